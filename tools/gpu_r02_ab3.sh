# round-2 A/B: V0 = build/var/libB.so (round-1 kernel), M = the tree's library, NF = build/var/libNF.so
cd $GRAFT_REPO_ROOT
O=gpurun_out/g4; mkdir -p $O
lib() { case $1 in M) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; V0) echo $PWD/build/var/libB.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
B="--no-e2e --no-cpu-baseline"
for rep in 1 2; do for v in V0 M NF; do for c in 2 1 4 5; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config $c --steps 10 --warmup 3 --dump-steps $B > $O/c${c}_${v}_$rep.json 2>$O/c${c}_${v}_$rep.err
  sleep 4
done; done; done
for v in M NF M; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --steps 200 --warmup 5 --dump-steps $B > $O/long_${v}_$RANDOM.json 2>&1
  sleep 20
done
