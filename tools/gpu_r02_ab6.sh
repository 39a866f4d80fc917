# round-2 A/B: E = tree library; P256 / P224 / T224 = slim variants (row pairing, 224 recovery threads)
cd $GRAFT_REPO_ROOT
O=gpurun_out/g7; mkdir -p $O
lib() { case $1 in E) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; V0) echo $PWD/build/var/libB.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
for v in P256 P224 T224; do
RAID6C_LIB=$(lib $v) timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -k "fullsize or long_run or c2 or config2 or config5 or config4" -m gpu -x -q > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
done
B="--no-e2e --no-cpu-baseline"
for rep in 1 2; do for v in E P256 P224 T224; do for c in 2 5 4; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config $c --steps 10 --warmup 3 $B > $O/c${c}_${v}_$rep.json 2>$O/c${c}_${v}_$rep.err
  sleep 3
done; done; done
for v in E P256 P224 T224; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --steps 200 --warmup 5 --dump-steps $B > $O/long_${v}.json 2>&1
  sleep 20
done
