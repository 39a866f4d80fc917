# partial last TMA tile (c1): T = tree library; NPT = slim variant without it
cd $GRAFT_REPO_ROOT
O=gpurun_out/g8; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; V0) echo $PWD/build/var/libB.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
B="--no-e2e --no-cpu-baseline"
for rep in 1 2 3; do for v in T NPT V0; do for c in 1; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config $c --steps 10 --warmup 3 $B > $O/c${c}_${v}_$rep.json 2>$O/c${c}_${v}_$rep.err
  sleep 3
done; done; done
for c in 2 4 5 3; do RAID6C_LIB=$(lib T) timeout 300 python bench.py --config $c --steps 10 --warmup 3 $B > $O/c${c}_T.json 2>$O/c${c}_T.err; done
RAID6C_LIB=$(lib T) timeout 300 python bench.py --config 1 --full --steps 5 > $O/c1lit_T.json 2>&1
timeout 1200 python bench.py --config 3 --sweep --steps 5 --warmup 3 > $O/sweep_c3.json 2>$O/sweep_c3.err; echo "sweep rc=$?" >> $O/sweep_c3.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zp_kernel -s 6 -c 2 -o $O/prof_c1 python bench.py --config 1 --steps 1 --warmup 3 $B --no-verify > $O/ncu_c1.log 2>&1; echo "ncu rc=$?" >> $O/ncu_c1.log
