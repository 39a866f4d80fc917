# round-2 A/B: M = tree library; NH, FL0, C12 = build/var variants (tools/build_variant.py); V0 = round-1
cd $GRAFT_REPO_ROOT
O=gpurun_out/g5; mkdir -p $O
lib() { case $1 in M) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; V0) echo $PWD/build/var/libB.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
RAID6C_LIB=$(lib C12) timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > $O/pytest_C12.log 2>&1; echo "rc=$?" >> $O/pytest_C12.log
B="--no-e2e --no-cpu-baseline"
for rep in 1 2; do for v in M NH FL0 C12 V0; do for c in 2 5 4 1; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config $c --steps 10 --warmup 3 $B > $O/c${c}_${v}_$rep.json 2>$O/c${c}_${v}_$rep.err
  sleep 3
done; done; done
for v in M C12; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --steps 200 --warmup 5 --dump-steps $B > $O/long_${v}.json 2>&1
  sleep 20
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zp_kernel -s 7 -c 1 -o $O/rec_c2 python bench.py --steps 1 --warmup 3 $B --no-verify > $O/ncu_c2.log 2>&1; echo "ncu rc=$?" >> $O/ncu_c2.log
