# round-2 A/B of recovery-kernel variants: V0 = build/var/libB.so (round-1 kernel), V1 = the tree's
# library, V2 = build/var/libV2.so; bash tools/gpu_r02_ab2.sh
cd $GRAFT_REPO_ROOT
O=gpurun_out/g3; mkdir -p $O
nvidia-smi -q -d POWER,CLOCK > $O/smi_power.txt 2>&1
lib() { case $1 in V1) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; V0) echo $PWD/build/var/libB.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
RAID6C_LIB=$(lib V2) timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py -m gpu -x -q > $O/pytest_V2.log 2>&1; echo "pytest rc=$?" >> $O/pytest_V2.log
B="--no-e2e --no-cpu-baseline"
for rep in 1 2; do for v in V0 V1 V2; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --steps 8 --warmup 3 --dump-steps $B > $O/short_${v}_$rep.json 2>$O/short_${v}_$rep.err
  sleep 8
done; done
for v in V0 V1 V2; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --steps 200 --warmup 5 --dump-steps $B > $O/long_${v}.json 2>$O/long_${v}.err
  sleep 15
  for c in 1 4 5; do
    RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config $c --steps 10 --warmup 3 --dump-steps $B > $O/c${c}_${v}.json 2>$O/c${c}_${v}.err
    sleep 5
  done
done
