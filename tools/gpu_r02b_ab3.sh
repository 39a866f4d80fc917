# A/B: half mask table for p = 233 (T = tree) vs the previous build (B)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab3; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next1.py tests/test_gpu_next2.py tests/test_gpu_xgpu.py -q -k "233 or rotation_unit or dd_solve" > $O/pytest_T.log 2>&1; echo "pytest T rc=$?"; tail -1 $O/pytest_T.log
B="--no-e2e --no-cpu-baseline --steps 10 --warmup 3"
for rep in 1 2; do for v in T B; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 2 --prime 233 $B > $O/p233_${v}_$rep.json 2>&1
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 2 --prime 233 --op update > $O/upd233_${v}_$rep.json 2>&1
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 2 $B > $O/c2_${v}_$rep.json 2>&1
done; done
python tools/ab_table.py $O/p233_*.json $O/c2_*.json
for f in $O/upd233_*.json; do echo "$f $(grep '^{' $f | cut -c1-250)"; done
