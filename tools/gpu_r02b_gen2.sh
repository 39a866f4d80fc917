# generic kernel: static-dispatch rotation (T) vs the first TMA version (G) vs the direct kernel (B)
cd $GRAFT_REPO_ROOT
O=gpurun_out/gen2; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_xgpu.py tests/test_gpu_next1.py tests/test_gpu_next2.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
B="--no-e2e --no-cpu-baseline --steps 5 --warmup 3"
for p in 67 83 103 127 163 211 251; do for v in T G; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 2 --prime $p $B > $O/p${p}_$v.json 2>&1
done; done
python tools/ab_table.py $O/p*.json
