# generic kernel, larger groups: 128 threads x 3 CTAs (tree) vs 256 threads x 2 CTAs (W256)
cd $GRAFT_REPO_ROOT
O=gpurun_out/gen4; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "generic_prime" > $O/pytest_T.log 2>&1; echo "pytest T rc=$?"; tail -1 $O/pytest_T.log
RAID6C_LIB=$(lib W256) timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "generic_prime" > $O/pytest_W.log 2>&1; echo "pytest W rc=$?"; tail -1 $O/pytest_W.log
B="--no-e2e --no-cpu-baseline --steps 5 --warmup 3"
for p in 67 127 131 139 163 197 211 251; do for v in T W256; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 2 --prime $p $B > $O/p${p}_$v.json 2>&1
done; done
python tools/ab_table.py $O/p*.json
