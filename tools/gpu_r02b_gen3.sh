# generic kernel, small groups (GB <= 56 B): 128 (tree) vs 192 vs 256 consumer threads per CTA
cd $GRAFT_REPO_ROOT
O=gpurun_out/gen3; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
for v in N192 N256; do
  RAID6C_LIB=$(lib $v) timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "generic_prime" > $O/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 $O/pytest_$v.log
done
B="--no-e2e --no-cpu-baseline --steps 5 --warmup 3"
for p in 67 71 79 83 103 107; do for v in T N192 N256; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 2 --prime $p $B > $O/p${p}_$v.json 2>&1
done; done
python tools/ab_table.py $O/p*.json
