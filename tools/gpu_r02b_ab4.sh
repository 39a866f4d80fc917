# A/B: p = 5 recovery with the per-item fold walk (F) vs the generic row loop (T)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab4; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
RAID6C_LIB=$(lib F) timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "5 and (recover_single or batch_encode or config1 or race or dd_solve or partial_last)" > $O/pytest_F.log 2>&1; echo "pytest F rc=$?"; tail -1 $O/pytest_F.log
B="--no-e2e --no-cpu-baseline --steps 20 --warmup 3"
for rep in 1 2 3; do for v in T F; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 1 $B > $O/c1_${v}_$rep.json 2>&1
done; done
python tools/ab_table.py $O/c1_*.json
