# A/B: T = tree (idle warps skip the partial tile), W = + per-warp output staging/stores, H = neither
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab1; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q > $O/pytest_T.log 2>&1; echo "pytest T rc=$?"; tail -1 $O/pytest_T.log
RAID6C_LIB=$(lib W) timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q > $O/pytest_W.log 2>&1; echo "pytest W rc=$?"; tail -1 $O/pytest_W.log
B="--no-e2e --no-cpu-baseline --steps 10 --warmup 3"
for rep in 1 2; do for v in T W H; do for c in 1 2 4 5; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config $c $B > $O/c${c}_${v}_$rep.json 2>&1
  sleep 2
done; done; done
python tools/ab_table.py $O/c*.json
