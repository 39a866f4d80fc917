# NEXT-4 over the self-launched multi-rank path (2 ranks sharing cuda:0 under gloo) + c3 sweep
cd $GRAFT_REPO_ROOT
O=gpurun_out/x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > $O/pytest_multirank.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_multirank.log
timeout 600 python bench.py --gpus 2 --dist-backend gloo --xgpu 2 --config 2 --stripes 16 --oracle-stripes 4 > $O/xgpu2_gloo.log 2>&1; echo "xgpu2 rc=$?"; grep '^{' $O/xgpu2_gloo.log | tail -1 | cut -c1-400
timeout 1500 python bench.py --config 3 --sweep > $O/sweep_c3.log 2>&1; echo "sweep rc=$?"; tail -c 1500 $O/sweep_c3.log
