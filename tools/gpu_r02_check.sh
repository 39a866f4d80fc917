set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
timeout 600 python bench.py --steps 30 --warmup 5 --dump-steps > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc=$?" >> gpurun_out/g1_bench.err
timeout 900 python bench.py --full --config 2 --steps 5 --warmup 3 > gpurun_out/g1_c2lit.json 2> gpurun_out/g1_c2lit.err; echo "c2lit rc=$?" >> gpurun_out/g1_c2lit.err
