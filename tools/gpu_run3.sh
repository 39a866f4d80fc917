cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench=$?"
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-budget 5 > gpurun_out/bench_c$c.log 2>&1; echo "c$c=$?"; done
