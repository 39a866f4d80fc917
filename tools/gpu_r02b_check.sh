# r02 (second session) sanity on one B200: GPU suite, smoke, default bench, c1 ncu with source
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02b
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 600 python bench.py --dump-steps > $O/bench_default.log 2>&1; echo "bench=$?"; grep '^{' $O/bench_default.log | tail -1 | cut -c1-300
timeout 300 python bench.py --config 1 --no-e2e --no-cpu-baseline --dump-steps > $O/bench_c1.log 2>&1; echo "c1=$?"; grep '^{' $O/bench_c1.log | tail -1 | cut -c1-300
F1="python bench.py --config 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zp_kernel -s 6 -c 2 -o $O/prof_c1 $F1 > $O/ncu_full_c1.log 2>&1; echo "ncu_full_c1=$?"
