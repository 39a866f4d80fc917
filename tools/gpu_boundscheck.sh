# Run the GPU test-suite, the smoke test and whole-config benches against the bounds-checked
# build (device asserts on every TMA row load / bulk store; stand-in for compute-sanitizer).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export RAID6C_LIB=$PWD/build/var/libCHK.so
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/chk_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/chk_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; echo "smoke=$?"
for c in 4 5; do timeout 900 python bench.py --config $c --full --warmup 3 > gpurun_out/chk_full_c$c.log 2>&1; echo "full c$c=$?"; done
for c in 1 2 3; do timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/chk_c$c.log 2>&1; echo "c$c=$?"; done
timeout 600 python bench.py --config 4 --xgpu 8 > gpurun_out/chk_xgpu.log 2>&1; echo "xgpu=$?"
grep -l "Assertion\|assert" gpurun_out/chk_*.log || echo "no device assertion fired"
