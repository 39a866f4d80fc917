cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TOOL=${1:-memcheck}
T="python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k single_matches_oracle_or_recover_single_all_pairs_or_batch_encode_and_mixed_or_unaligned_or_lost_strips"
K="${2:-}"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "$K" > gpurun_out/san_plain.log 2>&1 && timeout 2400 compute-sanitizer --tool $TOOL --target-processes all python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "$K" > gpurun_out/san_$TOOL.log 2>&1; echo "sanitizer=$?"
tail -5 gpurun_out/san_$TOOL.log
