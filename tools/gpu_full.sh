# Whole-config runs (c2/c4/c5 --full, strong-scaling shape at 1 GPU) and the c3 strip sweep.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
for c in 4 5 2; do
  timeout 900 python bench.py --config $c --full > gpurun_out/${TAG}_full_c$c.log 2>&1; echo "full c$c=$?"
  tail -1 gpurun_out/${TAG}_full_c$c.log | cut -c1-400
done
timeout 1200 python bench.py --config 3 --sweep > gpurun_out/${TAG}_sweep_c3.log 2>&1; echo "sweep=$?"
tail -1 gpurun_out/${TAG}_sweep_c3.log | cut -c1-300
