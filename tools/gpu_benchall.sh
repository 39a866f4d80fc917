cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
for c in 2 1 3 4 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_c$c.log 2>&1; echo "c$c=$?"; python - <<PY
import json
l=[x for x in open('gpurun_out/bench_${TAG}_c$c.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('c$c', d and d['value'], d and {k:(v['achieved_GBps'],v['frac_of_peak']) for k,v in d['kernels'].items()}, d and d['verified'])
PY
done
