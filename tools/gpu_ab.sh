# A/B timing of library variants: bash tools/gpu_ab.sh "A B C" "3 1 2"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in $1; do for c in $2; do
RAID6C_LIB=$PWD/build/var/lib$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline ${3:-} > gpurun_out/ab_${v}_c$c.log 2>&1
python - <<PY
import json
l=[x for x in open('gpurun_out/ab_${v}_c$c.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v c$c', d and {k:(v['achieved_GBps'],v['frac_of_peak']) for k,v in d['kernels'].items()}, d and d['verified']['mismatched_bytes'])
PY
done; done
