# Repeated A/B timing of library variants: bash tools/gpu_ab_rep.sh "A B C" "1 2" REPS [extra bench args]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
for rep in $(seq 1 ${3:-2}); do for c in $2; do for v in $1; do
RAID6C_LIB=$PWD/build/var/lib$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline ${4:-} > gpurun_out/ab/${v}_c${c}_$rep.log 2>&1
python - <<PY
import json
l=[x for x in open('gpurun_out/ab/${v}_c${c}_$rep.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v c$c rep$rep', d and {k:(v['avg_ms'],v['median_ms'],v['frac_of_peak']) for k,v in d['kernels'].items()}, d and d['verified']['ok'], d and d['clocks']['reasons'])
PY
done; done; done
