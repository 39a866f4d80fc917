# A/B of library variants on NEXT-1 ops: bash tools/gpu_ab_op.sh "A B" "1 2" "update scrub" [extra]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in $1; do for c in $2; do for op in $3; do
RAID6C_LIB=$PWD/build/var/lib$v.so timeout 300 python bench.py --config $c --op $op --steps 10 --warmup 3 ${4:-} > gpurun_out/abop_${v}_c${c}_$op.log 2>&1
python - <<PY
import json
l=[x for x in open('gpurun_out/abop_${v}_c${c}_$op.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v c$c $op', d and (d['roofline']['achieved'], d['roofline']['frac']), d and d['verified'])
PY
done; done; done
