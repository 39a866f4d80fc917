# A/B of library variants on NEXT-4 emulation: bash tools/gpu_ab_x.sh "A B" "1:4 2:8"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in $1; do for cg in $2; do c=${cg%%:*}; g=${cg##*:}
RAID6C_LIB=$PWD/build/var/lib$v.so timeout 300 python bench.py --config $c --xgpu $g --steps 10 --warmup 3 > gpurun_out/abx_${v}_c${c}_G$g.log 2>&1
python - <<PY
import json
l=[x for x in open('gpurun_out/abx_${v}_c${c}_G$g.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v c$c G$g', d and {k:v['frac_of_peak'] for k,v in d['kernels'].items()}, d and d['verified'])
PY
done; done
