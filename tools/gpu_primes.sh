# Per-prime c2-shaped throughput (N = 12, 4 MiB strips, 256 stripes) for library variants:
#   bash tools/gpu_primes.sh "gen main" "23 31 41"      (build/var/lib<variant>.so; "main" = the in-tree library)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for p in $2; do for v in $1; do
L=$PWD/build/var/lib$v.so; [ "$v" = main ] && L=$PWD/paper_cs_0611109_b200/libraid6c.so
RAID6C_LIB=$L timeout 300 python bench.py --config 2 --prime $p --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ${3:-} > gpurun_out/pr_${v}_p$p.log 2>&1
python - <<PY
import json
l=[x for x in open('gpurun_out/pr_${v}_p$p.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('p=$p $v', d and {k:(v['achieved_GBps'],v['frac_of_peak']) for k,v in d['kernels'].items()}, d and d['verified'])
PY
done; done
