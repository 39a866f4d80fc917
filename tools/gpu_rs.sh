cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# paper's comparison: Z_17 (16-bit words) vs RS at N = 16, plus the c2 workload (N = 12) and c4 (N = 58)
for spec in "2 16 zp 17" "2 16 rs 17" "2 12 zp 13" "2 12 rs 13" "4 58 rs 59" "5 60 rs 61"; do set -- $spec
extra=""; [ "$4" = "17" ] && extra="--prime 17"
timeout 600 python bench.py --config $1 --data-strips $2 --code $3 $extra --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/rs_$1_$2_$3_$4.log 2>&1; echo "c$1 N=$2 $3 p=$4 rc=$?"
grep '^{' gpurun_out/rs_$1_$2_$3_$4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k:(v['achieved_GBps'],v['frac_of_peak'],v['avg_ms']) for k,v in d['kernels'].items()}, d['verified'])"
done
