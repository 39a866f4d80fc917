cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=5 2>&1 | tail -9
for spec in "2 25" "2 17" "4 115" "5 121" "3 300" "1 9"; do set -- $spec
timeout 600 python bench.py --config $1 --data-strips $2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/next2_c$1_N$2.log 2>&1; echo "c$1 N=$2 rc=$?"
grep '^{' gpurun_out/next2_c$1_N$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k:(v['achieved_GBps'],v['frac_of_peak']) for k,v in d['kernels'].items()}, d['verified'])"
done
