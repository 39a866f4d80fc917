cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for op in update scrub; do for c in 2 1 3 4 5; do timeout 300 python bench.py --op $op --config $c --steps 10 --warmup 3 > gpurun_out/next1_${op}_c$c.log 2>&1; echo "$op c$c rc=$?"; grep '^{' gpurun_out/next1_${op}_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['verified'])"; done; done
