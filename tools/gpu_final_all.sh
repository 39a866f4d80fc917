# Full measurement refresh on one B200 (final build of the round): every bench line is written to
# gpurun_out/final/<name>.json (the last JSON line of the run), logs next to it.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final
mkdir -p $O
run() {  # run NAME TIMEOUT ARGS...
  local name=$1 to=$2; shift 2
  timeout $to python bench.py "$@" > $O/$name.log 2>&1; local rc=$?
  grep '^{' $O/$name.log | tail -1 > $O/$name.json
  echo "$name rc=$rc $(cut -c1-160 $O/$name.json)"
}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
run bench_default 900
for c in 1 2 3 4 5; do run bench_c$c 600 --config $c --no-e2e --no-cpu-baseline; done
for c in 2 4 5; do run full_c$c 900 --config $c --full; done
run sweep_c3 1200 --config 3 --sweep
run c1_literal 300 --config 1 --full --steps 5
for op in update scrub; do for c in 1 2 3 4 5; do run next1_${op}_c$c 600 --config $c --op $op; done; done
for spec in "2 25" "2 17" "4 115" "5 121" "3 300" "1 9"; do set -- $spec; run next2_c$1_N$2 600 --config $1 --data-strips $2 --no-e2e --no-cpu-baseline; done
for spec in "2 16 zp --prime 17" "2 16 rs --prime 17" "2 12 zp" "2 12 rs" "4 58 zp" "4 58 rs" "5 60 zp" "5 60 rs"; do set -- $spec
  run next3_c$1_N$2_$3${4:+_p17} 600 --config $1 --data-strips $2 --code $3 $4 $5 --no-e2e --no-cpu-baseline; done
for spec in "4 8" "5 8" "2 4" "2 8" "1 4" "3 8"; do set -- $spec; run next4_xgpu_c$1_G$2 600 --config $1 --xgpu $2; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 \
  bench.py --gpus 2 --xgpu 2 --dist-backend gloo --config 2 --stripes 32 > $O/next4_xgpu_ipc2.log 2>&1; echo "ipc2 rc=$?"
grep '^{' $O/next4_xgpu_ipc2.log | tail -1 > $O/next4_xgpu_ipc2.json
run impl_reference 600 --impl reference
# ncu: launch list of the default workload (2 timed steps) and a full-set capture of its encode + recover
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > $O/ncu_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c2.csv $B > $O/ncu_launch.log 2>&1; echo "ncu_launch=$?"
F="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
timeout 600 $F > $O/ncu_plain_full.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:zp_kernel -s 6 -c 2 -o $O/prof_c2 $F > $O/ncu_full.log 2>&1; echo "ncu_full=$?"
