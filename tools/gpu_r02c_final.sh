# Round-2 final measurement refresh on one B200: every bench line -> gpurun_out/r02c/<name>.json
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02c
mkdir -p $O
run() {  # run NAME TIMEOUT ARGS...
  local name=$1 to=$2; shift 2
  timeout $to python bench.py "$@" > $O/$name.log 2>&1; local rc=$?
  grep '^{' $O/$name.log | tail -1 > $O/$name.json
  echo "$name rc=$rc $(cut -c1-160 $O/$name.json)"
}
nvidia-smi -q -d POWER,CLOCK > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
run bench_default 900 --dump-steps
sleep 10
run bench_default_2 900 --steps 20 --warmup 5 --dump-steps --no-e2e
for c in 1 2 3 4 5; do sleep 5; run bench_c$c 600 --config $c --no-e2e --no-cpu-baseline --dump-steps; done
run full_c2 900 --config 2 --full --steps 5
run full_c4 1500 --config 4 --full
run full_c5 1800 --config 5 --full
run gpus2_gloo 900 --gpus 2 --dist-backend gloo --stripes 64 --no-e2e --oracle-stripes 8
run next4_xgpu_dist2_gloo 900 --gpus 2 --dist-backend gloo --xgpu 2 --config 2 --stripes 16 --oracle-stripes 4
run sweep_c3 1800 --config 3 --sweep
run c1_literal 300 --config 1 --full --steps 5
for op in update scrub; do for c in 1 2 3 4 5; do run next1_${op}_c$c 600 --config $c --op $op; done; done
for spec in "2 25" "2 17" "4 115" "5 121" "3 300" "1 9"; do set -- $spec; run next2_c$1_N$2 600 --config $1 --data-strips $2 --no-e2e --no-cpu-baseline; done
for spec in "4 8" "5 8" "2 4" "2 8" "1 4" "3 8"; do set -- $spec; run next4_xgpu_c$1_G$2 600 --config $1 --xgpu $2; done
for p in 233 127 251; do run prime_p$p 600 --config 2 --prime $p --no-e2e --no-cpu-baseline --steps 5; done
run impl_reference 600 --impl reference
# ncu: launch list of the default workload (2 timed steps) and full-set captures (c2, c1, generic p = 127)
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > $O/ncu_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c2.csv $B > $O/ncu_launch.log 2>&1; echo "ncu_launch=$?"
F="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:zp_kernel -s 6 -c 2 -o $O/prof_c2 $F > $O/ncu_full.log 2>&1; echo "ncu_full=$?"
F1="python bench.py --config 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:zp_kernel -s 6 -c 2 -o $O/prof_c1 $F1 > $O/ncu_full_c1.log 2>&1; echo "ncu_full_c1=$?"
FG="python bench.py --config 2 --prime 127 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:zp_generic -s 6 -c 2 -o $O/prof_g127 $FG > $O/ncu_full_g127.log 2>&1; echo "ncu_full_g127=$?"
mkdir -p $O/traffic
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for spec in "1 6 2" "2 6 2" "3 3 1" "4 6 2" "5 4 1"; do set -- $spec
  B="python bench.py --config $1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
  timeout 900 ncu --metrics $M --clock-control none -k regex:zp_kernel -s $2 -c $3 --csv --log-file $O/traffic/c$1.csv $B > $O/traffic/ncu_c$1.log 2>&1
  echo "traffic c$1 rc=$?"
done
