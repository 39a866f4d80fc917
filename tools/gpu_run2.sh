cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-budget 5 > gpurun_out/bench_c$c.log 2>&1; echo "c$c=$?"; done
for sb in 65536 131072 262144 524288 1048576 2097152 4194304 8388608 16777216; do timeout 300 python bench.py --config 3 --strip-bytes $sb --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sweep_c3_$sb.log 2>&1; echo "sweep $sb=$?"; done
timeout 600 $B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu=$?"
