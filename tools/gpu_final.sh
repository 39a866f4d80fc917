cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.log 2>&1; echo "bench=$?"
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
F="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
timeout 600 $F > gpurun_out/plain_full.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:zp_kernel -s 2 -c 2 -o gpurun_out/${TAG}_prof_c2 $F > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
