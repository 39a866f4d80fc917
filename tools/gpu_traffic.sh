# DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per launch of the timed step's kernels
# of `bench.py --config K --steps 1` for every config (the bench's own launch, not a smaller batch).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/traffic
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for spec in "1 6 2" "2 6 2" "3 3 1" "4 6 2" "5 4 1"; do set -- $spec
  B="python bench.py --config $1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
  timeout 600 $B > gpurun_out/traffic/plain_c$1.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:zp_kernel -s $2 -c $3 --csv --log-file gpurun_out/traffic/c$1.csv $B > gpurun_out/traffic/ncu_c$1.log 2>&1
  echo "c$1 rc=$?"
done
