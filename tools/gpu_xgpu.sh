# NEXT-4 measurements: emulated cross-GPU layout on one B200, plus the 2-process IPC rehearsal.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
for spec in "4 8" "2 4" "2 8" "5 8" "3 8" "1 4"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --xgpu $2 > gpurun_out/${TAG}_xgpu_c$1_G$2.log 2>&1; echo "xgpu c$1 G$2 rc=$?"
  tail -1 gpurun_out/${TAG}_xgpu_c$1_G$2.log | cut -c1-200
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --xgpu 2 --dist-backend gloo --config 2 --stripes 32 > gpurun_out/${TAG}_xgpu_ipc2.log 2>&1; echo "ipc2 rc=$?"
tail -1 gpurun_out/${TAG}_xgpu_ipc2.log | cut -c1-300
