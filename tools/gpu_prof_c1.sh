cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python tools/prof_configs.py 1"
timeout 600 $P > gpurun_out/prof_c1_plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:zp_kernel -s 2 -c 2 -o gpurun_out/prof_c1 $P > gpurun_out/prof_c1_ncu.log 2>&1; echo "ncu=$?"
tail -3 gpurun_out/prof_c1_ncu.log
