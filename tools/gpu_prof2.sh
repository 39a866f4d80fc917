cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python tools/prof_configs.py 1 3 4 5"
timeout 600 $P > gpurun_out/prof2_plain.log 2>&1 && timeout 2400 ncu --set full --clock-control none --import-source on -k regex:zp_kernel -c 16 -o gpurun_out/prof_cfgs $P > gpurun_out/prof2_ncu.log 2>&1; echo "ncu=$?"
tail -3 gpurun_out/prof2_ncu.log
