# ncu --set full of the NEXT-4 partial and combine kernels (c4 layout, 8 emulated ranks) and of
# the c1 encode (8 KiB-tile geometry).  Each command first runs once without ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
X="python bench.py --config 4 --xgpu 8 --steps 1 --warmup 3"
timeout 600 $X > gpurun_out/prof_x_plain.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:zp_kernel<\(int\)59, \(int\)[45]" -s 7 -c 2 -o gpurun_out/prof_next4 $X > gpurun_out/prof_next4_ncu.log 2>&1; echo "ncu next4=$?"
exit 0
P="python tools/prof_configs.py 1"
timeout 600 $P > gpurun_out/prof_c1b_plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:zp_kernel -s 2 -c 2 -o gpurun_out/prof_c1b $P > gpurun_out/prof_c1b_ncu.log 2>&1; echo "ncu c1=$?"
tail -n 2 gpurun_out/prof_next4_ncu.log
