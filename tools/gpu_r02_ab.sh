# round-2 A/B + profile call: bash tools/gpu_r02_ab.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/g2
O=gpurun_out/g2
B="--no-e2e --no-cpu-baseline"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for rep in 1 2; do for v in A B; do
  RAID6C_LIB=$([ $v = A ] && echo $PWD/paper_cs_0611109_b200/libraid6c.so || echo $PWD/build/var/lib$v.so) timeout 300 python bench.py --steps 8 --warmup 3 --dump-steps $B > $O/short_${v}_$rep.json 2>$O/short_${v}_$rep.err
  sleep 10
done; done
for v in A B; do
  RAID6C_LIB=$([ $v = A ] && echo $PWD/paper_cs_0611109_b200/libraid6c.so || echo $PWD/build/var/lib$v.so) timeout 300 python bench.py --steps 200 --warmup 5 --dump-steps $B > $O/long_${v}.json 2>$O/long_${v}.err
  sleep 20
  for c in 1 4 5; do
    RAID6C_LIB=$([ $v = A ] && echo $PWD/paper_cs_0611109_b200/libraid6c.so || echo $PWD/build/var/lib$v.so) timeout 300 python bench.py --config $c --steps 10 --warmup 3 --dump-steps $B > $O/c${c}_${v}.json 2>$O/c${c}_${v}.err
    sleep 5
  done
done
RAID6C_LIB=$PWD/build/var/libNOOP.so timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --oracle-stripes 4 > $O/noop.json 2> $O/noop.err; echo "noop rc=$?" >> $O/noop.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zp_kernel -s 7 -c 1 -o $O/rec_c2 python bench.py --steps 1 --warmup 3 $B --no-verify > $O/ncu_c2.log 2>&1; echo "ncu rc=$?" >> $O/ncu_c2.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zp_kernel -s 2 -c 2 -o $O/prof_c1 python tools/prof_configs.py 1 > $O/ncu_c1.log 2>&1; echo "ncu rc=$?" >> $O/ncu_c1.log
