# A/B of the p = 5 recovery geometry (config 1): T = 48 B x 224 (tree), G1 = 32 B x 256, G2 = 64 B x 128 (3 CTAs/SM), G3 = 64 B x 256
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab2; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
K="test_recover_single_all_pairs or test_batch_encode or test_config1_full or test_pipeline_race_stress or test_dd_solve_every_z or test_partial_last_tile or test_lost_strips"
for v in G1 G2 G3; do
  RAID6C_LIB=$(lib $v) timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "$K" > $O/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 $O/pytest_$v.log
done
B="--no-e2e --no-cpu-baseline --steps 20 --warmup 3"
for rep in 1 2 3; do for v in T G1 G2 G3; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 1 $B > $O/c1_${v}_$rep.json 2>&1
  sleep 1
done; done
for v in T G1 G2 G3; do RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 1 --full --steps 5 > $O/c1lit_$v.json 2>&1; done
python tools/ab_table.py $O/c1_*.json
for v in T G1 G2 G3; do echo "$v $(grep '^{' $O/c1lit_$v.json | cut -c1-200)"; done
