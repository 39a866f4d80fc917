# A/B: double-buffered output staging (one CTA barrier per item).
#   S1 = one buffer (round-2 kernel), D4 = two buffers where >= 4 TMA stages remain (c1, p = 257
#   recovery), D3 = two buffers where >= 3 remain (also c2's p = 13 recovery); slim libraries.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_outb; mkdir -p $O
lib() { echo $PWD/build/var/lib$1.so; }
for v in D4 D3; do
  RAID6C_LIB=$(lib $v) timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not prime" > $O/pytest_$v.log 2>&1
  echo "pytest $v rc=$?"; tail -1 $O/pytest_$v.log
done
B="--no-e2e --no-cpu-baseline --steps 10 --warmup 3"
for rep in 1 2; do for v in S1 D4 D3; do for c in 1 2 3 4 5; do
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config $c $B > $O/c${c}_${v}_$rep.json 2>&1
  sleep 2
done; done; done
python tools/ab_table.py $O/c*.json
