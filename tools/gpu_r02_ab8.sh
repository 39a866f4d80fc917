# T = tree library (EXT fold walk, recovery partial tile in small launches only); H = previous build
cd $GRAFT_REPO_ROOT
O=gpurun_out/g9; mkdir -p $O
lib() { case $1 in T) echo $PWD/paper_cs_0611109_b200/libraid6c.so;; *) echo $PWD/build/var/lib$1.so;; esac; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
B="--no-e2e --no-cpu-baseline"
for rep in 1 2; do for v in T H; do
  for spec in "2 25" "2 17" "4 115" "5 121"; do set -- $spec
    RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config $1 --data-strips $2 --steps 10 --warmup 3 $B > $O/n2_c$1_N$2_${v}_$rep.json 2>&1
  done
  RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 1 --steps 10 --warmup 3 $B > $O/c1_${v}_$rep.json 2>&1
done; done
for v in T H; do RAID6C_LIB=$(lib $v) timeout 300 python bench.py --config 1 --full --steps 5 > $O/c1lit_$v.json 2>&1; done
