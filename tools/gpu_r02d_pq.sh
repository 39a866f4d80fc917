# PQ-only recovery on the encode kernel: parity tests, config 2 as written (per class), config 1 literally
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02d_pq; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next2.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 900 python bench.py --config 2 --full --steps 5 > $O/full_c2.log 2>&1; echo "full_c2 rc=$?"
timeout 300 python bench.py --config 1 --full --steps 5 > $O/c1_literal.log 2>&1; echo "c1_literal rc=$?"
grep '^{' $O/full_c2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:v for k,v in d.items() if k in ('value','per_class','classes','verified')})" 2>&1 | cut -c1-1500
grep '^{' $O/c1_literal.log | tail -1 | cut -c1-1200
