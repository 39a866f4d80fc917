# Light recovery kernel (launches without DD): GPU tests, then config 2 as written per class (A: BASE = previous build, B: new)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02d_light; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
for rep in 1 2; do
  RAID6C_LIB=$PWD/build/var/libBASE.so timeout 900 python bench.py --config 2 --full --steps 5 --no-cpu-baseline > $O/full_c2_BASE_$rep.log 2>&1; echo "BASE rc=$?"
  timeout 900 python bench.py --config 2 --full --steps 5 --no-cpu-baseline > $O/full_c2_NEW_$rep.log 2>&1; echo "NEW rc=$?"
done
timeout 300 python bench.py --config 1 --full --steps 5 > $O/c1_literal.log 2>&1; echo "c1_literal rc=$?"
for f in $O/full_c2_*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$f'.split('/')[-1], 'enc', k['encode']['frac_of_peak'], {c:(v['ms_per_launch'],v['frac_of_peak']) for c,v in k['recover_by_class'].items()}, 'value', d['value'], 'ok', d['verified']['ok'])"; done
grep '^{' $O/c1_literal.log | tail -1 | cut -c1-900
