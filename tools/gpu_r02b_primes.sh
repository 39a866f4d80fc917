# Every odd prime <= 257 at the c2 shape (N = 12, 4 MiB x 256): encode + mixed recovery, oracle-sampled lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/primes; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_xgpu.py -q -x -k "generic or xgpu" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for p in 3 5 7 11 13 17 19 23 29 31 37 41 43 47 53 59 61 67 71 73 79 83 89 97 101 103 107 109 113 127 131 137 139 149 151 157 163 167 173 179 181 191 193 197 199 211 223 227 229 233 239 241 251 257; do
  timeout 300 python bench.py --config 2 --prime $p --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/p$p.log 2>&1
done
python - <<'PY'
import json, glob, os
out = {}
for f in sorted(glob.glob("gpurun_out/primes/p*.log"), key=lambda x: int(os.path.basename(x)[1:-4])):
    l = [x for x in open(f) if x.startswith("{")]
    p = int(os.path.basename(f)[1:-4])
    if not l:
        out[p] = None; continue
    d = json.loads(l[-1])
    out[p] = {"fast_path": d["fast_path"], **{k: {"GBps": v["achieved_GBps"], "frac": v["frac_of_peak"]} for k, v in d["kernels"].items()},
              "verified_ok": d["verified"]["ok"]}
json.dump(out, open("gpurun_out/primes/primes.json", "w"), indent=1)
for p, v in out.items():
    print(p, v and (v["fast_path"], v["encode"]["frac"], v["recover"]["frac"], v["verified_ok"]))
PY
