# K3 on the fp64 tensor cores (DMMA) vs the FMA pipe: parity subset + timings of both
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "global_solve or c3s or c5s or c2s or c1 or determin" 2>&1 | tail -4
rm -f gpurun_out/devrun_mma.log
for mma in 1 0; do
for a in "c5 --horizon 2 --set accel_fwd=1 --set outer_warm=1" "c3 --horizon 3 --set accel_fwd=1" "c4 --horizon 20 --set accel_fwd=1 --set outer_warm=1"; do
  echo "PD_K3_MMA=$mma $a" >> gpurun_out/devrun_mma.log
  PD_K3_MMA=$mma timeout 200 python tools/devrun.py $a >> gpurun_out/devrun_mma.log 2>&1
done
done
python - <<'PY'
import json
for l in open("gpurun_out/devrun_mma.log"):
    if not l.startswith("{"): print(l.strip()[:300]); continue
    d = json.loads(l); p = d["prof_all"]
    per = {k: round(1e3 * v[0] / max(v[1], 1), 1) for k, v in p.items() if v[1]}
    print(d["config"], "fwd", d["fwd_s"], "bwd", d["bwd_s"], "its", d["iters_fwd"]["mean"], d["iters_adj"]["mean"], "us/launch", per)
PY
