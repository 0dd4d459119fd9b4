mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?"
timeout 1200 python bench.py --config c5 --steps 1 --warmup 3 --cpu-sample-steps 0 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
python - <<'PY'
import json
for f in ("gpurun_out/bench_c3.json", "gpurun_out/bench_c5.json"):
    d = json.load(open(f))
    print(f, "value %.4g" % d["value"], "e2e %.4g" % d["e2e"]["value"], "K3 %.3f frac %.3f" % (d["roofline_k3"]["avg_launch_ms"], d["roofline_k3"]["frac"]), "K1 frac %.3f" % d["roofline_k1"]["frac"], d["clocks"])
PY
