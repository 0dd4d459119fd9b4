# K3 v4 check on the GPU: parity suite (v4 default) + c5 bench, then v3 for comparison
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pytest_k3v4.log 2>&1
echo "pytest rc=$?"; tail -n 5 gpurun_out/r2_pytest_k3v4.log
timeout 900 python bench.py --steps 1 --warmup 3 --cpu-sample-steps 0 --e2e-steps 1 > gpurun_out/r2_bench_c5_v4.json 2> gpurun_out/r2_bench_c5_v4.err
echo "bench v4 rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2_bench_c5_v4.json"))
print("v4", "value %.4g" % d["value"], "ms/step %.0f" % d["ms_per_step"], "K3 %.3f ms frac %.3f" % (d["roofline_k3"]["avg_launch_ms"], d["roofline_k3"]["frac"]), d["kernel_share"], d["iters"])
PY
