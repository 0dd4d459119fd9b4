# quick c5 K3 timing (+ optional K3 parity subset)
mkdir -p gpurun_out
if [ "$1" = "test" ]; then timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "global_solve or k3_switches or c5s_contact or bitwise" -p no:cacheprovider 2>&1 | tail -3; fi
timeout 900 python bench.py --steps 1 --warmup 3 --cpu-sample-steps 0 --e2e-steps 1 --horizon ${2:-20} > gpurun_out/quick_c5.json 2> gpurun_out/quick_c5.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/quick_c5.json"))
print("value %.4g" % d["value"], "ms/step %.0f" % d["ms_per_step"], "K3 %.4f ms frac %.3f" % (d["roofline_k3"]["avg_launch_ms"], d["roofline_k3"]["frac"]), "K1 %.4f ms" % d["roofline_k1"]["avg_launch_ms"], d["kernel_share"], d["iters"])
PY
