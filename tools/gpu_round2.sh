timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench c3 rc=$?"
timeout 1200 python bench.py --config c5 --steps 1 --warmup 3 --cpu-sample-steps 0 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "bench c5 rc=$?"
CMD="python bench.py --config c3 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 300 $CMD > gpurun_out/plain_bench_h1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c3_h1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench_c3.json", "gpurun_out/bench_c5.json"):
    try:
        d = json.load(open(f))
        print(f, "value %.4g" % d["value"], "ms/step %.0f" % d["ms_per_step"], "e2e %.4g" % d["e2e"]["value"],
              "K3 %.3f ms frac %.3f" % (d["roofline_k3"]["avg_launch_ms"], d["roofline_k3"]["frac"]),
              "K1 frac %.3f" % d["roofline_k1"]["frac"], d["kernel_share"], d["iters"], d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
