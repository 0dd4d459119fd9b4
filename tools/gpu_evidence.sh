# round evidence: ncu launch lists (per-kernel time + DRAM bytes) of the c3/c5 bench workloads (1 time step),
# traffic json, full captures of the K3 level kernel and K1, then the c3 and c5 bench lines
mkdir -p gpurun_out profiles
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CMD3="python bench.py --config c3 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 300 $CMD3 > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c3_h1.csv $CMD3 > gpurun_out/ncu_c3.log 2>&1
echo "c3 launch list rc=$?"
CMD5="python bench.py --config c5 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 600 $CMD5 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5_h1.csv $CMD5 > gpurun_out/ncu_c5.log 2>&1
echo "c5 launch list rc=$?"
python tools/ncu_traffic.py c3 gpurun_out/launches_c3_h1.csv profiles/ncu_traffic.json
python tools/ncu_traffic.py c5 gpurun_out/launches_c5_h1.csv profiles/ncu_traffic.json
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep_level|k_elem_residual|k_sweep_reduce" -c 5 -o gpurun_out/prof_c5_full $CMD5 > gpurun_out/ncu_c5_full.log 2>&1
echo "c5 full rc=$?"
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?"
timeout 1200 python bench.py --config c5 --steps 1 --warmup 3 --cpu-sample-steps 0 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench_c3.json", "gpurun_out/bench_c5.json"):
    try:
        d = json.load(open(f))
        print(f, "value %.4g" % d["value"], "ms/step %.0f" % d["ms_per_step"], "e2e %.4g" % d["e2e"]["value"],
              "K3 %.3f ms frac %.3f traffic %s" % (d["roofline_k3"]["avg_launch_ms"], d["roofline_k3"]["frac"], d["roofline_k3"]["traffic"]),
              "K1 frac %.3f" % d["roofline_k1"]["frac"], d["kernel_share"], d["iters"], d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
