CMD="python tools/devrun.py c5 --horizon 1 --set accel_fwd=1 --set max_iter_fwd=4 --set max_iter_adj=3"
timeout 200 $CMD > gpurun_out/plain_c5.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_sweep_items -s 20 -c 2 -o gpurun_out/prof_sweep2 $CMD > gpurun_out/ncu_sweep2.log 2>&1
echo "ncu rc=$?"
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
