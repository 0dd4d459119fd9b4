set -x
CMD="python tools/devrun.py c5 --horizon 1 --set accel_fwd=1 --set max_iter_fwd=4 --set max_iter_adj=3"
timeout 200 $CMD > gpurun_out/plain_c5.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_c5.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_sweep_items -s 8 -c 2 -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_sweep.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_elem_residual -s 2 -c 1 -o gpurun_out/prof_k1 $CMD > gpurun_out/ncu_k1.log 2>&1
timeout 500 python -m pytest tests -m gpu -q 2>&1 | tail -5
tail -3 gpurun_out/ncu_c5.log gpurun_out/ncu_sweep.log gpurun_out/ncu_k1.log
