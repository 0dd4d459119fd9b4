# ncu evidence for profiles/: launch list of a short bench run (same workload, 1 time step) and full
# captures of the top kernels (K3 item kernel, K3 reduce, K1) on c3 and c5
CMD="python bench.py --config c3 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 300 $CMD > gpurun_out/plain_bench_h1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c3_h1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
CMD5="python tools/devrun.py c5 --horizon 1 --set max_iter_fwd=3 --set max_iter_adj=2"
timeout 200 $CMD5 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep_flow|k_elem_residual|k_sweep_reduce" -s 40 -c 6 -o gpurun_out/prof_c5_full $CMD5 > gpurun_out/ncu_c5_full.log 2>&1
echo "c5 full rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum --clock-control none -k regex:"k_sweep_flow|k_elem_residual|k_sweep_reduce|k_elem_AN|k_to_solve|k_from_solve|k_gather" -c 400 --csv --log-file gpurun_out/launches_c5.csv $CMD5 > gpurun_out/ncu_c5_launch.log 2>&1
echo "c5 launch rc=$?"
