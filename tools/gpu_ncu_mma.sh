mkdir -p gpurun_out
CMD="python tools/devrun.py c5 --horizon 1 --set max_iter_fwd=2 --set max_iter_adj=1"
timeout 200 $CMD > gpurun_out/plain_c5b.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sweep|k_to_solve|k_from_solve" -c 200 --csv --log-file gpurun_out/launches_c5_mma.csv $CMD > gpurun_out/ncu_c5l.log 2>&1
echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_level -c 13 -o gpurun_out/prof_level_mma $CMD > gpurun_out/ncu_level.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_level.log
