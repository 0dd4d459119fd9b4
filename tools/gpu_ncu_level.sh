CMD="python tools/devrun.py c5 --horizon 1 --set max_iter_fwd=2 --set max_iter_adj=1"
timeout 200 $CMD > gpurun_out/plain_c5b.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_level -s 13 -c 14 -o gpurun_out/prof_level $CMD > gpurun_out/ncu_level.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_level.log
