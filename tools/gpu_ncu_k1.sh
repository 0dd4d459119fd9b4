mkdir -p gpurun_out
CMD="python tools/devrun.py c5 --horizon 1 --set max_iter_fwd=2 --set max_iter_adj=2"
timeout 200 $CMD > gpurun_out/plain_c5k1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_elem_residual|k_elem_AN_cached|k_mdot_partial|k_gather" -c 6 -o gpurun_out/prof_k1 $CMD > gpurun_out/ncu_k1.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_k1.log
