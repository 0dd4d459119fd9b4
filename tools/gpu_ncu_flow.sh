# full ncu of the dataflow sweep kernels (c3 and c5), after a clean plain run of the same command
for cfg in c3 c5; do
CMD="python tools/devrun.py $cfg --horizon 1 --set max_iter_fwd=2 --set max_iter_adj=1"
timeout 200 $CMD > gpurun_out/plain_$cfg.log 2>&1 && \
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_sweep_flow -s 2 -c 2 -o gpurun_out/prof_flow_$cfg $CMD > gpurun_out/ncu_flow_$cfg.log 2>&1
echo "$cfg ncu rc=$?"
done
