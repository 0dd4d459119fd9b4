# per-launch times of the K3 kernels in one c5 time step (ncu launch list, cold cache, serialised)
mkdir -p gpurun_out
CMD="python bench.py --config c5 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 600 $CMD > gpurun_out/k3l_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sweep|contact_fix" -c 400 --csv --log-file gpurun_out/k3_launches${1}.csv $CMD > gpurun_out/k3l_ncu.log 2>&1
echo "rc=$?"
