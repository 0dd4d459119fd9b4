# ncu --set full of the first K3 v4 level kernels and reduce of a c5 time step (after warm-up)
mkdir -p gpurun_out
CMD="python bench.py --config c5 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_warp|k_sweep_reduce4" -s 200 -c 6 -o gpurun_out/k3v4_full $CMD > gpurun_out/k3v4_full.log 2>&1
echo "rc=$?"
