# K1 (k_elem_residual) full capture with source counters on c5 (the forward's first launches)
mkdir -p gpurun_out
T=${1:-k1}
CMD="python bench.py --config c5 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_elem_residual" -s 2 -c 1 -o gpurun_out/${T}_full $CMD > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
