# K4 (k_elem_AN_cached) and the backward gather: duration, DRAM bytes and full metrics on c5 (one time step)
mkdir -p gpurun_out
T=${1:-k4}
CMD="python bench.py --config c5 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_elem_AN_cached|k_elem_jac" -c 4 -o gpurun_out/${T}_full $CMD > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
