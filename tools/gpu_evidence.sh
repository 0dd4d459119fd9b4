# Round evidence (run under gpurun): GPU tests, the c5 (headline) and c3 bench lines, ncu launch lists (per-launch
# time + DRAM bytes of one c5 / c3 time step), full captures of the K3 level/reduce kernels and K1.
# Usage: bash tools/gpu_evidence.sh <tag>   (outputs gpurun_out/<tag>_*)
T=${1:-r2}
mkdir -p gpurun_out profiles
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then  # (SKIP_TESTS=1: the GPU test suite is run by a separate call, tools/gpu_tests.sh)
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/${T}_pytest_gpu.log
fi
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/${T}_smoke.log
timeout 1500 python bench.py --steps 2 --warmup 3 > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --config c3 --steps 2 --warmup 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err; echo "bench c3 rc=$?"
# the on-box Newton-PCG comparison system on the headline workload
timeout 1500 python bench.py --solver newton --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 > gpurun_out/${T}_bench_c5_newton.json 2> gpurun_out/${T}_bench_c5_newton.err; echo "bench c5 newton rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CMD5="python bench.py --config c5 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 600 $CMD5 > gpurun_out/${T}_plain_c5.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -c 3500 --csv --log-file gpurun_out/${T}_launches_c5_h1.csv $CMD5 > gpurun_out/${T}_ncu_c5.log 2>&1
echo "c5 launch list rc=$?"
CMD3="python bench.py --config c3 --horizon 1 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0"
timeout 300 $CMD3 > gpurun_out/${T}_plain_c3.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -c 6000 --csv --log-file gpurun_out/${T}_launches_c3_h1.csv $CMD3 > gpurun_out/${T}_ncu_c3.log 2>&1
echo "c3 launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep_warp|k_sweep_reduce4" -s 300 -c 6 -o gpurun_out/${T}_full_c5 $CMD5 > gpurun_out/${T}_ncu_full.log 2>&1
echo "c5 full (K3) rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_elem_residual|k_elem_AN_cached|k_gather" -s 4 -c 3 -o gpurun_out/${T}_full_c5_elem $CMD5 > gpurun_out/${T}_ncu_full_elem.log 2>&1
echo "c5 full (K1/K4/K2) rc=$?"
