mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -k "not c5_full_batch_vs_oracle" -p no:cacheprovider > gpurun_out/r2_pytest1.log 2>&1
echo "pytest rc=$?"
tail -n 30 gpurun_out/r2_pytest1.log
timeout 1200 python bench.py --steps 2 --warmup 3 > gpurun_out/r2_bench_c5_a.json 2> gpurun_out/r2_bench_c5_a.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench_c5_a.json
