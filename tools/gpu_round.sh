# round deliverables: full GPU tests, c3 bench (default), launch list + full ncu of the top kernel (c3 bench cmd)
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench rc=$?"; tail -c 4000 gpurun_out/bench_c3.json
