# Round check (run under gpurun): all GPU tests, smoke, the c5 headline bench line.
# Usage: bash tools/gpu_check.sh <tag> [pytest -k expr]
T=${1:-chk}
K=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_smi.txt 2>&1
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
else
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
tail -n 25 gpurun_out/${T}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/${T}_smoke.log
timeout 1500 python bench.py --steps 2 --warmup 3 > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err; echo "bench c5 rc=$?"
tail -c 2500 gpurun_out/${T}_bench_c5.json
