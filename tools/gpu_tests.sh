# GPU tests only (optional -k expression)
mkdir -p gpurun_out
T=${1:-t}
K=${2:-}
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
else
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
fi
tail -25 gpurun_out/${T}_pytest.log
