# full round check: GPU tests, smoke, devrun timings, benches + launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
bash tools/gpu_quick.sh
bash tools/gpu_round2.sh
