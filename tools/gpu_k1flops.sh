mkdir -p gpurun_out
T=${1:-kf}
timeout 900 python bench.py --config c5 --horizon 10 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err; echo "c5 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/${T}_c5.json').read().strip().splitlines()[-1]); print(d['roofline_k1'])"
timeout 900 python bench.py --config c3 --horizon 10 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 > gpurun_out/${T}_c3.json 2> gpurun_out/${T}_c3.err; echo "c3 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/${T}_c3.json').read().strip().splitlines()[-1]); print(d['roofline_k1'])"
