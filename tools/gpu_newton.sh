# Newton-PCG forward (accel_fwd = 2): parity tests, then the PD vs Newton comparison on c3 / c5 (short horizons)
mkdir -p gpurun_out
T=${1:-nt}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "2-1 or accel_fwd2 or c3s_batched_shared_factor_parity" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/${T}_pytest.log
for C in c3 c5; do
for S in pd newton; do
timeout 900 python bench.py --config $C --solver $S --horizon 10 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 > gpurun_out/${T}_${C}_${S}.json 2> gpurun_out/${T}_${C}_${S}.err; echo "$C $S rc=$?"
python -c "import json,sys; d=json.loads(open('gpurun_out/${T}_${C}_${S}.json').read().strip().splitlines()[-1]); print('$C $S', round(d['value']/1e6,3), 'M', d['ms_per_step'], d['iters'], d['kernel_share'])" 2>&1 | tail -1
done; done
