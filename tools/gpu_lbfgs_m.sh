# L-BFGS memory sweep (developer probe): c5 / c3 throughput and iteration counts at a 20-step horizon per PD_LBFGS_M
mkdir -p gpurun_out
for cfg in c5 c3; do for m in 8 3 4 5 6; do
  echo -n "$cfg m=$m "
  PD_LBFGS_M=$m timeout 600 python bench.py --config $cfg --horizon 20 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3fM' % (d['value']/1e6), d['iters'], 'K3 %.1f us' % (d['roofline_k3']['avg_launch_ms']*1e3))"
done; done
