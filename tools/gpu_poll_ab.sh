# Iteration-control A/B (developer probe): throughput at a 20-step horizon with the polled host flag (default) vs
# the D2H copy + stream synchronisation of rounds 1-2c (PD_POLL=0), c5 and c3, plus the device timelines
for cfg in c5 c3; do for p in 0 1 0 1; do
  echo -n "$cfg PD_POLL=$p "
  PD_POLL=$p timeout 600 python bench.py --config $cfg --horizon 20 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3fM' % (d['value']/1e6), d['iters'], d['kernel_share'], 'K3 %.1f us' % (d['roofline_k3']['avg_launch_ms']*1e3))"
done; done
for cfg in c5 c3; do for p in 0 1; do
  echo "== timeline $cfg PD_POLL=$p"
  PD_POLL=$p timeout 600 python tools/timeline.py $cfg --horizon 2 --top 6 2>&1 | head -30
done; done
