# Active-set warm start probe (PD_ACTIVE_WARM=1, not Alg. 1 as printed, off by default): agreement with the default
# path on the contact configs, then c5 throughput at a 20-step horizon
timeout 900 python tools/active_warm_probe.py c5s c4s c4
for p in 0 1 0 1; do
  echo -n "c5 PD_ACTIVE_WARM=$p "
  PD_ACTIVE_WARM=$p timeout 600 python bench.py --config c5 --horizon 20 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3fM' % (d['value']/1e6), d['iters'], 'K3 %.1f us' % (d['roofline_k3']['avg_launch_ms']*1e3))"
done
