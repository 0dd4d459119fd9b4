# H0 scaling and fused-pass A/B (developer probe): throughput and iterations at a 20-step horizon, c5 and c3
run() {  # <label> <config> [ENV=...]
  echo -n "$1 $2 "
  env "${@:3}" timeout 600 python bench.py --config $2 --horizon 20 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3fM' % (d['value']/1e6), d['iters'], 'K3 %.1f us' % (d['roofline_k3']['avg_launch_ms']*1e3))"
}
for cfg in c5 c3; do
  run base $cfg X=0
  run gamma $cfg PD_LBFGS_GAMMA=1
  run nofuse $cfg PD_FUSE=0
  run base $cfg X=0
  run gamma $cfg PD_LBFGS_GAMMA=1
done
