# c3 K3 warp-count probe: A^-1 time per PD_K3_WARPS (the level launch's warp split; default 148 x 8)
for w in 1184 592 296 144 72; do PD_K3_WARPS=$w timeout 300 python tools/k3_time_probe.py c3 /tmp/k3ref_c3.pt 2>&1 | tail -1; done
for w in 1184 144; do echo -n "c3 bench warps=$w "; PD_K3_WARPS=$w timeout 600 python bench.py --config c3 --horizon 20 --steps 1 --warmup 3 --no-e2e --cpu-sample-steps 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3fM' % (d['value']/1e6), d['iters'], 'K3 %.1f us' % (d['roofline_k3']['avg_launch_ms']*1e3))"; done
