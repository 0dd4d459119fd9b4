mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "global_solve or c3s or c5s or c2s or c4s or c1 or determin" 2>&1 | tail -3
for w in 0 1; do
  timeout 300 python tools/devrun.py c5 --horizon 4 --set accel_fwd=1 --set outer_warm=1 --set lbfgs_warm=$w 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('lbfgs_warm=$w', 'fwd', d['fwd_s'], 'bwd', d['bwd_s'], 'its', d['iters_fwd'], d['outer'], d['nonconv'])
    else: print(l.strip()[:200])"
  timeout 300 python tools/devrun.py c4 --horizon 40 --set accel_fwd=1 --set outer_warm=1 --set lbfgs_warm=$w 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('c4 lbfgs_warm=$w', 'fwd', d['fwd_s'], 'its', d['iters_fwd'], d['outer'], d['nonconv'])"
done
for nb in 2 3 4; do
  PD_K3_NBUF=$nb timeout 300 python tools/timeline.py c5 --horizon 1 > gpurun_out/tl_c5_nb$nb.txt 2>&1
  echo "nbuf=$nb"; head -5 gpurun_out/tl_c5_nb$nb.txt | grep -E "span|sweep"
done
