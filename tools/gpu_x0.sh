for p in 0 1; do
  for cfg in "c5 --horizon 3" "c3 --horizon 3" "c4 --horizon 20"; do
    timeout 300 python tools/devrun.py $cfg --set accel_fwd=1 --set outer_warm=1 --set x0_predict=$p --reps 2 2>&1 | python -c "
import json,sys
ls=[l for l in sys.stdin if l.startswith('{')]
d=json.loads(ls[-1]) if ls else None
print('x0_predict=$p', d and d['config'], d and ('fwd', d['fwd_s'], 'bwd', d['bwd_s'], 'its', d['iters_fwd'], d['outer'], d['nonconv']))"
  done
done
