for m in 8 12 16; do
  for cfg in "c5 --horizon 3" "c3 --horizon 3"; do
    PD_LBFGS_M=$m timeout 300 python tools/devrun.py $cfg --set accel_fwd=1 --set outer_warm=1 --reps 2 2>&1 | python -c "
import json,sys
ls=[l for l in sys.stdin if l.startswith('{')]
d=json.loads(ls[-1]); print('m=$m', d['config'], 'fwd', d['fwd_s'], 'bwd', d['bwd_s'], 'its', d['iters_fwd'], d['nonconv'])"
  done
done
