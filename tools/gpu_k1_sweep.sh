# K1 register/occupancy sweep on c5 (rebuilds the library per setting; timing only)
for mb in ${MBS:-5 4 3}; do
  PD_K1_MIN_BLOCKS=$mb python -c "import paper_2101_05917_b200.buildlib as b; b.build(force=True)" > /dev/null
  echo -n "K1_MIN_BLOCKS=$mb: "
  timeout 600 python bench.py --steps 1 --warmup 3 --cpu-sample-steps 0 --e2e-steps 1 --horizon 10 > gpurun_out/k1_$mb.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k1_$mb.json'))
print('value %.4g' % d['value'], 'K1 %.4f ms frac %.3f' % (d['roofline_k1']['avg_launch_ms'], d['roofline_k1']['frac']), 'K3 %.4f' % d['roofline_k3']['avg_launch_ms'], d['kernel_share'])"
done
