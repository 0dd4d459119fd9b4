import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2101_05917_b200 as pdb
from pd_inputs import get_config, make_inputs
inp = make_inputs(get_config("c5"), steps=1)
sim = pdb.simulator_from_inputs(inp, max_steps=1)
B, N = inp["B"], 3 * inp["n_nodes"]
r = torch.randn(B, N, dtype=torch.float64, device="cuda"); o = torch.zeros_like(r)
for _ in range(3): sim.apply_Ainv(r, o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): sim.apply_Ainv(r, o)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("PD_K3_EXP", "0"), os.environ.get("PD_K3_V", "4"), "apply_Ainv %.1f us" % (e0.elapsed_time(e1) / 50 * 1e3))
