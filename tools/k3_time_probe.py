"""Developer probe: average time of one c5 (or argv[1]) A^-1 application through the C-ABI, with the K3 switches
of the environment (PD_K3_*); the solution of a seeded right-hand side is saved (first run) or compared bitwise /
by relative difference against the saved one (later runs).

    python tools/k3_time_probe.py [c5] [ref.pt]
"""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_2101_05917_b200 as pdb
from pd_inputs import get_config, make_inputs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
ref = sys.argv[2] if len(sys.argv) > 2 else None
inp = make_inputs(get_config(cfg), steps=1)
sim = pdb.simulator_from_inputs(inp, max_steps=1)
B, N = inp["B"], 3 * inp["n_nodes"]
g = torch.Generator(device="cuda").manual_seed(7)
r = torch.randn(B, N, dtype=torch.float64, device="cuda", generator=g); o = torch.zeros_like(r)
for _ in range(3): sim.apply_Ainv(r, o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for rep in range(3):
    e0.record()
    for _ in range(50): sim.apply_Ainv(r, o)
    e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 50 * 1e3)
knobs = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("PD_K3") or k == "PD_ND_LEAF")
msg = ""
if ref:
    if os.path.exists(ref):
        x = torch.load(ref).cuda()
        msg = "bitwise" if torch.equal(x, o) else "max rel diff %.2e" % ((x - o).abs().max() / x.abs().max()).item()
    else:
        torch.save(o.cpu(), ref)
        msg = "saved"
print(f"{cfg} [{knobs or 'default'}] apply_Ainv min {min(ts):.1f} us (reps {', '.join('%.1f' % t for t in ts)}) {msg}")
