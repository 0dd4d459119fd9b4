"""Timeline of one K3 solve (PD_K3_TRACE=1): per level, span, time waiting for inputs, data, reductions."""
import os
import sys

os.environ["PD_K3_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2101_05917_b200 as pdb
from pd_inputs import get_config, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
inp = make_inputs(get_config(name), steps=1)
sim = pdb.simulator_from_inputs(inp, contact_nodes=())
B, N = inp["B"], 3 * inp["n_nodes"]
rhs = torch.randn((B, N), dtype=torch.float64, device="cuda")
out = torch.zeros_like(rhs)
for _ in range(3):
    sim.apply_Ainv(rhs, out)
torch.cuda.synchronize()
tr = sim.k3_trace()
ok = tr[:, 0] > 0
t0 = tr[ok, 0].min()
tr = tr.astype(np.float64)
tr[:, :4] = (tr[:, :4] - t0) / 1e3  # us
tr[:, 6:8] = (tr[:, 6:8] - t0) / 1e3
nf = (tr.shape[0])
print("items", tr.shape[0], "span us %.1f" % (tr[ok, 3].max()))
wait = tr[ok, 1] - tr[ok, 0]
data = tr[ok, 2] - tr[ok, 1]
tail = tr[ok, 3] - tr[ok, 2]
print("per item us: wait mean %.1f max %.1f | data+compute mean %.1f max %.1f | output/reduce mean %.1f max %.1f" % (
    wait.mean(), wait.max(), data.mean(), data.max(), tail.mean(), tail.max()))
# coarse timeline: items finished per 10 us bucket
end = tr[ok, 3]
hist, edges = np.histogram(end, bins=40)
print("completions per bucket:", hist.tolist(), "bucket us %.1f" % (edges[1] - edges[0]))
warps = np.unique(tr[ok, 5]).size
print("warps used", warps, "SMs", np.unique(tr[ok, 4]).size)

# item-index windows (items are in level order: forward first, then backward)
nwin = 16
edges = np.linspace(0, tr.shape[0], nwin + 1).astype(int)
for a, b in zip(edges[:-1], edges[1:]):
    w = tr[a:b]
    w = w[w[:, 0] > -1e9]
    print("items %6d-%6d start %7.1f end %7.1f | wait %6.1f data %5.1f out %6.1f" % (
        a, b, w[:, 0].min(), w[:, 3].max(), (w[:, 1] - w[:, 0]).mean(), (w[:, 2] - w[:, 1]).mean(), (w[:, 3] - w[:, 2]).mean()))
# per-warp occupancy: gaps between consecutive items of the same warp
gaps, busy = [], []
for wid in np.unique(tr[ok, 5]):
    w = tr[ok & (tr[:, 5] == wid)]
    w = w[np.argsort(w[:, 0])]
    if len(w) > 1:
        gaps.extend((w[1:, 0] - w[:-1, 3]).tolist())
    busy.append(((w[:, 3] - w[:, 0]).sum(), len(w), w[:, 3].max() - w[:, 0].min()))
gaps = np.array(gaps)
busy = np.array(busy)
print("gap between items of a warp: mean %.2f us, max %.1f; items per warp mean %.1f max %d; warp busy/lifetime %.2f" % (
    gaps.mean(), gaps.max(), busy[:, 1].mean(), busy[:, 1].max(), busy[:, 0].sum() / busy[:, 2].sum()))

wr = tr[ok, 6] - tr[ok, 2]
cn = tr[ok, 7] - tr[ok, 6]
rd = tr[ok, 3] - tr[ok, 7]
print("out phase split: write %.2f  first-countdown %.2f  rest(reductions/signals) %.2f  (means, us)" % (wr.mean(), cn.mean(), rd.mean()))
