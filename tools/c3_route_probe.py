#!/usr/bin/env python
"""Developer probe (GPU): the soft and the stiff c3 sim over the whole horizon with the three forward routes
(accel_fwd 0 plain PD, 1 L-BFGS, 2 Newton-PCG), each against tests/golden/oracle_c3full.npz at the stored steps, and
the routes against each other at every step (first step where two routes separate by more than 1e-8).

    python tools/c3_route_probe.py [tol]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import test_gpu_fullsize as tf
    from gpu_common import rel, to_dev
    from paper_2101_05917_b200.shard import PER_SIM_KEYS, shared_youngs_ref
    from pd_inputs import get_config, make_inputs
    tol = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-13
    gd = dict(np.load(os.path.join(ROOT, "tests", "golden", "oracle_c3full.npz"), allow_pickle=False))
    T = int(gd["steps"])
    full = make_inputs(get_config("c3"), steps=T)
    sims = [int(b) for b in gd["sims"]]
    inp = dict(full)
    for k in PER_SIM_KEYS:
        if inp.get(k) is not None:
            inp[k] = inp[k][sims]
    inp["B"] = len(sims)
    traj = {}
    for route in (0, 1, 2):
        inp["youngs_ref"] = shared_youngs_ref(full["youngs"], bool(route))
        sim = tf._bench_sim(inp, tol_fwd=tol, tol_adj=10 * tol, accel_fwd=route, max_iter_fwd=20000)
        B, N = inp["B"], 3 * inp["n_nodes"]
        qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device="cuda")
        vt = torch.zeros_like(qt)
        st = sim.forward(to_dev(inp["q0"]), to_dev(inp["v0"]), T, f_ext=to_dev(inp["f_ext"]), actuation=None,
                         youngs=to_dev(inp["youngs"]), q_traj=qt, v_traj=vt)
        q = qt.cpu().numpy()
        traj[route] = q
        print(f"route {route}: nonconverged {st['n_nonconverged']}, iters/step mean {np.mean(st['iters_fwd']):.1f}", flush=True)
        for j, b in enumerate(sims):
            eq = [rel(q[j, i], gd[f"s{b}_q"][k]) for k, i in enumerate(gd["keep"])]
            print(f"  sim {b} vs golden q at stored steps: " + " ".join(f"{e:.1e}" for e in eq), flush=True)
    for a, c in ((0, 1), (0, 2), (1, 2)):
        for j, b in enumerate(sims):
            d = [rel(traj[a][j, i], traj[c][j, i]) for i in range(1, T + 1)]
            first = next((i + 1 for i, e in enumerate(d) if e > 1e-8), None)
            print(f"routes {a} vs {c}, sim {b}: max {max(d):.2e}, first step over 1e-8: {first}; around it: "
                  + (" ".join(f"{d[i]:.1e}" for i in range(max(0, first - 4), min(T, first + 3))) if first else "-"),
                  flush=True)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", "c3_route_probe.npz"),
                        **{f"q{r}": traj[r][:, 150:] for r in traj})


if __name__ == "__main__":
    main()
