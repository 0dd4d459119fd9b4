#!/usr/bin/env python
"""Developer probe (GPU): cost of the per-family CUDA-event profiler inside the timed region — one forward + backward
of a workload at a short horizon with pd_options.profile = 0 and 1 (device time by CUDA events around the pair).

    python tools/profile_cost_probe.py c5 20
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2101_05917_b200 as pdb
    from pd_inputs import get_config, make_inputs
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = get_config(name)
    inp = make_inputs(cfg, steps=T)
    dev = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
    B, N = inp["B"], 3 * inp["n_nodes"]
    act = None if inp["act"] is None else dev(inp["act"])
    a = [dev(inp["q0"]), dev(inp["v0"]), dev(inp["f_ext"]), dev(inp["youngs"])]
    gq, gv = dev(inp["c_q"]), dev(inp["c_v"])
    z = lambda: torch.zeros_like(gq)
    zb = lambda: torch.zeros(B, dtype=torch.float64, device="cuda")
    for prof in (0, 1, 0, 1):
        sim = pdb.simulator_from_inputs(inp, tol_fwd=cfg.tol, tol_adj=cfg.tol, max_steps=T, profile=prof, accel_fwd=1,
                                        outer_warm=1, check_every=1)

        def run():
            sim.forward(a[0], a[1], T, f_ext=a[2], actuation=act, youngs=a[3])
            sim.backward(gq, gv, z(), z(), z(), zb(), zb(), None if act is None else torch.zeros_like(act))
        run()
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        print(f"{name} T={T} profile={prof}: {ms:.2f} ms per forward+backward, {B * T * N / ms / 1e3:.3f} M DoF*steps/s",
              flush=True)
        del sim


if __name__ == "__main__":
    main()
