#!/usr/bin/env python
"""Developer probe: A^-1 applications per time step vs the per-sim iteration statistics (how much the batch loses to
sims that wait for the slowest one inside each Alg. 1 outer iteration).  python tools/solve_count.py c5 [T]"""
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
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    inp = make_inputs(get_config(name), steps=T)
    sim = pdb.simulator_from_inputs(inp, profile=1, max_steps=T)
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    B, N = inp["B"], 3 * inp["n_nodes"]
    act = None if inp["act"] is None else dev(inp["act"])
    st = sim.forward(dev(inp["q0"]), dev(inp["v0"]), T, f_ext=dev(inp["f_ext"]), actuation=act, youngs=dev(inp["youngs"]))
    pf = sim.profile()
    it = np.asarray(st["iters_fwd"]).reshape(B, T)
    outer = np.asarray(st["contact_outer"]).reshape(B, T) if st.get("contact_outer") is not None else None
    print("forward solves (K3 count):", pf["solve_K3"][1], "per step", pf["solve_K3"][1] / T)
    print("per-sim iterations per step: mean", it.mean(), "max over sims (per step, mean over steps)", it.max(0).mean())
    if outer is not None:
        print("outer iterations per step: mean", outer.mean(), "max", outer.max(0).mean())


if __name__ == "__main__":
    main()
