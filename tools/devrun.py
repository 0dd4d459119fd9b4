#!/usr/bin/env python
"""Developer timing probe (not the bench): one forward+backward of a config, possibly on a shortened
horizon, printing per-kernel-family device time, iteration counts and launches.

    python tools/devrun.py c3 --horizon 5 --set accel_fwd=1
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--horizon", type=int, default=0)
    ap.add_argument("--tol", type=float, default=0.0)
    ap.add_argument("--set", action="append", default=[], help="Simulator kwarg key=value")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2101_05917_b200 as pdb
    from pd_inputs import get_config, make_inputs
    cfg = get_config(a.config)
    T = a.horizon or cfg.steps
    inp = make_inputs(cfg, steps=T)
    kw = dict(profile=1)
    if a.tol:
        kw.update(tol_fwd=a.tol, tol_adj=a.tol)
    for kv in a.set:
        k, v = kv.split("=", 1)
        kw[k] = eval(v)
    t0 = time.perf_counter()
    sim = pdb.simulator_from_inputs(inp, **kw)
    setup = time.perf_counter() - t0
    dev = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
    B, N = inp["B"], 3 * inp["n_nodes"]
    qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device="cuda")
    vt = torch.zeros_like(qt)
    act = None if inp["act"] is None else dev(inp["act"])
    for rep in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = sim.forward(dev(inp["q0"]), dev(inp["v0"]), T, f_ext=dev(inp["f_ext"]), actuation=act,
                         youngs=dev(inp["youngs"]), q_traj=qt, v_traj=vt)
        torch.cuda.synchronize()
        tf = time.perf_counter() - t0
        pf = sim.profile()
        lf = sim.info()["launches"]
        gq = dev(inp["c_q"])
        gv = dev(inp["c_v"])
        t0 = time.perf_counter()
        sb = sim.backward(gq, gv, torch.zeros_like(gq), torch.zeros_like(gq), torch.zeros_like(gq),
                          torch.zeros(B, dtype=torch.float64, device="cuda"),
                          torch.zeros(B, dtype=torch.float64, device="cuda"), None if act is None else torch.zeros_like(act))
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        pb = sim.profile()
        lb = sim.info()["launches"]
        out = dict(config=a.config, T=T, B=B, dof=N, setup_s=round(setup, 3), info=sim.info(), fwd_s=round(tf, 4),
                   bwd_s=round(tb, 4), dof_steps_per_s=B * T * N / (tf + tb),
                   iters_fwd=dict(mean=float(st["iters_fwd"].mean()), max=int(st["iters_fwd"].max())),
                   iters_adj=dict(mean=float(sb["iters_adj"].mean()), max=int(sb["iters_adj"].max())),
                   outer=dict(mean=float(st["contact_outer"].mean()), max=int(st["contact_outer"].max())),
                   nonconv=(st["n_nonconverged"], sb["n_nonconverged"]), launches=(lf, lb),
                   prof_fwd={k: (round(v[0], 2), v[1]) for k, v in pf.items()},
                   prof_all={k: (round(v[0], 2), v[1]) for k, v in pb.items()}, kw=a.set)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
