#!/usr/bin/env python
"""Live per-launch timeline of one A^{-1} application (developer probe): torch.profiler (CUPTI) records the
kernels of a few pd_apply_Ainv calls; prints, for the last call, each launch's start (relative), duration,
overlap with / gap after the previous launch, and per-kernel totals.

    python tools/k3_trace.py c5 [--reps 5]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c5")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2101_05917_b200 as pdb
    from pd_inputs import get_config, make_inputs
    inp = make_inputs(get_config(a.config), steps=1)
    sim = pdb.simulator_from_inputs(inp, max_steps=1)
    B, N = inp["B"], 3 * inp["n_nodes"]
    r = torch.randn(B, N, dtype=torch.float64, device="cuda")
    o = torch.zeros_like(r)
    for _ in range(3):
        sim.apply_Ainv(r, o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        sim.apply_Ainv(r, o)
    e1.record()
    torch.cuda.synchronize()
    print("apply_Ainv (events, 20 reps) %.1f us" % (e0.elapsed_time(e1) / 20 * 1e3))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            sim.apply_Ainv(r, o)
        torch.cuda.synchronize()
    ks = []
    for e in prof.events():
        if e.device_type.name == "CUDA" and "pdb::" in e.name:
            ks.append((e.time_range.start, e.time_range.end, e.name))
    ks.sort()
    # one call = from a k_to_solve to the next k_to_solve
    starts = [i for i, k in enumerate(ks) if "k_to_solve" in k[2]]
    blk = ks[starts[-2]:starts[-1]] if len(starts) >= 2 else ks
    t0 = blk[0][0]
    prev_end = None
    tot = {}
    for s, e, n in blk:
        gap = "" if prev_end is None else "%+7.2f" % (s - prev_end)
        short = n.split("pdb::")[1].split("(")[0]
        print("%8.2f %7.2f %s  %s" % (s - t0, e - s, gap, short))
        prev_end = e
        tot.setdefault(short, [0, 0.0])
        tot[short][0] += 1
        tot[short][1] += e - s
    print("span %.1f us" % (blk[-1][1] - t0))
    for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print("  %-40s %4d %9.1f us" % (k, c, d))


if __name__ == "__main__":
    main()
