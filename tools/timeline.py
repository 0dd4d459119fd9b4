#!/usr/bin/env python
"""Device timeline of one forward+backward (developer probe, not the bench): torch.profiler (CUPTI) records
every kernel of the process, ours included, and every CUDA runtime call.  Prints GPU busy vs span, idle
gaps, per-kernel totals and the host-side runtime-call totals.

    python tools/timeline.py c3 --horizon 2 [--set accel_fwd=1 ...]
"""
import argparse
import collections
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--horizon", type=int, default=2)
    ap.add_argument("--set", action="append", default=[])
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--seq", type=int, default=0, help="print the kernels of the first solve (up to N)")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2101_05917_b200 as pdb
    from pd_inputs import get_config, make_inputs
    cfg = get_config(a.config)
    T = a.horizon
    inp = make_inputs(cfg, steps=T)
    kw = dict(profile=1, accel_fwd=1, outer_warm=1, check_every=1)
    for kv in a.set:
        k, v = kv.split("=", 1)
        kw[k] = eval(v)
    sim = pdb.simulator_from_inputs(inp, **kw)
    dev = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
    B, N = inp["B"], 3 * inp["n_nodes"]
    qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device="cuda")
    vt = torch.zeros_like(qt)
    act = None if inp["act"] is None else dev(inp["act"])
    args = [dev(inp["q0"]), dev(inp["v0"]), dev(inp["f_ext"]), dev(inp["youngs"])]
    gq, gv = dev(inp["c_q"]), dev(inp["c_v"])
    z = lambda: torch.zeros_like(gq)
    zb = lambda: torch.zeros(B, dtype=torch.float64, device="cuda")

    def run():
        st = sim.forward(args[0], args[1], T, f_ext=args[2], actuation=act, youngs=args[3], q_traj=qt, v_traj=vt)
        sb = sim.backward(gq, gv, z(), z(), z(), zb(), zb(), None if act is None else torch.zeros_like(act))
        return st, sb

    run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        st, sb = run()
        torch.cuda.synchronize()
    ev = prof.events()
    kern, rt = [], collections.defaultdict(lambda: [0.0, 0])
    for e in ev:
        dt = getattr(e, "device_type", None)
        if dt is not None and "CUDA" in str(dt):
            kern.append((e.time_range.start, e.time_range.end, e.name))
        elif e.name.startswith("cuda") or e.name.startswith("cu"):
            rt[e.name][0] += e.time_range.elapsed_us()
            rt[e.name][1] += 1
    kern.sort()
    span = kern[-1][1] - kern[0][0]
    busy, gaps, last = 0.0, [], kern[0][0]
    per = collections.defaultdict(lambda: [0.0, 0])
    for s, e, n in kern:
        busy += e - s
        if s > last:
            gaps.append(s - last)
        last = max(last, e)
        short = n.split("(")[0].replace("void ", "")[:48]
        per[short][0] += e - s
        per[short][1] += 1
    its_f, its_a = float(st["iters_fwd"].sum()), float(sb["iters_adj"].sum())
    print(json.dumps(dict(config=a.config, T=T, B=B, kernels=len(kern), span_ms=span / 1e3, busy_ms=busy / 1e3,
                          idle_ms=sum(gaps) / 1e3, gaps_over_5us=sum(1 for g in gaps if g > 5),
                          mean_gap_us=float(np.mean(gaps)) if gaps else 0.0, iters_fwd_sum=its_f, iters_adj_sum=its_a,
                          us_per_iter=span / max(1.0, (its_f + its_a) / B))))
    print("| kernel | total ms | count | avg us |")
    for n, (t, c) in sorted(per.items(), key=lambda x: -x[1][0])[:a.top]:
        print(f"| {n} | {t / 1e3:.3f} | {c} | {t / c:.1f} |")
    if a.seq:
        first = next(i for i, k in enumerate(kern) if "k_to_solve" in k[2])
        print("| # | kernel | us | gap before us |")
        for i in range(first, min(len(kern), first + a.seq)):
            print(f"| {i - first} | {kern[i][2].split('(')[0].replace('void ', '')[:40]} | {kern[i][1] - kern[i][0]:.1f} | "
                  f"{kern[i][0] - kern[i - 1][1]:.1f} |")
            if "k_from_solve" in kern[i][2]:
                break
    print("| runtime call | total ms | count | avg us |")
    for n, (t, c) in sorted(rt.items(), key=lambda x: -x[1][0])[:12]:
        print(f"| {n} | {t / 1e3:.3f} | {c} | {t / c:.1f} |")


if __name__ == "__main__":
    main()
