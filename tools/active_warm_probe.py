#!/usr/bin/env python
"""Developer probe (GPU): PD_ACTIVE_WARM=1 (a step's first Alg. 1 outer iteration starts from the previous step's final
active set instead of the empty set of P:339 — NOT the algorithm as printed, off by default) against the default path
on the contact configs: are the final active sets the same at every step, how far are the states apart, how many outer
and inner iterations does each take.

    python tools/active_warm_probe.py c5s c4s c4
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def run(name, warm):
    import torch
    import test_gpu_fullsize as tf
    from pd_inputs import get_config, make_inputs
    os.environ["PD_ACTIVE_WARM"] = "1" if warm else "0"
    inp = make_inputs(get_config(name))
    sim = tf._bench_sim(inp, tol_fwd=2e-14, tol_adj=1e-11, max_iter_fwd=6000)
    gpu = tf._run(torch, inp, sim)
    return gpu, np.asarray(sim.contact_sets())


def main():
    from gpu_common import rel
    for name in sys.argv[1:] or ["c5s", "c4s"]:
        a, sa = run(name, False)
        b, sb = run(name, True)
        same = bool(np.array_equal(sa, sb))
        first = None if same else int(np.argwhere((sa != sb).reshape(sa.shape[0], sa.shape[1], -1).any(axis=(0, 2)))[0, 0])
        dq = max(rel(b["q"][:, i], a["q"][:, i]) for i in range(1, a["q"].shape[1]))
        dg = max(rel(b[k], a[k]) for k in ("dq0", "dv0", "dfext"))
        print(f"{name}: sets equal {same} (first differing step {first}); max rel dq {dq:.2e}, max rel dgrad {dg:.2e}; "
              f"outer/step {np.mean(a['st']['contact_outer']):.2f} -> {np.mean(b['st']['contact_outer']):.2f}; "
              f"fwd iters/step {np.mean(a['st']['iters_fwd']):.1f} -> {np.mean(b['st']['iters_fwd']):.1f}; "
              f"nonconverged {a['st']['n_nonconverged']} / {b['st']['n_nonconverged']}", flush=True)


if __name__ == "__main__":
    main()
