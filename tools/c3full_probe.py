#!/usr/bin/env python
"""Developer probe: errors of the full-horizon c3 run against tests/golden/oracle_c3full.npz per stored step, for
several per-step solver tolerances (how the per-step error accumulates over the 200-step swing).

    python tools/c3full_probe.py 1e-12 1e-13 3e-14
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
    from gpu_common import rel
    from pd_inputs import get_config, make_inputs
    gd = dict(np.load(os.path.join(ROOT, "tests", "golden", "oracle_c3full.npz"), allow_pickle=False))
    T = int(gd["steps"])
    inp = make_inputs(get_config("c3"), steps=T)
    for tol in [float(a) for a in sys.argv[1:]] or [1e-12, 1e-13]:
        gpu = tf._run(torch, inp, tf._bench_sim(inp, tol_fwd=tol, tol_adj=10 * tol))
        print(f"tol_fwd {tol:g}: nonconverged fwd {gpu['st']['n_nonconverged']} adj {gpu['sb']['n_nonconverged']}, "
              f"fwd iters/step mean {np.mean(gpu['st']['iters_fwd']):.1f}", flush=True)
        for b in gd["sims"]:
            p = f"s{int(b)}_"
            eq = [rel(gpu["q"][b, i], gd[p + "q"][k]) for k, i in enumerate(gd["keep"])]
            ev = [rel(gpu["v"][b, i], gd[p + "v"][k]) for k, i in enumerate(gd["keep"])]
            eg = {k: rel(gpu[k][b], gd[p + k]) for k in ("dq0", "dv0", "dfext")}
            eg["dE"] = abs(gpu["dE"][b] - gd[p + "dE"]) / abs(gd[p + "dE"])
            print(f"  sim {int(b)}: max q {max(eq):.2e}, max v {max(ev):.2e}, v per stored step "
                  + " ".join(f"{e:.1e}" for e in ev) + " | grads " + " ".join(f"{k} {v:.1e}" for k, v in eg.items()),
                  flush=True)


if __name__ == "__main__":
    main()
