"""Write the oracle goldens the full-size GPU parity tests compare against (tests/golden/*.npz).

Every stored value comes from oracle/ (plus the seeded inputs of pd_inputs, which hold none of the
method's arithmetic) — nothing here imports or runs the CUDA path.  Rerun with

    python tools/make_goldens.py c5      # config c5, sim 0, first 2 steps (newton_pcg / pcg routes)
    python tools/make_goldens.py c3      # config c3, stiffest + softest sim, first 30 steps
    python tools/make_goldens.py c4      # config c4, the whole 150-step contact drop
    python tools/make_goldens.py c2      # config c2, the whole 100-step cantilever (4131 DoF)
    python tools/make_goldens.py c3full  # config c3, stiffest + softest sim, the whole 200-step horizon
    python tools/make_goldens.py c5long  # config c5, sim 0, first 4 steps (about 40 min on 8 host cores)

What is stored per sim: the states of every `every`-th step and of the last step (q, v), the Alg. 1 active
sets of every step, the per-step oracle statistics, and the gradients of the config's loss at the last
stored step: dL/dq0, dL/dv0, dL/df_ext (summed), dL/dE, dL/dnu, dL/dact.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import adjoint, pd  # noqa: E402
from pd_inputs import get_config, make_inputs  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")

# name -> (config, steps, sims (None = extremes of E), oracle tol, forward method, adjoint solver, every)
SPECS = {
    "c5": ("c5", 2, [0], 1e-13, "newton_pcg", "pcg", 1),
    "c3": ("c3", 30, None, 1e-13, "newton", "direct", 5),
    "c4": ("c4", 150, [0], 2e-14, "newton", "direct", 10),
    "c2": ("c2", 100, [0], 1e-13, "newton", "direct", 10),
    # the whole 200-step horizon of configs[2] (stiffest + softest sim): the soft beam's full swing
    "c3full": ("c3", 200, None, 1e-13, "newton", "direct", 20),
    # the softest c3 sim up to step 160, with the gradients of the tip loss at that horizon: the part of its swing
    # on which the minimiser of g is unique (reading 2.20; tools/c3_branch_probe.py)
    "c3soft160": ("c3", 160, [53], 1e-13, "newton", "direct", 20),
    # a longer c5 prefix (sim 0, 4 steps: the contact set changes again after the first impact steps)
    "c5long": ("c5", 4, [0], 1e-13, "newton_pcg", "pcg", 1),
}


def run(key):
    name, T, sims, tol, method, solver, every = SPECS[key]
    cfg = get_config(name)
    inp = make_inputs(cfg, steps=T)
    if sims is None:
        E = inp["youngs"]
        sims = [int(np.argmax(E)), int(np.argmin(E))]
    keep = sorted(set(list(range(every, T + 1, every)) + [T]))
    out = dict(config=name, steps=T, sims=np.asarray(sims), keep=np.asarray(keep), tol=tol, method=method,
               solver=solver)
    t0 = time.time()
    for b in sims:
        sc = pd.scene_from_inputs(inp)
        act = None if inp["act"] is None else inp["act"][b, :T]
        tr = pd.forward(sc, inp["q0"][b], inp["v0"][b], inp["f_ext"][b], inp["youngs"][b], act, steps=T, tol=tol,
                        fixed_iter=cfg.fixed_iter, method=method)
        print(f"{key} sim {b}: forward done {time.time() - t0:.0f} s", flush=True)
        L, gq, gv = adjoint.loss_and_grad(inp, b, tr["q"][-1], tr["v"][-1])
        g = adjoint.backward(sc, tr, inp["youngs"][b], gq, gv, act, solver=solver)
        print(f"{key} sim {b}: backward done {time.time() - t0:.0f} s", flush=True)
        p = f"s{b}_"
        out[p + "q"] = tr["q"][keep]
        out[p + "v"] = tr["v"][keep]
        out[p + "active"] = tr["active"]
        out[p + "iters"] = np.asarray([s["iters"] for s in tr["stats"]])
        out[p + "outer"] = np.asarray([s["outer"] for s in tr["stats"]])
        out[p + "res"] = np.asarray([s["res"] for s in tr["stats"]])
        out[p + "flag"] = np.asarray([s["flag"] for s in tr["stats"]])
        out[p + "vnorm"] = np.linalg.norm(tr["v"], axis=1)
        out[p + "loss"] = L
        for k in ("dq0", "dv0", "dfext", "dE", "dnu"):
            out[p + k] = g[k]
        if g["dact"] is not None:
            out[p + "dact"] = g["dact"]
    os.makedirs(GOLDEN, exist_ok=True)
    path = os.path.join(GOLDEN, f"oracle_{key}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.1f} MB) in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    for k in sys.argv[1:] or list(SPECS):
        run(k)
