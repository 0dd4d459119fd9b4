#!/usr/bin/env python
"""Oracle-only probe (no CUDA): is the minimiser of g unique along the soft c3 beam's late swing?

From the stored oracle state of sim 53 at step 160 (tests/golden/oracle_c3full.npz) run the oracle for 20 more steps
twice — method="newton" (the golden's route) and method="pd" (the literal local-global iteration from x_i) —
and print, per step, the distance between the two converged states and both objective values.  Two converged routes
that separate by far more than their tolerances have found different stationary points of the non-convex corotated
objective.

    python tools/c3_branch_probe.py [sim] [start_step] [steps] [pd_steps] [--save]

--save writes tests/golden/oracle_c3full_pdbranch.npz: the literal-PD route's states at the stored steps after the
start step (the branch the GPU follows), the per-step separation of the two routes and the objective values of both
at the first separated step.  The run stops at the first step the PD route does not converge to 1e-13 (its
stagnation exit; measured: step 186 of sim 53, residual 7e-6 after 276 iterations), so only step 180 is stored.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pd  # noqa: E402
from pd_inputs import get_config, make_inputs  # noqa: E402


def main():
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 53
    s0 = int(sys.argv[2]) if len(sys.argv) > 2 else 160
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    n_pd = int(sys.argv[4]) if len(sys.argv) > 4 else n   # the pd route continues alone up to this many steps
    gd = np.load(os.path.join(ROOT, "tests", "golden", "oracle_c3full.npz"))
    keep = list(gd["keep"])
    k = keep.index(s0)
    inp = make_inputs(get_config("c3"), steps=200)
    sc = pd.scene_from_inputs(inp)
    w = sc.w_of(inp["youngs"][b])
    q = {m: gd[f"s{b}_q"][k].copy() for m in ("newton", "pd")}
    v = {m: gd[f"s{b}_v"][k].copy() for m in ("newton", "pd")}
    sep, first_sep, g_at_sep, stored = [], 0, (0.0, 0.0), {}
    for i in range(max(n, n_pd)):
        out = {}
        for m in ("newton", "pd") if i < n else ("pd",):
            tr = pd.forward(sc, q[m], v[m], inp["f_ext"][b], inp["youngs"][b], None, steps=1, tol=1e-13, method=m)
            y = sc.y(q[m], v[m], inp["f_ext"][b])
            g, _ = sc.objective(tr["q"][-1], y, w, None)
            out[m] = (tr["q"][-1], tr["v"][-1], g, tr["stats"][-1]["iters"], tr["stats"][-1]["res"])
        step = s0 + i + 1
        if i < n:
            dq = np.linalg.norm(out["newton"][0] - out["pd"][0]) / np.linalg.norm(out["newton"][0])
            sep.append(dq)
            if not first_sep and dq > 1e-8:
                first_sep, g_at_sep = step, (out["newton"][2], out["pd"][2])
            print(f"step {step}: |q_newton - q_pd|/|q| = {dq:.2e}; newton g {out['newton'][2]:.12e} ({out['newton'][3]} its, "
                  f"res {out['newton'][4]:.1e}); pd g {out['pd'][2]:.12e} ({out['pd'][3]} its, res {out['pd'][4]:.1e})",
                  flush=True)
        else:
            print(f"step {step}: pd g {out['pd'][2]:.12e} ({out['pd'][3]} its, res {out['pd'][4]:.1e})", flush=True)
        for m in out:
            q[m], v[m] = out[m][0], out[m][1]
        if out["pd"][4] > 1e-13:  # the PD route's stagnation exit (oracle/pd.py pd_solve): no reference beyond here
            print(f"pd route not converged at step {step} (res {out['pd'][4]:.1e}): stop", flush=True)
            break
        if step in keep:
            stored[step] = (q["pd"].copy(), v["pd"].copy())
            kk = keep.index(step)
            for m in out:
                print(f"{m} vs golden at step {step}: "
                      f"{np.linalg.norm(q[m] - gd[f's{b}_q'][kk]) / np.linalg.norm(q[m]):.2e}", flush=True)
    if "--save" in sys.argv:
        steps = sorted(stored)
        path = os.path.join(ROOT, "tests", "golden", "oracle_c3full_pdbranch.npz")
        np.savez_compressed(path, sim=b, start=s0, steps=np.asarray(steps), q=np.stack([stored[t][0] for t in steps]),
                            v=np.stack([stored[t][1] for t in steps]), separation=np.asarray(sep),
                            first_separated_step=first_sep, g_newton_pd_at_separation=np.asarray(g_at_sep))
        print(f"wrote {path}", flush=True)


if __name__ == "__main__":
    main()
