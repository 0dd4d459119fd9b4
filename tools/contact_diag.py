"""Diagnostic: per-step GPU-vs-oracle errors on a contact config at several forward tolerances."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import paper_2101_05917_b200 as pdb
from gpu_common import oracle_run, rel, to_dev
from pd_inputs import get_config, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c4s"
inp = make_inputs(get_config(name))
tr, g, _, _ = oracle_run(inp, 0)
for accel in (0, 1):
    for tol in (1e-12, 1e-13, 3e-14):
        sim = pdb.simulator_from_inputs(inp, tol_fwd=tol, tol_adj=1e-11, accel_fwd=accel, max_iter_fwd=5000)
        B, T, N = inp["B"], inp["T"], 3 * inp["n_nodes"]
        qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device="cuda"); vt = torch.zeros_like(qt)
        st = sim.forward(to_dev(inp["q0"]), to_dev(inp["v0"]), T, f_ext=to_dev(inp["f_ext"]), youngs=to_dev(inp["youngs"]),
                         actuation=None if inp["act"] is None else to_dev(inp["act"]), q_traj=qt, v_traj=vt)
        q, v = qt.cpu().numpy()[0], vt.cpu().numpy()[0]
        eq = [rel(q[i], tr["q"][i]) for i in range(1, T + 1)]
        ev = [rel(v[i], tr["v"][i]) for i in range(1, T + 1)]
        dv = [np.linalg.norm(v[i] - tr["v"][i]) for i in range(1, T + 1)]
        print(f"accel={accel} tol={tol:g} nonconv={st['n_nonconverged']} its={st['iters_fwd'][0].tolist()}")
        print("  rel q:", " ".join(f"{x:.1e}" for x in eq))
        print("  rel v:", " ".join(f"{x:.1e}" for x in ev))
        print("  |dv| :", " ".join(f"{x:.1e}" for x in dv))
        print("  res  :", " ".join(f"{x:.1e}" for x in st["final_res_fwd"][0]))
