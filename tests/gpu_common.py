"""Shared helpers for the -m gpu parity tests (CUDA path via the C-ABI vs oracle/)."""
import numpy as np

from pd_inputs import get_config, make_inputs

TOL_PAR_FWD = 1e-12   # DESIGN.md §2.8 parity tolerance (forward)
TOL_PAR_ADJ = 1e-11   # (adjoint)
POS_TOL = 1e-9        # BASELINE.json north_star: positions / velocities
GRAD_TOL = 1e-6       # gradients


def torch_cuda():
    import torch
    return torch


def to_dev(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def oracle_run(inp, b, steps=None, tol=1e-13):
    """Oracle forward + backward for sim b (loss of SURVEY §8c.13)."""
    from oracle import adjoint, pd
    cfg = inp["cfg"]
    T = inp["T"] if steps is None else steps
    sc = pd.scene_from_inputs(inp)
    act = None if inp["act"] is None else inp["act"][b, :T]
    tr = pd.forward(sc, inp["q0"][b], inp["v0"][b], inp["f_ext"][b], inp["youngs"][b], act, steps=T,
                    tol=tol, fixed_iter=cfg.fixed_iter)
    L, gq, gv = adjoint.loss_and_grad(inp, b, tr["q"][-1], tr["v"][-1])
    g = adjoint.backward(sc, tr, inp["youngs"][b], gq, gv, act)
    return tr, g, gq, gv


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
