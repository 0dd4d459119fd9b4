"""Oracle backpropagation (test infrastructure only; see oracle/__init__.py).

Plain definition of the adjoint gradient:
  A_N = M/h^2 + Hess E_int(x_{i+1}) = A - dA
  dA  = sum_e w_e G_e^T dz_e*/dx
  u   = A_N^{-1} b,   b = dL/dx_{i+1} (+ dL/dv_{i+1}/h)           (eq:pre_adjoint)
  dL/dx_i = (1/h^2)(dy/dx_i)^T M u  (+ direct -dL/dv_{i+1}/h)
The oracle assembles A_N explicitly from the 9x9 projection Jacobians and solves
it directly (scipy sparse LU) — the BASELINE.json "direct dense solve of the
linearized adjoint" check, done sparsely.  The paper's fixed point / quasi-Newton
iteration converges to the same u; the GPU path runs that iteration.

Constrained DoFs (Dirichlet, and in contact steps the pinned normal DoFs of the
frozen active set, "the same modified matrix") carry u = 0.
Parameter gradients: implicit-function differentiation of eq:time_integration:
  dL/dw  = -sum_e sum_q V <G_q u_e, F_q - R_q>        (w = E/(1+nu), reading §8c.2)
  dL/dr  = w_m sum_q V n_hat_q^T (G_mq u_e)            (muscle)
  dL/df_ext(step) = u.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import energy, fem, pd


def hessian_blocks(scene, x, w, act=None):
    """Per-element 24x24 blocks of sum_q V [w G^T (I - dR/dF) G + w_m G_m^T (I - dp/dFm) G_m]."""
    F = fem.deformation_gradients(x, scene.hex8, scene.dx)
    J, R = energy.polar_jacobian(F)                                 # [m,8,9,9]
    G = fem.G_matrices(scene.dx)
    I9 = np.eye(9)
    H = w * scene.V * np.einsum("qka,mqkl,qlb->mab", G, I9 - J, G, optimize=True)
    if getattr(scene, "volume", False):                             # w_v G^T (I - dD/dF) G
        Jv = energy.volume_jacobian(F)
        H = H + w * scene.vol_ratio * scene.V * np.einsum("qka,mqkl,qlb->mab", G, I9 - Jv, G, optimize=True)
    if scene.muscle:
        Fm = np.einsum("mqij,mj->mqi", F, scene.fibers)             # F m_e (per-element fibers)
        r = np.broadcast_to(np.asarray(act)[:, None], Fm.shape[:-1])
        Jm, p, n_hat = energy.muscle_jacobian(Fm, r, scene.fibers[:, None, :])
        if scene.fiber_dir is None:
            Gm = fem.Gm_matrices(scene.dx, scene.fiber)
            H = H + scene.w_muscle * scene.V * np.einsum("qka,mqkl,qlb->mab", Gm, np.eye(3) - Jm, Gm, optimize=True)
        else:
            Gm = np.stack([fem.Gm_matrices(scene.dx, fe) for fe in scene.fibers])   # [m, q, 3, 24]
            H = H + scene.w_muscle * scene.V * np.einsum("mqka,mqkl,mqlb->mab", Gm, np.eye(3) - Jm, Gm,
                                                         optimize=True)
    return H


def assemble_AN(scene, x, w, act=None):
    """A_N = M/h^2 + Hess E_int."""
    K = fem.assemble_blocks(hessian_blocks(scene, x, w, act), scene.hex8, scene.n)
    return (sp.diags(scene.mass / scene.h ** 2) + K).tocsr()


def assemble_dA(scene, x, w, act=None):
    """dA = A - A_N = sum w G^T dz*/dx G."""
    return (scene.A(w) - assemble_AN(scene, x, w, act)).tocsr()


def solve_adjoint(scene, x, w, act, b, cons_mask, solver="direct", rtol=1e-13):
    """u = A_N^{-1} b on the unconstrained DoFs (0 on cons_mask).  solver="direct": sparse LU of A_N;
    solver="pcg": conjugate gradients preconditioned with the prefactorised A (the paper's accelerated
    fixed point, for meshes where the LU of A_N does not fit), to ||A_N u - b|| <= rtol ||b||."""
    AN = assemble_AN(scene, x, w, act)
    fr = ~cons_mask
    if solver == "pcg":
        facs = scene.axis_factors(w, cons_mask)
        u, _, _ = scene.pcg(lambda v: AN @ v, b, lambda r: scene.apply_axis_factors(facs, r), fr, rtol)
        return u
    u = np.zeros_like(b)
    u[fr] = spla.spsolve(AN[fr][:, fr].tocsc(), b[fr])
    return u


def param_terms(scene, x, u, act=None):
    """(dL/dw, dL/dr[m], dL/dw_v) contributions of one step (chain rule)."""
    F = fem.deformation_gradients(x, scene.hex8, scene.dx)
    R, S, V, s = energy.polar_svd(F)
    Gu = fem.deformation_gradients(u, scene.hex8, scene.dx)         # G_q u_e
    dw = -scene.V * np.sum(Gu * (F - R))
    dwv = -scene.V * np.sum(Gu * (F - energy.volume_project(F)[0])) if getattr(scene, "volume", False) else 0.0
    dr = None
    if scene.muscle:
        Fm = np.einsum("mqij,mj->mqi", F, scene.fibers)
        r = np.broadcast_to(np.asarray(act)[:, None], Fm.shape[:-1])
        p, n_hat, nrm = energy.muscle_project(Fm, r, scene.fibers[:, None, :])
        Gmu = np.einsum("mqij,mj->mqi", Gu, scene.fibers)
        dr = scene.w_muscle * scene.V * np.sum(n_hat * Gmu, axis=(-1, -2))
    return dw, dr, dwv


def backward(scene, traj, youngs, dL_dqT, dL_dvT, act=None, dL_dq_steps=None, dL_dv_steps=None, solver="direct"):
    """Reverse pass over a trajectory from oracle.pd.forward.

    Per-step losses L = sum_i l_i(q_i, v_i) (the Plant task's "loss at each time step"): optional
    dL_dq_steps, dL_dv_steps [T+1, 3n] are added to the adjoint of state i when the reverse pass reaches it.
    Returns dict(dq0, dv0, dfext (summed over steps), dfext_steps [T, 3n] (= u_i, dL/df_ext of step i),
    dE, dnu, dw, dact[T,m] or None)."""
    if pd.has_plane(scene):  # general contact plane: the adjoint in plane coordinates (vectors rotate)
        tr = dict(traj, q=pd.to_plane(scene, traj["q"], True), v=pd.to_plane(scene, traj["v"], False))
        vec = lambda a: None if a is None else pd.to_plane(scene, np.asarray(a, float), False)
        g = backward(pd.plane_scene(scene), tr, youngs, vec(dL_dqT), vec(dL_dvT), act, vec(dL_dq_steps),
                     vec(dL_dv_steps), solver)
        for k in ("dq0", "dv0", "dfext", "dfext_steps"):
            g[k] = pd.from_plane(scene, g[k], False)
        return g
    h = scene.h
    w = scene.w_of(youngs)
    T = traj["q"].shape[0] - 1
    ax = dL_dqT.copy()
    av = dL_dvT.copy()
    if dL_dq_steps is not None:
        ax = ax + dL_dq_steps[T]
    if dL_dv_steps is not None:
        av = av + dL_dv_steps[T]
    base = ~scene.free
    sticky = getattr(scene, "contact_mode", "frictionless") == "sticky"
    nodes = np.asarray(scene.contact_nodes)
    dfext = np.zeros(scene.N)
    dfext_steps = np.zeros((T, scene.N))
    dw_tot = 0.0
    dwv_tot = 0.0
    dact = np.zeros((T, scene.m)) if scene.muscle else None
    for i in range(T - 1, -1, -1):
        x1 = traj["q"][i + 1]
        cons = base.copy()
        pins = scene.pinned_dofs(nodes[traj["active"][i]]) if len(nodes) else np.zeros(0, np.int64)
        cons[pins] = True
        b = ax + av / h                                    # v_{i+1} = (x_{i+1} - x_i)/h
        b_pin = b[pins].copy()
        b[cons] = 0.0
        a_i = None if act is None else act[i]
        u = solve_adjoint(scene, x1, w, a_i, b, cons, solver)
        extra = None
        if sticky and len(pins):
            # x_{i+1,a} = x_{i,a}: dL/dx_{i,a} += b_a - (A_N u)_a  (u_a = 0)
            AN = assemble_AN(scene, x1, w, a_i)
            extra = np.zeros_like(b)
            extra[pins] = b_pin - (AN @ u)[pins]
        dw, dr, dwv = param_terms(scene, x1, u, a_i)
        dw_tot += dw
        dwv_tot += dwv
        if dr is not None:
            dact[i] = dr
        dfext += u
        dfext_steps[i] = u
        ax = scene.mass / h ** 2 * u - av / h              # (1/h^2)(dy/dx_i)^T M u - a_v/h
        if extra is not None:
            ax = ax + extra
        av = scene.mass / h * u                            # dy/dv_i = h I
        if dL_dq_steps is not None:
            ax = ax + dL_dq_steps[i]
        if dL_dv_steps is not None:
            av = av + dL_dv_steps[i]
        ax[base] = 0.0
        av[base] = 0.0
    dfext[base] = 0.0
    dfext_steps[:, base] = 0.0
    # w = 2 mu = E/(1+nu) (reading §8c.2) and, with the volume term, w_v = lambda = E nu/((1+nu)(1-2nu))
    # (SPEC lame_weights): dL/dE and dL/dnu by the chain rule through both weights
    nu = scene.poisson
    dE = dw_tot / (1.0 + nu) + dwv_tot * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    dnu = (-dw_tot * youngs / (1.0 + nu) ** 2
           + dwv_tot * youngs * (1.0 + 2.0 * nu ** 2) / ((1.0 + nu) ** 2 * (1.0 - 2.0 * nu) ** 2))
    return dict(dq0=ax, dv0=av, dfext=dfext, dfext_steps=dfext_steps, dw=dw_tot, dwv=dwv_tot,
                dE=dE, dnu=dnu, dact=dact)


def loss_and_grad(inp, b, q, v):
    """Loss of SURVEY §8c.13 for sim b and its terminal gradients (dL/dq_T, dL/dv_T)."""
    cfg = inp["cfg"]
    if cfg.loss == "linear_q":
        return float(inp["c_q"][b] @ q), inp["c_q"][b].copy(), np.zeros_like(v)
    if cfg.loss == "linear_qv":
        return (float(inp["c_q"][b] @ q + inp["c_v"][b] @ v), inp["c_q"][b].copy(),
                inp["c_v"][b].copy())
    if cfg.loss == "tip":
        idx = (3 * inp["tip_nodes"][:, None] + np.arange(3)[None, :]).ravel()
        diff = q[idx] - inp["tip_target"][b]
        g = np.zeros_like(q)
        g[idx] = 2.0 * diff
        return float(diff @ diff), g, np.zeros_like(v)
    raise ValueError(cfg.loss)
