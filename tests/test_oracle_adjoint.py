"""Pins for oracle/adjoint.py: Hessian, direct adjoint, and full-trajectory gradients vs FD."""
import dataclasses

import numpy as np
import pytest

from oracle import adjoint, pd
from pd_inputs import get_config, make_inputs


def _scene(name, **kw):
    cfg = get_config(name, **kw)
    inp = make_inputs(cfg)
    return pd.scene_from_inputs(inp), inp


def test_AN_is_jacobian_of_grad_g():
    # A_N = M/h^2 + Hess E_int: central FD of grad g along random directions.
    for name in ("c1", "c5s"):
        sc, inp = _scene(name)
        rng = np.random.default_rng(0)
        x = inp["q0"][0] + 5e-4 * rng.standard_normal(sc.N)
        act = None if inp["act"] is None else inp["act"][0, 0]
        y = sc.y(x, np.zeros(sc.N), np.zeros(sc.N))
        w = sc.w_of(1e5)
        AN = adjoint.assemble_AN(sc, x, w, act)
        d = rng.standard_normal(sc.N)
        eps = 1e-6
        _, gp = sc.objective(x + eps * d, y, w, act)
        _, gm = sc.objective(x - eps * d, y, w, act)
        fd = (gp - gm) / (2 * eps)
        np.testing.assert_allclose(AN @ d, fd, rtol=0, atol=1e-6 * np.abs(fd).max())
        np.testing.assert_allclose(AN.toarray(), AN.toarray().T, atol=1e-8 * abs(AN).max())


def test_dA_split_and_spectral_radius_at_rest():
    # A_N = A - dA; at rest R = I and dR/dF maps skew->skew, sym->0, so
    # dA = sum w G^T P_skew G and rho(A^{-1} dA) < 1 (the fixed point converges).
    sc, inp = _scene("c1")
    x = inp["rest"].ravel()
    w = sc.w_of(1e5)
    dA = adjoint.assemble_dA(sc, x, w).toarray()
    A = sc.A(w).toarray()
    fr = sc.free
    ev = np.linalg.eigvals(np.linalg.solve(A[fr][:, fr], dA[fr][:, fr]))
    rho = np.abs(ev).max()
    assert 0.3 < rho < 1.0


def test_zero_stiffness_closed_form():
    # SPEC backprop_step example: pure mass system, L = c^T x_1 ->
    # dL/dx_0 = c, dL/dv_0 = h c, dL/df_ext = h^2 M^{-1} c.
    sc, inp = _scene("c1", dirichlet="none")
    c = np.random.default_rng(1).standard_normal(sc.N)
    tr = pd.forward(sc, inp["q0"][0], inp["v0"][0], np.zeros(sc.N), 0.0, steps=1, tol=1e-14)
    g = adjoint.backward(sc, tr, 0.0, c, np.zeros(sc.N))
    np.testing.assert_allclose(g["dq0"], c, rtol=1e-12)
    np.testing.assert_allclose(g["dv0"], sc.h * c, rtol=1e-12)
    np.testing.assert_allclose(g["dfext"], sc.h ** 2 / sc.mass * c, rtol=1e-12)


def _fd_check(name, steps, params, rel, kw=None, tol=1e-14):
    sc, inp = _scene(name, **(kw or {}))
    b = 0
    act = None if inp["act"] is None else inp["act"][b, :steps].copy()
    base = dict(q0=inp["q0"][b].copy(), v0=inp["v0"][b].copy(), f=inp["f_ext"][b].copy(),
                E=float(inp["youngs"][b]), act=act)

    def run(p, sc=sc):
        s = sc if p.get("nu") is None else dataclasses.replace(sc, poisson=p["nu"])
        tr = pd.forward(s, p["q0"], p["v0"], p["f"], p["E"], p["act"], steps=steps, tol=tol)
        L, gq, gv = adjoint.loss_and_grad(inp, b, tr["q"][-1], tr["v"][-1])
        return L, tr, gq, gv, s

    L, tr, gq, gv, s = run(base)
    g = adjoint.backward(s, tr, base["E"], gq, gv, act)
    rng = np.random.default_rng(7)
    for key in params:
        if key in ("q0", "v0", "f"):
            d = rng.standard_normal(sc.N)
            d[~sc.free] = 0
            eps = {"q0": 1e-6, "v0": 1e-5, "f": 1e-5}[key]
            an = {"q0": g["dq0"], "v0": g["dv0"], "f": g["dfext"]}[key] @ d
        elif key == "E":
            d, eps, an = 1.0, 10.0, g["dE"]
        elif key == "nu":
            d, eps, an = 1.0, 1e-5, g["dnu"]
        elif key == "act":
            d = rng.standard_normal(base["act"].shape)
            eps, an = 1e-5, np.sum(g["dact"] * d)
        pp, pm = dict(base), dict(base)
        if key == "nu":
            pp["nu"], pm["nu"] = sc.poisson + eps, sc.poisson - eps
        else:
            pp[key] = base[key] + eps * d
            pm[key] = base[key] - eps * d
        fd = (run(pp)[0] - run(pm)[0]) / (2 * eps)
        assert abs(an - fd) <= rel * max(abs(fd), 1e-12), (key, an, fd)


def test_gradients_vs_central_fd_cantilever():
    # BASELINE.json self-check: central finite differences on tiny meshes, converged forwards.
    _fd_check("c1", 3, ["q0", "v0", "f", "E", "nu"], 1e-5, kw=dict(loss="linear_qv"))


def test_gradients_vs_central_fd_muscle():
    _fd_check("c5s", 2, ["q0", "v0", "act", "E"], 1e-5, kw=dict(contact=False))


def test_per_step_loss_and_time_varying_fext_vs_fd():
    # L = sum_i c_i . q_i + e_i . v_i with a time-varying f_ext; gradients w.r.t. q0 and
    # the per-step f_ext against central finite differences of the oracle forward (converged solves)
    from oracle import adjoint, pd
    from pd_inputs import get_config, make_inputs
    inp = make_inputs(get_config("c1"), steps=3)
    sc = pd.scene_from_inputs(inp)
    T, N = 3, sc.N
    rng = np.random.default_rng(7)
    cq = rng.standard_normal((T + 1, N))
    cv = rng.standard_normal((T + 1, N))
    fext = rng.standard_normal((T, N)) * 0.05
    fext[:, ~sc.free] = 0.0
    E = inp["youngs"][0]

    def L(q0, fe):
        tr = pd.forward(sc, q0, inp["v0"][0], fe, E, steps=T, tol=1e-13)
        return float(np.sum(cq * tr["q"]) + np.sum(cv * tr["v"])), tr

    _, tr = L(inp["q0"][0], fext)
    g = adjoint.backward(sc, tr, E, np.zeros(N), np.zeros(N), dL_dq_steps=cq, dL_dv_steps=cv)
    eps = 1e-6
    k = int(np.nonzero(sc.free)[0][7])
    for which in ("q0", "f1"):
        qp, qm = inp["q0"][0].copy(), inp["q0"][0].copy()
        fp, fm = fext.copy(), fext.copy()
        if which == "q0":
            qp[k] += eps
            qm[k] -= eps
        else:
            fp[1, k] += eps
            fm[1, k] -= eps
        fd = (L(qp, fp)[0] - L(qm, fm)[0]) / (2 * eps)
        an = g["dq0"][k] if which == "q0" else g["dfext_steps"][1, k]
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd)), (which, fd, an)


def test_gradients_vs_central_fd_volume():
    # volume-preserving term: with w_v = lambda the gradient wrt nu is no longer
    # a multiple of the one wrt E; both against central differences of the converged forward
    # (the residual floor of the forward is ~3e-14 with this term: converged runs at 1e-13)
    _fd_check("c2v", 2, ["q0", "v0", "E", "nu"], 1e-5, tol=1e-13)
    # (muscle case: w_m is the nominal-material constant of reading §8c.3, so nu is checked on c2v only)
    _fd_check("c5v", 2, ["q0", "act", "E"], 1e-5, kw=dict(contact=False), tol=1e-13)


def test_volume_AN_is_jacobian_of_grad_g():
    # A_N with the volume term = d(grad g)/dx by central differences on a deformed state
    sc, inp = _scene("c2v")
    rng = np.random.default_rng(3)
    x = inp["rest"].ravel() + 2e-3 * rng.standard_normal(sc.N)
    y = x + 1e-3 * rng.standard_normal(sc.N)
    w = sc.w_of(1e5)
    AN = adjoint.assemble_AN(sc, x, w)
    d = rng.standard_normal(sc.N)
    eps = 1e-7
    fd = (sc.objective(x + eps * d, y, w)[1] - sc.objective(x - eps * d, y, w)[1]) / (2 * eps)
    assert np.linalg.norm(AN @ d - fd) <= 1e-6 * np.linalg.norm(fd)


def test_gradients_vs_central_fd_fiber_field():
    # per-element fiber directions (SURVEY §8(b) material.fiber_dir): muscle energy (w_m/2)(||F m_e|| - r)^2 with
    # each element's own m_e; gradients wrt q0, v0, r and E against central differences (no contact)
    _fd_check("c5f", 2, ["q0", "v0", "act", "E"], 1e-5, kw=dict(contact=False))


def test_fiber_field_energy_closed_form_and_A():
    # Under an affine deformation x = F X every quad point has F_q = F, so the muscle energy of element e is exactly
    # 8 (w_m V / 2)(||F m_e|| - r_e)^2 (reading §8c.4), and x^T A_mus x = sum_e 8 w_m V ||F m_e||^2
    # for the muscle part of A (P:199-202 with G_m x = F m_e) -- written out here per element, not through G.
    from oracle import energy, fem, pd
    from pd_inputs import get_config, make_inputs
    inp = make_inputs(get_config("c5f", contact=False))
    sc = pd.scene_from_inputs(inp)
    F = np.array([[1.05, 0.10, -0.03], [0.02, 0.97, 0.08], [-0.04, 0.05, 1.02]])
    x = (inp["rest"] @ F.T).ravel()
    r = inp["act"][0, 0]
    sc_nm = pd.scene_from_inputs(inp)
    sc_nm.muscle = False
    w = sc.w_of(1e5)
    e_mus = sc.objective(x, x, w, r)[0] - sc_nm.objective(x, x, w)[0]
    m = inp["fiber_dir"]
    closed = sum(8 * 0.5 * sc.w_muscle * sc.V * (np.linalg.norm(F @ m[e]) - r[e]) ** 2 for e in range(sc.m))
    assert abs(e_mus - closed) <= 1e-12 * abs(closed)
    quad = x @ (sc.Kmus @ x)
    closed_q = sum(8 * sc.V * np.linalg.norm(F @ m[e]) ** 2 for e in range(sc.m))
    assert abs(quad - closed_q) <= 1e-12 * closed_q
    # a uniform field reproduces the uniform-fiber scene
    inp_u = dict(inp, fiber_dir=np.tile([1.0, 0.0, 0.0], (sc.m, 1)))
    sc_u, sc_0 = pd.scene_from_inputs(inp_u), pd.scene_from_inputs(dict(inp, fiber_dir=None))
    assert abs(sc_u.objective(x, x, w, r)[0] - sc_0.objective(x, x, w, r)[0]) <= 1e-13 * abs(sc_0.objective(x, x, w, r)[0])


def test_loss_gradients_vs_central_fd():
    # the terminal loss gradients of every loss kind (c3's squared tip error included) against
    # central differences of the loss value itself
    from oracle import adjoint
    from pd_inputs import get_config, make_inputs
    rng = np.random.default_rng(11)
    for name in ("c1", "c2s", "c3s"):
        inp = make_inputs(get_config(name))
        N = 3 * inp["n_nodes"]
        q = inp["rest"].ravel() + 0.01 * rng.standard_normal(N)
        v = 0.1 * rng.standard_normal(N)
        L, gq, gv = adjoint.loss_and_grad(inp, 0, q, v)
        for _ in range(3):
            dq, dv = rng.standard_normal(N), rng.standard_normal(N)
            eps = 1e-6
            fd = (adjoint.loss_and_grad(inp, 0, q + eps * dq, v + eps * dv)[0]
                  - adjoint.loss_and_grad(inp, 0, q - eps * dq, v - eps * dv)[0]) / (2 * eps)
            assert abs(fd - (gq @ dq + gv @ dv)) <= 1e-7 * max(1.0, abs(fd)), (name, fd)
        assert inp["cfg"].loss != "tip" or L > 0
