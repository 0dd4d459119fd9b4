"""Pins for the oracle's contact handling (Alg. 1 frictionless + constrained global solve)."""
import itertools

import numpy as np
import scipy.sparse.linalg as spla

from oracle import adjoint, pd
from pd_inputs import get_config, make_inputs


def test_alg2_and_capacitance_equal_direct_constrained_solve():
    # Alg. 2 with the Woodbury identity eq:woodbury, restated here from the
    # paper, and the capacitance form both reproduce the oracle's reduced direct
    # solve of eq:dirichlet/eq:complement when the pinned values are 0 (frictionless pins on z=0).
    inp = make_inputs(get_config("c4s"))
    sc = pd.scene_from_inputs(inp)
    A = sc.A(sc.w_of(1e5)).toarray()
    N = sc.N
    rng = np.random.default_rng(0)
    d = rng.standard_normal(N)
    Ci = np.sort(rng.choice(3 * inp["contact_nodes"] + 2, size=7, replace=False))
    # direct (the oracle's definition)
    cons = np.zeros(N, bool)
    cons[Ci] = True
    x = np.zeros(N)
    x[~cons] = np.linalg.solve(A[~cons][:, ~cons], d[~cons])
    # Alg. 2
    Ainv = np.linalg.inv(A)
    I_C = np.eye(N)[:, Ci]
    B1 = Ainv @ I_C
    B2 = I_C - B1 @ A[np.ix_(Ci, Ci)]
    B3 = np.hstack([B1, B2])
    # V P^T fetched from A: rows [A_{C, Cbar} (zero on C columns); I on C columns]
    VPt = np.zeros((2 * len(Ci), N))
    VPt[:len(Ci)] = A[Ci]
    VPt[:len(Ci)][:, Ci] = 0.0
    VPt[len(Ci):] = I_C.T
    B4 = np.eye(2 * len(Ci)) - VPt @ B3
    y1 = np.linalg.solve(A, d)
    y2 = np.concatenate([d @ B2, d @ B1])
    y3 = np.linalg.solve(B4, y2)
    xa = y1 + B3 @ y3
    xa[Ci] = 0.0
    np.testing.assert_allclose(xa, x, atol=1e-12 * np.abs(x).max())
    # capacitance: lambda = S^{-1}(0 - y1_C), x = y1 + A^{-1} I_C lambda
    S = Ainv[np.ix_(Ci, Ci)]
    lam = np.linalg.solve(S, -y1[Ci])
    xc = y1 + B1 @ lam
    np.testing.assert_allclose(xc, x, atol=1e-12 * np.abs(x).max())
    np.testing.assert_allclose(lam, (A @ x - d)[Ci], rtol=1e-9)


def test_contact_complementarity_and_impulse_balance():
    cfg = get_config("c4s")
    inp = make_inputs(cfg)
    sc = pd.scene_from_inputs(inp)
    w = sc.w_of(1e5)
    x, v = inp["q0"][0], inp["v0"][0]
    cand = sc.normal_dofs(sc.contact_nodes)
    seen = 0
    for i in range(cfg.steps):
        r = sc.step(x, v, inp["f_ext"][0], w, None, tol=1e-12)
        assert not r["flag"]
        act = r["active"]
        z = r["x"][cand]
        assert np.all(z >= -1e-6 * cfg.dx)                     # non-penetration (eq:lcp_normal)
        assert np.all(z[act] == 0.0)                           # pinned at the plane
        assert np.all(r["lam"][act] > 0)                       # compressive force on V_i
        # total contact impulse = momentum change minus gravity impulse (internal forces sum to 0)
        _, gg = sc.objective(r["x"], r["y"], w)
        lhs = gg[cand[act]].sum()
        rhs = (sc.mass / sc.h ** 2 * (r["x"] - r["y"]))[2::3].sum()
        assert abs(lhs - rhs) < 1e-9 * max(1.0, abs(rhs))
        seen += act.sum()
        x, v = r["x"], r["v"]
    assert seen > 0


def test_active_set_is_the_unique_kkt_point_by_enumeration():
    # Brute force over all 2^9 pinned sets of a 2x2x1 block (9 bottom candidates): the oracle's
    # final set is the only one whose solution is feasible (z >= 0) with lambda >= 0 (KKT of
    # min g s.t. z_j >= 0, eq:lcp_normal), and it has the lowest g among feasible sets.
    cfg = get_config("c4s", counts=(2, 2, 1), lift=0.0, max_tilt_deg=0.0)
    inp = make_inputs(cfg)
    sc = pd.scene_from_inputs(inp)
    w = sc.w_of(1e5)
    x = inp["q0"][0]
    v = np.zeros(sc.N)
    v[2::3] = -0.05
    v[0::3] = 0.02 * (inp["rest"][:, 1] - 0.01) / 0.01       # a little shear
    r = sc.step(x, v, np.zeros(sc.N), w, None, tol=1e-13)
    cand = sc.normal_dofs(sc.contact_nodes)
    y = r["y"]
    kkt = []
    for bits in itertools.product([False, True], repeat=len(cand)):
        act = np.array(bits)
        cons = ~sc.free
        cons[cand[act]] = True
        x0 = x.copy()
        x0[cand[act]] = 0.0
        xs, _, res = sc.newton_solve(x0, y, w, None, cons, tol=1e-13)
        g, gg = sc.objective(xs, y, w)
        if np.all(xs[cand] >= -1e-12) and np.all(gg[cand[act]] >= -1e-9):
            kkt.append((g, act))
    assert len(kkt) == 1
    np.testing.assert_array_equal(kkt[0][1], r["active"])
    assert r["active"].any()


def _sticky_block():
    """A 3x2x2 block standing on z = 0 under gravity, small horizontal push: every bottom node is active
    (lambda > 0) at every step, so the active set is locally constant and finite differences are valid."""
    from oracle import pd
    from pd_inputs import grid_mesh
    rest, hex8 = grid_mesh((3, 2, 2), 0.01)
    cand = np.nonzero(rest[:, 2] == 0.0)[0]
    sc = pd.Scene(rest=rest, hex8=hex8, dx=0.01, density=1e3, h=0.01, youngs=1e5, poisson=0.45,
                  gravity=np.array([0.0, 0.0, -9.81]), fixed_dofs=np.zeros(0, np.int64), contact_nodes=cand,
                  contact_mode="sticky")
    rng = np.random.default_rng(3)
    N = rest.size
    f = 0.002 * rng.standard_normal(N)                    # small horizontal push
    f[2::3] = 0.0
    v0 = np.zeros(N)
    return sc, rest.ravel().copy(), v0, f, rng


def test_sticky_nodes_do_not_move():
    # infinite friction: an active node keeps x_i in all three DoFs, its velocity is exactly 0
    from oracle import pd
    sc, q0, v0, f, _ = _sticky_block()
    tr = pd.forward(sc, q0, v0, f, 1e5, steps=3, tol=1e-13)
    cand = np.asarray(sc.contact_nodes)
    for i in range(3):
        act = cand[tr["active"][i]]
        assert act.size == cand.size                      # the standing block presses every bottom node
        pins = (3 * act[:, None] + np.arange(3)).ravel()
        assert np.array_equal(tr["q"][i + 1][pins], tr["q"][i][pins])
        assert np.all(tr["v"][i + 1][pins] == 0.0)


def test_sticky_gradients_vs_central_fd():
    # the adjoint with the pinned-value term dL/dx_{i,a} += b_a - (A_N u)_a against central FD, including a
    # DoF of a pinned node (where only that term carries the gradient)
    from oracle import adjoint, pd
    sc, q0, v0, f, rng = _sticky_block()
    N = q0.size
    cq, cv = rng.standard_normal(N), rng.standard_normal(N)

    def L(q, v):
        tr = pd.forward(sc, q, v, f, 1e5, steps=2, tol=1e-13)
        return float(cq @ tr["q"][-1] + cv @ tr["v"][-1]), tr

    _, tr = L(q0, v0)
    g = adjoint.backward(sc, tr, 1e5, cq, cv)
    pinned_dof = 3 * int(sc.contact_nodes[1]) + 0
    free_dof = 3 * int(np.nonzero(q0[2::3] > 0.015)[0][0]) + 1
    eps = 1e-7
    for k in (pinned_dof, free_dof):
        qp, qm = q0.copy(), q0.copy()
        qp[k] += eps
        qm[k] -= eps
        fd = (L(qp, v0)[0] - L(qm, v0)[0]) / (2 * eps)
        assert abs(fd - g["dq0"][k]) <= 1e-5 * max(1.0, abs(fd)), (k, fd, g["dq0"][k])
    # v0 of a pinned node has no effect (x_1 = x_0 there): its gradient is exactly (M/h) u_a = 0
    assert g["dv0"][pinned_dof] == 0.0


# ---- general contact plane n . x = d ("phi is a linear function and n ... a constant vector") ----
def test_plane_offset_is_a_translation():
    # The plane z = d is the plane z = 0 with the whole scene lifted by d: positions shift by d e_z, velocities,
    # active sets, iteration counts and every gradient are unchanged (the PD energy depends on x only through F).
    from oracle import adjoint
    inp = make_inputs(get_config("c4s"))
    sc0 = pd.scene_from_inputs(inp)
    d = 0.013
    sc1 = pd.scene_from_inputs(inp)
    sc1.plane_d = d
    q0, v0, f = inp["q0"][0], inp["v0"][0], inp["f_ext"][0]
    lift = np.zeros_like(q0)
    lift[2::3] = d
    t0 = pd.forward(sc0, q0, v0, f, 1e5, steps=inp["T"], tol=1e-13)
    t1 = pd.forward(sc1, q0 + lift, v0, f, 1e5, steps=inp["T"], tol=1e-13)
    np.testing.assert_array_equal(t0["active"], t1["active"])
    assert t0["active"].any()
    for i in range(inp["T"] + 1):
        assert np.linalg.norm(t1["q"][i] - lift - t0["q"][i]) <= 1e-11 * np.linalg.norm(t0["q"][i])
        assert np.linalg.norm(t1["v"][i] - t0["v"][i]) <= 1e-8 * max(1e-3, np.linalg.norm(t0["v"][i]))
    g0 = adjoint.backward(sc0, t0, 1e5, inp["c_q"][0], inp["c_v"][0])
    g1 = adjoint.backward(sc1, t1, 1e5, inp["c_q"][0], inp["c_v"][0])
    for k in ("dq0", "dv0", "dfext"):
        assert np.linalg.norm(g1[k] - g0[k]) <= 1e-7 * np.linalg.norm(g0[k]), k
    assert abs(g1["dE"] - g0["dE"]) <= 1e-7 * abs(g0["dE"])


def test_tilted_plane_kkt_in_world_coordinates():
    # c4p: the tilted plate falls on a 20-degree plane n . x = d.  Checked with the WORLD-frame objective (no
    # change of coordinates): at every step x_{i+1} is the KKT point of min g s.t. n . x_j >= d (frictionless):
    # active nodes lie exactly on the plane, carry a compressive normal force n . grad_j g >= 0 and no tangential
    # force; every other free DoF has grad g = 0; no candidate penetrates beyond eps_phi.
    cfg = get_config("c4p")
    inp = make_inputs(cfg)
    sc = pd.scene_from_inputs(inp)
    w = sc.w_of(1e5)
    n = np.asarray(cfg.plane_n) / np.linalg.norm(cfg.plane_n)
    dd = cfg.plane_d / np.linalg.norm(cfg.plane_n)
    tr = pd.forward(sc, inp["q0"][0], inp["v0"][0], inp["f_ext"][0], 1e5, steps=cfg.steps, tol=1e-13)
    cand = np.asarray(sc.contact_nodes)
    touched, slid = 0, 0.0
    for i in range(cfg.steps):
        x, xi, vi = tr["q"][i + 1], tr["q"][i], tr["v"][i]
        y = sc.y(xi, vi, inp["f_ext"][0])
        _, gg = sc.objective(x, y, w)
        scale = np.linalg.norm(sc.mass / sc.h ** 2 * y)
        X, G = x.reshape(-1, 3), gg.reshape(-1, 3)
        act = tr["active"][i]
        phi = X[cand] @ n - dd
        assert np.all(np.abs(phi[act]) <= 1e-12)
        assert np.all(phi >= -pd.EPS_PHI_REL * cfg.dx)
        lam = G[cand] @ n
        assert np.all(lam[act] >= -1e-9 * scale)
        tang = G[cand] - lam[:, None] * n[None, :]
        assert np.abs(tang[act]).max(initial=0.0) <= 1e-9 * scale
        rest_free = np.ones(sc.n, bool)
        rest_free[cand[act]] = False
        assert np.abs(G[rest_free]).max() <= 1e-9 * scale
        touched += int(act.sum())
        both = act & tr["active"][i - 1] if i > 0 else np.zeros_like(act)
        if both.any():  # frictionless: pinned nodes may slide along the plane
            slid = max(slid, np.abs((X[cand[both]] - xi.reshape(-1, 3)[cand[both]]) @ (np.eye(3) - np.outer(n, n))).max())
    assert touched > 0 and slid > 1e-6


def test_tilted_plane_gradients_vs_central_fd():
    # dL/dq0, dL/dv0 and dL/dE of L = c_q . q_T + c_v . v_T through contact steps on the tilted plane, against
    # central differences of the world-frame forward (the active sets do not change under the perturbation).
    from oracle import adjoint
    cfg = get_config("c4p", steps=6)
    inp = make_inputs(cfg)
    sc = pd.scene_from_inputs(inp)
    q0, v0, f = inp["q0"][0], inp["v0"][0], inp["f_ext"][0]
    cq, cv = inp["c_q"][0], inp["c_v"][0]

    def run(q, v, E):
        t = pd.forward(sc, q, v, f, E, steps=cfg.steps, tol=1e-13)
        return float(cq @ t["q"][-1] + cv @ t["v"][-1]), t

    L0, tr = run(q0, v0, 1e5)
    assert tr["active"].any()
    g = adjoint.backward(sc, tr, 1e5, cq, cv)
    rng = np.random.default_rng(3)
    eps = 1e-7
    for _ in range(2):
        dq = rng.standard_normal(q0.size)
        dv = rng.standard_normal(q0.size)
        lp, tp = run(q0 + eps * dq, v0 + eps * dv, 1e5)
        lm, tm = run(q0 - eps * dq, v0 - eps * dv, 1e5)
        assert np.array_equal(tp["active"], tr["active"]) and np.array_equal(tm["active"], tr["active"])
        fd = (lp - lm) / (2 * eps)
        an = g["dq0"] @ dq + g["dv0"] @ dv
        assert abs(fd - an) <= 1e-5 * max(1.0, abs(fd)), (fd, an)
    lp, _ = run(q0, v0, 1e5 * (1 + 1e-6))
    lm, _ = run(q0, v0, 1e5 * (1 - 1e-6))
    fd = (lp - lm) / (2e-6 * 1e5)
    assert abs(fd - g["dE"]) <= 1e-5 * max(1e-3, abs(fd)), (fd, g["dE"])
