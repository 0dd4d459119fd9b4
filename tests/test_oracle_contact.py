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
