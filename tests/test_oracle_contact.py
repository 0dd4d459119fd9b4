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
