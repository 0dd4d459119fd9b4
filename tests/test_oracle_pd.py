"""Pins for oracle/pd.py (forward) against closed forms, invariants and the paper's claims."""
import dataclasses

import numpy as np
import pytest

from oracle import fem, pd
from pd_inputs import get_config, make_inputs


def _scene(name, **kw):
    cfg = get_config(name, **kw)
    inp = make_inputs(cfg)
    return pd.scene_from_inputs(inp), inp


def test_y_closed_forms():
    sc, inp = _scene("c1")
    x = inp["q0"][0]
    zero = np.zeros_like(x)
    sc0 = dataclasses.replace(sc, gravity=np.zeros(3))
    np.testing.assert_array_equal(sc0.y(x, zero, zero), x)          # v=0, f=0 -> y = x
    v = np.random.default_rng(0).standard_normal(x.shape)
    # f_ext = -M g z-hat (gravity) -> y = x + h v - h^2 g z-hat (SPEC assemble_y)
    y = sc.y(x, v, zero)
    expect = x + sc.h * v
    expect[2::3] -= sc.h ** 2 * 9.81
    np.testing.assert_allclose(y, expect, rtol=0, atol=1e-15)


def test_grad_g_matches_finite_difference_of_g():
    # grad g = M/h^2 (x - y) + sum w G^T (Gx - z*) (eq:gradient; dz*/dx dropped by the
    # envelope theorem) must be the derivative of g (eq:opt).
    sc, inp = _scene("c1")
    rng = np.random.default_rng(1)
    x = inp["q0"][0] + 1e-3 * rng.standard_normal(sc.N)
    y = sc.y(x, np.zeros(sc.N), np.zeros(sc.N))
    w = sc.w_of(1e5)
    g0, gg = sc.objective(x, y, w)
    d = rng.standard_normal(sc.N)
    eps = 1e-7
    gp, _ = sc.objective(x + eps * d, y, w)
    gm, _ = sc.objective(x - eps * d, y, w)
    assert abs((gp - gm) / (2 * eps) - gg @ d) < 1e-6 * abs(gg @ d) + 1e-9


def test_rigid_rotation_zero_elastic_force():
    # BASELINE.json oracle self-check: zero elastic force under rigid rotation.
    sc, inp = _scene("c5s")
    from scipy.spatial.transform import Rotation
    Q = Rotation.from_rotvec([0.4, 1.2, -0.7]).as_matrix()
    x = (inp["rest"] @ Q.T + np.array([0.1, 0.2, 0.3])).ravel()
    z = sc.local_step(x, np.ones(sc.m))        # r = 1: ||Fm|| = 1 is on the muscle sphere
    E, gE = sc.elastic_terms(z, sc.w_of(1e5))
    assert E < 1e-20
    assert np.abs(gE).max() < 1e-9


def test_rest_without_gravity_stays_at_rest():
    # BASELINE.json self-check / SPEC step_pd example: exact fixed point after one iteration.
    sc, inp = _scene("c2s")
    sc = dataclasses.replace(sc, gravity=np.zeros(3))
    x = inp["rest"].ravel()
    zero = np.zeros_like(x)
    r = sc.step(x, zero, zero, sc.w_of(1e5), None, tol=1e-12, fixed_iter=1)
    np.testing.assert_allclose(r["x"], x, atol=1e-15)
    np.testing.assert_allclose(r["v"], 0, atol=1e-12)


def test_pd_objective_monotone():
    # PD local-global is block-coordinate descent on g: g never increases.
    sc, inp = _scene("c2s")
    x = inp["q0"][0]
    y = sc.y(x, inp["v0"][0] * 5, np.zeros(sc.N))
    w = sc.w_of(1e5)
    cons = ~sc.free
    gprev, _ = sc.objective(x, y, w)
    for _ in range(30):
        x = sc.pd_iteration(x, y, w, None, cons)
        g, _ = sc.objective(x, y, w)
        assert g <= gprev + 1e-13 * abs(gprev)
        gprev = g


def test_pd_and_newton_reach_the_same_minimiser():
    # The paper's PD iteration and Newton solve the same eq:time_integration.
    for name in ("c2s", "c5s"):
        sc, inp = _scene(name)
        x = inp["q0"][0]
        act = None if inp["act"] is None else inp["act"][0, 0]
        y = sc.y(x, inp["v0"][0], inp["f_ext"][0])
        w = sc.w_of(inp["youngs"][0])
        cons = ~sc.free
        xa, _, ra = sc.pd_solve(x, y, w, act, cons, tol=1e-12)
        xb, _, rb = sc.newton_solve(x, y, w, act, cons, tol=1e-13)
        assert ra <= 1e-12 and rb <= 1e-13
        assert np.linalg.norm(xa - xb) <= 1e-10 * np.linalg.norm(xb)


def test_dirichlet_exact_and_free_fall_ballistics():
    # Dirichlet DoFs keep their rest values exactly.
    sc, inp = _scene("c2s")
    tr = pd.forward(sc, inp["q0"][0], inp["v0"][0], inp["f_ext"][0], 1e5, steps=3, tol=1e-12)
    fx = inp["fixed_dofs"]
    np.testing.assert_array_equal(tr["q"][:, fx], np.broadcast_to(inp["q0"][0][fx], (4, len(fx))))
    # No Dirichlet, no contact: the centre of mass follows backward Euler ballistics exactly
    # (internal forces sum to zero): v_c' = v_c + h g, x_c' = x_c + h v_c' (SPEC step_pd example).
    sc, inp = _scene("c2s", dirichlet="none")
    rng = np.random.default_rng(3)
    q0 = inp["q0"][0] + 1e-3 * rng.standard_normal(sc.N)
    v0 = 0.1 * rng.standard_normal(sc.N)
    tr = pd.forward(sc, q0, v0, np.zeros(sc.N), 1e5, steps=3, tol=1e-13)
    M = sc.mass
    for i in range(3):
        vc = (M * tr["v"][i]).reshape(-1, 3).sum(0) / M[0::3].sum()
        vc1 = (M * tr["v"][i + 1]).reshape(-1, 3).sum(0) / M[0::3].sum()
        np.testing.assert_allclose(vc1, vc + sc.h * sc.gravity, atol=1e-9)
    # Momentum conservation with f_ext = 0 and no gravity (SPEC invariant).
    sc0 = dataclasses.replace(sc, gravity=np.zeros(3))
    tr = pd.forward(sc0, q0, v0, np.zeros(sc.N), 1e5, steps=3, tol=1e-13)
    P = [(M * v).reshape(-1, 3).sum(0) for v in tr["v"]]
    np.testing.assert_allclose(P[-1], P[0], atol=1e-12)


def test_c1_is_exactly_ten_pd_iterations():
    # c1: 10 local-global iterations per step from x^0 = x_i (reading §8c.6).
    sc, inp = _scene("c1")
    x, v = inp["q0"][0], inp["v0"][0]
    r = sc.step(x, v, inp["f_ext"][0], sc.w_of(1e5), None, tol=0, fixed_iter=10)
    y = sc.y(x, v, inp["f_ext"][0])
    xk = x.copy()
    for _ in range(10):
        xk = sc.pd_iteration(xk, y, sc.w_of(1e5), None, ~sc.free)
    np.testing.assert_array_equal(r["x"], xk)
    assert r["res"] > 1e-6        # far from converged, as the survey measured
