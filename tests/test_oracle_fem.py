"""Pins for oracle/fem.py against things the paper and mathematics fix (not the oracle itself)."""
import os

import numpy as np
import pytest

from oracle import fem
from pd_inputs import grid_mesh, get_config, make_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append([int(t) for t in line.split()])
    return rows


def test_cantilever_counts_match_paper():
    # PAPER.md:525 / Table tab:setting: 32x8x8 -> 2048 elements, 8019 DoFs, 243 Dirichlet.
    for nx, ny, nz, m, ndof, ndir in _golden("cantilever_mesh_counts.txt"):
        cfg = get_config("c3", counts=(nx, ny, nz))
        inp = make_inputs(cfg, batch=1, steps=1)
        assert inp["n_elems"] == m
        assert 3 * inp["n_nodes"] == ndof
        assert len(inp["fixed_dofs"]) == ndir


def test_tiny_counts():
    for nx, ny, nz, m, n, ndof in _golden("tiny_cantilever_counts.txt"):
        rest, hex8 = grid_mesh((nx, ny, nz), 0.01)
        assert hex8.shape == (m, 8) and rest.shape == (n, 3) and 3 * n == ndof
        assert all(len(set(h)) == 8 for h in hex8)


def _trilinear(xe, xi):
    """Independent trilinear interpolant x(xi) = sum_a N_a(xi) x_a (N written out, no dN)."""
    out = np.zeros(3)
    for a in range(8):
        s, t, u = 2 * (a & 1) - 1, 2 * ((a >> 1) & 1) - 1, 2 * ((a >> 2) & 1) - 1
        N = (1 + s * xi[0]) * (1 + t * xi[1]) * (1 + u * xi[2]) / 8.0
        out += N * xe[a]
    return out


def test_F_matches_finite_difference_of_interpolant():
    # F = dx/dX of the trilinear interpolant at each Gauss point (reading §8c.1),
    # computed here by central differences in reference coordinates, X = X0 + dx (xi+1)/2.
    rng = np.random.default_rng(0)
    dx = 0.01
    rest, hex8 = grid_mesh((1, 1, 1), dx)
    x = rest.ravel() + 0.002 * rng.standard_normal(24)
    F = fem.deformation_gradients(x, hex8, dx)[0]
    xe = x.reshape(8, 3)
    g = 1 / np.sqrt(3)
    for q in range(8):
        xi = np.array([(2 * (q & 1) - 1) * g, (2 * ((q >> 1) & 1) - 1) * g, (2 * ((q >> 2) & 1) - 1) * g])
        J = np.zeros((3, 3))
        for j in range(3):
            e = np.zeros(3)
            e[j] = 1e-6
            J[:, j] = (_trilinear(xe, xi + e) - _trilinear(xe, xi - e)) / 2e-6 * (2.0 / dx)
        np.testing.assert_allclose(F[q], J, atol=1e-8)


def test_rest_identity_and_affine_reproduction():
    # SPEC mesh invariants: rest -> F = I; x = Aff X + b -> F = Aff exactly.
    rng = np.random.default_rng(1)
    rest, hex8 = grid_mesh((3, 2, 2), 0.01)
    F = fem.deformation_gradients(rest.ravel(), hex8, 0.01)
    np.testing.assert_allclose(F, np.broadcast_to(np.eye(3), F.shape), atol=1e-12)
    Aff = rng.standard_normal((3, 3))
    b = rng.standard_normal(3)
    F = fem.deformation_gradients((rest @ Aff.T + b).ravel(), hex8, 0.01)
    np.testing.assert_allclose(F, np.broadcast_to(Aff, F.shape), atol=1e-11)


def test_lumped_mass_examples():
    # SPEC lumped_mass examples: single cube dx=1 rho=1 -> 0.125; 2x1x1 -> shared 0.25.
    rest, hex8 = grid_mesh((1, 1, 1), 1.0)
    np.testing.assert_allclose(fem.lumped_mass(hex8, 8, 1.0, 1.0), 0.125)
    rest, hex8 = grid_mesh((2, 1, 1), 1.0)
    m = fem.lumped_mass(hex8, 12, 1.0, 1.0).reshape(12, 3)[:, 0]
    shared = rest[:, 0] == 1.0
    np.testing.assert_allclose(m[shared], 0.25)
    np.testing.assert_allclose(m[~shared], 0.125)
    rest, hex8 = grid_mesh((4, 3, 2), 0.01)
    M = fem.lumped_mass(hex8, rest.shape[0], 0.01, 1e3)
    assert abs(M[0::3].sum() - 1e3 * 24 * 1e-6) < 1e-15


def _dirichlet_energy_3pt(xe, dx, w):
    """(w/2) * integral over the cube of ||dx/dX||_F^2 with a 3-point Gauss rule per axis and
    gradients by finite differences of the independent interpolant (exact for trilinear)."""
    pts = np.array([-np.sqrt(0.6), 0.0, np.sqrt(0.6)])
    wts = np.array([5 / 9, 8 / 9, 5 / 9])
    tot = 0.0
    for i, a in enumerate(pts):
        for j, b in enumerate(pts):
            for k, c in enumerate(pts):
                xi = np.array([a, b, c])
                J = np.zeros((3, 3))
                for d in range(3):
                    e = np.zeros(3)
                    e[d] = 1e-5
                    J[:, d] = (_trilinear(xe, xi + e) - _trilinear(xe, xi - e)) / 2e-5 * (2.0 / dx)
                tot += wts[i] * wts[j] * wts[k] * np.sum(J * J)
    return 0.5 * w * tot * (dx / 2) ** 3


def test_element_stiffness_is_exact_integral():
    # A's element block sum_q w V_q G_q^T G_q must equal the exact integral of the
    # quadratic form (8-point Gauss is exact for products of trilinear gradients).
    rng = np.random.default_rng(2)
    dx, w = 0.01, 3.7
    K = fem.element_stiffness(dx, w)
    for _ in range(3):
        xe = rng.standard_normal((8, 3)) * dx
        assert abs(0.5 * xe.ravel() @ K @ xe.ravel() - _dirichlet_energy_3pt(xe, dx, w)) \
            < 1e-6 * abs(_dirichlet_energy_3pt(xe, dx, w))


def test_A_properties():
    # A = M/h^2 + sum w G^T G: zero weight -> M/h^2; translations are in the
    # stiffness null space; A is SPD.
    inp = make_inputs(get_config("c1"))
    rest, hex8 = inp["rest"], inp["hex8"]
    n = rest.shape[0]
    M = fem.lumped_mass(hex8, n, 0.01, 1e3)
    A0 = fem.assemble_A(M, hex8, n, 0.01, 0.01, 0.0).toarray()
    np.testing.assert_allclose(A0, np.diag(M / 1e-4), atol=1e-12)
    A = fem.assemble_A(M, hex8, n, 0.01, 0.01, 6.9e4).toarray()
    c = np.tile([0.3, -1.0, 2.0], n)
    np.testing.assert_allclose(A @ c, M / 1e-4 * c, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(A, A.T, atol=1e-9)
    assert np.linalg.eigvalsh(A).min() > 0
