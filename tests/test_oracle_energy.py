"""Pins for oracle/energy.py: polar decomposition, its derivative, muscle projection."""
import numpy as np
import scipy.linalg
from scipy.spatial.transform import Rotation

from oracle import energy


def test_polar_special_cases():
    # SPEC project_corotated examples: F = I -> I; F = Q -> Q; F = diag(2,.5,1) -> I.
    R, *_ = energy.polar_svd(np.eye(3)[None])
    np.testing.assert_allclose(R[0], np.eye(3), atol=1e-15)
    Q = Rotation.from_rotvec([0.3, -1.1, 0.4]).as_matrix()
    R, *_ = energy.polar_svd(Q[None])
    np.testing.assert_allclose(R[0], Q, atol=1e-14)
    R, *_ = energy.polar_svd(np.diag([2.0, 0.5, 1.0])[None])
    np.testing.assert_allclose(R[0], np.eye(3), atol=1e-15)


def test_polar_matches_scipy_polar_and_is_rotation():
    rng = np.random.default_rng(0)
    F = rng.standard_normal((2000, 3, 3))
    R, S, V, s = energy.polar_svd(F)
    np.testing.assert_allclose(R @ np.swapaxes(R, 1, 2), np.broadcast_to(np.eye(3), R.shape), atol=1e-13)
    np.testing.assert_allclose(np.linalg.det(R), 1.0, atol=1e-13)
    np.testing.assert_allclose(S, np.swapaxes(S, 1, 2), atol=1e-13)
    np.testing.assert_allclose(R @ S, F, atol=1e-13)
    pos = np.linalg.det(F) > 0
    for k in np.nonzero(pos)[0][:300]:
        U, P = scipy.linalg.polar(F[k])        # library routine: for det F > 0, U in SO(3)
        np.testing.assert_allclose(R[k], U, atol=1e-12)


def test_polar_is_closest_rotation_for_inverted_F():
    # det F < 0: R must minimise ||F - Q||_F over SO(3) (the PD projection onto M = SO(3)).
    rng = np.random.default_rng(1)
    Qs = Rotation.random(20000, random_state=2).as_matrix()
    for _ in range(10):
        F = rng.standard_normal((3, 3))
        if np.linalg.det(F) > 0:
            F[:, 0] *= -1
        R, *_ = energy.polar_svd(F[None])
        best = np.min(np.sum((F[None] - Qs) ** 2, axis=(1, 2)))
        assert np.sum((F - R[0]) ** 2) <= best + 1e-12
        assert abs(np.linalg.det(R[0]) - 1) < 1e-13


def test_polar_derivative_vs_finite_difference():
    rng = np.random.default_rng(3)
    F = np.eye(3) + 0.3 * rng.standard_normal((50, 3, 3))
    dF = rng.standard_normal((50, 3, 3))
    R, S, V, s = energy.polar_svd(F)
    dR = energy.polar_derivative(R, V, s, dF)
    eps = 1e-6
    Rp, *_ = energy.polar_svd(F + eps * dF)
    Rm, *_ = energy.polar_svd(F - eps * dF)
    np.testing.assert_allclose(dR, (Rp - Rm) / (2 * eps), atol=5e-8)


def test_polar_derivative_at_identity():
    # SPEC: at F = I a skew dF maps to itself, a symmetric dF to zero.
    rng = np.random.default_rng(4)
    K = rng.standard_normal((3, 3))
    K = K - K.T
    Sym = rng.standard_normal((3, 3))
    Sym = Sym + Sym.T
    R, S, V, s = energy.polar_svd(np.eye(3)[None])
    np.testing.assert_allclose(energy.polar_derivative(R, V, s, K[None])[0], K, atol=1e-14)
    np.testing.assert_allclose(energy.polar_derivative(R, V, s, Sym[None])[0], 0, atol=1e-14)


def test_muscle_projection():
    m = np.array([1.0, 0, 0])
    p, n, nrm = energy.muscle_project(np.array([1.0, 0, 0])[None], np.array([0.5]), m)
    np.testing.assert_allclose(p[0], [0.5, 0, 0])
    rng = np.random.default_rng(5)
    Fm = rng.standard_normal(3)
    p, *_ = energy.muscle_project(Fm[None], np.array([np.linalg.norm(Fm)]), m)
    np.testing.assert_allclose(p[0], Fm, atol=1e-15)
    # p minimises ||Fm - q|| over the sphere ||q|| = r (sampling oracle, SPEC project_muscle).
    r = 0.9
    q = rng.standard_normal((100000, 3))
    q = r * q / np.linalg.norm(q, axis=1, keepdims=True)
    p, *_ = energy.muscle_project(Fm[None], np.array([r]), m)
    assert np.sum((Fm - p[0]) ** 2) <= np.min(np.sum((Fm - q) ** 2, axis=1)) + 1e-12
    # Jacobian vs central FD
    J, *_ = energy.muscle_jacobian(Fm[None], np.array([r]), m)
    Jfd = np.zeros((3, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = 1e-6
        Jfd[:, k] = (energy.muscle_project((Fm + e)[None], np.array([r]), m)[0][0]
                     - energy.muscle_project((Fm - e)[None], np.array([r]), m)[0][0]) / 2e-6
    np.testing.assert_allclose(J[0], Jfd, atol=1e-8)
