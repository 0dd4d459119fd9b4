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


# ----------------------------------------------------------------- volume preservation
def _rand_F(n, seed, scale=0.3):
    rng = np.random.default_rng(seed)
    F = np.eye(3) + scale * rng.standard_normal((n, 3, 3))
    return F[np.linalg.det(F) > 0.05]


def test_volume_projection_is_the_closest_det1_matrix():
    # D = U diag(Sigma + d*) V^T has det D = 1, and no det-1 neighbour D exp(eps X), tr X = 0, is closer
    from scipy.linalg import expm
    F = _rand_F(200, 0)
    D = energy.volume_project(F)[0]
    assert np.abs(np.linalg.det(D) - 1).max() < 1e-13
    rng = np.random.default_rng(1)
    dist = np.linalg.norm(F - D, axis=(1, 2))
    for _ in range(20):
        X = rng.standard_normal(F.shape)
        X -= np.trace(X, axis1=1, axis2=2)[:, None, None] * np.eye(3) / 3
        for eps in (1e-2, 1e-3):
            Dp = np.array([D[i] @ expm(eps * X[i]) for i in range(len(F))])
            assert np.all(np.linalg.norm(F - Dp, axis=(1, 2)) >= dist - 1e-14)


def test_volume_projection_special_cases():
    # fixed point on the manifold; rotation invariance D(Q F) = Q D(F); uniform scaling F = a I -> D = I
    F = _rand_F(50, 2)
    D = energy.volume_project(F)[0]
    np.testing.assert_allclose(energy.volume_project(D)[0], D, atol=1e-13)
    from scipy.spatial.transform import Rotation
    Q = Rotation.random(len(F), random_state=3).as_matrix()
    np.testing.assert_allclose(energy.volume_project(Q @ F)[0], Q @ D, atol=1e-12)
    for a in (0.5, 1.0, 2.0):
        np.testing.assert_allclose(energy.volume_project(a * np.eye(3)[None])[0][0], np.eye(3), atol=1e-14)
    # diagonal F: the KKT point in closed form, z_i (z_i - s_i) = -lam for all i
    s = np.array([[1.2, 0.9, 0.8], [0.7, 0.7, 1.5]])
    d, lam = energy.volume_kkt(s)
    z = s + d
    np.testing.assert_allclose(z * (z - s), -lam[:, None] * np.ones(3), atol=1e-13)
    np.testing.assert_allclose(np.prod(z, 1), 1.0, atol=1e-14)


def test_volume_kkt_jacobian_vs_finite_difference():
    # eq:vol_kkt: d(Sigma + d*)/dSigma against central differences of the KKT solution
    s = np.array([[1.2, 0.9, 0.8], [1.0, 1.0, 1.0], [0.6, 1.3, 1.1]])
    d, lam = energy.volume_kkt(s)
    J = energy.volume_dg(s, d, lam)
    eps = 1e-6
    for k in range(3):
        e = np.zeros(3)
        e[k] = eps
        gp = s + e + energy.volume_kkt(s + e)[0]
        gm = s - e + energy.volume_kkt(s - e)[0]
        np.testing.assert_allclose(J[:, :, k], (gp - gm) / (2 * eps), rtol=1e-7, atol=1e-9)


def test_volume_derivative_vs_finite_difference():
    # full dD/dF (KKT Jacobian + SVD chain rule) against central differences, including a repeated singular
    # value (F = diag(1.1, 0.9, 0.9) rotated) where the ratio (g_i - g_j)/(s_i - s_j) takes its limit
    from scipy.spatial.transform import Rotation
    F = _rand_F(100, 4)
    Q = Rotation.random(2, random_state=5).as_matrix()
    F = np.concatenate([F, (Q[0] @ np.diag([1.1, 0.9, 0.9]) @ Q[1])[None]], 0)
    rng = np.random.default_rng(6)
    dF = rng.standard_normal(F.shape)
    eps = 1e-6
    fd = (energy.volume_project(F + eps * dF)[0] - energy.volume_project(F - eps * dF)[0]) / (2 * eps)
    an = energy.volume_derivative(F, dF)
    err = np.linalg.norm(fd - an, axis=(1, 2)) / np.linalg.norm(fd, axis=(1, 2))
    assert err.max() < 1e-6, err.max()
