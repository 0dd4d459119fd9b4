"""Oracle PD projections and their derivatives (test infrastructure only).

Corotated: E = (w/2)||F - R||_F^2, R the rotation closest to F,
M = SO(3).  R "is computed from the polar decomposition of F"; the
oracle takes it from an SVD (numpy LAPACK), flipping the smallest singular
direction when det(U V^T) < 0 (reading §8c.5).  The GPU path uses a different
algorithm (Newton iteration), so agreement is evidence, not shared error.

dR/dF ("deriving the gradients of the rotation matrix in the polar
decomposition"): with F = R S, R^T dF - dF^T R = [w]x S + S [w]x = [(tr S I - S) w]x,
dR = R [w]x.  Eigenvalues of tr(S) I - S are floored at 1e-6 * max sigma (§8c.5).

Muscle: "projects Fm onto a spherical manifold ||p|| = r":
p = r Fm/||Fm|| (reading §8c.4), ||Fm|| = 0 -> p = r m.
"""
from __future__ import annotations

import numpy as np

CLAMP = 1e-6


def skew(w):
    """[w]x for w [..., 3]."""
    z = np.zeros(w.shape[:-1])
    return np.stack([
        np.stack([z, -w[..., 2], w[..., 1]], -1),
        np.stack([w[..., 2], z, -w[..., 0]], -1),
        np.stack([-w[..., 1], w[..., 0], z], -1)], -2)


def vee(W):
    """Inverse of skew for a skew-symmetric W: (W21, W02, W10)."""
    return np.stack([W[..., 2, 1], W[..., 0, 2], W[..., 1, 0]], -1)


def polar_svd(F):
    """Rotation part R and symmetric part S = R^T F of F [..., 3, 3] via SVD.

    Returns (R, S, V, s): S = V diag(s) V^T with s = (s1, s2, +-s3) sign-corrected."""
    U, s, Vt = np.linalg.svd(F)
    d = np.sign(np.linalg.det(U @ Vt))
    s = s.copy()
    s[..., 2] *= d
    U = U.copy()
    U[..., :, 2] *= d[..., None]
    R = U @ Vt
    V = np.swapaxes(Vt, -1, -2)
    S = V @ (s[..., :, None] * Vt)
    return R, S, V, s


def polar_derivative(R, V, s, dF):
    """dR[dF] = R [w]x,  (tr S I - S) w = vee(R^T dF - dF^T R), eigen-clamped."""
    W = np.swapaxes(R, -1, -2) @ dF
    W = W - np.swapaxes(W, -1, -2)
    rhs = vee(W)
    tr = s.sum(-1, keepdims=True)
    e = tr - s                                   # eigenvalues s_j + s_k
    floor = CLAMP * np.abs(s).max(-1, keepdims=True)
    e = np.maximum(e, floor)
    Vt = np.swapaxes(V, -1, -2)
    w = (V @ ((Vt @ rhs[..., None])[..., 0] / e)[..., None])[..., 0]
    return R @ skew(w)


def polar_jacobian(F):
    """J [..., 9, 9] with J[3i+j, 3k+l] = dR_ij / dF_kl (columns from unit dF)."""
    R, S, V, s = polar_svd(F)
    cols = []
    for k in range(9):
        E = np.zeros(F.shape)
        E[..., k // 3, k % 3] = 1.0
        cols.append(polar_derivative(R, V, s, E).reshape(F.shape[:-2] + (9,)))
    return np.stack(cols, -1), R


def muscle_project(Fm, r, m):
    """p = r Fm/||Fm||; ||Fm|| = 0 -> r m."""
    nrm = np.linalg.norm(Fm, axis=-1, keepdims=True)
    safe = np.where(nrm > 0, nrm, 1.0)
    n_hat = np.where(nrm > 0, Fm / safe, np.broadcast_to(np.asarray(m, float), Fm.shape))
    return np.asarray(r)[..., None] * n_hat, n_hat, nrm[..., 0]


def muscle_jacobian(Fm, r, m):
    """dp/d(Fm) = (r/||Fm||)(I - n n^T)."""
    p, n_hat, nrm = muscle_project(Fm, r, m)
    scale = np.where(nrm > 0, np.asarray(r) / np.where(nrm > 0, nrm, 1.0), 0.0)
    J = scale[..., None, None] * (np.eye(3) - n_hat[..., :, None] * n_hat[..., None, :])
    return J, p, n_hat
