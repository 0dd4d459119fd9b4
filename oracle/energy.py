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

Volume preservation: E = (w/2)||F - D||_F^2, D the projection of F onto {det D = 1}: with the
(sign-corrected) SVD F = U Sigma V^T, d* = argmin ||d||^2 s.t. prod_i (d_i + Sigma_ii) = 1, solved
here by Newton's method on its KKT system d + lam grad c(d) = 0, c(d) = 0, and D = U Sigma_D V^T,
Sigma_D = diag(d* + Sigma).  Its Jacobian: dd*/dSigma from the differentiated KKT system eq:vol_kkt
(P:999-1006); the rotation parts by the chain rule through the SVD.
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


# ----------------------------------------------------------------- volume preservation
def _c_grad_hess(z):
    """c(d) = prod(z) - 1 with z = Sigma + d: gradient prod_{j != i} z_j and Hessian prod_{k != i,j} z_k (0 diag)."""
    g = np.stack([z[..., 1] * z[..., 2], z[..., 0] * z[..., 2], z[..., 0] * z[..., 1]], -1)
    H = np.zeros(z.shape[:-1] + (3, 3))
    H[..., 0, 1] = H[..., 1, 0] = z[..., 2]
    H[..., 0, 2] = H[..., 2, 0] = z[..., 1]
    H[..., 1, 2] = H[..., 2, 1] = z[..., 0]
    return g, H


def volume_kkt(s, tol=1e-13, max_iter=60):
    """d* and lam* of min ||d||^2 s.t. prod(s + d) = 1 for signed singular values s [..., 3], by
    Newton's method on the KKT system from d = 0, lam = 0 (the paper names no solver: DESIGN.md
    §2.16).  Stops after the Newton step that follows the first iterate with KKT residual <= tol (quadratic
    convergence: that step lands at the fp64 rounding floor).  Returns (d, lam)."""
    d = np.zeros_like(s)
    lam = np.zeros(s.shape[:-1])
    last = False
    for _ in range(max_iter):
        z = s + d
        g, H = _c_grad_hess(z)
        r1 = d + lam[..., None] * g
        r2 = np.prod(z, -1) - 1.0
        if last:
            break
        if max(np.abs(r1).max(initial=0.0), np.abs(r2).max(initial=0.0)) <= tol:
            last = True
        K = np.zeros(s.shape[:-1] + (4, 4))
        K[..., :3, :3] = np.eye(3) + lam[..., None, None] * H
        K[..., :3, 3] = g
        K[..., 3, :3] = g
        rhs = -np.concatenate([r1, r2[..., None]], -1)
        step = np.linalg.solve(K, rhs[..., None])[..., 0]
        d = d + step[..., :3]
        lam = lam + step[..., 3]
    return d, lam


def volume_project(F):
    """D = U diag(Sigma + d*) V^T for F [..., 3, 3]; returns (D, U, V, s, d, lam)."""
    R, S, V, s = polar_svd(F)
    U = R @ V                                    # F = U diag(s) V^T with U, V in SO(3), s signed
    d, lam = volume_kkt(s)
    D = U @ ((s + d)[..., :, None] * np.swapaxes(V, -1, -2))
    return D, U, V, s, d, lam


def volume_dg(s, d, lam):
    """J = d(Sigma + d*)/dSigma = I + dd*/dSigma from the differentiated KKT system eq:vol_kkt:
    [I + lam Hc, gc; gc^T, 0] [dd; dlam] = [-lam Hc dSigma; -gc^T dSigma], dSigma one-hot."""
    z = s + d
    g, H = _c_grad_hess(z)
    K = np.zeros(s.shape[:-1] + (4, 4))
    K[..., :3, :3] = np.eye(3) + lam[..., None, None] * H
    K[..., :3, 3] = g
    K[..., 3, :3] = g
    rhs = np.zeros(s.shape[:-1] + (4, 3))
    rhs[..., :3, :] = -lam[..., None, None] * H
    rhs[..., 3, :] = -g
    sol = np.linalg.solve(K, rhs)                # columns: one-hot dSigma_k
    return np.eye(3) + sol[..., :3, :]


def volume_derivative(F, dF, proj=None):
    """dD[dF] for D = U diag(g(Sigma)) V^T: with P = U^T dF V, U^T dD V has diagonal J P_diag and, for i != j,
    (g_i - g_j)/(s_i - s_j) sym(P)_ij + (g_i + g_j)/(s_i + s_j) skew(P)_ij (the SVD chain rule);
    at s_i = s_j the first ratio is its limit J_ii - J_ij; s_i + s_j is floored at CLAMP max|s| like the rotation
    derivative."""
    D, U, V, s, d, lam = volume_project(F) if proj is None else proj
    J = volume_dg(s, d, lam)
    gv = s + d
    P = np.swapaxes(U, -1, -2) @ dF @ V
    M = np.zeros_like(P)
    M[..., [0, 1, 2], [0, 1, 2]] = (J @ P[..., [0, 1, 2], [0, 1, 2]][..., None])[..., 0]
    smax = np.abs(s).max(-1)
    for i in range(3):
        for j in range(3):
            if i == j:
                continue
            sym = 0.5 * (P[..., i, j] + P[..., j, i])
            skw = 0.5 * (P[..., i, j] - P[..., j, i])
            ds = s[..., i] - s[..., j]
            close = np.abs(ds) <= 1e-9 * smax
            r1 = np.where(close, J[..., i, i] - J[..., i, j], (gv[..., i] - gv[..., j]) / np.where(close, 1.0, ds))
            den = np.maximum(s[..., i] + s[..., j], CLAMP * smax)
            M[..., i, j] = r1 * sym + (gv[..., i] + gv[..., j]) / den * skw
    return U @ M @ np.swapaxes(V, -1, -2)


def volume_jacobian(F):
    """J [..., 9, 9] with J[3i+j, 3k+l] = dD_ij / dF_kl."""
    proj = volume_project(F)
    cols = []
    for k in range(9):
        E = np.zeros(F.shape)
        E[..., k // 3, k % 3] = 1.0
        cols.append(volume_derivative(F, E, proj).reshape(F.shape[:-2] + (9,)))
    return np.stack(cols, -1)
