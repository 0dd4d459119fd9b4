"""Oracle FEM discretisation (test infrastructure only; see oracle/__init__.py).

P:134  "n ... number of 3D nodes after FEM-discretization", x in R^{3n}, DoF = 3*node+axis.
P:189  "G ... mapping x to the local deformation gradients F".
P:969  "E is defined as an integral over each element, which ... becomes the sum of
        energy density functions evaluated at Gaussian quadratures" -> 8-point Gauss
        (reading §8c.1: trilinear hex, points at +-1/sqrt(3), V_q = dx^3/8).
P:141  "M ... is a lumped mass matrix" -> node mass = sum of rho*dx^3/8 over incident elements.
P:199-202  A = M/h^2 + sum_e w_e G_e^T G_e.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

GAUSS = 1.0 / np.sqrt(3.0)


def corner_signs():
    """Corner a = di + 2 dj + 4 dk -> (s, t, u) = (2di-1, 2dj-1, 2dk-1)."""
    out = np.zeros((8, 3))
    for a in range(8):
        di, dj, dk = a & 1, (a >> 1) & 1, (a >> 2) & 1
        out[a] = (2 * di - 1, 2 * dj - 1, 2 * dk - 1)
    return out


def quad_points():
    """Quad point q = qi + 2 qj + 4 qk at (xi, eta, zeta) = GAUSS * (2q*-1)."""
    return corner_signs() * GAUSS


def shape_grad(dx):
    """dN[q, a, j] = dN_a/dX_j at quad point q, for an axis-aligned cube of edge dx.

    N_a = (1 + s xi)(1 + t eta)(1 + u zeta)/8, X = X0 + dx (xi + 1)/2, so
    dN/dX = (2/dx) dN/dxi."""
    S = corner_signs()
    Q = quad_points()
    dN = np.zeros((8, 8, 3))
    for q in range(8):
        xi, eta, zeta = Q[q]
        for a in range(8):
            s, t, u = S[a]
            dN[q, a, 0] = s * (1 + t * eta) * (1 + u * zeta) / 8.0
            dN[q, a, 1] = t * (1 + s * xi) * (1 + u * zeta) / 8.0
            dN[q, a, 2] = u * (1 + s * xi) * (1 + t * eta) / 8.0
    return dN * (2.0 / dx)


def G_matrices(dx):
    """G_q in R^{9 x 24}: vec(F) (row-major, index 3i+j) from x_e (index 3a+i)."""
    dN = shape_grad(dx)
    G = np.zeros((8, 9, 24))
    for q in range(8):
        for a in range(8):
            for i in range(3):
                for j in range(3):
                    G[q, 3 * i + j, 3 * a + i] = dN[q, a, j]
    return G


def Gm_matrices(dx, m):
    """G_{m,q} in R^{3 x 24}: F m (muscle fiber direction m)."""
    dN = shape_grad(dx)
    dm = dN @ np.asarray(m, np.float64)          # [q, a]
    Gm = np.zeros((8, 3, 24))
    for q in range(8):
        for a in range(8):
            for i in range(3):
                Gm[q, i, 3 * a + i] = dm[q, a]
    return Gm


def deformation_gradients(x, hex8, dx):
    """F[e, q] = sum_a x_{a} (outer) dN[q, a]  -> shape [m, 8, 3, 3]."""
    xe = x.reshape(-1, 3)[hex8]                  # [m, 8(a), 3(i)]
    return np.einsum("mai,qaj->mqij", xe, shape_grad(dx))


def scatter_element_forces(P, hex8, dx, n_nodes):
    """sum_e sum_q G_eq^T vec(P_eq): P [m, 8, 3, 3] -> R^{3n} (P:209 'G_e^T')."""
    fe = np.einsum("mqij,qaj->mai", P, shape_grad(dx))   # [m, 8, 3]
    out = np.zeros((n_nodes, 3))
    np.add.at(out, hex8.ravel(), fe.reshape(-1, 3))
    return out.ravel()


def lumped_mass(hex8, n_nodes, dx, density):
    """Per-DoF lumped mass: each element spreads rho*dx^3 equally on its 8 nodes."""
    mn = np.zeros(n_nodes)
    np.add.at(mn, hex8.ravel(), density * dx ** 3 / 8.0)
    return np.repeat(mn, 3)


def element_stiffness(dx, w, w_m=0.0, fiber=(1.0, 0.0, 0.0)):
    """K_e = sum_q V_q [w G_q^T G_q + w_m G_mq^T G_mq]  (24 x 24), V_q = dx^3/8."""
    V = dx ** 3 / 8.0
    G = G_matrices(dx)
    K = w * V * np.einsum("qka,qkb->ab", G, G)
    if w_m:
        Gm = Gm_matrices(dx, fiber)
        K = K + w_m * V * np.einsum("qka,qkb->ab", Gm, Gm)
    return K


def assemble_blocks(Ke, hex8, n_nodes):
    """Sparse sum of per-element 24x24 blocks Ke[m,24,24] (or one shared block)."""
    m = hex8.shape[0]
    dofs = (3 * hex8[:, :, None] + np.arange(3)[None, None, :]).reshape(m, 24)
    rows = np.repeat(dofs[:, :, None], 24, axis=2)
    cols = np.repeat(dofs[:, None, :], 24, axis=1)
    if Ke.ndim == 2:
        vals = np.broadcast_to(Ke, (m, 24, 24))
    else:
        vals = Ke
    N = 3 * n_nodes
    return sp.csr_matrix((vals.ravel(), (rows.ravel(), cols.ravel())), shape=(N, N))


def assemble_A(mass, hex8, n_nodes, dx, h, w, w_m=0.0):
    """A = M/h^2 + sum_e sum_q w V G^T G (+ muscle)."""
    K = assemble_blocks(element_stiffness(dx, w, w_m), hex8, n_nodes)
    return (sp.diags(mass / h ** 2) + K).tocsr()
