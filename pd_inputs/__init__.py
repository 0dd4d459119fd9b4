"""Seeded synthetic workloads shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no G, no mass, no energy, no
solve).  It only builds the *inputs* the paper's problem statement names
("the inputs include the initial nodal positions x_0 and
velocities v_0, the external forces f_ext ... and the material parameters"):
a voxel hex mesh (rest node coordinates + 8-node connectivity), the Dirichlet
DoF list, the contact candidate node list V, and seeded random
draws.  Both the oracle (oracle/) and the CUDA path (paper_2101_05917_b200/)
consume these arrays; neither side's arithmetic lives here.

Configs c1..c5 are BASELINE.json configs[0..4]; the ``*s`` variants are
reduced copies of the same recipe used for element-by-element parity tests at
sizes the oracle finishes in seconds.  The recipe (seeds, distributions) is the
one SURVEY.md §8(d) fixes and DESIGN.md §3 restates.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = ["Config", "CONFIGS", "get_config", "grid_mesh", "make_inputs"]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    counts: tuple            # (nx, ny, nz) elements
    h: float                 # time step (s)
    steps: int               # T
    batch: int               # B independent simulations
    seed: int                # SeedSequence entropy
    dx: float = 0.01
    youngs: float = 1e5
    poisson: float = 0.45
    density: float = 1e3
    gravity: tuple = (0.0, 0.0, -9.81)
    tol: float = 1e-9        # throughput tolerance (BASELINE.json configs[1])
    fixed_iter: int = 0      # >0: run exactly this many plain PD iterations (c1)
    dirichlet: str = "none"  # "x0": all nodes on the x = 0 face fixed at rest
    contact: bool = False    # bottom-face nodes are contact candidates (plane z=0)
    contact_mode: str = "frictionless"  # or "sticky" (the paper's infinite-friction nodes)
    muscle: bool = False     # per-element fiber actuation along +x
    volume: bool = False     # volume-preserving PD energy with w_v = lambda
    loss: str = "linear_qv"  # "linear_q" | "linear_qv" | "tip"
    v0_std: float = 0.0      # N(0, v0_std) per free node component
    per_sim_youngs: bool = False  # lognormal(ln E, 0.3) per sim (c3)
    fext_std: float = 0.0    # N(0, fext_std) N per free DoF, constant in time (c3)
    lift: float = 0.0        # min z of the plate after tilt (c4)
    max_tilt_deg: float = 0.0
    plane_n: tuple = (0.0, 0.0, 1.0)  # contact plane n . x = plane_d; the plate is placed `lift` above it
    plane_d: float = 0.0
    fiber_field: bool = False  # per-element fiber directions: +x perturbed by N(0, 0.4^2) per component, normalised

    @property
    def n_nodes(self) -> int:
        nx, ny, nz = self.counts
        return (nx + 1) * (ny + 1) * (nz + 1)

    @property
    def n_elems(self) -> int:
        nx, ny, nz = self.counts
        return nx * ny * nz

    @property
    def n_dof(self) -> int:
        return 3 * self.n_nodes


CONFIGS = {
    # BASELINE.json configs[0]: tiny cantilever, exactly 10 PD iterations per step.
    "c1": Config("c1", (4, 2, 2), h=0.01, steps=10, batch=1, seed=1, fixed_iter=10,
                 dirichlet="x0", loss="linear_q"),
    # configs[1]: cantilever 16x8x8, v0 ~ N(0, 0.1), tol 1e-9.
    "c2": Config("c2", (16, 8, 8), h=0.01, steps=100, batch=1, seed=2, dirichlet="x0",
                 v0_std=0.1),
    # configs[2]: 64 cantilevers 32x8x8, per-sim lognormal E, f_ext N(0, 0.1 N), tip loss.
    "c3": Config("c3", (32, 8, 8), h=0.005, steps=200, batch=64, seed=3, dirichlet="x0",
                 per_sim_youngs=True, fext_std=0.1, loss="tip"),
    # configs[3]: contact drop of a 20x20x4 plate, tilt <= 10 deg, 0.02 m above z=0.
    "c4": Config("c4", (20, 20, 4), h=0.005, steps=150, batch=1, seed=4, contact=True,
                 lift=0.02, max_tilt_deg=10.0),
    # configs[4]: 64x32x32 actuated robot, B=8, muscle + bottom-face contact.
    "c5": Config("c5", (64, 32, 32), h=0.01, steps=200, batch=8, seed=5, contact=True,
                 muscle=True),
    # ---- reduced parity variants (same recipe, oracle-sized) ----
    "c2s": Config("c2s", (8, 4, 4), h=0.01, steps=8, batch=1, seed=102, dirichlet="x0",
                  v0_std=0.1),
    "c3s": Config("c3s", (8, 2, 2), h=0.005, steps=6, batch=5, seed=103, dirichlet="x0",
                  per_sim_youngs=True, fext_std=0.1, loss="tip"),
    "c4s": Config("c4s", (6, 5, 2), h=0.005, steps=12, batch=1, seed=104, contact=True,
                  lift=0.001, max_tilt_deg=10.0),
    "c5s": Config("c5s", (6, 4, 3), h=0.01, steps=6, batch=2, seed=105, contact=True,
                  muscle=True),
    # ---- volume-preserving energy variants: the c2 / c5 recipes with the volume term ----
    "c2v": Config("c2v", (8, 4, 4), h=0.01, steps=6, batch=2, seed=202, dirichlet="x0", v0_std=0.1,
                  per_sim_youngs=True, volume=True),
    # c4s on a tilted plane n . x = d (P:278 general linear phi; 20 deg slope, offset 13 mm): frictionless sliding
    "c4p": Config("c4p", (6, 5, 2), h=0.005, steps=12, batch=1, seed=104, contact=True,
                  lift=0.001, max_tilt_deg=10.0, plane_n=(0.296198, 0.171010, 0.939693), plane_d=0.013),
    # c5s with a per-element fiber field (SURVEY §8(b) material.fiber_dir): muscle + contact
    "c5f": Config("c5f", (6, 4, 3), h=0.01, steps=6, batch=2, seed=105, contact=True, muscle=True, fiber_field=True),
    "c5v": Config("c5v", (6, 4, 3), h=0.01, steps=5, batch=2, seed=205, contact=True, muscle=True, volume=True),
}


def get_config(name: str, **overrides) -> Config:
    cfg = CONFIGS[name]
    return dataclasses.replace(cfg, **overrides) if overrides else cfg


def grid_mesh(counts, dx, origin=(0.0, 0.0, 0.0)):
    """Voxel hex mesh: nodes lexicographic x-fastest, elements x-fastest,
    element corners a = di + 2 dj + 4 dk (SPEC mesh module).

    Returns (rest[n,3] float64, hex8[m,8] int32).  Pure indexing, no FEM."""
    nx, ny, nz = (int(c) for c in counts)
    if min(nx, ny, nz) < 1 or not dx > 0:
        raise ValueError("grid counts must be >= 1 and dx > 0")
    i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    # x-fastest: flatten with k slowest
    ii = i.transpose(2, 1, 0).ravel()
    jj = j.transpose(2, 1, 0).ravel()
    kk = k.transpose(2, 1, 0).ravel()
    rest = np.stack([ii, jj, kk], axis=1).astype(np.float64) * dx + np.asarray(origin, np.float64)

    def nid(a, b, c):
        return a + (nx + 1) * (b + (ny + 1) * c)

    ei, ej, ek = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ei = ei.transpose(2, 1, 0).ravel()
    ej = ej.transpose(2, 1, 0).ravel()
    ek = ek.transpose(2, 1, 0).ravel()
    hexes = []
    for dk in (0, 1):
        for dj in (0, 1):
            for di in (0, 1):
                hexes.append(nid(ei + di, ej + dj, ek + dk))
    hex8 = np.stack(hexes, axis=1).astype(np.int32)
    return rest, hex8


def _rotation(axis, angle):
    """Rodrigues rotation matrix (input preparation for the c4 tilt)."""
    a = np.asarray(axis, np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * (K @ K)


def make_inputs(cfg: Config, batch: Optional[int] = None, steps: Optional[int] = None):
    """Seeded inputs for one config.  Children of SeedSequence(cfg.seed) are
    spawned in the fixed order [v0, c_q, c_v, E_s, target, f_ext, tilt, act]
    (SURVEY §8d).  ``batch``/``steps`` truncate (a prefix of the same draws)."""
    B = cfg.batch if batch is None else int(batch)
    T = cfg.steps if steps is None else int(steps)
    ss = np.random.SeedSequence(cfg.seed)
    ch = ss.spawn(9)  # (child i depends on i only: the 9th, "fiber", leaves the first eight draws unchanged)
    rng = {name: np.random.default_rng(c) for name, c in
           zip(["v0", "cq", "cv", "E", "target", "fext", "tilt", "act", "fiber"], ch)}
    rest, hex8 = grid_mesh(cfg.counts, cfg.dx)
    n = rest.shape[0]
    m = hex8.shape[0]
    nx, ny, nz = cfg.counts

    # Dirichlet DoFs: every node on the x = 0 face, all three axes.
    if cfg.dirichlet == "x0":
        fixed_nodes = np.nonzero(rest[:, 0] == rest[:, 0].min())[0]
        fixed_dofs = (3 * fixed_nodes[:, None] + np.arange(3)[None, :]).ravel().astype(np.int32)
    else:
        fixed_dofs = np.zeros(0, np.int32)
    # Contact candidates V: bottom-face nodes (z = 0 face of the rest grid).
    if cfg.contact:
        contact_nodes = np.nonzero(rest[:, 2] == rest[:, 2].min())[0].astype(np.int32)
    else:
        contact_nodes = np.zeros(0, np.int32)

    free = np.ones(3 * n, bool)
    free[fixed_dofs] = False

    # Initial state.
    q_init = rest.copy()
    if cfg.contact and cfg.max_tilt_deg > 0:
        psi = rng["tilt"].uniform(0.0, 2 * math.pi, size=B)
        theta = np.deg2rad(rng["tilt"].uniform(0.0, cfg.max_tilt_deg, size=B))
    q0 = np.empty((B, 3 * n))
    for b in range(B):
        q = q_init.copy()
        if cfg.contact and cfg.max_tilt_deg > 0:
            Rm = _rotation((math.cos(psi[b]), math.sin(psi[b]), 0.0), theta[b])
            c = q.mean(axis=0)
            q = (q - c) @ Rm.T + c
            q[:, 2] += cfg.lift - q[:, 2].min()
            if tuple(cfg.plane_n) != (0.0, 0.0, 1.0) or cfg.plane_d != 0.0:  # lowest node `lift` above the plane
                nh = np.asarray(cfg.plane_n, float) / np.linalg.norm(cfg.plane_n)
                dh = cfg.plane_d / np.linalg.norm(cfg.plane_n)
                q += (cfg.lift + dh - (q @ nh).min()) * nh
        q0[b] = q.ravel()
    v0 = np.zeros((B, 3 * n))
    if cfg.v0_std > 0:
        v0[:, :] = rng["v0"].normal(0.0, cfg.v0_std, size=(B, 3 * n))
        v0[:, ~free] = 0.0
    c_q = rng["cq"].normal(0.0, 1.0, size=(B, 3 * n))
    c_v = rng["cv"].normal(0.0, 1.0, size=(B, 3 * n))
    if cfg.per_sim_youngs:
        youngs = np.exp(rng["E"].normal(math.log(cfg.youngs), 0.3, size=B))
    else:
        youngs = np.full(B, cfg.youngs)
    f_ext = np.zeros((B, 3 * n))
    if cfg.fext_std > 0:
        f_ext[:, :] = rng["fext"].normal(0.0, cfg.fext_std, size=(B, 3 * n))
        f_ext[:, ~free] = 0.0
    act = None
    if cfg.muscle:
        act = rng["act"].uniform(0.8, 1.2, size=(B, T, m))
    fiber_dir = None
    if cfg.fiber_field:
        f = np.array([1.0, 0.0, 0.0]) + rng["fiber"].normal(0.0, 0.4, size=(m, 3))
        fiber_dir = f / np.linalg.norm(f, axis=1, keepdims=True)
    # Tip loss (c3): nodes on the x = max face; seeded targets = rest tip
    # positions displaced by N(0, 1 cm) per component ("vs seeded targets").
    tip_nodes = np.nonzero(rest[:, 0] == rest[:, 0].max())[0].astype(np.int32)
    tip_target = np.repeat(rest[tip_nodes].ravel()[None, :], B, axis=0)
    tip_target = tip_target + rng["target"].normal(0.0, 0.01, size=tip_target.shape)

    return dict(cfg=cfg, B=B, T=T, rest=rest, hex8=hex8, n_nodes=n, n_elems=m,
                fixed_dofs=fixed_dofs, contact_nodes=contact_nodes,
                q0=q0, v0=v0, f_ext=f_ext, youngs=youngs, act=act, fiber_dir=fiber_dir,
                c_q=c_q, c_v=c_v, tip_nodes=tip_nodes, tip_target=tip_target)
