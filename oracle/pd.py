"""Oracle PD forward simulation (test infrastructure only; see oracle/__init__.py).

Implements, per simulation and per time step:
  y = x_i + h v_i + h^2 M^{-1} f_ext
  g(x) = 1/(2h^2) ||M^{1/2}(x - y)||^2 + E_int(x)             (P:150 eq:opt)
  E_int = sum_e sum_q V_q [w/2 ||F - R||^2 + w_m/2 ||Fm - p||^2]
  local step  z* = Proj_M(G x)                                (P:187 eq:pd_proj)
  global step A x = (1/h^2) M y + sum_e w_e G_e^T z_e*         (P:197 eq:pd_global, with M:
                                                               reading §8c.7)
  contact: Alg. 1 with frictionless normal pins on the plane n . x = d
           ("phi is a linear function and n ... a constant vector"; default z = 0;
           readings §8c.10, §8c.11), constrained solve eq:dirichlet/eq:complement
            with the coupling term kept (reading §8c.9).  A general plane is
           solved in coordinates x' = Q x - d e_z (Q a rotation with Q n = e_z): the PD
           energy is invariant under rigid motions (F' = Q F), gravity and forces rotate
           as vectors, and the plane becomes z' = 0.
  v_{i+1} = (x_{i+1} - x_i)/h                                  (eq:implicit_x)

The constrained global solve is the plain definition (a direct sparse solve of
the reduced system A_{CbarCbar} x_Cbar = d_Cbar - A_{Cbar C} xbar); the paper's
Woodbury route (Alg. 2) reaches the same x exactly and is checked against this
in tests.  c1 is an iteration (exactly `fixed_iter` PD iterations from x^0 = x_i,
reading §8c.6); every other config is the minimiser of g, to a relative residual
||grad g_free|| / ||(M/h^2) y_free|| <= tol (reading §8c.8).  The minimiser is
reached by one of three routes that tests show agree (SURVEY §8c "plain PD, PD
with L-BFGS, or a Newton polish"):
  method="newton"     (default) Newton on g with A_N = M/h^2 + Hess E_int and a direct
                      sparse LU solve per Newton step (small and mid-size meshes);
  method="pd"         the literal local-global iteration;
  method="newton_pcg" Newton on g whose step A_N d = -grad g is solved by conjugate
                      gradients preconditioned with the prefactorised A (the
                      BFGS-with-H0=A^{-1} of P:254-271 is the same Krylov space), for
                      meshes where a sparse LU of A_N does not fit (config c5).  A is
                      factored per coordinate axis: A = M/h^2 + sum w G^T G has no
                      coupling between axes (G maps every axis identically), which
                      `axis_factors` checks on the assembled matrix before using it.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import energy, fem

EPS_PHI_REL = 1e-6      # predictor penetration threshold eps_phi = 1e-6 dx (reading §8c.11)
MAX_OUTER = 10          # Alg. 1 "maximum iteration" (reading §8c.11)


@dataclasses.dataclass
class Scene:
    rest: np.ndarray
    hex8: np.ndarray
    dx: float
    density: float
    h: float
    youngs: float
    poisson: float
    gravity: np.ndarray
    fixed_dofs: np.ndarray
    contact_nodes: np.ndarray
    muscle: bool = False
    fiber: tuple = (1.0, 0.0, 0.0)
    contact_mode: str = "frictionless"   # or "sticky": the paper's infinite-friction model
    volume: bool = False                 # volume-preserving term of the background elasticity
    plane_n: tuple = (0.0, 0.0, 1.0)     # contact plane n . x = plane_d, unit normal into the free side
    plane_d: float = 0.0
    fiber_dir: Optional[np.ndarray] = None  # [m, 3] per-element fiber directions (normalised); None = `fiber`

    def __post_init__(self):
        self.n = self.rest.shape[0]
        self.N = 3 * self.n
        self.m = self.hex8.shape[0]
        self.mass = fem.lumped_mass(self.hex8, self.n, self.dx, self.density)
        self.V = self.dx ** 3 / 8.0
        self.free = np.ones(self.N, bool)
        self.free[self.fixed_dofs] = False
        self.Kcorot = fem.assemble_blocks(fem.element_stiffness(self.dx, 1.0), self.hex8, self.n)
        if self.fiber_dir is not None:
            f = np.asarray(self.fiber_dir, np.float64)
            self.fibers = f / np.linalg.norm(f, axis=1, keepdims=True)
            # per-element muscle blocks sum_q V G_mq^T G_mq with the element's own fiber
            self.Kmus = (fem.assemble_blocks(np.stack([fem.element_stiffness(self.dx, 0.0, 1.0, fe)
                                                       for fe in self.fibers]), self.hex8, self.n)
                         if self.muscle else None)
        else:
            self.fibers = np.broadcast_to(np.asarray(self.fiber, np.float64), (self.m, 3))
            self.Kmus = (fem.assemble_blocks(fem.element_stiffness(self.dx, 0.0, 1.0, self.fiber),
                                             self.hex8, self.n) if self.muscle else None)
        self._factors = {}

    # ---- material (reading §8c.2 / §8c.3) ----
    def w_of(self, youngs):
        """Corotated PD weight w = 2 mu = E/(1+nu) (SPEC lame_weights; reading §8c.2)."""
        return youngs / (1.0 + self.poisson)

    @property
    def vol_ratio(self):
        """w_v / w with w_v = lambda (Lame) and w = 2 mu (SPEC lame_weights):
        lambda / (2 mu) = nu / (1 - 2 nu); 0 without the volume term."""
        return self.poisson / (1.0 - 2.0 * self.poisson) if self.volume else 0.0

    @property
    def w_muscle(self):
        """w_m = 2 mu at the nominal material, constant (reading §8c.3)."""
        return self.youngs / (1.0 + self.poisson) if self.muscle else 0.0

    def A(self, w):
        """A = M/h^2 + sum (w + w_v) G^T G (+ w_m G_m^T G_m)  (both elastic terms have G = F)."""
        A = sp.diags(self.mass / self.h ** 2) + w * (1.0 + self.vol_ratio) * self.Kcorot
        if self.muscle:
            A = A + self.w_muscle * self.Kmus
        return A.tocsr()

    def factor(self, w, cons_mask):
        """Sparse LU of A restricted to unconstrained DoFs (library solve step)."""
        key = (float(w), cons_mask.tobytes())
        if key not in self._factors:
            A = self.A(w)
            fr = ~cons_mask
            Aff = A[fr][:, fr].tocsc()
            self._factors = {k: v for k, v in list(self._factors.items())[-4:]}
            self._factors[key] = (spla.splu(Aff), A[fr][:, cons_mask].tocsr())
        return self._factors[key]

    # ---- per-step quantities ----
    def y(self, x, v, f_ext):
        """y = x + h v + h^2 M^{-1} f_ext, gravity included in f_ext."""
        g = np.tile(self.gravity, self.n)
        return x + self.h * v + self.h ** 2 * (g + f_ext / self.mass)

    def local_step(self, x, act=None):
        """z* = Proj_M(G x) per quad point: R (SO(3)), D (det = 1) and p (muscle sphere)."""
        F = fem.deformation_gradients(x, self.hex8, self.dx)     # [m,8,3,3]
        R, S, V, s = energy.polar_svd(F)
        out = dict(F=F, R=R)
        if self.volume:
            out["D"] = energy.volume_project(F)[0]
        if self.muscle:
            Fm = np.einsum("mqij,mj->mqi", F, self.fibers)           # F m_e per quad point
            r = np.broadcast_to(np.asarray(act)[:, None], Fm.shape[:-1])
            p, n_hat, nrm = energy.muscle_project(Fm, r, self.fibers[:, None, :])
            out.update(Fm=Fm, p=p)
        return out

    def elastic_terms(self, z, w):
        """Element sums: E_int and grad E_int = sum w V G^T (F - R) (+ muscle)."""
        F, R = z["F"], z["R"]
        D = F - R
        E = 0.5 * w * self.V * np.sum(D * D)
        P = w * self.V * D
        if self.volume:
            wv = w * self.vol_ratio
            Dv = F - z["D"]
            E += 0.5 * wv * self.V * np.sum(Dv * Dv)
            P = P + wv * self.V * Dv
        if self.muscle:
            Dm = z["Fm"] - z["p"]
            E += 0.5 * self.w_muscle * self.V * np.sum(Dm * Dm)
            P = P + self.w_muscle * self.V * Dm[..., :, None] * self.fibers[:, None, None, :]
        grad = fem.scatter_element_forces(P, self.hex8, self.dx, self.n)
        return E, grad

    def rhs_d(self, y, z, w):
        """d = (1/h^2) M y + sum_e w_e G_e^T z_e*  (eq:pd_global, reading §8c.7)."""
        P = w * self.V * z["R"]
        if self.volume:
            P = P + w * self.vol_ratio * self.V * z["D"]
        if self.muscle:
            P = P + self.w_muscle * self.V * z["p"][..., :, None] * self.fibers[:, None, None, :]
        return self.mass / self.h ** 2 * y + fem.scatter_element_forces(P, self.hex8, self.dx, self.n)

    def objective(self, x, y, w, act=None):
        """g(x) (eq:opt) and grad g(x) = M/h^2 (x - y) + grad E_int (eq:time_integration)."""
        z = self.local_step(x, act)
        E, gE = self.elastic_terms(z, w)
        dxy = x - y
        g = 0.5 / self.h ** 2 * np.dot(self.mass * dxy, dxy) + E
        return g, self.mass / self.h ** 2 * dxy + gE

    def rel_residual(self, x, y, w, act, cons_mask):
        _, gg = self.objective(x, y, w, act)
        fr = ~cons_mask
        return np.linalg.norm(gg[fr]) / np.linalg.norm((self.mass / self.h ** 2 * y)[fr]), gg

    def pd_iteration(self, x, y, w, act, cons_mask):
        """One local-global iteration with DoFs in cons_mask held at their values in x."""
        z = self.local_step(x, act)
        d = self.rhs_d(y, z, w)
        lu, Afc = self.factor(w, cons_mask)
        fr = ~cons_mask
        xn = x.copy()
        xn[fr] = lu.solve(d[fr] - Afc @ x[cons_mask])
        return xn

    def pd_solve(self, x0, y, w, act, cons_mask, tol, fixed_iter=0, max_iter=20000):
        """Literal PD local-global iterations from x^0 to tol, or exactly
        fixed_iter iterations (c1).  Returns (x, iters, res).

        Stagnation exit (reading §8c.8): stop if the residual has not halved in 200 its."""
        x = x0.copy()
        if fixed_iter:
            for _ in range(fixed_iter):
                x = self.pd_iteration(x, y, w, act, cons_mask)
            res, _ = self.rel_residual(x, y, w, act, cons_mask)
            return x, fixed_iter, res
        hist = []
        for it in range(max_iter + 1):
            res, _ = self.rel_residual(x, y, w, act, cons_mask)
            hist.append(res)
            if res <= tol:
                return x, it, res
            if len(hist) > 200 and res > 0.5 * hist[-201]:
                return x, it, res
            x = self.pd_iteration(x, y, w, act, cons_mask)
        return x, max_iter, res

    def newton_solve(self, x0, y, w, act, cons_mask, tol, max_iter=200):
        """Minimiser of g (eq:opt) with DoFs in cons_mask held, by Newton's method with
        A_N = M/h^2 + Hess E_int and backtracking line search; falls back to
        the PD direction -A^{-1} grad g when the Newton direction is not a descent
        direction.  Reaches the same point PD converges to (tests check this)."""
        from . import adjoint
        x = x0.copy()
        fr = ~cons_mask
        scale = np.linalg.norm((self.mass / self.h ** 2 * y)[fr])
        g, gg = self.objective(x, y, w, act)
        res = np.linalg.norm(gg[fr]) / scale
        for it in range(max_iter + 1):
            if res <= tol:
                return x, it, res
            AN = adjoint.assemble_AN(self, x, w, act)
            d = np.zeros_like(x)
            try:
                d[fr] = -spla.spsolve(AN[fr][:, fr].tocsc(), gg[fr])
                ok = np.all(np.isfinite(d)) and gg[fr] @ d[fr] < 0
            except Exception:
                ok = False
            if not ok:
                lu, _ = self.factor(w, cons_mask)
                d[fr] = -lu.solve(gg[fr])
            slope = gg[fr] @ d[fr]
            t = 1.0
            for _ in range(60):
                gn, ggn = self.objective(x + t * d, y, w, act)
                resn = np.linalg.norm(ggn[fr]) / scale
                # Armijo on g; near the minimiser g stops resolving the decrease in
                # fp64, so a decrease of ||grad g|| is accepted there instead.
                if gn <= g + 1e-4 * t * slope or (res < 1e-6 and resn < res):
                    break
                t *= 0.5
            x = x + t * d
            g, gg, res = gn, ggn, resn
        return x, max_iter, res

    # ---- large meshes: A^{-1} per axis, A-preconditioned CG (method="newton_pcg") ----
    def axis_factors(self, w, cons_mask):
        """Preconditioner data for the CG routes: sparse LU of the diagonal axis blocks A[a::3, a::3] restricted
        to the Dirichlet-free DoFs of axis a (factored once per w; axes with the same free pattern share one LU).
        This is A^{-1} on the free DoFs only because A has no entries between different axes (checked here on
        the assembled A: P:199-202 with G acting on each axis alike).  DoFs in cons_mask beyond the
        Dirichlet ones (contact pins) are handled by restriction: z = (A^{-1} r_free)_free, the principal block
        of A^{-1} on the unconstrained DoFs, which is SPD and therefore a valid CG preconditioner."""
        base = ~self.free
        key = ("axes", float(w))
        if key not in self._factors:
            A = self.A(w).tocsr()
            Acoo = A.tocoo()
            cross = (Acoo.row % 3) != (Acoo.col % 3)
            if np.any(Acoo.data[cross] != 0.0):
                raise RuntimeError("A couples different axes: the per-axis factorisation does not apply")
            out, seen = [], {}
            for a in range(3):
                fr = ~base[a::3]
                k = fr.tobytes()
                if k not in seen:
                    Aa = A[a::3][:, a::3].tocsr()
                    seen[k] = spla.splu(Aa[fr][:, fr].tocsc(), permc_spec="MMD_AT_PLUS_A")
                out.append((fr, seen[k]))
            self._factors = {k: v for k, v in list(self._factors.items())[-4:]}
            self._factors[key] = out
        return self._factors[key], cons_mask.copy()

    @staticmethod
    def apply_axis_factors(facs, r):
        """z = (A^{-1} r)_free on the unconstrained DoFs (0 on cons_mask), r a full 3n vector."""
        axes, cons = facs
        r = np.where(cons, 0.0, r)
        z = np.zeros_like(r)
        for a, (fr, lu) in enumerate(axes):
            ra = r[a::3]
            za = np.zeros_like(ra)
            za[fr] = lu.solve(np.ascontiguousarray(ra[fr]))
            z[a::3] = za
        z[cons] = 0.0
        return z

    @staticmethod
    def pcg(matvec, b, precond, free, rtol, max_iter=5000):
        """Textbook preconditioned conjugate gradients for an SPD operator on the DoFs in `free` (the others stay
        0): stops when ||b - A u|| <= rtol ||b|| (the residual is recomputed from scratch before returning)."""
        u = np.zeros_like(b)
        bn = np.linalg.norm(b[free])
        if bn == 0.0:
            return u, 0, 0.0
        r = b.copy()
        r[~free] = 0.0
        z = precond(r)
        p = z.copy()
        rz = r @ z
        it = 0
        for it in range(1, max_iter + 1):
            q = matvec(p)
            q[~free] = 0.0
            alpha = rz / (p @ q)
            u += alpha * p
            r -= alpha * q
            if np.linalg.norm(r) <= 0.1 * rtol * bn:
                rt = b - matvec(u)
                rt[~free] = 0.0
                if np.linalg.norm(rt) <= rtol * bn:
                    break
                r = rt
            z = precond(r)
            rz_new = r @ z
            p = z + (rz_new / rz) * p
            rz = rz_new
        rt = b - matvec(u)
        rt[~free] = 0.0
        return u, it, np.linalg.norm(rt) / bn

    def newton_pcg_solve(self, x0, y, w, act, cons_mask, tol, max_iter=100):
        """Minimiser of g (eq:opt) with the DoFs in cons_mask held: Newton's method, each step A_N d = -grad g
        (A_N assembled) solved by A-preconditioned CG to 1e-4 of ||grad g|| (an inexact Newton step:
        the outer loop, not the inner accuracy, decides the converged point), Armijo backtracking on g (with the
        same fp64-floor rule as newton_solve)."""
        from . import adjoint
        x = x0.copy()
        fr = ~cons_mask
        scale = np.linalg.norm((self.mass / self.h ** 2 * y)[fr])
        facs = self.axis_factors(w, cons_mask)
        g, gg = self.objective(x, y, w, act)
        gg[cons_mask] = 0.0
        res = np.linalg.norm(gg) / scale
        for it in range(max_iter + 1):
            if res <= tol:
                return x, it, res
            AN = adjoint.assemble_AN(self, x, w, act)
            d, _, _ = self.pcg(lambda v: AN @ v, -gg, lambda r: self.apply_axis_factors(facs, r), fr, 1e-4)
            slope = gg @ d
            if not slope < 0:
                d = -self.apply_axis_factors(facs, gg)
                slope = gg @ d
            t = 1.0
            for _ in range(60):
                gn, ggn = self.objective(x + t * d, y, w, act)
                ggn[cons_mask] = 0.0
                resn = np.linalg.norm(ggn) / scale
                if gn <= g + 1e-4 * t * slope or (res < 1e-6 and resn < res):
                    break
                t *= 0.5
            x = x + t * d
            g, gg, res = gn, ggn, resn
        return x, max_iter, res

    def solve_step(self, x0, y, w, act, cons_mask, tol, fixed_iter=0, method="newton"):
        if fixed_iter or method == "pd":
            return self.pd_solve(x0, y, w, act, cons_mask, tol, fixed_iter)
        if method == "newton_pcg":
            return self.newton_pcg_solve(x0, y, w, act, cons_mask, tol)
        return self.newton_solve(x0, y, w, act, cons_mask, tol)

    # ---- contact (Alg. 1, frictionless normal pins on z = 0) ----
    def normal_dofs(self, nodes):
        return 3 * np.asarray(nodes, np.int64) + 2

    def pinned_dofs(self, nodes):
        """DoFs held by an active contact node: the normal DoF at the plane (frictionless, reading §2.10) or
        all three DoFs at the node's position x_i at the start of the step (sticky: "the contact node ... is
        fixed", infinite friction, P:321 / Alg. 1 line "x_{i+1,j} = x_{i,j}")."""
        nodes = np.asarray(nodes, np.int64)
        if self.contact_mode == "sticky":
            return (3 * nodes[:, None] + np.arange(3)[None, :]).ravel()
        return 3 * nodes + 2

    def step(self, x, v, f_ext, w, act, tol, fixed_iter=0, method="newton"):
        """One implicit step (Alg. 1 when contact candidates exist).

        Returns dict(x, v, active[|V|] bool, iters, outer, res, flag)."""
        y = self.y(x, v, f_ext)
        base = ~self.free
        if len(self.contact_nodes) == 0:
            xn, it, res = self.solve_step(x, y, w, act, base, tol, fixed_iter, method)
            return dict(x=xn, v=(xn - x) / self.h, active=np.zeros(0, bool), iters=it,
                        outer=0, res=res, flag=bool(res > tol and not fixed_iter), y=y)
        cand = self.normal_dofs(self.contact_nodes)
        eps_phi = EPS_PHI_REL * self.dx
        active = np.zeros(len(cand), bool)                     # V_i = empty
        total_it = 0
        flag = True
        margins = []
        sticky = self.contact_mode == "sticky"
        for outer in range(1, MAX_OUTER + 1):
            cons = base.copy()
            pins = self.pinned_dofs(self.contact_nodes[active])
            cons[pins] = True
            x0 = x.copy()                                       # x_{i+1} = x_i
            if not sticky:
                x0[pins] = 0.0                                  # frictionless: pinned at the plane
            # sticky: the pinned DoFs keep x_i, eq:complement with the coupling term (reading §2.9)
            xn, it, res = self.solve_step(x0, y, w, act, cons, tol, fixed_iter, method)
            total_it += it
            _, gg = self.objective(xn, y, w, act)
            lam = np.where(active, gg[cand], 0.0)              # lambda_j = 0 if j not in V_i
            phi = xn[cand]                                      # phi = z for the plane z = 0
            new = (phi < -eps_phi) | (lam > 0)
            margins.append((np.min(np.abs(phi + eps_phi)), np.min(np.abs(lam[active])) if active.any() else np.inf))
            if np.array_equal(new, active):
                flag = False
                break
            if outer == MAX_OUTER:
                break
            active = new
        return dict(x=xn, v=(xn - x) / self.h, active=active, iters=total_it, outer=outer,
                    res=res, flag=flag or bool(res > tol and not fixed_iter), y=y, lam=lam,
                    margins=margins)


def scene_from_inputs(inp, youngs=None):
    cfg = inp["cfg"]
    return Scene(rest=inp["rest"], hex8=inp["hex8"], dx=cfg.dx, density=cfg.density, h=cfg.h,
                 youngs=cfg.youngs if youngs is None else youngs, poisson=cfg.poisson,
                 gravity=np.asarray(cfg.gravity, float), fixed_dofs=inp["fixed_dofs"],
                 contact_nodes=inp["contact_nodes"], muscle=cfg.muscle, volume=getattr(cfg, "volume", False),
                 contact_mode=getattr(cfg, "contact_mode", "frictionless"),
                 plane_n=tuple(getattr(cfg, "plane_n", (0.0, 0.0, 1.0))), plane_d=getattr(cfg, "plane_d", 0.0),
                 fiber_dir=inp.get("fiber_dir"))


# ---- general contact plane n . x = d: a rigid change of world coordinates ----
def plane_rotation(n):
    """Rotation Q (rows t1, t2, n) with Q n = e_z: Gram-Schmidt from the coordinate axis least aligned
    with n; Q = I for n = e_z."""
    n = np.asarray(n, float) / np.linalg.norm(n)
    if np.array_equal(n, [0.0, 0.0, 1.0]):
        return np.eye(3)
    e = np.eye(3)[int(np.argmin(np.abs(n)))]
    t1 = e - (e @ n) * n
    t1 /= np.linalg.norm(t1)
    t2 = np.cross(n, t1)
    return np.vstack([t1, t2, n])


def has_plane(scene):
    return len(scene.contact_nodes) > 0 and (tuple(scene.plane_n) != (0.0, 0.0, 1.0) or scene.plane_d != 0.0)


def plane_scene(scene):
    """The same scene in plane coordinates x' = Q x - d e_z: gravity rotated, plane z' = 0 (cached)."""
    if getattr(scene, "_plane_scene", None) is None:
        Q = plane_rotation(scene.plane_n)
        scene._plane_scene = dataclasses.replace(scene, gravity=Q @ np.asarray(scene.gravity, float),
                                                 plane_n=(0.0, 0.0, 1.0), plane_d=0.0)
    return scene._plane_scene


def to_plane(scene, a, point):
    """[..., 3n] world -> plane coordinates (point: positions, x' = Q x - d e_z; else vectors, Q v)."""
    Q = plane_rotation(scene.plane_n)
    d = scene.plane_d / np.linalg.norm(scene.plane_n)
    b = np.asarray(a, float).reshape(a.shape[:-1] + (-1, 3)) @ Q.T
    if point:
        b[..., 2] -= d
    return b.reshape(a.shape)


def from_plane(scene, a, point):
    Q = plane_rotation(scene.plane_n)
    d = scene.plane_d / np.linalg.norm(scene.plane_n)
    b = np.asarray(a, float).reshape(a.shape[:-1] + (-1, 3)).copy()
    if point:
        b[..., 2] += d
    return (b @ Q).reshape(a.shape)


def forward(scene, q0, v0, f_ext, youngs, act=None, steps=1, tol=1e-12, fixed_iter=0,
            method="newton"):
    """Trajectory of one simulation: returns dict(q[T+1,3n], v[T+1,3n], active[T,|V|], stats).

    f_ext: [3n] constant or [T, 3n] per step."""
    if has_plane(scene):  # general plane: solve in plane coordinates, report in world coordinates
        fe = np.asarray(f_ext, dtype=np.float64)
        tr = forward(plane_scene(scene), to_plane(scene, np.asarray(q0, float), True),
                     to_plane(scene, np.asarray(v0, float), False), to_plane(scene, fe, False), youngs, act, steps,
                     tol, fixed_iter, method)
        tr["q"] = from_plane(scene, tr["q"], True)
        tr["v"] = from_plane(scene, tr["v"], False)
        return tr
    w = scene.w_of(youngs)
    q = [q0.copy()]
    vv = [v0.copy()]
    actives, stats = [], []
    f_ext = np.asarray(f_ext, dtype=np.float64)
    for i in range(steps):
        a = None if act is None else act[i]
        fe = f_ext[i] if f_ext.ndim == 2 else f_ext          # time-varying f_ext [T, 3n]
        r = scene.step(q[-1], vv[-1], fe, w, a, tol, fixed_iter, method)
        q.append(r["x"])
        vv.append(r["v"])
        actives.append(r["active"])
        stats.append({k: r[k] for k in ("iters", "outer", "res", "flag")})
    return dict(q=np.array(q), v=np.array(vv), active=np.array(actives), stats=stats)
