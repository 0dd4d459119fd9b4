"""B200-native DiffPD hot path (arXiv 2101.05917): PD forward + PD backpropagation.

Python surface = thin marshalling over the C-ABI in include/diffpd_b200.h.
PyTorch provides device memory and streams only; every step of the path runs
in libdiffpd_b200.so (sm_100a CUDA kernels + C++ host setup).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib

__all__ = ["Simulator", "PDError", "build"]


def build(force=False):
    from .buildlib import build as _b
    return _b(force=force)


class PDError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_lib.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _ptr(t, shape=None, name="array", device=None):
    """Device pointer of a contiguous fp64 CUDA tensor (or None), after checking what the C-ABI cannot:
    dtype float64, the handle's device and the exact shape the library will read or write (a float32 tensor
    or a short array would otherwise be read past its end)."""
    if t is None:
        return None
    import torch
    if not t.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor (the library takes device pointers)")
    if t.dtype != torch.float64:
        raise ValueError(f"{name}: expected dtype torch.float64, got {t.dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: tensor on {t.device}, the simulator's device is {device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Simulator:
    """One pd_sim handle: mesh + material + h + Dirichlet set + contact candidates."""

    def __init__(self, rest, hex8, dx, *, youngs, poisson, density, h, gravity=(0.0, 0.0, -9.81),
                 fixed_dofs=(), contact_nodes=(), muscle_w=0.0, fiber=(1.0, 0.0, 0.0),
                 tol_fwd=1e-9, tol_adj=1e-9, max_iter_fwd=20000, max_iter_adj=20000, fixed_iter=0,
                 accel_fwd=1, accel_adj=1, check_every=1, max_batch=1, max_steps=1, youngs_ref=0.0,
                 max_outer=10, eps_phi=None, profile=0, outer_warm=1, x0_predict=0, contact_mode=1,
                 lbfgs_warm=0, volume=False, plane_n=(0.0, 0.0, 1.0), plane_d=0.0, fiber_dir=None):
        self.lib = _lib.load()
        rest = np.ascontiguousarray(rest, dtype=np.float64)
        hex8 = np.ascontiguousarray(hex8, dtype=np.int32)
        self.n_nodes = rest.shape[0]
        self.n_elems = hex8.shape[0]
        self._keep = [rest, hex8]
        mesh = _lib.PdMesh(self.n_nodes, self.n_elems, rest.ctypes.data_as(_lib.dp),
                           hex8.ctypes.data_as(_lib.ip), float(dx))
        fib = None if fiber_dir is None else np.ascontiguousarray(fiber_dir, dtype=np.float64)
        if fib is not None and fib.shape != (self.n_elems, 3):
            raise ValueError(f"fiber_dir: expected shape ({self.n_elems}, 3), got {fib.shape}")
        self._keep.append(fib)
        mat = _lib.PdMaterial(float(youngs), float(poisson), float(density), float(muscle_w),
                              (C.c_double * 3)(*gravity), (C.c_double * 3)(*fiber), int(bool(volume)),
                              None if fib is None else fib.ctypes.data_as(_lib.dp))
        fixed = np.ascontiguousarray(fixed_dofs, dtype=np.int32)
        cand = np.ascontiguousarray(contact_nodes, dtype=np.int32)
        self._keep += [fixed, cand]
        opt = _lib.PdOptions(tol_fwd, tol_adj, max_iter_fwd, max_iter_adj, fixed_iter, accel_fwd, accel_adj,
                             check_every, max_batch, max_steps, youngs_ref,
                             cand.ctypes.data_as(_lib.ip) if len(cand) else None, len(cand), max_outer,
                             float(1e-6 * dx if eps_phi is None else eps_phi), int(profile), int(outer_warm),
                             int(contact_mode), int(x0_predict), int(lbfgs_warm),
                             (C.c_double * 3)(*[float(c) for c in plane_n]), float(plane_d))
        h_ = C.c_void_p()
        st = self.lib.pd_create(C.byref(mesh), C.byref(mat), float(h),
                                fixed.ctypes.data_as(_lib.ip) if len(fixed) else None, len(fixed),
                                C.byref(opt), C.byref(h_))
        if st != 0:
            raise PDError(st, self.lib.pd_last_error(None).decode())
        self.handle = h_
        import torch
        self.device = torch.device("cuda", torch.cuda.current_device())  # the handle's device (pd_create)
        self.n_contact = len(cand)
        self.max_batch, self.max_steps = max_batch, max_steps
        self.h = h

    def _check(self, st):
        if st != 0:
            raise PDError(st, self.lib.pd_last_error(self.handle).decode())

    def close(self):
        if getattr(self, "handle", None):
            self.lib.pd_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        out = (C.c_int64 * 8)()
        self._check(self.lib.pd_info(self.handle, out, 8))
        keys = ["n_nodes", "n_free_nodes", "n_supernodes", "n_levels", "nnz_L", "n_contact",
                "factor_ms", "launches"]
        return dict(zip(keys, list(out)))

    PROFILE_FAMILIES = ["local_K1", "gather_K2", "solve_K3", "AN_K4", "contact_K5", "param"]

    def profile(self):
        """{family: (total_ms, count)} since the last forward (needs profile=1)."""
        ms = (C.c_double * 6)()
        cnt = (C.c_int64 * 6)()
        self._check(self.lib.pd_profile(self.handle, ms, cnt, 6))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(self.PROFILE_FAMILIES)}

    def _stats(self, B, T):
        arrs = dict(iters_fwd=np.zeros(B * T, np.int32), iters_adj=np.zeros(B * T, np.int32),
                    contact_outer=np.zeros(B * T, np.int32), final_res_fwd=np.zeros(B * T),
                    final_res_adj=np.zeros(B * T))
        st = _lib.PdStats(arrs["iters_fwd"].ctypes.data_as(_lib.ip), arrs["iters_adj"].ctypes.data_as(_lib.ip),
                          arrs["contact_outer"].ctypes.data_as(_lib.ip),
                          arrs["final_res_fwd"].ctypes.data_as(_lib.dp),
                          arrs["final_res_adj"].ctypes.data_as(_lib.dp), 0)
        return st, arrs

    def forward(self, q0, v0, steps, f_ext=None, actuation=None, youngs=None, q_traj=None, v_traj=None):
        """q0, v0: CUDA fp64 [B, 3n]; f_ext [B, 3n] (constant) or [B, steps, 3n] (per step).
        Returns a stats dict (numpy [B, steps] arrays)."""
        B = q0.shape[0]
        N, m, dev = 3 * self.n_nodes, self.n_elems, self.device
        st, arrs = self._stats(B, steps)   # (B and steps against max_batch / max_steps: checked by pd_forward)
        per_step = f_ext is not None and f_ext.dim() == 3
        stride = N if per_step else 0
        args = [_ptr(q0, (B, N), "q0", dev), _ptr(v0, (B, N), "v0", dev),
                _ptr(f_ext, (B, steps, N) if per_step else (B, N), "f_ext", dev), stride,
                _ptr(actuation, (B, steps, m), "actuation", dev), _ptr(youngs, (B,), "youngs", dev), steps,
                _ptr(q_traj, (B, steps + 1, N), "q_traj", dev), _ptr(v_traj, (B, steps + 1, N), "v_traj", dev)]
        self._check(self.lib.pd_forward(self.handle, B, *args, C.byref(st), _stream()))
        self._B, self._T = B, steps
        out = {k: v.reshape(B, steps) for k, v in arrs.items() if k in ("iters_fwd", "final_res_fwd", "contact_outer")}
        out["n_nonconverged"] = st.n_nonconverged
        return out

    def backward(self, dL_dqT=None, dL_dvT=None, dL_dq0=None, dL_dv0=None, dL_dfext=None, dL_dE=None,
                 dL_dnu=None, dL_dact=None):
        B, T = self._B, self._T
        N, m, dev = 3 * self.n_nodes, self.n_elems, self.device
        st, arrs = self._stats(B, T)
        args = [_ptr(dL_dqT, (B, N), "dL_dqT", dev), _ptr(dL_dvT, (B, N), "dL_dvT", dev),
                _ptr(dL_dq0, (B, N), "dL_dq0", dev), _ptr(dL_dv0, (B, N), "dL_dv0", dev),
                _ptr(dL_dfext, (B, N), "dL_dfext", dev), _ptr(dL_dE, (B,), "dL_dE", dev),
                _ptr(dL_dnu, (B,), "dL_dnu", dev), _ptr(dL_dact, (B, T, m), "dL_dact", dev)]
        self._check(self.lib.pd_backward(self.handle, *args, C.byref(st), _stream()))
        out = {k: v.reshape(B, T) for k, v in arrs.items() if k in ("iters_adj", "final_res_adj")}
        out["n_nonconverged"] = st.n_nonconverged
        return out

    def backward_steps(self, dL_dq_steps=None, dL_dv_steps=None, dL_dq0=None, dL_dv0=None, dL_dfext_steps=None,
                       dL_dE=None, dL_dnu=None, dL_dact=None):
        """Per-step losses: dL_dq_steps / dL_dv_steps [B, T+1, 3n]; dL_dfext_steps output [B, T, 3n]."""
        B, T = self._B, self._T
        N, m, dev = 3 * self.n_nodes, self.n_elems, self.device
        st, arrs = self._stats(B, T)
        args = [_ptr(dL_dq_steps, (B, T + 1, N), "dL_dq_steps", dev), _ptr(dL_dv_steps, (B, T + 1, N), "dL_dv_steps", dev),
                _ptr(dL_dq0, (B, N), "dL_dq0", dev), _ptr(dL_dv0, (B, N), "dL_dv0", dev),
                _ptr(dL_dfext_steps, (B, T, N), "dL_dfext_steps", dev), _ptr(dL_dE, (B,), "dL_dE", dev),
                _ptr(dL_dnu, (B,), "dL_dnu", dev), _ptr(dL_dact, (B, T, m), "dL_dact", dev)]
        self._check(self.lib.pd_backward_steps(self.handle, *args, C.byref(st), _stream()))
        out = {k: v.reshape(B, T) for k, v in arrs.items() if k in ("iters_adj", "final_res_adj")}
        out["n_nonconverged"] = st.n_nonconverged
        return out

    def contact_sets(self):
        """Final Alg. 1 active set per (sim, step) of the last forward: bool [B, T, n_contact]."""
        out = np.zeros((self._B, self._T, self.n_contact), np.uint8)
        self._check(self.lib.pd_contact_sets(self.handle, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out.astype(bool)

    def _diag_B(self, x):
        return x.shape[0], 3 * self.n_nodes, self.n_elems, self.device

    def eval_objective(self, x, y, youngs=None, act=None, grad=None, g=None):
        B, N, m, dev = self._diag_B(x)
        self._check(self.lib.pd_eval_objective(self.handle, B, _ptr(x, (B, N), "x", dev), _ptr(y, (B, N), "y", dev),
                                               _ptr(youngs, (B,), "youngs", dev), _ptr(act, (B, m), "act", dev),
                                               _ptr(grad, (B, N), "grad", dev), _ptr(g, (B,), "g", dev), _stream()))

    def apply_Ainv(self, rhs, out):
        B, N, m, dev = self._diag_B(rhs)
        self._check(self.lib.pd_apply_Ainv(self.handle, B, _ptr(rhs, (B, N), "rhs", dev), _ptr(out, (B, N), "out", dev),
                                           _stream()))

    def apply_AN(self, x, p, out, youngs=None, act=None):
        B, N, m, dev = self._diag_B(x)
        self._check(self.lib.pd_apply_AN(self.handle, B, _ptr(x, (B, N), "x", dev), _ptr(youngs, (B,), "youngs", dev),
                                         _ptr(act, (B, m), "act", dev), _ptr(p, (B, N), "p", dev),
                                         _ptr(out, (B, N), "out", dev), _stream()))

    def polar_stats(self, x):
        """{'ns_iters': total Newton-Schulz iterations, 'ns_points', 'fallback_points'} of K1's polar on x [B][3n]."""
        B, N, m, dev = self._diag_B(x)
        out = (C.c_int64 * 3)()
        self._check(self.lib.pd_polar_stats(self.handle, B, _ptr(x, (B, N), "x", dev), out, _stream()))
        return dict(ns_iters=int(out[0]), ns_points=int(out[1]), fallback_points=int(out[2]))

    def project_rotations(self, x, R):
        B, N, m, dev = self._diag_B(x)
        self._check(self.lib.pd_project_rotations(self.handle, B, _ptr(x, (B, N), "x", dev),
                                                  _ptr(R, (B, m, 8, 9), "R", dev), _stream()))


def simulator_from_inputs(inp, **kw):
    """Convenience: a Simulator for a pd_inputs workload dict."""
    cfg = inp["cfg"]
    muscle_w = cfg.youngs / (1 + cfg.poisson) if cfg.muscle else 0.0
    args = dict(contact_mode=2 if getattr(cfg, "contact_mode", "frictionless") == "sticky" else 1,
                volume=getattr(cfg, "volume", False),
                youngs=cfg.youngs, poisson=cfg.poisson, density=cfg.density, h=cfg.h, gravity=cfg.gravity,
                fixed_dofs=inp["fixed_dofs"], contact_nodes=inp["contact_nodes"], muscle_w=muscle_w,
                fixed_iter=cfg.fixed_iter, tol_fwd=cfg.tol, max_batch=inp["B"], max_steps=inp["T"],
                plane_n=tuple(getattr(cfg, "plane_n", (0.0, 0.0, 1.0))), plane_d=getattr(cfg, "plane_d", 0.0),
                fiber_dir=inp.get("fiber_dir"))
    args.update(kw)
    if cfg.per_sim_youngs and "youngs_ref" not in kw:
        # plain PD needs the majorising A_ref (largest E of the batch); the quasi-Newton
        # forward/adjoint only use A_ref^{-1} as a preconditioner, where the geometric mean of the batch
        # extremes halves the worst-case condition number.  A sharded workload (shard.shard_inputs) carries the
        # value of the whole batch.
        from .shard import shared_youngs_ref
        accel = args.get("accel_fwd", 1)
        args["youngs_ref"] = inp.get("youngs_ref") or shared_youngs_ref(inp["youngs"], bool(accel))
    return Simulator(inp["rest"], inp["hex8"], cfg.dx, **args)
