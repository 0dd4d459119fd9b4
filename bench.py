#!/usr/bin/env python
"""bench.py — B200 DiffPD hot path: PD forward + PD backward throughput.

One bench "step" = one pass of the whole hot path over one batch: pd_forward over the
config's T time steps for its B sims (y, local step K1, gather K2, global solve K3, [contact
K5]) followed by pd_backward (adjoint PCG with K4 + K3, parameter terms) — SURVEY §8(a).
metric = (sims x time steps x DoF) / second (BASELINE.json "PD sim-steps/sec (forward+backward)
x DoF per B200"), DoF = 3 n (all nodal DoFs, as the configs quote them).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Default workload: c5 (BASELINE.json configs[4], 8 x 212k-DoF actuated robots with contact), the largest
single-GPU configuration and the one the north star's roofline target names.
N > 1 (torchrun): the configured batch is partitioned over the ranks (shard.shard_inputs: contiguous blocks of
sims, the shared factor's E_ref fixed from the whole batch) with no data-path collective; the time is the max
over ranks and `value` = the whole batch's DoF*steps / that time (total work fixed: "strong").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from pd_inputs import get_config, make_inputs  # noqa: E402

METRIC = "PD sim-steps/sec (forward+backward) x DoF per B200"
UNIT = "DoF*steps/s"
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 64 DFMA/clk/SM x 148 SMs x 1.965 GHz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--horizon", type=int, default=0, help="override T (time steps per trajectory)")
    ap.add_argument("--tol", type=float, default=0.0, help="override forward/adjoint tolerance")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-steps", type=int, default=2)
    ap.add_argument("--e2e-steps", type=int, default=3, help="timed iterations of the end-to-end leg (<= --steps)")
    ap.add_argument("--set", action="append", default=[], help="config override key=value (e.g. contact=False)")
    ap.add_argument("--solver", default="pd", choices=["pd", "newton"],
                    help="forward solver: pd = quasi-Newton PD (the product); newton = the Newton-PCG baseline "
                         "(SURVEY 8f-4, P:522-527) on the same kernels, for the on-box PD-vs-Newton comparison")
    return ap.parse_args()


def make_cfg(args):
    ov = {}
    for kv in args.set:
        k, v = kv.split("=", 1)
        ov[k] = eval(v, {}, {})
    if args.tol:
        ov["tol"] = args.tol
    return get_config(args.config, **ov)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- oracle (CPU)
# Bounded samples of each workload for the oracle timings (cpu_baseline, --impl reference): (grid override or
# None, sims, time steps).  c5's full grid costs the oracle minutes per sim-step (Newton with PCG),
# so its sample is the c5 recipe (contact + muscle, same h, material, seeds) on a 16x8x8 sub-grid.
CPU_SAMPLES = {"c5": ((16, 8, 8), 8, 1), "c3": (None, 8, 2), "c4": (None, 1, 2), "c2": (None, 1, 2),
               "c1": (None, 1, 10)}


def _oracle_one(args):
    """One oracle sim of a sample: forward + backward as they stand (worker process)."""
    name, counts, sims, steps, b = args
    import dataclasses
    from oracle import adjoint, pd
    cfg = get_config(name)
    if counts is not None:
        cfg = dataclasses.replace(cfg, counts=tuple(counts))
    inp = make_inputs(cfg, batch=sims, steps=steps)
    sc = pd.scene_from_inputs(inp)
    act = None if inp["act"] is None else inp["act"][b]
    tr = pd.forward(sc, inp["q0"][b], inp["v0"][b], inp["f_ext"][b], inp["youngs"][b], act,
                    steps=steps, tol=cfg.tol, fixed_iter=cfg.fixed_iter)
    L, gq, gv = adjoint.loss_and_grad(inp, b, tr["q"][-1], tr["v"][-1])
    adjoint.backward(sc, tr, inp["youngs"][b], gq, gv, act)
    return 3 * inp["n_nodes"] * steps


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        info = dict(l.split(":", 1) for l in out.splitlines() if ":" in l)
        return " ".join(info.get("Model name", "?").split()), int(info.get("CPU(s)", "0").strip() or 0)
    except Exception:
        return "unknown", os.cpu_count() or 0


def oracle_sample(cfg, sample_steps=None):
    """Time the oracle as it stands (forward + backward, the config's tolerance) on a bounded sample of the
    workload, one sim per worker process on the host's cores (the oracle itself is single-threaded NumPy)."""
    import multiprocessing as mproc
    counts, sims, steps = CPU_SAMPLES.get(cfg.name, (None, 1, 2))
    if sample_steps:
        steps = sample_steps
    model, logical = _cpu_model()
    workers = max(1, min(sims, os.cpu_count() or 1))
    jobs = [(cfg.name, counts, sims, steps, b) for b in range(sims)]
    t0 = time.perf_counter()
    with mproc.get_context("spawn").Pool(workers) as pool:
        units = sum(pool.map(_oracle_one, jobs))
    wall = time.perf_counter() - t0
    grid = "x".join(map(str, counts or cfg.counts))
    return dict(value=units / wall, unit=UNIT, cores=workers, kind="oracle",
                sample=f"{sims} sims x {steps} time steps of {cfg.name}"
                       f"{' recipe on a ' + grid + ' sub-grid' if counts else ''} (forward+backward, tol {cfg.tol:g}, "
                       f"{workers} worker processes, one sim each)",
                host_cpu=model, host_logical_cpus=logical, wall_s=wall)


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = make_cfg(args)
    vals = []
    res = None
    for _ in range(args.steps):
        res = oracle_sample(cfg)
        vals.append(res["value"])
    value = float(np.mean(vals))
    line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=args.gpus, steps=args.steps, warmup=args.warmup,
                ms_per_step=1e3 * res["wall_s"], higher_is_better=True, scaling="strong",
                vs_baseline=None, dtype="f64", data="synthetic", impl="reference",
                config=dict(workload=cfg.name, sample=res["sample"]),
                cpu_baseline=dict(value=value, unit=UNIT, cores=res["cores"], kind="oracle", sample=res["sample"],
                                  host_cpu=res["host_cpu"], host_logical_cpus=res["host_logical_cpus"]),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
            except ValueError:
                continue
            for k, v in zip(names, r[2:]):
                if "Active" in v and "Not" not in v:
                    reasons.add(k)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return dict(sm_mhz=statistics.median(loaded), sm_max_mhz=mx, reasons=sorted(reasons), samples=len(sm))


# ----------------------------------------------------------------------------- ours
# K1 operation count per quadrature point (an n-term dot product = n mul + (n-1) add): F = G_q x_e 135,
# det F 14, ||F||^2 17, 1/||F|| (rsqrt + 2 Newton steps) 12, the fallback test and X0 = c F 13, F - R / energy /
# stress 39, G_q^T P (24-term sums, 3 components) 141, energy butterfly 3 -> 374; muscle (Fm, ||Fm||, projection,
# energy, stress) 76; per Newton-Schulz iteration (X^T X 30, residual 15, Y 9, X Y 45) 99
K1_BASE_FLOPS, K1_MUSCLE_FLOPS, K1_NS_ITER_FLOPS = 374, 76, 99


def main_ours(args):
    import torch
    import paper_2101_05917_b200 as pdb

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = make_cfg(args)
    T = args.horizon or cfg.steps
    # the configured batch, partitioned over the ranks (E_ref of the shared factor from the whole batch)
    from paper_2101_05917_b200 import shard
    inp_all = make_inputs(cfg, steps=T)
    inp = shard.shard_inputs(inp_all, ws, rank) if ws > 1 else inp_all
    B, N = inp["B"], 3 * inp["n_nodes"]
    if B < 1:
        raise SystemExit(f"rank {rank}: --gpus {ws} exceeds the batch of {cfg.name} ({inp_all['B']} sims)")
    t_setup = time.perf_counter()
    sim = pdb.simulator_from_inputs(inp, tol_fwd=cfg.tol, tol_adj=cfg.tol, max_steps=T, profile=1,
                                    check_every=1, accel_fwd=2 if args.solver == "newton" else 1, outer_warm=1)
    setup_s = time.perf_counter() - t_setup
    info = sim.info()
    D = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    q0, v0, fext, E = D(inp["q0"]), D(inp["v0"]), D(inp["f_ext"]), D(inp["youngs"])
    act = None if inp["act"] is None else D(inp["act"])
    cq, cv = D(inp["c_q"]), D(inp["c_v"])
    tip = torch.as_tensor((3 * inp["tip_nodes"][:, None] + np.arange(3)[None]).ravel(), device=dev)
    target = D(inp["tip_target"])
    qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device=dev)
    vt = torch.zeros_like(qt)
    g = {k: torch.zeros((B, N), dtype=torch.float64, device=dev) for k in ("dq0", "dv0", "dfext")}
    dE = torch.zeros(B, dtype=torch.float64, device=dev)
    dnu = torch.zeros(B, dtype=torch.float64, device=dev)
    dact = None if act is None else torch.zeros_like(act)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > 126 MB L2

    def loss_grad(qT, vT):
        # user-side loss: linear in (q_T, v_T), or the c3 tip error
        if cfg.loss == "tip":
            gq = torch.zeros_like(qT)
            diff = qT[:, tip] - target
            gq[:, tip] = 2.0 * diff
            return (diff * diff).sum(1), gq, None
        L = (cq * qT).sum(1) + ((cv * vT).sum(1) if cfg.loss == "linear_qv" else 0.0)
        return L, cq, (cv if cfg.loss == "linear_qv" else None)

    stats = {}

    def one_step(q0_, v0_, fext_, E_, act_):
        st_f = sim.forward(q0_, v0_, T, f_ext=fext_, actuation=act_, youngs=E_, q_traj=qt, v_traj=vt)
        launches = sim.info()["launches"]
        L, gq, gv = loss_grad(qt[:, -1].contiguous(), vt[:, -1].contiguous())
        st_b = sim.backward(gq.contiguous(), None if gv is None else gv.contiguous(), g["dq0"], g["dv0"],
                            g["dfext"], dE, dnu, dact)
        launches += sim.info()["launches"]
        stats.update(fwd=st_f, bwd=st_b)
        return L, launches

    for _ in range(max(3, args.warmup)):
        one_step(q0, v0, fext, E, act)
    torch.cuda.synchronize()

    # ---------------- device-timed region (inputs resident in HBM)
    clocks = Clocks(local)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    total_ms, launches, prof = 0.0, 0, {}
    for _ in range(args.steps):
        flush.fill_(1.0)                           # L2 flush between timed iterations
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, nl = one_step(q0, v0, fext, E, act)
        e1.record()
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        launches += nl
        for k, (ms, c) in sim.profile().items():
            a, b = prof.get(k, (0.0, 0))
            prof[k] = (a + ms, b + c)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = shard.max_over_ranks(total_ms, ws, dev)
    ms_per_step = total_ms / args.steps
    units = inp_all["B"] * T * N           # the whole batch (every rank's sims)
    value = units / (ms_per_step / 1e3)

    # ---------------- K1's executed operation count on this workload (outside the timed region): the local step's
    # Newton-Schulz polar takes a data-dependent number of iterations; its mean over every quadrature point of the
    # trajectory's final states turns the per-point operation count of DESIGN.md §5 into K1's algorithmic flops
    k1_stats = sim.polar_stats(qt[:, T, :].contiguous())
    ns_mean = k1_stats["ns_iters"] / max(1, k1_stats["ns_points"])
    k1_flops_qp = K1_BASE_FLOPS + (K1_MUSCLE_FLOPS if act is not None else 0) + K1_NS_ITER_FLOPS * ns_mean

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        H = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64).pin_memory()
        host_in = [H(inp["q0"]), H(inp["v0"]), H(inp["f_ext"]), H(inp["youngs"])]
        if act is not None:
            host_in.append(H(inp["act"]))
        out_loss = torch.zeros(B, dtype=torch.float64).pin_memory()
        out_dE = torch.zeros(B, dtype=torch.float64).pin_memory()
        out_dq0 = torch.zeros((B, N), dtype=torch.float64).pin_memory()
        h2d = sum(t.numel() * 8 for t in host_in)
        d2h = (out_loss.numel() + out_dE.numel() + out_dq0.numel()) * 8
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e2e_ms = 0.0
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        for _ in range(e2e_steps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dv = [t.to(dev, non_blocking=True) for t in host_in]
            L, _ = one_step(dv[0], dv[1], dv[2], dv[3], dv[4] if act is not None else None)
            out_loss.copy_(L, non_blocking=True)
            out_dE.copy_(dE, non_blocking=True)
            out_dq0.copy_(g["dq0"], non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            e2e_ms += e0.elapsed_time(e1)
        e2e_ms = shard.max_over_ranks(e2e_ms, ws, dev)
        # the one end-of-run collective of the sharded path: per-sim losses of every rank
        all_loss = shard.gather_rows(out_loss.to(dev)[:, None], ws)
        assert all_loss.shape[0] == inp_all["B"]
        e2e = dict(value=units / (e2e_ms / e2e_steps / 1e3), unit=UNIT, h2d_bytes_per_step=h2d,
                   d2h_bytes_per_step=d2h, steps=e2e_steps)

    # ---------------- rooflines (live CUDA events per kernel family, pd_profile)
    nfree = info["n_free_nodes"]
    R = 3 * B
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    ncu = {}
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(cfg.name, {})
    except Exception:
        pass

    def roof_of(fam):
        ms_tot, cnt = prof.get(fam, (0.0, 0))
        if not cnt:
            return None
        avg_s = ms_tot / cnt / 1e3
        if fam == "solve_K3":
            # the scalar factor L_s streamed once per sweep (2 nnz(L_s) 8 B) + the solve vectors
            # (rhs in, y out+in, x out: 4 nfree R 8 B) + layout permutation in/out (2 3n B 8 B)
            alg = 2 * info["nnz_L"] * 8 + 4 * nfree * R * 8 + 2 * N * B * 8
            return dict(bound="hbm", achieved=alg / avg_s / 1e9, peak=hbm_peak, unit="GB/s",
                        frac=alg / avg_s / 1e9 / hbm_peak, traffic=ncu.get("solve_K3_dram_bytes"), kernel=fam,
                        algorithmic_bytes_per_launch=alg, avg_launch_ms=avg_s * 1e3,
                        peak_source="MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6650")
        # element kernels: fp64 flops per quadrature point (DESIGN.md §5 operation count; ncu-measured when
        # profiles/ncu_traffic.json has it)
        per_qp = {"local_K1": k1_flops_qp, "AN_K4": 420, "param": 700}.get(fam)
        if per_qp is None:
            return None
        flops = per_qp * 8 * inp["n_elems"] * B
        ach = flops / avg_s / 1e12
        r = dict(bound="alu", achieved=ach, peak=FP64_PEAK_TFLOPS, unit="TFLOP/s", frac=ach / FP64_PEAK_TFLOPS,
                 traffic=ncu.get(fam + "_dram_bytes"), kernel=fam, flops_per_qp=per_qp, avg_launch_ms=avg_s * 1e3,
                 peak_source="derived fp64 pipe peak: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (DESIGN.md §5)")
        if fam == "local_K1":
            r.update(flop_model=f"{K1_BASE_FLOPS} + {K1_MUSCLE_FLOPS if act is not None else 0} (muscle) + "
                                f"{K1_NS_ITER_FLOPS} x {ns_mean:.3f} Newton-Schulz iterations (measured mean over "
                                f"{k1_stats['ns_points']} quadrature points of the final states; "
                                f"{k1_stats['fallback_points']} fallback points counted at 0)")
        return r

    fam = max(prof, key=lambda k: prof[k][0])
    roof = roof_of(fam) or roof_of("solve_K3")
    share = {k: round(v[0] / max(1e-9, sum(x[0] for x in prof.values())), 4) for k, v in prof.items()}

    line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=ws, steps=args.steps, warmup=max(3, args.warmup),
                ms_per_step=ms_per_step, higher_is_better=True, scaling="strong", vs_baseline=None, dtype="f64",
                data="synthetic",
                config=dict(workload=cfg.name, batch=inp_all["B"], batch_per_gpu=B, time_steps=T, dof=N, tol=cfg.tol,
                            grid=list(cfg.counts), l2="flushed (256 MB write) before every timed iteration",
                            parallelism=f"batch partitioned over {ws} rank(s), no data-path collective",
                            solver="quasi-Newton PD (L-BFGS, H0 = gamma_b A^-1)" if args.solver == "pd"
                            else "Newton-PCG baseline (SURVEY 8f-4)",
                            # any developer switch in the environment is part of the measured configuration
                            # (PD_ACTIVE_WARM=1 is not Alg. 1 as printed: never the headline)
                            switches={k: v for k, v in sorted(os.environ.items()) if k.startswith("PD_")}),
                e2e=e2e, gpu_launches=launches, roofline=roof,
                roofline_k3=roof_of("solve_K3"), roofline_k1=roof_of("local_K1"),
                # the launch durations are CUDA-event times of a 1-in-N sample of each family's launches inside the
                # timed region (N = PD_PROF_EVERY, default 4; an event boundary interrupts the PDL chain)
                profile_sampling=f"1 in {os.environ.get('PD_PROF_EVERY', '4')} launches per kernel family",
                kernel_share=share,
                # per-sim means and, since the batch loop runs until its slowest sim converges, the mean over steps
                # of the per-step maximum over sims (what the batch actually pays)
                iters=dict(fwd_mean=float(np.mean(stats["fwd"]["iters_fwd"])),
                           adj_mean=float(np.mean(stats["bwd"]["iters_adj"])),
                           fwd_batch=float(np.mean(np.max(stats["fwd"]["iters_fwd"], axis=0))),
                           adj_batch=float(np.mean(np.max(stats["bwd"]["iters_adj"], axis=0))),
                           nonconverged=int(stats["fwd"]["n_nonconverged"] + stats["bwd"]["n_nonconverged"])),
                setup=dict(seconds=setup_s, factor_ms=info["factor_ms"], nnz_L=info["nnz_L"],
                           supernodes=info["n_supernodes"], levels=info["n_levels"]),
                clocks=clk)
    if rank == 0:
        if args.cpu_sample_steps > 0 and ws == 1:
            line["cpu_baseline"] = {k: v for k, v in oracle_sample(cfg).items() if k != "wall_s"}
        else:
            line["cpu_baseline"] = dict(value=None, unit=UNIT, cores=None, kind="oracle",
                                        sample="not run (--cpu-sample-steps 0, or N > 1: rank 0 at N = 1 only)")
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        main_ours(a)
