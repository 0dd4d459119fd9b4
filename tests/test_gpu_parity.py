"""CUDA path (C-ABI, sm_100a) vs the CPU oracle — element by element on seeded inputs.

Bars (BASELINE.json north_star): positions/velocities rel. 2-norm error <= 1e-9 per (sim, step),
gradients <= 1e-6 per output array per sim, all fp64; kernel-level hooks at 1e-12.
"""
import numpy as np
import pytest

from gpu_common import GRAD_TOL, POS_TOL, TOL_PAR_ADJ, TOL_PAR_FWD, oracle_run, rel, to_dev
from pd_inputs import get_config, make_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_05917_b200 as pdb
    pdb.build()
    return torch


def _sim(inp, **kw):
    import paper_2101_05917_b200 as pdb
    base = dict(tol_fwd=TOL_PAR_FWD, tol_adj=TOL_PAR_ADJ, contact_nodes=())
    base.update(kw)
    return pdb.simulator_from_inputs(inp, **base)


def _rand_states(inp, B, scale, seed):
    rng = np.random.default_rng(seed)
    x = np.repeat(inp["rest"].ravel()[None], B, 0) + scale * rng.standard_normal((B, 3 * inp["n_nodes"]))
    return x


# ----------------------------------------------------------------- kernel-level hooks
def test_rotations_match_oracle_polar(torch):
    from oracle import energy, fem
    inp = make_inputs(get_config("c5s"))
    sim = _sim(inp)
    for scale in (1e-3, 5e-3, 2e-2):          # 2e-2 (2 dx) inverts many elements: SVD fallback path
        x = _rand_states(inp, 2, scale, 0)
        R = torch.zeros((2, inp["n_elems"], 8, 9), dtype=torch.float64, device="cuda")
        sim.project_rotations(to_dev(x), R)
        R = R.cpu().numpy()
        for b in range(2):
            F = fem.deformation_gradients(x[b], inp["hex8"], 0.01)
            Ro, S, V, s = energy.polar_svd(F)
            ok = np.abs(s).min(-1) > 1e-6 * np.abs(s).max(-1)   # skip near-singular F (R not unique)
            gap = np.minimum(np.abs(s[..., 1] - s[..., 2]), np.abs(s[..., 0] - s[..., 2]))
            ok &= (np.abs(s[..., 1] + s[..., 2]) > 1e-6)
            d = np.abs(R[b].reshape(Ro.shape[:2] + (3, 3)) - Ro).max(axis=(-1, -2))
            assert d[ok].max() < 1e-11, (scale, d[ok].max())


@pytest.mark.parametrize("name", ["c1", "c3s", "c5s", "c2v", "c5v", "c5f"])
def test_objective_and_gradient(torch, name):
    from oracle import pd
    inp = make_inputs(get_config(name))
    B = inp["B"]
    sim = _sim(inp)
    x = _rand_states(inp, B, 1e-3, 1)
    rng = np.random.default_rng(2)
    y = x + 1e-3 * rng.standard_normal(x.shape)
    act = None if inp["act"] is None else np.ascontiguousarray(inp["act"][:, 0])
    grad = torch.zeros((B, 3 * inp["n_nodes"]), dtype=torch.float64, device="cuda")
    g = torch.zeros(B, dtype=torch.float64, device="cuda")
    sim.eval_objective(to_dev(x), to_dev(y), youngs=to_dev(inp["youngs"]),
                       act=None if act is None else to_dev(act), grad=grad, g=g)
    grad, g = grad.cpu().numpy(), g.cpu().numpy()
    for b in range(B):
        sc = pd.scene_from_inputs(inp)
        go, ggo = sc.objective(x[b], y[b], sc.w_of(inp["youngs"][b]), None if act is None else act[b])
        assert abs(g[b] - go) <= 1e-12 * abs(go)
        assert rel(grad[b], ggo) <= 1e-12


@pytest.mark.parametrize("name", ["c2s", "c3s", "c5s", "c5f"])
def test_global_solve_matches_direct(torch, name):
    # The prefactorised global step A^{-1} against a direct sparse solve of A on free DoFs.
    import scipy.sparse.linalg as spla
    from oracle import pd
    inp = make_inputs(get_config(name))
    B = inp["B"]
    sim = _sim(inp, youngs_ref=float(np.max(inp["youngs"])))
    rng = np.random.default_rng(3)
    rhs = rng.standard_normal((B, 3 * inp["n_nodes"]))
    out = torch.zeros_like(to_dev(rhs))
    sim.apply_Ainv(to_dev(rhs), out)
    out = out.cpu().numpy()
    sc = pd.scene_from_inputs(inp)
    w_ref = (np.max(inp["youngs"]) if inp["cfg"].per_sim_youngs else inp["cfg"].youngs) / (1 + sc.poisson)
    A = sc.A(w_ref)
    fr = sc.free
    for b in range(B):
        ref = np.zeros(sc.N)
        ref[fr] = spla.spsolve(A[fr][:, fr].tocsc(), rhs[b][fr])
        assert rel(out[b], ref) <= 1e-12
        assert np.all(out[b][~fr] == 0.0)


@pytest.mark.parametrize("name", ["c1", "c5s", "c2v", "c5v", "c5f"])
def test_AN_product_matches_assembled_hessian(torch, name):
    # Matrix-free A_N p vs the oracle's assembled A_N = A - dA.
    from oracle import adjoint, pd
    inp = make_inputs(get_config(name))
    B = inp["B"]
    sim = _sim(inp)
    x = _rand_states(inp, B, 1e-3, 4)
    p = np.random.default_rng(5).standard_normal(x.shape)
    act = None if inp["act"] is None else np.ascontiguousarray(inp["act"][:, 0])
    out = torch.zeros_like(to_dev(p))
    sim.apply_AN(to_dev(x), to_dev(p), out, youngs=to_dev(inp["youngs"]), act=None if act is None else to_dev(act))
    out = out.cpu().numpy()
    sc = pd.scene_from_inputs(inp)
    for b in range(B):
        AN = adjoint.assemble_AN(sc, x[b], sc.w_of(inp["youngs"][b]), None if act is None else act[b])
        assert rel(out[b], AN @ p[b]) <= 1e-12


def test_AN_product_clamp_branch(torch, monkeypatch):
    # The eigenvalue floor of the rotation derivative (reading §8c.5): the affine, inverted
    # deformation F0 = diag(1.1, 0.9, -(0.9 - 1e-9)) gives S = R^T F with s2 + s3 = 1e-9 < 1e-6 max sigma at every
    # quad point, so the floor binds (the clamped / Jacobi branch of rot_derivative_matrix).  In this regime R(F)
    # itself has condition 1/(s2 + s3) = 1e9: F carries rounding of ~1e-16 from x, so any two implementations of
    # R agree only to ~1e-16/(s2 + s3) ~ 1e-7, and the bar here is 100 eps/(s2 + s3) = 2.2e-5.  Getting the floor
    # wrong is an O(1) error: the same oracle product with the floor at 1e-7 instead of 1e-6 differs by > 1e-2.
    from oracle import adjoint, energy, pd
    inp = make_inputs(get_config("c2s"))
    sim = _sim(inp)
    gap = 1e-9
    F0 = np.diag([1.1, 0.9, -(0.9 - gap)])
    x = (inp["rest"] @ F0.T).ravel()[None]
    p = np.random.default_rng(7).standard_normal(x.shape)
    out = torch.zeros_like(to_dev(p))
    sim.apply_AN(to_dev(x), to_dev(p), out, youngs=to_dev(inp["youngs"]))
    sc = pd.scene_from_inputs(inp)
    _, _, _, sv = energy.polar_svd(F0[None])
    assert sv[0, 1] + sv[0, 2] < energy.CLAMP * np.abs(sv).max()      # the floor binds at every quad point
    ref = adjoint.assemble_AN(sc, x[0], sc.w_of(inp["youngs"][0])) @ p[0]
    assert rel(out.cpu().numpy()[0], ref) <= 100 * np.finfo(float).eps / gap
    monkeypatch.setattr(energy, "CLAMP", 1e-7)
    other = adjoint.assemble_AN(sc, x[0], sc.w_of(inp["youngs"][0])) @ p[0]
    assert rel(other, ref) > 1e-2


def test_AN_product_inverted_states(torch):
    # Random states at 2 dx (many inverted elements: SVD fallback of R, clamped or Jacobi paths of the rotation
    # derivative) against the oracle's assembled A_N.  Elements whose rotation is ill-conditioned
    # ((s_i + s_j) < 1e-3 max sigma: R itself is then determined only to ~1e-13 / 1e-3) are switched off by
    # p = 0 on their nodes; every other element, inverted or not, is compared at 1e-12.
    from oracle import adjoint, energy, fem, pd
    inp = make_inputs(get_config("c2s"))
    sim = _sim(inp)
    x = _rand_states(inp, 1, 2e-2, 9)
    F = fem.deformation_gradients(x[0], inp["hex8"], 0.01)
    _, _, _, sv = energy.polar_svd(F)
    pair = np.stack([sv[..., 0] + sv[..., 1], sv[..., 0] + sv[..., 2], sv[..., 1] + sv[..., 2]], -1)
    bad = (pair.min(-1) < 1e-3 * np.abs(sv).max(-1)).any(-1)
    inverted = (np.linalg.det(F) < 0).any(-1)
    assert inverted[~bad].sum() > 10, "the state should invert many well-conditioned elements"
    p = np.random.default_rng(10).standard_normal(x.shape)
    off = np.unique(inp["hex8"][bad])
    p.reshape(-1, 3)[off] = 0.0
    out = torch.zeros_like(to_dev(p))
    sim.apply_AN(to_dev(x), to_dev(p), out, youngs=to_dev(inp["youngs"]))
    sc = pd.scene_from_inputs(inp)
    AN = adjoint.assemble_AN(sc, x[0], sc.w_of(inp["youngs"][0]))
    assert rel(out.cpu().numpy()[0], AN @ p[0]) <= 1e-12


# ----------------------------------------------------------------- end to end
def _run_gpu(torch, inp, sim):
    B, T, N = inp["B"], inp["T"], 3 * inp["n_nodes"]
    qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device="cuda")
    vt = torch.zeros_like(qt)
    act = None if inp["act"] is None else to_dev(inp["act"][:, :T])
    st = sim.forward(to_dev(inp["q0"]), to_dev(inp["v0"]), T, f_ext=to_dev(inp["f_ext"]), actuation=act,
                     youngs=to_dev(inp["youngs"]), q_traj=qt, v_traj=vt)
    from oracle import adjoint
    q, v = qt.cpu().numpy(), vt.cpu().numpy()
    gq = np.zeros((B, N))
    gv = np.zeros((B, N))
    for b in range(B):
        _, gq[b], gv[b] = adjoint.loss_and_grad(inp, b, q[b, -1], v[b, -1])
    outs = {k: torch.zeros((B, N), dtype=torch.float64, device="cuda") for k in ("dq0", "dv0", "dfext")}
    dE = torch.zeros(B, dtype=torch.float64, device="cuda")
    dnu = torch.zeros(B, dtype=torch.float64, device="cuda")
    dact = None if act is None else torch.zeros_like(act)
    sb = sim.backward(to_dev(gq), to_dev(gv), outs["dq0"], outs["dv0"], outs["dfext"], dE, dnu, dact)
    res = dict(q=q, v=v, st=st, sb=sb, dE=dE.cpu().numpy(), dnu=dnu.cpu().numpy(),
               dact=None if dact is None else dact.cpu().numpy())
    res.update({k: t.cpu().numpy() for k, t in outs.items()})
    return res


def _compare(inp, gpu, sims):
    for b in sims:
        tr, g, _, _ = oracle_run(inp, b)
        for i in range(1, inp["T"] + 1):
            assert rel(gpu["q"][b, i], tr["q"][i]) <= POS_TOL, ("q", b, i, rel(gpu["q"][b, i], tr["q"][i]))
            vo = tr["v"][i]
            if np.linalg.norm(vo) > 0:
                assert rel(gpu["v"][b, i], vo) <= POS_TOL, ("v", b, i, rel(gpu["v"][b, i], vo))
            else:
                assert np.abs(gpu["v"][b, i]).max() <= 1e-12
        assert rel(gpu["dq0"][b], g["dq0"]) <= GRAD_TOL, ("dq0", rel(gpu["dq0"][b], g["dq0"]))
        assert rel(gpu["dv0"][b], g["dv0"]) <= GRAD_TOL, ("dv0", rel(gpu["dv0"][b], g["dv0"]))
        assert rel(gpu["dfext"][b], g["dfext"]) <= GRAD_TOL, ("dfext", rel(gpu["dfext"][b], g["dfext"]))
        assert abs(gpu["dE"][b] - g["dE"]) <= GRAD_TOL * abs(g["dE"]), ("dE", gpu["dE"][b], g["dE"])
        assert abs(gpu["dnu"][b] - g["dnu"]) <= GRAD_TOL * abs(g["dnu"]), ("dnu", gpu["dnu"][b], g["dnu"])
        if g["dact"] is not None:
            assert rel(gpu["dact"][b], g["dact"]) <= GRAD_TOL, ("dact", rel(gpu["dact"][b], g["dact"]))


def test_c1_fixed_iterations_parity(torch):
    # BASELINE.json configs[0]: exactly 10 local-global iterations per step (algorithmic parity).
    inp = make_inputs(get_config("c1"))
    gpu = _run_gpu(torch, inp, _sim(inp))
    assert np.all(gpu["st"]["iters_fwd"] == 10)
    _compare(inp, gpu, [0])


@pytest.mark.parametrize("accel_fwd,accel_adj", [(0, 1), (0, 0), (1, 1), (2, 1)])
def test_c2s_converged_parity(torch, accel_fwd, accel_adj):
    # plain PD / quasi-Newton / Newton-PCG forward; PD fixed point (eq:bp_update) / accelerated adjoint
    inp = make_inputs(get_config("c2s"))
    gpu = _run_gpu(torch, inp, _sim(inp, accel_fwd=accel_fwd, accel_adj=accel_adj))
    assert gpu["st"]["n_nonconverged"] == 0 and gpu["sb"]["n_nonconverged"] == 0
    _compare(inp, gpu, [0])


@pytest.mark.parametrize("accel_fwd", [0, 1, 2])
def test_c3s_batched_shared_factor_parity(torch, accel_fwd):
    # Per-sim E with ONE factor of A_ref: max E (plain PD) or the geometric mean of the
    # batch extremes (quasi-Newton); the oracle uses each sim's exact A_s.
    inp = make_inputs(get_config("c3s"))
    gpu = _run_gpu(torch, inp, _sim(inp, accel_fwd=accel_fwd))
    assert gpu["st"]["n_nonconverged"] == 0
    _compare(inp, gpu, range(inp["B"]))


def test_c5s_muscle_no_contact_parity(torch):
    inp = make_inputs(get_config("c5s", contact=False))
    gpu = _run_gpu(torch, inp, _sim(inp))
    assert gpu["st"]["n_nonconverged"] == 0
    _compare(inp, gpu, range(inp["B"]))


def test_bitwise_determinism(torch):
    # No float atomics anywhere: two runs are bitwise identical.
    inp = make_inputs(get_config("c3s"))
    sim = _sim(inp)
    a = _run_gpu(torch, inp, sim)
    b = _run_gpu(torch, inp, sim)
    for k in ("q", "v", "dq0", "dv0", "dfext", "dE", "dnu"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("env", [{"PD_K3_MMA": "0"}, {"PD_K3_NBUF": "3"}, {"PD_K3_NBUF": "4"}])
@pytest.mark.parametrize("name,batch", [("c3s", None), ("c5s", None), ("c3s", 10), ("c3s", 17)])
def test_k3_switches_match_direct(torch, monkeypatch, env, name, batch):
    # The K3 switches read at pd_create (FMA-pipe item product, deeper TMA rings) give the same A^{-1}
    # as a direct sparse solve (c3s: odd 3B -> the non-TMA right-hand-side path; c5s: contact ordering;
    # B = 10 / 17: 48-column chunks, where a deep ring must be clamped to the shared-memory limit).
    import scipy.sparse.linalg as spla
    from oracle import pd
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    inp = make_inputs(get_config(name), batch=batch)
    B = inp["B"]
    sim = _sim(inp, youngs_ref=float(np.max(inp["youngs"])))
    rhs = np.random.default_rng(4).standard_normal((B, 3 * inp["n_nodes"]))
    out = torch.zeros_like(to_dev(rhs))
    sim.apply_Ainv(to_dev(rhs), out)
    out = out.cpu().numpy()
    sc = pd.scene_from_inputs(inp)
    w_ref = (np.max(inp["youngs"]) if inp["cfg"].per_sim_youngs else inp["cfg"].youngs) / (1 + sc.poisson)
    A = sc.A(w_ref)
    fr = sc.free
    for b in range(B):
        ref = np.zeros(sc.N)
        ref[fr] = spla.spsolve(A[fr][:, fr].tocsc(), rhs[b][fr])
        assert rel(out[b], ref) <= 1e-12


@pytest.mark.parametrize("name", ["c3s", "c5s"])
@pytest.mark.parametrize("env", [{"PD_POLL": "0"}, {"PD_FUSE": "0"}, {"PD_POLL": "0", "PD_FUSE": "0"}])
def test_orchestration_switches_bitwise(torch, monkeypatch, env, name):
    # Iteration control by polled host flags (PD_POLL) and the fused layout / first-trial passes
    # (PD_FUSE) change how the same kernels' results are produced and read, not a single bit of them: trajectory,
    # iteration counts, active sets and every gradient equal the copy + synchronise / separate-pass path exactly
    # (c3s: per-sim E, sims converge at different iterations; c5s: contact + muscle).  Switches are read at pd_create.
    inp = make_inputs(get_config(name))
    kw = dict(contact_nodes=inp["contact_nodes"]) if name == "c5s" else {}
    kw.update(accel_fwd=1, outer_warm=1)
    ref = _run_gpu(torch, inp, _sim(inp, **kw))
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    alt_sim = _sim(inp, **kw)
    alt = _run_gpu(torch, inp, alt_sim)
    for k in ("q", "v", "dq0", "dv0", "dfext", "dE", "dnu"):
        assert np.array_equal(ref[k], alt[k]), k
    if ref["dact"] is not None:
        assert np.array_equal(ref["dact"], alt["dact"])
    for k in ("iters_fwd", "iters_adj"):
        a, b = ref["st" if k == "iters_fwd" else "sb"][k], alt["st" if k == "iters_fwd" else "sb"][k]
        assert np.array_equal(np.asarray(a), np.asarray(b)), k


@pytest.mark.parametrize("name", ["c4s", "c5s"])
def test_active_set_warm_start_probe_same_sets(torch, monkeypatch, name):
    # PD_ACTIVE_WARM=1 (off by default; NOT Alg. 1 as printed, which initialises V_i = empty at P:339): a step's first
    # outer iteration starts from the previous step's final active set.  The fixed point V' = V it stops at is the same:
    # final active sets identical at every step, states and gradients equal to the solver tolerance, fewer outer
    # iterations (the default path is the one compared with the oracle).
    inp = make_inputs(get_config(name))
    kw = dict(contact_nodes=inp["contact_nodes"], accel_fwd=1, outer_warm=1, tol_fwd=2e-14, max_iter_fwd=4000)
    ref_sim = _sim(inp, **kw)
    ref = _run_gpu(torch, inp, ref_sim)
    ref_sets = ref_sim.contact_sets()
    monkeypatch.setenv("PD_ACTIVE_WARM", "1")
    alt_sim = _sim(inp, **kw)
    alt = _run_gpu(torch, inp, alt_sim)
    assert np.array_equal(ref_sets, alt_sim.contact_sets())
    assert alt["st"]["n_nonconverged"] == 0 and alt["sb"]["n_nonconverged"] == 0
    B, T = inp["B"], inp["T"]
    for b in range(B):
        for i in range(1, T + 1):
            assert rel(alt["q"][b, i], ref["q"][b, i]) <= POS_TOL
        for k in ("dq0", "dv0", "dfext"):
            assert rel(alt[k][b], ref[k][b]) <= GRAD_TOL
    assert np.sum(alt["st"]["contact_outer"]) <= np.sum(ref["st"]["contact_outer"])


# ----------------------------------------------------------------- contact (K5, Alg. 1)
def _contact_parity(torch, name, accel_fwd=0, outer_warm=0, lbfgs_warm=0, tol_fwd=2e-14, **over):
    # The plate comes to rest on the plane, where ||v|| -> 0 and the relative velocity bar asks for
    # position agreement near the fp64 floor of the residual metric (~1e-14); the forward therefore
    # runs to 2e-14 here (measured: tools/contact_diag.py).
    inp = make_inputs(get_config(name, **over))
    sim = _sim(inp, contact_nodes=inp["contact_nodes"], accel_fwd=accel_fwd, outer_warm=outer_warm,
               lbfgs_warm=lbfgs_warm, tol_fwd=tol_fwd, max_iter_fwd=4000)
    gpu = _run_gpu(torch, inp, sim)
    sets = sim.contact_sets()
    # (sticky nodes under random actuation can make Alg. 1 cycle until its outer cap; such steps are flagged on
    # both sides and keep the last set, so only the adjoint must be free of flags there)
    if inp["cfg"].contact_mode != "sticky":
        assert gpu["st"]["n_nonconverged"] == 0
    assert gpu["sb"]["n_nonconverged"] == 0
    cand = 3 * inp["contact_nodes"] + 2
    n_active = 0
    for b in range(inp["B"]):
        tr, _, _, _ = oracle_run(inp, b)
        # bit-exact contact-set selection (BASELINE.json north_star) and identical Alg. 1 outer counts
        assert np.array_equal(sets[b], tr["active"]), ("active set", b)
        assert list(gpu["st"]["contact_outer"][b]) == [s["outer"] for s in tr["stats"]], b
        for i in range(inp["T"]):
            if inp["cfg"].contact_mode == "sticky":
                # active nodes hold all three DoFs at x_i exactly (infinite friction)
                nodes = inp["contact_nodes"][sets[b, i]]
                pins = (3 * nodes[:, None] + np.arange(3)).ravel()
                assert np.array_equal(gpu["q"][b, i + 1][pins], gpu["q"][b, i][pins])
            elif tuple(inp["cfg"].plane_n) == (0.0, 0.0, 1.0) and inp["cfg"].plane_d == 0.0:
                # pinned normal DoFs sit exactly on the plane z = 0 (eq:dirichlet with xbar = 0)
                assert np.all(gpu["q"][b, i + 1][cand[sets[b, i]]] == 0.0)
            else:
                # general plane n . x = d: pinned nodes on it up to the rounding of the change of coordinates
                nh = np.asarray(inp["cfg"].plane_n) / np.linalg.norm(inp["cfg"].plane_n)
                X = gpu["q"][b, i + 1].reshape(-1, 3)[inp["contact_nodes"][sets[b, i]]]
                assert np.all(np.abs(X @ nh - inp["cfg"].plane_d / np.linalg.norm(inp["cfg"].plane_n)) <= 1e-15)
        n_active += int(sets[b].sum())
    assert n_active > 0, "the workload never touched the plane"
    _compare(inp, gpu, range(inp["B"]))


@pytest.mark.parametrize("accel_fwd,outer_warm,lbfgs_warm", [(0, 0, 0), (1, 1, 0), (1, 1, 1), (2, 1, 0)])
def test_c4s_contact_drop_parity(torch, accel_fwd, outer_warm, lbfgs_warm):
    # BASELINE.json configs[3] recipe at oracle size: tilted plate dropped on z = 0, frictionless LCP.
    # (0, 0, 0) = literal Alg. 1 (plain PD corrector restarted from x_i); (1, 1, *) = the fast paths.
    _contact_parity(torch, "c4s", accel_fwd, outer_warm, lbfgs_warm)


@pytest.mark.parametrize("accel_fwd,outer_warm,lbfgs_warm", [(0, 0, 0), (1, 1, 0), (1, 1, 1), (2, 1, 0)])
def test_c5s_contact_muscle_parity(torch, accel_fwd, outer_warm, lbfgs_warm):
    # configs[4] recipe at oracle size: muscle actuation + bottom-face contact, B = 2.
    _contact_parity(torch, "c5s", accel_fwd, outer_warm, lbfgs_warm)


@pytest.mark.parametrize("accel_fwd,outer_warm", [(0, 0), (1, 1)])
def test_tilted_plane_contact_parity(torch, accel_fwd, outer_warm):
    # general contact plane n . x = d (20-degree slope, offset 13 mm, config c4p): the plate lands and
    # slides; bit-exact active sets and outer counts, positions / velocities / gradients in world coordinates
    _contact_parity(torch, "c4p", accel_fwd, outer_warm, 0)


def test_fiber_field_contact_muscle_parity(torch):
    # per-element fiber directions (material.fiber_dir): the c5 recipe at oracle size with a seeded
    # fiber field; forward, adjoint, dL/dr and bit-exact contact sets against the oracle
    _contact_parity(torch, "c5f", 1, 1, 0)


def test_contact_deterministic(torch):
    inp = make_inputs(get_config("c4s"))
    sim = _sim(inp, contact_nodes=inp["contact_nodes"])
    a = _run_gpu(torch, inp, sim)
    sa = sim.contact_sets()
    b = _run_gpu(torch, inp, sim)
    assert np.array_equal(sa, sim.contact_sets())
    for k in ("q", "v", "dq0", "dv0", "dfext", "dE", "dnu"):
        assert np.array_equal(a[k], b[k]), k


# ----------------------------------------------------------------- per-step losses, time-varying f_ext (8f.3)
@pytest.mark.parametrize("name", ["c2s", "c4s"])
def test_per_step_loss_time_varying_fext_parity(torch, name):
    from oracle import adjoint, pd
    inp = make_inputs(get_config(name))
    B, T, N = inp["B"], inp["T"], 3 * inp["n_nodes"]
    rng = np.random.default_rng(11)
    free = np.ones(N, bool)
    free[inp["fixed_dofs"]] = False
    fext = 0.02 * rng.standard_normal((B, T, N))
    fext[:, :, ~free] = 0.0
    cq = rng.standard_normal((B, T + 1, N))
    cv = rng.standard_normal((B, T + 1, N))
    sim = _sim(inp, contact_nodes=inp["contact_nodes"], tol_fwd=2e-14 if inp["cfg"].contact else 1e-12,
               max_iter_fwd=4000)
    qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device="cuda")
    vt = torch.zeros_like(qt)
    st = sim.forward(to_dev(inp["q0"]), to_dev(inp["v0"]), T, f_ext=to_dev(fext), youngs=to_dev(inp["youngs"]),
                     q_traj=qt, v_traj=vt)
    assert st["n_nonconverged"] == 0
    dq0 = torch.zeros((B, N), dtype=torch.float64, device="cuda")
    dfs = torch.zeros((B, T, N), dtype=torch.float64, device="cuda")
    dE = torch.zeros(B, dtype=torch.float64, device="cuda")
    sim.backward_steps(to_dev(cq), to_dev(cv), dq0, None, dfs, dE)
    q, dq0, dfs, dE = qt.cpu().numpy(), dq0.cpu().numpy(), dfs.cpu().numpy(), dE.cpu().numpy()
    sc = pd.scene_from_inputs(inp)
    tr = pd.forward(sc, inp["q0"][0], inp["v0"][0], fext[0], inp["youngs"][0], steps=T, tol=1e-13)
    for i in range(1, T + 1):
        assert rel(q[0, i], tr["q"][i]) <= POS_TOL
    g = adjoint.backward(sc, tr, inp["youngs"][0], np.zeros(N), np.zeros(N), dL_dq_steps=cq[0], dL_dv_steps=cv[0])
    assert rel(dq0[0], g["dq0"]) <= GRAD_TOL
    assert rel(dfs[0], g["dfext_steps"]) <= GRAD_TOL
    assert abs(dE[0] - g["dE"]) <= GRAD_TOL * abs(g["dE"])


# ----------------------------------------------------------------- sticky contact (the paper's model, 8f.1)
@pytest.mark.parametrize("name", ["c4s", "c5s", "c4p"])
def test_sticky_contact_parity(torch, name):
    # infinite friction: active candidates hold all three DoFs at x_i; constrained solve of all 3 columns,
    # adjoint with the pinned-value term (c4p: on the tilted plane, where the predictor's phi is n . x - d)
    _contact_parity(torch, name, 1, 1, contact_mode="sticky")


def test_tilted_plane_newton_pcg_parity(torch):
    # the Newton-PCG forward through the plane coordinates
    _contact_parity(torch, "c4p", 2, 1, 0)


def test_fiber_field_volume_parity(torch):
    # per-element fibers with the volume-preserving term (all three energies of the c5 family at once)
    _contact_parity(torch, "c5f", 1, 1, 0, volume=True, tol_fwd=5e-14)


# ----------------------------------------------------------------- volume-preserving energy (8f.2)
def test_c2v_volume_parity(torch):
    # corotated + volume-preserving background elasticity, per-sim E, 2 sims: forward and
    # gradients against the oracle; dL/dnu is no longer the corotated-only multiple -E/(1+nu) of dL/dE
    inp = make_inputs(get_config("c2v"))
    gpu = _run_gpu(torch, inp, _sim(inp, tol_fwd=5e-14))
    assert gpu["st"]["n_nonconverged"] == 0 and gpu["sb"]["n_nonconverged"] == 0
    _compare(inp, gpu, range(inp["B"]))
    nu = inp["cfg"].poisson
    for b in range(inp["B"]):
        corot_only = -inp["youngs"][b] / (1 + nu) * gpu["dE"][b]
        assert abs(gpu["dnu"][b] - corot_only) > 1e-3 * abs(gpu["dnu"][b])


def test_c5v_volume_contact_muscle_parity(torch):
    # the c5 recipe (contact + muscle) with the volume term: bit-exact active sets, states, gradients
    _contact_parity(torch, "c5v", 1, 1, 0, tol_fwd=5e-14)   # (residual floor ~3e-14 with the volume term)
