"""Edge cases of the C-ABI path on the GPU: argument/state errors, partial batches, single steps, the rest state,
an all-pinned contact set, and degenerate (inverted) elements."""
import numpy as np
import pytest

from gpu_common import rel, to_dev
from pd_inputs import get_config, grid_mesh, make_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_05917_b200 as pdb
    pdb.build()
    return torch


def test_state_and_argument_errors(torch):
    import paper_2101_05917_b200 as pdb
    from paper_2101_05917_b200 import _lib
    inp = make_inputs(get_config("c1"))
    sim = pdb.simulator_from_inputs(inp, max_batch=2, max_steps=3)
    z = torch.zeros((1, 3 * inp["n_nodes"]), dtype=torch.float64, device="cuda")
    sim._B, sim._T = 1, 1
    with pytest.raises(pdb.PDError) as e:          # backward before any forward
        sim.backward(z, None, torch.zeros_like(z))
    assert e.value.status == _lib.PD_ERR_STATE
    q = to_dev(np.repeat(inp["q0"], 3, 0))
    with pytest.raises(pdb.PDError) as e:          # B > max_batch
        sim.forward(q, torch.zeros_like(q), 1)
    assert e.value.status == _lib.PD_ERR_INVALID_ARGUMENT
    q = to_dev(inp["q0"])
    with pytest.raises(pdb.PDError) as e:          # steps > max_steps
        sim.forward(q, torch.zeros_like(q), 4)
    assert e.value.status == _lib.PD_ERR_INVALID_ARGUMENT
    with pytest.raises(ValueError):                # the binding checks dtype and shape before the C-ABI
        sim.forward(q.float(), torch.zeros_like(q), 1)
    with pytest.raises(ValueError):
        sim.forward(q, torch.zeros_like(q)[:, :-3].contiguous(), 1)
    with pytest.raises(pdb.PDError):               # a contact candidate that is also a Dirichlet node
        pdb.simulator_from_inputs(inp, contact_nodes=inp["fixed_dofs"][::3] // 3)
    with pytest.raises(pdb.PDError):               # repeated candidate
        pdb.simulator_from_inputs(inp, contact_nodes=np.array([5, 5], np.int32))
    with pytest.raises(pdb.PDError) as e:          # unknown forward route
        pdb.simulator_from_inputs(inp, accel_fwd=3)
    assert e.value.status == _lib.PD_ERR_INVALID_ARGUMENT
    with pytest.raises(pdb.PDError) as e:          # non-finite contact plane
        pdb.simulator_from_inputs(inp, contact_nodes=np.array([5], np.int32), plane_n=(0.0, float("nan"), 1.0))
    assert e.value.status == _lib.PD_ERR_INVALID_ARGUMENT
    inp5 = make_inputs(get_config("c5f", counts=(2, 2, 1), contact=False))
    bad = inp5["fiber_dir"].copy()
    bad[1] = 0.0
    with pytest.raises(pdb.PDError) as e:          # a zero fiber direction
        pdb.simulator_from_inputs(dict(inp5, fiber_dir=bad))
    assert e.value.status == _lib.PD_ERR_INVALID_ARGUMENT
    with pytest.raises(ValueError):                # fiber field of the wrong shape (binding check)
        pdb.simulator_from_inputs(dict(inp5, fiber_dir=bad[:-1]))


def test_partial_batch_and_single_step(torch):
    # max_batch 5 handle run with B = 2 and T = 1: same results as the first two sims of a B = 5 run
    import paper_2101_05917_b200 as pdb
    inp = make_inputs(get_config("c3s"), steps=1)
    kw = dict(tol_fwd=1e-12, tol_adj=1e-11, youngs_ref=float(np.max(inp["youngs"])))
    sim = pdb.simulator_from_inputs(inp, **kw)
    N = 3 * inp["n_nodes"]
    outs = []
    for B in (5, 2):
        qt = torch.zeros((B, 2, N), dtype=torch.float64, device="cuda")
        st = sim.forward(to_dev(inp["q0"][:B]), to_dev(inp["v0"][:B]), 1, f_ext=to_dev(inp["f_ext"][:B]),
                         youngs=to_dev(inp["youngs"][:B]), q_traj=qt)
        assert st["n_nonconverged"] == 0
        outs.append(qt.cpu().numpy())
    for b in range(2):
        assert rel(outs[1][b, 1], outs[0][b, 1]) <= 1e-11


def test_rest_state_without_gravity_stays_exactly(torch):
    # grad g(rest) = 0 exactly: the solve converges at iteration 0 and x, v stay bitwise at rest
    import paper_2101_05917_b200 as pdb
    rest, hex8 = grid_mesh((4, 3, 2), 0.01)
    sim = pdb.Simulator(rest, hex8, 0.01, youngs=1e5, poisson=0.45, density=1e3, h=0.01, gravity=(0.0, 0.0, 0.0),
                        max_batch=1, max_steps=3)
    N = rest.size
    q0 = to_dev(rest.reshape(1, -1))
    qt = torch.zeros((1, 4, N), dtype=torch.float64, device="cuda")
    vt = torch.zeros_like(qt)
    st = sim.forward(q0, torch.zeros_like(q0), 3, q_traj=qt, v_traj=vt)
    assert np.all(st["iters_fwd"] == 0)
    assert np.array_equal(qt.cpu().numpy()[0, -1], rest.ravel())
    assert np.all(vt.cpu().numpy() == 0.0)


def test_all_candidates_pinned(torch):
    # every bottom node pressed into the plane: the constrained root block has no free candidates (k = 0)
    import paper_2101_05917_b200 as pdb
    rest, hex8 = grid_mesh((3, 3, 2), 0.01)
    cand = np.nonzero(rest[:, 2] == 0.0)[0].astype(np.int32)
    sim = pdb.Simulator(rest, hex8, 0.01, youngs=1e5, poisson=0.45, density=1e3, h=0.01, contact_nodes=cand,
                        max_batch=1, max_steps=2, tol_fwd=1e-12, tol_adj=1e-11)
    N = rest.size
    q0 = to_dev(rest.reshape(1, -1))
    v0 = torch.zeros_like(q0)
    v0.view(-1, 3)[:, 2] = -0.5                      # moving into the plane
    qt = torch.zeros((1, 3, N), dtype=torch.float64, device="cuda")
    st = sim.forward(q0, v0, 2, q_traj=qt)
    sets = sim.contact_sets()
    assert sets.all()
    z = qt.cpu().numpy()[0, 1:, 2::3][:, cand]
    assert np.all(z == 0.0)
    assert st["n_nonconverged"] == 0
    g = torch.zeros_like(q0)
    sim.backward(to_dev(np.ones((1, N))), None, g)   # adjoint with every candidate pinned
    assert np.all(np.isfinite(g.cpu().numpy()))


def test_inverted_elements_project_to_rotations(torch):
    # det F <= 0 (inverted elements): the SVD path still returns proper rotations
    import paper_2101_05917_b200 as pdb
    rest, hex8 = grid_mesh((2, 2, 2), 0.01)
    sim = pdb.Simulator(rest, hex8, 0.01, youngs=1e5, poisson=0.45, density=1e3, h=0.01, max_batch=1, max_steps=1)
    x = rest.copy()
    x[:, 0] = -x[:, 0]                               # mirror: every element inverted
    R = torch.zeros((1, 8, 8, 9), dtype=torch.float64, device="cuda")
    sim.project_rotations(to_dev(x.reshape(1, -1)), R)
    R = R.cpu().numpy().reshape(-1, 3, 3)
    assert np.allclose(np.einsum("nij,nkj->nik", R, R), np.eye(3), atol=1e-12)
    assert np.allclose(np.linalg.det(R), 1.0, atol=1e-12)


def test_polar_stats_hook(torch):
    # pd_polar_stats (the K1 operation count of bench.py): at rest F = I, so every quadrature point takes exactly one
    # Newton-Schulz step (X0 = I is orthogonal); an inverted element takes the fallback path
    import paper_2101_05917_b200 as pdb
    inp = make_inputs(get_config("c1"))
    sim = pdb.simulator_from_inputs(inp)
    x = inp["rest"].ravel()[None].copy()
    st = sim.polar_stats(to_dev(x))
    assert st == dict(ns_iters=8 * inp["n_elems"], ns_points=8 * inp["n_elems"], fallback_points=0)
    x2 = x.copy().reshape(-1, 3)
    e0 = inp["hex8"][0]
    x2[e0[4:], 2] = x2[e0[:4], 2] - 0.01      # the element's top face below its bottom face: det F < 0
    st2 = sim.polar_stats(to_dev(x2.reshape(1, -1)))
    assert st2["fallback_points"] > 0 and st2["ns_points"] + st2["fallback_points"] == 8 * inp["n_elems"]
