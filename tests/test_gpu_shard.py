"""Batch-partitioned multi-rank path on one GPU: two ranks (gloo for the host-side
collectives) each run their contiguous block of the configured batch; the gathered per-sim results must be
BITWISE equal to the single-rank run of the whole batch (the per-sim reductions do not depend on the batch size,
and the shared factor's E_ref comes from the whole batch).  Both ranks use cuda:0 and never wait on each other's
kernels — only the final all-gather is collective."""
import os
import socket
import tempfile

import numpy as np
import pytest

from pd_inputs import get_config, make_inputs

pytestmark = pytest.mark.gpu

KEYS = ("qT", "vT", "dq0", "dv0", "dE", "dnu")


def _run(inp):
    import torch
    import paper_2101_05917_b200 as pdb
    from oracle import adjoint   # the test's loss; the arrays below are the CUDA path's
    B, T, N = inp["B"], inp["T"], 3 * inp["n_nodes"]
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")
    cfg = inp["cfg"]
    sim = pdb.simulator_from_inputs(inp, tol_fwd=1e-12, tol_adj=1e-11, max_steps=T, accel_fwd=1, outer_warm=1)
    qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device="cuda")
    vt = torch.zeros_like(qt)
    act = None if inp["act"] is None else dev(inp["act"][:, :T])
    sim.forward(dev(inp["q0"]), dev(inp["v0"]), T, f_ext=dev(inp["f_ext"]), actuation=act, youngs=dev(inp["youngs"]),
                q_traj=qt, v_traj=vt)
    q, v = qt.cpu().numpy(), vt.cpu().numpy()
    gq, gv = np.zeros((B, N)), np.zeros((B, N))
    for b in range(B):
        _, gq[b], gv[b] = adjoint.loss_and_grad(inp, b, q[b, -1], v[b, -1])
    dq0 = torch.zeros((B, N), dtype=torch.float64, device="cuda")
    dv0 = torch.zeros_like(dq0)
    dE = torch.zeros(B, dtype=torch.float64, device="cuda")
    dnu = torch.zeros_like(dE)
    sim.backward(dev(gq), dev(gv), dq0, dv0, None, dE, dnu, None if act is None else torch.zeros_like(act))
    sim.close()
    return dict(qT=q[:, -1], vT=v[:, -1], dq0=dq0.cpu().numpy(), dv0=dv0.cpu().numpy(), dE=dE.cpu().numpy(),
                dnu=dnu.cpu().numpy())


def _worker(rank, world, port, name, out_path):
    import torch
    import torch.distributed as dist
    from paper_2101_05917_b200 import shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    inp = shard.shard_inputs(make_inputs(get_config(name)), world, rank)
    r = _run(inp)
    full = {}
    for k in KEYS:
        loc = torch.as_tensor(r[k].reshape(inp["B"], -1))
        full[k] = shard.gather_rows(loc, world).numpy()
    if rank == 0:
        np.savez(out_path, **full)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["c3s", "c5s"])
def test_two_rank_partition_is_bitwise_single_rank(name):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_05917_b200 as pdb
    pdb.build()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "sharded.npz")
        mp.spawn(_worker, args=(2, _free_port(), name, path), nprocs=2, join=True)
        got = dict(np.load(path))
    ref = _run(make_inputs(get_config(name)))
    for k in KEYS:
        assert np.array_equal(got[k], ref[k].reshape(got[k].shape)), k
