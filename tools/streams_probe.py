#!/usr/bin/env python
"""Developer probe: one configured batch run as S concurrent handles (contiguous blocks of sims, one CUDA stream
and one host thread each) vs one handle; device time of forward+backward and bitwise equality of the results.

    python tools/streams_probe.py c5 --horizon 20 --streams 2
"""
import argparse
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--horizon", type=int, default=20)
    ap.add_argument("--streams", type=int, default=2)
    a = ap.parse_args()
    import torch
    import paper_2101_05917_b200 as pdb
    from paper_2101_05917_b200 import shard
    from pd_inputs import get_config, make_inputs
    cfg = get_config(a.config)
    T = a.horizon
    full = make_inputs(cfg, steps=T)

    class Lane:
        def __init__(self, inp):
            self.inp = inp
            self.sim = pdb.simulator_from_inputs(inp, tol_fwd=cfg.tol, tol_adj=cfg.tol, max_steps=T, accel_fwd=1,
                                                 outer_warm=1)
            D = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
            B, N = inp["B"], 3 * inp["n_nodes"]
            self.args = [D(inp["q0"]), D(inp["v0"]), D(inp["f_ext"]), D(inp["youngs"])]
            self.act = None if inp["act"] is None else D(inp["act"])
            self.cq, self.cv = D(inp["c_q"]), D(inp["c_v"])
            self.qt = torch.zeros((B, T + 1, N), dtype=torch.float64, device="cuda")
            self.vt = torch.zeros_like(self.qt)
            self.dq0 = torch.zeros((B, N), dtype=torch.float64, device="cuda")
            self.dE = torch.zeros(B, dtype=torch.float64, device="cuda")
            self.stream = torch.cuda.Stream()

        def step(self):
            with torch.cuda.stream(self.stream):
                self.sim.forward(self.args[0], self.args[1], T, f_ext=self.args[2], actuation=self.act,
                                 youngs=self.args[3], q_traj=self.qt, v_traj=self.vt)
                self.sim.backward(self.cq, self.cv, self.dq0, None, None, self.dE)

    def run(lanes):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for ln in lanes:
            ln.stream.wait_event(e0)
        th = [threading.Thread(target=ln.step) for ln in lanes]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for ln in lanes:
            torch.cuda.current_stream().wait_stream(ln.stream)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    one = [Lane(full)]
    many = [Lane(shard.shard_inputs(full, a.streams, r)) for r in range(a.streams)]
    for _ in range(2):
        run(one)
        run(many)
    t1 = min(run(one) for _ in range(2))
    ts = min(run(many) for _ in range(2))
    q1 = one[0].qt.cpu().numpy()
    qs = np.concatenate([ln.qt.cpu().numpy() for ln in many], 0)
    d1 = one[0].dq0.cpu().numpy()
    ds = np.concatenate([ln.dq0.cpu().numpy() for ln in many], 0)
    print(f"{a.config} T={T}: 1 handle {t1:.1f} ms, {a.streams} concurrent handles {ts:.1f} ms "
          f"(x{t1 / ts:.2f}); bitwise equal q: {np.array_equal(q1, qs)}, dL/dq0: {np.array_equal(d1, ds)}")


if __name__ == "__main__":
    main()
