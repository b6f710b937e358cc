"""Experiment: the C5 batch as S sub-batches on S CUDA streams (batch-interleaved path), so the latency-bound
upper-level launches of one sub-batch overlap with another's work.  Prints ms per fwd+bwd step for S = 1, 2, 4.
usage: python tools/two_streams.py [C5] [steps]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2207_09442_b200 import dnls as D  # noqa: E402
from paper_2207_09442_b200.layer import PoseGraphSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS[name]
B, K = cfg["B"], cfg["K"]
topo = synth.cube_topology(cfg["N"], dim=3, p=cfg["p"], mode=cfg["mode"], seed=0)
data = synth.cube_batch(topo, B, seed=0)
dev = torch.device("cuda", 0)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in data.items() if k != "gt"}
v = torch.randn(B, cfg["N"], 6, dtype=torch.float64, device=dev)
for S in (1, 2, 4):
    Bs = B // S
    streams = [torch.cuda.Stream() for _ in range(S)]
    subs = []
    for s in range(S):
        sl = slice(s * Bs, (s + 1) * Bs)
        solver = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=K)
        g, opt = solver.graph, solver.options
        opt.backward_mode = D.BWD_IMPLICIT
        ws = solver.workspace(Bs, opt)
        poses = t["poses0"][sl].clone()
        obj = torch.empty(Bs, dtype=torch.float64, device=dev)
        st = torch.empty(Bs, dtype=torch.int32, device=dev)
        it = torch.empty(Bs, dtype=torch.int32, device=dev)
        prob = D.make_problem(poses, t["meas"][sl], t["prior_meas"][sl], t["w_edge"], t["w_prior"], obj, st, it)
        ge = torch.zeros(topo.num_edges, dtype=torch.float64, device=dev)
        gp = torch.zeros(1, dtype=torch.float64, device=dev)
        subs.append((g, opt, ws, poses, prob, ge, gp, t["poses0"][sl], v[sl].contiguous()))

    def step():
        cur = torch.cuda.current_stream()
        ev0 = torch.cuda.Event()
        ev0.record(cur)
        for s, (g, opt, ws, poses, prob, ge, gp, p0, vv) in enumerate(subs):
            with torch.cuda.stream(streams[s]):
                streams[s].wait_event(ev0)
                poses.copy_(p0)
                D.dnls_forward(g, Bs, opt, prob, ws, stream=streams[s])
                D.dnls_backward_implicit(g, Bs, prob, vv, D.GRAD_TANGENT, ge, gp, 0, ws, stream=streams[s])
        for s in range(S):
            e = torch.cuda.Event()
            e.record(streams[s])
            cur.wait_event(e)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    print(f"{name} S={S} sub-batch {Bs}: {ms:.2f} ms per step, {B * K / ms * 1e3:.0f} problem-iter/s")
