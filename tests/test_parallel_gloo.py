"""Not-gpu tests of the batch-sharding / gradient-reduction logic (SURVEY.md §8(e), §4
"multi-node without a cluster"): world size 2 over gloo on CPU, the oracle as the per-shard
compute.  Per-element results of a 2-rank run are bitwise identical to the 1-rank run (seeds
per global element); the all-reduced weight gradient equals the full-batch sum to 1e-12."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import implicit as oimp
from oracle import lie as olie
from oracle import nls as onls
from paper_2207_09442_b200.parallel import allreduce_weight_grads, max_over_ranks, shard_range

N, GB, K = 16, 6, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard_compute(b0, b1):
    """Oracle fwd + implicit bwd for global elements [b0, b1): poses, objective, grad_w sums."""
    topo = synth.cube_topology(N, dim=2, p=0.7, seed=3)
    data = synth.cube_batch(topo, b1 - b0, seed=3, b_start=b0)
    res = onls.solve_batch("SE2", N, topo.edges, topo.prior_vars, data["poses0"], data["meas"], data["prior_meas"],
                           data["w_edge"], data["w_prior"], onls.Options(max_iterations=K, implicit=True))
    ge = np.zeros(topo.num_edges)
    gp = np.zeros(1)
    loss = 0.0
    poses = []
    for bl, r in enumerate(res):
        prob = onls.PGOProblem("SE2", N, topo.edges, topo.prior_vars, data["meas"][bl], data["prior_meas"][bl],
                               data["w_edge"], data["w_prior"])
        v = np.random.default_rng([7, b0 + bl]).standard_normal(N * 3)
        a, c, _ = oimp.implicit_weight_grads(prob, r.x, v, L_K=r.L_final)
        ge += a
        gp += c
        loss += r.objective
        poses.append(olie.from_homog(r.x))
    return np.stack(poses), ge, gp, loss


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b0, b1 = shard_range(GB, world, rank)
    poses, ge, gp, loss = shard_compute(b0, b1)
    g1, g2, l = allreduce_weight_grads(torch.from_numpy(ge), torch.from_numpy(gp), torch.tensor([loss], dtype=torch.float64))
    t = max_over_ranks(float(rank))
    out[rank] = (b0, b1, poses, g1.numpy(), g2.numpy(), float(l.item()), t)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    for gb in (1, 7, 128, 2048):
        for world in (1, 2, 3, 8):
            r = [shard_range(gb, world, k) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == gb
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_two_rank_gloo_matches_single_rank():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    full_poses, ge, gp, loss = shard_compute(0, GB)
    for r in range(2):
        b0, b1, poses, g1, g2, l, t = out[r]
        assert np.array_equal(poses, full_poses[b0:b1])               # bitwise per element
        assert np.max(np.abs(g1 - ge)) <= 1e-12 * np.max(np.abs(ge))  # only the summation order differs
        assert abs(g2[0] - gp[0]) <= 1e-12 * abs(gp[0]) + 1e-300
        assert abs(l - loss) <= 1e-12 * loss
        assert t == 1.0                                              # max over ranks


def shard_compute_robust(b0, b1, radius=0.4, eps=1e-3):
    """Welsch kernel (shared learnable radius) + DLM backward per element: weight and radius
    gradients of the shard."""
    from oracle import dlm as odlm
    topo = synth.cube_topology(N, dim=2, p=0.7, seed=5, outlier_ratio=0.3)
    data = synth.cube_batch(topo, b1 - b0, seed=5, b_start=b0)
    res = onls.solve_batch("SE2", N, topo.edges, topo.prior_vars, data["poses0"], data["meas"], data["prior_meas"],
                           data["w_edge"], data["w_prior"], onls.Options(max_iterations=K), radius=radius)
    ge, gp, gr = np.zeros(topo.num_edges), np.zeros(1), np.zeros(1)
    for bl, r in enumerate(res):
        prob = onls.PGOProblem("SE2", N, topo.edges, topo.prior_vars, data["meas"][bl], data["prior_meas"][bl],
                               data["w_edge"], data["w_prior"], radius=radius)
        v = np.random.default_rng([9, b0 + bl]).standard_normal(N * 3)
        a, c, Td = odlm.dlm_weight_grads(prob, r.x, v, eps)
        ge += a
        gp += c
        gr += odlm.dlm_radius_grad(prob, r.x, Td, eps)
    return ge, gp, gr


def _worker_robust(rank, world, port, out):
    from paper_2207_09442_b200.parallel import allreduce_shared_grads
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b0, b1 = shard_range(GB, world, rank)
    ge, gp, gr = shard_compute_robust(b0, b1)
    g1, g2, g3 = allreduce_shared_grads(torch.from_numpy(ge), torch.from_numpy(gp), torch.from_numpy(gr))
    out[rank] = (g1.numpy(), g2.numpy(), g3.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shared_radius_and_dlm():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker_robust, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ge, gp, gr = shard_compute_robust(0, GB)
    for r in range(2):
        g1, g2, g3 = out[r]
        assert np.max(np.abs(g1 - ge)) <= 1e-12 * np.max(np.abs(ge))
        assert abs(g2[0] - gp[0]) <= 1e-12 * abs(gp[0]) + 1e-300
        assert abs(g3[0] - gr[0]) <= 1e-12 * abs(gr[0]) + 1e-300


# ---- bench.py's own step wiring (shard() + reduce_step(), the code the timed step runs), 2 ranks over gloo
def _bench_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    cfg = dict(bench.CONFIGS["C5"])
    b0, b1 = bench.shard(cfg, world, rank)
    cfgw = dict(bench.CONFIGS["C2"])
    w0, w1 = bench.shard(cfgw, world, rank)
    poses, ge, gp, loss = shard_compute(*shard_range(GB, world, rank))
    obj = torch.tensor([loss, 0.0], dtype=torch.float64)   # reduce_step sums the per-element objectives
    red = bench.reduce_step(torch.from_numpy(ge), torch.from_numpy(gp), obj)
    out[rank] = ((b0, b1), (w0, w1), [r.numpy().copy() for r in red])
    dist.destroy_process_group()


def test_bench_step_wiring_two_ranks():
    import bench
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bench_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    # strong scaling (C5): contiguous halves of the 2048 global elements; weak (C2): 128 per rank
    assert out[0][0] == (0, 1024) and out[1][0] == (1024, 2048)
    assert out[0][1] == (0, 128) and out[1][1] == (128, 256)
    assert bench.shard(dict(bench.CONFIGS["C5"]), 1, 0) == (0, 2048)
    # the reduced gradients / loss equal the single-rank full-batch values (both ranks hold the same)
    _, ge1, gp1, l1 = shard_compute(0, GB)
    for r in range(world):
        ge, gp, loss = out[r][2]
        assert np.max(np.abs(ge - ge1)) <= 1e-12 * np.max(np.abs(ge1))
        assert np.max(np.abs(gp - gp1)) <= 1e-12 * np.max(np.abs(gp1))
        assert abs(loss[0] - l1) <= 1e-12 * l1
    assert all(np.array_equal(a, b) for a, b in zip(out[0][2], out[1][2]))
