#!/usr/bin/env python
"""Benchmark: batched SE3 pose-graph GN iterations/sec (fwd + implicit bwd) at 1/2/4/8 B200 --
BASELINE.json's metric, on the configuration it is quoted on.

One STEP = the whole hot path on one batch: reset poses to theta_0, dnls_forward
(K GN iterations + the final undamped linearise+factor at theta_K, implicit mode), then
dnls_backward_implicit (adjoint solve on the cached factor + weight-gradient contraction +
fixed-order batch reduction), and for N > 1 GPUs ONE all_reduce of [grad_w_edge | grad_w_prior |
loss] (paper_2207_09442_b200.parallel.allreduce_shared_grads).
value = (batch elements of all ranks) * K / T, T = device time of the K timed steps, max over ranks.

Default workload: BASELINE.json configs[4] = C5, SE3 Cube graph, 1024 poses, global batch 2048 split
over the N GPUs (strong scaling: 2048 at N=1, 256 per GPU at N=8), GN K = 10, implicit backward.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run with N
ranks (one per GPU, NCCL).  --impl reference times the fp64 CPU oracle (the reference arm of this
tier) on a bounded sample.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched SE3 pose-graph GN iterations/sec (fwd+implicit bwd) at 1/2/4/8 B200"
UNIT = "problem-iterations/s"
L2_BYTES = 126 * 1024 * 1024

CONFIGS = {
    "C1": dict(N=16, dim=2, B=4, K=10, opt="gn", p=0.2, mode="local", scaling="weak",
               desc="C1: SE2 pose graph, 16 poses + loop closures, batch 4, GN K=10"),
    "C2": dict(N=256, dim=3, B=128, K=10, opt="gn", p=0.2, mode="local", scaling="weak",
               desc="C2: SE3 cube pose graph, 256 poses, batch 128 per GPU, GN K=10 + implicit backward"),
    "C3": dict(N=4096, dim=3, B=16, K=10, opt="lm", p=0.2, mode="local", scaling="weak",
               desc="C3: SE3 pose graph, 4096 poses, batch 16 per GPU, LM K=10 + implicit backward"),
    "C3r": dict(N=4096, dim=3, B=16, K=10, opt="lm", p=0.2, mode="random", scaling="weak",
                desc="C3r: SE3 pose graph, 4096 poses, random loop closures (large supernodes), batch 16, LM K=10"),
    "C4": dict(N=1024, dim=3, B=256, K=10, opt="gn", p=0.2, mode="local", scaling="weak",
               desc="C4: SE3 pose graph, 1024 poses, batch 256 per GPU, GN K=10 + implicit backward (learnable w)"),
    "C5": dict(N=1024, dim=3, B=2048, K=10, opt="gn", p=0.2, mode="local", scaling="strong",
               desc="C5: SE3 pose graph, 1024 poses, batch 2048 split over the GPUs, GN K=10 + implicit + NCCL allreduce"),
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_fp64_peak():
    """Measured fp64 peak (profiles/r2_fp64_peak.json: cuBLAS DGEMM 8192^3, tools/fp64_peak.py), else the
    B200 datasheet label."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_fp64_peak.json")) as f:
            return float(json.load(f)["dgemm_tflops"]), "measured DGEMM (profiles/r2_fp64_peak.json)"
    except Exception:
        return 37.0, "datasheet label (37 TF/s)"


def ncu_traffic(config, batch):
    """ncu DRAM bytes per launch of the dominant kernel recorded for this config and batch (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            ent = json.load(f).get(config)
        return ent if isinstance(ent, dict) and ent.get("batch") == batch else None
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock / throttle reasons via NVML every 20 ms while running."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, m in names.items():
                    if r & m and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- host-side step wiring
def shard(cfg: dict, world: int, rank: int) -> tuple[int, int]:
    """[b0, b1) of the global batch solved by `rank`: strong scaling splits the
    config's batch, weak scaling gives every rank the config's batch (global indices continue)."""
    from paper_2207_09442_b200.parallel import shard_range
    if cfg["scaling"] == "weak":
        return rank * cfg["B"], (rank + 1) * cfg["B"]
    return shard_range(cfg["B"], world, rank)


def reduce_step(ge, gp, obj, extra=()):
    """The step's only exchange: ONE all_reduce(SUM) of [grad_w_edge | grad_w_prior | loss | extra]
    (parallel.allreduce_shared_grads; identity on one rank).  Returns the reduced tensors."""
    from paper_2207_09442_b200.parallel import allreduce_shared_grads
    return allreduce_shared_grads(ge, gp, obj.sum().reshape(1), *extra)


# ----------------------------------------------------------------------------- CPU oracle legs
def cpu_oracle_step(topo, data, cfg, elements, backward="implicit", eps=1e-3, radius=None, K=None):
    """Oracle fwd (K iterations [+ final factor]) + implicit or DLM bwd on the listed elements."""
    from oracle import dlm as odlm
    from oracle import implicit as oimp
    from oracle import lie as olie
    from oracle import nls as onls
    G = "SE3" if cfg["dim"] == 3 else "SE2"
    K = cfg["K"] if K is None else K
    with_bwd = backward in ("implicit", "dlm")
    opt = onls.Options(optimizer=cfg["opt"], max_iterations=K, implicit=(backward == "implicit"))
    v = np.ones(topo.num_poses * (6 if cfg["dim"] == 3 else 3))
    for b in elements:
        prob = onls.PGOProblem(G, topo.num_poses, topo.edges, topo.prior_vars, data["meas"][b],
                               data["prior_meas"][b], data["w_edge"], data["w_prior"], radius=radius)
        res = onls.optimize(prob, olie.to_homog(data["poses0"][b]), opt)
        if backward == "dlm":
            odlm.dlm_weight_grads(prob, res.x, v, eps)
        elif with_bwd and res.L_final is not None:
            oimp.implicit_weight_grads(prob, res.x, v, L_K=res.L_final)


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"), default=None)
    except Exception:
        return None


def cpu_baseline(cfg, n_elems, backward="implicit", eps=1e-3, radius=None):
    import synth
    topo = synth.cube_topology(cfg["N"], dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
    data = synth.cube_batch(topo, n_elems, seed=0)
    t0 = time.perf_counter()
    cpu_oracle_step(topo, data, cfg, range(n_elems), backward, eps, radius)
    dt = time.perf_counter() - t0
    return {"value": n_elems * cfg["K"] / dt, "unit": UNIT, "cores": cores(), "blas_threads": blas_threads(),
            "kind": "oracle",
            "sample": f"{n_elems} element(s) of {cfg['desc'].split(':')[0]} (fwd K={cfg['K']} + final factor + "
                      f"{backward} bwd), {dt:.1f} s, numpy/OpenBLAS fp64 dense n={cfg['N'] * (6 if cfg['dim'] == 3 else 3)}"}


def run_reference(args, cfg, rank):
    """Reference arm of this tier: the fp64 CPU oracle as it stands.  One step = ONE GN iteration
    (dense linearise, dense Cholesky, solve, retraction, objective) of one batch element of the
    workload; the implicit backward's extra factorisation (1/K of the work) is not included, so the
    value is an upper bound of the oracle's rate."""
    if rank != 0:
        return
    import synth
    topo = synth.cube_topology(cfg["N"], dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
    n_el = 1
    data = synth.cube_batch(topo, n_el, seed=0)
    for _ in range(args.warmup):
        cpu_oracle_step(topo, data, cfg, range(n_el), backward="none", K=1)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_oracle_step(topo, data, cfg, range(n_el), backward="none", K=1)
        ts.append(time.perf_counter() - t0)
    T = sum(ts) / len(ts)
    val = n_el * 1 / T
    sample = (f"one GN iteration of {n_el} batch element per step (dense n={topo.num_poses * (6 if cfg['dim'] == 3 else 3)}"
              f" linearise + Cholesky + solve + retraction), fp64 NumPy/OpenBLAS oracle; the implicit backward's "
              f"extra factorisation is not timed (upper bound of the oracle's rate)")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": T * 1e3, "higher_is_better": True, "scaling": cfg["scaling"],
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "sample": sample, "poses": cfg["N"], "edges": topo.num_edges,
                   "iterations": cfg["K"]},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores(), "blas_threads": blas_threads(),
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- launcher
def relaunch_distributed(args):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run, N ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def nccl_init_summary():
    """nRanks / NVLS lines NCCL wrote during communicator init (NCCL_DEBUG=INFO to a file)."""
    out = []
    for f in sorted(glob.glob("/tmp/dnls_nccl.*.log")):
        try:
            for ln in open(f):
                if "nRanks" in ln or "NVLS" in ln or "comm 0x" in ln and "Init COMPLETE" in ln:
                    out.append(ln.strip()[-160:])
        except Exception:
            pass
    return out[:8]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="dnls", choices=["dnls", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-factor-roofline", action="store_true")
    ap.add_argument("--cpu-elements", type=int, default=None)
    ap.add_argument("--flush", choices=["auto", "always", "never"], default="auto",
                    help="flush L2 between timed steps (auto: only when the step's working set is < 2x L2)")
    ap.add_argument("--backward", default="implicit", choices=["implicit", "dlm", "unroll", "truncated"],
                    help="backward mode timed in the step (dlm: PAPER.md:259-271, one augmented GN step; "
                         "unroll / truncated: PAPER.md:235-239, backprop through the recorded GN iterations)")
    ap.add_argument("--trunc-steps", type=int, default=5, help="truncated backward: iterations differentiated")
    ap.add_argument("--iters", type=int, default=None, help="override the config's K")
    ap.add_argument("--epsilon", type=float, default=1e-3, help="DLM epsilon")
    ap.add_argument("--optimizer", default=None, choices=["gn", "lm", "dogleg"],
                    help="override the config's inner optimizer (dogleg: PAPER.md:153 trust region)")
    ap.add_argument("--cluster", type=int, default=0, choices=[0, 1, 2, 4, 8],
                    help="CTAs per batch element in the forward (0 = automatic)")
    ap.add_argument("--welsch", type=float, default=None,
                    help="Welsch radius of the Between edges (PAPER.md:168 robust PGO); default: quadratic costs")
    ap.add_argument("--batch", type=int, default=None, help="override the config's (global) batch")
    ap.add_argument("--interleave", type=int, default=0, choices=[0, 1, 32],
                    help="dnls_options.batch_interleave: 0 automatic, 1 one CTA per element, 32 batch-interleaved "
                         "level-major path")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo + --share-gpu: multi-rank wiring test on one GPU)")
    ap.add_argument("--share-gpu", action="store_true", help="every rank uses cuda:0 (testing on a 1-GPU box)")
    ap.add_argument("--dump-shard", default=None, help="write this rank's theta_K / grads to <path>.rank<r>.npz")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.optimizer:
        cfg["opt"] = args.optimizer
    if args.batch:
        cfg["B"] = args.batch
    if args.iters is not None:
        cfg["K"] = args.iters
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_distributed(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist

    import synth
    from paper_2207_09442_b200 import dnls as D
    from paper_2207_09442_b200.layer import PoseGraphSolver

    dev_index = 0 if args.share_gpu else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if args.dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/dnls_nccl.%h.%p.log")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    # ---- data: per-rank shard of the global batch (per-element seeds -> shard independent)
    b0, b1 = shard(cfg, world, rank)
    B = b1 - b0
    topo = synth.cube_topology(cfg["N"], dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
    data = synth.cube_batch(topo, B, seed=0, b_start=b0)
    d = 6 if cfg["dim"] == 3 else 3
    group = D.SE3 if cfg["dim"] == 3 else D.SE2
    K = cfg["K"]
    t_sym = time.perf_counter()
    solver = PoseGraphSolver(group, topo.num_poses, topo.edges, topo.prior_vars, device=dev_index,
                             max_iterations=K, optimizer={"gn": D.GN, "lm": D.LM, "dogleg": D.DOGLEG}[cfg["opt"]])
    t_sym = time.perf_counter() - t_sym
    g = solver.graph
    st = solver.stats
    opt = solver.options
    dlm = args.backward == "dlm"
    unroll = args.backward in ("unroll", "truncated")
    opt.cluster_ctas = args.cluster
    opt.batch_interleave = args.interleave
    opt.backward_mode = {"implicit": D.BWD_IMPLICIT, "dlm": D.BWD_NONE, "unroll": D.BWD_UNROLL,
                         "truncated": D.BWD_TRUNCATED}[args.backward]
    opt.backward_steps = args.trunc_steps
    host = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in data.items() if k != "gt"}
    vgrad = torch.from_numpy(np.stack([np.random.default_rng([1, b]).standard_normal((topo.num_poses, d))
                                       for b in range(b0, b1)]))
    dv = {k: v.to(dev) for k, v in host.items()}
    dvg = vgrad.to(dev)
    poses = torch.empty_like(dv["poses0"])
    obj = torch.empty(B, dtype=torch.float64, device=dev)
    sts = torch.empty(B, dtype=torch.int32, device=dev)
    its = torch.empty(B, dtype=torch.int32, device=dev)
    E, P = topo.num_edges, int(topo.prior_vars.shape[0])
    ge = torch.zeros(E, dtype=torch.float64, device=dev)
    gp = torch.zeros(P, dtype=torch.float64, device=dev)
    ws = solver.workspace(B, opt)
    rad = None if args.welsch is None else torch.tensor([args.welsch], dtype=torch.float64, device=dev)
    gr = None if rad is None else torch.zeros(1, dtype=torch.float64, device=dev)
    prob = D.make_problem(poses, dv["meas"], dv["prior_meas"], dv["w_edge"], dv["w_prior"], obj, sts, its,
                          radius=rad)
    stream = torch.cuda.current_stream()
    # the step's working set: factor storage + per-slot scratch of the workspace, poses, measurements
    ws_bytes = ws.numel() + sum(v.numel() * v.element_size() for v in dv.values())
    flush_on = args.flush == "always" or (args.flush == "auto" and ws_bytes < 2 * L2_BYTES)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev) if flush_on else None
    reduced = [None]

    def step(record=None):
        poses.copy_(dv["poses0"])
        if record is not None:
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        D.dnls_forward(g, B, opt, prob, ws)
        if record is not None:
            b_.record(stream)
            record.append((a, b_))
        if dlm:
            D.dnls_backward_dlm(g, B, prob, dvg, D.GRAD_TANGENT, args.epsilon, ge, gp, 0, ws, grad_radius=gr)
        elif unroll:
            D.dnls_backward_unroll(g, B, prob, dvg, D.GRAD_TANGENT, ge, gp, 0, ws)
        else:
            D.dnls_backward_implicit(g, B, prob, dvg, D.GRAD_TANGENT, ge, gp, 0, ws, grad_radius=gr)
        reduced[0] = reduce_step(ge, gp, obj, () if gr is None else (gr,))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev_index).start()
    D.dnls_debug_launch_count(reset=True)
    ev_f, per_step = [], []
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(ev_f)
        e1.record(stream)
        per_step.append((e0, e1))
    t1.record(stream)
    launches = D.dnls_debug_launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    steps_ms = [a.elapsed_time(b) for a, b in per_step]
    # the timed region: the K steps end to end (with a flush the flush writes are excluded: sum of steps)
    T = (sum(steps_ms) if flush is not None else t0.elapsed_time(t1)) / 1e3
    Tf = sum(a.elapsed_time(b) for a, b in ev_f) / 1e3 / args.steps
    if world > 1:
        tt = torch.tensor([T, Tf], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        T, Tf = tt.tolist()
    total_elems = cfg["B"] if cfg["scaling"] == "strong" else B * world
    value = total_elems * K * args.steps / T
    ms_per_step = T / args.steps * 1e3

    if args.dump_shard:
        np.savez(f"{args.dump_shard}.rank{rank}.npz", poses=poses.cpu().numpy(), obj=obj.cpu().numpy(),
                 grads=torch.cat([r.reshape(-1) for r in reduced[0]]).cpu().numpy(), b0=b0, b1=b1)

    # ---- roofline of the dominant kernel.  Algorithmic bytes per SURVEY.md 8(d): a GN iteration moves
    # lin + factor + solve + update bytes per element (dnls_graph_stats), a factorisation 16 nnz(L) per element.
    per_iter = st["bytes_linearize"] + st["bytes_factor"] + st["bytes_solve"] + st["bytes_update"]
    alg_bytes = B * (K * per_iter + (0 if (dlm or unroll) else st["bytes_linearize"] + st["bytes_factor"]))
    peak, peak_src = load_peaks()
    fp64_peak, fp64_src = load_fp64_peak()
    tent = ncu_traffic(args.config, B)
    fbytes = 16.0 * st["nnz_L"] * B
    fflops = float(st["factor_flops"]) * B

    # the batch-interleaved path: CUDA events around each of the K + 1 factorisations of one forward
    # (DNLS_PHASE_TIMING) -- the numeric-factorisation kernel of north_star, timed in the configuration above
    os.environ["DNLS_PHASE_TIMING"] = "1"
    poses.copy_(dv["poses0"])
    D.dnls_forward(g, B, opt, prob, ws)
    del os.environ["DNLS_PHASE_TIMING"]
    phases = D.dnls_debug_phase_times(g)
    path = "batch-interleaved level-major (bl.cuh)" if phases else "one CTA per element (k_forward)"
    if phases:
        pm = statistics.median(phases)
        traffic = tent.get("dram_bytes_per_launch") if tent else None
        roofline = {
            "bound": "hbm", "achieved": fbytes / (pm / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
            "frac": fbytes / (pm / 1e3) / 1e9 / peak, "traffic": traffic,
            "traffic_over_algorithmic": None if traffic is None else traffic / fbytes,
            "kernel": "numeric factorisation: bl_subtree (the bottom subtrees of the elimination tree, one launch) + "
                      "per-level bl_update_items (chunked update lists) + bl_factor_red, PDL launches (one "
                      "factorisation of the batch)",
            "peak_source": peak_src, "alg_bytes_per_launch": fbytes, "kernel_ms": pm, "kernel_ms_min": min(phases),
            "factorisations_ms": phases,
            "fp64": {"flops_per_launch": fflops, "achieved_tflops": fflops / (pm / 1e3) / 1e12,
                     "peak_tflops": fp64_peak, "frac": fflops / (pm / 1e3) / 1e12 / fp64_peak,
                     "peak_source": fp64_src},
            "forward": {"kernels": "whole dnls_forward (K GN iterations + final factorisation)",
                        "alg_bytes": alg_bytes, "ms": Tf * 1e3, "frac": alg_bytes / Tf / 1e9 / peak},
            "traffic_source": tent.get("source") if tent else None,
            "note": "algorithmic bytes 16 nnz(L) B per factorisation (SURVEY.md 8(d) a3), median over the K+1 "
                    "factorisations of one forward (CUDA events on the stream); traffic = ncu dram read+write per "
                    "factorisation (cold-cache launch list, profiles/ncu_traffic.json): the left-looking updates "
                    "re-read source blocks that do not stay in L2",
        }
    else:
        traffic = tent.get("dram_bytes_per_launch") if tent else None
        roofline = {"bound": "hbm", "achieved": alg_bytes / Tf / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": alg_bytes / Tf / 1e9 / peak, "traffic": traffic, "kernel": "k_forward",
                    "peak_source": peak_src, "alg_bytes_per_launch": alg_bytes, "kernel_ms": Tf * 1e3,
                    "note": "algorithmic bytes = B*(K*(lin+factor+solve+update)" +
                            ("" if (dlm or unroll) else "+lin+factor") +
                            ") per SURVEY.md 8(d); traffic = ncu dram read+write of one launch (profiles/ncu_traffic.json)"}
        # factor-only leg: dnls_factorize on the assembled H(theta_0) of the same batch
        if not args.no_factor_roofline:
            fprob = D.make_problem(dv["poses0"], dv["meas"], dv["prior_meas"], dv["w_edge"], dv["w_prior"])
            fts = []
            for r in range(args.warmup + args.steps):
                D.dnls_linearize(g, B, fprob, None, D.DAMP_MARQUARDT, ws)
                a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                D.dnls_factorize(g, B, ws, sts)
                b_.record(stream)
                if r >= args.warmup:
                    fts.append((a, b_))
            torch.cuda.synchronize()
            fms = [a.elapsed_time(b) for a, b in fts]
            tfac = statistics.median(fms) / 1e3
            roofline["factor"] = {"kernel": "k_factorize", "bound": "hbm", "achieved": fbytes / tfac / 1e9,
                                  "peak": peak, "unit": "GB/s", "frac": fbytes / tfac / 1e9 / peak,
                                  "alg_bytes_per_launch": fbytes, "kernel_ms_median": tfac * 1e3,
                                  "kernel_ms_min": min(fms), "flops_per_launch": fflops,
                                  "fp64_frac": fflops / tfac / 1e12 / fp64_peak,
                                  "note": "16 nnz(L) B per launch (SURVEY.md 8(d) a3), standalone dnls_factorize"}

    # ---- e2e through the public API (PoseGraphSolver) with pinned host buffers: H2D of the step's inputs,
    # D2H of theta_K, the objective and the (reduced) gradients
    e2e = None
    if not args.no_e2e:
        pin = {k: v.pin_memory() for k, v in host.items()}
        pvg = vgrad.pin_memory()
        out_obj = torch.empty(B, dtype=torch.float64).pin_memory()
        out_pose = torch.empty(host["poses0"].shape, dtype=torch.float64).pin_memory()
        out_g = torch.empty(E + P + 1 + (0 if rad is None else 1), dtype=torch.float64).pin_memory()
        bi = sum(v.numel() * v.element_size() for v in pin.values()) + pvg.numel() * 8
        bo = out_obj.numel() * 8 + out_g.numel() * 8 + out_pose.numel() * 8
        # double-buffered device inputs: the H2D of step i+1 (copy stream) and the D2H of step i's results (a
        # second copy stream) overlap the compute of step i, as a serving pipeline would run; every step still
        # moves all of its inputs and results across PCIe inside the timed region (start event -> last D2H)
        nbuf = 2
        dbufs = [{k: torch.empty_like(v, device=dev) for k, v in pin.items()} for _ in range(nbuf)]
        dvgs = [torch.empty_like(pvg, device=dev) for _ in range(nbuf)]
        s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(nbuf)]     # inputs of buffer j have landed
        ev_free = [torch.cuda.Event() for _ in range(nbuf)]   # the compute reading buffer j has finished

        def e2e_load(j):
            s_h2d.wait_event(ev_free[j])
            with torch.cuda.stream(s_h2d):
                for k in pin:
                    dbufs[j][k].copy_(pin[k], non_blocking=True)
                dvgs[j].copy_(pvg, non_blocking=True)
            ev_in[j].record(s_h2d)

        def e2e_compute(j):
            stream.wait_event(ev_in[j])
            db = dbufs[j]
            P_, o_, _, _ = solver.forward(db["poses0"], db["meas"], db["prior_meas"], db["w_edge"],
                                          db["w_prior"], radius=rad, backward_mode=opt.backward_mode,
                                          backward_steps=args.trunc_steps)
            gs = solver.backward(P_, db["meas"], db["prior_meas"], db["w_edge"], db["w_prior"], dvgs[j],
                                 D.GRAD_TANGENT, mode="unroll" if unroll else args.backward, epsilon=args.epsilon,
                                 radius=rad)
            red = reduce_step(gs[0], gs[1], o_, tuple(gs[2:]))
            gcat = torch.cat([r.reshape(-1) for r in red])
            ev_free[j].record(stream)
            s_d2h.wait_event(ev_free[j])
            with torch.cuda.stream(s_d2h):
                for t in (gcat, o_, P_):
                    t.record_stream(s_d2h)
                out_g.copy_(gcat, non_blocking=True)
                out_obj.copy_(o_, non_blocking=True)
                out_pose.copy_(P_, non_blocking=True)

        def e2e_run(n, start=None):
            if start is not None:
                s_h2d.wait_event(start)
            e2e_load(0)
            for i in range(n):
                if i + 1 < n:
                    e2e_load((i + 1) % nbuf)
                e2e_compute(i % nbuf)
            stream.wait_stream(s_d2h)

        e2e_run(args.warmup)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if flush is not None:
            flush.fill_(1)
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_run(args.steps, start=a)
        b_.record(stream)
        torch.cuda.synchronize()
        Te = a.elapsed_time(b_) / 1e3
        if world > 1:
            tt = torch.tensor([Te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            Te = tt.item()
        e2e = {"value": total_elems * K * args.steps / Te, "unit": UNIT, "h2d_bytes_per_step": int(bi),
               "d2h_bytes_per_step": int(bo), "ms_per_step": Te / args.steps * 1e3,
               "note": "every step: pinned host inputs -> device, PoseGraphSolver.forward/backward, all_reduce, "
                       "theta_K + objective + gradients -> host; double-buffered inputs, the copies of adjacent "
                       "steps overlap the compute (two copy streams); time = start event -> last D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not unroll:
        n_el = args.cpu_elements if args.cpu_elements else (1 if cfg["N"] >= 1024 else 4)
        cpu = cpu_baseline(cfg, n_el, args.backward, args.epsilon, args.welsch)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "global_batch": total_elems, "batch_per_gpu": B,
                       "poses": cfg["N"], "edges": topo.num_edges, "iterations": K,
                       "optimizer": cfg["opt"], "backward": args.backward,
                       "backward_steps": args.trunc_steps if args.backward == "truncated" else None,
                       "workspace_bytes": int(ws.numel()),
                       "robust": "none" if args.welsch is None else f"welsch k={args.welsch}",
                       "l2": ("flushed between timed steps (256 MB write)" if flush is not None else
                              f"not flushed: the step's working set ({ws_bytes / 2**30:.2f} GiB per GPU) is larger "
                              f"than L2"),
                       "parallelism": f"dp{world}", "path": path, "nnz_L": st["nnz_L"], "supernodes": st["num_supernodes"],
                       "levels": st["num_levels"], "symbolic_ms": t_sym * 1e3},
            "step_ms": {"median": statistics.median(steps_ms), "min": min(steps_ms), "max": max(steps_ms)},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            # the library's own kernel launches inside the timed region (dnls_debug_launch_count)
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if world > 1:
            line["dist"] = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                            "nccl_init": nccl_init_summary() if args.dist_backend == "nccl" else None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
