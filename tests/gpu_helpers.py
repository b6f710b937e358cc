"""Shared helpers for the -m gpu parity tests: seeded inputs from synth/, oracle references
from oracle/, CUDA results through the C-ABI binding (paper_2207_09442_b200.dnls)."""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import implicit as oimp
from oracle import lie as olie
from oracle import nls as onls
from paper_2207_09442_b200 import dnls as D

DEV = torch.device("cuda", 0)

# tolerances (north_star: 1e-9 relative on solutions and objectives, 1e-6 on implicit gradients)
TOL_POSE = 1e-9
TOL_OBJ = 1e-9
TOL_GRAD = 1e-6


def to_dev(data):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for k, v in data.items()}


def make_case(N, dim=3, p=0.2, mode="local", seed=0, B=4, b_start=0, **noise):
    topo = synth.cube_topology(N, dim=dim, p=p, mode=mode, seed=seed)
    data = synth.cube_batch(topo, B, seed=seed, b_start=b_start, **noise)
    return topo, data


def oracle_results(topo, data, elements=None, **opt):
    G = "SE3" if topo.dim == 3 else "SE2"
    o = onls.Options(**opt)
    return onls.solve_batch(G, topo.num_poses, topo.edges, topo.prior_vars, data["poses0"], data["meas"],
                            data["prior_meas"], data["w_edge"], data["w_prior"], o, elements=elements,
                            radius=data.get("radius"))


def oracle_problem(topo, data, b):
    G = "SE3" if topo.dim == 3 else "SE2"
    we = data["w_edge"][b] if data["w_edge"].ndim == 2 else data["w_edge"]
    wp = data["w_prior"][b] if data["w_prior"].ndim == 2 else data["w_prior"]
    r = data.get("radius")
    rk = None if r is None else float(np.asarray(r).reshape(-1)[b if np.size(r) > 1 else 0])
    return onls.PGOProblem(G, topo.num_poses, topo.edges, topo.prior_vars, data["meas"][b], data["prior_meas"][b],
                           we, wp, radius=rk)


def pose_err(P_gpu, T_oracle_homog):
    ref = olie.from_homog(T_oracle_homog)
    return float(np.max(np.abs(P_gpu - ref)) / max(1.0, np.max(np.abs(ref))))


def rel_vec_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def graph_for(topo, device=0):
    group = D.SE3 if topo.dim == 3 else D.SE2
    return D.dnls_graph_create(group, topo.num_poses, topo.edges, topo.prior_vars, device)


def perm_matrix_indices(g):
    """Scalar permutation: H_perm = H[idx][:, idx] with idx from the pose permutation."""
    perm = D.dnls_graph_perm(g)
    d = g.d
    return (perm[:, None] * d + np.arange(d)[None, :]).reshape(-1)


__all__ = ["DEV", "TOL_POSE", "TOL_OBJ", "TOL_GRAD", "to_dev", "make_case", "oracle_results", "oracle_problem",
           "pose_err", "rel_vec_err", "graph_for", "perm_matrix_indices", "oimp", "olie", "onls", "D", "synth"]
