"""Pinned synthetic "Cube" pose-graph generator.

The paper gives only the knobs of its simulated Cube dataset -- number of poses,
loop-closure probability, outlier ratio (App. E.1, App. G.2).
Everything else here is our own pinned choice and is stated in DESIGN.md:

* ground-truth positions: the first N cells of a boustrophedon walk of an s^3 grid
  (s^2 in 2D), unit spacing; ground-truth rotations Haar-random (SE3, normalised
  Gaussian quaternion) or uniform angle (SE2);
* topology (shared by the batch, rng = default_rng([seed, 0])): odometry edges
  (k, k+1), then for k = 2..N-1 with probability p one loop closure (j, k), j < k-1,
  either to an earlier grid neighbour ("local", default) or uniform ("random");
* per batch element b (rng = default_rng([seed, 1, b]) with b the GLOBAL index, so
  data do not depend on how the batch is sharded): measurement noise and initial
  perturbation of the ground truth.

Noise model (deliberately NOT the method's Exp map, so this module holds none of the
method's arithmetic): a noise pose is [R(phi) | eps_t] where R(phi) is the rotation of
the unit quaternion normalise(1, phi/2) (a Gibbs/Cayley small rotation), phi ~
N(0, sigma_r^2 I) and eps_t ~ N(0, sigma_t^2 I).  In 2D the noise rotation is
R2(eps_theta).  Measurements Z_e = (T_i^gt)^-1 T_j^gt N_e, initial poses
T_k^0 = T_k^gt N_k.  All arrays are float64 and C-contiguous, poses stored as the top
rows of the homogeneous matrix: SE3 -> [3][4], SE2 -> [2][3] (row-major [R | t]).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def quat_to_rot(q: np.ndarray) -> np.ndarray:
    """Unit quaternion(s) (w, x, y, z) [..., 4] -> rotation matrices [..., 3, 3]."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def rot2(theta: np.ndarray) -> np.ndarray:
    """Planar rotation matrices [..., 2, 2]."""
    theta = np.asarray(theta, dtype=np.float64)
    c, s = np.cos(theta), np.sin(theta)
    R = np.empty(theta.shape + (2, 2))
    R[..., 0, 0] = c
    R[..., 0, 1] = -s
    R[..., 1, 0] = s
    R[..., 1, 1] = c
    return R


def _homog(R: np.ndarray, t: np.ndarray) -> np.ndarray:
    dim = R.shape[-1]
    T = np.zeros(R.shape[:-2] + (dim + 1, dim + 1))
    T[..., :dim, :dim] = R
    T[..., :dim, dim] = t
    T[..., dim, dim] = 1.0
    return T


def _inv_homog(T: np.ndarray) -> np.ndarray:
    dim = T.shape[-1] - 1
    R = T[..., :dim, :dim]
    t = T[..., :dim, dim]
    Rt = np.swapaxes(R, -1, -2)
    return _homog(Rt, -np.einsum("...ij,...j->...i", Rt, t))


def _grid_walk(N: int, dim: int) -> np.ndarray:
    """First N cells of a boustrophedon walk of an s^dim grid (consecutive cells adjacent)."""
    s = max(1, math.ceil(round(N ** (1.0 / dim), 12)))
    while s ** dim < N:
        s += 1
    cells = []
    row = 0
    layers = range(s) if dim == 3 else [0]
    for z in layers:
        ys = range(s) if z % 2 == 0 else range(s - 1, -1, -1)
        for y in ys:
            xs = range(s) if row % 2 == 0 else range(s - 1, -1, -1)
            for x in xs:
                cells.append((x, y, z) if dim == 3 else (x, y))
            row += 1
    return np.asarray(cells[:N], dtype=np.int64)


@dataclass
class CubeTopology:
    dim: int                 # 2 (SE2) or 3 (SE3)
    num_poses: int
    edges: np.ndarray        # int32 [E][2]  (i, j): measurement of T_i^-1 T_j
    prior_vars: np.ndarray   # int32 [P]
    gt: np.ndarray           # float64 [N][dim][dim+1]  ground-truth poses (top rows)
    outlier: np.ndarray      # bool [E]
    num_closures: int

    @property
    def num_edges(self) -> int:
        return int(self.edges.shape[0])


def cube_topology(N: int, dim: int = 3, p: float = 0.2, mode: str = "local",
                  seed: int = 0, outlier_ratio: float = 0.0) -> CubeTopology:
    """Topology + ground truth shared by the whole batch (rng = default_rng([seed, 0]))."""
    if dim not in (2, 3):
        raise ValueError("dim must be 2 or 3")
    if N < 2:
        raise ValueError("N >= 2 required")
    if mode not in ("local", "random"):
        raise ValueError("mode must be 'local' or 'random'")
    rng = np.random.default_rng([seed, 0])
    cells = _grid_walk(N, dim)
    if dim == 3:
        Rgt = quat_to_rot(rng.standard_normal((N, 4)))
    else:
        Rgt = rot2(rng.uniform(-math.pi, math.pi, size=N))
    gt = np.concatenate([Rgt, cells.astype(np.float64)[..., None]], axis=-1)

    index_of = {tuple(c): k for k, c in enumerate(cells.tolist())}
    offsets = []
    for ax in range(dim):
        for sgn in (-1, 1):
            o = [0] * dim
            o[ax] = sgn
            offsets.append(tuple(o))

    edges = [(k, k + 1) for k in range(N - 1)]
    closures = []
    for k in range(2, N):
        u = rng.random()
        if u >= p:
            continue
        if mode == "random":
            j = int(rng.integers(0, k - 1))
        else:
            c = tuple(cells[k].tolist())
            cand = []
            for o in offsets:
                nb = tuple(ci + oi for ci, oi in zip(c, o))
                j = index_of.get(nb)
                if j is not None and j < k - 1:
                    cand.append(j)
            cand.sort()
            if not cand:
                continue
            j = cand[int(rng.integers(0, len(cand)))]
        closures.append((j, k))
    edges += closures
    E = len(edges)
    outlier = np.zeros(E, dtype=bool)
    n_out = int(round(outlier_ratio * len(closures)))
    if n_out > 0:
        pick = rng.choice(len(closures), size=n_out, replace=False)
        outlier[(N - 1) + np.sort(pick)] = True
    return CubeTopology(dim=dim, num_poses=N, edges=np.asarray(edges, dtype=np.int32).reshape(E, 2),
                        prior_vars=np.zeros(1, dtype=np.int32), gt=np.ascontiguousarray(gt),
                        outlier=outlier, num_closures=len(closures))


def _noise_pose(rng, n: int, dim: int, sigma_t: float, sigma_r: float) -> np.ndarray:
    if dim == 3:
        phi = rng.standard_normal((n, 3)) * sigma_r
        q = np.concatenate([np.ones((n, 1)), 0.5 * phi], axis=1)
        R = quat_to_rot(q)
    else:
        R = rot2(rng.standard_normal(n) * sigma_r)
    t = rng.standard_normal((n, dim)) * sigma_t
    return _homog(R, t)


def cube_batch(topo: CubeTopology, batch: int, seed: int = 0, b_start: int = 0,
               sigma_t: float = 0.1, sigma_r: float = 0.05,
               init_sigma_t: float = 0.1, init_sigma_r: float = 0.05,
               outlier_sigma_t: float = 1.0, outlier_sigma_r: float = 0.5,
               zero_noise: bool = False) -> dict:
    """Per-element measurements and initial poses for global elements [b_start, b_start+batch).

    Returns dict with float64 arrays:
      poses0 [B][N][dim][dim+1], meas [B][E][dim][dim+1], prior_meas [B][P][dim][dim+1],
      w_edge [E] (ones), w_prior [P] (ones), gt [N][dim][dim+1].
    """
    dim, N, E = topo.dim, topo.num_poses, topo.num_edges
    P = int(topo.prior_vars.shape[0])
    Tgt = _homog(topo.gt[..., :dim], topo.gt[..., dim])
    Tinv = _inv_homog(Tgt)
    ii, jj = topo.edges[:, 0], topo.edges[:, 1]
    rel = np.einsum("eab,ebc->eac", Tinv[ii], Tgt[jj])
    poses0 = np.empty((batch, N, dim, dim + 1))
    meas = np.empty((batch, E, dim, dim + 1))
    prior = np.empty((batch, P, dim, dim + 1))
    n_out = int(topo.outlier.sum())
    for bl in range(batch):
        rng = np.random.default_rng([seed, 1, b_start + bl])
        Nm = _noise_pose(rng, E, dim, sigma_t, sigma_r)
        Ni = _noise_pose(rng, N, dim, init_sigma_t, init_sigma_r)
        No = _noise_pose(rng, n_out, dim, outlier_sigma_t, outlier_sigma_r) if n_out else None
        if zero_noise:
            Nm = _homog(np.broadcast_to(np.eye(dim), (E, dim, dim)), np.zeros((E, dim)))
            Ni = _homog(np.broadcast_to(np.eye(dim), (N, dim, dim)), np.zeros((N, dim)))
        Z = np.einsum("eab,ebc->eac", rel, Nm)
        if n_out and not zero_noise:
            Z[topo.outlier] = np.einsum("eab,ebc->eac", Z[topo.outlier], No)
        T0 = np.einsum("nab,nbc->nac", Tgt, Ni)
        meas[bl] = Z[:, :dim, :]
        poses0[bl] = T0[:, :dim, :]
        prior[bl] = Tgt[topo.prior_vars][:, :dim, :]
    return {
        "poses0": np.ascontiguousarray(poses0),
        "meas": np.ascontiguousarray(meas),
        "prior_meas": np.ascontiguousarray(prior),
        "w_edge": np.ones(E),
        "w_prior": np.ones(P),
        "gt": np.ascontiguousarray(topo.gt),
    }
