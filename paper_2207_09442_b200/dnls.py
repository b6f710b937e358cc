"""Thin Python binding of include/dnls.h -- same names, argument marshalling only.

Every compute step runs in libdnls' CUDA kernels; PyTorch only provides device memory,
the current CUDA stream and (for multi-GPU) process groups.  Tensors passed here must be
contiguous CUDA tensors of the documented dtype (float64 / int32); this module checks that
and raises otherwise -- there is no CPU path.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import DnlsOptions, DnlsProblem, DnlsStats, check, lib

SE2, SE3 = 3, 6
GN, LM, DOGLEG = 0, 1, 2
BWD_NONE, BWD_IMPLICIT, BWD_UNROLL, BWD_TRUNCATED = 0, 1, 2, 3
DAMP_MARQUARDT, DAMP_IDENTITY = 0, 1
GRAD_TANGENT, GRAD_MATRIX = 0, 1
ST_OK, ST_CONVERGED, ST_NOT_SPD, ST_SATURATED = 0, 1, 2, 3
ST_WARN_NOT_CONVERGED, ST_CODE_MASK = 0x100, 0xFF


def _ptr(t):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if not t.is_cuda:
        raise ValueError("libdnls takes CUDA tensors only (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _f64(t, name):
    if t is not None and t.dtype != torch.float64:
        raise TypeError(f"{name} must be float64, got {t.dtype}")
    return _ptr(t)


def _stream(stream=None, device=None):
    """The caller's stream, else the current stream OF THE GRAPH'S DEVICE (the C ABI switches to that
    device for the call, so the stream must belong to it)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def dnls_version_string() -> str:
    return lib().dnls_version_string().decode()


def dnls_last_error() -> str:
    return lib().dnls_last_error().decode()


def dnls_options_default(**overrides) -> DnlsOptions:
    o = DnlsOptions()
    lib().dnls_options_default(ctypes.byref(o))
    for k, v in overrides.items():
        if not hasattr(o, k):
            raise KeyError(k)
        setattr(o, k, v)
    return o


class Graph:
    """Owning handle of a dnls_graph (destroyed with the object)."""

    def __init__(self, handle, group, num_vars, num_edges, num_priors, device):
        self.handle = handle
        self.group, self.N, self.E, self.P, self.device = group, num_vars, num_edges, num_priors, device
        self.d = group
        self.pose_shape = (3, 4) if group == SE3 else (2, 3)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().dnls_graph_destroy(h)
            except Exception:
                pass
            self.handle = None


def dnls_graph_create(group: int, num_vars: int, edges_ij, prior_vars, device: int = 0) -> Graph:
    e = np.ascontiguousarray(np.asarray(edges_ij, dtype=np.int32).reshape(-1, 2))
    p = np.ascontiguousarray(np.asarray(prior_vars, dtype=np.int32).reshape(-1))
    out = ctypes.c_void_p()
    st = lib().dnls_graph_create(int(group), int(num_vars), int(e.shape[0]),
                                 e.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), int(p.shape[0]),
                                 p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), int(device), ctypes.byref(out))
    check(st, "dnls_graph_create")
    return Graph(out, int(group), int(num_vars), int(e.shape[0]), int(p.shape[0]), int(device))


def dnls_graph_stats(g: Graph) -> dict:
    s = DnlsStats()
    check(lib().dnls_graph_stats(g.handle, ctypes.byref(s)), "dnls_graph_stats")
    return {name: getattr(s, name) for name, _ in DnlsStats._fields_}


def _i32(n):
    a = np.zeros(max(int(n), 1), dtype=np.int32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def dnls_block_offsets(g: Graph):
    """(edge_desc [E][7], prior_desc [P][2]) int32: storage offsets / leading dims of each cost's H blocks."""
    ed = np.zeros((max(g.E, 1), 7), dtype=np.int32)
    pd = np.zeros((max(g.P, 1), 2), dtype=np.int32)
    check(lib().dnls_block_offsets(g.handle, ed.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                   pd.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), "dnls_block_offsets")
    return ed[:g.E], pd[:g.P]


def dnls_status_summary(status: torch.Tensor, stream=None):
    """Host-synchronous (n_failed, n_warned) of a device status[B]; raises DnlsError(6) if all failed."""
    if status.dtype != torch.int32:
        raise TypeError("status must be int32")
    nf, nw = ctypes.c_int32(0), ctypes.c_int32(0)
    check(lib().dnls_status_summary(_ptr(status), int(status.numel()), ctypes.byref(nf), ctypes.byref(nw),
                                    _stream(stream)), "dnls_status_summary")
    return nf.value, nw.value


def dnls_debug_phase_times(g: Graph, capacity: int = 4096) -> list:
    """Factorisation-phase times (ms) of the last batch-interleaved forward (needs DNLS_PHASE_TIMING=1)."""
    buf = np.zeros(capacity, dtype=np.float64)
    n = ctypes.c_int32(0)
    check(lib().dnls_debug_phase_times(g.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(capacity),
                                       ctypes.byref(n)), "dnls_debug_phase_times")
    return buf[:n.value].tolist()


def dnls_debug_launch_count(reset: bool = False) -> int:
    n = ctypes.c_int64(0)
    check(lib().dnls_debug_launch_count(ctypes.byref(n), 1 if reset else 0), "dnls_debug_launch_count")
    return int(n.value)


def dnls_graph_perm(g: Graph) -> np.ndarray:
    a, p = _i32(g.N)
    check(lib().dnls_graph_perm(g.handle, p), "dnls_graph_perm")
    return a[:g.N]


def dnls_graph_etree(g: Graph) -> np.ndarray:
    a, p = _i32(g.N)
    check(lib().dnls_graph_etree(g.handle, p), "dnls_graph_etree")
    return a[:g.N]


def dnls_graph_pattern(g: Graph):
    nnzb = dnls_graph_stats(g)["nnz_L_blocks"]
    cp, cpp = _i32(g.N + 1)
    ri, rip = _i32(nnzb)
    check(lib().dnls_graph_pattern(g.handle, cpp, rip), "dnls_graph_pattern")
    return cp[:g.N + 1], ri[:nnzb]


def dnls_graph_supernodes(g: Graph):
    S = dnls_graph_stats(g)["num_supernodes"]
    f, fp = _i32(S)
    n, np_ = _i32(S)
    lv, lvp = _i32(S)
    check(lib().dnls_graph_supernodes(g.handle, fp, np_, lvp), "dnls_graph_supernodes")
    return f[:S], n[:S], lv[:S]


def dnls_workspace_bytes(g: Graph, batch: int, opt: DnlsOptions | None = None) -> int:
    n = ctypes.c_size_t()
    check(lib().dnls_workspace_bytes(g.handle, int(batch), ctypes.byref(opt) if opt is not None else None,
                                     ctypes.byref(n)), "dnls_workspace_bytes")
    return int(n.value)


def alloc_workspace(g: Graph, batch: int, opt: DnlsOptions | None = None, device=None) -> torch.Tensor:
    nbytes = dnls_workspace_bytes(g, batch, opt)
    dev = torch.device("cuda", g.device) if device is None else device
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
    if ws.data_ptr() % 256:
        raise RuntimeError("workspace allocation not 256-byte aligned")
    return ws


def make_problem(poses, meas, prior_meas, w_edge, w_prior, objective=None, status=None, iterations=None,
                 radius=None):
    """dnls_problem from tensors.  prior_meas / weights with no batch axis are shared (stride 0).
    radius: Welsch radius of the Between edges, [1] shared or [B] per element, or None (quadratic)."""
    pr = DnlsProblem()
    pr.poses = _f64(poses, "poses")
    pr.meas = _f64(meas, "meas")
    pr.prior_meas = _f64(prior_meas, "prior_meas")
    pr.prior_meas_bstride = prior_meas[0].numel() if prior_meas is not None and prior_meas.dim() == 4 else 0
    pr.w_edge = _f64(w_edge, "w_edge")
    pr.w_edge_bstride = w_edge.shape[-1] if w_edge is not None and w_edge.dim() == 2 else 0
    pr.w_prior = _f64(w_prior, "w_prior")
    pr.w_prior_bstride = w_prior.shape[-1] if w_prior is not None and w_prior.dim() == 2 else 0
    pr.objective = _f64(objective, "objective")
    if status is not None and status.dtype != torch.int32:
        raise TypeError("status must be int32")
    if iterations is not None and iterations.dtype != torch.int32:
        raise TypeError("iterations must be int32")
    pr.status = _ptr(status)
    pr.iterations = _ptr(iterations)
    pr.radius = _f64(radius, "radius")
    pr.radius_bstride = 1 if radius is not None and radius.numel() > 1 else 0
    return pr


def dnls_forward(g: Graph, batch: int, opt: DnlsOptions, prob: DnlsProblem, workspace: torch.Tensor, stream=None):
    check(lib().dnls_forward(g.handle, int(batch), ctypes.byref(opt), ctypes.byref(prob), _ptr(workspace),
                             workspace.numel(), _stream(stream, g.device)), "dnls_forward")


def dnls_backward_implicit(g: Graph, batch: int, prob: DnlsProblem, grad_poses: torch.Tensor, grad_kind: int,
                           grad_w_edge, grad_w_prior, grad_bstride: int, workspace: torch.Tensor, stream=None,
                           grad_radius=None):
    check(lib().dnls_backward_implicit(g.handle, int(batch), ctypes.byref(prob), _f64(grad_poses, "grad_poses"),
                                       int(grad_kind), _f64(grad_w_edge, "grad_w_edge"),
                                       _f64(grad_w_prior, "grad_w_prior"), _f64(grad_radius, "grad_radius"),
                                       int(grad_bstride), _ptr(workspace), workspace.numel(), _stream(stream, g.device)),
          "dnls_backward_implicit")


def dnls_backward_dlm(g: Graph, batch: int, prob: DnlsProblem, grad_poses: torch.Tensor, grad_kind: int,
                      epsilon: float, grad_w_edge, grad_w_prior, grad_bstride: int, workspace: torch.Tensor,
                      stream=None, grad_radius=None):
    check(lib().dnls_backward_dlm(g.handle, int(batch), ctypes.byref(prob), _f64(grad_poses, "grad_poses"),
                                  int(grad_kind), float(epsilon), _f64(grad_w_edge, "grad_w_edge"),
                                  _f64(grad_w_prior, "grad_w_prior"), _f64(grad_radius, "grad_radius"),
                                  int(grad_bstride), _ptr(workspace), workspace.numel(), _stream(stream, g.device)),
          "dnls_backward_dlm")


def dnls_backward_unroll(g: Graph, batch: int, prob: DnlsProblem, grad_poses: torch.Tensor, grad_kind: int,
                         grad_w_edge, grad_w_prior, grad_bstride: int, workspace: torch.Tensor, stream=None,
                         grad_poses0=None):
    check(lib().dnls_backward_unroll(g.handle, int(batch), ctypes.byref(prob), _f64(grad_poses, "grad_poses"),
                                     int(grad_kind), _f64(grad_w_edge, "grad_w_edge"),
                                     _f64(grad_w_prior, "grad_w_prior"), _f64(grad_poses0, "grad_poses0"),
                                     int(grad_bstride), _ptr(workspace), workspace.numel(), _stream(stream, g.device)),
          "dnls_backward_unroll")


def dnls_linearize(g: Graph, batch: int, prob: DnlsProblem, lam, damping: int, workspace: torch.Tensor, stream=None):
    check(lib().dnls_linearize(g.handle, int(batch), ctypes.byref(prob), _f64(lam, "lambda"), int(damping),
                               _ptr(workspace), workspace.numel(), _stream(stream, g.device)), "dnls_linearize")


def dnls_factorize(g: Graph, batch: int, workspace: torch.Tensor, status=None, stream=None):
    check(lib().dnls_factorize(g.handle, int(batch), _ptr(workspace), workspace.numel(), _ptr(status),
                               _stream(stream, g.device)), "dnls_factorize")


def dnls_solve_factored(g: Graph, batch: int, workspace: torch.Tensor, rhs: torch.Tensor, x: torch.Tensor,
                        stream=None):
    check(lib().dnls_solve_factored(g.handle, int(batch), _ptr(workspace), workspace.numel(), _f64(rhs, "rhs"),
                                    _f64(x, "x"), _stream(stream, g.device)), "dnls_solve_factored")


def dnls_export_factor(g: Graph, batch: int, workspace: torch.Tensor, dense: torch.Tensor, stream=None):
    check(lib().dnls_export_factor(g.handle, int(batch), _ptr(workspace), workspace.numel(), _f64(dense, "dense"),
                                   _stream(stream, g.device)), "dnls_export_factor")


def dnls_import_matrix(g: Graph, batch: int, dense: torch.Tensor, workspace: torch.Tensor, stream=None):
    check(lib().dnls_import_matrix(g.handle, int(batch), _f64(dense, "dense"), _ptr(workspace), workspace.numel(),
                                   _stream(stream, g.device)), "dnls_import_matrix")


def dnls_export_rhs(g: Graph, batch: int, workspace: torch.Tensor, b: torch.Tensor, stream=None):
    check(lib().dnls_export_rhs(g.handle, int(batch), _ptr(workspace), workspace.numel(), _f64(b, "b"),
                                _stream(stream, g.device)), "dnls_export_rhs")
