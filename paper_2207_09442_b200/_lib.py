"""ctypes loader for the in-tree libdnls.so (include/dnls.h).  Argument marshalling only.

There is deliberately no fallback: if the CUDA library is missing or fails to load, every
entry point raises.  Build it with ``python -c "import __graft_entry__ as g; g.build()"``.
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# DNLS_LIB selects a development variant built next to it (lib/libdnls_<name>.so, e.g. "trace")
_VARIANT = os.environ.get("DNLS_LIB", "")
LIB_PATH = os.path.join(HERE, "lib", f"libdnls_{_VARIANT}.so" if _VARIANT else "libdnls.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "dnls.h")

c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_double_p = ctypes.POINTER(ctypes.c_double)


class DnlsOptions(ctypes.Structure):
    _fields_ = [
        ("optimizer", ctypes.c_int32),
        ("max_iterations", ctypes.c_int32),
        ("step_size", ctypes.c_double),
        ("lambda0", ctypes.c_double),
        ("lambda_min", ctypes.c_double),
        ("lambda_max", ctypes.c_double),
        ("lambda_down", ctypes.c_double),
        ("lambda_up", ctypes.c_double),
        ("damping", ctypes.c_int32),
        ("early_stop", ctypes.c_int32),
        ("abs_tol", ctypes.c_double),
        ("rel_tol", ctypes.c_double),
        ("backward_mode", ctypes.c_int32),
        ("cluster_ctas", ctypes.c_int32),
        ("trust_radius0", ctypes.c_double),
        ("trust_radius_max", ctypes.c_double),
        ("trust_radius_min", ctypes.c_double),
        ("backward_steps", ctypes.c_int32),
        ("batch_interleave", ctypes.c_int32),
    ]


class DnlsProblem(ctypes.Structure):
    _fields_ = [
        ("poses", ctypes.c_void_p),
        ("meas", ctypes.c_void_p),
        ("prior_meas", ctypes.c_void_p),
        ("prior_meas_bstride", ctypes.c_int64),
        ("w_edge", ctypes.c_void_p),
        ("w_edge_bstride", ctypes.c_int64),
        ("w_prior", ctypes.c_void_p),
        ("w_prior_bstride", ctypes.c_int64),
        ("objective", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("iterations", ctypes.c_void_p),
        ("radius", ctypes.c_void_p),
        ("radius_bstride", ctypes.c_int64),
    ]


class DnlsStats(ctypes.Structure):
    _fields_ = [
        ("group", ctypes.c_int32),
        ("num_vars", ctypes.c_int32),
        ("num_edges", ctypes.c_int32),
        ("num_priors", ctypes.c_int32),
        ("num_supernodes", ctypes.c_int32),
        ("num_levels", ctypes.c_int32),
        ("etree_height", ctypes.c_int32),
        ("max_supernode_cols", ctypes.c_int32),
        ("max_panel_rows", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
        ("nnz_H_blocks", ctypes.c_int64),
        ("nnz_L_blocks", ctypes.c_int64),
        ("nnz_L", ctypes.c_int64),
        ("storage_doubles", ctypes.c_int64),
        ("factor_flops", ctypes.c_double),
        ("solve_flops", ctypes.c_double),
        ("bytes_linearize", ctypes.c_double),
        ("bytes_factor", ctypes.c_double),
        ("bytes_solve", ctypes.c_double),
        ("bytes_update", ctypes.c_double),
        ("bytes_backward", ctypes.c_double),
        ("index_bytes", ctypes.c_int64),
        ("smem_bytes", ctypes.c_int64),
        ("resident_doubles", ctypes.c_int64),
    ]


_SIGS = {
    "dnls_version_string": (ctypes.c_char_p, []),
    "dnls_last_error": (ctypes.c_char_p, []),
    "dnls_options_default": (None, [ctypes.POINTER(DnlsOptions)]),
    "dnls_graph_create": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_int32_p, ctypes.c_int32,
                                         c_int32_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "dnls_graph_destroy": (None, [ctypes.c_void_p]),
    "dnls_graph_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DnlsStats)]),
    "dnls_graph_perm": (ctypes.c_int, [ctypes.c_void_p, c_int32_p]),
    "dnls_graph_etree": (ctypes.c_int, [ctypes.c_void_p, c_int32_p]),
    "dnls_graph_pattern": (ctypes.c_int, [ctypes.c_void_p, c_int32_p, c_int32_p]),
    "dnls_graph_supernodes": (ctypes.c_int, [ctypes.c_void_p, c_int32_p, c_int32_p, c_int32_p]),
    "dnls_workspace_bytes": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(DnlsOptions),
                                            ctypes.POINTER(ctypes.c_size_t)]),
    "dnls_forward": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(DnlsOptions),
                                    ctypes.POINTER(DnlsProblem), ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "dnls_backward_implicit": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(DnlsProblem),
                                              ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t,
                                              ctypes.c_void_p]),
    "dnls_backward_dlm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(DnlsProblem),
                                         ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_size_t, ctypes.c_void_p]),
    "dnls_linearize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(DnlsProblem), ctypes.c_void_p,
                                      ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "dnls_factorize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                                      ctypes.c_void_p, ctypes.c_void_p]),
    "dnls_solve_factored": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "dnls_export_factor": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "dnls_import_matrix": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_size_t, ctypes.c_void_p]),
    "dnls_debug_trace": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int64), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]),
    "dnls_export_rhs": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "dnls_backward_unroll": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(DnlsProblem),
                                            ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t,
                                            ctypes.c_void_p]),
    "dnls_debug_phase_times": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_int32, c_int32_p]),
    "dnls_debug_launch_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]),
    "dnls_block_offsets": (ctypes.c_int, [ctypes.c_void_p, c_int32_p, c_int32_p]),
    "dnls_status_summary": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_int32_p, c_int32_p, ctypes.c_void_p]),
}

_lib = None


def header_symbols(path: str = HEADER_PATH) -> list[str]:
    """Names of every DNLS_API function declared in include/dnls.h."""
    txt = open(path).read()
    return re.findall(r"DNLS_API\s+[\w\s\*]+?\b(dnls_\w+)\s*\(", txt)


def lib():
    """Load libdnls.so (raises if absent: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libdnls.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class DnlsError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().dnls_last_error().decode()
        super().__init__(f"{where} -> status {status}: {msg}")
        self.status = status


def check(status: int, where: str):
    if status != 0:
        raise DnlsError(status, where)
