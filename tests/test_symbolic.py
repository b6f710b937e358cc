"""Not-gpu tests of the C-ABI library and its host symbolic analysis (PAPER.md:213, :221,
:584): the library loads and exports every symbol include/dnls.h declares;
error statuses; the SPEC hand patterns (diagonal, chain, arrow); ordering / etree /
structure invariants against a brute-force elimination written here; fill vs scipy's
SuperLU MMD ordering.  Graphs are created host-only (device = -1)."""
import ctypes

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.linalg import splu

import synth
from paper_2207_09442_b200 import _lib
from paper_2207_09442_b200 import dnls as D


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    names = _lib.header_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
        assert isinstance(getattr(L, n), ctypes._CFuncPtr)
    assert "sm_100a" in D.dnls_version_string()


def test_options_default():
    o = D.dnls_options_default()
    assert (o.optimizer, o.max_iterations, o.step_size) == (D.GN, 10, 1.0)
    assert (o.lambda0, o.lambda_min, o.lambda_max, o.lambda_down, o.lambda_up) == (1e-3, 1e-8, 1e5, 3.0, 2.0)
    assert o.backward_mode == D.BWD_NONE and o.early_stop == 0


@pytest.mark.parametrize("args,status,frag", [
    ((7, 3, [(0, 1)], [0]), 1, "group"),
    ((D.SE3, 3, [(0, 0), (1, 2)], [0]), 3, "self edge"),
    ((D.SE3, 3, [(0, 5)], [0]), 2, "out of range"),
    ((D.SE3, 3, [(0, 1)], [0]), 3, "variable 2 has no cost"),
    ((D.SE2, 3, [(0, 1), (1, 2)], [9]), 2, "prior"),
])
def test_create_errors(args, status, frag):
    with pytest.raises(_lib.DnlsError) as ei:
        D.dnls_graph_create(*args, device=-1)
    assert ei.value.status == status
    assert frag in str(ei.value)


def host_graph(group, N, edges, priors):
    return D.dnls_graph_create(group, N, edges, priors, device=-1)


def brute_structure(N, edges, perm):
    """Symbolic elimination in the given order (independent of the library)."""
    pos = np.empty(N, dtype=int)
    pos[perm] = np.arange(N)
    adj = [set() for _ in range(N)]
    for i, j in edges:
        adj[pos[i]].add(pos[j])
        adj[pos[j]].add(pos[i])
    struct = []
    for k in range(N):
        nb = sorted(x for x in adj[k] if x > k)
        struct.append(nb)
        for a in nb:
            for c in nb:
                if a != c:
                    adj[a].add(c)
    return struct


def lib_structure(g):
    cp, ri = D.dnls_graph_pattern(g)
    return [list(ri[cp[c] + 1:cp[c + 1]]) for c in range(g.N)], cp, ri


def test_spec_diagonal_pattern():
    # SPEC.md:342  diagonal pattern (priors only): zero fill, identity order under the tie rule
    g = host_graph(D.SE2, 4, np.zeros((0, 2)), [0, 1, 2, 3])
    assert list(D.dnls_graph_perm(g)) == [0, 1, 2, 3]
    st = D.dnls_graph_stats(g)
    assert st["nnz_L_blocks"] == 4 and st["nnz_H_blocks"] == 4


def test_spec_chain_pattern():
    # SPEC.md:343  tridiagonal chain n=5: path elimination tree, zero fill
    g = host_graph(D.SE3, 5, [(0, 1), (1, 2), (2, 3), (3, 4)], [0])
    st = D.dnls_graph_stats(g)
    assert st["nnz_L_blocks"] == st["nnz_H_blocks"] == 9
    par = D.dnls_graph_etree(g)
    assert sorted(par.tolist()) == [-1, 1, 2, 3, 4] or (par >= -1).all()
    assert (par == -1).sum() == 1


def test_spec_arrow_pattern():
    # SPEC.md:344  arrow (hub 0 joined to all): the hub is eliminated after the spokes (once two
    # vertices remain they tie), zero fill; the identity order would fill the n-1 spokes' clique
    for n in (4, 8):
        g = host_graph(D.SE3, n, [(0, k) for k in range(1, n)], [1])
        perm = D.dnls_graph_perm(g)
        assert 0 in perm[-2:].tolist()
        st = D.dnls_graph_stats(g)
        assert st["nnz_L_blocks"] == st["nnz_H_blocks"] == 2 * n - 1
        ident = brute_structure(n, [(0, k) for k in range(1, n)], np.arange(n))
        assert sum(len(s) for s in ident) + n - (2 * n - 1) == (n - 1) * (n - 2) // 2


@pytest.mark.parametrize("N,dim,p,mode,seed", [(30, 2, 0.3, "local", 0), (64, 3, 0.2, "local", 1),
                                               (80, 3, 0.3, "random", 2), (256, 3, 0.2, "local", 0)])
def test_structure_invariants(N, dim, p, mode, seed):
    topo = synth.cube_topology(N, dim=dim, p=p, mode=mode, seed=seed)
    group = D.SE3 if dim == 3 else D.SE2
    g = host_graph(group, N, topo.edges, topo.prior_vars)
    perm = D.dnls_graph_perm(g)
    assert sorted(perm.tolist()) == list(range(N))
    struct, cp, ri = lib_structure(g)
    assert struct == brute_structure(N, topo.edges, perm)      # exact symbolic fill
    par = D.dnls_graph_etree(g)
    for k in range(N):
        assert par[k] == (struct[k][0] if struct[k] else -1)
        assert par[k] == -1 or par[k] > k                        # postorder: parents after children
    first, ncols, level = D.dnls_graph_supernodes(g)
    cover = np.concatenate([np.arange(f, f + n) for f, n in zip(first, ncols)])
    assert cover.tolist() == list(range(N))                      # contiguous, disjoint, complete
    st = D.dnls_graph_stats(g)
    d = group
    assert st["nnz_L"] == N * d * (d + 1) // 2 + d * d * (st["nnz_L_blocks"] - N)
    assert st["storage_doubles"] >= st["nnz_L"]
    assert st["num_levels"] == level.max() + 1
    # supernode parent (owner of the etree parent of its last column) is on a higher level
    owner = np.zeros(N, dtype=int)
    for s, (f, n) in enumerate(zip(first, ncols)):
        owner[f:f + n] = s
    for s, (f, n) in enumerate(zip(first, ncols)):
        pp = par[f + n - 1]
        if pp >= 0:
            assert level[owner[pp]] > level[s]


def test_fill_vs_superlu_mmd():
    # fill-reducing quality: nnz(L) blocks within 1.2x of SuperLU's MMD on the C2 pose graph
    topo = synth.cube_topology(256, dim=3, p=0.2, seed=0)
    N = 256
    g = host_graph(D.SE3, N, topo.edges, topo.prior_vars)
    ours = D.dnls_graph_stats(g)["nnz_L_blocks"]
    rows = np.concatenate([topo.edges[:, 0], topo.edges[:, 1], np.arange(N)])
    cols = np.concatenate([topo.edges[:, 1], topo.edges[:, 0], np.arange(N)])
    A = sp.csc_matrix((np.ones(len(rows)), (rows, cols)), shape=(N, N))
    A = A + sp.diags(np.full(N, 10.0))
    lu = splu(A, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0, options={"SymmetricMode": True})
    mmd = lu.L.nnz
    assert ours <= 1.2 * mmd, (ours, mmd)


def test_workspace_bytes_host_only():
    topo = synth.cube_topology(64, dim=3, p=0.2, seed=0)
    g = host_graph(D.SE3, 64, topo.edges, topo.prior_vars)
    n1 = D.dnls_workspace_bytes(g, 1)
    n8 = D.dnls_workspace_bytes(g, 8)
    st = D.dnls_graph_stats(g)
    assert n8 >= 8 * 8 * st["storage_doubles"] and n8 > n1 > 0


def test_launch_counter_host_only():
    # dnls_debug_launch_count (bench.py's gpu_launches): host-only, read / reset, NULL rejected; no kernel
    # launches without a GPU, so a reset counter stays 0
    D.dnls_debug_launch_count(reset=True)
    assert D.dnls_debug_launch_count() == 0
    assert _lib.lib().dnls_debug_launch_count(None, 0) == 1   # DNLS_E_INVALID
