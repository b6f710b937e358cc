"""-m gpu parity of the batch-interleaved level-major path (paper_2207_09442_b200/csrc/bl.cuh; DESIGN.md
"throughput path"; dnls_options.batch_interleave = 32) against the fp64 oracle (north_star tolerances: 1e-9
on poses / objectives, 1e-6 on implicit gradients) and against the per-element path, on ragged batches
(B not a multiple of 32), SE2 and SE3, parallel edges, early stop and per-element failures."""
import numpy as np
import pytest
import torch

from gpu_helpers import (DEV, TOL_GRAD, TOL_OBJ, TOL_POSE, D, make_case, oimp, olie, oracle_problem, oracle_results,
                         pose_err, rel_vec_err, to_dev)
from paper_2207_09442_b200.layer import PoseGraphSolver

pytestmark = pytest.mark.gpu


def solve(topo, data, K, bl, implicit=True, v=None, **opts):
    group = D.SE3 if topo.dim == 3 else D.SE2
    solver = PoseGraphSolver(group, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=K,
                             batch_interleave=32 if bl else 1, **opts)
    t = to_dev(data)
    P, obj, st, it = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                                    implicit=implicit)
    ge = gp = None
    if implicit and v is not None:
        ge, gp = solver.backward(P, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], torch.from_numpy(v).to(DEV),
                                 D.GRAD_TANGENT, per_element=True)
        ge, gp = ge.cpu().numpy(), gp.cpu().numpy()
    torch.cuda.synchronize()
    return P.cpu().numpy(), obj.cpu().numpy(), st.cpu().numpy(), it.cpu().numpy(), ge, gp


@pytest.mark.parametrize("N,dim,B,K,p,mode", [
    (16, 2, 4, 10, 0.2, "local"),      # C1
    (64, 3, 37, 8, 0.3, "local"),      # ragged batch: 37 = 32 + 5
    (40, 3, 5, 6, 0.4, "random"),
    (100, 2, 33, 6, 0.3, "random"),
])
def test_bl_forward_and_implicit_match_oracle(N, dim, B, K, p, mode):
    topo, data = make_case(N, dim=dim, p=p, mode=mode, seed=N + B, B=B)
    v = np.random.default_rng(N).standard_normal((B, N, 6 if dim == 3 else 3))
    P, obj, st, it, ge, gp = solve(topo, data, K, True, v=v)
    samples = sorted({0, 1, B // 2, B - 1})
    sub = {k: (val[samples] if k in ("poses0", "meas", "prior_meas") else val) for k, val in data.items()}
    res = oracle_results(topo, sub, max_iterations=K, implicit=True)
    for r, b in zip(res, samples):
        assert pose_err(P[b], r.x) <= TOL_POSE, b
        assert abs(obj[b] - r.objective) <= TOL_OBJ * r.objective + 1e-20
        assert (st[b] & 0xff) == r.status and it[b] == r.iterations
        prob = oracle_problem(topo, sub, samples.index(b))
        a, c, _ = oimp.implicit_weight_grads(prob, r.x, v[b].reshape(-1), L_K=r.L_final)
        assert rel_vec_err(np.concatenate([ge[b], gp[b]]), np.concatenate([a, c])) <= TOL_GRAD, b


def test_bl_matches_per_element_path_c2_size():
    # BASELINE.json configs[1] sizes (256 poses, batch 128): both GPU paths agree on every element
    topo, data = make_case(256, dim=3, p=0.2, seed=0, B=128)
    v = np.random.default_rng(5).standard_normal((128, 256, 6))
    a = solve(topo, data, 10, True, v=v)
    b = solve(topo, data, 10, False, v=v)
    assert np.max(np.abs(a[0] - b[0])) <= 1e-11 * max(1.0, np.max(np.abs(b[0])))
    assert np.max(np.abs(a[1] - b[1]) / b[1]) <= 1e-11
    assert np.array_equal(a[2] & 0xff, b[2] & 0xff) and np.array_equal(a[3], b[3])
    assert np.max(np.abs(a[4] - b[4])) <= 1e-9 * np.max(np.abs(b[4]))


def test_bl_parallel_edges_early_stop_and_failures():
    topo, data = make_case(30, dim=3, p=0.4, seed=2, B=6)
    # duplicate two edges (parallel edges share an off-diagonal block)
    e = topo.edges
    topo.edges = np.ascontiguousarray(np.concatenate([e, e[[3, 10]]], axis=0).astype(np.int32))
    data["meas"] = np.ascontiguousarray(np.concatenate([data["meas"], data["meas"][:, [3, 10]]], axis=1))
    data["w_edge"] = np.ones(topo.edges.shape[0])
    P, obj, st, it, _, _ = solve(topo, data, 12, True, implicit=False, early_stop=1, abs_tol=1e-12, rel_tol=1e-8)
    res = oracle_results(topo, data, max_iterations=12, early_stop=True, abs_tol=1e-12, rel_tol=1e-8)
    for b, r in enumerate(res):
        assert pose_err(P[b], r.x) <= TOL_POSE
        assert (st[b] & 0xff) == r.status and it[b] == r.iterations
    # a singular H (prior weight 0 on element-shared weights -> gauge freedom): every element NOT_SPD at
    # iteration 0, frozen at theta_0, zero gradient
    data["w_prior"] = np.zeros(1)
    P, obj, st, it, ge, gp = solve(topo, data, 3, True, v=np.ones((6, 30, 6)))
    assert np.all((st & 0xff) == D.ST_NOT_SPD) and np.all(it == 0)
    assert np.array_equal(P, data["poses0"])
    assert np.all(ge == 0) and np.all(gp == 0)


@pytest.mark.parametrize("dim,N,B,split,gw,lsolve", [(3, 64, 37, "4", "4", "1"), (2, 100, 33, "6", "8", "1"),
                                                    (3, 125, 40, "0", "16", "1"), (3, 64, 37, "4", "4", "0")])
def test_bl_large_batch_schedule_on_small_cases(monkeypatch, dim, N, B, split, gw, lsolve):
    # the schedule bench.py's C5 run uses (register-blocked update + persistent tail with chunked update lists
    # and dynamic unit scheduling + persistent tail solves) forced on small ragged batches, SE2 and SE3,
    # against the oracle; the plan reads the environment when the graph's batch-interleaved plan is built
    monkeypatch.setenv("DNLS_BL_UPD", "1")
    monkeypatch.setenv("DNLS_BL_PERSIST", gw)
    monkeypatch.setenv("DNLS_BL_SPLIT", split)
    monkeypatch.setenv("DNLS_BL_LSOLVE", lsolve)   # tail solves: level-parallel bl_lsolve / bl_persist_solve
    topo, data = make_case(N, dim=dim, p=0.3, mode="local", seed=N + B, B=B)
    v = np.random.default_rng(N).standard_normal((B, N, 6 if dim == 3 else 3))
    P, obj, st, it, ge, gp = solve(topo, data, 6, True, v=v)
    samples = sorted({0, B // 2, B - 1})
    sub = {k: (val[samples] if k in ("poses0", "meas", "prior_meas") else val) for k, val in data.items()}
    res = oracle_results(topo, sub, max_iterations=6, implicit=True)
    for r, b in zip(res, samples):
        assert pose_err(P[b], r.x) <= TOL_POSE, b
        assert abs(obj[b] - r.objective) <= TOL_OBJ * r.objective + 1e-20
        prob = oracle_problem(topo, sub, samples.index(b))
        a, c, _ = oimp.implicit_weight_grads(prob, r.x, v[b].reshape(-1), L_K=r.L_final)
        assert rel_vec_err(np.concatenate([ge[b], gp[b]]), np.concatenate([a, c])) <= TOL_GRAD, b


@pytest.mark.parametrize("dim,N,B,sub,subw", [(3, 256, 40, "4", "0"), (3, 256, 33, "8", "30"), (2, 100, 35, "100", "0"),
                                              (3, 64, 37, "0", "0"), (3, 256, 40, "10", "12")])
def test_bl_subtree_factorisation_matches_per_level_schedule(monkeypatch, dim, N, B, sub, subw):
    # bl_subtree (the bottom subtrees of the elimination tree as column tasks in one launch; sub = 100 puts the
    # whole tree in one subtree; subw caps the work of a subtree, the other low columns go through the filtered
    # per-level launches) against the chunked per-level schedule without subtrees: same contributions per target
    # in the same order up to the chunk split -- agreement to rounding, and with the oracle
    topo, data = make_case(N, dim=dim, p=0.3, mode="local", seed=N + B + 1, B=B)
    v = np.random.default_rng(N + 1).standard_normal((B, N, 6 if dim == 3 else 3))
    monkeypatch.setenv("DNLS_BL_UPD", "1")
    monkeypatch.setenv("DNLS_BL_SUB", "-1")
    ref = solve(topo, data, 5, True, v=v)
    monkeypatch.setenv("DNLS_BL_SUB", sub)
    monkeypatch.setenv("DNLS_BL_SUBW", subw)
    got = solve(topo, data, 5, True, v=v)
    assert np.max(np.abs(got[0] - ref[0])) <= 1e-11 * max(1.0, np.max(np.abs(ref[0])))
    assert np.max(np.abs(got[1] - ref[1]) / ref[1]) <= 1e-11
    assert np.array_equal(got[2], ref[2]) and np.array_equal(got[3], ref[3])
    # weight gradients as one vector per element (the prior weight's gradient is rounding noise at the optimum)
    gr = np.concatenate([ref[4], ref[5]], axis=1)
    gg = np.concatenate([got[4], got[5]], axis=1)
    for b in range(B):
        assert rel_vec_err(gg[b], gr[b]) <= 1e-9, b
    samples = [0, B - 1]
    subd = {k: (val[samples] if k in ("poses0", "meas", "prior_meas") else val) for k, val in data.items()}
    res = oracle_results(topo, subd, max_iterations=5, implicit=True)
    for r, b in zip(res, samples):
        assert pose_err(got[0][b], r.x) <= TOL_POSE, b
        assert abs(got[1][b] - r.objective) <= TOL_OBJ * r.objective + 1e-20


@pytest.mark.parametrize("dim,N,B,sub,lch,split,subw", [(3, 256, 40, "2", "1", "100", "0"),
                                                        (3, 256, 40, "6", "1", "100", "20"),
                                                        (3, 200, 35, "4", "3", "12", "0"),
                                                        (2, 100, 33, "-1", "2", "100", "0"),
                                                        (2, 100, 33, "3", "2", "100", "10"),
                                                        (3, 64, 37, "1", "6", "5", "0")])
def test_bl_chunked_level_updates_match_oracle(monkeypatch, dim, N, B, sub, lch, split, subw):
    # the large-batch schedule bench.py's C5 run uses -- bl_subtree for the bottom levels, per-level chunked
    # work items (bl_update_items; lch contributions per chunk, partials reduced in chunk order by
    # bl_factor_red), work-capped subtrees (subw; the other low columns in the filtered per-level launches), the
    # persistent tail from level `split` -- forced on small ragged SE2 / SE3 batches
    monkeypatch.setenv("DNLS_BL_UPD", "1")
    monkeypatch.setenv("DNLS_BL_SUB", sub)
    monkeypatch.setenv("DNLS_BL_SUBW", subw)
    monkeypatch.setenv("DNLS_BL_LCH", lch)
    monkeypatch.setenv("DNLS_BL_SPLIT", split)
    monkeypatch.setenv("DNLS_BL_PERSIST", "8")
    topo, data = make_case(N, dim=dim, p=0.3, mode="local", seed=N + B + 2, B=B)
    v = np.random.default_rng(N + 2).standard_normal((B, N, 6 if dim == 3 else 3))
    P, obj, st, it, ge, gp = solve(topo, data, 5, True, v=v)
    samples = sorted({0, B // 2, B - 1})
    subd = {k: (val[samples] if k in ("poses0", "meas", "prior_meas") else val) for k, val in data.items()}
    res = oracle_results(topo, subd, max_iterations=5, implicit=True)
    for r, b in zip(res, samples):
        assert pose_err(P[b], r.x) <= TOL_POSE, b
        assert abs(obj[b] - r.objective) <= TOL_OBJ * r.objective + 1e-20
        assert (st[b] & 0xff) == r.status and it[b] == r.iterations
        prob = oracle_problem(topo, subd, samples.index(b))
        a, c, _ = oimp.implicit_weight_grads(prob, r.x, v[b].reshape(-1), L_K=r.L_final)
        assert rel_vec_err(np.concatenate([ge[b], gp[b]]), np.concatenate([a, c])) <= TOL_GRAD, b
