"""TheseusLayer-style differentiable pose-graph layer over libdnls (PAPER.md:147-151
TheseusLayer "dict in -> dict out", Listing 1 :104-131, backward_mode "implicit").

``PoseGraphSolver`` owns a dnls_graph (one-time symbolic analysis) and a device workspace.
``pose_graph_layer(...)`` is a torch.autograd.Function: forward runs ``dnls_forward`` (K GN/LM
iterations, implicit mode keeps the factor of H(theta_K)); backward runs
``dnls_backward_implicit`` and returns gradients for the learnable cost weights.  Gradients
w.r.t. the initial poses are refused in implicit mode (Table 6 :726 "Cannot be used
for learning theta_init").
"""
from __future__ import annotations

import torch

from . import dnls as D


class PoseGraphSolver:
    def __init__(self, group: int, num_vars: int, edges, prior_vars, device: int | None = None, **options):
        if device is None:
            device = torch.cuda.current_device()
        self.graph = D.dnls_graph_create(group, num_vars, edges, prior_vars, device)
        self.device = torch.device("cuda", device)
        self.options = D.dnls_options_default(**options)
        self.stats = D.dnls_graph_stats(self.graph)
        self._ws = None
        self._ws_batch = -1
        self.generation = 0

    @property
    def group(self):
        return self.graph.group

    def workspace(self, batch: int, opt=None) -> torch.Tensor:
        nbytes = D.dnls_workspace_bytes(self.graph, batch, opt if opt is not None else self.options)
        if self._ws is None or self._ws_batch != batch or self._ws.numel() < nbytes:
            self._ws = D.alloc_workspace(self.graph, batch, opt if opt is not None else self.options, self.device)
            self._ws_batch = batch
        return self._ws

    def forward(self, poses, meas, prior_meas, w_edge, w_prior, implicit: bool = False, options=None, radius=None,
                backward_mode=None, backward_steps: int = 0):
        """Solve in place on a copy of ``poses``.  Returns (poses_K, objective, status, iterations).
        radius: Welsch radius tensor ([1] or [B]) of the Between edges, or None (quadratic costs).
        backward_mode: D.BWD_* (overrides ``implicit``); UNROLL / TRUNCATED record the per-iteration history
        (TRUNCATED: the last ``backward_steps`` iterations) for ``backward(mode="unroll")``."""
        opt = options if options is not None else self.options
        if backward_mode is None:
            backward_mode = D.BWD_IMPLICIT if implicit else D.BWD_NONE
        opt.backward_mode = backward_mode
        opt.backward_steps = int(backward_steps)
        B = poses.shape[0]
        out = poses.detach().clone().contiguous()
        obj = torch.empty(B, dtype=torch.float64, device=poses.device)
        st = torch.empty(B, dtype=torch.int32, device=poses.device)
        it = torch.empty(B, dtype=torch.int32, device=poses.device)
        ws = self.workspace(B, opt)
        prob = D.make_problem(out, meas.contiguous(), prior_meas.contiguous(), w_edge.detach().contiguous(),
                              w_prior.detach().contiguous(), obj, st, it,
                              radius=None if radius is None else radius.detach().contiguous())
        D.dnls_forward(self.graph, B, opt, prob, ws)
        self.generation += 1
        return out, obj, st, it

    def backward(self, poses_K, meas, prior_meas, w_edge, w_prior, grad_poses, grad_kind=D.GRAD_MATRIX,
                 per_element: bool = False, mode: str = "implicit", epsilon: float = 1e-3, radius=None,
                 grad_poses0=None):
        """Weight gradients for the upstream pose gradient: mode "implicit" (Prop. 1, cached factor
        of the last implicit forward) or "dlm" (direct loss minimisation, one
        augmented GN step from poses_K; no cached factor needed).  With a Welsch ``radius`` the
        result is (grad_w_edge, grad_w_prior, grad_radius), else (grad_w_edge, grad_w_prior)."""
        B = poses_K.shape[0]
        ws = self.workspace(B)
        E, P = self.graph.E, self.graph.P
        if per_element:
            ge = torch.zeros(B, max(E, P), dtype=torch.float64, device=poses_K.device)
            gp = torch.zeros(B, max(E, P), dtype=torch.float64, device=poses_K.device)
            stride = max(E, P)
        else:
            ge = torch.zeros(E, dtype=torch.float64, device=poses_K.device)
            gp = torch.zeros(P, dtype=torch.float64, device=poses_K.device)
            stride = 0
        rad = None if radius is None else radius.detach().contiguous()
        gr = None
        if rad is not None:   # laid out like the radius: shared [1] (batch sum) or per element [B]
            gr = torch.zeros(rad.numel(), dtype=torch.float64, device=poses_K.device)
        prob = D.make_problem(poses_K, meas.contiguous(), prior_meas.contiguous(), w_edge.detach().contiguous(),
                              w_prior.detach().contiguous(), radius=rad)
        if mode == "implicit":
            D.dnls_backward_implicit(self.graph, B, prob, grad_poses.contiguous(), grad_kind,
                                     ge if E else None, gp if P else None, stride, ws, grad_radius=gr)
        elif mode == "unroll":   # unroll / truncated: the history recorded by the last forward
            D.dnls_backward_unroll(self.graph, B, prob, grad_poses.contiguous(), grad_kind,
                                   ge if E else None, gp if P else None, stride, ws, grad_poses0=grad_poses0)
        elif mode == "dlm":
            D.dnls_backward_dlm(self.graph, B, prob, grad_poses.contiguous(), grad_kind, epsilon,
                                ge if E else None, gp if P else None, stride, ws, grad_radius=gr)
            self.generation += 1   # the workspace factor was overwritten
        else:
            raise ValueError(f"unknown backward mode {mode!r} (implicit | dlm | unroll)")
        if per_element:
            ge, gp = ge[:, :E], gp[:, :P]
        if rad is not None:
            return ge, gp, gr.reshape(rad.shape)
        return ge, gp


class _PoseGraphFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, solver, poses0, meas, prior_meas, w_edge, w_prior, radius=None, mode="implicit", epsilon=1e-3,
                steps=0):
        bmode = {"implicit": D.BWD_IMPLICIT, "dlm": D.BWD_NONE, "unroll": D.BWD_UNROLL,
                 "truncated": D.BWD_TRUNCATED}[mode]
        poses, obj, st, it = solver.forward(poses0, meas, prior_meas, w_edge, w_prior, radius=radius,
                                            backward_mode=bmode, backward_steps=steps)
        ctx.solver = solver
        ctx.mode, ctx.epsilon = mode, epsilon
        ctx.gen = solver.generation
        ctx.has_radius = radius is not None
        ctx.save_for_backward(poses, meas, prior_meas, w_edge, w_prior, *([radius] if radius is not None else []))
        ctx.mark_non_differentiable(obj, st, it)
        return poses, obj, st, it

    @staticmethod
    def backward(ctx, g_poses, g_obj, g_st, g_it):
        solver = ctx.solver
        if ctx.mode != "dlm" and solver.generation != ctx.gen:
            raise RuntimeError("pose_graph_layer: the solver ran another forward since this one; its cached "
                               "factor is gone (DNLS_E_STATE)")
        poses, meas, prior_meas, w_edge, w_prior, *rest = ctx.saved_tensors
        radius = rest[0] if ctx.has_radius else None
        if g_poses is None:
            g_poses = torch.zeros_like(poses)
        # per-element gradients when either weight is per element ([B][E] / [B][P]); a weight shared by the
        # batch (1-D) gets the batch sum of its per-element gradients
        per_el = w_edge.dim() == 2 or w_prior.dim() == 2
        out = solver.backward(poses, meas, prior_meas, w_edge, w_prior, g_poses, D.GRAD_MATRIX,
                              per_element=per_el, mode="unroll" if ctx.mode == "truncated" else ctx.mode,
                              epsilon=ctx.epsilon, radius=radius)
        ge, gp = out[0], out[1]
        if per_el:
            ge = ge if w_edge.dim() == 2 else ge.sum(0)
            gp = gp if w_prior.dim() == 2 else gp.sum(0)
        gr = out[2] if radius is not None and ctx.needs_input_grad[6] else None
        ge = ge if ctx.needs_input_grad[4] else None
        gp = gp if ctx.needs_input_grad[5] else None
        return None, None, None, None, ge, gp, gr, None, None, None


def pose_graph_layer(solver: PoseGraphSolver, poses0, meas, prior_meas, w_edge, w_prior, backward_mode="implicit",
                     epsilon=1e-3, radius=None, backward_steps=0):
    """Differentiable solve.  backward_mode "implicit" (Prop. 1, factor reuse), "dlm" (direct loss
    minimisation with step eps), "unroll" (backprop through every GN iteration) or
    "truncated" (through the last ``backward_steps``).  radius: learnable Welsch radius of
    the Between edges, [1] or [B], or None.  Returns (poses*, objective, status, iterations).
    theta_init gradients of the unroll modes are available from PoseGraphSolver.backward(grad_poses0=...)."""
    if backward_mode not in ("implicit", "dlm", "unroll", "truncated"):
        raise ValueError(f"unknown backward_mode {backward_mode!r}")
    if poses0.requires_grad or meas.requires_grad or prior_meas.requires_grad:
        raise ValueError("implicit backward gives no gradient for theta_init or measurements "
                         "(PAPER.md Table 6 :726); only w_edge / w_prior may require grad")
    return _PoseGraphFn.apply(solver, poses0, meas, prior_meas, w_edge, w_prior, radius, backward_mode, epsilon,
                              backward_steps)
