"""Batch sharding over torch.distributed ranks (one process per GPU).

Problems are independent: rank r solves the contiguous shard
[r*B/G, (r+1)*B/G) of the global batch with its own graph handle and workspace; the only
communication is one all_reduce(SUM) of [grad_w_edge, grad_w_prior, loss] per step for the
learnable cost weights shared by the batch (NCCL over NVLink on GPUs; gloo in the CPU tests).
The synthetic inputs are seeded per GLOBAL element index, so a G-rank run reproduces the
1-rank run element by element.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced shard of the global batch for `rank` (remainder to the first ranks)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError(f"bad world/rank {world}/{rank}")
    base, rem = divmod(int(global_batch), int(world))
    b0 = rank * base + min(rank, rem)
    return b0, b0 + base + (1 if rank < rem else 0)


def allreduce_weight_grads(grad_w_edge: torch.Tensor, grad_w_prior: torch.Tensor, loss: torch.Tensor,
                           group=None) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Sum the weight gradients and the loss over ranks with ONE all_reduce of E+P+1 doubles."""
    E, P = grad_w_edge.numel(), grad_w_prior.numel()
    buf = torch.cat([grad_w_edge.reshape(-1), grad_w_prior.reshape(-1), loss.reshape(-1)[:1]])
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf[:E].clone(), buf[E:E + P].clone(), buf[E + P:].clone()


def allreduce_shared_grads(*grads: torch.Tensor, group=None) -> list[torch.Tensor]:
    """Sum any set of gradients of parameters shared by the batch (weights, a shared Welsch radius,
    the loss) over ranks with ONE all_reduce of their concatenation (fixed order)."""
    sizes = [g.numel() for g in grads]
    buf = torch.cat([g.reshape(-1) for g in grads])
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    out, o = [], 0
    for g, n in zip(grads, sizes):
        out.append(buf[o:o + n].clone().reshape(g.shape))
        o += n
    return out


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
