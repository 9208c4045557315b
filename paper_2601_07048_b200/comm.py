"""Collective plumbing for the sharded path (torch.distributed).

NCCL moves device tensors over NVLink directly. With the gloo backend (CPU-only
collectives) device tensors are staged through host memory; that mode exists so
the multi-rank code paths run in CPU tests and on a single-GPU box.
"""

from __future__ import annotations


def _is_nccl(group=None) -> bool:
    import torch.distributed as dist

    return dist.get_backend(group) == "nccl"


def all_gather(t, group=None):
    """Concatenate `t` from every rank along a new leading dim: [world, *t.shape]."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = t.contiguous()
    src = t if (_is_nccl(group) or not t.is_cuda) else t.cpu()
    out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]) if t.dim() else (world,), dtype=t.dtype,
                      device=src.device)
    dist.all_gather_into_tensor(out, src if t.dim() else src.reshape(1), group=group)
    out = out.view((world,) + tuple(t.shape))
    return out.to(t.device, non_blocking=True) if out.device != t.device else out


def broadcast(t, src: int, group=None):
    import torch.distributed as dist

    if _is_nccl(group) or not t.is_cuda:
        dist.broadcast(t, src=src, group=group)
        return t
    h = t.cpu()
    dist.broadcast(h, src=src, group=group)
    t.copy_(h)
    return t


def all_reduce_max(t, group=None):
    import torch.distributed as dist

    if _is_nccl(group) or not t.is_cuda:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return t
    h = t.cpu()
    dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
    t.copy_(h)
    return t
