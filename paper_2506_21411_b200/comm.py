"""The collectives of the front end (strategies.py:83-96 AllGather, :48-80 TpHooks, :251-264
shared-gradient AllReduce), issued through torch.distributed.

On an NCCL group the call goes straight to NCCL on the device buffers (the production
path; NVLink / NVSwitch). A gloo group (the single-GPU multi-process tests, where several
ranks share one device and NCCL refuses duplicate GPUs) gets the same collective on host
copies of the device buffers, with identical semantics and rank ordering. No other code
in the package calls torch.distributed collectives directly.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class _Done:
    """Work handle of a collective that already completed (host-staged path)."""

    def wait(self):
        return True


def _staged(t: torch.Tensor, group) -> bool:
    return t.is_cuda and dist.get_backend(group) != "nccl"


def all_gather_into_tensor(out, inp, group=None, async_op=False):
    if not _staged(inp, group):
        return dist.all_gather_into_tensor(out, inp, group=group, async_op=async_op)
    host = torch.empty(out.numel(), dtype=out.dtype)   # gloo wants [world * n] for [n]
    dist.all_gather_into_tensor(host, inp.reshape(-1).cpu(), group=group)
    out.copy_(host.view(out.shape))
    return _Done() if async_op else None


def all_to_all_single(out, inp, group=None, async_op=False):
    if not _staged(inp, group):
        return dist.all_to_all_single(out, inp, group=group, async_op=async_op)
    host = torch.empty(out.numel(), dtype=out.dtype)
    dist.all_to_all_single(host, inp.reshape(-1).cpu(), group=group)
    out.copy_(host.view(out.shape))
    return _Done() if async_op else None


def all_reduce(t, group=None):
    if not _staged(t, group):
        return dist.all_reduce(t, group=group)
    host = t.cpu()
    dist.all_reduce(host, group=group)
    t.copy_(host)


def reduce_scatter_tensor(out, inp, group=None):
    if not _staged(inp, group):
        return dist.reduce_scatter_tensor(out, inp, group=group)
    host = torch.empty(out.numel(), dtype=out.dtype)
    dist.reduce_scatter_tensor(host, inp.reshape(-1).cpu(), group=group)
    out.copy_(host.view(out.shape))
