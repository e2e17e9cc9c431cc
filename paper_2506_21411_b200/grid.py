"""Process grid for D-CHAG inside data-parallel training.

Ranks are row-major over (dp, tp) as in the reference's ParallelConfig.coords
(config.py:180-186, fsdp = 1): tp fastest. The tp group of a rank is its channel-slab
group (the front end's collectives); the dp group holds the ranks with the same tp index
(gradient averaging, strategies.py:315-364)."""

from __future__ import annotations


def grid_coords(rank: int, tp: int) -> tuple[int, int]:
    """(tp_index, dp_index) of a rank (config.py:180-186 with fsdp = 1)."""
    return rank % tp, rank // tp


def make_groups(tp: int, dp: int):
    """torch.distributed groups of this rank: (tp_group, dp_group, tp_index, dp_index).
    Every rank must call it (new_group is collective)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    if world != tp * dp:
        raise ValueError(f"world size {world} != tp {tp} x dp {dp}")
    tp_i, dp_i = grid_coords(rank, tp)
    tp_group = dp_group = None
    for d in range(dp):
        g = dist.new_group([d * tp + t for t in range(tp)])
        if d == dp_i:
            tp_group = g
    for t in range(tp):
        g = dist.new_group([d * tp + t for d in range(dp)])
        if t == tp_i:
            dp_group = g
    return tp_group, dp_group, tp_i, dp_i
