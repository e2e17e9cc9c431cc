"""Process grid (paper_2506_21411_b200/grid.py): rank -> (tp, dp) coordinates as the
reference's ParallelConfig.coords (config.py:180-186) with fsdp = 1, and the tp / dp
groups on gloo (world_size 4 = tp 2 x dp 2)."""
import os
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_21411_b200.grid import grid_coords, make_groups

REF = "/root/reference/pkg/src"


@pytest.mark.parametrize("tp,dp", [(1, 4), (2, 2), (4, 2), (8, 1), (3, 3)])
def test_coords_row_major_tp_fastest(tp, dp):
    seen = set()
    for r in range(tp * dp):
        t, d = grid_coords(r, tp)
        assert r == d * tp + t and 0 <= t < tp and 0 <= d < dp
        seen.add((t, d))
    assert len(seen) == tp * dp


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not mounted")
def test_coords_match_reference():
    sys.path.insert(0, REF)
    try:
        from dchag.config import ParallelConfig
    finally:
        sys.path.remove(REF)
    for tp, dp in [(2, 2), (4, 2), (1, 3)]:
        pc = ParallelConfig(dchag_tp=tp, dp=dp)
        for r in range(tp * dp):
            t, f, d = pc.coords(r)
            assert f == 0 and (t, d) == grid_coords(r, tp)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    tpg, dpg, t, d = make_groups(2, 2)
    x = torch.tensor([float(rank)])
    dist.all_reduce(x, group=tpg)
    y = torch.tensor([float(rank)])
    dist.all_reduce(y, group=dpg)
    q.put((rank, t, d, float(x), float(y)))
    dist.destroy_process_group()


def test_groups_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29400 + os.getpid() % 500
    ps = [ctx.Process(target=_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
    for rank, t, d, xs, ys in res:
        assert (t, d) == (rank % 2, rank // 2)
        assert xs == sum(d * 2 + tt for tt in range(2))      # tp group: same dp index
        assert ys == sum(dd * 2 + t for dd in range(2))      # dp group: same tp index
