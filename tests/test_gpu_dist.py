"""Multi-rank front end on one GPU: world_size 2 and 3 processes share cuda:0 over gloo
(NCCL refuses two ranks on one device; comm.py stages the same collectives through host
memory). Runs tests/dist_checks.py: the position-split final layer (bitwise equal to the
AllGather schedule), the head-split final layer (strategies.py:48-80, :210-218) forward and
backward with its reduce-scatter, the replicated-final training step, the ledger byte
contract, data parallelism, and the head-split reload case -- every rank against the
float64 oracle / autograd. tools/dist_parity.py runs the same checks over NCCL on N GPUs."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_checks import run_checks
        lines = []
        worst = run_checks(log=lines.append)
        q.put((rank, worst, lines))
    except Exception as e:  # report instead of hanging the other ranks' queue reads
        import traceback
        q.put((rank, 1.0, [traceback.format_exc()]))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_front_end_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    report = "\n".join(line for _, _, lines in sorted(res) for line in lines)
    print(report)
    for rank, worst, _ in res:
        assert worst < 2e-2, (rank, worst, report)
    assert all(p.exitcode == 0 for p in procs), report
