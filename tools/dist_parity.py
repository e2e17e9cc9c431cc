"""Multi-GPU parity: torchrun --nproc-per-node N tools/dist_parity.py
One rank per GPU over NCCL; the checks themselves are tests/dist_checks.py (also run by
tests/test_gpu_dist.py with ranks as processes on one GPU). oracle/ is the checker only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from dist_checks import run_checks  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tp, rank = dist.get_world_size(), dist.get_rank()
    worst = run_checks(log=lambda m: print(m, flush=True),
                       ledger_dir=os.path.join(ROOT, "gpurun_out"))
    t = torch.tensor([worst], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"DIST_PARITY tp={tp} worst rel_err={float(t):.3e} -> "
              f"{'PASS' if float(t) < 2e-2 else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if float(t) < 2e-2 else 1)


if __name__ == "__main__":
    main()
