"""4-rank probe: the trainer's CUDA-graph step on a dedicated NCCL group (fe.process_group) vs
the default group, followed by an eager barrier on the default group."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NCCL_NVLS_ENABLE", "0")
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
mode = os.environ.get("PROBE_MODE", "group")
from paper_2506_21411_b200 import DchagFrontEnd  # noqa: E402
from paper_2506_21411_b200.train import DchagTrainer  # noqa: E402
pg = dist.new_group(list(range(world))) if mode == "group" else None
fe = DchagFrontEnd(16, 64, 128, 8, 256, 4, max_group=2, tp=world, rank=rank,
                   final_layer_tp_split=True, out_dtype=torch.float32, process_group=pg)
fe.init_weights(seed=0, all_ranks=False)
tr = DchagTrainer(fe)
img = torch.randn(2, fe.slab[1], 64, 128, device="cuda").to(torch.bfloat16)
probe = torch.randn(2, 1, fe.seq, 256, device="cuda")
gs = tr.capture(img, probe)
for _ in range(3):
    gs.replay()
torch.cuda.synchronize()
print(f"[{mode}] rank {rank}: replays done", flush=True)
dist.barrier()
print(f"[{mode}] rank {rank}: barrier after graph OK", flush=True)
t = torch.ones(1, device="cuda")
dist.all_reduce(t)
torch.cuda.synchronize()
print(f"[{mode}] rank {rank}: all_reduce after graph OK {t.item()}", flush=True)
gs.replay()
torch.cuda.synchronize()
dist.barrier()
print(f"[{mode}] rank {rank}: replay + barrier OK", flush=True)
gs.graph.reset()
dist.destroy_process_group()
