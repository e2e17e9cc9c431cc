"""Run a few front-end forwards of a bench workload (for ncu / compute-sanitizer)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2506_21411_b200 import DchagFrontEnd  # noqa: E402
from paper_2506_21411_b200.config import channel_slabs, max_group_for_depth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="hyperspectral")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--tp", type=int, default=1)
a = ap.parse_args()
wl = WORKLOADS[a.workload]
mg = max_group_for_depth([n for _, n in channel_slabs(wl["channels"], a.tp)], wl["depth"])
fe = DchagFrontEnd(wl["channels"], wl["image_h"], wl["image_w"], wl["patch"], wl["embed"],
                   wl["heads"], max_group=mg, tp=a.tp, rank=0)
fe.init_weights(seed=0, all_ranks=False)
off, cnt = fe.slab
x = torch.randn(a.batch, cnt, wl["image_h"], wl["image_w"], device="cuda").to(torch.bfloat16)
for _ in range(a.iters):
    if a.tp == 1:
        y = fe(x)
    else:  # single-GPU stand-in for the gather: replicate this rank's payload
        pay = fe.local_payload(x)
        y = fe.finish(torch.cat([pay] * a.tp), a.batch)
torch.cuda.synchronize()
print("ok", tuple(y.shape), float(y.float().abs().mean()))
