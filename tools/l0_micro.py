"""Time each front-end kernel of one workload with CUDA events (quick A/B probe)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2506_21411_b200 import DchagFrontEnd, _lib  # noqa: E402
from paper_2506_21411_b200.config import channel_slabs, max_group_for_depth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="hyperspectral")
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--channels", type=int, default=None, help="override (one rank's slab)")
a = ap.parse_args()
wl = dict(WORKLOADS[a.workload])
if a.channels:
    wl["channels"] = a.channels
mg = max_group_for_depth([n for _, n in channel_slabs(wl["channels"], 1)], wl["depth"])
fe = DchagFrontEnd(wl["channels"], wl["image_h"], wl["image_w"], wl["patch"], wl["embed"],
                   wl["heads"], max_group=mg)
fe.init_weights(seed=0, all_ranks=False)
x = torch.randn(a.batch, wl["channels"], wl["image_h"], wl["image_w"], device="cuda").to(torch.bfloat16)
plan = fe.launch_plan(a.batch)
acc = {}
ev = []
idx = {"i": 0}


def hook(name, phase, work=None):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    if phase == "pre":
        ev.append([plan[idx["i"]][1], e, None])
    else:
        ev[-1][2] = e
        idx["i"] += 1


for _ in range(3):
    fe(x)
_lib.set_launch_hook(hook)
for _ in range(a.iters):
    idx["i"] = 0
    fe(x)
torch.cuda.synchronize()
for site, s, e in ev:
    acc[site] = acc.get(site, 0.0) + s.elapsed_time(e) / a.iters
tot = sum(acc.values())
print(f"{a.workload} mode={os.environ.get('DCHAG_L0_DEBUG', '0')} total {tot:.3f} ms  " +
      "  ".join(f"{k}={v:.3f}" for k, v in acc.items()))
