"""Where the training step's time goes: forward/backward split and the top GPU kernels
(torch.profiler) for the TR workload (or --workload), one B200."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2506_21411_b200 import DchagFrontEnd  # noqa: E402
from paper_2506_21411_b200.config import channel_slabs, max_group_for_depth  # noqa: E402
from paper_2506_21411_b200.train import DchagTrainer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="train")
ap.add_argument("--batch", type=int, default=32)
a = ap.parse_args()
wl = WORKLOADS[a.workload]
mg = max_group_for_depth([n for _, n in channel_slabs(wl["channels"], 1)], wl["depth"])
fe = DchagFrontEnd(wl["channels"], wl["image_h"], wl["image_w"], wl["patch"], wl["embed"],
                   wl["heads"], max_group=mg, out_dtype=torch.float32)
fe.init_weights(seed=0, all_ranks=False)
tr = DchagTrainer(fe)
x = torch.randn(a.batch, wl["channels"], wl["image_h"], wl["image_w"], device="cuda").to(torch.bfloat16)
g = torch.randn(a.batch, 1, fe.seq, wl["embed"], device="cuda")
for _ in range(2):
    out, saved = tr.forward_train(x)
    tr.backward(saved, g)
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record()
out, saved = tr.forward_train(x)
e1.record()
tr.backward(saved, g)
e2.record()
torch.cuda.synchronize()
print(f"forward {e0.elapsed_time(e1):.2f} ms  backward {e1.elapsed_time(e2):.2f} ms")
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True) as prof:
    out, saved = tr.forward_train(x)
    tr.backward(saved, g)
    torch.cuda.synchronize()
evs = [e for e in prof.key_averages() if e.device_time_total > 0]
evs.sort(key=lambda e: -e.self_device_time_total)
tot = sum(e.self_device_time_total for e in evs)
print(f"total GPU time {tot / 1e3:.1f} ms")
for e in evs[:30]:
    print(f"{e.self_device_time_total / 1e3:8.2f} ms {e.count:5d}  {e.key[:90]}")
shp = [e for e in prof.key_averages(group_by_input_shape=True) if e.self_device_time_total > 0]
shp.sort(key=lambda e: -e.self_device_time_total)
print("-- by input shape")
for e in shp[:25]:
    print(f"{e.self_device_time_total / 1e3:8.2f} ms {e.count:5d}  {e.key[:30]:30s} {str(e.input_shapes)[:110]}")
