"""Timeline of CTA 0 in l0_node (clock64 per handshake) for one H1 forward."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

trace = torch.zeros(8 * 256, dtype=torch.int64, device="cuda")
os.environ["DCHAG_L0_TRACE_PTR"] = str(trace.data_ptr())
from bench import WORKLOADS  # noqa: E402
from paper_2506_21411_b200 import DchagFrontEnd  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hyperspectral"]
fe = DchagFrontEnd(wl["channels"], wl["image_h"], wl["image_w"], wl["patch"], wl["embed"],
                   wl["heads"], depth=wl["depth"])
fe.init_weights(seed=0, all_ranks=False)
x = torch.randn(32, wl["channels"], wl["image_h"], wl["image_w"], device="cuda").to(torch.bfloat16)
for _ in range(3):
    fe(x)
torch.cuda.synchronize()
t = trace.view(8, 256).cpu()
t0 = int(t[0, 0])
names = ["full", "slotfree", "issue", "img_sync", "built", "slot_sync", "pre_accfull", "accfull"]
print("q  " + " ".join(f"{n:>11s}" for n in names))
for q in range(0, 60):
    print(f"{q:3d} " + " ".join(f"{int(t[e, q]) - t0:11d}" for e in range(8)))
d = lambda e: [int(t[e, q + 1] - t[e, q]) for q in range(20, 50)]  # noqa: E731
import statistics  # noqa: E402
print("median per-stage period: issue", statistics.median(d(2)), "built", statistics.median(d(4)),
      "full", statistics.median(d(0)))
