"""Timeline of CTA 0 (the leader of the first CTA pair) in l0_node: clock64 per handshake."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

trace = torch.zeros(16 * 256, dtype=torch.int64, device="cuda")
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
tt = trace.view(16, 256).cpu()
t0 = int(tt[0, 0])
names = ["full", "post_issue", "pre_issue", "lds_done", "st_done"]
print("times in ns (globaltimer); rank 0 then rank 1")
print("q  " + " ".join(f"{n:>9s}" for n in names) + "  |" + " ".join(f"{n:>9s}" for n in names))
for q in range(0, 40):
    print(f"{q:3d} " + " ".join(f"{int(tt[e, q]) - t0:9d}" for e in range(5)) + "  |" +
          " ".join(f"{int(tt[8 + e, q]) - t0:9d}" for e in range(5)))
for r in (0, 1):
    t = tt[8 * r:8 * r + 8]
    qs = [q for q in range(20, 250) if all(int(t[e, q]) > t0 for e in (3, 4))]
    seg = lambda a, b: statistics.median([int(t[b, q] - t[a, q]) for q in qs])  # noqa: E731
    print(f"rank {r} median ns: lds_done->st_done", seg(3, 4))
t = tt[:8]
qs = [q for q in range(20, 250) if all(int(t[e, q]) > t0 for e in (1, 2, 3, 4))]
print("rank0 st_done->pre_issue", statistics.median([int(t[2, q] - t[4, q]) for q in qs]),
      " rank1 st_done->rank0 pre_issue",
      statistics.median([int(t[2, q] - tt[12, q]) for q in qs if int(tt[12, q]) > t0]),
      " pre->post issue", statistics.median([int(t[1, q] - t[2, q]) for q in qs]))
print("median issue period ns", statistics.median([int(t[2, q + 1] - t[2, q]) for q in qs
                                                   if q + 1 in qs]))
