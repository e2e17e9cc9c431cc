"""Per-item timeline of K_p0 (l0_logits_kernel) for CTAs 0..3 on the H1 forward (globaltimer,
DCHAG_P0_TRACE_PTR): 0 item top, 1 image landed, 2 max pass done (next item's copies issued
when single-buffered), 3 thread 0 done with the exp pass, 4 item end (after the barrier); 5 copies issued, 6 past the max-stat barrier, 7 exp pass done."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

trace = torch.zeros(4 * 8 * 64, dtype=torch.int64, device="cuda")
os.environ["DCHAG_P0_TRACE_PTR"] = str(trace.data_ptr())
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
tt = trace.view(4, 8, 64).cpu()
for cta in range(4):
    t = tt[cta]
    n = int((t[0] > 0).sum())
    ks = range(1, n - 1)
    med = lambda a, b: statistics.median([int(t[b, k] - t[a, k]) for k in ks])  # noqa: E731
    per = statistics.median([int(t[0, k + 1] - t[0, k]) for k in ks])
    print(f"CTA {cta}: items {n}, period {per} ns | top->landed {med(0, 1)}  max pass {med(1, 2)}"
          f"  exp pass {med(2, 3)}  barrier {med(3, 4)}")
    print(f"   issue {med(2, 5)}  to stat barrier {med(5, 6)}  exp+stores {med(6, 7)}  sums+pinv {med(7, 3)}")
