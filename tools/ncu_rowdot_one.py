"""One TR-shaped row-dot GEMM for an ncu capture (lean drain)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DCHAG_GEMM_DEBUG", "0")
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "rowdot_probe.py")).read()
exec(src.split("A = patches.permute")[0].replace("__file__", repr(os.path.abspath(__file__))))
for _ in range(5):
    run()  # noqa: F821
torch.cuda.synchronize()  # noqa: F821
