"""One K = 64 q | k GEMM shape for an ncu capture (tools/ncu_gemm_probe.sh)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DCHAG_GEMM_DEBUG", "0")
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gemm_epi_probe.py")).read()
exec(src.split("out_bytes = QK.numel()")[0].replace("__file__", repr(os.path.abspath(__file__))))
for _ in range(5):
    run()  # noqa: F821
torch.cuda.synchronize()  # noqa: F821
