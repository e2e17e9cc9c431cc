"""Times dchag_gemm_rowdot_heads (64-column head groups, the training step's level-0 dp partials)
at the TR node shape. Round-2 probe: without the bias add (-DDCHAG_ROWDOT_NOBIAS build) the
kernel took 91.5 us against 101 us."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_21411_b200 import _lib
B, S, PP, D, g = 32, 256, 64, 2048, 16
R = B * S
patches = torch.randn(B, g, S, PP, device="cuda").to(torch.bfloat16)
W = (torch.randn(g, D, PP, device="cuda") * 0.1).to(torch.bfloat16)
bias = torch.randn(g, D, device="cuda")
G = torch.randn(R, D, device="cuda").to(torch.bfloat16)
out = torch.empty(g, D // 64, R, device="cuda")
st = _lib.stream_handle()
def run():
    _lib.call("dchag_gemm_rowdot_heads", _lib.ptr(patches), g, B, S, PP, S * PP, g * S * PP, PP,
              _lib.ptr(W), D, D * PP, _lib.ptr(bias), D, _lib.ptr(G), D, 64, _lib.ptr(out), st)
for _ in range(3): run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(20): run()
e1.record(); torch.cuda.synchronize()
print(os.environ.get("DCHAG_LIB", "default"), f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
