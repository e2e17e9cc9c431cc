"""Times the level-0 backward T_c = patch_c^T (p_c * G) at the training node shape:
dchag_l0_tgrad (dV never stored) against dchag_l0_dv + bmm."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2506_21411_b200 import _lib  # noqa: E402

B, S, PP, D, H, NH, g = 32, 256, 64, 2048, 32, 4, 16
cnt, c0, R = g, 0, B * S
patches = torch.randn(B, cnt, S, PP, device="cuda").to(torch.bfloat16)
G = torch.randn(R, D, device="cuda").to(torch.bfloat16)
p = torch.rand(H // NH, g, R, NH, device="cuda").to(torch.bfloat16)
T = torch.empty(g, PP, D, device="cuda")
dV = torch.empty(g, R, D, device="cuda", dtype=torch.bfloat16)
posV = torch.randn(S, D, device="cuda")
Gpos = torch.empty(R, H, device="cuda")
st = _lib.stream_handle()
pt = patches.permute(1, 3, 0, 2).reshape(g, PP, R)


def tg():
    _lib.call("dchag_l0_tgrad", _lib.ptr(patches), cnt, c0, g, R, S, D, H, NH, PP, _lib.ptr(p), 0,
              _lib.ptr(G), _lib.ptr(T), st)


def dvbmm():
    _lib.call("dchag_l0_dv", g, R, D, H, NH, _lib.ptr(p), 0, _lib.ptr(G), _lib.ptr(posV), 0, S,
              _lib.ptr(Gpos), _lib.ptr(dV), st)
    torch.bmm(pt, dV, out_dtype=torch.float32)


def t(fn, n=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


tg()
T1 = T.clone()
dvbmm()
ref = torch.bmm(pt, (p.permute(1, 2, 0, 3).reshape(g, R, H).unsqueeze(-1) *
                     G.view(1, R, H, D // H)).reshape(g, R, D).to(torch.bfloat16),
                out_dtype=torch.float32)
err = ((T1 - ref).norm() / ref.norm()).item()
print(f"l0_tgrad {t(tg):.3f} ms   l0_dv + bmm {t(dvbmm):.3f} ms   rel err vs bmm {err:.2e}")
