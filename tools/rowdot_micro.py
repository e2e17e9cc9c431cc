"""Times the level-0 backward row-dot GEMM (dchag_gemm_rowdot) at the training shape against
the same GEMM storing V (dchag_gemm_bf16). DCHAG_GEMM_DEBUG ablations apply to both."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2506_21411_b200 import _lib  # noqa: E402

g, B, S, pp, D = 16, 32, 256, 64, 2048
R = B * S
cnt = g
patches = torch.randn(B, cnt, S, pp, device="cuda").to(torch.bfloat16)
Mt = (torch.randn(g, D, pp, device="cuda") * 0.1).to(torch.bfloat16)
Cb = torch.randn(g, D, device="cuda")
Gb = torch.randn(R, D, device="cuda").to(torch.bfloat16)
dpp = torch.empty(g, D // 32, R, device="cuda")
V = torch.empty(g, R, D, device="cuda", dtype=torch.bfloat16)
st = _lib.stream_handle()


def rowdot():
    _lib.call("dchag_gemm_rowdot", _lib.ptr(patches), g, B, S, pp, S * pp, cnt * S * pp, pp,
              _lib.ptr(Mt), D, D * pp, _lib.ptr(Cb), D, _lib.ptr(Gb), D, _lib.ptr(dpp), st)


def vstore():
    _lib.call("dchag_gemm_bf16", _lib.ptr(patches), g, B, S, pp, S * pp, cnt * S * pp, pp,
              _lib.ptr(Mt), D, D * pp, D, _lib.ptr(Cb), D, 0, 0, D, S, _lib.ptr(V), 0, R * D,
              S * D, D, 0, 0, 0, 0, st)


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


rowdot()
ref = (torch.einsum("bcsk,cdk->cbsd", patches.float(), Mt.float()).reshape(g, R, D) + Cb[:, None])
want = (ref * Gb.float()[None]).view(g, R, D // 32, 32).sum(-1).permute(0, 2, 1)
err = ((dpp - want).norm() / want.norm()).item()
print(f"rowdot rel err {err:.2e}; rowdot {t(rowdot):.3f} ms; vstore {t(vstore):.3f} ms "
      f"(debug={os.environ.get('DCHAG_GEMM_DEBUG', '0')})")
