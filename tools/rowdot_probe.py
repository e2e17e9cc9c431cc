"""Times dchag_gemm_rowdot at the TR level-0 node shape (16 channels, R = 8192, K = P^2 = 64,
N = D = 2048): the lean row-dot drain against the general one (DCHAG_GEMM_LEAN=0), and
checks both against torch: dot[g][n/32][m] = sum_{n in group} (A_g W_g^T + b_g)[m, n] G[m, n]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2506_21411_b200 import _lib  # noqa: E402

B, S, PP, D, g = 32, 256, 64, 2048, 16
R = B * S
patches = torch.randn(B, g, S, PP, device="cuda").to(torch.bfloat16)
W = (torch.randn(g, D, PP, device="cuda") * 0.1).to(torch.bfloat16)
bias = torch.randn(g, D, device="cuda")
G = torch.randn(R, D, device="cuda").to(torch.bfloat16)
out = torch.empty(g, D // 32, R, device="cuda")
st = _lib.stream_handle()


def run():
    _lib.call("dchag_gemm_rowdot", _lib.ptr(patches), g, B, S, PP, S * PP, g * S * PP, PP,
              _lib.ptr(W), D, D * PP, _lib.ptr(bias), D, _lib.ptr(G), D, _lib.ptr(out), st)


def timed(fn, n=20):
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


A = patches.permute(1, 0, 2, 3).reshape(g, R, PP).float()
ref = ((A @ W.float().transpose(1, 2) + bias[:, None, :]) * G.float()[None])
ref = ref.view(g, R, D // 32, 32).sum(-1).permute(0, 2, 1)
for lean in ("1", "0"):
    os.environ["DCHAG_GEMM_LEAN"] = lean
    ms = timed(run)
    run()
    torch.cuda.synchronize()
    err = ((out - ref).abs().max() / ref.abs().max()).item()
    print(f"lean={lean}: {ms * 1e3:7.1f} us  {2 * g * R * D * PP / ms / 1e9:6.0f} TFLOP/s  "
          f"rel err {err:.2e}")

# per-tile trace of the lean drain (DCHAG_GEMM_DEBUG bit 16; bit 4 drops the MMAs)
NEV = 19
trace = torch.zeros(NEV * 148 * 64, device="cuda", dtype=torch.int64)
os.environ["DCHAG_GEMM_LEAN"] = "1"


def run_tr():
    _lib.call("dchag_gemm_rowdot", _lib.ptr(patches), g, B, S, PP, S * PP, g * S * PP, PP,
              _lib.ptr(W), D, D * PP, _lib.ptr(bias), D, _lib.ptr(G), D,
              _lib.ptr(out), st)


os.environ["DCHAG_GEMM_TRACE_BUF"] = str(trace.data_ptr())
med = lambda x: x.flatten().median().item()  # noqa: E731
for dbg in ("16", "20"):
    os.environ["DCHAG_GEMM_DEBUG"] = dbg
    ms = timed(run_tr)
    trace.zero_()
    run_tr()
    torch.cuda.synchronize()
    tr = trace.view(NEV, 148, 64).cpu().double()
    t0 = tr[tr > 0].min()
    n = 40
    ev = (tr[:, :, :n] - t0) / 1e3
    lead = ev[:, 0::2]
    print(f"debug={dbg}: {ms * 1e3:.1f} us; tile period (epi) {med(ev[3, :, 1:] - ev[3, :, :-1]):.3f}"
          f" producer period {med(ev[0, :, 1:] - ev[0, :, :-1]):.3f}")
    print(f"   tempty->full {med(lead[2] - lead[1]):.3f}  full->epi {med(ev[3, 0::2] - lead[2]):.3f}"
          f"  epi(wait->release) {med(ev[4] - ev[3]):.3f}  release(i)->MMA tempty(i+2) "
          f"{med(lead[1, :, 2:] - ev[4, 0::2, :-2]):.3f}  release->loop top {med(ev[17, :, 1:] - ev[4, :, :-1]):.3f}"
          f"  top->wait {med(ev[18] - ev[17]):.3f}  wait {med(ev[3] - ev[18]):.3f}")
os.environ["DCHAG_GEMM_DEBUG"] = "0"
