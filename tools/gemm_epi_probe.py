"""Where does K_gemm's time go on an output-bound shape? Times the full_cross level-0 q | k
GEMM (K = P^2 = 64, N = 2D = 2048, bf16 out through the TMA-store epilogue) under the
DCHAG_GEMM_DEBUG probes: 0 full, 1 no stores, 2 no bias, 4 no MMA, 8 no epilogue groups.
A fill of the same bytes gives the write-bandwidth yardstick, cuBLAS the library one. Debug
probes run the general epilogue; debug 0 takes the lean one (DCHAG_GEMM_LEAN=0: general).
Round-2 finding (profiles/r02/gemm_epilogue.md): the general epilogue was instruction- and
dependency-latency bound (~350 instructions per 32 columns), not TMEM- or store-bound."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2506_21411_b200 import _lib  # noqa: E402

B, S, PP, D, g, C = 32, 256, 64, 1024, 8, 64
R = B * S
N = 2 * D
patches = torch.randn(B, C, S, PP, device="cuda").to(torch.bfloat16)
Mq = (torch.randn(g, N, PP, device="cuda") * 0.1).to(torch.bfloat16)
bias = torch.randn(g, N, device="cuda")
QK = torch.empty(g, R, N, device="cuda", dtype=torch.bfloat16)
st = _lib.stream_handle()


def run():
    _lib.call("dchag_gemm_bf16", _lib.ptr(patches), g, B, S, PP, S * PP, C * S * PP, PP,
              _lib.ptr(Mq), N, N * PP, N, _lib.ptr(bias), N, 0, 0, 0, 1, _lib.ptr(QK), 0, R * N,
              S * N, N, 0, 0, 0, 0, st)


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


out_bytes = QK.numel() * 2
for dbg in ("0", "1", "2", "8", "4", "12"):
    os.environ["DCHAG_GEMM_DEBUG"] = dbg
    ms = timed(run)
    print(f"debug={dbg:>2}: {ms * 1e3:8.1f} us  {out_bytes / ms / 1e6:7.0f} GB/s of output")
os.environ["DCHAG_GEMM_DEBUG"] = "0"
ms = timed(lambda: QK.fill_(1.0))
print(f"fill       : {ms * 1e3:8.1f} us  {out_bytes / ms / 1e6:7.0f} GB/s")
ref = (patches[:, :g].float().reshape(B, g, S, PP).permute(1, 0, 2, 3).reshape(g, R, PP)
       @ Mq.float().transpose(1, 2) + bias[:, None, :])
run()
torch.cuda.synchronize()
print("max err", (QK.float() - ref).abs().max().item(), "ref max", ref.abs().max().item())

# scaling: time vs the number of tiles (g children x N columns), probes 12 (pipeline only) / 0
print("g    N   tiles  dbg12_us  dbg8_us  full_us")
for gg in (1, 2, 4, 8):
    for NN in (256, 1024, 2048):
        def run2():
            _lib.call("dchag_gemm_bf16", _lib.ptr(patches), gg, B, S, PP, S * PP, C * S * PP, PP,
                      _lib.ptr(Mq), NN, N * PP, NN, _lib.ptr(bias), N, 0, 0, 0, 1, _lib.ptr(QK), 0,
                      R * N, S * N, N, 0, 0, 0, 0, st)
        res = []
        for dbg in ("12", "8", "0"):
            os.environ["DCHAG_GEMM_DEBUG"] = dbg
            res.append(timed(run2) * 1e3)
        print(f"{gg}  {NN:5d}  {gg * R // 256 * NN // 256:5d}  {res[0]:8.1f} {res[1]:8.1f} {res[2]:8.1f}")
os.environ["DCHAG_GEMM_DEBUG"] = "0"

# the same product by cuBLAS (one [g*R, 64] x [64, N] GEMM, bf16 out) and the single-CTA kernel
A2 = patches[:, :g].permute(1, 0, 2, 3).reshape(g * R, PP).contiguous()
W2 = Mq[0].t().contiguous().t()
out2 = torch.empty(g * R, N, device="cuda", dtype=torch.bfloat16)
ms = timed(lambda: torch.matmul(A2, Mq[0].t(), out=out2))
print(f"cuBLAS     : {ms * 1e3:8.1f} us  {out_bytes / ms / 1e6:7.0f} GB/s")
os.environ["DCHAG_GEMM_PAIR"] = "0"
for dbg in ("0", "12"):
    os.environ["DCHAG_GEMM_DEBUG"] = dbg
    ms = timed(run)
    print(f"single-CTA debug={dbg:>2}: {ms * 1e3:8.1f} us  {out_bytes / ms / 1e6:7.0f} GB/s")
os.environ["DCHAG_GEMM_PAIR"] = "1"
os.environ["DCHAG_GEMM_DEBUG"] = "0"

# per-tile event trace (debug bit 16): 0 producer past empty, 1 MMA past tempty, 2 MMA past
# full, 3 epilogue warp 2 past tfull, 4 epilogue warp 2 drained; per group gi of warp 2:
# 5+3gi TMEM load done, 6+3gi staging buffer free, 7+3gi store issued
NEV = 19
trace = torch.zeros(NEV * 148 * 64, device="cuda", dtype=torch.int64)


def run_tr():
    _lib.call("dchag_gemm_bf16", _lib.ptr(patches), g, B, S, PP, S * PP, C * S * PP, PP,
              _lib.ptr(Mq), N, N * PP, N, _lib.ptr(bias), N, 0, 0, 0, 1, _lib.ptr(QK), 0, R * N,
              S * N, N, trace.data_ptr(), 0, 0, 0, st)


for dbg in ("16", "17", "28"):
    os.environ["DCHAG_GEMM_DEBUG"] = dbg
    for _ in range(3):
        run_tr()
    trace.zero_()
    run_tr()
    torch.cuda.synchronize()
    tr = trace.view(NEV, 148, 64).cpu().double()
    t0 = tr[tr > 0].min()
    n = 20  # tiles per CTA that certainly exist
    ev = (tr[:, :, :n] - t0) / 1e3  # us
    lead = ev[:, 0::2]  # leader CTAs hold events 1, 2
    med = lambda x: x.flatten().median().item()  # noqa: E731
    print(f"debug={dbg}: tile period (epi) {med(ev[3, :, 1:] - ev[3, :, :-1]):.3f} us, "
          f"producer period {med(ev[0, :, 1:] - ev[0, :, :-1]):.3f}")
    print(f"   tempty->full {med(lead[2] - lead[1]):.3f}  full->epi {med(ev[3, 0::2] - lead[2]):.3f}"
          f"  epi {med(ev[4] - ev[3]):.3f}  epi done(i)->MMA tempty(i+2) "
          f"{med(lead[1, :, 2:] - ev[4, 0::2, :-2]):.3f}")
    print(f"   epi done(i)->loop top(i+1) {med(ev[17, :, 1:] - ev[4, :, :-1]):.3f}  top->wait "
          f"{med(ev[18] - ev[17]):.3f}  wait {med(ev[3] - ev[18]):.3f}  MMA full(i)->epi wait start(i)"
          f" {med(ev[18, 0::2] - lead[2]):.3f}")
    if False:
        prev = ev[3]
        parts = []
        for gi in range(4):
            for k, name in ((5, "ld"), (6, "buf"), (7, "st")):
                cur = ev[k + 3 * gi]
                if cur.abs().sum() == 0:
                    continue
                parts.append(f"g{gi}.{name} {med(cur - prev):.3f}")
                prev = cur
        print("   ", " ".join(parts))
os.environ["DCHAG_GEMM_DEBUG"] = "0"
