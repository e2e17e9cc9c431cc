"""Times dchag_l0_tgrad_te (the training step's level-0 [patch | 1]^T [p G | dl] kernel) at the
TR node shape (16 channels, R = 8192, D = 2048, H = 32)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2506_21411_b200 import _lib  # noqa: E402

B, S, PP, D, H, NH, g = 32, 256, 64, 2048, 32, 4, 16
R = B * S
patches = torch.randn(B, g, S, PP, device="cuda").to(torch.bfloat16)
G = torch.randn(R, D, device="cuda").to(torch.bfloat16)
p = torch.rand(H // NH, g, R, NH, device="cuda").to(torch.bfloat16)
dlb = torch.randn(g, H, R, device="cuda").to(torch.bfloat16)
Dp = 2304
TE = torch.zeros(g * PP + 128, Dp, device="cuda", dtype=torch.bfloat16)
st = _lib.stream_handle()


def te():
    _lib.call("dchag_l0_tgrad_te", _lib.ptr(patches), g, 0, g, R, S, D, H, NH, PP, _lib.ptr(p), 0,
              _lib.ptr(G), _lib.ptr(dlb), _lib.ptr(TE), Dp, g * PP, st)


def timed():
    for _ in range(3):
        te()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        te()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20


print(f"l0_tgrad_te {timed():.3f} ms per node")
if len(sys.argv) > 1:  # DCHAG_TE_DEBUG probes: 1 no scaling, 2 no MMA
    ref = None
    for dbg in sys.argv[1:]:
        os.environ["DCHAG_TE_DEBUG"] = dbg
        ms = timed()
        out = TE.float().clone()
        err = "" if ref is None else f"  max |diff| vs first {(out - ref).abs().max().item():.3g}"
        ref = out if ref is None else ref
        print(f"debug={dbg}: {ms:.3f} ms{err}")
    os.environ["DCHAG_TE_DEBUG"] = "0"

# one- vs two-channel CTAs (DCHAG_TE_CH=1 selects the one-channel kernel): equal bits, times
if os.environ.get("TE_AB"):
    outs = {}
    for ch in ("1", "2"):
        os.environ["DCHAG_TE_CH"] = ch
        TE.zero_()
        ms = timed()
        outs[ch] = TE.clone()
        print(f"channels per CTA {ch}: {ms:.4f} ms")
    os.environ.pop("DCHAG_TE_CH")
    print("bit-equal:", torch.equal(outs["1"], outs["2"]),
          "max |diff|", (outs["1"].float() - outs["2"].float()).abs().max().item())
