"""K_te (dchag_l0_tgrad_te, csrc/gemm.cu): the two-channel CTA form against the one-channel
form (DCHAG_TE_CH=1) on the same inputs, bit for bit, and both against a float64 torch
statement of the augmented level-0 product the kernel writes:

  TE[c*PP + k][d]      = sum_r patch_c[r][k] p_c[r][h(d)] G[r][d]
  TE[c*PP + k][D + h]  = sum_r patch_c[r][k] dl_c[r][h]
  TE[ones0 + c][d]     = sum_r p_c[r][h(d)] G[r][d]
  TE[ones0 + c][D + h] = sum_r dl_c[r][h]
(the level-0 backward of layers.py:103-123 with the tokenizer folded, see train.py)."""
import os

import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _run(g, B, S, D, H, NH, attention, seed):
    from paper_2506_21411_b200 import _lib as L
    PP = 64
    R = B * S
    gen = torch.Generator().manual_seed(seed)
    cnt = g + 3                      # slab wider than the node: channel offset c0 = 2
    patches = torch.randn(B, cnt, S, PP, generator=gen).to(torch.bfloat16).cuda()
    G = torch.randn(R, D, generator=gen).to(torch.bfloat16).cuda()
    p = torch.rand(H // NH, g, R, NH, generator=gen).to(torch.bfloat16).cuda()
    mix = torch.rand(g, generator=gen).cuda()
    dlb = torch.randn(g, H, R, generator=gen).to(torch.bfloat16).cuda() if attention else None
    te_ld = D + 128
    rows = g * PP + g

    def run(ch):
        old = os.environ.get("DCHAG_TE_CH")
        os.environ["DCHAG_TE_CH"] = ch
        try:
            TE = torch.zeros(rows, te_ld, device="cuda", dtype=torch.bfloat16)
            L.call("dchag_l0_tgrad_te", L.ptr(patches), cnt, 2, g, R, S, D, H, NH, PP,
                   L.ptr(p) if attention else 0, 0 if attention else L.ptr(mix), L.ptr(G),
                   L.ptr(dlb), L.ptr(TE), te_ld, g * PP, L.stream_handle())
            torch.cuda.synchronize()
            return TE
        finally:
            if old is None:
                os.environ.pop("DCHAG_TE_CH", None)
            else:
                os.environ["DCHAG_TE_CH"] = old

    one, two = run("1"), run("2")
    # float64 statement
    dh = D // H
    pt = patches[:, 2:2 + g].double().permute(1, 0, 2, 3).reshape(g, R, PP)     # [g][R][PP]
    if attention:
        ph = p.double().permute(1, 2, 0, 3).reshape(g, R, H)                     # [g][R][H]
    else:
        ph = mix.double()[:, None, None].expand(g, R, H)
    # the kernel scales G by p in bf16 before the MMA
    pG = (ph.repeat_interleave(dh, dim=2).float() * G.float()[None]).to(torch.bfloat16).double()
    want = torch.zeros(rows, te_ld, dtype=torch.float64, device="cuda")
    want[:g * PP, :D] = torch.einsum("grk,grd->gkd", pt, pG).reshape(g * PP, D)
    want[g * PP:, :D] = pG.sum(1)
    if attention:
        dl = dlb.double()                                                         # [g][H][R]
        want[:g * PP, D:D + H] = torch.einsum("grk,ghr->gkh", pt, dl).reshape(g * PP, H)
        want[g * PP:, D:D + H] = dl.sum(2)
    return one, two, want


@pytest.mark.parametrize("g,B,S,D,H,NH,attention", [
    (4, 2, 128, 512, 8, 4, True),
    (6, 1, 256, 1024, 16, 4, True),
    (4, 2, 64, 256, 2, 2, False),     # linear node: p = mix[c], no E columns
    (3, 2, 128, 512, 8, 4, True),     # odd channel count: one-channel CTAs only
])
def test_te_two_channel_ctas(g, B, S, D, H, NH, attention):
    one, two, want = _run(g, B, S, D, H, NH, attention, seed=g * 100 + D)
    assert torch.equal(one, two)
    assert rel_err(two.double().cpu().numpy(), want.cpu().numpy()) < 1e-2
