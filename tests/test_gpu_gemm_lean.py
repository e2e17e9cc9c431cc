"""The lean K_gemm drains (csrc/gemm.cu, LEAN 1-3) against a float64 torch reference of the
same bf16 operands, and against the general drain (DCHAG_GEMM_LEAN=0) on the same inputs.

  LEAN 1  plain bf16 tiles (bias, TMA stores)          dchag_gemm_bf16, Nv == N
  LEAN 2  row-dot tiles, 32- and 64-column groups      dchag_gemm_rowdot(_heads)
  LEAN 3  narrow fp32 logit-only tiles                 dchag_gemm_bf16, Nv == 0
(LEAN 4, the fused combine, is pinned by the bench-shape parity tests of the H1 forward.)
"""
import os

import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2506_21411_b200 import _lib as L
    return L


def _operands(G, Mo, Mi, K, N, seed):
    g = torch.Generator().manual_seed(seed)
    A = torch.randn(G, Mo, Mi, K, generator=g).to(torch.bfloat16).cuda()
    W = (torch.randn(G, N, K, generator=g) * 0.1).to(torch.bfloat16).cuda()
    b = torch.randn(G, N, generator=g).cuda()
    return A, W, b


def _ref(A, W, b):
    G, Mo, Mi, K = A.shape
    return (A.double().reshape(G, Mo * Mi, K) @ W.double().transpose(1, 2)
            + b.double()[:, None, :])


def _gemm_bf16(A, W, b, outV=None, outL=None):
    L = _lib()
    G, Mo, Mi, K = A.shape
    N = W.shape[1]
    Nv = N if outV is not None else 0
    L.call("dchag_gemm_bf16", L.ptr(A), G, Mo, Mi, K, Mo * Mi * K, Mi * K, K, L.ptr(W), N,
           N * K, Nv, L.ptr(b), N, 0, 0, 0, 1, L.ptr(outV), 0,
           Mo * Mi * N if outV is not None else 0, Mi * N if outV is not None else 0,
           N if outV is not None else 0, L.ptr(outL),
           Mo * Mi * N if outL is not None else 0, Mi * N if outL is not None else 0,
           N if outL is not None else 0, L.stream_handle())


def _both_drains(fn):
    """fn() under the lean drain and under DCHAG_GEMM_LEAN=0 (the general one)."""
    old = os.environ.get("DCHAG_GEMM_LEAN")
    try:
        os.environ["DCHAG_GEMM_LEAN"] = "1"
        lean = fn()
        os.environ["DCHAG_GEMM_LEAN"] = "0"
        general = fn()
    finally:
        if old is None:
            os.environ.pop("DCHAG_GEMM_LEAN", None)
        else:
            os.environ["DCHAG_GEMM_LEAN"] = old
    torch.cuda.synchronize()
    return lean, general


@pytest.mark.parametrize("G,Mo,Mi,K,N", [(2, 2, 256, 64, 2048), (1, 4, 128, 256, 512),
                                         (3, 1, 512, 1024, 256)])
def test_lean_bf16_tiles(G, Mo, Mi, K, N):
    A, W, b = _operands(G, Mo, Mi, K, N, seed=G * 31 + N)

    def run():
        out = torch.empty(G, Mo * Mi, N, device="cuda", dtype=torch.bfloat16)
        _gemm_bf16(A, W, b, outV=out)
        return out

    lean, general = _both_drains(run)
    want = _ref(A, W, b)
    assert rel_err(lean.double().cpu().numpy(), want.cpu().numpy()) < 1e-2
    # both drains round the same fp32 accumulator to bf16
    assert torch.equal(lean, general)


@pytest.mark.parametrize("G,Mo,Mi,K,N", [(4, 2, 256, 64, 16), (2, 2, 128, 128, 32)])
def test_lean_logit_tiles(G, Mo, Mi, K, N):
    A, W, b = _operands(G, Mo, Mi, K, N, seed=G * 7 + N)

    def run():
        out = torch.empty(G, Mo * Mi, N, device="cuda", dtype=torch.float32)
        _gemm_bf16(A, W, b, outL=out)
        return out

    lean, general = _both_drains(run)
    want = _ref(A, W, b)
    assert rel_err(lean.double().cpu().numpy(), want.cpu().numpy()) < 1e-5
    assert torch.allclose(lean, general, rtol=0, atol=0)


@pytest.mark.parametrize("group", [32, 64])
def test_lean_rowdot(group):
    """dot[g][n / group][m] = sum over the group's columns of (A W^T + b)[m, n] Gmat[m, n]."""
    L = _lib()
    G, Mo, Mi, K, N = 4, 2, 256, 64, 512
    A, W, b = _operands(G, Mo, Mi, K, N, seed=group)
    M = Mo * Mi
    Gm = torch.randn(M, N, generator=torch.Generator().manual_seed(5)).to(torch.bfloat16).cuda()

    def run(grp):
        out = torch.empty(G, N // grp, M, device="cuda")
        L.call("dchag_gemm_rowdot_heads", L.ptr(A), G, Mo, Mi, K, Mo * Mi * K, Mi * K, K,
               L.ptr(W), N, N * K, L.ptr(b), N, L.ptr(Gm), N, grp, L.ptr(out),
               L.stream_handle())
        return out

    v = _ref(A, W, b) * Gm.double()[None]
    want = v.view(G, M, N // group, group).sum(-1).permute(0, 2, 1)
    if group == 32:
        lean, general = _both_drains(lambda: run(32))
        assert rel_err(general.double().cpu().numpy(), want.cpu().numpy()) < 1e-4
    else:  # 64-column groups exist only on the lean drain
        lean = run(64)
        torch.cuda.synchronize()
        # equal to the 32-column sums added in pairs
        pairs = run(32).view(G, N // 64, 2, M).sum(2)
        torch.cuda.synchronize()
        assert torch.allclose(lean, pairs, rtol=1e-6, atol=1e-3)
    assert rel_err(lean.double().cpu().numpy(), want.cpu().numpy()) < 1e-4


def test_split3_matches_torch():
    """dchag_split3_bf16: [hi | lo | hi] with hi = bf16(x), lo = bf16(x - hi), strided rows."""
    L = _lib()
    g = torch.Generator().manual_seed(3)
    x = torch.randn(300, 200, generator=g).cuda()[:, :192]            # row stride 200
    out = torch.empty(300, 3 * 192, device="cuda", dtype=torch.bfloat16)
    L.call("dchag_split3_bf16", L.ptr(x), 300, 192, x.stride(0), L.ptr(out), 3 * 192,
           L.stream_handle())
    torch.cuda.synchronize()
    hi = x.to(torch.bfloat16)
    lo = (x - hi.float()).to(torch.bfloat16)
    assert torch.equal(out, torch.cat([hi, lo, hi], dim=1))


def test_p_normalize_matches_torch():
    """dchag_l0_p_normalize: p = e * pinv over the K_p0 node blocks [hg][g][R][NH]."""
    L = _lib()
    R, H, NH = 256, 8, 4
    gs = [3, 5]
    g = torch.Generator().manual_seed(4)
    e = [torch.rand(H // NH, c, R, NH, generator=g) for c in gs]
    pinv = torch.rand(len(gs), R, H, generator=g)
    flat = torch.cat([t.reshape(-1) for t in e]).to(torch.bfloat16).cuda()
    poff = torch.tensor([0, gs[0] * R * H], dtype=torch.int64, device="cuda")
    node_g = torch.tensor(gs, dtype=torch.int32, device="cuda")
    pin = pinv.cuda()
    out = torch.empty_like(flat)
    L.call("dchag_l0_p_normalize", L.ptr(flat), L.ptr(pin), L.ptr(out), L.ptr(poff),
           L.ptr(node_g), len(gs), max(gs), R, H, NH, L.stream_handle())
    torch.cuda.synchronize()
    at = 0
    for n, c in enumerate(gs):
        blk = flat[at:at + c * R * H].float().view(H // NH, c, R, NH)
        sc = pin[n].view(R, H // NH, NH).permute(1, 0, 2).unsqueeze(1)     # [hg, 1, R, NH]
        want = (blk * sc).to(torch.bfloat16)
        assert torch.equal(out[at:at + c * R * H].view(H // NH, c, R, NH), want)
        at += c * R * H
