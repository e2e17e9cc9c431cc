"""dchag_gemm_nt (the training backward's GEMM: tcgen05 with K-major or MN-major operands,
fp32 accumulate) against a float64 torch contraction of the same bf16 operands."""
import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2506_21411_b200 import _lib as L
    return L


def _gemm_nt(A, a_mn, B, b_mn, G, M, N, K, out, accumulate=0, Ki=None, sAko=None, lda=None,
             bias=None):
    L = _lib()
    lda = lda if lda is not None else (M if a_mn else K)
    Ki = Ki or K
    sAko = sAko if sAko is not None else Ki * lda
    ldb = N if b_mn else K
    L.call("dchag_gemm_nt", L.ptr(A), a_mn, lda, sAko, Ki, A[0].numel(), L.ptr(B), b_mn, ldb,
           B[0].numel(), G, M, N, K, L.ptr(bias), N if bias is not None else 0, L.ptr(out),
           int(out.dtype == torch.float32), accumulate, N, M * N, L.stream_handle())


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("G,M,N,K", [(2, 256, 256, 192), (1, 512, 320, 1024),
                                     (3, 256, 2048, 512), (1, 2048, 2048, 8192),
                                     (2, 256, 96, 128)])
def test_gemm_nt_layouts(a_mn, b_mn, G, M, N, K):
    if b_mn and N % 64:
        N = (N + 63) // 64 * 64
    g = torch.Generator().manual_seed(M + N + K + 7 * a_mn + 13 * b_mn)
    Am = torch.randn(G, M, K, generator=g).to(torch.bfloat16)          # logical A[g][m][k]
    Bn = torch.randn(G, N, K, generator=g).to(torch.bfloat16)          # logical B[g][n][k]
    A = (Am.transpose(1, 2) if a_mn else Am).contiguous().cuda()
    B = (Bn.transpose(1, 2) if b_mn else Bn).contiguous().cuda()
    want = torch.einsum("gmk,gnk->gmn", Am.double(), Bn.double())
    out = torch.empty(G, M, N, device="cuda")
    _gemm_nt(A, a_mn, B, b_mn, G, M, N, K, out)
    torch.cuda.synchronize()
    assert rel_err(out.double().cpu().numpy(), want.numpy()) < 1e-5
    # accumulate onto existing fp32 values; bf16 output
    base = torch.randn(G, M, N, generator=g).cuda()
    acc = base.clone()
    _gemm_nt(A, a_mn, B, b_mn, G, M, N, K, acc, accumulate=1)
    ob = torch.empty(G, M, N, device="cuda", dtype=torch.bfloat16)
    _gemm_nt(A, a_mn, B, b_mn, G, M, N, K, ob)
    torch.cuda.synchronize()
    assert rel_err(acc.double().cpu().numpy(), (want + base.double().cpu()).numpy()) < 1e-5
    assert rel_err(ob.double().cpu().numpy(), want.numpy()) < 5e-3


def test_gemm_nt_two_level_k_rows():
    """MN-major A whose K rows are two-level, as in the [B][C][S][PP] patch layout (k = (b, s):
    (k / S) * C*S*PP + (k % S) * PP + m): E_c = patch_c^T dl_c for one channel of a slab.
    Pixels padded to 256 columns (M % 256 == 0 for an MN-major operand)."""
    L = _lib()
    B_, C, S, PP, N, c = 3, 5, 256, 64, 64, 2
    g = torch.Generator().manual_seed(3)
    patches = torch.randn(B_, C, S, PP, generator=g).to(torch.bfloat16)
    dl = torch.randn(N, B_ * S, generator=g).to(torch.bfloat16).cuda()   # [N][K] K-major
    pad = torch.zeros(B_, C, S, 256, dtype=torch.bfloat16)
    pad[..., :PP] = patches
    pad = pad.cuda()
    out = torch.empty(256, N, device="cuda")
    L.call("dchag_gemm_nt", L.ptr(pad[:, c]), 1, 256, C * S * 256, S, 0, L.ptr(dl), 0, B_ * S, 0,
           1, 256, N, B_ * S, 0, 0, L.ptr(out), 1, 0, N, 256 * N, L.stream_handle())
    torch.cuda.synchronize()
    want = torch.einsum("bsk,nbs->kn", patches[:, c].double(), dl.double().cpu().view(N, B_, S))
    assert rel_err(out[:PP].double().cpu().numpy(), want.numpy()) < 1e-5
    assert float(out[PP:].abs().max()) == 0.0
