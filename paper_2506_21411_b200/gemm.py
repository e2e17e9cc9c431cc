"""Matrix products of the training step on the tcgen05 GEMM (dchag_gemm_nt).

`matmul(a, b)` is `a @ b` for bf16 operands in any of the layouts the backward produces:
each operand is read where it lies, K-major or MN-major (a transposed view such as
`x.t()` is MN-major: no copy), with fp32 accumulation into an fp32 (optionally
accumulating) or bf16 result. 2-D operands broadcast over the group dimension of a 3-D
partner. Shapes outside the kernel's tiling rules (M % 128, K % 64, N % 16; MN-major
operands M % 256, MN-major B N % 64) are zero-padded into scratch copies first -- only the small
test configurations need that; the benchmarked shapes run in place.
"""

from __future__ import annotations

import torch

from . import _lib


def _layout(t, k_dim):
    """(is_mn_major, leading stride) of a 2-D view whose K index is dimension k_dim."""
    other = 1 - k_dim
    if t.stride(k_dim) == 1 and t.size(k_dim) > 0:
        return 0, t.stride(other)
    if t.stride(other) == 1:
        return 1, t.stride(k_dim)
    return None, None


def _pad_kmajor(t, rows, cols):
    """Zero-padded contiguous [G][rows][cols] copy of a [G][r][c] tensor."""
    out = torch.zeros(t.shape[0], rows, cols, device=t.device, dtype=torch.bfloat16)
    out[:, :t.shape[1], :t.shape[2]] = t
    return out


def matmul(a, b, out=None, accumulate=False, out_dtype=torch.float32, bias=None, work=None):
    """out[g] (+)= a[g] @ b[g] (+ bias) with bf16 operands and fp32 accumulation.

    a [G, M, K] or [M, K]; b [G, K, N] or [K, N]; out [G, M, N] / [M, N] (created when None).
    accumulate=True adds into an fp32 `out`."""
    squeeze = a.dim() == 2 and b.dim() == 2
    a3 = a if a.dim() == 3 else a.unsqueeze(0)
    b3 = b if b.dim() == 3 else b.unsqueeze(0)
    G = max(a3.shape[0], b3.shape[0])
    M, K = a3.shape[1], a3.shape[2]
    N = b3.shape[2]
    if b3.shape[1] != K or (a3.shape[0] not in (1, G)) or (b3.shape[0] not in (1, G)):
        raise ValueError(f"matmul: shapes {tuple(a.shape)} @ {tuple(b.shape)}")
    if a3.dtype != torch.bfloat16 or b3.dtype != torch.bfloat16:
        raise TypeError("matmul: bf16 operands expected (convert the weights once per step)")
    if out is None:
        out = torch.empty(G, M, N, device=a.device, dtype=out_dtype)
        out_view = out
    else:
        out_view = out if out.dim() == 3 else out.unsqueeze(0)
    if accumulate and out_view.dtype != torch.float32:
        raise TypeError("matmul: accumulate needs an fp32 out")
    sAg = a3.stride(0) if a3.shape[0] == G and G > 1 else 0
    sBg = b3.stride(0) if b3.shape[0] == G and G > 1 else 0
    a_mn, lda = _layout(a3[0], 1)
    b_mn, ldb = _layout(b3[0].t(), 1)   # B_nt(n, k) = b[k][n]
    ok = (a_mn is not None and b_mn is not None and M % 128 == 0 and K % 64 == 0
          and N % 16 == 0 and (not (a_mn or b_mn) or M % 256 == 0) and (not b_mn or N % 64 == 0)
          and out_view.stride(-1) == 1
          and all((x * 2) % 16 == 0 for x in (lda, ldb, sAg, sBg))
          and a3.data_ptr() % 16 == 0 and b3.data_ptr() % 16 == 0)
    if not ok:
        return _matmul_padded(a3, b3, G, M, K, N, out_view, accumulate, bias, squeeze, out,
                              work)
    _lib.call("dchag_gemm_nt", _lib.ptr(a3), a_mn, lda, 0 if not a_mn else lda * K, K, sAg,
              _lib.ptr(b3), b_mn, ldb, sBg, G, M, N, K, _lib.ptr(bias),
              bias.stride(0) if bias is not None and bias.dim() == 2 else 0,
              _lib.ptr(out_view), int(out_view.dtype == torch.float32), int(accumulate),
              out_view.stride(-2), out_view.stride(0) if G > 1 else 0,
              _lib.stream_handle(), work=work)
    return out_view[0] if squeeze and out.dim() == 3 else out


def _matmul_padded(a3, b3, G, M, K, N, out_view, accumulate, bias, squeeze, out, work):
    """Tile-rule fallback: K-major zero-padded copies, product into a padded scratch."""
    Mp, Kp, Np = -(-M // 128) * 128, -(-K // 64) * 64, -(-N // 16) * 16
    A = _pad_kmajor(a3.expand(G, M, K), Mp, Kp)
    Bt = _pad_kmajor(b3.expand(G, K, N).transpose(1, 2), Np, Kp)
    tmp = torch.empty(G, Mp, Np, device=a3.device, dtype=torch.float32)
    bp = None
    if bias is not None:
        bp = torch.zeros(G, Np, device=a3.device, dtype=torch.float32)
        bp[:, :N] = bias.view(-1, N) if bias.dim() == 2 else bias.view(1, N)
    _lib.call("dchag_gemm_nt", _lib.ptr(A), 0, Kp, 0, Kp, Mp * Kp if G > 1 else 0, _lib.ptr(Bt),
              0, Kp, Np * Kp if G > 1 else 0, G, Mp, Np, Kp, _lib.ptr(bp), Np if bp is not None else 0,
              _lib.ptr(tmp), 1, 0, Np, Mp * Np if G > 1 else 0, _lib.stream_handle(), work=work)
    res = tmp[:, :M, :N]
    if accumulate:
        out_view.add_(res)
    else:
        out_view.copy_(res)
    return out_view[0] if squeeze and out.dim() == 3 else out
