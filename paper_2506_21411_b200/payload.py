"""Boundary payload of one rank: the rank's partial aggregate (root stream) already
projected into the shared final layer's value / logit space.

Layout (bytes): [ V : R*D bf16 | L : R*H fp32 ],  R = B*S rows (row r = b*S + s).
The AllGather (gather_shards, reference strategies.py:83-96; concatenation in rank order,
runtime.py:259) moves tp such payloads; rank j's block starts at j * nbytes.  The kernels
address the gathered buffer with exactly these offsets (frontend.DchagFrontEnd.finish).
"""

from __future__ import annotations

import torch


def payload_nbytes(R: int, D: int, H: int) -> int:
    return R * D * 2 + R * H * 4


def pack(V: torch.Tensor, L: torch.Tensor) -> torch.Tensor:
    """V [R, D] (any float), L [R, H] -> uint8 payload."""
    R, D = V.shape
    H = L.shape[1]
    out = torch.empty(payload_nbytes(R, D, H), dtype=torch.uint8, device=V.device)
    out[:R * D * 2].view(torch.bfloat16).copy_(V.reshape(-1).to(torch.bfloat16))
    out[R * D * 2:].view(torch.float32).copy_(L.reshape(-1).to(torch.float32))
    return out


def views(payload: torch.Tensor, R: int, D: int, H: int):
    """(V bf16 [R, D], L fp32 [R, H]) views of one rank's payload bytes."""
    V = payload[:R * D * 2].view(torch.bfloat16).view(R, D)
    L = payload[R * D * 2:R * D * 2 + R * H * 4].view(torch.float32).view(R, H)
    return V, L


def unpack(gathered: torch.Tensor, tp: int, R: int, D: int, H: int):
    """Gathered bytes [tp * nbytes] -> (V [tp, R, D] bf16, L [tp, R, H] fp32), rank order."""
    nb = payload_nbytes(R, D, H)
    if gathered.numel() != tp * nb:
        raise ValueError(f"gathered payload has {gathered.numel()} bytes, expected {tp * nb}")
    Vs, Ls = zip(*(views(gathered[j * nb:(j + 1) * nb], R, D, H) for j in range(tp)))
    return torch.stack(Vs), torch.stack(Ls)
