"""Weight folding: the algebra that lets the B200 path skip the token tensor.

Every D-CHAG single_query node (reference layers.py:103-123) has a learned query
that does not depend on the input, so with q' = q @ wq and
    U[:, h] = wk[:, h-blk] @ q'[h-blk] / sqrt(dh)                  (D x H)
its logits are x @ U and its context is ctx_h = (sum_c p_ch x_c) @ wv[:, h-blk].
Consequences used by the kernels:

* level 0 -- tokens x_c = patch_c @ tok.w[c] + tok.b[c] + chan_id[c] + pos[s]
  (model.py:51-64) fold into the node:  M_c = tok.w[c] @ wv,  Cb_c = (tok.b+chan_id)[c] @ wv,
  posV = pos @ wv, and the logit weights WU_c = tok.w[c] @ U, bU_c, posU = pos @ U.
* above level 0 -- a node's consumer (parent node, or the shared final layer for the
  root) only ever reads y @ [wv_par | U_par] (attention) or y @ w_par (linear,
  layers.py:141-146), so each node's output projection is folded with it:
  Wp = wo @ Wcons(par), bp = bo @ Wcons(par).  The node output y itself is never formed.
* the shared final layer ("agg.final", strategies.py:216-218) keeps Wp = wo, bp = bo.

`fold_rank` returns plain (untiled, float) torch tensors on the weights' device;
`pack_rank` casts/tiles them into the device buffers the kernels read.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from .config import ConfigError


def query_logit_weights(w, prefix, heads):
    """U (D x H) such that logits = x @ U (single_query, layers.py:103-120)."""
    wq, wk, q = w[f"{prefix}.wq"], w[f"{prefix}.wk"], w[f"{prefix}.q"]
    d = wk.shape[0]
    dh = d // heads
    qp = q @ wq
    return (wk.view(d, heads, dh) * qp.view(1, heads, dh)).sum(-1) / math.sqrt(dh)


def consumer_weight(w, prefix, kind, heads):
    """Wcons: what a consumer node reads of each input y: [wv | U] or w."""
    if kind == "linear":
        return w[f"{prefix}.w"], False
    return torch.cat([w[f"{prefix}.wv"], query_logit_weights(w, prefix, heads)], dim=1), True


def value_weight(w, prefix, kind):
    return w[f"{prefix}.w"] if kind == "linear" else w[f"{prefix}.wv"]


@dataclass
class FoldedRank:
    """Folded weights of one rank's slab tree + the shared final layer."""

    levels: tuple
    heads: int
    embed: int
    patch: int
    seq: int
    attn_l0: bool
    # level 0 (per slab channel c / per level-0 node n)
    l0_c0: list = field(default_factory=list)
    l0_g: list = field(default_factory=list)
    WU: torch.Tensor | None = None      # [C, PP, H]
    bU: torch.Tensor | None = None      # [C, H]
    posU: torch.Tensor | None = None    # [n0, S, H]
    M: torch.Tensor | None = None       # [C, PP, D]
    Cb: torch.Tensor | None = None      # [C, D]
    posV: torch.Tensor | None = None    # [n0, S, D]
    mix0: torch.Tensor | None = None    # [C] (linear level 0)
    # per level: projection of that level's nodes into their consumer
    Wp: list = field(default_factory=list)   # [n_l, D, N_l]
    bp: list = field(default_factory=list)   # [n_l, N_l]
    has_logits: list = field(default_factory=list)
    # per level >= 1: children of every node + linear mix
    comb_first: list = field(default_factory=list)
    comb_g: list = field(default_factory=list)
    comb_mix: list = field(default_factory=list)
    # final layer (attention over tp streams)
    Wf: torch.Tensor | None = None      # [D, D]
    bf: torch.Tensor | None = None      # [D]


def fold_rank(w, *, rank, slab, levels, embed, heads, patch, seq, variant, layer_kind):
    """Fold the front-end weights of `rank` (slab = (offset, count))."""
    if variant != "single_query":
        raise ConfigError("the fused B200 path implements agg_variant='single_query' "
                          "(full_cross is a later milestone; see DESIGN.md section 7)")
    off, cnt = slab
    d, h = embed, heads
    pre = f"agg.slab{rank}"
    depth = len(levels)
    tokw = w["tok.w"][off:off + cnt]                                  # [C, PP, D]
    tokb = w["tok.b"][off:off + cnt] + w["special.channel_id"][off:off + cnt]
    pos = w["special.pos"]
    attn = layer_kind != "linear"
    fr = FoldedRank(levels=tuple(levels), heads=h, embed=d, patch=patch, seq=seq, attn_l0=attn)

    # ---- level 0 (tokenizer folded)
    pp = patch * patch
    M, Cb, WU, bU, posU, posV, mix0 = [], [], [], [], [], [], []
    c = 0
    for gi, g in enumerate(levels[0]):
        node = f"{pre}.l0.g{gi}"
        Vw = value_weight(w, node, layer_kind)
        tw, tb = tokw[c:c + g], tokb[c:c + g]
        M.append(torch.matmul(tw, Vw))
        Cb.append(tb @ Vw)
        if attn:
            U = query_logit_weights(w, node, h)
            WU.append(torch.matmul(tw, U))
            bU.append(tb @ U)
            posU.append(pos @ U)
            posV.append(pos @ Vw)
        else:
            mix = w[f"{node}.mix"]
            mix0.append(mix)
            posV.append(mix.sum() * (pos @ Vw))
        fr.l0_c0.append(c)
        fr.l0_g.append(g)
        c += g
    fr.M, fr.Cb, fr.posV = torch.cat(M), torch.cat(Cb), torch.stack(posV)
    if attn:
        fr.WU, fr.bU, fr.posU = torch.cat(WU), torch.cat(bU), torch.stack(posU)
    else:
        fr.mix0 = torch.cat(mix0)

    # ---- projections of every level into its consumer
    for li, level in enumerate(levels):
        Wl, bl = [], []
        # consumer of each node of this level
        if li + 1 < depth:
            owners = []
            for gj, gcount in enumerate(levels[li + 1]):
                owners += [gj] * gcount
        for gi in range(len(level)):
            node = f"{pre}.l{li}.g{gi}"
            if li + 1 < depth:
                cons, ckind = f"{pre}.l{li + 1}.g{owners[gi]}", layer_kind
            else:
                cons, ckind = "agg.final", "cross_attention"
            Wc, logits = consumer_weight(w, cons, ckind, h)
            if layer_kind == "linear":
                Wl.append(Wc)
                bl.append(w[f"{node}.b"] @ Wc)
            else:
                Wl.append(w[f"{node}.wo"] @ Wc)
                bl.append(w[f"{node}.bo"] @ Wc)
        fr.Wp.append(torch.stack(Wl))
        fr.bp.append(torch.stack(bl))
        fr.has_logits.append(logits)
        if li >= 1:
            first, acc = [], 0
            for g in level:
                first.append(acc)
                acc += g
            fr.comb_first.append(first)
            fr.comb_g.append(list(level))
            if layer_kind == "linear":
                fr.comb_mix.append(torch.cat([w[f"{pre}.l{li}.g{gi}.mix"]
                                              for gi in range(len(level))]))
            else:
                fr.comb_mix.append(None)
    fr.Wf = w["agg.final.wo"]
    fr.bf = w["agg.final.bo"]
    return fr


# ----------------------------------------------------------------- device packing


@dataclass
class PackedRank:
    """Device buffers in the layouts the kernels read (see include/dchag.h)."""

    n0: int
    C: int
    C_pad: int
    KE: int
    HP: int
    NH: int                  # heads per K_l0 unit (fold.unit_heads)
    attn_l0: bool
    l0_c0: torch.Tensor
    l0_g: torch.Tensor
    l0_g_list: list
    WUt: torch.Tensor | None
    bU: torch.Tensor | None
    posU: torch.Tensor | None
    Mt: torch.Tensor
    Et: torch.Tensor
    posV0: torch.Tensor      # [n0][S][D] bf16: pos @ Vw_n, added to ctx by K_l0
    p_const: torch.Tensor | None
    Wp: list      # [n_l, N_l, D] bf16
    bp: list      # [n_l, N_l] fp32
    N: list
    comb_first: list
    comb_g: list
    comb_mix: list
    Wf: torch.Tensor
    bf: torch.Tensor
    levels: tuple
    # tp == 1: the root's value projection folded with the final layer (softmax over one
    # stream is exactly 1): out = ctx_root @ (Wp_root[:, :D] @ Wf) + (bp_root[:D] @ Wf + bf)
    Wdir: torch.Tensor = None   # [D_out][D] bf16 (n-major)
    bdir: torch.Tensor = None   # [D] fp32
    # final_layer_tp_split: this rank's column shard of Wf and its bias share (frontend)
    head_split: tuple | None = None


def refresh_packed(old: PackedRank, new: PackedRank) -> None:
    """Copy a fresh fold into an existing PackedRank's device buffers in place (same
    shapes: the tree and slab are fixed per module), so pointers captured by CUDA graphs or
    held by callers see the new weights."""
    import dataclasses
    for f in dataclasses.fields(old):
        a, b = getattr(old, f.name), getattr(new, f.name)
        if isinstance(a, torch.Tensor):
            a.copy_(b)
        elif isinstance(a, list) and a and any(isinstance(x, torch.Tensor) for x in a):
            for x, y in zip(a, b):
                if isinstance(x, torch.Tensor):
                    x.copy_(y)


def unit_heads(embed: int, heads: int) -> int:
    """Heads per K_l0 unit (its accumulator holds NH * dh <= 256 columns); also the head-group
    width of the K_p0 p layout."""
    return 2 if embed // heads == 128 else (4 if heads % 4 == 0 else 2)


def tile_values_l0(M, Cb, posV, l0_c0, l0_g, d, h, pp, device):
    """K_l0's value operands from the level-0 value folds M_c = tok.w[c] wv_n ([C, PP, D]),
    Cb_c = tb_c wv_n ([C, D]) and posV_n = pos wv_n ([n0, S, D]): Mt / Et as canonical UMMA
    blocks (dchag_tile_weights) and posV0 bf16. Shared by single_query and full_cross."""
    from . import _lib
    f32 = dict(device=device, dtype=torch.float32)
    stream = _lib.stream_handle()
    C = M.shape[0]
    C_pad = C + 64 // pp
    n0 = len(l0_g)
    KE = 16 * ((max(l0_g) + 15) // 16)

    def tile(src, nblk, K, N):
        src = src.to(**f32).contiguous()
        dst = torch.empty(nblk * N * K, device=device, dtype=torch.bfloat16)
        _lib.call("dchag_tile_weights", _lib.ptr(src), nblk, K, N, _lib.ptr(dst), stream)
        return dst

    # Mt [H][2 halves][C_pad*PP (channel-major K)][dh/2]: a CTA pair splits each head's dh
    # output columns, and one stage's K rows (CG channels) are one contiguous block per half
    dh = d // h
    hw = dh // 2
    Msrc = torch.zeros(h, C_pad, pp, 2, hw, **f32)
    Msrc[:, :C] = M.to(**f32).view(C, pp, h, 2, hw).permute(2, 0, 1, 3, 4)
    Mt = tile(Msrc.permute(0, 3, 1, 2, 4).reshape(h * 2, C_pad * pp, hw), h * 2, C_pad * pp, hw)
    # Et [n0][H][2][KE][dh/2]: row k = node-local channel
    Esrc = torch.zeros(n0, h, KE, 2, hw, **f32)
    for n, (c0, g) in enumerate(zip(l0_c0, l0_g)):
        Esrc[n, :, :g] = Cb[c0:c0 + g].to(**f32).view(g, h, 2, hw).permute(1, 0, 2, 3)
    Et = tile(Esrc.permute(0, 1, 3, 2, 4).reshape(n0 * h * 2, KE, hw), n0 * h * 2, KE, hw)
    posV0 = posV.to(**f32).to(torch.bfloat16).contiguous()
    return Mt, Et, posV0


def pack_rank(fr: FoldedRank, device) -> PackedRank:
    from . import _lib

    d, h, pp = fr.embed, fr.heads, fr.patch * fr.patch
    C = fr.M.shape[0]
    cg = 64 // pp
    C_pad = C + cg
    n0 = len(fr.l0_g)
    gmax = max(fr.l0_g)
    KE = 16 * ((gmax + 15) // 16)
    HP = 8 * ((h + 7) // 8)
    f32 = dict(device=device, dtype=torch.float32)
    stream = _lib.stream_handle()

    Mt, Et, posV0 = tile_values_l0(fr.M, fr.Cb, fr.posV, fr.l0_c0, fr.l0_g, d, h, pp, device)
    WUt = bU = posU = p_const = None
    if fr.attn_l0:
        wu = torch.zeros(C, HP, pp, **f32)
        wu[:, :h] = fr.WU.to(**f32).permute(0, 2, 1)
        WUt = wu.to(torch.bfloat16).contiguous()
        bU = torch.zeros(C, HP, **f32)
        bU[:, :h] = fr.bU.to(**f32)
        posU = torch.zeros(n0, fr.seq, HP, **f32)
        posU[:, :, :h] = fr.posU.to(**f32)
    else:
        # constant p table: p[poff[n] + c*H + h] = mix_c
        p_const = fr.mix0.to(**f32).view(C, 1).expand(C, h).to(torch.bfloat16).contiguous()
    i32 = dict(device=device, dtype=torch.int32)
    Wp, bp, N = [], [], []
    for W_l, b_l in zip(fr.Wp, fr.bp):
        Wp.append(W_l.to(**f32).transpose(1, 2).to(torch.bfloat16).contiguous())
        bp.append(b_l.to(**f32).contiguous())
        N.append(W_l.shape[2])
    comb_first = [torch.tensor(f, **i32) for f in fr.comb_first]
    comb_g = [torch.tensor(g, **i32) for g in fr.comb_g]
    comb_mix = [None if m is None else m.to(**f32).contiguous() for m in fr.comb_mix]
    Wr = fr.Wp[-1][0].to(**f32)[:, :d]                       # root value projection (x @ W)
    Wdir = (Wr @ fr.Wf.to(**f32)).t().to(torch.bfloat16).contiguous()
    bdir = (fr.bp[-1][0].to(**f32)[:d] @ fr.Wf.to(**f32) + fr.bf.to(**f32)).contiguous()
    return PackedRank(
        n0=n0, C=C, C_pad=C_pad, KE=KE, HP=HP, NH=unit_heads(d, h), attn_l0=fr.attn_l0,
        l0_c0=torch.tensor(fr.l0_c0, **i32), l0_g=torch.tensor(fr.l0_g, **i32),
        l0_g_list=list(fr.l0_g), WUt=WUt, bU=bU, posU=posU, Mt=Mt, Et=Et, posV0=posV0,
        p_const=p_const, Wp=Wp, bp=bp, N=N, comb_first=comb_first, comb_g=comb_g,
        comb_mix=comb_mix,
        Wf=fr.Wf.to(**f32).t().to(torch.bfloat16).contiguous(),
        bf=fr.bf.to(**f32).contiguous(), levels=fr.levels, Wdir=Wdir, bdir=bdir)
