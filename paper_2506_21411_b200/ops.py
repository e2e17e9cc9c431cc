"""Functional mirrors of the reference front-end API, on CUDA tensors.

Same names, argument order and meaning as the reference:

* ``tokenize_channels(images, tok_w, tok_b, chan_id, pos, patch)``   -- model.py:51-64
* ``flat_aggregate(tokens, w, prefix, variant, n_heads)``             -- model.py:67-73
* ``tree_aggregate(tokens, spec, w, prefix, layer_kind, variant, n_heads)`` -- model.py:76-97

These take already-formed tokens (the fused module path in frontend.py never forms
them). Each call lowers onto the same sm_100a kernels: dchag_unfold + dchag_gemm_bf16
(tokenizer), and per tree level a projection GEMM into the node's value/logit space plus
dchag_combine_strided (softmax-weighted child sum). Weights are dicts of tensors keyed
by the reference's dotted names, in the reference's [D_in, D_out] layout. Compute is bf16
with fp32 accumulation. Outputs are fp32 by default.
"""

from __future__ import annotations

import torch

from . import _lib
from .config import ConfigError, TreeSpec
from .fold import consumer_weight


def _bf(t):
    return t.to(device="cuda", dtype=torch.bfloat16).contiguous()


def _f32(t):
    return t.to(device="cuda", dtype=torch.float32).contiguous()


def _gemm(A, Mo, Mi, K, sAmo, sAmi, W_nk, bias, outV, sVmo, sVmi, outL=None, sLmo=0,
          sLmi=0, rowbias=None, rowbias_row=0, rowbias_period=1, outV_f32=False):
    """One-group dchag_gemm_bf16 call: out[m, n] = A[m, :] . W_nk[n, :] + bias[n] (+ rowbias)."""
    N = W_nk.shape[0]
    Nv = outV.shape[-1] if outV is not None else 0
    # unused strides of size-1 dims still have to be valid (non-zero) TMA strides
    sAmo = sAmo if Mo > 1 else Mi * sAmi
    sAg = Mo * Mi * K
    _lib.call("dchag_gemm_bf16", _lib.ptr(A), 1, Mo, Mi, K, sAg, sAmo, sAmi, _lib.ptr(W_nk), N,
              N * K, Nv, _lib.ptr(bias), N, _lib.ptr(rowbias), 0, rowbias_row,
              rowbias_period, _lib.ptr(outV), int(outV_f32), 0, sVmo, sVmi, _lib.ptr(outL), 0,
              sLmo, sLmi, _lib.stream_handle(),
              work={"site": "ops:gemm", "flops": 2 * Mo * Mi * K * N})


def tokenize_channels(images, tok_w, tok_b, chan_id, pos, patch, out_dtype=torch.float32):
    """[B, Cs, H, W] -> [B, Cs, S, D] tokens (model.py:51-64): unfold (tensor.py:303-323),
    per-channel GEMM on tcgen05, and tok.b + channel_id + pos fused in the epilogue."""
    B, C, Hh, Ww = images.shape
    if Hh % patch or Ww % patch:
        raise ConfigError(f"image {Hh}x{Ww} not divisible by patch {patch}")
    S, PP = (Hh // patch) * (Ww // patch), patch * patch
    D = tok_w.shape[-1]
    if S % 128 or PP % 16:
        raise ConfigError("tokenize_channels on sm_100a needs S % 128 == 0 and P*P % 16 == 0")
    img = _bf(images)
    patches = torch.empty(B, C, S, PP, device="cuda", dtype=torch.bfloat16)
    st = _lib.stream_handle()
    _lib.call("dchag_unfold", _lib.ptr(img), img.stride(0), img.stride(1), B, C, Hh, Ww, patch,
              _lib.ptr(patches), st)
    Wt = _bf(tok_w.transpose(1, 2))                   # [C, D, PP]
    bias = _f32(tok_b) + _f32(chan_id)                # [C, D]
    rb = _bf(pos)                                     # [S, D]
    out = torch.empty(B, C, S, D, device="cuda", dtype=out_dtype)
    _lib.call("dchag_gemm_bf16", _lib.ptr(patches), C, B, S, PP, S * PP, C * S * PP, PP,
              _lib.ptr(Wt), D, D * PP, D, _lib.ptr(bias), D, _lib.ptr(rb), 0, D, S,
              _lib.ptr(out), int(out_dtype == torch.float32), S * D, C * S * D, D, 0, 0, 0, 0,
              st)
    return out


_FC0_CACHE: dict = {}


def _fc_level0_fold(tok_w, tok_b, chan_id, pos, spec, tw, prefix, D, H):
    """Folded level-0 operands of a full_cross tree, once per weight version:
    per node (tok.w[c] [wq | wk | Wu])^T bf16 [g, 2D+H, PP] and tb_c [wq | wk | Wu] fp32
    [g, 2D+H] (tb = tok.b + chan_id); the positional query pos wq (bf16 [n0, S, D]); and the
    value folds K_l0 takes: M_c = tok.w[c] wv ([C, PP, D]), Cb_c = tb_c wv, posV_n = pos wv."""
    srcs = [tok_w, tok_b, chan_id, pos] + [tw[k] for k in sorted(tw)]
    key = (prefix, D, H, spec.levels) + tuple((t.data_ptr(), t._version, tuple(t.shape))
                                              for t in srcs)
    hit = _FC0_CACHE.get(prefix)
    if hit is not None and hit[0] == key:
        return hit[1]
    nodes, pq, Ms, Cbs, posV, c0s = [], [], [], [], [], []
    c0 = 0
    with torch.no_grad():
        tb = _f32(tok_b) + _f32(chan_id)
        p32 = _f32(pos)
        for gi, g in enumerate(spec.levels[0]):
            node = f"{prefix}.l0.g{gi}"
            Wnk, _, _ = _fc_node_weights(tw, node, D, H)          # [3D+H, D] bf16
            Wqku = torch.cat([tw[f"{node}.wq"], tw[f"{node}.wk"],
                              Wnk[3 * D:].float().t()], dim=1)      # [D, 2D+H]
            twc = _f32(tok_w[c0:c0 + g])
            M = torch.matmul(twc, Wqku)                             # [g, PP, 2D+H]
            nodes.append((_bf(M.transpose(1, 2)), (tb[c0:c0 + g] @ Wqku).contiguous()))
            pq.append(p32 @ tw[f"{node}.wq"])
            wv = tw[f"{node}.wv"]
            Ms.append(torch.matmul(twc, wv))
            Cbs.append(tb[c0:c0 + g] @ wv)
            posV.append(p32 @ wv)
            c0s.append(c0)
            c0 += g
    out = {"nodes": nodes, "posq": _bf(torch.stack(pq)), "M": torch.cat(Ms),
           "Cb": torch.cat(Cbs), "posV": torch.stack(posV), "c0s": c0s, "kl0": None}
    _FC0_CACHE[prefix] = (key, out)
    return out


def full_cross_level0(images, tok_w, tok_b, chan_id, pos, spec: TreeSpec, w, prefix, n_heads,
                      patch):
    """Level 0 of a full_cross tree with the tokenizer folded everywhere (tokens, and the
    children's values, never reach memory):
      1. q | k | u of every channel straight from the patches (K = P*P GEMM on the folded
         weights tok.w[c] [wq | wk | Wu], bias tb_c [...]; positional terms below),
      2. dchag_fullcross_weights -> per (child, head) weights w, written as K_l0's p operand
         (q gets the positional query pos wq; the key / u positional terms cancel in the
         softmaxes),
      3. dchag_l0_node (K_l0, tcgen05): ctx = sum_c w_c (patch_c M_c + Cb_c) + pos wv with
         M_c = tok.w[c] wv, the single_query level-0 kernel with p = w (sum_c w_c = 1),
      4. y = ctx wo + bo per node.
    Returns y bf16 [n0, R, D] (node-major rows r = b*S + s)."""
    from .fold import tile_values_l0, unit_heads
    B, C, Hh, Ww = images.shape
    D = tok_w.shape[-1]
    H = n_heads
    S, PP = (Hh // patch) * (Ww // patch), patch * patch
    R = B * S
    NQ = 2 * D + H
    img = images if images.dtype == torch.bfloat16 else images.to(torch.bfloat16)
    if img.stride(3) != 1 or img.stride(2) != Ww:
        img = img.contiguous()
    st = _lib.stream_handle()
    patches = torch.empty(B, C, S, PP, device="cuda", dtype=torch.bfloat16)
    _lib.call("dchag_unfold", _lib.ptr(img), img.stride(0), img.stride(1), B, C, Hh, Ww, patch,
              _lib.ptr(patches), st, work={"site": "ops:unfold", "bytes": 4 * img.numel()})
    tw = {k: _f32(v) for k, v in w.items() if k.startswith(prefix + ".")}
    fd = _fc_level0_fold(tok_w, tok_b, chan_id, pos, spec, tw, prefix, D, H)
    levels0 = spec.levels[0]
    n0 = len(levels0)
    if fd["kl0"] is None:
        fd["kl0"] = tile_values_l0(fd["M"], fd["Cb"], fd["posV"], fd["c0s"], list(levels0), D, H,
                                   PP, images.device)
    Mt, Et, posV0 = fd["kl0"]
    QK = torch.empty(C, R, 2 * D, device="cuda", dtype=torch.bfloat16)
    U = torch.empty(C, R, H, device="cuda", dtype=torch.float32)
    c0 = 0
    for gi, g in enumerate(levels0):
        Mq, bias = fd["nodes"][gi]                    # [g, NQ, PP] bf16, [g, NQ] fp32
        if H % 16:  # u too narrow for a GEMM of its own: one launch, u as the logit columns
            _lib.call("dchag_gemm_bf16", _lib.ptr(patches[:, c0]), g, B, S, PP, S * PP,
                      C * S * PP, PP, _lib.ptr(Mq), NQ, NQ * PP, 2 * D, _lib.ptr(bias), NQ,
                      0, 0, 0, 1, _lib.ptr(QK[c0]), 0, R * 2 * D, S * 2 * D, 2 * D,
                      _lib.ptr(U[c0]), R * H, S * H, H, st,
                      work={"site": "ops:fc_l0_qk", "flops": 2 * g * R * PP * NQ,
                            "bytes": g * R * (PP * 2 + 4 * D + 4 * H)})
        else:
            _lib.call("dchag_gemm_bf16", _lib.ptr(patches[:, c0]), g, B, S, PP, S * PP,
                      C * S * PP, PP, _lib.ptr(Mq), 2 * D, NQ * PP, 2 * D, _lib.ptr(bias), NQ,
                      0, 0, 0, 1, _lib.ptr(QK[c0]), 0, R * 2 * D, S * 2 * D, 2 * D, 0, 0, 0, 0,
                      st, work={"site": "ops:fc_l0_qk", "flops": 2 * g * R * PP * 2 * D,
                                "bytes": g * R * (PP + 2 * D) * 2})
            _lib.call("dchag_gemm_bf16", _lib.ptr(patches[:, c0]), g, B, S, PP, S * PP,
                      C * S * PP, PP, _lib.ptr(Mq[:, 2 * D:]), H, NQ * PP, 0,
                      _lib.ptr(bias[:, 2 * D:]), NQ, 0, 0, 0, 1, 0, 0, 0, 0, 0, _lib.ptr(U[c0]),
                      R * H, S * H, H, st,
                      work={"site": "ops:fc_l0_u", "flops": 2 * g * R * PP * H,
                            "bytes": g * R * (PP * 2 + H * 4)})
        c0 += g
    NH = unit_heads(D, H)
    poff, acc = [], 0
    for g in levels0:
        poff.append(acc)
        acc += g * R * H
    poff_t = _dev_i64(poff)
    pbuf = torch.empty(acc, device="cuda", dtype=torch.bfloat16)
    first_t, g_t = _dev_i32(fd["c0s"]), _dev_i32(levels0)
    _lib.call("dchag_fullcross_weights", n0, R, D, H, _lib.ptr(first_t), _lib.ptr(g_t),
              max(levels0), _lib.ptr(QK), R * 2 * D, 2 * D, _lib.ptr(U), R * H, 0,
              _lib.ptr(fd["posq"]), S, _lib.ptr(pbuf), _lib.ptr(poff_t), NH, st,
              work={"site": "ops:fullcross_weights", "bytes": C * R * (4 * D + 4 * H)})
    ctx = torch.empty(n0, R, D, device="cuda", dtype=torch.bfloat16)
    _lib.call("dchag_l0_node", _lib.ptr(img), img.stride(0), img.stride(1), B, Hh, Ww, patch, H,
              D, n0, _lib.ptr(first_t), _lib.ptr(g_t), _lib.ptr(poff_t), 1, _lib.ptr(pbuf), 0,
              _lib.ptr(Mt), C + 64 // PP, _lib.ptr(Et), 16 * ((max(levels0) + 15) // 16),
              _lib.ptr(posV0), _lib.ptr(ctx), st,
              work={"site": "ops:fc_l0_node", "flops": 2 * R * D * C * (PP + 1)})
    y = torch.empty(n0, R, D, device="cuda", dtype=torch.bfloat16)
    for k in range(n0):
        _, Wo, bo = _fc_node_weights(tw, f"{prefix}.l0.g{k}", D, H)
        _gemm(ctx[k], 1, R, D, 0, D, Wo, bo, y[k], 0, D)
    return y


def _dev_i64(vals):
    key = ("l", tuple(int(v) for v in vals))
    t = _SMALL.get(key)
    if t is None:
        t = _SMALL[key] = torch.tensor(key[1], device="cuda", dtype=torch.int64)
    return t


def _full_cross_tree(tokens, spec: TreeSpec, w, prefix, n_heads, out_dtype, x0=None):
    """full_cross nodes (layers.py:125-138): per node, the g children attend over each other
    (sdp_attention, layers.py:49-64), then a learned query rq reduces the g outputs. Folded:
    one projection GEMM per node gives [q | k | v | u] with u_jh = v_j,h . (wo rq)_h / sqrt(D)
    (the reduce's scores are linear in the attention outputs); dchag_fullcross_weights turns
    q, k, u into per-(child, head) weights w; dchag_combine_weighted sums the v rows; the
    node output is that sum @ wo + bo (exact: the reduce's softmax weights sum to 1)."""
    H = n_heads
    st = _lib.stream_handle()
    tw = {k: _f32(v) for k, v in w.items() if k.startswith(prefix + ".")}
    if x0 is not None:  # level-0 node outputs [n0, R, D] (full_cross_level0): start above
        B, S, D = tokens
        x = x0
    else:
        B, C, S, D = tokens.shape
        # node-major rows: x[j] is child j's [R, D]
        x = _bf(tokens).permute(1, 0, 2, 3).reshape(C, B * S, D).contiguous()
    R = B * S
    depth = len(spec.levels)
    for li, level in enumerate(spec.levels):
        if x0 is not None and li == 0:
            continue
        firsts, acc = [], 0
        for g in level:
            firsts.append(acc)
            acc += g
        nodes = [f"{prefix}.l{li}.g{gi}" for gi in range(len(level))]
        n_in = x.shape[0]
        QKV = torch.empty(n_in, R, 3 * D, device="cuda", dtype=torch.bfloat16)
        U = torch.empty(n_in, R, H, device="cuda", dtype=torch.float32)
        for node, f, g in zip(nodes, firsts, level):
            Wnk, _, _ = _fc_node_weights(tw, node, D, H)
            zero = _zeros(Wnk.shape[0])
            _gemm(x[f:f + g], 1, g * R, D, 0, D, Wnk, zero, QKV[f:f + g], 0, 3 * D,
                  U[f:f + g], 0, H)
        first_t = _dev_i32(firsts)
        g_t = _dev_i32(level)
        gmax = max(level)
        wts = torch.empty(len(level), R, gmax, H, device="cuda", dtype=torch.float32)
        _lib.call("dchag_fullcross_weights", len(level), R, D, H, _lib.ptr(first_t),
                  _lib.ptr(g_t), gmax, _lib.ptr(QKV), R * 3 * D, 3 * D, _lib.ptr(U), R * H,
                  _lib.ptr(wts), 0, S, 0, 0, 0, st,
                  work={"site": "ops:fullcross_weights", "bytes": n_in * R * (4 * D + 4 * H)})
        ctx = torch.empty(len(level), R, D, device="cuda", dtype=torch.bfloat16)
        _lib.call("dchag_combine_weighted", len(level), R, D, H, _lib.ptr(first_t),
                  _lib.ptr(g_t), gmax, _lib.ptr(QKV[:, :, 2 * D:]), R * 3 * D, 3 * D,
                  _lib.ptr(wts), _lib.ptr(ctx), st,
                  work={"site": "ops:combine_weighted", "bytes": n_in * R * 2 * D
                        + len(level) * R * 2 * D})
        last = li == depth - 1
        y = torch.empty(len(level), R, D, device="cuda",
                        dtype=out_dtype if last else torch.bfloat16)
        for k, node in enumerate(nodes):
            _, Wo, bo = _fc_node_weights(tw, node, D, H)
            _gemm(ctx[k], 1, R, D, 0, D, Wo, bo, y[k], 0, D, outV_f32=y.dtype == torch.float32)
        x = y
    return x.view(B, 1, S, D) if x.shape[0] == 1 else x.view(1, B, S, D).transpose(0, 1)


# bf16 operand forms of the full_cross node weights, folded once per weight version (an
# in-place update or a new tensor refolds; the forward never refolds unchanged weights)
_FC_CACHE: dict = {}
_SMALL: dict = {}


def _fc_node_weights(tw, node, D, H):
    """(W [q|k|v|u]^T bf16 [3D+H, D], wo^T bf16 [D, D], bo fp32) of a full_cross node:
    u_jh = v_j,h . (wo rq)_h / sqrt(D) (the rq reduce's scores are linear in the outputs)."""
    names = [f"{node}.{n}" for n in ("wq", "wk", "wv", "wo", "bo", "rq")]
    key = (node, D, H) + tuple((tw[n].data_ptr(), tw[n]._version, tuple(tw[n].shape))
                               for n in names)
    hit = _FC_CACHE.get(node)
    if hit is not None and hit[0] == key:
        return hit[1]
    dh = D // H
    with torch.no_grad():
        wr = tw[f"{node}.wo"] @ tw[f"{node}.rq"] / (D ** 0.5)                    # [D]
        Wu = (tw[f"{node}.wv"].view(D, H, dh) * wr.view(1, H, dh)).sum(-1)        # [D, H]
        Wc = torch.cat([tw[f"{node}.wq"], tw[f"{node}.wk"], tw[f"{node}.wv"], Wu], dim=1)
        val = (_bf(Wc.t()), _bf(tw[f"{node}.wo"].t()), _f32(tw[f"{node}.bo"]))
    _FC_CACHE[node] = (key, val)
    return val


def _zeros(n):
    t = _SMALL.get(("z", n))
    if t is None:
        t = _SMALL[("z", n)] = torch.zeros(n, device="cuda", dtype=torch.float32)
    return t


def _dev_i32(vals):
    """Device int32 table, made once per content (no per-call pageable H2D copy)."""
    key = ("i", tuple(int(v) for v in vals))
    t = _SMALL.get(key)
    if t is None:
        t = _SMALL[key] = torch.tensor(key[1], device="cuda", dtype=torch.int32)
    return t


def tree_aggregate(tokens, spec: TreeSpec, w, prefix, layer_kind, variant, n_heads,
                   out_dtype=torch.float32):
    """[B, C, S, D] -> [B, 1, S, D] (model.py:76-97): contiguous groups per level, node
    params under {prefix}.l{level}.g{group}."""
    if variant == "full_cross" and layer_kind != "linear":
        if sum(spec.levels[0]) != tokens.shape[1]:
            raise ConfigError(
                f"tree level 0 partitions {sum(spec.levels[0])} channels, input has "
                f"{tokens.shape[1]}")
        if max(max(lv) for lv in spec.levels) > 32:
            raise ConfigError("full_cross on sm_100a supports groups of <= 32 channels")
        return _full_cross_tree(tokens, spec, w, prefix, n_heads, out_dtype)
    if variant != "single_query" and layer_kind != "linear":
        raise ConfigError(f"unknown agg_variant {variant!r}")
    B, C, S, D = tokens.shape
    if sum(spec.levels[0]) != C:
        raise ConfigError(
            f"tree level 0 partitions {sum(spec.levels[0])} channels, input has {C}")
    if S % 128 or D % 64 or (D // n_heads) % 8:
        raise ConfigError("tree_aggregate on sm_100a needs S % 128 == 0 and D % 64 == 0")
    H = n_heads
    R = B * S
    st = _lib.stream_handle()
    tw = {k: _f32(v) for k, v in w.items() if k.startswith(prefix + ".")}
    x = _bf(tokens)
    # level inputs: x laid out [B][n_in][S][D] (level 0) or [n_in][R][D] (above)
    x_layout = "bsd"
    n_in = C
    depth = len(spec.levels)
    for li, level in enumerate(spec.levels):
        attn = layer_kind != "linear"
        nodes = [f"{prefix}.l{li}.g{gi}" for gi in range(len(level))]
        firsts, acc = [], 0
        for g in level:
            firsts.append(acc)
            acc += g
        # 1) project each node's inputs with its consumer weight Wcons = [wv | U] or w
        V = torch.empty(n_in, R, D, device="cuda", dtype=torch.bfloat16) if x_layout == "nrd" \
            else torch.empty(B, n_in, S, D, device="cuda", dtype=torch.bfloat16)
        L = None
        if attn:
            L = torch.empty(V.shape[:-1] + (H,), device="cuda", dtype=torch.float32)
        for node, f, g in zip(nodes, firsts, level):
            Wc, _ = consumer_weight(tw, node, layer_kind, H)          # [D, D(+H)]
            Wnk = _bf(Wc.t())
            zero = torch.zeros(Wnk.shape[0], device="cuda", dtype=torch.float32)
            if x_layout == "bsd":
                A = x[:, f:f + g]                                        # rows (b, j, s)
                _gemm(A, B, g * S, D, C * S * D, D, Wnk, zero, V[:, f:f + g], n_in * S * D, D,
                      L[:, f:f + g] if attn else None, n_in * S * H, H)
            else:
                A = x[f:f + g]
                _gemm(A, 1, g * R, D, 0, D, Wnk, zero, V[f:f + g], 0, D,
                      L[f:f + g] if attn else None, 0, H)
        # 2) combine children per node (+ linear bias b), then 3) node output projection
        ctx = torch.empty(len(level), R, D, device="cuda", dtype=torch.bfloat16)
        first_t = _dev_i32(firsts)
        g_t = _dev_i32(level)
        mix = None if attn else torch.cat([tw[f"{n}.mix"] for n in nodes]).contiguous()
        if x_layout == "bsd":
            sVj, sVb, sLj, sLb, rows_inner = S * D, n_in * S * D, S * H, n_in * S * H, S
        else:
            sVj, sVb, sLj, sLb, rows_inner = R * D, 0, R * H, 0, R
        _lib.call("dchag_combine_strided", len(level), R, D, H, _lib.ptr(first_t),
                  _lib.ptr(g_t), max(level), _lib.ptr(V), sVj, sVb, _lib.ptr(L), sLj, sLb,
                  rows_inner, _lib.ptr(mix), _lib.ptr(ctx), st)
        # node output y = ctx @ wo + bo (attention) or ctx + b (linear: w applied above)
        y = torch.empty(len(level), R, D, device="cuda",
                        dtype=out_dtype if li == depth - 1 else torch.bfloat16)
        for k, node in enumerate(nodes):
            if attn:
                _gemm(ctx[k], 1, R, D, 0, D, _bf(tw[f"{node}.wo"].t()),
                      tw[f"{node}.bo"].contiguous(), y[k], 0, D,
                      outV_f32=y.dtype == torch.float32)
            else:  # linear node: w was applied before the mix; only the bias remains
                torch.add(ctx[k], tw[f"{node}.b"], out=y[k])
        x, x_layout, n_in = y, "nrd", len(level)
    return x.view(B, 1, S, D) if x.shape[0] == 1 else x.view(1, B, S, D).transpose(0, 1)


def flat_aggregate(tokens, w, prefix, variant, n_heads, hooks=None, tag="aggregate",
                   out_dtype=torch.float32):
    """[B, Ck, S, D] -> [B, 1, S, D] (model.py:67-73): one node over all Ck tokens."""
    if hooks is not None:
        raise ConfigError("head-split hooks are not part of the sm_100a path")
    Ck = tokens.shape[1]
    node = {k.replace(prefix, f"{prefix}.__flat.l0.g0", 1): v for k, v in w.items()
            if k.startswith(prefix + ".")}
    return tree_aggregate(tokens, TreeSpec(((Ck,),)), node, f"{prefix}.__flat", "cross_attention",
                          variant, n_heads, out_dtype=out_dtype)


# ---------------------------------------------------------------- fp32 parity mode
# The reference is float64; BASELINE.json asks fp32 results within 1e-4 (max rel err). Every
# GEMM of this mode runs on the same tcgen05 kernel with each fp32 operand split into bf16
# high and low parts: [A_hi | A_lo | A_hi] . [W_hi | W_hi | W_lo] over a K three times as
# long = A W - A_lo W_lo (relative error ~2^-16, fp32 accumulation); combines run in fp32.

def _split3(x):
    """fp32 [..., K] -> bf16 [..., 3K] = [hi | lo | hi] (dchag_split3_bf16: one pass)."""
    x = _f32(x)
    K = x.shape[-1]
    x2 = x.reshape(-1, K)
    if x2.stride(-1) != 1 or x2.data_ptr() % 16 or x2.stride(0) % 4:
        x2 = x2.contiguous()
    out = torch.empty(x2.shape[0], 3 * K, device=x.device, dtype=torch.bfloat16)
    _lib.call("dchag_split3_bf16", _lib.ptr(x2), x2.shape[0], K, x2.stride(0), _lib.ptr(out),
              3 * K, _lib.stream_handle(),
              work={"site": "ops:split3", "bytes": x2.numel() * 10})
    return out.view(*x.shape[:-1], 3 * K)


_W3_CACHE: dict = {}


def _split_w3(W_dn):
    """bf16 [N, 3K] = [hi | hi | lo] of an fp32 weight [K, N], made once per weight version
    (keyed on storage, version counter and shape, like the full_cross fold cache)."""
    # the entry holds the source tensor itself: a hit needs the same live object at the same
    # version (a freed temporary's recycled storage can never match)
    key = (W_dn.data_ptr(), tuple(W_dn.shape), tuple(W_dn.stride()))
    hit = _W3_CACHE.get(key)
    if hit is not None and hit[0] is W_dn and hit[1] == W_dn._version:
        return hit[2]
    Wt = _f32(W_dn).t()
    hi = Wt.to(torch.bfloat16)
    lo = (Wt - hi.float()).to(torch.bfloat16)
    W3 = torch.cat([hi, hi, lo], dim=1).contiguous()
    if len(_W3_CACHE) > 256:
        _W3_CACHE.clear()
    _W3_CACHE[key] = (W_dn, W_dn._version, W3)
    return W3


def _gemm3(A, W_dn, bias, N_logit=0, out=None, out_L=None):
    """fp32 A [M, K] @ W_dn [K, N] + bias, fp32-accurate; returns fp32 [M, N - N_logit]
    (and the last N_logit columns separately), written into `out` / `out_L` when given
    (row-contiguous [M, N - N_logit] / [M, N_logit])."""
    M, K = A.shape
    N = W_dn.shape[1]
    if M % 128 or K % 16:
        raise ConfigError("fp32 mode needs rows % 128 == 0 and K % 16 == 0")
    A3 = _split3(A)
    W3 = _split_w3(W_dn)                                             # [N, 3K]
    Nv = N - N_logit
    V = out if out is not None else torch.empty(M, Nv, device="cuda", dtype=torch.float32)
    L = out_L if out_L is not None else torch.empty(M, max(N_logit, 1), device="cuda",
                                                    dtype=torch.float32)
    b = _f32(bias) if bias is not None else torch.zeros(N, device="cuda")
    _lib.call("dchag_gemm_bf16", _lib.ptr(A3), 1, 1, M, 3 * K, M * 3 * K, M * 3 * K, 3 * K,
              _lib.ptr(W3), N, N * 3 * K, Nv, _lib.ptr(b), N, 0, 0, N, 1, _lib.ptr(V), 1, 0, 0,
              Nv, _lib.ptr(L) if N_logit else 0, 0, 0, N_logit, _lib.stream_handle())
    return (V, L) if N_logit else V


def tokenize_channels_fp32(images, tok_w, tok_b, chan_id, pos, patch, node_major=False):
    """fp32 tokens [B, Cs, S, D] (model.py:51-64) with fp32-accurate GEMMs: one grouped
    split-bf16 GEMM over the channels (group = channel), tok.b + chan_id in its epilogue.
    node_major=True returns them as [Cs, B*S, D] (the tree's layout: no transposed copy)."""
    B, C, Hh, Ww = images.shape
    P = patch
    S, PP = (Hh // P) * (Ww // P), P * P
    D = tok_w.shape[-1]
    if (B * S) % 128 or PP % 16:
        raise ConfigError("fp32 mode needs B*S % 128 == 0 and P*P % 16 == 0")
    x = _f32(images)
    patches = x.reshape(B, C, Hh // P, P, Ww // P, P).permute(1, 0, 2, 4, 3, 5)
    patches = patches.reshape(C, B * S, PP)                           # unfold (tensor.py:303-323)
    A3 = _split3(patches)                                             # [C, R, 3 PP]
    Wt = _f32(tok_w).transpose(1, 2)                                  # [C, D, PP]
    hi = Wt.to(torch.bfloat16)
    lo = (Wt - hi.float()).to(torch.bfloat16)
    W3 = torch.cat([hi, hi, lo], dim=2).contiguous()                  # [C, D, 3 PP]
    bias = (_f32(tok_b) + _f32(chan_id)).contiguous()                 # [C, D]
    R, K3 = B * S, 3 * PP
    out = torch.empty(C, R, D, device="cuda", dtype=torch.float32)
    _lib.call("dchag_gemm_bf16", _lib.ptr(A3), C, 1, R, K3, R * K3, 0, K3, _lib.ptr(W3), D,
              D * K3, D, _lib.ptr(bias), D, 0, 0, 0, 1, _lib.ptr(out), 1, R * D, 0, D, 0, 0, 0, 0,
              _lib.stream_handle())
    if node_major:
        out.view(C, B, S, D).add_(_f32(pos)[None, None])
        return out
    return out.view(C, B, S, D).permute(1, 0, 2, 3) + _f32(pos)[None, None]


def tree_aggregate_fp32(tokens, spec: TreeSpec, w, prefix, layer_kind, n_heads, B=None):
    """fp32 [B, C, S, D] -> [B, 1, S, D] (model.py:76-97), single_query / linear nodes.
    A 3-D node-major [C, B*S, D] input (tokenize_channels_fp32(node_major=True)) needs B."""
    if tokens.dim() == 3:
        C, R, D = tokens.shape
        S = R // B
        x = _f32(tokens)
    else:
        B, C, S, D = tokens.shape
        R = B * S
        x = _f32(tokens).permute(1, 0, 2, 3).reshape(C, R, D).contiguous()
    H = n_heads
    st = _lib.stream_handle()
    tw = {k: _f32(v) for k, v in w.items() if k.startswith(prefix + ".")}
    attn = layer_kind != "linear"
    for li, level in enumerate(spec.levels):
        n_in = x.shape[0]
        nodes = [f"{prefix}.l{li}.g{gi}" for gi in range(len(level))]
        firsts, acc = [], 0
        for g in level:
            firsts.append(acc)
            acc += g
        V = torch.empty(n_in, R, D, device="cuda", dtype=torch.float32)
        L = torch.empty(n_in, R, H, device="cuda", dtype=torch.float32) if attn else None
        for node, f, g in zip(nodes, firsts, level):
            Wc, _ = consumer_weight(tw, node, layer_kind, H)
            if attn:
                _gemm3(x[f:f + g].reshape(g * R, D), Wc, None, N_logit=H,
                       out=V[f:f + g].view(g * R, D), out_L=L[f:f + g].view(g * R, H))
            else:
                _gemm3(x[f:f + g].reshape(g * R, D), Wc, None, out=V[f:f + g].view(g * R, D))
        ctx = torch.empty(len(level), R, D, device="cuda", dtype=torch.float32)
        first_t = _dev_i32(firsts)
        g_t = _dev_i32(level)
        mix = None if attn else torch.cat([tw[f"{n}.mix"] for n in nodes]).contiguous()
        _lib.call("dchag_combine_f32", len(level), R, D, H, _lib.ptr(first_t), _lib.ptr(g_t),
                  max(level), _lib.ptr(V), R * D, _lib.ptr(L), R * H, _lib.ptr(mix),
                  _lib.ptr(ctx), st)
        y = torch.empty(len(level), R, D, device="cuda", dtype=torch.float32)
        for k, node in enumerate(nodes):
            if attn:
                _gemm3(ctx[k], tw[f"{node}.wo"], tw[f"{node}.bo"], out=y[k])
            else:
                y[k] = ctx[k] + tw[f"{node}.b"]
        x = y
    return x.view(B, 1, S, D) if x.shape[0] == 1 else x.view(1, B, S, D).transpose(0, 1)


def flat_aggregate_fp32(tokens, w, prefix, n_heads):
    """fp32 single_query node over all Ck tokens (model.py:67-73)."""
    Ck = tokens.shape[1]
    node = {k.replace(prefix, f"{prefix}.__flat.l0.g0", 1): v for k, v in w.items()
            if k.startswith(prefix + ".")}
    return tree_aggregate_fp32(tokens, TreeSpec(((Ck,),)), node, f"{prefix}.__flat",
                               "cross_attention", n_heads)
