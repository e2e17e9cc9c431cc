"""CPU oracle for the D-CHAG channel front end -- TEST INFRASTRUCTURE ONLY.

This is a float64 numpy restatement of the reference algorithm
(`/root/reference/pkg/src/dchag`, a pure-Python/numpy simulator).  It exists
to check the CUDA path; only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s CPU-baseline leg may import it.  The product path
(`paper_2506_21411_b200`) never imports or calls it.

Parity pinning: `tests/test_oracle_golden.py` checks every function here
against golden vectors produced by the reference itself
(`tests/golden/make_golden.py` imports /root/reference and writes
`tests/golden/*.npz`), plus the reference's own brute-force oracles
(test_model.py:78-120) restated in `brute_force_single_query`.

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import math

import numpy as np

_REF = "/root/reference/pkg/src/dchag"


# -- layout -------------------------------------------------------------------


def unfold_patches(x: np.ndarray, patch: int) -> np.ndarray:
    """[..., C, H, W] -> [..., C, S, P*P]; token s = i*wp + j, pixel k = py*P + px.
    Restates tensor.py:303-323."""
    *lead, c, h, w = x.shape
    if h % patch or w % patch:
        raise ValueError(f"image {h}x{w} not divisible by patch {patch}")
    hp, wp = h // patch, w // patch
    v = x.reshape(*lead, c, hp, patch, wp, patch)
    nd = v.ndim
    perm = tuple(range(nd - 4)) + (nd - 4, nd - 2, nd - 3, nd - 1)
    return v.transpose(perm).reshape(*lead, c, hp * wp, patch * patch)


# -- layers -------------------------------------------------------------------


def tokenize_channels(images, tok_w, tok_b, chan_id, pos, patch):
    """tokens[b,c,s,:] = patch[b,c,s,:] @ tok_w[c] + tok_b[c] + chan_id[c] + pos[s].
    Restates model.py:51-64 (unfold + broadcast matmul + three adds)."""
    p = unfold_patches(np.asarray(images, np.float64), patch)          # [B,C,S,PP]
    tok = np.einsum("bcsk,ckd->bcsd", p, tok_w, optimize=True)
    tok = tok + tok_b[None, :, None, :]
    tok = tok + chan_id[None, :, None, :]
    return tok + pos[None, None, :, :]


def _softmax(x, axis=-1):
    """Max-subtracted softmax (tensor.py:194-205)."""
    m = x.max(axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=axis, keepdims=True)


def cross_attention_single_query(x, w, prefix, n_heads):
    """Learned-query reduce over the channel axis (-2) of x[..., Ck, D].
    Restates layers.py:103-123 literally (K and V projections formed)."""
    d = x.shape[-1]
    dh = d // n_heads
    k = x @ w[f"{prefix}.wk"]
    v = x @ w[f"{prefix}.wv"]
    q = w[f"{prefix}.q"] @ w[f"{prefix}.wq"]                              # [D]
    kh = k.reshape(*k.shape[:-1], n_heads, dh)                           # [..., Ck, H, dh]
    vh = v.reshape(*v.shape[:-1], n_heads, dh)
    logits = np.einsum("...chd,hd->...hc", kh, q.reshape(n_heads, dh)) / math.sqrt(dh)
    p = _softmax(logits, axis=-1)                                         # [..., H, Ck]
    ctx = np.einsum("...hc,...chd->...hd", p, vh).reshape(*x.shape[:-2], d)
    out = ctx @ w[f"{prefix}.wo"] + w[f"{prefix}.bo"]
    return out[..., None, :]                                              # [..., 1, D]


def cross_attention_full_cross(x, w, prefix, n_heads):
    """Ck x Ck self-attention over channels, then learned-rq reduce.
    Restates layers.py:125-138 with sdp_attention layers.py:49-64."""
    d = x.shape[-1]
    dh = d // n_heads
    q = x @ w[f"{prefix}.wq"]
    k = x @ w[f"{prefix}.wk"]
    v = x @ w[f"{prefix}.wv"]
    sh = lambda t: t.reshape(*t.shape[:-1], n_heads, dh)
    logits = np.einsum("...chd,...ehd->...hce", sh(q), sh(k)) / math.sqrt(dh)
    p = _softmax(logits, axis=-1)
    ctx = np.einsum("...hce,...ehd->...chd", p, sh(v)).reshape(x.shape)
    out = ctx @ w[f"{prefix}.wo"] + w[f"{prefix}.bo"]                     # [..., Ck, D]
    scores = out @ w[f"{prefix}.rq"] / math.sqrt(d)                      # [..., Ck]
    pr = _softmax(scores, axis=-1)
    return np.einsum("...c,...cd->...d", pr, out)[..., None, :]


def cross_attention_aggregate(x, w, prefix, variant, n_heads):
    """layers.py:94-138 dispatch."""
    if variant == "single_query":
        return cross_attention_single_query(x, w, prefix, n_heads)
    return cross_attention_full_cross(x, w, prefix, n_heads)


def linear_mix_aggregate(x, w, prefix):
    """out = (sum_g mix_g x_g) @ W + b.  Restates layers.py:141-146."""
    mixed = np.einsum("g,...gd->...d", w[f"{prefix}.mix"], x)
    return (mixed @ w[f"{prefix}.w"] + w[f"{prefix}.b"])[..., None, :]


def flat_aggregate(tokens, w, prefix, variant, n_heads):
    """[B,Ck,S,D] -> [B,1,S,D].  Restates model.py:67-73."""
    xt = tokens.transpose(0, 2, 1, 3)
    out = cross_attention_aggregate(xt, w, prefix, variant, n_heads)
    return out.transpose(0, 2, 1, 3)


def tree_aggregate(tokens, levels, w, prefix, layer_kind, variant, n_heads):
    """Hierarchical reduce; node params under {prefix}.l{li}.g{gi}.
    Restates model.py:76-97 (contiguous narrow per group, concat in group order)."""
    if sum(levels[0]) != tokens.shape[1]:
        raise ValueError(
            f"tree level 0 partitions {sum(levels[0])} channels, input has {tokens.shape[1]}")
    x = tokens.transpose(0, 2, 1, 3)                                      # [B,S,C,D]
    for li, level in enumerate(levels):
        outs, off = [], 0
        for gi, g in enumerate(level):
            xg = x[:, :, off:off + g]
            off += g
            node = f"{prefix}.l{li}.g{gi}"
            if layer_kind == "linear":
                outs.append(linear_mix_aggregate(xg, w, node))
            else:
                outs.append(cross_attention_aggregate(xg, w, node, variant, n_heads))
        x = np.concatenate(outs, axis=2)
    return x.transpose(0, 2, 1, 3)


def build_levels(n: int, max_group: int):
    """config.py:48-66 (greedy balanced contiguous grouping)."""
    levels = []
    while True:
        k = -(-n // max_group)
        base, rem = divmod(n, k)
        levels.append(tuple([base + 1] * rem + [base] * (k - rem)))
        if k == 1:
            return tuple(levels)
        n = k


def slabs(channels: int, tp: int):
    """Balanced contiguous slabs; equals strategies.py:162-164 when tp | C."""
    base, extra = divmod(channels, tp)
    out, off = [], 0
    for r in range(tp):
        cnt = base + (1 if r < extra else 0)
        out.append((off, cnt))
        off += cnt
    return out


def dchag_frontend(images, w, *, patch, heads, tp, max_group, variant="single_query",
                   layer_kind="cross_attention", return_streams=False):
    """Hot path of forward_loss_dchag_reference (model.py:180-201): per-slab
    tokenize + tree, streams concatenated in slab order (== the AllGather,
    runtime.py:259), shared final layer "agg.final".  Uneven slabs use the
    balanced extension; each rank r's tree is build_levels(c_r, max_group)."""
    streams = []
    for r, (off, cnt) in enumerate(slabs(images.shape[1], tp)):
        tok = tokenize_channels(images[:, off:off + cnt], w["tok.w"][off:off + cnt],
                                w["tok.b"][off:off + cnt],
                                w["special.channel_id"][off:off + cnt],
                                w["special.pos"], patch)
        streams.append(tree_aggregate(tok, build_levels(cnt, max_group), w,
                                      f"agg.slab{r}", layer_kind, variant, heads))
    gathered = np.concatenate(streams, axis=1)
    out = flat_aggregate(gathered, w, "agg.final", variant, heads)
    return (out, gathered) if return_streams else out


# -- parameters ------------------------------------------------------------


def apply_token_mask(agg, mask, mask_token):
    """model.py:100-108: agg [B,1,S,D] * (1 - m) + mask_token * m, m = mask[B,S]."""
    b, s = mask.shape
    m = mask.reshape(b, 1, s, 1)
    return agg * (1.0 - m) + mask_token.reshape(1, 1, 1, -1) * m


def vit_input(agg, mask, mask_token, meta, meta_w, meta_b):
    """model.py:100-108 + :111-117 (the trunk's first two steps): the masked aggregate
    prefixed by the metadata token, [B, S+1, D]."""
    b, _, s, d = agg.shape
    masked = apply_token_mask(agg, mask, mask_token)
    meta_tok = (meta @ meta_w + meta_b).reshape(b, 1, d)
    return np.concatenate([meta_tok, masked.reshape(b, s, d)], axis=1)


def frontend_param_specs(channels, image_h, image_w, patch, embed, tp, max_group,
                         variant="single_query", layer_kind="cross_attention"):
    """Names/shapes in the reference creation order (params.py:36-57, :99-115),
    front-end subset, with per-rank trees for uneven slabs."""
    s = (image_h // patch) * (image_w // patch)
    d = embed

    def node(prefix, g, kind):
        if kind == "linear":
            return [(f"{prefix}.mix", (g,), "normal"), (f"{prefix}.w", (d, d), "normal"),
                    (f"{prefix}.b", (d,), "zeros")]
        sp = [(f"{prefix}.q", (d,), "normal")] if variant == "single_query" else []
        sp += [(f"{prefix}.{n}", (d, d), "normal") for n in ("wq", "wk", "wv", "wo")]
        sp += [(f"{prefix}.bo", (d,), "zeros")]
        if variant == "full_cross":
            sp.append((f"{prefix}.rq", (d,), "normal"))
        return sp

    specs = [("tok.w", (channels, patch * patch, d), "normal"), ("tok.b", (channels, d), "zeros"),
             ("special.channel_id", (channels, d), "normal"), ("special.pos", (s, d), "normal")]
    for r, (_, cnt) in enumerate(slabs(channels, tp)):
        for li, level in enumerate(build_levels(cnt, max_group)):
            for gi, g in enumerate(level):
                specs += node(f"agg.slab{r}.l{li}.g{gi}", g, layer_kind)
    specs += node("agg.final", tp, "cross_attention")
    return specs


def random_params(specs, seed=0, std=0.02, bias_std=0.0):
    """Seeded truncated-normal(std) weights (rng.py:52-60 distribution, numpy
    PCG64 stream -- not the reference Philox stream); zero biases unless
    bias_std > 0 (used by tests to exercise the bias paths)."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape, init in specs:
        if init == "zeros":
            out[name] = rng.standard_normal(shape) * bias_std if bias_std else np.zeros(shape)
        else:
            v = rng.standard_normal(shape)
            bad = np.abs(v) > 2.0
            while bad.any():
                v[bad] = rng.standard_normal(int(bad.sum()))
                bad = np.abs(v) > 2.0
            out[name] = v * std
    return out


def rel_err(a, b, floor=1e-300):
    """max|a-b| / (max|a| + max|b|): the reference's parity metric (tests/conftest.py:8-13)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max(initial=0.0)
                 / (np.abs(a).max(initial=0.0) + np.abs(b).max(initial=0.0) + floor))


def brute_force_single_query(tokens, q, wq, wk, wv, wo, bo, heads):
    """Explicit-loop oracle of the learned-query reduce (test_model.py:78-97)."""
    b_, c, s, d = tokens.shape
    dh = d // heads
    out = np.zeros((b_, 1, s, d))
    qp = q @ wq
    for b in range(b_):
        for si in range(s):
            x = tokens[b, :, si, :]
            k, v = x @ wk, x @ wv
            merged = np.zeros(d)
            for h in range(heads):
                sl = slice(h * dh, (h + 1) * dh)
                lg = np.array([qp[sl] @ k[cc, sl] for cc in range(c)]) / np.sqrt(dh)
                e = np.exp(lg - lg.max())
                p = e / e.sum()
                merged[sl] = sum(p[cc] * v[cc, sl] for cc in range(c))
            out[b, 0, si, :] = merged @ wo + bo
    return out
