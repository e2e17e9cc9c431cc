"""float64 torch restatement of the reference front end WITH autograd -- test infrastructure.

It follows oracle/dchag_oracle.py line for line (which cites the reference file:line of
every step) but in torch, so `torch.autograd` gives the gradients of sum(out * probe) for
any configuration. tests/test_train_reference.py pins it to the golden gradients the
reference itself produced (tests/golden/*.npz, grad:* arrays). The GPU training tests
then compare the sm_100a backward against it.
"""
import math

import torch

import dchag_oracle as O


def _unfold(x, p):
    b, c, h, w = x.shape
    v = x.reshape(b, c, h // p, p, w // p, p).permute(0, 1, 2, 4, 3, 5)
    return v.reshape(b, c, (h // p) * (w // p), p * p)


def tokenize(images, tok_w, tok_b, cid, pos, p):
    pt = _unfold(images, p)
    return torch.einsum("bcsk,ckd->bcsd", pt, tok_w) + (tok_b + cid)[None, :, None, :] + pos


def single_query(x, w, prefix, heads):
    d = x.shape[-1]
    dh = d // heads
    k, v = x @ w[f"{prefix}.wk"], x @ w[f"{prefix}.wv"]
    q = w[f"{prefix}.q"] @ w[f"{prefix}.wq"]
    kh = k.reshape(*k.shape[:-1], heads, dh)
    vh = v.reshape(*v.shape[:-1], heads, dh)
    lg = torch.einsum("...chd,hd->...hc", kh, q.reshape(heads, dh)) / math.sqrt(dh)
    p = torch.softmax(lg, dim=-1)
    ctx = torch.einsum("...hc,...chd->...hd", p, vh).reshape(*x.shape[:-2], d)
    return (ctx @ w[f"{prefix}.wo"] + w[f"{prefix}.bo"])[..., None, :]


def full_cross(x, w, prefix, heads):
    """Ck x Ck channel self-attention + learned-rq reduce (oracle cross_attention_full_cross,
    layers.py:125-138 with sdp_attention :49-64)."""
    d = x.shape[-1]
    dh = d // heads
    sh = lambda t: t.reshape(*t.shape[:-1], heads, dh)  # noqa: E731
    q, k, v = x @ w[f"{prefix}.wq"], x @ w[f"{prefix}.wk"], x @ w[f"{prefix}.wv"]
    lg = torch.einsum("...chd,...ehd->...hce", sh(q), sh(k)) / math.sqrt(dh)
    p = torch.softmax(lg, dim=-1)
    ctx = torch.einsum("...hce,...ehd->...chd", p, sh(v)).reshape(x.shape)
    out = ctx @ w[f"{prefix}.wo"] + w[f"{prefix}.bo"]
    pr = torch.softmax(out @ w[f"{prefix}.rq"] / math.sqrt(d), dim=-1)
    return torch.einsum("...c,...cd->...d", pr, out)[..., None, :]


def linear_mix(x, w, prefix):
    mixed = torch.einsum("g,...gd->...d", w[f"{prefix}.mix"], x)
    return (mixed @ w[f"{prefix}.w"] + w[f"{prefix}.b"])[..., None, :]


def tree(tokens, levels, w, prefix, layer_kind, heads, variant="single_query"):
    x = tokens.permute(0, 2, 1, 3)
    for li, level in enumerate(levels):
        outs, off = [], 0
        for gi, g in enumerate(level):
            node = f"{prefix}.l{li}.g{gi}"
            xg = x[:, :, off:off + g]
            off += g
            outs.append(linear_mix(xg, w, node) if layer_kind == "linear"
                        else full_cross(xg, w, node, heads) if variant == "full_cross"
                        else single_query(xg, w, node, heads))
        x = torch.cat(outs, dim=2)
    return x.permute(0, 2, 1, 3)


def frontend(images, w, *, patch, heads, tp, max_group, layer_kind="cross_attention",
             variant="single_query"):
    streams = []
    for r, (off, cnt) in enumerate(O.slabs(images.shape[1], tp)):
        tok = tokenize(images[:, off:off + cnt], w["tok.w"][off:off + cnt],
                       w["tok.b"][off:off + cnt], w["special.channel_id"][off:off + cnt],
                       w["special.pos"], patch)
        streams.append(tree(tok, O.build_levels(cnt, max_group), w, f"agg.slab{r}", layer_kind,
                            heads, variant))
    gathered = torch.cat(streams, dim=1).permute(0, 2, 1, 3)
    final = full_cross if variant == "full_cross" else single_query
    return final(gathered, w, "agg.final", heads).permute(0, 2, 1, 3)


def grads(images, w_np, probe, **cfg):
    """(out, {name: grad}) of sum(out * probe) in float64."""
    w = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in w_np.items()}
    out = frontend(torch.as_tensor(images, dtype=torch.float64), w, **cfg)
    (out * torch.as_tensor(probe, dtype=torch.float64)).sum().backward()
    return out.detach().numpy(), {k: t.grad.numpy() if t.grad is not None else
                                  torch.zeros_like(t).numpy() for k, t in w.items()}
