"""float64 torch emulation of the folded execution plan the CUDA kernels implement.

Test infrastructure: it replays, op for op, what K_p0 / K_l0 / K_gemm / K_comb
compute (paper_2506_21411_b200/fold.py explains the algebra), so the CPU suite can
pin the *algebra* of the fused path to the oracle independently of the kernels.
"""
import torch

from paper_2506_21411_b200.fold import fold_rank


def unfold(images, p):
    b, c, h, w = images.shape
    v = images.reshape(b, c, h // p, p, w // p, p).permute(0, 1, 2, 4, 3, 5)
    return v.reshape(b, c, (h // p) * (w // p), p * p)


def emulate_rank(fr, images, heads):
    """images: [B, c_r, H, W] float64 -> (V_root [R, D], L_root [R, H], ctx_root [R, D])."""
    d, h = fr.embed, heads
    dh = d // h
    B = images.shape[0]
    pt = unfold(images, fr.patch)                                   # [B, C, S, PP]
    s = pt.shape[2]
    R = B * s
    pt = pt.permute(1, 0, 2, 3).reshape(pt.shape[1], R, -1)         # [C, R, PP]
    srow = torch.arange(R) % s
    ctxs = []
    for n, (c0, g) in enumerate(zip(fr.l0_c0, fr.l0_g)):
        Vc = torch.einsum("crk,ckd->crd", pt[c0:c0 + g], fr.M[c0:c0 + g]) + fr.Cb[c0:c0 + g, None]
        if fr.attn_l0:
            Lc = (torch.einsum("crk,ckh->crh", pt[c0:c0 + g], fr.WU[c0:c0 + g])
                  + fr.bU[c0:c0 + g, None] + fr.posU[n][srow][None])
            p = torch.softmax(Lc, dim=0)                            # [g, R, H]
        else:
            p = fr.mix0[c0:c0 + g].view(g, 1, 1).expand(g, R, h)
        pe = p.repeat_interleave(dh, dim=2)                         # [g, R, D]
        ctxs.append((pe * Vc).sum(0) + fr.posV[n][srow])
    ctx = torch.stack(ctxs)
    depth = len(fr.levels)
    for li in range(depth):
        out = torch.einsum("nrk,nkj->nrj", ctx, fr.Wp[li]) + fr.bp[li][:, None]
        V, L = out[..., :d], (out[..., d:] if fr.has_logits[li] else None)
        if li + 1 < depth:
            nxt = []
            for first, g, in zip(fr.comb_first[li], fr.comb_g[li]):
                if fr.comb_mix[li] is None:
                    p = torch.softmax(L[first:first + g], dim=0).repeat_interleave(dh, dim=2)
                else:
                    p = fr.comb_mix[li][first:first + g].view(g, 1, 1)
                nxt.append((p * V[first:first + g]).sum(0))
            ctx = torch.stack(nxt)
    return V[0], L[0], ctx[0]


def emulate_frontend(w, images, *, slabs, trees, embed, heads, patch, variant, layer_kind,
                     fold_root_final=False):
    """All ranks + AllGather (concat in rank order) + shared final layer.
    fold_root_final (tp == 1 only): the plan DchagFrontEnd runs at one stream -- the final
    softmax over one stream is 1, so out = ctx_root @ (Wp_root[:, :D] @ Wf) + (bp_root[:D]
    @ Wf + bf), one GEMM with the weights pack_rank folds (Wdir, bdir)."""
    dh = embed // heads
    Vs, Ls, fr = [], [], None
    for r, ((off, cnt), tree) in enumerate(zip(slabs, trees)):
        fr = fold_rank(w, rank=r, slab=(off, cnt), levels=tree, embed=embed, heads=heads,
                       patch=patch, seq=(images.shape[2] // patch) * (images.shape[3] // patch),
                       variant=variant, layer_kind=layer_kind)
        V, L, ctx_root = emulate_rank(fr, images[:, off:off + cnt], heads)
        if fold_root_final:
            assert len(slabs) == 1, "the root/final fold is the tp == 1 plan"
            Wdir = fr.Wp[-1][0][:, :embed] @ fr.Wf
            bdir = fr.bp[-1][0][:embed] @ fr.Wf + fr.bf
            return (ctx_root @ Wdir + bdir).view(images.shape[0], 1, -1, embed)
        Vs.append(V)
        Ls.append(L)
    V, L = torch.stack(Vs), torch.stack(Ls)
    p = torch.softmax(L, dim=0).repeat_interleave(dh, dim=2)
    ctx = (p * V).sum(0)
    out = ctx @ fr.Wf + fr.bf
    B = images.shape[0]
    return out.view(B, 1, -1, embed)
