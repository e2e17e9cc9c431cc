"""Training step of the D-CHAG front end: forward with saved activations + backward.

Reference semantics: `T.backward` over the hot path of forward_loss_dchag_reference /
dchag_forward_loss (model.py:180-201, strategies.py:195-218, tensor.py:395-413), gather
backward = local slice (strategies.py:91-94), and the special.pos gradient all-reduced over
the channel group (strategies.py:251-264).

Forward (`forward_train`) runs the sm_100a kernels: K_p0 + K_l0 for level 0 (tokens never
formed), and unfolded node projections above it, so every node output y is kept for the
weight gradients. The AllGather moves the root streams y_r themselves, in rank order. The
replicated final layer then projects them on every rank, so its gradients are identical
everywhere, as in the reference.

Backward (`backward`): the non-GEMM parts run on an sm_100a kernel, dchag_combine_bwd
(softmax-weighted child sum backward: dp, softmax backward, p*g). These are plain GEMMs
(cuBLAS through torch.matmul, bf16 in / fp32 accumulate):
  y = ctx wo + bo  ->  d wo = ctx^T g,  g_ctx = g wo^T
  [V | L] = y_child [wv | U]  ->  d wv = y^T gV,  dU = y^T dL,  g_y = gV wv^T + dL U^T
At level 0 each node's tokens are recomputed with the tcgen05 tokenizer GEMM
(dchag_gemm_bf16), one node at a time. That gives d tok.w = patches^T g_x,
d tok.b = d channel_id = sum_rows g_x, d pos = sum_{b,c} g_x.
dU -> (wk, q, wq) follows U[:, h] = wk[:, h-blk] (q wq)[h-blk] / sqrt(dh) (fold.py).
"""

from __future__ import annotations

import math
import os
import weakref

import torch

from . import _lib, comm
from .config import ConfigError
from .fold import query_logit_weights
from .frontend import DchagFrontEnd
from .payload import payload_nbytes  # noqa: F401  (layout reference)


def _bf(t):
    return t.to(torch.bfloat16).contiguous()


def _f32(t):
    return t.to(torch.float32).contiguous()


def _gemm(A, W_dn, bias=None, out_f32=False, rowbias=None, period=1, N_logit=0, out=None,
          out_l=None):
    """y[m, :] = A[m, :] @ W_dn + bias (+ rowbias[m % period]) with the sm_100a GEMM.
    A [M, K] bf16 (M % 128 == 0), W_dn [K, N] (reference x @ W layout). Columns >= N - N_logit
    come back as a separate fp32 tensor. `out` / `out_l` (contiguous) receive the results
    in place."""
    M, K = A.shape
    N = W_dn.shape[1]
    Nv = N - N_logit
    W = _bf_t(W_dn)
    b = _f32(bias) if bias is not None else torch.zeros(N, device=A.device)
    V = out if out is not None else torch.empty(
        M, Nv, device=A.device, dtype=torch.float32 if out_f32 else torch.bfloat16)
    L = out_l if out_l is not None else torch.empty(M, max(N_logit, 1), device=A.device,
                                                   dtype=torch.float32)
    rb = _bf(rowbias) if rowbias is not None else None
    _lib.call("dchag_gemm_bf16", _lib.ptr(A), 1, 1, M, K, M * K, M * K, K, _lib.ptr(W), N, N * K,
              Nv, _lib.ptr(b), N, _lib.ptr(rb), 0, N, period, _lib.ptr(V), int(out_f32), 0, 0, Nv,
              _lib.ptr(L) if N_logit else 0, 0, 0, N_logit, _lib.stream_handle())
    return (V, L) if N_logit else V


def _mm(a, b):
    """Plain GEMM on tensor cores: bf16 operands, fp32 accumulate (cuBLAS), fp32 result.
    bf16 copies of (fp32) weight operands are cached per tensor version."""
    a, b = _bfc(a), _bfc(b)
    if a.dim() == 2 and b.dim() == 2:
        return torch.mm(a, b, out_dtype=torch.float32)
    if a.dim() == 3 and b.dim() == 3:
        return torch.bmm(a, b, out_dtype=torch.float32)
    return torch.matmul(a, b).float()


# bf16 copies of the module's fp32 parameters (and their .t() / slice views), per parameter
# tensor object (checked through a weak reference, so a new tensor that reuses a freed
# address or id never sees a stale copy) and per tensor version
_BF_CACHE: dict = {}       # id(tensor) -> (weakref to it, {view key: bf16 copy})
_BF_WEIGHTS: set = set()   # ids of the module's parameter tensors (DchagTrainer)
_CAPTURING = [False]       # inside a CUDA-graph capture: conversions are recorded, not cached


def _cached(t, tag, make):
    base = t._base if t._base is not None else t
    if id(base) not in _BF_WEIGHTS or _CAPTURING[0] or base.numel() < 4096:
        return make()
    ent = _BF_CACHE.get(id(base))
    if ent is None or ent[0]() is not base:
        if len(_BF_CACHE) > 4096:
            _BF_CACHE.clear()
        ent = _BF_CACHE[id(base)] = (weakref.ref(base), {})
    per = ent[1]
    key = (tag, base._version, t.stride(), t.storage_offset(), tuple(t.shape))
    v = per.get(key)
    if v is None:
        if len(per) > 64:
            per.clear()
        v = per[key] = make()
    return v


def _bf_t(w):
    """Contiguous bf16 transpose of w; cached for the module's parameters (and views of them)."""
    return _cached(w, "T", lambda: _bf(w.t()))


def _bfc(t):
    """bf16 view of t; the module's fp32 parameters are converted once per version and cached
    (their .t() / slice views too). Temporaries are never cached (their storage is reused)."""
    if t.dtype == torch.bfloat16:
        return t
    return _cached(t, "bf", lambda: t.to(torch.bfloat16))


def _u_backward(w, prefix, dU, heads):
    """Gradients of wk, q, wq from dU where U[:,h] = wk[:,h-blk] q'[h-blk]/sqrt(dh), q' = q wq."""
    wk, wq, q = w[f"{prefix}.wk"], w[f"{prefix}.wq"], w[f"{prefix}.q"]
    d = wk.shape[0]
    dh = d // heads
    qp = q @ wq
    s = 1.0 / math.sqrt(dh)
    d_wk = (dU.view(d, heads, 1) * qp.view(1, heads, dh)).reshape(d, d) * s
    d_qp = (wk.view(d, heads, dh) * dU.view(d, heads, 1)).sum(0).reshape(d) * s
    return {f"{prefix}.wk": d_wk, f"{prefix}.wq": torch.outer(q, d_qp), f"{prefix}.q": wq @ d_qp}


class DchagTrainer:
    """Forward + backward of one rank's front end (tp ranks share the final layer)."""

    def __init__(self, fe: DchagFrontEnd, dp_group=None):
        """dp_group: the data-parallel group of this rank (grid.make_groups); backward()
        then averages every gradient over it (strategies.py:352-357)."""
        if fe.model.agg_variant != "single_query":
            raise ConfigError("training path implements agg_variant='single_query'")
        self.fe = fe
        self.dp_group = dp_group
        self._ints = {}

    def _dev_ints(self, vals, dtype, dev):
        """Small host-known index arrays on the device, made once (no copies inside a step,
        so the step can be captured in a CUDA graph)."""
        key = (tuple(int(v) for v in vals), dtype, str(dev))
        t = self._ints.get(key)
        if t is None:
            t = self._ints[key] = torch.tensor(key[0], device=dev, dtype=dtype)
        return t

    def capture(self, images, g_out, warmup: int = 2):
        """One training step (forward_train + backward) captured as a CUDA graph over the
        static buffers `images` / `g_out`: refill them in place and call .replay(). The
        folded kernel weights are read by pointer, so reload weights (or refold) before
        capturing again. Returns a GraphedStep with .out, .grads (written by every replay)
        and .launches (library kernel launches per replay)."""
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for _ in range(warmup):
                out, saved = self.forward_train(images)
                self.backward(saved, g_out)
        cur.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        n0 = _lib.LAUNCH_COUNT["n"]
        _CAPTURING[0] = True
        try:
            with torch.cuda.graph(graph):
                out, saved = self.forward_train(images)
                grads = self.backward(saved, g_out)
        finally:
            _CAPTURING[0] = False
        return GraphedStep(graph, out, grads, _lib.LAUNCH_COUNT["n"] - n0)

    # ---------------------------------------------------------------- forward
    def forward_local(self, images):
        """Slab tokenizer + tree of this rank up to its root stream (saved['y_root'])."""
        fe = self.fe
        m = fe.model
        pk = fe.prepare()
        w = fe.weights
        d, h, s = m.embed, m.heads, fe.seq
        attn = fe.strategy.agg_layer_kind != "linear"
        off, cnt = fe.slab
        if images.shape[1] == m.channels and fe.tp > 1:
            images = images[:, off:off + cnt]
        img = images.to(torch.bfloat16).contiguous()
        B = img.shape[0]
        R = B * s
        levels = fe.tree.levels
        pre = f"agg.slab{fe.rank}"
        saved = {"img": img, "B": B, "R": R}
        # ---- level 0 context via the fused kernels (p and ctx kept)
        dev = img.device
        st = _lib.stream_handle()
        if pk.attn_l0:
            poff, acc = [], 0
            for g in pk.l0_g_list:
                poff.append(acc)
                acc += g * R * h
            poff_t = self._dev_ints(poff, torch.int64, dev)
            pbuf = torch.empty(acc, device=dev, dtype=torch.bfloat16)
            pinv = torch.empty(pk.n0, R, h, device=dev, dtype=torch.float32)
            _lib.call("dchag_l0_logits", _lib.ptr(img), img.stride(0), img.stride(1), B,
                      m.image_h, m.image_w, m.patch, h, pk.HP, pk.NH, pk.n0, max(pk.l0_g_list),
                      _lib.ptr(pk.l0_c0), _lib.ptr(pk.l0_g), _lib.ptr(poff_t), _lib.ptr(pk.WUt),
                      _lib.ptr(pk.bU), _lib.ptr(pk.posU), _lib.ptr(pbuf), _lib.ptr(pinv), st)
            prow = 1
        else:
            poff_t = (pk.l0_c0.to(torch.int64) * h).contiguous()
            pbuf, prow, pinv = pk.p_const, 0, None
        ctx0 = torch.empty(pk.n0, R, d, device=dev, dtype=torch.bfloat16)
        # positional term of the level-0 context, pos @ Vw_n (x sum(mix) for linear nodes),
        # added by K_l0 in its drain
        posV0 = self._level0_posV().to(torch.bfloat16).contiguous()
        _lib.call("dchag_l0_node", _lib.ptr(img), img.stride(0), img.stride(1), B, m.image_h,
                  m.image_w, m.patch, h, d, pk.n0, _lib.ptr(pk.l0_c0), _lib.ptr(pk.l0_g),
                  _lib.ptr(poff_t), prow, _lib.ptr(pbuf), _lib.ptr(pinv), _lib.ptr(pk.Mt), pk.C_pad,
                  _lib.ptr(pk.Et), pk.KE, _lib.ptr(posV0), _lib.ptr(ctx0), st)
        saved["ctx"] = [ctx0]
        y = torch.empty(len(levels[0]), R, d, device=dev, dtype=torch.bfloat16)
        for gi in range(len(levels[0])):
            node = f"{pre}.l0.g{gi}"
            if attn:
                _gemm(ctx0[gi], w[f"{node}.wo"], w[f"{node}.bo"], out=y[gi])
            else:
                torch.add(ctx0[gi], w[f"{node}.b"], out=y[gi])
        saved["y"] = [y]
        saved["VL"] = []
        # ---- levels >= 1 (unfolded)
        for li in range(1, len(levels)):
            V, L, ctx, ynext = self._level_forward(y, levels[li], li, pre, attn, R)
            saved["VL"].append((V, L))
            saved["ctx"].append(ctx)
            saved["y"].append(ynext)
            y = ynext
        saved["y_root"] = y[0].contiguous()
        return saved

    def forward_train(self, images):
        """Full forward of this rank: slab tree, AllGather of the root streams (rank order,
        runtime.py:259), shared final layer.  Returns ([B,1,S,D] fp32, saved)."""
        _BF_WEIGHTS.clear()
        _BF_WEIGHTS.update(id(v) for v in self.fe.weights.values())
        saved = self.forward_local(images)
        fe = self.fe
        y_root = saved["y_root"]
        if fe.tp > 1:
            y_all = torch.empty((fe.tp,) + tuple(y_root.shape), device=y_root.device,
                                dtype=torch.bfloat16)
            comm.all_gather_into_tensor(y_all, y_root, group=fe.process_group)
            fe._log("AllGather", "forward", "dchag-boundary",
                    y_root.numel() * y_root.element_size())
        else:
            y_all = y_root.unsqueeze(0)
        return self.forward_final(y_all, saved), saved

    def forward_final(self, y_all, saved):
        """Shared final layer over the gathered streams y_all [tp, R, D] (replicated)."""
        fe = self.fe
        if fe.strategy.final_layer_tp_split and fe.tp > 1:
            return self._forward_final_split(y_all, saved)
        w = fe.weights
        d, h, s = fe.model.embed, fe.model.heads, fe.seq
        R, B = saved["R"], saved["B"]
        Wc = torch.cat([w["agg.final.wv"], query_logit_weights(w, "agg.final", h)], dim=1)
        Vf, Lf = _gemm(y_all.reshape(fe.tp * R, d), Wc, N_logit=h)
        Vf, Lf = Vf.view(fe.tp, R, d), Lf.view(fe.tp, R, h)
        ctx_f = self._combine(Vf, Lf, None, [0], [fe.tp], R)
        out = _gemm(ctx_f[0], w["agg.final.wo"], w["agg.final.bo"], out_f32=True)
        saved.update(y_all=y_all, Vf=Vf, Lf=Lf, ctx_f=ctx_f)
        return out.view(B, 1, s, d)

    def _level0_posV(self):
        """pos @ Wv_n for every level-0 node (x sum(mix) for linear nodes): one batched
        bf16 tensor-core GEMM with fp32 output (K_l0 adds it in bf16)."""
        fe = self.fe
        w = fe.weights
        pre = f"agg.slab{fe.rank}"
        pos = _bfc(w["special.pos"])
        n0 = len(fe.tree.levels[0])
        lin = fe.strategy.agg_layer_kind == "linear"
        Wv = torch.stack([_bfc(w[f"{pre}.l0.g{gi}.{'w' if lin else 'wv'}"]) for gi in range(n0)])
        out = torch.bmm(pos.unsqueeze(0).expand(n0, -1, -1), Wv, out_dtype=torch.float32)
        if lin:
            mixsum = torch.stack([w[f"{pre}.l0.g{gi}.mix"].float().sum() for gi in range(n0)])
            out.mul_(mixsum.view(n0, 1, 1))
        return out                                                       # [n0, S, D]

    def _combine(self, V, L, mix, firsts, gs, R, heads=None):
        n = len(firsts)
        d = V.shape[-1]
        h = heads or self.fe.model.heads
        ctx = torch.empty(n, R, d, device=V.device, dtype=torch.bfloat16)
        ft = self._dev_ints(firsts, torch.int32, V.device)
        gt = self._dev_ints(gs, torch.int32, V.device)
        _lib.call("dchag_combine", n, R, d, h, _lib.ptr(ft), _lib.ptr(gt), max(gs), _lib.ptr(V),
                  R * d, _lib.ptr(L), R * h, _lib.ptr(mix), _lib.ptr(ctx), _lib.stream_handle())
        return ctx

    def _level_forward(self, y_prev, level, li, pre, attn, R):
        w = self.fe.weights
        d, h = self.fe.model.embed, self.fe.model.heads
        nprev = y_prev.shape[0]
        V = torch.empty(nprev, R, d, device=y_prev.device, dtype=torch.bfloat16)
        L = torch.empty(nprev, R, h, device=y_prev.device, dtype=torch.float32) if attn else None
        firsts, acc = [], 0
        for gi, g in enumerate(level):
            firsts.append(acc)
            node = f"{pre}.l{li}.g{gi}"
            A = y_prev[acc:acc + g].reshape(g * R, d)
            if attn:
                Wc = torch.cat([w[f"{node}.wv"], query_logit_weights(w, node, h)], dim=1)
                _gemm(A, Wc, N_logit=h, out=V[acc:acc + g].view(g * R, d),
                      out_l=L[acc:acc + g].view(g * R, h))
            else:
                _gemm(A, w[f"{node}.w"], out=V[acc:acc + g].view(g * R, d))
            acc += g
        mix = None if attn else torch.cat([w[f"{pre}.l{li}.g{gi}.mix"]
                                           for gi in range(len(level))]).float().contiguous()
        ctx = self._combine(V, L, mix, firsts, list(level), R)
        y = torch.empty(len(level), R, d, device=y_prev.device, dtype=torch.bfloat16)
        for gi in range(len(level)):
            node = f"{pre}.l{li}.g{gi}"
            if attn:
                _gemm(ctx[gi], w[f"{node}.wo"], w[f"{node}.bo"], out=y[gi])
            else:
                torch.add(ctx[gi], w[f"{node}.b"], out=y[gi])
        return V, L, ctx, y

    # ---------------------------------------------------------------- backward
    def _combine_bwd(self, V, L, mix, G, firsts, gs, R, heads=None):
        """-> gV bf16 (V's shape), dL fp32 (attention) or dm fp32 [child, R] (linear)."""
        n = len(firsts)
        nch = V.shape[0]
        d = V.shape[-1]
        h = heads or self.fe.model.heads
        gV = torch.empty_like(V)
        dL = torch.empty(nch, R, h, device=V.device, dtype=torch.float32) if mix is None else None
        dm = torch.empty(nch, R, device=V.device, dtype=torch.float32) if mix is not None else None
        ft = self._dev_ints(firsts, torch.int32, V.device)
        gt = self._dev_ints(gs, torch.int32, V.device)
        _lib.call("dchag_combine_bwd", n, R, d, h, _lib.ptr(ft), _lib.ptr(gt), max(gs),
                  _lib.ptr(V), R * d, _lib.ptr(L), R * h, _lib.ptr(mix), _lib.ptr(_f32(G)),
                  _lib.ptr(dL), _lib.ptr(gV), _lib.ptr(dm), _lib.stream_handle())
        return gV, dL, dm

    def backward(self, saved, g_out):
        """Gradients of sum(out * g_out) w.r.t. this rank's parameters (reference names):
        the slab's tok.* / channel_id rows, its agg.slab{r}.*, the replicated agg.final.*,
        and special.pos all-reduced over the tp group."""
        _BF_WEIGHTS.clear()
        _BF_WEIGHTS.update(id(v) for v in self.fe.weights.values())
        grads, g_y = self.backward_final(saved, g_out)
        grads.update(self.backward_local(saved, g_y))
        if self.dp_group is not None:
            self._dp_average(grads)
        if self.fe.tp > 1:
            comm.all_reduce(grads["special.pos"], group=self.fe.process_group)
            self.fe._log("AllReduce", "optimizer", "shared-grad.special.pos",
                         (grads["special.pos"].numel(), grads["special.pos"].element_size()))
        return grads

    def _dp_average(self, grads):
        """Data-parallel gradient averaging (strategies.py:352-357: every gradient
        all-reduced over dp, x 1/dp), as ONE bucketed NCCL all-reduce of all gradients in
        name order instead of one call per tensor; the ledger records the reference's
        per-parameter events. special.pos is averaged here and summed over tp after."""
        import torch.distributed as dist
        ndp = dist.get_world_size(self.dp_group)
        if ndp == 1:
            return
        names = sorted(grads)
        flat = torch.cat([grads[k].reshape(-1).float() for k in names])
        comm.all_reduce(flat, group=self.dp_group)
        flat.mul_(1.0 / ndp)
        off = 0
        led = self.fe.ledger
        from . import ledger as LG
        for k in names:
            n = grads[k].numel()
            grads[k] = flat[off:off + n].view(grads[k].shape)
            off += n
            if led is not None:
                led.record(self.fe.rank, "AllReduce", "dp", "backward",
                           LG.allreduce_payload(n, 4, ndp), LG.DP_GRAD_TAG + k)

    def _own_heads(self):
        fe = self.fe
        h, d = fe.model.heads, fe.model.embed
        hc = h // fe.tp
        dh = d // h
        h0 = fe.rank * hc
        return h0, hc, slice(h0 * dh, (h0 + hc) * dh), slice(h0, h0 + hc)

    def _forward_final_split(self, y_all, saved):
        """final_layer_tp_split (strategies.py:211-215): this rank projects the gathered
        streams onto its own heads only (wv / wk / wq column shards, params.py:166-177),
        combines them, and its partial ctx_own @ wo[own rows] is summed over the tp group
        (TpHooks.allsum = ReduceScatter + AllGather; one all-reduce), bo added once."""
        fe = self.fe
        w = fe.weights
        d, h, s = fe.model.embed, fe.model.heads, fe.seq
        R, B = saved["R"], saved["B"]
        _, hc, cols, hs = self._own_heads()
        U = query_logit_weights(w, "agg.final", h)
        Wc = torch.cat([w["agg.final.wv"][:, cols], U[:, hs]], dim=1)
        dl = cols.stop - cols.start
        Vf, Lf = _gemm(y_all.reshape(fe.tp * R, d), Wc, N_logit=hc)
        Vf, Lf = Vf.view(fe.tp, R, dl), Lf.view(fe.tp, R, hc)
        ctx_f = self._combine(Vf, Lf, None, [0], [fe.tp], R, heads=hc)
        bo = w["agg.final.bo"] if fe.rank == 0 else torch.zeros_like(w["agg.final.bo"])
        out = _gemm(ctx_f[0], w["agg.final.wo"][cols], bo, out_f32=True)
        comm.all_reduce(out, group=fe.process_group)
        fe._log("AllReduce", "forward", "agg-final", (out.numel(), out.element_size()))
        saved.update(y_all=y_all, Vf=Vf, Lf=Lf, ctx_f=ctx_f)
        return out.view(B, 1, s, d)

    def _backward_final_split(self, saved, g_out):
        """Backward of the head-split final layer: shard grads (wv/wk/wq columns, wo rows of
        the own heads; bo and the fanned-out q in full), and the root-stream gradient by a
        ReduceScatter of every rank's partial gathered-stream gradient along the stream axis
        (the fused TpHooks.fanout RS + AG and gather slice, strategies.py:54-67, :91-94)."""
        fe = self.fe
        w = fe.weights
        d, h = fe.model.embed, fe.model.heads
        R = saved["R"]
        _, hc, cols, hs = self._own_heads()
        grads = {}
        g_out = _f32(g_out.reshape(R, d))
        ctx_f = saved["ctx_f"][0].float()
        grads["agg.final.bo"] = g_out.sum(0)
        grads["agg.final.wo"] = _mm(ctx_f.t(), g_out)                      # own rows
        g_ctx = _mm(g_out, w["agg.final.wo"][cols].t()).view(1, R, -1)
        gV, dL, _ = self._combine_bwd(saved["Vf"], saved["Lf"], None, g_ctx, [0], [fe.tp], R,
                                      heads=hc)
        y_all = saved["y_all"].reshape(fe.tp * R, d)
        grads["agg.final.wv"] = _mm(y_all.t(), gV.reshape(fe.tp * R, -1))  # own columns
        dU = torch.zeros(d, h, device=g_out.device, dtype=torch.float32)
        dU[:, hs] = _mm(y_all.t(), dL.reshape(fe.tp * R, hc))
        gu = _u_backward(w, "agg.final", dU, h)
        grads["agg.final.wk"] = gu["agg.final.wk"][:, cols].contiguous()
        grads["agg.final.wq"] = gu["agg.final.wq"][:, cols].contiguous()
        q_grad = gu["agg.final.q"].contiguous()
        comm.all_reduce(q_grad, group=fe.process_group)                   # fanout of q
        fe._log("AllReduce", "backward", "agg-final", (q_grad.numel(), q_grad.element_size()))
        grads["agg.final.q"] = q_grad
        U_own = query_logit_weights(w, "agg.final", h)[:, hs]
        g_part = (_mm(gV, w["agg.final.wv"][:, cols].t()) +
                  dL @ U_own.t()).contiguous()                            # [tp, R, D]
        g_y = torch.empty(R, d, device=g_out.device, dtype=torch.float32)
        comm.reduce_scatter_tensor(g_y, g_part.view(fe.tp * R, d), group=fe.process_group)
        fe._log("ReduceScatter", "backward", "agg-final", g_y.numel() * g_y.element_size())
        return grads, g_y.view(1, R, d)

    def backward_final(self, saved, g_out):
        """Final-layer grads (identical on every rank) and this rank's root-stream gradient
        (the local slice of the gathered gradient, strategies.py:91-94)."""
        fe = self.fe
        if fe.strategy.final_layer_tp_split and fe.tp > 1:
            return self._backward_final_split(saved, g_out)
        w = fe.weights
        d, h = fe.model.embed, fe.model.heads
        R = saved["R"]
        grads = {}
        g_out = _f32(g_out.reshape(R, d))
        # ---- final layer (replicated)
        ctx_f = saved["ctx_f"][0].float()
        grads["agg.final.bo"] = g_out.sum(0)
        grads["agg.final.wo"] = _mm(ctx_f.t(), g_out)
        g_ctx = _mm(g_out, w["agg.final.wo"].t()).view(1, R, d)
        gV, dL, _ = self._combine_bwd(saved["Vf"], saved["Lf"], None, g_ctx, [0], [fe.tp], R)
        y_all = saved["y_all"].reshape(fe.tp * R, d)
        grads["agg.final.wv"] = _mm(y_all.t(), gV.reshape(fe.tp * R, d))
        dU = _mm(y_all.t(), dL.reshape(fe.tp * R, h))
        grads.update(_u_backward(w, "agg.final", dU, h))
        U_f = query_logit_weights(w, "agg.final", h)
        # local slice of the gathered gradient (strategies.py:91-94): no collective
        g_y = (_mm(gV[fe.rank], w["agg.final.wv"].t()) + _mm(dL[fe.rank], U_f.t())).view(1, R, d)
        return grads, g_y

    def backward_local(self, saved, g_y):
        """Slab-tree and tokenizer grads from this rank's root-stream gradient g_y [1,R,D];
        special.pos is this rank's partial (summed over tp by backward())."""
        fe = self.fe
        m = fe.model
        w = fe.weights
        d, h, s, P = m.embed, m.heads, fe.seq, m.patch
        R, B = saved["R"], saved["B"]
        levels = fe.tree.levels
        pre = f"agg.slab{fe.rank}"
        attn = fe.strategy.agg_layer_kind != "linear"
        grads = {}
        # ---- levels >= 1, top down
        for li in range(len(levels) - 1, 0, -1):
            level = levels[li]
            ctx = saved["ctx"][li]
            V, L = saved["VL"][li - 1]
            y_prev = saved["y"][li - 1]
            G = torch.empty(len(level), R, d, device=g_y.device, dtype=torch.float32)
            for gi in range(len(level)):
                node = f"{pre}.l{li}.g{gi}"
                if attn:
                    grads[f"{node}.bo"] = g_y[gi].sum(0, dtype=torch.float32)
                    grads[f"{node}.wo"] = _mm(ctx[gi].t(), g_y[gi])
                    torch.mm(_bfc(g_y[gi]), _bfc(w[f"{node}.wo"]).t(), out_dtype=torch.float32,
                             out=G[gi])
                else:
                    grads[f"{node}.b"] = g_y[gi].sum(0, dtype=torch.float32)
                    G[gi] = g_y[gi]
            firsts, acc = [], 0
            for g in level:
                firsts.append(acc)
                acc += g
            mix = None if attn else torch.cat([w[f"{pre}.l{li}.g{gi}.mix"]
                                               for gi in range(len(level))]).float().contiguous()
            gV, dL, dm = self._combine_bwd(V, L, mix, G, firsts, list(level), R)
            # bf16 stream gradient (the operand every consumer GEMM takes), written in place:
            # g_prev = dl U^T, then += gV wv^T (cuBLAS, fp32 accumulation)
            g_prev = torch.empty(y_prev.shape, device=g_y.device, dtype=torch.bfloat16)
            for gi, (f0, g) in enumerate(zip(firsts, level)):
                node = f"{pre}.l{li}.g{gi}"
                Y = y_prev[f0:f0 + g].reshape(g * R, d)
                gv = gV[f0:f0 + g].reshape(g * R, d)
                if attn:
                    dl = dL[f0:f0 + g].reshape(g * R, h)
                    grads[f"{node}.wv"] = _mm(Y.t(), gv)
                    grads.update(_u_backward(w, node, _mm(Y.t(), dl), h))
                    U = query_logit_weights(w, node, h)
                    gp = g_prev[f0:f0 + g].view(g * R, d)
                    torch.mm(dl.to(torch.bfloat16), _bfc(U).t(), out=gp)
                    gp.addmm_(gv, _bfc(w[f"{node}.wv"]).t())
                else:
                    grads[f"{node}.w"] = _mm(Y.t(), gv)
                    grads[f"{node}.mix"] = dm[f0:f0 + g].sum(1)
                    torch.mm(gv, _bfc(w[f"{node}.w"]).t(), out=g_prev[f0:f0 + g].view(g * R, d))
            g_y = g_prev
        # ---- level 0, folded: tokens are never formed (their gradient neither). With
        # x_c = patch_c W_c + b_c + pos (model.py:51-64) and V_c = x_c wv, per node:
        #   V_c = patch_c (W_c wv) + b_c wv + pos wv     (K = P^2 GEMM per channel, tcgen05)
        #   dV_c = p_c * G (per head),  dp_c = G . V_c (per head),  dl_c = p_c (dp_c - G . ctx)
        #   T_c = patch_c^T dV_c  (P^2 x D),  E_c = patch_c^T dl_c  (P^2 x H)
        #   d wv = sum_c W_c^T T_c + b_c^T colsum(dV_c) + pos^T sum_b G
        #   d U  = sum_c W_c^T E_c + b_c^T colsum(dl_c)               (sum_c dl_c = 0)
        #   d W_c = T_c wv^T + E_c U^T,  d b_c = colsum(dV_c) wv^T + colsum(dl_c) U^T
        #   d pos[s] = sum_b G[b, s] wv^T
        # (linear nodes: p_c = mix_c, no dl, d mix_c = sum_r G . V_c)
        off, cnt = fe.slab
        img = saved["img"]
        ctx0 = saved["ctx"][0]
        pos = w["special.pos"]
        tokw = w["tok.w"][off:off + cnt]                                # [cnt, PP, D]
        tb = (w["tok.b"] + w["special.channel_id"])[off:off + cnt]      # [cnt, D]
        pp = P * P
        d_tokw = torch.zeros_like(tokw)
        d_tb = torch.zeros_like(tb)
        patches = torch.empty(B, cnt, s, pp, device=img.device, dtype=torch.bfloat16)
        _lib.call("dchag_unfold", _lib.ptr(img), img.stride(0), img.stride(1), B, cnt, m.image_h,
                  m.image_w, P, _lib.ptr(patches), _lib.stream_handle())
        pk = fe.prepare()
        pnorm = None
        if attn:  # normalised level-0 softmax (K_p0, no pinv), layout [node][hg][g][R][NH]
            poff, acc = [], 0
            for g in pk.l0_g_list:
                poff.append(acc)
                acc += g * R * h
            poff_t = self._dev_ints(poff, torch.int64, img.device)
            pnorm = torch.empty(acc, device=img.device, dtype=torch.bfloat16)
            _lib.call("dchag_l0_logits", _lib.ptr(img), img.stride(0), img.stride(1), B,
                      m.image_h, m.image_w, P, h, pk.HP, pk.NH, pk.n0, max(pk.l0_g_list),
                      _lib.ptr(pk.l0_c0), _lib.ptr(pk.l0_g), _lib.ptr(poff_t), _lib.ptr(pk.WUt),
                      _lib.ptr(pk.bU), _lib.ptr(pk.posU), _lib.ptr(pnorm), 0,
                      _lib.stream_handle())
        dh = d // h
        n0 = len(levels[0])
        wname = "wv" if attn else "w"
        # positional terms of every node at once (batched tensor-core GEMMs):
        # posV_n = pos Wv_n, and after the loop d pos = sum_n Gs_n Wv_n^T, d Wv_n += pos^T Gs_n
        Wv_all = torch.stack([_bfc(w[f"{pre}.l0.g{gi}.{wname}"]) for gi in range(n0)])
        pos_bf = _bfc(pos)
        posV_all = torch.bmm(pos_bf.unsqueeze(0).expand(n0, s, d), Wv_all,
                             out_dtype=torch.float32)                        # [n0, S, D]
        Gs_all = torch.empty(n0, s, d, device=img.device, dtype=torch.float32)
        use_tg = (pp == 64 and d % 128 == 0 and s % 64 == 0 and d // h in (64, 128)
                  and (not attn or pk.NH % 2 == 0)
                  and os.environ.get("DCHAG_TRAIN_TG", "1") != "0")
        c0, p_at = 0, 0
        for gi, g in enumerate(levels[0]):
            node = f"{pre}.l0.g{gi}"
            Wv = w[f"{node}.{wname}"]
            gyb = _bfc(g_y[gi])
            if attn:
                grads[f"{node}.bo"] = g_y[gi].sum(0, dtype=torch.float32)
                grads[f"{node}.wo"] = _mm(ctx0[gi].t(), gyb)
                Gb = torch.mm(gyb, _bfc(w[f"{node}.wo"]).t())            # [R, D] bf16
            else:
                grads[f"{node}.b"] = g_y[gi].sum(0, dtype=torch.float32)
                Gb = gyb
            # positional part of dp: Gpos[r, h] = G[r, h] . posV[s, h] (one pass over G), and
            # T_c = patch_c^T dV_c with dV_c = p_c * G per head: straight from patches, p and
            # G by K_tg (dV never stored) where its shape rules hold, else dV (bf16) + bmm
            Gpos = torch.empty(R, h, device=img.device, dtype=torch.float32)
            if attn:
                pblk = pnorm[p_at:p_at + g * R * h]
                p_at += g * R * h
                pptr, mptr, nh_ = _lib.ptr(pblk), 0, pk.NH
            else:
                mixv = w[f"{node}.mix"].float().contiguous()
                pptr, mptr, nh_ = 0, _lib.ptr(mixv), 1
            if use_tg:
                _lib.call("dchag_l0_dv", g, R, d, h, nh_, pptr, mptr, _lib.ptr(Gb),
                          _lib.ptr(posV_all[gi]), s, _lib.ptr(Gpos), 0, _lib.stream_handle())
                T = torch.empty(g, pp, d, device=img.device, dtype=torch.float32)
                _lib.call("dchag_l0_tgrad", _lib.ptr(patches), cnt, c0, g, R, s, d, h, nh_, pp,
                          pptr, mptr, _lib.ptr(Gb), _lib.ptr(T), _lib.stream_handle())
            else:
                dV = torch.empty(g, R, d, device=img.device, dtype=torch.bfloat16)
                _lib.call("dchag_l0_dv", g, R, d, h, nh_, pptr, mptr, _lib.ptr(Gb),
                          _lib.ptr(posV_all[gi]), s, _lib.ptr(Gpos), _lib.ptr(dV),
                          _lib.stream_handle())
                pt_ = patches[:, c0:c0 + g].permute(1, 3, 0, 2).reshape(g, pp, R)
                T = torch.bmm(pt_, dV, out_dtype=torch.float32)         # [g, PP, D]
            # dp_c[r, h] = G[r, h-cols] . V_c[r, h-cols] with V_c = patch_c Mt_c + Cb_c + posV:
            # the K = P^2 tcgen05 GEMM reduces each 32-column group of V_c against G in its
            # epilogue (V_c never reaches memory)
            Wc = tokw[c0:c0 + g]                                        # [g, PP, D]
            Mt = _bf(_mm(Wc.reshape(g * pp, d), Wv).view(g, pp, d).transpose(1, 2))  # [g, D, PP]
            Cb = _mm(tb[c0:c0 + g], Wv).contiguous()                   # [g, D]
            dpp = torch.empty(g, d // 32, R, device=img.device, dtype=torch.float32)
            A = patches[:, c0:c0 + g]
            _lib.call("dchag_gemm_rowdot", _lib.ptr(A), g, B, s, pp, s * pp, cnt * s * pp, pp,
                      _lib.ptr(Mt), d, d * pp, _lib.ptr(Cb), d, _lib.ptr(Gb), d, _lib.ptr(dpp),
                      _lib.stream_handle())
            if attn:
                pj = pblk.view(h // pk.NH, g, R, pk.NH).permute(1, 0, 3, 2).reshape(g, h, R)
                # softmax backward over the node's channels, one kernel:
                # dp = sum of the 32-column partials + Gpos, dl = p (dp - sum_c p dp)
                dlT = torch.empty(g, h, R, device=img.device, dtype=torch.float32)
                dlTb = torch.empty(g, h, R, device=img.device, dtype=torch.bfloat16)
                _lib.call("dchag_l0_softmax_bwd", g, R, h, pk.NH, dh, _lib.ptr(dpp),
                          _lib.ptr(Gpos), _lib.ptr(pblk), _lib.ptr(dlT), _lib.ptr(dlTb),
                          _lib.stream_handle())
            else:
                dp = dpp.view(g, h, dh // 32, R).sum(2) + Gpos.t().unsqueeze(0)   # [g, H, R]
                grads[f"{node}.mix"] = dp.sum((1, 2))
            pt = patches[:, c0:c0 + g].permute(1, 3, 0, 2).reshape(g, pp, R)   # patch_c^T
            if attn:  # colsum_r dV_j = sum_r p_jrh G_r (per head): a small GEMM, not a dV pass
                colV = torch.bmm(pj.permute(1, 0, 2), Gb.view(R, h, dh).permute(1, 0, 2),
                                 out_dtype=torch.float32)
                colV = colV.permute(1, 0, 2).reshape(g, d)             # [g, D]
            else:
                colV = w[f"{node}.mix"].float().view(g, 1) * Gb.sum(0, dtype=torch.float32).view(1, d)
            dWv = _mm(Wc.reshape(g * pp, d).t(), T.reshape(g * pp, d)) + _mm(tb[c0:c0 + g].t(), colV)
            d_tokw[c0:c0 + g] = _mm(T.reshape(g * pp, d), Wv.t()).view(g, pp, d)
            d_tb[c0:c0 + g] = _mm(colV, Wv.t())
            if attn:
                U = query_logit_weights(w, node, h)
                E = torch.bmm(pt, dlTb.transpose(1, 2), out_dtype=torch.float32)  # [g, PP, H]
                coll = dlT.sum(2)                                       # [g, H]
                dU = _mm(Wc.reshape(g * pp, d).t(), E.reshape(g * pp, h)) + _mm(tb[c0:c0 + g].t(), coll)
                grads.update(_u_backward(w, node, dU, h))
                d_tokw[c0:c0 + g] += _mm(E.reshape(g * pp, h), U.t()).view(g, pp, d)
                d_tb[c0:c0 + g] += _mm(coll, U.t())
            # positional term: sum_c dV_c = G (attention, sum_c p = 1) or (sum_c mix_c) G
            Gs = Gs_all[gi]
            torch.sum(Gb.view(B, s, d), 0, dtype=torch.float32, out=Gs)
            if not attn:
                Gs.mul_(w[f"{node}.mix"].float().sum())
            grads[f"{node}.{wname}"] = dWv
            c0 += g
        Gs_bf = Gs_all.to(torch.bfloat16)
        d_pos = torch.bmm(Gs_bf, Wv_all.transpose(1, 2), out_dtype=torch.float32).sum(0)
        dWv_pos = torch.bmm(pos_bf.t().unsqueeze(0).expand(n0, d, s), Gs_bf,
                            out_dtype=torch.float32)                    # [n0, D, D]
        for gi in range(n0):
            grads[f"{pre}.l0.g{gi}.{wname}"] += dWv_pos[gi]
        grads["tok.w"] = d_tokw
        grads["tok.b"] = d_tb
        grads["special.channel_id"] = d_tb.clone()
        grads["special.pos"] = d_pos  # partial; backward() all-reduces it (strategies.py:251-264)
        return grads

    def _tokens(self, patches, c0, g, B):
        """tokens[c][b*S + s] for slab channels c0..c0+g (tok.w @ patch + tok.b + chan_id + pos)."""
        fe = self.fe
        w = fe.weights
        off = fe.slab[0]
        d, s, pp = fe.model.embed, fe.seq, fe.model.patch ** 2
        C = patches.shape[1]
        Wt = _bf(w["tok.w"][off + c0:off + c0 + g].transpose(1, 2))        # [g, D, PP]
        bias = _f32((w["tok.b"] + w["special.channel_id"])[off + c0:off + c0 + g])
        rb = _bf(w["special.pos"])
        X = torch.empty(g, B * s, d, device=patches.device, dtype=torch.bfloat16)
        A = patches[:, c0:c0 + g]
        _lib.call("dchag_gemm_bf16", _lib.ptr(A), g, B, s, pp, s * pp, C * s * pp, pp, _lib.ptr(Wt),
                  d, d * pp, d, _lib.ptr(bias), d, _lib.ptr(rb), 0, d, s, _lib.ptr(X), 0,
                  B * s * d, s * d, d, 0, 0, 0, 0, _lib.stream_handle())
        return X


class GraphedStep:
    """A captured training step (DchagTrainer.capture)."""

    def __init__(self, graph, out, grads, launches):
        self.graph, self.out, self.grads, self.launches = graph, out, grads, launches

    def replay(self):
        self.graph.replay()
        _lib.LAUNCH_COUNT["n"] += self.launches
        return self.grads
