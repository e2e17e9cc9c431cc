"""Training step of a full_cross D-CHAG front end (agg_variant="full_cross").

Reference semantics: `T.backward` through full_cross nodes (layers.py:125-138 with
sdp_attention :49-64, tensor.py:395-413), the tokenizer (model.py:51-64), the AllGather's
local-slice backward (strategies.py:91-94) and the special.pos all-reduce
(strategies.py:251-264), as DchagTrainer does for single_query / linear trees.

Each node runs as in the forward mirror (ops._full_cross_tree): one projection GEMM to
[q | k | v | u] (u_jh = v_j,h . a_h with a = wo rq / sqrt(D): the rq reduce's scores are
linear in the node's outputs), the channel-attention weights (dchag_fullcross_weights),
the weighted value sum, and y = ctx wo + bo. The backward of the channel attention is one
kernel per (node, row) (dchag_fullcross_bwd: S, p2 and w recomputed on the tensor cores,
then dq, dk, dv and the row's contribution to d a); every matrix product is
dchag_gemm_nt / K_gemm:
  d bo = colsum(g_y), d wo = ctx^T g_y + (d a) rq^T / sqrt(D), G = g_y wo^T,
  d [wq | wk | wv] = x^T [dq | dk | dv],  d x = [dq | dk | dv] [wq | wk | wv]^T,
  d rq = wo^T d a / sqrt(D),
and at level 0 the tokenizer: d tok.w[c] = patch_c^T d x_c, d tok.b = d chan_id =
colsum(d x_c), d pos = sum over channels and images of d x (period S).
The tokens are materialised here (full_cross training is correctness-first; the forward's
folded level 0 is ops.full_cross_level0).
"""

from __future__ import annotations

import torch

from . import _lib, comm, ops
from .config import ConfigError
from .gemm import matmul


def _ptr(t):
    return int(t.data_ptr())


class FullCrossTrainer:
    """Forward + backward of one rank's full_cross front end."""

    def __init__(self, fe, dp_group=None):
        if fe.model.agg_variant != "full_cross" or fe.strategy.agg_layer_kind == "linear":
            raise ConfigError("FullCrossTrainer trains cross_attention nodes with "
                              "agg_variant='full_cross'")
        if fe.strategy.final_layer_tp_split and fe.tp > 1:
            raise ConfigError("full_cross training implements the replicated final layer")
        if max(max(lv) for lv in fe.tree.levels) > 16 or fe.tp > 16:
            raise ConfigError("full_cross training supports nodes of <= 16 inputs")
        if dp_group is not None:
            raise ConfigError("full_cross training: data-parallel averaging not implemented")
        self.fe = fe
        self.dp_group = dp_group
        self._ints = {}

    def _i32(self, vals):
        key = tuple(int(v) for v in vals)
        t = self._ints.get(key)
        if t is None:
            t = self._ints[key] = torch.tensor(key, device=self.fe.device, dtype=torch.int32)
        return t

    # ------------------------------------------------------------------ forward
    def _node_weights(self, node):
        """bf16 operands of one node from the current fp32 weights."""
        w = self.fe.weights
        D, H = self.fe.model.embed, self.fe.model.heads
        dh = D // H
        a = (w[f"{node}.wo"] @ w[f"{node}.rq"]) / (D ** 0.5)                  # [D]
        Wu = (w[f"{node}.wv"].view(D, H, dh) * a.view(1, H, dh)).sum(-1)      # [D, H]
        Wcat = torch.cat([w[f"{node}.wq"], w[f"{node}.wk"], w[f"{node}.wv"]], dim=1)
        Wt = torch.cat([Wcat, Wu], dim=1).t().to(torch.bfloat16).contiguous()  # [3D+H, D]
        return {"Wt": Wt, "Wcat": Wcat.to(torch.bfloat16).contiguous(), "a": a.contiguous(),
                "wo": w[f"{node}.wo"].to(torch.bfloat16).contiguous(),
                "bo": w[f"{node}.bo"].float().contiguous()}

    def _level(self, x, names, groups, R, out_f32=False):
        """One level of full_cross nodes over node-major inputs x [n_in, R, D]."""
        D, H = self.fe.model.embed, self.fe.model.heads
        n_in = x.shape[0]
        dev = x.device
        QKV = torch.empty(n_in, R, 3 * D, device=dev, dtype=torch.bfloat16)
        U = torch.empty(n_in, R, H, device=dev)
        nw = [self._node_weights(nm) for nm in names]
        firsts, acc = [], 0
        for g in groups:
            firsts.append(acc)
            acc += g
        zero = torch.zeros(3 * D + H, device=dev)
        for k, (f, g) in enumerate(zip(firsts, groups)):
            N = 3 * D + H
            _lib.call("dchag_gemm_bf16", _ptr(x[f]), 1, 1, g * R, D, g * R * D, 0, D,
                      _ptr(nw[k]["Wt"]), N, N * D, 3 * D, _ptr(zero), N, 0, 0, 0, 1,
                      _ptr(QKV[f]), 0, 0, 0, 3 * D, _ptr(U[f]), 0, 0, H, _lib.stream_handle(),
                      work={"site": "fc:qkvu", "flops": 2 * g * R * D * N})
        ft, gt = self._i32(firsts), self._i32(groups)
        n = len(groups)
        wts = torch.empty(n, R, max(groups), H, device=dev)
        _lib.call("dchag_fullcross_weights", n, R, D, H, _ptr(ft), _ptr(gt), max(groups),
                  _ptr(QKV), R * 3 * D, 3 * D, _ptr(U), R * H, _ptr(wts), 0, 1, 0, 0, 0,
                  _lib.stream_handle(), work={"site": "fc:weights"})
        ctx = torch.empty(n, R, D, device=dev, dtype=torch.bfloat16)
        _lib.call("dchag_combine_weighted", n, R, D, H, _ptr(ft), _ptr(gt), max(groups),
                  _ptr(QKV[:, :, 2 * D:]), R * 3 * D, 3 * D, _ptr(wts), _ptr(ctx),
                  _lib.stream_handle(), work={"site": "fc:combine"})
        y = torch.empty(n, R, D, device=dev,
                        dtype=torch.float32 if out_f32 else torch.bfloat16)
        for k in range(n):
            matmul(ctx[k], nw[k]["wo"], out=y[k], bias=nw[k]["bo"],
                   work={"site": "fc:wo", "flops": 2 * R * D * D})
        return {"x": x, "QKV": QKV, "U": U, "ctx": ctx, "nw": nw, "firsts": firsts,
                "groups": list(groups), "names": names}, y

    def forward_local(self, images):
        fe = self.fe
        m = fe.model
        w = fe.weights
        off, cnt = fe.slab
        if images.shape[1] == m.channels and fe.tp > 1:
            images = images[:, off:off + cnt]
        img = images if images.dtype == torch.bfloat16 else images.to(torch.bfloat16)
        img = img.contiguous()
        B = img.shape[0]
        S, D = fe.seq, m.embed
        R = B * S
        sl = slice(off, off + cnt)
        tok = ops.tokenize_channels(img, w["tok.w"][sl], w["tok.b"][sl],
                                    w["special.channel_id"][sl], w["special.pos"], m.patch,
                                    out_dtype=torch.bfloat16)                 # [B, C, S, D]
        x = tok.permute(1, 0, 2, 3).reshape(cnt, R, D).contiguous()
        saved = {"img": img, "B": B, "R": R, "levels": []}
        pre = f"agg.slab{fe.rank}"
        for li, level in enumerate(fe.tree.levels):
            names = [f"{pre}.l{li}.g{gi}" for gi in range(len(level))]
            lv, x = self._level(x, names, level, R)
            saved["levels"].append(lv)
        saved["y_root"] = x[0]
        return saved

    def forward_train(self, images):
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
        fe = self.fe
        R, B = saved["R"], saved["B"]
        lv, out = self._level(y_all.contiguous(), ["agg.final"], [fe.tp], R, out_f32=True)
        saved["final"] = lv
        return out.view(B, 1, fe.seq, fe.model.embed)

    # ---------------------------------------------------------------- backward
    def _level_backward(self, lv, g_y, R, grads):
        """Grads of one level's nodes from g_y [n, R, D]; returns d x [n_in, R, D] bf16."""
        fe = self.fe
        D, H = fe.model.embed, fe.model.heads
        dev = g_y.device
        n = len(lv["groups"])
        g16 = g_y if g_y.dtype == torch.bfloat16 else g_y.to(torch.bfloat16)
        sh = _lib.stream_handle()
        db = torch.empty(n, D, device=dev)
        work = torch.empty(n * (-(-R // 64)) * D, device=dev)
        _lib.call("dchag_colsum", _ptr(g16), 0, D, R * D, n, R, D, 1, _ptr(db), D, 0, 0, 0, 0,
                  _ptr(work), sh, work={"site": "fc:colsum"})
        G = torch.empty(n, R, D, device=dev)
        a = torch.stack([nw["a"] for nw in lv["nw"]]).contiguous()            # [n, D]
        for k, nw in enumerate(lv["nw"]):
            name = lv["names"][k]
            grads[f"{name}.bo"] = db[k]
            grads[f"{name}.wo"] = matmul(lv["ctx"][k].t(), g16[k],
                                         work={"site": "fc:dwo", "flops": 2 * R * D * D})
            matmul(g16[k], nw["wo"].t(), out=G[k],
                   work={"site": "fc:g", "flops": 2 * R * D * D})
        QKV = lv["QKV"]
        dQKV = torch.empty_like(QKV)
        dA = torch.empty(n, R, D, device=dev)
        ft, gt = self._i32(lv["firsts"]), self._i32(lv["groups"])
        _lib.call("dchag_fullcross_bwd", n, R, D, H, _ptr(ft), _ptr(gt), max(lv["groups"]),
                  _ptr(QKV), R * 3 * D, 3 * D, _ptr(lv["U"]), _ptr(G), _ptr(a), _ptr(dQKV),
                  _ptr(dA), sh, work={"site": "fc:attention_bwd"})
        da = torch.empty(n, D, device=dev)
        _lib.call("dchag_colsum", _ptr(dA), 1, D, R * D, n, R, D, 1, _ptr(da), D, 0, 0, 0, 0,
                  _ptr(work), sh, work={"site": "fc:colsum"})
        w = fe.weights
        x = lv["x"]
        dx = torch.empty(x.shape, device=dev, dtype=torch.bfloat16)
        for k, (f, g) in enumerate(zip(lv["firsts"], lv["groups"])):
            name = lv["names"][k]
            rq, wo = w[f"{name}.rq"], w[f"{name}.wo"]
            # a = wo rq / sqrt(D): d wo += d a rq^T / sqrt(D), d rq = wo^T d a / sqrt(D)
            grads[f"{name}.wo"] = grads[f"{name}.wo"] + torch.outer(da[k], rq) / (D ** 0.5)
            grads[f"{name}.rq"] = (wo.t() @ da[k]) / (D ** 0.5)
            X = x[f:f + g].reshape(g * R, D)
            dq = dQKV[f:f + g].reshape(g * R, 3 * D)
            dW = matmul(X.t(), dq, work={"site": "fc:dw", "flops": 2 * g * R * D * 3 * D})
            grads[f"{name}.wq"] = dW[:, :D]
            grads[f"{name}.wk"] = dW[:, D:2 * D]
            grads[f"{name}.wv"] = dW[:, 2 * D:]
            matmul(dq, lv["nw"][k]["Wcat"].t(), out=dx[f:f + g].view(g * R, D),
                   work={"site": "fc:dx", "flops": 2 * g * R * 3 * D * D})
        return dx

    def backward_final(self, saved, g_out):
        fe = self.fe
        R = saved["R"]
        grads = {}
        g = g_out.reshape(1, R, fe.model.embed).float().to(torch.bfloat16)
        d_all = self._level_backward(saved["final"], g, R, grads)          # [tp, R, D]
        return grads, d_all[fe.rank].unsqueeze(0)                          # local slice

    def backward_local(self, saved, g_y):
        fe = self.fe
        m = fe.model
        R, B = saved["R"], saved["B"]
        D, S, P = m.embed, fe.seq, m.patch
        PP = P * P
        grads = {}
        for lv in reversed(saved["levels"]):
            g_y = self._level_backward(lv, g_y, R, grads)
        # tokenizer (model.py:51-64): d tok.w[c] = patch_c^T dx_c, d tb = colsum, d pos
        img = saved["img"]
        cnt = img.shape[1]
        dev = img.device
        patches = torch.empty(B, cnt, S, PP, device=dev, dtype=torch.bfloat16)
        _lib.call("dchag_unfold", _ptr(img), img.stride(0), img.stride(1), B, cnt, m.image_h,
                  m.image_w, P, _ptr(patches), _lib.stream_handle(), work={"site": "fc:unfold"})
        pn = patches.permute(1, 0, 2, 3).reshape(cnt, R, PP)
        grads["tok.w"] = matmul(pn.transpose(1, 2), g_y,
                                work={"site": "fc:dtokw", "flops": 2 * cnt * R * PP * D})
        dtb = torch.empty(cnt, D, device=dev)
        work = torch.empty(cnt * (-(-R // 64)) * D, device=dev)
        _lib.call("dchag_colsum", _ptr(g_y), 0, D, R * D, cnt, R, D, 1, _ptr(dtb), D, 0, 0, 0,
                  0, _ptr(work), _lib.stream_handle(), work={"site": "fc:colsum"})
        grads["tok.b"] = dtb
        grads["special.channel_id"] = dtb.clone()
        dpos = torch.empty(S, D, device=dev)
        _lib.call("dchag_colsum", _ptr(g_y), 0, D, 0, 1, cnt * R, D, S, _ptr(dpos), 0, 0, 0, 0,
                  0, 0, _lib.stream_handle(), work={"site": "fc:colsum"})
        grads["special.pos"] = dpos
        return grads

    def backward(self, saved, g_out):
        grads, g_y = self.backward_final(saved, g_out)
        grads.update(self.backward_local(saved, g_y))
        if self.fe.tp > 1:
            comm.all_reduce(grads["special.pos"], group=self.fe.process_group)
            self.fe._log("AllReduce", "optimizer", "shared-grad.special.pos",
                         (grads["special.pos"].numel(), grads["special.pos"].element_size()))
        return grads
