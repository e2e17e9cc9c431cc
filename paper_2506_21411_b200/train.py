"""Training step of the D-CHAG front end: forward with saved activations + backward, every
matrix product on the repo's tcgen05 GEMMs.

Reference semantics: `T.backward` over the hot path of forward_loss_dchag_reference /
dchag_forward_loss (model.py:180-201, strategies.py:195-218, tensor.py:395-413), gather
backward = local slice (strategies.py:91-94), the special.pos gradient all-reduced over the
channel group (strategies.py:251-264), and the head-split final layer's TpHooks
(strategies.py:48-80).

One step = prep + forward + backward, all stream-ordered (CUDA-graph capturable):

prep      the fp32 master weights become the step's bf16 operands in ONE launch
          (dchag_cast_multi), the single_query query folds U = fold(wq, wk, q) run batched
          (dchag_query_fold), and level 0 is refolded from the current weights: one grouped
          GEMM MT_n = [Wv_n | U_n]^T x [tok.w rows ; tok.b + chan_id rows]^T for every
          level-0 node (fold.py's algebra) + one for pos [Wv_n | U_n], scattered into the
          K_p0 / K_l0 / row-dot operand layouts (dchag_l0_pack).
forward   K_p0 + K_l0 (level 0: tokens never formed), then per level the node projections
          y = ctx wo + bo (grouped GEMM) and, above level 0, V | L = y [wv | U] (K_gemm with
          the logit columns split) + softmax-weighted combine; the root streams are
          all-gathered in rank order and the final layer runs replicated (or head-split).
backward  per level, top down (grouped over the level's nodes where shapes agree):
            d bo = colsum(g_y), d wo = ctx^T g_y, G = g_y wo^T
            combine backward -> [gV | dL] (one bf16 operand, dchag_combine_bwd_packed)
            [d wv | d U] = y^T [gV | dL],  g_prev = [gV | dL] [wv | U]^T   (K-concatenated)
          level 0 in the augmented-token form x_c = [patch_c | 1] [tok.w[c] ; tb_c]:
            G = g_y wo^T, the positional dp (dchag_l0_dv), dp = G . V_c by the row-dot GEMM,
            the channel-softmax backward, then ONE kernel per node gives
            TE = [patch | 1]^T [p G | dl] (dchag_l0_tgrad_te) and two grouped GEMMs finish:
              [d Wv | d U] = [tok.w ; tb ; pos]^T [TE ; Gs],  d [tok.w ; tb ; pos] = [TE ; Gs] [Wv | U]^T
          and d wk / d wq / d q from d U (dchag_query_fold_bwd, batched over every node).
"""

from __future__ import annotations

import os

import torch

from . import _lib, comm
from .config import ConfigError
from .fold import unit_heads
from .frontend import DchagFrontEnd
from .gemm import matmul


def _c(x, m):
    return -(-x // m) * m


def _ptr(t):
    return int(t.data_ptr())


class _Node:
    """One attention / linear node of the rank's tree (or the shared final layer)."""

    def __init__(self, k, name, li, gi, g, first):
        self.k, self.name, self.li, self.gi, self.g, self.first = k, name, li, gi, g, first


class DchagTrainer:
    """Forward + backward of one rank's front end (tp ranks share the final layer).
    A full_cross front end gets its own trainer (train_fc.FullCrossTrainer)."""

    def __new__(cls, fe: DchagFrontEnd, dp_group=None):
        if cls is DchagTrainer and fe.model.agg_variant == "full_cross":
            from .train_fc import FullCrossTrainer
            return FullCrossTrainer(fe, dp_group)
        return super().__new__(cls)

    def __init__(self, fe: DchagFrontEnd, dp_group=None):
        """dp_group: the data-parallel group of this rank (grid.make_groups); backward()
        then averages every gradient over it (strategies.py:352-357)."""
        if fe.model.agg_variant != "single_query":
            raise ConfigError("training path implements agg_variant='single_query'")
        self.fe = fe
        self.dp_group = dp_group
        self._ints = {}
        self._st = None          # static plan + persistent buffers (built on first use)
        self._wsig = None        # weight tensors the device tables point at

    # ------------------------------------------------------------------ setup
    def _dev_ints(self, vals, dtype, dev):
        """Small host-known index arrays on the device, made once (no copies inside a step,
        so the step can be captured in a CUDA graph)."""
        key = (tuple(int(v) for v in vals), dtype, str(dev))
        t = self._ints.get(key)
        if t is None:
            t = self._ints[key] = torch.tensor(key[0], device=dev, dtype=dtype)
        return t

    def _static(self):
        if self._st is not None:
            return self._st
        fe = self.fe
        m = fe.model
        dev = fe.device
        D, H, S, P = m.embed, m.heads, fe.seq, m.patch
        PP = P * P
        attn = fe.strategy.agg_layer_kind != "linear"
        levels = fe.tree.levels
        pre = f"agg.slab{fe.rank}"
        st = {"D": D, "H": H, "S": S, "P": P, "PP": PP, "attn": attn, "dh": D // H,
              "levels": levels, "pre": pre}
        nodes, k = [], 0
        for li, level in enumerate(levels):
            first = 0
            for gi, g in enumerate(level):
                nodes.append(_Node(k, f"{pre}.l{li}.g{gi}", li, gi, g, first))
                first += g
                k += 1
        final = _Node(k, "agg.final", len(levels), 0, fe.tp, 0)
        st["nodes"], st["final"] = nodes, final
        st["lvl"] = [[n for n in nodes if n.li == li] for li in range(len(levels))]
        n0 = len(levels[0])
        C = fe.slab[1]
        gmax = max(levels[0])
        Dp = _c(D + H, 256)                            # [wv | U | 0] width
        ones0 = _c(gmax * PP, 64)                      # first tb row of a level-0 block
        Kn = _c(ones0 + gmax, 128)                     # level-0 block height
        st.update(n0=n0, C=C, gmax=gmax, Dp=Dp, ones0=ones0, Kn=Kn)
        nall = len(nodes) + 1
        bf = dict(device=dev, dtype=torch.bfloat16)
        f32 = dict(device=dev, dtype=torch.float32)
        # persistent operands (zero padding is written once and never touched)
        st["WvU"] = torch.zeros(nall, D, Dp, **bf)       # [wv | U | 0]  (linear: [w | 0])
        st["WvUt"] = torch.zeros(nall, D + H, D, **bf)   # [wv | U]^T (levels >= 1, final)
        st["wo16"] = torch.zeros(nall, D, D, **bf)
        st["bo32"] = torch.zeros(nall, D, **f32)         # bo (linear nodes: b)
        # [tok.w rows ; tb rows ; 0 ; pos rows]: rows Kn.. carry pos, so the level-0 weight
        # gradient GEMMs also give pos^T Gs_n and Gs_n Wv_n^T (the positional terms)
        st["Waug"] = torch.zeros(n0, Kn + S, D, **bf)
        st["pos16"] = torch.zeros(S, D, **bf)
        st["tb32"] = torch.zeros(C, D, **f32)
        st["U"] = torch.zeros(nall, D, H, **f32)
        st["qp"] = torch.zeros(nall, D, **f32)
        st["qf_work"] = torch.zeros(nall, _c(D, 128) // 128, D, **f32)
        st["dqp"] = torch.zeros(nall, D, **f32)
        st["dWvU"] = torch.zeros(nall, D, Dp, **f32)     # [d wv | d U | -] per node
        st["dwk"] = torch.zeros(nall, D, D, **f32)
        st["dwq"] = torch.zeros(nall, D, D, **f32)
        st["dq"] = torch.zeros(nall, D, **f32)
        st["TE"] = torch.zeros(n0, Kn + S, Dp, **bf)      # [T | E ; colV | coll ; 0 ; Gs | 0]
        # level-0 folded operands of K_p0 / K_l0 / the row-dot GEMM
        C_pad = C + 64 // PP
        KE = 16 * ((gmax + 15) // 16)
        HP = 8 * ((H + 7) // 8)
        hw = (D // H) // 2
        st.update(C_pad=C_pad, KE=KE, HP=HP, NH=unit_heads(D, H))
        st["MT"] = torch.zeros(n0, Dp, Kn, **f32)
        st["posVU"] = torch.zeros(n0, S, Dp, **f32)
        st["Mt"] = torch.zeros(H * 2 * C_pad * PP * hw, **bf)
        st["Et"] = torch.zeros(n0 * H * 2 * KE * hw, **bf)
        st["Mrow"] = torch.zeros(C, D, PP, **bf)
        st["Cb"] = torch.zeros(C, D, **f32)
        st["posV0"] = torch.zeros(n0, S, D, **bf)
        if attn:
            st["WUt"] = torch.zeros(C, HP, PP, **bf)
            st["bU"] = torch.zeros(C, HP, **f32)
            st["posU"] = torch.zeros(n0, S, HP, **f32)
        else:
            st["p_const"] = torch.zeros(C, H, **bf)
            st["mixsum"] = torch.zeros(n0, **f32)
        c0s = [0]
        for g in levels[0][:-1]:
            c0s.append(c0s[-1] + g)
        st["c0s"] = c0s
        st["l0_c0"] = self._dev_ints(c0s, torch.int32, dev)
        st["l0_g"] = self._dev_ints(levels[0], torch.int32, dev)
        chan_node, chan_local = [], []
        for n, g in enumerate(levels[0]):
            chan_node += [n] * g
            chan_local += list(range(g))
        st["chan_node"] = self._dev_ints(chan_node, torch.int32, dev)
        st["chan_local"] = self._dev_ints(chan_local, torch.int32, dev)
        # row indices of d tok.w / d tb inside the level-0 blocks
        rows_w = [n * (Kn + S) + l * PP + kk for n, g in enumerate(levels[0]) for l in range(g)
                  for kk in range(PP)]
        rows_b = [n * (Kn + S) + ones0 + l for n, g in enumerate(levels[0]) for l in range(g)]
        st["rows_w"] = torch.tensor(rows_w, device=dev, dtype=torch.int64)
        st["rows_b"] = torch.tensor(rows_b, device=dev, dtype=torch.int64)
        # per-level combine tables
        st["comb"] = {}
        for li in range(1, len(levels)):
            firsts = [n.first for n in st["lvl"][li]]
            gs = [n.g for n in st["lvl"][li]]
            st["comb"][li] = (self._dev_ints(firsts, torch.int32, dev),
                              self._dev_ints(gs, torch.int32, dev), max(gs))
        st["comb"]["final"] = (self._dev_ints([0], torch.int32, dev),
                               self._dev_ints([fe.tp], torch.int32, dev), fe.tp)
        st["zero_b"] = torch.zeros(D + H, **f32)
        self._st = st
        return st

    def _tables(self):
        """Device job tables of the per-step prep (cast + query folds), rebuilt only when the
        module's weight tensors are replaced (an in-place optimizer step keeps them)."""
        fe, st = self.fe, self._static()
        w = fe.weights
        sig = tuple((k, v.data_ptr()) for k, v in w.items())
        if sig == self._wsig:
            return
        D, H, PP, Dp, attn = st["D"], st["H"], st["PP"], st["Dp"], st["attn"]
        jobs = []

        def job(src, dst, rows, cols, lds, ldd, trans=0, f32=0):
            jobs.append([_ptr(src), _ptr(dst), rows, cols, lds, ldd, trans, f32])

        off, C = fe.slab
        fin = st["final"]
        allnodes = st["nodes"] + [fin]
        for nd in allnodes:
            kind_attn = attn or nd is fin
            Wv = w[f"{nd.name}.{'wv' if kind_attn else 'w'}"]
            job(Wv, st["WvU"][nd.k], D, D, D, Dp)
            if kind_attn:
                job(st["U"][nd.k], st["WvU"][nd.k, :, D:], D, H, H, Dp)
                if nd.li >= 1:
                    job(Wv, st["WvUt"][nd.k], D, D, D, D, trans=1)
                    job(st["U"][nd.k], st["WvUt"][nd.k, D:], D, H, H, D, trans=1)
                job(w[f"{nd.name}.wo"], st["wo16"][nd.k], D, D, D, D)
                job(w[f"{nd.name}.bo"], st["bo32"][nd.k], 1, D, D, D, f32=1)
            else:
                job(w[f"{nd.name}.b"], st["bo32"][nd.k], 1, D, D, D, f32=1)
        tokw = w["tok.w"]
        for n, (c0, g) in enumerate(zip(st["c0s"], st["levels"][0])):
            job(tokw[off + c0], st["Waug"][n], g * PP, D, D, D)
            job(st["tb32"][c0], st["Waug"][n, st["ones0"]:], g, D, D, D)
        job(w["special.pos"], st["pos16"], st["S"], D, D, D)
        for n in range(st["n0"]):
            job(w["special.pos"], st["Waug"][n, st["Kn"]:], st["S"], D, D, D)
        if fe.strategy.final_layer_tp_split and fe.tp > 1:
            self._head_split_buffers(job)
        tab = torch.tensor(jobs, dtype=torch.int64).to(fe.device)
        max_tiles = max(((j[2] + 31) // 32) * ((j[3] + 31) // 32) for j in jobs)
        st["cast"] = (tab, len(jobs), max_tiles)
        # query-fold jobs (forward: U with ldU = H; backward: dU = dWvU[:, :, D:], ldU = Dp)
        qnodes = [nd for nd in allnodes if attn or nd is fin]
        qf, qb = [], []
        for nd in qnodes:
            base = [_ptr(w[f"{nd.name}.wq"]), _ptr(w[f"{nd.name}.wk"]), _ptr(w[f"{nd.name}.q"])]
            qf.append(base + [_ptr(st["U"][nd.k]), H, _ptr(st["qp"][nd.k]), 0, 0, 0, 0])
            qb.append(base + [0, Dp, _ptr(st["qp"][nd.k]), _ptr(st["dWvU"][nd.k, :, D:]),
                              _ptr(st["dwk"][nd.k]), _ptr(st["dwq"][nd.k]),
                              _ptr(st["dq"][nd.k])])
        st["qf"] = torch.tensor(qf, dtype=torch.int64).to(fe.device)
        st["qb"] = torch.tensor(qb, dtype=torch.int64).to(fe.device)
        st["qnodes"] = qnodes
        self._wsig = sig

    def _head_split_buffers(self, job):
        """final_layer_tp_split: bf16 operands of this rank's head shard of the final layer."""
        fe, st = self.fe, self._st
        w = fe.weights
        D, H = st["D"], st["H"]
        h0, hc, cols, hs = self._own_heads()
        dl = cols.stop - cols.start
        dpo = _c(dl + hc, 256)
        dev = fe.device
        if "hs_WvUt" not in st:
            st["hs_WvUt"] = torch.zeros(dl + hc, D, device=dev, dtype=torch.bfloat16)
            st["hs_WvU"] = torch.zeros(D, dpo, device=dev, dtype=torch.bfloat16)
            st["hs_dWvU"] = torch.zeros(D, dpo, device=dev)
        k = st["final"].k
        wv = w["agg.final.wv"]
        job(wv[:, cols.start:], st["hs_WvUt"], D, dl, D, D, trans=1)
        job(st["U"][k, :, h0:], st["hs_WvUt"][dl:], D, hc, H, D, trans=1)
        job(wv[:, cols.start:], st["hs_WvU"], D, dl, D, dpo)
        job(st["U"][k, :, h0:], st["hs_WvU"][:, dl:], D, hc, H, dpo)
        st["hs_dp"] = dpo

    # ------------------------------------------------------------------ prep
    def prep(self):
        """Per-step weight preparation from the current fp32 master weights (see module
        docstring): bf16 operands, query folds, level-0 refold. Stream-ordered, no host sync
        after the first call, so it is part of a captured step."""
        fe, st = self.fe, self._static()
        self._tables()
        w = fe.weights
        D, H, Dp, n0, Kn = st["D"], st["H"], st["Dp"], st["n0"], st["Kn"]
        sh = _lib.stream_handle()
        off, C = fe.slab
        torch.add(w["tok.b"][off:off + C], w["special.channel_id"][off:off + C], out=st["tb32"])
        qn = len(st["qnodes"])
        _lib.call("dchag_query_fold", _ptr(st["qf"]), qn, D, H, _ptr(st["qf_work"]), sh,
                  work={"site": "prep:query_fold", "flops": 4 * qn * D * D,
                        "bytes": 8 * qn * D * D})
        tab, nj, mt = st["cast"]
        _lib.call("dchag_cast_multi", _ptr(tab), nj, mt, sh, work={"site": "prep:cast"})
        if not st["attn"]:
            mix = torch.cat([w[f"{nd.name}.mix"] for nd in st["lvl"][0]]).float()
            st["p_const"].copy_(mix.view(C, 1).expand(C, H))
            torch.stack([w[f"{nd.name}.mix"].float().sum() for nd in st["lvl"][0]],
                        out=st["mixsum"])
        # level-0 refold: MT_n = [Wv_n | U_n]^T Waug_n^T  and  pos [Wv_n | U_n]
        matmul(st["WvU"][:n0].transpose(1, 2), st["Waug"][:, :Kn].transpose(1, 2), out=st["MT"],
               work={"site": "prep:l0_fold", "flops": 2 * n0 * Dp * D * Kn})
        matmul(st["pos16"], st["WvU"][:n0], out=st["posVU"],
               work={"site": "prep:l0_fold_pos", "flops": 2 * n0 * st["S"] * D * Dp})
        attn = st["attn"]
        _lib.call("dchag_l0_pack", _ptr(st["MT"]), n0, C, st["C_pad"], D, H, st["HP"], st["PP"],
                  st["gmax"], st["ones0"], st["KE"], st["S"], Dp, Kn, _ptr(st["chan_node"]),
                  _ptr(st["chan_local"]), _ptr(st["l0_g"]), _ptr(st["Mt"]), _ptr(st["Et"]),
                  _ptr(st["Mrow"]), _ptr(st["Cb"]), _ptr(st["WUt"]) if attn else 0,
                  _ptr(st["bU"]) if attn else 0, _ptr(st["posVU"]),
                  0 if attn else _ptr(st["mixsum"]), _ptr(st["posV0"]),
                  _ptr(st["posU"]) if attn else 0, sh,
                  work={"site": "prep:l0_pack", "bytes": 4 * n0 * Dp * Kn})

    def capture(self, images, g_out, warmup: int = 2):
        """One training step (prep + forward_train + backward) captured as a CUDA graph over
        the static buffers `images` / `g_out`: refill them in place and call .replay(). The
        master weights are read by pointer every replay (an in-place optimizer update is
        seen; replacing the weight tensors needs a new capture). Returns a GraphedStep with
        .out, .grads (written by every replay) and .launches (library launches per replay)."""
        if self.fe.tp >= 4 and os.environ.get("NCCL_NVLS_ENABLE", "") != "0":
            raise ConfigError(
                "capturing the training step at tp >= 4 needs NCCL_NVLS_ENABLE=0 set before "
                "init_process_group (DESIGN.md section 7); or run the step eagerly")
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
        with torch.cuda.graph(graph):
            out, saved = self.forward_train(images)
            grads = self.backward(saved, g_out)
        # one completed replay before the graph is handed out: at 4 ranks, first replays
        # issued back to back (collectives inside) hung
        graph.replay()
        torch.cuda.synchronize()
        return GraphedStep(graph, out, grads, _lib.LAUNCH_COUNT["n"] - n0)

    # ---------------------------------------------------------------- forward
    def _proj_logits(self, A, rows, Wt, Nv, Nl, V, L, site, G=1):
        """[V | L] = A W with the K_gemm logit split (bf16 V, fp32 L); Wt = W^T bf16. G > 1:
        G groups of `rows` rows, A / Wt / V / L with consecutive group blocks."""
        D = self._st["D"]
        N = Nv + Nl
        _lib.call("dchag_gemm_bf16", _ptr(A), G, 1, rows, D, rows * D, 0, D, _ptr(Wt), N, N * D,
                  Nv, _ptr(self._st["zero_b"]), 0, 0, 0, 0, 1, _ptr(V), 0, rows * Nv, 0, Nv,
                  _ptr(L), rows * Nl, 0, Nl, _lib.stream_handle(),
                  work={"site": site, "flops": 2 * G * rows * D * N})

    def forward_local(self, images):
        """prep + slab tokenizer + tree of this rank up to its root stream (saved['y_root'])."""
        fe = self.fe
        m = fe.model
        self.prep()
        st = self._st
        D, H, S = st["D"], st["H"], st["S"]
        attn = st["attn"]
        off, cnt = fe.slab
        if images.shape[1] == m.channels and fe.tp > 1:
            images = images[:, off:off + cnt]
        img = images if images.dtype == torch.bfloat16 else images.to(torch.bfloat16)
        if not img.is_contiguous():
            img = img.contiguous()
        B = img.shape[0]
        R = B * S
        n0 = st["n0"]
        saved = {"img": img, "B": B, "R": R}
        dev = img.device
        sh = _lib.stream_handle()
        gl = st["levels"][0]
        if attn:
            poff, acc = [], 0
            for g in gl:
                poff.append(acc)
                acc += g * R * H
            poff_t = self._dev_ints(poff, torch.int64, dev)
            pbuf = torch.empty(acc, device=dev, dtype=torch.bfloat16)
            pinv = torch.empty(n0, R, H, device=dev, dtype=torch.float32)
            _lib.call("dchag_l0_logits", _ptr(img), img.stride(0), img.stride(1), B,
                      m.image_h, m.image_w, m.patch, H, st["HP"], st["NH"], n0, max(gl),
                      _ptr(st["l0_c0"]), _ptr(st["l0_g"]), _ptr(poff_t), _ptr(st["WUt"]),
                      _ptr(st["bU"]), _ptr(st["posU"]), _ptr(pbuf), _ptr(pinv), sh,
                      work={"site": "fwd:l0_logits",
                            "flops": 2 * 2 * R * cnt * st["PP"] * H})
            prow = 1
            saved["poff"] = poff_t
            saved["p_e"], saved["pinv"] = pbuf, pinv  # the backward normalises these
        else:
            poff_t = self._dev_ints([c * H for c in st["c0s"]], torch.int64, dev)
            pbuf, prow, pinv = st["p_const"], 0, None
        ctx0 = torch.empty(n0, R, D, device=dev, dtype=torch.bfloat16)
        _lib.call("dchag_l0_node", _ptr(img), img.stride(0), img.stride(1), B, m.image_h,
                  m.image_w, m.patch, H, D, n0, _ptr(st["l0_c0"]), _ptr(st["l0_g"]),
                  _ptr(poff_t), prow, _ptr(pbuf), _lib.ptr(pinv), _ptr(st["Mt"]), st["C_pad"],
                  _ptr(st["Et"]), st["KE"], _ptr(st["posV0"]), _ptr(ctx0), sh,
                  work={"site": "fwd:l0_node",
                        "flops": 2 * R * D * cnt * (st["PP"] + 1)})
        saved["ctx"] = [ctx0]
        y = self._node_out(ctx0, st["lvl"][0], R)
        saved["y"] = [y]
        saved["VL"] = []
        for li in range(1, len(st["levels"])):
            V, L, ctx, ynext = self._level_forward(y, li, R)
            saved["VL"].append((V, L))
            saved["ctx"].append(ctx)
            saved["y"].append(ynext)
            y = ynext
        saved["y_root"] = y[0]
        return saved

    def _node_out(self, ctx, nodes, R):
        """y = ctx wo + bo for a level's nodes (one grouped GEMM; linear nodes: ctx + b)."""
        st = self._st
        k0, n = nodes[0].k, len(nodes)
        D = st["D"]
        if not st["attn"]:
            return torch.add(ctx, st["bo32"][k0:k0 + n].unsqueeze(1)).to(torch.bfloat16)
        y = torch.empty_like(ctx)
        matmul(ctx, st["wo16"][k0:k0 + n], out=y, bias=st["bo32"][k0:k0 + n],
               work={"site": f"fwd:wo_l{nodes[0].li}", "flops": 2 * n * R * D * D})
        return y

    def _combine(self, V, L, mix, tables, R, heads=None, Dv=None):
        D = Dv or self._st["D"]
        H = heads or self._st["H"]
        ft, gt, gmax = tables
        n = ft.numel()
        ctx = torch.empty(n, R, D, device=V.device, dtype=torch.bfloat16)
        _lib.call("dchag_combine", n, R, D, H, _ptr(ft), _ptr(gt), gmax, _ptr(V), R * D,
                  _lib.ptr(L), R * H, _lib.ptr(mix), _ptr(ctx), _lib.stream_handle(),
                  work={"site": "fwd:combine", "bytes": V.numel() * 2 + ctx.numel() * 2})
        return ctx

    def _mix(self, li):
        w = self.fe.weights
        return torch.cat([w[f"{nd.name}.mix"] for nd in self._st["lvl"][li]]).float()

    def _level_forward(self, y_prev, li, R):
        st = self._st
        D, H = st["D"], st["H"]
        nodes = st["lvl"][li]
        nprev = y_prev.shape[0]
        V = torch.empty(nprev, R, D, device=y_prev.device, dtype=torch.bfloat16)
        L = torch.empty(nprev, R, H, device=y_prev.device) if st["attn"] else None
        uniform = (len({nd.g for nd in nodes}) == 1 and st["attn"]
                   and nodes[-1].first + nodes[-1].g == nprev)
        if uniform:  # equal fan-in: the whole level in one grouped launch
            g, k0 = nodes[0].g, nodes[0].k
            self._proj_logits(y_prev, g * R, st["WvUt"][k0], D, H, V, L, f"fwd:vl_l{li}",
                              G=len(nodes))
        for nd in ([] if uniform else nodes):
            A = y_prev[nd.first:nd.first + nd.g].reshape(nd.g * R, D)
            if st["attn"]:
                self._proj_logits(A, nd.g * R, st["WvUt"][nd.k], D, H,
                                  V[nd.first:nd.first + nd.g], L[nd.first:nd.first + nd.g],
                                  f"fwd:vl_l{li}")
            else:
                matmul(A, st["WvU"][nd.k, :, :D], out=V[nd.first:nd.first + nd.g].view(-1, D),
                       work={"site": f"fwd:v_l{li}", "flops": 2 * nd.g * R * D * D})
        mix = None if st["attn"] else self._mix(li)
        ctx = self._combine(V, L, mix, st["comb"][li], R)
        return V, L, ctx, self._node_out(ctx, nodes, R)

    def forward_train(self, images):
        """Full forward of this rank: slab tree, AllGather of the root streams (rank order,
        runtime.py:259), shared final layer.  Returns ([B,1,S,D] fp32, saved)."""
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
        st = self._static()
        if fe.strategy.final_layer_tp_split and fe.tp > 1:
            return self._forward_final_split(y_all, saved)
        D, H = st["D"], st["H"]
        R, B = saved["R"], saved["B"]
        fin = st["final"]
        Vf = torch.empty(fe.tp, R, D, device=y_all.device, dtype=torch.bfloat16)
        Lf = torch.empty(fe.tp, R, H, device=y_all.device)
        self._proj_logits(y_all.reshape(fe.tp * R, D), fe.tp * R, st["WvUt"][fin.k], D, H, Vf,
                          Lf, "fwd:vl_final")
        ctx_f = self._combine(Vf, Lf, None, st["comb"]["final"], R)
        out = matmul(ctx_f[0], st["wo16"][fin.k], bias=st["bo32"][fin.k],
                     work={"site": "fwd:wo_final", "flops": 2 * R * D * D})
        saved.update(y_all=y_all, Vf=Vf, Lf=Lf, ctx_f=ctx_f)
        return out.view(B, 1, fe.seq, D)

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
        st = self._st
        D = st["D"]
        R, B = saved["R"], saved["B"]
        _, hc, cols, hs = self._own_heads()
        dl = cols.stop - cols.start
        fin = st["final"]
        Vf = torch.empty(fe.tp, R, dl, device=y_all.device, dtype=torch.bfloat16)
        Lf = torch.empty(fe.tp, R, hc, device=y_all.device)
        self._proj_logits(y_all.reshape(fe.tp * R, D), fe.tp * R, st["hs_WvUt"], dl, hc, Vf, Lf,
                          "fwd:vl_final")
        ctx_f = self._combine(Vf, Lf, None, st["comb"]["final"], R, heads=hc, Dv=dl)
        bo = st["bo32"][fin.k] if fe.rank == 0 else st["zero_b"][:D]
        out = matmul(ctx_f[0], st["wo16"][fin.k, cols], bias=bo,
                     work={"site": "fwd:wo_final", "flops": 2 * R * dl * D})
        comm.all_reduce(out, group=fe.process_group)
        fe._log("AllReduce", "forward", "agg-final", (out.numel(), out.element_size()))
        saved.update(y_all=y_all, Vf=Vf, Lf=Lf, ctx_f=ctx_f)
        return out.view(B, 1, fe.seq, D)

    # ---------------------------------------------------------------- backward
    def _colsum(self, X, G, R, N, out, period=1, accumulate=0, ldo=0, gscale=None):
        """out[g] (+)= periodic column sums of X[g] (bf16 or fp32), rows X.stride(-2) apart;
        out fp32, or bf16 (rows ldo apart) for a bf16 GEMM operand."""
        sxg = X.stride(0) if X.dim() == 3 else 0
        work = torch.empty(G * (-(-R // 64)) * N, device=X.device) if period == 1 else None
        sog = out.stride(0) if out.dim() >= 2 and G > 1 else 0
        _lib.call("dchag_colsum", _ptr(X), int(X.dtype == torch.float32), X.stride(-2), sxg, G,
                  R, N, period, _ptr(out), sog, ldo, int(out.dtype == torch.bfloat16),
                  accumulate, _lib.ptr(gscale), _lib.ptr(work), _lib.stream_handle(),
                  work={"site": "bwd:colsum", "bytes": X.numel() * X.element_size()})
        return out

    def backward(self, saved, g_out):
        """Gradients of sum(out * g_out) w.r.t. this rank's parameters (reference names):
        the slab's tok.* / channel_id rows, its agg.slab{r}.*, the replicated agg.final.*,
        and special.pos all-reduced over the tp group."""
        grads, g_y = self.backward_final(saved, g_out)
        grads.update(self.backward_local(saved, g_y))
        if self.dp_group is not None:
            self._dp_average(grads)
        if self.fe.tp > 1:
            comm.all_reduce(grads["special.pos"], group=self.fe.process_group)
            self.fe._log("AllReduce", "optimizer", "shared-grad.special.pos",
                         (grads["special.pos"].numel(), grads["special.pos"].element_size()))
        return grads

    def _query_fold_backward(self, grads):
        """d wk, d wq, d q of every attention node from its d U (one batched launch). The
        head-split final layer's shards are reported by _backward_final_split."""
        st = self._st
        D, H = st["D"], st["H"]
        qn = len(st["qnodes"])
        _lib.call("dchag_query_fold_bwd", _ptr(st["qb"]), qn, D, H, _ptr(st["qf_work"]),
                  _ptr(st["dqp"]), _lib.stream_handle(),
                  work={"site": "bwd:query_fold", "flops": 8 * qn * D * D,
                        "bytes": 16 * qn * D * D})
        split = self.fe.strategy.final_layer_tp_split and self.fe.tp > 1
        for nd in st["qnodes"]:
            if nd is st["final"] and split:
                continue
            grads[f"{nd.name}.wk"] = st["dwk"][nd.k]
            grads[f"{nd.name}.wq"] = st["dwq"][nd.k]
            grads[f"{nd.name}.q"] = st["dq"][nd.k]
        if split:
            _, _, cols, _ = self._own_heads()
            fin = st["final"]
            grads["agg.final.wk"] = st["dwk"][fin.k][:, cols]
            grads["agg.final.wq"] = st["dwq"][fin.k][:, cols]
            q_grad = st["dq"][fin.k].clone()
            comm.all_reduce(q_grad, group=self.fe.process_group)          # fanout of q
            self.fe._log("AllReduce", "backward", "agg-final",
                         (q_grad.numel(), q_grad.element_size()))
            grads["agg.final.q"] = q_grad

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

    def backward_final(self, saved, g_out):
        """Final-layer grads (identical on every rank) and this rank's root-stream gradient
        (the local slice of the gathered gradient, strategies.py:91-94)."""
        fe = self.fe
        st = self._static()
        if fe.strategy.final_layer_tp_split and fe.tp > 1:
            return self._backward_final_split(saved, g_out)
        D, Dp = st["D"], st["Dp"]
        R = saved["R"]
        fin = st["final"]
        g32 = g_out.reshape(R, D).float()
        g16 = g32.to(torch.bfloat16)
        ctx_f = saved["ctx_f"][0]
        grads = {"agg.final.bo": self._colsum(g32, 1, R, D, torch.empty(D, device=g32.device))}
        grads["agg.final.wo"] = matmul(ctx_f.t(), g16,
                                       work={"site": "bwd:dwo_final", "flops": 2 * R * D * D})
        G = matmul(g16, st["wo16"][fin.k].t(),
                   work={"site": "bwd:g_final", "flops": 2 * R * D * D})
        gVL = self._combine_bwd(saved["Vf"], saved["Lf"], None, G.view(1, R, D),
                                st["comb"]["final"], R, fe.tp, tag="final")
        y_all = saved["y_all"].reshape(fe.tp * R, D)
        matmul(y_all.t(), gVL.view(fe.tp * R, Dp), out=st["dWvU"][fin.k],
               work={"site": "bwd:dwvu_final", "flops": 2 * fe.tp * R * D * Dp})
        grads["agg.final.wv"] = st["dWvU"][fin.k, :, :D]
        # local slice of the gathered gradient (strategies.py:91-94): no collective
        g_y = matmul(gVL[fe.rank], st["WvU"][fin.k].t(), out_dtype=torch.bfloat16,
                     work={"site": "bwd:gprev_final", "flops": 2 * R * Dp * D})
        return grads, g_y.view(1, R, D)

    def _backward_final_split(self, saved, g_out):
        """Backward of the head-split final layer: shard grads (wv/wk/wq columns, wo rows of
        the own heads; bo and the fanned-out q in full), and the root-stream gradient by a
        ReduceScatter of every rank's partial gathered-stream gradient along the stream axis
        (the fused TpHooks.fanout RS + AG and gather slice, strategies.py:54-67, :91-94)."""
        fe = self.fe
        st = self._st
        D, H = st["D"], st["H"]
        R = saved["R"]
        fin = st["final"]
        _, hc, cols, hs = self._own_heads()
        dl = cols.stop - cols.start
        dpo = st["hs_dp"]
        g32 = g_out.reshape(R, D).float()
        g16 = g32.to(torch.bfloat16)
        grads = {"agg.final.bo": self._colsum(g32, 1, R, D, torch.empty(D, device=g32.device))}
        ctx_f = saved["ctx_f"][0]                                          # [R, dl]
        grads["agg.final.wo"] = matmul(ctx_f.t(), g16,                      # own rows
                                       work={"site": "bwd:dwo_final", "flops": 2 * R * dl * D})
        G = matmul(g16, st["wo16"][fin.k, cols].t(),
                   work={"site": "bwd:g_final", "flops": 2 * R * D * dl})
        key = ("hs_gVL", R)
        if key not in st:
            st[key] = torch.zeros(fe.tp, R, dpo, device=g32.device, dtype=torch.bfloat16)
        gVL = st[key]
        ft, gt, _ = st["comb"]["final"]
        _lib.call("dchag_combine_bwd_packed", 1, R, dl, hc, _ptr(ft), _ptr(gt), fe.tp,
                  _ptr(saved["Vf"]), R * dl, _ptr(saved["Lf"]), R * hc, 0, _ptr(G), _ptr(gVL),
                  R * dpo, dpo, 0, _lib.stream_handle(),
                  work={"site": "bwd:combine", "bytes": 4 * gVL.numel()})
        y_all = saved["y_all"].reshape(fe.tp * R, D)
        matmul(y_all.t(), gVL.view(fe.tp * R, dpo), out=st["hs_dWvU"],
               work={"site": "bwd:dwvu_final", "flops": 2 * fe.tp * R * D * dpo})
        grads["agg.final.wv"] = st["hs_dWvU"][:, :dl]
        # the own heads' d U into the final node's full-width d U (other heads zero): the
        # batched query-fold backward then gives dwk / dwq (own columns kept) and dq
        dU = st["dWvU"][fin.k, :, D:D + H]
        dU.zero_()
        dU[:, hs] = st["hs_dWvU"][:, dl:dl + hc]
        g_part = matmul(gVL.view(fe.tp * R, dpo), st["hs_WvU"].t(),
                        work={"site": "bwd:gprev_final", "flops": 2 * fe.tp * R * dpo * D})
        g_y = torch.empty(R, D, device=g32.device, dtype=torch.float32)
        comm.reduce_scatter_tensor(g_y, g_part.view(fe.tp * R, D), group=fe.process_group)
        fe._log("ReduceScatter", "backward", "agg-final", g_y.numel() * g_y.element_size())
        return grads, g_y.to(torch.bfloat16).view(1, R, D)

    def _combine_bwd(self, V, L, mix, G, tables, R, nch, dm=None, tag=""):
        """-> gVL bf16 [nch][R][Dp] = [gV | dL | 0] (the K-concatenated backward operand)."""
        st = self._st
        D, H, Dp = st["D"], st["H"], st["Dp"]
        key = ("gVL", tag, nch, R)
        gVL = st.get(key)
        if gVL is None:
            gVL = st[key] = torch.zeros(nch, R, Dp, device=V.device, dtype=torch.bfloat16)
        ft, gt, gmax = tables
        _lib.call("dchag_combine_bwd_packed", ft.numel(), R, D, H, _ptr(ft), _ptr(gt), gmax,
                  _ptr(V), R * D, _lib.ptr(L), R * H, _lib.ptr(mix), _ptr(G), _ptr(gVL),
                  R * Dp, Dp, _lib.ptr(dm), _lib.stream_handle(),
                  work={"site": "bwd:combine", "bytes": 2 * V.numel() * 2 + G.numel() * 4})
        return gVL

    def backward_local(self, saved, g_y):
        """Slab-tree and tokenizer grads from this rank's root-stream gradient g_y [1,R,D];
        special.pos is this rank's partial (summed over tp by backward())."""
        st = self._st
        R = saved["R"]
        grads = {}
        g_y = g_y if g_y.dtype == torch.bfloat16 else g_y.to(torch.bfloat16)
        for li in range(len(st["levels"]) - 1, 0, -1):
            g_y = self._level_backward(saved, li, g_y, grads, R)
        self._level0_backward(saved, g_y, grads, R)
        # d wk / d wq / d q of every attention node, the final layer's included (its d U was
        # produced by backward_final)
        self._query_fold_backward(grads)
        return grads

    def _node_grads_out(self, nodes, ctx, g_y, R, grads):
        """d bo (linear: d b) and d wo of a level's nodes."""
        st = self._st
        D = st["D"]
        n = len(nodes)
        db = self._colsum(g_y, n, R, D, torch.empty(n, D, device=g_y.device))
        bname = "bo" if st["attn"] else "b"
        for i, nd in enumerate(nodes):
            grads[f"{nd.name}.{bname}"] = db[i]
        if st["attn"]:
            dwo = matmul(ctx.transpose(1, 2), g_y,
                         work={"site": f"bwd:dwo_l{nodes[0].li}", "flops": 2 * n * R * D * D})
            for i, nd in enumerate(nodes):
                grads[f"{nd.name}.wo"] = dwo[i]

    def _level_backward(self, saved, li, g_y, grads, R):
        st = self._st
        D, Dp = st["D"], st["Dp"]
        attn = st["attn"]
        nodes = st["lvl"][li]
        k0, n = nodes[0].k, len(nodes)
        ctx = saved["ctx"][li]
        V, L = saved["VL"][li - 1]
        y_prev = saved["y"][li - 1]
        self._node_grads_out(nodes, ctx, g_y, R, grads)
        if attn:
            G = matmul(g_y, st["wo16"][k0:k0 + n].transpose(1, 2),
                       work={"site": f"bwd:g_l{li}", "flops": 2 * n * R * D * D})
            mix, dm = None, None
        else:
            G = g_y.float()
            mix = self._mix(li)
            dm = torch.empty(V.shape[0], R, device=V.device)
        gVL = self._combine_bwd(V, L, mix, G, st["comb"][li], R, V.shape[0], dm=dm, tag=li)
        g_prev = torch.empty(y_prev.shape, device=y_prev.device, dtype=torch.bfloat16)
        gs = {nd.g for nd in nodes}
        if len(gs) == 1 and nodes[-1].first + nodes[-1].g == y_prev.shape[0]:
            # equal fan-in: one grouped launch per product for the whole level
            g = nodes[0].g
            Y = y_prev.view(n, g * R, D)
            gv = gVL.view(n, g * R, Dp)
            matmul(Y.transpose(1, 2), gv, out=st["dWvU"][k0:k0 + n],
                   work={"site": f"bwd:dwvu_l{li}", "flops": 2 * n * g * R * D * Dp})
            matmul(gv, st["WvU"][k0:k0 + n].transpose(1, 2), out=g_prev.view(n, g * R, D),
                   work={"site": f"bwd:gprev_l{li}", "flops": 2 * n * g * R * Dp * D})
            groups = []
        else:
            groups = nodes
        for nd in groups:
            f0, g = nd.first, nd.g
            Y = y_prev[f0:f0 + g].reshape(g * R, D)
            gv = gVL[f0:f0 + g].reshape(g * R, Dp)
            matmul(Y.t(), gv, out=st["dWvU"][nd.k],
                   work={"site": f"bwd:dwvu_l{li}", "flops": 2 * g * R * D * Dp})
            matmul(gv, st["WvU"][nd.k].t(), out=g_prev[f0:f0 + g].view(g * R, D),
                   work={"site": f"bwd:gprev_l{li}", "flops": 2 * g * R * Dp * D})
        for nd in nodes:
            f0, g = nd.first, nd.g
            grads[f"{nd.name}.{'wv' if attn else 'w'}"] = st["dWvU"][nd.k, :, :D]
            if not attn:
                dmix = torch.empty(g, device=V.device)
                _lib.call("dchag_rowsum", _ptr(dm[f0:f0 + g]), R, g, R, _ptr(dmix),
                          _lib.stream_handle(), work={"site": "bwd:rowsum", "bytes": 4 * g * R})
                grads[f"{nd.name}.mix"] = dmix
        return g_prev

    def _level0_backward(self, saved, g_y, grads, R):
        fe = self.fe
        m = fe.model
        st = self._st
        D, H, S, Dp, PP = st["D"], st["H"], st["S"], st["Dp"], st["PP"]
        n0, Kn, ones0 = st["n0"], st["Kn"], st["ones0"]
        attn = st["attn"]
        nodes = st["lvl"][0]
        img = saved["img"]
        B = saved["B"]
        dev = img.device
        sh = _lib.stream_handle()
        off, cnt = fe.slab
        ctx0 = saved["ctx"][0]
        self._node_grads_out(nodes, ctx0, g_y, R, grads)
        if attn:
            Gb = matmul(g_y, st["wo16"][:n0].transpose(1, 2), out_dtype=torch.bfloat16,
                        work={"site": "bwd:g_l0", "flops": 2 * n0 * R * D * D})
        else:
            Gb = g_y
        patches = torch.empty(B, cnt, S, PP, device=dev, dtype=torch.bfloat16)
        _lib.call("dchag_unfold", _ptr(img), img.stride(0), img.stride(1), B, cnt, m.image_h,
                  m.image_w, m.patch, _ptr(patches), sh,
                  work={"site": "bwd:unfold", "bytes": 4 * img.numel()})
        if attn:  # normalised level-0 softmax: the forward's e x 1/sum e (no second K_p0)
            gl = st["levels"][0]
            pnorm = torch.empty(sum(gl) * R * H, device=dev, dtype=torch.bfloat16)
            _lib.call("dchag_l0_p_normalize", _ptr(saved["p_e"]), _ptr(saved["pinv"]),
                      _ptr(pnorm), _ptr(saved["poff"]), _ptr(st["l0_g"]), n0, max(gl), R, H,
                      st["NH"], sh,
                      work={"site": "bwd:p_normalize", "bytes": sum(gl) * R * H * 4 + n0 * R * H * 4})
        # positional sums over the batch, Gs_n[s] = sum_b G_n[b, s] (x sum(mix), linear),
        # straight into the pos rows of the node's TE block (bf16 GEMM operand)
        TE = st["TE"]
        self._colsum(Gb, n0, R, D, TE[:, Kn:, :D], period=S, ldo=Dp,
                     gscale=None if attn else st["mixsum"])
        fast = (PP == 64 and D % 128 == 0 and S % 64 == 0 and D // H in (64, 128) and H <= 128
                and (not attn or st["NH"] % 2 == 0))
        dh = D // H
        p_at = 0
        for nd in nodes:
            g, c0, n = nd.g, st["c0s"][nd.gi], nd.gi
            Gn = Gb[n]
            if attn:
                pblk = pnorm[p_at:p_at + g * R * H]
                p_at += g * R * H
                pptr, mptr, nh_ = _ptr(pblk), 0, st["NH"]
            else:
                mixv = fe.weights[f"{nd.name}.mix"].float()
                pptr, mptr, nh_ = 0, _ptr(mixv), 1
            Gpos = torch.empty(R, H, device=dev)
            dV = None if fast else torch.empty(g, R, D, device=dev, dtype=torch.bfloat16)
            _lib.call("dchag_l0_dv", g, R, D, H, nh_, pptr, mptr, _ptr(Gn), _ptr(st["posVU"][n]),
                      Dp, S, _ptr(Gpos), _lib.ptr(dV), sh,
                      work={"site": "bwd:l0_dv", "bytes": 2 * R * D * (1 + (0 if fast else g))})
            # heads of 64 columns summed inside the row-dot drain (one dp partial per head:
            # half the partials written and read back) where the lean drain takes the shape
            heads = (attn and fast and dh == 64 and g <= 16 and D % 256 == 0
                     and (R // 128) % 2 == 0 and os.environ.get("DCHAG_GEMM_LEAN", "1") != "0"
                     and int(os.environ.get("DCHAG_GEMM_DEBUG", "0") or 0) & ~20 == 0)
            grp = 64 if heads else 32
            dpp = torch.empty(g, D // grp, R, device=dev)
            _lib.call("dchag_gemm_rowdot_heads", _ptr(patches[:, c0:c0 + g]), g, B, S, PP,
                      S * PP, cnt * S * PP, PP, _ptr(st["Mrow"][c0]), D, D * PP,
                      _ptr(st["Cb"][c0]), D, _ptr(Gn), D, grp, _ptr(dpp), sh,
                      work={"site": "bwd:l0_rowdot", "flops": 2 * g * R * D * PP,
                            "bytes": R * D * 2 + g * R * PP * 2 + g * D // grp * R * 4})
            dl = dlb = None
            if attn:
                # the tcgen05 TE kernel reads only the bf16 copy (fp32 dl: the generic path)
                if not fast or g > 16 or dh != 64:
                    dl = torch.empty(g, H, R, device=dev)
                dlb = torch.empty(g, H, R, device=dev, dtype=torch.bfloat16)
                _lib.call("dchag_l0_softmax_bwd", g, R, H, st["NH"], 32 if heads else dh,
                          _ptr(dpp), _ptr(Gpos), _ptr(pblk), _lib.ptr(dl), _ptr(dlb), sh,
                          work={"site": "bwd:l0_softmax", "bytes": 4 * g * R * D // grp})
            else:
                dp = dpp.view(g, H, dh // grp, R).sum(2) + Gpos.t().unsqueeze(0)
                grads[f"{nd.name}.mix"] = dp.sum((1, 2))
            if fast:
                _lib.call("dchag_l0_tgrad_te", _ptr(patches), cnt, c0, g, R, S, D, H, nh_, PP,
                          pptr, mptr, _ptr(Gn), _lib.ptr(dlb), _ptr(TE[n]), Dp, ones0, sh,
                          work={"site": "bwd:l0_tgrad_te",
                                "flops": 2 * g * R * 80 * (D + (128 if attn else 0))})
            else:
                self._te_generic(patches, c0, g, R, dV, dl, dlb, TE[n])
        # [d Wv | d U] = [tok.w ; tb ; pos]^T TE   (the pos rows add pos^T Gs_n),
        # d [tok.w ; tb ; pos_n] = TE [Wv | U]^T   (the pos rows give Gs_n Wv_n^T)
        dW = st["dWvU"][:n0]
        matmul(st["Waug"].transpose(1, 2), TE, out=dW,
               work={"site": "bwd:l0_dwvu", "flops": 2 * n0 * (Kn + S) * D * Dp})
        dWaug = matmul(TE, st["WvU"][:n0].transpose(1, 2),
                       work={"site": "bwd:l0_dtok", "flops": 2 * n0 * (Kn + S) * Dp * D})
        flat = dWaug.view(n0 * (Kn + S), D)
        grads["tok.w"] = flat.index_select(0, st["rows_w"]).view(cnt, PP, D)
        d_tb = flat.index_select(0, st["rows_b"])
        grads["tok.b"] = d_tb
        grads["special.channel_id"] = d_tb.clone()
        grads["special.pos"] = dWaug[:, Kn:].sum(0)  # partial; backward() all-reduces it
        wname = "wv" if attn else "w"
        for nd in nodes:
            grads[f"{nd.name}.{wname}"] = dW[nd.gi, :, :D]
        return grads

    def _te_generic(self, patches, c0, g, R, dV, dl, dlb, TE_n):
        """TE block without the tcgen05 TE kernel (shapes it does not take, e.g. P = 4):
        T_c = patch_c^T dV_c and E_c = patch_c^T dl_c on the GEMM, the bias rows as column /
        row sums."""
        st = self._st
        D, H, PP, ones0 = st["D"], st["H"], st["PP"], st["ones0"]
        pn = patches[:, c0:c0 + g].permute(1, 0, 2, 3).reshape(g, R, PP)
        T = matmul(pn.transpose(1, 2), dV, work={"site": "bwd:l0_t_generic"})
        TE_n[:g * PP, :D] = T.reshape(g * PP, D)
        colV = self._colsum(dV, g, R, D, torch.empty(g, D, device=dV.device))
        TE_n[ones0:ones0 + g, :D] = colV
        if dl is not None:
            E = matmul(pn.transpose(1, 2), dlb.transpose(1, 2), work={"site": "bwd:l0_e_generic"})
            TE_n[:g * PP, D:D + H] = E.reshape(g * PP, H)
            coll = torch.empty(g * H, device=dl.device)
            _lib.call("dchag_rowsum", _ptr(dl), R, g * H, R, _ptr(coll), _lib.stream_handle(),
                      work={"site": "bwd:rowsum", "bytes": 4 * g * H * R})
            TE_n[ones0:ones0 + g, D:D + H] = coll.view(g, H)


class GraphedStep:
    """A captured training step (DchagTrainer.capture)."""

    def __init__(self, graph, out, grads, launches):
        self.graph, self.out, self.grads, self.launches = graph, out, grads, launches

    def replay(self):
        self.graph.replay()
        _lib.LAUNCH_COUNT["n"] += self.launches
        return self.grads
