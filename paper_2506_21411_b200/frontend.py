"""DchagFrontEnd: the drop-in module for D-CHAG's channel front end on B200.

Constructor arguments are the reference's ModelConfig / StrategyConfig fields for
this path (config.py:70-84, :121-126); `depth` is optional and validated against
build_tree_spec(local_channels, max_group).depth.  Weights use the reference's
dotted names and [D_in, D_out] layout (params.py:1-24, :36-57), so a dict from
the reference's `create_master` loads 1:1 (`load_weights`).

forward(images[B, C_local or C, H, W]) -> [B, 1, S, D]   (model.py:180-201 hot path)

Execution per rank, all on the caller's current stream:
  K_p0  level-0 logits+softmax      (dchag_l0_logits)
  K_l0  level-0 context, tcgen05    (dchag_l0_node)
  K_gemm per level: node projection folded with its consumer (dchag_gemm_bf16)
  K_comb per level >= 1: softmax-weighted child sum (dchag_combine)
  AllGather of the root payload over NCCL (tp > 1), in rank order (runtime.py:259)
  K_comb + K_gemm: shared final layer.
"""

from __future__ import annotations

import math

import os

import torch

from . import _lib, comm
from .config import (ConfigError, ModelConfig, StrategyConfig, TreeSpec, build_tree_spec,
                     channel_slabs, max_group_for_depth)
from .fold import fold_rank, pack_rank, refresh_packed
from .payload import payload_nbytes, views


def frontend_param_specs(model: ModelConfig, strategy: StrategyConfig):
    """(name, shape, init) of the front-end parameters in the reference creation order
    (params.py:99-115), with one tree per rank slab (uneven slabs get their own trees)."""
    c, d, p = model.channels, model.embed, model.patch
    specs = [("tok.w", (c, p * p, d), "normal"), ("tok.b", (c, d), "zeros"),
             ("special.channel_id", (c, d), "normal"), ("special.pos", (model.seq, d), "normal")]

    def node(prefix, g, kind):
        if kind == "linear":
            return [(f"{prefix}.mix", (g,), "normal"), (f"{prefix}.w", (d, d), "normal"),
                    (f"{prefix}.b", (d,), "zeros")]
        out = [(f"{prefix}.q", (d,), "normal")] if model.agg_variant == "single_query" else []
        out += [(f"{prefix}.{n}", (d, d), "normal") for n in ("wq", "wk", "wv", "wo")]
        out.append((f"{prefix}.bo", (d,), "zeros"))
        if model.agg_variant == "full_cross":
            out.append((f"{prefix}.rq", (d,), "normal"))
        return out

    for r in range(strategy.tp_degree):
        tree = strategy.rank_tree(model, r)
        for li, level in enumerate(tree.levels):
            for gi, g in enumerate(level):
                specs += node(f"agg.slab{r}.l{li}.g{gi}", g, strategy.agg_layer_kind)
    specs += node("agg.final", strategy.tp_degree, "cross_attention")
    return specs


class DchagFrontEnd(torch.nn.Module):
    def __init__(self, channels: int, image_h: int, image_w: int, patch: int, embed: int,
                 heads: int, max_group: int | None = None, depth: int | None = None,
                 agg_variant: str = "single_query", agg_layer_kind: str = "cross_attention",
                 tp: int = 1, rank: int = 0, final_layer_tp_split: bool = False,
                 process_group=None, out_dtype=torch.bfloat16, device=None,
                 precision: str = "bf16", final_position_split: bool = True):
        super().__init__()
        self.model = ModelConfig(channels=channels, image_h=image_h, image_w=image_w,
                                 patch=patch, embed=embed, heads=heads,
                                 agg_variant=agg_variant, agg_layer_kind=agg_layer_kind)
        self.model.validate()
        slabs = channel_slabs(channels, tp)
        if max_group is None:
            if depth is None:
                raise ConfigError("give max_group or depth")
            max_group = max_group_for_depth([n for _, n in slabs], depth)
        self.strategy = StrategyConfig(kind="dchag", tp_degree=tp, max_group=max_group,
                                       agg_layer_kind=agg_layer_kind,
                                       final_layer_tp_split=final_layer_tp_split,
                                       uneven_slabs=True)
        self.strategy.validate(self.model)
        trees = [build_tree_spec(n, max_group) for _, n in slabs]
        if depth is not None and any(t.depth != depth for t in trees):
            raise ConfigError(
                f"depth {depth} disagrees with build_tree_spec(local_channels, {max_group}): "
                f"{sorted({t.depth for t in trees})}")
        if not 0 <= rank < tp:
            raise ConfigError(f"rank {rank} outside tp {tp}")
        self._check_gpu_shape()
        self.tp, self.rank = tp, rank
        self.slabs = slabs
        self.slab = slabs[rank]
        self.tree: TreeSpec = trees[rank]
        self.process_group = process_group
        self.out_dtype = out_dtype
        # tp > 1: exchange the root payload by position (all-to-all) and run the final
        # layer on R/tp rows per rank, then all-gather the outputs. The
        # per-row arithmetic is the same kernels on the same operands as the AllGather
        # schedule, so the result is bit-identical; only the bytes moved and the final
        # layer's work per rank shrink by ~tp.
        self.final_position_split = bool(final_position_split)
        self.ledger = None  # optional ledger.CommLedger: every collective issued is recorded
        # levels below the root: projection + parent combine in one K_gemm (COMB instance)
        self.fuse_combine = os.environ.get("DCHAG_FUSE_COMBINE", "1") != "0"
        self.combine_split = os.environ.get("DCHAG_COMBINE_SPLIT", "0") != "0"
        # tp > 1 device forward: batch chunks whose exchange overlaps the next chunk's kernels
        # (measured on 2 B200 at H2: 1 chunk 20.7k img/s, 2 chunks 18.9k, 4 chunks 18.3k --
        # the exchange is short and smaller launches lose more, so off by default)
        self.comm_chunks = int(os.environ.get("DCHAG_COMM_CHUNKS", "1"))
        if precision not in ("bf16", "fp32"):
            raise ConfigError(f"precision must be 'bf16' or 'fp32', got {precision!r}")
        if precision == "fp32" and agg_variant != "single_query":
            raise ConfigError("the fp32 parity mode implements agg_variant='single_query'")
        # "fp32": parity mode, results within 1e-4 of the float64 reference (BASELINE.json);
        # "bf16": the throughput path (bf16 operands, fp32 accumulation, within 2e-2)
        self.precision = precision
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        self.weights: dict[str, torch.Tensor] = {}
        self._packed = None
        self._packed_sig = None

    # ------------------------------------------------------------------ config
    def _check_gpu_shape(self):
        m = self.model
        dh = m.embed // m.heads
        s = m.seq
        wp = m.image_w // m.patch
        probs = []
        if dh not in (64, 128):
            probs.append(f"head dim {dh} not in (64, 128)")
        if m.heads % 2:
            probs.append(f"heads {m.heads} not even")
        if m.patch not in (4, 8):
            probs.append(f"patch {m.patch} not in (4, 8)")
        if s % 128:
            probs.append(f"tokens per image {s} not a multiple of 128")
        if 128 % wp:
            probs.append(f"patch columns {wp} do not divide 128")
        if probs:
            raise ConfigError("shape unsupported by the sm_100a kernels: " + "; ".join(probs))

    @property
    def seq(self) -> int:
        return self.model.seq

    def param_specs(self):
        return frontend_param_specs(self.model, self.strategy)

    # ----------------------------------------------------------------- weights
    def load_weights(self, master: dict) -> None:
        """Load reference-named weights (numpy or torch); the rank keeps what it needs:
        the channel slab of tok.*/special.channel_id, special.pos, its own agg.slab{r}.*
        and agg.final.* (params.py:180-221)."""
        keep = {}
        for name, shape, _ in self.param_specs():
            if name.startswith("agg.slab") and not name.startswith(f"agg.slab{self.rank}."):
                continue
            if name not in master:
                raise KeyError(f"missing weight {name}")
            t = torch.as_tensor(master[name])
            if tuple(t.shape) != tuple(shape):
                raise ConfigError(f"{name}: shape {tuple(t.shape)} != {shape}")
            keep[name] = t.to(device=self.device, dtype=torch.float32)
        self.weights = keep
        # a new weight set may differ in every derived buffer: fold from scratch (the
        # head-split final-layer shards live on the packed rank, so they go with it)
        self._packed = None
        self._packed_sig = None

    def needed_names(self):
        return [n for n, _, _ in self.param_specs()
                if not n.startswith("agg.slab") or n.startswith(f"agg.slab{self.rank}.")]

    def init_weights(self, seed: int = 0, std: float = 0.02, all_ranks: bool = True) -> dict:
        """Truncated-normal(std) weights, zero biases (the reference init distribution,
        params.py:139-150).  Every tensor has its own generator seeded from (seed, name), so
        ranks that build only their own slab's weights (all_ranks=False) agree on the
        shared ones.  Returns the named dict that was generated."""
        import zlib
        names = None if all_ranks else set(self.needed_names())
        master = {}
        for name, shape, init in self.param_specs():
            if names is not None and name not in names:
                continue
            if init == "zeros":
                master[name] = torch.zeros(shape, device=self.device)
                continue
            g = torch.Generator(device=self.device)
            g.manual_seed((seed * 1000003 + zlib.crc32(name.encode())) & 0x7FFFFFFFFFFF)
            v = torch.randn(shape, generator=g, device=self.device)
            bad = v.abs() > 2.0
            while bool(bad.any()):
                v[bad] = torch.randn(int(bad.sum()), generator=g, device=self.device)
                bad = v.abs() > 2.0
            master[name] = v * std
        self.load_weights(master)
        return master

    def _weights_signature(self):
        """Identity and in-place version of every loaded weight tensor: an optimizer step
        (in-place update) or a reassignment changes it."""
        return tuple((k, id(v), v._version) for k, v in self.weights.items())

    def prepare(self):
        """Fold + pack the weights for the kernels. The folded buffers are rebuilt whenever
        a loaded weight changes (reassigned, reloaded, or updated in place: the check keys on
        each tensor's version counter). A refold of an already packed rank writes into the
        existing device buffers, so CUDA graphs captured over them stay valid."""
        if self._unfolded():
            if not self.weights:
                raise RuntimeError("no weights loaded")
            return None  # full_cross / fp32 run the unfolded ops path on the reference weights
        if not self.weights:
            raise RuntimeError("no weights loaded")
        sig = self._weights_signature()
        if self._packed is None or self._packed_sig != sig:
            with torch.no_grad():
                fr = fold_rank(self.weights, rank=self.rank, slab=self.slab,
                               levels=self.tree.levels, embed=self.model.embed,
                               heads=self.model.heads, patch=self.model.patch, seq=self.seq,
                               variant=self.model.agg_variant,
                               layer_kind=self.strategy.agg_layer_kind)
                fresh = pack_rank(fr, self.device)
                if self._packed is None:
                    self._packed = fresh
                else:
                    refresh_packed(self._packed, fresh)
                    if self._packed.head_split is not None:
                        self._head_split_weights(self._packed, refresh=True)
            self._packed_sig = sig
        return self._packed

    # ------------------------------------------------------------------ forward
    def _unfolded(self):
        return self.model.agg_variant == "full_cross" or self.precision == "fp32"

    def _forward_full_cross(self, images, out=None):
        """agg_variant='full_cross' (layers.py:125-138): level 0 with the tokenizer folded
        (ops.full_cross_level0: q | k | u from the patches, the channel-attention weights,
        then K_l0 sums the children's values from the patches; tokens never formed), the
        levels above run ops._full_cross_tree on the node outputs,
        the [B,1,S,D] root streams are all-gathered in rank order and the shared final node
        runs over them (model.py:180-201 / strategies.py:199-218)."""
        from . import ops
        w = self.weights
        m = self.model
        off, cnt = self.slab
        sl = slice(off, off + cnt)
        if self.precision == "fp32":
            return self._forward_fp32(images, out)
        pre = f"agg.slab{self.rank}"
        if self.strategy.agg_layer_kind != "linear":
            # level 0 with the tokenizer folded into q / k / v / u (no token tensor)
            y0 = ops.full_cross_level0(images, w["tok.w"][sl], w["tok.b"][sl],
                                       w["special.channel_id"][sl], w["special.pos"],
                                       self.tree, w, pre, m.heads, m.patch)
            y = ops._full_cross_tree((images.shape[0], self.seq, m.embed), self.tree, w, pre,
                                     m.heads, torch.bfloat16, x0=y0)           # [B,1,S,D]
        else:
            tok = ops.tokenize_channels(images, w["tok.w"][sl], w["tok.b"][sl],
                                        w["special.channel_id"][sl], w["special.pos"], m.patch,
                                        out_dtype=torch.bfloat16)
            y = ops.tree_aggregate(tok, self.tree, w, pre, self.strategy.agg_layer_kind,
                                   "full_cross", m.heads, out_dtype=torch.bfloat16)
        if self.tp > 1:
            y = y.contiguous()
            allg = torch.empty((self.tp,) + tuple(y.shape), device=y.device, dtype=y.dtype)
            comm.all_gather_into_tensor(allg, y, group=self.process_group)
            self._log("AllGather", "forward", "dchag-boundary", y.numel() * y.element_size())
            gathered = allg.squeeze(2).permute(1, 0, 2, 3)                     # [B,tp,S,D]
        else:
            gathered = y
        res = ops.flat_aggregate(gathered, w, "agg.final", "full_cross", m.heads,
                                 out_dtype=self.out_dtype)
        if out is not None:
            out.copy_(res)
            return out
        return res

    def _forward_fp32(self, images, out=None):
        """fp32 parity mode (results within 1e-4 of the float64 reference): tokens, tree and
        final layer with fp32-accurate split-bf16 GEMMs and fp32 combines (ops.*_fp32)."""
        from . import ops
        w = self.weights
        m = self.model
        off, cnt = self.slab
        sl = slice(off, off + cnt)
        tok = ops.tokenize_channels_fp32(images.float(), w["tok.w"][sl], w["tok.b"][sl],
                                         w["special.channel_id"][sl], w["special.pos"], m.patch,
                                         node_major=True)
        y = ops.tree_aggregate_fp32(tok, self.tree, w, f"agg.slab{self.rank}",
                                    self.strategy.agg_layer_kind, m.heads,
                                    B=images.shape[0]).contiguous()
        if self.tp > 1:
            allg = torch.empty((self.tp,) + tuple(y.shape), device=y.device, dtype=y.dtype)
            comm.all_gather_into_tensor(allg, y, group=self.process_group)
            self._log("AllGather", "forward", "dchag-boundary", y.numel() * y.element_size())
            gathered = allg.squeeze(2).permute(1, 0, 2, 3)
        else:
            gathered = y
        res = ops.flat_aggregate_fp32(gathered, w, "agg.final", m.heads).to(self.out_dtype)
        if out is not None:
            out.copy_(res)
            return out
        return res

    def forward(self, images: torch.Tensor, return_payload: bool = False, out=None,
                h2d_chunks: int = 4):
        """[B, C or slab, H, W] images -> [B, 1, S, D] (model.py:180-201 front end).

        Device images run the rank's kernels on the current stream. Host images (pinned,
        for overlap) are streamed in `h2d_chunks` batch chunks: the copy of chunk k+1 on a
        side stream overlaps the kernels of chunk k (positions of different images are
        independent on this path, so chunking changes no result). `out`, when given, is
        the result buffer; a host `out` receives each chunk's rows as they finish."""
        pk = self.prepare()
        m = self.model
        if images.dim() != 4:
            raise ConfigError(f"images must be [B, C, H, W], got {tuple(images.shape)}")
        b, cin, himg, wimg = images.shape
        off, cnt = self.slab
        if (himg, wimg) != (m.image_h, m.image_w):
            raise ConfigError(f"image {himg}x{wimg} != configured {m.image_h}x{m.image_w}")
        if cin == m.channels and self.tp > 1:
            images = images[:, off:off + cnt]
        elif cin != cnt:
            raise ConfigError(f"images carry {cin} channels; rank {self.rank} expects {cnt} "
                              f"(its slab) or {m.channels} (all)")
        if out is not None and (tuple(out.shape) != (b, 1, self.seq, m.embed)
                                or out.dtype != self.out_dtype or not out.is_contiguous()):
            raise ConfigError(f"out must be a contiguous {self.out_dtype} tensor of shape "
                              f"{(b, 1, self.seq, m.embed)}")
        if self._unfolded():
            if not images.is_cuda or return_payload:
                raise ConfigError("agg_variant='full_cross' takes device images")
            return self._forward_full_cross(images, out)
        if not images.is_cuda:
            if return_payload:
                raise ConfigError("return_payload needs device images")
            return self._forward_host(images, pk, out, h2d_chunks)
        if images.dtype != torch.bfloat16:
            images = images.to(torch.bfloat16)
        if images.stride(3) != 1 or images.stride(2) != wimg:
            images = images.contiguous()
        dev_out = out if out is not None and out.is_cuda else None
        nc = self._comm_chunks(images.shape[0])
        if not return_payload and nc > 1:
            res = self._forward_pipelined(images, pk, dev_out, nc)
            if out is not None and not out.is_cuda:
                res = self._to_host(res, out)
            return res
        if self.tp == 1 and not return_payload:
            # one stream: the final layer's softmax is exactly 1, so the root projection and
            # the final projection fold into one GEMM writing the output
            B = images.shape[0]
            res = dev_out if dev_out is not None else torch.empty(
                B, 1, self.seq, m.embed, device=images.device, dtype=self.out_dtype)
            self.local_payload(images, pk, direct_out=res)
            if out is not None and not out.is_cuda:
                res = self._to_host(res, out)
            return res
        payload = self.local_payload(images, pk)
        if return_payload or not self._position_split(images.shape[0]):
            gathered = self.gather(payload)
            res = self.finish(gathered, images.shape[0], out=dev_out)
        else:
            res = self.exchange_finish(payload, images.shape[0], out=dev_out)
        if out is not None and not out.is_cuda:
            res = self._to_host(res, out)
        return (res, gathered) if return_payload else res

    @staticmethod
    def _to_host(res, out):
        """Copy a device result into the caller's host tensor and wait for it: like the
        reference's synchronous API, `out` is complete when forward returns."""
        out.copy_(res, non_blocking=True)
        torch.cuda.current_stream(res.device).synchronize()
        return out

    def vit_input(self, images, mask, mask_token, meta, meta_w, meta_b, out=None):
        """Front end + the trunk's input assembly: the aggregate with masked
        positions replaced by the mask token (model.py:100-108 apply_token_mask) and the
        metadata token prepended (model.py:111-117) -> [B, S+1, D] in out_dtype.
        mask [B, S] (1 = masked), mask_token [D] (`dec.mask`), meta [B, k] (k = 4 in the
        reference), meta_w [k, D] / meta_b [D] (`special.meta_w/b`).

        Device images on the folded plan (tp = 1, or the replicated final layer) fuse it into
        the final projection: its epilogue applies the mask and writes each row at its trunk
        position, and one small kernel writes the metadata rows (dchag_final_vit). The other
        schedules (position- / head-split final layer, full_cross, fp32 mode) assemble it
        from the forward's output (dchag_vit_tokens)."""
        m = self.model
        B, S, D = images.shape[0], self.seq, m.embed
        dev = self.device
        f32 = dict(device=dev, dtype=torch.float32)
        mask = torch.as_tensor(mask).to(**f32).reshape(B, S).contiguous()
        mtok = torch.as_tensor(mask_token).to(**f32).reshape(D).contiguous()
        meta = torch.as_tensor(meta).to(**f32).reshape(B, -1).contiguous()
        meta_w = torch.as_tensor(meta_w).to(**f32).reshape(meta.shape[1], D).contiguous()
        meta_b = torch.as_tensor(meta_b).to(**f32).reshape(D).contiguous()
        if out is None:
            out = torch.empty(B, S + 1, D, device=dev, dtype=self.out_dtype)
        elif tuple(out.shape) != (B, S + 1, D) or out.dtype != self.out_dtype or \
                not out.is_contiguous() or out.device != dev:
            raise ConfigError(f"out must be a contiguous {self.out_dtype} tensor of shape "
                              f"{(B, S + 1, D)} on {dev}")
        vit = (mask, mtok, meta, meta_w, meta_b)
        fused = (images.is_cuda and not self._unfolded() and self.comm_chunks == 1
                 and not self.strategy.final_layer_tp_split
                 and (self.tp == 1 or not self._position_split(B)))
        if fused:
            pk = self.prepare()
            img = self._check_images(images)
            if self.tp == 1:
                self.local_payload(img, pk, direct_out=out, vit=vit)
            else:
                self.finish(self.gather(self.local_payload(img, pk)), B, out=out, vit=vit)
            return out
        agg = self(images)
        meta_tok = (meta @ meta_w + meta_b).contiguous()
        _lib.call("dchag_vit_tokens", _lib.ptr(agg), int(agg.dtype == torch.float32), B, S, D,
                  _lib.ptr(mask), _lib.ptr(mtok), _lib.ptr(meta_tok), _lib.ptr(out),
                  _lib.stream_handle())
        return out

    def _final_vit(self, ctx, W, bias, B, out, vit):
        """Final projection with the trunk-input epilogue into out [B, S+1, D]."""
        m = self.model
        mask, mtok, meta, meta_w, meta_b = vit
        _lib.call("dchag_final_vit", _lib.ptr(ctx), B, self.seq, m.embed, _lib.ptr(W), m.embed,
                  _lib.ptr(bias), _lib.ptr(mask), _lib.ptr(mtok), _lib.ptr(meta), meta.shape[1],
                  _lib.ptr(meta_w), _lib.ptr(meta_b), _lib.ptr(out),
                  int(out.dtype == torch.float32), _lib.stream_handle())

    def _check_images(self, images):
        """Device images of this rank's slab as the kernels read them (bf16, row-contiguous)."""
        m = self.model
        off, cnt = self.slab
        if images.shape[1] == m.channels and self.tp > 1:
            images = images[:, off:off + cnt]
        elif images.shape[1] != cnt:
            raise ConfigError(f"images carry {images.shape[1]} channels; rank {self.rank} "
                              f"expects {cnt} (its slab) or {m.channels} (all)")
        if images.dtype != torch.bfloat16:
            images = images.to(torch.bfloat16)
        if images.stride(3) != 1 or images.stride(2) != m.image_w:
            images = images.contiguous()
        return images

    def _forward_host(self, images, pk, out, h2d_chunks):
        """Chunked H2D -> kernels -> (D2H) pipeline for host-resident images."""
        b, cnt, himg, wimg = images.shape
        if images.dtype != torch.bfloat16:
            images = images.to(torch.bfloat16)  # host-side cast; pass bf16 to avoid it
        dev = self.device
        cur = torch.cuda.current_stream(dev)
        cache = self.__dict__.setdefault("_cache", {})
        key = ("h2d", dev, b, cnt, himg, wimg)
        if key not in cache:
            cache[key] = (torch.empty(b, cnt, himg, wimg, device=dev, dtype=torch.bfloat16),
                          torch.cuda.Stream(dev))
        dbuf, side = cache[key]
        if out is None or out.is_cuda:
            res = out if out is not None else torch.empty(b, 1, self.seq, self.model.embed,
                                                          device=dev, dtype=self.out_dtype)
        else:
            res = torch.empty(b, 1, self.seq, self.model.embed, device=dev,
                              dtype=self.out_dtype)
        n = max(1, min(int(h2d_chunks), b))
        bounds = [(k * b) // n for k in range(n + 1)]
        # the staging buffer (and, for a host out, res) may still be read by earlier work
        side.wait_stream(cur)
        copied = []
        contig = images.is_contiguous()
        for k in range(n):
            b0, b1 = bounds[k], bounds[k + 1]
            with torch.cuda.stream(side):
                if contig:
                    dbuf[b0:b1].copy_(images[b0:b1], non_blocking=True)
                else:
                    for i in range(b0, b1):  # per-image contiguous runs (a channel slab)
                        dbuf[i].copy_(images[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
            copied.append(ev)
        for k in range(n):
            b0, b1 = bounds[k], bounds[k + 1]
            cur.wait_event(copied[k])
            if self.tp == 1:
                self.local_payload(dbuf[b0:b1], pk, direct_out=res[b0:b1])
            elif self._position_split(b1 - b0):
                self.exchange_finish(self.local_payload(dbuf[b0:b1], pk), b1 - b0,
                                     out=res[b0:b1])
            else:
                payload = self.local_payload(dbuf[b0:b1], pk)
                self.finish(self.gather(payload), b1 - b0, out=res[b0:b1])
            if out is not None and not out.is_cuda:
                done = torch.cuda.Event()
                done.record(cur)
                side.wait_event(done)
                with torch.cuda.stream(side):
                    out[b0:b1].copy_(res[b0:b1], non_blocking=True)
        if out is not None and not out.is_cuda:
            cur.wait_stream(side)
            cur.synchronize()  # a host `out` holds the result when forward returns
            return out
        return res

    def launch_plan(self, B: int):
        """Kernel launches of one forward in launch order, with the algorithmic work each
        does: (name, site, flops, bytes).  flops are the MMA flops of the folded plan
        (DESIGN.md section 5); bytes the compulsory HBM traffic."""
        pk = self.prepare()
        m = self.model
        d, h, s, pp = m.embed, m.heads, self.seq, m.patch * m.patch
        R = B * s
        G = sum(pk.l0_g_list)
        img_bytes = B * G * m.image_h * m.image_w * 2
        plan = []
        if pk.attn_l0:
            plan.append(("dchag_l0_logits", "l0_logits", 2 * 2 * R * G * pp * h,
                         img_bytes + R * G * h * 2))
        plan.append(("dchag_l0_node", "l0_node", 2 * R * d * G * (pp + 1),
                     img_bytes + (R * G * h * 2 if pk.attn_l0 else 0) + pk.n0 * R * d * 2))
        depth = len(pk.levels)
        for li in range(depth):
            n_l, N = len(pk.levels[li]), pk.N[li]
            if self._fused_level(pk, li, R):
                n_next = len(pk.levels[li + 1])
                plan.append(("dchag_gemm_bf16", f"gemm_logits_l{li}", 2 * R * n_l * d * h,
                             n_l * R * d * 2 + n_l * R * h * 4))
                plan.append(("dchag_child_softmax", f"child_softmax_l{li + 1}", 0,
                             2 * n_l * R * h * 4))
                plan.append(("dchag_gemm_combine", f"gemm_combine_l{li}", 2 * R * n_l * d * d,
                             n_l * R * d * 2 + n_l * d * d * 2 + n_next * R * d * 2))
                continue
            if li == depth - 1 and self.tp == 1:
                # root projection folded with the final layer (one stream)
                ob = 4 if self.out_dtype == torch.float32 else 2
                plan.append(("dchag_gemm_bf16", "gemm_root_final", 2 * R * d * d,
                             R * d * 2 + d * d * 2 + R * d * ob))
                return plan
            plan.append(("dchag_gemm_bf16", f"gemm_l{li}", 2 * R * n_l * d * N,
                         n_l * R * d * 2 + n_l * R * (d * 2 + (N - d) * 4) + n_l * N * d * 2))
            if li + 1 < depth:
                n_next = len(pk.levels[li + 1])
                plan.append(("dchag_combine", f"combine_l{li + 1}", 2 * R * n_l * d,
                             n_l * R * (d * 2 + h * 4) + n_next * R * d * 2))
        Rf = R // self.tp if self._position_split(B) else R   # rows of this rank's final
        if self.tp > 1:
            plan.append(("dchag_combine", "combine_final", 2 * Rf * self.tp * d,
                         self.tp * Rf * (d * 2 + h * 4) + Rf * d * 2))
        plan.append(("dchag_gemm_bf16", "gemm_final", 2 * Rf * d * d,
                     Rf * d * 2 + Rf * d * (4 if self.out_dtype == torch.float32 else 2)))
        return plan

    def gather(self, payload):
        """AllGather of the per-rank root payload in rank order (runtime.py:259)."""
        if self.tp == 1:
            return payload
        gathered = torch.empty(self.tp * payload.numel(), device=payload.device,
                               dtype=torch.uint8)
        comm.all_gather_into_tensor(gathered, payload, group=self.process_group)
        self._log("AllGather", "forward", "dchag-boundary", payload.numel())
        return gathered

    def _log(self, op, phase, tag, size):
        """Record one collective in self.ledger (ledger.py) with the reference's payload
        accounting. size: shard bytes (AllGather / ReduceScatter output chunk), buffer bytes
        (AllToAll), or (elements, itemsize) (AllReduce)."""
        if self.ledger is None:
            return
        from . import ledger as LG
        g = self.tp
        pay = {"AllGather": LG.allgather_payload, "ReduceScatter": LG.reduce_scatter_payload,
               "AllToAll": LG.alltoall_payload}.get(op)
        nbytes = pay(size, g) if pay else LG.allreduce_payload(size[0], size[1], g)
        self.ledger.record(self.rank, op, "tp", phase, nbytes, tag)

    def _comm_chunks(self, B):
        """Batch chunks of the pipelined tp > 1 forward (1 = no pipelining)."""
        n = self.comm_chunks
        while n > 1 and (B % n or not self._position_split(B // n)):
            n -= 1
        return n if self.tp > 1 else 1

    def _fused_level(self, pk, li, R):
        """Level li's projection fused with level li+1's combine (cross-attention parent)."""
        d, h = self.model.embed, self.model.heads
        return (self.fuse_combine and li + 1 < len(pk.levels) and pk.N[li] == d + h
                and R % 256 == 0 and d % 256 == 0 and (d // h) % 32 == 0 and h % 16 == 0)

    def _position_split(self, B):
        rows = B * self.seq
        return (self.final_position_split and self.tp > 1
                and not self.strategy.final_layer_tp_split
                and rows % (self.tp * 128) == 0)

    def exchange_start(self, payload, B, async_op=False):
        """First half of the position-split final layer: rank j receives rows
        [j R/tp, (j+1) R/tp) of every rank's root payload (one all-to-all of V, one of L).
        With async_op the exchange runs on NCCL's stream while later kernels proceed."""
        m = self.model
        d, h = m.embed, m.heads
        R = B * self.seq
        tp = self.tp
        Rl = R // tp
        dev = payload.device
        V, L = views(payload, R, d, h)
        Vx = torch.empty(tp, Rl, d, device=dev, dtype=torch.bfloat16)
        Lx = torch.empty(tp, Rl, h, device=dev, dtype=torch.float32)
        w1 = comm.all_to_all_single(Vx, V.view(tp, Rl, d), group=self.process_group,
                                    async_op=async_op)
        w2 = comm.all_to_all_single(Lx, L.view(tp, Rl, h), group=self.process_group,
                                    async_op=async_op)
        self._log("AllToAll", "forward", "dchag-boundary", payload.numel())
        return (B, Vx, Lx, (w1, w2) if async_op else ())

    def exchange_complete(self, state, out=None, async_op=False):
        """Second half: combine the tp streams of this rank's R/tp rows, final projection,
        all-gather of the outputs in rank (= row) order. Returns (out, pending work)."""
        B, Vx, Lx, works = state
        for wk in works:
            wk.wait()  # the current stream waits for the exchange
        pk = self.prepare()
        m = self.model
        d, h, s = m.embed, m.heads, self.seq
        R = B * s
        tp = self.tp
        Rl = R // tp
        dev = Vx.device
        st = _lib.stream_handle()
        ctx_f = torch.empty(1, Rl, d, device=dev, dtype=torch.bfloat16)
        first = self._final_first(dev)
        _lib.call("dchag_combine", 1, Rl, d, h, _lib.ptr(first[0]), _lib.ptr(first[1]), tp,
                  _lib.ptr(Vx), Rl * d, _lib.ptr(Lx), Rl * h, 0, _lib.ptr(ctx_f), st)
        part = torch.empty(Rl, d, device=dev, dtype=self.out_dtype)
        _lib.call("dchag_gemm_bf16", _lib.ptr(ctx_f), 1, 1, Rl, d, Rl * d, 0, d,
                  _lib.ptr(pk.Wf), d, d * d, d, _lib.ptr(pk.bf), d, 0, 0, 0, 1, _lib.ptr(part),
                  int(self.out_dtype == torch.float32), Rl * d, 0, d, 0, 0, 0, 0, st)
        if out is None:
            out = torch.empty(R, d, device=dev, dtype=self.out_dtype)
        wk = comm.all_gather_into_tensor(out.view(R, d), part, group=self.process_group,
                                         async_op=async_op)
        self._log("AllGather", "forward", "dchag-final-out",
                  part.numel() * part.element_size())
        return out.view(B, 1, s, d), wk

    def exchange_finish(self, payload, B, out=None):
        """Position-split final layer: exchange_start + exchange_complete, synchronous.
        Same per-row math as gather() + finish()."""
        res, _ = self.exchange_complete(self.exchange_start(payload, B), out)
        return res

    def _forward_pipelined(self, images, pk, out, n):
        """tp > 1, device images: the batch in n chunks, so the all-to-all of chunk k runs on
        NCCL's stream while the slab kernels of chunk k+1 run (positions are independent:
        same results as one chunk)."""
        b = images.shape[0]
        bounds = [(k * b) // n for k in range(n + 1)]
        res = out if out is not None else torch.empty(b, 1, self.seq, self.model.embed,
                                                      device=images.device, dtype=self.out_dtype)
        states = []
        for k in range(n):
            pay = self.local_payload(images[bounds[k]:bounds[k + 1]], pk)
            states.append(self.exchange_start(pay, bounds[k + 1] - bounds[k], async_op=True))
        works = []
        for k in range(n):
            _, wk = self.exchange_complete(states[k], out=res[bounds[k]:bounds[k + 1]],
                                           async_op=True)
            works.append(wk)
        for wk in works:
            wk.wait()
        return res

    def local_payload(self, img, pk=None, direct_out=None, vit=None):
        """Rank-local part: slab tree -> root payload [V bf16 R*D | L fp32 R*H] (bytes),
        V/L = the root stream projected into the final layer's value/logit space."""
        pk = pk or self.prepare()
        m = self.model
        d, h, s, p = m.embed, m.heads, self.seq, m.patch
        B = img.shape[0]
        R = B * s
        dev = img.device
        st = _lib.stream_handle()
        bf16 = dict(device=dev, dtype=torch.bfloat16)
        f32 = dict(device=dev, dtype=torch.float32)
        isb, isc = img.stride(0), img.stride(1)

        # ---- level 0
        if pk.attn_l0:
            poff_list, acc = [], 0
            for g in pk.l0_g_list:
                poff_list.append(acc)
                acc += g * R * h
            poff = self.dev_table(poff_list, torch.int64, dev)  # made once: no per-call H2D
            pbuf = torch.empty(acc, **bf16)
            # unnormalised e + 1/sum: K_l0 scales its accumulator (one exp per logit)
            pinv = torch.empty(pk.n0, R, h, **f32)
            _lib.call("dchag_l0_logits", _lib.ptr(img), isb, isc, B, m.image_h, m.image_w, p,
                      h, pk.HP, pk.NH, pk.n0, max(pk.l0_g_list), _lib.ptr(pk.l0_c0), _lib.ptr(pk.l0_g),
                      _lib.ptr(poff),
                      _lib.ptr(pk.WUt), _lib.ptr(pk.bU), _lib.ptr(pk.posU), _lib.ptr(pbuf),
                      _lib.ptr(pinv), st)
            prow = 1
        else:
            poff = (pk.l0_c0.to(torch.int64) * h).contiguous()
            pbuf = pk.p_const
            pinv = None
            prow = 0
        ctx = torch.empty(pk.n0, R, d, **bf16)
        _lib.call("dchag_l0_node", _lib.ptr(img), isb, isc, B, m.image_h, m.image_w, p, h, d,
                  pk.n0, _lib.ptr(pk.l0_c0), _lib.ptr(pk.l0_g), _lib.ptr(poff), prow,
                  _lib.ptr(pbuf), _lib.ptr(pinv), _lib.ptr(pk.Mt), pk.C_pad, _lib.ptr(pk.Et), pk.KE,
                  _lib.ptr(pk.posV0),
                  _lib.ptr(ctx), st)

        depth = len(pk.levels)
        payload = None
        for li in range(depth):
            n_l = len(pk.levels[li])
            N = pk.N[li]
            logits = N > d
            if self._fused_level(pk, li, R):
                # the children's logits for their parent (a thin GEMM over the logit rows of
                # the folded weights), then projection + softmax-weighted child sum in one
                # K_gemm (COMB): the child values never reach memory
                n_next = len(pk.levels[li + 1])
                Lpre = torch.empty(n_l, R, h, **f32)
                _lib.call("dchag_gemm_bf16", _lib.ptr(ctx), n_l, 1, R, d, R * d, 0, d,
                          _lib.ptr(pk.Wp[li][:, d:]), h, N * d, 0,
                          _lib.ptr(pk.bp[li][:, d:]), N, 0, 0, 0, 1, 0, 0, 0, 0, 0,
                          _lib.ptr(Lpre), R * h, 0, h, st)
                n_next = len(pk.levels[li + 1])
                _lib.call("dchag_child_softmax", _lib.ptr(Lpre), _lib.ptr(pk.comb_first[li]),
                          _lib.ptr(pk.comb_g[li]), n_next, R, h, st)
                # few parents -> few, long work units: split each parent's children in two
                # halves (partial sums under the full softmax) when that evens out the waves
                units = n_next * (R // 256) * (d // 256)
                split = 2 if (units < 5 * 74 and min(pk.levels[li + 1]) >= 2
                              and self.combine_split) else 1
                nxt = torch.empty(split, n_next, R, d, **bf16)
                _lib.call("dchag_gemm_combine", _lib.ptr(ctx), n_l, R, d, h, _lib.ptr(pk.Wp[li]),
                          N * d, _lib.ptr(pk.bp[li]), N, _lib.ptr(Lpre),
                          _lib.ptr(pk.comb_first[li]), _lib.ptr(pk.comb_g[li]), n_next, split,
                          _lib.ptr(nxt), st)
                ctx = nxt[0] if split == 1 else torch.add(nxt[0], nxt[1])
                continue
            if li == depth - 1 and direct_out is not None and vit is not None:
                # ... with the trunk-input epilogue (vit_input)
                self._final_vit(ctx, pk.Wdir, pk.bdir, B, direct_out, vit)
                return None
            if li == depth - 1 and direct_out is not None:
                # tp == 1: the root projection folded with the final layer writes the output
                _lib.call("dchag_gemm_bf16", _lib.ptr(ctx), 1, 1, R, d, R * d, 0, d,
                          _lib.ptr(pk.Wdir), d, d * d, d, _lib.ptr(pk.bdir), d, 0, 0, 0, 1,
                          _lib.ptr(direct_out), int(direct_out.dtype == torch.float32), R * d,
                          0, d, 0, 0, 0, 0, st)
                return None
            if li == depth - 1:
                # root: write straight into the gather payload (payload.py layout)
                payload = torch.empty(payload_nbytes(R, d, h), device=dev, dtype=torch.uint8)
                V, L = views(payload, R, d, h)
                V, L = V.view(1, R, d), L.view(1, R, h)
            else:
                V = torch.empty(n_l, R, d, **bf16)
                L = torch.empty(n_l, R, h, **f32) if logits else None
            rb = None  # level 0's positional term is added by K_l0 (posV0)
            _lib.call("dchag_gemm_bf16", _lib.ptr(ctx), n_l, 1, R, d, R * d, 0, d,
                      _lib.ptr(pk.Wp[li]), N, N * d, d, _lib.ptr(pk.bp[li]), N, _lib.ptr(rb),
                      s * N, N, s, _lib.ptr(V), 0, R * d, 0, d, _lib.ptr(L), R * h, 0, h, st)
            if li + 1 < depth:
                n_next = len(pk.levels[li + 1])
                ctx = torch.empty(n_next, R, d, **bf16)
                mix = pk.comb_mix[li]
                _lib.call("dchag_combine", n_next, R, d, h, _lib.ptr(pk.comb_first[li]),
                          _lib.ptr(pk.comb_g[li]), max(pk.levels[li + 1]), _lib.ptr(V), R * d,
                          _lib.ptr(None if mix is not None else L), R * h, _lib.ptr(mix),
                          _lib.ptr(ctx), st)
        return payload

    def finish(self, gathered, B, out=None, vit=None):
        """Shared final layer over the gathered streams -> [B, 1, S, D]."""
        pk = self.prepare()
        m = self.model
        d, h, s = m.embed, m.heads, self.seq
        R = B * s
        dev = gathered.device
        st = _lib.stream_handle()
        bf16 = dict(device=dev, dtype=torch.bfloat16)
        pb = gathered.numel() // self.tp
        if pb != payload_nbytes(R, d, h):
            raise ConfigError(f"gathered payload of {gathered.numel()} bytes does not match "
                              f"tp={self.tp}, B={B}")
        Vg = gathered.view(torch.bfloat16)
        Lg = gathered.view(torch.float32)
        if self.tp > 1:
            ctx_f = torch.empty(1, R, d, **bf16)
            first = self._final_first(dev)
            _lib.call("dchag_combine", 1, R, d, h, _lib.ptr(first[0]), _lib.ptr(first[1]),
                      self.tp, _lib.ptr(Vg), pb // 2, _lib.ptr(Lg[R * d // 2:]), pb // 4, 0,
                      _lib.ptr(ctx_f), st)
        else:
            ctx_f = Vg[:R * d].view(1, R, d)  # softmax over one stream is exactly 1
        if out is None:
            out = torch.empty(R, d, device=dev, dtype=self.out_dtype)
        if self.strategy.final_layer_tp_split and self.tp > 1:
            return self._finish_head_split(ctx_f, B, out)
        if vit is not None:
            self._final_vit(ctx_f, pk.Wf, pk.bf, B, out, vit)
            return out
        _lib.call("dchag_gemm_bf16", _lib.ptr(ctx_f), 1, 1, R, d, R * d, 0, d, _lib.ptr(pk.Wf),
                  d, d * d, d, _lib.ptr(pk.bf), d, 0, 0, 0, 1, _lib.ptr(out),
                  int(self.out_dtype == torch.float32), R * d, 0, d, 0, 0, 0, 0, st)
        return out.view(B, 1, s, d)

    def _finish_head_split(self, ctx_f, B, out):
        """final_layer_tp_split (strategies.py:211-215, layers.py:102-122 with TpHooks): this
        rank owns heads [r H/tp, (r+1) H/tp); its partial output ctx[:, own columns] @
        wo[own rows] (+ bo on rank 0) is summed over the tp group (the reference's allsum =
        ReduceScatter + AllGather, one NCCL all-reduce here)."""
        pk = self.prepare()
        m = self.model
        d, s = m.embed, self.seq
        R = B * s
        dev = ctx_f.device
        kc = d // self.tp
        c0 = self.rank * kc
        wf_loc, b_loc = self._head_split_weights(pk)
        part = torch.empty(R, d, device=dev, dtype=torch.float32)
        a = ctx_f.view(R, d)[:, c0:]                                # K = D/tp columns, row stride D
        _lib.call("dchag_gemm_bf16", _lib.ptr(a), 1, 1, R, kc, R * d, 0, d, _lib.ptr(wf_loc),
                  d, d * kc, d, _lib.ptr(b_loc), d, 0, 0, 0, 1, _lib.ptr(part), 1, R * d, 0, d,
                  0, 0, 0, 0, _lib.stream_handle())
        comm.all_reduce(part, group=self.process_group)
        self._log("AllReduce", "forward", "agg-final", (part.numel(), part.element_size()))
        out.copy_(part.view_as(out))
        return out.view(B, 1, s, d)

    def _head_split_weights(self, pk, refresh=False):
        """This rank's column shard of the folded final projection and its bias share
        (bo on rank 0 only). Kept on the packed rank, so a refold updates it in place."""
        kc = self.model.embed // self.tp
        c0 = self.rank * kc
        wf_loc = pk.Wf[:, c0:c0 + kc]                              # [D_out][D/tp] n-major
        if pk.head_split is None:
            pk.head_split = (wf_loc.contiguous(),
                             pk.bf.clone() if self.rank == 0 else torch.zeros_like(pk.bf))
        elif refresh:
            pk.head_split[0].copy_(wf_loc)
            if self.rank == 0:
                pk.head_split[1].copy_(pk.bf)
        return pk.head_split

    @staticmethod
    def combine_overflowed(reset: bool = True) -> bool:
        """Range guard of the fused level kernel (dchag_gemm_combine keeps its running child
        sum as fp16 x 2^8, range +-1.68e7): True if any forward since the last reset produced
        a partial sum outside that range (its output then holds inf). Synchronises the
        device; DCHAG_FUSE_COMBINE=0 selects the unfused levels, which have no such limit."""
        import ctypes
        flag = ctypes.c_int(0)
        _lib.call("dchag_combine_overflow", ctypes.byref(flag), int(reset))
        return bool(flag.value)

    def dev_table(self, vals, dtype, dev):
        """A small host-known index table on the device, made once per content: a forward
        (or a CUDA-graph capture) never issues a pageable H2D copy, which would synchronise
        the stream."""
        key = ("table", tuple(int(v) for v in vals), dtype, str(dev))
        cache = self.__dict__.setdefault("_cache", {})
        t = cache.get(key)
        if t is None:
            t = cache[key] = torch.tensor(key[1], device=dev, dtype=dtype)
        return t

    def _final_first(self, dev):
        return (self.dev_table([0], torch.int32, dev),
                self.dev_table([self.tp], torch.int32, dev))
