"""Generate golden vectors for the D-CHAG front end from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

For every case it builds weights with the reference's `create_master`
(params.py:139-150, RngState Philox stream) and images with `make_batch`
(synthetic.py:39-45), runs the reference hot path exactly as
forward_loss_dchag_reference composes it (model.py:180-201: per-slab
tokenize_channels + tree_aggregate, concat in slab order, flat_aggregate
"agg.final"), and writes inputs, front-end weights and outputs to
tests/golden/<case>.npz.  Large cases store float32-rounded weights/images and
recompute the reference output from those rounded values (upcast to f64), so
the golden output is exact for the stored inputs.

Backward goldens: the gradient of sum(out * probe) w.r.t. every front-end
parameter via the reference tape (tensor.py:395-413), the pattern of
test_model.py:66-70.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from dchag import tensor as T  # noqa: E402
from dchag.config import ModelConfig, StrategyConfig  # noqa: E402
from dchag.model import flat_aggregate, tokenize_channels, tree_aggregate  # noqa: E402
from dchag.params import create_master, rank_tree  # noqa: E402
from dchag.rng import RngState  # noqa: E402
from dchag.synthetic import make_batch  # noqa: E402
from dchag.tensor import Tensor  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

FRONT = ("tok.", "special.channel_id", "special.pos", "agg.")


def hot_path(w, model, strategy, images):
    """model.py:180-201 composed from the reference's own functions."""
    tp = strategy.tp_degree
    cloc = model.channels // tp
    tree = rank_tree(model, strategy)
    img = Tensor(images)
    streams = []
    for r in range(tp):
        tok = tokenize_channels(T.narrow(img, 1, r * cloc, cloc),
                                T.narrow(w["tok.w"], 0, r * cloc, cloc),
                                T.narrow(w["tok.b"], 0, r * cloc, cloc),
                                T.narrow(w["special.channel_id"], 0, r * cloc, cloc),
                                w["special.pos"], model.patch)
        streams.append(tree_aggregate(tok, tree, w, f"agg.slab{r}", strategy.agg_layer_kind,
                                      model.agg_variant, model.heads))
    gathered = streams[0] if tp == 1 else T.concat(streams, axis=1)
    out = flat_aggregate(gathered, w, "agg.final", model.agg_variant, model.heads)
    return out, gathered


def make_case(name, *, channels, image, patch, embed, heads, tp, max_group, batch,
              variant="single_query", layer_kind="cross_attention", seed=0, round32=False,
              grads=False, bias_scale=0.0):
    model = ModelConfig(channels=channels, image_h=image[0], image_w=image[1], patch=patch,
                        embed=embed, depth=0, heads=heads, agg_variant=variant,
                        decoder_depth=0, decoder_dim=8)
    model.validate()
    strat = StrategyConfig(kind="dchag", tp_degree=tp, max_group=max_group,
                           agg_layer_kind=layer_kind, vit_tp_split=False)
    strat.validate(model)
    master = create_master(model, strat, RngState(seed))
    master = {k: v for k, v in master.items() if k.startswith(FRONT)}
    if bias_scale:
        # exercise the bias paths (create_master zero-initialises biases)
        brng = RngState(seed + 100)
        for k in sorted(master):
            if k.endswith((".bo", ".b")) or k == "tok.b":
                master[k] = brng.normal(master[k].shape, bias_scale)
    images = make_batch(model, 11, 0, list(range(batch))).images
    if round32:
        master = {k: v.astype(np.float32).astype(np.float64) for k, v in master.items()}
        images = images.astype(np.float32).astype(np.float64)
    w = {k: Tensor(v, requires_grad=grads) for k, v in master.items()}
    out, gathered = hot_path(w, model, strat, images)
    payload = {"images": images, "out": out.data, "gathered": gathered.data,
               "levels": np.array(repr(rank_tree(model, strat).levels))}
    if grads:
        probe = RngState(seed + 7).normal(out.shape)
        loss = T.sum_all(T.mul(out, Tensor(probe)))
        T.backward(loss)
        payload["probe"] = probe
        for k, t in w.items():
            payload["grad:" + k] = t.grad if t.grad is not None else np.zeros(t.shape)
    for k, v in master.items():
        payload["w:" + k] = v
    meta = dict(channels=channels, image_h=image[0], image_w=image[1], patch=patch,
                embed=embed, heads=heads, tp=tp, max_group=max_group, batch=batch,
                variant=variant, layer_kind=layer_kind, seed=seed)
    payload["meta"] = np.array(repr(meta))
    dt = np.float32 if round32 else np.float64
    payload = {k: (v.astype(dt) if isinstance(v, np.ndarray) and v.dtype == np.float64 else v)
               for k, v in payload.items()}
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **payload)
    print(f"{name}: out {out.shape} -> {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def main():
    # reference-scale tiny cases (test_strategies.py:15-22 shapes), float64, with grads
    make_case("ref_tiny_sq_tp2", channels=8, image=(8, 8), patch=4, embed=8, heads=4,
              tp=2, max_group=2, batch=2, seed=6, grads=True, bias_scale=0.05)
    make_case("ref_tiny_lin_tp2", channels=8, image=(8, 8), patch=4, embed=8, heads=4,
              tp=2, max_group=2, batch=2, layer_kind="linear", seed=6, grads=True,
              bias_scale=0.05)
    make_case("ref_tiny_fc_tp2", channels=8, image=(8, 8), patch=4, embed=8, heads=2,
              tp=2, max_group=4, batch=1, variant="full_cross", seed=3, grads=True)
    make_case("ref_tiny_sq_tp1_g3", channels=10, image=(8, 8), patch=4, embed=8, heads=2,
              tp=1, max_group=4, batch=2, seed=9, grads=True, bias_scale=0.05)
    # GPU-shaped case (the "T" config of SURVEY section 8(d)): float32-rounded inputs
    make_case("T_sq_tp1", channels=16, image=(64, 64), patch=4, embed=128, heads=2,
              tp=1, max_group=8, batch=1, seed=0, round32=True, bias_scale=0.02)
    make_case("T_sq_tp2", channels=16, image=(64, 64), patch=4, embed=128, heads=2,
              tp=2, max_group=4, batch=1, seed=1, round32=True, bias_scale=0.02)
    # GPU-shaped training cases: gradients of sum(out * probe) through the front end
    make_case("Tg_sq_tp1", channels=8, image=(64, 32), patch=4, embed=128, heads=2,
              tp=1, max_group=4, batch=1, seed=2, round32=True, grads=True, bias_scale=0.02)
    make_case("Tg_sq_tp2", channels=8, image=(64, 32), patch=4, embed=128, heads=2,
              tp=2, max_group=2, batch=1, seed=3, round32=True, grads=True, bias_scale=0.02)
    make_case("Tg_lin_tp2", channels=8, image=(64, 32), patch=4, embed=128, heads=2,
              tp=2, max_group=2, batch=1, layer_kind="linear", seed=4, round32=True, grads=True,
              bias_scale=0.02)
    # full_cross training cases (agg_variant="full_cross": nodes and the final layer)
    make_case("Tg_fc_tp1", channels=8, image=(64, 32), patch=4, embed=128, heads=2,
              tp=1, max_group=4, batch=1, variant="full_cross", seed=5, round32=True,
              grads=True, bias_scale=0.02)
    make_case("Tg_fc_tp2", channels=8, image=(64, 32), patch=4, embed=128, heads=2,
              tp=2, max_group=2, batch=1, variant="full_cross", seed=6, round32=True,
              grads=True, bias_scale=0.02)


if __name__ == "__main__":
    main()
