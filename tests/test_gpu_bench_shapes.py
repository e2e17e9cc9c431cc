"""GPU parity at the exact shapes bench.py measures.

The GPU runs the benchmarked kernel instantiation in full (every channel, every tree node,
the full image); the CPU oracle (float64, oracle/dchag_oracle.py) is evaluated on the first
patch rows of the same images with the same weights and compared with those rows of the GPU
output. Positions are independent on this path (every op before the trunk is per (b, s):
model.py:51-64 tokenizer, layers.py:103-123 nodes over the channel axis, model.py:180-201),
so the crop changes nothing but the oracle's cost.

  H1  C500 128x128 P8 D1024 H16, max_group 16: groups of 16, 32 level-0 nodes, depth 3
      (also with D-CHAG-L linear nodes and with full_cross nodes)
  W   C128 128x256 P4 D1024 H16, max_group 64: KE = 64, S = 2048
  H8  C500 over 8 slabs (63 x4, 62 x4), max_group 4, all ranks in one process
  TR  fwd+bwd at D2048 H32 on a 24-channel slab with the TR tree (groups of 4, depth 3)
bf16 budget: rel_err <= 2e-2 (tests/conftest.py rel_err, the reference metric).
"""
import numpy as np
import pytest
import torch

import dchag_oracle as O
import torch_reference as TR
from conftest import rel_err

pytestmark = pytest.mark.gpu
BF16_TOL = 2e-2


def _master(fe, seed, bias_std=0.02):
    """Reference-named weights (truncated normal 0.02, per-name seeded so every rank agrees),
    with small random biases so the bias paths are exercised."""
    master = fe.init_weights(seed=seed)
    g = torch.Generator(device=fe.device).manual_seed(seed + 1)
    for k, v in master.items():
        if k in ("tok.b",) or k.endswith(".bo") or k.endswith(".b"):
            v.copy_(torch.randn(v.shape, generator=g, device=v.device) * bias_std)
    return master


def _frontends(cfg, tp, out_dtype=torch.float32):
    from paper_2506_21411_b200 import DchagFrontEnd
    return [DchagFrontEnd(cfg["channels"], cfg["image_h"], cfg["image_w"], cfg["patch"],
                          cfg["embed"], cfg["heads"], max_group=cfg["max_group"], tp=tp, rank=r,
                          out_dtype=out_dtype,
                          agg_layer_kind=cfg.get("layer_kind", "cross_attention"),
                          agg_variant=cfg.get("variant", "single_query"))
            for r in range(tp)]


def _gpu_forward(fes, master, img):
    """All tp ranks in one process: per-rank root payloads concatenated in rank order (the
    AllGather, runtime.py:259), then the shared final layer (strategies.py:216-218). tp = 1
    goes through the public forward (root projection folded with the final layer)."""
    tp = len(fes)
    for fe in fes[1:]:
        fe.load_weights(master)
    if tp == 1:
        return fes[0](img)
    pays = [fe.local_payload(img[:, fe.slab[0]:fe.slab[0] + fe.slab[1]]) for fe in fes]
    return fes[0].finish(torch.cat(pays), img.shape[0])


def _oracle_rows(cfg, master, img, tp, rows):
    """The float64 oracle on the first `rows` patch rows of every image."""
    P = cfg["patch"]
    wp = cfg["image_w"] // P
    w = {k: v.detach().float().cpu().numpy() for k, v in master.items()}
    w["special.pos"] = w["special.pos"][:rows * wp]
    x = img[:, :, :rows * P].float().cpu().numpy().astype(np.float64)
    return O.dchag_frontend(x, w, patch=P, heads=cfg["heads"], tp=tp,
                            max_group=cfg["max_group"],
                            layer_kind=cfg.get("layer_kind", "cross_attention"),
                            variant=cfg.get("variant", "single_query"))


SHAPES = {
    "H1": (dict(channels=500, image_h=128, image_w=128, patch=8, embed=1024, heads=16,
                max_group=16), 1, 2, 2),
    "H1_linear": (dict(channels=500, image_h=128, image_w=128, patch=8, embed=1024, heads=16,
                       max_group=16, layer_kind="linear"), 1, 2, 2),
    "H1_fullcross": (dict(channels=500, image_h=128, image_w=128, patch=8, embed=1024,
                          heads=16, max_group=16, variant="full_cross"), 1, 2, 2),
    "W": (dict(channels=128, image_h=128, image_w=256, patch=4, embed=1024, heads=16,
               max_group=64), 1, 2, 1),
    "H2": (dict(channels=500, image_h=128, image_w=128, patch=8, embed=1024, heads=16,
                max_group=8), 2, 2, 1),
    "H8": (dict(channels=500, image_h=128, image_w=128, patch=8, embed=1024, heads=16,
                max_group=4), 8, 2, 1),
}


@pytest.mark.parametrize("name", list(SHAPES))
def test_benchmarked_shape_matches_oracle(name):
    cfg, tp, B, rows = SHAPES[name]
    fes = _frontends(cfg, tp)
    if name == "H1":
        assert fes[0].tree.levels[0] == (16,) * 20 + (15,) * 12   # groups of 16, 32 nodes
        assert fes[0].tree.depth == 3
    if name == "W":
        assert fes[0].tree.levels == ((64, 64), (2,))
    if name == "H8":
        assert [f.slab[1] for f in fes] == [63] * 4 + [62] * 4
        assert all(f.tree.depth == 3 for f in fes)
    master = _master(fes[0], seed=7)
    gen = torch.Generator(device="cuda").manual_seed(3)
    img = torch.randn(B, cfg["channels"], cfg["image_h"], cfg["image_w"], device="cuda",
                      generator=gen).to(torch.bfloat16)
    out = _gpu_forward(fes, master, img)
    torch.cuda.synchronize()
    assert out.shape == (B, 1, fes[0].seq, cfg["embed"])
    assert torch.isfinite(out).all()
    want = _oracle_rows(cfg, master, img, tp, rows)
    got = out[:, :, :want.shape[2]].float().cpu().numpy()
    err = rel_err(got, want)
    assert err < BF16_TOL, (name, err)


def test_train_TR_slab_fwd_bwd_matches_autograd():
    """TR (D 2048, H 32, P8 128x128) forward + backward on a 24-channel slab whose tree has
    the TR slab's structure (groups of <= 4, depth 3: (4 x6), (3, 3), (2,)), against float64
    torch autograd of the reference restatement (tests/torch_reference.py)."""
    from paper_2506_21411_b200.train import DchagTrainer
    cfg = dict(channels=24, image_h=128, image_w=128, patch=8, embed=2048, heads=32,
               max_group=4)
    fe = _frontends(cfg, 1)[0]
    assert fe.tree.levels == ((4,) * 6, (3, 3), (2,))
    master = _master(fe, seed=11)
    gen = torch.Generator(device="cuda").manual_seed(5)
    img = torch.randn(1, 24, 128, 128, device="cuda", generator=gen).to(torch.bfloat16)
    probe = torch.randn(1, 1, fe.seq, 2048, device="cuda", generator=gen)
    tr = DchagTrainer(fe)
    out, saved = tr.forward_train(img)
    grads = tr.backward(saved, probe)
    torch.cuda.synchronize()
    w = {k: v.double().cpu().numpy() for k, v in master.items()}
    out_ref, g_ref = TR.grads(img.double().cpu().numpy(), w, probe.double().cpu().numpy(),
                              patch=8, heads=32, tp=1, max_group=4)
    assert rel_err(out.double().cpu().numpy(), out_ref) < BF16_TOL
    bad = {k: rel_err(grads[k].double().cpu().numpy(), g_ref[k]) for k in g_ref}
    worst = max(bad.values())
    assert worst < BF16_TOL, sorted(bad.items(), key=lambda kv: -kv[1])[:6]
