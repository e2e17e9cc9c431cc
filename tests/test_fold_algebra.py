"""The folded execution plan (fold.py + the kernels' arithmetic, emulated in float64
torch on CPU) reproduces the reference hot path (model.py:180-201) -- pins the
algebra of the fused B200 path independently of the CUDA code."""
import numpy as np
import pytest
import torch

import dchag_oracle as O
from conftest import load_golden, rel_err
from folded_emulator import emulate_frontend
from paper_2506_21411_b200.config import build_tree_spec, channel_slabs


def _run(meta, w, images, fold_root_final=False):
    tw = {k: torch.from_numpy(v) for k, v in w.items()}
    slabs = channel_slabs(meta["channels"], meta["tp"])
    trees = [build_tree_spec(n, meta["max_group"]).levels for _, n in slabs]
    return emulate_frontend(tw, torch.from_numpy(images), slabs=slabs, trees=trees,
                            embed=meta["embed"], heads=meta["heads"], patch=meta["patch"],
                            variant=meta["variant"], layer_kind=meta["layer_kind"],
                            fold_root_final=fold_root_final).numpy()


@pytest.mark.parametrize("case", ["ref_tiny_sq_tp2", "ref_tiny_lin_tp2", "ref_tiny_sq_tp1_g3",
                                  "T_sq_tp1", "T_sq_tp2"])
def test_folded_plan_matches_reference_golden(case):
    meta, z, w, _ = load_golden(case)
    out = _run(meta, w, z["images"].astype(np.float64))
    assert rel_err(out, z["out"]) < (1e-10 if z["out"].dtype == np.float64 else 1e-6)


@pytest.mark.parametrize("tp,layer_kind", [(3, "cross_attention"), (8, "cross_attention"),
                                           (3, "linear")])
def test_folded_plan_uneven_slabs(tp, layer_kind):
    # 22 channels over tp ranks: balanced slabs (extension), oracle composes per slab
    meta = dict(channels=22, image_h=16, image_w=16, patch=4, embed=16, heads=4, tp=tp,
                max_group=3, variant="single_query", layer_kind=layer_kind)
    specs = O.frontend_param_specs(22, 16, 16, 4, 16, tp, 3, layer_kind=layer_kind)
    w = O.random_params(specs, seed=3, std=0.2, bias_std=0.05)
    images = np.random.default_rng(1).standard_normal((2, 22, 16, 16))
    want = O.dchag_frontend(images, w, patch=4, heads=4, tp=tp, max_group=3,
                            layer_kind=layer_kind)
    assert rel_err(_run(meta, w, images), want) < 1e-10


@pytest.mark.parametrize("case", ["ref_tiny_sq_tp1_g3", "T_sq_tp1"])
def test_tp1_root_final_fold_matches_reference_golden(case):
    # the tp == 1 plan: root value projection and final layer as one GEMM (pack_rank Wdir)
    meta, z, w, _ = load_golden(case)
    out = _run(meta, w, z["images"].astype(np.float64), fold_root_final=True)
    assert rel_err(out, z["out"]) < (1e-10 if z["out"].dtype == np.float64 else 1e-6)
