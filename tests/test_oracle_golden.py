"""Pin the numpy oracle (oracle/dchag_oracle.py) to golden vectors produced by the
reference itself (tests/golden/make_golden.py) and to the reference's brute-force
layer oracle (pkg/tests/test_model.py:78-97)."""
import numpy as np
import pytest

import dchag_oracle as O
from conftest import load_golden, rel_err

CASES = ["ref_tiny_sq_tp2", "ref_tiny_lin_tp2", "ref_tiny_fc_tp2", "ref_tiny_sq_tp1_g3",
         "T_sq_tp1", "T_sq_tp2"]


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference_golden(case):
    meta, z, w, _ = load_golden(case)
    images = z["images"].astype(np.float64)
    out, gathered = O.dchag_frontend(images, w, patch=meta["patch"], heads=meta["heads"],
                                     tp=meta["tp"], max_group=meta["max_group"],
                                     variant=meta["variant"], layer_kind=meta["layer_kind"],
                                     return_streams=True)
    tol = 1e-12 if z["out"].dtype == np.float64 else 1e-6
    assert rel_err(out, z["out"]) < tol
    assert rel_err(gathered, z["gathered"]) < tol


@pytest.mark.parametrize("case", CASES)
def test_tree_levels_match_reference(case):
    meta, z, _, _ = load_golden(case)
    per_rank = meta["channels"] // meta["tp"]
    assert repr(O.build_levels(per_rank, meta["max_group"])) == str(z["levels"])


def test_single_query_matches_bruteforce():
    rng = np.random.default_rng(5)
    d, heads, c = 8, 2, 3
    w = {f"n.{k}": rng.standard_normal((d, d)) * 0.3 for k in ("wq", "wk", "wv", "wo")}
    w["n.q"] = rng.standard_normal(d)
    w["n.bo"] = rng.standard_normal(d) * 0.1
    tokens = rng.standard_normal((2, c, 5, d))
    got = O.flat_aggregate(tokens, w, "n", "single_query", heads)
    want = O.brute_force_single_query(tokens, w["n.q"], w["n.wq"], w["n.wk"], w["n.wv"],
                                      w["n.wo"], w["n.bo"], heads)
    assert rel_err(got, want) < 1e-12


def test_unfold_layout():
    x = np.arange(2 * 8 * 12, dtype=np.float64).reshape(1, 2, 8, 12)
    p = O.unfold_patches(x, 4)
    assert p.shape == (1, 2, 6, 16)
    # token s = i*wp + j, pixel k = py*P + px (tensor.py:303-323)
    i, j, py, px = 1, 2, 3, 1
    assert p[0, 1, i * 3 + j, py * 4 + px] == x[0, 1, i * 4 + py, j * 4 + px]


def test_vit_input_restatement_matches_reference():
    """oracle.vit_input vs the reference apply_token_mask + vit_forward's input assembly
    (model.py:100-117), run here from /root/reference (depth-0 trunk returns its input)."""
    import os
    import sys
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference tree not mounted")
    sys.path.insert(0, ref)
    try:
        from dchag.config import ModelConfig
        from dchag.model import apply_token_mask, vit_forward
        from dchag.tensor import Tensor
    finally:
        sys.path.remove(ref)
    rng = np.random.default_rng(3)
    B, S, D = 2, 16, 8
    agg = rng.standard_normal((B, 1, S, D))
    mask = (rng.random((B, S)) < 0.5).astype(np.float64)
    mtok, meta = rng.standard_normal(D), rng.standard_normal((B, 4))
    mw, mb = rng.standard_normal((4, D)), rng.standard_normal(D)
    model = ModelConfig(channels=2, image_h=16, image_w=16, patch=4, embed=D, heads=2,
                        depth=0, decoder_depth=0, decoder_dim=8)
    x = apply_token_mask(Tensor(agg), mask, Tensor(mtok))
    ref_out = vit_forward(x, Tensor(meta), {"special.meta_w": Tensor(mw),
                                            "special.meta_b": Tensor(mb)}, model)
    want = np.asarray(ref_out.data)
    got = O.vit_input(agg, mask, mtok, meta, mw, mb)
    assert np.allclose(got, want, rtol=0, atol=1e-12)
