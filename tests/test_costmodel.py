"""The reference cost model (costmodel.py:191-319) against this implementation's own accounting
(SURVEY.md f4), on the committed estimate fixture (tests/golden/costmodel.json, written by
make_costmodel_fixture.py from the reference itself).

Exact integer contracts: per-rank parameter bytes of the front end (tokenize + aggregate; the
reference's tokenize row also counts the trunk's metadata projection, 4D + D) and the
collective payloads of one step (boundary AllGather, shared special.pos gradient) in the
reference's ring accounting (ledger.py). The activation-memory side (the reference engine
materialises tokens; this one does not) is measured on the GPU by
tools/costmodel_validate.py (profiles/r02/costmodel_validate.json)."""
import json
import os

import pytest

from paper_2506_21411_b200 import ledger as LG
from paper_2506_21411_b200.config import ModelConfig, StrategyConfig, channel_slabs
from paper_2506_21411_b200.frontend import frontend_param_specs

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "costmodel.json")
CASES = json.load(open(FIX))


def _numel(shape):
    n = 1
    for s in shape:
        n *= s
    return n


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("pb", [2, 4, 8])
def test_param_bytes_match_cost_model(name, pb):
    cfg = CASES[name]["config"]
    est = CASES[name]["estimate"][str(pb)]
    c, d, tp = cfg["channels"], cfg["embed"], cfg["tp"]
    model = ModelConfig(channels=c, image_h=cfg["image_h"], image_w=cfg["image_w"],
                        patch=cfg["patch"], embed=d, heads=cfg["heads"],
                        agg_layer_kind=cfg["layer_kind"])
    strat = StrategyConfig(kind="dchag", tp_degree=tp, max_group=cfg["max_group"],
                           agg_layer_kind=cfg["layer_kind"], uneven_slabs=True)
    specs = frontend_param_specs(model, strat)
    cloc = max(n for _, n in channel_slabs(c, tp))   # the cost model rounds slabs up
    rank = 0                                          # rank 0 owns a largest slab
    tok = sum(_numel(s) for n, s, _ in specs if n in ("tok.w", "tok.b", "special.channel_id"))
    tok = tok // c * cloc + _numel([s for n, s, _ in specs if n == "special.pos"][0])
    agg = sum(_numel(s) for n, s, _ in specs if n.startswith(f"agg.slab{rank}.")
              or n.startswith("agg.final."))
    assert est["components"]["tokenize"]["params_bytes"] == (tok + 5 * d) * pb
    assert est["components"]["aggregate"]["params_bytes"] == agg * pb


@pytest.mark.parametrize("name", sorted(CASES))
def test_comm_bytes_match_cost_model(name):
    cfg = CASES[name]["config"]
    est = CASES[name]["estimate"]["2"]["comm"]
    b, d, tp = cfg["batch"], cfg["embed"], cfg["tp"]
    s = (cfg["image_h"] // cfg["patch"]) * (cfg["image_w"] // cfg["patch"])
    # boundary AllGather of each rank's [B,1,S,D] stream at 2-byte precision
    assert est["forward:tp"] == LG.allgather_payload(b * s * d * 2, tp)
    # shared special.pos gradient all-reduce (strategies.py:251-264), only when tp > 1
    assert est.get("optimizer:tp", 0) == (LG.allreduce_payload(s * d, 2, tp) if tp > 1 else 0)
