"""Writes tests/golden/costmodel.json: the reference cost model's per-rank estimate
(/root/reference/pkg/src/dchag/costmodel.py:191-319, `estimate`) for the front-end
components (tokenize, aggregate) and communication at the SURVEY.md section 8(d) configs.
Run in the container that has /root/reference (it is test infrastructure; the GPU box uses
the committed JSON):  python tests/golden/make_costmodel_fixture.py"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from dchag import costmodel as CM  # noqa: E402
from dchag.config import ModelConfig, StrategyConfig  # noqa: E402

CASES = {
    # name: (C, H, W, P, D, heads, tp, max_group, batch, layer_kind)
    "H1": (500, 128, 128, 8, 1024, 16, 1, 16, 32, "cross_attention"),
    "H2": (500, 128, 128, 8, 1024, 16, 2, 8, 32, "cross_attention"),
    "H4": (500, 128, 128, 8, 1024, 16, 4, 8, 32, "cross_attention"),
    "TR1": (500, 128, 128, 8, 2048, 32, 1, 16, 32, "cross_attention"),
    "TR2": (500, 128, 128, 8, 2048, 32, 2, 8, 32, "cross_attention"),
    "W": (128, 128, 256, 4, 1024, 16, 1, 64, 16, "cross_attention"),
    "H1_linear": (500, 128, 128, 8, 1024, 16, 1, 16, 32, "linear"),
    "T": (16, 64, 64, 4, 128, 2, 1, 8, 2, "cross_attention"),
}


def main():
    out = {}
    for name, (c, h, w, p, d, heads, tp, g, b, lk) in CASES.items():
        model = ModelConfig(channels=c, image_h=h, image_w=w, patch=p, embed=d, heads=heads,
                            depth=0, decoder_depth=0, decoder_dim=8, agg_variant="single_query")
        strat = StrategyConfig(kind="dchag", tp_degree=tp, max_group=g, agg_layer_kind=lk)
        per_pb = {}
        for pb in (2, 4, 8):
            rep = CM.estimate(model, strat, precision_bytes=pb, batch=b)
            comp = {k: {"params_bytes": int(v.params_bytes),
                        "activation_bytes": int(v.activation_bytes),
                        "grad_bytes": int(v.grad_bytes), "flops": int(v.flops)}
                    for k, v in rep.components.items() if k in ("tokenize", "aggregate")}
            per_pb[str(pb)] = {"components": comp,
                               "comm": {f"{ph}:{ax}": int(v) for (ph, ax), v in rep.comm.items()}}
        out[name] = {"config": dict(channels=c, image_h=h, image_w=w, patch=p, embed=d,
                                    heads=heads, tp=tp, max_group=g, batch=b, layer_kind=lk),
                     "estimate": per_pb}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "costmodel.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(path)


if __name__ == "__main__":
    main()
