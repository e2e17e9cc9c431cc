"""Measured device memory of the B200 front end against the reference cost model
(costmodel.py:191-319; the per-rank estimate is committed in tests/golden/costmodel.json by
tests/golden/make_costmodel_fixture.py). SURVEY.md f4.

For each config: parameter bytes (exact contract, also checked on CPU by
tests/test_costmodel.py), and the measured allocator peak above the resident weights for one
forward (and one training step for TR) against the model's activation (+ gradient) bytes at
2-byte precision. The reference engine materialises the token tensor and every node's
K/V; this path does not, so the measured/estimated ratio is the memory
the fused design saves. Prints one JSON document (profiles/r02/costmodel_validate.json)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_21411_b200 import DchagFrontEnd  # noqa: E402
from paper_2506_21411_b200.train import DchagTrainer  # noqa: E402

FIX = json.load(open(os.path.join(ROOT, "tests", "golden", "costmodel.json")))


def measure(name, train):
    cfg = FIX[name]["config"]
    est = FIX[name]["estimate"]["2"]["components"]
    torch.cuda.empty_cache()
    fe = DchagFrontEnd(cfg["channels"], cfg["image_h"], cfg["image_w"], cfg["patch"],
                       cfg["embed"], cfg["heads"], max_group=cfg["max_group"],
                       agg_layer_kind=cfg["layer_kind"])
    fe.init_weights(seed=0)
    params = sum(v.numel() for v in fe.weights.values())
    x = torch.randn(cfg["batch"], cfg["channels"], cfg["image_h"], cfg["image_w"],
                    device="cuda").to(torch.bfloat16)
    res = {"config": cfg, "params_elems": params,
           "ref_params_elems": (est["tokenize"]["params_bytes"] - 5 * cfg["embed"] * 2) // 2
           + est["aggregate"]["params_bytes"] // 2}
    ref_act = est["tokenize"]["activation_bytes"] + est["aggregate"]["activation_bytes"]
    if not train:
        fe.prepare()
        fe(x)
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        y = fe(x)
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base
        res.update(kind="forward", measured_peak_bytes=peak, ref_activation_bytes_bf16=ref_act,
                   ratio=peak / ref_act, output_bytes=y.numel() * y.element_size())
    else:
        tr = DchagTrainer(fe)
        probe = torch.randn(cfg["batch"], 1, fe.seq, cfg["embed"], device="cuda")
        out, saved = tr.forward_train(x)
        tr.backward(saved, probe)
        del out, saved
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        out, saved = tr.forward_train(x)
        grads = tr.backward(saved, probe)
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base
        ref = ref_act + est["tokenize"]["grad_bytes"] + est["aggregate"]["grad_bytes"]
        res.update(kind="train step", measured_peak_bytes=peak,
                   ref_activation_plus_grad_bytes_bf16=ref, ratio=peak / ref,
                   trainer_persistent_bytes=base)
        del grads
    return res


def main():
    out = {}
    for name, train in (("T", False), ("W", False), ("H1", False), ("H1_linear", False),
                        ("TR1", True)):
        out[name] = measure(name, train)
        print(name, json.dumps({k: v for k, v in out[name].items() if k != "config"}),
              file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
