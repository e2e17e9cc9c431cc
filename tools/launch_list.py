"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of bench.py into the
per-kernel share table (profiles/*_ncu_launches_*.txt). Only this repo's kernels count."""
import csv
import sys
from collections import OrderedDict

OURS = ("l0_node_kernel", "gemm_kernel", "l0_logits_kernel", "combine_kernel", "vit_tokens",
        "l0_dv_kernel", "combine_bwd_kernel", "unfold_kernel", "fullcross_weights",
        "combine_f32_kernel", "tile_weights_kernel")


def base(name):
    n = name.split("(")[0].replace("void ", "")
    n = n.split("<")[0]
    return n.split("::")[-1]


def main(path, title):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    seq = [(base(r[ki]), float(r[vi].replace(",", "")) / 1e3) for r in rows[h + 1:]
           if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    seq = [(k, us) for k, us in seq if k in OURS and k != "tile_weights_kernel"]
    agg = OrderedDict()
    for k, us in seq:
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values())
    print(title)
    print(f"{'kernel':20s} {'launches':>9s} {'total_us':>10s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:20s} {n:9d} {t:10.1f} {100 * t / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "# ncu launch list")
