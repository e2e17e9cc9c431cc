"""Summarise an ncu report (raw page) into the numbers the roofline needs."""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time_ns",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__mem_tensor_writes_op_stt.sum.pct_of_peak_sustained_elapsed": "tmem_st_pct",
    "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed": "tmem_ld_pct",
}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    for r in rows[2:]:
        out = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for k, name in KEYS.items():
            if k in hdr:
                out[name] = r[hdr.index(k)]
        stalls = []
        for i in stall_cols:
            try:
                stalls.append((float(r[i].replace(",", "")),
                               hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        stalls.sort(reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        out["top_stalls(pc-sample %)"] = [f"{n}={100 * v / tot:.0f}" for v, n in stalls[:7]]
        print(out)


if __name__ == "__main__":
    main(sys.argv[1])
