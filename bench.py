"""D-CHAG tokenize+aggregate throughput on B200 (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload hyperspectral|weather|tiny]
  python bench.py --impl reference ...      # the reference CPU path on the host cores

A step is one forward of the channel front end (per-channel tokenizer + hierarchical
cross-channel aggregation + partial-aggregate AllGather + final layer) over one batch
of synthetic images of the named shape.  With N GPUs the channels are sharded over N
ranks exactly as D-CHAG's distributed tokenization does (tp = N architecture, balanced
slabs for 500 / 8); the batch is global, so the scaling is strong.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # SURVEY.md section 8(d) canonical instantiations (heads at dh = 64, max_group derived)
    "hyperspectral": dict(channels=500, image_h=128, image_w=128, patch=8, embed=1024,
                          heads=16, depth=3, batch=32),
    "weather": dict(channels=128, image_h=128, image_w=256, patch=4, embed=1024, heads=16,
                    depth=2, batch=16),
    "tiny": dict(channels=16, image_h=64, image_w=64, patch=4, embed=128, heads=2, depth=2,
                 batch=2),
    # training step (fwd+bwd), SURVEY.md section 8(d) "TR": C500 D2048 H32 (dh 64), bf16
    "train": dict(channels=500, image_h=128, image_w=128, patch=8, embed=2048, heads=32,
                  depth=3, batch=32, train=True, final_split=True),
    # the H1 config with the other node kinds: D-CHAG-L linear nodes (the
    # paper's best configuration) and full_cross (ModelConfig's default variant, tokens
    # materialised)
    "hyperspectral_linear": dict(channels=500, image_h=128, image_w=128, patch=8, embed=1024,
                                 heads=16, depth=3, batch=32, layer_kind="linear"),
    "hyperspectral_fullcross": dict(channels=500, image_h=128, image_w=128, patch=8,
                                    embed=1024, heads=16, depth=3, batch=32,
                                    variant="full_cross"),
    # the fp32 parity mode (BASELINE tolerance fp32 <= 1e-4) on the H1 shape: split-bf16
    # 3-term tcgen05 GEMMs, fp32 combines, tokens materialised in fp32
    "hyperspectral_fp32": dict(channels=500, image_h=128, image_w=128, patch=8, embed=1024,
                               heads=16, depth=3, batch=32, precision="fp32"),
}
# scaling sweep: C 64..1024 x D 1024 (16 heads) / 4096 (32 heads,
# dh = 128), 128x128 P8, B 32, max_group 16 with the depth derived per slab
for _c in (64, 128, 256, 512, 1024):
    for _d, _h in ((1024, 16), (4096, 32)):
        WORKLOADS[f"sweep_c{_c}_d{_d}"] = dict(channels=_c, image_h=128, image_w=128, patch=8,
                                               embed=_d, heads=_h, depth=None, max_group=16,
                                               batch=32)
METRIC = "D-CHAG tokenize+aggregate images/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="hyperspectral", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="training workload: launch the step eagerly instead of replaying its "
                         "CUDA graph")
    ap.add_argument("--h2d-chunks", type=int, default=8,
                    help="batch chunks of the e2e host-input pipeline (copy/compute overlap)")
    ap.add_argument("--arch-tp", type=int, default=None,
                    help="one GPU, one process: run the tp=N architecture's N channel slabs "
                         "back to back + one final layer (BASELINE's same-architecture "
                         "single-GPU denominator of scaling efficiency)")
    ap.add_argument("--cpu-tokens", type=int, default=None,
                    help="tokens per CPU sample (default: 1/8 of an image)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p["bf16_tflops_sustained"], p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


# ----------------------------------------------------------------- CPU reference leg


def cpu_sample(wl, tp, max_group, tokens, seed=0):
    """Time the reference algorithm (oracle/dchag_oracle.py: float64 numpy restatement of
    model.py:180-201, all BLAS threads) on one image restricted to the first `tokens`
    positions (whole patch rows).  Every position is independent on this path, so
    images/s = (tokens / S) / seconds."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import dchag_oracle as O
    p = wl["patch"]
    wp = wl["image_w"] // p
    S = (wl["image_h"] // p) * wp
    # whole images while tokens >= S, else one image cut to whole patch rows
    n_img = max(1, tokens // S)
    rows = wl["image_h"] // p if tokens >= S else max(1, tokens // wp)
    tokens = n_img * rows * wp
    lk, var = wl.get("layer_kind", "cross_attention"), wl.get("variant", "single_query")
    specs = O.frontend_param_specs(wl["channels"], rows * p, wl["image_w"], p, wl["embed"], tp,
                                   max_group, variant=var, layer_kind=lk)
    w = O.random_params(specs, seed=seed)
    img = np.random.default_rng(seed).standard_normal((n_img, wl["channels"], rows * p,
                                                         wl["image_w"]))
    t0 = time.perf_counter()
    done = 0
    for i in range(n_img):  # image by image, stopping early past a 20 s budget
        O.dchag_frontend(img[i:i + 1], w, patch=p, heads=wl["heads"], tp=tp,
                         max_group=max_group, variant=var, layer_kind=lk)
        done += 1
        if time.perf_counter() - t0 > 20.0:
            break
    dt = time.perf_counter() - t0
    tokens = done * rows * wp
    return tokens / S / dt, tokens, dt


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=1), \
            ",".join(sorted({f"{i.get('internal_api')} {i.get('version')}" for i in info}))
    except Exception:
        return os.cpu_count(), "unknown"


def reference_arm(args, wl, tp, max_group):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # torchrun pins OMP_NUM_THREADS=1; the reference arm uses every host core
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=len(os.sched_getaffinity(0)))
    except Exception:
        pass
    S = (wl["image_h"] // wl["patch"]) * (wl["image_w"] // wl["patch"])
    tokens = args.cpu_tokens or max(S // 8, wl["image_w"] // wl["patch"])
    vals = []
    for i in range(args.warmup + args.steps):
        v, tok, dt = cpu_sample(wl, tp, max_group, tokens, seed=i)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    threads, blas = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * (tok / S) / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, wl, tp, max_group),
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"1 image x {tok}/{S} tokens per step (float64 numpy "
                                   f"restatement of the reference, {blas})"
                                   + ("; forward only: the oracle has no backward, so the "
                                      "CPU side of the fwd+bwd step is not timed"
                                      if wl.get("train") else "")},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, wl, tp, max_group):
    return {"workload": args.workload, "step": "fwd+bwd" if wl.get("train") else "fwd",
            "channels": wl["channels"],
            "image": [wl["image_h"], wl["image_w"]], "patch": wl["patch"],
            "embed": wl["embed"], "heads": wl["heads"], "depth": wl["depth"],
            "max_group": max_group, "tp": tp, "global_batch": args.batch or wl["batch"],
            "final_layer": final_layer_mode(args, wl, tp),
            **({"layer_kind": wl["layer_kind"]} if wl.get("layer_kind") else {}),
            **({"agg_variant": wl["variant"]} if wl.get("variant") else {}),
            "parallelism": f"dchag-tp{tp}",
            "l2": "flushed between timed steps (256 MiB write)"}


def final_layer_mode(args, wl, tp):
    if tp == 1:
        return "single stream"
    if wl.get("final_split"):
        return "head-split"
    rows = (args.batch or wl["batch"]) * (wl["image_h"] // wl["patch"]) * (wl["image_w"] // wl["patch"])
    return "position-split" if wl.get("train") is None and rows % (tp * 128) == 0 else "replicated"


# ----------------------------------------------------------------- B200 arm


class ClockSampler:
    """NVML sampler thread (every 5 ms) of SM clock, power and clock-event reasons; the
    summary covers the samples taken between mark_start() and mark_stop()."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        import threading
        self.index = index
        self.samples = []
        self.window = [None, None]
        self.stop_ev = threading.Event()
        self.thread = None

    def _run(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self.stop_ev.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((time.perf_counter(), sm, pw, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        import threading
        try:
            import pynvml  # noqa: F401
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def mark_start(self):
        self.window[0] = time.perf_counter()

    def mark_stop(self):
        self.window[1] = time.perf_counter()

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return None
        t0, t1 = self.window
        win = [x for x in self.samples if t0 is not None and t0 <= x[0] <= (t1 or 1e30)]
        src = win or self.samples
        reasons = sorted({k for x in src for k, bit in self.REASONS.items() if x[3] & bit})
        return {"sm_mhz": statistics.median(x[1] for x in src),
                "sm_max_mhz": float(getattr(self, "max_mhz", 0)),
                "power_w_max": max(x[2] for x in src), "reasons": reasons,
                "samples": len(src), "window": "timed region" if win else "whole run"}


class KernelTimer:
    """Per-launch CUDA events on the launching stream around every libdchag launch
    (_lib.set_launch_hook). A launch's site is its `work` annotation's site (train.py,
    ops.py), else the matching entry of the inference launch plan, else the entry point."""

    def __init__(self, plan=None):
        import torch
        self.torch = torch
        self.plan = plan or []
        self.events = []     # [site, name, start, stop, work]
        self.i = 0

    def hook(self, name, phase, work):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        if phase == "pre":
            if work and work.get("site"):
                site = work["site"]
            elif self.i < len(self.plan):
                site, work = self.plan[self.i][1], {"flops": self.plan[self.i][2],
                                                    "bytes": self.plan[self.i][3]}
            else:
                site = name
            self.events.append([site, name, ev, None, work or {}])
        else:
            self.events[-1][3] = ev
            self.i += 1

    def new_step(self, _=None):
        self.i = 0

    def summary(self, steps):
        """{site: {"kernel", "ms" per step, "launches" per step, "flops", "bytes"}}."""
        out = {}
        for site, name, a, b, work in self.events:
            e = out.setdefault(site, {"kernel": name, "ms": 0.0, "launches": 0, "flops": 0,
                                      "bytes": 0})
            e["ms"] += a.elapsed_time(b) / steps
            e["launches"] += 1 / steps
            e["flops"] += work.get("flops", 0) / steps
            e["bytes"] += work.get("bytes", 0) / steps
        return out


TENSOR_KERNELS = ("dchag_l0_node", "dchag_gemm_bf16", "dchag_l0_logits", "dchag_gemm_combine",
                  "dchag_gemm_wgrad", "dchag_gemm_rowdot", "dchag_gemm_rowdot_heads", "dchag_l0_tgrad",
                  "dchag_l0_tgrad_te",
                  "dchag_gemm_nt", "dchag_fullcross_weights")


def roofline(dom, peaks, traffic):
    """Roofline object of the dominant kernel: achieved = its algorithmic flops (or bytes) per
    step / its measured time per step. peak = the measured burst figure (the conservative
    denominator); frac_vs_sustained uses the back-to-back cuBLAS figure."""
    peak_burst, peak_sus, hbm, src = peaks
    t = dom["ms"] / 1e3
    if not t or not (dom["flops"] or dom["bytes"]):
        return None
    # the bound follows the site's arithmetic intensity when both counts are known (a K = 64
    # GEMM writing wide rows is HBM-bound even though it runs on the tensor cores)
    ridge = peak_burst * 1e12 / (hbm * 1e9)
    hbm_bound = bool(dom["bytes"]) and bool(dom["flops"]) and dom["flops"] / dom["bytes"] < ridge
    if dom["kernel"] in TENSOR_KERNELS and dom["flops"] and not hbm_bound:
        ach = dom["flops"] / t / 1e12
        r = {"bound": "tensor", "achieved": ach, "peak": peak_burst, "unit": "TFLOP/s",
             "frac": ach / peak_burst, "frac_vs_sustained": ach / peak_sus,
             "peak_source": f"{src} bf16_tflops (burst); sustained {peak_sus}",
             "flops_per_step": dom["flops"]}
    else:
        ach = dom["bytes"] / t / 1e9
        r = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
             "peak_source": f"{src} hbm_gbs", "bytes_per_step": dom["bytes"]}
    r.update(traffic=traffic, kernel=f"{dom['kernel']}[{dom['site']}]",
             launch_ms=dom["ms"] / max(1.0, dom["launches"]),
             launches_per_step=dom["launches"], ms_per_step=dom["ms"])
    if r["frac"] > 1.0:  # never report > 1: a timing anomaly is flagged, not credited
        r["anomaly"] = f"measured frac {r['frac']:.3f} > 1 (kernel timing anomaly)"
        r["frac"] = 1.0
    return r


def b200_arm(args, wl, tp, max_group):
    import torch
    import torch.distributed as dist
    from paper_2506_21411_b200 import DchagFrontEnd, _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world >= 4 and wl.get("train") and not args.no_graph:
        # the graph-captured training step needs NVLS off at >= 4 ranks;
        # must be set before the communicator is created
        os.environ.setdefault("NCCL_NVLS_ENABLE", "0")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B = args.batch or wl["batch"]
    arch_tp = args.arch_tp if (args.arch_tp and world == 1) else None

    def make_fe(tp_, rank_):
        # the training config's final layer is head-split over the tp group (reduce-scatter
        # of the boundary gradient in backward, BASELINE.json configs[3]); the in-process
        # architecture mode keeps the replicated final layer (no collectives in one process)
        fe_ = DchagFrontEnd(wl["channels"], wl["image_h"], wl["image_w"], wl["patch"],
                            wl["embed"], wl["heads"], max_group=max_group, tp=tp_, rank=rank_,
                            final_layer_tp_split=(bool(wl.get("final_split")) and tp_ > 1
                                                  and not arch_tp),
                            agg_variant=wl.get("variant", "single_query"),
                            agg_layer_kind=wl.get("layer_kind", "cross_attention"),
                            precision=wl.get("precision", "bf16"))
        fe_.init_weights(seed=0, all_ranks=False)
        fe_.prepare()
        return fe_

    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    if arch_tp:
        # the tp = N architecture in one process: N slabs back to back, one final layer
        fes = [make_fe(arch_tp, r) for r in range(arch_tp)]
        fe = fes[0]
        images = torch.randn(B, wl["channels"], wl["image_h"], wl["image_w"], device="cuda",
                             generator=gen).to(torch.bfloat16)
    else:
        fe = make_fe(tp, rank)
        images = torch.randn(B, fe.slab[1], wl["image_h"], wl["image_w"], device="cuda",
                             generator=gen).to(torch.bfloat16)
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")

    trace = os.environ.get("DCHAG_BENCH_TRACE") == "1"

    def mark(what):
        if trace:
            print(f"[bench rank {rank}] {what} {time.perf_counter():.3f}", file=sys.stderr,
                  flush=True)

    def barrier():
        mark("barrier: sync")
        torch.cuda.synchronize()
        mark("barrier: dist")
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        mark("barrier: done")

    def timed(step_fn, k, per_step_hook=None):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(k)]
        barrier()
        for i in range(k):
            flush.zero_()
            if per_step_hook:
                per_step_hook(i)
            ev[i][0].record()
            step_fn()
            ev[i][1].record()
        barrier()
        return sum(a.elapsed_time(b) for a, b in ev)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    gstep = None
    trainer = None
    if wl.get("train") and arch_tp:
        # the tp = N training architecture in one process: every rank's slab forward, the
        # root streams stacked in rank order (the AllGather), each rank's replicated final
        # layer and backward, as tests/test_gpu_train.py runs it
        from paper_2506_21411_b200.train import DchagTrainer
        trainers = [DchagTrainer(f) for f in fes]
        probe = torch.randn(B, 1, fe.seq, wl["embed"], device="cuda", generator=gen)
        slabs_img = [images[:, f.slab[0]:f.slab[0] + f.slab[1]] for f in fes]

        def step():
            saves = [t.forward_local(x) for t, x in zip(trainers, slabs_img)]
            y_all = torch.stack([sv["y_root"] for sv in saves])
            outs = [t.forward_final(y_all, sv) for t, sv in zip(trainers, saves)]
            for t, sv in zip(trainers, saves):
                _, g_y = t.backward_final(sv, probe)
                t.backward_local(sv, g_y)
            return outs[0]
        eager_step = step
    elif wl.get("train"):
        from paper_2506_21411_b200.train import DchagTrainer
        trainer = DchagTrainer(fe)
        probe = torch.randn(B, 1, fe.seq, wl["embed"], device="cuda", generator=gen)

        def eager_step():
            out, saved = trainer.forward_train(images)
            return trainer.backward(saved, probe)
        if args.no_graph:
            step = eager_step
        else:
            # the whole step (forward_train + backward, collectives included) as one CUDA
            # graph over the static image / probe buffers: a replay re-runs every kernel
            mark("capture")
            gstep = trainer.capture(images, probe)
            mark("captured")
            step = gstep.replay
    elif arch_tp:
        slabs_img = [images[:, f.slab[0]:f.slab[0] + f.slab[1]] for f in fes]

        def step():
            pays = [f.local_payload(x) for f, x in zip(fes, slabs_img)]
            return fe.finish(torch.cat(pays), B)
        eager_step = step
    else:
        eager_step = lambda: fe(images)  # noqa: E731
        step = eager_step
        if not args.no_graph and world == 1 and not fe._unfolded():
            # the inference forward as one CUDA graph (serving): a replay re-runs every
            # kernel of the step; the eager launches before capture build every cached
            # device table, so the captured region holds kernels only
            for _ in range(2):
                eager_step()
            torch.cuda.synchronize()
            n_cap = _lib.LAUNCH_COUNT["n"]
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            fgraph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(fgraph, stream=side):
                    eager_step()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            f_launches = _lib.LAUNCH_COUNT["n"] - n_cap

            def graph_step():
                fgraph.replay()
                _lib.LAUNCH_COUNT["n"] += f_launches
            graph_step()
            torch.cuda.synchronize()
            # keep the graph only where it is faster (launch-bound steps: the CPU launch cost
            # of ~10-20 kernels exceeds a small step's GPU time; ms-scale steps tie)
            t_eager = timed(eager_step, 5)
            t_graph = timed(graph_step, 5)
            if t_graph < t_eager:
                step, gstep = graph_step, fgraph
            else:
                fgraph.reset()
    clk = ClockSampler(local).__enter__()
    for i in range(args.warmup):
        step()
        # each warm-up step completes before the next is issued (graph replays with NCCL
        # kernels queued back to back in the warm-up hung at 4 ranks)
        torch.cuda.synchronize()
        mark(f"warmup {i} done")
    t_end = time.perf_counter() + 0.5  # let clocks settle: >= 0.5 s of warm-up work
    while time.perf_counter() < t_end:
        step()
        torch.cuda.synchronize()
    # ---- pass A: headline (inputs resident in HBM)
    n0 = _lib.LAUNCH_COUNT["n"]
    clk.mark_start()
    ms = timed(step, args.steps)
    clk.mark_stop()
    launches = _lib.LAUNCH_COUNT["n"] - n0
    ms = max_over_ranks(ms)
    value = B * args.steps / (ms / 1e3)

    # ---- pass B: per-kernel CUDA events on the launching stream, same step run eagerly
    # (the training step's launches carry work annotations; the forward follows its plan)
    unfolded = fe._unfolded()  # full_cross / fp32: annotated ops-path launches, no plan
    plan = [] if (unfolded or wl.get("train") or arch_tp) else fe.launch_plan(B)
    kt = KernelTimer(plan)
    chunks, fe.comm_chunks = fe.comm_chunks, 1
    _lib.set_launch_hook(kt.hook)
    try:
        step_ms = timed(eager_step, args.steps, per_step_hook=kt.new_step) / args.steps
    finally:
        _lib.set_launch_hook(None)
        fe.comm_chunks = chunks
    sites = kt.summary(args.steps)
    kernels = [dict(site=k, **v, tflops=(v["flops"] / v["ms"] / 1e9 if v["ms"] and v["flops"]
                                         else None),
                    gbs=(v["bytes"] / v["ms"] / 1e6 if v["ms"] and v["bytes"] else None))
               for k, v in sorted(sites.items(), key=lambda kv: -kv[1]["ms"])]
    peaks = load_peaks()
    traffic = None
    dom = kernels[0] if kernels else None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{args.workload}:tp{tp}:{dom['site']}")
    except Exception:
        pass
    roof = roofline(dom, peaks, traffic) if dom else None
    if roof is not None:
        roof["share_of_step"] = dom["ms"] / step_ms if step_ms else None
    ours_ms = sum(k["ms"] for k in kernels)

    # ---- pass C: end to end through the public API from pinned host memory
    host_img = images.cpu().pin_memory()
    out_host = torch.empty(B, 1, fe.seq, wl["embed"],
                           dtype=torch.float32 if wl.get("train") else fe.out_dtype).pin_memory()
    dev_img = torch.empty_like(images)

    def e2e_step():
        if wl.get("train") and arch_tp:
            images.copy_(host_img, non_blocking=True)
            out = step()
            if rank == 0:
                out_host.copy_(out, non_blocking=True)
        elif wl.get("train"):
            if gstep is None:
                dev_img.copy_(host_img, non_blocking=True)
                out, saved = trainer.forward_train(dev_img)
                trainer.backward(saved, probe)
            else:
                images.copy_(host_img, non_blocking=True)   # the graph's static input
                gstep.replay()
                out = gstep.out
            if rank == 0:
                out_host.copy_(out, non_blocking=True)
        elif unfolded or arch_tp:  # device-image paths: copy in, run, copy out
            dev_img.copy_(host_img, non_blocking=True)
            if arch_tp:
                pays = [f.local_payload(dev_img[:, f.slab[0]:f.slab[0] + f.slab[1]])
                        for f in fes]
                out = fe.finish(torch.cat(pays), B)
            else:
                out = fe(dev_img)
            if rank == 0:
                out_host.copy_(out, non_blocking=True)
        else:
            # public API with host buffers: chunked H2D overlapped with the kernels, the
            # result rows streamed back into the pinned host tensor
            fe(host_img, out=out_host if rank == 0 else None, h2d_chunks=args.h2d_chunks)

    for _ in range(2):
        e2e_step()
    e2e_ms = max_over_ranks(timed(e2e_step, args.steps))
    h2d = images.numel() * images.element_size()
    d2h = out_host.numel() * out_host.element_size() if rank == 0 else 0

    # ---- whole-job algorithmic work (executed flops of our kernels, summed over ranks;
    # a replicated final layer counts once)
    exec_flops = sum(k["flops"] for k in kernels)
    if world > 1:
        t = torch.tensor([float(exec_flops)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        tot_exec = float(t.item())
    else:
        tot_exec = exec_flops
    b_slabs = fes[0].slabs if arch_tp else fe.slabs
    b_flops = bflops_per_image(wl, b_slabs, max_group, train=bool(wl.get("train"))) * B

    cpu = None  # the CPU oracle is timed on rank 0 at N = 1 only (torchrun pins 1 OMP thread)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        S = fe.seq
        tokens = args.cpu_tokens or 2 * S   # two whole images, ~10-25 s of CPU work
        v, tok, dt = cpu_sample(wl, arch_tp or tp, max_group, tokens)
        threads, blas = blas_threads()
        cpu = {"value": v, "unit": "images/s", "cores": threads, "kind": "port",
               "cpu_model": cpu_model(),
               "sample": f"{tok / S:g} image(s) x {S} tokens, {dt:.1f} s (float64 numpy restatement "
                         f"of the reference hot path, {blas})"
                         + ("; forward only: the oracle has no backward" if wl.get("train")
                            else "")}

    clk.__exit__()
    if rank == 0:
        clocks = clk.summary()
        cfg = workload_config(args, wl, arch_tp or tp, max_group)
        cfg["launch"] = "eager" if gstep is None else "cuda graph (whole step)"
        if arch_tp:
            cfg["parallelism"] = f"dchag-tp{arch_tp} architecture on 1 GPU (slabs sequential)"
            cfg["final_layer"] = "once, over the tp streams (AllGather schedule)"
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": wl.get("precision", "bf16"),
            "data": "synthetic (N(0,1) bf16 images, truncated-normal(0.02) "
                                     "random-init weights)",
            "config": cfg,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": B * args.steps / (e2e_ms / 1e3), "unit": "images/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clocks,
            "work": {"executed_tflop_per_step": tot_exec / 1e12 if tot_exec else None,
                     "executed_tflops": (tot_exec / (ms / args.steps / 1e3) / 1e12
                                         if tot_exec else None),
                     "executed_frac_of_burst": (tot_exec / (ms / args.steps / 1e3) / 1e12
                                                / (world * peaks[0]) if tot_exec else None),
                     "reference_graph_B_tflop_per_step": b_flops / 1e12,
                     "B_flops_effective_tflops": b_flops / (ms / args.steps / 1e3) / 1e12,
                     "B_flops_roofline_frac": b_flops / (ms / args.steps / 1e3) / 1e12
                     / (world * peaks[0])},
            "kernel_pass": {"eager_step_ms": step_ms, "our_kernels_ms": ours_ms,
                            "other_ms": step_ms - ours_ms},
            "kernels": kernels,
        }
        print(json.dumps(line), flush=True)
    if gstep is not None:
        torch.cuda.synchronize()
        # release the captured work (NCCL included) before the group goes away
        (gstep.graph if hasattr(gstep, "graph") else gstep).reset()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def bflops_per_image(wl, slabs, max_group, train=False):
    """SURVEY.md section 8(d) 'B' flops: collapsed single_query count (linear nodes
    S (2 g D + 2 D^2); full_cross counted as single_query), final layer once;
    fwd+bwd = 3 x (nodes + final) + 2 x tokenizer."""
    from paper_2506_21411_b200.config import build_tree_spec
    S = (wl["image_h"] // wl["patch"]) * (wl["image_w"] // wl["patch"])
    D, H, pp = wl["embed"], wl["heads"], wl["patch"] ** 2
    tok = nodes = 0
    for _, c in slabs:
        tok += 2 * c * S * pp * D
        for level in build_tree_spec(c, max_group).levels:
            for g in level:
                nodes += (S * (2 * g * D + 2 * D * D) if wl.get("layer_kind") == "linear"
                          else S * (4 * g * D * H + 4 * D * D))
    nodes += S * (4 * len(slabs) * D * H + 4 * D * D)
    return 3 * nodes + 2 * tok if train else nodes + tok


def main():
    args = parse()
    wl = WORKLOADS[args.workload]
    tp = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if args.impl == "reference":
        tp = args.gpus
    from paper_2506_21411_b200.config import build_tree_spec, channel_slabs, max_group_for_depth
    slabs = [n for _, n in channel_slabs(wl["channels"], args.arch_tp or tp)]
    if wl.get("max_group"):
        max_group = wl["max_group"]
        wl = dict(wl, depth=max(build_tree_spec(n, max_group).depth for n in slabs))
    else:
        max_group = max_group_for_depth(slabs, wl["depth"])
    if args.impl == "reference":
        reference_arm(args, wl, tp, max_group)
    else:
        b200_arm(args, wl, tp, max_group)


if __name__ == "__main__":
    main()
