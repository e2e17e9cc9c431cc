"""Multi-GPU parity: torchrun --nproc-per-node N tools/dist_parity.py
Every rank runs its channel slab (tp = N, balanced slabs), the root payloads are
all-gathered over NCCL in rank order, the shared final layer runs on every rank, and
each rank's output is compared with the CPU oracle (oracle/ is the checker only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import dchag_oracle as O  # noqa: E402
from paper_2506_21411_b200 import DchagFrontEnd  # noqa: E402

CASES = [
    dict(channels=22, image_h=64, image_w=128, patch=8, embed=256, heads=4, max_group=3),
    dict(channels=37, image_h=64, image_w=64, patch=4, embed=128, heads=2, max_group=4),
    dict(channels=40, image_h=64, image_w=128, patch=8, embed=256, heads=4, max_group=4,
         layer_kind="linear"),
]


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tp, rank = dist.get_world_size(), dist.get_rank()
    worst = 0.0
    for meta, split in [(m, sp) for m in CASES for sp in (False, True)
                        if not sp or m["heads"] % tp == 0]:
        # batch 8: B*S = 1024 rows, so the position-split final layer (rows % (128 tp) == 0)
        # runs at tp <= 8; the AllGather schedule runs alongside and must match it bitwise
        lk = meta.get("layer_kind", "cross_attention")
        specs = O.frontend_param_specs(meta["channels"], meta["image_h"], meta["image_w"],
                                       meta["patch"], meta["embed"], tp, meta["max_group"],
                                       layer_kind=lk)
        w = O.random_params(specs, seed=7, std=0.05, bias_std=0.02)
        w = {k: v.astype(np.float32).astype(np.float64) for k, v in w.items()}
        img = np.random.default_rng(3).standard_normal(
            (8, meta["channels"], meta["image_h"], meta["image_w"]))
        img_bf = torch.from_numpy(img.astype(np.float32)).to(torch.bfloat16)
        fe = DchagFrontEnd(meta["channels"], meta["image_h"], meta["image_w"], meta["patch"],
                           meta["embed"], meta["heads"], max_group=meta["max_group"],
                           agg_layer_kind=lk, tp=tp, rank=rank, out_dtype=torch.float32,
                           final_layer_tp_split=split)
        fe.load_weights(w)
        from paper_2506_21411_b200.ledger import CommLedger
        fe.ledger = CommLedger()
        out = fe(img_bf.cuda()).cpu().numpy()  # full images: the rank slices its own slab
        # byte contract (test_strategies.py:195-208 restated for the bf16 payload): the
        # boundary is one collective per rank in the forward (AllGather of the root payload,
        # or its position-split all-to-all), nothing in the backward
        R_ = 8 * (meta["image_h"] // meta["patch"]) * (meta["image_w"] // meta["patch"])
        pay_ = R_ * (2 * meta["embed"] + 4 * meta["heads"])
        tot_, n_ = fe.ledger.query(phase="forward", tag="dchag-boundary")
        want_ = pay_ // tp * (tp - 1) if fe._position_split(8) and not split else pay_ * (tp - 1)
        nev_ = fe._comm_chunks(8) if not split else 1   # one exchange per batch chunk
        if n_ != nev_ or tot_ != want_:
            print(f"rank {rank}: boundary ledger {(tot_, n_)} != ({want_}, {nev_})", flush=True)
            worst = max(worst, 1.0)
        if not split:
            fe.final_position_split = False
            out_ag = fe(img_bf.cuda()).cpu().numpy()
            fe.final_position_split = True
            if not np.array_equal(out, out_ag):
                print(f"rank {rank}: position-split final differs from the AllGather schedule "
                      f"(max |diff| {np.abs(out - out_ag).max():.3e})", flush=True)
                worst = max(worst, 1.0)
        want = O.dchag_frontend(img_bf.float().numpy().astype(np.float64), w,
                                patch=meta["patch"], heads=meta["heads"], tp=tp,
                                max_group=meta["max_group"], layer_kind=lk)
        err = O.rel_err(out, want)
        worst = max(worst, err)
        mode = " head-split final" if split else (
            " position-split final (== AllGather bitwise)" if fe._position_split(8) else "")
        print(f"rank {rank}/{tp} C={meta['channels']} slab={fe.slab} {lk}{mode}: "
              f"rel_err={err:.3e}", flush=True)
    # training step over NCCL: forward_train (AllGather of root streams) + backward
    # (local-slice boundary, special.pos all-reduce), vs float64 autograd of the reference math
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch_reference as TRF
    from paper_2506_21411_b200.train import DchagTrainer
    specs = O.frontend_param_specs(13, 64, 128, 8, 256, tp, 2)
    w = O.random_params(specs, seed=9, std=0.05, bias_std=0.02)
    w = {k: v.astype(np.float32).astype(np.float64) for k, v in w.items()}
    rng = np.random.default_rng(6)
    img = torch.from_numpy(rng.standard_normal((2, 13, 64, 128)).astype(np.float32)).to(torch.bfloat16)
    probe = rng.standard_normal((2, 1, 128, 256))
    img64 = img.float().numpy().astype(np.float64)
    _, g_ref = TRF.grads(img64, w, probe, patch=8, heads=4, tp=tp, max_group=2)
    for split in (False, True) if 4 % tp == 0 else (False,):
        fe = DchagFrontEnd(13, 64, 128, 8, 256, 4, max_group=2, tp=tp, rank=rank,
                           out_dtype=torch.float32, final_layer_tp_split=split)
        fe.load_weights(w)
        trn = DchagTrainer(fe)
        from paper_2506_21411_b200.ledger import CommLedger
        fe.ledger = CommLedger()
        out, saved = trn.forward_train(img.cuda())
        grads = trn.backward(saved, torch.from_numpy(probe.astype(np.float32)).cuda())
        if fe.ledger.query(phase="backward", tag="dchag-boundary") != (0, 0) or \
                fe.ledger.query(phase="forward", tag="dchag-boundary")[1] != 1:
            print(f"rank {rank}: training ledger breaks the boundary contract", flush=True)
            worst = max(worst, 1.0)
        if rank == 0:
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            fe.ledger.to_csv(os.path.join(ROOT, "gpurun_out", f"ledger_tp{tp}"
                                          f"{'_split' if split else ''}.csv"))
        off, cnt = fe.slab
        dh = 256 // 4
        hc = 4 // tp
        cols = slice(rank * hc * dh, (rank + 1) * hc * dh)
        errs = {}
        for k, v in grads.items():
            v = v.double().cpu().numpy()
            ref = g_ref[k]
            if k in ("tok.w", "tok.b", "special.channel_id"):
                ref = ref[off:off + cnt]
            elif split and k in ("agg.final.wv", "agg.final.wk", "agg.final.wq"):
                ref = ref[:, cols]          # column shards of the own heads (params.py:166-177)
            elif split and k == "agg.final.wo":
                ref = ref[cols]             # row shard
            if np.abs(ref).max() < 1e-12:
                # exactly-zero reference gradient (e.g. the logit weights of a one-channel
                # node: its softmax is identically 1): require ours to be ~0 too
                errs[k] = float(np.abs(v).max() > 1e-6)
            else:
                errs[k] = O.rel_err(v, ref)
        terr = max(errs.values())
        worst = max(worst, terr)
        print(f"rank {rank}/{tp} train step{' (head-split final)' if split else ''}: "
              f"{len(errs)} grads, worst rel_err={terr:.3e} ({max(errs, key=errs.get)})",
              flush=True)
    # data parallel over the whole world (tp = 1, dp = N): every rank trains on
    # its own batch, gradients averaged by one bucketed all-reduce; check against the
    # average of the per-batch gradients computed locally without the dp group
    from paper_2506_21411_b200.grid import make_groups
    from paper_2506_21411_b200.ledger import CommLedger
    _, dp_group, _, dp_i = make_groups(1, tp)
    specs = O.frontend_param_specs(13, 64, 128, 8, 256, 1, 4)
    w = O.random_params(specs, seed=4, std=0.05, bias_std=0.02)
    w = {k: v.astype(np.float32).astype(np.float64) for k, v in w.items()}
    fe = DchagFrontEnd(13, 64, 128, 8, 256, 4, max_group=4, out_dtype=torch.float32)
    fe.load_weights(w)
    fe.ledger = CommLedger()
    imgs = [torch.from_numpy(np.random.default_rng(20 + i).standard_normal((2, 13, 64, 128))
                             .astype(np.float32)).to(torch.bfloat16).cuda() for i in range(tp)]
    probes = [torch.from_numpy(np.random.default_rng(40 + i).standard_normal((2, 1, 128, 256))
                               .astype(np.float32)).cuda() for i in range(tp)]
    trd = DchagTrainer(fe, dp_group=dp_group)
    _, sv = trd.forward_train(imgs[dp_i])
    g_dp = trd.backward(sv, probes[dp_i])
    tr1 = DchagTrainer(fe)
    acc = None
    for i in range(tp):
        _, sv = tr1.forward_train(imgs[i])
        gi = {k: v.double() for k, v in tr1.backward(sv, probes[i]).items()}
        acc = gi if acc is None else {k: acc[k] + gi[k] for k in acc}
    derr = max(O.rel_err(g_dp[k].double().cpu().numpy(), (acc[k] / tp).cpu().numpy())
               for k in acc)
    _, nev = fe.ledger.query(axis="dp", op="AllReduce")
    if nev != len(acc):
        derr = 1.0
    worst = max(worst, derr)
    print(f"rank {rank}/{tp} data-parallel (dp={tp}) averaged grads: worst rel_err={derr:.3e}, "
          f"{nev} dp ledger events", flush=True)
    t = torch.tensor([worst], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"DIST_PARITY tp={tp} worst rel_err={float(t):.3e} -> "
              f"{'PASS' if float(t) < 2e-2 else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if float(t) < 2e-2 else 1)


if __name__ == "__main__":
    main()
