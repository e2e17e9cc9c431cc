"""Multi-rank parity checks of the front end, shared by tests/test_gpu_dist.py (ranks as
processes on one GPU over gloo: the collectives go through comm.py's host-staged path) and
tools/dist_parity.py (one rank per GPU over NCCL under torchrun) -- test infrastructure.

Every rank runs its channel slab (tp = world, balanced slabs); the root payloads are
exchanged in rank order (AllGather, or the position-split all-to-all), the shared final
layer runs replicated, position-split or head-split, and each rank's output / gradients are
compared with the CPU oracle (float64) and the float64 autograd restatement
(tests/torch_reference.py). Also: the ledger byte contract of test_strategies.py:195-208,
data parallelism, and the head-split final layer after a weight reload (a fresh module must
agree bitwise).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)
import dchag_oracle as O  # noqa: E402
from paper_2506_21411_b200 import DchagFrontEnd  # noqa: E402

CASES = [
    dict(channels=22, image_h=64, image_w=128, patch=8, embed=256, heads=4, max_group=3),
    dict(channels=37, image_h=64, image_w=64, patch=4, embed=128, heads=2, max_group=4),
    dict(channels=40, image_h=64, image_w=128, patch=8, embed=256, heads=4, max_group=4,
         layer_kind="linear"),
]


def run_checks(log=print, ledger_dir=None):
    """Every check on the initialised default process group; returns the worst error
    (rel_err, or 1.0 for a broken contract) seen on this rank."""
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
            log(f"rank {rank}: boundary ledger {(tot_, n_)} != ({want_}, {nev_})")
            worst = max(worst, 1.0)
        if not split:
            fe.final_position_split = False
            out_ag = fe(img_bf.cuda()).cpu().numpy()
            fe.final_position_split = True
            if not np.array_equal(out, out_ag):
                log(f"rank {rank}: position-split final differs from the AllGather schedule "
                      f"(max |diff| {np.abs(out - out_ag).max():.3e})")
                worst = max(worst, 1.0)
        want = O.dchag_frontend(img_bf.float().numpy().astype(np.float64), w,
                                patch=meta["patch"], heads=meta["heads"], tp=tp,
                                max_group=meta["max_group"], layer_kind=lk)
        err = O.rel_err(out, want)
        worst = max(worst, err)
        mode = " head-split final" if split else (
            " position-split final (== AllGather bitwise)" if fe._position_split(8) else "")
        log(f"rank {rank}/{tp} C={meta['channels']} slab={fe.slab} {lk}{mode}: "
              f"rel_err={err:.3e}")
    # head-split final layer after a weight reload: the reloaded module must agree bitwise
    # with a fresh module given the same weights (the final-layer shards are derived from
    # the folded weights and must not outlive them)
    meta = CASES[0]
    if meta["heads"] % tp == 0:
        specs = O.frontend_param_specs(meta["channels"], meta["image_h"], meta["image_w"],
                                       meta["patch"], meta["embed"], tp, meta["max_group"])
        w1, w2 = (O.random_params(specs, seed=s_, std=0.05, bias_std=0.02) for s_ in (1, 2))
        img = torch.from_numpy(np.random.default_rng(8).standard_normal(
            (2, meta["channels"], meta["image_h"], meta["image_w"])).astype(np.float32))
        img = img.to(torch.bfloat16).cuda()
        mk = lambda: DchagFrontEnd(meta["channels"], meta["image_h"], meta["image_w"],  # noqa
                                   meta["patch"], meta["embed"], meta["heads"],
                                   max_group=meta["max_group"], tp=tp, rank=rank,
                                   out_dtype=torch.float32, final_layer_tp_split=True)
        fe = mk()
        fe.load_weights(w1)
        fe(img)
        fe.load_weights(w2)
        got = fe(img)
        fresh = mk()
        fresh.load_weights(w2)
        ok = torch.equal(got, fresh(img))
        log(f"rank {rank}/{tp} head-split final after weight reload == fresh module: {ok}")
        worst = max(worst, 0.0 if ok else 1.0)
    # training step over NCCL: forward_train (AllGather of root streams) + backward
    # (local-slice boundary, special.pos all-reduce), vs float64 autograd of the reference math
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
            log(f"rank {rank}: training ledger breaks the boundary contract")
            worst = max(worst, 1.0)
        if rank == 0 and ledger_dir:
            os.makedirs(ledger_dir, exist_ok=True)
            fe.ledger.to_csv(os.path.join(ledger_dir, f"ledger_tp{tp}"
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
        log(f"rank {rank}/{tp} train step{' (head-split final)' if split else ''}: "
              f"{len(errs)} grads, worst rel_err={terr:.3e} ({max(errs, key=errs.get)})")
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
    log(f"rank {rank}/{tp} data-parallel (dp={tp}) averaged grads: worst rel_err={derr:.3e}, "
          f"{nev} dp ledger events")
    return worst
