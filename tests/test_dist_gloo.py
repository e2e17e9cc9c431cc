"""N>1 host-side path on CPU (gloo, world_size 2 and 3): every rank folds only its own
slab's weights, packs its root payload (payload.py layout), the payloads are all-gathered
in rank order (all_gather_into_tensor, the NCCL call of the GPU path), and the shared final
layer over the unpacked streams reproduces the reference hot path (model.py:180-201) --
including uneven slabs (22 channels over 3 ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, meta, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import dchag_oracle as O
    from folded_emulator import emulate_rank
    from paper_2506_21411_b200.config import build_tree_spec, channel_slabs
    from paper_2506_21411_b200.fold import fold_rank
    from paper_2506_21411_b200.payload import pack, payload_nbytes, unpack

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lk = meta["layer_kind"]
        specs = O.frontend_param_specs(meta["C"], 16, 16, 4, meta["D"], world, meta["g"],
                                       layer_kind=lk)
        w = O.random_params(specs, seed=4, std=0.2, bias_std=0.05)
        images = np.random.default_rng(5).standard_normal((2, meta["C"], 16, 16))
        # the rank keeps only its own weights, exactly as DchagFrontEnd.load_weights
        slabs = channel_slabs(meta["C"], world)
        off, cnt = slabs[rank]
        tw = {k: torch.from_numpy(v) for k, v in w.items()
              if not k.startswith("agg.slab") or k.startswith(f"agg.slab{rank}.")}
        fr = fold_rank(tw, rank=rank, slab=(off, cnt),
                       levels=build_tree_spec(cnt, meta["g"]).levels, embed=meta["D"],
                       heads=meta["H"], patch=4, seq=16, variant="single_query", layer_kind=lk)
        V, L, _ = emulate_rank(fr, torch.from_numpy(images[:, off:off + cnt]), meta["H"])
        payload = pack(V, L)
        R = V.shape[0]
        assert payload.numel() == payload_nbytes(R, meta["D"], meta["H"])
        gathered = torch.empty(world * payload.numel(), dtype=torch.uint8)
        dist.all_gather_into_tensor(gathered, payload)
        Vg, Lg = unpack(gathered, world, R, meta["D"], meta["H"])
        dh = meta["D"] // meta["H"]
        p = torch.softmax(Lg.double(), dim=0).repeat_interleave(dh, dim=2)
        ctx = (p * Vg.double()).sum(0)
        out = (ctx @ fr.Wf + fr.bf).view(2, 1, 16, meta["D"]).numpy()
        want = O.dchag_frontend(images, w, patch=4, heads=meta["H"], tp=world,
                                max_group=meta["g"], layer_kind=lk)
        q.put((rank, O.rel_err(out, want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,meta", [
    (2, dict(C=12, D=16, H=4, g=3, layer_kind="cross_attention")),
    (3, dict(C=22, D=16, H=4, g=3, layer_kind="cross_attention")),
    (2, dict(C=10, D=16, H=2, g=2, layer_kind="linear")),
])
def test_gather_and_final_layer_match_reference(world, meta):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, meta, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in res:
        # V travels as bf16 (the GPU payload format): bf16 budget
        assert err < 2e-2, (rank, err)
