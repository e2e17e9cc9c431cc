"""Communication ledger of the collectives the front end issues over NCCL.

Restates the reference's ledger schema and per-rank payload accounting (runtime.py:30-90,
:93-99, :250-290) for the real NCCL calls, so the reference's byte contracts
(test_strategies.py:195-208: one boundary AllGather of S*D*itemsize*(tp-1) bytes per
rank and image in the forward, no boundary events in the backward) can be checked on the GPU.
Attach one with `fe.ledger = CommLedger()`; `DchagTrainer` records into the same object.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

DCHAG_BOUNDARY_TAG = "dchag-boundary"     # strategies.py:41
FINAL_OUT_TAG = "dchag-final-out"         # position-split final layer: output AllGather
FINAL_ALLSUM_TAG = "agg-final"            # head-split final layer: TpHooks.allsum
POS_GRAD_TAG = "shared-grad.special.pos"  # strategies.py:251-264 (phase "optimizer")
DP_GRAD_TAG = "dp-grad."                  # + parameter name (strategies.py:352-357)


@dataclass(frozen=True)
class CommEvent:
    rank: int
    seq: int
    op: str
    axis: str
    phase: str
    payload_bytes_per_rank: int
    tag: str


def allgather_payload(shard_nbytes: int, group: int) -> int:
    """Ring AllGather: every rank receives the other ranks' shards (runtime.py:93-94)."""
    return shard_nbytes * (group - 1)


def reduce_scatter_payload(chunk_nbytes: int, group: int) -> int:
    """Ring ReduceScatter: the AllGather count on the output chunk (runtime.py:275)."""
    return chunk_nbytes * (group - 1)


def allreduce_payload(n_elem: int, itemsize: int, group: int) -> int:
    """Ring AllReduce: 2 (g-1) chunks of ceil(n/g) elements (runtime.py:97-99)."""
    chunk = -(-n_elem // group)
    return 2 * chunk * itemsize * (group - 1)


def alltoall_payload(total_nbytes: int, group: int) -> int:
    """All-to-all of equal blocks: each rank sends (g-1)/g of its buffer (extension; the
    reference has no all-to-all)."""
    return total_nbytes // group * (group - 1)


class CommLedger:
    """Per-rank ordered collective events with the reference's query / CSV interface."""

    def __init__(self):
        self.per_rank: dict[int, list[CommEvent]] = {}

    def record(self, rank: int, op: str, axis: str, phase: str, payload: int, tag: str = ""):
        evs = self.per_rank.setdefault(rank, [])
        evs.append(CommEvent(rank, len(evs), op, axis, phase, int(payload), tag))

    def events(self):
        for rank in sorted(self.per_rank):
            yield from self.per_rank[rank]

    def query(self, phase: str | None = None, axis: str | None = None,
              op: str | None = None, tag: str | None = None,
              rank: int | None = None) -> tuple[int, int]:
        """(total payload bytes, event count) over matching events (runtime.py:62-81)."""
        total = count = 0
        for ev in self.events():
            if phase is not None and ev.phase != phase:
                continue
            if axis is not None and ev.axis != axis:
                continue
            if op is not None and ev.op != op:
                continue
            if tag is not None and ev.tag != tag:
                continue
            if rank is not None and ev.rank != rank:
                continue
            total += ev.payload_bytes_per_rank
            count += 1
        return total, count

    def to_csv(self, path) -> None:
        """Same columns as the reference ledger (runtime.py:83-90)."""
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["rank", "seq", "op", "axis", "phase", "payload_bytes_per_rank", "tag"])
            for ev in self.events():
                w.writerow([ev.rank, ev.seq, ev.op, ev.axis, ev.phase,
                            ev.payload_bytes_per_rank, ev.tag])
