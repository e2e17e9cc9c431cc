"""Communication ledger of the collectives the front end issues over NCCL.

The wire format is the reference's (runtime.py:83-90 CSV columns, runtime.py:62-81 query
semantics, runtime.py:93-99 / :250-290 ring payload accounting) so that the reference's byte
contracts (test_strategies.py:195-208: one boundary AllGather of S*D*itemsize*(tp-1) bytes per
rank and image in the forward, no boundary event in the backward) can be checked against the
real NCCL calls.  The container itself is a flat, append-only event log with a per-rank
sequence counter; per-rank views and queries are derived from it.

Attach one with `fe.ledger = CommLedger()`; `DchagTrainer` records into the same object.
"""

from __future__ import annotations

import csv
from collections import Counter
from typing import NamedTuple

DCHAG_BOUNDARY_TAG = "dchag-boundary"     # strategies.py:41
FINAL_OUT_TAG = "dchag-final-out"         # position-split final layer: output AllGather
FINAL_ALLSUM_TAG = "agg-final"            # head-split final layer: TpHooks.allsum
POS_GRAD_TAG = "shared-grad.special.pos"  # strategies.py:251-264 (phase "optimizer")
DP_GRAD_TAG = "dp-grad."                  # + parameter name (strategies.py:352-357)


class CommEvent(NamedTuple):
    """One collective as seen by one rank; field order = the CSV column order."""
    rank: int
    seq: int
    op: str
    axis: str
    phase: str
    payload_bytes_per_rank: int
    tag: str


CSV_COLUMNS = list(CommEvent._fields)


# ---- per-rank payload of one collective over a group of `group` ranks (ring algorithms)

def allgather_payload(shard_nbytes: int, group: int) -> int:
    """Every rank receives the group's other shards (runtime.py:93-94)."""
    return (group - 1) * shard_nbytes


def reduce_scatter_payload(chunk_nbytes: int, group: int) -> int:
    """Same count as the AllGather of the output chunk (runtime.py:275)."""
    return allgather_payload(chunk_nbytes, group)


def allreduce_payload(n_elem: int, itemsize: int, group: int) -> int:
    """ReduceScatter + AllGather of ceil(n/g)-element chunks (runtime.py:97-99)."""
    per_chunk = itemsize * ((n_elem + group - 1) // group)
    return 2 * (group - 1) * per_chunk


def alltoall_payload(total_nbytes: int, group: int) -> int:
    """Equal blocks: (g-1)/g of the buffer leaves each rank (extension; the reference has no
    all-to-all)."""
    return (group - 1) * (total_nbytes // group)


class CommLedger:
    """Ordered log of collective events with the reference's query / CSV interface."""

    def __init__(self):
        self._log: list[CommEvent] = []
        self._seq: Counter = Counter()

    def record(self, rank: int, op: str, axis: str, phase: str, payload: int, tag: str = ""):
        seq = self._seq[rank]
        self._seq[rank] = seq + 1
        self._log.append(CommEvent(rank, seq, op, axis, phase, int(payload), tag))

    @property
    def per_rank(self) -> dict:
        view: dict[int, list[CommEvent]] = {}
        for ev in self._log:
            view.setdefault(ev.rank, []).append(ev)
        return view

    def events(self):
        """All events, rank-major, each rank's in record order (runtime.py:58-60)."""
        return iter(sorted(self._log, key=lambda ev: (ev.rank, ev.seq)))

    def query(self, phase: str | None = None, axis: str | None = None,
              op: str | None = None, tag: str | None = None,
              rank: int | None = None) -> tuple[int, int]:
        """(total payload bytes, event count) of the events matching every given field;
        None matches anything (runtime.py:62-81)."""
        want = {k: v for k, v in (("phase", phase), ("axis", axis), ("op", op), ("tag", tag),
                                  ("rank", rank)) if v is not None}
        hits = [ev.payload_bytes_per_rank for ev in self._log
                if all(getattr(ev, k) == v for k, v in want.items())]
        return sum(hits), len(hits)

    def to_csv(self, path) -> None:
        """The reference ledger's CSV (runtime.py:83-90)."""
        with open(path, "w", newline="") as fh:
            out = csv.writer(fh)
            out.writerow(CSV_COLUMNS)
            out.writerows(self.events())
