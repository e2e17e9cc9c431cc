"""Communication ledger (paper_2506_21411_b200/ledger.py): the reference's payload
accounting (runtime.py:93-99, :250-290) and its query / CSV schema (runtime.py:62-90)."""
import csv
import os
import sys

import pytest

from paper_2506_21411_b200 import ledger as LG

REF = "/root/reference/pkg/src"


@pytest.mark.parametrize("g", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 7, 256, 1000, 4096])
def test_payload_formulas(g, n):
    assert LG.allgather_payload(n * 2, g) == n * 2 * (g - 1)
    assert LG.reduce_scatter_payload(n * 4, g) == n * 4 * (g - 1)
    assert LG.allreduce_payload(n, 4, g) == 2 * (-(-n // g)) * 4 * (g - 1)
    assert LG.alltoall_payload(n * g * 2, g) == n * 2 * (g - 1)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not mounted")
@pytest.mark.parametrize("g", [1, 2, 5, 8])
def test_payload_formulas_match_reference(g):
    sys.path.insert(0, REF)
    try:
        from dchag import runtime as RT
    finally:
        sys.path.remove(REF)
    for n in (1, 3, 64, 1001):
        assert LG.allgather_payload(n, g) == RT._ring_allgather_payload(n, g)
        assert LG.allreduce_payload(n, 8, g) == RT._ring_allreduce_payload(n, 8, g)


def test_query_and_csv(tmp_path):
    led = LG.CommLedger()
    for r in range(2):
        led.record(r, "AllGather", "tp", "forward", 100, LG.DCHAG_BOUNDARY_TAG)
        led.record(r, "AllReduce", "tp", "optimizer", 40, LG.POS_GRAD_TAG)
    assert led.query(phase="forward", tag=LG.DCHAG_BOUNDARY_TAG) == (200, 2)
    assert led.query(phase="backward", tag=LG.DCHAG_BOUNDARY_TAG) == (0, 0)
    assert led.query(op="AllReduce", rank=1) == (40, 1)
    assert [e.seq for e in led.per_rank[0]] == [0, 1]
    path = tmp_path / "ledger.csv"
    led.to_csv(path)
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["rank", "seq", "op", "axis", "phase", "payload_bytes_per_rank", "tag"]
    assert rows[1] == ["0", "0", "AllGather", "tp", "forward", "100", "dchag-boundary"]
    assert len(rows) == 5
