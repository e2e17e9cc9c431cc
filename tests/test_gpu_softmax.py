"""dchag_child_softmax (csrc/comb.cu): the softmax over a parent's children of the level >= 1
logits (layers.py:114-120), in place on L [children][R][H], against torch. Up to 16 children
take the register path (one load and one store per logit), more take the loop path."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("counts", [(2, 3), (15, 16), (16, 17), (40,), (1, 64, 7)])
def test_child_softmax_matches_torch(counts):
    from paper_2506_21411_b200 import _lib as L
    R, H = 384, 12
    total = sum(counts)
    gen = torch.Generator().manual_seed(sum(counts))
    logits = (torch.randn(total, R, H, generator=gen) * 4).cuda()
    first = torch.tensor([sum(counts[:i]) for i in range(len(counts))], dtype=torch.int32,
                         device="cuda")
    count = torch.tensor(counts, dtype=torch.int32, device="cuda")
    out = logits.clone()
    L.call("dchag_child_softmax", L.ptr(out), L.ptr(first), L.ptr(count), len(counts), R, H,
           L.stream_handle())
    torch.cuda.synchronize()
    at = 0
    for c in counts:
        want = torch.softmax(logits[at:at + c].double(), dim=0)
        torch.testing.assert_close(out[at:at + c].double(), want, rtol=1e-5, atol=1e-6)
        at += c
