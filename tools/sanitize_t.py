"""Tiny workload for compute-sanitizer (memcheck / racecheck / synccheck): the T config
forward (K_p0, K_l0, K_gemm, K_comb), a P8 forward at the fused-level shape (K_gemm COMB),
and one training step (every backward kernel), each checked against nothing -- the sanitizer
is the checker. Usage: compute-sanitizer --tool racecheck python tools/sanitize_t.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_21411_b200 import DchagFrontEnd  # noqa: E402
from paper_2506_21411_b200.train import DchagTrainer  # noqa: E402

torch.manual_seed(0)
fe = DchagFrontEnd(16, 64, 64, 4, 128, 2, max_group=8)          # T config
fe.init_weights(seed=0)
x = torch.randn(2, 16, 64, 64, device="cuda").to(torch.bfloat16)
fe(x)
fe2 = DchagFrontEnd(64, 64, 128, 8, 1024, 16, max_group=8)      # fused level (COMB), P8
fe2.init_weights(seed=1)
x2 = torch.randn(2, 64, 64, 128, device="cuda").to(torch.bfloat16)
fe2(x2)
fe3 = DchagFrontEnd(24, 64, 128, 8, 256, 4, max_group=4, out_dtype=torch.float32)
fe3.init_weights(seed=2)
tr = DchagTrainer(fe3)
x3 = torch.randn(2, 24, 64, 128, device="cuda").to(torch.bfloat16)
out, saved = tr.forward_train(x3)
tr.backward(saved, torch.randn_like(out))
torch.cuda.synchronize()
print("sanitize workload done")
