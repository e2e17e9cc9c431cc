import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_21411_b200 import DchagFrontEnd
from paper_2506_21411_b200.train import DchagTrainer
lk = sys.argv[1] if len(sys.argv) > 1 else "linear"
fe = DchagFrontEnd(12, 64, 128, 8, 256, 4, max_group=3, agg_layer_kind=lk, out_dtype=torch.float32)
fe.init_weights(seed=3, all_ranks=False)
tr = DchagTrainer(fe)
gen = torch.Generator(device="cuda").manual_seed(0)
img = torch.randn(2, 12, 64, 128, device="cuda", generator=gen).to(torch.bfloat16)
probe = torch.randn(2, 1, fe.seq, 256, device="cuda", generator=gen)
o1, _ = tr.forward_train(img.clone())
o2, _ = tr.forward_train(img.clone())
print("eager-eager equal", torch.equal(o1, o2), o1.abs().max().item())
y1 = fe(img.clone()); 
print("fe fwd vs train fwd rel", ((y1.float() - o1.float()).norm() / o1.norm()).item())
gs = tr.capture(img, probe)
gs.replay(); torch.cuda.synchronize()
print("graph vs eager same input rel", ((gs.out - o1).norm() / o1.norm()).item())
img2 = torch.randn(2, 12, 64, 128, device="cuda", generator=gen).to(torch.bfloat16)
o_before = gs.out.clone()
img.copy_(img2)
gs.replay(); torch.cuda.synchronize()
oe, _ = tr.forward_train(img2)
print("graph changed with input:", not torch.equal(o_before, gs.out),
      "graph vs eager(img2) rel", ((gs.out - oe).norm() / oe.norm()).item(),
      "graph vs eager(img1) rel", ((gs.out - o1).norm() / o1.norm()).item())
gs.replay(); torch.cuda.synchronize()
print("second replay vs eager(img2) rel", ((gs.out - oe).norm() / oe.norm()).item())
