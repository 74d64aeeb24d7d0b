"""One profiled training step (inside an NVTX range "step") after warm-up, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1712_02546_b200 import convpart as cp
from paper_1712_02546_b200.net import PartitionedNet

B = int(os.environ.get("B", "128"))
P = int(os.environ.get("P", "1"))      # simulated partition width (this process is rank 0 of P)
net = synth.paper_net("500:1500")
parts = [cp.cp_partition_plan([1.0] * P, K) for K in net.kernels]
pn = PartitionedNet(net.kernels, B, parts, rank=0, comm=None)
pn.load_params(synth.params(net, seed=42))
x, y = synth.images(B, 3, 32, 32)
pn.set_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
for _ in range(3):
    pn.step(0.01)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
pn.step(0.01)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("loss", pn.loss())
