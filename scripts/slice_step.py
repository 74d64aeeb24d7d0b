"""One rank's training step of the paper net at a P-way partition, on ONE GPU with no communicator
(comm=None, LOCAL dX: the compute-only step of bench.py's N=P breakdown), as CUDA-graph replays.
Run it under `ncu --metrics gpu__time_duration.sum` to get the per-kernel launch list of an N=P
rank's compute (ncu cannot profile the multi-rank run itself); without ncu it prints the step time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1712_02546_b200 import convpart as cp  # noqa: E402
from paper_1712_02546_b200.net import PartitionedNet  # noqa: E402

P, R, B = int(os.environ.get("P", "4")), int(os.environ.get("RANK_SLICE", "0")), 128
dev = torch.device("cuda", 0)
net = synth.paper_net("500:1500")
parts = [cp.cp_partition_plan([1.0] * P, K, 8) for K in net.kernels]
pn = PartitionedNet(net.kernels, B, parts, rank=R, comm=None, math=cp.CP_MATH_TF32, device=dev, head="partitioned",
                    in_hw=net.in_hw, fused=False)
pn.load_params(synth.params(net, seed=42))
x, y = synth.images(B, 3, net.in_hw, net.in_hw, step=0)
pn.set_batch(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
s = torch.cuda.current_stream(dev)
cs = torch.cuda.Stream(dev)
run = lambda: pn.step(0.01, cp.CP_DX_LOCAL, torch.cuda.current_stream(dev), cs, True)  # noqa: E731
for _ in range(2):
    run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for it in range(int(os.environ.get("STEPS", "10"))):
    flush.fill_(it)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"P": P, "rank": R, "ms_per_step": sorted(ts)[len(ts) // 2]}), flush=True)
