"""Compute-only step time of one rank of a P-way kernel split (no collectives: comm=None), to compare
with bench.py's N=P step and read off the exposed communication.  Prints one JSON line per P."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1712_02546_b200 import convpart as cp
from paper_1712_02546_b200.net import PartitionedNet

B = int(os.environ.get("B", "128"))
for P in [int(p) for p in os.environ.get("PS", "1,2,4").split(",")]:
    net = synth.paper_net("500:1500")
    parts = [cp.cp_partition_plan([1.0] * P, K) for K in net.kernels]
    pn = PartitionedNet(net.kernels, B, parts, rank=0, comm=None, head="partitioned")
    pn.load_params(synth.params(net, seed=42))
    x, y = synth.images(B, 3, 32, 32)
    pn.set_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(5):
            pn.step(0.01, cp.CP_DX_LOCAL, s, s, False)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            pn.step(0.01, cp.CP_DX_LOCAL, s, s, False)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"P": P, "B": B, "ms_median": ts[len(ts) // 2], "ms_min": ts[0]}), flush=True)
    del g
    pn.close()
