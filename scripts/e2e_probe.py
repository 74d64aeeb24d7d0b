"""Where does the e2e-vs-device gap go?  Time the graph-replayed paper-net step (N=1) in several
loop shapes, each K steps with the L2 flushed between steps outside the events:
  A  device: ev0, replay, ev1, host sync                           (bench value)
  B  e2e as bench: ev0, wait H2D, D2D x/labels, prefetch next, replay, D2H loss, ev1, host sync + read
  C  B without the per-step host sync (host runs ahead)
  D  B with the whole pre-step work enqueued before ev0 except the D2D copies (host gap check)
  E  ev0, D2D x/labels, replay, ev1 (no H2D at all)
  F  ev0, replay, D2H loss, ev1"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1712_02546_b200 import convpart as cp
from paper_1712_02546_b200.net import PartitionedNet

K = 20
net = synth.paper_net("500:1500")
B = 128
dev = torch.device("cuda", 0)
parts = [cp.cp_partition_plan([1.0], k) for k in net.kernels]
pn = PartitionedNet(net.kernels, B, parts, device=dev)
pn.load_params(synth.params(net, seed=42))
x, y = synth.images(B, 3, 32, 32)
xh, yh = torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()
pn.set_batch(xh.to(dev), yh.to(dev))
s = torch.cuda.current_stream()
cs = torch.cuda.Stream()
for _ in range(3):
    pn.step(0.01, cp.CP_DX_REDUCE_SCATTER, s, cs, True)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    pn.step(0.01, cp.CP_DX_REDUCE_SCATTER, torch.cuda.current_stream(), cs, True)
g.replay(); torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
cpy = torch.cuda.Stream()
stage = [(torch.empty_like(pn.x), torch.empty_like(pn.labels)) for _ in range(2)]
ready = [torch.cuda.Event() for _ in range(2)]
free = [torch.cuda.Event() for _ in range(2)]
lh = torch.empty(1).pin_memory()


def prefetch(k):
    j = k & 1
    with torch.cuda.stream(cpy):
        cpy.wait_event(free[j])
        stage[j][0].copy_(xh.reshape(-1), non_blocking=True)
        stage[j][1].copy_(yh, non_blocking=True)
        ready[j].record(cpy)


def run(mode):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for j in range(2):
        free[j].record(s)
    torch.cuda.synchronize()
    host = 0.0
    for k in range(K):
        j = k & 1
        flush.fill_(k & 0xFF)
        if mode == "D":
            if k == 0:
                cpy.wait_stream(s); prefetch(0)
            s.wait_event(ready[j])
        t0 = time.perf_counter()
        ev[k][0].record(s)
        if mode in ("B", "C"):
            if k == 0:
                cpy.wait_stream(s); prefetch(0)
            s.wait_event(ready[j])
        if mode in ("B", "C", "D", "E"):
            pn.x.copy_(stage[j][0] if mode != "E" else pn.x)
            pn.labels.copy_(stage[j][1] if mode != "E" else pn.labels)
        if mode in ("B", "C", "D"):
            free[j].record(s)
            if k + 1 < K:
                cpy.wait_stream(s); prefetch(k + 1)
        g.replay()
        if mode in ("B", "C", "D", "F"):
            lh.copy_(pn.head["loss"][:1], non_blocking=True)
        ev[k][1].record(s)
        host += time.perf_counter() - t0
        if mode != "C":
            ev[k][1].synchronize()
            _ = float(lh[0])
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / K
    print(f"{mode}: {ms:.4f} ms/step  ({B / ms * 1e3:.0f} img/s)  host enqueue {host / K * 1e3:.3f} ms/step", flush=True)


for rep in range(2):
    for m in "ABCDEF":
        run(m)
