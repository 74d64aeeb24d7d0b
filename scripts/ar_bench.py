"""Latency of the logits AllReduce (cp_allreduce_sum, one-shot over NVLink peer memory) vs NCCL, N ranks:
a CUDA graph of 50 back-to-back calls, CUDA events, max over ranks."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_1712_02546_b200 import convpart as cp

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
uid = [cp.cp_comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
comm = cp.cp_comm_create(uid[0], rank, world)
sym = cp.SymmetricBuffer(comm, 1 << 20, dev)   # first symmetric allocation creates the control line
buf = torch.ones(int(os.environ.get("N", "1280")), device=dev)
s = torch.cuda.current_stream(dev)
res = {}
for name, fn in (("oneshot", lambda st: cp.cp_allreduce_sum(comm, buf, st)),
                 ("nccl", lambda st: dist.all_reduce(buf))):
    for _ in range(5):
        fn(s)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(50):
            fn(torch.cuda.current_stream(dev))
    ts = []
    for it in range(10):
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize(dev)
        ts.append(e0.elapsed_time(e1) * 1e3 / 50)
    t = torch.tensor([sorted(ts)[len(ts) // 2]], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res[name] = round(float(t), 2)
    del g
if rank == 0:
    print(json.dumps({"world": world, "floats": buf.numel(), "us_per_call": res}), flush=True)
torch.cuda.synchronize(dev)
dist.barrier()
sym.free()
cp.cp_comm_destroy(comm)
dist.destroy_process_group()
