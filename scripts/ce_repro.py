"""Reproduce the CE-gather failure: paper net, replicated head, N ranks, one eager forward + backward,
a device sync + error check after every library call (rank-tagged progress on stderr)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import torch.distributed as dist
from paper_1712_02546_b200 import convpart as cp
from full_size import bench_setup

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
uid = [cp.cp_comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
comm = cp.cp_comm_create(uid[0], rank, world)
head = os.environ.get("HEAD", "replicated")
net, parts, pn, params, x, y = bench_setup(world, rank, comm, dev, head=head)
s = torch.cuda.current_stream(dev)
cs = torch.cuda.Stream(dev)


def step(name):
    try:
        torch.cuda.synchronize(dev)
        print(f"[r{rank}] ok after {name}", file=sys.stderr, flush=True)
    except Exception as e:
        print(f"[r{rank}] FAILED after {name}: {e}", file=sys.stderr, flush=True)
        raise


for it in range(2):
    inp = pn.x
    for i, L in enumerate(pn.layers):
        b = pn.buf[i]
        cp.conv_part_forward(L, inp, b["w"], b["b"], b["y"], b["saved"], b["ws"], s, cs)
        step(f"it{it} conv{i + 1} forward")
        inp = b["y"]
    last = next((m for m in pn.sym if m.tensor.data_ptr() == pn.buf[-1]["y"].data_ptr()), None)
    if last is not None:
        last.wait(s)
        step(f"it{it} symmetric wait (replicated head gather)")
    hd = pn.head
    cp.cp_fc_forward(pn.head_x, pn.B, pn.Hp, pn.Wp, pn.head_part, hd["wfc"], hd["bfc"], pn.O, hd["logits"], hd["ws"], s)
    step(f"it{it} fc forward")
    cp.cp_softmax_xent(hd["logits"], pn.labels, pn.B, pn.O, hd["loss"], hd["dlogits"], s)
    step(f"it{it} softmax")
    pn.backward(cp.CP_DX_REDUCE_SCATTER, s, cs, overlap=True)
    step(f"it{it} backward")
print(f"[r{rank}] done", file=sys.stderr, flush=True)
torch.cuda.synchronize(dev)
dist.barrier()
pn.close()
cp.cp_comm_destroy(comm)
dist.destroy_process_group()
