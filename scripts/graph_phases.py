"""Per-phase GPU time of one training step INSIDE its CUDA graph (external event-record nodes on the
compute stream between the phases), N ranks under torchrun, next to the same rank's compute-only step
(comm=None).  Unlike phase_times.py (eager launches) no host launch gaps enter the phases."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import synth
from paper_1712_02546_b200 import convpart as cp
from paper_1712_02546_b200.net import PartitionedNet

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
B = int(os.environ.get("B", "128"))
fused = os.environ.get("FUSED", "1") == "1"
comm = None
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
    uid = [cp.cp_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = cp.cp_comm_create(uid[0], rank, world)
net = synth.paper_net("500:1500")
parts = [cp.cp_partition_plan([1.0] * world, K) for K in net.kernels]


def phases(pn, s, cs):
    ev = []
    mark = lambda name: (ev.append((name, torch.cuda.Event(enable_timing=True, external=True))),  # noqa
                         ev[-1][1].record(torch.cuda.current_stream(dev)))
    mark("start")
    inp = pn.x
    for i, L in enumerate(pn.layers):
        b = pn.buf[i]
        cp.conv_part_forward(L, inp, b["w"], b["b"], b["y"], b["saved"], b["ws"], s, cs)
        inp = b["y"]
        mark(f"conv{i + 1}_fwd")
    hd = pn.head
    bias = hd["bfc"] if pn.rank == 0 else None
    cp.cp_fc_forward(pn.head_x, pn.B, pn.Hp, pn.Wp, pn.head_part, hd["wfc"], bias, pn.O, hd["logits"], hd["ws"], s)
    mark("fc_fwd")
    if pn.comm is not None:
        cp.cp_allreduce_softmax_xent(pn.comm, hd["logits"], pn.labels, pn.B, pn.O, hd["loss"], hd["dlogits"], s)
    else:
        cp.cp_softmax_xent(hd["logits"], pn.labels, pn.B, pn.O, hd["loss"], hd["dlogits"], s)
    mark("logits_allreduce+softmax")
    cp.cp_fc_backward(hd["dlogits"], pn.head_x, pn.B, pn.Hp, pn.Wp, pn.head_part, hd["wfc"], pn.O, pn.head_da,
                      hd["dwfc"], hd["dbfc"], hd["ws"], s)
    mark("fc_bwd")
    da = hd["da"]
    for i in reversed(range(len(pn.layers))):
        L, b = pn.layers[i], pn.buf[i]
        xin = pn.x if i == 0 else pn.buf[i - 1]["y"]
        if i > 0:
            cp.conv_part_backward_data(L, da, b["saved"], b["y"], b["w"], b["dx"],
                                       cp.CP_DX_REDUCE_SCATTER | cp.CP_DX_ASYNC | cp.CP_DX_ORDERED, b["ws"], s, cs)
            mark(f"conv{i + 1}_dgrad")
        cp.conv_part_backward_filter(L, da, b["saved"], b["y"], xin, b["dw"], b["db"], b["ws"], s)
        mark(f"conv{i + 1}_wgrad")
        if i > 0:
            cp.conv_part_wait(L, s)
            mark(f"conv{i + 1}_dx_wait")
            da = b["dx"]
    pn.sgd(0.01, s)
    mark("sgd")
    return ev


def run(pn, label):
    pn.load_params(synth.params(net, seed=42))
    x, y = synth.images(B, 3, 32, 32)
    pn.set_batch(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
    s, cs = torch.cuda.current_stream(dev), torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        phases(pn, s, cs)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ev = phases(pn, torch.cuda.current_stream(dev), cs)
    acc = None
    for it in range(25):
        flush.zero_()
        if comm is not None:
            torch.cuda.synchronize(dev)
            dist.barrier()
        g.replay()
        torch.cuda.synchronize(dev)
        if it >= 5:
            d = [(ev[k][0], ev[k - 1][1].elapsed_time(ev[k][1]) * 1e3) for k in range(1, len(ev))]
            acc = [[n, [t]] for n, t in d] if acc is None else [[n, a + [t]] for (n, a), (_, t) in zip(acc, d)]
    med = {n: sorted(a)[len(a) // 2] for n, a in acc}
    med["total_us"] = sum(med.values())
    print(json.dumps({"rank": rank, "world": world, "mode": label, "graph": True,
                      "us": {k: round(v, 1) for k, v in med.items()}}), flush=True)
    del g


pn = PartitionedNet(net.kernels, B, parts, rank=rank, comm=comm, device=dev, head="partitioned", fused=fused)
run(pn, "fused-gather" if fused and world > 1 else "nccl")
pn.close()
pn = PartitionedNet(net.kernels, B, parts, rank=rank, comm=None, device=dev, head="partitioned")
run(pn, "compute-only")
pn.close()
if comm is not None:
    torch.cuda.synchronize()
    dist.barrier()
    cp.cp_comm_destroy(comm)
    dist.destroy_process_group()
