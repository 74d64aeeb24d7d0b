"""Head kernels alone (FC forward + reduce, softmax-xent, FC backward) at the paper net's shapes: P=1
(all 1504 slots x 25 positions) and the P=4 partitioned head (rank 0's 376 slots), B=128; CUDA graph
of each call, L2 flushed between replays, CUDA events.  Variant libraries via CP_LIB."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1712_02546_b200 import convpart as cp

B, O, Hp = 128, 10, 5
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {"lib": os.environ.get("CP_LIB", "default")}
for P in (1, 4):
    full = cp.cp_partition_plan([1.0] * P, 1500)
    if P == 1:
        part = full
    else:   # rank 0's own channels only (partitioned head)
        part = cp.cp_partition.from_counts([full.k_count[0]])
    F = part.num_k * Hp * Hp
    Fg = sum(part.k_width[r] for r in range(part.n_ranks)) * Hp * Hp
    x = torch.randn(Fg * ((B + 31) // 32 * 32) + 64, device="cuda") * 0.1
    wg = torch.randn(O * Fg + 64, device="cuda") * 0.01
    bfc = torch.zeros(O, device="cuda")
    logits = torch.zeros(B * O, device="cuda")
    ws = torch.zeros(cp.cp_head_workspace_bytes(B, Hp, Hp, part, O) // 4 + 64, device="cuda")
    labels = torch.randint(0, O, (B,), dtype=torch.int32, device="cuda")
    loss = torch.zeros(1, device="cuda")
    dl = torch.zeros(B * O, device="cuda")
    dx = torch.zeros_like(x)
    dwg = torch.zeros_like(wg)
    dbfc = torch.zeros(O, device="cuda")
    calls = {
        "fc_fwd": lambda: cp.cp_fc_forward(x, B, Hp, Hp, part, wg, bfc, O, logits, ws, torch.cuda.current_stream()),
        "softmax": lambda: cp.cp_softmax_xent(logits, labels, B, O, loss, dl, torch.cuda.current_stream()),
        "fc_bwd": lambda: cp.cp_fc_backward(dl, x, B, Hp, Hp, part, wg, O, dx, dwg, dbfc, ws,
                                            torch.cuda.current_stream()),
    }
    res = {}
    for name, fn in calls.items():
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        ts = []
        for it in range(30):
            flush.fill_(it)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        res[name] = round(sorted(ts)[len(ts) // 2], 2)
        del g
    out[f"P{P}_us"] = res
print(json.dumps(out), flush=True)
