"""conv1 (image layer) pass times (CUDA-graph replays: GPU time only), old path (im2col + tc_fwd / unpool + tc_wgrad) vs the dedicated kernels
(CP_C1_FWD / CP_C1_WGRAD), paper net shapes, rank 0 of P simulated slices (no collectives), L2 flushed,
CUDA events; also checks old vs new outputs agree (TF32 tolerance) on the same inputs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1712_02546_b200 import convpart as cp

B = int(os.environ.get("B", "128"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for P in (1, 2, 4, 8):
    part = cp.cp_partition_plan([1.0] * P, 500)
    d = cp.cp_conv_desc()
    d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = B, 3, 32, 32, 500, 5, 5
    d.bias, d.relu, d.pool, d.math, d.input_kind = 1, 1, 1, cp.CP_MATH_TF32, cp.CP_INPUT_IMAGES
    d.out_part, d.rank, d.world = part, 0, P
    h = cp.conv_part_create(d, None)
    sz = cp.conv_part_query(h)
    w = torch.zeros(sz.w // 4, device="cuda")
    cp.cp_pack_conv_weights(d, torch.from_numpy(synth.normal((500, 3, 5, 5), 1, 0.05)).cuda(), w)
    b = torch.from_numpy(synth.normal((sz.b // 4,), 2, 0.05)).cuda()
    x = torch.from_numpy(synth.images(B, 3, 32, 32)[0]).cuda()
    ws = torch.zeros(sz.workspace, dtype=torch.uint8, device="cuda")
    y = torch.zeros(sz.y // 4, device="cuda")
    sv = torch.zeros(sz.saved, dtype=torch.uint8, device="cuda")
    da = torch.from_numpy(synth.normal((sz.y // 4,), 3, 1.0)).cuda()
    dw = torch.zeros(sz.w // 4, device="cuda")
    db = torch.zeros(max(sz.b // 4, 1), device="cuda")
    out = {}
    for mode in ("old", "new"):
        os.environ["CP_C1_FWD"] = os.environ["CP_C1_WGRAD"] = "1" if mode == "new" else "0"
        t = {"fwd": [], "bwd_filter": []}
        run_f = lambda: cp.conv_part_forward(h, x, w, b, y, sv, ws, torch.cuda.current_stream())  # noqa: E731
        run_b = lambda: cp.conv_part_backward_filter(h, da, sv, y, x, dw, db, ws, torch.cuda.current_stream())  # noqa
        run_f(); run_b(); torch.cuda.synchronize()
        graphs = {}
        for name, fn in (("fwd", run_f), ("bwd_filter", run_b)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            graphs[name] = g
        for it in range(12):
            for name in ("fwd", "bwd_filter"):
                flush.fill_(it)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graphs[name].replay()
                e1.record()
                torch.cuda.synchronize()
                if it >= 2:
                    t[name].append(e0.elapsed_time(e1))
        del graphs
        out[mode] = {"y": y.clone(), "sv": sv.clone(), "dw": dw.clone(), "db": db.clone(),
                     "ms": {k: sorted(v)[len(v) // 2] for k, v in t.items()}}
    rel = lambda a, r: float((a - r).abs().max() / r.abs().max().clamp_min(1e-30))
    line = {"P": P, "K_r": part.k_count[0], "old_ms": out["old"]["ms"], "new_ms": out["new"]["ms"],
            "y_rel": rel(out["new"]["y"], out["old"]["y"]), "codes_diff": int((out["new"]["sv"] != out["old"]["sv"]).sum()),
            "dw_rel": rel(out["new"]["dw"], out["old"]["dw"]), "db_rel": rel(out["new"]["db"], out["old"]["db"])}
    print(json.dumps(line), flush=True)
    cp.conv_part_destroy(h)
