"""Time the three conv2 passes of the paper net in isolation (CUDA events, L2 flushed between
reps) under layout/kernel variants.  Development aid for the roofline work; prints one JSON
line per variant."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02546_b200 import convpart as cp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=128)
ap.add_argument("--P", type=int, default=1)
ap.add_argument("--align", type=int, default=8)
ap.add_argument("--pool", type=int, default=1)
ap.add_argument("--K1", type=int, default=500)
ap.add_argument("--K2", type=int, default=1500)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--math", default="tf32")
ap.add_argument("--H", type=int, default=14, help="input height/width (scaled net conv2: 110)")
a = ap.parse_args()

B, P = a.B, a.P
align = 64 if a.math == "bf16" else a.align
p1 = cp.cp_partition_plan([1.0] * P, a.K1, align)
p2 = cp.cp_partition_plan([1.0] * P, a.K2, align)
d = cp.cp_conv_desc()
d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = B, a.K1, a.H, a.H, a.K2, 5, 5
d.bias, d.relu, d.pool = 1, 1, a.pool
d.math = {"tf32": cp.CP_MATH_TF32, "simt": cp.CP_MATH_FP32_SIMT, "bf16": cp.CP_MATH_BF16}[a.math]
d.input_kind = cp.CP_INPUT_GATHER
d.in_part, d.out_part, d.rank, d.world = p1, p2, 0, P
h = cp.conv_part_create(d, None)
sz = cp.conv_part_query(h)
dev = torch.device("cuda")
x = torch.rand(sz.x // 4, device=dev)
w = torch.randn(sz.w // 4, device=dev) * 0.01
b = torch.zeros(max(sz.b // 4, 1), device=dev)
y = torch.zeros(sz.y // 4, device=dev)
sv = torch.zeros(max(sz.saved, 1), dtype=torch.uint8, device=dev)
ws = torch.zeros(sz.workspace, dtype=torch.uint8, device=dev)
dy = torch.randn(sz.y // 4, device=dev)
dw = torch.zeros_like(w)
db = torch.zeros_like(b)
dx = torch.zeros(sz.dx // 4, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
t = {"fwd": [], "wgrad": [], "dgrad": []}
g = {"fwd": [], "dgrad": [], "wgrad": []}   # the tcgen05 GEMM launch alone (conv_part_timing events)
cp.conv_part_timing(h, True)
for r in range(a.reps + 2):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    flush.fill_(r)
    e[0].record(s)
    cp.conv_part_forward(h, x, w, b, y, sv, ws, s, s)
    e[1].record(s)
    cp.conv_part_backward_filter(h, dy, sv, y, x, dw, db, ws, s)
    e[2].record(s)
    cp.conv_part_backward_data(h, dy, sv, y, w, dx, cp.CP_DX_LOCAL, ws, s, s)
    e[3].record(s)
    torch.cuda.synchronize()
    if r >= 2:
        t["fwd"].append(e[0].elapsed_time(e[1]))
        t["wgrad"].append(e[1].elapsed_time(e[2]))
        t["dgrad"].append(e[2].elapsed_time(e[3]))
        for k, pss in (("fwd", 0), ("dgrad", 1), ("wgrad", 2)):
            g[k].append(cp.conv_part_kernel_time(h, pss))
Kr = p2.k_count[0]
flop = 2.0 * B * Kr * a.K1 * 25 * (a.H - 4) ** 2
med = {k: sorted(v)[len(v) // 2] for k, v in t.items()}
gm = {k: sorted(v)[len(v) // 2] for k, v in g.items()}
peak = 1651.7 * 1.1 / 2.25
print(json.dumps({"variant": vars(a), "cta_group": os.environ.get("CP_TC_CTA_GROUP", "2"), "own_kernels": Kr,
                  "ms": med, "tflops": {k: flop / (v / 1e3) / 1e12 for k, v in med.items()},
                  "gemm_ms": gm, "gemm_tflops": {k: flop / (v / 1e3) / 1e12 for k, v in gm.items() if v > 0},
                  "gemm_frac_of_807": {k: flop / (v / 1e3) / 1e12 / peak for k, v in gm.items() if v > 0}}))
cp.conv_part_destroy(h)
