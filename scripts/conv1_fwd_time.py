"""Time the conv1 forward (images input, im2col + tcgen05 GEMM + pooled epilogue) of the paper net alone
(CUDA events, L2 flushed between reps); one JSON line.  CP_TC_FWD_T_IMAGES=1 selects the transposed
kernel (pool in registers)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02546_b200 import convpart as cp  # noqa: E402

B, K, P = 128, 500, int(os.environ.get("P", "1"))
part = cp.cp_partition_plan([1.0] * P, K, 8)
d = cp.cp_conv_desc()
d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = B, 3, 32, 32, K, 5, 5
d.bias, d.relu, d.pool, d.math = 1, 1, 1, cp.CP_MATH_TF32
d.input_kind = cp.CP_INPUT_IMAGES
d.out_part, d.rank, d.world = part, 0, P
h = cp.conv_part_create(d, None)
sz = cp.conv_part_query(h)
dev = torch.device("cuda")
x = torch.rand(sz.x // 4, device=dev)
w = torch.randn(sz.w // 4, device=dev) * 0.05
b = torch.zeros(max(sz.b // 4, 1), device=dev)
y = torch.zeros(sz.y // 4, device=dev)
sv = torch.zeros(max(sz.saved, 1), dtype=torch.uint8, device=dev)
ws = torch.zeros(sz.workspace, dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
ts = []
for r in range(22):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.fill_(r)
    e0.record(s)
    cp.conv_part_forward(h, x, w, b, y, sv, ws, s, s)
    e1.record(s)
    torch.cuda.synchronize()
    if r >= 2:
        ts.append(e0.elapsed_time(e1))
print(json.dumps({"P": P, "fwdT_images": os.environ.get("CP_TC_FWD_T_IMAGES", "0"),
                  "conv1_fwd_ms_median": sorted(ts)[len(ts) // 2]}))
cp.conv_part_destroy(h)
