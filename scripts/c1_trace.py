"""Timeline of the conv1 forward kernel (experiment build with -DC1_TRACE): per-CTA globaltimer stamps."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_1712_02546_b200 import convpart as cp
B = 128
for P in (1, 8):
    part = cp.cp_partition_plan([1.0] * P, 500)
    d = cp.cp_conv_desc()
    d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = B, 3, 32, 32, 500, 5, 5
    d.bias, d.relu, d.pool, d.math, d.input_kind = 1, 1, 1, cp.CP_MATH_TF32, cp.CP_INPUT_IMAGES
    d.out_part, d.rank, d.world = part, 0, P
    h = cp.conv_part_create(d, None)
    sz = cp.conv_part_query(h)
    w = torch.zeros(sz.w // 4, device="cuda"); b = torch.zeros(max(sz.b // 4, 1), device="cuda")
    x = torch.from_numpy(synth.images(B, 3, 32, 32)[0]).cuda()
    ws = torch.zeros(sz.workspace, dtype=torch.uint8, device="cuda")
    y = torch.zeros(sz.y // 4, device="cuda"); sv = torch.zeros(sz.saved, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        cp.conv_part_forward(h, x, w, b, y, sv, ws)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (148 * 8))()
    cp.lib().cp_c1_trace(buf)
    t = np.array(buf, dtype=np.float64).reshape(148, 8)
    t0 = t[:, 0][t[:, 0] > 0].min()
    t = np.where(t > 0, (t - t0) / 1e3, np.nan)
    names = ["entry", "prologue", "1st set built", "1st acc full", "1st epi done", "last epi", "exit"]
    print(f"P={P}: us after the first CTA's entry: min / median / max over CTAs")
    for i, n in enumerate(names):
        col = t[:, i]
        print(f"  {n:14s} {np.nanmin(col):7.2f} {np.nanmedian(col):7.2f} {np.nanmax(col):7.2f}")
    cp.conv_part_destroy(h)
