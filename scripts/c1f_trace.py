"""conv1 forward per-set trace (experiment build with -DC1F_TRACE via CP_LIB): P=1 and P=4 of the paper net."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1712_02546_b200 import convpart as cp

B = 128
for P in (1, 4):
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
    for _ in range(3):
        cp.conv_part_forward(h, x, w, b, y, sv, ws)
    torch.cuda.synchronize()
    cp.conv_part_destroy(h)
