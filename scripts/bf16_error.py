"""Measured error of the bf16 operand mode (f4) per pass vs the fp64 oracle (max|gpu-ref|/max|ref|),
next to the TF32 mode on the same inputs.  One JSON line per (mode, P)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as orc, synth
from gpu_util import LocalLayer, dev, pack, unpack, rel_err
from paper_1712_02546_b200 import convpart as cp

B = 128
x, _ = synth.images(B, 3, 20, 20, step=3)
w1 = synth.normal((70, 3, 5, 5), 4, 0.05); b1 = synth.normal((70,), 5, 0.05)
w2 = synth.normal((300, 70, 5, 5), 6, 0.02); b2 = synth.normal((300,), 7, 0.02)
for name, m in (("tf32", cp.CP_MATH_TF32), ("bf16", cp.CP_MATH_BF16)):
    for P in (1, 2):
        al = 64 if m == cp.CP_MATH_BF16 else 8
        p1, p2 = cp.cp_partition_plan([1.0] * P, 70, al), cp.cp_partition_plan([1.0] * P, 300, al)
        L1 = LocalLayer(B, 3, 20, 70, 5, p1, None, m); L1.load(w1, b1); xd = dev(x); L1.forward(xd)
        y1 = L1.y_nchw()
        a1, _ = orc.relu_pool_fwd(orc.conv_fwd(x.astype(np.float64), w1.astype(np.float64), b1.astype(np.float64)))
        L2 = LocalLayer(B, 70, 8, 300, 5, p2, p1, m); L2.load(w2, b2); L2.forward(L1.y)
        y2 = L2.y_nchw()
        a2, _ = orc.relu_pool_fwd(orc.conv_fwd(y1, w2.astype(np.float64), b2.astype(np.float64)))
        da2 = synth.normal(y2.shape, 99, 1.0).astype(np.float32)
        dxs, dw2, _ = L2.backward(pack(da2, p2), L1.y)
        dy2 = orc.unpool_relu_bwd(da2.astype(np.float64), L2.argmax_nchw(), y2)
        print(json.dumps({"mode": name, "P": P, "fwd1": rel_err(y1, a1), "fwd2": rel_err(y2, a2),
                          "dgrad": rel_err(unpack(dxs, B, 70, 8, p1), orc.conv_dgrad(dy2, w2.astype(np.float64))),
                          "wgrad": rel_err(dw2, orc.conv_wgrad(dy2, y1, 5, 5))}), flush=True)
        L1.close(); L2.close()
