"""Per-pass diagnostics of the tcgen05 path vs the oracle (development aid)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle as orc  # noqa: E402
import synth  # noqa: E402
from gpu_util import LocalLayer, dev, pack, rel_err, unpack  # noqa: E402
from paper_1712_02546_b200 import convpart as cp  # noqa: E402


def stats(name, g, r):
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    print(f"{name:28s} rel={rel_err(g, r):.3e}  |g|max={np.abs(g).max():.3e} |r|max={np.abs(r).max():.3e} "
          f"nz(g)={np.count_nonzero(g) / g.size:.3f} nz(r)={np.count_nonzero(r) / r.size:.3f} "
          f"nan(g)={np.isnan(g).sum()}")


def run(B=32, H=12, K1=32, K2=32, math=cp.CP_MATH_TF32, seed=3):
    print(f"--- B={B} H={H} K1={K1} K2={K2} math={math}")
    x, _ = synth.images(B, 3, H, H, step=seed)
    w1 = synth.normal((K1, 3, 5, 5), seed + 1, 0.05)
    b1 = synth.normal((K1,), seed + 2, 0.05)
    Hp1 = (H - 4) // 2
    w2 = synth.normal((K2, K1, 5, 5), seed + 3, 0.02)
    b2 = synth.normal((K2,), seed + 4, 0.02)
    p1 = cp.cp_partition_plan([1.0], K1)
    p2 = cp.cp_partition_plan([1.0], K2)
    L1 = LocalLayer(B, 3, H, K1, 5, p1, None, math)
    L1.load(w1, b1)
    xd = dev(x)
    L1.forward(xd)
    torch.cuda.synchronize()
    z1 = orc.conv_fwd(x.astype(np.float64), w1.astype(np.float64), b1.astype(np.float64))
    a1, _ = orc.relu_pool_fwd(z1)
    y1 = L1.y_nchw()
    stats("conv1 fwd", y1, a1)
    L2 = LocalLayer(B, K1, Hp1, K2, 5, p2, p1, math)
    L2.load(w2, b2)
    L2.forward(L1.y)
    torch.cuda.synchronize()
    z2 = orc.conv_fwd(y1, w2.astype(np.float64), b2.astype(np.float64))
    a2, _ = orc.relu_pool_fwd(z2)
    y2 = L2.y_nchw()
    stats("conv2 fwd", y2, a2)
    am2 = L2.argmax_nchw()
    da2 = synth.normal(y2.shape, 99, 1.0).astype(np.float32)
    dxs, dw2, db2 = L2.backward(pack(da2, p2), L1.y)
    torch.cuda.synchronize()
    dy2 = orc.unpool_relu_bwd(da2.astype(np.float64), am2, y2)
    # GPU dY lives at the start of the workspace (gather input, TF32: no xcol / z regions)
    Ho2 = Hp1 - 4
    Bp = (B + 31) // 32 * 32
    Kc2 = p2.k_width[0]
    gdy = L2.ws[0][: Ho2 * Ho2 * Bp * Kc2 * 4].view(torch.float32).reshape(Ho2, Ho2, Bp, Kc2)
    gdy = gdy[:, :, :B, :K2].permute(2, 3, 0, 1).cpu().numpy()
    stats("dY2 (unpool)", gdy, dy2)
    stats("conv2 dgrad", unpack(dxs, B, K1, Hp1, p1), orc.conv_dgrad(dy2, w2.astype(np.float64)))
    stats("conv2 wgrad", dw2, orc.conv_wgrad(dy2, y1, 5, 5))
    stats("conv2 db", db2, orc.bias_grad(dy2))
    L1.close()
    L2.close()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for cfg in [dict(B=32, H=16, K1=32, K2=32), dict(B=32, H=16, K1=32, K2=32, math=cp.CP_MATH_FP32_SIMT),
                dict(B=40, H=20, K1=70, K2=300)]:
        try:
            run(**cfg)
        except Exception as e:  # keep going
            print("ERROR", type(e).__name__, e)
