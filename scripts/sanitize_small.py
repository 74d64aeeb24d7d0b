"""Small end-to-end exercise of every library kernel for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run): conv fwd/dgrad/wgrad in both math modes, 1-CTA and CTA-pair tiles,
split-K, spanning N tiles, the head and SGD, at tiny shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from gpu_util import LocalLayer, dev, pack  # noqa: E402
from paper_1712_02546_b200 import convpart as cp  # noqa: E402
from paper_1712_02546_b200.net import PartitionedNet, plan_even  # noqa: E402

torch.cuda.set_device(0)
for math in (cp.CP_MATH_TF32, cp.CP_MATH_FP32_SIMT):
    for P, B, align in [(1, 40, 8), (2, 64, 32)]:
        x, _ = synth.images(B, 3, 16, 16, step=1)
        p1 = cp.cp_partition_plan([1.0] * P, 40, align)
        p2 = cp.cp_partition_plan([1.0] * P, 96, align)
        L1 = LocalLayer(B, 3, 16, 40, 5, p1, None, math)
        L1.load(synth.normal((40, 3, 5, 5), 1, 0.05), synth.normal((40,), 2, 0.05))
        xd = dev(x)
        L1.forward(xd)
        L2 = LocalLayer(B, 40, 6, 96, 3, p2, p1, math, pool=True)
        L2.load(synth.normal((96, 40, 3, 3), 3, 0.05), synth.normal((96,), 4, 0.05))
        L2.forward(L1.y)
        da2 = synth.normal((B, 96, 2, 2), 5).astype(np.float32)
        dxs, _, _ = L2.backward(pack(da2, p2), L1.y)
        L1.backward(dxs, xd)
        torch.cuda.synchronize()
        L1.close()
        L2.close()
net = synth.NetSpec(kernels=(16, 40), in_hw=20, name="san")
pn = PartitionedNet(net.kernels, 32, plan_even(net.kernels, 1), in_hw=20)
pn.load_params(synth.params(net, seed=5))
x, y = synth.images(32, 3, 20, 20)
pn.set_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
pn.step(0.01)
torch.cuda.synchronize()
pn.close()
print("sanitize_small: ok")
