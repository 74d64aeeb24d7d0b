"""Stage-by-stage comparison of the LRN training step (SIMT mode, P=1) with the oracle (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as orc, synth
from gpu_util import unpack, rel_err, dev
from paper_1712_02546_b200 import convpart as cp
from paper_1712_02546_b200.net import PartitionedNet, plan_even
LRN = {"depth": 5, "alpha": 0.05, "beta": 0.75, "bias": 2.0}
net = synth.NetSpec(kernels=(24, 40), in_hw=20, name="small")
B = 40
params = synth.params(net, seed=12, std=0.05, bias_std=0.01)
x, y = synth.images(B, 3, 20, 20, step=2)
for lrn in (None, LRN):
    pn = PartitionedNet(net.kernels, B, plan_even(net.kernels, 1), math=cp.CP_MATH_FP32_SIMT, in_hw=20, lrn=lrn)
    pn.load_params(params)
    pn.set_batch(dev(x), dev(y, torch.int32))
    pn.forward(); torch.cuda.synchronize()
    rep = []
    for i, K in enumerate(net.kernels):
        if lrn:
            ho = pn.buf[i]["hw"]
            rep.append({"a": unpack(pn.buf[i]["yp"], B, K, ho // 2, pn.parts[i]),
                        "argmax": np.rint(unpack(pn.buf[i]["codes"].float(), B, K, ho // 2, pn.parts[i])).astype(np.uint8),
                        "pre": unpack(pn.buf[i]["y"], B, K, ho, pn.parts[i])})
        else:
            hp = 8 if i == 0 else 2
            am = torch.zeros(B * K * hp * hp, dtype=torch.uint8, device="cuda")
            cp.cp_unpack_saved(pn.buf[i]["saved"], B, hp, hp, pn.parts[i], 0, am)
            rep.append({"a": unpack(pn.buf[i]["y"], B, K, hp, pn.parts[i]), "argmax": am.reshape(B, K, hp, hp).cpu().numpy()})
    pn.backward(); torch.cuda.synchronize()
    p64 = {k: v.astype(np.float64) for k, v in params.items()}
    layers = [dict(L, lrn=lrn) if lrn else dict(L) for L in net.layers()]
    tr = orc.net_step(p64, x.astype(np.float64), y, 0.01, layers, replay=rep)
    print("== lrn" if lrn else "== plain", "loss", pn.loss(), tr["loss"])
    hp2 = 2
    print(" da(head)", rel_err(unpack(pn.head["da"], B, 40, hp2, pn.parts[1]), tr["da1"]))
    if lrn:
        print(" dpre2", rel_err(unpack(pn.buf[1]["dpre"], B, 40, 4, pn.parts[1]) * (rep[1]["pre"] > 0), tr["dy1"]))
        print(" a1 (conv2 input)", rel_err(rep[0]["a"], tr["in1"]))
    gw = pn.buf[1]["dw"]
    d = pn.descs[1]
    t = torch.zeros(40 * 24 * 25, device="cuda")
    cp.cp_unpack_conv_weights(d, gw, t)
    print(" dW1", rel_err(t.reshape(40, 24, 5, 5).cpu().numpy(), tr["grads"]["w1"]))
    print(" dW1 from the oracle's dy1 and the GPU's input:",
          rel_err(t.reshape(40, 24, 5, 5).cpu().numpy(), orc.conv_wgrad(tr["dy1"], rep[0]["a"], 5, 5)))
    pn.close()
