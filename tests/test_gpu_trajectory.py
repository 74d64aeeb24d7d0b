"""Multi-step loss-trajectory parity (SURVEY §8(c) protocol (iii); training progress S:L363).

Ten SGD steps of the kernel-partitioned network on the GPU (PartitionedNet, the bench's code path:
CUDA-graph-free eager calls of the same C ABI) next to ten steps of the fp64 oracle, each side on
its own parameter trajectory from the same seeded initialisation, a fresh seeded batch per step.
Decision replay per step (reading R15): the oracle's backward takes the GPU's pooling codes and ReLU
map of that step, so a flipped argmax cannot send the two gradients down different paths; the
forward disagreements are counted and reported, not failed.

Band: the loss is a mean of B cross-entropies of logits computed through two TF32 layers; each
layer's output is within the per-tensor 2e-3 bar (north_star), so the per-step loss must be within
2e-3 relative (TF32) / 1e-5 (FP32 SIMT) - the same bar as one step - for all ten steps: the
trajectories must not drift apart.  The oracle's own loss must also fall (training progresses).
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1712_02546_b200 import convpart as cp
    from gpu_util import TOL, dev, unpack


@pytest.mark.parametrize("math", ["simt", "tf32"])
def test_loss_trajectory_10_steps(orc, math):
    from paper_1712_02546_b200.net import PartitionedNet, plan_even
    m = cp.CP_MATH_FP32_SIMT if math == "simt" else cp.CP_MATH_TF32
    net = synth.NetSpec(kernels=(24, 40), in_hw=20, name="small")
    B, steps, lr = 40, 10, 0.05
    params = synth.params(net, seed=21, std=0.05, bias_std=0.01)
    pn = PartitionedNet(net.kernels, B, plan_even(net.kernels, 1), math=m, in_hw=20)
    pn.load_params(params)
    theta = {k: v.astype(np.float64) for k, v in params.items()}
    losses_gpu, losses_orc, flips = [], [], []
    x0, y0 = synth.images(B, 3, 20, 20, step=100)
    for k in range(steps):
        # a fixed probe batch every other step (progress is measurable on it), fresh batches between
        x, y = (x0, y0) if k % 2 == 0 else synth.images(B, 3, 20, 20, step=100 + k)
        pn.set_batch(dev(x), dev(y, torch.int32))
        pn.forward()
        torch.cuda.synchronize()
        rep, nflip = [], 0
        for i, K in enumerate(net.kernels):
            hp = (20 - 4) // 2 if i == 0 else 2
            a = unpack(pn.buf[i]["y"], B, K, hp, pn.parts[i])
            am = torch.zeros(B * K * hp * hp, dtype=torch.uint8, device="cuda")
            cp.cp_unpack_saved(pn.buf[i]["saved"], B, hp, hp, pn.parts[i], 0, am)
            rep.append({"a": a, "argmax": am.reshape(B, K, hp, hp).cpu().numpy()})
        pn.backward()
        pn.sgd(lr)
        tr = orc.net_step(theta, x.astype(np.float64), y, lr, net.layers(), replay=rep)
        for i in range(len(net.kernels)):
            nflip += int(np.sum((rep[i]["argmax"] != tr[f"argmax{i}"]) & (tr[f"a{i}"] > 0)))
        theta = tr["new_params"]
        losses_gpu.append(pn.loss())
        losses_orc.append(tr["loss"])
        flips.append(nflip)
    pn.close()
    print(f"\n[{math}] loss gpu {np.round(losses_gpu, 6).tolist()}\n[{math}] loss orc "
          f"{np.round(losses_orc, 6).tolist()}\n[{math}] argmax flips per step {flips}")
    rel = [abs(g - o) / abs(o) for g, o in zip(losses_gpu, losses_orc)]
    assert max(rel) <= TOL[m], f"loss trajectories apart: max rel {max(rel):.2e} > {TOL[m]:.0e} ({rel})"
    probe = losses_orc[0::2]
    assert probe[-1] < probe[0], f"oracle loss on the probe batch did not fall: {probe}"
    probe_g = losses_gpu[0::2]
    assert probe_g[-1] < probe_g[0], f"GPU loss on the probe batch did not fall: {probe_g}"
