"""GPU tests of the paper's probe (§4.1.1) and of BASELINE config C1 (-m gpu).

* conv_part_probe times this device's forward convolution of the layer's shapes on random data
  (P:L147), median of reps after warm-ups: positive, repeatable within 25 %
  (S:L184), roughly proportional to the kernel count ('doubling numK -> elapsed
  approximately doubles', +-30 %), and its times feed Eq. 1 / the planner.
* C1: one conv layer of 8 kernels on 32x32x3, batch 4, unsplit and 2-way split (LOCAL mode):
  forward/backward parity with the oracle and the split reproducing the unsplit layer.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1712_02546_b200 import convpart as cp
    from gpu_util import TOL, LocalLayer, assert_close, dev, pack, unpack


def _probe_desc(K):
    d = cp.cp_conv_desc()
    d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = 128, 500, 14, 14, K, 5, 5
    d.bias, d.relu, d.pool, d.math, d.input_kind = 1, 1, 1, cp.CP_MATH_TF32, cp.CP_INPUT_GATHER
    d.in_part = cp.cp_partition_plan([1.0], 500)
    d.out_part = cp.cp_partition_plan([1.0], K)
    d.rank, d.world = 0, 1
    return d


def test_probe_paper_layer():
    times = {}
    for K in (750, 1500):
        d = _probe_desc(K)
        scratch = torch.empty(cp.conv_part_probe_bytes(d), dtype=torch.uint8, device="cuda")
        t1 = cp.conv_part_probe(d, scratch, warmups=2, reps=5)
        t2 = cp.conv_part_probe(d, scratch, warmups=1, reps=5)
        assert t1 > 0 and t2 > 0
        assert abs(t1 - t2) <= 0.25 * max(t1, t2)                       # S:L184 stability
        times[K] = min(t1, t2)
        del scratch
    ratio = times[1500] / times[750]
    assert 1.4 <= ratio <= 2.6, ratio                                   # S:L185 (+-30 %)
    # probe times feed Eq. 1: a device twice as slow gets ~1/3 of the kernels
    plan = cp.cp_partition_plan([times[1500], 2 * times[1500]], 1500)
    assert plan.as_tuple()[1] == [1000, 500]


@pytest.mark.parametrize("math", ["simt", "tf32"])
def test_c1_tiny_config(orc, math):
    m = cp.CP_MATH_FP32_SIMT if math == "simt" else cp.CP_MATH_TF32
    B, K = 4, 8
    x, _ = synth.images(B, 3, 32, 32, step=0)
    w = synth.normal((K, 3, 5, 5), 11, 0.05)
    b = synth.normal((K,), 12, 0.05)
    z = orc.conv_fwd(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64))
    a, am = orc.relu_pool_fwd(z)
    outs = {}
    for P in (1, 2):
        part = cp.cp_partition_plan([1.0] * P, K)
        L = LocalLayer(B, 3, 32, K, 5, part, None, m)
        L.load(w, b)
        xd = dev(x)
        L.forward(xd)
        y = L.y_nchw()
        assert_close(y, a, TOL[m], f"C1 fwd P={P} ({math})")
        g = synth.normal(a.shape, 13).astype(np.float32)
        _, dw, db = L.backward(pack(g, part), xd)
        dy = orc.unpool_relu_bwd(g.astype(np.float64), L.argmax_nchw(), y)
        assert_close(dw, orc.conv_wgrad(dy, x.astype(np.float64), 5, 5), TOL[m], f"C1 wgrad P={P} ({math})")
        assert_close(db, orc.bias_grad(dy), 1e-5, f"C1 bias grad P={P} ({math})")
        outs[P] = y
        L.close()
    # the 2-way split reproduces the unsplit layer (same kernels per channel -> bitwise)
    assert np.array_equal(outs[1], outs[2])
