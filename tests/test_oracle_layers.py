"""Pins for the oracle's layer math (-m "not gpu").

Every check is against something other than the oracle itself: the paper's /
SPEC's printed worked examples (tests/golden/spec_layer_examples.txt), an
independent library (torch CPU float64 conv2d / autograd, numpy), closed forms,
central finite differences, adjoint identities and brute force.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth


def rnd(shape, seed, std=1.0):
    return synth.normal(shape, seed, std, np.float64)


# ------------------------------------------------------------------ SPEC worked examples
def test_conv_fwd_spec_examples(orc):
    z = orc.conv_fwd(np.zeros((1, 1, 3, 3)), rnd((1, 1, 2, 2), 1))
    assert z.shape == (1, 1, 2, 2) and np.all(z == 0)
    z = orc.conv_fwd(np.array([[[[1.0, 2], [3, 4]]]]), np.array([[[[2.0]]]]))
    assert np.array_equal(z[0, 0], [[2, 4], [6, 8]])
    z = orc.conv_fwd(np.zeros((1, 3, 32, 32)), np.zeros((50, 3, 5, 5)))
    assert z.shape == (1, 50, 28, 28)


def test_conv_bwd_spec_example(orc):
    x = np.array([[[[1.0, 2], [3, 4]]]])
    w = np.array([[[[2.0]]]])
    g = np.ones((1, 1, 2, 2))
    assert np.array_equal(orc.conv_dgrad(g, w)[0, 0], [[2, 2], [2, 2]])
    assert orc.conv_wgrad(g, x, 1, 1)[0, 0, 0, 0] == 10.0
    assert np.all(orc.conv_dgrad(np.zeros((1, 1, 2, 2)), w) == 0)


def test_shape_errors(orc):
    with pytest.raises(orc.OracleError, match="dimension"):
        orc.conv_fwd(np.zeros((1, 2, 8, 8)), np.zeros((3, 3, 5, 5)))
    with pytest.raises(orc.OracleError, match="dimension"):
        orc.relu_pool_fwd(np.zeros((1, 1, 3, 4)))


# ------------------------------------------------------------------ conv vs independent library
@pytest.mark.parametrize("B,C,H,K,R", [(2, 3, 9, 4, 5), (3, 5, 8, 7, 3), (1, 1, 6, 2, 1)])
def test_conv_fwd_matches_torch(orc, B, C, H, K, R):
    x, w, b = rnd((B, C, H, H + 1), 2), rnd((K, C, R, R), 3), rnd((K,), 4)
    ref = F.conv2d(torch.from_numpy(x), torch.from_numpy(w), torch.from_numpy(b)).numpy()
    np.testing.assert_allclose(orc.conv_fwd(x, w, b), ref, rtol=1e-12, atol=1e-12)


def test_conv_delta_kernel_is_shift(orc):
    """A delta kernel at (r0,s0) is a shifted copy of the input (closed form)."""
    x = rnd((2, 3, 10, 10), 5)
    w = np.zeros((3, 3, 5, 5))
    for c in range(3):
        w[c, c, 1, 3] = 1.0
    z = orc.conv_fwd(x, w)
    np.testing.assert_array_equal(z, x[:, :, 1:7, 3:9])


def test_conv_grads_match_torch_autograd(orc):
    x, w = rnd((2, 3, 9, 8), 6), rnd((4, 3, 3, 3), 7)
    g = rnd((2, 4, 7, 6), 8)
    xt = torch.from_numpy(x).requires_grad_()
    wt = torch.from_numpy(w).requires_grad_()
    F.conv2d(xt, wt).backward(torch.from_numpy(g))
    np.testing.assert_allclose(orc.conv_dgrad(g, w), xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(orc.conv_wgrad(g, x, 3, 3), wt.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(orc.bias_grad(g), g.sum(axis=(0, 2, 3)), rtol=1e-12)


def test_conv_finite_differences(orc):
    """Central FD, eps=1e-5, rel err < 1e-6 on a 1x2x6x6 input / 3x2x3x3 bank."""
    x, w, g = rnd((1, 2, 6, 6), 9), rnd((3, 2, 3, 3), 10), rnd((1, 3, 4, 4), 11)
    f = lambda xx, ww: float(np.sum(orc.conv_fwd(xx, ww) * g))
    dx, dw = orc.conv_dgrad(g, w), orc.conv_wgrad(g, x, 3, 3)
    eps = 1e-5
    for idx in [(0, 0, 0, 0), (0, 1, 2, 3), (0, 1, 5, 5), (0, 0, 3, 1)]:
        xp, xm = x.copy(), x.copy()
        xp[idx] += eps
        xm[idx] -= eps
        fd = (f(xp, w) - f(xm, w)) / (2 * eps)
        assert abs(fd - dx[idx]) <= 1e-6 * max(1.0, abs(dx[idx]))
    for idx in [(0, 0, 0, 0), (2, 1, 2, 1), (1, 0, 1, 2)]:
        wp, wm = w.copy(), w.copy()
        wp[idx] += eps
        wm[idx] -= eps
        fd = (f(x, wp) - f(x, wm)) / (2 * eps)
        assert abs(fd - dw[idx]) <= 1e-6 * max(1.0, abs(dw[idx]))


def test_conv_adjoint_identity(orc):
    """<conv(X,W),G> = <X, dgrad(G,W)> = <W, wgrad(G,X)> (exact adjoints)."""
    x, w = rnd((3, 4, 12, 12), 12), rnd((6, 4, 5, 5), 13)
    g = rnd((3, 6, 8, 8), 14)
    lhs = np.sum(orc.conv_fwd(x, w) * g)
    assert abs(lhs - np.sum(x * orc.conv_dgrad(g, w))) < 1e-10 * abs(lhs) + 1e-10
    assert abs(lhs - np.sum(w * orc.conv_wgrad(g, x, 5, 5))) < 1e-10 * abs(lhs) + 1e-10


def test_conv_points_match_dense(orc):
    x, w, b = rnd((2, 3, 10, 10), 15), rnd((5, 3, 5, 5), 16), rnd((5,), 17)
    z = orc.conv_fwd(x, w, b)
    g = np.random.default_rng(0)
    idx = np.stack([g.integers(0, n, 50) for n in z.shape], 1)
    np.testing.assert_array_equal(orc.conv_fwd_points(x, w, b, idx), z[tuple(idx.T)])
    dy = rnd((2, 5, 6, 6), 18)
    dx = orc.conv_dgrad(dy, w)
    idx = np.stack([g.integers(0, n, 50) for n in dx.shape], 1)
    np.testing.assert_array_equal(orc.conv_dgrad_points(dy, w, idx), dx[tuple(idx.T)])
    dw = orc.conv_wgrad(dy, x, 5, 5)
    idx = np.stack([g.integers(0, n, 50) for n in dw.shape], 1)
    np.testing.assert_array_equal(orc.conv_wgrad_points(dy, x, 5, 5, idx), dw[tuple(idx.T)])


def test_conv_kernel_independence(orc):
    """Output map j identical alone or inside the full bank, bitwise."""
    x, w = rnd((2, 3, 12, 12), 19), rnd((7, 3, 5, 5), 20)
    full = orc.conv_fwd(x, w)
    for j in range(7):
        np.testing.assert_array_equal(orc.conv_fwd(x, w[j:j + 1])[:, 0], full[:, j])


# ------------------------------------------------------------------ pooling / relu
def test_pool_spec_examples(orc):
    a, am = orc.relu_pool_fwd(np.array([[[[1.0, 2], [3, 4]]]]), relu=False)
    assert a[0, 0, 0, 0] == 4 and am[0, 0, 0, 0] == 3
    a, am = orc.relu_pool_fwd(np.full((1, 1, 4, 4), 7.0), relu=False)
    assert np.all(a == 7) and np.all(am == 0)                               # S:L78 tie -> first
    z = np.arange(16, dtype=np.float64).reshape(1, 1, 4, 4)
    a, _ = orc.relu_pool_fwd(z, relu=False)
    assert np.array_equal(a[0, 0], [[5, 7], [13, 15]])
    a, am = orc.relu_pool_fwd(np.array([[[[1.0, 2], [3, 4]]]]), relu=False)
    dy = orc.unpool_relu_bwd(np.ones((1, 1, 1, 1)), am, a, relu=False)
    assert np.array_equal(dy[0, 0], [[0, 0], [0, 1]])


def test_pool_matches_torch(orc):
    z = rnd((3, 4, 10, 8), 21)
    a, am = orc.relu_pool_fwd(z, relu=True)
    zt = torch.from_numpy(z).requires_grad_()
    at = F.max_pool2d(F.relu(zt), 2)
    np.testing.assert_array_equal(a, at.detach().numpy())
    g = rnd(a.shape, 22)
    at.backward(torch.from_numpy(g))
    dy = orc.unpool_relu_bwd(g, am, a, relu=True)
    np.testing.assert_array_equal(dy, zt.grad.numpy())   # continuous data: no ties


def test_pool_conservation_and_relu_mask(orc):
    z = rnd((2, 3, 6, 6), 23)
    a, am = orc.relu_pool_fwd(z, relu=False)
    g = rnd(a.shape, 24)
    dy = orc.unpool_relu_bwd(g, am, a, relu=False)
    assert dy.sum() == pytest.approx(g.sum(), abs=1e-12)
    assert np.count_nonzero(dy) == g.size
    # ReLU: windows whose max is <= 0 pass no gradient (reading R7, ReLU'(0)=0)
    a, am = orc.relu_pool_fwd(-np.abs(z), relu=True)
    assert np.all(a == 0) and np.all(am == 0)
    assert np.all(orc.unpool_relu_bwd(g, am, a, relu=True) == 0)


def test_relu_no_pool(orc):
    z = rnd((2, 3, 4, 4), 25)
    a, am = orc.relu_pool_fwd(z, relu=True, pool=False)
    assert am is None
    np.testing.assert_array_equal(a, np.maximum(z, 0))
    g = rnd(z.shape, 26)
    np.testing.assert_array_equal(orc.unpool_relu_bwd(g, None, a, relu=True, pool=False), g * (z > 0))


# ------------------------------------------------------------------ FC / softmax / SGD
def test_fc_examples_and_library(orc):
    b = np.array([0.5, -1.0, 2.0])
    assert np.array_equal(orc.fc_fwd(rnd((4, 6), 27), np.zeros((3, 6)), b), np.tile(b, (4, 1)))
    assert np.array_equal(orc.fc_fwd(np.array([[3.0, 4.0]]), np.eye(2), np.zeros(2)), [[3, 4]])
    a, w, bb = rnd((5, 36), 28), rnd((10, 36), 29), rnd((10,), 30)
    np.testing.assert_allclose(orc.fc_fwd(a, w, bb), a @ w.T + bb, rtol=1e-12)
    g = rnd((5, 10), 31)
    da, dw, db = orc.fc_bwd(g, a, w)
    np.testing.assert_allclose(da, g @ w, rtol=1e-12)
    np.testing.assert_allclose(dw, g.T @ a, rtol=1e-12)
    np.testing.assert_allclose(db, g.sum(0), rtol=1e-12)


def test_softmax_examples(orc):
    y = np.arange(6, dtype=np.int32) % 10
    loss, dl = orc.softmax_xent(np.zeros((6, 10)), y)
    assert loss == pytest.approx(math.log(10), abs=1e-12)
    loss, dl = orc.softmax_xent(np.array([[1000.0, -1000.0]]), np.array([0], np.int32))
    assert math.isfinite(loss) and loss == pytest.approx(0.0, abs=1e-12)
    assert np.all(np.isfinite(dl))
    logits = rnd((4, 10), 32)
    yy = np.array([3, 0, 9, 5], np.int32)
    loss, dl = orc.softmax_xent(logits, yy)
    np.testing.assert_allclose(dl.sum(1), 0, atol=1e-12)
    lt = torch.from_numpy(logits).requires_grad_()
    lref = F.cross_entropy(lt, torch.from_numpy(yy.astype(np.int64)))
    lref.backward()
    assert loss == pytest.approx(lref.item(), rel=1e-12)
    np.testing.assert_allclose(dl, lt.grad.numpy(), rtol=1e-10, atol=1e-14)
    with pytest.raises(orc.OracleError):
        orc.softmax_xent(logits, np.array([3, 0, 10, 5], np.int32))


def test_sgd_examples(orc):
    p = rnd((7,), 33)
    assert np.array_equal(orc.sgd(p, rnd((7,), 34), 0.0), p)
    assert np.array_equal(orc.sgd(np.array([1.0]), np.array([2.0]), 0.5), [0.0])


# ------------------------------------------------------------------ LRN (form S:L89-97)
def test_lrn_spec_examples(orc):
    out = orc.lrn_fwd(np.array([2.0]).reshape(1, 1, 1, 1), depth=1, alpha=1.0, beta=1.0, bias=1.0)
    assert out[0, 0, 0, 0] == pytest.approx(0.4, abs=1e-15)
    x = rnd((2, 5, 3, 3), 41)
    np.testing.assert_array_equal(orc.lrn_fwd(x, alpha=0.0, bias=1.0), x)   # S:L96 identity
    np.testing.assert_allclose(orc.lrn_fwd(x, alpha=0.0, beta=0.75, bias=2.0), x / 2.0 ** 0.75, rtol=1e-15)
    with pytest.raises(Exception):
        orc.lrn_fwd(x, depth=4)                                           # S:L93 even depth
    with pytest.raises(Exception):
        orc.lrn_fwd(x, bias=0.0)                                          # S:L92 bias > 0


@pytest.mark.parametrize("depth,alpha,beta,bias", [(5, 1e-4, 0.75, 2.0), (3, 0.3, 0.6, 1.5), (5, 0.05, 0.75, 1.0)])
def test_lrn_matches_torch(orc, depth, alpha, beta, bias):
    """torch's local_response_norm divides alpha by the window size: alpha_torch = alpha * depth."""
    x = rnd((2, 7, 4, 5), 42)
    ref = F.local_response_norm(torch.from_numpy(x), depth, alpha=alpha * depth, beta=beta, k=bias).numpy()
    np.testing.assert_allclose(orc.lrn_fwd(x, depth, alpha, beta, bias), ref, rtol=1e-13, atol=1e-15)
    xt = torch.from_numpy(x).requires_grad_()
    g = rnd(x.shape, 43)
    F.local_response_norm(xt, depth, alpha=alpha * depth, beta=beta, k=bias).backward(torch.from_numpy(g))
    np.testing.assert_allclose(orc.lrn_bwd(x, g, depth, alpha, beta, bias), xt.grad.numpy(), rtol=1e-12, atol=1e-14)


def test_lrn_finite_differences(orc):
    """random 1x5x4x4 input, backward vs central finite differences, rel err < 1e-6."""
    x = rnd((1, 5, 4, 4), 44)
    g = rnd(x.shape, 45)
    kw = dict(depth=5, alpha=0.2, beta=0.75, bias=1.5)   # alpha large enough that the cross terms matter
    din = orc.lrn_bwd(x, g, **kw)
    eps = 1e-6
    num = np.zeros_like(x)
    for idx in np.ndindex(*x.shape):
        xp, xm = x.copy(), x.copy()
        xp[idx] += eps
        xm[idx] -= eps
        num[idx] = (np.sum(g * orc.lrn_fwd(xp, **kw)) - np.sum(g * orc.lrn_fwd(xm, **kw))) / (2 * eps)
    assert np.max(np.abs(din - num)) / np.max(np.abs(num)) < 1e-6
