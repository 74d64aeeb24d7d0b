"""Partition invariants and whole-step pins for the oracle (-m "not gpu").

* concat(per-slice forward) == unsplit forward, bitwise
* sum of per-slice partial dX == unsplit dX within 1e-12 (north_star)
* per-slice wgrad == rows of unsplit wgrad, bitwise
* loss identical for any partition count (north_star)
* gather index map: constant maps per channel read back in channel order,
  padding slots zero, round trip exact
* the whole training step == torch float64 autograd of the same network
  (an independent library composition), and training makes progress
"""
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth


def small_net():
    return synth.NetSpec(kernels=(6, 10), in_hw=16, name="small")


def setup(net, B=3, bias_std=0.01, step=0):
    x, y = synth.images(B, 3, net.in_hw, net.in_hw, step=step)
    p = synth.params(net, seed=7, std=0.1, bias_std=bias_std)
    return {k: v.astype(np.float64) for k, v in p.items()}, x.astype(np.float64), y


def test_forward_concat_bitwise(orc):
    x = synth.normal((2, 4, 12, 12), 1).astype(np.float64)
    w = synth.normal((11, 4, 5, 5), 2).astype(np.float64)
    b = synth.normal((11,), 3).astype(np.float64)
    full = orc.conv_fwd(x, w, b)
    for P in (1, 2, 3, 4, 8):
        kb, kc, _ = orc.plan([1.0] * P, 11)
        parts = [orc.conv_fwd(x, w[kb[r]:kb[r] + kc[r]], b[kb[r]:kb[r] + kc[r]]) for r in range(P) if kc[r]]
        np.testing.assert_array_equal(np.concatenate(parts, 1), full)


def test_partial_dx_sum_and_wgrad_rows(orc):
    dy = synth.normal((2, 11, 8, 8), 4).astype(np.float64)
    w = synth.normal((11, 4, 5, 5), 5).astype(np.float64)
    x = synth.normal((2, 4, 12, 12), 6).astype(np.float64)
    full = orc.conv_dgrad(dy, w)
    dwf = orc.conv_wgrad(dy, x, 5, 5)
    for P in (2, 3, 4, 8):
        kb, kc, _ = orc.plan([1.0 + 0.1 * r for r in range(P)], 11)
        acc = np.zeros_like(full)
        for r in range(P):
            acc += orc.conv_dgrad(dy, w, kb[r], kb[r] + kc[r])
        assert np.max(np.abs(acc - full)) <= 1e-12 * np.max(np.abs(full))
        carried = orc.conv_dgrad(dy, w, 0, kb[0] + kc[0])           # carried-accumulator mode
        for r in range(1, P):
            orc.conv_dgrad(dy, w, kb[r], kb[r] + kc[r], accumulate_into=carried)
        np.testing.assert_array_equal(carried, full)
        for r in range(P):
            sl = slice(kb[r], kb[r] + kc[r])
            np.testing.assert_array_equal(orc.conv_wgrad(dy[:, sl], x, 5, 5), dwf[sl])


def test_gather_index_map(orc):
    B, C, H, W, Bp = 3, 7, 2, 3, 4
    x = np.zeros((B, C, H, W))
    for c in range(C):
        x[:, c] = c + 1.0                                            # distinct constant maps
    kb, kc, kw = orc.plan([1.0, 2.0, 1.5], C)
    g = orc.pack_gather(x, Bp, kb, kc, kw)
    start = 0
    for r in range(3):
        blk = g[start:start + H * W * Bp * kw[r]].reshape(H, W, Bp, kw[r])
        for slot in range(kw[r]):
            exp = (kb[r] + slot + 1.0) if slot < kc[r] else 0.0
            assert np.all(blk[:, :, :B, slot] == exp)
        assert np.all(blk[:, :, B:, :] == 0)                         # padded images
        start += H * W * Bp * kw[r]
    assert start == g.size
    # round trip: every real element appears exactly once
    xr = synth.normal((B, C, H, W), 9).astype(np.float64)
    gr = orc.pack_gather(xr, Bp, kb, kc, kw)
    assert np.sort(gr[gr != 0]).tolist() == np.sort(xr.ravel()).tolist()


def _read_gather_golden():
    """tests/golden/gather_layout_example.txt: the hand-written flat gather array."""
    path = os.path.join(os.path.dirname(__file__), "golden", "gather_layout_example.txt")
    kv, flat = {}, []
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("r"):
                flat += [float(v) for v in line.split(":", 1)[1].split()]
            else:
                for tok in line.split():
                    k, v = tok.split("=")
                    kv[k] = [int(u) for u in v.split(",")] if "," in v else int(v)
    return kv, np.array(flat)


def test_gather_layout_golden(orc):
    """Pins orc_pack_gather's (h, w, b, slot) order to a literal, hand-derived array (§8(c)
    item 9): with H != W and distinct values, an h<->w, b<->w or slot<->b swap changes it."""
    kv, expected = _read_gather_golden()
    B, C, H, W, Bp = kv["B"], kv["C"], kv["H"], kv["W"], kv["Bp"]
    b, c, h, w = np.meshgrid(np.arange(B), np.arange(C), np.arange(H), np.arange(W), indexing="ij")
    x = (1000 * b + 100 * c + 10 * h + w + 1).astype(np.float64)
    g = orc.pack_gather(x, Bp, kv["k_begin"], kv["k_count"], kv["k_width"])
    assert g.size == expected.size == sum(H * W * Bp * kw for kw in kv["k_width"])
    assert np.array_equal(g, expected)


def torch_step(params, x, y, net):
    """The same network in torch float64 autograd (independent composition)."""
    t = {k: torch.from_numpy(v).clone().requires_grad_() for k, v in params.items()}
    a = torch.from_numpy(x)
    for i in range(len(net.kernels)):
        a = F.conv2d(a, t[f"w{i}"], t[f"b{i}"])
        a = F.relu(a)
        a = F.max_pool2d(a, 2)
    logits = a.reshape(a.shape[0], -1) @ t["wfc"].T + t["bfc"]
    loss = F.cross_entropy(logits, torch.from_numpy(y.astype(np.int64)))
    loss.backward()
    return loss.item(), {k: v.grad.numpy() for k, v in t.items()}


def test_net_step_matches_torch(orc):
    net = small_net()
    params, x, y = setup(net)
    tr = orc.net_step(params, x, y, 0.01, net.layers())
    loss, grads = torch_step(params, x, y, net)
    assert tr["loss"] == pytest.approx(loss, rel=1e-12)
    for k, g in grads.items():
        np.testing.assert_allclose(tr["grads"][k], g, rtol=1e-9, atol=1e-13 * max(1, np.abs(g).max()))
    for k in params:
        np.testing.assert_array_equal(tr["new_params"][k], params[k] - 0.01 * tr["grads"][k])


@pytest.mark.parametrize("P", [2, 3, 4])
def test_net_step_partitioned_equals_unsplit(orc, P):
    net = small_net()
    params, x, y = setup(net)
    base = orc.net_step(params, x, y, 0.01, net.layers())
    part = []
    for K in net.kernels:
        kb, kc, _ = orc.plan([1.0 + 0.3 * r for r in range(P)], K)
        part.append((kb, kc))
    tr = orc.net_step(params, x, y, 0.01, net.layers(), part=part)
    assert tr["loss"] == base["loss"]                                 # forward is bitwise
    for k in base["grads"]:
        ref = base["grads"][k]
        assert np.max(np.abs(tr["grads"][k] - ref)) <= 1e-12 * max(np.abs(ref).max(), 1e-300)


def test_decision_replay_identity(orc):
    """Replaying the oracle's own decisions reproduces its backward exactly."""
    net = small_net()
    params, x, y = setup(net)
    base = orc.net_step(params, x, y, 0.01, net.layers())
    rep = [{"argmax": base[f"argmax{i}"], "a": base[f"a{i}"]} for i in range(2)]
    tr = orc.net_step(params, x, y, 0.01, net.layers(), replay=rep)
    for k in base["grads"]:
        np.testing.assert_array_equal(tr["grads"][k], base["grads"][k])


def test_training_progress(orc):
    """Loss on a fixed synthetic batch decreases over 20 SGD steps."""
    net = synth.tiny_net()
    params, x, y = setup(net, B=4, bias_std=0.0)
    losses = []
    for _ in range(20):
        tr = orc.net_step(params, x, y, 0.05, net.layers())
        losses.append(tr["loss"])
        params = tr["new_params"]
    assert losses[-1] < losses[0] - 1e-3


def test_net_step_with_lrn_matches_torch(orc):
    """Conv -> ReLU -> LRN -> Pool per conv layer, whole step vs torch float64 autograd."""
    net = small_net()
    params, x, y = setup(net)
    lrn = {"depth": 5, "alpha": 0.05, "beta": 0.75, "bias": 2.0}
    layers = [dict(L, lrn=lrn) for L in net.layers()]
    tr = orc.net_step(params, x, y, 0.01, layers)
    t = {k: torch.from_numpy(v).clone().requires_grad_() for k, v in params.items()}
    a = torch.from_numpy(x)
    for i in range(len(net.kernels)):
        a = F.relu(F.conv2d(a, t[f"w{i}"], t[f"b{i}"]))
        a = F.local_response_norm(a, 5, alpha=lrn["alpha"] * 5, beta=lrn["beta"], k=lrn["bias"])
        a = F.max_pool2d(a, 2)
    logits = a.reshape(a.shape[0], -1) @ t["wfc"].T + t["bfc"]
    loss = F.cross_entropy(logits, torch.from_numpy(y.astype(np.int64)))
    loss.backward()
    assert tr["loss"] == pytest.approx(loss.item(), rel=1e-12)
    for k, v in t.items():
        g = v.grad.numpy()
        np.testing.assert_allclose(tr["grads"][k], g, rtol=1e-9, atol=1e-13 * max(1, np.abs(g).max()))
