"""GPU parity of every pass through the C ABI against the fp64 oracle (-m gpu).

Per-pass parity on identical inputs: the oracle receives the same fp32
values the GPU holds (widened), including the GPU's own outputs of the previous pass;
backward passes replay the GPU's argmax/ReLU decisions (reading R15).
Tolerance: max|gpu-ref| <= tol * max|ref| per tensor, tol = 1e-5 (FP32 SIMT) or 2e-3
(TF32 tensor cores) — north_star.  P ranks are simulated on one GPU in LOCAL mode.
Sizes span several M/N tiles with ragged tails (B=40 -> padded batch 64; 300 kernels ->
two 256-wide N tiles; 70 input channels -> 32+32+8 channel chunks).
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1712_02546_b200 import convpart as cp
    from gpu_util import TOL, LocalLayer, assert_close, dev, pack, unpack
else:  # collected on CPU but skipped
    cp = None

MATHS = ["simt", "tf32"]


def math_id(m):
    return cp.CP_MATH_FP32_SIMT if m == "simt" else cp.CP_MATH_TF32


def parts_for(P, K, align=8):
    if P == 3:
        return cp.cp_partition_plan([1.0, 1.3, 2.1], K, align)   # uneven Eq. 1 map
    return cp.cp_partition_plan([1.0] * P, K, align)


def layer_data(B=40, H=20, K1=70, K2=300, seed=3):
    x, _ = synth.images(B, 3, H, H, step=seed)
    w1 = synth.normal((K1, 3, 5, 5), seed + 1, 0.05)
    b1 = synth.normal((K1,), seed + 2, 0.05)
    w2 = synth.normal((K2, K1, 5, 5), seed + 3, 0.02)
    b2 = synth.normal((K2,), seed + 4, 0.02)
    return x, w1, b1, w2, b2


def window_gap(z, relu=True):
    """Gap between the best and second-best value of each 2x2 window (after ReLU)."""
    if relu:
        z = np.maximum(z, 0)
    B, K, H, W = z.shape
    v = z.reshape(B, K, H // 2, 2, W // 2, 2).transpose(0, 1, 2, 4, 3, 5).reshape(B, K, H // 2, W // 2, 4)
    s = np.sort(v, -1)
    return s[..., 3] - s[..., 2]


# (P, B, align): B=20 -> one 32-image chunk (single-CTA tiles); align=32 -> block widths multiple
# of 32, so dgrad/wgrad N tiles span rank blocks; B=128 / 100 -> 128-image chunks: dgrad pixel
# mode (B=100: ragged, 28 padded images per chunk)
PB = [(1, 40, 8), (2, 40, 8), (3, 40, 8), (1, 20, 8), (2, 40, 32), (4, 40, 32), (2, 128, 8), (1, 100, 32)]


@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("P,B,align", PB)
def test_forward_parity(orc, math, P, B, align):
    _forward_parity(orc, math, P, B, align)


# Split forward (tc_fwd): own-slot counts just above a multiple of 256 run as a CTA-pair launch over the
# 256-multiple part + a transposed launch over the remainder (rank 0 of P=4 in the paper net: 375 slots).
# K2 = 330 at P=1 -> 336 slots (256 + 80); K2 = 750 at P=2 -> 376 (256 + 120); B = 64 / 128 (pair chunks)
@pytest.mark.parametrize("split", ["1", "0"])
@pytest.mark.parametrize("P,B,K2", [(1, 64, 330), (2, 64, 750), (2, 128, 750)])
def test_split_forward_parity(orc, monkeypatch, split, P, B, K2):
    monkeypatch.setenv("CP_TC_FWD_SPLIT", split)
    _forward_parity(orc, "tf32", P, B, 8, K2=K2, K1=40)


# conv1 forward work split (CP_C1_BALANCE): with more than one 128-kernel M tile per rank the CTAs take
# contiguous ranges of (B-set, M tile) units, so a B-set's tiles can be shared by two CTAs (each builds
# the set).  K1 = 300: 3 / 2 M tiles at P = 1 / 2, 80 B-sets -> 240 / 160 units on the SMs.
@pytest.mark.parametrize("balance", ["1", "0"])
@pytest.mark.parametrize("P,B", [(1, 40), (2, 40), (1, 128)])
def test_conv1_unit_split_parity(orc, monkeypatch, balance, P, B):
    monkeypatch.setenv("CP_C1_BALANCE", balance)
    _forward_parity(orc, "tf32", P, B, 8, K2=64, K1=300)


def _forward_parity(orc, math, P, B, align, K2=300, K1=70):
    m = math_id(math)
    x, w1, b1, w2, b2 = layer_data(B=B, K1=K1, K2=K2)
    B, K1, K2 = x.shape[0], w1.shape[0], w2.shape[0]
    p1, p2 = parts_for(P, K1, align), parts_for(P, K2, align)
    L1 = LocalLayer(B, 3, 20, K1, 5, p1, None, m)
    L1.load(w1, b1)
    xd = dev(x)
    L1.forward(xd)
    z1 = orc.conv_fwd(x.astype(np.float64), w1.astype(np.float64), b1.astype(np.float64))
    a1, am1 = orc.relu_pool_fwd(z1)
    y1 = L1.y_nchw()
    assert_close(y1, a1, TOL[m], f"conv1 fwd ({math}, P={P})")
    gap = window_gap(z1)
    bad = (L1.argmax_nchw() != am1) & (gap > 2 * TOL[m] * np.abs(a1).max()) & (a1 > 0)
    assert bad.sum() == 0, f"argmax disagreements on well-separated windows: {bad.sum()}"

    L2 = LocalLayer(B, K1, 8, K2, 5, p2, p1, m)
    L2.load(w2, b2)
    L2.forward(L1.y)
    z2 = orc.conv_fwd(y1, w2.astype(np.float64), b2.astype(np.float64))     # GPU's own A1 as input
    a2, am2 = orc.relu_pool_fwd(z2)
    assert_close(L2.y_nchw(), a2, TOL[m], f"conv2 fwd ({math}, P={P})")
    bad = (L2.argmax_nchw() != am2) & (window_gap(z2) > 2 * TOL[m] * np.abs(a2).max()) & (a2 > 0)
    assert bad.sum() == 0
    # padding slots and padded images are exactly zero
    ref = orc.pack_gather(L2.y_nchw(), (B + 31) // 32 * 32, *[np.array(v) for v in p2.as_tuple()])
    y = L2.y.cpu().numpy()[: ref.size]
    assert np.array_equal(y, ref.astype(np.float32))
    L1.close(); L2.close()


@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("P,B,align", PB)
def test_backward_parity(orc, math, P, B, align):
    m = math_id(math)
    x, w1, b1, w2, b2 = layer_data(B=B)
    B, K1, K2 = x.shape[0], w1.shape[0], w2.shape[0]
    p1, p2 = parts_for(P, K1, align), parts_for(P, K2, align)
    L1 = LocalLayer(B, 3, 20, K1, 5, p1, None, m)
    L1.load(w1, b1)
    xd = dev(x)
    L1.forward(xd)
    L2 = LocalLayer(B, K1, 8, K2, 5, p2, p1, m)
    L2.load(w2, b2)
    L2.forward(L1.y)
    y1, y2 = L1.y_nchw(), L2.y_nchw()
    am2 = L2.argmax_nchw()
    da2 = synth.normal(y2.shape, 99, 1.0).astype(np.float32)
    dxs, dw2, db2 = L2.backward(pack(da2, p2), L1.y)
    # oracle with decision replay (GPU argmax codes + GPU outputs)
    dy2 = orc.unpool_relu_bwd(da2.astype(np.float64), am2, y2)
    assert_close(unpack(dxs, B, K1, 8, p1), orc.conv_dgrad(dy2, w2.astype(np.float64)), TOL[m],
                 f"conv2 dgrad ({math}, P={P})")
    assert_close(dw2, orc.conv_wgrad(dy2, y1, 5, 5), TOL[m], f"conv2 wgrad ({math}, P={P})")
    assert_close(db2, orc.bias_grad(dy2), 1e-5, f"conv2 bias grad ({math}, P={P})")
    # conv1 backward_filter from the (replayed) gradient of its pooled output
    da1 = unpack(dxs, B, K1, 8, p1).astype(np.float32)
    _, dw1, db1 = L1.backward(pack(da1, p1), xd)
    dy1 = orc.unpool_relu_bwd(da1.astype(np.float64), L1.argmax_nchw(), y1)
    assert_close(dw1, orc.conv_wgrad(dy1, x.astype(np.float64), 5, 5), TOL[m], f"conv1 wgrad ({math}, P={P})")
    assert_close(db1, orc.bias_grad(dy1), 1e-5, f"conv1 bias grad ({math}, P={P})")
    L1.close(); L2.close()


@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("P,B", [(1, 40), (2, 40), (3, 20), (2, 128)])
def test_image_dgrad_parity(orc, math, P, B):
    """Row a14: conv_part_backward_data on an image layer (dX of the images, NCHW; S:L62-70 gradInput)
    vs orc_conv_dgrad, each rank's partial over its own kernels summed in rank order (LOCAL mode
    stands in for the all-reduce), with decision replay of the GPU's pooling codes."""
    m = math_id(math)
    x, w1, b1, _, _ = layer_data(B=B)
    B, K1 = x.shape[0], w1.shape[0]
    p1 = parts_for(P, K1)
    L1 = LocalLayer(B, 3, 20, K1, 5, p1, None, m)
    L1.load(w1, b1)
    xd = dev(x)
    L1.forward(xd)
    y1, am1 = L1.y_nchw(), L1.argmax_nchw()
    da1 = synth.normal(y1.shape, 98, 1.0).astype(np.float32)
    dag = pack(da1, p1)
    total = None
    for r in range(P):
        dx = torch.full((L1.sz[r].dx // 4,), float("nan"), device="cuda")
        cp.conv_part_backward_data(L1.h[r], dag, L1.saved[r], L1.y, L1.w[r], dx, cp.CP_DX_LOCAL, L1.ws[r])
        part = dx[: B * 3 * 20 * 20].reshape(B, 3, 20, 20).cpu().numpy().astype(np.float64)
        if p1.k_count[r] == 0:
            assert np.all(part == 0)
        total = part if total is None else total + part
    dy1 = orc.unpool_relu_bwd(da1.astype(np.float64), am1, y1)
    ref = orc.conv_dgrad(dy1, w1.astype(np.float64))
    # TF32 mode rounds dY to tf32 (the tensor-core operand precision) before the fp32 SIMT dgrad
    assert_close(total, ref, TOL[m], f"conv1 dgrad onto images ({math}, P={P})")
    L1.close()


def test_pack_roundtrip_bitexact(orc):
    g = np.random.default_rng(5)
    for P, counts in [(1, [13]), (3, [5, 0, 9]), (4, [8, 8, 8, 7])]:
        part = cp.cp_partition.from_counts(counts)
        x = g.standard_normal((37, sum(counts), 3, 3)).astype(np.float32)
        gd = pack(x, part)
        ref = orc.pack_gather(x.astype(np.float64), 64, *[np.array(v) for v in part.as_tuple()])
        assert np.array_equal(gd.cpu().numpy(), ref.astype(np.float32))
        assert np.array_equal(unpack(gd, 37, sum(counts), 3, part), x.astype(np.float64))


def test_head_parity(orc):
    B, K, H, O = 40, 37, 5, 10
    part = cp.cp_partition_plan([1.0, 2.0], K)
    a = np.maximum(synth.normal((B, K, H, H), 7), 0).astype(np.float32)
    wfc = synth.normal((O, K * H * H), 8, 0.05)
    bfc = synth.normal((O,), 9, 0.05)
    y = synth.images(B, step=4)[1]
    ag = pack(a, part)
    wg = torch.zeros(O * H * H * sum(part.k_width[:2]), device="cuda")
    cp.cp_pack_fc_weights(dev(wfc), O, H, H, part, wg)
    ws = torch.zeros(cp.cp_head_workspace_bytes(B, H, H, part, O), dtype=torch.uint8, device="cuda")
    logits = torch.zeros(B * O, device="cuda")
    cp.cp_fc_forward(ag, B, H, H, part, wg, dev(bfc), O, logits, ws)
    ref = orc.fc_fwd(a.astype(np.float64), wfc.astype(np.float64), bfc.astype(np.float64))
    assert_close(logits.reshape(B, O).cpu().numpy(), ref, 1e-5, "fc fwd")
    loss = torch.zeros(1, device="cuda")
    dl = torch.zeros(B * O, device="cuda")
    cp.cp_softmax_xent(logits, dev(y, torch.int32), B, O, loss, dl)
    rl, rdl = orc.softmax_xent(logits.reshape(B, O).cpu().numpy().astype(np.float64), y)
    assert abs(loss.item() - rl) <= 1e-5 * abs(rl)
    assert_close(dl.reshape(B, O).cpu().numpy(), rdl, 1e-5, "softmax grad")
    dxg = torch.full((ag.numel(),), float("nan"), device="cuda")
    dwg = torch.zeros_like(wg)
    dbf = torch.zeros(O, device="cuda")
    cp.cp_fc_backward(dl, ag, B, H, H, part, wg, O, dxg, dwg, dbf, ws)
    rda, rdw, rdb = orc.fc_bwd(dl.reshape(B, O).cpu().numpy().astype(np.float64), a.astype(np.float64),
                               wfc.astype(np.float64))
    assert_close(unpack(dxg, B, K, H, part), rda, 1e-5, "fc dx")
    dw = torch.zeros(O * K * H * H, device="cuda")
    cp.cp_unpack_fc_weights(dwg, O, H, H, part, dw)
    assert_close(dw.reshape(O, -1).cpu().numpy(), rdw, 1e-5, "fc dW")
    assert_close(dbf.cpu().numpy(), rdb, 1e-5, "fc db")
    # padded feature slots of dW stay exactly zero
    back = torch.zeros_like(wg)
    cp.cp_pack_fc_weights(dw, O, H, H, part, back)
    assert torch.equal(back, dwg)


@pytest.mark.parametrize("math", MATHS)
def test_full_step_p1(orc, math):
    """One whole training step (fwd, head, bwd, SGD) through PartitionedNet vs the oracle step
    with decision replay; every updated parameter within tolerance."""
    from paper_1712_02546_b200.net import PartitionedNet, plan_even
    m = math_id(math)
    net = synth.NetSpec(kernels=(24, 40), in_hw=20, name="small")
    B = 40
    params = synth.params(net, seed=11, std=0.05, bias_std=0.01)
    x, y = synth.images(B, 3, 20, 20, step=1)
    pn = PartitionedNet(net.kernels, B, plan_even(net.kernels, 1), math=m, in_hw=20)
    pn.load_params(params)
    pn.set_batch(dev(x), dev(y, torch.int32))
    pn.forward()
    torch.cuda.synchronize()
    rep = []
    for i, K in enumerate(net.kernels):
        hp = (20 - 4) // 2 if i == 0 else 2
        a = unpack(pn.buf[i]["y"], B, K, hp, pn.parts[i])
        am = torch.zeros(B * K * hp * hp, dtype=torch.uint8, device="cuda")
        cp.cp_unpack_saved(pn.buf[i]["saved"], B, hp, hp, pn.parts[i], 0, am)
        rep.append({"a": a, "argmax": am.reshape(B, K, hp, hp).cpu().numpy()})
    pn.backward()
    pn.sgd(0.01)
    new = pn.export_params()
    p64 = {k: v.astype(np.float64) for k, v in params.items()}
    tr = orc.net_step(p64, x.astype(np.float64), y, 0.01, net.layers(), replay=rep)
    assert abs(pn.loss() - tr["loss"]) <= TOL[m] * abs(tr["loss"])
    for k in p64:
        # compare the update (new - old) so the tolerance applies to the gradient step
        assert_close(new[k] - params[k], tr["new_params"][k] - p64[k], max(TOL[m], 1e-4), f"update of {k} ({math})")
    pn.close()


# ------------------------------------------------------------------ LRN + pool (NEXT row f2)
LRN_T = {"depth": 5, "alpha": 0.05, "beta": 0.75, "bias": 2.0}   # alpha large enough to matter


@pytest.mark.parametrize("P", [1, 2, 3])
def test_lrn_pool_parity(orc, P):
    """cp_lrn_pool_forward / _backward vs the oracle's LRN + pool on a gathered map whose channel
    windows cross (uneven) rank blocks; backward with decision replay of the GPU's pooling codes."""
    B, C, H = 40, 36, 8
    part = parts_for(P, C)
    a = np.abs(synth.normal((B, C, H, H), 51, 1.0)).astype(np.float32)
    a[a < 0.3] = 0.0                                          # post-ReLU maps carry zeros
    ag = pack(a, part)
    Bp = 64
    npool = (H // 2) ** 2 * Bp * sum(part.k_width[r] for r in range(part.n_ranks))
    y = torch.zeros(npool + 64, device="cuda")
    codes = torch.zeros(npool + 64, dtype=torch.uint8, device="cuda")
    cp.cp_lrn_pool_forward(ag, B, H, H, part, LRN_T, 0, y, codes)
    ref_y, _ = orc.relu_pool_fwd(orc.lrn_fwd(a.astype(np.float64), **LRN_T), relu=False)
    got_y = unpack(y, B, C, H // 2, part)
    assert_close(got_y, ref_y, 1e-5, f"LRN+pool forward (P={P})")
    got_am = np.rint(unpack(codes.float(), B, C, H // 2, part)).astype(np.uint8)
    dy = synth.normal(ref_y.shape, 52, 1.0).astype(np.float32)
    dyg = pack(dy, part)
    da = torch.zeros_like(ag)
    for r in range(P):
        cp.cp_lrn_pool_backward(dyg, ag, codes, B, H, H, part, r, LRN_T, da)
    dn = orc.unpool_relu_bwd(dy.astype(np.float64), got_am, got_y, relu=False)
    ref_da = orc.lrn_bwd(a.astype(np.float64), dn, **LRN_T)
    assert_close(unpack(da, B, C, H, part), ref_da, 1e-5, f"LRN+pool backward (P={P})")


def test_lrn_bad_config():
    part = parts_for(1, 8)
    t = torch.zeros(1024, device="cuda")
    c = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    with pytest.raises(cp.ConvPartError):
        cp.cp_lrn_pool_forward(t, 4, 4, 4, part, dict(LRN_T, depth=4), 0, t, c)
    with pytest.raises(cp.ConvPartError):
        cp.cp_lrn_pool_forward(t, 4, 4, 4, part, dict(LRN_T, bias=0.0), 0, t, c)


@pytest.mark.parametrize("math", MATHS)
def test_full_step_lrn_p1(orc, math):
    """Whole step of the paper-literal net (Conv -> ReLU -> LRN -> Pool per conv layer) vs the oracle
    step with decision replay (GPU pooling codes and pre-LRN ReLU map)."""
    from paper_1712_02546_b200.net import PartitionedNet, plan_even
    m = math_id(math)
    net = synth.NetSpec(kernels=(24, 40), in_hw=20, name="small")
    B = 40
    params = synth.params(net, seed=12, std=0.05, bias_std=0.01)
    x, y = synth.images(B, 3, 20, 20, step=2)
    pn = PartitionedNet(net.kernels, B, plan_even(net.kernels, 1), math=m, in_hw=20, lrn=LRN_T)
    pn.load_params(params)
    pn.set_batch(dev(x), dev(y, torch.int32))
    pn.forward()
    torch.cuda.synchronize()
    rep = []
    for i, K in enumerate(net.kernels):
        ho = pn.buf[i]["hw"]
        rep.append({"a": unpack(pn.buf[i]["yp"], B, K, ho // 2, pn.parts[i]),
                    "argmax": np.rint(unpack(pn.buf[i]["codes"].float(), B, K, ho // 2, pn.parts[i])).astype(np.uint8),
                    "pre": unpack(pn.buf[i]["y"], B, K, ho, pn.parts[i])})
    pn.backward()
    pn.sgd(0.01)
    new = pn.export_params()
    p64 = {k: v.astype(np.float64) for k, v in params.items()}
    layers = [dict(L, lrn=LRN_T) for L in net.layers()]
    tr = orc.net_step(p64, x.astype(np.float64), y, 0.01, layers, replay=rep)
    assert abs(pn.loss() - tr["loss"]) <= TOL[m] * abs(tr["loss"])
    for k in p64:
        # the update new - old is read back from fp32 weights: new was rounded at |w|, so the
        # comparison has a floor of ~2 eps32 max|w| / max|update| on top of the kernels' tolerance
        ref = tr["new_params"][k] - p64[k]
        floor = 2.0 * 2.0 ** -23 * np.abs(params[k]).max() / max(np.abs(ref).max(), 1e-30)
        assert_close(new[k] - params[k], ref, max(TOL[m], 1e-4) + floor, f"LRN update of {k} ({math})")
    pn.close()


# ------------------------------------------------------------------ BF16 operands (NEXT row f4, report-only)
@pytest.mark.parametrize("P,B", [(1, 40), (2, 40), (3, 40), (2, 128)])
def test_bf16_passes(orc, P, B):
    """CP_MATH_BF16: every pass with bf16 operand copies (kind::f16, fp32 accumulate) vs the fp64
    oracle at the report-only bound; partitions aligned to 64-slot widths."""
    m = cp.CP_MATH_BF16
    x, w1, b1, w2, b2 = layer_data(B=B)
    B, K1, K2 = x.shape[0], w1.shape[0], w2.shape[0]
    p1, p2 = parts_for(P, K1, 64), parts_for(P, K2, 64)
    L1 = LocalLayer(B, 3, 20, K1, 5, p1, None, m)
    L1.load(w1, b1)
    xd = dev(x)
    L1.forward(xd)
    a1, _ = orc.relu_pool_fwd(orc.conv_fwd(x.astype(np.float64), w1.astype(np.float64), b1.astype(np.float64)))
    y1 = L1.y_nchw()
    assert_close(y1, a1, TOL[m], f"bf16 conv1 fwd (P={P})")
    L2 = LocalLayer(B, K1, 8, K2, 5, p2, p1, m)
    L2.load(w2, b2)
    L2.forward(L1.y)
    a2, _ = orc.relu_pool_fwd(orc.conv_fwd(y1, w2.astype(np.float64), b2.astype(np.float64)))
    y2 = L2.y_nchw()
    assert_close(y2, a2, TOL[m], f"bf16 conv2 fwd (P={P})")
    da2 = synth.normal(y2.shape, 99, 1.0).astype(np.float32)
    dxs, dw2, db2 = L2.backward(pack(da2, p2), L1.y)
    dy2 = orc.unpool_relu_bwd(da2.astype(np.float64), L2.argmax_nchw(), y2)
    assert_close(unpack(dxs, B, K1, 8, p1), orc.conv_dgrad(dy2, w2.astype(np.float64)), TOL[m], f"bf16 dgrad (P={P})")
    assert_close(dw2, orc.conv_wgrad(dy2, y1, 5, 5), TOL[m], f"bf16 wgrad (P={P})")
    da1 = unpack(dxs, B, K1, 8, p1).astype(np.float32)
    _, dw1, _ = L1.backward(pack(da1, p1), xd)
    dy1 = orc.unpool_relu_bwd(da1.astype(np.float64), L1.argmax_nchw(), y1)
    assert_close(dw1, orc.conv_wgrad(dy1, x.astype(np.float64), 5, 5), TOL[m], f"bf16 conv1 wgrad (P={P})")
    L1.close(); L2.close()


def test_bf16_rejects_unaligned_partition():
    part = parts_for(1, 300, 8)    # width 304: not a multiple of 64
    d = cp.cp_conv_desc()
    d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = 40, 3, 20, 20, 300, 5, 5
    d.bias, d.relu, d.pool, d.math, d.input_kind = 1, 1, 1, cp.CP_MATH_BF16, cp.CP_INPUT_IMAGES
    d.out_part, d.rank, d.world = part, 0, 1
    with pytest.raises(cp.ConvPartError):
        cp.conv_part_create(d, None)


# Planner variants the default sizes do not reach (the environment overrides are read per call):
# wgrad tap-slowest unit order (large maps), with and without the stream tail (S = 1), the wgrad
# accumulation-length cap forcing split-K (long reductions), forward / dgrad split-K, single-CTA tiles,
# the transposed forward (also with multicast clusters).  (The forward halo boxes exist only in -DCP_TC_HALO_HOOK experiment builds:
# parity-checked there with CP_TC_FWD_HALO=1, scripts/halo_check.sh.)
VARIANTS = [{"CP_TC_WGRAD_ORDER": "1"}, {"CP_TC_WGRAD_ORDER": "1", "CP_TC_SPLIT_WGRAD": "1"},
            {"CP_TC_SPLIT_WGRAD": "1"}, {"CP_TC_ACC_TERMS": "1024"}, {"CP_TC_SPLIT_FWD": "3"},
            {"CP_TC_SPLIT_DGRAD": "2"}, {"CP_TC_CTA_GROUP": "1"}, {"CP_TC_FWD_T": "1"}, {"CP_TC_FWD_T_IMAGES": "1"},
            {"CP_TC_FWD_T": "1", "CP_TC_FWD_MC": "1"},   # multicast clusters (P=2 here: 2 CTAs)
            {"CP_TC_FWD_T": "0"}]   # the pair forward also where the planner picks the transposed one


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
@pytest.mark.parametrize("P,B,align", [(1, 128, 8), (2, 40, 32), (3, 40, 8)])
def test_planner_variants(orc, monkeypatch, env, P, B, align):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    test_forward_parity(orc, "tf32", P, B, align)
    test_backward_parity(orc, "tf32", P, B, align)


# Fused SGD (conv_part_backward_filter_sgd): the update w -= lr*dW, b -= lr*db runs where dW / db are final
# (wgrad epilogue, stream-tail / split-K reduce, bias reduce, conv1 reduce) and must equal
# backward_filter + conv_part_sgd_step bit for bit (same fma), with dW / db unchanged.  Cases: the
# stream tail (P=1, B=128), Eq. 1 maps (P=3), forced split-K (CP_TC_ACC_TERMS), no tail
# (CP_TC_WGRAD_TAIL=0), both layers (conv1: the image-layer kernel), and the SIMT mode (separate update).
@pytest.mark.parametrize("env", [{}, {"CP_TC_ACC_TERMS": "1024"}, {"CP_TC_WGRAD_TAIL": "0"}],
                         ids=["default", "split-K", "no-tail"])
@pytest.mark.parametrize("math,P,B", [("tf32", 1, 128), ("tf32", 3, 40), ("tf32", 2, 64), ("simt", 2, 40)])
def test_fused_sgd_bitwise(orc, monkeypatch, env, math, P, B):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    m = math_id(math)
    x, w1, b1, w2, b2 = layer_data(B=B)
    K1, K2 = w1.shape[0], w2.shape[0]
    p1, p2 = parts_for(P, K1), parts_for(P, K2)
    L1 = LocalLayer(B, 3, 20, K1, 5, p1, None, m)
    L1.load(w1, b1)
    xd = dev(x)
    L1.forward(xd)
    L2 = LocalLayer(B, K1, 8, K2, 5, p2, p1, m)
    L2.load(w2, b2)
    L2.forward(L1.y)
    lr = 0.0371
    for L, xin, hp, K in ((L2, L1.y, 2, K2), (L1, xd, 8, K1)):
        da = pack(synth.normal((B, K, hp, hp), 77, 1.0).astype(np.float32), L.out_part)
        for r in range(L.P):
            if not L.out_part.k_count[r]:
                continue
            args = (L.h[r], da, L.saved[r], L.y, xin)
            dw_a, db_a = torch.zeros_like(L.w[r]), torch.zeros_like(L.b[r])
            w_a, b_a = L.w[r].clone(), L.b[r].clone()
            cp.conv_part_backward_filter(*args, dw_a, db_a, L.ws[r])
            cp.conv_part_sgd_step(L.h[r], w_a, b_a, dw_a, db_a, lr)
            dw_b, db_b = torch.zeros_like(L.w[r]), torch.zeros_like(L.b[r])
            w_b, b_b = L.w[r].clone(), L.b[r].clone()
            cp.conv_part_backward_filter_sgd(*args, dw_b, db_b, w_b, b_b, lr, L.ws[r])
            torch.cuda.synchronize()
            tag = f"layer K={K} rank {r} ({math}, P={P}, {env})"
            assert torch.equal(dw_a, dw_b) and torch.equal(db_a, db_b), f"dW/db differ with the fused update: {tag}"
            assert torch.equal(w_a, w_b), f"fused weight update differs: {tag}"
            assert torch.equal(b_a, b_b), f"fused bias update differs: {tag}"
            assert not torch.equal(w_a, L.w[r]), f"no update happened: {tag}"
    L1.close(); L2.close()
