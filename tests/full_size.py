"""Sampled parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(PartitionedNet with bench.py's params, images, partition and flags, so the planner takes the same
decisions: CTA pairs, pixel-mode dgrad, stream tails, fused collectives at N>1):
  * configs[1]/[2]: the paper net 500:1500 on 32x32x3, batch 128, 1 GPU / N ranks;
  * configs[3] at its largest batch: the paper net, batch 1024, uneven (Eq. 1) partition, N ranks;
  * configs[4]: the scaled variant 512:2048 on 224x224x3, batch 256, N ranks.

The oracle cannot redo such a step element by element in seconds, so every pass is checked on
sampled outputs the oracle computes one by one (``conv_*_points``, pinned against the dense routines
in tests/test_oracle_layers.py), with decision replay (R15): each pass gets the GPU's own
previous outputs and pooling codes as inputs.  Samples always include the first and last image,
kernel, channel and pixel (ragged tile edges) plus seeded random points.  GPU tensors are unpacked
and sliced on the device; only the sampled images / kernels / channels are widened to fp64 on the
host (a full scaled-net map would be >10 GB in fp64).

Tolerance: north_star's TF32 bound, max|gpu-ref| <= 2e-3 * max|ref| over the sample.
Used by tests/test_gpu_full_size.py (1 GPU) and tests/multi_gpu_check.py (N ranks).
"""
import numpy as np
import torch

import oracle
import synth
from gpu_util import TOL, rel_err
from paper_1712_02546_b200 import convpart as cp


def bench_setup(world, rank, comm, dev, net=None, B=128, head="partitioned", fused=True, times=None):
    """bench.py's N-GPU workload: even partition (or Eq. 1 from per-rank `times`, as
    `bench.py --partition probe`), params seed 42, images step 0."""
    net = net or synth.paper_net("500:1500")
    parts = [cp.cp_partition_plan(times or [1.0] * world, K, 8) for K in net.kernels]
    from paper_1712_02546_b200.net import PartitionedNet
    pn = PartitionedNet(net.kernels, B, parts, rank=rank, comm=comm, math=cp.CP_MATH_TF32, device=dev, head=head,
                        in_hw=net.in_hw, fused=fused)
    params = synth.params(net, seed=42)
    pn.load_params(params)
    x, y = synth.images(B, 3, net.in_hw, net.in_hw, step=0)
    pn.set_batch(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
    return net, parts, pn, params, x, y


def _pick(rng, n, lo, hi, extra=()):
    """n indices in [lo, hi): the range ends first (so every column's entries 0 / 1 form the first /
    last corner), then `extra`, then seeded draws."""
    forced = [lo, hi - 1] + [e for e in extra if lo <= e < hi]
    return np.array(forced + list(rng.integers(lo, hi, size=max(n - len(forced), 0))), dtype=np.int64)[:n]


def _subset(rng, n, lo, hi):
    """Sorted distinct indices in [lo, hi), both ends included."""
    return np.unique(_pick(rng, n, lo, hi))


def _pooled_points(x, w, b, pts):
    """Oracle pooled value and code at pooled points (b,k,i,j): the 4 pre-activations of the window
    one by one (conv_fwd_points), then ReLU + 2x2 max-pool (relu_pool_fwd on the 2x2 window)."""
    n = len(pts)
    idx = np.empty((4 * n, 4), np.int64)
    for t, (dy, dx) in enumerate(((0, 0), (0, 1), (1, 0), (1, 1))):
        idx[t::4] = np.stack([pts[:, 0], pts[:, 1], 2 * pts[:, 2] + dy, 2 * pts[:, 3] + dx], 1)
    z = oracle.conv_fwd_points(x, w, b, idx).reshape(n, 1, 2, 2)
    a, am = oracle.relu_pool_fwd(z)
    zs = np.sort(np.maximum(z.reshape(n, 4), 0), 1)
    return a.reshape(n), am.reshape(n), zs[:, 3] - zs[:, 2]


def _nchw(g, B, C, H, part):
    """Gather-layout device buffer -> NCHW fp32 device tensor (library unpack kernel)."""
    out = torch.zeros(B * C * H * H, device=g.device)
    cp.cp_unpack_nchw(g, B, C, H, H, part, out)
    return out.reshape(B, C, H, H)


def _np(t):
    return t.cpu().numpy().astype(np.float64)


def check_step(pn, net, parts, params, x, y, rank, world, allgather, seed=7, n=384, n_img=6, n_k=10):
    """Run one forward + backward of `pn` (already loaded) and compare sampled outputs of every pass
    with the oracle.  allgather(obj) -> list over ranks (identity list at 1 GPU).  Returns failures."""
    dev = pn.device
    s = torch.cuda.current_stream(dev)
    cs = torch.cuda.Stream(dev)
    pn.forward(s, cs)
    pn.backward(cp.CP_DX_REDUCE_SCATTER, s, cs, overlap=True)
    torch.cuda.synchronize(dev)
    tol = TOL[cp.CP_MATH_TF32]
    rng = np.random.Generator(np.random.PCG64(seed))          # same draws on every rank
    fails = []
    B = pn.B
    (C1, _, K1, _, H1), (_, _, K2, _, H2) = net.shapes()
    own = [(parts[i].k_begin[rank], parts[i].k_count[rank]) for i in range(2)]
    imgs = _subset(rng, n_img, 0, B)
    it = torch.from_numpy(imgs).to(dev)

    def cmp(got, ref, what, t=tol):
        e = rel_err(got, ref)
        if not np.all(np.isfinite(got)) or e > t:
            fails.append(f"full-size {what}: max|gpu-ref|/max|ref| = {e:.3e} (tol {t:.0e})")

    def codes(i, Hp):
        k0, kr = own[i]
        o = torch.zeros(max(B * kr * Hp * Hp, 1), dtype=torch.uint8, device=dev)
        if kr:
            cp.cp_unpack_saved(pn.buf[i]["saved"], B, Hp, Hp, parts[i], rank, o)
        return o[: B * kr * Hp * Hp].reshape(B, kr, Hp, Hp)

    def gather_blocks(k0, t):
        """every rank's own-kernel slice (same images) -> all kernels, in kernel order"""
        got = sorted(allgather((k0, t)), key=lambda v: v[0])
        return np.concatenate([v[1] for v in got if v[1].shape[1]], 1)

    w0, b0 = params["w0"].astype(np.float64), params["b0"].astype(np.float64)
    w1, b1 = params["w1"].astype(np.float64), params["b1"].astype(np.float64)
    x_i = x[imgs].astype(np.float64)

    # ---------------------------------------------------------------- conv1 forward (gathered)
    a1 = _nchw(pn.buf[0]["y"], B, K1, H1, parts[0])           # every kernel on every rank
    am1 = codes(0, H1)
    a1_i = _np(a1[it])
    k0, kr = own[0]
    bnd = [parts[0].k_begin[r] for r in range(world)] + [parts[0].k_begin[r] + parts[0].k_count[r] - 1
                                                          for r in range(world)]
    pts = np.stack([_pick(rng, n, 0, len(imgs)), _pick(rng, n, 0, K1, bnd), _pick(rng, n, 0, H1),
                    _pick(rng, n, 0, H1)], 1)
    ref, refc, gap = _pooled_points(x_i, w0, b0, pts)
    cmp(a1_i[tuple(pts.T)], ref, "conv1 forward (gathered, all kernels)")
    m = (pts[:, 1] >= k0) & (pts[:, 1] < k0 + kr) & (gap > 2 * tol * np.abs(ref).max()) & (ref > 0)
    got_c = am1[it].cpu().numpy()[pts[m, 0], pts[m, 1] - k0, pts[m, 2], pts[m, 3]]
    if np.any(got_c != refc[m]):
        fails.append(f"full-size conv1 pooling codes: {(got_c != refc[m]).sum()} of {m.sum()} well-separated differ")

    # ---------------------------------------------------------------- conv2 forward
    a2 = _nchw(pn.buf[1]["y"], B, K2, H2, parts[1])           # own block valid (partitioned head) or all
    am2 = codes(1, H2)
    k0, kr = own[1]
    kset = (0, K2) if pn.head_mode == "replicated" else (k0, k0 + kr)
    a2_i = _np(a2[it])
    if kset[1] > kset[0]:
        pts = np.stack([_pick(rng, n, 0, len(imgs)), _pick(rng, n, *kset), _pick(rng, n, 0, H2),
                        _pick(rng, n, 0, H2)], 1)
        ref, refc, gap = _pooled_points(a1_i, w1, b1, pts)
        cmp(a2_i[tuple(pts.T)], ref, "conv2 forward (GPU conv1 output as input)")
        m = (pts[:, 1] >= k0) & (pts[:, 1] < k0 + kr) & (gap > 2 * tol * np.abs(ref).max()) & (ref > 0)
        got_c = am2[it].cpu().numpy()[pts[m, 0], pts[m, 1] - k0, pts[m, 2], pts[m, 3]]
        if np.any(got_c != refc[m]):
            fails.append(f"full-size conv2 pooling codes: {(got_c != refc[m]).sum()} of {m.sum()} well-separated "
                         "differ")
    a2_all_i = gather_blocks(k0, a2_i[:, k0:k0 + kr])            # the map the head saw, sampled images
    am2_all_i = gather_blocks(k0, am2[it].cpu().numpy())

    # ---------------------------------------------------------------- head (sampled images, dense)
    got_logits = pn.head["logits"][: B * pn.O].reshape(B, pn.O).cpu().numpy().astype(np.float64)
    cmp(got_logits[imgs], oracle.fc_fwd(a2_all_i, params["wfc"], params["bfc"]), "FC logits")
    loss, dl = oracle.softmax_xent(got_logits, y)              # on the GPU's logits (replay)
    if abs(pn.loss() - loss) > tol * abs(loss):
        fails.append(f"full-size loss {pn.loss()} vs oracle {loss}")
    da2 = _nchw(pn.head["da"], B, K2, H2, parts[1])
    da2_i = _np(da2[it])
    ref, _, _ = oracle.fc_bwd(dl[imgs], a2_all_i, params["wfc"])
    cmp(da2_i[:, k0:k0 + kr], ref[:, k0:k0 + kr], "FC backward dA (own block)")
    da2_all_i = gather_blocks(k0, da2_i[:, k0:k0 + kr])

    # ---------------------------------------------------------------- conv2 dgrad (summed over ranks)
    dy2_i = oracle.unpool_relu_bwd(da2_all_i, am2_all_i, a2_all_i)
    c0, cr = own[0]
    dx = _nchw(pn.buf[1]["dx"], B, K1, H1, parts[0])
    if cr:
        pts = np.stack([_pick(rng, n, 0, len(imgs)), _pick(rng, n, c0, c0 + cr), _pick(rng, n, 0, H1),
                        _pick(rng, n, 0, H1)], 1)
        ref = oracle.conv_dgrad_points(dy2_i, w1, pts)
        cmp(_np(dx[it])[tuple(pts.T)], ref, "conv2 dgrad, dX summed over every rank's kernels (own block)")

    # ---------------------------------------------------------------- wgrad / bias grad, own slices
    for i, (da_full, a_full, am, C) in enumerate([(dx, a1, am1, C1), (da2, a2, am2, K1)]):
        kb, kr_ = own[i]
        if not kr_:
            continue
        d = pn.descs[i]
        t = torch.zeros(kr_ * d.in_c * d.k_h * d.k_w, device=dev)
        cp.cp_unpack_conv_weights(d, pn.buf[i]["dw"], t)
        dw = t.reshape(kr_, d.in_c, d.k_h, d.k_w).cpu().numpy()
        db = pn.buf[i]["db"][:kr_].cpu().numpy()
        ks = _subset(rng, n_k, 0, kr_)                          # local kernel indices
        kt = torch.from_numpy(ks).to(dev)
        dy = oracle.unpool_relu_bwd(_np(da_full[:, kb + kt]), am[:, kt].cpu().numpy(), _np(a_full[:, kb + kt]))
        chans = _subset(rng, 12, 0, C)                          # input channels read by the sample
        if i == 0:
            xin = x[:, chans].astype(np.float64)
        else:
            xin = _np(a1[:, torch.from_numpy(chans).to(dev)])
        pts = np.stack([_pick(rng, n, 0, len(ks)), _pick(rng, n, 0, len(chans)), _pick(rng, n, 0, d.k_h),
                        _pick(rng, n, 0, d.k_w)], 1)
        ref = oracle.conv_wgrad_points(dy, xin, d.k_h, d.k_w, pts)
        cmp(dw[ks[pts[:, 0]], chans[pts[:, 1]], pts[:, 2], pts[:, 3]], ref, f"conv{i + 1} wgrad (own kernels)")
        cmp(db[ks], oracle.bias_grad(dy), f"conv{i + 1} bias grad (own kernels)", 1e-5)
    return fails
