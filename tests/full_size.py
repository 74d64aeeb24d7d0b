"""Sampled parity at BASELINE.json's full size (configs[1]/[2]: the paper net 500:1500 on 32x32x3,
batch 128), in the launch configuration bench.py times (PartitionedNet, same params/images, same
planner decisions: CTA pairs, pixel-mode dgrad, stream tails, fused collectives at N>1).

The oracle cannot redo a full 500:1500 step element by element in seconds, so every pass is checked
on sampled outputs the oracle computes one by one (``conv_*_points``, pinned against the dense
routines in tests/test_oracle_layers.py), with decision replay (R15): each pass gets the
GPU's own previous outputs and pooling codes as its inputs.  Samples always include the first and
last image, kernel, channel and pixel (ragged tile edges) plus seeded random interior points.

Tolerance: north_star's TF32 bound, max|gpu-ref| <= 2e-3 * max|ref| over the sample.
Used by tests/test_gpu_full_size.py (1 GPU) and tests/multi_gpu_check.py (N ranks).
"""
import numpy as np
import torch

import oracle
import synth
from gpu_util import TOL, rel_err, unpack
from paper_1712_02546_b200 import convpart as cp


def paper_setup(world, rank, comm, dev, head="partitioned", fused=True, B=128):
    """The bench.py N-GPU workload: paper net 500:1500, even partition, params seed 42, images step 0."""
    net = synth.paper_net("500:1500")
    parts = [cp.cp_partition_plan([1.0] * world, K, 8) for K in net.kernels]
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


def check_step(pn, net, parts, params, x, y, rank, world, allgather, seed=7, n=384):
    """Run one forward + backward of `pn` (already loaded) and compare sampled outputs of every pass
    with the oracle.  allgather(obj) -> list over ranks (identity list at 1 GPU).  Returns failures."""
    dev = pn.device
    s = torch.cuda.current_stream(dev)
    cs = torch.cuda.Stream(dev)
    pn.forward(s, cs)
    pn.backward(cp.CP_DX_REDUCE_SCATTER, s, cs, overlap=True)
    torch.cuda.synchronize(dev)
    tol = TOL[cp.CP_MATH_TF32]
    rng = np.random.Generator(np.random.PCG64(seed + 1000 * rank))
    fails = []
    B = pn.B
    K1, K2 = net.kernels
    H1, H2 = 14, 5                       # pooled sizes of conv1 / conv2 on 32x32 inputs
    p64 = {k: v.astype(np.float64) for k, v in params.items()}
    x64 = x.astype(np.float64)
    own = [(parts[i].k_begin[rank], parts[i].k_count[rank]) for i in range(2)]

    def cmp(got, ref, what, t=tol):
        e = rel_err(got, ref)
        if not np.all(np.isfinite(got)) or e > t:
            fails.append(f"full-size {what}: max|gpu-ref|/max|ref| = {e:.3e} (tol {t:.0e})")

    def codes(i, Hp):
        k0, kr = own[i]
        o = torch.zeros(max(B * kr * Hp * Hp, 1), dtype=torch.uint8, device=dev)
        if kr:
            cp.cp_unpack_saved(pn.buf[i]["saved"], B, Hp, Hp, parts[i], rank, o)
        return o[: B * kr * Hp * Hp].reshape(B, kr, Hp, Hp).cpu().numpy()

    # ---------------------------------------------------------------- forward
    a1 = unpack(pn.buf[0]["y"], B, K1, H1, parts[0])          # gathered: every kernel on every rank
    am1 = codes(0, H1)
    k0, kr = own[0]
    bnd = [parts[0].k_begin[r] for r in range(world)] + [parts[0].k_begin[r] + parts[0].k_count[r] - 1
                                                          for r in range(world)]
    pts = np.stack([_pick(rng, n, 0, B), _pick(rng, n, 0, K1, bnd), _pick(rng, n, 0, H1), _pick(rng, n, 0, H1)], 1)
    ref, refc, gap = _pooled_points(x64, p64["w0"], p64["b0"], pts)
    cmp(a1[tuple(pts.T)], ref, "conv1 forward (gathered, all kernels)")
    m = (pts[:, 1] >= k0) & (pts[:, 1] < k0 + kr) & (gap > 2 * tol * np.abs(ref).max()) & (ref > 0)
    got_c = am1[pts[m, 0], pts[m, 1] - k0, pts[m, 2], pts[m, 3]]
    if np.any(got_c != refc[m]):
        fails.append(f"full-size conv1 pooling codes: {(got_c != refc[m]).sum()} of {m.sum()} well-separated differ")

    a2_full = unpack(pn.buf[1]["y"], B, K2, H2, parts[1])     # own block valid (partitioned head) or all
    am2 = codes(1, H2)
    k0, kr = own[1]
    kset = (0, K2) if pn.head_mode == "replicated" else (k0, k0 + kr)
    pts = np.stack([_pick(rng, n, 0, B), _pick(rng, n, *kset), _pick(rng, n, 0, H2), _pick(rng, n, 0, H2)], 1)
    ref, refc, gap = _pooled_points(a1, p64["w1"], p64["b1"], pts)
    cmp(a2_full[tuple(pts.T)], ref, "conv2 forward (GPU conv1 output as input)")
    m = (pts[:, 1] >= k0) & (pts[:, 1] < k0 + kr) & (gap > 2 * tol * np.abs(ref).max()) & (ref > 0)
    got_c = am2[pts[m, 0], pts[m, 1] - k0, pts[m, 2], pts[m, 3]]
    if np.any(got_c != refc[m]):
        fails.append(f"full-size conv2 pooling codes: {(got_c != refc[m]).sum()} of {m.sum()} well-separated differ")

    # every rank's own conv2 block -> the full map the head saw (assembled only for the check)
    blocks = allgather((k0, a2_full[:, k0:k0 + kr], am2))
    a2 = np.concatenate([blk[1] for blk in sorted(blocks, key=lambda t: t[0]) if blk[1].shape[1]], 1)
    am2_all = np.concatenate([blk[2] for blk in sorted(blocks, key=lambda t: t[0]) if blk[2].shape[1]], 1)

    # ---------------------------------------------------------------- head (dense: it is small)
    logits = oracle.fc_fwd(a2, p64["wfc"], p64["bfc"])
    loss, dl = oracle.softmax_xent(logits, y)
    got_logits = pn.head["logits"][: B * pn.O].reshape(B, pn.O).cpu().numpy()
    cmp(got_logits, logits, "FC logits")
    if abs(pn.loss() - loss) > tol * abs(loss):
        fails.append(f"full-size loss {pn.loss()} vs oracle {loss}")
    da2_ref, _, _ = oracle.fc_bwd(dl, a2, p64["wfc"])
    da2_gpu = unpack(pn.head["da"], B, K2, H2, parts[1])
    cmp(da2_gpu[:, k0:k0 + kr], da2_ref[:, k0:k0 + kr], "FC backward dA (own block)")
    da2 = np.concatenate([d for _, d in sorted(allgather((k0, da2_gpu[:, k0:k0 + kr])), key=lambda t: t[0])
                          if d.shape[1]], 1)

    # ---------------------------------------------------------------- conv2 dgrad (summed over ranks)
    imgs = np.unique(_pick(rng, 6, 0, B))
    dy2_i = oracle.unpool_relu_bwd(da2[imgs], am2_all[imgs], a2[imgs])
    c0, cr = own[0]
    dx = unpack(pn.buf[1]["dx"], B, K1, H1, parts[0])
    if cr:
        pts = np.stack([_pick(rng, n, 0, len(imgs)), _pick(rng, n, c0, c0 + cr), _pick(rng, n, 0, H1),
                        _pick(rng, n, 0, H1)], 1)
        ref = oracle.conv_dgrad_points(dy2_i, p64["w1"], pts)
        got = dx[imgs[pts[:, 0]], pts[:, 1], pts[:, 2], pts[:, 3]]
        cmp(got, ref, "conv2 dgrad, dX summed over every rank's kernels (own block)")

    # ---------------------------------------------------------------- wgrad / bias grad of own slices
    def own_grads(i):
        d, (kb, kr_) = pn.descs[i], own[i]
        t = torch.zeros(max(kr_ * d.in_c * d.k_h * d.k_w, 1), device=dev)
        if kr_:
            cp.cp_unpack_conv_weights(d, pn.buf[i]["dw"], t)
        dw = t[: kr_ * d.in_c * d.k_h * d.k_w].reshape(kr_, d.in_c, d.k_h, d.k_w).cpu().numpy()
        return dw, pn.buf[i]["db"][:kr_].cpu().numpy()

    for i, (xin, da_all, Hp, C) in enumerate([(x64, dx, H1, 3), (a1, da2_gpu, H2, K1)]):
        kb, kr_ = own[i]
        if not kr_:
            continue
        dw, db = own_grads(i)
        ks = np.unique(_pick(rng, 10, 0, kr_))              # local kernel indices, incl. first/last
        am = am1 if i == 0 else am2
        a = a1 if i == 0 else a2_full
        dy = oracle.unpool_relu_bwd(da_all[:, kb + ks], am[:, ks], a[:, kb + ks])
        pts = np.stack([_pick(rng, n, 0, len(ks)), _pick(rng, n, 0, C), _pick(rng, n, 0, 5), _pick(rng, n, 0, 5)], 1)
        ref = oracle.conv_wgrad_points(dy, xin, 5, 5, pts)
        cmp(dw[ks[pts[:, 0]], pts[:, 1], pts[:, 2], pts[:, 3]], ref, f"conv{i + 1} wgrad (own kernels)")
        cmp(db[ks], oracle.bias_grad(dy), f"conv{i + 1} bias grad (own kernels)", 1e-5)
    return fails
