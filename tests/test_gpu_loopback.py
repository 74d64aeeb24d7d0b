"""Driver-visible parity of the fused multi-rank data paths on ONE GPU (rows a4 / a11 / f1).

P ranks are simulated in one process through a loopback communicator (cp_comm_create_loopback):
every rank has its own copy of each symmetric buffer, and the SAME library paths run as on P GPUs -
conv1's device barrier + local block write, conv2's forward kernel pushing its own input block into
every peer's copy from its warp 3 (chunk claims, release-adds on the peers' arrival counters) while
it consumes its own block first (the fused channel AllGather, Alg. 1 L19-22 P:L178-182, "reshapes
and rearranges" P:L235), and conv2's dgrad with the fused reduce-scatter of dX (north_star) in both variants: pull (each rank
keeps its partials in its own copy, the owner reads and sums them in rank order) and push (the dgrad
epilogue stores each input block's partial into its owner's receive slot, the owner sums the slots).

No kernel may spin on a later launch of the same process (one GPU, one stream), so:
  * gather: the ranks' conv2 forwards run in rank order; before rank r's kernel, the blocks of the
    ranks q > r that have not pushed yet are copied into rank r's copy by this harness and their
    arrival counters set to CP_GATHER_CHUNKS ("pre-satisfied"); right after the kernel those blocks
    are poisoned with NaN again, so that at the end every block of every copy holds exactly what
    the owning rank's kernel pushed (ranks q < r: pushed before rank r read them; q > r: pushed
    after the poison).  Every copy must equal the gathered output bit for bit, and the counters
    must read CP_GATHER_CHUNKS exactly where a push arrived after the consumer reset its line.
  * reduce-scatter: the library holds each rank's comm-stream tail (wait for the flags, rank-order
    slot sum) until every rank has issued its dgrad (the loopback contract in convpart.h).
Compared with the fp64 oracle (decision replay of the GPU's pooling codes): the gathered conv1
output (TF32 bar 2e-3), each rank's conv2 output, every partial (rank q's partial dX of block r: a receive
slot in push mode, rank q's own copy in pull mode) and the summed dX of each rank's block; in push mode
the sum must equal the fp32 rank-order sum of the slots bit for bit.  Cases include uneven Eq. 1 maps and ranks with zero kernels in a layer (the
copy-engine gather and zero-partial paths), and B=128 (pixel-mode dgrad), each over two steps.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1712_02546_b200 import convpart as cp
    from gpu_util import TOL, dev, pack, rel_err, unpack


class _Raw:
    """torch view of raw device memory (a simulated rank's flag line)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 2}


def raw_u32(ptr, n):
    return torch.as_tensor(_Raw(ptr, n, "<i4"), device="cuda")   # int32 view of the u32 counters (values <= 2^31)


CASES = [
    # name, P, B, conv1 partition, conv2 partition (times for Eq. 1, or explicit counts)
    ("P2-even", 2, 40, {"t": [1.0, 1.0]}, {"t": [1.0, 1.0]}),
    ("P3-eq1", 3, 40, {"t": [1.0, 1.3, 2.1]}, {"t": [1.0, 1.3, 2.1]}),
    ("P4-even-align32", 4, 40, {"t": [1.0] * 4, "align": 32}, {"t": [1.0] * 4, "align": 32}),
    ("P2-zero-kernel-conv1", 2, 40, {"counts": [36, 0]}, {"counts": [40, 32]}),
    ("P3-zero-kernel-conv2", 3, 40, {"counts": [12, 12, 12]}, {"counts": [0, 72, 0]}),
    ("P2-B128-pixel-dgrad", 2, 128, {"t": [1.0, 1.0]}, {"t": [1.0, 1.0]}),
    # 8 ranks (no 8-GPU box in the pool: the 8-way fused paths are exercised here)
    ("P8-even", 8, 40, {"t": [1.0] * 8}, {"t": [1.0] * 8}),
]


def make_part(spec, K):
    if "counts" in spec:
        return cp.cp_partition.from_counts(spec["counts"], spec.get("align", 8))
    return cp.cp_partition_plan(spec["t"], K, spec.get("align", 8))


def blocks(part, H, W, Bp):
    start, out = 0, []
    for r in range(part.n_ranks):
        n = H * W * Bp * part.k_width[r]
        out.append((start, start + n))
        start += n
    return out, start


@pytest.mark.parametrize("rs_mode", ["push", "pull", "ce"])
@pytest.mark.parametrize("name,P,B,s1,s2", CASES, ids=[c[0] for c in CASES])
def test_loopback_fused_collectives(orc, monkeypatch, name, P, B, s1, s2, rs_mode):
    monkeypatch.setenv("CP_RS_MODE", rs_mode)
    K1, K2, H0 = 36, 72, 20
    Bp = (B + 31) // 32 * 32
    p1, p2 = make_part(s1, K1), make_part(s2, K2)
    handles = cp.cp_comm_create_loopback(P)
    L1, L2, d1s, d2s = [], [], [], []
    for r in range(P):
        for i, (C, H, K, part, inp) in enumerate([(3, H0, K1, p1, None), (K1, 8, K2, p2, p1)]):
            d = cp.cp_conv_desc()
            d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = B, C, H, H, K, 5, 5
            d.bias, d.relu, d.pool, d.math = 1, 1, 1, cp.CP_MATH_TF32
            d.input_kind = cp.CP_INPUT_IMAGES if inp is None else cp.CP_INPUT_GATHER
            d.out_part = part
            if inp is not None:
                d.in_part = inp
                d.local_output = 1          # conv2's output stays rank-local (partitioned head)
            d.rank, d.world = r, P
            (L1 if i == 0 else L2).append(cp.conv_part_create(d, handles[r]))
            (d1s if i == 0 else d2s).append(d)
    sz1 = [cp.conv_part_query(h) for h in L1]
    sz2 = [cp.conv_part_query(h) for h in L2]
    # symmetric buffers: allocation k of every handle forms one buffer (same order on all ranks)
    y1 = [cp.SymmetricBuffer(handles[r], sz1[r].y, "cuda") for r in range(P)]
    dx2 = [cp.SymmetricBuffer(handles[r], sz2[r].dx_peer, "cuda") for r in range(P)]
    f_y1 = [raw_u32(cp.cp_symmetric_peer(handles[r], y1[r].ptr, r)[1], 64) for r in range(P)]
    f_dx = [raw_u32(cp.cp_symmetric_peer(handles[r], dx2[r].ptr, r)[1], 64) for r in range(P)]
    ws1 = [torch.zeros(s.workspace, dtype=torch.uint8, device="cuda") for s in sz1]
    ws2 = [torch.zeros(s.workspace, dtype=torch.uint8, device="cuda") for s in sz2]
    sv1 = [torch.zeros(max(s.saved, 1), dtype=torch.uint8, device="cuda") for s in sz1]
    sv2 = [torch.zeros(max(s.saved, 1), dtype=torch.uint8, device="cuda") for s in sz2]
    y2 = [torch.zeros(s.y // 4, device="cuda") for s in sz2]
    w1 = synth.normal((K1, 3, 5, 5), 31, 0.05)
    b1 = synth.normal((K1,), 32, 0.05)
    w2 = synth.normal((K2, K1, 5, 5), 33, 0.02)
    b2 = synth.normal((K2,), 34, 0.02)
    W1, B1, W2, B2 = [], [], [], []
    for r in range(P):
        for (W, Bb, d, sz, w, b, part) in [(W1, B1, d1s[r], sz1[r], w1, b1, p1), (W2, B2, d2s[r], sz2[r], w2, b2, p2)]:
            wt = torch.zeros(max(sz.w // 4, 1), device="cuda")
            cp.cp_pack_conv_weights(d, dev(w), wt)
            bt = torch.zeros(max(sz.b // 4, 1), device="cuda")
            k0, kr = part.k_begin[r], part.k_count[r]
            if kr:
                bt[:kr].copy_(dev(b[k0:k0 + kr]))
            W.append(wt)
            Bb.append(bt)
    blk1, n1 = blocks(p1, 8, 8, Bp)
    blk_in2, _ = blocks(p1, 8, 8, Bp)
    mb = max(e - s for s, e in blk_in2)
    s = torch.cuda.current_stream()
    cs = [torch.cuda.Stream() for _ in range(P)]
    chunks = cp.CP_GATHER_CHUNKS
    failures = []
    for step in range(2):
        x, _ = synth.images(B, 3, H0, H0, step=40 + step)
        xd = dev(x)
        # ---- conv1 forward on every rank: own block into the own copy (producer side of the gather)
        for r in range(P):
            cp.conv_part_forward(L1[r], xd, W1[r], B1[r], y1[r].tensor, sv1[r], ws1[r], s, s)
        # ---- conv2 forward in rank order: the consumer kernel pushes its block into every peer copy
        for r in range(P):
            for q in range(r + 1, P):       # not pushed yet: pre-satisfy (data + counter)
                a, e = blk1[q]
                y1[r].tensor[a:e].copy_(y1[q].tensor[a:e])
                f_y1[r][q] = chunks
            cp.conv_part_forward(L2[r], y1[r].tensor, W2[r], B2[r], y2[r], sv2[r], ws2[r], s, s)
            for q in range(r + 1, P):       # poison: rank q's own push must land here later
                a, e = blk1[q]
                y1[r].tensor[a:e].fill_(float("nan"))
        torch.cuda.synchronize()
        ref_g = torch.cat([y1[q].tensor[a:e] for q, (a, e) in enumerate(blk1)])
        for r in range(P):
            got = y1[r].tensor[:n1]
            if not torch.equal(got, ref_g):
                bad = int((got != ref_g).sum())
                failures.append(f"step {step}: rank {r}'s gathered copy differs from the blocks ({bad} elements)")
            fl = f_y1[r].cpu().numpy()
            exp = np.array([chunks if q > r else 0 for q in range(P)], np.uint32)
            if not np.array_equal(fl[:P], exp) or fl[32] != 0:
                failures.append(f"step {step}: rank {r} flag line {fl[:P].tolist()} claim {fl[32]} (expected "
                                f"{exp.tolist()} claim 0)")
        a1 = unpack(y1[0].tensor, B, K1, 8, p1)
        ref_a1, _ = orc.relu_pool_fwd(orc.conv_fwd(x.astype(np.float64), w1.astype(np.float64), b1.astype(np.float64)))
        e = rel_err(a1, ref_a1)
        if e > TOL[cp.CP_MATH_TF32]:
            failures.append(f"step {step}: gathered conv1 output rel err {e:.2e}")
        z2 = orc.conv_fwd(a1, w2.astype(np.float64), b2.astype(np.float64))
        ref_a2, _ = orc.relu_pool_fwd(z2)
        a2 = np.zeros_like(ref_a2)
        am2 = np.zeros(ref_a2.shape, np.uint8)
        for r in range(P):
            k0, kr = p2.k_begin[r], p2.k_count[r]
            if not kr:
                continue
            a2[:, k0:k0 + kr] = unpack(y2[r], B, K2, 2, p2)[:, k0:k0 + kr]
            am = torch.zeros(B * kr * 4, dtype=torch.uint8, device="cuda")
            cp.cp_unpack_saved(sv2[r], B, 2, 2, p2, r, am)
            am2[:, k0:k0 + kr] = am.reshape(B, kr, 2, 2).cpu().numpy()
        e = rel_err(a2, ref_a2)
        if e > TOL[cp.CP_MATH_TF32]:
            failures.append(f"step {step}: conv2 output (own blocks) rel err {e:.2e}")
        # ---- conv2 dgrad with the fused reduce-scatter (tails enqueued after the last rank's call)
        da2 = synth.normal(ref_a2.shape, 60 + step, 1.0).astype(np.float32)
        dag = pack(da2, p2)
        for r in range(P):
            dx2[r].tensor.fill_(float("nan"))
        for r in range(P):
            cp.conv_part_backward_data(L2[r], dag, sv2[r], y2[r], W2[r], dx2[r].tensor, cp.CP_DX_REDUCE_SCATTER,
                                       ws2[r], s, cs[r])
        torch.cuda.synchronize()
        dy2 = orc.unpool_relu_bwd(da2.astype(np.float64), am2, a2)
        ref_dx = orc.conv_dgrad(dy2, w2.astype(np.float64))
        for r in range(P):
            a, e_ = blk_in2[r]
            k0, kr = p1.k_begin[r], p1.k_count[r]
            nblk = e_ - a
            if rs_mode == "push":   # receive slots behind the gather layout of the owner's copy
                slots = [dx2[r].tensor[n1 + q * mb: n1 + q * mb + nblk] for q in range(P)]
                acc = slots[0].clone()
                for q in range(1, P):
                    acc += slots[q]
                if not torch.equal(acc, dx2[r].tensor[a:e_]):
                    failures.append(f"step {step}: rank {r}'s block is not the rank-order fp32 sum of its slots")
            else:                   # pull / ce: rank q's partial of block r stays in rank q's own copy (q != r)
                slots = [None if q == r else dx2[q].tensor[a:e_] for q in range(P)]
            if f_dx[r][:P].any().item():
                failures.append(f"step {step}: rank {r}'s dX flags not reset: {f_dx[r][:P].tolist()}")
            if not kr:
                continue
            Kw = p1.k_width[r]
            for q in range(P):
                if slots[q] is None:   # pull: the owner's own partial was summed in place
                    continue
                qk0, qkr = p2.k_begin[q], p2.k_count[q]
                got_q = slots[q].reshape(8, 8, Bp, Kw)[:, :, :B, :kr].permute(2, 3, 0, 1).cpu().numpy()
                if not qkr:
                    if np.any(got_q != 0):
                        failures.append(f"step {step}: zero-kernel rank {q}'s slot at rank {r} is not zero")
                    continue
                ref_q = orc.conv_dgrad(dy2, w2.astype(np.float64), qk0, qk0 + qkr)[:, k0:k0 + kr]
                e = rel_err(got_q, ref_q)
                if e > TOL[cp.CP_MATH_TF32]:
                    failures.append(f"step {step}: slot of rank {q} at rank {r} rel err {e:.2e}")
            got = dx2[r].tensor[a:e_].reshape(8, 8, Bp, Kw)[:, :, :B, :kr].permute(2, 3, 0, 1).cpu().numpy()
            e = rel_err(got, ref_dx[:, k0:k0 + kr])
            if e > TOL[cp.CP_MATH_TF32]:
                failures.append(f"step {step}: summed dX of rank {r}'s block rel err {e:.2e}")
    torch.cuda.synchronize()
    for h in L1 + L2:
        cp.conv_part_destroy(h)
    for b in y1 + dx2:
        b.free()
    for h in handles:
        cp.cp_comm_destroy(h)
    assert not failures, f"{name}:\n" + "\n".join(failures)
