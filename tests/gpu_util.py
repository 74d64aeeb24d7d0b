"""Test glue for GPU parity: build P simulated ranks of one layer on one GPU (LOCAL mode,
no collectives) and move tensors between the oracle's NCHW fp64 world and the library's
gather layout.  The concatenation / summation done here is test glue standing in for the
AllGather / partial-dX sum."""
import numpy as np
import torch

from paper_1712_02546_b200 import convpart as cp

TOL = {cp.CP_MATH_FP32_SIMT: 1e-5, cp.CP_MATH_TF32: 2e-3,   # north_star tolerances (max-abs / max|ref|)
       cp.CP_MATH_BF16: 1.5e-2}   # f4 report-only bf16 operands: 8-bit mantissas, K up to 12,800 (App. B)


def rel_err(gpu, ref):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    m = np.max(np.abs(ref))
    return float(np.max(np.abs(gpu - ref)) / (m if m > 0 else 1.0))


def assert_close(gpu, ref, tol, what):
    e = rel_err(gpu, ref)
    assert e <= tol, f"{what}: max|gpu-ref|/max|ref| = {e:.3e} > {tol:.1e}"
    return e


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


class LocalLayer:
    """All P ranks of one conv layer simulated on one GPU, sharing the gathered output."""

    def __init__(self, B, C, H, K, R, out_part, in_part=None, math=cp.CP_MATH_FP32_SIMT, relu=True, pool=True,
                 bias=True):
        self.P = out_part.n_ranks
        self.out_part, self.in_part = out_part, in_part
        self.B, self.C, self.H, self.K, self.R = B, C, H, K, R
        self.images = in_part is None
        self.pool = pool
        self.Ho = H - R + 1
        self.Hp = self.Ho // 2 if pool else self.Ho
        self.h, self.d, self.sz, self.ws = [], [], [], []
        for r in range(self.P):
            d = cp.cp_conv_desc()
            d.batch, d.in_c, d.in_h, d.in_w = B, C, H, H
            d.num_k, d.k_h, d.k_w = K, R, R
            d.bias, d.relu, d.pool, d.math = int(bias), int(relu), int(pool), math
            d.input_kind = cp.CP_INPUT_IMAGES if self.images else cp.CP_INPUT_GATHER
            d.out_part = out_part
            if in_part is not None:
                d.in_part = in_part
            d.rank, d.world = r, self.P
            h = cp.conv_part_create(d, None)
            sz = cp.conv_part_query(h)
            self.h.append(h)
            self.d.append(d)
            self.sz.append(sz)
            self.ws.append(torch.zeros(sz.workspace, dtype=torch.uint8, device="cuda"))
        self.y = torch.zeros(self.sz[0].y // 4, device="cuda")
        self.saved = [torch.zeros(max(s.saved, 1), dtype=torch.uint8, device="cuda") for s in self.sz]
        self.w = [torch.zeros(max(s.w // 4, 1), device="cuda") for s in self.sz]
        self.b = [torch.zeros(max(s.b // 4, 1), device="cuda") for s in self.sz]

    def load(self, w_kcrs, bias):
        wt = dev(w_kcrs)
        for r in range(self.P):
            cp.cp_pack_conv_weights(self.d[r], wt, self.w[r])
            k0, kr = self.out_part.k_begin[r], self.out_part.k_count[r]
            if kr:
                self.b[r][:kr].copy_(dev(bias[k0:k0 + kr]))

    def forward(self, x_dev):
        for r in range(self.P):
            cp.conv_part_forward(self.h[r], x_dev, self.w[r], self.b[r], self.y, self.saved[r], self.ws[r])

    def y_nchw(self):
        out = torch.zeros(self.B * self.K * self.Hp * self.Hp, device="cuda")
        cp.cp_unpack_nchw(self.y, self.B, self.K, self.Hp, self.Hp, self.out_part, out)
        return out.reshape(self.B, self.K, self.Hp, self.Hp).cpu().numpy().astype(np.float64)

    def argmax_nchw(self):
        parts = []
        for r in range(self.P):
            kr = self.out_part.k_count[r]
            if not kr:
                continue
            o = torch.zeros(self.B * kr * self.Hp * self.Hp, dtype=torch.uint8, device="cuda")
            cp.cp_unpack_saved(self.saved[r], self.B, self.Hp, self.Hp, self.out_part, r, o)
            parts.append(o.reshape(self.B, kr, self.Hp, self.Hp).cpu().numpy())
        return np.concatenate(parts, 1)

    def backward(self, dy_gathered, x_dev, dx_mode=cp.CP_DX_LOCAL):
        """Returns (sum of partial dx as device tensor or None, dW KCRS numpy, db numpy)."""
        dws, dbs, dx_sum = [], [], None
        for r in range(self.P):
            kr = self.out_part.k_count[r]
            dw = torch.zeros(max(self.sz[r].w // 4, 1), device="cuda")
            db = torch.zeros(max(self.sz[r].b // 4, 1), device="cuda")
            if not self.images:
                dx = torch.full((self.sz[r].dx // 4,), float("nan"), device="cuda")
                cp.conv_part_backward_data(self.h[r], dy_gathered, self.saved[r], self.y, self.w[r], dx, dx_mode,
                                           self.ws[r])
                dx_sum = dx.clone() if dx_sum is None else dx_sum + dx
            cp.conv_part_backward_filter(self.h[r], dy_gathered, self.saved[r], self.y, x_dev, dw, db, self.ws[r])
            if kr:
                t = torch.zeros(kr * self.C * self.R * self.R, device="cuda")
                cp.cp_unpack_conv_weights(self.d[r], dw, t)
                dws.append(t.reshape(kr, self.C, self.R, self.R).cpu().numpy().astype(np.float64))
                dbs.append(db[:kr].cpu().numpy().astype(np.float64))
        return dx_sum, np.concatenate(dws, 0), np.concatenate(dbs, 0)

    def close(self):
        for h in self.h:
            cp.conv_part_destroy(h)


def pack(x_nchw, part):
    B, C, H, W = x_nchw.shape
    Bp = (B + 31) // 32 * 32
    n = sum(H * W * Bp * part.k_width[r] for r in range(part.n_ranks))
    out = torch.full((n,), float("nan"), device="cuda")
    cp.cp_pack_nchw(dev(x_nchw), B, C, H, W, part, out)
    return out


def unpack(g, B, C, H, part):
    out = torch.zeros(B * C * H * H, device="cuda")
    cp.cp_unpack_nchw(g, B, C, H, H, part, out)
    return out.reshape(B, C, H, H).cpu().numpy().astype(np.float64)
