"""Kernel-partitioned training of the paper's CNN on one rank (SPMD over P ranks).

Host-side orchestration only: allocation of caller-owned device buffers (torch), and
the order of C-ABI calls that make one SGD training step of the §5.2 network
(P:L267-276): conv(5x5)+bias+ReLU+2x2 max-pool per conv layer (each rank its own
contiguous kernel slice, Alg. 1), channel AllGather of every conv output,
replicated FC + softmax loss head ("the master node is in charge of training
the remaining network"), backward with the same split: dgrad of the own slice and a
cross-rank sum of partial dX, wgrad local, SGD on the own slice.

Every arithmetic step runs in libconvpart's kernels; nothing here computes.
"""
from __future__ import annotations

import numpy as np
import torch

from . import convpart as cp


def _dev_bytes(n, device):
    return torch.empty(max(int(n), 16), dtype=torch.uint8, device=device)


def _f32(nbytes, device):
    return torch.zeros(max(int(nbytes) // 4, 4), dtype=torch.float32, device=device)


class PartitionedNet:
    """One rank's share of the kernel-partitioned network.

    kernels: conv kernel counts per layer (paper: (500, 1500)); parts: one cp_partition per
    conv layer (same n_ranks); comm: cp_comm handle or None (no collectives).
    """

    def __init__(self, kernels, batch, parts, rank=0, comm=None, math=cp.CP_MATH_TF32, in_c=3, in_hw=32,
                 ksize=5, classes=10, relu=True, pool=True, bias=True, device="cuda", head="replicated",
                 fused=False, lrn=None):
        """head: "replicated" - the last conv output is all-gathered and every rank runs the full FC
        head (the paper's master-side head, replicated); "partitioned" - the last conv output stays
        rank-local, each rank owns the FC columns of its channels, partial logits are summed with
        one AllReduce (identical logits/loss on every rank; no AllGather of the last layer).
        fused: B200 collective fusion - every all-gathered conv output and every dX is a
        symmetric (peer-mapped) buffer: the producer writes its block locally, the consuming layer's TF32
        forward kernel pushes that block into every peer's copy over NVLink while it computes on its own
        block first (each peer block is consumed once its arrival counter is complete), and the dgrad
        epilogue stores each input block's partial dX into its owner's receive slot (reduce-scatter
        without an NCCL kernel; the owner sums the slots in rank order).
        lrn: None, or LRN parameters {depth, alpha, beta, bias} (convpart.LRN_DEFAULT): every conv layer
        becomes Conv -> bias -> ReLU -> LRN -> Pool (NEXT row f2): the conv runs without
        pooling, its pre-pool output is gathered, every rank runs cp_lrn_pool_forward over all
        channels; backward needs the full pooled gradient (replicated head, all-reduced dX)."""
        self.device = torch.device(device)
        self.lrn = dict(lrn) if lrn else None
        if self.lrn:
            head = "replicated"    # the LRN backward needs the gradient of every channel
        self.head_mode = head if parts[0].n_ranks > 1 else "replicated"
        self.B, self.Bp, self.O = batch, (batch + 31) // 32 * 32, classes
        self.rank, self.world = rank, parts[0].n_ranks
        self.parts, self.comm, self.math = parts, comm, math
        self.layers, self.descs, self.sizes, self.buf, self.sym = [], [], [], [], []
        c, h, prev = in_c, in_hw, None
        for i, K in enumerate(kernels):
            d = cp.cp_conv_desc()
            d.batch, d.in_c, d.in_h, d.in_w = batch, c, h, h
            d.num_k, d.k_h, d.k_w = K, ksize, ksize
            d.bias, d.relu, d.pool, d.math = int(bias), int(relu), int(pool and not self.lrn), math
            d.input_kind = cp.CP_INPUT_IMAGES if prev is None else cp.CP_INPUT_GATHER
            d.out_part = parts[i]
            if prev is not None:
                d.in_part = prev
            d.rank, d.world = rank, self.world
            if i == len(kernels) - 1 and self.head_mode == "partitioned":
                d.local_output = 1
            hnd = cp.conv_part_create(d, comm)
            sz = cp.conv_part_query(hnd)
            self.layers.append(hnd)
            self.descs.append(d)
            self.sizes.append(sz)
            b = {
                "w": _f32(sz.w, self.device), "b": _f32(sz.b, self.device),
                "dw": _f32(sz.w, self.device), "db": _f32(sz.b, self.device),
                "y": self._symmetric(sz.y, fused and not d.local_output),
                "saved": _dev_bytes(sz.saved, self.device),
                "ws": _dev_bytes(sz.workspace, self.device),
            }
            if prev is not None:
                b["dx"] = self._symmetric(sz.dx_peer, fused) if fused else _f32(sz.dx, self.device)
            if self.lrn:
                # pooled gathered map + codes (all channels, computed by every rank), pre-pool gradient
                ho = h - ksize + 1
                cnt = sum(parts[i].k_width[r] for r in range(self.world))
                batch_p = (batch + 31) // 32 * 32
                npool = (ho // 2) * (ho // 2) * batch_p * cnt
                b["yp"] = _f32(npool * 4 + 256, self.device)
                b["codes"] = _dev_bytes(npool, self.device)
                b["dpre"] = _f32(sz.y, self.device)
                b["hw"] = ho
            self.buf.append(b)
            ho = h - ksize + 1
            h = ho // 2 if pool else ho
            c, prev = K, parts[i]
        self.Hp = self.Wp = h
        self.F = kernels[-1] * h * h
        last = parts[-1]
        if self.head_mode == "partitioned":
            # the head sees only this rank's block: a one-block partition of the own channels
            hp = cp.cp_partition()
            hp.n_ranks, hp.num_k = 1, last.k_count[rank]
            hp.k_begin[0], hp.k_count[0], hp.k_width[0] = 0, last.k_count[rank], last.k_width[rank]
            self.head_part = hp
            self.head_off = self.sizes[-1].y_offset // 4
        else:
            self.head_part = last
            self.head_off = 0
        last = self.head_part
        Fg = h * h * sum(last.k_width[: last.n_ranks])
        self.head = {
            # (max(.., 4): a rank without channels in the last layer still holds valid, empty head buffers)
            "wfc": torch.zeros(max(classes * Fg, 4), device=self.device), "bfc": torch.zeros(classes, device=self.device),
            "dwfc": torch.zeros(max(classes * Fg, 4), device=self.device), "dbfc": torch.zeros(classes, device=self.device),
            "logits": torch.zeros(batch * classes, device=self.device),
            "dlogits": torch.zeros(batch * classes, device=self.device),
            "loss": torch.zeros(4, device=self.device),
            "da": _f32(self.sizes[-1].y, self.device),
            "ws": _dev_bytes(cp.cp_head_workspace_bytes(batch, h, h, last, classes), self.device),
        }
        self.head_x = (self.buf[-1]["yp"] if self.lrn else self.buf[-1]["y"])[self.head_off:]
        self.head_da = self.head["da"][self.head_off:]
        self.x = torch.zeros(batch * in_c * in_hw * in_hw, device=self.device)
        self.labels = torch.zeros(batch, dtype=torch.int32, device=self.device)
        self.in_shape = (batch, in_c, in_hw, in_hw)

    def _symmetric(self, nbytes, symmetric):
        if not (symmetric and self.world > 1 and self.comm is not None and self.math == cp.CP_MATH_TF32):
            return _f32(nbytes, self.device)
        buf = cp.SymmetricBuffer(self.comm, max(int(nbytes), 16), self.device)
        self.sym.append(buf)
        return buf.tensor

    # ------------------------------------------------------------ parameters
    def load_params(self, params, stream=None):
        """params: dict of full fp32 numpy arrays (KCRS conv, [O,F] fc).  Packs this rank's slice."""
        for i, d in enumerate(self.descs):
            wfull = torch.from_numpy(np.ascontiguousarray(params[f"w{i}"], np.float32)).to(self.device)
            cp.cp_pack_conv_weights(d, wfull, self.buf[i]["w"], stream)
            k0, kr = self.parts[i].k_begin[self.rank], self.parts[i].k_count[self.rank]
            if kr:
                self.buf[i]["b"][:kr].copy_(torch.from_numpy(np.ascontiguousarray(params[f"b{i}"][k0:k0 + kr])))
        wfc_np = np.ascontiguousarray(params["wfc"], np.float32)
        if self.head_mode == "partitioned":
            k0, kr = self.parts[-1].k_begin[self.rank], self.parts[-1].k_count[self.rank]
            wfc_np = np.ascontiguousarray(wfc_np.reshape(self.O, -1, self.Hp * self.Wp)[:, k0:k0 + kr])
        wfc = torch.from_numpy(wfc_np.reshape(self.O, -1)).to(self.device)
        if wfc.numel():
            cp.cp_pack_fc_weights(wfc, self.O, self.Hp, self.Wp, self.head_part, self.head["wfc"], stream)
        self.head["bfc"].copy_(torch.from_numpy(np.ascontiguousarray(params["bfc"], np.float32)))
        torch.cuda.synchronize(self.device)

    def export_params(self):
        """This rank's rows (KCRS) of every conv layer and the full FC head, as numpy."""
        out = {}
        for i, d in enumerate(self.descs):
            kr = self.parts[i].k_count[self.rank]
            t = torch.zeros(max(kr * d.in_c * d.k_h * d.k_w, 1), device=self.device)
            if kr:
                cp.cp_unpack_conv_weights(d, self.buf[i]["w"], t)
            out[f"w{i}"] = t[: kr * d.in_c * d.k_h * d.k_w].reshape(kr, d.in_c, d.k_h, d.k_w)
            out[f"b{i}"] = self.buf[i]["b"][:kr]
        nf = self.head_part.num_k * self.Hp * self.Wp
        wfc = torch.zeros(max(self.O * nf, 1), device=self.device)
        if nf:
            cp.cp_unpack_fc_weights(self.head["wfc"], self.O, self.Hp, self.Wp, self.head_part, wfc)
        out["wfc"] = wfc[: self.O * nf].reshape(self.O, nf)   # own columns only when partitioned
        out["bfc"] = self.head["bfc"]
        torch.cuda.synchronize(self.device)
        return {k: v.detach().cpu().numpy().copy() for k, v in out.items()}

    def set_batch(self, x, labels):
        self.x.copy_(x.reshape(-1), non_blocking=True)
        self.labels.copy_(labels.reshape(-1), non_blocking=True)

    def bind_input(self, x, labels):
        """Read the images / labels of the following steps from these device buffers (e.g. an input
        pipeline's staging buffers, so no device copy precedes the step; a CUDA graph captured meanwhile
        keeps the pointers).  Returns the previous pair."""
        if x.numel() != self.x.numel() or x.device != self.x.device or x.dtype != torch.float32:
            raise ValueError("bind_input: images must be a float32 device tensor of the batch's size")
        if labels.numel() != self.labels.numel() or labels.dtype != torch.int32 or labels.device != self.x.device:
            raise ValueError("bind_input: labels must be an int32 device tensor of batch size")
        prev = (self.x, self.labels)
        self.x, self.labels = x.reshape(-1), labels.reshape(-1)
        return prev

    # ------------------------------------------------------------ one training step
    def forward(self, stream=None, comm_stream=None, head=True):
        """head=False: the conv stage only (every conv layer and its gather; no FC / loss) - bench.py's
        conv-stage images/s, with backward(head=False) starting from the fixed dA2 in head["da"]."""
        inp = self.x
        for i, L in enumerate(self.layers):
            b = self.buf[i]
            cp.conv_part_forward(L, inp, b["w"], b["b"], b["y"], b["saved"], b["ws"], stream, comm_stream)
            inp = b["y"]
            if self.lrn:
                sym = next((m for m in self.sym if m.tensor.data_ptr() == b["y"].data_ptr()), None)
                if sym is not None:
                    sym.wait(stream)
                cp.cp_lrn_pool_forward(b["y"], self.B, b["hw"], b["hw"], self.parts[i], self.lrn,
                                       self.math == cp.CP_MATH_TF32, b["yp"], b["codes"], stream)
                inp = b["yp"]
        hd = self.head
        last = next((m for m in self.sym if m.tensor.data_ptr() == self.buf[-1]["y"].data_ptr()), None)
        if last is not None and not self.lrn:
            last.wait(stream)   # replicated head reads the gathered last output
        if not head:
            return
        bias = hd["bfc"] if (self.head_mode == "replicated" or self.rank == 0) else None
        cp.cp_fc_forward(self.head_x, self.B, self.Hp, self.Wp, self.head_part, hd["wfc"], bias, self.O, hd["logits"],
                         hd["ws"], stream)
        if self.head_mode == "partitioned" and self.comm is not None:
            # the partial logits' AllReduce and the softmax in one launch (one-shot peer-memory path)
            cp.cp_allreduce_softmax_xent(self.comm, hd["logits"], self.labels, self.B, self.O, hd["loss"], hd["dlogits"],
                                         stream)
        else:
            cp.cp_softmax_xent(hd["logits"], self.labels, self.B, self.O, hd["loss"], hd["dlogits"], stream)

    def backward(self, dx_mode=cp.CP_DX_REDUCE_SCATTER, stream=None, comm_stream=None, overlap=True, head=True,
                 lr=None):
        """lr given: each conv layer's SGD step runs inside the backward pass - for a gather-input layer as a
        separate update on comm_stream right after its wgrad, overlapped with the next layer's backward
        (joined before returning); for the image layer fused into its backward-filter kernels
        (conv_part_backward_filter_sgd).  sgd(..., convs=False) then updates only the head."""
        hd = self.head
        s_main = stream if stream is not None else torch.cuda.current_stream(self.device)
        side = comm_stream is not None and comm_stream != s_main
        joined = True
        if head:
            cp.cp_fc_backward(hd["dlogits"], self.head_x, self.B, self.Hp, self.Wp, self.head_part, hd["wfc"],
                              self.O, self.head_da, hd["dwfc"], hd["dbfc"], hd["ws"], stream)
        da = hd["da"]
        n = len(self.layers)
        for i in reversed(range(n)):
            L, b = self.layers[i], self.buf[i]
            xin = self.x if i == 0 else self.buf[i - 1]["yp" if self.lrn else "y"]
            if self.lrn:
                # pooled gradient of every channel -> this rank's block of the pre-pool gradient
                cp.cp_lrn_pool_backward(da, b["y"], b["codes"], self.B, b["hw"], b["hw"], self.parts[i], self.rank,
                                        self.lrn, b["dpre"], stream)
                da = b["dpre"]
            if i > 0:
                # with several ranks the forward always runs a collective on every rank (gather or logits
                # AllReduce), which orders consecutive calls of the fused reduce-scatter (CP_DX_ORDERED);
                # LRN below needs every channel of the summed dX (all-reduce)
                mode = (cp.CP_DX_ALLREDUCE if self.lrn else dx_mode) | (cp.CP_DX_ASYNC if overlap else 0) | \
                    (cp.CP_DX_ORDERED if self.world > 1 else 0)
                cp.conv_part_backward_data(L, da, b["saved"], b["y"], b["w"], b["dx"], mode, b["ws"], stream,
                                           comm_stream)
            # wgrad needs no communication: it overlaps the dX reduction on the comm stream (§8(e))
            if lr is None or (i > 0 and side):
                cp.conv_part_backward_filter(L, da, b["saved"], b["y"], xin, b["dw"], b["db"], b["ws"], stream)
            else:
                cp.conv_part_backward_filter_sgd(L, da, b["saved"], b["y"], xin, b["dw"], b["db"], b["w"], b["b"], lr,
                                                 b["ws"], stream)
            if i > 0:
                if overlap:
                    cp.conv_part_wait(L, stream)
                if lr is not None and side:
                    # this layer's update (HBM-bound) on the comm stream - behind its dX reduction, which the
                    # main stream already waited for - while the next layer's backward runs on the SMs
                    ev = torch.cuda.Event()
                    ev.record(s_main)
                    comm_stream.wait_event(ev)
                    cp.conv_part_sgd_step(L, b["w"], b["b"], b["dw"], b["db"], lr, comm_stream)
                    joined = False
                da = b["dx"]
        if not joined:
            s_main.wait_stream(comm_stream)

    def sgd(self, lr, stream=None, head=True, convs=True):
        """SGD on the own conv slices (convs) and the head, one fused launch (cp_sgd_multi)."""
        pairs = []
        for i, b in enumerate(self.buf if convs else []):
            d, kr = self.descs[i], self.parts[i].k_count[self.rank]
            ktot = (self.sizes[i].w - 256) // 4 // max(kr, 1) if kr else 0
            pairs.append((b["w"], b["dw"], kr * ktot))
            pairs.append((b["b"], b["db"], kr))
        if head:
            pairs.append((self.head["wfc"], self.head["dwfc"]))
            pairs.append((self.head["bfc"], self.head["dbfc"]))
        if pairs:
            cp.cp_sgd_multi(pairs, lr, stream)

    def step(self, lr=0.01, dx_mode=cp.CP_DX_REDUCE_SCATTER, stream=None, comm_stream=None, overlap=True, head=True,
             fuse_sgd=False):
        """One SGD step; head=False: the conv stage with the head replaced by the fixed dA2 in head["da"]
        (SURVEY §8(d) conv-stage images/s).  fuse_sgd: the conv slices' update runs inside the backward
        pass (see backward(lr=...)) instead of one cp_sgd_multi launch at the end - measured no faster
        on B200, so off by default."""
        self.forward(stream, comm_stream, head)
        self.backward(dx_mode, stream, comm_stream, overlap, head, lr=lr if fuse_sgd else None)
        self.sgd(lr, stream, head, convs=not fuse_sgd)

    def loss(self):
        return float(self.head["loss"][0].item())

    def close(self):
        for L in self.layers:
            cp.conv_part_destroy(L)
        self.layers = []
        for b in self.buf:
            b.pop("y", None)
        self.head_x = None
        for s in self.sym:   # collective: every rank closes its net in the same order
            s.free()
        self.sym = []


def plan_even(kernels, world):
    return [cp.cp_partition_plan([1.0] * world, K) for K in kernels]
