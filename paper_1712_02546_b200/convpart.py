"""Thin ctypes binding of libconvpart (include/convpart.h): argument marshalling only.

Every step of the method runs in the library's CUDA kernels and NCCL calls; this module
never computes anything itself.  If the library is missing the import fails loudly
(no CPU fallback).  Names mirror the C ABI.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CP_LIB") or os.path.join(HERE, "libconvpart.so")   # CP_LIB: experiment builds

CP_MAX_RANKS = 16
CP_OK = 0
ERRORS = {-1: "CP_ERR_ARG", -2: "CP_ERR_SHAPE", -3: "CP_ERR_CONFIG", -4: "CP_ERR_DATA", -5: "CP_ERR_CUDA",
          -6: "CP_ERR_NCCL", -7: "CP_ERR_STATE", -8: "CP_ERR_UNSUPPORTED"}
CP_MATH_TF32, CP_MATH_FP32_SIMT, CP_MATH_BF16 = 0, 1, 2
CP_DX_ALLREDUCE, CP_DX_REDUCE_SCATTER, CP_DX_LOCAL, CP_DX_ASYNC, CP_DX_ORDERED = 0, 1, 2, 16, 64
CP_INPUT_IMAGES, CP_INPUT_GATHER = 0, 1

# every symbol include/convpart.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "cp_partition_plan", "cp_eq1_weights", "cp_comm_unique_id", "cp_comm_create", "cp_comm_destroy",
    "conv_part_create", "conv_part_query", "conv_part_destroy", "conv_part_probe_bytes", "conv_part_probe",
    "conv_part_forward", "conv_part_backward_data", "conv_part_backward_filter", "conv_part_backward_filter_sgd",
    "conv_part_wait", "conv_part_sgd_step",
    "cp_launch_count", "cp_last_error", "cp_pack_nchw", "cp_unpack_nchw", "cp_unpack_saved",
    "cp_pack_conv_weights", "cp_unpack_conv_weights", "cp_head_workspace_bytes", "cp_pack_fc_weights",
    "cp_unpack_fc_weights", "cp_fc_forward", "cp_softmax_xent", "cp_fc_backward", "cp_sgd",
    "cp_allreduce_sum", "cp_allreduce_softmax_xent", "cp_symmetric_alloc", "cp_symmetric_free", "cp_symmetric_wait", "conv_part_timing", "conv_part_kernel_time",
    "cp_sgd_multi", "cp_lrn_pool_forward", "cp_lrn_pool_backward", "cp_comm_create_loopback", "cp_symmetric_peer",
]
CP_GATHER_CHUNKS = 256   # convpart.h: a complete gather block raises its arrival counter to this


class cp_partition(ctypes.Structure):
    _fields_ = [("n_ranks", ctypes.c_int32), ("num_k", ctypes.c_int32),
                ("k_begin", ctypes.c_int32 * CP_MAX_RANKS), ("k_count", ctypes.c_int32 * CP_MAX_RANKS),
                ("k_width", ctypes.c_int32 * CP_MAX_RANKS)]

    def as_tuple(self):
        n = self.n_ranks
        return (list(self.k_begin[:n]), list(self.k_count[:n]), list(self.k_width[:n]))

    @classmethod
    def from_counts(cls, counts, align=8):
        p = cls()
        p.n_ranks = len(counts)
        p.num_k = int(sum(counts))
        b = 0
        for r, c in enumerate(counts):
            p.k_begin[r] = b
            p.k_count[r] = int(c)
            p.k_width[r] = (int(c) + align - 1) // align * align
            b += int(c)
        return p


class cp_conv_desc(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("in_c", ctypes.c_int32), ("in_h", ctypes.c_int32),
                ("in_w", ctypes.c_int32), ("num_k", ctypes.c_int32), ("k_h", ctypes.c_int32),
                ("k_w", ctypes.c_int32), ("bias", ctypes.c_int32), ("relu", ctypes.c_int32),
                ("pool", ctypes.c_int32), ("math", ctypes.c_int32), ("input_kind", ctypes.c_int32),
                ("out_part", cp_partition), ("in_part", cp_partition), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("local_output", ctypes.c_int32)]


class cp_sizes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_size_t)
                for n in ("w", "b", "x", "y", "y_block", "y_offset", "saved", "dx", "workspace", "dx_peer")]


class ConvPartError(RuntimeError):
    def __init__(self, fn, rc, msg):
        super().__init__(f"{fn} -> {ERRORS.get(rc, rc)}: {msg}")
        self.rc = rc


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libconvpart.so not built at {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, SZ, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_double
        pp = ctypes.POINTER(cp_partition)
        pd = ctypes.POINTER(cp_conv_desc)
        sig = {
            "cp_partition_plan": [ctypes.POINTER(D), I32, I32, I32, pp],
            "cp_eq1_weights": [ctypes.POINTER(D), I32, ctypes.POINTER(D)],
            "cp_comm_unique_id": [ctypes.c_char_p],
            "cp_comm_create": [ctypes.c_char_p, I32, I32, ctypes.POINTER(P)],
            "cp_comm_destroy": [P],
            "conv_part_create": [pd, P, ctypes.POINTER(P)],
            "conv_part_query": [P, ctypes.POINTER(cp_sizes)],
            "conv_part_destroy": [P],
            "conv_part_probe_bytes": [pd, ctypes.POINTER(SZ)],
            "conv_part_probe": [pd, I32, I32, P, SZ, P, ctypes.POINTER(D)],
            "conv_part_forward": [P, P, P, P, P, P, P, P, P],
            "conv_part_backward_data": [P, P, P, P, P, P, I32, P, P, P],
            "conv_part_backward_filter": [P, P, P, P, P, P, P, P, P],
            "conv_part_backward_filter_sgd": [P, P, P, P, P, P, P, P, P, ctypes.c_float, P, P],
            "conv_part_sgd_step": [P, P, P, P, P, ctypes.c_float, P],
            "conv_part_wait": [P, P],
            "cp_pack_nchw": [P, I32, I32, I32, I32, pp, P, P],
            "cp_unpack_nchw": [P, I32, I32, I32, I32, pp, P, P],
            "cp_unpack_saved": [P, I32, I32, I32, pp, I32, P, P],
            "cp_pack_conv_weights": [pd, P, P, P],
            "cp_unpack_conv_weights": [pd, P, P, P],
            "cp_head_workspace_bytes": [I32, I32, I32, pp, I32, ctypes.POINTER(SZ)],
            "cp_pack_fc_weights": [P, I32, I32, I32, pp, P, P],
            "cp_unpack_fc_weights": [P, I32, I32, I32, pp, P, P],
            "cp_fc_forward": [P, I32, I32, I32, pp, P, P, I32, P, P, P],
            "cp_softmax_xent": [P, P, I32, I32, P, P, P],
            "cp_fc_backward": [P, P, I32, I32, I32, pp, P, I32, P, P, P, P, P],
            "cp_sgd": [P, P, I64, ctypes.c_float, P],
            "cp_allreduce_sum": [P, P, I64, P],
            "cp_allreduce_softmax_xent": [P, P, P, I32, I32, P, P, P],
            "cp_symmetric_alloc": [P, SZ, ctypes.POINTER(P)],
            "cp_symmetric_free": [P, P],
            "cp_symmetric_wait": [P, P, P],
            "cp_comm_create_loopback": [I32, ctypes.POINTER(P)],
            "cp_symmetric_peer": [P, P, I32, ctypes.POINTER(P), ctypes.POINTER(P)],
            "conv_part_timing": [P, I32],
            "cp_sgd_multi": [ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(I64), I32, ctypes.c_float, P],
            "cp_lrn_pool_forward": [P, I32, I32, I32, pp, I32, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                    I32, P, P, P],
            "cp_lrn_pool_backward": [P, P, P, I32, I32, I32, pp, I32, I32, ctypes.c_float, ctypes.c_float,
                                     ctypes.c_float, P, P],
            "conv_part_kernel_time": [P, I32, ctypes.POINTER(ctypes.c_float)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.cp_launch_count.argtypes = []
        L.cp_launch_count.restype = ctypes.c_int64
        L.cp_last_error.argtypes = []
        L.cp_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc != CP_OK:
        raise ConvPartError(name, rc, lib().cp_last_error().decode(errors="replace"))
    return rc


def _ptr(t):
    """Device (or host) pointer of a torch tensor / None."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return ctypes.c_void_p(s)
    return ctypes.c_void_p(s.cuda_stream)


# ---------------------------------------------------------------- plan / comm
def cp_partition_plan(times, num_k, align=8):
    n = len(times)
    arr = (ctypes.c_double * n)(*[float(t) for t in times])
    out = cp_partition()
    _call("cp_partition_plan", arr, n, int(num_k), int(align), ctypes.byref(out))
    return out


def cp_eq1_weights(times):
    n = len(times)
    arr = (ctypes.c_double * n)(*[float(t) for t in times])
    out = (ctypes.c_double * n)()
    _call("cp_eq1_weights", arr, n, out)
    return list(out)


def cp_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _call("cp_comm_unique_id", buf)
    return buf.raw


def cp_comm_create(uid: bytes, rank: int, world: int):
    h = ctypes.c_void_p()
    _call("cp_comm_create", ctypes.c_char_p(uid), rank, world, ctypes.byref(h))
    return h


def cp_comm_destroy(h):
    _call("cp_comm_destroy", h)


def cp_comm_create_loopback(world):
    """`world` simulated ranks on the current GPU (tests of the fused paths): one handle per rank."""
    arr = (ctypes.c_void_p * world)()
    _call("cp_comm_create_loopback", int(world), arr)
    return [ctypes.c_void_p(arr[r]) for r in range(world)]


def cp_symmetric_peer(comm, local_ptr, rank):
    """(data pointer, flag-line pointer) of rank `rank`'s copy of a symmetric buffer, as ints."""
    d, f = ctypes.c_void_p(), ctypes.c_void_p()
    _call("cp_symmetric_peer", comm, ctypes.c_void_p(local_ptr), int(rank), ctypes.byref(d), ctypes.byref(f))
    return d.value, f.value


# ---------------------------------------------------------------- layers
def conv_part_create(desc: cp_conv_desc, comm=None):
    h = ctypes.c_void_p()
    _call("conv_part_create", ctypes.byref(desc), comm, ctypes.byref(h))
    return h


def conv_part_query(h) -> cp_sizes:
    s = cp_sizes()
    _call("conv_part_query", h, ctypes.byref(s))
    return s


def conv_part_destroy(h):
    _call("conv_part_destroy", h)


def conv_part_probe_bytes(desc):
    n = ctypes.c_size_t()
    _call("conv_part_probe_bytes", ctypes.byref(desc), ctypes.byref(n))
    return n.value


def conv_part_probe(desc, scratch, warmups=1, reps=3, stream=None):
    t = ctypes.c_double()
    _call("conv_part_probe", ctypes.byref(desc), warmups, reps, _ptr(scratch),
          scratch.numel() * scratch.element_size(), _stream(stream), ctypes.byref(t))
    return t.value


def conv_part_forward(h, x, w, b, y, saved, ws, stream=None, comm_stream=None):
    _call("conv_part_forward", h, _ptr(x), _ptr(w), _ptr(b), _ptr(y), _ptr(saved), _ptr(ws),
          _stream(stream), _stream(comm_stream))


def conv_part_backward_data(h, dy, saved, y, w, dx, dx_mode, ws, stream=None, comm_stream=None):
    _call("conv_part_backward_data", h, _ptr(dy), _ptr(saved), _ptr(y), _ptr(w), _ptr(dx), int(dx_mode),
          _ptr(ws), _stream(stream), _stream(comm_stream))


def conv_part_backward_filter(h, dy, saved, y, x, dw, db, ws, stream=None):
    _call("conv_part_backward_filter", h, _ptr(dy), _ptr(saved), _ptr(y), _ptr(x), _ptr(dw), _ptr(db),
          _ptr(ws), _stream(stream))


def conv_part_backward_filter_sgd(h, dy, saved, y, x, dw, db, w, b, lr, ws, stream=None):
    """backward_filter + the own slice's SGD step (w -= lr*dw, b -= lr*db) fused where dW / db are final."""
    _call("conv_part_backward_filter_sgd", h, _ptr(dy), _ptr(saved), _ptr(y), _ptr(x), _ptr(dw), _ptr(db), _ptr(w),
          _ptr(b), float(lr), _ptr(ws), _stream(stream))


def conv_part_wait(h, stream=None):
    _call("conv_part_wait", h, _stream(stream))


def conv_part_sgd_step(h, w, b, dw, db, lr, stream=None):
    _call("conv_part_sgd_step", h, _ptr(w), _ptr(b), _ptr(dw), _ptr(db), float(lr), _stream(stream))


def cp_launch_count() -> int:
    return int(lib().cp_launch_count())


# ---------------------------------------------------------------- helpers / head
def cp_pack_nchw(x, B, C, H, W, part, out, stream=None):
    _call("cp_pack_nchw", _ptr(x), B, C, H, W, ctypes.byref(part), _ptr(out), _stream(stream))


def cp_unpack_nchw(g, B, C, H, W, part, out, stream=None):
    _call("cp_unpack_nchw", _ptr(g), B, C, H, W, ctypes.byref(part), _ptr(out), _stream(stream))


def cp_unpack_saved(saved, B, Hp, Wp, part, rank, out, stream=None):
    _call("cp_unpack_saved", _ptr(saved), B, Hp, Wp, ctypes.byref(part), rank, _ptr(out), _stream(stream))


def cp_pack_conv_weights(desc, w, out, stream=None):
    _call("cp_pack_conv_weights", ctypes.byref(desc), _ptr(w), _ptr(out), _stream(stream))


def cp_unpack_conv_weights(desc, wg, out, stream=None):
    _call("cp_unpack_conv_weights", ctypes.byref(desc), _ptr(wg), _ptr(out), _stream(stream))


def cp_head_workspace_bytes(B, Hp, Wp, part, O):
    n = ctypes.c_size_t()
    _call("cp_head_workspace_bytes", B, Hp, Wp, ctypes.byref(part), O, ctypes.byref(n))
    return n.value


def cp_pack_fc_weights(wfc, O, Hp, Wp, part, out, stream=None):
    _call("cp_pack_fc_weights", _ptr(wfc), O, Hp, Wp, ctypes.byref(part), _ptr(out), _stream(stream))


def cp_unpack_fc_weights(wg, O, Hp, Wp, part, out, stream=None):
    _call("cp_unpack_fc_weights", _ptr(wg), O, Hp, Wp, ctypes.byref(part), _ptr(out), _stream(stream))


def cp_fc_forward(x, B, Hp, Wp, part, wg, bfc, O, logits, ws, stream=None):
    _call("cp_fc_forward", _ptr(x), B, Hp, Wp, ctypes.byref(part), _ptr(wg), _ptr(bfc), O, _ptr(logits),
          _ptr(ws), _stream(stream))


def cp_softmax_xent(logits, labels, B, O, loss, dlogits, stream=None):
    _call("cp_softmax_xent", _ptr(logits), _ptr(labels), B, O, _ptr(loss), _ptr(dlogits), _stream(stream))


def cp_fc_backward(dl, x, B, Hp, Wp, part, wg, O, dx, dwg, dbfc, ws, stream=None):
    _call("cp_fc_backward", _ptr(dl), _ptr(x), B, Hp, Wp, ctypes.byref(part), _ptr(wg), O, _ptr(dx), _ptr(dwg),
          _ptr(dbfc), _ptr(ws), _stream(stream))


def cp_allreduce_sum(comm, buf, stream=None):
    _call("cp_allreduce_sum", comm, _ptr(buf), buf.numel(), _stream(stream))


def cp_allreduce_softmax_xent(comm, logits, labels, B, O, loss, dlogits, stream=None):
    """Sum the partial logits over all ranks, then softmax cross-entropy - one launch on the one-shot path."""
    _call("cp_allreduce_softmax_xent", comm, _ptr(logits), _ptr(labels), int(B), int(O), _ptr(loss), _ptr(dlogits),
          _stream(stream))


class SymmetricBuffer:
    """Device memory from cp_symmetric_alloc, exposed to torch via __cuda_array_interface__."""

    def __init__(self, comm, nbytes, device):
        self.comm, self.nbytes = comm, int(nbytes)
        ptr = ctypes.c_void_p()
        _call("cp_symmetric_alloc", comm, self.nbytes, ctypes.byref(ptr))
        self.ptr = ptr.value
        self.__cuda_array_interface__ = {"shape": (self.nbytes // 4,), "typestr": "<f4",
                                         "data": (self.ptr, False), "version": 2}
        import torch
        self.tensor = torch.as_tensor(self, device=device)

    def wait(self, stream=None):
        """Before reading the gathered buffer outside conv_part_forward: wait for every peer's block."""
        _call("cp_symmetric_wait", self.comm, ctypes.c_void_p(self.ptr), _stream(stream))

    def free(self):
        if self.ptr:
            _call("cp_symmetric_free", self.comm, ctypes.c_void_p(self.ptr))
            self.ptr = None


def conv_part_timing(h, enable=True):
    _call("conv_part_timing", h, 1 if enable else 0)


def conv_part_kernel_time(h, pass_):
    ms = ctypes.c_float()
    _call("conv_part_kernel_time", h, int(pass_), ctypes.byref(ms))
    return ms.value


def cp_sgd_multi(pairs, lr, stream=None):
    """pairs: [(param, grad[, n])] of float32 device tensors; one fused update launch."""
    n = len(pairs)
    ps = (ctypes.c_void_p * max(n, 1))(*[t[0].data_ptr() for t in pairs])
    gs = (ctypes.c_void_p * max(n, 1))(*[t[1].data_ptr() for t in pairs])
    sz = (ctypes.c_int64 * max(n, 1))(*[int(t[2]) if len(t) > 2 else t[0].numel() for t in pairs])
    _call("cp_sgd_multi", ps, gs, sz, n, float(lr), _stream(stream))


LRN_DEFAULT = {"depth": 5, "alpha": 1e-4, "beta": 0.75, "bias": 2.0}


def cp_lrn_pool_forward(a, B, H, W, part, lrn, round_tf32, y, codes, stream=None):
    _call("cp_lrn_pool_forward", _ptr(a), B, H, W, ctypes.byref(part), int(lrn["depth"]), float(lrn["alpha"]),
          float(lrn["beta"]), float(lrn["bias"]), int(round_tf32), _ptr(y), _ptr(codes), _stream(stream))


def cp_lrn_pool_backward(dy, a, codes, B, H, W, part, rank, lrn, da, stream=None):
    _call("cp_lrn_pool_backward", _ptr(dy), _ptr(a), _ptr(codes), B, H, W, ctypes.byref(part), int(rank),
          int(lrn["depth"]), float(lrn["alpha"]), float(lrn["beta"]), float(lrn["bias"]), _ptr(da), _stream(stream))


def cp_sgd(p, g, lr, stream=None):
    _call("cp_sgd", _ptr(p), _ptr(g), p.numel(), float(lr), _stream(stream))
