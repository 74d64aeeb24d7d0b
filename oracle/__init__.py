"""fp64 CPU oracle for kernel-partitioned conv-layer training (arXiv 1712.02546).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA product path
(``paper_1712_02546_b200``) and neither imports the other; the only common
dependency is ``synth`` (seeded input generators, no arithmetic of the method).

The arithmetic lives in ``convnet_oracle.c`` (plain fp64 direct loops, fixed
summation order, OpenMP only over independent outputs).  This module is ctypes
marshalling plus :func:`net_step`, which composes the primitives in the order of
the paper's training loop (Alg. 1: for each layer, conv layers are
computed per kernel slice "same inputs but different kernels" and the master
"reshapes and rearranges" the maps).

Parity pins: see tests/test_oracle_*.py.  Unpinned: absolute loss values
(the paper reports none) -> "parity unpinned" for losses as absolute
numbers; everything else is pinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "convnet_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

_D = ctypes.POINTER(ctypes.c_double)
_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)
_U8 = ctypes.POINTER(ctypes.c_uint8)
_i = ctypes.c_int


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            sig = {
                "orc_conv_fwd": [_D, _i, _i, _i, _i, _D, _i, _i, _i, _D, _D],
                "orc_conv_fwd_points": [_D, _i, _i, _i, _i, _D, _i, _i, _i, _D, _I64, ctypes.c_int64, _D],
                "orc_conv_dgrad": [_D, _i, _i, _i, _i, _D, _i, _i, _i, _i, _i, _i, _D],
                "orc_conv_dgrad_points": [_D, _i, _i, _i, _i, _D, _i, _i, _i, _I64, ctypes.c_int64, _D],
                "orc_conv_wgrad": [_D, _i, _i, _i, _i, _D, _i, _i, _i, _D],
                "orc_conv_wgrad_points": [_D, _i, _i, _i, _i, _D, _i, _i, _i, _I64, ctypes.c_int64, _D],
                "orc_bias_grad": [_D, _i, _i, _i, _i, _D],
                "orc_relu_pool_fwd": [_D, _i, _i, _i, _i, _i, _i, _D, _U8],
                "orc_unpool_relu_bwd": [_D, _U8, _D, _i, _i, _i, _i, _i, _i, _D],
                "orc_lrn_fwd": [_D, _i, _i, _i, _i, _i, ctypes.c_double, ctypes.c_double, ctypes.c_double, _D],
                "orc_lrn_bwd": [_D, _D, _i, _i, _i, _i, _i, ctypes.c_double, ctypes.c_double, ctypes.c_double, _D],
                "orc_fc_fwd": [_D, _i, _i, _D, _D, _i, _D],
                "orc_fc_bwd": [_D, _D, _D, _i, _i, _i, _D, _D, _D],
                "orc_softmax_xent": [_D, _I32, _i, _i, _D, _D],
                "orc_sgd": [_D, _D, ctypes.c_int64, ctypes.c_double],
                "orc_eq1_weights": [_D, _i, _D],
                "orc_plan": [_D, _i, _i, _i, _I32, _I32, _I32],
                "orc_pack_gather": [_D, _i, _i, _i, _i, _i, _i, _I32, _I32, _I32, _D],
            }
            for name, args in sig.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = ctypes.c_int
            _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _chk(rc, what):
    if rc != 0:
        raise OracleError(f"{what}: status {rc}")


def _d(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, "oracle needs C-contiguous float64"
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- layer primitives
def conv_fwd(x, w, bias=None):
    """Valid cross-correlation, stride 1. x [B,C,H,W], w [K,C,R,S]."""
    x, w = _f64(x), _f64(w)
    B, C, H, W = x.shape
    K, C2, R, S = w.shape
    if C2 != C:
        raise OracleError(f"dimension error: input {x.shape} vs kernels {w.shape}")
    z = np.empty((B, K, H - R + 1, W - S + 1))
    b = None if bias is None else _f64(bias)
    _chk(lib().orc_conv_fwd(_d(x), B, C, H, W, _d(w), K, R, S, _d(b), _d(z)), "conv_fwd")
    return z


def conv_fwd_points(x, w, bias, idx):
    x, w = _f64(x), _f64(w)
    B, C, H, W = x.shape
    K, _, R, S = w.shape
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.shape[0])
    b = None if bias is None else _f64(bias)
    _chk(lib().orc_conv_fwd_points(_d(x), B, C, H, W, _d(w), K, R, S, _d(b),
                                   idx.ctypes.data_as(_I64), idx.shape[0], _d(out)), "conv_fwd_points")
    return out


def conv_dgrad(dy, w, k_begin=None, k_end=None, accumulate_into=None):
    """dX of the conv.  Optional kernel slice [k_begin,k_end) = one rank's partial dX."""
    dy, w = _f64(dy), _f64(w)
    B, K, P, Q = dy.shape
    K2, C, R, S = w.shape
    if K2 != K:
        raise OracleError(f"dimension error: gradOut {dy.shape} vs kernels {w.shape}")
    kb = 0 if k_begin is None else k_begin
    ke = K if k_end is None else k_end
    if accumulate_into is not None:
        dx = accumulate_into
        acc = 1
    else:
        dx = np.empty((B, C, P + R - 1, Q + S - 1))
        acc = 0
    _chk(lib().orc_conv_dgrad(_d(dy), B, K, P, Q, _d(w), C, R, S, kb, ke, acc, _d(dx)), "conv_dgrad")
    return dx


def conv_dgrad_points(dy, w, idx):
    dy, w = _f64(dy), _f64(w)
    B, K, P, Q = dy.shape
    _, C, R, S = w.shape
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.shape[0])
    _chk(lib().orc_conv_dgrad_points(_d(dy), B, K, P, Q, _d(w), C, R, S,
                                     idx.ctypes.data_as(_I64), idx.shape[0], _d(out)), "dgrad_points")
    return out


def conv_wgrad(dy, x, R, S):
    """dW of the conv.  dy [B,K,P,Q], x [B,C,H,W] -> dw [K,C,R,S]."""
    dy, x = _f64(dy), _f64(x)
    B, K, P, Q = dy.shape
    B2, C, H, W = x.shape
    if B2 != B or H != P + R - 1 or W != Q + S - 1:
        raise OracleError(f"dimension error: gradOut {dy.shape} vs input {x.shape}")
    dw = np.empty((K, C, R, S))
    _chk(lib().orc_conv_wgrad(_d(dy), B, K, P, Q, _d(x), C, R, S, _d(dw)), "conv_wgrad")
    return dw


def conv_wgrad_points(dy, x, R, S, idx):
    dy, x = _f64(dy), _f64(x)
    B, K, P, Q = dy.shape
    _, C, _, _ = x.shape
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.shape[0])
    _chk(lib().orc_conv_wgrad_points(_d(dy), B, K, P, Q, _d(x), C, R, S,
                                     idx.ctypes.data_as(_I64), idx.shape[0], _d(out)), "wgrad_points")
    return out


def bias_grad(dy):
    dy = _f64(dy)
    B, K, P, Q = dy.shape
    db = np.empty(K)
    _chk(lib().orc_bias_grad(_d(dy), B, K, P, Q, _d(db)), "bias_grad")
    return db


def relu_pool_fwd(z, relu=True, pool=True):
    """ReLU then 2x2/2 max-pool with first-max tie rule.  Returns (a, argmax)."""
    z = _f64(z)
    B, K, H, W = z.shape
    if pool:
        if H % 2 or W % 2:
            raise OracleError(f"dimension error: pooling input {z.shape} not divisible by 2")
        a = np.empty((B, K, H // 2, W // 2))
        am = np.empty((B, K, H // 2, W // 2), dtype=np.uint8)
        amp = am.ctypes.data_as(_U8)
    else:
        a = np.empty_like(z)
        am, amp = None, None
    _chk(lib().orc_relu_pool_fwd(_d(z), B, K, H, W, int(relu), int(pool), _d(a), amp), "relu_pool_fwd")
    return a, am


def unpool_relu_bwd(da, argmax, a, relu=True, pool=True):
    """Route da through max-pool argmax and the ReLU mask; decisions replayable."""
    da, a = _f64(da), _f64(a)
    B, K, Hp, Wp = da.shape
    if pool:
        argmax = np.ascontiguousarray(argmax, dtype=np.uint8)
        dy = np.empty((B, K, 2 * Hp, 2 * Wp))
        amp = argmax.ctypes.data_as(_U8)
    else:
        dy = np.empty_like(da)
        amp = None
    _chk(lib().orc_unpool_relu_bwd(_d(da), amp, _d(a), B, K, Hp, Wp, int(relu), int(pool), _d(dy)),
         "unpool_relu_bwd")
    return dy


LRN_DEFAULT = {"depth": 5, "alpha": 1e-4, "beta": 0.75, "bias": 2.0}


def lrn_fwd(x, depth=5, alpha=1e-4, beta=0.75, bias=2.0):
    """Cross-channel LRN (form S:L89-97): out = in * (bias + alpha*sum_window in^2)^-beta."""
    x = _f64(x)
    B, C, H, W = x.shape
    out = np.empty_like(x)
    _chk(lib().orc_lrn_fwd(_d(x), B, C, H, W, int(depth), float(alpha), float(beta), float(bias), _d(out)), "lrn_fwd")
    return out


def lrn_bwd(x, dout, depth=5, alpha=1e-4, beta=0.75, bias=2.0):
    """Gradient of lrn_fwd w.r.t. its input (chain rule written out)."""
    x, dout = _f64(x), _f64(dout)
    B, C, H, W = x.shape
    din = np.empty_like(x)
    _chk(lib().orc_lrn_bwd(_d(x), _d(dout), B, C, H, W, int(depth), float(alpha), float(beta), float(bias),
                           _d(din)), "lrn_bwd")
    return din


def fc_fwd(a, wfc, bfc):
    a = _f64(a).reshape(a.shape[0], -1)
    wfc, bfc = _f64(wfc), _f64(bfc)
    B, F = a.shape
    O = wfc.shape[0]
    if wfc.shape[1] != F:
        raise OracleError(f"dimension error: features {a.shape} vs weights {wfc.shape}")
    out = np.empty((B, O))
    _chk(lib().orc_fc_fwd(_d(a), B, F, _d(wfc), _d(bfc), O, _d(out)), "fc_fwd")
    return out


def fc_bwd(dlogits, a, wfc):
    shape = a.shape
    a = _f64(a).reshape(a.shape[0], -1)
    dlogits, wfc = _f64(dlogits), _f64(wfc)
    B, F = a.shape
    O = wfc.shape[0]
    da = np.empty((B, F))
    dw = np.empty((O, F))
    db = np.empty(O)
    _chk(lib().orc_fc_bwd(_d(dlogits), _d(a), _d(wfc), B, F, O, _d(da), _d(dw), _d(db)), "fc_bwd")
    return da.reshape(shape), dw, db


def softmax_xent(logits, y):
    logits = _f64(logits)
    y = np.ascontiguousarray(y, dtype=np.int32)
    B, O = logits.shape
    loss = ctypes.c_double(0.0)
    dl = np.empty((B, O))
    _chk(lib().orc_softmax_xent(_d(logits), y.ctypes.data_as(_I32), B, O, ctypes.byref(loss), _d(dl)),
         "softmax_xent")
    return loss.value, dl


def sgd(p, g, lr):
    p = _f64(p).copy()
    g = _f64(g)
    if p.shape != g.shape:
        raise OracleError(f"dimension error: params {p.shape} vs grads {g.shape}")
    _chk(lib().orc_sgd(_d(p), _d(g), p.size, float(lr)), "sgd")
    return p


def eq1_weights(t):
    t = _f64(t)
    w = np.empty_like(t)
    _chk(lib().orc_eq1_weights(_d(t), t.size, _d(w)), "eq1_weights")
    return w


def plan(t, num_k, align=8):
    """Eq. 1 + exact-integer largest remainder -> (k_begin, k_count, k_width) int32 arrays."""
    t = _f64(t)
    n = t.size
    kb = np.zeros(n, np.int32)
    kc = np.zeros(n, np.int32)
    kw = np.zeros(n, np.int32)
    _chk(lib().orc_plan(_d(t), n, int(num_k), int(align), kb.ctypes.data_as(_I32),
                        kc.ctypes.data_as(_I32), kw.ctypes.data_as(_I32)), "plan")
    return kb, kc, kw


def pack_gather(x_nchw, Bp, k_begin, k_count, k_width):
    """NCHW -> rank-blocked gather layout [r][H][W][Bp][Kc_r] (flat), §8(c) item 9."""
    x = _f64(x_nchw)
    B, C, H, W = x.shape
    kb = np.ascontiguousarray(k_begin, np.int32)
    kc = np.ascontiguousarray(k_count, np.int32)
    kw = np.ascontiguousarray(k_width, np.int32)
    total = int(sum(H * W * Bp * int(v) for v in kw))
    out = np.empty(total)
    _chk(lib().orc_pack_gather(_d(x), B, C, H, W, Bp, len(kw), kb.ctypes.data_as(_I32),
                               kc.ctypes.data_as(_I32), kw.ctypes.data_as(_I32), _d(out)), "pack_gather")
    return out


# ---------------------------------------------------------------- the network step
def net_step(params, x, y, lr, layers, part=None, replay=None):
    """One SGD training step of the conv net, unsplit or kernel-partitioned.

    params: dict with 'w{i}', 'b{i}' per conv layer i (KCRS / K) and 'wfc' [O,F], 'bfc' [O].
    layers: list of dicts {'relu': bool, 'pool': bool[, 'lrn': {depth, alpha, beta, bias}]} per conv
            layer; with 'lrn' the layer is Conv -> ReLU -> LRN -> Pool.
    part:   None (unsplit) or list per conv layer of (k_begin, k_count) arrays: the
            layer's kernels are evaluated slice by slice and concatenated in channel
            order (Alg. 1 L15-22); partial dX are summed in rank
            order (north_star "partial dX contributions are summed").
    replay: None or per-layer dict {'argmax': uint8 NCHW, 'a': pooled output[, 'pre': pre-LRN map]} —
            decision replay of a GPU's argmax/ReLU decisions in the backward pass (reading R15).
    Returns a trace dict with every intermediate and the updated params.
    """
    tr = {"x": _f64(x)}
    n = len(layers)
    act = tr["x"]
    for i, L in enumerate(layers):
        w, b = params[f"w{i}"], params[f"b{i}"]
        if part is None:
            z = conv_fwd(act, w, b)
        else:
            kb, kc = part[i]
            z = np.concatenate([conv_fwd(act, w[kb[r]:kb[r] + kc[r]], b[kb[r]:kb[r] + kc[r]])
                                for r in range(len(kb)) if kc[r] > 0], axis=1)
        lrn = L.get("lrn")
        if lrn:
            # Conv -> (bias, ReLU) -> Normalization -> Pool (reading R23)
            r_, _ = relu_pool_fwd(z, L["relu"], False)
            nrm = lrn_fwd(r_, **lrn)
            a, am = relu_pool_fwd(nrm, False, L["pool"])
            tr[f"pre{i}"], tr[f"nrm{i}"] = r_, nrm
        else:
            a, am = relu_pool_fwd(z, L["relu"], L["pool"])
        tr[f"in{i}"], tr[f"z{i}"], tr[f"a{i}"], tr[f"argmax{i}"] = act, z, a, am
        act = a
    logits = fc_fwd(act, params["wfc"], params["bfc"])
    loss, dlogits = softmax_xent(logits, y)
    da, dwfc, dbfc = fc_bwd(dlogits, act, params["wfc"])
    tr.update(logits=logits, loss=loss, dlogits=dlogits, dwfc=dwfc, dbfc=dbfc)
    grads = {"wfc": dwfc, "bfc": dbfc}
    for i in reversed(range(n)):
        L = layers[i]
        tr[f"da{i}"] = da
        am = tr[f"argmax{i}"] if replay is None else replay[i]["argmax"]
        a = tr[f"a{i}"] if replay is None else _f64(replay[i]["a"])
        if L.get("lrn"):
            dn = unpool_relu_bwd(da, am, a, False, L["pool"])
            dpre = lrn_bwd(tr[f"pre{i}"], dn, **L["lrn"])
            # ReLU' from the pre-LRN map (replay: the GPU's map decides, reading R15)
            pre = tr[f"pre{i}"] if replay is None or "pre" not in replay[i] else _f64(replay[i]["pre"])
            dy = unpool_relu_bwd(dpre, None, pre, L["relu"], False)
        else:
            dy = unpool_relu_bwd(da, am, a, L["relu"], L["pool"])
        w = params[f"w{i}"]
        R, S = w.shape[2], w.shape[3]
        inp = tr[f"in{i}"]
        tr[f"dy{i}"] = dy
        grads[f"b{i}"] = bias_grad(dy)
        grads[f"w{i}"] = conv_wgrad(dy, inp, R, S)
        if i > 0:
            if part is None:
                da = conv_dgrad(dy, w)
            else:
                kb, kc = part[i]
                da = np.zeros(inp.shape)
                for r in range(len(kb)):
                    if kc[r] > 0:
                        da += conv_dgrad(dy, w, kb[r], kb[r] + kc[r])
    tr["grads"] = grads
    tr["new_params"] = {k: sgd(v, grads[k], lr) for k, v in params.items()}
    return tr
