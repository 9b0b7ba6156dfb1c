"""Oracle primitives (fp64).  TEST INFRASTRUCTURE -- see oracle/__init__.py.

Each function restates the operator it implements, with the passage that
defines it.  conv2d is plain C loops (oracle_conv.c); the rest is numpy fp64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_conv.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build_native(force: bool = False) -> str:
    """Compile oracle_conv.c with gcc (plain -O2, no fast-math) -> liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off",
                               "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _native():
    global _lib
    with _lock:
        if _lib is None:
            build_native()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.POINTER(ctypes.c_double)
            i = ctypes.c_int
            lib.oracle_conv2d_nhwc.argtypes = [P, i, i, i, P, i, i, i, i, P, P]
            lib.oracle_conv2d_nhwc.restype = None
            _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ---------------------------------------------------------------------------
def round_bf16(v):
    """Round fp64 values to the nearest bf16 value, ties to even (mirror mode).

    bf16 = 8 significant bits.  With v = m * 2^e, 0.5 <= |m| < 1 (frexp), the
    nearest bf16 is rint(m * 2^8) * 2^(e-8); np.rint rounds half to even.
    (Magnitudes here stay far inside the bf16 normal range.)
    """
    v = np.asarray(v, dtype=np.float64)
    m, e = np.frexp(v)
    return np.ldexp(np.rint(m * 256.0), e - 8)


def conv2d(x, w, b, stride: int, pad: int):
    """2-D convolution of one NHWC sample x[H,W,C] with w[Co,k,k,C] (+ bias b[Co]).

    The 'convolutional operator' node of the DNN DAG (Sec. 2.2).
    Implemented in oracle_conv.c as the literal definition.
    """
    x = np.ascontiguousarray(x, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    H, W, C = x.shape
    Co, k, k2, Cw = w.shape
    assert k == k2 and Cw == C, (x.shape, w.shape)
    Ho = (H + 2 * pad - k) // stride + 1
    Wo = (W + 2 * pad - k) // stride + 1
    y = np.empty((Ho, Wo, Co), dtype=np.float64)
    bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
    _native().oracle_conv2d_nhwc(_ptr(x), H, W, C, _ptr(w), Co, k, stride, pad,
                                 None if bb is None else _ptr(bb), _ptr(y))
    return y


def dense(w, b, v):
    """The 'dense operator': y = W v + b, W[n_out, n_in]."""
    return np.asarray(w, np.float64) @ np.asarray(v, np.float64) + np.asarray(b, np.float64)


def relu(v):
    return np.maximum(v, 0.0)


def gap(h):
    """Global average pooling of one sample h[H,W,C] -> [C]: (1/HW) sum_{h,w}."""
    h = np.asarray(h, np.float64)
    return h.reshape(-1, h.shape[-1]).sum(axis=0) / float(h.shape[0] * h.shape[1])


def max_softmax(z):
    """Exit confidence of an internal classifier: max_j softmax(z)_j.

    Shallow-Deep: 'If one of the exits is confident about the prediction, the
    execution is stopped early'.  max softmax = 1/sum_j exp(z_j - max z).
    """
    z = np.asarray(z, np.float64)
    return 1.0 / np.exp(z - z.max()).sum()


def sigmoid(z):
    """SkipNet gate probability p = 1/(1+exp(-z)) (gate values)."""
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-np.asarray(z, np.float64)))


def argmax_lowest(z):
    """argmax with ties broken by the lowest index (np.argmax does this)."""
    return int(np.argmax(np.asarray(z)))


def option_a(h, c_out: int):
    """Parameter-free 'option A' shortcut: spatial subsample by 2, zero-pad channels.

    out = pad_c(h[::2, ::2, :]) with (c_out - c_in)/2 zero channels on each side
    (reading R7: the CIFAR ResNet convention).
    """
    h = np.asarray(h, np.float64)
    sub = h[::2, ::2, :]
    p = (c_out - h.shape[2]) // 2
    return np.pad(sub, ((0, 0), (0, 0), (p, c_out - h.shape[2] - p)))


def maxpool2d(h, k: int = 3, stride: int = 2, pad: int = 1):
    """Max pooling of one NHWC sample: y[ho][wo][c] = max over the k x k window at
    (ho*stride - pad, wo*stride - pad); out-of-range positions never win (-inf padding)."""
    h = np.asarray(h, np.float64)
    H, W, C = h.shape
    Ho = (H + 2 * pad - k) // stride + 1
    Wo = (W + 2 * pad - k) // stride + 1
    hp = np.full((H + 2 * pad, W + 2 * pad, C), -np.inf)
    hp[pad:pad + H, pad:pad + W] = h
    y = np.full((Ho, Wo, C), -np.inf)
    for r in range(k):
        for s in range(k):
            y = np.maximum(y, hp[r:r + stride * Ho:stride, s:s + stride * Wo:stride])
    return y
