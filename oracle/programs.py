"""The original (unrewritten) dynamic programs, interpreted one sample at a time.

TEST INFRASTRUCTURE -- see oracle/__init__.py.

Each program is the DyNN as written before DyCL's rewriting (Sec. 5.2,
L588-591): a loop over blocks with real ``if`` / ``return``, so the oracle is
the left-hand side of Eq. 2 (P_DyNN(x)).  Per sample it returns
the output logits, the path taken, and every predicate value it evaluated
(kind, value, threshold) so the harness can apply the 1e-3 band (reading R12).

Modes (reading R13; all three round the network input to bf16, the
a0 cast of Listing 2's pre-processing):
  'mirror'      -- the production numerics (fp32 residual stream): every tensor-
                   core operand is bf16 (RNE) -- the input of each conv / dense
                   layer is rounded, and so is a block's intermediate activation
                   (stored bf16); block outputs / sub-network outputs (the
                   residual stream) are NOT rounded.  Decisions are graded here.
  'mirror_bf16' -- every stored activation rounded to bf16 (the DYCL_PREC_BF16
                   storage mode).
  'exact'       -- no rounding after the bf16 input.
Pooled features, head/gate logits and predicates are never rounded.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .core import (conv2d, dense, gap, max_softmax, maxpool2d, option_a, relu,
                   round_bf16, sigmoid)


def _bf16_to_f64(bits):
    """Decode bf16 bit patterns: the value is the fp32 whose top half is the bits."""
    b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def prepare(W: dict) -> dict:
    """bf16 (uint16) tensors -> fp64; fp32 tensors -> fp64."""
    P = {}
    for k, v in W.items():
        v = np.asarray(v)
        P[k] = _bf16_to_f64(v) if v.dtype == np.uint16 else v.astype(np.float64)
    return P


def _operand(v, mode):
    """A tensor-core operand: bf16 in both mirror modes."""
    return round_bf16(v) if mode in ("mirror", "mirror_bf16") else v


def _inner(v, mode):
    """An activation consumed only by the next conv (stored bf16 in both mirror modes)."""
    return round_bf16(v) if mode in ("mirror", "mirror_bf16") else v


def _stream(v, mode):
    """A residual-stream / sub-network output tensor (bf16 only in mirror_bf16)."""
    return round_bf16(v) if mode == "mirror_bf16" else v


# ---------------------------------------------------------------------------
# Config 1: tiny early-exit MLP (BASELINE configs[0]).
#   h = x; for k in 0..2: h = relu(W_k h + b_k); z = H_k h + c_k
#          if k < 2 and maxsoftmax(z) >= tau: return (z, k)
#   return (z, 2)
# Early termination per Shallow-Deep; comparator '>=' is
# reading R1; the final head is the default exit (reading R3).
# ---------------------------------------------------------------------------
def mlp_ee(x, P, mode="mirror", tau=0.9):
    preds = []
    h = round_bf16(np.asarray(x, np.float64))                 # a0: input cast to bf16
    for k in range(3):
        h = _stream(relu(dense(P[f"fc{k}.w"], P[f"fc{k}.b"], _operand(h, mode))), mode)
        z = dense(P[f"head{k}.w"], P[f"head{k}.b"], h)
        if k < 2:
            conf = max_softmax(z)
            preds.append(("exit", conf, tau))
            if conf >= tau:
                return z, k, preds
    return z, 2, preds


# ---------------------------------------------------------------------------
# CIFAR ResNet pieces shared by configs 2 and 3 (He et al. basic block,
# 'option A' parameter-free shortcut at stage transitions).
# ---------------------------------------------------------------------------
def _block_io(i, per_stage, widths=(16, 32, 64)):
    s = (i - 1) // per_stage
    first = (i - 1) % per_stage == 0
    if s > 0 and first:
        return widths[s - 1], widths[s], 2
    return widths[s], widths[s], 1


def basic_block(h, P, i, per_stage, mode):
    """relu(conv2(relu(conv1(h) + b1)) + b2 + shortcut(h))."""
    ci, co, stride = _block_io(i, per_stage)
    t = _inner(relu(conv2d(_operand(h, mode), P[f"b{i}.c1.w"], P[f"b{i}.c1.b"], stride, 1)), mode)
    sc = h if stride == 1 else option_a(h, co)
    return _stream(relu(conv2d(t, P[f"b{i}.c2.w"], P[f"b{i}.c2.b"], 1, 1) + sc), mode)


def stem(x, P, mode):
    h = round_bf16(np.asarray(x, np.float64))                 # a0: input cast to bf16
    return _stream(relu(conv2d(h, P["stem.w"], P["stem.b"], 1, 1)), mode)


# ---------------------------------------------------------------------------
# Config 2: ShallowDeep-style early-exit ResNet-56 (BASELINE configs[1]).
#   h = stem(x); for blk in 1..27: h = block(h)
#       if blk in {5,11,16,22}: z = IC_k(GAP(h)); if maxsoftmax(z) >= tau: return (z, k)
#   return (FC_final(GAP(h)), 4)
# IC placement: reading R4.  Head = GAP -> FC (reading R5).
# ---------------------------------------------------------------------------
SDN_IC_AFTER = (5, 11, 16, 22)


def sdn_resnet56(x, P, mode="mirror", tau=0.9, features=None):
    preds = []
    h = stem(x, P, mode)
    k = 0
    for blk in range(1, 28):
        h = basic_block(h, P, blk, 9, mode)
        if blk in SDN_IC_AFTER:
            g = gap(h)
            if features is not None:
                features.append(g)
            z = dense(P[f"ic{k}.w"], P[f"ic{k}.b"], g)
            conf = max_softmax(z)
            preds.append(("exit", conf, tau))
            if conf >= tau:
                return z, k, preds
            k += 1
    g = gap(h)
    if features is not None:
        features.append(g)
    return dense(P["final.w"], P["final.b"], g), 4, preds


# ---------------------------------------------------------------------------
# Config 3: SkipNet-style gated ResNet-38 (BASELINE configs[2]).
# Listing 3: the first block always runs; for the others
#   'if mask == 0: x = (1 - mask) * prev  else: x = layer(x)'.
#   h = stem(x); h = block_1(h); mask = 0
#   for i in 2..18: p = sigmoid(gate_i(GAP(h)))           # gate on the block INPUT
#        if p > 0.5: h = block_i(h); mask |= 1 << (i-2)
#        else:       h = optionA(h) if i in {7,13} else h   # skip = identity path
#   return (FC(GAP(h)), mask)
# Comparator '>' : reading R2; transition skips: reading R7.
# ---------------------------------------------------------------------------
def skipnet_resnet38(x, P, mode="mirror", thr=0.5, gate_hook=None):
    preds = []
    h = stem(x, P, mode)
    h = basic_block(h, P, 1, 6, mode)
    mask = 0
    for i in range(2, 19):
        g = gap(h)
        z = dense(P[f"gate{i}.w"], P[f"gate{i}.b"], g)[0]
        if gate_hook is not None:
            gate_hook(i, g, z)
        p = sigmoid(z)
        preds.append(("gate", p, thr))
        if p > thr:
            h = basic_block(h, P, i, 6, mode)
            mask |= 1 << (i - 2)
        else:
            ci, co, stride = _block_io(i, 6)
            h = option_a(h, co) if stride == 2 else h
    return dense(P["final.w"], P["final.b"], gap(h)), mask, preds


# ---------------------------------------------------------------------------
# SkipNet with the recurrent gate (Table 3 ID 5 "ResNet38 + RNN"; SURVEY 8(f)3;
# reading R19).  Same trunk, same Listing-3 control flow as config 3; the gate of block i is
#   u = proj_i(GAP(h))                       (dense C_i -> n_in, bf16 weights, fp32 logits)
#   (hs, cs) = LSTMCell(u, (hs, cs))          (one cell shared by all gates, state carried across
#                                             gates in program order, zero before gate 2; torch
#                                             gate order i, f, g, o)
#   p = sigmoid(w_out_i . hs + b_out_i)       (per-gate calibrated output, fp32)
# and the cell steps at EVERY gate, whether the block then runs or not.
# ---------------------------------------------------------------------------
def lstm_cell(u, hs, cs, P):
    """One LSTM step (torch.nn.LSTMCell semantics), fp64."""
    gates = P["rnn.w_ih"] @ u + P["rnn.b_ih"] + P["rnn.w_hh"] @ hs + P["rnn.b_hh"]
    H = hs.shape[0]
    i_ = sigmoid(gates[0:H])
    f_ = sigmoid(gates[H:2 * H])
    g_ = np.tanh(gates[2 * H:3 * H])
    o_ = sigmoid(gates[3 * H:4 * H])
    cs = f_ * cs + i_ * g_
    return o_ * np.tanh(cs), cs


def skipnet_rnn_resnet38(x, P, mode="mirror", thr=0.5, gate_hook=None):
    preds = []
    h = stem(x, P, mode)
    h = basic_block(h, P, 1, 6, mode)
    H = int(P["rnn.hidden"])
    hs, cs = np.zeros(H), np.zeros(H)
    mask = 0
    for i in range(2, 19):
        g = gap(h)
        u = dense(P[f"proj{i}.w"], P[f"proj{i}.b"], g)
        hs, cs = lstm_cell(u, hs, cs, P)
        z = float(P[f"out{i}.w"] @ hs + P[f"out{i}.b"][0])
        if gate_hook is not None:
            gate_hook(i, g, hs, z)
        p = sigmoid(z)
        preds.append(("gate", p, thr))
        if p > thr:
            h = basic_block(h, P, i, 6, mode)
            mask |= 1 << (i - 2)
        else:
            ci, co, stride = _block_io(i, 6)
            h = option_a(h, co) if stride == 2 else h
    return dense(P["final.w"], P["final.b"], gap(h)), mask, preds


# ---------------------------------------------------------------------------
# Config 5: early-exit ResNet-50 v1.5 (BASELINE configs[4]).
#   h = maxpool(relu(conv7x7/2(x)))
#   for stage s in 1..4: for each bottleneck b: h = bottleneck(h)
#       if s in {1,2,3}: z = IC_s(GAP(h)); if maxsoftmax(z) >= tau: return (z, s-1)
#   return (FC(GAP(h)), 3)
# bottleneck(h) = relu(conv1x1(relu(conv3x3/stride(relu(conv1x1(h))))) + shortcut(h)),
# shortcut = conv1x1/stride(h) (projection) for the first block of a stage, else h.
# Exit placement: reading R6.  1000 classes.
# ---------------------------------------------------------------------------
R50_LAYERS = (3, 4, 6, 3)
R50_WIDTHS = (64, 128, 256, 512)


def bottleneck(h, P, s, b, mode):
    stride = 2 if (b == 0 and s > 1) else 1
    p = f"s{s}b{b}"
    t = _inner(relu(conv2d(_operand(h, mode), P[f"{p}.c1.w"], P[f"{p}.c1.b"], 1, 0)), mode)
    t = _inner(relu(conv2d(t, P[f"{p}.c2.w"], P[f"{p}.c2.b"], stride, 1)), mode)
    if b == 0:
        sc = _stream(conv2d(_operand(h, mode), P[f"{p}.proj.w"], P[f"{p}.proj.b"], stride, 0), mode)
    else:
        sc = h
    return _stream(relu(conv2d(t, P[f"{p}.c3.w"], P[f"{p}.c3.b"], 1, 0) + sc), mode)


def resnet50_ee(x, P, mode="mirror", tau=0.9, features=None):
    preds = []
    h = round_bf16(np.asarray(x, np.float64))                 # a0: input cast to bf16
    h = _stream(relu(conv2d(h, P["stem.w"], P["stem.b"], 2, 3)), mode)
    h = maxpool2d(h, 3, 2, 1)
    k = 0
    for s in range(1, 5):
        for b in range(R50_LAYERS[s - 1]):
            h = bottleneck(h, P, s, b, mode)
        if s < 4:
            g = gap(h)
            if features is not None:
                features.append(g)
            z = dense(P[f"ic{k}.w"], P[f"ic{k}.b"], g)
            conf = max_softmax(z)
            preds.append(("exit", conf, tau))
            if conf >= tau:
                return z, k, preds
            k += 1
    g = gap(h)
    if features is not None:
        features.append(g)
    return dense(P["final.w"], P["final.b"], g), 3, preds


PROGRAMS = {1: mlp_ee, 2: sdn_resnet56, 3: skipnet_resnet38, 5: resnet50_ee}


def run_batch(program, X, P, mode="mirror", threads=None, **kw):
    """Run ``program`` independently on every sample of X (no batching).

    Returns (logits [B, K] fp64, path [B] int64, preds list-of-lists).
    Samples are spread over a thread pool; the C conv releases the GIL.
    """
    threads = threads or len(os.sched_getaffinity(0))
    n = len(X)

    def one(i):
        return program(X[i], P, mode, **kw)

    if threads <= 1 or n <= 1:
        res = [one(i) for i in range(n)]
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            res = list(ex.map(one, range(n)))
    logits = np.stack([np.asarray(r[0], np.float64) for r in res]) if n else np.zeros((0, 10))
    path = np.array([r[1] for r in res], dtype=np.int64)
    preds = [r[2] for r in res]
    return logits, path, preds
