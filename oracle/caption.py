"""Image captioning En-Decoder: a CNN encoder and a soft-attention LSTM decoder
decoded greedily under a per-caption EOS / max-length loop guard.

TEST INFRASTRUCTURE -- see oracle/__init__.py.

The paper's En-Decoder is "Show, Attend and Tell" ("En-Decoder / Image caption /
token wise caption generation", L323 "En-Decoder ... uses two different types of attention
mechanisms to generate captions"; Table 3 IDs 7-8 pair a CNN with an LSTM, L814-815).  It is a
generative DyNN: its loop runs until the `If` node on the output token sees EOS (L265), under
the constant iteration bound of L267-268.  Reading R20 fixes the synthetic
architecture; per image, with the loop and the `if` as written:

    a = Encoder(x)                       CIFAR ResNet-38 trunk -> 8x8x64 feature map, the
                                         L = 64 annotation vectors a_j (D = 64)
    h = tanh(W_h mean(a) + b_h);  c = tanh(W_c mean(a) + b_c)
    y = BOS;  done = False;  L = max_len
    for t in 0..max_len-1:
        if done: out[t] = PAD; continue
        q = W_q h + b_q                                     (D)
        alpha = softmax_j(a_j . q / sqrt(D));  z = sum_j alpha_j a_j       (soft attention)
        (i, f, g, o) = W [E[y]; z; h] + b;  c = sig(f) c + sig(i) tanh(g);  h = sig(o) tanh(c)
        logits = W_o h + b_o;  tok = argmax (lowest index on ties)
        out[t] = tok;  y = tok;  if tok == EOS: done = True; L = t + 1
    return out, L

Modes as in programs.py / seq2seq.py: 'mirror' rounds every tensor-core operand to bf16 (the
encoder as config 3's trunk in mirror mode, then the feature map a (stored bf16), mean(a), h,
z and the word embedding rows (bf16 weights)); the state h, c, q, the attention weights and
the logits stay unrounded; 'exact' rounds nothing after the bf16 input and weights.
"""
from __future__ import annotations

import math

import numpy as np

from . import programs as prg
from .core import round_bf16, sigmoid


def _r(v, mode):
    return round_bf16(v) if mode in ("mirror", "mirror_bf16") else v


def encode(x, P, mode="mirror"):
    """CNN encoder: the CIFAR ResNet-38 trunk (config 3's blocks, all executed) -> [64, 64]
    annotation vectors (row j = pixel j of the 8x8 map, NHWC order), stored bf16 in mirror."""
    h = prg.stem(x, P, mode)
    for i in range(1, 19):
        h = prg.basic_block(h, P, i, 6, mode)
    a = np.asarray(h, np.float64).reshape(-1, h.shape[-1])
    return _r(a, mode)


def _softmax(e):
    e = e - e.max()
    p = np.exp(e)
    return p / p.sum()


def decode(a, P, cfg, mode="mirror", eos_bias=None, forced=None):
    """Greedy soft-attention LSTM decode of one image's annotation vectors a [L, D].
    Returns (tokens [max_len], length, top1 logit per step (nan after done), preds).
    eos_bias overrides b_o[EOS] (e.g. +-inf to pin lengths); forced = a token sequence fed as
    y instead of the decoder's own choice (teacher forcing)."""
    H, D = int(cfg["hidden"]), a.shape[1]
    max_len, pad, bos, eos = cfg["max_len"], cfg["pad"], cfg["bos"], cfg["eos"]
    abar = _r(a.mean(axis=0), mode)
    h = np.tanh(P["init.w"][:H] @ abar + P["init.b"][:H])
    c = np.tanh(P["init.w"][H:] @ abar + P["init.b"][H:])
    b_o = P["out.b"].copy()
    if eos_bias is not None:
        b_o[eos] = eos_bias
    out = np.full(max_len, pad, dtype=np.int64)
    top1 = np.full(max_len, np.nan)
    preds = []
    done = False
    length = max_len
    y = bos
    for t in range(max_len):
        if done:
            out[t] = pad                                      # constant assignment (Sec. 5.4)
            continue
        q = P["att.w"] @ _r(h, mode) + P["att.b"]
        alpha = _softmax(a @ q / math.sqrt(D))
        z = alpha @ a
        u = np.concatenate([P["emb"][y], _r(z, mode), _r(h, mode)])
        gates = P["lstm.w"] @ u + P["lstm.b"]
        i_, f_ = sigmoid(gates[:H]), sigmoid(gates[H:2 * H])
        g_, o_ = np.tanh(gates[2 * H:3 * H]), sigmoid(gates[3 * H:])
        c = f_ * c + i_ * g_
        h = o_ * np.tanh(c)
        z_out = P["out.w"] @ _r(h, mode) + b_o
        tok = int(np.argmax(z_out))                           # lowest index on ties (R11)
        srt = np.partition(z_out, -2)[-2:]
        preds.append(("token", (srt[1] - srt[0]) / max(1.0, abs(srt[1])), 0.0))
        out[t] = tok
        top1[t] = z_out[tok]
        y = tok if forced is None else int(forced[t])
        if y == eos:                                          # the If node on the output token
            done = True
            length = t + 1
    return out, length, top1, preds


def caption(x, P, cfg, mode="mirror", **kw):
    """Encoder + decoder for one image."""
    return decode(encode(x, P, mode), P, cfg, mode, **kw)


def prepare_caption(W: dict) -> dict:
    return prg.prepare(W)
