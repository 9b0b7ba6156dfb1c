"""Config 4: greedy seq2seq decoding with a per-sequence EOS / max-length loop guard.

TEST INFRASTRUCTURE -- see oracle/__init__.py.

The generative DyNN of the paper's study (AttentionNet = Vaswani Transformer,
PAPER.md L323; the `If` node "leverages the output token value to determine
whether the translation should be completed", L265), with the input-independent
loop bound the paper prescribes ("a flag that enforces a constant maximum number
of iterations", L267-268).  Run one sequence at a time, with the loop and the
`if` as written:

    m = Encoder(src);  y = [BOS];  done = False;  L = max_len
    for t in 0..max_len-1:
        if done: out[t] = PAD; continue                       # constant assignment
        z = LMhead(Decoder(y, m)[-1]);  z[EOS] += beta*(t+1 - LEN[src[0]])
        tok = argmax(z) (lowest index on ties);  out[t] = tok;  y.append(tok)
        if tok == EOS: done = True; L = t+1
    return out, L

Readings (R9/R10): post-LN layers (norm_first=False) without an extra final
LayerNorm, ReLU FFN, 8 heads x 64, sinusoidal PE, embeddings x sqrt(d), separate
source/target embeddings, untied LM head with bias, PAD=0 BOS=1 EOS=2, no source
padding, EOS counted in the length, PAD after done, length 64 when EOS never wins.
Decoding is incremental (cached K/V of earlier positions), which equals recomputing
the whole prefix for a causal decoder (tests pin it against torch's full recompute).

Modes as in programs.py: 'mirror' rounds every tensor-core operand and every
bf16-stored tensor (q/k/v, K/V caches, attention outputs, FFN hidden, the encoder's
attention probabilities P) to bf16,
keeps the residual stream, LayerNorm, softmax and logits unrounded; 'exact' rounds
nothing.  Matrix products use numpy's matmul (fp64) as the library primitive.
"""
from __future__ import annotations

import math

import numpy as np

from .core import round_bf16


def _r(v, mode):
    return round_bf16(v) if mode == "mirror" else v


def positional_encoding(n: int, d: int) -> np.ndarray:
    """PE[pos, 2i] = sin(pos / 10000^(2i/d)), PE[pos, 2i+1] = cos(pos / 10000^(2i/d))."""
    pos = np.arange(n, dtype=np.float64)[:, None]
    i2 = np.arange(0, d, 2, dtype=np.float64)[None, :]
    ang = pos / np.power(10000.0, i2 / d)
    pe = np.zeros((n, d))
    pe[:, 0::2] = np.sin(ang)
    pe[:, 1::2] = np.cos(ang)
    return pe


def layer_norm(x, g, b, eps=1e-5):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def _softmax_rows(s):
    s = s - s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    return e / e.sum(axis=-1, keepdims=True)


def attention(q, k, v, heads, mode, p_operand=False):
    """Multi-head scaled dot-product attention: q [nq, d], k/v [nk, d] (already bf16 in mirror).
    p_operand: the probabilities P are a tensor-core operand (the encoder's P x V runs on
    tcgen05), so mirror mode rounds P = softmax(.) to bf16 before P @ V (reading R18)."""
    nq, d = q.shape
    dh = d // heads
    out = np.empty((nq, d))
    for h in range(heads):
        sl = slice(h * dh, (h + 1) * dh)
        p = _softmax_rows(q[:, sl] @ k[:, sl].T / math.sqrt(dh))
        if p_operand:
            p = _r(p, mode)
        out[:, sl] = p @ v[:, sl]
    return _r(out, mode)                      # stored bf16: the out-projection's operand


def _linear(x, P, w, b, mode):
    return _r(x, mode) @ P[w].T + P[b]


def encoder(src, P, cfg, mode):
    d, H = cfg["d"], cfg["heads"]
    x = P["src_emb"][src] * math.sqrt(d) + positional_encoding(len(src), d)
    for l in range(cfg["enc_layers"]):
        p = f"enc{l}"
        qkv = _r(_linear(x, P, p + ".wqkv", p + ".bqkv", mode), mode)
        a = attention(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], H, mode, p_operand=True)
        x = layer_norm(_linear(a, P, p + ".wo", p + ".bo", mode) + x, P[p + ".ln1.g"], P[p + ".ln1.b"])
        h = _r(np.maximum(_linear(x, P, p + ".w1", p + ".b1", mode), 0.0), mode)
        x = layer_norm(_linear(h, P, p + ".w2", p + ".b2", mode) + x, P[p + ".ln2.g"], P[p + ".ln2.b"])
    return x


def greedy_decode(src, P, cfg, mode="mirror", eos_bias=None, max_steps=None, forced=None):
    """One sequence.  Returns (tokens [max_len] int, length, top1 logit per step [max_len]
    (nan after done), step-0 logits [V], preds).  eos_bias(t, src) overrides the length
    guard bias (e.g. -inf to force fixed-length decoding).

    forced (teacher forcing, SURVEY 8(c) "the oracle recomputes each step from the GPU's own
    prefix"): a token sequence fed as the decoder input instead of the oracle's own choice;
    out[t] is still the oracle's argmax at step t, the loop stops after forced[t] == EOS."""
    d, H, L = cfg["d"], cfg["heads"], cfg["max_len"]
    pad, bos, eos = cfg["pad"], cfg["bos"], cfg["eos"]
    m = encoder(src, P, cfg, mode)
    cross = []
    for l in range(cfg["dec_layers"]):
        p = f"dec{l}"
        kv = _r(_linear(m, P, p + ".wkv2", p + ".bkv2", mode), mode)
        cross.append((kv[:, :d], kv[:, d:]))
    kcache = [[] for _ in range(cfg["dec_layers"])]
    vcache = [[] for _ in range(cfg["dec_layers"])]
    pe = positional_encoding(L, d)
    out = np.full(L, pad, dtype=np.int64)
    top1 = np.full(L, np.nan)
    z0 = None
    preds = []
    done = False
    length = L
    tok_in = bos
    steps = L if max_steps is None else max_steps
    for t in range(steps):
        if done:
            out[t] = pad                                        # constant assignment (Sec. 5.4 strategy 2)
            continue
        x = (P["tgt_emb"][tok_in] * math.sqrt(d) + pe[t])[None, :]
        for l in range(cfg["dec_layers"]):
            p = f"dec{l}"
            qkv = _r(_linear(x, P, p + ".wqkv", p + ".bqkv", mode), mode)
            kcache[l].append(qkv[0, d:2 * d])
            vcache[l].append(qkv[0, 2 * d:])
            a = attention(qkv[:, :d], np.stack(kcache[l]), np.stack(vcache[l]), H, mode)
            x = layer_norm(_linear(a, P, p + ".wo", p + ".bo", mode) + x, P[p + ".ln1.g"], P[p + ".ln1.b"])
            q2 = _r(_linear(x, P, p + ".wq2", p + ".bq2", mode), mode)
            a2 = attention(q2, cross[l][0], cross[l][1], H, mode)
            x = layer_norm(_linear(a2, P, p + ".wo2", p + ".bo2", mode) + x, P[p + ".ln2.g"], P[p + ".ln2.b"])
            h = _r(np.maximum(_linear(x, P, p + ".w1", p + ".b1", mode), 0.0), mode)
            x = layer_norm(_linear(h, P, p + ".w2", p + ".b2", mode) + x, P[p + ".ln3.g"], P[p + ".ln3.b"])
        z = _linear(x, P, "lm.w", "lm.b", mode)[0]
        if eos_bias is None:
            z[eos] += float(P["beta"]) * (t + 1 - float(P["len_table"][src[0]]))
        else:
            z[eos] += eos_bias(t, src)
        if t == 0:
            z0 = z.copy()
        tok = int(np.argmax(z))                                 # lowest index on ties (reading R10)
        srt = np.partition(z, -2)[-2:]
        preds.append(("token", (srt[1] - srt[0]) / max(1.0, abs(srt[1])), 0.0))
        out[t] = tok
        top1[t] = z[tok]
        tok_in = tok if forced is None else int(forced[t])
        if tok_in == eos:                                          # the If node on the output token (L265)
            done = True
            length = t + 1
    return out, length, top1, z0, preds


def prepare_s2s(W: dict) -> dict:
    P = {}
    for k, v in W.items():
        v = np.asarray(v)
        P[k] = ((v.astype(np.uint32) << 16).view(np.float32).astype(np.float64) if v.dtype == np.uint16
                else v.astype(np.float64) if v.dtype != np.int32 else v)
    return P
