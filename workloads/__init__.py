"""Seeded synthetic workloads shared by the CUDA path and the oracle.

This module is the ONLY code both sides use.  It holds no arithmetic of the
method (no layer, predicate, compaction or scatter); it only draws numbers:

* network inputs (images, MLP vectors) as a pure function of
  (seed, global sample index, element index), so any subset can be
  regenerated independently (SURVEY.md §8(d) "Seeds");
* random-init weights of the five architectures (He-normal trunks, N(0,1/C)
  heads/gates), rounded once to bf16 (RNE) -- the weight file both sides read;
* application of frozen calibration constants (workloads/calib/*.json, written
  by the committed script ``oracle/calibrate.py``, which calls only oracle/).

Recipes are stated in DESIGN.md §3 ("Input recipe").
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# Listing 2: the host program's Normalize constants.
IMAGENET_MEAN = np.array([0.485, 0.456, 0.406], dtype=np.float32)
IMAGENET_STD = np.array([0.229, 0.224, 0.225], dtype=np.float32)

WEIGHT_SEED = 0
INPUT_SEED = 1
CALIB_SEED = 2
ORACLE_SUBSET_SEED = 3


# ----------------------------------------------------------------------------
# bf16 storage helpers (round-to-nearest-even of fp32 bit patterns).
# ----------------------------------------------------------------------------
def f32_to_bf16_bits(a) -> np.ndarray:
    """fp32 -> bf16 bit pattern (uint16), round to nearest, ties to even."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16).astype(np.uint16)
    # NaN stays NaN (not produced by the generators, guarded anyway)
    nan = np.isnan(a)
    if nan.any():
        r[nan] = 0x7FC0
    return r


def bf16_bits_to_f32(b) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32)


# ----------------------------------------------------------------------------
# Counter-based uniform generator: splitmix64 finaliser of (seed, sample, elem).
# ----------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_uniform(seed: int, sample: np.ndarray, elem: np.ndarray, stream: int = 0) -> np.ndarray:
    """u in [0,1) with 24 random bits: top 24 bits of splitmix64(key)/2^24."""
    with np.errstate(over="ignore"):
        key = (np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)) ^ (
            np.asarray(sample, dtype=np.uint64) * np.uint64(0x100000001B3)
            + np.asarray(elem, dtype=np.uint64) * np.uint64(0x9E3779B1)
            + np.uint64(stream) * np.uint64(0xA24BAED4963EE407))
    z = _splitmix64(key)
    return ((z >> np.uint64(40)).astype(np.float64) / float(1 << 24))


def _per_sample_normals(seed: int, idx: np.ndarray, n: int, stream: int) -> np.ndarray:
    """Box-Muller normals, shape [len(idx), n], from counter uniforms."""
    e = np.arange(n, dtype=np.uint64)[None, :]
    s = idx.astype(np.uint64)[:, None]
    u1 = counter_uniform(seed, s, 2 * e, stream)
    u2 = counter_uniform(seed, s, 2 * e + np.uint64(1), stream)
    u1 = np.maximum(u1, 1.0 / (1 << 25))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


def image_inputs(seed: int, start: int, count: int, hw: int = 32, idx=None) -> np.ndarray:
    """Normalized fp32 NHWC images [count, hw, hw, 3] (SURVEY §8(d) inputs).

    u ~ U[0,1) per pixel, per-sample contrast g = exp(0.5 N(0,1)), per-sample
    per-channel brightness b_c ~ N(0, 0.5^2);  p = 0.5 + g (u - 0.5) + 0.25 b_c;
    x = (p - mean_c) / std_c with Listing 2's constants.
    All per-pixel arithmetic in fp32, in this exact op order.
    """
    if idx is None:
        idx = np.arange(start, start + count, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    n = len(idx)
    nrm = _per_sample_normals(seed, idx, 4, stream=7)
    gamma = np.exp(0.5 * nrm[:, 0]).astype(np.float32)
    beta = (0.5 * nrm[:, 1:4]).astype(np.float32)
    elem = np.arange(hw * hw * 3, dtype=np.uint64)[None, :]
    u = counter_uniform(seed, idx.astype(np.uint64)[:, None], elem).astype(np.float32)
    u = u.reshape(n, hw, hw, 3)
    p = np.float32(0.5) + gamma[:, None, None, None] * (u - np.float32(0.5))
    p = p + np.float32(0.25) * beta[:, None, None, :]
    x = (p - IMAGENET_MEAN) / IMAGENET_STD
    return np.ascontiguousarray(x.astype(np.float32))


def mlp_inputs(seed: int, start: int, count: int, dim: int = 64, idx=None) -> np.ndarray:
    """fp32 [count, dim], x ~ N(0,1) (config 1: 'random fp32 inputs')."""
    if idx is None:
        idx = np.arange(start, start + count, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    return _per_sample_normals(seed, idx, dim, stream=3).astype(np.float32)


# ----------------------------------------------------------------------------
# Architectures (parameter shapes only) and seeded random-init weights.
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class ResNetCifarSpec:
    blocks_per_stage: int          # 9 -> ResNet-56, 6 -> ResNet-38
    widths: tuple = (16, 32, 64)

    @property
    def n_blocks(self):
        return 3 * self.blocks_per_stage

    def block_io(self, i: int):
        """1-based block i -> (c_in, c_out, stride, hw_in)."""
        s = (i - 1) // self.blocks_per_stage
        first = (i - 1) % self.blocks_per_stage == 0
        c_out = self.widths[s]
        if s > 0 and first:
            return self.widths[s - 1], c_out, 2, 32 >> (s - 1)
        return c_out, c_out, 1, 32 >> s


R56 = ResNetCifarSpec(9)
R38 = ResNetCifarSpec(6)
SDN_IC_AFTER = (5, 11, 16, 22)          # SURVEY §8(c) reading 4
SKIP_GATED = tuple(range(2, 19))        # reading 7: blocks 2..18 gated
NUM_CLASSES = 10
EXIT_TAU = 0.9                          # config 1 value, reused


class _Rng:
    """One independent PCG64 stream per tensor, in a fixed registration order."""

    def __init__(self, seed):
        self.seed = seed
        self.k = 0

    def next(self):
        self.k += 1
        return np.random.default_rng([self.seed, self.k])


def _he_conv(rng, co, k, ci, scale=1.0):
    std = math.sqrt(2.0 / (k * k * ci)) * scale
    return (rng.standard_normal((co, k, k, ci)) * std).astype(np.float32)


def _bias(rng, n, amp=0.05):
    return rng.uniform(-amp, amp, size=(n,)).astype(np.float32)


def _bf16(a):
    return f32_to_bf16_bits(a)


def load_calib(name: str):
    path = os.path.join(HERE, "calib", f"{name}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


def mlp_weights(seed: int = WEIGHT_SEED, head_scale: float = 4.0) -> dict:
    """Config 1: 3 dense blocks 64->64 ReLU, heads 64->10 after blocks 1,2 and final."""
    rng = _Rng(seed)
    W = {}
    for k in range(3):
        W[f"fc{k}.w"] = _bf16(rng.next().standard_normal((64, 64)) * math.sqrt(2.0 / 64))
        W[f"fc{k}.b"] = _bias(rng.next(), 64, 0.1)
    for k in range(3):
        W[f"head{k}.w"] = _bf16(rng.next().standard_normal((10, 64)) * (head_scale / 8.0))
        W[f"head{k}.b"] = _bias(rng.next(), 10, 0.1)
    return W


def resnet_cifar_trunk(spec: ResNetCifarSpec, seed: int) -> dict:
    """Stem 3->16 + basic blocks; conv2 of each block scaled by 1/sqrt(n_blocks)."""
    rng = _Rng(seed)
    W = {}
    W["stem.w"] = _bf16(_he_conv(rng.next(), 16, 3, 3))
    W["stem.b"] = _bias(rng.next(), 16)
    for i in range(1, spec.n_blocks + 1):
        ci, co, _, _ = spec.block_io(i)
        W[f"b{i}.c1.w"] = _bf16(_he_conv(rng.next(), co, 3, ci))
        W[f"b{i}.c1.b"] = _bias(rng.next(), co)
        W[f"b{i}.c2.w"] = _bf16(_he_conv(rng.next(), co, 3, co, 1.0 / math.sqrt(spec.n_blocks)))
        W[f"b{i}.c2.b"] = _bias(rng.next(), co)
    return W, rng


def _centered_head(H_raw: np.ndarray, scale: float, mu: np.ndarray):
    """w = bf16(scale * H_raw); b = -(w . mu) so logits = w (g - mu)."""
    w = _bf16(scale * H_raw)
    wf = bf16_bits_to_f32(w).astype(np.float64)
    b = (-(wf @ np.asarray(mu, dtype=np.float64))).astype(np.float32)
    return w, b


def sdn_r56_raw_heads(seed: int = WEIGHT_SEED) -> dict:
    """Raw (uncalibrated) IC and final head directions H ~ N(0, 1/C)."""
    rng = np.random.default_rng([seed, 1000])
    out = {}
    for k, blk in enumerate(SDN_IC_AFTER):
        c = R56.block_io(blk)[1]
        out[f"ic{k}"] = rng.standard_normal((NUM_CLASSES, c)) / math.sqrt(c)
    out["final"] = rng.standard_normal((NUM_CLASSES, 64)) / math.sqrt(64)
    return out


def sdn_r56_weights(seed: int = WEIGHT_SEED, calib=None) -> dict:
    """Config 2: ShallowDeep-style ResNet-56, ICs after blocks 5, 11, 16, 22."""
    W, _ = resnet_cifar_trunk(R56, seed)
    if calib is None:
        calib = load_calib("cfg2")
    raw = sdn_r56_raw_heads(seed)
    for name, H in raw.items():
        c = H.shape[1]
        if calib is not None:
            scale, mu = calib[name]["scale"], np.array(calib[name]["mu"])
        else:  # uncalibrated default (used only by the calibration script itself)
            scale, mu = 1.0, np.zeros(c)
        W[f"{name}.w"], W[f"{name}.b"] = _centered_head(H, scale, mu)
    W["tau"] = np.float32(EXIT_TAU)
    return W


def skipnet_r38_raw_gates(seed: int = WEIGHT_SEED) -> dict:
    rng = np.random.default_rng([seed, 2000])
    out = {}
    for i in SKIP_GATED:
        c = R38.block_io(i)[0]          # the gate sees the block INPUT (Listing 3)
        out[f"gate{i}"] = rng.standard_normal((1, c)) / math.sqrt(c)
    out["final"] = rng.standard_normal((NUM_CLASSES, 64)) / math.sqrt(64)
    return out


def skipnet_r38_weights(seed: int = WEIGHT_SEED, calib=None) -> dict:
    """Config 3: SkipNet-style ResNet-38 with 17 feed-forward gates (blocks 2..18)."""
    W, _ = resnet_cifar_trunk(R38, seed)
    if calib is None:
        calib = load_calib("cfg3")
    raw = skipnet_r38_raw_gates(seed)
    for i in SKIP_GATED:
        g = raw[f"gate{i}"]
        if calib is not None:
            s, a = calib[f"gate{i}"]["scale"], calib[f"gate{i}"]["median"]
        else:
            s, a = 1.0, 0.0
        W[f"gate{i}.w"] = _bf16(s * g)
        W[f"gate{i}.b"] = np.array([-s * a], dtype=np.float32)
    fin = raw["final"]
    mu = np.array(calib["final"]["mu"]) if calib is not None else np.zeros(64)
    W["final.w"], W["final.b"] = _centered_head(fin, 4.0, mu)
    W["thr"] = np.float32(0.5)
    return W


# ----------------------------------------------------------------------------
# SkipNet with the recurrent gate (Table 3 ID 5 "ResNet38 + RNN"; reading R19):
# the config-3 trunk, per-gate projections proj_i (C_i -> RNN_IN, N(0, 1/C_i), bf16) feeding one
# shared LSTM cell (hidden RNN_HIDDEN, torch.nn.LSTMCell's U(-1/sqrt(H), 1/sqrt(H)) init, fp32),
# and a raw output vector w_out ~ N(0, 1/H); per-gate calibration (oracle/calibrate.py) gives
# out_i.w = s_i w_out, out_i.b = -s_i a_i (a_i = median, s_i = 2/std of the raw w_out . h).
# ----------------------------------------------------------------------------
RNN_IN = 10
RNN_HIDDEN = 10


def skipnet_rnn_r38_raw(seed: int = WEIGHT_SEED) -> dict:
    rng = np.random.default_rng([seed, 3000])
    out = {}
    for i in SKIP_GATED:
        c = R38.block_io(i)[0]
        out[f"proj{i}.w"] = rng.standard_normal((RNN_IN, c)) / math.sqrt(c)
        out[f"proj{i}.b"] = rng.uniform(-0.05, 0.05, RNN_IN)
    k = 1.0 / math.sqrt(RNN_HIDDEN)
    H4 = 4 * RNN_HIDDEN
    out["rnn.w_ih"] = rng.uniform(-k, k, (H4, RNN_IN))
    out["rnn.w_hh"] = rng.uniform(-k, k, (H4, RNN_HIDDEN))
    out["rnn.b_ih"] = rng.uniform(-k, k, H4)
    out["rnn.b_hh"] = rng.uniform(-k, k, H4)
    out["w_out"] = rng.standard_normal(RNN_HIDDEN) / math.sqrt(RNN_HIDDEN)
    out["final"] = rng.standard_normal((NUM_CLASSES, 64)) / math.sqrt(64)
    return out


def skipnet_rnn_r38_weights(seed: int = WEIGHT_SEED, calib=None) -> dict:
    """SkipNet-style ResNet-38 with 17 recurrent (LSTM) gates on blocks 2..18."""
    W, _ = resnet_cifar_trunk(R38, seed)
    if calib is None:
        calib = load_calib("cfg3r")
    raw = skipnet_rnn_r38_raw(seed)
    for i in SKIP_GATED:
        W[f"proj{i}.w"] = _bf16(raw[f"proj{i}.w"])
        W[f"proj{i}.b"] = raw[f"proj{i}.b"].astype(np.float32)
        s, a = (calib[f"gate{i}"]["scale"], calib[f"gate{i}"]["median"]) if calib is not None else (1.0, 0.0)
        W[f"out{i}.w"] = (s * raw["w_out"]).astype(np.float32)
        W[f"out{i}.b"] = np.array([-s * a], dtype=np.float32)
    for k in ("rnn.w_ih", "rnn.w_hh", "rnn.b_ih", "rnn.b_hh"):
        W[k] = raw[k].astype(np.float32)
    W["rnn.n_in"] = np.int32(RNN_IN)
    W["rnn.hidden"] = np.int32(RNN_HIDDEN)
    fin = raw["final"]
    mu = np.array(calib["final"]["mu"]) if calib is not None else np.zeros(64)
    W["final.w"], W["final.b"] = _centered_head(fin, 4.0, mu)
    W["thr"] = np.float32(0.5)
    return W


# ----------------------------------------------------------------------------
# Config 5: early-exit ResNet-50 v1.5 (torchvision topology, BN folded into biases).
# ----------------------------------------------------------------------------
R50_LAYERS = (3, 4, 6, 3)
R50_WIDTHS = (64, 128, 256, 512)
R50_EXIT_AFTER_STAGE = (1, 2, 3)          # SURVEY §8(c) reading R6: exits after stages 1, 2, 3 + final
R50_CLASSES = 1000


def r50_blocks():
    """[(stage, block, c_in, width, c_out, stride)] in program order."""
    out = []
    c_in = 64
    for s, (n, w) in enumerate(zip(R50_LAYERS, R50_WIDTHS)):
        for b in range(n):
            stride = 2 if (b == 0 and s > 0) else 1
            out.append((s + 1, b, c_in, w, 4 * w, stride))
            c_in = 4 * w
    return out


def r50_raw_heads(seed: int = WEIGHT_SEED) -> dict:
    rng = np.random.default_rng([seed, 5000])
    out = {}
    for k, st in enumerate(R50_EXIT_AFTER_STAGE):
        c = 4 * R50_WIDTHS[st - 1]
        out[f"ic{k}"] = rng.standard_normal((R50_CLASSES, c)) / math.sqrt(c)
    out["final"] = rng.standard_normal((R50_CLASSES, 2048)) / math.sqrt(2048)
    return out


def resnet50_ee_weights(seed: int = WEIGHT_SEED, calib=None) -> dict:
    """Config 5: early-exit ResNet-50.  Conv weights [Co][k][k][Ci] bf16; conv3 of every
    bottleneck scaled by 1/sqrt(16) (16 residual blocks) to keep the stream bounded."""
    rng = _Rng(seed + 50)
    W = {}
    W["stem.w"] = _bf16(_he_conv(rng.next(), 64, 7, 3))
    W["stem.b"] = _bias(rng.next(), 64)
    for (s, b, ci, w, co, stride) in r50_blocks():
        p = f"s{s}b{b}"
        W[f"{p}.c1.w"] = _bf16(_he_conv(rng.next(), w, 1, ci))
        W[f"{p}.c1.b"] = _bias(rng.next(), w)
        W[f"{p}.c2.w"] = _bf16(_he_conv(rng.next(), w, 3, w))
        W[f"{p}.c2.b"] = _bias(rng.next(), w)
        W[f"{p}.c3.w"] = _bf16(_he_conv(rng.next(), co, 1, w, 1.0 / math.sqrt(16)))
        W[f"{p}.c3.b"] = _bias(rng.next(), co)
        if b == 0:
            W[f"{p}.proj.w"] = _bf16(_he_conv(rng.next(), co, 1, ci))
            W[f"{p}.proj.b"] = _bias(rng.next(), co)
    if calib is None:
        calib = load_calib("cfg5")
    raw = r50_raw_heads(seed)
    for name, H in raw.items():
        c = H.shape[1]
        if calib is not None:
            scale, mu = calib[name]["scale"], np.array(calib[name]["mu"])
        else:
            scale, mu = 1.0, np.zeros(c)
        W[f"{name}.w"], W[f"{name}.b"] = _centered_head(H, scale, mu)
    W["tau"] = np.float32(EXIT_TAU)
    return W


def image_inputs_torch(seed: int, start: int, count: int, hw: int, device="cuda"):
    """The SAME counter-based generator as image_inputs(), evaluated with torch on a
    device (for config 5's 39.5 GB of inputs).  Integer hash: int64 with wrap-around
    and masked logical shifts; per-pixel float math: the identical sequence of fp32
    IEEE operations (separate kernels, no fused multiply-add), so values are
    bit-identical to the numpy path (tests/test_workloads.py checks this).
    Per-sample gamma/beta come from the numpy path (4 transcendental draws per sample)."""
    import torch
    idx = np.arange(start, start + count, dtype=np.int64)
    nrm = _per_sample_normals(seed, idx, 4, stream=7)
    gamma = torch.from_numpy(np.exp(0.5 * nrm[:, 0]).astype(np.float32)).to(device)
    beta = torch.from_numpy((0.5 * nrm[:, 1:4]).astype(np.float32)).to(device)
    mean = torch.from_numpy(IMAGENET_MEAN).to(device)
    std = torch.from_numpy(IMAGENET_STD).to(device)

    def u64(v):
        v = int(v) & 0xFFFFFFFFFFFFFFFF
        return v - (1 << 64) if v >= (1 << 63) else v

    def lsr(x, k):                         # logical shift right of int64 bit patterns
        return (x >> k) & ((1 << (64 - k)) - 1)

    n_el = hw * hw * 3
    out = torch.empty((count, hw, hw, 3), dtype=torch.float32, device=device)
    elem = torch.arange(n_el, dtype=torch.int64, device=device)[None, :]
    C2, C3 = u64(0x100000001B3), u64(0x9E3779B1)
    seed_term = u64(seed * 0xD1B54A32D192ED03)
    blk = max(1, (1 << 25) // n_el)                     # samples per vectorised block
    half = torch.tensor(0.5, dtype=torch.float32, device=device)
    quarter = torch.tensor(0.25, dtype=torch.float32, device=device)
    for i0 in range(0, count, blk):
        i1 = min(count, i0 + blk)
        smp = torch.arange(start + i0, start + i1, dtype=torch.int64, device=device)[:, None]
        key = (smp * C2 + elem * C3) ^ seed_term          # stream 0
        z = key + u64(0x9E3779B97F4A7C15)
        z = (z ^ lsr(z, 30)) * u64(0xBF58476D1CE4E5B9)
        z = (z ^ lsr(z, 27)) * u64(0x94D049BB133111EB)
        z = z ^ lsr(z, 31)
        u = (lsr(z, 40).to(torch.float32) / float(1 << 24)).view(i1 - i0, hw, hw, 3)
        p = half + gamma[i0:i1, None, None, None] * (u - half)
        p = p + quarter * beta[i0:i1, None, None, :]
        out[i0:i1] = (p - mean) / std
    return out


# ----------------------------------------------------------------------------
# Config 4: 6+6 post-LN Transformer seq2seq, greedy decode with an EOS/length guard.
# ----------------------------------------------------------------------------
S2S = dict(vocab=32000, d=512, heads=8, d_ff=2048, enc_layers=6, dec_layers=6, src_len=64, max_len=64,
           pad=0, bos=1, eos=2, beta=16.0)


def token_inputs(seed: int, start: int, count: int, src_len: int = 64, vocab: int = 32000) -> np.ndarray:
    """int32 [count, src_len], tokens uniform on [3, vocab) (PAD/BOS/EOS never appear)."""
    idx = np.arange(start, start + count, dtype=np.uint64)[:, None]
    e = np.arange(src_len, dtype=np.uint64)[None, :]
    u = counter_uniform(seed, idx, e, stream=11)
    return (3 + np.floor(u * (vocab - 3))).astype(np.int32)


def seq2seq_weights(seed: int = WEIGHT_SEED) -> dict:
    """Embeddings N(0,1); linears N(0, 1/fan_in) (bf16); biases U(-0.05, 0.05);
    LayerNorm gamma = 1 + U(-0.1, 0.1), beta = U(-0.05, 0.05) (fp32).
    Length table LEN[v] = U{0..63} + 0.5 (fp32): with beta = 16 the EOS bias
    beta*(t+1-LEN[src[0]]) makes a sequence end after ~LEN+1 tokens."""
    c = S2S
    rng = _Rng(seed + 40)
    d, f, V = c["d"], c["d_ff"], c["vocab"]

    def lin(n_out, n_in):
        return _bf16(rng.next().standard_normal((n_out, n_in)) / math.sqrt(n_in))

    def ln():
        r = rng.next()
        return (1.0 + r.uniform(-0.1, 0.1, d)).astype(np.float32), r.uniform(-0.05, 0.05, d).astype(np.float32)

    W = {"src_emb": _bf16(rng.next().standard_normal((V, d))), "tgt_emb": _bf16(rng.next().standard_normal((V, d)))}
    for l in range(c["enc_layers"]):
        p = f"enc{l}"
        W[p + ".wqkv"], W[p + ".bqkv"] = lin(3 * d, d), _bias(rng.next(), 3 * d)
        W[p + ".wo"], W[p + ".bo"] = lin(d, d), _bias(rng.next(), d)
        W[p + ".ln1.g"], W[p + ".ln1.b"] = ln()
        W[p + ".w1"], W[p + ".b1"] = lin(f, d), _bias(rng.next(), f)
        W[p + ".w2"], W[p + ".b2"] = lin(d, f), _bias(rng.next(), d)
        W[p + ".ln2.g"], W[p + ".ln2.b"] = ln()
    for l in range(c["dec_layers"]):
        p = f"dec{l}"
        W[p + ".wqkv"], W[p + ".bqkv"] = lin(3 * d, d), _bias(rng.next(), 3 * d)
        W[p + ".wo"], W[p + ".bo"] = lin(d, d), _bias(rng.next(), d)
        W[p + ".ln1.g"], W[p + ".ln1.b"] = ln()
        W[p + ".wq2"], W[p + ".bq2"] = lin(d, d), _bias(rng.next(), d)
        W[p + ".wkv2"], W[p + ".bkv2"] = lin(2 * d, d), _bias(rng.next(), 2 * d)
        W[p + ".wo2"], W[p + ".bo2"] = lin(d, d), _bias(rng.next(), d)
        W[p + ".ln2.g"], W[p + ".ln2.b"] = ln()
        W[p + ".w1"], W[p + ".b1"] = lin(f, d), _bias(rng.next(), f)
        W[p + ".w2"], W[p + ".b2"] = lin(d, f), _bias(rng.next(), d)
        W[p + ".ln3.g"], W[p + ".ln3.b"] = ln()
    W["lm.w"], W["lm.b"] = lin(V, d), _bias(rng.next(), V)
    W["len_table"] = (rng.next().integers(0, c["max_len"], V) + 0.5).astype(np.float32)
    W["beta"] = np.float32(c["beta"])
    return W


# ----------------------------------------------------------------------------
# Image-captioning En-Decoder (reading R20): CIFAR ResNet-38 trunk encoder (its
# 8x8x64 output = 64 annotation vectors), soft-attention LSTM decoder (hidden 256, word
# embeddings 256, vocabulary 4096), greedy, EOS / max-len 32 guard.  EOS output bias calibrated
# (oracle/calibrate.py cfg4c) to a mean caption length of ~12.
# ----------------------------------------------------------------------------
CAP = dict(vocab=4096, emb=256, hidden=256, max_len=32, pad=0, bos=1, eos=2, L=64, D=64)
CAP_SEED_OFFSET = 6000


def caption_weights(seed: int = WEIGHT_SEED, calib=None) -> dict:
    W, _ = resnet_cifar_trunk(R38, seed + CAP_SEED_OFFSET)
    c = CAP
    V, E, H, D = c["vocab"], c["emb"], c["hidden"], c["D"]
    rng = _Rng([seed, 7000])
    k = 1.0 / math.sqrt(H)
    W["init.w"] = _bf16(rng.next().standard_normal((2 * H, D)) / math.sqrt(D) * 2.0)
    W["init.b"] = rng.next().uniform(-0.1, 0.1, 2 * H).astype(np.float32)
    W["att.w"] = _bf16(rng.next().standard_normal((D, H)) / math.sqrt(H) * 4.0)
    W["att.b"] = rng.next().uniform(-0.1, 0.1, D).astype(np.float32)
    W["emb"] = _bf16(rng.next().standard_normal((V, E)))
    W["lstm.w"] = _bf16(rng.next().uniform(-k, k, (4 * H, E + D + H)))
    W["lstm.b"] = rng.next().uniform(-2 * k, 2 * k, 4 * H).astype(np.float32)
    W["out.w"] = _bf16(rng.next().standard_normal((V, H)) / math.sqrt(H) * 8.0)
    W["out.b"] = rng.next().uniform(-0.1, 0.1, V).astype(np.float32)
    if calib is None:
        calib = load_calib("cfg4c")
    if calib is not None:
        W["out.b"][c["eos"]] = np.float32(calib["eos_bias"])
    return W


CONFIGS = {
    1: dict(name="mlp_ee", batch=32, desc="tiny early-exit MLP: 3 blocks width 64, 2 exit heads, tau 0.9, batch 32"),
    2: dict(name="sdn_resnet56", batch=4096, desc="ShallowDeep-style early-exit ResNet-56, 32x32x3, batch 4096, 4 ICs"),
    3: dict(name="skipnet_resnet38", batch=8192, desc="SkipNet-style gated ResNet-38, 32x32x3, batch 8192, 17 gates"),
    4: dict(name="seq2seq", batch=1024, desc="6+6 Transformer d=512 greedy decode, EOS/max-len 64 guard, batch 1024"),
    5: dict(name="resnet50_ee", batch=65536, desc="early-exit ResNet-50, 224x224x3, batch 65536, exits after stages 1-3"),
}
