"""Pins of the CPU oracle against things other than itself (runs without a GPU).

Each test names what fixes the expected value: a closed form, a value printed
in the paper/spec (tests/golden/*.json, cited), a library routine the case
reduces to (torch fp64), or an independent brute-force re-implementation.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
import workloads as wl
from oracle import programs as prg
from oracle.metrics import delta, eta, in_band
from tests import torch_ref as TR

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------- layers
@pytest.mark.parametrize("H,C,Co,k,stride,pad", [
    (8, 3, 5, 3, 1, 1), (9, 4, 6, 3, 2, 1), (7, 8, 4, 1, 2, 0), (12, 3, 8, 7, 2, 3), (5, 16, 16, 3, 1, 1)])
def test_conv2d_is_torch_conv2d(H, C, Co, k, stride, pad):
    """Library special case: the oracle conv equals torch.nn.functional.conv2d in fp64."""
    rng = np.random.default_rng(H * 100 + k)
    x = rng.standard_normal((H, H + 1, C))
    w = rng.standard_normal((Co, k, k, C))
    b = rng.standard_normal(Co)
    y = O.conv2d(x, w, b, stride, pad)
    t = torch.nn.functional.conv2d(torch.tensor(x).permute(2, 0, 1)[None], torch.tensor(w).permute(0, 3, 1, 2),
                                   torch.tensor(b), stride=stride, padding=pad)[0].permute(1, 2, 0).numpy()
    assert y.shape == t.shape
    np.testing.assert_allclose(y, t, rtol=0, atol=1e-12)


def test_round_bf16_matches_torch_cast_and_ties():
    rng = np.random.default_rng(7)
    v32 = (rng.standard_normal(20000) * np.exp(rng.uniform(-20, 20, 20000))).astype(np.float32)
    ref = torch.tensor(v32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(O.round_bf16(v32.astype(np.float64)), ref)
    # hand ties (bf16: 8 significant bits, ulp(1) = 2^-7): ties go to the even significand
    assert O.round_bf16(1 + 2 ** -8) == 1.0
    assert O.round_bf16(1 + 3 * 2 ** -8) == 1 + 2 ** -6
    assert O.round_bf16(-(1 + 2 ** -8 + 2 ** -30)) == -(1 + 2 ** -7)
    assert O.round_bf16(0.0) == 0.0


def test_option_a_is_subsample_and_symmetric_channel_pad():
    rng = np.random.default_rng(1)
    h = rng.standard_normal((8, 8, 16))
    a = O.option_a(h, 32)
    t = TR.shortcut_a(torch.tensor(h).permute(2, 0, 1)[None], 32)[0].permute(1, 2, 0).numpy()
    np.testing.assert_array_equal(a, t)
    assert a.shape == (4, 4, 32) and np.all(a[:, :, :8] == 0) and np.all(a[:, :, 24:] == 0)


# ------------------------------------------------------------------ predicates
def test_exit_confidence_closed_form():
    g = _gold("exit_closed_form.json")
    for c in g["cases"]:
        z = np.zeros(g["K"])
        z[0] = c["b"]
        conf = O.max_softmax(z)
        assert conf == pytest.approx(c["conf"], rel=1e-14)
        assert (conf >= g["tau"]) == c["exits"]
    z = np.zeros(g["K"])
    z[0] = g["b_star"]
    assert O.max_softmax(z) == pytest.approx(0.9, abs=1e-15)
    # shift invariance of softmax: adding a constant changes nothing
    assert O.max_softmax(z + 123.0) == pytest.approx(O.max_softmax(z), rel=1e-14)


def test_softmax_symmetry_and_argmax_ties():
    g = _gold("softmax_symmetry.json")
    assert O.max_softmax([0.0, 0.0, 0.0]) == pytest.approx(g["softmax_zeros3_max"], rel=1e-15)
    assert O.argmax_lowest(g["argmax_case"]["z"]) == g["argmax_case"]["argmax"]
    assert O.argmax_lowest(g["argmax_tie"]["z"]) == g["argmax_tie"]["argmax"]


def test_gate_at_half_skips():
    """Reading R2: execute iff p > 0.5, so sigma(0) = 0.5 skips."""
    assert O.sigmoid(0.0) == 0.5
    assert not (O.sigmoid(0.0) > 0.5)
    assert O.sigmoid(1e-9) > 0.5
    # the slope: sigma(ln 3) = 3/4, sigma(-ln 3) = 1/4 (closed form 1/(1+e^-z))
    assert O.sigmoid(np.log(3.0)) == pytest.approx(0.75, abs=1e-15)
    assert O.sigmoid(-np.log(3.0)) == pytest.approx(0.25, abs=1e-15)


def test_metrics_golden():
    g = _gold("metrics.json")
    a = [np.arange(10.0), np.ones(3)]
    assert delta(a, a) == pytest.approx(g["delta_identical"], abs=1e-12)
    b = [np.arange(10.0), np.ones(3)]
    b[1] = b[1].copy()
    b[1][2] += 1e-5
    assert delta(b, a) == pytest.approx(g["delta_one_1e-5"], abs=1e-6)
    v = [0] * 1000
    c = [1] * 830 + [0] * 170
    assert eta(c, v) == pytest.approx(g["eta_830_of_1000"])
    # unequal-length generations are inconsistent (reading R15)
    assert eta([np.array([1, 2])], [np.array([1, 2, 3])]) == 1.0


# ------------------------------------------------------------------- config 1
def _mlp_bruteforce(x, W, mode, tau=0.9):
    """Independent fp64 NumPy implementation of the 3-block early-exit MLP."""
    def f(name):
        a = np.asarray(W[name])
        if a.dtype == np.uint16:
            a = (a.astype(np.uint32) << 16).view(np.float32)
        return a.astype(np.float64)

    def op(v):      # tensor-core operand rounding (both mirror modes)
        return O.round_bf16(v) if mode != "exact" else v

    def store(v):   # stored-activation rounding (all-bf16 storage only)
        return O.round_bf16(v) if mode == "mirror_bf16" else v

    h = torch.tensor(np.float32(x)).to(torch.bfloat16).double().numpy()
    outs = []
    for k in range(3):
        h = store(np.maximum(f(f"fc{k}.w").dot(op(h)) + f(f"fc{k}.b"), 0))
        z = f(f"head{k}.w").dot(h) + f(f"head{k}.b")
        e = np.exp(z - z.max())
        outs.append((z, (e / e.sum()).max()))
    for k in range(2):
        if outs[k][1] >= tau:
            return outs[k][0], k
    return outs[2][0], 2


@pytest.mark.parametrize("mode", ["mirror", "mirror_bf16", "exact"])
def test_mlp_matches_bruteforce(mode):
    W = wl.mlp_weights()
    X = wl.mlp_inputs(wl.INPUT_SEED, 0, 32)
    P = prg.prepare(W)
    L, path, preds = O.run_batch(O.mlp_ee, X, P, mode, threads=1)
    for i in range(32):
        z, p = _mlp_bruteforce(X[i], W, mode)
        assert path[i] == p
        np.testing.assert_allclose(L[i], z, rtol=0, atol=1e-12)
    assert np.bincount(path, minlength=3).sum() == 32


def test_mlp_degenerate_thresholds():
    """tau > 1: never exits (static net, final head); tau <= 1/K: everyone exits at head 0."""
    W = wl.mlp_weights()
    X = wl.mlp_inputs(wl.INPUT_SEED, 0, 16)
    P = prg.prepare(W)
    _, p_hi, _ = O.run_batch(O.mlp_ee, X, P, "exact", threads=1, tau=1.01)
    _, p_lo, _ = O.run_batch(O.mlp_ee, X, P, "exact", threads=1, tau=0.1)
    assert np.all(p_hi == 2) and np.all(p_lo == 0)


# ------------------------------------------------------------------- config 2
@pytest.fixture(scope="module")
def r56():
    return wl.sdn_r56_weights()


def test_sdn_never_exit_is_static_resnet56(r56):
    """tau > 1 => the dynamic program is the static ResNet-56 + final head (torch fp64)."""
    X = wl.image_inputs(wl.INPUT_SEED, 0, 2)
    P = prg.prepare(r56)
    for i in range(2):
        z, path, preds = O.sdn_resnet56(X[i], P, "exact", tau=1.5)
        assert path == 4 and len(preds) == 4
        ref = TR.head(TR.static_resnet(X[i], r56, 9), r56, "final").numpy()
        np.testing.assert_allclose(z, ref, rtol=1e-12, atol=1e-12)


def test_sdn_all_exit_at_ic1_is_prefix_net(r56):
    """tau <= 1/K => every sample exits at IC after block 5 with that head's logits."""
    X = wl.image_inputs(wl.INPUT_SEED, 5, 2)
    P = prg.prepare(r56)
    for i in range(2):
        z, path, preds = O.sdn_resnet56(X[i], P, "exact", tau=0.1)
        assert path == 0 and len(preds) == 1
        ref = TR.head(TR.static_resnet(X[i], r56, 9, upto=5), r56, "ic0").numpy()
        np.testing.assert_allclose(z, ref, rtol=1e-12, atol=1e-12)


def test_sdn_mirror_rounding_points(r56):
    """Rounding points (reading R13): mirror_bf16 stores bf16 everywhere; mirror
    (fp32 stream) rounds exactly the conv operands: a block equals the exact
    block applied to a bf16-rounded conv1 input with the unrounded shortcut."""
    X = wl.image_inputs(wl.INPUT_SEED, 0, 1)
    P = prg.prepare(r56)
    h = prg.stem(X[0], P, "mirror_bf16")
    assert np.array_equal(O.round_bf16(h), h)
    h2 = prg.basic_block(h, P, 1, 9, "mirror_bf16")
    assert np.array_equal(O.round_bf16(h2), h2)
    hs = prg.stem(X[0], P, "mirror")
    assert not np.array_equal(O.round_bf16(hs), hs)          # the stream is not rounded
    hm = prg.basic_block(hs, P, 1, 9, "mirror")
    t = O.round_bf16(O.relu(O.conv2d(O.round_bf16(hs), P["b1.c1.w"], P["b1.c1.b"], 1, 1)))
    ref = O.relu(O.conv2d(t, P["b1.c2.w"], P["b1.c2.b"], 1, 1) + hs)
    np.testing.assert_array_equal(hm, ref)
    he = prg.basic_block(prg.stem(X[0], P, "exact"), P, 1, 9, "exact")
    for v in (h2, hm):
        assert np.max(np.abs(he - v)) < 0.05 * np.max(np.abs(he))


def test_sdn_calibrated_exit_histogram(r56):
    """The calibration makes the dynamic path branch (each exit taken) on held-out inputs."""
    X = wl.image_inputs(wl.INPUT_SEED, 0, 48)
    P = prg.prepare(r56)
    _, path, preds = O.run_batch(O.sdn_resnet56, X, P, "mirror")
    h = np.bincount(path, minlength=5)
    assert h.sum() == 48 and np.count_nonzero(h) >= 4
    for p, pr in zip(path, preds):          # path word = number of predicates evaluated - 1 on exit
        assert len(pr) == min(p + 1, 4)


# ------------------------------------------------------------------- config 3
@pytest.fixture(scope="module")
def r38():
    return wl.skipnet_r38_weights()


def _forced_gates(W, pattern):
    W = dict(W)
    for i in wl.SKIP_GATED:
        W[f"gate{i}.b"] = np.array([1e9 if pattern(i) else -1e9], np.float32)
    return W


@pytest.mark.parametrize("name,pattern", [
    ("all_execute", lambda i: True), ("all_skip", lambda i: False), ("even_blocks", lambda i: i % 2 == 0)])
def test_skipnet_forced_gates_equal_static_composition(r38, name, pattern):
    """Gate bias +-inf reduces SkipNet to a fixed static network (Listing 3 semantics)."""
    W = _forced_gates(r38, pattern)
    P = prg.prepare(W)
    X = wl.image_inputs(wl.INPUT_SEED, 11, 1)
    z, mask, preds = O.skipnet_resnet38(X[0], P, "exact")
    execd = {1} | {i for i in wl.SKIP_GATED if pattern(i)}
    assert mask == sum(1 << (i - 2) for i in wl.SKIP_GATED if pattern(i))
    ref = TR.head(TR.static_resnet(X[0], W, 6, exec_blocks=execd), W, "final").numpy()
    np.testing.assert_allclose(z, ref, rtol=1e-12, atol=1e-12)
    assert len(preds) == 17


def test_skipnet_calibrated_gates_branch(r38):
    X = wl.image_inputs(wl.INPUT_SEED, 0, 24)
    P = prg.prepare(r38)
    _, mask, preds = O.run_batch(O.skipnet_resnet38, X, P, "mirror")
    bits = np.array([bin(int(m)).count("1") for m in mask])
    assert len(set(mask.tolist())) > 10          # many distinct paths (2^17 possible)
    assert 3 <= bits.mean() <= 14


def test_band_exclusion():
    assert in_band([("exit", 0.9004, 0.9)])
    assert not in_band([("exit", 0.902, 0.9), ("gate", 0.3, 0.5)])


# ------------------------------------------------------------------- config 5
def test_maxpool_is_torch_maxpool():
    rng = np.random.default_rng(3)
    h = rng.standard_normal((13, 12, 8))
    y = O.maxpool2d(h, 3, 2, 1)
    t = torch.nn.functional.max_pool2d(torch.tensor(h).permute(2, 0, 1)[None], 3, 2, 1)[0].permute(1, 2, 0).numpy()
    np.testing.assert_array_equal(y, t)


def _torchvision_r50(W):
    """torchvision's ResNet-50 (v1.5) with our weights; BatchNorm reduced to a pure bias
    (weight 1, running mean 0, var 1 - eps -> y = x + b up to one fp64 rounding)."""
    import torchvision
    m = torchvision.models.resnet50(weights=None).double().eval()

    def setc(conv, bn, name):
        w = np.asarray(W[name + ".w"])
        w = (w.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        conv.weight.data = torch.tensor(w).permute(0, 3, 1, 2).contiguous()
        bn.weight.data.fill_(1.0)
        bn.bias.data = torch.tensor(np.asarray(W[name + ".b"], np.float64))
        bn.running_mean.zero_()
        bn.running_var.fill_(1.0 - bn.eps)

    setc(m.conv1, m.bn1, "stem")
    for s, layer in enumerate([m.layer1, m.layer2, m.layer3, m.layer4], start=1):
        for b, blk in enumerate(layer):
            p = f"s{s}b{b}"
            setc(blk.conv1, blk.bn1, p + ".c1")
            setc(blk.conv2, blk.bn2, p + ".c2")
            setc(blk.conv3, blk.bn3, p + ".c3")
            if blk.downsample is not None:
                setc(blk.downsample[0], blk.downsample[1], p + ".proj")
    fw = np.asarray(W["final.w"])
    m.fc.weight.data = torch.tensor((fw.astype(np.uint32) << 16).view(np.float32).astype(np.float64))
    m.fc.bias.data = torch.tensor(np.asarray(W["final.b"], np.float64))
    return m


def test_resnet50_never_exit_is_torchvision_resnet50():
    """tau > 1: the early-exit ResNet-50 program is torchvision's resnet50 (the v1.5 topology:
    stride in the 3x3, 1x1 projection shortcuts, 3x3/2 max-pool) with BN folded -- library
    special case, fp64, on a 64x64 input (the topology is resolution independent)."""
    W = wl.resnet50_ee_weights()
    m = _torchvision_r50(W)
    P = prg.prepare(W)
    X = wl.image_inputs(wl.INPUT_SEED, 0, 1, hw=64)
    z, path, preds = O.resnet50_ee(X[0], P, "exact", tau=1.5)
    assert path == 3 and len(preds) == 3
    xt = torch.tensor(X[0]).to(torch.bfloat16).double().permute(2, 0, 1)[None]
    with torch.no_grad():
        ref = m(xt)[0].numpy()
    np.testing.assert_allclose(z, ref, rtol=1e-10, atol=1e-10)


def test_resnet50_exit_after_stage1_is_prefix():
    """tau <= 1/K: every sample exits after stage 1 with IC0's logits on GAP(layer1(stem))."""
    W = wl.resnet50_ee_weights()
    m = _torchvision_r50(W)
    P = prg.prepare(W)
    X = wl.image_inputs(wl.INPUT_SEED, 1, 1, hw=64)
    z, path, _ = O.resnet50_ee(X[0], P, "exact", tau=1e-4)
    assert path == 0
    xt = torch.tensor(X[0]).to(torch.bfloat16).double().permute(2, 0, 1)[None]
    with torch.no_grad():
        h = m.layer1(m.maxpool(m.relu(m.bn1(m.conv1(xt)))))
        g = h.mean(dim=(2, 3))[0].numpy()
    wf = prg._bf16_to_f64(W["ic0.w"])
    np.testing.assert_allclose(z, wf @ g + W["ic0.b"], rtol=1e-10, atol=1e-10)


# ------------------------------------------------------------------- config 4
@pytest.fixture(scope="module")
def s2s():
    from oracle import seq2seq as S
    W = wl.seq2seq_weights()
    return W, S.prepare_s2s(W)


def _torch_s2s(P, cfg):
    """torch.nn Transformer layers (post-LN, ReLU, dropout 0) in fp64 with our weights."""
    import torch.nn as nn
    d, H, f = cfg["d"], cfg["heads"], cfg["d_ff"]
    enc = [nn.TransformerEncoderLayer(d, H, f, dropout=0.0, batch_first=True).double().eval()
           for _ in range(cfg["enc_layers"])]
    dec = [nn.TransformerDecoderLayer(d, H, f, dropout=0.0, batch_first=True).double().eval()
           for _ in range(cfg["dec_layers"])]
    T = lambda a: torch.tensor(np.asarray(a, np.float64))  # noqa: E731
    with torch.no_grad():
        for l, L in enumerate(enc):
            p = f"enc{l}"
            L.self_attn.in_proj_weight.copy_(T(P[p + ".wqkv"]))
            L.self_attn.in_proj_bias.copy_(T(P[p + ".bqkv"]))
            L.self_attn.out_proj.weight.copy_(T(P[p + ".wo"]))
            L.self_attn.out_proj.bias.copy_(T(P[p + ".bo"]))
            L.norm1.weight.copy_(T(P[p + ".ln1.g"])); L.norm1.bias.copy_(T(P[p + ".ln1.b"]))
            L.linear1.weight.copy_(T(P[p + ".w1"])); L.linear1.bias.copy_(T(P[p + ".b1"]))
            L.linear2.weight.copy_(T(P[p + ".w2"])); L.linear2.bias.copy_(T(P[p + ".b2"]))
            L.norm2.weight.copy_(T(P[p + ".ln2.g"])); L.norm2.bias.copy_(T(P[p + ".ln2.b"]))
        for l, L in enumerate(dec):
            p = f"dec{l}"
            L.self_attn.in_proj_weight.copy_(T(P[p + ".wqkv"]))
            L.self_attn.in_proj_bias.copy_(T(P[p + ".bqkv"]))
            L.self_attn.out_proj.weight.copy_(T(P[p + ".wo"]))
            L.self_attn.out_proj.bias.copy_(T(P[p + ".bo"]))
            L.norm1.weight.copy_(T(P[p + ".ln1.g"])); L.norm1.bias.copy_(T(P[p + ".ln1.b"]))
            L.multihead_attn.in_proj_weight.copy_(torch.cat([T(P[p + ".wq2"]), T(P[p + ".wkv2"])]))
            L.multihead_attn.in_proj_bias.copy_(torch.cat([T(P[p + ".bq2"]), T(P[p + ".bkv2"])]))
            L.multihead_attn.out_proj.weight.copy_(T(P[p + ".wo2"]))
            L.multihead_attn.out_proj.bias.copy_(T(P[p + ".bo2"]))
            L.norm2.weight.copy_(T(P[p + ".ln2.g"])); L.norm2.bias.copy_(T(P[p + ".ln2.b"]))
            L.linear1.weight.copy_(T(P[p + ".w1"])); L.linear1.bias.copy_(T(P[p + ".b1"]))
            L.linear2.weight.copy_(T(P[p + ".w2"])); L.linear2.bias.copy_(T(P[p + ".b2"]))
            L.norm3.weight.copy_(T(P[p + ".ln3.g"])); L.norm3.bias.copy_(T(P[p + ".ln3.b"]))
    return enc, dec


def test_seq2seq_fixed_length_is_torch_transformer_greedy(s2s):
    """EOS bias -inf => fixed-length greedy decoding == torch.nn Transformer layers (full-prefix
    recompute with a causal mask each step), exact mode: tokens equal, logits to 1e-9."""
    from oracle import seq2seq as S
    W, P = s2s
    cfg = dict(wl.S2S)
    src = wl.token_inputs(wl.INPUT_SEED, 7, 1)[0]
    steps = 6
    out, L, top1, z0, _ = S.greedy_decode(src, P, cfg, "exact", eos_bias=lambda t, s: -np.inf, max_steps=steps)
    enc, dec = _torch_s2s(P, cfg)
    d = cfg["d"]
    pe = torch.tensor(S.positional_encoding(64, d))
    with torch.no_grad():
        x = torch.tensor(P["src_emb"][src]) * math.sqrt(d) + pe[:len(src)]
        m = x[None]
        for L_ in enc:
            m = L_(m)
        y = [cfg["bos"]]
        for t in range(steps):
            yt = torch.tensor(P["tgt_emb"][np.array(y)]) * math.sqrt(d) + pe[:len(y)]
            h = yt[None]
            mask = torch.triu(torch.full((len(y), len(y)), float("-inf"), dtype=torch.float64), 1)
            for L_ in dec:
                h = L_(h, m, tgt_mask=mask)
            z = torch.tensor(P["lm.w"]) @ h[0, -1] + torch.tensor(P["lm.b"])
            z[cfg["eos"]] = -np.inf
            tok = int(torch.argmax(z))
            assert tok == out[t], (t, tok, out[t])
            assert abs(float(z[tok]) - top1[t]) < 1e-9
            if t == 0:
                zz = z.numpy().copy()
                zz[cfg["eos"]] = 0
                z0c = z0.copy()
                z0c[cfg["eos"]] = 0
                np.testing.assert_allclose(z0c, zz, rtol=1e-9, atol=1e-9)
            y.append(tok)


def test_seq2seq_length_guard(s2s):
    """Loop guard: EOS bias +inf ends every sequence after 1 token; with the length table the
    sequence ends at floor(LEN[src0]) + 1 when margins are large (beta = 16); PAD after done."""
    from oracle import seq2seq as S
    W, P = s2s
    cfg = dict(wl.S2S)
    src = wl.token_inputs(wl.INPUT_SEED, 0, 3)
    for i in range(3):
        out, L, top1, _, _ = S.greedy_decode(src[i], P, cfg, "exact", eos_bias=lambda t, s: np.inf)
        assert L == 1 and out[0] == cfg["eos"] and np.all(out[1:] == cfg["pad"]) and np.isnan(top1[1:]).all()
    for i in range(2):
        out, L, top1, _, preds = S.greedy_decode(src[i], P, cfg, "exact")
        assert L == int(np.floor(P["len_table"][src[i][0]])) + 1
        assert out[L - 1] == cfg["eos"] and np.all(out[L:] == cfg["pad"]) and cfg["eos"] not in out[:L - 1]
        assert len(preds) == L


def test_seq2seq_mirror_rounding_points(s2s, monkeypatch):
    """Mirror mode rounds exactly at the GPU's bf16 storage points (SURVEY 8(c) 'mirror'):
    every linear's operand, q/k/v (self and cross), attention outputs and the FFN hidden;
    residual stream, LayerNorm, softmax and logits unrounded.  Pinned against an independent
    composition of torch fp64 primitives (F.linear, F.scaled_dot_product_attention,
    F.layer_norm) with torch's own bf16 cast at those points, full-prefix recompute under a
    causal mask (so the K/V cache is the rounded k/v of earlier positions).  This pins the
    rounding POINTS: both sides use torch's cast as the rounding function (it rounds fp64 via
    fp32, a double rounding that differs from round_bf16's direct rounding on rare ties;
    round_bf16 itself is pinned by test_round_bf16_matches_torch_cast_and_ties)."""
    import torch.nn.functional as F
    from oracle import seq2seq as S
    W, P = s2s
    real_round = S.round_bf16
    monkeypatch.setattr(S, "round_bf16",
                        lambda v: torch.tensor(np.asarray(v, np.float64)).to(torch.bfloat16).double().numpy())
    cfg = dict(wl.S2S)
    d, H = cfg["d"], cfg["heads"]
    src = wl.token_inputs(wl.INPUT_SEED, 21, 1)[0]
    steps = 3
    out, _, top1, z0, _ = S.greedy_decode(src, P, cfg, "mirror", eos_bias=lambda t, s: -np.inf, max_steps=steps)
    T = lambda a: torch.tensor(np.asarray(a, np.float64))  # noqa: E731
    rb = lambda t: t.to(torch.bfloat16).to(torch.float64)  # noqa: E731

    def lin(x, w, b):
        return F.linear(rb(x), T(P[w]), T(P[b]))

    def mha(q, k, v, causal):
        sp = lambda t: t.reshape(t.shape[0], H, d // H).transpose(0, 1)  # noqa: E731
        o = F.scaled_dot_product_attention(sp(q)[None], sp(k)[None], sp(v)[None], is_causal=causal)[0]
        return rb(o.transpose(0, 1).reshape(q.shape[0], d))

    def mha_enc(q, k, v):
        # encoder: P x V on the tensor cores, so P itself is a bf16 operand (reading R18)
        sp = lambda t: t.reshape(t.shape[0], H, d // H).transpose(0, 1)  # noqa: E731
        p = torch.softmax(sp(q) @ sp(k).transpose(1, 2) / np.sqrt(d // H), dim=-1)
        o = rb(p) @ sp(v)
        return rb(o.transpose(0, 1).reshape(q.shape[0], d))

    def ln(x, p):
        return F.layer_norm(x, (d,), T(P[p + ".g"]), T(P[p + ".b"]), eps=1e-5)

    pe = T(S.positional_encoding(64, d))
    with torch.no_grad():
        m = T(P["src_emb"][src]) * np.sqrt(d) + pe[:len(src)]
        for l in range(cfg["enc_layers"]):
            p = f"enc{l}"
            qkv = rb(lin(m, p + ".wqkv", p + ".bqkv"))
            a = mha_enc(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:])
            m = ln(lin(a, p + ".wo", p + ".bo") + m, p + ".ln1")
            h = rb(F.relu(lin(m, p + ".w1", p + ".b1")))
            m = ln(lin(h, p + ".w2", p + ".b2") + m, p + ".ln2")
        y = [cfg["bos"]]
        for t in range(steps):
            x = T(P["tgt_emb"][np.array(y)]) * np.sqrt(d) + pe[:len(y)]
            for l in range(cfg["dec_layers"]):
                p = f"dec{l}"
                qkv = rb(lin(x, p + ".wqkv", p + ".bqkv"))
                a = mha(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], True)
                x = ln(lin(a, p + ".wo", p + ".bo") + x, p + ".ln1")
                q2 = rb(lin(x, p + ".wq2", p + ".bq2"))
                kv = rb(lin(m, p + ".wkv2", p + ".bkv2"))
                a2 = mha(q2, kv[:, :d], kv[:, d:], False)
                x = ln(lin(a2, p + ".wo2", p + ".bo2") + x, p + ".ln2")
                h = rb(F.relu(lin(x, p + ".w1", p + ".b1")))
                x = ln(lin(h, p + ".w2", p + ".b2") + x, p + ".ln3")
            z = lin(x[-1:], "lm.w", "lm.b")[0]
            z[cfg["eos"]] = -np.inf
            tok = int(torch.argmax(z))
            assert tok == out[t]
            assert abs(float(z[tok]) - top1[t]) <= 1e-9 * max(1.0, abs(top1[t]))
            if t == 0:
                zz, z0c = z.numpy().copy(), z0.copy()
                zz[cfg["eos"]] = z0c[cfg["eos"]] = 0
                np.testing.assert_allclose(z0c, zz, rtol=1e-9, atol=1e-9)
            y.append(tok)
    # and the rounding really happens: mirror differs from exact
    monkeypatch.setattr(S, "round_bf16", real_round)
    _, _, top1e, z0e, _ = S.greedy_decode(src, P, cfg, "exact", eos_bias=lambda t, s: -np.inf, max_steps=1)
    z0m = z0.copy()
    z0m[cfg["eos"]] = z0e[cfg["eos"]] = 0
    assert np.max(np.abs(z0m - z0e)) > 1e-6
