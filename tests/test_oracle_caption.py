"""Pins of the captioning En-Decoder oracle (reading R20)
against torch CPU fp64 library routines (runs without a GPU)."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import workloads as wl
from oracle import caption as C
from oracle import programs as prg
from tests import torch_ref as TR


@pytest.fixture(scope="module")
def cap():
    W = wl.caption_weights()
    return W, prg.prepare(W)


def _torch_decode(a, W, cfg, rb=None, eos_bias=None):
    """Independent composition: torch.nn.LSTMCell (fp64) on [E[y]; z] with h as the recurrent
    input, torch softmax attention, F.linear heads, torch.argmax greedy loop with the guard."""
    T = lambda v: torch.tensor(np.asarray(v, np.float64))  # noqa: E731
    exact = rb is None
    if exact:
        rb = lambda t: t  # noqa: E731
    H, E, D = cfg["hidden"], cfg["emb"], a.shape[1]
    w = T(prg._bf16_to_f64(W["lstm.w"]))
    cell = torch.nn.LSTMCell(E + D, H).double()
    with torch.no_grad():
        cell.weight_ih.copy_(w[:, :E + D])
        cell.weight_hh.copy_(w[:, E + D:])
        cell.bias_ih.copy_(T(W["lstm.b"]))
        cell.bias_hh.zero_()
    A = T(a)
    init_w, init_b = T(prg._bf16_to_f64(W["init.w"])), T(W["init.b"])
    abar = rb(A.mean(dim=0))
    h = torch.tanh(F.linear(abar, init_w[:H], init_b[:H]))[None]
    c = torch.tanh(F.linear(abar, init_w[H:], init_b[H:]))[None]
    emb = T(prg._bf16_to_f64(W["emb"]))
    att_w, att_b = T(prg._bf16_to_f64(W["att.w"])), T(W["att.b"])
    out_w, out_b = T(prg._bf16_to_f64(W["out.w"])), T(W["out.b"]).clone()
    if eos_bias is not None:
        out_b[cfg["eos"]] = eos_bias
    toks, top1, y, L = [], [], cfg["bos"], cfg["max_len"]
    with torch.no_grad():
        for t in range(cfg["max_len"]):
            q = F.linear(rb(h[0]), att_w, att_b)
            alpha = torch.softmax(A @ q / math.sqrt(D), dim=0)
            z = alpha @ A
            x = torch.cat([emb[y], rb(z)])[None]
            h, c = cell(x, (h, c)) if exact else _cell_rb(cell, x, h, c, rb)
            logits = F.linear(rb(h[0]), out_w, out_b)
            tok = int(torch.argmax(logits))
            toks.append(tok)
            top1.append(float(logits[tok]))
            y = tok
            if tok == cfg["eos"]:
                L = t + 1
                break
    return toks, L, top1


def _cell_rb(cell, x, h, c, rb):
    """LSTMCell with the recurrent operand rounded (the GPU's bf16 operand copy of h) while the
    state h, c themselves stay unrounded: W_hh applied to rb(h)."""
    gates = F.linear(x, cell.weight_ih, cell.bias_ih) + F.linear(rb(h), cell.weight_hh, cell.bias_hh)
    i, f, g, o = gates.chunk(4, dim=1)
    c2 = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(g)
    return torch.sigmoid(o) * torch.tanh(c2), c2


def test_encoder_is_torch_resnet38_trunk(cap):
    W, P = cap
    X = wl.image_inputs(wl.INPUT_SEED, 7, 1)
    a = C.encode(X[0], P, "exact")
    ref = TR.static_resnet(X[0], W, 6)[0].permute(1, 2, 0).reshape(-1, 64).numpy()
    np.testing.assert_allclose(a, ref, rtol=1e-12, atol=1e-12)


def test_decoder_exact_is_torch_lstmcell_greedy(cap):
    """exact mode == torch.nn.LSTMCell greedy loop (fp64): tokens, length, top-1 logits."""
    W, P = cap
    rng = np.random.default_rng(11)
    for _ in range(3):
        a = rng.standard_normal((64, 64)) * 0.5 + 0.5
        out, L, top1, _ = C.decode(a, P, wl.CAP, "exact")
        toks, L2, t2 = _torch_decode(a, W, wl.CAP)
        assert L == L2 and list(out[:L]) == toks
        assert np.all(out[L:] == wl.CAP["pad"])
        np.testing.assert_allclose(top1[:L], t2, rtol=1e-10, atol=1e-10)


def test_decoder_mirror_rounding_points(cap, monkeypatch):
    """mirror mode rounds exactly at the GPU's bf16 operand points (mean(a), h before each
    GEMM, z, the word embedding rows by construction); pinned against the torch composition
    with torch's bf16 cast at those points (both use torch's cast as the rounding function)."""
    W, P = cap
    monkeypatch.setattr(C, "round_bf16",
                        lambda v: torch.tensor(np.asarray(v, np.float64)).to(torch.bfloat16).double().numpy())
    rb = lambda t: t.to(torch.bfloat16).to(torch.float64)  # noqa: E731
    a = prg._bf16_to_f64(wl.f32_to_bf16_bits(np.random.default_rng(5).standard_normal((64, 64)) * 0.5 + 0.5))
    out, L, top1, _ = C.decode(a, P, wl.CAP, "mirror")
    toks, L2, t2 = _torch_decode(a, W, wl.CAP, rb=rb)
    assert L == L2 and list(out[:L]) == toks
    np.testing.assert_allclose(top1[:L], t2, rtol=1e-9, atol=1e-9)


def test_loop_guard_degenerate_eos(cap):
    """EOS bias +inf: every caption is [EOS] (length 1, PAD after); -inf: no EOS, length 32."""
    W, P = cap
    X = wl.image_inputs(wl.INPUT_SEED, 3, 2)
    for i in range(2):
        out, L, top1, preds = C.caption(X[i], P, wl.CAP, "exact", eos_bias=np.inf)
        assert L == 1 and out[0] == wl.CAP["eos"] and np.all(out[1:] == wl.CAP["pad"]) and np.isnan(top1[1:]).all()
        out, L, top1, preds = C.caption(X[i], P, wl.CAP, "exact", eos_bias=-np.inf)
        assert L == wl.CAP["max_len"] and wl.CAP["eos"] not in out and len(preds) == L


def test_teacher_forcing_with_own_output_is_free_running(cap):
    W, P = cap
    X = wl.image_inputs(wl.INPUT_SEED, 4, 1)
    a = C.encode(X[0], P, "mirror")
    out, L, top1, _ = C.decode(a, P, wl.CAP, "mirror")
    out2, L2, top2, _ = C.decode(a, P, wl.CAP, "mirror", forced=out)
    assert L == L2 and np.array_equal(out, out2) and np.allclose(top1[:L], top2[:L])


def test_calibrated_lengths_vary(cap):
    W, P = cap
    X = wl.image_inputs(wl.INPUT_SEED, 0, 12)
    Ls = [C.caption(X[i], P, wl.CAP, "mirror")[1] for i in range(12)]
    assert len(set(Ls)) >= 4 and 2 <= np.mean(Ls) <= 28
