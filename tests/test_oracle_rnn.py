"""Pins of the recurrent-gate SkipNet oracle (Table 3 ID 5 "ResNet38 + RNN",
PAPER.md L812; reading R19) against torch CPU fp64 library routines (runs without a GPU)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
import workloads as wl
from oracle import programs as prg
from tests import torch_ref as TR


@pytest.fixture(scope="module")
def r38r():
    return wl.skipnet_rnn_r38_weights()


def _torch_cell(W, cls):
    H, NI = int(W["rnn.hidden"]), int(W["rnn.n_in"])
    m = cls(NI, H).double()
    with torch.no_grad():
        sfx = "_l0" if cls is torch.nn.LSTM else ""
        getattr(m, "weight_ih" + sfx).copy_(torch.tensor(np.asarray(W["rnn.w_ih"], np.float64)))
        getattr(m, "weight_hh" + sfx).copy_(torch.tensor(np.asarray(W["rnn.w_hh"], np.float64)))
        getattr(m, "bias_ih" + sfx).copy_(torch.tensor(np.asarray(W["rnn.b_ih"], np.float64)))
        getattr(m, "bias_hh" + sfx).copy_(torch.tensor(np.asarray(W["rnn.b_hh"], np.float64)))
    return m


def test_lstm_cell_is_torch_lstmcell(r38r):
    """One step equals torch.nn.LSTMCell (gate order i, f, g, o; both biases) in fp64."""
    P = prg.prepare(r38r)
    cell = _torch_cell(r38r, torch.nn.LSTMCell)
    rng = np.random.default_rng(5)
    for _ in range(4):
        u, h, c = rng.standard_normal(10), rng.standard_normal(10), rng.standard_normal(10)
        ho, co = prg.lstm_cell(u, h, c, P)
        th, tc = cell(torch.tensor(u)[None], (torch.tensor(h)[None], torch.tensor(c)[None]))
        np.testing.assert_allclose(ho, th[0].detach().numpy(), rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(co, tc[0].detach().numpy(), rtol=1e-13, atol=1e-13)


def _forced(W, pattern):
    W = dict(W)
    for i in wl.SKIP_GATED:
        W[f"out{i}.b"] = np.array([1e9 if pattern(i) else -1e9], np.float32)
    return W


@pytest.mark.parametrize("name,pattern", [
    ("all_execute", lambda i: True), ("all_skip", lambda i: False), ("even_blocks", lambda i: i % 2 == 0)])
def test_rnn_forced_gates_equal_static_composition_and_torch_lstm(r38r, name, pattern):
    """Output bias +-inf fixes the path: the logits are the static network's (torch conv chain),
    and the gate state is torch.nn.LSTM run over the 17 gate inputs u_i = proj_i(GAP(block input))
    computed from the torch chain -- the cell steps at EVERY gate, executed or skipped, and the
    state carries across gates (not reset)."""
    W = _forced(r38r, pattern)
    P = prg.prepare(W)
    X = wl.image_inputs(wl.INPUT_SEED, 13, 1)
    seen = {}
    z, mask, preds = O.skipnet_rnn_resnet38(X[0], P, "exact",
                                            gate_hook=lambda i, g, hs, zz: seen.__setitem__(i, hs.copy()))
    assert mask == sum(1 << (i - 2) for i in wl.SKIP_GATED if pattern(i)) and len(preds) == 17
    execd = {1} | {i for i in wl.SKIP_GATED if pattern(i)}
    ref = TR.head(TR.static_resnet(X[0], W, 6, exec_blocks=execd), W, "final").numpy()
    np.testing.assert_allclose(z, ref, rtol=1e-12, atol=1e-12)
    # the gate inputs from the torch chain: block i's input is the output after blocks 1..i-1
    us = []
    for i in wl.SKIP_GATED:
        x = TR.static_resnet(X[0], W, 6, upto=i - 1, exec_blocks=execd)
        g = x.mean(dim=(2, 3))[0]
        us.append(F.linear(g, TR._w(W[f"proj{i}.w"]), TR._w(W[f"proj{i}.b"])))
    lstm = _torch_cell(W, torch.nn.LSTM)
    out, _ = lstm(torch.stack(us)[:, None, :])
    for k, i in enumerate(wl.SKIP_GATED):
        np.testing.assert_allclose(seen[i], out[k, 0].detach().numpy(), rtol=1e-11, atol=1e-12)


def test_rnn_zero_output_weights_skip_everything(r38r):
    """w_out = 0, b_out = 0 gives p = sigmoid(0) = 1/2 at every gate: reading R2 skips them all."""
    W = dict(r38r)
    for i in wl.SKIP_GATED:
        W[f"out{i}.w"] = np.zeros(10, np.float32)
        W[f"out{i}.b"] = np.zeros(1, np.float32)
    P = prg.prepare(W)
    X = wl.image_inputs(wl.INPUT_SEED, 2, 1)
    z, mask, preds = O.skipnet_rnn_resnet38(X[0], P, "exact")
    assert mask == 0 and all(p[1] == 0.5 for p in preds)
    ref = TR.head(TR.static_resnet(X[0], W, 6, exec_blocks={1}), W, "final").numpy()
    np.testing.assert_allclose(z, ref, rtol=1e-12, atol=1e-12)


def test_rnn_calibrated_gates_branch(r38r):
    X = wl.image_inputs(wl.INPUT_SEED, 0, 24)
    P = prg.prepare(r38r)
    _, mask, preds = O.run_batch(O.skipnet_rnn_resnet38, X, P, "mirror")
    bits = np.array([bin(int(m)).count("1") for m in mask])
    assert len(set(mask.tolist())) > 10
    assert 3 <= bits.mean() <= 14
