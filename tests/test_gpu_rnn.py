"""GPU tests of the recurrent-gate SkipNet (Table 3 ID 5 "ResNet38 + RNN",
PAPER.md L812; reading R19) through the C ABI (dycl_rnn_cell / dycl_gate_rnn), graded against
the oracle's mirror mode: decisions bit-exact outside the 1e-3 band, logits within 2e-2."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as wl
from oracle import programs as prg
from tests.parity import report

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

DEV = torch.device("cuda:0")


def _run(m, X):
    B = X.shape[0]
    x = torch.from_numpy(X).to(DEV)
    lg = torch.full((max(B, 1), 10), float("nan"), device=DEV)
    pa = torch.full((max(B, 1),), -7, dtype=torch.int32, device=DEV)
    m.run(x, lg, pa)
    torch.cuda.synchronize()
    return lg[:B].cpu().numpy(), pa[:B].cpu().numpy()


@pytest.fixture(scope="module")
def r38r():
    W = wl.skipnet_rnn_r38_weights()
    return W, P.build_skipnet_rnn_resnet38(W, 8192)


@pytest.mark.parametrize("B,start", [(256, 2000), (77, 500), (1, 9)])
def test_cfg3r_rnn_skipnet_parity(r38r, B, start):
    W, m = r38r
    X = wl.image_inputs(wl.INPUT_SEED, start, B)
    lg, pg = _run(m, X)
    lo, po, pr = O.run_batch(O.skipnet_rnn_resnet38, X, prg.prepare(W), "mirror")
    r = report(lg, pg, lo, po, pr)
    print("cfg3r", B, r)
    assert r["logit_rel_fail"] == 0 and r["outside_band_mismatch"] == 0, r


def test_cfg3r_full_batch_sampled_parity(r38r):
    """8192 rows (the config-3 batch, in-place gates): 512 sampled rows vs the oracle; the state
    is per original sample, so a permuted batch gives the permuted result bitwise."""
    W, m = r38r
    X = wl.image_inputs(wl.INPUT_SEED, 0, 8192)
    lg, pg = _run(m, X)
    assert np.isfinite(lg).all() and (pg >= 0).all() and (pg < (1 << 17)).all()
    idx = np.random.default_rng(wl.ORACLE_SUBSET_SEED).choice(8192, 512, replace=False)
    lo, po, pr = O.run_batch(O.skipnet_rnn_resnet38, X[idx], prg.prepare(W), "mirror")
    r = report(lg[idx], pg[idx], lo, po, pr)
    print("cfg3r full sampled", r, "mean executed", np.mean([bin(int(v)).count("1") for v in pg]))
    assert r["logit_rel_fail"] == 0 and r["outside_band_mismatch"] == 0, r
    perm = np.random.default_rng(4).permutation(512)
    l2, p2 = _run(m, X[:512][perm])
    assert np.array_equal(p2, pg[:512][perm]) and np.array_equal(l2, lg[:512][perm])


@pytest.mark.parametrize("name,pattern", [
    ("all_execute", lambda i: True), ("all_skip", lambda i: False), ("even_blocks", lambda i: i % 2 == 0)])
def test_cfg3r_forced_gates(name, pattern):
    W = dict(wl.skipnet_rnn_r38_weights())
    for i in wl.SKIP_GATED:
        W[f"out{i}.b"] = np.array([1e9 if pattern(i) else -1e9], np.float32)
    m = P.build_skipnet_rnn_resnet38(W, 64)
    X = wl.image_inputs(wl.INPUT_SEED, 40, 64)
    lg, pg = _run(m, X)
    want = sum(1 << (i - 2) for i in wl.SKIP_GATED if pattern(i))
    assert (pg == want).all()
    lo, po, pr = O.run_batch(O.skipnet_rnn_resnet38, X, prg.prepare(W), "mirror")
    r = report(lg, pg, lo, po, pr)
    assert r["logit_rel_fail"] == 0 and r["outside_band_mismatch"] == 0, r


def _status(fn, *a):
    try:
        fn(*a)
        return 0
    except D.DyclError as e:
        return e.status


def test_cfg3r_registration_errors():
    W = wl.skipnet_rnn_r38_weights()
    g = D.dycl_graph_create(0, 32, 32, 3)
    one = np.zeros(10, np.float32)
    # a recurrent gate before the cell exists: STATE
    assert _status(D.dycl_gate_rnn, g, 0, one, 0.0, 0.5, 0) == -5
    # bad sizes: INVALID_ARG; a second cell: STATE
    assert _status(D.dycl_rnn_cell, g, 0, 10, W["rnn.w_ih"], W["rnn.w_hh"], W["rnn.b_ih"], W["rnn.b_hh"]) == -1
    D.dycl_rnn_cell(g, 10, 10, W["rnn.w_ih"], W["rnn.w_hh"], W["rnn.b_ih"], W["rnn.b_hh"])
    assert _status(D.dycl_rnn_cell, g, 10, 10, W["rnn.w_ih"], W["rnn.w_hh"], W["rnn.b_ih"], W["rnn.b_hh"]) == -5
    # proj output width (7) != the cell's n_in (10): SHAPE_MISMATCH at finalize
    sn = D.dycl_subnet_begin(g)
    D.dycl_subnet_conv2d(g, sn, 3, 16, 3, 1, 1, W["stem.w"], W["stem.b"], D.DYCL_ACT_RELU, 0)
    D.dycl_subnet_end(g, sn)
    D.dycl_seq(g, sn)
    proj = D.dycl_subnet_begin(g)
    D.dycl_subnet_gap(g, proj)
    D.dycl_subnet_dense(g, proj, 16, 7, np.zeros((7, 16), np.uint16), np.zeros(7, np.float32), D.DYCL_ACT_NONE, 1)
    D.dycl_subnet_end(g, proj)
    blk = D.dycl_subnet_begin(g)
    D.dycl_subnet_block_begin(g, blk)
    D.dycl_subnet_conv2d(g, blk, 16, 16, 3, 1, 1, W["b2.c1.w"], W["b2.c1.b"], D.DYCL_ACT_RELU, 0)
    D.dycl_subnet_conv2d(g, blk, 16, 16, 3, 1, 1, W["b2.c2.w"], W["b2.c2.b"], D.DYCL_ACT_RELU, 1)
    D.dycl_subnet_end(g, blk)
    D.dycl_gate_rnn(g, proj, one, 0.0, 0.5, blk)
    fin = D.dycl_subnet_begin(g)
    D.dycl_subnet_gap(g, fin)
    D.dycl_subnet_dense(g, fin, 16, 10, np.zeros((10, 16), np.uint16), np.zeros(10, np.float32), D.DYCL_ACT_NONE, 1)
    D.dycl_subnet_end(g, fin)
    D.dycl_final(g, fin)
    assert _status(D.dycl_finalize, g, 4) == -2
    D.dycl_graph_destroy(g)
