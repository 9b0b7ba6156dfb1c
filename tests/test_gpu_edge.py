"""GPU tests of the method's degenerate cases and of the registration error codes.

Degenerate predicates (SURVEY 8(c) pins, run on the CUDA path through the C ABI and graded
against the oracle on the same settings):
  * tau > 1: no sample ever exits (the static network);
  * tau <= 1/K: every sample exits at the first head, so every later sub-network, head,
    compaction and scatter runs on 0 live rows (an exit that empties the batch);
  * SkipNet gate bias +-inf: all / no / alternate blocks executed (Listing 3 reduces to a
    static network);
  * decoder EOS bias +-inf (length table at -+1e6 with beta = 16): every length 1 / 64.
Registration errors: SHAPE_JOIN, SIGNATURE, SHAPE_MISMATCH, STATE, and a
batch above max_batch at run time.
"""
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


def _run(model, X):
    B = X.shape[0]
    x = torch.from_numpy(X).to(DEV)
    logits = torch.full((max(B, 1), model.K), float("nan"), device=DEV)
    path = torch.full((max(B, 1),), -7, dtype=torch.int32, device=DEV)
    counts = torch.full((64,), -1, dtype=torch.int32, device=DEV)
    model.run(x, logits, path, node_counts=counts)
    torch.cuda.synchronize()
    return logits[:B].cpu().numpy(), path[:B].cpu().numpy(), counts.cpu().numpy()


def _grade(W, model, program, X, **kw):
    lg, pg, cnt = _run(model, X)
    lo, po, pr = O.run_batch(program, X, prg.prepare(W), "mirror", **kw)
    r = report(lg, pg, lo, po, pr)
    assert r["outside_band_mismatch"] == 0 and r["logit_rel_fail"] == 0, r
    return lg, pg, cnt, r


# ------------------------------------------------------------ exits: tau > 1, tau <= 1/K
@pytest.mark.parametrize("tau,expect", [(1.5, "final"), (0.1, "first")])
def test_cfg1_degenerate_tau(tau, expect):
    W = wl.mlp_weights()
    X = wl.mlp_inputs(wl.INPUT_SEED, 0, 32)
    m = P.build_mlp_ee(W, 32, tau=tau)
    _, pg, _, _ = _grade(W, m, O.mlp_ee, X, tau=tau)
    assert (pg == (2 if expect == "final" else 0)).all()


@pytest.mark.parametrize("tau,expect", [(1.5, 4), (0.1, 0)])
def test_cfg2_degenerate_tau(tau, expect):
    W = wl.sdn_r56_weights()
    X = wl.image_inputs(wl.INPUT_SEED, 50, 96)
    m = P.build_sdn_resnet56(W, 128, tau=tau)
    _, pg, cnt, r = _grade(W, m, O.sdn_resnet56, X, tau=tau)
    assert (pg == expect).all(), np.bincount(pg)
    if expect == 0:
        # counts slot 1: survivors of exit 0 -- the rest of the chain ran on 0 live rows
        assert cnt[2] == 0, cnt[:12]


def test_cfg2_traced_program_differs_from_dynamic():
    """The trace baseline on the GPU path (Table 2): the program with every
    exit predicate frozen to "stay" (tau > 1, a trace of an input that ran to the final head)
    reproduces the dynamic run BITWISE for the inputs that take the final head in it -- the
    kernels are batch-position independent, so the compaction in between changes nothing --
    and differs for every input that exits early (eta > 0)."""
    from oracle.metrics import eta
    W = wl.sdn_r56_weights()
    X = wl.image_inputs(wl.INPUT_SEED, 4000, 256)
    ld, pd, _ = _run(P.build_sdn_resnet56(W, 256), X)
    lt, pt, _ = _run(P.build_sdn_resnet56(W, 256, tau=1.5), X)
    assert (pt == 4).all() and (pd < 4).any() and (pd == 4).any(), np.bincount(pd)
    fin = pd == 4
    assert np.array_equal(lt[fin], ld[fin])
    assert np.all(np.max(np.abs(lt[~fin] - ld[~fin]), axis=1) > 0)
    assert eta(list(np.argmax(lt, 1)), list(np.argmax(ld, 1))) > 0.0


@pytest.mark.parametrize("tau,expect", [(1.5, 3), (0.1, 0)])
def test_cfg5_degenerate_tau(tau, expect):
    W = wl.resnet50_ee_weights()
    X = wl.image_inputs(wl.INPUT_SEED, 77, 6, hw=224)
    m = P.build_resnet50_ee(W, 8, tau=tau)
    _, pg, _, _ = _grade(W, m, O.resnet50_ee, X, tau=tau)
    assert (pg == expect).all()


# ------------------------------------------------------------ gates: bias +-inf
def _forced_gates(W, pattern):
    W = dict(W)
    for i in wl.SKIP_GATED:
        W[f"gate{i}.b"] = np.array([1e9 if pattern(i) else -1e9], np.float32)
    return W


@pytest.mark.parametrize("name,pattern", [("all", lambda i: True), ("none", lambda i: False),
                                          ("even", lambda i: i % 2 == 0)])
def test_cfg3_forced_gates(name, pattern):
    W = _forced_gates(wl.skipnet_r38_weights(), pattern)
    X = wl.image_inputs(wl.INPUT_SEED, 60, 64)
    m = P.build_skipnet_resnet38(W, 64)
    _, pg, _, _ = _grade(W, m, O.skipnet_resnet38, X)
    want = sum(1 << (i - 2) for i in wl.SKIP_GATED if pattern(i))
    assert (pg == want).all(), (name, np.unique(pg))


# ------------------------------------------------------------ decoder: EOS bias +-inf
@pytest.mark.parametrize("len_value,expect", [(-1e6, 1), (1e6, 64)])
def test_cfg4_forced_lengths(len_value, expect):
    from tests.s2s_parity import compare_free_running, run_s2s
    from oracle import seq2seq as S
    W = dict(wl.seq2seq_weights())
    W["len_table"] = np.full_like(np.asarray(W["len_table"]), len_value)
    m = P.build_seq2seq(W, wl.S2S, 8)
    src = wl.token_inputs(wl.INPUT_SEED, 500, 3)
    tok, ln, top1, z0 = run_s2s(m, src)
    assert (ln == expect).all(), ln
    if expect == 1:
        assert (tok[:, 0] == wl.S2S["eos"]).all() and (tok[:, 1:] == wl.S2S["pad"]).all()
    else:
        assert (tok != wl.S2S["eos"]).all()
    rep = compare_free_running(S.prepare_s2s(W), src, tok, ln, top1, z0)
    assert rep["mismatch"] == 0 and rep["max_top1_rel"] <= 2e-2, rep


# ------------------------------------------------------------ registration errors
def _status(fn, *a):
    try:
        fn(*a)
    except D.DyclError as e:
        return e.status
    return 0


def _bits(shape, seed=0):
    return wl.f32_to_bf16_bits(np.random.default_rng(seed).standard_normal(shape) * 0.1)


def _head(g, c, k):
    h = D.dycl_subnet_begin(g)
    D.dycl_subnet_gap(g, h)
    D.dycl_subnet_dense(g, h, c, k, _bits((k, c)), np.zeros(k, np.float32), D.DYCL_ACT_NONE, 1)
    D.dycl_subnet_end(g, h)
    return h


def _conv_subnet(g, c_in, c_out, stride=1, residual=False):
    sn = D.dycl_subnet_begin(g)
    if residual:
        D.dycl_subnet_block_begin(g, sn)
    D.dycl_subnet_conv2d(g, sn, c_in, c_out, 3, stride, 1, _bits((c_out, 3, 3, c_in)), np.zeros(c_out, np.float32),
                         D.DYCL_ACT_RELU, 1 if residual else 0)
    D.dycl_subnet_end(g, sn)
    return sn


def test_error_shape_join():
    """A gate whose then-branch output joins neither identity nor option A (16 -> 48 channels)."""
    g = D.dycl_graph_create(0, 8, 8, 16)
    D.dycl_gate(g, _head(g, 16, 1), 0.5, _conv_subnet(g, 16, 48))
    D.dycl_final(g, _head(g, 48, 10))
    assert _status(D.dycl_finalize, g, 4) == -4
    D.dycl_graph_destroy(g)


def test_error_signature():
    """Exit and final heads disagree on K; a gate head with two logits."""
    g = D.dycl_graph_create(0, 8, 8, 16)
    D.dycl_seq(g, _conv_subnet(g, 16, 16))
    D.dycl_exit(g, _head(g, 16, 10), 0.9)
    D.dycl_final(g, _head(g, 16, 5))
    assert _status(D.dycl_finalize, g, 4) == -3
    D.dycl_graph_destroy(g)
    g = D.dycl_graph_create(0, 8, 8, 16)
    D.dycl_gate(g, _head(g, 16, 2), 0.5, _conv_subnet(g, 16, 16))
    D.dycl_final(g, _head(g, 16, 10))
    assert _status(D.dycl_finalize, g, 4) == -3
    D.dycl_graph_destroy(g)


def test_error_shape_mismatch_and_state():
    # conv c_in disagreeing with the propagated shape
    g = D.dycl_graph_create(0, 8, 8, 16)
    D.dycl_seq(g, _conv_subnet(g, 32, 32))
    D.dycl_final(g, _head(g, 32, 10))
    assert _status(D.dycl_finalize, g, 4) == -2
    D.dycl_graph_destroy(g)
    # residual whose shortcut is neither identity nor option A (16 -> 48, same H, W)
    g = D.dycl_graph_create(0, 8, 8, 16)
    D.dycl_seq(g, _conv_subnet(g, 16, 48, residual=True))
    D.dycl_final(g, _head(g, 48, 10))
    assert _status(D.dycl_finalize, g, 4) == -2
    D.dycl_graph_destroy(g)
    # a chain that does not end with dycl_final; run before finalize; batch > max_batch
    g = D.dycl_graph_create(0, 8, 8, 16)
    D.dycl_seq(g, _conv_subnet(g, 16, 16))
    assert _status(D.dycl_finalize, g, 4) == -5
    D.dycl_final(g, _head(g, 16, 10))
    x = torch.zeros((8, 8, 8, 16), device=DEV)
    lg = torch.empty((8, 10), device=DEV)
    pa = torch.empty(8, dtype=torch.int32, device=DEV)
    assert _status(D.dycl_run, g, x, 8, lg, pa) == -5
    D.dycl_finalize(g, 4)
    assert _status(D.dycl_finalize, g, 4) == -5
    assert _status(D.dycl_run, g, x, 8, lg, pa) == -2
    D.dycl_run(g, x, 4, lg, pa)
    torch.cuda.synchronize()
    assert set(pa[:4].cpu().tolist()) <= {0, -1}
    D.dycl_graph_destroy(g)
