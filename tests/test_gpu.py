"""GPU parity tests: the CUDA path (through the C ABI) vs the CPU oracle.

Run on a B200:  python -m pytest tests -m gpu -x -q
"""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as wl
from oracle import programs as prg
from tests.parity import report
from tests.s2s_parity import FLIP_NOISE_MARGIN, compare_free_running, compare_teacher_forced, run_s2s

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

DEV = torch.device("cuda:0")


def _bits_to_t(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(DEV)


def _t_to_f64(t):
    return (t.cpu().numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _planar(bits_nhwc):
    """NHWC bf16 bits -> the library's channel-planar layout [n][C/8][H][W][8]."""
    n, H, W, C = bits_nhwc.shape
    return np.ascontiguousarray(bits_nhwc.reshape(n, H, W, C // 8, 8).transpose(0, 3, 1, 2, 4))


def _unplanar(a, shape):
    n, H, W, C = shape
    return np.ascontiguousarray(a.reshape(n, C // 8, H, W, 8).transpose(0, 2, 3, 1, 4).reshape(n, H, W, C))


@pytest.fixture(scope="module")
def any_graph():
    g = D.dycl_graph_create(0, 1, 1, 8)
    yield g
    D.dycl_graph_destroy(g)


# ------------------------------------------------------------ a1 conv kernel
CONV_CASES = [
    # n, H, W, C, Cout, k, stride, pad, relu, res_mode
    (3, 32, 32, 16, 16, 3, 1, 1, 1, 0),
    (2, 32, 32, 16, 16, 3, 1, 1, 1, 1),
    (2, 32, 32, 16, 32, 3, 2, 1, 1, 2),     # option-A shortcut
    (4, 32, 32, 8, 16, 3, 1, 1, 1, 0),      # stem (C padded 3 -> 8)
    (5, 8, 8, 64, 64, 3, 1, 1, 1, 1),
    (5, 7, 7, 64, 128, 3, 1, 1, 0, 0),      # ragged M (245 rows), BN = 128
    (3, 7, 7, 32, 256, 1, 1, 0, 1, 0),      # BN = 256
    (2, 9, 9, 16, 512, 3, 2, 1, 1, 0),      # N tiling (2 x 256)
    (37, 1, 1, 64, 64, 1, 1, 0, 1, 0),      # dense layer
    (1, 12, 12, 24, 48, 7, 2, 3, 0, 0),     # 7x7 / stride 2 / pad 3
    (3, 16, 16, 32, 32, 3, 1, 1, 1, 1),     # stage-2 shape (halo mode)
    (3, 16, 16, 32, 64, 3, 2, 1, 1, 2),     # stage-2 -> 3 transition, option A
    (7, 8, 8, 64, 64, 3, 1, 1, 1, 0),       # odd sample count across 2-sample tiles
    (5, 32, 32, 16, 16, 3, 1, 1, 1, 1),
    (300, 1, 1, 512, 1536, 1, 1, 0, 0, 0),  # dense GEMM, TMA SW128 path (BN 256), ragged M
    (77, 1, 1, 128, 384, 1, 1, 0, 1, 1),    # dense GEMM BN 128 + residual + ReLU
    (9500, 1, 1, 64, 192, 1, 1, 0, 1, 0),   # dense GEMM, Cout = 64 * odd with >= num_sms/2 M tiles (BN 64)
]


TMA_CASES = [c for c in CONV_CASES if c[4] in (16, 32, 64) or (c[1] == c[2] == 1 and c[3] % 64 == 0 and c[4] % 64 == 0)]


ROWTAP_CASES = [c for c in TMA_CASES if c[5] == 3 and c[6] == 1 and c[7] == 1 and c[3] >= 16 and c[1] * c[2] >= 128]


# path 1: cp.async-fed kernel; 2: TMA kernel (row-tap mode where eligible); 3: TMA kernel, no row-tap
@pytest.mark.parametrize("path,case", [(1, c) for c in CONV_CASES] + [(2, c) for c in TMA_CASES] +
                         [(3, c) for c in ROWTAP_CASES],
                         ids=[f"cpasync-{c}" for c in CONV_CASES] + [f"tma-{c}" for c in TMA_CASES] +
                             [f"tma-norowtap-{c}" for c in ROWTAP_CASES])
def test_conv_kernel_matches_oracle_conv(any_graph, path, case):
    n, H, W, C, Co, k, st, pad, relu, res_mode = case
    rng = np.random.default_rng(abs(hash(case)) % 2**32)
    x = wl.f32_to_bf16_bits(rng.standard_normal((n, H, W, C)))
    w = wl.f32_to_bf16_bits(rng.standard_normal((Co, k, k, C)) * np.sqrt(2.0 / (k * k * C)))
    b = rng.uniform(-0.1, 0.1, Co).astype(np.float32)
    Ho, Wo = (H + 2 * pad - k) // st + 1, (W + 2 * pad - k) // st + 1
    res = None
    if res_mode == 1:
        res = wl.f32_to_bf16_bits(rng.standard_normal((n, Ho, Wo, Co)))
    elif res_mode == 2:
        res = wl.f32_to_bf16_bits(rng.standard_normal((n, 2 * Ho, 2 * Wo, Co // 2)))
    y = torch.zeros((n, Co // 8, Ho, Wo, 8), dtype=torch.int16, device=DEV)
    D.dycl_debug_conv2d(any_graph, _bits_to_t(_planar(x)), n, H, W, C, w, b, Co, k, st, pad, relu,
                        _bits_to_t(_planar(res)) if res is not None else None, res_mode, y, path)
    got = _unplanar(_t_to_f64(y), (n, Ho, Wo, Co))
    xf, wf = prg._bf16_to_f64(x), prg._bf16_to_f64(w)
    for i in range(n):
        ref = O.conv2d(xf[i], wf, b.astype(np.float64), st, pad)
        if res_mode == 1:
            ref = ref + prg._bf16_to_f64(res[i])
        elif res_mode == 2:
            ref = ref + O.option_a(prg._bf16_to_f64(res[i]), Co)
        if relu:
            ref = O.relu(ref)
        ref = O.round_bf16(ref)
        # fp32 tensor-core accumulation vs fp64: at most one bf16 rounding step apart
        tol = 2.0 ** -7 * np.abs(ref) + 1e-6
        bad = np.abs(got[i] - ref) > tol
        assert not bad.any(), (i, np.argwhere(bad)[:5], got[i][bad][:5], ref[bad][:5])
        assert np.mean(got[i] != ref) < 0.01


# NHWC im2col-TMA GEMM (config-5 layers): flat M across samples with ragged tails
NHWC_CASES = [
    # n, H, W, C, Cout, k, stride, pad, relu, res_mode
    (3, 14, 14, 64, 64, 1, 1, 0, 1, 0),      # 1x1, tiled A box, BN 64, M = 588 (ragged)
    (2, 14, 14, 128, 256, 1, 1, 0, 0, 1),    # 1x1 + identity shortcut, BN 256
    (3, 7, 7, 64, 128, 3, 1, 1, 1, 0),       # 3x3 im2col, 7x7 maps: tiles span 3 samples
    (2, 12, 10, 128, 128, 3, 1, 1, 1, 1),    # non-square, shortcut, two channel blocks
    (3, 14, 14, 64, 128, 3, 2, 1, 1, 0),     # 3x3 stride 2 (stage transition)
    (3, 14, 14, 128, 512, 1, 2, 0, 0, 0),    # 1x1 stride 2 projection, N tiling 2 x 256
    (2, 9, 9, 64, 64, 7, 2, 3, 1, 0),        # 7x7 stride 2 pad 3
    (4, 16, 16, 8, 64, 7, 2, 3, 1, 0),       # stem (C = 8): planar kernels, NHWC output
    (1, 1, 1, 64, 64, 1, 1, 0, 1, 0),        # single row
    # 3x3 / s1 / p1, 64 -> 64: the halo-tile kernel (conv_halo.cu; R output rows per tile, pitch W + 2)
    (2, 56, 56, 64, 64, 3, 1, 1, 1, 0),      # ResNet-50 stage 1: R = 2, P = 58
    (3, 14, 14, 64, 64, 3, 1, 1, 1, 0),      # R = 7, P = 16
    (2, 12, 30, 64, 64, 3, 1, 1, 0, 0),      # non-square, R = 4, P = 32 (128 rows), no ReLU
    (1, 9, 30, 64, 64, 3, 1, 1, 1, 0),       # R = 3 (9 / 3), P = 32
    (2, 8, 8, 64, 64, 3, 1, 1, 1, 0),        # 8 x 8: 80 of 128 rows real -> the im2col GEMM instead
    (2, 11, 47, 16, 64, 4, 1, 2, 1, 0),      # 4x4 / pad 2 over 16 channels (the 2x2 s2d stem's form): R = 2
    (2, 56, 56, 64, 256, 3, 1, 1, 1, 0),     # the 4x4 space-to-depth stem: N = 256 split over CTA pairs
    (3, 14, 14, 64, 128, 3, 1, 1, 0, 0),     # N = 128 in one CTA, R = 7
    (1, 9, 30, 64, 256, 3, 1, 1, 1, 0),      # N split, R = 3, a single sample
]
# row-tap GEMM form (path 5): 3x3 / s1 / p1, whole samples per 128-row tile, W | 32, Cout 64
ROWTAP_NHWC_CASES = [
    (5, 8, 8, 64, 64, 3, 1, 1, 1, 1),        # CIFAR stage 3 + identity shortcut, ragged last tile
    (7, 8, 8, 64, 64, 3, 1, 1, 0, 0),        # odd sample count, no ReLU
    (9, 4, 4, 128, 64, 3, 1, 1, 1, 0),       # 8 samples per tile, two channel blocks per tap
    (3, 8, 16, 64, 64, 3, 1, 1, 1, 1),       # non-square, W = 16
]


@pytest.mark.parametrize("path,case", [(4, c) for c in NHWC_CASES] + [(5, c) for c in ROWTAP_NHWC_CASES],
                         ids=[f"nhwc-{c}" for c in NHWC_CASES] + [f"nhwc-rowtap-{c}" for c in ROWTAP_NHWC_CASES])
def test_conv_gemm_nhwc_matches_oracle_conv(any_graph, path, case):
    n, H, W, C, Co, k, st, pad, relu, res_mode = case
    rng = np.random.default_rng(abs(hash(case)) % 2**32)
    x = wl.f32_to_bf16_bits(rng.standard_normal((n, H, W, C)))
    w = wl.f32_to_bf16_bits(rng.standard_normal((Co, k, k, C)) * np.sqrt(2.0 / (k * k * C)))
    b = rng.uniform(-0.1, 0.1, Co).astype(np.float32)
    Ho, Wo = (H + 2 * pad - k) // st + 1, (W + 2 * pad - k) // st + 1
    res = wl.f32_to_bf16_bits(rng.standard_normal((n, Ho, Wo, Co))) if res_mode == 1 else None
    y = torch.zeros((n, Ho, Wo, Co), dtype=torch.int16, device=DEV)
    D.dycl_debug_conv2d(any_graph, _bits_to_t(x), n, H, W, C, w, b, Co, k, st, pad, relu,
                        _bits_to_t(res) if res is not None else None, res_mode, y, path)
    got = _t_to_f64(y)
    xf, wf = prg._bf16_to_f64(x), prg._bf16_to_f64(w)
    for i in range(n):
        ref = O.conv2d(xf[i], wf, b.astype(np.float64), st, pad)
        if res_mode == 1:
            ref = ref + prg._bf16_to_f64(res[i])
        if relu:
            ref = O.relu(ref)
        ref = O.round_bf16(ref)
        tol = 2.0 ** -7 * np.abs(ref) + 1e-6
        bad = np.abs(got[i] - ref) > tol
        assert not bad.any(), (i, np.argwhere(bad)[:5], got[i][bad][:5], ref[bad][:5])
        assert np.mean(got[i] != ref) < 0.01


def test_conv_kernel_zero_rows(any_graph):
    y = torch.full((1, 4, 4, 16), 7, dtype=torch.int16, device=DEV)
    x = torch.zeros((1, 4, 4, 16), dtype=torch.int16, device=DEV)
    w = np.zeros((16, 3, 3, 16), np.uint16)
    D.dycl_debug_conv2d(any_graph, x, 0, 4, 4, 16, w, np.zeros(16, np.float32), 16, 3, 1, 1, 1, None, 0, y)
    assert torch.all(y == 7)


# ------------------------------------------------------------ whole programs
def _run_gpu(model, X):
    B = X.shape[0]
    x = torch.from_numpy(X).to(DEV)
    logits = torch.full((max(B, 1), model.K), float("nan"), device=DEV)
    path = torch.full((max(B, 1),), -7, dtype=torch.int32, device=DEV)
    model.run(x, logits, path)
    torch.cuda.synchronize()
    return logits[:B].cpu().numpy(), path[:B].cpu().numpy()


@pytest.fixture(scope="module")
def mlp():
    W = wl.mlp_weights()
    return W, P.build_mlp_ee(W, 64)


@pytest.fixture(scope="module")
def r56():
    W = wl.sdn_r56_weights()
    return W, P.build_sdn_resnet56(W, 4096)


@pytest.fixture(scope="module")
def r38():
    W = wl.skipnet_r38_weights()
    return W, P.build_skipnet_resnet38(W, 512)


def _parity(W, model, program, X, **kw):
    lg, pg = _run_gpu(model, X)
    lo, po, pr = O.run_batch(program, X, prg.prepare(W), "mirror", **kw)
    return report(lg, pg, lo, po, pr), lg, pg


def test_cfg1_mlp_parity(mlp):
    W, m = mlp
    X = wl.mlp_inputs(wl.INPUT_SEED, 0, 32)
    r, lg, pg = _parity(W, m, O.mlp_ee, X)
    print("cfg1", r)
    assert r["outside_band_mismatch"] == 0 and r["logit_rel_fail"] == 0
    assert set(np.unique(pg)) <= {0, 1, 2}


@pytest.mark.parametrize("B", [256, 203, 1])
def test_cfg2_sdn_parity(r56, B):
    W, m = r56
    X = wl.image_inputs(wl.INPUT_SEED, 1000, B)
    r, lg, pg = _parity(W, m, O.sdn_resnet56, X)
    print("cfg2", B, r)
    assert r["logit_rel_fail"] == 0
    assert r["outside_band_mismatch"] == 0, r


def test_cfg3_skipnet_parity(r38):
    W, m = r38
    X = wl.image_inputs(wl.INPUT_SEED, 2000, 256)
    r, lg, pg = _parity(W, m, O.skipnet_resnet38, X)
    print("cfg3", r)
    assert r["logit_rel_fail"] == 0
    assert r["outside_band_mismatch"] == 0, r


@pytest.mark.parametrize("cfg", [2, 3])
def test_bf16_storage_mode_vs_mirror_bf16(cfg):
    """DYCL_PREC_BF16 (all-bf16 storage, an opt-in mode BELOW the north star's logit bar) graded
    against the oracle's mirror_bf16 mode.  Decisions must still match bit-exactly outside the
    band.  Its logits drift past 2e-2 (measured 4.2e-2 on cfg2: bf16 rounding of the residual
    stream through 27 blocks, DESIGN R13) -- the reason the production mode is FP32_STREAM, which
    the other tests grade at 2e-2.  Here the drift is measured, reported and bounded at 6e-2."""
    if cfg == 2:
        W = wl.sdn_r56_weights()
        m = P.build_sdn_resnet56(W, 256, precision=D.DYCL_PREC_BF16)
        prog = O.sdn_resnet56
    else:
        W = wl.skipnet_r38_weights()
        m = P.build_skipnet_resnet38(W, 256, precision=D.DYCL_PREC_BF16)
        prog = O.skipnet_resnet38
    X = wl.image_inputs(wl.INPUT_SEED, 3000, 256)
    lg, pg = _run_gpu(m, X)
    lo, po, pr = O.run_batch(prog, X, prg.prepare(W), "mirror_bf16")
    r = report(lg, pg, lo, po, pr, rel=2e-2)
    print("bf16 storage cfg", cfg, r)
    assert r["outside_band_mismatch"] == 0, r
    assert r["max_logit_rel"] <= 6e-2, r


def test_empty_batch(r56):
    W, m = r56
    lg, pg = _run_gpu(m, np.zeros((0, 32, 32, 3), np.float32))
    assert lg.shape == (0, 10) and pg.shape == (0,)


def test_permutation_and_batch_size_invariance(r56):
    """Row i's result is bitwise independent of its batch position and the batch size."""
    W, m = r56
    X = wl.image_inputs(wl.INPUT_SEED, 0, 300)
    l1, p1 = _run_gpu(m, X)
    perm = np.random.default_rng(0).permutation(300)
    l2, p2 = _run_gpu(m, X[perm])
    assert np.array_equal(l2, l1[perm]) and np.array_equal(p2, p1[perm])
    l3, p3 = _run_gpu(m, X[:77])
    assert np.array_equal(l3, l1[:77]) and np.array_equal(p3, p1[:77])


def test_run_host_equals_run(r56):
    W, m = r56
    X = wl.image_inputs(wl.INPUT_SEED, 0, 128)
    l1, p1 = _run_gpu(m, X)
    lh = np.zeros((128, 10), np.float32)
    ph = np.zeros(128, np.int32)
    m.run_host(X, lh, ph)
    assert np.array_equal(lh, l1) and np.array_equal(ph, p1)


def test_run_host_batch_above_max_batch():
    """dycl_run_host with a batch 2.5x the graph's max_batch streams through in max_batch-row
    sub-chunks: bitwise the device runs' results (each sub-chunk run on its own), in input order,
    with global offsets carried (min margins identical)."""
    W = wl.sdn_r56_weights()
    m = P.build_sdn_resnet56(W, 200)
    X = wl.image_inputs(wl.INPUT_SEED, 5000, 500)
    l1, p1 = np.zeros((500, 10), np.float32), np.zeros(500, np.int32)
    for c0 in range(0, 500, 200):
        lg, pg = _run_gpu(m, X[c0:c0 + 200])
        l1[c0:c0 + 200], p1[c0:c0 + 200] = lg, pg
    lh = np.zeros((500, 10), np.float32)
    ph = np.zeros(500, np.int32)
    m.run_host(X, lh, ph)
    assert np.array_equal(lh, l1) and np.array_equal(ph, p1)
    mh = np.zeros(500, np.float32)
    m.run_host(X, lh, ph, global_offset=1000, min_margin=mh)
    assert np.array_equal(lh, l1) and np.array_equal(ph, p1) and np.isfinite(mh).any()


def test_run_host_pipelined_equals_run(r56):
    """A batch the host-buffer path splits into two uneven chunks (768 + 1732 rows): bitwise
    the device run's results, in input order."""
    W, m = r56
    X = wl.image_inputs(wl.INPUT_SEED, 3000, 2500)
    l1, p1 = _run_gpu(m, X)
    lh = np.zeros((2500, 10), np.float32)
    ph = np.zeros(2500, np.int32)
    m.run_host(X, lh, ph)
    assert np.array_equal(lh, l1) and np.array_equal(ph, p1)


def test_cfg2_full_batch_sampled_parity(r56):
    """BASELINE size (B = 4096, the bench launch configuration): sampled rows vs oracle."""
    W, m = r56
    X = wl.image_inputs(wl.INPUT_SEED, 0, 4096)
    lg, pg = _run_gpu(m, X)
    assert np.bincount(pg, minlength=5).sum() == 4096 and np.isfinite(lg).all()
    idx = np.random.default_rng(wl.ORACLE_SUBSET_SEED).choice(4096, 512, replace=False)
    lo, po, pr = O.run_batch(O.sdn_resnet56, X[idx], prg.prepare(W), "mirror")
    r = report(lg[idx], pg[idx], lo, po, pr)
    print("cfg2 full sampled", r)
    assert r["logit_rel_fail"] == 0 and r["outside_band_mismatch"] == 0, r


def test_cfg3_full_batch_sampled_parity():
    """BASELINE size (B = 8192, the bench launch configuration, in-place gates): sampled rows
    vs the oracle, plus the executed-block histogram's sanity."""
    W = wl.skipnet_r38_weights()
    m = P.build_skipnet_resnet38(W, 8192)
    X = wl.image_inputs(wl.INPUT_SEED, 0, 8192)
    lg, pg = _run_gpu(m, X)
    assert np.isfinite(lg).all() and (pg >= 0).all() and (pg < (1 << 17)).all()
    idx = np.random.default_rng(wl.ORACLE_SUBSET_SEED).choice(8192, 512, replace=False)
    lo, po, pr = O.run_batch(O.skipnet_resnet38, X[idx], prg.prepare(W), "mirror")
    r = report(lg[idx], pg[idx], lo, po, pr)
    print("cfg3 full sampled", r, "mean executed", np.mean([bin(int(v)).count("1") for v in pg]))
    assert r["logit_rel_fail"] == 0 and r["outside_band_mismatch"] == 0, r


def test_gates_in_place_equal_gather_merge():
    """The in-place gate form (executed rows rewritten through the row list) and the
    gather / merge form take the same paths; logits agree to fp32 reassociation (the
    in-place form pools through the fused-block GAP, the other through the head's GAP)."""
    import os
    W = wl.skipnet_r38_weights()
    X = wl.image_inputs(wl.INPUT_SEED, 500, 300)
    m1 = P.build_skipnet_resnet38(W, 300)
    lg1, pg1 = _run_gpu(m1, X)
    os.environ["DYCL_NO_INPLACE"] = "1"
    try:
        m2 = P.build_skipnet_resnet38(W, 300)
    finally:
        del os.environ["DYCL_NO_INPLACE"]
    lg2, pg2 = _run_gpu(m2, X)
    print("in place vs gather: path mismatches", int((pg1 != pg2).sum()),
          "max rel", float(np.max(np.abs(lg1 - lg2)) / np.max(np.abs(lg2))))
    assert np.array_equal(pg1, pg2)
    assert np.max(np.abs(lg1 - lg2)) <= 1e-5 * np.max(np.abs(lg2))


def test_zero_copy_exits_equal_gather():
    """Exits before a fused block hand the survivors over by row list (no gather): bitwise
    the same logits and paths as gathering them."""
    import os
    W = wl.sdn_r56_weights()
    X = wl.image_inputs(wl.INPUT_SEED, 900, 333)
    lg1, pg1 = _run_gpu(P.build_sdn_resnet56(W, 333), X)
    os.environ["DYCL_NO_ZERO_COPY"] = "1"
    try:
        m2 = P.build_sdn_resnet56(W, 333)
    finally:
        del os.environ["DYCL_NO_ZERO_COPY"]
    lg2, pg2 = _run_gpu(m2, X)
    assert np.array_equal(pg1, pg2) and np.array_equal(lg1, lg2)


def test_graph_replay_equals_direct_run(r56):
    """dycl_run's captured CUDA graph and the launch-by-launch run agree bitwise, across
    different data with the same io pointers (the graph is data-independent)."""
    import os
    W, m = r56
    B = 512
    x = torch.empty((B, 32, 32, 3), device=DEV)
    logits = torch.empty((B, 10), device=DEV)
    path = torch.empty(B, dtype=torch.int32, device=DEV)
    outs = []
    for start in (0, 7000):
        x.copy_(torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, start, B)))
        m.run(x, logits, path)
        torch.cuda.synchronize()
        outs.append((logits.cpu().numpy().copy(), path.cpu().numpy().copy()))
    os.environ["DYCL_GRAPH"] = "0"
    try:
        m2 = P.build_sdn_resnet56(W, 4096)
    finally:
        del os.environ["DYCL_GRAPH"]
    for k, start in enumerate((0, 7000)):
        x.copy_(torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, start, B)))
        m2.run(x, logits, path)
        torch.cuda.synchronize()
        assert np.array_equal(path.cpu().numpy(), outs[k][1])
        assert np.array_equal(logits.cpu().numpy(), outs[k][0])


# ------------------------------------------------------------------- config 5
@pytest.fixture(scope="module")
def r50():
    W = wl.resnet50_ee_weights()
    return W, P.build_resnet50_ee(W, 64)


def test_gpu_input_generator_matches_numpy():
    a = wl.image_inputs(wl.INPUT_SEED, 123, 3, hw=224)
    b = wl.image_inputs_torch(wl.INPUT_SEED, 123, 3, hw=224, device="cuda").cpu().numpy()
    assert np.array_equal(a, b)


def test_cfg5_resnet50_parity(r50):
    W, m = r50
    X = wl.image_inputs(wl.INPUT_SEED, 4000, 24, hw=224)
    r, lg, pg = _parity(W, m, O.resnet50_ee, X)
    print("cfg5", r)
    assert r["logit_rel_fail"] == 0
    assert r["outside_band_mismatch"] == 0, r


def test_cfg5_bench_chunk_sampled_parity():
    """The bench launch configuration (a graph finalised for 2048-sample chunks, run on a full
    chunk of GPU-generated inputs): 64 sampled rows per exit taken (256) vs the oracle."""
    W = wl.resnet50_ee_weights()
    m = P.build_resnet50_ee(W, 2048)
    x = wl.image_inputs_torch(wl.INPUT_SEED, 10000, 2048, hw=224, device="cuda")
    logits = torch.empty((2048, 1000), device=DEV)
    path = torch.empty(2048, dtype=torch.int32, device=DEV)
    m.run(x, logits, path)
    torch.cuda.synchronize()
    lg, pg = logits.cpu().numpy(), path.cpu().numpy()
    assert np.isfinite(lg).all() and set(np.unique(pg)) <= {0, 1, 2, 3}
    rng = np.random.default_rng(wl.ORACLE_SUBSET_SEED)
    idx = np.sort(np.concatenate([rng.choice(np.nonzero(pg == k)[0], min(64, int((pg == k).sum())), replace=False)
                                  for k in range(4)]))
    assert len(idx) >= 200, np.bincount(pg, minlength=4)
    X = wl.image_inputs(wl.INPUT_SEED, 0, 0, hw=224, idx=10000 + idx)
    lo, po, pr = O.run_batch(O.resnet50_ee, X, prg.prepare(W), "mirror")
    r = report(lg[idx], pg[idx], lo, po, pr)
    print("cfg5 chunk sampled", r)
    assert r["logit_rel_fail"] == 0 and r["outside_band_mismatch"] == 0, r


def test_cfg5_zero_copy_stage_entries_equal_gather():
    """cfg5 exits hand their survivors to the next stage by row list (default: the
    56x56 stage entry, 64-row A / 16-pixel projection boxes; DYCL_ZC_PROJ_MIN=4 adds the 28x28
    entry, 16-row A / 4-pixel projection boxes): bitwise the same logits and paths as gathering
    them, and fewer launches."""
    import os
    from paper_2307_04963_b200 import dycl as D
    W = wl.resnet50_ee_weights()
    B = 384
    x = wl.image_inputs_torch(wl.INPUT_SEED, 20000, B, hw=224, device="cuda")
    outs, launches = [], []
    for env in ({"DYCL_ZC_PROJ_MIN": "4"}, {}, {"DYCL_NO_ZERO_COPY": "1"}):
        os.environ.update(env)
        try:
            m = P.build_resnet50_ee(W, B)
        finally:
            for k in env:
                del os.environ[k]
        logits = torch.empty((B, 1000), device=DEV)
        path = torch.empty(B, dtype=torch.int32, device=DEV)
        m.run(x, logits, path)
        torch.cuda.synchronize()
        outs.append((logits.cpu().numpy(), path.cpu().numpy()))
        launches.append(D.dycl_launches_per_run(m.g))
        m.close()
    print("cfg5 paths", np.bincount(outs[0][1], minlength=4).tolist(), "launches (56x56 + 28x28 / 56x56 / none)", launches)
    assert all((outs[0][1] == k).sum() > 0 for k in range(4))
    for lg, pg in outs[1:]:
        assert np.array_equal(pg, outs[0][1]) and np.array_equal(lg, outs[0][0])
    assert launches[0] < launches[1] < launches[2]


def test_cfg5_empty_and_single():
    W = wl.resnet50_ee_weights()
    m = P.build_resnet50_ee(W, 8)
    X = wl.image_inputs(wl.INPUT_SEED, 321, 1, hw=224)
    lg, pg = _run_gpu(m, X)
    lo, po, pr = O.run_batch(O.resnet50_ee, X, prg.prepare(W), "mirror")
    r = report(lg, pg, lo, po, pr)
    assert r["logit_rel_fail"] == 0 and r["outside_band_mismatch"] == 0
    x0 = torch.empty((0, 224, 224, 3), device=DEV)
    m.run(x0, torch.empty((1, 1000), device=DEV), torch.empty(1, dtype=torch.int32, device=DEV))
    torch.cuda.synchronize()


# ------------------------------------------------------------------- config 4
@pytest.fixture(scope="module")
def s2s_model():
    from oracle import seq2seq as S
    W = wl.seq2seq_weights()
    return W, S.prepare_s2s(W), P.build_seq2seq(W, wl.S2S, 1024)


def _run_s2s(m, src):
    return run_s2s(m, src)


@pytest.mark.parametrize("B", [8, 5, 1])
def test_cfg4_seq2seq_parity(s2s_model, B):
    W, P_, m = s2s_model
    src = wl.token_inputs(wl.INPUT_SEED, 100, B)
    tok, ln, top1, z0 = _run_s2s(m, src)
    assert ((ln >= 1) & (ln <= 64)).all()
    for i in range(B):                              # PAD after the end, EOS at the end (unless 64)
        assert np.all(tok[i, ln[i]:] == wl.S2S["pad"])
        if ln[i] < 64:
            assert tok[i, ln[i] - 1] == wl.S2S["eos"]
    rep = compare_free_running(P_, src, tok, ln, top1, z0)
    print("cfg4", B, rep)
    assert rep["max_top1_rel"] <= 2e-2 and rep["max_z0_rel"] <= 2e-2, rep
    # production mode: a free-running divergence must come from a counted token flip whose
    # oracle margin (the oracle fed the GPU's own prefix) is inside the bf16 storage-noise floor;
    # every other teacher-forced step matches (bit-exact decisions are the BF16X3 mode's bar)
    if rep["mismatch"]:
        bad = rep["mismatch_idx"]
        tf = compare_teacher_forced(P_, src[bad], tok[bad], ln[bad], top1[bad])
        print("cfg4", B, "teacher-forced on the diverged sequences", tf)
        assert tf["step_mismatch"] >= 1 and tf["max_flip_margin"] < FLIP_NOISE_MARGIN, tf


def test_cfg4_full_batch_sampled_parity(s2s_model):
    """The bench launch configuration (1024 sequences), PRODUCTION bf16 mode: 128 sampled
    sequences free-running (tokens, lengths, top-1 logits) and 32 teacher-forced (every step's
    decision re-derived by the oracle from the GPU's own prefix) vs the mirror oracle.
    bf16 storage of q/k/v, K/V caches and attention outputs puts ~3e-3 relative noise on the
    logits, above the 1e-3 token band, so rare outside-band flips are expected here (measured
    2-4/128 sequences, 3-11/1014 teacher-forced steps, ~1 %) and are COUNTED (SURVEY 8(c) ladder: the bf16
    production mode is graded on logits <= 2e-2 and an outside-band mismatch count); bit-exact
    decisions are the BF16X3 parity mode's bar (test_cfg4_bf16x3_parity_mode_vs_exact)."""
    W, P_, m = s2s_model
    src = wl.token_inputs(wl.INPUT_SEED, 0, 1024)
    tok, ln, top1, z0 = _run_s2s(m, src)
    idx = np.sort(np.random.default_rng(wl.ORACLE_SUBSET_SEED).choice(1024, 128, replace=False))
    rep = compare_free_running(P_, src[idx], tok[idx], ln[idx], top1[idx], z0[idx])
    print("cfg4 full sampled", rep, "mean length", ln.mean())
    assert rep["mismatch"] <= 8 and rep["max_top1_rel"] <= 2e-2 and rep["max_z0_rel"] <= 2e-2, rep
    tf = compare_teacher_forced(P_, src[idx[:32]], tok[idx[:32]], ln[idx[:32]], top1[idx[:32]])
    print("cfg4 teacher forced", tf)
    assert tf["step_mismatch"] <= 0.02 * tf["steps"] and tf["max_top1_rel"] <= 2e-2, tf
    assert tf["max_flip_margin"] < FLIP_NOISE_MARGIN, tf
    # batch-position independence: a permuted sub-batch decodes identically
    perm = np.random.default_rng(1).permutation(64)
    tok2, ln2, _, _ = _run_s2s(m, src[:64][perm])
    assert np.array_equal(tok2, tok[:64][perm]) and np.array_equal(ln2, ln[:64][perm])
    th = np.zeros((64, 64), np.int32)
    lh = np.zeros(64, np.int32)
    m.run_host(src[:64], th, lh)
    assert np.array_equal(th, tok[:64]) and np.array_equal(lh, ln[:64])


@pytest.fixture(scope="module")
def s2s_parity_model():
    W = wl.seq2seq_weights()
    return W, P.build_seq2seq(W, wl.S2S, 1024, precision=D.DYCL_PREC_BF16X3_PARITY)


def test_cfg4_bf16x3_parity_mode_vs_exact(s2s_model, s2s_parity_model):
    """DYCL_PREC_BF16X3_PARITY (split-bf16 tensor-core products, fp32-accurate) graded against the
    oracle's EXACT (fp64) mode on the bench batch: tokens and lengths bit-exact outside the 1e-3
    band for 128 free-running and 32 teacher-forced sequences, top-1 logits within 1e-3."""
    from oracle import seq2seq as S
    W, m = s2s_parity_model
    P_ = s2s_model[1]
    src = wl.token_inputs(wl.INPUT_SEED, 0, 1024)
    tok, ln, top1, z0 = _run_s2s(m, src)
    idx = np.sort(np.random.default_rng(wl.ORACLE_SUBSET_SEED).choice(1024, 128, replace=False))
    rep = compare_free_running(P_, src[idx], tok[idx], ln[idx], top1[idx], z0[idx], mode="exact")
    print("cfg4 bf16x3 vs exact", rep)
    assert rep["mismatch"] == 0 and rep["max_top1_rel"] <= 1e-3 and rep["max_z0_rel"] <= 1e-3, rep
    tf = compare_teacher_forced(P_, src[idx[:32]], tok[idx[:32]], ln[idx[:32]], top1[idx[:32]], mode="exact")
    print("cfg4 bf16x3 teacher forced vs exact", tf)
    assert tf["step_mismatch"] == 0 and tf["max_top1_rel"] <= 1e-3, tf
    assert S is not None
