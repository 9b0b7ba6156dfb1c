"""Freeze the calibration constants of the synthetic models (run once, committed output).

TEST INFRASTRUCTURE: this script calls only oracle/ (and the seeded generator
``workloads``); it writes workloads/calib/cfg{2,3}.json, which both the CUDA
path and the oracle then read as model parameters.  No value here comes from
the CUDA path.

Why: random-init weights make every predicate degenerate (0 %
of samples exit, gates all ~0.5), so the dynamic path would never branch.
Recipe (SURVEY.md §8(d) "Calibration"), on 512 calibration
samples drawn with seed CALIB_SEED=2 (disjoint from the measured inputs):

* config 2 exit heads k=0..3: logits = w (g - mu_k), w = bf16(s_k H_k), with
  mu_k the calibration mean of the pooled features g at that IC and s_k found
  by bisection so that 25 % of the samples ARRIVING at head k exit
  (conf >= tau = 0.9); final head: s = 4, centred the same way.
* config 3 gates i=2..18, calibrated in order along the dynamic path:
  raw r = H_i . g, a_i = median(r), s_i = 2 / std(r); gate logit
  z = bf16(s_i H_i) . g - s_i a_i  (~50 % execute); final head s = 4, centred.

* SkipNet with recurrent gates (cfg3r, reading R19): as config 3 but on the raw LSTM output
  r = w_out . h after each gate's cell step; out_i = (s_i w_out, -s_i a_i) in fp32.

* captioning En-Decoder (cfg4c, reading R20): EOS output bias by bisection, mean length ~12.

Usage:  python -m oracle.calibrate [--n 512] [--cfg 2 3 3r 4c 5]
"""
from __future__ import annotations

import argparse
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import workloads as wl

from . import programs as prg
from .core import dense, gap, max_softmax, sigmoid


def _pool():
    return ThreadPoolExecutor(max_workers=len(os.sched_getaffinity(0)))


def calibrate_cfg2(n: int, mode: str = "mirror") -> dict:
    X = wl.image_inputs(wl.CALIB_SEED, 0, n)
    P = prg.prepare(wl.sdn_r56_weights(calib={
        k: {"scale": 1.0, "mu": [0.0] * c} for k, c in
        [("ic0", 16), ("ic1", 32), ("ic2", 32), ("ic3", 64), ("final", 64)]}))

    def feats(i):
        f = []
        prg.sdn_resnet56(X[i], P, mode, tau=2.0, features=f)   # tau > 1: never exits
        return f

    with _pool() as ex:
        F = list(ex.map(feats, range(n)))
    names = ["ic0", "ic1", "ic2", "ic3", "final"]
    G = {nm: np.stack([f[j] for f in F]) for j, nm in enumerate(names)}
    raw = wl.sdn_r56_raw_heads()
    out = {}
    arriving = np.ones(n, dtype=bool)
    for k in range(4):
        nm = f"ic{k}"
        g = G[nm]
        mu = g.mean(axis=0)

        def exits(s):
            w, b = wl._centered_head(raw[nm], s, mu)
            wf = prg._bf16_to_f64(w)
            conf = np.array([max_softmax(dense(wf, b, gi)) for gi in g])
            return conf >= wl.EXIT_TAU

        lo, hi = np.log(0.01), np.log(1000.0)
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            frac = exits(np.exp(mid))[arriving].mean()
            if frac < 0.25:
                lo = mid
            else:
                hi = mid
        s = float(np.exp(hi))
        ex_k = exits(s)
        out[nm] = {"scale": s, "mu": [float(v) for v in mu],
                   "exit_frac_of_arriving": float(ex_k[arriving].mean()),
                   "arriving": int(arriving.sum())}
        arriving &= ~ex_k
    out["final"] = {"scale": 4.0, "mu": [float(v) for v in G["final"].mean(axis=0)],
                    "arriving": int(arriving.sum())}
    out["_recipe"] = ("oracle/calibrate.py calibrate_cfg2: n=%d calibration samples "
                      "(seed %d), mode=%s, target 25%% exits of arriving, tau=%.2f"
                      % (n, wl.CALIB_SEED, mode, wl.EXIT_TAU))
    return out


def calibrate_cfg3(n: int, mode: str = "mirror") -> dict:
    X = wl.image_inputs(wl.CALIB_SEED, 0, n)
    W = wl.skipnet_r38_weights(calib=None)
    P = prg.prepare(W)
    raw = wl.skipnet_r38_raw_gates()
    with _pool() as ex:
        H = list(ex.map(lambda i: prg.basic_block(prg.stem(X[i], P, mode), P, 1, 6, mode), range(n)))
        out = {}
        executed = []
        for i in wl.SKIP_GATED:
            g = np.stack([gap(h) for h in H])
            r = g @ raw[f"gate{i}"][0]
            a = float(np.median(r))
            s = float(2.0 / r.std())
            w = prg._bf16_to_f64(wl.f32_to_bf16_bits(s * raw[f"gate{i}"]))[0]
            z = g @ w - s * a
            run = sigmoid(z) > 0.5
            executed.append(float(run.mean()))
            out[f"gate{i}"] = {"scale": s, "median": a, "exec_frac": float(run.mean())}
            ci, co, stride = prg._block_io(i, 6)

            def step(j, i=i, run=run, co=co, stride=stride):
                if run[j]:
                    return prg.basic_block(H[j], P, i, 6, mode)
                return prg.option_a(H[j], co) if stride == 2 else H[j]

            H = list(ex.map(step, range(n)))
    out["final"] = {"scale": 4.0, "mu": [float(v) for v in np.stack([gap(h) for h in H]).mean(axis=0)]}
    out["_recipe"] = ("oracle/calibrate.py calibrate_cfg3: n=%d calibration samples (seed %d), "
                      "mode=%s, gates in path order, a=median, s=2/std; mean executed %.2f/17"
                      % (n, wl.CALIB_SEED, mode, sum(executed)))
    return out


def calibrate_cfg3r(n: int, mode: str = "mirror") -> dict:
    """SkipNet with the recurrent gate (reading R19): gates in path order; per gate the raw
    output r = w_out . hs of the LSTM state after this gate's step, a = median(r), s = 2/std(r);
    the program's gate logit is then (s w_out)_fp32 . hs + (-s a)_fp32 (~50 % execute)."""
    X = wl.image_inputs(wl.CALIB_SEED, 0, n)
    W = wl.skipnet_rnn_r38_weights(calib=None)
    P = prg.prepare(W)
    raw = wl.skipnet_rnn_r38_raw()
    Hd = int(P["rnn.hidden"])
    with _pool() as ex:
        H = list(ex.map(lambda i: prg.basic_block(prg.stem(X[i], P, mode), P, 1, 6, mode), range(n)))
        hs = [np.zeros(Hd) for _ in range(n)]
        cs = [np.zeros(Hd) for _ in range(n)]
        out = {}
        executed = []
        for i in wl.SKIP_GATED:
            for j in range(n):
                u = dense(P[f"proj{i}.w"], P[f"proj{i}.b"], gap(H[j]))
                hs[j], cs[j] = prg.lstm_cell(u, hs[j], cs[j], P)
            r = np.array([raw["w_out"] @ h for h in hs])
            a = float(np.median(r))
            s = float(2.0 / r.std())
            w = np.float32(s * raw["w_out"]).astype(np.float64)
            b = float(np.float32(-s * a))
            run = np.array([sigmoid(w @ h + b) > 0.5 for h in hs])
            executed.append(float(run.mean()))
            out[f"gate{i}"] = {"scale": s, "median": a, "exec_frac": float(run.mean())}
            ci, co, stride = prg._block_io(i, 6)

            def step(j, i=i, run=run, co=co, stride=stride):
                if run[j]:
                    return prg.basic_block(H[j], P, i, 6, mode)
                return prg.option_a(H[j], co) if stride == 2 else H[j]

            H = list(ex.map(step, range(n)))
    out["final"] = {"scale": 4.0, "mu": [float(v) for v in np.stack([gap(h) for h in H]).mean(axis=0)]}
    out["_recipe"] = ("oracle/calibrate.py calibrate_cfg3r: n=%d calibration samples (seed %d), "
                      "mode=%s, recurrent gates in path order, a=median, s=2/std of w_out . h; mean executed "
                      "%.2f/17" % (n, wl.CALIB_SEED, mode, sum(executed)))
    return out


def calibrate_cfg4c(n: int, mode: str = "mirror", target: float = 12.0) -> dict:
    """Captioning En-Decoder (reading R20): the EOS output bias by bisection so the mean
    greedy caption length of n calibration images is ~target (of max_len 32)."""
    from . import caption as C
    X = wl.image_inputs(wl.CALIB_SEED, 0, n)
    P = prg.prepare(wl.caption_weights(calib={"eos_bias": 0.0}))
    with _pool() as ex:
        A = list(ex.map(lambda i: C.encode(X[i], P, mode), range(n)))

        def mean_len(b):
            return float(np.mean(list(ex.map(lambda a: C.decode(a, P, wl.CAP, mode, eos_bias=b)[1], A))))

        lo, hi = -20.0, 40.0                    # mean length decreases with the bias
        for _ in range(30):
            mid = 0.5 * (lo + hi)
            if mean_len(mid) > target:
                lo = mid
            else:
                hi = mid
        b = float(np.float32(0.5 * (lo + hi)))
        ml = mean_len(b)
    return {"eos_bias": b, "mean_length": ml,
            "_recipe": "oracle/calibrate.py calibrate_cfg4c: n=%d calibration images (seed %d), mode=%s, EOS "
                       "output bias by bisection to a mean greedy caption length of %.1f" % (n, wl.CALIB_SEED, mode,
                                                                                          target)}


def calibrate_cfg5(n: int, mode: str = "mirror") -> dict:
    """Config 5 heads (exits after stages 1-3, 1000 classes): same recipe as config 2."""
    X = wl.image_inputs(wl.CALIB_SEED, 0, n, hw=224)
    P = prg.prepare(wl.resnet50_ee_weights(calib={
        k: {"scale": 1.0, "mu": [0.0] * c} for k, c in [("ic0", 256), ("ic1", 512), ("ic2", 1024), ("final", 2048)]}))

    def feats(i):
        f = []
        prg.resnet50_ee(X[i], P, mode, tau=2.0, features=f)
        return f

    with _pool() as ex:
        F = list(ex.map(feats, range(n)))
    names = ["ic0", "ic1", "ic2", "final"]
    G = {nm: np.stack([f[j] for f in F]) for j, nm in enumerate(names)}
    raw = wl.r50_raw_heads()
    out = {}
    arriving = np.ones(n, dtype=bool)
    for k in range(3):
        nm = f"ic{k}"
        g = G[nm]
        mu = g.mean(axis=0)

        def exits(s):
            w, b = wl._centered_head(raw[nm], s, mu)
            wf = prg._bf16_to_f64(w)
            conf = np.array([max_softmax(dense(wf, b, gi)) for gi in g])
            return conf >= wl.EXIT_TAU

        lo, hi = np.log(0.01), np.log(1000.0)
        for _ in range(50):
            mid = 0.5 * (lo + hi)
            if exits(np.exp(mid))[arriving].mean() < 0.25:
                lo = mid
            else:
                hi = mid
        s = float(np.exp(hi))
        ex_k = exits(s)
        out[nm] = {"scale": s, "mu": [float(v) for v in mu],
                   "exit_frac_of_arriving": float(ex_k[arriving].mean()), "arriving": int(arriving.sum())}
        arriving &= ~ex_k
    out["final"] = {"scale": 4.0, "mu": [float(v) for v in G["final"].mean(axis=0)], "arriving": int(arriving.sum())}
    out["_recipe"] = ("oracle/calibrate.py calibrate_cfg5: n=%d calibration samples (seed %d), 224x224, mode=%s, "
                      "target 25%% exits of arriving, tau=%.2f" % (n, wl.CALIB_SEED, mode, wl.EXIT_TAU))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--cfg", nargs="*", default=["2", "3"], help="2 3 3r 5")
    ap.add_argument("--n5", type=int, default=128)
    a = ap.parse_args()
    os.makedirs(os.path.join(wl.HERE, "calib"), exist_ok=True)
    for c in a.cfg:
        res = {"2": lambda: calibrate_cfg2(a.n), "3": lambda: calibrate_cfg3(a.n), "3r": lambda: calibrate_cfg3r(a.n), "4c": lambda: calibrate_cfg4c(64),
               "5": lambda: calibrate_cfg5(a.n5)}[str(c)]()
        path = os.path.join(wl.HERE, "calib", f"cfg{c}.json")
        with open(path, "w") as f:
            json.dump(res, f, indent=1)
        print("wrote", path, res.get("_recipe"))


if __name__ == "__main__":
    main()
