"""Negative tests: what the method exists to prevent must be caught.

* Trace baseline (Table 2; §3.3): a DyNN converted by tracing
  keeps only the path one example took -- every predicate frozen to that example's decision.
  Run on other inputs it is no longer the dynamic program: eta > 0 against the oracle's
  dynamic run, while every input that happens to take the traced path agrees exactly.
  (DyCL's claim, Eq. 2, is the opposite: eta == 0 for every input.)
* An unstable compaction (survivors reordered inside an exit group) must fail the parity
  report's ordering check (tests/parity.report), which is what the GPU tests rely on.
CPU only: the oracle and the host-side checker.
"""
import numpy as np

import oracle as O
import workloads as wl
from oracle import programs as prg
from oracle.metrics import eta
from tests.parity import report


def _cfg1(n):
    W = wl.mlp_weights()
    X = wl.mlp_inputs(wl.INPUT_SEED, 0, n)
    return X, prg.prepare(W)


def test_traced_program_is_not_the_dynamic_program():
    X, P = _cfg1(256)
    lo, po, _ = O.run_batch(O.mlp_ee, X, P, "exact", threads=1)
    assert len(set(po.tolist())) == 3, np.bincount(po)          # every exit taken by some input
    # trace on the first input that ran to the final head (a "hard" example): every predicate
    # frozen to "do not exit" -- the static network (tau > 1 leaves no exit taken)
    k0 = int(np.nonzero(po == 2)[0][0])
    lt, pt, _ = O.run_batch(O.mlp_ee, X, P, "exact", threads=1, tau=1.5)
    assert np.all(pt == 2)
    same = po == 2
    assert same[k0]
    # inputs on the traced path: identical outputs (the trace is right for them) ...
    assert np.array_equal(lt[same], lo[same])
    # ... the rest get the final head's logits instead of their exit head's: inconsistent
    e = eta(list(np.argmax(lt, 1)), list(np.argmax(lo, 1)))
    assert e > 0.0
    assert np.all(np.max(np.abs(lt[~same] - lo[~same]), axis=1) > 0)
    # and a trace on an easy example (exits at head 0: tau below 1/K) is wrong the other way
    lf, pf, _ = O.run_batch(O.mlp_ee, X, P, "exact", threads=1, tau=0.05)
    first = po == 0
    assert np.all(pf == 0) and np.array_equal(lf[first], lo[first])
    assert eta(list(np.argmax(lf, 1)), list(np.argmax(lo, 1))) > 0.0


def test_unstable_compaction_fails_the_ordering_check():
    X, P = _cfg1(64)
    lo, po, pr = O.run_batch(O.mlp_ee, X, P, "mirror", threads=1)
    ok = report(lo, po, lo, po, pr)
    assert ok["outside_band_mismatch"] == 0 and ok["logit_rel_fail"] == 0
    # an unstable compaction: two survivors of the same exit written back in swapped order
    for k in range(3):
        idx = np.nonzero(po == k)[0]
        if len(idx) < 2:
            continue
        a, b = idx[0], idx[-1]
        lg, pg = lo.copy(), po.copy()
        lg[[a, b]] = lg[[b, a]]
        r = report(lg, pg, lo, po, pr)
        assert r["logit_rel_fail"] >= 1, (k, r)                  # the paths agree; the logits do not
    # survivors of different exits swapped: the decision check catches it
    a, b = int(np.nonzero(po == 0)[0][0]), int(np.nonzero(po == 2)[0][0])
    lg, pg = lo.copy(), po.copy()
    lg[[a, b]] = lg[[b, a]]
    pg[[a, b]] = pg[[b, a]]
    r = report(lg, pg, lo, po, pr)
    assert r["outside_band_mismatch"] >= 1 or r["band_excluded"] >= 1, r
