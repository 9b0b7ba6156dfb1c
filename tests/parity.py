"""Parity report: CUDA path vs oracle, per the north star's bar (tests only).

* decisions (path words) bit-exact for every sample whose predicates along the
  oracle's path are all outside the 1e-3 band (reading R11); band samples counted;
* logits within 2e-2 relative (L-inf, reading R12) for non-excluded samples;
* delta / eta per Eq. 1 reported.
"""
import numpy as np

from oracle.metrics import delta, eta, in_band


def report(gpu_logits, gpu_path, ora_logits, ora_path, ora_preds, band=1e-3, rel=2e-2):
    gpu_logits = np.asarray(gpu_logits, np.float64)
    n = len(ora_path)
    excl = np.array([in_band(p, band) for p in ora_preds], dtype=bool) if n else np.zeros(0, bool)
    pm = np.asarray(gpu_path) != np.asarray(ora_path)
    outside = pm & ~excl
    ok = ~excl & ~pm
    relerr = np.zeros(n)
    for i in np.nonzero(ok)[0]:
        relerr[i] = np.max(np.abs(gpu_logits[i] - ora_logits[i])) / max(np.max(np.abs(ora_logits[i])), 1e-30)
    return dict(
        n=n,
        band_excluded=int(excl.sum()),
        outside_band_mismatch=int(outside.sum()),
        mismatch_idx=np.nonzero(outside)[0].tolist(),
        max_logit_rel=float(relerr.max()) if n else 0.0,
        logit_rel_fail=int((relerr > rel).sum()),
        delta=delta(list(gpu_logits[ok]), list(np.asarray(ora_logits)[ok])) if ok.any() else -10.0,
        eta=eta(list(np.argmax(gpu_logits, 1)), list(np.argmax(ora_logits, 1))) if n else 0.0,
        path_hist=np.bincount(np.asarray(gpu_path) if np.asarray(gpu_path).max(initial=0) < 64 else [0]).tolist(),
    )
