"""Large-sample parity evidence (GPU box): the CUDA path in the bench launch configuration vs
the oracle on many seeded samples, stratified across exits for cfg5, free-running and
teacher-forced for cfg4.  Decisions must match bit-exactly outside the 1e-3 band (R12).

  python tools/parity_large.py [cfgs=2,3,5,4] [out.json]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as wl  # noqa: E402
from oracle import programs as prg  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402
from tests.parity import report  # noqa: E402

DEV = torch.device("cuda:0")


def run_img(model, x, K):
    B = x.shape[0]
    lg = torch.empty((B, K), device=DEV)
    pa = torch.empty(B, dtype=torch.int32, device=DEV)
    model.run(x, lg, pa)
    torch.cuda.synchronize()
    return lg.cpu().numpy(), pa.cpu().numpy()


def stratified(path, per, rng, n_classes):
    idx = []
    for k in range(n_classes):
        cand = np.nonzero(path == k)[0]
        if len(cand):
            idx.extend(rng.choice(cand, min(per, len(cand)), replace=False).tolist())
    return np.sort(np.array(idx, dtype=np.int64))


def main():
    cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "2,3,5,4").split(",")]
    outp = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/parity_large.json"
    out = {}
    rng = np.random.default_rng(wl.ORACLE_SUBSET_SEED)
    for cfg in cfgs:
        t0 = time.time()
        if cfg in (2, 3):
            W = wl.sdn_r56_weights() if cfg == 2 else wl.skipnet_r38_weights()
            B = 4096 if cfg == 2 else 8192
            m = (P.build_sdn_resnet56 if cfg == 2 else P.build_skipnet_resnet38)(W, B)
            X = wl.image_inputs(wl.INPUT_SEED, 0, B)
            lg, pg = run_img(m, torch.from_numpy(X).to(DEV), 10)
            idx = np.sort(rng.choice(B, 512, replace=False))
            lo, po, pr = O.run_batch(O.sdn_resnet56 if cfg == 2 else O.skipnet_resnet38, X[idx], prg.prepare(W),
                                     "mirror")
            out[f"cfg{cfg}"] = dict(report(lg[idx], pg[idx], lo, po, pr), batch=B, sampled=len(idx))
        elif cfg == 5:
            W = wl.resnet50_ee_weights()
            m = P.build_resnet50_ee(W, 2048)
            x = wl.image_inputs_torch(wl.INPUT_SEED, 0, 2048, hw=224, device="cuda")
            lg, pg = run_img(m, x, 1000)
            idx = stratified(pg, 64, rng, 4)
            X = wl.image_inputs(wl.INPUT_SEED, 0, 0, hw=224, idx=idx)
            lo, po, pr = O.run_batch(O.resnet50_ee, X, prg.prepare(W), "mirror")
            r = report(lg[idx], pg[idx], lo, po, pr)
            out["cfg5"] = dict(r, batch=2048, sampled=len(idx), stratified="64 per GPU exit")
        elif cfg == 4:
            from tests.s2s_parity import s2s_free_running, s2s_teacher_forced
            W = wl.seq2seq_weights()
            m4 = P.build_seq2seq(W, wl.S2S, 1024)
            src = wl.token_inputs(wl.INPUT_SEED, 0, 1024)
            idx = np.sort(rng.choice(1024, 128, replace=False))
            out["cfg4"] = s2s_free_running(m4, W, src, idx)
            out["cfg4_teacher_forced"] = s2s_teacher_forced(m4, W, src, idx[:32])
        out[f"cfg{cfg}"]["wall_s"] = round(time.time() - t0, 1)
        print(cfg, json.dumps(out[f"cfg{cfg}"]), flush=True)
    json.dump(out, open(outp, "w"), indent=1)


if __name__ == "__main__":
    main()
