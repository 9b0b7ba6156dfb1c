"""Parity evidence for profiles/: every config's CUDA path (through the C ABI, in the bench's
launch configuration where it differs) against the CPU oracle on seeded samples.  Decisions
must match bit-exactly outside the 1e-3 band (reading R12), logits within 2e-2 relative (R13).

  python tools/parity_report.py [out.json]        (GPU box; a few minutes of oracle CPU time)
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import workloads as wl  # noqa: E402
from oracle import programs as prg  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402
from tests.parity import report  # noqa: E402

DEV = torch.device("cuda:0")


def run_img(model, X, K):
    B = X.shape[0]
    x = torch.from_numpy(X).to(DEV)
    lg = torch.empty((B, K), device=DEV)
    pa = torch.empty(B, dtype=torch.int32, device=DEV)
    model.run(x, lg, pa)
    torch.cuda.synchronize()
    return lg.cpu().numpy(), pa.cpu().numpy()


def main():
    out = {}
    t0 = time.time()
    rng = np.random.default_rng(wl.ORACLE_SUBSET_SEED)
    # cfg 1: the whole bench batch
    W = wl.mlp_weights()
    X = wl.mlp_inputs(wl.INPUT_SEED, 0, 32)
    lg, pg = run_img(P.build_mlp_ee(W, 32), X, 10)
    lo, po, pr = O.run_batch(O.mlp_ee, X, prg.prepare(W), "mirror", threads=1)
    out["cfg1"] = dict(report(lg, pg, lo, po, pr), batch=32, sampled="all")
    # cfg 2 / 3: the bench batch, sampled rows
    for cfg, builder, prog, B, Wf, ns in [(2, P.build_sdn_resnet56, O.sdn_resnet56, 4096, wl.sdn_r56_weights, 128),
                                          (3, P.build_skipnet_resnet38, O.skipnet_resnet38, 8192,
                                           wl.skipnet_r38_weights, 96)]:
        W = Wf()
        X = wl.image_inputs(wl.INPUT_SEED, 0, B)
        lg, pg = run_img(builder(W, B), X, 10)
        idx = np.sort(rng.choice(B, ns, replace=False))
        lo, po, pr = O.run_batch(prog, X[idx], prg.prepare(W), "mirror")
        out[f"cfg{cfg}"] = dict(report(lg[idx], pg[idx], lo, po, pr), batch=B, sampled=int(ns))
    # cfg 5: one bench chunk (2048, GPU-generated inputs), sampled rows
    W = wl.resnet50_ee_weights()
    m = P.build_resnet50_ee(W, 2048)
    x = wl.image_inputs_torch(wl.INPUT_SEED, 0, 2048, hw=224, device="cuda")
    lg_t = torch.empty((2048, 1000), device=DEV)
    pa_t = torch.empty(2048, dtype=torch.int32, device=DEV)
    m.run(x, lg_t, pa_t)
    torch.cuda.synchronize()
    lg, pg = lg_t.cpu().numpy(), pa_t.cpu().numpy()
    idx = np.sort(rng.choice(2048, 24, replace=False))
    X = wl.image_inputs(wl.INPUT_SEED, 0, 0, hw=224, idx=idx)
    lo, po, pr = O.run_batch(O.resnet50_ee, X, prg.prepare(W), "mirror")
    out["cfg5"] = dict(report(lg[idx], pg[idx], lo, po, pr), batch=2048, sampled=24)
    # cfg 4: the bench batch, sampled sequences (tokens / lengths / top-1 logits)
    from concurrent.futures import ThreadPoolExecutor
    from oracle import seq2seq as S
    from oracle.metrics import in_band
    W = wl.seq2seq_weights()
    P_ = S.prepare_s2s(W)
    m4 = P.build_seq2seq(W, wl.S2S, 1024)
    src = wl.token_inputs(wl.INPUT_SEED, 0, 1024)
    L, V = wl.S2S["max_len"], wl.S2S["vocab"]
    s_t = torch.from_numpy(src).to(DEV)
    tok = torch.empty((1024, L), dtype=torch.int32, device=DEV)
    ln = torch.empty(1024, dtype=torch.int32, device=DEV)
    top1 = torch.empty((1024, L), device=DEV)
    z0 = torch.empty((1024, V), device=DEV)
    m4.run(s_t, tok, ln, top1, z0)
    torch.cuda.synchronize()
    tok, ln, top1, z0 = tok.cpu().numpy(), ln.cpu().numpy(), top1.cpu().numpy(), z0.cpu().numpy()
    idx = np.sort(rng.choice(1024, 16, replace=False))
    with ThreadPoolExecutor(8) as ex:
        res = list(ex.map(lambda i: S.greedy_decode(src[i], P_, wl.S2S, "mirror"), idx))
    rep = dict(n=len(idx), band_excluded=0, mismatch=0, max_top1_rel=0.0, max_z0_rel=0.0)
    for j, i in enumerate(idx):
        o_tok, o_len, o_top1, o_z0, preds = res[j]
        rep["max_z0_rel"] = max(rep["max_z0_rel"], float(np.max(np.abs(z0[i] - o_z0)) / np.max(np.abs(o_z0))))
        if in_band(preds):
            rep["band_excluded"] += 1
            continue
        if not (np.array_equal(tok[i], o_tok) and ln[i] == o_len):
            rep["mismatch"] += 1
            continue
        k = o_len
        rep["max_top1_rel"] = max(rep["max_top1_rel"], float(
            np.max(np.abs(top1[i, :k] - o_top1[:k]) / np.maximum(1.0, np.abs(o_top1[:k])))))
    out["cfg4"] = dict(rep, batch=1024, sampled=16, mean_length=float(ln.mean()))
    for v in out.values():
        v.pop("mismatch_idx", None)
    out["_bar"] = ("decisions bit-exact outside the 1e-3 band (R12); logits <= 2e-2 relative L-inf (R13); "
                   "oracle = per-sample fp64 interpreter, mirror mode")
    out["_wall_s"] = round(time.time() - t0, 1)
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_report.json"
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
