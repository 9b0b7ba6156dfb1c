"""Config-4 parity helpers (tests only): the CUDA decode vs the oracle's per-sequence greedy
decode, free-running and teacher-forced ("the oracle recomputes each step from
the GPU's own prefix").  Decisions are graded outside the 1e-3 band (reading R12)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

import workloads as wl
from oracle import seq2seq as S
from oracle.metrics import in_band

_P_CACHE = {}


def _prep(W):
    if id(W) not in _P_CACHE:
        _P_CACHE[id(W)] = S.prepare_s2s(W)
    return _P_CACHE[id(W)]


def run_s2s(m, src, dev="cuda:0"):
    B = src.shape[0]
    L, V = wl.S2S["max_len"], wl.S2S["vocab"]
    s = torch.from_numpy(np.ascontiguousarray(src)).to(dev)
    tok = torch.full((B, L), -5, dtype=torch.int32, device=dev)
    ln = torch.full((B,), -5, dtype=torch.int32, device=dev)
    top1 = torch.empty((B, L), device=dev)
    z0 = torch.empty((B, V), device=dev)
    m.run(s, tok, ln, top1, z0)
    torch.cuda.synchronize()
    return tok.cpu().numpy(), ln.cpu().numpy(), top1.cpu().numpy(), z0.cpu().numpy()


def _threads():
    return max(1, len(os.sched_getaffinity(0)))


def compare_free_running(P_, src, tok, ln, top1, z0, mode="mirror"):
    """Oracle free-running decode per sequence vs the GPU's tokens / lengths / top-1 logits."""
    with ThreadPoolExecutor(_threads()) as ex:
        res = list(ex.map(lambda i: S.greedy_decode(src[i], P_, wl.S2S, mode), range(len(src))))
    rep = dict(n=len(src), band_excluded=0, mismatch=0, max_top1_rel=0.0, max_z0_rel=0.0, mismatch_idx=[])
    for i, (o_tok, o_len, o_top1, o_z0, preds) in enumerate(res):
        rel0 = np.max(np.abs(z0[i] - o_z0)) / np.max(np.abs(o_z0))
        rep["max_z0_rel"] = max(rep["max_z0_rel"], float(rel0))
        if in_band(preds):
            rep["band_excluded"] += 1
            continue
        if not (np.array_equal(tok[i], o_tok) and ln[i] == o_len):
            rep["mismatch"] += 1
            rep["mismatch_idx"].append(i)
            continue
        k = o_len
        r = np.max(np.abs(top1[i, :k] - o_top1[:k]) / np.maximum(1.0, np.abs(o_top1[:k])))
        rep["max_top1_rel"] = max(rep["max_top1_rel"], float(r))
    return rep


# bf16 storage noise of the production mode on the LM logits (measured ~3e-3 relative, DESIGN.md
# R13 / SURVEY 8(c) ladder): a production-mode token flip is "explained" when the oracle's own
# top1 - top2 margin at that step (fed the GPU's prefix) is below this
FLIP_NOISE_MARGIN = 1e-2


def compare_teacher_forced(P_, src, tok, ln, top1, mode="mirror"):
    """Per step: the oracle, fed the GPU's own prefix, must choose the GPU's token at every
    step whose oracle margin lies outside the band; the chosen token's logit within 2e-2."""
    def one(i):
        return S.greedy_decode(src[i], P_, wl.S2S, mode, forced=tok[i])
    with ThreadPoolExecutor(_threads()) as ex:
        res = list(ex.map(one, range(len(src))))
    rep = dict(n=len(src), steps=0, band_steps=0, step_mismatch=0, max_top1_rel=0.0, max_flip_margin=0.0)
    for i, (o_tok, o_len, o_top1, _, preds) in enumerate(res):
        assert o_len == ln[i], (i, o_len, ln[i])       # the forced prefix decides the length
        for t in range(int(ln[i])):
            rep["steps"] += 1
            if in_band([preds[t]]):
                rep["band_steps"] += 1
                continue
            if o_tok[t] != tok[i, t]:
                rep["step_mismatch"] += 1
                rep["max_flip_margin"] = max(rep["max_flip_margin"], float(preds[t][1]))
                continue
            r = abs(top1[i, t] - o_top1[t]) / max(1.0, abs(o_top1[t]))
            rep["max_top1_rel"] = max(rep["max_top1_rel"], float(r))
    return rep


def s2s_free_running(m, W, src, idx, mode="mirror"):
    tok, ln, top1, z0 = run_s2s(m, src)
    rep = compare_free_running(_prep(W), src[idx], tok[idx], ln[idx], top1[idx], z0[idx], mode)
    rep.update(batch=len(src), sampled=len(idx), mean_length=float(ln.mean()))
    return rep


def s2s_teacher_forced(m, W, src, idx, mode="mirror"):
    tok, ln, top1, _ = run_s2s(m, src)
    rep = compare_teacher_forced(_prep(W), src[idx], tok[idx], ln[idx], top1[idx], mode)
    rep.update(batch=len(src), sampled=len(idx))
    return rep
