"""In-process A/B timing of config-5 chunks: graphs built under different DYCL_* environment
settings (read at graph creation / finalize), run alternately on the same inputs (development aid).

  python tools/ab5.py [chunk] [reps] VAR=VAL[,VAR=VAL] ...     (first variant: the default env)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
variants = [""] + sys.argv[3:]
W = wl.resnet50_ee_weights()
x = wl.image_inputs_torch(wl.INPUT_SEED, 0, B, hw=224)
models = []
for v in variants:
    saved = dict(os.environ)
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=")
        os.environ[k] = val
    models.append(P.build_resnet50_ee(W, B))
    os.environ.clear()
    os.environ.update(saved)
outs = []
for m in models:
    lg = torch.empty((B, 1000), device="cuda")
    pa = torch.empty(B, dtype=torch.int32, device="cuda")
    for _ in range(2):
        m.run(x, lg, pa)
    outs.append((lg, pa))
torch.cuda.synchronize()
times = [[] for _ in models]
for r in range(R):
    for i, m in enumerate(models):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.run(x, *outs[i])
        e1.record()
        torch.cuda.synchronize()
        times[i].append(e0.elapsed_time(e1))
ref_p = outs[0][1].cpu().numpy()
ref_l = outs[0][0].cpu().numpy()
for i, v in enumerate(variants):
    p = outs[i][1].cpu().numpy()
    l = outs[i][0].cpu().numpy()
    rel = float(np.max(np.abs(l - ref_l)) / np.max(np.abs(ref_l)))
    print(f"{v or 'default':40s} {np.median(times[i]):8.3f} ms/chunk (min {min(times[i]):.3f})  "
          f"paths {np.bincount(p, minlength=4).tolist()}  path diffs vs default {int((p != ref_p).sum())}  "
          f"max logit rel diff {rel:.2e}")
