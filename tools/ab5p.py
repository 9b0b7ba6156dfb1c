"""In-process A/B of config-5 chunks under DYCL_* environment variants (development aid):
sustained time of 3 back-to-back chunks per sample, variants interleaved, plus per-launch
CUDA-event times of the first launches (stem, pool, stage 1) from the library's profiler.

  python tools/ab5p.py [chunk] [reps] VAR=VAL[,VAR=VAL] ...     (first variant: the default env)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
R = int(sys.argv[2]) if len(sys.argv) > 2 else 6
variants = [""] + sys.argv[3:]
W = wl.resnet50_ee_weights()
x = wl.image_inputs_torch(wl.INPUT_SEED, 0, B, hw=224, device="cuda")
models = []
for v in variants:
    saved = dict(os.environ)
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=")
        os.environ[k] = val
    models.append(P.build_resnet50_ee(W, B))
    os.environ.clear()
    os.environ.update(saved)
outs = [(torch.empty((B, 1000), device="cuda"), torch.empty(B, dtype=torch.int32, device="cuda")) for _ in models]
for m, o in zip(models, outs):
    for _ in range(2):
        m.run(x, *o)
torch.cuda.synchronize()
times = [[] for _ in models]
lt = [[] for _ in models]
for r in range(R):
    for i, m in enumerate(models):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            m.run(x, *outs[i])
        e1.record()
        torch.cuda.synchronize()
        times[i].append(e0.elapsed_time(e1) / 3)
        D.dycl_set_profiling(m.g, 1)
        m.run(x, *outs[i])
        lt[i].append([p["ms"] for p in D.dycl_profile_read(m.g)])
        D.dycl_set_profiling(m.g, 0)
ref_p = outs[0][1].cpu().numpy()
for i, v in enumerate(variants):
    p = outs[i][1].cpu().numpy()
    n = min(len(t) for t in lt[i])
    med = np.median(np.array([t[:n] for t in lt[i]]), axis=0)
    print(f"{v or 'default':36s} {np.median(times[i]):8.3f} ms/chunk (min {min(times[i]):.3f}) profiled sum "
          f"{med.sum():.3f}  path diffs {int((p != ref_p).sum())}  launches 1-12: "
          + " ".join(f"{t:.3f}" for t in med[1:13]))
