"""Timing of config 5 (early-exit ResNet-50) chunks on one GPU (development aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
t0 = time.time()
m = P.build_resnet50_ee(wl.resnet50_ee_weights(), B)
x = wl.image_inputs_torch(wl.INPUT_SEED, 0, B, hw=224)
print("setup %.1fs" % (time.time() - t0))
lg = torch.empty((B, 1000), device="cuda")
pa = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(2):
    m.run(x, lg, pa)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    m.run(x, lg, pa)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"cfg5 B={B}: {ms:.2f} ms/chunk  {B / ms * 1e3:.0f} samples/s  path hist {np.bincount(pa.cpu().numpy(), minlength=4).tolist()}")
D.dycl_set_profiling(m.g, 1)
m.run(x, lg, pa)
prof = D.dycl_profile_read(m.g)
tot = {}
for p in prof:
    t = tot.setdefault(p["kind"], [0, 0.0, 0.0, 0.0])
    t[0] += 1; t[1] += p["ms"]; t[2] += p["bytes"]; t[3] += p["flops"]
for k, (n, t, b, f) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:8s} n={n:3d} {t:8.3f} ms  {b / t / 1e6 if t else 0:8.1f} GB/s  {f / t / 1e9 if t else 0:8.1f} TFLOP/s")
print(" ".join(f"{p['ms']*1e3:.0f}" if p["kind"] == "conv" else f"[{p['kind'][:3]} {p['ms']*1e3:.0f}]" for p in prof))
