"""Quick per-kernel timing of one config on the GPU (development aid, not the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else wl.CONFIGS[cfg]["batch"]
W = {1: wl.mlp_weights, 2: wl.sdn_r56_weights, 3: wl.skipnet_r38_weights}[cfg]()
m = P.BUILDERS[cfg](W, B)
X = wl.mlp_inputs(wl.INPUT_SEED, 0, B) if cfg == 1 else wl.image_inputs(wl.INPUT_SEED, 0, B)
x = torch.from_numpy(X).cuda()
lg = torch.empty((B, 10), device="cuda")
pa = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    m.run(x, lg, pa)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    m.run(x, lg, pa)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"cfg{cfg} B={B}: {ms:.3f} ms/step  {B / ms * 1e3:.0f} samples/s  launches={D.dycl_launches_per_run(m.g)}")
print("path hist", np.bincount(pa.cpu().numpy() if cfg != 3 else [0]).tolist())
D.dycl_set_profiling(m.g, 1)
m.run(x, lg, pa)
prof = D.dycl_profile_read(m.g)
tot = {}
for p in prof:
    t = tot.setdefault(p["kind"], [0, 0.0, 0.0, 0.0])
    t[0] += 1
    t[1] += p["ms"]
    t[2] += p["bytes"]
    t[3] += p["flops"]
for k, (n, t, b, f) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:8s} n={n:3d} {t:8.3f} ms  {b / t / 1e6 if t else 0:8.1f} GB/s  {f / t / 1e9 if t else 0:8.1f} TFLOP/s")
convs = [p for p in prof if p["kind"] == "conv"]
for p in convs[:8]:
    print(f"   conv {p['ms']*1e3:8.1f} us  {p['bytes']/p['ms']/1e6:8.1f} GB/s {p['flops']/p['ms']/1e9:8.1f} TF/s")
