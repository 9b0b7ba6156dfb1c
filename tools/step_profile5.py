"""One config-5 chunk (early-exit ResNet-50, 224x224) with per-launch CUDA-event timing,
algorithmic bytes / FLOPs and achieved rates (development tool; JSON to stdout).

  python tools/step_profile5.py [chunk] [warm]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
WARM = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m = P.build_resnet50_ee(wl.resnet50_ee_weights(), B)
x = wl.image_inputs_torch(wl.INPUT_SEED, 0, B, hw=224, device="cuda")
lg = torch.empty((B, 1000), device="cuda")
pa = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(WARM):
    m.run(x, lg, pa)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
m.run(x, lg, pa)
e1.record()
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1)
D.dycl_set_profiling(m.g, 1)
m.run(x, lg, pa)
prof = D.dycl_profile_read(m.g)
tot = sum(p["ms"] for p in prof)
rows = []
for i, p in enumerate(prof):
    ms = p["ms"]
    rows.append(dict(i=i, kind=p["kind"], ms=round(ms, 4), share=round(ms / tot, 4),
                     GBps=round(p["bytes"] / ms / 1e6, 1) if ms > 0 else 0,
                     TFLOPs=round(p["flops"] / ms / 1e9, 1) if ms > 0 else 0, rows=p.get("rows")))
json.dump(dict(chunk=B, step_ms=step_ms, profiled_total_ms=tot, paths=torch.bincount(pa, minlength=4).tolist(),
               launches=rows), sys.stdout, indent=0)
