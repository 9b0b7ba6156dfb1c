"""Run the a1 conv kernel alone on a config-2 stage shape (for ncu / timing)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import workloads as wl
from paper_2307_04963_b200 import dycl as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
H, C, Co, res_mode = [int(v) for v in (sys.argv[2:6] if len(sys.argv) > 5 else (32, 16, 16, 0))]
reps = 5
g = D.dycl_graph_create(0, 1, 1, 8)
rng = np.random.default_rng(0)
x = torch.randint(-30000, 30000, (n, H, H, C), dtype=torch.int16, device="cuda") & 0x3FFF
w = wl.f32_to_bf16_bits(rng.standard_normal((Co, 3, 3, C)) * 0.1)
b = np.zeros(Co, np.float32)
y = torch.zeros((n, H, H, Co), dtype=torch.int16, device="cuda")
res = torch.zeros((n, H, H, Co), dtype=torch.int16, device="cuda") if res_mode else None
path = int(sys.argv[6]) if len(sys.argv) > 6 else 0
for _ in range(reps):
    D.dycl_debug_conv2d(g, x, n, H, H, C, w, b, Co, 3, 1, 1, 1, res, res_mode, y, path)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    D.dycl_debug_conv2d(g, x, n, H, H, C, w, b, Co, 3, 1, 1, 1, res, res_mode, y, path)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
byt = n * H * H * (C + Co) * 2
print(f"conv n={n} {H}x{H}x{C}->{Co}: {ms*1e3:.1f} us/launch (incl. weight upload+sync), {byt/ms/1e6:.0f} GB/s algorithmic")
