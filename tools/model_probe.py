"""Run config-2 steps once (for ncu capture of specific launches)."""
import sys
import torch
sys.path.insert(0, ".")
import workloads as wl
from paper_2307_04963_b200 import programs as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m = P.build_sdn_resnet56(wl.sdn_r56_weights(), B)
x = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 0, B)).cuda()
lg = torch.empty((B, 10), device="cuda")
pa = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    m.run(x, lg, pa)
torch.cuda.synchronize()
