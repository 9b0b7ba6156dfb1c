"""Print fused-block phase timelines (CTA 0) for one block launch of config 2 (DYCL_TS=1)."""
import os
import sys

os.environ["DYCL_TS"] = sys.argv[1] if len(sys.argv) > 1 else "1"   # k > 1: k-th fused launch
import numpy as np
import torch
sys.path.insert(0, ".")
import workloads as wl
from paper_2307_04963_b200 import dycl as D
from paper_2307_04963_b200 import programs as P
B = 4096
m = P.build_sdn_resnet56(wl.sdn_r56_weights(), B)
x = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 0, B)).cuda()
lg = torch.empty((B, 10), device="cuda"); pa = torch.empty(B, dtype=torch.int32, device="cuda")
m.run(x, lg, pa); m.run(x, lg, pa)
ts = D.dycl_debug_timestamps(m.g)          # the LAST fused launch of the run (stage 2)
t0 = ts[0][ts[0] > 0].min()
names = ["cvt0", "cvt1", "e1s", "e1e", "e2s", "e2e", "m1s", "m1e", "m2s", "m2e", "prod"]
for i in range(8):
    print(i, " ".join(f"{n}={(ts[i][k]-t0)}" for k, n in enumerate(names)))
