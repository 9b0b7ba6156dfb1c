"""One chunk of a config through dycl_run, launch by launch (DYCL_GRAPH=0 set by the caller),
for an ncu launch list:  ncu -k regex:k_ ... python tools/ncu_chunk.py [cfg] [chunk]"""
import sys

import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
W = {2: wl.sdn_r56_weights, 3: wl.skipnet_r38_weights, 5: wl.resnet50_ee_weights}[cfg]()
m = P.BUILDERS[cfg](W, B)
x = (wl.image_inputs_torch(wl.INPUT_SEED, 0, B, hw=224, device="cuda") if cfg == 5 else
     torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 0, B)).cuda())
lg = torch.empty((B, m.K), device="cuda")
pa = torch.empty(B, dtype=torch.int32, device="cuda")
m.run(x, lg, pa)
torch.cuda.synchronize()
print("paths", torch.bincount(pa.long()).tolist())
