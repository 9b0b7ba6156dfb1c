"""One cfg2 (or cfg3: second argument 3) step with per-launch CUDA-event timing + algorithmic
bytes/flops (JSON to stdout).  python tools/step_profile.py [warm_runs] [cfg]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

CFG = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B = 4096 if CFG == 2 else 8192
m = (P.build_sdn_resnet56(wl.sdn_r56_weights(), B) if CFG == 2 else
     P.build_skipnet_resnet38(wl.skipnet_r38_weights(), B))
x = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 0, B)).cuda()
lg = torch.empty((B, 10), device="cuda")
pa = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    m.run(x, lg, pa)
torch.cuda.synchronize()
D.dycl_set_profiling(m.g, 1)
m.run(x, lg, pa)
prof = D.dycl_profile_read(m.g)
json.dump(prof, sys.stdout)
