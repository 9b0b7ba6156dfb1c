"""Config-5 parity of both storage precisions on N seeded samples (development tool):
FP32_STREAM vs the oracle's mirror mode and BF16 storage vs mirror_bf16 (reading R13)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import workloads as wl  # noqa: E402
from oracle import programs as prg  # noqa: E402
from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402
from tests.parity import report  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 48
W = wl.resnet50_ee_weights()
X = wl.image_inputs(wl.INPUT_SEED, 4000, N, hw=224)
out = {}
for name, prec, mode in [("fp32_stream", D.DYCL_PREC_FP32_STREAM, "mirror"), ("bf16", D.DYCL_PREC_BF16, "mirror_bf16")]:
    m = P.build_resnet50_ee(W, N, precision=prec)
    x = torch.from_numpy(X).cuda()
    lg = torch.empty((N, 1000), device="cuda")
    pa = torch.empty(N, dtype=torch.int32, device="cuda")
    m.run(x, lg, pa)
    torch.cuda.synchronize()
    lo, po, pr = O.run_batch(O.resnet50_ee, X, prg.prepare(W), mode)
    r = report(lg.cpu().numpy(), pa.cpu().numpy(), lo, po, pr)
    r.pop("mismatch_idx", None)
    out[name] = r
    print(name, r, flush=True)
json.dump(out, open("gpurun_out/cfg5_prec.json", "w"), indent=1)
