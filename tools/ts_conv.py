"""conv_gemm phase timeline (globaltimer ns, CTAs 0-7) of the k-th conv launch of a cfg2 run.
  python tools/ts_conv.py k [dbg]      (development; DYCL_TS_CONV=k)"""
import os
import sys

os.environ["DYCL_TS"] = "1"
os.environ["DYCL_TS_CONV"] = sys.argv[1] if len(sys.argv) > 1 else "6"
if len(sys.argv) > 2:
    os.environ["DYCL_CONV_DBG"] = sys.argv[2]
import torch  # noqa: E402
sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402
B = 4096
m = P.build_sdn_resnet56(wl.sdn_r56_weights(), B)
x = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 0, B)).cuda()
lg = torch.empty((B, 10), device="cuda"); pa = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    m.run(x, lg, pa)
torch.cuda.synchronize()
ts = D.dycl_debug_timestamps(m.g)
t0 = ts[:, 0].min()
names = ["start", "prolog", "bres", "mma_t0", "mma_end", "prod_t0", "prod_end", "epi_t0", "epi_end", "end"]
for i in range(8):
    print(i, f"tiles={ts[i][10]}", " ".join(f"{n}={(ts[i][k] - t0) / 1000:.2f}" for k, n in enumerate(names)))
