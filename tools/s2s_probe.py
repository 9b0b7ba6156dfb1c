"""One config-4 batch (for ncu launch lists)."""
import sys
import torch
sys.path.insert(0, ".")
import workloads as wl
from paper_2307_04963_b200 import programs as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = P.build_seq2seq(wl.seq2seq_weights(), wl.S2S, B)
src = torch.from_numpy(wl.token_inputs(wl.INPUT_SEED, 0, B)).cuda()
tok = torch.empty((B, 64), dtype=torch.int32, device="cuda")
ln = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    m.run(src, tok, ln)
torch.cuda.synchronize()
print("mean len", ln.float().mean().item())
