"""CPU oracle for DyCL-style dynamic-NN inference -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference the CUDA path is
graded against.  It interprets the ORIGINAL dynamic programs (real ``if`` /
``for`` / ``return``) one sample at a time, in fp64, exactly as the paper's
correctness contract states:  P_DyNN(x) = P_Host(x) for all x  (PAPER.md L528,
Sec. 5 Eq. 2).  It shares no code with ``paper_2307_04963_b200`` (no kernels,
headers, helpers or constant tables); the only common module is the seeded
input/weight generator ``workloads``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import, call, link or execute anything here.

Modes (readings R13-R14):
  * ``mirror`` -- bf16 rounding (round-to-nearest-even of the fp64 value) at
    the storage points of the production bf16 path; decisions are graded here;
  * ``exact``  -- fp64 everywhere after the bf16 weights/input.

Parity pins: tests/test_oracle.py.  Functions whose absolute values have no
pin beyond library cross-checks are marked "parity unpinned" where defined.
"""
from .core import (round_bf16, conv2d, dense, gap, relu, max_softmax, sigmoid,
                   argmax_lowest, option_a, maxpool2d)
from .programs import (mlp_ee, sdn_resnet56, skipnet_resnet38, skipnet_rnn_resnet38, resnet50_ee, run_batch,
                       PROGRAMS)
from .metrics import delta, eta

__all__ = [
    "round_bf16", "conv2d", "dense", "gap", "relu", "max_softmax", "sigmoid",
    "argmax_lowest", "option_a", "maxpool2d", "mlp_ee", "sdn_resnet56", "skipnet_resnet38", "skipnet_rnn_resnet38", "resnet50_ee",
    "run_batch", "PROGRAMS", "delta", "eta",
]
