"""dycl-b200: B200-native batched inference of rewritten dynamic neural networks (DyCL, arXiv 2307.04963).

Product path: ``libdycl.so`` (C ABI in include/dycl.h; sm_100a kernels in csrc/)
+ the ctypes binding ``dycl`` + the model registration ``programs``.
"""
from . import dycl  # noqa: F401
