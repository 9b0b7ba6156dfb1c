"""Build libdycl.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdycl.so")
SOURCES = ["api.cpp", "comm.cpp", "s2s_api.cpp", "conv_tc.cu", "conv_tma.cu", "conv_gemm.cu", "conv_halo.cu", "gemm_tma.cu", "block_fused.cu", "hostmod.cu", "s2s_kernels.cu", "cap.cu", "drb.cu"]
HEADERS = ["kernels.h", "comm.h", "drb.h", "ptx.cuh", "epilogue.cuh", "s2s_kernels.h", os.path.join("..", "..", "include", "dycl.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


def _nccl_include() -> str:
    """NCCL 2.28's headers (nccl.h + the device API, nccl_device/*) as shipped with the torch NCCL
    wheel: drb.cu computes LSA peer pointers with ncclGetPeerPointer (a header-inline device
    function); the host side resolves NCCL at run time."""
    try:
        import nvidia.nccl  # noqa: F401
        return os.path.join(list(nvidia.nccl.__path__)[0], "include")
    except Exception:
        return "/usr/include"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    bdir = os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    objs = [os.path.join(bdir, src + ".o") for src in SOURCES]

    def compile_one(src_obj):
        src, obj = src_obj
        cmd = [NVCC, *FLAGS, "-I", _nccl_include(), "-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, zip(SOURCES, objs)))
    tmp = LIB + f".{os.getpid()}.tmp"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
