"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports
every symbol include/dycl.h declares; host-side errors surface as statuses."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dycl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dycl_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_verbs():
    names = _declared()
    for v in ["dycl_subnet_begin", "dycl_subnet_conv2d", "dycl_subnet_dense", "dycl_exit", "dycl_gate",
              "dycl_final", "dycl_finalize", "dycl_run", "dycl_run_host"]:
        assert v in names


def test_library_exports_every_declared_symbol():
    from paper_2307_04963_b200 import build as B
    B.build()
    lib = ctypes.CDLL(B.LIB)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_wraps_every_symbol():
    from paper_2307_04963_b200 import dycl as D
    assert sorted(D.EXPORTS) == sorted(n for n in _declared())
    for n in D.EXPORTS:
        assert callable(getattr(D, n))


def test_no_gpu_create_fails_loudly():
    """Without a CUDA device the product path raises (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2307_04963_b200 import dycl as D
    with pytest.raises(D.DyclError) as e:
        D.dycl_graph_create(0, 32, 32, 3)
    assert "CUDA" in str(e.value)
    assert "device" in D.dycl_last_error(None).lower()


def test_null_and_bad_args_return_status():
    from paper_2307_04963_b200 import dycl as D
    L = D.lib()
    assert L.dycl_graph_destroy(None) == 0
    assert L.dycl_finalize(None, 10) == -1
    assert L.dycl_run(None, None, None) == -1
    assert L.dycl_graph_create(0, 0, 32, 3, None) == -1
