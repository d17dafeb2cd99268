"""The C-ABI library builds, loads and exports every symbol include/vdfcg.h declares;
host-only entry points work without a GPU; compute entry points fail loudly (there is no
CPU fallback) when no device is present."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2504_14897_b200 import _abi
from paper_2504_14897_b200.types import FitConfig, InvalidArgument

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2504_14897_b200 import api
    if not os.path.exists(api.LIB_PATH):
        from paper_2504_14897_b200 import build
        build.build()
    return api.lib()


def test_exports_every_header_symbol(lib):
    names = _abi.header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a(lib):
    import subprocess
    from paper_2504_14897_b200 import api
    out = subprocess.run(["cuobjdump", "--list-elf", api.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points(lib):
    from paper_2504_14897_b200 import api
    assert lib.vdfcg_abi_version() == 1
    assert lib.vdfcg_model_payload_bytes(2, 2) == 96
    assert lib.vdfcg_model_header_bytes(2, 1) == 59
    api.validate_fit_config(FitConfig(), 2)
    with pytest.raises(InvalidArgument, match="prune_threshold must be < 1/initial_components"):
        api.validate_fit_config(FitConfig(initial_components=12, prune_threshold=0.2), 2)


def test_no_cpu_fallback_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2504_14897_b200 import api
    h = C.c_void_p()
    rc = lib.vdfcg_ctx_create(0, C.byref(h))
    assert rc == _abi.VDFCG_CUDA_ERROR
    assert "no CPU fallback" in api.last_error()


def test_product_never_imports_oracle():
    """The product package must not reference the test-only oracle."""
    pkg = os.path.join(ROOT, "paper_2504_14897_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "liboracle" not in text, f
