"""CPU: the C-ABI library builds, loads and exports exactly what
include/kclique.h declares; without a GPU every compute entry fails loudly
(KC_ECUDA -> KcError), never silently on the CPU."""

import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "kclique.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|void|char)\s*\*?\s*(kc_\w+)\s*\(",
                                 src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2104_13209_b200 import _lib
    from paper_2104_13209_b200.build import build

    build()
    return _lib


def test_header_and_binding_agree(lib):
    assert header_symbols() == sorted(lib.EXPORTS)


def test_library_exports_every_symbol(lib):
    L = lib.load()
    for name in header_symbols():
        assert hasattr(L, name), name
    assert L.kc_abi_version() == 2


def test_sm100a_cubin_inside(lib):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and os.path.exists("/dev/nvidia0"),
                    reason="a GPU is visible")
def test_no_cpu_fallback_without_gpu(lib):
    if lib.device_count() > 0:
        pytest.skip("GPU visible")
    import paper_2104_13209_b200 as kc

    with pytest.raises(lib.KcError):
        kc.from_edges(np.array([[0, 1], [1, 2], [0, 2]], dtype=np.int64))
