"""CPU tests of the drop-in boundary: libgbxcu.so builds for sm_100a, loads,
exports every symbol include/gbxcu.h declares, and refuses to run without a
B200 (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2111_12055_b200 as gbx
from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    gbx.build()
    return gbx.load_library()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gbxcu.h")).read()
    return sorted(set(re.findall(r"\b(gbxcu_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    decl = declared_symbols()
    assert len(decl) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", gbx.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gbxcu_\w+)", out))
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    assert set(gbx.EXPORTS) == set(decl)
    for s in decl:
        getattr(lib, s)


def test_sm100a_only_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", gbx.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_abi_version(lib):
    assert lib.gbxcu_abi_version() == 2


def test_no_cpu_fallback_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    rc = lib.gbxcu_create(0, C.byref(h))
    assert rc == gbx.ECUDA
    with pytest.raises(gbx.CudaError):
        gbx.Device(0)
