"""The C-ABI boundary (include/qk.h): the library loads on a host without a
GPU and exports every entry point the header declares; device calls fail
loudly (QK_ERR_SIM) instead of falling back to the CPU."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "qk.h")
LIB = os.path.join(ROOT, "paper_2409_14697_b200", "libqk_b200.so")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("qk_create", "qk_destroy", "qk_set_basis", "qk_apply_block", "qk_ims_swap", "qk_xrs_swap",
                 "qk_norm", "qk_download", "qk_last_error", "qk_simulate", "qk_program_parse"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_no_torch_types_in_the_boundary():
    text = open(HEADER).read()
    assert "torch" not in text.replace("no CUDA, torch or C++ types", "")
    assert "extern \"C\"" in text


def test_device_calls_fail_loudly_without_gpu(qk):
    try:
        if qk.device_count() > 0:
            pytest.skip("GPU present")
    except qk.SimulationError:
        pass
    with pytest.raises(qk.SimulationError):
        qk.State(10)
