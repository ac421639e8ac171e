"""Host-side checks of the C-ABI library (no GPU needed, no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

import paper_2405_15013_b200 as ksb
from paper_2405_15013_b200 import build as kbuild


@pytest.fixture(scope="module")
def lib():
    kbuild.build()
    return ksb.load_library()


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "ks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(ks_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


def test_header_declarations_match_binding_list():
    assert _declared_functions() == sorted(ksb.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", ksb.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(ks_[a-z_0-9]+)$", out, flags=re.M))
    missing = [n for n in _declared_functions() if n not in exported]
    assert not missing, missing
    for n in _declared_functions():
        assert hasattr(lib, n)


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", ksb.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_status_strings_and_version(lib):
    assert lib.ks_abi_version() == 1
    for s, name in ksb.ks.STATUS.items():
        assert lib.ks_status_string(s).decode() == name


def test_pattern_validation_without_device(lib):
    h = lib.ks_pack_weights(0, 2, 2, 1, None)
    assert not h
    assert lib.ks_last_error() == 2                   # KS_ERR_PATTERN
    h = lib.ks_pack_weights(1 << 40, 1 << 40, 2, 1, None)
    assert not h and lib.ks_last_error() == 2
    h = lib.ks_pack_weights(1, 2, 2, 1, None)
    assert not h and lib.ks_last_error() == 1         # KS_ERR_INVALID_ARG (NULL K)


def test_null_handle_errors(lib):
    assert lib.ks_matmul(None, None, None, 1, 0, None) == 1
    assert lib.ks_set_math(None, 0) == 1
    arr = (ctypes.c_void_p * 1)(None)
    assert lib.ks_chain_ex(arr, 1, None, None, 4, 0, None) == 1
    assert lib.ks_chain_ex(arr, 0, None, None, 4, 0, None) == 1
    lib.ks_free(None)


def test_no_device_is_reported(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np
    K = np.ones(4, np.float32)
    h = lib.ks_pack_weights(1, 2, 2, 1, ctypes.c_void_p(K.ctypes.data))
    assert not h and lib.ks_last_error() == 5         # KS_ERR_DEVICE


def test_product_path_does_not_import_oracle():
    """The product package never references the oracle or a CPU fallback."""
    pkg = os.path.join(ROOT, "paper_2405_15013_b200")
    for dp, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dp, fn)).read()
                assert "oracle" not in txt.replace("oracle-", ""), fn
