"""The sm_100a library is a plain C ABI: it loads without a GPU and exports
every symbol include/rbd_b200.h declares; argument errors are reported
before any CUDA call."""
import ctypes
import os
import re

import pytest

from paper_2109_06976_b200 import codegen, kernels, models

HEADER = os.path.join(kernels.INCLUDE, "rbd_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^int (rbd_\w+)\(", text, flags=re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert set(kernels.ABI_SYMBOLS) == set(syms)


def test_library_exports_every_declared_symbol():
    m = models.load("chain7")
    lib = kernels.library(m)  # builds (nvcc cross-compiles) when missing
    for s in declared_symbols():
        assert hasattr(lib, s), s
    info = kernels.RbdInfo()
    assert lib.rbd_get_info(ctypes.byref(info)) == 0
    assert info.abi_version == 1 and info.n_dof == 7 and info.n_trees == 1
    assert info.robot.decode() == "chain7"
    assert info.fingerprint.decode() == codegen.model_hash(m)
    ni, e = ctypes.c_int32(), [ctypes.c_int64() for _ in range(3)]
    assert lib.rbd_alg_extents(4, ctypes.byref(ni), *[ctypes.byref(x) for x in e]) == 0
    assert (ni.value, [x.value for x in e]) == (3, [49, 49, 7])
    # argument errors come back as negative codes, no CUDA involved
    assert lib.rbd_launch(9, 1, None, None, None, None, None, None, 4, None) == -1
    assert lib.rbd_gradFD_f64(None, None, None, None, None, None, -1, None) == -1
    assert lib.rbd_gradFD_f64(None, None, None, None, None, None, 4, None) == -1
    assert lib.rbd_run_host(None, 4, 1, None, None, None, None, None, None, 4) == -2


def test_build_metadata_records_sm100a_and_registers():
    m = models.load("chain7")
    kernels.library(m)
    meta = kernels.build_meta(m)
    assert "arch=compute_100a,code=sm_100a" in " ".join(meta["nvcc_flags"])
    assert len(meta["ptxas"]) >= 10  # thread-per-knot and/or warp-specialised kernels per (alg, dtype)
    assert all("registers" in v for v in meta["ptxas"].values())
