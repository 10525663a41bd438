"""CPU-side checks of the C ABI: the in-tree library builds/loads and exports every symbol
include/mt.h declares; host-only entry points behave (no compute without a GPU)."""
import ctypes
import os
import re

import pytest

from paper_2301_10838_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mt_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    declared = header_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTS) == declared


def test_abi_version_and_status_strings(lib):
    assert lib.mt_abi_version() == 3
    for st in range(9):
        assert lib.mt_status_string(st)
    assert b"non-finite" in lib.mt_status_string(3)


def test_workspace_bytes(lib):
    assert _lib.mt_workspace_bytes((16, 16, 16), 6) > 4096 * 8
    assert _lib.mt_workspace_bytes((16, 16, 16), 5) == 0          # bad connectivity
    assert _lib.mt_workspace_bytes((16, 16, 2), 4) == 0           # conn 4 needs nz == 1
    assert _lib.mt_workspace_bytes((0, 16, 16), 6) > 0            # empty grid is valid
    assert _lib.mt_workspace_bytes((1 << 16, 1 << 16, 2), 6) == 0  # > 2^32 vertices
    a = _lib.mt_workspace_bytes((512, 512, 512), 6)
    assert a % 256 == 0 and a < 512 ** 3 * 57  # 16-B cells + 2n queue entries + <= n/2 records


def test_create_rejects_bad_args_without_gpu(lib):
    h = ctypes.c_void_p()
    dims = (ctypes.c_uint32 * 3)(4, 4, 4)
    assert lib.mt_create(ctypes.byref(h), dims, 5, 0, None, 0) == _lib.MT_ERR_INVALID_ARG
    assert lib.mt_create(ctypes.byref(h), dims, 6, 0, None, 0) == _lib.MT_ERR_WORKSPACE
    assert lib.mt_compute(None, None, None, 0, None) == _lib.MT_ERR_INVALID_ARG
    assert lib.mt_diagram(None, None, 0, None, None, None) == _lib.MT_ERR_INVALID_ARG
    lib.mt_destroy(None)


def test_sass_is_sm100a():
    """The library carries sm_100a SASS for every kernel (cuobjdump)."""
    import subprocess
    so = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_dist_host_entry_points_without_gpu(lib):
    """NCCL is loaded at run time (no link-time dependency); the unique id and the slab rule are
    host-only; creating a distributed context validates its arguments before touching NCCL."""
    uid = _lib.mt_get_unique_id()
    assert len(uid) == 128 and any(uid)
    assert _lib.mt_dist_slab_bounds(1024, 8) == [0, 128, 256, 384, 512, 640, 768, 896, 1024]
    assert _lib.mt_dist_workspace_bytes((64, 64, 64), 6, 0, 2) > 0
    assert _lib.mt_dist_workspace_bytes((64, 64, 64), 6, 2, 2) == 0      # rank out of range
    h = ctypes.c_void_p()
    dims = (ctypes.c_uint32 * 3)(64, 64, 64)
    idbuf = (ctypes.c_uint8 * 128)(*uid)
    assert lib.mt_create_dist(ctypes.byref(h), dims, 6, 3, 2, idbuf, 0, 0, None, 0) == _lib.MT_ERR_INVALID_ARG
    assert lib.mt_create_dist(ctypes.byref(h), dims, 6, 0, 65, idbuf, 0, 0, None, 0) == _lib.MT_ERR_INVALID_ARG
    assert lib.mt_create_dist(ctypes.byref(h), dims, 6, 0, 2, None, 0, 0, None, 0) == _lib.MT_ERR_INVALID_ARG


def test_wide_id_host_logic_without_gpu(lib):
    """a slab of a grid past 2^32 vertices is sized (its own ids fit the 32-bit
    view with room below and above); a slab too thick for the view is refused; the 64-bit entry
    points and the slab options validate their arguments before touching the device."""
    big = (2048, 2048, 1032)                                  # 4.33e9 vertices
    assert big[0] * big[1] * big[2] > 2 ** 32
    assert _lib.mt_workspace_bytes(big, 6) == 0               # one GPU: 32-bit ids
    assert _lib.mt_slab_workspace_bytes(big, 6, 0, 129) > 0   # a slab of 5.4e8 vertices
    assert _lib.mt_slab_workspace_bytes(big, 6, 0, 1023) == 0  # 1023 planes + 2 do not fit 2^32 - 1
    assert _lib.mt_dist_workspace_bytes(big, 6, 3, 8) > 0
    assert _lib.mt_dist_workspace_bytes(big, 6, 0, 1) == 0
    h = ctypes.c_void_p()
    dims = (ctypes.c_uint32 * 3)(*big)
    assert lib.mt_create_slab(ctypes.byref(h), dims, 6, 0, 129, 2, 0, None, 0) == _lib.MT_ERR_INVALID_ARG  # options
    assert lib.mt_create_slab(ctypes.byref(h), dims, 6, 0, 129, 0, 0, None, 0) == _lib.MT_ERR_WORKSPACE
    huge = (ctypes.c_uint32 * 3)(0xffffffff, 0xffffffff, 0xffffffff)    # ids past 2^63
    assert lib.mt_create_slab(ctypes.byref(h), huge, 6, 0, 1, 0, 0, None, 0) == _lib.MT_ERR_TOO_LARGE
    assert lib.mt_triplets64(None, None, 0, 0, None, None) == _lib.MT_ERR_INVALID_ARG
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    assert lib.mt_diagram64(None, None, 0, ctypes.byref(a), ctypes.byref(b), None) == _lib.MT_ERR_INVALID_ARG
    zb = (ctypes.c_uint32 * 3)(0, 8, 16)
    cnt = (ctypes.c_uint64 * 2)(0, 0)
    assert lib.mt_compute_global(None, None, cnt, zb, 2, None, 0, None, None) == _lib.MT_ERR_INVALID_ARG
    assert _lib.PAIR64_DTYPE.itemsize == 24 and _lib.TRIPLET64_DTYPE.itemsize == 16


def test_host_pipeline_and_dual_entry_points_validate_without_gpu(lib):
    """mt_compute_host / mt_compute_join_split reject bad arguments before touching the device."""
    vp = ctypes.c_void_p
    lib.mt_host_staging_bytes.restype = ctypes.c_size_t
    lib.mt_host_staging_bytes.argtypes = [vp]
    assert lib.mt_host_staging_bytes(None) == 0
    assert lib.mt_compute_host(None, 1, None, None, None, 0, None, 0, None, 0, None) == _lib.MT_ERR_INVALID_ARG
    assert lib.mt_compute_join_split(None, None, None, None, None, None) == _lib.MT_ERR_INVALID_ARG
