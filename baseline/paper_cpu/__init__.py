"""The paper's own method (Alg. 1-5 with 64-bit CAS) on all host cores with
OpenMP -- the analogue of the paper's OpenMP column (optional
second CPU baseline).  A reported baseline that bench.py times beside the GPU path; tests check
it against the oracle O1.  It shares no code with the oracle or the product package and neither
imports it."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tmt_cpu.c")
_SO = os.path.join(_HERE, "libtmt_cpu.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.tmt_cpu_merge_tree.restype = ctypes.c_int
            lib.tmt_cpu_merge_tree.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                               ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
            lib.tmt_cpu_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().tmt_cpu_max_threads())


def merge_tree(f, dims, conn: int = 6, split: bool = False, threads: int = 0) -> np.ndarray:
    """Triplet store T (uint64, s << 32 | v) of a float32 grid field, x fastest."""
    f = np.ascontiguousarray(f, dtype=np.float32).reshape(-1)
    nx, ny, nz = (int(d) for d in dims)
    if f.size != nx * ny * nz:
        raise ValueError("field size does not match dims")
    T = np.empty(f.size, dtype=np.uint64)
    st = _load().tmt_cpu_merge_tree(f.ctypes.data, nx, ny, nz, int(conn), int(bool(split)), T.ctypes.data,
                                    int(threads))
    if st != 0:
        raise RuntimeError(f"tmt_cpu status {st}")
    return T
