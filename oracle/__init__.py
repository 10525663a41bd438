"""Oracle for the merge-tree / 0-dim persistence hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under
``oracle/``.  The product package ``paper_2301_10838_b200`` never imports it,
and this package never imports the product (they share no code; the only
common input is the seeded field generator module ``paper_2301_10838_b200/fields.py``, which
holds none of the method's arithmetic).

Contents
--------
- ``merge_tree``  : O1, serial Kruskal/union-find with elder-rule pairing,
                    plain C (``mt_oracle.c``), PAPER.md:139-148 + 180-200.
- ``brute``       : O2, the triplet definition read literally by BFS over
                    sublevel sets, tiny inputs only.
- ``alg1``        : O3, the paper's Alg. 1-5 executed serially with the root
                    guard readings of DESIGN.md (R4/R5), any edge order.
- ``invariants``  : structural checks I1-I5 of DESIGN.md.

Pins (tests/test_oracle_pins.py): O1 == O2 on exhaustive/random tiny grids;
golden examples (tests/golden/*.txt, each cited); closed-form families
(checkerboard, constant, ramp); scipy.ndimage.label Betti-0 counts at sampled
thresholds.  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mt_oracle.c")
_SO = os.path.join(_HERE, "libmt_oracle.so")
_lock = threading.Lock()
_lib = None

PAIR_DTYPE = np.dtype([("birth_v", "<u4"), ("death_v", "<u4"), ("birth", "<f4"), ("death", "<f4")])

OK, INVALID, TOO_LARGE, NONFINITE, NOMEM, CAPACITY = 0, 1, 2, 3, 8, 9


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle status {status}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (no -ffast-math: IEEE compares matter)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.oracle_merge_tree.restype = ctypes.c_int
            lib.oracle_merge_tree.argtypes = [
                ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
            lib.oracle_triplet_at.restype = ctypes.c_int
            lib.oracle_triplet_at.argtypes = [
                ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                ctypes.c_uint32, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
            lib.oracle_triplet_at64.restype = ctypes.c_int
            lib.oracle_triplet_at64.argtypes = [
                ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
            lib.oracle_merge_tree_graph.restype = ctypes.c_int
            lib.oracle_merge_tree_graph.argtypes = [
                ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                ctypes.POINTER(ctypes.c_uint64)]
            _lib = lib
    return _lib


def merge_tree(f: np.ndarray, dims, conn: int = 6, split: bool = False, want_pairs: bool = True):
    """O1.  ``f``: float32 values, x fastest, ``dims`` = (nx, ny, nz).

    Returns ``(T, pairs, n_pairs, n_ess)`` with ``T`` a uint64 array
    (s << 32 | v) and ``pairs`` a PAIR_DTYPE array: finite pairs ascending by
    birth vertex, then essential classes ascending (death = +inf).
    """
    lib = _load()
    nx, ny, nz = (int(d) for d in dims)
    f = np.ascontiguousarray(f, dtype=np.float32).reshape(-1)
    n = nx * ny * nz
    if f.size != n:
        raise ValueError("f size does not match dims")
    T = np.empty(n, dtype=np.uint64)
    # a grid's strict minima form an independent set: at most ceil(n/2) diagram records
    cap = (n + 1) // 2 + 1 if want_pairs else 0
    pairs = np.empty(cap, dtype=PAIR_DTYPE)
    npairs, ness = ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = lib.oracle_merge_tree(f.ctypes.data if n else None, nx, ny, nz, int(conn), int(bool(split)),
                               T.ctypes.data if n else None,
                               pairs.ctypes.data if (want_pairs and n) else None, cap,
                               ctypes.byref(npairs), ctypes.byref(ness))
    if st != OK:
        raise OracleError(st)
    k = npairs.value + ness.value
    return T, (pairs[:k] if want_pairs else None), npairs.value, ness.value


def triplet_at(f: np.ndarray, dims, conn: int, u: int, split: bool = False, cap: int = 1 << 20):
    """O4: the triplet (s, v) of the single vertex u from the definition by
    bounded floods (oracle/mt_oracle.c: oracle_triplet_at64, 64-bit ids: any grid size), or None
    when a flood would visit more than ``cap`` vertices.  For sampled checks of full-size outputs."""
    f = np.ascontiguousarray(f, dtype=np.float32).reshape(-1)
    nx, ny, nz = (int(d) for d in dims)
    if f.size != nx * ny * nz:
        raise ValueError("f size does not match dims")
    s, v = ctypes.c_uint64(0), ctypes.c_uint64(0)
    rc = _load().oracle_triplet_at64(f.ctypes.data, nx, ny, nz, int(conn), int(bool(split)), int(u), int(cap),
                                     ctypes.byref(s), ctypes.byref(v))
    if rc < 0:
        raise OracleError(rc)
    return (int(s.value), int(v.value)) if rc == 1 else None


def merge_tree_graph(f: np.ndarray, row: np.ndarray, col: np.ndarray, split: bool = False):
    """O1 on an explicit graph in CSR form (neighbours of u: col[row[u]:row[u+1]]); same outputs
    as merge_tree.  Several components give several essential classes."""
    lib = _load()
    f = np.ascontiguousarray(f, dtype=np.float32).reshape(-1)
    row = np.ascontiguousarray(row, dtype=np.uint64)
    col = np.ascontiguousarray(col, dtype=np.uint32)
    n = f.size
    if row.size != n + 1:
        raise ValueError("row must have n+1 entries")
    T = np.empty(n, dtype=np.uint64)
    pairs = np.empty(max(n, 1), dtype=PAIR_DTYPE)
    npairs, ness = ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = lib.oracle_merge_tree_graph(f.ctypes.data if n else None, n, row.ctypes.data,
                                     col.ctypes.data if col.size else None, int(bool(split)),
                                     T.ctypes.data if n else None, pairs.ctypes.data, pairs.size, ctypes.byref(npairs),
                                     ctypes.byref(ness))
    if st != OK:
        raise OracleError(st)
    return T, pairs[: npairs.value + ness.value], npairs.value, ness.value


def csr_from_edges(n: int, edges) -> tuple[np.ndarray, np.ndarray]:
    """Symmetric CSR adjacency of an undirected edge list (each edge listed both ways)."""
    e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 2)
    src = np.concatenate([e[:, 0], e[:, 1]])
    dst = np.concatenate([e[:, 1], e[:, 0]])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    row = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(row, src + 1, 1)
    return np.cumsum(row).astype(np.uint64), dst.astype(np.uint32)


def filter_by_persistence(pairs: np.ndarray, n_pairs: int, eps: float) -> np.ndarray:
    """Finite pairs with persistence |f(b) - f(a)| > eps, then every essential class
    (short branches as topological noise; SPEC.md "filter_by_persistence").
    The persistence is computed in float32, the precision of the values."""
    fin = pairs[:n_pairs]
    pers = np.abs(fin["death"].astype(np.float32) - fin["birth"].astype(np.float32))
    return np.concatenate([fin[pers > np.float32(eps)], pairs[n_pairs:]])


def unpack(T: np.ndarray):
    """(s, v) halves of packed cells (s high, v low -- reading R11)."""
    T = np.asarray(T, dtype=np.uint64)
    return (T >> np.uint64(32)).astype(np.uint32), (T & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def pack(s, v):
    return (np.asarray(s, dtype=np.uint64) << np.uint64(32)) | np.asarray(v, dtype=np.uint64)
