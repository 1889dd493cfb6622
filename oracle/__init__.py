"""CPU oracle for the lossless homomorphic compression hot path — TEST INFRASTRUCTURE.

ctypes wrapper over ``oracle/liblhc_oracle.so`` (built from ``oracle/lhc_oracle.c``,
plain single-threaded C11, fp64 counters).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  It shares no code with ``paper_2402_07529_b200`` and imports nothing from it.

Every function cites the passage of PAPER.md (``P:L<n>``) it follows; the readings
taken where the paper is silent are listed in DESIGN.md §Readings.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lhc_oracle.c")
_LIB = os.path.join(_HERE, "liblhc_oracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no intrinsics, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", _SRC, "-o", _LIB]
        )
    return _LIB


class Params(ctypes.Structure):
    """Mirror of the oracle's ``ora_params`` (same field order as ``lhc_params``)."""

    _fields_ = [
        ("d", ctypes.c_uint32),
        ("m", ctypes.c_uint64),
        ("c", ctypes.c_uint64),
        ("k", ctypes.c_uint32),
        ("k_bloom", ctypes.c_uint32),
        ("L", ctypes.c_uint32),
        ("blocks", ctypes.c_uint32),
        ("seed", ctypes.c_uint64),
    ]


class _Stats(ctypes.Structure):
    _fields_ = [
        ("n_cand", ctypes.c_uint64),
        ("n_peeled", ctypes.c_uint64),
        ("rounds", ctypes.c_uint32),
        ("success", ctypes.c_int32),
        ("overflow", ctypes.c_int32),
    ]


@dataclass
class Stats:
    n_cand: int
    n_peeled: int
    rounds: int
    success: bool
    overflow: bool


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        u64, u32, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32
        vp = ctypes.c_void_p
        _lib.ora_mix64.restype = u64
        _lib.ora_mix64.argtypes = [u64]
        _lib.ora_hash.restype = u64
        _lib.ora_hash.argtypes = [u64, u32, u32, u64]
        _lib.ora_row_map.restype = None
        _lib.ora_row_map.argtypes = [P(Params), u32, u32, u64, P(u64), P(u32), P(ctypes.c_int)]
        _lib.ora_cell.restype = u64
        _lib.ora_cell.argtypes = [P(Params), u32, u64, P(ctypes.c_int)]
        _lib.ora_bit.restype = u64
        _lib.ora_bit.argtypes = [P(Params), u32, u64]
        _lib.ora_validate.restype = ctypes.c_int
        _lib.ora_validate.argtypes = [P(Params)]
        _lib.ora_compress_dense.restype = None
        _lib.ora_compress_dense.argtypes = [P(Params), vp, vp, vp]
        _lib.ora_compress_coo.restype = None
        _lib.ora_compress_coo.argtypes = [P(Params), u64, vp, vp, vp, vp]
        _lib.ora_aggregate.restype = None
        _lib.ora_aggregate.argtypes = [u64, u64, ctypes.c_int, vp, vp, vp, vp]
        _lib.ora_query.restype = u64
        _lib.ora_query.argtypes = [P(Params), vp, vp, u64]
        _lib.ora_peel_core.restype = u64
        _lib.ora_peel_core.argtypes = [u64, u32, vp, vp, u64, vp, vp, vp, vp, P(u32)]
        _lib.ora_finalize.restype = None
        _lib.ora_finalize.argtypes = [u64, u32, vp, vp, vp, vp, vp]
        _lib.ora_decompress.restype = ctypes.c_int
        _lib.ora_decompress.argtypes = [P(Params), vp, vp, u64, vp, vp, vp, vp, vp, P(_Stats)]
        del i32
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def params(d, m, c, k=3, k_bloom=0, L=1024, seed=0, blocks=0) -> Params:
    return Params(int(d), int(m), int(c), int(k), int(k_bloom), int(L), int(blocks),
                  int(seed) & (2**64 - 1))


INDEX_BITMAP = 255  # k_bloom value of the exact bitmap index


def k_bloom_of(p: Params) -> int:
    if p.k_bloom == INDEX_BITMAP:
        return 1
    return p.k_bloom or p.k


def n_words(p: Params) -> int:
    return int(p.m) // 32


# --- hashing (reading R1) ---------------------------------------------------------

def mix64(z: int) -> int:
    return int(lib().ora_mix64(z & (2**64 - 1)))


def hash64(seed: int, dom: int, j: int, i: int) -> int:
    return int(lib().ora_hash(seed & (2**64 - 1), dom, j, i))


def row_map(p: Params, dom: int, j: int, i: int):
    """(row, bias, sign) of input row i under probe j of domain dom."""
    row, bias, sign = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_int()
    lib().ora_row_map(ctypes.byref(p), dom, j, i, ctypes.byref(row), ctypes.byref(bias),
                      ctypes.byref(sign))
    return int(row.value), int(bias.value), int(sign.value)


def cell(p: Params, j: int, q: int):
    """(cell, sign) of coordinate q under Count Sketch hash j."""
    g = ctypes.c_int()
    e = lib().ora_cell(ctypes.byref(p), j, q, ctypes.byref(g))
    return int(e), int(g.value)


def bit(p: Params, j: int, q: int) -> int:
    """Bloom bit of coordinate q under probe j."""
    return int(lib().ora_bit(ctypes.byref(p), j, q))


def validate(p: Params) -> bool:
    return lib().ora_validate(ctypes.byref(p)) == 0


# --- Phase I ---------------------------------------------------------------------

def empty_sketch(p: Params):
    return np.zeros(n_words(p), np.uint32), np.zeros(int(p.c), np.float64)


def compress_dense(p: Params, x: np.ndarray, B=None, Y=None):
    """Alg. 1 Phase I on a dense fp32 gradient; accumulates into (B, Y)."""
    assert validate(p)
    x = np.ascontiguousarray(x, np.float32)
    assert x.shape == (p.d,)
    if B is None:
        B, Y = empty_sketch(p)
    lib().ora_compress_dense(ctypes.byref(p), _ptr(x), _ptr(B), _ptr(Y))
    return B, Y


def compress_coo(p: Params, idx: np.ndarray, val: np.ndarray, B=None, Y=None):
    """Alg. 1 Phase I on a COO gradient (every listed entry is inserted)."""
    assert validate(p)
    idx = np.ascontiguousarray(idx, np.uint32)
    val = np.ascontiguousarray(val, np.float32)
    if B is None:
        B, Y = empty_sketch(p)
    lib().ora_compress_coo(ctypes.byref(p), len(idx), _ptr(idx), _ptr(val), _ptr(B), _ptr(Y))
    return B, Y


def aggregate(Bs, Ys):
    """B = OR_w B_w, Y = sum_w Y_w."""
    Bs = [np.ascontiguousarray(b, np.uint32) for b in Bs]
    Ys = [np.ascontiguousarray(y, np.float64) for y in Ys]
    nw, c = len(Bs[0]), len(Ys[0])
    bp = (ctypes.c_void_p * len(Bs))(*[_ptr(b) for b in Bs])
    yp = (ctypes.c_void_p * len(Ys))(*[_ptr(y) for y in Ys])
    Bo = np.empty(nw, np.uint32)
    Yo = np.empty(c, np.float64)
    lib().ora_aggregate(nw, c, len(Bs), ctypes.addressof(bp), ctypes.addressof(yp), _ptr(Bo), _ptr(Yo))
    return Bo, Yo


# --- Phase II --------------------------------------------------------------------

def query(p: Params, B: np.ndarray) -> np.ndarray:
    """Ascending candidate list."""
    B = np.ascontiguousarray(B, np.uint32)
    n = int(lib().ora_query(ctypes.byref(p), _ptr(B), None, 0))
    cand = np.empty(max(n, 1), np.uint32)
    lib().ora_query(ctypes.byref(p), _ptr(B), _ptr(cand), n)
    return cand[:n]


@dataclass
class PeelResult:
    val: np.ndarray
    peeled: np.ndarray
    round_of: np.ndarray
    residual: np.ndarray
    n_peeled: int
    rounds: int


def peel_core(cells: np.ndarray, signs: np.ndarray, Y: np.ndarray, finalize: bool = True):
    """Peel an explicit incidence cells[n_items, k] / signs[n_items, k]
    over the sketch Y, then (if finalize) estimate unpeeled items by the residual
    median."""
    cells = np.ascontiguousarray(cells, np.uint64)
    signs = np.ascontiguousarray(signs, np.int8)
    n, k = cells.shape
    R = np.array(Y, np.float64, copy=True)
    val = np.zeros(max(n, 1), np.float64)
    peeled = np.zeros(max(n, 1), np.uint8)
    round_of = np.zeros(max(n, 1), np.uint32)
    rounds = ctypes.c_uint32()
    npeeled = lib().ora_peel_core(n, k, _ptr(cells), _ptr(signs), len(R), _ptr(R), _ptr(val),
                                  _ptr(peeled), _ptr(round_of), ctypes.byref(rounds))
    if finalize:
        lib().ora_finalize(n, k, _ptr(cells), _ptr(signs), _ptr(R), _ptr(peeled), _ptr(val))
    return PeelResult(val[:n], peeled[:n].astype(bool), round_of[:n], R, int(npeeled),
                      int(rounds.value))


@dataclass
class Decoded:
    cand: np.ndarray
    val: np.ndarray
    peeled: np.ndarray
    round_of: np.ndarray
    dense: np.ndarray | None
    stats: Stats


def decompress(p: Params, B: np.ndarray, Y: np.ndarray, dense: bool = True, cap: int | None = None):
    """Alg. 1 Phase II: query, peel, estimate, densify."""
    B = np.ascontiguousarray(B, np.uint32)
    Y = np.ascontiguousarray(Y, np.float64)
    if cap is None:
        cap = int(lib().ora_query(ctypes.byref(p), _ptr(B), None, 0))
    cand = np.zeros(max(cap, 1), np.uint32)
    val = np.zeros(max(cap, 1), np.float64)
    peeled = np.zeros(max(cap, 1), np.uint8)
    round_of = np.zeros(max(cap, 1), np.uint32)
    out = np.zeros(p.d, np.float64) if dense else None
    st = _Stats()
    rc = lib().ora_decompress(ctypes.byref(p), _ptr(B), _ptr(Y), cap, _ptr(cand), _ptr(val),
                              _ptr(peeled), _ptr(round_of), _ptr(out) if dense else None,
                              ctypes.byref(st))
    if rc != 0:
        raise ValueError("oracle: invalid parameters")
    n = min(int(st.n_cand), cap)
    stats = Stats(int(st.n_cand), int(st.n_peeled), int(st.rounds), bool(st.success),
                  bool(st.overflow))
    return Decoded(cand[:n], val[:n], peeled[:n].astype(bool), round_of[:n], out, stats)


def pipeline(p: Params, xs, dense: bool = True):
    """Compress every worker, aggregate, recover."""
    Bs, Ys = [], []
    for x in xs:
        B, Y = compress_dense(p, x)
        Bs.append(B)
        Ys.append(Y)
    B, Y = aggregate(Bs, Ys) if len(xs) > 1 else (Bs[0], Ys[0])
    return B, Y, decompress(p, B, Y, dense=dense)
