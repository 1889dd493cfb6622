"""ctypes binding of ``liblhc.so`` (include/lhc.h) — argument marshalling only.

Every function here has the name and argument order of the C ABI; torch tensors
are accepted where the ABI takes device pointers and are checked for device,
dtype, size and contiguity before the call.  All compute runs in the sm_100a
kernels of ``csrc/``; there is no CPU fallback: if the library is missing or a
call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblhc.so")
# experiment hook: load another build of the same sources (never a fallback)
LIB_PATH = os.environ.get("LHC_LIB", LIB_PATH)

LHC_OK, LHC_EINVAL, LHC_ECAPACITY, LHC_ECUDA, LHC_ECOMM = 0, 1, 2, 3, 4


class LhcError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed with status {code}: {msg}")
        self.code = code


class lhc_params(ctypes.Structure):
    """``lhc_params`` of include/lhc.h."""

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

    def __repr__(self):
        return (f"lhc_params(d={self.d}, m={self.m}, c={self.c}, k={self.k}, "
                f"k_bloom={self.k_bloom}, L={self.L}, blocks={self.blocks}, seed={self.seed:#x})")

    @property
    def kb(self) -> int:
        return self.k_bloom or self.k

    @property
    def words(self) -> int:
        return int(self.m) // 32

    @property
    def nrows(self) -> int:
        return (int(self.d) + self.L - 1) // self.L


class lhc_stats(ctypes.Structure):
    _fields_ = [
        ("n_cand", ctypes.c_uint64),
        ("n_peeled", ctypes.c_uint64),
        ("rounds", ctypes.c_uint32),
        ("success", ctypes.c_int32),
        ("overflow", ctypes.c_int32),
        ("entries", ctypes.c_uint32),
    ]


STATS_BYTES = ctypes.sizeof(lhc_stats)
assert STATS_BYTES == 32

_lib = None

EXPORTS = [
    "lhc_validate", "lhc_last_error", "lhc_bitmap_words", "lhc_decompress_workspace",
    "sketch_hash_rows", "sketch_clear", "sketch_compress", "sketch_compress_coo",
    "sketch_aggregate", "lhc_comm_layout", "lhc_ipc_handle", "lhc_comm_create",
    "sketch_allreduce", "lhc_comm_destroy", "sketch_decompress", "lhc_last_launch_count",
    "sketch_query", "sketch_peel", "sketch_peel_det", "sketch_decompress_det", "lhc_shard_layout", "lhc_shard_comm_create",
    "sketch_reduce_scatter", "sketch_allgather_decoded", "sketch_compress_batch",
    "sketch_clear_batch", "lhc_nvls_open", "lhc_nvls_bind", "sketch_allreduce_nvls",
    "sketch_reduce_scatter_nvls", "sketch_allgather_decoded_nvls", "lhc_nvls_destroy",
    "lhc_l2_persist",
]


def lib() -> ctypes.CDLL:
    """Load liblhc.so (raises if it was not built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make` or __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER(lhc_params)
        vp, u64, u32, i32, sz = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                 ctypes.c_int, ctypes.c_size_t)
        sig = {
            "lhc_validate": (i32, [P]),
            "lhc_last_error": (ctypes.c_char_p, []),
            "lhc_bitmap_words": (u64, [P]),
            "lhc_decompress_workspace": (sz, [P, u64]),
            "sketch_hash_rows": (i32, [P, u32, u64, vp, vp]),
            "sketch_clear": (i32, [P, vp, vp, vp]),
            "sketch_compress": (i32, [P, vp, vp, vp, vp, vp]),
            "sketch_compress_coo": (i32, [P, u64, vp, vp, vp, vp, vp, vp]),
            "sketch_aggregate": (i32, [P, i32, vp, vp, vp, vp, vp]),
            "lhc_comm_layout": (i32, [P, ctypes.POINTER(sz), ctypes.POINTER(sz),
                                      ctypes.POINTER(sz), ctypes.POINTER(sz)]),
            "lhc_ipc_handle": (i32, [vp, vp, ctypes.POINTER(u64)]),
            "lhc_comm_create": (i32, [i32, i32, vp, vp, vp, sz, P, ctypes.POINTER(vp)]),
            "sketch_allreduce": (i32, [vp, vp]),
            "lhc_comm_destroy": (None, [vp]),
            "sketch_decompress": (i32, [P, vp, vp, vp, sz, u64, vp, vp, vp, vp, vp, vp]),
            "lhc_last_launch_count": (i32, []),
            "sketch_query": (i32, [P, vp, vp, sz, u64, vp, vp, vp]),
            "sketch_peel": (i32, [P, vp, vp, sz, u64, vp, vp, vp, vp, vp, vp]),
            "sketch_peel_det": (i32, [P, vp, vp, sz, u64, vp, vp, vp, vp, vp, vp]),
            "sketch_decompress_det": (i32, [P, vp, vp, vp, sz, u64, vp, vp, vp, vp, vp, vp]),
            "lhc_shard_layout": (i32, [P, i32, u64, ctypes.POINTER(sz), ctypes.POINTER(sz),
                                       ctypes.POINTER(sz)]),
            "lhc_shard_comm_create": (i32, [i32, i32, vp, vp, vp, sz, P, u64,
                                            ctypes.POINTER(vp)]),
            "sketch_reduce_scatter": (i32, [vp, vp]),
            "sketch_allgather_decoded": (i32, [vp, vp, vp, vp, u64, u32, vp, vp]),
            "sketch_compress_batch": (i32, [P, i32, vp, vp, vp, vp, vp, vp]),
            "sketch_clear_batch": (i32, [P, i32, vp, vp, vp]),
            "lhc_nvls_open": (i32, [i32, i32, ctypes.c_char_p, sz, ctypes.POINTER(vp)]),
            "lhc_nvls_bind": (i32, [vp, ctypes.POINTER(vp), ctypes.POINTER(sz)]),
            "sketch_allreduce_nvls": (i32, [vp, P, vp]),
            "sketch_reduce_scatter_nvls": (i32, [vp, P, u64, vp]),
            "sketch_allgather_decoded_nvls": (i32, [vp, P, u64, vp, vp, vp, u64, u32, vp, vp]),
            "lhc_nvls_destroy": (None, [vp]),
            "lhc_l2_persist": (i32, [ctypes.c_double, ctypes.POINTER(sz)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().lhc_last_error().decode()


def last_launch_count() -> int:
    return int(lib().lhc_last_launch_count())


def l2_persist(fraction: float = 1.0) -> int:
    """Reserve `fraction` of the device's persisting-L2 set-aside, which the kernels'
    evict-last hints need to take effect (lhc_l2_persist); returns the bytes set."""
    out = ctypes.c_size_t(0)
    _check("lhc_l2_persist", lib().lhc_l2_persist(float(fraction), ctypes.byref(out)))
    return int(out.value)


def _check(fn: str, rc: int):
    if rc != LHC_OK:
        raise LhcError(fn, rc, last_error())


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev(t: torch.Tensor | None, dtype, numel: int | None, name: str) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs {numel}")
    return t.data_ptr()


def params(d, m, c, k=3, k_bloom=0, L=1024, seed=0, blocks=0) -> lhc_params:
    return lhc_params(int(d), int(m), int(c), int(k), int(k_bloom), int(L), int(blocks),
                      int(seed) & (2**64 - 1))


def lhc_validate(p: lhc_params) -> bool:
    return lib().lhc_validate(ctypes.byref(p)) == LHC_OK


def lhc_decompress_workspace(p: lhc_params, cap_cand: int) -> int:
    n = int(lib().lhc_decompress_workspace(ctypes.byref(p), int(cap_cand)))
    if n == 0:
        raise LhcError("lhc_decompress_workspace", LHC_EINVAL, last_error())
    return n


def sketch_hash_rows(p: lhc_params, dom: int, n_rows: int, out: torch.Tensor, stream=None):
    kk = p.k if dom == 0 else p.kb
    ptr = _dev(out, torch.int32, 2 * n_rows * kk, "out")
    _check("sketch_hash_rows",
           lib().sketch_hash_rows(ctypes.byref(p), dom, n_rows, ptr, _stream(stream)))


def sketch_clear(p: lhc_params, bitmap: torch.Tensor, counters: torch.Tensor, stream=None):
    _check("sketch_clear", lib().sketch_clear(
        ctypes.byref(p), _dev(bitmap, torch.int32, p.words, "bitmap"),
        _dev(counters, torch.float32, p.c, "counters"), _stream(stream)))


def sketch_compress(p: lhc_params, x: torch.Tensor, bitmap: torch.Tensor,
                    counters: torch.Tensor, nnz_out: torch.Tensor | None = None, stream=None):
    _check("sketch_compress", lib().sketch_compress(
        ctypes.byref(p), _dev(x, torch.float32, p.d, "x"),
        _dev(bitmap, torch.int32, p.words, "bitmap"),
        _dev(counters, torch.float32, p.c, "counters"),
        _dev(nnz_out, torch.int64, 1, "nnz_out"), _stream(stream)))


def _ptrs(ts, dtype, numel, name):
    return (ctypes.c_void_p * len(ts))(*[_dev(t, dtype, numel, name) for t in ts])


def sketch_compress_batch(p: lhc_params, xs, bitmaps, counters, ds=None,
                          nnz_out: torch.Tensor | None = None, stream=None):
    """xs[b] (len ds[b] <= p.d, default p.d) into (bitmaps[b], counters[b]), one launch."""
    n = len(xs)
    if not (n == len(bitmaps) == len(counters)) or n < 1:
        raise ValueError("need as many inputs as sketches")
    ds = [int(p.d)] * n if ds is None else [int(v) for v in ds]
    xp = (ctypes.c_void_p * n)(*[_dev(x, torch.float32, dd, "xs[]") for x, dd in zip(xs, ds)])
    dp = (ctypes.c_uint32 * n)(*ds)
    bp = _ptrs(bitmaps, torch.int32, None, "bitmaps[]")  # kept alive across the call
    yp = _ptrs(counters, torch.float32, p.c, "counters[]")
    _check("sketch_compress_batch", lib().sketch_compress_batch(
        ctypes.byref(p), n, ctypes.addressof(xp), ctypes.addressof(dp), ctypes.addressof(bp),
        ctypes.addressof(yp), _dev(nnz_out, torch.int64, 1, "nnz_out"), _stream(stream)))


def sketch_clear_batch(p: lhc_params, bitmaps, counters, stream=None):
    n = len(bitmaps)
    if n != len(counters) or n < 1:
        raise ValueError("need as many bitmaps as counter arrays")
    bp = _ptrs(bitmaps, torch.int32, p.words, "bitmaps[]")
    yp = _ptrs(counters, torch.float32, p.c, "counters[]")
    _check("sketch_clear_batch", lib().sketch_clear_batch(
        ctypes.byref(p), n, ctypes.addressof(bp), ctypes.addressof(yp), _stream(stream)))


def sketch_compress_coo(p: lhc_params, idx: torch.Tensor, val: torch.Tensor,
                        bitmap: torch.Tensor, counters: torch.Tensor,
                        bad_out: torch.Tensor | None = None, stream=None):
    """bad_out (int64[1] on the device, nullable) accumulates the number of entries
    with idx >= d, which are skipped."""
    nnz = idx.numel()
    if val.numel() != nnz:
        raise ValueError("idx and val differ in length")
    _check("sketch_compress_coo", lib().sketch_compress_coo(
        ctypes.byref(p), nnz, _dev(idx, torch.int32, nnz, "idx"),
        _dev(val, torch.float32, nnz, "val"), _dev(bitmap, torch.int32, p.words, "bitmap"),
        _dev(counters, torch.float32, p.c, "counters"), _dev(bad_out, torch.int64, 1, "bad_out"),
        _stream(stream)))


def sketch_aggregate(p: lhc_params, bitmaps, counters, out_bitmap: torch.Tensor,
                     out_counters: torch.Tensor, stream=None):
    n = len(bitmaps)
    if n != len(counters) or n < 1:
        raise ValueError("need as many bitmaps as counter arrays")
    bp = (ctypes.c_void_p * n)(*[_dev(b, torch.int32, p.words, "bitmaps[]") for b in bitmaps])
    yp = (ctypes.c_void_p * n)(*[_dev(y, torch.float32, p.c, "counters[]") for y in counters])
    _check("sketch_aggregate", lib().sketch_aggregate(
        ctypes.byref(p), n, ctypes.addressof(bp), ctypes.addressof(yp),
        _dev(out_bitmap, torch.int32, p.words, "out_bitmap"),
        _dev(out_counters, torch.float32, p.c, "out_counters"), _stream(stream)))


def sketch_decompress(p: lhc_params, bitmap: torch.Tensor, counters: torch.Tensor,
                      ws: torch.Tensor, cap_cand: int, out_idx: torch.Tensor,
                      out_val: torch.Tensor, out_peeled: torch.Tensor,
                      out_dense: torch.Tensor | None, stats: torch.Tensor, stream=None,
                      deterministic: bool = False):
    name = "sketch_decompress_det" if deterministic else "sketch_decompress"
    _check(name, getattr(lib(), name)(
        ctypes.byref(p), _dev(bitmap, torch.int32, p.words, "bitmap"),
        _dev(counters, torch.float32, p.c, "counters"), _dev(ws, torch.uint8, None, "ws"),
        ws.numel(), int(cap_cand), _dev(out_idx, torch.int32, cap_cand, "out_idx"),
        _dev(out_val, torch.float32, cap_cand, "out_val"),
        _dev(out_peeled, torch.uint8, cap_cand, "out_peeled"),
        _dev(out_dense, torch.float32, p.d, "out_dense"),
        _dev(stats, torch.uint8, STATS_BYTES, "stats"), _stream(stream)))


def sketch_query(p: lhc_params, bitmap, ws, cap_cand, out_idx, stats, stream=None):
    _check("sketch_query", lib().sketch_query(
        ctypes.byref(p), _dev(bitmap, torch.int32, p.words, "bitmap"),
        _dev(ws, torch.uint8, None, "ws"), ws.numel(), int(cap_cand),
        _dev(out_idx, torch.int32, cap_cand, "out_idx"),
        _dev(stats, torch.uint8, STATS_BYTES, "stats"), _stream(stream)))


def sketch_peel(p: lhc_params, counters, ws, cap_cand, out_idx, out_val, out_peeled, out_dense,
                stats, stream=None, deterministic: bool = False):
    """deterministic=True: sketch_peel_det (values independent of launch geometry)."""
    name = "sketch_peel_det" if deterministic else "sketch_peel"
    _check(name, getattr(lib(), name)(
        ctypes.byref(p), _dev(counters, torch.float32, p.c, "counters"),
        _dev(ws, torch.uint8, None, "ws"), ws.numel(), int(cap_cand),
        _dev(out_idx, torch.int32, cap_cand, "out_idx"),
        _dev(out_val, torch.float32, cap_cand, "out_val"),
        _dev(out_peeled, torch.uint8, cap_cand, "out_peeled"),
        _dev(out_dense, torch.float32, p.d, "out_dense"),
        _dev(stats, torch.uint8, STATS_BYTES, "stats"), _stream(stream)))


def lhc_comm_layout(p: lhc_params):
    vals = [ctypes.c_size_t() for _ in range(4)]
    _check("lhc_comm_layout", lib().lhc_comm_layout(ctypes.byref(p), *[ctypes.byref(v) for v in vals]))
    return tuple(int(v.value) for v in vals)


def lhc_ipc_handle(buf: torch.Tensor) -> tuple[bytes, int]:
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    _check("lhc_ipc_handle", lib().lhc_ipc_handle(buf.data_ptr(), h, ctypes.byref(off)))
    return h.raw, int(off.value)


def lhc_comm_create(rank: int, world: int, handles: list[bytes], offsets: list[int],
                    buf: torch.Tensor, p: lhc_params) -> int:
    hb = ctypes.create_string_buffer(b"".join(handles), 64 * world)
    ob = (ctypes.c_uint64 * world)(*offsets)
    out = ctypes.c_void_p()
    _check("lhc_comm_create", lib().lhc_comm_create(
        rank, world, hb, ob, buf.data_ptr(), buf.numel() * buf.element_size(), ctypes.byref(p),
        ctypes.byref(out)))
    return out.value


def sketch_allreduce(comm: int, stream=None):
    _check("sketch_allreduce", lib().sketch_allreduce(comm, _stream(stream)))


def lhc_shard_layout(ps: lhc_params, world: int, cap_items: int):
    """(slot_bytes, counters_off, total_bytes) of a sharded communication buffer."""
    vals = [ctypes.c_size_t() for _ in range(3)]
    _check("lhc_shard_layout", lib().lhc_shard_layout(ctypes.byref(ps), int(world), int(cap_items),
                                                      *[ctypes.byref(v) for v in vals]))
    return tuple(int(v.value) for v in vals)


def lhc_shard_comm_create(rank: int, world: int, handles: list[bytes], offsets: list[int],
                          buf: torch.Tensor, ps: lhc_params, cap_items: int) -> int:
    hb = ctypes.create_string_buffer(b"".join(handles), 64 * world)
    ob = (ctypes.c_uint64 * world)(*offsets)
    out = ctypes.c_void_p()
    _check("lhc_shard_comm_create", lib().lhc_shard_comm_create(
        rank, world, hb, ob, buf.data_ptr(), buf.numel() * buf.element_size(), ctypes.byref(ps),
        int(cap_items), ctypes.byref(out)))
    return out.value


def sketch_reduce_scatter(comm: int, stream=None):
    _check("sketch_reduce_scatter", lib().sketch_reduce_scatter(comm, _stream(stream)))


def sketch_allgather_decoded(comm: int, idx: torch.Tensor, val: torch.Tensor, stats: torch.Tensor,
                             shard_width: int, d: int, dense: torch.Tensor, stream=None):
    """n_items is read on the device from stats.n_cand (lhc_stats offset 0)."""
    _check("sketch_allgather_decoded", lib().sketch_allgather_decoded(
        comm, _dev(idx, torch.int32, None, "idx"), _dev(val, torch.float32, None, "val"),
        _dev(stats, torch.uint8, STATS_BYTES, "stats"), int(shard_width), int(d),
        _dev(dense, torch.float32, d, "dense"), _stream(stream)))


def lhc_nvls_open(rank: int, world: int, rendezvous: str, nbytes: int) -> int:
    out = ctypes.c_void_p()
    _check("lhc_nvls_open", lib().lhc_nvls_open(rank, world, rendezvous.encode(), int(nbytes),
                                                ctypes.byref(out)))
    return out.value


def lhc_nvls_bind(h: int) -> tuple[int, int]:
    ptr, size = ctypes.c_void_p(), ctypes.c_size_t()
    _check("lhc_nvls_bind", lib().lhc_nvls_bind(h, ctypes.byref(ptr), ctypes.byref(size)))
    return int(ptr.value), int(size.value)


def sketch_allreduce_nvls(h: int, p: lhc_params, stream=None):
    _check("sketch_allreduce_nvls", lib().sketch_allreduce_nvls(h, ctypes.byref(p), _stream(stream)))


def sketch_reduce_scatter_nvls(h: int, ps: lhc_params, cap_items: int, stream=None):
    _check("sketch_reduce_scatter_nvls",
           lib().sketch_reduce_scatter_nvls(h, ctypes.byref(ps), int(cap_items), _stream(stream)))


def sketch_allgather_decoded_nvls(h: int, ps: lhc_params, cap_items: int, idx, val, stats,
                                  shard_width: int, d: int, dense, stream=None):
    _check("sketch_allgather_decoded_nvls", lib().sketch_allgather_decoded_nvls(
        h, ctypes.byref(ps), int(cap_items), _dev(idx, torch.int32, None, "idx"),
        _dev(val, torch.float32, None, "val"), _dev(stats, torch.uint8, STATS_BYTES, "stats"),
        int(shard_width), int(d), _dev(dense, torch.float32, d, "dense"), _stream(stream)))


def lhc_nvls_destroy(h: int):
    lib().lhc_nvls_destroy(h)


class _DevPtr:
    """__cuda_array_interface__ view of a device allocation owned by liblhc.so."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def device_bytes(ptr: int, nbytes: int, device) -> torch.Tensor:
    """A uint8 tensor over nbytes at ptr (no copy; the caller keeps the owner alive)."""
    return torch.as_tensor(_DevPtr(ptr, nbytes), device=device)


def lhc_comm_destroy(comm: int):
    lib().lhc_comm_destroy(comm)


def read_stats(stats: torch.Tensor) -> dict:
    """Copy a device lhc_stats to the host (synchronises the current stream)."""
    raw = bytes(stats.cpu().numpy().tobytes())
    s = lhc_stats.from_buffer_copy(raw)
    return dict(n_cand=int(s.n_cand), n_peeled=int(s.n_peeled), rounds=int(s.rounds),
                success=bool(s.success), overflow=bool(s.overflow), entries=int(s.entries))
