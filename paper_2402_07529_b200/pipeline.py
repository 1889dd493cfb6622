"""User-facing objects over the C ABI: sketch buffers, the decoder, the NVLink
peer communicator and the whole Alg. 1 step (compress -> aggregate -> recover).

torch supplies device memory, streams and the process group used once to
exchange CUDA IPC handles; every step of the path runs in liblhc.so's kernels.
"""
from __future__ import annotations

import os

import torch

from . import _lib as L


class Sketch:
    """S(X) = [Y, B] (Alg. 1) in one device buffer laid out as
    [bitmap | counters | signals] (lhc_comm_layout), usable as an all-reduce buffer."""

    def __init__(self, p: L.lhc_params, device="cuda", buf: torch.Tensor | None = None):
        self.p = p
        b_off, y_off, s_off, total = L.lhc_comm_layout(p)
        # zero-initialised: the signal slots must start at zero (include/lhc.h)
        self.buf = torch.zeros(total, dtype=torch.uint8, device=device) if buf is None else buf
        self.bitmap = self.buf[b_off:b_off + p.words * 4].view(torch.int32)
        self.counters = self.buf[y_off:y_off + int(p.c) * 4].view(torch.float32)

    def clear(self, stream=None):
        L.sketch_clear(self.p, self.bitmap, self.counters, stream)

    def compress(self, x: torch.Tensor, nnz_out=None, stream=None):
        """Accumulate the dense gradient x into this sketch (Alg. 1 Phase I)."""
        L.sketch_compress(self.p, x, self.bitmap, self.counters, nnz_out, stream)

    def compress_coo(self, idx: torch.Tensor, val: torch.Tensor, bad_out=None, stream=None):
        """Accumulate a COO gradient; bad_out (device int64[1]) counts idx >= d (skipped)."""
        L.sketch_compress_coo(self.p, idx, val, self.bitmap, self.counters, bad_out, stream)

    @property
    def nbytes(self) -> int:
        return self.p.words * 4 + int(self.p.c) * 4


def aggregate(p: L.lhc_params, sketches, out: Sketch, stream=None):
    """out = OR / sum of the sketches, on one GPU."""
    L.sketch_aggregate(p, [s.bitmap for s in sketches], [s.counters for s in sketches],
                       out.bitmap, out.counters, stream)


class Decoder:
    """Phase II of Alg. 1 with preallocated workspace and outputs."""

    def __init__(self, p: L.lhc_params, cap_cand: int, dense: bool = True, device="cuda",
                 deterministic: bool = False):
        """deterministic=True decodes with sketch_peel_det: values, flags and dense
        output bit-identical across runs, launch geometries and ranks."""
        self.p = p
        self.deterministic = deterministic
        self.cap = int(min(cap_cand, p.d))
        self.ws = torch.empty(L.lhc_decompress_workspace(p, self.cap), dtype=torch.uint8,
                              device=device)
        self.idx = torch.empty(max(self.cap, 1), dtype=torch.int32, device=device)
        self.val = torch.empty(max(self.cap, 1), dtype=torch.float32, device=device)
        self.peeled = torch.empty(max(self.cap, 1), dtype=torch.uint8, device=device)
        self.dense = torch.empty(p.d, dtype=torch.float32, device=device) if dense else None
        self.stats = torch.zeros(L.STATS_BYTES, dtype=torch.uint8, device=device)

    def __call__(self, sketch: Sketch, stream=None):
        L.sketch_decompress(self.p, sketch.bitmap, sketch.counters, self.ws, self.cap, self.idx,
                            self.val, self.peeled, self.dense, self.stats, stream,
                            deterministic=self.deterministic)
        return self

    # the two steps of __call__, separately (for per-kernel timing)
    def query(self, sketch: Sketch, stream=None):
        L.sketch_query(self.p, sketch.bitmap, self.ws, self.cap, self.idx, self.stats, stream)

    def peel(self, sketch: Sketch, stream=None):
        L.sketch_peel(self.p, sketch.counters, self.ws, self.cap, self.idx, self.val, self.peeled,
                      self.dense, self.stats, stream, deterministic=self.deterministic)

    def read_stats(self) -> dict:
        return L.read_stats(self.stats)

    def coo(self):
        """(idx, val, peeled) views of the first n_cand slots (host sync)."""
        n = min(self.read_stats()["n_cand"], self.cap)
        return self.idx[:n], self.val[:n], self.peeled[:n]


def owned_workers(workers: int, rank: int, world: int) -> list[int]:
    """Workers a rank holds: w % world == rank (every worker exactly once)."""
    return [w for w in range(workers) if w % world == rank]


def exchange_handles(handle: bytes, offset: int, group=None):
    """All-gather every rank's (64-byte IPC handle, offset) over the process group;
    returns (handles, offsets) in rank order."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gathered = [None] * world
    dist.all_gather_object(gathered, (bytes(handle), int(offset)), group=group)
    if any(len(g[0]) != 64 for g in gathered):
        raise ValueError("IPC handles must be 64 bytes")
    return [g[0] for g in gathered], [g[1] for g in gathered]


class PeerComm:
    """NVLink P2P all-reduce of a Sketch across the ranks of a process group
    (one process per GPU).  Construction is collective."""

    def __init__(self, p: L.lhc_params, group=None, device=None):
        import torch.distributed as dist

        self.p = p
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.sketch = Sketch(p, device)
        torch.cuda.synchronize()
        handle, offset = L.lhc_ipc_handle(self.sketch.buf)
        handles, offsets = exchange_handles(handle, offset, group)
        self.handle = L.lhc_comm_create(self.rank, self.world, handles, offsets,
                                        self.sketch.buf, p)
        dist.barrier(group=group)

    def allreduce(self, stream=None):
        L.sketch_allreduce(self.handle, stream)

    def close(self):
        if self.handle:
            L.lhc_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NvlsBuffer:
    """A zeroed device buffer bound to an NVSwitch multicast object shared by the
    ranks of a process group (lhc_nvls_open / lhc_nvls_bind); construction is
    collective.  ``buf`` is the local (unicast) view."""

    _serial = 0

    def __init__(self, nbytes: int, group=None, device=None):
        import os

        import torch.distributed as dist

        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        device = device or torch.device("cuda", torch.cuda.current_device())
        NvlsBuffer._serial += 1
        name = [f"lhc-nvls-{os.getpid()}-{NvlsBuffer._serial}"]
        dist.broadcast_object_list(name, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        self.handle = L.lhc_nvls_open(self.rank, self.world, name[0], nbytes)
        dist.barrier(group=group)        # every device added before any binds
        ptr, size = L.lhc_nvls_bind(self.handle)
        dist.barrier(group=group)
        self.buf = L.device_bytes(ptr, size, device)

    def close(self):
        if self.handle:
            torch.cuda.synchronize()
            self.buf = None
            L.lhc_nvls_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NvlsComm:
    """In-switch all-reduce of a Sketch (sketch_allreduce_nvls): drop-in for PeerComm."""

    def __init__(self, p: L.lhc_params, group=None, device=None):
        self.p = p
        _, _, _, total = L.lhc_comm_layout(p)
        self.nvls = NvlsBuffer(total, group, device)
        self.rank, self.world = self.nvls.rank, self.nvls.world
        self.sketch = Sketch(p, buf=self.nvls.buf[:total])

    def allreduce(self, stream=None):
        L.sketch_allreduce_nvls(self.nvls.handle, self.p, stream)

    def close(self):
        self.nvls.close()


def reserve_l2(device=None):
    """The persisting-L2 set-aside the kernels' evict-last hints need (lhc_l2_persist),
    as the fraction LHC_L2_PERSIST gives (default 0: none).  With the whole set-aside
    the VGG19 compress runs 942 -> 774 us (the sketch stays in L2) but the decode
    slows more (1.53 -> 2.20 ms), even with the pinned lines demoted between the
    phases, so it is off by default."""
    frac = float(os.environ.get("LHC_L2_PERSIST", "0"))
    if frac <= 0:
        return 0
    with torch.cuda.device(torch.device(device) if device is not None else torch.cuda.current_device()):
        return L.l2_persist(frac)


class LosslessAllReduce:
    """One step of Alg. 1 for the workers a rank holds: compress every local
    gradient into the rank's sketch (homomorphic accumulation), make the
    sketch the all-rank OR/sum (NVLink P2P, or nothing on one GPU), and decode.

    ``per_worker=True`` keeps one sketch per local worker (the per-worker payload
    of the paper's API) and aggregates them on the GPU before the exchange.

    Every rank decodes the identical aggregated sketch.  With the default decode
    (sketch_peel) the flags, rounds and candidate set are identical on all ranks
    but fp32 values may differ in the last bits (residual deductions land in a
    scheduling-dependent order); ``deterministic=True`` decodes with
    sketch_peel_det, whose values are bit-identical on every rank and run."""

    def __init__(self, p: L.lhc_params, cap_cand: int, local_workers: int = 1,
                 per_worker: bool = True, comm: PeerComm | None = None, dense: bool = True,
                 device="cuda", deterministic: bool = False):
        self.p = p
        self.comm = comm
        reserve_l2(device)
        self.sketch = comm.sketch if comm is not None else Sketch(p, device)
        self.per_worker = per_worker and local_workers > 1
        self.worker_sketches = [Sketch(p, device) for _ in range(local_workers)] \
            if self.per_worker else []
        self.decoder = Decoder(p, cap_cand, dense=dense, device=device, deterministic=deterministic)

    def step(self, xs, stream=None):
        """xs: list of dense fp32 device gradients of this rank's workers."""
        return self._step([(x,) for x in xs], stream)

    def step_coo(self, coos, stream=None):
        """coos: list of (idx int32, val fp32) device COO gradients of this rank's
        workers (sketch_compress_coo); same result as step() on the dense form."""
        return self._step(list(coos), stream)

    def _step(self, items, stream):
        targets = self.worker_sketches if self.per_worker else [self.sketch]
        # cleared in reverse so the first sketches compressed are the last written (in L2)
        L.sketch_clear_batch(self.p, [t.bitmap for t in targets[::-1]], [t.counters for t in targets[::-1]],
                             stream)
        if self.per_worker:
            dst = self.worker_sketches[:len(items)]
        else:
            dst = [self.sketch] * len(items)
        if all(len(it) == 1 for it in items):   # dense: one launch for all workers
            L.sketch_compress_batch(self.p, [it[0] for it in items], [t.bitmap for t in dst],
                                    [t.counters for t in dst], stream=stream)
        else:
            for sk, it in zip(dst, items):
                sk.compress_coo(it[0], it[1], stream=stream)
        if self.per_worker:
            aggregate(self.p, self.worker_sketches, self.sketch, stream)
        if self.comm is not None and self.comm.world > 1:
            self.comm.allreduce(stream)
        return self.decoder(self.sketch, stream)


class _SlotSketch:
    """A Sketch-like view of slot q of a sharded buffer (bitmap and counters of one shard)."""

    def __init__(self, p: L.lhc_params, buf: torch.Tensor, base: int, y_off: int, words: int):
        self.p = p
        # the view spans the slot's whole bitmap region (the largest shard's words)
        self.bitmap = buf[base:base + words * 4].view(torch.int32)
        self.counters = buf[base + y_off:base + y_off + int(p.c) * 4].view(torch.float32)

    clear = Sketch.clear
    compress = Sketch.compress
    compress_coo = Sketch.compress_coo


class ShardedAllReduce:
    """Alg. 1 with a sharded decode (DESIGN.md NEXT-2): coordinate shard q has its
    own sub-sketch; every rank compresses its workers into all shards, the NVLink
    reduce-scatter leaves rank r with the aggregate of shard r, rank r decodes
    only shard r, and an all-gather of the decoded (index, value) lists gives
    every rank the identical dense sum.  Construction is collective; with one
    rank (no group) every shard is decoded locally.

    plan: sizing.ShardPlan with plan.shards == world size (or any shard count on
    one process, which then decodes every shard itself)."""

    def __init__(self, plan, k: int = 3, L_rows: int = 1024, seed: int = 0, cap_cand: int = 0,
                 local_workers: int = 1, per_worker: bool = True, group=None, device=None,
                 comm: str = "p2p", deterministic: bool = False):
        import torch.distributed as dist

        self.plan = plan
        s = plan.sizing
        distributed = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if distributed else 0
        self.world = dist.get_world_size(group) if distributed else 1
        if plan.shards != self.world and self.world != 1:
            raise ValueError(f"plan has {plan.shards} shards, world size is {self.world}")
        device = device or torch.device("cuda", torch.cuda.current_device())
        reserve_l2(device)
        self.ps = [L.params(plan.shard_d(q), plan.shard_m(q), s.c, k, s.k_bloom, L_rows, seed)
                   for q in range(plan.shards)]
        self.cap = int(cap_cand) or int(1.25 * s.n_cand_expected) + 4096
        # a multiple of 4 (the gather slots hold 16-byte vectors): the decoders and the
        # communicator then agree on when a shard's decode overflowed
        self.cap = (min(self.cap, plan.width) + 3) // 4 * 4
        self.slot_bytes, self.y_off, total = L.lhc_shard_layout(self.ps[0], self.world, self.cap)
        if comm not in ("p2p", "nvls"):
            raise ValueError("comm must be 'p2p' or 'nvls'")
        self.comm = comm if self.world > 1 else "none"
        self.nvls = None
        if self.comm == "nvls":   # the sharded buffer lives in the multicast-bound memory
            self.nvls = NvlsBuffer(total, group, device)
            self.buf = self.nvls.buf[:total]
        else:
            self.buf = torch.zeros(total, dtype=torch.uint8, device=device)
        words = self.ps[0].words
        self.slots = [_SlotSketch(self.ps[q], self.buf, q * self.slot_bytes, self.y_off, words)
                      for q in range(plan.shards)]
        self.per_worker = per_worker and local_workers > 1
        self.worker_bufs = []
        if self.per_worker:
            for _ in range(local_workers):
                b = torch.zeros(self.slot_bytes * plan.shards, dtype=torch.uint8, device=device)
                self.worker_bufs.append(
                    [_SlotSketch(self.ps[q], b, q * self.slot_bytes, self.y_off, words)
                     for q in range(plan.shards)])
        self.dense = torch.empty(plan.d, dtype=torch.float32, device=device)
        # the shards this process decodes: its own, or all of them on one rank
        self.owned = [self.rank] if self.world > 1 else list(range(plan.shards))
        self.decoders = {}
        for q in self.owned:
            lo, hi = plan.bounds(q)
            dec = Decoder(self.ps[q], self.cap, dense=False, device=device, deterministic=deterministic)
            dec.dense = self.dense[lo:hi]
            self.decoders[q] = dec
        self.decoder = self.decoders[self.owned[0]]
        self.handle = None
        if self.comm == "p2p":
            torch.cuda.synchronize()
            handle, offset = L.lhc_ipc_handle(self.buf)
            handles, offsets = exchange_handles(handle, offset, group)
            self.handle = L.lhc_shard_comm_create(self.rank, self.world, handles, offsets,
                                                  self.buf, self.ps[0], self.cap)
            dist.barrier(group=group)

    def shard_input(self, x: torch.Tensor, q: int) -> torch.Tensor:
        lo, hi = self.plan.bounds(q)
        return x[lo:hi]

    def step(self, xs, stream=None):
        """xs: dense fp32 device gradients (length d) of this rank's workers."""
        return self._step([(x,) for x in xs], stream)

    def step_coo(self, coos, stream=None):
        """coos: per local worker, a list of G (idx int32, val fp32) device COO
        gradients, one per shard, indices relative to the shard's first coordinate
        (split_coo); same result as step() on the dense form."""
        return self._step([tuple(c) for c in coos], stream, coo=True)

    def split_coo(self, idx, val):
        """Host helper: split a sorted COO gradient (numpy) into per-shard lists with
        shard-relative indices, for step_coo."""
        import numpy as np

        out = []
        for q in range(self.plan.shards):
            lo, hi = self.plan.bounds(q)
            a, b = np.searchsorted(idx, [lo, hi])
            out.append(((idx[a:b] - lo).astype(idx.dtype), val[a:b]))
        return out

    def _step(self, items, stream, coo=False):
        G = self.plan.shards
        targets = self.worker_bufs[:len(items)] if self.per_worker else [self.slots] * len(items)
        clear = self.worker_bufs if self.per_worker else [self.slots]
        flat = [sk for bufs in clear for sk in bufs]
        L.sketch_clear_batch(self.ps[0], [sk.bitmap for sk in flat[::-1]], [sk.counters for sk in flat[::-1]],
                             stream)
        if coo:
            for bufs, item in zip(targets, items):
                for q, sk in enumerate(bufs):
                    sk.compress_coo(item[q][0], item[q][1], stream=stream)
        else:   # every (worker, shard) pair in one launch
            xs, bms, ys, ds = [], [], [], []
            for bufs, item in zip(targets, items):
                for q, sk in enumerate(bufs):
                    xs.append(self.shard_input(item[0], q))
                    bms.append(sk.bitmap)
                    ys.append(sk.counters)
                    ds.append(self.plan.shard_d(q))
            L.sketch_compress_batch(self.ps[0], xs, bms, ys, ds=ds, stream=stream)
        if self.per_worker:
            for q in range(G):
                L.sketch_aggregate(self.ps[q], [b[q].bitmap for b in self.worker_bufs],
                                   [b[q].counters for b in self.worker_bufs],
                                   self.slots[q].bitmap, self.slots[q].counters, stream)
        self.reduce_scatter(stream)
        for q in self.owned:
            self.decoders[q](self.slots[q], stream)
        dec = self.decoder
        self.allgather(stream)
        return dec

    def reduce_scatter(self, stream=None):
        if self.comm == "p2p":
            L.sketch_reduce_scatter(self.handle, stream)
        elif self.comm == "nvls":
            L.sketch_reduce_scatter_nvls(self.nvls.handle, self.ps[0], self.cap, stream)

    def allgather(self, stream=None):
        dec = self.decoder
        if self.comm == "p2p":
            L.sketch_allgather_decoded(self.handle, dec.idx, dec.val, dec.stats, self.plan.width,
                                       self.plan.d, self.dense, stream)
        elif self.comm == "nvls":
            L.sketch_allgather_decoded_nvls(self.nvls.handle, self.ps[0], self.cap, dec.idx,
                                            dec.val, dec.stats, self.plan.width, self.plan.d,
                                            self.dense, stream)

    def close(self):
        if self.handle:
            L.lhc_comm_destroy(self.handle)
            self.handle = None
        if getattr(self, "nvls", None) is not None:
            self.nvls.close()
            self.nvls = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
