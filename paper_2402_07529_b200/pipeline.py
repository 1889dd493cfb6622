"""User-facing objects over the C ABI: sketch buffers, the decoder, the NVLink
peer communicator and the whole Alg. 1 step (compress -> aggregate -> recover).

torch supplies device memory, streams and the process group used once to
exchange CUDA IPC handles; every step of the path runs in liblhc.so's kernels.
"""
from __future__ import annotations

import torch

from . import _lib as L


class Sketch:
    """S(X) = [Y, B] (Alg. 1) in one device buffer laid out as
    [bitmap | counters | signals] (lhc_comm_layout), usable as an all-reduce buffer."""

    def __init__(self, p: L.lhc_params, device="cuda"):
        self.p = p
        b_off, y_off, s_off, total = L.lhc_comm_layout(p)
        # zero-initialised: the signal slots must start at zero (include/lhc.h)
        self.buf = torch.zeros(total, dtype=torch.uint8, device=device)
        self.bitmap = self.buf[b_off:b_off + p.words * 4].view(torch.int32)
        self.counters = self.buf[y_off:y_off + int(p.c) * 4].view(torch.float32)

    def clear(self, stream=None):
        L.sketch_clear(self.p, self.bitmap, self.counters, stream)

    def compress(self, x: torch.Tensor, nnz_out=None, stream=None):
        """Accumulate the dense gradient x into this sketch (Alg. 1 Phase I)."""
        L.sketch_compress(self.p, x, self.bitmap, self.counters, nnz_out, stream)

    def compress_coo(self, idx: torch.Tensor, val: torch.Tensor, stream=None):
        L.sketch_compress_coo(self.p, idx, val, self.bitmap, self.counters, stream)

    @property
    def nbytes(self) -> int:
        return self.p.words * 4 + int(self.p.c) * 4


def aggregate(p: L.lhc_params, sketches, out: Sketch, stream=None):
    """out = OR / sum of the sketches, on one GPU."""
    L.sketch_aggregate(p, [s.bitmap for s in sketches], [s.counters for s in sketches],
                       out.bitmap, out.counters, stream)


class Decoder:
    """Phase II of Alg. 1 with preallocated workspace and outputs."""

    def __init__(self, p: L.lhc_params, cap_cand: int, dense: bool = True, device="cuda"):
        self.p = p
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
                            self.val, self.peeled, self.dense, self.stats, stream)
        return self

    # the two steps of __call__, separately (for per-kernel timing)
    def query(self, sketch: Sketch, stream=None):
        L.sketch_query(self.p, sketch.bitmap, self.ws, self.cap, self.idx, self.stats, stream)

    def peel(self, sketch: Sketch, stream=None):
        L.sketch_peel(self.p, sketch.counters, self.ws, self.cap, self.idx, self.val, self.peeled,
                      self.dense, self.stats, stream)

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


class LosslessAllReduce:
    """One step of Alg. 1 for the workers a rank holds: compress every local
    gradient into the rank's sketch (homomorphic accumulation), make the
    sketch the all-rank OR/sum (NVLink P2P, or nothing on one GPU), and decode.

    ``per_worker=True`` keeps one sketch per local worker (the per-worker payload
    of the paper's API) and aggregates them on the GPU before the exchange."""

    def __init__(self, p: L.lhc_params, cap_cand: int, local_workers: int = 1,
                 per_worker: bool = True, comm: PeerComm | None = None, dense: bool = True,
                 device="cuda"):
        self.p = p
        self.comm = comm
        self.sketch = comm.sketch if comm is not None else Sketch(p, device)
        self.per_worker = per_worker and local_workers > 1
        self.worker_sketches = [Sketch(p, device) for _ in range(local_workers)] \
            if self.per_worker else []
        self.decoder = Decoder(p, cap_cand, dense=dense, device=device)

    def step(self, xs, stream=None):
        """xs: list of dense fp32 device gradients of this rank's workers."""
        return self._step([(x,) for x in xs], stream)

    def step_coo(self, coos, stream=None):
        """coos: list of (idx int32, val fp32) device COO gradients of this rank's
        workers (sketch_compress_coo); same result as step() on the dense form."""
        return self._step(list(coos), stream)

    def _step(self, items, stream):
        def compress(sk, item):
            if len(item) == 1:
                sk.compress(item[0], stream=stream)
            else:
                sk.compress_coo(item[0], item[1], stream=stream)

        if self.per_worker:
            for sk, item in zip(self.worker_sketches, items):
                sk.clear(stream)
                compress(sk, item)
            aggregate(self.p, self.worker_sketches, self.sketch, stream)
        else:
            self.sketch.clear(stream)
            for item in items:
                compress(self.sketch, item)
        if self.comm is not None and self.comm.world > 1:
            self.comm.allreduce(stream)
        return self.decoder(self.sketch, stream)
