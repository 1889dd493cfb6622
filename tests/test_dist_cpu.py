"""world_size-2 gloo tests of the N>1 host logic on CPU (-m "not gpu").

The GPU exchange itself (NVLink P2P) needs GPUs; here the same orchestration
runs over a real gloo process group: worker ownership, the IPC-handle exchange
protocol, and the homomorphic exchange semantics (OR of bitmaps, sum of
counters across ranks == the single-process aggregate), with the
oracle standing in for the per-rank compression."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from lhc_inputs import config
        from paper_2402_07529_b200.pipeline import exchange_handles, owned_workers
        from paper_2402_07529_b200.sizing import size_workload

        # ownership covers every worker exactly once
        mine = owned_workers(8, rank, world)
        allw = [None] * world
        dist.all_gather_object(allw, mine)
        assert sorted(sum(allw, [])) == list(range(8))

        # handle exchange protocol (fake 64-byte handles)
        h = bytes([rank]) * 64
        handles, offsets = exchange_handles(h, 256 * rank)
        assert handles == [bytes([r]) * 64 for r in range(world)]
        assert offsets == [256 * r for r in range(world)]

        # homomorphic exchange: per-rank sketches OR/summed across ranks
        wl = config("tiny", law="dyadic", workers=4, d=60_000)
        s = size_workload(wl.d, wl.density, wl.workers)
        p = oracle.params(wl.d, s.m, s.c, 3, 0, 1024, 77)
        B, Y = oracle.empty_sketch(p)
        for w in owned_workers(wl.workers, rank, world):
            oracle.compress_dense(p, wl.dense(w), B, Y)
        Yt = torch.from_numpy(Y.copy())
        dist.all_reduce(Yt)
        Bs = [torch.zeros(len(B), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(Bs, torch.from_numpy(B.view(np.int32).copy()))
        Bor = np.bitwise_or.reduce(np.stack([b.numpy().view(np.uint32) for b in Bs]), axis=0)
        Bref, Yref, ref = oracle.pipeline(p, [wl.dense(w) for w in range(wl.workers)])
        assert np.array_equal(Bor, Bref)
        assert np.array_equal(Yt.numpy(), Yref)
        dec = oracle.decompress(p, Bor, Yt.numpy())
        assert dec.stats.success and np.array_equal(dec.dense, ref.dense)

        # sharded decode protocol (NEXT-2a, reading R23) with the oracle standing in
        # for the kernels: per-shard sketches, reduce-scatter (sum/OR, keep the own
        # shard), decode the own shard, all-gather the decoded lists, assemble
        from paper_2402_07529_b200.sizing import shard_plan

        plan = shard_plan(wl.d, world, wl.density, wl.workers)
        ps = [oracle.params(plan.shard_d(r), plan.shard_m(r), plan.sizing.c, 3, 0, 1024, 77)
              for r in range(world)]
        lo, hi = plan.bounds(rank)
        mine = {}
        for r in range(world):
            Br, Yr = oracle.empty_sketch(ps[r])
            a, b = plan.bounds(r)
            for w in owned_workers(wl.workers, rank, world):
                oracle.compress_dense(ps[r], wl.dense(w)[a:b], Br, Yr)
            Yt = torch.from_numpy(Yr.copy())
            dist.all_reduce(Yt)                      # reduce (rank r keeps shard r)
            Bs = [torch.zeros(len(Br), dtype=torch.int32) for _ in range(world)]
            dist.all_gather(Bs, torch.from_numpy(Br.view(np.int32).copy()))
            if r == rank:
                Bo = np.bitwise_or.reduce(np.stack([t.numpy().view(np.uint32) for t in Bs]), axis=0)
                mine = oracle.decompress(ps[r], Bo, Yt.numpy())
        assert mine.stats.success
        lists = [None] * world
        dist.all_gather_object(lists, (mine.cand.astype(np.int64).tolist(), mine.val.tolist()))
        dense = np.zeros(wl.d)
        for r, (idx, val) in enumerate(lists):
            dense[plan.bounds(r)[0] + np.asarray(idx, dtype=np.int64)] = val
        exact = np.sum(np.stack([wl.dense(w).astype(np.float64) for w in range(wl.workers)]), axis=0)
        assert np.array_equal(dense, exact)              # lossless (dyadic law: exact sums)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(v == "ok" for v in res.values()), res
