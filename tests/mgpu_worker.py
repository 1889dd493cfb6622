"""Multi-GPU parity worker (launched by tests/test_gpu_multi.py under torchrun).

Each rank compresses the workers it owns (w % world == rank) into the NVLink
communication buffer, sketch_allreduce makes every rank's sketch the OR/sum over
all ranks, and every rank decodes.  Rank 0 checks against the CPU oracle; all
ranks check that their aggregated sketch bytes and decoded indices/flags are
identical across ranks.  Exit code 0 = pass.
"""
import os
import sys
import zlib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from lhc_inputs import config  # noqa: E402


def sharded(name, law, steps, rank, world, dev, comm="p2p"):
    """NEXT-2: reduce-scatter of per-shard sub-sketches, decode of the own shard,
    all-gather of the decoded lists.  Every rank checks its shard against the
    oracle on that coordinate range; all ranks must hold identical dense sums."""
    import paper_2402_07529_b200 as lhc
    from paper_2402_07529_b200.sizing import shard_plan

    wl = config(name, law=law)
    if name == "tiny":
        wl = config(name, law=law, workers=max(world, 2), d=20_000 * world)
    plan = shard_plan(wl.d, world, wl.density, wl.workers)
    mine = [w for w in range(wl.workers) if w % world == rank]
    xs = [torch.from_numpy(wl.dense(w)).to(dev) for w in mine]
    run = lhc.ShardedAllReduce(plan, seed=0x5BA4D, local_workers=len(xs), device=dev, comm=comm)
    for _ in range(steps):
        dec = run.step(xs)
    torch.cuda.synchronize()
    st = dec.read_stats()
    n = st["n_cand"]
    dense = run.dense.cpu().numpy()
    digest = torch.tensor([zlib.crc32(dense.tobytes())], dtype=torch.int64, device=dev)
    allg = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(allg, digest)
    ok = all(torch.equal(allg[0], a) for a in allg)
    import oracle

    lo, hi = plan.bounds(rank)
    p = run.ps[rank]
    op = oracle.params(p.d, p.m, p.c, p.k, p.k_bloom, p.L, p.seed)
    xs_all = [wl.dense(w) for w in range(wl.workers)]
    Bo, Yo, ref = oracle.pipeline(op, [x[lo:hi] for x in xs_all], dense=True)
    B = run.slots[rank].bitmap.cpu().numpy().view(np.uint32)
    Y = run.slots[rank].counters.cpu().numpy()
    idx = dec.idx[:n].cpu().numpy().view(np.uint32)
    val = dec.val[:n].cpu().numpy()
    ok &= np.array_equal(B, Bo)
    ok &= n == ref.stats.n_cand and np.array_equal(idx, ref.cand)
    ok &= np.array_equal(dec.peeled[:n].cpu().numpy().astype(bool), ref.peeled)
    ok &= st["rounds"] == ref.stats.rounds and st["success"] == ref.stats.success

    def close(a, b):
        if law == "dyadic":
            return np.array_equal(a.astype(np.float64), b)
        return bool(np.all(np.abs(a - b) <= 1e-7 + 1e-5 * np.abs(b)))

    ok &= close(Y, Yo) and close(val, ref.val) and close(dense[lo:hi], ref.dense)
    # the other shards: every rank holds what their owners decoded
    total = np.sum(np.stack(xs_all).astype(np.float64), axis=0)
    if law == "dyadic" and st["success"]:
        ok &= np.array_equal(dense[lo:hi].astype(np.float64), total[lo:hi])
    print(f"mgpu-sharded[{comm}] {name} world={world} rank={rank} n_cand={n} rounds={st['rounds']} "
          f"ok={ok}", flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    # rank 0 additionally checks the assembled dense sum of all shards (dyadic: exact)
    if rank == 0 and law == "dyadic":
        good = bool(np.array_equal(dense.astype(np.float64), total))
        print(f"mgpu-sharded dense == exact sum: {good}", flush=True)
        flag &= torch.tensor([1 if good else 0], device=dev)
    run.close()
    return flag.item() == 1


def sharded_overflow(rank, world, dev, comm="p2p"):
    """a shard whose decode overflows its candidate capacity must not
    leave stale values on the other ranks.  The last shard is made 8x denser than
    the others and the capacity is set between the two candidate counts, so only
    its owner overflows; every rank must then hold NaN on that shard's range and
    the exact sum everywhere else, and the owner's stats must report overflow."""
    import oracle
    import paper_2402_07529_b200 as lhc
    from lhc_inputs import rng_for, values
    from paper_2402_07529_b200.sizing import shard_plan

    W = 2
    d = 60_000 * world
    plan = shard_plan(d, world, 0.01, W)
    xs_all = []
    for w in range(W):
        rng = rng_for(777 + w)
        x = np.zeros(d, np.float32)
        for q in range(world):
            lo, hi = plan.bounds(q)
            rho = 0.08 if q == world - 1 else 0.01
            idx = rng.choice(hi - lo, int(rho * (hi - lo)), replace=False) + lo
            x[idx] = values(rng, len(idx), "dyadic")
        xs_all.append(x)
    s = plan.sizing
    n_cand = []
    for q in range(world):
        lo, hi = plan.bounds(q)
        op = oracle.params(plan.shard_d(q), plan.shard_m(q), s.c, 3, s.k_bloom, 1024, 0x0F0)
        Bq, Yq = oracle.aggregate(*zip(*[oracle.compress_dense(op, x[lo:hi]) for x in xs_all]))
        n_cand.append(len(oracle.query(op, Bq)))
    cap = (max(n_cand[:-1]) + n_cand[-1]) // 2 // 4 * 4
    assert max(n_cand[:-1]) <= cap < n_cand[-1], (n_cand, cap)
    mine = [w for w in range(W) if w % world == rank]
    xs = [torch.from_numpy(xs_all[w]).to(dev) for w in mine] or [torch.zeros(d, device=dev)]
    run = lhc.ShardedAllReduce(plan, seed=0x0F0, cap_cand=cap, local_workers=len(xs), device=dev,
                               comm=comm)
    dec = run.step(xs)
    torch.cuda.synchronize()
    st = dec.read_stats()
    dense = run.dense.cpu().numpy().astype(np.float64)
    total = np.sum(np.stack(xs_all).astype(np.float64), axis=0)
    lo_last, hi_last = plan.bounds(world - 1)
    ok = bool(np.isnan(dense[lo_last:hi_last]).all())
    ok &= bool(np.array_equal(dense[:lo_last], total[:lo_last]))
    if rank == world - 1:
        ok &= bool(st["overflow"]) and not st["success"]
    else:
        ok &= bool(st["success"]) and not st["overflow"]
    print(f"mgpu-sharded-overflow[{comm}] world={world} rank={rank} n_cand={n_cand} cap={cap} "
          f"ok={ok}", flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    run.close()
    return flag.item() == 1


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "ncf"
    law = sys.argv[2] if len(sys.argv) > 2 else "dyadic"
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    mode = sys.argv[4] if len(sys.argv) > 4 else "replicated"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    if mode in ("sharded-overflow", "sharded-nvls-overflow"):
        ok = sharded_overflow(rank, world, dev, "nvls" if "nvls" in mode else "p2p")
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    if mode in ("sharded", "sharded-nvls"):
        ok = sharded(name, law, steps, rank, world, dev, "nvls" if mode == "sharded-nvls" else "p2p")
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    import paper_2402_07529_b200 as lhc

    wl = config(name, law=law)
    if name == "tiny":
        wl = config(name, law=law, workers=max(world, 2))
    s = lhc.size_workload(wl.d, wl.density, wl.workers)
    p = lhc.params(wl.d, s.m, s.c, 3, 0, 1024, 0x1DC0DE)
    mine = [w for w in range(wl.workers) if w % world == rank]
    xs = [torch.from_numpy(wl.dense(w)).to(dev) for w in mine]
    comm = lhc.NvlsComm(p) if mode == "nvls" else lhc.PeerComm(p)
    run = lhc.LosslessAllReduce(p, min(wl.d, int(s.n_cand_expected * 1.5) + 4096),
                                local_workers=len(xs), comm=comm, device=dev)
    for _ in range(steps):  # repeated steps exercise the barrier epochs
        dec = run.step(xs)
    torch.cuda.synchronize()
    st = dec.read_stats()
    n = st["n_cand"]
    B = run.sketch.bitmap.cpu().numpy().view(np.uint32)
    Y = run.sketch.counters.cpu().numpy()
    idx = dec.idx[:n].cpu().numpy().view(np.uint32)
    peeled = dec.peeled[:n].cpu().numpy()
    val = dec.val[:n].cpu().numpy()
    # identical on every rank (the aggregate is reduced once per slice, then copied)
    digest = torch.tensor([zlib.crc32(a.tobytes()) for a in (B, Y, idx, peeled)] + [st["rounds"]],
                          dtype=torch.int64, device=dev)
    allg = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(allg, digest)
    ok = all(torch.equal(allg[0], a) for a in allg)
    if rank == 0:
        import oracle

        op = oracle.params(p.d, p.m, p.c, p.k, p.k_bloom, p.L, p.seed)
        Bo, Yo, ref = oracle.pipeline(op, [wl.dense(w) for w in range(wl.workers)], dense=False)
        ok &= np.array_equal(B, Bo)
        if law == "dyadic":
            ok &= np.array_equal(Y.astype(np.float64), Yo)
            ok &= np.array_equal(val.astype(np.float64), ref.val)
        else:
            ok &= bool(np.all(np.abs(Y - Yo) <= 1e-7 + 1e-5 * np.abs(Yo)))
            ok &= bool(np.all(np.abs(val - ref.val) <= 1e-7 + 1e-5 * np.abs(ref.val)))
        ok &= n == ref.stats.n_cand and np.array_equal(idx, ref.cand)
        ok &= np.array_equal(peeled.astype(bool), ref.peeled)
        ok &= st["rounds"] == ref.stats.rounds and st["success"] == ref.stats.success
        print(f"mgpu {name} world={world} n_cand={n} rounds={st['rounds']} ok={ok}", flush=True)
    if not ok:
        print(f"rank {rank}: mismatch (digests {[a.tolist() for a in allg]})", flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
