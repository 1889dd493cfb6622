"""Small runs of every kernel of liblhc.so, for compute-sanitizer.

    compute-sanitizer --tool memcheck   python tools/sanitize_run.py tiny
    compute-sanitizer --tool racecheck  python tools/sanitize_run.py 1m
    compute-sanitizer --tool synccheck  python tools/sanitize_run.py tiny

Kernels exercised: k_hash_rows, k_clear, k_compress_dense (batched, repeated
targets), k_compress_coo (incl. out-of-range entries), k_aggregate, k_query<3>,
k_pair_count / k_pair_scan / k_pair_scatter / k_build_cells (rows, compact),
k_peel<3> (insert, rows, compact), k_peel_blocked, k_pair_sort + k_peel_rows<3>
(deterministic decode), k_peel<0> / k_peel_rows<0> / k_query<0> (run-time k).
Each decode is checked against the CPU oracle (flags, rounds, values under the
dyadic law); the script exits non-zero on any mismatch.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2402_07529_b200 as lhc  # noqa: E402
from lhc_inputs import rng_for, support, values  # noqa: E402


def workers(d, nnz, W, seed):
    xs = []
    for w in range(W):
        rng = rng_for(seed + w)
        idx = support(rng, d, nnz)
        x = np.zeros(d, np.float32)
        x[idx] = values(rng, len(idx), "dyadic")
        xs.append(x)
    return xs


def check(name, dec, ref):
    st = dec.read_stats()
    n = st["n_cand"]
    ok = n == ref.stats.n_cand and st["rounds"] == ref.stats.rounds
    ok &= st["success"] == ref.stats.success and st["n_peeled"] == ref.stats.n_peeled
    ok &= np.array_equal(dec.idx[:n].cpu().numpy().view(np.uint32), ref.cand)
    ok &= np.array_equal(dec.peeled[:n].cpu().numpy().astype(bool), ref.peeled)
    ok &= np.array_equal(dec.val[:n].cpu().numpy().astype(np.float64), ref.val)
    print(f"  {name}: n_cand={n} rounds={st['rounds']} success={st['success']} ok={ok}", flush=True)
    return ok


def run(d, nnz, W, L=1024, k=3, blocks=0, seed=7):
    s = lhc.size_workload(d, nnz / d, W, L=L, k=k)
    c = s.c
    if blocks:
        S = max(1, -(-c // (blocks * k * L)))
        c = blocks * S * k * L
    p = lhc.params(d, s.m, c, k, 0, L, seed, blocks)
    op = oracle.params(p.d, p.m, p.c, p.k, p.k_bloom, p.L, p.seed, p.blocks)
    xs = workers(d, nnz, W, 100 + seed)
    _, _, ref = oracle.pipeline(op, xs)
    ok = True
    dev = torch.device("cuda", 0)
    # hash kernel
    out = torch.empty(2 * 64 * k, dtype=torch.int32, device=dev)
    lhc.sketch_hash_rows(p, 0, 64, out)
    # dense compress (per-worker sketches + aggregate) and every decode path
    modes = [("frontier/default", {}, False), ("frontier/rows", {"LHC_CELL_BUILD": "rows"}, False),
             ("frontier/compact", {"LHC_CELL_BUILD": "compact"}, False),
             ("frontier/insert", {"LHC_CELL_BUILD": "insert"}, False), ("deterministic", {}, True)]
    for name, env, det in modes:
        for kk, vv in env.items():
            os.environ[kk] = vv
        run_ = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W, deterministic=det)
        dec = run_.step([torch.from_numpy(x).to(dev) for x in xs])
        torch.cuda.synchronize()
        ok &= check(f"d={d} k={k} L={L} blocks={blocks} {name}", dec, ref)
        for kk in env:
            os.environ.pop(kk)
    # COO compress (with out-of-range entries, skipped and counted) into one sketch
    sk = lhc.Sketch(p, dev)
    sk.clear()
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    for x in xs:
        idx = np.flatnonzero(x).astype(np.uint32)
        idx2 = np.concatenate([idx, np.array([d, d + 7], np.uint32)])
        val2 = np.concatenate([x[idx], np.ones(2, np.float32)])
        sk.compress_coo(torch.from_numpy(idx2.view(np.int32)).to(dev), torch.from_numpy(val2).to(dev), bad)
    dec = lhc.Decoder(p, d, device=dev)
    dec(sk)
    torch.cuda.synchronize()
    ok &= int(bad.item()) == 2 * W
    ok &= check(f"d={d} coo", dec, ref)
    return ok


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    torch.cuda.set_device(0)
    ok = True
    if which == "tiny":
        ok &= run(10_000, 100, 2)
        ok &= run(10_000, 100, 2, L=32, k=4)          # run-time k kernels
        ok &= run(40_000, 400, 2, L=128, blocks=4)    # blocked sketch: k_peel_blocked
    else:
        ok &= run(1_000_003, 10_000, 3)
        ok &= run(1_000_003, 10_000, 3, L=128, blocks=16)
    print("SANITIZE-RUN", "OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
