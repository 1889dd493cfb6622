"""GPU parity: every step of the sm_100a path, through the C ABI, against the CPU
oracle on the same seeded inputs (-m gpu).

Bars (north star): bitmaps, candidate lists, peel flags, success and rounds
bit-exact; fp32 values within 1e-5 relative + 1e-7 absolute of the fp64 oracle
(|gpu - ora| <= 1e-7 + 1e-5 |ora|); under the dyadic law every fp32 sum is exact,
so values must be bit-identical too.
"""
import numpy as np
import pytest

from lhc_inputs import config, rng_for, support, values

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-7


@pytest.fixture(scope="module")
def lhc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2402_07529_b200 as lhc

    lhc.lib()
    return lhc


def U(t):
    return t.cpu().numpy().view(np.uint32)


def F(t):
    return t.cpu().numpy().astype(np.float64)


def gpu_params(lhc, d, m, c, k=3, kb=0, L=1024, seed=0):
    return lhc.params(d, m, c, k, kb, L, seed)


def ora_params(ora, p):
    return ora.params(p.d, p.m, p.c, p.k, p.k_bloom, p.L, p.seed, p.blocks)


def make_workers(d, nnz, W, seed, law="dyadic", structure="uniform", run=64, sigma=1e-3):
    xs = []
    for w in range(W):
        rng = rng_for(seed + w)
        idx = support(rng, d, nnz, structure, run)
        x = np.zeros(d, np.float32)
        x[idx] = values(rng, len(idx), law, sigma)
        xs.append(x)
    return xs


def assert_values(gpu, ref, exact):
    if exact:
        assert np.array_equal(gpu, ref)
    else:
        err = np.abs(gpu - ref)
        bad = err > ATOL + RTOL * np.abs(ref)
        assert not bad.any(), (int(bad.sum()), float(err.max()))


# ---------------------------------------------------------------- hash kernel --

@pytest.mark.parametrize("L", [32, 128, 1024])
def test_hash_rows_bit_exact(lhc, L):
    # the frozen row-map table (tests/golden/rowmap.json, written by
    # tools/make_golden_rowmap.py from oracle/ only; the oracle is pinned to it
    # in tests/test_oracle.py::test_row_map_golden_table)
    import json
    import os

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rowmap.json")))
    (t,) = [t for t in g["tables"] if t["L"] == L and t["d"] == 5_000_000]
    p = gpu_params(lhc, t["d"], 3 * L * t["S_B"], 3 * L * t["S_Y"], L=L, seed=t["seed"])
    n = 3000
    for dom in (0, 1):
        out = torch.empty(2 * n * 3, dtype=torch.int32, device="cuda")
        lhc.sketch_hash_rows(p, dom, n, out)
        got = U(out).reshape(n, 3, 2)
        ent = [e for e in t["entries"] if e[0] == dom]
        assert len(ent) == 3 * len(range(0, n, 7))
        for _, j, i, row, bias, sign in ent:
            assert got[i, j, 0] == row
            assert got[i, j, 1] == (bias | ((1 << 31) if sign < 0 else 0))


# ------------------------------------------------------------------ compress --

CASES = [
    # d, nnz per worker, W, L, structure
    (10_000, 100, 2, 1024, "uniform"),          # tiny config
    (1_000_003, 10_000, 3, 1024, "uniform"),    # many tiles + ragged tail
    (1_000_003, 10_000, 2, 32, "uniform"),      # smallest batch width
    (777_777, 30_000, 4, 256, "runs"),          # runs, L=256
    (4099, 4099, 1, 64, "uniform"),             # fully dense, tail < 4
]


@pytest.mark.parametrize("d,nnz,W,L,structure", CASES)
@pytest.mark.parametrize("law", ["dyadic", "gauss"])
def test_compress_dense(lhc, ora, d, nnz, W, L, structure, law):
    s = lhc.size_workload(d, nnz / d, W, L=L)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=77 + L)
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, W, 1000 + d % 97, law, structure)
    sk = lhc.Sketch(p)
    sk.clear()
    nnz_out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for x in xs:
        sk.compress(torch.from_numpy(x).cuda(), nnz_out)
    B, Y = None, None
    for x in xs:
        B, Y = ora.compress_dense(op, x, B, Y)
    assert np.array_equal(U(sk.bitmap), B)
    assert_values(F(sk.counters), Y, exact=(law == "dyadic"))
    assert int(nnz_out.item()) == sum(int((x != 0).sum()) for x in xs)


def test_step_coo_equals_step(lhc, ora):
    """LosslessAllReduce.step_coo (COO boundary) == step (dense boundary) == oracle."""
    d, nnz, W, L = 1_000_003, 10_000, 4, 1024
    s = lhc.size_workload(d, nnz / d, W, L=L)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=0xC00)
    xs = make_workers(d, nnz, W, 55, "dyadic")
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W)
    coos = []
    for x in xs:
        idx = np.flatnonzero(x).astype(np.uint32)
        coos.append((torch.from_numpy(idx.view(np.int32)).cuda(), torch.from_numpy(x[idx]).cuda()))
    dec = run.step_coo(coos)
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(ora_params(ora, p), xs)
    assert np.array_equal(U(run.sketch.bitmap), B)
    compare_decode(ora, dec, ref, exact=True)


def test_compress_coo(lhc, ora):
    d, L = 900_001, 512
    s = lhc.size_workload(d, 0.02, 1, L=L)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=5)
    rng = rng_for(42)
    idx = support(rng, d, 18_000, "runs", 64)
    val = values(rng, len(idx), "dyadic")
    val[::97] = 0.0  # listed zeros are still inserted
    sk = lhc.Sketch(p)
    sk.clear()
    sk.compress_coo(torch.from_numpy(idx.view(np.int32)).cuda(), torch.from_numpy(val).cuda())
    B, Y = ora.compress_coo(ora_params(ora, p), idx, val)
    assert np.array_equal(U(sk.bitmap), B)
    assert np.array_equal(F(sk.counters), Y)


@pytest.mark.parametrize("index", ["bloom", "bitmap"])
def test_compress_coo_out_of_range_flagged(lhc, ora, index):
    """Entries with idx >= d are skipped (nothing written: with the exact bitmap index
    such an index would address a word past the bitmap) and counted in bad_out."""
    d, L = 100_003, 1024
    s = lhc.size_workload(d, 0.02, 1, L=L)
    from paper_2402_07529_b200.sizing import INDEX_BITMAP
    kb = INDEX_BITMAP if index == "bitmap" else 0
    m = -(-d // L) * L if index == "bitmap" else s.m
    p = gpu_params(lhc, d, m, s.c, kb=kb, L=L, seed=6)
    rng = rng_for(43)
    idx = support(rng, d, 2_000, "uniform")
    val = values(rng, len(idx), "dyadic")
    bad_idx = np.array([d, d + 5, 2**32 - 1, 3 * d], np.uint32)
    all_idx = np.concatenate([idx, bad_idx])
    all_val = np.concatenate([val, np.ones(4, np.float32)])
    # guard words past the end of the bitmap and the counters
    bm = torch.zeros(p.words + 64, dtype=torch.int32, device="cuda")
    ct = torch.zeros(int(p.c) + 256, dtype=torch.float32, device="cuda")
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    lhc.sketch_compress_coo(p, torch.from_numpy(all_idx.view(np.int32)).cuda(),
                            torch.from_numpy(all_val).cuda(), bm, ct, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 4
    B, Y = ora.compress_coo(ora_params(ora, p), idx, val)
    assert np.array_equal(U(bm[:p.words]), B)
    assert np.array_equal(F(ct[:int(p.c)]), Y)
    assert not U(bm[p.words:]).any() and not F(ct[int(p.c):]).any()


@pytest.mark.parametrize("law", ["dyadic", "gauss"])
def test_negative_zero_and_exact_cancellation(lhc, ora, law):
    """R22: -0.0 is a zero (not inserted; "true indicates non-zero"); R12:
    coordinates where the workers' values cancel exactly stay candidates and recover
    an exact 0 (footnote P:L188).  Everything against the oracle."""
    d, nnz, W, L = 200_003, 3_000, 3, 1024
    s = lhc.size_workload(d, nnz / d, W, L=L)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=0xC0C0)
    xs = make_workers(d, nnz, W, 4242, law)
    rng = rng_for(99)
    # -0.0 at zeros of every worker (still zeros)
    for x in xs:
        zeros = np.flatnonzero(x == 0)
        x[rng.choice(zeros, 500, replace=False)] = -0.0
    # exact cancellation between workers 0 and 1 at 200 coordinates only they hold
    only = np.flatnonzero((xs[0] == 0) & (xs[1] == 0) & (xs[2] == 0))
    pos = rng.choice(only, 200, replace=False)
    v = values(rng, 200, law)  # same law as the rest (fp32 counters: |error| ~ |v| 2^-24)
    xs[0][pos] = v
    xs[1][pos] = -v
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(ora_params(ora, p), xs)
    assert np.array_equal(U(run.sketch.bitmap), B)
    st = compare_decode(ora, dec, ref, exact=(law == "dyadic"))
    assert st["success"]
    cand = set(ref.cand.tolist())
    assert all(int(q) in cand for q in pos)       # cancelled coordinates stay candidates ...
    dense = F(dec.dense)
    if law == "dyadic":                           # ... and recover an exact 0 (fp32 sums exact)
        assert np.all(dense[pos] == 0.0)
    else:                                         # ... or 0 within the tolerance (compare_decode)
        assert np.all(np.abs(dense[pos]) <= ATOL)
    # -0.0 coordinates set no index bit: with the exact bitmap they are not candidates
    from paper_2402_07529_b200.sizing import INDEX_BITMAP

    pb = gpu_params(lhc, d, -(-d // L) * L, s.c, kb=INDEX_BITMAP, L=L, seed=0xC0C1)
    runb = lhc.LosslessAllReduce(pb, cap_cand=d, local_workers=W)
    decb = runb.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    nb = decb.read_stats()["n_cand"]
    support = np.flatnonzero(np.any(np.stack(xs) != 0, axis=0))  # -0.0 != 0 is False
    assert np.array_equal(U(decb.idx[:nb]), support.astype(np.uint32))


def test_aggregate(lhc, ora):
    d, L, W = 500_000, 1024, 5
    s = lhc.size_workload(d, 0.01, W)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=9)
    op = ora_params(ora, p)
    xs = make_workers(d, 5000, W, 77)
    sks = []
    for x in xs:
        sk = lhc.Sketch(p)
        sk.clear()
        sk.compress(torch.from_numpy(x).cuda())
        sks.append(sk)
    out = lhc.Sketch(p)
    lhc.aggregate(p, sks, out)
    ref = [ora.compress_dense(op, x) for x in xs]
    B, Y = ora.aggregate([r[0] for r in ref], [r[1] for r in ref])
    assert np.array_equal(U(out.bitmap), B)
    assert np.array_equal(F(out.counters), Y)
    # in place (out aliases input 0)
    lhc.aggregate(p, sks, sks[0])
    assert np.array_equal(U(sks[0].bitmap), B)


# ---------------------------------------------------------------- decompress --

def run_decode(lhc, p, B, Y, cap=None, dense=True, det=False):
    """Decode oracle-independent sketch bytes B (u32) / Y (fp32) on the GPU."""
    sk = lhc.Sketch(p)
    sk.bitmap.copy_(torch.from_numpy(B.view(np.int32)))
    sk.counters.copy_(torch.from_numpy(Y.astype(np.float32)))
    dec = lhc.Decoder(p, cap if cap is not None else p.d, dense=dense, deterministic=det)
    dec(sk)
    torch.cuda.synchronize()
    return dec


def compare_decode(ora, dec, ref, exact):
    st = dec.read_stats()
    assert st["n_cand"] == ref.stats.n_cand
    assert st["overflow"] == ref.stats.overflow
    if ref.stats.overflow:
        assert not st["success"]
        return st
    n = st["n_cand"]
    assert np.array_equal(U(dec.idx[:n]), ref.cand)
    assert np.array_equal(dec.peeled[:n].cpu().numpy().astype(bool), ref.peeled)
    assert st["n_peeled"] == ref.stats.n_peeled
    assert st["rounds"] == ref.stats.rounds
    assert st["success"] == ref.stats.success
    assert_values(F(dec.val[:n]), ref.val, exact)
    if dec.dense is not None and ref.dense is not None:
        dense = F(dec.dense)
        assert_values(dense, ref.dense, exact)
        cand = np.zeros(len(dense), bool)
        cand[ref.cand] = True
        assert not dense[~cand].any()  # exact zeros off the candidate set
    return st


@pytest.mark.parametrize("d,nnz,W,L,structure", CASES)
@pytest.mark.parametrize("law", ["dyadic", "gauss"])
def test_pipeline(lhc, ora, d, nnz, W, L, structure, law):
    s = lhc.size_workload(d, nnz / d, W, L=L)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=0x5EED + d)
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, W, 31 + d % 13, law, structure)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(op, xs)
    assert np.array_equal(U(run.sketch.bitmap), B)
    assert_values(F(run.sketch.counters), Y, law == "dyadic")
    st = compare_decode(ora, dec, ref, law == "dyadic")
    if law == "dyadic" and st["success"]:
        assert np.array_equal(F(dec.dense), np.sum(np.stack(xs).astype(np.float64), axis=0))


@pytest.mark.parametrize("build", ["rows", "compact", "split", "insert"])
@pytest.mark.parametrize("d,nnz,W,L,structure", CASES)
def test_cell_build_paths(lhc, ora, d, nnz, W, L, structure, build, monkeypatch):
    """Both ways of building the peeling state (per-candidate reductions, or by
    destination row from the query masks) decode identically."""
    monkeypatch.setenv("LHC_CELL_BUILD", build)
    s = lhc.size_workload(d, nnz / d, W, L=L)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=0xB0B + d)
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, W, 17 + d % 11, "dyadic", structure)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(op, xs)
    compare_decode(ora, dec, ref, exact=True)


@pytest.mark.parametrize("build", ["default", "split"])
@pytest.mark.parametrize("gamma", [0.9, 1.1, 1.2, 1.25, 1.5])
def test_decode_threshold_sweep(lhc, ora, gamma, build, monkeypatch):
    # near and below the peeling threshold: flags, rounds and the median fallback
    # (also through the two-pass peel of the split state)
    if build != "default":
        monkeypatch.setenv("LHC_CELL_BUILD", build)
    d, L, n = 2_000_000, 1024, 40_000
    rng = rng_for(int(gamma * 100))
    idx = support(rng, d, n)
    x = np.zeros(d, np.float32)
    x[idx] = values(rng, n, "dyadic")
    m = 3 * L * ((12 * n) // (3 * L))
    c = 3 * L * max(1, int(round(gamma * n / (3 * L))))
    p = gpu_params(lhc, d, m, c, L=L, seed=int(gamma * 1000))
    op = ora_params(ora, p)
    B, Y = ora.compress_dense(op, x)
    ref = ora.decompress(op, B, Y)
    dec = run_decode(lhc, p, B, Y)
    # the GPU decodes fp32 counters; dyadic sums are exact so Y is the same bytes
    compare_decode(ora, dec, ref, exact=True)


@pytest.mark.parametrize("det", [False, True])
def test_overflow_and_caps(lhc, ora, det):
    d, L = 300_000, 1024
    p = gpu_params(lhc, d, 3 * L * 8, 3 * L * 16, L=L, seed=3)
    op = ora_params(ora, p)
    x = np.zeros(d, np.float32)
    x[::40] = 0.5
    B, Y = ora.compress_dense(op, x)
    n_c = len(ora.query(op, B))
    for cap in (10, n_c - 1, n_c, n_c + 5):
        ref = ora.decompress(op, B, Y, cap=cap)
        dec = run_decode(lhc, p, B, Y, cap=cap, det=det)
        compare_decode(ora, dec, ref, exact=True)


@pytest.mark.parametrize("L", [32, 64, 1024])
def test_query_mask_patterns(lhc, ora, L):
    """Query phase 2 works on 128-word groups (4096 coordinates), per word slot
    lane-serially or warp-cooperatively: a fully set group, runs of 64 and 256, sparse
    coordinates, a ragged last group (d not a multiple of 4096) and caps that cut a
    group in the middle; candidate list (and its truncated prefix) bit-exact."""
    d = 4096 * 37 + 1000 + 3
    rng = rng_for(4096 + L)
    x = np.zeros(d, np.float32)
    x[8192:12288] = 0.25                                  # one whole group
    for r in range(40):                                   # runs of 64 and 256
        a = 20000 + 1500 * r
        x[a:a + (64 if r % 2 else 256)] = -0.5
    sp = rng.choice(d, d // 100, replace=False)           # 1 % sparse
    x[sp] = 0.125
    x[d - 3:] = 1.0                                       # the ragged tail
    n = int(np.count_nonzero(x))
    s = lhc.size_workload(d, n / d, 1, L=L)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=0xA11 + L)
    op = ora_params(ora, p)
    B, Y = ora.compress_dense(op, x)
    cand = ora.query(op, B)
    assert len(cand) >= n
    ref = ora.decompress(op, B, Y)
    compare_decode(ora, run_decode(lhc, p, B, Y), ref, exact=True)
    for cap in (len(cand) - 1, len(cand) // 2 + 7, 4096 + 5):
        dec = run_decode(lhc, p, B, Y, cap=cap)
        st = dec.read_stats()
        assert st["n_cand"] == len(cand) and st["overflow"] and not st["success"]
        assert np.array_equal(U(dec.idx[:cap]), cand[:cap])


@pytest.mark.parametrize("det", [False, True])
def test_empty_and_degenerate(lhc, ora, det):
    L = 1024
    p = gpu_params(lhc, 5000, 3 * L, 3 * L, L=L, seed=1)
    op = ora_params(ora, p)
    B = np.zeros(p.words, np.uint32)
    Y = np.zeros(p.c, np.float64)
    dec = run_decode(lhc, p, B, Y, det=det)
    st = dec.read_stats()
    assert st["n_cand"] == 0 and st["success"] and st["rounds"] == 0
    assert not F(dec.dense).any()
    # d = 1
    p1 = gpu_params(lhc, 1, 3 * 32, 3 * 32, L=32, seed=2)
    x = np.array([0.25], np.float32)
    B, Y, ref = ora.pipeline(ora_params(ora, p1), [x])
    run = lhc.LosslessAllReduce(p1, cap_cand=1, deterministic=det)
    dec = run.step([torch.from_numpy(x).cuda()])
    torch.cuda.synchronize()
    compare_decode(ora, dec, ref, exact=True)
    assert F(dec.dense).tolist() == [0.25]


def test_determinism_of_indices_and_flags(lhc):
    d, L = 2_000_000, 1024
    s = lhc.size_workload(d, 0.01, 4)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=11)
    xs = [torch.from_numpy(x).cuda() for x in make_workers(d, 20_000, 4, 8, "gauss")]
    outs = []
    for _ in range(2):
        run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=4)
        dec = run.step(xs)
        torch.cuda.synchronize()
        st = dec.read_stats()
        n = st["n_cand"]
        outs.append((U(run.sketch.bitmap).copy(), U(dec.idx[:n]).copy(),
                     dec.peeled[:n].cpu().numpy().copy(), st["rounds"]))
    assert all(np.array_equal(a, b) for a, b in zip(outs[0][:3], outs[1][:3]))
    assert outs[0][3] == outs[1][3]


# ------------------------------------------------ exact bitmap index (NEXT-1) --

@pytest.mark.parametrize("d,nnz,W,L", [(10_000, 100, 2, 1024), (1_000_003, 10_000, 3, 1024),
                                      (777_777, 30_000, 4, 32)])
@pytest.mark.parametrize("law", ["dyadic", "gauss"])
def test_pipeline_exact_bitmap(lhc, ora, d, nnz, W, L, law):
    from paper_2402_07529_b200.sizing import INDEX_BITMAP

    s = lhc.size_workload(d, nnz / d, W, L=L, k_bloom=INDEX_BITMAP)
    p = gpu_params(lhc, d, s.m, s.c, kb=INDEX_BITMAP, L=L, seed=0xB17 + d)
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, W, 91 + d % 7, law)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(op, xs)
    assert np.array_equal(U(run.sketch.bitmap), B)
    assert_values(F(run.sketch.counters), Y, law == "dyadic")
    compare_decode(ora, dec, ref, law == "dyadic")


@pytest.mark.parametrize("frac", [0.70, 0.80, 0.856, 0.90, 0.95])
def test_vgg_table1_density_recovery_sweep(lhc, ora, frac):
    """Fig. 3-style single-GPU recovery at VGG19's Table 1 sparsity (30.4 % zeros,
    P:L322-344): one worker, exact bitmap index, counter array swept through c/d
    around the 85.6 % threshold. Below it the peel stalls and the median
    fallback decides values; every flag, round count and value must still equal
    the oracle's (dyadic values: bit-exact)."""
    from paper_2402_07529_b200.sizing import INDEX_BITMAP

    d, L = 1 << 20, 1024
    nnz = int(round(0.696 * d))
    s = lhc.size_workload(d, nnz / d, 1, L=L, k_bloom=INDEX_BITMAP)
    c = 3 * L * max(1, int(round(frac * d / (3 * L))))
    p = gpu_params(lhc, d, s.m, c, kb=INDEX_BITMAP, L=L, seed=0x344 + int(frac * 1000))
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, 1, 344, "dyadic")
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=1)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(op, xs)
    assert np.array_equal(U(run.sketch.bitmap), B)
    st = compare_decode(ora, dec, ref, exact=True)
    if frac >= 0.95:
        assert st["success"]
    if frac <= 0.70:
        assert not st["success"]


# ------------------------------------------------- BASELINE.json full sizes --

FULL = [
    ("ncf", {}),
    ("ncf", {"index": "bitmap"}),
    ("lstm", {}),
    ("bert", {"density": 0.01}),
    ("bert", {"density": 0.02}),
    ("bert", {"density": 0.05}),
    ("bert", {"density": 0.10}),
    ("bert", {"workers": 2}),
    ("bert", {"workers": 4}),
    ("vgg", {}),
    ("vgg", {"per_worker": True}),
]


@pytest.mark.slow
@pytest.mark.parametrize("name,over", FULL,
                         ids=[f"{n}-" + "-".join(f"{k}{v}" for k, v in o.items()) for n, o in FULL])
def test_full_size_configs(lhc, ora, name, over):
    """The bench's launch configuration (all of a rank's workers compressed into its
    one sketch, one decode; or per-worker sketches aggregated on the GPU) at the
    configs' full sizes — BERT over its 1/2/5/10 % density and 2/4/8-worker sweeps —
    compared in full with the oracle."""
    from paper_2402_07529_b200.sizing import INDEX_BITMAP

    over = dict(over)
    kb = INDEX_BITMAP if over.pop("index", "bloom") == "bitmap" else 0
    per_worker = over.pop("per_worker", False)
    wl = config(name, **over)
    s = lhc.size_workload(wl.d, wl.density, wl.workers, k_bloom=kb)
    p = gpu_params(lhc, wl.d, s.m, s.c, kb=kb, seed=0x1DC0DE)
    op = ora_params(ora, p)
    xs = [wl.dense(w) for w in range(wl.workers)]
    run = lhc.LosslessAllReduce(p, cap_cand=int(s.n_cand_expected * 1.5) + 1024,
                                local_workers=wl.workers, per_worker=per_worker)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(op, xs)
    assert np.array_equal(U(run.sketch.bitmap), B)
    assert_values(F(run.sketch.counters), Y, exact=False)
    st = compare_decode(ora, dec, ref, exact=False)
    assert st["success"]


@pytest.mark.slow
@pytest.mark.parametrize("gamma", [1.10, 1.20, 1.22, 1.25, 1.30, 1.50])
def test_vgg_gamma_sweep(lhc, ora, gamma):
    """VGG19-shaped sketch-size sweep near the peeling threshold (dyadic values:
    bit-exact everything, including the fallback estimates)."""
    wl = config("vgg", law="dyadic")
    s = lhc.size_workload(wl.d, wl.density, wl.workers, gamma=gamma)
    p = gpu_params(lhc, wl.d, s.m, s.c, seed=0x1DC0DE)
    op = ora_params(ora, p)
    xs = [wl.dense(w) for w in range(wl.workers)]
    run = lhc.LosslessAllReduce(p, cap_cand=int(s.n_cand_expected * 1.5), local_workers=wl.workers)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(op, xs, dense=False)
    assert np.array_equal(U(run.sketch.bitmap), B)
    compare_decode(ora, dec, ref, exact=True)


# ---------------------------------------- sharded layout, one process (NEXT-2) --

@pytest.mark.parametrize("d,nnz,W,G,kb", [
    (1_000_003, 10_000, 3, 4, 0),        # ragged last shard
    (1_000_003, 10_000, 3, 3, 255),      # exact bitmap: the last shard has a smaller m
    (300_000, 30_000, 2, 2, 0),
])
@pytest.mark.parametrize("law", ["dyadic", "gauss"])
def test_sharded_single_process(lhc, ora, d, nnz, W, G, kb, law):
    """Every shard is an independent sketch of its coordinate range: its
    bitmap, counters and decode equal the oracle's on that range with the
    shard's params, and the assembled dense output is the concatenation."""
    from paper_2402_07529_b200.sizing import shard_plan

    plan = shard_plan(d, G, nnz / d, W, k_bloom=kb)
    run = lhc.ShardedAllReduce(plan, seed=0x5AD + d, cap_cand=plan.width, local_workers=W)
    xs = make_workers(d, nnz, W, 7 + d % 5, law)
    for _ in range(2):    # the second step reuses the cleared buffers
        dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    dense = F(run.dense)
    for q in range(G):
        lo, hi = plan.bounds(q)
        p = run.ps[q]
        B, Y, ref = ora.pipeline(ora_params(ora, p), [x[lo:hi] for x in xs])
        bm = U(run.slots[q].bitmap)
        assert np.array_equal(bm[:p.words], B) and not bm[p.words:].any()
        assert_values(F(run.slots[q].counters), Y, law == "dyadic")
        compare_decode(ora, run.decoders[q], ref, law == "dyadic")
        assert_values(dense[lo:hi], ref.dense, law == "dyadic")
    assert dec is run.decoders[0]


def test_compress_batch_chained_and_repeated(lhc, ora):
    """sketch_compress_batch over more than 16 inputs (two launches) with repeated
    target sketches and ragged input lengths equals the oracle's per-input
    compression accumulated per target (homomorphism)."""
    d, W = 50_000, 18
    s = lhc.size_workload(d, 0.02, W)
    p = gpu_params(lhc, d, s.m, s.c, seed=0xBA7C)
    xs = make_workers(d, 1000, W, 5, "dyadic")
    ds = [d - 97 * (w % 3) for w in range(W)]          # some inputs shorter than d
    sks = [lhc.Sketch(p) for _ in range(3)]
    lhc.sketch_clear_batch(p, [k.bitmap for k in sks], [k.counters for k in sks])
    tgt = [sks[w % 3] for w in range(W)]
    lhc.sketch_compress_batch(p, [torch.from_numpy(x).cuda() for x in xs],
                              [t.bitmap for t in tgt], [t.counters for t in tgt], ds=ds)
    torch.cuda.synchronize()
    op = ora_params(ora, p)
    for r in range(3):
        parts = []
        for w in range(r, W, 3):
            x = xs[w].copy()
            x[ds[w]:] = 0.0                                  # coordinates past ds[w] are not read
            parts.append(ora.compress_dense(op, x))
        B, Y = ora.aggregate([a for a, _ in parts], [b for _, b in parts])
        assert np.array_equal(U(sks[r].bitmap), B)
        assert np.array_equal(F(sks[r].counters), Y)


@pytest.mark.parametrize("k,kb,L", [(3, 3, 1024), (4, 5, 1024), (3, 3, 256), (2, 1, 32)])
def test_compress_rows_ragged_one_sketch(lhc, ora, k, kb, L):
    """The row-major batched compress (every input into one sketch: a warp takes chunk
    row r of each input in turn; compile-time k = k_B = 3 or run-time k, k_B) with
    inputs of different lengths — one ending mid-chunk, one many chunks short, one
    shorter than a chunk — equals the oracle's per-input compressions accumulated
    (homomorphism)."""
    d = 50_000
    ds = [d, d - 97, d - 2048 - 5, 1000, d - 1]
    W = len(ds)
    s = lhc.size_workload(d, 0.02, W, L=L)
    m = kb * L * max(1, s.m // (kb * L))
    c = k * L * max(1, s.c // (k * L))
    p = gpu_params(lhc, d, m, c, k=k, kb=kb, L=L, seed=0x5EED + k)
    xs = make_workers(d, 1000, W, 9, "dyadic")
    sk = lhc.Sketch(p)
    sk.clear()
    lhc.sketch_compress_batch(p, [torch.from_numpy(x).cuda() for x in xs],
                              [sk.bitmap] * W, [sk.counters] * W, ds=ds)
    torch.cuda.synchronize()
    op = ora_params(ora, p)
    parts = []
    for x, dd in zip(xs, ds):
        x = x.copy()
        x[dd:] = 0.0
        parts.append(ora.compress_dense(op, x))
    B, Y = ora.aggregate([a for a, _ in parts], [b for _, b in parts])
    assert np.array_equal(U(sk.bitmap), B)
    assert np.array_equal(F(sk.counters), Y)


# ------------------------------- generic k / k_B (run-time k kernels, NEXT-4) --

@pytest.mark.parametrize("k,kb", [(2, 1), (4, 5), (3, 7), (5, 0)])
@pytest.mark.parametrize("law", ["dyadic", "gauss"])
@pytest.mark.parametrize("build", ["default", "split"])
def test_generic_k_and_probes(lhc, ora, k, kb, law, build, monkeypatch):
    """The run-time-k kernels (k != 3 or k_B != 3): bitmaps, candidates, flags and
    rounds exact, values exact/tol — including k = 2 below its peeling threshold,
    where most values come from the median (here: mean) fallback; also through the
    two-pass peel of the split state (run-time k)."""
    if build != "default":
        monkeypatch.setenv("LHC_CELL_BUILD", build)
    d, nnz, W = 300_000, 6_000, 2
    s = lhc.size_workload(d, nnz / d, W, k=k, k_bloom=kb)
    p = gpu_params(lhc, d, s.m, s.c, k=k, kb=kb, seed=0x6E + 16 * k + kb)
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, W, 3 + k, law)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(op, xs)
    assert np.array_equal(U(run.sketch.bitmap), B)
    assert_values(F(run.sketch.counters), Y, law == "dyadic")
    compare_decode(ora, dec, ref, law == "dyadic")


@pytest.mark.parametrize("density", [0.10, 0.30])
def test_paper_optimal_bloom_pipeline(lhc, ora, density):
    """NEXT-4: the paper's eps*-optimal Bloom filter (k_B = log2 1/eps* probes)
    end to end against the oracle, one worker at the given density."""
    from paper_2402_07529_b200.sizing import size_paper_optimal

    d = 500_000
    nnz = int(d * density)
    s = size_paper_optimal(d, nnz, C=32, gamma=1.30)
    assert s.k_bloom != 3
    p = gpu_params(lhc, d, s.m, s.c, kb=s.k_bloom, seed=0x0B7 + nnz)
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, 1, 21, "dyadic")
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=1)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B, Y, ref = ora.pipeline(op, xs)
    assert np.array_equal(U(run.sketch.bitmap), B)
    st = compare_decode(ora, dec, ref, True)
    assert st["success"]


# ------------------------------------------ NEXT-3: blocked Count Sketch (R25) --

def blocked_params(lhc, d, nnz, W, L, B, gamma=1.5, seed=0xB10C):
    s = lhc.size_workload(d, nnz / d, W, L=L)
    S = max(1, int(np.ceil(gamma * s.n_cand_expected / (B * 3 * L))))
    return lhc.params(d, s.m, B * 3 * S * L, 3, 0, L, seed + B, B)


@pytest.mark.parametrize("d,nnz,W,L,B", [
    (1_000_003, 10_000, 3, 128, 64),      # ragged tail, many blocks
    (300_000, 6_000, 2, 1024, 8),
    (777_777, 30_000, 4, 256, 33),         # B does not divide the row count
])
@pytest.mark.parametrize("law", ["dyadic", "gauss"])
@pytest.mark.parametrize("build", ["rowpeel", "blocked", "insert", "rows", "compact"])
def test_blocked_sketch_pipeline(lhc, ora, d, nnz, W, L, B, law, build, monkeypatch):
    """P:L206 blocks: every row map, the bitmap, counters, candidates, flags, rounds
    and values equal the oracle's on a blocked sketch — with the row peel (the
    default), the block-local shared-memory peel (k_peel_blocked) and through every
    build mode of the cell-frontier peel."""
    monkeypatch.delenv("LHC_CELL_BUILD", raising=False)
    if build not in ("rowpeel", "blocked"):
        monkeypatch.setenv("LHC_CELL_BUILD", build)
    p = blocked_params(lhc, d, nnz, W, L, B)
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, W, 50 + B, law)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W, deterministic=build == "rowpeel")
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    B_, Y, ref = ora.pipeline(op, xs)
    assert np.array_equal(U(run.sketch.bitmap), B_)
    assert_values(F(run.sketch.counters), Y, law == "dyadic")
    compare_decode(ora, dec, ref, law == "dyadic")


@pytest.mark.parametrize("law", ["dyadic", "gauss"])
def test_blocked_peel_falls_back_to_global(lhc, ora, law, monkeypatch):
    """A block whose destination rows collect more input rows than the block-local
    keys can count (> 127) hands the decode to the global peel, which produces the
    oracle's result; so does any block in an overloaded (failing) decode."""
    monkeypatch.delenv("LHC_CELL_BUILD", raising=False)
    d, L, B = 1000 * 256, 256, 2          # 500 rows per block onto S = 2 rows per partition
    p = lhc.params(d, 3 * 1024 * 64, B * 3 * 2 * L, 3, 0, L, 0xFA11, B)
    op = ora_params(ora, p)
    xs = make_workers(d, 800, 2, 77, law)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=2)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    _, _, ref = ora.pipeline(op, xs)
    compare_decode(ora, dec, ref, law == "dyadic")


@pytest.mark.parametrize("gamma", [1.25, 1.4])
def test_blocked_peel_failure_parity(lhc, ora, gamma, monkeypatch):
    """Near and below the per-block threshold some blocks stall: flags, rounds and the
    median-fallback values still equal the oracle's (dyadic law: exact)."""
    monkeypatch.delenv("LHC_CELL_BUILD", raising=False)
    p = blocked_params(lhc, 500_000, 8_000, 3, 128, 40, gamma=gamma, seed=0xF0 + int(gamma * 100))
    op = ora_params(ora, p)
    xs = make_workers(500_000, 8_000, 3, 91, "dyadic")
    run = lhc.LosslessAllReduce(p, cap_cand=500_000, local_workers=3)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    _, _, ref = ora.pipeline(op, xs)
    compare_decode(ora, dec, ref, True)


@pytest.mark.parametrize("gamma", [1.30, 1.05])
@pytest.mark.parametrize("law", ["gauss", "dyadic"])
def test_decode_deterministic_across_launch_geometries(lhc, ora, gamma, law, monkeypatch):
    """NEXT-3 (deterministic decode; P:L206 parallel rounds, P:L136 every worker
    recovers): the same aggregated sketch decoded 10 times by sketch_decompress_det
    with different grids gives bit-identical values, flags and dense output, under
    the Gaussian law where fp32 order matters — every value comes from the
    lowest-j pure cell and deductions are summed on an integer grid.  Flags, rounds
    and success equal the default decode's; under the dyadic law values are exact.
    gamma 1.05 stalls: the median fallback is covered too."""
    d, nnz, W, L = 3_000_017, 30_000, 4, 1024
    s = lhc.size_workload(d, nnz / d, W, L=L, gamma=gamma)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=0xDE7 + int(gamma * 100))
    xs = make_workers(d, nnz, W, 808, law, sigma=1e-3)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W)
    ref_dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    _, _, ref = ora.pipeline(ora_params(ora, p), xs)
    st0 = compare_decode(ora, ref_dec, ref, exact=(law == "dyadic"))
    if gamma < 1.2:
        assert not ref.stats.success
    outs = []
    for grid in [None, 1, 2, 7, 37, 148, 296, 1000, 3, 64]:
        if grid is None:
            monkeypatch.delenv("LHC_PEEL_GRID", raising=False)
        else:
            monkeypatch.setenv("LHC_PEEL_GRID", str(grid))
        dec = lhc.Decoder(p, d, deterministic=True)
        dec(run.sketch)
        torch.cuda.synchronize()
        st = compare_decode(ora, dec, ref, exact=(law == "dyadic"))
        assert {k: st[k] for k in ("n_cand", "n_peeled", "rounds", "success")} == \
            {k: st0[k] for k in ("n_cand", "n_peeled", "rounds", "success")}
        n = st["n_cand"]
        outs.append((dec.val[:n].cpu().numpy().tobytes(), dec.peeled[:n].cpu().numpy().tobytes(),
                     dec.dense.cpu().numpy().tobytes()))
    assert all(o == outs[0] for o in outs[1:])


@pytest.mark.parametrize("d,nnz,W,L,structure", CASES)
@pytest.mark.parametrize("law", ["dyadic", "gauss"])
def test_pipeline_deterministic_decode(lhc, ora, d, nnz, W, L, structure, law):
    """sketch_decompress_det over the small configs: candidates, flags, rounds and
    success bit-exact, values exact (dyadic) / within tolerance (Gaussian)."""
    s = lhc.size_workload(d, nnz / d, W, L=L)
    p = gpu_params(lhc, d, s.m, s.c, L=L, seed=0x5EED + d)
    xs = make_workers(d, nnz, W, 31 + d % 13, law, structure)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W, deterministic=True)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    _, _, ref = ora.pipeline(ora_params(ora, p), xs)
    compare_decode(ora, dec, ref, law == "dyadic")


@pytest.mark.parametrize("d,nnz,W,L,B,S,law", [
    (3_000_017, 30_000, 3, 1024, 4, 16, "dyadic"),    # 16-CTA clusters, ragged tail
    (3_000_017, 30_000, 3, 1024, 4, 16, "gauss"),
    (2_000_000, 20_000, 2, 256, 6, 16, "dyadic"),     # 8-CTA clusters (L = 256)
    (4_000_000, 60_000, 3, 1024, 2, 32, "dyadic"),    # near the threshold: many rounds
    (1_000_000, 30_000, 2, 1024, 2, 16, "dyadic"),    # overloaded: stalls, median fallback
])
@pytest.mark.parametrize("impl", ["cluster", "global"])
def test_cluster_blocked_peel(lhc, ora, d, nnz, W, L, B, S, law, impl, monkeypatch):
    """P:L206 blocks large enough for a thread-block cluster: the block's decode state
    lives in the cluster's distributed shared memory (peel_cluster.cu, on request), or
    the global peel decodes the blocked layout.  Candidates, flags, rounds, success and
    values (incl. the median fallback) equal the oracle's."""
    if impl == "cluster":
        monkeypatch.setenv("LHC_PEEL_CLUSTER", "1")
    else:
        monkeypatch.delenv("LHC_PEEL_CLUSTER", raising=False)
    s = lhc.size_workload(d, nnz / d, W, L=L)
    p = lhc.params(d, s.m, B * 3 * S * L, 3, 0, L, 0xC1C1 + d + B, B)
    op = ora_params(ora, p)
    xs = make_workers(d, nnz, W, 61 + B, law)
    run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=W)
    dec = run.step([torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    _, _, ref = ora.pipeline(op, xs)
    compare_decode(ora, dec, ref, law == "dyadic")
