"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it pins and is chosen so that a plausible slip in the
oracle (a dropped term, a wrong sign or index, a transposed operand) fails it.
Nothing here compares the oracle with itself or re-types its formulas.
"""
import json
import math
import os

import numpy as np
import pytest

from lhc_inputs import rng_for, support, values

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def P(ora, d, m, c, k=3, kb=0, L=1024, seed=0):
    return ora.params(d, m, c, k, kb, L, seed)


# ---------------------------------------------------------------- hashing (R1) --

def test_mix64_is_splitmix64(ora):
    # Published SplitMix64 output stream for state 0 (Steele/Lea/Flood 2014,
    # reference generator of xoshiro): state advances by the golden gamma.
    g = 0x9E3779B97F4A7C15
    expected = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    for n, e in enumerate(expected, 1):
        assert ora.mix64((n * g) % 2**64) == e


def test_row_map_statistics(ora):
    # Reading R1/R2: rows uniform inside partition j, bias uniform in [0, L),
    # signs balanced ("g_j(i) in {-1, 1}" symmetric for unbiasedness).
    L, S = 64, 50
    p = P(ora, d=4096 * L, m=3 * S * L, c=3 * S * L, L=L, seed=12345)
    n = 4000
    for dom in (0, 1):
        for j in range(3):
            rows, biases, signs = zip(*(ora.row_map(p, dom, j, i) for i in range(n)))
            rows = np.array(rows) - j * S
            assert rows.min() >= 0 and rows.max() < S
            # chi-square against uniform (df = S-1 / L-1), loose 1e-4-level bounds
            cr = np.bincount(rows, minlength=S)
            chi_r = ((cr - n / S) ** 2 / (n / S)).sum()
            assert chi_r < S - 1 + 6 * math.sqrt(2 * (S - 1))
            cb = np.bincount(np.array(biases), minlength=L)
            chi_b = ((cb - n / L) ** 2 / (n / L)).sum()
            assert chi_b < L - 1 + 6 * math.sqrt(2 * (L - 1))
            if dom == 0:
                frac = np.mean(np.array(signs) > 0)
                assert abs(frac - 0.5) < 4 * 0.5 / math.sqrt(n)


def test_hash_survey_golden_values(ora):
    # SURVEY.md §8c step 2 (the written hash spec; the paper gives none, P:L175,
    # P:L230) computed these three values from the spec, independently of the
    # oracle: dom and j occupy bits 56 and 48 of the packed key.
    assert ora.hash64(0, 0, 0, 0) == 0x48218226FF3CD4BF
    assert ora.hash64(0, 1, 0, 0) == 0x8B793569A9EFDF25
    assert ora.hash64(0xDEADBEEF, 0, 2, 12345) == 0x1563224AB3881EA0
    # and the row map fields of H(0, 0, 0, 0) the survey lists: bias 191 (H & 1023),
    # sign +1 (bit 16 of H clear)
    L, S = 1024, 5218
    p = P(ora, d=143_000_000, m=3 * S * L, c=3 * S * L, L=L, seed=0)
    row, bias, sign = ora.row_map(p, 0, 0, 0)
    assert (bias, sign) == (191, 1)
    assert row == (0x48218226 * S) >> 32


def test_row_map_golden_table(ora):
    # The frozen table (tests/golden/rowmap.json, written once by
    # tools/make_golden_rowmap.py and shared with the GPU hash test): packing
    # (j<<48, dom<<56), sign bit 16, bias mask and row reduction per partition.
    g = json.load(open(os.path.join(GOLDEN, "rowmap.json")))
    for s, dom, j, i, H in g["hash"]:
        assert ora.hash64(s, dom, j, i) == H, (s, dom, j, i)
    n_neg = n_17 = 0
    for t in g["tables"]:
        p = ora.params(t["d"], t["k_bloom"] * t["S_B"] * t["L"], t["k"] * t["S_Y"] * t["L"],
                       t["k"], t["k_bloom"], t["L"], t["seed"])
        for dom, j, i, row, bias, sign in t["entries"]:
            assert ora.row_map(p, dom, j, i) == (row, bias, sign), (t["L"], dom, j, i)
            if dom == 0:
                H = ora.hash64(t["seed"], 0, j, i)
                n_neg += sign < 0
                n_17 += ((H >> 16) & 1) != ((H >> 17) & 1)
    # the table has power against a sign taken from a neighbouring bit
    assert n_neg > 100 and n_17 > 100


def test_sketch_and_bloom_maps_independent(ora):
    # Reading R1: domain separation; identical maps would make the Bloom false
    # positives sit exactly on occupied counter rows.
    p = P(ora, d=1 << 20, m=3 * 1024 * 40, c=3 * 1024 * 40, seed=7)
    same = sum(ora.row_map(p, 0, 0, i)[:2] == ora.row_map(p, 1, 0, i)[:2] for i in range(1000))
    assert same < 10


# ------------------------------------------------------------- compression --

def _params_small(ora, L=1024, seed=99, S=8, d=None):
    d = d if d is not None else 20 * L
    return P(ora, d=d, m=3 * S * L, c=3 * S * L, L=L, seed=seed)


@pytest.mark.parametrize("L", [32, 256, 1024])
def test_single_insert_identity(ora, L):
    # inserting x_i adds g_j(i) x_i to exactly k cells (one per hash);
    # sets exactly k_B bits.  Partitioned reading R2: probe j in part j.
    S = 8
    p = _params_small(ora, L=L, S=S)
    rng = rng_for(5)
    for q in rng.integers(0, p.d, 20):
        x = np.zeros(p.d, np.float32)
        x[q] = 0.625
        B, Y = ora.compress_dense(p, x)
        bits = np.flatnonzero(np.unpackbits(B.view(np.uint8), bitorder="little"))
        assert len(bits) == 3
        assert sorted(b // (S * L) for b in bits) == [0, 1, 2]
        nz = np.flatnonzero(Y)
        assert len(nz) == 3
        assert sorted(e // (S * L) for e in nz) == [0, 1, 2]
        assert np.all(np.abs(Y[nz]) == 0.625)


@pytest.mark.parametrize("L", [32, 1024])
def test_full_row_rotation_is_a_bijection(ora, L):
    # a batch (input row) maps onto whole rows of Y and B, rotated by a
    # bias: a full input row must fill each destination row exactly once.
    S = 8
    p = _params_small(ora, L=L, S=S)
    i = 5
    x = np.zeros(p.d, np.float32)
    x[i * L:(i + 1) * L] = 1.0
    B, Y = ora.compress_dense(p, x)
    bits = np.unpackbits(B.view(np.uint8), bitorder="little").reshape(-1, L)
    full_rows = np.flatnonzero(bits.sum(1))
    assert len(full_rows) == 3 and np.all(bits[full_rows].sum(1) == L)
    Yr = Y.reshape(-1, L)
    rows = np.flatnonzero(np.abs(Yr).sum(1))
    assert len(rows) == 3
    for r in rows:
        assert np.all(np.abs(Yr[r]) == 1.0) and len(set(Yr[r])) == 1  # one sign per (row, j)


def test_rotation_keeps_consecutive_parameters_consecutive(ora):
    # P:L262 example: "the 2nd, 3rd, and 4th parameters of X_i could be mapped to
    # the 22nd, 23rd, and 24th parameters of Y_h1(i) ... and the 1022nd, 1023rd,
    # and 1st" — consecutive coordinates of a batch land on consecutive columns
    # modulo the width (reading R6: cyclic, 0-based).
    L = 1024
    p = _params_small(ora, L=L, S=4)
    shifts = set()
    for i in range(10):
        for j in range(3):
            cols = [ora.cell(p, j, i * L + t)[0] % L for t in (1, 2, 3)]
            rows = {ora.cell(p, j, i * L + t)[0] // L for t in (1, 2, 3)}
            assert len(rows) == 1
            assert (cols[1] - cols[0]) % L == 1 and (cols[2] - cols[1]) % L == 1
        # whole row: columns are a cyclic shift of 0..L-1
        cols = [ora.cell(p, 0, i * L + t)[0] % L for t in range(L)]
        shift = cols[0]
        assert cols == [(t + shift) % L for t in range(L)]
        shifts.add(shift)
    # "a random bias within the range [0..c-1]": the shift differs across batches
    assert len(shifts) >= 8


@pytest.mark.parametrize("L", [32, 1024])
def test_homomorphism(ora, L):
    # Y(sum X) = sum Y(X) and B(sum X) = OR B(X).  Dyadic values make
    # every fp sum exact, positive values exclude cancellation to zero.
    p = _params_small(ora, L=L, S=16, d=37 * L + 11)
    rng = rng_for(11)
    xs = []
    for w in range(3):
        x = np.zeros(p.d, np.float32)
        idx = support(rng, p.d, 300)
        x[idx] = np.abs(values(rng, len(idx), "dyadic"))
        xs.append(x)
    sk = [ora.compress_dense(p, x) for x in xs]
    Bsum, Ysum = ora.compress_dense(p, xs[0] + xs[1] + xs[2])
    Bor = sk[0][0] | sk[1][0] | sk[2][0]
    assert np.array_equal(Bsum, Bor)
    assert np.array_equal(Ysum, sk[0][1] + sk[1][1] + sk[2][1])
    # accumulating compressions into one sketch == compressing the sum
    B, Y = ora.compress_dense(p, xs[0])
    ora.compress_dense(p, xs[1], B, Y)
    ora.compress_dense(p, xs[2], B, Y)
    assert np.array_equal(B, Bsum) and np.array_equal(Y, Ysum)


def test_coo_equals_dense(ora):
    p = _params_small(ora, L=256, S=16, d=50_001)
    rng = rng_for(3)
    idx = support(rng, p.d, 900)
    val = values(rng, len(idx), "dyadic")
    x = np.zeros(p.d, np.float32)
    x[idx] = val
    B1, Y1 = ora.compress_dense(p, x)
    B2, Y2 = ora.compress_coo(p, idx, val)
    assert np.array_equal(B1, B2) and np.array_equal(Y1, Y2)


def test_negative_zero_is_zero(ora):
    # Zero-ness is the IEEE comparison x != 0 ("true indicates non-zero").
    p = _params_small(ora)
    x = np.zeros(p.d, np.float32)
    x[17] = -0.0
    B, Y = ora.compress_dense(p, x)
    assert not B.any() and not Y.any()


def test_aggregate_or_sum(ora):
    # B <- OR B, Y <- sum Y.
    rng = rng_for(8)
    Bs = [rng.integers(0, 2**32, 999, dtype=np.uint64).astype(np.uint32) for _ in range(5)]
    Ys = [rng.standard_normal(3072) for _ in range(5)]
    B, Y = ora.aggregate(Bs, Ys)
    assert np.array_equal(B, np.bitwise_or.reduce(np.stack(Bs), axis=0))
    np.testing.assert_allclose(Y, np.sum(np.stack(Ys), axis=0), rtol=1e-15, atol=1e-15)


# ------------------------------------------------------------------- query --

def test_query_no_false_negatives(ora):
    # the Bloom filter "never recognizes non-zero values as zero".
    p = P(ora, d=300_000, m=3 * 1024 * 4, c=3 * 1024 * 8, L=1024, seed=4)
    rng = rng_for(4)
    idx = support(rng, p.d, 3000)
    x = np.zeros(p.d, np.float32)
    x[idx] = 1.0
    B, _ = ora.compress_dense(p, x)
    cand = ora.query(p, B)
    assert np.all(np.diff(cand.astype(np.int64)) > 0)  # ascending, unique
    assert set(idx.tolist()) <= set(cand.tolist())


def test_query_exact_when_filter_sparse(ora):
    # With m >> n the false-positive rate (1-(1-k/m)^n)^k ~ 1e-11: the candidate
    # set is the support itself.
    L = 32
    p = P(ora, d=20_000, m=3 * L * 40_000, c=3 * L * 8, L=L, seed=21)
    rng = rng_for(21)
    idx = support(rng, p.d, 100)
    x = np.zeros(p.d, np.float32)
    x[idx] = 1.0
    B, _ = ora.compress_dense(p, x)
    assert np.array_equal(ora.query(p, B), idx)


@pytest.mark.parametrize("L", [32, 1024])
def test_query_false_positive_rate(ora, L):
    # P:L229-230 sizing: with n items and k probes into k partitions of m/k bits
    # the false-positive probability is (1 - (1 - k/m)^n)^k.
    d = 1 << 21
    n = 20_000
    m = 3 * L * ((6 * n) // (3 * L))
    p = P(ora, d=d, m=m, c=3 * L, L=L, seed=77)
    rng = rng_for(77)
    idx = support(rng, d, n)
    x = np.zeros(d, np.float32)
    x[idx] = 1.0
    B, _ = ora.compress_dense(p, x)
    fp = len(ora.query(p, B)) - n
    eps = (1 - (1 - 3 / m) ** n) ** 3
    expected = eps * (d - n)
    assert abs(fp - expected) < 0.08 * expected, (fp, expected)


# ------------------------------------------------------------------ peeling --

def test_fig1_worked_example(ora):
    g = json.load(open(os.path.join(GOLDEN, "fig1.json")))
    cells = np.array(g["cells"], np.uint64)
    signs = np.array(g["signs"], np.int8)
    vals = np.array(g["values"])
    Y = np.zeros(g["n_cells"])
    for s in range(3):
        for j in range(3):
            Y[cells[s, j]] += signs[s, j] * vals[s]
    r = ora.peel_core(cells, signs, Y)
    assert r.rounds == g["expected"]["rounds"]
    assert r.round_of.tolist() == g["expected"]["round_of"]
    assert r.peeled.tolist() == g["expected"]["peeled"]
    assert np.array_equal(r.val, vals)  # dyadic: exact
    assert np.all(r.residual == 0)


def _two_core_items(cells, n_cells):
    """Independent brute force of P:L204 ('the peeling process is equivalent to
    finding two cores'): delete any item that has a cell of degree one, until no
    such item remains.  Returns the set of surviving (unpeelable) items."""
    alive = set(range(len(cells)))
    changed = True
    while changed:
        changed = False
        deg = [0] * n_cells
        for s in alive:
            for e in cells[s]:
                deg[e] += 1
        for s in sorted(alive):
            if any(deg[e] == 1 for e in cells[s]):
                alive.discard(s)
                changed = True
                break
    return alive


def test_peel_equals_complement_of_two_core(ora):
    rng = rng_for(2024)
    for trial in range(120):
        n_cells = int(rng.integers(6, 30))
        n_items = int(rng.integers(1, 2 * n_cells // 3 + 2))
        cells = np.array([rng.choice(n_cells, 3, replace=False) for _ in range(n_items)], np.uint64)
        signs = rng.choice([-1, 1], (n_items, 3)).astype(np.int8)
        vals = values(rng, n_items, "dyadic").astype(np.float64)
        Y = np.zeros(n_cells)
        for s in range(n_items):
            for j in range(3):
                Y[cells[s, j]] += signs[s, j] * vals[s]
        r = ora.peel_core(cells, signs, Y, finalize=False)
        core = _two_core_items(cells.tolist(), n_cells)
        assert set(np.flatnonzero(~r.peeled).tolist()) == core
        # every peeled value is exact (P:L206 lossless)
        assert np.array_equal(r.val[r.peeled], vals[r.peeled])


@pytest.mark.parametrize("R", [1, 2, 5, 8, 13])
def test_two_ended_chain_round_count(ora, R):
    # Item r lives in cells {a_r, a_{r+1}, Z}; a_0 and a_R are private and the
    # shared cell Z has degree R, so the chain peels inward from both ends:
    # synchronous rounds = ceil(R/2) (one item per end per round).
    cells, signs = [], []
    Z = R + 1
    for r in range(R):
        cells.append([r, r + 1, Z])
        signs.append([1, -1, 1])
    cells = np.array(cells, np.uint64)
    signs = np.array(signs, np.int8)
    vals = np.arange(1, R + 1, dtype=np.float64) * 0.5
    Y = np.zeros(R + 2)
    for s in range(R):
        for j in range(3):
            Y[cells[s, j]] += signs[s, j] * vals[s]
    r = ora.peel_core(cells, signs, Y)
    assert r.rounds == (R + 1) // 2 if R > 1 else r.rounds == 1
    assert r.peeled.all() and np.array_equal(r.val, vals)
    expect = [min(s + 1, R - s) for s in range(R)]
    if R == 1:
        expect = [1]
    assert r.round_of.tolist() == expect


def test_unpeelable_pair_median_fallback(ora):
    # Two items sharing all three cells form a 2-core: nothing peels (P:L193 stop
    # rule) and both are estimated by the Count Sketch median.
    # a = 3, b = 1, signs a:(+,+,+), b:(+,-,+): Y = [4, 2, 4].
    cells = np.array([[0, 1, 2], [0, 1, 2]], np.uint64)
    signs = np.array([[1, 1, 1], [1, -1, 1]], np.int8)
    Y = np.array([4.0, 2.0, 4.0])
    r = ora.peel_core(cells, signs, Y)
    assert r.rounds == 0 and not r.peeled.any()
    # item a: median(4, 2, 4) = 4; item b: median(4, -2, 4) = 4
    assert r.val.tolist() == [4.0, 4.0]


def test_partial_peel_fallback_is_residual_median(ora):
    # Reading R11 ("Estimate the not recovered parameters of X from Y" after
    # the peel has deducted the recovered ones from Y).  Hand-built
    # incidence: z -> {2, 3, 4} peels in round 1 (cells 3 and 4 hold only z; the
    # lowest j, cell 3, gives its value); a -> {0, 1, 2} (+,+,+) and
    # b -> {0, 1, 2} (+,-,-) share all three cells: a 2-core, estimated.
    # a = 1, b = 2, z = 10:  Y = [3, -1, 1 - 2 + 10 = 9, 10, 10];
    # residual after z:      R = [3, -1, -1, 0, 0].
    # a: median(+3, -1, -1) = -1   (over Y it would be median(3, -1, 9) = 3)
    # b: median(+3, +1, +1) = +1   (over Y: median(3, 1, -9) = 1)
    cells = np.array([[0, 1, 2], [0, 1, 2], [2, 3, 4]], np.uint64)
    signs = np.array([[1, 1, 1], [1, -1, -1], [1, 1, 1]], np.int8)
    Y = np.array([3.0, -1.0, 9.0, 10.0, 10.0])
    r = ora.peel_core(cells, signs, Y)
    assert r.rounds == 1
    assert r.peeled.tolist() == [False, False, True]
    assert r.round_of.tolist() == [0, 0, 1]
    assert r.residual.tolist() == [3.0, -1.0, -1.0, 0.0, 0.0]
    assert r.val.tolist() == [-1.0, 1.0, 10.0]


def test_decompress_fallback_uses_the_residual(ora):
    # The same reading through the whole Phase II (ora_decompress): an
    # under-provisioned sketch (c = 288 cells for ~337 candidates) stalls after a
    # few rounds.  Independently of the oracle's peel and finalize: peeled values
    # are the true ones (exact, dyadic law), the residual is Y minus their signed
    # contributions at their cells, and every unpeeled candidate's value is the
    # median over j of g_j * residual.
    d, L, S, seed = 4096, 32, 3, 8
    p = ora.params(d, 3 * 32 * 40, 3 * L * S, 3, 3, L, seed)
    rng = rng_for(seed)
    idx = support(rng, d, 300, "uniform")
    x = np.zeros(d, np.float32)
    x[idx] = values(rng, len(idx), "dyadic")
    B, Y, dec = ora.pipeline(p, [x])
    assert 0 < dec.peeled.sum() < len(dec.cand) and not dec.stats.success
    truth = x[dec.cand].astype(np.float64)
    assert np.array_equal(dec.val[dec.peeled], truth[dec.peeled])
    maps = [[ora.cell(p, j, int(q)) for j in range(3)] for q in dec.cand]
    R = Y.copy()
    for s in np.flatnonzero(dec.peeled):
        for e, g in maps[s]:
            R[e] -= g * truth[s]
    differs = 0
    for s in np.flatnonzero(~dec.peeled):
        est_R = np.median([g * R[e] for e, g in maps[s]])
        est_Y = np.median([g * Y[e] for e, g in maps[s]])
        assert dec.val[s] == est_R
        differs += est_R != est_Y
    assert differs > 10  # the case separates the residual from the original Y


def test_even_k_median_is_mean_of_middle_pair(ora):
    cells = np.array([[0, 1, 2, 3], [0, 1, 2, 3]], np.uint64)
    signs = np.ones((2, 4), np.int8)
    Y = np.array([1.0, 5.0, 2.0, 9.0])
    r = ora.peel_core(cells, signs, Y)
    assert r.val.tolist() == [3.5, 3.5]


# ------------------------------------------------------------ full Phase II --

def _workers(d, nnz, W, seed, law="dyadic", structure="uniform", run=64):
    xs = []
    for w in range(W):
        rng = rng_for(seed + w)
        x = np.zeros(d, np.float32)
        idx = support(rng, d, nnz, structure, run)
        x[idx] = values(rng, len(idx), law)
        xs.append(x)
    return xs


@pytest.mark.parametrize("L,W,structure", [(1024, 2, "uniform"), (256, 4, "runs"), (32, 3, "uniform")])
def test_lossless_recovery_exact(ora, L, W, structure):
    # above the threshold the aggregate is recovered exactly;
    # non-candidates are exactly zero.  Dyadic values: every sum is exact.
    from paper_2402_07529_b200.sizing import size_for, union_support

    d = 200_003
    nnz = 1500
    s = size_for(d, union_support(d, nnz / d, W), L=L, gamma=1.5)
    p = P(ora, d, s.m, s.c, L=L, seed=0xC0FFEE)
    xs = _workers(d, nnz, W, 500, structure=structure)
    B, Y, dec = ora.pipeline(p, xs)
    truth = np.sum(np.stack(xs).astype(np.float64), axis=0)
    assert dec.stats.success and not dec.stats.overflow
    assert np.array_equal(dec.dense, truth)
    assert set(np.flatnonzero(truth).tolist()) <= set(dec.cand.tolist())
    assert dec.stats.rounds >= 1


def test_success_phase_transition(ora):
    # full recovery w.h.p. once the sketch holds >= gamma n cells
    # (gamma = 1.23; exact k=3 threshold 1.2218); well below it peeling stalls.
    d, n = 1 << 20, 12_000
    L = 256
    succ = {}
    for gamma in (1.05, 1.45):
        ok = 0
        for seed in range(6):
            rng = rng_for(900 + seed)
            idx = support(rng, d, n)
            x = np.zeros(d, np.float32)
            x[idx] = 1.0
            m = 3 * L * 2000  # ~ 128 bits/item: false positives negligible
            c = 3 * L * int(math.ceil(gamma * n / (3 * L)))
            p = P(ora, d, m, c, L=L, seed=seed)
            _, _, dec = ora.pipeline(p, [x], dense=False)
            ok += dec.stats.success
        succ[gamma] = ok
    assert succ[1.45] == 6 and succ[1.05] == 0


def test_856_percent_threshold_vgg_density(ora):
    # at VGG19's sparsity 30.4 % the recovery surges to 100 % once the
    # (counter) size passes 1.23 x (1 - 0.304) = 85.6 % of the original size.
    d = 1 << 16
    nnz = int(round(0.696 * d))
    L = 1024
    rng = rng_for(344)
    idx = support(rng, d, nnz)
    x = np.zeros(d, np.float32)
    x[idx] = values(rng, nnz, "dyadic")
    m = 3 * L * ((64 * d) // (3 * L))  # near-exact index, eps ~ 3e-5
    res = {}
    for frac in (0.70, 0.95):
        c = 3 * L * int(round(frac * d / (3 * L)))
        p = P(ora, d, m, c, L=L, seed=5)
        _, _, dec = ora.pipeline(p, [x])
        res[frac] = dec.stats
    assert not res[0.70].success and res[0.70].n_peeled < res[0.70].n_cand
    assert res[0.95].success


def test_rounds_decrease_with_provisioning(ora):
    # P:L332 / Fig. 3(c): more sketch -> fewer recovery iterations.
    d, n, L = 1 << 20, 15_000, 1024
    rng = rng_for(31)
    idx = support(rng, d, n)
    x = np.zeros(d, np.float32)
    x[idx] = 1.0
    m = 3 * L * 1000
    rounds = []
    for gamma in (1.3, 1.6, 2.5, 4.0):
        c = 3 * L * int(math.ceil(gamma * n / (3 * L)))
        _, _, dec = ora.pipeline(P(ora, d, m, c, L=L, seed=1), [x], dense=False)
        assert dec.stats.success
        rounds.append(dec.stats.rounds)
    assert rounds == sorted(rounds, reverse=True) and rounds[0] > rounds[-1]


def test_fallback_unbiased(ora):
    # the g_j factor makes collisions symmetric with zero mean, so the
    # median estimate of unpeeled parameters is unbiased (3-sigma test).  The
    # values are all positive, so without the signs the estimate would be biased.
    d, n, L = 1 << 18, 6000, 256
    errs = []
    for seed in range(8):
        rng = rng_for(4000 + seed)
        idx = support(rng, d, n)
        x = np.zeros(d, np.float32)
        x[idx] = np.abs(values(rng, n, "dyadic"))
        m = 3 * L * 500
        c = 3 * L * int(math.ceil(0.9 * n / (3 * L)))  # below threshold: peel stalls
        _, _, dec = ora.pipeline(P(ora, d, m, c, L=L, seed=seed), [x])
        un = ~dec.peeled
        assert un.sum() > 100
        errs.append(dec.val[un] - x[dec.cand[un]].astype(np.float64))
    e = np.concatenate(errs)
    assert abs(e.mean()) < 3 * e.std() / math.sqrt(len(e))


def test_overflow_flag(ora):
    d, L = 100_000, 1024
    p = P(ora, d, 3 * L * 4, 3 * L * 8, L=L, seed=3)
    x = np.zeros(d, np.float32)
    x[::50] = 1.0
    B, Y = ora.compress_dense(p, x)
    dec = ora.decompress(p, B, Y, cap=10)
    assert dec.stats.overflow and not dec.stats.success and dec.stats.n_cand > 10


def test_all_zero_gradient(ora):
    p = _params_small(ora)
    B, Y, dec = ora.pipeline(p, [np.zeros(p.d, np.float32)])
    assert dec.stats.n_cand == 0 and dec.stats.success and dec.stats.rounds == 0
    assert not dec.dense.any()


# ------------------------------------------------ exact bitmap index (NEXT-1) --

@pytest.mark.parametrize("L", [32, 1024])
def test_exact_bitmap_is_the_support(ora, L):
    # "allocating one bit per parameter - for each bit, true indicates
    # non-zero, while false indicates zero"; OR-homomorphic across workers.
    d = 50_003
    m = (d + L - 1) // L * L
    p = P(ora, d, m, 3 * L * 8, kb=ora.INDEX_BITMAP, L=L, seed=9)
    assert ora.validate(p)
    assert not ora.validate(P(ora, d, m + L, 3 * L * 8, kb=ora.INDEX_BITMAP, L=L))
    xs = _workers(d, 700, 3, 70)
    B = None
    Y = None
    for x in xs:
        B, Y = ora.compress_dense(p, x, B, Y)
    support = np.zeros(m, bool)
    for x in xs:
        support[:d] |= x != 0
    ref = np.packbits(support, bitorder="little").view(np.uint32)
    assert np.array_equal(B, ref)
    assert np.array_equal(ora.query(p, B), np.flatnonzero(support).astype(np.uint32))


def test_exact_bitmap_lossless(ora):
    from paper_2402_07529_b200.sizing import INDEX_BITMAP, size_for, union_support

    d, W, L = 300_001, 4, 1024
    s = size_for(d, union_support(d, 2000 / d, W), k_bloom=INDEX_BITMAP, L=L, gamma=1.4)
    p = P(ora, d, s.m, s.c, kb=ora.INDEX_BITMAP, L=L, seed=5)
    xs = _workers(d, 2000, W, 800)
    _, _, dec = ora.pipeline(p, xs)
    truth = np.sum(np.stack(xs).astype(np.float64), axis=0)
    assert dec.stats.success and np.array_equal(dec.dense, truth)
    assert dec.stats.n_cand == int((np.stack(xs) != 0).any(axis=0).sum())  # no false positives


# ------------------------------------------ NEXT-3: blocked Count Sketch (R25) --

def test_one_block_is_the_unblocked_sketch(ora):
    # P:L206 blocks: with a single block every map must equal the unblocked one
    d, L = 50 * 1024, 1024
    a = ora.params(d, 3 * L * 8, 3 * L * 20, 3, 0, L, 99, 0)
    b = ora.params(d, 3 * L * 8, 3 * L * 20, 3, 0, L, 99, 1)
    for q in range(0, d, 997):
        for j in range(3):
            assert ora.cell(a, j, q) == ora.cell(b, j, q)
            assert ora.bit(a, j, q) == ora.bit(b, j, q)   # the index is not blocked


def test_blocked_cells_stay_in_their_block(ora):
    # every coordinate of input row i lands in block i mod B, probe j in the j-th
    # partition of that block (S rows each), and the blocks are used evenly
    d, L, B, S = 97 * 256, 256, 7, 5
    c = B * 3 * S * L
    p = ora.params(d, 3 * L * 4, c, 3, 0, L, 7, B)
    used = np.zeros(c // L, np.int64)
    for q in range(0, d, 13):
        i = q // L
        for j in range(3):
            row = ora.cell(p, j, q)[0] // L
            lo = (i % B) * 3 * S + j * S
            assert lo <= row < lo + S, (q, j, row, lo)
            used[row] += 1
    per_block = used.reshape(B, 3 * S).sum(axis=1)
    assert per_block.min() > 0.8 * per_block.mean()


@pytest.mark.parametrize("B", [4, 16])
def test_blocked_sketch_is_lossless(ora, B):
    # the method stays exact with a blocked sketch at gamma_s = 1.5
    d, L, W, nnz = 64 * 128, 128, 3, 300
    n = d * (1 - (1 - nnz / d) ** W)
    S = max(1, math.ceil(1.5 * n / (B * 3 * L)))
    c = B * 3 * S * L
    p = ora.params(d, 3 * L * 64, c, 3, 0, L, 1234 + B, B)
    rng = rng_for(3100 + B)
    xs = []
    for w in range(W):
        x = np.zeros(d, np.float32)
        x[support(rng, d, nnz)] = values(rng, nnz, "dyadic")
        xs.append(x)
    _, _, ref = ora.pipeline(p, xs)
    assert ref.stats.success
    assert np.array_equal(ref.dense, np.sum(np.stack(xs).astype(np.float64), axis=0))
