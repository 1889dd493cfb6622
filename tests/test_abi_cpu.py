"""CPU-side checks of the C ABI (no GPU): liblhc.so loads, exports every symbol
include/lhc.h declares, and its host-side validation / sizing logic behaves.
No compute entry point is called with valid arguments here."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lhc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "return")))


@pytest.fixture(scope="module")
def lhc():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2402_07529_b200 as lhc

    return lhc


def test_library_exports_every_header_symbol(lhc):
    syms = header_symbols()
    assert "sketch_compress" in syms and "sketch_decompress" in syms and len(syms) >= 16
    L = lhc.lib()
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(lhc._lib.EXPORTS) <= set(syms)


def test_struct_layouts_match_header(lhc):
    # lhc_params: u32 d, u64 m, u64 c, u32 k, u32 k_bloom, u32 L, u64 seed (natural alignment)
    assert ctypes.sizeof(lhc.lhc_params) == 48
    assert lhc.lhc_params.m.offset == 8 and lhc.lhc_params.seed.offset == 40
    assert ctypes.sizeof(lhc._lib.lhc_stats) == 32


def test_validate(lhc):
    ok = lhc.params(10_000, 3072, 3072, 3, 0, 1024, 1)
    assert lhc.lhc_validate(ok)
    bad = [
        lhc.params(0, 3072, 3072),                 # d = 0
        lhc.params(10_000, 3072, 3000),            # c not a multiple of k*L
        lhc.params(10_000, 3000, 3072),            # m not a multiple of k_B*L
        lhc.params(10_000, 3072, 3072, 0),         # k = 0
        lhc.params(10_000, 3072, 3072, 9),         # k > 8
        lhc.params(10_000, 3072, 3072, L=48),      # L not a power of two
        lhc.params(10_000, 3072, 3072, L=2048),    # L > 1024
        lhc.params(10_000, 3072, 3 << 32),         # c >= 2^32
    ]
    for p in bad:
        assert not lhc.lhc_validate(p), p
    assert "c must" in lhc._lib.last_error() or "must" in lhc._lib.last_error()


def test_einval_before_any_launch(lhc):
    L = lhc.lib()
    bad = lhc.params(10_000, 3072, 3000)
    assert L.sketch_compress(ctypes.byref(bad), None, None, None, None, None) == lhc._lib.LHC_EINVAL
    ok = lhc.params(10_000, 3072, 3072)
    assert L.sketch_compress(ctypes.byref(ok), None, None, None, None, None) == lhc._lib.LHC_EINVAL
    assert L.sketch_decompress(ctypes.byref(ok), None, None, None, 0, 0, None, None, None, None,
                               None, None) == lhc._lib.LHC_EINVAL
    assert L.sketch_aggregate(ctypes.byref(ok), 0, None, None, None, None, None) == lhc._lib.LHC_EINVAL
    # misaligned pointers are rejected on the host
    assert L.sketch_compress(ctypes.byref(ok), 0x1004, 0x2000, 0x3000, None, None) == lhc._lib.LHC_EINVAL


def test_workspace_and_layout(lhc):
    p = lhc.params(32_000_000, 30904320, 3588096)
    ws = lhc.lhc_decompress_workspace(p, 3_000_000)
    # >= cell state (16 B/cell) + frontier (4 B/cell) + claims (4 B/candidate)
    assert ws >= 20 * 3588096 + 4 * 3_000_000
    b, y, s, total = lhc.lhc_comm_layout(p)
    assert b == 0 and y >= 30904320 // 8 and y % 256 == 0
    assert s >= y + 4 * 3588096 and total > s


# ------------------------------------------------------------ sizing (host) --

def test_sizing_matches_bloom_closed_form(lhc):
    from paper_2402_07529_b200 import sizing

    s = sizing.size_workload(32_000_000, 0.01, 8)
    assert s.m % (3 * 1024) == 0 and s.c % (3 * 1024) == 0
    n = 32_000_000 * (1 - 0.99 ** 8)
    assert abs(s.n_expected - n) < 1
    assert abs(s.eps - (1 - (1 - 3 / s.m) ** n) ** 3) < 1e-12
    assert s.c >= 1.3 * (n + s.eps * (32_000_000 - n))
    # the optimum is interior: cheaper than both neighbours on the grid
    cost = s.m + 32 * s.c
    for m2 in (int(s.m * 0.8) // 3072 * 3072, int(s.m * 1.25) // 3072 * 3072):
        eps = sizing.bloom_fp_rate(m2, n, 3)
        c2 = math.ceil(1.3 * (n + eps * (32_000_000 - n)) / 3072) * 3072
        assert m2 + 32 * c2 >= cost


def test_theory_pins(lhc):
    from paper_2402_07529_b200 import sizing

    # eps* = (ln^2 2 gamma C lambda)^-1
    assert abs(sizing.optimal_eps(32, 99, 1.23) - 5.341e-4) < 1e-6
    assert abs(sizing.optimal_eps(32, 9, 1.23) - 5.876e-3) < 1e-5
    assert sizing.optimal_eps(1, 0.5, 1.23) == 1.0  # clamp
    # f(0, x) = (x+1) H(1/(x+1)); H(1/2) = 1 -> f(0,1) = 2
    assert sizing.f0(1.0) == 2.0
    assert abs(sizing.f0(99) - 8.0793) < 1e-3
    # S_min(lambda=1, C=1) = 2n
    assert sizing.s_min_bits(1000, 1.0, 1) == 2000
    # n/ln2 log2(1/eps) bits; n=1e6, eps=0.01 -> 9,585,059 bits (ceil)
    assert math.ceil(sizing.bloom_bits(1e6, 0.01)) == 9_585_059
    # S1 + S2 < 1.6 S_min over a grid of bit widths and zero ratios
    worst = 0.0
    for C in (4, 8, 16, 32):
        for lam in (1, 9, 99, 999, 9999):
            s1, s2 = sizing.paper_sizes(1e4, lam, C)
            worst = max(worst, (s1 + s2) / sizing.s_min_bits(1e4, lam, C))
    assert worst < 1.6
    # 1.23 x (1 - 0.304) = 85.6 %
    assert round(1.23 * (1 - 0.304), 3) == 0.856


# ------------------------------------------------- sharded layout (host) --

@pytest.mark.parametrize("d,G", [(32_000_000, 8), (32_000_000, 2), (10_000_000, 3), (7_000, 3)])
def test_shard_plan_covers_d(lhc, d, G):
    from paper_2402_07529_b200.sizing import INDEX_BITMAP, shard_plan

    for kb in (0, INDEX_BITMAP):
        plan = shard_plan(d, G, 0.01, 8, k_bloom=kb)
        assert plan.width % 1024 == 0
        spans = [plan.bounds(q) for q in range(G)]
        assert spans[0][0] == 0 and spans[-1][1] == d
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))     # contiguous, disjoint
        assert all(plan.shard_d(q) > 0 for q in range(G))
        for q in range(G):
            p = lhc.params(plan.shard_d(q), plan.shard_m(q), plan.sizing.c, 3, kb, 1024, 1)
            assert lhc.lhc_validate(p), (q, p, lhc._lib.last_error())
            assert plan.shard_m(q) <= plan.sizing.m               # fits the largest slot


def test_shard_plan_rejects_empty_shards(lhc):
    from paper_2402_07529_b200.sizing import shard_plan

    with pytest.raises(ValueError):
        shard_plan(3000, 4, 0.01, 8)     # width 1024: the fourth shard would be empty


def test_shard_layout(lhc):
    from paper_2402_07529_b200.sizing import shard_plan

    plan = shard_plan(32_000_000, 8, 0.01, 8)
    s = plan.sizing
    # the G sub-sketches together are the size of the unsharded sketch (within rounding)
    full = lhc.size_workload(32_000_000, 0.01, 8)
    assert abs(8 * (s.m / 8 + 4 * s.c) - (full.m / 8 + 4 * full.c)) / (full.m / 8 + 4 * full.c) < 0.01
    ps = lhc.params(plan.width, s.m, s.c, 3, 0, 1024, 1)
    slot, y, total = lhc.lhc_shard_layout(ps, 8, 500_000)
    assert y >= s.m // 8 and y % 256 == 0 and slot >= y + 4 * s.c and slot % 256 == 0
    # slots + double-buffered staging + double-buffered gather lists + signals
    assert total >= 3 * 8 * slot + 2 * 8 * 500_000 * 8 + 512
    with pytest.raises(lhc.LhcError):
        lhc.lhc_shard_layout(ps, 9, 500_000)
    with pytest.raises(lhc.LhcError):
        lhc.lhc_shard_layout(ps, 8, 0)
    L = lhc.lib()
    assert L.sketch_reduce_scatter(None, None) == lhc._lib.LHC_EINVAL
    assert L.sketch_allgather_decoded(None, None, None, None, 4096, 10_000, None, None) == \
        lhc._lib.LHC_EINVAL


# ---------------------------------------- NEXT-4: paper-optimal Bloom sizing --

@pytest.mark.parametrize("density", [0.10, 0.30, 0.696])
def test_paper_optimal_sizing(lhc, density):
    """k_B = log2(1/eps*) probes, m = n/ln2 log2(1/eps*) bits,
    c = gamma n (1 + eps lambda); the realised partitioned-filter false-positive rate
    is close to eps*, and the total stays below 1.6 S_min."""
    from paper_2402_07529_b200 import sizing

    d = 10_000_000
    n = d * density
    s = sizing.size_paper_optimal(d, n, C=32, gamma=1.23)
    lam = (d - n) / n
    eps_star = sizing.optimal_eps(32, lam, 1.23)
    lg = math.log2(1 / eps_star)
    assert s.k_bloom == max(1, min(8, round(lg)))
    assert s.m % (s.k_bloom * 1024) == 0 and s.c % (3 * 1024) == 0
    assert abs(s.m - n / math.log(2) * lg) <= s.k_bloom * 1024
    assert 0.5 * eps_star < s.eps < 2.0 * eps_star
    assert abs(s.c - 1.23 * n * (1 + s.eps * lam)) <= 3 * 1024
    S = s.m + 32 * s.c
    assert S < 1.6 * sizing.s_min_bits(n, lam, 32)
    p = lhc.params(d, s.m, s.c, 3, s.k_bloom, 1024, 1)
    assert lhc.lhc_validate(p)


def test_blocked_sizing(lhc):
    """NEXT-3 sizing: c is a whole number of blocks of k partitions of S rows, about
    cells_per_block cells each, and at least the unblocked c (same provisioning)."""
    from paper_2402_07529_b200.sizing import size_blocked

    for L in (256, 1024):
        s, B = size_blocked(32_000_000, 0.01, 8, cells_per_block=12288, L=L)
        base = lhc.size_workload(32_000_000, 0.01, 8, L=L)
        S = round(12288 / (3 * L))
        assert s.c == B * 3 * S * L and s.c >= base.c and s.c - base.c < 3 * S * L
        assert s.m == base.m
        p = lhc.params(32_000_000, s.m, s.c, 3, 0, L, 1, B)
        assert lhc.lhc_validate(p)
    c_bad = 3 * L * (7 * 100 + 3)                                   # not a multiple of 7*3*L
    assert not lhc.lhc_validate(lhc.params(32_000_000, base.m, c_bad, 3, 0, L, 1, 7))
    assert lhc.lhc_validate(lhc.params(32_000_000, base.m, c_bad, 3, 0, L, 1, 0))
