"""Host-side sizing of the sketch S(X) = [Y, B] (no device work).

The workers must agree on (m, c) before any gradient is seen (reading R15), so
both are derived from the expected aggregate support:

* expected union support of W workers with independent supports of density rho
  (reading R19): ``n = d * (1 - (1 - rho)^W)``;
* Bloom false-positive rate of a partitioned filter with k_B probes over m bits
  (one partition of m/k_B bits per probe):
  ``eps(m) = (1 - (1 - k_B/m)^n)^k_B``;
* candidates ``n_c = n + eps * (d - n)`` (the table records
  ``eps (N - n)`` redundant values);
* Count Sketch cells ``c = gamma_s * n_c`` rounded up to a multiple of k*L, with
  the provisioning gamma_s >= gamma = 1.23 (reading R14: 1.30 default);
* m minimises the sketch bits ``m + 32 c`` over multiples of k_B*L.

Also the §3.3 theory helpers: S_min, the optimal eps and the
(S1, S2) sizes of the paper's Bloom + Count Sketch construction.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

GAMMA_PAPER = 1.23
GAMMA_DEFAULT = 1.30      # reading R14
GAMMA_STAR_K3 = 1.0 / 0.8184691  # exact 2-core threshold of random 3-hypergraphs


def union_support(d: int, density: float, workers: int) -> float:
    return d * (1.0 - (1.0 - density) ** workers)


def bloom_fp_rate(m: int, n: float, k_bloom: int) -> float:
    """False-positive rate of a k_bloom-partitioned Bloom filter of m bits, n items."""
    if m <= 0:
        return 1.0
    return (1.0 - (1.0 - k_bloom / m) ** n) ** k_bloom


@dataclass
class Sizing:
    d: int
    m: int
    c: int
    k: int
    k_bloom: int
    L: int
    n_expected: float
    eps: float
    n_cand_expected: float
    gamma: float

    @property
    def sketch_bytes(self) -> int:
        return self.m // 8 + 4 * self.c

    @property
    def ratio(self) -> float:
        """Sketch size / dense fp32 size."""
        return self.sketch_bytes / (4.0 * self.d)


def _round_up(x: float, q: int) -> int:
    return int(math.ceil(x / q)) * q


INDEX_BITMAP = 255  # k_bloom value of the exact bitmap index (include/lhc.h)


def size_for(d: int, n: float, k: int = 3, k_bloom: int = 0, L: int = 1024,
             gamma: float = GAMMA_DEFAULT) -> Sizing:
    """(m, c) minimising m + 32c for an expected aggregate support of n coordinates.

    k_bloom = INDEX_BITMAP selects the exact bitmap index of §3.2: m is one
    bit per coordinate (rounded up to whole rows), no false positives, c = gamma n."""
    if k_bloom == INDEX_BITMAP:
        n = max(float(n), 1.0)
        m = (d + L - 1) // L * L
        c = max(k * L, _round_up(gamma * n, k * L))
        return Sizing(d, m, c, k, INDEX_BITMAP, L, n, 0.0, n, gamma)
    kb = k_bloom or k
    qm, qc = kb * L, k * L
    n = max(float(n), 1.0)
    best = None
    # scan bits per expected item from 1 to 64 (fine grid), then refine locally
    grid = [0.25 * i for i in range(4, 257)]
    for bpe in grid:
        m = max(qm, _round_up(bpe * n, qm))
        eps = bloom_fp_rate(m, n, kb)
        nc = n + eps * (d - n)
        c = max(qc, _round_up(gamma * nc, qc))
        cost = m + 32 * c
        if best is None or cost < best[0]:
            best = (cost, m, c, eps, nc)
    _, m, c, eps, nc = best
    return Sizing(d, m, c, k, kb, L, n, eps, nc, gamma)


def size_workload(d: int, density: float, workers: int, **kw) -> Sizing:
    return size_for(d, union_support(d, density, workers), **kw)


def smaller_index(d: int, density: float, workers: int, **kw) -> int:
    """The index kind with the smaller sketch for this workload: 0 (Bloom filter
    with k probes) or INDEX_BITMAP (the paper's footnote P:L160: the Bloom filter is
    "only theoretically necessary when the sparsity is extremely high")."""
    bloom = size_workload(d, density, workers, **kw)
    exact = size_workload(d, density, workers, k_bloom=INDEX_BITMAP,
                          **{k: v for k, v in kw.items() if k != "k_bloom"})
    return INDEX_BITMAP if exact.sketch_bytes < bloom.sketch_bytes else 0


# ---- §3.3 theory ------------------------------------------------

def binary_entropy(x: float) -> float:
    if x <= 0.0 or x >= 1.0:
        return 0.0
    return -x * math.log2(x) - (1 - x) * math.log2(1 - x)


def f0(x: float) -> float:
    """f(0, x) = (x + 1) H(1 / (x + 1))."""
    return (x + 1.0) * binary_entropy(1.0 / (x + 1.0))


def s_min_bits(n: float, lam: float, C: int) -> float:
    """S_min = n f(0, lambda) + n log2(2^C - 1)."""
    return n * f0(lam) + n * math.log2(2.0 ** C - 1.0)


def optimal_eps(C: int, lam: float, gamma: float = GAMMA_PAPER) -> float:
    """eps = (ln^2 2 * gamma * C * lambda)^-1, clamped to 1."""
    return min(1.0, 1.0 / (math.log(2) ** 2 * gamma * C * lam))


def bloom_bits(n: float, eps: float) -> float:
    """n / ln 2 * log2(1/eps)."""
    return n / math.log(2) * math.log2(1.0 / eps)


def paper_sizes(n: float, lam: float, C: int, gamma: float = GAMMA_PAPER):
    """(S1, S2) of P:L244-247 at the optimal eps."""
    eps = optimal_eps(C, lam, gamma)
    s1 = bloom_bits(n, eps)
    s2 = gamma * C * n * (1.0 + eps * lam)
    return s1, s2


# ---- sharded decode (DESIGN.md NEXT-2) ----------------------------------------

@dataclass
class ShardPlan:
    """Coordinates [0, d) split into `shards` contiguous ranges of `width`
    coordinates (a multiple of 1024: whole compress tiles and whole rows); shard q
    is an independent sketch of its range, sized for its share of the support."""
    d: int
    shards: int
    width: int
    sizing: Sizing           # of the largest (full-width) shard

    def bounds(self, q: int) -> tuple[int, int]:
        lo = q * self.width
        return lo, min(self.d, lo + self.width)

    def shard_d(self, q: int) -> int:
        lo, hi = self.bounds(q)
        return hi - lo

    def shard_m(self, q: int) -> int:
        """m of shard q: equal on every shard, except the exact bitmap index
        (one bit per coordinate of the shard, whole rows)."""
        s = self.sizing
        if s.k_bloom == INDEX_BITMAP:
            return (self.shard_d(q) + s.L - 1) // s.L * s.L
        return s.m


def shard_plan(d: int, shards: int, density: float, workers: int, **kw) -> ShardPlan:
    if shards < 1:
        raise ValueError("shards must be >= 1")
    width = -(-d // shards)
    width = -(-width // 1024) * 1024
    if (shards - 1) * width >= d:
        raise ValueError(f"d={d} is too small for {shards} non-empty shards of {width}")
    return ShardPlan(d, shards, width, size_workload(width, density, workers, **kw))


# ---- NEXT-4: the paper's optimal Bloom configuration --------------

K_MAX = 8  # probes / hashes the kernels support (include/lhc.h)


def size_paper_optimal(d: int, n: float, C: int = 32, gamma: float = GAMMA_DEFAULT, k: int = 3,
                       L: int = 1024) -> Sizing:
    """The §3.3 construction: false-positive rate eps* = (ln^2 2 * gamma * C * lambda)^-1
    with lambda n = N - n, a Bloom filter of n/ln2 * log2(1/eps*) bits
    hashing every nonzero to log2(1/eps*) bits (rounded, at most K_MAX), and
    c = gamma (n + eps (N - n)) counters with eps the realised false-positive
    rate of the partitioned filter.  Rounded to the kernels' multiples (k_B L, k L)."""
    n = max(float(n), 1.0)
    lam = max((d - n) / n, 1e-12)
    eps_star = optimal_eps(C, lam, gamma)
    lg = math.log2(1.0 / eps_star) if eps_star < 1.0 else 0.0
    kb = max(1, min(K_MAX, int(round(lg))))
    m = max(kb * L, _round_up(n / math.log(2) * max(lg, 1.0), kb * L))
    eps = bloom_fp_rate(m, n, kb)
    nc = n + eps * (d - n)
    c = max(k * L, _round_up(gamma * nc, k * L))
    return Sizing(d, m, c, k, kb, L, n, eps, nc, gamma)


# ---- NEXT-3: blocked Count Sketch ----------------------------------------

def size_blocked(d: int, density: float, workers: int, cells_per_block: int = 12288,
                 k: int = 3, L: int = 1024, **kw) -> tuple[Sizing, int]:
    """Sizing of a blocked sketch: the unblocked (m, c) rule, then c rounded up to B
    blocks of k partitions of S rows (S*k*L cells per block, about cells_per_block)."""
    s = size_workload(d, density, workers, k=k, L=L, **kw)
    S = max(1, round(cells_per_block / (k * L)))
    blocks = max(1, math.ceil(s.c / (S * k * L)))
    c = blocks * S * k * L
    return Sizing(d, s.m, c, k, s.k_bloom, L, s.n_expected, s.eps, s.n_cand_expected, s.gamma), blocks
