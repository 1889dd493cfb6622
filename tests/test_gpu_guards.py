"""Out-of-bounds write checks of every kernel (-m gpu).

compute-sanitizer is not available on the GPU pool (runs under it are refused), so
SURVEY.md §4 T4 is covered the way the pool asks for: bounds checks of our own on
small cases, plus the comparison with the CPU oracle.  Every buffer a call writes
(sketches, workspace, candidate list, values, flags, dense output, stats) is a view
into a larger allocation whose guard bands before and after it are filled with a
canary; after the call every guard byte must still hold the canary, and the decode
must still equal the oracle's (flags, rounds, values exact under the dyadic law).
"""
import numpy as np
import pytest

from lhc_inputs import rng_for, support, values

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes on each side
CANARY = 0xA5


@pytest.fixture(scope="module")
def lhc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2402_07529_b200 as lhc

    lhc.lib()
    return lhc


class Guarded:
    """Views of `dtype[n]` inside canary-filled allocations."""

    def __init__(self):
        self.blocks = []

    def __call__(self, n, dtype, fill=None):
        itemsize = torch.empty(0, dtype=dtype).element_size()
        nbytes = max(1, n) * itemsize
        raw = torch.full((GUARD + nbytes + GUARD,), CANARY, dtype=torch.uint8, device="cuda")
        view = raw[GUARD:GUARD + nbytes].view(dtype)
        if fill is not None:
            view.fill_(fill)
        self.blocks.append((raw, nbytes))
        return view[:n] if n else view[:0]

    def intact(self):
        torch.cuda.synchronize()
        for raw, nbytes in self.blocks:
            head = raw[:GUARD]
            tail = raw[GUARD + nbytes:]
            if not (bool((head == CANARY).all()) and bool((tail == CANARY).all())):
                return False
        return True


def dyadic_workers(d, nnz, W, seed):
    xs = []
    for w in range(W):
        rng = rng_for(seed + w)
        idx = support(rng, d, nnz)
        x = np.zeros(d, np.float32)
        x[idx] = values(rng, len(idx), "dyadic")
        xs.append(x)
    return xs


CASES = [
    # d, nnz, W, L, k, blocks, gamma
    (10_000, 100, 2, 1024, 3, 0, 1.3),       # tiny config
    (1_000_003, 10_000, 3, 1024, 3, 0, 1.3),  # ragged tail
    (200_003, 3_000, 2, 32, 4, 0, 1.3),       # smallest L, run-time k
    (300_000, 6_000, 2, 128, 3, 8, 1.5),      # blocked sketch (k_peel_blocked)
    (500_000, 12_000, 2, 1024, 3, 0, 1.05),   # stalled decode (median fallback)
]


@pytest.mark.parametrize("d,nnz,W,L,k,blocks,gamma", CASES)
@pytest.mark.parametrize("decode", ["default", "deterministic", "split"])
def test_guard_bands_intact(lhc, ora, d, nnz, W, L, k, blocks, gamma, decode, monkeypatch):
    if decode == "split":  # the two-pass peel of the split state (forced at these sizes)
        if blocks:
            pytest.skip("the blocked sketch is peeled block-locally")
        monkeypatch.setenv("LHC_CELL_BUILD", "split")
    s = lhc.size_workload(d, nnz / d, W, L=L, k=k, gamma=gamma)
    c = s.c
    if blocks:
        S = max(1, -(-int(gamma * s.n_cand_expected) // (blocks * k * L)))
        c = blocks * S * k * L
    p = lhc.params(d, s.m, c, k, 0, L, 0x6A4D + d, blocks)
    op = ora.params(p.d, p.m, p.c, p.k, p.k_bloom, p.L, p.seed, p.blocks)
    xs = dyadic_workers(d, nnz, W, 500 + d % 7)
    _, _, ref = ora.pipeline(op, xs)
    g = Guarded()
    words, cells = p.words, int(p.c)
    bms = [g(words, torch.int32, 0) for _ in range(W)]
    cts = [g(cells, torch.float32, 0.0) for _ in range(W)]
    xin = [g(d, torch.float32) for _ in range(W)]
    for t, x in zip(xin, xs):
        t.copy_(torch.from_numpy(x))
    nnz_out = g(1, torch.int64, 0)
    # hash kernel
    hr = g(2 * 64 * k, torch.int32)
    lhc.sketch_hash_rows(p, 0, 64, hr)
    # clear, batched dense compress (one sketch per worker), aggregate into a fresh sketch
    lhc.sketch_clear_batch(p, bms, cts)
    lhc.sketch_compress_batch(p, xin, bms, cts, nnz_out=nnz_out)
    B = g(words, torch.int32, 0)
    Y = g(cells, torch.float32, 0.0)
    lhc.sketch_aggregate(p, bms, cts, B, Y)
    # row-major batched compress of all workers into one sketch (k_compress_rows)
    B3 = g(words, torch.int32, 0)
    Y3 = g(cells, torch.float32, 0.0)
    lhc.sketch_compress_batch(p, xin, [B3] * W, [Y3] * W)
    # COO compress of the same gradients into another sketch (plus out-of-range entries)
    B2 = g(words, torch.int32, 0)
    Y2 = g(cells, torch.float32, 0.0)
    bad = g(1, torch.int64, 0)
    for x in xs:
        idx = np.concatenate([np.flatnonzero(x), [d, d + 3]]).astype(np.uint32)
        val = np.concatenate([x[np.flatnonzero(x)], [1.0, 1.0]]).astype(np.float32)
        ti = g(len(idx), torch.int32)
        tv = g(len(val), torch.float32)
        ti.copy_(torch.from_numpy(idx.view(np.int32)))
        tv.copy_(torch.from_numpy(val))
        lhc.sketch_compress_coo(p, ti, tv, B2, Y2, bad)
    # decode
    cap = d
    ws = g(lhc.lhc_decompress_workspace(p, cap), torch.uint8)
    out_idx = g(cap, torch.int32)
    out_val = g(cap, torch.float32)
    out_pl = g(cap, torch.uint8)
    dense = g(d, torch.float32)
    stats = g(32, torch.uint8, 0)
    lhc.sketch_decompress(p, B, Y, ws, cap, out_idx, out_val, out_pl, dense, stats,
                          deterministic=(decode == "deterministic"))
    torch.cuda.synchronize()
    assert g.intact(), "a kernel wrote outside its buffer"
    assert int(bad.item()) == 2 * W
    assert np.array_equal(B.cpu().numpy().view(np.uint32), B2.cpu().numpy().view(np.uint32))
    assert np.array_equal(B.cpu().numpy().view(np.uint32), B3.cpu().numpy().view(np.uint32))
    assert np.array_equal(Y.cpu().numpy(), Y3.cpu().numpy())  # dyadic sums: exact in any order
    st = lhc.read_stats(stats)
    n = st["n_cand"]
    assert n == ref.stats.n_cand and st["rounds"] == ref.stats.rounds
    assert st["success"] == ref.stats.success and st["n_peeled"] == ref.stats.n_peeled
    assert np.array_equal(out_idx[:n].cpu().numpy().view(np.uint32), ref.cand)
    assert np.array_equal(out_pl[:n].cpu().numpy().astype(bool), ref.peeled)
    assert np.array_equal(out_val[:n].cpu().numpy().astype(np.float64), ref.val)
    assert np.array_equal(dense.cpu().numpy().astype(np.float64), ref.dense)
