// peel_rows.cu — Phase II steps 2-3 of Alg. 1 on sm_100a, organised by
// the rows of the batched layout instead of by single cells, with
// deterministic values.
//
// The synchronous peeling rounds of reading R10 ("figure out which indexes
// of Y are mapped by only one non-zero parameter ... deducting"; parallel
// rounds) run as two warp-cooperative phases per round over bit masks, with no
// frontier queue and no per-cell degree state:
//
//   X_r  one warp per destination row D of Y that round r-1 touched (all rows in
//        round 1).  The input rows that map into D under D's probe j are listed
//        in ascending order (a counting sort of the (input row, probe) pairs by
//        destination row).  Lane w owns the 32 cells 32w..32w+31 of D.  For every
//        listed row the lane loads one word of the row's REMAINING-candidate mask,
//        rotates it onto D's columns by the row's bias (two shuffles and a funnel
//        shift), and adds it into a saturating bit-sliced counter (ones, twos) and
//        into bit planes of the listed row's index (plane b ^= mask when bit b of
//        the index is set).  After the pass the pure cells — exactly one remaining
//        candidate, "mapped by only one" — are `ones & ~twos`, and the
//        planes hold, at a pure cell, the index of the listed row that owns its
//        candidate.  Each pure cell sets its candidate's bit in the claim mask of
//        probe j, and the owning input row is listed for Y_r.
//   Y_r  one warp per listed input row i.  Its candidates claimed this round are
//        the OR of the k claim masks; each takes its value from the pure cell of
//        the lowest claiming probe j (reading R10, as the oracle):
//        x_p = g_j(i) R[cell_j(p)] ("X_i can be deduced as g_j(i) Y_h_j(i)"),
//        written at its coordinate of the dense output, and is then deducted from
//        its other cells ("deducting Y_h_j(i) by g_j(i) X_i").  The row's
//        remaining mask loses the peeled bits; its destination rows are listed
//        for X_{r+1}.
//
// Residuals: R[e] = Y[e] + q * delta[e], where delta[e] is a 64-bit integer sum of
// the deductions -g x_p rounded to the fixed-point grid q (q = 2^(E-40), 2^E >
// max|Y|).  Integer sums commute, so R does not depend on the order in which the
// deductions land: the decode is deterministic — no launch geometry, scheduling
// or atomic order changes a bit of the output.  Under the dyadic law (values
// +-n 2^-12, sums < 2^12) every deduction is exact on the grid and every value
// bit-equals the oracle's; otherwise values stay within the fp32 tolerance of the
// fp64 oracle (the grid error, ~2^-40 max|Y| per deduction, is far below fp32's).
// A deduction too large for the grid sets Ctrl.fx_overflow and the decode
// reports failure.
//
// A grid barrier separates the phases; every read of a phase sees only what the
// previous phase wrote, so the peeled set, its round structure and `rounds` are
// exactly the synchronous rounds of the oracle.
//
// Finalize: candidates never peeled take the median over j of g_j R[cell_j(p)]
// (footnote P:L193; reading R11); the candidate list's values and flags
// are gathered by slot.
#include <cooperative_groups.h>
#include <cstdlib>

#include "launch.h"

namespace cg = cooperative_groups;

namespace lhc {

#ifndef LHC_ROWS_THREADS
#define LHC_ROWS_THREADS 256
#endif
constexpr int kRowsThreads = LHC_ROWS_THREADS;
constexpr int kRowsWarps = kRowsThreads / 32;
constexpr int kRowsUnroll = 8;
#ifndef LHC_ROWS_MINB
#define LHC_ROWS_MINB 3
#endif
#ifndef LHC_ROWS_TIMING
#define LHC_ROWS_TIMING 0
#endif  // listed rows whose mask words are in flight together

// Rank sort of each destination row's input-row list (the counting-sort scatter
// places them in an atomic order): entries of one row are distinct, so the rank of
// x is the number of smaller entries.  Warp per destination row.
__global__ void __launch_bounds__(256) k_pair_sort(uint64_t nD, const uint32_t* __restrict__ dst_off,
                                                   const uint32_t* __restrict__ src,
                                                   uint32_t* __restrict__ dst) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t D = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); D < nD; D += warps) {
        const uint32_t l0 = dst_off[D], l1 = dst_off[D + 1];
        for (uint32_t a = l0 + lane; a < l1; a += 32) {
            const uint32_t x = src[a];
            uint32_t rank = 0;
            for (uint32_t b = l0; b < l1; b++) rank += src[b] < x;
            dst[l0 + rank] = x;
        }
    }
}

// Rotation of a row mask between input-row columns and destination-row columns.
// Lane w holds word w of the source row (nw words, nw | 32); the result is word w
// of the row rotated so that bit t of the source lands at bit (t + s) mod L:
// destination word w takes source bits starting at (32 w - s) mod L.
__device__ __forceinline__ uint32_t rotate_row(uint32_t src_word, uint32_t s, uint32_t lane,
                                               const KParams& P) {
    const uint32_t sb = (32 * lane + P.L - s) & (P.L - 1);
    const uint32_t sw = sb >> 5, sh = sb & 31;
    const uint32_t lo = __shfl_sync(0xffffffffu, src_word, sw & (P.nw - 1));
    const uint32_t hi = __shfl_sync(0xffffffffu, src_word, (sw + 1) & (P.nw - 1));
    if (lane >= P.nw) return 0u;
    return sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
}

struct RowsArgs {
    KParams P;
    const float* counters;      // Y [c]
    const uint2* tabS;          // Count Sketch row maps [nrows * k]
    const uint32_t* gmask;      // candidate masks (query), words per mask
    const uint32_t* dst_off;    // [nD + 1]
    const uint32_t* dst_list;   // sorted input rows per destination row
    const uint32_t* cand;       // ascending candidate list [n_c]
    unsigned long long* delta;  // [c] fixed-point deductions
    uint32_t* rem;              // remaining-candidate masks
    uint32_t* claim;            // claim masks, k x words
    uint32_t* dmark;            // [nD]: last round for which D was listed for X
    uint32_t* ymark;            // [nrows]: last round for which row i was listed for Y
    uint32_t* xl;               // X worklists, 2 x nD destination rows (by round parity)
    uint32_t* yl;               // Y worklists, 2 x nrows input rows (by round parity)
    float* dense;               // [d] output
    float* out_val;
    uint8_t* out_peeled;
    lhc_stats* stats;
    Ctrl* ctrl;
    uint64_t cap;
    uint64_t words;             // words of a mask (whole rows: nrows * L / 32)
};

// Warp-aggregated append of the lanes' items (pred) to list[*n ...].
__device__ __forceinline__ void warp_append(bool pred, uint32_t item, uint32_t* list, uint32_t* n,
                                            uint32_t lane) {
    const uint32_t m = __ballot_sync(0xffffffffu, pred);
    if (!m) return;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(n, (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (pred) list[base + __popc(m & ((1u << lane) - 1))] = item;
}

// Per-warp shared memory: one staged entry per (lane, bit), so that the dependent
// loads of a lane's entries are issued together.
struct XSmem {
    uint32_t e[32][32];
};
constexpr int kLoads = 8;  // loads in flight per lane when a list is drained
constexpr int kYLoads = 4;
constexpr int kPlanes = 12; // bit planes of the listed-row index (lists <= 2^12, host-checked)

struct Fx {
    double q, inv_q;  // grid step and its inverse
};

// R[e] = Y[e] + q * delta[e], rounded once to fp32
__device__ __forceinline__ float residual(const RowsArgs& A, const Fx& fx, uint64_t e) {
    const double d = (double)(long long)__ldcg(A.delta + e);
    return (float)((double)__ldcg(A.counters + e) + d * fx.q);
}

// X_r for destination row D (warp-uniform).
template <int KT>
__device__ __forceinline__ void x_row(const RowsArgs& A, XSmem& sm, uint64_t D, uint32_t r,
                                      uint32_t lane) {
    const KParams& P = A.P;
    const uint32_t k = KT ? (uint32_t)KT : P.k;
    const uint32_t j = (uint32_t)((D % ((uint64_t)k * P.S_Y)) / P.S_Y);
    const uint32_t l0 = A.dst_off[D], l1 = A.dst_off[D + 1];
    const uint32_t n = l1 - l0;
    const uint32_t np = n > 1 ? 32 - __clz(n - 1) : 0;  // planes in use
    uint32_t ones = 0, twos = 0;
    uint32_t plane[kPlanes];
#pragma unroll
    for (int b = 0; b < kPlanes; b++) plane[b] = 0;
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t nc = min(32u, n - base);
        const uint32_t my_i = lane < nc ? A.dst_list[l0 + base + lane] : 0u;
        const uint32_t my_b = lane < nc ? map_bias(__ldg(A.tabS + (uint64_t)my_i * k + j)) : 0u;
        for (uint32_t u0 = 0; u0 < nc; u0 += kRowsUnroll) {
            uint32_t w[kRowsUnroll];
#pragma unroll
            for (int u = 0; u < kRowsUnroll; u++) {
                const uint32_t iu = __shfl_sync(0xffffffffu, my_i, (u0 + u) & 31);
                w[u] = (u0 + u < nc && lane < P.nw) ? __ldcg(A.rem + (uint64_t)iu * P.nw + lane) : 0u;
            }
#pragma unroll
            for (int u = 0; u < kRowsUnroll; u++) {
                const uint32_t bu = __shfl_sync(0xffffffffu, my_b, (u0 + u) & 31);
                const uint32_t x = rotate_row(w[u], bu, lane, P);
                twos |= ones & x;
                ones |= x;
                const uint32_t idx = base + u0 + u;  // warp-uniform
#pragma unroll
                for (int b = 0; b < kPlanes; b++)
                    if ((uint32_t)b < np && ((idx >> b) & 1u)) plane[b] ^= x;
            }
        }
    }
    const uint32_t pure = ones & ~twos;
    if (!__any_sync(0xffffffffu, pure != 0u)) return;
    // the owner of each pure cell: its listed-row index, read off the planes
    uint32_t ne = 0;
    for (uint32_t m = pure; m; m &= m - 1) {
        const uint32_t c = __ffs(m) - 1;
        uint32_t idx = 0;
#pragma unroll
        for (int b = 0; b < kPlanes; b++) idx |= ((plane[b] >> c) & 1u) << b;
        sm.e[ne++][lane] = idx << 5 | c;
    }
    uint32_t* claim = A.claim + (uint64_t)j * A.words;
    uint32_t* yl = A.yl + (uint64_t)(r & 1) * P.nrows;
    uint32_t* yn = &A.ctrl->yl_n[r & 1];
    const uint32_t nmax = __reduce_max_sync(0xffffffffu, ne);
    for (uint32_t q0 = 0; q0 < nmax; q0 += kLoads) {
        uint32_t iq[kLoads], yq[kLoads];
#pragma unroll
        for (int q = 0; q < kLoads; q++) iq[q] = q0 + q < ne ? A.dst_list[l0 + (sm.e[q0 + q][lane] >> 5)] : 0u;
#pragma unroll
        for (int q = 0; q < kLoads; q++) yq[q] = q0 + q < ne ? __ldg(A.tabS + (uint64_t)iq[q] * k + j).y : 0u;
#pragma unroll
        for (int q = 0; q < kLoads; q++) {
            const bool live = q0 + q < ne;
            if (live) {
                const uint32_t col = 32 * lane + (sm.e[q0 + q][lane] & 31);
                const uint64_t p = ((uint64_t)iq[q] << P.log2L) + ((col + P.L - (yq[q] & 0x7fffffffu)) & (P.L - 1));
                atomicOr(claim + (p >> 5), 1u << (p & 31));
            }
            const bool first = live && atomicExch(&A.ymark[iq[q]], r) != r;
            warp_append(first, iq[q], yl, yn, lane);
        }
    }
}

// Y_r for input row i (warp-uniform); returns the lane's number of peeled candidates.
template <int KT>
__device__ __forceinline__ uint32_t y_row(const RowsArgs& A, XSmem& sm, const Fx& fx, uint64_t i,
                                          uint32_t r, uint32_t lane) {
    const KParams& P = A.P;
    constexpr uint32_t NJ = KT ? KT : kMaxK;
    const uint32_t k = KT ? (uint32_t)KT : P.k;
    const uint64_t wi = i * P.nw + lane;
    const uint2 my_mp = lane < k ? __ldg(A.tabS + i * k + lane) : make_uint2(0u, 0u);
    uint32_t Dk[NJ], Yk[NJ];  // the row's maps, every lane (uniform shuffles)
#pragma unroll
    for (uint32_t j = 0; j < NJ; j++) {
        Dk[j] = __shfl_sync(0xffffffffu, my_mp.x, j);
        Yk[j] = __shfl_sync(0xffffffffu, my_mp.y, j);
    }
    const uint32_t rm = lane < P.nw ? __ldcg(A.rem + wi) : 0u;
    uint32_t cw[NJ];
#pragma unroll
    for (uint32_t j = 0; j < NJ; j++)
        cw[j] = (KT || j < k) && lane < P.nw ? __ldcg(A.claim + (uint64_t)j * A.words + wi) : 0u;
    // lowest claiming probe first: stage (j, bit) entries
    uint32_t N = 0, ne = 0;
#pragma unroll
    for (uint32_t j = 0; j < NJ; j++) {
        if (!KT && j >= k) break;
        if (cw[j]) A.claim[(uint64_t)j * A.words + wi] = 0u;  // ready for the next round
        for (uint32_t m = cw[j] & ~N; m; m &= m - 1) sm.e[ne++][lane] = j << 5 | (__ffs(m) - 1);
        N |= cw[j];
    }
    const uint32_t nmax = __reduce_max_sync(0xffffffffu, ne);
    for (uint32_t q0 = 0; q0 < nmax; q0 += kYLoads) {
        double yv[kYLoads];
        long long dv[kYLoads];
#pragma unroll
        for (int q = 0; q < kYLoads; q++) {
            const uint32_t en = q0 + q < ne ? sm.e[q0 + q][lane] : 0u;
            const uint32_t js = en >> 5, t = 32 * lane + (en & 31);
            uint32_t Dj = 0, yj = 0;
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++)
                if (j == js) Dj = Dk[j], yj = Yk[j];
            const uint64_t e = ((uint64_t)Dj << P.log2L) + ((t + (yj & 0x7fffffffu)) & (P.L - 1));
            yv[q] = q0 + q < ne ? (double)__ldcg(A.counters + e) : 0.0;
            dv[q] = q0 + q < ne ? (long long)__ldcg(A.delta + e) : 0ll;
        }
#pragma unroll
        for (int q = 0; q < kYLoads; q++) {
            if (q0 + q >= ne) continue;
            const uint32_t en = sm.e[q0 + q][lane];
            const uint32_t js = en >> 5, t = 32 * lane + (en & 31);
            uint32_t ys = 0;
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++)
                if (j == js) ys = Yk[j];
            const float val = ((ys >> 31) ? -1.f : 1.f) * (float)(yv[q] + (double)dv[q] * fx.q);
            A.dense[(i << P.log2L) + t] = val;
            // deduct g_j' x_p from the other cells (fixed point: order-free)
#pragma unroll
            for (uint32_t jj = 0; jj < NJ; jj++) {
                if ((!KT && jj >= k) || jj == js) continue;
                const double sc = (double)((Yk[jj] >> 31) ? val : -val) * fx.inv_q;
                if (fabs(sc) >= 0x1p61) atomicOr(&A.ctrl->fx_overflow, 1u);
                const uint64_t e = ((uint64_t)Dk[jj] << P.log2L) + ((t + (Yk[jj] & 0x7fffffffu)) & (P.L - 1));
                atomicAdd(A.delta + e, (unsigned long long)__double2ll_rn(sc));
            }
        }
    }
    if (__any_sync(0xffffffffu, N != 0u)) {
        if (lane < P.nw) A.rem[wi] = rm & ~N;
        const bool first = lane < k && atomicExch(&A.dmark[my_mp.x], r + 1) != r + 1;
        warp_append(first, my_mp.x, A.xl + (uint64_t)((r + 1) & 1) * (P.c >> P.log2L),
                    &A.ctrl->xl_n[(r + 1) & 1], lane);
    }
    return (uint32_t)__popc(N);
}

template <int KT>
__global__ void __launch_bounds__(kRowsThreads, LHC_ROWS_MINB) k_peel_rows(RowsArgs A) {
    cg::grid_group grid = cg::this_grid();
    const KParams& P = A.P;
    constexpr uint32_t NJ = KT ? KT : kMaxK;
    const uint32_t k = KT ? (uint32_t)KT : P.k;
    __shared__ XSmem sm_all[kRowsWarps];
    __shared__ uint32_t sh_cnt[2];
    const uint32_t lane = threadIdx.x & 31;
    XSmem& sm = sm_all[threadIdx.x >> 5];
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t gwarp = gtid >> 5, nwarps = gstride >> 5;
    const bool timer = blockIdx.x == 0 && threadIdx.x == 0;

    const uint64_t n_c = *(volatile unsigned long long*)&A.ctrl->n_cand;
    if (n_c > A.cap) {  // overflow: nothing is peeled (stats.overflow set by the query)
        if (gtid == 0) {
            A.stats->n_peeled = 0;
            A.stats->rounds = 0;
            A.stats->success = 0;
            A.stats->entries = 0;
        }
        return;
    }
    if (timer) A.ctrl->t[0] = globaltimer();
    const uint64_t nD = P.c >> P.log2L;
    // ---- init: rem = candidate masks, claims = 0, delta = 0, dense = 0, flags; max|Y|
    {
        const uint4* g4 = reinterpret_cast<const uint4*>(A.gmask);
        uint4* m4 = reinterpret_cast<uint4*>(A.rem);
        for (uint64_t u = gtid; u < A.words / 4; u += gstride) m4[u] = __ldcg(g4 + u);
        for (uint64_t u = 4 * (A.words / 4) + gtid; u < A.words; u += gstride) A.rem[u] = A.gmask[u];
        for (uint64_t u = gtid; u < (uint64_t)k * A.words; u += gstride) A.claim[u] = 0u;
        ulonglong2* z2 = reinterpret_cast<ulonglong2*>(A.delta);
        for (uint64_t u = gtid; u < P.c / 2; u += gstride) z2[u] = make_ulonglong2(0ull, 0ull);
        float4* d4 = reinterpret_cast<float4*>(A.dense);
        const uint64_t n4 = P.d / 4;
        for (uint64_t u = gtid; u < n4; u += gstride) __stcs(d4 + u, make_float4(0.f, 0.f, 0.f, 0.f));
        for (uint64_t u = 4 * n4 + gtid; u < P.d; u += gstride) A.dense[u] = 0.f;
        for (uint64_t u = gtid; u < nD; u += gstride) A.dmark[u] = 0u;
        for (uint64_t u = gtid; u < P.nrows; u += gstride) A.ymark[u] = 0u;
        float mx = 0.f;
        const float4* y4 = reinterpret_cast<const float4*>(A.counters);
        for (uint64_t u = gtid; u < P.c / 4; u += gstride) {
            const float4 y = __ldcg(y4 + u);
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(y.x), fabsf(y.y)), fmaxf(fabsf(y.z), fabsf(y.w))));
        }
        mx = __reduce_max_sync(0xffffffffu, __float_as_uint(mx)) ? __uint_as_float(
                 __reduce_max_sync(0xffffffffu, __float_as_uint(mx))) : 0.f;
        if (lane == 0 && mx > 0.f) atomicMax(&A.ctrl->ymax_bits, __float_as_uint(mx));
    }
    if (threadIdx.x == 0) sh_cnt[0] = sh_cnt[1] = 0;
    grid.sync();
    if (timer) A.ctrl->t[2] = globaltimer();
    Fx fx;
    {
        const float mx = __uint_as_float(*(volatile uint32_t*)&A.ctrl->ymax_bits);
        int E = 0;
        if (mx > 0.f) frexpf(mx, &E);  // mx < 2^E
        fx.q = ldexp(1.0, E - 40);
        fx.inv_q = ldexp(1.0, 40 - E);
    }

    uint64_t n_peeled = 0, work = 0;
    uint32_t rounds = 0;
    for (uint32_t r = 1;; r++) {
        unsigned long long* rc = &A.ctrl->rc[r % 3];
        if (gtid == 0) {
            A.ctrl->rc[(r + 1) % 3] = 0ull;  // last used in round r - 2
            if (r + 3 < (uint32_t)kCtrlTimes - 1) A.ctrl->t[r + 3] = globaltimer();
        }
        // ---- X_r: destination rows touched by round r - 1 (all rows in round 1) ----
        if (gtid == 0) A.ctrl->xl_n[(r + 1) & 1] = 0u;  // X_{r+1}'s list, last read in X_{r-1}
        const uint64_t nx = r == 1 ? nD : *(volatile uint32_t*)&A.ctrl->xl_n[r & 1];
        const uint32_t* xl = A.xl + (uint64_t)(r & 1) * nD;
        uint32_t n_x = 0;
        for (uint64_t q = gwarp; q < nx; q += nwarps) {
            const unsigned long long c0 = LHC_ROWS_TIMING ? clock64() : 0;
            x_row<KT>(A, sm, r == 1 ? q : xl[q], r, lane);
            if (LHC_ROWS_TIMING && lane == 0 && r < 128) atomicAdd(&A.ctrl->dbg[1][r], clock64() - c0);
            n_x++;
        }
        if (lane == 0 && n_x) atomicAdd(&sh_cnt[1], n_x);
        if (LHC_ROWS_TIMING && lane == 0 && r < (uint32_t)kCtrlTimes) atomicMax(&A.ctrl->tproc[r], globaltimer());
        grid.sync();
        if (LHC_ROWS_TIMING && gtid == 0 && r < (uint32_t)kCtrlTimes) A.ctrl->fsize[r] = (uint32_t)((globaltimer() - A.ctrl->t[r + 3]) / 100);
        // ---- Y_r: input rows that own the only candidate of a pure cell -------------
        if (gtid == 0) A.ctrl->yl_n[(r + 1) & 1] = 0u;  // X_{r+1} appends, last read in Y_{r-1}
        const uint64_t ny = *(volatile uint32_t*)&A.ctrl->yl_n[r & 1];
        const uint32_t* yl = A.yl + (uint64_t)(r & 1) * P.nrows;
        uint32_t n_y = 0;
        for (uint64_t q = gwarp; q < ny; q += nwarps) {
            const unsigned long long c0 = LHC_ROWS_TIMING ? clock64() : 0;
            n_y += y_row<KT>(A, sm, fx, yl[q], r, lane);
            if (LHC_ROWS_TIMING && lane == 0 && r < 128) atomicAdd(&A.ctrl->dbg[3][r], clock64() - c0);
        }
        n_y = __reduce_add_sync(0xffffffffu, n_y);  // y_row counts the lane's word
        if (LHC_ROWS_TIMING && lane == 0 && r < (uint32_t)kCtrlTimes) atomicMax(&A.ctrl->tflush[r], globaltimer());
        if (lane == 0 && n_y) atomicAdd(&sh_cnt[0], n_y);
        __syncthreads();
        if (threadIdx.x == 0) {
            if (sh_cnt[0]) atomicAdd(rc, (unsigned long long)sh_cnt[0]);
            if (sh_cnt[1]) atomicAdd(rc, (unsigned long long)sh_cnt[1] << 40);
            sh_cnt[0] = sh_cnt[1] = 0;
        }
        grid.sync();
        const unsigned long long v = *(volatile unsigned long long*)rc;
        const uint64_t np = v & ((1ull << 40) - 1);
        work += v >> 40;
        if (!np) break;
        n_peeled += np;
        rounds = r;
    }
    if (timer) A.ctrl->t[kCtrlTimes - 1] = globaltimer();

    // ---- finalize: median fallback, values and flags by slot ---------------
    for (uint64_t s = gtid; s < n_c; s += gstride) {
        const uint32_t p = __ldg(A.cand + s);
        const bool unpeeled = (__ldcg(A.rem + (p >> 5)) >> (p & 31)) & 1u;
        float val;
        if (!unpeeled) {
            val = __ldcg(A.dense + p);
        } else {
            const uint64_t i = p >> P.log2L;
            const uint32_t t = p & (P.L - 1);
            float v[NJ];
            for (uint32_t j = 0; j < k; j++) {
                const uint2 mp = __ldg(A.tabS + i * k + j);
                const uint64_t e = ((uint64_t)mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1));
                v[j] = map_sign(mp) * residual(A, fx, e);
            }
            for (uint32_t a = 1; a < k; a++) {  // insertion sort of <= 8 values
                const float x = v[a];
                int b = (int)a - 1;
                while (b >= 0 && v[b] > x) { v[b + 1] = v[b]; b--; }
                v[b + 1] = x;
            }
            val = (k & 1) ? v[k / 2] : 0.5f * (v[k / 2 - 1] + v[k / 2]);
            A.dense[p] = val;
        }
        A.out_val[s] = val;
        A.out_peeled[s] = unpeeled ? 0 : 1;
    }
    if (gtid == 0) {
        const bool fx_ok = *(volatile uint32_t*)&A.ctrl->fx_overflow == 0u;
        A.stats->n_peeled = n_peeled;
        A.stats->rounds = rounds;
        A.stats->success = n_peeled == n_c && fx_ok ? 1 : 0;
        A.stats->entries = work;  // destination-row work items of the X phases
        A.ctrl->rounds_dbg = rounds;
    }
}

static int rows_grid(int dev, bool k3) {
    static int cached[64][2] = {};
    if (dev < 64 && cached[dev][k3]) return cached[dev][k3];
    int per_sm = 0;
    const void* f = k3 ? (const void*)k_peel_rows<3> : (const void*)k_peel_rows<0>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kRowsThreads, 0);
    const int g = std::max(1, per_sm) * num_sms();
    if (dev < 64) cached[dev][k3] = g;
    return g;
}

cudaError_t launch_peel_rows(const KParams& P, const float* counters, const uint2* tabS,
                             const uint32_t* gmask, uint32_t* dst_off, uint32_t* pair_pos,
                             uint32_t* dst_tmp, uint32_t* dst_list, const uint32_t* cand,
                             unsigned long long* delta, uint32_t* rem, uint32_t* claim,
                             uint32_t* dmark, uint32_t* ymark, uint32_t* xl, uint32_t* yl,
                             float* dense, uint64_t cap, float* out_val, uint8_t* out_peeled,
                             Ctrl* ctrl, lhc_stats* stats, cudaStream_t s) {
    // (input row, probe) pairs by destination row, each row's list ascending
    launch_pair_lists(P, tabS, dst_off, pair_pos, dst_tmp, s);
    const uint64_t nD = P.c >> P.log2L;
    const uint32_t gs = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((nD + 7) / 8, (uint64_t)num_sms() * 16));
    k_pair_sort<<<gs, 256, 0, s>>>(nD, dst_off, dst_tmp, dst_list);
    count_launch();

    int dev = 0;
    cudaGetDevice(&dev);
    RowsArgs A{};
    A.P = P;
    A.counters = counters;
    A.tabS = tabS;
    A.gmask = gmask;
    A.dst_off = dst_off;
    A.dst_list = dst_list;
    A.cand = cand;
    A.delta = delta;
    A.rem = rem;
    A.claim = claim;
    A.dmark = dmark;
    A.ymark = ymark;
    A.xl = xl;
    A.yl = yl;
    A.dense = dense;
    A.out_val = out_val;
    A.out_peeled = out_peeled;
    A.stats = stats;
    A.ctrl = ctrl;
    A.cap = cap;
    A.words = (uint64_t)P.nrows * P.nw;
    void* args[] = {(void*)&A};
    const bool k3 = P.k == 3;
    int grid = rows_grid(dev, k3);
    if (const char* g = getenv("LHC_PEEL_GRID"))  // test hook: any co-resident grid gives the same bytes
        grid = std::max(1, std::min(grid, atoi(g)));
    cudaError_t err = cudaLaunchCooperativeKernel(k3 ? (const void*)k_peel_rows<3> : (const void*)k_peel_rows<0>,
                                                  dim3(grid), dim3(kRowsThreads), args, 0, s);
    count_launch();
    return err;
}

}  // namespace lhc
