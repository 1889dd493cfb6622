// peel.cu — Phase II steps 2-3 of Alg. 1 on sm_100a: the frontier-
// based parallel peeling decoder and the Count Sketch median
// fallback for what peeling cannot reach (footnote P:L193).
//
// One cooperative, persistent kernel (grid-wide barriers between phases) so that
// the whole round loop runs on the device with no host round trips:
//   build    cell state {key, R = Y} by destination row, without atomics on cells:
//            the (input row, probe) pairs are counting-sorted by destination row;
//            a warp per destination row rotates the query masks of its listed
//            input rows and sums key = sum over its candidates p of (2^32 + p)
//            (degree and coordinate sum) in shared memory, then writes the row once
//   F0       every cell of degree one is appended to the frontier queue as the
//            pair (cell, coordinate of its only candidate)
//   rounds   (synchronous, reading R10) for every queue entry (e, p) of the
//            previous round's segment: claim p (fetch-or of its bit — a candidate can
//            be the only one left in several cells; a stale entry whose candidate
//            was peeled meanwhile fails the claim), read val = sign * R[e] ("mapped by
//            only one non-zero parameter"; "X_i can be deduced as
//            g_j(i) * Y_h_j(i)"), write it to the dense output at p, and subtract
//            sign_j * val and (2^32 + p) from the other cells of p ("deducting
//            Y_h_j(i) by g_j(i) * X_i").  A cell
//            whose degree drops from 2 to 1 is appended for the next round with
//            its remaining candidate, which is the slot sum left in the key.  A
//            round consumes only the segment the previous round appended, so the
//            set of candidates peeled per round, and the number of rounds, are
//            exactly those of synchronous peeling.
//   finalize unpeeled candidates take the median over j of sign_j * R;
//            a warp per 1024-coordinate chunk assembles the chunk in shared memory
//            (zeros, the chunk's peeled values, its medians), writes the list values
//            of the chunk's candidate slots and the chunk of the dense output with
//            full-line stores.
// A peeled value is not stored at its coordinate during the rounds (a random 4-byte
// store into the 4d-byte output costs a partial-sector read-modify-write in HBM):
// it is appended as (coordinate, value) to its chunk's segment of a log whose
// segments start at the chunk's first candidate slot (the query's row offsets), so
// the appends of a chunk fill whole lines and the finalize reads them back in order.
// Queue appends go to warp-private shared-memory buffers (no block barrier inside a
// round; one global reservation per CTA and round, or per full buffer); every cell
// enters the queue at most once (c entries).  When the 8-byte state exceeds the L2
// but its 4-byte key array fits, the rounds run in two passes over a split state
// (peel_split: keys first, then the residuals replayed segment by segment).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "launch.h"

namespace cg = cooperative_groups;

namespace lhc {

#ifndef LHC_PEEL_TIMING
#define LHC_PEEL_TIMING 0
#endif
#ifndef LHC_PEEL_THREADS
#define LHC_PEEL_THREADS 512
#endif
constexpr int kPeelThreads = LHC_PEEL_THREADS;
#ifndef LHC_PEEL_MINB
#define LHC_PEEL_MINB 2  // 64 registers: two 512-thread CTAs per SM
#endif

__device__ __forceinline__ uint32_t cand_cell(const KParams& P, const uint2* __restrict__ tabS,
                                              uint32_t p, uint32_t j, uint32_t* neg) {
    const uint64_t i = p >> P.log2L;
    const uint32_t t = p & (P.L - 1);
    const uint2 mp = __ldg(tabS + i * P.k + j);
    *neg = mp.y >> 31;
    return (mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1));  // c < 2^32
}

constexpr int kRowsAhead = 8;  // listed rows whose mask words are loaded back to back

// In-place exclusive scan of a[0..n) by one block (a[n-1] becomes the total when
// the input's last element is 0).
__device__ void block_excl_scan(uint32_t* a, uint32_t n, uint32_t* sh) {
    const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t b = threadIdx.x * per, e = min(n, b + per);
    uint32_t sum = 0;
    // the thread's elements are loaded 8 at a time (independent loads in flight)
    for (uint32_t t0 = b; t0 < e; t0 += 8) {
        uint32_t v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) v[q] = t0 + q < e ? a[t0 + q] : 0u;
#pragma unroll
        for (int q = 0; q < 8; q++) sum += v[q];
    }
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; w++) {
            const uint32_t v = sh[w];
            sh[w] = run;
            run += v;
        }
    }
    __syncthreads();
    uint32_t run = sh[warp] + x - sum;
    for (uint32_t t0 = b; t0 < e; t0 += 8) {
        uint32_t v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) v[q] = t0 + q < e ? a[t0 + q] : 0u;
#pragma unroll
        for (int q = 0; q < 8; q++)
            if (t0 + q < e) {
                a[t0 + q] = run;
                run += v[q];
            }
    }
}

// queue-buffer entries per thread: a peel appends at most k - 1 cells, an F0
// pass at most 4
__host__ __device__ constexpr uint32_t peel_q_per_thread(uint32_t k) { return k - 1 > 4 ? k - 1 : 8; }

// Loads that must stay where they are written (issued before a dependent branch).
__device__ __forceinline__ uint32_t ld_nc_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_nc_u2(const uint2* p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_cg_f32(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}

// L2 eviction-priority hints (LHC_PEEL_HINTS): the decode state is reused every
// round, the dense output is written once per coordinate.
#ifndef LHC_PEEL_HINTS
#define LHC_PEEL_HINTS 1
#endif
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_hint(float* a, float v, uint64_t pol) {
    if (LHC_PEEL_HINTS)
        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
    else
        *a = v;
}
__device__ __forceinline__ void red_add_hint(float* a, float v, uint64_t pol) {
    if (LHC_PEEL_HINTS)
        asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
    else
        atomicAdd(a, v);
}
__device__ __forceinline__ unsigned long long atom_add_hint(unsigned long long* a, unsigned long long v,
                                                            uint64_t pol) {
    if (!LHC_PEEL_HINTS) return atomicAdd(a, v);
    unsigned long long old;
    asm volatile("atom.global.add.L2::cache_hint.u64 %0, [%1], %2, %3;"
                 : "=l"(old) : "l"(a), "l"(v), "l"(pol) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t atom_add_hint(uint32_t* a, uint32_t v, uint64_t pol) {
    if (!LHC_PEEL_HINTS) return atomicAdd(a, v);
    uint32_t old;
    asm volatile("atom.global.add.L2::cache_hint.u32 %0, [%1], %2, %3;"
                 : "=r"(old) : "l"(a), "r"(v), "l"(pol) : "memory");
    return old;
}

// The frontier queue and the value log are streamed (written once, read once a round
// or a phase later): evict-first so that they do not push the decode state out of L2.
#ifndef LHC_STREAM_QUEUE
#define LHC_STREAM_QUEUE 1
#endif
template <typename T>
__device__ __forceinline__ void st_stream(T* a, T v) {
    if (LHC_STREAM_QUEUE) __stcs(a, v); else *a = v;
}
template <typename T>
__device__ __forceinline__ T ld_stream(const T* a) {
    if (LHC_STREAM_QUEUE) return __ldcs(a);
    return *a;
}

// Block-aggregated append of the pairs in sh_q to the queue segment that starts
// at seg_base, through the low half of the round's counter rc.
__device__ __forceinline__ void flush_queue(uint2* sh_q, uint32_t* sh_n, uint32_t* sh_base,
                                            uint2* frontier, uint32_t seg_base,
                                            unsigned long long* rc) {
    __syncthreads();
    const uint32_t n = *sh_n;
    if (threadIdx.x == 0 && n) *sh_base = seg_base + (uint32_t)atomicAdd(rc, (unsigned long long)n);
    __syncthreads();  // every thread has read n: the count can be reset before the copy
    if (threadIdx.x == 0) *sh_n = 0;
    for (uint32_t a = threadIdx.x; a < n; a += blockDim.x) frontier[*sh_base + a] = sh_q[a];
    __syncthreads();
}

// Warp-private append buffers (kWarpQ entries of the shared queue buffer per warp):
// the warps of a CTA append without block barriers; a full buffer is flushed by its
// warp alone (one global reservation), the rest once per round by the CTA (one
// reservation for all its warps, with the round's peel count in the high half).
constexpr uint32_t kWarpQ = 512;
__device__ __forceinline__ void wq_push(bool has, uint2 v, uint2* wbuf, uint32_t& wn, uint2* frontier,
                                        uint32_t seg_base, unsigned long long* rc) {
    const uint32_t lane = threadIdx.x & 31;
    if (wn + 32 > kWarpQ) {  // warp-uniform
        __syncwarp();
        uint32_t b = 0;
        if (lane == 0) b = (uint32_t)atomicAdd(rc, (unsigned long long)wn);
        b = __shfl_sync(0xffffffffu, b, 0) + seg_base;
        for (uint32_t a = lane; a < wn; a += 32) st_stream(frontier + b + a, wbuf[a]);
        __syncwarp();
        wn = 0;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, has);
    if (has) wbuf[wn + __popc(m & ((1u << lane) - 1u))] = v;
    wn += __popc(m);
}
// End of a round: every warp's remaining entries, one reservation per CTA.
__device__ __forceinline__ void wq_round_end(uint2* wbuf, uint32_t& wn, uint32_t& wpeel, uint32_t* sh_wc,
                                             uint32_t* sh_wp, uint32_t* sh_base, uint2* frontier,
                                             uint32_t seg_base, unsigned long long* rc) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    __syncwarp();
    if (lane == 0) { sh_wc[warp] = wn; sh_wp[warp] = wpeel; }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0, pe = 0;
        for (uint32_t w = 0; w < nwarps; w++) {
            const uint32_t c = sh_wc[w];
            sh_wc[w] = tot;
            tot += c;
            pe += sh_wp[w];
        }
        *sh_base = tot || pe ? seg_base + (uint32_t)atomicAdd(rc, ((unsigned long long)pe << 32) + tot) : 0u;
    }
    __syncthreads();
    const uint32_t b = *sh_base + sh_wc[warp];
    for (uint32_t a = lane; a < wn; a += 32) st_stream(frontier + b + a, wbuf[a]);
    wn = 0;
    wpeel = 0;
}

// ---- cell state by destination row, without atomics on cells ---------------------
// (used when the cell state, 16 B per cell, does not fit in L2: then the
// per-candidate 64-bit reductions of the in-kernel insert go to HBM at random)
// The (input row i, probe j) pairs are counting-sorted by their destination row
// D = row_j(i) of Y (count with reservations, one-block scan, scatter); then a warp
// per destination row rotates the query masks of its listed input rows and sums
// key = sum over the row's candidates p of (2^32 + p) (degree and coordinate sum)
// in registers, lane w owning columns 32w .. 32w + 31, and writes the row's cells
// {key, R = Y} once.
__global__ void __launch_bounds__(256) k_pair_count(KParams P, const uint2* __restrict__ tabS,
                                                    uint32_t* dst_off, uint32_t* pair_pos) {
    const uint64_t n = (uint64_t)P.nrows * P.k;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
         q += (uint64_t)gridDim.x * blockDim.x)
        pair_pos[q] = atomicAdd(dst_off + __ldg(&tabS[q].x), 1u);
}

__global__ void __launch_bounds__(1024) k_pair_scan(uint32_t* dst_off, uint32_t n) {
    __shared__ uint32_t sh[32];
    block_excl_scan(dst_off, n, sh);
}


__global__ void __launch_bounds__(256) k_pair_scatter(KParams P, const uint2* __restrict__ tabS,
                                                      const uint32_t* __restrict__ dst_off,
                                                      const uint32_t* __restrict__ pair_pos,
                                                      uint32_t* __restrict__ dst_list) {
    const uint64_t n = (uint64_t)P.nrows * P.k;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
         q += (uint64_t)gridDim.x * blockDim.x)
        dst_list[dst_off[__ldg(&tabS[q].x)] + pair_pos[q]] = (uint32_t)(q / P.k);
}

#ifndef LHC_BUILD_MINB
#define LHC_BUILD_MINB 3  // 80 registers: 3 CTAs of 256 per SM (VGG build 167 -> 140 us)
#endif
// SPLIT (compact only): keys and residuals in two arrays, keys = cells_v[0, c),
// R = cells_v[c, 2c) as 4-byte words (the two-pass peel, peel_split).
template <bool COMPACT, bool SPLIT>
__global__ void __launch_bounds__(256, LHC_BUILD_MINB)
k_build_cells(KParams P, const float* __restrict__ counters, const uint2* __restrict__ tabS,
              const uint32_t* __restrict__ gmask, const uint32_t* __restrict__ dst_off,
              const uint32_t* __restrict__ dst_list, void* __restrict__ cells_v, Ctrl* ctrl,
              uint2* __restrict__ frontier) {
    using Acc = typename std::conditional<COMPACT, uint32_t, unsigned long long>::type;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = P.nw;
    const uint64_t nD = P.c >> P.log2L;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t D = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); D < nD;
         D += warps) {
        const uint32_t j = (uint32_t)((D % ((uint64_t)P.k * P.S_Y)) / P.S_Y);  // probe of row D
        Acc acc[32];
#pragma unroll
        for (int c = 0; c < 32; c++) acc[c] = 0;
        const uint32_t l0 = dst_off[D], l1 = dst_off[D + 1];
        if (COMPACT && l1 - l0 > kCompactMaxDeg && lane == 0) atomicOr(&ctrl->compact_fail, 1u);
        for (uint32_t base = l0; base < l1; base += 32) {
            // 32 listed rows at a time: lane r loads row r and its bias ...
            const uint32_t n = min(32u, l1 - base);
            const uint32_t my_i = lane < n ? dst_list[base + lane] : 0u;
            const uint32_t my_b = lane < n ? map_bias(__ldg(tabS + (uint64_t)my_i * P.k + j)) : 0u;
            // ... then kRowsAhead rows' mask words are loaded back to back
            for (uint32_t r0 = 0; r0 < n; r0 += kRowsAhead) {
                uint32_t mws[kRowsAhead], is[kRowsAhead], bs[kRowsAhead];
#pragma unroll
                for (int u = 0; u < kRowsAhead; u++) {
                    is[u] = __shfl_sync(0xffffffffu, my_i, (r0 + u) & 31);
                    bs[u] = __shfl_sync(0xffffffffu, my_b, (r0 + u) & 31);
                    mws[u] = (r0 + u < n && lane < nw) ? __ldg(gmask + (uint64_t)is[u] * nw + lane) : 0u;
                }
#pragma unroll
                for (int u = 0; u < kRowsAhead; u++) {
                    // destination word w = lane takes source bits (32w - b) mod L ..
                    const uint32_t b = bs[u];
                    const uint32_t sb = (32 * lane + P.L - b) & (P.L - 1);
                    const uint32_t sw = sb >> 5, sh = sb & 31;
                    const uint32_t lo = __shfl_sync(0xffffffffu, mws[u], sw & (nw - 1));
                    const uint32_t hi = __shfl_sync(0xffffffffu, mws[u], (sw + 1) & (nw - 1));
                    const uint32_t dst = lane < nw ? (sh ? (lo >> sh) | (hi << (32 - sh)) : lo) : 0u;
                    if (dst) {
                        if (COMPACT) {
                            const uint32_t add = (1u << 24) + is[u];
#pragma unroll
                            for (int c = 0; c < 32; c++)
                                if (dst & (1u << c)) acc[c] += add;
                        } else {
                            // coordinate of column 32w + c: i*L + (32w + c - b) mod L
                            const uint64_t pbase = ((uint64_t)is[u] << P.log2L) + (1ull << 32);
                            const uint32_t t0 = 32 * lane + P.L - b;
#pragma unroll
                            for (int c = 0; c < 32; c++)
                                if (dst & (1u << c)) acc[c] += pbase + ((t0 + c) & (P.L - 1));
                        }
                    }
                }
            }
        }
        // F0 fused: the row's cells of degree one are appended to the frontier queue
        // (one reservation per row) as (cell, id) — id as in the peel's F0
        uint32_t m1 = 0;
#pragma unroll
        for (int c = 0; c < 32; c++) m1 |= (uint32_t)((acc[c] >> (COMPACT ? 24 : 32)) == 1u) << c;
        if (lane >= nw) m1 = 0;
        uint32_t fpos;
        {
            const uint32_t n1 = __popc(m1);
            uint32_t x = n1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
            uint32_t base = 0;
            if (lane == 31 && tot) base = (uint32_t)atomicAdd(&ctrl->rc[0], (unsigned long long)tot);
            fpos = __shfl_sync(0xffffffffu, base, 31) + x - n1;
        }
        if (SPLIT && lane < nw) {
            const uint64_t e0 = (D << P.log2L) + 32 * lane;
            const float4* y4 = reinterpret_cast<const float4*>(counters + e0);
            uint4* k4 = reinterpret_cast<uint4*>(static_cast<uint32_t*>(cells_v) + e0);
            float4* r4 = reinterpret_cast<float4*>(static_cast<float*>(cells_v) + P.c + e0);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const float4 y = __ldcs(y4 + q);
                r4[q] = y;
                k4[q] = make_uint4((uint32_t)acc[4 * q], (uint32_t)acc[4 * q + 1], (uint32_t)acc[4 * q + 2],
                                   (uint32_t)acc[4 * q + 3]);
#pragma unroll
                for (int e = 0; e < 4; e++)
                    if ((m1 >> (4 * q + e)) & 1u)
                        frontier[fpos++] = make_uint2((uint32_t)(e0 + 4 * q + e),
                                                      ((uint32_t)acc[4 * q + e] & 0xffffffu) | (j << 24));
            }
        } else if (lane < nw) {
            const uint64_t e0 = (D << P.log2L) + 32 * lane;
            const float4* y4 = reinterpret_cast<const float4*>(counters + e0);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const float4 y = __ldcs(y4 + q);
                const float yv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    if ((m1 >> (4 * q + e)) & 1u)
                        frontier[fpos++] = make_uint2((uint32_t)(e0 + 4 * q + e),
                                                      COMPACT ? ((uint32_t)acc[4 * q + e] & 0xffffffu) | (j << 24)
                                                              : (uint32_t)acc[4 * q + e]);
                    if (COMPACT) {
                        CellC st;
                        st.key = (uint32_t)acc[4 * q + e];
                        st.R = yv[e];
                        static_cast<CellC*>(cells_v)[e0 + 4 * q + e] = st;
                    } else {
                        CellState st;
                        st.key = acc[4 * q + e];
                        st.R = yv[e];
                        st.pad = 0u;
                        static_cast<CellState*>(cells_v)[e0 + 4 * q + e] = st;
                    }
                }
            }
        }
    }
}

// (input row, probe) pairs counting-sorted by destination row: dst_off[nD + 1]
// offsets, dst_list the input rows (in an atomic order within a row)
void launch_pair_lists(const KParams& P, const uint2* tabS, uint32_t* dst_off, uint32_t* pair_pos,
                       uint32_t* dst_list, cudaStream_t s) {
    const uint64_t npairs = (uint64_t)P.nrows * P.k;
    const uint64_t nD = P.c >> P.log2L;
    const uint32_t gp = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((npairs + 255) / 256, (uint64_t)num_sms() * 8));
    cudaMemsetAsync(dst_off, 0, (nD + 1) * sizeof(uint32_t), s);
    k_pair_count<<<gp, 256, 0, s>>>(P, tabS, dst_off, pair_pos);
    k_pair_scan<<<1, 1024, 0, s>>>(dst_off, (uint32_t)nD + 1);
    k_pair_scatter<<<gp, 256, 0, s>>>(P, tabS, dst_off, pair_pos, dst_list);
    count_launch(3);
}

void launch_build_cells(const KParams& P, const float* counters, const uint2* tabS,
                        const uint32_t* gmask, uint32_t* dst_off, uint32_t* pair_pos,
                        uint32_t* dst_list, void* cells, Ctrl* ctrl, bool compact,
                        uint2* frontier, bool split, cudaStream_t s) {
    const uint64_t nD = P.c >> P.log2L;
#ifdef LHC_DEBUG_SYNC
#define DBG(name) { cudaError_t e_ = cudaStreamSynchronize(s); if (e_) fprintf(stderr, "%s: %s\n", name, cudaGetErrorString(e_)); else fprintf(stderr, "%s ok\n", name); }
#else
#define DBG(name)
#endif
    launch_pair_lists(P, tabS, dst_off, pair_pos, dst_list, s);
    DBG("pair_lists");
    const uint32_t gb = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((nD + 7) / 8, (uint64_t)num_sms() * 16));
    if (compact && split)
        k_build_cells<true, true><<<gb, 256, 0, s>>>(P, counters, tabS, gmask, dst_off, dst_list, cells,
                                                     ctrl, frontier);
    else if (compact)
        k_build_cells<true, false><<<gb, 256, 0, s>>>(P, counters, tabS, gmask, dst_off, dst_list, cells,
                                                      ctrl, frontier);
    else
        k_build_cells<false, false><<<gb, 256, 0, s>>>(P, counters, tabS, gmask, dst_off, dst_list, cells,
                                                       ctrl, frontier);
    DBG("build_cells");
    count_launch(1);
}

// KT: compile-time k (3) or 0 for a run-time k <= kMaxK.
// The two decode-state layouts: 16-byte cells keyed by coordinate (2^32 + p) and
// 8-byte cells keyed by input row (2^24 + i).  A frontier entry is (cell, id) with
// id = p (wide) or i | j << 24 (compact, j = the cell's probe).
template <bool COMPACT>
struct Cells {
    using T = typename std::conditional<COMPACT, CellC, CellState>::type;
    using K = typename std::conditional<COMPACT, uint32_t, unsigned long long>::type;
    static constexpr int kShift = COMPACT ? 24 : 32;
    __device__ static K one(uint32_t id) { return ((K)1 << kShift) + (K)id; }
    __device__ static uint32_t deg(K key) { return (uint32_t)(key >> kShift); }
    __device__ static uint32_t low(K key) { return (uint32_t)(key & (((K)1 << kShift) - 1)); }
};

// Finalize, a warp per 1024-coordinate chunk q with a 4 KB tile in shared memory
// (the queue buffer is free now): the chunk's candidates hold slots [s0, s1) of the
// list, its peeled values are log entries [s0, vfill[q]).  Unpeeled candidates take
// the median over j of sign_j * R; R of cell e is Rb[e * RS].
template <int KT, int RS>
__device__ void finalize_chunks(const KParams& P, const uint2* __restrict__ tabS,
                                const uint32_t* __restrict__ cand, float* dense, const float* Rb,
                                float* __restrict__ out_val, uint8_t* __restrict__ out_peeled,
                                uint64_t n_c, const uint32_t* __restrict__ rowoff, const uint2* vlog,
                                const uint32_t* vfill, uint2* sh_q) {
    constexpr uint32_t NJ = KT ? KT : kMaxK;
    const uint32_t k = KT ? (uint32_t)KT : P.k;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    {
        const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
        float* tile = reinterpret_cast<float*>(sh_q) + wib * (kTile + 32);
        uint32_t* pm = reinterpret_cast<uint32_t*>(tile + kTile);  // peeled bits of the chunk
        const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
        const uint32_t rsh = 10 - P.log2L;  // input rows per chunk = 2^rsh
        const uint64_t gw = gtid >> 5, nwarps = gstride >> 5;
        // the next chunk's bounds are loaded while this one is assembled; the first
        // 128 log entries and 128 candidate slots of a chunk are loaded together
        uint32_t n_s0 = 0, n_s1 = 0, n_f1 = 0;
        if (gw < nchunks) {
            n_s0 = __ldcg(rowoff + (gw << rsh));
            n_s1 = gw + 1 < nchunks ? __ldcg(rowoff + ((gw + 1) << rsh)) : (uint32_t)n_c;
            n_f1 = __ldcg(vfill + gw);
        }
        for (uint64_t q = gw; q < nchunks; q += nwarps) {
            const uint32_t s0 = n_s0, s1 = n_s1, f1 = n_f1;
            const uint64_t qn = q + nwarps;
            if (qn < nchunks) {
                n_s0 = __ldcg(rowoff + (qn << rsh));
                n_s1 = qn + 1 < nchunks ? __ldcg(rowoff + ((qn + 1) << rsh)) : (uint32_t)n_c;
                n_f1 = __ldcg(vfill + qn);
            }
            uint2 ent[4];
            uint32_t pc[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t a = s0 + lane + 32 * u;
                ent[u] = a < f1 ? __ldcs(vlog + a) : make_uint2(0u, 0u);
                pc[u] = a < s1 ? __ldg(cand + a) : 0u;
            }
            float4* t4 = reinterpret_cast<float4*>(tile);
#pragma unroll
            for (int u = 0; u < 8; u++) t4[lane + 32 * u] = make_float4(0.f, 0.f, 0.f, 0.f);
            pm[lane] = 0u;
            __syncwarp();
            for (uint32_t a0 = s0;;) {
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (a0 + lane + 32 * u < f1) {
                        const uint32_t off = ent[u].x & (kTile - 1);
                        tile[off] = __uint_as_float(ent[u].y);
                        atomicOr(pm + (off >> 5), 1u << (off & 31));
                    }
                a0 += 128;
                if (a0 >= f1) break;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const uint32_t a = a0 + lane + 32 * u;
                    ent[u] = a < f1 ? __ldcs(vlog + a) : make_uint2(0u, 0u);
                }
            }
            __syncwarp();
            for (uint32_t a0 = s0;;) {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const uint32_t sl = a0 + lane + 32 * u;
                    if (sl >= s1) continue;
                    const uint32_t p = pc[u];
                    const uint32_t off = p & (kTile - 1);
                    const bool pe = (pm[off >> 5] >> (off & 31)) & 1u;
                    float val;
                    if (pe) {
                        val = tile[off];
                    } else {
                        float v[NJ];
                        for (uint32_t j = 0; j < k; j++) {
                            uint32_t neg;
                            const uint32_t e = cand_cell(P, tabS, p, j, &neg);
                            v[j] = (neg ? -1.f : 1.f) * __ldcg(Rb + (uint64_t)e * RS);
                        }
                        for (uint32_t a = 1; a < k; a++) {  // insertion sort of <= 8 values
                            float x = v[a];
                            int b = (int)a - 1;
                            while (b >= 0 && v[b] > x) { v[b + 1] = v[b]; b--; }
                            v[b + 1] = x;
                        }
                        val = (k & 1) ? v[k / 2] : 0.5f * (v[k / 2 - 1] + v[k / 2]);
                        tile[off] = val;
                    }
                    out_peeled[sl] = pe ? 1 : 0;
                    out_val[sl] = val;
                }
                a0 += 128;
                if (a0 >= s1) break;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const uint32_t a = a0 + lane + 32 * u;
                    pc[u] = a < s1 ? __ldg(cand + a) : 0u;
                }
            }
            __syncwarp();
            if (dense) {
                const uint64_t c0 = q * kTile;
                if (c0 + kTile <= P.d) {
                    float4* o4 = reinterpret_cast<float4*>(dense + c0);
#pragma unroll
                    for (int u = 0; u < 8; u++) __stcs(o4 + lane + 32 * u, t4[lane + 32 * u]);
                } else {
                    for (uint32_t a = lane; c0 + a < P.d; a += 32) dense[c0 + a] = tile[a];
                }
            }
            __syncwarp();  // the tile is read before the next chunk clears it
        }
    }
}

// F0, the synchronous rounds and the finalize, on either layout.
template <int KT, bool COMPACT>
__device__ void peel_body(const KParams& P, const uint2* __restrict__ tabS,
                          const uint32_t* __restrict__ cand, float* dense, void* cells_v,
                          uint32_t* claim, uint2* frontier, Ctrl* ctrl, float* __restrict__ out_val,
                          uint8_t* __restrict__ out_peeled, lhc_stats* stats, uint64_t n_c,
                          const uint32_t* __restrict__ rowoff, uint2* vlog, uint32_t* vfill,
                          bool f0_done, uint2* sh_q, uint32_t* sh_n, uint32_t* sh_base,
                          uint32_t* sh_wc, uint32_t* sh_wp) {
    using C = Cells<COMPACT>;
    using Cell = typename C::T;
    using K = typename C::K;
    Cell* cells = static_cast<Cell*>(cells_v);
    cg::grid_group grid = cg::this_grid();
    constexpr uint32_t NJ = KT ? KT : kMaxK;
    const uint32_t k = KT ? (uint32_t)KT : P.k;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
    const uint64_t pl = pol_last();

    // F0 ("round 0"): cells of degree one with their candidate, through rc[0]
    // (already appended by the state build when the state was built by row)
    if (!f0_done) {
        // four cells per thread and pass (four loads in flight); one global
        // reservation per buffer-full, not per pass
        const uint32_t qcap = kPeelThreads * peel_q_per_thread(k);  // entries of sh_q
        for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < P.c; base += 4 * gstride) {
            K key[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint64_t e = base + u * gstride + threadIdx.x;
                key[u] = e < P.c ? __ldcg(&cells[e].key) : (K)0;
            }
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (C::deg(key[u]) == 1u) {
                    const uint32_t e = (uint32_t)(base + u * gstride + threadIdx.x);
                    const uint32_t id = COMPACT ? C::low(key[u]) | ((((e >> P.log2L) % (P.k * P.S_Y)) / P.S_Y) << 24)
                                                : C::low(key[u]);
                    sh_q[atomicAdd(sh_n, 1u)] = make_uint2(e, id);
                }
            __syncthreads();
            // the flush decision must be block-uniform: every thread reads the count
            // before any thread of the next pass appends (flush_queue has barriers)
            const bool flush = *sh_n + 4 * kPeelThreads > qcap || base + 4 * gstride >= P.c;
            __syncthreads();
            if (flush) flush_queue(sh_q, sh_n, sh_base, frontier, 0u, &ctrl->rc[0]);
        }
    }
    grid.sync();
    if (timer) ctrl->t[3] = globaltimer();

    uint2* wbuf = sh_q + (threadIdx.x >> 5) * kWarpQ;  // this warp's append buffer
    uint32_t wn = 0, wpeel = 0;
    uint32_t f_begin = 0;
    uint32_t f_end = (uint32_t)*(volatile unsigned long long*)&ctrl->rc[0];
    uint32_t n_peeled = 0, rounds = 0;
    for (uint32_t r = 1; f_begin < f_end; r++) {
        unsigned long long* rc = &ctrl->rc[r % 3];
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // counter of round r + 1 (last used r - 2)
            ctrl->rc[(r + 1) % 3] = 0ull;
            if (r < kCtrlTimes - 4) {
                ctrl->t[r + 3] = globaltimer();
                ctrl->fsize[r] = f_end - f_begin;
            }
        }
        for (uint64_t base = f_begin + blockIdx.x * (uint64_t)blockDim.x; base < f_end;
             base += gstride) {
            const uint64_t f = base + threadIdx.x;
            bool won = false;
            uint2 ap[NJ];  // the entries this one appends, by probe
            bool has[NJ];
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++) has[j] = false;
            if (f < f_end) {
                const uint2 ent = ld_stream(frontier + f);
                const uint32_t e = ent.x;
                // issued back to back (volatile loads are not sunk into the branch): the
                // pure cell's residual, the row maps of the candidate's input row and the
                // claim (fetch-or of the candidate's bit: a candidate can be the only one
                // left in several cells; a stale entry finds its bit already set)
                const float Re = ld_cg_f32(&cells[e].R);
                const uint32_t i = COMPACT ? (ent.y & 0xffffffu) : (ent.y >> P.log2L);
                const uint2* row = tabS + (uint64_t)i * k;
                uint2 mp[NJ];
#pragma unroll
                for (uint32_t j = 0; j < NJ; j++) {
                    if (!KT && j >= k) break;
                    mp[j] = ld_nc_u2(row + j);
                }
                uint32_t p, t;
                if (COMPACT) {  // column of the pure cell, rotated back by the row's bias
                    const uint32_t jp = ent.y >> 24;
                    uint32_t bj = 0;
#pragma unroll
                    for (uint32_t j = 0; j < NJ; j++)
                        if (j == jp) bj = map_bias(mp[j]);
                    t = ((e & (P.L - 1)) + P.L - bj) & (P.L - 1);
                    p = (i << P.log2L) + t;
                } else {
                    p = ent.y;
                    t = p & (P.L - 1);
                }
                const uint32_t bit = 1u << (p & 31);
                const uint32_t old = atomicOr(claim + (p >> 5), bit);
                if (!(old & bit)) {
                    uint32_t ev[NJ];
                    float ge = 1.f;
#pragma unroll
                    for (uint32_t j = 0; j < NJ; j++) {
                        if (!KT && j >= k) break;
                        ev[j] = (mp[j].x << P.log2L) + ((t + map_bias(mp[j])) & (P.L - 1));
                        if (ev[j] == e) ge = map_sign(mp[j]);
                    }
                    const float val = ge * Re;
                    // the value's place in its chunk's log segment: one L2-resident
                    // counter per chunk, one atomic per chunk and warp (runs of
                    // candidates peel together); the store waits behind the key atomics
                    const uint32_t q = p >> 10, lane = threadIdx.x & 31;
                    const uint32_t peers = __match_any_sync(__activemask(), q);
                    const uint32_t leader = __ffs(peers) - 1;
                    uint32_t lbase = 0;
                    if (lane == leader) lbase = atomicAdd(vfill + q, (uint32_t)__popc(peers));
                    won = true;
                    // all reductions first (independent), then the queue appends
                    const K dec = (K)0 - C::one(COMPACT ? i : p);
                    K rest[NJ];
#pragma unroll
                    for (uint32_t j = 0; j < NJ; j++) {
                        if (!KT && j >= k) break;
                        // the pure cell held only p: nothing reads its state again
                        if (ev[j] == e) continue;
                        red_add_hint(&cells[ev[j]].R, -map_sign(mp[j]) * val, pl);
                        rest[j] = atom_add_hint(&cells[ev[j]].key, dec, pl) + dec;
                    }
                    lbase = __shfl_sync(peers, lbase, leader) + __popc(peers & ((1u << lane) - 1u));
                    st_stream(vlog + lbase, make_uint2(p, __float_as_uint(val)));
#pragma unroll
                    for (uint32_t j = 0; j < NJ; j++) {
                        if (!KT && j >= k) break;
                        if (ev[j] != e && C::deg(rest[j]) == 1u) {
                            has[j] = true;
                            ap[j] = make_uint2(ev[j], COMPACT ? C::low(rest[j]) | (j << 24) : C::low(rest[j]));
                        }
                    }
                }
            }
            wpeel += __popc(__ballot_sync(0xffffffffu, won));
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++) {
                if (!KT && j >= k) break;
                wq_push(has[j], ap[j], wbuf, wn, frontier, f_end, rc);
            }
        }
        if (LHC_PEEL_TIMING && threadIdx.x == 0 && r < kCtrlTimes) atomicMax(&ctrl->tproc[r], globaltimer());
        wq_round_end(wbuf, wn, wpeel, sh_wc, sh_wp, sh_base, frontier, f_end, rc);
        grid.sync();
        const unsigned long long rcv = *(volatile unsigned long long*)rc;
        const uint32_t np = (uint32_t)(rcv >> 32);
        f_begin = f_end;
        f_end += (uint32_t)rcv;
        n_peeled += np;
        if (np) rounds++;
    }
    if (timer) ctrl->t[kCtrlTimes - 1] = globaltimer();

    finalize_chunks<KT, COMPACT ? 2 : 4>(P, tabS, cand, dense,
                                         reinterpret_cast<const float*>(cells) + (COMPACT ? 1 : 2),
                                         out_val, out_peeled, n_c, rowoff, vlog, vfill, sh_q);
    if (LHC_PEEL_TIMING && threadIdx.x == 0) atomicMax(&ctrl->t[1], globaltimer());
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        stats->n_peeled = n_peeled;
        stats->rounds = rounds;
        stats->success = (uint64_t)n_peeled == n_c ? 1 : 0;
        stats->entries = f_end;  // every entry appended was processed by a round
        ctrl->rounds_dbg = rounds;
    }
}

// Two-pass peel on the split compact state (keys[c], R[c]: 4 bytes each), used when
// the 8-byte cell state does not fit in L2.  The set of candidates peeled in each
// synchronous round depends only on the degrees, so
//   pass 1  runs the rounds on the keys alone (claim, key deductions, frontier
//           appends) and marks every entry whose claim succeeded (bit 31 of its id);
//           the end of each round's segment is kept in rend[] (<= c segments: every
//           cell enters the queue at most once and every segment is non-empty);
//   pass 2  replays the segments in order on the residuals alone: a marked entry
//           (e, i | j << 24) reads its value from its pure cell e and deducts it from
//           the other cells of its candidate, one grid barrier per segment —
//           all cells that fed a pure cell were peeled in earlier segments.
// Each pass works on half the state (VGG19: 64 MB), which then stays in L2.
template <int KT>
__device__ void peel_split(const KParams& P, const uint2* __restrict__ tabS,
                           const uint32_t* __restrict__ cand, float* dense, uint32_t* keys, float* R,
                           uint32_t* rend, uint32_t* claim, uint2* frontier, Ctrl* ctrl,
                           float* __restrict__ out_val, uint8_t* __restrict__ out_peeled,
                           lhc_stats* stats, uint64_t n_c, const uint32_t* __restrict__ rowoff,
                           uint2* vlog, uint32_t* vfill, uint2* sh_q, uint32_t* sh_wc,
                           uint32_t* sh_wp, uint32_t* sh_base) {
    using C = Cells<true>;
    cg::grid_group grid = cg::this_grid();
    constexpr uint32_t NJ = KT ? KT : kMaxK;
    const uint32_t k = KT ? (uint32_t)KT : P.k;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
    const uint64_t pl = pol_last();
    grid.sync();
    if (timer) ctrl->t[3] = globaltimer();

    // ---- pass 1: degrees only
    uint2* wbuf = sh_q + (threadIdx.x >> 5) * kWarpQ;  // this warp's append buffer
    uint32_t wn = 0, wpeel = 0;
    uint32_t f_begin = 0;
    uint32_t f_end = (uint32_t)*(volatile unsigned long long*)&ctrl->rc[0];
    uint32_t n_peeled = 0, rounds = 0, nseg = 0;
    for (uint32_t r = 1; f_begin < f_end; r++) {
        unsigned long long* rc = &ctrl->rc[r % 3];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctrl->rc[(r + 1) % 3] = 0ull;
            rend[r - 1] = f_end;  // segment r - 1 (0-based) is [rend[r - 2], rend[r - 1])
            if (r < kCtrlTimes - 4) {
                ctrl->t[r + 3] = globaltimer();
                ctrl->fsize[r] = f_end - f_begin;
            }
        }
        nseg = r;
        for (uint64_t base = f_begin + blockIdx.x * (uint64_t)blockDim.x; base < f_end; base += gstride) {
            const uint64_t f = base + threadIdx.x;
            bool won = false;
            uint2 ap[NJ];  // the entries this one appends, by probe
            bool has[NJ];
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++) has[j] = false;
            if (f < f_end) {
                const uint2 ent = ld_stream(frontier + f);
                const uint32_t e = ent.x, i = ent.y & 0xffffffu, jp = ent.y >> 24;
                const uint2* row = tabS + (uint64_t)i * k;
                uint2 mp[NJ];
#pragma unroll
                for (uint32_t j = 0; j < NJ; j++) {
                    if (!KT && j >= k) break;
                    mp[j] = ld_nc_u2(row + j);
                }
                uint32_t bj = 0;
#pragma unroll
                for (uint32_t j = 0; j < NJ; j++)
                    if (j == jp) bj = map_bias(mp[j]);
                const uint32_t t = ((e & (P.L - 1)) + P.L - bj) & (P.L - 1);
                const uint32_t p = (i << P.log2L) + t;
                const uint32_t bit = 1u << (p & 31);
                const uint32_t old = atomicOr(claim + (p >> 5), bit);
                if (!(old & bit)) {
                    won = true;
                    const uint32_t dec = 0u - C::one(i);
                    uint32_t rest[NJ];
#pragma unroll
                    for (uint32_t j = 0; j < NJ; j++) {
                        if (!KT && j >= k) break;
                        if (j == jp) continue;
                        ap[j].x = (mp[j].x << P.log2L) + ((t + map_bias(mp[j])) & (P.L - 1));
                        rest[j] = atom_add_hint(keys + ap[j].x, dec, pl) + dec;
                    }
                    st_stream(&frontier[f].y, ent.y | 0x80000000u);  // won: replayed by pass 2
#pragma unroll
                    for (uint32_t j = 0; j < NJ; j++) {
                        if (!KT && j >= k) break;
                        if (j != jp && C::deg(rest[j]) == 1u) {
                            has[j] = true;
                            ap[j].y = C::low(rest[j]) | (j << 24);
                        }
                    }
                }
            }
            wpeel += __popc(__ballot_sync(0xffffffffu, won));
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++) {
                if (!KT && j >= k) break;
                wq_push(has[j], ap[j], wbuf, wn, frontier, f_end, rc);
            }
        }
        wq_round_end(wbuf, wn, wpeel, sh_wc, sh_wp, sh_base, frontier, f_end, rc);
        grid.sync();
        const unsigned long long rcv = *(volatile unsigned long long*)rc;
        const uint32_t np = (uint32_t)(rcv >> 32);
        f_begin = f_end;
        f_end += (uint32_t)rcv;
        n_peeled += np;
        if (np) rounds++;
    }
    if (timer) ctrl->t[kCtrlTimes - 2] = globaltimer();

    // ---- pass 2: values, segment by segment (rend[] and the marks are ordered by the
    // last barrier of pass 1)
    for (uint32_t sgi = 0; sgi < nseg; sgi++) {
        const uint32_t b = sgi ? __ldcg(rend + sgi - 1) : 0u, en = __ldcg(rend + sgi);
        if (LHC_PEEL_TIMING && timer && sgi < kCtrlTimes) ctrl->tflush[sgi] = globaltimer();
        for (uint64_t f = b + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < en; f += gstride) {
            const uint2 ent = __ldcs(frontier + f);
            if (!(ent.y >> 31)) continue;
            const uint32_t e = ent.x, i = ent.y & 0xffffffu, jp = (ent.y >> 24) & 0x7fu;
            const float Re = ld_cg_f32(R + e);
            const uint2* row = tabS + (uint64_t)i * k;
            uint2 mp[NJ];
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++) {
                if (!KT && j >= k) break;
                mp[j] = ld_nc_u2(row + j);
            }
            uint32_t bj = 0;
            float ge = 1.f;
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++)
                if (j == jp) { bj = map_bias(mp[j]); ge = map_sign(mp[j]); }
            const uint32_t t = ((e & (P.L - 1)) + P.L - bj) & (P.L - 1);
            const uint32_t p = (i << P.log2L) + t;
            const float val = ge * Re;
            const uint32_t q = p >> 10, lane = threadIdx.x & 31;
            const uint32_t peers = __match_any_sync(__activemask(), q);
            const uint32_t leader = __ffs(peers) - 1;
            uint32_t lbase = 0;
            if (lane == leader) lbase = atomicAdd(vfill + q, (uint32_t)__popc(peers));
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++) {
                if (!KT && j >= k) break;
                if (j == jp) continue;
                red_add_hint(R + (mp[j].x << P.log2L) + ((t + map_bias(mp[j])) & (P.L - 1)),
                             -map_sign(mp[j]) * val, pl);
            }
            lbase = __shfl_sync(peers, lbase, leader) + __popc(peers & ((1u << lane) - 1u));
            st_stream(vlog + lbase, make_uint2(p, __float_as_uint(val)));
        }
        grid.sync();
    }
    if (timer) ctrl->t[kCtrlTimes - 1] = globaltimer();
    finalize_chunks<KT, 1>(P, tabS, cand, dense, R, out_val, out_peeled, n_c, rowoff, vlog, vfill, sh_q);
    if (LHC_PEEL_TIMING && threadIdx.x == 0) atomicMax(&ctrl->t[1], globaltimer());
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        stats->n_peeled = n_peeled;
        stats->rounds = rounds;
        stats->success = (uint64_t)n_peeled == n_c ? 1 : 0;
        stats->entries = f_end;
        ctrl->rounds_dbg = rounds;
    }
}

// KT: compile-time k (3) or 0 for a run-time k <= kMaxK.  mode: 0 = build the wide
// state here (per-candidate reductions), 1 = wide state prebuilt by destination
// row, 2 = compact state prebuilt by destination row (falls back to mode 0 if the
// build flagged a row with too many input rows), 4 = the same state split into key
// and residual arrays, peeled in two passes (peel_split; same fallback).
template <int KT>
__global__ void __launch_bounds__(kPeelThreads, KT ? LHC_PEEL_MINB : 1)
k_peel(KParams P, const float* __restrict__ counters, const uint2* __restrict__ tabS,
       const uint32_t* __restrict__ cand, float* dense, uint64_t cap, void* cells_v,
       uint32_t* claim, uint2* frontier, Ctrl* ctrl, float* __restrict__ out_val,
       uint8_t* __restrict__ out_peeled, lhc_stats* stats, const uint32_t* __restrict__ rowoff,
       uint2* vlog, uint32_t* vfill, int mode) {
    cg::grid_group grid = cg::this_grid();
    constexpr uint32_t NJ = KT ? KT : kMaxK;
    // queue buffer: kPeelThreads * peel_q_per_thread(k) entries of dynamic smem
    extern __shared__ uint2 sh_q[];
    __shared__ uint32_t sh_n, sh_base;
    __shared__ uint32_t sh_wc[32], sh_wp[32];
    const uint32_t k = KT ? (uint32_t)KT : P.k;

    const uint64_t n_c = *(volatile unsigned long long*)&ctrl->n_cand;
    if (n_c > cap) {  // overflow: nothing is peeled (stats.overflow set by the query)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            stats->n_peeled = 0;
            stats->rounds = 0;
            stats->success = 0;
            stats->entries = 0;
        }
        return;
    }
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
    if (threadIdx.x == 0) sh_n = 0;
    if (timer) ctrl->t[0] = globaltimer();
    if ((mode == 2 || mode == 4) && *(volatile uint32_t*)&ctrl->compact_fail) mode = 0;  // uniform
    if (mode == 3) {  // fallback after the blocked peel: only if a block could not be peeled
        if (!*(volatile uint32_t*)&ctrl->blk_fail) return;
        mode = 0;
    }
    __syncthreads();
    // claim bits cleared and the log segments' ends set to their chunks' first slots
    // (ordered before the rounds by the grid barriers below)
    for (uint64_t w = gtid; w < ((uint64_t)P.d + 31) / 32; w += gstride) __stcg(claim + w, 0u);
    {
        const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
        for (uint64_t q = gtid; q < nchunks; q += gstride) vfill[q] = __ldcg(rowoff + (q << (10 - P.log2L)));
    }

    if (mode == 0) {
        // (a compact build that failed may have appended to the queue: start it over;
        // nobody appends before the barriers below)
        if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->rc[0] = 0ull;
        CellState* cells = static_cast<CellState*>(cells_v);
        // cell state {key = 0, R = Y} (coalesced, 4 loads in flight per thread) ...
        uint64_t e = gtid;
        for (; e + 3 * gstride < P.c; e += 4 * gstride) {
            float y[4];
#pragma unroll
            for (int u = 0; u < 4; u++) y[u] = __ldcs(counters + e + u * gstride);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                CellState st;
                st.key = 0ull;
                st.R = y[u];
                st.pad = 0u;
                cells[e + u * gstride] = st;
            }
        }
        for (; e < P.c; e += gstride) {
            CellState st;
            st.key = 0ull;
            st.R = __ldcs(counters + e);
            st.pad = 0u;
            cells[e] = st;
        }
        grid.sync();
        // ... then every candidate p adds (2^32 + p) to the key of each of its cells
        for (uint64_t s = gtid; s < n_c; s += gstride) {
            const uint32_t p = __ldg(cand + s);
#pragma unroll
            for (uint32_t j = 0; j < NJ; j++) {
                if (!KT && j >= k) break;
                uint32_t neg;
                const uint32_t e2 = cand_cell(P, tabS, p, j, &neg);
                atomicAdd(&cells[e2].key, (1ull << 32) + p);
            }
        }
        grid.sync();
    }
    if (timer) ctrl->t[2] = globaltimer();
    if (mode == 4)
        peel_split<KT>(P, tabS, cand, dense, static_cast<uint32_t*>(cells_v),
                       static_cast<float*>(cells_v) + P.c, static_cast<uint32_t*>(cells_v) + 2 * P.c,
                       claim, frontier, ctrl, out_val, out_peeled, stats, n_c, rowoff, vlog, vfill, sh_q,
                       sh_wc, sh_wp, &sh_base);
    else if (mode == 2)
        peel_body<KT, true>(P, tabS, cand, dense, cells_v, claim, frontier, ctrl, out_val,
                            out_peeled, stats, n_c, rowoff, vlog, vfill, true, sh_q, &sh_n,
                            &sh_base, sh_wc, sh_wp);
    else
        peel_body<KT, false>(P, tabS, cand, dense, cells_v, claim, frontier, ctrl, out_val,
                             out_peeled, stats, n_c, rowoff, vlog, vfill, mode == 1, sh_q, &sh_n,
                             &sh_base, sh_wc, sh_wp);
}

constexpr uint64_t kSmallPeelCells = 1ull << 20;

// the queue buffer, reused by the finalize as one 4 KB tile (+ 128 B of bits) per warp
static size_t peel_smem(uint32_t k) {
    return std::max({(size_t)kPeelThreads * peel_q_per_thread(k) * sizeof(uint2),
                     (size_t)(kPeelThreads / 32) * (kTile + 32) * sizeof(float),
                     (size_t)(kPeelThreads / 32) * kWarpQ * sizeof(uint2)});
}

template <int KT>
static int peel_grid(int dev, uint32_t k, bool small) {
    static int cached[64][kMaxK + 1][2] = {};
    if (dev < 64 && cached[dev][k][small]) return cached[dev][k][small];
    const size_t smem = peel_smem(k);
    cudaFuncSetAttribute(k_peel<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peel<KT>, kPeelThreads, smem);
    // small decode states (a shard's): the rounds are barrier-bound and a grid
    // barrier over one CTA per SM is cheaper (NCF / 4: 162 vs 177 us)
    if (small) per_sm = 1;
    int g = std::max(1, per_sm) * num_sms();
    if (dev < 64) cached[dev][k][small] = g;
    return g;
}

cudaError_t launch_peel(const KParams& P, const float* counters, const uint2* tabS,
                        const uint32_t* cand, float* dense, uint64_t cap, void* cells,
                        uint32_t* claim, uint2* frontier, Ctrl* ctrl, float* out_val,
                        uint8_t* out_peeled, lhc_stats* stats, const uint32_t* rowoff,
                        uint2* vlog, uint32_t* vfill, int mode, cudaStream_t s) {
#ifdef LHC_DEBUG_SYNC
    if (getenv("LHC_DEBUG_SKIP_PEEL")) return cudaSuccess;
#endif
    int dev = 0;
    cudaGetDevice(&dev);
    const bool small = P.c <= kSmallPeelCells;
    KParams Pc = P;
    void* args[] = {(void*)&Pc,    (void*)&counters, (void*)&tabS,    (void*)&cand,
                    (void*)&dense, (void*)&cap,      (void*)&cells,   (void*)&claim,
                    (void*)&frontier, (void*)&ctrl,  (void*)&out_val, (void*)&out_peeled,
                    (void*)&stats, (void*)&rowoff, (void*)&vlog, (void*)&vfill, (void*)&mode};
    cudaError_t err;
    if (P.k == 3)
        err = cudaLaunchCooperativeKernel((const void*)k_peel<3>, dim3(peel_grid<3>(dev, 3, small)),
                                          dim3(kPeelThreads), args, peel_smem(3), s);
    else
        err = cudaLaunchCooperativeKernel((const void*)k_peel<0>, dim3(peel_grid<0>(dev, P.k, small)),
                                          dim3(kPeelThreads), args, peel_smem(P.k), s);
    count_launch();
    return err;
}

}  // namespace lhc
