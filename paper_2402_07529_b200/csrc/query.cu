// query.cu — Phase II step 1 (a parameter is a candidate iff "all the
// Bloom Filter's corresponding bits are set to one") on sm_100a: a streaming
// Bloom query over all d coordinates with an ordered stream compaction of the
// candidates.
//
// Work unit: one lane = one 32-coordinate source word; one warp = one chunk of
// 1024 coordinates; a CTA owns a contiguous range of chunks.  A source
// word of input row i is the AND over probes j of destination row rowB_j(i) of B
// rotated back by biasB_j(i): each lane loads word w of its row's destination row
// (128 contiguous bytes per row for L = 1024; B is L2-resident) and the rotation
// is two warp shuffles plus a funnel shift.  The row maps are hashed in-line by
// the lanes of the row (one hash per input row and probe).
//
// One cooperative kernel, one grid barrier:
//   phase 1  candidate masks of every chunk -> gmask (d/8 bytes) and per-CTA
//            totals; also the Count Sketch row-map table for the peel
//   phase 2  CTA prefix = sum of the totals of the CTAs before it, warp prefix =
//            + the totals of the warps before it; each warp expands its masks into
//            the ascending candidate list (below).
#include <cooperative_groups.h>

#include "launch.h"

namespace cg = cooperative_groups;

namespace lhc {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kQueryThreads = 256;  // 8 warps
constexpr int kQueryWarps = kQueryThreads / 32;
constexpr int kChunksPerWarp = 4;
constexpr uint32_t kQGroupWords = 128;  // phase-2 group: 4 words per lane, 4096 coordinates
constexpr size_t kQuerySmem = (size_t)kQueryWarps * kQGroupWords * 32 * sizeof(uint16_t);

// Candidate masks of kChunksPerWarp chunks (lane = word); all lanes must call.
// KB: compile-time number of Bloom probes (3) or 0 for a run-time k_bloom <= kMaxK.
template <int KB>
__device__ __forceinline__ void query_chunks(const KParams& P, const uint32_t* __restrict__ bitmap,
                                             uint64_t chunk0, uint32_t lane,
                                             uint32_t out[kChunksPerWarp]) {
    const uint32_t w = lane & (P.nw - 1);
    const uint32_t seg = lane & ~(P.nw - 1);
    const uint64_t nrows = P.nrows;
    constexpr uint32_t NJ = KB ? KB : kMaxK;
    const uint32_t kb = KB ? KB : P.kb;
    uint32_t dword[kChunksPerWarp][NJ];
    uint32_t bias[kChunksPerWarp][NJ];
#pragma unroll
    for (int it = 0; it < kChunksPerWarp; it++) {
        const uint64_t gw = (chunk0 + it) * 32 + lane;
        const uint64_t i = gw >> P.log2nw;
        const bool live = i < nrows;
        // row maps: lane seg + j hashes probe j of the row when the row spans >= kb lanes
        uint2 mine = make_uint2(0u, 0u);
        if (P.nw >= kb) {
            if (live && w < kb) mine = dom_map(P, 1, w, i);
        }
#pragma unroll
        for (uint32_t j = 0; j < NJ; j++) {
            if (j >= kb) break;
            uint2 mp;
            if (P.nw >= kb) {
                mp.x = __shfl_sync(kFull, mine.x, seg + j);
                mp.y = __shfl_sync(kFull, mine.y, seg + j);
            } else {
                mp = live ? dom_map(P, 1, j, i) : make_uint2(0u, 0u);
            }
            bias[it][j] = map_bias(mp);
            // every lane of a live row loads its word, even past d: the rotation
            // of the row's live words needs the whole destination row
            dword[it][j] = live ? __ldg(bitmap + (uint64_t)mp.x * P.nw + w) : 0u;
        }
    }
#pragma unroll
    for (int it = 0; it < kChunksPerWarp; it++) {
        const uint64_t gw = (chunk0 + it) * 32 + lane;
        uint32_t res = (gw >> P.log2nw) < nrows ? kFull : 0u;
#pragma unroll
        for (uint32_t j = 0; j < NJ; j++) {
            if (j >= kb) break;
            // source bit t of word w sits at destination bit (t + bias) mod L
            const uint32_t db = (32 * w + bias[it][j]) & (P.L - 1);
            const uint32_t dw = db >> 5, dh = db & 31;
            const uint32_t lo = __shfl_sync(kFull, dword[it][j], seg + dw);
            const uint32_t hi = __shfl_sync(kFull, dword[it][j], seg + ((dw + 1) & (P.nw - 1)));
            res &= dh ? (lo >> dh) | (hi << (32 - dh)) : lo;
        }
        const uint64_t q0 = gw << 5;  // clear coordinates >= d
        if (q0 >= P.d) res = 0u;
        else if (q0 + 32 > P.d) res &= (1u << (uint32_t)(P.d - q0)) - 1u;
        out[it] = res;
    }
}

// L = 1024 (one input row per chunk): masks of 8 chunks at once; the 8 * KB row
// maps are hashed by 8 * KB lanes in parallel and each lane's 8 * KB destination
// words are loaded back to back.  The rotation by bias = 32 b5 + dh: source word w
// is destination words w + b5 and w + b5 + 1 (shuffle indices wrap mod 32) funnel-
// shifted by dh.  FULL: all 8 chunks lie below d (no bound checks).
template <int KB, bool FULL>
__device__ __forceinline__ void query_chunks8_onerow(const KParams& P,
                                                     const uint32_t* __restrict__ bitmap,
                                                     uint64_t chunk0, uint64_t chunk_end,
                                                     uint32_t lane, uint32_t out[8]) {
    uint2 mine = make_uint2(0u, 0u);
    if (lane < 8 * KB) {
        const uint32_t cb = lane / KB, j = lane - cb * KB;
        if (FULL || chunk0 + cb < chunk_end) mine = dom_map(P, 1, j, chunk0 + cb);
    }
    uint32_t dword[8][KB], rot[8][KB];
#pragma unroll
    for (int cb = 0; cb < 8; cb++) {
#pragma unroll
        for (int j = 0; j < KB; j++) {
            const uint32_t rx = __shfl_sync(kFull, mine.x, cb * KB + j);
            // bias < L = 1024 in the low bits, the sign in bit 31: bits 5..9 are b5,
            // bits 0..4 dh (the funnel shift and the shuffle index use only those)
            rot[cb][j] = __shfl_sync(kFull, mine.y, cb * KB + j);
            dword[cb][j] = (FULL || chunk0 + cb < chunk_end) ? __ldg(bitmap + (uint64_t)rx * 32 + lane) : 0u;
        }
    }
#pragma unroll
    for (int cb = 0; cb < 8; cb++) {
        uint32_t res = (FULL || chunk0 + cb < chunk_end) ? kFull : 0u;
#pragma unroll
        for (int j = 0; j < KB; j++) {
            const uint32_t src = lane + (rot[cb][j] >> 5);
            const uint32_t lo = __shfl_sync(kFull, dword[cb][j], src);
            const uint32_t hi = __shfl_sync(kFull, dword[cb][j], src + 1);
            res &= __funnelshift_r(lo, hi, rot[cb][j]);
        }
        if (!FULL) {
            const uint64_t q0 = ((chunk0 + cb) * 32 + lane) << 5;  // clear coordinates >= d
            if (q0 >= P.d) res = 0u;
            else if (q0 + 32 > P.d) res &= (1u << (uint32_t)(P.d - q0)) - 1u;
        }
        out[cb] = res;
    }
}

// Each warp owns a contiguous sub-range of its CTA's chunks.  Phase 1 works on
// chunks (lane = word) and records the warp's candidate total; phase 2 walks the
// same sub-range in groups of 128 words (4096 coordinates; lane = four
// consecutive words, one 16-byte load): one warp scan of the lanes' popcounts
// gives every lane its first slot, the words' candidates are written (as 12-bit
// offsets in the group) into a warp-private shared-memory buffer — per word slot
// lane-serially or warp-cooperatively, whichever takes fewer steps — and the
// group's candidates leave in ascending order with coalesced stores.  (ncu: the
// kernel is issue-bound, so phase 2 pays one scan, one pair of warp barriers and
// one copy loop per group instead of per 32 words.)
#ifndef LHC_QUERY_MINB
#define LHC_QUERY_MINB 3
#endif
template <int KB>
__global__ void __launch_bounds__(kQueryThreads, LHC_QUERY_MINB)
k_query(KParams P, const uint32_t* __restrict__ bitmap, uint2* __restrict__ tabS,
        uint32_t* __restrict__ gmask, uint32_t* __restrict__ cta_total, uint64_t cap,
        uint32_t* __restrict__ out_idx, Ctrl* ctrl, lhc_stats* stats, uint32_t* __restrict__ rowoff) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t sh_warp[kQueryWarps];
    __shared__ unsigned long long sh_prefix;
    extern __shared__ uint16_t sh_buf[];  // per warp: one group's candidates (offsets in the group)
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
    const uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;  // chunks per CTA
    const uint64_t c_begin = min(nchunks, blockIdx.x * per), c_end = min(nchunks, c_begin + per);
    const uint64_t wper = (c_end - c_begin + kQueryWarps - 1) / kQueryWarps;  // chunks per warp
    const uint64_t wc_begin = min(c_end, c_begin + warp * wper), wc_end = min(c_end, wc_begin + wper);

    // Count Sketch row maps for the peel (grid-stride, independent of the query)
    {
        const uint64_t n = (uint64_t)P.nrows * P.k;
        for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
             q += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t i = q / P.k;
            tabS[q] = dom_map(P, 0, (uint32_t)(q - i * P.k), i);
        }
    }

    // phase 1: masks of this warp's chunks
    uint32_t my_cnt = 0;
    if (KB != 0 && P.L == 1024) {
        for (uint64_t c0 = wc_begin; c0 < wc_end; c0 += 8) {
            uint32_t m[8];
            if (c0 + 8 <= wc_end && (c0 + 8) * kTile <= (uint64_t)P.d)
                query_chunks8_onerow<KB ? KB : 1, true>(P, bitmap, c0, wc_end, lane, m);
            else
                query_chunks8_onerow<KB ? KB : 1, false>(P, bitmap, c0, wc_end, lane, m);
#pragma unroll
            for (int cb = 0; cb < 8; cb++)
                if (c0 + cb < wc_end) {
                    gmask[(c0 + cb) * 32 + lane] = m[cb];
                    my_cnt += __popc(m[cb]);
                }
        }
    } else {
        for (uint64_t c0 = wc_begin; c0 < wc_end; c0 += kChunksPerWarp) {
            uint32_t m[kChunksPerWarp];
            query_chunks<KB>(P, bitmap, c0, lane, m);
#pragma unroll
            for (int it = 0; it < kChunksPerWarp; it++)
                if (c0 + it < wc_end) {
                    gmask[(c0 + it) * 32 + lane] = m[it];
                    my_cnt += __popc(m[it]);
                }
        }
    }
    for (int o = 16; o; o >>= 1) my_cnt += __shfl_xor_sync(kFull, my_cnt, o);
    if (lane == 0) sh_warp[warp] = my_cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kQueryWarps; w++) t += sh_warp[w];
        cta_total[blockIdx.x] = t;
    }
    grid.sync();

    // phase 2: this CTA's prefix over the CTAs before it
    {
        unsigned long long acc = 0;
        for (uint32_t b = threadIdx.x; b < blockIdx.x; b += blockDim.x) acc += __ldcg(cta_total + b);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (threadIdx.x == 0) sh_prefix = 0;
        __syncthreads();
        if (lane == 0 && acc) atomicAdd(&sh_prefix, acc);
        __syncthreads();
    }
    unsigned long long run = sh_prefix;
    for (uint32_t v = 0; v < warp; v++) run += sh_warp[v];
    const uint32_t lt = (1u << lane) - 1u;
    uint16_t* buf = sh_buf + warp * kQGroupWords * 32;
    const uint64_t w_begin = wc_begin * 32, w_end = wc_end * 32;
    for (uint64_t w0 = w_begin; w0 < w_end; w0 += kQGroupWords) {
        // lane owns words w0 + 4 lane .. + 3 (w_end - w0 is a multiple of 32)
        const uint64_t wl = w0 + 4 * lane;
        uint4 mv = make_uint4(0u, 0u, 0u, 0u);
        if (wl < w_end) mv = __ldcg(reinterpret_cast<const uint4*>(gmask + wl));
        const uint32_t m[4] = {mv.x, mv.y, mv.z, mv.w};
        const uint32_t c = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
        uint32_t x = c;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        const uint32_t total = __shfl_sync(kFull, x, 31);
        if (total == 0) {
            // no candidates: only the row offsets
            if (wl < w_end) {
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if (((wl + k) & (P.nw - 1)) == 0) rowoff[(wl + k) >> P.log2nw] = (uint32_t)run;
            }
            continue;
        }
        __syncwarp();  // the previous group's copy has read the buffer
        uint32_t pos = x - c;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            // word slot k of every lane: lane-serial over the word's bits (max_l popc
            // steps) or, when fewer, the whole warp one nonzero word at a time (lane =
            // bit) — runs of candidates make a few words full and the rest sparse
            if (wl < w_end && ((wl + k) & (P.nw - 1)) == 0) rowoff[(wl + k) >> P.log2nw] = (uint32_t)(run + pos);
            const uint32_t pk = __popc(m[k]);
            const uint32_t nzk = __ballot_sync(kFull, m[k] != 0u);
            const uint32_t maxk = __reduce_max_sync(kFull, pk);
            if (maxk <= (uint32_t)__popc(nzk)) {
                uint32_t q = pos;
                const uint32_t base = 128 * lane + 32 * k;  // coordinate offset in the group
                for (uint32_t mm = m[k]; mm; mm &= mm - 1, q++) buf[q] = (uint16_t)(base + (__ffs(mm) - 1));
            } else {
                for (uint32_t nz = nzk; nz; nz &= nz - 1) {
                    const uint32_t wz = __ffs(nz) - 1;
                    const uint32_t mw = __shfl_sync(kFull, m[k], wz);
                    const uint32_t off = __shfl_sync(kFull, pos, wz);
                    if ((mw >> lane) & 1u) buf[off + __popc(mw & lt)] = (uint16_t)(128 * wz + 32 * k + lane);
                }
            }
            pos += pk;
        }
        __syncwarp();
        // coalesced copy of the group's candidates to their slots
        const uint32_t g0 = (uint32_t)(w0 << 5);
        if (run + total <= cap) {
            uint32_t* o = out_idx + run;
            for (uint32_t q = lane; q < total; q += 32) o[q] = g0 + buf[q];
        } else {
            for (uint32_t q = lane; q < total; q += 32)
                if (run + q < cap) out_idx[run + q] = g0 + buf[q];
        }
        run += total;
    }
    // the last warp of the last CTA ends at the grand total
    if (blockIdx.x == gridDim.x - 1 && warp == kQueryWarps - 1 && lane == 0) {
        unsigned long long total = sh_prefix;
        for (uint32_t v = 0; v < kQueryWarps; v++) total += sh_warp[v];
        ctrl->n_cand = total;
        ctrl->overflow = total > cap ? 1u : 0u;
        stats->n_cand = total;
        stats->overflow = total > cap ? 1 : 0;
    }
}

template <int KB>
static int query_grid(int dev) {
    static int cached[64] = {0};
    if (dev < 64 && cached[dev]) return cached[dev];
    cudaFuncSetAttribute(k_query<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQuerySmem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query<KB>, kQueryThreads, kQuerySmem);
    int g = std::max(1, per_sm) * num_sms();
    if (dev < 64) cached[dev] = g;
    return g;
}

uint32_t query_max_ctas() {
    int dev = 0;
    cudaGetDevice(&dev);
    return (uint32_t)std::max(query_grid<3>(dev), query_grid<0>(dev));
}

cudaError_t launch_query(const KParams& P, const uint32_t* bitmap, uint2* tabS, uint32_t* gmask,
                         uint32_t* cta_total, uint64_t cap, uint32_t* out_idx, Ctrl* ctrl,
                         lhc_stats* stats, uint32_t* rowoff, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    KParams Pc = P;
    void* args[] = {(void*)&Pc,      (void*)&bitmap, (void*)&tabS, (void*)&gmask,
                    (void*)&cta_total, (void*)&cap,  (void*)&out_idx, (void*)&ctrl,
                    (void*)&stats, (void*)&rowoff};
    cudaError_t e = P.kb == 3
        ? cudaLaunchCooperativeKernel((const void*)k_query<3>, dim3(query_grid<3>(dev)),
                                      dim3(kQueryThreads), args, kQuerySmem, s)
        : cudaLaunchCooperativeKernel((const void*)k_query<0>, dim3(query_grid<0>(dev)),
                                      dim3(kQueryThreads), args, kQuerySmem, s);
    count_launch();
    return e;
}

}  // namespace lhc
