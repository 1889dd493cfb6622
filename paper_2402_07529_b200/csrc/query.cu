// query.cu — Phase II step 1 (a parameter is a candidate iff "all the
// Bloom Filter's corresponding bits are set to one") on sm_100a: a streaming
// Bloom query over all d coordinates with an ordered stream compaction of the
// candidates.
//
// Work unit: one lane = one 32-coordinate source word; one warp = one chunk of
// 1024 coordinates; a CTA owns a contiguous range of 32-chunk tiles.  A source
// word of input row i is the AND over probes j of destination row rowB_j(i) of B
// rotated back by biasB_j(i): each lane loads word w of its row's destination row
// (128 contiguous bytes per row for L = 1024; B is L2-resident) and the rotation
// is two warp shuffles plus a funnel shift.  The row maps are hashed in-line by
// the lanes of the row (one hash per input row and probe).
//
// One cooperative kernel, one grid barrier:
//   phase 1  candidate masks of every chunk -> gmask (d/8 bytes), per-chunk counts,
//            per-CTA totals; also the Count Sketch row-map table for the peel
//   phase 2  CTA prefix = sum of the totals of the CTAs before it; chunk offsets
//            (kept in the workspace); candidates written in ascending order, one
//            coalesced store per nonzero mask word.
#include <cooperative_groups.h>

#include "launch.h"

namespace cg = cooperative_groups;

namespace lhc {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kQueryThreads = 256;  // 8 warps
constexpr int kQueryWarps = kQueryThreads / 32;
constexpr int kChunksPerWarp = 4;   // 8 warps * 4 = 32 chunks per tile
constexpr uint32_t kChunksPerTile = 32;

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t lane, uint32_t* total) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    *total = __shfl_sync(kFull, x, 31);
    return x - v;
}

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

template <int KB>
__global__ void __launch_bounds__(kQueryThreads)
k_query(KParams P, const uint32_t* __restrict__ bitmap, uint2* __restrict__ tabS,
        uint32_t* __restrict__ gmask, uint32_t* __restrict__ chunk_cnt,
        uint32_t* __restrict__ chunk_off, uint32_t* __restrict__ cta_total, uint64_t cap,
        uint32_t* __restrict__ out_idx, Ctrl* ctrl, lhc_stats* stats) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t sh_stage[kQueryWarps][kTile];
    __shared__ uint32_t sh_warp[kQueryWarps];
    __shared__ uint32_t sh_chunk[kChunksPerTile];
    __shared__ unsigned long long sh_prefix;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
    const uint64_t ntiles = (nchunks + kChunksPerTile - 1) / kChunksPerTile;
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t t_begin = blockIdx.x * per, t_end = min(ntiles, t_begin + per);

    // Count Sketch row maps for the peel (grid-stride, independent of the query)
    {
        const uint64_t n = (uint64_t)P.nrows * P.k;
        for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
             q += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t i = q / P.k;
            tabS[q] = dom_map(P, 0, (uint32_t)(q - i * P.k), i);
        }
    }

    // phase 1: masks and counts
    uint32_t my_total = 0;
    for (uint64_t tile = t_begin; tile < t_end; tile++) {
        const uint64_t c0 = tile * kChunksPerTile + warp * kChunksPerWarp;
        uint32_t m[kChunksPerWarp];
        query_chunks<KB>(P, bitmap, c0, lane, m);
#pragma unroll
        for (int it = 0; it < kChunksPerWarp; it++) {
            const uint64_t chunk = c0 + it;
            if (chunk < nchunks) {
                gmask[chunk * 32 + lane] = m[it];
                uint32_t cnt = __popc(m[it]);
                for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
                if (lane == 0) chunk_cnt[chunk] = cnt;
                my_total += cnt;
            }
        }
    }
    if (lane == 0) sh_warp[warp] = my_total;
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
        __syncthreads();
        if (threadIdx.x == 0) sh_prefix = 0;
        __syncthreads();
        if (lane == 0 && acc) atomicAdd(&sh_prefix, acc);
        __syncthreads();
    }
    unsigned long long run = sh_prefix;
    for (uint64_t tile = t_begin; tile < t_end; tile++) {
        // chunk offsets of the tile
        if (warp == 0) {
            const uint64_t chunk = tile * kChunksPerTile + lane;
            const uint32_t cnt = chunk < nchunks ? __ldcg(chunk_cnt + chunk) : 0u;
            uint32_t tot;
            const uint32_t ex = warp_excl_scan(cnt, lane, &tot);
            sh_chunk[lane] = ex;
            if (chunk < nchunks) chunk_off[chunk] = (uint32_t)(run + ex);  // n_c < 2^32
            if (lane == 0) sh_warp[0] = tot;
        }
        __syncthreads();
        const unsigned long long tile_base = run;
        run += sh_warp[0];
#pragma unroll 1
        for (int it = 0; it < kChunksPerWarp; it++) {
            const uint32_t cl = warp * kChunksPerWarp + it;
            const uint64_t chunk = tile * kChunksPerTile + cl;
            if (chunk >= nchunks) break;
            const uint32_t msk = __ldcg(gmask + chunk * 32 + lane);
            uint32_t tot;
            const uint32_t pre = warp_excl_scan(__popc(msk), lane, &tot);
            const unsigned long long out0 = tile_base + sh_chunk[cl];
            const uint32_t chunk_q0 = (uint32_t)(chunk * kTile);
            const uint32_t nz = __ballot_sync(kFull, msk != 0);
            uint32_t maxpop = __popc(msk);
            for (int o = 16; o; o >>= 1) maxpop = max(maxpop, __shfl_xor_sync(kFull, maxpop, o));
            if ((uint32_t)__popc(nz) <= maxpop) {
                // few, dense words: one coalesced store per nonzero word (its
                // candidates are consecutive slots)
                const uint32_t lt = (1u << lane) - 1u;
                for (uint32_t z = nz; z; z &= z - 1) {
                    const uint32_t w = __ffs(z) - 1;
                    const uint32_t mw = __shfl_sync(kFull, msk, w);
                    const uint32_t pw = __shfl_sync(kFull, pre, w);
                    if (mw & (1u << lane)) {
                        const unsigned long long pos = out0 + pw + __popc(mw & lt);
                        if (pos < cap) out_idx[pos] = chunk_q0 + 32 * w + lane;
                    }
                }
            } else {
                // many sparse words: each lane stages its word's candidates in shared
                // memory (max-popcount iterations), then a coalesced copy
                uint32_t pos = pre;
                for (uint32_t mm = msk; mm; mm &= mm - 1)
                    sh_stage[warp][pos++] = chunk_q0 + 32 * lane + (__ffs(mm) - 1);
                __syncwarp();
                for (uint32_t a = lane; a < tot; a += 32)
                    if (out0 + a < cap) out_idx[out0 + a] = sh_stage[warp][a];
                __syncwarp();
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const unsigned long long total = run;
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
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query<KB>, kQueryThreads, 0);
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
                         uint32_t* chunk_cnt, uint32_t* chunk_off, uint32_t* cta_total,
                         uint64_t cap, uint32_t* out_idx, Ctrl* ctrl, lhc_stats* stats,
                         cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    KParams Pc = P;
    void* args[] = {(void*)&Pc,        (void*)&bitmap,    (void*)&tabS,      (void*)&gmask,
                    (void*)&chunk_cnt, (void*)&chunk_off, (void*)&cta_total, (void*)&cap,
                    (void*)&out_idx,   (void*)&ctrl,      (void*)&stats};
    cudaError_t e = P.kb == 3
        ? cudaLaunchCooperativeKernel((const void*)k_query<3>, dim3(query_grid<3>(dev)),
                                      dim3(kQueryThreads), args, 0, s)
        : cudaLaunchCooperativeKernel((const void*)k_query<0>, dim3(query_grid<0>(dev)),
                                      dim3(kQueryThreads), args, 0, s);
    count_launch();
    return e;
}

}  // namespace lhc
