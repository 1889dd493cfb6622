// query.cu — Phase II step 1 ("verifying that all the Bloom Filter's
// corresponding bits are set to one") on sm_100a: a streaming Bloom query over
// all d coordinates with warp-ballot-free stream compaction of the candidates in
// ascending order, and the final densify (candidate values, exact zeros
// elsewhere).
//
// Work unit: one lane = one 32-coordinate source word; one warp = one 1024-
// coordinate chunk; one CTA (8 warps x 4 chunks) = one 32768-coordinate tile.
// A source word of input row i is the AND over probes j of the destination row
// rowB_j(i) of B rotated back by biasB_j(i): every lane loads word w of its row's
// destination row (a coalesced 128-byte row read for L = 1024, L2-resident since
// B is small) and the rotation is two warp shuffles plus a funnel shift.
#include "launch.h"

namespace lhc {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kQueryThreads = 256;           // 8 warps
constexpr int kChunksPerWarp = 4;            // 8 warps * 4 = 32 chunks per tile

// Candidate mask of global source word gw (coordinates [32 gw, 32 gw + 32)).
// All 32 lanes of the warp must call it (shuffles); lanes hold consecutive gw.
__device__ __forceinline__ uint32_t query_word(const KParams& P, const uint32_t* __restrict__ bitmap,
                                               const uint2* __restrict__ tabB, uint64_t gw,
                                               uint32_t lane) {
    // every lane of a row segment loads its destination word even past d: the
    // rotation of the row's live words needs the whole destination row
    const uint64_t i = gw >> P.log2nw;
    const bool live = i < P.nrows;
    const uint32_t w = (uint32_t)gw & (P.nw - 1);
    const uint32_t seg = lane & ~(P.nw - 1);
    uint32_t res = live ? kFull : 0u;
    for (uint32_t j = 0; j < P.kb; j++) {
        const uint2 mp = live ? __ldg(tabB + i * P.kb + j) : make_uint2(0u, 0u);
        const uint32_t dword = live ? __ldg(bitmap + (uint64_t)mp.x * P.nw + w) : 0u;
        // source bit t of word w sits at destination bit (t + bias) mod L
        const uint32_t db = (32 * w + map_bias(mp)) & (P.L - 1);
        const uint32_t dw = db >> 5, dh = db & 31;
        const uint32_t lo = __shfl_sync(kFull, dword, seg + dw);
        const uint32_t hi = __shfl_sync(kFull, dword, seg + ((dw + 1) & (P.nw - 1)));
        res &= dh ? (lo >> dh) | (hi << (32 - dh)) : lo;
    }
    const uint64_t q0 = gw << 5;  // clear coordinates >= d
    if (q0 >= P.d) res = 0u;
    else if (q0 + 32 > P.d) res &= (1u << (uint32_t)(P.d - q0)) - 1u;
    return res;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t lane, uint32_t* total) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    *total = __shfl_sync(kFull, x, 31);
    return x - v;
}

// Pass 1: candidates per tile.
__global__ void __launch_bounds__(kQueryThreads)
k_query_count(KParams P, const uint32_t* __restrict__ bitmap, const uint2* __restrict__ tabB,
              uint32_t* __restrict__ tile_cnt, uint32_t ntiles) {
    __shared__ uint32_t sh[kQueryThreads / 32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        uint32_t cnt = 0;
#pragma unroll
        for (int it = 0; it < kChunksPerWarp; it++) {
            const uint64_t chunk = (uint64_t)tile * 32 + warp * kChunksPerWarp + it;
            cnt += __popc(query_word(P, bitmap, tabB, chunk * 32 + lane, lane));
        }
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
        if (lane == 0) sh[warp] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int w = 0; w < kQueryThreads / 32; w++) t += sh[w];
            tile_cnt[tile] = t;
        }
        __syncthreads();
    }
}

// Pass 2: exclusive scan of the tile counts in one CTA; n_c and overflow.
__global__ void __launch_bounds__(1024)
k_query_scan(uint32_t* __restrict__ tile_cnt, uint32_t ntiles, uint64_t cap, Ctrl* ctrl,
             lhc_stats* stats) {
    __shared__ unsigned long long sh[32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = (ntiles + 1023) / 1024;
    const uint32_t b = tid * per, e = min(ntiles, b + per);
    unsigned long long sum = 0;
    for (uint32_t t = b; t < e; t++) sum += tile_cnt[t];
    // block exclusive scan of the per-thread sums
    unsigned long long x = sum;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(kFull, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = sh[lane];
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(kFull, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        sh[lane] = w;
    }
    __syncthreads();
    unsigned long long run = (warp ? sh[warp - 1] : 0ull) + x - sum;
    for (uint32_t t = b; t < e; t++) {
        uint32_t v = tile_cnt[t];
        tile_cnt[t] = (uint32_t)run;  // offsets < 2^32 (n_c <= d < 2^32)
        run += v;
    }
    if (tid == 1023) {
        const unsigned long long total = sh[31];
        ctrl->n_cand = total;
        ctrl->overflow = total > cap ? 1u : 0u;
        stats->n_cand = total;
        stats->overflow = total > cap ? 1 : 0;
    }
}

// Pass 3: write candidates ascending (slot = tile offset + chunk offset + lane
// prefix + rank of the bit) and the absolute offset of every chunk (densify).
__global__ void __launch_bounds__(kQueryThreads)
k_query_write(KParams P, const uint32_t* __restrict__ bitmap, const uint2* __restrict__ tabB,
              const uint32_t* __restrict__ tile_off, uint32_t* __restrict__ chunk_off,
              uint32_t ntiles, uint64_t cap, uint32_t* __restrict__ out_idx) {
    __shared__ uint32_t sh_cnt[32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        uint32_t msk[kChunksPerWarp], pre[kChunksPerWarp], tot[kChunksPerWarp];
#pragma unroll
        for (int it = 0; it < kChunksPerWarp; it++) {
            const uint64_t chunk = (uint64_t)tile * 32 + warp * kChunksPerWarp + it;
            msk[it] = query_word(P, bitmap, tabB, chunk * 32 + lane, lane);
            pre[it] = warp_excl_scan(__popc(msk[it]), lane, &tot[it]);
        }
        if (lane < kChunksPerWarp) {
            uint32_t t = tot[0];
#pragma unroll
            for (int it = 1; it < kChunksPerWarp; it++) if (lane == (uint32_t)it) t = tot[it];
            sh_cnt[warp * kChunksPerWarp + lane] = t;
        }
        __syncthreads();
        if (warp == 0) {
            uint32_t total;
            sh_cnt[lane] = warp_excl_scan(sh_cnt[lane], lane, &total);
        }
        __syncthreads();
        const uint32_t toff = tile_off[tile];
#pragma unroll
        for (int it = 0; it < kChunksPerWarp; it++) {
            const uint64_t chunk = (uint64_t)tile * 32 + warp * kChunksPerWarp + it;
            const uint32_t coff = toff + sh_cnt[warp * kChunksPerWarp + it];
            if (lane == 0 && chunk < nchunks) chunk_off[chunk] = coff;
            uint64_t pos = (uint64_t)coff + pre[it];
            const uint32_t q0 = (uint32_t)((chunk * 32 + lane) << 5);
            for (uint32_t mm = msk[it]; mm; mm &= mm - 1, pos++)
                if (pos < cap) out_idx[pos] = q0 + (__ffs(mm) - 1);
        }
        __syncthreads();
    }
}

// Densify: out_dense[p] = out_val[slot(p)] at candidates, 0 elsewhere; 128-bit
// streaming stores, one warp per 1024-coordinate chunk.
__global__ void __launch_bounds__(256)
k_densify(KParams P, const uint32_t* __restrict__ bitmap, const uint2* __restrict__ tabB,
          const uint32_t* __restrict__ chunk_off, uint64_t cap, const float* __restrict__ out_val,
          float* __restrict__ out_dense) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t chunk = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
         chunk < nchunks; chunk += warps) {
        const uint32_t msk = query_word(P, bitmap, tabB, chunk * 32 + lane, lane);
        uint32_t tot;
        const uint32_t pre = warp_excl_scan(__popc(msk), lane, &tot);
        const uint64_t base = chunk_off[chunk];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint32_t g = lane + 32 * q;  // float4 group of the chunk
            const uint32_t w = g >> 3, sh = (g & 7) * 4;
            const uint32_t mw = __shfl_sync(kFull, msk, w);
            const uint32_t pw = __shfl_sync(kFull, pre, w);
            const uint32_t nib = (mw >> sh) & 0xfu;
            float o[4] = {0.f, 0.f, 0.f, 0.f};
            if (nib) {
                uint64_t slot = base + pw + __popc(mw & ((1u << sh) - 1u));
#pragma unroll
                for (int e = 0; e < 4; e++)
                    if (nib & (1u << e)) {
                        o[e] = slot < cap ? out_val[slot] : 0.f;
                        slot++;
                    }
            }
            const uint64_t q0 = chunk * kTile + 4 * g;
            if (q0 + 3 < P.d) {
                __stcs(reinterpret_cast<float4*>(out_dense + q0), make_float4(o[0], o[1], o[2], o[3]));
            } else {
                for (int e = 0; e < 4; e++)
                    if (q0 + e < P.d) out_dense[q0 + e] = o[e];
            }
        }
    }
}

void launch_query_count(const KParams& P, const uint32_t* bitmap, const uint2* tabB,
                        uint32_t* tile_cnt, uint32_t ntiles, cudaStream_t s) {
    uint32_t blocks = std::min<uint32_t>(ntiles, (uint32_t)num_sms() * 8);
    k_query_count<<<blocks, kQueryThreads, 0, s>>>(P, bitmap, tabB, tile_cnt, ntiles);
    count_launch();
}

void launch_query_scan(uint32_t* tile_cnt, uint32_t ntiles, uint64_t cap, Ctrl* ctrl,
                       lhc_stats* stats, cudaStream_t s) {
    k_query_scan<<<1, 1024, 0, s>>>(tile_cnt, ntiles, cap, ctrl, stats);
    count_launch();
}

void launch_query_write(const KParams& P, const uint32_t* bitmap, const uint2* tabB,
                        const uint32_t* tile_off, uint32_t* chunk_off, uint32_t ntiles,
                        uint64_t cap, uint32_t* out_idx, cudaStream_t s) {
    uint32_t blocks = std::min<uint32_t>(ntiles, (uint32_t)num_sms() * 8);
    k_query_write<<<blocks, kQueryThreads, 0, s>>>(P, bitmap, tabB, tile_off, chunk_off, ntiles,
                                                   cap, out_idx);
    count_launch();
}

void launch_densify(const KParams& P, const uint32_t* bitmap, const uint2* tabB,
                    const uint32_t* chunk_off, uint64_t cap, const float* out_val,
                    float* out_dense, cudaStream_t s) {
    const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
    uint32_t blocks = (uint32_t)std::min<uint64_t>((nchunks + 7) / 8, (uint64_t)num_sms() * 8);
    k_densify<<<blocks, 256, 0, s>>>(P, bitmap, tabB, chunk_off, cap, out_val, out_dense);
    count_launch();
}

}  // namespace lhc
