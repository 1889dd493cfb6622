// compress.cu — Phase I of Alg. 1 on sm_100a: hash kernel, dense and
// COO compression into the Bloom filter B and the Count Sketch Y
// in the batched, rotated layout of §3.4.
#include "launch.h"

namespace lhc {

// ---------------------------------------------------------------------------
// Seeded hash kernel: one thread per (input row i, probe j) of one domain.
// ---------------------------------------------------------------------------
__global__ void k_hash_rows(KParams P, uint32_t dom, uint64_t n_rows, uint2* __restrict__ out) {
    const uint32_t kk = dom == 0 ? P.k : P.kb;
    const uint32_t S = dom == 0 ? P.S_Y : P.S_B;
    const uint64_t n = n_rows * kk;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
         q += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t i = q / kk;
        uint32_t j = (uint32_t)(q - i * kk);
        out[q] = row_map(P.seed, dom, j, i, S, P.L);
    }
}

void launch_hash_rows(const KParams& P, uint32_t dom, uint64_t n_rows, uint2* out,
                      cudaStream_t s) {
    const uint32_t kk = dom == 0 ? P.k : P.kb;
    uint64_t n = n_rows * kk;
    if (n == 0) return;
    uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms() * 16);
    k_hash_rows<<<blocks, 256, 0, s>>>(P, dom, n_rows, out);
    count_launch();
}

// ---------------------------------------------------------------------------
// Dense compression.
//
// One CTA of 256 threads processes a tile of 1024 consecutive coordinates per
// iteration (one 128-bit load per thread, next tile prefetched into registers);
// a tile holds 1024/L input rows.  Per tile:
//   1. threads < rows*(k+kb) compute the tile's row maps into shared memory
//      (one hash per input row and probe, "each batch shares the same
//      index");
//   2. the nonzero mask of the tile is built as 32 words with 8-lane OR
//      reductions of per-thread nibbles;
//   3. Bloom filter: thread (j, w) assembles destination word w of probe j's
//      row by a funnel shift of two source words (the rotation by bias_j, so a
//      row maps to exactly one row of B) and issues one atomicOr per nonzero
//      word — at most k_bloom*L/32 atomics per input row instead of one per bit;
//   4. Count Sketch: each nonzero adds sign_j * x to its k cells with a
//      fire-and-forget fp32 reduction (RED.ADD.F32 at L2).
// ---------------------------------------------------------------------------
constexpr int kCompressThreads = 256;

__device__ __forceinline__ float4 load_tile4(const float* __restrict__ x, uint64_t q, uint32_t d) {
    if (q + 3 < d) return __ldcs(reinterpret_cast<const float4*>(x + q));
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q < d) v.x = x[q];
    if (q + 1 < d) v.y = x[q + 1];
    if (q + 2 < d) v.z = x[q + 2];
    return v;
}

__global__ void __launch_bounds__(kCompressThreads)
k_compress_dense(KParams P, const float* __restrict__ x, uint32_t* __restrict__ bitmap,
                 float* __restrict__ counters, unsigned long long* __restrict__ nnz_out) {
    __shared__ uint2 sh_map[32 * 2 * kMaxK];
    __shared__ uint32_t sh_src[32];
    __shared__ unsigned long long sh_nnz;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ntiles = (uint32_t)((P.d + kTile - 1) / kTile);
    const uint32_t rpt_log2 = 10 - P.log2L;  // log2(rows per tile)
    const uint32_t kk = P.k + P.kb;
    const uint32_t n_map = (1u << rpt_log2) * kk;
    if (tid == 0) sh_nnz = 0;
    uint32_t my_nnz = 0;

    uint32_t tile = blockIdx.x;
    float4 v = tile < ntiles ? load_tile4(x, (uint64_t)tile * kTile + 4 * tid, P.d)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    for (; tile < ntiles; tile += gridDim.x) {
        const uint32_t next = tile + gridDim.x;
        float4 vn = make_float4(0.f, 0.f, 0.f, 0.f);
        if (next < ntiles) vn = load_tile4(x, (uint64_t)next * kTile + 4 * tid, P.d);
        const uint64_t row0 = ((uint64_t)tile * kTile) >> P.log2L;

        // 1. row maps of the tile's rows
        if (tid < n_map) {
            uint32_t r = tid / kk, jj = tid - r * kk;
            uint32_t dom = jj < P.k ? 0u : 1u;
            uint32_t j = dom ? jj - P.k : jj;
            sh_map[tid] = row_map(P.seed, dom, j, row0 + r, dom ? P.S_B : P.S_Y, P.L);
        }
        // 2. nonzero mask words (coordinate 4*tid+e of the tile = bit (4*lane+e)&31
        //    of tile word (4*tid+e)>>5 = warp*4 + lane/8)
        uint32_t nib = (v.x != 0.f ? 1u : 0u) | (v.y != 0.f ? 2u : 0u) | (v.z != 0.f ? 4u : 0u) |
                       (v.w != 0.f ? 8u : 0u);
        my_nnz += __popc(nib);
        uint32_t wv = nib << (4 * (lane & 7));
        wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
        wv |= __shfl_xor_sync(0xffffffffu, wv, 2);
        wv |= __shfl_xor_sync(0xffffffffu, wv, 4);
        if ((lane & 7) == 0) sh_src[warp * 4 + (lane >> 3)] = wv;
        __syncthreads();

        // 3. Bloom filter: thread (j = tid/32, tile word gw = tid%32)
        if (tid < 32 * P.kb) {
            const uint32_t j = tid >> 5, gw = tid & 31;
            const uint32_t r = gw >> P.log2nw, w = gw & (P.nw - 1);
            const uint2 mp = sh_map[r * kk + P.k + j];
            const uint32_t sb = (32 * w + P.L - map_bias(mp)) & (P.L - 1);  // (32w - bias) mod L
            const uint32_t sw = sb >> 5, sh = sb & 31;
            const uint32_t lo = sh_src[(r << P.log2nw) + sw];
            const uint32_t hi = sh_src[(r << P.log2nw) + ((sw + 1) & (P.nw - 1))];
            const uint32_t dst = sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
            if (dst) atomicOr(bitmap + (uint64_t)mp.x * P.nw + w, dst);
        }
        // 4. Count Sketch
        if (nib) {
            const uint32_t q = 4 * tid;
            const uint32_t r = q >> P.log2L, t0 = q & (P.L - 1);
            const float xv[4] = {v.x, v.y, v.z, v.w};
            for (uint32_t j = 0; j < P.k; j++) {
                const uint2 mp = sh_map[r * kk + j];
                const float g = map_sign(mp);
                const uint64_t base = (uint64_t)mp.x << P.log2L;
                const uint32_t b = map_bias(mp);
#pragma unroll
                for (int e = 0; e < 4; e++)
                    if (nib & (1u << e))
                        atomicAdd(counters + base + ((t0 + e + b) & (P.L - 1)), g * xv[e]);
            }
        }
        __syncthreads();
        v = vn;
    }
    if (nnz_out) {
        for (int o = 16; o; o >>= 1) my_nnz += __shfl_xor_sync(0xffffffffu, my_nnz, o);
        if (lane == 0 && my_nnz) atomicAdd(&sh_nnz, (unsigned long long)my_nnz);
        __syncthreads();
        if (tid == 0 && sh_nnz) atomicAdd(nnz_out, sh_nnz);
    }
}

void launch_compress_dense(const KParams& P, const float* x, uint32_t* bitmap, float* counters,
                           unsigned long long* nnz_out, cudaStream_t s) {
    uint32_t ntiles = (uint32_t)((P.d + kTile - 1) / kTile);
    uint32_t blocks = std::min<uint32_t>(ntiles, (uint32_t)num_sms() * 8);
    k_compress_dense<<<blocks, kCompressThreads, 0, s>>>(P, x, bitmap, counters, nnz_out);
    count_launch();
}

// ---------------------------------------------------------------------------
// COO compression: one thread per listed entry; bits are merged per warp when
// lanes hit the same word (sorted indices make neighbours share rows).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_compress_coo(KParams P, uint64_t nnz, const uint32_t* __restrict__ idx,
               const float* __restrict__ val, uint32_t* __restrict__ bitmap,
               float* __restrict__ counters) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < nnz; base += stride) {
        const uint64_t s = base + threadIdx.x;
        const bool live = s < nnz;
        uint32_t p = live ? idx[s] : 0u;
        float xv = live ? val[s] : 0.f;
        const uint64_t i = p >> P.log2L;
        const uint32_t t = p & (P.L - 1);
        for (uint32_t j = 0; j < P.kb; j++) {
            const uint2 mp = row_map(P.seed, 1, j, i, P.S_B, P.L);
            const uint64_t b = ((uint64_t)mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1));
            const uint64_t word = b >> 5;
            uint32_t bits = live ? (1u << (b & 31)) : 0u;
            // merge lanes that target the same word: one atomicOr per distinct word
            const uint32_t peers = __match_any_sync(0xffffffffu, live ? word : ~0ull);
            const uint32_t leader = __ffs(peers) - 1;
            const uint32_t acc = __reduce_or_sync(peers, bits);
            if (live && (threadIdx.x & 31) == leader) atomicOr(bitmap + word, acc);
        }
        if (live) {
            for (uint32_t j = 0; j < P.k; j++) {
                const uint2 mp = row_map(P.seed, 0, j, i, P.S_Y, P.L);
                const uint64_t e = ((uint64_t)mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1));
                atomicAdd(counters + e, map_sign(mp) * xv);
            }
        }
    }
}

void launch_compress_coo(const KParams& P, uint64_t nnz, const uint32_t* idx, const float* val,
                         uint32_t* bitmap, float* counters, cudaStream_t s) {
    if (nnz == 0) return;
    uint32_t blocks = (uint32_t)std::min<uint64_t>((nnz + 255) / 256, (uint64_t)num_sms() * 8);
    k_compress_coo<<<blocks, 256, 0, s>>>(P, nnz, idx, val, bitmap, counters);
    count_launch();
}

}  // namespace lhc
