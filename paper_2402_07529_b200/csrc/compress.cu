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
// One warp owns a chunk of 1024 consecutive coordinates at a time (1024/L input
// rows) and needs no block-level synchronisation:
//   1. eight 128-bit streaming loads per lane (the whole 4 KB chunk in flight);
//   2. lanes compute the chunk's row maps (one hash per input row and probe,
//      P:L261 "each batch shares the same index") into a warp-private slice of
//      shared memory;
//   3. the chunk's nonzero mask is assembled as 32 words, lane w holding word w
//      (8-lane OR reductions of per-lane nibbles);
//   4. Bloom filter: for probe j, lane w builds destination word w of its row's
//      destination row (the rotation by bias_j is two shuffles and a funnel
//      shift, so a row maps onto exactly one row of B) and issues one atomicOr
//      if it is nonzero — at most k_bloom*L/32 atomics per input row;
//   5. Count Sketch: each nonzero adds sign_j * x to its k cells with a
//      fire-and-forget fp32 reduction (RED.ADD.F32, performed at L2).
// ---------------------------------------------------------------------------
constexpr int kCompressThreads = 256;
constexpr int kCompressWarps = kCompressThreads / 32;
constexpr uint32_t kFullMask = 0xffffffffu;

__global__ void __launch_bounds__(kCompressThreads)
k_compress_dense(KParams P, const float* __restrict__ x, uint32_t* __restrict__ bitmap,
                 float* __restrict__ counters, unsigned long long* __restrict__ nnz_out) {
    extern __shared__ uint2 sh_map_all[];  // [warps][rows_per_chunk * (k + kb)]
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t kk = P.k + P.kb;
    const uint32_t rows = kTile >> P.log2L;  // input rows per chunk
    const uint32_t n_map = rows * kk;
    uint2* sh_map = sh_map_all + warp * n_map;
    const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
    const bool vec_ok = (P.d & 3u) == 0;
    uint32_t my_nnz = 0;

    for (uint64_t chunk = blockIdx.x * (uint64_t)kCompressWarps + warp; chunk < nchunks;
         chunk += (uint64_t)gridDim.x * kCompressWarps) {
        const uint64_t base = chunk * kTile;
        // 1. loads (lane owns float4 groups g = lane + 32 q)
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint64_t p0 = base + 4 * (lane + 32 * q);
            if (p0 + 3 < P.d && vec_ok) {
                v[q] = __ldcs(reinterpret_cast<const float4*>(x + p0));
            } else {
                v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (p0 < P.d) v[q].x = x[p0];
                if (p0 + 1 < P.d) v[q].y = x[p0 + 1];
                if (p0 + 2 < P.d) v[q].z = x[p0 + 2];
                if (p0 + 3 < P.d) v[q].w = x[p0 + 3];
            }
        }
        // 2. row maps of the chunk's rows (overlaps the loads)
        const uint64_t row0 = base >> P.log2L;
        for (uint32_t a = lane; a < n_map; a += 32) {
            const uint32_t r = a / kk, jj = a - r * kk;
            const uint32_t dom = jj < P.k ? 0u : 1u;
            sh_map[a] = row_map(P.seed, dom, dom ? jj - P.k : jj, row0 + r, dom ? P.S_B : P.S_Y, P.L);
        }
        __syncwarp();
        // 3. nonzero words: group g = lane + 32q covers coordinates 4g..4g+3, i.e. bits
        //    4*(lane%8).. of word g/8 = 4q + lane/8
        uint32_t nibs = 0, word = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint32_t nib = (v[q].x != 0.f ? 1u : 0u) | (v[q].y != 0.f ? 2u : 0u) |
                                 (v[q].z != 0.f ? 4u : 0u) | (v[q].w != 0.f ? 8u : 0u);
            nibs |= nib << (4 * q);
            uint32_t wv = nib << (4 * (lane & 7));
            wv |= __shfl_xor_sync(kFullMask, wv, 1);
            wv |= __shfl_xor_sync(kFullMask, wv, 2);
            wv |= __shfl_xor_sync(kFullMask, wv, 4);
            const uint32_t t = __shfl_sync(kFullMask, wv, 8 * (lane & 3));
            if ((lane >> 2) == (uint32_t)q) word = t;
        }
        my_nnz += __popc(nibs);
        if (!__any_sync(kFullMask, nibs != 0)) continue;
        // 4. Bloom filter, lane w = word w of the chunk
        {
            const uint32_t r = lane >> P.log2nw, w = lane & (P.nw - 1);
            const uint32_t seg = r << P.log2nw;
            for (uint32_t j = 0; j < P.kb; j++) {
                const uint2 mp = sh_map[r * kk + P.k + j];
                const uint32_t sb = (32 * w + P.L - map_bias(mp)) & (P.L - 1);  // (32w - bias) mod L
                const uint32_t sw = sb >> 5, sh = sb & 31;
                const uint32_t lo = __shfl_sync(kFullMask, word, seg + sw);
                const uint32_t hi = __shfl_sync(kFullMask, word, seg + ((sw + 1) & (P.nw - 1)));
                const uint32_t dst = sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
                if (dst) atomicOr(bitmap + (uint64_t)mp.x * P.nw + w, dst);
            }
        }
        // 5. Count Sketch
        if (nibs) {
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const uint32_t nib = (nibs >> (4 * q)) & 0xfu;
                if (!nib) continue;
                const uint32_t c0 = 4 * (lane + 32 * q);  // coordinate within the chunk
                const uint32_t r = c0 >> P.log2L, t0 = c0 & (P.L - 1);
                const float xv[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
                for (uint32_t j = 0; j < P.k; j++) {
                    const uint2 mp = sh_map[r * kk + j];
                    const float g = map_sign(mp);
                    const uint64_t rb = (uint64_t)mp.x << P.log2L;
                    const uint32_t b = map_bias(mp);
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        if (nib & (1u << e)) atomicAdd(counters + rb + ((t0 + e + b) & (P.L - 1)), g * xv[e]);
                }
            }
        }
        __syncwarp();  // sh_map is rewritten by the next chunk
    }
    if (nnz_out) {
        for (int o = 16; o; o >>= 1) my_nnz += __shfl_xor_sync(kFullMask, my_nnz, o);
        if (lane == 0 && my_nnz) atomicAdd(nnz_out, (unsigned long long)my_nnz);
    }
}

void launch_compress_dense(const KParams& P, const float* x, uint32_t* bitmap, float* counters,
                           unsigned long long* nnz_out, cudaStream_t s) {
    const uint64_t nchunks = ((uint64_t)P.d + kTile - 1) / kTile;
    const size_t smem = (size_t)kCompressWarps * (kTile >> P.log2L) * (P.k + P.kb) * sizeof(uint2);
    static int per_sm[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !per_sm[dev]) {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_compress_dense, kCompressThreads,
                                                      kCompressWarps * 32 * 2 * kMaxK * sizeof(uint2));
        per_sm[dev] = std::max(1, n);
    }
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((nchunks + kCompressWarps - 1) / kCompressWarps,
                                                         (uint64_t)num_sms() * (dev < 64 ? per_sm[dev] : 2));
    k_compress_dense<<<blocks, kCompressThreads, smem, s>>>(P, x, bitmap, counters, nnz_out);
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
