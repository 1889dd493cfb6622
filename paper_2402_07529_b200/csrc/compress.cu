// compress.cu — Phase I of Alg. 1 on sm_100a: hash kernel, dense and
// COO compression into the Bloom filter B and the Count Sketch Y
// in the batched, rotated layout of §3.4.
#include <cstdlib>
#include <cstring>

#include "launch.h"

namespace lhc {

// ---------------------------------------------------------------------------
// Seeded hash kernel: one thread per (input row i, probe j) of one domain.
// ---------------------------------------------------------------------------
__global__ void k_hash_rows(KParams P, uint32_t dom, uint64_t n_rows, uint2* __restrict__ out) {
    const uint32_t kk = dom == 0 ? P.k : P.kb;
    const uint64_t n = n_rows * kk;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
         q += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t i = q / kk;
        uint32_t j = (uint32_t)(q - i * kk);
        out[q] = dom_map(P, dom, j, i);
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
// Dense compression: two kernels with the same per-chunk work and different chunk
// orders — k_compress_rows (below; every input into one sketch: chunk row r of every
// input in turn, row maps hashed once per chunk row) and k_compress_dense (input
// after input; inputs into several sketches, e.g. per-worker sketches).
//
// One warp owns a chunk of 1024 consecutive coordinates at a time (1024/L input
// rows) and needs no block-level synchronisation:
//   1. the chunk (4 KB) arrives in the warp's shared-memory ring by a bulk async
//      copy (cp.async.bulk, the TMA engine, completing on an mbarrier), issued
//      kStages - 1 chunks ahead, with an L2 evict-first hint: x is read once and
//      the loads cost no registers;
//   2. lanes compute the chunk's row maps (one hash per input row and probe,
//      P:L261 "each batch shares the same index") into a warp-private slice of
//      shared memory;
//   3. word w of the chunk's nonzero mask is ballot(x[32w + lane] != 0); lane w
//      keeps word w;
//   4. Bloom filter: for probe j, lane w builds destination word w of its row's
//      destination row (the rotation by bias_j is two shuffles and a funnel
//      shift, so a row maps onto exactly one row of B) and issues one OR
//      reduction if it is nonzero — at most k_bloom*L/32 per input row;
//   5. Count Sketch: the chunk's nonzeros are compacted (coordinate, value) and
//      processed one per lane: sign_j * x is added to each of the k cells with a
//      fire-and-forget fp32 reduction at L2.
// The sketch reductions carry an L2 evict-last hint so that the streamed
// gradient does not evict the sketch lines they accumulate into.
// ---------------------------------------------------------------------------
#ifndef LHC_COMPRESS_WARPS
#define LHC_COMPRESS_WARPS 8  // input-major kernel: two 8-warp CTAs per SM
#endif
#ifndef LHC_COMPRESS_STAGES
#define LHC_COMPRESS_STAGES 2
#endif
constexpr int kCompressWarps = LHC_COMPRESS_WARPS;
constexpr int kCompressThreads = kCompressWarps * 32;
#ifndef LHC_ROWS_WARPS
#define LHC_ROWS_WARPS 12  // row-major kernel: one 12-warp CTA per SM (VGG19 934 -> 865 us vs two 8-warp CTAs)
#endif
constexpr int kRowsWarps = LHC_ROWS_WARPS;
constexpr int kRowsThreads = kRowsWarps * 32;
constexpr int kStages = LHC_COMPRESS_STAGES;
constexpr uint32_t kFullMask = 0xffffffffu;

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void red_add(float* a, float v, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void red_or(uint32_t* a, uint32_t v, uint64_t pol) {
    asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// one thread: expect `bytes` on the barrier and start the bulk copy gmem -> smem
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t pol) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// dynamic shared memory per warp: kStages chunk buffers, the compacted nonzeros'
// coordinates, the row maps, the stage barriers
__host__ __device__ constexpr size_t compress_warp_smem(uint32_t n_map) {
    return ((size_t)kStages * kTile * sizeof(float) + kTile * sizeof(uint16_t) +
            ((n_map * 8 + 15) / 16) * 16 + kStages * sizeof(uint64_t) + 127) / 128 * 128;
}

__global__ void __launch_bounds__(kCompressThreads)
k_compress_dense(KParams P, const __grid_constant__ CompressBatch B,
                 unsigned long long* __restrict__ nnz_out) {
    extern __shared__ __align__(128) unsigned char sh_all[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t kk = P.k + P.kb;
    const uint32_t n_map = (kTile >> P.log2L) * kk;  // row maps per chunk
    unsigned char* mine = sh_all + warp * compress_warp_smem(n_map);
    float* sh_x = reinterpret_cast<float*>(mine);                         // [kStages][kTile]
    uint16_t* sh_pos = reinterpret_cast<uint16_t*>(sh_x + kStages * kTile);
    uint2* sh_map = reinterpret_cast<uint2*>(sh_pos + kTile);
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sh_map) +
                                                ((n_map * 8 + 15) / 16) * 16);
    const uint64_t nchunks = B.start[B.n];  // chunks of all inputs
    const uint64_t stride = (uint64_t)gridDim.x * kCompressWarps;
    const uint64_t first = blockIdx.x * (uint64_t)kCompressWarps + warp;
#ifndef LHC_COMPRESS_POL
#define LHC_COMPRESS_POL 0
#endif
    uint64_t pol_keep, pol_stream, pol_norm;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_norm));
    pol_keep = (LHC_COMPRESS_POL & 1) ? pol_norm : policy_evict_last();
    pol_stream = (LHC_COMPRESS_POL & 2) ? pol_norm : policy_evict_first();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t my_nnz = 0;

    if (lane == 0) {
        for (int st = 0; st < kStages; st++) mbar_init(bar + st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // prologue: the first kStages - 1 chunks in flight
    // whole chunks are bulk-copied; the ragged last chunk of an input is loaded plainly
    // the chunks a warp visits increase monotonically, so the input of the chunk being
    // prefetched (pa) and of the chunk being processed (bi) only ever advance
    uint32_t pa = 0;
    uint64_t pa_start = 0, pa_next = B.n > 1 ? B.start[1] : nchunks, pa_full = B.d[0] / kTile;
    const float* pa_x = B.x[0];
    const uint32_t inter = B.interleave ? B.n : 0u;  // chunk g = row g / n of input g % n
    auto prefetch = [&](uint64_t g, uint32_t sa, bool fence) {
        if (g >= nchunks) return;
        if (inter) {
            const uint32_t b = (uint32_t)(g % inter);
            const uint64_t lc = g / inter;
            if (lc < B.d[b] / kTile) {
                if (fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk_load(sh_x + sa * kTile, B.x[b] + lc * kTile, kTile * 4, bar + sa, pol_stream);
            }
            return;
        }
        while (g >= pa_next) {
            pa++;
            pa_start = B.start[pa];
            pa_next = pa + 1 < B.n ? B.start[pa + 1] : nchunks;
            pa_full = B.d[pa] / kTile;
            pa_x = B.x[pa];
        }
        const uint64_t lc = g - pa_start;
        if (lc < pa_full) {
            if (fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(sh_x + sa * kTile, pa_x + lc * kTile, kTile * 4, bar + sa, pol_stream);
        }
    };
    if (lane == 0)
        for (int st = 0; st < kStages - 1; st++) prefetch(first + st * stride, st, false);
    uint32_t bi = 0;
    uint64_t bi_start = 0, bi_next = B.n > 1 ? B.start[1] : nchunks;
    uint32_t it = 0, phase = 0;
    for (uint64_t chunk = first; chunk < nchunks; chunk += stride, it++) {
        const uint32_t st = it % kStages;
        // refill: the stage consumed in the previous iteration takes chunk + (kStages-1) stride
        if (lane == 0) prefetch(chunk + (uint64_t)(kStages - 1) * stride, (it + kStages - 1) % kStages, true);
        uint64_t lchunk;
        if (inter) {
            bi = (uint32_t)(chunk % inter);
            lchunk = chunk / inter;
        } else {
            while (chunk >= bi_next) {
                bi++;
                bi_start = B.start[bi];
                bi_next = bi + 1 < B.n ? B.start[bi + 1] : nchunks;
            }
            lchunk = chunk - bi_start;
        }
        const uint32_t d_in = B.d[bi];
        const float* __restrict__ x = B.x[bi];
        uint32_t* __restrict__ bitmap = B.bitmap[bi];
        float* __restrict__ counters = B.counters[bi];
        const uint64_t base = lchunk * kTile;
        float* cx = sh_x + st * kTile;
        // row maps of the chunk's rows (overlap the copy)
        const uint64_t row0 = base >> P.log2L;
        for (uint32_t a = lane; a < n_map; a += 32) {
            const uint32_t r = a / kk, jj = a - r * kk;
            const uint32_t dom = jj < P.k ? 0u : 1u;
            sh_map[a] = dom_map(P, dom, dom ? jj - P.k : jj, row0 + r);
        }
        if (lchunk < (uint64_t)d_in / kTile) {
            // a stage's barrier completes one phase per bulk copy it received (ragged
            // chunks of the batch's inputs receive none): track its parity explicitly
            mbar_wait(bar + st, (phase >> st) & 1u);
            phase ^= 1u << st;
        } else {  // ragged last chunk: plain loads
            for (uint32_t a = lane; a < kTile; a += 32) cx[a] = base + a < d_in ? x[base + a] : 0.f;
        }
        __syncwarp();
        // nonzero words: lane w builds word w from its 32 values (eight 16-byte
        // shared loads, rotated by w so a quarter-warp hits distinct banks)
        uint32_t word = 0;
        {
            const float4* cw = reinterpret_cast<const float4*>(cx + 32 * lane);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const uint32_t qq = (q + lane) & 7;
                const float4 v = cw[qq];
                const uint32_t nib = (v.x != 0.f ? 1u : 0u) | (v.y != 0.f ? 2u : 0u) |
                                     (v.z != 0.f ? 4u : 0u) | (v.w != 0.f ? 8u : 0u);
                word |= nib << (4 * qq);
            }
        }
        const uint32_t nzw = __ballot_sync(kFullMask, word != 0);
        my_nnz += __popc(word);
        if (nzw) {  // uniform
            // Bloom filter, lane w = word w of the chunk
            const uint32_t r = lane >> P.log2nw, w = lane & (P.nw - 1);
            const uint32_t seg = r << P.log2nw;
            for (uint32_t j = 0; j < P.kb; j++) {
                const uint2 mp = sh_map[r * kk + P.k + j];
                const uint32_t sb = (32 * w + P.L - map_bias(mp)) & (P.L - 1);  // (32w - bias) mod L
                const uint32_t sw = sb >> 5, sh = sb & 31;
                const uint32_t lo = __shfl_sync(kFullMask, word, seg + sw);
                const uint32_t hi = __shfl_sync(kFullMask, word, seg + ((sw + 1) & (P.nw - 1)));
                const uint32_t dst = sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
                if (dst) red_or(bitmap + (uint64_t)mp.x * P.nw + w, dst, pol_keep);
            }
            // Count Sketch: sparse chunks — every lane walks its own word's bits;
            // dense chunks — compact the coordinates, then one nonzero per lane
            uint32_t maxpop = __popc(word);
            for (int o = 16; o; o >>= 1) maxpop = max(maxpop, __shfl_xor_sync(kFullMask, maxpop, o));
            if (maxpop <= 4) {
                for (uint32_t mm = word; mm; mm &= mm - 1) {
                    const uint32_t c0 = 32 * lane + (__ffs(mm) - 1);
                    const float v = cx[c0];
                    const uint32_t rr = c0 >> P.log2L, t = c0 & (P.L - 1);
                    for (uint32_t j = 0; j < P.k; j++) {
                        const uint2 mp = sh_map[rr * kk + j];
                        red_add(counters + ((uint64_t)mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1)),
                                map_sign(mp) * v, pol_keep);
                    }
                }
            } else {
                uint32_t n = 0;
                for (uint32_t z = nzw; z; z &= z - 1) {
                    const uint32_t wz = __ffs(z) - 1;
                    const uint32_t mw = __shfl_sync(kFullMask, word, wz);
                    if (mw & (1u << lane)) sh_pos[n + __popc(mw & lt)] = (uint16_t)(32 * wz + lane);
                    n += __popc(mw);
                }
                __syncwarp();
                for (uint32_t a = lane; a < n; a += 32) {
                    const uint32_t c0 = sh_pos[a];
                    const float v = cx[c0];
                    const uint32_t rr = c0 >> P.log2L, t = c0 & (P.L - 1);
                    for (uint32_t j = 0; j < P.k; j++) {
                        const uint2 mp = sh_map[rr * kk + j];
                        red_add(counters + ((uint64_t)mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1)),
                                map_sign(mp) * v, pol_keep);
                    }
                }
            }
        }
        __syncwarp();  // the stage buffer and the maps are rewritten next
    }
    if (nnz_out) {
        for (int o = 16; o; o >>= 1) my_nnz += __shfl_xor_sync(kFullMask, my_nnz, o);
        if (lane == 0 && my_nnz) atomicAdd(nnz_out, (unsigned long long)my_nnz);
    }
}

// Row-major order (the default): a warp takes chunk r of every input of the batch in
// turn (input b fastest), so the chunk's row maps — which depend only on the row
// — are hashed once for the n inputs, and the n inputs' reductions into the
// same destination rows follow each other.  KT / KBT: compile-time k and k_bloom (3),
// or 0 for run-time values.  The chunk's nonzeros are compacted (ascending
// coordinates in shared memory) before the Count Sketch reductions, one nonzero per
// lane: lane-serial over each lane's word when the words are sparse, warp-cooperative
// over the nonzero words when a few are dense.
template <int KT, int KBT>
__global__ void __launch_bounds__(kRowsThreads)
k_compress_rows(KParams P, const __grid_constant__ CompressBatch B, uint64_t nrc,
                unsigned long long* __restrict__ nnz_out) {
    extern __shared__ __align__(128) unsigned char sh_all[];
    constexpr uint32_t NK = KT ? KT : kMaxK, NKB = KBT ? KBT : kMaxK;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t k = KT ? (uint32_t)KT : P.k, kb = KBT ? (uint32_t)KBT : P.kb;
    const uint32_t kk = k + kb;
    const uint32_t n_map = (kTile >> P.log2L) * kk;  // row maps per chunk
    unsigned char* mine = sh_all + warp * compress_warp_smem(n_map);
    float* sh_x = reinterpret_cast<float*>(mine);  // [kStages][kTile]
    uint16_t* sh_pos = reinterpret_cast<uint16_t*>(sh_x + kStages * kTile);
    uint2* sh_map = reinterpret_cast<uint2*>(sh_pos + kTile);
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sh_map) +
                                                ((n_map * 8 + 15) / 16) * 16);
    const uint32_t n = B.n;
    const uint64_t stride = (uint64_t)gridDim.x * kRowsWarps;
    const uint64_t first = blockIdx.x * (uint64_t)kRowsWarps + warp;
    uint64_t pol_keep, pol_stream;
    {
        uint64_t pol_norm;
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_norm));
        pol_keep = (LHC_COMPRESS_POL & 1) ? pol_norm : policy_evict_last();
        pol_stream = (LHC_COMPRESS_POL & 2) ? pol_norm : policy_evict_first();
    }
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t my_nnz = 0;

    if (lane == 0) {
        for (int st = 0; st < kStages; st++) mbar_init(bar + st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // prefetch cursor (lane 0): unit (pr, pb) goes to the stage after the last one;
    // whole chunks are bulk-copied, a ragged last chunk is loaded plainly when used
    uint64_t pr = first;
    uint32_t pb = 0;
    auto issue = [&](uint32_t sa, bool fence) {
        if (pr < nrc && pr < B.d[pb] / kTile) {
            if (fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(sh_x + sa * kTile, B.x[pb] + pr * kTile, kTile * 4, bar + sa, pol_stream);
        }
        if (++pb == n) { pb = 0; pr += stride; }
    };
    if (lane == 0)
        for (int st = 0; st < kStages - 1; st++) issue((uint32_t)st, false);
    uint64_t cr = first;
    uint32_t cb = 0, it = 0, phase = 0;
    while (cr < nrc) {
        const uint32_t st = it % kStages;
        if (lane == 0) issue((it + kStages - 1) % kStages, true);
        if (cb == 0) {  // a new chunk row: its maps (the previous unit's readers are done)
            const uint64_t row0 = cr << (10 - P.log2L);
            for (uint32_t a = lane; a < n_map; a += 32) {
                const uint32_t r = a / kk, jj = a - r * kk;
                sh_map[a] = jj < k ? dom_map(P, 0, jj, row0 + r) : dom_map(P, 1, jj - k, row0 + r);
            }
        }
        const uint32_t d_in = B.d[cb];
        const uint64_t base = cr * kTile;
        float* cx = sh_x + st * kTile;
        const bool live = base < d_in;
        if (live) {
            if (cr < d_in / kTile) {
                mbar_wait(bar + st, (phase >> st) & 1u);
                phase ^= 1u << st;
            } else {  // ragged last chunk: plain loads
                const float* x = B.x[cb];
                for (uint32_t a = lane; a < kTile; a += 32) cx[a] = base + a < d_in ? x[base + a] : 0.f;
            }
        }
        __syncwarp();
        if (live) {
            // nonzero words: lane w builds word w from its 32 values (eight 16-byte
            // shared loads, rotated by w so a quarter-warp hits distinct banks)
            uint32_t word = 0;
            {
                const float4* cw = reinterpret_cast<const float4*>(cx + 32 * lane);
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const uint32_t qq = (q + lane) & 7;
                    const float4 v = cw[qq];
                    const uint32_t nib = (v.x != 0.f ? 1u : 0u) | (v.y != 0.f ? 2u : 0u) |
                                         (v.z != 0.f ? 4u : 0u) | (v.w != 0.f ? 8u : 0u);
                    word |= nib << (4 * qq);
                }
            }
            const uint32_t nzw = __ballot_sync(kFullMask, word != 0);
            const uint32_t pc = __popc(word);
            my_nnz += pc;
            if (nzw) {  // uniform
                uint32_t* __restrict__ bitmap = B.bitmap[cb];
                float* __restrict__ counters = B.counters[cb];
                // Bloom filter, lane w = word w of the chunk
                const uint32_t r = lane >> P.log2nw, w = lane & (P.nw - 1);
                const uint32_t seg = r << P.log2nw;
#pragma unroll
                for (uint32_t j = 0; j < NKB; j++) {
                    if (!KBT && j >= kb) break;
                    const uint2 mp = sh_map[r * kk + k + j];
                    const uint32_t sb = (32 * w + P.L - map_bias(mp)) & (P.L - 1);  // (32w - bias) mod L
                    const uint32_t sw = sb >> 5, sh = sb & 31;
                    const uint32_t lo = __shfl_sync(kFullMask, word, seg + sw);
                    const uint32_t hi = __shfl_sync(kFullMask, word, seg + ((sw + 1) & (P.nw - 1)));
                    const uint32_t dst = __funnelshift_r(lo, hi, sh);
                    if (dst) red_or(bitmap + (uint64_t)mp.x * P.nw + w, dst, pol_keep);
                }
                // compaction of the chunk's nonzero coordinates
                uint32_t total;
                if (__reduce_max_sync(kFullMask, pc) <= (uint32_t)__popc(nzw)) {
                    uint32_t x = pc;  // inclusive warp scan of the counts
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(kFullMask, x, o);
                        if (lane >= (uint32_t)o) x += y;
                    }
                    total = __shfl_sync(kFullMask, x, 31);
                    uint32_t off = x - pc;
                    for (uint32_t mm = word; mm; mm &= mm - 1) sh_pos[off++] = (uint16_t)(32 * lane + (__ffs(mm) - 1));
                } else {
                    total = 0;
                    for (uint32_t z = nzw; z; z &= z - 1) {
                        const uint32_t wz = __ffs(z) - 1;
                        const uint32_t mw = __shfl_sync(kFullMask, word, wz);
                        if (mw & (1u << lane)) sh_pos[total + __popc(mw & lt)] = (uint16_t)(32 * wz + lane);
                        total += __popc(mw);
                    }
                }
                __syncwarp();
                // Count Sketch: one nonzero per lane, sign_j * x into each of its k cells
                for (uint32_t a = lane; a < total; a += 32) {
                    const uint32_t c0 = sh_pos[a];
                    const float v = cx[c0];
                    const uint32_t rr = c0 >> P.log2L, t = c0 & (P.L - 1);
#pragma unroll
                    for (uint32_t j = 0; j < NK; j++) {
                        if (!KT && j >= k) break;
                        const uint2 mp = sh_map[rr * kk + j];
                        red_add(counters + ((uint64_t)mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1)),
                                map_sign(mp) * v, pol_keep);
                    }
                }
            }
        }
        __syncwarp();  // the stage buffer, the positions and the maps are rewritten next
        it++;
        if (++cb == n) { cb = 0; cr += stride; }
    }
    if (nnz_out) {
        for (int o = 16; o; o >>= 1) my_nnz += __shfl_xor_sync(kFullMask, my_nnz, o);
        if (lane == 0 && my_nnz) atomicAdd(nnz_out, (unsigned long long)my_nnz);
    }
}

void launch_compress_dense(const KParams& P, const CompressBatch& B, unsigned long long* nnz_out,
                           cudaStream_t s) {
    const uint64_t nchunks = B.start[B.n];
    const uint32_t n_map = (kTile >> P.log2L) * (P.k + P.kb);
    // (LHC_COMPRESS_IMPL=chunks: the input-major kernel, one chunk of one input per unit)
    static const bool env_chunks = [] {
        const char* e = getenv("LHC_COMPRESS_IMPL");
        return e && !strcmp(e, "chunks");
    }();
    bool by_chunks = env_chunks;
    const bool fast = P.k == 3 && P.kb == 3;
    // row-major order only when every input goes into the same sketch: with several
    // sketches it keeps all of them hot at once (VGG19, 8 per-worker sketches of 81 MB:
    // 1.91 ms vs 1.15 ms input-major)
    bool one_sketch = true;
    for (uint32_t b = 1; b < B.n; b++) one_sketch &= B.counters[b] == B.counters[0] && B.bitmap[b] == B.bitmap[0];
    if (!one_sketch) by_chunks = true;
    // warps per CTA: 8 for the input-major kernel, 12 for the row-major one (the
    // sharded decode's (worker, shard) batches take the input-major kernel and were
    // 15 % slower at 12)
    const int warps = by_chunks ? kCompressWarps : kRowsWarps;
    const size_t smem = warps * compress_warp_smem(n_map);
    const size_t smax = warps * compress_warp_smem(32 * 2 * kMaxK);
    const void* fn = by_chunks ? (const void*)k_compress_dense
                     : fast    ? (const void*)k_compress_rows<3, 3>
                               : (const void*)k_compress_rows<0, 0>;
    const int fi = by_chunks ? 0 : fast ? 1 : 2;
    static int per_sm[64][3][6] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int key = 10 - (int)P.log2L > 5 ? 5 : 10 - (int)P.log2L;
    if (dev < 64 && !per_sm[dev][fi][key]) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, warps * 32, smem);
        per_sm[dev][fi][key] = std::max(1, nb);
    }
    const int resident = dev < 64 ? per_sm[dev][fi][key] : 1;
    if (by_chunks) {
        const uint32_t blocks = (uint32_t)std::min<uint64_t>((nchunks + kCompressWarps - 1) / kCompressWarps,
                                                             (uint64_t)num_sms() * resident);
        k_compress_dense<<<blocks, kCompressThreads, smem, s>>>(P, B, nnz_out);
    } else {
        uint64_t nrc = 0;  // chunk rows: the longest input's chunks
        for (uint32_t b = 0; b < B.n; b++) nrc = std::max<uint64_t>(nrc, B.start[b + 1] - B.start[b]);
        const uint32_t blocks = (uint32_t)std::min<uint64_t>((nrc + kRowsWarps - 1) / kRowsWarps,
                                                             (uint64_t)num_sms() * resident);
        if (fast)
            k_compress_rows<3, 3><<<blocks, kRowsThreads, smem, s>>>(P, B, nrc, nnz_out);
        else
            k_compress_rows<0, 0><<<blocks, kRowsThreads, smem, s>>>(P, B, nrc, nnz_out);
    }
    count_launch();
}

// ---------------------------------------------------------------------------
// COO compression: one thread per listed entry; bits are merged per warp when
// lanes hit the same word (sorted indices make neighbours share rows).  An
// entry with idx >= d is skipped and counted into *bad_out (one atomic per warp).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_compress_coo(KParams P, uint64_t nnz, const uint32_t* __restrict__ idx,
               const float* __restrict__ val, uint32_t* __restrict__ bitmap,
               float* __restrict__ counters, unsigned long long* bad_out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < nnz; base += stride) {
        const uint64_t s = base + threadIdx.x;
        bool live = s < nnz;
        uint32_t p = live ? idx[s] : 0u;
        const bool bad = live && p >= P.d;
        const uint32_t nbad = __popc(__ballot_sync(0xffffffffu, bad));
        if (nbad && bad_out && (threadIdx.x & 31) == 0) atomicAdd(bad_out, (unsigned long long)nbad);
        if (bad) { live = false; p = 0u; }
        float xv = live ? val[s] : 0.f;
        const uint64_t i = p >> P.log2L;
        const uint32_t t = p & (P.L - 1);
        for (uint32_t j = 0; j < P.kb; j++) {
            const uint2 mp = dom_map(P, 1, j, i);
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
                const uint2 mp = dom_map(P, 0, j, i);
                const uint64_t e = ((uint64_t)mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1));
                atomicAdd(counters + e, map_sign(mp) * xv);
            }
        }
    }
}

void launch_compress_coo(const KParams& P, uint64_t nnz, const uint32_t* idx, const float* val,
                         uint32_t* bitmap, float* counters, unsigned long long* bad_out,
                         cudaStream_t s) {
    if (nnz == 0) return;
    uint32_t blocks = (uint32_t)std::min<uint64_t>((nnz + 255) / 256, (uint64_t)num_sms() * 8);
    k_compress_coo<<<blocks, 256, 0, s>>>(P, nnz, idx, val, bitmap, counters, bad_out);
    count_launch();
}

}  // namespace lhc
