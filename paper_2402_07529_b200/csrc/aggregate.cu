// aggregate.cu — single-GPU homomorphic aggregation (Alg. 1 comment, P:L148-149:
// "Y <- sum Y and B <- OR B"): a streaming, 128-bit vectorised OR over the
// Bloom filters and fp32 sum over the Count Sketches of n_in sketches.
#include "launch.h"

namespace lhc {

constexpr int kAggMaxIn = 16;

struct AggArgs {
    const uint32_t* b[kAggMaxIn];
    const float* y[kAggMaxIn];
    int n;
    int accumulate;  // 1: also add/OR the current output (chunked n_in > kAggMaxIn)
};

__global__ void __launch_bounds__(256)
k_aggregate(AggArgs A, uint64_t n_words, uint64_t c, uint32_t* ob, float* oy) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // Bloom filters: 16-byte groups of words, scalar tail
    const uint64_t nb4 = n_words / 4;
    for (uint64_t u = tid; u < nb4; u += stride) {
        uint4 acc = A.accumulate ? reinterpret_cast<const uint4*>(ob)[u] : make_uint4(0, 0, 0, 0);
        for (int r = 0; r < A.n; r++) {
            uint4 v = __ldcs(reinterpret_cast<const uint4*>(A.b[r]) + u);
            acc.x |= v.x; acc.y |= v.y; acc.z |= v.z; acc.w |= v.w;
        }
        reinterpret_cast<uint4*>(ob)[u] = acc;
    }
    for (uint64_t w = nb4 * 4 + tid; w < n_words; w += stride) {
        uint32_t acc = A.accumulate ? ob[w] : 0u;
        for (int r = 0; r < A.n; r++) acc |= A.b[r][w];
        ob[w] = acc;
    }
    // Count Sketches (c is a multiple of k*L >= 32): summed in ascending r
    const uint64_t nc4 = c / 4;
    for (uint64_t u = tid; u < nc4; u += stride) {
        float4 acc = A.accumulate ? reinterpret_cast<const float4*>(oy)[u]
                                  : __ldcs(reinterpret_cast<const float4*>(A.y[0]) + u);
        for (int r = A.accumulate ? 0 : 1; r < A.n; r++) {
            float4 v = __ldcs(reinterpret_cast<const float4*>(A.y[r]) + u);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        reinterpret_cast<float4*>(oy)[u] = acc;
    }
}

void launch_aggregate(uint64_t n_words, uint64_t c, int n_in, const uint32_t* const* bitmaps,
                      const float* const* counters, uint32_t* out_bitmap, float* out_counters,
                      cudaStream_t s) {
    const uint64_t units = std::max<uint64_t>(n_words / 4, c / 4);
    const uint32_t blocks =
        (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((units + 255) / 256, (uint64_t)num_sms() * 8));
    for (int r0 = 0; r0 < n_in; r0 += kAggMaxIn) {
        AggArgs A{};
        A.n = std::min(kAggMaxIn, n_in - r0);
        A.accumulate = r0 > 0;
        for (int r = 0; r < A.n; r++) {
            A.b[r] = bitmaps[r0 + r];
            A.y[r] = counters[r0 + r];
        }
        k_aggregate<<<blocks, 256, 0, s>>>(A, n_words, c, out_bitmap, out_counters);
        count_launch();
    }
}

// Zero a sketch with L2 evict-last stores: the lines stay L2-resident for the
// compress reductions that follow (a cold sketch costs one random DRAM sector
// read per first touch).
// clear up to kMaxBatch sketches: blockIdx.y = sketch.  L2 policy of the zero stores
// (LHC_CLEAR_POLICY): 0 evict-last, 1 normal, 2 evict-first
#ifndef LHC_CLEAR_POLICY
#define LHC_CLEAR_POLICY 0
#endif
struct ClearBatch {
    uint4* counters[kMaxBatch];
    uint32_t* bitmap[kMaxBatch];
};
__global__ void __launch_bounds__(256) k_clear(const __grid_constant__ ClearBatch C, uint64_t na,
                                               uint64_t nb) {
    uint64_t pol;
#if LHC_CLEAR_POLICY == 0
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#elif LHC_CLEAR_POLICY == 1
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    uint4* a = C.counters[blockIdx.y];
    uint32_t* b = C.bitmap[blockIdx.y];
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t u = tid; u < na; u += stride)
        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %1, %1, %1}, %2;" ::"l"(a + u), "r"(0u),
                     "l"(pol) : "memory");
    // bitmap words: 16-byte stores when the bitmap is 16-byte aligned, then the < 4-word tail
    uint64_t head = 0;
    if ((reinterpret_cast<uintptr_t>(b) & 15) == 0) {
        head = nb & ~uint64_t(3);
        uint4* b4 = reinterpret_cast<uint4*>(b);
        for (uint64_t u = tid; u < head / 4; u += stride)
            asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %1, %1, %1}, %2;" ::"l"(b4 + u),
                         "r"(0u), "l"(pol) : "memory");
    }
    for (uint64_t u = head + tid; u < nb; u += stride)
        asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(b + u), "r"(0u), "l"(pol)
                     : "memory");
}

void launch_clear(int n, uint32_t* const* bitmaps, uint64_t n_words, float* const* counters,
                  uint64_t c, cudaStream_t s) {
    // counters: c is a multiple of 32 floats; bitmap words: 16-byte groups + tail
    for (int b0 = 0; b0 < n; b0 += kMaxBatch) {
        const int nb = std::min(kMaxBatch, n - b0);
        ClearBatch C{};
        for (int b = 0; b < nb; b++) {
            C.counters[b] = reinterpret_cast<uint4*>(counters[b0 + b]);
            C.bitmap[b] = bitmaps[b0 + b];
        }
        const uint64_t units = std::max<uint64_t>(c / 4, n_words / 4);
        const uint32_t blocks = (uint32_t)std::max<uint64_t>(
            1, std::min<uint64_t>((units + 255) / 256, (uint64_t)num_sms() * 8 / nb + 1));
        k_clear<<<dim3(blocks, nb), 256, 0, s>>>(C, c / 4, n_words);
        count_launch();
    }
}

// Demote the lines of [p, p + bytes) to the normal L2 eviction priority.  Lines
// written or reduced with evict-last hints stay in the persisting-L2 set-aside
// (lhc_l2_persist) until demoted: the compress pins the sketch, the decode demotes
// it first so that its own working set gets the whole L2.
__global__ void __launch_bounds__(256) k_l2_demote(const char* p, uint64_t lines) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < lines;
         u += (uint64_t)gridDim.x * blockDim.x)
        asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(p + u * 128) : "memory");
}

void launch_l2_demote(const void* p, size_t bytes, cudaStream_t s) {
    if (!p || !bytes) return;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(127);
    const uint64_t lines = (reinterpret_cast<uintptr_t>(p) + bytes - a0 + 127) / 128;
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((lines + 255) / 256, (uint64_t)num_sms() * 8);
    k_l2_demote<<<blocks, 256, 0, s>>>(reinterpret_cast<const char*>(a0), lines);
    count_launch();
}

}  // namespace lhc
