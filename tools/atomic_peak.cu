// tools/atomic_peak.cu — measures the B200 L2 atomic throughput the peel and
// compress kernels are bound by (random RED.F32 / ATOM.ADD.64 / CAS over an
// array that fits in L2 and one that does not).  Standalone: nvcc -arch=sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
template <int OP>
__global__ void k(void* buf, uint32_t mask, uint32_t iters, unsigned long long* sink) {
    uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long acc = 0;
    for (uint32_t it = 0; it < iters; it++) {
        uint32_t i = hash32(tid * 7919u + it * 104729u) & mask;
        if (OP == 0) atomicAdd(reinterpret_cast<float*>(buf) + 2 * i, 1.0f);           // RED f32
        if (OP == 1) acc += atomicAdd(reinterpret_cast<unsigned long long*>(buf) + i, 1ull);  // ATOM u64
        if (OP == 2) acc += atomicCAS(reinterpret_cast<uint32_t*>(buf) + 2 * i, 0xffffffffu, 1u);
        if (OP == 3) acc += __ldcg(reinterpret_cast<unsigned long long*>(buf) + i);   // plain random load
        if (OP == 4) atomicAdd(reinterpret_cast<unsigned long long*>(buf) + i, 1ull);  // RED u64
        if (OP == 5) atomicAdd(reinterpret_cast<uint32_t*>(buf) + 2 * i, 1u);           // RED u32
        if (OP == 6) acc += atomicAdd(reinterpret_cast<uint32_t*>(buf) + 2 * i, 1u);    // ATOM u32
    }
    if (acc == 0x123456789ull) *sink = acc;
}
int main() {
    void* buf; unsigned long long* sink;
    cudaMalloc(&buf, 1ull << 31); cudaMalloc(&sink, 8); cudaMemset(buf, 0, 1ull << 31);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"RED.F32", "ATOM.ADD.U64(ret)", "ATOM.CAS.B32(ret)", "LDG.64 random",
                           "RED.ADD.U64", "RED.ADD.U32", "ATOM.ADD.U32(ret)"};
    for (uint32_t logb : {26u, 31u}) {  // 64 MB (L2-resident) and 2 GB (HBM)
        uint32_t mask = (uint32_t)((1ull << logb) / 8 - 1);
        for (int op = 0; op < 7; op++) {
            int blocks = sms * 8, threads = 256; uint32_t iters = 64;
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            for (int rep = 0; rep < 2; rep++) {
                cudaEventRecord(a);
                if (op == 0) k<0><<<blocks, threads>>>(buf, mask, iters, sink);
                if (op == 1) k<1><<<blocks, threads>>>(buf, mask, iters, sink);
                if (op == 2) k<2><<<blocks, threads>>>(buf, mask, iters, sink);
                if (op == 3) k<3><<<blocks, threads>>>(buf, mask, iters, sink);
                if (op == 4) k<4><<<blocks, threads>>>(buf, mask, iters, sink);
                if (op == 5) k<5><<<blocks, threads>>>(buf, mask, iters, sink);
                if (op == 6) k<6><<<blocks, threads>>>(buf, mask, iters, sink);
                cudaEventRecord(b); cudaEventSynchronize(b);
            }
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters;
            printf("%-20s footprint %5llu MB: %7.1f G ops/s\n", names[op], (1ull << logb) >> 20, ops / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
