// Microbenchmark: SM-driven stores into a peer GPU's memory over NVLink (one
// process, cudaDeviceEnablePeerAccess), for sizing the communication kernels.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_store_bench p2p_store_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void store_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n, int fence) {
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t u0 = tid; u0 < n; u0 += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int a = 0; a < U; a++)
            if (u0 + a * stride < n) v[a] = __ldcs(src + u0 + a * stride);
#pragma unroll
        for (int a = 0; a < U; a++)
            if (u0 + a * stride < n) dst[u0 + a * stride] = v[a];
    }
    if (fence) __threadfence_system();
}

// TMA-style bulk copy global(local) -> smem -> global(peer), one CTA pipeline
__global__ void bulk_kernel(char* __restrict__ dst, const char* __restrict__ src, size_t bytes, int chunk) {
    extern __shared__ __align__(128) char sm[];
    const size_t per = (size_t)chunk;
    for (size_t off = (size_t)blockIdx.x * per; off < bytes; off += (size_t)gridDim.x * per) {
        const size_t nb = off + per <= bytes ? per : bytes - off;
        // load (plain, coalesced) into smem
        for (size_t i = threadIdx.x * 16; i < nb; i += blockDim.x * 16)
            *reinterpret_cast<uint4*>(sm + i) = __ldcs(reinterpret_cast<const uint4*>(src + off + i));
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(dst + off), "r"((unsigned)__cvta_generic_to_shared(sm)), "r"((unsigned)nb) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    int n_dev = 0;
    cudaGetDeviceCount(&n_dev);
    if (n_dev < 2) { printf("needs 2 GPUs\n"); return 0; }
    cudaSetDevice(1);
    const size_t maxb = 64ull << 20;
    char* peer;
    cudaMalloc(&peer, maxb);
    cudaSetDevice(0);
    cudaDeviceEnablePeerAccess(1, 0);
    char* src;
    cudaMalloc(&src, maxb);
    cudaMemset(src, 1, maxb);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t sizes[] = {9ull << 20, 18ull << 20, 64ull << 20};
    for (size_t bytes : sizes) {
        const size_t n = bytes / 16;
        for (int cps : {1, 2, 4, 8}) {
            for (int thr : {256, 512, 1024}) {
                if (cps * thr > 2048) continue;
                for (int fence : {0, 1}) {
                    const int grid = cps * sms;
                    for (int w = 0; w < 3; w++)
                        store_kernel<4><<<grid, thr>>>((uint4*)peer, (const uint4*)src, n, fence);
                    cudaEventRecord(e0);
                    for (int it = 0; it < 10; it++)
                        store_kernel<4><<<grid, thr>>>((uint4*)peer, (const uint4*)src, n, fence);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    ms /= 10;
                    printf("st.v4  %5.1f MB  %d CTA/SM x %4d thr fence %d: %7.1f us  %6.0f GB/s\n",
                           bytes / 1048576.0, cps, thr, fence, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
                }
            }
        }
        for (int chunk : {8192, 16384, 32768}) {
            for (int cps : {1, 2, 4}) {
                const int grid = cps * sms;
                cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk);
                for (int w = 0; w < 3; w++) bulk_kernel<<<grid, 256, chunk>>>(peer, src, bytes, chunk);
                cudaEventRecord(e0);
                for (int it = 0; it < 10; it++) bulk_kernel<<<grid, 256, chunk>>>(peer, src, bytes, chunk);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                ms /= 10;
                printf("bulk   %5.1f MB  chunk %5d  %d CTA/SM: %7.1f us  %6.0f GB/s\n", bytes / 1048576.0,
                       chunk, cps, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
            }
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
