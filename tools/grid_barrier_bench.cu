// tools/grid_barrier_bench.cu — cost of a grid-wide barrier on B200: cooperative
// groups grid.sync() vs a gpu-scope counter barrier, at the peel kernel's grid.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void bar_gpu(uint32_t* bar, uint32_t& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        gen += gridDim.x;
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_gpu(bar) < gen) {}
    }
    __syncthreads();
}
__global__ void k_cg(int n, unsigned long long* t) {
    cg::grid_group g = cg::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < n; i++) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *t = clock64() - t0;
}
__global__ void k_own(int n, uint32_t* bar, unsigned long long* t) {
    uint32_t gen = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < n; i++) bar_gpu(bar, gen);
    if (blockIdx.x == 0 && threadIdx.x == 0) *t = clock64() - t0;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* bar; unsigned long long* t; cudaMalloc(&bar, 4); cudaMalloc(&t, 8);
    for (int per : {1, 2, 3, 4, 8}) {
        for (int threads : {256, 512, 1024}) {
            if (per * threads > 2048) continue;
            int grid = per * sms, n = 1000;
            void* a1[] = {&n, &t};
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, a1, 0, 0);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, a1, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms1; cudaEventElapsedTime(&ms1, e0, e1);
            cudaMemset(bar, 0, 4);
            void* a2[] = {&n, &bar, &t};
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void*)k_own, grid, threads, a2, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms2; cudaEventElapsedTime(&ms2, e0, e1);
            cudaError_t err = cudaGetLastError();
            printf("grid %5d x %4d: cg.sync %.2f us, gpu-scope counter %.2f us %s\n", grid, threads,
                   ms1 * 1e3 / n, ms2 * 1e3 / n, err ? cudaGetErrorString(err) : "");
        }
    }
}
