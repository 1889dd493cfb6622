// Probe: can this box create an NVLS multicast object, export it as a FABRIC
// handle, import it again, bind device memory and run multimem instructions?
// (single process, all visible GPUs).  Build: nvcc -o nvls_probe nvls_probe.cu -lcuda
#include <cstdio>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
    printf("%s failed: %d %s\n", #x, (int)r_, s_); return 1; } } while (0)

__global__ void mm_test(float* mc, float* out) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc) : "memory");
    out[0] = a; out[1] = b; out[2] = c; out[3] = d;
    unsigned o;
    asm volatile("multimem.ld_reduce.weak.global.or.b32 %0, [%1];" : "=r"(o) : "l"(mc + 4) : "memory");
    out[4] = __uint_as_float(o);
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 8), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

int main() {
    CK(cuInit(0));
    int n = 0;
    cudaGetDeviceCount(&n);
    printf("devices %d\n", n);
    CUmulticastObjectProp prop = {};
    prop.numDevices = n;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    prop.size = 2 << 20;
    CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    printf("mc granularity %zu\n", gran);
    prop.size = ((2 << 20) + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle mc;
    CK(cuMulticastCreate(&mc, &prop));
    int fd = -1;
    CK(cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    CUmemGenericAllocationHandle mc2;
    CK(cuMemImportFromShareableHandle(&mc2, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    printf("posix fd export/import ok (fd %d)\n", fd);
    for (int dv = 0; dv < n; dv++) CK(cuMulticastAddDevice(mc, dv));
    CUdeviceptr mcva[8], uva[8];
    for (int dv = 0; dv < n; dv++) {
        cudaSetDevice(dv);
        CUmemAllocationProp ap = {};
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = dv;
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        size_t ag = 0;
        CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
        CUmemGenericAllocationHandle mem;
        CK(cuMemCreate(&mem, prop.size, &ap, 0));
        CK(cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0));
        CK(cuMemAddressReserve(&uva[dv], prop.size, 0, 0, 0));
        CK(cuMemMap(uva[dv], prop.size, 0, mem, 0));
        CUmemAccessDesc acc = {};
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = dv;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CK(cuMemSetAccess(uva[dv], prop.size, &acc, 1));
        CK(cuMemAddressReserve(&mcva[dv], prop.size, 0, 0, 0));
        CK(cuMemMap(mcva[dv], prop.size, 0, mc, 0));
        CK(cuMemSetAccess(mcva[dv], prop.size, &acc, 1));
        float h[8] = {1.f + dv, 2.f, 3.f, 4.f, 0, 0, 0, 0};
        unsigned bits = 1u << dv;
        memcpy(&h[4], &bits, 4);
        cudaMemcpy((void*)uva[dv], h, sizeof(h), cudaMemcpyHostToDevice);
    }
    printf("bind/map ok\n");
    cudaSetDevice(0);
    float* out;
    cudaMalloc(&out, 64);
    cudaDeviceSynchronize();
    mm_test<<<1, 1>>>((float*)mcva[0], out);
    cudaError_t e = cudaDeviceSynchronize();
    float h[8];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    unsigned o;
    memcpy(&o, &h[4], 4);
    printf("kernel %s: sum %.1f %.1f %.1f %.1f  or 0x%x\n", cudaGetErrorString(e), h[0], h[1], h[2], h[3], o);
    for (int dv = 0; dv < n; dv++) {
        cudaSetDevice(dv);
        float g[12];
        cudaMemcpy(g, (void*)uva[dv], sizeof(g), cudaMemcpyDeviceToHost);
        printf("dev %d copy of the multimem.st: %.1f %.1f %.1f %.1f\n", dv, g[8], g[9], g[10], g[11]);
    }
    return 0;
}
