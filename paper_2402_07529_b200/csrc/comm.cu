// comm.cu — multi-GPU homomorphic aggregation (Alg. 1 comment, P:L148-149:
// "the API makes ... Y <- sum Y and B <- OR B") as a hand-written NVLink P2P
// all-reduce with mixed operators over CUDA-IPC-mapped peer buffers.
//
// Buffer of every rank: [bitmap (m/8 bytes, padded to 16) | counters (4c) | signals].
// One cooperative kernel per call, two-shot:
//   barrier A      every rank's compress has finished writing its buffer
//   reduce-scatter rank r owns 1/G of each region; it loads that slice from all G
//                  buffers over NVLink (128-bit loads), ORs the bitmap words /
//                  sums the counters in ascending rank order, stores locally
//   barrier B      every slice is reduced
//   all-gather     rank r copies the G-1 other reduced slices from their owners
//   barrier C      nobody reads our buffer any more (the caller may reuse it)
// Barriers: block 0 publishes the epoch to every peer's signal slot with a
// system-scope release store and spins on its own slots with acquire loads; the
// rest of the grid waits at a grid-wide barrier.  The epoch counter is kept on
// the device, so the call is CUDA-graph capturable and replayable.  Bytes per rank and direction:
// 2(G-1)/G * S.
#include <cooperative_groups.h>
#include <cuda.h>

#include <cstring>

#include "launch.h"

namespace cg = cooperative_groups;

namespace lhc {

constexpr int kMaxRanks = 8;
constexpr size_t kSignalBytes = 256;

struct ArArgs {
    const uint4* b[kMaxRanks];  // bitmap region of every rank (own one included)
    const float4* y[kMaxRanks]; // counter region of every rank
    uint32_t* sig[kMaxRanks];   // signal slots of every rank
    uint4* my_b;
    float4* my_y;
    uint64_t nb4, nc4;          // 16-byte units per region
    int rank, world;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Cross-rank barrier, executed by block 0 only (the grid syncs around it).
__device__ void xrank_barrier(const ArArgs& A, uint32_t epoch) {
    const int t = threadIdx.x;
    if (t < A.world && t != A.rank) {
        __threadfence_system();
        st_release_sys(A.sig[t] + A.rank, epoch);
    }
    if (t < A.world && t != A.rank) {
        const uint32_t* mine = A.sig[A.rank] + t;
        while ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void slice(uint64_t n, int q, int world, uint64_t* lo, uint64_t* hi) {
    *lo = n * q / world;
    *hi = n * (q + 1) / world;
}

// The barrier epoch lives in the rank's own signal area (slot kEpochSlot) and is
// advanced by the kernel itself, so a captured CUDA graph can be replayed.
constexpr int kEpochSlot = 32;

__global__ void __launch_bounds__(256) k_allreduce(ArArgs A) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    __shared__ uint32_t sh_epoch;
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) sh_epoch = *(volatile uint32_t*)(A.sig[A.rank] + kEpochSlot);
        __syncthreads();
    }
    const uint32_t epoch = blockIdx.x == 0 ? sh_epoch : 0u;

    if (blockIdx.x == 0) xrank_barrier(A, epoch + 1);
    grid.sync();

    // reduce-scatter of my slice
    uint64_t lo, hi;
    slice(A.nb4, A.rank, A.world, &lo, &hi);
    for (uint64_t u = lo + gtid; u < hi; u += gstride) {
        uint4 acc = __ldcg(A.b[0] + u);
        for (int r = 1; r < A.world; r++) {
            const uint4 v = __ldcg(A.b[r] + u);
            acc.x |= v.x; acc.y |= v.y; acc.z |= v.z; acc.w |= v.w;
        }
        A.my_b[u] = acc;
    }
    slice(A.nc4, A.rank, A.world, &lo, &hi);
    for (uint64_t u = lo + gtid; u < hi; u += gstride) {
        float4 acc = __ldcg(A.y[0] + u);
        for (int r = 1; r < A.world; r++) {
            const float4 v = __ldcg(A.y[r] + u);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        A.my_y[u] = acc;
    }
    grid.sync();
    if (blockIdx.x == 0) xrank_barrier(A, epoch + 2);
    grid.sync();

    // all-gather of the other slices
    for (int q = 0; q < A.world; q++) {
        if (q == A.rank) continue;
        slice(A.nb4, q, A.world, &lo, &hi);
        for (uint64_t u = lo + gtid; u < hi; u += gstride) A.my_b[u] = __ldcg(A.b[q] + u);
        slice(A.nc4, q, A.world, &lo, &hi);
        for (uint64_t u = lo + gtid; u < hi; u += gstride) A.my_y[u] = __ldcg(A.y[q] + u);
    }
    grid.sync();
    if (blockIdx.x == 0) {
        xrank_barrier(A, epoch + 3);
        if (threadIdx.x == 0) *(volatile uint32_t*)(A.sig[A.rank] + kEpochSlot) = epoch + 3;
    }
}

}  // namespace lhc

struct lhc_comm {
    int rank, world;
    lhc_params p;
    char* local;
    char* peers[lhc::kMaxRanks];
    void* opened[lhc::kMaxRanks];
    size_t bitmap_off, counters_off, signals_off, total;
    int grid;
};

using namespace lhc;

static void layout(const lhc_params* p, size_t* b, size_t* y, size_t* s, size_t* t) {
    *b = 0;
    *y = align_up(p->m / 8, 256);
    *s = align_up(*y + p->c * sizeof(float), 256);
    *t = *s + kSignalBytes;
}

extern "C" {

int lhc_comm_layout(const lhc_params* p, size_t* bitmap_off, size_t* counters_off,
                    size_t* signals_off, size_t* total_bytes) {
    if (int rc = validate(p)) return rc;
    size_t b, y, s, t;
    layout(p, &b, &y, &s, &t);
    if (bitmap_off) *bitmap_off = b;
    if (counters_off) *counters_off = y;
    if (signals_off) *signals_off = s;
    if (total_bytes) *total_bytes = t;
    return LHC_OK;
}

int lhc_ipc_handle(const void* dev_ptr, void* handle_out, uint64_t* offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return set_error(LHC_EINVAL, "NULL argument");
    // driver entry point resolved at run time: liblhc.so does not link libcuda
    typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        !fn)
        return set_error(LHC_ECOMM, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    CUresult r = reinterpret_cast<GetRange>(fn)(&base, &size, (CUdeviceptr)dev_ptr);
    if (r != CUDA_SUCCESS) return set_error(LHC_ECOMM, "cuMemGetAddressRange failed (%d)", (int)r);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
    if (e != cudaSuccess) return set_error(LHC_ECOMM, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
    memcpy(handle_out, &h, 64);
    *offset_out = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return LHC_OK;
}

int lhc_comm_create(int rank, int world, const void* handles, const uint64_t* offsets,
                    void* local_buf, size_t buf_bytes, const lhc_params* p, lhc_comm** out) {
    if (int rc = validate(p)) return rc;
    if (!out || !local_buf) return set_error(LHC_EINVAL, "NULL argument");
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
        return set_error(LHC_EINVAL, "world must be in [1, 8] and 0 <= rank < world");
    if (world > 1 && (!handles || !offsets)) return set_error(LHC_EINVAL, "NULL handles/offsets");
    if (((uintptr_t)local_buf & 255u) != 0) return set_error(LHC_EINVAL, "buffer must be 256-byte aligned");
    lhc_comm* c = new lhc_comm();
    c->rank = rank;
    c->world = world;
    c->p = *p;
    c->local = static_cast<char*>(local_buf);
    layout(p, &c->bitmap_off, &c->counters_off, &c->signals_off, &c->total);
    if (buf_bytes < c->total) {
        const size_t need = c->total;
        delete c;
        return set_error(LHC_ECAPACITY, "comm buffer too small: %zu < %zu", buf_bytes, need);
    }
    for (int q = 0; q < world; q++) {
        if (q == rank) {
            c->peers[q] = c->local;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, static_cast<const char*>(handles) + 64 * q, 64);
        void* ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (int a = 0; a < q; a++)
                if (c->opened[a]) cudaIpcCloseMemHandle(c->opened[a]);
            delete c;
            return set_error(LHC_ECOMM, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
        }
        c->opened[q] = ptr;
        c->peers[q] = static_cast<char*>(ptr) + offsets[q];
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_allreduce, 256, 0);
    c->grid = std::max(1, std::min(per_sm, 4)) * num_sms();
    *out = c;
    return LHC_OK;
}

int sketch_allreduce(lhc_comm* c, void* stream) {
    if (!c) return set_error(LHC_EINVAL, "NULL comm");
    reset_launches();
    if (c->world == 1) return LHC_OK;
    ArArgs A{};
    for (int q = 0; q < c->world; q++) {
        A.b[q] = reinterpret_cast<const uint4*>(c->peers[q] + c->bitmap_off);
        A.y[q] = reinterpret_cast<const float4*>(c->peers[q] + c->counters_off);
        A.sig[q] = reinterpret_cast<uint32_t*>(c->peers[q] + c->signals_off);
    }
    A.my_b = reinterpret_cast<uint4*>(c->local + c->bitmap_off);
    A.my_y = reinterpret_cast<float4*>(c->local + c->counters_off);
    A.nb4 = align_up(c->p.m / 8, 16) / 16;
    A.nc4 = c->p.c / 4;
    A.rank = c->rank;
    A.world = c->world;
    void* args[] = {(void*)&A};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_allreduce, dim3(c->grid), dim3(256),
                                                args, 0, (cudaStream_t)stream);
    count_launch();
    if (e != cudaSuccess) return set_error(LHC_ECUDA, "allreduce launch: %s", cudaGetErrorString(e));
    return LHC_OK;
}

void lhc_comm_destroy(lhc_comm* c) {
    if (!c) return;
    for (int q = 0; q < c->world; q++)
        if (c->opened[q]) cudaIpcCloseMemHandle(c->opened[q]);
    delete c;
}

}  // extern "C"
