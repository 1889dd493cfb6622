// comm.cu — multi-GPU homomorphic aggregation (Alg. 1 comment, P:L148-149:
// "the API makes ... Y <- sum Y and B <- OR B") as a hand-written NVLink P2P
// all-reduce with mixed operators over CUDA-IPC-mapped peer buffers.
//
// Buffer of every rank (lhc_comm_layout):
//   [bitmap B | counters Y | staging for B | staging for Y | signals]
// Each region is split into G contiguous slices of 16-byte units; rank q owns
// slice q.  One cooperative kernel per call, two-shot, every NVLink transfer a
// posted remote store (no remote loads):
//   push 1   rank r writes its slice q of B and Y into rank q's staging, slot r,
//            for every q != r                          ((G-1)/G * S bytes out)
//   barrier 1
//   reduce   rank q ORs / sums its own slice q with the G-1 staged copies in
//            ascending rank order (the same fp32 order on every rank), stores it,
//   push 2   and writes the reduced slice into every peer's B / Y   ((G-1)/G * S)
//   barrier 2
// No entry barrier is needed: push 1 only reads the caller's own sketch, and a
// rank's staging is rewritten only after it has passed barrier 2 of the
// previous call.  Barriers: every writing thread fences at system scope, the
// grid syncs, then block 0 publishes the epoch to every peer's signal slot with a
// system-scope release store and spins on its own slots with acquire loads.  The
// epoch counter lives on the device, so a captured CUDA graph can be replayed.
#include <cooperative_groups.h>
#include <cuda.h>

#include <cstring>

#include "launch.h"

namespace cg = cooperative_groups;

namespace lhc {

constexpr int kMaxRanks = 8;
constexpr size_t kSignalBytes = 256;
constexpr int kEpochSlot = 32;
constexpr int kU = 4;  // 16-byte units per thread and pass

struct ArArgs {
    uint4* b[kMaxRanks];    // B region of every rank (own one included)
    float4* y[kMaxRanks];   // Y region of every rank
    uint4* sb[kMaxRanks];   // B staging of every rank: G slots of sb_slot units
    float4* sy[kMaxRanks];  // Y staging of every rank: G slots of sy_slot units
    uint32_t* sig[kMaxRanks];
    uint64_t nb4, nc4;      // 16-byte units per region
    uint64_t sb_slot, sy_slot;
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

// Cross-rank barrier: all threads fence their remote stores, the grid syncs, block 0
// exchanges flags, the grid syncs again.
__device__ void xrank_barrier(cg::grid_group& grid, const ArArgs& A, uint32_t epoch) {
    __threadfence_system();
    grid.sync();
    if (blockIdx.x == 0) {
        const int t = threadIdx.x;
        if (t < A.world && t != A.rank) st_release_sys(A.sig[t] + A.rank, epoch);
        if (t < A.world && t != A.rank) {
            const uint32_t* mine = A.sig[A.rank] + t;
            while ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
            }
        }
    }
    grid.sync();
}

__device__ __forceinline__ void slice(uint64_t n, int q, int world, uint64_t* lo, uint64_t* hi) {
    *lo = n * q / world;
    *hi = n * (q + 1) / world;
}

__device__ __forceinline__ void combine(uint4& a, const uint4& v) {
    a.x |= v.x; a.y |= v.y; a.z |= v.z; a.w |= v.w;
}
__device__ __forceinline__ void combine(float4& a, const float4& v) {
    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
}

// push 1 for one region: my slice q -> rank q's staging slot `rank`
template <int G, typename T>
__device__ void push_slices(T* const* dst_stage, const T* src, uint64_t n, uint64_t slot, int rank,
                            uint64_t gtid, uint64_t gstride) {
#pragma unroll 1
    for (int d = 1; d < G; d++) {
        const int q = (rank + d) % G;  // stagger the destinations across ranks
        uint64_t lo, hi;
        slice(n, q, G, &lo, &hi);
        T* out = dst_stage[q] + (uint64_t)rank * slot - lo;
        for (uint64_t u0 = lo + gtid; u0 < hi; u0 += kU * gstride) {
            T v[kU];
#pragma unroll
            for (int a = 0; a < kU; a++) {
                const uint64_t u = u0 + a * gstride;
                if (u < hi) v[a] = __ldcs(src + u);
            }
#pragma unroll
            for (int a = 0; a < kU; a++) {
                const uint64_t u = u0 + a * gstride;
                if (u < hi) out[u] = v[a];
            }
        }
    }
}

// reduce my slice (own + G-1 staged copies, ascending rank), store it locally and
// into every peer's region
template <int G, typename T>
__device__ void reduce_push(T* const* region, const T* stage, uint64_t n, uint64_t slot, int rank,
                            uint64_t gtid, uint64_t gstride) {
    constexpr int U = G <= 2 ? 4 : G <= 4 ? 2 : 1;  // keeps U * G loads in flight
    uint64_t lo, hi;
    slice(n, rank, G, &lo, &hi);
    for (uint64_t u0 = lo + gtid; u0 < hi; u0 += U * gstride) {
        T v[U][G];
#pragma unroll
        for (int a = 0; a < U; a++) {
            const uint64_t u = u0 + a * gstride;
            if (u < hi) {
#pragma unroll
                for (int r = 0; r < G; r++)
                    v[a][r] = r == rank ? __ldcg(region[rank] + u) : __ldcg(stage + r * slot + (u - lo));
            }
        }
#pragma unroll
        for (int a = 0; a < U; a++) {
            const uint64_t u = u0 + a * gstride;
            if (u < hi) {
                T acc = v[a][0];
#pragma unroll
                for (int r = 1; r < G; r++) combine(acc, v[a][r]);
#pragma unroll
                for (int d = 0; d < G; d++) region[(rank + d) % G][u] = acc;
            }
        }
    }
}

#ifndef LHC_AR_TIMING
#define LHC_AR_TIMING 0
#endif
// debug: block 0 stamps the phase boundaries into signal slots 40.. (u64 each)
__device__ __forceinline__ void ar_stamp(const ArArgs& A, int k) {
    if (LHC_AR_TIMING && blockIdx.x == 0 && threadIdx.x == 0)
        reinterpret_cast<unsigned long long*>(A.sig[A.rank] + 40)[k] = globaltimer();
}

template <int G>
__global__ void __launch_bounds__(256) k_allreduce(ArArgs A) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t epoch = 0;
    if (blockIdx.x == 0) epoch = *(volatile uint32_t*)(A.sig[A.rank] + kEpochSlot);

    ar_stamp(A, 0);
    push_slices<G>(A.sb, A.b[A.rank], A.nb4, A.sb_slot, A.rank, gtid, gstride);
    push_slices<G>(A.sy, A.y[A.rank], A.nc4, A.sy_slot, A.rank, gtid, gstride);
    ar_stamp(A, 1);
    xrank_barrier(grid, A, epoch + 1);
    ar_stamp(A, 2);
    reduce_push<G>(A.b, A.sb[A.rank], A.nb4, A.sb_slot, A.rank, gtid, gstride);
    reduce_push<G>(A.y, A.sy[A.rank], A.nc4, A.sy_slot, A.rank, gtid, gstride);
    ar_stamp(A, 3);
    xrank_barrier(grid, A, epoch + 2);
    ar_stamp(A, 4);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *(volatile uint32_t*)(A.sig[A.rank] + kEpochSlot) = epoch + 2;
}


// ---------------------------------------------------------------------------
// Sharded aggregation (DESIGN.md NEXT-2, sharded decode).  The coordinates are
// split into G contiguous shards, shard q with its own sub-sketch; every rank's
// buffer is
//   [G slots of slot_units 16-byte units | staging: 2 x G slots | gather: 2 x G x
//    cap items (uint2) | signals + gather counts]
// slot q = [B_q | pad | Y_q], units [0, y_unit) combine with OR, the rest with +.
// sketch_reduce_scatter: push slot q -> rank q's staging[par][rank]; one barrier;
//   rank r reduces its slot r with the G-1 staged copies in ascending rank order.
// sketch_allgather_decoded: push my decoded (idx, val) list -> every peer's
//   gather[par][rank] (+ count); zero the peer-shard ranges of the local dense
//   output; one barrier; scatter every peer's list into them.
// Staging and gather areas alternate by call parity (per-op counters in the
// signal area), so one barrier per call suffices: a rank pushing in call k+1
// has passed call k's barrier, which every peer reached only after finishing
// call k-1, the last reader of the same-parity buffers.
// ---------------------------------------------------------------------------
constexpr int kRsCountSlot = 33;
constexpr int kAgCountSlot = 34;
constexpr int kGatherCountSlot = 64;  // u32 [2][kMaxRanks] from here

struct ShArgs {
    uint4* slots[kMaxRanks];  // slot region of every rank
    uint4* stage[kMaxRanks];  // staging region of every rank: [2][G][slot_units]
    uint2* gather[kMaxRanks]; // gather region of every rank: [2][G][cap]
    uint32_t* sig[kMaxRanks];
    uint64_t slot_units, y_unit, cap;
    int rank, world;
    // all-gather only
    const uint32_t* idx;
    const float* val;
    const unsigned long long* n_items;
    float* dense;
    uint64_t shard_width;
    uint32_t d;
};

template <int G>
__device__ void sh_barrier(cg::grid_group& grid, const ShArgs& A, uint32_t epoch) {
    ArArgs B{};
    for (int q = 0; q < G; q++) B.sig[q] = A.sig[q];
    B.rank = A.rank;
    B.world = G;
    xrank_barrier(grid, B, epoch);
}

template <int G>
__global__ void __launch_bounds__(256) k_reduce_scatter(ShArgs A) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t epoch = *(volatile uint32_t*)(A.sig[A.rank] + kEpochSlot);
    const uint32_t par = *(volatile uint32_t*)(A.sig[A.rank] + kRsCountSlot) & 1u;
    const uint64_t n = A.slot_units;
#pragma unroll 1
    for (int dd = 1; dd < G; dd++) {
        const int q = (A.rank + dd) % G;
        const uint4* src = A.slots[A.rank] + (uint64_t)q * n;
        uint4* out = A.stage[q] + ((uint64_t)par * G + A.rank) * n;
        for (uint64_t u0 = gtid; u0 < n; u0 += kU * gstride) {
            uint4 v[kU];
#pragma unroll
            for (int a = 0; a < kU; a++)
                if (u0 + a * gstride < n) v[a] = __ldcs(src + u0 + a * gstride);
#pragma unroll
            for (int a = 0; a < kU; a++)
                if (u0 + a * gstride < n) out[u0 + a * gstride] = v[a];
        }
    }
    sh_barrier<G>(grid, A, epoch + 1);
    constexpr int U = G <= 2 ? 4 : G <= 4 ? 2 : 1;
    uint4* mine = A.slots[A.rank] + (uint64_t)A.rank * n;
    const uint4* st = A.stage[A.rank] + (uint64_t)par * G * n;
    for (uint64_t u0 = gtid; u0 < n; u0 += U * gstride) {
        uint4 v[U][G];
#pragma unroll
        for (int a = 0; a < U; a++) {
            const uint64_t u = u0 + a * gstride;
            if (u < n) {
#pragma unroll
                for (int r = 0; r < G; r++) v[a][r] = r == A.rank ? __ldcg(mine + u) : __ldcg(st + r * n + u);
            }
        }
#pragma unroll
        for (int a = 0; a < U; a++) {
            const uint64_t u = u0 + a * gstride;
            if (u >= n) continue;
            if (u < A.y_unit) {
                uint4 acc = v[a][0];
#pragma unroll
                for (int r = 1; r < G; r++) combine(acc, v[a][r]);
                mine[u] = acc;
            } else {
                float4 acc = *reinterpret_cast<float4*>(&v[a][0]);
#pragma unroll
                for (int r = 1; r < G; r++) combine(acc, *reinterpret_cast<float4*>(&v[a][r]));
                mine[u] = *reinterpret_cast<uint4*>(&acc);
            }
        }
    }
    // every block read epoch / par before the barrier's grid syncs
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *(volatile uint32_t*)(A.sig[A.rank] + kEpochSlot) = epoch + 1;
        *(volatile uint32_t*)(A.sig[A.rank] + kRsCountSlot) = par + 1;
    }
}

constexpr uint32_t kOverflowMark = 0xFFFFFFFFu;

// dense[q*w, min(d, (q+1)*w)) = NaN: shard q's decode overflowed its capacity
__device__ __forceinline__ void fill_shard_nan(float* dense, int q, uint64_t w, uint32_t d,
                                               uint64_t gtid, uint64_t gstride) {
    const uint64_t lo = (uint64_t)q * w, hi = min((uint64_t)d, lo + w);
    for (uint64_t i = lo + gtid; i < hi; i += gstride) dense[i] = __int_as_float(0x7fc00000);
}

template <int G>
__global__ void __launch_bounds__(256) k_allgather_decoded(ShArgs A) {
    cg::grid_group grid = cg::this_grid();
    __shared__ __align__(16) float sh_tile[8][1024];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t epoch = *(volatile uint32_t*)(A.sig[A.rank] + kEpochSlot);
    const uint32_t par = *(volatile uint32_t*)(A.sig[A.rank] + kAgCountSlot) & 1u;
    // an overflowed own decode (n_items > cap: the peel did not run, the list is
    // stale) publishes kOverflowMark instead of a list; every rank then fills that
    // shard of its dense output with NaN, so the failure is visible everywhere
    const bool own_over = *A.n_items > A.cap;
    const uint64_t n = own_over ? 0 : *A.n_items;
    // A gather slot holds cap indices then cap values (cap a multiple of 4): the
    // decoded list travels as two 16-byte-vector streams.
    const uint64_t nv = n / 4;
    const uint4* src_i = reinterpret_cast<const uint4*>(A.idx);
    const uint4* src_v = reinterpret_cast<const uint4*>(A.val);
    // the whole grid pushes over NVLink; the peers' ranges of the local dense output are
    // assembled chunk by chunk after the barrier (no zeroing pass, no scattered stores)
    const uint64_t rtid = gtid, rstride = gstride;
    {
#pragma unroll 1
        for (int dd = 1; dd < G; dd++) {
            const int q = (A.rank + dd) % G;
            uint32_t* slot = reinterpret_cast<uint32_t*>(A.gather[q] + ((uint64_t)par * G + A.rank) * A.cap);
            uint4* di = reinterpret_cast<uint4*>(slot);
            uint4* dv = reinterpret_cast<uint4*>(slot + A.cap);
            for (uint64_t u = rtid; u < nv; u += rstride) {
                const uint4 a = __ldcg(src_i + u), b = __ldcg(src_v + u);
                di[u] = a;
                dv[u] = b;
            }
            for (uint64_t i = 4 * nv + rtid; i < n; i += rstride) {
                slot[i] = __ldcg(A.idx + i);
                slot[A.cap + i] = __float_as_uint(__ldcg(A.val + i));
            }
            if (rtid == 0)
                A.sig[q][kGatherCountSlot + par * kMaxRanks + A.rank] = own_over ? kOverflowMark : (uint32_t)n;
        }
    }
    sh_barrier<G>(grid, A, epoch + 1);
    if (own_over) fill_shard_nan(A.dense, A.rank, A.shard_width, A.d, gtid, gstride);
#pragma unroll 1
    for (int dd = 1; dd < G; dd++) {
        const int q = (A.rank + dd) % G;
        const uint32_t cnt = *(volatile uint32_t*)(A.sig[A.rank] + kGatherCountSlot + par * kMaxRanks + q);
        if (cnt == kOverflowMark) {
            fill_shard_nan(A.dense, q, A.shard_width, A.d, gtid, gstride);
            continue;
        }
        const uint64_t nq = min((uint64_t)cnt, A.cap);
        const uint32_t* slot = reinterpret_cast<const uint32_t*>(A.gather[A.rank] + ((uint64_t)par * G + q) * A.cap);
        const uint32_t* si = slot;
        const float* sv = reinterpret_cast<const float*>(slot + A.cap);
        // shard q = coordinates [q w, min(d, (q + 1) w)), its list ascending in
        // shard-local coordinates: a warp assembles a contiguous range of its
        // 1024-coordinate chunks in shared memory (zeros + the listed values) and
        // writes each chunk with full-line stores
        const uint64_t s0 = (uint64_t)q * A.shard_width;
        const uint64_t len = s0 < A.d ? min((uint64_t)A.shard_width, (uint64_t)A.d - s0) : 0;
        const uint64_t nch = (len + 1023) / 1024;
        const uint64_t nwarps = gstride >> 5, wid = gtid >> 5;
        const uint64_t cpw = (nch + nwarps - 1) / nwarps;
        const uint64_t c0 = min(nch, wid * cpw), c1 = min(nch, c0 + cpw);
        if (c0 < c1) {
            // first list entry of chunk c0 (binary search, every lane the same)
            uint64_t lo = 0, hi = nq;
            const uint64_t key = c0 * 1024;
            while (lo < hi) {
                const uint64_t mid = (lo + hi) / 2;
                if (__ldcs(si + mid) < key) lo = mid + 1; else hi = mid;
            }
            uint64_t pos = lo;
            float* tile = sh_tile[threadIdx.x >> 5];
            float4* t4 = reinterpret_cast<float4*>(tile);
            for (uint64_t c = c0; c < c1; c++) {
#pragma unroll
                for (int u = 0; u < 8; u++) t4[lane + 32 * u] = make_float4(0.f, 0.f, 0.f, 0.f);
                __syncwarp();
                const uint64_t cend = (c + 1) * 1024;
                for (;;) {
                    const uint64_t a = pos + lane;
                    const uint32_t ix = a < nq ? __ldcs(si + a) : 0xffffffffu;
                    const bool in = a < nq && ix < cend;
                    if (in) tile[ix & 1023] = __ldcs(sv + a);
                    const uint32_t nin = __popc(__ballot_sync(0xffffffffu, in));  // a prefix: sorted
                    pos += nin;
                    if (nin < 32) break;
                }
                __syncwarp();
                float* out = A.dense + s0 + c * 1024;
                if ((c + 1) * 1024 <= len) {
                    float4* o4 = reinterpret_cast<float4*>(out);
#pragma unroll
                    for (int u = 0; u < 8; u++) __stcs(o4 + lane + 32 * u, t4[lane + 32 * u]);
                } else {
                    for (uint64_t a = lane; c * 1024 + a < len; a += 32) out[a] = tile[a];
                }
                __syncwarp();
            }
        }
    }
    // every block read epoch / par before the barrier's grid syncs
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *(volatile uint32_t*)(A.sig[A.rank] + kEpochSlot) = epoch + 1;
        *(volatile uint32_t*)(A.sig[A.rank] + kAgCountSlot) = par + 1;
    }
}

}  // namespace lhc

struct lhc_comm {
    int rank, world;
    lhc_params p;
    char* local;
    char* peers[lhc::kMaxRanks];
    void* opened[lhc::kMaxRanks];
    size_t bitmap_off, counters_off, stage_b_off, stage_y_off, signals_off, total;
    int grid;
    // sharded communicator (lhc_shard_comm_create)
    int sharded;
    uint64_t slot_bytes, y_off, cap;
    size_t stage_off, gather_off;
};

using namespace lhc;

// [B | Y | staging B | staging Y | signals]; a staging area holds G slots of
// ceil(n/G) 16-byte units, at most n + kMaxRanks units for any G <= kMaxRanks.
static uint64_t units_b(const lhc_params* p) { return align_up(p->m / 8, 16) / 16; }
static uint64_t units_y(const lhc_params* p) { return p->c / 4; }
static void layout(const lhc_params* p, size_t* b, size_t* y, size_t* sb, size_t* sy, size_t* s,
                   size_t* t) {
    *b = 0;
    *y = align_up(p->m / 8, 256);
    *sb = align_up(*y + p->c * sizeof(float), 256);
    *sy = align_up(*sb + (units_b(p) + kMaxRanks) * 16, 256);
    *s = align_up(*sy + (units_y(p) + kMaxRanks) * 16, 256);
    *t = *s + kSignalBytes;
}

// sharded buffer: [G slots | staging 2 x G slots | gather 2 x G x cap x 8 B | signals 512 B]
static int shard_layout(const lhc_params* ps, int world, uint64_t cap, size_t* slot, size_t* y_off,
                        size_t* stage, size_t* gather, size_t* sig, size_t* total) {
    if (int rc = validate(ps)) return rc;
    if (world < 1 || world > kMaxRanks) return set_error(LHC_EINVAL, "world must be in [1, 8]");
    if (cap == 0 || cap >= (1ull << 32)) return set_error(LHC_EINVAL, "cap_items must be in [1, 2^32)");
    cap = (cap + 3) / 4 * 4;  // gather slots hold 16-byte vectors
    *y_off = align_up(ps->m / 8, 256);
    *slot = align_up(*y_off + ps->c * sizeof(float), 256);
    *stage = *slot * world;
    *gather = *stage + 2 * *slot * world;
    *sig = align_up(*gather + 2 * (size_t)world * cap * 8, 256);
    *total = *sig + 2 * kSignalBytes;
    return LHC_OK;
}

static int shard_grid() {
    const void* fns[] = {(const void*)k_reduce_scatter<2>, (const void*)k_reduce_scatter<3>,
                         (const void*)k_reduce_scatter<4>, (const void*)k_reduce_scatter<5>,
                         (const void*)k_reduce_scatter<6>, (const void*)k_reduce_scatter<7>,
                         (const void*)k_reduce_scatter<8>, (const void*)k_allgather_decoded<2>,
                         (const void*)k_allgather_decoded<3>, (const void*)k_allgather_decoded<4>,
                         (const void*)k_allgather_decoded<5>, (const void*)k_allgather_decoded<6>,
                         (const void*)k_allgather_decoded<7>, (const void*)k_allgather_decoded<8>};
    int per_sm = 4;
    for (const void* f : fns) {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, 256, 0);
        per_sm = std::min(per_sm, n);
    }
    return std::max(1, per_sm) * num_sms();
}

static ShArgs shard_args(const lhc_comm* c) {
    ShArgs A{};
    for (int q = 0; q < c->world; q++) {
        A.slots[q] = reinterpret_cast<uint4*>(c->peers[q]);
        A.stage[q] = reinterpret_cast<uint4*>(c->peers[q] + c->stage_off);
        A.gather[q] = reinterpret_cast<uint2*>(c->peers[q] + c->gather_off);
        A.sig[q] = reinterpret_cast<uint32_t*>(c->peers[q] + c->signals_off);
    }
    A.slot_units = c->slot_bytes / 16;
    A.y_unit = c->y_off / 16;
    A.cap = c->cap;
    A.rank = c->rank;
    A.world = c->world;
    return A;
}

static int launch_coop(const void* fn, const lhc_comm* c, ShArgs& A, void* stream, const char* what) {
    void* args[] = {(void*)&A};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(c->grid), dim3(256), args, 0, (cudaStream_t)stream);
    count_launch();
    if (e != cudaSuccess) return set_error(LHC_ECUDA, "%s launch: %s", what, cudaGetErrorString(e));
    return LHC_OK;
}

extern "C" {

int lhc_shard_layout(const lhc_params* ps, int world, uint64_t cap_items, size_t* slot_bytes,
                     size_t* counters_off, size_t* total_bytes) {
    size_t slot = 0, y = 0, st = 0, ga = 0, sg = 0, t = 0;
    if (int rc = shard_layout(ps, world, cap_items, &slot, &y, &st, &ga, &sg, &t)) return rc;
    if (slot_bytes) *slot_bytes = slot;
    if (counters_off) *counters_off = y;
    if (total_bytes) *total_bytes = t;
    return LHC_OK;
}

int lhc_comm_layout(const lhc_params* p, size_t* bitmap_off, size_t* counters_off,
                    size_t* signals_off, size_t* total_bytes) {
    if (int rc = validate(p)) return rc;
    size_t b, y, sb, sy, s, t;
    layout(p, &b, &y, &sb, &sy, &s, &t);
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
    layout(p, &c->bitmap_off, &c->counters_off, &c->stage_b_off, &c->stage_y_off, &c->signals_off,
           &c->total);
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
    // one grid size that is co-resident for every instantiation
    const void* fns[] = {(const void*)k_allreduce<2>, (const void*)k_allreduce<3>,
                         (const void*)k_allreduce<4>, (const void*)k_allreduce<5>,
                         (const void*)k_allreduce<6>, (const void*)k_allreduce<7>,
                         (const void*)k_allreduce<8>};
    int per_sm = 4;
    for (const void* f : fns) {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, 256, 0);
        per_sm = std::min(per_sm, n);
    }
    c->grid = std::max(1, per_sm) * num_sms();
    *out = c;
    return LHC_OK;
}

int sketch_allreduce(lhc_comm* c, void* stream) {
    if (!c) return set_error(LHC_EINVAL, "NULL comm");
    if (c->sharded) return set_error(LHC_EINVAL, "sharded communicator: use sketch_reduce_scatter");
    reset_launches();
    if (c->world == 1) return LHC_OK;
    ArArgs A{};
    const uint64_t nb4 = units_b(&c->p), nc4 = units_y(&c->p);
    for (int q = 0; q < c->world; q++) {
        A.b[q] = reinterpret_cast<uint4*>(c->peers[q] + c->bitmap_off);
        A.y[q] = reinterpret_cast<float4*>(c->peers[q] + c->counters_off);
        A.sb[q] = reinterpret_cast<uint4*>(c->peers[q] + c->stage_b_off);
        A.sy[q] = reinterpret_cast<float4*>(c->peers[q] + c->stage_y_off);
        A.sig[q] = reinterpret_cast<uint32_t*>(c->peers[q] + c->signals_off);
    }
    A.nb4 = nb4;
    A.nc4 = nc4;
    A.sb_slot = (nb4 + c->world - 1) / c->world;
    A.sy_slot = (nc4 + c->world - 1) / c->world;
    A.rank = c->rank;
    A.world = c->world;
    void* args[] = {(void*)&A};
    const void* fns[kMaxRanks + 1] = {nullptr,
                                      nullptr,
                                      (const void*)k_allreduce<2>,
                                      (const void*)k_allreduce<3>,
                                      (const void*)k_allreduce<4>,
                                      (const void*)k_allreduce<5>,
                                      (const void*)k_allreduce<6>,
                                      (const void*)k_allreduce<7>,
                                      (const void*)k_allreduce<8>};
    const void* fn = fns[c->world];
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(c->grid), dim3(256), args, 0,
                                                (cudaStream_t)stream);
    count_launch();
    if (e != cudaSuccess) return set_error(LHC_ECUDA, "allreduce launch: %s", cudaGetErrorString(e));
    return LHC_OK;
}

int lhc_shard_comm_create(int rank, int world, const void* handles, const uint64_t* offsets,
                          void* local_buf, size_t buf_bytes, const lhc_params* ps, uint64_t cap_items,
                          lhc_comm** out) {
    size_t slot = 0, y = 0, st = 0, ga = 0, sg = 0, t = 0;
    if (int rc = shard_layout(ps, world, cap_items, &slot, &y, &st, &ga, &sg, &t)) return rc;
    if (!out || !local_buf) return set_error(LHC_EINVAL, "NULL argument");
    if (rank < 0 || rank >= world) return set_error(LHC_EINVAL, "0 <= rank < world required");
    if (world > 1 && (!handles || !offsets)) return set_error(LHC_EINVAL, "NULL handles/offsets");
    if (((uintptr_t)local_buf & 255u) != 0) return set_error(LHC_EINVAL, "buffer must be 256-byte aligned");
    if (buf_bytes < t) return set_error(LHC_ECAPACITY, "shard buffer too small: %zu < %zu", buf_bytes, t);
    lhc_comm* c = new lhc_comm();
    c->rank = rank;
    c->world = world;
    c->p = *ps;
    c->local = static_cast<char*>(local_buf);
    c->sharded = 1;
    c->slot_bytes = slot;
    c->y_off = y;
    c->cap = (cap_items + 3) / 4 * 4;
    c->stage_off = st;
    c->gather_off = ga;
    c->signals_off = sg;
    c->total = t;
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
    c->grid = shard_grid();
    *out = c;
    return LHC_OK;
}

int sketch_reduce_scatter(lhc_comm* c, void* stream) {
    if (!c || !c->sharded) return set_error(LHC_EINVAL, "not a sharded communicator");
    reset_launches();
    if (c->world == 1) return LHC_OK;
    ShArgs A = shard_args(c);
    const void* fns[kMaxRanks + 1] = {nullptr, nullptr,
                                      (const void*)k_reduce_scatter<2>, (const void*)k_reduce_scatter<3>,
                                      (const void*)k_reduce_scatter<4>, (const void*)k_reduce_scatter<5>,
                                      (const void*)k_reduce_scatter<6>, (const void*)k_reduce_scatter<7>,
                                      (const void*)k_reduce_scatter<8>};
    return launch_coop(fns[c->world], c, A, stream, "reduce_scatter");
}

int sketch_allgather_decoded(lhc_comm* c, const uint32_t* idx, const float* val,
                             const unsigned long long* n_items, uint64_t shard_width, uint32_t d,
                             float* dense, void* stream) {
    if (!c || !c->sharded) return set_error(LHC_EINVAL, "not a sharded communicator");
    if (!idx || !val || !n_items || !dense) return set_error(LHC_EINVAL, "NULL argument");
    if (((uintptr_t)idx | (uintptr_t)val | (uintptr_t)dense) & 15u)
        return set_error(LHC_EINVAL, "idx, val and dense must be 16-byte aligned");
    if (shard_width == 0 || shard_width % 4 || (uint64_t)(c->world - 1) * shard_width >= d)
        return set_error(LHC_EINVAL, "shard_width must be a positive multiple of 4, every shard non-empty");
    reset_launches();
    if (c->world == 1) return LHC_OK;
    ShArgs A = shard_args(c);
    A.idx = idx;
    A.val = val;
    A.n_items = n_items;
    A.dense = dense;
    A.shard_width = shard_width;
    A.d = d;
    const void* fns[kMaxRanks + 1] = {nullptr, nullptr,
                                      (const void*)k_allgather_decoded<2>, (const void*)k_allgather_decoded<3>,
                                      (const void*)k_allgather_decoded<4>, (const void*)k_allgather_decoded<5>,
                                      (const void*)k_allgather_decoded<6>, (const void*)k_allgather_decoded<7>,
                                      (const void*)k_allgather_decoded<8>};
    return launch_coop(fns[c->world], c, A, stream, "allgather");
}

void lhc_comm_destroy(lhc_comm* c) {
    if (!c) return;
    for (int q = 0; q < c->world; q++)
        if (c->opened[q]) cudaIpcCloseMemHandle(c->opened[q]);
    delete c;
}

}  // extern "C"

// ===========================================================================
// NVLS: in-switch aggregation through an NVSwitch multicast object (DESIGN.md
// NEXT-2; the paper's in-network aggregation, P:L122-124 / P:L283, done by the
// switch).  Every rank binds its own physical buffer to one multicast object and
// maps it twice: unicast (local loads/stores, where the sketch is compressed) and
// multicast (multimem.* instructions, which the switch applies to every rank's
// copy):
//   multimem.ld_reduce .add.f32 / .or.b64   the switch reads the address on every
//                                           rank and returns the sum / OR
//   multimem.st                              one store reaches every rank's copy
//   multimem.red.add.u32                     barrier counter on every rank
// The multicast handle travels as a POSIX file descriptor over an abstract Unix
// socket (SCM_RIGHTS) from rank 0 to the others.
// ===========================================================================
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <chrono>
#include <thread>

namespace lhc {

constexpr size_t kNvlsSig = 4096;  // signal area at the end of the mapping
constexpr int kNvU = 4;            // multimem reductions in flight per thread

__device__ __forceinline__ void mm_or_b64(uint64_t* mc, uint64_t* out) {
    asm volatile("multimem.ld_reduce.weak.global.or.b64 %0, [%1];" : "=l"(*out) : "l"(mc) : "memory");
}
__device__ __forceinline__ float4 mm_add_v4f32(const float* mc) {
    float4 v;
    asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc) : "memory");
    return v;
}
__device__ __forceinline__ void mm_st_v4(float* mc, float4 v) {
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};"
                 ::"l"(mc), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void mm_st_u32(uint32_t* mc, uint32_t v) {
    asm volatile("multimem.st.weak.global.b32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}

struct NvArgs {
    char* uc;              // local (unicast) view of the buffer
    char* mc;              // multicast view
    uint32_t* sig_uc;      // [0] barrier counter (multicast-updated), [16] epoch (local)
    uint32_t* sig_mc;
    int rank, world;
    // regions in 16-byte units
    uint64_t lo, hi, y_unit;      // all-reduce: units [0, hi) (bitmap below y_unit); slice by rank
    uint64_t slot_units, cap;     // sharded layout
    uint64_t gather_off;
    const uint32_t* idx;
    const float* val;
    const unsigned long long* n_items;
    float* dense;
    uint64_t shard_width;
    uint32_t d;
};

// all ranks: every thread's writes are ordered before the switch-wide counter
// increment; block 0 waits for all ranks' increments
__device__ void nv_barrier(cg::grid_group& grid, const NvArgs& A, uint32_t target) {
    __threadfence_system();
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(A.sig_mc), "r"(1u) : "memory");
        while ((int32_t)(ld_acquire_sys(A.sig_uc) - target) < 0) {
        }
        asm volatile("fence.proxy.alias;" ::: "memory");
    }
    grid.sync();
}

#ifndef LHC_NV_TIMING
#define LHC_NV_TIMING 0
#endif
// debug: block 0 stamps phase boundaries into the signal area (u64 slots from byte 512)
__device__ __forceinline__ void nv_stamp(const NvArgs& A, int k) {
    if (LHC_NV_TIMING && blockIdx.x == 0 && threadIdx.x == 0)
        reinterpret_cast<unsigned long long*>(A.sig_uc + 128)[k] = globaltimer();
}

// 16-byte unit u of the multicast view: OR (bitmap) or sum (counters) over ranks
__device__ __forceinline__ float4 nv_reduce_unit(const NvArgs& A, uint64_t off_bytes, bool is_or) {
    if (is_or) {
        uint64_t a, b;
        mm_or_b64(reinterpret_cast<uint64_t*>(A.mc + off_bytes), &a);
        mm_or_b64(reinterpret_cast<uint64_t*>(A.mc + off_bytes + 8), &b);
        float4 v;
        v.x = __uint_as_float((uint32_t)a);
        v.y = __uint_as_float((uint32_t)(a >> 32));
        v.z = __uint_as_float((uint32_t)b);
        v.w = __uint_as_float((uint32_t)(b >> 32));
        return v;
    }
    return mm_add_v4f32(reinterpret_cast<const float*>(A.mc + off_bytes));
}

__global__ void __launch_bounds__(256) k_allreduce_nvls(NvArgs A) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t epoch = *(volatile uint32_t*)(A.sig_uc + 16);
    nv_stamp(A, 0);
    nv_barrier(grid, A, (epoch + 1) * (uint32_t)A.world);  // every rank's sketch is complete
    nv_stamp(A, 1);
    // kNvU switch reductions in flight per thread
    for (uint64_t u0 = A.lo + gtid; u0 < A.hi; u0 += kNvU * gstride) {
        float4 v[kNvU];
#pragma unroll
        for (int a = 0; a < kNvU; a++) {
            const uint64_t u = u0 + a * gstride;
            if (u < A.hi) v[a] = nv_reduce_unit(A, u * 16, u < A.y_unit);
        }
#pragma unroll
        for (int a = 0; a < kNvU; a++) {
            const uint64_t u = u0 + a * gstride;
            if (u < A.hi) mm_st_v4(reinterpret_cast<float*>(A.mc + u * 16), v[a]);
        }
    }
    nv_stamp(A, 2);
    nv_barrier(grid, A, (epoch + 2) * (uint32_t)A.world);  // every slice is everywhere
    nv_stamp(A, 3);
    if (blockIdx.x == 0 && threadIdx.x == 0) *(volatile uint32_t*)(A.sig_uc + 16) = epoch + 2;
}

// sharded layout: slot `rank` (locally) = OR / sum over ranks of their slot `rank`
__global__ void __launch_bounds__(256) k_reduce_scatter_nvls(NvArgs A) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t epoch = *(volatile uint32_t*)(A.sig_uc + 16);
    nv_barrier(grid, A, (epoch + 1) * (uint32_t)A.world);
    const uint64_t base = (uint64_t)A.rank * A.slot_units;
    uint4* out = reinterpret_cast<uint4*>(A.uc) + base;
    for (uint64_t u0 = gtid; u0 < A.slot_units; u0 += kNvU * gstride) {
        float4 v[kNvU];
#pragma unroll
        for (int a = 0; a < kNvU; a++) {
            const uint64_t u = u0 + a * gstride;
            if (u < A.slot_units) v[a] = nv_reduce_unit(A, (base + u) * 16, u < A.y_unit);
        }
#pragma unroll
        for (int a = 0; a < kNvU; a++) {
            const uint64_t u = u0 + a * gstride;
            if (u < A.slot_units) out[u] = *reinterpret_cast<const uint4*>(&v[a]);
        }
    }
    // the peers may rewrite their slots (next step) only after every rank read them
    nv_barrier(grid, A, (epoch + 2) * (uint32_t)A.world);
    if (blockIdx.x == 0 && threadIdx.x == 0) *(volatile uint32_t*)(A.sig_uc + 16) = epoch + 2;
}

// sharded layout: my decoded list -> gather slot [par][rank] of every rank with one
// multicast store per 16 bytes; zero the peer ranges of dense; barrier; scatter
__global__ void __launch_bounds__(256) k_allgather_nvls(NvArgs A) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t epoch = *(volatile uint32_t*)(A.sig_uc + 16);
    const uint32_t par = *(volatile uint32_t*)(A.sig_uc + 17) & 1u;
    const int G = A.world;
    const bool own_over = *A.n_items > A.cap;  // as in k_allgather_decoded
    const uint64_t n = own_over ? 0 : *A.n_items;
    const uint64_t slot_bytes = A.cap * 8;
    {
        const uint64_t off = A.gather_off + ((uint64_t)par * G + A.rank) * slot_bytes;
        float* di = reinterpret_cast<float*>(A.mc + off);
        float* dv = reinterpret_cast<float*>(A.mc + off + A.cap * 4);
        const uint64_t nv = (n + 3) / 4;  // the source lists hold >= n rounded up to 4? no: guard
        for (uint64_t u = gtid; u < nv; u += gstride) {
            float4 a, b;
            const uint64_t i0 = 4 * u;
            a.x = __uint_as_float(i0 + 0 < n ? __ldcg(A.idx + i0 + 0) : 0u);
            a.y = __uint_as_float(i0 + 1 < n ? __ldcg(A.idx + i0 + 1) : 0u);
            a.z = __uint_as_float(i0 + 2 < n ? __ldcg(A.idx + i0 + 2) : 0u);
            a.w = __uint_as_float(i0 + 3 < n ? __ldcg(A.idx + i0 + 3) : 0u);
            b.x = i0 + 0 < n ? __ldcg(A.val + i0 + 0) : 0.f;
            b.y = i0 + 1 < n ? __ldcg(A.val + i0 + 1) : 0.f;
            b.z = i0 + 2 < n ? __ldcg(A.val + i0 + 2) : 0.f;
            b.w = i0 + 3 < n ? __ldcg(A.val + i0 + 3) : 0.f;
            mm_st_v4(di + i0, a);
            mm_st_v4(dv + i0, b);
        }
        if (gtid == 0)
            mm_st_u32(reinterpret_cast<uint32_t*>(A.sig_mc) + 64 + par * kMaxRanks + A.rank,
                      own_over ? kOverflowMark : (uint32_t)n);
    }
    {
        const uint64_t lo = (uint64_t)A.rank * A.shard_width;
        const uint64_t hi = min((uint64_t)A.d, lo + A.shard_width);
        float4* d4 = reinterpret_cast<float4*>(A.dense);
        const uint64_t a4 = lo / 4, b4 = hi / 4, e4 = A.d / 4, own4 = b4 - a4;
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        for (uint64_t u = gtid; u < e4 - own4; u += gstride) __stcs(d4 + (u < a4 ? u : u + own4), z);
        for (uint64_t i = max(hi, 4 * e4) + gtid; i < A.d; i += gstride) A.dense[i] = 0.f;
    }
    nv_barrier(grid, A, (epoch + 1) * (uint32_t)A.world);
    if (own_over) fill_shard_nan(A.dense, A.rank, A.shard_width, A.d, gtid, gstride);
    for (int dd = 1; dd < G; dd++) {
        const int q = (A.rank + dd) % G;
        const uint32_t cnt = *(volatile uint32_t*)(A.sig_uc + 64 + par * kMaxRanks + q);
        if (cnt == kOverflowMark) {
            fill_shard_nan(A.dense, q, A.shard_width, A.d, gtid, gstride);
            continue;
        }
        const uint64_t nq = min((uint64_t)cnt, A.cap);
        const char* slot = A.uc + A.gather_off + ((uint64_t)par * G + q) * slot_bytes;
        const uint4* si = reinterpret_cast<const uint4*>(slot);
        const uint4* sv = reinterpret_cast<const uint4*>(slot + A.cap * 4);
        float* base = A.dense + (uint64_t)q * A.shard_width;
        for (uint64_t u = gtid; u < (nq + 3) / 4; u += gstride) {
            const uint4 a = __ldcs(si + u), b = __ldcs(sv + u);
            if (b.x) base[a.x] = __uint_as_float(b.x);
            if (b.y) base[a.y] = __uint_as_float(b.y);
            if (b.z) base[a.z] = __uint_as_float(b.z);
            if (b.w) base[a.w] = __uint_as_float(b.w);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *(volatile uint32_t*)(A.sig_uc + 16) = epoch + 1;
        *(volatile uint32_t*)(A.sig_uc + 17) = par + 1;
    }
}

}  // namespace lhc

struct lhc_nvls {
    int rank, world, dev;
    size_t size;  // mapping bytes (multiple of the multicast granularity)
    CUmemGenericAllocationHandle mc, mem;
    CUdeviceptr uc_va, mc_va;
    int opened, bound;
    int grid;
};

namespace {

void* drv(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess) return nullptr;
    return fn;
}
#define DRV(name) reinterpret_cast<decltype(&name)>(drv(#name))

int drv_err(const char* what, CUresult r) {
    return lhc::set_error(LHC_ECOMM, "%s failed (CUresult %d)", what, (int)r);
}

void sock_addr(const char* name, sockaddr_un* a, socklen_t* len) {
    memset(a, 0, sizeof(*a));
    a->sun_family = AF_UNIX;
    const size_t n = std::min(strlen(name), sizeof(a->sun_path) - 2);
    memcpy(a->sun_path + 1, name, n);  // abstract namespace
    *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

int send_fd(int sock, int fd) {
    char byte = 0;
    iovec io{&byte, 1};
    char ctrl[CMSG_SPACE(sizeof(int))] = {};
    msghdr m{};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof(ctrl);
    cmsghdr* c = CMSG_FIRSTHDR(&m);
    c->cmsg_level = SOL_SOCKET;
    c->cmsg_type = SCM_RIGHTS;
    c->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(c), &fd, sizeof(int));
    return sendmsg(sock, &m, 0) == 1 ? 0 : -1;
}

int recv_fd(int sock) {
    char byte = 0;
    iovec io{&byte, 1};
    char ctrl[CMSG_SPACE(sizeof(int))] = {};
    msghdr m{};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof(ctrl);
    if (recvmsg(sock, &m, 0) != 1) return -1;
    cmsghdr* c = CMSG_FIRSTHDR(&m);
    if (!c || c->cmsg_type != SCM_RIGHTS) return -1;
    int fd = -1;
    memcpy(&fd, CMSG_DATA(c), sizeof(int));
    return fd;
}

}  // namespace

using namespace lhc;

extern "C" {

int lhc_nvls_open(int rank, int world, const char* rendezvous, size_t bytes, lhc_nvls** out) {
    if (!out || !rendezvous || !*rendezvous) return set_error(LHC_EINVAL, "NULL argument");
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
        return set_error(LHC_EINVAL, "world must be in [1, 8] and 0 <= rank < world");
    if (bytes == 0) return set_error(LHC_EINVAL, "bytes must be > 0");
    auto cuDeviceGet_ = DRV(cuDeviceGet);
    auto cuMulticastGetGranularity_ = DRV(cuMulticastGetGranularity);
    auto cuMulticastCreate_ = DRV(cuMulticastCreate);
    auto cuMemExport_ = DRV(cuMemExportToShareableHandle);
    auto cuMemImport_ = DRV(cuMemImportFromShareableHandle);
    auto cuMulticastAddDevice_ = DRV(cuMulticastAddDevice);
    if (!cuDeviceGet_ || !cuMulticastGetGranularity_ || !cuMulticastCreate_ || !cuMemExport_ ||
        !cuMemImport_ || !cuMulticastAddDevice_)
        return set_error(LHC_ECOMM, "multicast driver entry points unavailable");
    int ord = 0;
    cudaGetDevice(&ord);
    cudaFree(nullptr);  // the runtime's primary context is current
    CUdevice dev;
    if (CUresult r = cuDeviceGet_(&dev, ord)) return drv_err("cuDeviceGet", r);
    auto cuMemRelease_ = DRV(cuMemRelease);
    CUmulticastObjectProp prop{};
    prop.numDevices = (unsigned)world;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    prop.size = bytes + kNvlsSig;
    size_t gran = 0;
    if (CUresult r = cuMulticastGetGranularity_(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED))
        return drv_err("cuMulticastGetGranularity", r);
    prop.size = (prop.size + gran - 1) / gran * gran;

    CUmemGenericAllocationHandle mc = 0;
    sockaddr_un addr;
    socklen_t alen;
    sock_addr(rendezvous, &addr, &alen);
    // once the multicast object exists (created or imported), every failure releases it
    auto release_mc = [&](int rc) {
        if (mc && cuMemRelease_) cuMemRelease_(mc);
        return rc;
    };
    if (rank == 0) {
        if (CUresult r = cuMulticastCreate_(&mc, &prop)) return drv_err("cuMulticastCreate", r);
        int fd = -1;
        if (CUresult r = cuMemExport_(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0))
            return release_mc(drv_err("cuMemExportToShareableHandle", r));
        int ls = socket(AF_UNIX, SOCK_STREAM, 0);
        if (ls < 0 || bind(ls, (sockaddr*)&addr, alen) != 0 || listen(ls, world) != 0) {
            if (ls >= 0) close(ls);
            close(fd);
            return release_mc(set_error(LHC_ECOMM, "rendezvous socket '%s' unavailable", rendezvous));
        }
        for (int i = 1; i < world; i++) {
            int c = accept(ls, nullptr, nullptr);
            if (c < 0 || send_fd(c, fd) != 0) {
                if (c >= 0) close(c);
                close(ls);
                close(fd);
                return release_mc(set_error(LHC_ECOMM, "sending the multicast handle failed"));
            }
            close(c);
        }
        close(ls);
        close(fd);
    } else {
        int s = -1;
        const auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            s = socket(AF_UNIX, SOCK_STREAM, 0);
            if (s >= 0 && connect(s, (sockaddr*)&addr, alen) == 0) break;
            if (s >= 0) close(s);
            s = -1;
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
                return set_error(LHC_ECOMM, "rank 0 did not open rendezvous '%s'", rendezvous);
            std::this_thread::sleep_for(std::chrono::milliseconds(5));
        }
        const int fd = recv_fd(s);
        close(s);
        if (fd < 0) return set_error(LHC_ECOMM, "receiving the multicast handle failed");
        CUresult r = cuMemImport_(&mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
        close(fd);
        if (r) return drv_err("cuMemImportFromShareableHandle", r);
    }
    if (CUresult r = cuMulticastAddDevice_(mc, dev)) return release_mc(drv_err("cuMulticastAddDevice", r));
    lhc_nvls* h = new lhc_nvls();
    h->rank = rank;
    h->world = world;
    h->dev = ord;
    h->size = prop.size;
    h->mc = mc;
    h->opened = 1;
    const void* fns[] = {(const void*)k_allreduce_nvls, (const void*)k_reduce_scatter_nvls,
                         (const void*)k_allgather_nvls};
    int per_sm = 4;
    for (const void* f : fns) {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, 256, 0);
        per_sm = std::min(per_sm, n);
    }
    h->grid = std::max(1, per_sm) * num_sms();
    *out = h;
    return LHC_OK;
}

int lhc_nvls_bind(lhc_nvls* h, void** local_ptr, size_t* size) {
    if (!h || !h->opened || h->bound) return set_error(LHC_EINVAL, "not an open, unbound NVLS handle");
    auto cuMemCreate_ = DRV(cuMemCreate);
    auto cuMulticastBindMem_ = DRV(cuMulticastBindMem);
    auto cuMemAddressReserve_ = DRV(cuMemAddressReserve);
    auto cuMemMap_ = DRV(cuMemMap);
    auto cuMemSetAccess_ = DRV(cuMemSetAccess);
    if (!cuMemCreate_ || !cuMulticastBindMem_ || !cuMemAddressReserve_ || !cuMemMap_ || !cuMemSetAccess_)
        return set_error(LHC_ECOMM, "virtual memory driver entry points unavailable");
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = h->dev;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // as the multicast object
    // a failure part-way unwinds what was done (mappings, reservations, binding,
    // the allocation), leaving the handle open and unbound
    auto cuMemUnmap_ = DRV(cuMemUnmap);
    auto cuMemAddressFree_ = DRV(cuMemAddressFree);
    auto cuMemRelease_ = DRV(cuMemRelease);
    auto cuMulticastUnbind_ = DRV(cuMulticastUnbind);
    bool created = false, bound_mc = false, uc_res = false, uc_map = false, mc_res = false, mc_map = false;
    auto unwind = [&](int rc) {
        if (mc_map && cuMemUnmap_) cuMemUnmap_(h->mc_va, h->size);
        if (mc_res && cuMemAddressFree_) cuMemAddressFree_(h->mc_va, h->size);
        if (uc_map && cuMemUnmap_) cuMemUnmap_(h->uc_va, h->size);
        if (uc_res && cuMemAddressFree_) cuMemAddressFree_(h->uc_va, h->size);
        CUdevice cd;
        auto cuDeviceGet_ = DRV(cuDeviceGet);
        if (bound_mc && cuMulticastUnbind_ && cuDeviceGet_ && !cuDeviceGet_(&cd, h->dev))
            cuMulticastUnbind_(h->mc, cd, 0, h->size);
        if (created && cuMemRelease_) cuMemRelease_(h->mem);
        h->uc_va = h->mc_va = 0;
        h->mem = 0;
        return rc;
    };
    if (CUresult r = cuMemCreate_(&h->mem, h->size, &ap, 0)) return drv_err("cuMemCreate", r);
    created = true;
    if (CUresult r = cuMulticastBindMem_(h->mc, 0, h->mem, 0, h->size, 0)) return unwind(drv_err("cuMulticastBindMem", r));
    bound_mc = true;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = h->dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (CUresult r = cuMemAddressReserve_(&h->uc_va, h->size, 0, 0, 0)) return unwind(drv_err("cuMemAddressReserve", r));
    uc_res = true;
    if (CUresult r = cuMemMap_(h->uc_va, h->size, 0, h->mem, 0)) return unwind(drv_err("cuMemMap", r));
    uc_map = true;
    if (CUresult r = cuMemSetAccess_(h->uc_va, h->size, &acc, 1)) return unwind(drv_err("cuMemSetAccess", r));
    if (CUresult r = cuMemAddressReserve_(&h->mc_va, h->size, 0, 0, 0)) return unwind(drv_err("cuMemAddressReserve", r));
    mc_res = true;
    if (CUresult r = cuMemMap_(h->mc_va, h->size, 0, h->mc, 0)) return unwind(drv_err("cuMemMap(multicast)", r));
    mc_map = true;
    if (CUresult r = cuMemSetAccess_(h->mc_va, h->size, &acc, 1)) return unwind(drv_err("cuMemSetAccess(multicast)", r));
    if (cudaMemset((void*)h->uc_va, 0, h->size) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        return unwind(set_error(LHC_ECUDA, "clearing the NVLS buffer failed"));
    h->bound = 1;
    if (local_ptr) *local_ptr = (void*)h->uc_va;
    if (size) *size = h->size - kNvlsSig;
    return LHC_OK;
}

static int nvls_launch(lhc_nvls* h, const void* fn, NvArgs& A, void* stream, const char* what) {
    A.uc = (char*)h->uc_va;
    A.mc = (char*)h->mc_va;
    A.sig_uc = reinterpret_cast<uint32_t*>(h->uc_va + h->size - kNvlsSig);
    A.sig_mc = reinterpret_cast<uint32_t*>(h->mc_va + h->size - kNvlsSig);
    A.rank = h->rank;
    A.world = h->world;
    void* args[] = {(void*)&A};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(h->grid), dim3(256), args, 0, (cudaStream_t)stream);
    count_launch();
    if (e != cudaSuccess) return set_error(LHC_ECUDA, "%s launch: %s", what, cudaGetErrorString(e));
    return LHC_OK;
}

int sketch_allreduce_nvls(lhc_nvls* h, const lhc_params* p, void* stream) {
    if (!h || !h->bound) return set_error(LHC_EINVAL, "NVLS handle not bound");
    if (int rc = validate(p)) return rc;
    size_t b, y, sb, sy, s, t;
    layout(p, &b, &y, &sb, &sy, &s, &t);
    const uint64_t units = (y + p->c * sizeof(float)) / 16;
    if (units * 16 > h->size - kNvlsSig) return set_error(LHC_ECAPACITY, "NVLS buffer too small");
    reset_launches();
    NvArgs A{};
    A.lo = units * h->rank / h->world;
    A.hi = units * (h->rank + 1) / h->world;
    A.y_unit = y / 16;
    return nvls_launch(h, (const void*)k_allreduce_nvls, A, stream, "allreduce_nvls");
}

int sketch_reduce_scatter_nvls(lhc_nvls* h, const lhc_params* ps, uint64_t cap_items, void* stream) {
    if (!h || !h->bound) return set_error(LHC_EINVAL, "NVLS handle not bound");
    size_t slot = 0, y = 0, st = 0, ga = 0, sg = 0, t = 0;
    if (int rc = shard_layout(ps, h->world, cap_items, &slot, &y, &st, &ga, &sg, &t)) return rc;
    if (t > h->size - kNvlsSig) return set_error(LHC_ECAPACITY, "NVLS buffer too small for the shard layout");
    reset_launches();
    NvArgs A{};
    A.slot_units = slot / 16;
    A.y_unit = y / 16;
    return nvls_launch(h, (const void*)k_reduce_scatter_nvls, A, stream, "reduce_scatter_nvls");
}

int sketch_allgather_decoded_nvls(lhc_nvls* h, const lhc_params* ps, uint64_t cap_items,
                                  const uint32_t* idx, const float* val,
                                  const unsigned long long* n_items, uint64_t shard_width, uint32_t d,
                                  float* dense, void* stream) {
    if (!h || !h->bound) return set_error(LHC_EINVAL, "NVLS handle not bound");
    size_t slot = 0, y = 0, st = 0, ga = 0, sg = 0, t = 0;
    if (int rc = shard_layout(ps, h->world, cap_items, &slot, &y, &st, &ga, &sg, &t)) return rc;
    if (t > h->size - kNvlsSig) return set_error(LHC_ECAPACITY, "NVLS buffer too small for the shard layout");
    if (!idx || !val || !n_items || !dense) return set_error(LHC_EINVAL, "NULL argument");
    if (((uintptr_t)dense) & 15u) return set_error(LHC_EINVAL, "dense must be 16-byte aligned");
    if (shard_width == 0 || shard_width % 4 || (uint64_t)(h->world - 1) * shard_width >= d)
        return set_error(LHC_EINVAL, "shard_width must be a positive multiple of 4, every shard non-empty");
    reset_launches();
    if (h->world == 1) return LHC_OK;
    NvArgs A{};
    A.cap = (cap_items + 3) / 4 * 4;
    A.gather_off = ga;
    A.idx = idx;
    A.val = val;
    A.n_items = n_items;
    A.dense = dense;
    A.shard_width = shard_width;
    A.d = d;
    return nvls_launch(h, (const void*)k_allgather_nvls, A, stream, "allgather_nvls");
}

void lhc_nvls_destroy(lhc_nvls* h) {
    if (!h) return;
    auto cuMemUnmap_ = DRV(cuMemUnmap);
    auto cuMemAddressFree_ = DRV(cuMemAddressFree);
    auto cuMemRelease_ = DRV(cuMemRelease);
    auto cuMulticastUnbind_ = DRV(cuMulticastUnbind);
    auto cuDeviceGet_ = DRV(cuDeviceGet);
    cudaDeviceSynchronize();
    if (h->bound && cuMemUnmap_ && cuMemAddressFree_) {
        cuMemUnmap_(h->uc_va, h->size);
        cuMemUnmap_(h->mc_va, h->size);
        cuMemAddressFree_(h->uc_va, h->size);
        cuMemAddressFree_(h->mc_va, h->size);
    }
    CUdevice dev;
    if (h->bound && cuMulticastUnbind_ && cuDeviceGet_ && !cuDeviceGet_(&dev, h->dev))
        cuMulticastUnbind_(h->mc, dev, 0, h->size);
    if (cuMemRelease_) {
        if (h->bound) cuMemRelease_(h->mem);
        if (h->opened) cuMemRelease_(h->mc);
    }
    delete h;
}

}  // extern "C"
