// lhc_internal.cuh — shared device helpers of the sm_100a kernels (not part of the ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/lhc.h"

namespace lhc {

constexpr int kMaxK = 8;          // max Count Sketch hashes / Bloom probes
constexpr uint32_t kTile = 1024;  // coordinates per compress tile / query chunk

// Kernel-side view of lhc_params with the derived sizes precomputed on the host.
struct KParams {
    uint64_t seed;
    uint64_t c;        // cells
    uint64_t m;        // bits
    uint32_t d;
    uint32_t k;        // sketch hashes
    uint32_t kb;       // bloom probes
    uint32_t L;        // batch width
    uint32_t log2L;
    uint32_t nw;       // 32-bit words per row = L/32
    uint32_t log2nw;
    uint32_t S_Y;      // rows per sketch partition
    uint32_t S_B;      // rows per bloom partition
    uint32_t nrows;    // ceil(d / L)
    uint32_t exact;    // 1: the index is the exact bitmap, bit p <-> coordinate p
    uint32_t blocks;   // 0, or Count Sketch blocks: row i -> block i mod blocks
};

// ---------------------------------------------------------------------------
// Hash (reading R1, include/lhc.h header comment).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__host__ __device__ __forceinline__ uint64_t hash_row(uint64_t seed, uint32_t dom, uint32_t j,
                                                      uint64_t i) {
    uint64_t key = ((uint64_t)dom << 56) | ((uint64_t)j << 48) | i;
    return mix64(seed ^ mix64(key + 0x9E3779B97F4A7C15ull));
}

// Packed row map: x = absolute row (partition j), y = bias | (sign<0) << 31.
__host__ __device__ __forceinline__ uint2 row_map(uint64_t seed, uint32_t dom, uint32_t j,
                                                  uint64_t i, uint32_t S, uint32_t L) {
    uint64_t H = hash_row(seed, dom, j, i);
    uint32_t row = j * S + (uint32_t)(((H >> 32) * (uint64_t)S) >> 32);
    uint32_t y = (uint32_t)(H & (uint64_t)(L - 1)) | ((uint32_t)((H >> 16) & 1u) << 31);
    return make_uint2(row, y);
}

// Row map of domain dom (0 = Count Sketch, 1 = index) for input row i under probe j.
// With the exact bitmap index ("one bit per parameter") the index row of
// input row i is row i itself, unrotated.
__host__ __device__ __forceinline__ uint2 dom_map(const KParams& P, uint32_t dom, uint32_t j,
                                                  uint64_t i) {
    if (dom == 1 && P.exact) return make_uint2((uint32_t)i, 0u);
    uint2 mp = row_map(P.seed, dom, j, i, dom ? P.S_B : P.S_Y, P.L);
    if (dom == 0 && P.blocks) mp.x += (uint32_t)(i % P.blocks) * P.k * P.S_Y;  // block base
    return mp;
}

__device__ __forceinline__ uint32_t map_bias(uint2 mp) { return mp.y & 0x7fffffffu; }
__device__ __forceinline__ float map_sign(uint2 mp) { return (mp.y >> 31) ? -1.0f : 1.0f; }

// Decode state of one Count Sketch cell, 16 bytes so one sector serves both.
//   key = sum over unpeeled candidates p in the cell of (2^32 + p) (p = coordinate):
//         the degree is key >> 32 exactly whenever it is 0 or 1 (then the
//         coordinate is (uint32)key), and >= 2 whenever the true degree is >= 2
//         (degree < 2^31 always holds since degree <= rows mapped to a cell < 2^27).
//   R   = residual counter.
struct __align__(16) CellState {
    unsigned long long key;
    float R;
    uint32_t pad;
};

// Compact decode state (8 bytes): key = sum over the cell's unpeeled candidates of
// (2^24 + input row i); degree 0 or 1 is exact (then the low 24 bits are the row
// of the only candidate, its column follows from the cell's column and the row's
// bias), degree >= 2 reads as >= 2 while degree * (2^24 + rows) < 2^32.  Used when
// the state does not fit in L2, input rows < 2^22 and no destination row receives
// more than kCompactMaxDeg input rows (checked on the device).
struct __align__(8) CellC {
    uint32_t key;
    float R;
};
constexpr uint32_t kCompactMaxDeg = 200;

// Control block of one decompress call (workspace, zeroed per call).
struct Ctrl {
    unsigned long long n_cand;  // written by the query scan
    uint32_t overflow;
    // Per-round counter, triple-buffered by round index r % 3: round r appends its
    // new frontier entries after the current segment through the low 32 bits of
    // rc[r % 3] and counts its peels in the high 32 bits; every block reads it
    // (one 64-bit load) after the grid barrier that ends round r, when it is
    // final, and block 0 resets it during round r + 2, when nobody uses it.
    unsigned long long rc[3];
    uint32_t rounds_dbg;
    uint32_t compact_fail;  // set by k_build_cells<compact> when a row is too full
    uint32_t blk_fail;      // set by k_peel_blocked when a block cannot be peeled in place
    uint32_t blk_done;      // blocks finished (the last one writes the stats)
    unsigned long long blk_peeled;
    uint32_t blk_rounds;
    uint32_t xl_n[2], yl_n[2];  // row peel worklist counts, by round parity
    uint32_t ymax_bits;         // row peel: max |Y| (fp32 bits), sets the fixed-point grid
    uint32_t fx_overflow;       // row peel: a deduction exceeded the fixed-point range
    // instrumentation (device globaltimer ns): t[0..3] phase starts, t[3 + r] start of
    // round r, t[kCtrlTimes-1] end of rounds; fsize[r] = queue segment of round r
    unsigned long long t[128];
    uint32_t fsize[128];
    unsigned long long tproc[128];  // per round: latest block finishing its entries
    unsigned long long tflush[128]; // per round: latest block finishing its appends
    unsigned long long dbg[4][128]; // row peel (LHC_ROWS_TIMING): per-round maxima of X / Y work items
};
constexpr int kCtrlTimes = 128;

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Sub-allocation of the decompress workspace.
struct WsLayout {
    size_t tabS, gmask, cta_total, cells, claim, frontier, dense, dst_off, pair_pos, dst_list, ctrl,
        rowoff, vlog, vfill, claim_k, dmark, dst_sorted, ymark, xl, yl, total;
    uint32_t nchunks;
};


inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace lhc
