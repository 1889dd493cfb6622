// peel.cu — Phase II steps 2-3 of Alg. 1 on sm_100a: the frontier-
// based parallel peeling decoder and the Count Sketch median
// fallback for what peeling cannot reach (footnote P:L193).
//
// One cooperative, persistent kernel (one CTA per SM slot, grid-wide barriers
// between phases) so that the whole round loop runs on the device with no host
// round trips:
//   init     cell state {key = 0, R = Y}; claim[s] = unclaimed
//   insert   every candidate s adds (2^32 + s) to the key of its k cells
//            (one 64-bit atomic per incidence: degree and slot sum together)
//   F0       every cell of degree one is appended to the frontier queue
//   rounds   (synchronous, reading R10) every frontier cell that is still pure
//            names its candidate s = low 32 bits of key ("mapped by only one
//            non-zero parameter"); the first claimer wins (atomicCAS on
//            claim[s]), reads val = sign * R[cell], and subtracts sign_j * val and
//            (2^32 + s) from all k cells of s ("deducting Y_h_j(i) by
//            g_j(i)*X_i"); a cell whose degree drops from 2 to 1 is
//            appended to the queue for the next round.  A round only consumes the
//            queue segment appended by the previous round, so rounds (and the set
//            of candidates peeled per round) are exactly the synchronous ones.
//   finalize unpeeled candidates take the median over j of sign_j * R.
// Pushes are aggregated per CTA in shared memory (one global atomic per CTA per
// round); every cell enters the queue at most once, so the queue holds c entries.
#include <cooperative_groups.h>

#include "launch.h"

namespace cg = cooperative_groups;

namespace lhc {

constexpr int kPeelThreads = 256;
constexpr uint32_t kUnclaimed = 0xffffffffu;

__device__ __forceinline__ uint64_t cand_cell(const KParams& P, const uint2* __restrict__ tabS,
                                              uint32_t p, uint32_t j, float* g) {
    const uint64_t i = p >> P.log2L;
    const uint32_t t = p & (P.L - 1);
    const uint2 mp = __ldg(tabS + i * P.k + j);
    *g = map_sign(mp);
    return ((uint64_t)mp.x << P.log2L) + ((t + map_bias(mp)) & (P.L - 1));
}

__device__ __forceinline__ unsigned long long ld_key(const CellState* c) {
    return __ldcg(&c->key);
}
__device__ __forceinline__ float ld_R(const CellState* c) { return __ldcg(&c->R); }

// Block-aggregated append of the (up to kMaxK per thread) cells in sh_q to the
// queue segment that starts at seg_base, through the round's counter qcnt.
__device__ __forceinline__ void flush_queue(uint32_t* sh_q, uint32_t* sh_n, uint32_t* sh_base,
                                            uint32_t* frontier, uint32_t seg_base, uint32_t* qcnt) {
    __syncthreads();
    const uint32_t n = *sh_n;
    if (threadIdx.x == 0 && n) *sh_base = seg_base + atomicAdd(qcnt, n);
    __syncthreads();
    for (uint32_t a = threadIdx.x; a < n; a += blockDim.x) frontier[*sh_base + a] = sh_q[a];
    __syncthreads();
    if (threadIdx.x == 0) *sh_n = 0;
    __syncthreads();
}

__global__ void __launch_bounds__(kPeelThreads)
k_peel(KParams P, const float* __restrict__ counters, const uint2* __restrict__ tabS,
       const uint32_t* __restrict__ cand, uint64_t cap, CellState* cells, uint32_t* claim,
       uint32_t* frontier, Ctrl* ctrl, float* __restrict__ out_val,
       uint8_t* __restrict__ out_peeled, lhc_stats* stats) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t sh_q[kPeelThreads * kMaxK];
    __shared__ uint32_t sh_n, sh_base, sh_peeled;

    const uint64_t n_c = *(volatile unsigned long long*)&ctrl->n_cand;
    if (n_c > cap) {  // overflow: nothing is peeled (stats.overflow set by the query scan)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            stats->n_peeled = 0;
            stats->rounds = 0;
            stats->success = 0;
        }
        return;
    }
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    if (threadIdx.x == 0) { sh_n = 0; sh_peeled = 0; }

    // init
    for (uint64_t e = gtid; e < P.c; e += gstride) {
        CellState cs;
        cs.key = 0ull;
        cs.R = __ldcs(counters + e);
        cs.pad = 0u;
        cells[e] = cs;
    }
    for (uint64_t s = gtid; s < n_c; s += gstride) claim[s] = kUnclaimed;
    grid.sync();

    // insert: degree and slot sum of every cell
    for (uint64_t s = gtid; s < n_c; s += gstride) {
        const uint32_t p = cand[s];
        for (uint32_t j = 0; j < P.k; j++) {
            float g;
            const uint64_t e = cand_cell(P, tabS, p, j, &g);
            atomicAdd(&cells[e].key, (1ull << 32) + s);
        }
    }
    grid.sync();

    // F0 ("round 0"): cells of degree one, appended through qcnt[0]
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < P.c; base += gstride) {
        const uint64_t e = base + threadIdx.x;
        if (e < P.c && (ld_key(cells + e) >> 32) == 1ull) sh_q[atomicAdd(&sh_n, 1u)] = (uint32_t)e;
        flush_queue(sh_q, &sh_n, &sh_base, frontier, 0u, &ctrl->qcnt[0]);
    }
    grid.sync();

    uint32_t f_begin = 0;
    uint32_t f_end = *(volatile uint32_t*)&ctrl->qcnt[0];
    uint32_t n_peeled = 0, rounds = 0;
    for (uint32_t r = 1; f_begin < f_end; r++) {
        uint32_t* qcnt = &ctrl->qcnt[r % 3];
        uint32_t* pcnt = &ctrl->pcnt[r % 3];
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // counters of round r + 1 (last used r - 2)
            ctrl->qcnt[(r + 1) % 3] = 0;
            ctrl->pcnt[(r + 1) % 3] = 0;
        }
        for (uint64_t base = f_begin + blockIdx.x * (uint64_t)blockDim.x; base < f_end;
             base += gstride) {
            const uint64_t f = base + threadIdx.x;
            if (f < f_end) {
                const uint32_t e = frontier[f];
                const unsigned long long key = ld_key(cells + e);
                if ((key >> 32) == 1ull) {
                    const uint32_t s = (uint32_t)key;
                    if (atomicCAS(claim + s, kUnclaimed, 1u) == kUnclaimed) {
                        const uint32_t p = cand[s];
                        float gs[kMaxK];
                        uint64_t es[kMaxK];
                        float ge = 1.f;
                        for (uint32_t j = 0; j < P.k; j++) {
                            es[j] = cand_cell(P, tabS, p, j, &gs[j]);
                            if (es[j] == e) ge = gs[j];
                        }
                        const float val = ge * ld_R(cells + e);
                        out_val[s] = val;
                        atomicAdd(&sh_peeled, 1u);
                        for (uint32_t j = 0; j < P.k; j++) {
                            atomicAdd(&cells[es[j]].R, -gs[j] * val);
                            const unsigned long long old =
                                atomicAdd(&cells[es[j]].key, 0ull - ((1ull << 32) + s));
                            if ((old >> 32) == 2ull) sh_q[atomicAdd(&sh_n, 1u)] = (uint32_t)es[j];
                        }
                    }
                }
            }
            flush_queue(sh_q, &sh_n, &sh_base, frontier, f_end, qcnt);
        }
        if (threadIdx.x == 0 && sh_peeled) {
            atomicAdd(pcnt, sh_peeled);
            sh_peeled = 0;
        }
        grid.sync();
        const uint32_t np = *(volatile uint32_t*)pcnt;
        f_begin = f_end;
        f_end += *(volatile uint32_t*)qcnt;
        n_peeled += np;
        if (np) rounds++;
    }

    // finalize: median estimate of unpeeled candidates
    for (uint64_t s = gtid; s < n_c; s += gstride) {
        const bool pe = __ldcg(claim + s) != kUnclaimed;
        out_peeled[s] = pe ? 1 : 0;
        if (!pe) {
            const uint32_t p = cand[s];
            float v[kMaxK];
            for (uint32_t j = 0; j < P.k; j++) {
                float g;
                const uint64_t e = cand_cell(P, tabS, p, j, &g);
                v[j] = g * ld_R(cells + e);
            }
            for (uint32_t a = 1; a < P.k; a++) {  // insertion sort of <= 8 values
                float x = v[a];
                int b = (int)a - 1;
                while (b >= 0 && v[b] > x) { v[b + 1] = v[b]; b--; }
                v[b + 1] = x;
            }
            out_val[s] = (P.k & 1) ? v[P.k / 2] : 0.5f * (v[P.k / 2 - 1] + v[P.k / 2]);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        stats->n_peeled = n_peeled;
        stats->rounds = rounds;
        stats->success = (uint64_t)n_peeled == n_c ? 1 : 0;
    }
}

static int peel_grid(int dev) {
    static int cached[64] = {0};
    if (dev < 64 && cached[dev]) return cached[dev];
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peel, kPeelThreads, 0);
    int g = std::max(1, per_sm) * num_sms();
    if (dev < 64) cached[dev] = g;
    return g;
}

cudaError_t launch_peel(const KParams& P, const float* counters, const uint2* tabS,
                        const uint32_t* cand, uint64_t cap, CellState* cells, uint32_t* claim,
                        uint32_t* frontier, Ctrl* ctrl, float* out_val, uint8_t* out_peeled,
                        lhc_stats* stats, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int grid = peel_grid(dev);
    KParams Pc = P;
    void* args[] = {(void*)&Pc,     (void*)&counters, (void*)&tabS,   (void*)&cand,
                    (void*)&cap,    (void*)&cells,    (void*)&claim,  (void*)&frontier,
                    (void*)&ctrl,   (void*)&out_val,  (void*)&out_peeled, (void*)&stats};
    cudaError_t err = cudaLaunchCooperativeKernel((const void*)k_peel, dim3(grid),
                                                  dim3(kPeelThreads), args, 0, s);
    count_launch();
    return err;
}

}  // namespace lhc
