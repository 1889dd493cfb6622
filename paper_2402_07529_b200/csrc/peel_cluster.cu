// peel_cluster.cu — Phase II steps 2-3 for a blocked Count Sketch with
// large blocks ("O(1) iterations by splitting the Count Sketch into multiple
// blocks of fixed size"; reading R25), one block per thread-block CLUSTER whose
// CTAs hold the block's decode state in their shared memory (distributed shared
// memory, DSMEM): the peeling rounds never touch L2 or HBM.
//
// Input row i hashes only into block i mod B, so blocks peel independently.  A
// cluster of CS CTAs (CS = 16 where the block's rows divide, else 8/4/2) takes
// blocks b = cluster, cluster + clusters, ...; CTA r of the cluster holds
//   * the cells [r cpc, (r+1) cpc) of the block (cpc = block cells / CS): the key
//     sum (2^24 + id) over the cell's remaining candidates (id = t L + col, t the
//     input row's index in the block) and the residual R, in shared memory;
//   * the block's input rows t = r, r + CS, ...: their candidate masks (from the
//     query), claim bits, first candidate slots and Count Sketch row maps.
// Phases of a block, separated by cluster barriers:
//   load     counters → R, keys = 0, masks / slots / maps of the CTA's rows
//   bound    input rows per destination row ≤ kClMaxRows (the key's degree byte
//            cannot carry); else the cluster flags blk_fail and the global peel
//            decodes the sketch instead (device-checked fallback)
//   insert   every candidate adds its key to its k cells (DSMEM atomics)
//   rounds   synchronous (reading R10): a cell whose key reads degree one names
//            its only candidate, which is claimed (first claimer wins), takes
//            val = g_j R[cell] ("mapped by only one non-zero parameter")
//            and is deducted from its other cells ("deducting ... by g_j(i) X_i");
//            a round examines only the cells the previous round brought to degree
//            one (all cells in round 1); the value lands in the dense output
//   final    unpeeled candidates take the median over j of g_j R; values
//            and flags are written at their slots
// Rounds are max-combined over blocks, as in the oracle (block-diagonal incidence).
#include <cooperative_groups.h>

#include "launch.h"

namespace cg = cooperative_groups;

namespace lhc {

constexpr int kClThreads = 1024;
constexpr uint32_t kClMaxRows = 127;    // listed input rows per destination row (degree byte)
constexpr uint32_t kClCellsPerThread = 32;
#ifndef LHC_CL_TIMING
#define LHC_CL_TIMING 0
#endif

struct ClArgs {
    KParams P;
    const float* counters;
    const uint2* tabS;
    const uint32_t* gmask;
    const uint32_t* rowoff;
    float* dense;        // zeroed by the launcher
    uint64_t cap;
    float* out_val;
    uint8_t* out_peeled;
    Ctrl* ctrl;
    lhc_stats* stats;
    uint32_t cs;         // CTAs per cluster
    uint32_t cpc;        // cells per CTA
    uint32_t rpc;        // input rows per CTA (upper bound)
};

struct ClLayout {
    size_t key, R, touch, mask, claim, wpre, first, maps, rpd, words;
};

__host__ __device__ inline ClLayout cl_layout(const KParams& P, uint32_t cs, uint32_t cpc, uint32_t rpc) {
    ClLayout l{};
    size_t o = 0;
    l.key = o;   o += cpc;
    l.R = o;     o += cpc;
    l.touch = o; o += 2 * ((cpc + 31) / 32);
    l.mask = o;  o += (size_t)rpc * P.nw;
    l.claim = o; o += (size_t)rpc * P.nw;
    l.wpre = o;  o += (size_t)rpc * P.nw;
    l.first = o; o += rpc;
    o = (o + 1) & ~(size_t)1;
    l.maps = o;  o += 2 * (size_t)rpc * P.k;
    l.rpd = o;   o += (size_t)P.k * P.S_Y / cs;
    l.words = o;
    return l;
}

template <int KT>
__global__ void __launch_bounds__(kClThreads, 1) k_peel_cluster(const __grid_constant__ ClArgs A) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ uint32_t sh_warp[32];
    __shared__ uint32_t sh_flag[4];   // [0..1] round counters (CTA 0), [2] fail, [3] broadcast
    __shared__ uint32_t sh_peeled;
    cg::cluster_group cluster = cg::this_cluster();
    const KParams& P = A.P;
    constexpr uint32_t NJ = KT ? KT : kMaxK;
    const uint32_t k = KT ? (uint32_t)KT : P.k;
    const uint32_t L = P.L, nw = P.nw, CS = A.cs, cpc = A.cpc;
    const uint32_t r = cluster.block_rank();
    const uint32_t SL = P.S_Y * L;                 // cells per partition of a block
    const uint32_t cb = k * SL;                     // cells per block
    const uint32_t rows_per_cta = k * P.S_Y / CS;   // destination rows per CTA
    const ClLayout ly = cl_layout(P, CS, cpc, A.rpc);
    uint32_t* key = sm + ly.key;
    float* R = reinterpret_cast<float*>(sm + ly.R);
    uint32_t* touch = sm + ly.touch;
    uint32_t* mask = sm + ly.mask;
    uint32_t* claim = sm + ly.claim;
    uint32_t* wpre = sm + ly.wpre;
    uint32_t* first = sm + ly.first;
    uint2* maps = reinterpret_cast<uint2*>(sm + ly.maps);
    uint32_t* rpd = sm + ly.rpd;
    const uint32_t ncw = (cpc + 31) / 32;
    const uint32_t tid = threadIdx.x;
    const uint32_t cpt = (cpc + blockDim.x - 1) / blockDim.x;  // cells per thread (<= 32)
    const uint32_t n_clusters = gridDim.x / CS;
    const uint32_t cid = blockIdx.x / CS;

    const uint64_t n_c = *(volatile unsigned long long*)&A.ctrl->n_cand;
    if (n_c > A.cap) return;  // overflow: the stats were set by the query (uniform)

    for (uint32_t b = cid; b < P.blocks; b += n_clusters) {
        const uint32_t nrb = b < P.nrows ? (P.nrows - 1 - b) / P.blocks + 1 : 0;  // rows of block b
        const uint32_t nmy = nrb > r ? (nrb - 1 - r) / CS + 1 : 0;                // this CTA's rows
        const uint64_t cbase = (uint64_t)b * cb + (uint64_t)r * cpc;             // first cell of this CTA
        const uint32_t rbase = b * k * P.S_Y;                                     // first destination row
        const bool tm = LHC_CL_TIMING && tid == 0 && r == 0;
        unsigned long long t0 = tm ? globaltimer() : 0ull, t1 = 0, t2 = 0, t3 = 0;
        if (tid == 0) {
            sh_peeled = 0;
            sh_flag[0] = sh_flag[1] = sh_flag[2] = 0;
        }
        // ---- load
        for (uint32_t e = tid; e < cpc; e += blockDim.x) {
            key[e] = 0u;
            R[e] = __ldcs(A.counters + cbase + e);
        }
        for (uint32_t a = tid; a < 2 * ncw; a += blockDim.x) touch[a] = a < ncw ? ~0u : 0u;
        for (uint32_t a = tid; a < rows_per_cta; a += blockDim.x) rpd[a] = 0u;
        for (uint32_t a = tid; a < nmy * nw; a += blockDim.x) {
            const uint32_t u = a / nw, w = a - u * nw;
            const uint64_t i = b + (uint64_t)(r + u * CS) * P.blocks;
            mask[a] = __ldcg(A.gmask + i * nw + w);
            claim[a] = 0u;
        }
        for (uint32_t u = tid; u < nmy; u += blockDim.x)
            first[u] = __ldcg(A.rowoff + b + (uint64_t)(r + u * CS) * P.blocks);
        for (uint32_t a = tid; a < nmy * k; a += blockDim.x) {
            const uint32_t u = a / k, j = a - u * k;
            maps[a] = __ldg(&A.tabS[(b + (uint64_t)(r + u * CS) * P.blocks) * k + j]);
        }
        __syncthreads();
        // exclusive prefix of the candidates over this CTA's words (slots at the end)
        {
            const uint32_t nwords = nmy * nw;
            const uint32_t per = (nwords + blockDim.x - 1) / blockDim.x;
            const uint32_t w0 = tid * per, w1 = min(nwords, w0 + per);
            uint32_t sum = 0;
            for (uint32_t a = w0; a < w1; a++) sum += __popc(mask[a]);
            const uint32_t lane = tid & 31, warp = tid >> 5;
            uint32_t x = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            if (lane == 31) sh_warp[warp] = x;
            __syncthreads();
            if (tid == 0) {
                uint32_t run = 0;
                for (uint32_t v = 0; v < blockDim.x / 32; v++) {
                    const uint32_t c = sh_warp[v];
                    sh_warp[v] = run;
                    run += c;
                }
            }
            __syncthreads();
            uint32_t run = sh_warp[warp] + x - sum;
            for (uint32_t a = w0; a < w1; a++) {
                wpre[a] = run;
                run += __popc(mask[a]);
            }
        }
        cluster.sync();  // every CTA of the cluster loaded before any remote access
        // ---- degree bound: input rows per destination row of the block
        for (uint32_t a = tid; a < nmy * k; a += blockDim.x) {
            const uint32_t D = maps[a].x - rbase;
            atomicAdd(cluster.map_shared_rank(rpd, D / rows_per_cta) + D % rows_per_cta, 1u);
        }
        cluster.sync();
        {
            uint32_t bad = 0;
            for (uint32_t a = tid; a < rows_per_cta; a += blockDim.x) bad |= rpd[a] > kClMaxRows;
            bad = __syncthreads_or(bad);
            if (tid == 0 && bad) atomicOr(cluster.map_shared_rank(sh_flag, 0) + 2, 1u);
        }
        cluster.sync();
        if (tid == 0) sh_flag[3] = *(volatile uint32_t*)(cluster.map_shared_rank(sh_flag, 0) + 2);
        __syncthreads();
        if (sh_flag[3]) {  // uniform over the cluster
            if (tid == 0 && r == 0) atomicOr(&A.ctrl->blk_fail, 1u);
            cluster.sync();
            continue;
        }
        if (tm) t1 = globaltimer();
        // ---- insert: every candidate of this CTA's rows into its k cells
        for (uint32_t a = tid; a < nmy * nw; a += blockDim.x) {
            const uint32_t u = a / nw, w = a - u * nw;
            uint32_t mm = mask[a];
            if (!mm) continue;
            const uint32_t t = r + u * CS;
            for (uint32_t j = 0; j < k; j++) {
                const uint2 mp = maps[u * k + j];
                const uint32_t rowl = (mp.x - rbase) * L, bias = map_bias(mp);
                for (uint32_t m2 = mm; m2; m2 &= m2 - 1) {
                    const uint32_t col = 32 * w + (__ffs(m2) - 1);
                    const uint32_t e = rowl + ((col + bias) & (L - 1));
                    atomicAdd(cluster.map_shared_rank(key, e / cpc) + e % cpc, (1u << 24) + t * L + col);
                }
            }
        }
        cluster.sync();
        if (tm) t2 = globaltimer();
        // ---- synchronous rounds
        uint32_t rounds = 0;
        for (uint32_t cur = 0, rd = 0;; cur ^= 1u, rd++) {
            uint32_t* tc = touch + cur * ncw;
            if (tid == 0 && r == 0) sh_flag[(rd + 1) & 1] = 0u;  // last read in round rd - 1
            // A: pure cells among the marked ones (thread: cells [tid cpt, (tid+1) cpt))
            const uint32_t c0 = tid * cpt;
            uint32_t pure = 0u;
            if (c0 < cpc) {
                const uint32_t w0 = c0 >> 5, s0 = c0 & 31;
                uint64_t bits = (uint64_t)tc[w0] | (w0 + 1 < ncw ? (uint64_t)tc[w0 + 1] << 32 : 0ull);
                uint32_t cand = (uint32_t)(bits >> s0) & (cpt >= 32 ? ~0u : ((1u << cpt) - 1u));
                for (; cand; cand &= cand - 1) {
                    const uint32_t s2 = __ffs(cand) - 1;
                    if (c0 + s2 < cpc && (key[c0 + s2] >> 24) == 1u) pure |= 1u << s2;
                }
            }
            const uint32_t any = __syncthreads_or(pure != 0u);
            if (tid == 0 && any) atomicAdd(cluster.map_shared_rank(sh_flag, 0) + (rd & 1), 1u);
            cluster.sync();
            if (tid == 0) sh_flag[3] = *(volatile uint32_t*)(cluster.map_shared_rank(sh_flag, 0) + (rd & 1));
            for (uint32_t a = tid; a < ncw; a += blockDim.x) tc[a] = 0u;  // read: free for round rd + 2
            __syncthreads();
            if (!sh_flag[3]) break;  // no pure cell in the cluster's block (uniform)
            rounds++;
            // B: peel them
            uint32_t my_peeled = 0;
            for (uint32_t pm = pure; pm; pm &= pm - 1) {
                const uint32_t e = c0 + (__ffs(pm) - 1);
                const uint32_t kv = key[e];
                if ((kv >> 24) != 1u) continue;
                const uint32_t id = kv & 0xffffffu;
                const uint32_t t = id / L, col = id - t * L, w = col >> 5, bit = 1u << (col & 31);
                const uint32_t ro = t % CS, u = t / CS;
                if (atomicOr(cluster.map_shared_rank(claim, ro) + u * nw + w, bit) & bit) continue;
                const uint64_t i = b + (uint64_t)t * P.blocks;
                const uint32_t je = (r * cpc + e) / SL;
                uint2 mp[NJ];
#pragma unroll
                for (uint32_t j = 0; j < NJ; j++) {
                    if (!KT && j >= k) break;
                    mp[j] = dom_map(P, 0, j, i);
                }
                float ge = 1.f;
#pragma unroll
                for (uint32_t j = 0; j < NJ; j++)
                    if (j == je) ge = map_sign(mp[j]);
                const float val = ge * R[e];
                A.dense[(i << P.log2L) + col] = val;
#pragma unroll
                for (uint32_t j = 0; j < NJ; j++) {
                    if ((!KT && j >= k) || j == je) continue;
                    const uint32_t ej = (mp[j].x - rbase) * L + ((col + map_bias(mp[j])) & (L - 1));
                    const uint32_t oj = ej / cpc, lj = ej % cpc;
                    atomicAdd(cluster.map_shared_rank(R, oj) + lj, -map_sign(mp[j]) * val);
                    const uint32_t one = (1u << 24) + id;
                    const uint32_t now = atomicSub(cluster.map_shared_rank(key, oj) + lj, one) - one;
                    if ((now >> 24) == 1u)
                        atomicOr(cluster.map_shared_rank(touch, oj) + (cur ^ 1u) * ncw + (lj >> 5), 1u << (lj & 31));
                }
                my_peeled++;
            }
            if (my_peeled) atomicAdd(&sh_peeled, my_peeled);
            cluster.sync();  // the round's deductions and marks are visible cluster-wide
        }
        if (tm) t3 = globaltimer();
        // ---- finalize: the CTA's rows — flags, values, medians of the unpeeled
        for (uint32_t a = tid; a < nmy * nw; a += blockDim.x) {
            uint32_t mm = mask[a];
            if (!mm) continue;
            const uint32_t u = a / nw, w = a - u * nw;
            const uint32_t t = r + u * CS;
            const uint64_t i = b + (uint64_t)t * P.blocks;
            const uint32_t cl = claim[a];
            const uint64_t slot0 = (uint64_t)first[u] + wpre[a] - wpre[u * nw];
            for (uint32_t q = 0; mm; mm &= mm - 1, q++) {
                const uint32_t c = __ffs(mm) - 1, col = 32 * w + c;
                const uint64_t p = (i << P.log2L) + col;
                const bool pe = (cl >> c) & 1u;
                float val;
                if (pe) {
                    val = __ldcg(A.dense + p);
                } else {
                    float v[NJ];
                    for (uint32_t j = 0; j < k; j++) {
                        const uint2 mp = maps[u * k + j];
                        const uint32_t ej = (mp.x - rbase) * L + ((col + map_bias(mp)) & (L - 1));
                        v[j] = map_sign(mp) * *cluster.map_shared_rank(R + ej % cpc, ej / cpc);
                    }
                    for (uint32_t x = 1; x < k; x++) {  // insertion sort of <= 8 values
                        const float y = v[x];
                        int z = (int)x - 1;
                        while (z >= 0 && v[z] > y) { v[z + 1] = v[z]; z--; }
                        v[z + 1] = y;
                    }
                    val = (k & 1) ? v[k / 2] : 0.5f * (v[k / 2 - 1] + v[k / 2]);
                    A.dense[p] = val;
                }
                A.out_val[slot0 + q] = val;
                A.out_peeled[slot0 + q] = pe ? 1 : 0;
            }
        }
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&A.ctrl->blk_peeled, (unsigned long long)sh_peeled);
            if (r == 0) atomicMax(&A.ctrl->blk_rounds, rounds);
        }
        if (tm) {  // debug: summed phase durations (ns) of the clusters' CTA 0 in ctrl->t[8..12]
            const unsigned long long t4 = globaltimer();
            atomicAdd(&A.ctrl->t[8], t1 - t0);
            atomicAdd(&A.ctrl->t[9], t2 - t1);
            atomicAdd(&A.ctrl->t[10], t3 - t2);
            atomicAdd(&A.ctrl->t[11], t4 - t3);
            atomicAdd(&A.ctrl->t[12], 1ull);
        }
        cluster.sync();  // no CTA still reads this block's shared memory remotely
    }
    // the last CTA to finish writes the stats
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(&A.ctrl->blk_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && tid == 0 && !*(volatile uint32_t*)&A.ctrl->blk_fail) {
        const unsigned long long np = *(volatile unsigned long long*)&A.ctrl->blk_peeled;
        A.stats->n_peeled = np;
        A.stats->rounds = *(volatile uint32_t*)&A.ctrl->blk_rounds;
        A.stats->success = np == n_c ? 1 : 0;
        A.stats->entries = 0;
    }
}

static uint32_t cl_rows_per_block(const KParams& P) {
    return P.blocks ? (P.nrows + P.blocks - 1) / P.blocks : 0;
}

// Cluster size for a blocked sketch (0: the cluster peel does not apply): the
// largest of 16 / 8 / 4 / 2 that divides the block's destination rows and leaves
// at most 32 cells per thread and a shared-memory footprint within the opt-in.
uint32_t peel_cluster_size(const KParams& P) {
    if (!P.blocks || P.nrows == 0) return 0;
    if ((uint64_t)cl_rows_per_block(P) * P.L >= (1u << 24)) return 0;  // 24-bit ids
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    for (uint32_t cs : {16u, 8u, 4u, 2u}) {
        if ((P.k * P.S_Y) % cs) continue;
        const uint32_t cpc = P.k * P.S_Y * P.L / cs;
        if (cpc > (uint32_t)kClThreads * kClCellsPerThread) continue;
        if (cpc < (uint32_t)kClThreads) continue;  // blocks small enough for one CTA: k_peel_blocked
        const uint32_t rpc = (cl_rows_per_block(P) + cs - 1) / cs;
        const size_t bytes = cl_layout(P, cs, cpc, rpc).words * 4;
        if (bytes + 1024 <= (size_t)optin) return cs;
    }
    return 0;
}

template <int KT>
static cudaError_t launch_cluster(const ClArgs& A, size_t smem, cudaStream_t s) {
    auto fn = k_peel_cluster<KT>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (A.cs > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = A.cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(A.cs);
    int max_clusters = 0;
    cudaOccupancyMaxActiveClusters(&max_clusters, (const void*)fn, &cfg);
    const uint32_t nclus = (uint32_t)std::max(1, std::min<int>(max_clusters, (int)A.P.blocks));
    cfg.gridDim = dim3(nclus * A.cs);
    return cudaLaunchKernelEx(&cfg, fn, A);
}

cudaError_t launch_peel_cluster(const KParams& P, uint32_t cs, const float* counters, const uint2* tabS,
                                const uint32_t* gmask, const uint32_t* rowoff, float* dense,
                                uint64_t cap, float* out_val, uint8_t* out_peeled, Ctrl* ctrl,
                                lhc_stats* stats, cudaStream_t s) {
    ClArgs A{};
    A.P = P;
    A.counters = counters;
    A.tabS = tabS;
    A.gmask = gmask;
    A.rowoff = rowoff;
    A.dense = dense;
    A.cap = cap;
    A.out_val = out_val;
    A.out_peeled = out_peeled;
    A.ctrl = ctrl;
    A.stats = stats;
    A.cs = cs;
    A.cpc = P.k * P.S_Y * P.L / cs;
    A.rpc = (cl_rows_per_block(P) + cs - 1) / cs;
    const size_t smem = cl_layout(P, cs, A.cpc, A.rpc).words * 4;
    // the dense output is zeroed first: the peel writes only candidates' values
    cudaMemsetAsync(dense, 0, (size_t)P.d * sizeof(float), s);
    cudaError_t e = P.k == 3 ? launch_cluster<3>(A, smem, s) : launch_cluster<0>(A, smem, s);
    count_launch();
    return e;
}

}  // namespace lhc
