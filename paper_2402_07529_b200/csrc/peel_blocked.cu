// peel_blocked.cu — Phase II steps 2-3 for a blocked Count Sketch
// ("O(1) iterations by splitting the Count Sketch into multiple blocks of
// fixed size"; reading R25): input row i hashes only into block i mod B, so the
// peeling of different blocks is independent.  One CTA peels one block entirely
// in shared memory:
//   load   the block's counters (R), the query masks of its input rows and their
//          first candidate slots (from the query), and zero its dense ranges
//   insert every candidate p of the block adds (2^24 + local id) to the 32-bit key
//          of each of its k cells (shared-memory atomics; the degree is key >> 24,
//          exact whenever it is 0 or 1; the per-destination-row row counts are
//          checked first so the degree cannot overflow 8 bits)
//   rounds synchronous (reading R10): every thread scans its cells for degree 1
//          into a register bitmask, __syncthreads, then peels them — claim bit
//          (first claimer wins), val = sign * R, subtract from the other cells —
//          __syncthreads; the rounds end when no cell of the block is pure
//   final  median over j of sign_j * R for the candidates peeling did not reach
//          (P:L155); values land in out_val / out_peeled at their slots and in the
//          dense output at their coordinates
// Block rounds are max-combined, so `rounds` equals the synchronous rounds of the
// whole (block-diagonal) incidence, as in the oracle.  A block whose destination
// rows collect more than kBlkMaxRows input rows sets ctrl->blk_fail and the global peel
// (k_peel, launched after in fallback mode) decodes the sketch instead.
#include "launch.h"

namespace lhc {

#ifndef LHC_BLK_THREADS
#define LHC_BLK_THREADS 1024
#endif
constexpr int kBlkThreads = LHC_BLK_THREADS;
constexpr int kBlkCellsPerThread = 32;  // a thread's pure-cell bitmask is one word
// key = sum (2^24 + local id): with local ids < 2^24 and at most 127 input rows per
// destination row (so degree <= 127), degree + carry of the id sum stays < 256 and
// equals 1 only when the true degree is 1
constexpr uint32_t kBlkMaxRows = 127;
#ifndef LHC_BLK_TIMING
#define LHC_BLK_TIMING 0
#endif

struct BlkArgs {
    KParams P;
    const float* counters;
    const uint2* tabS;
    const uint32_t* gmask;
    const uint32_t* rowoff;
    float* dense;
    uint64_t cap;
    float* out_val;
    uint8_t* out_peeled;
    Ctrl* ctrl;
    lhc_stats* stats;
    uint32_t rpb;  // input rows per block (upper bound)
};

// shared-memory layout of one block (32-bit words)
__host__ __device__ inline size_t blk_smem_words(const KParams& P, uint32_t rpb) {
    const size_t cb = (size_t)P.k * P.S_Y * P.L;           // cells of a block
    return 2 * cb                                          // key, R
           + 2 * (size_t)rpb * P.nw                        // masks, claim bits
           + rpb                                           // first slots
           + (size_t)P.k * P.S_Y                           // input rows per destination row
           + 2 * (size_t)rpb * P.k + 1                     // row maps (uint2) of the block's rows
           + (size_t)rpb * P.nw                            // block-local index of each word's first candidate
           + cb                                            // values of the block's candidates
           + 2 * ((cb + 31) / 32);                         // cells to examine: this round's, the next's
}

__global__ void __launch_bounds__(kBlkThreads) k_peel_blocked(const __grid_constant__ BlkArgs A) {
    extern __shared__ uint32_t sm[];
    const KParams& P = A.P;
    const uint32_t k = P.k, L = P.L, nw = P.nw;
    const uint32_t SL = P.S_Y * L;                         // cells per partition of a block
    const uint32_t cb = k * SL;
    uint32_t* key = sm;
    float* R = reinterpret_cast<float*>(sm + cb);
    uint32_t* mask = sm + 2 * cb;
    uint32_t* claim = mask + (size_t)A.rpb * nw;
    uint32_t* first = claim + (size_t)A.rpb * nw;
    uint32_t* rows_per_dst = first + A.rpb;
    const size_t maps_off = ((size_t)(rows_per_dst + k * P.S_Y - sm) + 1) & ~(size_t)1;  // 8-byte aligned
    uint2* maps = reinterpret_cast<uint2*>(sm + maps_off);                             // [rpb][k]
    uint32_t* wpre = reinterpret_cast<uint32_t*>(maps + (size_t)A.rpb * k);            // [rpb][nw]
    float* cval = reinterpret_cast<float*>(wpre + (size_t)A.rpb * nw);                 // [cb]
    const uint32_t ncw = (cb + 31) / 32;                   // words of a cell bitmask
    uint32_t* touch = reinterpret_cast<uint32_t*>(cval + cb);                          // [2][ncw]
    __shared__ uint32_t sh_warp[32];
    __shared__ uint32_t sh_nb;
    const uint32_t cells_per_thread = (cb + blockDim.x - 1) / blockDim.x;  // <= kBlkCellsPerThread

    __shared__ uint32_t sh_peeled, sh_rounds, sh_fail;
    const uint64_t n_c = *(volatile unsigned long long*)&A.ctrl->n_cand;
    if (n_c > A.cap) return;  // overflow: the stats were set by the query

    for (uint32_t b = blockIdx.x; b < P.blocks; b += gridDim.x) {
        __syncthreads();  // the previous block's readers of the shared flags are done
        const uint32_t nrb = b < P.nrows ? (P.nrows - 1 - b) / P.blocks + 1 : 0;  // rows of block b
        const uint64_t cbase = (uint64_t)b * cb;           // first cell of the block
        const uint32_t rbase = b * k * P.S_Y;              // first destination row
        if (threadIdx.x == 0) { sh_peeled = 0; sh_rounds = 0; sh_fail = 0; }
        unsigned long long tb0 = 0, tb1 = 0, tb2 = 0, tb3 = 0;
        if (LHC_BLK_TIMING && threadIdx.x == 0) tb0 = globaltimer();
        // ---- load
        for (uint32_t e = threadIdx.x; e < cb; e += blockDim.x) {
            key[e] = 0u;
            R[e] = __ldcs(A.counters + cbase + e);
        }
        for (uint32_t a = threadIdx.x; a < k * P.S_Y; a += blockDim.x) rows_per_dst[a] = 0u;
        for (uint32_t a = threadIdx.x; a < nrb * nw; a += blockDim.x) {
            const uint32_t t = a / nw, w = a - t * nw;
            const uint64_t i = b + (uint64_t)t * P.blocks;
            mask[a] = __ldcg(A.gmask + i * nw + w);
            claim[a] = 0u;
        }
        for (uint32_t t = threadIdx.x; t < nrb; t += blockDim.x)
            first[t] = __ldcg(A.rowoff + b + (uint64_t)t * P.blocks);
        for (uint32_t a = threadIdx.x; a < nrb * k; a += blockDim.x) {
            const uint32_t t = a / k, j = a - t * k;
            maps[a] = __ldg(&A.tabS[((uint64_t)b + (uint64_t)t * P.blocks) * k + j]);
        }
        // the block's dense ranges are zeroed (values land there later)
        for (uint32_t a = threadIdx.x; a < nrb * (L / 4); a += blockDim.x) {
            const uint32_t t = a / (L / 4), u = a - t * (L / 4);
            const uint64_t q0 = ((uint64_t)b + (uint64_t)t * P.blocks) * L + 4 * u;
            if (q0 + 4 <= P.d) __stcs(reinterpret_cast<float4*>(A.dense + q0), make_float4(0.f, 0.f, 0.f, 0.f));
            else for (uint64_t q = q0; q < P.d; q++) A.dense[q] = 0.f;
        }
        __syncthreads();
        // ---- degree bound: input rows per destination row of the block
        for (uint32_t a = threadIdx.x; a < nrb * k; a += blockDim.x)
            atomicAdd(&rows_per_dst[maps[a].x - rbase], 1u);
        __syncthreads();
        for (uint32_t a = threadIdx.x; a < k * P.S_Y; a += blockDim.x)
            if (rows_per_dst[a] > kBlkMaxRows) sh_fail = 1u;
        __syncthreads();
        if (sh_fail) {
            if (threadIdx.x == 0) atomicOr(&A.ctrl->blk_fail, 1u);
            continue;  // uniform
        }
        if (LHC_BLK_TIMING && threadIdx.x == 0) tb1 = globaltimer();
        // ---- insert: (row t, word w) pairs, every set bit a candidate
        for (uint32_t a = threadIdx.x; a < nrb * nw; a += blockDim.x) {
            const uint32_t t = a / nw, w = a - t * nw;
            uint32_t mm = mask[a];
            if (!mm) continue;
            for (uint32_t j = 0; j < k; j++) {
                const uint2 mp = maps[t * k + j];
                const uint32_t rowl = (mp.x - rbase) * L, bias = map_bias(mp);
                for (uint32_t m2 = mm; m2; m2 &= m2 - 1) {
                    const uint32_t col = 32 * w + (__ffs(m2) - 1);
                    atomicAdd(&key[rowl + ((col + bias) & (L - 1))], (1u << 24) + t * L + col);
                }
            }
        }
        // block-local candidate index of every word's first candidate (exclusive scan
        // of the words' popcounts: thread = a run of consecutive words)
        {
            const uint32_t nwords = nrb * nw;
            const uint32_t per = (nwords + blockDim.x - 1) / blockDim.x;
            const uint32_t w0 = threadIdx.x * per, w1 = min(nwords, w0 + per);
            uint32_t sum = 0;
            for (uint32_t a = w0; a < w1; a++) sum += __popc(mask[a]);
            const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            uint32_t x = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            if (lane == 31) sh_warp[warp] = x;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t run = 0;
                for (uint32_t v = 0; v < blockDim.x / 32; v++) {
                    const uint32_t c = sh_warp[v];
                    sh_warp[v] = run;
                    run += c;
                }
                sh_nb = run;
            }
            __syncthreads();
            uint32_t run = sh_warp[warp] + x - sum;
            for (uint32_t a = w0; a < w1; a++) {
                wpre[a] = run;
                run += __popc(mask[a]);
            }
        }
        __syncthreads();
        // values go through shared memory (written out row by row at the end) unless the
        // block holds more candidates than cells (such a block cannot be peeled anyway)
        const bool staged = sh_nb <= cb;
        if (LHC_BLK_TIMING && threadIdx.x == 0) tb2 = globaltimer();
        // ---- synchronous rounds
        // Only a cell whose degree dropped to one in the previous round can be pure in
        // this one (every pure cell's candidate is peeled in its round), so a round
        // examines the cells marked in its bitmask (all cells in round 1) and marks
        // for the next round the cells its removals bring from degree two to one.
        // Thread t examines the cells [t*cpt, (t+1)*cpt).
        for (uint32_t a = threadIdx.x; a < 2 * ncw; a += blockDim.x) touch[a] = a < ncw ? ~0u : 0u;
        __syncthreads();
        unsigned long long tb_round = LHC_BLK_TIMING ? globaltimer() : 0ull;
        for (uint32_t cur = 0;; cur ^= 1u) {
            uint32_t* tc = touch + cur * ncw;
            uint32_t* tn = touch + (cur ^ 1u) * ncw;
            // A: pure cells at the start of the round among the marked ones
            const uint32_t c0 = threadIdx.x * cells_per_thread;
            uint32_t pure = 0u;
            if (c0 < cb) {
                const uint32_t w0 = c0 >> 5, sh = c0 & 31;
                uint64_t bits = (uint64_t)tc[w0] | (w0 + 1 < ncw ? (uint64_t)tc[w0 + 1] << 32 : 0ull);
                bits >>= sh;
                uint32_t cand = (uint32_t)bits & (cells_per_thread >= 32 ? ~0u : ((1u << cells_per_thread) - 1u));
                for (; cand; cand &= cand - 1) {
                    const uint32_t s2 = __ffs(cand) - 1;
                    if (c0 + s2 < cb && (key[c0 + s2] >> 24) == 1u) pure |= 1u << s2;
                }
            }
            if (!__syncthreads_or(pure != 0u)) break;
            // (this round's marks are read: clear them for the round after next)
            for (uint32_t a = threadIdx.x; a < ncw; a += blockDim.x) tc[a] = 0u;
            // B: peel them
            uint32_t my_peeled = 0;
            for (uint32_t pm = pure; pm; pm &= pm - 1) {
                const uint32_t e = c0 + (__ffs(pm) - 1);
                const uint32_t kv = key[e];
                if ((kv >> 24) != 1u) continue;  // its only candidate was peeled via another cell
                const uint32_t id = kv & 0xffffffu;
                const uint32_t t = id / L, col = id - t * L, w = col >> 5, bit = 1u << (col & 31);
                if (atomicOr(&claim[t * nw + w], bit) & bit) continue;  // claimed via another cell
                const uint64_t i = b + (uint64_t)t * P.blocks;
                const uint32_t je = e / SL;
                const uint2 mpe = maps[t * k + je];
                const float val = map_sign(mpe) * R[e];
                for (uint32_t j = 0; j < k; j++) {
                    // every cell of p loses it (its pure cell too: degree 0, not marked)
                    if (j == je) {
                        atomicSub(&key[e], (1u << 24) + id);
                        continue;
                    }
                    const uint2 mp = maps[t * k + j];
                    const uint32_t ej = (mp.x - rbase) * L + ((col + map_bias(mp)) & (L - 1));
                    atomicAdd(&R[ej], -map_sign(mp) * val);
                    // the new key reads degree one exactly when it is one (the id sum of
                    // two candidates may carry into the degree byte: test the new key)
                    const uint32_t now = atomicSub(&key[ej], (1u << 24) + id) - ((1u << 24) + id);
                    if ((now >> 24) == 1u) atomicOr(&tn[ej >> 5], 1u << (ej & 31));
                }
                const uint32_t ci = wpre[t * nw + w] + __popc(mask[t * nw + w] & (bit - 1u));
                if (staged) {
                    cval[ci] = val;
                } else {  // slot = first slot of the row + candidates before col in the row
                    const uint64_t slot = (uint64_t)first[t] + ci - wpre[t * nw];
                    A.out_val[slot] = val;
                    A.out_peeled[slot] = 1;
                    A.dense[i * L + col] = val;
                }
                my_peeled++;
            }
            // the barrier that ends the round (the next scan sees every update)
            const uint32_t any = __syncthreads_or(my_peeled != 0u);
            if (my_peeled) atomicAdd(&sh_peeled, my_peeled);
            if (any && threadIdx.x == 0) sh_rounds++;
            if (LHC_BLK_TIMING && threadIdx.x == 0 && sh_rounds < 128) {  // per round: time, peeled
                const unsigned long long tr = globaltimer();
                atomicAdd(&A.ctrl->tproc[sh_rounds], tr - tb_round);
                atomicAdd(&A.ctrl->tflush[sh_rounds], (unsigned long long)sh_peeled);
                tb_round = tr;
            }
        }
        if (LHC_BLK_TIMING && threadIdx.x == 0) tb3 = globaltimer();
        // ---- finalize: median estimate of the block's unpeeled candidates
        for (uint32_t a = threadIdx.x; a < nrb * nw; a += blockDim.x) {
            const uint32_t t = a / nw, w = a - t * nw;
            uint32_t left = mask[a] & ~claim[a];
            if (!left) continue;
            const uint64_t i = b + (uint64_t)t * P.blocks;
            for (; left; left &= left - 1) {
                const uint32_t c = __ffs(left) - 1, col = 32 * w + c;
                float v[kMaxK];
                for (uint32_t j = 0; j < k; j++) {
                    const uint2 mp = maps[t * k + j];
                    v[j] = map_sign(mp) * R[(mp.x - rbase) * L + ((col + map_bias(mp)) & (L - 1))];
                }
                for (uint32_t x = 1; x < k; x++) {  // insertion sort of <= 8 values
                    const float y = v[x];
                    int z = (int)x - 1;
                    while (z >= 0 && v[z] > y) { v[z + 1] = v[z]; z--; }
                    v[z + 1] = y;
                }
                const float val = (k & 1) ? v[k / 2] : 0.5f * (v[k / 2 - 1] + v[k / 2]);
                const uint32_t ci = wpre[a] + __popc(mask[a] & ((1u << c) - 1u));
                if (staged) {
                    cval[ci] = val;
                } else {
                    const uint64_t slot = (uint64_t)first[t] + ci - wpre[t * nw];
                    A.out_val[slot] = val;
                    A.out_peeled[slot] = 0;
                    A.dense[i * L + col] = val;
                }
            }
        }
        __syncthreads();
        // ---- outputs, word by word (consecutive threads: consecutive words of a row)
        if (staged) {
            for (uint32_t a = threadIdx.x; a < nrb * nw; a += blockDim.x) {
                uint32_t mm = mask[a];
                if (!mm) continue;
                const uint32_t t = a / nw, w = a - t * nw;
                const uint64_t i = b + (uint64_t)t * P.blocks;
                const uint32_t cl = claim[a];
                const uint64_t slot0 = (uint64_t)first[t] + wpre[a] - wpre[t * nw];
                for (uint32_t r = 0; mm; mm &= mm - 1, r++) {
                    const uint32_t c = __ffs(mm) - 1;
                    const float val = cval[wpre[a] + r];
                    A.out_val[slot0 + r] = val;
                    A.out_peeled[slot0 + r] = (cl >> c) & 1u;
                    A.dense[i * L + 32 * w + c] = val;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            atomicAdd(&A.ctrl->blk_peeled, (unsigned long long)sh_peeled);
            atomicMax(&A.ctrl->blk_rounds, sh_rounds);
            if (LHC_BLK_TIMING) {  // debug: summed phase durations (ns) in ctrl->t[8..12]
                const unsigned long long tb4 = globaltimer();
                atomicAdd(&A.ctrl->t[8], tb1 - tb0);
                atomicAdd(&A.ctrl->t[9], tb2 - tb1);
                atomicAdd(&A.ctrl->t[10], tb3 - tb2);
                atomicAdd(&A.ctrl->t[11], tb4 - tb3);
                atomicAdd(&A.ctrl->t[12], 1ull);
            }
        }
        __syncthreads();
    }
    // the last CTA to finish writes the stats
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&A.ctrl->blk_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0 && !*(volatile uint32_t*)&A.ctrl->blk_fail) {
        const unsigned long long np = *(volatile unsigned long long*)&A.ctrl->blk_peeled;
        A.stats->n_peeled = np;
        A.stats->rounds = *(volatile uint32_t*)&A.ctrl->blk_rounds;
        A.stats->success = np == n_c ? 1 : 0;
        A.stats->entries = 0;
    }
}

static uint32_t rows_per_block(const KParams& P) {
    return P.blocks ? (P.nrows + P.blocks - 1) / P.blocks : 0;
}

bool peel_blocked_fits(const KParams& P) {
    if (!P.blocks || P.nrows == 0) return false;
    const size_t bytes = blk_smem_words(P, rows_per_block(P)) * 4;
    if ((uint64_t)P.k * P.S_Y * P.L > (uint64_t)kBlkThreads * kBlkCellsPerThread) return false;
    if ((uint64_t)rows_per_block(P) * P.L >= (1u << 24)) return false;  // 24-bit local ids
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return bytes + 64 <= (size_t)optin;
}

cudaError_t launch_peel_blocked(const KParams& P, const float* counters, const uint2* tabS,
                                const uint32_t* gmask, const uint32_t* rowoff, float* dense,
                                uint64_t cap, float* out_val, uint8_t* out_peeled, Ctrl* ctrl,
                                lhc_stats* stats, cudaStream_t s) {
    BlkArgs A{};
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
    A.rpb = rows_per_block(P);
    const size_t smem = blk_smem_words(P, A.rpb) * 4;
    cudaFuncSetAttribute(k_peel_blocked, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peel_blocked, kBlkThreads, smem);
    const uint32_t grid = (uint32_t)std::min<uint64_t>(P.blocks, (uint64_t)std::max(1, per_sm) * num_sms());
    k_peel_blocked<<<grid, kBlkThreads, smem, s>>>(A);
    count_launch();
    return cudaGetLastError();
}

}  // namespace lhc
