/*
 * lhc.h — C ABI of the B200 (sm_100a) hot path of lossless homomorphic gradient
 * compression (arXiv 2402.07529, "Accelerating Distributed Deep Learning using
 * Lossless Homomorphic Compression").  PAPER.md lines are cited as P:L<n>.
 *
 * Algorithm 1: every worker compresses its gradient X into
 * S(X) = [Y, B] (Count Sketch Y + Bloom-filter index B), the aggregation API
 * makes Y <- sum Y and B <- OR B without decompressing, and every
 * worker recovers sum X by peeling and estimation.
 *
 * Conventions for every call below
 *   - All array pointers are DEVICE pointers unless stated otherwise; every
 *     compute call is asynchronous and stream-ordered on `stream` (a
 *     cudaStream_t passed as void*; NULL = the legacy default stream).
 *   - The caller owns every buffer.  The library allocates nothing except the
 *     small state object of lhc_comm_create.
 *   - Shape and argument errors are detected synchronously on the host and
 *     returned as LHC_EINVAL before anything is launched.  Data-dependent
 *     conditions (candidate overflow, a stalled peel) are reported through the
 *     device-resident lhc_stats, never by a host synchronisation (Alg. 1 estimates
 *     the unpeeled parameters instead of failing).  A failed launch
 *     returns LHC_ECUDA; lhc_last_error() gives the message (thread-local).
 *   - Two sketches can be merged only if their lhc_params are identical
 *     (merge-compatibility); the caller enforces it.
 *   - Bit b of a Bloom filter is bit (b & 31) of 32-bit word (b >> 5).
 *   - Alignment: x, counters, bitmaps, out_dense and the workspace must be
 *     16-byte aligned (LHC_EINVAL otherwise).
 *   - Calls on distinct buffers are thread-safe.
 *
 * Layout (§3.4 "Locality Optimization"): coordinate p of the
 * gradient is (input row i = p / L, column t = p % L).  Each input row i and
 * probe j has one (row, bias, sign) triple (reading R4: "each batch shares the
 * same index"); probe j of the Count Sketch lives in partition j of Y (rows
 * [j*S_Y, (j+1)*S_Y), S_Y = c/(k*L); reading R2: "three different indexes"),
 * probe j of the Bloom filter in partition j of B (S_B = m/(k_bloom*L)):
 *   cell_j(p) = row_j(i)*L + (t + bias_j(i)) mod L          (Y: fp32 cells)
 *   bit_j(p)  = rowB_j(i)*L + (t + biasB_j(i)) mod L        (B: bits)
 * The hash (reading R1; the paper gives none) is
 *   mix64(z) = SplitMix64 finalizer
 *   H(seed,dom,j,i) = mix64(seed ^ mix64(((dom<<56)|(j<<48)|i) + 0x9E3779B97F4A7C15))
 *   row = j*S + ((H>>32)*S >> 32), bias = H & (L-1), sign = bit16(H) ? -1 : +1,
 * dom 0 = Count Sketch (S = S_Y), dom 1 = Bloom filter (S = S_B).
 */
#ifndef LHC_H
#define LHC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Sizes of one sketch S(X) = [Y, B] (Alg. 1). */
typedef struct lhc_params {
    uint32_t d;        /* gradient coordinates, 1 <= d < 2^32 (paper: N)            */
    uint64_t m;        /* Bloom-filter bits, multiple of k_bloom*L, m/L < 2^32     */
    uint64_t c;        /* Count Sketch cells, multiple of k*L, c < 2^32 (size of Y) */
    uint32_t k;        /* Count Sketch hashes, 1..8 (paper: 3)                      */
    uint32_t k_bloom;  /* Bloom probes, 0..8; 0 means k (paper: log 1/eps);        *
                        * LHC_INDEX_BITMAP: the exact bitmap index of §3.2 (one bit *
                        * per parameter, bit p = coordinate p; requires m = ceil(d/L)*L)    */
    uint32_t L;        /* batch width, power of two in [32, 1024] (paper: c=1024)  */
    uint32_t blocks;   /* 0: one Count Sketch over all rows; B > 0: the sketch is split into
                          B blocks of k partitions ("splitting the Count Sketch into
                          multiple blocks of fixed size"): input row i hashes only into
                          block i mod B (c must be a multiple of B*k*L)                    */
    uint64_t seed;     /* hash seed; every rank must use the same one                       */
} lhc_params;

/* k_bloom value selecting the exact bitmap index instead of a Bloom filter. */
#define LHC_INDEX_BITMAP 255u

/* Device-resident decode statistics (§4.1.1 metrics). */
typedef struct lhc_stats {
    uint64_t n_cand;   /* candidates n_c returned by the Bloom query (may exceed cap)        */
    uint64_t n_peeled; /* candidates recovered exactly by peeling ("recovery rate" numerator) */
    uint32_t rounds;   /* synchronous peeling rounds that peeled something ("iterations")    */
    int32_t success;   /* 1 iff n_peeled == n_cand and no overflow (lossless)        */
    int32_t overflow;  /* 1 iff n_cand > cap_cand: outputs truncated, nothing peeled         */
    uint32_t entries;  /* frontier entries the rounds processed (F0 included; one claim each) */
} lhc_stats;

enum {
    LHC_OK = 0,
    LHC_EINVAL = 1,    /* invalid argument, shape or alignment                         */
    LHC_ECAPACITY = 2, /* workspace too small                                          */
    LHC_ECUDA = 3,     /* a CUDA call or launch failed                                 */
    LHC_ECOMM = 4      /* peer mapping / IPC failure                                   */
};

/* ---- host helpers (synchronous, no device work) ------------------------- */

/* LHC_OK if the parameters satisfy every constraint listed in lhc_params. */
int lhc_validate(const lhc_params* p);
/* Human-readable text of the last error on the calling thread (never NULL). */
const char* lhc_last_error(void);
/* Number of 32-bit words of the Bloom filter: m / 32. */
uint64_t lhc_bitmap_words(const lhc_params* p);
/* Bytes of device workspace sketch_decompress needs for at most cap_cand
 * candidates (0 on invalid parameters). */
size_t lhc_decompress_workspace(const lhc_params* p, uint64_t cap_cand);

/* ---- Phase I: compression (Alg. 1) ---------------------------- */

/* Seeded hash kernel: writes the per-input-row map of domain dom (0 = Count
 * Sketch, 1 = Bloom filter) for input rows [0, n_rows):
 *   out[2*(i*kk + j)]     = row_j(i)       (absolute row of Y or B, partition j)
 *   out[2*(i*kk + j) + 1] = bias_j(i) | (sign_j(i) < 0) << 31
 * with kk = k (dom 0) or k_bloom (dom 1).  out holds 2*n_rows*kk u32. */
int sketch_hash_rows(const lhc_params* p, uint32_t dom, uint64_t n_rows, uint32_t* out,
                     void* stream);

/* Zero a sketch (bitmap: m/32 words, counters: c floats) before compression. */
int sketch_clear(const lhc_params* p, uint32_t* bitmap, float* counters, void* stream);
/* sketch_clear of n sketches in one launch (HOST arrays of n device pointers). */
int sketch_clear_batch(const lhc_params* p, int n, uint32_t* const* bitmaps, float* const* counters,
                       void* stream);

/* Compress a dense fp32 gradient x[d] (Alg. 1 Phase I; Count Sketch P:L175,
 * Bloom filter P:L230, batched layout P:L262).  Every coordinate with
 * x[p] != 0.0f (IEEE compare: -0.0 counts as zero) sets its k_bloom bits in
 * bitmap[m/32] (bitwise OR) and adds sign_j*x[p] to its k cells of
 * counters[c] (fp32 atomic add, round-to-nearest; order-dependent rounding).
 * ACCUMULATES: compressing several gradients into one sketch yields the
 * aggregate sketch of their sum (the homomorphism of P:L137).  nnz_out
 * (device, nullable) is incremented by the number of nonzeros. */
int sketch_compress(const lhc_params* p, const float* x, uint32_t* bitmap, float* counters,
                    unsigned long long* nnz_out, void* stream);

/* n dense gradients in one launch (per 16 inputs): input b, xs[b][ds[b]] with
 * ds[b] <= p->d (ds NULL: every input has p->d coordinates), is accumulated into
 * (bitmaps[b], counters[b]) with the hash functions of p — the same result as n
 * sketch_compress calls.  Sketches may repeat (homomorphic accumulation);
 * a shorter input is a coordinate shard sketched with its own row range (DESIGN.md
 * NEXT-2).  xs, bitmaps, counters: HOST arrays of n device pointers, each 16-byte
 * aligned; nnz_out (device, nullable) receives the total nonzero count. */
int sketch_compress_batch(const lhc_params* p, int n, const float* const* xs, const uint32_t* ds,
                          uint32_t* const* bitmaps, float* const* counters,
                          unsigned long long* nnz_out, void* stream);

/* Same from a COO gradient: idx[nnz] (each < d, distinct), val[nnz].  Every
 * listed entry is inserted, including val == 0 (the index describes the listed
 * support).  Accumulates like sketch_compress.  An entry with idx >= d is a
 * data-dependent error: it is skipped (nothing is written for it) and counted
 * into *bad_out (device, nullable; accumulated, the caller zeroes it). */
int sketch_compress_coo(const lhc_params* p, uint64_t nnz, const uint32_t* idx,
                        const float* val, uint32_t* bitmap, float* counters,
                        unsigned long long* bad_out, void* stream);

/* ---- aggregation (Alg. 1: Y <- sum Y, B <- OR B) ---------------- */

/* Single-GPU aggregation of n_in sketches (e.g. workers simulated on one GPU):
 * out_bitmap = OR_r bitmaps[r], out_counters = sum_r counters[r] (fp32, summed
 * in ascending r).  bitmaps/counters are HOST arrays of n_in device pointers;
 * out may alias bitmaps[0]/counters[0]. */
int sketch_aggregate(const lhc_params* p, int n_in, const uint32_t* const* bitmaps,
                     const float* const* counters, uint32_t* out_bitmap, float* out_counters,
                     void* stream);

/* Multi-GPU aggregation over NVLink peer memory (one process per GPU).
 * The communication buffer of every rank holds [bitmap | counters | signals]
 * at the offsets lhc_comm_layout returns; compress straight into it.
 * lhc_ipc_handle exports a buffer (CUDA IPC handle, 64 bytes, plus the offset
 * of dev_ptr inside its allocation); the caller exchanges them (e.g. with
 * torch.distributed.all_gather_object) and passes all world handles/offsets to
 * lhc_comm_create, which maps the peers' buffers.  sketch_allreduce then makes
 * every rank's [bitmap | counters] the OR / sum over all ranks, in place, with
 * a two-shot reduce-scatter + all-gather over NVLink and system-scope flag
 * barriers (counters summed in ascending rank order: identical on all ranks). */
typedef struct lhc_comm lhc_comm;
int lhc_comm_layout(const lhc_params* p, size_t* bitmap_off, size_t* counters_off,
                    size_t* signals_off, size_t* total_bytes);
int lhc_ipc_handle(const void* dev_ptr, void* handle_out /*64 bytes*/, uint64_t* offset_out);
int lhc_comm_create(int rank, int world, const void* handles /*world*64 bytes, host*/,
                    const uint64_t* offsets /*world, host*/, void* local_buf, size_t buf_bytes,
                    const lhc_params* p, lhc_comm** out);
int sketch_allreduce(lhc_comm* comm, void* stream);
void lhc_comm_destroy(lhc_comm* comm);

/* Sharded aggregation and decode (DESIGN.md NEXT-2).  The coordinates [0, d)
 * are split into `world` contiguous shards of shard_width coordinates (a
 * multiple of 1024; the last shard ragged, none empty); shard q is an
 * independent sketch of x[q*shard_width ...] with its own params ps_q (equal m
 * and c on every shard; d = the shard's width; for the exact bitmap index the
 * last shard's m = ceil(d_q/L)*L).  Every rank's buffer holds `world` slots of
 * slot_bytes; slot q = [bitmap of shard q | counters of shard q at
 * counters_off].  lhc_shard_layout gives the sizes for the LARGEST shard's
 * params ps and a per-shard item capacity cap_items (< 2^32); the buffer must
 * be zero-initialised and 256-byte aligned.
 *   sketch_reduce_scatter   slot `rank` of every rank becomes the OR / sum over
 *       all ranks of their slot `rank` (counters summed in ascending rank
 *       order); the other slots are left as they were.  One NVLink push of
 *       (world-1)/world of the sketch per rank, one cross-rank barrier.
 *   sketch_allgather_decoded  after the rank decoded its shard (sketch_query +
 *       sketch_peel on slot `rank`, out_dense = dense + rank*shard_width):
 *       idx[n]/val[n] with n = *n_items (device; e.g. &stats->n_cand, clamped to
 *       cap_items) are pushed to every peer, and every other shard's range of
 *       dense[d] is overwritten with exactly the values its owner decoded
 *       (0 elsewhere).  Every rank ends with the identical dense sum.  idx, val
 *       and dense must be 16-byte aligned.  If an owner's *n_items exceeds
 *       cap_items (its decode overflowed and did not run), it publishes an
 *       overflow mark instead of its list and EVERY rank, the owner included,
 *       fills that shard's range of dense with NaN: a failed shard is visible on
 *       all ranks, never silently stale.
 * A sharded communicator is created by lhc_shard_comm_create (same handle
 * exchange as lhc_comm_create) and released by lhc_comm_destroy; calling
 * sketch_allreduce on it, or the sharded calls on a plain one, is LHC_EINVAL.
 * All ranks must issue the same sequence of calls. */
int lhc_shard_layout(const lhc_params* ps, int world, uint64_t cap_items, size_t* slot_bytes,
                     size_t* counters_off, size_t* total_bytes);
int lhc_shard_comm_create(int rank, int world, const void* handles /*world*64 bytes, host*/,
                          const uint64_t* offsets /*world, host*/, void* local_buf,
                          size_t buf_bytes, const lhc_params* ps, uint64_t cap_items,
                          lhc_comm** out);
int sketch_reduce_scatter(lhc_comm* comm, void* stream);
int sketch_allgather_decoded(lhc_comm* comm, const uint32_t* idx, const float* val,
                             const unsigned long long* n_items /*device*/, uint64_t shard_width,
                             uint32_t d, float* dense, void* stream);

/* In-switch aggregation over an NVSwitch multicast object (NVLS; DESIGN.md
 * NEXT-2 — the paper's in-network aggregation, P:L122-124 / P:L283, done by the
 * switch).  Collective setup, every rank of the same `world`:
 *   lhc_nvls_open  rank 0 creates a multicast object of >= bytes (+ a 4 KB signal
 *                  area) and hands it to the other ranks over the abstract Unix
 *                  socket `rendezvous` (a name unique to this group); every rank
 *                  adds its current device.  LHC_ECOMM if the box has no NVLS.
 *   (all ranks must return from lhc_nvls_open before any calls lhc_nvls_bind,
 *    e.g. a process-group barrier in between)
 *   lhc_nvls_bind  binds a zeroed buffer of this device to the object and returns
 *                  its local pointer and usable size: lay the sketch out in it
 *                  exactly as for lhc_comm_layout (replicated) or
 *                  lhc_shard_layout (sharded) and compress straight into it.
 * Then, with the same call sequence on every rank:
 *   sketch_allreduce_nvls        [bitmap | counters] (lhc_comm_layout offsets) becomes
 *        the OR / sum over ranks on every rank: each rank reduces a 1/world slice
 *        with multimem.ld_reduce (the switch reads every rank's copy) and writes
 *        it to every rank with one multimem.st; two switch-counter barriers.
 *   sketch_reduce_scatter_nvls   sharded layout: slot `rank` becomes the OR / sum
 *        over ranks of their slot `rank` (multimem.ld_reduce, local store).
 *   sketch_allgather_decoded_nvls  as sketch_allgather_decoded, the list written
 *        once with multicast stores (the switch replicates it to every rank).
 * The in-switch fp32 sum is identical on every rank (one rank reduces each
 * element and broadcasts it) but its order is the switch's, not ascending rank.
 * lhc_nvls_destroy unmaps and releases (after the last call completed). */
typedef struct lhc_nvls lhc_nvls;
int lhc_nvls_open(int rank, int world, const char* rendezvous, size_t bytes, lhc_nvls** out);
int lhc_nvls_bind(lhc_nvls* h, void** local_ptr, size_t* size);
int sketch_allreduce_nvls(lhc_nvls* h, const lhc_params* p, void* stream);
int sketch_reduce_scatter_nvls(lhc_nvls* h, const lhc_params* ps, uint64_t cap_items, void* stream);
int sketch_allgather_decoded_nvls(lhc_nvls* h, const lhc_params* ps, uint64_t cap_items,
                                  const uint32_t* idx, const float* val,
                                  const unsigned long long* n_items /*device*/,
                                  uint64_t shard_width, uint32_t d, float* dense, void* stream);
void lhc_nvls_destroy(lhc_nvls* h);

/* ---- Phase II: recovery (Alg. 1) ----------------------------- */

/* Decode an aggregated sketch [bitmap, counters] (not modified):
 *   1. Bloom query over all d coordinates (a coordinate is a candidate
 *      iff all its k_bloom bits are set); the n_c candidates are written in
 *      ascending order to out_idx[cap_cand]; slot s names out_idx[s].
 *   2. Peeling: synchronous rounds; every cell holding exactly one
 *      unpeeled candidate recovers it (val = sign * residual) and the value is
 *      subtracted from the candidate's other cells.
 *   3. Estimation of candidates peeling did not reach: median over j
 *      of sign_j * residual (reading R11).
 *   out_val[s], out_peeled[s] (1 = recovered exactly, 0 = estimated) for
 *   s < n_c; out_dense[d] (nullable) = value at candidates, exactly 0 elsewhere.
 * ws: lhc_decompress_workspace(p, cap_cand) bytes.  stats: device lhc_stats.
 * If n_c > cap_cand, stats.overflow = 1 and the outputs are undefined. */
int sketch_decompress(const lhc_params* p, const uint32_t* bitmap, const float* counters,
                      void* ws, size_t ws_bytes, uint64_t cap_cand, uint32_t* out_idx,
                      float* out_val, uint8_t* out_peeled, float* out_dense, lhc_stats* stats,
                      void* stream);

/* sketch_decompress in two stream-ordered steps sharing one workspace (call
 * them in this order with the same ws and cap_cand):
 *   sketch_query  step 1 — candidates to out_idx, n_cand / overflow to stats
 *   sketch_peel   steps 2-3 — out_val, out_peeled, n_peeled / rounds / success,
 *                 and out_dense (nullable): every coordinate < d is written,
 *                 the value at candidates and exactly 0 elsewhere; when NULL
 *                 only the list outputs are produced.  The workspace includes
 *                 a log of 8 bytes per candidate slot (peeled values bucketed
 *                 by 1024-coordinate chunk) and a dense scratch for blocked
 *                 sketches. */
int sketch_query(const lhc_params* p, const uint32_t* bitmap, void* ws, size_t ws_bytes,
                 uint64_t cap_cand, uint32_t* out_idx, lhc_stats* stats, void* stream);
int sketch_peel(const lhc_params* p, const float* counters, void* ws, size_t ws_bytes,
                uint64_t cap_cand, const uint32_t* out_idx, float* out_val, uint8_t* out_peeled,
                float* out_dense, lhc_stats* stats, void* stream);

/* Deterministic decode (DESIGN.md NEXT-3): sketch_peel with values that do not
 * depend on launch geometry, scheduling or atomic order — the same aggregated
 * sketch gives the same bytes on every rank and every run.  Same arguments,
 * workspace and outputs as sketch_peel (call after sketch_query); flags, rounds
 * and success are identical to sketch_peel's.  Each candidate takes its value
 * from its lowest-j pure cell (the oracle's rule, reading R10) and deductions
 * are accumulated on a 64-bit fixed-point grid (integer sums commute), so values
 * are bit-exact under the dyadic law and within the fp32 tolerance otherwise.
 * Synchronous rounds organised by sketch row (peel_rows.cu).  Requires no
 * destination row to receive more than 4096 input rows (nrows <= 2048 S_Y; else
 * LHC_EINVAL).  sketch_decompress_det = sketch_query + sketch_peel_det. */
int sketch_peel_det(const lhc_params* p, const float* counters, void* ws, size_t ws_bytes,
                    uint64_t cap_cand, const uint32_t* out_idx, float* out_val, uint8_t* out_peeled,
                    float* out_dense, lhc_stats* stats, void* stream);
int sketch_decompress_det(const lhc_params* p, const uint32_t* bitmap, const float* counters,
                          void* ws, size_t ws_bytes, uint64_t cap_cand, uint32_t* out_idx,
                          float* out_val, uint8_t* out_peeled, float* out_dense, lhc_stats* stats,
                          void* stream);

/* Number of kernel launches the last successful call of each entry point made
 * on this thread (bench accounting of `gpu_launches`). */
int lhc_last_launch_count(void);

/* Reserve `fraction` (0..1) of the current device's maximum persisting-L2 set-aside
 * (cudaLimitPersistingL2CacheSize; a device-wide setting of the calling process).
 * The kernels mark the lines they reuse with L2 evict-last hints (the sketch during
 * the compress, "random memory access lead to frequent cache misses"; the
 * decode state during the peel); those hints only protect lines inside this
 * set-aside, which is 0 by default.  *set_bytes (may be NULL) receives the bytes
 * reserved.  LHC_EINVAL for a fraction outside [0, 1]; LHC_ECUDA if the runtime
 * refuses the limit. */
int lhc_l2_persist(double fraction, size_t* set_bytes);

#ifdef __cplusplus
}
#endif
#endif /* LHC_H */
