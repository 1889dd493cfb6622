// api.cu — the C ABI of include/lhc.h: host-side validation, workspace layout and
// launch sequencing.  All compute happens in the kernels of compress.cu,
// aggregate.cu, query.cu, peel.cu and comm.cu; nothing here touches data.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "launch.h"

namespace lhc {

static thread_local char g_err[512] = "no error";
static thread_local int g_launches = 0;

void count_launch(int n) { g_launches += n; }
void reset_launches() { g_launches = 0; }

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && cached[dev]) return cached[dev];
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    if (dev < 64) cached[dev] = n;
    return n;
}

int l2_bytes() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && cached[dev]) return cached[dev];
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrL2CacheSize, dev);
    if (n <= 0) n = 126 << 20;
    if (dev < 64) cached[dev] = n;
    return n;
}

int set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

static int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(LHC_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return LHC_OK;
}

static uint32_t ilog2(uint32_t x) {
    uint32_t r = 0;
    while ((1u << r) < x) r++;
    return r;
}

int validate(const lhc_params* p) {
    if (!p) return set_error(LHC_EINVAL, "params is NULL");
    if (p->d == 0) return set_error(LHC_EINVAL, "d must be >= 1");
    if (p->k == 0 || p->k > (uint32_t)kMaxK) return set_error(LHC_EINVAL, "k must be in [1, 8]");
    if (p->L < 32 || p->L > 1024 || (p->L & (p->L - 1)))
        return set_error(LHC_EINVAL, "L must be a power of two in [32, 1024]");
    if (p->k_bloom == LHC_INDEX_BITMAP) {
        const uint64_t rows = ((uint64_t)p->d + p->L - 1) / p->L;
        if (p->m != rows * p->L) return set_error(LHC_EINVAL, "exact bitmap index needs m = ceil(d/L)*L");
    } else if (p->k_bloom > (uint32_t)kMaxK) {
        return set_error(LHC_EINVAL, "k_bloom must be in [0, 8] or LHC_INDEX_BITMAP");
    }
    const uint32_t kb = p->k_bloom == LHC_INDEX_BITMAP ? 1u : p->k_bloom ? p->k_bloom : p->k;
    if (p->c == 0 || p->c % ((uint64_t)p->k * p->L)) return set_error(LHC_EINVAL, "c must be a positive multiple of k*L");
    if (p->m == 0 || p->m % ((uint64_t)kb * p->L)) return set_error(LHC_EINVAL, "m must be a positive multiple of k_bloom*L");
    if (p->c >= (1ull << 32)) return set_error(LHC_EINVAL, "c must be < 2^32");
    if (p->m / p->L >= (1ull << 32)) return set_error(LHC_EINVAL, "m/L must be < 2^32");
    if (p->blocks && p->c % ((uint64_t)p->blocks * p->k * p->L))
        return set_error(LHC_EINVAL, "c must be a multiple of blocks*k*L");
    return LHC_OK;
}

KParams kparams(const lhc_params* p) {
    KParams K{};
    K.seed = p->seed;
    K.c = p->c;
    K.m = p->m;
    K.d = p->d;
    K.k = p->k;
    K.exact = p->k_bloom == LHC_INDEX_BITMAP ? 1u : 0u;
    K.kb = K.exact ? 1u : p->k_bloom ? p->k_bloom : p->k;
    K.L = p->L;
    K.log2L = ilog2(p->L);
    K.nw = p->L / 32;
    K.log2nw = ilog2(K.nw);
    K.blocks = p->blocks;
    // rows per Count Sketch partition (per block when the sketch is blocked)
    K.S_Y = (uint32_t)(p->c / ((uint64_t)(p->blocks ? p->blocks : 1) * K.k * p->L));
    K.S_B = (uint32_t)(p->m / ((uint64_t)K.kb * p->L));
    K.nrows = (uint32_t)(((uint64_t)p->d + p->L - 1) / p->L);
    return K;
}

WsLayout ws_layout(const KParams& P, uint64_t cap) {
    WsLayout W{};
    const uint64_t nrows = P.nrows;
    W.nchunks = (uint32_t)(((uint64_t)P.d + kTile - 1) / kTile);
    size_t o = 0;
    W.ctrl = o;      o = align_up(o + sizeof(Ctrl), 256);
    W.tabS = o;      o = align_up(o + nrows * P.k * sizeof(uint2), 256);
    W.gmask = o;     o = align_up(o + (size_t)W.nchunks * 32 * sizeof(uint32_t), 256);
    W.cta_total = o; o = align_up(o + kMaxQueryCtas * sizeof(uint32_t), 256);
    W.cells = o;     o = align_up(o + P.c * sizeof(CellState), 256);
    W.claim = o;     o = align_up(o + (size_t)W.nchunks * 32 * sizeof(uint32_t), 256);  // 1 bit per coordinate
    W.frontier = o;  o = align_up(o + P.c * sizeof(uint2), 256);
    W.dense = o;     o = align_up(o + (size_t)W.nchunks * kTile * sizeof(float), 256);
    W.dst_off = o;   o = align_up(o + ((P.c >> P.log2L) + 1) * sizeof(uint32_t), 256);
    W.pair_pos = o;  o = align_up(o + (size_t)P.nrows * P.k * sizeof(uint32_t), 256);
    W.dst_list = o;  o = align_up(o + (size_t)P.nrows * P.k * sizeof(uint32_t), 256);
    W.rowoff = o;    o = align_up(o + ((size_t)P.nrows + 1) * sizeof(uint32_t), 256);
    // peeled (coordinate, value) pairs, bucketed by 1024-coordinate chunk at the
    // chunk's candidate slots (one end pointer per chunk)
    W.vlog = o;      o = align_up(o + std::max<uint64_t>(std::min<uint64_t>(cap, P.d), 1) * sizeof(uint2), 256);
    W.vfill = o;     o = align_up(o + ((size_t)W.nchunks + 1) * sizeof(uint32_t), 256);
    // row peel (peel_rows.cu): claim masks per probe, per-row flags and worklists,
    // sorted destination-row lists (the fixed-point deductions use `cells`, the
    // remaining masks `claim`)
    W.claim_k = o;   o = align_up(o + (size_t)P.k * W.nchunks * 32 * sizeof(uint32_t), 256);
    W.dmark = o;     o = align_up(o + (P.c >> P.log2L) * sizeof(uint32_t), 256);
    W.dst_sorted = o; o = align_up(o + (size_t)P.nrows * P.k * sizeof(uint32_t), 256);
    W.ymark = o;     o = align_up(o + (size_t)P.nrows * sizeof(uint32_t), 256);
    W.xl = o;        o = align_up(o + 2 * (P.c >> P.log2L) * sizeof(uint32_t), 256);
    W.yl = o;        o = align_up(o + 2 * (size_t)P.nrows * sizeof(uint32_t), 256);
    W.total = o;
    return W;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
static bool aligned4(const void* p) { return ((uintptr_t)p & 3u) == 0; }

}  // namespace lhc

using namespace lhc;

extern "C" {

int lhc_validate(const lhc_params* p) { return validate(p); }

const char* lhc_last_error(void) { return g_err; }

int lhc_last_launch_count(void) { return g_launches; }

// set by lhc_l2_persist: evict-last lines stay pinned in the set-aside, so the decode
// demotes the sketch (and its own state when it is done)
static bool g_l2_persist = false;

int lhc_l2_persist(double fraction, size_t* set_bytes) {
    if (!(fraction >= 0.0 && fraction <= 1.0)) return set_error(LHC_EINVAL, "fraction outside [0, 1]");
    int dev = 0, mx = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess)
        return set_error(LHC_ECUDA, "persisting L2 attribute: %s", cudaGetErrorString(cudaGetLastError()));
    const size_t bytes = (size_t)((double)mx * fraction);
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) != cudaSuccess)
        return set_error(LHC_ECUDA, "persisting L2 limit: %s", cudaGetErrorString(cudaGetLastError()));
    if (set_bytes) *set_bytes = bytes;
    g_l2_persist = bytes > 0;
    return LHC_OK;
}

uint64_t lhc_bitmap_words(const lhc_params* p) { return validate(p) ? 0 : p->m / 32; }

size_t lhc_decompress_workspace(const lhc_params* p, uint64_t cap_cand) {
    if (validate(p)) return 0;
    return ws_layout(kparams(p), cap_cand).total;
}

int sketch_hash_rows(const lhc_params* p, uint32_t dom, uint64_t n_rows, uint32_t* out,
                     void* stream) {
    reset_launches();
    if (int rc = validate(p)) return rc;
    if (dom > 1) return set_error(LHC_EINVAL, "dom must be 0 or 1");
    if (!out && n_rows) return set_error(LHC_EINVAL, "out is NULL");
    if (n_rows >= (1ull << 48)) return set_error(LHC_EINVAL, "n_rows must be < 2^48");
    launch_hash_rows(kparams(p), dom, n_rows, reinterpret_cast<uint2*>(out), (cudaStream_t)stream);
    return check_launch("sketch_hash_rows");
}

int sketch_clear(const lhc_params* p, uint32_t* bitmap, float* counters, void* stream) {
    reset_launches();
    if (int rc = validate(p)) return rc;
    if (!bitmap || !counters) return set_error(LHC_EINVAL, "NULL sketch buffer");
    if (!aligned16(counters)) return set_error(LHC_EINVAL, "counters must be 16-byte aligned");
    launch_clear(1, &bitmap, p->m / 32, &counters, p->c, (cudaStream_t)stream);
    return check_launch("sketch_clear");
}

int sketch_clear_batch(const lhc_params* p, int n, uint32_t* const* bitmaps, float* const* counters,
                       void* stream) {
    reset_launches();
    if (int rc = validate(p)) return rc;
    if (n < 1 || !bitmaps || !counters) return set_error(LHC_EINVAL, "need n >= 1 sketches");
    for (int b = 0; b < n; b++)
        if (!bitmaps[b] || !counters[b] || !aligned16(counters[b]))
            return set_error(LHC_EINVAL, "sketch %d is NULL or its counters not 16-byte aligned", b);
    launch_clear(n, bitmaps, p->m / 32, counters, p->c, (cudaStream_t)stream);
    return check_launch("sketch_clear_batch");
}

static void compress_batches(const KParams& P, int n, const float* const* xs, const uint32_t* ds,
                             uint32_t* const* bitmaps, float* const* counters,
                             unsigned long long* nnz_out, cudaStream_t s) {
    for (int b0 = 0; b0 < n; b0 += kMaxBatch) {
        CompressBatch B{};
        B.n = (uint32_t)std::min(kMaxBatch, n - b0);
        uint64_t start = 0;
        for (uint32_t b = 0; b < B.n; b++) {
            B.x[b] = xs[b0 + b];
            B.bitmap[b] = bitmaps[b0 + b];
            B.counters[b] = counters[b0 + b];
            B.d[b] = ds ? ds[b0 + b] : P.d;
            B.start[b] = start;
            start += ((uint64_t)B.d[b] + kTile - 1) / kTile;
        }
        B.start[B.n] = start;
        bool same = B.n > 1;
        for (uint32_t b = 1; b < B.n; b++) same &= B.d[b] == B.d[0];
        // (input-major kernel only, i.e. inputs into several sketches: the one-sketch
        // case takes the row-major kernel, compress.cu) interleave the inputs row by
        // row when their sketch is well beyond L2 (then the lines a row's reductions
        // touch are reused by the other inputs before they are evicted; measured:
        // BERT 10 %, 387 MB sketch, 3.04 -> 2.02 ms); otherwise the input-major order
        // streams each input once (VGG: 1.09 vs 1.14 ms)
        const size_t sketch = (size_t)P.m / 8 + (size_t)P.c * 4;
        bool inter = same && sketch > (size_t)l2_bytes() * 3 / 2;
        if (const char* ev = getenv("LHC_COMPRESS_INTERLEAVE")) inter = same && strcmp(ev, "0") != 0;
        B.interleave = inter ? 1u : 0u;
        if (start) launch_compress_dense(P, B, nnz_out, s);
    }
}

int sketch_compress(const lhc_params* p, const float* x, uint32_t* bitmap, float* counters,
                    unsigned long long* nnz_out, void* stream) {
    reset_launches();
    if (int rc = validate(p)) return rc;
    if (!x || !bitmap || !counters) return set_error(LHC_EINVAL, "NULL buffer");
    if (!aligned16(x) || !aligned16(counters) || !aligned16(bitmap))
        return set_error(LHC_EINVAL, "x, bitmap and counters must be 16-byte aligned");
    compress_batches(kparams(p), 1, &x, nullptr, &bitmap, &counters, nnz_out, (cudaStream_t)stream);
    return check_launch("sketch_compress");
}

int sketch_compress_batch(const lhc_params* p, int n, const float* const* xs, const uint32_t* ds,
                          uint32_t* const* bitmaps, float* const* counters,
                          unsigned long long* nnz_out, void* stream) {
    reset_launches();
    if (int rc = validate(p)) return rc;
    if (n < 1 || !xs || !bitmaps || !counters) return set_error(LHC_EINVAL, "need n >= 1 inputs");
    for (int b = 0; b < n; b++) {
        if (!xs[b] || !bitmaps[b] || !counters[b])
            return set_error(LHC_EINVAL, "input %d has a NULL buffer", b);
        if (!aligned16(xs[b]) || !aligned16(bitmaps[b]) || !aligned16(counters[b]))
            return set_error(LHC_EINVAL, "input %d: x, bitmap and counters must be 16-byte aligned", b);
        if (ds && ds[b] > p->d) return set_error(LHC_EINVAL, "ds[%d] = %u > d", b, ds[b]);
    }
    compress_batches(kparams(p), n, xs, ds, bitmaps, counters, nnz_out, (cudaStream_t)stream);
    return check_launch("sketch_compress_batch");
}

int sketch_compress_coo(const lhc_params* p, uint64_t nnz, const uint32_t* idx,
                        const float* val, uint32_t* bitmap, float* counters,
                        unsigned long long* bad_out, void* stream) {
    reset_launches();
    if (int rc = validate(p)) return rc;
    if (nnz && (!idx || !val)) return set_error(LHC_EINVAL, "NULL idx/val");
    if (!bitmap || !counters) return set_error(LHC_EINVAL, "NULL sketch buffer");
    if (nnz > p->d) return set_error(LHC_EINVAL, "nnz > d");
    if (nnz && (!aligned4(idx) || !aligned4(val) || !aligned4(counters) || !aligned4(bitmap)))
        return set_error(LHC_EINVAL, "idx, val, bitmap and counters must be 4-byte aligned");
    launch_compress_coo(kparams(p), nnz, idx, val, bitmap, counters, bad_out, (cudaStream_t)stream);
    return check_launch("sketch_compress_coo");
}

int sketch_aggregate(const lhc_params* p, int n_in, const uint32_t* const* bitmaps,
                     const float* const* counters, uint32_t* out_bitmap, float* out_counters,
                     void* stream) {
    reset_launches();
    if (int rc = validate(p)) return rc;
    if (n_in < 1 || !bitmaps || !counters) return set_error(LHC_EINVAL, "need n_in >= 1 inputs");
    if (!out_bitmap || !out_counters) return set_error(LHC_EINVAL, "NULL output");
    for (int r = 0; r < n_in; r++)
        if (!bitmaps[r] || !counters[r] || !aligned16(bitmaps[r]) || !aligned16(counters[r]))
            return set_error(LHC_EINVAL, "input %d is NULL or not 16-byte aligned", r);
    if (!aligned16(out_bitmap) || !aligned16(out_counters))
        return set_error(LHC_EINVAL, "outputs must be 16-byte aligned");
    launch_aggregate(p->m / 32, p->c, n_in, bitmaps, counters, out_bitmap, out_counters,
                     (cudaStream_t)stream);
    return check_launch("sketch_aggregate");
}

namespace {
struct WsView {
    KParams P;
    WsLayout W;
    Ctrl* ctrl;
    uint2* tabS;
    uint32_t *gmask, *cta_total, *claim;
    CellState* cells;
    uint2* frontier;
    float* dense;
    uint32_t *dst_off, *pair_pos, *dst_list;
    uint32_t* rowoff;
    uint2* vlog;
    uint32_t* vfill;
    uint32_t *claim_k, *dmark, *dst_sorted, *ymark, *xl, *yl;
};

int ws_view(const lhc_params* p, void* ws, size_t ws_bytes, uint64_t* cap_cand, WsView* v) {
    if (int rc = validate(p)) return rc;
    if (!ws) return set_error(LHC_EINVAL, "NULL workspace");
    if (!aligned16(ws)) return set_error(LHC_EINVAL, "workspace must be 16-byte aligned");
    if (*cap_cand > p->d) *cap_cand = p->d;
    v->P = kparams(p);
    v->W = ws_layout(v->P, *cap_cand);
    if (ws_bytes < v->W.total)
        return set_error(LHC_ECAPACITY, "workspace too small: %zu < %zu bytes", ws_bytes, v->W.total);
    char* b = static_cast<char*>(ws);
    v->rowoff = reinterpret_cast<uint32_t*>(b + v->W.rowoff);
    v->vlog = reinterpret_cast<uint2*>(b + v->W.vlog);
    v->vfill = reinterpret_cast<uint32_t*>(b + v->W.vfill);
    v->ctrl = reinterpret_cast<Ctrl*>(b + v->W.ctrl);
    v->tabS = reinterpret_cast<uint2*>(b + v->W.tabS);
    v->gmask = reinterpret_cast<uint32_t*>(b + v->W.gmask);
    v->cta_total = reinterpret_cast<uint32_t*>(b + v->W.cta_total);
    v->cells = reinterpret_cast<CellState*>(b + v->W.cells);
    v->claim = reinterpret_cast<uint32_t*>(b + v->W.claim);
    v->frontier = reinterpret_cast<uint2*>(b + v->W.frontier);
    v->dense = reinterpret_cast<float*>(b + v->W.dense);
    v->dst_off = reinterpret_cast<uint32_t*>(b + v->W.dst_off);
    v->pair_pos = reinterpret_cast<uint32_t*>(b + v->W.pair_pos);
    v->dst_list = reinterpret_cast<uint32_t*>(b + v->W.dst_list);
    v->claim_k = reinterpret_cast<uint32_t*>(b + v->W.claim_k);
    v->dmark = reinterpret_cast<uint32_t*>(b + v->W.dmark);
    v->dst_sorted = reinterpret_cast<uint32_t*>(b + v->W.dst_sorted);
    v->ymark = reinterpret_cast<uint32_t*>(b + v->W.ymark);
    v->xl = reinterpret_cast<uint32_t*>(b + v->W.xl);
    v->yl = reinterpret_cast<uint32_t*>(b + v->W.yl);
    return LHC_OK;
}
}  // namespace

int sketch_query(const lhc_params* p, const uint32_t* bitmap, void* ws, size_t ws_bytes,
                 uint64_t cap_cand, uint32_t* out_idx, lhc_stats* stats, void* stream) {
    reset_launches();
    WsView v;
    if (int rc = ws_view(p, ws, ws_bytes, &cap_cand, &v)) return rc;
    if (!bitmap || !stats) return set_error(LHC_EINVAL, "NULL buffer");
    if (cap_cand && !out_idx) return set_error(LHC_EINVAL, "NULL out_idx");
    if (query_max_ctas() > kMaxQueryCtas) return set_error(LHC_ECUDA, "device too large for the query grid");
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(v.ctrl, 0, sizeof(Ctrl), s) != cudaSuccess) return check_launch("memset");
    if (cudaMemsetAsync(stats, 0, sizeof(lhc_stats), s) != cudaSuccess) return check_launch("memset");
    if (g_l2_persist) launch_l2_demote(bitmap, v.P.m / 8, s);
    cudaError_t e = launch_query(v.P, bitmap, v.tabS, v.gmask, v.cta_total, cap_cand, out_idx,
                                 v.ctrl, stats, v.rowoff, s);
    if (e != cudaSuccess) return set_error(LHC_ECUDA, "query launch: %s", cudaGetErrorString(e));
    return check_launch("sketch_query");
}

int sketch_peel(const lhc_params* p, const float* counters, void* ws, size_t ws_bytes,
                uint64_t cap_cand, const uint32_t* out_idx, float* out_val, uint8_t* out_peeled,
                float* out_dense, lhc_stats* stats, void* stream) {
    reset_launches();
    WsView v;
    if (int rc = ws_view(p, ws, ws_bytes, &cap_cand, &v)) return rc;
    if (!counters || !stats) return set_error(LHC_EINVAL, "NULL buffer");
    if (!aligned16(counters)) return set_error(LHC_EINVAL, "counters must be 16-byte aligned");
    if (out_dense && !aligned16(out_dense)) return set_error(LHC_EINVAL, "out_dense must be 16-byte aligned");
    if (cap_cand && (!out_idx || !out_val || !out_peeled)) return set_error(LHC_EINVAL, "NULL output");
    cudaStream_t s = (cudaStream_t)stream;
    float* dense = out_dense ? out_dense : v.dense;  // zeroed by the peel kernel
    // cell state larger than half the L2: build it by destination row (no random
    // HBM reductions), compact (8 B/cell) when the input rows fit in 22 bits;
    // otherwise the in-kernel per-candidate insert is faster.
    // (LHC_CELL_BUILD=rows|compact|insert overrides the choice; results are identical)
    // A blocked sketch is peeled block by block in shared memory; the global
    // peel then runs only if a block could not be (mode 3: fallback, device-checked).
    int mode = p->c * sizeof(CellState) > (size_t)l2_bytes() / 2 ? 1 : 0;
    if (mode == 1 && v.P.nrows <= (1u << 22)) mode = 2;
    // compact state beyond the L2: keys and residuals in two arrays, peeled in two
    // passes that each keep half of it in L2 — when that half fits (VGG19: 1.74 ->
    // 1.45 ms; LSTM, 118 MB of keys: 1.72 -> 1.98 ms) (LHC_PEEL_SPLIT=0/1 overrides)
    bool split = p->c * sizeof(CellC) > (size_t)l2_bytes() / 2 &&
                 p->c * sizeof(uint32_t) <= (size_t)l2_bytes() * 7 / 10;
    if (const char* es = getenv("LHC_PEEL_SPLIT")) split = !strcmp(es, "1");
    bool blocked = peel_blocked_fits(v.P);
    if (const char* ev = getenv("LHC_CELL_BUILD")) {
        if (!strcmp(ev, "rows")) mode = 1, blocked = false;
        if (!strcmp(ev, "compact")) mode = v.P.nrows <= (1u << 22) ? 2 : 1, blocked = false, split = false;
        if (!strcmp(ev, "split")) mode = v.P.nrows <= (1u << 22) ? 2 : 1, blocked = false, split = true;
        if (!strcmp(ev, "insert")) mode = 0, blocked = false;
    }
    // large blocks, one per thread-block cluster with the state in distributed shared
    // memory (peel_cluster.cu): correct but slower than the global peel on the same
    // layout (VGG19, 82 blocks of 196,608 cells: 5.0 ms vs 2.2 ms — DSMEM atomics
    // across 16 CTAs sustain ~56 G/s in total), so only on request (LHC_PEEL_CLUSTER=1)
    const char* ecl = getenv("LHC_PEEL_CLUSTER");
    uint32_t cl_size = v.P.blocks && ecl && !strcmp(ecl, "1") ? peel_cluster_size(v.P) : 0u;
    if (getenv("LHC_CELL_BUILD")) cl_size = 0;
    if (cl_size) {
        cudaError_t ec = launch_peel_cluster(v.P, cl_size, counters, v.tabS, v.gmask, v.rowoff, dense,
                                             cap_cand, out_val, out_peeled, v.ctrl, stats, s);
        if (ec != cudaSuccess) return set_error(LHC_ECUDA, "cluster peel launch: %s", cudaGetErrorString(ec));
        mode = 3;
        blocked = false;
    }
    if (blocked) {
        cudaError_t eb = launch_peel_blocked(v.P, counters, v.tabS, v.gmask, v.rowoff, dense, cap_cand,
                                             out_val, out_peeled, v.ctrl, stats, s);
        if (eb != cudaSuccess) return set_error(LHC_ECUDA, "blocked peel launch: %s", cudaGetErrorString(eb));
        mode = 3;
    }
    if (mode == 2 && split) mode = 4;
    if (mode == 1 || mode == 2 || mode == 4)
        launch_build_cells(v.P, counters, v.tabS, v.gmask, v.dst_off, v.pair_pos, v.dst_list,
                           v.cells, v.ctrl, mode != 1, v.frontier, mode == 4, s);
    // the global peel writes every coordinate of the dense output itself (chunk by
    // chunk, after the rounds); with no dense output it writes only the list values
    if (g_l2_persist) launch_l2_demote(counters, v.P.c * sizeof(float), s);
    cudaError_t e = launch_peel(v.P, counters, v.tabS, out_idx, out_dense, cap_cand, v.cells, v.claim,
                                v.frontier, v.ctrl, out_val, out_peeled, stats, v.rowoff, v.vlog,
                                v.vfill, mode, s);
    if (e != cudaSuccess) return set_error(LHC_ECUDA, "peel launch: %s", cudaGetErrorString(e));
    if (g_l2_persist) {  // the peel's evict-last state
        launch_l2_demote(v.cells, v.P.c * (mode == 2 || mode == 4 ? sizeof(CellC) : sizeof(CellState)), s);
        launch_l2_demote(v.claim, ((size_t)v.P.d + 7) / 8, s);
    }
    return check_launch("sketch_peel");
}

int sketch_peel_det(const lhc_params* p, const float* counters, void* ws, size_t ws_bytes,
                    uint64_t cap_cand, const uint32_t* out_idx, float* out_val, uint8_t* out_peeled,
                    float* out_dense, lhc_stats* stats, void* stream) {
    reset_launches();
    WsView v;
    if (int rc = ws_view(p, ws, ws_bytes, &cap_cand, &v)) return rc;
    if (!counters || !stats) return set_error(LHC_EINVAL, "NULL buffer");
    if (!aligned16(counters)) return set_error(LHC_EINVAL, "counters must be 16-byte aligned");
    if (out_dense && !aligned16(out_dense)) return set_error(LHC_EINVAL, "out_dense must be 16-byte aligned");
    if (cap_cand && (!out_idx || !out_val || !out_peeled)) return set_error(LHC_EINVAL, "NULL output");
    // the row peel tracks a pure cell's owner in 12 bit planes: a destination row
    // may list at most 4096 input rows (hashed uniformly: nrows <= 2048 S_Y)
    const uint64_t s_blk = v.P.blocks ? v.P.S_Y : v.P.S_Y;
    const uint64_t rows_per_part = v.P.blocks ? (v.P.nrows + v.P.blocks - 1) / v.P.blocks : v.P.nrows;
    if (rows_per_part > 2048ull * s_blk)
        return set_error(LHC_EINVAL, "deterministic decode: %llu input rows onto %llu rows per partition",
                         (unsigned long long)rows_per_part, (unsigned long long)s_blk);
    float* dense = out_dense ? out_dense : v.dense;
    cudaError_t er = launch_peel_rows(v.P, counters, v.tabS, v.gmask, v.dst_off, v.pair_pos,
                                      v.dst_list, v.dst_sorted, out_idx,
                                      reinterpret_cast<unsigned long long*>(v.cells), v.claim,
                                      v.claim_k, v.dmark, v.ymark, v.xl, v.yl, dense, cap_cand,
                                      out_val, out_peeled, v.ctrl, stats, (cudaStream_t)stream);
    if (er != cudaSuccess) return set_error(LHC_ECUDA, "row peel launch: %s", cudaGetErrorString(er));
    return check_launch("sketch_peel_det");
}

int sketch_decompress_det(const lhc_params* p, const uint32_t* bitmap, const float* counters,
                          void* ws, size_t ws_bytes, uint64_t cap_cand, uint32_t* out_idx,
                          float* out_val, uint8_t* out_peeled, float* out_dense, lhc_stats* stats,
                          void* stream) {
    if (int rc = sketch_query(p, bitmap, ws, ws_bytes, cap_cand, out_idx, stats, stream)) return rc;
    int n = lhc_last_launch_count();
    if (int rc = sketch_peel_det(p, counters, ws, ws_bytes, cap_cand, out_idx, out_val, out_peeled,
                                 out_dense, stats, stream))
        return rc;
    n += lhc_last_launch_count();
    reset_launches();
    count_launch(n);
    return LHC_OK;
}

int sketch_decompress(const lhc_params* p, const uint32_t* bitmap, const float* counters,
                      void* ws, size_t ws_bytes, uint64_t cap_cand, uint32_t* out_idx,
                      float* out_val, uint8_t* out_peeled, float* out_dense, lhc_stats* stats,
                      void* stream) {
    if (int rc = sketch_query(p, bitmap, ws, ws_bytes, cap_cand, out_idx, stats, stream)) return rc;
    int n = lhc_last_launch_count();
    if (int rc = sketch_peel(p, counters, ws, ws_bytes, cap_cand, out_idx, out_val, out_peeled,
                             out_dense, stats, stream))
        return rc;
    n += lhc_last_launch_count();
    reset_launches();
    count_launch(n);
    return LHC_OK;
}

}  // extern "C"
