// launch.h — host-side launchers of the sm_100a kernels (internal to liblhc.so).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "lhc_internal.cuh"

namespace lhc {

int num_sms();           // SM count of the current device (cached per device)
void count_launch(int n = 1);  // bench accounting (thread-local)
void reset_launches();
int set_error(int code, const char* fmt, ...);
int validate(const lhc_params* p);
KParams kparams(const lhc_params* p);

void launch_hash_rows(const KParams& P, uint32_t dom, uint64_t n_rows, uint2* out, cudaStream_t s);
// up to kMaxBatch dense inputs compressed by one launch: input b (d[b] <= P.d
// coordinates) into (bitmap[b], counters[b]); its chunks are the global chunk
// indices [start[b], start[b + 1])
constexpr int kMaxBatch = 16;
struct CompressBatch {
    const float* x[kMaxBatch];
    uint32_t* bitmap[kMaxBatch];
    float* counters[kMaxBatch];
    uint64_t start[kMaxBatch + 1];
    uint32_t d[kMaxBatch];
    uint32_t n;
    // 1: every input has the same d and the global chunk g is row-chunk g / n of
    // input g % n — the n inputs' chunk i are compressed together, so their
    // reductions into the same destination rows (the row maps depend only on the
    // row) hit each sketch line while it is in L2
    uint32_t interleave;
};
void launch_l2_demote(const void* p, size_t bytes, cudaStream_t s);
void launch_compress_dense(const KParams& P, const CompressBatch& B, unsigned long long* nnz_out,
                           cudaStream_t s);
void launch_compress_coo(const KParams& P, uint64_t nnz, const uint32_t* idx, const float* val,
                         uint32_t* bitmap, float* counters, unsigned long long* bad_out,
                         cudaStream_t s);
void launch_clear(int n, uint32_t* const* bitmaps, uint64_t n_words, float* const* counters,
                  uint64_t c, cudaStream_t s);
void launch_aggregate(uint64_t n_words, uint64_t c, int n_in, const uint32_t* const* bitmaps,
                      const float* const* counters, uint32_t* out_bitmap, float* out_counters,
                      cudaStream_t s);
// query + compaction (query.cu)
constexpr uint32_t kMaxQueryCtas = 4096;
cudaError_t launch_query(const KParams& P, const uint32_t* bitmap, uint2* tabS, uint32_t* gmask,
                         uint32_t* cta_total, uint64_t cap, uint32_t* out_idx, Ctrl* ctrl,
                         lhc_stats* stats, uint32_t* rowoff, cudaStream_t s);
// block-local peel of a blocked sketch (peel.cu); false if a block does not fit
bool peel_blocked_fits(const KParams& P);
cudaError_t launch_peel_blocked(const KParams& P, const float* counters, const uint2* tabS,
                                const uint32_t* gmask, const uint32_t* rowoff, float* dense,
                                uint64_t cap, float* out_val, uint8_t* out_peeled, Ctrl* ctrl,
                                lhc_stats* stats, cudaStream_t s);
uint32_t query_max_ctas();
// cluster-level (DSMEM) peel of a blocked sketch with large blocks (peel_cluster.cu):
// the cluster size to use, or 0 when it does not apply
uint32_t peel_cluster_size(const KParams& P);
cudaError_t launch_peel_cluster(const KParams& P, uint32_t cs, const float* counters, const uint2* tabS,
                                const uint32_t* gmask, const uint32_t* rowoff, float* dense,
                                uint64_t cap, float* out_val, uint8_t* out_peeled, Ctrl* ctrl,
                                lhc_stats* stats, cudaStream_t s);

// peeling decoder (peel.cu)
void launch_pair_lists(const KParams& P, const uint2* tabS, uint32_t* dst_off, uint32_t* pair_pos,
                       uint32_t* dst_list, cudaStream_t s);
// row-organised synchronous peel with deterministic values (peel_rows.cu)
cudaError_t launch_peel_rows(const KParams& P, const float* counters, const uint2* tabS,
                             const uint32_t* gmask, uint32_t* dst_off, uint32_t* pair_pos,
                             uint32_t* dst_tmp, uint32_t* dst_list, const uint32_t* cand,
                             unsigned long long* delta, uint32_t* rem, uint32_t* claim,
                             uint32_t* dmark, uint32_t* ymark, uint32_t* xl, uint32_t* yl,
                             float* dense, uint64_t cap, float* out_val, uint8_t* out_peeled,
                             Ctrl* ctrl, lhc_stats* stats, cudaStream_t s);
void launch_build_cells(const KParams& P, const float* counters, const uint2* tabS,
                        const uint32_t* gmask, uint32_t* dst_off, uint32_t* pair_pos,
                        uint32_t* dst_list, void* cells, Ctrl* ctrl, bool compact,
                        uint2* frontier, bool split, cudaStream_t s);
cudaError_t launch_peel(const KParams& P, const float* counters, const uint2* tabS,
                        const uint32_t* cand, float* dense, uint64_t cap, void* cells,
                        uint32_t* claim, uint2* frontier, Ctrl* ctrl, float* out_val,
                        uint8_t* out_peeled, lhc_stats* stats, const uint32_t* rowoff,
                        uint2* vlog, uint32_t* vfill, int mode, cudaStream_t s);
int l2_bytes();

WsLayout ws_layout(const KParams& P, uint64_t cap);

}  // namespace lhc
