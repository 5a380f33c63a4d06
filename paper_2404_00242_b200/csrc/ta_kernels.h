// ta_kernels.h -- launch interface of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ta_internal.h"

namespace ta {

// One attention launch over a list of units for all local kv heads
// (grid.y = kv head).  Rows of a unit are (slot, q-head-in-group) pairs,
// row = slot * G + g; q head index (local) = kv_head * G + g.
struct AttnArgs {
    const void* k;            // layer base of the K pool, local kv head 0
    const void* v;
    int64_t head_stride;      // elements between kv heads in the pool
    const void* q;            // [L][hq_loc][D]
    void* out;                // [L][hq_loc][D] out dtype
    float* lse;               // [L][hq_loc] natural log, or nullptr
    float* part_o;            // [n_part][hq_loc][D]
    float* part_lse;          // [n_part][hq_loc] (log2 domain)
    const UnitDesc* units;
    int n_units;
    const int32_t* tok_row;
    const uint32_t* tok_be;
    const int32_t* slot_leaf;
    const int32_t* slot_part;
    int G;
    int hq_loc;
    int n_kv_loc;
    int D;
    float scale_log2;         // log2(e) / sqrt(D)
    int kv_bf16;
    int out_bf16;
    // MMA path: TMA tensor maps over the whole K / V pools ([rows][D] bf16,
    // rows = layer * n_loc * head_rows + head * head_rows + page * P + slot)
    const void* tmap_k;       // CUtensorMap[4] (16/32/64/128-row boxes; host memory, copied into params)
    const void* tmap_v;
    int64_t layer_row0;
    int64_t head_rows;
    const int32_t* grp_row;
    const uint32_t* grp_info;
    long long* trace;         // optional per-tile clock64 trace of CTA (0,0)
};

struct MergeArgs {
    const float* part_o;
    const float* part_lse;
    const int32_t* merge_leaf;
    const int32_t* merge_begin;
    const int32_t* merge_parts;
    int n_merge;
    void* out;
    float* lse;
    int hq_loc;
    int D;
    int out_bf16;
};

// FMA path (sparse chunks / fp32): max_rows in {8, 16}.
cudaError_t launch_attn_fma(const AttnArgs& a, int max_rows, cudaStream_t s);
// tcgen05/TMEM path (dense bf16 chunks, D in {64,128}).
cudaError_t launch_attn_mma(const AttnArgs& a, cudaStream_t s);
bool mma_supported(int D, int kv_bf16);
// encode the TMA descriptor (128 B, CUtensorMap) of a [rows][D] bf16 pool
bool make_pool_tmap(void* tmap_out, const void* base, int64_t rows, int D, int box_rows);
cudaError_t launch_merge(const MergeArgs& a, cudaStream_t s);
// dst rows[i] <- src row i, for n_loc kv heads: src [n][n_loc][D], dst pool
cudaError_t launch_kv_scatter(const void* src_k, const void* src_v, void* dst_k, void* dst_v,
                              const int32_t* rows, int n, int n_loc, int64_t head_stride, int D,
                              int esize, cudaStream_t s);

}  // namespace ta
