// ta_kernels.h -- launch interface of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ta_internal.h"

namespace ta {

// One persistent launch per layer (grid = schedule CTAs, one per SM).  A CTA
// walks its items (see ta_internal.h); rows of an item are (slot, q head in
// the GQA group) pairs, row = slot * G + g, local q head = head * G + g.
// Per-step counts, at offset 0 of the schedule metadata blob (device).
struct DevCounts {
    int32_t n_empty;     // empty leaf-heads
    int32_t n_merge;     // merge records
    int32_t n_append;    // rows of ta_kv_append (tokens appended before the last ta_prepare)
    int32_t n_partials;
    int32_t pad[60];
};
static_assert(sizeof(DevCounts) == 256, "DevCounts layout");

// fused-merge counters: one per merge record, kCntStride words apart (own L2 line)
constexpr int kCntStride = 32;

struct AttnArgs {
    // KV pools of this layer.  FMA path: element pointers + per-head stride.
    const void* k;
    const void* v;
    int64_t head_stride;      // elements between kv heads
    // MMA path: TMA maps over the whole pools ([rows][D] bf16, rows =
    // (layer * n_loc + head) * head_rows + page * P + slot)
    const void* tmap_k;       // CUtensorMap[4] (16/32/64/128-row boxes), host memory
    const void* tmap_v;
    int64_t layer_row0;
    int64_t head_rows;
    // queries / outputs, leaves() order
    const void* q;            // [L][hq_loc][D] kv dtype
    void* out;                // [L][hq_loc][D] out dtype
    float* lse;               // [L][hq_loc] natural log, or nullptr
    float* part_o;            // [n_part][G][D] fp32, O / l
    float* part_lse;          // [n_part][G] log2 domain
    // schedule (device copies of Schedule)
    const TileDesc* tiles;
    const TileMeta* tile_meta;
    const int32_t* grp_row;
    const uint32_t* grp_info;
    const ItemDesc* items;
    const int32_t* cta_begin;
    const int32_t* slot_leaf;
    const int32_t* slot_out;
    const DevCounts* counts;  // per-step counts (device; graph-stable pointer)
    const int4* merge_rec;    // [n_merge] {leaf, local kv head, first partial id, count}
    const int32_t* part_merge;// partial id -> merge record
    unsigned* merge_cnt;      // fused merge: per record, partials published (self-resetting)
    int fused_merge;          // 1: records merged at the end of the attention launch (tcgen05 kernel)
    const int32_t* cta_pub_begin;   // [n_ctas + 1] into cta_pub
    const int2* cta_pub;            // (record, partials this CTA wrote)
    const int32_t* cta_own_begin;   // [n_ctas + 1] into cta_own
    const int32_t* cta_own;         // records the CTA merges
    const int32_t* empty;     // [n_empty][2] (leaf, head)
    const uint8_t* cta_heads; // tcgen05 kernel: per-CTA schedule blobs (ta_internal.h, namespace blob)
    const uint8_t* cta_tails;
    int n_ctas;
    int G;
    int hq_loc;
    int D;
    float scale_log2;         // log2(e) / sqrt(D)
    int kv_bf16;
    int out_bf16;
    long long* trace;         // optional clock64 trace (debug builds of the launch: a separate instantiation)
    int prefetch_tiles;       // first tiles of each CTA prefetched into L2 before the dependency wait
    // tcgen05 kernel, fused decode-step append (ta_kv_append deferred into
    // this launch): the step's new rows [n][n_loc][D] (nullptr: none) and
    // per CTA the rows it writes into this layer's pools before loading them
    // tcgen05 kernel, host-buffer attend: q lands by an asynchronous copy on
    // another stream, announced by a stream write of q_seq to *q_flag (nullptr:
    // q is ready when the launch starts)
    const unsigned* q_flag;
    unsigned q_seq;
    const void* app_k;
    const void* app_v;
    const int4* app_cta;      // [n_ctas] {begin, end, first CTA-local tile, 0}
    const int4* app_list;     // {append index, local head, pool row, 0}
    int early_kv;             // tcgen05 kernel: the CTA's leading tiles that no pending ta_kv_append row
                              // touches (blob header) are loaded before the dependency wait
    unsigned long long* timeline;   // debug: [4] = attn first start, attn last end, merge first start, merge last end (ns)
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for the current device,
// once per (kernel, device): the attribute is per device, so a process with
// contexts on several GPUs sets it on each.
cudaError_t set_smem_attr_once(const void* kernel, int bytes);

// tcgen05/TMEM path (bf16, D = 128).
cudaError_t launch_attn_mma(const AttnArgs& a, bool pdl, cudaStream_t s);
bool mma_supported(int D, int kv_bf16);
// encode the TMA descriptor (128 B, CUtensorMap) of a [rows][D] bf16 pool
bool make_pool_tmap(void* tmap_out, const void* base, int64_t rows, int D, int box_rows);
// FMA path (fp32 or bf16, D in {16, 32, 64, 128}, rows per lane <= 8 or 16).
cudaError_t launch_attn_fma(const AttnArgs& a, int max_rows, bool pdl, cudaStream_t s);
// groups per tile the FMA kernel stages (2 stages of K and V fit in SMEM)
int fma_tile_groups(int D, int esize);
// split-K merge of the partial records (after the attention launch); a fixed
// grid of 4 x n_sms CTAs loops over counts->n_merge records (graph-stable)
cudaError_t launch_merge(const AttnArgs& a, int n_sms, bool pdl, cudaStream_t s);
// ta_lse_merge: n_parts partial results of the same rows -> their merge (prefix split)
cudaError_t launch_lse_merge(const float* part_o, const float* part_lse, int n_parts, int64_t rows, int d, void* out,
                             int out_bf16, float* lse_out, cudaStream_t s);
// ta_kv_append: src rows [n][n_loc][D] -> pool rows rows[i] for every local
// head, n = counts->n_append read on the device (graph-stable, fixed grid)
cudaError_t launch_kv_append(const void* src_k, const void* src_v, void* dst_k, void* dst_v, const int32_t* rows,
                             const DevCounts* counts, int n_loc, int64_t head_stride, int D, int esize, int n_sms,
                             cudaStream_t s);
// dst rows[i] <- src row i, for n_loc kv heads: src [n][n_loc][D], dst pool
cudaError_t launch_kv_scatter(const void* src_k, const void* src_v, void* dst_k, void* dst_v,
                              const int32_t* rows, int n, int n_loc, int64_t head_stride, int D,
                              int esize, cudaStream_t s);

}  // namespace ta
