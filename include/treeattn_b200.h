/*
 * treeattn_b200.h -- C ABI of the B200-native DeFT-Flatten decode path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/treeattn, paths below relative to it).
 * The reference is a header-only C++ library with no FFI of its own; the
 * entry points here are exactly what a binding of its hot path needs:
 *
 *   reference call                                   | replaced by
 *   -------------------------------------------------+---------------------------
 *   DecodingTree(root_tokens, KvLifecycle*)  tree.hpp:40-51   | ta_tree_new
 *   DecodingTree::restore(root, nodes, kv)   tree.hpp:207-238 | ta_tree_restore
 *   DecodingTree::branch                     tree.hpp:74-97   | ta_tree_branch
 *   DecodingTree::prune                      tree.hpp:100-116 | ta_tree_prune
 *   DecodingTree::append_tokens              tree.hpp:119-129 | ta_tree_append
 *   DecodingTree::leaves                     tree.hpp:55      | ta_tree_leaves
 *   PagePool(dim, page_size) + KvLifecycle   kv_cache.hpp:33-147 | ta_ctx_create (device pool)
 *   PagePool::page_count/free_page_count/live_slots kv_cache.hpp:43-45 | ta_pool_stats
 *   KvHandle::refs[t] (TokenRef)             kv_cache.hpp:14-22 | ta_pool_token_ref
 *   PagePool::write_kv                       kv_cache.hpp:104-116 | ta_kv_write
 *   partition_flatten                        partition.hpp:212-253 | ta_plan_flatten
 *   plan_to_json                             serde.hpp:41-61  | ta_plan_json
 *   run_iteration(tree, Flatten, bs, pool, queries, params)
 *                                            attention.hpp:293-334 | ta_prepare + ta_attend
 *   io_measured / io_analytical(Flatten)     io_model.hpp:144-170 | ta_io_stats
 *
 * Errors: every entry returns a ta_status; ta_last_error() returns the
 * thread-local message, mirroring the reference's exception text
 * (invalid_argument / out_of_range / logic_error).  No exception crosses
 * this boundary.  There is no CPU fallback: attention entry points on a
 * context without a device fail with TA_ERR_NO_DEVICE.
 */
#ifndef TREEATTN_B200_H
#define TREEATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TA_ABI_VERSION 2

typedef int ta_status;
enum {
    TA_OK = 0,
    TA_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    TA_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range */
    TA_ERR_LOGIC = 3,            /* std::logic_error */
    TA_ERR_CUDA = 4,
    TA_ERR_NO_DEVICE = 5,
    TA_ERR_OUT_OF_MEMORY = 6,
};

enum { TA_F32 = 0, TA_BF16 = 1 };

/* Partition strategies (partition.hpp:16, same order).  Flatten is the hot
 * path; the others are the paper's ablations (DeFT-Node, DeFT-Node-Chunk and
 * the query-guided split of Flash-Decoding / Radix attention), runnable on the
 * same kernels: select with ta_set_option(ctx, "strategy", s). */
enum { TA_STRATEGY_Q_GUIDED = 0, TA_STRATEGY_NODE = 1, TA_STRATEGY_NODE_CHUNK = 2, TA_STRATEGY_FLATTEN = 3 };

/* IO model (io_model.hpp:16-26, same order) */
enum {
    TA_ALG_NAIVE = 0, TA_ALG_FLASH_DECODING = 1, TA_ALG_RADIX = 2, TA_ALG_TREE_ATTN_MEDUSA = 3,
    TA_ALG_TREE_ATTN_SPECINFER = 4, TA_ALG_NODE = 5, TA_ALG_NODE_CHUNK = 6, TA_ALG_FLATTEN = 7
};
typedef struct ta_cost_params {  /* CostParams (common.hpp:15-31) */
    int d_head, n_heads, n_layers, dtype_bytes;
} ta_cost_params;
typedef struct ta_io_report {     /* IoReport (io_model.hpp:62-72) */
    uint64_t kv_bytes, q_bytes, mask_bytes, partial_bytes;
} ta_io_report;

typedef struct ta_shape {
    int n_layers;        /* independent KV pools, one per layer */
    int n_q_heads;       /* h_q of the model (AttentionParams::n_heads for MHA) */
    int n_kv_heads;      /* h_kv (== n_q_heads for the reference's MHA) */
    int d_head;          /* AttentionParams::d_head */
    int kv_dtype;        /* TA_F32 | TA_BF16 : KV pool and query dtype */
    int out_dtype;       /* TA_F32 | TA_BF16 : attention output dtype */
    int page_tokens;     /* PagePool page_size (kv_cache.hpp:35), default 16 */
    int kv_head_begin;   /* first kv head owned by this context (head sharding) */
    int n_local_kv_heads;/* kv heads owned by this context (0 = all) */
    int64_t max_pages;   /* device page capacity per (layer, kv head) pool */
} ta_shape;

typedef struct ta_ctx ta_ctx;

const char* ta_last_error(void);
int ta_abi_version(void);

/* device < 0 creates a host-only context (tree, page accounting, planner). */
ta_status ta_ctx_create(int device, const ta_shape* shape, ta_ctx** out);
ta_status ta_ctx_destroy(ta_ctx* ctx);
/* tuning knobs: "use_mma", "fma_max_rows", "mma_max_rows", "tile_groups",
 * "tile_cost", "box_cost", "row_cost", "item_cost", "item_cost_many", "many_items",
 * "minmax", "num_ctas", "final_direct", "fused_merge", "pdl", "fuse_append", "host_q_poll",
 * "prefetch_tiles"; debug: "trace_ptr", "timeline_ptr" */
ta_status ta_set_option(ta_ctx* ctx, const char* key, int64_t value);

/* ---- DecodingTree (tree mutations drive the page pool like KvLifecycle) -- */
ta_status ta_tree_new(ta_ctx* ctx, int64_t root_tokens, int32_t* root_out);
ta_status ta_tree_restore(ta_ctx* ctx, int32_t root, int n, const int32_t* ids,
                          const int32_t* parents, const int64_t* token_counts);
ta_status ta_tree_branch(ta_ctx* ctx, int32_t at, int n, const int64_t* child_token_counts,
                         int32_t* created);
ta_status ta_tree_prune(ta_ctx* ctx, int32_t at);
ta_status ta_tree_append(ta_ctx* ctx, int32_t leaf, int64_t n);
/* append_tokens on many leaves in one call (the decode step of gen_few_shot,
 * workloads.hpp:98-111): leaves NULL = every leaf in leaves() order (n must be
 * the leaf count), counts NULL = one token each.  All or nothing. */
ta_status ta_tree_append_leaves(ta_ctx* ctx, int n, const int32_t* leaves, const int64_t* counts);
/* leaves in DFS pre-order; *n receives the count (out may be NULL to size) */
ta_status ta_tree_leaves(ta_ctx* ctx, int32_t* out, int cap, int* n);

typedef struct ta_tree_info {
    int32_t root;
    int32_t node_count;
    int32_t n_leaves;
    int32_t next_id;
    int64_t total_tokens;
    int64_t path_tokens_sum; /* sum of root-to-leaf path lengths (F_s numerator) */
} ta_tree_info;
ta_status ta_tree_get_info(ta_ctx* ctx, ta_tree_info* out);
/* snapshot in ascending id order; *n receives node count */
ta_status ta_tree_snapshot(ta_ctx* ctx, int32_t* ids, int32_t* parents, int64_t* counts,
                           int cap, int* n);

/* ---- PagePool accounting ------------------------------------------------ */
ta_status ta_pool_stats(ta_ctx* ctx, int64_t* page_count, int64_t* free_pages,
                        int64_t* live_slots);
ta_status ta_pool_token_ref(ta_ctx* ctx, int32_t node, int64_t token, int32_t* page,
                            int32_t* slot);

/* ---- KV content ----------------------------------------------------------
 * Rows [n_tok][n_local_kv_heads][d_head] in kv_dtype, for tokens
 * [tok_begin, tok_begin+n_tok) of `node` in `layer`.  src_on_device selects
 * device or host source pointers.  stream: cudaStream_t (NULL = default). */
ta_status ta_kv_write(ta_ctx* ctx, int layer, int32_t node, int64_t tok_begin, int64_t n_tok,
                      const void* k, const void* v, int src_on_device, void* stream);

/* ---- Decode-step KV append (PagePool::write_kv of the step's new tokens,
 * kv_cache.hpp:104-116, batched and asynchronous).  The pool rows of every
 * token appended (ta_tree_append / ta_tree_append_leaves) since the previous
 * ta_prepare are uploaded by the next ta_prepare; ta_kv_append then writes
 * that layer's rows k, v [n_rows][n_local_kv_heads][d_head] (device, in
 * append order) with one kernel and no host synchronisation.  The row count
 * is read on the device, so the call can live in a captured CUDA graph.
 * With the tcgen05 kernel (bf16, d 128, fused merge) and option
 * "fuse_append" (default 1) the call launches nothing: it records k / v, and
 * the layer's next ta_attend writes each row from the CTA that loads it,
 * right before its tile (k / v must stay valid until that ta_attend). */
ta_status ta_kv_append(ta_ctx* ctx, int layer, const void* k, const void* v, void* stream);
/* rows the last ta_prepare uploaded for ta_kv_append */
int64_t ta_kv_append_rows(ta_ctx* ctx);
/* Captured launches (ta_attend, ta_kv_append in a CUDA graph) stay valid
 * across ta_prepare calls while this value is unchanged; it changes when a
 * larger schedule relocates the metadata / scratch buffers. */
int64_t ta_graph_epoch(ta_ctx* ctx);

/* ---- Plan (bit-exact partition_flatten) ---------------------------------- */
typedef struct ta_plan_view {
    int block_size;
    int n_groups;
    const int32_t* seg_begin;   /* [n_groups+1] */
    const int32_t* q_begin;     /* [n_groups+1] */
    const int32_t* seg_node;    /* [n_segs] */
    const int64_t* seg_offset;
    const int64_t* seg_len;
    const uint64_t* seg_mask;
    const int32_t* queries;     /* leaf NodeIds */
} ta_plan_view;
/* The context's plan (partition_flatten unless the "strategy" option selects
 * another partition.hpp strategy); arrays stay valid until the next plan call
 * on this context */
ta_status ta_plan_flatten(ta_ctx* ctx, int block_size, ta_plan_view* out);
/* plan_to_json(make_plan(tree, strategy, bs)).dump(); *len excludes the NUL */
ta_status ta_plan_json(ta_ctx* ctx, int block_size, char* buf, size_t cap, size_t* len);
/* io_measured(make_plan(tree, strategy, bs), params) (io_model.hpp:158-170) */
ta_status ta_io_measured(ta_ctx* ctx, int block_size, const ta_cost_params* params, ta_io_report* out);
/* io_analytical(tree, algorithm, params, bs) (io_model.hpp:88-153) */
ta_status ta_io_analytical(ta_ctx* ctx, int algorithm, const ta_cost_params* params, int block_size,
                           ta_io_report* out);

/* ---- Attention ------------------------------------------------------------
 * ta_prepare: plan + device schedule + metadata upload for the current tree
 * (once per decode step; reused by every layer).  ta_attend: one layer;
 * q  [n_leaves][n_local_q_heads][d_head] in kv_dtype, leaves() order;
 * out [n_leaves][n_local_q_heads][d_head] in out_dtype;
 * lse (optional, may be NULL) [n_leaves][n_local_q_heads] fp32, natural log.
 * Leaves whose path holds no tokens get lse = -inf and out = 0 (they are
 * absent from the reference's AttentionOutput map).
 * Ordering: ta_attend waits for the previous kernel on `stream` before it
 * reads q or writes out / lse (programmatic dependent launch).  KV pools are
 * written only by ta_kv_write (synchronous) and ta_kv_append (rows known at
 * ta_prepare), so with option "early_kv" = 1 a CTA starts loading its
 * leading KV tiles -- those no pending ta_kv_append row touches -- before
 * that wait (off by default; a caller that writes the pools by other means
 * on the same stream must leave it off). */
ta_status ta_prepare(ta_ctx* ctx, int block_size, void* stream);
/* Decode-step fast path of ta_prepare: when the only mutations since the last
 * ta_prepare are ta_tree_append_leaves and every new token extends its leaf's
 * tail group of the current device schedule (same page, group not full), the
 * schedule is patched in place instead of re-planned (the flatten plan is
 * rebuilt on demand by the plan queries).  Number of such prepares so far. */
int64_t ta_fast_prepares(ta_ctx* ctx);
ta_status ta_attend(ta_ctx* ctx, int layer, const void* q, void* out, float* lse, void* stream);
/* End-to-end variant over HOST buffers (pinned or pageable): H2D q, attend,
 * D2H out, synchronised on `stream` before returning. */
ta_status ta_attend_host(ta_ctx* ctx, int layer, const void* q_host, void* out_host,
                         void* stream);
/* Pipelined host-buffer variant: enqueues H2D q (context copy-in stream),
 * attend (on `stream`), D2H out (context copy-out stream) and returns.
 * Consecutive calls overlap the copy-in of one call, the attention of the
 * previous one and the copy-out of the one before (three device slots).  Host
 * buffers should be pinned for the copies to be asynchronous; out_host is
 * complete after ta_attend_host_wait.  Reference analogue: run_iteration's
 * host-side inputs and AttentionOutput (attention.hpp:293-334), batched. */
ta_status ta_attend_host_async(ta_ctx* ctx, int layer, const void* q_host, void* out_host,
                               void* stream);
ta_status ta_attend_host_wait(ta_ctx* ctx);

/* Cross-GPU prefix split: merge n_parts partial results of the
 * same rows -- each the attention of a row over a disjoint token range, as
 * ta_attend returns it (out fp32 normalised, lse natural log, -inf for a row
 * with no tokens in that range) -- into the attention over the union:
 * tree_reduce (attention.hpp:209-233) in part order.  part_o [n_parts][rows][d]
 * fp32, part_lse [n_parts][rows]; out [rows][d] (out_bf16: bf16 else fp32),
 * lse_out [rows] (optional).  Device pointers, 16-byte aligned; d % 4 == 0,
 * n_parts <= 32.  No context needed (device = the current one). */
ta_status ta_lse_merge(const float* part_o, const float* part_lse, int n_parts, int64_t rows, int d, void* out,
                       int out_bf16, float* lse_out, void* stream);

typedef struct ta_io_stats {
    int64_t n_chunks;          /* flatten chunks (sibling groups fused) */
    int64_t n_groups;          /* reference QkvGroups */
    int64_t n_units;           /* items (CTA work runs, all local kv heads) */
    int64_t n_units_mma;       /* items run by the tcgen05 kernel */
    int64_t n_partials;        /* (unit, query) partial records per kv head */
    int64_t kv_bytes;          /* unique KV bytes read per layer (this shard) */
    int64_t kv_bytes_loaded;   /* KV bytes the schedule loads (incl. row-block re-reads) */
    int64_t q_bytes;           /* query bytes per layer */
    int64_t out_bytes;         /* output bytes per layer */
    int64_t partial_bytes;     /* off-chip partial (m,l,O) bytes written+read per layer */
    int64_t meta_bytes;        /* schedule metadata uploaded per step */
    int64_t flops;             /* masked-in attention flops per layer (4*d per q-head-token) */
    int64_t host_plan_ns;      /* last ta_prepare: plan (partition) time on the host */
    int64_t host_schedule_ns;  /* ... device-schedule build */
    int64_t host_upload_ns;    /* ... staging copy + upload enqueue (excluding any wait for the GPU) */
} ta_io_stats;
ta_status ta_io_stats_get(ta_ctx* ctx, ta_io_stats* out);

/* Device schedule of the current tree (built on the host; works on host-only
 * contexts; layout described in DESIGN.md section 3).  CTA c runs items
 * [cta_begin[c], cta_begin[c+1]).  items: [n_items][8] int32 = {head,
 * tile_begin, tile_end, slot_begin, n_slots, out_begin, lane, flags}.
 * tiles: [n_tiles][4] int32 = raw 16-byte tile records {grp_begin,
 * ng | nbox << 8 | ntok << 16, boxes 0-3, boxes 4-7}.  Group g covers
 * (grp_info[g] & 0xff) tokens at pool rows grp_row[g] + i (row = page *
 * page_tokens + slot), attended by the item's local slots
 * [(info >> 8) & 0xfff, info >> 20).  slot_out per item slot: -1 - leaf
 * (final output written directly), a partial id, or INT32_MIN (slot unused
 * by the item).  Arrays stay valid until the next schedule call. */
typedef struct ta_schedule_view {
    int32_t n_ctas;
    const int32_t* cta_begin;   /* [n_ctas + 1] */
    int32_t n_items;
    const int32_t* items;
    int32_t n_tiles;
    const int32_t* tiles;
    int32_t n_grp;
    const int32_t* grp_row;
    const uint32_t* grp_info;
    int32_t n_slot_leaf;
    const int32_t* slot_leaf;   /* leaf index in leaves() order */
    int32_t n_slot_out;
    const int32_t* slot_out;
    int32_t n_partials;
    const int32_t* part_merge;  /* partial id -> merge record */
    int32_t n_merge;
    const int32_t* merge_leaf;
    const int32_t* merge_head;
    const int32_t* merge_begin; /* [n_merge + 1] */
    const int32_t* merge_parts;
    int32_t n_empty;
    const int32_t* empty;       /* [n_empty][2] (leaf, local kv head) */
    int32_t n_lanes;
    int32_t use_mma;
    int32_t fused_merge;        /* 1: records merged at the end of the attention launch: CTA c
                                   publishes cta_pub[cta_pub_begin[c] ..] = (record, partials it
                                   wrote), then merges records cta_own[cta_own_begin[c] ..] */
    const int32_t* cta_pub_begin;  /* [n_ctas + 1] (fused_merge only, else NULL) */
    const int32_t* cta_pub;        /* [n][2] */
    const int32_t* cta_own_begin;  /* [n_ctas + 1] */
    const int32_t* cta_own;        /* [n_merge] */
} ta_schedule_view;
ta_status ta_schedule_get(ta_ctx* ctx, int block_size, ta_schedule_view* out);

/* number of kernels ta_attend launches per call (for launch accounting) */
int ta_launches_per_attend(ta_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
