/*
 * treeattn_oracle.h -- CPU restatement of the reference's DeFT-Flatten path.
 *
 * TEST INFRASTRUCTURE ONLY.  This oracle is the checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product library (paper_2404_00242_b200) never links it.
 *
 * Every function restates one reference function; the citation is next to
 * each declaration (paths relative to /root/reference/proj).
 */
#ifndef TREEATTN_ORACLE_H
#define TREEATTN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- std::mt19937_64 + libstdc++ distributions (synth.hpp:33-37, 80-111) -- */
typedef struct to_rng {
    uint64_t mt[312];
    int idx;
} to_rng;

void to_rng_seed(to_rng* r, uint64_t seed);
uint64_t to_rng_next(to_rng* r);
/* std::uniform_real_distribution<float>(a, b) as implemented by libstdc++ */
float to_rng_uniform_float(to_rng* r, float a, float b);
/* std::uniform_int_distribution<T>(a, b) for any 64-bit-range T (libstdc++ 13) */
int64_t to_rng_uniform_int(to_rng* r, int64_t a, int64_t b);

/* ---- deterministic content (synth.hpp:20-69) ---------------------------- */
uint64_t to_mix64(uint64_t x);                                      /* synth.hpp:20-27 */
uint64_t to_content_seed(uint64_t seed, uint64_t a, uint64_t b);    /* synth.hpp:29-31 */
void to_fill_uniform(float* v, int64_t n, uint64_t seed);           /* synth.hpp:33-37 */
/* K/V rows of tokens [t0, t0+n) of `node`, each `dim` floats (synth.hpp:41-50) */
void to_fill_node_kv(int32_t node, int64_t t0, int64_t n, int dim, uint64_t seed,
                     float* keys, float* values);
/* query vector of `leaf` (synth.hpp:56-69) */
void to_fill_query(int32_t leaf, int dim, uint64_t seed, float* q);

/* ---- DecodingTree (tree.hpp:38-269) ------------------------------------ */
typedef struct to_tree to_tree;

to_tree* to_tree_new(int64_t root_tokens);                          /* tree.hpp:40-51 */
to_tree* to_tree_restore(int32_t root, int n, const int32_t* ids,   /* tree.hpp:207-238 */
                         const int32_t* parents, const int64_t* counts);
void to_tree_free(to_tree* t);
/* error codes: 0 ok, -1 invalid_argument, -2 out_of_range */
int to_tree_branch(to_tree* t, int32_t at, int n, const int64_t* counts,
                   int32_t* created);                               /* tree.hpp:74-97 */
int to_tree_prune(to_tree* t, int32_t at);                          /* tree.hpp:100-116 */
int to_tree_append(to_tree* t, int32_t leaf, int64_t n);            /* tree.hpp:119-129 */
int32_t to_tree_root(const to_tree* t);
int to_tree_node_count(const to_tree* t);
int to_tree_n_leaves(const to_tree* t);
const int32_t* to_tree_leaves(const to_tree* t);                    /* tree.hpp:55, 257-262 */
int64_t to_tree_total_tokens(const to_tree* t);
int64_t to_tree_path_tokens(const to_tree* t, int32_t leaf);        /* tree.hpp:132-141 */
int64_t to_tree_token_count(const to_tree* t, int32_t id);
int32_t to_tree_parent(const to_tree* t, int32_t id);
/* snapshot in ascending id order (workloads.hpp:25-34); returns node count */
int to_tree_snapshot(const to_tree* t, int32_t* ids, int32_t* parents, int64_t* counts);
/* pre-order DFS (tree.hpp:161-166); returns count */
int to_tree_dfs(const to_tree* t, int32_t* out);

/* seeded random tree through the public mutation API (synth.hpp:71-111) */
to_tree* to_random_tree(to_rng* rng, int max_leaves, int64_t max_tokens,
                        int64_t max_node_tokens, int max_branch_width, int mutation_steps);

/* ---- PartitionPlan / partition_flatten (partition.hpp:37-126, 212-253) --- */
typedef struct to_plan {
    int n_groups;
    int block_size;
    int* group_id;        /* [n_groups] */
    int* seg_begin;       /* [n_groups+1] prefix into segs */
    int* q_begin;         /* [n_groups+1] prefix into queries */
    int32_t* seg_node;    /* [n_segs] */
    int64_t* seg_offset;  /* [n_segs] */
    int64_t* seg_len;     /* [n_segs] */
    uint64_t* seg_mask;   /* [n_segs] */
    int32_t* queries;     /* [n_queries] */
    int seg_cap, q_cap, g_cap;
} to_plan;

to_plan* to_partition_flatten(const to_tree* t, int block_size);    /* partition.hpp:212-253 */
void to_plan_free(to_plan* p);

/* ---- attention (attention.hpp:63-288) ---------------------------------- */
/* KV content per node: keys[node] -> [token_count][dim] floats */
typedef struct to_kv {
    int dim;
    int n_nodes;               /* ids 0..n_nodes-1 addressable */
    const float* const* keys;
    const float* const* values;
} to_kv;

/*
 * Stage 1 for one group (attention.hpp:117-204), Scalar=float when
 * use_double==0 else double.  Writes at most |query_ids| partials:
 * part_query[i], part_out[i*dim..], part_lse[i*n_heads..]; returns count.
 * queries[leaf] -> q vector (dim floats).
 */
int to_group_attention(const to_plan* p, int g, const float* const* queries,
                       const to_kv* kv, int d_head, int n_heads, int tile_size,
                       int use_double, int32_t* part_query, double* part_out,
                       double* part_lse);
/* Stage 2 (attention.hpp:209-233): merge n partials; returns 0 or -3 (logic_error) */
int to_tree_reduce(int n, const double* const* outs, const double* const* lses,
                   int d_head, int n_heads, double* out);
/*
 * run_iteration with the Flatten strategy (attention.hpp:293-334).
 * out: [n_leaves][dim] in tree.leaves() order; present[i]=1 iff the leaf
 * appears in the reference's AttentionOutput map.  Returns 0 or error.
 */
int to_run_iteration_flatten(const to_tree* t, int block_size, const float* const* queries,
                             const to_kv* kv, int d_head, int n_heads, int tile_size,
                             int use_double, double* out, uint8_t* present);
/* dense fp64 oracle (attention.hpp:237-288); out [n_leaves][dim] in leaves() order */
void to_naive_attention(const to_tree* t, const float* const* queries, const to_kv* kv,
                        int d_head, int n_heads, double* out);
/* attention.hpp:337-346 */
double to_relative_error(const double* got, const double* ref, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
