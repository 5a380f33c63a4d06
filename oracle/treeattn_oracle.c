/*
 * treeattn_oracle.c -- plain-C restatement of the reference's DeFT-Flatten
 * decode path (/root/reference/proj/include/treeattn/*.hpp).
 *
 * TEST INFRASTRUCTURE ONLY (see treeattn_oracle.h).  It is the checker the
 * CUDA path is compared against; it is never linked into the product.
 *
 * Parity of this restatement is pinned against the reference itself: the
 * golden fixtures in tests/golden/ are produced by oracle/_ref (the unmodified
 * reference headers compiled by oracle/Makefile) via oracle/make_golden.py,
 * and tests/test_oracle_golden.py checks this file against them.
 *
 * Build flags matter for bit-exactness with the reference: -O2 without
 * -march=native (x86-64 baseline has no FMA, so no contraction) and
 * -ffp-contract=off, identical to the _ref build.
 */
#include "treeattn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ========================================================================
 * std::mt19937_64 (C++11 [rand.eng.mt] parameters) and the libstdc++-13
 * distribution algorithms used by synth.hpp / workloads.hpp.
 * ====================================================================== */
#define MT_N 312
#define MT_M 156

void to_rng_seed(to_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

static void mt_twist(to_rng* r) {
    const uint64_t upper = ~0ULL << 31, lower = ~upper, a = 0xb5026f5aa96619e9ULL;
    int k;
    for (k = 0; k < MT_N - MT_M; ++k) {
        uint64_t y = (r->mt[k] & upper) | (r->mt[k + 1] & lower);
        r->mt[k] = r->mt[k + MT_M] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    for (; k < MT_N - 1; ++k) {
        uint64_t y = (r->mt[k] & upper) | (r->mt[k + 1] & lower);
        r->mt[k] = r->mt[k + (MT_M - MT_N)] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    uint64_t y = (r->mt[MT_N - 1] & upper) | (r->mt[0] & lower);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    r->idx = 0;
}

uint64_t to_rng_next(to_rng* r) {
    if (r->idx >= MT_N) mt_twist(r);
    uint64_t z = r->mt[r->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71d67fffeda60000ULL;
    z ^= (z << 37) & 0xfff7eee000000000ULL;
    z ^= (z >> 43);
    return z;
}

/* generate_canonical<float, 24>(mt19937_64): one draw, float(x) / 2^64,
 * clamped below 1 with nextafter; then a + (b - a) * u in float. */
float to_rng_uniform_float(to_rng* r, float a, float b) {
    float sum = (float)to_rng_next(r);
    float tmp = 18446744073709551616.0f; /* 2^64, exact in float */
    float u = sum / tmp;
    if (u >= 1.0f) u = nextafterf(1.0f, 0.0f);
    return u * (b - a) + a;
}

/* uniform_int_distribution downscaling path for a 64-bit generator:
 * Lemire's nearly-divisionless method with 128-bit products (_S_nd). */
int64_t to_rng_uniform_int(to_rng* r, int64_t a, int64_t b) {
    uint64_t urange = (uint64_t)b - (uint64_t)a;
    uint64_t ret;
    if (urange == ~0ULL) {
        ret = to_rng_next(r);
    } else {
        uint64_t erange = urange + 1;
        unsigned __int128 product = (unsigned __int128)to_rng_next(r) * erange;
        uint64_t low = (uint64_t)product;
        if (low < erange) {
            uint64_t threshold = (0 - erange) % erange;
            while (low < threshold) {
                product = (unsigned __int128)to_rng_next(r) * erange;
                low = (uint64_t)product;
            }
        }
        ret = (uint64_t)(product >> 64);
    }
    return (int64_t)(ret + (uint64_t)a);
}

/* ========================================================================
 * synth.hpp:20-69
 * ====================================================================== */
uint64_t to_mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

uint64_t to_content_seed(uint64_t seed, uint64_t a, uint64_t b) {
    return to_mix64(seed ^ to_mix64(a * 0x9e3779b97f4a7c15ULL + b));
}

void to_fill_uniform(float* v, int64_t n, uint64_t seed) {
    to_rng r;
    to_rng_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) v[i] = to_rng_uniform_float(&r, -1.0f, 1.0f);
}

void to_fill_node_kv(int32_t node, int64_t t0, int64_t n, int dim, uint64_t seed,
                     float* keys, float* values) {
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t t = (uint64_t)(t0 + i);
        if (keys) to_fill_uniform(keys + i * dim, dim, to_content_seed(seed, (uint64_t)node, 2 * t));
        if (values)
            to_fill_uniform(values + i * dim, dim, to_content_seed(seed, (uint64_t)node, 2 * t + 1));
    }
}

void to_fill_query(int32_t leaf, int dim, uint64_t seed, float* q) {
    to_fill_uniform(q, dim, to_content_seed(seed ^ 0xabcdef12ULL, (uint64_t)leaf, 0));
}

/* ========================================================================
 * DecodingTree (tree.hpp:38-269): ids are sequential and never reused;
 * children in insertion order; leaves() is the DFS pre-order leaf list.
 * ====================================================================== */
struct to_tree {
    int cap;
    int32_t next_id;
    int32_t root;
    int n_alive;
    uint8_t* alive;
    int32_t* parent;
    int64_t* count;
    int32_t** kids;
    int* n_kids;
    int* kids_cap;
    int32_t* leaves;
    int n_leaves;
};

static void tree_reserve(to_tree* t, int need) {
    if (need <= t->cap) return;
    int nc = t->cap ? t->cap : 16;
    while (nc < need) nc *= 2;
    t->alive = (uint8_t*)realloc(t->alive, (size_t)nc);
    t->parent = (int32_t*)realloc(t->parent, sizeof(int32_t) * nc);
    t->count = (int64_t*)realloc(t->count, sizeof(int64_t) * nc);
    t->kids = (int32_t**)realloc(t->kids, sizeof(int32_t*) * nc);
    t->n_kids = (int*)realloc(t->n_kids, sizeof(int) * nc);
    t->kids_cap = (int*)realloc(t->kids_cap, sizeof(int) * nc);
    t->leaves = (int32_t*)realloc(t->leaves, sizeof(int32_t) * nc);
    for (int i = t->cap; i < nc; ++i) {
        t->alive[i] = 0;
        t->parent[i] = -1;
        t->count[i] = 0;
        t->kids[i] = NULL;
        t->n_kids[i] = 0;
        t->kids_cap[i] = 0;
    }
    t->cap = nc;
}

static void kid_push(to_tree* t, int32_t p, int32_t c) {
    if (t->n_kids[p] == t->kids_cap[p]) {
        t->kids_cap[p] = t->kids_cap[p] ? 2 * t->kids_cap[p] : 4;
        t->kids[p] = (int32_t*)realloc(t->kids[p], sizeof(int32_t) * t->kids_cap[p]);
    }
    t->kids[p][t->n_kids[p]++] = c;
}

static int alive(const to_tree* t, int32_t id) {
    return id >= 0 && id < t->cap && t->alive[id];
}

/* tree.hpp:298-301 pre-order, children in stored order (iterative) */
static int dfs_from(const to_tree* t, int32_t at, int32_t* out) {
    int n = 0, sp = 0;
    int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * (size_t)(t->cap + 1));
    stack[sp++] = at;
    while (sp) {
        int32_t v = stack[--sp];
        out[n++] = v;
        for (int i = t->n_kids[v] - 1; i >= 0; --i) stack[sp++] = t->kids[v][i];
    }
    free(stack);
    return n;
}

/* tree.hpp:309-314 */
static void rebuild_leaves(to_tree* t) {
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)t->cap);
    int n = dfs_from(t, t->root, order);
    t->n_leaves = 0;
    for (int i = 0; i < n; ++i)
        if (t->n_kids[order[i]] == 0) t->leaves[t->n_leaves++] = order[i];
    free(order);
}

static to_tree* tree_alloc(void) {
    to_tree* t = (to_tree*)calloc(1, sizeof(to_tree));
    t->root = -1;
    return t;
}

to_tree* to_tree_new(int64_t root_tokens) {
    if (root_tokens < 1) return NULL; /* invalid_argument in tree.hpp:42-43 */
    to_tree* t = tree_alloc();
    tree_reserve(t, 16);
    t->root = t->next_id++;
    t->alive[t->root] = 1;
    t->count[t->root] = root_tokens;
    t->parent[t->root] = -1;
    t->n_alive = 1;
    rebuild_leaves(t);
    return t;
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

to_tree* to_tree_restore(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                         const int64_t* counts) {
    to_tree* t = tree_alloc();
    int32_t maxid = root;
    for (int i = 0; i < n; ++i) {
        if (ids[i] < 0) { to_tree_free(t); return NULL; }
        if (ids[i] > maxid) maxid = ids[i];
    }
    tree_reserve(t, maxid + 1);
    t->root = root;
    for (int i = 0; i < n; ++i) {
        if (t->alive[ids[i]]) { to_tree_free(t); return NULL; } /* duplicate node id */
        t->alive[ids[i]] = 1;
        t->parent[ids[i]] = parents[i];
        t->count[ids[i]] = counts[i];
        if (ids[i] + 1 > t->next_id) t->next_id = ids[i] + 1;
    }
    t->n_alive = n;
    if (!alive(t, root)) { to_tree_free(t); return NULL; }
    /* children pushed in ascending id order (std::map iteration, tree.hpp:223-233) */
    int32_t* sorted = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    memcpy(sorted, ids, sizeof(int32_t) * (size_t)n);
    qsort(sorted, (size_t)n, sizeof(int32_t), cmp_i32);
    for (int i = 0; i < n; ++i) {
        int32_t id = sorted[i];
        if (id == root) {
            if (t->parent[id] != -1) { free(sorted); to_tree_free(t); return NULL; }
            continue;
        }
        if (!alive(t, t->parent[id])) { free(sorted); to_tree_free(t); return NULL; }
        kid_push(t, t->parent[id], id);
    }
    free(sorted);
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)t->cap);
    /* guard against cycles: cap the walk */
    int reach = dfs_from(t, root, order);
    free(order);
    if (reach != n) { to_tree_free(t); return NULL; }
    rebuild_leaves(t);
    return t;
}

void to_tree_free(to_tree* t) {
    if (!t) return;
    for (int i = 0; i < t->cap; ++i) free(t->kids[i]);
    free(t->alive); free(t->parent); free(t->count); free(t->kids);
    free(t->n_kids); free(t->kids_cap); free(t->leaves);
    free(t);
}

int to_tree_branch(to_tree* t, int32_t at, int n, const int64_t* counts, int32_t* created) {
    if (!alive(t, at)) return -2;
    if (t->n_kids[at] != 0) return -1;
    for (int i = 0; i < n; ++i)
        if (counts[i] < 0) return -1;
    tree_reserve(t, t->next_id + n + 1);
    for (int i = 0; i < n; ++i) {
        int32_t id = t->next_id++;
        t->alive[id] = 1;
        t->parent[id] = at;
        t->count[id] = counts[i];
        t->n_kids[id] = 0;
        kid_push(t, at, id);
        if (created) created[i] = id;
        t->n_alive++;
    }
    rebuild_leaves(t);
    return 0;
}

int to_tree_prune(to_tree* t, int32_t at) {
    if (at == t->root) return -1;
    if (!alive(t, at)) return -2;
    int32_t p = t->parent[at];
    for (int i = 0; i < t->n_kids[p]; ++i)
        if (t->kids[p][i] == at) {
            memmove(&t->kids[p][i], &t->kids[p][i + 1], sizeof(int32_t) * (size_t)(t->n_kids[p] - i - 1));
            t->n_kids[p]--;
            break;
        }
    int32_t* doomed = (int32_t*)malloc(sizeof(int32_t) * (size_t)t->cap);
    int nd = dfs_from(t, at, doomed);
    for (int i = 0; i < nd; ++i) {
        t->alive[doomed[i]] = 0;
        t->n_kids[doomed[i]] = 0;
        t->n_alive--;
    }
    free(doomed);
    rebuild_leaves(t);
    return 0;
}

int to_tree_append(to_tree* t, int32_t leaf, int64_t n) {
    if (!alive(t, leaf)) return -2;
    if (t->n_kids[leaf] != 0) return -1;
    if (n < 1) return -1;
    t->count[leaf] += n;
    return 0;
}

int32_t to_tree_root(const to_tree* t) { return t->root; }
int to_tree_node_count(const to_tree* t) { return t->n_alive; }
int to_tree_n_leaves(const to_tree* t) { return t->n_leaves; }
const int32_t* to_tree_leaves(const to_tree* t) { return t->leaves; }
int64_t to_tree_token_count(const to_tree* t, int32_t id) { return alive(t, id) ? t->count[id] : -1; }
int32_t to_tree_parent(const to_tree* t, int32_t id) { return alive(t, id) ? t->parent[id] : -1; }

int64_t to_tree_total_tokens(const to_tree* t) {
    int64_t s = 0;
    for (int i = 0; i < t->cap; ++i)
        if (t->alive[i]) s += t->count[i];
    return s;
}

int64_t to_tree_path_tokens(const to_tree* t, int32_t leaf) {
    int64_t s = 0;
    for (int32_t cur = leaf; cur != -1; cur = t->parent[cur]) s += t->count[cur];
    return s;
}

int to_tree_snapshot(const to_tree* t, int32_t* ids, int32_t* parents, int64_t* counts) {
    int n = 0;
    for (int i = 0; i < t->cap; ++i)
        if (t->alive[i]) {
            if (ids) ids[n] = i;
            if (parents) parents[n] = t->parent[i];
            if (counts) counts[n] = t->count[i];
            n++;
        }
    return n;
}

int to_tree_dfs(const to_tree* t, int32_t* out) { return dfs_from(t, t->root, out); }

/* synth.hpp:80-111 */
to_tree* to_random_tree(to_rng* rng, int max_leaves, int64_t max_tokens, int64_t max_node_tokens,
                        int max_branch_width, int mutation_steps) {
    to_tree* t = to_tree_new(to_rng_uniform_int(rng, 1, max_node_tokens));
    int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)(max_branch_width + 1));
    for (int step = 0; step < mutation_steps; ++step) {
        const int nl = t->n_leaves;
        const int32_t leaf = t->leaves[to_rng_uniform_int(rng, 0, nl - 1)];
        const int can_branch = nl + max_branch_width <= max_leaves &&
                               to_tree_total_tokens(t) + max_branch_width <= max_tokens;
        if (can_branch && to_rng_next(rng) % 3 == 0) {
            const int w = (int)to_rng_uniform_int(rng, 2, max_branch_width);
            int64_t budget = max_tokens - to_tree_total_tokens(t);
            for (int i = 0; i < w; ++i) {
                int64_t c = to_rng_uniform_int(rng, 1, max_node_tokens);
                int64_t cap = budget / w;
                if (cap < 1) cap = 1;
                if (cap < c) c = cap;
                counts[i] = c;
                budget -= c;
            }
            to_tree_branch(t, leaf, w, counts, NULL);
        } else {
            int64_t n = to_rng_uniform_int(rng, 1, max_node_tokens / 4 + 1);
            int64_t room = max_tokens - to_tree_total_tokens(t);
            if (room < n) n = room;
            if (n >= 1) to_tree_append(t, leaf, n);
        }
    }
    free(counts);
    return t;
}

/* ========================================================================
 * partition.hpp: AncestorIndex (:76-95), emit_groups (:102-126),
 * partition_flatten (:212-253).  Restated literally: queries_for_node walks
 * the subtree and filters leaves() (tree.hpp:169-178); the ancestor test
 * walks parent links.
 * ====================================================================== */
static int attends(const to_tree* t, int32_t leaf, int32_t node) {
    for (int32_t cur = leaf; cur != -1; cur = t->parent[cur])
        if (cur == node) return 1;
    return 0;
}

static void plan_push_group(to_plan* p) {
    if (p->n_groups + 2 > p->g_cap) {
        p->g_cap = p->g_cap ? 2 * p->g_cap : 64;
        p->group_id = (int*)realloc(p->group_id, sizeof(int) * (size_t)p->g_cap);
        p->seg_begin = (int*)realloc(p->seg_begin, sizeof(int) * (size_t)p->g_cap);
        p->q_begin = (int*)realloc(p->q_begin, sizeof(int) * (size_t)p->g_cap);
    }
}

static void plan_push_seg(to_plan* p, int at, int32_t node, int64_t off, int64_t len, uint64_t mask) {
    if (at + 1 > p->seg_cap) {
        p->seg_cap = p->seg_cap ? 2 * p->seg_cap : 256;
        p->seg_node = (int32_t*)realloc(p->seg_node, sizeof(int32_t) * (size_t)p->seg_cap);
        p->seg_offset = (int64_t*)realloc(p->seg_offset, sizeof(int64_t) * (size_t)p->seg_cap);
        p->seg_len = (int64_t*)realloc(p->seg_len, sizeof(int64_t) * (size_t)p->seg_cap);
        p->seg_mask = (uint64_t*)realloc(p->seg_mask, sizeof(uint64_t) * (size_t)p->seg_cap);
    }
    p->seg_node[at] = node;
    p->seg_offset[at] = off;
    p->seg_len[at] = len;
    p->seg_mask[at] = mask;
}

static void plan_push_query(to_plan* p, int at, int32_t q) {
    if (at + 1 > p->q_cap) {
        p->q_cap = p->q_cap ? 2 * p->q_cap : 256;
        p->queries = (int32_t*)realloc(p->queries, sizeof(int32_t) * (size_t)p->q_cap);
    }
    p->queries[at] = q;
}

/* partition.hpp:102-126 */
static void emit_groups(to_plan* p, const to_tree* t, int n_pend, const int32_t* pn,
                        const int64_t* po, const int64_t* pl, int nq, const int32_t* queries) {
    const int split = nq > 64;
    for (int base = 0; base < nq; base += 64) {
        const int count = (nq - base) < 64 ? (nq - base) : 64;
        plan_push_group(p);
        const int g = p->n_groups;
        const int s0 = p->seg_begin[g], q0 = p->q_begin[g];
        int ns = 0, any = 0;
        for (int j = 0; j < count; ++j) plan_push_query(p, q0 + j, queries[base + j]);
        for (int s = 0; s < n_pend; ++s) {
            uint64_t mask = 0;
            for (int j = 0; j < count; ++j)
                if (attends(t, queries[base + j], pn[s])) mask |= 1ULL << j;
            if (mask == 0 && !split) continue;
            plan_push_seg(p, s0 + ns, pn[s], po[s], pl[s], mask);
            ns++;
            any = any || mask != 0;
        }
        if (any) {
            p->group_id[g] = g;
            p->n_groups++;
            p->seg_begin[g + 1] = s0 + ns;
            p->q_begin[g + 1] = q0 + count;
        }
    }
}

to_plan* to_partition_flatten(const to_tree* t, int block_size) {
    if (block_size < 1) return NULL;
    to_plan* p = (to_plan*)calloc(1, sizeof(to_plan));
    p->block_size = block_size;
    plan_push_group(p);
    p->seg_begin[0] = 0;
    p->q_begin[0] = 0;

    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)t->cap);
    int n_order = dfs_from(t, t->root, order);
    int32_t* sub = (int32_t*)malloc(sizeof(int32_t) * (size_t)t->cap);
    uint8_t* qset = (uint8_t*)calloc((size_t)t->cap, 1);
    uint8_t* want = (uint8_t*)calloc((size_t)t->cap, 1);
    int32_t* ordered = (int32_t*)malloc(sizeof(int32_t) * (size_t)(t->n_leaves + 1));
    int cap_pend = 64, n_pend = 0;
    int32_t* pn = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap_pend);
    int64_t* po = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap_pend);
    int64_t* pl = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap_pend);
    int64_t fill = 0;

    for (int oi = 0; oi <= n_order; ++oi) {
        const int final_flush = oi == n_order;
        int64_t remaining = final_flush ? 0 : t->count[order[oi]];
        int64_t offset = 0;
        const int32_t id = final_flush ? -1 : order[oi];
        for (;;) {
            int do_flush = 0;
            if (!final_flush && remaining > 0) {
                int64_t take = remaining < (block_size - fill) ? remaining : (block_size - fill);
                if (n_pend == cap_pend) {
                    cap_pend *= 2;
                    pn = (int32_t*)realloc(pn, sizeof(int32_t) * (size_t)cap_pend);
                    po = (int64_t*)realloc(po, sizeof(int64_t) * (size_t)cap_pend);
                    pl = (int64_t*)realloc(pl, sizeof(int64_t) * (size_t)cap_pend);
                }
                pn[n_pend] = id; po[n_pend] = offset; pl[n_pend] = take; n_pend++;
                /* add_queries_of(id): queries_for_node (tree.hpp:169-178) */
                if (t->n_kids[id] == 0) {
                    qset[id] = 1;
                } else {
                    int ns = dfs_from(t, id, sub);
                    for (int i = 0; i < ns; ++i)
                        if (t->n_kids[sub[i]] == 0) want[sub[i]] = 1;
                    for (int i = 0; i < t->n_leaves; ++i)
                        if (want[t->leaves[i]]) qset[t->leaves[i]] = 1;
                    for (int i = 0; i < ns; ++i) want[sub[i]] = 0;
                }
                offset += take;
                remaining -= take;
                fill += take;
                if (fill == block_size) do_flush = 1;
            } else if (final_flush) {
                do_flush = 1;
            }
            if (do_flush && n_pend > 0) {
                int nq = 0;
                for (int i = 0; i < t->n_leaves; ++i)
                    if (qset[t->leaves[i]]) ordered[nq++] = t->leaves[i];
                emit_groups(p, t, n_pend, pn, po, pl, nq, ordered);
                for (int i = 0; i < t->n_leaves; ++i) qset[t->leaves[i]] = 0;
                n_pend = 0;
                fill = 0;
            }
            if (final_flush || remaining <= 0) break;
        }
    }
    free(order); free(sub); free(qset); free(want); free(ordered);
    free(pn); free(po); free(pl);
    return p;
}

void to_plan_free(to_plan* p) {
    if (!p) return;
    free(p->group_id); free(p->seg_begin); free(p->q_begin);
    free(p->seg_node); free(p->seg_offset); free(p->seg_len); free(p->seg_mask);
    free(p->queries);
    free(p);
}

/* ========================================================================
 * attention.hpp:117-204  group_attention<Scalar>
 * ====================================================================== */
#define DEFINE_GROUP_ATTN(NAME, S, EXP, SQRT)                                                    \
static int NAME(const to_plan* p, int g, const float* const* queries, const to_kv* kv,          \
                int d_head, int n_heads, int tile_size, int32_t* part_query,                    \
                double* part_out, double* part_lse) {                                           \
    const int dim = d_head * n_heads;                                                           \
    const int s0 = p->seg_begin[g], s1 = p->seg_begin[g + 1];                                   \
    int n_tokens = 0;                                                                           \
    for (int s = s0; s < s1; ++s) n_tokens += (int)p->seg_len[s];                               \
    const float** krow = (const float**)malloc(sizeof(float*) * (size_t)(n_tokens + 1));       \
    const float** vrow = (const float**)malloc(sizeof(float*) * (size_t)(n_tokens + 1));       \
    uint64_t* tmask = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n_tokens + 1));            \
    int k = 0;                                                                                  \
    for (int s = s0; s < s1; ++s)                                                               \
        for (int64_t t = 0; t < p->seg_len[s]; ++t, ++k) {                                      \
            const int64_t tok = p->seg_offset[s] + t;                                           \
            krow[k] = kv->keys[p->seg_node[s]] + tok * dim;                                     \
            vrow[k] = kv->values[p->seg_node[s]] + tok * dim;                                   \
            tmask[k] = p->seg_mask[s];                                                          \
        }                                                                                       \
    const S scale = (S)1 / SQRT((S)d_head);                                                     \
    S* qv = (S*)malloc(sizeof(S) * (size_t)dim);                                                \
    S* acc = (S*)malloc(sizeof(S) * (size_t)d_head);                                            \
    S* scores = (S*)malloc(sizeof(S) * (size_t)(tile_size + 1));                                \
    int n_out = 0;                                                                              \
    const int q0 = p->q_begin[g], q1 = p->q_begin[g + 1];                                       \
    for (int j = 0; j < q1 - q0; ++j) {                                                         \
        const int32_t leaf = p->queries[q0 + j];                                                \
        const float* qsrc = queries[leaf];                                                      \
        if (!qsrc) { n_out = -1; break; }                                                       \
        for (int i = 0; i < dim; ++i) qv[i] = (S)qsrc[i];                                       \
        double* pout = part_out + (size_t)n_out * dim;                                          \
        double* plse = part_lse + (size_t)n_out * n_heads;                                      \
        int attended_any = 0;                                                                   \
        for (int h = 0; h < n_heads; ++h) {                                                     \
            const S* qh = qv + (size_t)h * d_head;                                              \
            S run_max = -(S)INFINITY, run_den = 0;                                              \
            for (int d = 0; d < d_head; ++d) acc[d] = 0;                                        \
            int attended = 0;                                                                   \
            for (int tile = 0; tile < n_tokens; tile += tile_size) {                            \
                const int tile_end = n_tokens < tile + tile_size ? n_tokens : tile + tile_size; \
                S tile_max = -(S)INFINITY;                                                      \
                int tile_any = 0;                                                               \
                for (int t = tile; t < tile_end; ++t) {                                         \
                    if (!((tmask[t] >> j) & 1)) continue;                                       \
                    const float* kk = krow[t] + (size_t)h * d_head;                             \
                    S dacc = 0;                                                                 \
                    for (int i = 0; i < d_head; ++i) dacc += qh[i] * (S)kk[i];                  \
                    const S sc = dacc * scale;                                                  \
                    scores[t - tile] = sc;                                                      \
                    tile_max = (tile_max < sc) ? sc : tile_max;                                 \
                    tile_any = 1;                                                               \
                }                                                                               \
                if (!tile_any) continue;                                                        \
                const S new_max = attended ? ((run_max < tile_max) ? tile_max : run_max)        \
                                           : tile_max;                                          \
                if (attended && new_max != run_max) {                                           \
                    const S r = EXP(run_max - new_max);                                         \
                    run_den *= r;                                                               \
                    for (int d = 0; d < d_head; ++d) acc[d] *= r;                               \
                }                                                                               \
                run_max = new_max;                                                              \
                for (int t = tile; t < tile_end; ++t) {                                         \
                    if (!((tmask[t] >> j) & 1)) continue;                                       \
                    const S w = EXP(scores[t - tile] - run_max);                                \
                    run_den += w;                                                               \
                    const float* vv = vrow[t] + (size_t)h * d_head;                             \
                    for (int d = 0; d < d_head; ++d) acc[d] += w * (S)vv[d];                    \
                }                                                                               \
                attended = 1;                                                                   \
            }                                                                                   \
            if (attended) {                                                                     \
                attended_any = 1;                                                               \
                plse[h] = (double)run_max + log((double)run_den);                               \
                for (int d = 0; d < d_head; ++d)                                                \
                    pout[(size_t)h * d_head + d] = (double)(acc[d] / run_den);                  \
            } else {                                                                            \
                plse[h] = -INFINITY;                                                            \
                for (int d = 0; d < d_head; ++d) pout[(size_t)h * d_head + d] = 0.0;            \
            }                                                                                   \
        }                                                                                       \
        if (attended_any) part_query[n_out++] = leaf;                                           \
    }                                                                                           \
    free(krow); free(vrow); free(tmask); free(qv); free(acc); free(scores);                     \
    return n_out;                                                                               \
}

DEFINE_GROUP_ATTN(group_attention_f, float, expf, sqrtf)
DEFINE_GROUP_ATTN(group_attention_d, double, exp, sqrt)

int to_group_attention(const to_plan* p, int g, const float* const* queries, const to_kv* kv,
                       int d_head, int n_heads, int tile_size, int use_double,
                       int32_t* part_query, double* part_out, double* part_lse) {
    return use_double ? group_attention_d(p, g, queries, kv, d_head, n_heads, tile_size,
                                          part_query, part_out, part_lse)
                      : group_attention_f(p, g, queries, kv, d_head, n_heads, tile_size,
                                          part_query, part_out, part_lse);
}

/* attention.hpp:209-233 */
int to_tree_reduce(int n, const double* const* outs, const double* const* lses, int d_head,
                   int n_heads, double* out) {
    if (n == 0) return -3;
    double* num = (double*)malloc(sizeof(double) * (size_t)d_head);
    for (int h = 0; h < n_heads; ++h) {
        double m = -INFINITY;
        for (int i = 0; i < n; ++i) m = (m < lses[i][h]) ? lses[i][h] : m;
        if (!isfinite(m)) { free(num); return -3; }
        double den = 0;
        for (int d = 0; d < d_head; ++d) num[d] = 0.0;
        for (int i = 0; i < n; ++i) {
            if (!isfinite(lses[i][h])) continue;
            const double w = exp(lses[i][h] - m);
            den += w;
            for (int d = 0; d < d_head; ++d) num[d] += w * outs[i][(size_t)h * d_head + d];
        }
        for (int d = 0; d < d_head; ++d) out[(size_t)h * d_head + d] = num[d] / den;
    }
    free(num);
    return 0;
}

/* attention.hpp:293-334 with Strategy::Flatten */
int to_run_iteration_flatten(const to_tree* t, int block_size, const float* const* queries,
                             const to_kv* kv, int d_head, int n_heads, int tile_size,
                             int use_double, double* out, uint8_t* present) {
    const int dim = d_head * n_heads;
    const int L = t->n_leaves;
    memset(present, 0, (size_t)L);
    int any_query = 0;
    for (int i = 0; i < L; ++i)
        if (queries[t->leaves[i]]) any_query = 1;
    if (!any_query) return 0;
    to_plan* p = to_partition_flatten(t, block_size);
    if (!p) return -1;
    int total_q = p->q_begin[p->n_groups];
    double* pout = (double*)malloc(sizeof(double) * (size_t)(total_q + 1) * dim);
    double* plse = (double*)malloc(sizeof(double) * (size_t)(total_q + 1) * n_heads);
    int32_t* pq = (int32_t*)malloc(sizeof(int32_t) * (size_t)(total_q + 1));
    int n_part = 0;
    int rc = 0;
    for (int g = 0; g < p->n_groups; ++g) {
        int k = to_group_attention(p, g, queries, kv, d_head, n_heads, tile_size, use_double,
                                   pq + n_part, pout + (size_t)n_part * dim,
                                   plse + (size_t)n_part * n_heads);
        if (k < 0) { rc = -1; break; }
        n_part += k;
    }
    if (rc == 0) {
        /* by_query: partials in group order per leaf; reduce per leaf */
        const double** o = (const double**)malloc(sizeof(double*) * (size_t)(n_part + 1));
        const double** l = (const double**)malloc(sizeof(double*) * (size_t)(n_part + 1));
        for (int li = 0; li < L && rc == 0; ++li) {
            const int32_t leaf = t->leaves[li];
            int n = 0;
            for (int i = 0; i < n_part; ++i)
                if (pq[i] == leaf) {
                    o[n] = pout + (size_t)i * dim;
                    l[n] = plse + (size_t)i * n_heads;
                    n++;
                }
            if (n == 0) continue;
            if (to_tree_reduce(n, o, l, d_head, n_heads, out + (size_t)li * dim) != 0) rc = -3;
            present[li] = 1;
        }
        free(o); free(l);
    }
    free(pout); free(plse); free(pq);
    to_plan_free(p);
    return rc;
}

/* attention.hpp:237-288 */
void to_naive_attention(const to_tree* t, const float* const* queries, const to_kv* kv,
                        int d_head, int n_heads, double* out) {
    const int dim = d_head * n_heads;
    const double scale = 1.0 / sqrt((double)d_head);
    int32_t* chain = (int32_t*)malloc(sizeof(int32_t) * (size_t)t->cap);
    for (int li = 0; li < t->n_leaves; ++li) {
        const int32_t leaf = t->leaves[li];
        double* o = out + (size_t)li * dim;
        for (int i = 0; i < dim; ++i) o[i] = 0.0;
        const float* q = queries[leaf];
        if (!q) continue;
        int nc = 0;
        for (int32_t cur = leaf; cur != -1; cur = t->parent[cur]) chain[nc++] = cur;
        int64_t rows = 0;
        for (int c = 0; c < nc; ++c) rows += t->count[chain[c]];
        double* scores = (double*)malloc(sizeof(double) * (size_t)(rows + 1));
        for (int h = 0; h < n_heads; ++h) {
            const float* qh = q + (size_t)h * d_head;
            double m = -INFINITY;
            int64_t r = 0;
            for (int c = nc - 1; c >= 0; --c) {
                const int32_t id = chain[c];
                for (int64_t tk = 0; tk < t->count[id]; ++tk, ++r) {
                    const float* k = kv->keys[id] + tk * dim + (size_t)h * d_head;
                    double s = 0;
                    for (int d = 0; d < d_head; ++d) s += (double)qh[d] * (double)k[d];
                    scores[r] = s * scale;
                    m = (m < scores[r]) ? scores[r] : m;
                }
            }
            double den = 0;
            for (int64_t i = 0; i < rows; ++i) den += exp(scores[i] - m);
            r = 0;
            for (int c = nc - 1; c >= 0; --c) {
                const int32_t id = chain[c];
                for (int64_t tk = 0; tk < t->count[id]; ++tk, ++r) {
                    const double w = exp(scores[r] - m) / den;
                    const float* v = kv->values[id] + tk * dim + (size_t)h * d_head;
                    for (int d = 0; d < d_head; ++d) o[(size_t)h * d_head + d] += w * (double)v[d];
                }
            }
        }
        free(scores);
    }
    free(chain);
}

double to_relative_error(const double* got, const double* ref, int64_t n) {
    double md = 0, mr = 0;
    for (int64_t i = 0; i < n; ++i) {
        double d = fabs(got[i] - ref[i]);
        md = md < d ? d : md;
        double a = fabs(ref[i]);
        mr = mr < a ? a : mr;
    }
    return md / (mr + 1e-12);
}
