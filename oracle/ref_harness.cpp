// ref_harness.cpp -- extern "C" driver over the UNMODIFIED reference headers
// at /root/reference/proj/include (compiled in place by oracle/Makefile into
// oracle/_ref/libtreeattn_ref.so; nothing from the reference is copied here).
//
// TEST INFRASTRUCTURE ONLY: used to (a) generate the golden fixtures under
// tests/golden/ (oracle/make_golden.py) and (b) time the reference CPU path
// for bench.py's `--impl reference` arm / cpu_baseline.  The product never
// links it.
//
// Entry points mirror the reference's public calls:
//   trees / traces  : DecodingTree::restore, gen_few_shot, gen_reasoning,
//                     gen_speculative, preset_trace, random_tree
//   instances       : instance_from_snapshot (+ a GQA expansion and an
//                     arbitrary-content variant), PagePool::write_kv
//   attention       : run_iteration (attention.hpp:293), naive_attention (:237)
//   plan            : make_plan + plan_to_json (serde.hpp:41-61), io_measured
#include <malloc.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "treeattn/treeattn.hpp"

using namespace treeattn;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        g_err = std::string("invalid_argument: ") + e.what();
        return -1;
    } catch (const std::out_of_range& e) {
        g_err = std::string("out_of_range: ") + e.what();
        return -2;
    } catch (const std::logic_error& e) {
        g_err = std::string("logic_error: ") + e.what();
        return -3;
    } catch (const std::exception& e) {
        g_err = std::string("exception: ") + e.what();
        return -4;
    }
}

struct SnapList {
    std::vector<TreeSnapshot> snaps;
    std::vector<int> iteration;
    std::vector<int> query_count;
};

struct Instance {
    std::unique_ptr<PagePool> pool;
    std::unique_ptr<DecodingTree> tree;
    std::map<NodeId, QueryVec> queries;
    AttentionParams params;
};

std::vector<TreeNode> nodes_from(int n, const int32_t* ids, const int32_t* parents,
                                 const int64_t* counts) {
    std::vector<TreeNode> nodes(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
        nodes[i].id = ids[i];
        nodes[i].parent = parents[i];
        nodes[i].token_count = counts[i];
    }
    return nodes;
}

SnapList* from_trace(const Trace& tr) {
    auto* s = new SnapList;
    for (const auto& it : tr) {
        s->snaps.push_back(it.tree);
        s->iteration.push_back(it.iteration);
        s->query_count.push_back(it.query_count);
    }
    return s;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

// --- runtime knobs for timing runs (attention.hpp:52-57) -----------------
void ref_set_threads(int n) {
    std::string v = std::to_string(n);
    setenv("TREEATTN_THREADS", v.c_str(), 1);
}

// Equivalent of MALLOC_MMAP_THRESHOLD_/MALLOC_TRIM_THRESHOLD_ for the
// per-group gather buffers (kv_cache.hpp:119-137); see BASELINE.md §4.
void ref_tune_malloc() {
    mallopt(M_MMAP_THRESHOLD, 32 * 1024 * 1024);
    mallopt(M_TRIM_THRESHOLD, 1 << 30);
    mallopt(M_ARENA_MAX, 64);
}

// --- snapshot lists ------------------------------------------------------
void* ref_trace_few_shot(int64_t prefix, int branches, int iterations) {
    SnapList* out = nullptr;
    guarded([&] { out = from_trace(gen_few_shot(prefix, branches, iterations)); return 0; });
    return out;
}

void* ref_trace_preset(const char* name) {
    SnapList* out = nullptr;
    guarded([&] { out = from_trace(preset_trace(name)); return 0; });
    return out;
}

// Any WorkloadSpec JSON accepted by spec_from_json (workloads.hpp:331-370).
void* ref_trace_spec_json(const char* json) {
    SnapList* out = nullptr;
    guarded([&] {
        out = from_trace(generate(spec_from_json(nlohmann::json::parse(json))));
        return 0;
    });
    return out;
}

// n trees from one rng stream, as the reference tests draw them
// (e.g. attention_test.cpp:157-176, partition_test.cpp:232-256).
void* ref_random_trees(uint64_t seed, int n, int max_leaves, int64_t max_tokens,
                       int64_t max_node_tokens, int max_branch_width, int mutation_steps) {
    auto* s = new SnapList;
    std::mt19937_64 rng(seed);
    RandomTreeConfig cfg;
    cfg.max_leaves = max_leaves;
    cfg.max_tokens = max_tokens;
    cfg.max_node_tokens = max_node_tokens;
    cfg.max_branch_width = max_branch_width;
    cfg.mutation_steps = mutation_steps;
    for (int i = 0; i < n; ++i) {
        DecodingTree t = random_tree(rng, cfg);
        s->snaps.push_back(TreeSnapshot::of(t));
        s->iteration.push_back(i);
        s->query_count.push_back(static_cast<int>(t.leaves().size()));
    }
    return s;
}

int ref_snaps_len(void* h) { return static_cast<int>(static_cast<SnapList*>(h)->snaps.size()); }

int ref_snaps_iteration(void* h, int i) { return static_cast<SnapList*>(h)->iteration.at(i); }

// Copies snapshot i; returns node count (call with nullptr buffers to size).
int ref_snaps_get(void* h, int i, int32_t* root, int32_t* ids, int32_t* parents, int64_t* counts) {
    const TreeSnapshot& s = static_cast<SnapList*>(h)->snaps.at(i);
    if (root) *root = s.root;
    if (ids)
        for (std::size_t k = 0; k < s.nodes.size(); ++k) {
            ids[k] = s.nodes[k].id;
            parents[k] = s.nodes[k].parent;
            counts[k] = s.nodes[k].token_count;
        }
    return static_cast<int>(s.nodes.size());
}

void ref_snaps_free(void* h) { delete static_cast<SnapList*>(h); }

// --- tree queries ----------------------------------------------------------
// leaves() of the restored tree (tree.hpp:55); returns count.
int ref_tree_leaves(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                    const int64_t* counts, int32_t* out) {
    return guarded([&] {
        DecodingTree t = DecodingTree::restore(root, nodes_from(n, ids, parents, counts));
        const auto& l = t.leaves();
        if (out) std::copy(l.begin(), l.end(), out);
        return static_cast<int>(l.size());
    });
}

// plan_to_json(make_plan(tree, strategy, bs)).dump(); malloc'd string.
char* ref_plan_json(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                    const int64_t* counts, const char* strategy, int block_size) {
    char* out = nullptr;
    guarded([&] {
        DecodingTree t = DecodingTree::restore(root, nodes_from(n, ids, parents, counts));
        const std::string s =
            plan_to_json(make_plan(t, strategy_from_name(strategy), block_size)).dump();
        out = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(out, s.c_str(), s.size() + 1);
        return 0;
    });
    return out;
}

// io_measured(make_plan(...)) (io_model.hpp:158-170): kv, q, mask, partial.
int ref_io_measured(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                    const int64_t* counts, const char* strategy, int block_size, int d_head,
                    int n_heads, int n_layers, int dtype_bytes, uint64_t* out4) {
    return guarded([&] {
        DecodingTree t = DecodingTree::restore(root, nodes_from(n, ids, parents, counts));
        CostParams cp{d_head, n_heads, n_layers, dtype_bytes};
        IoReport r = io_measured(make_plan(t, strategy_from_name(strategy), block_size), cp);
        out4[0] = r.kv_bytes;
        out4[1] = r.q_bytes;
        out4[2] = r.mask_bytes;
        out4[3] = r.partial_bytes;
        return 0;
    });
}

// io_analytical (io_model.hpp:91-153) kv/q/mask/partial for a named algorithm.
int ref_io_analytical(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                      const int64_t* counts, const char* algorithm, int block_size, int d_head,
                      int n_heads, int n_layers, int dtype_bytes, uint64_t* out4) {
    return guarded([&] {
        DecodingTree t = DecodingTree::restore(root, nodes_from(n, ids, parents, counts));
        CostParams cp{d_head, n_heads, n_layers, dtype_bytes};
        IoReport r = io_analytical(t, algorithm_from_name(algorithm), cp, block_size);
        out4[0] = r.kv_bytes;
        out4[1] = r.q_bytes;
        out4[2] = r.mask_bytes;
        out4[3] = r.partial_bytes;
        return 0;
    });
}

// --- instances -------------------------------------------------------------
// instance_from_snapshot (synth.hpp:130-144): MHA content at n_heads*d_head.
void* ref_instance_new(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                       const int64_t* counts, int d_head, int n_heads, uint64_t seed) {
    Instance* inst = nullptr;
    guarded([&] {
        auto in = std::make_unique<Instance>();
        in->params.d_head = d_head;
        in->params.n_heads = n_heads;
        in->pool = std::make_unique<PagePool>(in->params.dim());
        in->tree = std::make_unique<DecodingTree>(
            DecodingTree::restore(root, nodes_from(n, ids, parents, counts), in->pool.get()));
        fill_tree_kv(*in->pool, *in->tree, seed);
        in->queries = make_queries(*in->tree, in->params, seed);
        inst = in.release();
        return 0;
    });
    return inst;
}

// GQA expansion: content generated by fill_tree_kv at
// h_kv*d_head, q heads h read kv head h / (h_q/h_kv), queries by make_queries
// at h_q*d_head.  The reference then runs MHA over the expanded pool.
void* ref_instance_new_gqa(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                           const int64_t* counts, int d_head, int h_q, int h_kv, uint64_t seed) {
    Instance* inst = nullptr;
    guarded([&] {
        if (h_kv < 1 || h_q % h_kv != 0) throw std::invalid_argument("gqa: h_q % h_kv != 0");
        const int grp = h_q / h_kv;
        auto nodes = nodes_from(n, ids, parents, counts);
        PagePool kvpool(d_head * h_kv);
        DecodingTree kvtree = DecodingTree::restore(root, nodes, &kvpool);
        fill_tree_kv(kvpool, kvtree, seed);

        auto in = std::make_unique<Instance>();
        in->params.d_head = d_head;
        in->params.n_heads = h_q;
        in->pool = std::make_unique<PagePool>(in->params.dim());
        in->tree = std::make_unique<DecodingTree>(DecodingTree::restore(root, nodes, in->pool.get()));
        std::vector<float> k(static_cast<std::size_t>(in->params.dim()));
        std::vector<float> v(k.size());
        for (NodeId id : in->tree->node_ids()) {
            const KvHandle& src = kvpool.handle(id);
            const KvHandle& dst = in->pool->handle(id);
            GatheredKv g = kvpool.gather(src.refs);
            for (int t = 0; t < g.rows; ++t) {
                for (int h = 0; h < h_q; ++h)
                    for (int d = 0; d < d_head; ++d) {
                        const std::size_t s = static_cast<std::size_t>(t) * g.dim + (h / grp) * d_head + d;
                        k[static_cast<std::size_t>(h) * d_head + d] = g.keys[s];
                        v[static_cast<std::size_t>(h) * d_head + d] = g.values[s];
                    }
                in->pool->write_kv(dst, t, k, v);
            }
        }
        in->queries = make_queries(*in->tree, in->params, seed);
        inst = in.release();
        return 0;
    });
    return inst;
}

// Arbitrary content (e.g. bf16-rounded K/V/Q).
// keys/values: nodes in ascending id order, each [token_count][dim];
// q: [n_leaves][dim] in leaves() order.
void* ref_instance_new_content(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                               const int64_t* counts, int d_head, int n_heads, const float* keys,
                               const float* values, const float* q) {
    Instance* inst = nullptr;
    guarded([&] {
        auto in = std::make_unique<Instance>();
        in->params.d_head = d_head;
        in->params.n_heads = n_heads;
        const int dim = in->params.dim();
        in->pool = std::make_unique<PagePool>(dim);
        in->tree = std::make_unique<DecodingTree>(
            DecodingTree::restore(root, nodes_from(n, ids, parents, counts), in->pool.get()));
        std::size_t off = 0;
        for (NodeId id : in->tree->node_ids()) {
            const KvHandle& h = in->pool->handle(id);
            for (std::size_t t = 0; t < h.refs.size(); ++t, off += dim)
                in->pool->write_kv(h, static_cast<int>(t),
                                   std::span<const float>(keys + off, dim),
                                   std::span<const float>(values + off, dim));
        }
        std::size_t qi = 0;
        for (NodeId leaf : in->tree->leaves()) {
            QueryVec qv;
            qv.leaf = leaf;
            qv.q.assign(q + qi * dim, q + (qi + 1) * dim);
            in->queries.emplace(leaf, std::move(qv));
            ++qi;
        }
        inst = in.release();
        return 0;
    });
    return inst;
}

void ref_instance_free(void* h) { delete static_cast<Instance*>(h); }

int ref_instance_dim(void* h) { return static_cast<Instance*>(h)->params.dim(); }

int ref_instance_leaves(void* h, int32_t* out) {
    const auto& l = static_cast<Instance*>(h)->tree->leaves();
    if (out) std::copy(l.begin(), l.end(), out);
    return static_cast<int>(l.size());
}

// Node rows in token order via PagePool::gather (kv_cache.hpp:119-137).
int ref_instance_node_kv(void* h, int32_t node, float* keys, float* values) {
    return guarded([&] {
        auto* in = static_cast<Instance*>(h);
        const KvHandle& kh = in->pool->handle(node);
        GatheredKv g = in->pool->gather(kh.refs);
        if (keys) std::copy(g.keys.begin(), g.keys.end(), keys);
        if (values) std::copy(g.values.begin(), g.values.end(), values);
        return g.rows;
    });
}

int ref_instance_queries(void* h, float* q) {
    auto* in = static_cast<Instance*>(h);
    const int dim = in->params.dim();
    int i = 0;
    for (NodeId leaf : in->tree->leaves()) {
        const auto& v = in->queries.at(leaf).q;
        std::copy(v.begin(), v.end(), q + static_cast<std::size_t>(i) * dim);
        ++i;
    }
    return i;
}

// run_iteration (attention.hpp:293-334).  out: [n_leaves][dim] leaves() order,
// present[i] = leaf i appears in the AttentionOutput map.  seconds: wall time.
int ref_run_iteration(void* h, const char* strategy, int block_size, int use_double,
                      int tile_size, double* out, uint8_t* present, double* seconds) {
    return guarded([&] {
        auto* in = static_cast<Instance*>(h);
        AttentionParams p = in->params;
        p.use_double = use_double != 0;
        p.tile_size = tile_size;
        const auto t0 = std::chrono::steady_clock::now();
        auto [got, plan] =
            run_iteration(*in->tree, strategy_from_name(strategy), block_size, *in->pool,
                          in->queries, p);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        const int dim = p.dim();
        int i = 0;
        for (NodeId leaf : in->tree->leaves()) {
            auto it = got.find(leaf);
            if (present) present[i] = it != got.end();
            if (out && it != got.end())
                std::copy(it->second.begin(), it->second.end(), out + static_cast<std::size_t>(i) * dim);
            ++i;
        }
        return 0;
    });
}

// naive_attention (attention.hpp:237-288); out as above.
int ref_naive(void* h, double* out, double* seconds) {
    return guarded([&] {
        auto* in = static_cast<Instance*>(h);
        const auto t0 = std::chrono::steady_clock::now();
        AttentionOutput got = naive_attention(*in->tree, in->queries, *in->pool, in->params);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        const int dim = in->params.dim();
        int i = 0;
        for (NodeId leaf : in->tree->leaves()) {
            auto it = got.find(leaf);
            if (it != got.end())
                std::copy(it->second.begin(), it->second.end(), out + static_cast<std::size_t>(i) * dim);
            ++i;
        }
        return 0;
    });
}

// --- synth primitives, for pinning the C restatement -----------------------
void ref_fill_uniform(float* v, int64_t n, uint64_t seed) {
    std::vector<float> x(static_cast<std::size_t>(n));
    detail::fill_uniform(x, seed);
    std::copy(x.begin(), x.end(), v);
}

uint64_t ref_content_seed(uint64_t seed, uint64_t a, uint64_t b) {
    return detail::content_seed(seed, a, b);
}

}  // extern "C"
