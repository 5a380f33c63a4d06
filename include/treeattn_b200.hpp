// treeattn_b200.hpp -- drop-in replacement of the reference's run_iteration
// (attention.hpp:293-334) on the B200 path, header-only, built only on the C
// ABI (treeattn_b200.h).  Include it next to the reference's headers
// (<treeattn/treeattn.hpp> must be on the include path) and call
// treeattn::b200::run_iteration instead of treeattn::run_iteration.  Exceptions
// map back from ta_status exactly as the reference throws them.
//
// Compiled and run by tests/cpp/shim_run_iteration.cpp against the reference
// itself (oracle/Makefile, target shim_test; pytest -m gpu
// tests/test_cpp_shim.py).
#pragma once

#include <treeattn/treeattn.hpp>

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "treeattn_b200.h"

namespace treeattn::b200 {

inline void check(ta_status s) {
    if (s == TA_OK) return;
    const std::string m = ta_last_error();
    if (s == TA_ERR_INVALID_ARGUMENT) throw std::invalid_argument(m);
    if (s == TA_ERR_OUT_OF_RANGE) throw std::out_of_range(m);
    throw std::logic_error(m);   // logic / CUDA / device errors
}

// One device context per (model, GPU); the tree and its pages are mirrored in.
struct Context {
    ta_ctx* ctx = nullptr;
    explicit Context(const AttentionParams& p, int64_t max_pages, int device = 0) {
        ta_shape s{};
        s.n_layers = 1;
        s.n_q_heads = p.n_heads;
        s.n_kv_heads = p.n_heads;
        s.d_head = p.d_head;
        s.kv_dtype = TA_F32;   // the reference's pool is fp32
        s.out_dtype = TA_F32;
        s.page_tokens = 16;
        s.max_pages = max_pages;
        check(ta_ctx_create(device, &s, &ctx));
    }
    ~Context() { ta_ctx_destroy(ctx); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
};

// run_iteration(tree, Flatten, bs, pool, queries, params), attention.hpp:293-334
inline std::pair<AttentionOutput, PartitionPlan> run_iteration(Context& c, const DecodingTree& tree, int block_size,
                                                               const PagePool& pool,
                                                               const std::map<NodeId, QueryVec>& queries,
                                                               const AttentionParams& params) {
    // 1. tree description = the reference's snapshot {id, parent, token_count} (tree.hpp:207-238)
    std::vector<int32_t> ids, parents;
    std::vector<int64_t> counts;
    for (NodeId id : tree.node_ids()) {   // ascending ids (std::map order)
        ids.push_back((int32_t)id);
        parents.push_back((int32_t)tree.node(id).parent);
        counts.push_back((int64_t)tree.node(id).token_count);
    }
    check(ta_tree_restore(c.ctx, (int32_t)tree.root(), (int)ids.size(), ids.data(), parents.data(), counts.data()));
    // 2. KV rows: PagePool::gather of each node (kv_cache.hpp:119-137) -> ta_kv_write
    for (NodeId id : tree.node_ids()) {
        const int64_t n = tree.node(id).token_count;
        if (n == 0) continue;
        GatheredKv kv = pool.gather(pool.handle(id).refs);
        check(ta_kv_write(c.ctx, 0, (int32_t)id, 0, n, kv.keys.data(), kv.values.data(), /*src_on_device=*/0, nullptr));
    }
    // 3. queries in leaves() order, [L][h][d]
    const auto leaves = tree.leaves();
    const size_t hd = (size_t)params.n_heads * params.d_head;
    std::vector<float> q(leaves.size() * hd, 0.f), out(leaves.size() * hd);
    for (size_t i = 0; i < leaves.size(); ++i)
        if (auto it = queries.find(leaves[i]); it != queries.end())
            std::copy(it->second.q.begin(), it->second.q.end(), q.begin() + i * hd);
    // 4. plan + schedule + attention (one layer), host buffers in and out
    check(ta_prepare(c.ctx, block_size, nullptr));
    check(ta_attend_host(c.ctx, 0, q.data(), out.data(), nullptr));
    // 5. AttentionOutput: map<leaf, vector<double>[h*d]> for leaves with a query and a path
    AttentionOutput result;
    for (size_t i = 0; i < leaves.size(); ++i)
        if (queries.count(leaves[i]) && tree.path_tokens(leaves[i]) > 0)
            result[leaves[i]] = std::vector<double>(out.begin() + i * hd, out.begin() + (i + 1) * hd);
    // 6. the plan: make_plan(tree, Flatten, bs) is byte-identical to ta_plan_json
    return {std::move(result), make_plan(tree, Strategy::Flatten, block_size)};
}

}  // namespace treeattn::b200
