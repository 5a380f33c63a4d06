// Runs INTEGRATION.md's drop-in (include/treeattn_b200.hpp) against the
// reference's own run_iteration on the same trees and content: the reference
// headers from /root/reference (compiled here by oracle/Makefile, target
// shim_test), the B200 path through the C ABI on cuda:0.
//
// Cases: fig2 (partition_test.cpp:181-194), the demo tree (SURVEY §8d config
// A at 1 layer, 4 heads x d128), 20 random trees (synth.hpp:80-111, seed
// 2024, d 16/64/128), and the reference's error behaviour (an unknown node
// throws std::out_of_range through the shim).  Gates: relative_error
// (attention.hpp:337-346) <= 1e-5 per leaf against the reference's fp64
// engine, the same leaf set, and plan_to_json identical to ta_plan_json.
// Exit 0 on success.
#include <cstdio>
#include <random>

#include "treeattn_b200.hpp"

using namespace treeattn;

static int failures = 0;

static double compare(const AttentionOutput& got, const AttentionOutput& ref, const char* what) {
    double worst = 0;
    if (got.size() != ref.size()) {
        std::printf("FAIL %s: %zu leaves vs %zu\n", what, got.size(), ref.size());
        ++failures;
        return 1e30;
    }
    for (const auto& [leaf, r] : ref) {
        auto it = got.find(leaf);
        if (it == got.end()) {
            std::printf("FAIL %s: leaf %lld missing\n", what, (long long)leaf);
            ++failures;
            return 1e30;
        }
        worst = std::max(worst, relative_error(it->second, r));
    }
    if (worst > 1e-5) {
        std::printf("FAIL %s: relative_error %.3e\n", what, worst);
        ++failures;
    }
    return worst;
}

static void run_case(const DecodingTree& tree, const PagePool& pool, const std::map<NodeId, QueryVec>& queries,
                     const AttentionParams& params, int block_size, const char* what) {
    AttentionParams dp = params;
    dp.use_double = true;
    const auto ref = treeattn::run_iteration(tree, Strategy::Flatten, block_size, pool, queries, dp);
    int64_t pages = 16;
    for (NodeId id : tree.node_ids()) pages += (tree.node(id).token_count + 15) / 16;
    b200::Context c(params, pages);
    const auto got = b200::run_iteration(c, tree, block_size, pool, queries, params);
    const double err = compare(got.first, ref.first, what);
    // the plan the shim returns and the device's plan are the reference's plan
    size_t len = 0;
    b200::check(ta_plan_json(c.ctx, block_size, nullptr, 0, &len));
    std::string js(len + 1, '\0');
    b200::check(ta_plan_json(c.ctx, block_size, js.data(), js.size(), &len));
    js.resize(len);
    if (plan_to_json(ref.second).dump() != js || plan_to_json(got.second).dump() != js) {
        std::printf("FAIL %s: plan_to_json differs from ta_plan_json\n", what);
        ++failures;
    }
    std::printf("%-28s leaves %3zu  relative_error %.2e\n", what, ref.first.size(), err);
}

int main() {
    {   // fig2: two-cascaded tree (partition_test.cpp:181-194), bs 6
        AttentionParams p{16, 2};
        PagePool pool(p.dim());
        DecodingTree t(4, &pool);
        t.branch(t.root(), {2, 2});
        fill_tree_kv(pool, t, 7);
        run_case(t, pool, make_queries(t, p, 7), p, 6, "fig2");
    }
    {   // demo tree: 1k prefix + 4 x 128 (config A shape, 4 heads)
        AttentionParams p{128, 4};
        PagePool pool(p.dim());
        DecodingTree t(1024, &pool);
        t.branch(t.root(), {128, 128, 128, 128});
        fill_tree_kv(pool, t, 42);
        run_case(t, pool, make_queries(t, p, 42), p, 128, "demo 1k+4x128");
    }
    std::mt19937_64 rng(2024);
    const int dims[3] = {16, 64, 128};
    for (int i = 0; i < 20; ++i) {
        AttentionParams p{dims[i % 3], 1 + i % 3};
        RandomTreeConfig cfg;
        cfg.max_leaves = 24;
        cfg.max_tokens = 1500;
        auto inst = make_instance(rng, p, 1000 + i, cfg);
        char what[64];
        std::snprintf(what, sizeof what, "random %2d (d%d h%d)", i, p.d_head, p.n_heads);
        run_case(inst.tree, *inst.pool, inst.queries, p, 32 + 16 * (i % 7), what);
    }
    {   // error mapping: an unknown node is std::out_of_range, as in the reference
        AttentionParams p{16, 1};
        b200::Context c(p, 64);
        int32_t root = -1;
        b200::check(ta_tree_new(c.ctx, 10, &root));
        bool thrown = false;
        try {
            int64_t n = 3;
            int32_t kid = -1;
            b200::check(ta_tree_branch(c.ctx, 12345, 1, &n, &kid));
        } catch (const std::out_of_range&) {
            thrown = true;
        }
        if (!thrown) {
            std::printf("FAIL error mapping: no std::out_of_range\n");
            ++failures;
        }
    }
    std::printf(failures ? "FAILED (%d)\n" : "OK\n", failures);
    return failures ? 1 : 0;
}
