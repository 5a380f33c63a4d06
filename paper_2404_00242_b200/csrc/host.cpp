// host.cpp -- tree mirror, page accounting, bit-exact flatten planner and the
// device schedule builder.  Reference citations are relative to
// /root/reference/proj/include/treeattn.
#include <algorithm>
#include <cstring>
#include <atomic>
#include <cstdio>
#include <numeric>
#include <unordered_map>
#include <cstddef>

#include "ta_internal.h"
#include "treeattn_b200.h"

namespace ta {

void fail(int code, const std::string& msg) { throw Error(code, msg); }

// Tree versions are globally unique so a cached plan can never be mistaken
// for the plan of a different (restored / recreated) tree.
static std::atomic<uint64_t> g_tree_version{1};
static uint64_t next_version() { return g_tree_version.fetch_add(1); }

// ===========================================================================
// Tree (tree.hpp:38-269)
// ===========================================================================
void Tree::reserve(int32_t n) {
    if ((int32_t)alive.size() >= n) return;
    int32_t cap = std::max<int32_t>(16, (int32_t)alive.size());
    while (cap < n) cap *= 2;
    alive.resize(cap, 0);
    parent.resize(cap, -1);
    count.resize(cap, 0);
    kids.resize(cap);
    leaf_lo.resize(cap, 0);
    leaf_hi.resize(cap, 0);
}

void Tree::subtree(int32_t at, std::vector<int32_t>& out) const {
    out.clear();
    std::vector<int32_t> stack{at};
    while (!stack.empty()) {
        int32_t v = stack.back();
        stack.pop_back();
        out.push_back(v);
        for (auto it = kids[v].rbegin(); it != kids[v].rend(); ++it) stack.push_back(*it);
    }
}

// leaves() / depth_first_order() (tree.hpp:161-166, 257-262) plus, per node,
// the [lo, hi) range of leaf indices in its subtree: because leaves are in
// DFS order, queries_for_node (tree.hpp:169-178) is exactly that range.
void Tree::rebuild() {
    subtree(root, dfs);
    leaves.clear();
    for (int32_t id : dfs)
        if (kids[id].empty()) {
            leaf_lo[id] = (int32_t)leaves.size();
            leaf_hi[id] = leaf_lo[id] + 1;
            leaves.push_back(id);
        }
    for (auto it = dfs.rbegin(); it != dfs.rend(); ++it) {
        const int32_t id = *it;
        if (!kids[id].empty()) {
            leaf_lo[id] = leaf_lo[kids[id].front()];
            leaf_hi[id] = leaf_hi[kids[id].back()];
        }
    }
    version = next_version();
}

void Tree::create(int64_t root_tokens) {
    if (root_tokens < 1) fail(TA_ERR_INVALID_ARGUMENT, "new_tree: root_token_count must be >= 1");
    KvHook* h = hook;
    *this = Tree{};
    hook = h;
    reserve(16);
    root = next_id++;
    alive[root] = 1;
    count[root] = root_tokens;
    n_alive = 1;
    if (hook) hook->on_alloc(root, root_tokens);
    rebuild();
}

void Tree::restore(int32_t r, int n, const int32_t* ids, const int32_t* parents, const int64_t* counts) {
    KvHook* h = hook;
    *this = Tree{};
    int32_t maxid = r;
    for (int i = 0; i < n; ++i) {
        if (ids[i] < 0) fail(TA_ERR_INVALID_ARGUMENT, "restore: negative node id");
        maxid = std::max(maxid, ids[i]);
    }
    reserve(maxid + 1);
    root = r;
    for (int i = 0; i < n; ++i) {
        if (alive[ids[i]]) fail(TA_ERR_INVALID_ARGUMENT, "restore: duplicate node id");
        alive[ids[i]] = 1;
        parent[ids[i]] = parents[i];
        count[ids[i]] = counts[i];
        next_id = std::max(next_id, ids[i] + 1);
    }
    n_alive = n;
    // children in ascending id order (std::map iteration, tree.hpp:223-233)
    for (int32_t id = 0; id < (int32_t)alive.size(); ++id) {
        if (!alive[id]) continue;
        if (id == root) {
            if (parent[id] != -1) fail(TA_ERR_INVALID_ARGUMENT, "restore: root must have no parent");
            continue;
        }
        if (!contains(parent[id])) fail(TA_ERR_INVALID_ARGUMENT, "restore: dangling parent link");
        kids[parent[id]].push_back(id);
    }
    if (!contains(root)) fail(TA_ERR_INVALID_ARGUMENT, "restore: unreachable or cyclic nodes");
    // reachability (a cycle among non-root nodes is unreachable from root)
    std::vector<int32_t> reach;
    {
        std::vector<uint8_t> seen(alive.size(), 0);
        std::vector<int32_t> stack{root};
        while (!stack.empty()) {
            int32_t v = stack.back();
            stack.pop_back();
            if (seen[v]) continue;
            seen[v] = 1;
            reach.push_back(v);
            for (int32_t c : kids[v]) stack.push_back(c);
        }
    }
    if ((int)reach.size() != n) fail(TA_ERR_INVALID_ARGUMENT, "restore: unreachable or cyclic nodes");
    rebuild();
    hook = h;
    if (hook)
        for (int32_t id : dfs) hook->on_alloc(id, count[id]);
}

std::vector<int32_t> Tree::branch(int32_t at, const int64_t* counts, int n) {
    if (!contains(at)) fail(TA_ERR_OUT_OF_RANGE, "branch: unknown node id " + std::to_string(at));
    if (!kids[at].empty()) fail(TA_ERR_INVALID_ARGUMENT, "branch: only leaves may branch");
    for (int i = 0; i < n; ++i)
        if (counts[i] < 0) fail(TA_ERR_INVALID_ARGUMENT, "branch: negative child token count");
    reserve(next_id + n + 1);
    std::vector<int32_t> created;
    const int32_t first_id = next_id;
    try {
        for (int i = 0; i < n; ++i) {
            const int32_t id = next_id;
            if (hook) hook->on_alloc(id, counts[i]);   // atomic: allocates all of the child's pages or none
            ++next_id;
            alive[id] = 1;
            parent[id] = at;
            count[id] = counts[i];
            kids[id].clear();
            kids[at].push_back(id);
            created.push_back(id);
            ++n_alive;
        }
    } catch (...) {
        // a bounded device pool ran out part way: undo the children created so
        // far, so the tree and the pool stay consistent (the reference's pool is
        // unbounded and never gets here)
        for (int32_t id : created) {
            if (hook) hook->on_free(id);
            alive[id] = 0;
            --n_alive;
        }
        kids[at].clear();
        next_id = first_id;
        throw;
    }
    rebuild();
    return created;
}

void Tree::prune(int32_t at) {
    if (at == root) fail(TA_ERR_INVALID_ARGUMENT, "prune: cannot prune the root");
    if (!contains(at)) fail(TA_ERR_OUT_OF_RANGE, "prune: unknown node id " + std::to_string(at));
    std::vector<int32_t> doomed;
    subtree(at, doomed);
    auto& pk = kids[parent[at]];
    pk.erase(std::find(pk.begin(), pk.end(), at));
    for (int32_t id : doomed) {
        if (hook) hook->on_free(id);
        alive[id] = 0;
        kids[id].clear();
        --n_alive;
    }
    rebuild();
}

void Tree::append(int32_t leaf, int64_t n) {
    if (!contains(leaf)) fail(TA_ERR_OUT_OF_RANGE, "append_tokens: unknown node id " + std::to_string(leaf));
    if (!kids[leaf].empty()) fail(TA_ERR_INVALID_ARGUMENT, "append_tokens: target is not a leaf");
    if (n < 1) fail(TA_ERR_INVALID_ARGUMENT, "append_tokens: n must be >= 1");
    count[leaf] += n;
    if (hook) hook->on_extend(leaf, n);
    version = next_version();
}

int64_t Tree::total_tokens() const {
    int64_t s = 0;
    for (int32_t id : dfs) s += count[id];
    return s;
}

int64_t Tree::path_tokens(int32_t leaf) const {
    int64_t s = 0;
    for (int32_t cur = leaf; cur != -1; cur = parent[cur]) s += count[cur];
    return s;
}

// ===========================================================================
// PagePool accounting (kv_cache.hpp:33-187)
// ===========================================================================
int32_t PagePool::acquire_page(int32_t owner) {
    int32_t pid;
    if (!free_list.empty()) {
        pid = free_list.back();
        free_list.pop_back();
    } else {
        if (capacity >= 0 && (int64_t)pages.size() >= capacity)
            fail(TA_ERR_OUT_OF_MEMORY, "PagePool: device page capacity exhausted (" +
                                           std::to_string(capacity) + " pages)");
        pid = (int32_t)pages.size();
        pages.emplace_back();
    }
    pages[pid].owner = owner;
    pages[pid].used = 0;
    pages[pid].live = 0;
    return pid;
}

void PagePool::allocate(int32_t node, int64_t n) {
    if (n < 0) fail(TA_ERR_INVALID_ARGUMENT, "allocate: negative token count");
    if (handles.count(node)) fail(TA_ERR_LOGIC, "allocate: node already has a handle");
    handles.emplace(node, Handle{});
    try {
        extend(node, n);
    } catch (...) {
        handles.erase(node);
        throw;
    }
}

void PagePool::extend(int32_t node, int64_t n) {
    auto it = handles.find(node);
    if (it == handles.end()) fail(TA_ERR_LOGIC, "extend: no handle for node");
    Handle& h = it->second;
    if (capacity >= 0) {   // all or nothing: check the page demand before taking any
        const int64_t room = h.pages.empty() ? 0 : page_size - pages[h.pages.back()].used;
        const int64_t need = n > room ? (n - room + page_size - 1) / page_size : 0;
        const int64_t avail = (int64_t)free_list.size() + capacity - (int64_t)pages.size();
        if (need > avail)
            fail(TA_ERR_OUT_OF_MEMORY, "PagePool: device page capacity exhausted (" + std::to_string(capacity) +
                                           " pages, " + std::to_string(need) + " more needed, " + std::to_string(avail) +
                                           " free)");
    }
    // Fill this node's tail page first; never share a page across nodes.
    while (n > 0) {
        if (!h.pages.empty()) {
            Page& p = pages[h.pages.back()];
            if (p.used < page_size) {
                const int64_t take = std::min<int64_t>(n, page_size - p.used);
                p.used += (int32_t)take;
                p.live += (int32_t)take;
                live_slots += take;
                h.n_tokens += take;
                n -= take;
                continue;
            }
        }
        const int32_t pid = acquire_page(node);
        h.pages.push_back(pid);
        const int64_t take = std::min<int64_t>(n, page_size);
        pages[pid].used = (int32_t)take;
        pages[pid].live = (int32_t)take;
        live_slots += take;
        h.n_tokens += take;
        n -= take;
    }
}

void PagePool::release(int32_t node) {
    auto it = handles.find(node);
    if (it == handles.end()) fail(TA_ERR_LOGIC, "free: handle not live (double free?)");
    // refs are released in token order; each page is released when its last
    // live slot goes (kv_cache.hpp:95-100)
    for (int32_t pid : it->second.pages) {
        Page& p = pages[pid];
        live_slots -= p.live;
        p.live = 0;
        p.owner = -1;
        p.used = 0;
        free_list.push_back(pid);
    }
    handles.erase(it);
}

const PagePool::Handle& PagePool::handle(int32_t node) const {
    auto it = handles.find(node);
    if (it == handles.end()) fail(TA_ERR_LOGIC, "PagePool: no handle for node " + std::to_string(node));
    return it->second;
}

void PagePool::reset() {
    pages.clear();
    free_list.clear();
    handles.clear();
    live_slots = 0;
}

// ===========================================================================
// The reference's partition strategies (partition.hpp:97-262) via leaf
// intervals.  Leaves are in DFS order, so a node's queries
// (queries_for_node, tree.hpp:169-178) are the contiguous leaf interval
// [lo, hi) of its subtree, and every mask word is a contiguous run of bits.
//
// Emitter::flush(segments) is emit_groups (partition.hpp:102-126) for one
// chunk: the query list is the union of the segments' intervals in leaves()
// order; > 64 queries give 64-query slices that keep every segment (even
// with mask 0), else mask-0 segments are dropped; a group is emitted iff
// some mask is set.  It also records the chunk view the device schedule is
// built from.  Bit-exact with plan_to_json for every strategy.
// ===========================================================================
static inline uint64_t run_mask(int b, int e) {
    if (e <= b) return 0;
    const int n = e - b;
    return (n >= 64 ? ~0ULL : ((1ULL << n) - 1)) << b;
}

namespace {

struct Seg {
    int32_t node;
    int64_t off, len;
};

struct Emitter {
    const Tree& t;
    Plan& P;
    std::vector<std::pair<int32_t, int32_t>> iv;
    std::vector<int32_t> Q;

    void chunk_view(const std::vector<Seg>& segs) {
        for (std::size_t s = 0; s < segs.size(); ++s) {
            P.cseg_node.push_back(segs[s].node);
            P.cseg_offset.push_back(segs[s].off);
            P.cseg_len.push_back(segs[s].len);
            P.cseg_lo.push_back(iv[s].first);
            P.cseg_hi.push_back(iv[s].second);
        }
        P.chunk_seg_begin.push_back((int32_t)P.cseg_node.size());
        P.chunk_q.insert(P.chunk_q.end(), Q.begin(), Q.end());
        P.chunk_q_begin.push_back((int32_t)P.chunk_q.size());
    }

    void flush(const std::vector<Seg>& segs) {
        if (segs.empty()) return;
        iv.clear();
        for (const Seg& s : segs) iv.emplace_back(t.leaf_lo[s.node], t.leaf_hi[s.node]);
        std::vector<std::pair<int32_t, int32_t>> sorted = iv;
        std::stable_sort(sorted.begin(), sorted.end());
        Q.clear();
        int32_t end = -1;
        for (auto [lo, hi] : sorted) {
            const int32_t from = std::max(lo, end);
            for (int32_t q = from; q < hi; ++q) Q.push_back(q);
            end = std::max(end, hi);
        }
        chunk_view(segs);
        // reference groups
        const int nq = (int)Q.size();
        const bool split = nq > 64;
        for (int base = 0; base < nq; base += 64) {
            const int cnt = std::min(64, nq - base);
            const std::size_t seg_mark = P.seg_node.size();
            bool any = false;
            for (std::size_t s = 0; s < segs.size(); ++s) {
                const int b = (int)(std::lower_bound(Q.begin(), Q.end(), iv[s].first) - Q.begin());
                const int e = (int)(std::lower_bound(Q.begin(), Q.end(), iv[s].second) - Q.begin());
                const int bb = std::clamp(b, base, base + cnt) - base;
                const int ee = std::clamp(e, base, base + cnt) - base;
                const uint64_t mask = run_mask(bb, ee);
                if (mask == 0 && !split) continue;
                P.seg_node.push_back(segs[s].node);
                P.seg_offset.push_back(segs[s].off);
                P.seg_len.push_back(segs[s].len);
                P.seg_mask.push_back(mask);
                any = any || mask != 0;
            }
            if (!any) {
                P.seg_node.resize(seg_mark);
                P.seg_offset.resize(seg_mark);
                P.seg_len.resize(seg_mark);
                P.seg_mask.resize(seg_mark);
                continue;
            }
            for (int j = 0; j < cnt; ++j) P.queries.push_back(t.leaves[Q[base + j]]);
            P.seg_begin.push_back((int32_t)P.seg_node.size());
            P.q_begin.push_back((int32_t)P.queries.size());
        }
    }
};

}  // namespace

// partition_flatten (partition.hpp:212-253): stream tokens in DFS pre-order,
// skip 0-token nodes, flush every block_size tokens and at the end.
void plan_flatten(const Tree& t, int bs, Plan& P) {
    if (bs < 1) fail(TA_ERR_INVALID_ARGUMENT, "partition: block_size must be >= 1");
    P = Plan{};
    P.block_size = bs;
    P.strategy = TA_STRATEGY_FLATTEN;
    Emitter em{t, P, {}, {}};
    std::vector<Seg> pend;
    int64_t fill = 0;
    for (int32_t id : t.dfs) {
        int64_t remaining = t.count[id], offset = 0;
        while (remaining > 0) {
            const int64_t take = std::min<int64_t>(remaining, bs - fill);
            pend.push_back({id, offset, take});
            offset += take;
            remaining -= take;
            fill += take;
            if (fill == bs) {
                em.flush(pend);
                pend.clear();
                fill = 0;
            }
        }
    }
    em.flush(pend);
}

// partition_node (partition.hpp:176-187) / partition_node_chunk (:190-207):
// one chunk per live node, or per block_size piece of it, with the node's
// queries.
static void plan_node(const Tree& t, int bs, bool chunked, Plan& P) {
    if (chunked && bs < 1) fail(TA_ERR_INVALID_ARGUMENT, "partition: block_size must be >= 1");
    P = Plan{};
    P.block_size = chunked ? bs : 0;
    P.strategy = chunked ? TA_STRATEGY_NODE_CHUNK : TA_STRATEGY_NODE;
    Emitter em{t, P, {}, {}};
    std::vector<Seg> one(1);
    for (int32_t id : t.dfs) {
        const int64_t n = t.count[id];
        if (n == 0) continue;
        const int64_t step = chunked ? bs : n;
        for (int64_t off = 0; off < n; off += step) {
            one[0] = {id, off, std::min<int64_t>(step, n - off)};
            em.flush(one);
        }
    }
}

// partition_q_guided (partition.hpp:133-173): one group per leaf, its whole
// root-to-leaf KV cut into blocks, every mask word 1 (shared prefixes are
// loaded once per query: the redundancy the KV-guided strategies remove).
static void plan_q_guided(const Tree& t, int bs, Plan& P) {
    if (bs < 1) fail(TA_ERR_INVALID_ARGUMENT, "partition: block_size must be >= 1");
    P = Plan{};
    P.block_size = bs;
    P.strategy = TA_STRATEGY_Q_GUIDED;
    std::vector<int32_t> chain;
    std::vector<Seg> segs;
    for (int32_t li = 0; li < (int32_t)t.leaves.size(); ++li) {
        const int32_t leaf = t.leaves[li];
        chain.clear();
        for (int32_t cur = leaf; cur != -1; cur = t.parent[cur]) chain.push_back(cur);
        std::reverse(chain.begin(), chain.end());
        int64_t fill = 0;
        auto flush = [&] {
            if (segs.empty()) return;
            for (const Seg& s : segs) {
                P.seg_node.push_back(s.node);
                P.seg_offset.push_back(s.off);
                P.seg_len.push_back(s.len);
                P.seg_mask.push_back(1);
                P.cseg_node.push_back(s.node);
                P.cseg_offset.push_back(s.off);
                P.cseg_len.push_back(s.len);
                P.cseg_lo.push_back(li);
                P.cseg_hi.push_back(li + 1);
            }
            P.queries.push_back(leaf);
            P.seg_begin.push_back((int32_t)P.seg_node.size());
            P.q_begin.push_back((int32_t)P.queries.size());
            P.chunk_seg_begin.push_back((int32_t)P.cseg_node.size());
            P.chunk_q.push_back(li);
            P.chunk_q_begin.push_back((int32_t)P.chunk_q.size());
            segs.clear();
            fill = 0;
        };
        for (int32_t id : chain) {
            int64_t remaining = t.count[id], offset = 0;
            while (remaining > 0) {
                const int64_t take = std::min<int64_t>(remaining, bs - fill);
                segs.push_back({id, offset, take});
                offset += take;
                remaining -= take;
                fill += take;
                if (fill == bs) flush();
            }
        }
        flush();
    }
}

// make_plan (partition.hpp:255-262)
void make_plan(const Tree& t, int strategy, int bs, Plan& P) {
    switch (strategy) {
        case TA_STRATEGY_Q_GUIDED: plan_q_guided(t, bs, P); return;
        case TA_STRATEGY_NODE: plan_node(t, bs, false, P); return;
        case TA_STRATEGY_NODE_CHUNK: plan_node(t, bs, true, P); return;
        case TA_STRATEGY_FLATTEN: plan_flatten(t, bs, P); return;
        default: fail(TA_ERR_INVALID_ARGUMENT, "unknown strategy " + std::to_string(strategy));
    }
}

// plan_to_json(plan).dump() (serde.hpp:41-61): nlohmann objects are key-sorted
// and dumped without whitespace.
std::string plan_json(const Tree& t, const Plan& p) {
    std::string s = "{\"block_size\":" + std::to_string(p.block_size) + ",\"groups\":[";
    char buf[32];
    for (int g = 0; g < p.n_groups(); ++g) {
        if (g) s += ',';
        s += "{\"id\":" + std::to_string(g) + ",\"masks\":[";
        for (int k = p.seg_begin[g]; k < p.seg_begin[g + 1]; ++k) {
            std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)p.seg_mask[k]);
            if (k > p.seg_begin[g]) s += ',';
            s += '"';
            s += buf;
            s += '"';
        }
        s += "],\"queries\":[";
        for (int k = p.q_begin[g]; k < p.q_begin[g + 1]; ++k) {
            if (k > p.q_begin[g]) s += ',';
            s += std::to_string(p.queries[k]);
        }
        s += "],\"segments\":[";
        for (int k = p.seg_begin[g]; k < p.seg_begin[g + 1]; ++k) {
            if (k > p.seg_begin[g]) s += ',';
            s += "{\"len\":" + std::to_string(p.seg_len[k]) + ",\"node\":" + std::to_string(p.seg_node[k]) +
                 ",\"offset\":" + std::to_string(p.seg_offset[k]) + "}";
        }
        s += "]}";
    }
    static const char* names[] = {"q-guided", "node", "node-chunk", "flatten"};
    s += "],\"strategy\":\"";
    s += names[p.strategy];
    s += "\"}";
    (void)t;
    return s;
}

// ===========================================================================
// Device schedule (see ta_internal.h for the vocabulary).
//
// 1. Stripes.  Walk the flatten chunks in order.  A chunk whose query set fits
//    a row tile (|Q| <= S = max_rows / G slots) joins the open stripe while
//    the union of query sets still fits; a wider chunk joins an open wide
//    stripe with the identical query set.  Queries that persist across chunks
//    (shared prefixes, long branches) therefore accumulate on chip.
// 2. Lanes.  A stripe with |Q| slots is cut into ceil(|Q| / S) balanced slot
//    blocks; each block streams only the stripe tokens its slots attend, as
//    16-row groups (consecutive pool rows, one slot range) and 8-group tiles.
//    The blocks of a wide stripe read the same KV; they are adjacent in the
//    sequence so they run concurrently and the repeat reads hit L2.
// 3. CTA runs.  The sequence (head, lane, tile) is cut into num_ctas
//    contiguous runs of equal cost (box rows + a fixed per-tile cost); each
//    run's maximal (head, lane) pieces are its items.
// 4. Outputs.  A leaf-head attended by one item is written directly; else
//    its items write partials that are merged in item order (tree_reduce,
//    attention.hpp:209-233): at the end of the attention launch by the record's
//    owner CTA (fused merge) or by the merge launch after it.
// ===========================================================================
namespace {

struct Stripe {
    int c0 = 0, c1 = 0;             // chunk range [c0, c1) (chunks with no queries skipped inside)
    std::vector<int32_t> qset;      // sorted leaf indices
    bool wide = false;
};

struct Lane {
    int32_t slot_begin = 0, n_slots = 0;
    int32_t tile_begin = 0, tile_end = 0;
};

}  // namespace

void build_schedule(const Tree& t, const PagePool& pool, const Plan& plan, int G, int n_heads,
                    const SchedOptions& opt, Schedule& S) {
    S.clear();   // keeps the vectors' capacity: no reallocation (and page faults) per step
    S.n_leaves = (int32_t)t.leaves.size();
    const int P = pool.page_size;
    const int nc = plan.n_chunks();
    const int max_rows = opt.use_mma ? opt.max_rows : opt.fma_max_rows;
    const int S_max = std::max(1, max_rows / std::max(1, G));
    const int TG = std::clamp(opt.tile_groups, 1, 8);
    if (S_max > 128) fail(TA_ERR_INVALID_ARGUMENT, "schedule: more than 128 slots per lane");

    // ---- 1. stripes
    S.kv_tokens_unique = t.total_tokens();   // one pass over the tree's KV (ablation plans load more)
    std::vector<Stripe> stripes;
    std::vector<int32_t> tmp;
    for (int c = 0; c < nc; ++c) {
        const int qb = plan.chunk_q_begin[c], qe = plan.chunk_q_begin[c + 1];
        const int nq = qe - qb;
        if (nq == 0) continue;
        const int32_t* q = plan.chunk_q.data() + qb;
        Stripe* cur = stripes.empty() || !opt.fuse_chunks ? nullptr : &stripes.back();
        if (nq > S_max) {
            if (cur && cur->wide && (int)cur->qset.size() == nq && std::equal(q, q + nq, cur->qset.begin())) {
                cur->c1 = c + 1;
                continue;
            }
            stripes.push_back({c, c + 1, std::vector<int32_t>(q, q + nq), true});
            continue;
        }
        if (cur && !cur->wide) {
            tmp.clear();
            std::set_union(cur->qset.begin(), cur->qset.end(), q, q + nq, std::back_inserter(tmp));
            if ((int)tmp.size() <= S_max) {
                cur->qset.swap(tmp);
                cur->c1 = c + 1;
                continue;
            }
        }
        stripes.push_back({c, c + 1, std::vector<int32_t>(q, q + nq), false});
    }
    S.n_stripes = (int64_t)stripes.size();

    // ---- 2. lanes: groups and tiles
    std::vector<Lane> lanes;
    for (const Stripe& st : stripes) {
        const int nq = (int)st.qset.size();
        const int nb = (nq + S_max - 1) / S_max;
        for (int k = 0; k < nb; ++k) {
            Lane ln;
            const int a = (int)((int64_t)nq * k / nb), b = (int)((int64_t)nq * (k + 1) / nb);
            ln.slot_begin = (int32_t)S.slot_leaf.size();
            ln.n_slots = b - a;
            S.slot_leaf.insert(S.slot_leaf.end(), st.qset.begin() + a, st.qset.begin() + b);
            const int32_t* sl = S.slot_leaf.data() + ln.slot_begin;
            ln.tile_begin = (int32_t)S.tiles.size();
            int32_t g_open = -1;        // open group (may take more tokens)
            int32_t tile_g0 = (int32_t)S.grp_row.size();
            auto close_tile = [&](bool force) {
                const int32_t ng = (int32_t)S.grp_row.size() - tile_g0;
                if (ng == 0 || (!force && ng < TG)) return;
                TileDesc td{};
                td.grp_begin = tile_g0;
                td.ng = (uint8_t)ng;
                int ntok = 0;
                for (int g = 0; g < ng; ++g) ntok += (int)(S.grp_info[tile_g0 + g] & 0xffu);
                td.ntok = (uint16_t)ntok;
                // TMA boxes: runs of full, row-contiguous groups as 8/4/2/1-group boxes
                int nbx = 0, g = 0;
                while (g < ng) {
                    int run = 1;
                    while (g + run < ng && (S.grp_info[tile_g0 + g + run - 1] & 0xffu) == 16u &&
                           S.grp_row[tile_g0 + g + run] == S.grp_row[tile_g0 + g] + 16 * run)
                        ++run;
                    while (run > 0) {
                        int sz = 3;
                        while ((1 << sz) > run) --sz;
                        td.box[nbx++] = (uint8_t)((g << 2) | sz);
                        g += 1 << sz;
                        run -= 1 << sz;
                    }
                }
                td.nbox = (uint8_t)nbx;
                S.tiles.push_back(td);
                tile_g0 = (int32_t)S.grp_row.size();
                g_open = -1;
            };
            for (int c = st.c0; c < st.c1; ++c) {
                for (int s = plan.chunk_seg_begin[c]; s < plan.chunk_seg_begin[c + 1]; ++s) {
                    const int32_t lo = plan.cseg_lo[s], hi = plan.cseg_hi[s];
                    const int bb = (int)(std::lower_bound(sl, sl + ln.n_slots, lo) - sl);
                    const int ee = (int)(std::lower_bound(sl, sl + ln.n_slots, hi) - sl);
                    if (bb >= ee) continue;
                    const auto& h = pool.handle(plan.cseg_node[s]);
                    const int64_t off = plan.cseg_offset[s], len = plan.cseg_len[s];
                    // runs of consecutive pool rows (within a page) are added in bulk
                    for (int64_t k2 = 0; k2 < len;) {
                        const int64_t tok = off + k2;
                        int32_t row = (int32_t)(h.pages[tok / P] * P + tok % P);
                        int run = (int)std::min<int64_t>(len - k2, P - tok % P);
                        k2 += run;
                        while (run > 0) {
                            if (g_open >= 0) {
                                const uint32_t info = S.grp_info[g_open];
                                const int cnt = (int)(info & 0xffu);
                                if (cnt < 16 && S.grp_row[g_open] + cnt == row && (int)((info >> 8) & 0xfffu) == bb &&
                                    (int)(info >> 20) == ee) {
                                    const int take = std::min(run, 16 - cnt);
                                    S.grp_info[g_open] = grp_pack(cnt + take, bb, ee);
                                    row += take;
                                    run -= take;
                                    continue;
                                }
                            }
                            if ((int32_t)S.grp_row.size() - tile_g0 == TG) close_tile(false);
                            g_open = (int32_t)S.grp_row.size();
                            const int take = std::min(run, 16);
                            S.grp_row.push_back(row);
                            S.grp_info.push_back(grp_pack(take, bb, ee));
                            row += take;
                            run -= take;
                        }
                    }
                }
            }
            close_tile(true);
            ln.tile_end = (int32_t)S.tiles.size();
            if (ln.tile_end > ln.tile_begin) lanes.push_back(ln);
        }
    }
    S.n_lanes = (int32_t)lanes.size();
    for (const Lane& ln : lanes) S.max_lane_rows = std::max<int32_t>(S.max_lane_rows, ln.n_slots * G);
    S.tile_meta.resize(S.tiles.size());
    for (std::size_t i = 0; i < S.tiles.size(); ++i) {
        TileMeta& tm = S.tile_meta[i];
        std::memset(&tm, 0, sizeof tm);
        for (int g = 0; g < S.tiles[i].ng; ++g) {
            tm.info[g] = S.grp_info[S.tiles[i].grp_begin + g];
            tm.row[g] = S.grp_row[S.tiles[i].grp_begin + g];
        }
    }

    // ---- 3. CTA runs over the (head, lane, tile) sequence.  Cost of a tile:
    // its box rows (KV bytes) + a fixed per-tile cost + a softmax cost growing
    // with its attended (row, token) pairs; every item a CTA starts costs
    // item_cost more.  (A max(streaming, softmax) model and an L2 discount for
    // the re-read row blocks of wide stripes measured worse.)
    const int n_tiles = (int)S.tiles.size();
    std::vector<int32_t> tile_lane(n_tiles);
    for (int li = 0; li < (int)lanes.size(); ++li)
        for (int i = lanes[li].tile_begin; i < lanes[li].tile_end; ++i) tile_lane[i] = li;
    std::vector<int64_t> tcost(n_tiles);
    int64_t tile_sum = 0;   // per head
    for (int i = 0; i < n_tiles; ++i) {
        // softmax work: attended (row, token) pairs, in units of a dense 128 x 128 tile
        int64_t pairs = 0;
        for (int g = 0; g < S.tiles[i].ng; ++g) {
            const uint32_t info = S.grp_info[S.tiles[i].grp_begin + g];
            pairs += (int64_t)(info & 0xffu) * (int64_t)((info >> 20) - ((info >> 8) & 0xfffu)) * G;
        }
        tcost[i] = 16LL * S.tiles[i].ng + opt.tile_cost + (int64_t)opt.box_cost * S.tiles[i].nbox +
                   (int64_t)opt.row_cost * pairs / (128 * 128);
        tile_sum += tcost[i];
        S.kv_rows_loaded += 16LL * S.tiles[i].ng * n_heads;
    }
    const int n_cta = std::max(1, opt.num_ctas);
    // returns the most items any CTA got
    auto partition = [&](int item_cost) -> int {
        S.items.clear();
        S.cta_begin.assign(1, 0);
        const int64_t per_head = (int64_t)item_cost * (int64_t)lanes.size() + tile_sum;
        // each CTA boundary opens one more item than the (head, lane) count
        const int64_t total = per_head * n_heads + (int64_t)item_cost * (n_cta - 1);
        int cta = 0;
        int64_t acc = 0;
        ItemDesc* open = nullptr;
        for (int h = 0; h < n_heads; ++h) {
            for (int i = 0; i < n_tiles; ++i) {
                // boundary of CTA `cta` at cost (cta + 1) * total / n_cta (nearest tile edge)
                while (cta < n_cta - 1 && 2 * (acc * n_cta) >= (2LL * (cta + 1) * total - tcost[i] * n_cta)) {
                    S.cta_begin.push_back((int32_t)S.items.size());
                    ++cta;
                    open = nullptr;
                }
                const int li = tile_lane[i];
                if (!open || open->head != h || open->lane != li) {
                    ItemDesc it{};
                    it.head = h;
                    it.lane = li;
                    it.tile_begin = i;
                    it.tile_end = i;
                    it.slot_begin = lanes[li].slot_begin;
                    it.n_slots = lanes[li].n_slots;
                    S.items.push_back(it);
                    open = &S.items.back();
                    acc += item_cost;
                }
                open->tile_end = i + 1;
                acc += tcost[i];
            }
        }
        while ((int)S.cta_begin.size() < n_cta + 1) S.cta_begin.push_back((int32_t)S.items.size());
        int most = 0;
        for (int c = 0; c < n_cta; ++c) most = std::max(most, S.cta_begin[c + 1] - S.cta_begin[c]);
        return most;
    };
    // Min-max variant: the smallest per-CTA budget B for which a greedy cut of
    // the sequence into runs of cost <= B needs at most n_cta runs (binary
    // search on B; each greedy pass finds a run's end by galloping search on
    // prefix sums of tile costs and lane-segment starts).  The equal-split
    // cut above rounds every boundary to a tile edge and can leave the
    // heaviest CTA up to a tile plus an item over the mean.
    auto partition_minmax = [&](int item_cost) -> int {
        const int64_t N = (int64_t)n_heads * n_tiles;
        if (N == 0) {
            S.items.clear();
            S.cta_begin.assign(n_cta + 1, 0);
            return 0;
        }
        // prefix sums over the sequence (kept across calls: no page faults per step):
        // P[x] = cost of positions [0, x), NB[x] = lane-segment starts at positions 1..x
        static thread_local std::vector<int64_t> P;
        static thread_local std::vector<int32_t> NB;
        P.resize(N + 1);
        NB.resize(N + 1);
        P[0] = 0;
        int64_t maxt = 0;
        {
            int64_t x = 0;
            int32_t nb = 0;
            for (int h = 0; h < n_heads; ++h)
                for (int i = 0; i < n_tiles; ++i, ++x) {
                    P[x + 1] = P[x] + tcost[i];
                    maxt = std::max(maxt, tcost[i]);
                    if (x > 0 && (i == 0 || tile_lane[i] != tile_lane[i - 1])) ++nb;
                    NB[x] = nb;
                }
        }
        auto cost = [&](int64_t a, int64_t b) { return P[b] - P[a] + (int64_t)item_cost * (1 + NB[b - 1] - NB[a]); };
        auto runs = [&](int64_t cap, std::vector<int64_t>* cuts) {
            int64_t a = 0, guess = std::max<int64_t>(1, N / n_cta);
            int n = 0;
            while (a < N) {
                // the largest b with cost(a, b) <= cap (at least a + 1): gallop from
                // the previous run's length (runs are similar), then bisect
                int64_t lo, hi;
                const int64_t g = std::min(N, a + guess);
                if (g == a + 1 || cost(a, g) <= cap) {
                    int64_t step = std::max<int64_t>(1, guess / 4);
                    lo = g;
                    while (lo + step <= N && cost(a, lo + step) <= cap) {
                        lo += step;
                        step *= 2;
                    }
                    hi = std::min(N, lo + step - 1);
                } else {
                    // cost(a, g) > cap: the answer is in [a + 1, top]; gallop down
                    int64_t step = std::max<int64_t>(1, guess / 4), top = g - 1, bot = top - step;
                    while (bot > a && cost(a, bot) > cap) {
                        top = bot - 1;
                        step *= 2;
                        bot = top - step;
                    }
                    lo = std::max(a + 1, bot);
                    hi = std::max(lo, top);
                    if (cost(a, lo) > cap) hi = lo;   // a single position over the cap still forms a run
                }
                while (lo < hi) {
                    const int64_t mid = (lo + hi + 1) / 2;
                    if (cost(a, mid) <= cap) lo = mid; else hi = mid - 1;
                }
                if (cuts) cuts->push_back(lo);
                guess = std::max<int64_t>(1, lo - a);
                a = lo;
                if (++n > n_cta && !cuts) return n;   // infeasible budget: stop counting
            }
            return n;
        };
        const int64_t total = cost(0, N);
        // greedy with budget >= mean + largest piece never needs more than n_cta runs
        int64_t lo = std::max<int64_t>(maxt + item_cost, (total + n_cta - 1) / n_cta);
        int64_t hi = (total + n_cta - 1) / n_cta + maxt + item_cost;
        while (runs(hi, nullptr) > n_cta) hi += maxt + item_cost;   // (defensive)
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (runs(mid, nullptr) <= n_cta) hi = mid; else lo = mid + 1;
        }
        std::vector<int64_t> cuts;
        runs(lo, &cuts);
        S.items.clear();
        S.cta_begin.assign(1, 0);
        int64_t a = 0;
        int h = 0, i = 0;   // position a as (head, tile)
        for (const int64_t b : cuts) {
            ItemDesc* open = nullptr;
            for (int64_t x = a; x < b; ++x, ++i) {
                if (i == n_tiles) {
                    i = 0;
                    ++h;
                }
                const int li = tile_lane[i];
                if (!open || open->head != h || open->lane != li) {
                    ItemDesc it{};
                    it.head = h;
                    it.lane = li;
                    it.tile_begin = i;
                    it.tile_end = i;
                    it.slot_begin = lanes[li].slot_begin;
                    it.n_slots = lanes[li].n_slots;
                    S.items.push_back(it);
                    open = &S.items.back();
                }
                open->tile_end = i + 1;
            }
            S.cta_begin.push_back((int32_t)S.items.size());
            a = b;
        }
        while ((int)S.cta_begin.size() < n_cta + 1) S.cta_begin.push_back((int32_t)S.items.size());
        int most = 0;
        for (int c = 0; c < n_cta; ++c) most = std::max(most, S.cta_begin[c + 1] - S.cta_begin[c]);
        return most;
    };
    if (opt.minmax) {
        if (partition_minmax(opt.item_cost) > opt.many_items && opt.item_cost_many > opt.item_cost)
            partition_minmax(opt.item_cost_many);
    } else
    // Item switches cost 3.6-4.6 us each (per-CTA fit of traced durations,
    // profiles/r1_summary.md): where CTAs would run many short items (token
    // trees, many small branches) they are charged more, which measured
    // faster there (spec t256 -9 %); schedules of few long items keep the
    // base cost (few-shot is faster with it).
    if (partition(opt.item_cost) > opt.many_items && opt.item_cost_many > opt.item_cost) partition(opt.item_cost_many);

    // ---- 4. outputs: touched slots, direct vs partial, merge lists
    const int L = S.n_leaves;
    std::vector<int32_t> cover((size_t)L * n_heads, 0);
    // slots a tile attends, as a 128-bit mask (a lane has <= 128 slots): built
    // once per tile, OR-ed over an item's tiles (items of every head share them)
    static thread_local std::vector<uint64_t> tmask;
    tmask.assign(2 * S.tiles.size(), 0);
    auto range_bits = [](int lo, int hi, uint64_t& w0, uint64_t& w1) {   // bits [lo, hi)
        auto word = [](int lo_, int hi_) -> uint64_t {   // within one 64-bit word, 0 <= lo_ <= hi_ <= 64
            if (hi_ <= lo_) return 0;
            const uint64_t top = hi_ == 64 ? ~0ull : ((1ull << hi_) - 1);
            return top & ~((1ull << lo_) - 1);
        };
        w0 |= word(std::min(lo, 64), std::min(hi, 64));
        w1 |= word(std::max(lo, 64) - 64, std::max(hi, 64) - 64);
    };
    for (std::size_t i = 0; i < S.tiles.size(); ++i) {
        const TileDesc& td = S.tiles[i];
        for (int g = 0; g < td.ng; ++g) {
            const uint32_t info = S.grp_info[td.grp_begin + g];
            range_bits((int)((info >> 8) & 0xfffu), (int)(info >> 20), tmask[2 * i], tmask[2 * i + 1]);
        }
    }
    for (ItemDesc& it : S.items) {
        uint64_t m0 = 0, m1 = 0;
        for (int i = it.tile_begin; i < it.tile_end; ++i) {
            m0 |= tmask[2 * i];
            m1 |= tmask[2 * i + 1];
        }
        it.out_begin = (int32_t)S.slot_out.size();
        for (int j = 0; j < it.n_slots; ++j) {
            if ((j < 64 ? m0 >> j : m1 >> (j - 64)) & 1ull) {
                cover[(size_t)S.slot_leaf[it.slot_begin + j] * n_heads + it.head]++;
                S.slot_out.push_back(0);
            } else {
                S.slot_out.push_back(kSlotUnused);
            }
        }
    }
    // Partial ids are contiguous per merge record (record mi owns ids
    // [merge_begin[mi], merge_begin[mi+1]) in item order), so a merge reads
    // them without an id list.
    std::vector<int32_t> rec((size_t)L * n_heads, -1);  // leaf-head -> merge record
    std::vector<int32_t> rec_n;                          // partials per record (counting sort)
    for (int ii = 0; ii < (int)S.items.size(); ++ii) {
        const ItemDesc& it = S.items[ii];
        for (int j = 0; j < it.n_slots; ++j) {
            int32_t& code = S.slot_out[it.out_begin + j];
            if (code == kSlotUnused) continue;
            const int32_t leaf = S.slot_leaf[it.slot_begin + j];
            const size_t key = (size_t)leaf * n_heads + it.head;
            if (opt.final_direct && cover[key] == 1) {
                code = -1 - leaf;
                continue;
            }
            if (rec[key] < 0) {
                rec[key] = (int32_t)rec_n.size();
                rec_n.push_back(0);
                S.merge_leaf.push_back(leaf);
                S.merge_head.push_back(it.head);
            }
            code = rec[key];   // temporarily: the record
            rec_n[rec[key]]++;
        }
    }
    const int nrec = (int)rec_n.size();
    S.merge_begin.resize(nrec + 1);
    S.merge_begin[0] = 0;
    for (int mi = 0; mi < nrec; ++mi) S.merge_begin[mi + 1] = S.merge_begin[mi] + rec_n[mi];
    S.n_partials = S.merge_begin[nrec];
    S.part_merge.resize(S.n_partials);
    S.merge_parts.resize(S.n_partials);
    std::vector<int32_t> fill(S.merge_begin.begin(), S.merge_begin.end() - 1);
    for (const ItemDesc& it : S.items)   // item order within each record
        for (int j = 0; j < it.n_slots; ++j) {
            int32_t& code = S.slot_out[it.out_begin + j];
            if (code < 0) continue;
            const int mi = code;
            code = fill[mi]++;
            S.part_merge[code] = mi;
            S.merge_parts[code] = code;
        }
    S.merge_rec.resize(nrec);
    for (int mi = 0; mi < nrec; ++mi)
        S.merge_rec[mi] = {S.merge_leaf[mi], S.merge_head[mi], S.merge_begin[mi], rec_n[mi]};
    for (ItemDesc& it : S.items)
        for (int j = 0; j < it.n_slots; ++j)
            if (S.slot_out[it.out_begin + j] >= 0) it.pad |= 1;   // holds partials: takes part in merges
    // Fused merge (tcgen05 kernel): no merge launch.  At its end, after all
    // its items, a CTA publishes the partials it wrote (per record: how many)
    // and only then merges the records it owns.  Publication never waits, so
    // no CTA's wait can block another's: any ownership is deadlock-free while
    // every CTA is resident (<= one per SM).  Records are spread evenly over
    // the CTAs by merge work (rows x partials).
    S.fused_merge = opt.fused_merge;
    if (opt.fused_merge) {
        const int n_cta = (int)S.cta_begin.size() - 1;
        std::vector<int32_t> owner(nrec, -1);
        S.cta_pub_begin.assign(1, 0);
        std::vector<int32_t> cnt_here(nrec, 0), touched_recs;
        for (int c = 0; c < n_cta; ++c) {
            touched_recs.clear();
            for (int ii = S.cta_begin[c]; ii < S.cta_begin[c + 1]; ++ii) {
                const ItemDesc& it = S.items[ii];
                for (int j = 0; j < it.n_slots; ++j) {
                    const int32_t code = S.slot_out[it.out_begin + j];
                    if (code < 0) continue;
                    const int mi = S.part_merge[code];
                    if (cnt_here[mi]++ == 0) touched_recs.push_back(mi);
                }
            }
            for (int mi : touched_recs) {
                S.cta_pub.push_back({mi, cnt_here[mi]});
                cnt_here[mi] = 0;
            }
            S.cta_pub_begin.push_back((int32_t)S.cta_pub.size());
        }
        // even split of the records' merge work (G rows x (1 + partials) each)
        // into contiguous record ranges, one per CTA
        {
            int64_t total = 0;
            for (int mi = 0; mi < nrec; ++mi) total += 1 + rec_n[mi];
            int64_t acc = 0;
            for (int mi = 0; mi < nrec; ++mi) {
                owner[mi] = (int)std::min<int64_t>(n_cta - 1, (acc * n_cta) / std::max<int64_t>(1, total));
                acc += 1 + rec_n[mi];
            }
        }
        std::vector<int32_t> own_n(n_cta + 1, 0);
        int n_own_total = 0;
        for (int mi = 0; mi < nrec; ++mi)
            if (owner[mi] >= 0) {
                own_n[owner[mi] + 1]++;
                ++n_own_total;
            }
        S.cta_own_begin.assign(n_cta + 1, 0);
        for (int c = 0; c < n_cta; ++c) S.cta_own_begin[c + 1] = S.cta_own_begin[c] + own_n[c + 1];
        S.cta_own.resize(n_own_total);
        std::vector<int32_t> pos(S.cta_own_begin.begin(), S.cta_own_begin.end() - 1);
        for (int mi = 0; mi < nrec; ++mi)
            if (owner[mi] >= 0) S.cta_own[pos[owner[mi]]++] = mi;
    }
    for (int32_t l = 0; l < L; ++l)
        for (int h = 0; h < n_heads; ++h)
            if (cover[(size_t)l * n_heads + h] == 0) {
                S.empty.push_back(l);
                S.empty.push_back(h);
            }
    for (int32_t l : t.leaves) S.masked_q_tokens += t.path_tokens(l);
}

// Per-CTA schedule blobs (ta_internal.h, namespace blob): the tcgen05
// kernel's SMEM staging laid out on the host, so a CTA's first round trip
// (one fixed-size head copy) brings everything it needs to start streaming.
void build_cta_blobs(Schedule& S, const std::vector<int32_t>& pending_rows) {
    using namespace blob;
    const int n_cta = (int)S.cta_begin.size() - 1;
    S.cta_heads.assign((size_t)std::max(n_cta, 1) * HEAD_BYTES, 0);
    S.cta_tails.clear();
    auto put = [](std::vector<uint8_t>& v, const void* p, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(p);
        v.insert(v.end(), b, b + n);
    };
    auto pad16 = [](std::vector<uint8_t>& v) { v.resize((v.size() + 15) & ~size_t(15), 0); };
    std::vector<int32_t> slots;
    std::vector<TileDesc> tds;
    std::vector<TileMeta> tms;
    std::vector<int32_t> tids;   // global tile index of each staged tile
    std::vector<std::pair<int32_t, uint32_t>> copies;   // (tile, blob offset of its TileMeta copy)
    for (int c = 0; c < n_cta; ++c) {
        uint8_t* head = S.cta_heads.data() + (size_t)c * HEAD_BYTES;
        int32_t* hdr = reinterpret_cast<int32_t*>(head + HDR);
        int32_t* ioff = reinterpret_cast<int32_t*>(head + IOFF);
        int32_t* soff = reinterpret_cast<int32_t*>(head + SOFF);
        const int it0 = S.cta_begin[c], ni = S.cta_begin[c + 1] - it0;
        const int ni_s = std::min(ni, MAXI);
        tds.clear();
        tms.clear();
        tids.clear();
        slots.clear();
        int off = 0, so = 0;
        for (int k = 0; k < ni_s; ++k) {
            const ItemDesc& it = S.items[it0 + k];
            ioff[k] = off;
            soff[k] = so;
            off += it.tile_end - it.tile_begin;
            so += it.n_slots;
            for (int t = it.tile_begin; t < it.tile_end && (int)tds.size() < MAXT; ++t) {
                tds.push_back(S.tiles[t]);
                tms.push_back(S.tile_meta[t]);
                tids.push_back(t);
            }
            for (int j = 0; j < it.n_slots && (int)slots.size() < MAXS; ++j) slots.push_back(S.slot_leaf[it.slot_begin + j]);
        }
        ioff[ni_s] = off;
        soff[ni_s] = so;
        const int nt_s = (int)tds.size(), ns_s = (int)slots.size();
        int n_own = 0, n_pub = 0, o0 = 0, pb0 = 0;
        if (S.fused_merge) {
            o0 = S.cta_own_begin[c];
            n_own = S.cta_own_begin[c + 1] - o0;
            pb0 = S.cta_pub_begin[c];
            n_pub = S.cta_pub_begin[c + 1] - pb0;
        }
        hdr[N_ITEMS] = ni;
        hdr[N_TILES] = nt_s;
        hdr[N_SLOTS] = ns_s;
        hdr[N_OWN] = n_own;
        hdr[N_PUB] = n_pub;
        hdr[IT0] = it0;
        hdr[O0] = o0;
        hdr[PB0] = pb0;
        // leading tiles (<= 2: the ring) free of rows the step's ta_kv_append
        // writes: the kernel may load them before its dependency wait
        int early = 0;
        for (; early < std::min(nt_s, 2); ++early) {
            bool hit = false;
            for (int g = 0; g < tds[early].ng && !hit; ++g) {
                const int32_t r0 = tms[early].row[g], r1 = r0 + (int32_t)(tms[early].info[g] & 0xffu);
                auto it = std::lower_bound(pending_rows.begin(), pending_rows.end(), r0);
                hit = it != pending_rows.end() && *it < r1;
            }
            if (hit) break;
        }
        hdr[N_EARLY] = early;
        std::memcpy(head + H_ITEMS, S.items.data() + it0, (size_t)std::min(ni_s, HI) * sizeof(ItemDesc));
        std::memcpy(head + H_TD, tds.data(), (size_t)std::min(nt_s, HT) * sizeof(TileDesc));
        std::memcpy(head + H_TM, tms.data(), (size_t)std::min(nt_s, HT) * sizeof(TileMeta));
        std::memcpy(head + H_SLOT, slots.data(), (size_t)std::min(ns_s, HS) * 4);
        // tail sections
        hdr[TAIL_OFF] = (int32_t)S.cta_tails.size();
        size_t b0 = S.cta_tails.size();
        if (ni_s > HI) put(S.cta_tails, S.items.data() + it0 + HI, (size_t)(ni_s - HI) * sizeof(ItemDesc));
        hdr[T_ITEMS] = (int32_t)(S.cta_tails.size() - b0);
        b0 = S.cta_tails.size();
        if (nt_s > HT) put(S.cta_tails, tds.data() + HT, (size_t)(nt_s - HT) * sizeof(TileDesc));
        hdr[T_TD] = (int32_t)(S.cta_tails.size() - b0);
        b0 = S.cta_tails.size();
        for (int lt = 0; lt < nt_s; ++lt)
            copies.push_back({tids[lt], lt < HT ? (uint32_t)((size_t)c * HEAD_BYTES + H_TM + lt * sizeof(TileMeta))
                                                 : (uint32_t)(b0 + (lt - HT) * sizeof(TileMeta)) | 0x80000000u});
        if (nt_s > HT) put(S.cta_tails, tms.data() + HT, (size_t)(nt_s - HT) * sizeof(TileMeta));
        hdr[T_TM] = (int32_t)(S.cta_tails.size() - b0);
        b0 = S.cta_tails.size();
        if (ns_s > HS) put(S.cta_tails, slots.data() + HS, (size_t)(ns_s - HS) * 4);
        pad16(S.cta_tails);
        hdr[T_SLOT] = (int32_t)(S.cta_tails.size() - b0);
        b0 = S.cta_tails.size();
        const int no_s = std::min(n_own, MAXO), np_s = std::min(n_pub, MAXP);
        for (int x = 0; x < no_s; ++x) put(S.cta_tails, &S.merge_rec[S.cta_own[o0 + x]], 16);
        hdr[T_OWN] = (int32_t)(S.cta_tails.size() - b0);
        b0 = S.cta_tails.size();
        if (no_s) put(S.cta_tails, S.cta_own.data() + o0, (size_t)no_s * 4);
        pad16(S.cta_tails);
        hdr[T_OWNID] = (int32_t)(S.cta_tails.size() - b0);
        b0 = S.cta_tails.size();
        if (np_s) put(S.cta_tails, S.cta_pub.data() + pb0, (size_t)np_s * 8);
        pad16(S.cta_tails);
        hdr[T_PUB] = (int32_t)(S.cta_tails.size() - b0);
    }
    if (S.cta_tails.empty()) S.cta_tails.resize(16, 0);
    // copies by tile (counting sort)
    S.tile_copy_begin.assign(S.tiles.size() + 1, 0);
    for (const auto& cp : copies) S.tile_copy_begin[cp.first + 1]++;
    for (size_t t = 0; t < S.tiles.size(); ++t) S.tile_copy_begin[t + 1] += S.tile_copy_begin[t];
    S.tile_copy.assign(copies.size(), 0);
    std::vector<int32_t> pos(S.tile_copy_begin.begin(), S.tile_copy_begin.end() - 1);
    for (const auto& cp : copies) S.tile_copy[pos[cp.first]++] = cp.second;
}

void build_tail_map(const Tree& t, const PagePool& pool, Schedule& S) {
    S.grp_tile.assign(S.grp_row.size(), -1);
    for (size_t i = 0; i < S.tiles.size(); ++i)
        for (int g = 0; g < S.tiles[i].ng; ++g) S.grp_tile[S.tiles[i].grp_begin + g] = (int32_t)i;
    // a leaf's last token is the last row of its group (nothing follows it in its page)
    std::unordered_map<int32_t, int32_t> last_row;   // pool row -> group
    last_row.reserve(S.grp_row.size() * 2);
    for (size_t g = 0; g < S.grp_row.size(); ++g) last_row[S.grp_row[g] + (int32_t)(S.grp_info[g] & 0xffu) - 1] = (int32_t)g;
    S.tail_grp.assign(t.alive.size(), -1);
    const int P = pool.page_size;
    for (int32_t leaf : t.leaves) {
        const int64_t n = t.count[leaf];
        if (n == 0) continue;
        const auto& h = pool.handle(leaf);
        const int32_t row = (int32_t)(h.pages[(n - 1) / P] * P + (n - 1) % P);
        auto it = last_row.find(row);
        if (it != last_row.end()) S.tail_grp[leaf] = it->second;
    }
}

bool patch_schedule_appends(Schedule& S, const PagePool& pool,
                            const std::vector<std::pair<int32_t, int64_t>>& appends) {
    if (S.tail_grp.empty() || S.tile_copy_begin.empty()) return false;
    const int P = pool.page_size;
    // dry run: every token extends its leaf's tail group by the next pool row
    std::unordered_map<int32_t, int32_t> cnt;   // group -> count after the appends so far
    for (const auto& [leaf, tok] : appends) {
        if (leaf < 0 || leaf >= (int32_t)S.tail_grp.size() || S.tail_grp[leaf] < 0) return false;
        const int32_t g = S.tail_grp[leaf];
        auto it = cnt.find(g);
        const int32_t c0 = it != cnt.end() ? it->second : (int32_t)(S.grp_info[g] & 0xffu);
        const auto& h = pool.handle(leaf);
        const int32_t row = (int32_t)(h.pages[tok / P] * P + tok % P);
        if (c0 >= 16 || S.grp_row[g] + c0 != row) return false;
        cnt[g] = c0 + 1;
    }
    // apply: the group's count in grp_info, in the tile metadata and in every
    // CTA blob's copy of it
    for (const auto& [g, c] : cnt) {
        const uint32_t info = S.grp_info[g];
        const uint32_t ninfo = (info & ~0xffu) | (uint32_t)c;
        const int added = c - (int)(info & 0xffu);
        S.grp_info[g] = ninfo;
        const int32_t t = S.grp_tile[g];
        const int gi = g - S.tiles[t].grp_begin;
        S.tile_meta[t].info[gi] = ninfo;
        S.tiles[t].ntok = (uint16_t)(S.tiles[t].ntok + added);
        for (int32_t k = S.tile_copy_begin[t]; k < S.tile_copy_begin[t + 1]; ++k) {
            const uint32_t off = S.tile_copy[k];
            uint8_t* base = (off & 0x80000000u) ? S.cta_tails.data() + (off & 0x7fffffffu) : S.cta_heads.data() + off;
            std::memcpy(base + offsetof(TileMeta, info) + 4 * gi, &ninfo, 4);
        }
    }
    S.kv_tokens_unique += (int64_t)appends.size();
    S.masked_q_tokens += (int64_t)appends.size();   // each new token is on exactly one leaf's path
    return true;
}

void build_append_lists(Schedule& S, int n_heads, const std::vector<int32_t>& pending_rows,
                        const std::vector<int32_t>& tail_groups) {
    const int n_cta = (int)S.cta_begin.size() - 1;
    const int n_tiles = (int)S.tiles.size();
    if ((int64_t)S.tile_loc.size() != (int64_t)n_heads * n_tiles) {
        S.tile_loc.assign((size_t)n_heads * n_tiles, -1);
        for (int c = 0; c < n_cta; ++c) {
            int gt = 0;
            for (int i = S.cta_begin[c]; i < S.cta_begin[c + 1]; ++i) {
                const ItemDesc& it = S.items[i];
                for (int t = it.tile_begin; t < it.tile_end; ++t, ++gt)
                    S.tile_loc[(size_t)it.head * n_tiles + t] = (c << 16) | std::min(gt, 0xffff);
            }
        }
    }
    S.app_cta.assign((size_t)4 * n_cta, 0);
    S.app_list.clear();
    if (pending_rows.empty() || n_cta == 0) return;
    // (append index, tile) for every group holding a pending row
    std::vector<std::pair<int32_t, int32_t>> hits;
    const bool known = tail_groups.size() == pending_rows.size();
    if (known) {
        for (size_t i = 0; i < pending_rows.size(); ++i)
            if (tail_groups[i] >= 0) hits.push_back({(int32_t)i, S.grp_tile[tail_groups[i]]});
    } else {
        std::vector<std::pair<int32_t, int32_t>> sorted;   // (row, append index)
        sorted.reserve(pending_rows.size());
        for (size_t i = 0; i < pending_rows.size(); ++i) sorted.push_back({pending_rows[i], (int32_t)i});
        std::sort(sorted.begin(), sorted.end());
        for (int t = 0; t < n_tiles; ++t)
            for (int g = S.tiles[t].grp_begin; g < S.tiles[t].grp_begin + S.tiles[t].ng; ++g) {
                const int32_t r0 = S.grp_row[g], r1 = r0 + (int32_t)(S.grp_info[g] & 0xffu);
                for (auto it = std::lower_bound(sorted.begin(), sorted.end(), std::make_pair(r0, INT32_MIN));
                     it != sorted.end() && it->first < r1; ++it)
                    hits.push_back({it->second, t});
            }
    }
    // per CTA (counting sort): {append index, head, pool row}
    std::vector<int32_t> n_per(n_cta + 1, 0);
    for (const auto& [i, t] : hits)
        for (int h = 0; h < n_heads; ++h) {
            const int32_t loc = S.tile_loc[(size_t)h * n_tiles + t];
            if (loc >= 0) ++n_per[(loc >> 16) + 1];
        }
    for (int c = 0; c < n_cta; ++c) n_per[c + 1] += n_per[c];
    S.app_list.assign((size_t)4 * n_per[n_cta], 0);
    std::vector<int32_t> fill(n_per.begin(), n_per.end() - 1);
    for (int c = 0; c < n_cta; ++c) {
        S.app_cta[4 * c] = n_per[c];
        S.app_cta[4 * c + 1] = n_per[c + 1];
        S.app_cta[4 * c + 2] = INT32_MAX;
    }
    for (const auto& [i, t] : hits)
        for (int h = 0; h < n_heads; ++h) {
            const int32_t loc = S.tile_loc[(size_t)h * n_tiles + t];
            if (loc < 0) continue;
            const int c = loc >> 16, gt = loc & 0xffff;
            int32_t* e = &S.app_list[(size_t)4 * fill[c]++];
            e[0] = i;
            e[1] = h;
            e[2] = pending_rows[i];
            S.app_cta[4 * c + 2] = std::min(S.app_cta[4 * c + 2], gt);
        }
}

}  // namespace ta
