// host.cpp -- tree mirror, page accounting, bit-exact flatten planner and the
// device schedule builder.  Reference citations are relative to
// /root/reference/proj/include/treeattn.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <numeric>

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
    for (int i = 0; i < n; ++i) {
        const int32_t id = next_id++;
        alive[id] = 1;
        parent[id] = at;
        count[id] = counts[i];
        kids[id].clear();
        kids[at].push_back(id);
        created.push_back(id);
        ++n_alive;
        if (hook) hook->on_alloc(id, counts[i]);
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
    extend(node, n);
}

void PagePool::extend(int32_t node, int64_t n) {
    auto it = handles.find(node);
    if (it == handles.end()) fail(TA_ERR_LOGIC, "extend: no handle for node");
    Handle& h = it->second;
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
// partition_flatten (partition.hpp:212-253) via leaf intervals.
//
// Walk nodes in DFS pre-order, stream their tokens, cut every block_size
// tokens (0-token nodes contribute nothing).  Per flush the query list is the
// union of the segments' leaf intervals in leaves() order; a segment's mask
// bit j is set iff query j lies in the segment node's interval, i.e. a
// contiguous run.  >64 queries: 64-query slices that keep every segment
// (emit_groups, partition.hpp:102-126).  Bit-exact with plan_to_json.
// ===========================================================================
static inline uint64_t run_mask(int b, int e) {
    if (e <= b) return 0;
    const int n = e - b;
    return (n >= 64 ? ~0ULL : ((1ULL << n) - 1)) << b;
}

void plan_flatten(const Tree& t, int bs, Plan& P) {
    if (bs < 1) fail(TA_ERR_INVALID_ARGUMENT, "partition: block_size must be >= 1");
    P = Plan{};
    P.block_size = bs;
    struct Pend {
        int32_t node;
        int64_t off, len;
    };
    std::vector<Pend> pend;
    std::vector<std::pair<int32_t, int32_t>> iv;
    std::vector<int32_t> Q;
    int64_t fill = 0;

    auto flush = [&] {
        if (pend.empty()) return;
        iv.clear();
        for (const Pend& s : pend) iv.emplace_back(t.leaf_lo[s.node], t.leaf_hi[s.node]);
        std::vector<std::pair<int32_t, int32_t>> sorted = iv;
        std::stable_sort(sorted.begin(), sorted.end());
        Q.clear();
        int32_t end = -1;
        for (auto [lo, hi] : sorted) {
            const int32_t from = std::max(lo, end);
            for (int32_t q = from; q < hi; ++q) Q.push_back(q);
            end = std::max(end, hi);
        }
        // chunk view
        for (std::size_t s = 0; s < pend.size(); ++s) {
            P.cseg_node.push_back(pend[s].node);
            P.cseg_offset.push_back(pend[s].off);
            P.cseg_len.push_back(pend[s].len);
            P.cseg_lo.push_back(iv[s].first);
            P.cseg_hi.push_back(iv[s].second);
        }
        P.chunk_seg_begin.push_back((int32_t)P.cseg_node.size());
        P.chunk_q.insert(P.chunk_q.end(), Q.begin(), Q.end());
        P.chunk_q_begin.push_back((int32_t)P.chunk_q.size());
        // reference groups
        const int nq = (int)Q.size();
        const bool split = nq > 64;
        for (int base = 0; base < nq; base += 64) {
            const int cnt = std::min(64, nq - base);
            const std::size_t seg_mark = P.seg_node.size();
            bool any = false;
            for (std::size_t s = 0; s < pend.size(); ++s) {
                const int b = (int)(std::lower_bound(Q.begin(), Q.end(), iv[s].first) - Q.begin());
                const int e = (int)(std::lower_bound(Q.begin(), Q.end(), iv[s].second) - Q.begin());
                const int bb = std::clamp(b, base, base + cnt) - base;
                const int ee = std::clamp(e, base, base + cnt) - base;
                const uint64_t mask = run_mask(bb, ee);
                if (mask == 0 && !split) continue;
                P.seg_node.push_back(pend[s].node);
                P.seg_offset.push_back(pend[s].off);
                P.seg_len.push_back(pend[s].len);
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
        pend.clear();
        fill = 0;
    };

    for (int32_t id : t.dfs) {
        int64_t remaining = t.count[id], offset = 0;
        while (remaining > 0) {
            const int64_t take = std::min<int64_t>(remaining, bs - fill);
            pend.push_back({id, offset, take});
            offset += take;
            remaining -= take;
            fill += take;
            if (fill == bs) flush();
        }
    }
    flush();
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
    s += "],\"strategy\":\"flatten\"}";
    (void)t;
    return s;
}

// ===========================================================================
// Device schedule.
//
// Every flatten chunk is one unit of KV streaming work.  Its query list is
// cut into blocks of at most S slots (S = rows-per-unit / G, rows being
// (query, q-head-in-group) pairs); a block keeps only the segments some of
// its queries attend.  Consecutive chunks whose blocks fit together are
// merged into one unit (a span), so queries that persist across chunks
// (shared prefixes) accumulate on-chip and leave one (m, l, O) partial per
// span instead of one per chunk.  Leaves covered by a single unit are
// written directly; the rest are merged by the merge kernel in unit order.
// ===========================================================================
namespace {

struct Piece {
    int32_t node;
    int64_t off, len;
    int32_t lo, hi;
};

constexpr int kMaxUnitGroups = 256;  // = MAX_GRP of attn_mma.cu

struct OpenUnit {
    std::vector<int32_t> slots;  // sorted leaf indices
    std::vector<Piece> pieces;
    int64_t tokens = 0;
    int64_t grp_est = 0;         // upper bound on 16-row TMA groups
    int last_chunk = -1;
    bool mma = false;
};

void sorted_union(const std::vector<int32_t>& a, const int32_t* b, int nb, std::vector<int32_t>& out) {
    out.clear();
    std::set_union(a.begin(), a.end(), b, b + nb, std::back_inserter(out));
}

}  // namespace

void build_schedule(const Tree& t, const PagePool& pool, const Plan& plan, int G,
                    int n_kv_heads_local, bool bf16, const SchedOptions& opt, Schedule& S) {
    S = Schedule{};
    S.n_leaves = (int32_t)t.leaves.size();
    const int P = pool.page_size;
    const int nc = plan.n_chunks();

    // --- per-chunk path and query blocks
    struct Block {
        int chunk;
        int q0, q1;  // into plan.chunk_q
        bool mma;
        int64_t tokens;
        int64_t grp_est;
    };
    std::vector<Block> blocks;
    int64_t work_tokens = 0;
    for (int c = 0; c < nc; ++c) {
        const int qb = plan.chunk_q_begin[c], qe = plan.chunk_q_begin[c + 1];
        const int nq = qe - qb;
        if (nq == 0) continue;
        const int64_t rows = (int64_t)nq * G;
        const bool mma = bf16 && opt.use_mma && rows > opt.fma_max_rows;
        const int cap_rows = mma ? opt.mma_max_rows : opt.fma_max_rows;
        const int S_slots = std::max(1, cap_rows / G);
        const int nb = (nq + S_slots - 1) / S_slots;
        for (int k = 0; k < nb; ++k) {
            const int a = qb + (int)((int64_t)nq * k / nb);
            const int b = qb + (int)((int64_t)nq * (k + 1) / nb);
            int64_t toks = 0, grp = 0;
            for (int s = plan.chunk_seg_begin[c]; s < plan.chunk_seg_begin[c + 1]; ++s)
                if (plan.cseg_hi[s] > plan.chunk_q[a] && plan.cseg_lo[s] <= plan.chunk_q[b - 1]) {
                    toks += plan.cseg_len[s];
                    grp += (plan.cseg_len[s] + 15) / 16 + 1;
                }
            blocks.push_back({c, a, b, mma, toks, grp});
            work_tokens += toks;
        }
        for (int s = plan.chunk_seg_begin[c]; s < plan.chunk_seg_begin[c + 1]; ++s)
            S.kv_tokens_unique += plan.cseg_len[s];
    }

    // span length: aim at ~2 waves of CTAs over all kv heads
    int64_t span = opt.span_tokens;
    if (span <= 0) {
        const int64_t target_units = std::max<int64_t>(1, (2LL * opt.num_sms) / std::max(1, n_kv_heads_local));
        span = std::max<int64_t>(plan.block_size, (work_tokens + target_units - 1) / target_units);
    }

    // --- greedy span merge
    std::vector<OpenUnit> done, open;
    std::vector<int32_t> tmp;
    auto close_stale = [&](int chunk) {
        for (std::size_t i = 0; i < open.size();) {
            if (open[i].last_chunk < chunk - 1) {
                done.push_back(std::move(open[i]));
                open.erase(open.begin() + (long)i);
            } else {
                ++i;
            }
        }
    };
    for (const Block& bl : blocks) {
        close_stale(bl.chunk);
        const int cap_rows = bl.mma ? opt.mma_max_rows : opt.fma_max_rows;
        const int S_slots = std::max(1, cap_rows / G);
        const int32_t* bq = plan.chunk_q.data() + bl.q0;
        const int nb = bl.q1 - bl.q0;
        int pick = -1;
        for (std::size_t i = 0; i < open.size(); ++i) {
            OpenUnit& u = open[i];
            if (u.mma != bl.mma || u.last_chunk != bl.chunk - 1) continue;
            if (u.tokens + bl.tokens > span) continue;
            // MMA units keep their group metadata in SMEM: <= kMaxUnitGroups boxes
            if (u.mma && u.grp_est + bl.grp_est > kMaxUnitGroups) continue;
            sorted_union(u.slots, bq, nb, tmp);
            if ((int)tmp.size() > S_slots) continue;
            // prefer exact continuation of the same query block
            if (pick < 0 || (int)tmp.size() == (int)u.slots.size()) pick = (int)i;
        }
        if (pick < 0) {
            open.emplace_back();
            open.back().mma = bl.mma;
            pick = (int)open.size() - 1;
        }
        OpenUnit& u = open[pick];
        sorted_union(u.slots, bq, nb, tmp);
        u.slots = tmp;
        for (int s = plan.chunk_seg_begin[bl.chunk]; s < plan.chunk_seg_begin[bl.chunk + 1]; ++s)
            if (plan.cseg_hi[s] > bq[0] && plan.cseg_lo[s] <= bq[nb - 1]) {
                // the segment's interval must intersect the block itself
                const int32_t* lo_it = std::lower_bound(bq, bq + nb, plan.cseg_lo[s]);
                if (lo_it == bq + nb || *lo_it >= plan.cseg_hi[s]) continue;
                // attended only by this chunk's block: the unit may hold other
                // slots (from neighbouring chunks) that belong to a sibling block here
                u.pieces.push_back({plan.cseg_node[s], plan.cseg_offset[s], plan.cseg_len[s],
                                    std::max(plan.cseg_lo[s], bq[0]), std::min(plan.cseg_hi[s], bq[nb - 1] + 1)});
                u.tokens += plan.cseg_len[s];
            }
        u.grp_est += bl.grp_est;
        u.last_chunk = bl.chunk;
    }
    for (auto& u : open) done.push_back(std::move(u));

    // --- leaf coverage counts -> direct vs partial
    std::vector<int32_t> cover(S.n_leaves, 0);
    for (const auto& u : done)
        for (int32_t l : u.slots) cover[l]++;

    std::vector<std::vector<int32_t>> leaf_parts(S.n_leaves);
    auto emit = [&](const OpenUnit& u, std::vector<UnitDesc>& dst) {
        UnitDesc d;
        d.tok_begin = (int32_t)S.tok_row.size();
        d.slot_begin = (int32_t)S.slot_leaf.size();
        d.n_slots = (int32_t)u.slots.size();
        for (int32_t l : u.slots) {
            S.slot_leaf.push_back(l);
            if (opt.final_direct && cover[l] == 1) {
                S.slot_part.push_back(-1 - l);
            } else {
                leaf_parts[l].push_back(S.n_partials);
                S.slot_part.push_back(S.n_partials++);
            }
        }
        for (const Piece& pc : u.pieces) {
            const int b = (int)(std::lower_bound(u.slots.begin(), u.slots.end(), pc.lo) - u.slots.begin());
            const int e = (int)(std::lower_bound(u.slots.begin(), u.slots.end(), pc.hi) - u.slots.begin());
            const auto& h = pool.handle(pc.node);
            for (int64_t k = 0; k < pc.len; ++k) {
                const int64_t tok = pc.off + k;
                S.tok_row.push_back((int32_t)(h.pages[tok / P] * P + tok % P));
                S.tok_be.push_back((uint32_t)b | ((uint32_t)e << 16));
            }
        }
        d.n_tokens = (int32_t)(S.tok_row.size() - d.tok_begin);
        S.kv_tokens_loaded += d.n_tokens;
        d.grp_begin = (int32_t)S.grp_row.size();
        d.n_grp = 0;
        d.pad0 = d.pad1 = 0;
        if (u.mma) {
            for (int32_t k = d.tok_begin; k < d.tok_begin + d.n_tokens;) {
                const int32_t row0 = S.tok_row[k];
                const uint32_t be = S.tok_be[k];
                int cnt = 1;
                while (cnt < 16 && k + cnt < d.tok_begin + d.n_tokens && S.tok_row[k + cnt] == row0 + cnt &&
                       S.tok_be[k + cnt] == be)
                    ++cnt;
                S.grp_row.push_back(row0);
                S.grp_info.push_back(grp_pack(cnt, (int)(be & 0xffffu), (int)(be >> 16)));
                k += cnt;
            }
            d.n_grp = (int32_t)S.grp_row.size() - d.grp_begin;
            if (d.n_grp > kMaxUnitGroups) fail(TA_ERR_LOGIC, "schedule: MMA unit exceeds its group capacity");
            S.kv_tokens_loaded += 16LL * d.n_grp - d.n_tokens;  // box over-read
        }
        dst.push_back(d);
    };
    for (const auto& u : done) emit(u, u.mma ? S.units_mma : S.units_fma);

    S.merge_begin.push_back(0);
    for (int32_t l = 0; l < S.n_leaves; ++l) {
        if (opt.final_direct && cover[l] == 1) continue;
        S.merge_leaf.push_back(l);
        S.merge_parts.insert(S.merge_parts.end(), leaf_parts[l].begin(), leaf_parts[l].end());
        S.merge_begin.push_back((int32_t)S.merge_parts.size());
    }
    for (int32_t l : t.leaves) S.masked_q_tokens += t.path_tokens(l);
}

}  // namespace ta
