// ta_internal.h -- host-side data structures of the B200 DeFT-Flatten path.
//
// Tree / page pool / planner mirror the reference semantics (citations are
// relative to /root/reference/proj/include/treeattn); the device schedule and
// kernels are this framework's own design.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace ta {

// ---------------------------------------------------------------------------
// Errors: mapped 1:1 to the reference's exception classes at the C boundary.
struct Error : std::exception {
    int code;
    std::string msg;
    Error(int c, std::string m) : code(c), msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};
[[noreturn]] void fail(int code, const std::string& msg);

// ---------------------------------------------------------------------------
// DecodingTree (tree.hpp:38-269): ids sequential and never reused; children in
// insertion order (ascending id after restore); leaves() in DFS pre-order.
// Flat arrays indexed by node id plus derived DFS data rebuilt per mutation.
class KvHook {
public:
    virtual ~KvHook() = default;
    virtual void on_alloc(int32_t node, int64_t n) = 0;   // KvLifecycle (tree.hpp:19-25)
    virtual void on_extend(int32_t node, int64_t n) = 0;
    virtual void on_free(int32_t node) = 0;
};

struct Tree {
    int32_t root = -1;
    int32_t next_id = 0;
    int32_t n_alive = 0;
    std::vector<uint8_t> alive;
    std::vector<int32_t> parent;
    std::vector<int64_t> count;
    std::vector<std::vector<int32_t>> kids;
    KvHook* hook = nullptr;

    // derived (rebuild())
    std::vector<int32_t> dfs;      // pre-order
    std::vector<int32_t> leaves;   // leaf ids, DFS order
    std::vector<int32_t> leaf_lo;  // per id: [lo, hi) range of leaf indices under it
    std::vector<int32_t> leaf_hi;
    uint64_t version = 0;

    bool contains(int32_t id) const { return id >= 0 && id < (int32_t)alive.size() && alive[id]; }
    void reserve(int32_t n);
    void rebuild();
    void create(int64_t root_tokens);                                   // tree.hpp:40-51
    void restore(int32_t root, int n, const int32_t* ids, const int32_t* parents,
                 const int64_t* counts);                                // tree.hpp:207-238
    std::vector<int32_t> branch(int32_t at, const int64_t* counts, int n);   // tree.hpp:74-97
    void prune(int32_t at);                                             // tree.hpp:100-116
    void append(int32_t leaf, int64_t n);                               // tree.hpp:119-129
    int64_t total_tokens() const;
    int64_t path_tokens(int32_t leaf) const;
    void subtree(int32_t at, std::vector<int32_t>& out) const;
};

// ---------------------------------------------------------------------------
// PagePool accounting (kv_cache.hpp:33-187): page-per-node ownership, tail
// fill, LIFO free list.  Token t of a node lives at pages[t / P], slot t % P.
struct PagePool : KvHook {
    int page_size = 16;
    int64_t capacity = -1;  // device page capacity (-1: unbounded, host-only)
    struct Page {
        int32_t owner = -1;
        int32_t used = 0;
        int32_t live = 0;
    };
    struct Handle {
        std::vector<int32_t> pages;
        int64_t n_tokens = 0;
    };
    std::vector<Page> pages;
    std::vector<int32_t> free_list;
    std::unordered_map<int32_t, Handle> handles;
    int64_t live_slots = 0;

    void allocate(int32_t node, int64_t n);   // kv_cache.hpp:56-66
    void extend(int32_t node, int64_t n);     // kv_cache.hpp:68-89
    void release(int32_t node);               // kv_cache.hpp:91-102
    int32_t acquire_page(int32_t owner);      // kv_cache.hpp:158-173
    const Handle& handle(int32_t node) const;
    void reset();
    void on_alloc(int32_t node, int64_t n) override { allocate(node, n); }
    void on_extend(int32_t node, int64_t n) override { extend(node, n); }
    void on_free(int32_t node) override { release(node); }
};

// ---------------------------------------------------------------------------
// Reference plan (partition.hpp:37-68) plus the fused chunk view the device
// schedule is built from.
struct Plan {
    int block_size = 128;
    int strategy = 3;                          // TA_STRATEGY_* (partition.hpp:16): flatten by default
    // QkvGroups exactly as partition_flatten emits them
    std::vector<int32_t> seg_begin{0}, q_begin{0};
    std::vector<int32_t> seg_node, queries;
    std::vector<int64_t> seg_offset, seg_len;
    std::vector<uint64_t> seg_mask;
    // chunks = one per flush (sibling groups of a >64-query split fused)
    std::vector<int32_t> chunk_seg_begin{0};   // into cseg_*
    std::vector<int32_t> chunk_q_begin{0};     // into chunk_q
    std::vector<int32_t> cseg_node;
    std::vector<int64_t> cseg_offset, cseg_len;
    std::vector<int32_t> cseg_lo, cseg_hi;     // attending leaf-index interval
    std::vector<int32_t> chunk_q;              // sorted leaf indices
    int n_groups() const { return (int)seg_begin.size() - 1; }
    int n_chunks() const { return (int)chunk_seg_begin.size() - 1; }
};

void plan_flatten(const Tree& t, int block_size, Plan& out);   // partition.hpp:212-253
void make_plan(const Tree& t, int strategy, int block_size, Plan& out);   // partition.hpp:255-262
std::string plan_json(const Tree& t, const Plan& p);           // serde.hpp:41-61

// ---------------------------------------------------------------------------
// Device schedule (this framework's layout).
//
//   stripe  a maximal run of consecutive flatten chunks whose query sets fit
//           one row tile together (or, for chunks with more queries than a
//           tile holds, runs of chunks with the identical query set)
//   lane    one row block of a stripe: a fixed, sorted list of query slots
//           (leaf indices, <= max_rows / G of them) and the stripe tokens any
//           of those slots attend, cut into 16-row groups and tiles
//   group   <= 16 tokens at consecutive pool rows with one attending slot
//           range [b, e) (local slot indices of the lane): one TMA box row set
//   tile    <= 8 groups (<= 128 tokens): one KV stage / one MMA N extent
//   item    a run of tiles of one lane for one kv head, processed by one CTA
//           with its (m, l, O) kept on chip; a CTA owns a contiguous run of
//           the (head, lane, tile) sequence balanced by cost
// Items whose leaf-head is covered by one item write the final output
// directly.  Otherwise the leaf-head's items write (O/l, log2 lse) partial
// records, merged in item order (deterministic): at the end of the attention
// launch by the record's owner CTA (fused merge, tcgen05 kernel), or by the
// merge launch (FMA kernel).
struct TileDesc {          // 16 bytes, read by the device
    int32_t grp_begin;     // into grp_row / grp_info
    uint8_t ng;            // groups in the tile (1..8)
    uint8_t nbox;          // TMA boxes covering them
    uint16_t ntok;         // real tokens
    uint8_t box[8];        // (first group << 2) | log2(box rows / 16)
};
static_assert(sizeof(TileDesc) == 16, "TileDesc layout");

// The tile's groups packed for single-load access by the device (no load
// depends on another): slot ranges + counts, and first pool rows.
struct TileMeta {          // 64 bytes
    uint32_t info[8];      // grp_pack(count, b, e); 0 past ng
    int32_t row[8];        // first pool row of each group
};
static_assert(sizeof(TileMeta) == 64, "TileMeta layout");

struct ItemDesc {          // 32 bytes, read by the device
    int32_t head;          // local kv head
    int32_t tile_begin, tile_end;
    int32_t slot_begin;    // into slot_leaf (the lane's slots)
    int32_t n_slots;
    int32_t out_begin;     // into slot_out: one code per slot of the item
    int32_t lane;
    int32_t pad;
};
static_assert(sizeof(ItemDesc) == 32, "ItemDesc layout");

constexpr int32_t kSlotUnused = INT32_MIN;   // slot_out: slot not attended in this item

// Per-CTA schedule blob of the tcgen05 kernel, built on the host in the
// kernel's SMEM layout so a CTA stages its schedule with bulk copies: a
// fixed-size head (one copy round trip, enough to start streaming) and a
// variable tail (issued once the head has landed; read from tile HT, item HI,
// slot HS on).  Entries past the SMEM capacities are read from the global
// schedule arrays.
namespace blob {
constexpr int MAXI = 32, MAXT = 112, MAXS = 512, MAXO = 32, MAXP = 64;   // SMEM capacities
constexpr int HI = 2, HT = 4, HS = 128;                                  // head part
enum { N_ITEMS, N_TILES, N_SLOTS, N_OWN, N_PUB, IT0, TAIL_OFF, O0, PB0, T_ITEMS, T_TD, T_TM, T_SLOT, T_OWN, T_OWNID,
       T_PUB, N_EARLY, NHDR };
constexpr int HDR = 0;                        // int32[NHDR]: counts are staged counts except N_ITEMS / N_OWN / N_PUB
constexpr int IOFF = 80;                      // int32[MAXI + 1]: CTA-local first tile of each staged item
constexpr int SOFF = IOFF + 144;              // int32[MAXI + 1]: CTA-local first slot of each staged item
constexpr int H_ITEMS = SOFF + 144;           // ItemDesc[HI]
constexpr int H_TD = H_ITEMS + HI * 32;       // TileDesc[HT]
constexpr int H_TM = H_TD + HT * 16;          // TileMeta[HT]
constexpr int H_SLOT = H_TM + HT * 64;        // int32[HS]
constexpr int HEAD_BYTES = H_SLOT + HS * 4;   // tail: items, tiles, metas, slots, own records, own ids, pubs (16-byte sections)
static_assert(NHDR * 4 <= IOFF && (MAXI + 1) * 4 <= 144 && HEAD_BYTES % 16 == 0 && H_ITEMS % 16 == 0, "blob layout");
}  // namespace blob

inline uint32_t grp_pack(int count, int b, int e) {
    return (uint32_t)count | ((uint32_t)b << 8) | ((uint32_t)e << 20);
}

struct Schedule {
    std::vector<TileDesc> tiles;
    std::vector<TileMeta> tile_meta;  // per tile, packed copy of its groups
    std::vector<int32_t> grp_row;     // first pool row of the group (page * P + slot)
    std::vector<uint32_t> grp_info;   // grp_pack(count, b, e)
    std::vector<ItemDesc> items;
    std::vector<int32_t> cta_begin;   // [n_ctas + 1] into items
    std::vector<int32_t> slot_leaf;   // lanes' slots: leaf index (leaves() order)
    std::vector<int32_t> slot_out;    // per item slot: -1 - leaf (direct), partial id, or kSlotUnused
    std::vector<int32_t> part_merge;  // partial id -> merge record
    std::vector<int32_t> merge_leaf, merge_head;  // merge record -> leaf index, local kv head
    std::vector<int32_t> merge_begin; // [n_merge + 1] into merge_parts
    std::vector<int32_t> merge_parts; // partial ids in merge order (item order; contiguous per record)
    struct MergeRec {
        int32_t leaf, head, pbegin, n;
    };
    std::vector<MergeRec> merge_rec;  // device copy: one 16-byte load per record
    // fused merge (tcgen05 kernel): per CTA, the records it wrote partials for
    // (record, partial count) and the records it merges at its end
    bool fused_merge = false;
    struct Pub {
        int32_t rec, n;
    };
    std::vector<int32_t> cta_pub_begin;   // [n_ctas + 1] into cta_pub
    std::vector<Pub> cta_pub;
    std::vector<int32_t> cta_own_begin;   // [n_ctas + 1] into cta_own
    std::vector<int32_t> cta_own;         // merge records
    // decode-step fast path (tcgen05 schedules, patch_schedule_appends): per
    // node id the group holding a leaf's last token (-1: none), group -> tile,
    // and where the CTA blobs keep copies of each tile's TileMeta (byte offsets;
    // bit 31 set: into cta_tails, else into cta_heads)
    std::vector<int32_t> tail_grp;
    std::vector<int32_t> grp_tile;
    std::vector<int32_t> tile_copy_begin;
    std::vector<uint32_t> tile_copy;
    // fused decode-step append (tcgen05 kernel): (local head, tile) -> the CTA
    // running it and its CTA-local tile index (cta << 16 | gt; -1: none), and
    // per step the rows each CTA writes before loading them (ta_kv_append
    // deferred into ta_attend): per CTA {begin, end, first local tile, 0} into
    // app_list {append index, local head, pool row, 0}
    std::vector<int32_t> tile_loc;
    std::vector<int32_t> app_cta;     // int4 per CTA
    std::vector<int32_t> app_list;    // int4 per entry
    std::vector<uint8_t> cta_heads;   // [n_ctas][blob::HEAD_BYTES]
    std::vector<uint8_t> cta_tails;   // packed tails (16-byte sections)
    std::vector<int32_t> empty;       // [n][2] (leaf, local head) pairs with no path tokens
    int32_t n_lanes = 0;
    int32_t max_lane_rows = 0;        // max rows (slots x G) of any lane
    int32_t n_partials = 0;
    int32_t n_leaves = 0;
    int64_t kv_tokens_unique = 0;     // per kv head
    int64_t kv_rows_loaded = 0;       // box rows loaded, all local heads
    int64_t masked_q_tokens = 0;      // sum over leaves of path tokens (flops / (4 d h_q))
    int64_t n_stripes = 0;

    void clear() {
        tiles.clear(); tile_meta.clear(); grp_row.clear(); grp_info.clear(); items.clear(); cta_begin.clear();
        slot_leaf.clear(); slot_out.clear(); part_merge.clear(); merge_leaf.clear(); merge_head.clear();
        merge_begin.clear(); merge_parts.clear(); merge_rec.clear(); empty.clear();
        fused_merge = false;
        cta_pub_begin.clear(); cta_pub.clear(); cta_own_begin.clear(); cta_own.clear();
        cta_heads.clear(); cta_tails.clear();
        tail_grp.clear(); grp_tile.clear(); tile_copy_begin.clear(); tile_copy.clear();
        tile_loc.clear(); app_cta.clear(); app_list.clear();
        n_lanes = n_partials = n_leaves = max_lane_rows = 0;
        kv_tokens_unique = kv_rows_loaded = masked_q_tokens = n_stripes = 0;
    }
};

struct SchedOptions {
    int max_rows = 128;        // rows (slots x G) per lane: 128 for the MMA kernel, 8/16 for FMA
    int tile_groups = 8;       // groups per tile
    int num_ctas = 148;        // persistent grid
    int tile_cost = 24;        // fixed per-tile cost, in box rows
    int box_cost = 0;          // per TMA box of a tile (partial tiles of scattered rows issue more), in box rows
    int row_cost = 15;         // softmax cost of a dense tile (128 x 128 attended pairs), in box rows
                               // (swept: 15 beats 60 by 3 % on few-shot, 14 % on 70B, ties on reasoning)
    int item_cost = 300;       // cost of starting an item (Q load, epilogue), in box rows
    int item_cost_many = 450;  // ... when the base cost leaves some CTA more than many_items items
    int many_items = 4;
    int minmax = 1;            // CTA runs: 1 min-max budget (binary search; measured better on
                               // every config), 0 equal split points
    bool fuse_chunks = true;   // stripes span consecutive plan chunks (flatten); the ablation
                               // strategies run each plan group as its own stripe
    bool use_mma = true;       // bf16 d128 only
    int fma_max_rows = 8;      // rows per lane of the FMA kernel (8 or 16)
    bool final_direct = true;  // single-item leaf-heads written directly
    bool fused_merge = false;  // split leaf-heads merged inside the attention launch, at the end of the
                               // record's owner CTA after every CTA has published its partial counts
                               // (tcgen05 kernel, all CTAs co-resident); else by the merge launch
    int64_t trace_ptr = 0;     // debug: device buffer for the kernel's clock64 trace
};

void build_schedule(const Tree& t, const PagePool& pool, const Plan& plan, int group_size,
                    int n_kv_heads_local, const SchedOptions& opt, Schedule& out);
// Decode-step fast path: the leaf-tail map of a built schedule (after
// build_cta_blobs), and the in-place patch for tokens appended to leaves since
// (leaf node, token index) -- every new token must extend its leaf's tail group
// by the next pool row (same page, group not full); false (nothing changed)
// otherwise, and the caller rebuilds.
void build_tail_map(const Tree& t, const PagePool& pool, Schedule& S);
bool patch_schedule_appends(Schedule& S, const PagePool& pool,
                            const std::vector<std::pair<int32_t, int64_t>>& appends);
// per-CTA head / tail blobs of a built schedule (tcgen05 kernel)
// pending_rows: pool rows the step's ta_kv_append writes (sorted); a CTA's
// leading tiles without any of them may be loaded before the dependency wait
void build_cta_blobs(Schedule& S, const std::vector<int32_t>& pending_rows);
// the fused append's per-CTA row lists for the rows appended since the last
// prepare (pending_rows, in append order); tail_groups[i] >= 0: the group of
// pending row i is known (fast path), else found by a scan of the groups
void build_append_lists(Schedule& S, int n_heads, const std::vector<int32_t>& pending_rows,
                        const std::vector<int32_t>& tail_groups);

}  // namespace ta
