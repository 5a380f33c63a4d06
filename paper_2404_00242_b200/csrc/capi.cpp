// capi.cpp -- extern "C" boundary (include/treeattn_b200.h).  Owns the
// context: tree mirror, page accounting, device KV pools, per-step schedule
// metadata and scratch.  No exception crosses the boundary; there is no CPU
// fallback for attention.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "ta_internal.h"
#include "ta_kernels.h"
#include "treeattn_b200.h"

using namespace ta;

struct ta_ctx {
    int device = -1;
    ta_shape shape{};
    int G = 1;
    int hq_loc = 1;
    int esize = 4;
    int out_esize = 4;
    Tree tree;
    PagePool pool;
    Plan plan;
    Schedule sched;
    SchedOptions opt;
    bool plan_valid = false;
    uint64_t plan_version = ~0ull;
    int plan_bs = -1;
    bool prepared = false;
    uint64_t prepared_version = ~0ull;
    int prepared_bs = -1;
    // decode-step fast path: tokens appended by ta_tree_append_leaves since the
    // last ta_prepare, as (leaf, token index), while no other mutation happened
    std::vector<std::pair<int32_t, int64_t>> fast_log;
    uint64_t fast_log_version = ~0ull;   // tree version after the last logged append
    bool fast_bad = true;
    int64_t n_fast_prepares = 0;
    int64_t n_noop_prepares = 0;        // ta_prepare calls that found nothing to rebuild

    // TMA descriptors (CUtensorMap, 128 B) over the whole K / V pools
    alignas(64) unsigned char tmap_k[512];   // CUtensorMap for 16/32/64/128-row boxes
    alignas(64) unsigned char tmap_v[512];
    bool tmaps_ok = false;

    // device pools: one K and one V slab per layer, [n_loc][max_pages][P][D]
    void* kv_k = nullptr;
    void* kv_v = nullptr;
    int64_t layer_elems = 0;  // elements per layer slab
    int64_t head_stride = 0;  // elements per (layer, head) pool

    // schedule metadata: one device blob of fixed-offset parts (see
    // upload_schedule) + double-buffered pinned staging
    void* meta_dev = nullptr;
    std::vector<size_t> meta_part_off, meta_part_cap;
    size_t meta_bytes_total = 0;
    void* meta_host[2] = {nullptr, nullptr};
    cudaEvent_t meta_done[2] = {nullptr, nullptr};
    int meta_buf = 0;
    int64_t graph_epoch = 0;      // bumped whenever a relocation invalidates captured launches
    const DevCounts* d_counts = nullptr;
    const int32_t* d_append_rows = nullptr;
    int64_t n_append = 0;         // tokens whose rows the last ta_prepare uploaded for ta_kv_append
    int64_t t_plan_ns = 0, t_sched_ns = 0, t_upload_ns = 0;   // host time of the last ta_prepare
    std::vector<int32_t> pending_rows;   // pool rows of tokens appended since the last ta_prepare
    std::vector<int32_t> pending_sorted; // (sorted copy for the schedule blobs)
    bool host_q_poll = true;             // option "host_q_poll": attend_host_async's kernel waits for q on the device
    bool fuse_append = true;             // option "fuse_append": ta_kv_append deferred into ta_attend (tcgen05 path)
    std::vector<const void*> app_k, app_v;   // per layer: new rows recorded by ta_kv_append for the next ta_attend
    const int32_t* d_app_cta = nullptr;
    const int32_t* d_app_list = nullptr;
    bool early_kv = false;               // option "early_kv": leading KV tiles loaded before the dependency wait
                                         // (off: in the 32-layer graph it measured +0.9 µs per few-shot layer,
                                         // the early loads competing with the previous launch's merge phase)
    const TileDesc* d_tiles = nullptr;
    const TileMeta* d_tile_meta = nullptr;
    const int32_t* d_grp_row = nullptr;
    const uint32_t* d_grp_info = nullptr;
    const ItemDesc* d_items = nullptr;
    const int32_t* d_cta_begin = nullptr;
    const int32_t* d_slot_leaf = nullptr;
    const int32_t* d_slot_out = nullptr;
    const int4* d_merge_rec = nullptr;
    const int32_t* d_part_merge = nullptr;
    const int32_t* d_empty = nullptr;
    const int32_t* d_cta_pub_begin = nullptr;
    const int2* d_cta_pub = nullptr;
    const int32_t* d_cta_own_begin = nullptr;
    const int32_t* d_cta_own = nullptr;
    const uint8_t* d_cta_heads = nullptr;
    const uint8_t* d_cta_tails = nullptr;
    unsigned* merge_cnt = nullptr;   // fused merge counters, one per merge record
    size_t merge_cnt_n = 0;          // capacity (records)
    bool fused_merge = true;         // option "fused_merge"
    int strategy = TA_STRATEGY_FLATTEN;   // option "strategy": the partition.hpp strategy planned
    bool pdl = true;
    int prefetch_tiles = 2;
    int64_t trace = 0;  // debug: device buffer for the MMA kernel's pipeline trace
    int64_t timeline = 0;   // debug: per-launch start/end timestamps
    int num_sms = 148;

    // host copy of the schedule for ta_schedule_get
    Schedule dbg_sched;

    // partial scratch: o [part_rec_cap][G][D] then lse [part_rec_cap][G]
    float* part = nullptr;
    size_t part_rec_cap = 0;

    // staging for kv writes and host-buffer attend
    void* stage_dev = nullptr;
    size_t stage_cap = 0;
    void* stage_host = nullptr;
    size_t stage_host_cap = 0;
    void* io_dev = nullptr;
    size_t io_cap = 0;
    // pipelined host-buffer attend (ta_attend_host_async): a ring of device
    // q / out slots; H2D and D2H on their own streams so that consecutive
    // calls overlap copy-in, attention and copy-out
    static constexpr int kIoSlots = 3;
    struct IoSlot {
        void* dev = nullptr;
        size_t cap = 0;
        cudaEvent_t h2d = nullptr, kern = nullptr, d2h = nullptr;
        bool used = false;
    };
    IoSlot io_slot[kIoSlots];
    int io_next = 0;
    // q-ready flags of the io slots (device words written by stream memory
    // operations after each copy-in; the tcgen05 kernel polls its slot's
    // flag instead of the compute stream waiting on an event, which would
    // cut the launch chain between consecutive layers)
    unsigned* io_flags = nullptr;
    unsigned io_seq[kIoSlots] = {0, 0, 0};
    const unsigned* q_flag = nullptr;   // set for the duration of one attend_impl
    unsigned q_seq = 0;
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;

    ~ta_ctx() {
        if (device >= 0) {
            cudaSetDevice(device);
            cudaFree(kv_k);
            cudaFree(kv_v);
            cudaFree(meta_dev);
            cudaFreeHost(meta_host[0]);
            cudaFreeHost(meta_host[1]);
            cudaFree(part);
            cudaFree(merge_cnt);
            cudaFree(stage_dev);
            cudaFreeHost(stage_host);
            cudaFree(io_dev);
            cudaFree(io_flags);
            for (IoSlot& sl : io_slot) {
                cudaFree(sl.dev);
                if (sl.h2d) cudaEventDestroy(sl.h2d);
                if (sl.kern) cudaEventDestroy(sl.kern);
                if (sl.d2h) cudaEventDestroy(sl.d2h);
            }
            if (h2d_stream) cudaStreamDestroy(h2d_stream);
            if (d2h_stream) cudaStreamDestroy(d2h_stream);
            for (cudaEvent_t e : meta_done)
                if (e) cudaEventDestroy(e);
        }
    }
};

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& m) {
    g_err = m;
    return code;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return TA_OK;
    } catch (const Error& e) {
        return set_err(e.code, e.msg);
    } catch (const std::bad_alloc&) {
        return set_err(TA_ERR_OUT_OF_MEMORY, "host allocation failed");
    } catch (const std::exception& e) {
        return set_err(TA_ERR_LOGIC, e.what());
    }
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(e == cudaErrorMemoryAllocation ? TA_ERR_OUT_OF_MEMORY : TA_ERR_CUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
}

void need_device(const ta_ctx* c) {
    if (c->device < 0) fail(TA_ERR_NO_DEVICE, "context has no CUDA device (host-only context)");
}

void grow_dev(void** p, size_t* cap, size_t need) {
    if (need <= *cap) return;
    size_t n = std::max(need, *cap * 2);
    cudaFree(*p);
    *p = nullptr;
    cuda_check(cudaMalloc(p, n), "cudaMalloc");
    *cap = n;
}

void grow_host(void** p, size_t* cap, size_t need) {
    if (need <= *cap) return;
    size_t n = std::max(need, *cap * 2);
    cudaFreeHost(*p);
    *p = nullptr;
    cuda_check(cudaMallocHost(p, n), "cudaMallocHost");
    *cap = n;
}

void ensure_plan(ta_ctx* c, int bs) {
    if (c->plan_valid && c->plan_version == c->tree.version && c->plan_bs == bs && c->plan.strategy == c->strategy)
        return;
    make_plan(c->tree, c->strategy, bs, c->plan);
    c->plan_valid = true;
    c->plan_version = c->tree.version;
    c->plan_bs = bs;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

extern "C" {

const char* ta_last_error(void) { return g_err.c_str(); }
int ta_abi_version(void) { return TA_ABI_VERSION; }

ta_status ta_ctx_create(int device, const ta_shape* s, ta_ctx** out) {
    return guard([&] {
        if (!s || !out) fail(TA_ERR_INVALID_ARGUMENT, "ta_ctx_create: null argument");
        ta_shape sh = *s;
        if (sh.page_tokens == 0) sh.page_tokens = 16;
        if (sh.n_local_kv_heads == 0) sh.n_local_kv_heads = sh.n_kv_heads - sh.kv_head_begin;
        if (sh.n_layers < 1 || sh.n_q_heads < 1 || sh.n_kv_heads < 1 || sh.d_head < 1 || sh.page_tokens < 1)
            fail(TA_ERR_INVALID_ARGUMENT, "ta_ctx_create: dimensions must be positive");
        if (sh.n_q_heads % sh.n_kv_heads != 0)
            fail(TA_ERR_INVALID_ARGUMENT, "ta_ctx_create: n_q_heads must be a multiple of n_kv_heads");
        if (sh.kv_head_begin < 0 || sh.n_local_kv_heads < 1 || sh.kv_head_begin + sh.n_local_kv_heads > sh.n_kv_heads)
            fail(TA_ERR_INVALID_ARGUMENT, "ta_ctx_create: bad kv head shard");
        if ((sh.kv_dtype != TA_F32 && sh.kv_dtype != TA_BF16) || (sh.out_dtype != TA_F32 && sh.out_dtype != TA_BF16))
            fail(TA_ERR_INVALID_ARGUMENT, "ta_ctx_create: dtype must be TA_F32 or TA_BF16");
        if (device >= 0 && sh.d_head != 8 && sh.d_head != 16 && sh.d_head != 32 && sh.d_head != 64 && sh.d_head != 128)
            fail(TA_ERR_INVALID_ARGUMENT, "ta_ctx_create: d_head must be 8, 16, 32, 64 or 128 on the device");
        auto c = std::make_unique<ta_ctx>();
        c->shape = sh;
        c->G = sh.n_q_heads / sh.n_kv_heads;
        c->hq_loc = sh.n_local_kv_heads * c->G;
        c->esize = sh.kv_dtype == TA_BF16 ? 2 : 4;
        c->out_esize = sh.out_dtype == TA_BF16 ? 2 : 4;
        c->pool.page_size = sh.page_tokens;
        c->tree.hook = &c->pool;
        if (device >= 0) {
            int n = 0;
            if (cudaGetDeviceCount(&n) != cudaSuccess || device >= n)
                fail(TA_ERR_NO_DEVICE, "ta_ctx_create: CUDA device " + std::to_string(device) + " not available");
            cuda_check(cudaSetDevice(device), "cudaSetDevice");
            c->device = device;
            if (sh.max_pages < 1) fail(TA_ERR_INVALID_ARGUMENT, "ta_ctx_create: max_pages must be >= 1");
            c->pool.capacity = sh.max_pages;
            c->head_stride = sh.max_pages * sh.page_tokens * (int64_t)sh.d_head;
            c->layer_elems = c->head_stride * sh.n_local_kv_heads;
            const size_t bytes = (size_t)c->layer_elems * sh.n_layers * c->esize;
            c->app_k.assign(sh.n_layers, nullptr);
            c->app_v.assign(sh.n_layers, nullptr);
            cuda_check(cudaMalloc(&c->kv_k, bytes), "cudaMalloc(K pool)");
            cuda_check(cudaMalloc(&c->kv_v, bytes), "cudaMalloc(V pool)");
            // Zeroed once: the tcgen05 kernel loads whole 16-row boxes, so the
            // unwritten tail rows of a node's last page are read too.  Their P is
            // exactly 0, but 0 * NaN would poison O if reused memory held NaNs.
            cuda_check(cudaMemset(c->kv_k, 0, bytes), "cudaMemset(K pool)");
            cuda_check(cudaMemset(c->kv_v, 0, bytes), "cudaMemset(V pool)");
            for (cudaEvent_t& e : c->meta_done)
                cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            cudaDeviceProp prop;
            cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
            c->num_sms = prop.multiProcessorCount;
            c->opt.num_ctas = prop.multiProcessorCount;
            if (mma_supported(sh.d_head, sh.kv_dtype == TA_BF16)) {
                const int64_t rows = (int64_t)sh.n_layers * sh.n_local_kv_heads * sh.max_pages * sh.page_tokens;
                c->tmaps_ok = true;
                for (int i = 0; i < 4; ++i)
                    c->tmaps_ok = c->tmaps_ok && make_pool_tmap(c->tmap_k + 128 * i, c->kv_k, rows, sh.d_head, 16 << i) &&
                                  make_pool_tmap(c->tmap_v + 128 * i, c->kv_v, rows, sh.d_head, 16 << i);
                if (!c->tmaps_ok) fail(TA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the KV pools");
            }
        }
        c->opt.use_mma = mma_supported(sh.d_head, sh.kv_dtype == TA_BF16);
        *out = c.release();
    });
}

ta_status ta_ctx_destroy(ta_ctx* c) {
    delete c;
    return TA_OK;
}

ta_status ta_set_option(ta_ctx* c, const char* key, int64_t v) {
    return guard([&] {
        const std::string k = key ? key : "";
        if (k == "fma_max_rows") {
            if (v < 1 || v > 16) fail(TA_ERR_INVALID_ARGUMENT, "fma_max_rows must be in [1, 16]");
            c->opt.fma_max_rows = (int)v;
        } else if (k == "use_mma") {
            c->opt.use_mma = v != 0 && mma_supported(c->shape.d_head, c->shape.kv_dtype == TA_BF16);
        } else if (k == "mma_max_rows") {
            if (v < 1 || v > 128) fail(TA_ERR_INVALID_ARGUMENT, "mma_max_rows must be in [1, 128]");
            c->opt.max_rows = (int)v;
        } else if (k == "tile_groups") {
            if (v < 1 || v > 8) fail(TA_ERR_INVALID_ARGUMENT, "tile_groups must be in [1, 8]");
            c->opt.tile_groups = (int)v;
        } else if (k == "tile_cost") {
            if (v < 0) fail(TA_ERR_INVALID_ARGUMENT, "tile_cost must be >= 0");
            c->opt.tile_cost = (int)v;
        } else if (k == "box_cost") {
            if (v < 0) fail(TA_ERR_INVALID_ARGUMENT, "box_cost must be >= 0");
            c->opt.box_cost = (int)v;
        } else if (k == "row_cost") {
            if (v < 0) fail(TA_ERR_INVALID_ARGUMENT, "row_cost must be >= 0");
            c->opt.row_cost = (int)v;
        } else if (k == "item_cost") {
            if (v < 0) fail(TA_ERR_INVALID_ARGUMENT, "item_cost must be >= 0");
            c->opt.item_cost = (int)v;
        } else if (k == "item_cost_many") {
            if (v < 0) fail(TA_ERR_INVALID_ARGUMENT, "item_cost_many must be >= 0");
            c->opt.item_cost_many = (int)v;
        } else if (k == "minmax") {
            c->opt.minmax = v != 0;
        } else if (k == "many_items") {
            if (v < 1) fail(TA_ERR_INVALID_ARGUMENT, "many_items must be >= 1");
            c->opt.many_items = (int)v;
        } else if (k == "num_ctas") {
            if (v < 1 || v > 65535) fail(TA_ERR_INVALID_ARGUMENT, "num_ctas must be in [1, 65535]");
            c->opt.num_ctas = (int)v;
        } else if (k == "final_direct") {
            c->opt.final_direct = v != 0;
        } else if (k == "pdl") {
            c->pdl = v != 0;
        } else if (k == "prefetch_tiles") {
            if (v < 0 || v > 32) fail(TA_ERR_INVALID_ARGUMENT, "prefetch_tiles must be in [0, 32]");
            c->prefetch_tiles = (int)v;
        } else if (k == "timeline_ptr") {
            c->timeline = v;
        } else if (k == "trace_ptr") {
            c->trace = v;
        } else if (k == "host_q_poll") {
            c->host_q_poll = v != 0;
        } else if (k == "fuse_append") {
            c->fuse_append = v != 0;
        } else if (k == "early_kv") {
            c->early_kv = v != 0;
        } else if (k == "fused_merge") {
            c->fused_merge = v != 0;
        } else if (k == "strategy") {
            if (v < TA_STRATEGY_Q_GUIDED || v > TA_STRATEGY_FLATTEN)
                fail(TA_ERR_INVALID_ARGUMENT, "strategy must be a TA_STRATEGY_* value");
            c->strategy = (int)v;
            c->plan_valid = false;
        } else {
            fail(TA_ERR_INVALID_ARGUMENT, "unknown option " + k);
        }
        // launch-only knobs keep the prepared schedule
        if (k != "trace_ptr" && k != "timeline_ptr" && k != "pdl" && k != "prefetch_tiles" && k != "early_kv" &&
            k != "host_q_poll")
            c->prepared = false;
    });
}

// --------------------------------------------------------------------- tree
ta_status ta_tree_new(ta_ctx* c, int64_t root_tokens, int32_t* root) {
    return guard([&] {
        if (root_tokens < 1) fail(TA_ERR_INVALID_ARGUMENT, "new_tree: root_token_count must be >= 1");
        c->pool.reset();
        c->pending_rows.clear();
        c->tree.create(root_tokens);
        if (root) *root = c->tree.root;
    });
}

ta_status ta_tree_restore(ta_ctx* c, int32_t root, int n, const int32_t* ids, const int32_t* parents,
                          const int64_t* counts) {
    return guard([&] {
        // validate on a scratch tree first so a bad snapshot leaves ctx intact
        Tree probe;
        probe.restore(root, n, ids, parents, counts);
        // ... and check the page demand before the pool is reset
        if (c->pool.capacity >= 0) {
            int64_t need = 0;
            for (int i = 0; i < n; ++i) need += (counts[i] + c->pool.page_size - 1) / c->pool.page_size;
            if (need > c->pool.capacity)
                fail(TA_ERR_OUT_OF_MEMORY, "restore: snapshot needs " + std::to_string(need) + " pages, capacity is " +
                                               std::to_string(c->pool.capacity));
        }
        c->pool.reset();
        c->pending_rows.clear();
        c->tree.restore(root, n, ids, parents, counts);
    });
}

ta_status ta_tree_branch(ta_ctx* c, int32_t at, int n, const int64_t* counts, int32_t* created) {
    return guard([&] {
        auto ids = c->tree.branch(at, counts, n);
        if (created) std::memcpy(created, ids.data(), ids.size() * sizeof(int32_t));
    });
}

ta_status ta_tree_prune(ta_ctx* c, int32_t at) {
    return guard([&] { c->tree.prune(at); });
}

// the new tokens' pool rows, queued for the next ta_prepare (ta_kv_append)
static void queue_rows(ta_ctx* c, int32_t leaf, int64_t t0, int64_t n) {
    const auto& h = c->pool.handle(leaf);
    const int P = c->pool.page_size;
    for (int64_t t = t0; t < t0 + n; ++t) c->pending_rows.push_back((int32_t)(h.pages[t / P] * P + t % P));
}

ta_status ta_tree_append(ta_ctx* c, int32_t leaf, int64_t n) {
    return guard([&] {
        const int64_t t0 = c->tree.contains(leaf) ? c->tree.count[leaf] : 0;
        c->tree.append(leaf, n);
        queue_rows(c, leaf, t0, n);
    });
}

ta_status ta_tree_append_leaves(ta_ctx* c, int n, const int32_t* leaves, const int64_t* counts) {
    return guard([&] {
        // the decode step of gen_few_shot (workloads.hpp:98-111): append_tokens
        // (tree.hpp:119-129) on many leaves at once.  Validated and checked
        // against the page capacity first, so it applies to all or none.
        std::vector<int32_t> ids;
        if (leaves) {
            ids.assign(leaves, leaves + n);
        } else {
            ids = c->tree.leaves;
            if (n >= 0 && n != (int)ids.size())
                fail(TA_ERR_INVALID_ARGUMENT, "append_leaves: n must equal the leaf count when leaves is NULL");
        }
        std::vector<uint8_t> seen(c->tree.alive.size(), 0);
        int64_t pages = 0;
        const int P = c->pool.page_size;
        for (size_t i = 0; i < ids.size(); ++i) {
            const int32_t id = ids[i];
            const int64_t k = counts ? counts[i] : 1;
            if (!c->tree.contains(id)) fail(TA_ERR_OUT_OF_RANGE, "append_tokens: unknown node id " + std::to_string(id));
            if (!c->tree.kids[id].empty()) fail(TA_ERR_INVALID_ARGUMENT, "append_tokens: target is not a leaf");
            if (k < 1) fail(TA_ERR_INVALID_ARGUMENT, "append_tokens: n must be >= 1");
            if (seen[id]++) fail(TA_ERR_INVALID_ARGUMENT, "append_leaves: leaf listed twice");
            const int64_t have = c->tree.count[id], room = (P - have % P) % P;
            if (k > room) pages += (k - room + P - 1) / P;
        }
        if (c->pool.capacity >= 0 &&
            pages > (int64_t)c->pool.free_list.size() + c->pool.capacity - (int64_t)c->pool.pages.size())
            fail(TA_ERR_OUT_OF_MEMORY, "append_leaves: device page capacity exhausted");
        const uint64_t v0 = c->tree.version;
        const bool chain = c->prepared && !c->fast_bad &&
                           (c->fast_log.empty() ? v0 == c->prepared_version : v0 == c->fast_log_version);
        for (size_t i = 0; i < ids.size(); ++i) {
            const int64_t k = counts ? counts[i] : 1, t0 = c->tree.count[ids[i]];
            c->tree.append(ids[i], k);
            queue_rows(c, ids[i], t0, k);
            if (chain)
                for (int64_t j = 0; j < k; ++j) c->fast_log.push_back({ids[i], t0 + j});
        }
        if (chain) c->fast_log_version = c->tree.version;
        else c->fast_bad = true;
    });
}

int64_t ta_graph_epoch(ta_ctx* c) { return c ? c->graph_epoch : -1; }

int64_t ta_fast_prepares(ta_ctx* c) { return c ? c->n_fast_prepares : -1; }

// ta_kv_append is fused into ta_attend: tcgen05 schedules with the fused merge
static bool fused_append(const ta_ctx* c) {
    return c->fuse_append && c->sched.fused_merge && (int)c->app_k.size() == c->shape.n_layers;
}

ta_status ta_kv_append(ta_ctx* c, int layer, const void* k, const void* v, void* stream) {
    return guard([&] {
        need_device(c);
        if (!c->prepared) fail(TA_ERR_LOGIC, "kv_append: call ta_prepare after appending tokens");
        if (layer < 0 || layer >= c->shape.n_layers) fail(TA_ERR_INVALID_ARGUMENT, "kv_append: layer out of range");
        if (!k || !v) fail(TA_ERR_INVALID_ARGUMENT, "kv_append: null key/value");
        if (((uintptr_t)k | (uintptr_t)v) & 15) fail(TA_ERR_INVALID_ARGUMENT, "kv_append: rows must be 16-byte aligned");
        if (fused_append(c)) {
            // written by the layer's next ta_attend, each row by the CTA that
            // loads it, right before its tile: no launch of its own
            c->app_k[layer] = k;
            c->app_v[layer] = v;
            return;
        }
        cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
        char* dk = (char*)c->kv_k + (size_t)layer * c->layer_elems * c->esize;
        char* dv = (char*)c->kv_v + (size_t)layer * c->layer_elems * c->esize;
        cuda_check(launch_kv_append(k, v, dk, dv, c->d_append_rows, c->d_counts, c->shape.n_local_kv_heads,
                                    c->head_stride, c->shape.d_head, c->esize, c->num_sms, (cudaStream_t)stream),
                   "kv_append");
    });
}

int64_t ta_kv_append_rows(ta_ctx* c) { return c && c->prepared ? c->n_append : 0; }

ta_status ta_tree_leaves(ta_ctx* c, int32_t* out, int cap, int* n) {
    return guard([&] {
        const int k = (int)c->tree.leaves.size();
        if (n) *n = k;
        if (out) std::memcpy(out, c->tree.leaves.data(), sizeof(int32_t) * std::min(k, cap));
    });
}

ta_status ta_tree_get_info(ta_ctx* c, ta_tree_info* o) {
    return guard([&] {
        if (c->tree.root < 0) fail(TA_ERR_LOGIC, "no tree");
        o->root = c->tree.root;
        o->node_count = c->tree.n_alive;
        o->n_leaves = (int32_t)c->tree.leaves.size();
        o->next_id = c->tree.next_id;
        o->total_tokens = c->tree.total_tokens();
        int64_t p = 0;
        for (int32_t l : c->tree.leaves) p += c->tree.path_tokens(l);
        o->path_tokens_sum = p;
    });
}

ta_status ta_tree_snapshot(ta_ctx* c, int32_t* ids, int32_t* parents, int64_t* counts, int cap, int* n) {
    return guard([&] {
        int k = 0;
        for (int32_t id = 0; id < (int32_t)c->tree.alive.size(); ++id) {
            if (!c->tree.alive[id]) continue;
            if (ids && k < cap) {
                ids[k] = id;
                parents[k] = c->tree.parent[id];
                counts[k] = c->tree.count[id];
            }
            ++k;
        }
        if (n) *n = k;
    });
}

// --------------------------------------------------------------------- pool
ta_status ta_pool_stats(ta_ctx* c, int64_t* page_count, int64_t* free_pages, int64_t* live_slots) {
    return guard([&] {
        if (page_count) *page_count = (int64_t)c->pool.pages.size();
        if (free_pages) *free_pages = (int64_t)c->pool.free_list.size();
        if (live_slots) *live_slots = c->pool.live_slots;
    });
}

ta_status ta_pool_token_ref(ta_ctx* c, int32_t node, int64_t token, int32_t* page, int32_t* slot) {
    return guard([&] {
        const auto& h = c->pool.handle(node);
        if (token < 0 || token >= h.n_tokens) fail(TA_ERR_INVALID_ARGUMENT, "token index out of range");
        const int P = c->pool.page_size;
        if (page) *page = h.pages[token / P];
        if (slot) *slot = (int32_t)(token % P);
    });
}

ta_status ta_kv_write(ta_ctx* c, int layer, int32_t node, int64_t t0, int64_t n, const void* k,
                      const void* v, int src_on_device, void* stream) {
    return guard([&] {
        need_device(c);
        if (layer < 0 || layer >= c->shape.n_layers) fail(TA_ERR_INVALID_ARGUMENT, "write_kv: layer out of range");
        const auto& h = c->pool.handle(node);
        if (t0 < 0 || n < 0 || t0 + n > h.n_tokens)
            fail(TA_ERR_INVALID_ARGUMENT, "write_kv: token index out of range");
        if (n == 0) return;
        if (!k || !v) fail(TA_ERR_INVALID_ARGUMENT, "write_kv: null key/value");
        if (src_on_device && (((uintptr_t)k | (uintptr_t)v) & 15))
            fail(TA_ERR_INVALID_ARGUMENT, "write_kv: device key/value rows must be 16-byte aligned");
        cudaStream_t s = (cudaStream_t)stream;
        cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
        const int P = c->pool.page_size;
        const int D = c->shape.d_head, nl = c->shape.n_local_kv_heads;
        const size_t row_bytes = (size_t)nl * D * c->esize;
        const size_t rows_bytes = align_up((size_t)n * 4, 256);
        const size_t data_bytes = src_on_device ? 0 : align_up((size_t)n * row_bytes, 256);
        grow_dev(&c->stage_dev, &c->stage_cap, rows_bytes + 2 * data_bytes);
        grow_host(&c->stage_host, &c->stage_host_cap, rows_bytes);
        int32_t* rows_h = (int32_t*)c->stage_host;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t tok = t0 + i;
            rows_h[i] = (int32_t)(h.pages[tok / P] * P + tok % P);
        }
        char* base = (char*)c->stage_dev;
        cuda_check(cudaMemcpyAsync(base, rows_h, n * 4, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(rows)");
        const void* sk = k;
        const void* sv = v;
        if (!src_on_device) {
            cuda_check(cudaMemcpyAsync(base + rows_bytes, k, n * row_bytes, cudaMemcpyHostToDevice, s), "H2D k");
            cuda_check(cudaMemcpyAsync(base + rows_bytes + data_bytes, v, n * row_bytes, cudaMemcpyHostToDevice, s),
                       "H2D v");
            sk = base + rows_bytes;
            sv = base + rows_bytes + data_bytes;
        }
        char* dk = (char*)c->kv_k + (size_t)layer * c->layer_elems * c->esize;
        char* dv = (char*)c->kv_v + (size_t)layer * c->layer_elems * c->esize;
        cuda_check(launch_kv_scatter(sk, sv, dk, dv, (const int32_t*)base, (int)n, nl, c->head_stride, D, c->esize, s),
                   "kv_scatter");
        // the pinned row list / device staging are reused by the next call
        cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    });
}

// --------------------------------------------------------------------- plan
ta_status ta_plan_flatten(ta_ctx* c, int bs, ta_plan_view* out) {
    return guard([&] {
        if (c->tree.root < 0) fail(TA_ERR_LOGIC, "no tree");
        ensure_plan(c, bs);
        const Plan& p = c->plan;
        out->block_size = p.block_size;
        out->n_groups = p.n_groups();
        out->seg_begin = p.seg_begin.data();
        out->q_begin = p.q_begin.data();
        out->seg_node = p.seg_node.data();
        out->seg_offset = p.seg_offset.data();
        out->seg_len = p.seg_len.data();
        out->seg_mask = p.seg_mask.data();
        out->queries = p.queries.data();
    });
}

ta_status ta_plan_json(ta_ctx* c, int bs, char* buf, size_t cap, size_t* len) {
    return guard([&] {
        if (c->tree.root < 0) fail(TA_ERR_LOGIC, "no tree");
        ensure_plan(c, bs);
        const std::string s = plan_json(c->tree, c->plan);
        if (len) *len = s.size();
        if (buf && cap) {
            const size_t k = std::min(cap - 1, s.size());
            std::memcpy(buf, s.data(), k);
            buf[k] = 0;
        }
    });
}

// ------------------------------------------------------------------ IO model
// io_measured / io_analytical (io_model.hpp:88-170) over the context's tree.
static void check_params(const ta_cost_params* p) {
    if (!p) fail(TA_ERR_INVALID_ARGUMENT, "CostParams: null");
    if (p->d_head <= 0 || p->n_heads <= 0 || p->n_layers <= 0)
        fail(TA_ERR_INVALID_ARGUMENT, "CostParams: dimensions must be positive");
    if (p->dtype_bytes != 2 && p->dtype_bytes != 4 && p->dtype_bytes != 8)
        fail(TA_ERR_INVALID_ARGUMENT, "CostParams: dtype_bytes must be 2, 4 or 8");
}

ta_status ta_io_measured(ta_ctx* c, int bs, const ta_cost_params* p, ta_io_report* out) {
    return guard([&] {
        if (c->tree.root < 0) fail(TA_ERR_LOGIC, "no tree");
        check_params(p);
        ensure_plan(c, bs);
        const Plan& P = c->plan;
        const uint64_t u = (uint64_t)p->n_heads * p->n_layers * p->dtype_bytes, d = (uint64_t)p->d_head;
        ta_io_report r{};
        for (int g = 0; g < P.n_groups(); ++g) {
            uint64_t kv_len = 0;   // QkvGroup::kv_length: sum of its segment lengths
            for (int k = P.seg_begin[g]; k < P.seg_begin[g + 1]; ++k) kv_len += (uint64_t)P.seg_len[k];
            r.kv_bytes += 2 * d * kv_len * u;
            r.q_bytes += (uint64_t)(P.q_begin[g + 1] - P.q_begin[g]) * d * u;
            r.mask_bytes += (uint64_t)(P.seg_begin[g + 1] - P.seg_begin[g]) * 8 * (uint64_t)p->n_layers;
        }
        *out = r;   // fused execution writes no partials
    });
}

ta_status ta_io_analytical(ta_ctx* c, int algo, const ta_cost_params* p, int bs, ta_io_report* out) {
    return guard([&] {
        if (c->tree.root < 0) fail(TA_ERR_LOGIC, "no tree");
        check_params(p);
        const Tree& t = c->tree;
        const uint64_t u = (uint64_t)p->n_heads * p->n_layers * p->dtype_bytes, d = (uint64_t)p->d_head;
        uint64_t n_tree = 0, live = 0, chunked = 0, sum_paths = 0;
        for (int32_t id : t.dfs) {
            const uint64_t tc = (uint64_t)t.count[id];
            n_tree += tc;
            if (tc == 0) continue;
            live++;
            chunked += (tc + (uint64_t)bs - 1) / (uint64_t)bs;
        }
        for (int32_t l : t.leaves) sum_paths += (uint64_t)t.path_tokens(l);
        const uint64_t ln = t.leaves.size();
        uint64_t k = 1;
        ta_io_report r{};
        uint64_t qkt = 0, scaled = 0, mask_add = 0, softmax = 0, dense_mask = 0;
        switch (algo) {
            case TA_ALG_NAIVE:
                r.kv_bytes = 2 * d * sum_paths * u;
                qkt = scaled = softmax = 2 * sum_paths * u;
                break;
            case TA_ALG_FLASH_DECODING:
            case TA_ALG_RADIX:
                r.kv_bytes = 2 * d * sum_paths * u;
                break;
            case TA_ALG_TREE_ATTN_MEDUSA:
                r.kv_bytes = 2 * d * n_tree * u;
                qkt = scaled = mask_add = softmax = 2 * ln * n_tree * u;
                dense_mask = ln * n_tree * u;
                break;
            case TA_ALG_TREE_ATTN_SPECINFER:
                r.kv_bytes = 2 * d * n_tree * ln * u;
                r.mask_bytes = (ln * n_tree + 63) / 64 * u;
                break;
            case TA_ALG_NODE:
                r.kv_bytes = 2 * d * n_tree * u;
                k = live;
                break;
            case TA_ALG_NODE_CHUNK:
                r.kv_bytes = 2 * d * n_tree * u;
                k = chunked;
                break;
            case TA_ALG_FLATTEN:
                r.kv_bytes = 2 * d * n_tree * u;
                r.mask_bytes = n_tree * u;
                k = (n_tree + (uint64_t)bs - 1) / (uint64_t)bs;
                break;
            default:
                fail(TA_ERR_INVALID_ARGUMENT, "unknown algorithm " + std::to_string(algo));
        }
        r.partial_bytes = qkt + scaled + mask_add + softmax + dense_mask;
        r.q_bytes = k * ln * d * u;
        *out = r;
    });
}

// ---------------------------------------------------------------- attention
namespace {

// schedule options as the selected kernel needs them
SchedOptions effective_opts(const ta_ctx* c) {
    SchedOptions o = c->opt;
    o.use_mma = o.use_mma && mma_supported(c->shape.d_head, c->shape.kv_dtype == TA_BF16);
    if (!o.use_mma) o.tile_groups = fma_tile_groups(c->shape.d_head, c->esize);
    // The merge runs inside the tcgen05 launch when every CTA can be resident
    // at once (one CTA per SM): a record's last item then waits only for
    // items of earlier CTAs, which are running or done.
    o.fused_merge = o.use_mma && c->fused_merge && o.num_ctas <= c->num_sms;
    // the ablation strategies run every plan group as its own stripe
    o.fuse_chunks = c->strategy == TA_STRATEGY_FLATTEN;
    return o;
}

// Row capacity of the FMA kernel instantiation for a schedule whose widest
// lane has `rows` rows (a lane always holds whole GQA groups: rows <= max(G,
// fma_max_rows)).  ta_prepare rejects G > kFmaMaxRows on the FMA path.
constexpr int kFmaMaxRows = 16;
int fma_rows(int rows) { return rows <= 4 ? 4 : rows <= 8 ? 8 : 16; }

}  // namespace

// ---------------------------------------------------------------------------
// Schedule metadata upload.  Every part lives at a FIXED offset of one device
// blob with room to grow (x1.5 when exceeded); the per-step counts sit in a
// header at offset 0 that the kernels read on the device.  Kernel arguments
// therefore stay valid from one ta_prepare to the next, so a captured CUDA
// graph of the layer calls (and of ta_kv_append) replays correctly after
// every re-plan; only a capacity growth relocates buffers, which bumps
// ta_graph_epoch.  Pinned staging is double-buffered: ta_prepare for the next
// step never waits for the current step's upload.
enum {
    P_HDR, P_TILES, P_TMETA, P_GROW, P_GINFO, P_ITEMS, P_CTAB, P_SLEAF, P_SOUT, P_MREC, P_PMERGE, P_PUBB, P_PUB,
    P_EMPTY, P_OWNB, P_OWN, P_APPEND, P_HEADS, P_TAILS, P_APPC, P_APPL, NPART
};

static void upload_schedule(ta_ctx* c, cudaStream_t s) {
    const Schedule& S = c->sched;
    DevCounts hdr{};
    hdr.n_empty = (int32_t)(S.empty.size() / 2);
    hdr.n_merge = (int32_t)S.merge_rec.size();
    hdr.n_append = (int32_t)c->pending_rows.size();
    hdr.n_partials = S.n_partials;
    const std::pair<const void*, size_t> src[NPART] = {
        {&hdr, sizeof hdr},
        {S.tiles.data(), S.tiles.size() * sizeof(TileDesc)},
        {S.tile_meta.data(), S.tile_meta.size() * sizeof(TileMeta)},
        {S.grp_row.data(), S.grp_row.size() * 4},
        {S.grp_info.data(), S.grp_info.size() * 4},
        {S.items.data(), S.items.size() * sizeof(ItemDesc)},
        {S.cta_begin.data(), S.cta_begin.size() * 4},
        {S.slot_leaf.data(), S.slot_leaf.size() * 4},
        {S.slot_out.data(), S.slot_out.size() * 4},
        {S.merge_rec.data(), S.merge_rec.size() * 16},
        {S.part_merge.data(), S.part_merge.size() * 4},
        {S.cta_pub_begin.data(), S.cta_pub_begin.size() * 4},
        {S.cta_pub.data(), S.cta_pub.size() * 8},
        {S.empty.data(), S.empty.size() * 4},
        {S.cta_own_begin.data(), S.cta_own_begin.size() * 4},
        {S.cta_own.data(), S.cta_own.size() * 4},
        {c->pending_rows.data(), c->pending_rows.size() * 4},
        {S.cta_heads.data(), S.cta_heads.size()},
        {S.cta_tails.data(), S.cta_tails.size()},
        {S.app_cta.data(), S.app_cta.size() * 4},
        {S.app_list.data(), S.app_list.size() * 4},
    };
    static_assert(sizeof(src) / sizeof(src[0]) == NPART, "parts");
    // capacities (bytes): grow all exceeded parts by 1.5x, keep the rest
    bool relocate = c->meta_part_cap.size() != NPART;
    if (relocate) c->meta_part_cap.assign(NPART, 0);
    for (int i = 0; i < NPART; ++i)
        if (src[i].second > c->meta_part_cap[i]) relocate = true;
    const int G = c->G, D = c->shape.d_head;
    const size_t n_part = (size_t)std::max(1, S.n_partials), n_rec = std::max<size_t>(1, S.merge_rec.size());
    if (n_part > c->part_rec_cap || n_rec > c->merge_cnt_n) relocate = true;
    if (relocate) {
        // every relocation invalidates captured launches: make them rare
        cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        size_t off = 0;
        c->meta_part_off.assign(NPART, 0);
        for (int i = 0; i < NPART; ++i) {
            if (src[i].second > c->meta_part_cap[i])
                c->meta_part_cap[i] = std::max<size_t>(256, align_up(src[i].second * 3 / 2, 256));
            c->meta_part_off[i] = off;
            off += c->meta_part_cap[i];
        }
        c->meta_bytes_total = off;
        cudaFree(c->meta_dev);
        c->meta_dev = nullptr;
        cuda_check(cudaMalloc(&c->meta_dev, off), "cudaMalloc(schedule metadata)");
        for (int b = 0; b < 2; ++b) {
            cudaFreeHost(c->meta_host[b]);
            c->meta_host[b] = nullptr;
            cuda_check(cudaMallocHost(&c->meta_host[b], off), "cudaMallocHost(schedule staging)");
        }
        if (n_part > c->part_rec_cap) {
            c->part_rec_cap = std::max(n_part * 3 / 2, c->part_rec_cap);
            cudaFree(c->part);
            c->part = nullptr;
            cuda_check(cudaMalloc(&c->part, c->part_rec_cap * G * (D + 1) * sizeof(float)), "cudaMalloc(partials)");
        }
        if (n_rec > c->merge_cnt_n) {
            c->merge_cnt_n = std::max(n_rec * 3 / 2, c->merge_cnt_n);
            cudaFree(c->merge_cnt);
            c->merge_cnt = nullptr;
            cuda_check(cudaMalloc(&c->merge_cnt, c->merge_cnt_n * kCntStride * sizeof(unsigned)), "cudaMalloc(merge counters)");
            cuda_check(cudaMemsetAsync(c->merge_cnt, 0, c->merge_cnt_n * kCntStride * sizeof(unsigned), s), "cudaMemsetAsync");
        }
        ++c->graph_epoch;
    }
    const int b = c->meta_buf;
    c->meta_buf ^= 1;
    // the upload that last used this staging buffer (two prepares ago) is done
    cuda_check(cudaEventSynchronize(c->meta_done[b]), "cudaEventSynchronize");
    const auto u0 = std::chrono::steady_clock::now();
    char* h = (char*)c->meta_host[b];
    size_t extent = 0;
    for (int i = 0; i < NPART; ++i) {
        if (src[i].second) std::memcpy(h + c->meta_part_off[i], src[i].first, src[i].second);
        if (src[i].second) extent = c->meta_part_off[i] + src[i].second;
    }
    cuda_check(cudaMemcpyAsync(c->meta_dev, h, extent, cudaMemcpyHostToDevice, s), "metadata upload");
    cuda_check(cudaEventRecord(c->meta_done[b], s), "cudaEventRecord");
    c->t_upload_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - u0).count();
    char* d = (char*)c->meta_dev;
    auto at = [&](int i) { return (const void*)(d + c->meta_part_off[i]); };
    c->d_counts = (const DevCounts*)at(P_HDR);
    c->d_tiles = (const TileDesc*)at(P_TILES);
    c->d_tile_meta = (const TileMeta*)at(P_TMETA);
    c->d_grp_row = (const int32_t*)at(P_GROW);
    c->d_grp_info = (const uint32_t*)at(P_GINFO);
    c->d_items = (const ItemDesc*)at(P_ITEMS);
    c->d_cta_begin = (const int32_t*)at(P_CTAB);
    c->d_slot_leaf = (const int32_t*)at(P_SLEAF);
    c->d_slot_out = (const int32_t*)at(P_SOUT);
    c->d_merge_rec = (const int4*)at(P_MREC);
    c->d_part_merge = (const int32_t*)at(P_PMERGE);
    c->d_cta_pub_begin = (const int32_t*)at(P_PUBB);
    c->d_cta_pub = (const int2*)at(P_PUB);
    c->d_empty = (const int32_t*)at(P_EMPTY);
    c->d_cta_own_begin = (const int32_t*)at(P_OWNB);
    c->d_cta_own = (const int32_t*)at(P_OWN);
    c->d_append_rows = (const int32_t*)at(P_APPEND);
    c->d_cta_heads = (const uint8_t*)at(P_HEADS);
    c->d_cta_tails = (const uint8_t*)at(P_TAILS);
    c->d_app_cta = (const int32_t*)at(P_APPC);
    c->d_app_list = (const int32_t*)at(P_APPL);
    c->n_append = (int64_t)c->pending_rows.size();
    c->pending_rows.clear();
    // The fused-merge counters are self-resetting; zero them only after a
    // failed launch may have left them dirty (ta_ctx_reset_counters) or on
    // relocation above.
}

ta_status ta_prepare(ta_ctx* c, int bs, void* stream) {
    return guard([&] {
        need_device(c);
        if (c->tree.root < 0) fail(TA_ERR_LOGIC, "no tree");
        cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
        // one decode step = plan + schedule + metadata upload, reused by every layer
        const auto t0 = std::chrono::steady_clock::now();
        // nothing changed since the last prepare (same tree version, block size
        // and options; no appends logged): the device schedule stands
        if (c->prepared && c->prepared_version == c->tree.version && c->prepared_bs == bs && c->fast_log.empty() &&
            !c->early_kv && c->n_append == 0) {
            c->t_plan_ns = c->t_sched_ns = c->t_upload_ns = 0;
            ++c->n_noop_prepares;
            return;
        }
        // decode-step fast path: only ta_tree_append_leaves since the last
        // prepare, and every new token extends its leaf's tail group -> patch the
        // schedule in place (the flatten plan is rebuilt on demand only).  Off
        // with early_kv (its per-CTA early-tile counts depend on the new rows).
        if (c->prepared && !c->fast_bad && !c->fast_log.empty() && c->tree.version == c->fast_log_version &&
            c->prepared_bs == bs && c->strategy == TA_STRATEGY_FLATTEN && c->sched.fused_merge && !c->early_kv &&
            patch_schedule_appends(c->sched, c->pool, c->fast_log)) {
            if (c->fuse_append) {
                std::vector<int32_t> tg(c->fast_log.size());
                for (size_t i = 0; i < tg.size(); ++i) tg[i] = c->sched.tail_grp[c->fast_log[i].first];
                build_append_lists(c->sched, c->shape.n_local_kv_heads, c->pending_rows, tg);
            }
            const auto t2f = std::chrono::steady_clock::now();
            c->plan_valid = false;
            upload_schedule(c, (cudaStream_t)stream);
            c->t_plan_ns = 0;
            c->t_sched_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t2f - t0).count();
            c->prepared_version = c->tree.version;
            c->fast_log.clear();
            ++c->n_fast_prepares;
            return;
        }
        c->fast_log.clear();
        c->fast_bad = false;
        make_plan(c->tree, c->strategy, bs, c->plan);
        const auto t1 = std::chrono::steady_clock::now();
        c->plan_valid = true;
        c->plan_version = c->tree.version;
        c->plan_bs = bs;
        const SchedOptions o = effective_opts(c);
        // a lane holds whole GQA groups: the kernels' row capacity bounds G
        if (o.use_mma && c->G > 128)
            fail(TA_ERR_INVALID_ARGUMENT, "prepare: GQA group size " + std::to_string(c->G) +
                                              " exceeds the tensor-core kernel's 128 rows");
        if (!o.use_mma && c->G > kFmaMaxRows)
            fail(TA_ERR_INVALID_ARGUMENT, "prepare: GQA group size " + std::to_string(c->G) +
                                              " exceeds the FMA kernel's 16 rows (use bf16 KV with d_head 128)");
        build_schedule(c->tree, c->pool, c->plan, c->G, c->shape.n_local_kv_heads, o, c->sched);
        if (o.use_mma) {
            c->pending_sorted.assign(c->pending_rows.begin(), c->pending_rows.end());
            std::sort(c->pending_sorted.begin(), c->pending_sorted.end());
            build_cta_blobs(c->sched, c->pending_sorted);
            if (c->sched.fused_merge) build_tail_map(c->tree, c->pool, c->sched);
            if (c->sched.fused_merge && c->fuse_append)
                build_append_lists(c->sched, c->shape.n_local_kv_heads, c->pending_rows, {});
        }
        const auto t2 = std::chrono::steady_clock::now();
        upload_schedule(c, (cudaStream_t)stream);
        c->t_plan_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
        c->t_sched_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count();
        c->prepared = true;
        c->prepared_version = c->tree.version;
        c->prepared_bs = bs;
    });
}

static void attend_impl(ta_ctx* c, int layer, const void* q, void* out, float* lse, cudaStream_t s) {
    if (!c->prepared || c->prepared_version != c->tree.version)
        fail(TA_ERR_LOGIC, "ta_attend: tree changed since ta_prepare (call ta_prepare first)");
    if (layer < 0 || layer >= c->shape.n_layers) fail(TA_ERR_INVALID_ARGUMENT, "attend: layer out of range");
    const Schedule& S = c->sched;
    const int D = c->shape.d_head;
    AttnArgs a{};
    a.k = (const char*)c->kv_k + (size_t)layer * c->layer_elems * c->esize;
    a.v = (const char*)c->kv_v + (size_t)layer * c->layer_elems * c->esize;
    a.head_stride = c->head_stride;
    a.tmap_k = c->tmap_k;
    a.tmap_v = c->tmap_v;
    a.head_rows = c->shape.max_pages * c->shape.page_tokens;
    a.layer_row0 = (int64_t)layer * c->shape.n_local_kv_heads * a.head_rows;
    a.q = q;
    a.out = out;
    a.lse = lse;
    a.part_o = c->part;
    a.part_lse = c->part + c->part_rec_cap * c->G * D;
    a.counts = c->d_counts;
    a.tiles = c->d_tiles;
    a.tile_meta = c->d_tile_meta;
    a.grp_row = c->d_grp_row;
    a.grp_info = c->d_grp_info;
    a.items = c->d_items;
    a.cta_begin = c->d_cta_begin;
    a.slot_leaf = c->d_slot_leaf;
    a.slot_out = c->d_slot_out;
    a.merge_rec = c->d_merge_rec;
    a.part_merge = c->d_part_merge;
    a.merge_cnt = c->merge_cnt;
    a.fused_merge = S.fused_merge ? 1 : 0;
    a.cta_pub_begin = c->d_cta_pub_begin;
    a.cta_pub = c->d_cta_pub;
    a.cta_own_begin = c->d_cta_own_begin;
    a.cta_own = c->d_cta_own;
    a.empty = c->d_empty;
    a.cta_heads = c->d_cta_heads;
    a.cta_tails = c->d_cta_tails;
    a.n_ctas = (int)S.cta_begin.size() - 1;
    a.G = c->G;
    a.hq_loc = c->hq_loc;
    a.D = D;
    a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
    a.kv_bf16 = c->shape.kv_dtype == TA_BF16;
    a.out_bf16 = c->shape.out_dtype == TA_BF16;
    a.trace = reinterpret_cast<long long*>(c->trace);
    a.timeline = reinterpret_cast<unsigned long long*>(c->timeline);
    a.prefetch_tiles = c->prefetch_tiles;
    a.early_kv = c->early_kv ? 1 : 0;
    a.q_flag = c->q_flag;
    a.q_seq = c->q_seq;
    if (fused_append(c) && c->app_k[layer]) {
        a.app_k = c->app_k[layer];
        a.app_v = c->app_v[layer];
        a.app_cta = (const int4*)c->d_app_cta;
        a.app_list = (const int4*)c->d_app_list;
        c->app_k[layer] = c->app_v[layer] = nullptr;   // one append per step and layer
    }

    const SchedOptions o = effective_opts(c);
    // both kernels move q / out / lse rows in 16-byte units
    if (!q || !out) fail(TA_ERR_INVALID_ARGUMENT, "attend: null q or out");
    if (((uintptr_t)out | (uintptr_t)q) & 15) fail(TA_ERR_INVALID_ARGUMENT, "attend: q and out must be 16-byte aligned");
    cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
    if (o.use_mma)
        cuda_check(launch_attn_mma(a, c->pdl, s), "attn_mma");
    else
        cuda_check(launch_attn_fma(a, fma_rows(S.max_lane_rows), c->pdl, s), "attn_fma");
    // always launched on the merge-launch path, so a captured step stays
    // valid when a re-plan adds or removes merge records
    if (!S.fused_merge) cuda_check(launch_merge(a, c->num_sms, c->pdl, s), "merge");
}

ta_status ta_attend(ta_ctx* c, int layer, const void* q, void* out, float* lse, void* stream) {
    return guard([&] {
        need_device(c);
        attend_impl(c, layer, q, out, lse, (cudaStream_t)stream);
    });
}

ta_status ta_attend_host(ta_ctx* c, int layer, const void* q_host, void* out_host, void* stream) {
    return guard([&] {
        need_device(c);
        cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
        cudaStream_t s = (cudaStream_t)stream;
        const size_t L = c->tree.leaves.size();
        const size_t qb = L * c->hq_loc * c->shape.d_head * c->esize;
        const size_t ob = L * c->hq_loc * c->shape.d_head * c->out_esize;
        grow_dev(&c->io_dev, &c->io_cap, align_up(qb, 256) + ob);
        char* dq = (char*)c->io_dev;
        char* dout = dq + align_up(qb, 256);
        cuda_check(cudaMemcpyAsync(dq, q_host, qb, cudaMemcpyHostToDevice, s), "H2D q");
        attend_impl(c, layer, dq, dout, nullptr, s);
        cuda_check(cudaMemcpyAsync(out_host, dout, ob, cudaMemcpyDeviceToHost, s), "D2H out");
        cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    });
}

// cuStreamWriteValue32 (driver API, reached through the runtime's entry-point
// query so the library links only cudart); nullptr when unavailable
typedef int (*WriteValue32Fn)(void* stream, unsigned long long addr, unsigned value, unsigned flags);
static WriteValue32Fn write_value32() {
    static WriteValue32Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (WriteValue32Fn) nullptr;
        return (WriteValue32Fn)p;
    }();
    return fn;
}

ta_status ta_attend_host_async(ta_ctx* c, int layer, const void* q_host, void* out_host, void* stream) {
    return guard([&] {
        need_device(c);
        cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
        cudaStream_t s = (cudaStream_t)stream;
        if (!c->h2d_stream) {
            cuda_check(cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking), "cudaStreamCreate");
            cuda_check(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking), "cudaStreamCreate");
            for (auto& sl : c->io_slot) {
                cuda_check(cudaEventCreateWithFlags(&sl.h2d, cudaEventDisableTiming), "cudaEventCreate");
                cuda_check(cudaEventCreateWithFlags(&sl.kern, cudaEventDisableTiming), "cudaEventCreate");
                cuda_check(cudaEventCreateWithFlags(&sl.d2h, cudaEventDisableTiming), "cudaEventCreate");
            }
        }
        const size_t L = c->tree.leaves.size();
        const size_t qb = L * c->hq_loc * c->shape.d_head * c->esize;
        const size_t ob = L * c->hq_loc * c->shape.d_head * c->out_esize;
        const size_t need = align_up(qb, 256) + ob;
        auto& sl = c->io_slot[c->io_next];
        c->io_next = (c->io_next + 1) % ta_ctx::kIoSlots;
        if (need > sl.cap) {
            if (sl.used) cuda_check(cudaEventSynchronize(sl.d2h), "cudaEventSynchronize");
            cudaFree(sl.dev);
            sl.dev = nullptr;
            sl.cap = 0;
            cuda_check(cudaMalloc(&sl.dev, need), "cudaMalloc(io slot)");
            sl.cap = need;
        }
        char* dq = (char*)sl.dev;
        char* dout = dq + align_up(qb, 256);
        // the slot's previous use (its copy-out, hence its attention) is complete
        if (sl.used) cuda_check(cudaStreamWaitEvent(c->h2d_stream, sl.d2h, 0), "cudaStreamWaitEvent");
        cuda_check(cudaMemcpyAsync(dq, q_host, qb, cudaMemcpyHostToDevice, c->h2d_stream), "H2D q");
        const int si = (int)(&sl - c->io_slot);
        const bool poll = c->host_q_poll && effective_opts(c).use_mma && write_value32() != nullptr;
        if (poll) {
            // the kernel waits for q on the device: no cross-stream dependency
            // on the compute stream, so consecutive layers stay chained
            if (!c->io_flags) {
                cuda_check(cudaMalloc(&c->io_flags, 256), "cudaMalloc(io flags)");
                cuda_check(cudaMemset(c->io_flags, 0, 256), "cudaMemset(io flags)");
            }
            const unsigned seq = ++c->io_seq[si];
            if (write_value32()(c->h2d_stream, (unsigned long long)(uintptr_t)(c->io_flags + si), seq, 0) != 0)
                fail(TA_ERR_CUDA, "cuStreamWriteValue32 failed");
            c->q_flag = c->io_flags + si;
            c->q_seq = seq;
        } else {
            cuda_check(cudaEventRecord(sl.h2d, c->h2d_stream), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(s, sl.h2d, 0), "cudaStreamWaitEvent");
        }
        attend_impl(c, layer, dq, dout, nullptr, s);
        c->q_flag = nullptr;
        cuda_check(cudaEventRecord(sl.kern, s), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(c->d2h_stream, sl.kern, 0), "cudaStreamWaitEvent");
        cuda_check(cudaMemcpyAsync(out_host, dout, ob, cudaMemcpyDeviceToHost, c->d2h_stream), "D2H out");
        cuda_check(cudaEventRecord(sl.d2h, c->d2h_stream), "cudaEventRecord");
        sl.used = true;
    });
}

ta_status ta_attend_host_wait(ta_ctx* c) {
    return guard([&] {
        need_device(c);
        if (c->d2h_stream) cuda_check(cudaStreamSynchronize(c->d2h_stream), "cudaStreamSynchronize");
    });
}

ta_status ta_io_stats_get(ta_ctx* c, ta_io_stats* o) {
    return guard([&] {
        if (!c->prepared) fail(TA_ERR_LOGIC, "ta_io_stats: call ta_prepare first");
        const Schedule& S = c->sched;
        const int64_t D = c->shape.d_head, nl = c->shape.n_local_kv_heads;
        const int64_t L = (int64_t)c->tree.leaves.size();
        std::memset(o, 0, sizeof(*o));
        o->n_chunks = c->plan.n_chunks();
        o->n_groups = c->plan.n_groups();
        o->n_units = (int64_t)S.items.size();
        o->n_units_mma = effective_opts(c).use_mma ? (int64_t)S.items.size() : 0;
        o->n_partials = S.n_partials;
        o->kv_bytes = S.kv_tokens_unique * 2 * nl * D * c->esize;
        o->kv_bytes_loaded = S.kv_rows_loaded * 2 * D * c->esize;
        o->q_bytes = L * c->hq_loc * D * c->esize;
        o->out_bytes = L * c->hq_loc * D * c->out_esize;
        o->partial_bytes = (int64_t)S.n_partials * c->G * (D + 1) * 4 * 2;
        o->meta_bytes = (int64_t)(S.tiles.size() * (sizeof(TileDesc) + sizeof(TileMeta)) +
                                  S.items.size() * sizeof(ItemDesc)) +
                        (int64_t)(S.grp_row.size() + S.grp_info.size() + S.cta_begin.size() + S.slot_leaf.size() +
                                  S.slot_out.size() + 4 * S.merge_rec.size() + S.part_merge.size() + S.empty.size() +
                                  S.cta_pub_begin.size() + 2 * S.cta_pub.size() + S.cta_own_begin.size() +
                                  S.cta_own.size()) * 4;
        o->flops = S.masked_q_tokens * c->hq_loc * 4 * D;
        o->host_plan_ns = c->t_plan_ns;
        o->host_schedule_ns = c->t_sched_ns;
        o->host_upload_ns = c->t_upload_ns;
    });
}

ta_status ta_schedule_get(ta_ctx* c, int bs, ta_schedule_view* o) {
    return guard([&] {
        if (c->tree.root < 0) fail(TA_ERR_LOGIC, "no tree");
        ensure_plan(c, bs);
        Schedule& S = c->dbg_sched;
        build_schedule(c->tree, c->pool, c->plan, c->G, c->shape.n_local_kv_heads, effective_opts(c), S);
        std::memset(o, 0, sizeof(*o));
        o->n_ctas = (int32_t)S.cta_begin.size() - 1;
        o->cta_begin = S.cta_begin.data();
        o->n_items = (int32_t)S.items.size();
        o->items = reinterpret_cast<const int32_t*>(S.items.data());
        o->n_tiles = (int32_t)S.tiles.size();
        o->tiles = reinterpret_cast<const int32_t*>(S.tiles.data());
        o->n_grp = (int32_t)S.grp_row.size();
        o->grp_row = S.grp_row.data();
        o->grp_info = S.grp_info.data();
        o->n_slot_leaf = (int32_t)S.slot_leaf.size();
        o->slot_leaf = S.slot_leaf.data();
        o->n_slot_out = (int32_t)S.slot_out.size();
        o->slot_out = S.slot_out.data();
        o->n_partials = S.n_partials;
        o->part_merge = S.part_merge.data();
        o->n_merge = (int32_t)S.merge_leaf.size();
        o->merge_leaf = S.merge_leaf.data();
        o->merge_head = S.merge_head.data();
        o->merge_begin = S.merge_begin.data();
        o->merge_parts = S.merge_parts.data();
        o->n_empty = (int32_t)(S.empty.size() / 2);
        o->empty = S.empty.data();
        o->n_lanes = S.n_lanes;
        o->use_mma = effective_opts(c).use_mma ? 1 : 0;
        o->fused_merge = S.fused_merge ? 1 : 0;
        if (S.fused_merge) {
            o->cta_pub_begin = S.cta_pub_begin.data();
            o->cta_pub = reinterpret_cast<const int32_t*>(S.cta_pub.data());
            o->cta_own_begin = S.cta_own_begin.data();
            o->cta_own = S.cta_own.data();
        }
    });
}

ta_status ta_lse_merge(const float* part_o, const float* part_lse, int n_parts, int64_t rows, int d, void* out,
                       int out_bf16, float* lse_out, void* stream) {
    return guard([&] {
        if (!part_o || !part_lse || !out) fail(TA_ERR_INVALID_ARGUMENT, "lse_merge: null pointer");
        if (n_parts < 1 || n_parts > 32) fail(TA_ERR_INVALID_ARGUMENT, "lse_merge: n_parts must be in [1, 32]");
        if (rows < 0 || d < 1) fail(TA_ERR_INVALID_ARGUMENT, "lse_merge: bad rows / d");
        if (((uintptr_t)part_o | (uintptr_t)out) & 15) fail(TA_ERR_INVALID_ARGUMENT, "lse_merge: pointers must be 16-byte aligned");
        cuda_check(launch_lse_merge(part_o, part_lse, n_parts, rows, d, out, out_bf16, lse_out, (cudaStream_t)stream),
                   "lse_merge");
    });
}

int ta_launches_per_attend(ta_ctx* c) {
    if (!c || !c->prepared) return 0;
    return c->sched.fused_merge ? 1 : 2;
}

}  // extern "C"
