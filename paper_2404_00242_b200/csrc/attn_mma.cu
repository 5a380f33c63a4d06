// attn_mma.cu -- persistent tcgen05/TMEM chunk attention (bf16 KV, D = 128).
//
// One launch per layer, one CTA per SM.  A CTA walks its items (a run of
// tiles of one lane for one kv head, see ta_internal.h).  Rows of an item
// are (query slot, q head in the GQA group) pairs, <= 128 of them, one per
// TMEM lane.  Per tile (<= 8 groups of 16 pool rows = <= 128 tokens):
//   TMA (warp 0)    K/V boxes -> separate K and V rings (128B swizzle), 2
//                   stages each; runs ahead across items.  Two stages per SM
//                   already keep HBM saturated; a deeper ring only adds
//                   queueing latency (paid at every CTA's start and end)
//   QK  (warp 1)    S = Q K^T  (M=128, N=16*groups, K=128), Q from TMEM
//                   -> S buffer (t & 1) in TMEM
//   PV  (warp 2)    O += P V   (M=128, N=128, K=16*groups), P from TMEM
//   softmax (warps 3-10, thread = TMEM lane = row, two column halves)
//                   pass 1: tcgen05.ld S -> tree-masked row max; exchange
//                   with the other half; online softmax in base 2 with lazy
//                   O rescale; pass 2: tcgen05.ld S -> P = exp2 -> bf16 ->
//                   tcgen05.st into TMEM.  Warps none of whose rows attend
//                   the tile (sparse lanes) skip the exponentials.
// TMEM: S0 [0,128) S1 [128,256) O [256,384) Q0 [384,448) Q1 [448,512) (Q
// double-buffered by item parity; P aliased into the S buffer it came from).
// At an item's end the softmax warps write each attended row either as the
// final output (its leaf-head is covered by this item alone) or as an
// (O/l, log2 lse) partial record, by bulk async copies.
// Schedule staging: the CTA's per-CTA blob (ta_internal.h, namespace blob),
// a fixed head by one bulk copy, the tail behind it.
// Fused merge (no merge launch): at its end, once its copies have landed, a
// CTA publishes how many partials it wrote per merge record, then merges the
// records it owns (owners spread evenly by merge work; two rows per warp).
// Every CTA publishes before it waits and every CTA is resident (<= one per
// SM), so no wait can block a publication.  The FMA kernel's schedules use
// merge.cu as a second launch instead.
//
// Reference semantics: group_attention (attention.hpp:117-204) over every
// chunk a leaf attends; tree_reduce (attention.hpp:209-233) at the owner
// CTA's end (or in merge.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "ta_ptx.cuh"

namespace ta {
namespace {

using namespace dev;

constexpr int BM = 128;                                  // rows per item (TMEM lanes)
constexpr int DH = 128;                                  // head dim
#ifndef TA_NK
#define TA_NK 2
#endif
#ifndef TA_NV
#define TA_NV 2
#endif
#ifndef TA_NQ
#define TA_NQ 2   // threads per softmax row, each owning 128 / TA_NQ columns: 2 or 4
#endif
constexpr int NQ = TA_NQ;                                // threads per row (column splits)
constexpr int CPT = 128 / NQ;                            // S / O / Q columns per softmax thread
constexpr int GPT = 8 / NQ;                              // 16-column S groups per softmax thread
constexpr int NTHREADS = 96 + 128 * NQ;                  // 3 issuer warps + 4 * NQ softmax warps
constexpr int NSOFT = 128 * NQ;                          // softmax threads
static_assert(NQ == 1 || NQ == 2 || NQ == 4, "column splits");
constexpr int NK = TA_NK;                                // K ring depth (a K tile is released by its QK)
constexpr int NV = TA_NV;                                // V ring depth (a V tile waits for the softmax and PV)
constexpr int HALF = BM * 128;                           // one 64-column half of a [128][128] bf16 tile
constexpr int TILE = 2 * HALF;                           // 32 KB
constexpr int SMEM_K = 0;                                // K stage s at s * TILE
constexpr int SMEM_V = NK * TILE;                        // V stage s at SMEM_V + s * TILE
constexpr int SMEM_BAR = SMEM_V + NV * TILE;
constexpr int SMEM_RED = SMEM_BAR + 256;                 // [2 parity][NQ split][128] fp32 row max
constexpr int SMEM_REDL = SMEM_RED + 2 * NQ * BM * 4;    // [NQ split][128] fp32 row sum
// the CTA's schedule (ta_internal.h, namespace blob): header + per-item tile /
// slot offsets, items, tile descriptors and metadata, slot leaves, and the
// fused merge's owned records and publications, staged by bulk copies
using blob::MAXI;
using blob::MAXT;
using blob::MAXS;
using blob::MAXO;
using blob::MAXP;
using blob::HI;
using blob::HT;
using blob::HS;
// epilogue staging: one row of O / l (this thread's CPT columns) per thread,
// written to global by bulk async copies
#ifndef TA_EPI_PASSES
#define TA_EPI_PASSES 1
#endif
constexpr int EPI_PASSES = TA_EPI_PASSES;                // fp32 rows staged in 1 or 2 column passes
constexpr int EPI_ROW = CPT * 4 / EPI_PASSES + 16;
constexpr int SMEM_EPI = SMEM_REDL + NQ * BM * 4;       // [softmax warps][32 rows][EPI_ROW]
constexpr int SMEM_HDR = SMEM_EPI + NSOFT * EPI_ROW;     // blob header + IOFF + SOFF (blob::H_ITEMS bytes)
constexpr int SMEM_ITEM = SMEM_HDR + blob::H_ITEMS;      // ItemDesc[MAXI]
constexpr int SMEM_TD = SMEM_ITEM + MAXI * 32;           // TileDesc[MAXT]
constexpr int SMEM_TM = SMEM_TD + MAXT * 16;             // TileMeta[MAXT]
constexpr int SMEM_SLOT = SMEM_TM + MAXT * 64;           // int[MAXS]
constexpr int SMEM_OWN = SMEM_SLOT + MAXS * 4;           // int4[MAXO]
constexpr int SMEM_OWNID = SMEM_OWN + MAXO * 16;         // int[MAXO]
constexpr int SMEM_PUB = SMEM_OWNID + MAXO * 4;          // int2[MAXP]: (record, partials written here)
constexpr int SMEM_BYTES = SMEM_PUB + MAXP * 8 + 1024;   // + alignment slack
static_assert(SMEM_HDR % 16 == 0 && SMEM_ITEM % 16 == 0 && SMEM_SLOT % 16 == 0 && SMEM_OWN % 16 == 0, "bulk copy alignment");
static_assert(SMEM_BYTES <= 232448, "shared memory budget");
constexpr int SOFT0 = 3;                                 // first softmax warp
constexpr int TRACE_TID = SOFT0 * 32;                    // thread that records the softmax trace
constexpr int TMEM_COLS = 512;
constexpr int TMEM_S = 0, TMEM_O = 256, TMEM_Q = 384;   // S0, S1 (P aliased), O, Q0, Q1 (item parity)
constexpr float kLazy = 8.0f;                            // rescale O only when the max grows by > 2^8
// A/B ablations and the light CTA-phase trace (scripts/build_variant.sh,
// scripts/light_spans.py); never defined in the product build
#ifndef TA_ABL_NOMMA
#define TA_ABL_NOMMA 0    // issuers commit without issuing MMAs (timing only, with TA_ABL_STREAM)
#endif
#ifndef TA_ABL_STREAM
#define TA_ABL_STREAM 0   // softmax warps release each tile without reading S (timing only)
#endif
#ifndef TA_ABL_NOEPI
#define TA_ABL_NOEPI 0    // no epilogue stores (timing only)
#endif
#ifndef TA_LIGHT_TRACE
#define TA_LIGHT_TRACE 0  // product kernel records CTA entry / items done / exit (globaltimer) into AttnArgs::trace
#endif
#define TA_LIGHT(slot, dep)                                                                        \
    do {                                                                                           \
        if constexpr (TA_LIGHT_TRACE && !TRACE) {                                                  \
            if (a.trace) {                                                                         \
                unsigned long long t_;                                                             \
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_) : "r"((unsigned)(dep)) : "memory"); \
                a.trace[blockIdx.x * TRACE_SLOTS + (slot)] = (long long)t_;                        \
            }                                                                                      \
        }                                                                                          \
    } while (0)
#ifndef TA_ABL_NOMERGE
#define TA_ABL_NOMERGE 0  // publish but do not wait / merge (timing only)
#endif
#ifndef TA_ABL_NOPUB
#define TA_ABL_NOPUB 0    // no fused merge (timing only)
#endif

// Per-tile barriers are double-buffered by tile parity (S_FULL, S_FREE,
// P_FULL, O_FULL): the softmax warps may run one tile ahead of the PV
// issuer, and a waiter must never be two phases behind its barrier.
enum { FULLK = 0, FULLV = NK, EMPTYK = NK + NV, EMPTYV = 2 * NK + NV, S_FULL = 2 * (NK + NV), S_FREE = S_FULL + 2,
       P_FULL = S_FULL + 4, O_FULL = S_FULL + 6, Q_FULL = S_FULL + 8, Q_FREE = S_FULL + 10, META_HEAD = S_FULL + 12,
       META_TAIL = S_FULL + 13, APPEND = S_FULL + 14, NBAR = S_FULL + 15 };
constexpr int TMEM_SLOT = 240;                           // offset of the TMEM address in the barrier block
static_assert(NBAR * 8 <= TMEM_SLOT, "barriers overlap the TMEM slot");

// Optional pipeline trace (a separate TRACE=true instantiation, launched only
// when AttnArgs::trace or ::timeline is set): per CTA 256
// int64 slots: [0] start / [1] end (%globaltimer ns), [2] SM id, [3] tiles, [4] / [5] clock64 at start / end,
// then per tile t < 27 (clock64, 8 slots): [8+8t] K loads issued, [+1] S
// seen by softmax, [+2] S loaded + masked, [+3] row max exchanged, [+4]
// O_FULL(t-1) seen, [+5] O rescaled, [+6] P published, [+7] item epilogue
// done (last tile of an item only).
constexpr int TRACE_SLOTS = 256, TRACE_TILES = 20;   // tiles: slots 8..167 (168.. phase marks)
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t;
}
// epilogue phases ([0] O_FULL seen, [1] fenced, [4] l exchanged, [3] stores begin, [2]
// stores done): slots 240.. for the CTA's first item, 248.. for its last; slot
// 224 + w: softmax warp w's last epilogue end; 232 + c: O columns c loaded
#define TA_TRACE_EPI(a, item, k)                                                                   \
    do {                                                                                           \
        if constexpr (TRACE) {                                                                     \
            if ((a).trace && threadIdx.x == TRACE_TID) {                                           \
                if ((item) == 0) (a).trace[blockIdx.x * TRACE_SLOTS + 240 + (k)] = clock64();      \
                (a).trace[blockIdx.x * TRACE_SLOTS + 248 + (k)] = clock64();                       \
            }                                                                                      \
        }                                                                                          \
    } while (0)
// phase marks at slots 180..191 (debug): clock64 (cheap; a %globaltimer read
// costs ~1 us and would distort the phases), max over the CTA's writers.  The
// asm takes `dep` as an input so it cannot issue before that value exists (a
// timer read right after a barrier is otherwise not ordered by it).  Slots
// 192..195: globaltimer / clock64 at entry and at the end, to place each
// CTA's clocks on the global timeline.
#define TA_MARK(a, k, dep)                                                                          \
    do {                                                                                           \
        if constexpr (TRACE) {                                                                     \
            if ((a).trace) {                                                                       \
                unsigned long long _t;                                                             \
                asm volatile("mov.u64 %0, %%clock64;" : "=l"(_t) : "r"((unsigned)(dep)) : "memory"); \
                atomicMax(reinterpret_cast<unsigned long long*>((a).trace) + blockIdx.x * TRACE_SLOTS + (k), _t); \
            }                                                                                      \
        }                                                                                          \
    } while (0)
// per-item marks of the first 3 items (slots 198 + 8 * item + j): 0 QK
// issuer past Q_FULL, 1 first QK committed, 2 epilogue saw O_FULL, 3 staging
// free, 4 copies issued, 5 first PV committed, 6 softmax item setup done,
// 7 softmax at the first tile's S wait
#define TA_TRACE_ITEM(a, item, j)                                                                  \
    do {                                                                                           \
        if constexpr (TRACE) {                                                                     \
            if ((a).trace && (item) < 3) (a).trace[blockIdx.x * TRACE_SLOTS + 198 + 8 * (item) + (j)] = clock64(); \
        }                                                                                          \
    } while (0)
#define TA_TRACE(a, t, k)                                                                          \
    do {                                                                                           \
        if constexpr (TRACE) {                                                                     \
            if ((a).trace && (t) < TRACE_TILES) (a).trace[blockIdx.x * TRACE_SLOTS + 8 + 8 * (t) + (k)] = clock64(); \
        }                                                                                          \
    } while (0)

// ---- fused merge: the owner's wait for the published partial counts.  One
// counter per 128-byte line: every waiting warp polls its line, and packed
// counters turned a few L2 lines into hot spots that slowed the publications
// themselves.
#ifndef TA_POLL_NS
#define TA_POLL_NS 256
#endif
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Spin until `target` pieces are in.  A schedule bug must fail loudly, not
// hang the GPU: trap after ~4e9 SM clocks (2 s at the boost clock).  The
// timeout reads clock64 (cheap), never %globaltimer (slow to read: it
// stretched every poll to ~1 us).
__device__ __forceinline__ void wait_pieces(const unsigned* cnt, unsigned target) {
    if (ld_acquire(cnt) >= target) return;
    const long long t0 = clock64();
    while (ld_acquire(cnt) < target) {
        __nanosleep(TA_POLL_NS);
        if (clock64() - t0 > 4000000000LL) __trap();
    }
}

struct TmapSet {
    CUtensorMap k[4];   // boxes of 16, 32, 64, 128 pool rows x 64 columns
    CUtensorMap v[4];
};

template <bool TRACE>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_mma_kernel(const __grid_constant__ TmapSet tm, const AttnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + SMEM_BAR;
    auto BAR = [&](int i) { return bar0 + 8u * (uint32_t)i; };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SMEM_BAR + TMEM_SLOT);
    float* red = reinterpret_cast<float*>(smem + SMEM_RED);
    float* redl = reinterpret_cast<float*>(smem + SMEM_REDL);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (TRACE && threadIdx.x == 0 && a.timeline) {   // debug: CTA entry (first / last over the grid)
        timeline_mark(a.timeline, 4, true);
        timeline_mark(a.timeline, 4, false);
    }
    if (TRACE && a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * TRACE_SLOTS + 192] = gtimer();
        a.trace[blockIdx.x * TRACE_SLOTS + 193] = clock64();
    }
    if (threadIdx.x == 0) TA_MARK(a, 180, blockIdx.x);
    if (TA_LIGHT_TRACE && !TRACE && a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * TRACE_SLOTS] = gtimer();
        unsigned smid_;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));
        a.trace[blockIdx.x * TRACE_SLOTS + 41] = smid_;
    }
    ItemDesc* s_item = reinterpret_cast<ItemDesc*>(smem + SMEM_ITEM);
    TileDesc* s_td = reinterpret_cast<TileDesc*>(smem + SMEM_TD);
    TileMeta* s_tm = reinterpret_cast<TileMeta*>(smem + SMEM_TM);
    int* s_slot = reinterpret_cast<int*>(smem + SMEM_SLOT);
    int4* s_own = reinterpret_cast<int4*>(smem + SMEM_OWN);
    int* s_own_id = reinterpret_cast<int*>(smem + SMEM_OWNID);
    int2* s_pub = reinterpret_cast<int2*>(smem + SMEM_PUB);
    const int32_t* s_hdr = reinterpret_cast<const int32_t*>(smem + SMEM_HDR);
    const int* s_ioff = reinterpret_cast<const int*>(smem + SMEM_HDR + blob::IOFF);
    const int* s_soff = reinterpret_cast<const int*>(smem + SMEM_HDR + blob::SOFF);

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * (NK + NV); ++i) mbar_init(BAR(FULLK + i), 1);   // FULLK, FULLV, EMPTYK, EMPTYV
        for (int i = 0; i < 2; ++i) {
            mbar_init(BAR(S_FULL + i), 1);
            mbar_init(BAR(S_FREE + i), 1);
            mbar_init(BAR(P_FULL + i), NSOFT);
            mbar_init(BAR(O_FULL + i), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(BAR(Q_FULL + i), NSOFT);
            mbar_init(BAR(Q_FREE + i), 1);
        }
        mbar_init(BAR(META_HEAD), 1);
        mbar_init(BAR(META_TAIL), 1);
        mbar_init(BAR(APPEND), NSOFT);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
        // the schedule head: host-written before the launch, so read before the
        // dependency wait; one round trip brings what the first tiles need
        const uint8_t* hb = a.cta_heads + (size_t)blockIdx.x * blob::HEAD_BYTES;
        mbar_expect_tx(BAR(META_HEAD), blob::HEAD_BYTES);
        bulk_g2s(sbase + SMEM_HDR, hb, blob::H_ITEMS, BAR(META_HEAD));
        bulk_g2s(sbase + SMEM_ITEM, hb + blob::H_ITEMS, HI * 32, BAR(META_HEAD));
        bulk_g2s(sbase + SMEM_TD, hb + blob::H_TD, HT * 16, BAR(META_HEAD));
        bulk_g2s(sbase + SMEM_TM, hb + blob::H_TM, HT * 64, BAR(META_HEAD));
        bulk_g2s(sbase + SMEM_SLOT, hb + blob::H_SLOT, HS * 4, BAR(META_HEAD));
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp == 0 && lane == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            prefetch_tmap(&tm.k[i]);
            prefetch_tmap(&tm.v[i]);
        }
    }
    tc_fence_before();
    __syncthreads();   // barriers initialised, TMEM address written
    tc_fence_after();
    if (threadIdx.x == 0) TA_LIGHT(38, *tmem_slot);   // barriers initialised, TMEM allocated
    mbar_wait(BAR(META_HEAD), 0);
    if (threadIdx.x == 0) TA_LIGHT(39, s_hdr[0]);      // schedule head landed
    const int n_items = s_hdr[blob::N_ITEMS], it0 = s_hdr[blob::IT0];
    const int ni_s = min(n_items, MAXI);
    const int nt_s = s_hdr[blob::N_TILES];   // staged tiles: CTA tile index < nt_s
    const int ns_s = s_hdr[blob::N_SLOTS];   // staged slot leaves
    if (threadIdx.x == 0) {
        // the tail: everything past the head's items / tiles / slots, and the
        // fused merge's lists (needed from tile HT / item HI / slot HS on)
        const uint8_t* tb = a.cta_tails + s_hdr[blob::TAIL_OFF];
        const uint32_t dst[7] = {sbase + SMEM_ITEM + HI * 32, sbase + SMEM_TD + HT * 16, sbase + SMEM_TM + HT * 64,
                                 sbase + SMEM_SLOT + HS * 4,  sbase + SMEM_OWN,          sbase + SMEM_OWNID,
                                 sbase + SMEM_PUB};
        uint32_t tot = 0;
        for (int i = 0; i < 7; ++i) tot += (uint32_t)s_hdr[blob::T_ITEMS + i];
        mbar_expect_tx(BAR(META_TAIL), tot);
        uint32_t off = 0;
        for (int i = 0; i < 7; ++i) {
            const uint32_t n = (uint32_t)s_hdr[blob::T_ITEMS + i];
            if (n) bulk_g2s(dst[i], tb + off, n, BAR(META_TAIL));
            off += n;
        }
    }
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) TA_MARK(a, 181, tmem);
    if (TRACE && threadIdx.x == 0 && a.timeline) {   // debug: schedule staged
        timeline_mark(a.timeline, 6, true);
        timeline_mark(a.timeline, 6, false);
    }
    pdl_launch_dependents();
    // warm L2 with the first tiles' KV and the first item's query rows while
    // the previous launch drains (prefetches carry no ordering obligations).
    // Issued by the PV issuer's lanes, idle until the first P: from the
    // producer's thread they delayed its own first loads by ~1.5 µs.  Tiles
    // the producer loads before the wait (n_early) need none.
    if (warp == 2 && lane < a.prefetch_tiles && lane < min(nt_s, HT) && lane >= (a.early_kv ? s_hdr[blob::N_EARLY] : 0)) {
        int k = 0;
        while (s_ioff[k + 1] <= lane) ++k;
        if (k < HI) {   // else its item is in the tail
            const int64_t row0 = a.layer_row0 + (int64_t)s_item[k].head * a.head_rows;
            const TileDesc td = s_td[lane];
            uint64_t boxes;
            std::memcpy(&boxes, td.box, 8);
#pragma unroll 1
            for (int b = 0; b < td.nbox; ++b, boxes >>= 8) {
                const int g = (int)(boxes & 0xffu) >> 2, sz = (int)(boxes & 3u);
                const int row = (int)(row0 + s_tm[lane].row[g]);
                tma_prefetch_2d(&tm.k[sz], 0, row);
                tma_prefetch_2d(&tm.k[sz], 64, row);
                tma_prefetch_2d(&tm.v[sz], 0, row);
                tma_prefetch_2d(&tm.v[sz], 64, row);
            }
        }
    }
    if (warp >= SOFT0 && n_items > 0) {
        const int r = (warp & 3) * 32 + lane, h = (warp - SOFT0) >> 2;
        const ItemDesc I0 = s_item[0];
        if (r < I0.n_slots * a.G && r / a.G < ns_s) {
            const __nv_bfloat16* qp = reinterpret_cast<const __nv_bfloat16*>(a.q) +
                                      ((size_t)s_slot[r / a.G] * a.hq_loc + I0.head * a.G + r % a.G) * DH + CPT * h;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(qp));
        }
    }
    // previous launch finished: queries, outputs, partial scratch are ours.  The
    // producer waits inside its loop, after loading the leading tiles no
    // pending ta_kv_append row touches (KV is written only by ta_kv_write,
    // synchronous, or ta_kv_append, whose rows the host knows)
    const int n_early = a.early_kv ? s_hdr[blob::N_EARLY] : 0;
    if (!(warp == 0 && lane == 0)) pdl_wait();
    if (threadIdx.x == 32) TA_LIGHT(40, s_hdr[1]);   // after the dependency wait (warp 1)
    if (TRACE && threadIdx.x == 0) timeline_mark(a.timeline, 0, true);
    if (TRACE && a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * TRACE_SLOTS] = gtimer();
        a.trace[blockIdx.x * TRACE_SLOTS + 4] = clock64();
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[blockIdx.x * TRACE_SLOTS + 2] = smid;
    }
    // schedule accessors: k = CTA-local item index, lt = CTA-local tile index
    bool tail_in = false;   // this thread has seen the tail land
    auto need_tail = [&]() {
        if (!tail_in) {
            mbar_wait(BAR(META_TAIL), 0);
            tail_in = true;
        }
    };
    auto item_at = [&](int k) -> ItemDesc {
        if (k >= HI) need_tail();
        return k < MAXI ? s_item[k] : a.items[it0 + k];
    };
    auto td_at = [&](int lt, int t) -> TileDesc {
        if (lt >= HT) need_tail();
        return lt < nt_s ? s_td[lt] : a.tiles[t];
    };
    auto tm_at = [&](int lt, int t) -> const TileMeta* {
        if (lt >= HT) need_tail();
        return lt < nt_s ? &s_tm[lt] : &a.tile_meta[t];
    };
    auto leaf_at = [&](int k, const ItemDesc& I, int jj) -> int {   // leaf of slot jj of item k
        if (k < ni_s) {
            const int x = s_soff[k] + jj;
            if (x < ns_s) {
                if (x >= HS) need_tail();
                return s_slot[x];
            }
        }
        return a.slot_leaf[I.slot_begin + jj];
    };

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int gt = 0;
            // fused append: the first tile holding a row this launch writes
            const int app_gt = a.app_k ? a.app_cta[blockIdx.x].z : INT_MAX;
            for (int k = 0; k < n_items; ++k) {
                const ItemDesc I = item_at(k);
                const int64_t row0 = a.layer_row0 + (int64_t)I.head * a.head_rows;
                for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                    if (gt == n_early) pdl_wait();
                    if (gt == app_gt) mbar_wait(BAR(APPEND), 0);   // the softmax warps wrote the rows
                    const TileDesc td = td_at(gt, t);
                    const TileMeta* tmp = tm_at(gt, t);
                    const int s = gt % NK, sv = gt % NV;
                    const uint32_t ph = (uint32_t)(gt / NK) & 1u, phv = (uint32_t)(gt / NV) & 1u;
                    const uint32_t kdst = sbase + SMEM_K + (uint32_t)s * TILE;
                    const uint32_t vdst = sbase + SMEM_V + (uint32_t)sv * TILE;
                    const uint32_t bytes = (uint32_t)td.ng * 4096u;
                    mbar_wait(BAR(EMPTYK + s), ph ^ 1);
                    mbar_expect_tx(BAR(FULLK + s), bytes);
                    uint64_t boxes;   // the 8 box codes in a register (no local-memory indexing)
                    std::memcpy(&boxes, td.box, 8);
#pragma unroll 1   // rolled: unrolled TMA issue sequences bloated the kernel's code (I-cache)
                    for (int b = 0; b < td.nbox; ++b, boxes >>= 8) {
                        const int g = (int)(boxes & 0xffu) >> 2, sz = (int)(boxes & 3u);
                        const int row = (int)(row0 + tmp->row[g]);
                        tma_load_2d(kdst + g * 2048, &tm.k[sz], 0, row, BAR(FULLK + s));
                        tma_load_2d(kdst + HALF + g * 2048, &tm.k[sz], 64, row, BAR(FULLK + s));
                    }
                    TA_TRACE(a, gt, 0);
                    if (gt == 0) TA_MARK(a, 183, bytes);
                    if (gt == 0) TA_LIGHT(2, bytes);
                    mbar_wait(BAR(EMPTYV + sv), phv ^ 1);
                    TA_TRACE(a, gt, 4);
                    mbar_expect_tx(BAR(FULLV + sv), bytes);
                    std::memcpy(&boxes, td.box, 8);
#pragma unroll 1
                    for (int b = 0; b < td.nbox; ++b, boxes >>= 8) {
                        const int g = (int)(boxes & 0xffu) >> 2, sz = (int)(boxes & 3u);
                        const int row = (int)(row0 + tmp->row[g]);
                        tma_load_2d(vdst + g * 2048, &tm.v[sz], 0, row, BAR(FULLV + sv));
                        tma_load_2d(vdst + HALF + g * 2048, &tm.v[sz], 64, row, BAR(FULLV + sv));
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== QK issuer: S = Q K^T =====================
        if (lane == 0) {
            int gt = 0;
            for (int k = 0; k < n_items; ++k) {
                const ItemDesc I = item_at(k);
                const int qb = k & 1;   // Q buffer of this item
                mbar_wait(BAR(Q_FULL + qb), (k >> 1) & 1);
                TA_TRACE_ITEM(a, k, 0);
                for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                    const int ng = td_at(gt, t).ng;
                    const int s = gt % NK, sb = gt & 1;
                    mbar_wait(BAR(FULLK + s), (uint32_t)(gt / NK) & 1u);
                    if (gt >= 2) mbar_wait(BAR(S_FREE + sb), ((gt >> 1) - 1) & 1);
                    tc_fence_after();
                    const uint32_t sK = sbase + SMEM_K + (uint32_t)s * TILE;
                    const uint32_t id = idesc_bf16(BM, 16 * ng, 0, 0);
#pragma unroll
                    for (int kq = 0; kq < (TA_ABL_NOMMA ? 0 : DH / 16); ++kq) {
                        const uint32_t off = (uint32_t)((kq >> 2) * HALF + (kq & 3) * 32);
                        mma_bf16_ts(tmem + TMEM_S + sb * 128, tmem + TMEM_Q + 64 * qb + 8 * kq, sdesc(sK + off, 16, 1024), id,
                                    kq > 0);
                    }
                    mma_commit(BAR(S_FULL + sb));
                    if (t == I.tile_begin) TA_TRACE_ITEM(a, k, 1);
                    mma_commit(BAR(EMPTYK + s));
                }
                mma_commit(BAR(Q_FREE + qb));
            }
        }
    } else if (warp == 2) {
        // ===================== PV issuer: O += P V =====================
        if (lane == 0) {
            int gt = 0;
            for (int k = 0; k < n_items; ++k) {
                const ItemDesc I = item_at(k);
                for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                    const int ng = td_at(gt, t).ng;
                    const int s = gt % NV;
                    const int sb = gt & 1;
                    mbar_wait(BAR(FULLV + s), (uint32_t)(gt / NV) & 1u);
                    mbar_wait(BAR(P_FULL + sb), (gt >> 1) & 1);
                    tc_fence_after();
                    const uint32_t sV = sbase + SMEM_V + (uint32_t)s * TILE;
                    const uint32_t id = idesc_bf16(BM, DH, 0, 1);
                    const bool first = t == I.tile_begin;
                    // P of group kk: bf16 pairs in columns [16kk, 16kk+8) of S buffer sb
                    for (int kk = 0; kk < (TA_ABL_NOMMA ? 0 : ng); ++kk)
                        mma_bf16_ts(tmem + TMEM_O, tmem + TMEM_S + sb * 128 + 16 * kk, sdesc(sV + kk * 2048, HALF, 1024),
                                    id, (!first || kk > 0) ? 1u : 0u);
                    mma_commit(BAR(EMPTYV + s));
                    if (first) TA_TRACE_ITEM(a, k, 5);
                    mma_commit(BAR(S_FREE + sb));
                    mma_commit(BAR(O_FULL + sb));
                }
            }
        }
        // leaf-heads with no path tokens (their outputs are not read in this
        // launch): the idle lanes, after the PV issuer's loop
        __syncwarp();
        if (lane > 0) fill_empty(a, lane - 1, 31);
    } else {
        // ===================== softmax / epilogue (256 threads) =====================
        const int q4 = warp & 3;                 // TMEM lane quadrant of this warp (warps 3..10)
        const int h = (warp - SOFT0) >> 2;       // column split (S groups GPT*h.., O / Q columns CPT*h..)
        const int r = q4 * 32 + lane;            // row == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
        const int G = a.G;
        const float sc = a.scale_log2;

        // Q row of an item (this thread: dims [64h, 64h+64) of row r = 32
        // packed bf16 pairs) -> registers -> (once the previous item's QK is
        // complete) tcgen05.st into the Q columns
        constexpr int QV = CPT / 8;   // uint4 of this thread's Q dims
        auto q_row = [&](const ItemDesc& I, int leaf) -> const uint4* {
            return reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.q) +
                                                  ((size_t)leaf * a.hq_loc + I.head * G + r % G) * DH) + QV * h;
        };
        auto q_fetch = [&](const ItemDesc& I, int leaf, uint4 (&v)[QV]) {
            if (leaf >= 0) {
                const uint4* src = q_row(I, leaf);
#pragma unroll
                for (int c = 0; c < QV; ++c) v[c] = src[c];
            } else {
#pragma unroll
                for (int c = 0; c < QV; ++c) v[c] = make_uint4(0, 0, 0, 0);
            }
        };
        auto q_store = [&](const uint4 (&v)[QV], int qb) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
#pragma unroll
            for (int c = 0; c < QV / 4; ++c) TA_TMEM_ST16(tmem + lane_addr + TMEM_Q + 64 * qb + (CPT / 2) * h + 16 * c, (w + 16 * c));
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(BAR(Q_FULL + qb));
        };

        if (a.app_k) {
            // fused ta_kv_append: this CTA's share of the step's new K / V rows
            // into this layer's pools (a warp per row: lanes 0-15 K, 16-31 V),
            // visible to the TMA loads the producer issues after the barrier
            const int4 ce = a.app_cta[blockIdx.x];
            const int n_loc = a.hq_loc / G;
            for (int e = ce.x + (warp - SOFT0); e < ce.y; e += NSOFT / 32) {
                const int4 en = a.app_list[e];
                const bool is_v = lane >= 16;
                const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(is_v ? a.app_v : a.app_k) +
                                                                  ((size_t)en.x * n_loc + en.y) * DH);
                uint4* dst = reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(reinterpret_cast<const __nv_bfloat16*>(is_v ? a.v : a.k)) +
                                                      ((size_t)en.y * a.head_rows + en.z) * DH);
                dst[lane & 15] = src[lane & 15];
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
            mbar_arrive(BAR(APPEND));
        }
        if (a.q_flag) {
            // host-buffer attend: q's copy-in (another stream) has landed
            // (a lost copy must fail loudly, not hang the GPU: trap after ~4 s)
            const long long t0 = clock64();
            while ((int)(ld_acquire(a.q_flag) - a.q_seq) < 0) {
                __nanosleep(64);
                if (clock64() - t0 > 8000000000LL) __trap();
            }
        }
        if (n_items > 0) {
            const ItemDesc I0 = item_at(0);
            uint4 qv[QV];
            q_fetch(I0, r < I0.n_slots * G ? leaf_at(0, I0, r / G) : -1, qv);
            q_store(qv, 0);
        }
        int gt = 0;
        for (int k = 0; k < n_items; ++k) {
            const ItemDesc I = item_at(k);
            const int nrows = I.n_slots * G;
            const bool live_row = r < nrows;
            const int j = live_row ? r / G : 0;      // local query slot
            const int g_in = r % G;
            const bool warp_live = q4 * 32 < nrows;
            float m = -INFINITY, l = 0.f;
            // this row's output code; the next item's Q goes to the other Q
            // buffer during this item's first tile (L2-prefetched before it)
            const bool has_next = k + 1 < n_items;
            const int code = live_row ? a.slot_out[I.out_begin + j] : kSlotUnused;
            int nleaf = -1;
            if (has_next) {
                const ItemDesc In = item_at(k + 1);
                nleaf = r < In.n_slots * G ? leaf_at(k + 1, In, r / G) : -1;
                if (nleaf >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(q_row(In, nleaf)));
            }
            if (threadIdx.x == TRACE_TID) TA_TRACE_ITEM(a, k, 6);
            for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                const TileDesc td = td_at(gt, t);
                uint32_t info[GPT];
                if constexpr (GPT == 8) {
                    const uint4* inf = reinterpret_cast<const uint4*>(tm_at(gt, t)->info);
                    const uint4 i0 = inf[0], i1 = inf[1];
                    info[0] = i0.x; info[1] = i0.y; info[2] = i0.z; info[3] = i0.w;
                    info[4] = i1.x; info[5] = i1.y; info[6] = i1.z; info[7] = i1.w;
                } else if constexpr (GPT == 4) {
                    const uint4 inf = *reinterpret_cast<const uint4*>(tm_at(gt, t)->info + 4 * h);
                    info[0] = inf.x; info[1] = inf.y; info[2] = inf.z; info[3] = inf.w;
                } else {
                    const uint2 inf = *reinterpret_cast<const uint2*>(tm_at(gt, t)->info + 2 * h);
                    info[0] = inf.x; info[1] = inf.y;
                }
                const int ng = td.ng;
                const int g0 = GPT * h;
                // per group: number of leading columns this row attends (0: none)
                int lim[GPT];
                bool att = false;
#pragma unroll
                for (int g = 0; g < GPT; ++g) {
                    const int b = (int)((info[g] >> 8) & 0xfffu), e = (int)(info[g] >> 20);
                    lim[g] = (live_row && g0 + g < ng && j >= b && j < e) ? (int)(info[g] & 0xffu) : 0;
                    att |= lim[g] > 0;
                }
                const bool warp_att = __any_sync(0xffffffffu, att);
                const int sb = gt & 1;
                const uint32_t s_addr = tmem + lane_addr + TMEM_S + sb * 128;
                if (threadIdx.x == TRACE_TID && t == I.tile_begin) TA_TRACE_ITEM(a, k, 7);
                mbar_wait(BAR(S_FULL + sb), (gt >> 1) & 1);
                if (threadIdx.x == TRACE_TID) TA_TRACE(a, gt, 1);
                tc_fence_after();
                // S of my column split into registers (one pass), tree mask, row max
                uint32_t rv[GPT][16];
                float mx = -INFINITY;
                if (warp_att && !TA_ABL_STREAM) {
                    // groups past ng hold stale columns; lim == 0 masks them
#pragma unroll
                    for (int g = 0; g < GPT; ++g) TA_TMEM_LD16(s_addr + (g0 + g) * 16, rv[g]);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
#pragma unroll
                        for (int g = 0; g < GPT; ++g) {
                            rv[g][c] = c < lim[g] ? rv[g][c] : 0xff800000u;   // -inf
                            mx = fmaxf(mx, __uint_as_float(rv[g][c]));
                        }
                    }
                }
                if (threadIdx.x == TRACE_TID) TA_TRACE(a, gt, 2);
                // combine the column splits of the row (partner warps: same quadrant)
                float* rd = red + (gt & 1) * NQ * BM;
                rd[h * BM + r] = mx;
                if constexpr (NQ > 1) named_bar(1 + q4, 32 * NQ);
#pragma unroll
                for (int q = 1; q < NQ; ++q) mx = fmaxf(mx, rd[((h + q) % NQ) * BM + r]);
                mx *= sc;
                if (threadIdx.x == TRACE_TID) TA_TRACE(a, gt, 3);
                // lazy rescale: keep the stale max unless it grew by > kLazy (both
                // threads of a row decide alike).  The O correction is warp-collective
                // and the only reason to wait for PV(t-1) here.
                const bool grow = mx > m + kLazy;
                float f = 1.f;
                if (grow) {
                    if (m != -INFINITY) f = ex2(m - mx);
                    l *= f;
                    m = mx;
                }
                if (t > I.tile_begin && __any_sync(0xffffffffu, grow && f != 1.f)) {
                    mbar_wait(BAR(O_FULL + (sb ^ 1)), ((gt - 1) >> 1) & 1);   // PV(t-1) done
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < CPT / 16; ++c) {
                        uint32_t o[16];
                        TA_TMEM_LD16(tmem + lane_addr + TMEM_O + h * CPT + c * 16, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
                        TA_TMEM_ST16(tmem + lane_addr + TMEM_O + h * CPT + c * 16, o);
                    }
                }
                if (threadIdx.x == TRACE_TID) TA_TRACE(a, gt, 5);
                if (warp_att && !TA_ABL_STREAM) {
                    // P = exp2(s * scale - m) -> bf16 pairs -> S columns [16g, 16g+8); l += sum(P)
                    const float negm = m == -INFINITY ? 0.f : -m;
                    float la = 0.f;
                    // P past ng lands in S columns PV never reads
#pragma unroll
                    for (int g = 0; g < GPT; ++g) {
                        uint32_t pk[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const float p0 = ex2(fmaf(__uint_as_float(rv[g][2 * c]), sc, negm));
                            const float p1 = ex2(fmaf(__uint_as_float(rv[g][2 * c + 1]), sc, negm));
                            la += p0 + p1;
                            pk[c] = pack_bf16(p0, p1);
                        }
                        TA_TMEM_ST8(s_addr + 16 * (g0 + g), pk);
                    }
                    l += la;
                } else if (warp_live) {
                    // no row of this warp attends my half of the tile: P = 0
                    const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
                    for (int g = 0; g < GPT; ++g)
                        if (g0 + g < ng) TA_TMEM_ST8(s_addr + 16 * (g0 + g), z);
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(BAR(P_FULL + sb));
                if (threadIdx.x == TRACE_TID) TA_TRACE(a, gt, 6);
                if (threadIdx.x == TRACE_TID && gt == 0) TA_MARK(a, 184, __float_as_uint(l));
                if (threadIdx.x == TRACE_TID && gt == 0) TA_LIGHT(3, __float_as_uint(l));
                if (threadIdx.x == TRACE_TID && gt == 4) TA_LIGHT(7, __float_as_uint(l));
                if (threadIdx.x == TRACE_TID && gt + 1 == s_ioff[ni_s]) TA_LIGHT(4, __float_as_uint(l));
                if (threadIdx.x == TRACE_TID) TA_MARK(a, 185, __float_as_uint(l));
                if (has_next && t == I.tile_begin) {
                    // next item's Q -> the other Q buffer (free once item k-1's QK is done)
                    uint4 qv[QV];
                    q_fetch(item_at(k + 1), nleaf, qv);
                    if (k >= 1) mbar_wait(BAR(Q_FREE + ((k + 1) & 1)), ((k - 1) >> 1) & 1);
                    tc_fence_after();
                    q_store(qv, (k + 1) & 1);
                }
            }

            // ---- epilogue
            mbar_wait(BAR(O_FULL + ((gt - 1) & 1)), ((gt - 1) >> 1) & 1);   // PV(last) and all before it
            TA_TRACE_EPI(a, k, 0);
            if (threadIdx.x == TRACE_TID) TA_TRACE_ITEM(a, k, 2);
            tc_fence_after();
            TA_TRACE_EPI(a, k, 1);
            redl[h * BM + r] = l;
            if constexpr (NQ > 1) named_bar(1 + q4, 32 * NQ);
#pragma unroll
            for (int q = 1; q < NQ; ++q) l += redl[((h + q) % NQ) * BM + r];
            if (threadIdx.x == TRACE_TID) TA_MARK(a, 186, __float_as_uint(l));
            TA_TRACE_EPI(a, k, 4);
            const float inv = l > 0.f ? 1.f / l : 0.f;
            const float lse2 = m + log2f(l);
            if (code != kSlotUnused && h == 0) {
                if (code < 0) {
                    if (a.lse) a.lse[(size_t)(-1 - code) * a.hq_loc + I.head * G + g_in] = lse2 * kLn2;
                } else {
                    a.part_lse[(size_t)code * G + g_in] = lse2;
                }
            }
            if (warp_live && !TA_ABL_NOEPI) {
                // O / l -> this thread's staging row (its TMEM lane = output row,
                // its 64 columns), then one bulk async copy of the row to the
                // final output or the partial record: the stores drain in the
                // background instead of stalling the softmax warps behind the
                // saturated read stream.  Compact loops: this code runs once per
                // item, I-cache cold.
                {
                const uint32_t srow = sbase + SMEM_EPI + (uint32_t)(((warp - SOFT0) * 32 + lane) * EPI_ROW);
                const bool st_bf16 = code < 0 && a.out_bf16;
                // the row's previous bulk copy (an earlier item) has read the staging
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                TA_TRACE_EPI(a, k, 3);
                if (threadIdx.x == TRACE_TID) TA_TRACE_ITEM(a, k, 3);
                // fp32 rows go out in EPI_PASSES column passes through a staging
                // row of 256 / EPI_PASSES bytes (the SMEM it saves deepens the V ring)
                const int npass = st_bf16 ? 1 : EPI_PASSES;
                const int cpp = (CPT / 16) / npass;   // 16-column chunks per pass
                char* dst = nullptr;
                if (code != kSlotUnused)
                    dst = code >= 0 ? reinterpret_cast<char*>(a.part_o + ((size_t)code * G + g_in) * DH + CPT * h)
                                    : reinterpret_cast<char*>(a.out) +
                                          (((size_t)(-1 - code) * a.hq_loc + I.head * G + g_in) * DH + CPT * h) * (a.out_bf16 ? 2 : 4);
#pragma unroll 1
                for (int pass = 0; pass < npass; ++pass) {
                    if (pass > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll 1
                    for (int c = pass * cpp; c < (pass + 1) * cpp; ++c) {
                        uint32_t o[16];
                        TA_TMEM_LD16(tmem + lane_addr + TMEM_O + h * CPT + c * 16, o);
                        tmem_wait_ld();
                        float f[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(o[i]) * inv;
                        if (st_bf16) {
                            sts128(srow + (uint32_t)(c * 32), pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]),
                                   pack_bf16(f[6], f[7]));
                            sts128(srow + (uint32_t)(c * 32 + 16), pack_bf16(f[8], f[9]), pack_bf16(f[10], f[11]),
                                   pack_bf16(f[12], f[13]), pack_bf16(f[14], f[15]));
                        } else {
                            const uint32_t o16 = (uint32_t)((c - pass * cpp) * 64);
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                sts128(srow + o16 + 16 * q, __float_as_uint(f[4 * q]), __float_as_uint(f[4 * q + 1]),
                                       __float_as_uint(f[4 * q + 2]), __float_as_uint(f[4 * q + 3]));
                        }
                    }
                    if (dst) {
                        const uint32_t nb = st_bf16 ? (uint32_t)(CPT * 2) : (uint32_t)(CPT * 4) / npass;
                        fence_proxy_async();   // the staging writes -> visible to the bulk copy
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + pass * nb), "r"(srow),
                                     "r"(nb)
                                     : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        TA_MARK(a, 187, srow);
                        if (threadIdx.x == TRACE_TID && k + 1 == n_items) TA_LIGHT(5, srow);
                    }
                }
                }
            }
            TA_TRACE_EPI(a, k, 2);
            if (threadIdx.x == TRACE_TID) TA_TRACE_ITEM(a, k, 4);
            tc_fence_before();
            if (threadIdx.x == TRACE_TID) TA_TRACE(a, gt - 1, 7);
            if constexpr (TRACE) {
                if (a.trace && lane == 0) a.trace[blockIdx.x * TRACE_SLOTS + 224 + warp - SOFT0] = clock64();
            }
        }
    }

    // the epilogues' bulk copies are complete (writes performed) before exit
    // or, with the fused merge, before this CTA's partials are published
    if (warp >= SOFT0) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        if (a.fused_merge) asm volatile("fence.proxy.async.global;" ::: "memory");
        TA_MARK(a, 188, lane);
        if (threadIdx.x == TRACE_TID) TA_LIGHT(35, lane);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TA_MARK(a, 196, s_ioff[0]);
    if (threadIdx.x == 0) TA_LIGHT(36, s_ioff[0]);
    if (TA_LIGHT_TRACE && !TRACE && a.trace && threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_) : "r"(s_ioff[0]) : "memory");
        a.trace[blockIdx.x * TRACE_SLOTS + 6] = (long long)t_;
    }
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
    if (a.fused_merge && !TA_ABL_NOPUB) {
        need_tail();
        // read here, not kept live across the item loop (register pressure)
        const int n_own = s_hdr[blob::N_OWN], o0 = s_hdr[blob::O0];
        const int n_pub = s_hdr[blob::N_PUB], pb0 = s_hdr[blob::PB0];
        // 1. publish: per record this CTA wrote partials for, one release-add
        //    of their count
#ifndef TA_PUB
#define TA_PUB 0   // A/B: 0 fence.acq_rel + relaxed red, 1 red.release, 2 no ordering (timing only)
#endif
        if (TA_PUB == 0 && (int)threadIdx.x < n_pub) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if ((int)threadIdx.x < n_pub) TA_MARK(a, 197, n_pub);
        if (threadIdx.x == 0) TA_LIGHT(37, n_pub);
        for (int i = threadIdx.x; i < n_pub; i += NTHREADS) {
            const int2 pb = i < MAXP ? s_pub[i] : a.cta_pub[pb0 + i];
            if (TA_PUB == 1)
                asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.merge_cnt + (size_t)pb.x * kCntStride), "r"(pb.y) : "memory");
            else
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(a.merge_cnt + (size_t)pb.x * kCntStride), "r"(pb.y) : "memory");
        }
        if ((int)threadIdx.x < n_pub) TA_MARK(a, 189, n_pub);
        if (threadIdx.x == 0) TA_LIGHT(9, n_pub);
        // 2. merge the records this CTA owns: one warp per (record, q head),
        //    tree_reduce in item order, every partial's loads in flight at
        //    once (merge_record_row).  Every CTA has published before it waits
        //    here, so no wait can block a publication.
        const int G = a.G;
        // two rows per warp (half-warp merges): every owned row in one round
        const int hw = lane >> 4;
        for (int row0 = TA_ABL_NOMERGE ? n_own * G : 2 * warp; row0 < n_own * G; row0 += 2 * (NTHREADS / 32)) {
            const int row = row0 + hw;
            const bool active = row < n_own * G;
            const int k = active ? row / G : 0;
            const int id = k < MAXO ? s_own_id[k] : a.cta_own[o0 + k];
            const int4 rec = k < MAXO ? s_own[k] : __ldg(a.merge_rec + id);
            if (active && (lane & 15) == 0) wait_pieces(a.merge_cnt + (size_t)id * kCntStride, (unsigned)rec.w);
            __syncwarp();
            if (lane == 0) TA_MARK(a, 190, rec.w);
            merge_record_row_half(a, rec, row % G, lane & 15, active);
        }
        __syncthreads();
        // the counters are ours alone now: reset them for the next launch
        // (which publishes only after its dependency wait, i.e. after this grid)
        for (int x = threadIdx.x; x < n_own; x += NTHREADS) a.merge_cnt[(size_t)(x < MAXO ? s_own_id[x] : a.cta_own[o0 + x]) * kCntStride] = 0u;
    }
    if (threadIdx.x == 0) TA_MARK(a, 191, *tmem_slot);
    if (TA_LIGHT_TRACE && !TRACE && a.trace && threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_) : "r"(s_ioff[0]) : "memory");
        a.trace[blockIdx.x * TRACE_SLOTS + 1] = (long long)t_;
    }
    if (TRACE && a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * TRACE_SLOTS + 195] = clock64();
        a.trace[blockIdx.x * TRACE_SLOTS + 194] = gtimer();
    }
    if (TRACE && threadIdx.x == 0) timeline_mark(a.timeline, 0, false);
    if (TRACE && a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * TRACE_SLOTS + 1] = gtimer();
        a.trace[blockIdx.x * TRACE_SLOTS + 5] = clock64();
        int nt = 0;
        for (int k = 0; k < n_items; ++k) nt += item_at(k).tile_end - item_at(k).tile_begin;
        a.trace[blockIdx.x * TRACE_SLOTS + 3] = nt;
    }
}

}  // namespace

bool mma_supported(int D, int kv_bf16) { return kv_bf16 && D == DH; }

bool make_pool_tmap(void* tmap_out, const void* base, int64_t rows, int D, int box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    CUtensorMap* m = reinterpret_cast<CUtensorMap*>(tmap_out);
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

cudaError_t launch_attn_mma(const AttnArgs& a, bool pdl, cudaStream_t s) {
    if (!mma_supported(a.D, a.kv_bf16)) return cudaErrorNotSupported;
    const bool trace = (a.trace && !TA_LIGHT_TRACE) || a.timeline;
    cudaError_t e = set_smem_attr_once(trace ? (const void*)attn_mma_kernel<true> : (const void*)attn_mma_kernel<false>,
                                       SMEM_BYTES);
    if (e != cudaSuccess) return e;
    TmapSet tm;
    std::memcpy(tm.k, a.tmap_k, sizeof(tm.k));
    std::memcpy(tm.v, a.tmap_v, sizeof(tm.v));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.n_ctas);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return trace ? cudaLaunchKernelEx(&cfg, attn_mma_kernel<true>, tm, a)
                 : cudaLaunchKernelEx(&cfg, attn_mma_kernel<false>, tm, a);
}

}  // namespace ta
