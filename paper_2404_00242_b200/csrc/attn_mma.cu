// attn_mma.cu -- persistent tcgen05/TMEM chunk attention (bf16 KV, D = 128).
//
// One launch per layer, one CTA per SM.  A CTA walks its items (a run of
// tiles of one lane for one kv head, see ta_internal.h).  Rows of an item
// are (query slot, q head in the GQA group) pairs, <= 128 of them, one per
// TMEM lane.  Per tile (<= 8 groups of 16 pool rows = <= 128 tokens):
//   TMA (warp 0)    K/V boxes -> SMEM ring (128B swizzle), 3 stages, K and V
//                   on separate barriers; runs ahead across items
//   QK  (warp 1)    S = Q K^T  (M=128, N=16*groups, K=128), Q from TMEM
//                   -> S buffer (t & 1) in TMEM
//   PV  (warp 2)    O += P V   (M=128, N=128, K=16*groups), P from TMEM
//   softmax (warps 4-11, thread = TMEM lane = row, two column halves)
//                   pass 1: tcgen05.ld S -> tree-masked row max; exchange
//                   with the other half; online softmax in base 2 with lazy
//                   O rescale; pass 2: tcgen05.ld S -> P = exp2 -> bf16 ->
//                   tcgen05.st into TMEM.  Warps none of whose rows attend
//                   the tile (sparse lanes) skip the exponentials.
// TMEM: S0 [0,128) S1 [128,256) O [256,384) P [384,448) Q [448,512); the
// whole SMEM budget goes to the KV ring.
// At an item's end the softmax warps write each attended row either as the
// final output (its leaf-head is covered by this item alone) or as an
// (O/l, log2 lse) partial record that merge.cu combines right after.
//
// Reference semantics: group_attention (attention.hpp:117-204) over every
// chunk a leaf attends; tree_reduce (attention.hpp:209-233) in merge.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "ta_ptx.cuh"

namespace ta {
namespace {

using namespace dev;

constexpr int BM = 128;                                  // rows per item (TMEM lanes)
constexpr int DH = 128;                                  // head dim
constexpr int NSTAGE = 3;                                // KV ring depth
constexpr int HALF = BM * 128;                           // one 64-column half of a [128][128] bf16 tile
constexpr int TILE = 2 * HALF;                           // 32 KB
constexpr int STAGE = 2 * TILE;                          // K + V
constexpr int SMEM_KV = 0;                               // stage s: K at s*STAGE, V at +TILE
constexpr int SMEM_BAR = NSTAGE * STAGE;                 // 196608
constexpr int SMEM_RED = SMEM_BAR + 256;                 // [2 parity][2 half][128] fp32 row max
constexpr int SMEM_REDL = SMEM_RED + 2 * 2 * BM * 4;     // [2 half][128] fp32 row sum
constexpr int SMEM_BYTES = SMEM_REDL + 2 * BM * 4 + 1024;   // + alignment slack
constexpr int NTHREADS = 384;
constexpr int NSOFT = 256;
constexpr int TMEM_COLS = 512;
constexpr int TMEM_S = 0, TMEM_O = 256, TMEM_P = 384, TMEM_Q = 448;
constexpr float kLazy = 8.0f;                            // rescale O only when the max grows by > 2^8

enum { FULLK = 0, FULLV = 3, EMPTYK = 6, EMPTYV = 9, S_FULL = 12, S_FREE = 14, P_FULL = 16, O_FULL = 17, Q_FULL = 18,
       Q_FREE = 19, NBAR = 20 };

// Optional pipeline trace (debug; AttnArgs::trace != nullptr): per CTA 256
// int64 slots: [0] start / [1] end (%globaltimer ns), [2] SM id, [3] tiles,
// then per tile t < 31 (clock64, 8 slots): [8+8t] K loads issued, [+1] S
// seen by softmax, [+2] S loaded + masked, [+3] row max exchanged, [+4]
// O_FULL(t-1) seen, [+5] O rescaled, [+6] P published, [+7] item epilogue
// done (last tile of an item only).
constexpr int TRACE_SLOTS = 256, TRACE_TILES = 31;
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TA_TRACE_EPI(a, k)                                                                         \
    do {                                                                                           \
        if ((a).trace && threadIdx.x == 128) (a).trace[blockIdx.x * TRACE_SLOTS + 248 + (k)] = clock64(); \
    } while (0)
#define TA_TRACE(a, t, k)                                                                          \
    do {                                                                                           \
        if ((a).trace && (t) < TRACE_TILES) (a).trace[blockIdx.x * TRACE_SLOTS + 8 + 8 * (t) + (k)] = clock64(); \
    } while (0)

struct TmapSet {
    CUtensorMap k[4];   // boxes of 16, 32, 64, 128 pool rows x 64 columns
    CUtensorMap v[4];
};

__global__ void __launch_bounds__(NTHREADS, 1)
    attn_mma_kernel(const __grid_constant__ TmapSet tm, const AttnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + SMEM_BAR;
    auto BAR = [&](int i) { return bar0 + 8u * (uint32_t)i; };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SMEM_BAR + 192);
    float* red = reinterpret_cast<float*>(smem + SMEM_RED);
    float* redl = reinterpret_cast<float*>(smem + SMEM_REDL);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int it0 = a.cta_begin[blockIdx.x], it1 = a.cta_begin[blockIdx.x + 1];

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * NSTAGE; ++i) mbar_init(BAR(FULLK + i), 1);       // FULLK, FULLV
        for (int i = 0; i < 2 * NSTAGE; ++i) mbar_init(BAR(EMPTYK + i), 1);      // EMPTYK, EMPTYV
        for (int i = 0; i < 2; ++i) {
            mbar_init(BAR(S_FULL + i), 1);
            mbar_init(BAR(S_FREE + i), NSOFT);
        }
        mbar_init(BAR(P_FULL), NSOFT);
        mbar_init(BAR(O_FULL), 1);
        mbar_init(BAR(Q_FULL), NSOFT);
        mbar_init(BAR(Q_FREE), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
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
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_launch_dependents();
    pdl_wait();   // previous launch finished: queries, outputs, partial scratch are ours
    if (a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * TRACE_SLOTS] = gtimer();
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[blockIdx.x * TRACE_SLOTS + 2] = smid;
    }

    // next tile of this CTA after tile t of item ii (-1: none); *nii = its item
    auto next_tile = [&](int ii, int t, int tile_end, int* nii) -> int {
        if (t + 1 < tile_end) {
            *nii = ii;
            return t + 1;
        }
        *nii = ii + 1;
        return ii + 1 < it1 ? a.items[ii + 1].tile_begin : -1;
    };

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0 && it0 < it1) {
            int gt = 0, ii = it0;
            ItemDesc I = a.items[ii];
            int t = I.tile_begin;
            TileDesc td = a.tiles[t];
            int4 rlo = *reinterpret_cast<const int4*>(a.tile_meta[t].row);
            int4 rhi = *reinterpret_cast<const int4*>(a.tile_meta[t].row + 4);
            while (true) {
                // prefetch the next tile's descriptor and rows (independent loads)
                int nii;
                const int nt = next_tile(ii, t, I.tile_end, &nii);
                TileDesc ntd{};
                int4 nrlo{}, nrhi{};
                if (nt >= 0) {
                    ntd = a.tiles[nt];
                    nrlo = *reinterpret_cast<const int4*>(a.tile_meta[nt].row);
                    nrhi = *reinterpret_cast<const int4*>(a.tile_meta[nt].row + 4);
                }
                const int rows8[8] = {rlo.x, rlo.y, rlo.z, rlo.w, rhi.x, rhi.y, rhi.z, rhi.w};
                auto row_of = [&](int g) {   // register select (no local-memory indexing)
                    int v = rows8[0];
#pragma unroll
                    for (int k = 1; k < 8; ++k) v = g == k ? rows8[k] : v;
                    return v;
                };
                const int64_t row0 = a.layer_row0 + (int64_t)I.head * a.head_rows;
                const int s = gt % NSTAGE;
                const uint32_t ph = (uint32_t)(gt / NSTAGE) & 1u;
                const uint32_t kdst = sbase + SMEM_KV + (uint32_t)s * STAGE;
                const uint32_t vdst = kdst + TILE;
                const uint32_t bytes = (uint32_t)td.ng * 4096u;
                mbar_wait(BAR(EMPTYK + s), ph ^ 1);
                mbar_expect_tx(BAR(FULLK + s), bytes);
                for (int b = 0; b < td.nbox; ++b) {
                    const int g = td.box[b] >> 2, sz = td.box[b] & 3;
                    const int row = (int)(row0 + row_of(g));
                    tma_load_2d(kdst + g * 2048, &tm.k[sz], 0, row, BAR(FULLK + s));
                    tma_load_2d(kdst + HALF + g * 2048, &tm.k[sz], 64, row, BAR(FULLK + s));
                }
                TA_TRACE(a, gt, 0);
                mbar_wait(BAR(EMPTYV + s), ph ^ 1);
                mbar_expect_tx(BAR(FULLV + s), bytes);
                for (int b = 0; b < td.nbox; ++b) {
                    const int g = td.box[b] >> 2, sz = td.box[b] & 3;
                    const int row = (int)(row0 + row_of(g));
                    tma_load_2d(vdst + g * 2048, &tm.v[sz], 0, row, BAR(FULLV + s));
                    tma_load_2d(vdst + HALF + g * 2048, &tm.v[sz], 64, row, BAR(FULLV + s));
                }
                ++gt;
                if (nt < 0) break;
                if (nii != ii) {
                    ii = nii;
                    I = a.items[ii];
                }
                t = nt;
                td = ntd;
                rlo = nrlo;
                rhi = nrhi;
            }
        }
    } else if (warp == 1) {
        // ===================== QK issuer: S = Q K^T =====================
        if (lane == 0) {
            int gt = 0;
            for (int ii = it0; ii < it1; ++ii) {
                const ItemDesc I = a.items[ii];
                int ng = a.tiles[I.tile_begin].ng;
                mbar_wait(BAR(Q_FULL), (ii - it0) & 1);
                for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                    const int ng_next = t + 1 < I.tile_end ? a.tiles[t + 1].ng : 0;
                    const int s = gt % NSTAGE, sb = gt & 1;
                    mbar_wait(BAR(FULLK + s), (uint32_t)(gt / NSTAGE) & 1u);
                    if (gt >= 2) mbar_wait(BAR(S_FREE + sb), ((gt >> 1) - 1) & 1);
                    tc_fence_after();
                    const uint32_t sK = sbase + SMEM_KV + (uint32_t)s * STAGE;
                    const uint32_t id = idesc_bf16(BM, 16 * ng, 0, 0);
#pragma unroll
                    for (int k = 0; k < DH / 16; ++k) {
                        const uint32_t off = (uint32_t)((k >> 2) * HALF + (k & 3) * 32);
                        mma_bf16_ts(tmem + TMEM_S + sb * 128, tmem + TMEM_Q + 8 * k, sdesc(sK + off, 16, 1024), id, k > 0);
                    }
                    mma_commit(BAR(S_FULL + sb));
                    mma_commit(BAR(EMPTYK + s));
                    ng = ng_next;
                }
                mma_commit(BAR(Q_FREE));
            }
        }
    } else if (warp == 2) {
        // ===================== PV issuer: O += P V =====================
        if (lane == 0) {
            int gt = 0;
            for (int ii = it0; ii < it1; ++ii) {
                const ItemDesc I = a.items[ii];
                int ng = a.tiles[I.tile_begin].ng;
                for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                    const int ng_next = t + 1 < I.tile_end ? a.tiles[t + 1].ng : 0;
                    const int s = gt % NSTAGE;
                    mbar_wait(BAR(FULLV + s), (uint32_t)(gt / NSTAGE) & 1u);
                    mbar_wait(BAR(P_FULL), gt & 1);
                    tc_fence_after();
                    const uint32_t sV = sbase + SMEM_KV + (uint32_t)s * STAGE + TILE;
                    const uint32_t id = idesc_bf16(BM, DH, 0, 1);
                    const bool first = t == I.tile_begin;
                    for (int kk = 0; kk < ng; ++kk)
                        mma_bf16_ts(tmem + TMEM_O, tmem + TMEM_P + 8 * kk, sdesc(sV + kk * 2048, HALF, 1024), id,
                                    (!first || kk > 0) ? 1u : 0u);
                    mma_commit(BAR(EMPTYV + s));
                    mma_commit(BAR(O_FULL));
                    ng = ng_next;
                }
            }
        }
    } else if (warp == 3) {
        fill_empty(a, lane);
    } else {
        // ===================== softmax / epilogue (256 threads) =====================
        const int q4 = warp & 3;                 // TMEM lane quadrant of this warp
        const int h = (warp - 4) >> 2;           // column half (S groups 4h..4h+3, O / Q columns 64h..)
        const int r = q4 * 32 + lane;            // row == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
        const int G = a.G;
        const float sc = a.scale_log2;

        // Q rows of item ii (this thread: dims [64h, 64h+64) of row r, i.e.
        // 32 packed bf16 pairs): global loads into registers, then (once the
        // previous item's QK is complete) tcgen05.st into the Q columns
        auto q_fetch = [&](int ii, uint4 (&v)[8]) {
            const ItemDesc I = a.items[ii];
            if (r < I.n_slots * G) {
                const int leaf = a.slot_leaf[I.slot_begin + r / G];
                const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.q) +
                                                                  ((size_t)leaf * a.hq_loc + I.head * G + r % G) * DH);
#pragma unroll
                for (int c = 0; c < 8; ++c) v[c] = src[8 * h + c];
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) v[c] = make_uint4(0, 0, 0, 0);
            }
        };
        auto q_store = [&](const uint4 (&v)[8]) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
            TA_TMEM_ST16(tmem + lane_addr + TMEM_Q + 32 * h, w);
            TA_TMEM_ST16(tmem + lane_addr + TMEM_Q + 32 * h + 16, (w + 16));
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(BAR(Q_FULL));
        };

        if (it0 < it1) {
            uint4 qv[8];
            q_fetch(it0, qv);
            q_store(qv);
        }
        int gt = 0;
        for (int ii = it0; ii < it1; ++ii) {
            const ItemDesc I = a.items[ii];
            const int nrows = I.n_slots * G;
            const bool live_row = r < nrows;
            const int j = live_row ? r / G : 0;      // local query slot
            const int g_in = r % G;
            const bool warp_live = q4 * 32 < nrows;
            float m = -INFINITY, l = 0.f;
            // this thread's half of the tile metadata, prefetched a tile ahead
            TileDesc td = a.tiles[I.tile_begin];
            uint4 inf = *reinterpret_cast<const uint4*>(a.tile_meta[I.tile_begin].info + 4 * h);

            for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                TileDesc ntd{};
                uint4 ninf{};
                if (t + 1 < I.tile_end) {
                    ntd = a.tiles[t + 1];
                    ninf = *reinterpret_cast<const uint4*>(a.tile_meta[t + 1].info + 4 * h);
                }
                const int ng = td.ng;
                const int g0 = 4 * h;
                const uint32_t info[4] = {inf.x, inf.y, inf.z, inf.w};
                // per group: number of leading columns this row attends (0: none)
                int lim[4];
                bool att = false;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int b = (int)((info[g] >> 8) & 0xfffu), e = (int)(info[g] >> 20);
                    lim[g] = (live_row && g0 + g < ng && j >= b && j < e) ? (int)(info[g] & 0xffu) : 0;
                    att |= lim[g] > 0;
                }
                const bool warp_att = __any_sync(0xffffffffu, att);
                const int sb = gt & 1;
                const uint32_t s_addr = tmem + lane_addr + TMEM_S + sb * 128;
                mbar_wait(BAR(S_FULL + sb), (gt >> 1) & 1);
                if (threadIdx.x == 128) TA_TRACE(a, gt, 1);
                tc_fence_after();
                // pass 1: masked row max of my half (scale > 0 commutes with max)
                float mx = -INFINITY;
                if (warp_att) {
#pragma unroll
                    for (int g2 = 0; g2 < 4; g2 += 2) {
                        if (g0 + g2 < ng) {
                            uint32_t rr[32];
                            TA_TMEM_LD16(s_addr + (g0 + g2) * 16, rr);
                            if (g0 + g2 + 1 < ng) TA_TMEM_LD16(s_addr + (g0 + g2 + 1) * 16, (rr + 16));
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                if (c < lim[g2]) mx = fmaxf(mx, __uint_as_float(rr[c]));
                                if (c < lim[g2 + 1]) mx = fmaxf(mx, __uint_as_float(rr[16 + c]));
                            }
                        }
                    }
                }
                if (threadIdx.x == 128) TA_TRACE(a, gt, 2);
                // combine the two column halves of the row (partner warp: same quadrant)
                float* rd = red + (gt & 1) * 2 * BM;
                rd[h * BM + r] = mx;
                named_bar(1 + q4, 64);
                mx = fmaxf(mx, rd[(h ^ 1) * BM + r]) * sc;
                if (threadIdx.x == 128) TA_TRACE(a, gt, 3);
                // lazy rescale: keep the stale max unless it grew by > kLazy (both
                // threads of a row decide alike).  The O correction is warp-collective.
                const bool grow = mx > m + kLazy;
                float f = 1.f;
                if (grow) {
                    if (m != -INFINITY) f = ex2(m - mx);
                    l *= f;
                    m = mx;
                }
                if (gt > 0) mbar_wait(BAR(O_FULL), (gt - 1) & 1);   // PV(t-1) done: P free, O settled
                if (threadIdx.x == 128) TA_TRACE(a, gt, 4);
                tc_fence_after();
                if (t > I.tile_begin && __any_sync(0xffffffffu, grow && f != 1.f)) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[16];
                        TA_TMEM_LD16(tmem + lane_addr + TMEM_O + h * 64 + c * 16, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
                        TA_TMEM_ST16(tmem + lane_addr + TMEM_O + h * 64 + c * 16, o);
                    }
                }
                if (threadIdx.x == 128) TA_TRACE(a, gt, 5);
                if (warp_att) {
                    // pass 2: P = exp2(s * scale - m) -> bf16 pairs -> TMEM; l += sum(P)
                    const float negm = m == -INFINITY ? 0.f : -m;
                    float la = 0.f;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (g0 + g < ng) {
                            uint32_t rr[16];
                            TA_TMEM_LD16(s_addr + (g0 + g) * 16, rr);
                            tmem_wait_ld();
                            uint32_t pk[8];
#pragma unroll
                            for (int c = 0; c < 8; ++c) {
                                const float p0 = 2 * c < lim[g] ? ex2(fmaf(__uint_as_float(rr[2 * c]), sc, negm)) : 0.f;
                                const float p1 =
                                    2 * c + 1 < lim[g] ? ex2(fmaf(__uint_as_float(rr[2 * c + 1]), sc, negm)) : 0.f;
                                la += p0 + p1;
                                pk[c] = pack_bf16(p0, p1);
                            }
                            TA_TMEM_ST8(tmem + lane_addr + TMEM_P + 8 * (g0 + g), pk);
                        }
                    }
                    l += la;
                } else if (warp_live) {
                    // no row of this warp attends my half of the tile: P = 0
                    const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        if (g0 + g < ng) TA_TMEM_ST8(tmem + lane_addr + TMEM_P + 8 * (g0 + g), z);
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(BAR(S_FREE + sb));
                mbar_arrive(BAR(P_FULL));
                if (threadIdx.x == 128) TA_TRACE(a, gt, 6);
                td = ntd;
                inf = ninf;
            }

            // ---- epilogue.  Next item's Q: global loads now, TMEM after O is out
            const bool has_next = ii + 1 < it1;
            uint4 qv[8];
            if (has_next) q_fetch(ii + 1, qv);
            mbar_wait(BAR(O_FULL), (gt - 1) & 1);
            TA_TRACE_EPI(a, 0);
            tc_fence_after();
            redl[h * BM + r] = l;
            named_bar(1 + q4, 64);
            l += redl[(h ^ 1) * BM + r];
            const float inv = l > 0.f ? 1.f / l : 0.f;
            const float lse2 = m + log2f(l);
            const int code = live_row ? a.slot_out[I.out_begin + j] : kSlotUnused;
            const int hq = I.head * G + g_in;
            if (warp_live) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[16];
                    const int col = h * 64 + c * 16;
                    TA_TMEM_LD16(tmem + lane_addr + TMEM_O + col, o);
                    tmem_wait_ld();
                    if (code != kSlotUnused) {
                        const float* of = reinterpret_cast<const float*>(o);
                        if (code < 0) {
                            const int leaf = -1 - code;
                            store_row<16>(a.out, ((size_t)leaf * a.hq_loc + hq) * DH + col, of, inv, a.out_bf16);
                            if (c == 0 && h == 0 && a.lse) a.lse[(size_t)leaf * a.hq_loc + hq] = lse2 * kLn2;
                        } else {
                            store_row<16>(a.part_o, ((size_t)code * G + g_in) * DH + col, of, inv, 0);
                            if (c == 0 && h == 0) a.part_lse[(size_t)code * G + g_in] = lse2;
                        }
                    }
                }
            }
            TA_TRACE_EPI(a, 1);
            if (has_next) {
                mbar_wait(BAR(Q_FREE), (ii - it0) & 1);
                tc_fence_after();
                q_store(qv);
            } else {
                tc_fence_before();
            }
            if (threadIdx.x == 128) TA_TRACE(a, gt - 1, 7);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * TRACE_SLOTS + 1] = gtimer();
        int nt = 0;
        for (int ii = it0; ii < it1; ++ii) nt += a.items[ii].tile_end - a.items[ii].tile_begin;
        a.trace[blockIdx.x * TRACE_SLOTS + 3] = nt;
    }
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
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
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        if (e != cudaSuccess) return e;
        configured = true;
    }
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
    return cudaLaunchKernelEx(&cfg, attn_mma_kernel, tm, a);
}

}  // namespace ta
