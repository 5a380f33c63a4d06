// attn_mma.cu -- persistent tcgen05/TMEM chunk attention (bf16 KV, D = 128).
//
// One launch per layer, one CTA per SM.  A CTA walks its items (a run of
// tiles of one lane for one kv head, see ta_internal.h).  Rows of an item
// are (query slot, q head in the GQA group) pairs, <= 128 of them, one per
// TMEM lane.  Per tile (<= 8 groups of 16 pool rows = <= 128 tokens):
//   TMA (warp 0)    K/V boxes -> SMEM stage (128B swizzle), 2 stages, K and
//                   V on separate barriers; runs ahead across items
//   QK  (warp 1)    S = Q K^T  (M=128, N=16*groups, K=128)  -> TMEM [0,128)
//   PV  (warp 2)    O += P V   (M=128, N=128, K=16*groups)  -> TMEM [128,256)
//   softmax (warps 4-11, thread = TMEM lane = row, two column halves)
//                   tcgen05.ld S -> tree mask (slot range per group) ->
//                   online softmax in base 2 with lazy O rescale -> P bf16
//                   -> SMEM (swizzled K-major)
// At an item's end the softmax warps write each attended row either as the
// final output (its leaf-head is covered by this item alone) or as an
// (O/l, lse) partial; the CTA whose arrival completes a leaf-head's partial
// set merges it (last-arriver merge, partials read back from L2).  The next
// item's Q is staged before the epilogue, so QK of its first tile overlaps it.
//
// Reference semantics: group_attention (attention.hpp:117-204) over every
// chunk a leaf attends, and tree_reduce (attention.hpp:209-233), fused.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "ta_ptx.cuh"

namespace ta {
namespace {

using namespace dev;

constexpr int BM = 128;                                  // rows per item (TMEM lanes)
constexpr int DH = 128;                                  // head dim
constexpr int NSTAGE = 2;
constexpr int HALF = BM * 128;                           // one 64-column half of a [128][128] bf16 tile
constexpr int TILE = 2 * HALF;                           // 32 KB
constexpr int SMEM_Q = 0;
constexpr int SMEM_P = TILE;
constexpr int SMEM_KV = 2 * TILE;                        // stage s: K at +s*2*TILE, V at +TILE
constexpr int SMEM_BAR = SMEM_KV + NSTAGE * 2 * TILE;    // 196608
constexpr int SMEM_RED = SMEM_BAR + 256;                 // [2 parity][2 half][128] fp32 row max
constexpr int SMEM_REDL = SMEM_RED + 2 * 2 * BM * 4;     // [2 half][128] fp32 row sum
constexpr int SMEM_FLAG = SMEM_REDL + 2 * BM * 4;        // [128] merge flags per slot
constexpr int SMEM_BYTES = SMEM_FLAG + BM * 4 + 1024;    // + alignment slack
constexpr int NTHREADS = 384;
constexpr int NSOFT = 256;
constexpr int TMEM_COLS = 256;
constexpr int TMEM_S = 0, TMEM_O = 128;
constexpr float kLazy = 8.0f;                            // rescale O only when the max grows by > 2^8

enum { FULLK = 0, FULLV = 2, EMPTYK = 4, EMPTYV = 6, S_FULL = 8, S_FREE = 9, P_FULL = 10, O_FULL = 11, Q_FULL = 12,
       Q_FREE = 13, NBAR = 14 };
enum { BAR_ALL_SOFT = 5 };                               // named barriers 1..4: quadrant pairs

// byte offset of 16-byte chunk c16 (0..15 over 128 columns) of row r of a
// [128][128] bf16 K-major SW128 tile stored as two 64-column halves
__device__ __forceinline__ uint32_t sw128_off(int r, int c16) {
    const int half = c16 >> 3, ch = c16 & 7;
    return (uint32_t)(half * HALF + (r >> 3) * 1024 + (r & 7) * 128 + ((ch ^ (r & 7)) << 4));
}

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
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SMEM_BAR + 128);
    float* red = reinterpret_cast<float*>(smem + SMEM_RED);
    float* redl = reinterpret_cast<float*>(smem + SMEM_REDL);
    int* flag = reinterpret_cast<int*>(smem + SMEM_FLAG);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int it0 = a.cta_begin[blockIdx.x], it1 = a.cta_begin[blockIdx.x + 1];

    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(BAR(i), 1);
        mbar_init(BAR(S_FULL), 1);
        mbar_init(BAR(S_FREE), NSOFT);
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
    pdl_wait();   // previous launch (layer) finished: counters, partials, outputs are ours

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int gt = 0;
            for (int ii = it0; ii < it1; ++ii) {
                const ItemDesc I = a.items[ii];
                const int64_t row0 = a.layer_row0 + (int64_t)I.head * a.head_rows;
                for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                    const TileDesc td = a.tiles[t];
                    int rows[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b)
                        rows[b] = b < td.nbox ? (int)(row0 + a.grp_row[td.grp_begin + (td.box[b] >> 2)]) : 0;
                    const int s = gt & 1;
                    const uint32_t kdst = sbase + SMEM_KV + (uint32_t)s * 2 * TILE;
                    const uint32_t vdst = kdst + TILE;
                    const uint32_t bytes = (uint32_t)td.ng * 4096u;
                    mbar_wait(BAR(EMPTYK + s), ((gt >> 1) & 1) ^ 1);
                    mbar_expect_tx(BAR(FULLK + s), bytes);
                    for (int b = 0; b < td.nbox; ++b) {
                        const int g = td.box[b] >> 2, sz = td.box[b] & 3;
                        tma_load_2d(kdst + g * 2048, &tm.k[sz], 0, rows[b], BAR(FULLK + s));
                        tma_load_2d(kdst + HALF + g * 2048, &tm.k[sz], 64, rows[b], BAR(FULLK + s));
                    }
                    mbar_wait(BAR(EMPTYV + s), ((gt >> 1) & 1) ^ 1);
                    mbar_expect_tx(BAR(FULLV + s), bytes);
                    for (int b = 0; b < td.nbox; ++b) {
                        const int g = td.box[b] >> 2, sz = td.box[b] & 3;
                        tma_load_2d(vdst + g * 2048, &tm.v[sz], 0, rows[b], BAR(FULLV + s));
                        tma_load_2d(vdst + HALF + g * 2048, &tm.v[sz], 64, rows[b], BAR(FULLV + s));
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== QK issuer: S = Q K^T =====================
        if (lane == 0) {
            const uint32_t sQ = sbase + SMEM_Q;
            int gt = 0;
            for (int ii = it0; ii < it1; ++ii) {
                const ItemDesc I = a.items[ii];
                mbar_wait(BAR(Q_FULL), (ii - it0) & 1);
                for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                    const int ng = a.tiles[t].ng;
                    const int s = gt & 1;
                    mbar_wait(BAR(FULLK + s), (gt >> 1) & 1);
                    if (gt > 0) mbar_wait(BAR(S_FREE), (gt - 1) & 1);
                    tc_fence_after();
                    const uint32_t sK = sbase + SMEM_KV + (uint32_t)s * 2 * TILE;
                    const uint32_t id = idesc_bf16(BM, 16 * ng, 0, 0);
#pragma unroll
                    for (int k = 0; k < DH / 16; ++k) {
                        const uint32_t off = (uint32_t)((k >> 2) * HALF + (k & 3) * 32);
                        mma_bf16(tmem + TMEM_S, sdesc(sQ + off, 16, 1024), sdesc(sK + off, 16, 1024), id, k > 0);
                    }
                    mma_commit(BAR(S_FULL));
                    mma_commit(BAR(EMPTYK + s));
                }
                mma_commit(BAR(Q_FREE));
            }
        }
    } else if (warp == 2) {
        // ===================== PV issuer: O += P V =====================
        if (lane == 0) {
            const uint32_t sP = sbase + SMEM_P;
            int gt = 0;
            for (int ii = it0; ii < it1; ++ii) {
                const ItemDesc I = a.items[ii];
                for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                    const int ng = a.tiles[t].ng;
                    const int s = gt & 1;
                    mbar_wait(BAR(FULLV + s), (gt >> 1) & 1);
                    mbar_wait(BAR(P_FULL), gt & 1);
                    tc_fence_after();
                    const uint32_t sV = sbase + SMEM_KV + (uint32_t)s * 2 * TILE + TILE;
                    const uint32_t id = idesc_bf16(BM, DH, 0, 1);
                    const bool first = t == I.tile_begin;
                    for (int kk = 0; kk < ng; ++kk) {
                        const uint32_t poff = (uint32_t)((kk >> 2) * HALF + (kk & 3) * 32);
                        mma_bf16(tmem + TMEM_O, sdesc(sP + poff, 16, 1024), sdesc(sV + kk * 2048, HALF, 1024), id,
                                 (!first || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(BAR(EMPTYV + s));
                    mma_commit(BAR(O_FULL));
                }
            }
        }
    } else if (warp == 3) {
        fill_empty(a, lane);
    } else {
        // ===================== softmax / epilogue (256 threads) =====================
        const int q4 = warp & 3;                 // TMEM lane quadrant of this warp
        const int h = (warp - 4) >> 2;           // column half (S groups 4h..4h+3, O columns 64h..)
        const int r = q4 * 32 + lane;            // row == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
        const int G = a.G;
        const float sc = a.scale_log2;

        // stage the Q rows of item ii (this thread: 8 of the 16 chunks of row r)
        auto load_q = [&](int ii) {
            const ItemDesc I = a.items[ii];
            const int nrows = I.n_slots * G;
            if (r < nrows) {
                const int leaf = a.slot_leaf[I.slot_begin + r / G];
                const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.q) +
                                                                  ((size_t)leaf * a.hq_loc + I.head * G + r % G) * DH);
                uint4 v[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) v[c] = src[8 * h + c];
#pragma unroll
                for (int c = 0; c < 8; ++c) sts128(sbase + SMEM_Q + sw128_off(r, 8 * h + c), v[c].x, v[c].y, v[c].z, v[c].w);
            }
            fence_proxy_async();
            mbar_arrive(BAR(Q_FULL));
        };

        if (it0 < it1) load_q(it0);
        int gt = 0;
        for (int ii = it0; ii < it1; ++ii) {
            const ItemDesc I = a.items[ii];
            const int nrows = I.n_slots * G;
            const bool live_row = r < nrows;
            const int j = live_row ? r / G : 0;      // local query slot
            const int g_in = r % G;
            const bool warp_live = q4 * 32 < nrows;
            float m = -INFINITY, l = 0.f;

            for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
                const TileDesc td = a.tiles[t];
                const int ng = td.ng;
                const int g0 = 4 * h;
                uint32_t info[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) info[g] = (g0 + g < ng) ? a.grp_info[td.grp_begin + g0 + g] : 0u;
                mbar_wait(BAR(S_FULL), gt & 1);
                tc_fence_after();
                float sv[64];
                if (warp_live) {
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (g0 + g < ng) {
                            uint32_t rr[16];
                            TA_TMEM_LD16(tmem + lane_addr + TMEM_S + (g0 + g) * 16, rr);
#pragma unroll
                            for (int c = 0; c < 16; ++c) sv[g * 16 + c] = __uint_as_float(rr[c]);
                        }
                    }
                    tmem_wait_ld();
                }
                tc_fence_before();
                mbar_arrive(BAR(S_FREE));

                // tree mask on the raw scores (scale > 0 commutes with max)
                float mx = -INFINITY;
                if (warp_live) {
                    float mxa[4];
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        mxa[g] = -INFINITY;
                        if (g0 + g < ng) {
                            const int cnt = (int)(info[g] & 0xffu), b = (int)((info[g] >> 8) & 0xfffu),
                                      e = (int)(info[g] >> 20);
                            const int lim = (live_row && j >= b && j < e) ? cnt : 0;
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                const float v = c < lim ? sv[g * 16 + c] : -INFINITY;
                                sv[g * 16 + c] = v;
                                mxa[g] = fmaxf(mxa[g], v);
                            }
                        }
                    }
                    mx = fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3]));
                }
                // combine the two column halves of the row (partner warp: same quadrant)
                float* rd = red + (gt & 1) * 2 * BM;
                rd[h * BM + r] = mx;
                named_bar(1 + q4, 64);
                mx = fmaxf(mx, rd[(h ^ 1) * BM + r]) * sc;
                // lazy rescale: keep the stale max unless it grew by > kLazy (both
                // threads of a row decide alike).  The O correction is warp-collective.
                const bool grow = mx > m + kLazy;
                float f = 1.f;
                if (grow) {
                    if (m != -INFINITY) f = ex2(m - mx);
                    l *= f;
                    m = mx;
                }
                if (gt > 0) mbar_wait(BAR(O_FULL), (gt - 1) & 1);   // PV(t-1) done: P buffer free, O settled
                if (t > I.tile_begin && __any_sync(0xffffffffu, grow && f != 1.f)) {
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[16];
                        TA_TMEM_LD16(tmem + lane_addr + TMEM_O + h * 64 + c * 16, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
                        TA_TMEM_ST16(tmem + lane_addr + TMEM_O + h * 64 + c * 16, o);
                    }
                    tmem_wait_st();
                }
                if (warp_live) {
                    // P = exp2(s * scale - m) -> bf16 -> SMEM; l += sum(P)
                    const float negm = m == -INFINITY ? 0.f : -m;
                    float la[4];
                    const uint32_t prow = sbase + SMEM_P;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        la[g] = 0.f;
                        if (g0 + g < ng) {
                            uint32_t pk[8];
#pragma unroll
                            for (int c = 0; c < 8; ++c) {
                                const float p0 = ex2(fmaf(sv[g * 16 + 2 * c], sc, negm));
                                const float p1 = ex2(fmaf(sv[g * 16 + 2 * c + 1], sc, negm));
                                la[g] += p0 + p1;
                                pk[c] = pack_bf16(p0, p1);
                            }
                            sts128(prow + sw128_off(r, 2 * (g0 + g)), pk[0], pk[1], pk[2], pk[3]);
                            sts128(prow + sw128_off(r, 2 * (g0 + g) + 1), pk[4], pk[5], pk[6], pk[7]);
                        }
                    }
                    l += (la[0] + la[1]) + (la[2] + la[3]);
                    fence_proxy_async();
                }
                tc_fence_before();
                mbar_arrive(BAR(P_FULL));
            }

            // next item's Q (QK of this item is complete once Q_FREE fires)
            if (ii + 1 < it1) {
                mbar_wait(BAR(Q_FREE), (ii - it0) & 1);
                load_q(ii + 1);
            }

            // ---- epilogue: O / l -> final output or partial record
            mbar_wait(BAR(O_FULL), (gt - 1) & 1);
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
            tc_fence_before();
            if (I.pad & 1) {
                // last-arriver merge of the leaf-heads this item holds partials of
                __threadfence();
                named_bar(BAR_ALL_SOFT, NSOFT);
                if (live_row && g_in == 0 && h == 0) {
                    int f = 0;
                    if (code >= 0) {
                        const int mi = a.part_merge[code];
                        const int need = a.merge_begin[mi + 1] - a.merge_begin[mi];
                        if (atomicAdd(a.counters + mi, 1) == need - 1) {
                            a.counters[mi] = 0;   // self-reset for the next launch
                            f = 1;
                        }
                    }
                    flag[j] = f;
                }
                named_bar(BAR_ALL_SOFT, NSOFT);
                if (live_row && code >= 0 && flag[j]) {
                    __threadfence();
                    const int mi = a.part_merge[code];
                    merge_row<64>(a, mi, g_in, hq, a.merge_leaf[mi], h * 64);
                }
                named_bar(BAR_ALL_SOFT, NSOFT);   // flag[] reuse
            }
        }
    }

    tc_fence_before();
    __syncthreads();
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
