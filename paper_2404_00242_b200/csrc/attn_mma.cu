// attn_mma.cu -- tcgen05/TMEM path of the chunk attention (dense bf16 units).
//
// One CTA runs one unit for one kv head: up to 128 rows (query slot x q head
// in the GQA group) against a span of flatten chunks streamed as tiles of up
// to 8 TMA boxes (16 pool rows each, 128 tokens).  Per tile:
//   TMA (warp 0)   K/V boxes -> SMEM stage (128B swizzle), 2 stages
//   MMA (warp 1)   S = Q K^T   (M=128, N=16*boxes, K=128)  -> TMEM cols [0,128)
//                  O += P V    (M=128, N=128, K=16*boxes)  -> TMEM cols [128,256)
//   softmax (warps 2-5, thread = TMEM lane = row)
//                  tcgen05.ld S -> tree mask (slot range per box) -> online
//                  softmax in base 2 with lazy O rescale (only when the row max
//                  grows by > 2^8) -> P (bf16) -> SMEM (swizzled K-major)
// O and the row statistics stay on chip for the whole span; one (m, l, O)
// record per row leaves the SM at the end (or the final output directly).
//
// Reference semantics: group_attention (attention.hpp:117-204) per chunk and
// tree_reduce (attention.hpp:209-233) across chunks, fused.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>

#include "ta_kernels.h"

namespace ta {
namespace {

constexpr int BM = 128;           // rows per unit (TMEM lanes)
constexpr int BN = 128;           // tokens per tile (8 boxes of 16)
constexpr int DH = 128;           // head dim handled by this kernel
constexpr int NSTAGE = 2;
constexpr int HALF = BM * 128;    // bytes of one 64-column half of a [128][128] bf16 tile
constexpr int TILE = 2 * HALF;    // 32 KB
constexpr int SMEM_Q = 0;
constexpr int SMEM_P = TILE;
constexpr int SMEM_KV = 2 * TILE;                        // stage s: K at +s*2*TILE, V at +TILE
constexpr int SMEM_BAR = SMEM_KV + NSTAGE * 2 * TILE;    // 196608
constexpr int SMEM_RED = SMEM_BAR + 256;                 // [2][128] fp32 row exchange
constexpr int MAX_GRP = 256;                             // groups per unit held in SMEM (host caps units)
constexpr int SMEM_GRP = SMEM_RED + 2 * BM * 4;          // [MAX_GRP] row, [MAX_GRP] info
constexpr int SMEM_TBOX = SMEM_GRP + 2 * MAX_GRP * 4;
constexpr int SMEM_BYTES = SMEM_TBOX + (MAX_GRP / 8) * 16 + 1024;  // + alignment slack
constexpr int NTHREADS = 384;
constexpr int TMEM_COLS = 256;
constexpr int TMEM_S = 0, TMEM_O = 128;
constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLazy = 8.0f;     // rescale O only when the max grows by > 2^8

// ----------------------------------------------------------------- PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor, SWIZZLE_128B, sm_100 version bit.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 instruction descriptor: f32 accumulate, bf16 A/B.
__device__ __forceinline__ uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

#define TMEM_LD16(addr, r)                                                                                     \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),         \
                   "=r"(r[15])                                                                                  \
                 : "r"(addr))
#define TMEM_ST16(addr, r)                                                                                     \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
                 ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])      \
                 : "memory")
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

// byte offset of 16-byte chunk `c16` (0..15 across 128 columns) of row r in a
// [128][128] bf16 K-major SW128 tile stored as two 64-column halves
__device__ __forceinline__ uint32_t sw128_off(int r, int c16) {
    const int half = c16 >> 3, ch = c16 & 7;
    return (uint32_t)(half * HALF + (r >> 3) * 1024 + (r & 7) * 128 + ((ch ^ (r & 7)) << 4));
}

// Warp roles (384 threads):
//   warp 0      TMA producer (one lane)
//   warp 1      QK issuer (one lane); owns the TMEM allocation
//   warp 2      PV issuer (one lane)
//   warp 3      idle
//   warps 4-11  softmax: warp w handles TMEM lane quadrant (w & 3) and the
//               64-column half h = (w - 4) >> 2 of every S tile, so each row is
//               shared by two threads (row max exchanged through SMEM).
// QK and PV are issued by different threads so PV(t) never waits behind the
// data of tile t+1, and a stage is released as soon as PV(t) has read it.
constexpr int NSOFT = 256;

// TMA descriptors for boxes of 16, 32, 64, 128 pool rows, K and V.
struct TmapSet {
    CUtensorMap k[4];
    CUtensorMap v[4];
};
// trace slots per tile: 0 producer issue, 1 QK: data seen, 2 QK issued, 3 softmax: S seen,
// 4 softmax: P published, 5 PV issued, 6 producer: stage free seen
#define TRACE(t, slot)                                                                         \
    do {                                                                                        \
        if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && (t) < 64)                          \
            a.trace[(t) * 8 + (slot)] = clock64();                                              \
    } while (0)

__global__ void __launch_bounds__(NTHREADS, 1)
    attn_mma_kernel(const __grid_constant__ TmapSet tm, const AttnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
    const uint32_t bar0 = smem_u32(bars);
    auto BAR = [&](int i) { return bar0 + 8u * (uint32_t)i; };
    // K and V have their own full/empty barriers: K(t+2) is loaded as soon as
    // QK(t) has consumed stage t&1, V(t+2) once PV(t) has.
    enum { FULLK = 0, FULLV = 2, EMPTYK = 4, EMPTYV = 6, S_FULL = 8, S_FREE = 9, P_FULL = 10, O_FULL = 11,
           Q_FULL = 12, G_FULL = 13 };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SMEM_BAR + 128);
    float* red = reinterpret_cast<float*>(smem + SMEM_RED);   // [2][128] row-max halves, then l halves
    int32_t* g_row = reinterpret_cast<int32_t*>(smem + SMEM_GRP);
    // per tile: [0] = number of TMA boxes, [1..8] = (first group << 2) | log2(box rows / 16)
    uint8_t* t_box = smem + SMEM_TBOX;
    uint32_t* g_info = reinterpret_cast<uint32_t*>(smem + SMEM_GRP + MAX_GRP * 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kvh = blockIdx.y;
    const UnitDesc U = a.units[blockIdx.x];
    const int G = a.G;
    const int nrows = U.n_slots * G;
    const int ntiles = (U.n_grp + 7) >> 3;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(BAR(i), 1);
        mbar_init(BAR(S_FULL), 1);
        mbar_init(BAR(S_FREE), NSOFT);
        mbar_init(BAR(P_FULL), NSOFT);
        mbar_init(BAR(O_FULL), 1);
        mbar_init(BAR(Q_FULL), NSOFT);
        mbar_init(BAR(G_FULL), 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    long long t_begin = 0;
    if (a.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                asm volatile("prefetch.tensormap [%0];" ::"l"(&tm.k[i]) : "memory");
                asm volatile("prefetch.tensormap [%0];" ::"l"(&tm.v[i]) : "memory");
            }
            const int64_t row0 = a.layer_row0 + (int64_t)kvh * a.head_rows;
            mbar_wait(BAR(G_FULL), 0);
            for (int t = 0; t < ntiles; ++t) {
                const int s = t & 1;
                const int ng = min(8, U.n_grp - 8 * t);
                const uint32_t kdst = sbase + SMEM_KV + (uint32_t)s * 2 * TILE;
                const uint32_t vdst = kdst + TILE;
                const uint8_t* bx = t_box + 16 * t;
                const int nb = bx[0];
                const uint32_t bytes = (uint32_t)ng * 2u * 2048u;
                mbar_wait(BAR(EMPTYK + s), ((t >> 1) & 1) ^ 1);
                TRACE(t, 6);
                mbar_expect_tx(BAR(FULLK + s), bytes);
                for (int b = 0; b < nb; ++b) {
                    const int g = bx[1 + b] >> 2, sz = bx[1 + b] & 3;
                    const int row = (int)(row0 + g_row[8 * t + g]);
                    tma_load_2d(kdst + g * 2048, &tm.k[sz], 0, row, BAR(FULLK + s));
                    tma_load_2d(kdst + HALF + g * 2048, &tm.k[sz], 64, row, BAR(FULLK + s));
                }
                mbar_wait(BAR(EMPTYV + s), ((t >> 1) & 1) ^ 1);
                mbar_expect_tx(BAR(FULLV + s), bytes);
                for (int b = 0; b < nb; ++b) {
                    const int g = bx[1 + b] >> 2, sz = bx[1 + b] & 3;
                    const int row = (int)(row0 + g_row[8 * t + g]);
                    tma_load_2d(vdst + g * 2048, &tm.v[sz], 0, row, BAR(FULLV + s));
                    tma_load_2d(vdst + HALF + g * 2048, &tm.v[sz], 64, row, BAR(FULLV + s));
                }
                TRACE(t, 0);
            }
        }
    } else if (warp == 1) {
        // ===================== QK issuer: S = Q K^T =====================
        if (lane == 0) {
            const uint32_t sQ = sbase + SMEM_Q;
            mbar_wait(BAR(Q_FULL), 0);
            for (int t = 0; t < ntiles; ++t) {
                const int s = t & 1;
                mbar_wait(BAR(FULLK + s), (t >> 1) & 1);
                TRACE(t, 1);
                if (t > 0) mbar_wait(BAR(S_FREE), (t - 1) & 1);
                tc_fence_after();
                const int ng = min(8, U.n_grp - 8 * t);
                const uint32_t sK = sbase + SMEM_KV + (uint32_t)s * 2 * TILE;
                const uint32_t id = idesc_bf16(BM, 16 * ng, 0, 0);
#pragma unroll
                for (int k = 0; k < DH / 16; ++k) {
                    const uint32_t off = (uint32_t)((k >> 2) * HALF + (k & 3) * 32);
                    mma_bf16(tmem + TMEM_S, sdesc(sQ + off, 16, 1024), sdesc(sK + off, 16, 1024), id, k > 0);
                }
                mma_commit(BAR(S_FULL));
                mma_commit(BAR(EMPTYK + s));
                TRACE(t, 2);
            }
        }
    } else if (warp == 2) {
        // ===================== PV issuer: O += P V =====================
        if (lane == 0) {
            const uint32_t sP = sbase + SMEM_P;
            for (int t = 0; t < ntiles; ++t) {
                const int s = t & 1;
                mbar_wait(BAR(FULLV + s), (t >> 1) & 1);
                mbar_wait(BAR(P_FULL), t & 1);
                tc_fence_after();
                const int ng = min(8, U.n_grp - 8 * t);
                const uint32_t sV = sbase + SMEM_KV + (uint32_t)s * 2 * TILE + TILE;
                const uint32_t id = idesc_bf16(BM, DH, 0, 1);
                for (int kk = 0; kk < ng; ++kk) {
                    const uint32_t poff = (uint32_t)((kk >> 2) * HALF + (kk & 3) * 32);
                    mma_bf16(tmem + TMEM_O, sdesc(sP + poff, 16, 1024), sdesc(sV + kk * 2048, HALF, 1024), id,
                             (t > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(BAR(EMPTYV + s));
                mma_commit(BAR(O_FULL));
                TRACE(t, 5);
            }
        }
    } else if (warp == 3) {
        // ===================== group metadata -> SMEM (once per unit) =====================
        for (int g = lane; g < U.n_grp; g += 32) {
            g_row[g] = a.grp_row[U.grp_begin + g];
            g_info[g] = a.grp_info[U.grp_begin + g];
        }
        __syncwarp();
        // box plan per tile: runs of full, row-contiguous groups are loaded as
        // power-of-two boxes (8/4/2/1 groups); the box bytes always
        // equal 16 rows per group (masked rows are never read)
        for (int t = lane; t < ntiles; t += 32) {
            const int ng = min(8, U.n_grp - 8 * t);
            uint8_t* bx = t_box + 16 * t;
            int nb = 0, g = 0;
            while (g < ng) {
                int run = 1;  // full contiguous groups starting at g (the last may be partial)
                while (g + run < ng && (g_info[8 * t + g + run - 1] & 0xffu) == 16u &&
                       g_row[8 * t + g + run] == g_row[8 * t + g] + 16 * run)
                    ++run;
                while (run > 0) {
                    int sz = 3;
                    while ((1 << sz) > run) --sz;
                    bx[1 + nb++] = (uint8_t)((g << 2) | sz);
                    g += 1 << sz;
                    run -= 1 << sz;
                }
            }
            bx[0] = (uint8_t)nb;
        }
        __syncwarp();
        mbar_arrive(BAR(G_FULL));
    } else if (warp >= 4) {
        // ===================== softmax / epilogue (256 threads) =====================
        const int q4 = warp & 3;                 // TMEM lane quadrant of this warp
        const int h = (warp - 4) >> 2;           // column half (S groups 4h..4h+3, O cols 64h..)
        const int r = q4 * 32 + lane;            // row == TMEM lane
        const bool live_row = r < nrows;
        const int j = live_row ? r / G : -1;     // local query slot
        const int hq = kvh * G + (live_row ? r % G : 0);
        const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
        const bool warp_live = q4 * 32 < nrows;

        // Q row -> SMEM (K-major SW128); this thread writes 8 of the 16 chunks
        {
            const uint4* src = nullptr;
            if (live_row) {
                const int leaf = a.slot_leaf[U.slot_begin + j];
                src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.q) +
                                                     ((size_t)leaf * a.hq_loc + hq) * DH);
            }
#pragma unroll
            for (int c = 8 * h; c < 8 * h + 8; ++c) {
                const uint4 v = live_row ? src[c] : make_uint4(0, 0, 0, 0);
                sts128(sbase + SMEM_Q + sw128_off(r, c), v.x, v.y, v.z, v.w);
            }
        }
        fence_proxy_async();
        mbar_arrive(BAR(Q_FULL));

        float m = -INFINITY, l = 0.f;
        const float sc = a.scale_log2;
        mbar_wait(BAR(G_FULL), 0);
        for (int t = 0; t < ntiles; ++t) {
            const int ng = min(8, U.n_grp - 8 * t);
            const int g0 = 4 * h;
            mbar_wait(BAR(S_FULL), t & 1);
            if (threadIdx.x == 128) TRACE(t, 3);
            tc_fence_after();
            float sv[64];
            if (warp_live) {
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    if (g0 + g < ng) {
                        uint32_t rr[16];
                        TMEM_LD16(tmem + lane_addr + TMEM_S + (g0 + g) * 16, rr);
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
                const uint32_t* gi = g_info + 8 * t + g0;
                float mxa[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    mxa[g] = -INFINITY;
                    if (g0 + g < ng) {
                        const uint32_t info = gi[g];
                        const int cnt = (int)(info & 0xffu), b = (int)((info >> 8) & 0xfffu), e = (int)(info >> 20);
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
            // combine the two halves of the row
            red[h * BM + r] = mx;
            asm volatile("bar.sync 1, %0;" ::"n"(NSOFT) : "memory");
            mx = fmaxf(mx, red[(h ^ 1) * BM + r]) * sc;
            // lazy rescale: keep the stale max unless it grew by > kLazy (both
            // threads of a row take the same decision).  The O correction is
            // warp-collective, so a warp takes it when any of its rows needs it.
            const bool grow = mx > m + kLazy;
            float f = 1.f;
            if (grow) {
                if (m != -INFINITY) f = ex2(m - mx);
                l *= f;
                m = mx;
            }
            if (t > 0) mbar_wait(BAR(O_FULL), (t - 1) & 1);
            if (t > 0 && __any_sync(0xffffffffu, grow && f != 1.f)) {
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[16];
                    TMEM_LD16(tmem + lane_addr + TMEM_O + h * 64 + c * 16, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
                    TMEM_ST16(tmem + lane_addr + TMEM_O + h * 64 + c * 16, o);
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
            if (threadIdx.x == 128) TRACE(t, 4);
        }

        // epilogue: O / l -> partial or final output (this thread: 64 columns)
        if (ntiles > 0) {
            mbar_wait(BAR(O_FULL), (ntiles - 1) & 1);
            tc_fence_after();
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NSOFT) : "memory");  // red[] reuse
        red[h * BM + r] = l;
        asm volatile("bar.sync 1, %0;" ::"n"(NSOFT) : "memory");
        l += red[(h ^ 1) * BM + r];
        const float inv = (live_row && l > 0.f) ? 1.f / l : 0.f;
        const float lse2 = m + log2f(l);
        int pid = 0;
        if (live_row) pid = a.slot_part[U.slot_begin + j];
        if (warp_live) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t o[16];
                const int col = h * 64 + c * 16;
                TMEM_LD16(tmem + lane_addr + TMEM_O + col, o);
                tmem_wait_ld();
                if (live_row) {
                    if (pid < 0) {
                        const int leaf = -1 - pid;
                        const size_t base = ((size_t)leaf * a.hq_loc + hq) * DH + col;
                        if (a.out_bf16) {
                            uint4 w0, w1;
                            uint32_t* p0 = &w0.x;
                            uint32_t* p1 = &w1.x;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                p0[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
                                p1[i] = pack_bf16(__uint_as_float(o[8 + 2 * i]) * inv,
                                                  __uint_as_float(o[9 + 2 * i]) * inv);
                            }
                            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) + base);
                            dst[0] = w0;
                            dst[1] = w1;
                        } else {
                            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + base);
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                dst[i] = make_float4(__uint_as_float(o[4 * i]) * inv, __uint_as_float(o[4 * i + 1]) * inv,
                                                     __uint_as_float(o[4 * i + 2]) * inv,
                                                     __uint_as_float(o[4 * i + 3]) * inv);
                        }
                        if (c == 0 && h == 0 && a.lse) a.lse[(size_t)leaf * a.hq_loc + hq] = lse2 * kLn2;
                    } else {
                        float4* dst = reinterpret_cast<float4*>(a.part_o + ((size_t)pid * a.hq_loc + hq) * DH + col);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            dst[i] = make_float4(__uint_as_float(o[4 * i]) * inv, __uint_as_float(o[4 * i + 1]) * inv,
                                                 __uint_as_float(o[4 * i + 2]) * inv, __uint_as_float(o[4 * i + 3]) * inv);
                        if (c == 0 && h == 0) a.part_lse[(size_t)pid * a.hq_loc + hq] = lse2;
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (a.trace && threadIdx.x == 0) {
        long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        const int cta = blockIdx.y * gridDim.x + blockIdx.x;
        if (cta < 4096) {
            unsigned smid;
            asm("mov.u32 %0, %%smid;" : "=r"(smid));
            a.trace[512 + 4 * cta] = t_begin;
            a.trace[512 + 4 * cta + 1] = t_end;
            a.trace[512 + 4 * cta + 2] = smid;
            a.trace[512 + 4 * cta + 3] = ((long long)U.n_grp << 32) | (unsigned)nrows;
        }
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

cudaError_t launch_attn_mma(const AttnArgs& a, cudaStream_t s) {
    if (a.n_units == 0) return cudaSuccess;
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
    dim3 grid(a.n_units, a.n_kv_loc);
    attn_mma_kernel<<<grid, NTHREADS, SMEM_BYTES, s>>>(tm, a);
    return cudaGetLastError();
}

}  // namespace ta
