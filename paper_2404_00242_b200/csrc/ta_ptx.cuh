// ta_ptx.cuh -- sm_100a PTX helpers shared by the kernels (mbarriers, TMA,
// tcgen05/TMEM, PDL) and the empty-leaf fill.
#pragma once

#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>

#include "ta_kernels.h"

namespace ta {
namespace dev {

constexpr float kLn2 = 0.69314718055994530942f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ------------------------------------------------------------------ mbarrier
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

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
// bulk copy global -> shared (16-byte aligned, size a multiple of 16), completing on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// TMA prefetch of a box into L2 (no SMEM, no barrier)
__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(tmap), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------------ tcgen05
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor, SWIZZLE_128B, sm_100 version bit.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 instruction descriptor: f32 accumulate, bf16 A/B, A/B major bits.
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
// A operand from TMEM (K-major, bf16 pairs packed per 32-bit column, row = lane)
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

#define TA_TMEM_LD16(addr, r)                                                                                  \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),         \
                   "=r"(r[15])                                                                                  \
                 : "r"(addr))
#define TA_TMEM_ST16(addr, r)                                                                                  \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
                 ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])      \
                 : "memory")
#define TA_TMEM_ST8(addr, r)                                                                                   \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(r[0]), \
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])                    \
                 : "memory")
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ misc
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Programmatic dependent launch: let the next launch on the stream start its
// prologue now; wait for the previous launch's memory before touching shared
// state (queries, outputs, partials).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t;
}
// debug timeline: first start / last end of a launch (atomics on slots k, k+1)
__device__ __forceinline__ void timeline_mark(unsigned long long* tl, int k, bool start) {
    if (!tl) return;
    if (start) atomicMin(tl + k, gtimer_ns());
    else atomicMax(tl + k + 1, gtimer_ns());
}

// Store NV consecutive fp32 values (NV % 8 == 0) as the output dtype.
template <int NV>
__device__ __forceinline__ void store_row(void* out, size_t base, const float* v, float scale, int out_bf16) {
    if (out_bf16) {
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + base);
#pragma unroll
        for (int i = 0; i < NV / 8; ++i)
            dst[i] = make_uint4(pack_bf16(v[8 * i] * scale, v[8 * i + 1] * scale), pack_bf16(v[8 * i + 2] * scale, v[8 * i + 3] * scale),
                                pack_bf16(v[8 * i + 4] * scale, v[8 * i + 5] * scale), pack_bf16(v[8 * i + 6] * scale, v[8 * i + 7] * scale));
    } else {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + base);
#pragma unroll
        for (int i = 0; i < NV / 4; ++i)
            dst[i] = make_float4(v[4 * i] * scale, v[4 * i + 1] * scale, v[4 * i + 2] * scale, v[4 * i + 3] * scale);
    }
}

// tree_reduce (attention.hpp:209-233) of one merge record row (q head g of
// the record's leaf-head) by one warp: lane k < n holds partial k's log2-lse,
// every lane sums its DPL columns over the partials (ids rec.z .. rec.z +
// rec.w - 1, contiguous), 8 partials' loads in flight at a time.  Fixed
// order: the result does not depend on which CTA produced what when.
template <int DPL>
__device__ __forceinline__ void ldcg_cols(const float* p, float (&f)[DPL]) {
    if constexpr (DPL == 4) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
        f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
    } else if constexpr (DPL == 2) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(p));
        f[0] = v.x; f[1] = v.y;
    } else {
        f[0] = __ldcg(p);
    }
}

template <int DPL>
__device__ __forceinline__ void merge_record_row(const AttnArgs& a, int4 rec, int g, int lane) {
    constexpr int PB = 8;
    const int D = a.D, G = a.G;
    const int hq = rec.y * G + g;
    const bool active = lane * DPL < D;
    float acc[DPL];
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
    float M = -INFINITY, den = 0.f;
    for (int base = 0; base < rec.w; base += 32) {
        const int np = min(32, rec.w - base);
        const int p0 = rec.z + base;
        const float lp = lane < np ? __ldcg(a.part_lse + (size_t)(p0 + lane) * G + g) : -INFINITY;
        float v[PB][DPL];
#pragma unroll
        for (int u = 0; u < PB; ++u) {
            if (active && u < np) {
                ldcg_cols<DPL>(a.part_o + ((size_t)(p0 + u) * G + g) * D + lane * DPL, v[u]);
            } else {
#pragma unroll
                for (int i = 0; i < DPL; ++i) v[u][i] = 0.f;
            }
        }
        float bm = lp;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
        if (bm == -INFINITY) continue;
        const float nm = fmaxf(M, bm);
        const float rescale = M == -INFINITY ? 0.f : ex2(M - nm);
        den *= rescale;
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[i] *= rescale;
        M = nm;
        const float w = lp == -INFINITY ? 0.f : ex2(lp - M);
        float ws = w;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, off);
        den += ws;
        for (int p = 0; p < np; p += PB) {
            if (p > 0) {
#pragma unroll
                for (int u = 0; u < PB; ++u) {
                    if (active && p + u < np) {
                        ldcg_cols<DPL>(a.part_o + ((size_t)(p0 + p + u) * G + g) * D + lane * DPL, v[u]);
                    } else {
#pragma unroll
                        for (int i = 0; i < DPL; ++i) v[u][i] = 0.f;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < PB; ++u) {
                const float wu = __shfl_sync(0xffffffffu, w, (p + u) & 31);
#pragma unroll
                for (int i = 0; i < DPL; ++i) acc[i] = fmaf(p + u < np ? wu : 0.f, v[u][i], acc[i]);
            }
        }
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    const size_t ob = ((size_t)rec.x * a.hq_loc + hq) * D;
    if (active) {
        if (a.out_bf16) {
            if constexpr (DPL == 4) {
                *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.out) + ob + lane * 4) =
                    make_uint2(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv));
            } else {
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    reinterpret_cast<__nv_bfloat16*>(a.out)[ob + lane * DPL + i] = __float2bfloat16_rn(acc[i] * inv);
            }
        } else {
#pragma unroll
            for (int i = 0; i < DPL; ++i) reinterpret_cast<float*>(a.out)[ob + lane * DPL + i] = acc[i] * inv;
        }
    }
    if (lane == 0 && a.lse) a.lse[(size_t)rec.x * a.hq_loc + hq] = M == -INFINITY ? -INFINITY : (M + log2f(den)) * kLn2;
}

// Half-warp variant for D = 128: lanes [16 hw, 16 hw + 16) merge one row, 8
// columns per lane, so a warp merges two rows at once; up to 16 partials' lse
// (lane k: partial k) and 8 partials' columns in flight per round trip.
__device__ __forceinline__ void merge_record_row_half(const AttnArgs& a, int4 rec, int g, int lane16, bool active) {
    constexpr int PB = 8;
    const int G = a.G;
    const int hq = rec.y * G + g;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    float M = -INFINITY, den = 0.f;
    const int n = active ? rec.w : 0;
    const int nmax = max(n, __shfl_xor_sync(0xffffffffu, n, 16));   // the warp's two rows: one trip count
    for (int base = 0; base < nmax; base += 16) {
        const int np = max(0, min(16, n - base));
        const int p0 = rec.z + base;
        const float lp = lane16 < np ? __ldcg(a.part_lse + (size_t)(p0 + lane16) * G + g) : -INFINITY;
        float4 v[PB][2];
#pragma unroll
        for (int u = 0; u < PB; ++u) {
            if (u < np) {
                const float4* src = reinterpret_cast<const float4*>(a.part_o + ((size_t)(p0 + u) * G + g) * 128 + lane16 * 8);
                v[u][0] = __ldcg(src);
                v[u][1] = __ldcg(src + 1);
            } else {
                v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        float bm = lp;
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
        const float nm = fmaxf(M, bm);
        const float rescale = (M == -INFINITY || nm == -INFINITY) ? 0.f : ex2(M - nm);
        if (nm != -INFINITY) {
            den *= rescale;
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] *= rescale;
            M = nm;
        }
        const float w = (lp == -INFINITY || M == -INFINITY) ? 0.f : ex2(lp - M);
        float ws = w;
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, off);
        den += ws;
        for (int p = 0; p < 16; p += PB) {
            if (p > 0) {
#pragma unroll
                for (int u = 0; u < PB; ++u) {
                    if (p + u < np) {
                        const float4* src =
                            reinterpret_cast<const float4*>(a.part_o + ((size_t)(p0 + p + u) * G + g) * 128 + lane16 * 8);
                        v[u][0] = __ldcg(src);
                        v[u][1] = __ldcg(src + 1);
                    } else {
                        v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < PB; ++u) {
                const float wu = __shfl_sync(0xffffffffu, w, (threadIdx.x & 16) + ((p + u) & 15));
                const float ww = p + u < np ? wu : 0.f;
                acc[0] = fmaf(ww, v[u][0].x, acc[0]);
                acc[1] = fmaf(ww, v[u][0].y, acc[1]);
                acc[2] = fmaf(ww, v[u][0].z, acc[2]);
                acc[3] = fmaf(ww, v[u][0].w, acc[3]);
                acc[4] = fmaf(ww, v[u][1].x, acc[4]);
                acc[5] = fmaf(ww, v[u][1].y, acc[5]);
                acc[6] = fmaf(ww, v[u][1].z, acc[6]);
                acc[7] = fmaf(ww, v[u][1].w, acc[7]);
            }
        }
    }
    if (!active) return;
    const float inv = den > 0.f ? 1.f / den : 0.f;
    const size_t ob = ((size_t)rec.x * a.hq_loc + hq) * 128 + lane16 * 8;
    store_row<8>(a.out, ob, acc, inv, a.out_bf16);
    if (lane16 == 0 && a.lse) a.lse[(size_t)rec.x * a.hq_loc + hq] = M == -INFINITY ? -INFINITY : (M + log2f(den)) * kLn2;
}

// Leaf-heads whose path holds no tokens: out = 0, lse = -inf (they are
// absent from the reference's AttentionOutput).  `nl` lanes (ids 0..nl-1) of
// one warp, strided over CTAs.
__device__ __forceinline__ void fill_empty(const AttnArgs& a, int lane, int nl = 32) {
    const int n_empty = a.counts->n_empty;
    for (int e = blockIdx.x; e < n_empty; e += gridDim.x) {
        const int leaf = a.empty[2 * e], head = a.empty[2 * e + 1];
        const size_t base = ((size_t)leaf * a.hq_loc + (size_t)head * a.G) * a.D;
        for (int i = lane; i < a.G * a.D; i += nl) {
            if (a.out_bf16)
                reinterpret_cast<__nv_bfloat16*>(a.out)[base + i] = __float2bfloat16_rn(0.f);
            else
                reinterpret_cast<float*>(a.out)[base + i] = 0.f;
        }
        if (a.lse)
            for (int g = lane; g < a.G; g += nl) a.lse[(size_t)leaf * a.hq_loc + head * a.G + g] = -INFINITY;
    }
}

}  // namespace dev
}  // namespace ta
