// attn_fma.cu -- FMA path of the chunk attention (sparse chunks, fp32 KV),
// the split-K (m, l, O) merge, and the KV scatter used by ta_kv_write.
//
// Reference semantics: group_attention (attention.hpp:117-204) computes, per
// query and head, an online softmax over the group's tokens whose mask bit
// is set; tree_reduce (attention.hpp:209-233) merges a query's partials by
// LSE weighting.  Here one CTA runs a whole unit (a span of consecutive
// flatten chunks for a block of query slots and one kv head): the KV rows
// are staged in shared memory once with cp.async (double-buffered tiles of
// TT tokens), and every (slot, q-head) row that shares the tile consumes
// them.  The mask is the slot range [b, e) per token (a contiguous run, as
// every reference mask word is).  Each warp owns TT/8 tokens of every tile
// and keeps its own running (m, l, O) for all rows; warps are merged once at
// the end of the unit, so nothing leaves the SM per chunk.
#include <cuda_bf16.h>

#include <cfloat>
#include <cmath>

#include "ta_kernels.h"

namespace ta {
namespace {

constexpr float kLn2 = 0.69314718055994530942f;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ void load8(const float* p, float (&f)[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0];
    const float4 b = reinterpret_cast<const float4*>(p)[1];
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 x = __bfloat1622float2(h[i]);
        f[2 * i] = x.x;
        f[2 * i + 1] = x.y;
    }
}

template <int N>
__device__ __forceinline__ void loadN(const float* p, float (&f)[N]) {
    if constexpr (N == 4) {
        const float4 a = *reinterpret_cast<const float4*>(p);
        f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    } else if constexpr (N == 2) {
        const float2 a = *reinterpret_cast<const float2*>(p);
        f[0] = a.x; f[1] = a.y;
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) f[i] = p[i];
    }
}
template <int N>
__device__ __forceinline__ void loadN(const __nv_bfloat16* p, float (&f)[N]) {
    if constexpr (N == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(p);
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
    } else if constexpr (N == 2) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
        f[0] = a.x; f[1] = a.y;
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) f[i] = __bfloat162float(p[i]);
    }
}

__device__ __forceinline__ void store_out(void* out, size_t idx, float v, int bf16) {
    if (bf16)
        reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
    else
        reinterpret_cast<float*>(out)[idx] = v;
}

template <typename T, int D>
struct FmaCfg {
    static constexpr int NW = 8;
    static constexpr int TT_RAW = 65536 / (2 * D * (int)sizeof(T));
    static constexpr int TT = TT_RAW < 512 ? TT_RAW : 512;   // tokens per tile
    static constexpr int TPW = TT / NW;                       // tokens per warp
    static constexpr int DQ = D < 32 ? D : 32;                // dims per lane (QK)
    static constexpr int LPT = D / DQ;                        // lanes per token
    static constexpr int NT = TPW * LPT / 32;                 // tokens per lane
    static constexpr int ROWE = D + 16 / (int)sizeof(T);      // padded smem row
    static constexpr int DPL = D >= 32 ? D / 32 : 1;          // dims per lane (PV)
    static constexpr int PVL = D / DPL;                       // active PV lanes
    static constexpr int CPR = D * (int)sizeof(T) / 16;       // 16-byte chunks per row
    static_assert(NT >= 1 && TPW * LPT % 32 == 0, "tile shape");
    static_assert(DQ % 8 == 0, "D must be a multiple of 8");
};

template <typename T, int D, int R>
constexpr size_t fma_smem_bytes() {
    using C = FmaCfg<T, D>;
    size_t kv = 2ull * 2 * C::TT * C::ROWE * sizeof(T);
    size_t be = 2ull * C::TT * 4;
    size_t qs = (size_t)R * C::LPT * (C::DQ + 4) * 4;
    size_t pb = (size_t)C::NW * C::TPW * R * 4;
    size_t comb = (size_t)C::NW * R * (D + 2) * 4;
    size_t a = kv + be + qs + pb;
    return a > comb ? a : comb;
}

template <typename T, int D, int R>
__global__ void __launch_bounds__(256, 1) attn_fma_kernel(const AttnArgs a) {
    using C = FmaCfg<T, D>;
    constexpr int TT = C::TT, TPW = C::TPW, DQ = C::DQ, LPT = C::LPT, NT = C::NT, ROWE = C::ROWE;
    constexpr int DPL = C::DPL, CPR = C::CPR, EPC = 16 / (int)sizeof(T);
    extern __shared__ __align__(16) uint8_t smem[];
    T* Ks = reinterpret_cast<T*>(smem);
    T* Vs = Ks + 2 * TT * ROWE;
    uint32_t* be_s = reinterpret_cast<uint32_t*>(Vs + 2 * TT * ROWE);
    float* qs = reinterpret_cast<float*>(be_s + 2 * TT);
    float* pbuf = qs + R * LPT * (DQ + 4);

    const int kvh = blockIdx.y;
    const UnitDesc U = a.units[blockIdx.x];
    const int G = a.G;
    const int nrows = U.n_slots * G;
    const T* kb = reinterpret_cast<const T*>(a.k) + (size_t)kvh * a.head_stride;
    const T* vb = reinterpret_cast<const T*>(a.v) + (size_t)kvh * a.head_stride;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // queries of the unit's rows, pre-scaled by log2(e)/sqrt(D)
    for (int i = tid; i < R * D; i += 256) {
        const int r = i / D, d = i % D;
        float v = 0.f;
        if (r < nrows) {
            const int leaf = a.slot_leaf[U.slot_begin + r / G];
            const int hq = kvh * G + r % G;
            v = to_f(reinterpret_cast<const T*>(a.q)[((size_t)leaf * a.hq_loc + hq) * D + d]) * a.scale_log2;
        }
        qs[(r * LPT + d / DQ) * (DQ + 4) + d % DQ] = v;
    }

    auto issue = [&](int tile, int st) {
        const int t0 = tile * TT;
        const int nv = min(TT, U.n_tokens - t0);
        const int32_t* rows = a.tok_row + U.tok_begin + t0;
        for (int c = tid; c < nv * CPR; c += 256) {
            const int row = c / CPR, ch = c % CPR;
            const size_t g = (size_t)rows[row] * D + ch * EPC;
            cp_async16(Ks + (st * TT + row) * ROWE + ch * EPC, kb + g);
            cp_async16(Vs + (st * TT + row) * ROWE + ch * EPC, vb + g);
        }
        for (int t = tid; t < TT; t += 256) be_s[st * TT + t] = t < nv ? a.tok_be[U.tok_begin + t0 + t] : 0u;
        cp_async_commit();
    };

    float m[R], l[R], acc[R][DPL];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[r][i] = 0.f;
    }

    const int tl = lane / LPT, part = lane % LPT;
    const int ntiles = (U.n_tokens + TT - 1) / TT;
    issue(0, 0);
    for (int it = 0; it < ntiles; ++it) {
        const int st = it & 1;
        if (it + 1 < ntiles) {
            issue(it + 1, st ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int nv = min(TT, U.n_tokens - it * TT);
        const T* Kst = Ks + st * TT * ROWE;
        const T* Vst = Vs + st * TT * ROWE;
        const uint32_t* bes = be_s + st * TT;

        // ---- scores: lane group (tl) owns NT tokens, LPT lanes split D
        float s[NT][R];
#pragma unroll
        for (int k = 0; k < NT; ++k)
#pragma unroll
            for (int r = 0; r < R; ++r) s[k][r] = 0.f;
#pragma unroll
        for (int dc = 0; dc < DQ / 8; ++dc) {
            float kf[NT][8];
#pragma unroll
            for (int k = 0; k < NT; ++k) {
                const int tok = warp * TPW + tl + k * (32 / LPT);
                load8(Kst + tok * ROWE + part * DQ + dc * 8, kf[k]);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (r < nrows) {
                    const float* qp = qs + (r * LPT + part) * (DQ + 4) + dc * 8;
                    const float4 qa = *reinterpret_cast<const float4*>(qp);
                    const float4 qb = *reinterpret_cast<const float4*>(qp + 4);
#pragma unroll
                    for (int k = 0; k < NT; ++k)
                        s[k][r] += kf[k][0] * qa.x + kf[k][1] * qa.y + kf[k][2] * qa.z + kf[k][3] * qa.w +
                                   kf[k][4] * qb.x + kf[k][5] * qb.y + kf[k][6] * qb.z + kf[k][7] * qb.w;
                }
            }
        }
#pragma unroll
        for (int off = 1; off < LPT; off <<= 1)
#pragma unroll
            for (int k = 0; k < NT; ++k)
#pragma unroll
                for (int r = 0; r < R; ++r) s[k][r] += __shfl_xor_sync(0xffffffffu, s[k][r], off);

        // ---- tree mask: token attended by slots [b, e)
#pragma unroll
        for (int k = 0; k < NT; ++k) {
            const int tok = warp * TPW + tl + k * (32 / LPT);
            const uint32_t be = bes[tok];
            const int b = (int)(be & 0xffffu), e = (int)(be >> 16);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int j = r / G;
                if (j < b || j >= e) s[k][r] = -INFINITY;
            }
        }

        // ---- online softmax (base 2), per warp running state
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r < nrows) {
                float tm = s[0][r];
#pragma unroll
                for (int k = 1; k < NT; ++k) tm = fmaxf(tm, s[k][r]);
#pragma unroll
                for (int off = LPT; off < 32; off <<= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, off));
                if (tm > m[r]) {
                    const float alpha = exp2f(m[r] - tm);
                    l[r] *= alpha;
#pragma unroll
                    for (int i = 0; i < DPL; ++i) acc[r][i] *= alpha;
                    m[r] = tm;
                }
                const bool live = m[r] != -INFINITY;
#pragma unroll
                for (int k = 0; k < NT; ++k) {
                    const float p = live ? exp2f(s[k][r] - m[r]) : 0.f;
                    if (part == 0) {
                        l[r] += p;
                        pbuf[(warp * TPW + tl + k * (32 / LPT)) * R + r] = p;
                    }
                }
            }
        }
        __syncwarp();

        // ---- O += P V : lane owns DPL output dims
        const int ntw = min(TPW, nv - warp * TPW);
        if (lane < C::PVL) {
            for (int tw = 0; tw < ntw; ++tw) {
                const int tok = warp * TPW + tw;
                float vf[DPL];
                loadN<DPL>(Vst + tok * ROWE + lane * DPL, vf);
                const float* pp = pbuf + (warp * TPW + tw) * R;
#pragma unroll
                for (int r4 = 0; r4 < R; r4 += 4) {
                    if (r4 < nrows) {
                        const float4 p4 = *reinterpret_cast<const float4*>(pp + r4);
                        const float pr[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
                        for (int q = 0; q < 4; ++q)
#pragma unroll
                            for (int i = 0; i < DPL; ++i) acc[r4 + q][i] += pr[q] * vf[i];
                    }
                }
            }
        }
        __syncwarp();
        __syncthreads();
    }

    // ---- merge the 8 warps' states, then write partial or final output
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) l[r] += __shfl_xor_sync(0xffffffffu, l[r], off);
    float* acc_s = reinterpret_cast<float*>(smem);
    float* m_s = acc_s + C::NW * R * D;
    float* l_s = m_s + C::NW * R;
    if (lane < C::PVL) {
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (r < nrows)
#pragma unroll
                for (int i = 0; i < DPL; ++i) acc_s[(warp * R + r) * D + lane * DPL + i] = acc[r][i];
    }
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            m_s[warp * R + r] = m[r];
            l_s[warp * R + r] = l[r];
        }
    }
    __syncthreads();
    for (int idx = tid; idx < nrows * D; idx += 256) {
        const int r = idx / D, d = idx % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < C::NW; ++w) M = fmaxf(M, m_s[w * R + r]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < C::NW; ++w) {
            const float mw = m_s[w * R + r];
            if (mw != -INFINITY) {
                const float sc = exp2f(mw - M);
                L += l_s[w * R + r] * sc;
                O += acc_s[(w * R + r) * D + d] * sc;
            }
        }
        O = O / L;
        const float lse2 = M + log2f(L);
        const int j = r / G, hq = kvh * G + r % G;
        const int pid = a.slot_part[U.slot_begin + j];
        if (pid < 0) {
            const int leaf = -1 - pid;
            store_out(a.out, ((size_t)leaf * a.hq_loc + hq) * D + d, O, a.out_bf16);
            if (d == 0 && a.lse) a.lse[(size_t)leaf * a.hq_loc + hq] = lse2 * kLn2;
        } else {
            a.part_o[((size_t)pid * a.hq_loc + hq) * D + d] = O;
            if (d == 0) a.part_lse[(size_t)pid * a.hq_loc + hq] = lse2;
        }
    }
}

template <typename T, int D, int R>
cudaError_t launch_fma_t(const AttnArgs& a, cudaStream_t s) {
    constexpr size_t smem = fma_smem_bytes<T, D, R>();
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_fma_kernel<T, D, R>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid(a.n_units, a.n_kv_loc);
    attn_fma_kernel<T, D, R><<<grid, 256, smem, s>>>(a);
    return cudaGetLastError();
}

template <typename T, int R>
cudaError_t launch_fma_d(const AttnArgs& a, cudaStream_t s) {
    switch (a.D) {
        case 16: return launch_fma_t<T, 16, R>(a, s);
        case 32: return launch_fma_t<T, 32, R>(a, s);
        case 64: return launch_fma_t<T, 64, R>(a, s);
        case 128: return launch_fma_t<T, 128, R>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

// ---------------------------------------------------------------------------
// Split-K merge (tree_reduce, attention.hpp:209-233) for leaves covered by
// more than one unit; partials are consumed in a fixed (unit) order so the
// result is independent of CTA scheduling.
template <int DPL>
__device__ __forceinline__ void load_dpl(const float* p, float (&f)[DPL]) {
    if constexpr (DPL == 4) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
    } else if constexpr (DPL == 2) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        f[0] = v.x; f[1] = v.y;
    } else {
        f[0] = p[0];
    }
}

// one warp per (merged leaf, q head); lane p fetches partial p's id and lse
// (all in flight at once), weights are broadcast by shuffle, and the O loads
// of all partials are independent (no dependent-load chain).  Lane i owns
// output dims [i*DPL, (i+1)*DPL) (D < 32: lanes >= D idle).
template <int DPL>
__global__ void __launch_bounds__(256) merge_kernel(const MergeArgs a) {
    const int wid = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (wid >= a.n_merge * a.hq_loc) return;
    const int mi = wid / a.hq_loc, hq = wid % a.hq_loc;
    const int leaf = a.merge_leaf[mi];
    const int p0 = a.merge_begin[mi], p1 = a.merge_begin[mi + 1];
    const int D = a.D;
    const bool active = lane * DPL < D;
    float acc[DPL];
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
    float M = -INFINITY, den = 0.f;
    for (int base = p0; base < p1; base += 32) {
        const int np = min(32, p1 - base);
        int pid = 0;
        float lp = -INFINITY;
        if (lane < np) {
            pid = a.merge_parts[base + lane];
            lp = a.part_lse[(size_t)pid * a.hq_loc + hq];
        }
        float bm = lp;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
        if (bm == -INFINITY) continue;
        const float nm = fmaxf(M, bm);
        const float rescale = M == -INFINITY ? 0.f : exp2f(M - nm);
        den *= rescale;
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[i] *= rescale;
        M = nm;
        const float w = lp == -INFINITY ? 0.f : exp2f(lp - M);
        float ws = w;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, off);
        den += ws;
        int p = 0;
        for (; p + 4 <= np; p += 4) {
            float v[4][DPL];
            float wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int id = __shfl_sync(0xffffffffu, pid, p + u);
                wv[u] = __shfl_sync(0xffffffffu, w, p + u);
                if (active) load_dpl<DPL>(a.part_o + ((size_t)id * a.hq_loc + hq) * D + lane * DPL, v[u]);
            }
            if (active)
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int i = 0; i < DPL; ++i) acc[i] += wv[u] * v[u][i];
        }
        for (; p < np; ++p) {
            const int id = __shfl_sync(0xffffffffu, pid, p);
            const float wp = __shfl_sync(0xffffffffu, w, p);
            if (active) {
                float v[DPL];
                load_dpl<DPL>(a.part_o + ((size_t)id * a.hq_loc + hq) * D + lane * DPL, v);
#pragma unroll
                for (int i = 0; i < DPL; ++i) acc[i] += wp * v[i];
            }
        }
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    const size_t base = ((size_t)leaf * a.hq_loc + hq) * D;
    if (active)
#pragma unroll
        for (int i = 0; i < DPL; ++i) store_out(a.out, base + lane * DPL + i, acc[i] * inv, a.out_bf16);
    if (lane == 0 && a.lse) a.lse[(size_t)leaf * a.hq_loc + hq] = M == -INFINITY ? -INFINITY : (M + log2f(den)) * kLn2;
}

// ---------------------------------------------------------------------------
// KV scatter: src rows [n][n_loc][D] -> pool rows (page*P + slot) per head.
__global__ void kv_scatter_kernel(const uint4* __restrict__ sk, const uint4* __restrict__ sv,
                                  uint4* __restrict__ dk, uint4* __restrict__ dv,
                                  const int32_t* __restrict__ rows, int n, int n_loc,
                                  int64_t head_stride_v, int row_v) {
    const int64_t total = (int64_t)n * n_loc * row_v;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % row_v);
        const int64_t th = i / row_v;
        const int h = (int)(th % n_loc);
        const int t = (int)(th / n_loc);
        const int64_t dst = h * head_stride_v + (int64_t)rows[t] * row_v + c;
        dk[dst] = sk[i];
        dv[dst] = sv[i];
    }
}

}  // namespace

cudaError_t launch_attn_fma(const AttnArgs& a, int max_rows, cudaStream_t s) {
    if (a.n_units == 0) return cudaSuccess;
    if (max_rows <= 8) return a.kv_bf16 ? launch_fma_d<__nv_bfloat16, 8>(a, s) : launch_fma_d<float, 8>(a, s);
    return a.kv_bf16 ? launch_fma_d<__nv_bfloat16, 16>(a, s) : launch_fma_d<float, 16>(a, s);
}

cudaError_t launch_merge(const MergeArgs& a, cudaStream_t s) {
    if (a.n_merge == 0) return cudaSuccess;
    const int warps = a.n_merge * a.hq_loc;
    const int blocks = (warps + 7) / 8;
    if (a.D >= 128) merge_kernel<4><<<blocks, 256, 0, s>>>(a);
    else if (a.D >= 64) merge_kernel<2><<<blocks, 256, 0, s>>>(a);
    else merge_kernel<1><<<blocks, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_kv_scatter(const void* src_k, const void* src_v, void* dst_k, void* dst_v,
                              const int32_t* rows, int n, int n_loc, int64_t head_stride, int D,
                              int esize, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int row_v = D * esize / 16;
    const int64_t hs_v = head_stride * esize / 16;
    const int64_t total = (int64_t)n * n_loc * row_v;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    kv_scatter_kernel<<<blocks, 256, 0, s>>>((const uint4*)src_k, (const uint4*)src_v, (uint4*)dst_k,
                                             (uint4*)dst_v, rows, n, n_loc, hs_v, row_v);
    return cudaGetLastError();
}

}  // namespace ta
