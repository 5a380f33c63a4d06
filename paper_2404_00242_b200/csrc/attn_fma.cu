// attn_fma.cu -- persistent warp-FMA chunk attention (fp32 or bf16 KV, any
// supported D, <= 8 or 16 rows per lane) and the KV scatter of ta_kv_write.
//
// Same schedule as the tcgen05 kernel (items of tiles of 16-row groups, see
// ta_internal.h), for sparse lanes and for dtypes / head dims the tensor-core
// path does not take.  A CTA (8 warps) stages each tile's K/V rows in SMEM
// once (cp.async, 2 stages); warp w owns tokens [w*TPW, (w+1)*TPW) of every
// tile (in sub-batches of SB = 64/R tokens) and keeps its own running
// (m, l, O) for all rows of the item:
//   QK   lane owns D/32 dims; the SB x R partial dot products are reduced
//        across the warp by a butterfly transpose-reduction (one shuffle per
//        dot product), leaving each lane with whole scores
//   mask token >= group count, or row's slot outside the group's [b, e)
//   P    exp2 online softmax; P goes through a per-warp SMEM buffer and is
//        read back as broadcasts for O += P V (lane owns D/32 dims)
// The warps' states are merged once per item, then written as the final
// output or as a partial record for merge.cu.
//
// Reference semantics: group_attention (attention.hpp:117-204) and
// tree_reduce (attention.hpp:209-233).
#include <algorithm>
#include <cfloat>

#include "ta_ptx.cuh"

namespace ta {
namespace {

using namespace dev;

__device__ __forceinline__ void cp_async16(uint32_t s, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
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
        f[0] = p[0];
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
        f[0] = __bfloat162float(p[0]);
    }
}

template <typename T, int D>
struct FmaCfg {
    static constexpr int NW = 8;
    static constexpr int TG0 = 32768 / (16 * D * (int)sizeof(T));
    static constexpr int TG = TG0 < 8 ? TG0 : 8;              // groups per tile (= fma_tile_groups)
    static constexpr int TROWS = 16 * TG;                     // rows per tile stage
    static constexpr int TPW = TROWS / NW;                    // tokens per warp per tile
    static constexpr int DPL = D >= 32 ? D / 32 : 1;          // dims per lane
    static constexpr int CPR = D * (int)sizeof(T) / 16;       // 16-byte chunks per row
    static_assert(TG >= 1 && TPW >= 1, "tile shape");
};

constexpr int FMAXI = 32, FMAXT = 48;   // staged items / tiles per CTA (the rest read from global)
constexpr size_t FMETA_BYTES = FMAXI * 32 + 256 + FMAXT * (16 + 64);

template <typename T, int D, int R>
constexpr size_t fma_smem_bytes() {
    using C = FmaCfg<T, D>;
    return 2ull * 2 * C::TROWS * D * sizeof(T)            // K, V stages
           + (size_t)C::NW * 64 * 4                       // P buffers (64 per warp)
           + (size_t)C::NW * R * (D + 2) * 4              // warp combine
           + FMETA_BYTES;                                 // staged schedule
}

template <typename T, int D, int R>
__global__ void __launch_bounds__(256, 1) attn_fma_kernel(const AttnArgs a) {
    using C = FmaCfg<T, D>;
    constexpr int NW = C::NW, TROWS = C::TROWS, TPW = C::TPW, DPL = C::DPL, CPR = C::CPR;
    constexpr int SB = 64 / R < TPW ? 64 / R : TPW;   // tokens per sub-batch (64 dot products)
    static_assert(TPW % SB == 0, "sub-batches");
    constexpr int NV = SB * R;                  // partial dots per lane before the reduction
    constexpr int VPL = NV / 32;                // whole scores per lane after it
    static_assert(NV % 32 == 0 && VPL >= 1, "SB * R must be a multiple of 32");
    static_assert(R % VPL == 0, "rows per lane");
    constexpr int RCLS = R / VPL;               // lanes l, l + RCLS, ... hold the same rows
    extern __shared__ __align__(16) uint8_t smem[];
    T* Ks = reinterpret_cast<T*>(smem);
    T* Vs = Ks + 2 * TROWS * D;
    float* pbuf = reinterpret_cast<float*>(Vs + 2 * TROWS * D);
    float* acc_s = pbuf + NW * 64;
    float* m_s = acc_s + NW * R * D;
    float* l_s = m_s + NW * R;

    ItemDesc* s_item = reinterpret_cast<ItemDesc*>(l_s + NW * R);
    int* s_ioff = reinterpret_cast<int*>(s_item + FMAXI);
    TileDesc* s_td = reinterpret_cast<TileDesc*>(s_ioff + 64);
    TileMeta* s_tm = reinterpret_cast<TileMeta*>(s_td + FMAXT);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int it0 = a.cta_begin[blockIdx.x], it1 = a.cta_begin[blockIdx.x + 1];
    const int n_items = it1 - it0;
    const int G = a.G;
    // stage the CTA's schedule (host-written: read before the dependency wait)
    const int ni_s = min(n_items, FMAXI);
    for (int k = tid; k < ni_s; k += 256) s_item[k] = a.items[it0 + k];
    __syncthreads();
    if (tid == 0) {
        int off = 0;
        for (int k = 0; k < ni_s; ++k) {
            s_ioff[k] = off;
            off += s_item[k].tile_end - s_item[k].tile_begin;
        }
        s_ioff[ni_s] = off;
    }
    __syncthreads();
    const int nt_s = min(s_ioff[ni_s], FMAXT);
    for (int x = tid; x < nt_s; x += 256) {
        int k = 0;
        while (s_ioff[k + 1] <= x) ++k;
        const int t = s_item[k].tile_begin + x - s_ioff[k];
        s_td[x] = a.tiles[t];
        s_tm[x] = a.tile_meta[t];
    }
    __syncthreads();
    auto item_at = [&](int k) -> ItemDesc { return k < FMAXI ? s_item[k] : a.items[it0 + k]; };
    auto td_at = [&](int lt, int t) -> TileDesc { return lt < nt_s ? s_td[lt] : a.tiles[t]; };
    auto tm_at = [&](int lt, int t) -> const TileMeta* { return lt < nt_s ? &s_tm[lt] : &a.tile_meta[t]; };
    pdl_launch_dependents();
    pdl_wait();
    if (warp == NW - 1) fill_empty(a, lane);
    if (n_items == 0) return;

    // cp.async of one tile's K/V rows into stage st (tile t of item k, CTA tile lt)
    auto issue = [&](int k, int t, int lt, int st) {
        const ItemDesc I = item_at(k);
        const TileDesc td = td_at(lt, t);
        const TileMeta* tmp = tm_at(lt, t);
        const T* kb = reinterpret_cast<const T*>(a.k) + (size_t)I.head * a.head_stride;
        const T* vb = reinterpret_cast<const T*>(a.v) + (size_t)I.head * a.head_stride;
        const uint32_t ks = smem_u32(Ks + st * TROWS * D), vs = smem_u32(Vs + st * TROWS * D);
        for (int c = tid; c < td.ng * 16 * CPR; c += 256) {
            const int rr = c / CPR, ch = c % CPR;
            if ((rr & 15) >= (int)(tmp->info[rr >> 4] & 0xffu)) continue;
            const size_t g = ((size_t)tmp->row[rr >> 4] + (rr & 15)) * D;
            cp_async16(ks + (uint32_t)(rr * D * sizeof(T) + ch * 16), reinterpret_cast<const uint8_t*>(kb + g) + ch * 16);
            cp_async16(vs + (uint32_t)(rr * D * sizeof(T) + ch * 16), reinterpret_cast<const uint8_t*>(vb + g) + ch * 16);
        }
        cp_async_commit();
    };
    // (item, tile) cursor of the next tile to stage (runs ahead across items)
    int nx_k = 0, nx_t = item_at(0).tile_begin, nx_lt = 0;
    auto advance = [&]() {
        ++nx_lt;
        if (++nx_t >= item_at(nx_k).tile_end && ++nx_k < n_items) nx_t = item_at(nx_k).tile_begin;
    };
    issue(nx_k, nx_t, nx_lt, 0);
    advance();
    int gt = 0;

    for (int ii = 0; ii < n_items; ++ii) {
        const ItemDesc I = item_at(ii);
        const int nrows = I.n_slots * G;
        // queries of the item's rows in registers, pre-scaled by log2(e)/sqrt(D)
        float q[R][DPL];
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int i = 0; i < DPL; ++i) q[r][i] = 0.f;
            if (r < nrows && lane * DPL < D) {
                const int leaf = a.slot_leaf[I.slot_begin + r / G];
                loadN<DPL>(reinterpret_cast<const T*>(a.q) + ((size_t)leaf * a.hq_loc + I.head * G + r % G) * D +
                               lane * DPL,
                           q[r]);
#pragma unroll
                for (int i = 0; i < DPL; ++i) q[r][i] *= a.scale_log2;
            }
        }
        float m[R], acc[R][DPL], lsum[VPL];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            m[r] = -INFINITY;
#pragma unroll
            for (int i = 0; i < DPL; ++i) acc[r][i] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < VPL; ++k) lsum[k] = 0.f;

        for (int t = I.tile_begin; t < I.tile_end; ++t, ++gt) {
            const int st = gt & 1;
            if (nx_k < n_items) {
                issue(nx_k, nx_t, nx_lt, st ^ 1);
                advance();
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const TileDesc td = td_at(gt, t);
            const int grp = (warp * TPW) >> 4, c0 = (warp * TPW) & 15;
            const uint32_t info = grp < td.ng ? tm_at(gt, t)->info[grp] : 0u;
            const int cnt = max(0, min(TPW, (int)(info & 0xffu) - c0));    // valid tokens of this warp
            const int b = (int)((info >> 8) & 0xfffu), e = (int)(info >> 20);
            const T* Kst = Ks + (st * TROWS + warp * TPW) * D;
            const T* Vst = Vs + (st * TROWS + warp * TPW) * D;
            for (int sb = 0; sb < cnt; sb += SB) {
                const int cnt_sb = min(SB, cnt - sb);
                // ---- partial dots v[tok * R + r] over this lane's dims
                float v[NV];
#pragma unroll
                for (int tk = 0; tk < SB; ++tk) {
                    float kf[DPL];
                    if (tk < cnt_sb && lane * DPL < D) {
                        loadN<DPL>(Kst + (sb + tk) * D + lane * DPL, kf);
                    } else {
#pragma unroll
                        for (int i = 0; i < DPL; ++i) kf[i] = 0.f;
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        float s = 0.f;
#pragma unroll
                        for (int i = 0; i < DPL; ++i) s = fmaf(q[r][i], kf[i], s);
                        v[tk * R + r] = s;
                    }
                }
                // ---- butterfly transpose-reduction: lane l ends with v[l*VPL .. +VPL)
#pragma unroll
                for (int st5 = 0; st5 < 5; ++st5) {
                    const int off = 16 >> st5, n = NV >> st5;
                    const bool upper = (lane & off) != 0;
#pragma unroll
                    for (int i = 0; i < NV / 2; ++i) {
                        if (i < n / 2) {
                            const float send = upper ? v[i] : v[i + n / 2];
                            const float keep = upper ? v[i + n / 2] : v[i];
                            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                        }
                    }
                }
                // ---- mask; my values: index l*VPL + k -> (token, row)
                float mx[VPL];
#pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    const int idx = lane * VPL + k;
                    const int tk = idx / R, r = idx % R;
                    const int jj = r / G;
                    const bool ok = tk < cnt_sb && r < nrows && jj >= b && jj < e;
                    v[k] = ok ? v[k] : -INFINITY;
                    mx[k] = v[k];
                }
#pragma unroll
                for (int off = RCLS; off < 32; off <<= 1)
#pragma unroll
                    for (int k = 0; k < VPL; ++k) mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
                // ---- online softmax: every lane learns every row's new max
                float alpha_mine[VPL], m_mine[VPL];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float tmx = __shfl_sync(0xffffffffu, mx[r % VPL], r / VPL);
                    const float nm = fmaxf(m[r], tmx);
                    const float alpha = (nm == -INFINITY) ? 1.f : ex2(m[r] - nm);
#pragma unroll
                    for (int i = 0; i < DPL; ++i) acc[r][i] *= alpha;
                    m[r] = nm;
#pragma unroll
                    for (int k = 0; k < VPL; ++k)
                        if ((lane * VPL + k) % R == r) {
                            alpha_mine[k] = alpha;
                            m_mine[k] = nm;
                        }
                }
                float* pw = pbuf + warp * SB * R;
#pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    const float p = v[k] == -INFINITY ? 0.f : ex2(v[k] - m_mine[k]);
                    lsum[k] = lsum[k] * alpha_mine[k] + p;
                    pw[lane * VPL + k] = p;
                }
                __syncwarp();
                // ---- O += P V
                if (lane * DPL < D) {
                    for (int tk = 0; tk < cnt_sb; ++tk) {
                        float vf[DPL];
                        loadN<DPL>(Vst + (sb + tk) * D + lane * DPL, vf);
#pragma unroll
                        for (int r4 = 0; r4 < R; r4 += 4) {
                            const float4 p4 = *reinterpret_cast<const float4*>(pw + tk * R + r4);
                            const float pr[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u)
#pragma unroll
                                for (int i = 0; i < DPL; ++i) acc[r4 + u][i] = fmaf(pr[u], vf[i], acc[r4 + u][i]);
                        }
                    }
                }
                __syncwarp();
            }
            __syncthreads();   // stage st is refilled by the next issue
        }

        // ---- merge the warps' states
#pragma unroll
        for (int k = 0; k < VPL; ++k)
#pragma unroll
            for (int off = RCLS; off < 32; off <<= 1) lsum[k] += __shfl_xor_sync(0xffffffffu, lsum[k], off);
        if (lane * DPL < D)
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int i = 0; i < DPL; ++i) acc_s[(warp * R + r) * D + lane * DPL + i] = acc[r][i];
        if (lane < RCLS)
#pragma unroll
            for (int k = 0; k < VPL; ++k) l_s[warp * R + (lane * VPL + k) % R] = lsum[k];
        if (lane == 0)
#pragma unroll
            for (int r = 0; r < R; ++r) m_s[warp * R + r] = m[r];
        __syncthreads();
        for (int idx = tid; idx < nrows * D; idx += 256) {
            const int r = idx / D, d = idx % D;
            const int j = r / G, gq = r % G;
            const int code = a.slot_out[I.out_begin + j];
            if (code == kSlotUnused) continue;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < NW; ++w) M = fmaxf(M, m_s[w * R + r]);
            float L = 0.f, O = 0.f;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const float mw = m_s[w * R + r];
                if (mw != -INFINITY) {
                    const float s = ex2(mw - M);
                    L += l_s[w * R + r] * s;
                    O += acc_s[(w * R + r) * D + d] * s;
                }
            }
            O = L > 0.f ? O / L : 0.f;
            const float lse2 = M + log2f(L);
            const int hq = I.head * G + gq;
            if (code < 0) {
                const int leaf = -1 - code;
                const size_t o = ((size_t)leaf * a.hq_loc + hq) * D + d;
                if (a.out_bf16)
                    reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(O);
                else
                    reinterpret_cast<float*>(a.out)[o] = O;
                if (d == 0 && a.lse) a.lse[(size_t)leaf * a.hq_loc + hq] = lse2 * kLn2;
            } else {
                a.part_o[((size_t)code * G + gq) * D + d] = O;
                if (d == 0) a.part_lse[(size_t)code * G + gq] = lse2;
            }
        }
        __syncthreads();   // acc_s / m_s / l_s reuse
    }
}

template <typename T, int D, int R>
cudaError_t launch_fma_t(const AttnArgs& a, bool pdl, cudaStream_t s) {
    constexpr size_t smem = fma_smem_bytes<T, D, R>();
    cudaError_t e = set_smem_attr_once((const void*)attn_fma_kernel<T, D, R>, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.n_ctas);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, attn_fma_kernel<T, D, R>, a);
}

template <typename T, int R>
cudaError_t launch_fma_d(const AttnArgs& a, bool pdl, cudaStream_t s) {
    switch (a.D) {
        case 8: return launch_fma_t<T, 8, R>(a, pdl, s);
        case 16: return launch_fma_t<T, 16, R>(a, pdl, s);
        case 32: return launch_fma_t<T, 32, R>(a, pdl, s);
        case 64: return launch_fma_t<T, 64, R>(a, pdl, s);
        case 128: return launch_fma_t<T, 128, R>(a, pdl, s);
        default: return cudaErrorInvalidValue;
    }
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

// ta_kv_append: n = counts->n_append rows, read on the device (a captured
// decode step stays valid as the number of new tokens changes)
__global__ void kv_append_kernel(const uint4* __restrict__ sk, const uint4* __restrict__ sv, uint4* __restrict__ dk,
                                 uint4* __restrict__ dv, const int32_t* __restrict__ rows,
                                 const DevCounts* __restrict__ counts, int n_loc, int64_t head_stride_v, int row_v) {
    // the next launch (this layer's attention) may start its prologue now; the
    // sources (the caller's K/V projection) are ready once the previous launch is
    pdl_launch_dependents();
    const int64_t total = (int64_t)counts->n_append * n_loc * row_v;
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
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

cudaError_t launch_kv_append(const void* src_k, const void* src_v, void* dst_k, void* dst_v, const int32_t* rows,
                             const DevCounts* counts, int n_loc, int64_t head_stride, int D, int esize, int n_sms,
                             cudaStream_t s) {
    const int row_v = D * esize / 16;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * n_sms);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kv_append_kernel, (const uint4*)src_k, (const uint4*)src_v, (uint4*)dst_k,
                              (uint4*)dst_v, rows, counts, n_loc, (int64_t)(head_stride * esize / 16), row_v);
}

int fma_tile_groups(int D, int esize) {
    const int tg = 32768 / (16 * D * esize);
    return tg < 8 ? tg : 8;
}

cudaError_t launch_attn_fma(const AttnArgs& a, int max_rows, bool pdl, cudaStream_t s) {
    if (max_rows <= 4) return a.kv_bf16 ? launch_fma_d<__nv_bfloat16, 4>(a, pdl, s) : launch_fma_d<float, 4>(a, pdl, s);
    if (max_rows <= 8) return a.kv_bf16 ? launch_fma_d<__nv_bfloat16, 8>(a, pdl, s) : launch_fma_d<float, 8>(a, pdl, s);
    return a.kv_bf16 ? launch_fma_d<__nv_bfloat16, 16>(a, pdl, s) : launch_fma_d<float, 16>(a, pdl, s);
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
