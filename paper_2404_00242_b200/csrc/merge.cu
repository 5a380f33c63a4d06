// merge.cu -- split-K partial merge (tree_reduce, attention.hpp:209-233).
//
// Runs right after the attention launch of a layer (programmatic dependent
// launch: its CTAs start as the attention CTAs retire and wait for their
// memory).  One warp per (leaf-head merge record, q head in the group):
// lane k fetches partial k's id and log2-lse (all in flight at once), the
// weights 2^(lse_k - M) / sum are broadcast by shuffle, and every lane sums
// its D/32 columns over the partials with independent loads.  Partials are
// consumed in the schedule's fixed (item) order, so the result does not
// depend on CTA timing.  The partial records were written by the attention
// launch moments earlier and are read from L2.
#include "ta_ptx.cuh"

namespace ta {
namespace {

using namespace dev;

template <int DPL>
__device__ __forceinline__ void ld_cols(const float* p, float (&f)[DPL]) {
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
__global__ void __launch_bounds__(256) merge_kernel(const AttnArgs a, int n_merge) {
    pdl_launch_dependents();
    pdl_wait();   // the attention launch's partials are complete
    const int wid = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (wid >= n_merge * a.G) return;
    const int mi = wid / a.G, g = wid % a.G;
    const int leaf = a.merge_leaf[mi];
    const int pb = a.merge_begin[mi], pe = a.merge_begin[mi + 1];
    const int D = a.D;
    const int hq = a.merge_head[mi] * a.G + g;
    const bool active = lane * DPL < D;
    float acc[DPL];
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
    float M = -INFINITY, den = 0.f;
    for (int base = pb; base < pe; base += 32) {
        const int np = min(32, pe - base);
        int pid = 0;
        float lp = -INFINITY;
        if (lane < np) {
            pid = a.merge_parts[base + lane];
            lp = __ldcg(a.part_lse + (size_t)pid * a.G + g);
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
        for (int p = 0; p < np; p += 8) {
            float v[8][DPL];
            float wv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int id = __shfl_sync(0xffffffffu, pid, (p + u) & 31);
                wv[u] = p + u < np ? __shfl_sync(0xffffffffu, w, (p + u) & 31) : 0.f;
                if (active && p + u < np) {
                    ld_cols<DPL>(a.part_o + ((size_t)id * a.G + g) * D + lane * DPL, v[u]);
                } else {
#pragma unroll
                    for (int i = 0; i < DPL; ++i) v[u][i] = 0.f;
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int i = 0; i < DPL; ++i) acc[i] = fmaf(wv[u], v[u][i], acc[i]);
        }
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    const size_t base = ((size_t)leaf * a.hq_loc + hq) * D;
    if (active) {
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
            const size_t o = base + lane * DPL + i;
            if (a.out_bf16)
                reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(acc[i] * inv);
            else
                reinterpret_cast<float*>(a.out)[o] = acc[i] * inv;
        }
    }
    if (lane == 0 && a.lse) a.lse[(size_t)leaf * a.hq_loc + hq] = M == -INFINITY ? -INFINITY : (M + log2f(den)) * kLn2;
}

}  // namespace

cudaError_t launch_merge(const AttnArgs& a, int n_merge, bool pdl, cudaStream_t s) {
    if (n_merge == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((n_merge * a.G + 7) / 8);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (a.D >= 128) return cudaLaunchKernelEx(&cfg, merge_kernel<4>, a, n_merge);
    if (a.D >= 64) return cudaLaunchKernelEx(&cfg, merge_kernel<2>, a, n_merge);
    return cudaLaunchKernelEx(&cfg, merge_kernel<1>, a, n_merge);
}

}  // namespace ta
