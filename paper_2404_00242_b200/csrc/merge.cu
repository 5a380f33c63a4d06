// merge.cu -- split-K partial merge (tree_reduce, attention.hpp:209-233).
//
// Runs right after the attention launch of a layer (programmatic dependent
// launch: its CTAs start as the attention CTAs retire and wait for their
// memory).  One warp per (leaf-head merge record, q head in the group).  A
// record's partial ids are contiguous, so after the one 16-byte record load
// (read before the dependency wait) every partial's log2-lse (lane k:
// partial k) and every partial's columns (lane: D/32 columns of each) are
// loaded at once -- one memory round trip after the wait.  Partials are combined in the schedule's fixed (item)
// order, so the result does not depend on CTA timing.  The records were
// written moments earlier and are read from L2.
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

constexpr int PB = 8;   // partials loaded per batch (all in flight together)

template <int DPL>
__global__ void __launch_bounds__(128) merge_kernel(const AttnArgs a, int n_merge) {
    pdl_launch_dependents();
    const int wid = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const bool live = wid < n_merge * a.G;
    const int mi = live ? wid / a.G : 0, g = wid % a.G;
    // the record is host-written schedule metadata: read it before the wait
    const int4 rec = live ? __ldg(a.merge_rec + mi) : make_int4(0, 0, 0, 0);   // leaf, head, first partial, count
    pdl_wait();   // the attention launch's partials are complete
    if (!live) return;
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
        // this chunk's lse (lane k) and the first batch of columns, together
        const float lp = lane < np ? __ldcg(a.part_lse + (size_t)(p0 + lane) * G + g) : -INFINITY;
        float v[PB][DPL];
#pragma unroll
        for (int u = 0; u < PB; ++u) {
            if (active && u < np) {
                ld_cols<DPL>(a.part_o + ((size_t)(p0 + u) * G + g) * D + lane * DPL, v[u]);
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
                        ld_cols<DPL>(a.part_o + ((size_t)(p0 + p + u) * G + g) * D + lane * DPL, v[u]);
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
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
            const size_t o = ob + lane * DPL + i;
            if (a.out_bf16)
                reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(acc[i] * inv);
            else
                reinterpret_cast<float*>(a.out)[o] = acc[i] * inv;
        }
    }
    if (lane == 0 && a.lse) a.lse[(size_t)rec.x * a.hq_loc + hq] = M == -INFINITY ? -INFINITY : (M + log2f(den)) * kLn2;
}

}  // namespace

cudaError_t launch_merge(const AttnArgs& a, int n_merge, bool pdl, cudaStream_t s) {
    if (n_merge == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((n_merge * a.G + 3) / 4);
    cfg.blockDim = dim3(128);
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
