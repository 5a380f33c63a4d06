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
#include <mutex>
#include <vector>

#include "ta_ptx.cuh"

namespace ta {
namespace {

using namespace dev;

template <int DPL>
__global__ void __launch_bounds__(128, 8) merge_kernel(const AttnArgs a) {
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31;
    // counts and records are host-written schedule metadata: read before the wait
    const int n_rows = a.counts->n_merge * a.G;
    int wid = blockIdx.x * 4 + (threadIdx.x >> 5);
    int4 rec = wid < n_rows ? __ldg(a.merge_rec + wid / a.G) : make_int4(0, 0, 0, 0);   // leaf, head, first partial, count
    pdl_wait();   // the attention launch's partials are complete
    if (threadIdx.x == 0) timeline_mark(a.timeline, 2, true);
    for (; wid < n_rows; wid += gridDim.x * 4) {
        merge_record_row<DPL>(a, rec, wid % a.G, lane);
        const int nx = wid + gridDim.x * 4;
        if (nx < n_rows) rec = __ldg(a.merge_rec + nx / a.G);
    }
    if (threadIdx.x == 0) timeline_mark(a.timeline, 2, false);
}

// ta_lse_merge: one warp per row; lane k < n holds part k's lse, every lane
// DPL columns of each part (all parts' loads in flight), combined in part order.
template <int DPL>
__global__ void __launch_bounds__(256) lse_merge_kernel(const float* __restrict__ part_o, const float* __restrict__ part_lse,
                                                        int n_parts, int64_t rows, int d, void* out, int out_bf16,
                                                        float* lse_out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const float lp = lane < n_parts ? part_lse[(int64_t)lane * rows + row] : -INFINITY;
    float M = lp;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    const float w = (lp == -INFINITY) ? 0.f : __expf(lp - M);
    float den = w;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
    for (int c0 = lane * DPL; c0 < d; c0 += 32 * DPL) {
        float acc[DPL];
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
        for (int p = 0; p < n_parts; ++p) {
            const float wp = __shfl_sync(0xffffffffu, w, p);
            float v[DPL];
            ldcg_cols<DPL>(part_o + ((int64_t)p * rows + row) * d + c0, v);
#pragma unroll
            for (int i = 0; i < DPL; ++i) acc[i] = fmaf(wp, v[i], acc[i]);
        }
        const float inv = den > 0.f ? 1.f / den : 0.f;
        if (out_bf16) {
#pragma unroll
            for (int i = 0; i < DPL; ++i)
                reinterpret_cast<__nv_bfloat16*>(out)[row * d + c0 + i] = __float2bfloat16_rn(acc[i] * inv);
        } else {
#pragma unroll
            for (int i = 0; i < DPL; ++i) reinterpret_cast<float*>(out)[row * d + c0 + i] = acc[i] * inv;
        }
    }
    if (lane == 0 && lse_out) lse_out[row] = M == -INFINITY ? -INFINITY : M + logf(den);
}

}  // namespace

cudaError_t launch_lse_merge(const float* part_o, const float* part_lse, int n_parts, int64_t rows, int d, void* out,
                             int out_bf16, float* lse_out, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((rows + 7) / 8);
    if (d % 4 == 0) lse_merge_kernel<4><<<grid, 256, 0, s>>>(part_o, part_lse, n_parts, rows, d, out, out_bf16, lse_out);
    else lse_merge_kernel<1><<<grid, 256, 0, s>>>(part_o, part_lse, n_parts, rows, d, out, out_bf16, lse_out);
    return cudaGetLastError();
}

cudaError_t launch_merge(const AttnArgs& a, int n_sms, bool pdl, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(4 * n_sms);   // fixed: the record count is read on the device
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (a.D >= 128) return cudaLaunchKernelEx(&cfg, merge_kernel<4>, a);
    if (a.D >= 64) return cudaLaunchKernelEx(&cfg, merge_kernel<2>, a);
    return cudaLaunchKernelEx(&cfg, merge_kernel<1>, a);
}

}  // namespace ta

namespace ta {

cudaError_t set_smem_attr_once(const void* kernel, int bytes) {
    struct Key {
        const void* k;
        int dev;
    };
    static std::mutex mu;
    static std::vector<Key> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    for (const Key& k : done)
        if (k.k == kernel && k.dev == dev) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.push_back({kernel, dev});
    return e;
}

}  // namespace ta
