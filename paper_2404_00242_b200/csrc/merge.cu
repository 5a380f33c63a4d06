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

}  // namespace

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
