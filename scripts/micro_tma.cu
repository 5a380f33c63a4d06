// micro_tma.cu -- streaming ceiling of the KV staging design on one B200.
// Each CTA streams `tiles` tiles of K+V (128 rows x 256 B each = 64 KB/tile)
// through `S` shared-memory stages, loading each tile as 128/H TMA boxes of
// H rows x 64 cols (x2 column halves).  A consumer warp releases a stage as
// soon as it lands (no math): this is the memory-side ceiling of the design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_tma scripts/micro_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint32_t bar) { asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(bar) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t b) { asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
    asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const void* map, int c0, int c1, uint32_t bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar) : "memory");
}

template <int H, int S>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mv,
                                                       int tiles, int rows_total, int share, int seq) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(sm + S * 65536);
    const uint32_t b0 = smem_u32(bars);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * S; ++i) mbar_init(b0 + 8 * i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        for (int t = 0; t < tiles; ++t) {
            const int s = t % S;
            mbar_wait(b0 + 8 * (S + s), ((t / S) & 1) ^ 1);
            mbar_expect(b0 + 8 * s, 65536);
            const uint32_t dst = smem_u32(sm + s * 65536);
            // pseudo-random tile base row (128-row aligned), distinct per CTA/tile
            // share > 0: groups of `share` CTAs read the same tile sequence
            // (share < 0: the same, each CTA of a group offset by one tile)
            const int grp = share > 0 ? share : (share < 0 ? -share : 1);
            const long long tile_id = share == 0 ? (long long)blockIdx.x * tiles + t
                                                 : (long long)(blockIdx.x / grp) * tiles + (share > 0 ? t : (t + blockIdx.x % grp) % tiles);
            // hashed tile positions, or (seq) contiguous tile runs
            const int row0 = seq ? (int)((tile_id % (rows_total / 128)) * 128)
                                 : (int)((tile_id * 2654435761LL) % (rows_total / 128)) * 128;
            for (int b = 0; b < 128 / H; ++b) {
                tma2d(dst + b * H * 128, &mk, 0, row0 + b * H, b0 + 8 * s);
                tma2d(dst + 16384 + b * H * 128, &mk, 64, row0 + b * H, b0 + 8 * s);
                tma2d(dst + 32768 + b * H * 128, &mv, 0, row0 + b * H, b0 + 8 * s);
                tma2d(dst + 49152 + b * H * 128, &mv, 64, row0 + b * H, b0 + 8 * s);
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int t = 0; t < tiles; ++t) {
            const int s = t % S;
            mbar_wait(b0 + 8 * s, (t / S) & 1);
            mbar_arrive(b0 + 8 * (S + s));
        }
    }
    __syncthreads();
}

template <int H, int S>
float run(CUtensorMap& mk, CUtensorMap& mv, int ctas, int tiles, int rows, int share = 0, int seq = 0) {
    const int smem = S * 65536 + 2048;
    cudaFuncSetAttribute(stream_kernel<H, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    stream_kernel<H, S><<<ctas, 64, smem>>>(mk, mv, tiles, rows, share, seq);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) stream_kernel<H, S><<<ctas, 64, smem>>>(mk, mv, tiles, rows, share, seq);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 5.0 * ctas * tiles * 65536.0;
    const float gbs = (float)(bytes / (ms * 1e-3) / 1e9);
    printf("H=%3d S=%d ctas=%4d tiles=%3d share=%2d seq=%d : %8.1f GB/s  (%s)\n", H, S, ctas, tiles, share, seq, gbs, cudaGetErrorString(cudaGetLastError()));
    return gbs;
}

int main() {
    const int rows = 8 << 20;  // 8M rows x 256 B = 2 GiB per tensor
    void *k, *v;
    cudaMalloc(&k, (size_t)rows * 256);
    cudaMalloc(&v, (size_t)rows * 256);
    cudaMemset(k, 1, (size_t)rows * 256);
    cudaMemset(v, 1, (size_t)rows * 256);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    auto make = [&](CUtensorMap* m, void* base, int H) {
        cuuint64_t dims[2] = {128, (cuuint64_t)rows};
        cuuint64_t str[1] = {256};
        cuuint32_t box[2] = {64, (cuuint32_t)H};
        cuuint32_t es[2] = {1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap k16, v16, k128, v128;
    make(&k16, k, 16); make(&v16, v, 16); make(&k128, k, 128); make(&v128, v, 128);
    for (int ctas : {148, 296}) {
        run<16, 2>(k16, v16, ctas, 64, rows);
        run<16, 3>(k16, v16, ctas, 64, rows);
        run<128, 2>(k128, v128, ctas, 64, rows);
        run<128, 3>(k128, v128, ctas, 64, rows);
    }
    run<16, 2>(k16, v16, 112, 16, rows);
    run<128, 2>(k128, v128, 112, 16, rows);
    run<16, 3>(k16, v16, 112, 16, rows);
    // L2-resident working sets (a 16k-token prefix x 8 heads = 128k rows, 64 MB
    // of K+V; and 32k rows, 16 MB): the ceiling for re-read tiles that hit L2
    for (int small : {131072, 32768}) {
        printf("L2-resident working set: %d rows (%.0f MB K+V)\n", small, small * 512.0 / 1e6);
        run<128, 2>(k128, v128, 148, 64, small);
        run<128, 3>(k128, v128, 148, 64, small);
        run<16, 2>(k16, v16, 148, 64, small);
    }
    // tiles shared by groups of CTAs (the lanes of a wide stripe), 1 GB of
    // rows (L2-resident only through the sharing)
    printf("shared tile sequences (2 GiB tensors: a tile comes from DRAM once per group)\n");
    for (int sh : {1, 2, 4, 8, -2, -4, -8}) run<128, 2>(k128, v128, 148, 64, rows, sh);
    for (int sh : {8, -8}) run<128, 3>(k128, v128, 148, 64, rows, sh);
    printf("contiguous tile runs\n");
    for (int sh : {0, 2, 8, -8}) run<128, 2>(k128, v128, 148, 64, rows, sh, 1);
    run<128, 2>(k128, v128, 148, 64, 131072, 0, 1);
    return 0;
}
