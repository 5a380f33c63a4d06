// attn_mma.cu -- tcgen05/TMEM path of the chunk attention (dense bf16 chunks).
// (placeholder until the tcgen05 kernel lands; the scheduler never routes
// units here while mma_supported() is false)
#include "ta_kernels.h"

namespace ta {

bool mma_supported(int D, int kv_bf16) { (void)D; (void)kv_bf16; return false; }

cudaError_t launch_attn_mma(const AttnArgs& a, cudaStream_t s) {
    (void)a; (void)s;
    return cudaErrorNotSupported;
}

}  // namespace ta
