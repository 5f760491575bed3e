// mulmod_l16.cu — ecm_mulmod_batch kernels for L = 16 (one translation unit per width so the
// build compiles the widths in parallel; the kernels are in mulmod_kernels.cuh).
#include "mulmod_kernels.cuh"

namespace ecm {
template cudaError_t launch_mulmod_L<16>(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out,
                                 size_t count, uint32_t iters, uint32_t flags, cudaStream_t s, size_t* wave);
}  // namespace ecm
