// fp32 SIMT layer kernels for the n_out <= 4 layers of the training path (narrow_layers.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fv {
namespace nl {

int32_t narrow_fwd(const float* x, int64_t ldx, int K, const float* W, const float* b, int act, float* y,
                   int64_t ldy, int64_t M, int N, cudaStream_t st);
int32_t narrow_dx(const float* dz, int64_t ldz, int N, const float* W, int K, const uint32_t* bits,
                  const float* fmask, int64_t ldm, float* dx, int64_t lddx, int64_t M, cudaStream_t st);
int32_t narrow_dw(const float* x, int64_t ldx, int K, const float* dz, int64_t ldz, int N, float* dW, float* db,
                  int64_t M, cudaStream_t st);

}  // namespace nl
}  // namespace fv
