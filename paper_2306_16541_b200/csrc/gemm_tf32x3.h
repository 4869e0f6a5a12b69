// Split-precision (3xTF32) tcgen05 layer GEMMs of the training path (gemm_tf32x3.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fv {
namespace g3 {

struct RowsArgs {
  const float* A; int64_t lda; int K;          // A (M x K) row-major, K <= 256
  const float* W; int64_t sbn, sbk; int N;     // B(n,k) = W[n*sbn + k*sbk], N <= 128
  const float* bias; int act;                  // epilogue: + bias[n]; act 1 = ReLU
  const float* mask; int64_t ldm;              // epilogue: * (mask[m*ldm + n] > 0) if mask
  float* out; int64_t ldo; int64_t M;
  uint32_t* bits_out = nullptr;                // epilogue: bit (y > 0) per output, [M][ceil(N/32)] words
  const uint32_t* bits_in = nullptr;           // epilogue: * bit, [M][ceil(N/32)] words (ReLU mask as bits)
  // filled by rows_gemm
  int Np = 0, nkc = 0, nsteps = 0, tma = 0, tma_out = 0, stages = 0;
};

struct DwArgs3 {
  const float* X; int64_t ldx; int K;          // layer input (M x K), K <= 128
  const float* Z; int64_t ldz; int N;          // dZ (M x N), already ReLU-masked, N <= 128
  float* dW;                                   // (K x N) row-major, accumulated
  float* db;                                   // (N) accumulated, may be null
  int64_t M;
  // filled by dw_gemm
  int64_t rows_per_cta = 0;
  int nxb = 0, nzb = 0, tmaX = 0, tmaZ = 0, stages = 0;
};

int32_t rows_gemm(RowsArgs a, cudaStream_t st);
int32_t dw_gemm(DwArgs3 a, cudaStream_t st);

}  // namespace g3
}  // namespace fv
