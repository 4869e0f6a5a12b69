// Fused multi-tensor Adam (ad:880-912): one pass over a flat fp32 master buffer holding
// every trainable block, per-segment learning rate, bias correction, optional fp16
// shadow copy of a sub-range (the hash table used by the forward).  A first pass flags
// non-finite gradients; the update pass is skipped entirely when the flag is set, which
// mirrors the reference raising TrainingError before touching any parameter (ad:898-902).
#include <cuda_runtime.h>
#include "fv_common.cuh"
#include "fv_internal.h"

namespace fv {

struct AdamSegs {
  int64_t end[32];
  float lr[32];
  int n;
};

__device__ __forceinline__ int seg_of(const AdamSegs& s, int64_t e) {
  int k = 0;
  while (k < s.n - 1 && e >= s.end[k]) ++k;
  return k;
}

__global__ void k_adam_check(const float* __restrict__ grad, int64_t n, AdamSegs segs, int32_t* __restrict__ flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    if (!isfinite(grad[e])) atomicCAS(flag, 0, 1 + seg_of(segs, e));
  }
}

__global__ void k_adam_update(float* __restrict__ p, const float* __restrict__ grad, float* __restrict__ m,
                              float* __restrict__ v, int64_t n, AdamSegs segs, float b1, float b2, float eps,
                              float bc1, float bc2, __half* __restrict__ half, int64_t hb, int64_t he,
                              const int32_t* __restrict__ flag) {
  if (*flag != 0) return;
  const float rb1 = 1.f / bc1, rb2 = 1.f / bc2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float g = grad[e];
    const float mm = b1 * m[e] + (1.f - b1) * g;
    const float vv = b2 * v[e] + (1.f - b2) * g * g;
    m[e] = mm;
    v[e] = vv;
    const float lr = segs.lr[seg_of(segs, e)];
    const float pn = p[e] - lr * (mm * rb1) / (sqrtf(vv * rb2) + eps);
    p[e] = pn;
    if (half && e >= hb && e < he) half[e - hb] = __float2half_rn(pn);
  }
}

}  // namespace fv

using namespace fv;

extern "C" int32_t fv_adam_step(float* d_param, const float* d_grad, float* d_m, float* d_v, int64_t n,
                                const int64_t* seg_end, const float* lr, int32_t n_seg, int32_t step, float beta1,
                                float beta2, float eps, void* d_half, int64_t half_begin, int64_t half_end,
                                int32_t* d_flag, void* stream) {
  if (n < 0 || n_seg < 1 || n_seg > 32 || step < 1 || !seg_end || !lr || !d_flag)
    return set_error(FV_EDIM, "fv_adam_step: bad arguments");
  AdamSegs s{};
  s.n = n_seg;
  for (int i = 0; i < n_seg; ++i) { s.end[i] = seg_end[i]; s.lr[i] = lr[i]; }
  if (s.end[n_seg - 1] != n) return set_error(FV_EDIM, "fv_adam_step: last segment end != n");
  const float bc1 = (float)(1.0 - pow((double)beta1, step));
  const float bc2 = (float)(1.0 - pow((double)beta2, step));
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  if (n == 0) return FV_OK;
  k_adam_check<<<grid, 256, 0, st>>>(d_grad, n, s, d_flag);
  k_adam_update<<<grid, 256, 0, st>>>(d_param, d_grad, d_m, d_v, n, s, beta1, beta2, eps, bc1, bc2, (__half*)d_half,
                                      half_begin, half_end, d_flag);
  return check_launch("fv_adam_step");
}
