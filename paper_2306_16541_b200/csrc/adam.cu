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

// Both passes stream float4s (the flat buffer is 16-byte aligned; a scalar tail covers
// n % 4); each element still picks its own segment's learning rate.
__global__ void k_adam_check(const float* __restrict__ grad, int64_t n, AdamSegs segs, int32_t* __restrict__ flag) {
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(grad);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 g = g4[i];
    if (!(isfinite(g.x) && isfinite(g.y) && isfinite(g.z) && isfinite(g.w))) {
      const float gv[4] = {g.x, g.y, g.z, g.w};
      for (int k = 0; k < 4; ++k)
        if (!isfinite(gv[k])) atomicCAS(flag, 0, 1 + seg_of(segs, 4 * i + k));
    }
  }
  for (int64_t e = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(grad[e])) atomicCAS(flag, 0, 1 + seg_of(segs, e));
}

__device__ __forceinline__ float adam_one(float& p, float g, float& m, float& v, float lr, float b1, float b2,
                                          float eps, float rb1, float rb2) {
  m = b1 * m + (1.f - b1) * g;
  v = b2 * v + (1.f - b2) * g * g;
  p = p - lr * (m * rb1) / (sqrtf(v * rb2) + eps);
  return p;
}

__global__ void k_adam_update(float* __restrict__ p, const float* __restrict__ grad, float* __restrict__ m,
                              float* __restrict__ v, int64_t n, AdamSegs segs, float b1, float b2, float eps,
                              float bc1, float bc2, __half* __restrict__ half, int64_t hb, int64_t he,
                              const int32_t* __restrict__ flag) {
  if (*flag != 0) return;
  const float rb1 = 1.f / bc1, rb2 = 1.f / bc2;
  const int64_t n4 = n / 4;
  const bool hvec = half && (hb % 4 == 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    const float4 gg = reinterpret_cast<const float4*>(grad)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    const int64_t e = 4 * i;
    const int s0 = seg_of(segs, e), s3 = seg_of(segs, e + 3);
    const float l0 = segs.lr[s0];
    const float l3 = segs.lr[s3];
    const float l1 = s0 == s3 ? l0 : segs.lr[seg_of(segs, e + 1)];
    const float l2 = s0 == s3 ? l0 : segs.lr[seg_of(segs, e + 2)];
    adam_one(pp.x, gg.x, mm.x, vv.x, l0, b1, b2, eps, rb1, rb2);
    adam_one(pp.y, gg.y, mm.y, vv.y, l1, b1, b2, eps, rb1, rb2);
    adam_one(pp.z, gg.z, mm.z, vv.z, l2, b1, b2, eps, rb1, rb2);
    adam_one(pp.w, gg.w, mm.w, vv.w, l3, b1, b2, eps, rb1, rb2);
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (half && e + 3 >= hb && e < he) {
      if (hvec && e >= hb && e + 3 < he) {
        const __half2 a = __floats2half2_rn(pp.x, pp.y), b = __floats2half2_rn(pp.z, pp.w);
        uint2 u;
        u.x = *reinterpret_cast<const uint32_t*>(&a);
        u.y = *reinterpret_cast<const uint32_t*>(&b);
        *reinterpret_cast<uint2*>(half + (e - hb)) = u;
      } else {
        const float pv[4] = {pp.x, pp.y, pp.z, pp.w};
        for (int k = 0; k < 4; ++k)
          if (e + k >= hb && e + k < he) half[e + k - hb] = __float2half_rn(pv[k]);
      }
    }
  }
  for (int64_t e = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float pe = p[e], me = m[e], ve = v[e];
    adam_one(pe, grad[e], me, ve, segs.lr[seg_of(segs, e)], b1, b2, eps, rb1, rb2);
    p[e] = pe; m[e] = me; v[e] = ve;
    if (half && e >= hb && e < he) half[e - hb] = __float2half_rn(pe);
  }
}

// Set *flag to `code` (first writer wins) if any of x[0..n) is non-finite.
__global__ void k_check_finite(const float* __restrict__ x, int64_t n, int32_t code, int32_t* __restrict__ flag) {
  bool bad = false;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[e]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicCAS(flag, 0, code);
}

}  // namespace fv

using namespace fv;

extern "C" int32_t fv_check_finite(const float* d_x, int64_t n, int32_t code, int32_t* d_flag, void* stream) {
  if (n < 0 || !d_flag || code == 0 || (n > 0 && !d_x)) return set_error(FV_EDIM, "fv_check_finite: bad arguments");
  if (n == 0) return FV_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_check_finite<<<grid, 256, 0, (cudaStream_t)stream>>>(d_x, n, code, d_flag);
  return check_launch("fv_check_finite");
}

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
  if (n == 0) return FV_OK;
  if ((reinterpret_cast<uintptr_t>(d_param) | reinterpret_cast<uintptr_t>(d_grad) | reinterpret_cast<uintptr_t>(d_m) |
       reinterpret_cast<uintptr_t>(d_v)) & 15)
    return set_error(FV_EDIM, "fv_adam_step: buffers must be 16-byte aligned");
  if (d_half && (reinterpret_cast<uintptr_t>(d_half) & 7)) return set_error(FV_EDIM, "fv_adam_step: fp16 copy must be 8-byte aligned");
  const int grid = (int)std::min<int64_t>((n / 4 + 255) / 256 + 1, 148 * 8);
  k_adam_check<<<grid, 256, 0, st>>>(d_grad, n, s, d_flag);
  k_adam_update<<<grid, 256, 0, st>>>(d_param, d_grad, d_m, d_v, n, s, beta1, beta2, eps, bc1, bc2, (__half*)d_half,
                                      half_begin, half_end, d_flag);
  return check_launch("fv_adam_step");
}
