// fused_forward (fu:145-193): the reference's fixed-width (64) MLP evaluated chunk by chunk
// with every layer's weights resident on chip -- one launch for the whole network.
//
// A persistent CTA stages ALL layers' weights (zero-padded to 64x64 fp32, + bias) in shared
// memory once, then walks 128-row chunks: the chunk's input rows land in a 128x64 activation
// buffer, each layer computes the next buffer (ReLU on all but the last layer) and only the
// final out_dim columns go back to HBM.  HBM traffic is therefore in_dim + out_dim floats per
// row instead of 2 x 64 per layer.  fp32 FMAs accumulate every output over k = 0..63 in
// order, so a row's result does not depend on the chunk it falls in (the reference's bitwise
// chunk invariance, t_fused:69-76) and matches naive_forward (fu:132-142) to fp32 rounding.
#include <cuda_runtime.h>
#include "fv_internal.h"

namespace fv {

constexpr int FW = 64;            // fu:29 WIDTH
constexpr int FCH = 128;          // rows per chunk (fu:31 CHUNK)
constexpr int FMAX_LAYERS = 8;

struct FusedMlpArgs {
  const float* w[FMAX_LAYERS];    // (in_i, out_i) row-major
  const float* b[FMAX_LAYERS];    // (out_i) or NULL
  int n_layers, in_dim, out_dim;
};

// smem: n_layers x (64*64 + 64) weights/biases, then two 128 x (64+1) activation buffers
// (+1 column padding so the row-strided reads of a warp fall in distinct banks).
constexpr int ALD = FW + 1;

__global__ void __launch_bounds__(256) k_fused_mlp(FusedMlpArgs a, const float* __restrict__ x, int64_t m,
                                                   float* __restrict__ y) {
  extern __shared__ float sm[];
  float* sw = sm;                                           // [L][64*64]
  float* sb = sm + a.n_layers * FW * FW;                    // [L][64]
  float* act0 = sb + a.n_layers * FW;                       // [128][65]
  float* act1 = act0 + FCH * ALD;
  const int t = threadIdx.x;
  for (int l = 0; l < a.n_layers; ++l) {
    const int kin = l == 0 ? a.in_dim : FW;
    const int nout = l == a.n_layers - 1 ? a.out_dim : FW;
    for (int e = t; e < FW * FW; e += blockDim.x) {
      const int k = e / FW, j = e % FW;
      sw[l * FW * FW + e] = (k < kin && j < nout) ? a.w[l][k * nout + j] : 0.f;
    }
    for (int j = t; j < FW; j += blockDim.x) sb[l * FW + j] = (j < nout && a.b[l]) ? a.b[l][j] : 0.f;
  }
  // thread tile: rows rg + 32 i (i = 0..3) x columns c0 .. c0 + 7 (32 row groups x 8 column
  // groups = 128 x 64); a warp covers 4 row groups (broadcast reads) x all 64 columns
  const int rg = t >> 3, cg = t & 7;
  const int c0 = cg * 8;
  const int64_t nchunks = (m + FCH - 1) / FCH;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t row0 = ch * FCH;
    const int rows = (int)(m - row0 < FCH ? m - row0 : (int64_t)FCH);
    __syncthreads();                      // weights staged / previous chunk's reads done
    for (int e = t; e < FCH * FW; e += blockDim.x) {
      const int r = e / FW, k = e % FW;
      act0[r * ALD + k] = (r < rows && k < a.in_dim) ? x[(row0 + r) * a.in_dim + k] : 0.f;
    }
    float* in = act0;
    float* out = act1;
    for (int l = 0; l < a.n_layers; ++l) {
      __syncthreads();
      const float* W = sw + l * FW * FW;
      float acc[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
      // rows rg + 32 i (i = 0..3): a warp's 4 row groups x 8 column groups
#pragma unroll 4
      for (int k = 0; k < FW; ++k) {
        float av[4], wv[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = in[(rg + 32 * i) * ALD + k];
        const float4 w0 = *reinterpret_cast<const float4*>(W + k * FW + c0);
        const float4 w1 = *reinterpret_cast<const float4*>(W + k * FW + c0 + 4);
        wv[0] = w0.x; wv[1] = w0.y; wv[2] = w0.z; wv[3] = w0.w;
        wv[4] = w1.x; wv[5] = w1.y; wv[6] = w1.z; wv[7] = w1.w;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = __fmaf_rn(av[i], wv[j], acc[i][j]);
      }
      const bool last = l == a.n_layers - 1;
      const float* B = sb + l * FW;
      if (!last) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) out[(rg + 32 * i) * ALD + c0 + j] = fmaxf(__fadd_rn(acc[i][j], B[c0 + j]), 0.f);
        float* tmp = in; in = out; out = tmp;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rg + 32 * i;
          if (r >= rows) continue;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (c0 + j < a.out_dim) y[(row0 + r) * a.out_dim + c0 + j] = __fadd_rn(acc[i][j], B[c0 + j]);
        }
      }
    }
  }
}

}  // namespace fv

using namespace fv;

extern "C" int32_t fv_fused_mlp_fwd(const float* d_x, int64_t m, int32_t in_dim, int32_t out_dim, int32_t n_layers,
                                    const float* const* d_w, const float* const* d_b, float* d_y, void* stream) {
  if (m < 0 || in_dim < 1 || in_dim > FW || out_dim < 1 || out_dim > FW || n_layers < 2 || n_layers > FMAX_LAYERS ||
      !d_w || (m > 0 && (!d_x || !d_y)))
    return set_error(FV_EDIM, "fv_fused_mlp_fwd: bad arguments (in/out width 1..64, 2..8 layers)");
  if (m == 0) return FV_OK;
  FusedMlpArgs a{};
  a.n_layers = n_layers; a.in_dim = in_dim; a.out_dim = out_dim;
  for (int l = 0; l < n_layers; ++l) {
    if (!d_w[l]) return set_error(FV_EDIM, "fv_fused_mlp_fwd: null weight");
    a.w[l] = d_w[l];
    a.b[l] = d_b ? d_b[l] : nullptr;
  }
  const size_t smem = (size_t)(n_layers * (FW * FW + FW) + 2 * FCH * ALD) * sizeof(float);
  cudaFuncSetAttribute(k_fused_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nchunks = (m + FCH - 1) / FCH;
  const int grid = (int)std::min<int64_t>(nchunks, (int64_t)n_sm);
  k_fused_mlp<<<grid, 256, smem, (cudaStream_t)stream>>>(a, d_x, m, d_y);
  return check_launch("fv_fused_mlp_fwd");
}
