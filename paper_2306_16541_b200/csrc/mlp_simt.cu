// fp32 SIMT MLP kernels: the 1e-5-parity path (config 1), the FusedMlp width-64 evaluator
// in float32 (fu:182-193) and the training-time linear backward (ad:417-422).
// Layer convention of the reference: y = act(x @ W + b), W stored (in, out) (ad:403-425).
#include <cuda_runtime.h>
#include "fv_common.cuh"
#include "fv_internal.h"

namespace fv {

constexpr int BM = 64, BN = 64, BK = 16;

// C[m, n] = act( sum_k A(m,k) * B(k,n) + bias[n] )
//   A(m,k) = a[m*lda + k]                      (row-major activations)
//   MASK_A: A(m,k) *= (amask[m*lda + k] > 0)   (ReLU backward mask taken from y)
//   B(k,n) = b[k*sbk + n*sbn]                  (W: sbk=N, sbn=1 ; W^T: sbk=1, sbn=ldW)
template <bool MASK_A>
__global__ void __launch_bounds__(256) k_gemm_f32(const float* __restrict__ a, const float* __restrict__ amask,
                                                  int64_t lda, const float* __restrict__ b, int64_t sbk,
                                                  int64_t sbn, const float* __restrict__ bias,
                                                  float* __restrict__ c, int64_t ldc, int64_t M, int K, int N,
                                                  int act) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      const int mm = e / BK, kk = e % BK;
      const int64_t gm = m0 + mm;
      const int gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < K) {
        v = a[gm * lda + gk];
        if (MASK_A) v = amask[gm * lda + gk] > 0.f ? v : 0.f;
      }
      As[kk][mm] = v;
    }
    for (int e = threadIdx.x; e < BN * BK; e += 256) {
      const int kk = e / BN, nn = e % BN;
      const int gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < K && gn < N) ? b[gk * sbk + gn * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j] + (bias ? bias[gn] : 0.f);
      if (act == 1) v = fmaxf(v, 0.f);
      c[gm * ldc + gn] = v;
    }
  }
}

// dW[k, n] += sum_m x[m,k] * dz[m,n],  dz = dy * (y > 0 if relu);  db[n] += sum_m dz[m,n]
constexpr int DW_ROWS = 2048;
__global__ void __launch_bounds__(256) k_linear_dw(const float* __restrict__ x, const float* __restrict__ y,
                                                   const float* __restrict__ dy, float* __restrict__ dw,
                                                   float* __restrict__ db, int64_t M, int K, int N, int act) {
  __shared__ float Xs[BK][BM + 4];
  __shared__ float Zs[BK][BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int k0 = blockIdx.x * BM;  // dW row tile (input features)
  const int n0 = blockIdx.y * BN;  // dW col tile (outputs)
  const int64_t r0 = (int64_t)blockIdx.z * DW_ROWS;
  const int64_t r1 = r0 + DW_ROWS < M ? r0 + DW_ROWS : M;
  float acc[4][4] = {};
  float bacc = 0.f;  // per-thread partial of db for column n0 + (threadIdx.x % 64), rows strided
  for (int64_t rr = r0; rr < r1; rr += BK) {
    for (int e = threadIdx.x; e < BK * BM; e += 256) {
      const int r = e / BM, kk = e % BM;
      const int64_t gr = rr + r;
      Xs[r][kk] = (gr < r1 && k0 + kk < K) ? x[gr * K + k0 + kk] : 0.f;
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      const int r = e / BN, nn = e % BN;
      const int64_t gr = rr + r;
      float v = 0.f;
      if (gr < r1 && n0 + nn < N) {
        v = dy[gr * N + n0 + nn];
        if (act == 1 && !(y[gr * N + n0 + nn] > 0.f)) v = 0.f;
      }
      Zs[r][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < BK; ++r) {
      float xv[4], zv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = Xs[r][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) zv[j] = Zs[r][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xv[i], zv[j], acc[i][j]);
    }
    if (db && blockIdx.x == 0 && threadIdx.x < BN) {
#pragma unroll
      for (int r = 0; r < BK; ++r) bacc += Zs[r][threadIdx.x];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gk = k0 + ty * 4 + i;
    if (gk >= K) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn < N && acc[i][j] != 0.f) atomicAdd(dw + (int64_t)gk * N + gn, acc[i][j]);
    }
  }
  if (db && blockIdx.x == 0 && threadIdx.x < BN && n0 + threadIdx.x < N && bacc != 0.f)
    atomicAdd(db + n0 + threadIdx.x, bacc);
}

int32_t linear_fwd(const float* x, const float* w, const float* b, float* y, int64_t m, int k, int n, int act,
                   cudaStream_t st) {
  dim3 grid((unsigned)((m + BM - 1) / BM), (unsigned)((n + BN - 1) / BN));
  k_gemm_f32<false><<<grid, 256, 0, st>>>(x, nullptr, k, w, n, 1, b, y, n, m, k, n, act);
  return check_launch("linear_fwd");
}

// ---------------------------------------------------------------- fp32 field (config 1)

// posenc of x_skel (ad:581-600): [x, per band k: w_k sin(x 2^k pi), w_k cos(x 2^k pi)];
// angle = x * float32(2^k pi) then sinf/cosf, as numpy float32 does.
__global__ void k_posenc(fv_field f, const float4* __restrict__ xs, int64_t n, float eps_w, float* __restrict__ pe) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int D = 3 + 6 * f.pe_bands;
  const float4 v = xs[p];
  float* o = pe + p * D;
  if (!(v.w > eps_w)) {
    for (int j = 0; j < D; ++j) o[j] = 0.f;
    return;
  }
  const float x[3] = {v.x, v.y, v.z};
  o[0] = x[0]; o[1] = x[1]; o[2] = x[2];
  for (int k = 0; k < f.pe_bands; ++k) {
    const float freq = __fmul_rn((float)(1 << k), 3.14159265358979323846f);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const float ang = __fmul_rn(x[j], freq);
      float s, c;
      sincosf(ang, &s, &c);
      o[3 + 6 * k + j] = __fmul_rn(f.pe_w[k], s);
      o[3 + 6 * k + 3 + j] = __fmul_rn(f.pe_w[k], c);
    }
  }
}

__global__ void k_xfinal_hash(fv_hash h, const float4* __restrict__ xs, const float* __restrict__ xres, int64_t n,
                              float eps_w, float* __restrict__ feat, float* __restrict__ xfinal) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const float4 v = xs[p];
  const int F = 2 * h.n_levels;
  if (!(v.w > eps_w)) {
    for (int j = 0; j < F; ++j) feat[p * F + j] = 0.f;
    if (xfinal) xfinal[3 * p] = xfinal[3 * p + 1] = xfinal[3 * p + 2] = 0.f;
    return;
  }
  float x0 = v.x, x1 = v.y, x2 = v.z;
  if (xres) {
    x0 = __fadd_rn(x0, xres[3 * p]); x1 = __fadd_rn(x1, xres[3 * p + 1]); x2 = __fadd_rn(x2, xres[3 * p + 2]);
  }
  if (xfinal) { xfinal[3 * p] = x0; xfinal[3 * p + 1] = x1; xfinal[3 * p + 2] = x2; }
  float xn[3]; bool mask[3];
  hash_norm(h, x0, x1, x2, xn, mask);
  for (int l = 0; l < h.n_levels; ++l) {
    HashCell c;
    hash_level_cell(xn, h.res[l], c);
    const float2 fv2 = hash_level_feat(h, l, c);
    feat[p * F + 2 * l] = fv2.x;
    feat[p * F + 2 * l + 1] = fv2.y;
  }
}

__global__ void k_heads(const float4* __restrict__ xs, const float* __restrict__ hd, int64_t n, float eps_w,
                        float4* __restrict__ rgbs) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (!(xs[p].w > eps_w)) { rgbs[p] = make_float4(0.f, 0.f, 0.f, 0.f); return; }
  const float* h = hd + 4 * p;
  rgbs[p] = make_float4(sigmoidf_(h[0]), sigmoidf_(h[1]), sigmoidf_(h[2]), softplusf_(h[3] - 1.f));
}

// b0' = b0 + pose @ W0[D:, :]
__global__ void k_offset_bias(const float* __restrict__ w0, const float* __restrict__ b0, const float* __restrict__ pose,
                              int d_pe, int n_pose, int n_out, float* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_out) return;
  float acc = b0 ? b0[j] : 0.f;
  for (int k = 0; k < n_pose; ++k) acc = fmaf(pose[k], w0[(int64_t)(d_pe + k) * n_out + j], acc);
  out[j] = acc;
}

constexpr int64_t F32_CHUNK = 131072;
constexpr int OFF_W = 128, RAD_W = 64;

size_t field_f32_work_bytes(int64_t n) {
  const int64_t c = n < F32_CHUNK ? n : F32_CHUNK;
  // pe(39) + 2 x 128 hidden + xres 3 + feat 32 + head 4, padded
  return (size_t)c * (40 + 2 * OFF_W + 4 + 32 + 4) * sizeof(float) + 256;
}

int32_t field_fwd_f32(const fv_field* f, const fv_hash* h, const float4* xs, int64_t n, float eps_w, float4* rgbs,
                      float* xfinal, void* work, size_t work_bytes, cudaStream_t st) {
  if (work_bytes < field_f32_work_bytes(n)) return set_error(FV_EDIM, "field fp32: workspace too small");
  const int D = 3 + 6 * f->pe_bands;
  const int64_t cmax = n < F32_CHUNK ? n : F32_CHUNK;
  float* pe = (float*)work;
  float* ha = pe + cmax * 40;
  float* hb = ha + cmax * OFF_W;
  float* xres = hb + cmax * OFF_W;
  float* feat = xres + cmax * 4;
  float* hd = feat + cmax * 32;
  const int F = 2 * h->n_levels;
  for (int64_t s0 = 0; s0 < n; s0 += F32_CHUNK) {
    const int64_t c = (n - s0) < F32_CHUNK ? (n - s0) : F32_CHUNK;
    const unsigned g = (unsigned)((c + 127) / 128);
    const float* xres_p = nullptr;
    if (f->offset_enabled) {
      k_posenc<<<g, 128, 0, st>>>(*f, xs + s0, c, eps_w, pe);
      if (int32_t e = linear_fwd(pe, f->d_off_w[0], f->d_off_b0_eff, ha, c, D, OFF_W, 1, st)) return e;
      if (int32_t e = linear_fwd(ha, f->d_off_w[1], f->d_off_b[1], hb, c, OFF_W, OFF_W, 1, st)) return e;
      if (int32_t e = linear_fwd(hb, f->d_off_w[2], f->d_off_b[2], ha, c, OFF_W, OFF_W, 1, st)) return e;
      if (int32_t e = linear_fwd(ha, f->d_off_w[3], f->d_off_b[3], hb, c, OFF_W, OFF_W, 1, st)) return e;
      if (int32_t e = linear_fwd(hb, f->d_off_w[4], f->d_off_b[4], xres, c, OFF_W, 3, 0, st)) return e;
      xres_p = xres;
    }
    k_xfinal_hash<<<g, 128, 0, st>>>(*h, xs + s0, xres_p, c, eps_w, feat, xfinal ? xfinal + 3 * s0 : nullptr);
    if (int32_t e = linear_fwd(feat, f->d_rad_w[0], f->d_rad_b[0], ha, c, F, RAD_W, 1, st)) return e;
    if (int32_t e = linear_fwd(ha, f->d_rad_w[1], f->d_rad_b[1], hb, c, RAD_W, RAD_W, 1, st)) return e;
    if (int32_t e = linear_fwd(hb, f->d_rad_w[2], f->d_rad_b[2], hd, c, RAD_W, 4, 0, st)) return e;
    k_heads<<<g, 128, 0, st>>>(xs + s0, hd, c, eps_w, rgbs + s0);
  }
  return check_launch("field_fwd_f32");
}

}  // namespace fv

using namespace fv;

extern "C" int32_t fv_linear_fwd(const float* d_x, const float* d_w, const float* d_b, float* d_y, int64_t m,
                                 int32_t k_in, int32_t n_out, int32_t act, void* stream) {
  if (m < 0 || k_in < 1 || n_out < 1 || (act != 0 && act != 1)) return set_error(FV_EDIM, "fv_linear_fwd: bad shape");
  if (m == 0) return FV_OK;
  return linear_fwd(d_x, d_w, d_b, d_y, m, k_in, n_out, act, (cudaStream_t)stream);
}

extern "C" int32_t fv_linear_bwd(const float* d_x, const float* d_w, const float* d_y, const float* d_dy, float* d_dx,
                                 float* d_dw, float* d_db, int64_t m, int32_t k_in, int32_t n_out, int32_t act,
                                 void* stream) {
  if (m < 0 || k_in < 1 || n_out < 1 || (act != 0 && act != 1)) return set_error(FV_EDIM, "fv_linear_bwd: bad shape");
  if (m == 0) return FV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (d_dx) {
    dim3 grid((unsigned)((m + BM - 1) / BM), (unsigned)((k_in + BN - 1) / BN));
    if (act == 1)
      k_gemm_f32<true><<<grid, 256, 0, st>>>(d_dy, d_y, n_out, d_w, 1, n_out, nullptr, d_dx, k_in, m, n_out, k_in, 0);
    else
      k_gemm_f32<false><<<grid, 256, 0, st>>>(d_dy, nullptr, n_out, d_w, 1, n_out, nullptr, d_dx, k_in, m, n_out, k_in, 0);
  }
  if (d_dw) {
    dim3 grid((unsigned)((k_in + BM - 1) / BM), (unsigned)((n_out + BN - 1) / BN), (unsigned)((m + DW_ROWS - 1) / DW_ROWS));
    k_linear_dw<<<grid, 256, 0, st>>>(d_x, d_y, d_dy, d_dw, d_db, m, k_in, n_out, act);
  }
  return check_launch("fv_linear_bwd");
}

extern "C" int32_t fv_offset_bias(const fv_field* field, const float* d_pose, int32_t n_pose, float* d_b0_eff,
                                  void* stream) {
  if (!field || n_pose < 0) return set_error(FV_EDIM, "fv_offset_bias: bad arguments");
  const int d_pe = 3 + 6 * field->pe_bands;
  k_offset_bias<<<1, 128, 0, (cudaStream_t)stream>>>(field->d_off_w[0], field->d_off_b[0], d_pose, d_pe, n_pose, 128,
                                                     d_b0_eff);
  return check_launch("fv_offset_bias");
}
