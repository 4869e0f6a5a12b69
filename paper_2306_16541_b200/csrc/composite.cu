// Front-to-back compositing with likelihood gating (Eq 3) and its
// division-free reverse scan (ad:815-837 style), one thread per ray, transmittance in a
// register, samples visited in depth order with early termination (T < eps_t).
// The sequential per-ray order equals oracle/composite.py, so T and rgb match it to the
// last bit whenever the per-sample inputs do.
#include <cuda_runtime.h>
#include "fv_common.cuh"
#include "fv_internal.h"
#include "layout.cuh"

namespace fv {


__device__ __forceinline__ int64_t sidx(const CompIn& in, int64_t r, int i, int n) {
  return in.blocked ? sample_index(r, i, n) : r * n + i;
}

// Samples are read in chunks of CH (all loads of a chunk issued before the sequential
// arithmetic consumes them: with few rays per SM -- 6,144 in a training step -- the
// per-sample load latency, not bandwidth, bounds a one-sample-at-a-time loop; with a full
// frame of rays CH = 1 keeps registers low and occupancy high).  The arithmetic and its
// order are the same for every CH.
constexpr int kFewRays = 65536;

template <int CH>
__global__ void k_composite_fwd(CompIn in, int64_t n_rays, int n, float3 bg, float eps_w, float eps_t,
                                const int32_t* __restrict__ out_pix, float* __restrict__ rgb_out,
                                float* __restrict__ alpha_out, float* __restrict__ trans) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f;
  int i = 0;
  bool stop = false;
  for (int i0 = 0; i0 < n && !stop; i0 += CH) {
    float Lc[CH], dc[CH];
    float4 vc[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (i0 + k < n) {
        const int64_t s = sidx(in, r, i0 + k, n);
        Lc[k] = in.lik[s * in.lik_stride];
        if (!in.skip_bg) {                 // independent loads (no wait on the likelihood)
          vc[k] = in.rgbs[s];
          dc[k] = in.delta[s];
        } else {
          // background samples carry sigma = 0 (abar = 0, T unchanged): with a compacted
          // field their [c, sigma] slot was never written, so it is not read
          const bool skip = !(Lc[k] > eps_w);
          vc[k] = skip ? make_float4(0.f, 0.f, 0.f, 0.f) : in.rgbs[s];
          dc[k] = skip ? 0.f : in.delta[s];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (i0 + k >= n) break;
      if (eps_t > 0.f && T < eps_t) { stop = true; break; }
      i = i0 + k + 1;
      if (trans) trans[r * (n + 1) + i0 + k] = T;
      if (in.skip_bg && !(Lc[k] > eps_w)) continue;
      const float4 v = vc[k];
      const float a = __fsub_rn(1.f, expf(-__fmul_rn(v.w, dc[k])));
      const float gate = fminf(fmaxf(__fdiv_rn(Lc[k], eps_w), 0.f), 1.f);
      const float ab = __fmul_rn(a, gate);
      const float w = __fmul_rn(T, ab);
      cr = __fadd_rn(cr, __fmul_rn(w, v.x));
      cg = __fadd_rn(cg, __fmul_rn(w, v.y));
      cb = __fadd_rn(cb, __fmul_rn(w, v.z));
      T = __fmul_rn(T, __fsub_rn(1.f, ab));
    }
  }
  if (trans) for (int j = i; j <= n; ++j) trans[r * (n + 1) + j] = T;
  cr = __fadd_rn(cr, __fmul_rn(T, bg.x));
  cg = __fadd_rn(cg, __fmul_rn(T, bg.y));
  cb = __fadd_rn(cb, __fmul_rn(T, bg.z));
  const int64_t o = out_pix ? out_pix[r] : r;
  rgb_out[3 * o] = cr; rgb_out[3 * o + 1] = cg; rgb_out[3 * o + 2] = cb;
  alpha_out[o] = __fsub_rn(1.f, T);
}

// Q_N = bg, Q_i = ab_i c_i + (1-ab_i) Q_{i+1};  P_N = 1, P_i = (1-ab_i) P_{i+1}
// d rgb/d ab_i = T_i (c_i - Q_{i+1});  d alpha/d ab_i = T_i P_{i+1}   (eps_t must be 0)
template <int CH>
__global__ void k_composite_bwd(CompIn in, const float* __restrict__ trans, int64_t n_rays, int n, float3 bg,
                                float eps_w, const float* __restrict__ drgb, const float* __restrict__ dalpha,
                                float4* __restrict__ dout) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const float gr = drgb[3 * r], gg = drgb[3 * r + 1], gb = drgb[3 * r + 2];
  const float ga = dalpha ? dalpha[r] : 0.f;
  float qr = bg.x, qg = bg.y, qb = bg.z, P = 1.f;
  for (int i1 = n - 1; i1 >= 0; i1 -= CH) {           // chunks of CH samples, back to front
    float4 vc[CH];
    float dc[CH], Lc[CH], Tc[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int i = i1 - k;
      if (i >= 0) {
        const int64_t s = sidx(in, r, i, n);
        vc[k] = in.rgbs[s];
        dc[k] = in.delta[s];
        Lc[k] = in.lik[s * in.lik_stride];
        Tc[k] = trans[r * (n + 1) + i];
      }
    }
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int i = i1 - k;
      if (i < 0) break;
      const int64_t s = sidx(in, r, i, n);
      const float4 v = vc[k];
      const float d = dc[k];
      const float e = expf(-v.w * d);
      const float a = 1.f - e;
      const float gate = fminf(fmaxf(Lc[k] / eps_w, 0.f), 1.f);
      const float ab = a * gate;
      const float Ti = Tc[k];
      const float dab = Ti * (gr * (v.x - qr) + gg * (v.y - qg) + gb * (v.z - qb) + ga * P);
      const float wt = Ti * ab;
      dout[s] = make_float4(wt * gr, wt * gg, wt * gb, dab * gate * d * e);
      qr = ab * v.x + (1.f - ab) * qr;
      qg = ab * v.y + (1.f - ab) * qg;
      qb = ab * v.z + (1.f - ab) * qb;
      P *= 1.f - ab;
    }
  }
}

int32_t composite_fwd(const CompIn& in, int64_t n_rays, int n, const float* bg, float eps_w, float eps_t,
                      const int32_t* out_pix, float* rgb, float* alpha, float* trans, cudaStream_t st) {
  if (n_rays == 0) return FV_OK;
  const unsigned grid = (unsigned)((n_rays + 127) / 128);
  const float3 b = make_float3(bg[0], bg[1], bg[2]);
  if (n_rays < kFewRays)
    k_composite_fwd<8><<<grid, 128, 0, st>>>(in, n_rays, n, b, eps_w, eps_t, out_pix, rgb, alpha, trans);
  else
    k_composite_fwd<1><<<grid, 128, 0, st>>>(in, n_rays, n, b, eps_w, eps_t, out_pix, rgb, alpha, trans);
  return check_launch("composite_fwd");
}

int32_t composite_bwd(const CompIn& in, const float* trans, int64_t n_rays, int n, const float* bg, float eps_w,
                      const float* drgb, const float* dalpha, float4* dout, cudaStream_t st) {
  if (n_rays == 0) return FV_OK;
  const unsigned grid = (unsigned)((n_rays + 127) / 128);
  const float3 b = make_float3(bg[0], bg[1], bg[2]);
  if (n_rays < kFewRays)
    k_composite_bwd<8><<<grid, 128, 0, st>>>(in, trans, n_rays, n, b, eps_w, drgb, dalpha, dout);
  else
    k_composite_bwd<1><<<grid, 128, 0, st>>>(in, trans, n_rays, n, b, eps_w, drgb, dalpha, dout);
  return check_launch("composite_bwd");
}

// One marching round of the front-to-back compositor (early termination): live
// ray j (= live[j], or j when live == NULL) continues from its persistent state (T, rgb) over
// the round's K samples (round slot layout, march_round), with exactly the per-sample rule and
// float32 operation order of k_composite_fwd<skip_bg>, so the final pixel is bitwise the
// single-pass result.  A ray retires -- its pixel is written -- when it missed the box
// (count 0), when T fell below eps_t (the next sample would not be composited) or in the last
// round; otherwise its state is stored and it is appended to next_live (warp-aggregated
// atomic), the next round's ray list.  Whole warps iterate together (ballot), grid-stride.
__global__ void k_composite_round(const float4* __restrict__ rgbs, const float* __restrict__ delta,
                                  const float* __restrict__ lik, int K, int i0, int n, const int32_t* __restrict__ live,
                                  const int32_t* __restrict__ n_live, int64_t n_rays,
                                  const int32_t* __restrict__ ray_count, float4* __restrict__ state, float3 bg,
                                  float eps_w, float eps_t, const int32_t* __restrict__ out_pix,
                                  float* __restrict__ rgb_out, float* __restrict__ alpha_out,
                                  int32_t* __restrict__ next_live, int32_t* __restrict__ next_n) {
  const int64_t n_j = live ? (int64_t)*n_live : n_rays;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool last = i0 + K >= n;
  for (int64_t jb = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; jb < n_j; jb += stride) {
    const int64_t j = jb + lane;
    const bool valid = j < n_j;
    bool cont = false;
    if (valid) {
      const int64_t ray = live ? (int64_t)live[j] : j;
      float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f;
      if (i0 > 0) { const float4 q = state[ray]; T = q.x; cr = q.y; cg = q.z; cb = q.w; }
      bool stop = ray_count[ray] == 0;
      for (int il = 0; il < K && !stop; ++il) {
        if (eps_t > 0.f && T < eps_t) { stop = true; break; }
        const int64_t s = sample_index(j, il, K);
        const float L = lik[s];
        if (!(L > eps_w)) continue;
        const float4 v = rgbs[s];
        const float a = __fsub_rn(1.f, expf(-__fmul_rn(v.w, delta[s])));
        const float gate = fminf(fmaxf(__fdiv_rn(L, eps_w), 0.f), 1.f);
        const float ab = __fmul_rn(a, gate);
        const float w = __fmul_rn(T, ab);
        cr = __fadd_rn(cr, __fmul_rn(w, v.x));
        cg = __fadd_rn(cg, __fmul_rn(w, v.y));
        cb = __fadd_rn(cb, __fmul_rn(w, v.z));
        T = __fmul_rn(T, __fsub_rn(1.f, ab));
      }
      stop = stop || last || (eps_t > 0.f && T < eps_t);
      if (stop) {
        cr = __fadd_rn(cr, __fmul_rn(T, bg.x));
        cg = __fadd_rn(cg, __fmul_rn(T, bg.y));
        cb = __fadd_rn(cb, __fmul_rn(T, bg.z));
        const int64_t o = out_pix ? out_pix[ray] : ray;
        rgb_out[3 * o] = cr; rgb_out[3 * o + 1] = cg; rgb_out[3 * o + 2] = cb;
        alpha_out[o] = __fsub_rn(1.f, T);
      } else {
        state[ray] = make_float4(T, cr, cg, cb);
        cont = true;
      }
    }
    const uint32_t ballot = __ballot_sync(0xffffffffu, cont);
    if (ballot) {
      int32_t base = 0;
      if (lane == 0) base = atomicAdd(next_n, __popc(ballot));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (cont) next_live[base + __popc(ballot & ((1u << lane) - 1u))] = (int32_t)(live ? live[j] : j);
    }
  }
}

int32_t composite_round(const float4* rgbs, const float* delta, const float* lik, int K, int i0, int n,
                        const int32_t* live, const int32_t* n_live, int64_t n_rays, const int32_t* ray_count,
                        float4* state, const float* bg, float eps_w, float eps_t, const int32_t* out_pix, float* rgb,
                        float* alpha, int32_t* next_live, int32_t* next_n, cudaStream_t st) {
  if (n_rays == 0) return FV_OK;
  cudaMemsetAsync(next_n, 0, sizeof(int32_t), st);
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = std::min<int64_t>((n_rays + 127) / 128, (int64_t)n_sm * 16);
  k_composite_round<<<(unsigned)blocks, 128, 0, st>>>(rgbs, delta, lik, K, i0, n, live, n_live, n_rays, ray_count,
                                                      state, make_float3(bg[0], bg[1], bg[2]), eps_w, eps_t, out_pix,
                                                      rgb, alpha, next_live, next_n);
  return check_launch("composite_round");
}

}  // namespace fv

using namespace fv;

namespace fv {
// transmittance (ad:815-837): T[r, 0] = 1, T[r, i + 1] = T[r, i] * atten[r, i] in fp32, the
// exclusive running product of the per-sample attenuations 1 - opacity (one thread per ray).
__global__ void k_transmittance(const float* __restrict__ atten, int64_t R, int N, float* __restrict__ T) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= R) return;
  const float* a = atten + r * N;
  float* t = T + r * (N + 1);
  float acc = 1.f;
  t[0] = acc;
  for (int i = 0; i < N; ++i) {
    acc = __fmul_rn(acc, a[i]);
    t[i + 1] = acc;
  }
}

// Its division-free reverse scan (ad:828-835): b = g[N]; gx[N-1] = T[N-1] b; for j = N-1..1:
// b = g[j] + atten[j] b, gx[j-1] = T[j-1] b -- exact zeros in atten are safe.
__global__ void k_transmittance_bwd(const float* __restrict__ atten, const float* __restrict__ T,
                                    const float* __restrict__ g, int64_t R, int N, float* __restrict__ gx) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= R || N == 0) return;
  const float* a = atten + r * N;
  const float* t = T + r * (N + 1);
  const float* gr = g + r * (N + 1);
  float* o = gx + r * N;
  float b = gr[N];
  o[N - 1] = t[N - 1] * b;
  for (int j = N - 1; j > 0; --j) {
    b = __fadd_rn(gr[j], __fmul_rn(a[j], b));
    o[j - 1] = t[j - 1] * b;
  }
}
}  // namespace fv

extern "C" int32_t fv_transmittance(const float* d_atten, int64_t n_rays, int32_t n_samples, float* d_trans,
                                    void* stream) {
  if (n_rays < 0 || n_samples < 0 || (n_rays > 0 && (!d_atten || !d_trans)))
    return set_error(FV_EDIM, "fv_transmittance: bad arguments");
  if (n_rays == 0) return FV_OK;
  fv::k_transmittance<<<(unsigned)((n_rays + 127) / 128), 128, 0, (cudaStream_t)stream>>>(d_atten, n_rays, n_samples,
                                                                                         d_trans);
  return check_launch("fv_transmittance");
}

extern "C" int32_t fv_transmittance_bwd(const float* d_atten, const float* d_trans, const float* d_g, int64_t n_rays,
                                        int32_t n_samples, float* d_gatten, void* stream) {
  if (n_rays < 0 || n_samples < 0 || (n_rays > 0 && n_samples > 0 && (!d_atten || !d_trans || !d_g || !d_gatten)))
    return set_error(FV_EDIM, "fv_transmittance_bwd: bad arguments");
  if (n_rays == 0 || n_samples == 0) return FV_OK;
  fv::k_transmittance_bwd<<<(unsigned)((n_rays + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      d_atten, d_trans, d_g, n_rays, n_samples, d_gatten);
  return check_launch("fv_transmittance_bwd");
}

extern "C" int32_t fv_composite_fwd(const float* d_rgbs, const float* d_delta, const float* d_lik, int32_t lik_stride,
                                    int32_t blocked, int64_t n_rays, int32_t n_samples, const float bg[3], float eps_w,
                                    float eps_t, float* d_rgb, float* d_alpha, float* d_trans, void* stream) {
  if (n_rays < 0 || n_samples < 1 || !bg || eps_w <= 0.f || lik_stride < 1)
    return set_error(FV_EDIM, "fv_composite_fwd: bad arguments");
  CompIn in{(const float4*)d_rgbs, d_delta, d_lik, lik_stride, blocked != 0};
  return composite_fwd(in, n_rays, n_samples, bg, eps_w, eps_t, nullptr, d_rgb, d_alpha, d_trans, (cudaStream_t)stream);
}

extern "C" int32_t fv_composite_bwd(const float* d_rgbs, const float* d_delta, const float* d_lik, int32_t lik_stride,
                                    int32_t blocked, const float* d_trans, int64_t n_rays, int32_t n_samples,
                                    const float bg[3], float eps_w, const float* d_drgb, const float* d_dalpha,
                                    float* d_drgbs, void* stream) {
  if (n_rays < 0 || n_samples < 1 || !bg || !d_trans || lik_stride < 1)
    return set_error(FV_EDIM, "fv_composite_bwd: bad arguments");
  CompIn in{(const float4*)d_rgbs, d_delta, d_lik, lik_stride, blocked != 0};
  return composite_bwd(in, d_trans, n_rays, n_samples, bg, eps_w, d_drgb, d_dalpha, (float4*)d_drgbs,
                       (cudaStream_t)stream);
}
