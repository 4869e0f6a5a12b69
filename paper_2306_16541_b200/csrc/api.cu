// C-ABI glue: errors, version, the fused render orchestration and the occupancy builder.
#include <cuda_runtime.h>
#include <cstring>
#include "fv_common.cuh"
#include "fv_internal.h"
#include "layout.cuh"

namespace fv {

static thread_local char g_err[512] = "";

int32_t set_error(int32_t code, const char* msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

int32_t check_launch(const char* where) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return FV_ELAUNCH;
  }
  return FV_OK;
}


static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct RenderWork {
  float* lik; float* delta; float4* rgbs; float4* xsc; int32_t* idx; int32_t* count; float4* rgbsc;
  void* fwork; size_t fbytes;
};

// workspace: per-sample likelihood / spacing / [c, sigma] (full ray-block-major layout),
// the march's compacted foreground stream (x, L) + sample ids + counter, and for the fp32
// path a compacted [c, sigma] buffer and the SIMT layer scratch.
static size_t carve(void* base, int64_t S, int precision, RenderWork* w) {
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  const size_t o_l = take((size_t)S * 4), o_d = take((size_t)S * 4), o_r = take((size_t)S * 16);
  const size_t o_x = take((size_t)S * 16), o_i = take((size_t)S * 4), o_c = take(16);
  const size_t o_rc = take(precision == 0 ? (size_t)S * 16 : 0);
  const size_t fb = precision == 0 ? field_f32_work_bytes(S) : 0;
  const size_t o_f = take(fb);
  if (w) {
    uint8_t* b = (uint8_t*)base;
    w->lik = (float*)(b + o_l); w->delta = (float*)(b + o_d); w->rgbs = (float4*)(b + o_r);
    w->xsc = (float4*)(b + o_x); w->idx = (int32_t*)(b + o_i); w->count = (int32_t*)(b + o_c);
    w->rgbsc = (float4*)(b + o_rc); w->fwork = b + o_f; w->fbytes = fb;
  }
  return off;
}

__global__ void k_scatter4(const float4* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                           float4* __restrict__ dst) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) dst[idx[j]] = src[j];
}

int32_t field_fwd(const fv_field* f, const fv_hash* h, const float4* xs, int64_t n, float eps_w, float4* rgbs,
                  float* xfinal, void* work, size_t work_bytes, cudaStream_t st) {
  if (f->precision == 0) return field_fwd_f32(f, h, xs, n, eps_w, rgbs, xfinal, work, work_bytes, st);
  if (f->precision == 1) return field_fwd_tc(f, h, xs, n, eps_w, rgbs, xfinal, st);
  return set_error(FV_EUNSUPPORTED, "fv_field: precision must be 0 (fp32) or 1 (fp16 tcgen05)");
}

// occupancy probe points: cell c (x-major), sub-point j in 2x2x2
__global__ void k_occ_points(fv_march m, fv_warp w, float4* __restrict__ xs) {
  __shared__ __align__(16) float sg[FV_MAX_BONES * 12];
  fill_bones_x2(sg, w.d_g, w.n_bones);
  __syncthreads();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= OCC_RES * OCC_RES * OCC_RES * 8) return;
  const int cell = e >> 3, j = e & 7;
  const int c[3] = {cell / (OCC_RES * OCC_RES), (cell / OCC_RES) % OCC_RES, cell % OCC_RES};
  const int sub[3] = {(j >> 2) & 1, (j >> 1) & 1, j & 1};
  float p[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float cw = __fdiv_rn(__fsub_rn(m.obox_max[k], m.obox_min[k]), (float)OCC_RES);
    p[k] = __fadd_rn(m.obox_min[k], __fmul_rn(__fadd_rn((float)c[k], sub[k] ? 0.75f : 0.25f), cw));
  }
  float xsk[3];
  const float L = warp_point<false>(w, sg, m.eps_w, p[0], p[1], p[2], xsk);
  xs[e] = make_float4(xsk[0], xsk[1], xsk[2], L);
}

__global__ void k_occ_bits(const float4* __restrict__ xs, const float4* __restrict__ rgbs, float eps_w, float thr,
                           uint32_t* __restrict__ occ) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;  // 32768 cells, blockDim multiple of 32
  bool on = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int e = cell * 8 + j;
    on = on || (xs[e].w > eps_w && rgbs[e].w > thr);
  }
  const uint32_t word = __ballot_sync(0xffffffffu, on);
  if ((threadIdx.x & 31) == 0) occ[cell >> 5] = word;
}

constexpr int OCC_PTS = OCC_RES * OCC_RES * OCC_RES * 8;

}  // namespace fv

using namespace fv;

extern "C" int32_t fv_version(void) { return 100; }
extern "C" const char* fv_last_error(void) { return g_err; }
extern "C" void fv_struct_sizes(int64_t* out) {
  out[0] = sizeof(fv_camera); out[1] = sizeof(fv_march); out[2] = sizeof(fv_warp);
  out[3] = sizeof(fv_hash); out[4] = sizeof(fv_field); out[5] = sizeof(fv_scene_merge);
}
extern "C" int32_t fv_device_sm(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

extern "C" size_t fv_field_workspace_bytes(int64_t n, int32_t precision) {
  return precision == 0 ? field_f32_work_bytes(n) : 0;
}

extern "C" int32_t fv_field_fwd(const fv_field* field, const fv_hash* hash, const float* d_xs, int64_t n, float eps_w,
                                float* d_rgbs, float* d_xfinal, void* d_work, size_t work_bytes, void* stream) {
  if (!field || n < 0) return set_error(FV_EDIM, "fv_field_fwd: bad arguments");
  if (int32_t e = check_hash(hash)) return e;
  if (n == 0) return FV_OK;
  return field_fwd(field, hash, (const float4*)d_xs, n, eps_w, (float4*)d_rgbs, d_xfinal, d_work, work_bytes,
                   (cudaStream_t)stream);
}

extern "C" size_t fv_render_workspace_bytes(int64_t n_rays, int32_t n_samples, int32_t precision) {
  return carve(nullptr, padded_rays(n_rays) * n_samples, precision, nullptr);
}

// ev (optional, 5 events): recorded before the march, after the march, between the two
// tensor-core field kernels, after the field and after the compositor (stage timing).
static int32_t render_fwd(const fv_camera* cam, const fv_march* march, const fv_warp* warp, const fv_hash* hash,
                          const fv_field* field, int64_t n_rays, void* d_work, size_t work_bytes, float* d_rgb,
                          float* d_alpha, int32_t* d_count, cudaStream_t st, cudaEvent_t* ev) {
  if (!cam || !march || !warp || !hash || !field || n_rays < 0 || march->n_samples < 1)
    return set_error(FV_EDIM, "fv_render_fwd: bad arguments");
  if (int32_t e = check_hash(hash)) return e;
  if (int32_t e = check_warp(warp)) return e;
  if (n_rays == 0) return FV_OK;
  const int N = march->n_samples;
  const int64_t S = padded_rays(n_rays) * N;
  if (work_bytes < carve(nullptr, S, field->precision, nullptr))
    return set_error(FV_EDIM, "fv_render_fwd: workspace too small");
  RenderWork w;
  carve(d_work, S, field->precision, &w);
  if (ev) cudaEventRecord(ev[0], st);
  if (int32_t e = march_compact(cam, march, warp, n_rays, w.lik, w.delta, w.xsc, w.idx, w.count, d_count, st)) return e;
  if (ev) cudaEventRecord(ev[1], st);
  if (field->precision == 1) {  // tensor-core field over the foreground stream, count stays on the device
    if (int32_t e = field_fwd_tc(field, hash, w.xsc, S, march->eps_w, w.rgbs, nullptr, st, w.count, w.idx,
                                 ev ? ev[2] : nullptr))
      return e;
  } else {                      // fp32 parity path: host needs the count for its chunked SIMT layers
    if (ev) cudaEventRecord(ev[2], st);
    int32_t n_fg = 0;
    cudaMemcpyAsync(&n_fg, w.count, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("fv_render_fwd count");
    if (n_fg > 0) {
      if (int32_t e = field_fwd(field, hash, w.xsc, n_fg, march->eps_w, w.rgbsc, nullptr, w.fwork, w.fbytes, st))
        return e;
      k_scatter4<<<(unsigned)((n_fg + 255) / 256), 256, 0, st>>>(w.rgbsc, w.idx, n_fg, w.rgbs);
    }
  }
  if (ev) cudaEventRecord(ev[3], st);
  CompIn in{w.rgbs, w.delta, w.lik, 1, true, true};
  const int32_t* out_pix = march->out_by_pixel ? march->d_pix : nullptr;
  if (march->out_by_pixel && !march->d_pix) return set_error(FV_EDIM, "fv_render_fwd: out_by_pixel needs d_pix");
  const int32_t e = composite_fwd(in, n_rays, N, march->bg, march->eps_w, march->eps_t, out_pix, d_rgb, d_alpha,
                                  nullptr, st);
  if (ev) cudaEventRecord(ev[4], st);
  return e;
}

extern "C" int32_t fv_render_fwd(const fv_camera* cam, const fv_march* march, const fv_warp* warp, const fv_hash* hash,
                                 const fv_field* field, int64_t n_rays, void* d_work, size_t work_bytes, float* d_rgb,
                                 float* d_alpha, int32_t* d_count, void* stream) {
  return render_fwd(cam, march, warp, hash, field, n_rays, d_work, work_bytes, d_rgb, d_alpha, d_count,
                    (cudaStream_t)stream, nullptr);
}

// Same render with CUDA events between its stages; synchronises and returns the device
// times (ms) of march+warp, residual MLP, hash+radiance, compositor, total in stage_ms[5]
// and the number of foreground samples the field evaluated in *n_fg.
extern "C" int32_t fv_render_fwd_timed(const fv_camera* cam, const fv_march* march, const fv_warp* warp,
                                       const fv_hash* hash, const fv_field* field, int64_t n_rays, void* d_work,
                                       size_t work_bytes, float* d_rgb, float* d_alpha, float* stage_ms,
                                       int64_t* n_fg, void* stream) {
  cudaEvent_t ev[5];
  for (auto& e : ev) cudaEventCreate(&e);
  cudaStream_t st = (cudaStream_t)stream;
  int32_t err = render_fwd(cam, march, warp, hash, field, n_rays, d_work, work_bytes, d_rgb, d_alpha, nullptr, st, ev);
  if (!err) {
    cudaEventSynchronize(ev[4]);
    float t[4];
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    for (int i = 0; i < 4; ++i) stage_ms[i] = t[i];
    cudaEventElapsedTime(&stage_ms[4], ev[0], ev[4]);
    if (n_fg) {
      RenderWork w;
      carve(d_work, padded_rays(n_rays) * march->n_samples, field->precision, &w);
      int32_t c = 0;
      cudaMemcpy(&c, w.count, sizeof(int32_t), cudaMemcpyDeviceToHost);
      *n_fg = c;
    }
    err = check_launch("fv_render_fwd_timed");
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return err;
}

extern "C" size_t fv_occupancy_workspace_bytes(int32_t precision) {
  return align256((size_t)OCC_PTS * 16) * 2 + (precision == 0 ? field_f32_work_bytes(OCC_PTS) : 0);
}

extern "C" int32_t fv_occupancy_build(const fv_march* march, const fv_warp* warp, const fv_hash* hash,
                                      const fv_field* field, float threshold, void* d_work, size_t work_bytes,
                                      uint32_t* d_occ, void* stream) {
  if (!march || !warp || !hash || !field || !d_occ) return set_error(FV_EDIM, "fv_occupancy_build: null argument");
  if (int32_t e = check_warp(warp)) return e;
  if (work_bytes < fv_occupancy_workspace_bytes(field->precision))
    return set_error(FV_EDIM, "fv_occupancy_build: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* b = (uint8_t*)d_work;
  float4* xs = (float4*)b;
  float4* rgbs = (float4*)(b + align256((size_t)OCC_PTS * 16));
  void* fw = b + 2 * align256((size_t)OCC_PTS * 16);
  k_occ_points<<<OCC_PTS / 128, 128, 0, st>>>(*march, *warp, xs);
  if (int32_t e = check_launch("occ_points")) return e;
  if (int32_t e = field_fwd(field, hash, xs, OCC_PTS, march->eps_w, rgbs, nullptr, fw,
                            field->precision == 0 ? field_f32_work_bytes(OCC_PTS) : 0, st))
    return e;
  k_occ_bits<<<OCC_RES * OCC_RES * OCC_RES / 128, 128, 0, st>>>(xs, rgbs, march->eps_w, threshold, d_occ);
  return check_launch("fv_occupancy_build");
}
