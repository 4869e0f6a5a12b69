// C-ABI glue: errors, version, the fused render orchestration and the occupancy builder.
#include <cuda_runtime.h>
#include <climits>
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
// Marching rounds (early termination): per-ray state (T, rgb), two live-ray lists with their
// device counts, the per-ray sample counts, one foreground counter per round.
constexpr int kMaxRounds = 64;
struct RoundWork {
  float4* state; int32_t* live[2]; int32_t* n_live; int32_t* ray_count; int32_t* counts;
};

static size_t carve(void* base, int64_t S, int precision, RenderWork* w, int64_t n_rays = 0,
                    RoundWork* rw = nullptr) {
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  const size_t o_l = take((size_t)S * 4), o_d = take((size_t)S * 4), o_r = take((size_t)S * 16);
  const size_t o_x = take((size_t)S * 16), o_i = take((size_t)S * 4), o_c = take(16);
  const size_t o_rc = take(precision == 0 ? (size_t)S * 16 : 0);
  const size_t fb = precision == 0 ? field_f32_work_bytes(S) : 0;
  const size_t o_f = take(fb);
  // round bookkeeping (always reserved: 28 B per ray)
  const size_t o_st = take((size_t)n_rays * 16), o_l0 = take((size_t)n_rays * 4), o_l1 = take((size_t)n_rays * 4);
  const size_t o_rcn = take((size_t)n_rays * 4), o_nl = take(2 * 4), o_cn = take(kMaxRounds * 4);
  uint8_t* b = (uint8_t*)base;
  if (w) {
    w->lik = (float*)(b + o_l); w->delta = (float*)(b + o_d); w->rgbs = (float4*)(b + o_r);
    w->xsc = (float4*)(b + o_x); w->idx = (int32_t*)(b + o_i); w->count = (int32_t*)(b + o_c);
    w->rgbsc = (float4*)(b + o_rc); w->fwork = b + o_f; w->fbytes = fb;
  }
  if (rw) {
    rw->state = (float4*)(b + o_st); rw->live[0] = (int32_t*)(b + o_l0); rw->live[1] = (int32_t*)(b + o_l1);
    rw->ray_count = (int32_t*)(b + o_rcn); rw->n_live = (int32_t*)(b + o_nl); rw->counts = (int32_t*)(b + o_cn);
  }
  return off;
}

static int round_size(const fv_march* m) {
  const int N = m->n_samples, K = m->round_samples;
  if (!(m->eps_t > 0.f) || K <= 0 || K >= N) return N;
  return std::max(K, (N + kMaxRounds - 1) / kMaxRounds);
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
  return carve(nullptr, padded_rays(n_rays) * n_samples, precision, nullptr, n_rays);
}

// Field over one compacted foreground stream (count on the device): tensor cores read the
// count themselves; the fp32 parity path needs it on the host for its chunked SIMT layers.
static int32_t field_stream(const fv_field* field, const fv_hash* hash, const RenderWork& w, int64_t S, float eps_w,
                            int32_t* count, cudaStream_t st, cudaEvent_t mid) {
  if (field->precision == 1)
    return field_fwd_tc(field, hash, w.xsc, S, eps_w, w.rgbs, nullptr, st, count, w.idx, mid);
  if (mid) cudaEventRecord(mid, st);
  int32_t n_fg = 0;
  cudaMemcpyAsync(&n_fg, count, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("fv_render_fwd count");
  if (n_fg > 0) {
    if (int32_t e = field_fwd(field, hash, w.xsc, n_fg, eps_w, w.rgbsc, nullptr, w.fwork, w.fbytes, st)) return e;
    k_scatter4<<<(unsigned)((n_fg + 255) / 256), 256, 0, st>>>(w.rgbsc, w.idx, n_fg, w.rgbs);
  }
  return FV_OK;
}

// ev (optional, 5 events per round): recorded before the march, after the march, between
// the two tensor-core field kernels, after the field and after the compositor (stage timing).
// Single pass (eps_t == 0 or round_samples >= N): march all N samples of every ray, field on
// the foreground stream, composite.  Marching rounds: K samples of every live ray
// per round, field on the round's foreground stream, composite into the rays' persistent
// (T, rgb); rays whose T fell below eps_t retire, so their later samples are never marched,
// warped or evaluated.  Both produce bitwise the same pixels.
static int32_t render_fwd(const fv_camera* cam, const fv_march* march, const fv_warp* warp, const fv_hash* hash,
                          const fv_field* field, int64_t n_rays, void* d_work, size_t work_bytes, float* d_rgb,
                          float* d_alpha, int32_t* d_count, cudaStream_t st, cudaEvent_t* ev, int* n_rounds_out) {
  if (!cam || !march || !warp || !hash || !field || n_rays < 0 || march->n_samples < 1)
    return set_error(FV_EDIM, "fv_render_fwd: bad arguments");
  if (int32_t e = check_hash(hash)) return e;
  if (int32_t e = check_warp(warp)) return e;
  if (n_rays == 0) return FV_OK;
  const int N = march->n_samples;
  if (padded_rays(n_rays) * (int64_t)N > (int64_t)INT32_MAX)
    return set_error(FV_EDIM, "fv_render_fwd: n_rays x n_samples exceeds 2^31 - 1 sample slots (sample ids are "
                              "int32): render the rays in chunks");
  const int K = round_size(march);
  const int64_t S = padded_rays(n_rays) * K;
  if (work_bytes < carve(nullptr, padded_rays(n_rays) * N, field->precision, nullptr, n_rays))
    return set_error(FV_EDIM, "fv_render_fwd: workspace too small");
  RenderWork w;
  RoundWork rw;
  carve(d_work, S, field->precision, &w, n_rays, &rw);
  const int32_t* out_pix = march->out_by_pixel ? march->d_pix : nullptr;
  if (march->out_by_pixel && !march->d_pix) return set_error(FV_EDIM, "fv_render_fwd: out_by_pixel needs d_pix");
  if (K == N) {
    if (n_rounds_out) *n_rounds_out = 1;
    if (ev) cudaEventRecord(ev[0], st);
    if (int32_t e = march_compact(cam, march, warp, n_rays, w.lik, w.delta, w.xsc, w.idx, w.count, d_count, st))
      return e;
    if (ev) cudaEventRecord(ev[1], st);
    if (int32_t e = field_stream(field, hash, w, S, march->eps_w, w.count, st, ev ? ev[2] : nullptr)) return e;
    if (ev) cudaEventRecord(ev[3], st);
    CompIn in{w.rgbs, w.delta, w.lik, 1, true, true};
    const int32_t e = composite_fwd(in, n_rays, N, march->bg, march->eps_w, march->eps_t, out_pix, d_rgb, d_alpha,
                                    nullptr, st);
    if (ev) cudaEventRecord(ev[4], st);
    return e;
  }
  const int rounds = (N + K - 1) / K;
  if (n_rounds_out) *n_rounds_out = rounds;
  for (int r = 0; r < rounds; ++r) {
    const int i0 = r * K, Kr = std::min(K, N - i0);
    const int32_t* live = r == 0 ? nullptr : rw.live[(r + 1) & 1];
    const int32_t* n_live = r == 0 ? nullptr : rw.n_live + ((r + 1) & 1);
    cudaEvent_t* e5 = ev ? ev + 5 * r : nullptr;
    if (e5) cudaEventRecord(e5[0], st);
    if (int32_t e = march_round(cam, march, warp, n_rays, i0, Kr, live, n_live, w.lik, w.delta, w.xsc, w.idx,
                                rw.counts + r, rw.ray_count, st))
      return e;
    if (e5) cudaEventRecord(e5[1], st);
    if (int32_t e = field_stream(field, hash, w, padded_rays(n_rays) * Kr, march->eps_w, rw.counts + r, st,
                                 e5 ? e5[2] : nullptr))
      return e;
    if (e5) cudaEventRecord(e5[3], st);
    if (int32_t e = composite_round(w.rgbs, w.delta, w.lik, Kr, i0, N, live, n_live, n_rays, rw.ray_count, rw.state,
                                    march->bg, march->eps_w, march->eps_t, out_pix, d_rgb, d_alpha, rw.live[r & 1],
                                    rw.n_live + (r & 1), st))
      return e;
    if (e5) cudaEventRecord(e5[4], st);
  }
  if (d_count) cudaMemcpyAsync(d_count, rw.ray_count, (size_t)n_rays * 4, cudaMemcpyDeviceToDevice, st);
  return check_launch("fv_render_fwd rounds");
}

extern "C" int32_t fv_render_fwd(const fv_camera* cam, const fv_march* march, const fv_warp* warp, const fv_hash* hash,
                                 const fv_field* field, int64_t n_rays, void* d_work, size_t work_bytes, float* d_rgb,
                                 float* d_alpha, int32_t* d_count, void* stream) {
  return render_fwd(cam, march, warp, hash, field, n_rays, d_work, work_bytes, d_rgb, d_alpha, d_count,
                    (cudaStream_t)stream, nullptr, nullptr);
}

// Same render with CUDA events between its stages (summed over marching rounds);
// synchronises and returns the device times (ms) of march+warp, residual MLP, hash+radiance,
// compositor, total in stage_ms[5] and the number of foreground samples the field evaluated
// (all rounds) in *n_fg.
extern "C" int32_t fv_render_fwd_timed(const fv_camera* cam, const fv_march* march, const fv_warp* warp,
                                       const fv_hash* hash, const fv_field* field, int64_t n_rays, void* d_work,
                                       size_t work_bytes, float* d_rgb, float* d_alpha, float* stage_ms,
                                       int64_t* n_fg, void* stream) {
  const int max_ev = 5 * kMaxRounds;
  cudaEvent_t ev[5 * kMaxRounds];
  for (int i = 0; i < max_ev; ++i) cudaEventCreate(&ev[i]);
  cudaStream_t st = (cudaStream_t)stream;
  int rounds = 1;
  int32_t err = render_fwd(cam, march, warp, hash, field, n_rays, d_work, work_bytes, d_rgb, d_alpha, nullptr, st, ev,
                           &rounds);
  if (!err) {
    cudaEventSynchronize(ev[5 * rounds - 1]);
    for (int i = 0; i < 5; ++i) stage_ms[i] = 0.f;
    for (int r = 0; r < rounds; ++r) {
      for (int i = 0; i < 4; ++i) {
        float t = 0.f;
        cudaEventElapsedTime(&t, ev[5 * r + i], ev[5 * r + i + 1]);
        stage_ms[i] += t;
      }
    }
    cudaEventElapsedTime(&stage_ms[4], ev[0], ev[5 * rounds - 1]);
    if (n_fg) {
      const int N = march->n_samples, K = round_size(march);
      RenderWork w;
      RoundWork rw;
      carve(d_work, padded_rays(n_rays) * K, field->precision, &w, n_rays, &rw);
      int32_t c[kMaxRounds] = {0};
      if (K == N) cudaMemcpy(c, w.count, sizeof(int32_t), cudaMemcpyDeviceToHost);
      else cudaMemcpy(c, rw.counts, sizeof(int32_t) * rounds, cudaMemcpyDeviceToHost);
      int64_t tot = 0;
      for (int r = 0; r < rounds; ++r) tot += c[r];
      *n_fg = tot;
    }
    err = check_launch("fv_render_fwd_timed");
  }
  for (int i = 0; i < max_ev; ++i) cudaEventDestroy(ev[i]);
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
