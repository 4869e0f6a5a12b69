// Depth-ordered joint compositing of several independently posed subjects (BASELINE
// config 5; the paper's multi-person future work).  Builder-
// defined, PARITY UNPINNED: the reference has no multi-subject code (S:8).
//
// Each subject is rendered by the single-subject path in its own frame (world camera
// shifted by -offset, background 0), giving per pixel its premultiplied colour C_s and
// alpha_s = 1 - T_s over its box.  Subject boxes are disjoint (scene placement guarantees
// it), so along any ray their sample intervals are disjoint and the front-to-back
// composite of all samples factorises exactly in entry-depth order:
//     C = sum_s (prod_{j before s} T_j) C_s + (prod_s T_s) bg,   alpha = 1 - prod_s T_s.
// Entry depths come from the same float32 ray + slab arithmetic as the ray-march kernel
// (fv_common.cuh), so the order is the one the samples were generated in.
#include <cuda_runtime.h>
#include "fv_common.cuh"
#include "fv_internal.h"

namespace fv {

__global__ void __launch_bounds__(256) k_scene_merge(fv_scene_merge m, int64_t pix0, int64_t n_pix,
                                                     float* __restrict__ rgb, float* __restrict__ alpha) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_pix) return;
  const int64_t p = pix0 + q;                      // pixel id; outputs are image-sized
  float te[FV_MAX_SUBJECTS];
  int ord[FV_MAX_SUBJECTS];
  int nh = 0;
  for (int s = 0; s < m.n_subjects; ++s) {
    const Ray r = make_ray(m.cam[s], (int32_t)p);
    float t0, t1;
    if (!slab(r, m.box_min, m.box_max, t0, t1)) continue;
    int k = nh++;                                  // insertion sort by entry depth (stable in s)
    while (k > 0 && te[k - 1] > t0) { te[k] = te[k - 1]; ord[k] = ord[k - 1]; --k; }
    te[k] = t0;
    ord[k] = s;
  }
  float T = 1.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
  for (int k = 0; k < nh; ++k) {
    const int s = ord[k];
    const float* cs = m.d_rgb[s] + 3 * p;
    c0 = __fadd_rn(c0, __fmul_rn(T, cs[0]));
    c1 = __fadd_rn(c1, __fmul_rn(T, cs[1]));
    c2 = __fadd_rn(c2, __fmul_rn(T, cs[2]));
    T = __fmul_rn(T, __fsub_rn(1.f, m.d_alpha[s][p]));
  }
  rgb[3 * p] = __fadd_rn(c0, __fmul_rn(T, m.bg[0]));
  rgb[3 * p + 1] = __fadd_rn(c1, __fmul_rn(T, m.bg[1]));
  rgb[3 * p + 2] = __fadd_rn(c2, __fmul_rn(T, m.bg[2]));
  alpha[p] = __fsub_rn(1.f, T);
}

}  // namespace fv

using namespace fv;

extern "C" int32_t fv_scene_composite(const fv_scene_merge* m, int64_t pix0, int64_t n_pix, float* d_rgb,
                                      float* d_alpha, void* stream) {
  if (!m || pix0 < 0 || n_pix < 0 || m->n_subjects < 1 || m->n_subjects > FV_MAX_SUBJECTS || !d_rgb || !d_alpha)
    return set_error(FV_EDIM, "fv_scene_composite: bad arguments (1..FV_MAX_SUBJECTS subjects)");
  for (int s = 0; s < m->n_subjects; ++s) {
    if (!m->d_rgb[s] || !m->d_alpha[s]) return set_error(FV_EDIM, "fv_scene_composite: null subject buffer");
    if ((int64_t)m->cam[s].width * m->cam[s].height < pix0 + n_pix)
      return set_error(FV_EDIM, "fv_scene_composite: camera smaller than the pixel count");
  }
  if (n_pix == 0) return FV_OK;
  k_scene_merge<<<(unsigned)((n_pix + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*m, pix0, n_pix, d_rgb, d_alpha);
  return check_launch("fv_scene_composite");
}
