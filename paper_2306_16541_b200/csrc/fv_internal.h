// Internal helpers for the C-ABI layer: thread-local error messages and launch checks.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/fv_api.h"

namespace fv {
struct PeW { float w[8]; };
int32_t set_error(int32_t code, const char* msg);
int32_t check_launch(const char* where);
int32_t check_hash(const fv_hash* h);
// 1 <= K <= FV_MAX_BONES, 2 <= G <= FV_MAX_VOL_RES (packed cell index fits int32)
int32_t check_warp(const fv_warp* w);
int32_t field_fwd_f32(const fv_field* f, const fv_hash* h, const float4* xs, int64_t n, float eps_w, float4* rgbs,
                      float* xfinal, void* work, size_t work_bytes, cudaStream_t st);
size_t field_f32_work_bytes(int64_t n);
int32_t field_fwd_tc(const fv_field* f, const fv_hash* h, const float4* xs, int64_t n, float eps_w, float4* rgbs,
                     float* xfinal, cudaStream_t st, const int32_t* d_count = nullptr, const int32_t* idx = nullptr,
                     cudaEvent_t mid_event = nullptr);
int32_t march_compact(const fv_camera* cam, const fv_march* march, const fv_warp* warp, int64_t n_rays, float* lik,
                      float* delta, float4* xsc, int32_t* idx, int32_t* count, int32_t* ray_count, cudaStream_t st,
                      uint8_t* flags = nullptr);
int32_t march_round(const fv_camera* cam, const fv_march* march, const fv_warp* warp, int64_t n_rays, int32_t i0,
                    int32_t K, const int32_t* live, const int32_t* n_live, float* lik, float* delta, float4* xsc,
                    int32_t* idx, int32_t* count, int32_t* ray_count, cudaStream_t st);
struct CompIn {
  const float4* rgbs;   // [c, sigma] per sample
  const float* delta;   // per sample
  const float* lik;     // per sample, stride lik_stride floats
  int lik_stride;
  bool blocked;         // sample layout: ray-block-major (render) or ray-major [R][N]
  bool skip_bg = false; // L <= eps_w samples are skipped (their rgbs slot is unwritten)
};
int32_t composite_fwd(const CompIn& in, int64_t n_rays, int n, const float* bg, float eps_w, float eps_t,
                      const int32_t* out_pix, float* rgb, float* alpha, float* trans, cudaStream_t st);
int32_t composite_bwd(const CompIn& in, const float* trans, int64_t n_rays, int n, const float* bg, float eps_w,
                      const float* drgb, const float* dalpha, float4* dout, cudaStream_t st);
int32_t composite_round(const float4* rgbs, const float* delta, const float* lik, int K, int i0, int n,
                        const int32_t* live, const int32_t* n_live, int64_t n_rays, const int32_t* ray_count,
                        float4* state, const float* bg, float eps_w, float eps_t, const int32_t* out_pix, float* rgb,
                        float* alpha, int32_t* next_live, int32_t* next_n, cudaStream_t st);
int32_t field_fwd(const fv_field* f, const fv_hash* h, const float4* xs, int64_t n, float eps_w, float4* rgbs,
                  float* xfinal, void* work, size_t work_bytes, cudaStream_t st);
}  // namespace fv
