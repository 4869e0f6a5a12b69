// Sample layout shared by the march, field and composite kernels.
//
// Rays are grouped in blocks of RB = 32 rays; sample i of ray (block b, lane l) lives at
//     s = (b * N + i) * RB + l
// so one warp of 32 consecutive samples holds 32 neighbouring rays at the same depth
// index: their world points, bone points and canonical points are spatially close,
// which keeps the weight-volume and hash-table gathers on few cache lines (full frames
// are traversed in 8x4 pixel tiles, see render.py).  A 128-row MMA tile = 4 depths x 32 rays.
#pragma once
#include <cstdint>

namespace fv {
constexpr int RB = 32;

__host__ __device__ __forceinline__ int64_t padded_rays(int64_t n_rays) {
  return (n_rays + RB - 1) / RB * RB;
}
__host__ __device__ __forceinline__ int64_t sample_index(int64_t ray, int32_t i, int32_t n) {
  return ((ray / RB) * n + i) * RB + (ray % RB);
}
__host__ __device__ __forceinline__ void sample_coords(int64_t s, int32_t n, int64_t& ray, int32_t& i) {
  const int64_t l = s % RB;
  const int64_t q = s / RB;
  i = (int32_t)(q % n);
  ray = (q / n) * RB + l;
}
}  // namespace fv
