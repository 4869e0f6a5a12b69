// Device-side building blocks shared by the freeview sm_100a kernels.
//
// Everything index-critical (ray generation, slab test, sample depths, occupancy cell,
// warp grid coordinates, hash-grid vertex) is written with explicit round-to-nearest
// intrinsics (__fmul_rn / __fadd_rn / __fsub_rn / __fdiv_rn) in the exact order of the
// float32 oracle (oracle/camera.py, oracle/warp.py, oracle/encoding.py), so no FMA
// contraction can change a rounding and integer outputs (sample counts, skip masks,
// hash indices, foreground flags) match the oracle bit for bit.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include "../../include/fv_api.h"

namespace fv {

// Debug builds (-DFV_DEBUG=1; compute-sanitizer is not available on the GPU pool): bounds
// checks on the gathers and staging writes that trap with the failing condition.
#ifndef FV_DEBUG
#define FV_DEBUG 0
#endif
#if FV_DEBUG
#define FV_ASSERT(cond)                                                                     \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("FV_ASSERT %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,      \
             (int)blockIdx.x, (int)threadIdx.x);                                            \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define FV_ASSERT(cond) do {} while (0)
#endif

constexpr uint32_t PRIME_Y = 2654435761u;
constexpr uint32_t PRIME_Z = 805459861u;
constexpr int OCC_RES = 32;

// ---------------------------------------------------------------- camera / sampling
struct Ray { float ox, oy, oz, dx, dy, dz; };

// cap:73-82 restated in float32: d = normalize((K^-1 [px+.5, py+.5, 1]) @ R), o = centre.
__device__ __forceinline__ Ray make_ray(const fv_camera& cam, int32_t pix) {
  const float px = __fadd_rn((float)(pix % cam.width), 0.5f);
  const float py = __fadd_rn((float)(pix / cam.width), 0.5f);
  float dc[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    dc[i] = __fadd_rn(__fadd_rn(__fmul_rn(cam.kinv[3 * i + 0], px), __fmul_rn(cam.kinv[3 * i + 1], py)),
                      cam.kinv[3 * i + 2]);
  float d[3];
#pragma unroll
  for (int j = 0; j < 3; ++j)
    d[j] = __fadd_rn(__fadd_rn(__fmul_rn(dc[0], cam.rot[j]), __fmul_rn(dc[1], cam.rot[3 + j])),
                     __fmul_rn(dc[2], cam.rot[6 + j]));
  const float n = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(d[0], d[0]), __fmul_rn(d[1], d[1])),
                                       __fmul_rn(d[2], d[2])));
  Ray r;
  r.ox = cam.center[0]; r.oy = cam.center[1]; r.oz = cam.center[2];
  r.dx = __fdiv_rn(d[0], n); r.dy = __fdiv_rn(d[1], n); r.dz = __fdiv_rn(d[2], n);
  return r;
}

// Slab test; fminf/fmaxf ignore the NaN of 0*inf exactly like numpy fmin/fmax.
__device__ __forceinline__ bool slab(const Ray& r, const float* bmin, const float* bmax,
                                     float& t_enter, float& t_exit) {
  const float o[3] = {r.ox, r.oy, r.oz};
  const float d[3] = {r.dx, r.dy, r.dz};
  float tn[3], tf[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float inv = __fdiv_rn(1.0f, d[j]);
    const float t0 = __fmul_rn(__fsub_rn(bmin[j], o[j]), inv);
    const float t1 = __fmul_rn(__fsub_rn(bmax[j], o[j]), inv);
    tn[j] = fminf(t0, t1);
    tf[j] = fmaxf(t0, t1);
  }
  t_enter = fmaxf(fmaxf(fmaxf(tn[0], tn[1]), tn[2]), 0.0f);
  t_exit = fminf(fminf(tf[0], tf[1]), tf[2]);
  return t_exit > t_enter;
}

__device__ __forceinline__ uint32_t hash_u32(uint32_t seed, uint32_t pix, uint32_t i) {
  uint32_t h = seed ^ (pix * 0x9E3779B1u) ^ ((i + 1u) * 0x85EBCA77u);
  h ^= h >> 16; h *= 0x7FEB352Du;
  h ^= h >> 15; h *= 0x846CA68Bu;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ float jitter_u(uint32_t seed, uint32_t pix, uint32_t i) {
  return __fmul_rn((float)(hash_u32(seed, pix, i) >> 8), 5.9604644775390625e-08f);  // 2^-24
}

// t_i = t_enter + (i + u_i) * step
__device__ __forceinline__ float sample_t(float t_enter, float step, int i, float u) {
  return __fadd_rn(t_enter, __fmul_rn(__fadd_rn((float)i, u), step));
}

__device__ __forceinline__ bool occ_test(const uint32_t* occ, const float* bmin, const float* scale,
                                         float x, float y, float z) {
  const float p[3] = {x, y, z};
  int c[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float q = floorf(__fmul_rn(__fsub_rn(p[j], bmin[j]), scale[j]));
    c[j] = q < 0.f ? 0 : (q > (float)(OCC_RES - 1) ? OCC_RES - 1 : (int)q);
  }
  const int cell = (c[0] * OCC_RES + c[1]) * OCC_RES + c[2];
  return (__ldg(occ + (cell >> 5)) >> (cell & 31)) & 1u;
}

// ---------------------------------------------------------------- skeleton warp
#ifndef FV_WARP_UNROLL
#define FV_WARP_UNROLL 2
#endif
constexpr int kWarpUnroll = FV_WARP_UNROLL;

// Corner-packed weight volume: for channel i and padded-grid cell (ix,iy,iz) in [0,G]^3 the
// 8 corner values vp[i, ix+a, iy+b, iz+c] are stored contiguously (one 16-byte word in fp16,
// two in fp32) as x-pairs Z_q = (v[0,b,c], v[1,b,c]), q = 2b + c (k_warp_pack), so one
// gather replaces the 8 of ad:767-773.  load_corners returns them in a*4+b*2+c order.
__device__ __forceinline__ void load_corners_x2(const void* vol, int half, size_t cell, float2 (&z)[4]) {
  if (half) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(vol) + cell);
    const __half2* h = reinterpret_cast<const __half2*>(&w);
#pragma unroll
    for (int q = 0; q < 4; ++q) z[q] = __half22float2(h[q]);
  } else {
    const float4 a = __ldg(reinterpret_cast<const float4*>(vol) + 2 * cell);
    const float4 b = __ldg(reinterpret_cast<const float4*>(vol) + 2 * cell + 1);
    z[0] = make_float2(a.x, a.y); z[1] = make_float2(a.z, a.w); z[2] = make_float2(b.x, b.y); z[3] = make_float2(b.z, b.w);
  }
}

__device__ __forceinline__ void load_corners(const void* vol, int half, size_t cell, float (&cv)[8]) {
  float2 z[4];
  load_corners_x2(vol, half, cell, z);
#pragma unroll
  for (int q = 0; q < 4; ++q) { cv[q] = z[q].x; cv[4 + q] = z[q].y; }
}

// Grid coordinates of bone point p for the volume (ad:746-753); returns inside flag.
__device__ __forceinline__ bool warp_cell(const fv_warp& w, const float (&p)[3], int (&i0)[3], float (&f)[3]) {
  bool inside = true;
  const float gp1 = (float)(w.vol_res + 1);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float u = __fmaf_rn(__fsub_rn(p[j], w.wbox_min[j]), w.wscale[j], 1.0f);
    inside = inside && (u >= 0.0f) && (u <= gp1);
    float fl = floorf(u);
    fl = fl < 0.f ? 0.f : (fl > (float)w.vol_res ? (float)w.vol_res : fl);
    i0[j] = (int)fl;
    f[j] = __fsub_rn(u, fl);
  }
  return inside;
}

// Trilinear blend of ad:767-773 as seven lerps v0 + f (v1 - v0), each one FMA
// (oracle.warp._lerp32): z, then y, then x.
__device__ __forceinline__ float lerp_fma(float v0, float v1, float t) {
  return __fmaf_rn(t, __fsub_rn(v1, v0), v0);
}

__device__ __forceinline__ float trilerp8(const float (&f)[3], const float (&cv)[8]) {
  const float c00 = lerp_fma(cv[0], cv[1], f[2]), c01 = lerp_fma(cv[2], cv[3], f[2]);
  const float c10 = lerp_fma(cv[4], cv[5], f[2]), c11 = lerp_fma(cv[6], cv[7], f[2]);
  return lerp_fma(lerp_fma(c00, c01, f[1]), lerp_fma(c10, c11, f[1]), f[0]);
}

// <= 32 bones x 129^3 cells fits int32 (fv_warp_pack checks the volume size)
__device__ __forceinline__ size_t vol_cell_index(int bone, int res, const int (&i0)[3]) {
  const int s = res + 1;
  return (size_t)(unsigned)(((bone * s + i0[0]) * s + i0[1]) * s + i0[2]);
}

// Bone transforms in shared memory for warp_point: per bone the 12 floats of G_i
// (R row-major, t) reordered as [R00 R10 R01 R11 | R02 R12 t0 t1 | R20 R21 R22 t2], so rows
// 0 and 1 of p = x R^T + t go through one packed f32x2 FMA chain (nibble table below).
__device__ __forceinline__ void fill_bones_x2(float* sg, const float* g, int n_bones) {
  for (int i = threadIdx.x; i < n_bones * 12; i += blockDim.x) {
    const int b = i / 12, k = i % 12;
    sg[i] = g[b * 12 + (int)((0xB876A9524130ull >> (4 * k)) & 15u)];
  }
}

// p = x @ R^T + t (row convention, sk:171-172) on the fill_bones_x2 layout: the FMA chain of
// oracle.warp.bone_points, rows 0/1 as packed f32x2 (per lane the scalar operations)
__device__ __forceinline__ void bone_point_x2(const float* g, float x0, float x1, float x2, float (&p)[3]) {
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4 a = g4[0], b = g4[1], c = g4[2];
  const float2 p01 = __fadd2_rn(__ffma2_rn(make_float2(b.x, b.y), make_float2(x2, x2),
                                           __ffma2_rn(make_float2(a.z, a.w), make_float2(x1, x1),
                                                      __fmul2_rn(make_float2(a.x, a.y), make_float2(x0, x0)))),
                                make_float2(b.z, b.w));
  p[0] = p01.x;
  p[1] = p01.y;
  p[2] = __fadd_rn(__fmaf_rn(c.z, x2, __fmaf_rn(c.y, x1, __fmul_rn(c.x, x0))), c.w);
}

// v0 + t (v1 - v0) on two lanes; v1 - v0 as fma(v0, -1, v1) (exact product, one rounding),
// so each lane is bitwise lerp_fma.
__device__ __forceinline__ float2 lerp_fma2(float2 v0, float2 v1, float2 t) {
  return __ffma2_rn(t, __ffma2_rn(v0, make_float2(-1.f, -1.f), v1), v0);
}

// Full skeleton warp of one point with G in shared memory (sg: K*12 floats, fill_bones_x2).
// Returns L; xs = sum_i w_i p_i / L (0 if L <= eps_w).  Optional per-bone weights out.
// Per bone, the x/y coordinates of the bone point and grid position, the three lerp levels
// of the trilinear blend (over x-pairs of corners) and the (s0, s1) accumulation run as
// packed f32x2 FMAs: each lane performs exactly the scalar operation of bone_point_x2 /
// warp_cell / trilerp8 (oracle.warp), so results are unchanged bit for bit.
template <bool STORE_W, int HALF = -1>
__device__ __forceinline__ float warp_point(const fv_warp& w, const float* sg, float eps_w,
                                            float x0, float x1, float x2, float (&xs)[3],
                                            float* w_out = nullptr, size_t w_stride = 0) {
  float lik = 0.f, s2 = 0.f;
  float2 s01 = make_float2(0.f, 0.f);
  const int K = w.n_bones;
  const int G = w.vol_res;
  const float gp1 = (float)(G + 1), gmax = (float)G;
  const float2 nmin01 = make_float2(-w.wbox_min[0], -w.wbox_min[1]), sc01 = make_float2(w.wscale[0], w.wscale[1]);
  const float2 one2 = make_float2(1.f, 1.f), mone2 = make_float2(-1.f, -1.f);
  const float2 X0 = make_float2(x0, x0), X1 = make_float2(x1, x1), X2 = make_float2(x2, x2);
  const int half = HALF < 0 ? w.vol_half : HALF;
  // cell index from the bit patterns of t = u_clamped +rd 2^23 (bits = 0x4B000000 + floor):
  // idx = ((i s + fx) s + fy) s + fz with the 0x4B000000 (s^2 + s + 1) bias folded into the
  // per-bone base (uint32 wrap-around; the true index fits)
  const uint32_t s1 = (uint32_t)G + 1u, s2c = s1 * s1;
  const uint32_t bias = 0x4B000000u * (s2c + s1 + 1u);
  const uint32_t gbits = __float_as_uint(gp1);
#pragma unroll kWarpUnroll
  for (int i = 0; i < K; ++i) {
    const float4* g4 = reinterpret_cast<const float4*>(sg + 12 * i);   // 48-byte rows
    const float4 a = g4[0], b = g4[1], c = g4[2];
    // p01 = (x R^T + t)[0..1], p2 (bone_point's FMA chain)
    const float2 p01 = __fadd2_rn(__ffma2_rn(make_float2(b.x, b.y), X2,
                                             __ffma2_rn(make_float2(a.z, a.w), X1, __fmul2_rn(make_float2(a.x, a.y), X0))),
                                  make_float2(b.z, b.w));
    const float p2 = __fadd_rn(__fmaf_rn(c.z, x2, __fmaf_rn(c.y, x1, __fmul_rn(c.x, x0))), c.w);
    // grid position (warp_cell): u = (p - min) * scale + 1, inside iff u in [0, G+1]
    const float2 u01 = __ffma2_rn(__fadd2_rn(p01, nmin01), sc01, one2);
    const float u2 = __fmaf_rn(__fsub_rn(p2, w.wbox_min[2]), w.wscale[2], 1.0f);
    // inside <=> 0 <= u <= G+1 on all axes <=> max of the bit patterns <= bits(G+1): u >= 0
    // has the sign bit clear (u = q s + 1 never rounds to -0) and NaN / negative patterns
    // compare above.  For an inside u only the top clamp remains, and floor needs no XU op:
    // t = min(u, G) +rd 2^23 holds floor in its low mantissa bits, fl = t - 2^23 exactly and
    // fr = u - fl exactly (= warp_cell).
    const bool inside = max(max(__float_as_uint(u01.x), __float_as_uint(u01.y)), __float_as_uint(u2)) <= gbits;
    float wi = 0.f;
    if (inside) {
      const float t0 = __fadd_rd(fminf(u01.x, gmax), 8388608.f);
      const float t1 = __fadd_rd(fminf(u01.y, gmax), 8388608.f);
      const float t2 = __fadd_rd(fminf(u2, gmax), 8388608.f);
      const float2 fl01 = __fadd2_rn(make_float2(t0, t1), make_float2(-8388608.f, -8388608.f));
      const float2 fr01 = __ffma2_rn(fl01, mone2, u01);                       // u - floor(u)
      const float fr2 = __fsub_rn(u2, __fsub_rn(t2, 8388608.f));
      const uint32_t cell = ((uint32_t)i * s1 * s2c - bias) + __float_as_uint(t0) * s2c +
                            __float_as_uint(t1) * s1 + __float_as_uint(t2);
      FV_ASSERT(cell < (uint32_t)K * s1 * s2c);
      float2 z[4];
      load_corners_x2(w.d_vol_packed, half, (size_t)cell, z);
      const float2 tz = make_float2(fr2, fr2), ty = make_float2(fr01.y, fr01.y);
      const float2 q = lerp_fma2(lerp_fma2(z[0], z[1], tz), lerp_fma2(z[2], z[3], tz), ty);   // (c_{a=0}, c_{a=1})
      wi = lerp_fma(q.x, q.y, fr01.x);
    }
    if (STORE_W) w_out[(size_t)i * w_stride] = wi;
    lik = __fadd_rn(lik, wi);
    s01 = __ffma2_rn(make_float2(wi, wi), p01, s01);
    s2 = __fmaf_rn(wi, p2, s2);
  }
  if (lik > eps_w) {
    xs[0] = __fdiv_rn(s01.x, lik); xs[1] = __fdiv_rn(s01.y, lik); xs[2] = __fdiv_rn(s2, lik);
  } else {
    xs[0] = xs[1] = xs[2] = 0.f;
  }
  return lik;
}

// ---------------------------------------------------------------- warp aggregation
// Sum v over each run of consecutive lanes holding the same key (segmented inclusive scan,
// 5 shuffle steps); returns true on the run's last lane, which then holds the run total.
// Lanes of one key that are not contiguous form several runs (each still correct).  The
// backward kernels' warps are 32 neighbouring rays of a patch row at one depth, so a
// cell's lanes are contiguous and this replaces one serial leader loop per group.
template <int N, typename K>
__device__ __forceinline__ bool seg_sum(float (&v)[N], K key, int lane) {
  const K prev = __shfl_up_sync(0xffffffffu, key, 1);
  const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || prev != key);
  if (heads == 0xffffffffu) return true;            // all runs of one (fine levels): nothing to sum
  const int start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
  // the longest run bounds the scan depth: skip the shuffle steps no run needs
  const int longest = (int)__reduce_max_sync(0xffffffffu, (unsigned)(lane - start + 1));
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    if (d >= longest) break;
    const bool add = lane - d >= start;
#pragma unroll
    for (int j = 0; j + 1 < N; j += 2) {   // pairs of values: one packed f32x2 add
      const float2 y = make_float2(__shfl_up_sync(0xffffffffu, v[j], d), __shfl_up_sync(0xffffffffu, v[j + 1], d));
      if (add) {
        const float2 r = __fadd2_rn(make_float2(v[j], v[j + 1]), y);
        v[j] = r.x;
        v[j + 1] = r.y;
      }
    }
    if (N & 1) {
      const float y = __shfl_up_sync(0xffffffffu, v[N - 1], d);
      if (add) v[N - 1] += y;
    }
  }
  return lane == 31 || ((heads >> (lane + 1)) & 1u);
}

// ---------------------------------------------------------------- hash grid
struct HashCell { int i0[3]; float f[3]; };

__device__ __forceinline__ void hash_norm(const fv_hash& h, float x0, float x1, float x2, float (&xn)[3],
                                          bool (&mask)[3]) {
  const float x[3] = {x0, x1, x2};
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float raw = __fmul_rn(__fsub_rn(x[j], h.cmin[j]), h.cinv[j]);
    mask[j] = (raw >= 0.f) && (raw <= 1.f);
    xn[j] = fminf(fmaxf(raw, 0.f), 1.f);
  }
}

__device__ __forceinline__ void hash_level_cell(const float (&xn)[3], int res, HashCell& c) {
  const float rf = (float)res;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float pos = __fmul_rn(xn[j], rf);
    float fl = floorf(pos);
    fl = fminf(fl, rf - 1.0f);
    c.i0[j] = (int)fl;
    c.f[j] = __fsub_rn(pos, fl);
  }
}

__device__ __forceinline__ uint32_t hash_index(int dense, int res, uint32_t mask_T, uint32_t x, uint32_t y,
                                               uint32_t z) {
  if (dense) {
    const uint32_t s = (uint32_t)res + 1u;
    return x + y * s + z * (s * s);
  }
  return (x ^ (y * PRIME_Y) ^ (z * PRIME_Z)) & mask_T;
}

// Features of one level (F = 2).
__device__ __forceinline__ float2 hash_level_feat(const fv_hash& h, int l, const HashCell& c,
                                                  uint32_t* idx_out = nullptr) {
  const float wx[2] = {__fsub_rn(1.0f, c.f[0]), c.f[0]};
  const float wy[2] = {__fsub_rn(1.0f, c.f[1]), c.f[1]};
  const float wz[2] = {__fsub_rn(1.0f, c.f[2]), c.f[2]};
  const uint32_t maskT = (1u << h.log2_T) - 1u;
  const uint32_t off = h.offset[l];
  uint32_t gidx[8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
        gidx[a * 4 + b * 2 + cc] = off + hash_index(h.dense[l], h.res[l], maskT, c.i0[0] + a, c.i0[1] + b, c.i0[2] + cc);
#if FV_DEBUG
#pragma unroll
  for (int q = 0; q < 8; ++q)
    FV_ASSERT(gidx[q] - off < (h.dense[l] ? (uint32_t)(h.res[l] + 1) * (h.res[l] + 1) * (h.res[l] + 1) : maskT + 1u));
#endif
  float2 v[8];
  if (h.table_half) {
    const __half2* t = reinterpret_cast<const __half2*>(h.d_table);
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __half22float2(__ldg(t + gidx[q]));
  } else {
    const float2* t = reinterpret_cast<const float2*>(h.d_table);
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldg(t + gidx[q]);
  }
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const float wgt = __fmul_rn(__fmul_rn(wx[a], wy[b]), wz[cc]);
        const int q = a * 4 + b * 2 + cc;
        acc.x = __fadd_rn(acc.x, __fmul_rn(wgt, v[q].x));
        acc.y = __fadd_rn(acc.y, __fmul_rn(wgt, v[q].y));
      }
  if (idx_out) {
#pragma unroll
    for (int q = 0; q < 8; ++q) idx_out[q] = gidx[q];
  }
  return acc;
}

// Lane-paired gathers of NL levels (fp16 or fp32 table): lanes (2p, 2p+1) serve the
// samples of both lanes; lane parity a = lane & 1 fetches the x-corner a of each sample.  A
// cell's two x-corners differ only in low index bits (same 128-byte line ~99% of the time),
// so in one warp instruction 16 samples x 2 corners touch 16 lines instead of 32 -- half
// the L1 wavefronts of the per-sample form at the same load count.  8 NL independent gathers
// are in flight per thread before any is consumed.  Corner indices are strength-reduced
// (y+1 -> +PRIME_Y or +s, z+1 -> +PRIME_Z or +s^2, same uint32 arithmetic as hash_index)
// and each lane blends its four corners as lerps (z, then y) scaled by its x weight; one
// shuffle per feature adds the partner's partial.  The blend order differs from the
// oracle's (a,b,c) sum by fp32 rounding only: used where features are rounded to fp16.
// IDX (verification only, k_hash_index_paired): also return the global table index of every
// corner this lane fetches, idx_out[q * 8 + k] (sample A) and idx_out[q * 8 + 4 + k] (sample
// B) for x-corner a = lane parity and k = 2 b + c.
template <int NL, bool IDX = false>
__device__ __forceinline__ void hash_levels_paired(const fv_hash& h, int l0, const float (&xn_self)[3],
                                                   float2 (&out)[NL], uint32_t* idx_out = nullptr) {
  const uint32_t maskT = (1u << h.log2_T) - 1u;
  const uint32_t a = threadIdx.x & 1u;
  // A = the even lane's sample, B = the odd lane's, for both lanes of a pair: each load
  // instruction then has the pair fetching the two x-corners of the same sample
  float xA[3], xB[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float other = __shfl_xor_sync(0xffffffffu, xn_self[j], 1);
    xA[j] = a ? other : xn_self[j];
    xB[j] = a ? xn_self[j] : other;
  }
  const float wsgn = a ? 1.f : -1.f, wbase = a ? 0.f : 1.f;   // w_x(a) = wbase + wsgn * f_x
  uint32_t iA[4 * NL], iB[4 * NL];
  uint32_t lofs[NL];
  float fA[NL][3], fB[NL][3];
#pragma unroll
  for (int q = 0; q < NL; ++q) {
    const int l = l0 + q < h.n_levels ? l0 + q : h.n_levels - 1;
    const int res = h.res[l];
    lofs[q] = h.offset[l];
    HashCell cA, cB;
    hash_level_cell(xA, res, cA);
    hash_level_cell(xB, res, cB);
#pragma unroll
    for (int j = 0; j < 3; ++j) { fA[q][j] = cA.f[j]; fB[q][j] = cB.f[j]; }
    const uint32_t xa = (uint32_t)cA.i0[0] + a, xb = (uint32_t)cB.i0[0] + a;
    if (h.dense[l]) {
      const uint32_t sy = (uint32_t)res + 1u, sz = sy * sy;
      const uint32_t bA = xa + (uint32_t)cA.i0[1] * sy + (uint32_t)cA.i0[2] * sz;
      const uint32_t bB = xb + (uint32_t)cB.i0[1] * sy + (uint32_t)cB.i0[2] * sz;
      iA[q * 4 + 0] = bA; iA[q * 4 + 1] = bA + sz; iA[q * 4 + 2] = bA + sy; iA[q * 4 + 3] = bA + sy + sz;
      iB[q * 4 + 0] = bB; iB[q * 4 + 1] = bB + sz; iB[q * 4 + 2] = bB + sy; iB[q * 4 + 3] = bB + sy + sz;
    } else {
      const uint32_t yA0 = (uint32_t)cA.i0[1] * PRIME_Y, yA1 = yA0 + PRIME_Y;
      const uint32_t zA0 = (uint32_t)cA.i0[2] * PRIME_Z, zA1 = zA0 + PRIME_Z;
      const uint32_t yB0 = (uint32_t)cB.i0[1] * PRIME_Y, yB1 = yB0 + PRIME_Y;
      const uint32_t zB0 = (uint32_t)cB.i0[2] * PRIME_Z, zB1 = zB0 + PRIME_Z;
      iA[q * 4 + 0] = (xa ^ yA0 ^ zA0) & maskT; iA[q * 4 + 1] = (xa ^ yA0 ^ zA1) & maskT;
      iA[q * 4 + 2] = (xa ^ yA1 ^ zA0) & maskT; iA[q * 4 + 3] = (xa ^ yA1 ^ zA1) & maskT;
      iB[q * 4 + 0] = (xb ^ yB0 ^ zB0) & maskT; iB[q * 4 + 1] = (xb ^ yB0 ^ zB1) & maskT;
      iB[q * 4 + 2] = (xb ^ yB1 ^ zB0) & maskT; iB[q * 4 + 3] = (xb ^ yB1 ^ zB1) & maskT;
    }
  }
#if FV_DEBUG
#pragma unroll
  for (int q = 0; q < NL; ++q) {
    const int l = l0 + q < h.n_levels ? l0 + q : h.n_levels - 1;
    const uint32_t lim = h.dense[l] ? (uint32_t)(h.res[l] + 1) * (h.res[l] + 1) * (h.res[l] + 1) : maskT + 1u;
#pragma unroll
    for (int k = 0; k < 4; ++k) FV_ASSERT(iA[q * 4 + k] < lim && iB[q * 4 + k] < lim);
  }
#endif
  if constexpr (IDX) {
#pragma unroll
    for (int q = 0; q < NL; ++q)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        idx_out[q * 8 + k] = lofs[q] + iA[q * 4 + k];
        idx_out[q * 8 + 4 + k] = lofs[q] + iB[q * 4 + k];
      }
  }
  float2 vA[4 * NL], vB[4 * NL];
  if (h.table_half) {
#pragma unroll
    for (int q = 0; q < NL; ++q) {
      const __half2* t = reinterpret_cast<const __half2*>(h.d_table) + lofs[q];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        vA[q * 4 + k] = __half22float2(__ldg(t + iA[q * 4 + k]));
        vB[q * 4 + k] = __half22float2(__ldg(t + iB[q * 4 + k]));
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < NL; ++q) {
      const float2* t = reinterpret_cast<const float2*>(h.d_table) + lofs[q];
#pragma unroll
      for (int k = 0; k < 4; ++k) { vA[q * 4 + k] = __ldg(t + iA[q * 4 + k]); vB[q * 4 + k] = __ldg(t + iB[q * 4 + k]); }
    }
  }
#pragma unroll
  for (int q = 0; q < NL; ++q) {
    // corners k = 2b + c of this lane's x-corner a: lerp in z (c), then y (b), scale by w_x(a)
    const float2* va = vA + q * 4;
    const float2* vb = vB + q * 4;
    float2 pA, pB;
    {
      const float fy = fA[q][1], fz = fA[q][2];
      const float c0x = fmaf(fz, va[1].x - va[0].x, va[0].x), c0y = fmaf(fz, va[1].y - va[0].y, va[0].y);
      const float c1x = fmaf(fz, va[3].x - va[2].x, va[2].x), c1y = fmaf(fz, va[3].y - va[2].y, va[2].y);
      const float wx = fmaf(wsgn, fA[q][0], wbase);
      pA = make_float2(wx * fmaf(fy, c1x - c0x, c0x), wx * fmaf(fy, c1y - c0y, c0y));
    }
    {
      const float fy = fB[q][1], fz = fB[q][2];
      const float c0x = fmaf(fz, vb[1].x - vb[0].x, vb[0].x), c0y = fmaf(fz, vb[1].y - vb[0].y, vb[0].y);
      const float c1x = fmaf(fz, vb[3].x - vb[2].x, vb[2].x), c1y = fmaf(fz, vb[3].y - vb[2].y, vb[2].y);
      const float wx = fmaf(wsgn, fB[q][0], wbase);
      pB = make_float2(wx * fmaf(fy, c1x - c0x, c0x), wx * fmaf(fy, c1y - c0y, c0y));
    }
    // even lane keeps sample A: own a=0 partial of A + partner's a=1 partial of A
    const float sx = a ? pA.x : pB.x, sy = a ? pA.y : pB.y;      // what the partner needs
    const float rx = __shfl_xor_sync(0xffffffffu, sx, 1), ry = __shfl_xor_sync(0xffffffffu, sy, 1);
    const float2 mine = a ? pB : pA;
    out[q] = l0 + q < h.n_levels ? make_float2(mine.x + rx, mine.y + ry) : make_float2(0.f, 0.f);
  }
}

// ---------------------------------------------------------------- heads
__device__ __forceinline__ float sigmoidf_(float x) {
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}
__device__ __forceinline__ float softplusf_(float x) { return log1pf(expf(-fabsf(x))) + fmaxf(x, 0.f); }

// MUFU forms for the fp16 tensor-core field (absolute error ~1e-7, far inside its 1e-3 bar)
__device__ __forceinline__ float sigmoid_fast(float x) { return __frcp_rn(1.f + __expf(-x)); }
__device__ __forceinline__ float softplus_fast(float x) { return __logf(1.f + __expf(-fabsf(x))) + fmaxf(x, 0.f); }

}  // namespace fv
