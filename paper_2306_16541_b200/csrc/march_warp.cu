// Ray march + skeleton warp kernels (S:410-413 sampling, S:327-336 warp; ad:728-773).
#include <climits>
#include <cuda_runtime.h>
#include "fv_common.cuh"
#include "layout.cuh"
#include "fv_internal.h"

namespace fv {

// W^c (C,G,G,G) -> corner-packed [K][(G+1)^3][8], zero padding of ad:755-756 folded in.
// Corner order within a cell: x-pairs Z_q = (v[0,b,c], v[1,b,c]) for q = 2b + c, i.e. the
// a*4+b*2+c indices (0,4, 1,5, 2,6, 3,7), so the blend runs as packed f32x2 lerps.
template <typename T>
__global__ void k_warp_pack(const float* __restrict__ vol, int K, int G, T* __restrict__ out) {
  const int s = G + 1;
  const int64_t total = (int64_t)K * s * s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = e;
    const int iz = q % s; q /= s;
    const int iy = q % s; q /= s;
    const int ix = q % s; q /= s;
    const int ch = (int)q;
    float v[8];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          // padded index (ix+a, iy+b, iz+c) -> original (.. - 1)
          const int x = ix + a - 1, y = iy + b - 1, z = iz + c - 1;
          const bool in = x >= 0 && x < G && y >= 0 && y < G && z >= 0 && z < G;
          v[a * 4 + b * 2 + c] = in ? vol[(((int64_t)ch * G + x) * G + y) * G + z] : 0.f;
        }
    if constexpr (sizeof(T) == 2) {
      __half2 h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) h[q] = __floats2half2_rn(v[q], v[4 + q]);
      reinterpret_cast<uint4*>(out)[e] = *reinterpret_cast<uint4*>(h);
    } else {
      float4* o = reinterpret_cast<float4*>(out) + 2 * e;
      o[0] = make_float4(v[0], v[4], v[1], v[5]);
      o[1] = make_float4(v[2], v[6], v[3], v[7]);
    }
  }
}

__global__ void k_warp_fwd(fv_warp w, float eps_w, const float* __restrict__ x, int64_t n,
                           float* __restrict__ xskel, float* __restrict__ lik, uint8_t* __restrict__ fg,
                           float* __restrict__ wout) {
  __shared__ __align__(16) float sg[FV_MAX_BONES * 12];
  fill_bones_x2(sg, w.d_g, w.n_bones);
  __syncthreads();
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  float xs[3];
  float L;
  if (wout) L = warp_point<true>(w, sg, eps_w, x[3 * p], x[3 * p + 1], x[3 * p + 2], xs, wout + p, (size_t)n);
  else L = warp_point<false>(w, sg, eps_w, x[3 * p], x[3 * p + 1], x[3 * p + 2], xs);
  xskel[3 * p] = xs[0]; xskel[3 * p + 1] = xs[1]; xskel[3 * p + 2] = xs[2];
  lik[p] = L;
  fg[p] = L > eps_w;
}

// Compacted foreground stream written by the render march (COMPACT): fg samples only.
struct Compact {
  float* lik;        // [S] likelihood of every sample (0 outside box / empty cell)
  float4* xsc;       // [<= S] (x_skel, L) of foreground samples
  int32_t* idx;      // [<= S] their sample index
  int32_t* count;    // device counter (zeroed before the launch)
  uint8_t* flags;    // optional [S] per-sample bits: 1 ray hits the box, 2 occupancy cell on
                     // (or no grid), 4 foreground (L > eps_w) -- the skip/fg masks for parity
};

// One marching round (early termination): samples [i0, i0 + K) of the rays in a
// live list.  Slot layout as layout.cuh with K samples per ray and the live-list position j
// in place of the ray: s = ((j / 32) K + (i - i0)) 32 + j % 32.  live == NULL: every ray
// (j = ray), the single-pass render (i0 = 0, K = N).
struct MarchRound {
  int32_t i0, K;
  const int32_t* live;     // [n_live] ray ids, or NULL
  const int32_t* n_live;   // device count of live rays (NULL: n_rays)
};

// Per-ray setup of a slot: ray id, pixel, direction, slab interval and bin width (make_ray /
// slab / step of the oracle).
struct RaySetup {
  float dx, dy, dz, t0, t1, step;
  int32_t pix, ray;      // ray < 0: no ray (padding or past the live count)
};

__device__ __forceinline__ RaySetup ray_setup(const fv_camera& cam, const fv_march& m, const MarchRound& rd,
                                              int64_t j, int64_t n_j, bool& hit) {
  RaySetup q;
  q.ray = -1; q.pix = 0; q.dx = q.dy = q.dz = q.t0 = q.t1 = q.step = 0.f;
  hit = false;
  if (j < n_j) {
    const int64_t ray = rd.live ? (int64_t)rd.live[j] : j;
    const int32_t pix = m.d_pix ? m.d_pix[ray] : (int32_t)(m.pix_offset + ray);
    const Ray r = make_ray(cam, pix);
    float t0, t1;
    hit = slab(r, m.obox_min, m.obox_max, t0, t1);
    q.ray = (int32_t)ray; q.pix = pix;
    q.dx = r.dx; q.dy = r.dy; q.dz = r.dz; q.t0 = t0; q.t1 = t1;
    q.step = hit ? __fdiv_rn(__fsub_rn(t1, t0), (float)m.n_samples) : 0.f;
  }
  return q;
}

// Branch-free occ_test (same float32 cell index: floor, clamp to [0, 31]).
__device__ __forceinline__ bool occ_test_nb(const uint32_t* occ, const float* bmin, const float* scale, float x,
                                            float y, float z) {
  const float p[3] = {x, y, z};
  int c[3];
#pragma unroll
  for (int j = 0; j < 3; ++j)
    c[j] = (int)fminf(fmaxf(floorf(__fmul_rn(__fsub_rn(p[j], bmin[j]), scale[j])), 0.f), (float)(OCC_RES - 1));
  const int cell = (c[0] * OCC_RES + c[1]) * OCC_RES + c[2];
  return (__ldg(occ + (cell >> 5)) >> (cell & 31)) & 1u;
}

// One thread per sample slot.  Writes xs[s] = (x_skel, L) with L = 0 for samples outside the
// box or in empty occupancy cells, delta[s], optional x[s].  COMPACT: writes lik[s] instead of
// xs[s] and appends each foreground sample (L > eps_w) to the compacted stream -- one
// atomicAdd per 128-thread block, warp ballots inside, so a block's survivors stay contiguous
// (4 depths x 32 neighbouring rays) and the field kernels skip background samples entirely.
// Block-uniform grid-stride loop over 128-slot tiles (a round's slot count is only known on
// the device), launched with enough blocks for one tile each in the single pass.  (Measured
// and not kept: a persistent grid with the bone table staged once per CTA, 2.12 -> 2.40 ms;
// warp 0 computing the 32 rays' setup for the tile's 4 depth warps through shared memory,
// +0.15 ms -- the barrier costs more than the redundant ray setup.)
#ifndef FV_MARCH_DPT
#define FV_MARCH_DPT 8
#endif
#ifndef FV_MARCH_STASH
#define FV_MARCH_STASH 1
#endif
constexpr int MARCH_DPT = FV_MARCH_DPT;   // consecutive depths per thread

template <bool COMPACT>
#ifndef FV_MARCH_MINB
#define FV_MARCH_MINB 8   // <= 64 registers: 8 blocks of 4 warps per SM
#endif
__global__ void __launch_bounds__(128, FV_MARCH_MINB) k_march_warp(fv_camera cam, fv_march m, fv_warp w, int64_t n_rays,
                                                    float4* __restrict__ xs_out, float* __restrict__ delta_out,
                                                    float* __restrict__ x_out, int32_t* __restrict__ count_out,
                                                    Compact cmp, MarchRound rd) {
  __shared__ __align__(16) float sg[FV_MAX_BONES * 12];
  __shared__ int32_t wcount[4], wbase;
#if FV_MARCH_STASH
  // the tile's foreground samples, staged so the whole tile (32 rays x 4 DPT consecutive
  // depths) lands contiguously in the compacted stream with one global atomic
  __shared__ float4 stash_x[COMPACT ? 128 * MARCH_DPT : 1];
  __shared__ int32_t stash_i[COMPACT ? 128 * MARCH_DPT : 1];
  __shared__ int32_t scount;
#endif
  fill_bones_x2(sg, w.d_g, w.n_bones);
  __syncthreads();
  const int N = m.n_samples, K = rd.K;
  const int64_t n_j = rd.n_live ? (int64_t)*rd.n_live : n_rays;     // rays in this round
  const int64_t n_rb = padded_rays(n_j) / RB;                         // blocks of 32 rays
#ifndef FV_MARCH_INTERLEAVE
#define FV_MARCH_INTERLEAVE 1
#endif
  constexpr int DPT = MARCH_DPT, TILE_DEPTHS = 4 * DPT;
  const int64_t tiles_per_rb = (K + TILE_DEPTHS - 1) / TILE_DEPTHS;
  const int64_t n_tiles = n_rb * tiles_per_rb;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // tile = one block of 32 rays x 4 DPT consecutive depths, one ray per lane.  Iteration d
  // covers the tile's depths [4 d, 4 d + 4), warp w depth 4 d + w (INTERLEAVED: the block's
  // 128 slots of an iteration -- one compaction, contiguous in the foreground stream -- are 4
  // consecutive depths of 32 neighbouring rays, the locality the field kernels' gathers
  // want), or (FV_MARCH_INTERLEAVE 0) warp w takes depths [w DPT, (w + 1) DPT) and carries
  // t_{i+1} over as t_i of its next slot.  Either way the ray setup (pixel, direction, slab,
  // bin width) is computed once per DPT slots.  (Measured and not kept: the block's 4 warps
  // on 4 neighbouring ray blocks at the same depths -- k_radiance_tc 4.58 -> 4.71 ms: depth
  // neighbours share more hash cells than ray neighbours.)  With FV_MARCH_STASH the tile's
  // foreground samples are staged in shared memory and appended to the compacted stream with
  // ONE atomic, so the whole tile (32 rays x 32 consecutive depths) is contiguous there:
  // fewer barriers, and consecutive radiance tiles (on one SM's warpgroups) share lines.
  constexpr bool INTERLEAVE = FV_MARCH_INTERLEAVE;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t jb = tile / tiles_per_rb;
    const int il0 = (int)(tile % tiles_per_rb) * TILE_DEPTHS + (INTERLEAVE ? wid : wid * DPT);
    const int64_t j = jb * RB + lane;
    bool hit;
    const RaySetup rs = ray_setup(cam, m, rd, j, n_j, hit);
    float t_carry = 0.f;
    bool carry = false;
#if FV_MARCH_STASH
    if (COMPACT && threadIdx.x == 0) scount = 0;
    if (COMPACT) __syncthreads();
#endif
#pragma unroll 1
    for (int d = 0; d < DPT; ++d) {
      const int il = il0 + (INTERLEAVE ? 4 * d : d);
      const bool slot_ok = il < K;                                   // warp-uniform
      const int64_t s = (jb * K + il) * RB + lane;
      const int32_t i = rd.i0 + il;
      float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
      float delta = 0.f;
      bool occ = false;
      if (slot_ok && rs.ray >= 0) {
        const int32_t pix = rs.pix;
        if (hit) {
          const float t = carry ? t_carry
                                : sample_t(rs.t0, rs.step, i, m.jitter ? jitter_u(m.seed, (uint32_t)pix, i) : 0.5f);
          if (i + 1 < N) {
            const float un = m.jitter ? jitter_u(m.seed, (uint32_t)pix, i + 1) : 0.5f;
            t_carry = sample_t(rs.t0, rs.step, i + 1, un);
            carry = !INTERLEAVE;
            delta = __fsub_rn(t_carry, t);
          } else {
            const float u0 = m.jitter ? jitter_u(m.seed, (uint32_t)pix, 0) : 0.5f;
            delta = __fadd_rn(__fsub_rn(rs.t1, t), __fsub_rn(sample_t(rs.t0, rs.step, 0, u0), rs.t0));
          }
          const float px = __fadd_rn(cam.center[0], __fmul_rn(t, rs.dx));
          const float py = __fadd_rn(cam.center[1], __fmul_rn(t, rs.dy));
          const float pz = __fadd_rn(cam.center[2], __fmul_rn(t, rs.dz));
          if (x_out) { x_out[3 * s] = px; x_out[3 * s + 1] = py; x_out[3 * s + 2] = pz; }
          occ = m.d_occ == nullptr || occ_test_nb(m.d_occ, m.obox_min, m.occ_scale, px, py, pz);
          if (occ) {
            float xsk[3];
            const float L = w.vol_half ? warp_point<false, 1>(w, sg, m.eps_w, px, py, pz, xsk)
                                       : warp_point<false, 0>(w, sg, m.eps_w, px, py, pz, xsk);
            out = make_float4(xsk[0], xsk[1], xsk[2], L);
          }
        } else if (x_out) {
          x_out[3 * s] = x_out[3 * s + 1] = x_out[3 * s + 2] = 0.f;
        }
        if (i == 0 && count_out) count_out[rs.ray] = hit ? N : 0;
      } else if (x_out && slot_ok) {
        x_out[3 * s] = x_out[3 * s + 1] = x_out[3 * s + 2] = 0.f;
      }
      if (!COMPACT) {
        if (slot_ok) {
          xs_out[s] = out;
          delta_out[s] = delta;
        }
        continue;
      }
      const bool fg = slot_ok && out.w > m.eps_w;
      const uint32_t ballot = __ballot_sync(0xffffffffu, fg);
#if FV_MARCH_STASH
      {
        int base = 0;
        if (lane == 0 && ballot) base = atomicAdd(&scount, __popc(ballot));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (fg) {
          const int k = base + __popc(ballot & ((1u << lane) - 1u));
          FV_ASSERT(k < 128 * MARCH_DPT);
          stash_x[k] = out;
          stash_i[k] = (int32_t)s;
        }
        if (slot_ok) {
          cmp.lik[s] = out.w;
          delta_out[s] = delta;
          if (cmp.flags) cmp.flags[s] = (uint8_t)((hit ? 1 : 0) | (occ ? 2 : 0) | (fg ? 4 : 0));
        }
        continue;
      }
#endif
      if (lane == 0) wcount[wid] = __popc(ballot);
      __syncthreads();
      if (threadIdx.x == 0) wbase = atomicAdd(cmp.count, wcount[0] + wcount[1] + wcount[2] + wcount[3]);
      __syncthreads();
      if (slot_ok) {
        cmp.lik[s] = out.w;
        delta_out[s] = delta;
        if (cmp.flags) cmp.flags[s] = (uint8_t)((hit ? 1 : 0) | (occ ? 2 : 0) | (fg ? 4 : 0));
      }
      if (fg) {
        int off = wbase;
        for (int qq = 0; qq < wid; ++qq) off += wcount[qq];
        off += __popc(ballot & ((1u << lane) - 1u));
        cmp.xsc[off] = out;
        cmp.idx[off] = (int32_t)s;
      }
      __syncthreads();                   // wcount / wbase are reused by the next slot
    }
#if FV_MARCH_STASH
    if (COMPACT) {
      __syncthreads();
      if (threadIdx.x == 0) wbase = scount ? atomicAdd(cmp.count, scount) : 0;
      __syncthreads();
      for (int k = threadIdx.x; k < scount; k += blockDim.x) {
        cmp.xsc[wbase + k] = stash_x[k];
        cmp.idx[wbase + k] = stash_i[k];
      }
      __syncthreads();                   // the stash is refilled by the next tile
    }
#endif
  }
}

// Grid for k_march_warp: one tile (32 rays x 4 MARCH_DPT depths) per block, capped at 64
// waves of resident blocks (the block loop covers the rest).
template <bool COMPACT>
static unsigned march_grid(int64_t n_rays, int K) {
  static int per_sm[2] = {0, 0};
  int& b = per_sm[COMPACT ? 1 : 0];
  if (b == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_march_warp<COMPACT>, 128, 0);
    if (b < 1) b = 1;
  }
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = padded_rays(n_rays) / RB * ((K + 4 * MARCH_DPT - 1) / (4 * MARCH_DPT));
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)n_sm * b * 64));
}

// d x_skel -> d W^c (C,G,G,G) via dw_i = <dxs, p_i - x_skel>/L and the trilinear scatter.
// dvol[i, corner] += trilinear weight * dL/dw_i (ad:778-789 bincount scatter); dL/dw_i =
// dL/dx_skel . (G_i(x) - x_skel) / L.  Warp-aggregated like k_hash_bwd: lanes sharing a
// bone cell (a warp = 32 neighbouring rays at one depth, ~8 rays per 1/32-box cell) sum
// their 8 corner terms with a segmented shuffle scan and the run's last lane issues the
// atomics.
// With WANT_G the kernel also returns dL/dG_i (oracle.warp.skeleton_warp_bwd_g):
// dL/dp_i = (w_i / L) g + dw_i * dw_i/dp_i (trilinear gradient of the bone's W^c channel),
// dR_i += dp_i x^T, dt_i += dp_i, reduced over the warp by shuffles, over the block in shared
// memory and over the grid with one atomicAdd per (bone, entry) per block.
template <bool WANT_G>
__global__ void __launch_bounds__(128) k_warp_bwd(fv_warp w, float eps_w, const float* __restrict__ x, int64_t n,
                                                  const float* __restrict__ dxs, float* __restrict__ dvol,
                                                  float* __restrict__ dg) {
  __shared__ __align__(16) float sg[FV_MAX_BONES * 12];
  __shared__ float sdg[WANT_G ? FV_MAX_BONES * 12 : 1];
  fill_bones_x2(sg, w.d_g, w.n_bones);
  if (WANT_G)
    for (int i = threadIdx.x; i < w.n_bones * 12; i += blockDim.x) sdg[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool live = q0 < n;
  const int64_t q = live ? q0 : n - 1;
  const float g0 = dxs[3 * q], g1 = dxs[3 * q + 1], g2 = dxs[3 * q + 2];
  live = live && !(g0 == 0.f && g1 == 0.f && g2 == 0.f);
  if (!__any_sync(0xffffffffu, live)) {
    if (WANT_G) goto flush;            // every block still publishes its (partial) dG
    return;
  }
  {
  const float x0 = x[3 * q], x1 = x[3 * q + 1], x2 = x[3 * q + 2];
  float xsk[3];
  const float L = warp_point<false>(w, sg, eps_w, x0, x1, x2, xsk);
  live = live && (L > eps_w);
  const float invL = live ? 1.f / L : 0.f;
  const int G = w.vol_res;
  for (int i = 0; i < w.n_bones; ++i) {
    float p[3];
    bone_point_x2(sg + 12 * i, x0, x1, x2, p);
    int i0[3]; float f[3];
    const bool in = warp_cell(w, p, i0, f);
    const float dw = (g0 * (p[0] - xsk[0]) + g1 * (p[1] - xsk[1]) + g2 * (p[2] - xsk[2])) * invL;
    if (WANT_G) {
      float dp[3] = {0.f, 0.f, 0.f};
      if (live && in) {
        float cv[8];
        load_corners(w.d_vol_packed, w.vol_half, vol_cell_index(i, G, i0), cv);
        const float wi = trilerp8(f, cv);
        const float gy0 = 1.f - f[1], gz0 = 1.f - f[2];
        // trilinear gradient in grid units (corner order a*4 + b*2 + c = x, y, z)
        const float dfx = gy0 * gz0 * (cv[4] - cv[0]) + gy0 * f[2] * (cv[5] - cv[1]) +
                          f[1] * gz0 * (cv[6] - cv[2]) + f[1] * f[2] * (cv[7] - cv[3]);
        const float gx0 = 1.f - f[0];
        const float dfy = gx0 * gz0 * (cv[2] - cv[0]) + gx0 * f[2] * (cv[3] - cv[1]) +
                          f[0] * gz0 * (cv[6] - cv[4]) + f[0] * f[2] * (cv[7] - cv[5]);
        const float dfz = gx0 * gy0 * (cv[1] - cv[0]) + gx0 * f[1] * (cv[3] - cv[2]) +
                          f[0] * gy0 * (cv[5] - cv[4]) + f[0] * f[1] * (cv[7] - cv[6]);
        const float a = wi * invL;
        dp[0] = a * g0 + dw * dfx * w.wscale[0];
        dp[1] = a * g1 + dw * dfy * w.wscale[1];
        dp[2] = a * g2 + dw * dfz * w.wscale[2];
      }
      float v[12] = {dp[0] * x0, dp[0] * x1, dp[0] * x2, dp[1] * x0, dp[1] * x1, dp[1] * x2,
                     dp[2] * x0, dp[2] * x1, dp[2] * x2, dp[0], dp[1], dp[2]};
#pragma unroll
      for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int j = 0; j < 12; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < 12; ++j) atomicAdd(&sdg[12 * i + j], v[j]);
      }
    }
    const bool any = live && in && dw != 0.f && dvol != nullptr;
    const float wx[2] = {1.f - f[0], f[0]}, wy[2] = {1.f - f[1], f[1]}, wz[2] = {1.f - f[2], f[2]};
    float v[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {   // ((wx wy) wz) dw, the z-pair of each (x, y) corner as f32x2
      const float t = wx[q >> 1] * wy[q & 1];
      const float2 p = __fmul2_rn(__fmul2_rn(make_float2(t, t), make_float2(wz[0], wz[1])), make_float2(dw, dw));
      v[2 * q] = p.x;
      v[2 * q + 1] = p.y;
    }
    const uint32_t key = any ? (uint32_t)vol_cell_index(i, G, i0) : (0xFFFFFFFFu - (uint32_t)lane);
    const bool lead = seg_sum<8>(v, key, lane) && any;
    if (lead) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int vx = i0[0] + (c >> 2) - 1, vy = i0[1] + ((c >> 1) & 1) - 1, vz = i0[2] + (c & 1) - 1;
        if (vx < 0 || vx >= G || vy < 0 || vy >= G || vz < 0 || vz >= G) continue;
        atomicAdd(dvol + (((int64_t)i * G + vx) * G + vy) * G + vz, v[c]);
      }
    }
  }
  }
flush:
  if (WANT_G) {
    __syncthreads();
    for (int j = threadIdx.x; j < w.n_bones * 12; j += blockDim.x)
      if (sdg[j] != 0.f) atomicAdd(dg + j, sdg[j]);
  }
}

// sample_bone_channels (ad:728-773) on its own: channel i of W^c at the bone-i points pts[i]
// (K,n,3) -> (K,n), the trilinear sample warp_point takes per bone (zero outside the padded
// grid).
__global__ void k_sample_bone_channels(fv_warp w, const float* __restrict__ pts, int64_t n, float* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)w.n_bones * n) return;
  const int i = (int)(e / n);
  const float p[3] = {pts[3 * e], pts[3 * e + 1], pts[3 * e + 2]};
  int i0[3];
  float f[3];
  float v = 0.f;
  if (warp_cell(w, p, i0, f)) {
    float cv[8];
    load_corners(w.d_vol_packed, w.vol_half, vol_cell_index(i, w.vol_res, i0), cv);
    v = trilerp8(f, cv);
  }
  out[e] = v;
}

// Backward of sample_bone_channels (ad:775-806) for an upstream gradient g (K,n):
// dvol[i, corner] += trilinear weight * g (the reference's bincount scatter, ad:778-789;
// fp32 atomics into the unpadded (C,G,G,G) grid, padding corners dropped) and
// dpts[i, n] = (d out / d u) * g * scale (ad:790-805), both zero for points outside.
__global__ void k_sample_bone_channels_bwd(fv_warp w, const float* __restrict__ pts, int64_t n,
                                           const float* __restrict__ g, float* __restrict__ dvol,
                                           float* __restrict__ dpts) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)w.n_bones * n) return;
  const int i = (int)(e / n);
  const float p[3] = {pts[3 * e], pts[3 * e + 1], pts[3 * e + 2]};
  int i0[3];
  float f[3];
  const bool in = warp_cell(w, p, i0, f);
  const float gv = in ? g[e] : 0.f;
  if (dpts) {
    float d[3] = {0.f, 0.f, 0.f};
    if (in) {
      float cv[8];
      load_corners(w.d_vol_packed, w.vol_half, vol_cell_index(i, w.vol_res, i0), cv);
      const float gx0 = 1.f - f[0], gy0 = 1.f - f[1], gz0 = 1.f - f[2];
      d[0] = gy0 * gz0 * (cv[4] - cv[0]) + gy0 * f[2] * (cv[5] - cv[1]) + f[1] * gz0 * (cv[6] - cv[2]) +
             f[1] * f[2] * (cv[7] - cv[3]);
      d[1] = gx0 * gz0 * (cv[2] - cv[0]) + gx0 * f[2] * (cv[3] - cv[1]) + f[0] * gz0 * (cv[6] - cv[4]) +
             f[0] * f[2] * (cv[7] - cv[5]);
      d[2] = gx0 * gy0 * (cv[1] - cv[0]) + gx0 * f[1] * (cv[3] - cv[2]) + f[0] * gy0 * (cv[5] - cv[4]) +
             f[0] * f[1] * (cv[7] - cv[6]);
    }
    dpts[3 * e] = d[0] * gv * w.wscale[0];
    dpts[3 * e + 1] = d[1] * gv * w.wscale[1];
    dpts[3 * e + 2] = d[2] * gv * w.wscale[2];
  }
  if (dvol && in && gv != 0.f) {
    const int G = w.vol_res;
    const float wx[2] = {1.f - f[0], f[0]}, wy[2] = {1.f - f[1], f[1]}, wz[2] = {1.f - f[2], f[2]};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int a = c >> 2, b = (c >> 1) & 1, z = c & 1;
      const int vx = i0[0] + a - 1, vy = i0[1] + b - 1, vz = i0[2] + z - 1;
      if (vx < 0 || vx >= G || vy < 0 || vy >= G || vz < 0 || vz >= G) continue;
      atomicAdd(dvol + (((int64_t)i * G + vx) * G + vy) * G + vz, wx[a] * wy[b] * wz[z] * gv);
    }
  }
}

}  // namespace fv

namespace fv {
int32_t check_warp(const fv_warp* w) {
  if (!w) return set_error(FV_EDIM, "null fv_warp");
  if (w->n_bones < 1 || w->n_bones > FV_MAX_BONES) return set_error(FV_EDIM, "fv_warp: bad bone count");
  if (w->vol_res < 2 || w->vol_res > FV_MAX_VOL_RES) return set_error(FV_EDIM, "fv_warp: bad volume resolution");
  return FV_OK;
}
}  // namespace fv

using namespace fv;

extern "C" int32_t fv_warp_pack(const float* d_vol, int32_t channels, const fv_warp* warp, void* d_vol_packed,
                                void* stream) {
  if (!warp || !d_vol || !d_vol_packed) return set_error(FV_EDIM, "fv_warp_pack: null argument");
  if (int32_t e = check_warp(warp)) return e;
  if (warp->n_bones > channels) return set_error(FV_EDIM, "fv_warp_pack: more bones than volume channels");
  const int64_t cells = (int64_t)warp->n_bones * (warp->vol_res + 1) * (warp->vol_res + 1) * (warp->vol_res + 1);
  const int grid = (int)std::min<int64_t>((cells + 255) / 256, 148 * 16);
  cudaStream_t st = (cudaStream_t)stream;
  if (warp->vol_half)
    k_warp_pack<__half><<<grid, 256, 0, st>>>(d_vol, warp->n_bones, warp->vol_res, (__half*)d_vol_packed);
  else
    k_warp_pack<float><<<grid, 256, 0, st>>>(d_vol, warp->n_bones, warp->vol_res, (float*)d_vol_packed);
  return check_launch("fv_warp_pack");
}

extern "C" int32_t fv_warp_fwd(const fv_warp* warp, float eps_w, const float* d_x, int64_t n, float* d_xskel,
                               float* d_lik, uint8_t* d_fg, float* d_w, void* stream) {
  if (!warp || n < 0) return set_error(FV_EDIM, "fv_warp_fwd: bad arguments");
  if (int32_t e = check_warp(warp)) return e;
  if (n == 0) return FV_OK;
  k_warp_fwd<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*warp, eps_w, d_x, n, d_xskel, d_lik,
                                                                             d_fg, d_w);
  return check_launch("fv_warp_fwd");
}

extern "C" int32_t fv_sample_bone_channels(const fv_warp* warp, const float* d_pts, int64_t n, float* d_out,
                                           void* stream) {
  if (!warp || n < 0 || (n > 0 && (!d_pts || !d_out))) return set_error(FV_EDIM, "fv_sample_bone_channels: bad arguments");
  if (int32_t e = check_warp(warp)) return e;
  if (n == 0) return FV_OK;
  const int64_t total = (int64_t)warp->n_bones * n;
  k_sample_bone_channels<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*warp, d_pts, n, d_out);
  return check_launch("fv_sample_bone_channels");
}

extern "C" int32_t fv_sample_bone_channels_bwd(const fv_warp* warp, const float* d_pts, int64_t n, const float* d_g,
                                               float* d_dvol, float* d_dpts, void* stream) {
  if (!warp || n < 0 || (n > 0 && (!d_pts || !d_g))) return set_error(FV_EDIM, "fv_sample_bone_channels_bwd: bad arguments");
  if (int32_t e = check_warp(warp)) return e;
  if (n == 0 || (!d_dvol && !d_dpts)) return FV_OK;
  const int64_t total = (int64_t)warp->n_bones * n;
  k_sample_bone_channels_bwd<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*warp, d_pts, n, d_g,
                                                                                                d_dvol, d_dpts);
  return check_launch("fv_sample_bone_channels_bwd");
}

extern "C" int32_t fv_warp_bwd(const fv_warp* warp, float eps_w, const float* d_x, int64_t n,
                               const float* d_dxskel, float* d_dvol, void* stream) {
  if (!warp || n < 0) return set_error(FV_EDIM, "fv_warp_bwd: bad arguments");
  if (int32_t e = check_warp(warp)) return e;
  if (n == 0) return FV_OK;
  k_warp_bwd<false><<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*warp, eps_w, d_x, n, d_dxskel,
                                                                                    d_dvol, nullptr);
  return check_launch("fv_warp_bwd");
}

// fv_warp_bwd that also accumulates dL/dG_i into d_dg [K][12] (R row-major, t); d_dvol may
// be NULL (no volume gradient).
extern "C" int32_t fv_warp_bwd_g(const fv_warp* warp, float eps_w, const float* d_x, int64_t n,
                                 const float* d_dxskel, float* d_dvol, float* d_dg, void* stream) {
  if (!warp || n < 0 || !d_dg) return set_error(FV_EDIM, "fv_warp_bwd_g: bad arguments");
  if (int32_t e = check_warp(warp)) return e;
  if (n == 0) return FV_OK;
  k_warp_bwd<true><<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*warp, eps_w, d_x, n, d_dxskel,
                                                                                   d_dvol, d_dg);
  return check_launch("fv_warp_bwd_g");
}

extern "C" int32_t fv_march_warp(const fv_camera* cam, const fv_march* march, const fv_warp* warp, int64_t n_rays,
                                 float* d_xs, float* d_delta, float* d_x, int32_t* d_count, void* stream) {
  if (!cam || !march || !warp || n_rays < 0 || march->n_samples < 1)
    return set_error(FV_EDIM, "fv_march_warp: bad arguments");
  if (int32_t e = check_warp(warp)) return e;
  if (n_rays == 0) return FV_OK;
  k_march_warp<false><<<march_grid<false>(n_rays, march->n_samples), 128, 0, (cudaStream_t)stream>>>(
      *cam, *march, *warp, n_rays, (float4*)d_xs, d_delta, d_x, d_count, Compact{},
      MarchRound{0, march->n_samples, nullptr, nullptr});
  return check_launch("fv_march_warp");
}

namespace fv {
// render-path march: likelihood per sample + compacted foreground stream (count zeroed here)
int32_t march_compact(const fv_camera* cam, const fv_march* march, const fv_warp* warp, int64_t n_rays, float* lik,
                      float* delta, float4* xsc, int32_t* idx, int32_t* count, int32_t* ray_count, cudaStream_t st,
                      uint8_t* flags) {
  cudaMemsetAsync(count, 0, sizeof(int32_t), st);
  k_march_warp<true><<<march_grid<true>(n_rays, march->n_samples), 128, 0, st>>>(*cam, *march, *warp, n_rays, nullptr, delta,
                                                                      nullptr, ray_count,
                                                                      Compact{lik, xsc, idx, count, flags},
                                                                      MarchRound{0, march->n_samples, nullptr, nullptr});
  return check_launch("march_compact");
}

// One marching round over a live-ray list (count zeroed here): samples [i0, i0 + K) of the
// n_live rays in live (device), slots in the round layout; n_rays bounds n_live.
int32_t march_round(const fv_camera* cam, const fv_march* march, const fv_warp* warp, int64_t n_rays, int32_t i0,
                    int32_t K, const int32_t* live, const int32_t* n_live, float* lik, float* delta, float4* xsc,
                    int32_t* idx, int32_t* count, int32_t* ray_count, cudaStream_t st) {
  cudaMemsetAsync(count, 0, sizeof(int32_t), st);
  k_march_warp<true><<<march_grid<true>(n_rays, K), 128, 0, st>>>(*cam, *march, *warp, n_rays, nullptr, delta,
                                                                  nullptr, ray_count,
                                                                  Compact{lik, xsc, idx, count, nullptr},
                                                                  MarchRound{i0, K, live, n_live});
  return check_launch("march_round");
}
}  // namespace fv

// The render path's own march (the kernel fv_render_fwd launches), exposed so its integer
// outputs can be checked bit for bit: per-sample likelihood (0 where skipped), spacing and
// flags, the compacted foreground stream (x_skel, L) + sample ids and its length, per-ray
// sample counts.  Sample slots are ray-block-major (layout.cuh).
extern "C" int32_t fv_march_compact(const fv_camera* cam, const fv_march* march, const fv_warp* warp, int64_t n_rays,
                                    float* d_lik, float* d_delta, float* d_xsc, int32_t* d_idx, int32_t* d_n_fg,
                                    int32_t* d_count, uint8_t* d_flags, void* stream) {
  if (!cam || !march || !warp || n_rays < 0 || march->n_samples < 1 || !d_lik || !d_delta || !d_xsc || !d_idx ||
      !d_n_fg)
    return set_error(FV_EDIM, "fv_march_compact: bad arguments");
  if (int32_t e = check_warp(warp)) return e;
  if (padded_rays(n_rays) * (int64_t)march->n_samples > (int64_t)INT32_MAX)
    return set_error(FV_EDIM, "fv_march_compact: n_rays x n_samples exceeds 2^31 - 1 sample slots (int32 sample ids)");
  if (n_rays == 0) return cudaMemsetAsync(d_n_fg, 0, sizeof(int32_t), (cudaStream_t)stream) == cudaSuccess
                              ? FV_OK : check_launch("fv_march_compact");
  return march_compact(cam, march, warp, n_rays, d_lik, d_delta, (float4*)d_xsc, d_idx, d_n_fg, d_count,
                       (cudaStream_t)stream, d_flags);
}
