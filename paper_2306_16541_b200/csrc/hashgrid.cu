// Multiresolution hash-grid encoding, forward and backward (builder-defined; the
// definition and its float32 operation order live in oracle/encoding.py).
#include <cuda_runtime.h>
#include "fv_common.cuh"
#include "fv_internal.h"

namespace fv {

// One thread per sample, levels in turn; the 2L features of the block's 128 rows are
// staged in shared memory and stored as contiguous runs (coalesced) instead of 2L strided
// 4-byte stores per thread.
__global__ void __launch_bounds__(128) k_hash_fwd(fv_hash h, const float* __restrict__ x, int64_t n,
                                                  float* __restrict__ feat, uint32_t* __restrict__ index) {
  __shared__ float sf[128 * (2 * FV_MAX_LEVELS + 1)];
  const int t = threadIdx.x;
  const int64_t p0 = (int64_t)blockIdx.x * 128;
  const int64_t p = p0 + t;
  const int F = 2 * h.n_levels, L1 = F + 1;
  if (p < n) {
    float xn[3]; bool mask[3];
    hash_norm(h, x[3 * p], x[3 * p + 1], x[3 * p + 2], xn, mask);
    for (int l = 0; l < h.n_levels; ++l) {
      HashCell c;
      hash_level_cell(xn, h.res[l], c);
      uint32_t idx[8];
      const float2 f = hash_level_feat(h, l, c, index ? idx : nullptr);
      sf[t * L1 + 2 * l] = f.x;
      sf[t * L1 + 2 * l + 1] = f.y;
      if (index) {
#pragma unroll
        for (int q = 0; q < 8; ++q) index[(p * h.n_levels + l) * 8 + q] = idx[q];
      }
    }
  }
  __syncthreads();
  const int64_t rows = n - p0 < 128 ? n - p0 : 128;
  float* dst = feat + p0 * F;
  for (int64_t i = t; i < rows * F; i += 128) dst[i] = sf[(i / F) * L1 + i % F];
}

// dtable += w_corner * dfeat (float2 vector atomics); dx = sum_l d feat_l / d x.
// Warp aggregation: a warp holds 32 neighbouring rays at one depth, so at the coarse levels
// many lanes share a cell.  Lanes are grouped by (level cell) with __match_any_sync; a
// group's lowest lane sums the members' 8 corner contributions through shared memory and
// issues one float2 atomic per corner (singletons -- most lanes at the fine levels -- add
// directly).  Summation order inside a group differs from a per-sample scatter by fp32
// rounding only (the reference's gather0 scatter-add, ad:335-344, is order-free).
__device__ __forceinline__ void red2(float2* p, float2 v) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" :: "l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void red4(float2* p, float2 a, float2 b) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(p), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y)
               : "memory");
}
// The 8 corner updates of one cell: an x-corner pair whose entries form an aligned 16-byte
// pair (indices 2k, 2k+1 -- always the case for even x on hashed levels, where x+1 only
// flips index bit 0) goes out as one v4 reduction instead of two v2.
__device__ __forceinline__ void scatter8(float2* dt2, const uint32_t (&gi)[8], const float2 (&v)[8], bool v4ok) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t i0 = gi[q], i1 = gi[q + 4];
    if (v4ok && (i0 ^ i1) == 1u) {
      if (i0 < i1) red4(dt2 + i0, v[q], v[q + 4]);
      else red4(dt2 + i1, v[q + 4], v[q]);
    } else {
      red2(dt2 + i0, v[q]);
      red2(dt2 + i1, v[q + 4]);
    }
  }
}

__global__ void __launch_bounds__(128) k_hash_bwd(fv_hash h, const float* __restrict__ x, int64_t n,
                                                  const float* __restrict__ dfeat, float* __restrict__ dtable,
                                                  float* __restrict__ dx) {
  __shared__ float2 scratch[4][8][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t p0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool valid = p0 < n;
  const int64_t p = valid ? p0 : n - 1;
  float xn[3]; bool mask[3];
  hash_norm(h, x[3 * p], x[3 * p + 1], x[3 * p + 2], xn, mask);
  const uint32_t maskT = (1u << h.log2_T) - 1u;
  float2* dt2 = reinterpret_cast<float2*>(dtable);
  const bool v4ok = (reinterpret_cast<uintptr_t>(dtable) & 15) == 0;
  // corner indices + table values of level l+1 are fetched while level l is processed
  auto corners = [&](int l, HashCell& c, uint32_t (&gi)[8], float2 (&tv)[8]) {
    hash_level_cell(xn, h.res[l], c);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      gi[q] = h.offset[l] + hash_index(h.dense[l], h.res[l], maskT, c.i0[0] + (q >> 2), c.i0[1] + ((q >> 1) & 1),
                                       c.i0[2] + (q & 1));
      FV_ASSERT(gi[q] - h.offset[l] <
                (h.dense[l] ? (uint32_t)(h.res[l] + 1) * (h.res[l] + 1) * (h.res[l] + 1) : maskT + 1u));
    }
    if (dx) {
      if (h.table_half) {
#pragma unroll
        for (int q = 0; q < 8; ++q) tv[q] = __half22float2(__ldg(reinterpret_cast<const __half2*>(h.d_table) + gi[q]));
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) tv[q] = __ldg(reinterpret_cast<const float2*>(h.d_table) + gi[q]);
      }
    }
  };
  float gx = 0.f, gy = 0.f, gz = 0.f;
  HashCell cn;
  uint32_t gin[8];
  float2 tvn[8];
  corners(0, cn, gin, tvn);
  for (int l = 0; l < h.n_levels; ++l) {
    const float2 gg = valid ? *reinterpret_cast<const float2*>(dfeat + p * (2 * h.n_levels) + 2 * l)
                            : make_float2(0.f, 0.f);
    const float g0 = gg.x, g1 = gg.y;
    const HashCell c = cn;
    uint32_t gi[8];
    float2 tv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { gi[q] = gin[q]; tv[q] = tvn[q]; }
    if (l + 1 < h.n_levels) corners(l + 1, cn, gin, tvn);
    const float wx[2] = {1.f - c.f[0], c.f[0]}, wy[2] = {1.f - c.f[1], c.f[1]}, wz[2] = {1.f - c.f[2], c.f[2]};
    float2 v[8];
    float px = 0.f, py = 0.f, pz = 0.f;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int q = a * 4 + b * 2 + cc;
          const float wgt = wx[a] * wy[b] * wz[cc];
          v[q] = make_float2(wgt * g0, wgt * g1);
          if (dx) {
            const float gv = g0 * tv[q].x + g1 * tv[q].y;
            px += (a ? 1.f : -1.f) * wy[b] * wz[cc] * gv;
            py += wx[a] * (b ? 1.f : -1.f) * wz[cc] * gv;
            pz += wx[a] * wy[b] * (cc ? 1.f : -1.f) * gv;
          }
        }
    const float rf = (float)h.res[l];
    gx += px * rf; gy += py * rf; gz += pz * rf;
    const bool any = valid && (g0 != 0.f || g1 != 0.f);
    const uint64_t key = any ? ((uint64_t)(uint32_t)c.i0[0] | ((uint64_t)(uint32_t)c.i0[1] << 21) |
                                ((uint64_t)(uint32_t)c.i0[2] << 42))
                             : (~0ull - (uint64_t)lane);
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    const unsigned multi = __ballot_sync(0xffffffffu, grp != (1u << lane));
    if (grp == (1u << lane)) {
      if (any) scatter8(dt2, gi, v, v4ok);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) scratch[wib][q][lane] = v[q];
      __syncwarp(multi);
      if (lane == __ffs(grp) - 1 && any) {
        unsigned rest = grp & (grp - 1);
        while (rest) {
          const int o = __ffs(rest) - 1;
          rest &= rest - 1;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float2 w = scratch[wib][q][o];
            v[q].x += w.x;
            v[q].y += w.y;
          }
        }
        scatter8(dt2, gi, v, v4ok);
      }
      __syncwarp(multi);
    }
  }
  if (dx && valid) {
    dx[3 * p] = mask[0] ? gx * h.cinv[0] : 0.f;
    dx[3 * p + 1] = mask[1] ? gy * h.cinv[1] : 0.f;
    dx[3 * p + 2] = mask[2] ? gz * h.cinv[2] : 0.f;
  }
}

int32_t check_hash(const fv_hash* h) {
  if (!h || h->n_levels < 1 || h->n_levels > FV_MAX_LEVELS || h->n_feat != 2 || h->log2_T < 4 || h->log2_T > 26 ||
      !h->d_table)
    return set_error(FV_EDIM, "fv_hash: unsupported configuration (levels 1..16, F = 2, log2_T 4..26)");
  return FV_OK;
}

}  // namespace fv

using namespace fv;

extern "C" int32_t fv_hash_fwd(const fv_hash* hash, const float* d_x, int64_t n, float* d_feat, uint32_t* d_index,
                               void* stream) {
  if (int32_t e = check_hash(hash)) return e;
  if (n < 0) return set_error(FV_EDIM, "fv_hash_fwd: n < 0");
  if (n == 0) return FV_OK;
  k_hash_fwd<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*hash, d_x, n, d_feat, d_index);
  return check_launch("fv_hash_fwd");
}

extern "C" int32_t fv_hash_bwd(const fv_hash* hash, const float* d_x, int64_t n, const float* d_dfeat,
                               float* d_dtable, float* d_dx, void* stream) {
  if (int32_t e = check_hash(hash)) return e;
  if (n < 0) return set_error(FV_EDIM, "fv_hash_bwd: n < 0");
  if (n == 0) return FV_OK;
  if ((reinterpret_cast<uintptr_t>(d_dfeat) & 7) || (reinterpret_cast<uintptr_t>(d_dtable) & 7))
    return set_error(FV_EDIM, "fv_hash_bwd: d_dfeat / d_dtable must be 8-byte aligned");
  k_hash_bwd<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*hash, d_x, n, d_dfeat, d_dtable, d_dx);
  return check_launch("fv_hash_bwd");
}
