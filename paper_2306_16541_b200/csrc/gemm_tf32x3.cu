// Training-time MLP layer GEMMs on 5th-gen tensor cores, split-precision 3xTF32
// (a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi, fp32 accumulate in TMEM -> ~fp32 accurate):
// the layer ops of the reference training step, `linear` forward (ad:403-416) and its
// backward (ad:417-422), for the tall-skinny shapes of the path (M = samples, K, N <= 128).
//
// Both kernels are persistent (one CTA per SM) and warp-specialised:
//   warp 0       TMA producer  : cp.async.bulk.tensor 128-byte-swizzled boxes -> smem ring
//   warp 1       MMA issuer    : one thread issues tcgen05.mma.kind::tf32, commits to mbarriers
//   warps 4..7   converter     : splits each landed stage in place into hi (= rna_tf32(x)) and
//                                lo (= x - hi) tiles (or loads unaligned operands itself)
//   warps 8..11  epilogue      : TMEM -> registers -> bias / ReLU / ReLU-mask -> HBM
//                                (k_rows only; double-buffered accumulators overlap the
//                                next tile's MMAs)
//
// k_rows : out[M x N] = epi(A[M x K] . B),  B(n,k) = W[n*sbn + k*sbk] resident in smem.
//          Forward (B = W^T view, + bias, ReLU) and dX (B = W view, ReLU mask of the layer
//          input).  A is K-major SWIZZLE_128B (TMA box 32 fp32 x 128 rows).
// k_dw   : dW^T[N x K] (+ db as one extra column) += dZ^T . [X | 1] over a contiguous
//          sample range per CTA.  Both operands are MN-major SWIZZLE_128B boxes of
//          32 features x 32 samples, i.e. exactly the row-major activations as TMA lands
//          them -- no transposing copy.  A constant ones box appended to X turns
//          db = colsum(dZ) into column 32*ceil(K/32) of the same accumulator.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include "fv_common.cuh"
#include "fv_internal.h"
#include "tc_sm100.cuh"
#include "gemm_tf32x3.h"

namespace fv {
#ifndef FV_G3_OBUF
#define FV_G3_OBUF 1   // per-warp output staging buffers (1 frees a ring stage)
#endif
namespace g3 {

// ------------------------------------------------------------------------- device helpers
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// tcgen05 shared-memory descriptor; layout type at bits 61..63: 2 = SWIZZLE_128B (16-byte
// chunks, K-major operands here), 1 = SWIZZLE_128B_BASE32B (32-byte chunks: the only 128-byte
// swizzle the tensor core accepts for MN-major 32-bit (tf32) operands)
template <uint32_t LAYOUT = 2>
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)LAYOUT << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      :: "r"(tc::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(tc::smem_u32(src)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// round-to-nearest (ties away) to tf32 = cvt.rna.tf32.f32 for finite inputs, as 2 integer
// ops on the bit pattern (the cvt is emulated with an extra inf/nan guard we do not need)
__device__ __forceinline__ float rna_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ void split4(const float4 v, float4& hi, float4& lo) {
  hi = make_float4(rna_tf32(v.x), rna_tf32(v.y), rna_tf32(v.z), rna_tf32(v.w));
  lo = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
}

// byte offset of 16-byte unit u (0..7) of row r inside a 128B-swizzled region of 128-byte rows
__device__ __forceinline__ uint32_t sw_off(uint32_t r, uint32_t u) { return r * 128u + ((u ^ (r & 7u)) << 4); }
// same for the 32-byte-chunk variant (TMA SWIZZLE_128B_ATOM_32B / UMMA SWIZZLE_128B_BASE32B):
// 32-byte chunk index (address bits 5..6) XOR row bits 0..1 (address bits 7..8)
__device__ __forceinline__ uint32_t sw32_off(uint32_t r, uint32_t u) { return r * 128u + ((u << 4) ^ ((r & 3u) << 5)); }

// 4 consecutive fp32 of a row at columns [k, k+4) with zero fill beyond ncol / for invalid rows
__device__ __forceinline__ float4 load4(const float* row, int k, int ncol, bool vec, bool ok) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!ok || k >= ncol) return v;
  if (vec && k + 3 < ncol) return __ldg(reinterpret_cast<const float4*>(row + k));
  v.x = __ldg(row + k);
  if (k + 1 < ncol) v.y = __ldg(row + k + 1);
  if (k + 2 < ncol) v.z = __ldg(row + k + 2);
  if (k + 3 < ncol) v.w = __ldg(row + k + 3);
  return v;
}

constexpr int kStageA = 128 * 128;       // bytes of one 128-row x 32-fp32 swizzled A tile

// ============================================================================ k_rows
// TMEM map (512 columns): accumulators [0,128) and [128,256); A stages t = 0..3 at
// 256 + 64t: hi in the first 32 columns, lo in the next 32 (lane = tile row, column = k).
constexpr int kAStages = 4;

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
               :: "r"(d), "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}

__global__ void __launch_bounds__(384, 1) k_rows(RowsArgs a, const __grid_constant__ CUtensorMap tmA,
                                                const __grid_constant__ CUtensorMap tmO) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8], aready[kAStages], afree[kAStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float sbias[128];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ST = a.stages;
  const uint32_t bchunk = (uint32_t)a.Np * 128u;          // bytes of one 32-wide K chunk of B
  uint8_t* sBhi = sm;
  uint8_t* sBlo = sm + a.nkc * bchunk;
  uint8_t* sRaw = sm + 2 * a.nkc * bchunk;                 // raw A stages (TMA destination)

  // B (tiny, L2-resident) -> split hi/lo, swizzled K-major, by every thread
  const int Kp = a.nkc * 32;
  for (int i = tid; i < a.Np * Kp; i += blockDim.x) {
    const int n = i % a.Np, k = i / a.Np;
    const float w = (n < a.N && k < a.K) ? __ldg(a.W + (int64_t)n * a.sbn + (int64_t)k * a.sbk) : 0.f;
    const float hi = rna_tf32(w);
    const uint32_t off = (uint32_t)(k >> 5) * bchunk + sw_off(n, (k & 31) >> 2) + (k & 3) * 4;
    *reinterpret_cast<float*>(sBhi + off) = hi;
    *reinterpret_cast<float*>(sBlo + off) = w - hi;
  }
  if (tid < 128) sbias[tid] = (a.bias && tid < a.N) ? __ldg(a.bias + tid) : 0.f;
  if (tid == 0) {
    for (int s = 0; s < 8; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 128); }
    for (int s = 0; s < kAStages; ++s) { tc::mbar_init(&aready[s], 128); tc::mbar_init(&afree[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 128); }
    tc::mbar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  const int64_t ntiles = (a.M + 127) / 128;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && a.tma) {
      const bool pf_bytes = a.mask && (a.ldm % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.mask) & 15) == 0);
      uint32_t g = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int c = 0; c < a.nkc; ++c, ++g) {
          const int s = g % ST;
          tc::mbar_wait(&empty[s], ((g / ST) & 1) ^ 1);
          mbar_expect_tx(&full[s], kStageA);
          tma_load_2d(sRaw + s * kStageA, &tmA, &full[s], c * 32, (int)(tile * 128));
          if (c == 0 && pf_bytes) {   // the epilogue's ReLU-mask rows of this tile: DRAM -> L2 now
            const int64_t rows = (a.M - tile * 128) < 128 ? (a.M - tile * 128) : 128;
            bulk_prefetch_l2(a.mask + tile * 128 * a.ldm, (uint32_t)(rows * a.ldm * 4));
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (A from TMEM)
    if (lane == 0) {
      const uint32_t id = idesc_tf32(128, a.Np, 0, 0);
      uint32_t g = 0, it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t acc = it & 1;
        tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t d = tbase + acc * 128;
        for (int c = 0; c < a.nkc; ++c, ++g) {
          const int t = g % kAStages;
          tc::mbar_wait(&aready[t], (g / kAStages) & 1);
          tc::fence_after();
          const uint32_t ahi = tbase + 256 + t * 64, alo = ahi + 32;
          const uint32_t bhi = tc::smem_u32(sBhi + c * bchunk), blo = tc::smem_u32(sBlo + c * bchunk);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (c * 4 + j >= a.nsteps) break;
            const uint64_t dbh = desc_sw128(bhi + j * 32, 16, 1024), dbl = desc_sw128(blo + j * 32, 16, 1024);
            mma_tf32_ts(d, alo + 8 * j, dbh, id, (c | j) ? 1u : 0u);   // small terms first
            mma_tf32_ts(d, ahi + 8 * j, dbl, id, 1u);
            mma_tf32_ts(d, ahi + 8 * j, dbh, id, 1u);
          }
          tc::mma_commit(&afree[t]);
        }
        tc::mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ converter: row ct of the tile
    const int ct = tid - 128, quarter = warp & 3;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const bool vec = (a.lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.A) & 15) == 0);
    uint32_t g = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t m = tile * 128 + ct;
      for (int c = 0; c < a.nkc; ++c, ++g) {
        float4 v[8];
        if (a.tma) {
          const int s = g % ST;
          tc::mbar_wait(&full[s], (g / ST) & 1);
          const uint8_t* raw = sRaw + s * kStageA;
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const float4*>(raw + sw_off(ct, u));
          mbar_arrive(&empty[s]);
        } else {
          const float* row = a.A + m * a.lda;
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = load4(row, c * 32 + 4 * u, a.K, vec, m < a.M);
        }
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float4 h, l;
          split4(v[u], h, l);
          hi[4 * u] = __float_as_uint(h.x); hi[4 * u + 1] = __float_as_uint(h.y);
          hi[4 * u + 2] = __float_as_uint(h.z); hi[4 * u + 3] = __float_as_uint(h.w);
          lo[4 * u] = __float_as_uint(l.x); lo[4 * u + 1] = __float_as_uint(l.y);
          lo[4 * u + 2] = __float_as_uint(l.z); lo[4 * u + 3] = __float_as_uint(l.w);
        }
        const int t = g % kAStages;
        tc::mbar_wait(&afree[t], ((g / kAStages) & 1) ^ 1);
        tc::fence_after();
        const uint32_t ta = tbase + lane_off + 256 + t * 64;
        tc::tmem_st32(ta, hi);
        tc::tmem_st32(ta + 32, lo);
        tc::tmem_st_wait();
        tc::fence_before();
        mbar_arrive(&aready[t]);
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue
    // Row et of the tile per thread, 32-column groups; the TMEM load of group cg+1 is in
    // flight while group cg is processed.  Output: each warp stages its 32 rows x 32
    // columns in a 128B-swizzled smem buffer (double-buffered per warp) and one lane issues
    // a TMA bulk-tensor store; direct row stores when TMA cannot address the output.
    // ReLU bits in/out: one uint32 per 32 columns per row.
    const int et = tid - 256, quarter = warp & 3;
    const bool vout = (a.ldo % 4 == 0) && (a.N % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0) &&
                      (!a.mask || ((a.ldm % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.mask) & 15) == 0)));
    const int ngroups = (a.Np + 31) / 32, nw = (a.N + 31) / 32;
    uint8_t* wbuf = sRaw + ST * kStageA + quarter * FV_G3_OBUF * 4096;
    uint32_t it = 0, wcount = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const uint32_t acc = it & 1;
      const int64_t m = tile * 128 + et;
      const bool rowok = m < a.M;
      uint32_t mb[4] = {~0u, ~0u, ~0u, ~0u};
      if (a.bits_in && rowok) {
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (w < nw) mb[w] = __ldg(a.bits_in + m * nw + w);
      }
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::fence_after();
      const uint32_t taddr = tbase + acc * 128 + ((uint32_t)(quarter * 32) << 16);
      float va[16], vb[16];
      tc::tmem_ld16(taddr, va);
      if (16 < a.Np) tc::tmem_ld16(taddr + 16, vb);
      tc::tmem_ld_wait();
      for (int cg = 0; cg < ngroups; ++cg) {
        const int n0 = 32 * cg;
        const bool more = cg + 1 < ngroups;
        float na[16], nb[16];
        if (more) {
          tc::tmem_ld16(taddr + n0 + 32, na);
          if (n0 + 48 < a.Np) tc::tmem_ld16(taddr + n0 + 48, nb);
        } else {                          // accumulator fully read: the MMA may reuse it
          tc::fence_before();
          mbar_arrive(&tempty[acc]);
        }
        float4 ma[4], mbf[4];
        if (a.mask && vout && rowok) {   // float mask (legacy form)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ma[q] = n0 + 4 * q < a.N ? __ldg(reinterpret_cast<const float4*>(a.mask + m * a.ldm + n0 + 4 * q))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            mbf[q] = n0 + 16 + 4 * q < a.N
                         ? __ldg(reinterpret_cast<const float4*>(a.mask + m * a.ldm + n0 + 16 + 4 * q))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        uint32_t bits = 0;
        const uint32_t mw = cg == 0 ? mb[0] : cg == 1 ? mb[1] : cg == 2 ? mb[2] : mb[3];
        // bias of the 32 columns as 8 broadcast float4 shared loads
        float bias[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 b4 = *reinterpret_cast<const float4*>(sbias + ((n0 + 4 * q) & 127));
          bias[4 * q] = b4.x; bias[4 * q + 1] = b4.y; bias[4 * q + 2] = b4.z; bias[4 * q + 3] = b4.w;
        }
        const uint32_t live = a.N - n0 >= 32 ? 0xFFFFFFFFu : ((1u << (a.N - n0)) - 1u);   // columns < N
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float y = va[j] + bias[j];
          if (a.act == 1) y = fmaxf(y, 0.f);
          va[j] = y;
          float z = vb[j] + bias[16 + j];
          if (a.act == 1) z = fmaxf(z, 0.f);
          vb[j] = z;
        }
        if (a.bits_in) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            va[j] = (mw >> j) & 1u ? va[j] : 0.f;
            vb[j] = (mw >> (16 + j)) & 1u ? vb[j] : 0.f;
          }
        }
        if (a.mask) {   // legacy float-mask form
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (vout) {
              const float4 x = ma[q], z = mbf[q];
              va[4 * q] = x.x > 0.f ? va[4 * q] : 0.f;     va[4 * q + 1] = x.y > 0.f ? va[4 * q + 1] : 0.f;
              va[4 * q + 2] = x.z > 0.f ? va[4 * q + 2] : 0.f; va[4 * q + 3] = x.w > 0.f ? va[4 * q + 3] : 0.f;
              vb[4 * q] = z.x > 0.f ? vb[4 * q] : 0.f;     vb[4 * q + 1] = z.y > 0.f ? vb[4 * q + 1] : 0.f;
              vb[4 * q + 2] = z.z > 0.f ? vb[4 * q + 2] : 0.f; vb[4 * q + 3] = z.w > 0.f ? vb[4 * q + 3] : 0.f;
            } else if (rowok) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int n = n0 + 4 * q + e;
                if (n < a.N && !(__ldg(a.mask + m * a.ldm + n) > 0.f)) va[4 * q + e] = 0.f;
                if (n + 16 < a.N && !(__ldg(a.mask + m * a.ldm + n + 16) > 0.f)) vb[4 * q + e] = 0.f;
              }
            }
          }
        }
        if (a.bits_out) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            bits |= (va[j] > 0.f ? 1u : 0u) << j;
            bits |= (vb[j] > 0.f ? 1u : 0u) << (16 + j);
          }
          bits &= live;
        }
        if (a.bits_out && rowok) a.bits_out[m * nw + cg] = bits;
        if (a.tma_out) {
          uint8_t* ob = wbuf + (FV_G3_OBUF == 2 ? (wcount & 1) * 4096 : 0);
          if (lane == 0) bulk_wait_read<FV_G3_OBUF - 1>();      // the store that used this buffer has read it
          __syncwarp();
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<float4*>(ob + sw_off(lane, u)) = make_float4(va[4 * u], va[4 * u + 1], va[4 * u + 2], va[4 * u + 3]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<float4*>(ob + sw_off(lane, 4 + u)) =
                make_float4(vb[4 * u], vb[4 * u + 1], vb[4 * u + 2], vb[4 * u + 3]);
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmO, ob, n0, (int)(tile * 128 + quarter * 32));
            bulk_commit();
          }
          ++wcount;
        } else if (rowok) {
          auto store16 = [&](const float (&v)[16], int nb0) {
            if (vout) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int n = nb0 + 4 * q;
                if (n >= a.N) break;
                *reinterpret_cast<float4*>(a.out + m * a.ldo + n) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (nb0 + j < a.N) a.out[m * a.ldo + nb0 + j] = v[j];
            }
          };
          store16(va, n0);
          if (n0 + 16 < a.Np) store16(vb, n0 + 16);
        }
        if (more) {
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) { va[j] = na[j]; vb[j] = nb[j]; }
        }
      }
    }
    if (a.tma_out && lane == 0) bulk_wait_read<0>();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_free<512>(tbase);
}

// ============================================================================ k_dw
// Stage layout (smem): Z raw [4 boxes] | X hi [nxb + 1 boxes] | X lo [nxb + 1]; the split
// dZ^T operand lives in TMEM (A stage t at columns 256 + 64t: hi 32 columns, lo 32), the
// accumulator D = dW^T (+ db column) in columns [0, 32*nxb + 16).
constexpr int kDwS = 32;                  // samples per stage (4 MMA k-steps of 8)
constexpr int kBox = kDwS * 128;          // bytes of one 32-feature x 32-sample swizzled box

__global__ void __launch_bounds__(384, 1) k_dw(DwArgs3 a, const __grid_constant__ CUtensorMap tmX,
                                               const __grid_constant__ CUtensorMap tmZ) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[4], conv[4], empty[4], tfull;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ST = a.stages;
  const int nxb1 = a.nxb + 1;                               // X boxes + the ones box
  const uint32_t stage_bytes = (uint32_t)(4 + 2 * nxb1) * kBox;
  auto zraw = [&](int s) { return sm + s * stage_bytes; };
  auto xhi = [&](int s) { return sm + s * stage_bytes + 4 * kBox; };
  auto xlo = [&](int s) { return sm + s * stage_bytes + (4 + nxb1) * kBox; };

  // zero every stage (Z boxes TMA never writes, X padding); the ones box is 1.0 everywhere
  // (hi = 1, lo = 0), so each of its columns of D is colsum(dZ) whatever the swizzle
  for (uint32_t i = tid; i < ST * stage_bytes / 16; i += blockDim.x) {
    const uint32_t o = i % (stage_bytes / 16);
    const bool ones = o >= (4 + a.nxb) * kBox / 16 && o < (4 + nxb1) * kBox / 16;
    const float v = ones ? 1.f : 0.f;
    reinterpret_cast<float4*>(sm)[i] = make_float4(v, v, v, v);
  }
  if (tid == 0) {
    // narrow unaligned dZ: the producer warp's 32 lanes also arrive (cp.async completion)
    const uint32_t nfull = (!a.tmaZ && a.N <= 16) ? 33u : 1u;
    for (int s = 0; s < 4; ++s) { tc::mbar_init(&full[s], nfull); tc::mbar_init(&conv[s], 256); tc::mbar_init(&empty[s], 1); }
    tc::mbar_init(&tfull, 1);
    tc::mbar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r1 = min(r0 + a.rows_per_cta, a.M);
  const int nchunk = r1 > r0 ? (int)((r1 - r0 + kDwS - 1) / kDwS) : 0;
  const int nprime = 32 * a.nxb + 16;

  if (warp == 0) {
    // producer: TMA boxes (lane 0); a narrow unaligned dZ (N <= 16, e.g. the 3-wide residual
    // output) is gathered by all 32 lanes with 4-byte cp.async straight into the swizzled
    // zraw box, completion tracked by the same full barrier (cp.async.mbarrier.arrive.noinc)
    const bool zcoop = !a.tmaZ && a.N <= 16;
    const uint32_t bytes = (uint32_t)((a.tmaZ ? a.nzb : 0) + (a.tmaX ? a.nxb : 0)) * kBox;
    for (int g = 0; g < nchunk; ++g) {
      const int s = g % ST;
      const int64_t row0 = r0 + (int64_t)g * kDwS;
      if (zcoop || lane == 0) tc::mbar_wait(&empty[s], ((g / ST) & 1) ^ 1);
      if (zcoop) {
        for (int e = lane; e < kDwS * a.N; e += 32) {
          const int r = e / a.N, nn = e % a.N;
          uint8_t* dst = zraw(s) + r * 128 + ((nn * 4) ^ ((r & 3) << 5));
          if (row0 + r < r1) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(tc::smem_u32(dst)),
                         "l"(a.Z + (row0 + r) * a.ldz + nn) : "memory");
          } else {
            *reinterpret_cast<float*>(dst) = 0.f;
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(tc::smem_u32(&full[s])) : "memory");
      }
      if (lane == 0) {
        if (bytes) mbar_expect_tx(&full[s], bytes); else mbar_arrive(&full[s]);
        if (a.tmaZ)
          for (int b = 0; b < a.nzb; ++b) tma_load_2d(zraw(s) + b * kBox, &tmZ, &full[s], 32 * b, (int)row0);
        if (a.tmaX)
          for (int b = 0; b < a.nxb; ++b) tma_load_2d(xhi(s) + b * kBox, &tmX, &full[s], 32 * b, (int)row0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id = idesc_tf32(128, nprime, 0, 1);      // A = dZ^T K-major in TMEM, B MN-major
      for (int g = 0; g < nchunk; ++g) {
        const int s = g % ST;
        tc::mbar_wait(&conv[s], (g / ST) & 1);
        tc::fence_after();
        const uint32_t ah = tbase + 256 + 64 * s, al = ah + 32;
        const uint32_t bh = tc::smem_u32(xhi(s)), bl = tc::smem_u32(xlo(s));
#pragma unroll
        for (int j = 0; j < kDwS / 8; ++j) {
          // MN-major, 32-byte-chunk swizzle: 4-sample k-groups 512 B apart, 32-feature groups kBox apart
          const uint64_t dbh = desc_sw128<1>(bh + j * 1024, kBox, 512), dbl = desc_sw128<1>(bl + j * 1024, kBox, 512);
          mma_tf32_ts(tbase, al + 8 * j, dbh, id, (g | j) ? 1u : 0u);
          mma_tf32_ts(tbase, ah + 8 * j, dbl, id, 1u);
          mma_tf32_ts(tbase, ah + 8 * j, dbh, id, 1u);
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(&tfull);
    }
  } else if (warp >= 4) {
    // two converter warpgroups: half h owns samples [16h, 16h + 16) of every chunk (TMEM
    // columns) and every other X unit; both see all 128 TMEM lanes (warp quarter = lanes)
    const int t256 = tid - 128, half = t256 >> 7, ct = t256 & 127, quarter = warp & 3;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const bool vx = (a.ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
    const int n = ct;                                         // this thread's TMEM lane = output neuron
    const bool zcoop = !a.tmaZ && a.N <= 16;          // dZ gathered into zraw by the producer
    for (int g = 0; g < nchunk; ++g) {
      const int s = g % ST;
      const int64_t row0 = r0 + (int64_t)g * kDwS;
      tc::mbar_wait(&full[s], (g / ST) & 1);
      // dZ^T row n, samples [16h, 16h+16) -> hi/lo -> TMEM lane n
      uint32_t hi[16], lo[16];
      if (a.tmaZ || zcoop) {
        const uint8_t* zb = zraw(s) + (n >> 5) * kBox;
        const uint32_t nb = (uint32_t)(n & 31) * 4;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int r = 16 * half + j;
          const float v = *reinterpret_cast<const float*>(zb + r * 128 + (nb ^ ((r & 3u) << 5)));
          const float h = rna_tf32(v);
          hi[j] = __float_as_uint(h);
          lo[j] = __float_as_uint(v - h);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t row = row0 + 16 * half + j;
          const float v = (n < a.N && row < r1) ? __ldg(a.Z + row * a.ldz + n) : 0.f;
          const float h = rna_tf32(v);
          hi[j] = __float_as_uint(h);
          lo[j] = __float_as_uint(v - h);
        }
      }
      const uint32_t ta = tbase + lane_off + 256 + 64 * s + 16 * half;
      tc::tmem_st16(ta, hi);
      tc::tmem_st16(ta + 32, lo);
      // X -> hi (in place) / lo tiles in smem
      float4* h4 = reinterpret_cast<float4*>(xhi(s));
      float4* l4 = reinterpret_cast<float4*>(xlo(s));
      if (a.tmaX) {
        for (int q = t256; q < a.nxb * (kBox / 16); q += 256) {
          float4 h, l;
          split4(h4[q], h, l);
          h4[q] = h;
          l4[q] = l;
        }
      } else {
        for (int q = t256; q < a.nxb * (kBox / 16); q += 256) {
          const int b = q / (kBox / 16), r = (q / 8) % kDwS, u = q % 8;
          const int64_t row = row0 + r;
          float4 h, l;
          split4(load4(a.X + row * a.ldx, 32 * b + 4 * u, a.K, vx, row < r1), h, l);
          const uint32_t off = (b * kBox + sw32_off(r, u)) >> 4;
          h4[off] = h;
          l4[off] = l;
        }
      }
      tc::tmem_st_wait();
      tc::fence_before();
      tc::fence_proxy_async();
      mbar_arrive(&conv[s]);
    }
    // epilogue: TMEM lane n = output neuron, column k = input feature (column 32*nxb = db);
    // half h reads the 16-column blocks 2i + h
    if (nchunk > 0) {
      tc::mbar_wait(&tfull, 0);
      tc::fence_after();
      const uint32_t taddr = tbase + lane_off;
      for (int c0 = 16 * half; c0 < nprime; c0 += 32) {
        float v[16];
        tc::tmem_ld16(taddr + c0, v);
        tc::tmem_ld_wait();
        if (n < a.N) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int k = c0 + j;
            if (v[j] == 0.f) continue;
            if (k < a.K) atomicAdd(a.dW + (int64_t)k * a.N + n, v[j]);
            else if (k == 32 * a.nxb && a.db) atomicAdd(a.db + n, v[j]);
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_free<512>(tbase);
}

// ============================================================================ host side
// FV_G3_NOTMA=1: converter / producer warps load every operand themselves (exercises the
// path unaligned operands take; the tests also reach it with odd row strides)
static bool no_tma() {
  static const int v = [] { const char* e = std::getenv("FV_G3_NOTMA"); return e && e[0] == '1' ? 1 : 0; }();
  return v != 0;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// fp32 [rows x cols] with row stride ld (elements), box 32 columns x box_rows rows, 128B swizzle.
// Returns false when TMA cannot address it (row stride / base not 16-byte aligned).
static bool make_tmap(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld, int box_rows,
                      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  if (no_tma()) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 4) % 16 || rows < 1 || cols < 1) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

static constexpr int kSmemMax = 227 * 1024;

int32_t rows_gemm(RowsArgs a, cudaStream_t st) {
  if (a.N < 1 || a.N > 128 || a.K < 1 || a.K > 256) return set_error(FV_EDIM, "rows_gemm: unsupported shape");
  a.Np = (a.N + 15) / 16 * 16;
  a.nkc = (a.K + 31) / 32;
  a.nsteps = (a.K + 7) / 8;
  if (a.M == 0) return FV_OK;
  CUtensorMap tm{}, to{};
  a.tma = make_tmap(&tm, a.A, a.K, a.M, a.lda, 128) ? 1 : 0;
  a.tma_out = make_tmap(&to, a.out, a.N, a.M, a.ldo, 32) ? 1 : 0;
  const int bbytes = 2 * a.nkc * a.Np * 128;
  const int obytes = a.tma_out ? FV_G3_OBUF * kStageA : 0;
  a.stages = std::min(6, (kSmemMax - 2048 - bbytes - obytes) / kStageA);
  if (a.stages < 2) return set_error(FV_EDIM, "rows_gemm: B operand too large for shared memory");
  const size_t smem = 1024 + bbytes + (size_t)a.stages * kStageA + obytes;
  cudaFuncSetAttribute(k_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = (a.M + 127) / 128;
  const int grid = (int)std::min<int64_t>(ntiles, num_sms());
  k_rows<<<grid, 384, smem, st>>>(a, tm, to);
  return check_launch("k_rows");
}

int32_t dw_gemm(DwArgs3 a, cudaStream_t st) {
  if (a.N < 1 || a.N > 128 || a.K < 1 || a.K > 128) return set_error(FV_EDIM, "dw_gemm: unsupported shape");
  if (a.M == 0) return FV_OK;
  a.nxb = (a.K + 31) / 32;
  a.nzb = (a.N + 31) / 32;
  CUtensorMap tx{}, tz{};
  a.tmaX = make_tmap(&tx, a.X, a.K, a.M, a.ldx, kDwS, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ? 1 : 0;
  a.tmaZ = make_tmap(&tz, a.Z, a.N, a.M, a.ldz, kDwS, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ? 1 : 0;
  const int ncta = num_sms();
  a.rows_per_cta = ((a.M + ncta - 1) / ncta + kDwS - 1) / kDwS * kDwS;
  const int grid = (int)((a.M + a.rows_per_cta - 1) / a.rows_per_cta);
  const int stage_bytes = (4 + 2 * (a.nxb + 1)) * kBox;
  a.stages = std::min(4, (kSmemMax - 1024) / stage_bytes);
  const size_t smem = 1024 + (size_t)a.stages * stage_bytes;
  cudaFuncSetAttribute(k_dw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_dw<<<grid, 384, smem, st>>>(a, tx, tz);
  return check_launch("k_dw");
}

}  // namespace g3
}  // namespace fv
