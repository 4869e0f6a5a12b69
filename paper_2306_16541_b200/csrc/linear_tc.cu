// Training-time MLP layers on 5th-gen tensor cores, kind::tf32 (fp32 storage, TF32 math,
// fp32 accumulation): the layer ops of the reference training step (ad:403-425 forward,
// ad:417-422 backward) for the tall-skinny shapes of the path (M = samples, K, N <= 128).
//
// Why TF32 rather than fp16 here: dW reduces over ~786K samples of gradients that are
// 1e-9..1e-5 in magnitude -- below fp16's normal range -- and the layers are memory bound
// (fp32 activations in HBM), so TF32's half MMA rate costs nothing.
//
// k_lin_tc   : out[M x N] = epi(A[M x K] . B) with B(n,k) = W[n*sbn + k*sbk]; covers
//              forward (B = W^T view, bias + act) and dX (B = W view, ReLU mask of the
//              layer input applied in the epilogue so the next GEMM reads dZ directly).
// k_lin_dw_tc: dW[K x N] += X^T . dZ over a slice of samples per CTA; both operands are
//              transposed while staging into shared memory so the MMA sees K-major tiles
//              (MN-major TF32 needs the 128B/32B-atom swizzle; the transposing fill is
//              bank-conflict free instead).
#include <cuda_runtime.h>
#include "fv_common.cuh"
#include "fv_internal.h"
#include "tc_sm100.cuh"
#include "gemm_tf32x3.h"
#include <cstdlib>

namespace fv {

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

template <uint32_t NC>
__device__ __forceinline__ void tmem_alloc_n(uint32_t* dst) { tc::tmem_alloc<NC>(dst); }

constexpr int KC = 32;  // K elements staged per chunk (4 MMAs of K = 8)

struct LinArgs {
  const float* A; int64_t lda; int K;          // A (M x K) row-major
  const float* W; int64_t sbn, sbk; int N;     // B(n,k) = W[n*sbn + k*sbk]
  int Kp, Np;                                  // padded: Kp % 32 == 0, Np % 16 == 0, Np <= 128
  const float* bias; int act;                  // epilogue: + bias[n], act 1 = ReLU
  const float* mask; int64_t ldm;              // epilogue: * (mask[m*ldm + n] > 0) if mask
  float* out; int64_t ldo; int64_t M;
  int split;                                   // 1: 3xTF32 (hi*hi + hi*lo + lo*hi), ~fp32 accurate
};

// hi = fp32 rounded to TF32 (low 13 mantissa bits zero), lo = x - hi (exact)
__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// word (row r, chunk c) of an R-row K-major tf32 tile: 4 floats at c*R*16 + r*16 bytes
__device__ __forceinline__ uint32_t kmaj(int R, int r, int k) { return (uint32_t)((k >> 2) * R * 4 + r * 4 + (k & 3)); }

__global__ void __launch_bounds__(128) k_lin_tc(LinArgs a) {
  extern __shared__ __align__(1024) float sm[];
  // smem: B hi [Np x Kp] (+ B lo), then 2 stages of A hi [128 x KC] (+ A lo)
  const int nsplit = a.split ? 2 : 1;
  float* sB = sm;
  float* sBlo = sm + a.Np * a.Kp;
  float* sA = sm + nsplit * a.Np * a.Kp;
  const int astage = nsplit * 128 * KC;
  __shared__ uint64_t bars[2];
  __shared__ uint32_t tmem;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < a.Np * a.Kp; i += 128) {
    const int n = i / a.Kp, k = i % a.Kp;
    const float w = (n < a.N && k < a.K) ? __ldg(a.W + n * a.sbn + k * a.sbk) : 0.f;
    if (a.split) {
      const float hi = tf32_hi(w);
      sB[kmaj(a.Np, n, k)] = hi;
      sBlo[kmaj(a.Np, n, k)] = w - hi;
    } else {
      sB[kmaj(a.Np, n, k)] = w;
    }
  }
  if (warp == 0) tc::tmem_alloc<128>(&tmem);
  if (t == 0) { tc::mbar_init(&bars[0], 1); tc::mbar_init(&bars[1], 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem;
  const uint32_t trow = tbase + ((uint32_t)(warp * 32) << 16);
  const uint32_t id = idesc_tf32(128, a.Np);
  const int nchunk = a.Kp / KC;
  // rows 16-byte aligned -> float4 loads (a K % 4 tail reads the row padding and is zeroed)
  const bool vec = (a.lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.A) & 15) == 0);
  const bool vout = (a.ldo % 4 == 0) && (a.N % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0) &&
                    (!a.mask || ((a.ldm % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.mask) & 15) == 0)));
  uint32_t used[2] = {0, 0};      // commits issued per stage
  const int64_t ntiles = (a.M + 127) / 128;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t m0 = tile * 128;
    for (int c = 0; c < nchunk; ++c) {
      const int st = (int)((used[0] + used[1]) & 1);
      if (used[st]) tc::mbar_wait(&bars[st], (used[st] - 1) & 1);   // MMAs reading this stage are done
      float* S = sA + st * astage;
      float* Slo = S + 128 * KC;
      // row t of the tile, columns [c*KC, c*KC+KC): conflict-free 16-byte stores
      const int64_t m = m0 + t;
      const float* src = a.A + m * a.lda + c * KC;
#pragma unroll
      for (int j = 0; j < KC / 4; ++j) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        const int k = c * KC + 4 * j;
        if (m < a.M) {
          if (vec) {
            if (k < a.K) {
              v = __ldg(reinterpret_cast<const float4*>(src + 4 * j));
              if (k + 3 >= a.K) { v.w = 0.f; if (k + 2 >= a.K) v.z = 0.f; if (k + 1 >= a.K) v.y = 0.f; }
            }
          } else {
            v.x = k < a.K ? __ldg(src + 4 * j) : 0.f;         v.y = k + 1 < a.K ? __ldg(src + 4 * j + 1) : 0.f;
            v.z = k + 2 < a.K ? __ldg(src + 4 * j + 2) : 0.f; v.w = k + 3 < a.K ? __ldg(src + 4 * j + 3) : 0.f;
          }
        }
        if (a.split) {
          const float4 hi = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
          *reinterpret_cast<float4*>(S + kmaj(128, t, 4 * j)) = hi;
          *reinterpret_cast<float4*>(Slo + kmaj(128, t, 4 * j)) =
              make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
        } else {
          *reinterpret_cast<float4*>(S + kmaj(128, t, 4 * j)) = v;
        }
      }
      tc::fence_proxy_async();
      __syncthreads();
      if (t == 0) {
        tc::fence_after();
#pragma unroll
        for (int j = 0; j < KC / 8; ++j) {
          const uint32_t aoff = j * 2 * 128 * 16, boff = (c * (KC / 4) + j * 2) * a.Np * 16;
          const uint64_t ad = tc::make_desc(tc::smem_u32(S) + aoff, 128 * 16, 128);
          const uint64_t bd = tc::make_desc(tc::smem_u32(sB) + boff, a.Np * 16, 128);
          if (a.split) {  // small terms first, the dominant hi*hi last
            mma_tf32(tbase, tc::make_desc(tc::smem_u32(Slo) + aoff, 128 * 16, 128), bd, id, (c | j) ? 1u : 0u);
            mma_tf32(tbase, ad, tc::make_desc(tc::smem_u32(sBlo) + boff, a.Np * 16, 128), id, 1u);
            mma_tf32(tbase, ad, bd, id, 1u);
          } else {
            mma_tf32(tbase, ad, bd, id, (c | j) ? 1u : 0u);
          }
        }
        tc::mma_commit(&bars[st]);
      }
      __syncwarp();
      used[st]++;
    }
    const int last = (int)((used[0] + used[1] - 1) & 1);
    tc::mbar_wait(&bars[last], (used[last] - 1) & 1);
    tc::fence_after();
    const int64_t m = m0 + t;
    for (int n0 = 0; n0 < a.Np; n0 += 16) {
      float v[16];
      tc::tmem_ld16(trow + n0, v);
      tc::tmem_ld_wait();
      if (m < a.M) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          v[j] += (a.bias && n0 + j < a.N) ? a.bias[n0 + j] : 0.f;
          if (a.act == 1) v[j] = fmaxf(v[j], 0.f);
        }
        if (vout) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int n = n0 + 4 * q;
            if (n >= a.N) break;
            float4 y = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            if (a.mask) {
              const float4 mk = __ldg(reinterpret_cast<const float4*>(a.mask + m * a.ldm + n));
              y.x = mk.x > 0.f ? y.x : 0.f; y.y = mk.y > 0.f ? y.y : 0.f;
              y.z = mk.z > 0.f ? y.z : 0.f; y.w = mk.w > 0.f ? y.w : 0.f;
            }
            *reinterpret_cast<float4*>(a.out + m * a.ldo + n) = y;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = n0 + j;
            if (n < a.N) {
              float y = v[j];
              if (a.mask && !(a.mask[m * a.ldm + n] > 0.f)) y = 0.f;
              a.out[m * a.ldo + n] = y;
            }
          }
        }
      }
    }
    tc::fence_before();
    __syncthreads();
  }
  if (warp == 0) tc::tmem_free<128>(tbase);
}

struct DwArgs {
  const float* X; int64_t ldx; int K;          // layer input  (M x K)
  const float* Z; int64_t ldz; int N;          // dZ           (M x N), already ReLU-masked
  int Np;                                      // N padded to 16 (<= 128); K <= 128 (M' = 128)
  float* dW;                                   // (K x N) accumulate
  int64_t M, rows_per_cta;
};

// D[k][n] = sum_s X[s][k] dZ[s][n]: A' = X^T (128 x samples), B' = dZ^T (Np x samples).
// Staging transposes through registers: every thread issues all of its chunk loads before
// any shared store (the load->store-per-element form was latency bound), only the
// ceil(K/8) k-blocks that exist are staged (rows >= K stay zero from the prologue), and
// db = colsum(dZ) is reduced from the staged dZ^T tile.  The reduction over ~10^6 samples
// of sign-mixed products cancels heavily, so both operands are split hi/lo (3xTF32).
constexpr int KW = 16;                   // samples per dW chunk (2 MMAs of K = 8, x3 split)

__global__ void __launch_bounds__(128) k_lin_dw_tc(DwArgs a, float* __restrict__ db) {
  extern __shared__ __align__(1024) float sm[];
  const int zt = a.Np * KW;              // floats of one dZ^T tile
  // stage layout: X hi [128 x KW] | X lo | Z hi [Np x KW] | Z lo
  const int stage_f = 2 * 128 * KW + 2 * zt;
  __shared__ uint64_t bars[2];
  __shared__ uint32_t tmem;
  const int t = threadIdx.x, warp = t >> 5;
  const int kblk = (a.K + 7) / 8;
  for (int i = t; i < 2 * stage_f; i += 128) {    // zero everything once (rows k >= 8*kblk stay 0)
    sm[i] = 0.f;
  }
  if (warp == 0) tc::tmem_alloc<128>(&tmem);
  if (t == 0) { tc::mbar_init(&bars[0], 1); tc::mbar_init(&bars[1], 1); tc::mbar_fence_init(); }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem;
  const uint32_t id = idesc_tf32(128, a.Np);
  const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r1 = r0 + a.rows_per_cta < a.M ? r0 + a.rows_per_cta : a.M;
  const int nx = kblk;                   // X elements per thread per chunk (kblk*8*KW/128)
  const int nz = a.Np / 8;               // Z elements per thread per chunk (Np*KW/128)
  const int nzb = a.Np / 8;
  float dbacc = 0.f;
  uint32_t used[2] = {0, 0};
  int chunk = 0;
  for (int64_t s0 = r0; s0 < r1; s0 += KW, ++chunk) {
    const int st = chunk & 1;
    float vx[16], vz[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {       // e -> (s4 = e&3, k8 = (e>>2)&7, block): lanes cover 32 words
      if (i < nx) {
        const int e = t + 128 * i;
        const int q = e >> 5, k = (q % kblk) * 8 + ((e >> 2) & 7), s = (q / kblk) * 4 + (e & 3);
        const int64_t row = s0 + s;
        vx[i] = (k < a.K && row < r1) ? __ldg(a.X + row * a.ldx + k) : 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < nz) {
        const int e = t + 128 * i;
        const int q = e >> 5, n = (q % nzb) * 8 + ((e >> 2) & 7), s = (q / nzb) * 4 + (e & 3);
        const int64_t row = s0 + s;
        vz[i] = (n < a.N && row < r1) ? __ldg(a.Z + row * a.ldz + n) : 0.f;
      }
    }
    if (used[st]) tc::mbar_wait(&bars[st], (used[st] - 1) & 1);   // MMAs of 2 chunks ago are done
    float* SX = sm + st * stage_f;
    float* SXl = SX + 128 * KW;
    float* SZ = SXl + 128 * KW;
    float* SZl = SZ + zt;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < nx) {
        const int e = t + 128 * i;
        const int q = e >> 5;
        const uint32_t o = kmaj(128, (q % kblk) * 8 + ((e >> 2) & 7), (q / kblk) * 4 + (e & 3));
        const float hi = tf32_hi(vx[i]);
        SX[o] = hi;
        SXl[o] = vx[i] - hi;
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < nz) {
        const int e = t + 128 * i;
        const int q = e >> 5;
        const uint32_t o = kmaj(a.Np, (q % nzb) * 8 + ((e >> 2) & 7), (q / nzb) * 4 + (e & 3));
        const float hi = tf32_hi(vz[i]);
        SZ[o] = hi;
        SZl[o] = vz[i] - hi;
      }
    }
    tc::fence_proxy_async();
    __syncthreads();
    if (t == 0) {
      tc::fence_after();
#pragma unroll
      for (int j = 0; j < KW / 8; ++j) {
        const uint32_t ao = j * 2 * 128 * 16, bo = j * 2 * a.Np * 16;
        const uint64_t ad = tc::make_desc(tc::smem_u32(SX) + ao, 128 * 16, 128);
        const uint64_t bd = tc::make_desc(tc::smem_u32(SZ) + bo, a.Np * 16, 128);
        mma_tf32(tbase, tc::make_desc(tc::smem_u32(SXl) + ao, 128 * 16, 128), bd, id, (chunk | j) ? 1u : 0u);
        mma_tf32(tbase, ad, tc::make_desc(tc::smem_u32(SZl) + bo, a.Np * 16, 128), id, 1u);
        mma_tf32(tbase, ad, bd, id, 1u);
      }
      tc::mma_commit(&bars[st]);
    }
    __syncwarp();
    if (db && t < a.Np) {                // row t of dZ^T (hi + lo): KW samples as conflict-free float4
#pragma unroll
      for (int j = 0; j < KW / 4; ++j) {
        const float4 h4 = *reinterpret_cast<const float4*>(SZ + j * a.Np * 4 + t * 4);
        const float4 l4 = *reinterpret_cast<const float4*>(SZl + j * a.Np * 4 + t * 4);
        dbacc += ((h4.x + l4.x) + (h4.y + l4.y)) + ((h4.z + l4.z) + (h4.w + l4.w));
      }
    }
    used[st]++;
  }
  if (chunk > 0) {
    const int last = (chunk - 1) & 1;
    tc::mbar_wait(&bars[last], (used[last] - 1) & 1);
    tc::fence_after();
    const uint32_t trow = tbase + ((uint32_t)(warp * 32) << 16);
    for (int n0 = 0; n0 < a.Np; n0 += 16) {
      float v[16];
      tc::tmem_ld16(trow + n0, v);
      tc::tmem_ld_wait();
      if (t < a.K) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (n0 + j < a.N && v[j] != 0.f) atomicAdd(a.dW + (int64_t)t * a.N + n0 + j, v[j]);
      }
    }
    if (db && t < a.N && dbacc != 0.f) atomicAdd(db + t, dbacc);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<128>(tbase);
}

static int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int32_t lin_tc(const LinArgs& a, cudaStream_t st) {
  if (a.Np > 128 || a.Np % 16 || a.Kp % KC || a.Kp > 256) return set_error(FV_EDIM, "lin_tc: unsupported shape");
  const size_t smem = (size_t)((a.split ? 2 : 1) * (a.Np * a.Kp + 2 * 128 * KC)) * 4;
  cudaFuncSetAttribute(k_lin_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = (a.M + 127) / 128;
  const int grid = (int)std::min<int64_t>(ntiles, 2 * num_sms());
  k_lin_tc<<<grid, 128, smem, st>>>(a);
  return check_launch("k_lin_tc");
}

int32_t lin_dw_tc(const DwArgs& a0, float* db, cudaStream_t st) {
  DwArgs a = a0;
  if (a.Np > 128 || a.Np % 16 || a.K > 128) return set_error(FV_EDIM, "lin_dw_tc: unsupported shape");
  const int ncta = 3 * num_sms();
  a.rows_per_cta = ((a.M + ncta - 1) / ncta + KW - 1) / KW * KW;
  const int grid = (int)((a.M + a.rows_per_cta - 1) / a.rows_per_cta);
  const size_t smem = (size_t)2 * (2 * 128 * KW + 2 * a.Np * KW) * 4;
  cudaFuncSetAttribute(k_lin_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_lin_dw_tc<<<grid, 128, smem, st>>>(a, db);
  return check_launch("k_lin_dw_tc");
}

static int pad(int x, int m) { return (x + m - 1) / m * m; }

// FV_LEGACY_LIN=1 selects the round-1 per-CTA kernels (A/B timing only)
static bool legacy() {
  static const int v = [] { const char* e = std::getenv("FV_LEGACY_LIN"); return e && e[0] == '1' ? 1 : 0; }();
  return v != 0;
}

}  // namespace fv

using namespace fv;

// y = act(x @ W + b) with TF32 tensor cores.  W (k_in, n_out) row-major; x rows have
// stride ldx >= k_in, y rows stride ldy >= n_out.
extern "C" int32_t fv_linear_fwd_tc(const float* d_x, int64_t ldx, const float* d_w, const float* d_b, float* d_y,
                                    int64_t ldy, int64_t m, int32_t k_in, int32_t n_out, int32_t act, void* stream) {
  if (m < 0 || k_in < 1 || k_in > 256 || n_out < 1 || n_out > 128 || ldx < k_in || ldy < n_out)
    return set_error(FV_EDIM, "fv_linear_fwd_tc: bad shape");
  if (m == 0) return FV_OK;
  // forward activations feed the next layer and, through x_final, the hash-cell positions,
  // so the forward runs split-precision 3xTF32 (~fp32); backward GEMMs are plain TF32
  if (!legacy()) {
    g3::RowsArgs r{d_x, ldx, k_in, d_w, 1, n_out, n_out, d_b, act, nullptr, 0, d_y, ldy, m};
    return g3::rows_gemm(r, (cudaStream_t)stream);
  }
  LinArgs a{d_x, ldx, k_in, d_w, 1, n_out, n_out, pad(k_in, KC), pad(n_out, 16), d_b, act, nullptr, 0, d_y, ldy, m, 1};
  return lin_tc(a, (cudaStream_t)stream);
}

// Backward of fv_linear_fwd_tc given dz = dL/d(pre-activation) (already masked):
//   dx = (dz @ W^T) * (x_mask > 0 if x_mask)     (x_mask = the layer input, i.e. the previous
//                                                  layer's ReLU output -> dz of that layer)
//   dW += x^T dz ; db += colsum(dz)
extern "C" int32_t fv_linear_bwd_tc(const float* d_x, int64_t ldx, const float* d_w, const float* d_dz, int64_t ldz,
                                    float* d_dx, int64_t lddx, const float* d_xmask, float* d_dw, float* d_db,
                                    int64_t m, int32_t k_in, int32_t n_out, void* stream) {
  if (m < 0 || k_in < 1 || k_in > 128 || n_out < 1 || n_out > 128 || ldx < k_in || ldz < n_out)
    return set_error(FV_EDIM, "fv_linear_bwd_tc: bad shape");
  if (m == 0) return FV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (d_dx) {
    // dx[m, k] = sum_n dz[m, n] W[k, n]  : K' = n_out, N' = k_in, B(n'=k, k'=n) = W[k*n_out + n]
    if (!legacy()) {
      g3::RowsArgs r{d_dz, ldz, n_out, d_w, n_out, 1, k_in, nullptr, 0, d_xmask, ldx, d_dx, lddx, m};
      if (int32_t e = g3::rows_gemm(r, st)) return e;
    } else {
      LinArgs a{d_dz, ldz, n_out, d_w, n_out, 1, k_in, pad(n_out, KC), pad(k_in, 16), nullptr, 0, d_xmask, ldx,
                d_dx, lddx, m, 1};   // dx feeds the rest of the backward chain: 3xTF32 too
      if (int32_t e = lin_tc(a, st)) return e;
    }
  }
  if (d_dw) {
    if (!legacy()) {
      g3::DwArgs3 w{d_x, ldx, k_in, d_dz, ldz, n_out, d_dw, d_db, m};
      if (int32_t e = g3::dw_gemm(w, st)) return e;
    } else {
      DwArgs a{d_x, ldx, k_in, d_dz, ldz, n_out, pad(n_out, 16), d_dw, m, 0};
      if (int32_t e = lin_dw_tc(a, d_db, st)) return e;
    }
  }
  return FV_OK;
}

// Bit-mask forms (training path): the forward also writes the ReLU mask as bits
// (bit j of word w of row m <-> output column 32w + j is > 0, [m][ceil(n_out/32)] words),
// and the backward applies such bits to dx instead of reading the float activations.
extern "C" int32_t fv_linear_fwd_tc_bits(const float* d_x, int64_t ldx, const float* d_w, const float* d_b,
                                         float* d_y, int64_t ldy, int64_t m, int32_t k_in, int32_t n_out,
                                         int32_t act, uint32_t* d_relu_bits, void* stream) {
  if (m < 0 || k_in < 1 || k_in > 256 || n_out < 1 || n_out > 128 || ldx < k_in || ldy < n_out)
    return set_error(FV_EDIM, "fv_linear_fwd_tc_bits: bad shape");
  if (m == 0) return FV_OK;
  g3::RowsArgs r{d_x, ldx, k_in, d_w, 1, n_out, n_out, d_b, act, nullptr, 0, d_y, ldy, m};
  r.bits_out = d_relu_bits;
  return g3::rows_gemm(r, (cudaStream_t)stream);
}

extern "C" int32_t fv_linear_bwd_tc_bits(const float* d_x, int64_t ldx, const float* d_w, const float* d_dz,
                                         int64_t ldz, float* d_dx, int64_t lddx, const uint32_t* d_xmask_bits,
                                         float* d_dw, float* d_db, int64_t m, int32_t k_in, int32_t n_out,
                                         void* stream) {
  if (m < 0 || k_in < 1 || k_in > 128 || n_out < 1 || n_out > 128 || ldx < k_in || ldz < n_out)
    return set_error(FV_EDIM, "fv_linear_bwd_tc_bits: bad shape");
  if (m == 0) return FV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (d_dx) {
    g3::RowsArgs r{d_dz, ldz, n_out, d_w, n_out, 1, k_in, nullptr, 0, nullptr, 0, d_dx, lddx, m};
    r.bits_in = d_xmask_bits;
    if (int32_t e = g3::rows_gemm(r, st)) return e;
  }
  if (d_dw) {
    g3::DwArgs3 w{d_x, ldx, k_in, d_dz, ldz, n_out, d_dw, d_db, m};
    if (int32_t e = g3::dw_gemm(w, st)) return e;
  }
  return FV_OK;
}
