// Layers with a narrow side (n_out <= 4: the residual MLP's 128 -> 3 output layer and the
// radiance MLP's 64 -> 4 head; `linear` ad:403-425) in fp32 SIMT.  A 128-row tensor-core
// tile would waste 124 of 128 MMA rows/columns on them and their operands do not fit the
// TMA boxes (12-byte rows), so these kernels simply stream the wide operand once, coalesced,
// with fp32 FMA accumulation (at least as accurate as the split-precision 3xTF32 GEMMs):
//   k_narrow_fwd : y[s][n] = act(sum_k x[s][k] W[k][n] + b[n])      warp per row, lanes split k
//   k_narrow_dx  : dx[s][k] = (sum_n dz[s][n] W[k][n]) * mask(s,k)    warp per row, lanes split k
//   k_narrow_dw  : dW[k][n] += sum_s x[s][k] dz[s][n], db[n] += sum_s dz[s][n]
#include <cuda_runtime.h>
#include "fv_internal.h"
#include "narrow_layers.h"

namespace fv {
namespace nl {

constexpr int kMaxN = 4;
constexpr int kRowsPerWarp = 4;            // rows in flight per warp iteration

// A row of K <= 128 columns is read by LPR = 32, 16 or 8 lanes (K > 64, > 32, <= 32), 4
// consecutive columns each, so 32 / LPR rows share one warp-wide load instruction.
__device__ __forceinline__ void load_row4(const float* row, int k, int K, bool vec, float (&v)[4]) {
  if (vec && k + 3 < K) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(row + k));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = k + j < K ? __ldg(row + k + j) : 0.f;
  }
}

template <int N, int LPR>
__global__ void __launch_bounds__(256) k_narrow_fwd(const float* __restrict__ x, int64_t ldx, int K,
                                                    const float* __restrict__ W, const float* __restrict__ b, int act,
                                                    float* __restrict__ y, int64_t ldy, int64_t M) {
  constexpr int RPI = 32 / LPR;                     // rows per warp-wide instruction
  __shared__ float sW[128 * kMaxN];
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) sW[i] = W[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane / LPR, li = lane % LPR;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  const int k0 = 4 * li;
  float w[4][N];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int n = 0; n < N; ++n) w[j][n] = k0 + j < K ? sW[(k0 + j) * N + n] : 0.f;
  constexpr int STEP = kRowsPerWarp * RPI;
  for (int64_t r0 = warp * STEP; r0 < M; r0 += nwarps * STEP) {
    float xv[kRowsPerWarp][4];
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q) {
      const int64_t r = r0 + q * RPI + sub;
      if (r < M) load_row4(x + r * ldx, k0, K, vec, xv[q]);
      else { xv[q][0] = xv[q][1] = xv[q][2] = xv[q][3] = 0.f; }
    }
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q) {
      const int64_t r = r0 + q * RPI + sub;
      float acc[N];
#pragma unroll
      for (int n = 0; n < N; ++n) {
        acc[n] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[n] = fmaf(xv[q][j], w[j][n], acc[n]);
      }
#pragma unroll
      for (int o = LPR / 2; o; o >>= 1)
#pragma unroll
        for (int n = 0; n < N; ++n) acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], o);
      if (li < N && r < M) {
        float v = acc[0];
#pragma unroll
        for (int n = 1; n < N; ++n) v = li == n ? acc[n] : v;
        v += b ? __ldg(b + li) : 0.f;
        if (act == 1) v = fmaxf(v, 0.f);
        y[r * ldy + li] = v;
      }
    }
  }
}

// dx row of K <= 128 columns (LPR lanes per row, 4 columns each); bits (one uint32 per 32
// columns) or a float mask zero the ReLU-inactive inputs.
// A warp handles 32 rows per iteration: lane l stages row l's dz (N floats) and ReLU-bit
// words in shared memory (one coalesced load batch for the 32 rows, the next batch already
// in flight), then the rows are written LPR lanes x 4 columns at a time (the kernel is a
// write stream of K floats per row).
template <int N, int LPR>
__global__ void __launch_bounds__(256) k_narrow_dx(const float* __restrict__ dz, int64_t ldz, const float* __restrict__ W,
                                                   int K, const uint32_t* __restrict__ bits,
                                                   const float* __restrict__ fmask, int64_t ldm,
                                                   float* __restrict__ dx, int64_t lddx, int64_t M) {
  constexpr int RPI = 32 / LPR;
  __shared__ float sW[128 * kMaxN];
  __shared__ float sdz[8][32 * N];
  __shared__ uint32_t sbits[8][32 * 4];
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) sW[i] = W[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, sub = lane / LPR, li = lane % LPR;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nw = (K + 31) / 32;
  const bool vout = (lddx % 4 == 0) && ((reinterpret_cast<uintptr_t>(dx) & 15) == 0) &&
                    (!fmask || ((ldm % 4 == 0) && ((reinterpret_cast<uintptr_t>(fmask) & 15) == 0)));
  const int k0 = 4 * li;
  float w[4][N];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int n = 0; n < N; ++n) w[j][n] = k0 + j < K ? sW[(k0 + j) * N + n] : 0.f;
  float gn[N];
  uint32_t bn[4];
  auto fetch = [&](int64_t g0) {   // lane l: row g0 + l
    const int64_t r = g0 + lane;
    const bool ok = r < M;
#pragma unroll
    for (int n = 0; n < N; ++n) gn[n] = ok ? __ldg(dz + r * ldz + n) : 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) bn[q] = (bits && ok && q < nw) ? __ldg(bits + r * nw + q) : 0xFFFFFFFFu;
  };
  int64_t g0 = warp * 32;
  if (g0 < M) fetch(g0);
  for (; g0 < M; g0 += nwarps * 32) {
#pragma unroll
    for (int n = 0; n < N; ++n) sdz[wib][lane * N + n] = gn[n];
#pragma unroll
    for (int q = 0; q < 4; ++q) sbits[wib][lane * 4 + q] = bn[q];
    __syncwarp();
    if (g0 + nwarps * 32 < M) fetch(g0 + nwarps * 32);   // next batch in flight during the stores
#pragma unroll 4
    for (int it = 0; it < 32 / RPI; ++it) {
      const int rr = it * RPI + sub;
      const int64_t r = g0 + rr;
      if (r >= M || k0 >= K) continue;
      float g[N];
#pragma unroll
      for (int n = 0; n < N; ++n) g[n] = sdz[wib][rr * N + n];
      const uint32_t mb = sbits[wib][rr * 4 + (k0 >> 5)];
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int n = 0; n < N; ++n) acc = fmaf(g[n], w[j][n], acc);
        if (bits && !((mb >> ((k0 + j) & 31)) & 1u)) acc = 0.f;
        o[j] = acc;
      }
      float* dst = dx + r * lddx + k0;
      if (fmask) {
        const float* mrow = fmask + r * ldm + k0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (k0 + j < K && !(__ldg(mrow + j) > 0.f)) o[j] = 0.f;
      }
      if (vout && k0 + 3 < K) {
        *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (k0 + j < K) dst[j] = o[j];
      }
    }
    __syncwarp();
  }
}

// dW: block-private partial sums over a contiguous row range (LPR lanes per row, lane owns
// columns 4li..4li+3 of x), folded across the row groups of a warp by shuffles and across
// the block's warps in shared memory, then one atomicAdd per weight.
template <int N, int LPR>
__global__ void __launch_bounds__(256) k_narrow_dw(const float* __restrict__ x, int64_t ldx, int K,
                                                   const float* __restrict__ dz, int64_t ldz,
                                                   float* __restrict__ dW, float* __restrict__ db, int64_t M,
                                                   int64_t rows_per_block) {
  constexpr int RPI = 32 / LPR;
  __shared__ float red[8][128 * kMaxN + kMaxN];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, sub = lane / LPR, li = lane % LPR;
  const bool vec = (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  const int64_t rb = (int64_t)blockIdx.x * rows_per_block;
  const int64_t re = rb + rows_per_block < M ? rb + rows_per_block : M;
  const int k0 = 4 * li;
  float acc[4][N], accb[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    accb[n] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][n] = 0.f;
  }
  constexpr int STEP = kRowsPerWarp * RPI;
  for (int64_t r0 = rb + wib * STEP; r0 < re; r0 += 8 * STEP) {
    float xv[kRowsPerWarp][4], g[kRowsPerWarp][N];
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q) {
      const int64_t r = r0 + q * RPI + sub;
      const bool ok = r < re;
      if (ok) load_row4(x + r * ldx, k0, K, vec, xv[q]);
      else { xv[q][0] = xv[q][1] = xv[q][2] = xv[q][3] = 0.f; }
#pragma unroll
      for (int n = 0; n < N; ++n) g[q][n] = ok ? __ldg(dz + r * ldz + n) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q)
#pragma unroll
      for (int n = 0; n < N; ++n) {
        accb[n] += g[q][n];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j][n] = fmaf(xv[q][j], g[q][n], acc[j][n]);
      }
  }
#pragma unroll
  for (int o = 16; o >= LPR; o >>= 1)                // fold the row groups of the warp
#pragma unroll
    for (int n = 0; n < N; ++n) {
      accb[n] += __shfl_xor_sync(0xffffffffu, accb[n], o);
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j][n] += __shfl_xor_sync(0xffffffffu, acc[j][n], o);
    }
  if (sub == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int n = 0; n < N; ++n) red[wib][(k0 + j) * N + n] = acc[j][n];
    if (li == 0) {
#pragma unroll
      for (int n = 0; n < N; ++n) red[wib][128 * N + n] = accb[n];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K * N + N; i += blockDim.x) {
    const int src = i < K * N ? i : 128 * N + (i - K * N);
    float s = 0.f;
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) s += red[w8][src];
    if (s == 0.f) continue;
    if (i < K * N) atomicAdd(dW + i, s);
    else if (db) atomicAdd(db + (i - K * N), s);
  }
}

static int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

#define FV_NARROW_SWITCH(KERNEL, GRID, ...)                                                  \
  do {                                                                                       \
    const int lpr = K > 64 ? 32 : (K > 32 ? 16 : 8);                                         \
    switch (N * 100 + lpr) {                                                                 \
      case 132: KERNEL<1, 32><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                     \
      case 116: KERNEL<1, 16><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                     \
      case 108: KERNEL<1, 8><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                      \
      case 232: KERNEL<2, 32><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                     \
      case 216: KERNEL<2, 16><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                     \
      case 208: KERNEL<2, 8><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                      \
      case 332: KERNEL<3, 32><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                     \
      case 316: KERNEL<3, 16><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                     \
      case 308: KERNEL<3, 8><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                      \
      case 432: KERNEL<4, 32><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                     \
      case 416: KERNEL<4, 16><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                     \
      default: KERNEL<4, 8><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                       \
    }                                                                                        \
  } while (0)

static int grid_rows(int64_t M, int K) {
  const int rpi = K > 64 ? 1 : (K > 32 ? 2 : 4);
  const int64_t warps = (M + kRowsPerWarp * rpi - 1) / (kRowsPerWarp * rpi);
  return (int)std::min<int64_t>((warps + 7) / 8, (int64_t)sms() * 16);
}

int32_t narrow_fwd(const float* x, int64_t ldx, int K, const float* W, const float* b, int act, float* y,
                   int64_t ldy, int64_t M, int N, cudaStream_t st) {
  if (N < 1 || N > kMaxN || K < 1 || K > 128) return set_error(FV_EDIM, "narrow_fwd: shape");
  const int grid = grid_rows(M, K);
  FV_NARROW_SWITCH(k_narrow_fwd, grid, x, ldx, K, W, b, act, y, ldy, M);
  return check_launch("k_narrow_fwd");
}

int32_t narrow_dx(const float* dz, int64_t ldz, int N, const float* W, int K, const uint32_t* bits,
                  const float* fmask, int64_t ldm, float* dx, int64_t lddx, int64_t M, cudaStream_t st) {
  if (N < 1 || N > kMaxN || K < 1 || K > 128) return set_error(FV_EDIM, "narrow_dx: shape");
  const int grid = (int)std::min<int64_t>(((M + 31) / 32 + 7) / 8, (int64_t)sms() * 8);
  FV_NARROW_SWITCH(k_narrow_dx, grid, dz, ldz, W, K, bits, fmask, ldm, dx, lddx, M);
  return check_launch("k_narrow_dx");
}

int32_t narrow_dw(const float* x, int64_t ldx, int K, const float* dz, int64_t ldz, int N, float* dW, float* db,
                  int64_t M, cudaStream_t st) {
  if (N < 1 || N > kMaxN || K < 1 || K > 128) return set_error(FV_EDIM, "narrow_dw: shape");
  const int blocks = sms() * 4;
  int64_t rpb = (M + blocks - 1) / blocks;
  rpb = (rpb + 8 * kRowsPerWarp * 4 - 1) / (8 * kRowsPerWarp * 4) * (8 * kRowsPerWarp * 4);
  const int grid = (int)((M + rpb - 1) / rpb);
  FV_NARROW_SWITCH(k_narrow_dw, grid, x, ldx, K, dz, ldz, dW, db, M, rpb);
  return check_launch("k_narrow_dw");
}

}  // namespace nl
}  // namespace fv
