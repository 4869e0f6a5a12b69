// Probe: D = A * B^T with the A operand in TMEM (tcgen05.mma ... [a_tmem], b_desc), written
// by tcgen05.st from registers: thread r of the warpgroup owns row r = TMEM lane r and stores
// word j = half2(A[r][2j], A[r][2j+1]) (low half = even k) at column a_base + j.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tc_selftest_ts.cu -o tc_selftest_ts
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2306_16541_b200/csrc/tc_sm100.cuh"

using namespace fv;
constexpr int K = 48, N = 128;

__global__ void __launch_bounds__(128) probe(const __half* A, const __half* B, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  for (int r = t; r < N; r += 128)
    for (int c = 0; c < K / 8; ++c)
      *reinterpret_cast<uint4*>(smem + tc::op_off(N, r, c)) = *reinterpret_cast<const uint4*>(B + r * K + c * 8);
  if (warp == 0) tc::tmem_alloc<256>(&tmem_base);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tb = tmem_base, lane = (uint32_t)(warp * 32) << 16;
  uint32_t w[K / 2];
  for (int j = 0; j < K / 2; ++j) w[j] = *reinterpret_cast<const uint32_t*>(A + t * K + 2 * j);
  tc::tmem_st8(tb + lane + 128, w);
  tc::tmem_st16(tb + lane + 136, w + 8);
  tc::tmem_st_wait();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (t == 0) {
    for (int k = 0; k < K / 16; ++k)
      tc::mma_f16_ts(tb, tb + 128 + k * 8, tc::make_desc(tc::smem_u32(smem) + k * 2 * N * 16, N * 16, 128),
                     tc::idesc_f16(128, N), k > 0);
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tb + lane + c0, v);
    tc::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) D[t * N + c0 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<256>(tb);
}

int main() {
  std::vector<__half> a(128 * K), b(N * K);
  std::vector<float> af(128 * K), bf(N * K), d(128 * N);
  srand(1);
  for (int i = 0; i < 128 * K; ++i) { a[i] = __float2half((rand() % 17 - 8) / 8.f); af[i] = __half2float(a[i]); }
  for (int i = 0; i < N * K; ++i) { b[i] = __float2half((rand() % 13 - 6) / 4.f); bf[i] = __half2float(b[i]); }
  __half *da, *db; float* dd;
  cudaMalloc(&da, a.size() * 2); cudaMalloc(&db, b.size() * 2); cudaMalloc(&dd, d.size() * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  probe<<<1, 128, N * K * 2>>>(da, db, dd);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)af[r * K + k] * bf[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - d[r * N + n]));
    }
  printf("A-in-TMEM probe K=%d N=%d: %s, max |err| = %g -> %s\n", K, N, cudaGetErrorString(e), maxerr,
         maxerr < 1e-3 ? "PASS" : "FAIL");
  return maxerr < 1e-3 ? 0 : 1;
}
