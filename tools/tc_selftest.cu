// Standalone probe: one CTA computes D = A * B^T (fp16 in, fp32 accum) with tcgen05 for
// several (K, N) shapes at M = 128 and checks against a host reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I.. tc_selftest.cu -o tc_selftest
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2306_16541_b200/csrc/tc_sm100.cuh"

using namespace fv;

template <int K, int N>
__global__ void __launch_bounds__(128) gemm_probe(const __half* A, const __half* B, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                       // 128*K*2 bytes
  uint8_t* sB = smem + 128 * K * 2;         // N*K*2 bytes
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  // A: row t
  for (int c = 0; c < K / 8; ++c) {
    uint4 w = *reinterpret_cast<const uint4*>(A + t * K + c * 8);
    *reinterpret_cast<uint4*>(sA + tc::op_off(128, t, c)) = w;
  }
  for (int r = t; r < N; r += 128)
    for (int c = 0; c < K / 8; ++c) {
      uint4 w = *reinterpret_cast<const uint4*>(B + r * K + c * 8);
      *reinterpret_cast<uint4*>(sB + tc::op_off(N, r, c)) = w;
    }
  if (warp == 0) tc::tmem_alloc<(N < 32 ? 32 : N)>(&tmem_base);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tb = tmem_base;
  if (t == 0) {
    const uint32_t id = tc::idesc_f16(128, N);
    for (int k = 0; k < K / 16; ++k) {
      uint64_t ad = tc::make_desc(tc::smem_u32(sA) + k * 2 * 128 * 16, 128 * 16, 128);
      uint64_t bd = tc::make_desc(tc::smem_u32(sB) + k * 2 * N * 16, N * 16, 128);
      tc::mma_f16(tb, ad, bd, id, k > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) D[t * N + c0 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<(N < 32 ? 32 : N)>(tb);
}

template <int K, int N>
int run() {
  std::vector<__half> A(128 * K), B(N * K);
  std::vector<float> Af(128 * K), Bf(N * K), D(128 * N);
  srand(K * 1000 + N);
  for (int i = 0; i < 128 * K; ++i) { float x = (rand() % 2001 - 1000) / 1000.f; A[i] = __float2half(x); Af[i] = __half2float(A[i]); }
  for (int i = 0; i < N * K; ++i) { float x = (rand() % 2001 - 1000) / 1000.f; B[i] = __float2half(x); Bf[i] = __half2float(B[i]); }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  size_t sm = 128 * K * 2 + N * K * 2;
  cudaFuncSetAttribute(gemm_probe<K, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  gemm_probe<K, N><<<1, 128, sm>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("K=%d N=%d CUDA error %s\n", K, N, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)Af[m * K + k] * Bf[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
    }
  printf("K=%d N=%d maxerr=%.3e %s\n", K, N, maxerr, maxerr < 1e-3 ? "OK" : "FAIL");
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return maxerr < 1e-3 ? 0 : 1;
}

int main() {
  int bad = 0;
  bad |= run<64, 128>();
  bad |= run<48, 128>();
  bad |= run<128, 16>();
  bad |= run<32, 64>();
  bad |= run<128, 128>();
  return bad;
}
