// Probe: kind::tf32 tcgen05 MMA with K-major and MN-major (no swizzle) smem operands.
// D[M=128 x N] = A[M x K] * B[N x K]^T, fp32 in memory, TF32 math, fp32 accumulate.
// K-major tile (R rows x K): 16-byte word (row r, k-chunk c = 4 elements) at c*R*16 + r*16
//   -> LBO = R*16 (k-chunks), SBO = 128 (8-row groups); one MMA = K 8 = 2 chunks.
// MN-major tile (R rows x K): core matrix = 8 k-rows x 16 B (4 consecutive rows r);
//   word (r-group g = r/4, k) at g*128 + (k%8)*16 + (k/8)*LBO, element r%4 inside
//   -> SBO = 128 (MN 16-byte groups), LBO = (R/4)*128 (8-deep k groups).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2306_16541_b200/csrc/tc_sm100.cuh"

using namespace fv;

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

// element (r, k) of an R x K operand -> float offset in smem
__host__ __device__ inline uint32_t off_kmaj(int R, int r, int k) { return (k / 4) * R * 4 + r * 4 + (k % 4); }
__host__ __device__ inline uint32_t off_mnmaj(int R, int r, int k) {
  return (r / 4) * 32 + (k % 8) * 4 + (k / 8) * (R / 4) * 32 + (r % 4);
}

template <int K, int N, int AMN, int BMN>
__global__ void probe(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) float sm[];
  float* sA = sm;
  float* sB = sm + 128 * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * K; i += 128) {
    const int r = i / K, k = i % K;
    sA[AMN ? off_mnmaj(128, r, k) : off_kmaj(128, r, k)] = A[i];
  }
  for (int i = t; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    sB[BMN ? off_mnmaj(N, r, k) : off_kmaj(N, r, k)] = B[i];
  }
  if (warp == 0) tc::tmem_alloc<128>(&tbase);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (t == 0) {
    const uint32_t id = idesc_tf32(128, N, AMN, BMN);
    for (int kk = 0; kk < K / 8; ++kk) {
      uint64_t ad, bd;
      if (AMN) ad = tc::make_desc(tc::smem_u32(sA) + kk * (128 / 4) * 128, (128 / 4) * 128, 128);
      else ad = tc::make_desc(tc::smem_u32(sA) + kk * 2 * 128 * 16, 128 * 16, 128);
      if (BMN) bd = tc::make_desc(tc::smem_u32(sB) + kk * (N / 4) * 128, (N / 4) * 128, 128);
      else bd = tc::make_desc(tc::smem_u32(sB) + kk * 2 * N * 16, N * 16, 128);
      mma_tf32(tbase, ad, bd, id, kk > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) D[t * N + c0 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<128>(tbase);
}

template <int K, int N, int AMN, int BMN>
int run() {
  std::vector<float> A(128 * K), B(N * K), D(128 * N);
  srand(K * 7 + N + AMN * 3 + BMN * 5);
  for (auto& x : A) x = (rand() % 2001 - 1000) / 1000.f;
  for (auto& x : B) x = (rand() % 2001 - 1000) / 1000.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t sm = (128 * K + N * K) * 4;
  cudaFuncSetAttribute(probe<K, N, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  probe<K, N, AMN, BMN><<<1, 128, sm>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("K=%d N=%d amn=%d bmn=%d CUDA error %s\n", K, N, AMN, BMN, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  const bool ok = maxerr < 2e-3 * maxref;
  printf("tf32 K=%d N=%d a_mn=%d b_mn=%d maxerr=%.3e (ref %.2f) %s\n", K, N, AMN, BMN, maxerr, maxref, ok ? "OK" : "FAIL");
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return ok ? 0 : 1;
}

int main() {
  int bad = 0;
  bad |= run<32, 64, 0, 0>();
  bad |= run<32, 64, 1, 0>();
  bad |= run<32, 64, 0, 1>();
  bad |= run<32, 64, 1, 1>();
  bad |= run<128, 128, 1, 1>();
  bad |= run<64, 16, 0, 1>();
  return bad;
}
