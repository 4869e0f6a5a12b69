// Microbenchmark: tcgen05.ld throughput (bytes/cycle/SM) vs warps and load shape.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tmem_ld_rate.cu -o tmem_ld_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2306_16541_b200/csrc/tc_sm100.cuh"
using namespace fv;

template <int NC>  // columns per tcgen05.ld (32x32b.xNC)
__device__ __forceinline__ void ld_cols(uint32_t taddr, uint32_t (&r)[NC]);
template <> __device__ __forceinline__ void ld_cols<16>(uint32_t a, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(a));
}
template <> __device__ __forceinline__ void ld_cols<32>(uint32_t a, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(a));
}

// W warps (multiple of 4); warp w reads lanes 32*(w%4).., columns [ (w/4)*span, +span ) in
// chunks of NC, INF chunks in flight before one wait.
template <int W, int NC, int INF>
__global__ void k_ld(int reps, long long* cyc, uint32_t* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tb);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const int groups = W / 4, span = 256 / groups;
  const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * span;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int c = 0; c < span; c += NC * INF) {
      uint32_t v[INF][NC];
#pragma unroll
      for (int i = 0; i < INF; ++i) ld_cols<NC>(base + c + i * NC, v[i]);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < INF; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc ^= v[i][j];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x1234567u) sink[threadIdx.x] = acc;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tb);
}

template <int W, int NC, int INF>
void run(int nsm, long long* d, uint32_t* sink) {
  const int reps = 1000;
  k_ld<W, NC, INF><<<nsm, W * 32>>>(reps, d, sink);
  k_ld<W, NC, INF><<<nsm, W * 32>>>(reps, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double bytes = (double)reps * 128 * 256 * 4;  // 128 lanes x 256 columns x 4 B per rep
  printf("warps %2d  x%-3d  in-flight %d : %6.1f B/cyc/SM  %s\n", W, NC, INF, bytes / avg, cudaGetErrorString(e));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 512 * sizeof(long long));
  cudaMalloc(&sink, 4096);
  run<4, 16, 1>(nsm, d, sink);
  run<4, 16, 4>(nsm, d, sink);
  run<4, 32, 2>(nsm, d, sink);
  run<4, 32, 4>(nsm, d, sink);
  run<8, 16, 4>(nsm, d, sink);
  run<8, 32, 2>(nsm, d, sink);
  run<16, 16, 4>(nsm, d, sink);
  run<16, 32, 2>(nsm, d, sink);
  return 0;
}
