// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16) on one CTA per SM for
// operand modes that matter to the field kernels:
//   ss_none   A and B from smem, SWIZZLE_NONE K-chunk-major (the layout tc_sm100.cuh uses)
//   ss_128b   A and B from smem, SWIZZLE_128B descriptors (timing only, data is garbage)
//   ts_none   A from TMEM, B from smem SWIZZLE_NONE
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tc_rate.cu -o tc_rate
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2306_16541_b200/csrc/tc_sm100.cuh"

using namespace fv;

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = tc::make_desc(saddr, lbo, sbo);
  return d | ((uint64_t)layout << 61);
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
      :: "r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}

template <int MODE, int N>
__global__ void __launch_bounds__(128) k_rate(int reps, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x;
  for (int i = t; i < (128 * 128 * 2 + N * 128 * 2) / 16; i += 128)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3C003C00u, 0x3C003C00u, 0, 0);
  if ((t >> 5) == 0) tc::tmem_alloc<512>(&tmem_base);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tb = tmem_base;
  const uint32_t sA = tc::smem_u32(smem), sB = sA + 128 * 128 * 2;
  constexpr uint32_t idesc = MODE >= 3 ? ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                                          ((uint32_t)(128 >> 4) << 24))
                                       : tc::idesc_f16(128, N);
  if (t == 0) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 0) {
          tc::mma_f16(tb, tc::make_desc(sA + k * 4096, 2048, 128), tc::make_desc(sB + k * 2 * N * 16, N * 16, 128),
                      idesc, 1u);
        } else if (MODE == 1) {   // 128B swizzle: rows of 128 B, 8-row groups of 1024 B, +32 B per K=16
          const uint32_t kb = (k & 3) * 32 + (k >> 2) * 128 * 128;
          tc::mma_f16(tb, desc_sw(sA + kb, 16, 1024, 2), desc_sw(sB + (k & 3) * 32 + (k >> 2) * N * 128, 16, 1024, 2),
                      idesc, 1u);
        } else if (MODE == 2) {   // A in TMEM columns [256, 320): K=16 fp16 = 8 columns per MMA
          mma_ts(tb, tb + 256 + k * 8, tc::make_desc(sB + k * 2 * N * 16, N * 16, 128), idesc, 1u);
        } else if (MODE == 3) {   // kind::tf32, A in TMEM (K=8 = 8 columns), B SW128 K-major
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                       :: "r"(tb), "r"(tb + 256 + k * 8), "l"(desc_sw(sB + (k & 3) * 32 + (k >> 2) * N * 128, 16, 1024, 2)),
                          "r"(idesc), "r"(1u));
        } else {                  // kind::tf32, A and B SW128 K-major in smem
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                       :: "r"(tb), "l"(desc_sw(sA + (k & 3) * 32 + (k >> 2) * 128 * 128, 16, 1024, 2)),
                          "l"(desc_sw(sB + (k & 3) * 32 + (k >> 2) * N * 128, 16, 1024, 2)), "r"(idesc), "r"(1u));
        }
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if ((t >> 5) == 0) tc::tmem_free<512>(tb);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
         "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
         "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// One 256-thread team doing what a k_offset_tc layer does, serially: 9 MMAs (K=144,
// N=128) + commit, all wait, epilogue, proxy fence, named barrier.
// F bit0: TMEM ld + cvt, bit1: fence+barrier, bit2: STS of A, bit3: tcgen05.st of A,
// bit4: A operand from TMEM (ts mode).
__device__ __forceinline__ bool getenv_dummy() { return false; }

template <int F, int TEAMS = 1, int TW = 8>
__global__ void __launch_bounds__(1024) k_layer_lat(int reps, long long* cycles, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[TEAMS];
  __shared__ uint32_t tmem_base;
  constexpr int TT = TW * 32, NCOL = 128 / (TW / 4);   // threads per team, columns per warp
  const int warp = threadIdx.x >> 5, team = threadIdx.x / TT, t = threadIdx.x % TT;
  for (int i = threadIdx.x; i < (TEAMS + 1) * 128 * 144 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3C003C00u, 0x3C003C00u, 0, 0);
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  if (threadIdx.x == 0) { for (int i = 0; i < TEAMS; ++i) tc::mbar_init(&bars[i], 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  uint64_t& bar = bars[team];
  const uint32_t tb = tmem_base + team * (TEAMS > 2 ? 128 : 256);
  uint8_t* A = smem + (1 + team) * 128 * 144 * 2;
  const uint32_t sB = tc::smem_u32(smem), sA = tc::smem_u32(A);
  const int quad = warp & 3, half = (warp >> 2) % (TW / 4), row = quad * 32 + (t & 31);
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t taddr = tb + lane_off + half * NCOL;
  const uint32_t aaddr = tb + 128 + lane_off + half * NCOL / 2;   // A operand columns [128, 200) of the team
  constexpr uint32_t idesc = tc::idesc_f16(128, 128);
  uint32_t phase = 0, acc = 0;
  long long t0 = clock64();
  long long ph[4] = {0, 0, 0, 0}, tp = t0;   // bar, mma wait, ld+cvt, st
  for (int r = 0; r < reps; ++r) {
    if (F & 2) {
      if (F & 4) tc::fence_proxy_async();
      if (F & 8) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc::fence_before();
      asm volatile("bar.sync %0, %1;" :: "r"(1 + team), "r"(TT) : "memory");
    }
    { long long c = clock64(); ph[0] += c - tp; tp = c; }
    if (t == 0) {
      tc::fence_after();
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        if (F & 16)
          mma_ts(tb, tb + 128 + k * 8, tc::make_desc(sB + k * 4096, 2048, 128), idesc, k > 0);
        else
          tc::mma_f16(tb, tc::make_desc(sA + k * 4096, 2048, 128), tc::make_desc(sB + k * 4096, 2048, 128), idesc,
                      k > 0);
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, phase);
    phase ^= 1u;
    tc::fence_after();
    { long long c = clock64(); ph[1] += c - tp; tp = c; }
    if (F & 1) {
      float v[NCOL / 16][16];
#pragma unroll
      for (int g = 0; g < NCOL / 16; ++g) tc::tmem_ld16(taddr + g * 16, v[g]);
      tc::tmem_ld_wait();
      { long long c = clock64(); ph[2] += c - tp; tp = c; }
      uint32_t w[NCOL / 2];
#pragma unroll
      for (int j = 0; j < NCOL / 2; ++j) {
        uint32_t r;
        asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[j / 8][2 * (j % 8) + 1]), "f"(v[j / 8][2 * (j % 8)]));
        w[j] = r;
      }
      if (F & 4) {
#pragma unroll
        for (int g = 0; g < NCOL / 8; ++g)
          *reinterpret_cast<uint4*>(A + tc::op_off(128, row, (NCOL / 8) * half + g)) =
              make_uint4(w[4 * g], w[4 * g + 1], w[4 * g + 2], w[4 * g + 3]);
      } else if (F & 8) {
        if constexpr (NCOL == 64) {
          tmem_st32(aaddr, w);
        } else {
          uint32_t w2[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) w2[j] = w[j % (NCOL / 2)];
          tmem_st32(aaddr, w2);   // (timing stand-in: x16 would do)
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int j = 0; j < NCOL / 2; ++j) acc ^= w[j];
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (blockIdx.x == 0 && t == 0 && getenv_dummy())
    printf("   team %d warp-role %s: bar %.0f  mma-wait %.0f  ld %.0f  rest %.0f cyc/layer\n", team,
           t == 0 ? "issuer" : "half0 ", ph[0] / (double)reps, ph[1] / (double)reps, ph[2] / (double)reps,
           ((t1 - t0) - ph[0] - ph[1] - ph[2]) / (double)reps);
  if (acc == 0x12345678u) sink[t] = acc;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tb);
}

// Contention probe: warp 0 (thread 0) streams MMAs (N=128, K=16) for `reps` x 8; warps
// 4..7 stream tcgen05.ld x16 over columns [256, 384) in parallel (MODE bit0: MMAs on,
// bit1: loads on).  Reports cycles of each role.
template <int MODE>
__global__ void __launch_bounds__(256) k_contend(int reps, long long* cycles, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 2 * 128 * 128 * 2 / 16; i += 256)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3C003C00u, 0x3C003C00u, 0, 0);
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tb = tmem_base, sA = tc::smem_u32(smem), sB = sA + 128 * 128 * 2;
  constexpr uint32_t idesc = tc::idesc_f16(128, 128);
  uint32_t acc = 0;
  long long t0 = clock64(), t1 = t0;
  if ((MODE & 1) && t == 0) {
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        tc::mma_f16(tb, tc::make_desc(sA + k * 4096, 2048, 128), tc::make_desc(sB + k * 4096, 2048, 128), idesc, 1u);
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    t1 = clock64();
    cycles[blockIdx.x * 2] = t1 - t0;
  }
  if ((MODE & 2) && warp >= 4) {
    const uint32_t a = tb + 256 + ((uint32_t)((warp & 3) * 32) << 16);
    for (int r = 0; r < reps; ++r) {
      float v[4][16];
#pragma unroll
      for (int g = 0; g < 4; ++g) tc::tmem_ld16(a + ((r & 1) * 64) + g * 16, v[g]);
      tc::tmem_ld_wait();
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int j = 0; j < 16; ++j) acc ^= __float_as_uint(v[g][j]);
    }
    t1 = clock64();
    if (t == 128) cycles[blockIdx.x * 2 + 1] = t1 - t0;
  }
  if (acc == 0x12345678u) sink[t] = acc;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tb);
}

template <int MODE>
void run_contend(const char* name, long long* d_cyc, int nsm, int reps_mma, int reps_ld) {
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4096);
  const int smem = 2 * 128 * 128 * 2;
  cudaFuncSetAttribute(k_contend<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(d_cyc, 0, 512 * sizeof(long long));
  const int reps = MODE == 2 ? reps_ld : reps_mma;
  k_contend<MODE><<<nsm, 256, smem>>>(reps, d_cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, d_cyc, 2 * nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double m = 0, l = 0;
  for (int i = 0; i < nsm; ++i) { m += h[2 * i]; l += h[2 * i + 1]; }
  m /= nsm; l /= nsm;
  printf("contend %-10s mma %7.1f cyc/MMA   ld %6.1f B/cyc (4 warps, 16 KB per rep)  %s\n", name,
         m / (reps * 8.0), l > 0 ? reps * 16384.0 / l : 0.0, cudaGetErrorString(e));
}

template <int PHASES, int TEAMS = 1, int TW = 8>
void run_lat(const char* name, long long* d_cyc, int nsm) {
  const int reps = 2000, smem = (TEAMS + 1) * 128 * 144 * 2;
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(k_layer_lat<PHASES, TEAMS, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_layer_lat<PHASES, TEAMS, TW><<<nsm, TW * 32 * TEAMS, smem>>>(reps, d_cyc, sink);
  k_layer_lat<PHASES, TEAMS, TW><<<nsm, TW * 32 * TEAMS, smem>>>(reps, d_cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d_cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  printf("layer %-22s tw=%2d teams=%d %7.1f cyc/layer/team (MMA floor 576)  %s\n", name, TW, TEAMS, avg / nsm / reps,
         cudaGetErrorString(e));
}

template <int MODE, int N>
void run(const char* name, long long* d_cyc, int nsm) {
  const int reps = 2000;
  const int smem = 128 * 128 * 2 + N * 128 * 2;
  cudaFuncSetAttribute(k_rate<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_rate<MODE, N><<<nsm, 128, smem>>>(reps, d_cyc);
  k_rate<MODE, N><<<nsm, 128, smem>>>(reps, d_cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d_cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double per = avg / (reps * 8.0);
  printf("%-8s N=%3d  %7.1f cyc/MMA  (floor %d)  %s\n", name, N, per, 128 * N / 256, cudaGetErrorString(e));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 512 * sizeof(long long));
  if (getenv("LAYER")) {
    run_lat<16 + 11, 2, 8>("ts +ld/cvt+tmem.st", d, nsm);
    run_lat<16 + 11, 2, 16>("ts +ld/cvt+tmem.st", d, nsm);
    run_lat<16 + 2, 2, 8>("ts mma+wait+bar", d, nsm);
    run_lat<16 + 2, 2, 16>("ts mma+wait+bar", d, nsm);
    run_lat<16 + 3, 2, 8>("ts +ld/cvt (no st)", d, nsm);
    return 0;
  }
  if (getenv("CONTEND")) {
    run_contend<2>("ld only", d, nsm, 2000, 2000);
    run_contend<1>("mma only", d, nsm, 2000, 2000);
    run_contend<3>("mma+ld", d, nsm, 2000, 2000);
    return 0;
  }
  if (getenv("TF32")) {
    run<2, 128>("f16_ts", d, nsm);
    run<3, 128>("tf32_ts", d, nsm);
    run<4, 128>("tf32_ss", d, nsm);
    run<3, 144>("tf32_ts", d, nsm);
    run<3, 64>("tf32_ts", d, nsm);
    return 0;
  }
  if (getenv("FULL")) {
  run<0, 128>("ss_none", d, nsm);
  run<1, 128>("ss_128b", d, nsm);
  run<2, 128>("ts_none", d, nsm);
  run<0, 64>("ss_none", d, nsm);
  run<1, 64>("ss_128b", d, nsm);
  run<2, 64>("ts_none", d, nsm);
  run<0, 256>("ss_none", d, nsm);
  run<1, 256>("ss_128b", d, nsm);
  run<2, 256>("ts_none", d, nsm);
  run<0, 16>("ss_none", d, nsm);
  run<0, 32>("ss_none", d, nsm);
  }
  run_lat<7, 2, 8>("ss +ld/cvt+STS", d, nsm);
  run_lat<7, 3, 8>("ss +ld/cvt+STS", d, nsm);
  run_lat<7, 4, 4>("ss +ld/cvt+STS", d, nsm);
  run_lat<7, 3, 4>("ss +ld/cvt+STS", d, nsm);
  run_lat<2, 3, 8>("ss mma+wait+bar", d, nsm);
  run_lat<2, 4, 4>("ss mma+wait+bar", d, nsm);
  run_lat<16 + 11, 2, 8>("ts +ld/cvt+tmem.st", d, nsm);
  return 0;
}
