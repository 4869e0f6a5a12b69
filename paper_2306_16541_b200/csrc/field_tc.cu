// Fused canonical field on 5th-gen tensor cores (sm_100a, tcgen05 + TMEM):
//   posenc(x_skel) -> offset MLP 39(48)->128->128->128->128->3(16)   (ResidualNet)
//   x_final = x_skel + x_res                                        (Eq 12)
//   hash-grid features (16 levels x 2)                              (builder-defined)
//   radiance MLP 32->64->64->4(16) + heads c = sigmoid, sigma = softplus(h-1)
//
// Design (the B200 restatement of the Fig-4 "fully fused" scheme, fu:1-14, fu:145-179):
//  * two persistent kernels, one CTA per SM each, with the MLP weights resident in shared
//    memory as fp16 UMMA B operands (loaded once per CTA):
//      k_offset_tc   posenc + residual MLP (112 KB of weights), pure tensor-core work,
//                    writes x_final in place of x_skel;
//      k_radiance_ws hash-grid gathers + radiance MLP + heads (19 KB of weights), so
//                    ~200 KB of the SM's L1 stays free for the table gathers (profiling
//                    the single fused kernel showed its 126-230 KB of smem starving L1);
//                    warp-specialised: 6 gather warpgroups feed TMEM feature slots to one
//                    MLP warpgroup (k_radiance_tc: every warpgroup gathers and runs its MLP);
//  * NWG warpgroups per CTA each own a 128-sample tile: thread t <-> sample row t <->
//    TMEM lane t.  Activations live in an fp16 A-operand buffer rewritten in place
//    layer after layer; accumulators live in TMEM;
//  * one elected thread per warpgroup issues the tcgen05.mma chain of a layer
//    (M = 128, N = 16..128, K = 16 per instruction) and commits to an mbarrier; the
//    128 threads run the epilogue (tcgen05.ld -> bias, ReLU -> fp16 -> smem) which is
//    the next layer's A operand.  Warpgroups interleave, so one WG's gathers/epilogue
//    overlap another WG's MMAs.
#include <cuda_runtime.h>
#include <cstdlib>
#include "fv_common.cuh"
#include "fv_internal.h"
#include "tc_sm100.cuh"

#ifndef FV_OFF_LEAD
#define FV_OFF_LEAD 2
#endif
#ifndef FV_RAD_NL
#define FV_RAD_NL 2   // hash levels per gather batch in k_radiance_tc
#endif
namespace fv {

// ---- weight pack layout (bytes) ------------------------------------------------------
// Every tensor-core layer except the offset MLP's last carries its bias inside the GEMM:
// K = activations + a 16-row bias group whose first two rows are the fp16 hi/lo split of
// the fp32 bias (b - hi(b) in fp16: ~2^-22 relative), multiplied by A columns = 1.0.
// Offset layer 0 uses the posenc pad columns 46/47 for the per-frame b0' (patched into the
// smem copy by the kernel).
constexpr uint32_t OF_KH = 144;                           // hidden-layer K (128 + bias group)
constexpr uint32_t PK_OFF0 = 0;                           // [128 x 48]
constexpr uint32_t PK_OFF1 = PK_OFF0 + 128 * 48 * 2;      // [128 x 144]
constexpr uint32_t PK_OFF2 = PK_OFF1 + 128 * OF_KH * 2;
constexpr uint32_t PK_OFF3 = PK_OFF2 + 128 * OF_KH * 2;
constexpr uint32_t PK_OFF4 = PK_OFF3 + 128 * OF_KH * 2;   // [16 x 128]
constexpr uint32_t RA_K0 = 48, RA_KH = 80;                // radiance K incl. the bias group
constexpr uint32_t PK_RAD0 = PK_OFF4 + 16 * 128 * 2;      // [64 x 48]  (32 features + bias group)
constexpr uint32_t PK_RAD1 = PK_RAD0 + 64 * RA_K0 * 2;    // [64 x 80]  (64 hidden + bias group)
constexpr uint32_t PK_RAD2 = PK_RAD1 + 64 * RA_KH * 2;    // [16 x 80]
constexpr uint32_t PK_WEND = PK_RAD2 + 16 * RA_KH * 2;    // 148480
// fp32 biases: off b1,b2,b3 (128 each), off b4 (16), rad b0 (64), rad b1 (64), rad b2 (16)
constexpr uint32_t BI_OFF1 = 0, BI_OFF2 = 128, BI_OFF3 = 256, BI_OFF4 = 384, BI_RAD0 = 400, BI_RAD1 = 464,
                   BI_RAD2 = 528, BI_END = 544;
constexpr uint32_t PK_BYTES = PK_WEND + BI_END * 4;       // 150656

struct PackLayer { uint32_t off; int N, K, n_true, k_true; };

// (in,out) fp32 weight -> B operand [N rows x K] fp16, K-chunk-major (tc_sm100.cuh).
__global__ void k_field_pack(fv_field f, uint8_t* __restrict__ pack) {
  const PackLayer L[8] = {
      {PK_OFF0, 128, 48, 128, 3 + 6 * f.pe_bands}, {PK_OFF1, 128, OF_KH, 128, 128}, {PK_OFF2, 128, OF_KH, 128, 128},
      {PK_OFF3, 128, OF_KH, 128, 128},            {PK_OFF4, 16, 128, 3, 128},       {PK_RAD0, 64, RA_K0, 64, 32},
      {PK_RAD1, 64, RA_KH, 64, 64},               {PK_RAD2, 16, RA_KH, 4, 64}};
  const float* W[8] = {f.d_off_w[0], f.d_off_w[1], f.d_off_w[2], f.d_off_w[3], f.d_off_w[4],
                       f.d_rad_w[0], f.d_rad_w[1], f.d_rad_w[2]};
  const int layer = blockIdx.y;
  const PackLayer pl = L[layer];
  const int words = pl.N * (pl.K / 8);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < words; e += gridDim.x * blockDim.x) {
    const int nrow = e % pl.N, c = e / pl.N;
    __half hv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = 8 * c + j;
      const float v = (k < pl.k_true && nrow < pl.n_true) ? W[layer][(int64_t)k * pl.n_true + nrow] : 0.f;
      hv[j] = __float2half_rn(v);
      if (layer != 0 && layer != 4 && k >= pl.k_true) {   // bias group: rows (hi, lo, 0 ...)
        const float b = nrow >= pl.n_true ? 0.f : (layer < 4 ? f.d_off_b[layer][nrow] : f.d_rad_b[layer - 5][nrow]);
        const __half hi = __float2half_rn(b);
        hv[j] = k == pl.k_true ? hi : (k == pl.k_true + 1 ? __float2half_rn(b - __half2float(hi)) : __float2half_rn(0.f));
      }
    }
    *reinterpret_cast<uint4*>(pack + pl.off + tc::op_off(pl.N, nrow, c)) = *reinterpret_cast<uint4*>(hv);
  }
  if (layer == 0 && blockIdx.x == 0) {
    float* bias = reinterpret_cast<float*>(pack + PK_WEND);
    for (int i = threadIdx.x; i < (int)BI_END; i += blockDim.x) {
      float v = 0.f;
      if (i < 384) v = f.d_off_b[1 + i / 128][i % 128];
      else if (i < 400) v = (i - 384) < 3 ? f.d_off_b[4][i - 384] : 0.f;
      else if (i < 464) v = f.d_rad_b[0][i - 400];
      else if (i < 528) v = f.d_rad_b[1][i - 464];
      else v = (i - 528) < 4 ? f.d_rad_b[2][i - 528] : 0.f;
      bias[i] = v;
    }
  }
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}

// fp16x2 helper: relu + round + pack in one conversion, (lo, hi) -> half2(max(lo,0), max(hi,0))
__device__ __forceinline__ uint32_t cvt_relu_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// ---- shared prologue: copy [w_begin, w_end) of the pack and `nbias` biases into smem
template <int NWG, uint32_t TCOLS>
__device__ __forceinline__ void tc_prologue(const uint8_t* pack, uint32_t w_begin, uint32_t w_end, uint32_t b_begin,
                                            uint32_t nbias, uint8_t* smem, float* sbias, uint64_t* bars,
                                            uint32_t* tmem_base) {
  const uint4* src = reinterpret_cast<const uint4*>(pack + w_begin);
  uint4* dst = reinterpret_cast<uint4*>(smem);
  for (int i = threadIdx.x; i < (int)((w_end - w_begin) / 16); i += blockDim.x) dst[i] = __ldg(src + i);
  const float* bsrc = reinterpret_cast<const float*>(pack + PK_WEND) + b_begin;
  for (int i = threadIdx.x; i < (int)nbias; i += blockDim.x) sbias[i] = bsrc[i];
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<TCOLS>(tmem_base);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NWG; ++i) tc::mbar_init(&bars[i], 1);
    tc::mbar_fence_init();
  }
}

__device__ __forceinline__ void tc_prologue_sync() {
  tc::fence_proxy_async();  // weight stores -> visible to the tensor-core proxy
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
}

#ifndef FV_OFF_PROF
#define FV_OFF_PROF 0
#endif
#if FV_OFF_PROF
__device__ long long g_off_prof[2 * 32 * 10];
#endif

// ---- k_offset_tc: xs (x_skel, L) -> out (x_final, L) ------------------------------------
// (Measured in round 2 and not kept: 16 worker warps + 1 MMA-issuer warp
// serving two tile slots through mbarriers, 2.91 -> 4.22 ms -- the issuing thread blocks
// ~850 cycles per 9-MMA batch and the two slots then serialise; the hidden-layer bias added
// in the epilogue instead of the K = 144 bias group, 2.91 -> 3.22 ms -- 3 fewer MMAs per
// tile, but the longer epilogue is on each team's critical chain.)
// Activations never touch shared memory: each layer's A operand lives in TMEM next to its
// accumulator (tcgen05.mma with A from TMEM), so the MMAs read only the weights from smem
// (64 of the SM's 128 B/cycle) and the epilogue is tcgen05.ld -> ReLU+fp16 cvt ->
// tcgen05.st.  (With A in smem, N = 128 MMAs use all of the smem bandwidth and the
// epilogue's stores stall them: tools/tc_rate.cu measures 2175 vs 1743 cycles per layer.)
// A team of 8 warps (two warpgroups) owns a 128-sample tile: warp w reads TMEM lane quadrant
// w%4 and accumulator columns [64*(w/4%2), +64).  Biases ride in the GEMM (pack layout).
// TMEM per team: D = columns [0, 128), A = [128, 200) (K = 144 fp16 pairs), the next
// tile's posenc [200, 224), the last layer's accumulator [224, 240); 2 teams.
constexpr uint32_t OF_W = PK_RAD0 - PK_OFF0;               // 126976
constexpr uint32_t OF_B4 = OF_W;                           // off b4: 16 floats
constexpr uint32_t OF_SMEM = OF_B4 + 64;
constexpr uint32_t OF_TA = 128;                            // A-operand column offset in a team
constexpr uint32_t OF_TPE = 200;                           // next tile's posenc (layer-0 A, 24 columns)
constexpr uint32_t OF_TD4 = 224;                           // layer-4 accumulator (16 columns)

// One layer of a team with A in TMEM: A stores done -> barrier -> one thread issues K/16
// MMAs (8 A columns each) + commit -> `overlap()` (independent work of the waiting
// threads) -> everyone waits.
struct NoOverlap { __device__ __forceinline__ void operator()() const {} };
// A batch of MMAs issued by `issue()` (one thread) with the same barrier/commit/wait protocol.
template <typename I>
__device__ __forceinline__ void layer_issue_ts(uint64_t* bar, uint32_t& phase, int t, int grp, I&& issue) {
  tc::tmem_st_wait();
  tc::fence_before();
  named_bar(1 + grp, 256);
  if (t == 0) {
    tc::fence_after();
    issue();
    tc::mma_commit(bar);
  }
  __syncwarp();
  tc::mbar_wait(bar, phase);
  phase ^= 1u;
  tc::fence_after();
}

template <int K, int N, int NTHR, typename F = NoOverlap>
__device__ __forceinline__ void layer_mma_ts(uint32_t tcol, const uint8_t* Wt, uint64_t* bar, uint32_t& phase,
                                             int t, int grp, F&& overlap = F()) {
  tc::tmem_st_wait();
  tc::fence_before();
  named_bar(1 + grp, NTHR);
  if (t == 0) {
    tc::fence_after();
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    const uint32_t b0 = tc::smem_u32(Wt);
#pragma unroll
    for (int k = 0; k < K / 16; ++k)
      tc::mma_f16_ts(tcol, tcol + OF_TA + k * 8, tc::make_desc(b0 + k * 2 * N * 16, N * 16, 128), idesc,
                     k > 0 ? 1u : 0u);
    tc::mma_commit(bar);
  }
  __syncwarp();
  overlap();
  tc::mbar_wait(bar, phase);
  phase ^= 1u;
  tc::fence_after();
}

// 64 accumulator columns -> ReLU -> fp16 pairs -> 32 A-operand columns
// WIDE: two 32-column loads (offset kernel) instead of four 16-column ones (the radiance
// kernel at 96 registers spills with the wide form)
template <bool WIDE = false>
__device__ __forceinline__ void epi_relu64_ts(uint32_t dsrc, uint32_t adst) {
  if constexpr (!WIDE) {
    float v[4][16];
#pragma unroll
    for (int g = 0; g < 4; ++g) tc::tmem_ld16(dsrc + g * 16, v[g]);
    tc::tmem_ld_wait();
    uint32_t w[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) w[j] = cvt_relu_h2(v[j >> 3][2 * (j & 7)], v[j >> 3][2 * (j & 7) + 1]);
    tc::tmem_st32(adst, w);
    return;
  }
  float v[2][32];
  tc::tmem_ld32(dsrc, v[0]);
  tc::tmem_ld32(dsrc + 32, v[1]);
  tc::tmem_ld_wait();
  uint32_t w[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) w[j] = cvt_relu_h2(v[j >> 4][2 * (j & 15)], v[j >> 4][2 * (j & 15) + 1]);
  tc::tmem_st32(adst, w);
}

template <int TEAMS>
__global__ void __launch_bounds__(TEAMS * 256, 1)
    k_offset_tc(fv_field f, const float4* __restrict__ xs, int64_t n, float eps_w, float4* __restrict__ out,
                float* __restrict__ xfinal, const int32_t* __restrict__ d_count) {
  static_assert(TEAMS == 1 || TEAMS == 2, "256 TMEM columns per team");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[TEAMS];
  __shared__ uint32_t tmem_base;
  __shared__ int lead_done;   // team 0's completed batches (counted up to FV_OFF_LEAD)
  if (threadIdx.x == 0) lead_done = 0;
  constexpr uint32_t TCOLS = TEAMS == 1 ? 256 : 512;
  float* sB4 = reinterpret_cast<float*>(smem + OF_B4);
  tc_prologue<TEAMS, TCOLS>(reinterpret_cast<const uint8_t*>(f.d_tc_pack), PK_OFF0, PK_RAD0, BI_OFF4, 16, smem,
                            sB4, bars, &tmem_base);
  // per-frame layer-0 bias b0' as weight rows K = 46 (hi) / 47 (lo) of the smem copy
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    const float b = f.d_off_b0_eff[i];
    const __half hi = __float2half_rn(b);
    __half* w = reinterpret_cast<__half*>(smem + PK_OFF0 + tc::op_off(128, i, 5));
    w[6] = hi;
    w[7] = __float2half_rn(b - __half2float(hi));
  }
  tc_prologue_sync();

  const int warp = threadIdx.x >> 5, team = threadIdx.x >> 8, tt = threadIdx.x & 255;
  const int quad = warp & 3, half = (warp >> 2) & 1;
  const int row = quad * 32 + (threadIdx.x & 31);
  const uint32_t tcol = tmem_base + team * 256;
  const uint32_t lane = (uint32_t)(quad * 32) << 16;
  const uint32_t dsrc = tcol + lane + half * 64;              // this thread's accumulator columns
  const uint32_t adst = tcol + lane + OF_TA + half * 32;      // ... and its A-operand columns
  if (half == 0) {   // constant bias group of the hidden layers: A columns 64..71 = (1, 1), 0, ...
    const uint32_t ones[8] = {0x3C003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    tc::tmem_st8(tcol + lane + OF_TA + 64, ones);
  }
  uint64_t* bar = &bars[team];
  uint32_t phase = 0;
  if (d_count) n = min((int64_t)*d_count, n);   // compacted foreground stream of the march
  const int64_t ntiles = (n + 127) / 128;
  const int64_t tstep = (int64_t)gridDim.x * TEAMS;
  int64_t tile = (int64_t)blockIdx.x * TEAMS + team;
  // posenc of one sample -> this thread's 12 A-operand words (columns [12*half, +12) of the
  // 24 holding 39 values, zero pad, ones at k = 46/47): sin/cos(pi x) once per coordinate,
  // higher bands by double-angle recurrences (error 2^k ulp << fp16 resolution)
  // posenc of one sample -> this thread's 12 A-operand words: the 48 fp16 columns hold the 39
  // values, zero pad and ones at k = 46/47; warpgroup half 0 owns columns [0, 24) (raw xyz,
  // bands 0-2, band 3 sine), half 1 columns [24, 48) (band 3 cosine, bands 4-5, pad, ones),
  // so each half computes only its own 24 values: sin/cos(pi 2^k0 x) once per coordinate
  // (k0 = 0 or 3), the other bands by double-angle recurrences (error 2^k ulp << fp16).
  auto posenc12 = [&](const float4 v, int64_t s, uint32_t (&w)[12]) {
    const bool fg = s < n && v.w > eps_w;
    const float xx[3] = {fg ? v.x : 0.f, fg ? v.y : 0.f, fg ? v.z : 0.f};
    __half pe[24];
    if (half == 0) {
      pe[0] = __float2half_rn(xx[0]); pe[1] = __float2half_rn(xx[1]); pe[2] = __float2half_rn(xx[2]);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float sv, cv;
        sincospif(xx[j], &sv, &cv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float wk = k < f.pe_bands ? f.pe_w[k] : 0.f;
          pe[3 + 6 * k + j] = __float2half_rn(wk * sv);                 // k = 3: column 21 + j
          if (k < 3) pe[6 + 6 * k + j] = __float2half_rn(wk * cv);
          const float s2 = 2.f * sv * cv, c2 = (cv - sv) * (cv + sv);
          sv = s2; cv = c2;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float sv, cv;
        sincospif(8.f * xx[j], &sv, &cv);                                // band 3: 2^3 pi x
#pragma unroll
        for (int k = 3; k < 6; ++k) {
          const float wk = k < f.pe_bands ? f.pe_w[k] : 0.f;
          if (k > 3) pe[3 + 6 * k + j - 24] = __float2half_rn(wk * sv);
          pe[6 + 6 * k + j - 24] = __float2half_rn(wk * cv);             // k = 3: column 24 + j
          const float s2 = 2.f * sv * cv, c2 = (cv - sv) * (cv + sv);
          sv = s2; cv = c2;
        }
      }
#pragma unroll
      for (int j = 39 - 24; j < 46 - 24; ++j) pe[j] = __float2half_rn(0.f);
      pe[46 - 24] = pe[47 - 24] = __float2half_rn(1.f);
    }
    const uint32_t* pw = reinterpret_cast<const uint32_t*>(pe);
#pragma unroll
    for (int i = 0; i < 12; ++i) w[i] = pw[i];
  };
  // Software pipeline per team:
  //  * the input is loaded two tiles ahead and the next tile's posenc is computed (and
  //    stored to its own TMEM block, OF_TPE) while this tile's layer-1 MMAs run;
  //  * the last layer (N = 16, accumulator block OF_TD4) of tile t-1 and layer 0 of tile t
  //    are independent, so they go out as ONE batch with one commit: 4 MMA round trips per
  //    tile instead of 5.
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 vcur = tile * 128 + row < n ? xs[tile * 128 + row] : zero4;
  float4 vnext = (tile + tstep) * 128 + row < n ? xs[(tile + tstep) * 128 + row] : zero4;
  const uint32_t pe_dst = tcol + lane + OF_TPE + half * 12;
  {
    uint32_t pw[12];
    posenc12(vcur, tile * 128 + row, pw);
    tc::tmem_st8(pe_dst, pw);
    tc::tmem_st4(pe_dst + 8, pw + 8);
  }
  const auto emit = [&](const float4 v, int64_t s) {   // x_final = x_skel + x_res of one sample
    float o[16];
    tc::tmem_ld16(tcol + lane + OF_TD4, o);
    tc::tmem_ld_wait();
    if (s < n) {
      const bool fg = v.w > eps_w;
      const float y0 = v.x + (o[0] + sB4[0]), y1 = v.y + (o[1] + sB4[1]), y2 = v.z + (o[2] + sB4[2]);
      out[s] = fg ? make_float4(y0, y1, y2, v.w) : make_float4(0.f, 0.f, 0.f, v.w);
      if (xfinal) {
        xfinal[3 * s] = fg ? y0 : 0.f; xfinal[3 * s + 1] = fg ? y1 : 0.f; xfinal[3 * s + 2] = fg ? y2 : 0.f;
      }
    }
  };
  const uint32_t b4 = tc::smem_u32(smem + PK_OFF4), b0 = tc::smem_u32(smem + PK_OFF0);
  float4 vprev = zero4;
  int64_t sprev = -1;
  const auto lead = [&] {
    if (TEAMS == 2 && team == 0 && tt == 0) {
      volatile int* p = &lead_done;
      if (*p < FV_OFF_LEAD) *p = *p + 1;
    }
  };
#if FV_OFF_PROF
  // timeline probe (alt builds only): CTA 0, thread 0 of each team records clock64 at 10
  // points per tile for its first 32 tiles -> g_off_prof[team][tile][10]
  int ptile = 0;
  const bool prec = blockIdx.x == 0 && tt == 0;
  auto P = [&](int k) { if (prec && ptile < 32) g_off_prof[(team * 32 + ptile) * 10 + k] = clock64(); };
#else
  auto P = [&](int) {};
#endif
  for (; tile < ntiles; tile += tstep) {
    const int64_t s = tile * 128 + row;
    const float4 v = vcur;
    P(0);
    // [layer 4 of the previous tile] + layer 0 of this tile, one commit
    layer_issue_ts(bar, phase, tt, team, [&] {
      // De-phase the two teams: team 1 starts once team 0 has FV_OFF_LEAD batches done, so
      // one team's epilogues run under the other's MMAs instead of both teams' at once.
      if (TEAMS == 2 && team == 1 && sprev < 0)
        while (*reinterpret_cast<volatile int*>(&lead_done) < FV_OFF_LEAD) {}
      if (sprev >= 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc::mma_f16_ts(tcol + OF_TD4, tcol + OF_TA + k * 8, tc::make_desc(b4 + k * 2 * 16 * 16, 16 * 16, 128),
                         tc::idesc_f16(128, 16), k > 0 ? 1u : 0u);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k)
        tc::mma_f16_ts(tcol, tcol + OF_TPE + k * 8, tc::make_desc(b0 + k * 2 * 128 * 16, 128 * 16, 128),
                       tc::idesc_f16(128, 128), k > 0 ? 1u : 0u);
    });
    P(1);
    lead();
    P(2);
    epi_relu64_ts<true>(dsrc, adst);
    P(3);
    // Work hidden under the MMAs of layers 1-3 (which write D, not D4 or the posenc block):
    // the next tile's posenc (each warpgroup half computes its own 24 columns) and input,
    // and the previous tile's x_final (FV_OFF_SCHED picks the windows).  The next B0
    // batch's tmem_st_wait + team barrier orders the posenc stores before its layer-0 MMAs.
#ifndef FV_OFF_SCHED
#define FV_OFF_SCHED 5
#endif
    const int64_t s1 = s + tstep * 128, s2 = s1 + tstep * 128;
    const auto posenc_next = [&] {
      uint32_t pw[12];
      posenc12(vnext, s1, pw);
      tc::tmem_st8(pe_dst, pw);
      tc::tmem_st4(pe_dst + 8, pw + 8);
    };
    constexpr int SCHED = FV_OFF_SCHED;
    // window of: posenc half 0, posenc half 1, input advance, emit
    constexpr int W_PE0 = SCHED == 4 ? 2 : 1, W_PE1 = 1, W_IN = SCHED == 4 ? 2 : 1, W_EMIT = SCHED == 2 ? 2 : 3;
    const auto window = [&](int wdx) {
      if (wdx == W_PE0 && half == 0) posenc_next();
      if (wdx == W_PE1 && half == 1) posenc_next();
      if (wdx == W_IN) { vcur = vnext; vnext = s2 < n ? xs[s2] : zero4; }
      if (wdx == W_EMIT && sprev >= 0 && half == 0) emit(vprev, sprev);
    };
    layer_mma_ts<OF_KH, 128, 256>(tcol, smem + PK_OFF1, bar, phase, tt, team, [&] { window(1); });
    P(4);
    lead();
    epi_relu64_ts<true>(dsrc, adst);
    P(5);
    layer_mma_ts<OF_KH, 128, 256>(tcol, smem + PK_OFF2, bar, phase, tt, team, [&] { window(2); });
    P(6);
    lead();
    epi_relu64_ts<true>(dsrc, adst);
    P(7);
    layer_mma_ts<OF_KH, 128, 256>(tcol, smem + PK_OFF3, bar, phase, tt, team, [&] { window(3); });
    P(8);
    lead();
    epi_relu64_ts<true>(dsrc, adst);
    P(9);
#if FV_OFF_PROF
    ++ptile;
#endif
    const bool fg = s < n && v.w > eps_w;
    vprev = fg ? v : make_float4(0.f, 0.f, 0.f, v.w);
    sprev = s;
  }
  if (sprev >= 0) {   // layer 4 of the team's last tile
    layer_issue_ts(bar, phase, tt, team, [&] {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        tc::mma_f16_ts(tcol + OF_TD4, tcol + OF_TA + k * 8, tc::make_desc(b4 + k * 2 * 16 * 16, 16 * 16, 128),
                       tc::idesc_f16(128, 16), k > 0 ? 1u : 0u);
    });
    if (half == 0) emit(vprev, sprev);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<TCOLS>(tmem_base);
}

// ---- k_radiance_tc: (x_final, L) -> (c, sigma) ----------------------------------------
// Hash features and hidden activations live in TMEM (tcgen05.st; MMAs take A from TMEM)
// and the biases ride in the GEMM, so the only shared-memory traffic is the tensor core
// reading the 17 KB of weights: the L1 data pipe is left to the table gathers, which
// bound this kernel.  (The smem-A version spent ~25% of the pipe's wavefronts on the
// MLP's STS/LDS.)  TMEM per warpgroup: D = columns [0, 64), A = [64, 96): features
// (words 0..15) or hidden activations (words 0..31); the bias group (8 columns = (1, 1),
// 0, ...) that every layer's last K step reads is one block at column 480 shared by all
// warpgroups (5 x 96 + 8 <= 512; with <= 4 warpgroups each keeps its own at A + 32).
// 5 warpgroups gathering 2 levels per batch beat 4 gathering 4 (more warps, 96 registers).
constexpr uint32_t RA_SMEM = PK_WEND - PK_RAD0;          // 19456 B of weights
constexpr uint32_t RA_TA = 64;                           // A-operand column offset
constexpr uint32_t RA_TCOLS_WG = 128;                    // TMEM columns per warpgroup (104 used)

// K_ACT activations (K_ACT/16 steps from A words 0..) + the bias step (A words 32..39).
template <int K_ACT, int N>
__device__ __forceinline__ void layer_mma_rad(uint32_t tcol, const uint8_t* Wt, uint64_t* bar, uint32_t& phase,
                                              int t, int wg, uint32_t bias_a) {
  tc::tmem_st_wait();
  tc::fence_before();
  named_bar(1 + wg, 128);
  if (t == 0) {
    tc::fence_after();
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    const uint32_t b0 = tc::smem_u32(Wt);
#pragma unroll
    for (int k = 0; k <= K_ACT / 16; ++k) {
      const uint32_t a = k < K_ACT / 16 ? tcol + RA_TA + k * 8 : bias_a;
      tc::mma_f16_ts(tcol, a, tc::make_desc(b0 + k * 2 * N * 16, N * 16, 128), idesc, k > 0 ? 1u : 0u);
    }
    tc::mma_commit(bar);
  }
  __syncwarp();
  tc::mbar_wait(bar, phase);
  phase ^= 1u;
  tc::fence_after();
}

template <int NWG>
__global__ void __launch_bounds__(NWG * 128, 1)
    k_radiance_tc(fv_field f, fv_hash h, const float4* __restrict__ xf, int64_t n, float eps_w,
                  float4* __restrict__ rgbs, const int32_t* __restrict__ d_count, const int32_t* __restrict__ idx) {
  // <= 4 warpgroups: 128 columns each (D 64 | A 32 | own bias group 8); 5: 96 each (D | A)
  // and one bias group shared by all at column 480 (it is the same constant in every row)
  constexpr uint32_t WGC = NWG <= 4 ? RA_TCOLS_WG : 96;
  static_assert(NWG * WGC + (NWG <= 4 ? 0 : 8) <= 512, "TMEM");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[NWG];
  __shared__ uint32_t tmem_base;
  constexpr uint32_t TCOLS = NWG * RA_TCOLS_WG <= 256 ? 256 : 512;
  tc_prologue<NWG, TCOLS>(reinterpret_cast<const uint8_t*>(f.d_tc_pack), PK_RAD0, PK_WEND, 0, 0, smem, nullptr,
                          bars, &tmem_base);
  tc_prologue_sync();

  const int warp = threadIdx.x >> 5, wg = threadIdx.x >> 7, t = threadIdx.x & 127;
  const uint32_t tcol = tmem_base + wg * WGC;
  const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t trow = tcol + lane;              // this thread's accumulator row
  const uint32_t arow = tcol + lane + RA_TA;      // ... and its A-operand row
  const uint32_t bias_a = NWG <= 4 ? tcol + RA_TA + 32 : tmem_base + 480;
  if (NWG <= 4 || wg == 0) {
    const uint32_t ones[8] = {0x3C003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    tc::tmem_st8(NWG <= 4 ? arow + 32 : tmem_base + lane + 480, ones);
  }
  if (NWG > 4) {   // the shared bias group is written by warpgroup 0, read by every MMA
    tc::tmem_st_wait();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  uint64_t* bar = &bars[wg];
  uint32_t phase = 0;
#if FV_DEBUG
  const int64_t n_slots = n;              // the full layout's size: every scatter slot is below it
#endif
  if (d_count) n = min((int64_t)*d_count, n);
  const int64_t ntiles = (n + 127) / 128;
  const int64_t tstep = (int64_t)gridDim.x * NWG;
  int64_t tile = (int64_t)blockIdx.x * NWG + wg;
  float4 vnext = make_float4(0.f, 0.f, 0.f, 0.f);
  int32_t onext = 0;                      // output slot (scatter index of the compacted stream)
  if (tile * 128 + t < n) {
    vnext = xf[tile * 128 + t];
    onext = idx ? idx[tile * 128 + t] : (int32_t)(tile * 128 + t);
  }
  for (; tile < ntiles; tile += tstep) {
    const int64_t s = tile * 128 + t;
    const float4 v = vnext;
    const int64_t o_s = idx ? (int64_t)onext : s;
    if (s + tstep * 128 < n) {            // prefetch the warpgroup's next tile (input + scatter slot)
      vnext = xf[s + tstep * 128];
      if (idx) onext = idx[s + tstep * 128];
    }
    const bool fg = s < n && v.w > eps_w;
    {  // hash-grid features -> A words 0..15 (NL levels = NL words per batch)
      float xn[3]; bool msk[3];
      hash_norm(h, fg ? v.x : 0.f, fg ? v.y : 0.f, fg ? v.z : 0.f, xn, msk);
      constexpr int NL = FV_RAD_NL;       // levels whose 8 NL gathers per lane are in flight together
#pragma unroll 1
      for (int c = 0; c < 16 / NL; ++c) {
        float2 fv[NL];
        hash_levels_paired<NL>(h, NL * c, xn, fv);
        uint32_t w[NL];
#pragma unroll
        for (int q = 0; q < NL; ++q) w[q] = tc::pack_half2(fg ? fv[q].x : 0.f, fg ? fv[q].y : 0.f);
        if constexpr (NL == 1) tc::tmem_st1(arow + NL * c, w);
        else if constexpr (NL == 2) tc::tmem_st2(arow + NL * c, w);
        else if constexpr (NL == 4) tc::tmem_st4(arow + NL * c, w);
        else tc::tmem_st8(arow + NL * c, w);
      }
    }
    layer_mma_rad<32, 64>(tcol, smem + (PK_RAD0 - PK_RAD0), bar, phase, t, wg, bias_a);
    epi_relu64_ts(trow, arow);
    layer_mma_rad<64, 64>(tcol, smem + (PK_RAD1 - PK_RAD0), bar, phase, t, wg, bias_a);
    epi_relu64_ts(trow, arow);
    layer_mma_rad<64, 16>(tcol, smem + (PK_RAD2 - PK_RAD0), bar, phase, t, wg, bias_a);
    float o[16];
    tc::tmem_ld16(trow, o);
    tc::tmem_ld_wait();
    if (s < n) {
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      if (fg) r = make_float4(sigmoid_fast(o[0]), sigmoid_fast(o[1]), sigmoid_fast(o[2]), softplus_fast(o[3] - 1.f));
      FV_ASSERT(o_s >= 0 && o_s < n_slots);
      rgbs[o_s] = r;                         // scatter back to the full sample layout
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<TCOLS>(tmem_base);
}

// ---- k_radiance_ws: warp-specialised variant (FV_RAD_WS) -------------------------------
// NG gather warpgroups only gather: each writes its tile's 32 fp16 features into one of two
// TMEM slots (16 columns each) and arrives on the slot's `full` barrier; ONE MLP warpgroup
// runs the radiance MLP of every tile (layer-0 A = the slot, commit -> the slot's `empty`
// barrier) and scatters (c, sigma).  The gathering warps never wait on an MMA.
// TMEM: MLP D [0, 64), hidden A [64, 96), bias ones [96, 104); slots from column 128.
// bounded mbarrier wait: traps (with a message) instead of hanging if a phase never completes
__device__ __forceinline__ void mbar_wait_guard(uint64_t* bar, uint32_t parity) {
  const uint32_t a = tc::smem_u32(bar);
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, P1;\n\t}\n" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    if (it > (1u << 26)) {   // a phase that never completes is a bug: report and fail, do not hang
      printf("k_radiance_ws: mbarrier wait timed out (block %d thread %d)\n", (int)blockIdx.x, (int)threadIdx.x);
      __trap();
    }
  }
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(tc::smem_u32(bar)) : "memory");
}

#ifndef FV_RAD_WS_SLOTS
#define FV_RAD_WS_SLOTS 2   // feature slots per gather warpgroup
#endif

template <int NG>
__global__ void __launch_bounds__((NG + 1) * 128, 1)
    k_radiance_ws(fv_field f, fv_hash h, const float4* __restrict__ xf, int64_t n, float eps_w,
                  float4* __restrict__ rgbs, const int32_t* __restrict__ d_count, const int32_t* __restrict__ idx) {
  constexpr int SL = FV_RAD_WS_SLOTS;
  static_assert(128 + NG * SL * 16 <= 512, "TMEM");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[1];
  __shared__ uint64_t full[NG][SL], empty[NG][SL];
  __shared__ int32_t meta[NG][SL][128];     // scatter slot (>= 0 fg, <= -2 background at -(m+2), -1 none)
  __shared__ int sel[2];
  __shared__ uint32_t tmem_base;
  tc_prologue<1, 512>(reinterpret_cast<const uint8_t*>(f.d_tc_pack), PK_RAD0, PK_WEND, 0, 0, smem, nullptr, bars,
                      &tmem_base);
  if (threadIdx.x == 0) {
    for (int g = 0; g < NG; ++g)
      for (int k = 0; k < SL; ++k) { tc::mbar_init(&full[g][k], 128); tc::mbar_init(&empty[g][k], 1); }
    tc::mbar_fence_init();
  }
  tc_prologue_sync();
  const int warp = threadIdx.x >> 5, wg = threadIdx.x >> 7, t = threadIdx.x & 127;
  const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t tb = tmem_base;
  if (d_count) n = min((int64_t)*d_count, n);
  const int64_t ntiles = (n + 127) / 128;
  const int64_t tstep = (int64_t)gridDim.x * NG;
  if (wg < NG) {
    // ------------------------------------------------------------ gather warpgroup wg
    const uint32_t slot0 = tb + lane + 128 + (uint32_t)(wg * SL) * 16;
    int64_t tile = (int64_t)blockIdx.x * NG + wg;
    float4 vnext = make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t onext = 0;
    if (tile * 128 + t < n) {
      vnext = xf[tile * 128 + t];
      onext = idx ? idx[tile * 128 + t] : (int32_t)(tile * 128 + t);
    }
    for (int i = 0; tile < ntiles; tile += tstep, ++i) {
      const int k = i % SL;
      const int64_t s = tile * 128 + t;
      const float4 v = vnext;
      const int32_t o_s = idx ? onext : (int32_t)s;
      if (s + tstep * 128 < n) {
        vnext = xf[s + tstep * 128];
        if (idx) onext = idx[s + tstep * 128];
      }
      const bool fg = s < n && v.w > eps_w;
      float xn[3]; bool msk[3];
      hash_norm(h, fg ? v.x : 0.f, fg ? v.y : 0.f, fg ? v.z : 0.f, xn, msk);
      if (i >= SL) mbar_wait_guard(&empty[wg][k], ((i / SL) - 1) & 1);   // the MLP took this slot's last tile
      tc::fence_after();
      const uint32_t slot = slot0 + (uint32_t)k * 16;
      constexpr int NL = FV_RAD_NL;
#pragma unroll 1
      for (int c = 0; c < 16 / NL; ++c) {
        float2 fv[NL];
        hash_levels_paired<NL>(h, NL * c, xn, fv);
        uint32_t w[NL];
#pragma unroll
        for (int q = 0; q < NL; ++q) w[q] = tc::pack_half2(fg ? fv[q].x : 0.f, fg ? fv[q].y : 0.f);
        if constexpr (NL == 1) tc::tmem_st1(slot + NL * c, w);
        else if constexpr (NL == 2) tc::tmem_st2(slot + NL * c, w);
        else if constexpr (NL == 4) tc::tmem_st4(slot + NL * c, w);
        else tc::tmem_st8(slot + NL * c, w);
      }
      meta[wg][k][t] = s < n ? (fg ? o_s : -o_s - 2) : -1;
      tc::tmem_st_wait();
      tc::fence_before();
      mbar_arrive_cta(&full[wg][k]);
    }
  } else {
    // ------------------------------------------------------------ MLP warpgroup
    const uint32_t trow = tb + lane, arow = tb + lane + RA_TA, bias_a = tb + 96;
    {
      const uint32_t ones[8] = {0x3C003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      tc::tmem_st8(tb + lane + 96, ones);
      tc::tmem_st_wait();
    }
    uint64_t* bar = &bars[0];
    uint32_t phase = 0;
    const auto mlp_layer = [&](int K_ACT16, uint32_t a_act, const uint8_t* Wt, int N) {
      tc::fence_before();
      named_bar(1, 128);
      if (t == 0) {
        tc::fence_after();
        const uint32_t idesc = tc::idesc_f16(128, N);
        const uint32_t b0 = tc::smem_u32(Wt);
        for (int kk = 0; kk <= K_ACT16; ++kk) {
          const uint32_t a = kk < K_ACT16 ? a_act + kk * 8 : bias_a;
          tc::mma_f16_ts(tb, a, tc::make_desc(b0 + kk * 2 * N * 16, N * 16, 128), idesc, kk > 0 ? 1u : 0u);
        }
      }
    };
    const auto epi = [&] {   // D (64 columns) -> ReLU -> fp16 -> hidden A, in 16-column pieces
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float v[16];
        tc::tmem_ld16(trow + g * 16, v);
        tc::tmem_ld_wait();
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = cvt_relu_h2(v[2 * j], v[2 * j + 1]);
        tc::tmem_st8(arow + g * 8, w);
      }
      tc::tmem_st_wait();
    };
    const auto process = [&](int g, int i) {
      const int k = i % SL;
      mbar_wait_guard(&full[g][k], (i / SL) & 1);
      tc::fence_after();
      const int32_t m = meta[g][k][t];
      const uint32_t slot = tb + 128 + (uint32_t)(g * SL + k) * 16;
      mlp_layer(2, slot, smem + (PK_RAD0 - PK_RAD0), 64);
      if (t == 0) { tc::mma_commit(&empty[g][k]); tc::mma_commit(bar); }
      __syncwarp();
      mbar_wait_guard(bar, phase); phase ^= 1u;
      tc::fence_after();
      epi();
      mlp_layer(4, tb + RA_TA, smem + (PK_RAD1 - PK_RAD0), 64);
      if (t == 0) tc::mma_commit(bar);
      __syncwarp();
      mbar_wait_guard(bar, phase); phase ^= 1u;
      tc::fence_after();
      epi();
      mlp_layer(4, tb + RA_TA, smem + (PK_RAD2 - PK_RAD0), 16);
      if (t == 0) tc::mma_commit(bar);
      __syncwarp();
      mbar_wait_guard(bar, phase); phase ^= 1u;
      tc::fence_after();
      float o[16];
      tc::tmem_ld16(trow, o);
      tc::tmem_ld_wait();
      if (m != -1) {
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m >= 0) r = make_float4(sigmoid_fast(o[0]), sigmoid_fast(o[1]), sigmoid_fast(o[2]), softplus_fast(o[3] - 1.f));
        rgbs[m >= 0 ? m : -m - 2] = r;
      }
    };
    for (int i = 0;; ++i) {
      bool any = false;
      for (int g = 0; g < NG; ++g) {
        const int64_t tile = (int64_t)blockIdx.x * NG + g + (int64_t)i * tstep;
        if (tile >= ntiles) continue;
        any = true;
        process(g, i);
      }
      if (!any) break;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem_base);
}

// Tuned configuration (round-1 sweeps on B200, SS4): residual MLP with 2
// 8-warp teams per SM (all 512 TMEM columns; 124 KB of weights in smem), hash+radiance
// with 4 warpgroups and 4-level batched gathers.
#ifndef FV_RAD_NWG
#define FV_RAD_NWG 5   // warpgroups per CTA in k_radiance_tc (5 x 96 TMEM columns + shared bias group)
#endif
constexpr int OFF_TEAMS = 2, RAD_NWG = FV_RAD_NWG;

static int sm_count() {
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  return n_sm;
}

static void launch_offset(const fv_field* f, const float4* xs, int64_t n, float eps_w, float4* out, float* xfinal,
                          const int32_t* d_count, cudaStream_t st) {
  const size_t smem = OF_SMEM;
  cudaFuncSetAttribute(k_offset_tc<OFF_TEAMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = (n + 127) / 128;
  const int grid = (int)std::min<int64_t>((ntiles + OFF_TEAMS - 1) / OFF_TEAMS, sm_count());
  k_offset_tc<OFF_TEAMS><<<grid, OFF_TEAMS * 256, smem, st>>>(*f, xs, n, eps_w, out, xfinal, d_count);
}

#ifndef FV_RAD_WS
#define FV_RAD_WS 6   // k_radiance_ws with 6 gather warpgroups + 1 MLP warpgroup (0: k_radiance_tc)
#endif
static void launch_radiance(const fv_field* f, const fv_hash* h, const float4* xf, int64_t n, float eps_w,
                            float4* rgbs, const int32_t* d_count, const int32_t* idx, cudaStream_t st) {
#if FV_RAD_WS
  {
    constexpr int NG = FV_RAD_WS;
    cudaFuncSetAttribute(k_radiance_ws<NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RA_SMEM);
    const int64_t ntiles = (n + 127) / 128;
    const int grid = (int)std::min<int64_t>((ntiles + NG - 1) / NG, sm_count());
    k_radiance_ws<NG><<<grid, (NG + 1) * 128, RA_SMEM, st>>>(*f, *h, xf, n, eps_w, rgbs, d_count, idx);
    return;
  }
#endif
  const size_t smem = RA_SMEM;
  cudaFuncSetAttribute(k_radiance_tc<RAD_NWG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = (n + 127) / 128;
  const int grid = (int)std::min<int64_t>((ntiles + RAD_NWG - 1) / RAD_NWG, sm_count());
  k_radiance_tc<RAD_NWG><<<grid, RAD_NWG * 128, smem, st>>>(*f, *h, xf, n, eps_w, rgbs, d_count, idx);
}

// x_skel -> x_final -> (c, sigma).  Dense form (d_count == NULL): x_final goes to rgbs as
// scratch and the radiance kernel overwrites it in place.  Compacted form (render path):
// xs is the march's foreground stream of *d_count samples (<= n), x_final overwrites it in
// place and (c, sigma) are scattered to rgbs[idx[j]] in the full sample layout.
int32_t field_fwd_tc(const fv_field* f, const fv_hash* h, const float4* xs, int64_t n, float eps_w, float4* rgbs,
                     float* xfinal, cudaStream_t st, const int32_t* d_count, const int32_t* idx,
                     cudaEvent_t mid_event) {
  if (!f->d_tc_pack) return set_error(FV_EDIM, "field tc: d_tc_pack is NULL (call fv_field_pack)");
  if (!f->d_off_b0_eff) return set_error(FV_EDIM, "field tc: d_off_b0_eff is NULL (call fv_offset_bias)");
  if (h->n_levels * h->n_feat != 32 || f->pe_bands > 6)
    return set_error(FV_EUNSUPPORTED, "field tc: needs 16x2 hash features and <= 6 PE bands");
  if (n == 0) return FV_OK;
  const float4* src = xs;
  if (f->offset_enabled) {
    float4* dst = d_count ? const_cast<float4*>(xs) : rgbs;
    launch_offset(f, xs, n, eps_w, dst, xfinal, d_count, st);
    if (int32_t e = check_launch("k_offset_tc")) return e;
    src = dst;
  } else if (xfinal) {
    return set_error(FV_EUNSUPPORTED, "field tc: x_final output needs the residual stage enabled");
  }
  if (mid_event) cudaEventRecord(mid_event, st);
  launch_radiance(f, h, src, n, eps_w, rgbs, d_count, idx, st);
  return check_launch("k_radiance_tc");
}

// Verification twin of k_radiance_tc's gather stage: the same hash_norm +
// hash_levels_paired<FV_RAD_NL> calls on canonical points x (n,3), returning every corner's
// global table index idx (n, L, 8) (corner a*4 + b*2 + c) and the blended features (n, 2L).
// One thread per sample, whole warps (the pairing shuffles need both lanes of a pair).
__global__ void k_hash_index_paired(fv_hash h, const float* __restrict__ x, int64_t n, uint32_t* __restrict__ idx,
                                    float* __restrict__ feat) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = p < n;
  const int64_t q = live ? p : n - 1;
  float xn[3]; bool msk[3];
  hash_norm(h, x[3 * q], x[3 * q + 1], x[3 * q + 2], xn, msk);
  const uint32_t a = threadIdx.x & 1u;
  constexpr int NL = FV_RAD_NL;
  for (int c = 0; c < 16 / NL; ++c) {
    float2 fv[NL];
    uint32_t io[NL * 8];
    hash_levels_paired<NL, true>(h, NL * c, xn, fv, io);
    const int64_t sA = p & ~(int64_t)1, sB = sA + 1;     // the even lane's / the odd lane's sample
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int lev = NL * c + l;
      if (lev >= h.n_levels) break;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (sA < n) idx[(sA * h.n_levels + lev) * 8 + a * 4 + k] = io[l * 8 + k];
        if (sB < n) idx[(sB * h.n_levels + lev) * 8 + a * 4 + k] = io[l * 8 + 4 + k];
      }
      if (live) { feat[p * 2 * h.n_levels + 2 * lev] = fv[l].x; feat[p * 2 * h.n_levels + 2 * lev + 1] = fv[l].y; }
    }
  }
}

// Gather-rate probe (measurement, bench.py): k_radiance_tc's gather stage alone -- the same
// hash_norm + hash_levels_paired<FV_RAD_NL> loop over all levels, persistent warpgroups, one
// sample per thread -- with the features summed into a per-thread sink instead of the MLP.
// mode 0: the given canonical points (the frame's real foreground stream); mode 1: uniformly
// random points in the box (hash of the sample id), i.e. no reuse beyond chance: the rate of
// compulsory L1-miss gathers from the L2-resident table with the production access pattern.
__global__ void __launch_bounds__(256) k_gather_probe(fv_hash h, const float4* __restrict__ xf, int64_t n, int mode,
                                                      float* __restrict__ sink) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t s = base + threadIdx.x;
    float x0, x1, x2;
    if (mode == 0) {
      const float4 v = xf[s < n ? s : n - 1];
      x0 = v.x; x1 = v.y; x2 = v.z;
    } else {
      uint32_t k = (uint32_t)s * 0x9E3779B9u + 0x7F4A7C15u;
      k ^= k >> 16; k *= 0x85EBCA6Bu; k ^= k >> 13; k *= 0xC2B2AE35u; k ^= k >> 16;
      const uint32_t k2 = k * 0x27D4EB2Fu + 0x165667B1u, k3 = (k2 ^ (k2 >> 15)) * 0x2C1B3C6Du;
      x0 = h.cmin[0] + (float)(k >> 8) * (1.0f / 16777216.0f) / h.cinv[0];
      x1 = h.cmin[1] + (float)(k2 >> 8) * (1.0f / 16777216.0f) / h.cinv[1];
      x2 = h.cmin[2] + (float)(k3 >> 8) * (1.0f / 16777216.0f) / h.cinv[2];
    }
    float xn[3]; bool msk[3];
    hash_norm(h, x0, x1, x2, xn, msk);
    constexpr int NL = FV_RAD_NL;
#pragma unroll 1
    for (int c = 0; c < 16 / NL; ++c) {
      float2 fv[NL];
      hash_levels_paired<NL>(h, NL * c, xn, fv);
#pragma unroll
      for (int q = 0; q < NL; ++q) acc += fv[q].x + fv[q].y;
    }
  }
  sink[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

}  // namespace fv

using namespace fv;

extern "C" int32_t fv_gather_probe(const fv_hash* hash, const float* d_xf, int64_t n, int32_t mode, float* d_sink,
                                   int64_t sink_len, void* stream) {
  if (int32_t e = check_hash(hash)) return e;
  if (n < 0 || (mode == 0 && n > 0 && !d_xf) || mode < 0 || mode > 1 || !d_sink)
    return set_error(FV_EDIM, "fv_gather_probe: bad arguments");
  if (hash->n_levels != 16) return set_error(FV_EUNSUPPORTED, "fv_gather_probe: 16 levels");
  if (n == 0) return FV_OK;
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, std::min<int64_t>((int64_t)n_sm * 8, sink_len / 256));
  if (blocks < 1) return set_error(FV_EDIM, "fv_gather_probe: sink too small (>= 256 floats)");
  k_gather_probe<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(*hash, (const float4*)d_xf, n, mode, d_sink);
  return check_launch("fv_gather_probe");
}

extern "C" int32_t fv_hash_index_paired(const fv_hash* hash, const float* d_x, int64_t n, uint32_t* d_index,
                                        float* d_feat, void* stream) {
  if (int32_t e = check_hash(hash)) return e;
  if (n < 0 || (n > 0 && (!d_x || !d_index || !d_feat))) return set_error(FV_EDIM, "fv_hash_index_paired: bad arguments");
  if (n == 0) return FV_OK;
  k_hash_index_paired<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*hash, d_x, n, d_index, d_feat);
  return check_launch("fv_hash_index_paired");
}

#if FV_OFF_PROF
// alt builds only (tools/prof_offset.py): the timeline probe of k_offset_tc
extern "C" int32_t fv_debug_offset_prof(long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, g_off_prof, sizeof(g_off_prof)) == cudaSuccess ? FV_OK : FV_ELAUNCH;
}
#endif

extern "C" size_t fv_field_pack_bytes(void) { return PK_BYTES; }

// residual_offset + warp_point composition on the tensor cores:
// xs (n,4) = [x_skel, L] -> out (n,4) = [x_final, L]  (one k_offset_tc launch)
extern "C" int32_t fv_residual_offset(const fv_field* field, const float* d_xs, int64_t n, float eps_w, float* d_out,
                                      void* stream) {
  if (!field || n < 0) return set_error(FV_EDIM, "fv_residual_offset: bad arguments");
  if (field->precision != 1 || !field->d_tc_pack || !field->d_off_b0_eff)
    return set_error(FV_EUNSUPPORTED, "fv_residual_offset: tensor-core path only (precision 1, packed weights)");
  if (n == 0) return FV_OK;
  launch_offset(field, (const float4*)d_xs, n, eps_w, (float4*)d_out, nullptr, nullptr, (cudaStream_t)stream);
  return check_launch("fv_residual_offset");
}

extern "C" int32_t fv_field_pack(const fv_field* field, void* d_tc_pack, void* stream) {
  if (!field || !d_tc_pack) return set_error(FV_EDIM, "fv_field_pack: null argument");
  if (field->pe_bands < 1 || field->pe_bands > 6) return set_error(FV_EUNSUPPORTED, "fv_field_pack: 1..6 PE bands");
  k_field_pack<<<dim3(16, 8), 256, 0, (cudaStream_t)stream>>>(*field, (uint8_t*)d_tc_pack);
  return check_launch("fv_field_pack");
}
