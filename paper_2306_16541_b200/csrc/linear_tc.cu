// C-ABI entry points of the training-time MLP layers on 5th-gen tensor cores (the layer
// ops of the reference training step: `linear` forward ad:403-416, backward ad:417-422).
// The kernels are the split-precision 3xTF32 warp-specialised GEMMs of gemm_tf32x3.cu:
// forward and dX on k_rows, dW (+ db) on k_dw.
//
// Layers with n_out <= 4 (the 128 -> 3 residual output and the 64 -> 4 radiance head) go to
// the fp32 SIMT kernels of narrow_layers.cu instead: a 128-wide MMA tile would be ~97% padding.
//
// Why TF32x3 rather than fp16 here: the training forward must reproduce the oracle's
// float32 x_final (it picks the hash cells the gradient is scattered into), and dW reduces
// over ~786K samples of gradients that are 1e-9..1e-5 in magnitude -- below fp16's normal
// range -- with heavy sign cancellation; the layers are HBM-bound on fp32 activations, so
// the three MMAs per product are (almost) free.
#include <cuda_runtime.h>
#include "fv_internal.h"
#include "gemm_tf32x3.h"
#include "narrow_layers.h"

using namespace fv;

// y = act(x @ W + b).  W (k_in, n_out) row-major; x rows have stride ldx >= k_in, y rows
// stride ldy >= n_out.
extern "C" int32_t fv_linear_fwd_tc(const float* d_x, int64_t ldx, const float* d_w, const float* d_b, float* d_y,
                                    int64_t ldy, int64_t m, int32_t k_in, int32_t n_out, int32_t act, void* stream) {
  if (m < 0 || k_in < 1 || k_in > 256 || n_out < 1 || n_out > 128 || ldx < k_in || ldy < n_out)
    return set_error(FV_EDIM, "fv_linear_fwd_tc: bad shape");
  if (m == 0) return FV_OK;
  if (n_out <= 4 && k_in <= 128) return nl::narrow_fwd(d_x, ldx, k_in, d_w, d_b, act, d_y, ldy, m, n_out, (cudaStream_t)stream);
  g3::RowsArgs r{d_x, ldx, k_in, d_w, 1, n_out, n_out, d_b, act, nullptr, 0, d_y, ldy, m};
  return g3::rows_gemm(r, (cudaStream_t)stream);
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
    if (n_out <= 4) {
      if (int32_t e = nl::narrow_dx(d_dz, ldz, n_out, d_w, k_in, nullptr, d_xmask, ldx, d_dx, lddx, m, st)) return e;
    } else {
      g3::RowsArgs r{d_dz, ldz, n_out, d_w, n_out, 1, k_in, nullptr, 0, d_xmask, ldx, d_dx, lddx, m};
      if (int32_t e = g3::rows_gemm(r, st)) return e;
    }
  }
  if (d_dw) {
    if (n_out <= 4) {
      if (int32_t e = nl::narrow_dw(d_x, ldx, k_in, d_dz, ldz, n_out, d_dw, d_db, m, st)) return e;
    } else {
      g3::DwArgs3 w{d_x, ldx, k_in, d_dz, ldz, n_out, d_dw, d_db, m};
      if (int32_t e = g3::dw_gemm(w, st)) return e;
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
  if (n_out <= 4 && k_in <= 128 && !d_relu_bits)
    return nl::narrow_fwd(d_x, ldx, k_in, d_w, d_b, act, d_y, ldy, m, n_out, (cudaStream_t)stream);
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
    if (n_out <= 4) {
      if (int32_t e = nl::narrow_dx(d_dz, ldz, n_out, d_w, k_in, d_xmask_bits, nullptr, 0, d_dx, lddx, m, st)) return e;
    } else {
      g3::RowsArgs r{d_dz, ldz, n_out, d_w, n_out, 1, k_in, nullptr, 0, nullptr, 0, d_dx, lddx, m};
      r.bits_in = d_xmask_bits;
      if (int32_t e = g3::rows_gemm(r, st)) return e;
    }
  }
  if (d_dw) {
    if (n_out <= 4) {
      if (int32_t e = nl::narrow_dw(d_x, ldx, k_in, d_dz, ldz, n_out, d_dw, d_db, m, st)) return e;
    } else {
      g3::DwArgs3 w{d_x, ldx, k_in, d_dz, ldz, n_out, d_dw, d_db, m};
      if (int32_t e = g3::dw_gemm(w, st)) return e;
    }
  }
  return FV_OK;
}
