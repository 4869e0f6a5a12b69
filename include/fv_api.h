/* fv_api.h -- C ABI of libfvcuda.so, the sm_100a implementation of the freeview
 * per-ray-sample path (inverse-LBS warp -> offset MLP -> hash grid -> radiance MLP ->
 * compositing, plus backward and Adam).
 *
 * The reference (arxiv 2306.16541 "freeview", /root/reference/pkg) is pure Python and
 * exposes no FFI; each entry point below replaces one reference operator (cited per
 * function as file:line; ad = pkg/src/freeview/autodiff.py, fu = fused.py,
 * S = SPEC.md).  Binding: ctypes (paper_2306_16541_b200/_lib.py).
 *
 * Conventions
 *  - every pointer argument named d_* is a DEVICE pointer owned by the caller; the
 *    library never allocates or frees device memory (workspaces are caller-provided);
 *  - `stream` is a cudaStream_t passed as void*; all work is enqueued on it, nothing
 *    synchronises unless the function says so;
 *  - no hidden shared state: per-call constants travel in the parameter structs, so calls
 *    on different streams / host threads are independent; the only library state is the
 *    thread-local message fv_last_error() returns (per host thread, never shared);
 *  - return value: FV_OK or one of the FV_E* codes; the Python layer maps
 *    FV_EDIM -> DimensionError, FV_ENONFINITE -> TrainingError, others -> RuntimeError.
 */
#ifndef FV_API_H
#define FV_API_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FV_OK 0
#define FV_EDIM 1        /* shape / size / configuration error */
#define FV_ENONFINITE 2  /* non-finite value detected (Adam gradients) */
#define FV_ELAUNCH 3     /* CUDA launch / runtime error */
#define FV_EUNSUPPORTED 4

#define FV_MAX_BONES 32
#define FV_MAX_VOL_RES 128
#define FV_MAX_LEVELS 16
#define FV_MAX_SUBJECTS 8

/* ---- parameter blocks (plain data, host memory) ----------------------------------- */

typedef struct fv_camera {
  float kinv[9];    /* K^-1 row-major                      (cap:73-82) */
  float rot[9];     /* world->camera R row-major           (cap:62-71) */
  float center[3];  /* camera centre -R^T t                (cap:69-71) */
  int32_t width, height;
} fv_camera;

typedef struct fv_march {
  float obox_min[3], obox_max[3]; /* observation-space sampling box */
  int32_t n_samples;              /* N samples per ray                                 */
  int32_t jitter;                 /* 0: bin midpoints, 1: counter-hash jitter          */
  uint32_t seed;
  float eps_w;                    /* foreground likelihood threshold 1e-4      */
  float eps_t;                    /* early-termination transmittance (0 = off)         */
  float bg[3];                    /* background colour                         */
  const uint32_t* d_occ;          /* 32^3 occupancy bitfield (1024 words) or NULL      */
  float occ_scale[3];             /* float32(32 / (obox_max - obox_min))               */
  const int32_t* d_pix;           /* optional list of linear pixel ids (NULL = 0..R-1) */
  int32_t pix_offset;             /* first pixel id when d_pix == NULL                 */
  int32_t out_by_pixel;           /* 1: rgb/alpha written at the pixel id (image), 0: ray */
  int32_t round_samples;          /* marching-round size K: with eps_t > 0 and 0 < K < N the
                                     render marches K samples per live ray per round and
                                     retires rays whose T fell below eps_t (0: one pass) */
} fv_march;

typedef struct fv_warp {
  int32_t n_bones;                /* K <= FV_MAX_BONES                                 */
  int32_t vol_res;                /* G (32), 2 <= G <= FV_MAX_VOL_RES                  */
  int32_t vol_half;               /* corner-packed volume dtype: 0 fp32, 1 fp16        */
  const void* d_vol_packed;       /* [K][(G+1)^3][8] corner-packed weights             */
  const float* d_g;               /* [K][12] G_i = (R row-major 9, t 3), device        */
  float wbox_min[3];              /* canonical box of W^c                              */
  float wscale[3];                /* float32((G-1)/(wbox_max-wbox_min))  (ad:746)      */
} fv_warp;

/* Multi-subject scene (BASELINE config 5; builder-defined, parity unpinned): per-subject
 * renders over disjoint boxes merged front to back in entry-depth order. */
typedef struct fv_scene_merge {
  int32_t n_subjects;                      /* 1..FV_MAX_SUBJECTS                         */
  fv_camera cam[FV_MAX_SUBJECTS];          /* subject-local cameras (world cam - offset) */
  float box_min[3], box_max[3];            /* subject box in subject-local coordinates   */
  const float* d_rgb[FV_MAX_SUBJECTS];     /* [n_pix][3] premultiplied, background 0     */
  const float* d_alpha[FV_MAX_SUBJECTS];   /* [n_pix]                                    */
  float bg[3];                             /* scene background                           */
} fv_scene_merge;

typedef struct fv_hash {
  int32_t n_levels, n_feat, log2_T;
  int32_t res[FV_MAX_LEVELS];
  int32_t dense[FV_MAX_LEVELS];
  uint32_t offset[FV_MAX_LEVELS];
  int32_t table_half;             /* table dtype: 0 fp32, 1 fp16                       */
  const void* d_table;            /* [entries][n_feat]                                 */
  float cmin[3], cinv[3];         /* canonical normalisation                           */
} fv_hash;

typedef struct fv_field {
  int32_t precision;              /* 0: fp32 SIMT (1e-5 parity), 1: fp16 tcgen05       */
  int32_t pe_bands;               /* 6                                                  */
  float pe_w[8];                  /* Hann band weights (ad:574-578)                     */
  int32_t offset_enabled;         /* residual stage                             */
  /* fp32 weights, (in,out) row-major as the reference stores them (ad:403-425) */
  const float* d_off_w[5]; const float* d_off_b[5];   /* 111->128->128->128->128->3     */
  const float* d_rad_w[3]; const float* d_rad_b[3];   /* 32->64->64->4                  */
  const float* d_off_b0_eff;      /* [128] b0 + Omega @ W0[39:111] (per frame)          */
  const void* d_tc_pack;          /* fp16 tcgen05 weight pack (fv_field_pack) or NULL   */
} fv_field;

/* ---- misc ---------------------------------------------------------------------------- */

int32_t fv_version(void);                       /* ABI version (100 = 1.0)            */
const char* fv_last_error(void);                /* thread-local message of last error */
int32_t fv_device_sm(void);                     /* SM count of the current device     */
/* sizeof of the 6 parameter structs (camera, march, warp, hash, field, scene_merge) -> out[6];
 * lets a binding verify its struct layout without a GPU. */
void fv_struct_sizes(int64_t* out);

/* ---- warp (ad:728-808) ----------------------------------------------------- */

/* W^c (C,G,G,G) fp32 softmax output -> corner-packed volume of the first K channels,
 * fp32 or fp16 (warp->vol_half).  Replaces the zero-padded grid of ad:755-756. */
int32_t fv_warp_pack(const float* d_vol, int32_t channels, const fv_warp* warp,
                     void* d_vol_packed, void* stream);

/* Skeleton warp of n points: x (n,3) -> x_skel (n,3), L (n), fg (n) uint8; optional
 * per-bone weights w (K,n) (NULL to skip).  S:327-336 / ad:728-773. */
int32_t fv_warp_fwd(const fv_warp* warp, float eps_w, const float* d_x, int64_t n,
                    float* d_xskel, float* d_lik, uint8_t* d_fg, float* d_w, void* stream);

/* sample_bone_channels (reference freeview.autodiff, ad:728-773) on its own: channel i of the
 * packed W^c at the bone-i points, pts (K,n,3) -> out (K,n), K = warp->n_bones; zero outside
 * the one-voxel-padded grid.  Same trilinear sample as inside fv_warp_fwd. */
int32_t fv_sample_bone_channels(const fv_warp* warp, const float* d_pts, int64_t n, float* d_out, void* stream);

/* Backward of fv_sample_bone_channels (ad:775-806) for upstream g (K,n): d vol (C,G,G,G) fp32
 * accumulated (trilinear-weight scatter, atomics; may be NULL) and d pts (K,n,3) written
 * (may be NULL); points outside the padded grid get zero gradient. */
int32_t fv_sample_bone_channels_bwd(const fv_warp* warp, const float* d_pts, int64_t n, const float* d_g,
                                    float* d_dvol, float* d_dpts, void* stream);

/* d x_skel (n,3) -> d W^c (C,G,G,G) fp32 (accumulated, atomics).  ad:775-789 + Eq 9. */
int32_t fv_warp_bwd(const fv_warp* warp, float eps_w, const float* d_x, int64_t n,
                    const float* d_dxskel, float* d_dvol, void* stream);
/* fv_warp_bwd that also accumulates dL/dG_i (the gradient into the motion bases, for pose
 * refinement) into d_dg [K][12] = (R row-major, t); d_dvol may be NULL. */
int32_t fv_warp_bwd_g(const fv_warp* warp, float eps_w, const float* d_x, int64_t n,
                      const float* d_dxskel, float* d_dvol, float* d_dg, void* stream);

/* ---- hash grid (builder-defined; PARITY UNPINNED) ------------------------------------- */

int32_t fv_hash_fwd(const fv_hash* hash, const float* d_x, int64_t n, float* d_feat,
                    uint32_t* d_index /* (n, L, 8) or NULL */, void* stream);

/* d feat (n, L*F) -> d table (entries, F) fp32 (accumulated) and d x (n,3) (or NULL). */
int32_t fv_hash_bwd(const fv_hash* hash, const float* d_x, int64_t n, const float* d_dfeat,
                    float* d_dtable, float* d_dx, void* stream);

/* Verification entry for the production gather path: the lane-paired, strength-reduced
 * index arithmetic k_radiance_tc uses (hash_levels_paired) on canonical points x (n,3) ->
 * every corner's global table index (n, L, 8) and the blended features (n, 2L).  Lets the
 * bit-exact index bar be checked on the path the headline render runs, not only on
 * fv_hash_fwd's separate scalar form. */
int32_t fv_hash_index_paired(const fv_hash* hash, const float* d_x, int64_t n, uint32_t* d_index,
                             float* d_feat, void* stream);

/* Measurement probe (bench.py): the gather stage of the fused radiance kernel alone (same
 * lane-paired pattern, all levels, features summed into d_sink, >= 256 x blocks floats) over
 * n canonical points xf (n,4) = [x_final, .] (mode 0) or n uniformly random box points
 * (mode 1: compulsory-miss gathers from the L2-resident table -- the measured gather
 * ceiling the radiance kernel is graded against besides HBM). */
int32_t fv_gather_probe(const fv_hash* hash, const float* d_xf, int64_t n, int32_t mode, float* d_sink,
                        int64_t sink_len, void* stream);

/* ---- MLPs (ad:403-425; fu:132-227) ---------------------------------------------------- */

/* Dense fp32 layer y = act(x @ W + b), W (k_in, n_out) row-major; act 0 none, 1 relu. */
int32_t fv_linear_fwd(const float* d_x, const float* d_w, const float* d_b, float* d_y,
                      int64_t m, int32_t k_in, int32_t n_out, int32_t act, void* stream);

/* Backward of fv_linear_fwd: given y and dy -> dx (may be NULL), dW += x^T dz, db += sum dz. */
int32_t fv_linear_bwd(const float* d_x, const float* d_w, const float* d_y, const float* d_dy,
                      float* d_dx, float* d_dw, float* d_db, int64_t m, int32_t k_in,
                      int32_t n_out, int32_t act, void* stream);

/* fused_forward (fu:145-193): the reference's fixed-width MLP (n_layers 2..8; weights[l]
 * (in_l, out_l) row-major device pointers in a HOST array, widths in_dim -> 64 -> ... -> 64 ->
 * out_dim, in/out <= 64; biases[l] device pointers or a NULL array) on x (m, in_dim) ->
 * y (m, out_dim), ReLU on all but the last layer.  One launch: all weights resident in
 * shared memory, 128-row chunks with on-chip activations, fp32 FMAs in fixed order. */
int32_t fv_fused_mlp_fwd(const float* d_x, int64_t m, int32_t in_dim, int32_t out_dim, int32_t n_layers,
                         const float* const* d_w, const float* const* d_b, float* d_y, void* stream);

/* Pack the fp32 field weights into the fp16 tcgen05 operand layout (+ fp32 biases).
 * Workspace d_tc_pack must hold fv_field_pack_bytes() bytes. */
size_t fv_field_pack_bytes(void);
int32_t fv_field_pack(const fv_field* field, void* d_tc_pack, void* stream);

/* Per-frame folded bias b0' = b0 + pose @ W0[3+6L:, :] (pose: n_pose floats, device). */
int32_t fv_offset_bias(const fv_field* field, const float* d_pose, int32_t n_pose,
                       float* d_b0_eff, void* stream);

/* Field on n canonical samples: xs (n,4) = [x_skel, L] (foreground iff L > eps_w) ->
 * rgbs (n,4) = [c, sigma] fp32 (zeros on background); optional x_final (n,3).
 * S:346-358 (residual offset on posenc) + hash grid + S:419-427 (radiance heads).
 * Workspace: fv_field_workspace_bytes(n, precision) bytes (0 for the tcgen05 path). */
size_t fv_field_workspace_bytes(int64_t n, int32_t precision);
/* Residual stage alone (tensor-core path): xs (n,4) [x_skel, L] -> out (n,4) [x_final, L].
 * query_radiance alone is fv_field_fwd with offset_enabled = 0. */
int32_t fv_residual_offset(const fv_field* field, const float* d_xs, int64_t n, float eps_w,
                           float* d_out, void* stream);
int32_t fv_field_fwd(const fv_field* field, const fv_hash* hash, const float* d_xs, int64_t n,
                     float eps_w, float* d_rgbs, float* d_xfinal, void* d_work, size_t work_bytes,
                     void* stream);

/* ---- compositing (ad:815-837) ---------------------------------------------- */

/* transmittance (reference freeview.autodiff, ad:815-837): attenuations atten (R,N) = 1 - opacity
 * -> T (R,N+1), T[r,0] = 1, T[r,i+1] = T[r,i] atten[r,i] in fp32 (exclusive running product). */
int32_t fv_transmittance(const float* d_atten, int64_t n_rays, int32_t n_samples, float* d_trans, void* stream);
/* Its division-free reverse scan (ad:828-835): upstream g (R,N+1) and the forward's T ->
 * d atten (R,N) (written, not accumulated); exact zeros in atten are safe. */
int32_t fv_transmittance_bwd(const float* d_atten, const float* d_trans, const float* d_g, int64_t n_rays,
                             int32_t n_samples, float* d_gatten, void* stream);

/* rays r (R), N samples each: rgbs (R*N,4) [rgb, sigma], delta (R*N), lik (R*N)
 * -> rgb (R,3), alpha (R); optional T (R,N+1) for backward.  Sample layout: ray-major
 * [R][N] (blocked = 0) or the render's ray-block-major layout (blocked = 1). */
int32_t fv_composite_fwd(const float* d_rgbs, const float* d_delta, const float* d_lik,
                         int32_t lik_stride, int32_t blocked, int64_t n_rays, int32_t n_samples,
                         const float bg[3], float eps_w, float eps_t, float* d_rgb,
                         float* d_alpha, float* d_trans, void* stream);

/* Division-free reverse scan: d rgb (R,3), d alpha (R) -> d rgbs (R*N,4) [dc, dsigma]. */
int32_t fv_composite_bwd(const float* d_rgbs, const float* d_delta, const float* d_lik,
                         int32_t lik_stride, int32_t blocked, const float* d_trans,
                         int64_t n_rays, int32_t n_samples, const float bg[3], float eps_w,
                         const float* d_drgb, const float* d_dalpha, float* d_drgbs,
                         void* stream);

/* ---- training-step operators ---------------------------------------------------------- */

/* posenc of x_skel (xs (n,4) = [x_skel, L]; zero rows where L <= eps_w) -> (n, 3+6*bands)
 * with Hann band weights w (ad:574-600); backward accumulates into dx (n,3) (ad:602-609). */
int32_t fv_posenc_fwd(const float* d_xs, int64_t n, float eps_w, int32_t bands, const float* w,
                      float* d_pe, int64_t ld, void* stream);
/* TF32 tensor-core layer ops (training): y = act(x @ W + b); backward from dz (masked
 * pre-activation gradient): dx = (dz @ W^T) * (x_mask > 0) [x_mask may be NULL],
 * dW += x^T dz, db += colsum(dz).  Rows may be padded (ld >= width). */
int32_t fv_linear_fwd_tc(const float* d_x, int64_t ldx, const float* d_w, const float* d_b,
                         float* d_y, int64_t ldy, int64_t m, int32_t k_in, int32_t n_out,
                         int32_t act, void* stream);
int32_t fv_linear_bwd_tc(const float* d_x, int64_t ldx, const float* d_w, const float* d_dz,
                         int64_t ldz, float* d_dx, int64_t lddx, const float* d_xmask,
                         float* d_dw, float* d_db, int64_t m, int32_t k_in, int32_t n_out,
                         void* stream);
/* Same layer ops with the ReLU mask as bits: the forward writes bit (y > 0) of every output
 * ([m][ceil(n_out/32)] uint32 words, bit j of word w <-> column 32w + j; d_relu_bits may be
 * NULL) and the backward masks dx with such bits of the layer input ([m][ceil(k_in/32)]). */
int32_t fv_linear_fwd_tc_bits(const float* d_x, int64_t ldx, const float* d_w, const float* d_b,
                              float* d_y, int64_t ldy, int64_t m, int32_t k_in, int32_t n_out,
                              int32_t act, uint32_t* d_relu_bits, void* stream);
int32_t fv_linear_bwd_tc_bits(const float* d_x, int64_t ldx, const float* d_w, const float* d_dz,
                              int64_t ldz, float* d_dx, int64_t lddx, const uint32_t* d_xmask_bits,
                              float* d_dw, float* d_db, int64_t m, int32_t k_in, int32_t n_out,
                              void* stream);
int32_t fv_posenc_bwd(const float* d_xs, int64_t n, float eps_w, int32_t bands, const float* w,
                      const float* d_dpe, int64_t ld, float* d_dx, void* stream);
/* x_final = x_skel + x_res on foreground rows; d_xres may be NULL. */
int32_t fv_xfinal(const float* d_xs, const float* d_xres, int64_t n, float eps_w, float* d_xf,
                  void* stream);
/* radiance heads c = sigmoid(h[:3]), sigma = softplus(h[3]-1) and backward. */
int32_t fv_heads_fwd(const float* d_xs, const float* d_h, int64_t n, float eps_w, float* d_rgbs,
                     void* stream);
int32_t fv_heads_bwd(const float* d_xs, const float* d_h, const float* d_drgbs, int64_t n,
                     float eps_w, float* d_dh, void* stream);
/* softmax over the channel axis of a (C, V) volume (ad:711-721); bwd accumulates. */
int32_t fv_softmax0_fwd(const float* d_a, int32_t channels, int64_t voxels, float* d_out,
                        void* stream);
int32_t fv_softmax0_bwd(const float* d_out, const float* d_g, int32_t channels, int64_t voxels,
                        float* d_da, void* stream);
/* SPEC compute_loss on patches: rgb rows are G patches of size x size pixels,
 * each row-major; target gathered by d_pix.  loss[0..2] = (lam_mse*MSE + lam_perc*GD, MSE,
 * GD) with GD the multi-scale gradient-difference proxy of the perceptual term;
 * d_drgb = d loss[0] / d rgb. */
int32_t fv_patch_loss(const float* d_rgb, const float* d_target, const int32_t* d_pix, int32_t n_patches,
                      int32_t size, float lam_mse, float lam_perc, float* d_loss, float* d_drgb,
                      void* stream);
/* L2 loss over rays (target gathered at pixel ids, or row r when d_pix is NULL):
 * *d_loss = mean((rgb - t)^2) (device scalar), d_drgb = its gradient. */
int32_t fv_mse_loss(const float* d_rgb, const float* d_target, const int32_t* d_pix,
                    int64_t n_rays, float* d_loss, float* d_drgb, void* stream);

/* ---- fused render (the hot path) ------------------------------------------------------ */

/* Workspace bytes for rendering n_rays rays of n_samples samples with field precision. */
size_t fv_render_workspace_bytes(int64_t n_rays, int32_t n_samples, int32_t precision);

/* Ray generation + slab + stratified sampling + occupancy skip + skeleton warp, one thread
 * per sample.  Outputs per sample: xs (R*N,4) = [x_skel, L] (L = 0 if skipped),
 * delta (R*N), x (R*N,3) world position (may be NULL); per ray: count (R) int32. */
int32_t fv_march_warp(const fv_camera* cam, const fv_march* march, const fv_warp* warp,
                      int64_t n_rays, float* d_xs, float* d_delta, float* d_x,
                      int32_t* d_count, void* stream);

/* The render path's own march + foreground compaction (what fv_render_fwd launches first):
 * per sample slot (ray-block-major, R padded to 32) lik (L, 0 where skipped), delta, and
 * optional flags (uint8: 1 ray hits the box, 2 occupancy cell on or no grid, 4 L > eps_w);
 * the compacted foreground stream xsc (<= S, 4) = [x_skel, L] with its slot ids idx and its
 * length *d_n_fg (device int32); per-ray sample counts d_count (may be NULL).
 * padded(n_rays) x n_samples must stay below 2^31 (int32 slot ids; FV_EDIM otherwise). */
int32_t fv_march_compact(const fv_camera* cam, const fv_march* march, const fv_warp* warp, int64_t n_rays,
                         float* d_lik, float* d_delta, float* d_xsc, int32_t* d_idx, int32_t* d_n_fg,
                         int32_t* d_count, uint8_t* d_flags, void* stream);

/* Full forward: rays -> rgb (3 floats) and alpha per ray (or per pixel, out_by_pixel),
 * per-ray sample counts (may be NULL).  d_work >= fv_render_workspace_bytes().
 * padded(n_rays) x n_samples must stay below 2^31 sample slots (FV_EDIM otherwise; the
 * Python Renderer splits larger ray sets into chunks of whole 32-ray blocks).
 * There is no single fv_render_bwd: the training step differentiates the
 * render by the per-op sequence of the reference Tape (ad:114-134) -- fv_composite_bwd,
 * fv_heads_bwd, fv_linear_bwd_tc_bits (radiance MLP), fv_hash_bwd, fv_linear_bwd_tc_bits
 * (residual MLP), fv_posenc_bwd, fv_warp_bwd[_g], fv_softmax0_bwd -- over activations its
 * forward keeps (the render path's compacted streams are not kept); INTEGRATION.md. */
int32_t fv_render_fwd(const fv_camera* cam, const fv_march* march, const fv_warp* warp,
                      const fv_hash* hash, const fv_field* field, int64_t n_rays,
                      void* d_work, size_t work_bytes, float* d_rgb, float* d_alpha,
                      int32_t* d_count, void* stream);

/* Joint compositing of per-subject renders for pixel ids pix0 .. pix0+n_pix-1 (subject and
 * output buffers image-sized, indexed by pixel id):
 * rgb = sum_s (prod_{j before s} T_j) C_s + (prod T) bg, alpha = 1 - prod T, subjects ordered
 * by ray entry depth (same float32 slab as fv_march_warp). */
int32_t fv_scene_composite(const fv_scene_merge* m, int64_t pix0, int64_t n_pix, float* d_rgb,
                           float* d_alpha, void* stream);

/* fv_render_fwd with CUDA events between its stages (measurement): synchronises, writes
 * stage_ms[5] = {march+warp+compaction, residual MLP, hash+radiance, compositor, total}
 * and the number of foreground samples the field evaluated to *n_fg (may be NULL). */
int32_t fv_render_fwd_timed(const fv_camera* cam, const fv_march* march, const fv_warp* warp,
                            const fv_hash* hash, const fv_field* field, int64_t n_rays,
                            void* d_work, size_t work_bytes, float* d_rgb, float* d_alpha,
                            float* stage_ms, int64_t* n_fg, void* stream);

/* ---- occupancy (builder-defined; PARITY UNPINNED) ------------------------------------- */

/* Evaluate density at 2x2x2 sub-cell points of each of the 32^3 observation-box cells
 * through warp + field; bit (x*32+y)*32+z is set when any point has L > eps_w and
 * sigma > threshold.  Workspace: fv_occupancy_workspace_bytes(field->precision). */
size_t fv_occupancy_workspace_bytes(int32_t precision);
int32_t fv_occupancy_build(const fv_march* march, const fv_warp* warp, const fv_hash* hash,
                           const fv_field* field, float threshold, void* d_work,
                           size_t work_bytes, uint32_t* d_occ, void* stream);

/* ---- Adam (ad:880-912) ---------------------------------------------------------------- */

/* Sets *d_flag (device int32) to `code` (!= 0; first writer wins) if any of x[0..n) is not
 * finite -- the per-block check adam_step makes before touching any parameter (ad:898-902). */
int32_t fv_check_finite(const float* d_x, int64_t n, int32_t code, int32_t* d_flag, void* stream);

/* In-place bias-corrected Adam over n params; lr per segment: seg_end (n_seg) exclusive
 * end offsets, lr (n_seg).  Writes an fp16 copy of [half_begin, half_end) into d_half
 * (if non-NULL).  Non-finite grads set *d_flag to 1 + segment index (device int32) and
 * skip the update of that element. */
int32_t fv_adam_step(float* d_param, const float* d_grad, float* d_m, float* d_v, int64_t n,
                     const int64_t* seg_end, const float* lr, int32_t n_seg, int32_t step,
                     float beta1, float beta2, float eps, void* d_half, int64_t half_begin,
                     int64_t half_end, int32_t* d_flag, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FV_API_H */
