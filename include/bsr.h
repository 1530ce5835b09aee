/*
 * bsr.h -- C-ABI of the B200-native tile rasterizer ("Beta-splat renderer", libbsr.so).
 *
 * Drop-in boundary for the hot path of /root/reference (betasplat, arXiv 2501.18630):
 *
 *   reference (pkg/src/betasplat/...)                     this ABI
 *   ---------------------------------------------------   ------------------------------
 *   rasterizer.render_tiled        rasterizer.py:194-211   bsr_forward
 *   rasterizer.render_backward     rasterizer.py:230-321   bsr_backward
 *     (_view_setup :88-103, project_arrays primitive.py:221-277, sh_basis
 *      appearance.py:235-261, _depth_order :83-85, tile_bins :161-191,
 *      project_backward primitive.py:302-367, _sh_basis_grad appearance.py:264-300)
 *   core.forward_tiled             _raster.pyx:130-155     bsr_core_forward_tiled
 *   core.backward                  _raster.pyx:244-287     bsr_core_backward
 *   training.loss / ssim           training.py:51-131      bsr_loss_l1_dssim
 *   training.adam_step             training.py:258-273     bsr_adam_step
 *   training.loss direct terms     training.py:112-124     bsr_regularizers
 *   training.inject_noise          training.py:276-292     bsr_inject_noise
 *   training.exponential_lr        training.py:134-145     bsr_lr_schedule (device-side)
 *   mcmc.find_dead                 mcmc.py:32-36           bsr_find_dead
 *   mcmc.plan_relocation           mcmc.py:49-70           bsr_sample_live
 *   mcmc.apply_relocation          mcmc.py:86-106          bsr_apply_relocation
 *   mcmc.grow                      mcmc.py:108-146         bsr_sample_live + bsr_grow
 *   sceneio.save/load_checkpoint   sceneio.py:467-564      bsr_checkpoint_pack / _unpack
 *   compression.morton_keys/sort   compression.py:34-66    bsr_codec_sort
 *   compression.pack / unpack      compression.py:141-250  bsr_codec_encode / _decode
 *
 * Conventions
 *   - Every pointer is DEVICE memory owned by the caller unless stated; the library
 *     allocates nothing.  Scratch/state lives in a caller-provided "frame" buffer sized
 *     by bsr_frame_bytes(); forward writes the saved state backward reads (the
 *     reference recomputes projection/sort/binning in backward, rasterizer.py:243-251).
 *   - Every call is stream-ordered on the given cudaStream_t (passed as void*), reentrant
 *     per stream, no global mutable state, no host synchronisation except
 *     bsr_frame_status() (which synchronises the stream to read counters).
 *   - Every function returns an int status (BSR_OK = 0).  No C++ exception crosses the ABI.
 *   - Layouts follow PrimitiveSet / Camera (primitive.py:83-137, 387-426), fp32 on device:
 *       positions (N,3), rotations (N,4) wxyz unnormalised, log_scales (N,3),
 *       opacity_raw (N,) pre-sigmoid, shapes (N,) Beta shape b, sh (N,K,3) DC first.
 *     Images are (H,W,3) / (H,W) row-major, pixel (row i, col j) at (x=j, y=i).
 */
#ifndef BSR_H_
#define BSR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum bsr_status {
    BSR_OK = 0,
    BSR_ERR_BAD_ARG = 1,          /* ValueError in the reference (shape/dtype/size)        */
    BSR_ERR_CAPACITY = 2,         /* tile-entry capacity exceeded: retry with entries_needed */
    BSR_ERR_CUDA = 3,             /* a CUDA runtime error (launch / async fault)            */
    BSR_ERR_DEGENERATE_QUAT = 4,  /* DegenerateQuaternionError (primitive.py:44-56)         */
    BSR_ERR_FRAME_TOO_SMALL = 5,  /* frame buffer smaller than bsr_frame_bytes()            */
};

/* Pinhole camera (primitive.py:83-137); world_to_camera row-major 4x4. */
typedef struct bsr_camera {
    double world_to_camera[16];
    double fx, fy, cx, cy;
    int32_t width, height;
} bsr_camera;

/* Colour models (appearance.py). */
enum bsr_color_model {
    BSR_COLOR_SH = 0, /* real SH, sh (N,K,3), K = (degree+1)^2 <= 16 (SH adapter) */
    BSR_COLOR_SB = 1, /* Spherical Beta (the reference's default): base_colors (N,3),
                         lobe_axes (N,M,3), lobe_colors (N,M,3), M <= 4 (appearance.py:82-163) */
};

/* Primitive parameters, device fp32 SoA (PrimitiveSet layout, primitive.py:387-426). */
typedef struct bsr_scene {
    const float *positions, *rotations, *log_scales, *opacity_raw, *shapes, *sh;
    int64_t n;
    int32_t sh_coeffs;   /* SH: K = (degree+1)^2, degree <= 3 */
    int32_t color_model; /* bsr_color_model */
    const float *base_colors, *lobe_axes, *lobe_colors; /* SB arrays */
    int32_t lobes;       /* SB: M */
    int32_t reserved;
    /* Optional: this view's fp32 colours precomputed by bsr_view_colors, (N, 4) float
     * (rgb + pad).  bsr_forward then reads them instead of the appearance parameters (a
     * multi-view step reads the SH coefficients once for all its views, not once per
     * view); the colours are the same bits preprocess would compute.  NULL: evaluate. */
    const float *view_rgb;
} bsr_scene;

/* Per-parameter gradient buffers (device fp32, same shapes); bsr_backward ADDS into them.
 * Only the pointers of the scene's colour model are used. */
typedef struct bsr_grads {
    float *positions, *rotations, *log_scales, *opacity_raw, *shapes, *sh;
    float *base_colors, *lobe_axes, *lobe_colors;
    /* 0: the gradients are ADDED into these buffers (multi-view accumulation); nonzero:
     * they are WRITTEN -- every primitive's rows, culled ones zeroed, screen_grad_norm too --
     * so the caller needs no memset and no buffer is read back (not with a deferred colour
     * chain, bsr_backward_deferred_color / drgb). */
    int32_t overwrite;
} bsr_grads;

/* Forward outputs (device; any pointer may be NULL to skip that output). */
typedef struct bsr_outputs {
    float *color;          /* (H,W,3) max(raw, 0)                          rasterizer.py:136 */
    float *raw;            /* (H,W,3) composite incl. background             _raster.pyx:124  */
    float *alpha;          /* (H,W)   1 - T                                                  */
    float *transmittance;  /* (H,W)   final T                                                */
    float *depth;          /* (H,W)   sum_k w_k z_k (extension, no background term)          */
    int32_t *pixel_count;  /* (H,W)   contributors per pixel (extension)                     */
    int32_t *contributions;/* (N,)    pixels each primitive contributed to, ADDED into       */
    int32_t defer_contributions; /* nonzero: bsr_forward adds only the fp64 replay's part of
                            contributions (flagged pixels from their flag point on); the raster's
                            part is added by bsr_contributions() on the same frame, when (if)
                            the caller needs the counts -- counting inside the forward raster
                            costs it ~18% (config 4) */
} bsr_outputs;

/* Optional profiling hooks (caller-owned; pass NULL to disable).
 *   stats:  device uint64[4] the kernels ADD into: [0] forward evaluated (pixel, entry)
 *           pairs (passing the bounds test, up to termination = the roofline's P_f),
 *           [1] forward contributions, [2] backward evaluated pairs (P_b), [3] reserved.
 *   events: caller-created cudaEvent_t handles (void*), recorded on the stream at stage
 *           boundaries.  bsr_forward: [0] start, [1] preprocess, [2] depth sort,
 *           [3] emit, [4] tile sort + ranges, [5] raster, [6] fp64 replay.
 *           bsr_backward: [0] start, [1] raster backward, [2] fp64 replay,
 *           [3] preprocess backward.  NULL entries are skipped. */
typedef struct bsr_profile {
    unsigned long long *stats;
    void *events[8];
} bsr_profile;

typedef struct bsr_frame_info {
    int64_t visible;         /* V: primitives kept by projection                           */
    int64_t entries;         /* E: (tile, primitive) entries                               */
    int64_t entries_needed;  /* E required (== entries unless capacity was exceeded)       */
    int64_t flagged_pixels;  /* pixels re-composited in fp64 (near a decision threshold)   */
    int32_t status;          /* first error raised on the device side (bsr_status)         */
    int32_t reserved;
} bsr_frame_info;

/* ---- version / capability -------------------------------------------------------- */
int bsr_version(int32_t *major, int32_t *minor);
const char *bsr_status_string(int32_t status);

/* ---- frame (state + scratch) sizing ------------------------------------------------- */
int bsr_frame_bytes(int64_t n, int32_t width, int32_t height, int64_t entry_cap,
                    uint64_t *bytes);

/* ---- full pipeline (render_tiled / render_backward) -------------------------------- */
int bsr_forward(const bsr_scene *scene, const bsr_camera *camera, const float background[3],
                void *frame, uint64_t frame_bytes, int64_t entry_cap, const bsr_outputs *out,
                const bsr_profile *profile, void *stream);
/* The raster's part of the contributions of a forward run with defer_contributions, ADDED
 * into contributions (N,): re-walks every pixel's certified entries on the unchanged frame
 * (same decisions, no outputs written).  Call at most once per forward. */
int bsr_contributions(const bsr_scene *scene, const bsr_camera *camera, const float background[3],
                      void *frame, uint64_t frame_bytes, int64_t entry_cap, int32_t *contributions,
                      void *stream);
/* fp32 colours of every primitive for each of `views` camera centres (world, double[3]
 * each): rgb[v][i][0..2] (4 floats per primitive), exactly the values bsr_forward's
 * preprocess computes for that view -- feed rgb + v*N*4 as bsr_scene.view_rgb. */
int bsr_view_colors(const bsr_scene *scene, const double *centers, int32_t views, float *rgb, void *stream);
/* Synchronises `stream`, then reports counters / device-side errors of the last forward. */
int bsr_frame_status(const void *frame, bsr_frame_info *info, void *stream);
/* Asynchronous status (no sync): enqueues on `stream` a copy of the frame's counters into
 * caller-owned host memory `snapshot` of bsr_frame_snapshot_bytes() bytes (pinned, so the
 * copy is truly asynchronous); once the stream has passed that point (e.g. an event
 * recorded after the call has completed) bsr_frame_snapshot_decode() reports what
 * bsr_frame_status() would have.  Lets render_tiled skip the per-call stream sync. */
int bsr_frame_snapshot_bytes(uint64_t *bytes);
int bsr_frame_status_async(const void *frame, void *snapshot, void *stream);
int bsr_frame_snapshot_decode(const void *snapshot, bsr_frame_info *info);
/* Deterministic backward (the reference's bitwise determinism for a fixed input,
 * SPEC.md:334, _raster.pyx:273-286): the same gradients as bsr_backward, but every
 * per-primitive partial is summed as a 64-bit fixed-point integer (two passes: magnitude
 * bound, then the sums), so results are bitwise identical run to run whatever order the
 * device's atomics land in.  det_ws: caller-owned device workspace of
 * bsr_det_workspace_bytes(n) bytes, 256-byte aligned.  drgb: as bsr_backward_deferred_color
 * (SH colour, multi-view), or NULL for the full chain. */
int bsr_det_workspace_bytes(int64_t n, uint64_t *bytes);
int bsr_backward_deterministic(const bsr_scene *scene, const bsr_camera *camera, const float background[3],
                               void *frame, uint64_t frame_bytes, int64_t entry_cap, const float *d_color,
                               const float *d_depth, const bsr_grads *grads, float *screen_grad_norm,
                               float *drgb, void *det_ws, uint64_t det_ws_bytes, void *stream);
/* d_color: (H,W,3) dL/d color (clamped image); d_depth: (H,W) or NULL. */
int bsr_backward(const bsr_scene *scene, const bsr_camera *camera, const float background[3],
                 void *frame, uint64_t frame_bytes, int64_t entry_cap, const float *d_color,
                 const float *d_depth, const bsr_grads *grads, float *screen_grad_norm,
                 const bsr_profile *profile, void *stream);

/* Multi-view steps, SH colour: bsr_backward_deferred_color is bsr_backward except that
 * the SH / view-direction part of the chain is not applied; drgb (device, float4 per
 * primitive, 16-byte aligned) receives (dL/dr, dL/dg, dL/db, 0), zero where culled.
 * bsr_color_grad_views then applies `views` such buffers ([views][N] float4, contiguous)
 * at once: grads.sh += sum_v basis(dir_v) (x) d_rgb_v, grads.positions += sum_v the
 * view-direction chain, dir_v = normalize(position - centers[v]) (host double[views][3]).
 * Same gradients as per-view bsr_backward calls (appearance.py:264-318,
 * rasterizer.py:287-289), with the coefficient gradients read and written once per step. */
int bsr_backward_deferred_color(const bsr_scene *scene, const bsr_camera *camera,
                                const float background[3], void *frame, uint64_t frame_bytes,
                                int64_t entry_cap, const float *d_color, const float *d_depth,
                                const bsr_grads *grads, float *screen_grad_norm,
                                const bsr_profile *profile, float *drgb, void *stream);
int bsr_color_grad_views(const bsr_scene *scene, const float *drgb, const double *centers,
                         int32_t views, const bsr_grads *grads, void *stream);

/* ---- core seam (backend.get_core(): forward_tiled / backward on depth-sorted input) -- */
/* Inputs are DEVICE fp64 arrays exactly as the reference core receives them
 * (_raster.pyx:130-134): means (V,2), conics (V,3), opac (V,), betas (V,), colors (V,3),
 * bounds (V,4) int32 [x0,x1,y0,y1], offsets (T+1,) int64, lists (E,) int64. */
int bsr_core_scratch_bytes(int64_t v, int32_t width, int32_t height, int64_t n_entries,
                           uint64_t *bytes);
int bsr_core_forward_tiled(int64_t v, const double *means, const double *conics,
                           const double *opac, const double *betas, const double *colors,
                           const int32_t *bounds, int32_t height, int32_t width,
                           const double background[3], int32_t tile_size, const int64_t *offsets,
                           const int64_t *lists, int64_t n_entries, double alpha_min,
                           double t_stop, float *raw, float *transmittance,
                           int32_t *contrib, int32_t *pixel_count, void *scratch,
                           uint64_t scratch_bytes, int64_t *flagged_out, void *stream);
int bsr_core_backward(int64_t v, const double *means, const double *conics, const double *opac,
                      const double *betas, const double *colors, const int32_t *bounds,
                      int32_t height, int32_t width, const double background[3],
                      const float *d_raw, int32_t tile_size, const int64_t *offsets,
                      const int64_t *lists, int64_t n_entries, double alpha_min, double t_stop,
                      float *d_means, float *d_conics, float *d_opac, float *d_betas,
                      float *d_colors, void *scratch, uint64_t scratch_bytes, void *stream);

/* ---- loss (training.loss with lambda_opacity = lambda_scale = 0) ------------------- */
/* rendered/target (H,W,3); raw (H,W,3) or NULL: when given, the clamp chain
 * d_raw = d_image * [raw >= 0] (rasterizer.py:253) is fused into the output.
 * loss_out: device double[3] = {loss, l1, ssim}.  scratch: bsr_loss_scratch_bytes(). */
int bsr_loss_scratch_bytes(int32_t width, int32_t height, uint64_t *bytes);
int bsr_loss_l1_dssim(const float *rendered, const float *target, const float *raw,
                      int32_t width, int32_t height, double lambda_ssim, double *loss_out,
                      float *d_image, void *scratch, uint64_t scratch_bytes, void *stream);

/* ---- Adam (training.adam_step), flat parameter buffer with per-group lr ----------- */
/* Groups are contiguous ranges [group_end[g-1], group_end[g]) of the flat buffers. */
int bsr_adam_step(float *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                  int64_t count, int32_t n_groups, const int64_t *group_end /* host */,
                  const float *group_lr /* host */, int64_t step, double beta1, double beta2,
                  double eps, void *stream);
/* Same update with the step count kept in device memory (int64, incremented by the call):
 * no host value changes between steps, so a captured CUDA graph can replay it. */
int bsr_adam_step_device(float *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                         int64_t count, int32_t n_groups, const int64_t *group_end /* host */,
                         const float *group_lr /* host */, int64_t *step_counter, double beta1,
                         double beta2, double eps, void *stream);

/* ---- training-loop neighbours ---------------------------------- */
/* Group table of a flat, group-major parameter buffer (primitive.group_layout): group g
 * occupies elements [start[g], start[g] + width[g] * n) with width[g] floats per primitive.
 * The four named groups must have widths 3 / 4 / 3 / 1. */
#define BSR_MAX_GROUPS 16
typedef struct bsr_layout {
    int64_t n;
    int32_t n_groups;
    int32_t width[BSR_MAX_GROUPS];
    int64_t start[BSR_MAX_GROUPS];
    int32_t g_positions, g_rotations, g_log_scales, g_opacity; /* group indices */
} bsr_layout;

/* training.exponential_lr x scene scale (training.py:134-145, TrainConfig.position_lr
 * :206-215) evaluated on the device from a step counter, so a captured CUDA graph of the
 * training step follows the schedule. */
typedef struct bsr_lr_schedule {
    double lr_init, lr_final;
    int64_t max_steps, delay_steps;
    double delay_mult, scale;
} bsr_lr_schedule;
double bsr_scheduled_lr(const bsr_lr_schedule *sched, int64_t step); /* host helper */

/* Device-step Adam whose group `sched_group` (the positions) takes its learning rate from
 * `sched` at the step being taken (TrainConfig.group_lrs, training.py:217-227). */
int bsr_adam_step_scheduled(float *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                            int64_t count, int32_t n_groups, const int64_t *group_end /* host */,
                            const float *group_lr /* host */, int64_t *step_counter,
                            const bsr_lr_schedule *sched, int32_t sched_group, double beta1,
                            double beta2, double eps, void *stream);


/* One-kernel optimizer step for captured training loops: device step count in
 * step_counter[0] (step_counter: device int64[2], [1] is scratch kept 0 between calls),
 * bumped by the kernel's last block; optional schedule as bsr_adam_step_scheduled
 * (sched may be NULL); zero_grads != 0 clears the gradients after use (the next step
 * accumulates from zero without a separate memset). */
int bsr_adam_step_fused(float *params, float *grads, float *exp_avg, float *exp_avg_sq, int64_t count,
                        int32_t n_groups, const int64_t *group_end /* host */,
                        const float *group_lr /* host */, int64_t *step_counter,
                        const bsr_lr_schedule *sched, int32_t sched_group, double beta1, double beta2,
                        double eps, int32_t zero_grads, void *stream);

/* training.loss direct terms (training.py:112-124): grads[opacity_raw] += lo * o (1 - o),
 * grads[log_scales] += ls * exp(log_scales); loss[0] += lo * sum(o) + ls * sum(s) (device
 * double, may be NULL). */
int bsr_regularizers(const float *params, const bsr_layout *layout, double lambda_opacity,
                     double lambda_scale, float *grads, double *loss, void *stream);

/* training.inject_noise (training.py:276-292): positions += noise_lr * position_lr *
 * (1 - o)^100 * Sigma * eta.  eta: device (N,3) fp32 normals, or NULL for on-device
 * Philox4x32-10 + Box-Muller keyed by (seed, offset + *step_counter, index).  sched != NULL
 * replaces position_lr by the schedule at *step_counter (device int64).  status (device
 * int32, may be NULL) receives BSR_ERR_DEGENERATE_QUAT. */
int bsr_inject_noise(float *params, const bsr_layout *layout, double noise_lr, double position_lr,
                     const bsr_lr_schedule *sched, const int64_t *step_counter, const float *eta,
                     uint64_t seed, uint64_t offset, int32_t *status, void *stream);

/* MCMC densification (mcmc.py).  scratch: bsr_mcmc_scratch_bytes(n) device bytes. */
int bsr_mcmc_scratch_bytes(int64_t n, uint64_t *bytes);
/* mcmc.find_dead (mcmc.py:32-36): dead[0..*count) = ascending indices with
 * sigmoid(opacity_raw) < threshold.  dead: device int64 capacity n; count: device int64. */
int bsr_find_dead(const float *opacity_raw, int64_t n, double threshold, int64_t *dead,
                  int64_t *count, void *scratch, uint64_t scratch_bytes, void *stream);
/* The multinomial draw of mcmc.plan_relocation / mcmc.grow (mcmc.py:49-70, 108-128):
 * live = {o >= threshold} minus exclude[0..*exclude_count); out[k] = live index drawn
 * with odds o / sum(o), k < min(*n_draw_dev, n_draw) (n_draw_dev may be NULL), exactly
 * numpy Generator.choice(live, p=...) when `uniforms` holds numpy's rng.random(draws)
 * (else Philox uniforms from (seed, offset)).  counts (device int32, n) = draws per index
 * (zeroed by the call); live_count (device int64) = |live| (0: nothing drawn, the
 * caller raises AllDeadError). */
int bsr_sample_live(const float *opacity_raw, int64_t n, double threshold, const int64_t *exclude,
                    const int64_t *exclude_count, int64_t exclude_cap, const int64_t *n_draw_dev,
                    int64_t n_draw, const double *uniforms, uint64_t seed, uint64_t offset,
                    int64_t *out, int32_t *counts, int64_t *live_count, void *scratch,
                    uint64_t scratch_bytes, void *stream);
/* mcmc.apply_relocation (mcmc.py:86-106): every dead row takes its target's parameters,
 * dead and target rows the opacity logit(max(1 - (1 - o)^(1/(counts[t]+1)), floor)) and
 * zeroed moments (exp_avg / exp_avg_sq may be NULL). */
int bsr_apply_relocation(float *params, const bsr_layout *layout, float *exp_avg, float *exp_avg_sq,
                         const int64_t *dead, const int64_t *targets, const int64_t *dead_count,
                         int64_t dead_cap, const int32_t *counts, double floor_, void *stream);
/* mcmc.grow after the draw (mcmc.py:128-146): dst (layout for n + n_add) = src rows, then
 * n_add copies of sources[] with the adjusted opacity (also written to the sources);
 * moments copied, zeroed for the sources and the new rows. */
int bsr_grow(const float *src_params, const bsr_layout *src_layout, const float *src_exp_avg,
             const float *src_exp_avg_sq, float *dst_params, const bsr_layout *dst_layout,
             float *dst_exp_avg, float *dst_exp_avg_sq, const int64_t *sources, int64_t n_add,
             const int32_t *counts, double floor_, void *stream);

/* ---- checkpoints (sceneio.save_checkpoint / load_checkpoint, sceneio.py:467-564) ------ */
/* records: device (N, n_props) fp64, row-major (the PLY vertex block of the reference's
 * checkpoint); property q of primitive i <-> flat[prop_start[q] + prop_stride[q] * i]
 * (host tables, n_props <= 64).  unpack rounds to fp32; pack widens exactly. */
int bsr_checkpoint_unpack(const double *records, int64_t n, int32_t n_props, const int64_t *prop_start,
                          const int32_t *prop_stride, float *flat, void *stream);
int bsr_checkpoint_pack(const float *flat, int64_t n, int32_t n_props, const int64_t *prop_start,
                        const int32_t *prop_stride, double *records, void *stream);

/* ---- post-training codec (compression.py:34-250; docs/formats.md "Archives") ----------
 * The device side of compression.pack / unpack; PNG encoding of the byte grids stays on
 * the host (OpenCV, as sceneio.write_png / read_png).  Attribute group g holds channels
 * [0, channels) of primitive i at flat[start + stride * i + c]; its codes occupy
 * rows * cols * channels bytes (row-major grid, channel-interleaved, zero padding) at the
 * running byte offset of the groups before it in `codes`; its min / max at the running
 * channel offset in mins / maxs.  Position byte planes: planes[b][cell][axis] = byte b of
 * the fp32 bits (4 x rows x cols x 3 bytes).  8-bit quantisation only (QUANT_BITS). */
typedef struct {
    int64_t start;
    int32_t stride;
    int32_t channels; /* 1..4 */
} bsr_codec_group;

size_t bsr_codec_scratch_bytes(int64_t n);
/* compression.morton_keys + sort_primitives: keys_out (n, original order; may be NULL)
 * and perm (n) = the stable argsort of the keys. */
int bsr_codec_sort(const float *positions /* (n,3) */, int64_t n, uint64_t *keys_out, int64_t *perm,
                   void *scratch, size_t scratch_bytes, void *stream);
/* compression.pack minus the file I/O: grid cell j holds primitive perm[j] (perm NULL:
 * j).  mins / maxs (device, one per channel) receive quantize_attribute's ranges; a
 * non-finite value sets *status (device, may be NULL) to BSR_ERR_BAD_ARG. */
int bsr_codec_encode(const float *flat, const float *positions, int64_t n, const int64_t *perm,
                     int32_t n_groups, const bsr_codec_group *groups /* host */, int32_t rows,
                     int32_t cols, uint8_t *planes, uint8_t *codes, double *mins, double *maxs,
                     int32_t *status, void *scratch, size_t scratch_bytes, void *stream);
/* compression.unpack minus the file I/O: fp32 positions from the planes (bit-exact), every
 * group dequantised in fp64 (mins (1 - t) + maxs t, t = code / 255) and rounded to fp32. */
int bsr_codec_decode(const uint8_t *planes, const uint8_t *codes, const double *mins, const double *maxs,
                     int64_t n, int32_t n_groups, const bsr_codec_group *groups /* host */, int32_t rows,
                     int32_t cols, float *flat, float *positions, void *stream);

/* ---- parity / debug: export the binning of the last forward (synchronises) ---------- */
/* order (V): compact index per depth rank (== np.argsort(depths, kind="stable"),
 * rasterizer.py:83-85, over the visible subset in source order); src_index (V): source
 * index of each compact primitive (batch.indices); bounds (V,4) compact order; lists (E):
 * compact index per tile entry (tile_bins, rasterizer.py:161-191); ranges (T,2): per-tile
 * [start, end).  Any pointer may be NULL. */
int bsr_debug_export(const void *frame, int64_t n, int32_t width, int32_t height,
                     int64_t entry_cap, int32_t *order, int32_t *src_index, int32_t *bounds,
                     int32_t *lists, int32_t *ranges, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BSR_H_ */
