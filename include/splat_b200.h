/*
 * splat_b200 — C ABI of the B200 (sm_100a) gradient-aware render + spline
 * upscale path.  libsplat_b200.so exports exactly the functions below.
 *
 * Conventions
 *  - Every pointer argument is DEVICE memory unless the comment says "host".
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *    default stream), performs no host synchronisation and allocates nothing:
 *    scratch comes from caller-provided workspaces sized by the *_bytes query.
 *  - Return value: SPLAT_OK or one of the error codes; splat_last_error()
 *    gives the message (thread-local).  The Python layer maps the codes onto
 *    the reference exception classes (splinesplat core.py:28-41).
 *  - Images are row-major HWC float32.  A "gradient image" is the packed
 *    (H, W, 4, 3) buffer [color, d_dx, d_dy, d_dxdy] plus planar (4, H, W)
 *    alpha state and an (H, W) int32 contrib_count — the fields of the
 *    reference GradientImage (raster_forward.py:27-40) in float32.
 *
 * Each entry point cites the reference interface it replaces (file:line in
 * /root/reference/pkg/src/splinesplat).  INTEGRATION.md shows the ctypes
 * binding.
 */
#ifndef SPLAT_B200_H
#define SPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPLAT_OK 0
#define SPLAT_ERR_DIMENSION 1   /* DimensionError        (core.py:36) */
#define SPLAT_ERR_PARAMETER 2   /* ParameterError        (core.py:28) */
#define SPLAT_ERR_SCALE 3       /* UnsupportedScaleError (core.py:40) */
#define SPLAT_ERR_CAPACITY 4    /* tile-pair buffer too small: retry larger */
#define SPLAT_ERR_CUDA 100      /* CUDA runtime error (message in splat_last_error) */

#define SPLAT_ABI_VERSION 1

/* Storage-order scene on the device: the reference Scene arrays
 * (core.py:75-93) as float64.  n may be 0. */
typedef struct {
    int64_t n;
    const double *means;          /* (n,2) */
    const double *log_scales;     /* (n,2) */
    const double *rotations;      /* (n)   */
    const double *opacity_logits; /* (n)   */
    const double *colors;         /* (n,3) */
    const double *depths;         /* (n)   */
} splat_scene_t;

/* Pinhole camera for the 3D front-end: world -> camera
 * x_c = R x_w + t (R row-major), pixel = (fx x/z + cx, fy y/z + cy) on the
 * camera image, points with z <= near_plane are culled. */
typedef struct {
    double R[9];
    double t[3];
    double fx, fy, cx, cy;
    double near_plane;
} splat_camera_t;

/* One camera view (host values).  The render of view v at W x H equals the
 * reference render_forward of Scene(means - (ox, oy), ..., reference_resolution
 * = (W/kx_ratio...)) with kx = out_w / ref_w, ky = out_h / ref_h exactly as
 * prepare_scene computes them (raster_forward.py:81-85). */
typedef struct {
    double kx, ky;     /* render-resolution scale per axis */
    double ox, oy;     /* pan, subtracted from means before scaling */
    double bg[3];      /* background colour (Scene.background) */
} splat_view_t;

/* Caller-owned outputs of one render (a GradientImage). */
typedef struct {
    float *planes;     /* (H,W,4,3) color, d_dx, d_dy, d_dxdy */
    float *alpha;      /* (4,H,W) alpha, alpha_dx, alpha_dy, alpha_dxdy */
    int32_t *count;    /* (H,W) contrib_count */
    uint32_t *last;    /* (H,W) private: tile-list end of the last contributor */
    double *state;     /* (H,W,4) private float64 terminal (T, A_x, A_y, A_xy); NULL = inference */
} splat_gimg_t;

/* Pointers into a frame workspace (for inspection / the stage-level API). */
typedef struct {
    int16_t *bboxes;        /* (n,4) x0,x1,y0,y1 half-open, rank order (prepare_scene bboxes) */
    uint32_t *touched;      /* (n) tiles touched per rank, 0 when invalid */
    uint32_t *offsets;      /* (n+1) exclusive scan of touched */
    uint32_t *keys;         /* (capacity) tile id per pair (only with SPLAT_BIN_KEYS) */
    uint32_t *ranks;        /* (capacity) sorted rank per pair */
    uint32_t *ranges;       /* (ntiles,2) [start,end) into keys/ranks */
    uint32_t *counters;     /* [0]=pairs [1]=overflow [2]=fix-up pixels [3]=raster work cursor;
                               [4]=sticky overflow (never cleared by the library: the caller
                               zeroes it); [5]=tiles too long for the shared-memory sort */
    uint32_t *fixup;        /* (H*W) pixels re-rendered by the exact float64 pass */
    float *pack;            /* (n,16) float32 per-view pack */
} splat_frame_ptrs_t;

const char *splat_last_error(void);
int splat_abi_version(void);
/* Number of kernels this library has launched since load (all streams). */
uint64_t splat_kernel_launches(void);
/* 1 for the checked build (device-side SPLAT_DCHECK bounds / protocol checks, `make checked`), else 0. */
int splat_build_checked(void);

/* ---- per-scene preparation (view independent) --------------------------
 * Stable depth argsort (raster_forward.py:59-61) and the view-independent
 * float64 terms of prepare_scene (raster_forward.py:86-110): e^{-2l}, cos,
 * sin, sigma = logistic(logit), q = log(max(sigma*255,1)), n00/n01/n11, e1*e2. */
size_t splat_scene_const_bytes(int64_t n);
size_t splat_scene_workspace_bytes(int64_t n);
int splat_scene_prepare(const splat_scene_t *scene, void *const_buf, size_t const_bytes,
                        void *workspace, size_t ws_bytes, void *stream);
/* Recompute the view-independent terms after a parameter update, keeping the
 * depth order already in const_buf (depths are not optimised, fit.py:163-166). */
int splat_scene_refresh(const splat_scene_t *scene, void *const_buf, size_t const_bytes, void *stream);
/* rank -> storage index (int32, n) inside const_buf (sort_by_depth output) */
const int32_t *splat_scene_order(const void *const_buf, int64_t n);

/* ---- per-view render with analytic gradients ---------------------------
 * render_forward (raster_forward.py:152-187): preprocess (prepare_scene),
 * tile binning with a device radix sort (bin_tiles), the 16x16-tile
 * front-to-back rasterizer (_kernels.forward_region, _kernels.py:32-129) and
 * an exact float64 re-render of pixels whose termination decision was too
 * close to call in float32.  train != 0 also writes the private float64
 * terminal state needed by splat_render_backward. */
size_t splat_frame_workspace_bytes(int64_t n, int width, int height, int64_t pair_capacity);
int splat_frame_pointers(void *workspace, int64_t n, int width, int height, int64_t pair_capacity,
                         splat_frame_ptrs_t *out /* host */);
int splat_render_forward(const void *scene_const, int64_t n, const splat_view_t *view /* host */,
                         int width, int height, int train, const splat_gimg_t *out /* host struct */,
                         void *workspace, size_t ws_bytes, int64_t pair_capacity, void *stream);
/* Stage-level entry points (inspection; the fused call above runs them all). */
int splat_prepare_view(const void *scene_const, int64_t n, const splat_view_t *view, int width,
                       int height, void *workspace, size_t ws_bytes, int64_t pair_capacity,
                       void *stream);
/* flags: SPLAT_BIN_OFFSETS also fills `offsets` (rank-major pair slots, needed by
 * splat_render_backward; splat_render_forward sets it when train != 0);
 * SPLAT_BIN_KEYS also fills `keys` (the tile id of every pair, for inspection —
 * the rasterizer only reads `ranges` and `ranks`). */
#define SPLAT_BIN_OFFSETS 1
#define SPLAT_BIN_KEYS 2
/* SPLAT_BIN_ATOMIC forces the binning path used for very large tile grids
 * (per-pair global atomics + per-tile sort); same output, for testing. */
#define SPLAT_BIN_ATOMIC 4
/* SPLAT_BIN_COUNT_ONLY stops after the per-tile counts: counters[0] = the pair count
 * (capacity calibration; no pairs are written, so any pair_capacity is accepted). */
#define SPLAT_BIN_COUNT_ONLY 8
int splat_bin_tiles(int64_t n, int width, int height, void *workspace, size_t ws_bytes,
                    int64_t pair_capacity, int flags, void *stream);
/* Rasterizer + exact fix-up pass alone, on a frame already prepared and binned
 * by the two calls above (render_forward = prepare_view + bin_tiles + rasterize).
 * `train`: bit 0 = training mode (float64 state); bit 1 (SPLAT_RASTER_DEFER_FIXUP) =
 * launch the raster kernel only, the caller then runs splat_fixup on the same stream
 * (stage timing: the two kernels have different rooflines). */
#define SPLAT_RASTER_DEFER_FIXUP 2
int splat_rasterize(const void *scene_const, int64_t n, const splat_view_t *view, int width,
                    int height, int train, const splat_gimg_t *out, void *workspace, size_t ws_bytes,
                    int64_t pair_capacity, void *stream);
/* The exact float64 re-render of the pixels splat_rasterize(..., train | SPLAT_RASTER_DEFER_FIXUP)
 * flagged (the reference's acc = acc + alpha (1 - acc) chain, _kernels.py:88-111). */
int splat_fixup(const void *scene_const, int64_t n, const splat_view_t *view, int width, int height,
                int train, const splat_gimg_t *out, void *workspace, size_t ws_bytes, int64_t pair_capacity,
                void *stream);
/* ---- view batches (the throughput path) ---------------------------------
 * One per-view workspace set; views are assigned round-robin (view i -> slot i % nslots) and
 * every view's prepare -> bin -> rasterize (+ fix-up) -> upscale chain is enqueued on its
 * slot's stream, in view order, with no host synchronisation: render_forward + upscale_spline
 * (raster_forward.py:152-187, spline.py:162-178) for a whole batch from one call (the
 * per-view host cost is the kernel launches only).  outs[i]: (out_h, out_w, 3) float32 frame
 * of view i; plan from splat_upscale_plan(width, height, out_w, out_h). */
typedef struct {
    void *workspace;        /* frame workspace (splat_frame_workspace_bytes), 256-byte aligned */
    size_t ws_bytes;
    int64_t pair_capacity;
    splat_gimg_t image;     /* the slot's GradientImage buffers (state may be NULL) */
    void *stream;
} splat_slot_t;
int splat_render_views(const void *scene_const, int64_t n, const splat_view_t *views, int nviews, int width,
                       int height, const splat_slot_t *slots, int nslots, float *const *outs, int out_w,
                       int out_h, int clamp, const void *plan);

/* Exact float64 RenderPack of a view (prepare_scene means/conics/sigmas,
 * raster_forward.py:86-102), rank order: pack64 (n,6) = mx,my,a,b,c,sigma;
 * colors64 (n,3) may be NULL.  Inspection only (the rasterizer uses float32). */
int splat_view_pack64(const void *scene_const, int64_t n, const splat_view_t *view, double *pack64,
                      void *stream);

/* render_at_points (raster_forward.py:190-233): blended colour (npts,3) float64
 * at arbitrary positions (render pixels), every valid splat in rank order with
 * the cull / clamp / early-termination rules; pack64 / valid from a prepared
 * view (splat_view_pack64, the frame's touched flags), colours (n,3) float64 in
 * rank order, background (3) host array.  state (npts, 2n) uint8 (may be NULL):
 * per point the splats that blended, then the ones clamped. */
int splat_render_points(const double *pack64, const double *colors, const uint8_t *valid, int64_t n,
                        const double *xs, const double *ys, int64_t npts, const double *background, double *out,
                        uint8_t *state, void *stream);

/* ---- reverse mode -------------------------------------------------------
 * render_backward (raster_backward.py:73-153) for a frame rendered with
 * train != 0 (its workspace still holds the bins): replays each pixel's
 * contributors back to front (_kernels.backward_region, _kernels.py:132-365),
 * reduces per-(splat, tile) partials in fixed order and chains them into the
 * stored parametrisation.  adjoint = (H,W,4,3) [w, wx, wy, wxy] (PixelAdjoint).
 * grads (float32, 11n) = [d_means (n,2) | d_log_scales (n,2) | d_rotations (n) |
 * d_opacity_logits (n) | d_colors (n,3)] in storage order; accumulate != 0 adds. */
size_t splat_backward_workspace_bytes(int64_t n, int64_t pair_capacity);
int splat_render_backward(const void *scene_const, const splat_scene_t *scene /* host struct */,
                          const splat_view_t *view /* host */, int width, int height,
                          const splat_gimg_t *fwd /* host struct */, const float *adjoint, void *workspace,
                          size_t ws_bytes, int64_t pair_capacity, void *bwd_workspace, size_t bwd_bytes,
                          float *grads, int accumulate, void *stream);
/* The same backward, stopping before the parametrisation chain: adds this
 * view's render-space terms per rank, (n, 9) float32 [d_colour(3), d_sigma-term,
 * d_mean (x kx, x ky), d_conic (/ kx^2, / kx ky, / ky^2)], into rank_grads
 * (accumulate != 0) or overwrites them.  Summed over views, one
 * splat_chain_grads maps them to parameter gradients: the multi-view training
 * step pays the chain (raster_backward.py:126-152) once, not once per view. */
int splat_render_backward_rank(const void *scene_const, const splat_scene_t *scene, const splat_view_t *view,
                               int width, int height, const splat_gimg_t *fwd, const float *adjoint,
                               void *workspace, size_t ws_bytes, int64_t pair_capacity, void *bwd_workspace,
                               size_t bwd_bytes, float *rank_grads, int accumulate, void *stream);
int splat_chain_grads(const void *scene_const, const splat_scene_t *scene, const float *rank_grads, float *grads,
                      int accumulate, void *stream);

/* ---- training loss and optimizer ----------------------------------------
 * loss (fit.py:94-108) with ssim_with_grad (baselines.py:170-203):
 * value[0] = (1-l) L1 + l (1 - SSIM), value[1] = SSIM (device float64);
 * adjoint (H,W,3) = dL/dpred.  pred/target are (H,W,3) float32. */
size_t splat_loss_workspace_bytes(int width, int height);
int splat_loss(const float *pred, const float *target, int width, int height, double ssim_weight,
               float *adjoint, double *value, void *workspace, size_t ws_bytes, void *stream);
/* adam_step (fit.py:144-160) on one parameter group: float64 params and
 * moments, float32 gradients; bc1/bc2 = 1 - beta^t computed by the caller. */
int splat_adam_step(double *params, const float *grads, double *m, double *v, int64_t count, double lr,
                    double beta1, double beta2, double bc1, double bc2, double eps, void *stream);
/* The same step over up to 8 groups in one launch (fit.py:144-160's loop over groups):
 * group k = (params[k], grads[k], m[k], v[k], counts[k] elements, lrs[k]). */
int splat_adam_step_groups(int ngroups, double *const *params, const float *const *grads, double *const *m,
                           double *const *v, const int64_t *counts, const double *lrs, double beta1, double beta2,
                           double bc1, double bc2, double eps, void *stream);

/* 3D EWA front-end: n 3D Gaussians (means (n,3), log_scales
 * (n,3), quaternions (n,4) w,x,y,z, opacity logits (n)) seen by `camera` ->
 * the 2D scene arrays (means (n,2) in camera-image pixels, log_scales (n,2),
 * rotations (n), opacity logits (n; -100 behind the near plane), depths (n) =
 * camera z) in the reference's 2D parametrisation (core.py:175-182), float64.
 * The colours pass through unchanged. */
int splat_project_3d(int64_t n, const double *means3, const double *log_scales3, const double *quats,
                     const double *opacity_logits, const splat_camera_t *camera, double *means2,
                     double *log_scales2, double *rotations, double *opacity_logits_out, double *depths,
                     void *stream);

/* dst += src over `count` floats: folds per-stream gradient buffers (views
 * rendered concurrently) into one in a fixed order (deterministic sum of the
 * per-view gradients, raster_backward.py's outputs summed over views). */
int splat_grad_accumulate(float *dst, const float *src, int64_t count, void *stream);

/* ---- spline upscaler ----------------------------------------------------
 * upscale_spline (spline.py:162-178): (H,W,4,3) gradient planes -> (Ho,Wo,3).
 * upscale_backward (spline.py:191-243): (Ho,Wo,3) adjoint -> (H,W,4,3). */
size_t splat_upscale_plan_bytes(int in_w, int in_h, int out_w, int out_h);
/* Per-axis maps (floor(s), Hermite weights) for one (in, out) size pair;
 * reusable by every upscale of that size (spline.py:102-112). */
int splat_upscale_plan(int in_w, int in_h, int out_w, int out_h, void *plan, void *stream);
int splat_upscale_forward(const float *src, int in_w, int in_h, float *out, int out_w, int out_h,
                          int clamp, const void *plan, void *stream);
int splat_upscale_backward(const float *adjoint, int out_w, int out_h, float *dsrc, int in_w,
                           int in_h, void *stream);
/* fd_gradients / fd_gradients_backward (spline.py:274-297). */
int splat_fd_gradients(const float *image, int width, int height, float *planes, void *stream);
int splat_fd_gradients_backward(const float *dplanes, int width, int height, float *dimage,
                                float *scratch /* (H,W,3) */, void *stream);

/* ---- wire formats --------------------------------------
 * GIMG gradient dump body (io.py:100-137 save/load_gradient_dump): 16 planar
 * float32 (H,W) planes — colour RGB, d_dx RGB, d_dy RGB, d_dxdy RGB, alpha,
 * alpha_dx, alpha_dy, alpha_dxdy — from / to the device layout (planes
 * (H,W,4,3), alpha (4,H,W)).  The caller writes / checks the 12-byte header.
 * unpack zeroes `count` (H,W) when it is non-NULL (a dump has no counts). */
int splat_gimg_pack(const float *planes, const float *alpha, int width, int height, float *out,
                    void *stream);
int splat_gimg_unpack(const float *in, int width, int height, float *planes, float *alpha, int32_t *count,
                      void *stream);
/* encode_display (io.py:28-31): clip [0,1], ^(1/2.2), x255, round half even -> uint8. */
int splat_encode_display(const float *image, int64_t count, uint8_t *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLAT_B200_H */
