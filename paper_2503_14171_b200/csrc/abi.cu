// extern "C" boundary of libsplat_b200.so (declared in include/splat_b200.h).
#include <cstdio>
#include <atomic>
#include <cstring>

#include "kernels.cuh"

namespace splat {

static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int set_error(int code, const char* msg) {
    std::snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

int set_cuda_error(cudaError_t e, const char* what) {
    std::snprintf(g_err, sizeof(g_err), "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return SPLAT_ERR_CUDA;
}

int device_sms(int& sms) {
    static PerDevice<int> cache;
    return cache.get(sms, [](int& v) {
        int dev = 0;
        SPLAT_CUDA_CHECK(cudaGetDevice(&dev));
        SPLAT_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return SPLAT_OK;
    });
}

size_t scene_workspace_bytes_impl(int64_t n);
int scene_prepare_impl(const splat_scene_t& s, void* const_buf, void* ws, cudaStream_t stream);
int scene_refresh_impl(const splat_scene_t& s, void* const_buf, cudaStream_t stream);
int launch_pack64(const SceneConst& sc, const ViewConst& vc, double* out, cudaStream_t stream);
size_t backward_workspace_bytes_impl(int64_t n, int64_t cap);
size_t loss_workspace_bytes_impl(int w, int h);
int loss_impl(const float* pred, const float* target, int w, int h, double lam, float* adj, double* value,
              void* ws, cudaStream_t stream);
int adam_groups_impl(int ngroups, double* const* p, const float* const* g, double* const* m, double* const* v,
                     const int64_t* count, const double* lr, double b1, double b2, double bc1, double bc2, double eps,
                     cudaStream_t stream);
int adam_impl(double* p, const float* g, double* m, double* v, int64_t count, double lr, double b1, double b2,
              double bc1, double bc2, double eps, cudaStream_t stream);
int launch_raster_backward(const SceneConst& sc, const splat_scene_t& scene, const ViewConst& vc,
                           const FrameLayout& L, char* ws, const splat_gimg_t& fwd, const float* adj,
                           char* bws, float* grads, int accumulate, cudaStream_t stream, float* rank_out);
int launch_chain(const SceneConst& sc, const splat_scene_t& scene, const float* rank_grads, float* grads,
                 int accumulate, cudaStream_t stream);
int upscale_forward_impl(const float* src, int in_w, int in_h, float* out, int out_w, int out_h,
                         int clamp, const void* plan, cudaStream_t stream);
size_t upscale_plan_bytes_impl(int out_w, int out_h);
int upscale_plan_impl(int in_w, int in_h, int out_w, int out_h, void* plan, cudaStream_t stream);
int upscale_backward_impl(const float* adj, int out_w, int out_h, float* dsrc, int in_w, int in_h,
                          cudaStream_t stream);
int fd_forward_impl(const float* img, int w, int h, float* planes, cudaStream_t stream);
int fd_backward_impl(const float* dplanes, int w, int h, float* tmp, float* out, cudaStream_t stream);

int gimg_pack_impl(const float* planes, const float* alpha, int w, int h, float* out, cudaStream_t stream);
int gimg_unpack_impl(const float* in, int w, int h, float* planes, float* alpha, int32_t* count,
                     cudaStream_t stream);
int encode_display_impl(const float* img, int64_t n, uint8_t* out, cudaStream_t stream);
int accumulate_impl(float* dst, const float* src, int64_t n, cudaStream_t stream);
int points_impl(const double* pack, const double* colors, const uint8_t* valid, int64_t n, const double* xs,
                const double* ys, int64_t npts, const double* bg, double* out, uint8_t* state,
                cudaStream_t stream);
int project_impl(int64_t n, const double* mu, const double* ls3, const double* quat, const double* logit,
                 const splat_camera_t& cam, double* means2, double* ls2, double* rot2, double* logit_out,
                 double* depth, cudaStream_t stream);

static int check_dims(int width, int height) {
    if (width <= 0 || height <= 0)
        return set_error(SPLAT_ERR_DIMENSION, "output dimensions must be positive");
    if (width > 32767 || height > 32767)
        return set_error(SPLAT_ERR_DIMENSION, "render dimensions above 32767 are not supported");
    return SPLAT_OK;
}

}  // namespace splat

using namespace splat;

extern "C" {

const char* splat_last_error(void) { return g_err; }
int splat_abi_version(void) { return SPLAT_ABI_VERSION; }
uint64_t splat_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }
int splat_build_checked(void) { return SPLAT_CHECKS; }

size_t splat_scene_const_bytes(int64_t n) { return const_layout(n).total; }
size_t splat_scene_workspace_bytes(int64_t n) { return scene_workspace_bytes_impl(n); }

int splat_scene_prepare(const splat_scene_t* scene, void* const_buf, size_t const_bytes, void* workspace,
                        size_t ws_bytes, void* stream) {
    if (!scene || scene->n < 0) return set_error(SPLAT_ERR_PARAMETER, "invalid scene");
    if (scene->n >= (int64_t)1 << 31) return set_error(SPLAT_ERR_PARAMETER, "too many splats");
    if (const_bytes < const_layout(scene->n).total || ws_bytes < scene_workspace_bytes_impl(scene->n))
        return set_error(SPLAT_ERR_PARAMETER, "scene buffers too small");
    return scene_prepare_impl(*scene, const_buf, workspace, (cudaStream_t)stream);
}

int splat_scene_refresh(const splat_scene_t* scene, void* const_buf, size_t const_bytes, void* stream) {
    if (!scene || scene->n < 0) return set_error(SPLAT_ERR_PARAMETER, "invalid scene");
    if (const_bytes < const_layout(scene->n).total) return set_error(SPLAT_ERR_PARAMETER, "scene buffer too small");
    return scene_refresh_impl(*scene, const_buf, (cudaStream_t)stream);
}

const int32_t* splat_scene_order(const void* const_buf, int64_t n) {
    return scene_const_view(const_buf, n).order;
}

size_t splat_frame_workspace_bytes(int64_t n, int width, int height, int64_t pair_capacity) {
    return frame_layout(n, width, height, pair_capacity).total;
}

int splat_frame_pointers(void* workspace, int64_t n, int width, int height, int64_t pair_capacity,
                         splat_frame_ptrs_t* out) {
    FrameLayout L = frame_layout(n, width, height, pair_capacity);
    char* w = (char*)workspace;
    out->bboxes = (int16_t*)(w + L.bboxes);
    out->touched = (uint32_t*)(w + L.touched);
    out->offsets = (uint32_t*)(w + L.offsets);
    out->keys = (uint32_t*)(w + L.keys0);
    out->ranks = (uint32_t*)(w + L.vals0);
    out->ranges = (uint32_t*)(w + L.ranges);
    out->counters = (uint32_t*)(w + L.counters);
    out->fixup = (uint32_t*)(w + L.fixup);
    out->pack = (float*)(w + L.pack);
    return SPLAT_OK;
}

int splat_prepare_view(const void* scene_const, int64_t n, const splat_view_t* view, int width,
                       int height, void* workspace, size_t ws_bytes, int64_t pair_capacity, void* stream) {
    int rc = check_dims(width, height);
    if (rc) return rc;
    FrameLayout L = frame_layout(n, width, height, pair_capacity);
    if (ws_bytes < L.total) return set_error(SPLAT_ERR_PARAMETER, "frame workspace too small");
    if ((uintptr_t)workspace & 255) return set_error(SPLAT_ERR_PARAMETER, "frame workspace must be 256-byte aligned");
    return launch_preprocess(scene_const_view(scene_const, n), make_view_const(*view), L, (char*)workspace,
                             (cudaStream_t)stream);
}

int splat_bin_tiles(int64_t n, int width, int height, void* workspace, size_t ws_bytes,
                    int64_t pair_capacity, int flags, void* stream) {
    int rc = check_dims(width, height);
    if (rc) return rc;
    FrameLayout L = frame_layout(n, width, height, pair_capacity);
    if (ws_bytes < L.total) return set_error(SPLAT_ERR_PARAMETER, "frame workspace too small");
    if ((uintptr_t)workspace & 255) return set_error(SPLAT_ERR_PARAMETER, "frame workspace must be 256-byte aligned");
    return launch_binning(L, (char*)workspace, flags, (cudaStream_t)stream);
}

int splat_view_pack64(const void* scene_const, int64_t n, const splat_view_t* view, double* pack64,
                      void* stream) {
    return launch_pack64(scene_const_view(scene_const, n), make_view_const(*view), pack64,
                         (cudaStream_t)stream);
}

int splat_render_forward(const void* scene_const, int64_t n, const splat_view_t* view, int width, int height,
                         int train, const splat_gimg_t* out, void* workspace, size_t ws_bytes,
                         int64_t pair_capacity, void* stream) {
    int rc = check_dims(width, height);
    if (rc) return rc;
    if (train && !out->state) return set_error(SPLAT_ERR_PARAMETER, "train mode needs the state buffer");
    FrameLayout L = frame_layout(n, width, height, pair_capacity);
    if (ws_bytes < L.total) return set_error(SPLAT_ERR_PARAMETER, "frame workspace too small");
    if ((uintptr_t)workspace & 255) return set_error(SPLAT_ERR_PARAMETER, "frame workspace must be 256-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    SceneConst sc = scene_const_view(scene_const, n);
    ViewConst vc = make_view_const(*view);
    char* w = (char*)workspace;
    if ((rc = launch_preprocess(sc, vc, L, w, s))) return rc;
    if ((rc = launch_binning(L, w, train ? SPLAT_BIN_OFFSETS : 0, s))) return rc;
    return launch_raster_forward(sc, vc, L, w, *out, train != 0, s);
}

int splat_rasterize(const void* scene_const, int64_t n, const splat_view_t* view, int width, int height,
                    int train, const splat_gimg_t* out, void* workspace, size_t ws_bytes,
                    int64_t pair_capacity, void* stream) {
    int rc = check_dims(width, height);
    if (rc) return rc;
    const bool tr = train & 1, defer = train & SPLAT_RASTER_DEFER_FIXUP;
    if (tr && !out->state) return set_error(SPLAT_ERR_PARAMETER, "train mode needs the state buffer");
    FrameLayout L = frame_layout(n, width, height, pair_capacity);
    if (ws_bytes < L.total) return set_error(SPLAT_ERR_PARAMETER, "frame workspace too small");
    if ((uintptr_t)workspace & 255) return set_error(SPLAT_ERR_PARAMETER, "frame workspace must be 256-byte aligned");
    return launch_raster_forward(scene_const_view(scene_const, n), make_view_const(*view), L,
                                 (char*)workspace, *out, tr, (cudaStream_t)stream, !defer);
}
int splat_fixup(const void* scene_const, int64_t n, const splat_view_t* view, int width, int height, int train,
                const splat_gimg_t* out, void* workspace, size_t ws_bytes, int64_t pair_capacity, void* stream) {
    int rc = check_dims(width, height);
    if (rc) return rc;
    if ((train & 1) && !out->state) return set_error(SPLAT_ERR_PARAMETER, "train mode needs the state buffer");
    FrameLayout L = frame_layout(n, width, height, pair_capacity);
    if (ws_bytes < L.total) return set_error(SPLAT_ERR_PARAMETER, "frame workspace too small");
    if ((uintptr_t)workspace & 255) return set_error(SPLAT_ERR_PARAMETER, "frame workspace must be 256-byte aligned");
    return launch_fixup(scene_const_view(scene_const, n), make_view_const(*view), L, (char*)workspace, *out,
                        (train & 1) != 0, (cudaStream_t)stream);
}

size_t splat_upscale_plan_bytes(int in_w, int in_h, int out_w, int out_h) {
    (void)in_w;
    (void)in_h;
    return upscale_plan_bytes_impl(out_w, out_h);
}

int splat_upscale_plan(int in_w, int in_h, int out_w, int out_h, void* plan, void* stream) {
    if (in_w <= 0 || in_h <= 0) return set_error(SPLAT_ERR_DIMENSION, "empty source image");
    if (out_w < in_w || out_h < in_h)
        return set_error(SPLAT_ERR_SCALE, "output must be at least source size");
    return upscale_plan_impl(in_w, in_h, out_w, out_h, plan, (cudaStream_t)stream);
}

size_t splat_backward_workspace_bytes(int64_t n, int64_t pair_capacity) {
    return backward_workspace_bytes_impl(n, pair_capacity);
}

int splat_render_backward(const void* scene_const, const splat_scene_t* scene, const splat_view_t* view,
                          int width, int height, const splat_gimg_t* fwd, const float* adjoint, void* workspace,
                          size_t ws_bytes, int64_t pair_capacity, void* bwd_workspace, size_t bwd_bytes,
                          float* grads, int accumulate, void* stream) {
    int rc = check_dims(width, height);
    if (rc) return rc;
    if (!fwd || !fwd->state || !fwd->last)
        return set_error(SPLAT_ERR_PARAMETER, "backward needs a training-mode forward (state + last)");
    FrameLayout L = frame_layout(scene->n, width, height, pair_capacity);
    if (ws_bytes < L.total) return set_error(SPLAT_ERR_PARAMETER, "frame workspace too small");
    if ((uintptr_t)workspace & 255) return set_error(SPLAT_ERR_PARAMETER, "frame workspace must be 256-byte aligned");
    if (bwd_bytes < backward_workspace_bytes_impl(scene->n, pair_capacity))
        return set_error(SPLAT_ERR_PARAMETER, "backward workspace too small");
    return launch_raster_backward(scene_const_view(scene_const, scene->n), *scene, make_view_const(*view), L,
                                  (char*)workspace, *fwd, adjoint, (char*)bwd_workspace, grads, accumulate,
                                  (cudaStream_t)stream, nullptr);
}

int splat_render_backward_rank(const void* scene_const, const splat_scene_t* scene, const splat_view_t* view,
                               int width, int height, const splat_gimg_t* fwd, const float* adjoint,
                               void* workspace, size_t ws_bytes, int64_t pair_capacity, void* bwd_workspace,
                               size_t bwd_bytes, float* rank_grads, int accumulate, void* stream) {
    int rc = check_dims(width, height);
    if (rc) return rc;
    if (!fwd || !fwd->state || !fwd->last)
        return set_error(SPLAT_ERR_PARAMETER, "backward needs a training-mode forward (state + last)");
    FrameLayout L = frame_layout(scene->n, width, height, pair_capacity);
    if (ws_bytes < L.total) return set_error(SPLAT_ERR_PARAMETER, "frame workspace too small");
    if ((uintptr_t)workspace & 255) return set_error(SPLAT_ERR_PARAMETER, "frame workspace must be 256-byte aligned");
    if (bwd_bytes < backward_workspace_bytes_impl(scene->n, pair_capacity))
        return set_error(SPLAT_ERR_PARAMETER, "backward workspace too small");
    return launch_raster_backward(scene_const_view(scene_const, scene->n), *scene, make_view_const(*view), L,
                                  (char*)workspace, *fwd, adjoint, (char*)bwd_workspace, nullptr, accumulate,
                                  (cudaStream_t)stream, rank_grads);
}

int splat_chain_grads(const void* scene_const, const splat_scene_t* scene, const float* rank_grads, float* grads,
                      int accumulate, void* stream) {
    return launch_chain(scene_const_view(scene_const, scene->n), *scene, rank_grads, grads, accumulate,
                        (cudaStream_t)stream);
}

size_t splat_loss_workspace_bytes(int width, int height) { return loss_workspace_bytes_impl(width, height); }

int splat_loss(const float* pred, const float* target, int width, int height, double ssim_weight, float* adjoint,
               double* value, void* workspace, size_t ws_bytes, void* stream) {
    if (width <= 0 || height <= 0) return set_error(SPLAT_ERR_DIMENSION, "empty image");
    if (ssim_weight < 0.0 || ssim_weight > 1.0) return set_error(SPLAT_ERR_PARAMETER, "ssim_weight must be in [0, 1]");
    if (ssim_weight > 0.0 && (width < 11 || height < 11))
        return set_error(SPLAT_ERR_DIMENSION, "ssim requires images of at least 11 pixels per side");
    if (ws_bytes < loss_workspace_bytes_impl(width, height))
        return set_error(SPLAT_ERR_PARAMETER, "loss workspace too small");
    return loss_impl(pred, target, width, height, ssim_weight, adjoint, value, workspace, (cudaStream_t)stream);
}

int splat_adam_step(double* params, const float* grads, double* m, double* v, int64_t count, double lr,
                    double beta1, double beta2, double bc1, double bc2, double eps, void* stream) {
    return adam_impl(params, grads, m, v, count, lr, beta1, beta2, bc1, bc2, eps, (cudaStream_t)stream);
}

int splat_adam_step_groups(int ngroups, double* const* params, const float* const* grads, double* const* m,
                           double* const* v, const int64_t* counts, const double* lrs, double beta1, double beta2,
                           double bc1, double bc2, double eps, void* stream) {
    if (!params || !grads || !m || !v || !counts || !lrs) return set_error(SPLAT_ERR_PARAMETER, "null group arrays");
    return adam_groups_impl(ngroups, params, grads, m, v, counts, lrs, beta1, beta2, bc1, bc2, eps,
                            (cudaStream_t)stream);
}

int splat_render_views(const void* scene_const, int64_t n, const splat_view_t* views, int nviews, int width,
                       int height, const splat_slot_t* slots, int nslots, float* const* outs, int out_w, int out_h,
                       int clamp, const void* plan) {
    int rc = check_dims(width, height);
    if (rc) return rc;
    if (nviews < 0 || (nviews > 0 && (!views || !slots || nslots <= 0 || !outs)))
        return set_error(SPLAT_ERR_PARAMETER, "invalid view batch");
    if (!plan) return set_error(SPLAT_ERR_PARAMETER, "upscale plan required (splat_upscale_plan)");
    if (out_w < width || out_h < height) return set_error(SPLAT_ERR_SCALE, "output must be at least source size");
    if (n > 0 && nviews > 0 && !scene_const) return set_error(SPLAT_ERR_PARAMETER, "scene constants required");
    for (int i = 0; i < nviews; ++i)
        if (!outs[i]) return set_error(SPLAT_ERR_PARAMETER, "null output frame in the batch");
    for (int k = 0; k < nslots && k < nviews; ++k) {
        const splat_slot_t& sl = slots[k];
        const FrameLayout L = frame_layout(n, width, height, sl.pair_capacity);
        if (sl.ws_bytes < L.total) return set_error(SPLAT_ERR_PARAMETER, "frame workspace too small");
        if ((uintptr_t)sl.workspace & 255) return set_error(SPLAT_ERR_PARAMETER, "frame workspace must be 256-byte aligned");
        if ((uintptr_t)sl.image.planes & 15) return set_error(SPLAT_ERR_PARAMETER, "image planes must be 16-byte aligned");
    }
    const SceneConst sc = scene_const_view(scene_const, n);
    for (int i = 0; i < nviews; ++i) {
        const splat_slot_t& sl = slots[i % nslots];
        const FrameLayout L = frame_layout(n, width, height, sl.pair_capacity);
        const ViewConst vc = make_view_const(views[i]);
        char* w = (char*)sl.workspace;
        cudaStream_t s = (cudaStream_t)sl.stream;
        if ((out_w & 3) == 0 && ((uintptr_t)outs[i] & 15)) return set_error(SPLAT_ERR_PARAMETER, "output must be 16-byte aligned");
        if ((rc = launch_preprocess(sc, vc, L, w, s))) return rc;
        if ((rc = launch_binning(L, w, 0, s))) return rc;
        if ((rc = launch_raster_forward(sc, vc, L, w, sl.image, false, s))) return rc;
        if ((rc = upscale_forward_impl(sl.image.planes, width, height, outs[i], out_w, out_h, clamp, plan, s))) return rc;
    }
    return SPLAT_OK;
}

int splat_upscale_forward(const float* src, int in_w, int in_h, float* out, int out_w, int out_h, int clamp,
                          const void* plan, void* stream) {
    if (in_w <= 0 || in_h <= 0) return set_error(SPLAT_ERR_DIMENSION, "empty source image");
    if (out_w < in_w || out_h < in_h)
        return set_error(SPLAT_ERR_SCALE, "output must be at least source size");
    if (!plan) return set_error(SPLAT_ERR_PARAMETER, "upscale plan required (splat_upscale_plan)");
    // source rows are staged with 16-byte bulk copies; rows of out_w % 4 == 0 frames are
    // written with 16-byte (bulk / vector) stores
    if ((uintptr_t)src & 15) return set_error(SPLAT_ERR_PARAMETER, "source planes must be 16-byte aligned");
    if ((out_w & 3) == 0 && ((uintptr_t)out & 15))
        return set_error(SPLAT_ERR_PARAMETER, "output must be 16-byte aligned");
    return upscale_forward_impl(src, in_w, in_h, out, out_w, out_h, clamp, plan, (cudaStream_t)stream);
}

int splat_upscale_backward(const float* adjoint, int out_w, int out_h, float* dsrc, int in_w, int in_h,
                           void* stream) {
    if (in_w <= 0 || in_h <= 0) return set_error(SPLAT_ERR_DIMENSION, "empty source image");
    if (out_w < in_w || out_h < in_h)
        return set_error(SPLAT_ERR_SCALE, "output must be at least source size");
    return upscale_backward_impl(adjoint, out_w, out_h, dsrc, in_w, in_h, (cudaStream_t)stream);
}

int splat_fd_gradients(const float* image, int width, int height, float* planes, void* stream) {
    if (width < 2 || height < 2)
        return set_error(SPLAT_ERR_DIMENSION, "finite differences need at least 2x2 pixels");
    return fd_forward_impl(image, width, height, planes, (cudaStream_t)stream);
}

int splat_fd_gradients_backward(const float* dplanes, int width, int height, float* dimage,
                                float* scratch, void* stream) {
    if (width < 2 || height < 2)
        return set_error(SPLAT_ERR_DIMENSION, "finite differences need at least 2x2 pixels");
    return fd_backward_impl(dplanes, width, height, scratch, dimage, (cudaStream_t)stream);
}

int splat_gimg_pack(const float* planes, const float* alpha, int width, int height, float* out, void* stream) {
    if (width <= 0 || height <= 0) return set_error(SPLAT_ERR_DIMENSION, "image dimensions must be positive");
    return gimg_pack_impl(planes, alpha, width, height, out, (cudaStream_t)stream);
}

int splat_gimg_unpack(const float* in, int width, int height, float* planes, float* alpha, int32_t* count,
                      void* stream) {
    if (width <= 0 || height <= 0) return set_error(SPLAT_ERR_DIMENSION, "image dimensions must be positive");
    return gimg_unpack_impl(in, width, height, planes, alpha, count, (cudaStream_t)stream);
}

int splat_project_3d(int64_t n, const double* means3, const double* log_scales3, const double* quats,
                     const double* opacity_logits, const splat_camera_t* camera, double* means2,
                     double* log_scales2, double* rotations, double* opacity_logits_out, double* depths,
                     void* stream) {
    if (n < 0) return set_error(SPLAT_ERR_DIMENSION, "negative splat count");
    if (!camera) return set_error(SPLAT_ERR_PARAMETER, "camera is required");
    if (!(camera->fx > 0.0) || !(camera->fy > 0.0) || !(camera->near_plane > 0.0))
        return set_error(SPLAT_ERR_PARAMETER, "camera focal lengths and near plane must be positive");
    return project_impl(n, means3, log_scales3, quats, opacity_logits, *camera, means2, log_scales2, rotations,
                        opacity_logits_out, depths, (cudaStream_t)stream);
}

int splat_render_points(const double* pack64, const double* colors, const uint8_t* valid, int64_t n,
                        const double* xs, const double* ys, int64_t npts, const double* background, double* out,
                        uint8_t* state, void* stream) {
    if (n < 0 || npts < 0) return set_error(SPLAT_ERR_DIMENSION, "negative size");
    return points_impl(pack64, colors, valid, n, xs, ys, npts, background, out, state, (cudaStream_t)stream);
}

int splat_grad_accumulate(float* dst, const float* src, int64_t count, void* stream) {
    if (count < 0) return set_error(SPLAT_ERR_DIMENSION, "negative element count");
    return accumulate_impl(dst, src, count, (cudaStream_t)stream);
}

int splat_encode_display(const float* image, int64_t count, uint8_t* out, void* stream) {
    if (count < 0) return set_error(SPLAT_ERR_DIMENSION, "negative element count");
    return encode_display_impl(image, count, out, (cudaStream_t)stream);
}

}  // extern "C"
