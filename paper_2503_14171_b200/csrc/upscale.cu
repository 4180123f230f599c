// Bicubic Hermite spline upscaler (forward and exact transpose) for sm_100a.
//
// upscale_spline (spline.py:145-178): per unit subdomain F = C A C^T built
// from the four corner pixels' value / d/dx / d/dy / d2/dxdy planes (border
// corners replicate the edge pixel, spline.py:115-142), evaluated at the
// centre-aligned source coordinate s = (u + .5) / (n_out / n_in) - .5
// (spline.py:102-112).  Written here in the equivalent Hermite-basis form
// out = sum_k sum_l hx_k(tx) hy_l(ty) F[k, l], factored as a y pass shared by
// every output pixel of a row (G) followed by a 4-term x pass, then clamped
// to [0, 1] (spline.py:178).
//
// Memory: the source is the packed (H, W, 4, 3) float32 gradient image (48 B
// per pixel).  A CTA owns an 8 x 128 output tile; the source rectangle it
// needs is staged into shared memory with bulk async copies (TMA,
// cp.async.bulk -> UBLKCP) on an mbarrier, one copy per source row.  Output
// rows are written with 16-byte vector stores.  The kernel is HBM-bound:
// 12 B per output pixel written + 48 B per source pixel read.
//
// upscale_backward (spline.py:191-243) is the gather-form transpose: one CTA
// per 8 x 16 source tile first contracts the adjoint along x for every output
// row it influences, then along y, writing each source pixel's 12 adjoints
// exactly once — no atomics, deterministic.
#include <cmath>

#include "kernels.cuh"

namespace splat {

namespace {

constexpr int kUpRows = 8;
constexpr int kUpCols = 128;

struct AxisMap {
    int i0;        // floor(s)
    float h[4];    // Hermite weights: value@0, value@1, slope@0, slope@1
};

__device__ __forceinline__ AxisMap axis_map(int u, double scale) {
    // spline.py:106-111, float64 like numpy: s = (u + .5) / scale - .5
    double s = __dsub_rn(__ddiv_rn((double)u + 0.5, scale), 0.5);
    double f = floor(s);
    double t = s - f;
    double t2 = t * t, t3 = t2 * t;
    AxisMap m;
    m.i0 = (int)f;
    m.h[0] = (float)(1.0 - 3.0 * t2 + 2.0 * t3);
    m.h[1] = (float)(3.0 * t2 - 2.0 * t3);
    m.h[2] = (float)(t - 2.0 * t2 + t3);
    m.h[3] = (float)(t3 - t2);
    return m;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(256) upscale_fwd_kernel(const float* __restrict__ src, int in_w,
                                                          int in_h, float* __restrict__ out, int out_w,
                                                          int out_h, double scale_x, double scale_y,
                                                          int clamp, int span_cols, int span_rows) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ AxisMap s_cmap[kUpCols];
    __shared__ AxisMap s_rmap[kUpRows];
    __shared__ int s_box[4];
    __shared__ __align__(8) unsigned long long s_bar;

    const int tid = threadIdx.x;
    const int U0 = blockIdx.x * kUpCols, V0 = blockIdx.y * kUpRows;
    float* s_src = reinterpret_cast<float*>(smem);                 // span_rows x span_cols x 12
    float* s_g = s_src + (size_t)span_rows * span_cols * 12;       // kUpRows x span_cols x 6

    if (tid < kUpCols) {
        int u = min(U0 + tid, out_w - 1);
        s_cmap[tid] = axis_map(u, scale_x);
    } else if (tid < kUpCols + kUpRows) {
        int v = min(V0 + tid - kUpCols, out_h - 1);
        s_rmap[tid - kUpCols] = axis_map(v, scale_y);
    }
    if (tid == 0) {
        int ulast = min(U0 + kUpCols, out_w) - 1, vlast = min(V0 + kUpRows, out_h) - 1;
        AxisMap a = axis_map(U0, scale_x), b = axis_map(ulast, scale_x);
        AxisMap c = axis_map(V0, scale_y), d = axis_map(vlast, scale_y);
        s_box[0] = clampi(a.i0, 0, in_w - 1);
        s_box[1] = clampi(b.i0 + 1, 0, in_w - 1);
        s_box[2] = clampi(c.i0, 0, in_h - 1);
        s_box[3] = clampi(d.i0 + 1, 0, in_h - 1);
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const int x0 = s_box[0], ncols = s_box[1] - s_box[0] + 1;
    const int y0 = s_box[2], nrows = s_box[3] - s_box[2] + 1;

    // TMA bulk copies: one contiguous source row segment (ncols * 48 B) per row
    if (tid == 0) {
        uint32_t bytes = (uint32_t)(ncols * 48) * (uint32_t)nrows;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar)),
                     "r"(bytes)
                     : "memory");
        for (int r = 0; r < nrows; ++r) {
            const float* g = src + ((size_t)(y0 + r) * in_w + x0) * 12;
            float* d = s_src + (size_t)r * span_cols * 12;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(d)),
                "l"(g), "r"((uint32_t)(ncols * 48)), "r"(smem_u32(&s_bar))
                : "memory");
        }
    }
    // wait for the transaction bytes (phase 0)
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                : "=r"(done)
                : "r"(smem_u32(&s_bar))
                : "memory");
        }
    }

    // y pass: G[v][x] = (value-in-x, slope-in-x) along output row v
    const int nv = min(kUpRows, out_h - V0);
    for (int e = tid; e < nv * ncols; e += blockDim.x) {
        int v = e / ncols, x = e - v * ncols;
        const AxisMap& rm = s_rmap[v];
        int ra = clampi(rm.i0, 0, in_h - 1) - y0, rb = clampi(rm.i0 + 1, 0, in_h - 1) - y0;
        const float* pa = s_src + ((size_t)ra * span_cols + x) * 12;
        const float* pb = s_src + ((size_t)rb * span_cols + x) * 12;
        float* gd = s_g + ((size_t)v * span_cols + x) * 6;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            // value planes: f and f_y ; slope planes: f_x and f_xy
            gd[c] = rm.h[0] * pa[c] + rm.h[1] * pb[c] + rm.h[2] * pa[6 + c] + rm.h[3] * pb[6 + c];
            gd[3 + c] = rm.h[0] * pa[3 + c] + rm.h[1] * pb[3 + c] + rm.h[2] * pa[9 + c] + rm.h[3] * pb[9 + c];
        }
    }
    __syncthreads();

    // x pass: each thread writes 4 consecutive output pixels of one row
    const int v = tid >> 5;
    const int ug = (tid & 31) * 4;
    if (v < nv) {
        const int vrow = V0 + v;
        float o[12];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const AxisMap& cm = s_cmap[ug + i];
            int xa = clampi(cm.i0, 0, in_w - 1) - x0, xb = clampi(cm.i0 + 1, 0, in_w - 1) - x0;
            const float* ga = s_g + ((size_t)v * span_cols + xa) * 6;
            const float* gb = s_g + ((size_t)v * span_cols + xb) * 6;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float val = cm.h[0] * ga[c] + cm.h[1] * gb[c] + cm.h[2] * ga[3 + c] + cm.h[3] * gb[3 + c];
                if (clamp) val = fminf(fmaxf(val, 0.f), 1.f);
                o[3 * i + c] = val;
            }
        }
        const int u = U0 + ug;
        float* dst = out + ((size_t)vrow * out_w + u) * 3;
        if (u + 3 < out_w && (out_w & 3) == 0) {
            float4* d4 = reinterpret_cast<float4*>(dst);
            d4[0] = make_float4(o[0], o[1], o[2], o[3]);
            d4[1] = make_float4(o[4], o[5], o[6], o[7]);
            d4[2] = make_float4(o[8], o[9], o[10], o[11]);
        } else {
            for (int i = 0; i < 4 && u + i < out_w; ++i)
                for (int c = 0; c < 3; ++c) dst[3 * i + c] = o[3 * i + c];
        }
    }
}

// ---- backward -----------------------------------------------------------------

constexpr int kBwRows = 16;
constexpr int kBwCols = 16;

// First and last output index whose floor(s) lies in [lo, hi] (monotone map).
__device__ int first_out_with_i0_ge(int lo, int n_out, double scale) {
    // smallest u with i0(u) >= lo
    double guess = floor(((double)lo + 0.5) * scale - 0.5) - 2.0;
    int u = guess < 0 ? 0 : (int)guess;
    while (u < n_out && axis_map(u, scale).i0 < lo) ++u;
    while (u > 0 && axis_map(u - 1, scale).i0 >= lo) --u;
    return u;
}

__global__ void __launch_bounds__(256) upscale_bwd_kernel(const float* __restrict__ adj, int out_w,
                                                          int out_h, float* __restrict__ dsrc, int in_w,
                                                          int in_h, double scale_x, double scale_y,
                                                          int max_u, int max_v) {
    extern __shared__ __align__(16) unsigned char smem[];
    // layout: umap[max_u], vmap[max_v], dG[max_v][kBwCols][6]
    AxisMap* s_umap = reinterpret_cast<AxisMap*>(smem);
    AxisMap* s_vmap = s_umap + max_u;
    float* s_dg = reinterpret_cast<float*>(s_vmap + max_v);
    __shared__ int s_rng[4];
    __shared__ int s_cu[kBwCols][2];

    const int tid = threadIdx.x;
    const int X0 = blockIdx.x * kBwCols, Y0 = blockIdx.y * kBwRows;
    const int X1 = min(X0 + kBwCols, in_w) - 1, Y1 = min(Y0 + kBwRows, in_h) - 1;
    if (tid == 0) {
        // outputs touching source columns [X0, X1]: i0 in [X0 - 1, X1] (edge clamps included)
        int ulo = first_out_with_i0_ge(X0 - 1, out_w, scale_x);
        int uhi = first_out_with_i0_ge(X1 + 1, out_w, scale_x);
        if (X0 == 0) ulo = 0;
        if (X1 == in_w - 1) uhi = out_w;
        int vlo = first_out_with_i0_ge(Y0 - 1, out_h, scale_y);
        int vhi = first_out_with_i0_ge(Y1 + 1, out_h, scale_y);
        if (Y0 == 0) vlo = 0;
        if (Y1 == in_h - 1) vhi = out_h;
        s_rng[0] = ulo;
        s_rng[1] = min(uhi, ulo + max_u);
        s_rng[2] = vlo;
        s_rng[3] = min(vhi, vlo + max_v);
    }
    __syncthreads();
    const int ulo = s_rng[0], nu = s_rng[1] - s_rng[0];
    const int vlo = s_rng[2], nv = s_rng[3] - s_rng[2];
    for (int i = tid; i < nu; i += blockDim.x) s_umap[i] = axis_map(ulo + i, scale_x);
    for (int i = tid; i < nv; i += blockDim.x) s_vmap[i] = axis_map(vlo + i, scale_y);
    __syncthreads();
    if (tid < kBwCols) {
        // u range (within [ulo, ulo+nu)) whose corners can hit column X0 + tid
        int x = X0 + tid, a = nu, b = 0;
        for (int i = 0; i < nu; ++i) {
            int xa = clampi(s_umap[i].i0, 0, in_w - 1), xb = clampi(s_umap[i].i0 + 1, 0, in_w - 1);
            if (xa == x || xb == x) {
                a = min(a, i);
                b = max(b, i + 1);
            }
        }
        s_cu[tid][0] = a;
        s_cu[tid][1] = b;
    }
    __syncthreads();
    // x contraction: dG[v][x] (value part, slope part) for every output row v
    const int ncx = X1 - X0 + 1;
    for (int e = tid; e < nv * ncx; e += blockDim.x) {
        int vi = e / ncx, xi = e - vi * ncx;
        int x = X0 + xi;
        const float* arow = adj + (size_t)(vlo + vi) * out_w * 3;
        float dv[3] = {0.f, 0.f, 0.f}, ds[3] = {0.f, 0.f, 0.f};
        for (int i = s_cu[xi][0]; i < s_cu[xi][1]; ++i) {
            const AxisMap& m = s_umap[i];
            int xa = clampi(m.i0, 0, in_w - 1), xb = clampi(m.i0 + 1, 0, in_w - 1);
            float w0 = (xa == x ? m.h[0] : 0.f) + (xb == x ? m.h[1] : 0.f);
            float w1 = (xa == x ? m.h[2] : 0.f) + (xb == x ? m.h[3] : 0.f);
            const float* a = arow + (size_t)(ulo + i) * 3;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float g = a[c];
                dv[c] = fmaf(w0, g, dv[c]);
                ds[c] = fmaf(w1, g, ds[c]);
            }
        }
        float* d = s_dg + ((size_t)vi * kBwCols + xi) * 6;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            d[c] = dv[c];
            d[3 + c] = ds[c];
        }
    }
    __syncthreads();
    // y contraction: one source pixel per thread
    const int yi = tid / kBwCols, xi = tid % kBwCols;
    const int y = Y0 + yi, x = X0 + xi;
    if (y <= Y1 && x <= X1) {
        float f[3] = {0, 0, 0}, fx[3] = {0, 0, 0}, fy[3] = {0, 0, 0}, fxy[3] = {0, 0, 0};
        for (int vi = 0; vi < nv; ++vi) {
            const AxisMap& m = s_vmap[vi];
            int ya = clampi(m.i0, 0, in_h - 1), yb = clampi(m.i0 + 1, 0, in_h - 1);
            if (ya != y && yb != y) continue;
            float w0 = (ya == y ? m.h[0] : 0.f) + (yb == y ? m.h[1] : 0.f);
            float w1 = (ya == y ? m.h[2] : 0.f) + (yb == y ? m.h[3] : 0.f);
            const float* d = s_dg + ((size_t)vi * kBwCols + xi) * 6;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                f[c] = fmaf(w0, d[c], f[c]);
                fy[c] = fmaf(w1, d[c], fy[c]);
                fx[c] = fmaf(w0, d[3 + c], fx[c]);
                fxy[c] = fmaf(w1, d[3 + c], fxy[c]);
            }
        }
        float4* o = reinterpret_cast<float4*>(dsrc + ((size_t)y * in_w + x) * 12);
        o[0] = make_float4(f[0], f[1], f[2], fx[0]);
        o[1] = make_float4(fx[1], fx[2], fy[0], fy[1]);
        o[2] = make_float4(fy[2], fxy[0], fxy[1], fxy[2]);
    }
}

// ---- finite-difference derivative planes (spline.py:246-297) -----------------

__device__ __forceinline__ float diff1(const float* f, int i, int n, int stride) {
    // central difference, one-sided at the borders (spline.py:246-253)
    if (i == 0) return f[stride] - f[0];
    if (i == n - 1) return f[(size_t)(n - 1) * stride] - f[(size_t)(n - 2) * stride];
    return 0.5f * (f[(size_t)(i + 1) * stride] - f[(size_t)(i - 1) * stride]);
}

__global__ void fd_kernel(const float* __restrict__ img, int w, int h, float* __restrict__ planes) {
    int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    float out[12];
    for (int c = 0; c < 3; ++c) {
        const float* base = img + c;
        out[c] = base[((size_t)y * w + x) * 3];
        out[3 + c] = diff1(base + (size_t)y * w * 3, x, w, 3);
        out[6 + c] = diff1(base + (size_t)x * 3, y, h, w * 3);
        // d_dxdy = diff_x(diff_y(image)) (spline.py:285)
        auto dy_at = [&](int xx) { return diff1(base + (size_t)xx * 3, y, h, w * 3); };
        float v;
        if (x == 0) v = dy_at(1) - dy_at(0);
        else if (x == w - 1) v = dy_at(w - 1) - dy_at(w - 2);
        else v = 0.5f * (dy_at(x + 1) - dy_at(x - 1));
        out[9 + c] = v;
    }
    float4* o = reinterpret_cast<float4*>(planes + ((size_t)y * w + x) * 12);
    o[0] = make_float4(out[0], out[1], out[2], out[3]);
    o[1] = make_float4(out[4], out[5], out[6], out[7]);
    o[2] = make_float4(out[8], out[9], out[10], out[11]);
}

// transpose of diff1 along one axis, evaluated at index i (spline.py:256-264)
__device__ __forceinline__ float diff1_t(const float* g, int i, int n, int stride) {
    float v = 0.f;
    if (i - 1 >= 1 && i - 1 <= n - 2) v += 0.5f * g[(size_t)(i - 1) * stride];
    if (i + 1 >= 1 && i + 1 <= n - 2) v -= 0.5f * g[(size_t)(i + 1) * stride];
    if (i == 1) v += g[0];
    if (i == 0) v -= g[0];
    if (i == n - 1) v += g[(size_t)(n - 1) * stride];
    if (i == n - 2) v -= g[(size_t)(n - 1) * stride];
    return v;
}

// tmp = Dx^T d_dxdy (per channel, (H,W,3))
__global__ void fd_bwd_x_kernel(const float* __restrict__ dplanes, int w, int h, float* __restrict__ tmp) {
    int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    for (int c = 0; c < 3; ++c)
        tmp[((size_t)y * w + x) * 3 + c] = diff1_t(dplanes + (size_t)y * w * 12 + 9 + c, x, w, 12);
}

// out = d_color + Dx^T d_dx + Dy^T (d_dy + tmp)
__global__ void fd_bwd_kernel(const float* __restrict__ dplanes, const float* __restrict__ tmp, int w,
                              int h, float* __restrict__ out) {
    int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    for (int c = 0; c < 3; ++c) {
        size_t o = ((size_t)y * w + x);
        float v = dplanes[o * 12 + c];
        v += diff1_t(dplanes + (size_t)y * w * 12 + 3 + c, x, w, 12);
        v += diff1_t(dplanes + (size_t)x * 12 + 6 + c, y, h, w * 12);
        v += diff1_t(tmp + (size_t)x * 3 + c, y, h, w * 3);
        out[o * 3 + c] = v;
    }
}

}  // namespace

int upscale_forward_impl(const float* src, int in_w, int in_h, float* out, int out_w, int out_h,
                         int clamp, cudaStream_t stream) {
    if (out_w <= 0 || out_h <= 0) return SPLAT_OK;
    double sx = (double)out_w / (double)in_w, sy = (double)out_h / (double)in_h;
    int span_cols = (int)ceil(kUpCols / sx) + 3;
    int span_rows = (int)ceil(kUpRows / sy) + 3;
    if (span_cols > in_w) span_cols = in_w;
    if (span_rows > in_h) span_rows = in_h;
    size_t smem = (size_t)span_rows * span_cols * 12 * 4 + (size_t)kUpRows * span_cols * 6 * 4;
    static int configured = 0;
    if (!configured) {
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(upscale_fwd_kernel,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = 1;
    }
    if (smem > 200 * 1024) return set_error(SPLAT_ERR_DIMENSION, "upscale tile exceeds shared memory");
    dim3 grid(ceil_div(out_w, kUpCols), ceil_div(out_h, kUpRows));
    upscale_fwd_kernel<<<grid, 256, smem, stream>>>(src, in_w, in_h, out, out_w, out_h, sx, sy, clamp,
                                                    span_cols, span_rows); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int upscale_backward_impl(const float* adj, int out_w, int out_h, float* dsrc, int in_w, int in_h,
                          cudaStream_t stream) {
    double sx = (double)out_w / (double)in_w, sy = (double)out_h / (double)in_h;
    int max_u = (int)ceil((kBwCols + 2) * sx) + 8;
    int max_v = (int)ceil((kBwRows + 2) * sy) + 8;
    size_t smem = (size_t)(max_u + max_v) * sizeof(AxisMap) + (size_t)max_v * kBwCols * 6 * 4;
    static int configured = 0;
    if (!configured) {
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(upscale_bwd_kernel,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = 1;
    }
    if (smem > 200 * 1024) return set_error(SPLAT_ERR_DIMENSION, "upscale backward tile too large");
    dim3 grid(ceil_div(in_w, kBwCols), ceil_div(in_h, kBwRows));
    upscale_bwd_kernel<<<grid, 256, smem, stream>>>(adj, out_w, out_h, dsrc, in_w, in_h, sx, sy, max_u,
                                                    max_v); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int fd_forward_impl(const float* img, int w, int h, float* planes, cudaStream_t stream) {
    dim3 grid(ceil_div(w, 128), h);
    fd_kernel<<<grid, 128, 0, stream>>>(img, w, h, planes); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int fd_backward_impl(const float* dplanes, int w, int h, float* tmp, float* out, cudaStream_t stream) {
    dim3 grid(ceil_div(w, 128), h);
    fd_bwd_x_kernel<<<grid, 128, 0, stream>>>(dplanes, w, h, tmp); note_launch();
    fd_bwd_kernel<<<grid, 128, 0, stream>>>(dplanes, tmp, w, h, out); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

}  // namespace splat
