// Training loss and optimizer kernels (sm_100a).
//
// loss (fit.py:94-108): L = (1 - lam) mean|p - t| + lam (1 - SSIM(p, t)) and its
// adjoint dL/dp = (1 - lam) sign(p - t) / size - lam dSSIM/dp.  SSIM follows
// baselines.py:116-203: 11-tap Gaussian window (sigma 1.5), zero-padded
// separable correlation, per-channel mean of the SSIM map over the interior
// crop [5:H-5, 5:W-5], C1 = 1e-4, C2 = 9e-4; its gradient is
//   F(g_ux) + 2 x F(g_vx) + y F(g_vxy)   (the window is self-adjoint),
// with g_* the per-pixel coefficient maps (non-zero on the interior only).
//
//   ssim_stats_kernel : per 32x32 tile and channel, the five filtered moments
//                       (two separable passes through shared memory), the
//                       SSIM map summed per tile (fixed order), and the three
//                       coefficient maps written to global memory.
//   ssim_grad_kernel  : filters the coefficient maps, adds the L1 term and
//                       writes the adjoint; per-tile |p - t| partial sums.
//   loss_finish_kernel: fixed-order reduction of the per-tile partials.
//
// adam_kernel: bias-corrected Adam (fit.py:144-160) on float64 parameters and
// moments with float32 gradients.
#include <cmath>

#include "kernels.cuh"

namespace splat {

namespace {

constexpr int kS = 32;            // output tile
constexpr int kR = 5;             // window radius
constexpr int kHalo = kS + 2 * kR;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;   // baselines.py:17-18

__constant__ float c_win[11];
__constant__ double c_wind[11];

// Moments x, y, x^2, y^2, xy of one channel, filtered in float64: the SSIM
// variances are differences of nearly equal second moments, and their float32
// rounding (amplified by cancellation in the splat-gradient sums) would exceed
// the 1e-3 gradient tolerance.  Inputs and the outputs' consumers stay float32.
constexpr size_t kStatsSmem = 2 * (size_t)kHalo * (kHalo + 1) * 4 + 5 * (size_t)kHalo * kS * 8;

// 1/x for x > 0: float32 reciprocal + two float64 Newton steps (~1 ulp)
__device__ __forceinline__ double rcp64(double x) {
    float f;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"((float)x));
    double r = (double)f;
    r = r * fma(-x, r, 2.0);
    r = r * fma(-x, r, 2.0);
    return r;
}

__global__ void __launch_bounds__(256, 3) ssim_stats_kernel(const float* __restrict__ pred,
                                                         const float* __restrict__ target, int w, int h,
                                                         double gscale, float* __restrict__ coef,
                                                         double* __restrict__ part_ssim) {
    extern __shared__ __align__(16) unsigned char sm[];
    float(*s_x)[kHalo + 1] = reinterpret_cast<float(*)[kHalo + 1]>(sm);
    float(*s_y)[kHalo + 1] = reinterpret_cast<float(*)[kHalo + 1]>(sm + (size_t)kHalo * (kHalo + 1) * 4);
    double* s_h = reinterpret_cast<double*>(sm + 2 * (size_t)kHalo * (kHalo + 1) * 4);   // [5][kHalo][kS]
    __shared__ double s_red[8];
    const int tid = threadIdx.x;
    // the three channel CTAs of a tile are adjacent in launch order, so the interleaved
    // (H, W, 3) pred / target sectors one of them fetches are L2 hits for the other two
    const int ch = blockIdx.x % 3, bx = blockIdx.x / 3, gx = gridDim.x / 3;
    const int X0 = bx * kS, Y0 = blockIdx.y * kS;
    double local = 0.0;
    // load the channel tile with a zero halo (zero padding: correlate1d mode="constant")
    for (int e = tid; e < kHalo * kHalo; e += 256) {
        const int r = e / kHalo, c = e - r * kHalo;
        const int gy = Y0 + r - kR, gx = X0 + c - kR;
        float xv = 0.f, yv = 0.f;
        if (gy >= 0 && gy < h && gx >= 0 && gx < w) {
            const size_t o = ((size_t)gy * w + gx) * 3 + ch;
            xv = pred[o];
            yv = target[o];
        }
        s_x[r][c] = xv;
        s_y[r][c] = yv;
    }
    __syncthreads();
    // horizontal pass, register-blocked: one (row, 4 consecutive columns) item per thread step
    for (int e = tid; e < kHalo * (kS / 4); e += 256) {
        const int r = e / (kS / 4), c0 = (e - r * (kS / 4)) * 4;
        double m[4][5];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 5; ++q) m[i][q] = 0.0;
#pragma unroll
        for (int t = 0; t < 14; ++t) {
            const double xv = s_x[r][c0 + t], yv = s_y[r][c0 + t];
            const double xx = xv * xv, yy = yv * yv, xy = xv * yv;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = t - i;
                if (k < 0 || k > 10) continue;
                const double wk = c_wind[k];
                m[i][0] = fma(wk, xv, m[i][0]);
                m[i][1] = fma(wk, yv, m[i][1]);
                m[i][2] = fma(wk, xx, m[i][2]);
                m[i][3] = fma(wk, yy, m[i][3]);
                m[i][4] = fma(wk, xy, m[i][4]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 5; ++q) s_h[((size_t)q * kHalo + r) * kS + c0 + i] = m[i][q];
    }
    __syncthreads();
    // vertical pass, register-blocked: thread = (column, 4 consecutive rows) -> exactly 256 items
    {
        const int c = tid & (kS - 1), r0 = (tid >> 5) * 4;
        double m[4][5];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 5; ++q) m[i][q] = 0.0;
#pragma unroll
        for (int t = 0; t < 14; ++t) {
            double hv[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) hv[q] = s_h[((size_t)q * kHalo + r0 + t) * kS + c];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = t - i;
                if (k < 0 || k > 10) continue;
                const double wk = c_wind[k];
#pragma unroll
                for (int q = 0; q < 5; ++q) m[i][q] = fma(wk, hv[q], m[i][q]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int gy = Y0 + r0 + i, gx = X0 + c;
            if (gy >= h || gx >= w) continue;
            const double ux = m[i][0], uy = m[i][1];
            const double sxx = m[i][2] - ux * ux, syy = m[i][3] - uy * uy, sxy = m[i][4] - ux * uy;
            const double n1 = 2.0 * ux * uy + kC1, n2 = 2.0 * sxy + kC2;
            const double d1 = ux * ux + uy * uy + kC1, d2 = sxx + syy + kC2;
            const bool interior = gy >= kR && gy < h - kR && gx >= kR && gx < w - kR;
            float gux = 0.f, gvx = 0.f, gvxy = 0.f;
            if (interior) {
                const double r1 = rcp64(d1), r2 = rcp64(d2);
                const double pq = n1 * r1, qq = n2 * r2;
                local += pq * qq;
                gux = (float)(gscale * (qq * (2.0 * uy * d1 - 2.0 * ux * n1) * (r1 * r1) +
                                        pq * (-2.0 * uy * r2 + 2.0 * ux * n2 * (r2 * r2))));
                gvx = (float)(gscale * pq * (-n2 * (r2 * r2)));
                gvxy = (float)(gscale * pq * (2.0 * r2));
            }
            // planar coefficient maps [(ch * 3 + q)][H][W]: coalesced stores and loads
            const size_t hw = (size_t)h * w, o = (size_t)gy * w + gx;
            coef[(size_t)(ch * 3) * hw + o] = gux;
            coef[(size_t)(ch * 3 + 1) * hw + o] = gvx;
            coef[(size_t)(ch * 3 + 2) * hw + o] = gvxy;
        }
    }
    // fixed-order block reduction of the SSIM map sum
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
    if ((tid & 31) == 0) s_red[tid >> 5] = local;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int i = 0; i < 8; ++i) t += s_red[i];
        part_ssim[((size_t)ch * gridDim.y + blockIdx.y) * gx + bx] = t;
    }
}

__global__ void __launch_bounds__(256) ssim_grad_kernel(const float* __restrict__ pred,
                                                        const float* __restrict__ target, int w, int h,
                                                        const float* __restrict__ coef, float l1_scale,
                                                        float lam, float* __restrict__ adj,
                                                        float* __restrict__ part_l1) {
    __shared__ float s_c[3][kHalo][kHalo + 1];
    __shared__ float s_h[3][kHalo][kS + 1];
    __shared__ float s_red[8];
    const int tid = threadIdx.x;
    // the three channel CTAs of a tile are adjacent in launch order, so the interleaved
    // (H, W, 3) pred / target sectors one of them fetches are L2 hits for the other two
    const int ch = blockIdx.x % 3, bx = blockIdx.x / 3, gx = gridDim.x / 3;
    const int X0 = bx * kS, Y0 = blockIdx.y * kS;
    float local = 0.f;
    for (int e = tid; e < kHalo * kHalo; e += 256) {
        const int r = e / kHalo, c = e - r * kHalo;
        const int gy = Y0 + r - kR, gx = X0 + c - kR;
        float a = 0.f, b = 0.f, d = 0.f;
        if (gy >= 0 && gy < h && gx >= 0 && gx < w) {
            const size_t hw = (size_t)h * w, o = (size_t)gy * w + gx;
            a = coef[(size_t)(ch * 3) * hw + o];
            b = coef[(size_t)(ch * 3 + 1) * hw + o];
            d = coef[(size_t)(ch * 3 + 2) * hw + o];
        }
        s_c[0][r][c] = a;
        s_c[1][r][c] = b;
        s_c[2][r][c] = d;
    }
    __syncthreads();
    // horizontal pass, register-blocked: (row, 4 consecutive columns) per item
    for (int e = tid; e < kHalo * (kS / 4); e += 256) {
        const int r = e / (kS / 4), c0 = (e - r * (kS / 4)) * 4;
        float m[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 3; ++q) m[i][q] = 0.f;
#pragma unroll
        for (int t = 0; t < 14; ++t) {
            float v[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) v[q] = s_c[q][r][c0 + t];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = t - i;
                if (k < 0 || k > 10) continue;
                const float wk = c_win[k];
#pragma unroll
                for (int q = 0; q < 3; ++q) m[i][q] = fmaf(wk, v[q], m[i][q]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 3; ++q) s_h[q][r][c0 + i] = m[i][q];
    }
    __syncthreads();
    // vertical pass, register-blocked: (column, 4 consecutive rows) per thread
    {
        const int c = tid & (kS - 1), r0 = (tid >> 5) * 4;
        float m[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 3; ++q) m[i][q] = 0.f;
#pragma unroll
        for (int t = 0; t < 14; ++t) {
            float v[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) v[q] = s_h[q][r0 + t][c];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = t - i;
                if (k < 0 || k > 10) continue;
                const float wk = c_win[k];
#pragma unroll
                for (int q = 0; q < 3; ++q) m[i][q] = fmaf(wk, v[q], m[i][q]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int gy = Y0 + r0 + i, gx = X0 + c;
            if (gy >= h || gx >= w) continue;
            const size_t o = ((size_t)gy * w + gx) * 3 + ch;
            const float x = pred[o], y = target[o];
            const float dssim = m[i][0] + 2.f * x * m[i][1] + y * m[i][2];
            const float diff = x - y;
            const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
            adj[o] = l1_scale * sgn - lam * dssim;
            local += fabsf(diff);
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
    if ((tid & 31) == 0) s_red[tid >> 5] = local;
    __syncthreads();
    if (tid == 0) {
        float t = 0.f;
        for (int i = 0; i < 8; ++i) t += s_red[i];
        part_l1[((size_t)ch * gridDim.y + blockIdx.y) * gx + bx] = t;
    }
}

// value = (1 - lam) * sum|d| / size + lam * (1 - mean_c(sum_ssim_c / inner))
// 3 x 256 threads: channel c = threadIdx.x / 256 sums its partials with stride 256,
// then fixed-order warp and block reductions (deterministic).
__global__ void __launch_bounds__(768) loss_finish_kernel(const double* __restrict__ part_ssim,
                                                          const float* __restrict__ part_l1, int nparts_per_ch,
                                                          double size, double inner, double lam,
                                                          double* __restrict__ value) {
    __shared__ double s[3][8][2];
    const int ch = threadIdx.x >> 8, i0 = threadIdx.x & 255, lane = threadIdx.x & 31, wid = i0 >> 5;
    double ss = 0.0, l1 = 0.0;
    for (int i = i0; i < nparts_per_ch; i += 256) {
        ss += part_ssim[(size_t)ch * nparts_per_ch + i];
        l1 += (double)part_l1[(size_t)ch * nparts_per_ch + i];
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, d);
        l1 += __shfl_xor_sync(0xffffffffu, l1, d);
    }
    if (lane == 0) {
        s[ch][wid][0] = ss;
        s[ch][wid][1] = l1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ssim = 0.0, l1t = 0.0;
        for (int c = 0; c < 3; ++c) {
            double sc = 0.0, lc = 0.0;
            for (int w = 0; w < 8; ++w) {
                sc += s[c][w][0];
                lc += s[c][w][1];
            }
            ssim += sc / inner;
            l1t += lc;
        }
        ssim /= 3.0;
        value[0] = (1.0 - lam) * (l1t / size) + (lam > 0.0 ? lam * (1.0 - ssim) : 0.0);
        value[1] = ssim;
    }
}

__global__ void adam_kernel(double* __restrict__ p, const float* __restrict__ g, double* __restrict__ m,
                            double* __restrict__ v, int64_t count, double lr, double b1, double b2,
                            double bc1, double bc2, double eps) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double gi = (double)g[i];
    const double mi = b1 * m[i] + (1.0 - b1) * gi;
    const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] = p[i] - lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
}

// dst += src (float32): folds per-stream gradient buffers into one, in a fixed order.
__global__ void accumulate_kernel(float* __restrict__ dst, const float* __restrict__ src, int64_t n) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i + 3 < n) {
        float4 a = *reinterpret_cast<const float4*>(dst + i);
        const float4 b = *reinterpret_cast<const float4*>(src + i);
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
        *reinterpret_cast<float4*>(dst + i) = a;
    } else {
        for (int64_t k = i; k < n; ++k) dst[k] += src[k];
    }
}

}  // namespace

int accumulate_impl(float* dst, const float* src, int64_t n, cudaStream_t stream) {
    if (n <= 0) return SPLAT_OK;
    const int64_t threads = (n + 3) / 4;
    accumulate_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(dst, src, n); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

size_t loss_workspace_bytes_impl(int w, int h) {
    size_t nparts = (size_t)ceil_div(w, kS) * ceil_div(h, kS) * 3;
    return (size_t)w * h * 9 * 4 + 16 + nparts * 3 * 8 + nparts * 3 * 4 + 256;
}

int loss_impl(const float* pred, const float* target, int w, int h, double lam, float* adj, double* value,
              void* ws, cudaStream_t stream) {
    static PerDevice<bool> win_set;   // __constant__ tables and attributes are per device
    bool ok = false;
    const int rc = win_set.get(ok, [](bool& v) {
        double wd[11], sum = 0.0;
        for (int k = 0; k < 11; ++k) {
            const double x = k - 5;
            wd[k] = std::exp(-(x * x) / (2.0 * 1.5 * 1.5));
            sum += wd[k];
        }
        float wf[11];
        for (int k = 0; k < 11; ++k) {
            wd[k] /= sum;
            wf[k] = (float)wd[k];
        }
        SPLAT_CUDA_CHECK(cudaMemcpyToSymbol(c_win, wf, sizeof(wf)));
        SPLAT_CUDA_CHECK(cudaMemcpyToSymbol(c_wind, wd, sizeof(wd)));
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(ssim_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)kStatsSmem));
        v = true;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    const int gx = ceil_div(w, kS), gy = ceil_div(h, kS);
    const size_t nparts = (size_t)gx * gy;
    float* coef = (float*)ws;
    double* part_ssim = (double*)((char*)ws + (((size_t)w * h * 9 * 4 + 15) & ~(size_t)15));
    float* part_l1 = (float*)(part_ssim + nparts * 3);
    const double inner = (double)(h - 2 * kR) * (double)(w - 2 * kR);
    const double size = (double)w * h * 3;
    const double gscale = 1.0 / (inner * 3.0);
    dim3 grid(3 * gx, gy);   // channel fastest (see ssim_stats_kernel)
    if (lam > 0.0) {
        ssim_stats_kernel<<<grid, 256, kStatsSmem, stream>>>(pred, target, w, h, gscale, coef, part_ssim); note_launch();
    } else {
        SPLAT_CUDA_CHECK(cudaMemsetAsync(coef, 0, (size_t)w * h * 9 * 4, stream));
        SPLAT_CUDA_CHECK(cudaMemsetAsync(part_ssim, 0, nparts * 3 * 8, stream));
    }
    ssim_grad_kernel<<<grid, 256, 0, stream>>>(pred, target, w, h, coef, (float)((1.0 - lam) / size), (float)lam,
                                               adj, part_l1); note_launch();
    loss_finish_kernel<<<1, 768, 0, stream>>>(part_ssim, part_l1, (int)nparts, size, inner, lam, value);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int adam_impl(double* p, const float* g, double* m, double* v, int64_t count, double lr, double b1, double b2,
              double bc1, double bc2, double eps, cudaStream_t stream) {
    if (count <= 0) return SPLAT_OK;
    adam_kernel<<<(unsigned)((count + 255) / 256), 256, 0, stream>>>(p, g, m, v, count, lr, b1, b2, bc1, bc2,
                                                                      eps); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

}  // namespace splat
