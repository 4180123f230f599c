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
//
// A CTA owns a 32-column strip of one channel over kSegTiles tile rows and walks it
// down in 32-row chunks: each image row's horizontal moments are computed once
// (a ring of 42 rows in shared memory carries the 10 rows the next chunk's vertical
// window shares with this one), so the horizontal pass does 32 rows of work per
// 32 output rows instead of 42, in exactly one (row, 4 columns) item per thread;
// the next chunk's input rows land by cp.async while this chunk computes.
#ifndef SSIM_SEG_TILES
#define SSIM_SEG_TILES 6
#endif
#ifndef SSIM_PREFETCH
#define SSIM_PREFETCH 0   // 1: double-buffered input rows (76 KB: 2 CTAs/SM); 0: one buffer (65 KB: 3 CTAs/SM)
#endif
constexpr int kSegTiles = SSIM_SEG_TILES;
constexpr int kInBufs = SSIM_PREFETCH ? 2 : 1;
constexpr int kInStride = 45;   // = 1 mod 4: the four rows a warp's (row, 4 columns) items touch hit distinct banks
constexpr int kRing = kS + 2 * kR;   // 42 rows of horizontal moments
struct StatsSmem {
    float x[kInBufs][kS][kInStride];   // input rows of the current (/ next) chunk (x: pred, y: target)
    float y[kInBufs][kS][kInStride];
    double hm[5][kRing][kS];         // horizontal moments, ring over image rows
    double red[8];
};
constexpr size_t kStatsSmem = sizeof(StatsSmem);

__device__ __forceinline__ void cp_async4_zfill(void* smem, const void* gmem, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(valid ? 4 : 0)
                 : "memory");
}

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
    StatsSmem& S = *reinterpret_cast<StatsSmem*>(sm);
    const int tid = threadIdx.x;
    // the three channel CTAs of a strip are adjacent in launch order, so the interleaved
    // (H, W, 3) pred / target sectors one of them fetches are L2 hits for the other two
    const int ch = blockIdx.x % 3, bx = blockIdx.x / 3, gx = gridDim.x / 3;
    const int gy = (h + kS - 1) / kS;
    const int ty0 = blockIdx.y * kSegTiles, nchunks = min(kSegTiles, gy - ty0);
    const int X0 = bx * kS, Yseg = ty0 * kS;
    // input rows [gy0, gy0 + nrows) of the strip (+ halo columns), zero outside the image
    auto load_rows = [&](int buf, int gy0, int nrows) {
        for (int e = tid; e < nrows * kHalo; e += 256) {
            const int r = e / kHalo, c = e - r * kHalo;
            const int yy = gy0 + r, xx = X0 + c - kR;
            const bool ok = yy >= 0 && yy < h && xx >= 0 && xx < w;
            const size_t o = ok ? ((size_t)yy * w + xx) * 3 + ch : 0;
            cp_async4_zfill(&S.x[buf][r][c], pred + o, ok);
            cp_async4_zfill(&S.y[buf][r][c], target + o, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // horizontal moments of input rows [gy0, gy0 + nrows) (in buffer buf) into the ring
    auto hpass = [&](int buf, int gy0, int nrows) {
        for (int e = tid; e < nrows * (kS / 4); e += 256) {
            const int r = e / (kS / 4), c0 = (e - r * (kS / 4)) * 4;
            double m[4][5];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 5; ++q) m[i][q] = 0.0;
#pragma unroll
            for (int t = 0; t < 14; ++t) {
                const double xv = S.x[buf][r][c0 + t], yv = S.y[buf][r][c0 + t];
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
            const int slot = (gy0 + r - (Yseg - kR)) % kRing;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 5; ++q) S.hm[q][slot][c0 + i] = m[i][q];
        }
    };
    // the segment's top halo rows [Yseg - 5, Yseg + 5), then chunk 0's rows [Yseg + 5, Yseg + 37)
    load_rows(kInBufs - 1, Yseg - kR, 2 * kR);
    if (SSIM_PREFETCH) load_rows(0, Yseg + kR, kS);
    if (SSIM_PREFETCH) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    hpass(kInBufs - 1, Yseg - kR, 2 * kR);
    if (SSIM_PREFETCH) asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    for (int k = 0; k < nchunks; ++k) {
        const int y0 = Yseg + k * kS, b = SSIM_PREFETCH ? (k & 1) : 0;
        if (SSIM_PREFETCH) {
            if (k + 1 < nchunks) load_rows(b ^ 1, y0 + kS + kR, kS);   // buffer b^1 was read before the last barrier
        } else {
            load_rows(0, y0 + kR, kS);   // the buffer was read before the last barrier
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
        }
        hpass(b, y0 + kR, kS);
        __syncthreads();
        // vertical pass, register-blocked: thread = (column, 4 consecutive rows) -> exactly 256 items
        double local = 0.0;
        {
            const int c = tid & (kS - 1), r0 = (tid >> 5) * 4;
            const int base = y0 + r0 - kR - (Yseg - kR);   // ring index of the window's first row
            double m[4][5];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 5; ++q) m[i][q] = 0.0;
#pragma unroll
            for (int t = 0; t < 14; ++t) {
                const int slot = (base + t) % kRing;
                double hv[5];
#pragma unroll
                for (int q = 0; q < 5; ++q) hv[q] = S.hm[q][slot][c];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int kk = t - i;
                    if (kk < 0 || kk > 10) continue;
                    const double wk = c_wind[kk];
#pragma unroll
                    for (int q = 0; q < 5; ++q) m[i][q] = fma(wk, hv[q], m[i][q]);
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int yy = y0 + r0 + i, xx = X0 + c;
                if (yy >= h || xx >= w) continue;
                const double ux = m[i][0], uy = m[i][1];
                const double sxx = m[i][2] - ux * ux, syy = m[i][3] - uy * uy, sxy = m[i][4] - ux * uy;
                const double n1 = 2.0 * ux * uy + kC1, n2 = 2.0 * sxy + kC2;
                const double d1 = ux * ux + uy * uy + kC1, d2 = sxx + syy + kC2;
                const bool interior = yy >= kR && yy < h - kR && xx >= kR && xx < w - kR;
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
                const size_t hw = (size_t)h * w, o = (size_t)yy * w + xx;
                coef[(size_t)(ch * 3) * hw + o] = gux;
                coef[(size_t)(ch * 3 + 1) * hw + o] = gvx;
                coef[(size_t)(ch * 3 + 2) * hw + o] = gvxy;
            }
        }
        // fixed-order block reduction of the chunk's (= one 32x32 tile's) SSIM map sum
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
        if ((tid & 31) == 0) S.red[tid >> 5] = local;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int i = 0; i < 8; ++i) t += S.red[i];
            part_ssim[((size_t)ch * gy + ty0 + k) * gx + bx] = t;
        }
        // (the next chunk's hpass overwrites ring rows this chunk's vertical pass read;
        //  its S.red writes come after the next barrier)
        __syncthreads();
    }
}

// The gradient filter walks the same strips: the three coefficient maps' horizontal
// passes go to a 42-row ring, one 32-row chunk (= one output tile) at a time.
struct GradSmem {
    float c[2][3][kS][kInStride];   // coefficient-map rows of the current / next chunk (+ halo columns)
    float h[3][kRing][kS + 1];   // horizontal passes, ring over image rows
    float red[8];
};

__global__ void __launch_bounds__(256) ssim_grad_kernel(const float* __restrict__ pred,
                                                        const float* __restrict__ target, int w, int h,
                                                        const float* __restrict__ coef, float l1_scale,
                                                        float lam, float* __restrict__ adj,
                                                        float* __restrict__ part_l1) {
    extern __shared__ __align__(16) unsigned char gsm[];
    GradSmem& S = *reinterpret_cast<GradSmem*>(gsm);
    const int tid = threadIdx.x;
    // the three channel CTAs of a strip are adjacent in launch order, so the interleaved
    // (H, W, 3) pred / target sectors one of them fetches are L2 hits for the other two
    const int ch = blockIdx.x % 3, bx = blockIdx.x / 3, gx = gridDim.x / 3;
    const int gy = (h + kS - 1) / kS;
    const int ty0 = blockIdx.y * kSegTiles, nchunks = min(kSegTiles, gy - ty0);
    const int X0 = bx * kS, Yseg = ty0 * kS;
    const size_t hw = (size_t)h * w;
    auto load_rows = [&](int buf, int gy0, int nrows) {
        for (int e = tid; e < nrows * kHalo; e += 256) {
            const int r = e / kHalo, c = e - r * kHalo;
            const int yy = gy0 + r, xx = X0 + c - kR;
            const bool ok = yy >= 0 && yy < h && xx >= 0 && xx < w;
            const size_t o = ok ? (size_t)yy * w + xx : 0;
#pragma unroll
            for (int q = 0; q < 3; ++q)
                cp_async4_zfill(&S.c[buf][q][r][c], coef + (size_t)(ch * 3 + q) * hw + o, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // horizontal pass, register-blocked: (row, 4 consecutive columns) per item
    auto hpass = [&](int buf, int gy0, int nrows) {
        for (int e = tid; e < nrows * (kS / 4); e += 256) {
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
                for (int q = 0; q < 3; ++q) v[q] = S.c[buf][q][r][c0 + t];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int k = t - i;
                    if (k < 0 || k > 10) continue;
                    const float wk = c_win[k];
#pragma unroll
                    for (int q = 0; q < 3; ++q) m[i][q] = fmaf(wk, v[q], m[i][q]);
                }
            }
            const int slot = (gy0 + r - (Yseg - kR)) % kRing;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 3; ++q) S.h[q][slot][c0 + i] = m[i][q];
        }
    };
    load_rows(1, Yseg - kR, 2 * kR);   // the segment's top halo rows, then chunk 0's rows
    load_rows(0, Yseg + kR, kS);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    hpass(1, Yseg - kR, 2 * kR);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    for (int k = 0; k < nchunks; ++k) {
        const int y0 = Yseg + k * kS, b = k & 1;
        if (k + 1 < nchunks) load_rows(b ^ 1, y0 + kS + kR, kS);   // buffer b^1 was read before the last barrier
        // this thread's output pixels' pred / target, loaded before the filter passes
        const int c = tid & (kS - 1), r0 = (tid >> 5) * 4;
        float px[4], py[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int yy = y0 + r0 + i, xx = X0 + c;
            const bool ok = yy < h && xx < w;
            const size_t o = ok ? ((size_t)yy * w + xx) * 3 + ch : 0;
            px[i] = ok ? pred[o] : 0.f;
            py[i] = ok ? target[o] : 0.f;
        }
        hpass(b, y0 + kR, kS);
        __syncthreads();
        float local = 0.f;
        {
            const int base = y0 + r0 - kR - (Yseg - kR);
            float m[4][3];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 3; ++q) m[i][q] = 0.f;
#pragma unroll
            for (int t = 0; t < 14; ++t) {
                const int slot = (base + t) % kRing;
                float v[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) v[q] = S.h[q][slot][c];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int kk = t - i;
                    if (kk < 0 || kk > 10) continue;
                    const float wk = c_win[kk];
#pragma unroll
                    for (int q = 0; q < 3; ++q) m[i][q] = fmaf(wk, v[q], m[i][q]);
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int yy = y0 + r0 + i, xx = X0 + c;
                if (yy >= h || xx >= w) continue;
                const size_t o = ((size_t)yy * w + xx) * 3 + ch;
                const float x = px[i], y = py[i];
                const float dssim = m[i][0] + 2.f * x * m[i][1] + y * m[i][2];
                const float diff = x - y;
                const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
                adj[o] = l1_scale * sgn - lam * dssim;
                local += fabsf(diff);
            }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
        if ((tid & 31) == 0) S.red[tid >> 5] = local;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            float t = 0.f;
            for (int i = 0; i < 8; ++i) t += S.red[i];
            part_l1[((size_t)ch * gy + ty0 + k) * gx + bx] = t;
        }
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

// All parameter groups of one step in one launch: a block-range per group (blocks of
// 256 threads x 2 elements), the pair of elements loaded as double2 / float2 where
// aligned.  Same per-element arithmetic as adam_kernel.
constexpr int kAdamMaxGroups = 8;
struct AdamGroups {
    double* p[kAdamMaxGroups];
    const float* g[kAdamMaxGroups];
    double* m[kAdamMaxGroups];
    double* v[kAdamMaxGroups];
    int64_t count[kAdamMaxGroups];
    double lr[kAdamMaxGroups];
    int64_t block0[kAdamMaxGroups + 1];   // first block of each group
    int ngroups;
};

__device__ __forceinline__ void adam_one(double& p, double& m, double& v, float g, double lr, double b1, double b2,
                                         double bc1, double bc2, double eps) {
    const double gi = (double)g;
    const double mi = b1 * m + (1.0 - b1) * gi;
    const double vi = b2 * v + (1.0 - b2) * gi * gi;
    m = mi;
    v = vi;
    p = p - lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
}

__global__ void __launch_bounds__(256) adam_groups_kernel(AdamGroups a, double b1, double b2, double bc1,
                                                          double bc2, double eps) {
    int k = 0;
    while (k + 1 < a.ngroups && (int64_t)blockIdx.x >= a.block0[k + 1]) ++k;
    const int64_t i = (((int64_t)blockIdx.x - a.block0[k]) * 256 + threadIdx.x) * 2;
    const int64_t n = a.count[k];
    if (i >= n) return;
    double* p = a.p[k] + i;
    double* m = a.m[k] + i;
    double* v = a.v[k] + i;
    const float* g = a.g[k] + i;
    const double lr = a.lr[k];
    const bool vec = i + 1 < n && ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(m) |
                                    reinterpret_cast<uintptr_t>(v)) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(g) & 7) == 0;
    if (vec) {
        double2 pp = *reinterpret_cast<double2*>(p), mm = *reinterpret_cast<double2*>(m),
                vv = *reinterpret_cast<double2*>(v);
        const float2 gg = *reinterpret_cast<const float2*>(g);
        adam_one(pp.x, mm.x, vv.x, gg.x, lr, b1, b2, bc1, bc2, eps);
        adam_one(pp.y, mm.y, vv.y, gg.y, lr, b1, b2, bc1, bc2, eps);
        *reinterpret_cast<double2*>(p) = pp;
        *reinterpret_cast<double2*>(m) = mm;
        *reinterpret_cast<double2*>(v) = vv;
    } else {
        for (int64_t j = 0; j < 2 && i + j < n; ++j) adam_one(p[j], m[j], v[j], g[j], lr, b1, b2, bc1, bc2, eps);
    }
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
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(ssim_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)sizeof(GradSmem)));
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
    if (lam > 0.0) {   // grids: channel fastest (see ssim_stats_kernel)
        const dim3 sgrid(3 * gx, ceil_div(gy, kSegTiles));
        ssim_stats_kernel<<<sgrid, 256, kStatsSmem, stream>>>(pred, target, w, h, gscale, coef, part_ssim); note_launch();
    } else {
        SPLAT_CUDA_CHECK(cudaMemsetAsync(coef, 0, (size_t)w * h * 9 * 4, stream));
        SPLAT_CUDA_CHECK(cudaMemsetAsync(part_ssim, 0, nparts * 3 * 8, stream));
    }
    ssim_grad_kernel<<<dim3(3 * gx, ceil_div(gy, kSegTiles)), 256, sizeof(GradSmem), stream>>>(pred, target, w, h, coef, (float)((1.0 - lam) / size), (float)lam,
                                               adj, part_l1); note_launch();
    loss_finish_kernel<<<1, 768, 0, stream>>>(part_ssim, part_l1, (int)nparts, size, inner, lam, value);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int adam_groups_impl(int ngroups, double* const* p, const float* const* g, double* const* m, double* const* v,
                     const int64_t* count, const double* lr, double b1, double b2, double bc1, double bc2, double eps,
                     cudaStream_t stream) {
    if (ngroups < 0 || ngroups > kAdamMaxGroups) return set_error(SPLAT_ERR_PARAMETER, "0..8 parameter groups");
    AdamGroups a{};
    a.ngroups = ngroups;
    int64_t blocks = 0;
    for (int k = 0; k < ngroups; ++k) {
        if (count[k] < 0) return set_error(SPLAT_ERR_PARAMETER, "negative group size");
        a.p[k] = p[k];
        a.g[k] = g[k];
        a.m[k] = m[k];
        a.v[k] = v[k];
        a.count[k] = count[k];
        a.lr[k] = lr[k];
        a.block0[k] = blocks;
        blocks += (count[k] + 511) / 512;
    }
    a.block0[ngroups] = blocks;
    if (blocks == 0) return SPLAT_OK;
    adam_groups_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a, b1, b2, bc1, bc2, eps); note_launch();
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
