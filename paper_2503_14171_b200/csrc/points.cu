// render_at_points (raster_forward.py:190-233): the blended colour at arbitrary
// continuous positions, with the rasterizer's sort / cull / clamp / early
// termination rules, for finite-difference validation of the analytic gradient
// planes.  One thread per point walks every valid splat in rank order in
// float64 with the reference's operation order (numpy evaluates left to right,
// unfused), so the result is the reference's to the last bit up to exp().
#include <cmath>

#include "kernels.cuh"

namespace splat {
namespace {

constexpr double kPtCull = 1.0 / 255.0, kPtClamp = 0.999, kPtTerm = 1e-4;

__global__ void points_kernel(const double* __restrict__ pack, const double* __restrict__ colors,
                              const uint8_t* __restrict__ valid, int64_t n, const double* __restrict__ xs,
                              const double* __restrict__ ys, int64_t npts, double bg0, double bg1, double bg2,
                              double* __restrict__ out, uint8_t* __restrict__ state) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= npts) return;
    const double x = xs[k], y = ys[k];
    double b0 = 0.0, b1 = 0.0, b2 = 0.0, acc = 0.0;
    bool done = false;
    for (int64_t i = 0; i < n; ++i) {
        if (!valid[i]) continue;
        const double* p = pack + 6 * i;
        const double dx = __dsub_rn(x, p[0]), dy = __dsub_rn(y, p[1]);
        const double t1 = __dmul_rn(__dmul_rn(p[2], dx), dx);
        const double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, p[3]), dx), dy);
        const double t3 = __dmul_rn(__dmul_rn(p[4], dy), dy);
        const double expo = -__dadd_rn(__dadd_rn(t1, t2), t3);
        const double a_raw = __dmul_rn(p[5], exp(expo));
        const double alpha = a_raw < kPtClamp ? a_raw : kPtClamp;
        const bool use = (a_raw >= kPtCull) && !done;
        if (state) {
            state[k * 2 * n + i] = use;
            state[k * 2 * n + n + i] = use && (a_raw > kPtClamp);
        }
        if (!use) continue;
        const double t = __dsub_rn(1.0, acc);
        const double ta = __dmul_rn(t, alpha);
        b0 = __dadd_rn(b0, __dmul_rn(ta, colors[3 * i]));
        b1 = __dadd_rn(b1, __dmul_rn(ta, colors[3 * i + 1]));
        b2 = __dadd_rn(b2, __dmul_rn(ta, colors[3 * i + 2]));
        acc = __dadd_rn(acc, __dmul_rn(alpha, t));
        done = __dsub_rn(1.0, acc) < kPtTerm;
    }
    const double rem = __dsub_rn(1.0, acc);
    out[3 * k] = __dadd_rn(b0, __dmul_rn(rem, bg0));
    out[3 * k + 1] = __dadd_rn(b1, __dmul_rn(rem, bg1));
    out[3 * k + 2] = __dadd_rn(b2, __dmul_rn(rem, bg2));
}

}  // namespace

int points_impl(const double* pack, const double* colors, const uint8_t* valid, int64_t n, const double* xs,
                const double* ys, int64_t npts, const double* bg, double* out, uint8_t* state,
                cudaStream_t stream) {
    if (npts == 0) return SPLAT_OK;
    points_kernel<<<(unsigned)((npts + 127) / 128), 128, 0, stream>>>(pack, colors, valid, n, xs, ys, npts, bg[0],
                                                                     bg[1], bg[2], out, state);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

}  // namespace splat
