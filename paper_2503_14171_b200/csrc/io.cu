// Wire formats either side of the hot path.
//
//   GIMG gradient dump (reference io.py:100-137): "GIMG", u32 width, u32 height,
//   then 16 little-endian float32 (H, W) planes in the order
//   color R,G,B, d_dx R,G,B, d_dy R,G,B, d_dxdy R,G,B, alpha, alpha_dx,
//   alpha_dy, alpha_dxdy.  The device GradientImage keeps colour + derivatives
//   pixel-interleaved (H, W, 4, 3) for the upscaler, so writing / reading a
//   dump is a transpose: one thread per pixel reads its 48 contiguous bytes and
//   writes 12 planar values (coalesced across the warp), or the reverse.
//
//   Display encoding (io.py:28-37): clip to [0, 1], x^(1/2.2), x 255, round half
//   to even, uint8 — computed in float64 like numpy.
#include "kernels.cuh"

namespace splat {
namespace {

__global__ void gimg_pack_kernel(const float4* __restrict__ planes, const float* __restrict__ alpha, int64_t P,
                                 float* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = planes[3 * i], b = planes[3 * i + 1], c = planes[3 * i + 2];
        const float v[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
        for (int k = 0; k < 12; ++k) out[k * P + i] = v[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) out[(12 + k) * P + i] = alpha[k * P + i];
    }
}

__global__ void gimg_unpack_kernel(const float* __restrict__ in, int64_t P, float4* __restrict__ planes,
                                   float* __restrict__ alpha, int32_t* __restrict__ count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        float v[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) v[k] = in[k * P + i];
        planes[3 * i] = make_float4(v[0], v[1], v[2], v[3]);
        planes[3 * i + 1] = make_float4(v[4], v[5], v[6], v[7]);
        planes[3 * i + 2] = make_float4(v[8], v[9], v[10], v[11]);
#pragma unroll
        for (int k = 0; k < 4; ++k) alpha[k * P + i] = in[(12 + k) * P + i];
        if (count) count[i] = 0;   // a dump carries no contributor counts (io.py:128)
    }
}

__global__ void encode_display_kernel(const float* __restrict__ img, int64_t n, uint8_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double x = (double)img[i];
        x = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);   // np.clip (NaN stays NaN -> 0 below)
        const double y = pow(x, 1.0 / 2.2) * 255.0;
        const double r = rint(y);                    // round half to even, as np.round
        out[i] = (uint8_t)(r >= 0.0 && r <= 255.0 ? (int)r : 0);
    }
}

int grid_for(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

int gimg_pack_impl(const float* planes, const float* alpha, int w, int h, float* out, cudaStream_t stream) {
    const int64_t P = (int64_t)w * h;
    gimg_pack_kernel<<<grid_for(P), 256, 0, stream>>>((const float4*)planes, alpha, P, out);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int gimg_unpack_impl(const float* in, int w, int h, float* planes, float* alpha, int32_t* count,
                     cudaStream_t stream) {
    const int64_t P = (int64_t)w * h;
    gimg_unpack_kernel<<<grid_for(P), 256, 0, stream>>>(in, P, (float4*)planes, alpha, count);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int encode_display_impl(const float* img, int64_t n, uint8_t* out, cudaStream_t stream) {
    if (n == 0) return SPLAT_OK;
    encode_display_kernel<<<grid_for(n), 256, 0, stream>>>(img, n, out);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

}  // namespace splat
