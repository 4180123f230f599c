// 3D EWA front-end: 3D Gaussians seen by
// a pinhole camera -> the 2D splat scene the rest of the path consumes.
//
//   m      = R mu + t                          (camera space)
//   Sigma3 = Rq diag(exp(2 s)) Rq^T            (quaternion q, log-scales s)
//   J      = [[fx/z, 0, -fx x/z^2], [0, fy/z, -fy y/z^2]]
//   Sigma2 = (J R) Sigma3 (J R)^T              (local affine approximation)
//   mean2  = (fx x/z + cx, fy y/z + cy)        (pixels of the camera image)
//
// Sigma2 is then written in the reference's 2D parametrisation
// (core.py:175-182: Sigma = R(theta) diag(exp(2 l1), exp(2 l2)) R(theta)^T):
// theta = atan2(2 b, a - c) / 2 is the major axis, l1/l2 = ln(lambda_max/min) / 2.
// Depth = z (front to back after the stable sort).  Gaussians with z <= near
// get an opacity logit of -100 (sigma ~ 4e-44 < 1/255: invalid, as the
// reference culls low opacity).  Everything in float64.  The reference package
// is 2D-only, so this stage is pinned to the float64 numpy restatement in
// oracle/oracle.py (project_gaussians), not to reference outputs.
#include <cmath>

#include "kernels.cuh"

namespace splat {
namespace {

__global__ void project_kernel(int64_t n, const double* __restrict__ mu, const double* __restrict__ ls3,
                               const double* __restrict__ quat, const double* __restrict__ logit_in,
                               splat_camera_t cam, double* __restrict__ means2, double* __restrict__ ls2,
                               double* __restrict__ rot2, double* __restrict__ logit_out,
                               double* __restrict__ depth) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* R = cam.R;
    const double px = mu[3 * i], py = mu[3 * i + 1], pz = mu[3 * i + 2];
    const double x = R[0] * px + R[1] * py + R[2] * pz + cam.t[0];
    const double y = R[3] * px + R[4] * py + R[5] * pz + cam.t[1];
    const double z = R[6] * px + R[7] * py + R[8] * pz + cam.t[2];
    depth[i] = z;
    if (!(z > cam.near_plane)) {
        means2[2 * i] = cam.cx;
        means2[2 * i + 1] = cam.cy;
        ls2[2 * i] = 0.0;
        ls2[2 * i + 1] = 0.0;
        rot2[i] = 0.0;
        logit_out[i] = -100.0;
        return;
    }
    // rotation matrix of the (normalised) quaternion w, x, y, z
    double qw = quat[4 * i], qx = quat[4 * i + 1], qy = quat[4 * i + 2], qz = quat[4 * i + 3];
    const double qn = 1.0 / sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    qw *= qn;
    qx *= qn;
    qy *= qn;
    qz *= qn;
    const double Q[9] = {1.0 - 2.0 * (qy * qy + qz * qz), 2.0 * (qx * qy - qw * qz), 2.0 * (qx * qz + qw * qy),
                         2.0 * (qx * qy + qw * qz), 1.0 - 2.0 * (qx * qx + qz * qz), 2.0 * (qy * qz - qw * qx),
                         2.0 * (qx * qz - qw * qy), 2.0 * (qy * qz + qw * qx), 1.0 - 2.0 * (qx * qx + qy * qy)};
    const double s2[3] = {exp(2.0 * ls3[3 * i]), exp(2.0 * ls3[3 * i + 1]), exp(2.0 * ls3[3 * i + 2])};
    // M = J R Q (2 x 3); Sigma2 = M diag(s2) M^T
    const double iz = 1.0 / z;
    const double J0[3] = {cam.fx * iz, 0.0, -cam.fx * x * iz * iz};
    const double J1[3] = {0.0, cam.fy * iz, -cam.fy * y * iz * iz};
    double JR0[3], JR1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        JR0[c] = J0[0] * R[c] + J0[1] * R[3 + c] + J0[2] * R[6 + c];
        JR1[c] = J1[0] * R[c] + J1[1] * R[3 + c] + J1[2] * R[6 + c];
    }
    double M0[3], M1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        M0[c] = JR0[0] * Q[c] + JR0[1] * Q[3 + c] + JR0[2] * Q[6 + c];
        M1[c] = JR1[0] * Q[c] + JR1[1] * Q[3 + c] + JR1[2] * Q[6 + c];
    }
    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a += M0[k] * M0[k] * s2[k];
        b += M0[k] * M1[k] * s2[k];
        c += M1[k] * M1[k] * s2[k];
    }
    const double h = 0.5 * (a + c), d = sqrt(0.25 * (a - c) * (a - c) + b * b);
    const double lmax = h + d;
    const double lmin = fmax(h - d, 1e-12 * lmax);   // rank-deficient projections stay positive definite
    means2[2 * i] = cam.fx * x * iz + cam.cx;
    means2[2 * i + 1] = cam.fy * y * iz + cam.cy;
    ls2[2 * i] = 0.5 * log(lmax);
    ls2[2 * i + 1] = 0.5 * log(lmin);
    rot2[i] = 0.5 * atan2(2.0 * b, a - c);
    logit_out[i] = logit_in[i];
}

}  // namespace

int project_impl(int64_t n, const double* mu, const double* ls3, const double* quat, const double* logit,
                 const splat_camera_t& cam, double* means2, double* ls2, double* rot2, double* logit_out,
                 double* depth, cudaStream_t stream) {
    if (n == 0) return SPLAT_OK;
    project_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(n, mu, ls3, quat, logit, cam, means2, ls2,
                                                                    rot2, logit_out, depth);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

}  // namespace splat
