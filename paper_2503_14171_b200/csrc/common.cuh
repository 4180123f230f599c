// Shared definitions for the sm_100a render + upscale kernels.
#pragma once
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <cuda_runtime.h>

#include "../../include/splat_b200.h"

namespace splat {

constexpr int kTile = 16;                 // raster_forward.py:24
constexpr int kBlock = 256;               // one 16x16 tile per CTA
constexpr double kAlphaClamp = 0.999;     // core.py:23
constexpr double kAlphaCull = 1.0 / 255.0;  // core.py:24
constexpr double kEarlyTerm = 1e-4;       // core.py:25
// _kernels.py:29 LOG_CULL = float(np.log(1/255)); bit pattern taken from numpy.
constexpr double kLogCull = -5.541263545158426;

// Rank-ordered, view-independent per-splat constants (computed once per scene
// on the device).  Struct-of-arrays, float64 unless noted.
struct SceneConst {
    int64_t n;
    const int32_t* order;   // rank -> storage index (stable depth argsort)
    const int32_t* rank_of; // storage index -> rank (inverse permutation)
    const double* mean;     // (n,2) means gathered into rank order
    const double* n00;      // e1 c^2 + e2 s^2          (raster_forward.py:96)
    const double* n01;      // (e1 - e2) s c            (raster_forward.py:97)
    const double* n11;      // e1 s^2 + e2 c^2          (raster_forward.py:98)
    const double* e1e2;     // e1 * e2                  (raster_forward.py:108)
    const double* sigma;    // logistic(opacity_logit)  (raster_forward.py:89)
    const double* q;        // log(max(sigma/(1/255),1)) (raster_forward.py:107)
    const float4* color;    // (n) float32 rgb_ colours in rank order
};

// Per-view float32 pack the rasterizer consumes (rank order, 64 bytes).
struct __align__(16) PackF {
    float mxh, myh, mxl, myl;     // render-space mean as float hi + lo parts ((x, y) pairs for FADD2)
    float a, c, nb2, l2sig;       // conic a, c (adjacent for FMUL2), nb2 = -2 b (exact), log2(sigma)
    // decision thresholds of eval_fast with its qcull-relative tolerance folded in (directed
    // rounding): qcull (1 + 2^-19) up, qcull (1 - 2^-19) down, qclamp + 2^-19 qcull up,
    // qclamp - 2^-19 qcull down; qcull = ln(255 sigma), qclamp = ln(sigma / 0.999)
    float cull_hi, cull_lo, clamp_hi, clamp_lo;
    float ex, ey, pad2, pad3;     // half extents of the cull ellipse; pad2: 4x2-group Q-norm bound (pre-filters only)
};

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Device-side invariant checks of the checked build (`make checked` ->
// libsplat_b200_checked.so): index and protocol bounds of the shared-memory rings,
// staging buffers and scattered stores.  A violated check prints and traps, so the
// launch fails loudly; the default build compiles them out.  (compute-sanitizer is
// not available on this pool: this build plus the guard-band tests stand in for it.)
#ifndef SPLAT_CHECKS
#define SPLAT_CHECKS 0
#endif
#if SPLAT_CHECKS
#define SPLAT_DCHECK(cond)                                                                          \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("SPLAT_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                             \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define SPLAT_DCHECK(cond) \
    do {                   \
    } while (0)
#endif

}  // namespace splat

#define SPLAT_CUDA_CHECK(expr)                                   \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) return splat::set_cuda_error(_e, #expr); \
    } while (0)

namespace splat {
void note_launch();  // counts kernels launched by this library (splat_kernel_launches)
int set_cuda_error(cudaError_t e, const char* what);
int set_error(int code, const char* msg);

// Launch configuration that is per device (the dynamic shared-memory opt-in of
// cudaFuncSetAttribute, occupancy-derived grids, __constant__ tables): one
// entry per device ordinal, initialised once under a mutex, so a process that
// drives several GPUs, or calls from several host threads, configures each
// device exactly once.  `init(T&)` returns SPLAT_OK or an error code.
template <class T>
class PerDevice {
public:
    template <class F>
    int get(T& out, F&& init) {
        int dev = 0;
        SPLAT_CUDA_CHECK(cudaGetDevice(&dev));
        if (dev < 0 || dev >= kMaxDevices) return set_error(SPLAT_ERR_PARAMETER, "device ordinal out of range");
        if (!ready_[dev].load(std::memory_order_acquire)) {
            std::lock_guard<std::mutex> lock(mu_);
            if (!ready_[dev].load(std::memory_order_relaxed)) {
                T v{};
                const int rc = init(v);
                if (rc != SPLAT_OK) return rc;
                val_[dev] = v;
                ready_[dev].store(true, std::memory_order_release);
            }
        }
        out = val_[dev];
        return SPLAT_OK;
    }

private:
    static constexpr int kMaxDevices = 64;
    std::atomic<bool> ready_[kMaxDevices] = {};
    T val_[kMaxDevices] = {};
    std::mutex mu_;
};

// SM count of the current device (cached per device).
int device_sms(int& sms);
}  // namespace splat
