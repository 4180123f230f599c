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

constexpr int kUpRows = 16;

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

// ---- upscale plan: per-axis maps computed once per (in, out) size ------------------------
// Table entry for output index u: i0 = floor(s) and the 4 Hermite weights,
// s = (u + .5) / (n_out / n_in) - .5 in float64 exactly as numpy computes it.
// Tables are padded to a multiple of the tile size (tail entries repeat the
// last index) so every tile's slice can be bulk-copied without bounds checks.
constexpr int kPlanPad = 256;

__global__ void plan_kernel(int n_out, int n_pad, double scale, int* __restrict__ i0,
                            float4* __restrict__ w) {
    int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_pad) return;
    AxisMap m = axis_map(min(u, n_out - 1), scale);
    i0[u] = m.i0;
    w[u] = make_float4(m.h[0], m.h[1], m.h[2], m.h[3]);
}

struct PlanView {
    const int* ci0;
    const float4* cw;
    const int* ri0;
    const float4* rw;
};

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// Persistent upscaler.  Each CTA walks output tiles of kUpRows x tile_c
// pixels; for tile i+1 it issues the TMA bulk copies (source rows, column and
// row maps) into the other shared-memory stage before computing tile i, so
// HBM reads overlap the arithmetic and the 16-byte output stores.
__global__ void __launch_bounds__(256) upscale_fwd_kernel(const float* __restrict__ src, int in_w,
                                                          int in_h, float* __restrict__ out, int out_w,
                                                          int out_h, int clamp, PlanView plan, int tile_c,
                                                          int span_c, int span_r) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ int s_box[2][4];

    const int tid = threadIdx.x;
    const int ntx = (out_w + tile_c - 1) / tile_c;
    const int nty = (out_h + kUpRows - 1) / kUpRows;
    const int ntiles = ntx * nty;
    const size_t src_floats = (size_t)span_r * span_c * 12;
    float* const s_src0 = reinterpret_cast<float*>(smem);                 // 2 stages of span_r x span_c x 12
    float* const s_g = s_src0 + 2 * src_floats;                           // kUpRows x span_c x 6
    // per-stage map slices: [cw tile_c float4][rw kUpRows float4][ci0 tile_c int][ri0 kUpRows int]
    unsigned char* const s_map0 = reinterpret_cast<unsigned char*>(s_g + (size_t)kUpRows * span_c * 6);
    const size_t map_bytes = (size_t)tile_c * 20 + kUpRows * 20;
#define STAGE_SRC(b) (s_src0 + (size_t)(b) * src_floats)
#define STAGE_CW(b) reinterpret_cast<float4*>(s_map0 + (size_t)(b) * map_bytes)
#define STAGE_RW(b) reinterpret_cast<float4*>(s_map0 + (size_t)(b) * map_bytes + (size_t)tile_c * 16)
#define STAGE_CI(b) reinterpret_cast<int*>(s_map0 + (size_t)(b) * map_bytes + (size_t)tile_c * 16 + kUpRows * 16)
#define STAGE_RI(b) reinterpret_cast<int*>(s_map0 + (size_t)(b) * map_bytes + (size_t)tile_c * 20 + kUpRows * 16)
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[0])));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    // thread 0: compute the source box of tile t and launch its copies into stage b
    auto issue = [&](int t, int b) {
        const int U0 = (t % ntx) * tile_c, V0 = (t / ntx) * kUpRows;
        const int ulast = min(U0 + tile_c, out_w) - 1, vlast = min(V0 + kUpRows, out_h) - 1;
        const int x0 = clampi(plan.ci0[U0], 0, in_w - 1), x1 = clampi(plan.ci0[ulast] + 1, 0, in_w - 1);
        const int y0 = clampi(plan.ri0[V0], 0, in_h - 1), y1 = clampi(plan.ri0[vlast] + 1, 0, in_h - 1);
        s_box[b][0] = x0;
        s_box[b][1] = x1 - x0 + 1;
        s_box[b][2] = y0;
        s_box[b][3] = y1 - y0 + 1;
        const uint32_t row_bytes = (uint32_t)(x1 - x0 + 1) * 48u;
        const uint32_t bytes = row_bytes * (uint32_t)(y1 - y0 + 1) + (uint32_t)tile_c * 20u + kUpRows * 20u;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar[b])),
                     "r"(bytes)
                     : "memory");
        for (int r = 0; r <= y1 - y0; ++r)
            bulk_copy(STAGE_SRC(b) + (size_t)r * span_c * 12, src + ((size_t)(y0 + r) * in_w + x0) * 12,
                      row_bytes, &s_bar[b]);
        bulk_copy(STAGE_CW(b), plan.cw + U0, (uint32_t)tile_c * 16u, &s_bar[b]);
        bulk_copy(STAGE_CI(b), plan.ci0 + U0, (uint32_t)tile_c * 4u, &s_bar[b]);
        bulk_copy(STAGE_RW(b), plan.rw + V0, kUpRows * 16u, &s_bar[b]);
        bulk_copy(STAGE_RI(b), plan.ri0 + V0, kUpRows * 4u, &s_bar[b]);
    };

    int t = blockIdx.x;
    if (t < ntiles && tid == 0) issue(t, 0);
    uint32_t phases = 0u;  // bit b = parity of stage b's next completion
    for (int b = 0; t < ntiles; t += gridDim.x, b ^= 1) {
        const int tn = t + gridDim.x;
        if (tn < ntiles && tid == 0) issue(tn, b ^ 1);
        mbar_wait(&s_bar[b], (phases >> b) & 1u);
        phases ^= 1u << b;
        const int U0 = (t % ntx) * tile_c, V0 = (t / ntx) * kUpRows;
        const int x0 = s_box[b][0], ncols = s_box[b][1], y0 = s_box[b][2];
        const int nv = min(kUpRows, out_h - V0);
        const float* sb = STAGE_SRC(b);
        const float4* s_rwb = STAGE_RW(b);
        const int* s_rib = STAGE_RI(b);
        const float4* s_cwb = STAGE_CW(b);
        const int* s_cib = STAGE_CI(b);
        // y pass: G[v][x] = (value-in-x, slope-in-x) of output row v at source column x.
        // Source records (48 B) are read as 3 x LDS.128 and G records (24 B) written as
        // 3 x STS.64: both strides are bank-conflict free.
        for (int e = tid; e < nv * ncols; e += blockDim.x) {
            const int v = e / ncols, x = e - v * ncols;
            const float4 h = s_rwb[v];
            const int ri = s_rib[v];
            const int ra = clampi(ri, 0, in_h - 1) - y0, rb = clampi(ri + 1, 0, in_h - 1) - y0;
            const float4* pa = reinterpret_cast<const float4*>(sb + ((size_t)ra * span_c + x) * 12);
            const float4* pb = reinterpret_cast<const float4*>(sb + ((size_t)rb * span_c + x) * 12);
            const float4 a0 = pa[0], a1 = pa[1], a2 = pa[2];
            const float4 b0 = pb[0], b1 = pb[1], b2 = pb[2];
            // record = [f0 f1 f2 fx0 | fx1 fx2 fy0 fy1 | fy2 fxy0 fxy1 fxy2]
            const float fa[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
            const float fb[12] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
            float g[6];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                g[c] = fmaf(h.x, fa[c], fmaf(h.y, fb[c], fmaf(h.z, fa[6 + c], h.w * fb[6 + c])));
                g[3 + c] = fmaf(h.x, fa[3 + c], fmaf(h.y, fb[3 + c], fmaf(h.z, fa[9 + c], h.w * fb[9 + c])));
            }
            float2* gd = reinterpret_cast<float2*>(s_g + ((size_t)v * span_c + x) * 6);
            gd[0] = make_float2(g[0], g[1]);
            gd[1] = make_float2(g[2], g[3]);
            gd[2] = make_float2(g[4], g[5]);
        }
        __syncthreads();
        // x pass: 4 consecutive output pixels per thread and step
        const int groups_per_row = tile_c / 4;
        const int nu = min(tile_c, out_w - U0);
        for (int e = tid; e < nv * groups_per_row; e += blockDim.x) {
            const int v = e / groups_per_row, ug = (e - v * groups_per_row) * 4;
            if (ug >= nu) continue;
            float o[12];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int uu = min(ug + i, nu - 1);
                const float4 h = s_cwb[uu];
                const int ci = s_cib[uu];
                const int xa = clampi(ci, 0, in_w - 1) - x0, xb = clampi(ci + 1, 0, in_w - 1) - x0;
                const float2* ga = reinterpret_cast<const float2*>(s_g + ((size_t)v * span_c + xa) * 6);
                const float2* gb = reinterpret_cast<const float2*>(s_g + ((size_t)v * span_c + xb) * 6);
                const float2 a0 = ga[0], a1 = ga[1], a2 = ga[2], b0 = gb[0], b1 = gb[1], b2 = gb[2];
                const float A[6] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y};
                const float B[6] = {b0.x, b0.y, b1.x, b1.y, b2.x, b2.y};
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    float val = fmaf(h.x, A[c], fmaf(h.y, B[c], fmaf(h.z, A[3 + c], h.w * B[3 + c])));
                    if (clamp) val = fminf(fmaxf(val, 0.f), 1.f);
                    o[3 * i + c] = val;
                }
            }
            float* dst = out + ((size_t)(V0 + v) * out_w + U0 + ug) * 3;
            if (ug + 3 < nu && (out_w & 3) == 0) {
                float4* d4 = reinterpret_cast<float4*>(dst);
                __stcs(d4, make_float4(o[0], o[1], o[2], o[3]));
                __stcs(d4 + 1, make_float4(o[4], o[5], o[6], o[7]));
                __stcs(d4 + 2, make_float4(o[8], o[9], o[10], o[11]));
            } else {
                for (int i = 0; i < 4 && ug + i < nu; ++i)
                    for (int c = 0; c < 3; ++c) dst[3 * i + c] = o[3 * i + c];
            }
        }
        __syncthreads();
    }
#undef STAGE_SRC
#undef STAGE_CW
#undef STAGE_RW
#undef STAGE_CI
#undef STAGE_RI
}

// ---- integer factors (x2, x4: the benchmark configurations) ------------------------------
// With out = F * in exactly, output column u = F m + j maps to a fixed phase
// (i0 - m, t) that repeats every F pixels, so the Hermite weights are per-phase
// constants and no per-column maps are needed.  A CTA computes a 16-row x
// (64 F)-column output tile: one TMA bulk copy per source row into shared
// memory, the y pass G[v][x] for the tile's source columns, then each thread
// emits 4 consecutive pixels of a row (3 x 16-byte streaming stores) from the
// G records of the F-aligned cells they fall in.  Clamping to [0, 1] is the
// .sat modifier of the last FMA (spline.py:178).

__device__ __forceinline__ float fma_sat(float a, float b, float c) {
    float r;
    asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__host__ __device__ constexpr int int_tile_cols(int F) { return 32 * F; }

// Hermite weights of phase j for integer factor F: t_j = (j + .5) / F (the
// fractional position of output pixel F m + F/2 + j inside cell m).  The values
// are dyadic rationals, exact in float32, and become FFMA immediates.
__host__ __device__ constexpr float hermite_w(int F, int j, int k) {
    const double t = (j + 0.5) / F, t2 = t * t, t3 = t2 * t;
    return (float)(k == 0 ? 1.0 - 3.0 * t2 + 2.0 * t3
                          : k == 1 ? 3.0 * t2 - 2.0 * t3 : k == 2 ? t - 2.0 * t2 + t3 : t3 - t2);
}

template <int F, bool CLAMP>
__global__ void __launch_bounds__(256) upscale_int_kernel(const float* __restrict__ src, int in_w, int in_h,
                                                          float* __restrict__ out, int out_w, int out_h,
                                                          int span_c, int span_r) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[2];
    constexpr int TC = int_tile_cols(F);
    constexpr int GPR = TC / 4;            // 4-pixel groups per output row
    constexpr int NREC = 4 / F + 2;        // G records a group touches
    constexpr int GCOLS = TC / F + 2;      // G columns (cells) of a tile
    constexpr int CROWS = kUpRows / F + 1; // cell rows overlapping a tile's rows
    const int tid = threadIdx.x;
    const int ntx = (out_w + TC - 1) / TC, nty = (out_h + kUpRows - 1) / kUpRows, ntiles = ntx * nty;
    const size_t src_floats = (size_t)span_r * span_c * 12;
    float* const s_src0 = reinterpret_cast<float*>(smem);
    float* const s_g = s_src0 + 2 * src_floats;
    float4* const s_xpose = reinterpret_cast<float4*>(s_g + (size_t)kUpRows * GCOLS * 6);  // 8 warps x 96
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[0])));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // source box of a tile: cells U0/F - 1 .. (U0 + TC)/F (clamped), rows likewise
    auto box = [&](int t, int& x0, int& ncols, int& y0, int& nrows) {
        const int U0 = (t % ntx) * TC, V0 = (t / ntx) * kUpRows;
        x0 = max(U0 / F - 1, 0);
        ncols = min((U0 + TC) / F, in_w - 1) - x0 + 1;
        y0 = max(V0 / F - 1, 0);
        nrows = min((V0 + kUpRows) / F, in_h - 1) - y0 + 1;
    };
    auto issue = [&](int t, int b) {
        int x0, ncols, y0, nrows;
        box(t, x0, ncols, y0, nrows);
        const uint32_t row_bytes = (uint32_t)ncols * 48u;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar[b])),
                     "r"(row_bytes * (uint32_t)nrows)
                     : "memory");
        float* dst = s_src0 + (size_t)b * src_floats;
        for (int r = 0; r < nrows; ++r)
            bulk_copy(dst + (size_t)r * span_c * 12, src + ((size_t)(y0 + r) * in_w + x0) * 12, row_bytes,
                      &s_bar[b]);
    };

    int t = blockIdx.x;
    if (t < ntiles && tid == 0) issue(t, 0);
    uint32_t phases = 0u;
    for (int b = 0; t < ntiles; t += gridDim.x, b ^= 1) {
        // prefetch the next tile into the other stage while this one is computed
        if (t + (int)gridDim.x < ntiles && tid == 0) issue(t + gridDim.x, b ^ 1);
        mbar_wait(&s_bar[b], (phases >> b) & 1u);
        phases ^= 1u << b;
        const int U0 = (t % ntx) * TC, V0 = (t / ntx) * kUpRows;
        const int cx0 = U0 / F - 1, cy0 = V0 / F - 1;
        int x0, ncols, y0, nrows;
        box(t, x0, ncols, y0, nrows);
        const float* sb = s_src0 + (size_t)b * src_floats;
        const int nv = min(kUpRows, out_h - V0);
        // y pass, one item per (cell row, cell column): the cell's two corner rows are
        // read once (6 x LDS.128) and give the G records of its F output rows
        // G[v][gc] = (value-in-x, slope-in-x) at corner column cx0 + gc.
        for (int it = tid; it < CROWS * GCOLS; it += blockDim.x) {
            const int cr = it / GCOLS, gc = it - cr * GCOLS;
            const int n = cy0 + cr;
            const int ra = clampi(n, 0, in_h - 1) - y0, rb = clampi(n + 1, 0, in_h - 1) - y0;
            const int xc = clampi(cx0 + gc, 0, in_w - 1) - x0;
            const float4* pa = reinterpret_cast<const float4*>(sb + ((size_t)ra * span_c + xc) * 12);
            const float4* pb = reinterpret_cast<const float4*>(sb + ((size_t)rb * span_c + xc) * 12);
            const float4 a0 = pa[0], a1 = pa[1], a2 = pa[2];
            const float4 b0 = pb[0], b1 = pb[1], b2 = pb[2];
            // record = [f0 f1 f2 fx0 | fx1 fx2 fy0 fy1 | fy2 fxy0 fxy1 fxy2]
            const float fa[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
            const float fb[12] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
#pragma unroll
            for (int j = 0; j < F; ++j) {
                const int v = F * n + F / 2 + j - V0;   // output row of phase j in cell row n
                if (v < 0 || v >= nv) continue;
                const float h0 = hermite_w(F, j, 0), h1 = hermite_w(F, j, 1);
                const float h2 = hermite_w(F, j, 2), h3 = hermite_w(F, j, 3);
                float g[6];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    g[c] = fmaf(h0, fa[c], fmaf(h1, fb[c], fmaf(h2, fa[6 + c], h3 * fb[6 + c])));
                    g[3 + c] = fmaf(h0, fa[3 + c], fmaf(h1, fb[3 + c], fmaf(h2, fa[9 + c], h3 * fb[9 + c])));
                }
                float2* gd = reinterpret_cast<float2*>(s_g + ((size_t)v * GCOLS + gc) * 6);
                gd[0] = make_float2(g[0], g[1]);
                gd[1] = make_float2(g[2], g[3]);
                gd[2] = make_float2(g[4], g[5]);
            }
        }
        __syncthreads();
        // x pass: thread -> 4 consecutive pixels u = U0 + ug .. +3 of row v, whose corner
        // columns are the cells base-1 .. base+4/F (NREC G records, each loaded once)
        const int nu = min(TC, out_w - U0);
        for (int e = tid; e < nv * GPR; e += blockDim.x) {
            const int v = e / GPR, ug = (e - v * GPR) * 4;
            if (ug >= nu) continue;
            const int r0 = (U0 + ug) / F - 1 - cx0;   // G column of record 0
            const float2* gp = reinterpret_cast<const float2*>(s_g + ((size_t)v * GCOLS + r0) * 6);
            float R[NREC][6];
#pragma unroll
            for (int k = 0; k < NREC; ++k) {
                const float2 q0 = gp[3 * k], q1 = gp[3 * k + 1], q2 = gp[3 * k + 2];
                R[k][0] = q0.x;
                R[k][1] = q0.y;
                R[k][2] = q1.x;
                R[k][3] = q1.y;
                R[k][4] = q2.x;
                R[k][5] = q2.y;
            }
            float o[12];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                // pixel U0 + ug + i (U0 + ug is a multiple of F): phase and left record are static
                const int jx = (i + F / 2) % F;
                const int ka = (i + F / 2) / F;
                const float h0 = hermite_w(F, jx, 0), h1 = hermite_w(F, jx, 1);
                const float h2 = hermite_w(F, jx, 2), h3 = hermite_w(F, jx, 3);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float part = fmaf(h1, R[ka + 1][c], fmaf(h2, R[ka][3 + c], h3 * R[ka + 1][3 + c]));
                    o[3 * i + c] = CLAMP ? fma_sat(h0, R[ka][c], part) : fmaf(h0, R[ka][c], part);
                }
            }
            // the lanes of one row segment (GPR = 32 or 16 groups) transpose their
            // 48-byte outputs through shared memory so every 16-byte store
            // instruction writes whole 128-byte lines (512 or 2 x 256 contiguous bytes)
            if ((out_w & 3) == 0 && nu == TC) {
                const int lane = tid & 31, li = lane % GPR;
                float4* w4 = s_xpose + (tid >> 5) * 96 + (lane / GPR) * 3 * GPR;
                w4[3 * li] = make_float4(o[0], o[1], o[2], o[3]);
                w4[3 * li + 1] = make_float4(o[4], o[5], o[6], o[7]);
                w4[3 * li + 2] = make_float4(o[8], o[9], o[10], o[11]);
                __syncwarp();
                float4* d4 = reinterpret_cast<float4*>(out + ((size_t)(V0 + v) * out_w + U0) * 3);
                __stcs(d4 + li, w4[li]);
                __stcs(d4 + GPR + li, w4[GPR + li]);
                __stcs(d4 + 2 * GPR + li, w4[2 * GPR + li]);
                __syncwarp();
            } else {
                float* dst = out + ((size_t)(V0 + v) * out_w + U0 + ug) * 3;
                for (int i = 0; i < 4 && ug + i < nu; ++i)
                    for (int c = 0; c < 3; ++c) dst[3 * i + c] = o[3 * i + c];
            }
        }
        __syncthreads();
    }
}

// x4 fast path (the headline configuration).  One thread owns one cell row n
// and one 4-pixel column group g: output rows 4n+2 .. 4n+5 (phases 0..3 of
// the cell) x pixels 4g .. 4g+3 (phases 2,3 of cell g-1 and 0,1 of cell g).
// It reads its 6 corner records (corner columns g-1..g+1, rows n, n+1) from
// the TMA-staged source tile once, runs y pass + x pass in registers (no
// shared-memory intermediate, no barrier between the passes) and writes
// 4 rows x 48 bytes with 16-byte streaming stores.  A CTA = UP_X4_WARPS warps
// = as many cell rows x 32 groups; persistent, double-buffered.  One warp per
// CTA (105 registers, 3.6K per CTA) is the default: such a CTA fits in the
// registers the persistent raster of another view leaves free on each SM, so
// in the multi-stream pipeline part of the upscale runs beside that raster;
// alone it is also faster (26.5 -> 24.6 us at C3, 78% of measured HBM peak)
// although each source row is staged twice (tiles of 1 cell row need 2 rows).
constexpr int kX4Groups = 32;                // groups (4 px) per tile row = one warp
#ifndef UP_X4_WARPS
#define UP_X4_WARPS 1
#endif
#ifndef UP_X4_GRID_PER_SM
#define UP_X4_GRID_PER_SM 0   // 0: occupancy
#endif
constexpr int kX4CellRows = UP_X4_WARPS;     // cell rows per tile = warps per CTA
constexpr int kX4SpanC = kX4Groups + 2;      // corner columns of a tile
constexpr int kX4SpanR = kX4CellRows + 1;    // corner rows of a tile

#ifndef UP_TMA_STORE
#define UP_TMA_STORE 1
#endif
#ifndef UP_X4_MINB
#define UP_X4_MINB (UP_X4_WARPS == 1 ? 16 : 1)
#endif
template <bool CLAMP>
__global__ void __launch_bounds__(32 * UP_X4_WARPS, UP_X4_MINB) upscale_x4_kernel(const float* __restrict__ src, int in_w, int in_h,
                                                         float* __restrict__ out, int out_w, int out_h) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[2];
    constexpr size_t kStage = (size_t)kX4SpanR * kX4SpanC * 12;   // floats per stage
    float* const s_src0 = reinterpret_cast<float*>(smem);
    float4* const s_xp = reinterpret_cast<float4*>(s_src0 + 2 * kStage);  // warps x 96 float4
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ngx = (out_w / 4 + kX4Groups - 1) / kX4Groups;     // tiles along x
    const int ngy = (in_h + 1 + kX4CellRows - 1) / kX4CellRows;  // cell rows -1 .. in_h-1
    const int ntiles = ngx * ngy;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[0])));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // tile t: groups g0 .. g0+31, cell rows n0 .. n0+7 (n0 = 8 ty - 1); its corner box is
    // columns g0-1 .. g0+32 and rows n0 .. n0+8, clamped to the image (edge replication)
    auto box = [&](int t, int& x0, int& ncols, int& y0, int& nrows) {
        const int g0 = (t % ngx) * kX4Groups, n0 = (t / ngx) * kX4CellRows - 1;
        x0 = max(g0 - 1, 0);
        ncols = min(g0 + kX4Groups, in_w - 1) - x0 + 1;
        y0 = max(n0, 0);
        nrows = min(n0 + kX4CellRows, in_h - 1) - y0 + 1;
    };
    auto issue = [&](int t, int b) {
        int x0, ncols, y0, nrows;
        box(t, x0, ncols, y0, nrows);
        const uint32_t row_bytes = (uint32_t)ncols * 48u;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar[b])),
                     "r"(row_bytes * (uint32_t)nrows)
                     : "memory");
        float* dst = s_src0 + (size_t)b * kStage;
        for (int r = 0; r < nrows; ++r)
            bulk_copy(dst + (size_t)r * kX4SpanC * 12, src + ((size_t)(y0 + r) * in_w + x0) * 12, row_bytes,
                      &s_bar[b]);
    };

    int t = blockIdx.x;
    if (t < ntiles && tid == 0) issue(t, 0);
    uint32_t phases = 0u;
    for (int b = 0; t < ntiles; t += gridDim.x, b ^= 1) {
        if (t + (int)gridDim.x < ntiles && tid == 0) issue(t + gridDim.x, b ^ 1);
        mbar_wait(&s_bar[b], (phases >> b) & 1u);
        phases ^= 1u << b;
        int x0, ncols, y0, nrows;
        box(t, x0, ncols, y0, nrows);
        const int g = (t % ngx) * kX4Groups + lane;
        const int n = (t / ngx) * kX4CellRows - 1 + warp;
        const unsigned active = __ballot_sync(0xffffffffu, g < out_w / 4);
        if (g < out_w / 4 && n < in_h) {
            const float* sb = s_src0 + (size_t)b * kStage;
            // corner records: columns g-1, g, g+1; rows n, n+1 (edge-clamped)
            float rec[2][3][12];
#pragma unroll
            for (int ry = 0; ry < 2; ++ry) {
                const int row = clampi(n + ry, 0, in_h - 1) - y0;
                SPLAT_DCHECK(row >= 0 && row < nrows && row < kX4SpanR);
#pragma unroll
                for (int cx = 0; cx < 3; ++cx) {
                    const int col = clampi(g - 1 + cx, 0, in_w - 1) - x0;
                    SPLAT_DCHECK(col >= 0 && col < ncols && col < kX4SpanC);
                    const float4* p = reinterpret_cast<const float4*>(sb + ((size_t)row * kX4SpanC + col) * 12);
                    const float4 q0 = p[0], q1 = p[1], q2 = p[2];
                    float* r = rec[ry][cx];
                    r[0] = q0.x; r[1] = q0.y; r[2] = q0.z; r[3] = q0.w;
                    r[4] = q1.x; r[5] = q1.y; r[6] = q1.z; r[7] = q1.w;
                    r[8] = q2.x; r[9] = q2.y; r[10] = q2.z; r[11] = q2.w;
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {              // output row 4n + 2 + j
                const int v = 4 * n + 2 + j;
                if (v < 0 || v >= out_h) continue;
                const float h0 = hermite_w(4, j, 0), h1 = hermite_w(4, j, 1);
                const float h2 = hermite_w(4, j, 2), h3 = hermite_w(4, j, 3);
                // y pass: value-in-x (f, fy) and slope-in-x (fx, fxy) per corner column
                float G[3][6];
#pragma unroll
                for (int cx = 0; cx < 3; ++cx)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float* a = rec[0][cx];
                        const float* bb = rec[1][cx];
                        G[cx][c] = fmaf(h0, a[c], fmaf(h1, bb[c], fmaf(h2, a[6 + c], h3 * bb[6 + c])));
                        G[cx][3 + c] = fmaf(h0, a[3 + c], fmaf(h1, bb[3 + c], fmaf(h2, a[9 + c], h3 * bb[9 + c])));
                    }
                // x pass: pixel i has phase (i + 2) % 4 in cell g - 1 + (i >= 2)
                float o[12];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int jx = (i + 2) % 4, ka = (i + 2) / 4;
                    const float w0 = hermite_w(4, jx, 0), w1 = hermite_w(4, jx, 1);
                    const float w2 = hermite_w(4, jx, 2), w3 = hermite_w(4, jx, 3);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float part = fmaf(w1, G[ka + 1][c], fmaf(w2, G[ka][3 + c], w3 * G[ka + 1][3 + c]));
                        o[3 * i + c] = CLAMP ? fma_sat(w0, G[ka][c], part) : fmaf(w0, G[ka][c], part);
                    }
                }
#if UP_TMA_STORE
                // the warp's 128 pixels (1536 B) go to shared memory (double-buffered per
                // warp) and leave as one bulk copy (TMA engine), not 96 LSU stores
                const int sb_i = j & 1;
                float4* w4 = s_xp + (warp * 2 + sb_i) * 96;
                if (lane == 0)   // the bulk copy that last read this buffer has finished reading
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp(active);
                w4[3 * lane] = make_float4(o[0], o[1], o[2], o[3]);
                w4[3 * lane + 1] = make_float4(o[4], o[5], o[6], o[7]);
                w4[3 * lane + 2] = make_float4(o[8], o[9], o[10], o[11]);
                const int gw = (t % ngx) * kX4Groups;        // first group of this warp row
                float4* d4 = reinterpret_cast<float4*>(out + ((size_t)v * out_w + 4 * gw) * 3);
                const int nvalid = 3 * min(kX4Groups, out_w / 4 - gw);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp(active);
                if (lane == 0) {
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d4),
                                 "r"(smem_u32(w4)), "r"((uint32_t)nvalid * 16u)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
#else
                // transpose the warp's 128 pixels (1536 B) through shared memory so each
                // 16-byte store instruction writes 512 contiguous bytes (whole lines)
                float4* w4 = s_xp + warp * 96;
                w4[3 * lane] = make_float4(o[0], o[1], o[2], o[3]);
                w4[3 * lane + 1] = make_float4(o[4], o[5], o[6], o[7]);
                w4[3 * lane + 2] = make_float4(o[8], o[9], o[10], o[11]);
                __syncwarp(active);
                const int gw = (t % ngx) * kX4Groups;        // first group of this warp row
                float4* d4 = reinterpret_cast<float4*>(out + ((size_t)v * out_w + 4 * gw) * 3);
                const int nvalid = 3 * min(kX4Groups, out_w / 4 - gw);
                const int nact = __popc(active);   // active lanes are 0 .. nact-1
                for (int k = lane; k < nvalid; k += nact) __stcs(d4 + k, w4[k]);
                __syncwarp(active);
#endif
            }
        }
        __syncthreads();   // stage b is refilled by the prefetch of the next iteration
    }
#if UP_TMA_STORE
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
}

// x2 fast path (C2 / C4).  Same design as the x4 kernel: one thread owns one
// cell row n and one 4-pixel column group g, i.e. output rows 2n+1, 2n+2
// (phases 0, 1 of the cell row) x pixels 4g .. 4g+3 (phase 1 of cell 2g-1,
// phases 0, 1 of cell 2g, phase 0 of cell 2g+1).  Per corner column 2g-1 ..
// 2g+2 it reads the two corner records (rows n, n+1) once and keeps only the
// y-pass results G (value-in-x, slope-in-x) of both output rows; the x pass
// then runs in registers.  A CTA = 8 warps = 8 cell rows x 32 groups (16 x 128
// output pixels); persistent, TMA-staged source double buffer, TMA bulk stores.
constexpr int kX2Groups = 32;
#ifndef UP_X2_WARPS
#define UP_X2_WARPS 4
#endif
constexpr int kX2CellRows = UP_X2_WARPS;   // cell rows per tile = warps per CTA
constexpr int kX2SpanC = 2 * kX2Groups + 2;   // corner columns 2 g0 - 1 .. 2 g0 + 64
constexpr int kX2SpanR = kX2CellRows + 1;
#ifndef UP_X2_MINB
#define UP_X2_MINB (UP_X2_WARPS == 1 ? 14 : 2)
#endif

template <bool CLAMP>
__global__ void __launch_bounds__(32 * UP_X2_WARPS, UP_X2_MINB) upscale_x2_kernel(const float* __restrict__ src, int in_w,
                                                                     int in_h, float* __restrict__ out,
                                                                     int out_w, int out_h) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[2];
    constexpr size_t kStage = (size_t)kX2SpanR * kX2SpanC * 12;
    float* const s_src0 = reinterpret_cast<float*>(smem);
    float4* const s_xp = reinterpret_cast<float4*>(s_src0 + 2 * kStage);  // warps x 2 x 96 float4
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ngx = (out_w / 4 + kX2Groups - 1) / kX2Groups;
    const int ngy = (in_h + 1 + kX2CellRows - 1) / kX2CellRows;   // cell rows -1 .. in_h-1
    const int ntiles = ngx * ngy;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[0])));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    auto box = [&](int t, int& x0, int& ncols, int& y0, int& nrows) {
        const int g0 = (t % ngx) * kX2Groups, n0 = (t / ngx) * kX2CellRows - 1;
        x0 = max(2 * g0 - 1, 0);
        ncols = min(2 * g0 + 2 * kX2Groups, in_w - 1) - x0 + 1;
        y0 = max(n0, 0);
        nrows = min(n0 + kX2CellRows, in_h - 1) - y0 + 1;
    };
    auto issue = [&](int t, int b) {
        int x0, ncols, y0, nrows;
        box(t, x0, ncols, y0, nrows);
        const uint32_t row_bytes = (uint32_t)ncols * 48u;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar[b])),
                     "r"(row_bytes * (uint32_t)nrows)
                     : "memory");
        float* dst = s_src0 + (size_t)b * kStage;
        for (int r = 0; r < nrows; ++r)
            bulk_copy(dst + (size_t)r * kX2SpanC * 12, src + ((size_t)(y0 + r) * in_w + x0) * 12, row_bytes,
                      &s_bar[b]);
    };

    int t = blockIdx.x;
    if (t < ntiles && tid == 0) issue(t, 0);
    uint32_t phases = 0u;
    int sb_i = 0;   // this warp's store buffer (alternates per issued row store)
    for (int b = 0; t < ntiles; t += gridDim.x, b ^= 1) {
        if (t + (int)gridDim.x < ntiles && tid == 0) issue(t + gridDim.x, b ^ 1);
        mbar_wait(&s_bar[b], (phases >> b) & 1u);
        phases ^= 1u << b;
        int x0, ncols, y0, nrows;
        box(t, x0, ncols, y0, nrows);
        const int gw = (t % ngx) * kX2Groups;        // first group of this tile row
        const int g = gw + lane;
        const int n = (t / ngx) * kX2CellRows - 1 + warp;
        const unsigned active = __ballot_sync(0xffffffffu, g < out_w / 4);
        if (g < out_w / 4 && n < in_h) {
            const float* sb = s_src0 + (size_t)b * kStage;
            const int ra = clampi(n, 0, in_h - 1) - y0, rb = clampi(n + 1, 0, in_h - 1) - y0;
            // y pass per corner column 2g-1 .. 2g+2 (edge-clamped): G[j][cx] for output row 2n+1+j
            float G[2][4][6];
#pragma unroll
            for (int cx = 0; cx < 4; ++cx) {
                const int col = clampi(2 * g - 1 + cx, 0, in_w - 1) - x0;
                SPLAT_DCHECK(col >= 0 && col < ncols && col < kX2SpanC && ra >= 0 && rb < nrows && rb < kX2SpanR);
                const float4* pa = reinterpret_cast<const float4*>(sb + ((size_t)ra * kX2SpanC + col) * 12);
                const float4* pb = reinterpret_cast<const float4*>(sb + ((size_t)rb * kX2SpanC + col) * 12);
                const float4 a0 = pa[0], a1 = pa[1], a2 = pa[2];
                const float4 b0 = pb[0], b1 = pb[1], b2 = pb[2];
                const float a[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
                const float bb[12] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const float h0 = hermite_w(2, j, 0), h1 = hermite_w(2, j, 1);
                    const float h2 = hermite_w(2, j, 2), h3 = hermite_w(2, j, 3);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        G[j][cx][c] = fmaf(h0, a[c], fmaf(h1, bb[c], fmaf(h2, a[6 + c], h3 * bb[6 + c])));
                        G[j][cx][3 + c] = fmaf(h0, a[3 + c], fmaf(h1, bb[3 + c], fmaf(h2, a[9 + c], h3 * bb[9 + c])));
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {              // output row 2n + 1 + j
                const int v = 2 * n + 1 + j;
                if (v < 0 || v >= out_h) continue;
                // x pass: pixel i has phase (i + 1) % 2 in cell 2g - 1 + (i + 1) / 2
                float o[12];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int jx = (i + 1) % 2, ka = (i + 1) / 2;
                    const float w0 = hermite_w(2, jx, 0), w1 = hermite_w(2, jx, 1);
                    const float w2 = hermite_w(2, jx, 2), w3 = hermite_w(2, jx, 3);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float part =
                            fmaf(w1, G[j][ka + 1][c], fmaf(w2, G[j][ka][3 + c], w3 * G[j][ka + 1][3 + c]));
                        o[3 * i + c] = CLAMP ? fma_sat(w0, G[j][ka][c], part) : fmaf(w0, G[j][ka][c], part);
                    }
                }
                // the warp's 128 pixels (1536 B) leave as one TMA bulk store
                float4* w4 = s_xp + (warp * 2 + sb_i) * 96;
                sb_i ^= 1;
                if (lane == 0)   // the bulk store that last read this buffer has finished reading
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp(active);
                w4[3 * lane] = make_float4(o[0], o[1], o[2], o[3]);
                w4[3 * lane + 1] = make_float4(o[4], o[5], o[6], o[7]);
                w4[3 * lane + 2] = make_float4(o[8], o[9], o[10], o[11]);
                float4* d4 = reinterpret_cast<float4*>(out + ((size_t)v * out_w + 4 * gw) * 3);
                const int nvalid = 3 * min(kX2Groups, out_w / 4 - gw);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp(active);
                if (lane == 0) {
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d4),
                                 "r"(smem_u32(w4)), "r"((uint32_t)nvalid * 16u)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
        }
        // lanes past the image's right edge skip the stores: keep the store-buffer parity
        // warp-uniform (lane 0 stores whenever the warp stores)
        sb_i = __shfl_sync(0xffffffffu, sb_i, 0);
        __syncthreads();   // stage b is refilled by the prefetch of the next iteration
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

// Exact-x4 backward (out = 4 x in on both axes): source pixel x is corner b of
// cell x-1 for outputs 4x-2..4x+1 (phases 0..3) and corner a of cell x for
// outputs 4x+2..4x+5; at the borders the clamped corner coincides with x and
// both weights apply (the transpose of the edge replication, spline.py:232-243).
// Per CTA: 32 x 8 source pixels.  x pass: each warp stages whole output-row
// segments of the adjoint (coalesced) in shared memory and every lane contracts
// its source column's 8-wide window into value / slope partial sums; y pass: one
// source pixel per thread contracts 8 rows of those.
constexpr int kB4Cols = 32, kB4Rows = 8;
constexpr int kB4WinC = 4 * kB4Cols + 8, kB4WinR = 4 * kB4Rows + 8;
constexpr size_t kB4Smem = sizeof(float) * (8 * 2 * kB4WinC * 3 + kB4WinR * kB4Cols * 6);

__device__ __forceinline__ void x4_weights(int j, int x, int n, float& wv, float& ws) {
    if (j < 4) {   // x = corner b of cell x-1, phase j
        wv = hermite_w(4, j, 1);
        ws = hermite_w(4, j, 3);
        if (x == 0) {   // cell -1: corner a clamps onto x as well
            wv += hermite_w(4, j, 0);
            ws += hermite_w(4, j, 2);
        }
    } else {       // x = corner a of cell x, phase j-4
        wv = hermite_w(4, j - 4, 0);
        ws = hermite_w(4, j - 4, 2);
        if (x == n - 1) {   // cell n-1: corner b clamps onto x as well
            wv += hermite_w(4, j - 4, 1);
            ws += hermite_w(4, j - 4, 3);
        }
    }
}

__global__ void __launch_bounds__(256) upscale_bwd_x4_kernel(const float* __restrict__ adj,
                                                             float* __restrict__ dsrc, int in_w, int in_h) {
    extern __shared__ __align__(16) unsigned char b4_smem[];
    auto& s_row = *reinterpret_cast<float(*)[8][2][kB4WinC * 3]>(b4_smem);   // per warp, double-buffered
    auto& s_g = *reinterpret_cast<float(*)[kB4WinR][kB4Cols][6]>(b4_smem + sizeof(float) * 8 * 2 * kB4WinC * 3);
    const int out_w = 4 * in_w, out_h = 4 * in_h;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int X0 = blockIdx.x * kB4Cols, Y0 = blockIdx.y * kB4Rows;
    const int u0 = 4 * X0 - 2, v0 = 4 * Y0 - 2;
    const int x = X0 + lane;
    // adjoint row vi of the window (zero outside the image) -> buffer k of this warp, by cp.async
    auto load_row = [&](int vi, int k) {
        const int v = v0 + vi;
        const bool vok = v >= 0 && v < out_h;
        float* row = s_row[warp][k];
        for (int e = lane; e < kB4WinC * 3; e += 32) {
            const int u = u0 + e / 3;
            const bool ok = vok && u >= 0 && u < out_w;
            const float* src = ok ? adj + ((size_t)v * out_w + u0) * 3 + e : adj;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(row + e)), "l"(src),
                         "r"(ok ? 4 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float wv[8], ws[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x4_weights(j, x, in_w, wv[j], ws[j]);
    load_row(warp, 0);
    for (int vi = warp, k = 0; vi < kB4WinR; vi += 8, k ^= 1) {
        if (vi + 8 < kB4WinR) {   // the next row streams in while this one is contracted
            load_row(vi + 8, k ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        const float* row = s_row[warp][k];
        float a[3] = {0.f, 0.f, 0.f}, b[3] = {0.f, 0.f, 0.f};
        // the lane's 8 output pixels x 3 channels = 24 floats from byte 48 * lane: six 16-byte
        // loads, conflict-free per 8-lane phase (scalar loads at a 12-float lane stride: 4-way)
        float gv[24];
        {
            const float4* g4 = reinterpret_cast<const float4*>(row + 12 * lane);
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                const float4 t = g4[q];
                gv[4 * q] = t.x;
                gv[4 * q + 1] = t.y;
                gv[4 * q + 2] = t.z;
                gv[4 * q + 3] = t.w;
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                a[c] = fmaf(wv[j], gv[3 * j + c], a[c]);
                b[c] = fmaf(ws[j], gv[3 * j + c], b[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            s_g[vi][lane][c] = a[c];
            s_g[vi][lane][3 + c] = b[c];
        }
        __syncwarp();
    }
    __syncthreads();
    const int yi = threadIdx.x >> 5, xi = lane;
    const int y = Y0 + yi;
    if (y >= in_h || x >= in_w) return;
    float f[3] = {0, 0, 0}, fx[3] = {0, 0, 0}, fy[3] = {0, 0, 0}, fxy[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float hv, hs;
        x4_weights(i, y, in_h, hv, hs);
        const float* d = s_g[4 * yi + i][xi];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            f[c] = fmaf(hv, d[c], f[c]);
            fy[c] = fmaf(hs, d[c], fy[c]);
            fx[c] = fmaf(hv, d[3 + c], fx[c]);
            fxy[c] = fmaf(hs, d[3 + c], fxy[c]);
        }
    }
    float4* o = reinterpret_cast<float4*>(dsrc + ((size_t)y * in_w + x) * 12);
    o[0] = make_float4(f[0], f[1], f[2], fx[0]);
    o[1] = make_float4(fx[1], fx[2], fy[0], fy[1]);
    o[2] = make_float4(fy[2], fxy[0], fxy[1], fxy[2]);
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

size_t upscale_plan_bytes_impl(int out_w, int out_h) {
    size_t pw = (size_t)((out_w + kPlanPad - 1) / kPlanPad) * kPlanPad;
    size_t ph = (size_t)((out_h + kPlanPad - 1) / kPlanPad) * kPlanPad;
    return (pw + ph) * 20 + 64;
}

static PlanView plan_view(const void* plan, int out_w) {
    size_t pw = (size_t)((out_w + kPlanPad - 1) / kPlanPad) * kPlanPad;
    const char* b = (const char*)plan;
    PlanView v;
    v.cw = (const float4*)b;
    v.ci0 = (const int*)(b + pw * 16);
    v.rw = (const float4*)(b + pw * 20);
    return v;
}

int upscale_plan_impl(int in_w, int in_h, int out_w, int out_h, void* plan, cudaStream_t stream) {
    int pw = (out_w + kPlanPad - 1) / kPlanPad * kPlanPad;
    int ph = (out_h + kPlanPad - 1) / kPlanPad * kPlanPad;
    char* b = (char*)plan;
    float4* cw = (float4*)b;
    int* ci0 = (int*)(b + (size_t)pw * 16);
    float4* rw = (float4*)(b + (size_t)pw * 20);
    int* ri0 = (int*)(b + (size_t)pw * 20 + (size_t)ph * 16);
    plan_kernel<<<ceil_div(pw, 256), 256, 0, stream>>>(out_w, pw, (double)out_w / (double)in_w, ci0, cw); note_launch();
    plan_kernel<<<ceil_div(ph, 256), 256, 0, stream>>>(out_h, ph, (double)out_h / (double)in_h, ri0, rw); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

template <int F, bool CLAMP>
static int upscale_int_launch(const float* src, int in_w, int in_h, float* out, int out_w, int out_h,
                              cudaStream_t stream) {
    constexpr int TC = int_tile_cols(F);
    const int span_c = TC / F + 3, span_r = kUpRows / F + 3;
    const size_t smem = 2 * (size_t)span_r * span_c * 48 + (size_t)kUpRows * (TC / F + 2) * 24 + 8 * 96 * 16;
    static PerDevice<int> slots;   // resident CTAs per device (attribute set once per device)
    int cap = 0;
    const int rc = slots.get(cap, [smem](int& v) {
        int per_sm = 0, sms = 148;
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(upscale_int_kernel<F, CLAMP>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SPLAT_CUDA_CHECK(
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, upscale_int_kernel<F, CLAMP>, 256, smem));
        const int e = device_sms(sms);
        if (e != SPLAT_OK) return e;
        v = max(per_sm, 1) * sms;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    const int ntiles = ceil_div(out_w, TC) * ceil_div(out_h, kUpRows);
    const int grid = max(1, min(ntiles, cap));
    upscale_int_kernel<F, CLAMP><<<grid, 256, smem, stream>>>(src, in_w, in_h, out, out_w, out_h, span_c,
                                                              span_r); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

template <bool CLAMP>
static int upscale_x4_launch(const float* src, int in_w, int in_h, float* out, int out_w, int out_h,
                             cudaStream_t stream) {
    const size_t smem = 2 * (size_t)kX4SpanR * kX4SpanC * 48 + kX4CellRows * 96 * 16 * (UP_TMA_STORE ? 2 : 1);
    static PerDevice<int> slots;
    int cap = 0;
    const int rc = slots.get(cap, [smem](int& v) {
        int per_sm = 0, sms = 148;
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(upscale_x4_kernel<CLAMP>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SPLAT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, upscale_x4_kernel<CLAMP>,
                                                                       32 * kX4CellRows, smem));
        if (UP_X4_GRID_PER_SM > 0) per_sm = UP_X4_GRID_PER_SM;
        const int e = device_sms(sms);
        if (e != SPLAT_OK) return e;
        v = max(per_sm, 1) * sms;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    const int ntiles = ceil_div(out_w / 4, kX4Groups) * ceil_div(in_h + 1, kX4CellRows);
    const int grid = max(1, min(ntiles, cap));
    upscale_x4_kernel<CLAMP><<<grid, 32 * kX4CellRows, smem, stream>>>(src, in_w, in_h, out, out_w, out_h);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

template <bool CLAMP>
static int upscale_x2_launch(const float* src, int in_w, int in_h, float* out, int out_w, int out_h,
                             cudaStream_t stream) {
    const size_t smem = 2 * (size_t)kX2SpanR * kX2SpanC * 48 + kX2CellRows * 2 * 96 * 16;
    static PerDevice<int> slots;
    int cap = 0;
    const int rc = slots.get(cap, [smem](int& v) {
        int per_sm = 0, sms = 148;
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(upscale_x2_kernel<CLAMP>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SPLAT_CUDA_CHECK(
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, upscale_x2_kernel<CLAMP>, 32 * kX2CellRows, smem));
        const int e = device_sms(sms);
        if (e != SPLAT_OK) return e;
        v = max(per_sm, 1) * sms;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    const int ntiles = ceil_div(out_w / 4, kX2Groups) * ceil_div(in_h + 1, kX2CellRows);
    const int grid = max(1, min(ntiles, cap));
    upscale_x2_kernel<CLAMP><<<grid, 32 * kX2CellRows, smem, stream>>>(src, in_w, in_h, out, out_w, out_h);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int upscale_forward_impl(const float* src, int in_w, int in_h, float* out, int out_w, int out_h,
                         int clamp, const void* plan, cudaStream_t stream) {
#ifdef TIMING_SKIP_UP
    return SPLAT_OK;
#endif
    if (out_w <= 0 || out_h <= 0) return SPLAT_OK;
    if (out_w == 4 * in_w && out_h == 4 * in_h)
        return clamp ? upscale_x4_launch<true>(src, in_w, in_h, out, out_w, out_h, stream)
                     : upscale_x4_launch<false>(src, in_w, in_h, out, out_w, out_h, stream);
    if (out_w == 2 * in_w && out_h == 2 * in_h && (out_w & 3) == 0)
        return clamp ? upscale_x2_launch<true>(src, in_w, in_h, out, out_w, out_h, stream)
                     : upscale_x2_launch<false>(src, in_w, in_h, out, out_w, out_h, stream);
    if (out_w == 2 * in_w && out_h == 2 * in_h)
        return clamp ? upscale_int_launch<2, true>(src, in_w, in_h, out, out_w, out_h, stream)
                     : upscale_int_launch<2, false>(src, in_w, in_h, out, out_w, out_h, stream);
    double sx = (double)out_w / (double)in_w, sy = (double)out_h / (double)in_h;
    int tile_c = sx >= 4.0 ? 256 : (sx >= 2.0 ? 128 : 64);
    int span_c = (int)ceil((tile_c - 1) / sx) + 3;
    int span_r = (int)ceil((kUpRows - 1) / sy) + 3;
    if (span_c > in_w) span_c = in_w;
    if (span_r > in_h) span_r = in_h;
    size_t smem = 2 * (size_t)span_r * span_c * 48 + (size_t)kUpRows * span_c * 24 +
                  2 * ((size_t)tile_c * 20 + kUpRows * 20);
    static PerDevice<int> opt_in;
    int max_smem = 0;
    const int rc = opt_in.get(max_smem, [](int& v) {
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(upscale_fwd_kernel,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        v = 220 * 1024;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    if (smem > (size_t)max_smem) return set_error(SPLAT_ERR_DIMENSION, "upscale tile exceeds shared memory");
    int per_sm = 0;
    SPLAT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, upscale_fwd_kernel, 256, smem));
    int sms = 148;
    const int rs = device_sms(sms);
    if (rs != SPLAT_OK) return rs;
    int ntiles = ceil_div(out_w, tile_c) * ceil_div(out_h, kUpRows);
    int grid = per_sm * sms;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    PlanView pv = plan_view(plan, out_w);
    int pw = (out_w + kPlanPad - 1) / kPlanPad * kPlanPad;
    int ph = (out_h + kPlanPad - 1) / kPlanPad * kPlanPad;
    pv.ri0 = (const int*)((const char*)plan + (size_t)pw * 20 + (size_t)ph * 16);
    upscale_fwd_kernel<<<grid, 256, smem, stream>>>(src, in_w, in_h, out, out_w, out_h, clamp, pv, tile_c,
                                                    span_c, span_r); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int upscale_backward_impl(const float* adj, int out_w, int out_h, float* dsrc, int in_w, int in_h,
                          cudaStream_t stream) {
    double sx = (double)out_w / (double)in_w, sy = (double)out_h / (double)in_h;
    int max_u = (int)ceil((kBwCols + 2) * sx) + 8;
    int max_v = (int)ceil((kBwRows + 2) * sy) + 8;
    size_t smem = (size_t)(max_u + max_v) * sizeof(AxisMap) + (size_t)max_v * kBwCols * 6 * 4;
    if (out_w == 4 * in_w && out_h == 4 * in_h) {   // the x4 training path (C5)
        dim3 g4(ceil_div(in_w, kB4Cols), ceil_div(in_h, kB4Rows));
        static PerDevice<bool> b4_configured;
        bool b4ok = false;
        const int b4rc = b4_configured.get(b4ok, [](bool& v) {
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(upscale_bwd_x4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)kB4Smem));
            v = true;
            return SPLAT_OK;
        });
        if (b4rc != SPLAT_OK) return b4rc;
        upscale_bwd_x4_kernel<<<g4, 256, kB4Smem, stream>>>(adj, dsrc, in_w, in_h);
        note_launch();
        SPLAT_CUDA_CHECK(cudaGetLastError());
        return SPLAT_OK;
    }
    static PerDevice<bool> configured;
    bool ok = false;
    const int rc = configured.get(ok, [](bool& v) {
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(upscale_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              200 * 1024));
        v = true;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    if (smem > 200 * 1024) return set_error(SPLAT_ERR_DIMENSION, "upscale backward tile too large");
    dim3 grid(ceil_div(in_w, kBwCols), ceil_div(in_h, kBwRows));
    upscale_bwd_kernel<<<grid, 256, smem, stream>>>(adj, out_w, out_h, dsrc, in_w, in_h, sx, sy, max_u, max_v);
    note_launch();
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
