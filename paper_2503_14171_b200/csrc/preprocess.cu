// Scene preparation, per-view preprocessing and tile binning.
//
//   scene_prepare  : sort_by_depth (raster_forward.py:59-61) as a stable
//                    device radix sort of order-preserving float64 keys, and the
//                    view-independent terms of prepare_scene (raster_forward.py:
//                    86-110) evaluated once per scene.
//   preprocess     : per-view rescale / conic / cull-ellipse bbox
//                    (raster_forward.py:79-123) with the reference's float64
//                    expression trees and explicitly rounded (non-fused) ops, so
//                    the integer bboxes and validity are bit-identical.
//   emit + sort    : duplicate (tile, rank) pairs in rank order, stable radix
//                    sort on the tile bits, per-tile [start, end) ranges
//                    (bin_tiles, raster_forward.py:136-149).
#include <cmath>

#include "kernels.cuh"

namespace splat {

namespace {

inline size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

// ---- scene constants ------------------------------------------------------

__global__ void depth_keys_kernel(const double* __restrict__ depths, int64_t n,
                                  uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = depths[i];
    if (d == 0.0) d = 0.0;  // -0.0 and +0.0 compare equal in argsort
    uint64_t b = (uint64_t)__double_as_longlong(d);
    // order-preserving map: flip all bits of negatives, the sign bit of positives
    keys[i] = (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
    idx[i] = (uint32_t)i;
}

__global__ void scene_const_kernel(int64_t n, const uint32_t* __restrict__ order,
                                   const double* __restrict__ means, const double* __restrict__ ls,
                                   const double* __restrict__ rot, const double* __restrict__ logit,
                                   const double* __restrict__ colors, int32_t* __restrict__ order_out,
                                   int32_t* __restrict__ rank_of,
                                   double* __restrict__ mean_r, double* __restrict__ n00,
                                   double* __restrict__ n01, double* __restrict__ n11,
                                   double* __restrict__ e1e2, double* __restrict__ sigma,
                                   double* __restrict__ q, float4* __restrict__ color) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t s = order[r];
    order_out[r] = (int32_t)s;
    rank_of[s] = (int32_t)r;
    mean_r[2 * r] = means[2 * s];
    mean_r[2 * r + 1] = means[2 * s + 1];
    // raster_forward.py:89, 94-98 — same operation order, no contraction
    double sg = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-logit[s])));
    double e1 = exp(__dmul_rn(-2.0, ls[2 * s]));
    double e2 = exp(__dmul_rn(-2.0, ls[2 * s + 1]));
    double c = cos(rot[s]);
    double sn = sin(rot[s]);
    n00[r] = __dadd_rn(__dmul_rn(__dmul_rn(e1, c), c), __dmul_rn(__dmul_rn(e2, sn), sn));
    n01[r] = __dmul_rn(__dmul_rn(__dsub_rn(e1, e2), sn), c);
    n11[r] = __dadd_rn(__dmul_rn(__dmul_rn(e1, sn), sn), __dmul_rn(__dmul_rn(e2, c), c));
    e1e2[r] = __dmul_rn(e1, e2);
    sigma[r] = sg;
    // raster_forward.py:107: log(max(sigma / ALPHA_CULL, 1))
    double ratio = __ddiv_rn(sg, kAlphaCull);
    q[r] = log(ratio > 1.0 ? ratio : 1.0);
    color[r] = make_float4((float)colors[3 * s], (float)colors[3 * s + 1], (float)colors[3 * s + 2],
                           0.f);
}

// ---- per-view preprocess ----------------------------------------------------

__device__ __forceinline__ int64_t clip64(int64_t v, int64_t lo, int64_t hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

__global__ void preprocess_kernel(SceneConst sc, ViewConst vc, int width, int height,
                                  PackF* __restrict__ pack, short4* __restrict__ bboxes,
                                  uint32_t* __restrict__ touched) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= sc.n) return;
    // raster_forward.py:86 means[order] * [kx, ky] (view pan applied first)
    double mx = __dmul_rn(__dsub_rn(sc.mean[2 * r], vc.ox), vc.kx);
    double my = __dmul_rn(__dsub_rn(sc.mean[2 * r + 1], vc.oy), vc.ky);
    // raster_forward.py:99-101
    double a = __ddiv_rn(sc.n00[r], vc.c00);
    double b = __ddiv_rn(sc.n01[r], vc.c01);
    double c = __ddiv_rn(sc.n11[r], vc.c11);
    double sg = sc.sigma[r];
    double q = sc.q[r];
    // raster_forward.py:108-121
    double det = __ddiv_rn(sc.e1e2[r], vc.cdet);
    double rx = __dsqrt_rn(__ddiv_rn(__dmul_rn(q, c), det));
    double ry = __dsqrt_rn(__ddiv_rn(__dmul_rn(q, a), det));
    int64_t x0 = clip64((int64_t)floor(__dsub_rn(mx, rx)) - 1, 0, width);
    int64_t x1 = clip64((int64_t)ceil(__dadd_rn(mx, rx)) + 1, 0, width);
    int64_t y0 = clip64((int64_t)floor(__dsub_rn(my, ry)) - 1, 0, height);
    int64_t y1 = clip64((int64_t)ceil(__dadd_rn(my, ry)) + 1, 0, height);
    bool valid = (sg >= kAlphaCull) && (x1 > x0) && (y1 > y0);
    bboxes[r] = make_short4((short)x0, (short)x1, (short)y0, (short)y1);
    uint32_t cnt = 0;
    if (valid) {
        uint32_t tx0 = (uint32_t)x0 / kTile, tx1 = (uint32_t)(x1 - 1) / kTile;
        uint32_t ty0 = (uint32_t)y0 / kTile, ty1 = (uint32_t)(y1 - 1) / kTile;
        cnt = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
    }
    touched[r] = cnt;
    PackF p;
    p.mxh = (float)mx;
    p.mxl = (float)(mx - (double)p.mxh);
    p.myh = (float)my;
    p.myl = (float)(my - (double)p.myh);
    p.a = (float)a;
    p.b = (float)b;
    p.c = (float)c;
    p.sigma = (float)sg;
    p.qcull = (float)q;
    p.qclamp = (float)log(sg / kAlphaClamp);
    p.pad0 = (float)(b / a);  // ellipse-rectangle test: edge minimisers (raster_fwd.cu)
    p.pad1 = (float)(b / c);
    // cull-ellipse half extents (the reference's rx, ry) with a 1e-3 px + 1e-5 relative
    // margin: every pixel centre that can contribute lies in mean +- (ex, ey)
    p.ex = (float)(rx * (1.0 + 1e-5) + 1e-3);
    p.ey = (float)(ry * (1.0 + 1e-5) + 1e-3);
    p.pad2 = 0.f;
    p.pad3 = 0.f;
    pack[r] = p;
}

// Pair emission, warp-cooperative: the 32 ranks of a warp own the contiguous
// slot range [offsets[r0], offsets[r0+32]); lane l writes slots l, l+32, ...
// (coalesced) after a 5-step shuffle binary search for the slot's owner rank.
// Pairs of one rank are written in row-major tile order, ranks ascending
// (raster_forward.py:141-148 append order).
__global__ void emit_pairs_kernel(int64_t n, const short4* __restrict__ bboxes,
                                  const uint32_t* __restrict__ touched,
                                  const uint32_t* __restrict__ offsets, int ntx, int64_t cap,
                                  uint32_t* __restrict__ keys, uint32_t* __restrict__ ranks,
                                  uint32_t* __restrict__ counters) {
    const int lane = threadIdx.x & 31;
    const int64_t r0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane;
    if (r0 >= n) return;
    const int64_t r = r0 + lane;
    const bool have = r < n;
    const uint32_t cnt = have ? touched[r] : 0u;
    const uint32_t off = have ? offsets[r] : 0u;
    const uint32_t off0 = __shfl_sync(0xffffffffu, off, 0);
    const uint32_t incl = (have ? off - off0 : 0u) + cnt;          // inclusive end of this lane's slots
    uint32_t warp_total = incl;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) warp_total = max(warp_total, __shfl_xor_sync(0xffffffffu, warp_total, d));
    const uint32_t key = have ? incl : 0xffffffffu;                // monotone search key
    int tx0 = 0, ty0 = 0, nx = 1;
    if (cnt) {
        const short4 bb = bboxes[r];
        tx0 = bb.x / kTile;
        ty0 = bb.z / kTile;
        nx = (bb.y - 1) / kTile - tx0 + 1;
    }
    if ((int64_t)off0 + warp_total > cap && lane == 0) {
        atomicOr(&counters[1], 1u);
        atomicOr(&counters[4], 1u);  // sticky until the caller clears it
    }
    for (uint32_t sb = 0; sb < warp_total; sb += 32) {   // uniform trip count: full-warp shuffles
        const uint32_t s = sb + lane;
        // owner = first lane whose inclusive end exceeds s
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t e = __shfl_sync(0xffffffffu, key, lo + step - 1);
            if (e <= s) lo += step;
        }
        const uint32_t start = __shfl_sync(0xffffffffu, incl - cnt, lo);
        const int otx0 = __shfl_sync(0xffffffffu, tx0, lo);
        const int oty0 = __shfl_sync(0xffffffffu, ty0, lo);
        const int onx = __shfl_sync(0xffffffffu, nx, lo);
        const int64_t slot = (int64_t)off0 + s;
        if (s < warp_total && slot < cap) {
            const uint32_t li = s - start;
            const int ty = oty0 + (int)(li / (uint32_t)onx), tx = otx0 + (int)(li % (uint32_t)onx);
            keys[slot] = (uint32_t)(ty * ntx + tx);
            ranks[slot] = (uint32_t)(r0 + lo);
        }
    }
}

__global__ void tile_ranges_kernel(const uint32_t* __restrict__ keys, const uint32_t* counters,
                                   int64_t cap, int ntiles, uint32_t* __restrict__ ranges) {
    int64_t np = counters[0];
    if (np > cap) np = cap;
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= np) return;
    uint32_t k = keys[j];
    if (k >= (uint32_t)ntiles) return;  // defensive: never index past the range table
    if (j == 0 || keys[j - 1] != k) ranges[2 * k] = (uint32_t)j;
    if (j == np - 1 || keys[j + 1] != k) ranges[2 * k + 1] = (uint32_t)(j + 1);
}

__global__ void pack64_kernel(SceneConst sc, ViewConst vc, double* __restrict__ out) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= sc.n) return;
    double* o = out + 6 * r;
    o[0] = __dmul_rn(__dsub_rn(sc.mean[2 * r], vc.ox), vc.kx);
    o[1] = __dmul_rn(__dsub_rn(sc.mean[2 * r + 1], vc.oy), vc.ky);
    o[2] = __ddiv_rn(sc.n00[r], vc.c00);
    o[3] = __ddiv_rn(sc.n01[r], vc.c01);
    o[4] = __ddiv_rn(sc.n11[r], vc.c11);
    o[5] = sc.sigma[r];
}

int tile_key_bits(int ntiles) {
    int bits = 0;
    while ((1 << bits) < ntiles) ++bits;
    return bits == 0 ? 8 : ((bits + 7) / 8) * 8;
}

}  // namespace

// ---- layouts ----------------------------------------------------------------

ConstLayout const_layout(int64_t n) {
    ConstLayout L;
    size_t o = 0;
    size_t nn = (size_t)(n > 0 ? n : 1);
    L.order = o; o = align_up(o + nn * 4);
    L.rank_of = o; o = align_up(o + nn * 4);
    L.mean = o; o = align_up(o + nn * 16);
    L.n00 = o; o = align_up(o + nn * 8);
    L.n01 = o; o = align_up(o + nn * 8);
    L.n11 = o; o = align_up(o + nn * 8);
    L.e1e2 = o; o = align_up(o + nn * 8);
    L.sigma = o; o = align_up(o + nn * 8);
    L.q = o; o = align_up(o + nn * 8);
    L.color = o; o = align_up(o + nn * 16);
    L.total = o;
    return L;
}

SceneConst scene_const_view(const void* buf, int64_t n) {
    ConstLayout L = const_layout(n);
    const char* b = (const char*)buf;
    SceneConst s;
    s.n = n;
    s.order = (const int32_t*)(b + L.order);
    s.rank_of = (const int32_t*)(b + L.rank_of);
    s.mean = (const double*)(b + L.mean);
    s.n00 = (const double*)(b + L.n00);
    s.n01 = (const double*)(b + L.n01);
    s.n11 = (const double*)(b + L.n11);
    s.e1e2 = (const double*)(b + L.e1e2);
    s.sigma = (const double*)(b + L.sigma);
    s.q = (const double*)(b + L.q);
    s.color = (const float4*)(b + L.color);
    return s;
}

FrameLayout frame_layout(int64_t n, int width, int height, int64_t cap) {
    FrameLayout L;
    L.n = n;
    L.cap = cap;
    L.width = width;
    L.height = height;
    L.ntx = ceil_div(width, kTile);
    L.nty = ceil_div(height, kTile);
    size_t nn = (size_t)(n > 0 ? n : 1);
    size_t cc = (size_t)(cap > 0 ? cap : 1);
    size_t o = 0;
    L.bboxes = o; o = align_up(o + nn * 8);
    L.touched = o; o = align_up(o + (nn + 1) * 4);
    L.offsets = o; o = align_up(o + (nn + 1) * 4);
    L.scan_scratch = o; o = align_up(o + (size_t)scan_scratch_words(n + 1) * 4);
    L.keys0 = o; o = align_up(o + cc * 4);
    L.vals0 = o; o = align_up(o + cc * 4);
    L.keys1 = o; o = align_up(o + cc * 4);
    L.vals1 = o; o = align_up(o + cc * 4);
    L.sort_scratch = o; o = align_up(o + (size_t)radix_scratch_words(cap) * 4);
    L.ranges = o; o = align_up(o + (size_t)L.ntx * L.nty * 8);
    L.counters = o; o = align_up(o + 16 * 4);
    L.fixup = o; o = align_up(o + (size_t)width * height * 4 + 4);
    L.pack = o; o = align_up(o + nn * sizeof(PackF));
    L.total = o;
    return L;
}

ViewConst make_view_const(const splat_view_t& v) {
    ViewConst c;
    c.kx = v.kx;
    c.ky = v.ky;
    c.ox = v.ox;
    c.oy = v.oy;
    // Python evaluates these left to right in float64 (raster_forward.py:99-101, 108)
    c.c00 = (2.0 * v.kx) * v.kx;
    c.c01 = (2.0 * v.kx) * v.ky;
    c.c11 = (2.0 * v.ky) * v.ky;
    c.cdet = (((4.0 * v.kx) * v.kx) * v.ky) * v.ky;
    for (int i = 0; i < 3; ++i) c.bg[i] = (float)v.bg[i];
    return c;
}

// ---- launchers --------------------------------------------------------------

size_t scene_workspace_bytes_impl(int64_t n) {
    size_t nn = (size_t)(n > 0 ? n : 1);
    return align_up(nn * 8) * 2 + align_up(nn * 4) * 2 + align_up((size_t)radix_scratch_words(n) * 4);
}

int scene_prepare_impl(const splat_scene_t& s, void* const_buf, void* ws, cudaStream_t stream) {
    int64_t n = s.n;
    if (n == 0) return SPLAT_OK;
    size_t nn = (size_t)n;
    char* w = (char*)ws;
    uint64_t* k0 = (uint64_t*)w;
    uint64_t* k1 = (uint64_t*)(w + align_up(nn * 8));
    uint32_t* v0 = (uint32_t*)(w + 2 * align_up(nn * 8));
    uint32_t* v1 = (uint32_t*)(w + 2 * align_up(nn * 8) + align_up(nn * 4));
    uint32_t* scratch = (uint32_t*)(w + 2 * align_up(nn * 8) + 2 * align_up(nn * 4));
    int blocks = (int)((n + 255) / 256);
    depth_keys_kernel<<<blocks, 256, 0, stream>>>(s.depths, n, k0, v0); note_launch();
    int alt = 0;
    radix_sort_pairs<uint64_t>(k0, v0, k1, v1, nullptr, n, n, 0, 64, scratch, &alt, stream);
    const uint32_t* order = alt ? v1 : v0;
    ConstLayout L = const_layout(n);
    char* b = (char*)const_buf;
    scene_const_kernel<<<blocks, 256, 0, stream>>>(
        n, order, s.means, s.log_scales, s.rotations, s.opacity_logits, s.colors,
        (int32_t*)(b + L.order), (int32_t*)(b + L.rank_of), (double*)(b + L.mean), (double*)(b + L.n00),
        (double*)(b + L.n01),
        (double*)(b + L.n11), (double*)(b + L.e1e2), (double*)(b + L.sigma), (double*)(b + L.q),
        (float4*)(b + L.color)); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

// Recompute the view-independent terms for updated parameters, keeping the
// existing depth order (depths are not optimised: fit.py:163-166).
int scene_refresh_impl(const splat_scene_t& s, void* const_buf, cudaStream_t stream) {
    const int64_t n = s.n;
    if (n == 0) return SPLAT_OK;
    ConstLayout L = const_layout(n);
    char* b = (char*)const_buf;
    scene_const_kernel<<<(int)((n + 255) / 256), 256, 0, stream>>>(
        n, (const uint32_t*)(b + L.order), s.means, s.log_scales, s.rotations, s.opacity_logits, s.colors,
        (int32_t*)(b + L.order), (int32_t*)(b + L.rank_of), (double*)(b + L.mean), (double*)(b + L.n00),
        (double*)(b + L.n01),
        (double*)(b + L.n11), (double*)(b + L.e1e2), (double*)(b + L.sigma), (double*)(b + L.q),
        (float4*)(b + L.color)); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int launch_preprocess(const SceneConst& sc, const ViewConst& vc, const FrameLayout& L, char* ws,
                      cudaStream_t stream) {
    uint32_t* counters = (uint32_t*)(ws + L.counters);
    SPLAT_CUDA_CHECK(cudaMemsetAsync(counters, 0, 4 * 4, stream));  // [4..] are sticky
    if (sc.n == 0) return SPLAT_OK;
    int blocks = (int)((sc.n + 255) / 256);
    preprocess_kernel<<<blocks, 256, 0, stream>>>(sc, vc, L.width, L.height,
                                                  (PackF*)(ws + L.pack), (short4*)(ws + L.bboxes),
                                                  (uint32_t*)(ws + L.touched)); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int launch_binning(const FrameLayout& L, char* ws, cudaStream_t stream) {
    uint32_t* counters = (uint32_t*)(ws + L.counters);
    uint32_t* ranges = (uint32_t*)(ws + L.ranges);
    int ntiles = L.ntx * L.nty;
    SPLAT_CUDA_CHECK(cudaMemsetAsync(ranges, 0, (size_t)ntiles * 8, stream));
    if (L.n == 0) return SPLAT_OK;
    uint32_t* touched = (uint32_t*)(ws + L.touched);
    uint32_t* offsets = (uint32_t*)(ws + L.offsets);
    exclusive_scan_u32(touched, offsets, L.n, (uint32_t*)(ws + L.scan_scratch), &counters[0], stream);
    int blocks = (int)((L.n + 255) / 256);
    uint32_t* k0 = (uint32_t*)(ws + L.keys0);
    uint32_t* v0 = (uint32_t*)(ws + L.vals0);
    uint32_t* k1 = (uint32_t*)(ws + L.keys1);
    uint32_t* v1 = (uint32_t*)(ws + L.vals1);
    emit_pairs_kernel<<<blocks, 256, 0, stream>>>(L.n, (const short4*)(ws + L.bboxes), touched,
                                                  offsets, L.ntx, L.cap, k0, v0, counters); note_launch();
    int alt = 0;
    radix_sort_pairs<uint32_t>(k0, v0, k1, v1, counters, 0, L.cap, 0, tile_key_bits(ntiles),
                               (uint32_t*)(ws + L.sort_scratch), &alt, stream);
    const uint32_t* keys = alt ? k1 : k0;
    int rblocks = (int)((L.cap + 255) / 256);
    if (rblocks > 0)
        tile_ranges_kernel<<<rblocks, 256, 0, stream>>>(keys, counters, L.cap, ntiles, ranges); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int launch_pack64(const SceneConst& sc, const ViewConst& vc, double* out, cudaStream_t stream) {
    if (sc.n == 0) return SPLAT_OK;
    pack64_kernel<<<(int)((sc.n + 255) / 256), 256, 0, stream>>>(sc, vc, out); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

bool sorted_in_alt(int ntiles) { return (tile_key_bits(ntiles) / 8) % 2 == 1; }

}  // namespace splat
