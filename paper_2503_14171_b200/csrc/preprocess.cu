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
//   binning      : per-4096-rank-block tile histograms, column scan, staged
//                    counting-sort fill -> per-tile lists in the reference's
//                    append order and [start, end) ranges (bin_tiles,
//                    raster_forward.py:136-149); see "tile binning" below.
#include <cmath>
#ifdef TIMING_SKIP_BIN
#include <set>
#endif

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

#ifndef PACK_ALL
#define PACK_ALL 0
#endif
#ifndef PRE_THREADS
#define PRE_THREADS 64   // 64 x 46 registers fit beside a persistent raster CTA set (C3 1896 -> 1911 frames/s)
#endif
#ifndef PRE_MINB
#define PRE_MINB 1
#endif
__global__ void __launch_bounds__(PRE_THREADS, PRE_MINB) preprocess_kernel(SceneConst sc, ViewConst vc, int width, int height,
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
    p.nb2 = -2.f * (float)b;   // exact scaling of the float32 conic b
    p.c = (float)c;
    // al = 2^(log2 sigma - log2(e) qf): one FFMA + EX2 (the float32 rounding of log2 sigma,
    // |log2 sigma| <= 8, is <= 2^-22 absolute, inside eval_fast's rel budget)
    p.l2sig = (float)log2(sg);
    // eval_fast's tests qf > qcull + tol etc. with tol = (s + qcull) 2^-19 become
    // qf - 2^-19 s > cull_hi etc.: the qcull-relative part of the tolerance is added here
    // exactly (double) and rounded outward, so the float32 path does one FMA per side.
    // qcull and qclamp are the float32 values the tolerance was designed around (qclamp:
    // ln(sigma / 0.999) in float32, <= 2 ulp; 2^-19 qcull >= 16 ulp(qclamp) when clamping
    // is possible, qclamp < qcull).
    {
        const float qc = (float)q;
        const float ql = logf((float)sg / (float)kAlphaClamp);
        const double tq = (double)qc * 1.9073486328125e-06;   // 2^-19 qcull, exact
        p.cull_hi = __double2float_ru((double)qc + tq);
        p.cull_lo = __double2float_rd((double)qc - tq);
        p.clamp_hi = __double2float_ru((double)ql + tq);
        p.clamp_lo = __double2float_rd((double)ql - tq);
    }
    // cull-ellipse half extents (the reference's rx, ry) with a 1e-3 px + 1e-5 relative
    // margin: every pixel centre that can contribute lies in mean +- (ex, ey)
    p.ex = (float)(rx * (1.0 + 1e-5) + 1e-3);
    p.ey = (float)(ry * (1.0 + 1e-5) + 1e-3);
    // group pre-filter of the rasterizer (Q-norm triangle inequality): a 4x2 block of pixel
    // centres with centre G can hold a pixel with Q(p - m) <= q only if
    // sqrt(Q(G - m)) <= sqrt(q) + max_{|u|<=1.5,|v|<=.5} sqrt(Q(u, v)); pad2 is that bound squared,
    // widened by 1e-5 relative + 1e-4 (float32 conic and test rounding are far below)
    {
        const double rq = sqrt(2.25 * a + 0.25 * c + 1.5 * fabs(b));
        const double rt = sqrt(q) + rq;
        p.pad2 = (float)(rt * rt * (1.0 + 1e-5) + 1e-4);
    }
    p.pad3 = 0.f;
    // only splats that reach a tile list are ever read through the pack (raster, fix-up,
    // backward): off-screen / culled splats skip the 64-byte store
#if PACK_ALL
    pack[r] = p;
#else
    if (cnt != 0) pack[r] = p;
#endif
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

// ---- tile binning ------------------------------------------------------------
// bin_tiles (raster_forward.py:136-149) appends each valid rank, in rank order,
// to the list of every tile its bbox touches.  Ranks are cut into blocks of
// kBinBlock consecutive ranks; then
//   1. count: per block, a tile histogram in shared memory -> row of hist[block][tile]
//   2. column scan: per tile, exclusive prefix over blocks (two levels:
//      groups of kColGroup rows, then the group sums) + the tile totals
//   3. scan of the tile totals -> each list's [start, end)
//   4. fill: each block counting-sorts its pairs by tile in shared memory,
//      sorts each (block, tile) run by rank (runs are a few entries long) and
//      writes it at start[tile] + prefix[block][tile]: lists come out exactly in
//      the reference's append order, deterministically, without a global sort.
// Tile grids too large for the shared-memory tables fall back to per-pair
// global atomics + a per-tile sort (same result).

#ifndef BIN_BLOCK
#define BIN_BLOCK 4096
#endif
#ifndef BIN_STAGE
#define BIN_STAGE 16384
#endif
constexpr int kBinBlock = BIN_BLOCK;   // ranks per block (a histogram row) on large grids
#ifndef BIN_THREADS
#define BIN_THREADS 1024
#endif
constexpr int kBinThreads = BIN_THREADS;   // kBinBlock / kBinThreads ranks per thread
constexpr int kBinRPT = kBinBlock / kBinThreads;
// Small grids bin in half-size blocks: a block's (block, tile) runs are then half as long, and
// the fill's per-entry rank count within its run (quadratic in the run length) shrinks 4x,
// while the per-block tile tables stay small (C5, 510 tiles: fill 72 -> 52 us; C3, 2040
// tiles, keeps 4096: 2048 there costs 4.6 us of extra table work per view).
// Small scenes halve the blocks further until there is at least one block per SM (C2:
// 200k splats were 49 blocks of 4096 for 148 SMs).
constexpr int kBinSmallGridTiles = 1024;
constexpr int64_t kBinMinBlocks = 148;
static_assert(kBinRPT >= 4 && kBinRPT % 4 == 0, "block sizes kBinRPT, /2, /4 ranks per thread");
static int bin_rpt(int ntiles, int64_t n) {
    int r = ntiles < kBinSmallGridTiles ? kBinRPT / 2 : kBinRPT;
    while (r > kBinRPT / 4 && (n + (int64_t)r * kBinThreads - 1) / ((int64_t)r * kBinThreads) < kBinMinBlocks) r /= 2;
    return r;
}
constexpr int kBinStage = BIN_STAGE;   // staged pairs per pass of the fill (2 CTAs/SM fit)
constexpr int kColGroup = 16;        // rows per column-scan group
constexpr int kBinSmemMax = 200 * 1024;

__device__ __forceinline__ void tile_rect(short4 bb, int& tx0, int& tx1, int& ty0, int& ty1) {
    tx0 = bb.x / kTile;
    tx1 = (bb.y - 1) / kTile;
    ty0 = bb.z / kTile;
    ty1 = (bb.w - 1) / kTile;
}

__device__ __forceinline__ void write_range(int t, const uint32_t* tile_start, const uint32_t* tile_count,
                                            uint32_t* ranges, int64_t cap) {
    const uint32_t st = tile_start[t];
    ranges[2 * t] = (uint32_t)min((int64_t)st, cap);
    ranges[2 * t + 1] = (uint32_t)min((int64_t)st + tile_count[t], cap);
}

__device__ __forceinline__ void put_rank(uint32_t pos, uint32_t r, int64_t cap, uint32_t* ranks, uint32_t* counters) {
    if ((int64_t)pos < cap) {
        ranks[pos] = r;
    } else {
        atomicOr(&counters[1], 1u);
        atomicOr(&counters[4], 1u);  // sticky until the caller clears it
    }
}

// Tile rectangle of rank r, or an empty one (tx1 < tx0) for untouched ranks.
struct BinRect {
    int r, tx0, tx1, ty0, ty1;
};

__device__ __forceinline__ BinRect bin_rect(int64_t n, int64_t r, const short4* bboxes, const uint32_t* touched) {
    BinRect q{(int)r, 0, -1, 0, -1};
    if (r < n) {
        const uint32_t c = __ldg(touched + r);   // both loads in flight together
        const short4 bb = __ldg(bboxes + r);
        if (c != 0) tile_rect(bb, q.tx0, q.tx1, q.ty0, q.ty1);
    }
    return q;
}

template <int RPT>
__global__ void __launch_bounds__(kBinThreads) count_rows_kernel(int64_t n, const short4* __restrict__ bboxes,
                                                                 const uint32_t* __restrict__ touched, int ntx,
                                                                 int ntiles, uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t h[];
    constexpr int64_t kBlk = (int64_t)RPT * kBinThreads;
    const int64_t nblk = (n + kBlk - 1) / kBlk;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        for (int t = threadIdx.x; t < ntiles; t += blockDim.x) h[t] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const BinRect q = bin_rect(n, blk * kBlk + j * kBinThreads + threadIdx.x, bboxes, touched);
            for (int ty = q.ty0; ty <= q.ty1; ++ty)
                for (int tx = q.tx0; tx <= q.tx1; ++tx) atomicAdd(&h[ty * ntx + tx], 1u);
        }
        __syncthreads();
        uint32_t* row = hist + (size_t)blk * ntiles;
        for (int t = threadIdx.x; t < ntiles; t += blockDim.x) row[t] = h[t];
        __syncthreads();
    }
}

// Per (group, tile): exclusive prefix within the group's rows (into pre; hist keeps the
// counts, which the fill uses as its block's histogram) and the group sum.
__global__ void colscan_rows_kernel(int ntiles, int nrows, const uint32_t* __restrict__ hist,
                                    uint32_t* __restrict__ pre, uint32_t* __restrict__ part) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int g = blockIdx.y;
    if (t >= ntiles) return;
    const int r0 = g * kColGroup, nr = min(kColGroup, nrows - r0);
    const uint32_t* col = hist + (size_t)r0 * ntiles + t;
    uint32_t* out = pre + (size_t)r0 * ntiles + t;
    uint32_t v[kColGroup];
#pragma unroll
    for (int i = 0; i < kColGroup; ++i) v[i] = i < nr ? col[(size_t)i * ntiles] : 0u;   // all loads in flight
    uint32_t run = 0;
#pragma unroll
    for (int i = 0; i < kColGroup; ++i) {
        if (i < nr) out[(size_t)i * ntiles] = run;
        run += v[i];
    }
    part[(size_t)g * ntiles + t] = run;
}

// Per tile: exclusive prefix over the group sums (in place) and the tile total.
__global__ void colscan_groups_kernel(int ntiles, int ngroups, uint32_t* __restrict__ part,
                                      uint32_t* __restrict__ tile_count, uint32_t* __restrict__ counters) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) counters[5] = 0;
    if (t >= ntiles) return;
    uint32_t run = 0;
    for (int g0 = 0; g0 < ngroups; g0 += 16) {   // 16 loads in flight, then the prefix
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = g0 + i < ngroups ? part[(size_t)(g0 + i) * ntiles + t] : 0u;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (g0 + i < ngroups) part[(size_t)(g0 + i) * ntiles + t] = run;
            run += v[i];
        }
    }
    tile_count[t] = run;
}

// In-place exclusive scan of a[0, m) by the whole CTA; returns the total.
__device__ uint32_t block_exclusive_scan(uint32_t* a, int m, uint32_t* wsum) {
    const int per = (m + blockDim.x - 1) / blockDim.x;
    const int i0 = min((int)threadIdx.x * per, m), i1 = min(i0 + per, m);
    uint32_t local = 0;
    for (int i = i0; i < i1; ++i) local += a[i];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = local;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += v;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        const uint32_t v = lane < nw ? wsum[lane] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += u;
        }
        if (lane < nw) wsum[lane] = x - v;   // exclusive warp offsets
        if (lane == 31) wsum[32] = x;        // total
    }
    __syncthreads();
    uint32_t run = wsum[wid] + inc - local;
    for (int i = i0; i < i1; ++i) {
        const uint32_t v = a[i];
        a[i] = run;
        run += v;
    }
    const uint32_t total = wsum[32];
    __syncthreads();
    return total;
}

static_assert(kTile == 16, "tile rectangles below use shifts");

// Packed bbox of rank r, all-zero (an empty tile rectangle) for untouched ranks.
__device__ __forceinline__ short4 bin_box(int64_t n, int64_t r, const short4* bboxes, const uint32_t* touched) {
    short4 bb = make_short4(0, 0, 0, 0);
    if (r < n) {
        const uint32_t c = __ldg(touched + r);   // both loads in flight together
        const short4 b = __ldg(bboxes + r);
        if (c != 0) bb = b;
    }
    return bb;
}

// One CTA (1024 threads): per tile, exclusive prefix over the group sums (in
// place) and the tile total, then the exclusive scan of the totals into each
// list's start (and the pair count) — what colscan_groups_kernel plus a
// multi-kernel device scan did, in one launch (grids up to kScanTilesMax tiles).
constexpr int kScanTilesMax = 16384;
// above this many (group, tile) column entries the single-CTA fused scan is the bottleneck
// (C4: 46 groups x 5100 tiles took 29 us in one CTA)
constexpr int64_t kFusedScanWork = 65536;
__global__ void __launch_bounds__(1024) colscan_groups_scan_kernel(int ntiles, int ngroups, uint32_t* __restrict__ part,
                                                                   uint32_t* __restrict__ tile_count,
                                                                   uint32_t* __restrict__ tile_start,
                                                                   uint32_t* __restrict__ counters) {
    extern __shared__ uint32_t s_cnt[];
    __shared__ uint32_t wsum[33];
    if (threadIdx.x == 0) counters[5] = 0;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
        uint32_t run = 0;
        for (int g0 = 0; g0 < ngroups; g0 += 16) {   // 16 loads in flight, then the prefix
            uint32_t v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = g0 + i < ngroups ? part[(size_t)(g0 + i) * ntiles + t] : 0u;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (g0 + i < ngroups) part[(size_t)(g0 + i) * ntiles + t] = run;
                run += v[i];
            }
        }
        tile_count[t] = run;
        s_cnt[t] = run;
    }
    __syncthreads();
    const uint32_t total = block_exclusive_scan(s_cnt, ntiles, wsum);
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) tile_start[t] = s_cnt[t];
    if (threadIdx.x == 0) counters[0] = total;
}

// One CTA: exclusive scan of the tile totals into each list's start and the pair count
// (the second half of colscan_groups_scan_kernel, after a multi-CTA colscan_groups_kernel).
__global__ void __launch_bounds__(1024) tile_scan_kernel(int ntiles, const uint32_t* __restrict__ tile_count,
                                                         uint32_t* __restrict__ tile_start,
                                                         uint32_t* __restrict__ counters) {
    extern __shared__ uint32_t s_cnt[];
    __shared__ uint32_t wsum[33];
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_cnt[t] = tile_count[t];
    __syncthreads();
    const uint32_t total = block_exclusive_scan(s_cnt, ntiles, wsum);
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) tile_start[t] = s_cnt[t];
    if (threadIdx.x == 0) counters[0] = total;
}

template <int RPT>
__global__ void __launch_bounds__(kBinThreads, 2) fill_rows_kernel(
    int64_t n, const short4* __restrict__ bboxes, const uint32_t* __restrict__ touched, int ntx, int ntiles,
    const uint32_t* __restrict__ hist, const uint32_t* __restrict__ pre, const uint32_t* __restrict__ part,
    const uint32_t* __restrict__ tile_start,
    const uint32_t* __restrict__ tile_count, uint32_t* __restrict__ ranges, int64_t cap,
    uint32_t* __restrict__ ranks, uint32_t* __restrict__ keys, uint32_t* __restrict__ counters,
    const uint32_t* __restrict__ offsets, uint32_t* __restrict__ slot_pos, uint8_t* __restrict__ rmask) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ uint32_t wsum[33];
    __shared__ int pass_end;
    uint32_t* loff = smem;                 // per tile: count -> local start -> cursor
    uint32_t* gbase = smem + ntiles;       // per tile: global slot of this block's run, minus its local start
    uint32_t* stage = gbase + ntiles;      // staged ranks of the current pass
    uint16_t* stile = (uint16_t*)(stage + kBinStage);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x)
        write_range(t, tile_start, tile_count, ranges, cap);
    constexpr int64_t kBlk = (int64_t)RPT * kBinThreads;
    const int64_t nblk = (n + kBlk - 1) / kBlk;
    const float inv_ntx = 1.0f / (float)ntx;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        short4 bb[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j)
            bb[j] = bin_box(n, blk * kBlk + j * kBinThreads + threadIdx.x, bboxes, touched);
        // this block's tile histogram is count_rows' row (no second counting pass)
        const uint32_t* crow = hist + (size_t)blk * ntiles;
        for (int t = threadIdx.x; t < ntiles; t += blockDim.x) loff[t] = crow[t];
        __syncthreads();
        const uint32_t* hrow = pre + (size_t)blk * ntiles;
        const uint32_t* prow = part + (size_t)(blk / kColGroup) * ntiles;
        const uint32_t total = block_exclusive_scan(loff, ntiles, wsum);
        for (int t = threadIdx.x; t < ntiles; t += blockDim.x) gbase[t] = tile_start[t] + prow[t] + hrow[t] - loff[t];
        // passes over tile ranges whose pairs fit the stage (one pass unless the block is dense)
        int t0 = 0;
        while (t0 < ntiles) {
            if (total <= kBinStage) {
                if (threadIdx.x == 0) pass_end = ntiles;
            } else if (threadIdx.x == 0) {
                // largest t1 whose tiles [t0, t1) hold <= kBinStage pairs; a single
                // tile holds <= kBlk pairs of a block, so t1 > t0
                int lo = t0 + 1, hi = ntiles;
                const uint32_t lim = loff[t0] + kBinStage;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    const uint32_t e = mid < ntiles ? loff[mid] : total;
                    if (e <= lim) lo = mid;
                    else hi = mid - 1;
                }
                pass_end = lo;
            }
            __syncthreads();
            const int t1 = pass_end;
            const uint32_t s0 = loff[t0];
            const uint32_t s1 = t1 < ntiles ? loff[t1] : total;
            __syncthreads();   // everyone has read loff[t0], loff[t1] before the cursors move
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const uint32_t r = (uint32_t)(blk * kBlk + j * kBinThreads + threadIdx.x);
                for (int ty = bb[j].z >> 4; ty <= (bb[j].w - 1) >> 4; ++ty) {
                    const int row = ty * ntx;
                    for (int tx = bb[j].x >> 4; tx <= (bb[j].y - 1) >> 4; ++tx) {
                        const int t = row + tx;
                        if (t < t0 || t >= t1) continue;
                        const uint32_t idx = atomicAdd(&loff[t], 1u) - s0;
                        SPLAT_DCHECK(idx < (uint32_t)kBinStage);
                        stage[idx] = r;
                        stile[idx] = (uint16_t)t;
                    }
                }
            }
            __syncthreads();
            // each (block, tile) run [a, e) is a handful of entries: an entry's place in
            // its run is the number of smaller ranks in it (ranks are distinct)
            const int m = (int)(s1 - s0);
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const int t = stile[i];
                const uint32_t v = stage[i];
                const int a = t == t0 ? 0 : (int)(loff[t - 1] - s0);
                const int e = (int)(loff[t] - s0);
                uint32_t below = 0;
                SPLAT_DCHECK(a <= i && i < e && e <= m);
                for (int j = a; j < e; ++j) below += stage[j] < v;
                const uint32_t pos = gbase[t] + s0 + (uint32_t)a + below;
                put_rank(pos, v, cap, ranks, counters);
                if ((int64_t)pos < cap) {
                    if (keys) keys[pos] = (uint32_t)t;
                    const short4 b = bboxes[v];   // the block's boxes: L1 / L2 hits
                    // t / ntx without an integer division: (t + 0.5) / ntx is >= 0.5 / ntx away
                    // from an integer, far beyond the float32 error for t < 2^16
                    const int ty = __float2int_rd(((float)t + 0.5f) * inv_ntx), tx = t - ty * ntx;
                    rmask[pos] = (uint8_t)rect_mask(b, tx, ty);
                    if (slot_pos) {   // training: emission slot -> list position (see slot_map_kernel)
                        const int tx0 = b.x >> 4, ty0 = b.z >> 4, nx = ((b.y - 1) >> 4) - tx0 + 1;
                        const int64_t e = (int64_t)offsets[v] + (ty - ty0) * nx + (tx - tx0);
                        if (e < cap) slot_pos[e] = pos;
                    }
                }
            }
            __syncthreads();
            t0 = t1;
        }
    }
}

// Large-grid path: the per-pair rectangle masks once the lists are sorted.
__global__ void rect_mask_kernel(int ntx, const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ ranks,
                                 const short4* __restrict__ bboxes, uint8_t* __restrict__ rmask) {
    const int t = blockIdx.x;
    const uint32_t st = ranges[2 * t], en = ranges[2 * t + 1];
    for (uint32_t j = st + threadIdx.x; j < en; j += blockDim.x)
        rmask[j] = (uint8_t)rect_mask(bboxes[ranks[j]], t % ntx, t / ntx);
}

// Training mode: list position of every pair, indexed by its emission slot
// offsets[r] + (tile index inside r's tile rectangle) — the backward writes
// per-pair partials at list positions and reduces them per rank through this map.
__global__ void slot_map_kernel(int ntx, const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ ranks,
                                const short4* __restrict__ bboxes, const uint32_t* __restrict__ offsets,
                                int64_t cap, uint32_t* __restrict__ slot_pos) {
    const int t = blockIdx.x;
    const int tx = t % ntx, ty = t / ntx;
    const uint32_t st = ranges[2 * t], en = ranges[2 * t + 1];
    for (uint32_t j = st + threadIdx.x; j < en; j += blockDim.x) {
        const uint32_t r = ranks[j];
        const short4 bb = bboxes[r];
        const int tx0 = bb.x >> 4, ty0 = bb.z >> 4, nx = ((bb.y - 1) >> 4) - tx0 + 1;
        const int64_t e = (int64_t)offsets[r] + (ty - ty0) * nx + (tx - tx0);
        if (e < cap) slot_pos[e] = j;
    }
}

// Fallback for tile grids too large for the shared-memory tables: global atomics.
__global__ void count_tiles_kernel(int64_t n, const short4* __restrict__ bboxes,
                                   const uint32_t* __restrict__ touched, int ntx,
                                   uint32_t* __restrict__ tile_count) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n || touched[r] == 0) return;
    int tx0, tx1, ty0, ty1;
    tile_rect(bboxes[r], tx0, tx1, ty0, ty1);
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(&tile_count[ty * ntx + tx], 1u);
}

__global__ void init_ranges_kernel(int ntiles, const uint32_t* __restrict__ tile_start,
                                   const uint32_t* __restrict__ tile_count, uint32_t* __restrict__ ranges,
                                   uint32_t* __restrict__ cursor, int64_t cap, uint32_t* __restrict__ counters) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) counters[5] = 0;
    if (t >= ntiles) return;
    write_range(t, tile_start, tile_count, ranges, cap);
    cursor[t] = tile_start[t];
}

__global__ void fill_tiles_kernel(int64_t n, const short4* __restrict__ bboxes,
                                  const uint32_t* __restrict__ touched, int ntx, int64_t cap,
                                  uint32_t* __restrict__ cursor, uint32_t* __restrict__ ranks,
                                  uint32_t* __restrict__ counters) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n || touched[r] == 0) return;
    int tx0, tx1, ty0, ty1;
    tile_rect(bboxes[r], tx0, tx1, ty0, ty1);
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx)
            put_rank(atomicAdd(&cursor[ty * ntx + tx], 1u), (uint32_t)r, cap, ranks, counters);
}

constexpr int kSegThreads = 256;
constexpr int kSegSmall = 8192;      // per-tile lists up to this length: 32 KB smem bitonic, one CTA per tile
constexpr int kSegThreadsLarge = 1024;
constexpr int kSegChunk = 32768;     // longer lists: 128 KB chunks sorted in smem, then merged in HBM

__device__ void bitonic_sort_smem(uint32_t* a, int P) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t x = a[i], y = a[ixj];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        a[i] = y;
                        a[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Sort src[0, L) (L <= P_max) through shared memory into dst (may alias src).
__device__ void sort_run_smem(const uint32_t* src, uint32_t* dst, int L, uint32_t* seg) {
    int P = 1;
    while (P < L) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) seg[i] = i < L ? src[i] : 0xffffffffu;
    __syncthreads();
    bitonic_sort_smem(seg, P);
    for (int i = threadIdx.x; i < L; i += blockDim.x) dst[i] = seg[i];
    __syncthreads();
}

__device__ __forceinline__ int lower_bound_u32(const uint32_t* a, int n, uint32_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One CTA per tile.  Lists longer than kSegSmall are queued for the large kernel.
__global__ void __launch_bounds__(kSegThreads) segsort_kernel(int ntiles, const uint32_t* __restrict__ ranges,
                                                              uint32_t* __restrict__ ranks,
                                                              uint32_t* __restrict__ keys,
                                                              uint32_t* __restrict__ big_list,
                                                              uint32_t* __restrict__ counters) {
    extern __shared__ __align__(16) uint32_t seg[];
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint32_t st = ranges[2 * t], en = ranges[2 * t + 1];
        const int L = (int)(en - st);
        if (L == 0) continue;
        if (L > kSegSmall) {
            if (threadIdx.x == 0) big_list[atomicAdd(&counters[5], 1u)] = (uint32_t)t;
            continue;
        }
        sort_run_smem(ranks + st, ranks + st, L, seg);
        if (keys)
            for (int i = threadIdx.x; i < L; i += blockDim.x) keys[st + i] = (uint32_t)t;
    }
}

// Long lists (rare: a tile covered by > kSegSmall splats): one CTA per tile sorts
// kSegChunk runs in shared memory, then merges runs pairwise in HBM (ranks are
// unique inside a list, so each element's merged position is its index in its own
// run plus a lower_bound in the partner run), ping-ponging through `alt`.
__global__ void __launch_bounds__(kSegThreadsLarge) segsort_large_kernel(const uint32_t* __restrict__ ranges,
                                                                         uint32_t* __restrict__ ranks,
                                                                         uint32_t* __restrict__ alt,
                                                                         uint32_t* __restrict__ keys,
                                                                         const uint32_t* __restrict__ big_list,
                                                                         const uint32_t* __restrict__ counters) {
    extern __shared__ __align__(16) uint32_t seg[];
    const int nbig = (int)counters[5];
    for (int w = blockIdx.x; w < nbig; w += gridDim.x) {
        const int t = (int)big_list[w];
        const uint32_t st = ranges[2 * t];
        const int L = (int)(ranges[2 * t + 1] - st);
        uint32_t* a = ranks + st;
        uint32_t* b = alt + st;
        for (int c = 0; c < L; c += kSegChunk) sort_run_smem(a + c, a + c, min(kSegChunk, L - c), seg);
        for (int run = kSegChunk; run < L; run <<= 1) {
            for (int i = threadIdx.x; i < L; i += blockDim.x) {
                const int k = i / run;
                const int base = (k & ~1) * run;
                const int pb = (k ^ 1) * run;
                int pos = i;
                if (pb < L) {
                    const int pn = min(run, L - pb);
                    pos = base + (i - k * run) + lower_bound_u32(a + pb, pn, a[i]);
                }
                b[pos] = a[i];
            }
            __syncthreads();
            uint32_t* tmp = a;
            a = b;
            b = tmp;
        }
        if (a != ranks + st)
            for (int i = threadIdx.x; i < L; i += blockDim.x) ranks[st + i] = a[i];
        if (keys)
            for (int i = threadIdx.x; i < L; i += blockDim.x) keys[st + i] = (uint32_t)t;
        __syncthreads();
    }
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
    L.vals0 = o; o = align_up(o + (cc + kPairPad) * 4);
    L.vals1 = o; o = align_up(o + cc * 4);   // merge buffer for very long tile lists
    L.slot_pos = o; o = align_up(o + cc * 4);   // training: list position of each emission slot
    L.tile_scan = o; o = align_up(o + (size_t)scan_scratch_words((int64_t)L.ntx * L.nty) * 4);
    L.ranges = o; o = align_up(o + (size_t)L.ntx * L.nty * 8);
    L.tile_count = o; o = align_up(o + (size_t)L.ntx * L.nty * 4 + 4);
    L.tile_start = o; o = align_up(o + (size_t)L.ntx * L.nty * 4 + 4);
    L.cursor = o; o = align_up(o + (size_t)L.ntx * L.nty * 4);
    {
        const size_t blk = (size_t)bin_rpt(L.ntx * L.nty, n) * kBinThreads;
        const size_t rows = (size_t)(nn + blk - 1) / blk;
        const size_t groups = (rows + kColGroup - 1) / kColGroup;
        L.bin_hist = o; o = align_up(o + rows * L.ntx * L.nty * 4);
        L.bin_pre = o; o = align_up(o + rows * L.ntx * L.nty * 4);
        L.bin_part = o; o = align_up(o + groups * L.ntx * L.nty * 4);
    }
    L.big_list = o; o = align_up(o + (size_t)L.ntx * L.nty * 4);
    L.counters = o; o = align_up(o + 32 * 4);   // [16..] only in RASTER_STATS builds
    L.fixup = o; o = align_up(o + (size_t)width * height * 4 + 4);
    L.pack = o; o = align_up(o + nn * sizeof(PackF));
    L.rmask = o; o = align_up(o + cc + kPairPad);   // per pair: rect_mask of its tile (u8)
    L.bwd_hi = o; o = align_up(o + (size_t)L.ntx * L.nty * 8 * 4);   // backward: replay start per rectangle
    L.bwd_cursor = o; o = align_up(o + 16);                          // backward: work-unit counter
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
#ifdef TIMING_SKIP_PRE   // timing-only builds (tools/marginal.sh): measure a stage's marginal cost
    if (L.n > 0) return SPLAT_OK;
#endif
    uint32_t* counters = (uint32_t*)(ws + L.counters);
    SPLAT_CUDA_CHECK(cudaMemsetAsync(counters, 0, 4 * 4, stream));  // [4..] are sticky
    if (sc.n == 0) return SPLAT_OK;
    int blocks = (int)((sc.n + PRE_THREADS - 1) / PRE_THREADS);
    preprocess_kernel<<<blocks, PRE_THREADS, 0, stream>>>(sc, vc, L.width, L.height,
                                                  (PackF*)(ws + L.pack), (short4*)(ws + L.bboxes),
                                                  (uint32_t*)(ws + L.touched)); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int launch_binning(const FrameLayout& L, char* ws, int flags, cudaStream_t stream) {
#ifdef TIMING_SKIP_BIN   // bin each workspace once, then reuse its lists (tools/same_view_probe.py)
    {
        static std::set<const char*> binned;
        if (L.n > 0 && !(flags & (SPLAT_BIN_KEYS | SPLAT_BIN_OFFSETS)) && !binned.insert(ws).second) return SPLAT_OK;
    }
#endif
    const bool with_offsets = flags & SPLAT_BIN_OFFSETS;
    uint32_t* counters = (uint32_t*)(ws + L.counters);
    uint32_t* ranges = (uint32_t*)(ws + L.ranges);
    const int ntiles = L.ntx * L.nty;
    uint32_t* tile_count = (uint32_t*)(ws + L.tile_count);
    uint32_t* tile_start = (uint32_t*)(ws + L.tile_start);
    if (L.n == 0) {
        SPLAT_CUDA_CHECK(cudaMemsetAsync(ranges, 0, (size_t)ntiles * 8, stream));
        return SPLAT_OK;
    }
    const uint32_t* touched = (const uint32_t*)(ws + L.touched);
    const short4* bboxes = (const short4*)(ws + L.bboxes);
    if (with_offsets)   // rank-major pair slots for the backward's partials
        exclusive_scan_u32(touched, (uint32_t*)(ws + L.offsets), L.n, (uint32_t*)(ws + L.scan_scratch), nullptr,
                           stream);
    uint32_t* ranks = (uint32_t*)(ws + L.vals0);
    uint32_t* keys = (flags & SPLAT_BIN_KEYS) ? (uint32_t*)(ws + L.keys0) : nullptr;
    uint32_t* scan_tmp = (uint32_t*)(ws + L.tile_scan);
    const int rpt = bin_rpt(ntiles, L.n);
    const int64_t bin_blk = (int64_t)rpt * kBinThreads;
    const int64_t nrows = (L.n + bin_blk - 1) / bin_blk;
    const int ngroups = (int)((nrows + kColGroup - 1) / kColGroup);
    const int fill_smem = 8 * ntiles + 6 * kBinStage;
    const bool staged = ntiles <= 65535 && fill_smem <= kBinSmemMax && L.cap < 0xffffffffLL &&
                        !(flags & SPLAT_BIN_ATOMIC);
    if (staged) {
        static PerDevice<bool> configured;
        bool ok = false;
        const int rc = configured.get(ok, [](bool& v) {
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(count_rows_kernel<kBinRPT>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kBinSmemMax));
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(fill_rows_kernel<kBinRPT>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kBinSmemMax));
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(count_rows_kernel<kBinRPT / 2>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kBinSmemMax));
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(fill_rows_kernel<kBinRPT / 2>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kBinSmemMax));
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(count_rows_kernel<kBinRPT / 4>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kBinSmemMax));
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(fill_rows_kernel<kBinRPT / 4>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kBinSmemMax));
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(colscan_groups_scan_kernel,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kScanTilesMax * 4));
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(tile_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  kScanTilesMax * 4));
            v = true;
            return SPLAT_OK;
        });
        if (rc != SPLAT_OK) return rc;
        uint32_t* hist = (uint32_t*)(ws + L.bin_hist);
        uint32_t* pre = (uint32_t*)(ws + L.bin_pre);
        uint32_t* part = (uint32_t*)(ws + L.bin_part);
        const int grid = (int)(nrows < 148 * 2 ? nrows : 148 * 2);
        auto count = rpt == kBinRPT       ? count_rows_kernel<kBinRPT>
                     : rpt == kBinRPT / 2 ? count_rows_kernel<kBinRPT / 2>
                                          : count_rows_kernel<kBinRPT / 4>;
        count<<<grid, kBinThreads, ntiles * 4, stream>>>(L.n, bboxes, touched, L.ntx, ntiles, hist);
        note_launch();
        colscan_rows_kernel<<<dim3(ceil_div(ntiles, 128), ngroups), 128, 0, stream>>>(ntiles, (int)nrows, hist,
                                                                                     pre, part);
        note_launch();
        if (ntiles <= kScanTilesMax && (int64_t)ngroups * ntiles <= kFusedScanWork) {
            colscan_groups_scan_kernel<<<1, 1024, ntiles * 4, stream>>>(ntiles, ngroups, part, tile_count,
                                                                        tile_start, counters);
            note_launch();
        } else if (ntiles <= kScanTilesMax) {   // many groups x tiles: the column prefixes over many CTAs
            colscan_groups_kernel<<<ceil_div(ntiles, 128), 128, 0, stream>>>(ntiles, ngroups, part, tile_count,
                                                                            counters);
            note_launch();
            tile_scan_kernel<<<1, 1024, ntiles * 4, stream>>>(ntiles, tile_count, tile_start, counters);
            note_launch();
        } else {
            colscan_groups_kernel<<<ceil_div(ntiles, 128), 128, 0, stream>>>(ntiles, ngroups, part, tile_count,
                                                                            counters);
            note_launch();
            exclusive_scan_u32(tile_count, tile_start, ntiles, scan_tmp, &counters[0], stream);
        }
        if (flags & SPLAT_BIN_COUNT_ONLY) {   // counters[0] holds the pair count
            SPLAT_CUDA_CHECK(cudaGetLastError());
            return SPLAT_OK;
        }
        auto fill = rpt == kBinRPT       ? fill_rows_kernel<kBinRPT>
                    : rpt == kBinRPT / 2 ? fill_rows_kernel<kBinRPT / 2>
                                         : fill_rows_kernel<kBinRPT / 4>;
        fill<<<grid, kBinThreads, fill_smem, stream>>>(L.n, bboxes, touched, L.ntx, ntiles, hist, pre, part,
                                                                  tile_start, tile_count, ranges, L.cap, ranks,
                                                                  keys, counters, (const uint32_t*)(ws + L.offsets),
                                                                  with_offsets ? (uint32_t*)(ws + L.slot_pos) : nullptr,
                                                                  (uint8_t*)(ws + L.rmask));
        note_launch();
        SPLAT_CUDA_CHECK(cudaGetLastError());
        return SPLAT_OK;
    } else {
        const int blocks = (int)((L.n + 255) / 256);
        SPLAT_CUDA_CHECK(cudaMemsetAsync(tile_count, 0, (size_t)ntiles * 4, stream));
        count_tiles_kernel<<<blocks, 256, 0, stream>>>(L.n, bboxes, touched, L.ntx, tile_count); note_launch();
        exclusive_scan_u32(tile_count, tile_start, ntiles, scan_tmp, &counters[0], stream);
        if (flags & SPLAT_BIN_COUNT_ONLY) {
            SPLAT_CUDA_CHECK(cudaGetLastError());
            return SPLAT_OK;
        }
        uint32_t* cursor = (uint32_t*)(ws + L.cursor);
        init_ranges_kernel<<<ceil_div(ntiles, 256), 256, 0, stream>>>(ntiles, tile_start, tile_count, ranges,
                                                                      cursor, L.cap, counters); note_launch();
        fill_tiles_kernel<<<blocks, 256, 0, stream>>>(L.n, bboxes, touched, L.ntx, L.cap, cursor, ranks, counters);
        note_launch();
    }
    static PerDevice<bool> configured;
    bool ok = false;
    const int rc = configured.get(ok, [](bool& v) {
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(segsort_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              kSegChunk * 4));
        v = true;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    uint32_t* big = (uint32_t*)(ws + L.big_list);
    segsort_kernel<<<ntiles, kSegThreads, kSegSmall * 4, stream>>>(ntiles, ranges, ranks, keys, big, counters);
    note_launch();
    segsort_large_kernel<<<148, kSegThreadsLarge, kSegChunk * 4, stream>>>(ranges, ranks, (uint32_t*)(ws + L.vals1),
                                                                          keys, big, counters);
    note_launch();
    rect_mask_kernel<<<ntiles, 256, 0, stream>>>(L.ntx, ranges, ranks, bboxes, (uint8_t*)(ws + L.rmask));
    note_launch();
    if (with_offsets) {
        slot_map_kernel<<<ntiles, 256, 0, stream>>>(L.ntx, ranges, ranks, bboxes, (const uint32_t*)(ws + L.offsets),
                                                    L.cap, (uint32_t*)(ws + L.slot_pos));
        note_launch();
    }
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int launch_pack64(const SceneConst& sc, const ViewConst& vc, double* out, cudaStream_t stream) {
    if (sc.n == 0) return SPLAT_OK;
    pack64_kernel<<<(int)((sc.n + 255) / 256), 256, 0, stream>>>(sc, vc, out); note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}



}  // namespace splat
