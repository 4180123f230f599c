// Front-to-back gradient rasterizer (forward) for sm_100a.
//
// Semantics: _kernels.forward_region (_kernels.py:32-129) per pixel, on the
// 16x16 tile lists of bin_tiles.  One CTA per tile, 8 warps, each warp owns an
// 8x4 pixel rectangle (one pixel per lane).  Candidates are staged in shared
// memory 256 at a time together with an 8-bit mask of the warp rectangles
// their bbox touches; a warp walks only the candidates whose mask bit is set
// (warp-level bbox rejection) and leaves as soon as all its pixels terminated
// (warp-level early termination).
//
// Precision design: every blending decision of the reference
// — cull (alpha < 1/255), clamp (alpha > 0.999) and early termination
// (1 - A < 1e-4) — is decided in float32 with a rigorous error bound; a
// candidate whose cull/clamp test falls inside the bound is re-evaluated with
// the reference's exact float64 arithmetic, and a pixel whose termination test
// falls inside the bound is re-rendered by `fixup_kernel` with the exact
// float64 blend chain.  The decisions (hence contrib_count and every per-tile
// contributor list) therefore equal the reference's; values are float32.
#include <cmath>

#include <cstring>

#include "footprint.cuh"

namespace splat {

namespace {

struct RasterArgs {
    SceneConst sc;
    ViewConst vc;
    int width, height, ntx;
    const uint32_t* ranges;
    const uint32_t* ranks;
    const uint8_t* rmask;
    const PackF* pack;
    const short4* bboxes;
    float* planes;
    float* alpha;
    int32_t* count;
    uint32_t* last;
    double* state;
    uint32_t* fixup;
    uint32_t* counters;
};

#ifndef RASTER_FFMA2
#define RASTER_FFMA2 1
#endif

// Per-pixel blend state (_kernels.py:41-57 accumulators).  T is the
// transmittance 1 - A; TRAIN keeps the A-state in float64 for the backward
// inversion.
template <bool TRAIN>
struct Blend {
    float b[3], bx[3], by[3], bxy[3];
    float T, ax, ay, axy;          // float32 state (inference)
    double Td, axd, ayd, axyd;     // float64 state (training)
    float err;                     // absolute error bound of T, excluding the per-step product roundings
    int n;
    uint32_t last;

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int c = 0; c < 3; ++c) b[c] = bx[c] = by[c] = bxy[c] = 0.f;
        T = 1.f;
        ax = ay = axy = 0.f;
        Td = 1.0;
        axd = ayd = axyd = 0.0;
        err = 0.f;
        n = 0;
        last = 0;
    }

    // Inference blend from the raw gradient factors (gx, gy, h = gx gy - 2b; zero when
    // clamped): a_x = al gx etc. are folded into the blend terms
    //   tx = al (T gx - A_x),  ty = al (T gy - A_y),  txy = al (T h - A_y gx - A_x gy - A_xy)
    // and the state advances by them (A_x += tx, T -= T al).
    __device__ __forceinline__ void add_raw(float al, float gx, float gy, float h, const float4& col) {
        const float2 al2 = make_float2(al, al);
        const float2 txty = fmul2(al2, ffma2(make_float2(T, T), make_float2(gx, gy), make_float2(-ax, -ay)));
        const float txy = al * fmaf(-ax, gy, fmaf(-ay, gx, fmaf(T, h, -axy)));
        const float ta = T * al;
        const float2 tab2 = make_float2(ta, txy);
        const float cc[3] = {col.x, col.y, col.z};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float2 c2 = make_float2(cc[c], cc[c]);
            const float2 p = ffma2(c2, txty, make_float2(bx[c], by[c]));
            const float2 q = ffma2(c2, tab2, make_float2(b[c], bxy[c]));
            bx[c] = p.x;
            by[c] = p.y;
            b[c] = q.x;
            bxy[c] = q.y;
        }
        const float2 n2 = fadd2(make_float2(ax, ay), txty);
        ax = n2.x;
        ay = n2.y;
        axy += txy;
        T -= ta;
        ++n;
    }

    // One contributor (_kernels.py:88-109).  om = 1 - alpha (exactly 1e-3 when clamped).
    __device__ __forceinline__ void add(float al, float gax, float gay, float gaxy, float om,
                                        const float4& col) {
        float t, sx, sy, sxy;
        if (TRAIN) {
            t = (float)Td;
            sx = (float)axd;
            sy = (float)ayd;
            sxy = (float)axyd;
        } else {
            t = T;
            sx = ax;
            sy = ay;
            sxy = axy;
        }
#if RASTER_FFMA2
        const float2 tg = fmul2(make_float2(t, t), make_float2(gax, gay));        // (t gax, t gay)
        const float2 txty = fsub2(tg, fmul2(make_float2(sx, sy), make_float2(al, al)));
        const float tx_ = txty.x, ty_ = txty.y;
#else
        float tx_ = t * gax - sx * al;
        float ty_ = t * gay - sy * al;
#endif
        float txy = ((t * gaxy - sy * gax) - sxy * al) - sx * gay;
        float ta = t * al;
        float cc[3] = {col.x, col.y, col.z};
#if RASTER_FFMA2
        // (bx, by) and (b, bxy) per channel as packed pairs: 6 FFMA2 instead of 12 FFMA
        const float2 txy2 = make_float2(tx_, ty_), tab2 = make_float2(ta, txy);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float2 c2 = make_float2(cc[c], cc[c]);
            const float2 p = ffma2(c2, txy2, make_float2(bx[c], by[c]));
            const float2 q = ffma2(c2, tab2, make_float2(b[c], bxy[c]));
            bx[c] = p.x;
            by[c] = p.y;
            b[c] = q.x;
            bxy[c] = q.y;
        }
#else
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            bx[c] = fmaf(cc[c], tx_, bx[c]);
            by[c] = fmaf(cc[c], ty_, by[c]);
            bxy[c] = fmaf(cc[c], txy, bxy[c]);
            b[c] = fmaf(cc[c], ta, b[c]);
        }
#endif
        if (TRAIN) {
            double a = al, gx = gax, gy = gay, gxy = gaxy, o = om;
            double nx = fma(axd, o, Td * gx);
            double ny = fma(ayd, o, Td * gy);
            double nxy = fma(axyd, o, Td * gxy) - axd * gy - ayd * gx;
            (void)a;
            axd = nx;
            ayd = ny;
            axyd = nxy;
            Td = Td * o;
            T = (float)Td;
        } else {
            // the state advances by this contributor's blend terms:
            //   A_x' = A_x om + t a_x = A_x + tx, likewise y and xy, and T' = T - t al
            // (T - ta rounds ta once more: <= 2^-24 ta, carried by eval_fast's `rel`)
#if RASTER_FFMA2
            const float2 nxy2 = fadd2(make_float2(ax, ay), make_float2(tx_, ty_));
            ax = nxy2.x;
            ay = nxy2.y;
#else
            ax += tx_;
            ay += ty_;
#endif
            axy += txy;
            T -= ta;
            (void)om;
        }
        ++n;
    }
};

template <bool TRAIN>
__device__ __forceinline__ void write_pixel(const RasterArgs& p, int px, int py, const Blend<TRAIN>& s) {
    int64_t o = (int64_t)py * p.width + px;
    float bgc[3] = {p.vc.bg[0], p.vc.bg[1], p.vc.bg[2]};
    float T = s.T, sx, sy, sxy;
    if (TRAIN) {
        sx = (float)s.axd;
        sy = (float)s.ayd;
        sxy = (float)s.axyd;
    } else {
        sx = s.ax;
        sy = s.ay;
        sxy = s.axy;
    }
    float v[12];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        v[c] = fmaf(T, bgc[c], s.b[c]);          // _kernels.py:112-115
        v[3 + c] = s.bx[c] - sx * bgc[c];        // _kernels.py:116-118
        v[6 + c] = s.by[c] - sy * bgc[c];
        v[9 + c] = s.bxy[c] - sxy * bgc[c];
    }
    float4* dst = reinterpret_cast<float4*>(p.planes + 12 * o);
    dst[0] = make_float4(v[0], v[1], v[2], v[3]);
    dst[1] = make_float4(v[4], v[5], v[6], v[7]);
    dst[2] = make_float4(v[8], v[9], v[10], v[11]);
    int64_t P = (int64_t)p.width * p.height;
    p.alpha[o] = TRAIN ? (float)(1.0 - s.Td) : 1.f - T;
    p.alpha[P + o] = sx;
    p.alpha[2 * P + o] = sy;
    p.alpha[3 * P + o] = sxy;
    p.count[o] = s.n;
    if (TRAIN) p.last[o] = s.last;
    if (TRAIN) {
        double2* st = reinterpret_cast<double2*>(p.state + 4 * o);
        st[0] = make_double2(s.Td, s.axd);
        st[1] = make_double2(s.ayd, s.axyd);
    }
}

constexpr float kTermF = 1e-4f;
#ifndef RASTER_THREADS
#define RASTER_THREADS 128
#endif
constexpr int kRasterThreads = RASTER_THREADS;
constexpr int kWarps = kRasterThreads / 32;   // warps per CTA of the persistent raster
constexpr int kRects = 8;                     // 8x4 rectangles per 16x16 tile

// One candidate at one pixel: the certified decision (kCulled / kContrib /
// kClamped) and the canonical float32 values.  `rp` points at the candidate's
// rank (read only on the rare exact path).
template <bool TRAIN>
__device__ __forceinline__ int decide_candidate(const RasterArgs& p, const PackF& g, const uint32_t* rp,
                                                float cx, float cy, float& al, float& gax, float& gay,
                                                float& gaxy, float& rel) {
    // inference: raw gradient factors (see Blend::add_raw); training: al-scaled
    int st = eval_fast<!TRAIN>(g, cx, cy, al, gax, gay, gaxy, rel);
    if (st == kUnsure) {
        double a64;
        // (int)cx == px: the centres are px + 0.5, exact in float32
        st = eval_exact(p.sc, p.vc, p.bboxes, *rp, (int)cx, (int)cy, &a64);
        if (st != kCulled) canonical_values<!TRAIN>(g, cx, cy, st, al, gax, gay, gaxy);
        if (st == kClamped) rel = 1.6e-5f;   // as eval_fast's clamped branch
    }
    return st;
}

// Blend one contributor (st != kCulled) and run the termination test.
template <bool TRAIN>
__device__ __forceinline__ void apply_candidate(int st, float al, float gax, float gay, float gaxy, float rel,
                                                const float4& col, uint32_t j, Blend<TRAIN>& s, bool& active,
                                                bool& flagged) {
    // training keeps the reference's om = 1e-3 for clamped splats (the backward inverts
    // with it); inference advances T by T al and uses om = 1 - al only in the error
    // recurrence, with the clamped `rel` of eval_fast covering 1 - 0.999f != 1e-3
    float om = 1.f - al;
    if (TRAIN && st == kClamped) om = 1.0e-3f;
    // Absolute error of T: |om - om_exact| <= al rel, so
    // err_k <= om err_{k-1} + T_{k-1} al rel (+ one rounding of the product per
    // step, <= 1.2e-7 T_k including the 1e-3f clamp constant, added at decision
    // time from the step count n).  No division per step.
    if (TRAIN) s.err = fmaf(s.err, om, (s.T * al) * rel);
    else s.err = fmaf(-s.err, al, fmaf(s.T * al, rel, s.err));   // err (1 - al) + ta rel, no om
    if (TRAIN) s.add(al, gax, gay, gaxy, om, col);
    else s.add_raw(al, gax, gay, gaxy, col);
    if (TRAIN) s.last = j + 1;   // contributor-list end: the backward's replay start (training only)
    // err stays far below 1e-6 (flagged pixels stop), so T > 1.02e-4 is never a decision.
    const float T = s.T;
    if (T <= 1.02e-4f) {
        // 1.0625 covers the first-order terms and the float32 rounding of err itself;
        // 2.1e-11 the rounding of 1e-4f and of the compares.
        const float m = fmaf(1.0625f, fmaf((float)s.n, 1.2e-7f * 1.02e-4f, s.err), 2.1e-11f);
        if (T < kTermF - m) {
            active = false;  // certainly terminated (_kernels.py:110-111)
        } else if (T <= kTermF + m) {
            active = false;  // too close to call in float32: exact re-render
            flagged = true;
        }
    }
}

// An undecidable candidate (its float32 footprint test inside the guard band) stops the pixel
// and flags it for the exact float64 re-render of fixup_kernel, which decides every candidate
// of the pixel exactly anyway -- instead of calling the float64 test from the blend loop.
// Inference: ~600 instead of ~230 fix-up pixels per C3 view, but the loop drops from 96
// registers + stack to 70 registers and 7 persistent CTAs per SM (raster 388 -> 346 us);
// training: 96 -> 80 registers at 6 CTAs per SM (C5 raster 227 -> 191 us).
#ifndef RASTER_UNSURE_TO_FIXUP
#define RASTER_UNSURE_TO_FIXUP 1
#endif
#ifndef RASTER_UNSURE_TO_FIXUP_TRAIN
#define RASTER_UNSURE_TO_FIXUP_TRAIN 1
#endif
template <bool TRAIN>
__device__ __forceinline__ void blend_candidate(const RasterArgs& p, const PackF& g, const float4& col,
                                                const uint32_t* rp, uint32_t j, float cx, float cy,
                                                Blend<TRAIN>& s, bool& active, bool& flagged) {
    float al, gax, gay, gaxy, rel;
#if RASTER_UNSURE_TO_FIXUP || RASTER_UNSURE_TO_FIXUP_TRAIN
    if (TRAIN ? RASTER_UNSURE_TO_FIXUP_TRAIN : RASTER_UNSURE_TO_FIXUP) {
        const int st = eval_fast<!TRAIN>(g, cx, cy, al, gax, gay, gaxy, rel);
        if (st == kUnsure) {
            active = false;
            flagged = true;
            return;
        }
        if (st != kCulled) apply_candidate<TRAIN>(st, al, gax, gay, gaxy, rel, col, j, s, active, flagged);
        return;
    }
#endif
    const int st = decide_candidate<TRAIN>(p, g, rp, cx, cy, al, gax, gay, gaxy, rel);
    if (st != kCulled) apply_candidate<TRAIN>(st, al, gax, gay, gaxy, rel, col, j, s, active, flagged);
}

// Each warp streams its tile's candidate list itself (no block barriers), compacted
// to the pairs whose bbox reaches its 8x4 rectangle (see raster_fwd_kernel).  The
// rectangle is split into four 4x2 groups of 8 lanes; per chunk of 32 staged
// candidates each group gets its own in-order list (extent box + Q-norm bound), and
// step k of the blend loop advances every group by one of ITS candidates (four
// candidates per warp instruction stream).
#ifndef RASTER_STATS
#define RASTER_STATS 0   // work counters for tools/raster_stats.py
#endif
#ifndef RASTER_MIN_BLOCKS
// inference: 7 x 128 threads x 70 registers, no spills, since an undecidable candidate hands its
// pixel to the fix-up instead of calling the float64 test in the blend loop (with that call the
// loop needed 96 registers and a stack frame: 5 CTAs per SM)
#define RASTER_MIN_BLOCKS 7
#endif
#ifndef RASTER_MIN_BLOCKS_TRAIN
#define RASTER_MIN_BLOCKS_TRAIN 6   // training (float64 state): 80 registers, no spills, 6 CTAs per SM
#endif
#ifndef RASTER_UNROLL
#define RASTER_UNROLL 3   // inference blend steps per loop iteration (at 7 CTAs/SM: 3 > 2 > 4 > 1)
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Pair batches: the tile list (ranks + per-pair rectangle masks, written by the
// binning) is read 128 pairs at a time with TMA bulk copies (cp.async.bulk ->
// UBLKCP, completion on a per-warp mbarrier), aligned down to 16 pairs.
constexpr int kBatch = 128;
constexpr int kQueue = 256;   // compaction ring: < 32 queued + one batch always fit

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}

template <bool TRAIN>
__global__ void __launch_bounds__(kRasterThreads, TRAIN ? RASTER_MIN_BLOCKS_TRAIN : RASTER_MIN_BLOCKS)
    raster_fwd_kernel(RasterArgs p) {
    // per warp, double-buffered: chunk c+1 is fetched with cp.async (LDGSTS) while chunk c blends
    // 80-byte stride: the four groups' candidates of a step fall on different banks
    struct PackS {
        PackF f;
        float4 col;   // the candidate's colour rides in the fifth 16-byte slot
    };
    __shared__ PackS s_packs[kWarps][2][32];
#define S_PACK(w, b, i) (s_packs[w][b][i].f)
#define S_COL(w, b, i) (s_packs[w][b][i].col)
    __shared__ uint32_t s_rank[kWarps][2][32];
    __shared__ uint32_t s_pos[kWarps][TRAIN ? 2 : 1][32];                 // list positions (training)
    __shared__ __align__(16) uint32_t s_braw[kWarps][2][kBatch];          // batch: ranks
    __shared__ __align__(16) uint32_t s_bmask[kWarps][2][kBatch / 4];     // batch: rect masks (u8 x 4)
    __shared__ uint32_t s_qr[kWarps][kQueue];                             // queue: ranks
    __shared__ uint32_t s_qp[kWarps][TRAIN ? kQueue : 1];                 // queue: list positions
    __shared__ __align__(8) uint64_t s_bbar[kWarps][2];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane >> 3, li = lane & 7;
    const uint32_t nunits = (uint32_t)(p.ntx * ((p.height + kTile - 1) / kTile)) * kRects;
    const uint32_t lt_mask = (1u << lane) - 1u;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_addr(&s_bbar[warp][0])));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_addr(&s_bbar[warp][1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t bphase = 0u;   // parity of the next completion of batch buffer k (bit k)

    // Persistent, per-warp dynamic scheduling: a warp claims (tile, 8x4 rectangle)
    // units from a global counter, so neither slow warps of a CTA nor the last wave
    // leave SM slots idle.  Units are tile-major (neighbouring warps share a tile list
    // in L2 at about the same time).
    for (;;) {
        uint32_t unit = 0;
        if (lane == 0) unit = atomicAdd(&p.counters[3], 1u);
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit >= nunits) break;
        const int tile = (int)(unit / kRects), wr = (int)(unit % kRects);
        const int tile_x = tile % p.ntx, tile_y = tile / p.ntx;
        const int rx0 = tile_x * kTile + (wr & 1) * 8, ry0 = tile_y * kTile + (wr >> 1) * 4;
        const int px = rx0 + (q & 1) * 4 + (li & 3), py = ry0 + (q >> 1) * 2 + (li >> 2);
        const bool inside = px < p.width && py < p.height;
        const float cx = (float)px + 0.5f, cy = (float)py + 0.5f;
        const float X0 = (float)rx0 + 0.5f, Y0 = (float)ry0 + 0.5f;
        const uint32_t start = p.ranges[2 * tile], end = p.ranges[2 * tile + 1];
        SPLAT_DCHECK(start <= end);

        Blend<TRAIN> s;
        s.init();
        s.last = start;
        bool active = inside;
        bool flagged = false;

        if (__any_sync(0xffffffffu, active) && start < end) {
            // The tile list is compacted to the pairs whose bbox reaches this warp's
            // rectangle (binning's rect masks, ~40% of the list at C3) before any
            // candidate is staged: batches of 128 pairs land in shared memory by bulk
            // copy, a ballot scan appends the kept (rank, position) pairs in list order to
            // a per-warp ring, and chunks of 32 kept candidates are staged from the ring.
            const uint32_t b0 = start & ~15u;
            auto issue_batch = [&](uint32_t bstart, int k) {   // lane 0
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(&s_bbar[warp][k])),
                             "r"((uint32_t)(kBatch * 4 + kBatch)) : "memory");
                bulk_g2s(&s_braw[warp][k][0], p.ranks + bstart, kBatch * 4, &s_bbar[warp][k]);
                bulk_g2s(&s_bmask[warp][k][0], p.rmask + bstart, kBatch, &s_bbar[warp][k]);
            };
            if (lane == 0) {
                issue_batch(b0, 0);
                if (b0 + kBatch < end) issue_batch(b0 + kBatch, 1);
            }
            uint32_t bnext = b0;         // first pair of the next batch to scan
            uint32_t qh = 0, qt = 0;     // ring head (next to stage) / tail (next free)
            // scan batches until 32 candidates are queued or the list is exhausted
            auto refill = [&]() {
                while (qt - qh < 32u && bnext < end) {
                    const int k = (int)((bnext - b0) / kBatch) & 1;
                    mbar_wait_parity(&s_bbar[warp][k], (bphase >> k) & 1u);
                    bphase ^= 1u << k;
                    const uint32_t m4 = s_bmask[warp][k][lane];
                    const uint32_t pos0 = bnext + 4u * (uint32_t)lane;
                    uint32_t keep = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t pos = pos0 + (uint32_t)j;
                        if (((m4 >> (8 * j + wr)) & 1u) && pos >= start && pos < end) keep |= 1u << j;
                    }
                    const uint32_t c = __popc(keep);
                    const uint32_t v0 = __ballot_sync(0xffffffffu, c & 1u), v1 = __ballot_sync(0xffffffffu, c & 2u),
                                   v2 = __ballot_sync(0xffffffffu, c & 4u);
                    uint32_t at = qt + __popc(v0 & lt_mask) + 2u * __popc(v1 & lt_mask) + 4u * __popc(v2 & lt_mask);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if ((keep >> j) & 1u) {
                            s_qr[warp][at & (kQueue - 1)] = s_braw[warp][k][4 * lane + j];
                            if (TRAIN) s_qp[warp][at & (kQueue - 1)] = pos0 + (uint32_t)j;
                            ++at;
                        }
                    qt += __popc(v0) + 2u * __popc(v1) + 4u * __popc(v2);
                    SPLAT_DCHECK(qt - qh <= (uint32_t)kQueue && at <= qt);
                    __syncwarp();   // the batch buffer is read: it may be refilled
                    bnext += kBatch;
                    if (lane == 0 && bnext + kBatch < end) issue_batch(bnext + kBatch, k);
                }
                __syncwarp();
            };
            // lane copies queued candidate qh + lane into chunk buffer b; returns the chunk size
            auto stage = [&](int b) -> int {
                const int n = (int)min(32u, qt - qh);
                if (lane < n) {
                    const uint32_t e = (qh + (uint32_t)lane) & (kQueue - 1);
                    const uint32_t r = s_qr[warp][e];
                    SPLAT_DCHECK((int64_t)r < p.sc.n);
                    SPLAT_DCHECK(!TRAIN || (s_qp[warp][TRAIN ? e : 0] >= start && s_qp[warp][TRAIN ? e : 0] < end));
                    const float4* src = reinterpret_cast<const float4*>(p.pack + r);
                    float4* dst = reinterpret_cast<float4*>(&S_PACK(warp, b, lane));
                    cp_async16(dst, src);
                    cp_async16(dst + 1, src + 1);
                    cp_async16(dst + 2, src + 2);
                    cp_async16(dst + 3, src + 3);
                    cp_async16(&S_COL(warp, b, lane), p.sc.color + r);
                    s_rank[warp][b][lane] = r;
                    if (TRAIN) s_pos[warp][TRAIN ? b : 0][lane] = s_qp[warp][TRAIN ? e : 0];
                }
                cp_async_commit();   // one group per chunk (possibly empty)
                qh += (uint32_t)n;
                return n;
            };
            refill();
            int ncur = stage(0);
            int b = 0;
            while (ncur > 0) {
                refill();
                const int nnext = stage(b ^ 1);
                cp_async_wait1();   // chunk b landed (the next one may still be in flight)
                __syncwarp();
                uint32_t gmask = 0;   // bit g: candidate reaches group g's 4x2 rectangle
                if (lane < ncur) {
                    const PackF g = S_PACK(warp, b, lane);
                    // groups: the cull ellipse's extent box against each 4x2 rectangle
                    const float lx = g.mxh - g.ex, hx = g.mxh + g.ex;
                    const float ly = g.myh - g.ey, hy = g.myh + g.ey;
                    const uint32_t c0 = (lx <= X0 + 3.f && hx >= X0) ? 1u : 0u;
                    const uint32_t c1 = (lx <= X0 + 7.f && hx >= X0 + 4.f) ? 1u : 0u;
                    const uint32_t r0 = (ly <= Y0 + 1.f && hy >= Y0) ? 1u : 0u;
                    const uint32_t r1 = (ly <= Y0 + 3.f && hy >= Y0 + 2.f) ? 1u : 0u;
                    gmask = (c0 & r0) | ((c1 & r0) << 1) | ((c0 & r1) << 2) | ((c1 & r1) << 3);
                    if (gmask) gmask &= group_qnorm_mask(g, X0, Y0);
                }
                int cnt_max = 0;
                uint32_t my_mask = 0;   // this lane's group: candidates of the chunk, walked low to high
#if RASTER_STATS
                int cnt_sum = 0;
#endif
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const uint32_t mq = __ballot_sync(0xffffffffu, (gmask >> qq) & 1u);
                    cnt_max = max(cnt_max, __popc(mq));
                    if (qq == q) my_mask = mq;
#if RASTER_STATS
                    cnt_sum += __popc(mq);
#endif
                }
#if RASTER_STATS   // tools/raster_stats.py: chunks, steps, group entries (counters[8..13] as u64)
                if (lane == 0) {
                    atomicAdd((unsigned long long*)&p.counters[8], 1ull);
                    atomicAdd((unsigned long long*)&p.counters[10], (unsigned long long)cnt_max);
                    atomicAdd((unsigned long long*)&p.counters[12], (unsigned long long)cnt_sum);
                }
#endif
                __syncwarp();
                // RASTER_UNROLL steps per iteration in inference (a step with an empty list is a
                // no-op, so the tail needs no guard): less loop-back and termination-vote
                // overhead.  Training keeps one step (its float64 state has no registers to spare).
                constexpr int kU = TRAIN ? 1 : RASTER_UNROLL;
                for (int k = 0; k < cnt_max; k += kU) {
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
#if RASTER_STATS
                        const uint32_t ev = __ballot_sync(0xffffffffu, active && my_mask != 0u);
                        if (lane == 0) atomicAdd((unsigned long long*)&p.counters[14], (unsigned long long)__popc(ev));
                        const int n_before = s.n;
#endif
                        if (active && my_mask != 0u) {
                            const int idx = __ffs(my_mask) - 1;
                            my_mask &= my_mask - 1u;
                            SPLAT_DCHECK(idx < ncur);
                            blend_candidate<TRAIN>(p, S_PACK(warp, b, idx), S_COL(warp, b, idx),
                                                   &s_rank[warp][b][idx], TRAIN ? s_pos[warp][TRAIN ? b : 0][idx] : 0u,
                                                   cx, cy, s, active, flagged);
                        }
#if RASTER_STATS   // steps in which some lane evaluated but none contributed (counters[16..17] as u64)
                        {
                            const uint32_t con = __ballot_sync(0xffffffffu, s.n != n_before);
                            if (lane == 0 && ev != 0u && con == 0u) atomicAdd((unsigned long long*)&p.counters[16], 1ull);
                            if (lane == 0 && ev != 0u) atomicAdd((unsigned long long*)&p.counters[18], (unsigned long long)__popc(con));
                        }
#endif
                    }
                    if (((k + kU) & 7) == 0 && !__any_sync(0xffffffffu, active)) break;
                }
                if (!__any_sync(0xffffffffu, active)) break;
                __syncwarp();
                ncur = nnext;
                b ^= 1;
            }
            cp_async_wait0();
            // batches still in flight must land before their buffers and barriers are reused
            // (the batches in flight are always those at bnext and bnext + kBatch below end)
            for (int i = 0; i < 2 && bnext < end; ++i) {
                const int k = (int)((bnext - b0) / kBatch) & 1;
                mbar_wait_parity(&s_bbar[warp][k], (bphase >> k) & 1u);
                bphase ^= 1u << k;
                bnext += kBatch;
            }
            __syncwarp();
        }
        if (inside) {
            const int ox = (int)cx, oy = (int)cy;   // == px, py (only the float centres stay live)
            write_pixel<TRAIN>(p, ox, oy, s);
            if (flagged) {
                uint32_t slot = atomicAdd(&p.counters[2], 1u);
                p.fixup[slot] = (uint32_t)(oy * p.width + ox);
            }
        }
    }
}

// Exact re-render of flagged pixels: one CTA per pixel.  Per segment of up to
// kFixSeg candidates of the tile list:
//   A. all threads screen their candidates with the certified float32 test
//      (loads of 4 candidates per thread issued back to back);
//   B. the survivors, compacted in list order, get the exact float64
//      reference test (_kernels.py:61-80) spread over the whole CTA;
//   C. warp 0 walks the contributors in list order, running the reference's
//      float64 accumulation `acc = acc + alpha * (1 - acc)` for the
//      termination decision (_kernels.py:105-111) and the same float32 (or
//      TRAIN float64) value recurrences as the main pass.
// Launch shapes.  Inference: one warp at <= 64 registers and a 128-candidate segment
// (6 KB), small enough to co-reside with the next view's persistent raster (7 CTAs per
// SM leave 2816 registers and ~20 KB of shared memory), so the latency-bound fix-up of
// view k overlaps the raster of view k+1 in the multi-stream pipeline without taking a
// raster CTA slot.  Training keeps the wide shape: its float64 blend state would spill
// at 64 registers.
#ifndef FIX_SEG
#define FIX_SEG 2048
#endif
#ifndef FIX_THREADS
#define FIX_THREADS 512
#endif
// Inference shape: one warp per pixel, 128-candidate segments (6 KB of shared memory, 64
// registers), so a fix-up CTA fits beside the 7 persistent raster CTAs of an SM (they leave
// 2816 registers): the 64-thread shape blocked a raster CTA slot per resident fix-up CTA (C3
// 2410 -> 2455 frames/s with this shape and 8 CTAs per SM in the grid).
#ifndef FIX_MINB_INF
#define FIX_MINB_INF 32
#endif
#ifndef FIX_THREADS_INF
#define FIX_THREADS_INF 32
#endif
#ifndef FIX_SEG_INF
#define FIX_SEG_INF 128
#endif
#ifndef FIX_GRID_INF
#define FIX_GRID_INF (148 * 8)
#endif
#ifndef FIX_GRID
#define FIX_GRID (148 * 2)
#endif
template <bool TRAIN>
struct FixShape {
    static constexpr int kSeg = TRAIN ? FIX_SEG : FIX_SEG_INF;
    static constexpr int kThreads = TRAIN ? FIX_THREADS : FIX_THREADS_INF;
    static constexpr int kMinBlocks = TRAIN ? 1 : FIX_MINB_INF;   // 32 x 32 threads: <= 64 registers
    static constexpr int kPer = kSeg / kThreads;
    static_assert(kPer <= 32 && kSeg % kThreads == 0, "candidates per thread fit the keep mask");
};

template <bool TRAIN>
struct FixShared {
    static constexpr int kSeg = FixShape<TRAIN>::kSeg;
    double a64[kSeg];
    float4 val[kSeg];   // al, ax, ay, axy (compacted survivors)
    float4 col[kSeg];
    uint32_t idx[kSeg]; // list index of each survivor
    int8_t st[kSeg];
    uint32_t wcount[FixShape<TRAIN>::kThreads / 32];
    int nsurv;
    int done;
};

template <bool TRAIN>
__global__ void __launch_bounds__(FixShape<TRAIN>::kThreads, FixShape<TRAIN>::kMinBlocks) fixup_kernel(RasterArgs p) {
    constexpr int kFixSeg = FixShape<TRAIN>::kSeg, kFixThreads = FixShape<TRAIN>::kThreads;
    constexpr int kFixPer = FixShape<TRAIN>::kPer;
    extern __shared__ __align__(16) unsigned char fix_raw[];
    FixShared<TRAIN>& S = *reinterpret_cast<FixShared<TRAIN>*>(fix_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t nfix = p.counters[2];
    for (uint32_t w = blockIdx.x; w < nfix; w += gridDim.x) {
        const uint32_t pix = p.fixup[w];
        SPLAT_DCHECK(pix < (uint32_t)(p.width * p.height));
        const int px = (int)(pix % (uint32_t)p.width), py = (int)(pix / (uint32_t)p.width);
        const int tile = (py / kTile) * p.ntx + px / kTile;
        const int wrect = ((py % kTile) / 4) * 2 + (px % kTile) / 8;   // the pixel's 8x4 rectangle
        const uint32_t start = p.ranges[2 * tile], end = p.ranges[2 * tile + 1];
        const float cx = (float)px + 0.5f, cy = (float)py + 0.5f;
        Blend<TRAIN> s;
        s.init();
        s.last = start;
        double acc = 0.0;
        if (tid == 0) S.done = 0;
        for (uint32_t seg = start; seg < end; seg += kFixSeg) {
            const int nseg = (int)min((uint32_t)kFixSeg, end - seg);
            // A: float32 screen; candidate i = tid * kFixPer + u keeps list order per thread
            // (candidates whose bbox misses the pixel's 8x4 rectangle -- binning's rect mask --
            // cannot reach it: their pack is never loaded)
            uint32_t rr[kFixPer], rm = 0;
#pragma unroll
            for (int u = 0; u < kFixPer; ++u) {
                const int i = tid * kFixPer + u;
                rr[u] = i < nseg ? p.ranks[seg + i] : 0u;
                if (i < nseg && ((p.rmask[seg + i] >> wrect) & 1u)) rm |= 1u << u;
            }
            uint32_t keepm = 0;
#pragma unroll
            for (int u = 0; u < kFixPer; ++u) {
                const int i = tid * kFixPer + u;
                if ((rm >> u) & 1u) {
                    const PackF g = p.pack[rr[u]];
                    float al, gax, gay, gaxy, rel;
                    if (eval_fast(g, cx, cy, al, gax, gay, gaxy, rel) != kCulled) keepm |= 1u << u;
                }
            }
            // compact the survivors in list order (block-wide exclusive scan of popcounts)
            const uint32_t cnt = __popc(keepm);
            uint32_t incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            if (lane == 31) S.wcount[wid] = incl;
            __syncthreads();
            uint32_t base = 0, total = 0;
#pragma unroll
            for (int k = 0; k < kFixThreads / 32; ++k) {
                const uint32_t c = S.wcount[k];
                base += k < wid ? c : 0u;
                total += c;
            }
            base += incl - cnt;
#pragma unroll
            for (int u = 0; u < kFixPer; ++u)
                if ((keepm >> u) & 1u) S.idx[base++] = (uint32_t)(tid * kFixPer + u);
            __syncthreads();
            // B: exact float64 test of the survivors, spread over the CTA
            for (uint32_t k = tid; k < total; k += kFixThreads) {
                const uint32_t i = S.idx[k];
                const uint32_t r = p.ranks[seg + i];
                double a64 = 0.0;
                float al = 0.f, gax = 0.f, gay = 0.f, gaxy = 0.f;
                int st = eval_exact_inl(p.sc, p.vc, p.bboxes, r, px, py, &a64);
                if (st != kCulled) {
                    canonical_values(p.pack[r], cx, cy, st, al, gax, gay, gaxy);
                    S.col[k] = p.sc.color[r];
                }
                S.st[k] = (int8_t)st;
                S.a64[k] = a64;
                S.val[k] = make_float4(al, gax, gay, gaxy);
            }
            __syncthreads();
            // C: the reference's ordered accumulation
            if (tid < 32) {
                bool done = false;
                for (uint32_t c0 = 0; c0 < total && !done; c0 += 32) {
                    uint32_t bits = __ballot_sync(0xffffffffu, c0 + lane < total && S.st[c0 + lane] != kCulled);
                    while (bits) {
                        const uint32_t k = c0 + __ffs(bits) - 1;
                        bits &= bits - 1;
                        const float4 v = S.val[k];
                        const float om = S.st[k] == kClamped ? 1.0e-3f : 1.f - v.x;
                        s.add(v.x, v.y, v.z, v.w, om, S.col[k]);
                        s.last = seg + S.idx[k] + 1;
                        const double t = __dsub_rn(1.0, acc);
                        acc = __dadd_rn(acc, __dmul_rn(S.a64[k], t));
                        if (__dsub_rn(1.0, acc) < kEarlyTerm) {
                            done = true;
                            break;
                        }
                    }
                }
                if (lane == 0 && done) S.done = 1;
            }
            __syncthreads();
            if (S.done) break;
        }
        if (tid == 0) write_pixel<TRAIN>(p, px, py, s);
        __syncthreads();
    }
}


static RasterArgs raster_args(const SceneConst& sc, const ViewConst& vc, const FrameLayout& L, char* ws,
                              const splat_gimg_t& out) {
    RasterArgs a;
    a.sc = sc;
    a.vc = vc;
    a.width = L.width;
    a.height = L.height;
    a.ntx = L.ntx;
    a.ranges = (const uint32_t*)(ws + L.ranges);
    a.ranks = (const uint32_t*)(ws + L.vals0);
    a.rmask = (const uint8_t*)(ws + L.rmask);
    a.pack = (const PackF*)(ws + L.pack);
    a.bboxes = (const short4*)(ws + L.bboxes);
    a.planes = out.planes;
    a.alpha = out.alpha;
    a.count = out.count;
    a.last = out.last;
    a.state = out.state;
    a.fixup = (uint32_t*)(ws + L.fixup);
    a.counters = (uint32_t*)(ws + L.counters);
    return a;
}

struct RasterGrids {
    int inf, train;
};

static int raster_grids(RasterGrids& gr) {
    static PerDevice<RasterGrids> grids;
    return grids.get(gr, [](RasterGrids& g) {
        int per_sm = 0, sms = 148;
        const int e = device_sms(sms);
        if (e != SPLAT_OK) return e;
        SPLAT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raster_fwd_kernel<false>, kRasterThreads, 0));
#ifdef RASTER_GRID_PER_SM   // fewer persistent CTAs than fit: room for other streams' kernels beside them
        per_sm = min(per_sm, RASTER_GRID_PER_SM);
#endif
        g.inf = max(per_sm, 1) * sms;
        SPLAT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raster_fwd_kernel<true>, kRasterThreads, 0));
        g.train = max(per_sm, 1) * sms;
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(fixup_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)sizeof(FixShared<false>)));
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(fixup_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)sizeof(FixShared<true>)));
        return SPLAT_OK;
    });
}

}  // namespace

// The exact re-render of the pixels the raster kernel flagged (counters[2] of the frame).
int launch_fixup(const SceneConst& sc, const ViewConst& vc, const FrameLayout& L, char* ws, const splat_gimg_t& out,
                 bool train, cudaStream_t stream) {
    RasterGrids gr{};
    const int rc = raster_grids(gr);
    if (rc != SPLAT_OK) return rc;
    RasterArgs a = raster_args(sc, vc, L, ws, out);
    if (train) {
        fixup_kernel<true><<<FIX_GRID, FixShape<true>::kThreads, sizeof(FixShared<true>), stream>>>(a); note_launch();
    } else {
#ifndef TIMING_SKIP_FIX
        fixup_kernel<false><<<FIX_GRID_INF, FixShape<false>::kThreads, sizeof(FixShared<false>), stream>>>(a);
        note_launch();
#endif
    }
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int launch_raster_forward(const SceneConst& sc, const ViewConst& vc, const FrameLayout& L, char* ws,
                          const splat_gimg_t& out, bool train, cudaStream_t stream, bool with_fixup) {
    RasterGrids gr{};
    const int rc = raster_grids(gr);
    if (rc != SPLAT_OK) return rc;
    RasterArgs a = raster_args(sc, vc, L, ws, out);
    // counters[2] = fix-up pixels, counters[3] = work-unit cursor of the persistent raster
    SPLAT_CUDA_CHECK(cudaMemsetAsync(a.counters + 2, 0, 8, stream));
    if (train) {
        raster_fwd_kernel<true><<<gr.train, kRasterThreads, 0, stream>>>(a); note_launch();
    } else {
        raster_fwd_kernel<false><<<gr.inf, kRasterThreads, 0, stream>>>(a); note_launch();
    }
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return with_fixup ? launch_fixup(sc, vc, L, ws, out, train, stream) : SPLAT_OK;
}

}  // namespace splat
