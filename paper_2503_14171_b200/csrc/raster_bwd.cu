// Reverse-mode rasterizer (sm_100a): _kernels.backward_region
// (_kernels.py:132-365) + the fixed-order reduction and parametrisation chain
// of render_backward (raster_backward.py:87-152).
//
// Per pixel (lane) the contributor list is replayed back to front from the
// forward's `last` index with the same certified decisions and canonical
// float32 footprint values as the forward pass, so the replay is exact.  The
// accumulated-alpha state is inverted in float64 starting from the private
// float64 terminal state the training forward wrote:
//   T_{k-1} = T_k / om_k,  A_{x,k-1} = (A_{x,k} - T_{k-1} a_x) / om_k, ...
// Each 4x2 lane group walks its own candidate list; per candidate the group's
// nine gradient terms are reduce-scattered over its 8 lanes.
//
// Two organisations of the same per-candidate work (BWD_V2 selects; both built,
// tests pass on either):
// * raster_bwd2_kernel (default): persistent warps own (tile, 8x4 rectangle)
//   units, walk only the pairs whose bbox reaches the rectangle (binning's rect
//   masks, TMA-loaded 128-pair windows scanned back to front) and write one
//   partial per (pair, rectangle); reduce_pairs2_kernel sums them per splat.
// * raster_bwd_kernel: one 8-warp CTA per tile; the warps' partials meet in a
//   shared-memory ring after every 32-pair batch, one partial per (tile, splat)
//   pair; reduce_pairs_kernel sums each splat's pairs in tile order.
// No atomics in either: results are bitwise repeatable.
#include <cmath>

#include "footprint.cuh"

namespace splat {

namespace {

constexpr int kBwBatch = 32;
constexpr int kWarps_bw = kBlock / 32;
constexpr int kG = 9;   // d_color(3), d_sigma, d_mean(2), d_conic(3)

struct BwdArgs {
    SceneConst sc;
    ViewConst vc;
    int width, height, ntx;
    const uint32_t* ranges;
    const uint32_t* ranks;
    const PackF* pack;
    const short4* bboxes;
    const uint32_t* offsets;   // pair offset of each rank (emission order)
    const uint32_t* last;
    const int32_t* count;
    const double* state;       // (H,W,4) terminal T, A_x, A_y, A_xy
    const float* adj;          // (H,W,4,3) w, wx, wy, wxy
    float* partial;            // (pairs, 9) per (splat, tile) partial, emission order
};

// Reduce-scatter of the nine terms over the 8 lanes of a 4x2 group (lane bits
// 2, 1, 0): lane li of the group ends with the group sum of term li; g8 gets the
// sum of term 8.  Fixed order, deterministic.
__device__ __forceinline__ float group_reduce9(const float (&g)[kG], int li, float& g8) {
    const bool b2 = li & 4, b1 = li & 2, b0 = li & 1;
    float h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float send = b2 ? g[i] : g[i + 4];
        const float keep = b2 ? g[i + 4] : g[i];
        h[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    float q[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = b1 ? h[i] : h[i + 2];
        const float keep = b1 ? h[i + 2] : h[i];
        q[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    const float send = b0 ? q[0] : q[1];
    const float keep = b0 ? q[1] : q[0];
    const float v = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    float e = g[8];
    e += __shfl_xor_sync(0xffffffffu, e, 4);
    e += __shfl_xor_sync(0xffffffffu, e, 2);
    e += __shfl_xor_sync(0xffffffffu, e, 1);
    g8 = e;
    return v;
}



// Batches of kBwBatch candidates are walked back to front by every warp of the
// tile independently.  Per-batch, per-warp partials go to one of kRing shared
// slots; the last warp to finish a batch sums its slot in fixed warp order and
// writes the (splat, tile) partials, then releases the slot for batch + kRing.
// Warps thus drift up to kRing batches apart instead of meeting at a block
// barrier after every batch (their per-batch work differs with coverage).
constexpr int kRing = 4;

struct BwdShared {
    struct {
        PackF f;
        float4 pad;   // 80-byte stride: the four groups' candidates fall on different banks
    } pack[kWarps_bw][kBwBatch];
    float4 col[kWarps_bw][kBwBatch];
    uint32_t rank[kWarps_bw][kBwBatch];
    float part[kRing][kWarps_bw][kBwBatch][kG];
    float gpart[kWarps_bw][4][kBwBatch][kG];   // per 4x2 group partials of the current batch
    uint8_t list[kWarps_bw][4][kBwBatch];      // per group candidate lists (ascending)
    uint32_t touch[kRing][kWarps_bw];
    int done[kRing];
    int epoch[kRing];
    uint32_t hi[kWarps_bw];
};

__global__ void __launch_bounds__(kBlock, 2) raster_bwd_kernel(BwdArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdShared& S = *reinterpret_cast<BwdShared*>(smem_raw);
    auto& s_pack = S.pack;
    auto& s_col = S.col;
    auto& s_rank = S.rank;

    const int tile = blockIdx.x;
    const int tile_x = tile % p.ntx, tile_y = tile / p.ntx;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rx0 = tile_x * kTile + (warp & 1) * 8, ry0 = tile_y * kTile + (warp >> 1) * 4;
    // four 4x2 lane groups (as in the forward): group q walks its own candidate list
    const int q = lane >> 3, li = lane & 7;
    const int px = rx0 + (q & 1) * 4 + (li & 3), py = ry0 + (q >> 1) * 2 + (li >> 2);
    const bool inside = px < p.width && py < p.height;
    const float cx = (float)px + 0.5f, cy = (float)py + 0.5f;
    const float X0 = (float)rx0 + 0.5f, Y0 = (float)ry0 + 0.5f;
    const uint32_t start = p.ranges[2 * tile], end = p.ranges[2 * tile + 1];

    // per-pixel inputs
    const int64_t o = (int64_t)py * p.width + px;
    uint32_t my_last = start;
    float w[12];
    double T = 1.0, ax = 0.0, ay = 0.0, axy = 0.0;
    bool live = false;
    if (inside) {
        my_last = p.last[o];
        const float4* a4 = reinterpret_cast<const float4*>(p.adj + 12 * o);
        const float4 w0 = a4[0], w1 = a4[1], w2 = a4[2];
        w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
        w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
        w[8] = w2.x; w[9] = w2.y; w[10] = w2.z; w[11] = w2.w;
        bool nz = false;
#pragma unroll
        for (int i = 0; i < 12; ++i) nz |= (w[i] != 0.f);
        live = nz && p.count[o] > 0;   // _kernels.py:155-174
        const double2* st = reinterpret_cast<const double2*>(p.state + 4 * o);
        const double2 s0 = st[0], s1 = st[1];
        T = s0.x;
        ax = s0.y;
        ay = s1.x;
        axy = s1.y;
    } else {
#pragma unroll
        for (int i = 0; i < 12; ++i) w[i] = 0.f;
    }
    // behind-colour state, the background acting as a far splat (_kernels.py:218-229)
    // (channels 0, 1 as packed pairs, channel 2 scalar)
    float2 bh01 = make_float2(p.vc.bg[0], p.vc.bg[1]), bhx01 = make_float2(0.f, 0.f);
    float2 bhy01 = make_float2(0.f, 0.f), bhxy01 = make_float2(0.f, 0.f);
    float bh2 = p.vc.bg[2], bhx2 = 0.f, bhy2 = 0.f, bhxy2 = 0.f;
    const float2 W0p = make_float2(w[0], w[1]), WXp = make_float2(w[3], w[4]);
    const float2 WYp = make_float2(w[6], w[7]), WXYp = make_float2(w[9], w[10]);

    // block-wide highest list end among live pixels
    uint32_t hi = live ? my_last : start;
    hi = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t warp_hi = hi;
    if (lane == 0) S.hi[warp] = hi;
    if (tid < kRing) {
        S.done[tid] = 0;
        S.epoch[tid] = 0;
    }
    __syncthreads();
    hi = start;
#pragma unroll
    for (int k = 0; k < kWarps_bw; ++k) hi = max(hi, S.hi[k]);
    int bi = 0;   // batch index (back to front)
    // pairs no live pixel reaches back to get zero partials: every pair of the
    // tile list is written exactly once (at its list position, so this tile's
    // partials are one contiguous run) and the buffer needs no clearing
    for (uint32_t e = (hi - start) * kG + tid; e < (end - start) * kG; e += kBlock)
        p.partial[(size_t)start * kG + e] = 0.f;

    // the batch's ranks are loaded one batch ahead (one dependent global load less per batch)
    auto batch_lo = [&](uint32_t tp) { return (tp - start > (uint32_t)kBwBatch) ? tp - kBwBatch : start; };
    uint32_t r_cur = 0;
    if (hi > start && batch_lo(hi) + lane < hi) r_cur = p.ranks[batch_lo(hi) + lane];
    for (uint32_t top = hi; top > start; top = batch_lo(top), ++bi) {
        const uint32_t lo = batch_lo(top);
        const int nb = (int)(top - lo);
        const int slot = bi % kRing, round = bi / kRing;
        const uint32_t r = r_cur;
        if (lo > start) {
            const uint32_t lo2 = batch_lo(lo);
            r_cur = lo2 + lane < lo ? p.ranks[lo2 + lane] : 0u;
        }
        // this warp stages the batch and culls it against its own rectangle
        // (skipped when none of its live pixels reaches back this far)
        const bool work = lo < warp_hi;
        bool keep = false;
        SPLAT_DCHECK(nb >= 1 && nb <= kBwBatch);
        if (lane < nb) {
            SPLAT_DCHECK((int64_t)r < p.sc.n);
            s_rank[warp][lane] = r;
            if (work) {
                const PackF g = p.pack[r];
                keep = ellipse_hits_rect(g, X0, X0 + 7.f, Y0, Y0 + 3.f);
                s_pack[warp][lane].f = g;
                s_col[warp][lane] = p.sc.color[r];
            }
        }
        uint32_t gmask = 0;   // bit g: candidate reaches group g's 4x2 rectangle
        if (keep) {
            const PackF& g = s_pack[warp][lane].f;
            const float lx = g.mxh - g.ex, hx = g.mxh + g.ex;
            const float ly = g.myh - g.ey, hy = g.myh + g.ey;
            const uint32_t c0 = (lx <= X0 + 3.f && hx >= X0) ? 1u : 0u;
            const uint32_t c1 = (lx <= X0 + 7.f && hx >= X0 + 4.f) ? 1u : 0u;
            const uint32_t r0 = (ly <= Y0 + 1.f && hy >= Y0) ? 1u : 0u;
            const uint32_t r1 = (ly <= Y0 + 3.f && hy >= Y0 + 2.f) ? 1u : 0u;
            gmask = (c0 & r0) | ((c1 & r0) << 1) | ((c0 & r1) << 2) | ((c1 & r1) << 3);
            if (gmask) gmask &= group_qnorm_mask(g, X0, Y0);
        }
        const uint32_t lt = (1u << lane) - 1u;
        int cnt_my = 0, cnt_max = 0;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            const uint32_t mq = __ballot_sync(0xffffffffu, (gmask >> qq) & 1u);
            if ((gmask >> qq) & 1u) S.list[warp][qq][__popc(mq & lt)] = (uint8_t)lane;
            const int c = __popc(mq);
            cnt_max = max(cnt_max, c);
            if (qq == q) cnt_my = c;
        }
        __syncwarp();
        uint32_t tmask = 0;   // this lane's group: candidates it produced partials for
        for (int k = 0; k < cnt_max; ++k) {   // back to front within each group's list
            const bool has = k < cnt_my;
            const int idx = has ? S.list[warp][q][cnt_my - 1 - k] : 0;
            float gr[kG];
#pragma unroll
            for (int i = 0; i < kG; ++i) gr[i] = 0.f;
            bool contrib = false;
            if (has && live && lo + idx < my_last) {
                const PackF g = s_pack[warp][idx].f;
                float al, gax, gay, gaxy, rel;
                int st = eval_fast(g, cx, cy, al, gax, gay, gaxy, rel);
                if (st == kUnsure) {
                    double a64;
                    st = eval_exact(p.sc, p.vc, p.bboxes, s_rank[warp][idx], px, py, &a64);
                    if (st != kCulled) canonical_values(g, cx, cy, st, al, gax, gay, gaxy);
                }
                if (st != kCulled) {
                    contrib = true;
                    const float4 col = s_col[warp][idx];
                    // invert the accumulated-alpha state across this splat (float64)
                    const double om = st == kClamped ? (double)1.0e-3f : (double)(1.f - al);
                    // 1/om: float32 reciprocal refined by two float64 Newton steps (|rel err| ~ 1e-16)
                    double inv = (double)fast_rcp((float)om);
                    inv = inv * fma(-om, inv, 2.0);
                    inv = inv * fma(-om, inv, 2.0);
                    const double Tp = T * inv;
                    const double axp = (ax - Tp * (double)gax) * inv;
                    const double ayp = (ay - Tp * (double)gay) * inv;
                    const double axyp = (axy - Tp * (double)gaxy + axp * (double)gay + ayp * (double)gax) * inv;
                    const float t = (float)Tp, sx = (float)axp, sy = (float)ayp, sxy = (float)axyp;
                    // blend coefficients of this splat (_kernels.py:253-262)
                    const float ta = t * al;
                    const float2 cxy = fsub2(fmul2(make_float2(t, t), make_float2(gax, gay)),
                                             fmul2(make_float2(sx, sy), make_float2(al, al)));
                    const float cxx = ((t * gaxy - sxy * al) - sy * gax) - sx * gay;
                    // per-channel adjoint terms u0..u3 and their sums: channels 0 and 1 as
                    // packed pairs, channel 2 scalar
                    const float2 T2 = make_float2(t, t);
                    const float2 d01 = fsub2(make_float2(col.x, col.y), bh01);
                    const float2 u0p = fmul2(T2, d01);
                    const float2 u1p = fsub2(fmul2(make_float2(-sx, -sx), d01), fmul2(T2, bhx01));
                    const float2 u2p = fsub2(fmul2(make_float2(-sy, -sy), d01), fmul2(T2, bhy01));
                    const float2 u3p = fsub2(ffma2(make_float2(sy, sy), bhx01,
                                                   ffma2(make_float2(sx, sx), bhy01,
                                                         fmul2(make_float2(-sxy, -sxy), d01))),
                                             fmul2(T2, bhxy01));
                    const float2 grp = ffma2(WXYp, make_float2(cxx, cxx),
                                             ffma2(WYp, make_float2(cxy.y, cxy.y),
                                                   ffma2(WXp, make_float2(cxy.x, cxy.x),
                                                         fmul2(W0p, make_float2(ta, ta)))));
                    const float2 abp = ffma2(WXYp, u3p, ffma2(WYp, u2p, ffma2(WXp, u1p, fmul2(W0p, u0p))));
                    const float2 abxp = ffma2(WXp, u0p, fmul2(WXYp, u2p));
                    const float2 abyp = ffma2(WYp, u0p, fmul2(WXYp, u1p));
                    const float2 abxyp = fmul2(WXYp, u0p);
                    const float d2 = col.z - bh2;
                    const float u0 = t * d2;
                    const float u1 = -sx * d2 - t * bhx2;
                    const float u2 = -sy * d2 - t * bhy2;
                    const float u3 = ((-sxy * d2 + sx * bhy2) + sy * bhx2) - t * bhxy2;
                    gr[0] = grp.x;
                    gr[1] = grp.y;
                    gr[2] = w[2] * ta + w[5] * cxy.x + w[8] * cxy.y + w[11] * cxx;
                    const float abar = (abp.x + abp.y) + (w[2] * u0 + w[5] * u1 + w[8] * u2 + w[11] * u3);
                    const float abar_x = (abxp.x + abxp.y) + (w[5] * u0 + w[11] * u2);
                    const float abar_y = (abyp.x + abyp.y) + (w[8] * u0 + w[11] * u1);
                    const float abar_xy = (abxyp.x + abxyp.y) + w[11] * u0;
                    if (st != kClamped) {   // _kernels.py:291-336
                        const float dx = (cx - g.mxh) - g.mxl, dy = (cy - g.myh) - g.myl;
                        const float ca = g.a, cb = -0.5f * g.nb2, ccn = g.c;
                        const float gx = -(2.f * ca * dx + 2.f * cb * dy);
                        const float gy = -(2.f * cb * dx + 2.f * ccn * dy);
                        const float hxy = gx * gy - 2.f * cb;
                        // the reference's per-parameter sums share S = abar + abar_x gx + abar_y gy
                        // + abar_xy hxy and P = abar_x + abar_xy gy, Q = abar_y + abar_xy gx:
                        //   d sigma = al S / sigma (the / sigma in the chain), d mean = al (-g S
                        //   + 2 (a P + b Q, b P + c Q)), d conic = al (-D S - ...)
                        const float S = ((abar + abar_x * gx) + abar_y * gy) + abar_xy * hxy;
                        gr[3] = al * S;
                        const float P = abar_x + abar_xy * gy, Q = abar_y + abar_xy * gx;
                        gr[4] = al * (-gx * S + 2.f * (ca * P + cb * Q));
                        gr[5] = al * (-gy * S + 2.f * (cb * P + ccn * Q));
                        gr[6] = al * (-(dx * dx) * S - 2.f * dx * P);
                        gr[7] = al * ((-(2.f * dx * dy) * S - 2.f * dy * P) - 2.f * (dx * Q + abar_xy));
                        gr[8] = al * (-(dy * dy) * S - 2.f * dy * Q);
                    }
                    // advance the behind-colour state through this splat (_kernels.py:337-357)
                    const float omf = (float)om;
                    {
                        const float2 O2 = make_float2(omf, omf);
                        const float2 GX = make_float2(gax, gax), GY = make_float2(gay, gay);
                        const float2 nbx = ffma2(O2, bhx01, fmul2(GX, d01));
                        const float2 nby = ffma2(O2, bhy01, fmul2(GY, d01));
                        const float2 nbxy = fsub2(fsub2(ffma2(O2, bhxy01, fmul2(make_float2(gaxy, gaxy), d01)),
                                                        fmul2(GY, bhx01)),
                                                  fmul2(GX, bhy01));
                        bh01 = ffma2(O2, bh01, fmul2(make_float2(al, al), make_float2(col.x, col.y)));
                        bhx01 = nbx;
                        bhy01 = nby;
                        bhxy01 = nbxy;
                        const float nbx2 = omf * bhx2 + gax * d2;
                        const float nby2 = omf * bhy2 + gay * d2;
                        const float nbxy2 = ((omf * bhxy2 + gaxy * d2) - gay * bhx2) - gax * bhy2;
                        bh2 = omf * bh2 + al * col.z;
                        bhx2 = nbx2;
                        bhy2 = nby2;
                        bhxy2 = nbxy2;
                    }
                    T = Tp;
                    ax = axp;
                    ay = ayp;
                    axy = axyp;
                }
            }
            const uint32_t cb = __ballot_sync(0xffffffffu, contrib);
            if (cb) {
                float g8;
                const float v = group_reduce9(gr, li, g8);
                if ((cb >> (q * 8)) & 0xffu) {
                    S.gpart[warp][q][idx][li] = v;
                    if (li == 0) S.gpart[warp][q][idx][8] = g8;
                    tmask |= 1u << idx;
                }
            }
        }
        __syncwarp();
        uint32_t gm[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) gm[g] = __shfl_sync(0xffffffffu, tmask, g * 8);
        const uint32_t touched = gm[0] | gm[1] | gm[2] | gm[3];
        // wait until the slot's previous batch has been reduced
        if (lane == 0)
            while (*(volatile int*)&S.epoch[slot] != round) __nanosleep(64);
        __syncwarp();
        __threadfence_block();
        if ((touched >> lane) & 1u) {   // this warp's partial of candidate `lane`, groups in fixed order
            float acc[kG];
#pragma unroll
            for (int i = 0; i < kG; ++i) acc[i] = 0.f;
#pragma unroll
            for (int g = 0; g < 4; ++g)
                if ((gm[g] >> lane) & 1u) {
#pragma unroll
                    for (int i = 0; i < kG; ++i) acc[i] += S.gpart[warp][g][lane][i];
                }
#pragma unroll
            for (int i = 0; i < kG; ++i) S.part[slot][warp][lane][i] = acc[i];
        }
        // publish; the last warp of the batch reduces the slot.  Every lane fences its
        // own partial stores and the warp converges before lane 0's release, so the
        // partials are ordered before the `done` increment the reducer acquires.
        __threadfence_block();
        __syncwarp();
        int prev = 0;
        if (lane == 0) {
            S.touch[slot][warp] = touched;
            __threadfence_block();
            prev = atomicAdd(&S.done[slot], 1);
        }
        prev = __shfl_sync(0xffffffffu, prev, 0);
        SPLAT_DCHECK(prev >= 0 && prev < kWarps_bw);
        if (prev == kWarps_bw - 1) {
            __threadfence_block();
            // fixed warp order: one partial per (splat, tile) pair, at its list position
            if (lane < nb) {
                float acc[kG];
#pragma unroll
                for (int i = 0; i < kG; ++i) acc[i] = 0.f;
#pragma unroll
                for (int ww = 0; ww < kWarps_bw; ++ww) {
                    if ((*(volatile uint32_t*)&S.touch[slot][ww] >> lane) & 1u) {
#pragma unroll
                        for (int i = 0; i < kG; ++i) acc[i] += S.part[slot][ww][lane][i];
                    }
                }
                {
                    SPLAT_DCHECK(lo + lane >= start && lo + lane < end);
                    float* dst = p.partial + (size_t)(lo + lane) * kG;
#pragma unroll
                    for (int i = 0; i < kG; ++i) dst[i] = acc[i];
                }
            }
            __syncwarp();   // every lane's reads of the slot precede its release
            if (lane == 0) {
                S.done[slot] = 0;
                __threadfence_block();
                *(volatile int*)&S.epoch[slot] = round + 1;
            }
        }
        __syncwarp();
    }
}

// Per rank: sum its (splat, tile) partials in tile order, the reference's fixed
// tile-order reduction (raster_backward.py:116-124).  The rank's pairs are the
// emission slots offsets[r] .. + touched[r] (tile-rectangle order); slot_pos
// maps each to its list position, where the backward left the partial.
// Per-term view scales for the rank-order accumulation across views (all 1 for the
// single-view path): d_mean x kx / ky and d_conic / (kx^2, kx ky, ky^2), so that a
// view-independent chain (kx = ky = 1) maps the sum over views in one pass.
struct TermScales {
    double s[kG];
};

__global__ void reduce_pairs_kernel(int64_t n, const uint32_t* __restrict__ touched,
                                    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ slot_pos,
                                    const float* __restrict__ partial, int64_t cap, float* __restrict__ g_rank,
                                    TermScales sc, int accumulate) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    float g[kG];
#pragma unroll
    for (int i = 0; i < kG; ++i) g[i] = 0.f;
    const uint32_t off = offsets[r];
    const uint32_t cnt = (uint32_t)min((int64_t)touched[r], cap - (int64_t)off > 0 ? cap - (int64_t)off : (int64_t)0);
    // four pairs' gathers in flight at a time, summed in tile order
    for (uint32_t k = 0; k < cnt; k += 4) {
        uint32_t pos[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pos[u] = k + u < cnt ? slot_pos[off + k + u] : 0xffffffffu;
        float v[4][kG];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float* src = partial + (size_t)(pos[u] == 0xffffffffu ? 0u : pos[u]) * kG;
#pragma unroll
            for (int i = 0; i < kG; ++i) v[u][i] = pos[u] == 0xffffffffu ? 0.f : __ldg(src + i);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (pos[u] != 0xffffffffu) {
#pragma unroll
                for (int i = 0; i < kG; ++i) g[i] += v[u][i];
            }
    }
#pragma unroll
    for (int i = 0; i < kG; ++i) {
        const float v = sc.s[i] == 1.0 ? g[i] : (float)((double)g[i] * sc.s[i]);
        float* d = g_rank + (size_t)r * kG + i;
        *d = accumulate ? *d + v : v;
    }
}

// Per splat, in storage order (coalesced gradient stores): chain the render-space
// gradients of its rank into the stored parametrisation (raster_backward.py:126-152).
// grads layout (float32, n = scene size):
//   [d_means (n,2) | d_log_scales (n,2) | d_rotations (n) | d_opacity_logits (n) | d_colors (n,3)]
__global__ void chain_kernel(int64_t n, const int32_t* __restrict__ rank_of, const float* __restrict__ g_rank,
                             const double* __restrict__ ls, const double* __restrict__ rot,
                             const double* __restrict__ sigma_r, double kx, double ky, int accumulate,
                             float* __restrict__ grads) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int64_t r = rank_of[s];
    float g[kG];
#pragma unroll
    for (int i = 0; i < kG; ++i) g[i] = g_rank[(size_t)r * kG + i];
    const double sg = sigma_r[r];
    const double d_sigma = (double)g[3] / sg;
    const double dn00 = (double)g[6] / (2.0 * kx * kx);
    const double dn01 = (double)g[7] / (2.0 * kx * ky);
    const double dn11 = (double)g[8] / (2.0 * ky * ky);
    const double e1 = exp(-2.0 * ls[2 * s]), e2 = exp(-2.0 * ls[2 * s + 1]);
    double sn, c;
    sincos(rot[s], &sn, &c);
    const double d_l1 = -2.0 * e1 * (dn00 * c * c + dn01 * sn * c + dn11 * sn * sn);
    const double d_l2 = -2.0 * e2 * (dn00 * sn * sn - dn01 * sn * c + dn11 * c * c);
    const double sin2 = 2.0 * sn * c, cos2 = c * c - sn * sn;
    const double d_rot = (e2 - e1) * sin2 * dn00 + (e1 - e2) * cos2 * dn01 + (e1 - e2) * sin2 * dn11;
    const float v[9] = {(float)((double)g[4] * kx), (float)((double)g[5] * ky), (float)d_l1, (float)d_l2,
                        (float)d_rot, (float)(d_sigma * sg * (1.0 - sg)), g[0], g[1], g[2]};
    float* dst[9] = {grads + 2 * s, grads + 2 * s + 1, grads + 2 * n + 2 * s, grads + 2 * n + 2 * s + 1,
                     grads + 4 * n + s, grads + 5 * n + s, grads + 6 * n + 3 * s, grads + 6 * n + 3 * s + 1,
                     grads + 6 * n + 3 * s + 2};
#pragma unroll
    for (int i = 0; i < 9; ++i) *dst[i] = accumulate ? *dst[i] + v[i] : v[i];
}


// ---- decoupled backward (v2) -------------------------------------------------------
// The same per-pixel replay, inversion and per-candidate gradient terms as
// raster_bwd_kernel, reorganised like the forward: persistent warps claim (tile, 8x4
// rectangle) units from a global counter, walk ONLY the pairs whose bbox reaches their
// rectangle (binning's rect masks; 128-pair TMA batches scanned back to front into a
// per-warp ring), and write one partial per (pair, rectangle) -- the warp's four group
// sums added in fixed order -- instead of meeting the tile's other warps at a
// shared-memory ring after every batch.  reduce_pairs2_kernel then sums, per splat, the
// rectangles of each of its tiles in fixed order (rect 0..7) and the tiles in tile order:
// still no atomics, bitwise repeatable.  Rectangles a pair's bbox misses, and list
// positions at or above the last contributor of every live pixel of the rectangle
// (hi2[unit]), contribute zero and are never read.
#ifndef BWD_V2
#define BWD_V2 1
#endif
#ifndef BW2_WARPS
#define BW2_WARPS 4
#endif
#ifndef BW2_EXACT
#define BW2_EXACT eval_exact_inl   // inlined: no call frame in the replay loop (eval_exact: 296-byte stack, C5 -1.4%)
#endif
#ifndef BW2_UNROLL
#define BW2_UNROLL 1   // candidate steps per loop iteration
#endif
#ifndef BW2_MIN_BLOCKS
#define BW2_MIN_BLOCKS 4
#endif
constexpr int kBw2Warps = BW2_WARPS;
constexpr int kBw2Unroll = BW2_UNROLL;
constexpr int kBw2Threads = 32 * kBw2Warps;
constexpr int kBw2Batch = 128;
constexpr int kBw2Queue = 256;
constexpr int kGS = 12;   // floats per (pair, rectangle) partial: three 16-byte stores

struct Bwd2Args {
    SceneConst sc;
    ViewConst vc;
    int width, height, ntx;
    uint32_t nunits;
    const uint32_t* ranges;
    const uint32_t* ranks;
    const uint8_t* rmask;
    const PackF* pack;
    const short4* bboxes;
    const uint32_t* last;
    const int32_t* count;
    const double* state;
    const float* adj;
    float* partial2;      // (cap, 8 rects, kGS) by list position
    uint32_t* hi2;        // (ntiles * 8) replay start of each rectangle
    uint32_t* cursor;     // work-unit counter (zeroed per launch)
};

struct Bwd2Shared {
    struct PackS {
        PackF f;
        float4 col;
    } pack[kBw2Warps][2][32];
    uint32_t rank[kBw2Warps][2][32];
    uint32_t pos[kBw2Warps][2][32];
    __align__(16) uint32_t braw[kBw2Warps][2][kBw2Batch];
    __align__(16) uint32_t bmask[kBw2Warps][2][kBw2Batch / 4];
    uint32_t qr[kBw2Warps][kBw2Queue];
    uint32_t qp[kBw2Warps][kBw2Queue];
    float gpart[kBw2Warps][4][32][kG];
    __align__(8) uint64_t bar[kBw2Warps][2];
};

__device__ __forceinline__ uint32_t bw_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16_bw(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(bw_smem(smem)), "l"(gmem) : "memory");
}

__global__ void __launch_bounds__(kBw2Threads, BW2_MIN_BLOCKS) raster_bwd2_kernel(Bwd2Args p) {
    extern __shared__ __align__(16) unsigned char smem2_raw[];
    Bwd2Shared& S = *reinterpret_cast<Bwd2Shared*>(smem2_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane >> 3, li = lane & 7;
    const uint32_t gt_mask = ~((2u << lane) - 1u);   // lanes above this one
    if (lane == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bw_smem(&S.bar[warp][0])));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bw_smem(&S.bar[warp][1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t bphase = 0u;
    for (;;) {
        uint32_t unit = 0;
        if (lane == 0) unit = atomicAdd(p.cursor, 1u);
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit >= p.nunits) break;
        const int tile = (int)(unit / 8), wr = (int)(unit % 8);
        const int tile_x = tile % p.ntx, tile_y = tile / p.ntx;
        const int rx0 = tile_x * kTile + (wr & 1) * 8, ry0 = tile_y * kTile + (wr >> 1) * 4;
        const int px = rx0 + (q & 1) * 4 + (li & 3), py = ry0 + (q >> 1) * 2 + (li >> 2);
        const bool inside = px < p.width && py < p.height;
        const float cx = (float)px + 0.5f, cy = (float)py + 0.5f;
        const float X0 = (float)rx0 + 0.5f, Y0 = (float)ry0 + 0.5f;
        const uint32_t start = p.ranges[2 * tile], end = p.ranges[2 * tile + 1];
        // per-pixel inputs (as raster_bwd_kernel)
        const int64_t o = (int64_t)py * p.width + px;
        uint32_t my_last = start;
        float w[12];
        double T = 1.0, ax = 0.0, ay = 0.0, axy = 0.0;
        bool live = false;
        if (inside) {
            my_last = p.last[o];
            const float4* a4 = reinterpret_cast<const float4*>(p.adj + 12 * o);
            const float4 w0 = a4[0], w1 = a4[1], w2 = a4[2];
            w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
            w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
            w[8] = w2.x; w[9] = w2.y; w[10] = w2.z; w[11] = w2.w;
            bool nz = false;
#pragma unroll
            for (int i = 0; i < 12; ++i) nz |= (w[i] != 0.f);
            live = nz && p.count[o] > 0;   // _kernels.py:155-174
            const double2* st = reinterpret_cast<const double2*>(p.state + 4 * o);
            const double2 s0 = st[0], s1 = st[1];
            T = s0.x;
            ax = s0.y;
            ay = s1.x;
            axy = s1.y;
        } else {
#pragma unroll
            for (int i = 0; i < 12; ++i) w[i] = 0.f;
        }
        float2 bh01 = make_float2(p.vc.bg[0], p.vc.bg[1]), bhx01 = make_float2(0.f, 0.f);
        float2 bhy01 = make_float2(0.f, 0.f), bhxy01 = make_float2(0.f, 0.f);
        float bh2 = p.vc.bg[2], bhx2 = 0.f, bhy2 = 0.f, bhxy2 = 0.f;
        const float2 W0p = make_float2(w[0], w[1]), WXp = make_float2(w[3], w[4]);
        const float2 WYp = make_float2(w[6], w[7]), WXYp = make_float2(w[9], w[10]);
        const uint32_t warp_hi = __reduce_max_sync(0xffffffffu, live ? my_last : start);
        if (lane == 0) p.hi2[unit] = warp_hi;
        if (warp_hi > start) {
            // windows of 128 positions aligned to 16, from the top down: window k covers
            // [top - 128 (k + 1), top - 128 k), copied from max(that, 0) so buffer index i is
            // position wbot + i
            const int64_t top = ((int64_t)warp_hi + 15) & ~(int64_t)15;
            auto issue_batch = [&](int64_t wtop, int k) {   // lane 0
                const int64_t wbot = wtop - kBw2Batch, lo = wbot < 0 ? 0 : wbot;
                const uint32_t nel = (uint32_t)(wtop - lo), skip = (uint32_t)(lo - wbot);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bw_smem(&S.bar[warp][k])),
                             "r"(nel * 5u) : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        bw_smem(&S.braw[warp][k][skip])),
                    "l"(p.ranks + lo), "r"(nel * 4u), "r"(bw_smem(&S.bar[warp][k]))
                    : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        bw_smem(reinterpret_cast<uint8_t*>(&S.bmask[warp][k][0]) + skip)),
                    "l"(p.rmask + lo), "r"(nel), "r"(bw_smem(&S.bar[warp][k]))
                    : "memory");
            };
            // windows exist while their top is above start
            if (lane == 0) {
                issue_batch(top, 0);
                if (top - kBw2Batch > (int64_t)start) issue_batch(top - kBw2Batch, 1);
            }
            int64_t wnext = top;   // top of the next window to scan
            int kwin = 0;          // its index (buffer kwin & 1)
            uint32_t qh = 0, qt = 0;
            auto refill = [&]() {
                while (qt - qh < 32u && wnext > (int64_t)start) {
                    const int k = kwin & 1;
                    asm volatile("" ::: "memory");
                    {
                        uint32_t done = 0;
                        const uint32_t par = (bphase >> k) & 1u;
                        while (!done) {
                            asm volatile(
                                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                                : "=r"(done)
                                : "r"(bw_smem(&S.bar[warp][k])), "r"(par)
                                : "memory");
                        }
                    }
                    bphase ^= 1u << k;
                    const int64_t wbot = wnext - kBw2Batch;
                    const uint32_t m4 = S.bmask[warp][k][lane];
                    uint32_t keep = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int64_t pos = wbot + 4 * lane + j;
                        if (((m4 >> (8 * j + wr)) & 1u) && pos >= (int64_t)start && pos < (int64_t)warp_hi)
                            keep |= 1u << j;
                    }
                    const uint32_t c = __popc(keep);
                    const uint32_t v0 = __ballot_sync(0xffffffffu, c & 1u), v1 = __ballot_sync(0xffffffffu, c & 2u),
                                   v2 = __ballot_sync(0xffffffffu, c & 4u);
                    // descending positions: higher lanes, and higher j within a lane, come first
                    uint32_t at = qt + __popc(v0 & gt_mask) + 2u * __popc(v1 & gt_mask) + 4u * __popc(v2 & gt_mask);
#pragma unroll
                    for (int j = 3; j >= 0; --j)
                        if ((keep >> j) & 1u) {
                            S.qr[warp][at & (kBw2Queue - 1)] = S.braw[warp][k][4 * lane + j];
                            S.qp[warp][at & (kBw2Queue - 1)] = (uint32_t)(wbot + 4 * lane + j);
                            ++at;
                        }
                    qt += __popc(v0) + 2u * __popc(v1) + 4u * __popc(v2);
                    SPLAT_DCHECK(qt - qh <= (uint32_t)kBw2Queue);
                    __syncwarp();
                    wnext -= kBw2Batch;
                    ++kwin;
                    if (lane == 0 && wnext - kBw2Batch > (int64_t)start) issue_batch(wnext - kBw2Batch, k);
                }
                __syncwarp();
            };
            auto stage = [&](int b) -> int {
                const int n = (int)min(32u, qt - qh);
                if (lane < n) {
                    const uint32_t e = (qh + (uint32_t)lane) & (kBw2Queue - 1);
                    const uint32_t r = S.qr[warp][e];
                    SPLAT_DCHECK((int64_t)r < p.sc.n);
                    const float4* src = reinterpret_cast<const float4*>(p.pack + r);
                    float4* dst = reinterpret_cast<float4*>(&S.pack[warp][b][lane].f);
                    cp_async16_bw(dst, src);
                    cp_async16_bw(dst + 1, src + 1);
                    cp_async16_bw(dst + 2, src + 2);
                    cp_async16_bw(dst + 3, src + 3);
                    cp_async16_bw(&S.pack[warp][b][lane].col, p.sc.color + r);
                    S.rank[warp][b][lane] = r;
                    S.pos[warp][b][lane] = S.qp[warp][e];
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
                qh += (uint32_t)n;
                return n;
            };
            refill();
            int ncur = stage(0);
            int b = 0;
            while (ncur > 0) {
                refill();
                const int nnext = stage(b ^ 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                __syncwarp();
                uint32_t gmask = 0;   // bit g: candidate `lane` reaches group g's 4x2 rectangle
                if (lane < ncur) {
                    const PackF& g = S.pack[warp][b][lane].f;
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
                uint32_t my_mask = 0;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const uint32_t mq = __ballot_sync(0xffffffffu, (gmask >> qq) & 1u);
                    cnt_max = max(cnt_max, __popc(mq));
                    if (qq == q) my_mask = mq;
                }
                uint32_t tmask = 0;   // this lane's group: candidates it produced partials for
#pragma unroll kBw2Unroll
                for (int k = 0; k < cnt_max; ++k) {   // chunk index ascending = list position descending
                    const bool has = my_mask != 0u;
                    const int idx = has ? __ffs(my_mask) - 1 : 0;
                    if (has) my_mask &= my_mask - 1u;
                    float gr[kG];
#pragma unroll
                    for (int i = 0; i < kG; ++i) gr[i] = 0.f;
                    bool contrib = false;
                    if (has && live && S.pos[warp][b][idx] < my_last) {
                        const PackF g = S.pack[warp][b][idx].f;
                        float al, gax, gay, gaxy, rel;
                        int st = eval_fast(g, cx, cy, al, gax, gay, gaxy, rel);
                        if (st == kUnsure) {
                            double a64;
                            st = BW2_EXACT(p.sc, p.vc, p.bboxes, S.rank[warp][b][idx], px, py, &a64);
                            if (st != kCulled) canonical_values(g, cx, cy, st, al, gax, gay, gaxy);
                        }
                        if (st != kCulled) {
                            contrib = true;
                            const float4 col = S.pack[warp][b][idx].col;
                            // invert the accumulated-alpha state across this splat (float64)
                            const double om = st == kClamped ? (double)1.0e-3f : (double)(1.f - al);
                            // 1/om: float32 reciprocal refined by two float64 Newton steps (|rel err| ~ 1e-16)
                            double inv = (double)fast_rcp((float)om);
                            inv = inv * fma(-om, inv, 2.0);
                            inv = inv * fma(-om, inv, 2.0);
                            const double Tp = T * inv;
                            const double axp = (ax - Tp * (double)gax) * inv;
                            const double ayp = (ay - Tp * (double)gay) * inv;
                            const double axyp = (axy - Tp * (double)gaxy + axp * (double)gay + ayp * (double)gax) * inv;
                            const float t = (float)Tp, sx = (float)axp, sy = (float)ayp, sxy = (float)axyp;
                            // blend coefficients of this splat (_kernels.py:253-262)
                            const float ta = t * al;
                            const float2 cxy = fsub2(fmul2(make_float2(t, t), make_float2(gax, gay)),
                                                     fmul2(make_float2(sx, sy), make_float2(al, al)));
                            const float cxx = ((t * gaxy - sxy * al) - sy * gax) - sx * gay;
                            // per-channel adjoint terms u0..u3 and their sums: channels 0 and 1 as
                            // packed pairs, channel 2 scalar
                            const float2 T2 = make_float2(t, t);
                            const float2 d01 = fsub2(make_float2(col.x, col.y), bh01);
                            const float2 u0p = fmul2(T2, d01);
                            const float2 u1p = fsub2(fmul2(make_float2(-sx, -sx), d01), fmul2(T2, bhx01));
                            const float2 u2p = fsub2(fmul2(make_float2(-sy, -sy), d01), fmul2(T2, bhy01));
                            const float2 u3p = fsub2(ffma2(make_float2(sy, sy), bhx01,
                                                           ffma2(make_float2(sx, sx), bhy01,
                                                                 fmul2(make_float2(-sxy, -sxy), d01))),
                                                     fmul2(T2, bhxy01));
                            const float2 grp = ffma2(WXYp, make_float2(cxx, cxx),
                                                     ffma2(WYp, make_float2(cxy.y, cxy.y),
                                                           ffma2(WXp, make_float2(cxy.x, cxy.x),
                                                                 fmul2(W0p, make_float2(ta, ta)))));
                            const float2 abp = ffma2(WXYp, u3p, ffma2(WYp, u2p, ffma2(WXp, u1p, fmul2(W0p, u0p))));
                            const float2 abxp = ffma2(WXp, u0p, fmul2(WXYp, u2p));
                            const float2 abyp = ffma2(WYp, u0p, fmul2(WXYp, u1p));
                            const float2 abxyp = fmul2(WXYp, u0p);
                            const float d2 = col.z - bh2;
                            const float u0 = t * d2;
                            const float u1 = -sx * d2 - t * bhx2;
                            const float u2 = -sy * d2 - t * bhy2;
                            const float u3 = ((-sxy * d2 + sx * bhy2) + sy * bhx2) - t * bhxy2;
                            gr[0] = grp.x;
                            gr[1] = grp.y;
                            gr[2] = w[2] * ta + w[5] * cxy.x + w[8] * cxy.y + w[11] * cxx;
                            const float abar = (abp.x + abp.y) + (w[2] * u0 + w[5] * u1 + w[8] * u2 + w[11] * u3);
                            const float abar_x = (abxp.x + abxp.y) + (w[5] * u0 + w[11] * u2);
                            const float abar_y = (abyp.x + abyp.y) + (w[8] * u0 + w[11] * u1);
                            const float abar_xy = (abxyp.x + abxyp.y) + w[11] * u0;
                            if (st != kClamped) {   // _kernels.py:291-336
                                const float dx = (cx - g.mxh) - g.mxl, dy = (cy - g.myh) - g.myl;
                                const float ca = g.a, cb = -0.5f * g.nb2, ccn = g.c;
                                const float gx = -(2.f * ca * dx + 2.f * cb * dy);
                                const float gy = -(2.f * cb * dx + 2.f * ccn * dy);
                                const float hxy = gx * gy - 2.f * cb;
                                // the reference's per-parameter sums share S = abar + abar_x gx + abar_y gy
                                // + abar_xy hxy and P = abar_x + abar_xy gy, Q = abar_y + abar_xy gx:
                                //   d sigma = al S / sigma (the / sigma in the chain), d mean = al (-g S
                                //   + 2 (a P + b Q, b P + c Q)), d conic = al (-D S - ...)
                                const float S = ((abar + abar_x * gx) + abar_y * gy) + abar_xy * hxy;
                                gr[3] = al * S;
                                const float P = abar_x + abar_xy * gy, Q = abar_y + abar_xy * gx;
                                gr[4] = al * (-gx * S + 2.f * (ca * P + cb * Q));
                                gr[5] = al * (-gy * S + 2.f * (cb * P + ccn * Q));
                                gr[6] = al * (-(dx * dx) * S - 2.f * dx * P);
                                gr[7] = al * ((-(2.f * dx * dy) * S - 2.f * dy * P) - 2.f * (dx * Q + abar_xy));
                                gr[8] = al * (-(dy * dy) * S - 2.f * dy * Q);
                            }
                            // advance the behind-colour state through this splat (_kernels.py:337-357)
                            const float omf = (float)om;
                            {
                                const float2 O2 = make_float2(omf, omf);
                                const float2 GX = make_float2(gax, gax), GY = make_float2(gay, gay);
                                const float2 nbx = ffma2(O2, bhx01, fmul2(GX, d01));
                                const float2 nby = ffma2(O2, bhy01, fmul2(GY, d01));
                                const float2 nbxy = fsub2(fsub2(ffma2(O2, bhxy01, fmul2(make_float2(gaxy, gaxy), d01)),
                                                                fmul2(GY, bhx01)),
                                                          fmul2(GX, bhy01));
                                bh01 = ffma2(O2, bh01, fmul2(make_float2(al, al), make_float2(col.x, col.y)));
                                bhx01 = nbx;
                                bhy01 = nby;
                                bhxy01 = nbxy;
                                const float nbx2 = omf * bhx2 + gax * d2;
                                const float nby2 = omf * bhy2 + gay * d2;
                                const float nbxy2 = ((omf * bhxy2 + gaxy * d2) - gay * bhx2) - gax * bhy2;
                                bh2 = omf * bh2 + al * col.z;
                                bhx2 = nbx2;
                                bhy2 = nby2;
                                bhxy2 = nbxy2;
                            }
                            T = Tp;
                            ax = axp;
                            ay = ayp;
                            axy = axyp;
                        }
                    }
                    const uint32_t cb = __ballot_sync(0xffffffffu, contrib);
                    if (cb) {
                        float g8;
                        const float v = group_reduce9(gr, li, g8);
                        if ((cb >> (q * 8)) & 0xffu) {
                            S.gpart[warp][q][idx][li] = v;
                            if (li == 0) S.gpart[warp][q][idx][8] = g8;
                            tmask |= 1u << idx;
                        }
                    }
                }
                __syncwarp();
                uint32_t gm[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) gm[g] = __shfl_sync(0xffffffffu, tmask, g * 8);
                if (lane < ncur) {   // this rectangle's partial of candidate `lane`, groups in fixed order
                    float acc[kG];
#pragma unroll
                    for (int i = 0; i < kG; ++i) acc[i] = 0.f;
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        if ((gm[g] >> lane) & 1u) {
#pragma unroll
                            for (int i = 0; i < kG; ++i) acc[i] += S.gpart[warp][g][lane][i];
                        }
                    const uint32_t pos = S.pos[warp][b][lane];
                    SPLAT_DCHECK(pos >= start && pos < warp_hi);
                    float4* d = reinterpret_cast<float4*>(p.partial2 + ((size_t)pos * 8 + wr) * kGS);
                    d[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                    d[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
                    d[2] = make_float4(acc[8], 0.f, 0.f, 0.f);
                }
                __syncwarp();
                ncur = nnext;
                b ^= 1;
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            // windows still in flight: at wnext and wnext - kBw2Batch while above start
            for (int i = 0; i < 2 && wnext > (int64_t)start; ++i) {
                const int k = kwin & 1;
                uint32_t done = 0;
                const uint32_t par = (bphase >> k) & 1u;
                while (!done) {
                    asm volatile(
                        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                        : "=r"(done)
                        : "r"(bw_smem(&S.bar[warp][k])), "r"(par)
                        : "memory");
                }
                bphase ^= 1u << k;
                wnext -= kBw2Batch;
                ++kwin;
            }
            __syncwarp();
        }
    }
}

// Per rank: the sum over its tiles (tile order) of the sum over the tile's rectangles its
// bbox reaches (rect order) of the rectangle's partial -- zero where the rectangle's
// replay started below the pair (position >= hi2).
__global__ void reduce_pairs2_kernel(int64_t n, int ntx, const uint32_t* __restrict__ touched,
                                     const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ slot_pos,
                                     const short4* __restrict__ bboxes, const uint32_t* __restrict__ hi2,
                                     const float* __restrict__ partial2,
                                     int64_t cap, float* __restrict__ g_rank, TermScales sc, int accumulate) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    float g[kG];
#pragma unroll
    for (int i = 0; i < kG; ++i) g[i] = 0.f;
    const uint32_t off = offsets[r];
    const uint32_t cnt = (uint32_t)min((int64_t)touched[r], cap - (int64_t)off > 0 ? cap - (int64_t)off : (int64_t)0);
    if (cnt) {
        const short4 bb = bboxes[r];
        const int tx0 = bb.x >> 4, ty0 = bb.z >> 4, nx = ((bb.y - 1) >> 4) - tx0 + 1;
        int tx = tx0, ty = ty0;
        for (uint32_t k = 0; k < cnt; ++k) {
            // the rect mask is recomputed (as the binning computed it) and the rectangles'
            // replay starts loaded beside the position: one dependent step to the partials
            const uint32_t pos = slot_pos[off + k];
            const int t = ty * ntx + tx;
            const uint32_t m = rect_mask(bb, tx, ty);
            uint32_t h[8];
#pragma unroll
            for (int rect = 0; rect < 8; ++rect) h[rect] = ((m >> rect) & 1u) ? __ldg(hi2 + 8 * t + rect) : 0u;
#pragma unroll
            for (int rect = 0; rect < 8; ++rect) {
                if (pos < h[rect]) {
                    const float4* s = reinterpret_cast<const float4*>(partial2 + ((size_t)pos * 8 + rect) * kGS);
                    const float4 a = __ldg(s), c = __ldg(s + 1);
                    const float e = __ldg(reinterpret_cast<const float*>(s + 2));
                    g[0] += a.x; g[1] += a.y; g[2] += a.z; g[3] += a.w;
                    g[4] += c.x; g[5] += c.y; g[6] += c.z; g[7] += c.w;
                    g[8] += e;
                }
            }
            if (++tx - tx0 == nx) {
                tx = tx0;
                ++ty;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < kG; ++i) {
        const float v = sc.s[i] == 1.0 ? g[i] : (float)((double)g[i] * sc.s[i]);
        float* d = g_rank + (size_t)r * kG + i;
        *d = accumulate ? *d + v : v;
    }
}

}  // namespace

// partials: (cap, kG) per pair (v1) or (cap, 8 rects, kGS) per (pair, rectangle) (v2)
constexpr size_t kPartialBytes = BWD_V2 ? 8 * kGS * 4 : kG * 4;

size_t backward_workspace_bytes_impl(int64_t n, int64_t cap) {
    size_t nn = (size_t)(n > 0 ? n : 1), cc = (size_t)(cap > 0 ? cap : 1);
    return ((cc * kPartialBytes + 255) & ~size_t(255)) + nn * kG * 4;
}

int launch_raster_backward(const SceneConst& sc, const splat_scene_t& scene, const ViewConst& vc,
                           const FrameLayout& L, char* ws, const splat_gimg_t& fwd, const float* adj,
                           char* bws, float* grads, int accumulate, cudaStream_t stream, float* rank_out) {
    const size_t nn = (size_t)(L.n > 0 ? L.n : 1), cc = (size_t)(L.cap > 0 ? L.cap : 1);
    float* partial = (float*)bws;
    if (L.n == 0) return SPLAT_OK;
    float* g_rank = (float*)(bws + ((cc * kPartialBytes + 255) & ~size_t(255)));
    (void)nn;
    const int blocks = (int)((L.n + 255) / 256);
    TermScales ts;
    for (int i = 0; i < kG; ++i) ts.s[i] = 1.0;
    if (rank_out) {   // rank-order, view-scaled terms accumulated for one chain over all views
        ts.s[4] = vc.kx;
        ts.s[5] = vc.ky;
        ts.s[6] = 1.0 / (vc.kx * vc.kx);
        ts.s[7] = 1.0 / (vc.kx * vc.ky);
        ts.s[8] = 1.0 / (vc.ky * vc.ky);
    }
    if (BWD_V2) {
        Bwd2Args a;
        a.sc = sc;
        a.vc = vc;
        a.width = L.width;
        a.height = L.height;
        a.ntx = L.ntx;
        a.nunits = (uint32_t)L.ntx * (uint32_t)L.nty * 8u;
        a.ranges = (const uint32_t*)(ws + L.ranges);
        a.ranks = (const uint32_t*)(ws + L.vals0);
        a.rmask = (const uint8_t*)(ws + L.rmask);
        a.pack = (const PackF*)(ws + L.pack);
        a.bboxes = (const short4*)(ws + L.bboxes);
        a.last = fwd.last;
        a.count = fwd.count;
        a.state = fwd.state;
        a.adj = adj;
        a.partial2 = partial;
        a.hi2 = (uint32_t*)(ws + L.bwd_hi);
        a.cursor = (uint32_t*)(ws + L.bwd_cursor);
        static PerDevice<int> grid2;
        int g2 = 0;
        const int rc2 = grid2.get(g2, [](int& v) {
            SPLAT_CUDA_CHECK(cudaFuncSetAttribute(raster_bwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)sizeof(Bwd2Shared)));
            int per_sm = 0;
            SPLAT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raster_bwd2_kernel, kBw2Threads,
                                                                           sizeof(Bwd2Shared)));
            int sms = 0;
            const int e = device_sms(sms);
            if (e != SPLAT_OK) return e;
            v = sms * (per_sm > 0 ? per_sm : 1);
            return SPLAT_OK;
        });
        if (rc2 != SPLAT_OK) return rc2;
        SPLAT_CUDA_CHECK(cudaMemsetAsync(a.cursor, 0, 4, stream));
        const int nblk = (int)std::min<int64_t>(g2, ((int64_t)a.nunits + kBw2Warps - 1) / kBw2Warps);
        raster_bwd2_kernel<<<nblk, kBw2Threads, sizeof(Bwd2Shared), stream>>>(a); note_launch();
        reduce_pairs2_kernel<<<blocks, 256, 0, stream>>>(
            L.n, L.ntx, (const uint32_t*)(ws + L.touched), (const uint32_t*)(ws + L.offsets),
            (const uint32_t*)(ws + L.slot_pos), (const short4*)(ws + L.bboxes), a.hi2, partial, L.cap, rank_out ? rank_out : g_rank, ts, rank_out ? accumulate : 0);
        note_launch();
        if (!rank_out) {
            chain_kernel<<<blocks, 256, 0, stream>>>(L.n, sc.rank_of, g_rank, scene.log_scales, scene.rotations,
                                                     sc.sigma, vc.kx, vc.ky, accumulate, grads);
            note_launch();
        }
        SPLAT_CUDA_CHECK(cudaGetLastError());
        return SPLAT_OK;
    }
    BwdArgs a;
    a.sc = sc;
    a.vc = vc;
    a.width = L.width;
    a.height = L.height;
    a.ntx = L.ntx;
    a.ranges = (const uint32_t*)(ws + L.ranges);
    a.ranks = (const uint32_t*)(ws + L.vals0);
    a.pack = (const PackF*)(ws + L.pack);
    a.bboxes = (const short4*)(ws + L.bboxes);
    a.offsets = (const uint32_t*)(ws + L.offsets);
    a.last = fwd.last;
    a.count = fwd.count;
    a.state = fwd.state;
    a.adj = adj;
    a.partial = partial;
    static PerDevice<bool> configured;
    bool ok = false;
    const int rc = configured.get(ok, [](bool& v) {
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(raster_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)sizeof(BwdShared)));
        v = true;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    raster_bwd_kernel<<<L.ntx * L.nty, kBlock, sizeof(BwdShared), stream>>>(a); note_launch();
    if (rank_out) {
        reduce_pairs_kernel<<<blocks, 256, 0, stream>>>(L.n, (const uint32_t*)(ws + L.touched),
                                                        (const uint32_t*)(ws + L.offsets),
                                                        (const uint32_t*)(ws + L.slot_pos), partial, L.cap, rank_out,
                                                        ts, accumulate);
        note_launch();
        SPLAT_CUDA_CHECK(cudaGetLastError());
        return SPLAT_OK;
    }
    reduce_pairs_kernel<<<blocks, 256, 0, stream>>>(L.n, (const uint32_t*)(ws + L.touched),
                                                    (const uint32_t*)(ws + L.offsets),
                                                    (const uint32_t*)(ws + L.slot_pos), partial, L.cap, g_rank, ts, 0);
    note_launch();
    chain_kernel<<<blocks, 256, 0, stream>>>(L.n, sc.rank_of, g_rank, scene.log_scales, scene.rotations, sc.sigma,
                                             vc.kx, vc.ky, accumulate, grads);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

int launch_chain(const SceneConst& sc, const splat_scene_t& scene, const float* rank_grads, float* grads,
                 int accumulate, cudaStream_t stream) {
    if (scene.n == 0) return SPLAT_OK;
    chain_kernel<<<(int)((scene.n + 255) / 256), 256, 0, stream>>>(scene.n, sc.rank_of, rank_grads, scene.log_scales,
                                                                  scene.rotations, sc.sigma, 1.0, 1.0, accumulate,
                                                                  grads);
    note_launch();
    SPLAT_CUDA_CHECK(cudaGetLastError());
    return SPLAT_OK;
}

}  // namespace splat
