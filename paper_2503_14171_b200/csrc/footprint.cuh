// Certified per-pixel footprint evaluation shared by the forward and backward
// rasterizers: the float32 fast path with a rigorous error bound, the exact
// float64 reference evaluation it falls back to, and the canonical float32
// values both passes blend with (so the backward replays the forward's
// decisions and values bit for bit).
#pragma once
#include <cmath>
#include <cstring>

#include "kernels.cuh"

namespace splat {
namespace {

enum : int { kCulled = 0, kContrib = 1, kClamped = 2, kUnsure = 3 };


// Exact reference evaluation of one candidate at one pixel centre
// (_kernels.py:61-80, float64, every operation individually rounded).
__device__ __forceinline__ int eval_exact_inl(const SceneConst& sc, const ViewConst& vc,
                                              const short4* bboxes, uint32_t r, int px, int py,
                                              double* alpha64) {
    short4 bb = bboxes[r];
    if (px < bb.x || px >= bb.y || py < bb.z || py >= bb.w) return kCulled;
    double mx = __dmul_rn(__dsub_rn(sc.mean[2 * r], vc.ox), vc.kx);
    double my = __dmul_rn(__dsub_rn(sc.mean[2 * r + 1], vc.oy), vc.ky);
    double ca = __ddiv_rn(sc.n00[r], vc.c00);
    double cb = __ddiv_rn(sc.n01[r], vc.c01);
    double cc = __ddiv_rn(sc.n11[r], vc.c11);
    double dx = __dsub_rn((double)px + 0.5, mx);
    double dy = __dsub_rn((double)py + 0.5, my);
    double t1 = __dmul_rn(__dmul_rn(ca, dx), dx);
    double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, cb), dx), dy);
    double t3 = __dmul_rn(__dmul_rn(cc, dy), dy);
    double expo = -__dadd_rn(__dadd_rn(t1, t2), t3);
    if (expo < kLogCull) return kCulled;
    double araw = __dmul_rn(sc.sigma[r], exp(expo));
    if (araw < kAlphaCull) return kCulled;
    if (araw > kAlphaClamp) {
        *alpha64 = kAlphaClamp;
        return kClamped;
    }
    *alpha64 = araw;
    return kContrib;
}

// Out-of-line copy for the main pass, where the exact path is rare and must
// not inflate the register footprint of the hot loop.
__device__ __noinline__ int eval_exact(const SceneConst& sc, const ViewConst& vc, const short4* bboxes,
                                       uint32_t r, int px, int py, double* alpha64) {
    return eval_exact_inl(sc, vc, bboxes, r, px, py, alpha64);
}

// 2^x via MUFU.EX2 (flush-to-zero: results below 2^-126 are far below the cull).
// Max relative error 2^-22, inside the 2^-20 budget of eval_fast's `rel`.
__device__ __forceinline__ float fast_exp2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float fast_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Float32 footprint with a certified decision (_kernels.py:65-87).  Returns
// kCulled / kContrib / kClamped when the float32 evaluation decides the
// reference's tests with margin, kUnsure otherwise.  `al` etc. are the
// canonical float32 values used for blending (identical in the backward pass);
// `rel` receives the relative error bound of `al`.
__device__ __forceinline__ uint64_t f2_bits(float2 v) {
    uint64_t r;
    memcpy(&r, &v, 8);
    return r;
}
__device__ __forceinline__ float2 bits_f2(uint64_t r) {
    float2 v;
    memcpy(&v, &r, 8);
    return v;
}
// Packed float32x2 arithmetic (sm_100 FADD2 / FMUL2 / FFMA2): two IEEE ops per instruction.
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
    return bits_f2(r);
}

// RAW: return the gradient factors (gx, gy, h = gx gy - 2b) instead of
// (al gx, al gy, al h) — the inference blend multiplies by al itself.
template <bool RAW = false>
__device__ __forceinline__ int eval_fast(const PackF& g, float cx, float cy, float& al, float& ax,
                                         float& ay, float& axy, float& rel) {
    // (dx, dy) = ((cx, cy) - (mxh, myh)) - (mxl, myl), and (a dx, c dy) as packed pairs
    const float2 d = fsub2(fsub2(make_float2(cx, cy), make_float2(g.mxh, g.myh)), make_float2(g.mxl, g.myl));
    const float dx = d.x, dy = d.y;
    const float2 acd = fmul2(make_float2(g.a, g.c), d);
    const float adx = acd.x;
    const float2 t13 = fmul2(acd, d);   // (a dx dx, c dy dy)
    float t1 = t13.x;
    float t2 = ((-g.nb2) * dx) * dy;   // (2b dx) dy
    float t3 = t13.y;
    float qf = (t1 + t2) + t3;
    float s = (t1 + fabsf(t2)) + t3;
    // |qf - Q_exact| <= ~8 ulp * s; conic/mean rounding adds ~4 ulp * s.  2^-19 * s is a 2x margin
    // (the one rounding of lo/hi below adds <= 0.5 ulp * s).  The tests are qf -+ tol against the
    // thresholds with tol = (s + qcull) 2^-19; the qcull part is folded into the pack's
    // outward-rounded cull_hi/lo, clamp_hi/lo.  (s + qcull = 0: every test below is "unsure".)
    const float lo = fmaf(s, -1.9073486e-06f, qf), hi = fmaf(s, 1.9073486e-06f, qf);
    // |al - alpha_ref| / al <= 2^-21 s (Q) + 2^-20 (exp2 approx 2^-22; rounding of the
    // argument, of log2(e) and of log2(sigma), each <= 2^-22 absolute for |argument| <= 8);
    // + 2^-24 for the extra rounding of t al in the forward's T' = T - t al
    if (lo > g.cull_hi) return kCulled;   // (rel after the cull test: culls are half the evaluations)
    rel = fmaf(s, 4.7683716e-07f, 1.0132790e-06f);
    if (hi >= g.cull_lo) return kUnsure;
    if (lo <= g.clamp_hi) {
        if (hi < g.clamp_lo) {
            al = 0.999f;
            ax = 0.f;
            ay = 0.f;
            axy = 0.f;
            // 1 - 0.999f = 1e-3 (1 - 1.3e-5): the inference blend's T - T al carries that
            // relative error of om (= 1.3e-8 / al), which this bound covers
            rel = 1.6e-5f;
            return kClamped;
        }
        return kUnsure;
    }
    al = fast_exp2(fmaf(qf, -1.44269504f, g.l2sig));
    // (gx, gy) = -2 ((b dy, b dx) + (a dx, c dy)) = (-2b) (dy, dx) + (-2) (a dx, c dy), bit for bit
    const float2 gxy = ffma2(make_float2(g.nb2, g.nb2), make_float2(dy, dx), fmul2(acd, make_float2(-2.f, -2.f)));
    if (RAW) {
        ax = gxy.x;
        ay = gxy.y;
        axy = fmaf(gxy.x, gxy.y, g.nb2);
    } else {
        const float2 axy2 = fmul2(make_float2(al, al), gxy);
        ax = axy2.x;
        ay = axy2.y;
        axy = al * fmaf(gxy.x, gxy.y, g.nb2);
    }
    return kContrib;
}

// Values of a candidate whose decision came from the exact path.
template <bool RAW = false>
__device__ __forceinline__ void canonical_values(const PackF& g, float cx, float cy, int st, float& al,
                                                 float& ax, float& ay, float& axy) {
    if (st == kClamped) {
        al = 0.999f;
        ax = ay = axy = 0.f;
        return;
    }
    float dx = (cx - g.mxh) - g.mxl;
    float dy = (cy - g.myh) - g.myl;
    float adx = g.a * dx;
    const float b = -0.5f * g.nb2, b2 = -g.nb2;
    float qf = ((adx * dx) + ((b2 * dx) * dy)) + ((g.c * dy) * dy);
    al = fast_exp2(fmaf(qf, -1.44269504f, g.l2sig));
    float gx = -2.f * fmaf(b, dy, adx);
    float gy = -2.f * fmaf(b, dx, g.c * dy);
    if (RAW) {
        ax = gx;
        ay = gy;
        axy = fmaf(gx, gy, -b2);
    } else {
        ax = al * gx;
        ay = al * gy;
        axy = al * fmaf(gx, gy, -b2);
    }
}

// Group pre-filter: bit g set unless the cull ellipse certainly misses 4x2
// group g of the 8x4 pixel-centre rectangle whose first centre is (X0, Y0)
// (groups: bit 0 at (X0, Y0), bit 1 at x + 4, bit 2 at y + 2, bit 3 at both).
// Q-norm triangle inequality at each group centre G: some centre p of the group
// has Q(p - m) <= q only if Q(G - m) <= pad2 (preprocess_kernel).  The float32
// error of Q(G - m) is <= 8 ulp (t1 + |t2| + t3) <= 16 ulp (t1 + t3) for a
// positive-definite form, which the 2^-18 (t1 + t3) allowance covers.
__device__ __forceinline__ uint32_t group_qnorm_mask(const PackF& g, float X0, float Y0) {
    const float2 d0 = fsub2(fsub2(make_float2(X0 + 1.5f, Y0 + 0.5f), make_float2(g.mxh, g.myh)),
                            make_float2(g.mxl, g.myl));
    const float2 dxs = make_float2(d0.x, d0.x + 4.f), dys = make_float2(d0.y, d0.y + 2.f);
    const float2 t1 = fmul2(fmul2(make_float2(g.a, g.a), dxs), dxs);
    const float2 t3 = fmul2(fmul2(make_float2(g.c, g.c), dys), dys);
    const float2 bx = fmul2(make_float2(-g.nb2, -g.nb2), dxs);
    // groups 0, 1 (row dys.x) and 2, 3 (row dys.y)
    const float2 s01 = fadd2(t1, make_float2(t3.x, t3.x));
    const float2 s23 = fadd2(t1, make_float2(t3.y, t3.y));
    const float2 q01 = ffma2(bx, make_float2(dys.x, dys.x), s01);
    const float2 q23 = ffma2(bx, make_float2(dys.y, dys.y), s23);
    const float2 k = make_float2(-3.8146973e-06f, -3.8146973e-06f);
    const float2 l01 = ffma2(s01, k, q01), l23 = ffma2(s23, k, q23);
    const float tau = g.pad2;
    return (l01.x <= tau ? 1u : 0u) | (l01.y <= tau ? 2u : 0u) | (l23.x <= tau ? 4u : 0u) |
           (l23.y <= tau ? 8u : 0u);
}

// Conservative "does the cull ellipse {Q <= qcull} reach the pixel-centre
// rectangle [X0,X1] x [Y0,Y1]" test.  The minimum of the positive-definite
// form over the rectangle is at the centre (if inside) or on an edge, where it
// is a 1-D quadratic minimised in closed form.  Each edge value is lowered by
// a bound on its float32 error (2^-18 (a u^2 + c v^2) >= 8 ulp * s) before the
// comparison, and NaNs keep the candidate, so no contributing candidate is
// ever rejected.  cull_hi >= qcull keeps the test conservative; b/a and b/c are
// approximate quotients (a perturbed edge minimiser only raises the edge value by O(eps^2),
// far inside the 2^-18 margin).
__device__ __forceinline__ bool ellipse_hits_rect(const PackF& g, float X0, float X1, float Y0, float Y1) {
    const float u0 = (X0 - g.mxh) - g.mxl, u1 = (X1 - g.mxh) - g.mxl;
    const float v0 = (Y0 - g.myh) - g.myl, v1 = (Y1 - g.myh) - g.myl;
    if (u0 <= 0.f && u1 >= 0.f && v0 <= 0.f && v1 >= 0.f) return true;
    const float b2 = -g.nb2, b = -0.5f * g.nb2;
    const float ba = __fdividef(b, g.a), bc = __fdividef(b, g.c);
    float lo = 3.0e38f;
    auto edge = [&](float u, float v) {
        float t1 = (g.a * u) * u, t3 = (g.c * v) * v;
        float qv = fmaf(b2 * u, v, t1 + t3);
        lo = fminf(lo, fmaf(-(t1 + t3), 3.8146973e-06f, qv));
    };
    // vertical edges u = u0, u1: v* = -(b/c) u clamped
    edge(u0, fminf(fmaxf(-bc * u0, v0), v1));
    edge(u1, fminf(fmaxf(-bc * u1, v0), v1));
    // horizontal edges v = v0, v1: u* = -(b/a) v clamped
    edge(fminf(fmaxf(-ba * v0, u0), u1), v0);
    edge(fminf(fmaxf(-ba * v1, u0), u1), v1);
    return !(lo > fmaf(g.cull_hi, 3.8146973e-06f, g.cull_hi));
}

}  // namespace
}  // namespace splat
