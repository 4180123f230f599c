// Internal launcher declarations shared by the .cu files of libsplat_b200.
#pragma once
#include "common.cuh"

namespace splat {

// sort.cu
int64_t scan_scratch_words(int64_t n);
int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* scratch,
                       uint32_t* total_out, cudaStream_t stream);
int64_t radix_blocks(int64_t cap);
int64_t radix_scratch_words(int64_t cap);
int radix_passes(int bits);
template <typename K>
int radix_sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                     int64_t n_host, int64_t cap, int begin_bit, int end_bit, uint32_t* scratch,
                     int* result_in_alt, cudaStream_t stream);

// Frame workspace layout (all offsets 256-byte aligned).
struct FrameLayout {
    size_t bboxes, touched, offsets, scan_scratch, keys0, vals0, vals1, slot_pos, tile_scan,
        ranges, tile_count, tile_start, cursor, big_list, bin_hist, bin_pre, bin_part, counters, fixup, pack, rmask, bwd_hi, bwd_cursor, total;
    int64_t n, cap;
    int width, height, ntx, nty;
};
FrameLayout frame_layout(int64_t n, int width, int height, int64_t cap);

// Tail padding of the per-pair arrays (ranks, rect masks): the rasterizer streams them
// in 128-pair batches aligned down to 16 pairs, so a batch may read up to this many
// entries past the last pair.
constexpr int kPairPad = 160;

// The rasterizer's 8x4-pixel rectangles of a 16x16 tile: rectangle (col, row), col 0..1,
// row 0..3, is bit 2 row + col.  Bit set when the pair's bbox [x0, x1) x [y0, y1) overlaps
// the rectangle's pixels: the reference tests each pixel against the bbox
// (_kernels.py:61-64), so a rectangle whose bit is clear never sees the candidate.
__device__ __forceinline__ uint32_t rect_mask(short4 bb, int tx, int ty) {
    const int px0 = tx * kTile, py0 = ty * kTile;
    uint32_t cols = 0, m = 0;
#pragma unroll
    for (int c = 0; c < 2; ++c)
        if (bb.x < px0 + 8 * c + 8 && bb.y > px0 + 8 * c) cols |= 1u << c;
#pragma unroll
    for (int r = 0; r < 4; ++r)
        if (bb.z < py0 + 4 * r + 4 && bb.w > py0 + 4 * r) m |= cols << (2 * r);
    return m;
}

// Scene-constant layout inside const_buf.
struct ConstLayout {
    size_t order, rank_of, mean, n00, n01, n11, e1e2, sigma, q, color, total;
};
ConstLayout const_layout(int64_t n);
SceneConst scene_const_view(const void* buf, int64_t n);

// Per-view scalar constants, all computed on the host with the reference's
// float64 expression trees (raster_forward.py:81-85, 99-101, 108).
struct ViewConst {
    double kx, ky, ox, oy;
    double c00, c01, c11, cdet;  // 2kx*kx, 2kx*ky, 2ky*ky, 4kx*kx*ky*ky
    float bg[3];
};
ViewConst make_view_const(const splat_view_t& v);

int launch_preprocess(const SceneConst& sc, const ViewConst& vc, const FrameLayout& L, char* ws,
                      cudaStream_t stream);
int launch_binning(const FrameLayout& L, char* ws, int flags, cudaStream_t stream);
int launch_raster_forward(const SceneConst& sc, const ViewConst& vc, const FrameLayout& L, char* ws,
                          const splat_gimg_t& out, bool train, cudaStream_t stream, bool with_fixup = true);
int launch_fixup(const SceneConst& sc, const ViewConst& vc, const FrameLayout& L, char* ws,
                 const splat_gimg_t& out, bool train, cudaStream_t stream);

}  // namespace splat
