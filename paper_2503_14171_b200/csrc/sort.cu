// Device primitives for tile binning: exclusive scan and a stable LSD radix
// sort of (key, value) pairs.  Hand-written for sm_100a (no CUB): the binning
// pass only needs the tile-id bits sorted, because pairs are emitted in rank
// order and the sort is stable (raster_forward.py:136-149 appends ranks to each
// tile list in ascending order).
#include "kernels.cuh"

namespace splat {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;                       // per thread
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096 per block

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread (1024 threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = warp_incl_scan(v, lane);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = s_warp[lane];
        uint32_t wi = warp_incl_scan(w, lane);
        s_warp[lane] = wi - w;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    uint32_t r = s_warp[warp] + inc - v;
    *total = s_warp[32];
    return r;
}

__global__ void scan_reduce_kernel(const uint32_t* __restrict__ in, int64_t n,
                                   uint32_t* __restrict__ partials) {
    __shared__ uint32_t s_warp[33];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) s += in[base + i];
    uint32_t total;
    block_excl_scan(s, s_warp, &total);
    if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

// Single block: exclusive scan of the per-block partials in place.
__global__ void scan_partials_kernel(uint32_t* partials, int64_t nparts) {
    __shared__ uint32_t s_warp[33];
    uint32_t carry = 0;
    for (int64_t base = 0; base < nparts; base += kScanThreads) {
        int64_t i = base + threadIdx.x;
        uint32_t v = i < nparts ? partials[i] : 0;
        uint32_t total;
        uint32_t e = block_excl_scan(v, s_warp, &total);
        if (i < nparts) partials[i] = carry + e;
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[nparts] = carry;
}

__global__ void scan_down_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                 int64_t n, const uint32_t* __restrict__ partials, int64_t nparts,
                                 uint32_t* total_out) {
    __shared__ uint32_t s_warp[33];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    uint32_t total;
    uint32_t e = block_excl_scan(s, s_warp, &total) + partials[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = e;
        e += v[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        out[n] = partials[nparts];
        if (total_out) *total_out = partials[nparts];
    }
}

// ---------------------------------------------------------------------------
// Radix sort.  8-bit digits; each CTA owns kSortTile consecutive items and
// processes them in rounds of 256 (one per thread) so the scatter is stable:
// intra-warp rank from __match_any_sync, inter-warp prefix per digit in smem,
// inter-block offsets from a digit-major exclusive scan of block histograms.

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;
constexpr int kSortTile = kSortThreads * kSortRounds;  // 4096

__device__ __forceinline__ uint32_t sort_count(const uint32_t* n_dev, int64_t n_host, int64_t cap) {
    int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    return (uint32_t)(n < cap ? n : cap);
}

// BITS-wide digits: 8 for multi-pass sorts (64-bit depth keys, >11-bit tile ids),
// up to 11 so a 2040-tile (960x540) frame's tile ids sort in ONE pass.
template <typename K, int BITS>
__global__ void __launch_bounds__(kSortThreads)
radix_upsweep_kernel(const K* __restrict__ keys, const uint32_t* n_dev, int64_t n_host, int64_t cap,
                     int shift, uint32_t* __restrict__ hist, int nblocks) {
    constexpr int D = 1 << BITS;
    constexpr uint32_t M = D - 1;
    __shared__ uint32_t h[D];
    for (int d = threadIdx.x; d < D; d += kSortThreads) h[d] = 0;
    __syncthreads();
    uint32_t n = sort_count(n_dev, n_host, cap);
    int64_t base = (int64_t)blockIdx.x * kSortTile;
    if (base < n) {
        for (int r = 0; r < kSortRounds; ++r) {
            int64_t i = base + r * kSortThreads + threadIdx.x;
            if (i < n) atomicAdd(&h[(uint32_t)(keys[i] >> shift) & M], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += kSortThreads) hist[(int64_t)d * nblocks + blockIdx.x] = h[d];
}

// Downsweep: warp w of the CTA owns the contiguous sub-chunk
// [base + w*32*R, base + (w+1)*32*R) and keeps its R items per lane in
// registers.  Pass 1 counts digits per warp (one __match_any_sync per item,
// the group leader accumulates into the warp's counters).  The CTA then
// derives each item's position in the block-locally sorted order (digit-major,
// stable) and its digit's global base.  Pass 2 writes items to shared memory at
// their local position; finally the CTA streams shared memory out, so each
// digit run is written to global memory with consecutive stores.
template <typename K, int BITS>
__global__ void __launch_bounds__(kSortThreads)
radix_downsweep_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                       K* __restrict__ kout, uint32_t* __restrict__ vout,
                       const uint32_t* n_dev, int64_t n_host, int64_t cap, int shift,
                       const uint32_t* __restrict__ hist, int nblocks) {
    constexpr int R = kSortRounds;
    constexpr int D = 1 << BITS;
    constexpr uint32_t M = D - 1;
    constexpr int G = D / kSortThreads;                                         // digits per thread
    extern __shared__ __align__(16) unsigned char sm[];
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(sm);                          // [8][D]
    uint32_t* s_gbase = s_cnt + 8 * D;                                          // [D]
    uint32_t* s_scan = s_gbase + D;                                             // [32]
    K* s_k = reinterpret_cast<K*>(sm + ((size_t)9 * D + 32) * 4);               // [kSortTile]
    uint32_t* s_v = reinterpret_cast<uint32_t*>(s_k + kSortTile);              // [kSortTile]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = sort_count(n_dev, n_host, cap);
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    if (base >= n) return;
    const int nblk = (int)min((int64_t)kSortTile, (int64_t)n - base);
    const int64_t sub = base + (int64_t)warp * 32 * R;
    const uint32_t lt_mask = (1u << lane) - 1u;
    K k[R];
    uint32_t v[R], peers[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = sub + r * 32 + lane;
        const bool valid = i < n;
        k[r] = valid ? kin[i] : K(0);
        v[r] = valid ? vin[i] : 0u;
    }
    uint32_t* my_cnt = s_cnt + warp * D;
    for (int d = lane; d < D; d += 32) my_cnt[d] = 0;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const bool valid = sub + r * 32 + lane < n;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        const uint32_t d = (uint32_t)(k[r] >> shift) & M;
        peers[r] = 0;
        if (valid) {
            peers[r] = __match_any_sync(vmask, d);
            if ((peers[r] & lt_mask) == 0) my_cnt[d] += __popc(peers[r]);
        }
        __syncwarp();
    }
    __syncthreads();
    // thread t owns digits [t*G, (t+1)*G): warp prefix, block total, block-local offset
    uint32_t tot[G];
    uint32_t local = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int d = tid * G + g;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const uint32_t c = s_cnt[w * D + d];
            s_cnt[w * D + d] = run;
            run += c;
        }
        tot[g] = run;
        local += run;
    }
    uint32_t incl = local;   // exclusive scan of `local` over the 256 threads
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, dd);
        if (lane >= dd) incl += o;
    }
    if (lane == 31) s_scan[warp] = incl;
    __syncthreads();
    uint32_t loff = incl - local;
    for (int w = 0; w < warp; ++w) loff += s_scan[w];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int d = tid * G + g;
#pragma unroll
        for (int w = 0; w < 8; ++w) s_cnt[w * D + d] += loff;
        s_gbase[d] = hist[(int64_t)d * nblocks + blockIdx.x] - loff;
        loff += tot[g];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t d = (uint32_t)(k[r] >> shift) & M;
        uint32_t pos = 0;
        if (peers[r]) pos = my_cnt[d] + __popc(peers[r] & lt_mask);
        __syncwarp();
        if (peers[r]) {
            if ((peers[r] & lt_mask) == 0) my_cnt[d] += __popc(peers[r]);
            s_k[pos] = k[r];
            s_v[pos] = v[r];
        }
        __syncwarp();
    }
    __syncthreads();
    for (int i = tid; i < nblk; i += kSortThreads) {
        const K kk = s_k[i];
        const uint32_t pos = s_gbase[(uint32_t)(kk >> shift) & M] + (uint32_t)i;
        kout[pos] = kk;
        vout[pos] = s_v[i];
    }
}

template <typename K, int BITS>
constexpr size_t downsweep_smem() {
    return ((size_t)9 * (1 << BITS) + 32) * 4 + (size_t)kSortTile * (sizeof(K) + 4);
}

}  // namespace

int64_t scan_scratch_words(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* scratch,
                       uint32_t* total_out, cudaStream_t stream) {
    int64_t nparts = (n + kScanTile - 1) / kScanTile;
    if (nparts == 0) nparts = 1;
    scan_reduce_kernel<<<(unsigned)nparts, kScanThreads, 0, stream>>>(in, n, scratch); note_launch();
    scan_partials_kernel<<<1, kScanThreads, 0, stream>>>(scratch, nparts); note_launch();
    scan_down_kernel<<<(unsigned)nparts, kScanThreads, 0, stream>>>(in, out, n, scratch, nparts,
                                                                     total_out); note_launch();
    return SPLAT_OK;
}

int64_t radix_blocks(int64_t cap) { return (cap + kSortTile - 1) / kSortTile; }

constexpr int kMaxDigits = 2048;   // widest single pass (11 bits)

int64_t radix_scratch_words(int64_t cap) {
    int64_t nb = radix_blocks(cap);
    if (nb == 0) nb = 1;
    return kMaxDigits * nb + 1 + scan_scratch_words(kMaxDigits * nb + 1);
}

int radix_passes(int bits) { return bits <= 0 ? 0 : (bits <= 11 ? 1 : (bits + 7) / 8); }

template <typename K, int BITS>
static int radix_pass(const K* src_k, const uint32_t* src_v, K* dst_k, uint32_t* dst_v, const uint32_t* n_dev,
                      int64_t n_host, int64_t cap, int shift, uint32_t* hist, uint32_t* hscan, int nb,
                      cudaStream_t stream) {
    static PerDevice<bool> configured;
    bool ok = false;
    const int rc = configured.get(ok, [](bool& v) {
        SPLAT_CUDA_CHECK(cudaFuncSetAttribute(radix_downsweep_kernel<K, BITS>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)downsweep_smem<K, BITS>()));
        v = true;
        return SPLAT_OK;
    });
    if (rc != SPLAT_OK) return rc;
    radix_upsweep_kernel<K, BITS><<<nb, kSortThreads, 0, stream>>>(src_k, n_dev, n_host, cap, shift, hist, nb); note_launch();
    exclusive_scan_u32(hist, hist, (int64_t)(1 << BITS) * nb, hscan, nullptr, stream);
    radix_downsweep_kernel<K, BITS><<<nb, kSortThreads, downsweep_smem<K, BITS>(), stream>>>(
        src_k, src_v, dst_k, dst_v, n_dev, n_host, cap, shift, hist, nb); note_launch();
    return SPLAT_OK;
}

// Stable LSD sort of (key, value) on key bits [begin_bit, end_bit): one 11-bit
// pass when the range fits (tile ids of frames up to 2048 tiles), else 8-bit passes.
template <typename K>
int radix_sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                     int64_t n_host, int64_t cap, int begin_bit, int end_bit, uint32_t* scratch,
                     int* result_in_alt, cudaStream_t stream) {
    int nb = (int)radix_blocks(cap);
    if (nb == 0) nb = 1;
    uint32_t* hist = scratch;
    uint32_t* hscan = scratch + (int64_t)kMaxDigits * nb + 1;
    K* src_k = keys;
    uint32_t* src_v = vals;
    K* dst_k = keys_alt;
    uint32_t* dst_v = vals_alt;
    int alt = 0;
    const int bits = end_bit - begin_bit;
    int rc;
    if (radix_passes(bits) == 1 && bits > 8) {
        if ((rc = radix_pass<K, 11>(src_k, src_v, dst_k, dst_v, n_dev, n_host, cap, begin_bit, hist, hscan, nb,
                                    stream)))
            return rc;
        alt = 1;
    } else {
        for (int shift = begin_bit; shift < end_bit; shift += 8) {
            if ((rc = radix_pass<K, 8>(src_k, src_v, dst_k, dst_v, n_dev, n_host, cap, shift, hist, hscan, nb,
                                       stream)))
                return rc;
            K* tk = src_k; src_k = dst_k; dst_k = tk;
            uint32_t* tv = src_v; src_v = dst_v; dst_v = tv;
            alt ^= 1;
        }
    }
    *result_in_alt = alt;
    return SPLAT_OK;
}

template int radix_sort_pairs<uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, const uint32_t*,
                                        int64_t, int64_t, int, int, uint32_t*, int*, cudaStream_t);
template int radix_sort_pairs<uint64_t>(uint64_t*, uint32_t*, uint64_t*, uint32_t*, const uint32_t*,
                                        int64_t, int64_t, int, int, uint32_t*, int*, cudaStream_t);

}  // namespace splat
