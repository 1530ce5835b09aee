// Frame = caller-provided device buffer holding the saved forward state and the scratch
// of one render.  Layout is a pure function of (n, W, H, entry_cap) so forward and
// backward carve identical views.
#pragma once

#include "common.cuh"

namespace bsr {

// Keys per thread in a sort / emit partition: 16 (4096 per CTA) for large inputs, 4 (1024
// per CTA) while the input would give fewer than ~2 CTAs per SM at 16.
constexpr int64_t kSmallSortCap = 148 * 2 * 4096;
inline int sort_items(int64_t cap) { return cap <= kSmallSortCap ? 4 : 16; }
constexpr int kDepthPasses = 4;                      // 32-bit (fp32-depth) keys + fp64 fixup
constexpr int kRec64 = 8;                            // doubles per fp64 side record
constexpr int kGradStride = 12;                      // raster grad accumulator floats/primitive
constexpr int kSide64 = 6;                           // fp64 side doubles per primitive (FrameView::side64)
// primitives whose fp32 r2 error bound exceeds this are evaluated in fp64 by the raster
#ifndef BSR_UNSAFE_R2_ERR
#define BSR_UNSAFE_R2_ERR 2.0e-5f
#endif
constexpr float kUnsafeR2Err = BSR_UNSAFE_R2_ERR;

struct Counters {
    uint32_t visible;        // V
    uint32_t entries;        // E (0 on overflow)
    unsigned long long entries_needed;
    uint32_t flagged;        // flagged pixels
    int32_t status;          // first device-side error
    uint32_t depth_ticket[kDepthPasses];   // global depth sort (parity export only)
    uint32_t depth_key_max_inv;  // max(~key) == ~min(key) over the 32-bit depth keys
    uint32_t depth_plan[kDepthPasses + 1];
    uint32_t big_tiles;      // crowded tiles queued by tile_sort for tile_sort_big (ids in tile_cur)
    uint32_t mid_tiles;      // tiles queued by tile_sort for tile_sort_mid (ids in tile_cnt)
    uint32_t pad[3];
};

// Deterministic accumulation of the backward's per-primitive partials
// (bsr_backward_deterministic): float atomics land in a run-dependent order and their sums
// differ in the last bits, so in this mode every value is added as a 64-bit fixed-point
// integer (integer addition is associative: the sum does not depend on the order).  Pass 1
// (mode 1) records per primitive and slot the largest magnitude that will be added
// (atomicMax on the float bits, itself order-independent); pass 2 (mode 2) recomputes the
// same values and adds round(v * 2^(38 - e)), e = exponent of that bound, so every term is
// below 2^39 in magnitude and up to 2^24 terms fit in 63 bits with a resolution of
// bound * 2^-39; a finalize kernel converts the sums back (det_finalize in api.cu).
constexpr int kDetSlots = 12;  // grad_acc's 11 slots (fp64-path xy partials reuse 0..4)
struct DetAcc {
    int mode;                  // 0: off (float / fp64 atomics), 1: bound pass, 2: fixed-point pass
    uint32_t *bound;           // [N][kDetSlots] float bits of max |value|
    unsigned long long *acc;   // [N][kDetSlots] fixed-point sums (two's complement)
};

__device__ __forceinline__ int det_exp(uint32_t bound_bits) { return (int)((bound_bits >> 23) & 0xff) - 127; }

__device__ __forceinline__ void det_add(const DetAcc &d, uint32_t c, int slot, double v) {
    const int64_t k = (int64_t)kDetSlots * c + slot;
    if (d.mode == 1) {
        const float av = fabsf((float)v);
        if (av > 0.f) atomicMax(d.bound + k, __float_as_uint(av));
    } else if (v != 0.0) {
        const long long qv = __double2ll_rn(ldexp(v, 38 - det_exp(d.bound[k])));
        atomicAdd(d.acc + k, (unsigned long long)qv);
    }
}

struct FrameView {
    // --- zeroed every forward (one memset) ---
    Counters *ctr;
    uint2 *tile_ranges;      // [n_tiles] (start, end)
    uint32_t *tile_cnt;      // [n_tiles << cnt_shift] entries per tile (tile_cnt_at)
    uint32_t *tile_cur;      // [n_tiles << cnt_shift] scatter cursors (tile_cur_at)
    uint32_t *tile_order;    // [n_tiles] tiles by decreasing entry count (log2 buckets; bin_scan):
                             // the raster kernels' CTA -> tile map, heavy tiles first
    // --- not zeroed ---
    uint32_t *depth_hist;    // [4][256]                  global depth sort: parity export only,
    uint32_t *depth_status;  // [4][ceil(N/4096)][256]     zeroed by bsr_debug_export
    Record *rec;             // [N] by source index (valid where tile_count > 0)
    double *rec64;           // [N][8] fp64 {mean x, y, conic a, b, c, opacity, beta, depth}:
                             // the fp64 replay's geometry and the raster's path for fp32-unsafe
                             // primitives (Record.c.w < 0)
    uint32_t *dkeys[2];      // [N] fp32-depth keys by source index ([1]: parity-export sort)
    uint64_t *dkey64;        // [N] fp64 depth bits by source index (tie fixup)
    uint32_t *dvals[2];      // [N] parity-export depth sort values (ping-pong)
    uint32_t *tile_count;    // [N] tiles touched by source index, 0 = culled
    uint64_t *tent;          // [Ecap] (fp32 depth key << 32 | source index), scattered per tile
    uint32_t *lists;         // [Ecap] source index per tile entry in depth order (tile_ranges)
    uint32_t *emask;         // [Ecap] sub-block occupancy mask of every tile entry the forward raster
                             // reached (raster.cuh entry_tile_mask), reused by the backward
    uint32_t *mask_end;      // [n_tiles] emask holds the tile's entries [range.x, mask_end) (the
                             // batches the forward raster processed before its pixels finished)
    float *t_final;          // [H*W]
    uint32_t *last;          // [H*W] local end index of last contributor (0: none / flagged)
    uint2 *flags;            // [H*W] (pixel, local entry index where fp32 became ambiguous)
    double *replay_state;    // [H*W][6] by flag slot: raw(3), raw_depth, T, last  (fp64, flagged only)
    double *split_state;     // [H*W][6] by flag slot, at the split point: T, prefix colour(3) + depth
    float4 *bwd_init;        // [H*W] flagged pixels: the raster backward's starting "behind" state
                             // (colour(3), depth) at the flag point, t_final holds -T there
    float4 *needle;          // [N] needle words of records with c.w < 0 (raster.cuh), NaN: fp64 path
    uint32_t *vis_hint;      // visible count of the previous forward on this frame (a
                             // scheduling hint for preprocess only: any value is safe)
    float *grad_acc;         // [N][12] raster gradient accumulators by source index (zeroed by backward):
                             // [0..4] geometry partials in the record's whitened frame (u, w) =
                             // L^T (px - mean), Q = L L^T:  sum d_x (u, w, u^2, u w, w^2)
                             // (d_x = dL/dr2), [5] d opacity, [6] d beta, [7..9] d rgb, [10] d z
    double *side64;          // [N][kSide64] fp64 side data of fp32-unsafe records (Record.c.w < 0) that
                             // take the fp64 path (needle word .x NaN): with a positive-definite
                             // conic (needle word .y == 1) [0..2] = its fp64 factor (l11, l21,
                             // l22); without one (.y == 0) [0..4] = xy-frame geometry partials
                             // summed in fp64 (add_geom64; zeroed by preprocess, re-zeroed when
                             // preprocess_bwd consumes them)
    DetAcc det;              // deterministic-backward workspace (mode 0 outside bsr_backward_deterministic)
    // --- sizes ---
    int64_t n, entry_cap;
    int W, H, tiles_x, tiles_y, n_tiles;
    int cnt_shift;  // log2 of the word stride of tile_cnt / tile_cur (tile_cnt_at)
    int64_t depth_parts;
    int depth_items;  // sort_items() of the (parity-export) depth sort
    uint64_t zero_bytes, total_bytes;
};

// Per-tile counters (hot REDs / atomics), 2^cnt_shift words apart.
__host__ __device__ __forceinline__ uint32_t *tile_cnt_at(const FrameView &f, uint32_t t) {
    return f.tile_cnt + ((size_t)t << f.cnt_shift);
}
__host__ __device__ __forceinline__ uint32_t *tile_cur_at(const FrameView &f, uint32_t t) {
    return f.tile_cur + ((size_t)t << f.cnt_shift);
}

// Carve the frame.  base == nullptr computes sizes only.
inline FrameView carve_frame(void *base, int64_t n, int W, int H, int64_t entry_cap) {
    FrameView f;
    f.n = n;
    f.entry_cap = entry_cap;
    f.det.mode = 0;
    f.det.bound = nullptr;
    f.det.acc = nullptr;
    f.W = W;
    f.H = H;
    f.tiles_x = (W + BSR_TILE - 1) / BSR_TILE;
    f.tiles_y = (H + BSR_TILE - 1) / BSR_TILE;
    f.n_tiles = f.tiles_x * f.tiles_y;
    f.depth_items = sort_items(n);
    f.depth_parts = div_up(n > 0 ? n : 1, (int64_t)BSR_BLOCK * f.depth_items);
    const int64_t npx = (int64_t)W * H;
    uint64_t off = 0;
    char *b = static_cast<char *>(base);
    auto take = [&](uint64_t bytes) -> void * {
        off = align_up(off, 256);
        void *p = b ? b + off : nullptr;
        off += bytes;
        return p;
    };
    f.ctr = (Counters *)take(sizeof(Counters));
    f.tile_ranges = (uint2 *)take(8ull * f.n_tiles);
    // small frames spread their tile counters (few tiles take millions of REDs: packed, they
    // share a few L2 lines and the RED rate depends on how those lines hash to L2 slices)
    // (bin_scan keeps spread counters in shared memory: at most 8192 tiles)
    f.cnt_shift = f.n_tiles <= 4096 ? 5 : (f.n_tiles <= 8192 ? 3 : 0);
    f.tile_cnt = (uint32_t *)take(4ull * f.n_tiles << f.cnt_shift);
    f.tile_cur = (uint32_t *)take(4ull * f.n_tiles << f.cnt_shift);
    f.tile_order = (uint32_t *)take(4ull * f.n_tiles);
    off = align_up(off, 256);
    f.zero_bytes = off;
    f.vis_hint = (uint32_t *)take(4);
    f.depth_hist = (uint32_t *)take(4ull * kDepthPasses * 256);
    f.depth_status = (uint32_t *)take(4ull * kDepthPasses * f.depth_parts * 256);
    f.rec = (Record *)take(sizeof(Record) * (uint64_t)n);
    f.rec64 = (double *)take(8ull * kRec64 * n);
    f.dkeys[0] = (uint32_t *)take(4ull * n);
    f.dkeys[1] = (uint32_t *)take(4ull * n);
    f.dkey64 = (uint64_t *)take(8ull * n);
    f.dvals[0] = (uint32_t *)take(4ull * n);
    f.dvals[1] = (uint32_t *)take(4ull * n);
    f.tile_count = (uint32_t *)take(4ull * n);
    f.tent = (uint64_t *)take(8ull * entry_cap);
    f.lists = (uint32_t *)take(4ull * entry_cap);
    f.emask = (uint32_t *)take(4ull * entry_cap);
    f.t_final = (float *)take(4ull * npx);
    f.last = (uint32_t *)take(4ull * npx);
    f.flags = (uint2 *)take(8ull * npx);
    f.replay_state = (double *)take(8ull * 6 * npx);
    f.grad_acc = (float *)take(4ull * kGradStride * n);
    f.needle = (float4 *)take(16ull * n);
    f.side64 = (double *)take(8ull * kSide64 * n);
    f.mask_end = (uint32_t *)take(4ull * f.n_tiles);
    f.split_state = (double *)take(8ull * 6 * npx);
    f.bwd_init = (float4 *)take(16ull * npx);
    f.total_bytes = align_up(off, 256);
    return f;
}

// xy-frame geometry partials summed in fp64 (raster_bwd / replay_bwd) for the records that
// have no usable factor (fp64-path records whose conic is not positive definite in fp64):
// without a whitened frame their conic gradient's short-axis part is a cancellation of
// large xy terms, so it is formed from the fp64 mean / conic and summed in fp64.
__device__ __forceinline__ void add_geom64(const FrameView &f, uint32_t c, double d_x, double dx, double dy,
                                           double ca, double cb, double cc) {
    const double ga = ca * dx + cb * dy, gb = cb * dx + cc * dy;
    const double v[5] = {-2.0 * d_x * ga, -2.0 * d_x * gb, d_x * dx * dx, 2.0 * d_x * dx * dy, d_x * dy * dy};
    if (f.det.mode) {
        for (int q = 0; q < 5; ++q) det_add(f.det, c, q, v[q]);
        return;
    }
    double *g = f.side64 + (int64_t)kSide64 * c;
    for (int q = 0; q < 5; ++q) atomicAdd(g + q, v[q]);
}

}  // namespace bsr
