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
// primitives whose fp32 r2 error bound exceeds this are evaluated in fp64 by the raster
constexpr float kUnsafeR2Err = 2.0e-5f;

struct Counters {
    uint32_t visible;        // V
    uint32_t entries;        // E (0 on overflow)
    unsigned long long entries_needed;
    uint32_t flagged;        // flagged pixels
    int32_t status;          // first device-side error
    uint32_t pre_ticket;     // preprocess partition ticket
    uint32_t emit_ticket;
    uint32_t depth_ticket[kDepthPasses];
    uint32_t tile_ticket[4];
    uint32_t depth_key_max_inv;  // max(~key) == ~min(key) over the 32-bit depth keys
    uint32_t big_emit;           // primitives whose tile rectangle is emitted cooperatively
    uint32_t depth_plan[kDepthPasses + 1];
    uint32_t tile_plan[4 + 1];
    uint32_t pad[6];
};

struct FrameView {
    // --- zeroed every forward (one memset) ---
    Counters *ctr;
    uint32_t *depth_hist;    // [4][256]
    uint32_t *tile_hist;     // [4][256]
    uint32_t *pre_status;    // [ceil(N/256)]
    uint32_t *depth_status;  // [4][ceil(N/4096)][256]
    unsigned long long *emit_status;  // [ceil(N/4096)]
    uint32_t *tile_status;   // [tile_passes][ceil(Ecap/4096)][256]
    uint2 *tile_ranges;      // [n_tiles] (start, end)
    // --- not zeroed ---
    Record *rec;             // [N] compact order
    uint32_t *src_of;        // [N] compact -> source index (batch.indices)
    double *rec64;           // [N][8] fp64 {mean x, y, conic a, b, c, opacity, beta, depth}:
                             // the fp64 replay's geometry and the raster's path for fp32-unsafe
                             // primitives (Record.c.w < 0)
    uint32_t *dkeys[2];      // [N] fp32-depth keys (ping-pong)
    uint64_t *dkey64;        // [N] fp64 depth bits, compact order (tie fixup)
    uint32_t *dvals[2];      // [N] compact index (ping-pong)
    uint32_t *tile_count;    // [N] tiles touched, compact order
    uint4 *big;              // [N] (compact index, entry offset lo, hi, count) of big rects
    uint32_t *tkeys[2];      // [Ecap] tile ids (ping-pong)
    uint32_t *tvals[2];      // [Ecap] compact index (ping-pong)
    float *t_final;          // [H*W]
    uint32_t *last;          // [H*W] local end index of last contributor (0: none / flagged)
    uint2 *flags;            // [H*W] (pixel, local entry index where fp32 became ambiguous)
    double *replay_state;    // [H*W][6] raw(3), raw_depth, T, last  (fp64, flagged only)
    float *grad_acc;         // [N][12] raster gradient accumulators (zeroed by backward)
    // --- sizes ---
    int64_t n, entry_cap;
    int W, H, tiles_x, tiles_y, n_tiles, tile_passes;
    int64_t pre_parts, depth_parts, tile_parts;
    int depth_items, tile_items;  // sort_items() of the depth sort / emission and the tile sort
    uint64_t zero_bytes, total_bytes;
};

inline int tile_key_passes(int n_tiles) {
    int p = 1;
    while (p < 4 && (uint64_t)(n_tiles - 1) >= (1ull << (8 * p))) ++p;
    return p;
}

// Carve the frame.  base == nullptr computes sizes only.
inline FrameView carve_frame(void *base, int64_t n, int W, int H, int64_t entry_cap) {
    FrameView f;
    f.n = n;
    f.entry_cap = entry_cap;
    f.W = W;
    f.H = H;
    f.tiles_x = (W + BSR_TILE - 1) / BSR_TILE;
    f.tiles_y = (H + BSR_TILE - 1) / BSR_TILE;
    f.n_tiles = f.tiles_x * f.tiles_y;
    f.tile_passes = tile_key_passes(f.n_tiles);
    f.pre_parts = div_up(n > 0 ? n : 1, BSR_BLOCK);
    f.depth_items = sort_items(n);
    f.tile_items = sort_items(entry_cap);
    f.depth_parts = div_up(n > 0 ? n : 1, (int64_t)BSR_BLOCK * f.depth_items);
    f.tile_parts = div_up(entry_cap > 0 ? entry_cap : 1, (int64_t)BSR_BLOCK * f.tile_items);
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
    f.depth_hist = (uint32_t *)take(4ull * kDepthPasses * 256);
    f.tile_hist = (uint32_t *)take(4ull * 4 * 256);
    f.pre_status = (uint32_t *)take(4ull * f.pre_parts);
    f.depth_status = (uint32_t *)take(4ull * kDepthPasses * f.depth_parts * 256);
    f.emit_status = (unsigned long long *)take(8ull * f.depth_parts);
    f.tile_status = (uint32_t *)take(4ull * f.tile_passes * f.tile_parts * 256);
    f.tile_ranges = (uint2 *)take(8ull * f.n_tiles);
    off = align_up(off, 256);
    f.zero_bytes = off;
    f.rec = (Record *)take(sizeof(Record) * (uint64_t)n);
    f.src_of = (uint32_t *)take(4ull * n);
    f.rec64 = (double *)take(8ull * kRec64 * n);
    f.dkeys[0] = (uint32_t *)take(4ull * n);
    f.dkeys[1] = (uint32_t *)take(4ull * n);
    f.dkey64 = (uint64_t *)take(8ull * n);
    f.dvals[0] = (uint32_t *)take(4ull * n);
    f.dvals[1] = (uint32_t *)take(4ull * n);
    f.tile_count = (uint32_t *)take(4ull * n);
    f.big = (uint4 *)take(16ull * n);
    f.tkeys[0] = (uint32_t *)take(4ull * entry_cap);
    f.tkeys[1] = (uint32_t *)take(4ull * entry_cap);
    f.tvals[0] = (uint32_t *)take(4ull * entry_cap);
    f.tvals[1] = (uint32_t *)take(4ull * entry_cap);
    f.t_final = (float *)take(4ull * npx);
    f.last = (uint32_t *)take(4ull * npx);
    f.flags = (uint2 *)take(8ull * npx);
    f.replay_state = (double *)take(8ull * 6 * npx);
    f.grad_acc = (float *)take(4ull * kGradStride * n);
    f.total_bytes = align_up(off, 256);
    return f;
}

}  // namespace bsr
