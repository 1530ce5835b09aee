// K3b / K3d: tile binning (rasterizer.py:161-191).
//
// emit:   in depth-rank order r (perm from the depth sort), every primitive writes one
//         (tile id, compact index) entry per tile of its bounds rectangle, row-major within
//         the rectangle.  The exclusive scan of per-rank tile counts that places the
//         entries is fused into the same kernel (single pass, 64-bit decoupled look-back),
//         and the total E is checked against the caller's capacity (overflow -> status
//         BSR_ERR_CAPACITY, nothing written, entries_needed reported for a retry).
// ranges: after the stable tile sort, per-tile [start, end) from key boundaries
//         (== np.bincount + cumsum offsets).
#include "frame.cuh"

namespace bsr {

constexpr uint32_t kBigRect = 64;  // rectangles with more tiles are emitted by a whole CTA
constexpr unsigned long long kFlag64Agg = 1ull << 62;
constexpr unsigned long long kFlag64Prefix = 2ull << 62;
constexpr unsigned long long kValue64Mask = (1ull << 62) - 1;

template <int kEmitItems>
__global__ void __launch_bounds__(BSR_BLOCK) emit_kernel(FrameView f) {
    constexpr int kEmitTile = BSR_BLOCK * kEmitItems;
    __shared__ uint32_t s_part;
    __shared__ unsigned long long s_warp[BSR_BLOCK / 32], s_excl;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) s_part = atomicAdd(&f.ctr->emit_ticket, 1u);
    __syncthreads();
    const uint32_t V = f.ctr->visible;
    const int64_t part = s_part;
    const int64_t base = part * kEmitTile;
    if (base >= (int64_t)V) return;
    const int64_t nparts = div_up(V, kEmitTile);
    const uint32_t *perm = f.dvals[f.ctr->depth_plan[kDepthPasses] & 1u];
    // blocked arrangement: thread t owns ranks base + t*ITEMS .. +ITEMS
    uint32_t cidx[kEmitItems], cnt[kEmitItems];
    unsigned long long tsum = 0;
#pragma unroll
    for (int i = 0; i < kEmitItems; ++i) {
        const int64_t r = base + (int64_t)t * kEmitItems + i;
        if (r < (int64_t)V) {
            cidx[i] = perm[r];
            cnt[i] = f.tile_count[cidx[i]];
        } else {
            cidx[i] = 0;
            cnt[i] = 0;
        }
        tsum += cnt[i];
    }
    // block exclusive scan of thread sums
    unsigned long long x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {  // block total -> aggregate, warp-parallel look-back -> prefix
        const unsigned long long mine = lane < BSR_BLOCK / 32 ? s_warp[lane] : 0ull;
        unsigned long long incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const unsigned long long run = __shfl_sync(0xffffffffu, incl, 31);
        if (lane < BSR_BLOCK / 32) s_warp[lane] = incl - mine;
        unsigned long long excl = 0;
        volatile unsigned long long *st = f.emit_status;
        if (part == 0) {
            if (lane == 0) {
                __threadfence();
                st[0] = kFlag64Prefix | run;
            }
        } else {
            if (lane == 0) {
                __threadfence();
                st[part] = kFlag64Agg | run;
            }
            excl = warp_lookback<unsigned long long>(f.emit_status, part, 1, kFlag64Prefix, kValue64Mask);
            if (lane == 0) {
                __threadfence();
                st[part] = kFlag64Prefix | (excl + run);
            }
        }
        if (lane == 0) {
            s_excl = excl;
            if (part == nparts - 1) {
                const unsigned long long total = excl + run;
                f.ctr->entries_needed = total;
                if (total > (unsigned long long)f.entry_cap) {
                    f.ctr->entries = 0;
                    raise_status(&f.ctr->status, BSR_ERR_CAPACITY);
                } else {
                    f.ctr->entries = (uint32_t)total;
                }
            }
        }
    }
    __syncthreads();
    unsigned long long off = s_excl + s_warp[warp] + (x - tsum);
    const int tiles_x = f.tiles_x;
#pragma unroll 1
    for (int i = 0; i < kEmitItems; ++i) {
        if (cnt[i] == 0) continue;
        if (off + cnt[i] > (unsigned long long)f.entry_cap) return;  // overflow: caller retries
        if (cnt[i] > kBigRect) {  // load balance: near-plane primitives cover whole frames
            const uint32_t slot = atomicAdd(&f.ctr->big_emit, 1u);
            f.big[slot] = make_uint4(cidx[i], (uint32_t)off, (uint32_t)(off >> 32), cnt[i]);
            off += cnt[i];
            continue;
        }
        const int4 bd = f.rec[cidx[i]].d;
        const int tx0 = bd.x / BSR_TILE, tx1 = bd.y / BSR_TILE;
        const int ty0 = bd.z / BSR_TILE, ty1 = bd.w / BSR_TILE;
        uint32_t *kout = f.tkeys[0] + off;
        uint32_t *vout = f.tvals[0] + off;
        int j = 0;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx, ++j) {
                kout[j] = (uint32_t)(ty * tiles_x + tx);
                vout[j] = cidx[i];
            }
        off += cnt[i];
    }
}

// Cooperative emission of the big rectangles queued by emit_kernel: one CTA per rectangle,
// consecutive threads write consecutive (row-major) entries.
__global__ void __launch_bounds__(BSR_BLOCK) emit_big_kernel(FrameView f) {
    const uint32_t nbig = f.ctr->big_emit;
    for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {
        const uint4 it = f.big[b];
        const int4 bd = f.rec[it.x].d;
        const int tx0 = bd.x / BSR_TILE, ty0 = bd.z / BSR_TILE;
        const uint32_t spanx = (uint32_t)(bd.y / BSR_TILE - tx0 + 1);
        const unsigned long long off = (unsigned long long)it.y | ((unsigned long long)it.z << 32);
        uint32_t *kout = f.tkeys[0] + off;
        uint32_t *vout = f.tvals[0] + off;
        for (uint32_t j = threadIdx.x; j < it.w; j += BSR_BLOCK) {
            const uint32_t ty = ty0 + j / spanx, tx = tx0 + j % spanx;
            kout[j] = ty * (uint32_t)f.tiles_x + tx;
            vout[j] = it.x;
        }
    }
}

__global__ void tile_ranges_kernel(FrameView f) {
    const uint32_t E = f.ctr->entries;
    const uint32_t sel = f.ctr->tile_plan[f.tile_passes] & 1u;
    const uint32_t *keys = f.tkeys[sel];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        if (i == 0 || keys[i - 1] != k) f.tile_ranges[k].x = i;
        if (i == E - 1 || keys[i + 1] != k) f.tile_ranges[k].y = i + 1;
    }
}

int launch_emit(const FrameView &f, cudaStream_t st) {
    if (f.n == 0) return BSR_OK;
    if (f.depth_items == 4)
        emit_kernel<4><<<(unsigned)div_up(f.n, BSR_BLOCK * 4), BSR_BLOCK, 0, st>>>(f);
    else
        emit_kernel<16><<<(unsigned)div_up(f.n, BSR_BLOCK * 16), BSR_BLOCK, 0, st>>>(f);
    emit_big_kernel<<<148 * 4, BSR_BLOCK, 0, st>>>(f);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

int launch_tile_ranges(const FrameView &f, cudaStream_t st) {
    if (f.entry_cap == 0) return BSR_OK;
    const unsigned blocks = (unsigned)imin64(div_up(f.entry_cap, BSR_BLOCK), 148 * 16);
    tile_ranges_kernel<<<blocks, BSR_BLOCK, 0, st>>>(f);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
