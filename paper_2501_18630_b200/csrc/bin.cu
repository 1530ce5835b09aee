// K3: tile binning (rasterizer.py:83-85 _depth_order + :161-191 tile_bins).
//
// The reference sorts the visible primitives by depth (stable) and then stably sorts the
// (tile, depth rank) entries by tile, so each tile's list is its primitives in global
// depth order with source-index ties.  That order is a property of each tile alone, so
// the B200 path builds it per tile instead of sorting twice globally:
//
//   (counts)              every visible primitive adds one per tile of its bounds
//                         rectangle to that tile's count (RED), warp-cooperatively; done
//                         at the end of preprocess (preprocess.cu), which has the rectangle
//                         in registers (bin_entries<COUNT> is the standalone variant)
//   bin_scan              one CTA: exclusive scan of the tile counts -> tile ranges, E,
//                         capacity check (overflow -> BSR_ERR_CAPACITY, entries_needed)
//   bin_entries<SCATTER>  each entry takes a slot in its tile (atomic cursor) and writes
//                         (fp32 depth key << 32 | source index)
//   tile_sort             one CTA per tile sorts its entries ascending by that 64-bit key
//                         (bucket sort in shared memory up to kSortSmem entries, bitonic in
//                         place in global memory beyond), then re-orders runs of equal fp32 keys by
//                         (fp64 depth, source index); writes the compact indices.
//
// fp32 rounding of the depth is monotone, so (fp32 key, then fp64 depth, then compact
// index) is exactly the reference's order (source index order == source order of the
// visible primitives).  Nothing here needs a host synchronisation: counts and E live in
// device memory, grids are sized by capacity with early exits.
#include <algorithm>

#include "frame.cuh"

namespace bsr {

constexpr uint32_t kBigRect = 512;   // rectangles with more tiles are binned by a whole CTA
constexpr int kSortSmem = 4096;      // entries sorted in shared memory (32 KB of u64)

struct RectInfo {
    int tx0, ty0, spanx;
};

__device__ __forceinline__ RectInfo rect_of(const FrameView &f, uint32_t c) {
    const int4 bd = f.rec[c].d;
    RectInfo r;
    r.tx0 = bd.x / BSR_TILE;
    r.ty0 = bd.z / BSR_TILE;
    r.spanx = bd.y / BSR_TILE - r.tx0 + 1;
    return r;
}

__device__ __forceinline__ bool over_capacity(const FrameView &f) {
    return f.ctr->entries_needed > (unsigned long long)f.entry_cap;
}

// Warp-cooperative binning of compact primitives [32 w, 32 w + 32): lane l owns primitive
// 32 w + l; the warp's entries (inclusive prefix `incl` over the lanes) are taken
// round-robin by the lanes, each finding its entry's owner by a 5-step search over the
// prefix.  COUNT: tile_cnt[t] += 1.  Otherwise: slot = tile_cur[t]++, write the entry.
//
// Rectangles of more than kBigRect tiles (near-plane primitives can cover whole frames) are
// queued in shared memory and binned by the whole CTA after its warps are done (a warp takes
// its own when the CTA's queue is full).
constexpr int kBigQueue = 64;

template <bool COUNT>
__device__ __forceinline__ void bin_one(const FrameView &f, uint32_t t, uint64_t key) {
    if (COUNT) {
        atomicAdd(tile_cnt_at(f, t), 1u);
    } else {
        const uint32_t slot = atomicAdd(tile_cur_at(f, t), 1u);
        f.tent[f.tile_ranges[t].x + slot] = key;
    }
}

// Scatter of up to U entries per thread with every cursor atomic in flight before the first
// store (the store needs the atomic's returned slot: one at a time, each warp would wait a
// full L2 round trip per entry).
template <int U>
__device__ __forceinline__ void scatter_u(const FrameView &f, const uint32_t (&t)[U], const bool (&ok)[U],
                                          const uint64_t (&key)[U]) {
    uint32_t slot[U], at[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (ok[u]) slot[u] = atomicAdd(tile_cur_at(f, t[u]), 1u);
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (ok[u]) at[u] = f.tile_ranges[t[u]].x;
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (ok[u]) f.tent[at[u] + slot[u]] = key[u];
}
#ifndef BSR_SCATTER_U
#define BSR_SCATTER_U 4
#endif
constexpr int kScatterU = BSR_SCATTER_U;

template <bool COUNT>
__device__ __forceinline__ void bin_rect(const FrameView &f, uint32_t c, uint32_t cnt, uint32_t j0, uint32_t step) {
    const RectInfo r = rect_of(f, c);
    const uint64_t key = COUNT ? 0ull : (((uint64_t)f.dkeys[0][c] << 32) | c);
    auto tile_of = [&](uint32_t j) {
        const uint32_t row = j / (uint32_t)r.spanx;
        return (uint32_t)(r.ty0 + (int)row) * (uint32_t)f.tiles_x + (uint32_t)(r.tx0 + (int)(j - row * r.spanx));
    };
    if (COUNT) {
        for (uint32_t j = j0; j < cnt; j += step) bin_one<true>(f, tile_of(j), key);
        return;
    }
    for (uint32_t j = j0; j < cnt; j += kScatterU * step) {
        uint32_t t[kScatterU];
        bool ok[kScatterU];
        uint64_t k[kScatterU];
#pragma unroll
        for (int u = 0; u < kScatterU; ++u) {
            const uint32_t ju = j + u * step;
            ok[u] = ju < cnt;
            t[u] = ok[u] ? tile_of(ju) : 0u;
            k[u] = key;
        }
        scatter_u<kScatterU>(f, t, ok, k);
    }
}

template <bool COUNT>
__global__ void __launch_bounds__(BSR_BLOCK) bin_entries_kernel(FrameView f) {
    pdl_wait();
    __shared__ uint2 s_big[kBigQueue];
    __shared__ int s_nbig;
    const uint32_t V = (uint32_t)f.n;  // every primitive; culled ones have tile_count 0
    if (!COUNT && over_capacity(f)) return;
    if (threadIdx.x == 0) s_nbig = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (BSR_BLOCK / 32);
    for (int64_t w = (blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x) >> 5; w * 32 < (int64_t)V; w += nwarps) {
        const uint32_t c = (uint32_t)(w * 32 + lane);
        uint32_t cnt = 0;
        RectInfo r{0, 0, 1};
        uint64_t key = 0;
        uint32_t own_big = 0;  // big rectangle this lane could not queue
        if (c < V) {
            cnt = f.tile_count[c];
            if (cnt > kBigRect) {  // the whole CTA takes it after the warp loop
                const int slot = atomicAdd(&s_nbig, 1);
                if (slot < kBigQueue) s_big[slot] = make_uint2(c, cnt);
                else own_big = cnt;
                cnt = 0;
            } else if (cnt) {
                r = rect_of(f, c);
                if (!COUNT) key = ((uint64_t)f.dkeys[0][c] << 32) | c;
            }
        }
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        // entry e of the warp: its owner lane (number of lanes whose inclusive prefix is <= e)
        // and tile
        auto entry = [&](uint32_t e, uint32_t &t, uint64_t &okey) {
            int lo = 0;
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, lo + s - 1);
                if (v <= e) lo += s;
            }
            const int owner = min(lo, 31);
            const uint32_t oin = __shfl_sync(0xffffffffu, incl, owner);
            const uint32_t ocnt = __shfl_sync(0xffffffffu, cnt, owner);
            const int tx0 = __shfl_sync(0xffffffffu, r.tx0, owner);
            const int ty0 = __shfl_sync(0xffffffffu, r.ty0, owner);
            const int spanx = __shfl_sync(0xffffffffu, r.spanx, owner);
            okey = __shfl_sync(0xffffffffu, key, owner);
            const uint32_t local = e - (oin - ocnt);
            const uint32_t row = local / (uint32_t)spanx;
            t = (uint32_t)(ty0 + (int)row) * (uint32_t)f.tiles_x + (uint32_t)(tx0 + (int)(local - row * spanx));
        };
        if (COUNT) {
            for (uint32_t base = 0; base < total; base += 32) {
                uint32_t t;
                uint64_t okey;
                entry(base + lane, t, okey);
                if (base + lane < total) bin_one<true>(f, t, okey);
            }
        } else {
            for (uint32_t base = 0; base < total; base += 32 * kScatterU) {
                uint32_t t[kScatterU];
                bool ok[kScatterU];
                uint64_t k[kScatterU];
#pragma unroll
                for (int u = 0; u < kScatterU; ++u) {
                    const uint32_t e = base + 32 * u + lane;
                    entry(e, t[u], k[u]);
                    ok[u] = e < total;
                }
                scatter_u<kScatterU>(f, t, ok, k);
            }
        }
        // queue overflow: the warp bins those rectangles itself
        unsigned ob = __ballot_sync(0xffffffffu, own_big != 0);
        while (ob) {
            const int src = __ffs(ob) - 1;
            ob &= ob - 1;
            const uint32_t bc = __shfl_sync(0xffffffffu, c, src), bn = __shfl_sync(0xffffffffu, own_big, src);
            bin_rect<COUNT>(f, bc, bn, lane, 32);
        }
    }
    __syncthreads();
    const int nbig = min(s_nbig, kBigQueue);
    for (int b = 0; b < nbig; ++b) bin_rect<COUNT>(f, s_big[b].x, s_big[b].y, threadIdx.x, BSR_BLOCK);
}

// One CTA of 1024 threads: tile ranges from the counts (== np.bincount + cumsum offsets).
// The counts stream through in chunks of 4096 (one uint4 per thread, coalesced), each
// chunk is block-scanned (warp shuffles + one word per warp in shared memory) and its
// ranges written back coalesced; a running total carries across chunks.
constexpr int kScanThreads = 1024, kScanChunk = 4 * kScanThreads, kScanSmemTiles = 8192;
__global__ void __launch_bounds__(kScanThreads) bin_scan_kernel(FrameView f) {
    pdl_wait();
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_total, s_chunk;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int T = f.n_tiles;
    const bool vec = (T & 3) == 0;  // uint4 / 2 x uint4 accesses stay aligned
    // spread counters (small frames, FrameView::cnt_shift): read once, kept in shared memory
    __shared__ uint32_t s_cnt[kScanSmemTiles];
    const bool cached = f.cnt_shift > 0;  // implies T <= kScanSmemTiles
    auto count = [&](int i) { return cached ? s_cnt[i] : *tile_cnt_at(f, i); };
    // pass 1: the total (capacity check before any range is written), 64-bit
    unsigned long long mine = 0;
    for (int i = 4 * t; i < T; i += kScanChunk)
        for (int k = 0; k < 4; ++k) {
            const uint32_t c = i + k < T ? *tile_cnt_at(f, i + k) : 0u;
            if (cached && i + k < T) s_cnt[i + k] = c;
            mine += c;
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) s_w[warp] = mine;
    __syncthreads();
    if (warp == 0) {
        unsigned long long x = s_w[lane];
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) {
            s_total = x;
            *f.vis_hint = f.ctr->visible;  // preprocess of the next forward reads it
            f.ctr->entries_needed = x;
            if (x > (unsigned long long)f.entry_cap) {
                f.ctr->entries = 0;
                raise_status(&f.ctr->status, BSR_ERR_CAPACITY);
            } else {
                f.ctr->entries = (uint32_t)x;
            }
        }
    }
    __syncthreads();
    const bool over = s_total > (unsigned long long)f.entry_cap;  // every tile empty: the caller retries larger
    // pass 2: exclusive scan chunk by chunk (E <= entry_cap < 2^31 when not over)
    unsigned long long carry = 0;
    for (int base = 0; base < T; base += kScanChunk) {
        const int i = base + 4 * t;
        uint32_t c[4];
        if (f.cnt_shift == 0 && vec && i < T) {
            const uint4 c4 = *reinterpret_cast<const uint4 *>(f.tile_cnt + i);
            c[0] = c4.x;
            c[1] = c4.y;
            c[2] = c4.z;
            c[3] = c4.w;
        } else {
            for (int k = 0; k < 4; ++k) c[k] = i + k < T ? count(i + k) : 0u;
        }
        const uint32_t sum = c[0] + c[1] + c[2] + c[3];
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        __syncthreads();  // s_w / s_chunk of the previous chunk are consumed
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const unsigned long long v = s_w[lane];
            unsigned long long x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            s_w[lane] = x - v;  // exclusive warp offsets
            if (lane == 31) s_chunk = x;
        }
        __syncthreads();
        unsigned long long run = carry + s_w[warp] + (incl - sum);
        uint2 r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            r[k] = over ? make_uint2(0u, 0u) : make_uint2((uint32_t)run, (uint32_t)(run + c[k]));
            run += c[k];
        }
        if (vec && i < T) {
            uint4 *dst = reinterpret_cast<uint4 *>(f.tile_ranges + i);
            dst[0] = make_uint4(r[0].x, r[0].y, r[1].x, r[1].y);
            dst[1] = make_uint4(r[2].x, r[2].y, r[3].x, r[3].y);
        } else {
            for (int k = 0; k < 4; ++k)
                if (i + k < T) f.tile_ranges[i + k] = r[k];
        }
        carry += s_chunk;
    }
    // pass 3: the raster CTA -> tile map, tiles by decreasing entry count (log2 buckets, order
    // inside a bucket arbitrary: every tile is independent), so the heaviest tiles of a
    // crowded frame start first instead of forming the tail of the raster kernels
    constexpr int kOrdBuckets = 33;
    __shared__ uint32_t s_hist[kOrdBuckets], s_cur[kOrdBuckets];
    if (t < kOrdBuckets) s_hist[t] = 0u;
    __syncthreads();
    auto bucket = [&](int i) {  // 0 = heaviest
        const uint32_t c = over ? 0u : count(i);
        return c == 0u ? kOrdBuckets - 1 : __clz(c);
    };
    for (int i = t; i < T; i += kScanThreads) atomicAdd(&s_hist[bucket(i)], 1u);
    __syncthreads();
    if (t == 0) {
        uint32_t run = 0;
        for (int b = 0; b < kOrdBuckets; ++b) {
            s_cur[b] = run;
            run += s_hist[b];
        }
    }
    __syncthreads();
    for (int i = t; i < T; i += kScanThreads) f.tile_order[atomicAdd(&s_cur[bucket(i)], 1u)] = (uint32_t)i;
}

// Ascending bitonic sort of a[0, n) with virtual +inf padding to the next power of two
// N: every compare-exchange keeps the smaller value at the lower index (first stage of
// each merge compares i with its mirror, the rest are half-cleaners), so pairs whose upper
// index is >= n are skipped.  All threads of the CTA call it.
template <typename P, typename Sync>
__device__ void bitonic_sort(P a, int n, int me, int nthreads, Sync sync) {
    int N = 1;
    while (N < n) N <<= 1;
    for (int k = 2; k <= N; k <<= 1) {
        for (int i = me; i < N / 2; i += nthreads) {
            const int h = k >> 1;
            const int lo = ((i & ~(h - 1)) << 1) | (i & (h - 1)), hi = lo ^ (k - 1);
            if (hi < n) {
                const uint64_t x = a[lo], y = a[hi];
                if (y < x) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
        }
        sync();
        for (int j = k >> 2; j >= 1; j >>= 1) {
            for (int i = me; i < N / 2; i += nthreads) {
                const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;
                if (hi < n) {
                    const uint64_t x = a[lo], y = a[hi];
                    if (y < x) {
                        a[lo] = y;
                        a[hi] = x;
                    }
                }
            }
            sync();
        }
    }
}
template <typename P>
__device__ void bitonic_sort_block(P a, int n) {
    bitonic_sort(a, n, (int)threadIdx.x, (int)blockDim.x, [] { __syncthreads(); });
}
template <typename P>
__device__ void bitonic_sort_warp(P a, int n) {
    bitonic_sort(a, n, (int)(threadIdx.x & 31), 32, [] { __syncwarp(); });
}

// Runs of equal fp32 keys: re-order by (fp64 depth, source index); the thread at the
// start of each run insertion-sorts it (runs are rare and short).
template <typename P>
__device__ void fixup_ties(P a, int n, const uint64_t *dkey64) {
    for (int i = threadIdx.x; i + 1 < n; i += blockDim.x) {
        const uint32_t ki = (uint32_t)(a[i] >> 32);
        if ((uint32_t)(a[i + 1] >> 32) != ki || (i > 0 && (uint32_t)(a[i - 1] >> 32) == ki)) continue;
        int j = i + 2;
        while (j < n && (uint32_t)(a[j] >> 32) == ki) ++j;
        for (int p = i + 1; p < j; ++p) {
            const uint64_t vp = a[p];
            const uint64_t dp = dkey64[(uint32_t)vp];
            int q = p;
            while (q > i) {
                const uint64_t vq = a[q - 1];
                const uint64_t dq = dkey64[(uint32_t)vq];
                if (dq < dp || (dq == dp && (uint32_t)vq < (uint32_t)vp)) break;
                a[q] = vq;
                --q;
            }
            a[q] = vp;
        }
    }
    __syncthreads();
}

// Per-tile order by the fp32 depth key.  Equal keys are re-ordered by fixup_ties anyway,
// so the sort need not be stable: a bucket sort on the tile's key range, shared-memory
// atomics for the scatter, insertion sort inside the (tiny) buckets; buckets of more than
// kMaxBucket entries get a warp each and a bitonic network.  The buckets are equi-depth
// rather than equal-width: a coarse histogram (kCoarse bins, linear in the key) gives every
// coarse bin a share of the nb fine buckets proportional to its entries, so the dense
// depth clusters of crowded tiles are split finely instead of piling into a few big
// buckets.  Every step of the mapping is monotone in the key.
constexpr int kBuckets = 1024;
constexpr int kCoarse = 256;
constexpr int kEquiDepthMin = 1024;  // tiles with more entries get the coarse histogram
#ifndef BSR_MAX_BUCKET
#define BSR_MAX_BUCKET 16
#endif
constexpr int kMaxBucket = BSR_MAX_BUCKET;  // larger buckets: one warp each, bitonic
static_assert(kSortSmem / (kMaxBucket + 1) < 2 * kCoarse, "big-bucket list must fit in cbase / cnf");

template <int NB>
struct SortSmem {
    uint32_t start[NB + kCoarse], cur[NB + kCoarse];
    // cbase / cnf: coarse-bin fine-bucket base / count while bucketing; afterwards the
    // same words hold the list of big buckets (at most kSortSmem / (kMaxBucket + 1) < 2 kCoarse)
    uint32_t cbase[kCoarse], cnf[kCoarse];
    // the crowded-tile variant (NB = kBigBuckets) can have up to kBigSortSmem / (kMaxBucket + 1)
    // big buckets: its own list
    uint32_t bigbuf[NB >= 4096 ? 1280 : 1];
    __device__ uint32_t *bigl() { return NB >= 4096 ? bigbuf : cbase; }
    uint32_t w[BSR_BLOCK / 32];
    uint32_t kmin, kmax, big;
};

// Sort tile `tile`'s entries (n <= capacity of s) into f.lists; all threads of the CTA.
template <int NB>
__device__ void sort_tile(const FrameView &f, int tile, uint64_t *s, SortSmem<NB> &sm) {
    const uint2 rg = f.tile_ranges[tile];
    const int n = (int)(rg.y - rg.x);
    if (n == 0) return;
    const int t = threadIdx.x, lane = t & 31;
    uint64_t *g = f.tent + rg.x;
    uint32_t *out = f.lists + rg.x;
    if (n == 1) {
        if (t == 0) out[0] = (uint32_t)g[0];
        return;
    }
    // key range
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int i = t; i < n; i += BSR_BLOCK) {
        const uint32_t k = (uint32_t)(g[i] >> 32);
        kmin = min(kmin, k);
        kmax = max(kmax, k);
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (t == 0) {
        sm.kmin = 0xffffffffu;
        sm.kmax = 0u;
        sm.big = 0u;
    }
    int nb = 1;
    while (nb < n && nb < NB) nb <<= 1;
    // equal-width buckets for ordinary tiles (linear in the key); equi-depth for crowded ones
    const bool eq = n > kEquiDepthMin;
    const int nc = eq ? min(nb, kCoarse) : 1;
    if (eq)
        for (int b = t; b < nc; b += BSR_BLOCK) sm.cnf[b] = 0u;
    else
        for (int b = t; b < nb; b += BSR_BLOCK) sm.start[b] = 0u;
    __syncthreads();
    if (lane == 0) {
        atomicMin(&sm.kmin, kmin);
        atomicMax(&sm.kmax, kmax);
    }
    __syncthreads();
    kmin = sm.kmin;
    // position t = (key - kmin) * bins / span in fp32 (monotone in the key)
    const float cscale = (float)(eq ? nc : nb) / ((float)(sm.kmax - kmin) + 1.0f);
    auto cpos = [&](uint64_t e) { return (float)((uint32_t)(e >> 32) - kmin) * cscale; };
    auto cbin = [&](float tc) { return min(nc - 1, (int)tc); };
    int nf = nb;
    if (eq) {
        for (int i = t; i < n; i += BSR_BLOCK) atomicAdd(&sm.cnf[cbin(cpos(g[i]))], 1u);
        __syncthreads();
        // fine buckets per coarse bin ~ its share of the entries (>= 1), exclusive prefix -> base
        if (t < 32) {
            constexpr int kPerC = kCoarse / 32;
            uint32_t v[kPerC], tot = 0;
#pragma unroll
            for (int q = 0; q < kPerC; ++q) {
                const int c = kPerC * t + q;
                const uint32_t cnt = c < nc ? sm.cnf[c] : 0u;
                v[q] = c < nc ? max(1u, (uint32_t)(((uint64_t)cnt * (uint32_t)nb + (uint32_t)n - 1) / (uint32_t)n)) : 0u;
                tot += v[q];
            }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (t >= o) incl += y;
            }
            uint32_t run = incl - tot;
#pragma unroll
            for (int q = 0; q < kPerC; ++q) {
                const int c = kPerC * t + q;
                if (c < nc) {
                    sm.cbase[c] = run;
                    sm.cnf[c] = v[q];
                }
                run += v[q];
            }
            if (t == 31) sm.big = incl;  // total fine buckets (reset below)
        }
        __syncthreads();
        nf = (int)sm.big;
        for (int b = t; b < nf; b += BSR_BLOCK) sm.start[b] = 0u;
        __syncthreads();
        if (t == 0) sm.big = 0u;
    }
    auto bucket = [&](uint64_t e) {
        const float tc = cpos(e);
        if (!eq) return min(nb - 1, (int)tc);
        const int c = cbin(tc);
        const uint32_t k = sm.cnf[c];
        return (int)sm.cbase[c] + min((int)k - 1, (int)(fminf(tc - (float)c, 0.99999994f) * (float)k));
    };
    for (int i = t; i < n; i += BSR_BLOCK) atomicAdd(&sm.start[bucket(g[i])], 1u);
    __syncthreads();
    {
        // exclusive scan of the fine bucket counts (up to (NB + kCoarse) / 256 per thread)
        constexpr int kPer = (NB + kCoarse) / BSR_BLOCK;
        uint32_t v[kPer], tot = 0;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int b = kPer * t + q;
            v[q] = b < nf ? sm.start[b] : 0u;
            tot += v[q];
        }
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) sm.w[t >> 5] = incl;
        __syncthreads();
        uint32_t run = incl - tot;
        for (int w = 0; w < (t >> 5); ++w) run += sm.w[w];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int b = kPer * t + q;
            if (b < nf) {
                sm.start[b] = run;
                sm.cur[b] = run;
            }
            run += v[q];
        }
    }
    __syncthreads();
    for (int i = t; i < n; i += BSR_BLOCK) {
        const uint64_t e = g[i];
        s[atomicAdd(&sm.cur[bucket(e)], 1u)] = e;
    }
    __syncthreads();
    // small buckets: insertion sort by one thread; large ones (keys bunched in the tile's
    // range): queued, then a warp each runs a bitonic network on it
    for (int b = t; b < nf; b += BSR_BLOCK) {
        const int lo = (int)sm.start[b], hi = (int)sm.cur[b];
        if (hi - lo > kMaxBucket) {
            sm.bigl()[atomicAdd(&sm.big, 1u)] = (uint32_t)b;
            continue;
        }
        for (int p = lo + 1; p < hi; ++p) {
            const uint64_t x = s[p];
            int q = p;
            while (q > lo && s[q - 1] > x) {
                s[q] = s[q - 1];
                --q;
            }
            s[q] = x;
        }
    }
    __syncthreads();
    for (uint32_t k = t >> 5; k < sm.big; k += BSR_BLOCK / 32) {
        const int b = (int)sm.bigl()[k];
        const int lo = (int)sm.start[b];
        bitonic_sort_warp(s + lo, (int)sm.cur[b] - lo);
    }
    __syncthreads();
    fixup_ties(s, n, f.dkey64);
    for (int i = t; i < n; i += BSR_BLOCK) out[i] = (uint32_t)s[i];
    __syncthreads();  // s / sm are reused by the next tile of a persistent CTA
}

// one CTA per tile: up to kSortSmem entries in shared memory; crowded tiles are left to
// tile_sort_big_kernel
// one CTA per tile for tiles of up to kSortSmall entries (28 KB of shared memory: 7 CTAs per
// SM instead of 5; measured 512 / 1024 / 2048: config 4 0.510 / 0.465 / 0.454 ms);
// larger ones are queued: up to kSortSmem entries for tile_sort_mid_kernel (queue in
// tile_cnt, free after bin_scan), beyond for tile_sort_big_kernel (queue in tile_cur)
#ifndef BSR_SORT_SMALL
#define BSR_SORT_SMALL 2048
#endif
constexpr int kSortSmall = BSR_SORT_SMALL;
__global__ void __launch_bounds__(BSR_BLOCK) tile_sort_kernel(FrameView f) {
    pdl_wait();
    __shared__ uint64_t s[kSortSmall];
    __shared__ SortSmem<kBuckets> sm;
    if (over_capacity(f)) return;
    const uint2 rg = f.tile_ranges[blockIdx.x];
    const int n = (int)(rg.y - rg.x);
    if (n > kSortSmall) {
        if (threadIdx.x == 0) {
            if (n > kSortSmem) f.tile_cur[atomicAdd(&f.ctr->big_tiles, 1u)] = blockIdx.x;
            else f.tile_cnt[atomicAdd(&f.ctr->mid_tiles, 1u)] = blockIdx.x;
        }
        return;
    }
    sort_tile<kBuckets>(f, blockIdx.x, s, sm);
}

constexpr int kMidSortCtas = 148 * 5;
__global__ void __launch_bounds__(BSR_BLOCK) tile_sort_mid_kernel(FrameView f) {
    pdl_wait();
    __shared__ uint64_t s[kSortSmem];
    __shared__ SortSmem<kBuckets> sm;
    if (over_capacity(f)) return;
    const uint32_t nmid = f.ctr->mid_tiles;
    for (uint32_t k = blockIdx.x; k < nmid; k += gridDim.x) sort_tile<kBuckets>(f, (int)f.tile_cnt[k], s, sm);
}

// Crowded tiles (more than kSortSmem entries; config 4's dense cluster reaches ~4200):
// the same bucket sort with kBigSortSmem entries in dynamic shared memory and 4x the fine
// buckets; tile_sort_kernel queues the crowded tiles (their ids in tile_cur, the count in
// Counters::big_tiles) and kBigSortCtas CTAs take them grid-stride; beyond kBigSortSmem the
// in-place bitonic network in global memory.
constexpr int kBigSortSmem = 20480;  // 160 KB of u64 keys
constexpr int kBigBuckets = 4096;
constexpr int kBigSortCtas = 148;
static_assert(kBigSortSmem / (kMaxBucket + 1) < 1280, "big-bucket list bound (SortSmem::bigbuf)");

struct BigSortSmem {
    uint64_t s[kBigSortSmem];
    SortSmem<kBigBuckets> sm;
};

__global__ void __launch_bounds__(BSR_BLOCK) tile_sort_big_kernel(FrameView f) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char big_smem[];
    BigSortSmem &b = *reinterpret_cast<BigSortSmem *>(big_smem);
    if (over_capacity(f)) return;
    const uint32_t nbig = f.ctr->big_tiles;
    for (uint32_t k = blockIdx.x; k < nbig; k += gridDim.x) {
        const int tile = (int)f.tile_cur[k];
        const uint2 rg = f.tile_ranges[tile];
        const int n = (int)(rg.y - rg.x);
        if (n <= kBigSortSmem) {
            sort_tile<kBigBuckets>(f, tile, b.s, b.sm);
            continue;
        }
        uint64_t *g = f.tent + rg.x;
        bitonic_sort_block(g, n);
        fixup_ties(g, n, f.dkey64);
        for (int i = threadIdx.x; i < n; i += BSR_BLOCK) f.lists[rg.x + i] = (uint32_t)g[i];
        __syncthreads();
    }
}

static unsigned entry_blocks(const FrameView &f) {
    return (unsigned)imin64(div_up(f.n, BSR_BLOCK), 148 * 16);
}

// counts -> ranges (profile stage "bin count")
// (the per-tile counts themselves are taken by preprocess, preprocess.cu)
int launch_bin_count(const FrameView &f, cudaStream_t st) {
    if (f.n == 0) return BSR_OK;
    BSR_CUDA_TRY((pdl_launch(bin_scan_kernel, dim3(1), dim3(kScanThreads), 0, st, f)));
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

// entries -> their tiles (profile stage "bin scatter")
int launch_bin_scatter(const FrameView &f, cudaStream_t st) {
    if (f.n == 0) return BSR_OK;
    BSR_CUDA_TRY((pdl_launch(bin_entries_kernel<false>, dim3(entry_blocks(f)), dim3(BSR_BLOCK), 0, st, f)));
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

// per-tile depth order (profile stage "tile sort")
int launch_tile_sort(const FrameView &f, cudaStream_t st) {
    if (f.n == 0 || f.n_tiles == 0) return BSR_OK;
    BSR_CUDA_TRY((pdl_launch(tile_sort_kernel, dim3(f.n_tiles), dim3(BSR_BLOCK), 0, st, f)));
    BSR_CUDA_TRY((pdl_launch(tile_sort_mid_kernel, dim3((unsigned)std::min(f.n_tiles, kMidSortCtas)), dim3(BSR_BLOCK), 0,
                             st, f)));
    static SmemAttrOnce attr;
    BSR_CUDA_TRY(attr.ensure(tile_sort_big_kernel, sizeof(BigSortSmem)));
    BSR_CUDA_TRY((pdl_launch(tile_sort_big_kernel, dim3((unsigned)std::min(f.n_tiles, kBigSortCtas)), dim3(BSR_BLOCK),
                             sizeof(BigSortSmem), st, f)));
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
