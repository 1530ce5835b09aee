// K3a / K3c: hand-written onesweep LSD radix sort (stable), 8-bit digits.
//
// The global depth order (np.argsort(depths, kind="stable"), rasterizer.py:83-85) for the
// parity export: 32-bit keys = fp32-rounded camera z (monotone), values = compact index
// (ascending source index), then the fp64 tie fixup below.  The per-frame binning does
// not need it (bin.cu sorts each tile's entries by the same key).
//
// Fully device-driven (no host sync): the element count lives in device memory, one
// histogram kernel computes every digit place at once, a 1-block plan kernel scans them,
// marks digit places that are constant across all keys as skipped (after subtracting the
// minimum key) and precomputes which ping-pong buffer each pass reads; pass kernels with
// nothing to do exit immediately.  Each pass is a single kernel: partition ticket ->
// warp-level match_any ranking -> per-digit decoupled look-back -> shared-memory
// staging -> coalesced scatter.
//
// HBM roofline per pass: n * 2 * (sizeof(K) + 4) bytes.
#include "frame.cuh"
#include "sort.cuh"

namespace bsr {

template <typename K>
__device__ __forceinline__ K sort_bias(const SortArgs<K> &a) {
    return a.bias_inv ? (K)(~(*a.bias_inv)) : (K)0;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, K bias, int pass) {
    return (uint32_t)(((K)(key - bias) >> (8 * pass)) & 0xFF);
}

template <typename K>
__global__ void __launch_bounds__(BSR_BLOCK) sort_hist_kernel(SortArgs<K> a) {
    __shared__ uint32_t h[sizeof(K)][256];
    const int P = a.passes;
    for (int i = threadIdx.x; i < P * 256; i += BSR_BLOCK) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t n = *a.count;
    const K bias = sort_bias(a);
    const K *keys = a.keys[0];
    for (uint32_t i = blockIdx.x * BSR_BLOCK + threadIdx.x; i < n; i += gridDim.x * BSR_BLOCK) {
        const K k = keys[i];
        for (int p = 0; p < P; ++p) atomicAdd(&h[p][digit_of(k, bias, p)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P * 256; i += BSR_BLOCK) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(a.hist + i, v);
    }
}

// One block of 256 threads: per place, exclusive-scan the histogram in place and decide
// whether the place is active (keys differ in it).
template <typename K>
__global__ void __launch_bounds__(BSR_BLOCK) sort_plan_kernel(SortArgs<K> a) {
    __shared__ uint32_t s[256];
    __shared__ int s_const;
    const int t = threadIdx.x;
    const uint32_t n = *a.count;
    uint32_t cur = 0;
    for (int p = 0; p < a.passes; ++p) {
        const uint32_t v = a.hist[p * 256 + t];
        if (t == 0) s_const = 0;
        __syncthreads();
        if (v == n) s_const = 1;  // all keys share this digit (or n == 0)
        s[t] = v;
        __syncthreads();
        // Hillis-Steele inclusive scan
        for (int o = 1; o < 256; o <<= 1) {
            uint32_t x = t >= o ? s[t - o] : 0;
            __syncthreads();
            s[t] += x;
            __syncthreads();
        }
        a.hist[p * 256 + t] = s[t] - v;
        const bool active = !s_const && n > 1;
        if (t == 0) a.plan[p] = cur | (active ? 0x100u : 0u);
        if (active) cur ^= 1u;
        __syncthreads();
    }
    if (t == 0) a.plan[a.passes] = cur;
}

template <typename K, int kSortItems>
__global__ void __launch_bounds__(BSR_BLOCK) sort_pass_kernel(SortArgs<K> a, int pass) {
    constexpr int kSortTile = BSR_BLOCK * kSortItems;
    const uint32_t plan = a.plan[pass];
    if (!(plan & 0x100u)) return;
    const uint32_t src = plan & 1u;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K *s_keys = reinterpret_cast<K *>(smem_raw);
    uint32_t *s_vals = reinterpret_cast<uint32_t *>(s_keys + kSortTile);
    uint32_t *s_whist = s_vals + kSortTile;             // [8][256]
    uint32_t *s_excl = s_whist + 8 * 256;               // [256] block-exclusive digit start
    uint32_t *s_gbase = s_excl + 256;                   // [256] global start for this block
    __shared__ uint32_t s_part;

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) s_part = atomicAdd(a.tickets + pass, 1u);
    for (int i = t; i < 8 * 256; i += BSR_BLOCK) s_whist[i] = 0;
    __syncthreads();
    const uint32_t n = *a.count;
    const int64_t part = s_part;
    const int64_t base = part * kSortTile;
    if (base >= (int64_t)n) return;
    const K bias = sort_bias(a);
    const K *keys_in = a.keys[src];
    const uint32_t *vals_in = a.vals[src];

    K k[kSortItems];
    uint32_t v[kSortItems], d[kSortItems], rank[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int64_t idx = base + warp * (32 * kSortItems) + i * 32 + lane;
        const bool ok = idx < (int64_t)n;
        k[i] = ok ? keys_in[idx] : (K)0;
        v[i] = ok ? vals_in[idx] : 0u;
        d[i] = ok ? digit_of(k[i], bias, pass) : 256u;
    }
    // warp-level stable ranking: items in (i, lane) order == input order
    uint32_t *wh = s_whist + warp * 256;
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const uint32_t peers = __match_any_sync(0xffffffffu, d[i]);
        const int leader = __ffs(peers) - 1;
        uint32_t before = 0;
        if (lane == leader && d[i] < 256u) {
            before = wh[d[i]];
            wh[d[i]] = before + __popc(peers);
        }
        before = __shfl_sync(0xffffffffu, before, leader);
        rank[i] = before + __popc(peers & lt_mask);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, block count, look-back, global base
    {
        const int dg = t;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const uint32_t c = s_whist[w * 256 + dg];
            s_whist[w * 256 + dg] = run;
            run += c;
        }
        uint32_t *st = a.status + ((int64_t)pass * a.max_parts) * 256 + dg;
        uint32_t excl = 0;
        if (part == 0) {
            st_release(st, kFlagPrefix | run);
        } else {
            st_release(st + part * 256, kFlagAgg | run);
            // look back 8 predecessors per round trip (independent loads in flight)
            for (int64_t hi = part - 1; hi >= 0; hi -= 8) {
                uint32_t s[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) s[q] = hi - q >= 0 ? ld_volatile(st + (hi - q) * 256) : kFlagPrefix;
                bool done = false;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    while ((s[q] & ~kValueMask) == 0) s[q] = ld_volatile(st + (hi - q) * 256);
                    excl += s[q] & kValueMask;
                    if (s[q] & kFlagPrefix) {
                        done = true;
                        break;
                    }
                }
                if (done) break;
            }
            st_release(st + part * 256, kFlagPrefix | (excl + run));
        }
        s_gbase[dg] = a.hist[pass * 256 + dg] + excl;
        s_excl[dg] = run;  // scanned below
    }
    __syncthreads();
    // block exclusive scan of per-digit counts (256 values, one per thread)
    {
        uint32_t x = s_excl[t];
        const uint32_t own = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        __shared__ uint32_t s_wsum[8];
        if (lane == 31) s_wsum[warp] = x;
        __syncthreads();
        uint32_t wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
        s_excl[t] = wpre + x - own;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        if (d[i] < 256u) {
            const uint32_t pos = s_excl[d[i]] + s_whist[warp * 256 + d[i]] + rank[i];
            s_keys[pos] = k[i];
            s_vals[pos] = v[i];
        }
    }
    __syncthreads();
    const int64_t cnt = min((int64_t)kSortTile, (int64_t)n - base);
    K *keys_out = a.keys[src ^ 1u];
    uint32_t *vals_out = a.vals[src ^ 1u];
#pragma unroll 4
    for (int i = 0; i < kSortItems; ++i) {
        const int pos = i * BSR_BLOCK + t;  // (coalesced within each digit run)
        if (pos < cnt) {
            const K key = s_keys[pos];
            const uint32_t dg = digit_of(key, bias, pass);
            const uint32_t o = s_gbase[dg] + (pos - s_excl[dg]);
            keys_out[o] = key;
            vals_out[o] = s_vals[pos];
        }
    }
}

template <typename K, int ITEMS>
size_t sort_smem_bytes() {
    return (size_t)BSR_BLOCK * ITEMS * (sizeof(K) + 4) + 4 * (8 * 256 + 256 + 256);
}

template <typename K, int ITEMS>
static int launch_passes(const SortArgs<K> &a, int64_t cap, cudaStream_t st) {
    static SmemAttrOnce attr;
    const size_t smem = sort_smem_bytes<K, ITEMS>();
    BSR_CUDA_TRY(attr.ensure(sort_pass_kernel<K, ITEMS>, smem));
    const unsigned parts = (unsigned)div_up(cap, BSR_BLOCK * ITEMS);
    for (int p = 0; p < a.passes; ++p) sort_pass_kernel<K, ITEMS><<<parts, BSR_BLOCK, smem, st>>>(a, p);
    return BSR_OK;
}

template <typename K>
int launch_sort(const SortArgs<K> &a, int64_t cap, cudaStream_t st) {
    if (cap <= 0) return BSR_OK;
    const unsigned hist_blocks = (unsigned)imin64(div_up(cap, 4096), 148 * 4);
    sort_hist_kernel<K><<<hist_blocks, BSR_BLOCK, 0, st>>>(a);
    sort_plan_kernel<K><<<1, BSR_BLOCK, 0, st>>>(a);
    const int rc = a.items == 4 ? launch_passes<K, 4>(a, cap, st) : launch_passes<K, 16>(a, cap, st);
    if (rc) return rc;
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

template int launch_sort<uint32_t>(const SortArgs<uint32_t> &, int64_t, cudaStream_t);
template int launch_sort<uint64_t>(const SortArgs<uint64_t> &, int64_t, cudaStream_t);

// After sorting the fp32-rounded depths, primitives whose fp32 keys tie are re-ordered by
// their exact fp64 depth (then compact index): rounding is monotone, so this yields exactly
// np.argsort(fp64 depths, kind="stable").  Runs of equal fp32 keys are short; the thread
// at the start of each run insertion-sorts it.
__global__ void depth_fixup_kernel(FrameView f) {
    const uint32_t V = f.ctr->visible;
    const uint32_t sel = f.ctr->depth_plan[kDepthPasses] & 1u;
    const uint32_t *k = f.dkeys[sel];
    uint32_t *v = f.dvals[sel];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < V; i += gridDim.x * blockDim.x) {
        const uint32_t ki = k[i];
        if (k[i + 1] != ki || (i > 0 && k[i - 1] == ki)) continue;  // not the start of a run
        uint32_t j = i + 2;
        while (j < V && k[j] == ki) ++j;
        for (uint32_t a = i + 1; a < j; ++a) {
            const uint32_t va = v[a];
            const uint64_t da = f.dkey64[va];
            uint32_t b = a;
            while (b > i) {
                const uint32_t vb = v[b - 1];
                const uint64_t db = f.dkey64[vb];
                if (db < da || (db == da && vb < va)) break;
                v[b] = vb;
                --b;
            }
            v[b] = va;
        }
    }
}

int launch_depth_sort(const FrameView &f, cudaStream_t st) {
    SortArgs<uint32_t> a;
    a.keys[0] = f.dkeys[0];
    a.keys[1] = f.dkeys[1];
    a.vals[0] = f.dvals[0];
    a.vals[1] = f.dvals[1];
    a.count = &f.ctr->visible;
    a.bias_inv = &f.ctr->depth_key_max_inv;
    a.hist = f.depth_hist;
    a.plan = f.ctr->depth_plan;
    a.status = f.depth_status;
    a.tickets = f.ctr->depth_ticket;
    a.passes = kDepthPasses;
    a.items = f.depth_items;
    a.max_parts = f.depth_parts;
    int rc = launch_sort(a, f.n, st);
    if (rc) return rc;
    if (f.n > 1) {
        depth_fixup_kernel<<<(unsigned)imin64(div_up(f.n, BSR_BLOCK), 148 * 8), BSR_BLOCK, 0, st>>>(f);
        BSR_LAUNCH_CHECK();
    }
    return BSR_OK;
}

}  // namespace bsr
