// Post-training codec on the device (compression.py:34-250,
// docs/formats.md "Archives").
//
// pack:  Morton keys of the positions quantised to 21 bits per axis in their bounding box
//        (compression.py:34-59) -> stable sort (compression.py:62-66; the LSD radix sort of
//        sort.cu on 64-bit keys) -> per attribute group: per-channel min / max and uniform
//        8-bit codes (compression.py:69-90) laid row-major into a rows x cols grid with zero
//        padding (compression.py:106-117); positions as the four byte planes of their fp32
//        bits (compression.py:160-166).
// unpack: byte planes -> fp32 positions (bit-exact), codes -> mins (1 - t) + maxs t in fp64
//        (compression.py:93-103), rounded once to the fp32 parameter buffer.
// The host only moves bytes: PNG encoding / decoding stays in OpenCV exactly as the
// reference calls it (sceneio.write_png / read_png).
//
// Everything is integer / byte work plus a few fp64 ops per value: HBM-bound.  This file
// is compiled with -fmad=false so the fp64 expressions round exactly like numpy's.
#include "frame.cuh"
#include "sort.cuh"

namespace bsr {

constexpr int kCodecMaxGroups = 64;
constexpr int kCodecMaxChannels = 4 * kCodecMaxGroups;
constexpr double kMortonMax = 2097151.0;  // 2^21 - 1
constexpr double kLevels = 255.0;         // QUANT_BITS = 8

struct CodecTable {
    int n_groups;
    int64_t start[kCodecMaxGroups];     // flat offset of primitive 0, channel 0
    int32_t stride[kCodecMaxGroups];    // floats between consecutive primitives
    int32_t ch[kCodecMaxGroups];        // channels (1..4)
    int64_t code_off[kCodecMaxGroups];  // byte offset of the group's grid in `codes`
    int32_t mm_off[kCodecMaxGroups];    // first channel's slot in mins / maxs
};

// order-preserving float <-> uint32 (for atomicMin / atomicMax)
__device__ __forceinline__ uint32_t f2o(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

struct CodecScratch {
    uint32_t *count;    // [1]
    uint32_t *tickets;  // [8]
    uint32_t *plan;     // [9]
    uint32_t *hist;     // [8][256]
    uint32_t *mm;       // [2][kCodecMaxChannels] ordered min, max
    uint64_t *keys[2];
    uint32_t *vals[2];
    uint32_t *status;   // [8][parts][256]
    int64_t parts;
    int items;
};

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static size_t carve(void *base, int64_t n, CodecScratch *s) {
    const int items = sort_items(n);
    const int64_t parts = div_up(n > 0 ? n : 1, (int64_t)BSR_BLOCK * items);
    char *p = (char *)base;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *r = p ? p + off : nullptr;
        off += align256(bytes);
        return r;
    };
    char *hdr = take(256);
    char *hist = take(8 * 256 * 4);
    char *mm = take(2 * kCodecMaxChannels * 4);
    char *status = take((size_t)8 * parts * 256 * 4);
    const size_t zero_bytes = off;  // header, hist, min/max and status are cleared per call
    char *k0 = take(8 * (size_t)n), *k1 = take(8 * (size_t)n);
    char *v0 = take(4 * (size_t)n), *v1 = take(4 * (size_t)n);
    if (s) {
        s->count = (uint32_t *)hdr;
        s->tickets = (uint32_t *)hdr + 4;
        s->plan = (uint32_t *)hdr + 16;
        s->hist = (uint32_t *)hist;
        s->mm = (uint32_t *)mm;
        s->status = (uint32_t *)status;
        s->keys[0] = (uint64_t *)k0;
        s->keys[1] = (uint64_t *)k1;
        s->vals[0] = (uint32_t *)v0;
        s->vals[1] = (uint32_t *)v1;
        s->parts = parts;
        s->items = items;
    }
    return s ? zero_bytes : off;
}

__global__ void codec_init_kernel(uint32_t *count, uint32_t n, uint32_t *mm) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = n;
    for (int c = threadIdx.x; c < kCodecMaxChannels; c += blockDim.x) {
        mm[c] = 0xffffffffu;              // min
        mm[kCodecMaxChannels + c] = 0u;   // max
    }
}

// Per-channel min / max of every group (grid.y = group); flags non-finite values
// (quantize_attribute raises, compression.py:75-76).
__global__ void codec_minmax_kernel(const float *__restrict__ base, int64_t n, CodecTable t, uint32_t *mm,
                                    int32_t *status) {
    const int g = blockIdx.y;
    const int C = t.ch[g];
    uint32_t lo[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[4] = {0u, 0u, 0u, 0u};
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float *p = base + t.start[g] + (int64_t)t.stride[g] * i;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (c < C) {
                const float v = p[c];
                bad |= !isfinite(v);
                const uint32_t o = f2o(v);
                lo[c] = min(lo[c], o);
                hi[c] = max(hi[c], o);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            lo[c] = min(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], s));
            hi[c] = max(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], s));
        }
    }
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        for (int c = 0; c < C; ++c) {
            atomicMin(mm + t.mm_off[g] + c, lo[c]);
            atomicMax(mm + kCodecMaxChannels + t.mm_off[g] + c, hi[c]);
        }
        if (bad && status) atomicCAS(status, 0, (int32_t)BSR_ERR_BAD_ARG);
    }
}

__global__ void codec_minmax_finish_kernel(const uint32_t *mm, int channels, double *mins, double *maxs) {
    const int c = threadIdx.x;
    if (c >= channels) return;
    mins[c] = (double)o2f(mm[c]);
    maxs[c] = (double)o2f(mm[kCodecMaxChannels + c]);
}

// compression.py:34-42
__device__ __forceinline__ uint64_t spread_bits_21(uint64_t v) {
    v &= 0x1FFFFFull;
    v = (v | (v << 32)) & 0x1F00000000FFFFull;
    v = (v | (v << 16)) & 0x1F0000FF0000FFull;
    v = (v | (v << 8)) & 0x100F00F00F00F00Full;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

// compression.py:45-59: codes = clip(round((p - lo) / span * (2^21 - 1)), 0, 2^21 - 1)
__global__ void morton_kernel(const float *__restrict__ pos, int64_t n, const uint32_t *mm, uint64_t *keys,
                              uint32_t *vals, uint64_t *keys_out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t key = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double lo = (double)o2f(mm[a]);
        double span = (double)o2f(mm[kCodecMaxChannels + a]) - lo;
        if (span == 0.0) span = 1.0;
        double q = rint(((double)pos[3 * i + a] - lo) / span * kMortonMax);
        q = fmin(fmax(q, 0.0), kMortonMax);
        key |= spread_bits_21((uint64_t)q) << a;
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
    if (keys_out) keys_out[i] = key;
}

__global__ void perm_kernel(const CodecScratch s, int64_t n, int64_t *perm) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t sel = s.plan[8] & 1u;
    perm[i] = (int64_t)s.vals[sel][i];
}

// compression.py:69-90 for one value: round((v - min) / span * 255) if span > 0 else 0
__device__ __forceinline__ uint8_t quantize8(float x, double mn, double mx) {
    const double span = mx - mn;
    if (!(span > 0.0)) return 0;
    return (uint8_t)rint(((double)x - mn) / span * kLevels);
}

// One thread per grid cell (row-major, cells >= n are zero padding).
__global__ void codec_encode_kernel(const float *__restrict__ flat, const float *__restrict__ pos, int64_t n,
                                    const int64_t *__restrict__ perm, CodecTable t, int64_t cells,
                                    const double *__restrict__ mins, const double *__restrict__ maxs,
                                    uint8_t *planes, uint8_t *codes) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= cells) return;
    const int64_t src = j < n ? (perm ? perm[j] : j) : -1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const uint32_t bits = src >= 0 ? __float_as_uint(pos[3 * src + a]) : 0u;
#pragma unroll
        for (int b = 0; b < 4; ++b) planes[(int64_t)b * cells * 3 + 3 * j + a] = (uint8_t)(bits >> (8 * b));
    }
    for (int g = 0; g < t.n_groups; ++g) {
        const int C = t.ch[g];
        const float *p = src >= 0 ? flat + t.start[g] + (int64_t)t.stride[g] * src : nullptr;
        uint8_t *o = codes + t.code_off[g] + j * C;
        for (int c = 0; c < C; ++c) {
            const int k = t.mm_off[g] + c;
            o[c] = p ? quantize8(p[c], mins[k], maxs[k]) : (uint8_t)0;
        }
    }
}

// compression.py:199-212 + 93-103: one thread per primitive.
__global__ void codec_decode_kernel(const uint8_t *__restrict__ planes, const uint8_t *__restrict__ codes,
                                    const double *__restrict__ mins, const double *__restrict__ maxs, int64_t n,
                                    CodecTable t, int64_t cells, float *flat, float *pos) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        uint32_t bits = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) bits |= (uint32_t)planes[(int64_t)b * cells * 3 + 3 * i + a] << (8 * b);
        pos[3 * i + a] = __uint_as_float(bits);
    }
    for (int g = 0; g < t.n_groups; ++g) {
        const int C = t.ch[g];
        const uint8_t *c8 = codes + t.code_off[g] + i * C;
        float *o = flat + t.start[g] + (int64_t)t.stride[g] * i;
        for (int c = 0; c < C; ++c) {
            const int k = t.mm_off[g] + c;
            const double tt = (double)c8[c] / kLevels;
            o[c] = (float)(mins[k] * (1.0 - tt) + maxs[k] * tt);
        }
    }
}

static int make_table(int32_t n_groups, const bsr_codec_group *groups, int64_t cells, CodecTable &t,
                      int *channels) {
    if (n_groups < 0 || n_groups > kCodecMaxGroups || (n_groups > 0 && !groups)) return BSR_ERR_BAD_ARG;
    t.n_groups = n_groups;
    int64_t off = 0;
    int mm = 0;
    for (int g = 0; g < n_groups; ++g) {
        const bsr_codec_group &q = groups[g];
        if (q.channels < 1 || q.channels > 4 || q.stride < q.channels || q.start < 0) return BSR_ERR_BAD_ARG;
        t.start[g] = q.start;
        t.stride[g] = q.stride;
        t.ch[g] = q.channels;
        t.code_off[g] = off;
        t.mm_off[g] = mm;
        off += cells * q.channels;
        mm += q.channels;
    }
    if (channels) *channels = mm;
    return BSR_OK;
}

}  // namespace bsr

using namespace bsr;

extern "C" size_t bsr_codec_scratch_bytes(int64_t n) {
    return carve(nullptr, n < 0 ? 0 : n, nullptr);
}

extern "C" int bsr_codec_sort(const float *positions, int64_t n, uint64_t *keys_out, int64_t *perm, void *scratch,
                              size_t scratch_bytes, void *stream) {
    if (n < 0 || n > 0x7fffffffLL || (n > 0 && (!positions || !perm || !scratch)) ||
        (n > 0 && scratch_bytes < bsr_codec_scratch_bytes(n)))
        return BSR_ERR_BAD_ARG;
    if (n == 0) return BSR_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CodecScratch s;
    const size_t zero = carve(scratch, n, &s);
    BSR_CUDA_TRY(cudaMemsetAsync(scratch, 0, zero, st));
    codec_init_kernel<<<1, 256, 0, st>>>(s.count, (uint32_t)n, s.mm);
    CodecTable t;
    bsr_codec_group pg{0, 3, 3};
    make_table(1, &pg, 0, t, nullptr);
    const unsigned blocks = (unsigned)imin64(div_up(n, BSR_BLOCK), 148 * 8);
    codec_minmax_kernel<<<dim3(blocks, 1), BSR_BLOCK, 0, st>>>(positions, n, t, s.mm, nullptr);
    morton_kernel<<<(unsigned)div_up(n, BSR_BLOCK), BSR_BLOCK, 0, st>>>(positions, n, s.mm, s.keys[0], s.vals[0],
                                                                       keys_out);
    BSR_LAUNCH_CHECK();
    SortArgs<uint64_t> a;
    a.keys[0] = s.keys[0];
    a.keys[1] = s.keys[1];
    a.vals[0] = s.vals[0];
    a.vals[1] = s.vals[1];
    a.count = s.count;
    a.bias_inv = nullptr;
    a.hist = s.hist;
    a.plan = s.plan;
    a.status = s.status;
    a.tickets = s.tickets;
    a.passes = 8;
    a.items = s.items;
    a.max_parts = s.parts;
    const int rc = launch_sort(a, n, st);
    if (rc) return rc;
    perm_kernel<<<(unsigned)div_up(n, BSR_BLOCK), BSR_BLOCK, 0, st>>>(s, n, perm);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_codec_encode(const float *flat, const float *positions, int64_t n, const int64_t *perm,
                                int32_t n_groups, const bsr_codec_group *groups, int32_t rows, int32_t cols,
                                uint8_t *planes, uint8_t *codes, double *mins, double *maxs, int32_t *status,
                                void *scratch, size_t scratch_bytes, void *stream) {
    const int64_t cells = (int64_t)rows * cols;
    CodecTable t;
    int channels = 0;
    if (n < 1 || rows < 1 || cols < 1 || cells < n || !flat || !positions || !planes || !mins || !maxs ||
        !scratch || scratch_bytes < bsr_codec_scratch_bytes(n) || (n_groups > 0 && !codes))
        return BSR_ERR_BAD_ARG;
    int rc = make_table(n_groups, groups, cells, t, &channels);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    CodecScratch s;
    const size_t zero = carve(scratch, n, &s);
    BSR_CUDA_TRY(cudaMemsetAsync(scratch, 0, zero, st));
    codec_init_kernel<<<1, 256, 0, st>>>(s.count, (uint32_t)n, s.mm);
    if (n_groups > 0) {
        const unsigned blocks = (unsigned)imin64(div_up(n, BSR_BLOCK), 148 * 2);
        codec_minmax_kernel<<<dim3(blocks, n_groups), BSR_BLOCK, 0, st>>>(flat, n, t, s.mm, status);
        codec_minmax_finish_kernel<<<1, kCodecMaxChannels, 0, st>>>(s.mm, channels, mins, maxs);
    }
    codec_encode_kernel<<<(unsigned)div_up(cells, BSR_BLOCK), BSR_BLOCK, 0, st>>>(flat, positions, n, perm, t, cells,
                                                                                 mins, maxs, planes, codes);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_codec_decode(const uint8_t *planes, const uint8_t *codes, const double *mins,
                                const double *maxs, int64_t n, int32_t n_groups, const bsr_codec_group *groups,
                                int32_t rows, int32_t cols, float *flat, float *positions, void *stream) {
    const int64_t cells = (int64_t)rows * cols;
    CodecTable t;
    if (n < 0 || rows < 1 || cols < 1 || cells < n) return BSR_ERR_BAD_ARG;
    if (n == 0) return BSR_OK;
    if (!planes || !flat || !positions || (n_groups > 0 && (!codes || !mins || !maxs))) return BSR_ERR_BAD_ARG;
    const int rc = make_table(n_groups, groups, cells, t, nullptr);
    if (rc) return rc;
    codec_decode_kernel<<<(unsigned)div_up(n, BSR_BLOCK), BSR_BLOCK, 0, (cudaStream_t)stream>>>(
        planes, codes, mins, maxs, n, t, cells, flat, positions);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}
