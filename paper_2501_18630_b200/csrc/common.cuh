// Internal definitions shared by the libbsr kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bsr.h"

#define BSR_TILE 16
#define BSR_MAX_LOBES 4
#define BSR_BLOCK 256

namespace bsr {

// Constants of the reference contract (rasterizer.py:28-30, primitive.py:22-25,
// kernel.py:24-28).
constexpr double kNearPlane = 0.01;
constexpr double kCovConditioning = 0.3;
constexpr int kBoundsGuard = 1;
constexpr double kShapeClamp = 10.0;
constexpr double kBaseExponent = 4.0;
constexpr float kEdgeGradClamp = 1e7f;

// Device-side error word values (bsr_status); first error wins (atomicCAS from 0).
__device__ __forceinline__ void raise_status(int32_t *status, int32_t code) {
    atomicCAS(reinterpret_cast<int *>(status), 0, code);
}

// ----------------------------------------------------------------------------------
// Camera as seen by kernels.
struct KCam {
    double R[9];  // world->camera rotation, row-major
    double t[3];
    double center[3];  // -R^T t
    double fx, fy, cx, cy;
    int W, H, tiles_x, tiles_y;
};

inline KCam make_kcam(const bsr_camera &c) {
    KCam k;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) k.R[3 * i + j] = c.world_to_camera[4 * i + j];
        k.t[i] = c.world_to_camera[4 * i + 3];
    }
    for (int j = 0; j < 3; ++j)
        k.center[j] = -(k.R[0 + j] * k.t[0] + k.R[3 + j] * k.t[1] + k.R[6 + j] * k.t[2]);
    k.fx = c.fx;
    k.fy = c.fy;
    k.cx = c.cx;
    k.cy = c.cy;
    k.W = c.width;
    k.H = c.height;
    k.tiles_x = (c.width + BSR_TILE - 1) / BSR_TILE;
    k.tiles_y = (c.height + BSR_TILE - 1) / BSR_TILE;
    return k;
}

// ----------------------------------------------------------------------------------
// Raster record: one per visible primitive, compact (source) order, 64 B.
//   A: mean_x - x0, mean_y - y0, conic a, conic b      (mean stored relative to its
//      bounds corner so dx = (px - x0) - rel loses no bits at large pixel coordinates)
//   B: conic c, opacity, beta, depth z
//   C: r, g, b, kR = bound on |r2(fp32) - r2(exact)| over the footprint (error analysis,
//      raster.cuh); NEGATIVE kR marks an fp32-unsafe (ill-conditioned) primitive whose r2 /
//      alpha the raster evaluates in fp64 from FrameView::rec64.  The source index lives
//      is the record index itself (records are indexed by source index).
//   D: x0, x1, y0, y1 (inclusive pixel bounds, primitive.py:252-262)
struct __align__(16) Record {
    float4 a, b, c;
    int4 d;
};
static_assert(sizeof(Record) == 64, "record must be 64 B");

// fp64 projected primitive (primitive.py:221-277), the single source of truth used by
// preprocess AND by the fp64 replay of flagged pixels (same code => same bits).
struct Proj64 {
    double mx, my;       // mean2d
    double c00, c01, c11;  // conditioned cov2d
    double ca, cb, cc;   // conic
    double tx, ty, tz;   // camera-space point
    int x0, x1, y0, y1;  // bounds (inclusive)
    bool visible;
    bool degenerate;
};

// Lookback status word: [31:30] flag (0 none, 1 aggregate, 2 inclusive prefix), [29:0] value.
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
    return *reinterpret_cast<const volatile uint32_t *>(p);
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    __threadfence();
    *reinterpret_cast<volatile uint32_t *>(p) = v;
}

// Exclusive prefix over predecessors [0, part) via decoupled look-back on `status`.
__device__ __forceinline__ uint32_t lookback_exclusive(const uint32_t *status, int part) {
    uint32_t excl = 0;
    for (int j = part - 1; j >= 0;) {
        uint32_t s = ld_volatile(status + j);
        if ((s & ~kValueMask) == 0) continue;  // spin until published
        excl += s & kValueMask;
        if (s & kFlagPrefix) break;
        --j;
    }
    return excl;
}

// ---- TMA bulk copies (cp.async.bulk, global -> shared, mbarrier completion) ----------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Dispatch a templated launcher on the colour model: CM = K (SH coefficients) or -M (SB).
#define BSR_DISPATCH_CM(sc, LAUNCH)                                         \
    do {                                                                   \
        if ((sc).color_model == BSR_COLOR_SB) {                            \
            switch ((sc).lobes) {                                          \
                case 0: LAUNCH(0); break;                                  \
                case 1: LAUNCH(-1); break;                                 \
                case 2: LAUNCH(-2); break;                                 \
                case 3: LAUNCH(-3); break;                                 \
                case 4: LAUNCH(-4); break;                                 \
                default: return BSR_ERR_BAD_ARG;                           \
            }                                                              \
        } else {                                                           \
            switch ((sc).sh_coeffs) {                                      \
                case 1: LAUNCH(1); break;                                  \
                case 4: LAUNCH(4); break;                                  \
                case 9: LAUNCH(9); break;                                  \
                case 16: LAUNCH(16); break;                                \
                default: return BSR_ERR_BAD_ARG;                           \
            }                                                              \
        }                                                                  \
    } while (0)

// Warp-parallel decoupled look-back (called by ALL 32 lanes of one warp): lane l reads the
// status of predecessor part-1-l, 32 predecessors per L2 round trip instead of one; the
// nearest inclusive prefix ends the walk.  `stride` separates consecutive partitions.
template <typename W>
__device__ __forceinline__ W warp_lookback(const W *status, int64_t part, int64_t stride, W flag_prefix,
                                           W value_mask) {
    const int lane = threadIdx.x & 31;
    W excl = 0;
    int64_t hi = part - 1;
    while (true) {
        const int64_t j = hi - lane;
        W s;
        if (j >= 0) {
            do {
                s = *reinterpret_cast<const volatile W *>(status + j * stride);
            } while ((s & ~value_mask) == 0);
        } else {
            s = flag_prefix;  // virtual inclusive prefix 0 before partition 0
        }
        const unsigned pm = __ballot_sync(0xffffffffu, (s & flag_prefix) != 0);
        const int first = pm ? __ffs(pm) - 1 : 32;
        W v = lane <= first ? (s & value_mask) : (W)0;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pm) return excl;
        hi -= 32;
    }
}

__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ inline int64_t div_up(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline uint64_t align_up(uint64_t a, uint64_t b) { return (a + b - 1) / b * b; }

}  // namespace bsr

namespace bsr {
// ---- programmatic dependent launch (sm_90+): hot-path kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's grid is launched while
// its predecessor in the stream drains (no launch gap between dependent kernels, also
// inside captured CUDA graphs).  Every such kernel calls pdl_wait() before it touches
// memory; griddepcontrol.wait returns once the predecessor grid has completed and its
// writes are visible (immediately for a normal launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

bool pdl_enabled();  // api.cu (BSR_NO_PDL=1 disables, for A/B measurements)

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute: set it once per
// (kernel, device) -- a process may drive several GPUs.  Each call site owns its flags.
struct SmemAttrOnce {
    bool done[64] = {};
    template <typename... KArgs>
    cudaError_t ensure(void (*kernel)(KArgs...), size_t bytes) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
        return e;
    }
};
}  // namespace bsr

#define BSR_CUDA_TRY(expr)                                      \
    do {                                                        \
        cudaError_t _e = (expr);                                \
        if (_e != cudaSuccess) return BSR_ERR_CUDA;             \
    } while (0)
#define BSR_LAUNCH_CHECK() BSR_CUDA_TRY(cudaGetLastError())
