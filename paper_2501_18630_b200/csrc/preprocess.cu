// K1+K2 preprocess: fp64 EWA projection (primitive.py:221-277), SH colour
// (appearance.py:235-261 via the SH adapter), opacity / Beta exponent.  Records are indexed
// by the source index (culled primitives get tile_count 0): the reference's visible
// subset ``idx = nonzero(vis)[keep]`` keeps source order, so every later stage can use
// the source index as the batch index without a compaction pass.
//
// Compiled with -fmad=false: the fp64 integer outputs (bounds, depth keys) must follow
// the reference's rounding, and replay.cu recomputes the same primitives bit-identically.
//
// HBM roofline: N*(48 + 12K) B read, V*(64 + 8 + 4 + 4) B written.
#include "frame.cuh"
#include "appearance.cuh"
#include "project.cuh"
#include "raster.cuh"

namespace bsr {

// CTA size NT: 4-warp CTAs (30 KB of staging each for SH-3, up to 7 CTAs per SM) for scenes
// up to kPreSmallMaxN primitives -- small scenes (config 1: one wave) spread evenly over the
// SMs; 8-warp CTAs above (measured: 1M / 3M configs 6% / 11% faster at 128 threads, the 6M
// config 11% faster at 256)
constexpr int64_t kPreSmallMaxN = 4 << 20;

struct PreArgs {
    bsr_scene sc;
    KCam cam;
    FrameView f;
};

// Bound on |r2_fp32 - r2_exact| for any pixel of the footprint (bounds box: |dx| <= ex + 2,
// |dy| <= ey + 2 around the mean, ex = sqrt(Sigma'_00)) of the factored evaluation in
// eval_pair (raster.cuh chol_r2_error_bound).
__device__ __forceinline__ double r2_error_bound(const Proj64 &p, double l11, double l21, double l22) {
    return chol_r2_error_bound(l11, l21, l22, sqrt(p.c00) + 2.0, sqrt(p.c11) + 2.0);
}

// Shared-memory staging of one CTA's 256 primitives: the parameter blocks are contiguous
// per CTA, so one elected thread moves the geometry (48 B per primitive) with TMA bulk
// copies (cp.async.bulk + mbarrier); partial / misaligned blocks fall back to cooperative
// loads.  The appearance payload (192 B per primitive for SH-3) is needed only for visible
// primitives: when at least half of the CTA is visible it comes in one more bulk copy,
// otherwise each visible thread copies its own row with cp.async (wide views of large
// scenes and mostly-culled CTAs).  When the previous forward on this frame kept at least
// half of the primitives (FrameView::vis_hint) the appearance block is requested together
// with the geometry instead, so its latency overlaps the projection (measured with the
// current CTA sizes: config 2 0.090 -> 0.080 ms, config 3 0.251 -> 0.237, config 4 0.616 ->
// 0.605; a build A/B with -DBSR_EAGER_APP_MAX_N=0, scripts/gpu/ab.sh).
#ifndef BSR_EAGER_APP_MAX_N
#define BSR_EAGER_APP_MAX_N (1ll << 40)  // no size limit (build knob for A/B runs)
#endif
constexpr int64_t kEagerAppMaxN = BSR_EAGER_APP_MAX_N;
constexpr uint32_t kPreBigRect = 512;  // tile rectangles counted by the whole CTA
// Appearance payload: SH -> sh[256][3K];  SB -> base[256][3] | axes[256][3M] | cols[256][3M]
template <int CM, int kPreThreads>
struct PreSmem {
    float pos[kPreThreads * 3], rot[kPreThreads * 4], ls[kPreThreads * 3], op[kPreThreads], shp[kPreThreads];
    float app[kPreThreads * AppTraits<CM>::floats];
};

// The fp32 colour of one primitive seen from `center` (appearance payload rows as staged):
// shared by preprocess and bsr_view_colors so both produce the same bits.
template <int CM>
__device__ __forceinline__ void view_color(const float *pos, const double *center, const float *pa, const float *pb,
                                           const float *pc, float rgb[3]) {
    float vx = pos[0] - (float)center[0], vy = pos[1] - (float)center[1], vz = pos[2] - (float)center[2];
    const float inv = rsqrtf(vx * vx + vy * vy + vz * vz);
    if constexpr (AppTraits<CM>::sh)
        app_color32<CM>(pa, nullptr, nullptr, vx * inv, vy * inv, vz * inv, rgb);
    else
        app_color32<CM>(pa, pb, pc, vx * inv, vy * inv, vz * inv, rgb);
}

// bsr_view_colors: one thread per primitive reads its appearance row once and evaluates it
// for every view (views <= kMaxColorViews per launch); rgb[v][i] as float4.
constexpr int kMaxColorViews = 64;
struct ViewColorArgs {
    bsr_scene sc;
    double center[kMaxColorViews][3];
    int views;
    float4 *rgb;
};

template <int CM>
__global__ void __launch_bounds__(256) view_colors_kernel(__grid_constant__ const ViewColorArgs a) {
    pdl_wait();
    using Tr = AppTraits<CM>;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.sc.n) return;
    float row[Tr::floats];
    const float *src_a = Tr::sh ? a.sc.sh + 3 * Tr::K * i : a.sc.base_colors + 3 * i;
    for (int q = 0; q < (Tr::sh ? 3 * Tr::K : 3); ++q) row[q] = __ldg(src_a + q);
    if constexpr (!Tr::sh) {
        for (int q = 0; q < 3 * Tr::M; ++q) {
            row[3 + q] = __ldg(a.sc.lobe_axes + 3 * Tr::M * i + q);
            row[3 + 3 * Tr::M + q] = __ldg(a.sc.lobe_colors + 3 * Tr::M * i + q);
        }
    }
    const float pos[3] = {a.sc.positions[3 * i], a.sc.positions[3 * i + 1], a.sc.positions[3 * i + 2]};
    for (int v = 0; v < a.views; ++v) {
        float rgb[3];
        view_color<CM>(pos, a.center[v], row, row + 3, row + 3 + 3 * Tr::M, rgb);
        a.rgb[(int64_t)v * a.sc.n + i] = make_float4(rgb[0], rgb[1], rgb[2], 0.f);
    }
}

int launch_view_colors(const bsr_scene &sc, const double *centers, int views, float *rgb, cudaStream_t st) {
    if (sc.n == 0 || views == 0) return BSR_OK;
    for (int v0 = 0; v0 < views; v0 += kMaxColorViews) {
        ViewColorArgs a;
        a.sc = sc;
        a.views = views - v0 < kMaxColorViews ? views - v0 : kMaxColorViews;
        for (int v = 0; v < a.views; ++v)
            for (int c = 0; c < 3; ++c) a.center[v][c] = centers[3 * (v0 + v) + c];
        a.rgb = reinterpret_cast<float4 *>(rgb) + (int64_t)v0 * sc.n;
        const unsigned blocks = (unsigned)div_up(sc.n, (int64_t)256);
#define BSR_VC_LAUNCH(CM) BSR_CUDA_TRY((pdl_launch(view_colors_kernel<CM>, dim3(blocks), dim3(256), 0, st, a)))
        BSR_DISPATCH_CM(sc, BSR_VC_LAUNCH);
#undef BSR_VC_LAUNCH
    }
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

template <int CM, int kPreThreads>
__global__ void __launch_bounds__(kPreThreads, kPreThreads == 128 ? 7 : 3) preprocess_fwd_kernel(PreArgs args) {
    pdl_wait();
    using Tr = AppTraits<CM>;
    const FrameView &f = args.f;
    extern __shared__ __align__(16) unsigned char pre_smem_raw[];
    PreSmem<CM, kPreThreads> &sm = *reinterpret_cast<PreSmem<CM, kPreThreads> *>(pre_smem_raw);
    float *app_a = sm.app;                                  // SH coeffs / SB base colours
    float *app_b = sm.app + kPreThreads * (Tr::sh ? 0 : 3);   // SB lobe axes
    float *app_c = app_b + kPreThreads * 3 * Tr::M;           // SB lobe colours
    __shared__ __align__(8) uint64_t s_bar[2];  // geometry, appearance
    __shared__ int s_bulk;
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t n = args.sc.n;
    const bsr_scene &sc = args.sc;
    const int64_t part = blockIdx.x;
    const int64_t base = part * kPreThreads;
    const int64_t cnt = imin64(kPreThreads, n - base);
    const float *app_src_a = Tr::sh ? sc.sh + 3 * Tr::K * base : sc.base_colors + 3 * base;
    __shared__ int s_eager;
    auto issue_app = [&]() {  // one elected thread: the CTA's whole appearance block
        const uint32_t bapp = kPreThreads * 4 * Tr::floats;
        mbar_expect_tx(&s_bar[1], bapp);
        if constexpr (Tr::sh) {
            bulk_g2s(app_a, app_src_a, bapp, &s_bar[1]);
        } else {
            bulk_g2s(app_a, app_src_a, kPreThreads * 12, &s_bar[1]);
            if constexpr (Tr::M > 0) {
                bulk_g2s(app_b, sc.lobe_axes + 3 * Tr::M * base, kPreThreads * 12 * Tr::M, &s_bar[1]);
                bulk_g2s(app_c, sc.lobe_colors + 3 * Tr::M * base, kPreThreads * 12 * Tr::M, &s_bar[1]);
            }
        }
    };
    if (tid == 0) {
        uintptr_t al = reinterpret_cast<uintptr_t>(sc.positions) | reinterpret_cast<uintptr_t>(sc.rotations) |
                       reinterpret_cast<uintptr_t>(sc.log_scales) | reinterpret_cast<uintptr_t>(sc.opacity_raw) |
                       reinterpret_cast<uintptr_t>(sc.shapes);
        if constexpr (Tr::sh)
            al |= reinterpret_cast<uintptr_t>(sc.sh);
        else
            al |= reinterpret_cast<uintptr_t>(sc.base_colors) | reinterpret_cast<uintptr_t>(sc.lobe_axes) |
                  reinterpret_cast<uintptr_t>(sc.lobe_colors);
        const bool bulk = cnt == kPreThreads && (al & 15) == 0;
        s_bulk = bulk;
        if (bulk) {
            mbar_init(&s_bar[0], 1);
            mbar_init(&s_bar[1], 1);
            const uint32_t b3 = kPreThreads * 12, b4 = kPreThreads * 16, b1 = kPreThreads * 4;
            mbar_expect_tx(&s_bar[0], 2 * b3 + b4 + 2 * b1);
            bulk_g2s(sm.pos, sc.positions + 3 * base, b3, &s_bar[0]);
            bulk_g2s(sm.rot, sc.rotations + 4 * base, b4, &s_bar[0]);
            bulk_g2s(sm.ls, sc.log_scales + 3 * base, b3, &s_bar[0]);
            bulk_g2s(sm.op, sc.opacity_raw + base, b1, &s_bar[0]);
            bulk_g2s(sm.shp, sc.shapes + base, b1, &s_bar[0]);
            const bool eager = !sc.view_rgb && n <= kEagerAppMaxN && 2 * (int64_t)*f.vis_hint >= n;
            s_eager = eager;
            if (eager) issue_app();
        }
    }
    __syncthreads();
    const int64_t i = base + tid;
    const bool bulk = s_bulk;
    if (bulk) {
        mbar_wait(&s_bar[0], 0);
    } else {
        for (int q = tid; q < cnt * 3; q += kPreThreads) {
            sm.pos[q] = sc.positions[3 * base + q];
            sm.ls[q] = sc.log_scales[3 * base + q];
        }
        for (int q = tid; q < cnt * 4; q += kPreThreads) sm.rot[q] = sc.rotations[4 * base + q];
        for (int q = tid; q < cnt; q += kPreThreads) {
            sm.op[q] = sc.opacity_raw[base + q];
            sm.shp[q] = sc.shapes[base + q];
        }
        if (sc.view_rgb) {
            // colours precomputed (bsr_view_colors): no appearance payload
        } else if constexpr (Tr::sh) {
            for (int q = tid; q < cnt * 3 * Tr::K; q += kPreThreads) app_a[q] = app_src_a[q];
        } else {
            for (int q = tid; q < cnt * 3; q += kPreThreads) app_a[q] = app_src_a[q];
            for (int q = tid; q < cnt * 3 * Tr::M; q += kPreThreads) {
                app_b[q] = sc.lobe_axes[3 * Tr::M * base + q];
                app_c[q] = sc.lobe_colors[3 * Tr::M * base + q];
            }
        }
        __syncthreads();
    }

    bool vis = false;
    Record r;
    uint64_t key = 0;
    uint32_t key32 = 0;
    bool unsafe = false;
    double m64[kRec64];
    uint32_t tcount = 0;
    Proj64 p;
    if (i < n) {
        p = project64(sm.pos + 3 * tid, sm.rot + 4 * tid, sm.ls + 3 * tid, args.cam);
        if (p.degenerate) raise_status(&f.ctr->status, BSR_ERR_DEGENERATE_QUAT);
        vis = p.visible;
    }
    // visible count (statistics / frame_status); records are indexed by the source index
    // itself, so no compaction (and no cross-CTA dependency) is needed: the order of the
    // visible subset the reference's ``batch.indices`` defines is the source order
    {
        const uint32_t ballot = __ballot_sync(0xffffffffu, vis);
        if (lane == 0 && ballot) atomicAdd(&f.ctr->visible, (uint32_t)__popc(ballot));
    }
    // appearance payload of the visible primitives (the non-bulk path staged everything)
    bool app_bulk = false;
    if (sc.view_rgb) {
        // colours precomputed (bsr_view_colors): nothing to stage
    } else if (bulk && s_eager) {
        app_bulk = true;  // requested with the geometry
    } else if (bulk) {
        const int nvis = __syncthreads_count(vis);
        app_bulk = 2 * nvis >= kPreThreads;
        if (app_bulk) {
            if (tid == 0) issue_app();
        } else if (vis) {  // own row only; read back by this thread alone
            constexpr int F = Tr::sh ? 3 * Tr::K : 3;
            if constexpr (F % 4 == 0) {
                for (int q = 0; q < F; q += 4) cp_async16(app_a + F * tid + q, app_src_a + F * tid + q);
            } else {
                for (int q = 0; q < F; ++q) cp_async4(app_a + F * tid + q, app_src_a + F * tid + q);
            }
            if constexpr (!Tr::sh) {
                for (int q = 0; q < 3 * Tr::M; ++q) {
                    cp_async4(app_b + 3 * Tr::M * tid + q, sc.lobe_axes + 3 * Tr::M * i + q);
                    cp_async4(app_c + 3 * Tr::M * tid + q, sc.lobe_colors + 3 * Tr::M * i + q);
                }
            }
            cp_async_commit();
        }
    }
    // every thread waits for a requested bulk copy (a CTA must not retire with one in flight)
    if (app_bulk) mbar_wait(&s_bar[1], 0);
    if (vis) {
        float rgb[3];
        if (sc.view_rgb) {
            const float4 c4 = __ldg(reinterpret_cast<const float4 *>(sc.view_rgb) + i);
            rgb[0] = c4.x;
            rgb[1] = c4.y;
            rgb[2] = c4.z;
        } else {
            if (!app_bulk && bulk) cp_async_wait<0>();
            const float *pos = sm.pos + 3 * tid;
            view_color<CM>(pos, args.cam.center, app_a + (Tr::sh ? 3 * Tr::K : 3) * tid, app_b + 3 * Tr::M * tid,
                           app_c + 3 * Tr::M * tid, rgb);
        }
        const double o = sigmoid64((double)sm.op[tid]);
        const double beta = shape_to_exponent64((double)sm.shp[tid]);
        double l11, l21, l22;
        const bool pd = conic_cholesky(p.ca, p.cb, p.cc, l11, l21, l22);
        r.a = make_float4((float)(p.mx - p.x0), (float)(p.my - p.y0), (float)l11, (float)l21);
        r.b = make_float4((float)l22, (float)o, (float)beta, (float)p.tz);
        float kr = pd ? (float)r2_error_bound(p, l11, l21, l22) : 1.0f;
        unsafe = !pd || kr > kUnsafeR2Err;
        if (unsafe) {  // needle (compensated fp32) if its bound allows, else the fp64 path
            float4 nw = make_float4(__int_as_float(0x7fc00000), pd ? 1.f : 0.f, 0.f, 0.f);
            if (pd) {
                const float kn = (float)needle_r2_error_bound(l11, l21, sqrt(p.c00) + 2.0, sqrt(p.c11) + 2.0);
                if (kn <= kUnsafeR2Err) {
                    kr = kn;
                    nw = needle_word(l11, l21, p.mx - p.x0, p.my - p.y0);
                }
            }
            f.needle[i] = nw;
            if (nw.x != nw.x) {  // fp64 path: its factor, or zeroed xy-frame fp64 accumulators
                double2 *s64 = reinterpret_cast<double2 *>(f.side64 + kSide64 * (int64_t)i);
                s64[0] = make_double2(pd ? l11 : 0.0, pd ? l21 : 0.0);
                s64[1] = make_double2(pd ? l22 : 0.0, 0.0);
                s64[2] = make_double2(0.0, 0.0);
            }
        }
        r.c = make_float4(rgb[0], rgb[1], rgb[2], record_err_word(kr, (double)r.b.z, unsafe));
        m64[0] = p.mx;
        m64[1] = p.my;
        m64[2] = p.ca;
        m64[3] = p.cb;
        m64[4] = p.cc;
        m64[5] = o;
        m64[6] = beta;
        m64[7] = p.tz;
        r.d = make_int4(p.x0, p.x1, p.y0, p.y1);
        key = (uint64_t)__double_as_longlong(p.tz);  // tz > 0.01: bits are monotonic
        key32 = (uint32_t)__float_as_int((float)p.tz);  // monotone rounding of tz
        tcount = (uint32_t)((p.x1 / BSR_TILE - p.x0 / BSR_TILE + 1) * (p.y1 / BSR_TILE - p.y0 / BSR_TILE + 1));
    }
    // min depth key for the radix plan: max of the complement
    const uint32_t inv = __reduce_max_sync(0xffffffffu, vis ? ~key32 : 0u);
    if (lane == 0 && inv) atomicMax(&f.ctr->depth_key_max_inv, inv);
    if (i < n) f.tile_count[i] = tcount;  // 0: culled
    // ---- tile_bins counts (rasterizer.py:161-191), fused here instead of a second pass
    //      over the records: the warp's entries are spread over its lanes round-robin
    //      (owner found by a search over the inclusive prefix), one RED per entry;
    //      rectangles of more than kPreBigRect tiles are counted by the whole CTA at the end
    {
        __shared__ uint4 s_big[32];  // first tile, span x, tiles
        __shared__ int s_nbig;
        if (tid == 0) s_nbig = 0;
        __syncthreads();
        uint32_t cnt = tcount;
        const int tx0 = vis ? p.x0 / BSR_TILE : 0, ty0 = vis ? p.y0 / BSR_TILE : 0;
        const int spanx = vis ? p.x1 / BSR_TILE - tx0 + 1 : 1;
        uint32_t own_big = 0;
        if (cnt > kPreBigRect) {
            const int slot = atomicAdd(&s_nbig, 1);
            if (slot < 32) s_big[slot] = make_uint4((uint32_t)(ty0 * f.tiles_x + tx0), (uint32_t)spanx, cnt, 0u);
            else own_big = cnt;
            cnt = 0;
        }
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t b = 0; b < total; b += 32) {
            const uint32_t e = b + lane;
            int lo = 0;
#pragma unroll
            for (int sft = 16; sft; sft >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, lo + sft - 1);
                if (v <= e) lo += sft;
            }
            const int owner = min(lo, 31);
            const uint32_t oin = __shfl_sync(0xffffffffu, incl, owner);
            const uint32_t ocnt = __shfl_sync(0xffffffffu, cnt, owner);
            const int otx = __shfl_sync(0xffffffffu, tx0, owner), oty = __shfl_sync(0xffffffffu, ty0, owner);
            const int osp = __shfl_sync(0xffffffffu, spanx, owner);
            if (e >= total) continue;
            const uint32_t local = e - (oin - ocnt), row = local / (uint32_t)osp;
            atomicAdd(tile_cnt_at(f, (uint32_t)(oty + (int)row) * (uint32_t)f.tiles_x + (uint32_t)otx + (local - row * osp)), 1u);
        }
        unsigned ob = __ballot_sync(0xffffffffu, own_big != 0);  // queue overflow: the warp itself
        while (ob) {
            const int src = __ffs(ob) - 1;
            ob &= ob - 1;
            const uint32_t bn = __shfl_sync(0xffffffffu, own_big, src);
            const int btx = __shfl_sync(0xffffffffu, tx0, src), bty = __shfl_sync(0xffffffffu, ty0, src);
            const int bsp = __shfl_sync(0xffffffffu, spanx, src);
            for (uint32_t j = lane; j < bn; j += 32) {
                const uint32_t row = j / (uint32_t)bsp;
                atomicAdd(tile_cnt_at(f, (uint32_t)(bty + (int)row) * (uint32_t)f.tiles_x + (uint32_t)btx + (j - row * bsp)), 1u);
            }
        }
        __syncthreads();
        const int nbig = min(s_nbig, 32);
        for (int q = 0; q < nbig; ++q) {
            const uint32_t t0 = s_big[q].x, bsp = s_big[q].y, bn = s_big[q].z;
            for (uint32_t j = tid; j < bn; j += kPreThreads) {
                const uint32_t row = j / bsp;
                atomicAdd(tile_cnt_at(f, t0 + row * (uint32_t)f.tiles_x + (j - row * bsp)), 1u);
            }
        }
    }
    if (vis) {
        const int64_t c = i;
        f.rec[c] = r;
        double4 *d = reinterpret_cast<double4 *>(f.rec64 + kRec64 * (int64_t)c);
        d[0] = make_double4(m64[0], m64[1], m64[2], m64[3]);
        d[1] = make_double4(m64[4], m64[5], m64[6], m64[7]);
        f.dkeys[0][c] = key32;
        f.dkey64[c] = key;
    }
}

template <int CM, int NT>
static int launch_pre_k(const PreArgs &a, cudaStream_t st) {
    const size_t smem = sizeof(PreSmem<CM, NT>);
    static SmemAttrOnce attr;
    BSR_CUDA_TRY(attr.ensure(preprocess_fwd_kernel<CM, NT>, smem));
    const unsigned blocks = (unsigned)div_up(a.sc.n, NT);
    BSR_CUDA_TRY((pdl_launch(preprocess_fwd_kernel<CM, NT>, dim3(blocks), dim3(NT), smem, st, a)));
    return BSR_OK;
}

int launch_preprocess(const bsr_scene &sc, const KCam &cam, const FrameView &f, cudaStream_t st) {
    if (sc.n == 0) return BSR_OK;
    PreArgs a{sc, cam, f};
    int rc = BSR_OK;
    const bool small = sc.n <= kPreSmallMaxN;
#define BSR_PRE_LAUNCH(CM) rc = small ? launch_pre_k<CM, 128>(a, st) : launch_pre_k<CM, 256>(a, st)
    BSR_DISPATCH_CM(sc, BSR_PRE_LAUNCH);
#undef BSR_PRE_LAUNCH
    if (rc) return rc;
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
