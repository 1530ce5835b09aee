#include <stdlib.h>
// C-ABI entry points of libbsr.so (declared in include/bsr.h): stream-ordered
// orchestration of the kernels.  No allocation, no host sync except bsr_frame_status.
#include <math.h>
#include <string.h>

#include "frame.cuh"
#include "raster.cuh"

namespace bsr {
// kernel launchers (one per translation unit)
int launch_preprocess(const bsr_scene &, const KCam &, const FrameView &, cudaStream_t);
int launch_depth_sort(const FrameView &, cudaStream_t);
int launch_bin_count(const FrameView &, cudaStream_t);
int launch_raster_count(const FrameView &, int32_t *, const float[3], float, float, cudaStream_t);
int launch_bin_scatter(const FrameView &, cudaStream_t);
int launch_tile_sort(const FrameView &, cudaStream_t);
int launch_raster_fwd(const FrameView &, const bsr_outputs &, const float bg[3], float, float,
                      const uint32_t *, const uint2 *, const Record *, unsigned long long *,
                      cudaStream_t);
int launch_raster_bwd(const FrameView &, const float *, bool, const float *, const float bg[3],
                      float, const uint32_t *, const uint2 *, const Record *, unsigned long long *,
                      cudaStream_t);
int launch_replay_scene(bool, const FrameView &, const bsr_scene &, const KCam &, const bsr_outputs &,
                        const double bg[3], double, double, const float *, const float *,
                        cudaStream_t);
int launch_replay_arrays(bool, const FrameView &, const double *, const double *, const double *,
                         const double *, const double *, const int32_t *, const uint32_t *,
                         const uint2 *, const bsr_outputs &, const double bg[3], double, double,
                         const float *, cudaStream_t);
int launch_preprocess_bwd(const bsr_scene &, const KCam &, const FrameView &, const bsr_grads &,
                          float *, float4 *, cudaStream_t);
int launch_color_views(const bsr_scene &, const bsr_grads &, const float4 *, const double *, int, cudaStream_t);

constexpr double kAlphaMin = 1.0 / 255.0;  // rasterizer.py:28
constexpr double kTStop = 1e-4;            // rasterizer.py:29

// raster-gradient accumulators of the visible primitives (3 float4 each)
__global__ void zero_acc_kernel(FrameView f) {
    pdl_wait();
    const int64_t n3 = f.n * (kGradStride / 4);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n3; q += (int64_t)gridDim.x * blockDim.x)
        if (f.tile_count[q / (kGradStride / 4)])
            reinterpret_cast<float4 *>(f.grad_acc)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ---- core seam helpers ------------------------------------------------------------
struct CoreView {
    FrameView f;
    uint32_t *lists;
    uint2 *ranges;
    uint64_t bytes;
};

inline CoreView carve_core(void *base, int64_t v, int W, int H, int64_t e) {
    // reuse the frame layout for the per-pixel state + records, add lists/ranges
    CoreView c;
    c.f = carve_frame(base, v, W, H, 0);
    uint64_t off = c.f.total_bytes;
    char *b = static_cast<char *>(base);
    c.lists = b ? (uint32_t *)(b + off) : nullptr;
    off = align_up(off + 4ull * (e > 0 ? e : 1), 256);
    c.ranges = b ? (uint2 *)(b + off) : nullptr;
    off = align_up(off + 8ull * c.f.n_tiles, 256);
    c.bytes = off;
    return c;
}

__global__ void core_pack_kernel(int64_t v, const double *means, const double *conics,
                                 const double *opac, const double *betas, const double *colors,
                                 const int32_t *bounds, Record *rec, double *rec64, float4 *needle,
                                 double *side64) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= v) return;
    const int x0 = bounds[4 * k], x1 = bounds[4 * k + 1], y0 = bounds[4 * k + 2], y1 = bounds[4 * k + 3];
    Record r;
    // factored conic + r2 error coefficient as in preprocess.cu (extents from the conic's inverse)
    const double ca = conics[3 * k], cb = conics[3 * k + 1], cc = conics[3 * k + 2];
    double l11, l21, l22;
    const bool pd = conic_cholesky(ca, cb, cc, l11, l21, l22);
    r.a = make_float4((float)(means[2 * k] - x0), (float)(means[2 * k + 1] - y0), (float)l11, (float)l21);
    r.b = make_float4((float)l22, (float)opac[k], (float)betas[k], 0.f);
    const double det = ca * cc - cb * cb;
    const double ex = det > 0 ? sqrt(fabs(cc / det)) : 1e30, ey = det > 0 ? sqrt(fabs(ca / det)) : 1e30;
    const double kr = pd ? chol_r2_error_bound(l11, l21, l22, ex + 2.0, ey + 2.0) : 1.0;
    const bool unsafe = !pd || (float)kr > kUnsafeR2Err;
    if (unsafe) {  // core seam: fp64 path (its factor, or zeroed xy-frame fp64 accumulators)
        needle[k] = make_float4(__int_as_float(0x7fc00000), pd ? 1.f : 0.f, 0.f, 0.f);
        double *s64 = side64 + kSide64 * k;
        for (int q = 0; q < kSide64; ++q) s64[q] = 0.0;
        if (pd) {
            s64[0] = l11;
            s64[1] = l21;
            s64[2] = l22;
        }
    }
    r.c = make_float4((float)colors[3 * k], (float)colors[3 * k + 1], (float)colors[3 * k + 2],
                      record_err_word(kr, (double)r.b.z, unsafe));
    double *d = rec64 + kRec64 * k;
    d[0] = means[2 * k];
    d[1] = means[2 * k + 1];
    d[2] = ca;
    d[3] = cb;
    d[4] = cc;
    d[5] = opac[k];
    d[6] = betas[k];
    d[7] = 0.0;
    r.d = make_int4(x0, x1, y0, y1);
    rec[k] = r;
}

__global__ void core_lists_kernel(const int64_t *offsets, const int64_t *lists, int64_t e,
                                  int n_tiles, uint32_t *lists32, uint2 *ranges) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < e) lists32[i] = (uint32_t)lists[i];
    if (i < n_tiles) ranges[i] = make_uint2((uint32_t)offsets[i], (uint32_t)offsets[i + 1]);
}

__global__ void core_unpack_kernel(FrameView f, int64_t v, float *d_means, float *d_conics, float *d_opac,
                                   float *d_betas, float *d_colors) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= v) return;
    const float *g = f.grad_acc + k * kGradStride;
    double l11, l21, l22;
    if (!record_factor64(f, (uint32_t)k, l11, l21, l22)) {  // xy-frame partials summed in fp64
        const double *g64 = f.side64 + kSide64 * k;
        d_means[2 * k] = (float)g64[0];
        d_means[2 * k + 1] = (float)g64[1];
        d_conics[3 * k] = (float)g64[2];
        d_conics[3 * k + 1] = (float)g64[3];
        d_conics[3 * k + 2] = (float)g64[4];
    } else {  // whitened-frame partials (frame.cuh grad_acc): d mean = -2 L M, G = L^-T H L^-1
        const double mu = g[0], mw = g[1], h00 = g[2], h01 = g[3], h11 = g[4];
        d_means[2 * k] = (float)(-2.0 * l11 * mu);
        d_means[2 * k + 1] = (float)(-2.0 * (l21 * mu + l22 * mw));
        const double i00 = 1.0 / l11, i11 = 1.0 / l22, i10 = -l21 / (l11 * l22);
        d_conics[3 * k] = (float)(i00 * i00 * h00 + 2.0 * i00 * i10 * h01 + i10 * i10 * h11);
        d_conics[3 * k + 1] = (float)(2.0 * (i00 * h01 * i11 + i10 * h11 * i11));
        d_conics[3 * k + 2] = (float)(i11 * i11 * h11);
    }
    d_opac[k] = g[5];
    d_betas[k] = g[6];
    d_colors[3 * k] = g[7];
    d_colors[3 * k + 1] = g[8];
    d_colors[3 * k + 2] = g[9];
}

__global__ void set_visible_kernel(FrameView f, uint32_t v) { f.ctr->visible = v; }

// Per host thread and device: a side stream plus fork/join events, used to run the fp64
// replay of the flagged pixels concurrently with the fp32 raster backward (both only add
// into grad_acc; the pixels are disjoint).  Works eagerly and under stream capture (the
// fork/join become graph edges).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

inline int side_stream(SideStream **out) {
    static thread_local SideStream per_dev[64];
    int dev = 0;
    BSR_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return BSR_ERR_CUDA;
    SideStream &ss = per_dev[dev];
    if (!ss.s) {
        // highest priority: the latency-bound replay CTAs are dispatched as soon as raster
        // CTAs retire instead of queueing behind the whole raster grid
        int lo = 0, hi = 0;
        BSR_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        BSR_CUDA_TRY(cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, hi));
        BSR_CUDA_TRY(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
        BSR_CUDA_TRY(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
    }
    *out = &ss;
    return BSR_OK;
}

inline int mark(const bsr_profile *p, int i, cudaStream_t st) {
    if (p && p->events[i]) BSR_CUDA_TRY(cudaEventRecord((cudaEvent_t)p->events[i], st));
    return BSR_OK;
}

}  // namespace bsr

using namespace bsr;

namespace bsr {
bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("BSR_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}
}  // namespace bsr

static bool bad_camera(const bsr_camera *c) {
    return !c || c->width < 1 || c->height < 1 || !(c->fx > 0) || !(c->fy > 0);
}

static bool bad_scene(const bsr_scene *s) {
    if (!s || s->n < 0 || s->n >= (1ll << 31)) return true;
    if (reinterpret_cast<uintptr_t>(s->view_rgb) & 15) return true;
    if (s->n > 0 && (!s->positions || !s->rotations || !s->log_scales || !s->opacity_raw || !s->shapes))
        return true;
    if (s->color_model == BSR_COLOR_SB) {
        if (s->lobes < 0 || s->lobes > BSR_MAX_LOBES) return true;
        if (s->n > 0 && (!s->base_colors || (s->lobes > 0 && (!s->lobe_axes || !s->lobe_colors)))) return true;
        return false;
    }
    if (s->color_model != BSR_COLOR_SH) return true;
    if (!(s->sh_coeffs == 1 || s->sh_coeffs == 4 || s->sh_coeffs == 9 || s->sh_coeffs == 16)) return true;
    return s->n > 0 && !s->sh;
}

static bool bad_grads(const bsr_scene *s, const bsr_grads *g) {
    if (!g) return true;
    if (s->n == 0) return false;
    if (!g->positions || !g->rotations || !g->log_scales || !g->opacity_raw || !g->shapes) return true;
    if (s->color_model == BSR_COLOR_SB)
        return !g->base_colors || (s->lobes > 0 && (!g->lobe_axes || !g->lobe_colors));
    return !g->sh;
}

extern "C" int bsr_version(int32_t *major, int32_t *minor) {
    if (major) *major = 0;
    if (minor) *minor = 1;
    return BSR_OK;
}

extern "C" const char *bsr_status_string(int32_t s) {
    switch (s) {
        case BSR_OK: return "ok";
        case BSR_ERR_BAD_ARG: return "bad argument (shape / dtype / size)";
        case BSR_ERR_CAPACITY: return "tile-entry capacity exceeded";
        case BSR_ERR_CUDA: return "CUDA error";
        case BSR_ERR_DEGENERATE_QUAT: return "quaternion norm below 1e-12";
        case BSR_ERR_FRAME_TOO_SMALL: return "frame buffer too small";
        default: return "unknown status";
    }
}

extern "C" int bsr_frame_bytes(int64_t n, int32_t width, int32_t height, int64_t entry_cap,
                               uint64_t *bytes) {
    if (!bytes || n < 0 || width < 1 || height < 1 || entry_cap < 0 || entry_cap >= (1ll << 31))
        return BSR_ERR_BAD_ARG;
    *bytes = carve_frame(nullptr, n, width, height, entry_cap).total_bytes;
    return BSR_OK;
}

extern "C" int bsr_forward(const bsr_scene *scene, const bsr_camera *camera, const float background[3],
                           void *frame, uint64_t frame_bytes, int64_t entry_cap,
                           const bsr_outputs *out, const bsr_profile *prof, void *stream) {
    if (bad_scene(scene) || bad_camera(camera) || !background || !frame || !out ||
        entry_cap < 0 || entry_cap >= (1ll << 31))
        return BSR_ERR_BAD_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const FrameView f = carve_frame(frame, scene->n, camera->width, camera->height, entry_cap);
    if (frame_bytes < f.total_bytes) return BSR_ERR_FRAME_TOO_SMALL;
    const KCam cam = make_kcam(*camera);
    int rc;
    unsigned long long *stats = prof ? prof->stats : nullptr;
    if ((rc = mark(prof, 0, st))) return rc;
    BSR_CUDA_TRY(cudaMemsetAsync(frame, 0, f.zero_bytes, st));
    if ((rc = launch_preprocess(*scene, cam, f, st))) return rc;
    if ((rc = mark(prof, 1, st))) return rc;
    if ((rc = launch_bin_count(f, st))) return rc;
    if ((rc = mark(prof, 2, st))) return rc;
    if ((rc = launch_bin_scatter(f, st))) return rc;
    if ((rc = mark(prof, 3, st))) return rc;
    if ((rc = launch_tile_sort(f, st))) return rc;
    if ((rc = mark(prof, 4, st))) return rc;
    bsr_outputs out_raster = *out;  // deferred contributions: the replay counts its part now
    if (out->defer_contributions) out_raster.contributions = nullptr;
    if ((rc = launch_raster_fwd(f, out_raster, background, (float)kAlphaMin, (float)kTStop, nullptr, nullptr,
                                nullptr, stats, st)))
        return rc;
    if ((rc = mark(prof, 5, st))) return rc;
    const double bg64[3] = {background[0], background[1], background[2]};
    if ((rc = launch_replay_scene(true, f, *scene, cam, *out, bg64, kAlphaMin, kTStop, nullptr, nullptr, st)))
        return rc;
    return mark(prof, 6, st);
}

extern "C" int bsr_frame_status(const void *frame, bsr_frame_info *info, void *stream) {
    if (!frame || !info) return BSR_ERR_BAD_ARG;
    Counters c;
    BSR_CUDA_TRY(cudaMemcpyAsync(&c, frame, sizeof(Counters), cudaMemcpyDeviceToHost,
                                 (cudaStream_t)stream));
    BSR_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    info->visible = c.visible;
    info->entries = c.entries;
    info->entries_needed = (int64_t)c.entries_needed;
    info->flagged_pixels = c.flagged;
    info->status = c.status;
    info->reserved = 0;
    return c.status;
}

namespace bsr {
int launch_view_colors(const bsr_scene &sc, const double *centers, int views, float *rgb, cudaStream_t st);
}

extern "C" int bsr_view_colors(const bsr_scene *scene, const double *centers, int32_t views, float *rgb,
                               void *stream) {
    if (bad_scene(scene) || views < 0 || (views > 0 && (!centers || !rgb)) ||
        (reinterpret_cast<uintptr_t>(rgb) & 15))
        return BSR_ERR_BAD_ARG;
    return launch_view_colors(*scene, centers, views, rgb, (cudaStream_t)stream);
}

extern "C" int bsr_frame_snapshot_bytes(uint64_t *bytes) {
    if (!bytes) return BSR_ERR_BAD_ARG;
    *bytes = sizeof(Counters);
    return BSR_OK;
}

extern "C" int bsr_frame_status_async(const void *frame, void *snapshot, void *stream) {
    if (!frame || !snapshot) return BSR_ERR_BAD_ARG;
    BSR_CUDA_TRY(cudaMemcpyAsync(snapshot, frame, sizeof(Counters), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    return BSR_OK;
}

extern "C" int bsr_frame_snapshot_decode(const void *snapshot, bsr_frame_info *info) {
    if (!snapshot || !info) return BSR_ERR_BAD_ARG;
    Counters c;
    memcpy(&c, snapshot, sizeof(Counters));
    info->visible = c.visible;
    info->entries = c.entries;
    info->entries_needed = (int64_t)c.entries_needed;
    info->flagged_pixels = c.flagged;
    info->status = c.status;
    info->reserved = 0;
    return c.status;
}

// Deterministic mode: fixed-point sums -> grad_acc (float) / side64 (the xy-frame fp64
// partials of fp64-path records without a factor), for every visible primitive.
__global__ void det_finalize_kernel(FrameView f) {
    pdl_wait();
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < f.n; c += (int64_t)gridDim.x * blockDim.x) {
        if (!f.tile_count[c]) continue;
        double l11, l21, l22;
        const bool factor = record_factor64(f, (uint32_t)c, l11, l21, l22);
        for (int k = 0; k < 11; ++k) {
            const int64_t q = (int64_t)kDetSlots * c + k;
            const uint32_t b = f.det.bound[q];
            const double v = b ? ldexp((double)(long long)f.det.acc[q], det_exp(b) - 38) : 0.0;
            if (k < 5 && !factor)
                f.side64[kSide64 * c + k] = v;
            else
                f.grad_acc[kGradStride * c + k] = (float)v;
        }
    }
}

static int backward_impl(const bsr_scene *scene, const bsr_camera *camera, const float background[3],
                         void *frame, uint64_t frame_bytes, int64_t entry_cap, const float *d_color,
                         const float *d_depth, const bsr_grads *grads, float *screen_grad_norm,
                         const bsr_profile *prof, float *drgb, void *stream, void *det_ws = nullptr) {
    if (bad_scene(scene) || bad_camera(camera) || !background || !frame || !d_color || bad_grads(scene, grads))
        return BSR_ERR_BAD_ARG;
    if (drgb && (scene->color_model != BSR_COLOR_SH || grads->overwrite)) return BSR_ERR_BAD_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const FrameView f = carve_frame(frame, scene->n, camera->width, camera->height, entry_cap);
    if (frame_bytes < f.total_bytes) return BSR_ERR_FRAME_TOO_SMALL;
    if (scene->n == 0) return BSR_OK;
    const KCam cam = make_kcam(*camera);
    int rc;
    if ((rc = mark(prof, 0, st))) return rc;
    BSR_CUDA_TRY((pdl_launch(zero_acc_kernel, dim3((unsigned)imin64(div_up(f.n * kGradStride / 4, BSR_BLOCK), 148 * 8)), dim3(BSR_BLOCK), 0, st, f)));
    BSR_LAUNCH_CHECK();
    const double bg64_[3] = {background[0], background[1], background[2]};
    if (det_ws) {
        // deterministic mode (frame.cuh DetAcc): bound pass, fixed-point pass, finalize;
        // replay and raster run in sequence on the caller's stream
        bsr_outputs none_;
        memset(&none_, 0, sizeof(none_));
        FrameView fd = f;
        fd.det.bound = static_cast<uint32_t *>(det_ws);
        fd.det.acc = reinterpret_cast<unsigned long long *>(
            static_cast<char *>(det_ws) + align_up(4ull * kDetSlots * f.n, 256));
        BSR_CUDA_TRY(cudaMemsetAsync(det_ws, 0, align_up(4ull * kDetSlots * f.n, 256) + 8ull * kDetSlots * f.n, st));
        for (int mode = 1; mode <= 2; ++mode) {
            fd.det.mode = mode;
            if ((rc = launch_replay_scene(false, fd, *scene, cam, none_, bg64_, kAlphaMin, kTStop, d_color, d_depth, st)))
                return rc;
            if ((rc = launch_raster_bwd(fd, d_color, true, d_depth, background, (float)kAlphaMin, nullptr, nullptr,
                                        nullptr, nullptr, st)))
                return rc;
        }
        BSR_CUDA_TRY((pdl_launch(det_finalize_kernel, dim3(148 * 8), dim3(BSR_BLOCK), 0, st, fd)));
        BSR_LAUNCH_CHECK();
        if ((rc = mark(prof, 1, st))) return rc;
        if ((rc = mark(prof, 2, st))) return rc;
        if ((rc = launch_preprocess_bwd(*scene, cam, f, *grads, screen_grad_norm, reinterpret_cast<float4 *>(drgb), st)))
            return rc;
        return mark(prof, 3, st);
    }
    // fork: the fp64 replay of the flagged pixels runs beside the fp32 raster backward
    SideStream *ss = nullptr;
    if ((rc = side_stream(&ss))) return rc;
    BSR_CUDA_TRY(cudaEventRecord(ss->fork, st));
    BSR_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    bsr_outputs none;
    memset(&none, 0, sizeof(none));
    const double bg64[3] = {background[0], background[1], background[2]};
    if ((rc = launch_replay_scene(false, f, *scene, cam, none, bg64, kAlphaMin, kTStop, d_color, d_depth,
                                  ss->s)))
        return rc;
    BSR_CUDA_TRY(cudaEventRecord(ss->join, ss->s));
    if ((rc = launch_raster_bwd(f, d_color, true, d_depth, background, (float)kAlphaMin, nullptr, nullptr,
                                nullptr, prof ? prof->stats : nullptr, st)))
        return rc;
    if ((rc = mark(prof, 1, st))) return rc;
    BSR_CUDA_TRY(cudaStreamWaitEvent(st, ss->join, 0));  // join
    if ((rc = mark(prof, 2, st))) return rc;
    if ((rc = launch_preprocess_bwd(*scene, cam, f, *grads, screen_grad_norm, reinterpret_cast<float4 *>(drgb), st)))
        return rc;
    return mark(prof, 3, st);
}

extern "C" int bsr_contributions(const bsr_scene *scene, const bsr_camera *camera, const float background[3],
                                 void *frame, uint64_t frame_bytes, int64_t entry_cap, int32_t *contributions,
                                 void *stream) {
    if (bad_scene(scene) || bad_camera(camera) || !background || !frame || !contributions || entry_cap < 0 ||
        entry_cap >= (1ll << 31))
        return BSR_ERR_BAD_ARG;
    const FrameView f = carve_frame(frame, scene->n, camera->width, camera->height, entry_cap);
    if (frame_bytes < f.total_bytes) return BSR_ERR_FRAME_TOO_SMALL;
    if (scene->n == 0) return BSR_OK;
    return launch_raster_count(f, contributions, background, (float)kAlphaMin, (float)kTStop, (cudaStream_t)stream);
}

extern "C" int bsr_det_workspace_bytes(int64_t n, uint64_t *bytes) {
    if (!bytes || n < 0) return BSR_ERR_BAD_ARG;
    *bytes = align_up(4ull * kDetSlots * (uint64_t)n, 256) + 8ull * kDetSlots * (uint64_t)n;
    return BSR_OK;
}

extern "C" int bsr_backward_deterministic(const bsr_scene *scene, const bsr_camera *camera,
                                          const float background[3], void *frame, uint64_t frame_bytes,
                                          int64_t entry_cap, const float *d_color, const float *d_depth,
                                          const bsr_grads *grads, float *screen_grad_norm, float *drgb,
                                          void *det_ws, uint64_t det_ws_bytes, void *stream) {
    uint64_t need = 0;
    if (!det_ws || bsr_det_workspace_bytes(scene ? scene->n : 0, &need) || det_ws_bytes < need ||
        (reinterpret_cast<uintptr_t>(det_ws) & 255) || (drgb && (reinterpret_cast<uintptr_t>(drgb) & 15)))
        return BSR_ERR_BAD_ARG;
    return backward_impl(scene, camera, background, frame, frame_bytes, entry_cap, d_color, d_depth, grads,
                         screen_grad_norm, nullptr, drgb, stream, det_ws);
}

extern "C" int bsr_backward(const bsr_scene *scene, const bsr_camera *camera, const float background[3],
                            void *frame, uint64_t frame_bytes, int64_t entry_cap, const float *d_color,
                            const float *d_depth, const bsr_grads *grads, float *screen_grad_norm,
                            const bsr_profile *prof, void *stream) {
    return backward_impl(scene, camera, background, frame, frame_bytes, entry_cap, d_color, d_depth, grads,
                         screen_grad_norm, prof, nullptr, stream);
}

extern "C" int bsr_backward_deferred_color(const bsr_scene *scene, const bsr_camera *camera,
                                           const float background[3], void *frame, uint64_t frame_bytes,
                                           int64_t entry_cap, const float *d_color, const float *d_depth,
                                           const bsr_grads *grads, float *screen_grad_norm,
                                           const bsr_profile *prof, float *drgb, void *stream) {
    if (!drgb || (reinterpret_cast<uintptr_t>(drgb) & 15)) return BSR_ERR_BAD_ARG;
    return backward_impl(scene, camera, background, frame, frame_bytes, entry_cap, d_color, d_depth, grads,
                         screen_grad_norm, prof, drgb, stream);
}

extern "C" int bsr_color_grad_views(const bsr_scene *scene, const float *drgb, const double *centers,
                                    int32_t views, const bsr_grads *grads, void *stream) {
    if (bad_scene(scene) || bad_grads(scene, grads) || scene->color_model != BSR_COLOR_SH || views < 0 ||
        (views > 0 && (!drgb || !centers)) || (reinterpret_cast<uintptr_t>(drgb) & 15))
        return BSR_ERR_BAD_ARG;
    return launch_color_views(*scene, *grads, reinterpret_cast<const float4 *>(drgb), centers, views,
                              (cudaStream_t)stream);
}

// ---- core seam ---------------------------------------------------------------------
extern "C" int bsr_core_scratch_bytes(int64_t v, int32_t width, int32_t height, int64_t n_entries,
                                      uint64_t *bytes) {
    if (!bytes || v < 0 || width < 1 || height < 1 || n_entries < 0) return BSR_ERR_BAD_ARG;
    *bytes = carve_core(nullptr, v, width, height, n_entries).bytes;
    return BSR_OK;
}

static int core_prepare(const CoreView &c, int64_t v, const double *means, const double *conics,
                        const double *opac, const double *betas, const double *colors,
                        const int32_t *bounds, const int64_t *offsets, const int64_t *lists,
                        int64_t n_entries, cudaStream_t st) {
    BSR_CUDA_TRY(cudaMemsetAsync(c.f.ctr, 0, c.f.zero_bytes, st));
    if (v > 0)
        core_pack_kernel<<<(unsigned)div_up(v, BSR_BLOCK), BSR_BLOCK, 0, st>>>(v, means, conics, opac, betas,
                                                                               colors, bounds, c.f.rec, c.f.rec64, c.f.needle, c.f.side64);
    const int64_t m = imax64(n_entries, c.f.n_tiles);
    core_lists_kernel<<<(unsigned)div_up(imax64(m, 1), BSR_BLOCK), BSR_BLOCK, 0, st>>>(
        offsets, lists, n_entries, c.f.n_tiles, c.lists, c.ranges);
    set_visible_kernel<<<1, 1, 0, st>>>(c.f, (uint32_t)v);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_core_forward_tiled(int64_t v, const double *means, const double *conics,
                                      const double *opac, const double *betas, const double *colors,
                                      const int32_t *bounds, int32_t height, int32_t width,
                                      const double background[3], int32_t tile_size,
                                      const int64_t *offsets, const int64_t *lists, int64_t n_entries,
                                      double alpha_min, double t_stop, float *raw, float *transmittance,
                                      int32_t *contrib, int32_t *pixel_count, void *scratch,
                                      uint64_t scratch_bytes, int64_t *flagged_out, void *stream) {
    if (tile_size != BSR_TILE || v < 0 || v >= (1ll << 31) || height < 1 || width < 1 || !background ||
        !offsets || (n_entries > 0 && !lists) || !scratch)
        return BSR_ERR_BAD_ARG;
    const CoreView c = carve_core(scratch, v, width, height, n_entries);
    if (scratch_bytes < c.bytes) return BSR_ERR_FRAME_TOO_SMALL;
    cudaStream_t st = (cudaStream_t)stream;
    int rc;
    if ((rc = core_prepare(c, v, means, conics, opac, betas, colors, bounds, offsets, lists, n_entries, st)))
        return rc;
    bsr_outputs out;
    memset(&out, 0, sizeof(out));
    out.raw = raw;
    out.transmittance = transmittance;
    out.contributions = contrib;
    out.pixel_count = pixel_count;
    const float bg[3] = {(float)background[0], (float)background[1], (float)background[2]};
    if ((rc = launch_raster_fwd(c.f, out, bg, (float)alpha_min, (float)t_stop, c.lists, c.ranges, c.f.rec, nullptr, st)))
        return rc;
    if ((rc = launch_replay_arrays(true, c.f, means, conics, opac, betas, colors, bounds, c.lists, c.ranges,
                                   out, background, alpha_min, t_stop, nullptr, st)))
        return rc;
    if (flagged_out) {
        Counters h;
        BSR_CUDA_TRY(cudaMemcpyAsync(&h, c.f.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
        BSR_CUDA_TRY(cudaStreamSynchronize(st));
        *flagged_out = h.flagged;
    }
    return BSR_OK;
}

extern "C" int bsr_core_backward(int64_t v, const double *means, const double *conics, const double *opac,
                                 const double *betas, const double *colors, const int32_t *bounds,
                                 int32_t height, int32_t width, const double background[3],
                                 const float *d_raw, int32_t tile_size, const int64_t *offsets,
                                 const int64_t *lists, int64_t n_entries, double alpha_min, double t_stop,
                                 float *d_means, float *d_conics, float *d_opac, float *d_betas,
                                 float *d_colors, void *scratch, uint64_t scratch_bytes, void *stream) {
    if (tile_size != BSR_TILE || v < 0 || v >= (1ll << 31) || height < 1 || width < 1 || !background ||
        !offsets || (n_entries > 0 && !lists) || !scratch || !d_raw)
        return BSR_ERR_BAD_ARG;
    const CoreView c = carve_core(scratch, v, width, height, n_entries);
    if (scratch_bytes < c.bytes) return BSR_ERR_FRAME_TOO_SMALL;
    cudaStream_t st = (cudaStream_t)stream;
    int rc;
    if ((rc = core_prepare(c, v, means, conics, opac, betas, colors, bounds, offsets, lists, n_entries, st)))
        return rc;
    // replay the forward to recover the saved per-pixel state (the reference core
    // recomputes the forward inside backward too, _raster.pyx:191-241)
    bsr_outputs none;
    memset(&none, 0, sizeof(none));
    const float bg[3] = {(float)background[0], (float)background[1], (float)background[2]};
    if ((rc = launch_raster_fwd(c.f, none, bg, (float)alpha_min, (float)t_stop, c.lists, c.ranges, c.f.rec, nullptr,
                                st)))
        return rc;
    if ((rc = launch_replay_arrays(true, c.f, means, conics, opac, betas, colors, bounds, c.lists, c.ranges,
                                   none, background, alpha_min, t_stop, nullptr, st)))
        return rc;
    if (v > 0)
        BSR_CUDA_TRY(cudaMemsetAsync(c.f.grad_acc, 0, 4ull * kGradStride * v, st));
    if ((rc = launch_raster_bwd(c.f, d_raw, false, nullptr, bg, (float)alpha_min, c.lists, c.ranges, c.f.rec,
                                nullptr, st)))
        return rc;
    if ((rc = launch_replay_arrays(false, c.f, means, conics, opac, betas, colors, bounds, c.lists, c.ranges,
                                   none, background, alpha_min, t_stop, d_raw, st)))
        return rc;
    if (v > 0)
        core_unpack_kernel<<<(unsigned)div_up(v, BSR_BLOCK), BSR_BLOCK, 0, st>>>(c.f, v, d_means, d_conics, d_opac, d_betas,
                                                                                 d_colors);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

// ---- debug / parity export -----------------------------------------------------------
// The frame indexes everything by source index; the export reports the reference's batch
// (compact) indices: comp[i] = rank of visible primitive i among the visible ones.
namespace bsr {
__global__ void __launch_bounds__(1024) export_compact_kernel(FrameView f, uint32_t *comp, int32_t *src,
                                                               int32_t *bounds) {
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_carry;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) s_carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < f.n; b0 += 1024) {
        const int64_t i = b0 + t;
        const uint32_t v = (i < f.n && f.tile_count[i]) ? 1u : 0u;
        const uint32_t m = __ballot_sync(0xffffffffu, v);
        if (lane == 0) s_w[warp] = __popc(m);
        __syncthreads();
        uint32_t base = s_carry;
        for (int w = 0; w < warp; ++w) base += s_w[w];
        const uint32_t c = base + __popc(m & ((1u << lane) - 1u));
        if (v) {
            comp[i] = c;
            if (src) src[c] = (int32_t)i;
            if (bounds) {
                const int4 d = f.rec[i].d;
                bounds[4 * c] = d.x;
                bounds[4 * c + 1] = d.y;
                bounds[4 * c + 2] = d.z;
                bounds[4 * c + 3] = d.w;
            }
        }
        __syncthreads();
        if (t == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < 32; ++w) tot += s_w[w];
            s_carry += tot;
        }
        __syncthreads();
    }
}
// depth-sort inputs in compact order: keys[c] = fp32 key of its source, vals[c] = source
__global__ void export_keys_kernel(FrameView f, const uint32_t *comp) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= f.n || !f.tile_count[i]) return;
    f.dkeys[1][comp[i]] = f.dkeys[0][i];
    f.dvals[1][comp[i]] = (uint32_t)i;
}
__global__ void export_map_kernel(const uint32_t *comp, const uint32_t *in, int32_t *out, int64_t m) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < m) out[k] = (int32_t)comp[in[k]];
}
}  // namespace bsr

extern "C" int bsr_debug_export(const void *frame, int64_t n, int32_t width, int32_t height,
                                int64_t entry_cap, int32_t *order, int32_t *src_index,
                                int32_t *bounds, int32_t *lists, int32_t *ranges, void *stream) {
    if (!frame || n < 0 || width < 1 || height < 1) return BSR_ERR_BAD_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const FrameView f = carve_frame(const_cast<void *>(frame), n, width, height, entry_cap);
    Counters c;
    BSR_CUDA_TRY(cudaMemcpyAsync(&c, f.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    BSR_CUDA_TRY(cudaStreamSynchronize(st));
    if (f.n == 0) return BSR_OK;
    // scratch (the gradient accumulator is zeroed by every backward before use):
    //   comp [N] | saved dkeys[0] [N] | sorted-order staging [N]
    uint32_t *comp = reinterpret_cast<uint32_t *>(f.grad_acc);
    uint32_t *saved = comp + f.n;
    uint32_t *tmp = saved + f.n;
    export_compact_kernel<<<1, 1024, 0, st>>>(f, comp, src_index, bounds);
    BSR_LAUNCH_CHECK();
    if (order && c.visible) {
        // the global depth order is not part of the per-frame binning (bin.cu sorts per
        // tile); compute it here with the onesweep depth sort over the compact keys
        BSR_CUDA_TRY(cudaMemcpyAsync(saved, f.dkeys[0], 4ull * f.n, cudaMemcpyDeviceToDevice, st));
        export_keys_kernel<<<(unsigned)div_up(f.n, BSR_BLOCK), BSR_BLOCK, 0, st>>>(f, comp);
        BSR_CUDA_TRY(cudaMemcpyAsync(f.dkeys[0], f.dkeys[1], 4ull * c.visible, cudaMemcpyDeviceToDevice, st));
        BSR_CUDA_TRY(cudaMemcpyAsync(f.dvals[0], f.dvals[1], 4ull * c.visible, cudaMemcpyDeviceToDevice, st));
        BSR_CUDA_TRY(cudaMemsetAsync(f.depth_hist, 0, 4ull * kDepthPasses * 256, st));
        BSR_CUDA_TRY(cudaMemsetAsync(f.depth_status, 0, 4ull * kDepthPasses * f.depth_parts * 256, st));
        BSR_CUDA_TRY(cudaMemsetAsync(f.ctr->depth_ticket, 0, sizeof(c.depth_ticket), st));
        BSR_CUDA_TRY(cudaMemsetAsync(f.ctr->depth_plan, 0, sizeof(c.depth_plan), st));
        int rc = launch_depth_sort(f, st);  // values: source indices; fixup reads dkey64[source]
        if (rc) return rc;
        BSR_CUDA_TRY(cudaMemcpyAsync(&c, f.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
        BSR_CUDA_TRY(cudaStreamSynchronize(st));
        BSR_CUDA_TRY(cudaMemcpyAsync(tmp, f.dvals[c.depth_plan[kDepthPasses] & 1u], 4ull * c.visible,
                                     cudaMemcpyDeviceToDevice, st));
        export_map_kernel<<<(unsigned)div_up(c.visible, BSR_BLOCK), BSR_BLOCK, 0, st>>>(comp, tmp, order, c.visible);
        BSR_CUDA_TRY(cudaMemcpyAsync(f.dkeys[0], saved, 4ull * f.n, cudaMemcpyDeviceToDevice, st));
    }
    if (lists && c.entries)
        export_map_kernel<<<(unsigned)div_up(c.entries, BSR_BLOCK), BSR_BLOCK, 0, st>>>(comp, f.lists, lists,
                                                                                       c.entries);
    if (ranges)
        BSR_CUDA_TRY(cudaMemcpyAsync(ranges, f.tile_ranges, 8ull * f.n_tiles, cudaMemcpyDeviceToDevice, st));
    BSR_LAUNCH_CHECK();
    BSR_CUDA_TRY(cudaStreamSynchronize(st));
    return BSR_OK;
}
