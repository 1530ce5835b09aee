// K1+K2 preprocess: fp64 EWA projection (primitive.py:221-277), SH colour
// (appearance.py:235-261 via the SH adapter), opacity / Beta exponent, and an
// order-preserving compaction of the visible subset (the reference's
// ``idx = nonzero(vis)[keep]``) in ONE pass with decoupled look-back.
//
// Compiled with -fmad=false: the fp64 integer outputs (bounds, depth keys) must follow
// the reference's rounding, and replay.cu recomputes the same primitives bit-identically.
//
// HBM roofline: N*(48 + 12K) B read, V*(64 + 8 + 4 + 4) B written.
#include "frame.cuh"
#include "project.cuh"

namespace bsr {

struct PreArgs {
    bsr_scene sc;
    KCam cam;
    FrameView f;
};

// Bound on |r2_fp32 - r2_exact| for any pixel of the footprint (r2 <= 1), accounting for
// the fp32 rounding of the record (mean relative to the bounds corner, conic) and of the
// r2 evaluation in eval_pair (raster.cuh):  eps * (8 S + 3 (GX + GY)) with
//   S  = |a| ex^2 + 2|b| ex ey + |c| ey^2            (|terms| of the quadratic form)
//   GX = (|a| ex + |b| ey)(2 ex + 3), GY = (|b| ex + |c| ey)(2 ey + 3)  (d r2 / d mean x
//        the mean's representation error, |mean - corner| <= extent + 2)
__device__ __forceinline__ double r2_error_bound(const Proj64 &p) {
    const double ex = sqrt(p.c00), ey = sqrt(p.c11);
    const double a = fabs(p.ca), b = fabs(p.cb), c = fabs(p.cc);
    const double S = a * ex * ex + 2.0 * b * ex * ey + c * ey * ey;
    const double GX = (a * ex + b * ey) * (2.0 * ex + 3.0);
    const double GY = (b * ex + c * ey) * (2.0 * ey + 3.0);
    return 5.9604644775390625e-08 * (8.0 * S + 3.0 * (GX + GY)) * 1.5;
}

template <int K>
__device__ __forceinline__ void load_sh(const float *sh, int64_t i, float *dst) {
    const float *p = sh + i * (int64_t)K * 3;
    if ((K * 3) % 4 == 0 && (reinterpret_cast<uintptr_t>(sh) & 15) == 0) {
        const float4 *p4 = reinterpret_cast<const float4 *>(p);
#pragma unroll
        for (int j = 0; j < K * 3 / 4; ++j) {
            float4 v = __ldg(p4 + j);
            dst[4 * j] = v.x;
            dst[4 * j + 1] = v.y;
            dst[4 * j + 2] = v.z;
            dst[4 * j + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < K * 3; ++j) dst[j] = __ldg(p + j);
    }
}

template <int K>
__global__ void __launch_bounds__(BSR_BLOCK) preprocess_fwd_kernel(PreArgs args) {
    const FrameView &f = args.f;
    __shared__ uint32_t s_part, s_warp[BSR_BLOCK / 32], s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_part = atomicAdd(&f.ctr->pre_ticket, 1u);
    __syncthreads();
    const int64_t part = s_part;
    const int64_t i = part * BSR_BLOCK + tid;
    const int64_t n = args.sc.n;

    bool vis = false;
    Record r;
    uint64_t key = 0;
    uint32_t key32 = 0;
    bool unsafe = false;
    double m64[5];
    uint32_t tcount = 0;
    if (i < n) {
        float pos[3] = {__ldg(args.sc.positions + 3 * i), __ldg(args.sc.positions + 3 * i + 1),
                        __ldg(args.sc.positions + 3 * i + 2)};
        float q[4] = {__ldg(args.sc.rotations + 4 * i), __ldg(args.sc.rotations + 4 * i + 1),
                      __ldg(args.sc.rotations + 4 * i + 2), __ldg(args.sc.rotations + 4 * i + 3)};
        float ls[3] = {__ldg(args.sc.log_scales + 3 * i), __ldg(args.sc.log_scales + 3 * i + 1),
                       __ldg(args.sc.log_scales + 3 * i + 2)};
        Proj64 p = project64(pos, q, ls, args.cam);
        if (p.degenerate) raise_status(&f.ctr->status, BSR_ERR_DEGENERATE_QUAT);
        if (p.visible) {
            vis = true;
            float shv[3 * K];
            load_sh<K>(args.sc.sh, i, shv);
            double rgb[3];
            sh_color64<K>(shv, pos, args.cam, rgb);
            const double o = sigmoid64((double)__ldg(args.sc.opacity_raw + i));
            const double beta = shape_to_exponent64((double)__ldg(args.sc.shapes + i));
            r.a = make_float4((float)(p.mx - p.x0), (float)(p.my - p.y0), (float)p.ca, (float)p.cb);
            r.b = make_float4((float)p.cc, (float)o, (float)beta, (float)p.tz);
            const float kr = (float)r2_error_bound(p);
            unsafe = kr > kUnsafeR2Err;
            r.c = make_float4((float)rgb[0], (float)rgb[1], (float)rgb[2], unsafe ? -kr : kr);
            m64[0] = p.mx;
            m64[1] = p.my;
            m64[2] = p.ca;
            m64[3] = p.cb;
            m64[4] = p.cc;
            r.d = make_int4(p.x0, p.x1, p.y0, p.y1);
            key = (uint64_t)__double_as_longlong(p.tz);  // tz > 0.01: bits are monotonic
            key32 = (uint32_t)__float_as_int((float)p.tz);  // monotone rounding of tz
            tcount = (uint32_t)((p.x1 / BSR_TILE - p.x0 / BSR_TILE + 1) *
                                (p.y1 / BSR_TILE - p.y0 / BSR_TILE + 1));
        }
    }
    // block-exclusive rank of visible primitives (source order preserved)
    const uint32_t ballot = __ballot_sync(0xffffffffu, vis);
    const uint32_t local = __popc(ballot & ((1u << lane) - 1));
    if (lane == 0) s_warp[warp] = __popc(ballot);
    // min depth key for the radix plan: max of the complement
    const uint32_t inv = __reduce_max_sync(0xffffffffu, vis ? ~key32 : 0u);
    if (lane == 0 && inv) atomicMax(&f.ctr->depth_key_max_inv, inv);
    __syncthreads();
    if (tid == 0) {
        uint32_t run = 0;
        for (int w = 0; w < BSR_BLOCK / 32; ++w) {
            uint32_t c = s_warp[w];
            s_warp[w] = run;
            run += c;
        }
        const uint32_t total = run;
        if (part == 0) {
            st_release(f.pre_status, kFlagPrefix | total);
            s_excl = 0;
        } else {
            st_release(f.pre_status + part, kFlagAgg | total);
            const uint32_t excl = lookback_exclusive(f.pre_status, (int)part);
            st_release(f.pre_status + part, kFlagPrefix | (excl + total));
            s_excl = excl;
        }
        if (part == f.pre_parts - 1) f.ctr->visible = s_excl + total;
    }
    __syncthreads();
    if (vis) {
        const uint32_t c = s_excl + s_warp[warp] + local;
        f.rec[c] = r;
        f.src_of[c] = (uint32_t)i;
        if (unsafe) {
            double *d = f.rec64 + 6 * (int64_t)c;
            for (int q = 0; q < 5; ++q) d[q] = m64[q];
        }
        f.dkeys[0][c] = key32;
        f.dkey64[c] = key;
        f.dvals[0][c] = c;
        f.tile_count[c] = tcount;
    }
}

int launch_preprocess(const bsr_scene &sc, const KCam &cam, const FrameView &f, cudaStream_t st) {
    if (sc.n == 0) return BSR_OK;
    PreArgs a{sc, cam, f};
    switch (sc.sh_coeffs) {
        case 1: preprocess_fwd_kernel<1><<<(unsigned)f.pre_parts, BSR_BLOCK, 0, st>>>(a); break;
        case 4: preprocess_fwd_kernel<4><<<(unsigned)f.pre_parts, BSR_BLOCK, 0, st>>>(a); break;
        case 9: preprocess_fwd_kernel<9><<<(unsigned)f.pre_parts, BSR_BLOCK, 0, st>>>(a); break;
        case 16: preprocess_fwd_kernel<16><<<(unsigned)f.pre_parts, BSR_BLOCK, 0, st>>>(a); break;
        default: return BSR_ERR_BAD_ARG;
    }
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
