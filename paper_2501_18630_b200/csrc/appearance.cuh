// View-dependent colour models (appearance.py), selected at compile time by CM:
//   CM > 0   real spherical harmonics with K = CM coefficients per channel (degree <= 3),
//            sh (N, K, 3) -- the SH adapter of SURVEY 8(c), appearance.py:192-318
//   CM <= 0  Spherical Beta with M = -CM lobes (the reference's default model,
//            appearance.py:82-163): base colour (N,3), lobe axes (N,M,3) = direction *
//            exp(sharpness), lobe colours (N,M,3);  response dot(axis_hat, v)^(4 |axis|)
//            for positive dots, exactly 0 otherwise.
#pragma once

#include "common.cuh"

namespace bsr {

constexpr double kAxisEps = 1e-8;  // appearance.py:24

template <int CM>
struct AppTraits {
    static constexpr bool sh = CM > 0;
    static constexpr int K = CM > 0 ? CM : 1;
    static constexpr int M = CM > 0 ? 0 : -CM;
    // floats per primitive in the staged payload: SH 3K; SB base 3 + axes 3M + colours 3M
    static constexpr int floats = CM > 0 ? 3 * CM : 3 + 6 * (-CM);
};

// ---- fp32 evaluation from a staged payload (preprocess) --------------------------------
// SH payload: sh[3K] of this primitive.  SB payload pointers: base[3], axes[3M], cols[3M].
template <int CM>
__device__ __forceinline__ void app_color32(const float *p0, const float *p1, const float *p2, float x,
                                            float y, float z, float rgb[3]) {
    using Tr = AppTraits<CM>;
    if constexpr (Tr::sh) {
        constexpr int K = Tr::K;
        float b[16];
        b[0] = 0.28209479177387814f;
        if constexpr (K > 1) {
            const float C1 = 0.4886025119029199f;
            b[1] = -C1 * y;
            b[2] = C1 * z;
            b[3] = -C1 * x;
        }
        if constexpr (K > 4) {
            const float xx = x * x, yy = y * y, zz = z * z;
            b[4] = 1.0925484305920792f * x * y;
            b[5] = -1.0925484305920792f * y * z;
            b[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
            b[7] = -1.0925484305920792f * x * z;
            b[8] = 0.5462742152960396f * (xx - yy);
            if constexpr (K > 9) {
                b[9] = -0.5900435899266435f * y * (3.f * xx - yy);
                b[10] = 2.890611442640554f * x * y * z;
                b[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
                b[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
                b[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
                b[14] = 1.445305721320277f * z * (xx - yy);
                b[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
            }
        }
        float r = 0.f, g = 0.f, bl = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            r = __fmaf_rn(b[k], p0[3 * k], r);
            g = __fmaf_rn(b[k], p0[3 * k + 1], g);
            bl = __fmaf_rn(b[k], p0[3 * k + 2], bl);
        }
        rgb[0] = r;
        rgb[1] = g;
        rgb[2] = bl;
    } else {
        rgb[0] = p0[0];
        rgb[1] = p0[1];
        rgb[2] = p0[2];
#pragma unroll
        for (int m = 0; m < Tr::M; ++m) {
            float ax = p1[3 * m], ay = p1[3 * m + 1], az = p1[3 * m + 2];
            float nrm = sqrtf(ax * ax + ay * ay + az * az);
            if (nrm < (float)kAxisEps) {
                ax = 0.f;
                ay = 0.f;
                az = 1.f;
                nrm = 1.f;
            }
            const float w = fminf(fmaxf((ax * x + ay * y + az * z) / nrm, 0.f), 1.f);
            const float resp = w > 0.f ? exp2f(4.0f * nrm * __log2f(w)) : 0.f;
            rgb[0] = __fmaf_rn(resp, p2[3 * m], rgb[0]);
            rgb[1] = __fmaf_rn(resp, p2[3 * m + 1], rgb[1]);
            rgb[2] = __fmaf_rn(resp, p2[3 * m + 2], rgb[2]);
        }
    }
}

// ---- fp64 evaluation from global memory (fp64 replay; reference expression order) -------
template <int CM>
__device__ __forceinline__ void app_color64(const bsr_scene &sc, int64_t i, double x, double y, double z,
                                            double rgb[3]) {
    using Tr = AppTraits<CM>;
    if constexpr (Tr::sh) {
        constexpr int K = Tr::K;
        double b[16];
        const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
        b[0] = C0;
        if constexpr (K > 1) {
            b[1] = -C1 * y;
            b[2] = C1 * z;
            b[3] = -C1 * x;
        }
        if constexpr (K > 4) {
            const double xx = x * x, yy = y * y, zz = z * z;
            b[4] = 1.0925484305920792 * x * y;
            b[5] = -1.0925484305920792 * y * z;
            b[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
            b[7] = -1.0925484305920792 * x * z;
            b[8] = 0.5462742152960396 * (xx - yy);
            if constexpr (K > 9) {
                b[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
                b[10] = 2.890611442640554 * x * y * z;
                b[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
                b[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
                b[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
                b[14] = 1.445305721320277 * z * (xx - yy);
                b[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
            }
        }
        const float *sh = sc.sh + i * 3 * K;
        double r = 0.0, g = 0.0, bl = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            r += b[k] * (double)sh[3 * k];
            g += b[k] * (double)sh[3 * k + 1];
            bl += b[k] * (double)sh[3 * k + 2];
        }
        rgb[0] = r;
        rgb[1] = g;
        rgb[2] = bl;
    } else {
        constexpr int M = Tr::M;
        const float *bc = sc.base_colors + 3 * i;
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const float *ap = sc.lobe_axes + (i * M + m) * 3;
            const float *cp = sc.lobe_colors + (i * M + m) * 3;
            double ax = ap[0], ay = ap[1], az = ap[2];
            double nrm = sqrt((ax * ax + ay * ay) + az * az);
            if (nrm < kAxisEps) {
                ax = 0.0;
                ay = 0.0;
                az = 1.0;
                nrm = 1.0;
            }
            const double dot = (ax / nrm * x + ay / nrm * y) + az / nrm * z;
            const double w = fmin(fmax(dot, 0.0), 1.0);
            const double resp = w > 0.0 ? pow(w, 4.0 * nrm) : 0.0;
            acc[0] += resp * (double)cp[0];
            acc[1] += resp * (double)cp[1];
            acc[2] += resp * (double)cp[2];
        }
        rgb[0] = (double)bc[0] + acc[0];
        rgb[1] = (double)bc[1] + acc[1];
        rgb[2] = (double)bc[2] + acc[2];
    }
}

}  // namespace bsr
