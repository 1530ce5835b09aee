// K6 preprocess_bwd: per visible primitive, chain the raster gradients (grad_acc) back to
// the unconstrained parameters -- the tail of render_backward (rasterizer.py:262-320):
//   opacity sigmoid chain (:292-293), Beta exponent chain (:296-299),
//   conic -> conditioned covariance  dSigma' = -Inv G Inv  (:302-312),
//   project_backward + _rotation_grad_to_quat (primitive.py:302-367),
//   SH colour chain (appearance.py:264-318, the SH adapter of SURVEY 8(c)) and the
//   view-direction -> position chain (rasterizer.py:287-289),
//   plus the depth extension  z = R[2].p + t[2].
// Gradients are ADDED into the caller's per-parameter buffers (multi-view accumulation).
// HBM roofline: V * (48 B grad_acc + 240 B params read + 240 B grads RMW) at SH-3.
#include "appearance.cuh"
#include "frame.cuh"
#include "raster.cuh"

namespace bsr {

struct PreBwdArgs {
    bsr_scene sc;
    KCam cam;
    FrameView f;
    bsr_grads g;
    float *screen_grad_norm;
    float4 *drgb;  // deferred colour chain: (dL/dr, dL/dg, dL/db, 0) per primitive, or nullptr
};

template <int K>
__device__ __forceinline__ void sh_basis_and_grad(float x, float y, float z, float *b, float (*db)[3]) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    b[0] = C0;
    db[0][0] = db[0][1] = db[0][2] = 0.f;
    if constexpr (K > 1) {
        b[1] = -C1 * y;
        b[2] = C1 * z;
        b[3] = -C1 * x;
        db[1][0] = 0.f; db[1][1] = -C1; db[1][2] = 0.f;
        db[2][0] = 0.f; db[2][1] = 0.f; db[2][2] = C1;
        db[3][0] = -C1; db[3][1] = 0.f; db[3][2] = 0.f;
    }
    if constexpr (K > 4) {
        const float xx = x * x, yy = y * y, zz = z * z;
        const float c20 = 1.0925484305920792f, c21 = -1.0925484305920792f, c22 = 0.31539156525252005f,
                    c23 = -1.0925484305920792f, c24 = 0.5462742152960396f;
        b[4] = c20 * x * y;
        b[5] = c21 * y * z;
        b[6] = c22 * (2.f * zz - xx - yy);
        b[7] = c23 * x * z;
        b[8] = c24 * (xx - yy);
        db[4][0] = c20 * y; db[4][1] = c20 * x; db[4][2] = 0.f;
        db[5][0] = 0.f; db[5][1] = c21 * z; db[5][2] = c21 * y;
        db[6][0] = -2.f * c22 * x; db[6][1] = -2.f * c22 * y; db[6][2] = 4.f * c22 * z;
        db[7][0] = c23 * z; db[7][1] = 0.f; db[7][2] = c23 * x;
        db[8][0] = 2.f * c24 * x; db[8][1] = -2.f * c24 * y; db[8][2] = 0.f;
        if constexpr (K > 9) {
            const float c30 = -0.5900435899266435f, c31 = 2.890611442640554f, c32 = -0.4570457994644658f,
                        c33 = 0.3731763325901154f, c34 = -0.4570457994644658f, c35 = 1.445305721320277f,
                        c36 = -0.5900435899266435f;
            b[9] = c30 * y * (3.f * xx - yy);
            b[10] = c31 * x * y * z;
            b[11] = c32 * y * (4.f * zz - xx - yy);
            b[12] = c33 * z * (2.f * zz - 3.f * xx - 3.f * yy);
            b[13] = c34 * x * (4.f * zz - xx - yy);
            b[14] = c35 * z * (xx - yy);
            b[15] = c36 * x * (xx - 3.f * yy);
            db[9][0] = c30 * 6.f * x * y; db[9][1] = c30 * (3.f * xx - 3.f * yy); db[9][2] = 0.f;
            db[10][0] = c31 * y * z; db[10][1] = c31 * x * z; db[10][2] = c31 * x * y;
            db[11][0] = c32 * -2.f * x * y; db[11][1] = c32 * (4.f * zz - xx - 3.f * yy); db[11][2] = c32 * 8.f * y * z;
            db[12][0] = c33 * -6.f * x * z; db[12][1] = c33 * -6.f * y * z; db[12][2] = c33 * (6.f * zz - 3.f * xx - 3.f * yy);
            db[13][0] = c34 * (4.f * zz - 3.f * xx - yy); db[13][1] = c34 * -2.f * x * y; db[13][2] = c34 * 8.f * x * z;
            db[14][0] = c35 * 2.f * x * z; db[14][1] = c35 * -2.f * y * z; db[14][2] = c35 * (xx - yy);
            db[15][0] = c36 * (3.f * xx - 3.f * yy); db[15][1] = c36 * -6.f * x * y; db[15][2] = 0.f;
        }
    }
}

// Colour-model backward: accumulates the parameter gradients of primitive i and returns
// d rgb / d view-direction (added into ddx/ddy/ddz).
//   SH: d_sh[k,c] = basis_k d_rgb[c];  d_dir = dbasis^T (sh . d_rgb)     (appearance.py:264-318)
//   SB: sb_grad_many (appearance.py:127-163)
template <int CM>
__device__ __forceinline__ void app_backward(const bsr_scene &sc, const bsr_grads &g, int64_t i, float vx,
                                             float vy, float vz, float dr, float dg, float dbl, float &ddx,
                                             float &ddy, float &ddz, float4 *srow = nullptr) {
    const bool ovw = g.overwrite != 0;  // write instead of add (bsr_grads::overwrite)
    using Tr = AppTraits<CM>;
    if constexpr (Tr::sh) {
        constexpr int K = Tr::K;
        float b[16], db[16][3];
        sh_basis_and_grad<K>(vx, vy, vz, b, db);
        if ((3 * K) % 4 == 0 && srow) {
            // the warp staged this row (preprocess_bwd_kernel): coefficients in, coefficient
            // gradients out (overwrite mode; the warp stores the rows coalesced)
            // four coefficients = three float4 at a time
#pragma unroll
            for (int g4 = 0; g4 < K / 4; ++g4) {
                const float4 v0 = srow[3 * g4], v1 = srow[3 * g4 + 1], v2 = srow[3 * g4 + 2];
                const float sv[12] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y, v2.z, v2.w};
                float gv[12];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int k = 4 * g4 + kk;
                    const float dbk = sv[3 * kk] * dr + sv[3 * kk + 1] * dg + sv[3 * kk + 2] * dbl;
                    ddx += db[k][0] * dbk;
                    ddy += db[k][1] * dbk;
                    ddz += db[k][2] * dbk;
                    gv[3 * kk] = 0.f + b[k] * dr;
                    gv[3 * kk + 1] = 0.f + b[k] * dg;
                    gv[3 * kk + 2] = 0.f + b[k] * dbl;
                }
                srow[3 * g4] = make_float4(gv[0], gv[1], gv[2], gv[3]);
                srow[3 * g4 + 1] = make_float4(gv[4], gv[5], gv[6], gv[7]);
                srow[3 * g4 + 2] = make_float4(gv[8], gv[9], gv[10], gv[11]);
            }
            return;
        }
        // coefficients and their gradients move as float4 when a row of K*3 floats is
        // 16-byte aligned (K = 4, 16); coalescing-friendly vs 3K scalar accesses
        float shv[3 * K], gsv[3 * K];
        const float *shp = sc.sh + i * 3 * K;
        float *gsh = g.sh + i * 3 * K;
        const bool sh16 = ((reinterpret_cast<uintptr_t>(sc.sh) | reinterpret_cast<uintptr_t>(g.sh)) & 15) == 0;
        if ((3 * K) % 4 == 0 && sh16) {
#pragma unroll
            for (int q = 0; q < 3 * K / 4; ++q) {
                const float4 x4 = __ldg(reinterpret_cast<const float4 *>(shp) + q);
                const float4 g4 = ovw ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<const float4 *>(gsh)[q];
                shv[4 * q] = x4.x; shv[4 * q + 1] = x4.y; shv[4 * q + 2] = x4.z; shv[4 * q + 3] = x4.w;
                gsv[4 * q] = g4.x; gsv[4 * q + 1] = g4.y; gsv[4 * q + 2] = g4.z; gsv[4 * q + 3] = g4.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3 * K; ++q) {
                shv[q] = __ldg(shp + q);
                gsv[q] = ovw ? 0.f : gsh[q];
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            gsv[3 * k] += b[k] * dr;
            gsv[3 * k + 1] += b[k] * dg;
            gsv[3 * k + 2] += b[k] * dbl;
            const float dbk = shv[3 * k] * dr + shv[3 * k + 1] * dg + shv[3 * k + 2] * dbl;
            ddx += db[k][0] * dbk;
            ddy += db[k][1] * dbk;
            ddz += db[k][2] * dbk;
        }
        if ((3 * K) % 4 == 0 && sh16) {
#pragma unroll
            for (int q = 0; q < 3 * K / 4; ++q)
                reinterpret_cast<float4 *>(gsh)[q] =
                    make_float4(gsv[4 * q], gsv[4 * q + 1], gsv[4 * q + 2], gsv[4 * q + 3]);
        } else {
#pragma unroll
            for (int q = 0; q < 3 * K; ++q) gsh[q] = gsv[q];
        }
    } else {
        constexpr int M = Tr::M;
        auto put = [&](float *dst, float v) {
            if (ovw) *dst = v; else *dst += v;
        };
        put(g.base_colors + 3 * i, dr);  // d base = upstream
        put(g.base_colors + 3 * i + 1, dg);
        put(g.base_colors + 3 * i + 2, dbl);
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const int64_t o = (i * M + m) * 3;
            float ax = sc.lobe_axes[o], ay = sc.lobe_axes[o + 1], az = sc.lobe_axes[o + 2];
            float nrm = sqrtf(ax * ax + ay * ay + az * az);
            if (nrm < (float)kAxisEps) {  // effective axis +z (appearance.py:76-78)
                ax = 0.f;
                ay = 0.f;
                az = 1.f;
                nrm = 1.f;
            }
            const float inrm = 1.f / nrm;
            const float ux = ax * inrm, uy = ay * inrm, uz = az * inrm;
            const float w = fminf(fmaxf(ux * vx + uy * vy + uz * vz, 0.f), 1.f);
            const float expo = 4.0f * nrm;
            const float cr = sc.lobe_colors[o], cg = sc.lobe_colors[o + 1], cb = sc.lobe_colors[o + 2];
            if (!(w > 1e-12f)) {  // outside the lobe's support: exactly zero gradients
                if (ovw)
                    for (int q = 0; q < 3; ++q) g.lobe_colors[o + q] = g.lobe_axes[o + q] = 0.f;
                continue;
            }
            const float lw = __logf(w);
            const float resp = __expf(expo * lw);
            const float resp_dw = expo * __expf((expo - 1.0f) * lw);
            put(g.lobe_colors + o, resp * dr);
            put(g.lobe_colors + o + 1, resp * dg);
            put(g.lobe_colors + o + 2, resp * dbl);
            const float d_resp = dr * cr + dg * cg + dbl * cb;
            const float d_w = d_resp * resp_dw;
            const float d_norm = d_resp * resp * lw * 4.0f;
            const float dux = d_w * vx, duy = d_w * vy, duz = d_w * vz;
            const float dot = dux * ux + duy * uy + duz * uz;
            put(g.lobe_axes + o, (dux - dot * ux) * inrm + d_norm * ux);
            put(g.lobe_axes + o + 1, (duy - dot * uy) * inrm + d_norm * uy);
            put(g.lobe_axes + o + 2, (duz - dot * uz) * inrm + d_norm * uz);
            ddx += d_w * ux;
            ddy += d_w * uy;
            ddz += d_w * uz;
        }
    }
}

// Geometric chain of one primitive (primitive.py:302-367, project_backward +
// _rotation_grad_to_quat), in fp64: from d mean2d and the symmetric d cov2d (already mapped
// from the raster's conic partials) to the position / log-scale / rotation gradients.
// Adds the log-scale and rotation gradients and returns d position (without the
// view-direction part).  fp64 because the 3D covariance chain of an anisotropic primitive
// cancels: a small-axis scale gradient is a ~kappa times smaller projection of xy-frame terms.
template <typename T>
__device__ __forceinline__ void geom_chain(const PreBwdArgs &a, int64_t i, T dmx, T dmy, T gm00, T gs01, T gm11,
                                           float dz, float &dpx_out, float &dpy_out, float &dpz_out) {
    const bsr_scene &sc = a.sc;
    const KCam &cam = a.cam;
    const T px = sc.positions[3 * i], py = sc.positions[3 * i + 1], pz = sc.positions[3 * i + 2];
    T R[9];
    for (int k = 0; k < 9; ++k) R[k] = (T)cam.R[k];
    const T tx = R[0] * px + R[1] * py + R[2] * pz + (T)cam.t[0];
    const T ty = R[3] * px + R[4] * py + R[5] * pz + (T)cam.t[1];
    const T tz = R[6] * px + R[7] * py + R[8] * pz + (T)cam.t[2];
    const T fx = (T)cam.fx, fy = (T)cam.fy;
    const bool rot16 = ((reinterpret_cast<uintptr_t>(sc.rotations) | reinterpret_cast<uintptr_t>(a.g.rotations)) & 15) == 0;
    float4 q4;
    if (rot16) {
        q4 = __ldg(reinterpret_cast<const float4 *>(sc.rotations) + i);
    } else {
        q4 = make_float4(sc.rotations[4 * i], sc.rotations[4 * i + 1], sc.rotations[4 * i + 2], sc.rotations[4 * i + 3]);
    }
    // The chain's inputs (1 / |q|, exp(log_scale), 1 / t_z) come from fp32 transcendentals
    // refined by one fp64 Newton step where a quotient feeds a cancellation (relative
    // error <= ~1e-7 on an input is the fp32 parameters' own precision); the linear
    // algebra below, where the cancellations happen, runs in T.  fp64 division, sqrt and
    // exp sequences dominated the latency of the fp64 variant.
    T qw = q4.x, qx = q4.y, qy = q4.z, qz = q4.w;
    const T qq = qw * qw + qx * qx + qy * qy + qz * qz;
    T iqn = (T)rsqrtf((float)qq);
    iqn = iqn * ((T)1.5 - (T)0.5 * qq * iqn * iqn);  // Newton step on 1 / sqrt(qq)
    qw *= iqn;
    qx *= iqn;
    qy *= iqn;
    qz *= iqn;
    const T one = 1, two = 2;
    T Q[9] = {one - two * (qy * qy + qz * qz), two * (qx * qy - qw * qz), two * (qx * qz + qw * qy),
              two * (qx * qy + qw * qz), one - two * (qx * qx + qz * qz), two * (qy * qz - qw * qx),
              two * (qx * qz - qw * qy), two * (qy * qz + qw * qx), one - two * (qx * qx + qy * qy)};
    T s2[3];
    for (int k = 0; k < 3; ++k) {
        const T s = (T)expf(sc.log_scales[3 * i + k]);
        s2[k] = s * s;
    }
    T Sig[9];
    for (int r = 0; r < 3; ++r)
        for (int col = 0; col < 3; ++col)
            Sig[3 * r + col] = Q[3 * r] * s2[0] * Q[3 * col] + Q[3 * r + 1] * s2[1] * Q[3 * col + 1] +
                               Q[3 * r + 2] * s2[2] * Q[3 * col + 2];
    T itz = (T)(1.0f / (float)tz);
    itz = itz * (two - tz * itz);  // Newton step on 1 / t_z
    const T itz2 = itz * itz;
    const T J00 = fx * itz, J02 = -fx * tx * itz2, J11 = fy * itz, J12 = -fy * ty * itz2;
    T Am[6];
    for (int j = 0; j < 3; ++j) {
        Am[j] = J00 * R[j] + J02 * R[6 + j];
        Am[3 + j] = J11 * R[3 + j] + J12 * R[6 + j];
    }
    const T Gm[4] = {gm00, gs01, gs01, gm11};
    // g_sigma = A^T g_m A (3x3)
    T gS[9];
    for (int r = 0; r < 3; ++r)
        for (int col = 0; col < 3; ++col) {
            T v = 0;
            for (int u = 0; u < 2; ++u)
                for (int w = 0; w < 2; ++w) v += Am[3 * u + r] * Gm[2 * u + w] * Am[3 * w + col];
            gS[3 * r + col] = v;
        }
    // g_a = 2 g_m A Sigma (2x3); g_jac = g_a R^T
    T gA[6];
    for (int u = 0; u < 2; ++u)
        for (int j = 0; j < 3; ++j) {
            T v = 0;
            for (int w = 0; w < 2; ++w)
                for (int k = 0; k < 3; ++k) v += Gm[2 * u + w] * Am[3 * w + k] * Sig[3 * k + j];
            gA[3 * u + j] = two * v;
        }
    T gJ[6];
    for (int u = 0; u < 2; ++u)
        for (int j = 0; j < 3; ++j)
            gJ[3 * u + j] = gA[3 * u] * R[3 * j] + gA[3 * u + 1] * R[3 * j + 1] + gA[3 * u + 2] * R[3 * j + 2];
    // g_t = J^T d_mean + dJ/dt terms (primitive.py:328-337)
    T gt0 = J00 * dmx, gt1 = J11 * dmy, gt2 = J02 * dmx + J12 * dmy;
    gt0 += gJ[2] * (-fx * itz2);
    gt1 += gJ[5] * (-fy * itz2);
    gt2 += gJ[0] * (-fx * itz2) + gJ[2] * (two * fx * tx * itz2 * itz) + gJ[4] * (-fy * itz2) +
           gJ[5] * (two * fy * ty * itz2 * itz);
    gt2 += (T)dz;  // depth extension: z = t_z
    dpx_out = (float)(gt0 * R[0] + gt1 * R[3] + gt2 * R[6]);
    dpy_out = (float)(gt0 * R[1] + gt1 * R[4] + gt2 * R[7]);
    dpz_out = (float)(gt0 * R[2] + gt1 * R[5] + gt2 * R[8]);
    // Sigma = Q diag(s^2) Q^T: g_rot = 2 gS Q diag(s^2); g_d_i = (Q^T gS Q)_ii
    T gR[9];
    for (int r = 0; r < 3; ++r)
        for (int col = 0; col < 3; ++col)
            gR[3 * r + col] = two * (gS[3 * r] * Q[col] + gS[3 * r + 1] * Q[3 + col] + gS[3 * r + 2] * Q[6 + col]) * s2[col];
    for (int k = 0; k < 3; ++k) {
        T v = 0;
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) v += Q[3 * j + k] * gS[3 * j + l] * Q[3 * l + k];
        const float gls = (float)(v * two * s2[k]);
        if (a.g.overwrite) a.g.log_scales[3 * i + k] = gls; else a.g.log_scales[3 * i + k] += gls;
    }
    // _rotation_grad_to_quat (primitive.py:348-367)
    {
        const T w = qw, x = qx, y = qy, z = qz;
        const T *g = gR;
        const T gw = two * (-z * g[1] + y * g[2] + z * g[3] - x * g[5] - y * g[6] + x * g[7]);
        const T gx = two * (y * g[1] + z * g[2] + y * g[3] - two * x * g[4] - w * g[5] + z * g[6] + w * g[7] - two * x * g[8]);
        const T gy = two * (-two * y * g[0] + x * g[1] + w * g[2] + x * g[3] + z * g[5] - w * g[6] + z * g[7] - two * y * g[8]);
        const T gz = two * (-two * z * g[0] - w * g[1] + x * g[2] + w * g[3] - two * z * g[4] + y * g[5] + x * g[6] + y * g[7]);
        const T dot = gw * w + gx * x + gy * y + gz * z;
        const float r0 = (float)((gw - dot * w) * iqn), r1 = (float)((gx - dot * x) * iqn);
        const float r2 = (float)((gy - dot * y) * iqn), r3 = (float)((gz - dot * z) * iqn);
        if (rot16) {
            float4 *gr = reinterpret_cast<float4 *>(a.g.rotations) + i;
            float4 gq = a.g.overwrite ? make_float4(0.f, 0.f, 0.f, 0.f) : *gr;
            gq.x += r0;
            gq.y += r1;
            gq.z += r2;
            gq.w += r3;
            *gr = gq;
        } else {
            const bool ow = a.g.overwrite != 0;
            float *gr = a.g.rotations + 4 * i;
            gr[0] = (ow ? 0.f : gr[0]) + r0;
            gr[1] = (ow ? 0.f : gr[1]) + r1;
            gr[2] = (ow ? 0.f : gr[2]) + r2;
            gr[3] = (ow ? 0.f : gr[3]) + r3;
        }
    }
}

template <int K>
__device__ __forceinline__ void prebwd_one(const PreBwdArgs &a, int64_t c, float4 *srow = nullptr) {
    const float *acc = a.f.grad_acc + (int64_t)c * kGradStride;
    const float4 g1 = *reinterpret_cast<const float4 *>(acc + 4);
    const float4 g2 = *reinterpret_cast<const float4 *>(acc + 8);
    const float d_o = g1.y, d_beta = g1.z;
    const float dr = g1.w, dg = g2.x, dbl = g2.y;
    const int64_t i = c;
    const bsr_scene &sc = a.sc;
    const KCam &cam = a.cam;

    // ---- opacity / shape chains
    const float oraw = sc.opacity_raw[i];
    const float o = oraw >= 0.f ? 1.f / (1.f + expf(-oraw)) : expf(oraw) / (1.f + expf(oraw));
    const bool ovw = a.g.overwrite != 0;
    const float gop = d_o * o * (1.f - o);
    if (ovw) a.g.opacity_raw[i] = gop; else a.g.opacity_raw[i] += gop;
    const float bsh = sc.shapes[i];
    const float beta = 4.f * expf(fminf(fmaxf(bsh, -10.f), 10.f));
    const float gsp = fabsf(bsh) <= 10.f ? d_beta * beta : 0.f;
    if (ovw) a.g.shapes[i] = gsp; else a.g.shapes[i] += gsp;

    // ---- the geometric chain runs in fp64 in prebwd_geom_kernel (after this kernel)
    float dpx = 0.f, dpy = 0.f, dpz = 0.f;
    const float px = sc.positions[3 * i], py = sc.positions[3 * i + 1], pz = sc.positions[3 * i + 2];
    // ---- colour chain (SH or Spherical Beta) + view direction -> position; deferred for
    //      multi-view steps (bsr_color_grad_views applies every view's chain at once)
    if (a.drgb) {
        a.drgb[i] = make_float4(dr, dg, dbl, 0.f);
    } else {
        float vx = px - (float)cam.center[0], vy = py - (float)cam.center[1], vz = pz - (float)cam.center[2];
        const float vn = sqrtf(vx * vx + vy * vy + vz * vz);
        const float ivn = 1.f / vn;
        vx *= ivn;
        vy *= ivn;
        vz *= ivn;
        float ddx = 0.f, ddy = 0.f, ddz = 0.f;
        app_backward<K>(sc, a.g, i, vx, vy, vz, dr, dg, dbl, ddx, ddy, ddz, srow);
        const float dd = ddx * vx + ddy * vy + ddz * vz;
        dpx += (ddx - dd * vx) * ivn;
        dpy += (ddy - dd * vy) * ivn;
        dpz += (ddz - dd * vz) * ivn;
    }
    if (!a.drgb) {
        if (ovw) {
            a.g.positions[3 * i] = dpx;
            a.g.positions[3 * i + 1] = dpy;
            a.g.positions[3 * i + 2] = dpz;
        } else {
            a.g.positions[3 * i] += dpx;
            a.g.positions[3 * i + 1] += dpy;
            a.g.positions[3 * i + 2] += dpz;
        }
    }
}

// bsr_grads::overwrite: the rows of a culled primitive (its gradients are zero,
// rasterizer.py:262-320) -- written here since nothing else touches them
template <int CM>
__device__ __forceinline__ void zero_rows(const PreBwdArgs &a, int64_t i, bool sh_staged = false) {
    using Tr = AppTraits<CM>;
    const bsr_grads &g = a.g;
    for (int q = 0; q < 3; ++q) g.positions[3 * i + q] = g.log_scales[3 * i + q] = 0.f;
    if ((reinterpret_cast<uintptr_t>(g.rotations) & 15) == 0)
        reinterpret_cast<float4 *>(g.rotations)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    else
        for (int q = 0; q < 4; ++q) g.rotations[4 * i + q] = 0.f;
    g.opacity_raw[i] = g.shapes[i] = 0.f;
    if constexpr (Tr::sh) {
        if (sh_staged) {  // the warp's coalesced row store writes it
            if (a.screen_grad_norm) a.screen_grad_norm[i] = 0.f;
            return;
        }
        float *row = g.sh + 3 * Tr::K * i;
        if ((3 * Tr::K) % 4 == 0 && (reinterpret_cast<uintptr_t>(g.sh) & 15) == 0) {
            for (int q = 0; q < 3 * Tr::K / 4; ++q) reinterpret_cast<float4 *>(row)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            for (int q = 0; q < 3 * Tr::K; ++q) row[q] = 0.f;
        }
    } else {
        for (int q = 0; q < 3; ++q) g.base_colors[3 * i + q] = 0.f;
        for (int q = 0; q < 3 * Tr::M; ++q) g.lobe_axes[3 * Tr::M * i + q] = g.lobe_colors[3 * Tr::M * i + q] = 0.f;
    }
    if (a.screen_grad_norm) a.screen_grad_norm[i] = 0.f;
}

// Each warp takes 64 consecutive source indices and runs the visible ones densely (32
// per pass, ballot-compacted); culled primitives get no gradient (rasterizer.py:262-320
// leaves them zero).
constexpr int kPreBwdChunk = 64;
// 4-warp CTAs: small scenes (config 1: one wave) spread over more SMs
constexpr int kPreBwdThreads = 128;

// SH rows (3K floats, K = 4 / 16: whole float4s) of the warp's chunk are staged through
// shared memory in overwrite mode: loaded and stored by the warp with lane-contiguous
// 16-byte accesses (a thread per row would touch 32 rows 3K floats apart per access), the
// culled rows' zeros included.
static_assert(kPreBwdChunk == 64, "two visibility words per warp chunk");
template <int CM>
struct PreBwdStage {
    static constexpr bool on = AppTraits<CM>::sh && (3 * AppTraits<CM>::K) % 4 == 0;
    static constexpr int rw = on ? 3 * AppTraits<CM>::K / 4 : 0;  // float4 per row
    static constexpr int rs = rw | 1;  // row stride: odd, so 8 lanes' float4 rows hit distinct banks
    static constexpr size_t bytes = (size_t)(kPreBwdThreads / 32) * kPreBwdChunk * rs * 16;
};

template <int K>
__global__ void __launch_bounds__(kPreBwdThreads) preprocess_bwd_kernel(__grid_constant__ const PreBwdArgs a) {
    pdl_wait();
    using St = PreBwdStage<K>;
    extern __shared__ float4 pbw_stage[];
    const int lane = threadIdx.x & 31;
    const int64_t c0 = ((blockIdx.x * (int64_t)kPreBwdThreads + threadIdx.x) >> 5) * kPreBwdChunk;
    if (c0 >= a.f.n) return;
    const bool stage = St::on && a.g.overwrite && !a.drgb &&
                       ((reinterpret_cast<uintptr_t>(a.sc.sh) | reinterpret_cast<uintptr_t>(a.g.sh)) & 15) == 0;
    float4 *wbuf = pbw_stage + (threadIdx.x >> 5) * (kPreBwdChunk * St::rs);
    uint32_t m[kPreBwdChunk / 32];
    int tot = 0;
#pragma unroll
    for (int q = 0; q < kPreBwdChunk / 32; ++q) {
        const int64_t c = c0 + 32 * q + lane;
        const bool vis = c < a.f.n && a.f.tile_count[c] != 0;
        m[q] = __ballot_sync(0xffffffffu, vis);
        tot += __popc(m[q]);
        if (a.drgb && c < a.f.n && !vis) a.drgb[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a.g.overwrite && c < a.f.n && !vis) zero_rows<K>(a, c, stage);
    }
    const int rows = (int)min((int64_t)kPreBwdChunk, a.f.n - c0);
    if (St::on && stage) {
        const float4 *src = reinterpret_cast<const float4 *>(a.sc.sh) + c0 * St::rw;
        for (int u = lane; u < rows * St::rw; u += 32) {
            const int row = u / St::rw;
            if (((row < 32 ? m[0] : m[1]) >> (row & 31)) & 1u) wbuf[u + row * (St::rs - St::rw)] = __ldg(src + u);
        }
        __syncwarp();
    }
    for (int base = 0; base < tot; base += 32) {
        int r = base + lane;
        if (r >= tot) break;
        int q = 0;
#pragma unroll
        for (int k = 0; k < kPreBwdChunk / 32 - 1; ++k)
            if (q == k && r >= __popc(m[k])) {
                r -= __popc(m[k]);
                q = k + 1;
            }
        const int row = 32 * q + (int)__fns(m[q], 0, r + 1);
        prebwd_one<K>(a, c0 + row, (St::on && stage) ? wbuf + row * St::rs : nullptr);
    }
    if (St::on && stage) {
        __syncwarp();
        float4 *dst = reinterpret_cast<float4 *>(a.g.sh) + c0 * St::rw;
        for (int u = lane; u < rows * St::rw; u += 32) {
            const int row = u / St::rw;
            dst[u] = (((row < 32 ? m[0] : m[1]) >> (row & 31)) & 1u) ? wbuf[u + row * (St::rs - St::rw)]
                                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

// Geometric chain of every visible primitive, fp64 (geom_chain): the raster's geometry
// partials are mapped to d mean2d / d cov2d with the record's factor L (whitened frame,
// frame.cuh grad_acc):  d mean = -2 L M,  d cov2d = -Q G Q = -L H L^T  (Q = L L^T,
// G = L^-T H L^-1 the conic gradient, rasterizer.py:302-312), so no inverse of the
// ill-conditioned conic is formed (the factor of each record class: raster.cuh
// record_factor64).  fp64-path records without a factor carry xy-frame conic partials
// summed in fp64 (side64, cleared here) and use the fp64 conic.
template <bool DRGB>
__device__ __forceinline__ void prebwd_geom_one(const PreBwdArgs &a, int64_t i) {
    const FrameView &f = a.f;
    if (DRGB) {  // deferred colour chain: this kernel also does prebwd_one's non-colour part
        const float *acc = f.grad_acc + i * kGradStride;
        const float4 g1 = *reinterpret_cast<const float4 *>(acc + 4);
        const float4 g2 = *reinterpret_cast<const float4 *>(acc + 8);
        const float oraw = a.sc.opacity_raw[i];
        const float o = oraw >= 0.f ? 1.f / (1.f + expf(-oraw)) : expf(oraw) / (1.f + expf(oraw));
        a.g.opacity_raw[i] += g1.y * o * (1.f - o);
        const float bsh = a.sc.shapes[i];
        if (fabsf(bsh) <= 10.f) a.g.shapes[i] += g1.z * (4.f * expf(fminf(fmaxf(bsh, -10.f), 10.f)));
        a.drgb[i] = make_float4(g1.w, g2.x, g2.y, 0.f);
    }
    double dmx, dmy, gm00, gs01, gm11;
    double l11, l21, l22;
    if (record_factor64(f, (uint32_t)i, l11, l21, l22)) {
        const float *acc = f.grad_acc + i * kGradStride;
        const float4 g0 = *reinterpret_cast<const float4 *>(acc);
        const double mu = g0.x, mw = g0.y, h00 = g0.z, h01 = g0.w, h11 = acc[4];
        dmx = -2.0 * l11 * mu;
        dmy = -2.0 * (l21 * mu + l22 * mw);
        gm00 = -(l11 * l11 * h00);
        gs01 = -(l11 * (h00 * l21 + h01 * l22));
        gm11 = -((l21 * h00 + l22 * h01) * l21 + (l21 * h01 + l22 * h11) * l22);
    } else {  // no factor: xy-frame conic partials summed in fp64, fp64 conic
        double2 *g2 = reinterpret_cast<double2 *>(f.side64 + kSide64 * i);
        const double2 u0 = g2[0], u1 = g2[1], u2 = g2[2];
        g2[0] = g2[1] = g2[2] = make_double2(0.0, 0.0);
        const double *m64 = f.rec64 + kRec64 * i;
        const double ia = m64[2], ib = m64[3], ic = m64[4];
        const double dA = u1.x, Gb = 0.5 * u1.y, dC = u2.x;
        dmx = u0.x;
        dmy = u0.y;
        const double m00 = dA * ia + Gb * ib, m01 = dA * ib + Gb * ic;  // G Q
        const double m10 = Gb * ia + dC * ib, m11 = Gb * ib + dC * ic;
        gm00 = -(ia * m00 + ib * m10);
        gs01 = -0.5 * ((ia * m01 + ib * m11) + (ib * m00 + ic * m10));
        gm11 = -(ib * m01 + ic * m11);
    }
    const float dz = f.grad_acc[i * kGradStride + 10];
    float dpx, dpy, dpz;
    geom_chain<double>(a, i, dmx, dmy, gm00, gs01, gm11, dz, dpx, dpy, dpz);
    a.g.positions[3 * i] += dpx;
    a.g.positions[3 * i + 1] += dpy;
    a.g.positions[3 * i + 2] += dpz;
    if (a.screen_grad_norm) a.screen_grad_norm[i] = (float)sqrt(dmx * dmx + dmy * dmy);
}

// 6 resident CTAs per SM (80 registers; the fp64 chain then spills ~0.5 KB to L1, which the
// extra warps hide: measured 4 / 5 / 6 / 7 / 8 per SM, config 3 0.281 / 0.264 / 0.260 /
// 0.269 / 0.275 ms per view, config 4 preprocess_bwd 0.904 / 0.878 / 0.860 / 0.901 / 0.941 ms)
#ifndef BSR_GEOM_MINB
#define BSR_GEOM_MINB 6
#endif
// DRGB: the multi-view deferred-colour mode, where the fp32 colour kernel has nothing
// left but the opacity / shape chains and the d rgb store -- done here instead, so that
// mode runs one kernel per view, not two.
template <bool DRGB>
__global__ void __launch_bounds__(kPreBwdThreads, BSR_GEOM_MINB) prebwd_geom_kernel(__grid_constant__ const PreBwdArgs a) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t c0 = ((blockIdx.x * (int64_t)kPreBwdThreads + threadIdx.x) >> 5) * kPreBwdChunk;
    if (c0 >= a.f.n) return;
    uint32_t m[kPreBwdChunk / 32];
    int tot = 0;
#pragma unroll
    for (int q = 0; q < kPreBwdChunk / 32; ++q) {
        const int64_t c = c0 + 32 * q + lane;
        const bool vis = c < a.f.n && a.f.tile_count[c] != 0;
        m[q] = __ballot_sync(0xffffffffu, vis);
        tot += __popc(m[q]);
        if (DRGB && c < a.f.n && !vis) a.drgb[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int base = 0; base < tot; base += 32) {
        int r = base + lane;
        if (r >= tot) break;
        int q = 0;
#pragma unroll
        for (int k = 0; k < kPreBwdChunk / 32 - 1; ++k)
            if (q == k && r >= __popc(m[k])) {
                r -= __popc(m[k]);
                q = k + 1;
            }
        prebwd_geom_one<DRGB>(a, c0 + 32 * q + (int)__fns(m[q], 0, r + 1));
    }
}

int launch_preprocess_bwd(const bsr_scene &sc, const KCam &cam, const FrameView &f,
                          const bsr_grads &g, float *screen_grad_norm, float4 *drgb, cudaStream_t st) {
    if (f.n == 0) return BSR_OK;
    PreBwdArgs a{sc, cam, f, g, screen_grad_norm, drgb};
    const unsigned blocks = (unsigned)div_up(f.n, (int64_t)kPreBwdChunk * (kPreBwdThreads / 32));
    if (drgb) {  // deferred colour chain (SH, multi-view, accumulating): one fused kernel
        BSR_CUDA_TRY((pdl_launch(prebwd_geom_kernel<true>, dim3(blocks), dim3(kPreBwdThreads), 0, st, a)));
        BSR_LAUNCH_CHECK();
        return BSR_OK;
    }
#define BSR_PREBWD_LAUNCH(CM)                                                                                   \
    do {                                                                                                        \
        static SmemAttrOnce attr;                                                                               \
        BSR_CUDA_TRY(attr.ensure(preprocess_bwd_kernel<CM>, PreBwdStage<CM>::bytes));                           \
        BSR_CUDA_TRY((pdl_launch(preprocess_bwd_kernel<CM>, dim3(blocks), dim3(kPreBwdThreads),                  \
                                 PreBwdStage<CM>::bytes, st, a)));                                              \
    } while (0)
    BSR_DISPATCH_CM(sc, BSR_PREBWD_LAUNCH);
#undef BSR_PREBWD_LAUNCH
    BSR_CUDA_TRY((pdl_launch(prebwd_geom_kernel<false>, dim3(blocks), dim3(kPreBwdThreads), 0, st, a)));
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

// ---- deferred multi-view colour chain (SH colour) ---------------------------------------
// For a step over several views the SH part of the chain is linear in each view's d rgb:
//   d sh[k] = sum_v basis_k(dir_v) d_rgb_v,   d dir_v = dbasis(dir_v)^T (sh . d_rgb_v)
// (appearance.py:264-318, rasterizer.py:287-289), so instead of a read-modify-write of
// the 3K coefficient gradients per view, preprocess_bwd stores d_rgb_v (16 B) and this
// kernel applies all views at once: SH coefficients read once, their gradients written
// once.
constexpr int kMaxViewsPerPass = 32;

struct ColorViewsArgs {
    bsr_scene sc;
    bsr_grads g;
    const float4 *drgb;  // [views][n]
    int views;
    float center[kMaxViewsPerPass][3];
};

// One CTA owns 128 consecutive primitives.  Its inputs are contiguous runs in HBM (the 3K
// coefficients, and per view 128 x 16 B of d rgb), so one elected thread streams them into
// shared memory with TMA bulk copies: the coefficients once, the views in chunks of
// kViewChunk through a two-slot ring, so a whole chunk of views is in flight per CTA
// instead of one 16 B load per thread.  The coefficient gradients leave through shared
// memory as one coalesced read-modify-write of the CTA's contiguous run.
constexpr int kCvThreads = 128;
constexpr int kViewChunk = 8;

template <int K>
constexpr size_t color_views_smem() {
    return 2 * kViewChunk * kCvThreads * sizeof(float4) + (size_t)kCvThreads * 3 * K * sizeof(float) + 64;
}

template <int K>
__global__ void __launch_bounds__(kCvThreads) color_views_kernel(ColorViewsArgs a) {
    extern __shared__ __align__(128) unsigned char cv_smem[];
    float4 *s_d = reinterpret_cast<float4 *>(cv_smem);                   // [2][kViewChunk][128]
    float *s_sh = reinterpret_cast<float *>(s_d + 2 * kViewChunk * kCvThreads);  // [128][3K]
    uint64_t *bar = reinterpret_cast<uint64_t *>(s_sh + kCvThreads * 3 * K);      // sh, slot 0, slot 1
    const int64_t n = a.sc.n;
    const int64_t i0 = blockIdx.x * (int64_t)kCvThreads;
    const int cnt = (int)(n - i0 < kCvThreads ? n - i0 : kCvThreads);
    const int t = threadIdx.x;
    const int chunks = (a.views + kViewChunk - 1) / kViewChunk;
    auto issue = [&](int c) {  // views [c*kViewChunk, ...) -> slot c & 1
        const int v0 = c * kViewChunk, nv = a.views - v0 < kViewChunk ? a.views - v0 : kViewChunk;
        uint64_t *b = bar + 1 + (c & 1);
        mbar_expect_tx(b, (uint32_t)(nv * cnt * sizeof(float4)));
        for (int v = 0; v < nv; ++v)
            bulk_g2s(s_d + ((c & 1) * kViewChunk + v) * kCvThreads, a.drgb + (int64_t)(v0 + v) * n + i0,
                     (uint32_t)(cnt * sizeof(float4)), b);
    };
    if (t == 0) {
        for (int q = 0; q < 3; ++q) mbar_init(bar + q, 1);
    }
    __syncthreads();
    pdl_wait();  // d rgb comes from the preceding backward
    const float *src_sh = a.sc.sh + i0 * 3 * K;
    const uint32_t sh_bytes = (uint32_t)(cnt * 3 * K * sizeof(float));
    const bool sh_bulk = ((reinterpret_cast<uintptr_t>(src_sh) | sh_bytes) & 15) == 0;
    if (t == 0) {
        if (sh_bulk) {
            mbar_expect_tx(bar, sh_bytes);
            bulk_g2s(s_sh, src_sh, sh_bytes, bar);
        }
        issue(0);
        if (chunks > 1) issue(1);
    }
    if (!sh_bulk) {  // a 16 B-misaligned run (K = 1 or 9, partial CTA): coalesced plain loads
        for (int e = t; e < cnt * 3 * K; e += kCvThreads) s_sh[e] = src_sh[e];
        __syncthreads();
    }
    const bool live = t < cnt;
    const int64_t i = i0 + t;
    float px = 0.f, py = 0.f, pz = 0.f;
    if (live) px = a.sc.positions[3 * i], py = a.sc.positions[3 * i + 1], pz = a.sc.positions[3 * i + 2];
    float sh[3 * K], dsh[3 * K];
    if (sh_bulk) mbar_wait(bar, 0);
#pragma unroll
    for (int q = 0; q < 3 * K; ++q) {
        sh[q] = s_sh[t * 3 * K + q];
        dsh[q] = 0.f;
    }
    float dpx = 0.f, dpy = 0.f, dpz = 0.f;
    bool any = false;
    for (int c = 0; c < chunks; ++c) {
        mbar_wait(bar + 1 + (c & 1), (c >> 1) & 1);
        const int v0 = c * kViewChunk, nv = a.views - v0 < kViewChunk ? a.views - v0 : kViewChunk;
        const float4 *slot = s_d + (c & 1) * kViewChunk * kCvThreads;
        for (int v = 0; v < nv && live; ++v) {
            const float4 d = slot[v * kCvThreads + t];
            if (d.x == 0.f && d.y == 0.f && d.z == 0.f) continue;
            any = true;
            float vx = px - a.center[v0 + v][0], vy = py - a.center[v0 + v][1], vz = pz - a.center[v0 + v][2];
            const float vn = sqrtf(vx * vx + vy * vy + vz * vz);
            const float ivn = 1.f / vn;
            vx *= ivn;
            vy *= ivn;
            vz *= ivn;
            float b[16], db[16][3];
            sh_basis_and_grad<K>(vx, vy, vz, b, db);
            float ddx = 0.f, ddy = 0.f, ddz = 0.f;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                dsh[3 * k] += b[k] * d.x;
                dsh[3 * k + 1] += b[k] * d.y;
                dsh[3 * k + 2] += b[k] * d.z;
                const float dbk = sh[3 * k] * d.x + sh[3 * k + 1] * d.y + sh[3 * k + 2] * d.z;
                ddx += db[k][0] * dbk;
                ddy += db[k][1] * dbk;
                ddz += db[k][2] * dbk;
            }
            const float dd = ddx * vx + ddy * vy + ddz * vz;
            dpx += (ddx - dd * vx) * ivn;
            dpy += (ddy - dd * vy) * ivn;
            dpz += (ddz - dd * vz) * ivn;
        }
        __syncthreads();  // slot c & 1 is free again
        if (t == 0 && c + 2 < chunks) issue(c + 2);
    }
    if (live && any) {
        a.g.positions[3 * i] += dpx;
        a.g.positions[3 * i + 1] += dpy;
        a.g.positions[3 * i + 2] += dpz;
    }
    // coefficient gradients: registers -> shared (own row) -> one coalesced RMW of the run
    if (!__syncthreads_or(any)) return;
#pragma unroll
    for (int q = 0; q < 3 * K; ++q) s_sh[t * 3 * K + q] = dsh[q];
    __syncthreads();
    float *gsh = a.g.sh + i0 * 3 * K;
    for (int e = t; e < cnt * 3 * K; e += kCvThreads) gsh[e] += s_sh[e];
}

int launch_color_views(const bsr_scene &sc, const bsr_grads &g, const float4 *drgb, const double *centers,
                       int views, cudaStream_t st) {
    if (sc.n == 0 || views == 0) return BSR_OK;
    for (int v0 = 0; v0 < views; v0 += kMaxViewsPerPass) {
        ColorViewsArgs a;
        a.sc = sc;
        a.g = g;
        a.drgb = drgb + (int64_t)v0 * sc.n;
        a.views = views - v0 < kMaxViewsPerPass ? views - v0 : kMaxViewsPerPass;
        for (int v = 0; v < a.views; ++v)
            for (int c = 0; c < 3; ++c) a.center[v][c] = (float)centers[3 * (v0 + v) + c];
        const unsigned blocks = (unsigned)div_up(sc.n, kCvThreads);
#define BSR_CV_LAUNCH(K)                                                                                     \
    do {                                                                                                     \
        static SmemAttrOnce attr;                                                                            \
        BSR_CUDA_TRY(attr.ensure(color_views_kernel<K>, color_views_smem<K>()));                             \
        BSR_CUDA_TRY((pdl_launch(color_views_kernel<K>, dim3(blocks), dim3(kCvThreads), color_views_smem<K>(), st, a))); \
    } while (0)
        switch (sc.sh_coeffs) {
            case 1: BSR_CV_LAUNCH(1); break;
            case 4: BSR_CV_LAUNCH(4); break;
            case 9: BSR_CV_LAUNCH(9); break;
            case 16: BSR_CV_LAUNCH(16); break;
            default: return BSR_ERR_BAD_ARG;
        }
#undef BSR_CV_LAUNCH
    }
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
