/*
 * ORACLE -- test infrastructure only.  Never linked into the product library; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it, as the checker.
 *
 * Plain-C fp64 restatement of the reference raster core
 *   /root/reference/pkg/src/betasplat/_raster.pyx
 *     _tile_forward   (:74-127)  per-pixel front-to-back compositing over a tile list
 *     forward_tiled   (:130-155) prange over tiles + fixed-order contribution merge
 *     _tile_backward  (:158-241) per-pixel front-to-back replay, per-entry staging
 *     backward        (:244-287) prange over tiles + fixed-order gradient merge
 * with the same expression trees and operation order (compiled with -ffp-contract=off,
 * like pkg/setup.py:13), so raw / T / contributions come out bit-identical to the
 * compiled reference core (pinned in tests/test_oracle.py).
 *
 * Extensions the reference does not produce, needed by the north-star contract:
 *   - per-pixel contributor count and last contributing entry (bit-exact targets),
 *   - per-pixel evaluated pair count (the roofline's P_f),
 *   - an accumulated-depth channel D = sum_k w_k z_k (no background term) and its
 *     backward, formed exactly like the reference's colour channels with bg = 0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const double EDGE_GRAD_CLAMP = 1e7; /* _raster.pyx:21 */

typedef struct {
    const double *means, *conics, *opac, *betas, *colors, *depths;
    const int32_t *bounds;
    int height, width, tile_size, tiles_x;
    const double *bg;
    const int64_t *offsets, *lists;
    double alpha_min, t_stop;
} scene_t;

/* _raster.pyx:74-127 */
static void tile_forward(const scene_t *s, int tile, double *raw, double *trans, double *depth_out,
                         int64_t *stage_contrib, int32_t *pix_count, int64_t *pix_last,
                         int64_t *pix_pairs) {
    int tx0 = (tile % s->tiles_x) * s->tile_size;
    int ty0 = (tile / s->tiles_x) * s->tile_size;
    int tx1 = tx0 + s->tile_size - 1;
    int ty1 = ty0 + s->tile_size - 1;
    if (tx1 > s->width - 1) tx1 = s->width - 1;
    if (ty1 > s->height - 1) ty1 = s->height - 1;
    int64_t lo = s->offsets[tile], hi = s->offsets[tile + 1];
    for (int py = ty0; py <= ty1; ++py) {
        for (int px = tx0; px <= tx1; ++px) {
            double t = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, dacc = 0.0;
            int32_t count = 0;
            int64_t last = -1, pairs = 0;
            for (int64_t e = lo; e < hi; ++e) {
                int k = (int)s->lists[e];
                const int32_t *b = s->bounds + 4 * (int64_t)k;
                if (px < b[0] || px > b[1]) continue;
                if (py < b[2] || py > b[3]) continue;
                ++pairs;
                double dx = px - s->means[2 * k + 0];
                double dy = py - s->means[2 * k + 1];
                const double *cn = s->conics + 3 * (int64_t)k;
                double r2 = cn[0] * dx * dx + 2.0 * cn[1] * dx * dy + cn[2] * dy * dy;
                double x = fmin(fmax(r2, 0.0), 1.0);
                double kernel = pow(1.0 - x, s->betas[k]);
                double alpha = s->opac[k] * kernel;
                if (alpha < s->alpha_min) continue;
                double weight = alpha * t;
                const double *col = s->colors + 3 * (int64_t)k;
                c0 = c0 + weight * col[0];
                c1 = c1 + weight * col[1];
                c2 = c2 + weight * col[2];
                if (s->depths) dacc = dacc + weight * s->depths[k];
                t = t * (1.0 - alpha);
                stage_contrib[e] += 1;
                ++count;
                last = e;
                if (t < s->t_stop) break;
            }
            int64_t p = (int64_t)py * s->width + px;
            raw[3 * p + 0] = c0 + s->bg[0] * t;
            raw[3 * p + 1] = c1 + s->bg[1] * t;
            raw[3 * p + 2] = c2 + s->bg[2] * t;
            trans[p] = t;
            if (depth_out) depth_out[p] = dacc;
            if (pix_count) pix_count[p] = count;
            if (pix_last) pix_last[p] = last;
            if (pix_pairs) pix_pairs[p] = pairs;
        }
    }
}

/* _raster.pyx:130-155.  Outputs are caller-allocated; contrib has V entries. */
void oracle_forward_tiled(int v, const double *means, const double *conics, const double *opac,
                          const double *betas, const double *colors, const double *depths,
                          const int32_t *bounds, int height, int width, const double *bg,
                          int tile_size, const int64_t *offsets, const int64_t *lists,
                          int64_t n_entries, int threads, double alpha_min, double t_stop,
                          double *raw, double *trans, double *depth_out, int64_t *contrib,
                          int32_t *pix_count, int64_t *pix_last, int64_t *pix_pairs) {
    scene_t s = {means, conics, opac, betas, colors, depths, bounds, height, width, tile_size,
                 (width + tile_size - 1) / tile_size, bg, offsets, lists, alpha_min, t_stop};
    int n_tiles = ((width + tile_size - 1) / tile_size) * ((height + tile_size - 1) / tile_size);
    int64_t *stage = (int64_t *)calloc(n_entries > 0 ? n_entries : 1, sizeof(int64_t));
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int tile = 0; tile < n_tiles; ++tile)
        tile_forward(&s, tile, raw, trans, depth_out, stage, pix_count, pix_last, pix_pairs);
    memset(contrib, 0, sizeof(int64_t) * (size_t)v);
    for (int64_t e = 0; e < n_entries; ++e) contrib[s.lists[e]] += stage[e];
    free(stage);
}

#define NSTAGE 11 /* reference's 10 partials + d_depth */

/* _raster.pyx:158-241 (+ the depth channel, formed like a colour channel with bg = 0) */
static void tile_backward(const scene_t *s, int tile, const double *raw, const double *raw_depth,
                          const double *d_raw, const double *d_depth, double *stage) {
    int tx0 = (tile % s->tiles_x) * s->tile_size;
    int ty0 = (tile / s->tiles_x) * s->tile_size;
    int tx1 = tx0 + s->tile_size - 1;
    int ty1 = ty0 + s->tile_size - 1;
    if (tx1 > s->width - 1) tx1 = s->width - 1;
    if (ty1 > s->height - 1) ty1 = s->height - 1;
    int64_t lo = s->offsets[tile], hi = s->offsets[tile + 1];
    for (int py = ty0; py <= ty1; ++py) {
        for (int px = tx0; px <= tx1; ++px) {
            int64_t p = (int64_t)py * s->width + px;
            double t = 1.0, p0 = 0.0, p1 = 0.0, p2 = 0.0, pd = 0.0;
            double g0 = d_raw[3 * p + 0], g1 = d_raw[3 * p + 1], g2 = d_raw[3 * p + 2];
            double gd = d_depth ? d_depth[p] : 0.0;
            for (int64_t e = lo; e < hi; ++e) {
                int k = (int)s->lists[e];
                const int32_t *bb = s->bounds + 4 * (int64_t)k;
                if (px < bb[0] || px > bb[1]) continue;
                if (py < bb[2] || py > bb[3]) continue;
                double dx = px - s->means[2 * k + 0];
                double dy = py - s->means[2 * k + 1];
                double a = s->conics[3 * k + 0], b = s->conics[3 * k + 1], c = s->conics[3 * k + 2];
                double r2 = a * dx * dx + 2.0 * b * dx * dy + c * dy * dy;
                double x = fmin(fmax(r2, 0.0), 1.0);
                double kernel = pow(1.0 - x, s->betas[k]);
                double alpha = s->opac[k] * kernel;
                if (alpha < s->alpha_min) continue;
                double weight = alpha * t;
                const double *col = s->colors + 3 * (int64_t)k;
                double cr0 = weight * col[0];
                double cr1 = weight * col[1];
                double cr2 = weight * col[2];
                double behind0 = raw[3 * p + 0] - p0 - cr0;
                double behind1 = raw[3 * p + 1] - p1 - cr1;
                double behind2 = raw[3 * p + 2] - p2 - cr2;
                double g_dot_col = g0 * col[0] + g1 * col[1] + g2 * col[2];
                double g_dot_behind = g0 * behind0 + g1 * behind1 + g2 * behind2;
                double d_alpha = g_dot_col * t - g_dot_behind / (1.0 - alpha);
                double crd = 0.0;
                if (d_depth) {
                    double z = s->depths[k];
                    crd = weight * z;
                    double behindd = raw_depth[p] - pd - crd;
                    d_alpha = d_alpha + (gd * z * t - gd * behindd / (1.0 - alpha));
                }
                double *st = stage + NSTAGE * e;
                st[7] += weight * g0;
                st[8] += weight * g1;
                st[9] += weight * g2;
                st[10] += weight * gd;
                st[5] += d_alpha * kernel;
                double d_kernel = d_alpha * s->opac[k];
                if (x < 1.0) {
                    st[6] += d_kernel * kernel * log(1.0 - x);
                    double dkdx = -s->betas[k] * pow(1.0 - x, s->betas[k] - 1.0);
                    if (dkdx < -EDGE_GRAD_CLAMP) dkdx = -EDGE_GRAD_CLAMP;
                    double d_x = d_kernel * dkdx;
                    st[0] += -d_x * 2.0 * (a * dx + b * dy);
                    st[1] += -d_x * 2.0 * (b * dx + c * dy);
                    st[2] += d_x * dx * dx;
                    st[3] += d_x * 2.0 * dx * dy;
                    st[4] += d_x * dy * dy;
                }
                p0 = p0 + cr0;
                p1 = p1 + cr1;
                p2 = p2 + cr2;
                pd = pd + crd;
                t = t * (1.0 - alpha);
                if (t < s->t_stop) break;
            }
        }
    }
}

/* _raster.pyx:244-287.  Output arrays (V-sized) are overwritten. */
void oracle_backward(int v, const double *means, const double *conics, const double *opac,
                     const double *betas, const double *colors, const double *depths,
                     const int32_t *bounds, int height, int width, const double *bg,
                     const double *raw, const double *raw_depth, const double *d_raw,
                     const double *d_depth, int tile_size, const int64_t *offsets,
                     const int64_t *lists, int64_t n_entries, int threads, double alpha_min,
                     double t_stop, double *d_means, double *d_conics, double *d_opac,
                     double *d_betas, double *d_colors, double *d_depths) {
    scene_t s = {means, conics, opac, betas, colors, depths, bounds, height, width, tile_size,
                 (width + tile_size - 1) / tile_size, bg, offsets, lists, alpha_min, t_stop};
    int n_tiles = ((width + tile_size - 1) / tile_size) * ((height + tile_size - 1) / tile_size);
    double *stage = (double *)calloc((size_t)(n_entries > 0 ? n_entries : 1) * NSTAGE, sizeof(double));
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int tile = 0; tile < n_tiles; ++tile)
        tile_backward(&s, tile, raw, raw_depth, d_raw, d_depth, stage);
    memset(d_means, 0, sizeof(double) * 2 * (size_t)v);
    memset(d_conics, 0, sizeof(double) * 3 * (size_t)v);
    memset(d_opac, 0, sizeof(double) * (size_t)v);
    memset(d_betas, 0, sizeof(double) * (size_t)v);
    memset(d_colors, 0, sizeof(double) * 3 * (size_t)v);
    if (d_depths) memset(d_depths, 0, sizeof(double) * (size_t)v);
    /* fixed merge order (_raster.pyx:273-286) */
    for (int64_t e = 0; e < n_entries; ++e) {
        int k = (int)lists[e];
        const double *st = stage + NSTAGE * e;
        d_means[2 * k + 0] += st[0];
        d_means[2 * k + 1] += st[1];
        d_conics[3 * k + 0] += st[2];
        d_conics[3 * k + 1] += st[3];
        d_conics[3 * k + 2] += st[4];
        d_opac[k] += st[5];
        d_betas[k] += st[6];
        d_colors[3 * k + 0] += st[7];
        d_colors[3 * k + 1] += st[8];
        d_colors[3 * k + 2] += st[9];
        if (d_depths) d_depths[k] += st[10];
    }
    free(stage);
}
