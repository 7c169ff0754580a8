/*
 * ORACLE — test infrastructure only.  Never linked into the product library.
 *
 * Plain-C restatement of the reference's per-frame binning and per-tile
 * compositing loops, used by tests/ (as the checker), by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * legs.  Each function cites the reference code it restates
 * (paths under /root/reference/pkg/src/betasplat).
 *
 * Differences from the reference that do not change results:
 *   - one call handles every tile of a frame (the reference calls the numba
 *     kernels once per tile from a thread pool, raster.py:284-311,426-433);
 *   - the forward additionally reports the per-pixel contributor count (the
 *     number of splats a pixel iterated before the transmittance early-out,
 *     which the reference accumulates only as a total, _tiles.py:35);
 *   - per-tile partial gradients are written into one flat array indexed by
 *     list position and reduced tile by tile in fixed tile order, as
 *     gradients.py:164-173 does with np.add.at.
 *
 * Arithmetic is evaluated in the same order as the Python source, with FMA
 * contraction disabled (-ffp-contract=off), matching numba's default.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* raster.py:252-266 build_tiles: for every 16x16 tile in row-major order,
 * keep the depth-ordered splats whose [mean2 -/+ radii] box touches the tile
 * (inclusive bounds, last tile clipped to the image).  Same two-level mask as
 * the reference (row mask, raster.py:260-261, then the column test per tile),
 * on bounds precomputed in rank order.  `lo`/`hi` are (n_order, 2) rank-
 * ordered mean2 -/+ radii.  fill == 0: write per-tile counts into `out`,
 * return K.  fill == 1: write ids (order[r]) at tile_start[t]... into `out`. */
int64_t oracle_build_tiles(int width, int height, int tile, int64_t n_order, const int64_t *order,
                           const double *lo, const double *hi, const int64_t *tile_start, int64_t *out,
                           int fill) {
    int tx_n = (width + tile - 1) / tile, ty_n = (height + tile - 1) / tile;
    int64_t total = 0;
#pragma omp parallel reduction(+ : total)
    {
        int64_t *cand = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_order > 0 ? n_order : 1));
#pragma omp for schedule(dynamic, 1)
        for (int ty = 0; ty < ty_n; ++ty) {
            double y0 = (double)(ty * tile), y1 = (double)((ty + 1) * tile < height ? (ty + 1) * tile : height);
            int64_t nc = 0;
            for (int64_t r = 0; r < n_order; ++r)
                if (hi[2 * r + 1] >= y0 && lo[2 * r + 1] <= y1) cand[nc++] = r;
            for (int tx = 0; tx < tx_n; ++tx) {
                double x0 = (double)(tx * tile), x1 = (double)((tx + 1) * tile < width ? (tx + 1) * tile : width);
                int t = ty * tx_n + tx;
                int64_t c = 0, w = fill ? tile_start[t] : 0;
                for (int64_t j = 0; j < nc; ++j) {
                    int64_t r = cand[j];
                    if (hi[2 * r] >= x0 && lo[2 * r] <= x1) {
                        if (fill) out[w++] = order[r];
                        ++c;
                    }
                }
                if (!fill) out[t] = c;
                total += c;
            }
        }
        free(cand);
    }
    return total;
}

/* _tiles.py:19-56 tile_forward, applied to every tile of the frame.
 * p2 is (n,2,2) row-major.  Outputs are full-image arrays; hit is per
 * primitive.  Returns the total number of splat-pixel visits. */
int64_t oracle_raster_forward(int width, int height, int tile, const int64_t *tile_start,
                              const int64_t *tile_ids, const double *mean2, const double *p2,
                              const double *og, const double *bx, const double *color,
                              const double *bg, double tau_sq, double clamp, double t_min,
                              double *rgb, double *asum, double *tstop, int32_t *count,
                              uint8_t *hit) {
    int tx_n = (width + tile - 1) / tile, ty_n = (height + tile - 1) / tile;
    int64_t visits_total = 0;
#pragma omp parallel for schedule(dynamic, 2) reduction(+ : visits_total)
    for (int t = 0; t < tx_n * ty_n; ++t) {
        int ty = t / tx_n, tx = t % tx_n;
        int ya = ty * tile, yb = (ty + 1) * tile < height ? (ty + 1) * tile : height;
        int xa = tx * tile, xb = (tx + 1) * tile < width ? (tx + 1) * tile : width;
        int64_t s = tile_start[t], e = tile_start[t + 1];
        for (int y = ya; y < yb; ++y) {
            for (int x = xa; x < xb; ++x) {
                double px = x + 0.5, py = y + 0.5;
                double T = 1.0, a0 = 0.0, a1 = 0.0, a2 = 0.0, ws = 0.0;
                int32_t c = 0;
                for (int64_t q = s; q < e; ++q) {
                    if (T < t_min) break;
                    ++c;
                    int64_t i = tile_ids[q];
                    double dx = px - mean2[2 * i], dy = py - mean2[2 * i + 1];
                    const double *P = p2 + 4 * i;
                    double m = P[0] * dx * dx + 2.0 * P[1] * dx * dy + P[3] * dy * dy;
                    if (m >= tau_sq) continue;
                    double a = og[i] * exp(bx[i] * log1p(-m / tau_sq));
                    if (a > clamp) {
                        a = clamp;
                        hit[i] = 1; /* benign race: every writer stores 1 */
                    }
                    double w = a * T;
                    a0 += w * color[3 * i];
                    a1 += w * color[3 * i + 1];
                    a2 += w * color[3 * i + 2];
                    ws += w;
                    T *= 1.0 - a;
                }
                int64_t pix = (int64_t)y * width + x;
                rgb[3 * pix] = a0 + T * bg[0];
                rgb[3 * pix + 1] = a1 + T * bg[1];
                rgb[3 * pix + 2] = a2 + T * bg[2];
                asum[pix] = ws;
                tstop[pix] = T;
                count[pix] = c;
                visits_total += c;
            }
        }
    }
    return visits_total;
}

/* _tiles.py:59-127 tile_backward for every tile, partials per list position
 * (pg: K x 10 = mean2[2], p2[00,01,10,11], og, bx, color[3] -> 11 slots),
 * then the fixed-tile-order scatter of gradients.py:161-173 minus the
 * -P g P conversion (left to the caller, it is linear). */
void oracle_raster_backward(int width, int height, int tile, const int64_t *tile_start,
                            const int64_t *tile_ids, const double *mean2, const double *p2,
                            const double *og, const double *bx, const double *color,
                            const double *bg, double tau_sq, double clamp, double t_min,
                            const double *g_img, double *pg /* K x 11 scratch */,
                            double *g_mean2, double *g_p2, double *g_og, double *g_bx,
                            double *g_color) {
    int tx_n = (width + tile - 1) / tile, ty_n = (height + tile - 1) / tile;
    int ntiles = tx_n * ty_n;
#pragma omp parallel
    {
        int64_t cap = 0;
        double *abuf = NULL, *mbuf = NULL, *tbuf = NULL;
#pragma omp for schedule(dynamic, 2)
        for (int t = 0; t < ntiles; ++t) {
            int ty = t / tx_n, tx = t % tx_n;
            int ya = ty * tile, yb = (ty + 1) * tile < height ? (ty + 1) * tile : height;
            int xa = tx * tile, xb = (tx + 1) * tile < width ? (tx + 1) * tile : width;
            int64_t s = tile_start[t], e = tile_start[t + 1], k = e - s;
            memset(pg + 11 * s, 0, sizeof(double) * 11 * (size_t)k);
            if (k == 0) continue;
            if (k > cap) {
                free(abuf); free(mbuf); free(tbuf);
                cap = k;
                abuf = malloc(sizeof(double) * cap);
                mbuf = malloc(sizeof(double) * cap);
                tbuf = malloc(sizeof(double) * cap);
            }
            for (int y = ya; y < yb; ++y) {
                for (int x = xa; x < xb; ++x) {
                    double px = x + 0.5, py = y + 0.5;
                    double T = 1.0;
                    int64_t kstop = 0;
                    for (int64_t j = 0; j < k; ++j) {
                        if (T < t_min) break;
                        kstop = j + 1;
                        int64_t i = tile_ids[s + j];
                        double dx = px - mean2[2 * i], dy = py - mean2[2 * i + 1];
                        const double *P = p2 + 4 * i;
                        double m = P[0] * dx * dx + 2.0 * P[1] * dx * dy + P[3] * dy * dy;
                        tbuf[j] = T;
                        mbuf[j] = m;
                        if (m >= tau_sq) { abuf[j] = 0.0; continue; }
                        double a = og[i] * exp(bx[i] * log1p(-m / tau_sq));
                        if (a > clamp) a = clamp;
                        abuf[j] = a;
                        T *= 1.0 - a;
                    }
                    int64_t pix = (int64_t)y * width + x;
                    double g0 = g_img[3 * pix], g1 = g_img[3 * pix + 1], g2 = g_img[3 * pix + 2];
                    double suffix = (g0 * bg[0] + g1 * bg[1] + g2 * bg[2]) * T;
                    for (int64_t j = kstop - 1; j >= 0; --j) {
                        double a = abuf[j];
                        if (a == 0.0) continue;
                        int64_t i = tile_ids[s + j];
                        double *q = pg + 11 * (s + j);
                        double ti = tbuf[j], w = a * ti;
                        q[8] += w * g0;
                        q[9] += w * g1;
                        q[10] += w * g2;
                        double gc = g0 * color[3 * i] + g1 * color[3 * i + 1] + g2 * color[3 * i + 2];
                        double ga = gc * ti - suffix / (1.0 - a);
                        suffix += gc * w;
                        if (a >= clamp) continue;
                        double kv = a / og[i], xs = mbuf[j] / tau_sq;
                        double gk = ga * og[i];
                        q[6] += ga * kv;
                        q[7] += gk * kv * log1p(-xs);
                        double gm = gk * kv * (-bx[i] / (1.0 - xs)) / tau_sq;
                        double dx = px - mean2[2 * i], dy = py - mean2[2 * i + 1];
                        const double *P = p2 + 4 * i;
                        double pd0 = P[0] * dx + P[1] * dy;
                        double pd1 = P[1] * dx + P[3] * dy;
                        q[0] -= 2.0 * gm * pd0;
                        q[1] -= 2.0 * gm * pd1;
                        q[2] += gm * dx * dx;
                        q[3] += gm * dx * dy;
                        q[4] += gm * dx * dy;
                        q[5] += gm * dy * dy;
                    }
                }
            }
        }
        free(abuf); free(mbuf); free(tbuf);
    }
    /* fixed-order reduction over tiles (gradients.py:164-173) */
    for (int t = 0; t < ntiles; ++t) {
        for (int64_t q = tile_start[t]; q < tile_start[t + 1]; ++q) {
            int64_t i = tile_ids[q];
            const double *v = pg + 11 * q;
            g_mean2[2 * i] += v[0];
            g_mean2[2 * i + 1] += v[1];
            g_p2[4 * i] += v[2];
            g_p2[4 * i + 1] += v[3];
            g_p2[4 * i + 2] += v[4];
            g_p2[4 * i + 3] += v[5];
            g_og[i] += v[6];
            g_bx[i] += v[7];
            g_color[3 * i] += v[8];
            g_color[3 * i + 1] += v[9];
            g_color[3 * i + 2] += v[10];
        }
    }
}
