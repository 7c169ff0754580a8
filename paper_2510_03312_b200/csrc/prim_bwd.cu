// K10 prim_bwd: chain the accumulated screen-space gradients back to the raw
// N-D Beta parameters, one thread per primitive, fp64.
//
// Reference: gradients.py:161 (conic -> covariance), :179-204
// (_projection_backward), :207-280 (_slice_backward), :283-300
// (_clamp_eig_adjoint), :120-123 (regularisers, added once per step).
//
// The forward intermediates (~120 doubles per primitive at C = 4) are
// recomputed by the same prim_geom() the preprocess kernel runs instead of
// being stored: at 1M primitives storing them would cost ~1 GB of HBM writes
// and reads per view, recomputing costs ~2 kflop of fp64 per primitive.
#include <cuda_runtime.h>

#include <type_traits>

#include "ubs_common.cuh"

namespace ubs {

// adjoint of X -> V max(L, floor) V^T for symmetric X (gradients.py:283-300)
template <int D>
__device__ inline void floor_adjoint(const double (&lam)[D], const double (&E)[D][D], double floor,
                                     const double (&g)[D][D], double (&out)[D][D]) {
    double f[D], fp[D], K[D][D], gt[D][D], tmp[D][D];
    for (int i = 0; i < D; ++i) {
        f[i] = fmax(lam[i], floor);
        fp[i] = lam[i] > floor ? 1.0 : 0.0;
    }
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            const double dl = lam[i] - lam[j];
            K[i][j] = fabs(dl) > 1e-12 ? (f[i] - f[j]) / dl : 0.5 * (fp[i] + fp[j]);
        }
    // gt = E^T g E
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            double s = 0.0;
            for (int k = 0; k < D; ++k) s += g[i][k] * E[k][j];
            tmp[i][j] = s;
        }
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            double s = 0.0;
            for (int k = 0; k < D; ++k) s += E[k][i] * tmp[k][j];
            gt[i][j] = s * K[i][j];
        }
    // out = E gt E^T
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            double s = 0.0;
            for (int k = 0; k < D; ++k) s += E[i][k] * gt[k][j];
            tmp[i][j] = s;
        }
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            double s = 0.0;
            for (int k = 0; k < D; ++k) s += tmp[i][k] * E[j][k];
            out[i][j] = s;
        }
}

// Compaction: primitives whose chain can be nonzero (any of the 10 screen-space
// gradients nonzero, a saturated gate, or regularisers requested).
template <typename GT>
__global__ void __launch_bounds__(256)
prim_active_kernel(const GT *__restrict__ grad2d, const uint16_t *__restrict__ flags, int64_t n, int add_reg,
                   uint32_t *__restrict__ active, uint32_t *__restrict__ count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool need = false;
    if (i < n) {
        bool nz = false;
        if constexpr (sizeof(GT) == 4) {  // 3 aligned 16 B loads per 48 B record
            const float4 *q = reinterpret_cast<const float4 *>(grad2d + i * kGrad2dStride);
            const float4 x = q[0], y = q[1], z = q[2];
            nz = x.x != 0.f || x.y != 0.f || x.z != 0.f || x.w != 0.f || y.x != 0.f || y.y != 0.f ||
                 y.z != 0.f || y.w != 0.f || z.x != 0.f || z.y != 0.f;
        } else {
            const double2 *q = reinterpret_cast<const double2 *>(grad2d + i * kGrad2dStride);
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const double2 x = q[k];
                nz |= x.x != 0.0 || x.y != 0.0;
            }
        }
        need = nz || add_reg || (flags[i] & UBS_F_GATE_SAT);
    }
    // one atomic per CTA (a per-warp atomic on the single counter serialises
    // ~n/32 atomics per view)
    __shared__ uint32_t wcnt[8], cta_base;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) wcnt[wid] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            const uint32_t c = wcnt[w];
            wcnt[w] = t;
            t += c;
        }
        cta_base = t ? atomicAdd(count, t) : 0u;
    }
    __syncthreads();
    if (need) active[cta_base + wcnt[wid] + __popc(m & ((1u << lane) - 1u))] = (uint32_t)i;
}

#ifndef UBS_PRIM_BWD_MIN_CTAS
#define UBS_PRIM_BWD_MIN_CTAS 1
#endif
// kCached: the frame's scene statics are current (UbsView.statics): the
// forward's query-invariant half is read back instead of recomputed
template <int C, typename PT, typename GT, typename OT, bool kCached>
__global__ void __launch_bounds__(128, UBS_PRIM_BWD_MIN_CTAS)
prim_bwd_kernel(const UbsView v, GT *__restrict__ grad2d, OT *__restrict__ out, int add_reg,
                double reg_o, double reg_s, uint32_t *__restrict__ nonfinite, const uint32_t *__restrict__ active,
                const uint32_t *__restrict__ active_count) {
    constexpr int P = 14 + 6 * C;
    constexpr int CC = PrimGeom<C>::CC;
    int64_t limit = v.n;
    if (active) {
        const int64_t na = (int64_t)*active_count;
        // statics pay off once most primitives are active (their block-strided
        // reads are then dense); a sparse active set recomputes instead: both
        // variants are launched (grid-stride, so the idle one costs a few
        // microseconds), each keeps its regime
        if constexpr (kCached) {
            if (4 * na < v.n) return;
        } else {
            if (v.statics && 4 * na >= v.n) return;
        }
        limit = na;
    }
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < limit;
         t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = active ? (int64_t)active[t] : t;
    const PT *rec = reinterpret_cast<const PT *>(v.params) + i * P;
    PrimGeom<C> g;
    double mu_x[3];
    if constexpr (kCached) prim_geom_cached<C, PT>(rec, i, v, g, mu_x);
    else prim_geom<C, PT>(rec, v, g, mu_x);

    // grad2d holds raw per-pixel moments (raster_bwd kernels); the per-splat
    // factors of tile_backward (_tiles.py:114-127) are applied here once:
    //   g_mean2 = -2 c P sum(h d), g_P = c sum(h d d^T) (both off-diagonals get
    //   the dx dy moment), c = -beta / tau; g_og = sum(g_a a) / og
    GT *qp = grad2d + i * kGrad2dStride;
    GT q[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) {
        q[k] = qp[k];
        qp[k] = GT(0);  // consumed: every row the raster touched is active, so the buffer is left all-zero
    }
    const double p00 = g.p2[0], p01 = g.p2[1], p11 = g.p2[2];
    const double cm = -g.beta_x / v.set.tau_sq;
    const double sx = q[0], sy = q[1];
    const double gm2x = -2.0 * cm * (p00 * sx + p01 * sy), gm2y = -2.0 * cm * (p01 * sx + p11 * sy);
    const double gPa = cm * (double)q[2], gPc = cm * (double)q[3], gPb = cm * (double)q[4];
    const double g_og = g.og != 0.0 ? (double)q[5] / g.og : 0.0, g_bx = q[6];
    const double gcol[3] = {(double)q[7], (double)q[8], (double)q[9]};

    // conic -> covariance: g_cov2 = -P g_P P (gradients.py:161)
    double gc2[2][2];
    {
        // t = g_P P
        const double t00 = gPa * p00 + gPc * p01, t01 = gPa * p01 + gPc * p11;
        const double t10 = gPc * p00 + gPb * p01, t11 = gPc * p01 + gPb * p11;
        gc2[0][0] = -(p00 * t00 + p01 * t10);
        gc2[0][1] = -(p00 * t01 + p01 * t11);
        gc2[1][0] = -(p01 * t00 + p11 * t10);
        gc2[1][1] = -(p01 * t01 + p11 * t11);
    }
    // screen floor adjoint + symmetrisation (gradients.py:181-184)
    double gpre[2][2];
    if (g.floored2) {
        double lam[2], E[2][2];
        eigh2(g.raw2[0], g.raw2[1], g.raw2[2], lam, E);
        floor_adjoint<2>(lam, E, v.set.screen_cov_floor, gc2, gpre);
    } else {
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) gpre[a][b] = gc2[a][b];
    }
    double graw[2][2];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) graw[a][b] = 0.5 * (gpre[a][b] + gpre[b][a]);

    // projection adjoint (gradients.py:185-204)
    double gcov3[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double s = 0.0;
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c) s += g.V[r][a] * graw[r][c] * g.V[c][b];
            gcov3[a][b] = s;
        }
    double gV[2][3];
    for (int r = 0; r < 2; ++r)
        for (int b = 0; b < 3; ++b) {
            double s = 0.0;
            for (int c = 0; c < 2; ++c) {
                const double gs = graw[r][c] + graw[c][r];
                double vc = 0.0;
                for (int k = 0; k < 3; ++k) vc += g.V[c][k] * g.cov3[k][b];
                s += gs * vc;
            }
            gV[r][b] = s;
        }
    const double *Rc = v.cam.rot;
    double gJ[2][3];
    for (int r = 0; r < 2; ++r)
        for (int b = 0; b < 3; ++b) gJ[r][b] = gV[r][0] * Rc[3 * b] + gV[r][1] * Rc[3 * b + 1] + gV[r][2] * Rc[3 * b + 2];
    const double z = g.z, x = g.tcam[0], y = g.tcam[1], fx = v.cam.fx, fy = v.cam.fy;
    const double z2 = z * z, z3 = z2 * z;
    double gt[3];
    gt[0] = gm2x * fx / z + gJ[0][2] * (-fx / z2);
    gt[1] = gm2y * fy / z + gJ[1][2] * (-fy / z2);
    gt[2] = -gm2x * fx * x / z2 - gm2y * fy * y / z2 + gJ[0][0] * (-fx / z2) + gJ[1][1] * (-fy / z2) +
            gJ[0][2] * (2.0 * fx * x / z3) + gJ[1][2] * (2.0 * fy * y / z3);
    const double vis = g.visible ? 1.0 : 0.0;
    double gmean3[3];
    for (int k = 0; k < 3; ++k)
        gmean3[k] = (gt[0] * vis) * Rc[k] + (gt[1] * vis) * Rc[3 + k] + (gt[2] * vis) * Rc[6 + k];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) gcov3[a][b] *= vis;

    // slice adjoint (gradients.py:207-280)
    double o_mu_x[3], o_mu_q[CC], o_rot[3], o_sx[3], o_lqx[CC][3], o_sq[CC], o_bx, o_bq[CC], o_op, o_col[3];
    for (int k = 0; k < 3; ++k) { o_mu_x[k] = gmean3[k]; o_col[k] = gcol[k]; o_rot[k] = 0.0; o_sx[k] = 0.0; }
    o_bx = g_bx * g.beta_x;
    o_op = g_og * g.gate * g.opacity * (1.0 - g.opacity);
    const double g_gate = g_og * g.opacity;

    double gM[CC][CC], gdelta[CC], gbq[CC], gSxq[3][CC];
    for (int a = 0; a < CC; ++a) {
        gdelta[a] = 0.0;
        gbq[a] = 0.0;
        o_mu_q[a] = 0.0; o_sq[a] = 0.0; o_bq[a] = 0.0;
        for (int b = 0; b < CC; ++b) gM[a][b] = 0.0;
        for (int b = 0; b < 3; ++b) { gSxq[b][a] = 0.0; o_lqx[a][b] = 0.0; }
    }
    if constexpr (C > 0) {
        // gate (gradients.py:224-234); a saturated gate gives 0 * inf = NaN
        // exactly like the reference, which then raises GradientError
        const double gg = g_gate * g.gate;
        double gw[C];
        for (int k = 0; k < C; ++k) {
            const double gd = gg * (-4.0 * g.beta_q[k] / (1.0 - g.d_gate[k]));
            gbq[k] += gg * 4.0 * log1p(-g.d_gate[k]);
            const double s = g.s_tanh[k];
            const double msk = v.set.gate_symmetric ? (s > 0.0 ? 1.0 : (s < 0.0 ? -1.0 : 0.0)) : (s > 0.0 ? 1.0 : 0.0);
            gw[k] = gd * msk * 0.5 * (1.0 - s * s);
        }
        for (int a = 0; a < C; ++a)
            for (int b = 0; b < C; ++b) gM[a][b] += gw[a] * g.delta[b];
        for (int b = 0; b < C; ++b) {
            double s = 0.0;
            for (int a = 0; a < C; ++a) s += g.M[a][b] * gw[a];
            gdelta[b] += s;
        }
        // conditional mean (gradients.py:237-243)
        double gvv[C], gu[C];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < C; ++b) gSxq[a][b] = gmean3[a] * g.v[b];
        for (int b = 0; b < C; ++b) gvv[b] = g.Sxq[0][b] * gmean3[0] + g.Sxq[1][b] * gmean3[1] + g.Sxq[2][b] * gmean3[2];
        for (int a = 0; a < C; ++a)
            for (int b = 0; b < C; ++b) gM[a][b] += gvv[a] * g.u[b];
        for (int b = 0; b < C; ++b) {
            double s = 0.0;
            for (int a = 0; a < C; ++a) s += g.M[a][b] * gvv[a];
            gu[b] = s;
        }
        for (int k = 0; k < C; ++k) {
            gbq[k] += gu[k] * g.delta[k];
            gdelta[k] += gu[k] * g.beta_q[k];
        }
    }

    // conditional covariance through the PSD floor (gradients.py:246-257)
    double gsym[3][3];
    if (g.floored3) {
        double lam[3], E[3][3];
        eigh3(g.sym3, lam, E);
        floor_adjoint<3>(lam, E, g.floor_eps, gcov3, gsym);
    } else {
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) gsym[a][b] = gcov3[a][b];
    }
    double gSx[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) gSx[a][b] = 0.5 * (gsym[a][b] + gsym[b][a]);

    double gSq[CC][CC];
    if constexpr (C > 0) {
        double Q[C][C];  // M diag(beta_q)
        for (int a = 0; a < C; ++a)
            for (int b = 0; b < C; ++b) Q[a][b] = g.M[a][b] * g.beta_q[b];
        double gneg[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) gneg[a][b] = -gSx[a][b];
        // gneg H and gneg^T H (3xC)
        double nH[3][C], nTH[3][C];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < C; ++b) {
                double s1 = 0.0, s2 = 0.0;
                for (int k = 0; k < 3; ++k) {
                    s1 += gneg[a][k] * g.Sxq[k][b];
                    s2 += gneg[k][a] * g.Sxq[k][b];
                }
                nH[a][b] = s1;
                nTH[a][b] = s2;
            }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < C; ++b) {
                double s = 0.0;
                for (int k = 0; k < C; ++k) s += nH[a][k] * Q[b][k] + nTH[a][k] * Q[k][b];
                gSxq[a][b] += s;
            }
        double gq[C][C];  // H^T gneg H
        for (int a = 0; a < C; ++a)
            for (int b = 0; b < C; ++b) {
                double s = 0.0;
                for (int k = 0; k < 3; ++k) s += g.Sxq[k][a] * nH[k][b];
                gq[a][b] = s;
            }
        for (int a = 0; a < C; ++a)
            for (int b = 0; b < C; ++b) gM[a][b] += gq[a][b] * g.beta_q[b];
        for (int j = 0; j < C; ++j) {
            double s = 0.0;
            for (int k = 0; k < C; ++k) s += g.M[j][k] * gq[k][j];
            gbq[j] += s;
        }
        // inverse of the query block: g_Sq = -M gM M (gradients.py:260)
        double t[C][C];
        for (int a = 0; a < C; ++a)
            for (int b = 0; b < C; ++b) {
                double s = 0.0;
                for (int k = 0; k < C; ++k) s += gM[a][k] * g.M[k][b];
                t[a][b] = s;
            }
        for (int a = 0; a < C; ++a)
            for (int b = 0; b < C; ++b) {
                double s = 0.0;
                for (int k = 0; k < C; ++k) s += g.M[a][k] * t[k][b];
                gSq[a][b] = -s;
            }
        for (int k = 0; k < C; ++k) o_mu_q[k] = -gdelta[k];
    }

    // factor blocks (gradients.py:263-280)
    double gLx[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += (gSx[a][k] + gSx[k][a]) * g.Lx[k][b];
            if constexpr (C > 0) {
                for (int k = 0; k < C; ++k) s += gSxq[a][k] * g.lqx[k][b];
            }
            gLx[a][b] = s;
        }
    if constexpr (C > 0) {
        for (int a = 0; a < C; ++a)
            for (int b = 0; b < 3; ++b) {
                double s = 0.0;
                for (int k = 0; k < 3; ++k) s += gSxq[k][a] * g.Lx[k][b];
                for (int k = 0; k < C; ++k) s += (gSq[a][k] + gSq[k][a]) * g.lqx[k][b];
                o_lqx[a][b] = s;
            }
        for (int k = 0; k < C; ++k) {
            o_sq[k] = 2.0 * g.sq[k] * gSq[k][k] * g.sq[k];
            o_bq[k] = gbq[k] * g.beta_q[k];
        }
    }
    double gR[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) gR[a][b] = gLx[a][b] * g.sx[b];
    for (int k = 0; k < 3; ++k)
        o_sx[k] = (gLx[0][k] * g.R[0][k] + gLx[1][k] * g.R[1][k] + gLx[2][k] * g.R[2][k]) * g.sx[k];
    o_rot[0] = gR[2][1] - gR[1][2];
    o_rot[1] = gR[0][2] - gR[2][0];
    o_rot[2] = gR[1][0] - gR[0][1];

    if (add_reg) {
        // gradients.py:120-123 (once per step, not per view)
        o_op += reg_o * g.opacity * (1.0 - g.opacity);
        for (int k = 0; k < 3; ++k) o_sx[k] += reg_s * g.sx[k];
        if constexpr (C > 0) {
            for (int k = 0; k < C; ++k) o_sq[k] += reg_s * g.sq[k];
        }
    }

    // += into the packed gradient record (PARAM_FIELDS order)
    OT *dst = out + i * P;
    double vals[P];
    int o = 0;
    for (int k = 0; k < 3; ++k) vals[o++] = o_mu_x[k];
    for (int k = 0; k < C; ++k) vals[o++] = o_mu_q[k];
    for (int k = 0; k < 3; ++k) vals[o++] = o_rot[k];
    for (int k = 0; k < 3; ++k) vals[o++] = o_sx[k];
    for (int a = 0; a < C; ++a)
        for (int b = 0; b < 3; ++b) vals[o++] = o_lqx[a][b];
    for (int k = 0; k < C; ++k) vals[o++] = o_sq[k];
    vals[o++] = o_bx;
    for (int k = 0; k < C; ++k) vals[o++] = o_bq[k];
    vals[o++] = o_op;
    for (int k = 0; k < 3; ++k) vals[o++] = o_col[k];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const OT nv = (OT)((double)dst[k] + vals[k]);
        dst[k] = nv;
        bad |= !isfinite((double)nv);
    }
    if (bad && nonfinite) atomicOr(nonfinite, 1u);
    }
}

template <int C, typename PT>
static void launch_bwd(const UbsView &v, const UbsGradBuffers &gb, int add_reg, bool g2d_f64, cudaStream_t s) {
    // grid-stride: at most 8 CTAs per SM's worth (255 registers: 2 resident per SM)
    const unsigned blocks = (unsigned)min((int64_t)148 * 16, (v.n + 127) / 128);
    if (gb.active) {
        const unsigned ab = (unsigned)((v.n + 255) / 256);
        cudaMemsetAsync(gb.active_count, 0, sizeof(uint32_t), s);
        if (g2d_f64)
            prim_active_kernel<double><<<ab, 256, 0, s>>>((const double *)gb.grad2d, gb.flags, v.n, add_reg, gb.active,
                                                          gb.active_count);
        else
            prim_active_kernel<float><<<ab, 256, 0, s>>>((const float *)gb.grad2d, gb.flags, v.n, add_reg, gb.active,
                                                         gb.active_count);
    }
    auto run = [&](auto cached) {
        constexpr bool kC = decltype(cached)::value;
        if (g2d_f64) {
            if (gb.grad_f64)
                prim_bwd_kernel<C, PT, double, double, kC><<<blocks, 128, 0, s>>>(
                    v, (double *)gb.grad2d, (double *)gb.grad_params, add_reg, gb.reg_opacity, gb.reg_scale, gb.nonfinite, gb.active, gb.active_count);
            else
                prim_bwd_kernel<C, PT, double, float, kC><<<blocks, 128, 0, s>>>(
                    v, (double *)gb.grad2d, (float *)gb.grad_params, add_reg, gb.reg_opacity, gb.reg_scale, gb.nonfinite, gb.active, gb.active_count);
        } else {
            if (gb.grad_f64)
                prim_bwd_kernel<C, PT, float, double, kC><<<blocks, 128, 0, s>>>(
                    v, (float *)gb.grad2d, (double *)gb.grad_params, add_reg, gb.reg_opacity, gb.reg_scale, gb.nonfinite, gb.active, gb.active_count);
            else
                prim_bwd_kernel<C, PT, float, float, kC><<<blocks, 128, 0, s>>>(
                    v, (float *)gb.grad2d, (float *)gb.grad_params, add_reg, gb.reg_opacity, gb.reg_scale, gb.nonfinite, gb.active, gb.active_count);
        }
    };
    if (v.statics) run(std::true_type{});  // dense active sets (or no compaction): read the statics back
    if (!v.statics || gb.active) run(std::false_type{});  // sparse active sets: recompute
}

}  // namespace ubs

using namespace ubs;

extern "C" int ubs_prim_backward(const UbsView *v, const UbsGradBuffers *gb, int32_t add_regularisers,
                                 ubs_stream_t stream) {
    if (!v || !gb || !gb->grad2d || !gb->grad_params) return UBS_E_ARGS;
    if (gb->active && (!gb->flags || !gb->active_count)) return UBS_E_ARGS;
    if (v->n == 0) return UBS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const bool pf64 = v->param_f64 != 0, g64 = gb->grad2d_f64 != 0;
    switch (v->n_dims) {
        case 3: pf64 ? launch_bwd<0, double>(*v, *gb, add_regularisers, g64, s)
                     : launch_bwd<0, float>(*v, *gb, add_regularisers, g64, s); break;
        case 6: pf64 ? launch_bwd<3, double>(*v, *gb, add_regularisers, g64, s)
                     : launch_bwd<3, float>(*v, *gb, add_regularisers, g64, s); break;
        case 7: pf64 ? launch_bwd<4, double>(*v, *gb, add_regularisers, g64, s)
                     : launch_bwd<4, float>(*v, *gb, add_regularisers, g64, s); break;
        default: return UBS_E_ARGS;
    }
    UBS_CUDA_CHECK();
    return UBS_OK;
}

UBS_CHECKED_ACCESSOR(prim_bwd)
