// Shared device code for the B200 UBS render path (sm_100a).
//
// The per-primitive math (conditioning + projection) is evaluated in fp64,
// one thread per primitive.  B200 runs fp64 at half the fp32 rate, and the
// survey measured that fp32 geometry mis-bins primitives and reorders depth
// ties, so bit-exact binning needs fp64 here.  The same
// routine feeds the preprocess kernel and the backward chain (which
// recomputes instead of storing ~120 doubles per primitive).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ubs_b200.h"

namespace ubs {

// Bounds-checked build (-DUBS_CHECKED; tests/test_gpu_checked.py): every
// guarded index is tested on the device, a failing test sets its bit in
// g_checked_status (read with ubs_debug_checked_status) and the access is
// skipped.  The product build compiles the guards away.  (compute-sanitizer
// is not available on the GPU pool, so this is the memory-safety evidence.)
#ifdef UBS_CHECKED
__device__ unsigned int g_checked_status;
__device__ __forceinline__ bool ubs_guard(bool ok, unsigned int bit) {
    if (!ok) atomicOr(&g_checked_status, bit);
    return ok;
}
#define UBS_GUARD(cond, bit) ::ubs::ubs_guard((cond), (bit))
// one status word per translation unit (whole-program compilation): each .cu
// exports its own reader, ubs_debug_checked_<tu>
#define UBS_CHECKED_ACCESSOR(tu)                                                                  \
    extern "C" int ubs_debug_checked_##tu(unsigned int *out, int reset) {                        \
        if (cudaDeviceSynchronize() != cudaSuccess) return -2;                                     \
        if (cudaMemcpyFromSymbol(out, ::ubs::g_checked_status, sizeof(unsigned int)) != cudaSuccess) \
            return -2;                                                                             \
        if (reset) {                                                                               \
            const unsigned int z = 0;                                                              \
            cudaMemcpyToSymbol(::ubs::g_checked_status, &z, sizeof(z));                             \
        }                                                                                          \
        return 0;                                                                                  \
    }
#else
#define UBS_GUARD(cond, bit) true
#define UBS_CHECKED_ACCESSOR(tu)
#endif
// guard bits
enum : unsigned int {
    kChkOwner = 1u << 0,      // binning FlatStage owner[] slot
    kChkLocate = 1u << 1,     // binning flat index -> (rank lane, bucket)
    kChkBucket = 1u << 2,     // binning per-warp bucket counter index
    kChkEntry = 1u << 3,      // binning level-1 entry write
    kChkList = 1u << 4,       // binning level-2 tile-list write
    kChkRank = 1u << 5,       // depth sort slot / rank write
    kChkGrid = 1u << 6,       // preprocess tile-grid corner
    kChkSplat = 1u << 7,      // raster shared splat index / ballot word
    kChkHit = 1u << 8,        // raster alpha_clamped write
    kChkFix = 1u << 9,        // raster fix-up list write
    kChkPixel = 1u << 10,     // raster image write
    kChkPair = 1u << 11,      // raster / backward tile-list read
    kChkGrad = 1u << 12,      // backward grad2d / partial write
};

constexpr int kTile = 16;
constexpr int kTileThreads = kTile * kTile;
constexpr uint64_t kInvisibleKey = 0xFFFFFFFFFFFFFFFFull;
constexpr int kGrad2dStride = 12;  // 10 raw moment sums (see ubs_b200.h UbsGradBuffers.grad2d) + pad[2]

// fp64 raster record: exactly the operands tile_forward reads (_tiles.py:36-50).
struct __align__(16) Rec64 {
    double mx, my;          // mean2
    double p00, p01, p11;   // inverse screen covariance (raster.py:436-446)
    double og, bx;          // gated opacity, spatial exponent
    double cr, cg, cb;      // raw colour (not activated, raster.py:297)
};
static_assert(sizeof(Rec64) == 80, "Rec64 layout");

// fp32 raster record, 64 B = 4 x 16 B vector loads.
//  r0: fx, fy = floor(mean2) as exact floats, ox, oy = 0.5 - frac(mean2)
//      -> dx = (px - fx) + ox: the first difference is exact (integers
//      < 2^24), so dx is accurate to ~1e-7 px at any image size
//  r1: u00, u01, u11 (P = U^T U, m = (u00 dx + u01 dy)^2 + (u11 dy)^2),
//      tau + E (E bounds |m32 - m64| over the splat's support)
//  r2: beta_x, colour
//  r3: eb = beta_x * E, og, qc (lg2/ex2 approximation bound), log2(og)
struct __align__(16) Rec32 {
    float4 r0, r1, r2, r3;
};
static_assert(sizeof(Rec32) == 64, "Rec32 layout");

// --- fp64 helpers with contraction disabled: the tile loops must round like
// numba (no FMA contraction by default) so the contributor count decision
// T < t_min matches the reference.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

template <typename PT>
__device__ __forceinline__ double ld(const PT *p, int64_t i) { return (double)p[i]; }

// ---------------------------------------------------------------------------
// small dense fp64 linear algebra
// ---------------------------------------------------------------------------

// Cholesky of a CxC SPD matrix (row-major), LAPACK dpotrf failure rule:
// a pivot that is not > 0 (or NaN) fails.
template <int C>
__device__ __forceinline__ bool cholesky(const double (&A)[C][C], double (&L)[C][C]) {
#pragma unroll
    for (int j = 0; j < C; ++j) {
        double s = A[j][j];
#pragma unroll
        for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
        if (!(s > 0.0)) return false;
        const double d = sqrt(s), inv_d = 1.0 / d;
        L[j][j] = d;
#pragma unroll
        for (int i = j + 1; i < C; ++i) {
            double t = A[i][j];
#pragma unroll
            for (int k = 0; k < j; ++k) t -= L[i][k] * L[j][k];
            L[i][j] = t * inv_d;
        }
#pragma unroll
        for (int i = 0; i < j; ++i) L[i][j] = 0.0;
    }
    return true;
}

// inverse from a Cholesky factor: A^-1 = L^-T L^-1
template <int C>
__device__ __forceinline__ void chol_inverse(const double (&L)[C][C], double (&M)[C][C]) {
    double Li[C][C], inv[C];
#pragma unroll
    for (int j = 0; j < C; ++j) inv[j] = 1.0 / L[j][j];
#pragma unroll
    for (int j = 0; j < C; ++j) {
#pragma unroll
        for (int i = 0; i < C; ++i) Li[i][j] = 0.0;
        Li[j][j] = inv[j];
#pragma unroll
        for (int i = j + 1; i < C; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = j; k < i; ++k) s += L[i][k] * Li[k][j];
            Li[i][j] = -s * inv[i];
        }
    }
#pragma unroll
    for (int i = 0; i < C; ++i)
#pragma unroll
        for (int j = 0; j < C; ++j) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < C; ++k) s += Li[k][i] * Li[k][j];
            M[i][j] = s;
        }
}

// Symmetric 3x3 eigen-decomposition by cyclic Jacobi; ascending eigenvalues,
// eigenvectors as columns of V.  Only reached for primitives whose
// conditioned covariance needs the PSD floor (rare), so robustness beats speed.
__device__ inline void eigh3(const double (&A)[3][3], double (&w)[3], double (&V)[3][3]) {
    double a[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            a[i][j] = A[i][j];
            V[i][j] = (i == j) ? 1.0 : 0.0;
        }
    for (int sweep = 0; sweep < 32; ++sweep) {
        double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
        double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
        if (off == 0.0 || off <= 1e-300 || off < 1e-18 * scale) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double apq = a[p][q];
                if (apq == 0.0) continue;
                double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
                double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {
                    double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - s * akq;
                    a[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - s * aqk;
                    a[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {
                    double vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = c * vkp - s * vkq;
                    V[k][q] = s * vkp + c * vkq;
                }
            }
    }
    for (int i = 0; i < 3; ++i) w[i] = a[i][i];
    // sort ascending (selection sort, swap columns)
    for (int i = 0; i < 2; ++i) {
        int m = i;
        for (int j = i + 1; j < 3; ++j)
            if (w[j] < w[m]) m = j;
        if (m != i) {
            double t = w[i]; w[i] = w[m]; w[m] = t;
            for (int k = 0; k < 3; ++k) { double u = V[k][i]; V[k][i] = V[k][m]; V[k][m] = u; }
        }
    }
}

// Symmetric 2x2 eigen-decomposition [[a,b],[b,d]], ascending, columns of V.
__device__ inline void eigh2(double a, double b, double d, double (&w)[2], double (&V)[2][2]) {
    double h = 0.5 * (a + d), g = 0.5 * (a - d);
    double r = sqrt(g * g + b * b);
    w[0] = h - r;
    w[1] = h + r;
    if (b == 0.0) {
        if (a <= d) { V[0][0] = 1; V[1][0] = 0; V[0][1] = 0; V[1][1] = 1; }
        else { V[0][0] = 0; V[1][0] = 1; V[0][1] = 1; V[1][1] = 0; }
        if (a == d) { V[0][0] = 1; V[1][0] = 0; V[0][1] = 0; V[1][1] = 1; }
        return;
    }
    // eigenvector of the larger eigenvalue, from the better conditioned row
    double x1, y1;
    if (g >= 0.0) { x1 = g + r; y1 = b; } else { x1 = b; y1 = r - g; }
    double nrm = sqrt(x1 * x1 + y1 * y1);
    x1 /= nrm; y1 /= nrm;
    V[0][1] = x1; V[1][1] = y1;
    V[0][0] = -y1; V[1][0] = x1;
}

// ---------------------------------------------------------------------------
// Per-primitive conditioning + projection (fp64).
// slicing.py:185-235 (with covariance.py:57-159, kernels.py:18-25) and
// raster.py:95-134.
// ---------------------------------------------------------------------------
template <int C>
struct PrimGeom {
    static constexpr int CC = C > 0 ? C : 1;
    // activated parameters
    double sx[3], sq[CC], lqx[CC][3], R[3][3], Lx[3][3];
    double beta_x, beta_q[CC], opacity, color[3];
    // conditioning
    double Sxq[3][CC], M[CC][CC];
    double delta[CC], u[CC], v[CC], mean3[3];
    double sym3[3][3], cov3[3][3], floor_eps;
    double s_tanh[CC], d_gate[CC], gate, og;
    double log2_op, lsum;  // log2(opacity) (query-invariant) and the gate's log: log2(og) = log2_op + lsum log2(e)
    bool valid, floored3;
    // projection
    double tcam[3], z, mean2[2], V[2][3], raw2[3], cov2[3], p2[3], radii[2];
    bool in_front, floored2, visible;
};

template <int C, typename PT>
__device__ inline void load_params(const PT *rec, double (&mu_x)[3], double *mu_q, double (&rot)[3],
                                   double (&sxr)[3], double *lqx /*C*3*/, double *sqr, double &bxr,
                                   double *bqr, double &oraw, double (&col)[3]) {
    int o = 0;
    for (int k = 0; k < 3; ++k) mu_x[k] = (double)rec[o++];
    for (int k = 0; k < C; ++k) mu_q[k] = (double)rec[o++];
    for (int k = 0; k < 3; ++k) rot[k] = (double)rec[o++];
    for (int k = 0; k < 3; ++k) sxr[k] = (double)rec[o++];
    for (int k = 0; k < 3 * C; ++k) lqx[k] = (double)rec[o++];
    for (int k = 0; k < C; ++k) sqr[k] = (double)rec[o++];
    bxr = (double)rec[o++];
    for (int k = 0; k < C; ++k) bqr[k] = (double)rec[o++];
    oraw = (double)rec[o++];
    for (int k = 0; k < 3; ++k) col[k] = (double)rec[o++];
}

__device__ __forceinline__ double sigmoid64(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

// R = I + A (A skew from (a1, a2, a3), covariance.py:57-72) and Lx = R diag(sx)
template <int C>
__device__ __forceinline__ void static_rotation(const double (&rot)[3], PrimGeom<C> &g) {
    g.R[0][0] = 1.0;     g.R[0][1] = -rot[2]; g.R[0][2] = rot[1];
    g.R[1][0] = rot[2];  g.R[1][1] = 1.0;     g.R[1][2] = -rot[0];
    g.R[2][0] = -rot[1]; g.R[2][1] = rot[0];  g.R[2][2] = 1.0;
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) g.Lx[i][k] = g.R[i][k] * g.sx[k];
}

// Sx = Lx Lx^T (covariance.py:104-119)
template <int C>
__device__ __forceinline__ void static_sx(const PrimGeom<C> &g, double (&Sx)[3][3]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            Sx[i][j] = g.Lx[i][0] * g.Lx[j][0] + g.Lx[i][1] * g.Lx[j][1] + g.Lx[i][2] * g.Lx[j][2];
}

// raw = Sx - Sxq M diag(beta_q) Sqx (slicing.py:210-211), sym3 = (raw + raw^T) / 2
template <int C>
__device__ __forceinline__ void static_sym3(PrimGeom<C> &g, const double (&Sx)[3][3]) {
    double raw[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) raw[i][j] = Sx[i][j];
    if constexpr (C > 0) {
        double H[3][C];  // Sxq M
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < C; ++k) {
                double s = 0.0;
                for (int j = 0; j < C; ++j) s += g.Sxq[i][j] * g.M[j][k];
                H[i][k] = s;
            }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double s = 0.0;
                for (int k = 0; k < C; ++k) s += H[i][k] * g.beta_q[k] * g.Sxq[j][k];
                raw[i][j] = Sx[i][j] - s;
            }
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) g.sym3[i][j] = 0.5 * (raw[i][j] + raw[j][i]);
}

// Query-invariant half of slice_scene (slicing.py:185-235): activations,
// Sx, the query block inverse M, Sxq, the conditional covariance with its PSD
// floor, opacity and beta_x.  Depends on the parameters and psd_floor_scale
// only, so a scene's statics are computed once per parameter version
// (ubs_scene_statics) and shared by every view; prim_view does the rest with
// the same operations in the same order, so both routes give identical bits.
template <int C, typename PT>
__device__ inline void prim_static(const PT *rec, const UbsSettings &set, PrimGeom<C> &g, double (&mu_x)[3],
                                   double (&mu_q)[PrimGeom<C>::CC]) {
    constexpr int CC = PrimGeom<C>::CC;
    double rot[3], sxr[3], lq[CC * 3], sqr[CC], bxr, bqr[CC], oraw;
    load_params<C>(rec, mu_x, mu_q, rot, sxr, lq, sqr, bxr, bqr, oraw, g.color);

    for (int k = 0; k < 3; ++k) g.sx[k] = exp(sxr[k]);
    static_rotation<C>(rot, g);
    double Sx[3][3];
    static_sx<C>(g, Sx);

    g.beta_x = 4.0 * exp(bxr);
    g.opacity = sigmoid64(oraw);
    g.log2_op = log2(g.opacity);
    g.valid = true;

    if constexpr (C > 0) {
        for (int k = 0; k < C; ++k) {
            g.sq[k] = exp(sqr[k]);
            g.beta_q[k] = exp(bqr[k]);
            for (int j = 0; j < 3; ++j) g.lqx[k][j] = lq[3 * k + j];
        }
        double Sq[C][C];
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < C; ++k)
                g.Sxq[i][k] = g.Lx[i][0] * g.lqx[k][0] + g.Lx[i][1] * g.lqx[k][1] + g.Lx[i][2] * g.lqx[k][2];
        bool finite = true;
        for (int i = 0; i < C; ++i)
            for (int j = 0; j < C; ++j) {
                double s = g.lqx[i][0] * g.lqx[j][0] + g.lqx[i][1] * g.lqx[j][1] + g.lqx[i][2] * g.lqx[j][2];
                if (i == j) s += g.sq[i] * g.sq[i];
                Sq[i][j] = s;
                finite &= isfinite(s);
            }
        // invert_query_block (covariance.py:122-149): Cholesky test, one
        // 1e-8 jitter, still failing -> degenerate with identity slot
        double L[C][C];
        bool ok = finite && cholesky<C>(Sq, L);
        if (finite && !ok) {
            for (int i = 0; i < C; ++i) Sq[i][i] += 1e-8;
            ok = cholesky<C>(Sq, L);
        }
        if (ok) {
            chol_inverse<C>(L, g.M);
        } else {
            g.valid = false;
            for (int i = 0; i < C; ++i)
                for (int j = 0; j < C; ++j) g.M[i][j] = (i == j) ? 1.0 : 0.0;
        }
    }

    // conditional covariance, symmetrised (slicing.py:210-212), then the PSD
    // eigen floor (slicing.py:212-222)
    static_sym3<C>(g, Sx);
    g.floor_eps = set.psd_floor_scale * (Sx[0][0] + Sx[1][1] + Sx[2][2]) / 3.0;
    {
        // cheap test first: sym - eps I positive definite <=> lambda_min > eps
        double T[3][3], L3[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) T[i][j] = g.sym3[i][j] - (i == j ? g.floor_eps : 0.0);
        bool pd = cholesky<3>(T, L3);
        g.floored3 = false;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) g.cov3[i][j] = g.sym3[i][j];
        if (!pd) {
            double w[3], Vv[3][3];
            eigh3(g.sym3, w, Vv);
            if (w[0] < g.floor_eps) {
                g.floored3 = true;
                for (int k = 0; k < 3; ++k) w[k] = fmax(w[k], g.floor_eps);
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j)
                        g.cov3[i][j] = Vv[i][0] * w[0] * Vv[j][0] + Vv[i][1] * w[1] * Vv[j][1] +
                                       Vv[i][2] * w[2] * Vv[j][2];
            }
        }
    }
}

// Per-view half of slice_scene (conditional mean slicing.py:205-208, opacity
// gate :224-228) and project_scene (raster.py:99-131) on top of prim_static.
// exact_s: always evaluate s_tanh (the debug dump and the backward read it);
// otherwise an asymmetric-gate dimension with 0.5 dr <= 0 skips tanh and
// log1p: there s = tanh(0.5 dr) <= 0, d = max(s, 0) = 0 and 4 beta log1p(-0)
// adds a signed zero, so lsum and the gate are bit-identical (s_tanh is then
// only known to be <= 0, all the flags use).
template <int C>
__device__ inline void prim_view(PrimGeom<C> &g, const double (&mu_x)[3], const double (&mu_q)[PrimGeom<C>::CC],
                                 const UbsView &v, bool exact_s = true) {
    double mean3[3] = {mu_x[0], mu_x[1], mu_x[2]};
    g.gate = 1.0;
    g.lsum = 0.0;
    if constexpr (C > 0) {
        // conditional mean (slicing.py:205-208)
        for (int k = 0; k < C; ++k) {
            g.delta[k] = v.query[k] - mu_q[k];
            g.u[k] = g.beta_q[k] * g.delta[k];
        }
        for (int i = 0; i < C; ++i) {
            double s = 0.0;
            for (int k = 0; k < C; ++k) s += g.M[i][k] * g.u[k];
            g.v[i] = s;
        }
        for (int i = 0; i < 3; ++i) {
            double s = 0.0;
            for (int k = 0; k < C; ++k) s += g.Sxq[i][k] * g.v[k];
            mean3[i] = mu_x[i] + s;
        }
        // opacity gate (slicing.py:224-228)
        double lsum = 0.0;
        for (int i = 0; i < C; ++i) {
            double dr = 0.0;
            for (int k = 0; k < C; ++k) dr += g.M[i][k] * g.delta[k];
            const double h = 0.5 * dr;
            if (!exact_s && !v.set.gate_symmetric && !(h > 0.0)) {
                g.s_tanh[i] = h;  // <= 0 (or NaN, as tanh would give)
                g.d_gate[i] = 0.0;
                continue;
            }
            double s = tanh(h);
            g.s_tanh[i] = s;
            double d = v.set.gate_symmetric ? fabs(s) : fmax(s, 0.0);
            g.d_gate[i] = d;
            lsum += 4.0 * g.beta_q[i] * log1p(-d);
        }
        g.gate = exp(lsum);
        g.lsum = lsum;
    }
    for (int i = 0; i < 3; ++i) g.mean3[i] = mean3[i];
    g.og = g.opacity * g.gate;

    // projection (raster.py:99-131)
    const double *Rc = v.cam.rot;
    for (int i = 0; i < 3; ++i)
        g.tcam[i] = Rc[3 * i] * mean3[0] + Rc[3 * i + 1] * mean3[1] + Rc[3 * i + 2] * mean3[2] + v.cam.trans[i];
    g.in_front = g.tcam[2] > v.set.near_plane;
    g.z = g.in_front ? g.tcam[2] : 1.0;
    const double z = g.z, x = g.tcam[0], y = g.tcam[1];
    const double fx = v.cam.fx, fy = v.cam.fy;
    const double iz = 1.0 / z;
    g.mean2[0] = fx * x * iz + v.cam.cx;
    g.mean2[1] = fy * y * iz + v.cam.cy;
    double J[2][3] = {{fx * iz, 0.0, -fx * x * iz * iz}, {0.0, fy * iz, -fy * y * iz * iz}};
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k) g.V[i][k] = J[i][0] * Rc[k] + J[i][1] * Rc[3 + k] + J[i][2] * Rc[6 + k];
    double VC[2][3];
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k)
            VC[i][k] = g.V[i][0] * g.cov3[0][k] + g.V[i][1] * g.cov3[1][k] + g.V[i][2] * g.cov3[2][k];
    double r00 = VC[0][0] * g.V[0][0] + VC[0][1] * g.V[0][1] + VC[0][2] * g.V[0][2];
    double r01 = VC[0][0] * g.V[1][0] + VC[0][1] * g.V[1][1] + VC[0][2] * g.V[1][2];
    double r10 = VC[1][0] * g.V[0][0] + VC[1][1] * g.V[0][1] + VC[1][2] * g.V[0][2];
    double r11 = VC[1][0] * g.V[1][0] + VC[1][1] * g.V[1][1] + VC[1][2] * g.V[1][2];
    g.raw2[0] = r00;
    g.raw2[1] = 0.5 * (r01 + r10);
    g.raw2[2] = r11;
    {
        double w[2], E[2][2];
        // the floor test needs only the smaller eigenvalue (eigh2's own
        // arithmetic, so the same bits); eigenvectors only for floored splats
        {
            const double h = 0.5 * (g.raw2[0] + g.raw2[2]), gg = 0.5 * (g.raw2[0] - g.raw2[2]);
            const double r = sqrt(gg * gg + g.raw2[1] * g.raw2[1]);
            g.floored2 = h - r < v.set.screen_cov_floor;
        }
        if (g.floored2) {
            eigh2(g.raw2[0], g.raw2[1], g.raw2[2], w, E);
            double f0 = fmax(w[0], v.set.screen_cov_floor), f1 = fmax(w[1], v.set.screen_cov_floor);
            g.cov2[0] = E[0][0] * f0 * E[0][0] + E[0][1] * f1 * E[0][1];
            g.cov2[1] = E[0][0] * f0 * E[1][0] + E[0][1] * f1 * E[1][1];
            g.cov2[2] = E[1][0] * f0 * E[1][0] + E[1][1] * f1 * E[1][1];
        } else {
            g.cov2[0] = g.raw2[0];
            g.cov2[1] = g.raw2[1];
            g.cov2[2] = g.raw2[2];
        }
    }
    const double a = g.cov2[0], b = g.cov2[1], d = g.cov2[2];
    const double idet = 1.0 / (a * d - b * b);
    g.p2[0] = d * idet;
    g.p2[1] = -b * idet;
    g.p2[2] = a * idet;
    g.radii[0] = sqrt(v.set.tau_sq * a);
    g.radii[1] = sqrt(v.set.tau_sq * d);
    const double mg = v.set.cull_margin;
    const double lox = g.mean2[0] - g.radii[0], hix = g.mean2[0] + g.radii[0];
    const double loy = g.mean2[1] - g.radii[1], hiy = g.mean2[1] + g.radii[1];
    bool on_screen = (hix >= -mg) && (lox <= v.cam.width + mg) && (hiy >= -mg) && (loy <= v.cam.height + mg);
    g.visible = g.in_front && on_screen && g.valid;
}

template <int C, typename PT>
__device__ inline void prim_geom(const PT *rec, const UbsView &v, PrimGeom<C> &g, double (&mu_x)[3]) {
    double mu_q[PrimGeom<C>::CC];
    prim_static<C, PT>(rec, v.set, g, mu_x, mu_q);
    prim_view<C>(g, mu_x, mu_q, v);
}

// Scene statics, tiled structure of arrays: blocks of kStaticBlock
// primitives, each block holding D fp64 fields then R raw fields at parameter
// precision, field-major inside the block (every field load of a warp is one
// coalesced access at a constant offset from the block base).
//   fp64: beta_q[C] | M upper triangle, row-major [C(C+1)/2] | Sxq[3][C] |
//         cov3[3][3] | opacity | beta_x | floor_eps | flags | log2(opacity)
//   raw:  mu_x[3] | mu_q[C] | color[3]
// flags: 1 = valid (query block invertible), 2 = PSD-floored.
constexpr int kStaticBlock = 128;

template <int C>
struct StaticLayout {
    static constexpr int kBetaQ = 0;
    static constexpr int kM = kBetaQ + C;
    static constexpr int kSxq = kM + C * (C + 1) / 2;
    static constexpr int kCov3 = kSxq + 3 * C;
    static constexpr int kOpacity = kCov3 + 9;
    static constexpr int kBetaX = kOpacity + 1;
    static constexpr int kFloorEps = kBetaX + 1;
    static constexpr int kFlags = kFloorEps + 1;
    static constexpr int kLog2Op = kFlags + 1;
    static constexpr int D = kLog2Op + 1;
    static constexpr int R = 6 + C;
};

__host__ __device__ inline size_t static_block_bytes(int n_dims, int param_f64) {
    const int C = n_dims - 3;
    const int D = C + C * (C + 1) / 2 + 3 * C + 14;
    const int R = 6 + C;
    return (size_t)kStaticBlock * (size_t)(8 * D + (param_f64 ? 8 : 4) * R);
}

__host__ __device__ inline size_t statics_bytes(int64_t n, int n_dims, int param_f64) {
    return (size_t)((n + kStaticBlock - 1) / kStaticBlock) * static_block_bytes(n_dims, param_f64);
}

// fp64 and raw field bases of primitive i (field f at [f * kStaticBlock])
template <int C, typename PT>
__device__ __forceinline__ void static_slot(void *buf, int64_t i, double *&d, PT *&r) {
    using L = StaticLayout<C>;
    constexpr size_t kBlock = (size_t)kStaticBlock * (8 * L::D + sizeof(PT) * L::R);
    char *blk = reinterpret_cast<char *>(buf) + (size_t)(i / kStaticBlock) * kBlock;
    const int t = (int)(i % kStaticBlock);
    d = reinterpret_cast<double *>(blk) + t;
    r = reinterpret_cast<PT *>(blk + (size_t)kStaticBlock * 8 * L::D) + t;
}

template <int C, typename PT>
__device__ inline void store_statics(void *buf, int64_t i, const PrimGeom<C> &g, const double (&mu_x)[3],
                                     const double (&mu_q)[PrimGeom<C>::CC]) {
    using L = StaticLayout<C>;
    constexpr int S = kStaticBlock;
    double *d;
    PT *r;
    static_slot<C, PT>(buf, i, d, r);
    for (int k = 0; k < C; ++k) d[(L::kBetaQ + k) * S] = g.beta_q[k];
    int o = L::kM;
    for (int a = 0; a < C; ++a)
        for (int b = a; b < C; ++b) d[(o++) * S] = g.M[a][b];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < C; ++k) d[(L::kSxq + a * C + k) * S] = g.Sxq[a][k];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d[(L::kCov3 + 3 * a + b) * S] = g.cov3[a][b];
    d[L::kOpacity * S] = g.opacity;
    d[L::kBetaX * S] = g.beta_x;
    d[L::kFloorEps * S] = g.floor_eps;
    d[L::kFlags * S] = (double)((g.valid ? 1 : 0) | (g.floored3 ? 2 : 0));
    d[L::kLog2Op * S] = g.log2_op;
    for (int k = 0; k < 3; ++k) r[k * S] = (PT)mu_x[k];
    for (int k = 0; k < C; ++k) r[(3 + k) * S] = (PT)mu_q[k];
    for (int k = 0; k < 3; ++k) r[(3 + C + k) * S] = (PT)g.color[k];
}

// M is symmetric bit for bit (chol_inverse sums Li[k][i] Li[k][j] in the same
// k order for (i, j) and (j, i)), so its upper triangle restores it exactly;
// the floored cov3 (V w V^T with left-to-right products) is not, so all nine
// entries are kept.
// kGlobal: buf is device memory (read-only path); else a shared-memory copy
// of the primitive's statics block (preprocess_views_kernel)
template <typename T, bool kGlobal>
__device__ __forceinline__ T ld_statics(const T *p) {
    if constexpr (kGlobal) return __ldg(p);
    else return *p;
}

template <int C, typename PT, bool kGlobal = true>
__device__ inline void load_statics(const void *buf, int64_t i, PrimGeom<C> &g, double (&mu_x)[3],
                                    double (&mu_q)[PrimGeom<C>::CC]) {
    using L = StaticLayout<C>;
    constexpr int S = kStaticBlock;
    double *d;
    PT *r;
    static_slot<C, PT>(const_cast<void *>(buf), i, d, r);
    for (int k = 0; k < C; ++k) g.beta_q[k] = ld_statics<double, kGlobal>(d + (L::kBetaQ + k) * S);
    int o = L::kM;
    for (int a = 0; a < C; ++a)
        for (int b = a; b < C; ++b) g.M[a][b] = g.M[b][a] = ld_statics<double, kGlobal>(d + (o++) * S);
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < C; ++k) g.Sxq[a][k] = ld_statics<double, kGlobal>(d + (L::kSxq + a * C + k) * S);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) g.cov3[a][b] = ld_statics<double, kGlobal>(d + (L::kCov3 + 3 * a + b) * S);
    g.opacity = ld_statics<double, kGlobal>(d + L::kOpacity * S);
    g.beta_x = ld_statics<double, kGlobal>(d + L::kBetaX * S);
    g.floor_eps = ld_statics<double, kGlobal>(d + L::kFloorEps * S);
    const int fl = (int)ld_statics<double, kGlobal>(d + L::kFlags * S);
    g.valid = (fl & 1) != 0;
    g.floored3 = (fl & 2) != 0;
    g.log2_op = ld_statics<double, kGlobal>(d + L::kLog2Op * S);
    for (int k = 0; k < 3; ++k) mu_x[k] = (double)ld_statics<PT, kGlobal>(r + k * S);
    for (int k = 0; k < C; ++k) mu_q[k] = (double)ld_statics<PT, kGlobal>(r + (3 + k) * S);
    for (int k = 0; k < 3; ++k) g.color[k] = (double)ld_statics<PT, kGlobal>(r + (3 + C + k) * S);
}

// prim_geom for primitive i of a scene whose statics are current: the
// query-invariant half is read back (load_statics: the bits prim_static
// computed) instead of recomputed -- no Cholesky, inverse or eigen floor --
// and only what the adjoint needs beyond the statics is rebuilt from the
// parameters with prim_static's own helpers: sx, R, Lx, sq, lqx and, for a
// floored conditional covariance, the pre-floor sym3.  Same bits as
// prim_geom (gradients.py:179-280 reads all of them).
template <int C, typename PT>
__device__ inline void prim_geom_cached(const PT *rec, int64_t i, const UbsView &v, PrimGeom<C> &g,
                                        double (&mu_x)[3]) {
    constexpr int CC = PrimGeom<C>::CC;
    double mu_q[CC];
    load_statics<C, PT, true>(v.statics, i, g, mu_x, mu_q);
    double mx[3], mq[CC], rot[3], sxr[3], lq[CC * 3], sqr[CC], bxr, bqr[CC], oraw, col[3];
    load_params<C>(rec, mx, mq, rot, sxr, lq, sqr, bxr, bqr, oraw, col);
    for (int k = 0; k < 3; ++k) g.sx[k] = exp(sxr[k]);
    static_rotation<C>(rot, g);
    if constexpr (C > 0) {
        for (int k = 0; k < C; ++k) {
            g.sq[k] = exp(sqr[k]);
            for (int j = 0; j < 3; ++j) g.lqx[k][j] = lq[3 * k + j];
        }
    }
    if (g.floored3) {
        double Sx[3][3];
        static_sx<C>(g, Sx);
        static_sym3<C>(g, Sx);
    } else {
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) g.sym3[a][b] = g.cov3[a][b];  // prim_static's cov3 = sym3 when unfloored
    }
    prim_view<C>(g, mu_x, mu_q, v);
}

// Device-side capacity guard for the pair buffers: true (and the overflow
// status bit set) when this frame's K exceeds the caller's capacity.
__device__ __forceinline__ bool pairs_overflow(const unsigned long long *n_pairs, int64_t capacity,
                                               uint32_t *status) {
    if (n_pairs && (int64_t)*n_pairs > capacity) {
        if (status && threadIdx.x == 0) atomicOr(status, (uint32_t)UBS_S_PAIR_OVERFLOW);
        return true;
    }
    return false;
}

}  // namespace ubs

#define UBS_CUDA_CHECK()                                   \
    do {                                                   \
        if (cudaPeekAtLastError() != cudaSuccess) {        \
            (void)cudaGetLastError();                      \
            return UBS_E_CUDA;                             \
        }                                                  \
    } while (0)
