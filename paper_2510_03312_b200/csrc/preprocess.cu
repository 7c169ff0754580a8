// K1 preprocess: conditioning + projection + tile rect, one thread per primitive.
//
// Reference: slicing.py:185-235 (slice_scene), raster.py:95-134 (project_scene),
// raster.py:252-266 (build_tiles' inclusive AABB test, restated as an exact
// rect formula: SURVEY.md Appendix A).
//
// HBM: reads 4P B of parameters, writes 8 (depth key) + 8 (rect) + 4 (count)
// + 2 (flags) + 64/80 B (raster record) per primitive.  Arithmetic is fp64.
// Parameters are staged into shared memory with coalesced loads (the UBS1
// record is AoS with a 56..152 B stride; one thread per record would issue
// 32 scattered 4 B loads per warp instruction).
#include <cuda_runtime.h>

#include <cmath>

#include "ubs_common.cuh"

namespace ubs {

constexpr int kPreThreads = 128;

// Scene statics: the query-invariant half of slice_scene for every primitive
// (prim_static), written field-major (StaticLayout) for coalesced reads.
template <int C, typename PT>
__global__ void __launch_bounds__(kPreThreads)
statics_kernel(const UbsView v, void *out) {
    constexpr int P = 14 + 6 * C;
    __shared__ PT stage[kPreThreads * P];
    const int64_t base = (int64_t)blockIdx.x * kPreThreads;
    const int64_t n = v.n;
    const int nloc = (int)min((int64_t)kPreThreads, n - base);
    const PT *src = reinterpret_cast<const PT *>(v.params) + base * P;
    for (int k = threadIdx.x; k < nloc * P; k += kPreThreads) stage[k] = src[k];
    __syncthreads();
    const int t = threadIdx.x;
    if (t >= nloc) return;
    PrimGeom<C> g;
    double mu_x[3], mu_q[PrimGeom<C>::CC];
    prim_static<C, PT>(stage + t * P, v.set, g, mu_x, mu_q);
    store_statics<C, PT>(out, base + t, g, mu_x, mu_q);
}

// Block-wide visible count, pair total and depth range of one view, added to
// the view's counters with one atomic each per CTA: warp totals by
// single-instruction reductions (REDUX) into per-warp shared slots, summed by
// thread 0 (no shared-memory atomics).  The depth range is kept at the
// granularity of the keys' high 32 bits (lo rounded down, hi up): it still
// bounds every visible key, which is all the depth bucketing needs.
struct PreAgg {
    uint32_t vis[kPreThreads / 32], pairs[kPreThreads / 32], kmin[kPreThreads / 32], kmax[kPreThreads / 32];
};

__device__ __forceinline__ void preprocess_aggregate(PreAgg &agg, const UbsPrimBuffers &pb, bool vis,
                                                     uint32_t my_count, unsigned long long my_key) {
    const uint32_t full = 0xffffffffu;
    const int w = threadIdx.x >> 5;
    const unsigned ballot = __ballot_sync(full, vis);
    const uint32_t wsum = __reduce_add_sync(full, my_count);  // < 2^32 per warp
    const uint32_t khi = (uint32_t)(my_key >> 32);
    const uint32_t kmin = __reduce_min_sync(full, vis ? khi : 0xffffffffu);
    const uint32_t kmax = __reduce_max_sync(full, vis ? khi : 0u);
    if ((threadIdx.x & 31) == 0) {
        agg.vis[w] = (uint32_t)__popc(ballot);
        agg.pairs[w] = wsum;
        agg.kmin[w] = kmin;
        agg.kmax[w] = kmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t nv = 0, lo = 0xffffffffu, hi = 0u;
        unsigned long long np = 0;
#pragma unroll
        for (int k = 0; k < kPreThreads / 32; ++k) {
            nv += agg.vis[k];
            np += agg.pairs[k];
            lo = min(lo, agg.kmin[k]);
            hi = max(hi, agg.kmax[k]);
        }
        if (nv) {
            atomicAdd(pb.n_visible, nv);
            atomicMin(pb.depth_range, (unsigned long long)lo << 32);
            atomicMax(pb.depth_range + 1, ((unsigned long long)hi << 32) | 0xffffffffull);
        }
        if (np) atomicAdd(pb.n_pairs, np);
    }
}

// The per-view outputs of primitive i once g holds its view-dependent
// geometry (prim_view / prim_geom): depth key, tile rect and count (plus the
// rect's corners in the 2D difference array), flags, raster records.
template <int C>
__device__ __forceinline__ void preprocess_emit(const UbsView &v, const UbsPrimBuffers &pb, int want_rec32,
                                                int64_t i, const PrimGeom<C> &g, double sqrt_tau, bool &vis,
                                                uint32_t &my_count, unsigned long long &my_key) {
    const int W = v.cam.width, H = v.cam.height;
    const int TX = (W + kTile - 1) / kTile, TY = (H + kTile - 1) / kTile;
    uint32_t count = 0;
    uint64_t rect = 0;
    vis = g.visible;
    if (vis) {
        // inclusive tile test of raster.py:261-264 as a closed form:
        // tile tx is hit iff hi >= 16 tx and lo <= min(16 (tx+1), W)
        const double lox = g.mean2[0] - g.radii[0], hix = g.mean2[0] + g.radii[0];
        const double loy = g.mean2[1] - g.radii[1], hiy = g.mean2[1] + g.radii[1];
        if (hix >= 0.0 && lox <= (double)W && hiy >= 0.0 && loy <= (double)H) {
            // x / 16 == x * 0.0625 exactly (a power-of-two scale)
            constexpr double kInvTile = 1.0 / kTile;
            double tx0 = fmax(0.0, ceil(lox * kInvTile) - 1.0), tx1 = fmin((double)(TX - 1), floor(hix * kInvTile));
            double ty0 = fmax(0.0, ceil(loy * kInvTile) - 1.0), ty1 = fmin((double)(TY - 1), floor(hiy * kInvTile));
            if (tx1 >= tx0 && ty1 >= ty0) {
                uint64_t a = (uint64_t)tx0, b = (uint64_t)ty0, c = (uint64_t)tx1, d = (uint64_t)ty1;
                rect = a | (b << 16) | (c << 32) | (d << 48);
                count = (uint32_t)((c - a + 1) * (d - b + 1));
                // 2D difference array: a prefix sum over it gives every tile's pair count
                const int gw = TX + 1;
                if (!UBS_GUARD(c + 1 <= (uint64_t)TX && d + 1 <= (uint64_t)TY, kChkGrid)) return;
                atomicAdd(pb.tile_grid + (int)b * gw + (int)a, 1);
                atomicAdd(pb.tile_grid + (int)b * gw + (int)c + 1, -1);
                atomicAdd(pb.tile_grid + ((int)d + 1) * gw + (int)a, -1);
                atomicAdd(pb.tile_grid + ((int)d + 1) * gw + (int)c + 1, 1);
            }
        }
    }
    my_key = vis ? (unsigned long long)__double_as_longlong(g.tcam[2]) : kInvisibleKey;
    pb.depth_key[i] = my_key;
    pb.rect[i] = rect;
    pb.tile_count[i] = count;
    my_count = count;
    uint16_t fl = (vis ? UBS_F_VISIBLE : 0) | (g.valid ? 0 : UBS_F_DEGENERATE) |
                  (g.floored3 ? UBS_F_FLOOR3 : 0) | (g.floored2 ? UBS_F_FLOOR2 : 0);
    if constexpr (C > 0) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            fl |= (g.s_tanh[k] > 0.0 ? 1 : 0) << (8 + k);
            if (g.d_gate[k] == 1.0) fl |= UBS_F_GATE_SAT;
        }
    }

    // raster records: only visible primitives' are ever read (the depth order,
    // the tile lists and the backward hold visible ids only), so invisible
    // ones are not written
    if (vis && pb.rec64) {
        Rec64 r;
        r.mx = g.mean2[0]; r.my = g.mean2[1];
        r.p00 = g.p2[0]; r.p01 = g.p2[1]; r.p11 = g.p2[2];
        r.og = g.og; r.bx = g.beta_x;
        r.cr = g.color[0]; r.cg = g.color[1]; r.cb = g.color[2];
        reinterpret_cast<Rec64 *>(pb.rec64)[i] = r;
    }
    if (vis && want_rec32 && pb.rec32) {
        // P = U^T U with U upper triangular (Cholesky of P, transposed)
        const double u00 = sqrt(g.p2[0]);
        const double u01 = g.p2[1] / u00;
        const double u11 = sqrt(fmax(g.p2[2] - u01 * u01, 0.0));
        const double fxm = floor(g.mean2[0]), fym = floor(g.mean2[1]);
        const bool in_range = fabs(g.mean2[0]) < 4.0e6 && fabs(g.mean2[1]) < 4.0e6 && isfinite(u11);
        // E bounds |m32 - m64| over the support (m < tau => |dx| < rx, |dy| < ry,
        // |y0|, |y1| < sqrt(tau)), with u = 2^-24 the fp32 unit roundoff:
        //   dx = ((tx 16 - fx) + ox) + lx   |d dx| <= u (2|dx| + 15.5)
        //        (ox rounded; the tile offset, |.| <= |dx| + 15, and the add of
        //        the pixel's column lx in 0..15 rounded once each: raster.cu tile_offset)
        //   y0 = fma(u01, dy, u00 dx)  |d y0| <= u (|u00|(4|dx| + 16) + |u01|(4|dy| + 16) + |y0|)
        //                              (either product may be the separately rounded one)
        //   y1 = u11 dy                |d y1| <= u (|u11|(3|dy| + 16) + |y1|)
        //   m  = fma(y0, y0, y1 y1)    |d m|  <= 2|y0||d y0| + 2|y1||d y1| + 2 u tau
        // (u.. rounded to fp32 included), times a 1.25 safety factor.
        const double u = 5.9604644775390625e-08;
        const double st = sqrt_tau;
        const double rx = g.radii[0], ry = g.radii[1];
        double E = 1.25 * u * (2.0 * st * (fabs(u00) * (4.0 * rx + 16.0) + fabs(u01) * (4.0 * ry + 16.0) + st) +
                               2.0 * st * (fabs(u11) * (3.0 * ry + 16.0) + st) + 2.0 * v.set.tau_sq);
        double eb = in_range ? g.beta_x * E : INFINITY;
        if (!isfinite(eb)) fl |= UBS_F_THIN;
        Rec32 r;
        r.r0 = make_float4(in_range ? (float)fxm : 0.f, in_range ? (float)fym : 0.f,
                           (float)(0.5 - (g.mean2[0] - fxm)), (float)(0.5 - (g.mean2[1] - fym)));
        r.r1 = make_float4((float)u00, (float)u01, (float)u11, (float)(v.set.tau_sq + E));
        r.r2 = make_float4((float)g.beta_x, (float)g.color[0], (float)g.color[1], (float)g.color[2]);
        // qc: lg2.approx absolute error 2^-22.6 (near 1) times ln2 beta, ex2.approx
        // relative error 2^-22, og / log2(og) representation; the |arg|-relative
        // parts are added per visit in the raster (2.1e-7 |arg|)
        const double qc = 0.6931471805599453 * g.beta_x * 1.6e-7 + 4.0e-7;
        // log2(og) = log2(opacity) + lsum log2(e): the gate's log is already
        // formed and log2(opacity) is query-invariant (a scene static); the
        // fp64 result differs from log2(og) by ~1e-16 relative, far below
        // the fp32 rounding the per-visit 2.1e-7 |arg| term covers
        const double log2_og = g.log2_op + g.lsum * 1.4426950408889634;
        r.r3 = make_float4((float)eb, (float)g.og, (float)qc, (float)log2_og);
        reinterpret_cast<Rec32 *>(pb.rec32)[i] = r;
    }
    pb.flags[i] = fl;

}

// kStatic: the query-invariant half comes from v.statics (ubs_scene_statics)
// and only prim_view runs here; otherwise the whole of prim_geom.
template <int C, typename PT, bool kStatic>
__global__ void __launch_bounds__(kPreThreads, kStatic ? 5 : 4)
preprocess_kernel(const UbsView v, const UbsPrimBuffers pb, int want_rec32) {
    constexpr int P = 14 + 6 * C;
    __shared__ PT stage[kStatic ? 1 : kPreThreads * P];
    __shared__ PreAgg agg;
    const int64_t base = (int64_t)blockIdx.x * kPreThreads;
    const int64_t n = v.n;
    const int nloc = (int)min((int64_t)kPreThreads, n - base);
    if constexpr (!kStatic) {
        const PT *src = reinterpret_cast<const PT *>(v.params) + base * P;
        for (int k = threadIdx.x; k < nloc * P; k += kPreThreads) stage[k] = src[k];
    }
    __syncthreads();
    const int t = threadIdx.x;
    bool vis = false;
    uint32_t my_count = 0;
    unsigned long long my_key = ~0ull;
    if (t < nloc) {
        const int64_t i = base + t;
        PrimGeom<C> g;
        double mu_x[3];
        if constexpr (kStatic) {
            double mu_q[PrimGeom<C>::CC];
            load_statics<C, PT>(v.statics, i, g, mu_x, mu_q);
            prim_view<C>(g, mu_x, mu_q, v, false);
        } else {
            prim_geom<C, PT>(stage + t * P, v, g, mu_x);
        }
        preprocess_emit<C>(v, pb, want_rec32, i, g, sqrt(v.set.tau_sq), vis, my_count, my_key);
    }
    preprocess_aggregate(agg, pb, vis, my_count, my_key);
}

// Several views of one scene from one read of its statics: the CTA's
// 128-primitive statics block (StaticLayout, 16..62 KB contiguous) is pulled
// into shared memory with one TMA bulk copy, then every view runs prim_view
// from it.  Per view this saves the statics read (352 B per primitive at 7D
// of the ~520 B a view moves), which is most of preprocess's HBM traffic;
// the arithmetic and outputs are those of preprocess_kernel<C, PT, true>.
constexpr int kMaxViews = UBS_MAX_VIEWS;

struct PreViews {
    UbsView v[kMaxViews];
    UbsPrimBuffers pb[kMaxViews];
    double sqrt_tau;  // sqrt(tau_sq) of the group (same settings), host-computed: IEEE sqrt, same bits
    int nv;
    int want_rec32;
};

template <int C, typename PT>
__global__ void __launch_bounds__(kPreThreads, 4)
preprocess_views_kernel(const __grid_constant__ PreViews m) {
    using L = StaticLayout<C>;
    constexpr uint32_t kBlockBytes = (uint32_t)kStaticBlock * (8 * L::D + sizeof(PT) * L::R);
    static_assert(kStaticBlock == kPreThreads && kBlockBytes % 16 == 0, "statics block = CTA, 16 B multiple");
    extern __shared__ __align__(128) unsigned char st_block[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ PreAgg agg;
    const int64_t base = (int64_t)blockIdx.x * kPreThreads;
    const int nloc = (int)min((int64_t)kPreThreads, m.v[0].n - base);
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const char *src = reinterpret_cast<const char *>(m.v[0].statics) + (size_t)blockIdx.x * kBlockBytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kBlockBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(st_block)),
            "l"(src), "r"(kBlockBytes), "r"(bar)
            : "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(bar)
        : "memory");
    const int t = threadIdx.x;
    for (int k = 0; k < m.nv; ++k) {
        const UbsView &v = m.v[k];
        const UbsPrimBuffers &pb = m.pb[k];
        bool vis = false;
        uint32_t my_count = 0;
        unsigned long long my_key = ~0ull;
        if (t < nloc) {
            PrimGeom<C> g;
            double mu_x[3], mu_q[PrimGeom<C>::CC];
            load_statics<C, PT, false>(st_block, t, g, mu_x, mu_q);  // slot t of the staged block
            prim_view<C>(g, mu_x, mu_q, v, false);
            preprocess_emit<C>(v, pb, m.want_rec32, base + t, g, m.sqrt_tau, vis, my_count, my_key);
        }
        preprocess_aggregate(agg, pb, vis, my_count, my_key);
        __syncthreads();  // thread 0 has read agg before the next view's warps overwrite it
    }
}

// FrameCache.slices / .proj (slicing.py:153-182, raster.py:46-60): a
// separate kernel that recomputes each primitive's geometry on the frame's
// own route (statics or inline) and writes the include/ubs_b200.h
// UBS_DEBUG_* row.  Fields of the query-invariant half (l_x, rotation, s_x,
// s_q, the cov3 eigen pair) are only known on the inline route; d_raw and
// both eigen pairs are recomputed with prim_view's / eigh's own arithmetic.
// Kept out of the preprocess kernels so the debug path's eigen solvers cost
// their hot path no registers.
template <int C, typename PT, bool kStatic>
__global__ void __launch_bounds__(kPreThreads)
preprocess_debug_kernel(const UbsView v, double *__restrict__ debug) {
    constexpr int P = 14 + 6 * C;
    const int64_t i = (int64_t)blockIdx.x * kPreThreads + threadIdx.x;
    if (i >= v.n) return;
    PrimGeom<C> g;
    double mu_x[3];
    if constexpr (kStatic) {
        double mu_q[PrimGeom<C>::CC];
        load_statics<C, PT>(v.statics, i, g, mu_x, mu_q);
        prim_view<C>(g, mu_x, mu_q, v, true);
    } else {
        prim_geom<C, PT>(reinterpret_cast<const PT *>(v.params) + i * P, v, g, mu_x);
    }
    const bool vis = g.visible;
    double *d = debug + i * UBS_DEBUG_STRIDE;
    for (int k = 0; k < UBS_DEBUG_STRIDE; ++k) d[k] = 0.0;
    d[0] = g.tcam[2];
    d[1] = g.mean2[0]; d[2] = g.mean2[1];
    d[3] = g.p2[0]; d[4] = g.p2[1]; d[5] = g.p2[2];
    d[6] = g.radii[0]; d[7] = g.radii[1];
    d[8] = g.og; d[9] = g.beta_x;
    d[10] = g.cov2[0]; d[11] = g.cov2[1]; d[12] = g.cov2[2];
    d[13] = g.cov3[0][0]; d[14] = g.cov3[0][1]; d[15] = g.cov3[0][2];
    d[16] = g.cov3[1][1]; d[17] = g.cov3[1][2]; d[18] = g.cov3[2][2];
    d[19] = g.tcam[0]; d[20] = g.tcam[1]; d[21] = g.tcam[2];
    d[22] = g.mean3[0]; d[23] = g.mean3[1]; d[24] = g.mean3[2];
    d[25] = g.gate; d[26] = g.opacity;
    d[31] = g.floor_eps;
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) d[UBS_DEBUG_VMAT + 3 * r + c] = g.V[r][c];
    {
        double w[2], E[2][2];
        eigh2(g.raw2[0], g.raw2[1], g.raw2[2], w, E);
        d[UBS_DEBUG_COV2_EIG] = w[0]; d[UBS_DEBUG_COV2_EIG + 1] = w[1];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) d[UBS_DEBUG_COV2_EIG + 2 + 2 * r + c] = E[r][c];
    }
    if (!v.statics) {
        double w[3], E[3][3];
        eigh3(g.sym3, w, E);
        for (int k = 0; k < 3; ++k) d[UBS_DEBUG_COV3_EIG + k] = w[k];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                d[UBS_DEBUG_COV3_EIG + 3 + 3 * r + c] = E[r][c];
                d[UBS_DEBUG_LX + 3 * r + c] = g.Lx[r][c];
                d[UBS_DEBUG_ROT + 3 * r + c] = g.R[r][c];
            }
        for (int k = 0; k < 3; ++k) d[UBS_DEBUG_SX + k] = g.sx[k];
    }
    for (int k = 0; k < 3; ++k) d[UBS_DEBUG_COLOR + k] = g.color[k];
    if constexpr (C > 0) {
        for (int k = 0; k < C; ++k) {
            d[27 + k] = g.s_tanh[k];
            d[UBS_DEBUG_BETA_Q + k] = g.beta_q[k];
            d[UBS_DEBUG_DELTA + k] = g.delta[k];
            d[UBS_DEBUG_U + k] = g.u[k];
            d[UBS_DEBUG_V + k] = g.v[k];
            d[UBS_DEBUG_D_GATE + k] = g.d_gate[k];
            double dr = 0.0;  // prim_view's d_raw, same accumulation order
            for (int j = 0; j < C; ++j) dr += g.M[k][j] * g.delta[j];
            d[UBS_DEBUG_D_RAW + k] = dr;
            for (int j = 0; j < C; ++j) d[UBS_DEBUG_M_INV + 4 * k + j] = g.M[k][j];
            for (int r = 0; r < 3; ++r) d[UBS_DEBUG_SIGMA_XQ + 4 * r + k] = g.Sxq[r][k];
            if (!v.statics) d[UBS_DEBUG_SQ + k] = g.sq[k];
        }
    }
    d[UBS_DEBUG_FLAGS] = (g.valid ? 1.0 : 0.0) + (g.floored3 ? 2.0 : 0.0) + (g.floored2 ? 4.0 : 0.0) +
                         (vis ? 8.0 : 0.0) + (v.statics ? 0.0 : 16.0);
}

template <int C, typename PT>
static void launch_debug(const UbsView &v, double *debug, cudaStream_t s) {
    const int64_t blocks = (v.n + kPreThreads - 1) / kPreThreads;
    if (v.statics)
        preprocess_debug_kernel<C, PT, true><<<(unsigned)blocks, kPreThreads, 0, s>>>(v, debug);
    else
        preprocess_debug_kernel<C, PT, false><<<(unsigned)blocks, kPreThreads, 0, s>>>(v, debug);
}

static int launch_debug_any(const UbsView &v, double *debug, cudaStream_t s) {
    const bool f64 = v.param_f64 != 0;
    switch (v.n_dims) {
        case 3: f64 ? launch_debug<0, double>(v, debug, s) : launch_debug<0, float>(v, debug, s); break;
        case 6: f64 ? launch_debug<3, double>(v, debug, s) : launch_debug<3, float>(v, debug, s); break;
        case 7: f64 ? launch_debug<4, double>(v, debug, s) : launch_debug<4, float>(v, debug, s); break;
        default: return UBS_E_ARGS;
    }
    return UBS_OK;
}

template <int C, typename PT>
static int launch_views(const PreViews &m, cudaStream_t s) {
    using L = StaticLayout<C>;
    constexpr size_t kBlockBytes = (size_t)kStaticBlock * (8 * L::D + sizeof(PT) * L::R);
    // (a host-side attribute write, once per group launch; no cached state)
    if (cudaFuncSetAttribute(preprocess_views_kernel<C, PT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kBlockBytes) != cudaSuccess)
        return UBS_E_CUDA;
    const int64_t blocks = (m.v[0].n + kPreThreads - 1) / kPreThreads;
    preprocess_views_kernel<C, PT><<<(unsigned)blocks, kPreThreads, kBlockBytes, s>>>(m);
    return UBS_OK;
}

template <int C, typename PT>
static void launch_pre(const UbsView &v, const UbsPrimBuffers &pb, int want32, cudaStream_t s) {
    const int64_t blocks = (v.n + kPreThreads - 1) / kPreThreads;
    if (v.statics)
        preprocess_kernel<C, PT, true><<<(unsigned)blocks, kPreThreads, 0, s>>>(v, pb, want32);
    else
        preprocess_kernel<C, PT, false><<<(unsigned)blocks, kPreThreads, 0, s>>>(v, pb, want32);
}

template <int C, typename PT>
static void launch_statics(const UbsView &v, void *out, cudaStream_t s) {
    const int64_t blocks = (v.n + kPreThreads - 1) / kPreThreads;
    statics_kernel<C, PT><<<(unsigned)blocks, kPreThreads, 0, s>>>(v, out);
}

}  // namespace ubs

using namespace ubs;

extern "C" int ubs_abi_version(void) { return UBS_ABI_VERSION; }

extern "C" const char *ubs_build_info(void) {
    return "ubs_b200 sm_100a; fp64 preprocess (scene statics); depth bucket sort; two-level 8x4-tile binning; "
           "tile-per-CTA raster fp32 (certified, fp64 fix-up) / fp64";
}

static int preprocess_check(const UbsView *v, const UbsPrimBuffers *pb, int32_t want_rec32) {
    if (!v || !pb || !pb->n_visible || !pb->n_pairs) return UBS_E_ARGS;
    if (v->set.tile_size != kTile) return UBS_E_ARGS;
    if (v->n < 0 || (v->n > 0 && !v->params)) return UBS_E_ARGS;
    if (!pb->depth_key || !pb->rect || !pb->tile_count || !pb->flags) return UBS_E_ARGS;
    if (!pb->rec64 && !(want_rec32 && pb->rec32)) return UBS_E_ARGS;
    if (!pb->tile_grid || !pb->depth_range) return UBS_E_ARGS;
    return UBS_OK;
}

static int preprocess_reset(const UbsView *v, const UbsPrimBuffers *pb, cudaStream_t s) {
    if (cudaMemsetAsync(pb->depth_range, 0xFF, 8, s) != cudaSuccess ||
        cudaMemsetAsync(pb->depth_range + 1, 0, 8, s) != cudaSuccess)
        return UBS_E_CUDA;
    const int TX = (v->cam.width + kTile - 1) / kTile, TY = (v->cam.height + kTile - 1) / kTile;
    if (cudaMemsetAsync(pb->tile_grid, 0, sizeof(int32_t) * (size_t)(TX + 1) * (TY + 1), s) != cudaSuccess)
        return UBS_E_CUDA;
    return UBS_OK;
}

extern "C" int ubs_preprocess(const UbsView *v, const UbsPrimBuffers *pb, int32_t want_rec32,
                              ubs_stream_t stream) {
    const int rc = preprocess_check(v, pb, want_rec32);
    if (rc != UBS_OK) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (preprocess_reset(v, pb, s) != UBS_OK) return UBS_E_CUDA;
    if (v->n == 0) return UBS_OK;
    const bool f64 = v->param_f64 != 0;
    switch (v->n_dims) {
        case 3: f64 ? launch_pre<0, double>(*v, *pb, want_rec32, s)
                    : launch_pre<0, float>(*v, *pb, want_rec32, s); break;
        case 6: f64 ? launch_pre<3, double>(*v, *pb, want_rec32, s)
                    : launch_pre<3, float>(*v, *pb, want_rec32, s); break;
        case 7: f64 ? launch_pre<4, double>(*v, *pb, want_rec32, s)
                    : launch_pre<4, float>(*v, *pb, want_rec32, s); break;
        default: return UBS_E_ARGS;
    }
    if (pb->debug && launch_debug_any(*v, pb->debug, s) != UBS_OK) return UBS_E_ARGS;
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" int ubs_preprocess_views(const UbsView *views, const UbsPrimBuffers *pbs, int32_t n_views,
                                    int32_t want_rec32, ubs_stream_t stream) {
    if (!views || !pbs || n_views < 1) return UBS_E_ARGS;
    const UbsView &v0 = views[0];
    for (int k = 0; k < n_views; ++k) {
        const int rc = preprocess_check(views + k, pbs + k, want_rec32);
        if (rc != UBS_OK) return rc;
        const UbsView &v = views[k];
        // one scene: the views differ in camera and query only
        if (!v.statics || v.statics != v0.statics || v.params != v0.params || v.n != v0.n ||
            v.n_dims != v0.n_dims || v.param_f64 != v0.param_f64 || v.set.tau_sq != v0.set.tau_sq)
            return UBS_E_ARGS;
    }
    cudaStream_t s = (cudaStream_t)stream;
    for (int k = 0; k < n_views; ++k) {
        const int rc = preprocess_reset(views + k, pbs + k, s);
        if (rc != UBS_OK) return rc;
    }
    if (v0.n == 0) return UBS_OK;
    for (int k0 = 0; k0 < n_views; k0 += kMaxViews) {
        PreViews m;
        m.nv = min(kMaxViews, n_views - k0);
        m.want_rec32 = want_rec32;
        m.sqrt_tau = sqrt(v0.set.tau_sq);
        for (int k = 0; k < m.nv; ++k) {
            m.v[k] = views[k0 + k];
            m.pb[k] = pbs[k0 + k];
        }
        const bool f64 = v0.param_f64 != 0;
        int rc;
        switch (v0.n_dims) {
            case 3: rc = f64 ? launch_views<0, double>(m, s) : launch_views<0, float>(m, s); break;
            case 6: rc = f64 ? launch_views<3, double>(m, s) : launch_views<3, float>(m, s); break;
            case 7: rc = f64 ? launch_views<4, double>(m, s) : launch_views<4, float>(m, s); break;
            default: return UBS_E_ARGS;
        }
        if (rc != UBS_OK) return rc;
    }
    for (int k = 0; k < n_views; ++k)
        if (pbs[k].debug && launch_debug_any(views[k], pbs[k].debug, s) != UBS_OK) return UBS_E_ARGS;
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" size_t ubs_statics_bytes(int64_t n, int32_t n_dims, int32_t param_f64) {
    if (n < 0 || (n_dims != 3 && n_dims != 6 && n_dims != 7)) return 0;
    return statics_bytes(n, n_dims, param_f64);
}

extern "C" int ubs_scene_statics(const UbsView *v, void *statics, ubs_stream_t stream) {
    if (!v || v->n < 0 || (v->n > 0 && (!v->params || !statics))) return UBS_E_ARGS;
    if (v->n == 0) return UBS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const bool f64 = v->param_f64 != 0;
    switch (v->n_dims) {
        case 3: f64 ? launch_statics<0, double>(*v, statics, s) : launch_statics<0, float>(*v, statics, s); break;
        case 6: f64 ? launch_statics<3, double>(*v, statics, s) : launch_statics<3, float>(*v, statics, s); break;
        case 7: f64 ? launch_statics<4, double>(*v, statics, s) : launch_statics<4, float>(*v, statics, s); break;
        default: return UBS_E_ARGS;
    }
    UBS_CUDA_CHECK();
    return UBS_OK;
}

UBS_CHECKED_ACCESSOR(preprocess)
