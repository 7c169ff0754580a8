// Tile rasterizer: forward composite, fp64 fix-up, backward replay.
//
// Reference: _tiles.py:19-56 (tile_forward), _tiles.py:59-127 (tile_backward),
// raster.py:284-316 (per-tile driver and assembly), gradients.py:142-173
// (per-tile partials scattered with np.add.at).
//
// Layout: one 16x16 tile per CTA, one pixel per thread (256 threads).  The
// tile's depth-ordered id list is walked in batches of 256: each thread
// gathers one splat record into shared memory (vector loads), then every
// thread walks the batch from shared memory.  A CTA stops staging once
// __syncthreads_count says all 256 pixels crossed the transmittance cut.
//
// Two forward precisions:
//  * fp64: the reference's arithmetic, same operation order, no FMA
//    contraction (mul/add helpers) -> images to ~1e-15, counts exact.
//  * fp32: each pixel also accumulates a first-order bound on the relative
//    error of its transmittance (from the per-splat bound E on |m32 - m64|
//    and the float rounding of alpha).  Pixels whose cut decision
//    (T < t_min), alpha-clamp decision or image error are not certain under
//    that bound are appended to a fix-up list and recomputed in fp64 by
//    raster_fixup_kernel (one warp per pixel, sequential blend => the
//    reference's rounding), so contributor counts and alpha_clamped flags
//    stay bit-exact while 99+% of pixels take the fp32 path.
#include <cuda_runtime.h>

#include <type_traits>

#include <cub/device/device_scan.cuh>

#include "ubs_common.cuh"
#include "f32x2.cuh"

namespace ubs {

#ifdef UBS_FWD_STATS
// profiling build only (scratch tooling, not the product library): walk statistics
// 0 warp-visits | 1 warp-visits with no lane in support | 2 lane-visits in support |
// 3 active lanes over warp-visits | 4 warp-visits with a lane above clamp_lo |
// 5 warp-visits with a lane below tmin_hi | 6 CTA batches | 7 warps whose walk ended by the cut
__device__ unsigned long long g_fwd_stats[8];
extern "C" int ubs_debug_fwd_stats(unsigned long long *out, int reset) {
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out, g_fwd_stats, sizeof(g_fwd_stats)) != cudaSuccess) return -2;
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_fwd_stats, z, sizeof(z));
    }
    return 0;
}
#define FWD_STAT(k, v) do { if ((threadIdx.x & 31) == (__ffs(__activemask()) - 1)) atomicAdd(&g_fwd_stats[k], (unsigned long long)(v)); } while (0)
#else
#define FWD_STAT(k, v) do { } while (0)
#endif

struct RasterParams {
    int W, H, TX;
    double tau, clamp, tmin;
    double bg[3];
    // the fp32 kernels' constants, rounded once on the host exactly as the
    // kernels' own casts would (kernel-parameter operands: a register-starved
    // kernel re-reads them for free instead of re-converting a double)
    float tau_f, inv_tau_f, clamp_f, omc_f, tmin_f;
    const unsigned long long *n_pairs;  // device K, checked against pair_capacity
    int64_t pair_capacity;
    uint32_t list_cap;                  // per-tile list cap (binning materialised only this prefix)
    uint32_t *status;                   // UBS_S_LIST_TRUNC when a capped list ran out too early
};

// [start, end) of the materialised part of a tile's list; `capped` when the
// real list is longer (running out of it with unsaturated pixels is an error)
__device__ __forceinline__ void tile_span(const RasterParams &P, const uint32_t *ranges, int tile, uint32_t &start,
                                          uint32_t &end, bool &capped) {
    start = ranges[2 * tile];
    const uint32_t len = ranges[2 * tile + 1] - start;
    capped = len > P.list_cap;
    end = start + (capped ? P.list_cap : len);
}

static RasterParams make_params(const UbsView &v, const UbsPrimBuffers &pb, const UbsBinBuffers &bb) {
    RasterParams p;
    p.n_pairs = pb.n_pairs;
    p.pair_capacity = bb.pair_capacity;
    p.list_cap = bb.list_cap ? bb.list_cap : 0xFFFFFFFFu;
    p.status = bb.status;
    p.W = v.cam.width;
    p.H = v.cam.height;
    p.TX = (p.W + kTile - 1) / kTile;
    p.tau = v.set.tau_sq;
    p.clamp = v.set.alpha_clamp;
    p.tmin = v.set.transmittance_min;
    p.tau_f = (float)p.tau;
    p.inv_tau_f = (float)(1.0 / p.tau);
    p.clamp_f = (float)p.clamp;
    p.omc_f = (float)(1.0 - p.clamp);
    p.tmin_f = (float)p.tmin;
    for (int k = 0; k < 3; ++k) p.bg[k] = v.background[k];
    return p;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long x, unsigned long long *red) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kTileThreads / 32; ++w) t += red[w];
    return t;
}

// ---------------------------------------------------------------------------
// forward, fp32 with certified fall-back to fp64
// ---------------------------------------------------------------------------
// Linear worst-case bound on the relative transmittance error above which a
// pixel is re-done in fp64 regardless of its decisions.  The bound adds every
// per-visit error with the same sign, so it overestimates the real fp32 error
// (~1e-5, measured against the oracle in tests/) by 10-100x; this threshold
// only catches pathological splats (needle conics, huge beta at the support
// edge), the image tolerance itself is asserted by the parity tests.
constexpr float kImgErrTol = 1.0e-3f;

// 16 B shared-memory load at a 32-bit shared address (keeps the splat walk
// in 32-bit shared offsets instead of generic 64-bit pointers); the record
// offset is an immediate, so every field of a record shares one address
// register
template <int OFF = 0>
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "r"(a), "n"(OFF));
    return v;
}

template <int OFF = 0>
__device__ __forceinline__ float2 lds64(uint32_t a) {
    float2 v;
    asm("ld.shared.v2.f32 {%0, %1}, [%2+%3];" : "=f"(v.x), "=f"(v.y) : "r"(a), "n"(OFF));
    return v;
}

// 1 << p in one instruction (bmsk: width-1 mask at position p)
__device__ __forceinline__ uint32_t bit_at(uint32_t p) {
    uint32_t m;
    asm("bmsk.clamp.b32 %0, %1, 1;" : "=r"(m) : "r"(p));
    return m;
}

// position of the most significant set bit (x != 0)
__device__ __forceinline__ uint32_t msb_pos(uint32_t x) {
    uint32_t p;
    asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(x));
    return p;
}

__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// An upper bound of 1 / x for normal x > 0, at most 12.5% above it, from one
// integer subtract (ALU pipe) instead of a MUFU.RCP: for x = 2^e (1 + f),
// 0x7F000000 - bits(x) is the float 2^(-e-1) (2 - f) (2^-e when f = 0), and
// x times it is (1 + f)(2 - f) / 2 in [1, 1.125].  Always finite (so 0 times
// it is 0, never NaN); for a subnormal x it is ~2^127 and no longer a bound,
// but there x sits within 1e-38 of the support edge and any error bound
// scaled by it is far above every certification threshold anyway.
__device__ __forceinline__ float rcp_upper(float x) {
    return __int_as_float(0x7F000000 - __float_as_int(x));
}

// Warp cover mask of one splat over a 16x16 tile whose warps are 8x4 pixel
// blocks (warp w covers columns 8 (w & 1) .. +7, rows 4 (w >> 1) .. +3).
// The conic factor maps a pixel offset to y0 = u00 dx + u01 dy, y1 = u11 dy
// (u00, u11 >= 0) and m = y0^2 + y1^2; over a warp's box both are linear, so
// their ranges come from the box corners and z0^2 + z1^2 (z = distance of
// each range from 0) is a lower bound of m over the box.  Bit w is clear only
// when that bound, less a 1e-5 relative slack in y0 (a hundred ulp of the
// terms, above the fp32 rounding of this test and of the per-pixel m), is
// still >= (tau + E)(1 + 1e-4): every pixel of the warp would have skipped
// the splat without raising its edge flag, so culling never changes a bit.
// Splat offset from the tile origin, (tx 16 - fx) + ox: the integer part is
// exact, so this is one rounding; a pixel's dx is then xa + lx (lx = 0..15 its
// column in the tile), the formula the preprocess error bound E covers
// (|d dx| <= u (2 |dx| + 15.5)).  fwd32 and bwd32 both stage it in shared
// memory so their in-support tests agree bit for bit.
__device__ __forceinline__ float2 tile_offset(const float4 r0, int tx, int ty) {
    return make_float2(((float)(tx * kTile) - r0.x) + r0.z, ((float)(ty * kTile) - r0.y) + r0.w);
}

__device__ __forceinline__ uint32_t warp_cover_mask(const float xa0, const float ya0, const float4 r1) {
    const float u00 = r1.x, u01 = r1.y, u11 = r1.z;
    const float thr = r1.w * (1.0f + 1.0e-4f);
    if (!isfinite(u00 + u01 + u11 + thr + xa0 + ya0)) return 0xffu;  // fmaxf would drop a NaN
    float clo[2], chi[2], cs[2];
#pragma unroll
    for (int wx = 0; wx < 2; ++wx) {
        clo[wx] = u00 * (xa0 + (float)(8 * wx));
        chi[wx] = u00 * (xa0 + (float)(8 * wx + 7));
        cs[wx] = fmaf(1.0e-5f, fabsf(clo[wx]) + fabsf(chi[wx]), 1.0e-6f);
    }
    uint32_t mask = 0;
#pragma unroll
    for (int wy = 0; wy < 4; ++wy) {
        const float ya = ya0 + (float)(4 * wy), yb = ya + 3.0f;
        const float z1 = fmaxf(0.0f, fmaxf(u11 * ya, -(u11 * yb)));
        const float z1sq = z1 * z1;
        const float ua = u01 * ya, ub = u01 * yb;
        const float umin = fminf(ua, ub), umax = fmaxf(ua, ub);
        const float us = 1.0e-5f * (fabsf(ua) + fabsf(ub));
#pragma unroll
        for (int wx = 0; wx < 2; ++wx) {
            const float z0 = fmaxf(fmaxf(clo[wx] + umin, -(chi[wx] + umax)) - (cs[wx] + us), 0.0f);
            if (fmaf(z0, z0, z1sq) < thr) mask |= 1u << (2 * wy + wx);
        }
    }
    return mask;
}

__device__ __forceinline__ uint32_t warp_cover_mask(const float4 r0, const float4 r1, int tx, int ty) {
    const float2 o = tile_offset(r0, tx, ty);
    return warp_cover_mask(o.x, o.y, r1);
}

// Per visit (in support): alpha = 2^(beta * lg2(1 - m/tau) + log2(og)) with
// the MUFU lg2/ex2 approximations; their error (qc, and 2.1e-7 per unit of
// the exponent) is part of the per-visit relative alpha bound
//     q = eb / (tau - m) + qc + 2.1e-7 |arg|
// (1 / (tau - m) taken as rcp_upper's bound, at most 12.5% above it),
// and D, the bound on |T32 - T64|, accumulates D (1 - a) + T a q + 2u T: the
// first-order error of T (D / T = sum a q / (1 - a) + 2u per visit).
// T and D change only on in-support visits, so the reference's cut test
// (T < t_min before each splat) and its certification band are evaluated
// right after each update: the next splat is iterated iff T >= t_min, exactly
// as in tile_forward.  Each warp walks only the splats whose cover mask has
// its bit (per-warp ballot words), and the contributor count is the list
// position where the pixel stopped (tile_forward counts every iterated splat).
__global__ void __launch_bounds__(kTileThreads)
raster_fwd32_kernel(const RasterParams P, const uint32_t *__restrict__ ranges, const uint32_t *__restrict__ ids,
                    const Rec32 *__restrict__ recs, float *__restrict__ image, float *__restrict__ asum,
                    float *__restrict__ tstop, int32_t *__restrict__ ncontrib, uint8_t *__restrict__ hit,
                    unsigned long long *__restrict__ visits, uint32_t *__restrict__ fix_list,
                    uint32_t *__restrict__ fix_count) {
    constexpr int kWarps = kTileThreads / 32;
    __shared__ Rec32 srec[kTileThreads];
    __shared__ uint32_t sid[kTileThreads];
    __shared__ uint32_t swm[kWarps][kWarps];  // [walking warp][loading warp] ballot words
    __shared__ unsigned long long red[kWarps];
    if (pairs_overflow(P.n_pairs, P.pair_capacity, nullptr)) return;
    const int tile = blockIdx.x;
    const int ty = tile / P.TX, tx = tile - ty * P.TX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const float lxf = (float)(px - tx * kTile), lyf = (float)(py - ty * kTile);
    const bool inside = px < P.W && py < P.H;
    uint32_t start, end;
    bool capped;
    tile_span(P, ranges, tile, start, end, capped);
    const float tau = (float)P.tau, inv_tau = (float)(1.0 / P.tau);
    const float clamp = (float)P.clamp, one_minus_clamp = (float)(1.0 - P.clamp);
    // alpha below clamp_lo cannot be clamp-ambiguous unless its error bound is
    // so large that D > kImgErrTol T flags the pixel anyway: a(1+q) > clamp
    // with a < clamp_lo implies a q / (1 - a) > clamp - clamp_lo >> kImgErrTol
    const float clamp_lo = clamp - 0.05f;
    const float tmin = (float)P.tmin;
    const float tmin_hi = tmin * (1.0f + 4.0e-3f);
    float T = 1.0f, a0 = 0.f, a1 = 0.f, a2 = 0.f;
    float D = 0.f;  // bound on |T32 - T64|
    uint32_t cnt = inside ? end - start : 0u;
    int flag = 0;
    float edge = 1.0f;  // min over out-of-support visits of m - (tau + E): < 0 flags the pixel
    bool done = !inside;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(srec);
    for (uint32_t b = start; b < end; b += kTileThreads) {
        if (__syncthreads_count(done) == kTileThreads) break;
        if (threadIdx.x == 0) FWD_STAT(6, 1);
        const uint32_t q = b + threadIdx.x;
        uint32_t cover = 0;
        if (q < end && UBS_GUARD((int64_t)q < P.pair_capacity, kChkPair)) {
            const uint32_t id = ids[q];
            const float4 *r = reinterpret_cast<const float4 *>(recs + id);
            float4 *d = reinterpret_cast<float4 *>(srec + threadIdx.x);
            sid[threadIdx.x] = id;
            const float4 r0 = __ldg(r), r1 = __ldg(r + 1);
            const float2 o = tile_offset(r0, tx, ty);
            d[0] = make_float4(o.x, o.y, r0.z, r0.w);
            d[1] = r1;
            d[2] = __ldg(r + 2);
            d[3] = __ldg(r + 3);
            cover = warp_cover_mask(o.x, o.y, r1);
        }
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t word = __ballot_sync(0xffffffffu, (cover >> w) & 1u);
            if (lane == 0) swm[w][warp] = __brev(word);  // splat order from the highest bit down
        }
        __syncthreads();
        if (!done) {
            const int nw = (int)((min((uint32_t)kTileThreads, end - b) + 31u) >> 5);
            for (int k = 0; k < nw && !done; ++k) {
                uint32_t bits = swm[warp][k];
                // bit p of the reversed word is splat 32 k + 31 - p, at stop - 64 p
                const uint32_t stop = sbase + (uint32_t)(32 * k + 31) * (uint32_t)sizeof(Rec32);
                while (bits) {
                    const uint32_t p = msb_pos(bits);
                    bits ^= bit_at(p);
                    const uint32_t ra = stop - (p << 6);
                    const float4 r0 = lds128<0>(ra), r1 = lds128<16>(ra);
                    const float dx = r0.x + lxf;  // tile_offset + column in the tile
                    const float dy = r0.y + lyf;
                    const float y0 = fmaf(r1.x, dx, r1.y * dy);
                    const float y1 = r1.z * dy;
                    const float m = fmaf(y0, y0, y1 * y1);
#ifdef UBS_FWD_STATS
                    {
                        const unsigned am = __activemask();
                        const unsigned inb = __ballot_sync(am, m < tau);
                        FWD_STAT(0, 1);
                        FWD_STAT(1, inb == 0u);
                        FWD_STAT(2, __popc(inb));
                        FWD_STAT(3, __popc(am));
                    }
#endif
                    if (m >= tau) {
                        edge = fminf(edge, m - r1.w);  // support edge within the m-error band
                        continue;
                    }
                    const float4 r2 = lds128<32>(ra), r3 = lds128<48>(ra);
                    const float arg = fmaf(r2.x, lg2_approx(fmaf(-m, inv_tau, 1.0f)), r3.w);
                    float a = ex2_approx(arg);
                    // relative alpha bound q = eb / (tau - m) + qc + 2.1e-7 |arg|
                    const float qrel = fmaf(r3.x, rcp_upper(tau - m), fmaf(fabsf(arg), 2.1e-7f, r3.z));
                    float om = 1.0f - a;
                    // T (1 - a) as T - a T: rounds a T and the difference (<= u T in
                    // all, inside the 2u T rounding term of D), and keeps T's register
                    float w = a * T;
                    float Tn = T - w;
#ifdef UBS_FWD_STATS
                    FWD_STAT(4, __any_sync(__activemask(), a > clamp_lo));
                    FWD_STAT(5, __any_sync(__activemask(), Tn < tmin_hi));
#endif
                    // blend + error-bound update: D' = D (1 - a) + T a q + rounding of
                    // 1 - a and of T (1 - a)
                    auto blend = [&]() {
                        a0 = fmaf(w, r2.y, a0);
                        a1 = fmaf(w, r2.z, a1);
                        a2 = fmaf(w, r2.w, a2);
                        D = fmaf(D, om, w * qrel);
                        T = Tn;
                        D = fmaf(1.2e-7f, T, D);
                    };
                    // one test for both rare cases (~3% of visits): alpha in the clamp
                    // band, or T about to cross the cut band
                    if (a > clamp_lo || Tn < tmin_hi) {
                        if (a > clamp_lo) {
                            if (a > clamp) {
                                if (a * (1.0f - qrel) > clamp &&
                                UBS_GUARD(32 * k + 31 - (int)p >= 0 && 32 * k + 31 - (int)p < kTileThreads, kChkSplat))
                                hit[sid[32 * k + 31 - (int)p]] = 1;
                                else flag = 1;
                                a = clamp;
                                om = one_minus_clamp;
                                w = a * T;
                                Tn = T - w;
                            } else {
                                flag |= (a * (1.0f + qrel) > clamp);
                            }
                        }
                        blend();
                        if (T < tmin_hi) {
                            const float slack = fmaf(1.0e-6f, tmin, D);
                            if (T < tmin) {
                                // the reference stops before the next splat; ending the walk
                                // through the loop condition (bits = 0, !done) avoids a
                                // divergent break
                                flag |= (T > tmin - slack);
                                done = true;
                                cnt = b - start + (uint32_t)(32 * k + 31) - p + 1u;
                                bits = 0u;
                            } else {
                                flag |= (T < tmin + slack);
                            }
                        }
                    } else {
                        blend();
                    }
                }
            }
        }
    }
    if (capped && inside && !done) atomicOr(P.status, (uint32_t)UBS_S_LIST_TRUNC);
    if (D > kImgErrTol * T || edge < 0.0f) flag = 1;
    if (inside && UBS_GUARD((int64_t)py * P.W + px < (int64_t)P.W * P.H, kChkPixel)) {
        const int64_t pix = (int64_t)py * P.W + px;
        image[3 * pix] = fmaf(T, (float)P.bg[0], a0);
        image[3 * pix + 1] = fmaf(T, (float)P.bg[1], a1);
        image[3 * pix + 2] = fmaf(T, (float)P.bg[2], a2);
        asum[pix] = 1.0f - T;  // sum_i a_i T_i telescopes to 1 - T
        tstop[pix] = T;
        ncontrib[pix] = (int32_t)cnt;
    }
    const bool fl = flag && inside;
    const unsigned fb = __ballot_sync(0xffffffffu, fl);
    if (fb) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(fix_count, (uint32_t)__popc(fb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (fl && UBS_GUARD((int64_t)base + __popc(fb & ((1u << lane) - 1u)) < (int64_t)P.W * P.H, kChkFix))
            fix_list[base + __popc(fb & ((1u << lane) - 1u))] = (uint32_t)((int64_t)py * P.W + px);
    }
    __syncthreads();
    const unsigned long long tot = block_sum_u64((unsigned long long)cnt, red);
    if (threadIdx.x == 0 && tot) atomicAdd(visits, tot);
}

// ---------------------------------------------------------------------------
// forward, fp32, two pixels per lane with Blackwell's packed fp32x2 math
// ---------------------------------------------------------------------------
// Same algorithm, records, error bound and decisions as raster_fwd32_kernel,
// pixel for pixel: each of the 4 warps of a 128-thread CTA owns an 8x8 block
// of the 16x16 tile = two of the 8x4 blocks, and each lane carries the pixel
// pair (x, y) and (x, y + 4) -- one from each block.  The walk (bit scan,
// record address, shared loads) is paid once per pair, and the per-pixel
// arithmetic runs as sm_100 FADD2 / FMUL2 / FFMA2 instructions on the pair
// (PTX add/mul/fma.rn.f32x2, IEEE round-to-nearest per element, so every
// pixel sees exactly the scalar kernel's operations and roundings; uniform
// operands are broadcast by the .F32 operand selector, no moves).  MUFU
// transcendentals stay scalar.  A warp walks a splat when its cover mask has
// either block's bit; a pixel whose block bit is clear is out of support
// (every pixel of a culled block would skip the splat: warp_cover_mask).
// f32x2 pair helpers: f32x2.cuh

constexpr int kX2Threads = kTileThreads / 2;  // 128: 4 warps x 32 lanes x 2 pixels
constexpr int kX2Warps = kX2Threads / 32;

__global__ void __launch_bounds__(kX2Threads)
raster_fwd32x2_kernel(const RasterParams P, const uint32_t *__restrict__ ranges, const uint32_t *__restrict__ ids,
                      const Rec32 *__restrict__ recs, float *__restrict__ image, float *__restrict__ asum,
                      float *__restrict__ tstop, int32_t *__restrict__ ncontrib, uint8_t *__restrict__ hit,
                      unsigned long long *__restrict__ visits, uint32_t *__restrict__ fix_list,
                      uint32_t *__restrict__ fix_count) {
    constexpr int kBatch = kTileThreads;      // 256 records per batch, 2 staged per thread
    constexpr int kWords = kBatch / 32;
    __shared__ Rec32 srec[kBatch];
    __shared__ uint32_t sid[kBatch];
    __shared__ uint32_t swm[kX2Warps][kWords];  // [walking warp][record word] ballot words
    __shared__ unsigned long long red[kX2Warps];
    if (pairs_overflow(P.n_pairs, P.pair_capacity, nullptr)) return;
    const int tile = blockIdx.x;
    const int ty = tile / P.TX, tx = tile - ty * P.TX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wx = warp & 1, wy = warp >> 1;
    // this warp's two 8x4 blocks are warp_cover_mask bits 2 (2 wy) + wx and that + 2
    const int lx = 8 * wx + (lane & 7), ly = 8 * wy + (lane >> 3);  // pixel 0; pixel 1 is 4 rows down
    const int px = tx * kTile + lx, py0 = ty * kTile + ly, py1 = py0 + 4;
    const bool in0 = px < P.W && py0 < P.H, in1 = px < P.W && py1 < P.H;
    uint32_t start, end;
    bool capped;
    tile_span(P, ranges, tile, start, end, capped);
    const float tau = (float)P.tau, inv_tau = (float)(1.0 / P.tau);
    const float clamp = (float)P.clamp;
    const float clamp_lo = clamp - 0.05f;
    const float og_lo = clamp_lo / (1.0f + 1.0e-4f);
    const float tmin = (float)P.tmin;
    const float tmin_hi = tmin * (1.0f + 4.0e-3f);
    const float lxf = (float)lx;
    const f32x2 lyf = pk2((float)ly, (float)(ly + 4));
    // per-pixel state as scalars (packed ops read T0:T1 as an adjacent pair; a
    // loop-carried f32x2 would cost a register-pair copy per visit in ptxas)
    float T0 = 1.0f, T1 = 1.0f, D0 = 0.0f, D1 = 0.0f;
    float c00 = 0.0f, c01 = 0.0f, c10 = 0.0f, c11 = 0.0f, c20 = 0.0f, c21 = 0.0f;
    float edge0 = 1.0f, edge1 = 1.0f;
    uint32_t cnt0 = in0 ? end - start : 0u, cnt1 = in1 ? end - start : 0u;
    int flag0 = 0, flag1 = 0;
    bool done0 = !in0, done1 = !in1;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(srec);
    for (uint32_t b = start; b < end; b += kBatch) {
        if (__syncthreads_count(done0 && done1) == kX2Threads) break;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int jl = i * kX2Threads + (int)threadIdx.x;
            const uint32_t q = b + (uint32_t)jl;
            uint32_t cover = 0;
            if (q < end && UBS_GUARD((int64_t)q < P.pair_capacity, kChkPair)) {
                const uint32_t id = ids[q];
                const float4 *r = reinterpret_cast<const float4 *>(recs + id);
                float4 *d = reinterpret_cast<float4 *>(srec + jl);
                sid[jl] = id;
                const float4 r0 = __ldg(r), r1 = __ldg(r + 1);
                const float2 o = tile_offset(r0, tx, ty);
                d[0] = make_float4(o.x, o.y, r0.z, r0.w);
                d[1] = r1;
                d[2] = __ldg(r + 2);
                d[3] = __ldg(r + 3);
                cover = warp_cover_mask(o.x, o.y, r1);
            }
#pragma unroll
            for (int w = 0; w < kX2Warps; ++w) {
                const int c0w = 2 * (2 * (w >> 1)) + (w & 1);
                const uint32_t word = __ballot_sync(0xffffffffu, ((cover >> c0w) | (cover >> (c0w + 2))) & 1u);
                if (lane == 0) swm[w][jl >> 5] = __brev(word);  // splat order from the highest bit down
            }
        }
        __syncthreads();
        if (!(done0 && done1)) {
            const int nw = (int)((min((uint32_t)kBatch, end - b) + 31u) >> 5);
            for (int k = 0; k < nw && !(done0 && done1); ++k) {
                uint32_t bits = swm[warp][k];
                // bit p of the reversed word is splat 32 k + 31 - p, at stop - 64 p
                const uint32_t stop = sbase + (uint32_t)(32 * k + 31) * (uint32_t)sizeof(Rec32);
                while (bits) {
                    const uint32_t p = msb_pos(bits);
                    bits ^= bit_at(p);
                    const uint32_t ra = stop - (p << 6);
                    const float4 r0 = lds128<0>(ra), r1 = lds128<16>(ra);
                    const float dx = r0.x + lxf;  // the pair shares its column
                    const f32x2 dy = add2(dup2(r0.y), lyf);
                    const f32x2 y0 = fma2(dup2(r1.x), dup2(dx), mul2(dup2(r1.y), dy));
                    const f32x2 y1 = mul2(dup2(r1.z), dy);
                    const float2 m = up2(fma2(y0, y0, mul2(y1, y1)));
                    const bool s0 = !done0 && m.x < tau, s1 = !done1 && m.y < tau;
                    const f32x2 m2 = pk2(m.x, m.y);
                    const f32x2 tm = sub2(dup2(tau), m2);
                    // support edge within the m-error band, m in [tau, tau + E): there
                    // (tau - m) (tau + E - m) <= 0, elsewhere > 0 (in-support pixels too).
                    // A done pixel is tested as well: that band is ~1e-5 tau wide, a flag
                    // there is only a spare fix-up.
                    const float2 eg = up2(mul2(tm, sub2(dup2(r1.w), m2)));
                    edge0 = fminf(edge0, eg.x);
                    edge1 = fminf(edge1, eg.y);
                    if (!(s0 || s1)) continue;
                    const float4 r2 = lds128<32>(ra), r3 = lds128<48>(ra);
                    const float2 omx = up2(fma2(m2, dup2(-inv_tau), dup2(1.0f)));
                    const f32x2 arg = fma2(dup2(r2.x), pk2(lg2_approx(omx.x), lg2_approx(omx.y)), dup2(r3.w));
                    const float2 ag = up2(arg);
                    float a0 = s0 ? ex2_approx(ag.x) : 0.0f, a1 = s1 ? ex2_approx(ag.y) : 0.0f;
                    // q = eb / (tau - m) + qc + 2.1e-7 |arg|, with |arg| = -arg (arg =
                    // beta lg2(1 - x) + log2(og) <= 0 up to the lg2 approximation's
                    // 2^-22 near 1, whose 1e-13 effect hides in qc's 4e-7 term)
                    const float2 tmv = up2(tm);
                    const float2 qr = up2(fma2(dup2(r3.x), pk2(rcp_upper(tmv.x), rcp_upper(tmv.y)),
                                               fma2(arg, dup2(-2.1e-7f), dup2(r3.z))));
                    // zero for a pixel not in support: its w = 0, and q may be +-inf
                    // (m == tau, or eb = inf for a thin splat) where 0 q would be NaN
                    const f32x2 q = pk2(s0 ? qr.x : 0.0f, s1 ? qr.y : 0.0f);
                    // alpha <= og (1 + 1e-5) (omx <= 1, MUFU error): a splat with og below
                    // clamp_lo / (1 + 1e-4) never reaches the band -- a warp-uniform test
                    if (r3.y > og_lo && (a0 > clamp_lo || a1 > clamp_lo)) {
                        // clamp band (rare; scalar per pixel, as raster_fwd32_kernel)
                        const float2 qv = up2(q);
                        if (a0 > clamp_lo) {
                            if (a0 > clamp) {
                                if (a0 * (1.0f - qv.x) > clamp &&
                                    UBS_GUARD(32 * k + 31 - (int)p < kBatch, kChkSplat))
                                    hit[sid[32 * k + 31 - (int)p]] = 1;
                                else flag0 = 1;
                                a0 = clamp;  // 1 - clamp == one_minus_clamp exactly
                            } else {
                                flag0 |= (a0 * (1.0f + qv.x) > clamp);
                            }
                        }
                        if (a1 > clamp_lo) {
                            if (a1 > clamp) {
                                if (a1 * (1.0f - qv.y) > clamp &&
                                    UBS_GUARD(32 * k + 31 - (int)p < kBatch, kChkSplat))
                                    hit[sid[32 * k + 31 - (int)p]] = 1;
                                else flag1 = 1;
                                a1 = clamp;
                            } else {
                                flag1 |= (a1 * (1.0f + qv.y) > clamp);
                            }
                        }
                    }
                    // blend + error-bound update of the pair:
                    // D' = D (1 - a) + T a q + rounding of 1 - a and of T (1 - a)
                    const f32x2 a2 = pk2(a0, a1);
                    const float2 w = up2(mul2(a2, pk2(T0, T1)));
                    const float2 om = up2(sub2(dup2(1.0f), a2));
                    const float2 wq = up2(mul2(pk2(w.x, w.y), q));
                    c00 = fmaf(w.x, r2.y, c00);
                    c01 = fmaf(w.y, r2.y, c01);
                    c10 = fmaf(w.x, r2.z, c10);
                    c11 = fmaf(w.y, r2.z, c11);
                    c20 = fmaf(w.x, r2.w, c20);
                    c21 = fmaf(w.y, r2.w, c21);
                    D0 = fmaf(D0, om.x, wq.x);
                    D1 = fmaf(D1, om.y, wq.y);
                    T0 = T0 - w.x;  // T (1 - a) as T - a T (see raster_fwd32_kernel)
                    T1 = T1 - w.y;
                    D0 = fmaf(1.2e-7f, T0, D0);
                    D1 = fmaf(1.2e-7f, T1, D1);
                    const float2 Tn = make_float2(T0, T1);
                    if ((s0 && Tn.x < tmin_hi) | (s1 && Tn.y < tmin_hi)) {
                        // the cut (rare; scalar per pixel): the reference stops before the
                        // next splat once T < t_min; certified within D + 1e-6 t_min
                        const float2 Dv = make_float2(D0, D1);
                        const uint32_t pos = b - start + (uint32_t)(32 * k + 31) - p + 1u;
                        if (s0 && Tn.x < tmin_hi) {
                            const float slack = fmaf(1.0e-6f, tmin, Dv.x);
                            if (Tn.x < tmin) {
                                flag0 |= (Tn.x > tmin - slack);
                                flag0 |= Dv.x > kImgErrTol * Tn.x;
                                done0 = true;
                                cnt0 = pos;
                            } else {
                                flag0 |= (Tn.x < tmin + slack);
                            }
                        }
                        if (s1 && Tn.y < tmin_hi) {
                            const float slack = fmaf(1.0e-6f, tmin, Dv.y);
                            if (Tn.y < tmin) {
                                flag1 |= (Tn.y > tmin - slack);
                                flag1 |= Dv.y > kImgErrTol * Tn.y;
                                done1 = true;
                                cnt1 = pos;
                            } else {
                                flag1 |= (Tn.y < tmin + slack);
                            }
                        }
                        if (done0 && done1) bits = 0u;  // ends the walk through the loop condition
                    }
                }
            }
        }
    }
    if (capped && ((in0 && !done0) || (in1 && !done1))) atomicOr(P.status, (uint32_t)UBS_S_LIST_TRUNC);
    const float2 Tf = make_float2(T0, T1), Df = make_float2(D0, D1), C0 = make_float2(c00, c01),
                 C1 = make_float2(c10, c11), C2 = make_float2(c20, c21);
    if (!done0 && Df.x > kImgErrTol * Tf.x) flag0 = 1;
    if (!done1 && Df.y > kImgErrTol * Tf.y) flag1 = 1;
    if (!(edge0 > 0.0f)) flag0 = 1;  // some visit had m in [tau, tau + E)
    if (!(edge1 > 0.0f)) flag1 = 1;
    [[maybe_unused]] const int64_t npix = (int64_t)P.W * P.H;  // bounds guards (checked builds)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const bool inside = h ? in1 : in0;
        const int py = h ? py1 : py0;
        const float Th = h ? Tf.y : Tf.x;
        if (inside && UBS_GUARD((int64_t)py * P.W + px < npix, kChkPixel)) {
            const int64_t pix = (int64_t)py * P.W + px;
            image[3 * pix] = fmaf(Th, (float)P.bg[0], h ? C0.y : C0.x);
            image[3 * pix + 1] = fmaf(Th, (float)P.bg[1], h ? C1.y : C1.x);
            image[3 * pix + 2] = fmaf(Th, (float)P.bg[2], h ? C2.y : C2.x);
            asum[pix] = 1.0f - Th;  // sum_i a_i T_i telescopes to 1 - T
            tstop[pix] = Th;
            ncontrib[pix] = (int32_t)(h ? cnt1 : cnt0);
        }
        const bool fl = (h ? flag1 : flag0) && inside;
        const unsigned fb = __ballot_sync(0xffffffffu, fl);
        if (fb) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(fix_count, (uint32_t)__popc(fb));
            base = __shfl_sync(0xffffffffu, base, 0);
            const uint32_t at = base + __popc(fb & ((1u << lane) - 1u));
            if (fl && UBS_GUARD((int64_t)at < npix, kChkFix)) fix_list[at] = (uint32_t)((int64_t)py * P.W + px);
        }
    }
    // processed_pixels: every pixel's count, one atomic per CTA
    unsigned long long c = (unsigned long long)cnt0 + (unsigned long long)cnt1;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) red[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < kX2Warps; ++w) tot += red[w];
        if (tot) atomicAdd(visits, tot);
    }
}

// ---------------------------------------------------------------------------
// forward, fp64 (bit-faithful to tile_forward)
// ---------------------------------------------------------------------------
// The reference's per-pixel loop in its operation order (no FMA contraction),
// on the fp32 kernel's 8x4-pixel warps: each warp walks only the splats whose
// cover mask has its bit.  The masks come from each record's fp64 conic
// rounded to the fp32 factor form with a 1e-3 relative margin on tau (far
// above that rounding), so a culled splat is one every pixel of the warp
// evaluates to m >= tau in fp64 anyway; the contributor count is the list
// position where T first fell below t_min (tile_forward counts every iterated
// splat), exactly as in the fp32 kernel.
__device__ __forceinline__ uint32_t warp_cover_mask64(const Rec64 &r, float tau, int tx, int ty) {
    if (!(fabs(r.mx) < 4.0e6 && fabs(r.my) < 4.0e6) || !(r.p00 > 0.0)) return 0xffu;
    const double fx = floor(r.mx), fy = floor(r.my);
    const double u00 = sqrt(r.p00), u01 = r.p01 / u00;
    const double u11 = sqrt(fmax(r.p11 - u01 * u01, 0.0));
    const float4 r0 = make_float4((float)fx, (float)fy, (float)(0.5 - (r.mx - fx)), (float)(0.5 - (r.my - fy)));
    const float4 r1 = make_float4((float)u00, (float)u01, (float)u11, tau * 1.001f);
    return warp_cover_mask(r0, r1, tx, ty);
}

__global__ void __launch_bounds__(kTileThreads)
raster_fwd64_kernel(const RasterParams P, const uint32_t *__restrict__ ranges, const uint32_t *__restrict__ ids,
                    const Rec64 *__restrict__ recs, double *__restrict__ image, double *__restrict__ asum,
                    double *__restrict__ tstop, int32_t *__restrict__ ncontrib, uint8_t *__restrict__ hit,
                    unsigned long long *__restrict__ visits) {
    constexpr int kWarps = kTileThreads / 32;
    __shared__ Rec64 srec[kTileThreads];
    __shared__ uint32_t sid[kTileThreads];
    __shared__ uint32_t swm[kWarps][kWarps];
    __shared__ unsigned long long red[kWarps];
    if (pairs_overflow(P.n_pairs, P.pair_capacity, nullptr)) return;
    const int tile = blockIdx.x;
    const int ty = tile / P.TX, tx = tile - ty * P.TX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = px < P.W && py < P.H;
    uint32_t start, end;
    bool capped;
    tile_span(P, ranges, tile, start, end, capped);
    const double pxc = (double)px + 0.5, pyc = (double)py + 0.5;
    const double tau = P.tau, clamp = P.clamp, tmin = P.tmin;
    double T = 1.0, a0 = 0.0, a1 = 0.0, a2 = 0.0, ws = 0.0;
    uint32_t cnt = inside ? end - start : 0u;
    bool done = !inside;
    for (uint32_t b = start; b < end; b += kTileThreads) {
        if (__syncthreads_count(done) == kTileThreads) break;
        const uint32_t q = b + threadIdx.x;
        uint32_t cover = 0;
        if (q < end) {
            const uint32_t id = ids[q];
            sid[threadIdx.x] = id;
            const Rec64 r = recs[id];
            srec[threadIdx.x] = r;
            cover = warp_cover_mask64(r, (float)tau, tx, ty);
        }
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t word = __ballot_sync(0xffffffffu, (cover >> w) & 1u);
            if (lane == 0) swm[w][warp] = word;
        }
        __syncthreads();
        if (!done) {
            const int nw = (int)((min((uint32_t)kTileThreads, end - b) + 31u) >> 5);
            for (int k = 0; k < nw && !done; ++k) {
                uint32_t bits = swm[warp][k];
                while (bits) {
                    const int j = (k << 5) + __ffs(bits) - 1;  // ascending list order
                    bits &= bits - 1u;
                    const Rec64 &r = srec[j];
                    const double dx = sub(pxc, r.mx), dy = sub(pyc, r.my);
                    const double m = add(add(mul(mul(r.p00, dx), dx), mul(mul(mul(2.0, r.p01), dx), dy)),
                                         mul(mul(r.p11, dy), dy));
                    if (m >= tau) continue;
                    double a = mul(r.og, exp(mul(r.bx, log1p(-m / tau))));
                    if (a > clamp) {
                        a = clamp;
                        hit[sid[j]] = 1;
                    }
                    const double w = mul(a, T);
                    a0 = add(a0, mul(w, r.cr));
                    a1 = add(a1, mul(w, r.cg));
                    a2 = add(a2, mul(w, r.cb));
                    ws = add(ws, w);
                    T = mul(T, sub(1.0, a));
                    if (T < tmin) {  // the reference stops before the next splat
                        done = true;
                        cnt = b - start + (uint32_t)j + 1u;
                        bits = 0u;
                    }
                }
            }
        }
    }
    if (capped && inside && !done) atomicOr(P.status, (uint32_t)UBS_S_LIST_TRUNC);
    if (inside) {
        const int64_t pix = (int64_t)py * P.W + px;
        image[3 * pix] = add(a0, mul(T, P.bg[0]));
        image[3 * pix + 1] = add(a1, mul(T, P.bg[1]));
        image[3 * pix + 2] = add(a2, mul(T, P.bg[2]));
        asum[pix] = ws;
        tstop[pix] = T;
        ncontrib[pix] = (int32_t)cnt;
    }
    __syncthreads();
    const unsigned long long tot = block_sum_u64((unsigned long long)cnt, red);
    if (threadIdx.x == 0 && tot) atomicAdd(visits, tot);
}

#ifndef UBS_FIX_THREADS
#define UBS_FIX_THREADS 128
#endif
#ifndef UBS_FIX_CTAS_PER_SM
#define UBS_FIX_CTAS_PER_SM 4
#endif
constexpr int kFixThreads = UBS_FIX_THREADS;  // fix-up CTA size; grid = 148 x UBS_FIX_CTAS_PER_SM

// fp64 replay of flagged pixels: one warp per pixel, chunks of 32 splats.
//  1. lanes evaluate alpha_k (reference formula and rounding, clamp applied)
//     and 1 - alpha_k in parallel;
//  2. lane 0 runs the only truly sequential part, T_{k+1} = T_k (1 - alpha_k),
//     exactly as tile_forward rounds it, straight through the chunk (T is
//     non-increasing, so the early-out index is a ballot count of T_k >= t_min)
//     and publishes T_k through shared memory;
//  3. lanes accumulate w_k = alpha_k T_k times colour in per-lane sums, reduced
//     once per pixel (summation order differs from the reference only at the
//     1e-16 level; T, the contributor count and the clamp flags are exact).
__global__ void __launch_bounds__(kFixThreads)
raster_fixup_kernel(const RasterParams P, const uint32_t *__restrict__ ranges, const uint32_t *__restrict__ ids,
                    const Rec64 *__restrict__ recs, const uint32_t *__restrict__ fix_list,
                    const uint32_t *__restrict__ fix_count, float *__restrict__ image, float *__restrict__ asum,
                    float *__restrict__ tstop, int32_t *__restrict__ ncontrib, uint8_t *__restrict__ hit,
                    unsigned long long *__restrict__ visits) {
    __shared__ double s_om[kFixThreads / 32][32], s_T[kFixThreads / 32][33];
    if (pairs_overflow(P.n_pairs, P.pair_capacity, nullptr)) return;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const uint32_t nfix = *fix_count;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const double tau = P.tau, clamp = P.clamp, tmin = P.tmin;
    for (uint32_t wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nfix; wi += warps) {
        const uint32_t pix = fix_list[wi];
        const int py = pix / P.W, px = pix - py * P.W;
        const int tile = (py / kTile) * P.TX + px / kTile;
        uint32_t start, end;
        bool capped;
        tile_span(P, ranges, tile, start, end, capped);
        const double pxc = (double)px + 0.5, pyc = (double)py + 0.5;
        double T = 1.0, a0 = 0.0, a1 = 0.0, a2 = 0.0, ws = 0.0;
        double l0 = 0.0, l1 = 0.0, l2 = 0.0, lw = 0.0;
        int cnt = 0;
        bool done = false;
        uint32_t q = start + lane;
        uint32_t id = q < end ? ids[q] : 0u;
        for (uint32_t b = start; b < end && !done; b += 32) {
            double a = 0.0, cr = 0.0, cg = 0.0, cb = 0.0;
            const bool valid = q < end;
            if (valid) {
                const Rec64 r = recs[id];
                const double dx = sub(pxc, r.mx), dy = sub(pyc, r.my);
                const double m = add(add(mul(mul(r.p00, dx), dx), mul(mul(mul(2.0, r.p01), dx), dy)),
                                     mul(mul(r.p11, dy), dy));
                if (m < tau) a = mul(r.og, exp(mul(r.bx, log1p(-m / tau))));
                cr = r.cr; cg = r.cg; cb = r.cb;
            }
            const uint32_t my_id = id;
            // prefetch the next chunk's id while the chain runs
            q += 32;
            id = q < end ? ids[q] : 0u;
            const bool clamped = a > clamp;
            if (clamped) a = clamp;
            s_om[wl][lane] = sub(1.0, a);
            __syncwarp();
            const int nb = (int)min(32u, end - b);
            if (lane == 0) {
                // T_k = T_{k-1} (1 - a_{k-1}) for the whole chunk, unconditionally:
                // T is non-increasing, so the reference's stop (first T_k < t_min)
                // is the count of T_k >= t_min; lanes past the list have 1 - 0 == 1
                double t = T;
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    s_T[wl][k] = t;
                    t = mul(t, s_om[wl][k]);
                }
                s_T[wl][32] = t;
            }
            __syncwarp();
            const double Tk = s_T[wl][lane];
            const int stop = __popc(__ballot_sync(0xffffffffu, lane < nb && Tk >= tmin));
            cnt += stop;
            done = stop < nb;
            if (lane < stop && a != 0.0) {
                const double w = mul(a, Tk);
                l0 += w * cr;
                l1 += w * cg;
                l2 += w * cb;
                lw += w;
                if (clamped) hit[my_id] = 1;
            }
            T = s_T[wl][stop];
            if (!done && T < tmin) done = true;  // crossed on the chunk's last splat
            __syncwarp();
        }
        // per-lane partial sums, reduced once (summation order differs from the
        // reference's sequential sum only at the 1e-16 level)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
            l2 += __shfl_xor_sync(0xffffffffu, l2, o);
            lw += __shfl_xor_sync(0xffffffffu, lw, o);
        }
        a0 = l0; a1 = l1; a2 = l2; ws = lw;
        if (lane == 0 && capped && !done) atomicOr(P.status, (uint32_t)UBS_S_LIST_TRUNC);
        if (lane == 0) {
            image[3 * (int64_t)pix] = (float)add(a0, mul(T, P.bg[0]));
            image[3 * (int64_t)pix + 1] = (float)add(a1, mul(T, P.bg[1]));
            image[3 * (int64_t)pix + 2] = (float)add(a2, mul(T, P.bg[2]));
            asum[pix] = (float)ws;
            tstop[pix] = (float)T;
            const int old = ncontrib[pix];
            ncontrib[pix] = cnt;
            if (old != cnt) atomicAdd(visits, (unsigned long long)(long long)(cnt - old));
        }
    }
}

// ---------------------------------------------------------------------------
// backward: reverse replay of the blend (tile_backward), warp-reduced atomics
// ---------------------------------------------------------------------------
// alpha (clamped), 1 - alpha, and the operands of its derivative at a pixel
struct SplatEval {
    double dx, dy, m, a, om, og, bx, c0, c1, c2;
};

__device__ __forceinline__ void eval_splat(const Rec64 &r, int px, int py, double tau, double clamp,
                                           double one_minus_clamp, SplatEval &e) {
    e.dx = sub((double)px + 0.5, r.mx);
    e.dy = sub((double)py + 0.5, r.my);
    e.m = add(add(mul(mul(r.p00, e.dx), e.dx), mul(mul(mul(2.0, r.p01), e.dx), e.dy)), mul(mul(r.p11, e.dy), e.dy));
    e.og = r.og; e.bx = r.bx; e.c0 = r.cr; e.c1 = r.cg; e.c2 = r.cb;
    e.a = (e.m < tau) ? mul(e.og, exp(mul(e.bx, log1p(-e.m / tau)))) : 0.0;
    if (e.a > clamp) e.a = clamp;
    e.om = sub(1.0, e.a);
}

__device__ __forceinline__ double log1p_(double x) { return log1p(x); }
__device__ __forceinline__ double rcp_(double x) { return 1.0 / x; }

// One pixel's share of tile_backward (_tiles.py:97-127) for one splat, in
// the reference's operation order, T_i rebuilt by division from T_final;
// the pixel's sums are ADDED to v (raw moments: prim_bwd applies -2 P,
// -beta / tau and 1 / og per primitive).  Returns whether alpha != 0.
__device__ __forceinline__ bool bwd64_pixel(const Rec64 &r, int px, int py, double tau, double clamp,
                                            double one_minus_clamp, double g0, double g1, double g2, double &T,
                                            double &suffix, double (&v)[16]) {
    SplatEval e;
    eval_splat(r, px, py, tau, clamp, one_minus_clamp, e);
    if (e.a == (double)0) return false;
    const double iom = rcp_(e.om);
    const double ti = T * iom;
    const double w = e.a * ti;
    v[7] += w * g0;
    v[8] += w * g1;
    v[9] += w * g2;
    const double gc = g0 * e.c0 + g1 * e.c1 + g2 * e.c2;
    const double ga = gc * ti - suffix * iom;
    suffix += gc * w;
    T = ti;
    if (e.a < clamp) {
        const double x = e.m / tau;
        const double gaa = ga * e.a;
        v[5] += gaa;
        v[6] += gaa * log1p_(-x);
        const double h = gaa / ((double)1 - x);
        v[0] += h * e.dx;
        v[1] += h * e.dy;
        v[2] += h * e.dx * e.dx;
        v[3] += h * e.dx * e.dy;
        v[4] += h * e.dy * e.dy;
    }
    return true;
}

// Warp sums of 10 per-lane values in 12 exchanges (a 3-level split takes 14):
// a reduce-scatter over lane bit 16 (components 0-4 stay with the lower
// half, 5-9 go to the upper), then over bit 8 on the pairs (0,1), (2,3) of
// each half's five with the fifth summed on both sides, over bit 4 on the
// remaining pair and the fifth, over bit 2 between that component and the
// fifth, and a last butterfly over bit 1.  Lane l ends with component
// reduce10_index(l) of its half (-1 for the lanes whose copy is not the one
// reported: odd lanes, and the redundant holders of the fifth).
template <typename T>
__device__ __forceinline__ T warp_reduce10_value(T (&v)[16], int lane) {
    const bool u16 = (lane & 16) != 0, u8 = (lane & 8) != 0, u4 = (lane & 4) != 0, u2 = (lane & 2) != 0;
    T w[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {  // bit 16: lower keeps 0-4, upper keeps 5-9
        const T send = u16 ? v[i] : v[i + 5];
        const T keep = u16 ? v[i + 5] : v[i];
        w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    T x[3];
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // bit 8: pairs (0, 1), (2, 3)
        const T send = u8 ? w[2 * j] : w[2 * j + 1];
        const T keep = u8 ? w[2 * j + 1] : w[2 * j];
        x[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    x[2] = w[4] + __shfl_xor_sync(0xffffffffu, w[4], 8);
    T y0, y1;
    {  // bit 4: pair (x0, x1), and the fifth
        const T send = u4 ? x[0] : x[1];
        const T keep = u4 ? x[1] : x[0];
        y0 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        y1 = x[2] + __shfl_xor_sync(0xffffffffu, x[2], 4);
    }
    // bit 2: lower keeps y0 (a pair component), upper keeps the fifth
    const T send = u2 ? y0 : y1;
    const T keep = u2 ? y1 : y0;
    T r = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}
__device__ __forceinline__ int reduce10_index(int lane) {
    if (lane & 1) return -1;
    const int base = (lane & 16) ? 5 : 0;
    if (lane & 2) return (lane & 12) ? -1 : base + 4;  // the fifth: one reporter per half
    // pair component: bit 4 picks the pair (0,1) / (2,3), bit 8 its member
    return base + 2 * ((lane >> 2) & 1) + ((lane >> 3) & 1);
}

// fp64 backward (tile_backward, _tiles.py:59-127) in the reference's operation order
__global__ void __launch_bounds__(kTileThreads)
raster_bwd64_kernel(const RasterParams P, const uint32_t *__restrict__ ranges, const uint32_t *__restrict__ ids,
                  const Rec64 *__restrict__ recs, const double *__restrict__ tstop,
                  const int32_t *__restrict__ ncontrib, const double *__restrict__ g_image, double *__restrict__ grad2d) {
    constexpr int kWarps = kTileThreads / 32;
    __shared__ Rec64 srec[kTileThreads];
    __shared__ uint32_t sid[kTileThreads];
    __shared__ uint32_t swm[kWarps][kWarps];  // [walking warp][loading warp] ballot words
    __shared__ int smax;
    if (pairs_overflow(P.n_pairs, P.pair_capacity, nullptr)) return;
    const int tile = blockIdx.x;
    const int ty = tile / P.TX, tx = tile - ty * P.TX;
    // the forward kernels' 8x4-pixel warps, walking only the splats whose
    // cover mask (from the fp64 conic, 1e-3 margin: raster_fwd64_kernel) has
    // their bit -- a culled splat has alpha == 0 at every pixel of the warp
    const int warp = threadIdx.x >> 5;
    const int px = tx * kTile + (warp & 1) * 8 + (threadIdx.x & 7);
    const int py = ty * kTile + (warp >> 1) * 4 + ((threadIdx.x & 31) >> 3);
    const bool inside = px < P.W && py < P.H;
    const uint32_t start = ranges[2 * tile];
    const int64_t pix = (int64_t)py * P.W + px;
    int my_cnt = 0;
    double T = 0, g0 = 0, g1 = 0, g2 = 0;
    if (threadIdx.x == 0) smax = 0;
    __syncthreads();
    if (inside) {
        my_cnt = ncontrib[pix];
        T = tstop[pix];
        g0 = g_image[3 * pix];
        g1 = g_image[3 * pix + 1];
        g2 = g_image[3 * pix + 2];
        atomicMax(&smax, my_cnt);
    }
    __syncthreads();
    const int max_cnt = smax;
    int warp_cnt = my_cnt;  // this warp's largest contributor count: splats beyond it are skipped
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) warp_cnt = max(warp_cnt, __shfl_xor_sync(0xffffffffu, warp_cnt, o));
    const double tau = (double)P.tau, clamp = (double)P.clamp, one_minus_clamp = (double)(1.0 - P.clamp);
    double suffix = (g0 * (double)P.bg[0] + g1 * (double)P.bg[1] + g2 * (double)P.bg[2]) * T;
    const int lane = threadIdx.x & 31;
    for (int hi = max_cnt; hi > 0; hi -= kTileThreads) {
        const int lo = hi > kTileThreads ? hi - kTileThreads : 0;
        __syncthreads();
        const int q = lo + (int)threadIdx.x;
        uint32_t cover = 0;
        if (q < hi) {
            const uint32_t id = ids[start + q];
            sid[threadIdx.x] = id;
            const Rec64 r = recs[id];
            srec[threadIdx.x] = r;
            cover = warp_cover_mask64(r, (float)tau, tx, ty);
        }
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t word = __ballot_sync(0xffffffffu, (cover >> w) & 1u);
            if (lane == 0) swm[w][warp] = word;
        }
        __syncthreads();
        const int top = min(hi, warp_cnt) - lo;  // splats [lo, lo + top) concern this warp
        for (int kw = (top - 1) >> 5; kw >= 0; --kw) {
          uint32_t bits = swm[warp][kw];
          const int lim = top - 32 * kw;  // keep bits < lim
          if (lim < 32) bits &= (1u << lim) - 1u;
          while (bits) {
            const int bpos = 31 - __clz(bits);
            bits ^= 1u << bpos;
            const int j = lo + 32 * kw + bpos;
            double v[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
            bool contrib = false;
            if (j < my_cnt) contrib = bwd64_pixel(srec[j - lo], px, py, tau, clamp, one_minus_clamp, g0, g1, g2, T, suffix, v);
            if (__any_sync(0xffffffffu, contrib)) {
                const double mine = warp_reduce10_value(v, lane);
                const int idx = reduce10_index(lane);
                if (idx >= 0 && mine != (double)0)
                    atomicAdd(grad2d + (int64_t)sid[j - lo] * kGrad2dStride + idx, mine);
            }
          }
        }
    }
}

// fp32 backward (tile_backward, _tiles.py:59-127): the forward's 8x4-pixel
// warps walk, from the end of the list towards its front, only the splats
// whose cover mask has their bit (a culled splat has alpha == 0 at every
// pixel of the warp, so it contributes nothing), with the forward's exact
// alpha expression (the same bits, so T_i = T_{i+1} / (1 - alpha_i) unwinds
// the forward's chain) and MUFU reciprocals / lg2 in the derivatives:
//   d alpha / d og = alpha / og,  d alpha / d beta = alpha ln(1 - x),
//   d alpha / d m = -alpha beta / (tau (1 - x)),  x = m / tau.
// The 10 per-splat sums (raw moments: sum h d, sum h d d^T with
// h = g_alpha alpha / (1 - x), sum g_alpha alpha, sum g_alpha alpha ln(1 - x),
// sum w g_rgb) are warp reduce-scattered and added with atomics; prim_bwd turns
// them into d/d mean2 = -2 (-beta/tau) P sum h d, d/d P = (-beta/tau) sum h d d^T,
// d/d og = sum / og, d/d beta = sum g_alpha alpha ln(1 - x) (_tiles.py:97-127).
// NP pixels per lane: warp w owns NP of the forward's 8x4 blocks stacked in
// one 8-pixel column (blocks blk0 + 2 r), walks the splats whose cover mask
// has any of their bits, evaluates only the covered blocks' pixels (warp-
// uniform branches) and reduces the NP pixels' sums once: splats are several
// 8x4 blocks wide at the benchmark scales, so the union visits far fewer
// (warp, splat) pairs than the blocks separately, and the reduce + atomic --
// more than half of a visit's instructions -- is paid once per pair.  NP = 2
// (7D 3M view: 5.2 M -> 2.84 M reductions, 843 -> 737 us).  NP = 4 (64
// threads per tile, 128-record batches, the pixels' read-only state in
// shared memory) removes another 20% of the instructions: alone it runs ~8%
// slower (fewer, longer warps), beside other views' kernels (the training
// backend's views in flight) ~2% of the step faster; the caller picks
// (UbsGradBuffers.bwd_pixels_per_lane).


struct BwdPixel {
    float pxf, pyf, T, g0, g1, g2, suffix;
    int cnt;
};

// Deterministic backward (UbsGradBuffers.deterministic): instead of adding
// its warp sums into grad2d with atomics (arrival order), one warp per tile
// writes each splat's tile partial to a slot of its own -- primitive i owns
// slots slot_off[i] .. + tile_count[i], one per tile of its rect in row-major
// order (the order build_tiles visits tiles, raster.py:252-266) -- and
// det_reduce_kernel adds every primitive's partials in slot order: the same
// bits on every run (the reference's guarantee, raster.py:1-8,
// gradients.py:164-173), at the cost of a K x 10 partial buffer.
template <typename T>
struct DetOut {
    const uint32_t *slot_off;  // n + 1: exclusive prefix of tile_count
    const uint64_t *rect;      // UbsPrimBuffers.rect
    T *part;                   // capacity x 10 partial sums (zeroed per view)
    int64_t capacity;          // slots
};

// slot of (primitive with rect q, tile tx, ty): its base + the tile's row-major index in the rect
__device__ __forceinline__ uint32_t det_slot(uint32_t base, uint64_t q, int tx, int ty) {
    const int tx0 = (int)(q & 0xFFFF), ty0 = (int)((q >> 16) & 0xFFFF), tx1 = (int)((q >> 32) & 0xFFFF);
    return base + (uint32_t)((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
}

__device__ __forceinline__ bool bwd_visit(BwdPixel &p, const float g0, const float g1, const float g2, const float4 r0, const float4 r1, uint32_t ra, float tau,
                                          float inv_tau, float clamp, float one_minus_clamp, float (&v)[16]) {
    constexpr float kLn2 = 0.6931471805599453f;
    const float dx = r0.x + p.pxf;  // tile_offset + column in the tile (p.pxf is tile-local)
    const float dy = r0.y + p.pyf;
    const float y0 = fmaf(r1.x, dx, r1.y * dy);
    const float y1 = r1.z * dy;
    const float m = fmaf(y0, y0, y1 * y1);
    if (!(m < tau)) return false;
    const float4 r2 = lds128<32>(ra), r3 = lds128<48>(ra);
    const float omx = fmaf(-m, inv_tau, 1.0f);  // 1 - x
    const float L = lg2_approx(omx);
    float a = ex2_approx(fmaf(r2.x, L, r3.w));  // the forward's alpha
    if (a == 0.0f) return false;
    const bool clamped = a > clamp;
    float om = 1.0f - a;
    if (clamped) {
        a = clamp;
        om = one_minus_clamp;
    }
    const float iom = rcp_approx(om);
    const float ti = p.T * iom;
    const float w = a * ti;
    v[7] += w * g0;
    v[8] += w * g1;
    v[9] += w * g2;
    const float gc = fmaf(g0, r2.y, fmaf(g1, r2.z, g2 * r2.w));
    const float ga = fmaf(gc, ti, -p.suffix * iom);
    p.suffix = fmaf(gc, w, p.suffix);
    p.T = ti;
    if (!clamped) {
        // raw moments; prim_bwd applies the per-splat factors
        // (-2 P, -beta / tau, 1 / og) once per primitive
        const float gaa = ga * a;
        v[5] += gaa;
        v[6] += gaa * (L * kLn2);  // gaa ln(1 - x)
        const float h = gaa * rcp_approx(omx);
        const float hx = h * dx, hy = h * dy;
        v[0] += hx;
        v[1] += hy;
        v[2] += hx * dx;
        v[3] += hx * dy;
        v[4] += hy * dy;
    }
    return true;
}

template <int NP, bool kDet>
__global__ void __launch_bounds__(kTileThreads / NP, NP == 8 ? 24 : 4 * NP)  // 64 registers (NP = 8: 85)
raster_bwd32_kernel(const RasterParams P, const uint32_t *__restrict__ ranges, const uint32_t *__restrict__ ids,
                    const Rec32 *__restrict__ recs, const float *__restrict__ tstop,
                    const int32_t *__restrict__ ncontrib, const float *__restrict__ g_image,
                    float *__restrict__ grad2d, const DetOut<float> det) {
    constexpr int kThreads = kTileThreads / NP;
    // NP = 2: 2 records per thread, half the barriers of 128; NP = 8 (one warp
    // per tile): 64, so ~24 one-warp CTAs fit an SM's shared memory
    constexpr int kBatch = NP == 8 ? 64 : NP >= 4 ? 128 : 256;
    constexpr int kWords = kBatch / 32;
    constexpr int kBlocks = kTileThreads / 32;  // the forward's 8x4 blocks per tile
    // NP = 8: one warp per tile owning all 8 blocks (one reduction per
    // (tile, splat)); kDet (NP = 8 only): tile partials written to per-
    // (primitive, tile) slots instead of atomics
    static_assert(!kDet || NP == 8, "deterministic mode is the one-warp-per-tile layout");
    constexpr bool kOneWarp = NP == 8;
    __shared__ Rec32 srec[kBatch];
    __shared__ uint32_t sid[kBatch];
    __shared__ uint32_t sslot[kDet ? kBatch : 1];
    __shared__ uint32_t swm[kBlocks][kWords];  // [8x4 block][batch word] ballot words
    __shared__ int smax;
    // NP >= 4: each pixel's read-only state (g_image, contributor count) lives
    // in shared memory instead of registers
    constexpr bool kSmemG = NP >= 4;
    __shared__ float4 sg[kSmemG ? NP : 1][kSmemG ? kThreads : 1];
    if (pairs_overflow(P.n_pairs, P.pair_capacity, nullptr)) return;
    const int tile = blockIdx.x;
    const int ty = tile / P.TX, tx = tile - ty * P.TX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int blk0 = (warp & 1) + 2 * NP * (warp >> 1);  // blocks blk0 + 2 r, r < NP (NP = 8: blocks r)
    const uint32_t start = ranges[2 * tile];
    BwdPixel px[NP];
    int my_max = 0;
    if (threadIdx.x == 0) smax = 0;
    __syncthreads();
#pragma unroll
    for (int h = 0; h < NP; ++h) {
        const int blk = kOneWarp ? h : blk0 + 2 * h;
        const int x = tx * kTile + (blk & 1) * 8 + (lane & 7);
        const int y = ty * kTile + (blk >> 1) * 4 + (lane >> 3);
        BwdPixel &p = px[h];
        p.pxf = (float)(x - tx * kTile);
        p.pyf = (float)(y - ty * kTile);
        p.cnt = 0;
        p.T = p.g0 = p.g1 = p.g2 = 0.f;
        if (x < P.W && y < P.H) {
            const int64_t pix = (int64_t)y * P.W + x;
            p.cnt = ncontrib[pix];
            p.T = tstop[pix];
            p.g0 = g_image[3 * pix];
            p.g1 = g_image[3 * pix + 1];
            p.g2 = g_image[3 * pix + 2];
        }
        p.suffix = (p.g0 * (float)P.bg[0] + p.g1 * (float)P.bg[1] + p.g2 * (float)P.bg[2]) * p.T;
        my_max = max(my_max, p.cnt);
        if constexpr (kSmemG) sg[h][threadIdx.x] = make_float4(p.g0, p.g1, p.g2, __int_as_float(p.cnt));
    }
    int warp_cnt = my_max;  // this warp's largest contributor count: splats beyond it are skipped
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) warp_cnt = max(warp_cnt, __shfl_xor_sync(0xffffffffu, warp_cnt, o));
    if (lane == 0) atomicMax(&smax, warp_cnt);
    __syncthreads();
    const int max_cnt = smax;
    const float tau = (float)P.tau, inv_tau = (float)(1.0 / P.tau);
    const float clamp = (float)P.clamp, one_minus_clamp = (float)(1.0 - P.clamp);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(srec);
    // batches aligned from the list front, walked back to front
    for (int lo = ((max_cnt - 1) / kBatch) * kBatch; lo >= 0 && max_cnt > 0; lo -= kBatch) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kBatch / kThreads; ++i) {
            const int jl = i * kThreads + (int)threadIdx.x;
            const int q = lo + jl;
            uint32_t cover = 0;
            if (q < max_cnt) {
                const uint32_t id = ids[start + q];
                const float4 *r = reinterpret_cast<const float4 *>(recs + id);
                float4 *d = reinterpret_cast<float4 *>(srec + jl);
                sid[jl] = id;
                if constexpr (kDet) sslot[jl] = det_slot(det.slot_off[id], det.rect[id], tx, ty);
                const float4 r0 = __ldg(r), r1 = __ldg(r + 1);
                const float2 o = tile_offset(r0, tx, ty);
                d[0] = make_float4(o.x, o.y, r0.z, r0.w);
                d[1] = r1;
                d[2] = __ldg(r + 2);
                d[3] = __ldg(r + 3);
                cover = warp_cover_mask(o.x, o.y, r1);
            }
#pragma unroll
            for (int w = 0; w < kBlocks; ++w) {
                const uint32_t word = __ballot_sync(0xffffffffu, (cover >> w) & 1u);
                if (lane == 0) swm[w][jl >> 5] = word;
            }
        }
        __syncthreads();
        const int top = min(kBatch, warp_cnt - lo);  // splats [lo, lo + top) concern this warp
        for (int k = (top - 1) >> 5; k >= 0; --k) {
            uint32_t wr[NP], bits = 0;
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                wr[h] = swm[kOneWarp ? h : blk0 + 2 * h][k];
                bits |= wr[h];
            }
            const int lim = top - 32 * k;  // keep bits < lim
            if (lim < 32) bits &= (1u << lim) - 1u;
            while (bits) {
                const uint32_t b = msb_pos(bits), bm = bit_at(b);
                bits ^= bm;
                const int jj = 32 * k + (int)b;  // index inside the batch
                const uint32_t ra = sbase + (uint32_t)jj * (uint32_t)sizeof(Rec32);
                const float4 r0 = lds128<0>(ra), r1 = lds128<16>(ra);
                float v[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
                bool contrib = false;
#pragma unroll
                for (int h = 0; h < NP; ++h) {
                    if (!(wr[h] & bm)) continue;
                    if constexpr (kSmemG) {
                        const float4 gq = sg[h][threadIdx.x];
                        if (lo + jj < __float_as_int(gq.w))
                            contrib |= bwd_visit(px[h], gq.x, gq.y, gq.z, r0, r1, ra, tau, inv_tau, clamp,
                                                 one_minus_clamp, v);
                    } else if (lo + jj < px[h].cnt) {
                        contrib |= bwd_visit(px[h], px[h].g0, px[h].g1, px[h].g2, r0, r1, ra, tau, inv_tau, clamp,
                                             one_minus_clamp, v);
                    }
                }
                if (__any_sync(0xffffffffu, contrib)) {
                    const float mine = warp_reduce10_value(v, lane);
                    const int idx = reduce10_index(lane);
                    if (idx >= 0 && mine != 0.0f) {
                        if constexpr (kDet) {
                            const uint32_t sl = sslot[jj];
                            if ((int64_t)sl < det.capacity) det.part[(int64_t)sl * 10 + idx] = mine;
                        } else if (UBS_GUARD(jj >= 0 && jj < kBatch && idx >= 0 && idx < 10, kChkGrad)) {
                            atomicAdd(grad2d + (int64_t)sid[jj] * kGrad2dStride + idx, mine);
                        }
                    }
                }
            }
        }
    }
}

// Deterministic mode, fp64 (tile_backward in the reference's operation
// order): one warp per tile, 8 pixels per lane (pixel lane + 32 h of the
// tile, row-major), the list walked back to front in batches of 32 staged
// records; each splat's per-lane sums over the 8 pixels are warp-reduced once
// and written to the splat's (primitive, tile) slot.
__global__ void __launch_bounds__(32)
raster_bwd64_det_kernel(const RasterParams P, const uint32_t *__restrict__ ranges, const uint32_t *__restrict__ ids,
                        const Rec64 *__restrict__ recs, const double *__restrict__ tstop,
                        const int32_t *__restrict__ ncontrib, const double *__restrict__ g_image,
                        const DetOut<double> det) {
    __shared__ Rec64 srec[32];
    __shared__ uint32_t sslot[32];
    __shared__ double sg[8][3][32];
    __shared__ int scnt[8][32];
    if (pairs_overflow(P.n_pairs, P.pair_capacity, nullptr)) return;
    const int tile = blockIdx.x;
    const int ty = tile / P.TX, tx = tile - ty * P.TX;
    const int lane = threadIdx.x;
    const uint32_t start = ranges[2 * tile];
    double T[8], suffix[8];
    int my_max = 0;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        const int p = lane + 32 * h;
        const int x = tx * kTile + (p & 15), y = ty * kTile + (p >> 4);
        int cnt = 0;
        double t = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
        if (x < P.W && y < P.H) {
            const int64_t pix = (int64_t)y * P.W + x;
            cnt = ncontrib[pix];
            t = tstop[pix];
            g0 = g_image[3 * pix];
            g1 = g_image[3 * pix + 1];
            g2 = g_image[3 * pix + 2];
        }
        T[h] = t;
        suffix[h] = (g0 * P.bg[0] + g1 * P.bg[1] + g2 * P.bg[2]) * t;
        sg[h][0][lane] = g0;
        sg[h][1][lane] = g1;
        sg[h][2][lane] = g2;
        scnt[h][lane] = cnt;
        my_max = max(my_max, cnt);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
    const double tau = P.tau, clamp = P.clamp, one_minus_clamp = 1.0 - P.clamp;
    for (int lo = ((my_max - 1) / 32) * 32; lo >= 0 && my_max > 0; lo -= 32) {
        __syncwarp();
        const int q = lo + lane;
        if (q < my_max) {
            const uint32_t id = ids[start + q];
            srec[lane] = recs[id];
            sslot[lane] = det_slot(det.slot_off[id], det.rect[id], tx, ty);
        }
        __syncwarp();
        for (int jj = min(32, my_max - lo) - 1; jj >= 0; --jj) {
            double v[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
            bool contrib = false;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const int p = lane + 32 * h;
                if (lo + jj < scnt[h][lane])
                    contrib |= bwd64_pixel(srec[jj], tx * kTile + (p & 15), ty * kTile + (p >> 4), tau, clamp,
                                           one_minus_clamp, sg[h][0][lane], sg[h][1][lane], sg[h][2][lane], T[h],
                                           suffix[h], v);
            }
            if (__any_sync(0xffffffffu, contrib)) {
                const double mine = warp_reduce10_value(v, lane);
                const int idx = reduce10_index(lane);
                if (idx >= 0 && mine != 0.0) {
                    const uint32_t sl = sslot[jj];
                    if ((int64_t)sl < det.capacity) det.part[(int64_t)sl * 10 + idx] = mine;
                }
            }
        }
    }
}

// Deterministic mode: each primitive adds its (primitive, tile) partials in
// slot order (its rect's tiles, row-major) into grad2d.
template <typename T>
__global__ void det_reduce_kernel(const uint32_t *__restrict__ slot_off, const uint32_t *__restrict__ tile_count,
                                  const T *__restrict__ part, int64_t n, int64_t capacity, T *__restrict__ grad2d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t cnt = tile_count[i];
    if (cnt == 0) return;
    const int64_t base = slot_off[i];
    if (base + cnt > capacity) return;
    T acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t t = 0; t < cnt; ++t) {
        const T *q = part + (base + t) * 10;
#pragma unroll
        for (int c = 0; c < 10; ++c) acc[c] += q[c];
    }
    T *g = grad2d + i * kGrad2dStride;
#pragma unroll
    for (int c = 0; c < 10; ++c)
        if (acc[c] != (T)0) g[c] += acc[c];
}

// Packed fp32x2 backward: raster_bwd32_kernel's layouts with NP = 4 / 8
// pixels per lane evaluated as NP / 2 vertical pixel pairs (h, h + 1: the same
// column, 4 rows apart) with FADD2 / FMUL2 / FFMA2 on the pair.  Every pixel
// runs the scalar kernel's alpha expression bit for bit (so T_i = T_{i+1} /
// (1 - alpha_i) unwinds the forward's chain exactly); the per-splat sums are
// accumulated as pairs and folded once before the warp reduction, so they
// differ from the scalar kernel's only in float summation order.  A pair with
// a pixel in the clamp band takes the scalar bwd_visit (rare).
// 11 CTAs per SM = 80 registers for the four-pixel layout: at the 64 of 16 CTAs
// the kernel spilled its cover words and counts and re-derived its constants
// every visit (323 -> 261 instructions per visited splat; 7D 3M 1080p view
// 0.99 -> 0.77 ms, training step 48 -> 54 it/s)
#ifndef UBS_BWD4_MIN_CTAS
#define UBS_BWD4_MIN_CTAS 11
#endif
template <int NP>
__global__ void __launch_bounds__(kTileThreads / NP, NP == 8 ? 16 : UBS_BWD4_MIN_CTAS)
raster_bwd32x2_kernel(const RasterParams P, const uint32_t *__restrict__ ranges, const uint32_t *__restrict__ ids,
                      const Rec32 *__restrict__ recs, const float *__restrict__ tstop,
                      const int32_t *__restrict__ ncontrib, const float *__restrict__ g_image,
                      float *__restrict__ grad2d) {
    static_assert(NP == 4 || NP == 8, "pairs of pixels per lane");
    constexpr int NQ = NP / 2;                   // pixel pairs per lane
    constexpr int kThreads = kTileThreads / NP;  // 64 (NP = 4) or 32 (NP = 8)
    constexpr int kBatch = NP == 8 ? 64 : 128;
    constexpr int kWords = kBatch / 32;
    constexpr int kBlocks = kTileThreads / 32;
    constexpr bool kOneWarp = NP == 8;
    __shared__ Rec32 srec[kBatch];
    __shared__ uint32_t sid[kBatch];
    __shared__ uint32_t swm[kBlocks][kWords];
    __shared__ int smax;
    // per pair: (g0a, g0b, g1a, g1b), (g2a, g2b, -, -): adjacent pair halves for FFMA2
    __shared__ float4 sgp[NQ][2][kThreads];
    if (pairs_overflow(P.n_pairs, P.pair_capacity, nullptr)) return;
    const int tile = blockIdx.x;
    const int ty = tile / P.TX, tx = tile - ty * P.TX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int blk0 = (warp & 1) + 2 * NP * (warp >> 1);
    const int ridx = reduce10_index(lane);  // this lane's reduced component (-1: none)
    const uint32_t start = ranges[2 * tile];
    float T[NP], S[NP], pyf[NP];  // S: the suffix sum of tile_backward (_tiles.py:97-127)
    int cnt[NP];
    int my_max = 0;
    if (threadIdx.x == 0) smax = 0;
    __syncthreads();
    // pixel h of the lane lies in 8x4 block blk(h); pixels 2p and 2p + 1 are
    // vertical neighbours (the same column, 4 rows apart): NP = 4: blocks
    // blk0 + 2h; NP = 8 (the whole tile): block column h >> 2, block row h & 3
    auto blk_of = [&](int h) { return kOneWarp ? (h >> 2) + 2 * (h & 3) : blk0 + 2 * h; };
#pragma unroll
    for (int h = 0; h < NP; ++h) {
        const int blk = blk_of(h);
        const int x = tx * kTile + (blk & 1) * 8 + (lane & 7);
        const int y = ty * kTile + (blk >> 1) * 4 + (lane >> 3);
        pyf[h] = (float)(y - ty * kTile);
        cnt[h] = 0;
        T[h] = 0.f;
        float g0 = 0.f, g1 = 0.f, g2 = 0.f;
        if (x < P.W && y < P.H) {
            const int64_t pix = (int64_t)y * P.W + x;
            cnt[h] = ncontrib[pix];
            T[h] = tstop[pix];
            g0 = g_image[3 * pix];
            g1 = g_image[3 * pix + 1];
            g2 = g_image[3 * pix + 2];
        }
        S[h] = (g0 * (float)P.bg[0] + g1 * (float)P.bg[1] + g2 * (float)P.bg[2]) * T[h];
        my_max = max(my_max, cnt[h]);
        float *gp = reinterpret_cast<float *>(&sgp[h >> 1][0][threadIdx.x]);
        float *gq = reinterpret_cast<float *>(&sgp[h >> 1][1][threadIdx.x]);
        gp[h & 1] = g0;
        gp[2 + (h & 1)] = g1;
        gq[h & 1] = g2;
    }
    int warp_cnt = my_max;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) warp_cnt = max(warp_cnt, __shfl_xor_sync(0xffffffffu, warp_cnt, o));
    if (lane == 0) atomicMax(&smax, warp_cnt);
    __syncthreads();
    const int max_cnt = smax;
    const float tau = P.tau_f, inv_tau = P.inv_tau_f;
    const float clamp = P.clamp_f, one_minus_clamp = P.omc_f;
    const float og_hi = clamp / (1.0f + 1.0e-4f);
    constexpr float kLn2 = 0.6931471805599453f;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(srec);
    for (int lo = ((max_cnt - 1) / kBatch) * kBatch; lo >= 0 && max_cnt > 0; lo -= kBatch) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kBatch / kThreads; ++i) {
            const int jl = i * kThreads + (int)threadIdx.x;
            const int q = lo + jl;
            uint32_t cover = 0;
            if (q < max_cnt && UBS_GUARD((int64_t)start + q < P.pair_capacity, kChkPair)) {
                const uint32_t id = ids[start + q];
                const float4 *r = reinterpret_cast<const float4 *>(recs + id);
                float4 *d = reinterpret_cast<float4 *>(srec + jl);
                sid[jl] = id;
                const float4 r0 = __ldg(r), r1 = __ldg(r + 1);
                const float2 o = tile_offset(r0, tx, ty);
                d[0] = make_float4(o.x, o.y, r0.z, r0.w);
                d[1] = r1;
                d[2] = __ldg(r + 2);
                d[3] = __ldg(r + 3);
                cover = warp_cover_mask(o.x, o.y, r1);
            }
#pragma unroll
            for (int w = 0; w < kBlocks; ++w) {
                const uint32_t word = __ballot_sync(0xffffffffu, (cover >> w) & 1u);
                if (lane == 0) swm[w][jl >> 5] = word;
            }
        }
        __syncthreads();
        const int top = min(kBatch, warp_cnt - lo);
        for (int k = (top - 1) >> 5; k >= 0; --k) {
            uint32_t wr[NP], bits = 0;
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                wr[h] = swm[blk_of(h)][k];
                bits |= wr[h];
            }
            const int lim = top - 32 * k;
            if (lim < 32) bits &= (1u << lim) - 1u;
            while (bits) {
                const uint32_t b = msb_pos(bits), bm = bit_at(b);
                bits ^= bm;
                const int jj = 32 * k + (int)b;
                const int j = lo + jj;  // list position
                const uint32_t ra = sbase + (uint32_t)jj * (uint32_t)sizeof(Rec32);
                const float2 r0 = lds64<0>(ra);  // tile offset (xa, ya)
                const float4 r1 = lds128<16>(ra);
                // Per-splat sums V of the lane's pixel pairs.  The first pair that
                // has a pixel in support anywhere in the warp writes V, later pairs
                // add to it: no per-visit zeroing.  In a writing pair, lanes with no
                // pixel in support run the body on alpha = 0, which writes exact
                // zeros and leaves T and S bit-for-bit unchanged (1 - 0 = 1, whose
                // reciprocal is exactly 1); in an adding pair they skip.
                f32x2 V[10];
                auto pair = [&](auto p_, auto init_) -> bool {
                    constexpr int p = decltype(p_)::value;
                    constexpr bool init = decltype(init_)::value;
                    const int h0 = 2 * p, h1 = 2 * p + 1;
                    const bool e0 = (wr[h0] & bm) && j < cnt[h0], e1 = (wr[h1] & bm) && j < cnt[h1];
                    if (init ? !__any_sync(0xffffffffu, e0 || e1) : !(e0 || e1)) return false;
                    const float dx = r0.x + (float)((blk_of(h0) & 1) * 8 + (lane & 7));  // the pair's column
                    const f32x2 dy = add2(dup2(r0.y), pk2(pyf[h0], pyf[h1]));
                    const f32x2 y0 = fma2(dup2(r1.x), dup2(dx), mul2(dup2(r1.y), dy));
                    const f32x2 y1 = mul2(dup2(r1.z), dy);
                    const float2 m = up2(fma2(y0, y0, mul2(y1, y1)));
                    const bool s0 = e0 && m.x < tau, s1 = e1 && m.y < tau;
                    if (init ? !__any_sync(0xffffffffu, s0 || s1) : !(s0 || s1)) return false;
                    const float4 r2 = lds128<32>(ra), r3 = lds128<48>(ra);
                    const float2 omx = up2(fma2(pk2(m.x, m.y), dup2(-inv_tau), dup2(1.0f)));
                    // pixels not in support take omx = 1: lg2 = 0, 1 / omx = 1 (finite), alpha = 0 below
                    const float ox0 = s0 ? omx.x : 1.0f, ox1 = s1 ? omx.y : 1.0f;
                    const f32x2 L = pk2(lg2_approx(ox0), lg2_approx(ox1));
                    const float2 ag = up2(fma2(dup2(r2.x), L, dup2(r3.w)));
                    float a0 = s0 ? ex2_approx(ag.x) : 0.0f, a1 = s1 ? ex2_approx(ag.y) : 0.0f;
                    float2 om = up2(sub2(dup2(1.0f), pk2(a0, a1)));
                    float am0 = a0, am1 = a1;  // alpha in the raw moments: 0 for a clamped pixel
                    // alpha <= og (1 + 1e-5): a splat with og below clamp / (1 + 1e-4) is never
                    // clamped -- a warp-uniform test ahead of the per-pixel one
                    if (r3.y > og_hi && (a0 > clamp || a1 > clamp)) {
                        // clamp band (rare): alpha = clamp, 1 - alpha = 1 - clamp, and no
                        // moments (tile_backward skips d/d m, og, beta at the clamp)
                        if (a0 > clamp) {
                            a0 = clamp;
                            om.x = one_minus_clamp;
                            am0 = 0.0f;
                        }
                        if (a1 > clamp) {
                            a1 = clamp;
                            om.y = one_minus_clamp;
                            am1 = 0.0f;
                        }
                    }
                    const f32x2 a2 = pk2(a0, a1);
                    const f32x2 iom = pk2(rcp_approx(om.x), rcp_approx(om.y));
                    const f32x2 ti = mul2(pk2(T[h0], T[h1]), iom);  // T_i rebuilt from T_{i+1} (the forward's alpha)
                    const f32x2 w = mul2(a2, ti);
                    const float4 gA = sgp[p][0][threadIdx.x], gB = sgp[p][1][threadIdx.x];
                    const f32x2 g0 = pk2(gA.x, gA.y), g1 = pk2(gA.z, gA.w), g2 = pk2(gB.x, gB.y);
                    const f32x2 gc = fma2(g0, dup2(r2.y), fma2(g1, dup2(r2.z), mul2(g2, dup2(r2.w))));
                    const f32x2 Sp = pk2(S[h0], S[h1]);
                    // ga = gc T_i - suffix / (1 - a)  (fmaf(gc, ti, -suffix * iom) per pixel)
                    const f32x2 ga = fma2(gc, ti, sub2(0ull, mul2(Sp, iom)));
                    const float2 Sn = up2(fma2(gc, w, Sp));
                    const float2 Tn = up2(ti);
                    S[h0] = Sn.x;
                    S[h1] = Sn.y;
                    T[h0] = Tn.x;
                    T[h1] = Tn.y;
                    // raw moments (not clamped here); alpha = 0 pixels add exact zeros
                    const f32x2 gaa = mul2(ga, pk2(am0, am1));
                    const f32x2 gln = mul2(L, dup2(kLn2));  // ln(1 - x)
                    const f32x2 hh = mul2(gaa, pk2(rcp_approx(ox0), rcp_approx(ox1)));
                    const f32x2 hx = mul2(hh, dup2(dx)), hy = mul2(hh, dy);
                    if constexpr (init) {
                        V[7] = mul2(w, g0);
                        V[8] = mul2(w, g1);
                        V[9] = mul2(w, g2);
                        V[5] = gaa;
                        V[6] = mul2(gaa, gln);
                        V[0] = hx;
                        V[1] = hy;
                        V[2] = mul2(hx, dup2(dx));
                        V[3] = mul2(hx, dy);
                        V[4] = mul2(hy, dy);
                    } else {
                        V[7] = fma2(w, g0, V[7]);
                        V[8] = fma2(w, g1, V[8]);
                        V[9] = fma2(w, g2, V[9]);
                        V[5] = add2(V[5], gaa);
                        V[6] = fma2(gaa, gln, V[6]);
                        V[0] = add2(V[0], hx);
                        V[1] = add2(V[1], hy);
                        V[2] = fma2(hx, dup2(dx), V[2]);
                        V[3] = fma2(hx, dy, V[3]);
                        V[4] = fma2(hy, dy, V[4]);
                    }
                    return true;
                };
                using Yes = std::integral_constant<bool, true>;
                using No = std::integral_constant<bool, false>;
                // any_in: warp-uniform (the writing pair's vote), the reduction's gate
                bool any_in = false;
                bool both = false;
                if constexpr (NQ == 2) {
                    // the splat meets both 8x8 halves of the warp: the two pixel pairs
                    // are evaluated together, without per-pair branches, so their
                    // lg2 -> ex2 -> rcp chains interleave (pixels not in support run
                    // on alpha = 0: exact zeros, T and S unchanged bit for bit)
                    bool e[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) e[h] = (wr[h] & bm) && j < cnt[h];
                    both = __any_sync(0xffffffffu, e[0] || e[1]) && __any_sync(0xffffffffu, e[2] || e[3]);
                    if (both) {
                        const float dx = r0.x + (float)((blk_of(0) & 1) * 8 + (lane & 7));  // both pairs' column
                        float2 m[2];
                        f32x2 dyp[2];
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            dyp[p] = add2(dup2(r0.y), pk2(pyf[2 * p], pyf[2 * p + 1]));
                            const f32x2 y0 = fma2(dup2(r1.x), dup2(dx), mul2(dup2(r1.y), dyp[p]));
                            const f32x2 y1 = mul2(dup2(r1.z), dyp[p]);
                            m[p] = up2(fma2(y0, y0, mul2(y1, y1)));
                        }
                        bool sp[4];
                        sp[0] = e[0] && m[0].x < tau;
                        sp[1] = e[1] && m[0].y < tau;
                        sp[2] = e[2] && m[1].x < tau;
                        sp[3] = e[3] && m[1].y < tau;
                        any_in = __any_sync(0xffffffffu, sp[0] || sp[1] || sp[2] || sp[3]);
                        if (any_in) {
                            const float4 r2 = lds128<32>(ra), r3 = lds128<48>(ra);
                            float ox[4], al[4], am[4], omv[4];
                            f32x2 L[2];
#pragma unroll
                            for (int p = 0; p < 2; ++p) {
                                const float2 omx = up2(fma2(pk2(m[p].x, m[p].y), dup2(-inv_tau), dup2(1.0f)));
                                ox[2 * p] = sp[2 * p] ? omx.x : 1.0f;
                                ox[2 * p + 1] = sp[2 * p + 1] ? omx.y : 1.0f;
                                L[p] = pk2(lg2_approx(ox[2 * p]), lg2_approx(ox[2 * p + 1]));
                                const float2 ag = up2(fma2(dup2(r2.x), L[p], dup2(r3.w)));
                                al[2 * p] = sp[2 * p] ? ex2_approx(ag.x) : 0.0f;
                                al[2 * p + 1] = sp[2 * p + 1] ? ex2_approx(ag.y) : 0.0f;
                                const float2 o2 = up2(sub2(dup2(1.0f), pk2(al[2 * p], al[2 * p + 1])));
                                omv[2 * p] = o2.x;
                                omv[2 * p + 1] = o2.y;
                            }
#pragma unroll
                            for (int h = 0; h < 4; ++h) am[h] = al[h];  // 0 when clamped
                            if (r3.y > og_hi && (al[0] > clamp || al[1] > clamp || al[2] > clamp || al[3] > clamp)) {
#pragma unroll
                                for (int h = 0; h < 4; ++h)
                                    if (al[h] > clamp) {  // clamp band (rare)
                                        al[h] = clamp;
                                        omv[h] = one_minus_clamp;
                                        am[h] = 0.0f;
                                    }
                            }
#pragma unroll
                            for (int p = 0; p < 2; ++p) {
                                const int h0 = 2 * p, h1 = 2 * p + 1;
                                const f32x2 a2 = pk2(al[h0], al[h1]);
                                const f32x2 iom = pk2(rcp_approx(omv[h0]), rcp_approx(omv[h1]));
                                const f32x2 ti = mul2(pk2(T[h0], T[h1]), iom);
                                const f32x2 w = mul2(a2, ti);
                                const float4 gA = sgp[p][0][threadIdx.x], gB = sgp[p][1][threadIdx.x];
                                const f32x2 g0 = pk2(gA.x, gA.y), g1 = pk2(gA.z, gA.w), g2 = pk2(gB.x, gB.y);
                                const f32x2 gc = fma2(g0, dup2(r2.y), fma2(g1, dup2(r2.z), mul2(g2, dup2(r2.w))));
                                const f32x2 Sp = pk2(S[h0], S[h1]);
                                const f32x2 ga = fma2(gc, ti, sub2(0ull, mul2(Sp, iom)));
                                const float2 Sn = up2(fma2(gc, w, Sp));
                                const float2 Tn = up2(ti);
                                S[h0] = Sn.x;
                                S[h1] = Sn.y;
                                T[h0] = Tn.x;
                                T[h1] = Tn.y;
                                const f32x2 gaa = mul2(ga, pk2(am[h0], am[h1]));
                                const f32x2 gln = mul2(L[p], dup2(kLn2));
                                const f32x2 hh = mul2(gaa, pk2(rcp_approx(ox[h0]), rcp_approx(ox[h1])));
                                const f32x2 hx = mul2(hh, dup2(dx)), hy = mul2(hh, dyp[p]);
                                if (p == 0) {
                                    V[7] = mul2(w, g0);
                                    V[8] = mul2(w, g1);
                                    V[9] = mul2(w, g2);
                                    V[5] = gaa;
                                    V[6] = mul2(gaa, gln);
                                    V[0] = hx;
                                    V[1] = hy;
                                    V[2] = mul2(hx, dup2(dx));
                                    V[3] = mul2(hx, dyp[p]);
                                    V[4] = mul2(hy, dyp[p]);
                                } else {
                                    V[7] = fma2(w, g0, V[7]);
                                    V[8] = fma2(w, g1, V[8]);
                                    V[9] = fma2(w, g2, V[9]);
                                    V[5] = add2(V[5], gaa);
                                    V[6] = fma2(gaa, gln, V[6]);
                                    V[0] = add2(V[0], hx);
                                    V[1] = add2(V[1], hy);
                                    V[2] = fma2(hx, dup2(dx), V[2]);
                                    V[3] = fma2(hx, dyp[p], V[3]);
                                    V[4] = fma2(hy, dyp[p], V[4]);
                                }
                            }
                        }
                    }
                }
                if (!both) {  // one half (or none): the pair chain, pair by pair
                    auto step = [&](auto p_) {
                        if (any_in) pair(p_, No{});
                        else any_in = pair(p_, Yes{});
                    };
                    step(std::integral_constant<int, 0>{});
                    step(std::integral_constant<int, 1>{});
                    if constexpr (NQ > 2) {
                        step(std::integral_constant<int, 2>{});
                        step(std::integral_constant<int, 3>{});
                    }
                }
                if (any_in) {
                    float v[16];
#pragma unroll
                    for (int c = 0; c < 10; ++c) {
                        const float2 t = up2(V[c]);
                        v[c] = t.x + t.y;
                    }
                    const float mine = warp_reduce10_value(v, lane);
                    if (ridx >= 0 && mine != 0.0f &&
                        UBS_GUARD(jj >= 0 && jj < kBatch && ridx < 10, kChkGrad))
                        atomicAdd(grad2d + (int64_t)sid[jj] * kGrad2dStride + ridx, mine);
                }
            }
        }
    }
}

}  // namespace ubs

using namespace ubs;

extern "C" int ubs_raster_forward(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                                  const UbsImageBuffers *ib, ubs_stream_t stream) {
    if (!v || !pb || !bb || !ib || !ib->image || !ib->alpha_sum || !ib->t_stop || !ib->n_contrib ||
        !ib->hit_clamp || !ib->visits)
        return UBS_E_ARGS;
    const RasterParams P = make_params(*v, *pb, *bb);
    const int n_tiles = P.TX * ((P.H + kTile - 1) / kTile);
    cudaStream_t s = (cudaStream_t)stream;
    if (ib->raster_f64) {
        if (!pb->rec64) return UBS_E_ARGS;
        raster_fwd64_kernel<<<n_tiles, kTileThreads, 0, s>>>(
            P, bb->tile_ranges, bb->tile_ids, (const Rec64 *)pb->rec64, (double *)ib->image, (double *)ib->alpha_sum,
            (double *)ib->t_stop, ib->n_contrib, ib->hit_clamp, ib->visits);
    } else {
        if (!pb->rec32 || !pb->rec64 || !ib->fix_list || !ib->fix_count) return UBS_E_ARGS;
        if (ib->raster_scalar)
            raster_fwd32_kernel<<<n_tiles, kTileThreads, 0, s>>>(
                P, bb->tile_ranges, bb->tile_ids, (const Rec32 *)pb->rec32, (float *)ib->image, (float *)ib->alpha_sum,
                (float *)ib->t_stop, ib->n_contrib, ib->hit_clamp, ib->visits, ib->fix_list, ib->fix_count);
        else
            raster_fwd32x2_kernel<<<n_tiles, kX2Threads, 0, s>>>(
                P, bb->tile_ranges, bb->tile_ids, (const Rec32 *)pb->rec32, (float *)ib->image, (float *)ib->alpha_sum,
                (float *)ib->t_stop, ib->n_contrib, ib->hit_clamp, ib->visits, ib->fix_list, ib->fix_count);
    }
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" int ubs_raster_fixup(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                                const UbsImageBuffers *ib, ubs_stream_t stream) {
    if (!v || !pb || !bb || !ib) return UBS_E_ARGS;
    if (ib->raster_f64) return UBS_OK;  // nothing to fix: the fp64 raster is the reference arithmetic
    if (!pb->rec64 || !ib->fix_list || !ib->fix_count) return UBS_E_ARGS;
    const RasterParams P = make_params(*v, *pb, *bb);
    // one pass over the device-counted list, grid-stride over ~4 warps per SM:
    // the fix-up's cost is its tail, so it keeps a small footprint beside the
    // other frames' rasters (148 x 128 threads: 2008 vs 1997 fps for 592 x 256)
    raster_fixup_kernel<<<148 * UBS_FIX_CTAS_PER_SM, kFixThreads, 0, (cudaStream_t)stream>>>(
        P, bb->tile_ranges, bb->tile_ids, (const Rec64 *)pb->rec64, ib->fix_list, ib->fix_count, (float *)ib->image,
        (float *)ib->alpha_sum, (float *)ib->t_stop, ib->n_contrib, ib->hit_clamp, ib->visits);
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" int ubs_raster_backward(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                                   const UbsImageBuffers *ib, const UbsGradBuffers *gb, ubs_stream_t stream) {
    if (!v || !pb || !bb || !ib || !gb || !gb->g_image || !gb->grad2d) return UBS_E_ARGS;
    if ((gb->grad2d_f64 != 0) != (ib->raster_f64 != 0)) return UBS_E_ARGS;
    if (gb->bwd_pixels_per_lane != 0 && gb->bwd_pixels_per_lane != 2 && gb->bwd_pixels_per_lane != 4 &&
        gb->bwd_pixels_per_lane != 8)
        return UBS_E_ARGS;
    const RasterParams P = make_params(*v, *pb, *bb);
    const int n_tiles = P.TX * ((P.H + kTile - 1) / kTile);
    cudaStream_t s = (cudaStream_t)stream;
    if (gb->deterministic) {
        if (!gb->det_slot_off || !gb->det_partials || !gb->det_temp || !pb->rect || !pb->tile_count || v->n < 1)
            return v->n == 0 ? UBS_OK : UBS_E_ARGS;
        size_t need = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, need, pb->tile_count, gb->det_slot_off, (int)v->n + 1);
        if (need > gb->det_temp_bytes) return UBS_E_CAPACITY;
        // tile_count[n] is not an element: scan n, then slot_off[n] = K by the reduce's bound check
        if (cub::DeviceScan::ExclusiveSum(gb->det_temp, need, pb->tile_count, gb->det_slot_off, (int)v->n, s) !=
            cudaSuccess)
            return UBS_E_CUDA;
        const size_t elem = ib->raster_f64 ? 8 : 4;
        if (cudaMemsetAsync(gb->det_partials, 0, (size_t)gb->det_capacity * 10 * elem, s) != cudaSuccess)
            return UBS_E_CUDA;
        const unsigned rb = (unsigned)((v->n + 255) / 256);
        if (ib->raster_f64) {
            const DetOut<double> det{gb->det_slot_off, pb->rect, (double *)gb->det_partials, gb->det_capacity};
            raster_bwd64_det_kernel<<<n_tiles, 32, 0, s>>>(P, bb->tile_ranges, bb->tile_ids, (const Rec64 *)pb->rec64,
                                                          (const double *)ib->t_stop, ib->n_contrib,
                                                          (const double *)gb->g_image, det);
            det_reduce_kernel<double><<<rb, 256, 0, s>>>(gb->det_slot_off, pb->tile_count, det.part, v->n,
                                                         det.capacity, (double *)gb->grad2d);
        } else {
            const DetOut<float> det{gb->det_slot_off, pb->rect, (float *)gb->det_partials, gb->det_capacity};
            raster_bwd32_kernel<8, true><<<n_tiles, kTileThreads / 8, 0, s>>>(
                P, bb->tile_ranges, bb->tile_ids, (const Rec32 *)pb->rec32, (const float *)ib->t_stop, ib->n_contrib,
                (const float *)gb->g_image, (float *)gb->grad2d, det);
            det_reduce_kernel<float><<<rb, 256, 0, s>>>(gb->det_slot_off, pb->tile_count, det.part, v->n,
                                                        det.capacity, (float *)gb->grad2d);
        }
        UBS_CUDA_CHECK();
        return UBS_OK;
    }
    const DetOut<float> none{nullptr, nullptr, nullptr, 0};
    if (ib->raster_f64) {
        raster_bwd64_kernel<<<n_tiles, kTileThreads, 0, s>>>(
            P, bb->tile_ranges, bb->tile_ids, (const Rec64 *)pb->rec64, (const double *)ib->t_stop, ib->n_contrib,
            (const double *)gb->g_image, (double *)gb->grad2d);
    } else {
        // 0 / 4: packed pairs, four pixels per lane (the default: ~0.71 ms against
        // ~0.86 for two scalar pixels per lane on a 7D 3M 1080p view); 2 / 8 and
        // raster_scalar: one pixel per lane (the packed one-warp 8-pixel layout: 0.88 ms at 121
        // registers, 16 warps per SM)
        const int ppl = gb->bwd_pixels_per_lane ? gb->bwd_pixels_per_lane : 4;
        if (ppl == 4 && !ib->raster_scalar)
            raster_bwd32x2_kernel<4><<<n_tiles, kTileThreads / 4, 0, s>>>(
                P, bb->tile_ranges, bb->tile_ids, (const Rec32 *)pb->rec32, (const float *)ib->t_stop, ib->n_contrib,
                (const float *)gb->g_image, (float *)gb->grad2d);
        else if (ppl == 8)
            raster_bwd32_kernel<8, false><<<n_tiles, kTileThreads / 8, 0, s>>>(
                P, bb->tile_ranges, bb->tile_ids, (const Rec32 *)pb->rec32, (const float *)ib->t_stop, ib->n_contrib,
                (const float *)gb->g_image, (float *)gb->grad2d, none);
        else if (ppl == 4)
            raster_bwd32_kernel<4, false><<<n_tiles, kTileThreads / 4, 0, s>>>(
                P, bb->tile_ranges, bb->tile_ids, (const Rec32 *)pb->rec32, (const float *)ib->t_stop, ib->n_contrib,
                (const float *)gb->g_image, (float *)gb->grad2d, none);
        else
            raster_bwd32_kernel<2, false><<<n_tiles, kTileThreads / 2, 0, s>>>(
                P, bb->tile_ranges, bb->tile_ids, (const Rec32 *)pb->rec32, (const float *)ib->t_stop, ib->n_contrib,
                (const float *)gb->g_image, (float *)gb->grad2d, none);
    }
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" size_t ubs_det_temp_bytes(int64_t n) {
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (int)(n > 0 ? n : 1) + 1);
    return need;
}

UBS_CHECKED_ACCESSOR(raster)
