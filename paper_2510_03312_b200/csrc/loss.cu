// Loss image gradient: L1 + (1 - SSIM) and its exact adjoint.
//
// Reference: gradients.py:110-116 (g_image = scale * ((1-l) sign(diff)/size
// - l * g_ssim)), metrics.py:35-114 (separable 11-tap sigma 1.5 Gaussian
// window with reflect padding folded into a banded operator; the adjoint is
// the transposed operator).
//
// Images with both sides >= 12 take the two tiled kernels below; smaller
// ones four separable global passes: horizontal blur of (a, b, a^2, b^2, ab),
// vertical blur + pointwise SSIM map and its pointwise adjoint, vertical
// adjoint, horizontal adjoint + combine.  The adjoint of the reflect-folded blur is a
// gather: output j collects from every (row, tap) whose reflected source is j.
#include <cuda_runtime.h>

#include "ubs_common.cuh"
#include "f32x2.cuh"

namespace ubs {

struct BlurTaps {
    double k[11];
};

__device__ __forceinline__ int reflect_idx(int i, int n) {
    // metrics.py:43-46: period 2n-2, no edge duplication
    const int period = n > 1 ? 2 * n - 2 : 1;
    i = abs(i) % period;
    return i >= n ? period - i : i;
}

// forward blur along an axis of length n (interior points skip the reflect)
template <typename T, typename F>
__device__ __forceinline__ T blur_fwd(const BlurTaps &w, int j, int n, F get) {
    T s = 0;
    if (j >= 5 && j + 5 < n) {
#pragma unroll
        for (int t = 0; t < 11; ++t) s += (T)w.k[t] * get(j - 5 + t);
    } else {
#pragma unroll
        for (int t = 0; t < 11; ++t) s += (T)w.k[t] * get(reflect_idx(j - 5 + t, n));
    }
    return s;
}

// adjoint blur: sum over (r, t) with reflect(r - 5 + t) == j of k[t] g[r]
template <typename T, typename F>
__device__ __forceinline__ T blur_adj(const BlurTaps &w, int j, int n, F get) {
    T s = 0;
    if (n >= 12 && j >= 6 && j + 7 < n) {
        // interior: only the direct source p = j contributes, all taps in range
#pragma unroll
        for (int t = 0; t < 11; ++t) s += (T)w.k[t] * get(j + 5 - t);
        return s;
    }
    if (n < 12) {
        for (int r = 0; r < n; ++r)
#pragma unroll
            for (int t = 0; t < 11; ++t)
                if (reflect_idx(r - 5 + t, n) == j) s += (T)w.k[t] * get(r);
        return s;
    }
    // n >= 12: a source position p in [-5, n+4] reflects onto j iff p == j,
    // p == -j (1 <= j <= 5) or p == 2n-2-j (n-6 <= j <= n-2)
    int ps[3];
    int np = 0;
    ps[np++] = j;
    if (j >= 1 && j <= 5) ps[np++] = -j;
    if (j >= n - 6 && j <= n - 2) ps[np++] = 2 * n - 2 - j;
    for (int c = 0; c < np; ++c) {
        const int p = ps[c];
#pragma unroll
        for (int t = 0; t < 11; ++t) {
            const int r = p + 5 - t;
            if (r >= 0 && r < n) s += (T)w.k[t] * get(r);
        }
    }
    return s;
}

template <typename T>
__global__ void ssim_hblur_kernel(const T *__restrict__ a, const T *__restrict__ b, int H, int W, BlurTaps w,
                                  T *__restrict__ h5) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t N = (int64_t)H * W * 3;
    if (idx >= N) return;
    const int c = (int)(idx % 3);
    const int64_t yx = idx / 3;
    const int x = (int)(yx % W);
    const int64_t row = (yx / W) * W;
    T s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    const bool interior = x >= 5 && x + 5 < W;
#pragma unroll
    for (int t = 0; t < 11; ++t) {
        const int64_t q = (row + (interior ? x - 5 + t : reflect_idx(x - 5 + t, W))) * 3 + c;
        const T av = a[q], bv = b[q], k = (T)w.k[t];
        s0 += k * av;
        s1 += k * bv;
        s2 += k * (av * av);
        s3 += k * (bv * bv);
        s4 += k * (av * bv);
    }
    h5[idx] = s0;
    h5[N + idx] = s1;
    h5[2 * N + idx] = s2;
    h5[3 * N + idx] = s3;
    h5[4 * N + idx] = s4;
}

template <typename T>
__global__ void ssim_vblur_map_kernel(const T *__restrict__ a, const T *__restrict__ b, const T *__restrict__ h5,
                                      int H, int W, BlurTaps w, T *__restrict__ g3, double *__restrict__ sums) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t N = (int64_t)H * W * 3;
    double l1 = 0.0, sm = 0.0;
    if (idx < N) {
        const int64_t rc = idx % ((int64_t)W * 3);  // x*3 + c
        const int y = (int)(idx / ((int64_t)W * 3));
        const int64_t rs = (int64_t)W * 3;
        T m[5];
#pragma unroll
        for (int qd = 0; qd < 5; ++qd) {
            const T *src = h5 + qd * N + rc;
            m[qd] = blur_fwd<T>(w, y, H, [&](int r) { return src[(int64_t)r * rs]; });
        }
        const T C1 = (T)(0.01 * 0.01), C2 = (T)(0.03 * 0.03);
        const T mu_a = m[0], mu_b = m[1];
        const T va = m[2] - mu_a * mu_a, vb = m[3] - mu_b * mu_b, cab = m[4] - mu_a * mu_b;
        const T n1 = (T)2 * mu_a * mu_b + C1, n2 = (T)2 * cab + C2;
        const T d1 = mu_a * mu_a + mu_b * mu_b + C1, d2 = va + vb + C2;
        const T den = d1 * d2;
        const T s = n1 * n2 / den;
        const T g = (T)(1.0 / (double)N);
        const T g_n1 = g * n2 / den, g_n2 = g * n1 / den;
        const T g_den = -g * s / den;
        const T g_d1 = g_den * d2, g_d2 = g_den * d1;
        const T g_cab = (T)2 * g_n2;
        const T g_mu_a = (T)2 * mu_b * g_n1 + (T)2 * mu_a * g_d1 - (T)2 * mu_a * g_d2 - mu_b * g_cab;
        g3[idx] = g_mu_a;
        g3[N + idx] = g_d2;   // g_E[a^2]
        g3[2 * N + idx] = g_cab;  // g_E[ab]
        sm = (double)s;
        l1 = fabs((double)a[idx] - (double)b[idx]);
    }
    // block reduction of (sum |diff|, sum ssim)
    for (int o = 16; o > 0; o >>= 1) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
    }
    __shared__ double red[2][32];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { red[0][wid] = l1; red[1][wid] = sm; }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        l1 = lane < nw ? red[0][lane] : 0.0;
        sm = lane < nw ? red[1][lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
            sm += __shfl_xor_sync(0xffffffffu, sm, o);
        }
        if (lane == 0) {  // per-block partials, summed in block order by loss_sums_kernel
            sums[2 * blockIdx.x] = l1;
            sums[2 * blockIdx.x + 1] = sm;
        }
    }
}

template <typename T>
__global__ void ssim_vadj_kernel(const T *__restrict__ g3, int H, int W, BlurTaps w, T *__restrict__ v3) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t N = (int64_t)H * W * 3;
    if (idx >= N) return;
    const int64_t rc = idx % ((int64_t)W * 3);
    const int y = (int)(idx / ((int64_t)W * 3));
    const int64_t rs = (int64_t)W * 3;
#pragma unroll
    for (int qd = 0; qd < 3; ++qd) {
        const T *src = g3 + qd * N + rc;
        v3[qd * N + idx] = blur_adj<T>(w, y, H, [&](int r) { return src[(int64_t)r * rs]; });
    }
}

template <typename T>
__global__ void ssim_hadj_combine_kernel(const T *__restrict__ a, const T *__restrict__ b, const T *__restrict__ v3,
                                         int H, int W, BlurTaps w, double lambda_ssim, double scale,
                                         T *__restrict__ g_image) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t N = (int64_t)H * W * 3;
    if (idx >= N) return;
    const int c = (int)(idx % 3);
    const int64_t yx = idx / 3;
    const int x = (int)(yx % W);
    const int64_t row = (yx / W) * W;
    T adj[3];
#pragma unroll
    for (int qd = 0; qd < 3; ++qd) {
        const T *src = v3 + qd * N;
        adj[qd] = blur_adj<T>(w, x, W, [&](int r) { return src[(row + r) * 3 + c]; });
    }
    const T av = a[idx], bv = b[idx];
    const T gs = adj[0] + adj[1] * (T)2 * av + adj[2] * bv;
    const T diff = av - bv;
    const T sgn = diff > (T)0 ? (T)1 : (diff < (T)0 ? (T)-1 : (T)0);
    g_image[idx] = (T)scale * ((T)(1.0 - lambda_ssim) * sgn / (T)N - (T)lambda_ssim * gs);
}

// ---------------------------------------------------------------------------
// Tiled path (both sides >= 12): two kernels over kSsimTW x kSsimTH pixel
// tiles, all three channels, the blurs in shared memory.
//   fwd: a, b over the tile's halo (reflected loads: exactly the padded
//        image); horizontal blur of (a, b, a^2, b^2, ab), each thread a run
//        of kSsimHPx outputs from one register window of source pixels;
//        vertical blur, each thread kSsimVRows outputs of one column from a
//        streamed window of rows; SSIM map and its pointwise adjoint -> g3
//        (3 maps) + the L1 / SSIM sums;
//   adj: g3 over the tile's halo (zero outside the image), vertical then
//        horizontal transpose blur (the same register windows), combine with
//        a, b.
// Every output sums its taps in ascending tap order, as the per-output loops
// of the small-image path do.  For n >= 12 every source of output j's adjoint
// lies in [j-5, j+5] (the reflections p = -j and p = 2n-2-j only reach j < 6 /
// j > n-8): interior outputs take the plain taps k[j - r + 5], the 12 border
// ones fold the reflected taps, sum_t k[t] [reflect(r - 5 + t) == j].
constexpr int kSsimTW = 32, kSsimTH = 16, kSsimR = 5;
constexpr int kSsimCols = kSsimTW * 3;                  // floats per tile row
constexpr int kSsimHaloCols = kSsimCols + 6 * kSsimR;   // + 5 px each side
constexpr int kSsimHaloRows = kSsimTH + 2 * kSsimR;
constexpr int kSsimThreads = 256;
constexpr int kSsimHPx = 4;    // horizontal-blur outputs per thread (forward)
constexpr int kSsimVRows = 8;  // vertical-blur outputs per thread; also the adjoint's horizontal run
static_assert(kSsimTH % kSsimVRows == 0 && kSsimTW % kSsimHPx == 0 && kSsimTW % kSsimVRows == 0, "tile");

// reflect() for the halo of an n >= 12 axis: i in [-5, n + 4]
__device__ __forceinline__ int reflect_near(int i, int n) { return i < 0 ? -i : (i >= n ? 2 * n - 2 - i : i); }

// sum_t k[t] [reflect(r - 5 + t) == j] for n >= 12 and |j - r| <= 5: the
// padded position p = r - 5 + t lies in [j - 10, j + 10], where reflect() is
// one mirror at most, so p is j itself, -j (j >= 1) or 2n - 2 - j (j <= n - 2)
template <typename T>
__device__ __forceinline__ T fold_weight(const T *__restrict__ sk, int j, int r, int n) {
    T s = 0;
    const int td = j - r + kSsimR, tl = -j - r + kSsimR, th = 2 * n - 2 - j - r + kSsimR;
    if (td >= 0 && td <= 10) s += sk[td];
    if (j >= 1 && tl >= 0 && tl <= 10) s += sk[tl];
    if (j <= n - 2 && th >= 0 && th <= 10) s += sk[th];
    return s;
}

template <typename T>
__global__ void __launch_bounds__(kSsimThreads)
ssim_fwd_tile_kernel(const T *__restrict__ a, const T *__restrict__ b, int H, int W, BlurTaps w,
                     T *__restrict__ g3, double *__restrict__ sums) {
    extern __shared__ __align__(16) unsigned char ssim_smem[];
    T(*h5)[kSsimHaloRows][kSsimCols] = reinterpret_cast<T(*)[kSsimHaloRows][kSsimCols]>(ssim_smem);
    T(*sab)[kSsimHaloRows][kSsimHaloCols] = reinterpret_cast<T(*)[kSsimHaloRows][kSsimHaloCols]>(
        ssim_smem + sizeof(T) * 5 * kSsimHaloRows * kSsimCols);
    const int x0 = blockIdx.x * kSsimTW, y0 = blockIdx.y * kSsimTH;
    const int64_t rs = (int64_t)W * 3;
    T k[11];
#pragma unroll
    for (int t = 0; t < 11; ++t) k[t] = (T)w.k[t];
    // a, b over the halo with reflected rows and columns: the padded image
    // (rows / columns past n + 4 feed no output inside the image: zero)
#pragma unroll 4  // several halo loads in flight per thread
    for (int e = threadIdx.x; e < kSsimHaloRows * kSsimHaloCols; e += kSsimThreads) {
        const int yy = e / kSsimHaloCols, hc = e - yy * kSsimHaloCols;
        const int hp = hc / 3, c = hc - 3 * hp;
        const int px = x0 - kSsimR + hp, py = y0 - kSsimR + yy;
        T av = 0, bv = 0;
        if (px < W + kSsimR && py < H + kSsimR) {
            const int64_t q = (int64_t)reflect_near(py, H) * rs + (int64_t)reflect_near(px, W) * 3 + c;
            av = a[q];
            bv = b[q];
        }
        sab[0][yy][hc] = av;
        sab[1][yy][hc] = bv;
    }
    __syncthreads();
    // horizontal blur: item = (halo row, run of kSsimHPx pixels, channel)
    constexpr int kRuns = kSsimTW / kSsimHPx;
    for (int it = threadIdx.x; it < kSsimHaloRows * kRuns * 3; it += kSsimThreads) {
        const int yy = it / (kRuns * 3), rem = it - yy * (kRuns * 3);
        const int g = rem / 3, c = rem - 3 * g;
        const int p0 = g * kSsimHPx;  // first output pixel of the run (tile-relative)
        if (x0 + p0 >= W) continue;
        T acc[kSsimHPx][5];
#pragma unroll
        for (int o = 0; o < kSsimHPx; ++o)
#pragma unroll
            for (int q = 0; q < 5; ++q) acc[o][q] = 0;
#pragma unroll
        for (int i = 0; i < kSsimHPx + 10; ++i) {  // halo pixel p0 + i = padded column x - 5 + t, t = i - o
            const T av = sab[0][yy][(p0 + i) * 3 + c], bv = sab[1][yy][(p0 + i) * 3 + c];
            const T aa = av * av, bb = bv * bv, ab = av * bv;
#pragma unroll
            for (int o = 0; o < kSsimHPx; ++o) {
                const int t = i - o;
                if (t >= 0 && t <= 10) {
                    acc[o][0] += k[t] * av;
                    acc[o][1] += k[t] * bv;
                    acc[o][2] += k[t] * aa;
                    acc[o][3] += k[t] * bb;
                    acc[o][4] += k[t] * ab;
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kSsimHPx; ++o)
#pragma unroll
            for (int q = 0; q < 5; ++q) h5[q][yy][(p0 + o) * 3 + c] = acc[o][q];
    }
    __syncthreads();
    // vertical blur + SSIM: item = (column, run of kSsimVRows rows)
    const int64_t N = (int64_t)H * W * 3;
    const T g = (T)(1.0 / (double)N);
    const T C1 = (T)(0.01 * 0.01), C2 = (T)(0.03 * 0.03);
    double l1 = 0.0, sm = 0.0;
    for (int it = threadIdx.x; it < kSsimCols * (kSsimTH / kSsimVRows); it += kSsimThreads) {
        const int rg = it / kSsimCols, cc = it - rg * kSsimCols;
        const int x = x0 + cc / 3, ty0 = rg * kSsimVRows;
        if (x >= W || y0 + ty0 >= H) continue;
        T acc[kSsimVRows][5];
#pragma unroll
        for (int o = 0; o < kSsimVRows; ++o)
#pragma unroll
            for (int q = 0; q < 5; ++q) acc[o][q] = 0;
#pragma unroll
        for (int i = 0; i < kSsimVRows + 10; ++i) {  // halo row ty0 + i, tap t = i - o
            T hv[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) hv[q] = h5[q][ty0 + i][cc];
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) {
                const int t = i - o;
                if (t >= 0 && t <= 10)
#pragma unroll
                    for (int q = 0; q < 5; ++q) acc[o][q] += k[t] * hv[q];
            }
        }
#pragma unroll
        for (int o = 0; o < kSsimVRows; ++o) {
            const int y = y0 + ty0 + o;
            if (y >= H) break;
            const T mu_a = acc[o][0], mu_b = acc[o][1];
            const T va = acc[o][2] - mu_a * mu_a, vb = acc[o][3] - mu_b * mu_b, cab = acc[o][4] - mu_a * mu_b;
            const T n1 = (T)2 * mu_a * mu_b + C1, n2 = (T)2 * cab + C2;
            const T d1 = mu_a * mu_a + mu_b * mu_b + C1, d2 = va + vb + C2;
            const T den = d1 * d2;
            const T inv = (T)1 / den;
            const T sv = n1 * n2 * inv;
            const T g_n1 = g * n2 * inv, g_n2 = g * n1 * inv;
            const T g_den = -g * sv * inv;
            const T g_d1 = g_den * d2, g_d2 = g_den * d1;
            const T g_cab = (T)2 * g_n2;
            const T g_mu_a = (T)2 * mu_b * g_n1 + (T)2 * mu_a * g_d1 - (T)2 * mu_a * g_d2 - mu_b * g_cab;
            const int64_t idx = (int64_t)y * rs + (int64_t)x0 * 3 + cc;
            g3[idx] = g_mu_a;
            g3[N + idx] = g_d2;       // g_E[a^2]
            g3[2 * N + idx] = g_cab;  // g_E[ab]
            sm += (double)sv;
            const T av = sab[0][ty0 + o + kSsimR][cc + 3 * kSsimR], bv = sab[1][ty0 + o + kSsimR][cc + 3 * kSsimR];
            l1 += fabs((double)av - (double)bv);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
    }
    __shared__ double red[2][kSsimThreads / 32];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { red[0][wid] = l1; red[1][wid] = sm; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int q = 0; q < kSsimThreads / 32; ++q) { t0 += red[0][q]; t1 += red[1][q]; }
        const int64_t bid = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;  // per-block partials
        sums[2 * bid] = t0;
        sums[2 * bid + 1] = t1;
    }
}

template <typename T>
__global__ void __launch_bounds__(kSsimThreads)
ssim_adj_tile_kernel(const T *__restrict__ a, const T *__restrict__ b, const T *__restrict__ g3, int H, int W,
                     BlurTaps w, double lambda_ssim, double scale, T *__restrict__ g_image) {
    extern __shared__ __align__(16) unsigned char ssim_smem[];
    T(*gs)[kSsimHaloRows][kSsimHaloCols] = reinterpret_cast<T(*)[kSsimHaloRows][kSsimHaloCols]>(ssim_smem);
    T(*vs)[kSsimTH][kSsimHaloCols] = reinterpret_cast<T(*)[kSsimTH][kSsimHaloCols]>(
        ssim_smem + sizeof(T) * 3 * kSsimHaloRows * kSsimHaloCols);
    const int x0 = blockIdx.x * kSsimTW, y0 = blockIdx.y * kSsimTH;
    const int64_t rs = (int64_t)W * 3, N = (int64_t)H * W * 3;
    __shared__ T sk[11];  // the taps, for the border folds' dynamic indexing
    T k[11];
#pragma unroll
    for (int t = 0; t < 11; ++t) k[t] = (T)w.k[t];
    if (threadIdx.x == 0)
#pragma unroll
        for (int t = 0; t < 11; ++t) sk[t] = k[t];
    // g3 over rows y0-5 .. y0+TH+5 and columns (x0-5)*3 .. (x0+TW+5)*3, zero outside
#pragma unroll 4  // several halo loads in flight per thread
    for (int e = threadIdx.x; e < kSsimHaloRows * kSsimHaloCols; e += kSsimThreads) {
        const int yy = e / kSsimHaloCols, hc = e - yy * kSsimHaloCols;
        const int y = y0 - kSsimR + yy, xf = x0 * 3 - 3 * kSsimR + hc;  // float column
        T v0 = 0, v1 = 0, v2 = 0;
        if (y >= 0 && y < H && xf >= 0 && xf < W * 3) {
            const int64_t q = (int64_t)y * rs + xf;
            v0 = g3[q];
            v1 = g3[N + q];
            v2 = g3[2 * N + q];
        }
        gs[0][yy][hc] = v0;
        gs[1][yy][hc] = v1;
        gs[2][yy][hc] = v2;
    }
    __syncthreads();
    // vertical transpose blur: item = (halo column, run of kSsimVRows rows)
    for (int it = threadIdx.x; it < kSsimHaloCols * (kSsimTH / kSsimVRows); it += kSsimThreads) {
        const int rg = it / kSsimHaloCols, hc = it - rg * kSsimHaloCols;
        const int ty0 = rg * kSsimVRows, yb = y0 + ty0;
        if (yb >= 6 && yb + kSsimVRows - 1 + 7 < H) {
            T acc[kSsimVRows][3];
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) acc[o][0] = acc[o][1] = acc[o][2] = 0;
            // output row ty0 + o takes source halo row ty0 + i with tap t = 10 - (i - o);
            // descending i walks every output's taps in ascending order
#pragma unroll
            for (int i = kSsimVRows + 9; i >= 0; --i) {
                const T s0 = gs[0][ty0 + i][hc], s1 = gs[1][ty0 + i][hc], s2 = gs[2][ty0 + i][hc];
#pragma unroll
                for (int o = 0; o < kSsimVRows; ++o) {
                    const int t = 10 - (i - o);
                    if (t >= 0 && t <= 10) {
                        acc[o][0] += k[t] * s0;
                        acc[o][1] += k[t] * s1;
                        acc[o][2] += k[t] * s2;
                    }
                }
            }
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) {
                vs[0][ty0 + o][hc] = acc[o][0];
                vs[1][ty0 + o][hc] = acc[o][1];
                vs[2][ty0 + o][hc] = acc[o][2];
            }
        } else {
            for (int o = 0; o < kSsimVRows; ++o) {  // border rows: folded reflected taps
                const int y = yb + o;
                T s0 = 0, s1 = 0, s2 = 0;
                if (y < H) {
                    for (int d = -kSsimR; d <= kSsimR; ++d) {
                        const int r = y + d;
                        if (r < 0 || r >= H) continue;
                        const T kw = fold_weight<T>(sk, y, r, H);
                        const int yy = ty0 + o + kSsimR + d;
                        s0 += kw * gs[0][yy][hc];
                        s1 += kw * gs[1][yy][hc];
                        s2 += kw * gs[2][yy][hc];
                    }
                }
                vs[0][ty0 + o][hc] = s0;
                vs[1][ty0 + o][hc] = s1;
                vs[2][ty0 + o][hc] = s2;
            }
        }
    }
    __syncthreads();
    // horizontal transpose blur: item = (row, run of kSsimVRows pixels, channel);
    // the three sums go to shared memory (over the g3 halo, dead since the
    // vertical pass's barrier) so the combine
    // below reads a, b and writes the gradient coalesced
    T(*adj)[kSsimTH][kSsimCols] = reinterpret_cast<T(*)[kSsimTH][kSsimCols]>(ssim_smem);
    constexpr int kRuns = kSsimTW / kSsimVRows;
    for (int it = threadIdx.x; it < kSsimTH * kRuns * 3; it += kSsimThreads) {
        const int ty = it / (kRuns * 3), rem = it - ty * (kRuns * 3);
        const int g = rem / 3, c = rem - 3 * g;
        const int p0 = g * kSsimVRows, xb = x0 + p0, y = y0 + ty;
        if (y >= H || xb >= W) continue;
        T hacc[kSsimVRows][3];
        if (xb >= 6 && xb + kSsimVRows - 1 + 7 < W) {
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) hacc[o][0] = hacc[o][1] = hacc[o][2] = 0;
            // output pixel p0 + o takes halo pixel p0 + i with tap t = 10 - (i - o)
#pragma unroll
            for (int i = kSsimVRows + 9; i >= 0; --i) {
                const int hc = (p0 + i) * 3 + c;
                const T s0 = vs[0][ty][hc], s1 = vs[1][ty][hc], s2 = vs[2][ty][hc];
#pragma unroll
                for (int o = 0; o < kSsimVRows; ++o) {
                    const int t = 10 - (i - o);
                    if (t >= 0 && t <= 10) {
                        hacc[o][0] += k[t] * s0;
                        hacc[o][1] += k[t] * s1;
                        hacc[o][2] += k[t] * s2;
                    }
                }
            }
        } else {
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) {  // border columns: folded reflected taps
                const int x = xb + o;
                T s0 = 0, s1 = 0, s2 = 0;
                if (x < W) {
                    for (int d = -kSsimR; d <= kSsimR; ++d) {
                        const int r = x + d;
                        if (r < 0 || r >= W) continue;
                        const T kw = fold_weight<T>(sk, x, r, W);
                        const int hc = (p0 + o + kSsimR + d) * 3 + c;
                        s0 += kw * vs[0][ty][hc];
                        s1 += kw * vs[1][ty][hc];
                        s2 += kw * vs[2][ty][hc];
                    }
                }
                hacc[o][0] = s0;
                hacc[o][1] = s1;
                hacc[o][2] = s2;
            }
        }
#pragma unroll
        for (int o = 0; o < kSsimVRows; ++o) {
            adj[0][ty][p0 * 3 + c + 3 * o] = hacc[o][0];
            adj[1][ty][p0 * 3 + c + 3 * o] = hacc[o][1];
            adj[2][ty][p0 * 3 + c + 3 * o] = hacc[o][2];
        }
    }
    static_assert(3 * kSsimTH * kSsimCols <= 3 * kSsimHaloRows * kSsimHaloCols, "adj fits over gs");
    __syncthreads();
    // combine (gradients.py:110-116), coalesced over the tile's rows
    const T w_l1 = (T)(1.0 - lambda_ssim) / (T)N, w_ssim = (T)lambda_ssim, sc = (T)scale;
    for (int e = threadIdx.x; e < kSsimTH * kSsimCols; e += kSsimThreads) {
        const int ty = e / kSsimCols, cc = e - ty * kSsimCols;
        const int y = y0 + ty, x = x0 + cc / 3;
        if (y >= H || x >= W) continue;
        const int64_t idx = (int64_t)y * rs + (int64_t)x0 * 3 + cc;
        const T av = a[idx], bv = b[idx];
        const T gsum = adj[0][ty][cc] + adj[1][ty][cc] * (T)2 * av + adj[2][ty][cc] * bv;
        const T diff = av - bv;
        const T sgn = diff > (T)0 ? (T)1 : (diff < (T)0 ? (T)-1 : (T)0);
        g_image[idx] = sc * (w_l1 * sgn - w_ssim * gsum);
    }
}

// ---------------------------------------------------------------------------
// fp32 tiled path on packed pairs (sm_100 FFMA2): the tiles, passes, taps and
// per-element operation order of ssim_fwd_tile_kernel / ssim_adj_tile_kernel
// -- so the same bits -- with (a, b), (a^2, b^2), (mu_a, mu_b), (E[a^2], E[b^2])
// and the adjoint's (g_mu_a, g_E[a^2]) carried as f32x2 pairs: one FFMA2 per
// tap for two of the blurred quantities, 64-bit shared loads and stores.  The
// halo loads walk rows with one warp per row, the per-lane source columns
// computed once (no per-element division).
#ifndef UBS_SSIM_ROW_UNROLL
#define UBS_SSIM_ROW_UNROLL 4
#endif
constexpr int kSsimRowUnroll = UBS_SSIM_ROW_UNROLL;  // halo rows in flight per warp

__device__ __forceinline__ void ssim_col_sources(int x0col, int lane, int W, int (&colq)[4]) {
    // float column lane + 32 j of the forward halo (pixel x0 - 5 + hc / 3): its
    // reflected source column, or -1 past W + 4 (those feed no output)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int hc = lane + 32 * j, hp = hc / 3, c = hc - 3 * hp;
        const int px = x0col - kSsimR + hp;
        colq[j] = (hc < kSsimHaloCols && px < W + kSsimR) ? reflect_near(px, W) * 3 + c : -1;
    }
}

__global__ void __launch_bounds__(kSsimThreads)
ssim_fwd_x2_kernel(const float *__restrict__ a, const float *__restrict__ b, int H, int W, BlurTaps w,
                   float *__restrict__ g3, double *__restrict__ sums) {
    extern __shared__ __align__(16) unsigned char ssim_smem[];
    f32x2(*sab)[kSsimHaloCols] = reinterpret_cast<f32x2(*)[kSsimHaloCols]>(ssim_smem);  // (a, b)
    f32x2(*hab)[kSsimCols] = reinterpret_cast<f32x2(*)[kSsimCols]>(sab + kSsimHaloRows);  // (mu_a, mu_b) rows
    f32x2(*hsq)[kSsimCols] = hab + kSsimHaloRows;                                          // (E[a^2], E[b^2])
    float(*hxy)[kSsimCols] = reinterpret_cast<float(*)[kSsimCols]>(hsq + kSsimHaloRows);   // E[ab]
    const int x0 = blockIdx.x * kSsimTW, y0 = blockIdx.y * kSsimTH;
    const int64_t rs = (int64_t)W * 3;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float k[11];
#pragma unroll
    for (int t = 0; t < 11; ++t) k[t] = (float)w.k[t];
    int colq[4];
    ssim_col_sources(x0, lane, W, colq);
#pragma unroll kSsimRowUnroll
    for (int yy = warp; yy < kSsimHaloRows; yy += kSsimThreads / 32) {
        const int py = y0 - kSsimR + yy;
        const bool rowok = py < H + kSsimR;
        const int64_t rq = rowok ? (int64_t)reflect_near(py, H) * rs : 0;
        float av[4], bv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            av[j] = 0.0f;
            bv[j] = 0.0f;
            if (rowok && colq[j] >= 0) {
                av[j] = a[rq + colq[j]];
                bv[j] = b[rq + colq[j]];
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (lane + 32 * j < kSsimHaloCols) sab[yy][lane + 32 * j] = pk2(av[j], bv[j]);
    }
    __syncthreads();
    // horizontal blur: item = (halo row, run of kSsimHPx pixels, channel)
    constexpr int kRuns = kSsimTW / kSsimHPx;
    for (int it = threadIdx.x; it < kSsimHaloRows * kRuns * 3; it += kSsimThreads) {
        const int yy = it / (kRuns * 3), rem = it - yy * (kRuns * 3);
        const int g = rem / 3, c = rem - 3 * g;
        const int p0 = g * kSsimHPx;
        if (x0 + p0 >= W) continue;
        f32x2 aab[kSsimHPx], asq[kSsimHPx];
        float axy[kSsimHPx];
#pragma unroll
        for (int o = 0; o < kSsimHPx; ++o) {
            aab[o] = 0ull;
            asq[o] = 0ull;
            axy[o] = 0.0f;
        }
#pragma unroll
        for (int i = 0; i < kSsimHPx + 10; ++i) {
            const f32x2 sv = sab[yy][(p0 + i) * 3 + c];
            const f32x2 sq = mul2(sv, sv);  // (a a, b b)
            const float2 s2 = up2(sv);
            const float xy = s2.x * s2.y;
#pragma unroll
            for (int o = 0; o < kSsimHPx; ++o) {
                const int t = i - o;
                if (t >= 0 && t <= 10) {
                    aab[o] = fma2(dup2(k[t]), sv, aab[o]);
                    asq[o] = fma2(dup2(k[t]), sq, asq[o]);
                    axy[o] = fmaf(k[t], xy, axy[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kSsimHPx; ++o) {
            const int col = (p0 + o) * 3 + c;
            hab[yy][col] = aab[o];
            hsq[yy][col] = asq[o];
            hxy[yy][col] = axy[o];
        }
    }
    __syncthreads();
    // vertical blur + SSIM: item = (column, run of kSsimVRows rows)
    const int64_t N = (int64_t)H * W * 3;
    const float g = (float)(1.0 / (double)N);
    const float C1 = (float)(0.01 * 0.01), C2 = (float)(0.03 * 0.03);
    double l1 = 0.0, sm = 0.0;
    for (int it = threadIdx.x; it < kSsimCols * (kSsimTH / kSsimVRows); it += kSsimThreads) {
        const int rg = it / kSsimCols, cc = it - rg * kSsimCols;
        const int x = x0 + cc / 3, ty0 = rg * kSsimVRows;
        if (x >= W || y0 + ty0 >= H) continue;
        f32x2 vab[kSsimVRows], vsq[kSsimVRows];
        float vxy[kSsimVRows];
#pragma unroll
        for (int o = 0; o < kSsimVRows; ++o) {
            vab[o] = 0ull;
            vsq[o] = 0ull;
            vxy[o] = 0.0f;
        }
#pragma unroll
        for (int i = 0; i < kSsimVRows + 10; ++i) {
            const f32x2 hv = hab[ty0 + i][cc], hq = hsq[ty0 + i][cc];
            const float hx = hxy[ty0 + i][cc];
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) {
                const int t = i - o;
                if (t >= 0 && t <= 10) {
                    vab[o] = fma2(dup2(k[t]), hv, vab[o]);
                    vsq[o] = fma2(dup2(k[t]), hq, vsq[o]);
                    vxy[o] = fmaf(k[t], hx, vxy[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kSsimVRows; ++o) {
            const int y = y0 + ty0 + o;
            if (y >= H) break;
            const float2 mu = up2(vab[o]), e2 = up2(vsq[o]);
            const float mu_a = mu.x, mu_b = mu.y;
            const float va = e2.x - mu_a * mu_a, vb = e2.y - mu_b * mu_b, cab = vxy[o] - mu_a * mu_b;
            const float n1 = 2.0f * mu_a * mu_b + C1, n2 = 2.0f * cab + C2;
            const float d1 = mu_a * mu_a + mu_b * mu_b + C1, d2 = va + vb + C2;
            const float den = d1 * d2;
            const float inv = 1.0f / den;
            const float sv = n1 * n2 * inv;
            const float g_n1 = g * n2 * inv, g_n2 = g * n1 * inv;
            const float g_den = -g * sv * inv;
            const float g_d1 = g_den * d2, g_d2 = g_den * d1;
            const float g_cab = 2.0f * g_n2;
            const float g_mu_a = 2.0f * mu_b * g_n1 + 2.0f * mu_a * g_d1 - 2.0f * mu_a * g_d2 - mu_b * g_cab;
            const int64_t idx = (int64_t)y * rs + (int64_t)x0 * 3 + cc;
            g3[idx] = g_mu_a;
            g3[N + idx] = g_d2;       // g_E[a^2]
            g3[2 * N + idx] = g_cab;  // g_E[ab]
            sm += (double)sv;
            const float2 ab = up2(sab[ty0 + o + kSsimR][cc + 3 * kSsimR]);
            l1 += fabs((double)ab.x - (double)ab.y);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
    }
    __shared__ double red[2][kSsimThreads / 32];
    if (lane == 0) {
        red[0][warp] = l1;
        red[1][warp] = sm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int q = 0; q < kSsimThreads / 32; ++q) {
            t0 += red[0][q];
            t1 += red[1][q];
        }
        const int64_t bid = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
        sums[2 * bid] = t0;
        sums[2 * bid + 1] = t1;
    }
}

__global__ void __launch_bounds__(kSsimThreads)
ssim_adj_x2_kernel(const float *__restrict__ a, const float *__restrict__ b, const float *__restrict__ g3, int H,
                   int W, BlurTaps w, double lambda_ssim, double scale, float *__restrict__ g_image) {
    extern __shared__ __align__(16) unsigned char ssim_smem[];
    f32x2(*gs01)[kSsimHaloCols] = reinterpret_cast<f32x2(*)[kSsimHaloCols]>(ssim_smem);        // (g_mu_a, g_E[a^2])
    float(*gs2)[kSsimHaloCols] = reinterpret_cast<float(*)[kSsimHaloCols]>(gs01 + kSsimHaloRows);  // g_E[ab]
    f32x2(*vs01)[kSsimHaloCols] = reinterpret_cast<f32x2(*)[kSsimHaloCols]>(gs2 + kSsimHaloRows);
    float(*vs2)[kSsimHaloCols] = reinterpret_cast<float(*)[kSsimHaloCols]>(vs01 + kSsimTH);
    const int x0 = blockIdx.x * kSsimTW, y0 = blockIdx.y * kSsimTH;
    const int64_t rs = (int64_t)W * 3, N = (int64_t)H * W * 3;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the combine's a, b loads issued first: their latency hides behind the blurs
    constexpr int kComb = kSsimTH * kSsimCols / kSsimThreads;
    static_assert(kSsimTH * kSsimCols % kSsimThreads == 0, "combine items per thread");
    float ca[kComb], cb[kComb];
#pragma unroll
    for (int r = 0; r < kComb; ++r) {
        const int e = threadIdx.x + r * kSsimThreads;
        const int ty = e / kSsimCols, cc = e - ty * kSsimCols;
        const int y = y0 + ty, x = x0 + cc / 3;
        ca[r] = 0.0f;
        cb[r] = 0.0f;
        if (y < H && x < W) {
            const int64_t idx = (int64_t)y * rs + (int64_t)x0 * 3 + cc;
            ca[r] = a[idx];
            cb[r] = b[idx];
        }
    }
    __shared__ float sk[11];  // the taps, for the border folds' dynamic indexing
    float k[11];
#pragma unroll
    for (int t = 0; t < 11; ++t) k[t] = (float)w.k[t];
    if (threadIdx.x == 0)
#pragma unroll
        for (int t = 0; t < 11; ++t) sk[t] = k[t];
    // g3 over rows y0-5 .. y0+TH+5 and float columns (x0-5)*3 .. (x0+TW+5)*3, zero outside
#pragma unroll kSsimRowUnroll
    for (int yy = warp; yy < kSsimHaloRows; yy += kSsimThreads / 32) {
        const int y = y0 - kSsimR + yy;
        const bool rowok = y >= 0 && y < H;
        float v0[4], v1[4], v2[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int hc = lane + 32 * j, xf = x0 * 3 - 3 * kSsimR + hc;
            v0[j] = 0.0f;
            v1[j] = 0.0f;
            v2[j] = 0.0f;
            if (rowok && hc < kSsimHaloCols && xf >= 0 && xf < W * 3) {
                const int64_t q = (int64_t)y * rs + xf;
                v0[j] = g3[q];
                v1[j] = g3[N + q];
                v2[j] = g3[2 * N + q];
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int hc = lane + 32 * j;
            if (hc < kSsimHaloCols) {
                gs01[yy][hc] = pk2(v0[j], v1[j]);
                gs2[yy][hc] = v2[j];
            }
        }
    }
    __syncthreads();
    // vertical transpose blur: item = (halo column, run of kSsimVRows rows)
    for (int it = threadIdx.x; it < kSsimHaloCols * (kSsimTH / kSsimVRows); it += kSsimThreads) {
        const int rg = it / kSsimHaloCols, hc = it - rg * kSsimHaloCols;
        const int ty0 = rg * kSsimVRows, yb = y0 + ty0;
        if (yb >= 6 && yb + kSsimVRows - 1 + 7 < H) {
            f32x2 acc01[kSsimVRows];
            float acc2[kSsimVRows];
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) {
                acc01[o] = 0ull;
                acc2[o] = 0.0f;
            }
            // output row ty0 + o takes source halo row ty0 + i with tap t = 10 - (i - o);
            // descending i walks every output's taps in ascending order
#pragma unroll
            for (int i = kSsimVRows + 9; i >= 0; --i) {
                const f32x2 s01 = gs01[ty0 + i][hc];
                const float s2 = gs2[ty0 + i][hc];
#pragma unroll
                for (int o = 0; o < kSsimVRows; ++o) {
                    const int t = 10 - (i - o);
                    if (t >= 0 && t <= 10) {
                        acc01[o] = fma2(dup2(k[t]), s01, acc01[o]);
                        acc2[o] = fmaf(k[t], s2, acc2[o]);
                    }
                }
            }
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) {
                vs01[ty0 + o][hc] = acc01[o];
                vs2[ty0 + o][hc] = acc2[o];
            }
        } else {
            for (int o = 0; o < kSsimVRows; ++o) {  // border rows: folded reflected taps
                const int y = yb + o;
                float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f;
                if (y < H) {
                    for (int d = -kSsimR; d <= kSsimR; ++d) {
                        const int r = y + d;
                        if (r < 0 || r >= H) continue;
                        const float kw = fold_weight<float>(sk, y, r, H);
                        const int yy = ty0 + o + kSsimR + d;
                        const float2 g01 = up2(gs01[yy][hc]);
                        s0 += kw * g01.x;
                        s1 += kw * g01.y;
                        s2 += kw * gs2[yy][hc];
                    }
                }
                vs01[ty0 + o][hc] = pk2(s0, s1);
                vs2[ty0 + o][hc] = s2;
            }
        }
    }
    __syncthreads();
    // horizontal transpose blur: item = (row, run of kSsimVRows pixels, channel);
    // the sums go to shared memory over the (dead) g3 halo for the coalesced combine
    float(*adj)[kSsimTH][kSsimCols] = reinterpret_cast<float(*)[kSsimTH][kSsimCols]>(ssim_smem);
    static_assert(3 * kSsimTH * kSsimCols * 4 <= 12 * kSsimHaloRows * kSsimHaloCols, "adj fits over gs");
    constexpr int kRuns = kSsimTW / kSsimVRows;
    for (int it = threadIdx.x; it < kSsimTH * kRuns * 3; it += kSsimThreads) {
        const int ty = it / (kRuns * 3), rem = it - ty * (kRuns * 3);
        const int g = rem / 3, c = rem - 3 * g;
        const int p0 = g * kSsimVRows, xb = x0 + p0, y = y0 + ty;
        if (y >= H || xb >= W) continue;
        f32x2 h01[kSsimVRows];
        float h2[kSsimVRows];
        if (xb >= 6 && xb + kSsimVRows - 1 + 7 < W) {
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) {
                h01[o] = 0ull;
                h2[o] = 0.0f;
            }
            // output pixel p0 + o takes halo pixel p0 + i with tap t = 10 - (i - o)
#pragma unroll
            for (int i = kSsimVRows + 9; i >= 0; --i) {
                const int hc = (p0 + i) * 3 + c;
                const f32x2 s01 = vs01[ty][hc];
                const float s2 = vs2[ty][hc];
#pragma unroll
                for (int o = 0; o < kSsimVRows; ++o) {
                    const int t = 10 - (i - o);
                    if (t >= 0 && t <= 10) {
                        h01[o] = fma2(dup2(k[t]), s01, h01[o]);
                        h2[o] = fmaf(k[t], s2, h2[o]);
                    }
                }
            }
        } else {
#pragma unroll
            for (int o = 0; o < kSsimVRows; ++o) {  // border columns: folded reflected taps
                const int x = xb + o;
                float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f;
                if (x < W) {
                    for (int d = -kSsimR; d <= kSsimR; ++d) {
                        const int r = x + d;
                        if (r < 0 || r >= W) continue;
                        const float kw = fold_weight<float>(sk, x, r, W);
                        const int hc = (p0 + o + kSsimR + d) * 3 + c;
                        const float2 g01 = up2(vs01[ty][hc]);
                        s0 += kw * g01.x;
                        s1 += kw * g01.y;
                        s2 += kw * vs2[ty][hc];
                    }
                }
                h01[o] = pk2(s0, s1);
                h2[o] = s2;
            }
        }
#pragma unroll
        for (int o = 0; o < kSsimVRows; ++o) {
            const float2 hv = up2(h01[o]);
            adj[0][ty][p0 * 3 + c + 3 * o] = hv.x;
            adj[1][ty][p0 * 3 + c + 3 * o] = hv.y;
            adj[2][ty][p0 * 3 + c + 3 * o] = h2[o];
        }
    }
    __syncthreads();
    // combine (gradients.py:110-116), coalesced over the tile's rows
    const float w_l1 = (float)(1.0 - lambda_ssim) / (float)N, w_ssim = (float)lambda_ssim, sc = (float)scale;
#pragma unroll
    for (int r = 0; r < kComb; ++r) {
        const int e = threadIdx.x + r * kSsimThreads;
        const int ty = e / kSsimCols, cc = e - ty * kSsimCols;
        const int y = y0 + ty, x = x0 + cc / 3;
        if (y >= H || x >= W) continue;
        const int64_t idx = (int64_t)y * rs + (int64_t)x0 * 3 + cc;
        const float av = ca[r], bv = cb[r];
        const float gsum = adj[0][ty][cc] + adj[1][ty][cc] * 2.0f * av + adj[2][ty][cc] * bv;
        const float diff = av - bv;
        const float sgn = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
        g_image[idx] = sc * (w_l1 * sgn - w_ssim * gsum);
    }
}

// The loss terms' per-block partials summed in block order by one CTA (a
// fixed summation order: the loss value is bitwise reproducible, unlike
// float atomics in arrival order), then added to the caller's sums.
__global__ void __launch_bounds__(256) loss_sums_kernel(const double *__restrict__ part, int64_t nb,
                                                        double *__restrict__ sums) {
    double t0 = 0.0, t1 = 0.0;
    for (int64_t i = threadIdx.x; i < nb; i += 256) {
        t0 += part[2 * i];
        t1 += part[2 * i + 1];
    }
    for (int o = 16; o > 0; o >>= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
    }
    __shared__ double red[2][8];
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = t0;
        red[1][threadIdx.x >> 5] = t1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < 8; ++w) { a += red[0][w]; b += red[1][w]; }
        sums[0] += a;
        sums[1] += b;
    }
}

static int64_t loss_part_offset(int H, int W, int elem) {
    // partials live after the 11 N working maps, 16-byte aligned
    return (((int64_t)11 * H * W * 3 * elem + 15) / 16) * 16;
}

static BlurTaps make_taps() {
    BlurTaps w;
    double s = 0.0;
    for (int t = 0; t < 11; ++t) {
        const double u = (t - 5) / 1.5;
        w.k[t] = exp(-0.5 * u * u);
        s += w.k[t];
    }
    for (int t = 0; t < 11; ++t) w.k[t] /= s;
    return w;
}

template <typename T>
static void run_loss(const T *a, const T *b, int H, int W, double lam, double scale, T *g, double *sums, T *scr,
                     cudaStream_t s) {
    const int64_t N = (int64_t)H * W * 3;
    const BlurTaps w = make_taps();
    const int thr = 256;
    const unsigned blocks = (unsigned)((N + thr - 1) / thr);
    T *h5 = scr, *g3 = scr + 5 * N, *v3 = scr + 8 * N;
    double *part = reinterpret_cast<double *>(reinterpret_cast<char *>(scr) + loss_part_offset(H, W, sizeof(T)));
    if (H >= 12 && W >= 12) {
        const dim3 grid((W + kSsimTW - 1) / kSsimTW, (H + kSsimTH - 1) / kSsimTH);
        const size_t fwd_smem = sizeof(T) * (5 * kSsimHaloRows * kSsimCols + 2 * kSsimHaloRows * kSsimHaloCols);
        const size_t adj_smem = sizeof(T) * 3 * (kSsimHaloRows + kSsimTH) * kSsimHaloCols;
        cudaFuncSetAttribute(ssim_fwd_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem);
        cudaFuncSetAttribute(ssim_adj_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)adj_smem);
        if constexpr (sizeof(T) == 4) {
#ifndef UBS_SSIM_SCALAR
            // packed pairs: the same smem footprint and bits as the scalar tiles
            cudaFuncSetAttribute(ssim_fwd_x2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem);
            cudaFuncSetAttribute(ssim_adj_x2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)adj_smem);
            ssim_fwd_x2_kernel<<<grid, kSsimThreads, fwd_smem, s>>>(a, b, H, W, w, g3, part);
            loss_sums_kernel<<<1, 256, 0, s>>>(part, (int64_t)grid.x * grid.y, sums);
            ssim_adj_x2_kernel<<<grid, kSsimThreads, adj_smem, s>>>(a, b, g3, H, W, w, lam, scale, g);
            return;
#endif
        }
        ssim_fwd_tile_kernel<T><<<grid, kSsimThreads, fwd_smem, s>>>(a, b, H, W, w, g3, part);
        loss_sums_kernel<<<1, 256, 0, s>>>(part, (int64_t)grid.x * grid.y, sums);
        ssim_adj_tile_kernel<T><<<grid, kSsimThreads, adj_smem, s>>>(a, b, g3, H, W, w, lam, scale, g);
        return;
    }
    ssim_hblur_kernel<T><<<blocks, thr, 0, s>>>(a, b, H, W, w, h5);
    ssim_vblur_map_kernel<T><<<blocks, thr, 0, s>>>(a, b, h5, H, W, w, g3, part);
    loss_sums_kernel<<<1, 256, 0, s>>>(part, (int64_t)blocks, sums);
    ssim_vadj_kernel<T><<<blocks, thr, 0, s>>>(g3, H, W, w, v3);
    ssim_hadj_combine_kernel<T><<<blocks, thr, 0, s>>>(a, b, v3, H, W, w, lam, scale, g);
}

}  // namespace ubs

using namespace ubs;

extern "C" size_t ubs_loss_scratch_bytes(int32_t height, int32_t width, int32_t f64) {
    // 11 N working maps + two fp64 partials per block (at most one block per 256 elements)
    const int64_t N = (int64_t)height * width * 3;
    return (size_t)loss_part_offset(height, width, f64 ? 8 : 4) + (size_t)16 * ((N + 255) / 256 + 1);
}

extern "C" int ubs_loss_image_grad(const void *image, const void *target, int32_t height, int32_t width,
                                   int32_t f64, double lambda_ssim, double scale, void *g_image,
                                   double *loss_parts, void *scratch, ubs_stream_t stream) {
    if (!image || !target || !g_image || !loss_parts || !scratch || height < 1 || width < 1) return UBS_E_ARGS;
    cudaStream_t s = (cudaStream_t)stream;
    if (f64)
        run_loss<double>((const double *)image, (const double *)target, height, width, lambda_ssim, scale,
                         (double *)g_image, loss_parts, (double *)scratch, s);
    else
        run_loss<float>((const float *)image, (const float *)target, height, width, lambda_ssim, scale,
                        (float *)g_image, loss_parts, (float *)scratch, s);
    UBS_CUDA_CHECK();
    return UBS_OK;
}

UBS_CHECKED_ACCESSOR(loss)
