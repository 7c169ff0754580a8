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
        if (lane == 0) {
            atomicAdd(sums, l1);
            atomicAdd(sums + 1, sm);
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
//   fwd: horizontal blur of (a, b, a^2, b^2, ab) over the tile's halo rows
//        (reflected loads: exactly the padded blur), vertical blur from shared
//        memory, SSIM map and its pointwise adjoint -> g3 (3 maps) + sums;
//   adj: g3 over the tile's halo (zero outside the image), vertical then
//        horizontal transpose blur in shared memory, combine with a, b.
// For n >= 12 every source of output j's adjoint lies in [j-5, j+5] (the
// reflections p = -j and p = 2n-2-j only reach j < 6 / j > n-8): interior
// outputs take the plain taps k[j - r + 5], the 12 border ones fold the
// reflected taps, sum_t k[t] [reflect(r - 5 + t) == j].
constexpr int kSsimTW = 32, kSsimTH = 16, kSsimR = 5;
constexpr int kSsimCols = kSsimTW * 3;                  // floats per tile row
constexpr int kSsimHaloCols = kSsimCols + 6 * kSsimR;   // + 5 px each side
constexpr int kSsimHaloRows = kSsimTH + 2 * kSsimR;

template <typename T>
__device__ __forceinline__ T fold_weight(const BlurTaps &w, int j, int r, int n) {
    T s = 0;
#pragma unroll
    for (int t = 0; t < 11; ++t)
        if (reflect_idx(r - kSsimR + t, n) == j) s += (T)w.k[t];
    return s;
}

template <typename T>
__global__ void __launch_bounds__(256)
ssim_fwd_tile_kernel(const T *__restrict__ a, const T *__restrict__ b, int H, int W, BlurTaps w,
                     T *__restrict__ g3, double *__restrict__ sums) {
    extern __shared__ __align__(16) unsigned char ssim_smem[];
    T(*h5)[kSsimHaloRows][kSsimCols] = reinterpret_cast<T(*)[kSsimHaloRows][kSsimCols]>(ssim_smem);
    T(*sab)[kSsimHaloRows][kSsimHaloCols] = reinterpret_cast<T(*)[kSsimHaloRows][kSsimHaloCols]>(
        ssim_smem + sizeof(T) * 5 * kSsimHaloRows * kSsimCols);
    const int x0 = blockIdx.x * kSsimTW, y0 = blockIdx.y * kSsimTH;
    const int64_t rs = (int64_t)W * 3;
    // a, b over the halo with reflected rows and columns: the padded image
    for (int e = threadIdx.x; e < kSsimHaloRows * kSsimHaloCols; e += blockDim.x) {
        const int yy = e / kSsimHaloCols, hc = e - yy * kSsimHaloCols;
        const int px = x0 - kSsimR + hc / 3, c = hc % 3;
        T av = 0, bv = 0;
        if (px < W + kSsimR) {
            const int64_t q = (int64_t)reflect_idx(y0 - kSsimR + yy, H) * rs + (int64_t)reflect_idx(px, W) * 3 + c;
            av = a[q];
            bv = b[q];
        }
        sab[0][yy][hc] = av;
        sab[1][yy][hc] = bv;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kSsimHaloRows * kSsimCols; e += blockDim.x) {
        const int yy = e / kSsimCols, cc = e - yy * kSsimCols;
        const int x = x0 + cc / 3;
        T s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
        if (x < W) {
#pragma unroll
            for (int t = 0; t < 11; ++t) {  // padded column x - 5 + t at halo column cc + 3 t
                const T av = sab[0][yy][cc + 3 * t], bv = sab[1][yy][cc + 3 * t], k = (T)w.k[t];
                s0 += k * av;
                s1 += k * bv;
                s2 += k * (av * av);
                s3 += k * (bv * bv);
                s4 += k * (av * bv);
            }
        }
        h5[0][yy][cc] = s0;
        h5[1][yy][cc] = s1;
        h5[2][yy][cc] = s2;
        h5[3][yy][cc] = s3;
        h5[4][yy][cc] = s4;
    }
    __syncthreads();
    const int64_t N = (int64_t)H * W * 3;
    double l1 = 0.0, sm = 0.0;
    for (int e = threadIdx.x; e < kSsimTH * kSsimCols; e += blockDim.x) {
        const int ty = e / kSsimCols, cc = e - ty * kSsimCols;
        const int y = y0 + ty, x = x0 + cc / 3;
        if (y >= H || x >= W) continue;
        T m[5];
#pragma unroll
        for (int qd = 0; qd < 5; ++qd) {
            T s = 0;
#pragma unroll
            for (int t = 0; t < 11; ++t) s += (T)w.k[t] * h5[qd][ty + t][cc];
            m[qd] = s;
        }
        const T C1 = (T)(0.01 * 0.01), C2 = (T)(0.03 * 0.03);
        const T mu_a = m[0], mu_b = m[1];
        const T va = m[2] - mu_a * mu_a, vb = m[3] - mu_b * mu_b, cab = m[4] - mu_a * mu_b;
        const T n1 = (T)2 * mu_a * mu_b + C1, n2 = (T)2 * cab + C2;
        const T d1 = mu_a * mu_a + mu_b * mu_b + C1, d2 = va + vb + C2;
        const T den = d1 * d2;
        const T sv = n1 * n2 / den;
        const T g = (T)(1.0 / (double)N);
        const T g_n1 = g * n2 / den, g_n2 = g * n1 / den;
        const T g_den = -g * sv / den;
        const T g_d1 = g_den * d2, g_d2 = g_den * d1;
        const T g_cab = (T)2 * g_n2;
        const T g_mu_a = (T)2 * mu_b * g_n1 + (T)2 * mu_a * g_d1 - (T)2 * mu_a * g_d2 - mu_b * g_cab;
        const int64_t idx = (int64_t)y * rs + (int64_t)x0 * 3 + cc;
        g3[idx] = g_mu_a;
        g3[N + idx] = g_d2;       // g_E[a^2]
        g3[2 * N + idx] = g_cab;  // g_E[ab]
        sm += (double)sv;
        l1 += fabs((double)a[idx] - (double)b[idx]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
    }
    __shared__ double red[2][8];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { red[0][wid] = l1; red[1][wid] = sm; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { t0 += red[0][k]; t1 += red[1][k]; }
        atomicAdd(sums, t0);
        atomicAdd(sums + 1, t1);
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
ssim_adj_tile_kernel(const T *__restrict__ a, const T *__restrict__ b, const T *__restrict__ g3, int H, int W,
                     BlurTaps w, double lambda_ssim, double scale, T *__restrict__ g_image) {
    extern __shared__ __align__(16) unsigned char ssim_smem[];
    T(*gs)[kSsimHaloRows][kSsimHaloCols] = reinterpret_cast<T(*)[kSsimHaloRows][kSsimHaloCols]>(ssim_smem);
    T(*vs)[kSsimTH][kSsimHaloCols] = reinterpret_cast<T(*)[kSsimTH][kSsimHaloCols]>(
        ssim_smem + sizeof(T) * 3 * kSsimHaloRows * kSsimHaloCols);
    const int x0 = blockIdx.x * kSsimTW, y0 = blockIdx.y * kSsimTH;
    const int64_t rs = (int64_t)W * 3, N = (int64_t)H * W * 3;
    // g3 over rows y0-5 .. y0+TH+5 and columns (x0-5)*3 .. (x0+TW+5)*3, zero outside
    for (int e = threadIdx.x; e < kSsimHaloRows * kSsimHaloCols; e += blockDim.x) {
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
    // vertical transpose blur for the tile's rows, all halo columns
    for (int e = threadIdx.x; e < kSsimTH * kSsimHaloCols; e += blockDim.x) {
        const int ty = e / kSsimHaloCols, hc = e - ty * kSsimHaloCols;
        const int y = y0 + ty;
        T s0 = 0, s1 = 0, s2 = 0;
        if (y < H) {
            if (y >= 6 && y + 7 < H) {
#pragma unroll
                for (int t = 0; t < 11; ++t) {  // source row r = y + 5 - t, at yy = ty + 10 - t
                    const T k = (T)w.k[t];
                    s0 += k * gs[0][ty + 10 - t][hc];
                    s1 += k * gs[1][ty + 10 - t][hc];
                    s2 += k * gs[2][ty + 10 - t][hc];
                }
            } else {
                for (int d = -kSsimR; d <= kSsimR; ++d) {
                    const int r = y + d;
                    if (r < 0 || r >= H) continue;
                    const T k = fold_weight<T>(w, y, r, H);
                    s0 += k * gs[0][ty + kSsimR + d][hc];
                    s1 += k * gs[1][ty + kSsimR + d][hc];
                    s2 += k * gs[2][ty + kSsimR + d][hc];
                }
            }
        }
        vs[0][ty][hc] = s0;
        vs[1][ty][hc] = s1;
        vs[2][ty][hc] = s2;
    }
    __syncthreads();
    // horizontal transpose blur + combine (gradients.py:110-116)
    for (int e = threadIdx.x; e < kSsimTH * kSsimCols; e += blockDim.x) {
        const int ty = e / kSsimCols, cc = e - ty * kSsimCols;
        const int y = y0 + ty, x = x0 + cc / 3;
        if (y >= H || x >= W) continue;
        const int hc0 = cc + 3 * kSsimR;  // this element in halo columns
        T adj0 = 0, adj1 = 0, adj2 = 0;
        if (x >= 6 && x + 7 < W) {
#pragma unroll
            for (int t = 0; t < 11; ++t) {  // source column x + 5 - t
                const int hc = hc0 + 3 * (kSsimR - t);
                const T k = (T)w.k[t];
                adj0 += k * vs[0][ty][hc];
                adj1 += k * vs[1][ty][hc];
                adj2 += k * vs[2][ty][hc];
            }
        } else {
            for (int d = -kSsimR; d <= kSsimR; ++d) {
                const int r = x + d;
                if (r < 0 || r >= W) continue;
                const T k = fold_weight<T>(w, x, r, W);
                const int hc = hc0 + 3 * d;
                adj0 += k * vs[0][ty][hc];
                adj1 += k * vs[1][ty][hc];
                adj2 += k * vs[2][ty][hc];
            }
        }
        const int64_t idx = (int64_t)y * rs + (int64_t)x0 * 3 + cc;
        const T av = a[idx], bv = b[idx];
        const T gsum = adj0 + adj1 * (T)2 * av + adj2 * bv;
        const T diff = av - bv;
        const T sgn = diff > (T)0 ? (T)1 : (diff < (T)0 ? (T)-1 : (T)0);
        g_image[idx] = (T)scale * ((T)(1.0 - lambda_ssim) * sgn / (T)N - (T)lambda_ssim * gsum);
    }
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
    if (H >= 12 && W >= 12) {
        const dim3 grid((W + kSsimTW - 1) / kSsimTW, (H + kSsimTH - 1) / kSsimTH);
        const size_t fwd_smem = sizeof(T) * (5 * kSsimHaloRows * kSsimCols + 2 * kSsimHaloRows * kSsimHaloCols);
        const size_t adj_smem = sizeof(T) * 3 * (kSsimHaloRows + kSsimTH) * kSsimHaloCols;
        cudaFuncSetAttribute(ssim_fwd_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem);
        cudaFuncSetAttribute(ssim_adj_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)adj_smem);
        ssim_fwd_tile_kernel<T><<<grid, 256, fwd_smem, s>>>(a, b, H, W, w, g3, sums);
        ssim_adj_tile_kernel<T><<<grid, 256, adj_smem, s>>>(a, b, g3, H, W, w, lam, scale, g);
        return;
    }
    ssim_hblur_kernel<T><<<blocks, thr, 0, s>>>(a, b, H, W, w, h5);
    ssim_vblur_map_kernel<T><<<blocks, thr, 0, s>>>(a, b, h5, H, W, w, g3, sums);
    ssim_vadj_kernel<T><<<blocks, thr, 0, s>>>(g3, H, W, w, v3);
    ssim_hadj_combine_kernel<T><<<blocks, thr, 0, s>>>(a, b, v3, H, W, w, lam, scale, g);
}

}  // namespace ubs

using namespace ubs;

extern "C" size_t ubs_loss_scratch_bytes(int32_t height, int32_t width, int32_t f64) {
    return (size_t)11 * height * width * 3 * (f64 ? 8 : 4);
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
