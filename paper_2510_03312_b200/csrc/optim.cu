// Training-step epilogue on the flat (n x P) parameter buffer.
//
// Reference: optim.py:115-135 (adam_step: bias-corrected Adam, per-field
// learning-rate group, shapes clamped to [-5, 5] after the update,
// kernels.py:57-60) and gradients.py:120-123 (regularisers, added once per
// step).  One fused elementwise pass: read param/grad/m/v, write param/m/v;
// memory bound (16-32 B per element).
#include <cuda_runtime.h>

#include "ubs_common.cuh"

namespace ubs {

struct AdamCols {
    float lr[64];          // learning rate of each record column
    uint64_t clamp_mask;   // columns clamped to [-5, 5] after the step (b_x, b_q)
    uint64_t frozen_mask;  // columns not updated (freeze_shapes)
    uint64_t opa_mask;     // opacity_raw column (regulariser sigmoid term)
    uint64_t scale_mask;   // s_x_raw and s_q_raw columns (regulariser exp term)
};

// The next step's starting gradient of one updated parameter (regulariser_kernel's
// value on a zeroed buffer: the same fp64 arithmetic and rounding) and its
// share of the regulariser sums.
template <typename GT>
__device__ __forceinline__ GT next_reg_grad(double p, uint64_t bit, const AdamCols &cols, double reg_o, double reg_s,
                                            double &so, double &ss) {
    if (cols.opa_mask & bit) {
        const double o = sigmoid64(p);
        so += o;
        return (GT)((double)GT(0) + reg_o * o * (1.0 - o));
    }
    if (cols.scale_mask & bit) {
        const double e = exp(p);
        ss += e;
        return (GT)((double)GT(0) + reg_s * e);
    }
    return GT(0);
}

__device__ __forceinline__ void block_add_sums(double so, double ss, double *sums) {
    for (int o = 16; o > 0; o >>= 1) {
        so += __shfl_xor_sync(0xffffffffu, so, o);
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    __shared__ double red[2][8];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = so;
        red[1][w] = ss;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            a += red[0][k];
            b += red[1][k];
        }
        atomicAdd(sums, a);
        atomicAdd(sums + 1, b);
    }
}

// fp32 path: the flat n*P buffer is processed as float4 quads (16 B vector
// loads of param/grad/m/v); each quad's column comes from one division, the
// per-column learning rate and clamp/frozen bits from shared memory.
// kNext: also write the next step's starting gradient over grads (and add the
// regulariser sums): the regularised epilogue
template <bool kNext>
__global__ void __launch_bounds__(256)
adam_f32_kernel(float *__restrict__ params, float *__restrict__ grads, float *__restrict__ m,
                float *__restrict__ v, int64_t total, int P, AdamCols cols, float b1, float b2, float inv_bc1,
                float inv_bc2, float eps, double reg_o, double reg_s, double *__restrict__ sums) {
    double so = 0.0, ss = 0.0;
    __shared__ float slr[64];
    __shared__ uint64_t smask[2];
    if (threadIdx.x < 64) slr[threadIdx.x] = cols.lr[threadIdx.x];
    if (threadIdx.x == 0) { smask[0] = cols.clamp_mask; smask[1] = cols.frozen_mask; }
    __syncthreads();
    const int64_t nq = total / 4;
    for (int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; qi < nq; qi += (int64_t)gridDim.x * blockDim.x) {
        float4 pp = reinterpret_cast<float4 *>(params)[qi];
        const float4 gg = reinterpret_cast<const float4 *>(grads)[qi];  // read before the kNext overwrite
        float4 mm = reinterpret_cast<float4 *>(m)[qi];
        float4 vv = reinterpret_cast<float4 *>(v)[qi];
        int c = (int)((qi * 4) % P);
        float *pe = &pp.x, *me = &mm.x, *ve = &vv.x;
        const float *ge = &gg.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if ((smask[1] >> c) & 1ull) {
                pe[e] = fminf(fmaxf(pe[e], -5.0f), 5.0f);  // frozen: clamp only (optim.py:122-135)
            } else {
                const float g = ge[e];
                const float mi = fmaf(b1, me[e], (1.0f - b1) * g);
                const float vi = fmaf(b2, ve[e], (1.0f - b2) * g * g);
                me[e] = mi;
                ve[e] = vi;
                float p = pe[e] - __fdividef(slr[c] * mi * inv_bc1, sqrtf(vi * inv_bc2) + eps);
                if ((smask[0] >> c) & 1ull) p = fminf(fmaxf(p, -5.0f), 5.0f);
                pe[e] = p;
            }
            c = (c + 1 == P) ? 0 : c + 1;
        }
        reinterpret_cast<float4 *>(params)[qi] = pp;
        reinterpret_cast<float4 *>(m)[qi] = mm;
        reinterpret_cast<float4 *>(v)[qi] = vv;
        if constexpr (kNext) {
            int c2 = (int)((qi * 4) % P);
            float4 gn;
            float *gne = &gn.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                gne[e] = next_reg_grad<float>((double)pe[e], 1ull << c2, cols, reg_o, reg_s, so, ss);
                c2 = (c2 + 1 == P) ? 0 : c2 + 1;
            }
            reinterpret_cast<float4 *>(grads)[qi] = gn;
        }
    }
    if constexpr (kNext) {
        if (sums) block_add_sums(so, ss, sums);
    }
}

// generic path (fp64 parameters or gradients, or a tail): one element per thread
template <typename PT, typename GT, bool kNext>
__global__ void __launch_bounds__(256)
adam_kernel(PT *__restrict__ params, GT *__restrict__ grads, float *__restrict__ m, float *__restrict__ v,
            int64_t begin, int64_t total, int P, AdamCols cols, float b1, float b2, float inv_bc1, float inv_bc2,
            float eps, double reg_o, double reg_s, double *__restrict__ sums) {
    double so = 0.0, ss = 0.0;
    for (int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % P);
        if ((cols.frozen_mask >> c) & 1ull) {
            params[i] = (PT)fmin(fmax((double)params[i], -5.0), 5.0);
            if constexpr (kNext) grads[i] = next_reg_grad<GT>((double)params[i], 1ull << c, cols, reg_o, reg_s, so, ss);
            continue;
        }
        const double g = (double)grads[i];
        const float mi = fmaf(b1, m[i], (1.0f - b1) * (float)g);
        const float vi = fmaf(b2, v[i], (1.0f - b2) * (float)(g * g));
        m[i] = mi;
        v[i] = vi;
        double p = (double)params[i] - (double)cols.lr[c] * ((double)mi * inv_bc1) / (sqrt((double)vi * inv_bc2) + eps);
        if ((cols.clamp_mask >> c) & 1ull) p = fmin(fmax(p, -5.0), 5.0);
        params[i] = (PT)p;
        if constexpr (kNext) grads[i] = next_reg_grad<GT>((double)params[i], 1ull << c, cols, reg_o, reg_s, so, ss);
    }
    if constexpr (kNext) {
        if (sums) block_add_sums(so, ss, sums);
    }
}

// g_opacity_raw += reg_o * o (1 - o); g_s_x_raw += reg_s exp(s_x_raw); g_s_q_raw += reg_s exp(s_q_raw)
template <typename PT, typename GT>
__global__ void regulariser_kernel(const PT *__restrict__ params, GT *__restrict__ grads, int64_t n, int C,
                                   double reg_o, double reg_s) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int P = 14 + 6 * C;
    const PT *r = params + i * P;
    GT *g = grads + i * P;
    const int o_sx = 3 + C + 3, o_sq = o_sx + 3 + 3 * C, o_op = o_sq + C + 1 + C;
    const double o = sigmoid64((double)r[o_op]);
    g[o_op] = (GT)((double)g[o_op] + reg_o * o * (1.0 - o));
    for (int k = 0; k < 3; ++k) g[o_sx + k] = (GT)((double)g[o_sx + k] + reg_s * exp((double)r[o_sx + k]));
    for (int k = 0; k < C; ++k) g[o_sq + k] = (GT)((double)g[o_sq + k] + reg_s * exp((double)r[o_sq + k]));
}

// sums[0] += sum sigmoid(opacity_raw), sums[1] += sum exp(s_x_raw) + sum exp(s_q_raw)
// (the regulariser value, gradients.py:120-123), fp64, one grid-stride pass
template <typename PT>
__global__ void regulariser_value_kernel(const PT *__restrict__ params, int64_t n, int C, double *__restrict__ sums) {
    const int P = 14 + 6 * C;
    const int o_sx = 3 + C + 3, o_sq = o_sx + 3 + 3 * C, o_op = o_sq + C + 1 + C;
    double so = 0.0, ss = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const PT *r = params + i * P;
        so += sigmoid64((double)r[o_op]);
        for (int k = 0; k < 3; ++k) ss += exp((double)r[o_sx + k]);
        for (int k = 0; k < C; ++k) ss += exp((double)r[o_sq + k]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        so += __shfl_xor_sync(0xffffffffu, so, o);
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    __shared__ double red[2][8];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { red[0][w] = so; red[1][w] = ss; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { a += red[0][k]; b += red[1][k]; }
        atomicAdd(sums, a);
        atomicAdd(sums + 1, b);
    }
}

}  // namespace ubs

using namespace ubs;

// lr_group: [position, opacity, scale, other] (optim.py:77-89)
static int adam_launch(void *params, int32_t param_f64, void *grads, int32_t grad_f64, float *m, float *v, int64_t n,
                       int32_t n_dims, const double *lr_group, int32_t step, int32_t freeze_shapes, bool next,
                       double reg_o, double reg_s, double *sums, ubs_stream_t stream) {
    if (!params || !grads || !m || !v || !lr_group || step < 1) return UBS_E_ARGS;
    if (n_dims != 3 && n_dims != 6 && n_dims != 7) return UBS_E_ARGS;
    if (n == 0) return UBS_OK;
    const int C = n_dims - 3, P = 14 + 6 * C;
    AdamCols cols{};
    // column -> learning-rate group, PARAM_FIELDS order
    int c = 0;
    auto put = [&](int count, double lr, bool clampc, uint64_t *reg_mask = nullptr) {
        for (int k = 0; k < count; ++k, ++c) {
            cols.lr[c] = (float)lr;
            if (clampc) {
                cols.clamp_mask |= 1ull << c;
                if (freeze_shapes) cols.frozen_mask |= 1ull << c;
            }
            if (reg_mask) *reg_mask |= 1ull << c;
        }
    };
    const double pos = lr_group[0], opa = lr_group[1], scl = lr_group[2], oth = lr_group[3];
    put(3, pos, false);                        // mu_x
    put(C, oth, false);                        // mu_q
    put(3, oth, false);                        // rot
    put(3, scl, false, &cols.scale_mask);      // s_x_raw
    put(3 * C, oth, false);                    // l_qx
    put(C, scl, false, &cols.scale_mask);      // s_q_raw
    put(1, oth, true);                         // b_x
    put(C, oth, true);                         // b_q
    put(1, opa, false, &cols.opa_mask);        // opacity_raw
    put(3, oth, false);                        // color
    const float b1 = 0.9f, b2 = 0.999f;
    const float inv_bc1 = (float)(1.0 / (1.0 - pow(0.9, step))), inv_bc2 = (float)(1.0 / (1.0 - pow(0.999, step)));
    const int64_t total = n * P;
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned grid = 148 * 8;
    int64_t begin = 0;
    const bool aligned = ((uintptr_t)params % 16 == 0) && ((uintptr_t)grads % 16 == 0) && ((uintptr_t)m % 16 == 0) &&
                         ((uintptr_t)v % 16 == 0);
#define UBS_ADAM_ARGS b1, b2, inv_bc1, inv_bc2, 1e-8f, reg_o, reg_s, sums
    if (!param_f64 && !grad_f64 && aligned) {
        if (next)
            adam_f32_kernel<true><<<grid, 256, 0, s>>>((float *)params, (float *)grads, m, v, total, P, cols, UBS_ADAM_ARGS);
        else
            adam_f32_kernel<false><<<grid, 256, 0, s>>>((float *)params, (float *)grads, m, v, total, P, cols, UBS_ADAM_ARGS);
        begin = (total / 4) * 4;
    }
    if (begin < total) {
        auto run = [&](auto pt, auto gt) {
            using PT = decltype(pt);
            using GT = decltype(gt);
            if (next)
                adam_kernel<PT, GT, true><<<grid, 256, 0, s>>>((PT *)params, (GT *)grads, m, v, begin, total, P, cols, UBS_ADAM_ARGS);
            else
                adam_kernel<PT, GT, false><<<grid, 256, 0, s>>>((PT *)params, (GT *)grads, m, v, begin, total, P, cols, UBS_ADAM_ARGS);
        };
        if (param_f64) {
            if (grad_f64) run(0.0, 0.0);
            else run(0.0, 0.0f);
        } else {
            if (grad_f64) run(0.0f, 0.0);
            else run(0.0f, 0.0f);
        }
    }
#undef UBS_ADAM_ARGS
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" int ubs_adam_step(void *params, int32_t param_f64, const void *grads, int32_t grad_f64, float *m,
                             float *v, int64_t n, int32_t n_dims, const double *lr_group, int32_t step,
                             int32_t freeze_shapes, ubs_stream_t stream) {
    // the plain step never writes grads (the kernels' kNext = false path)
    return adam_launch(params, param_f64, const_cast<void *>(grads), grad_f64, m, v, n, n_dims, lr_group, step,
                       freeze_shapes, false, 0.0, 0.0, nullptr, stream);
}

extern "C" int ubs_adam_step_regularised(void *params, int32_t param_f64, void *grads, int32_t grad_f64, float *m,
                                         float *v, int64_t n, int32_t n_dims, const double *lr_group, int32_t step,
                                         int32_t freeze_shapes, double next_reg_opacity, double next_reg_scale,
                                         double *next_reg_sums, ubs_stream_t stream) {
    return adam_launch(params, param_f64, grads, grad_f64, m, v, n, n_dims, lr_group, step, freeze_shapes, true,
                       next_reg_opacity, next_reg_scale, next_reg_sums, stream);
}

extern "C" int ubs_add_regularisers(const void *params, int32_t param_f64, void *grads, int32_t grad_f64, int64_t n,
                                    int32_t n_dims, double reg_opacity, double reg_scale, ubs_stream_t stream) {
    if (!params || !grads) return UBS_E_ARGS;
    if (n_dims != 3 && n_dims != 6 && n_dims != 7) return UBS_E_ARGS;
    if (n == 0) return UBS_OK;
    const int C = n_dims - 3;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    if (param_f64) {
        if (grad_f64) regulariser_kernel<double, double><<<blocks, 256, 0, s>>>((const double *)params, (double *)grads, n, C, reg_opacity, reg_scale);
        else regulariser_kernel<double, float><<<blocks, 256, 0, s>>>((const double *)params, (float *)grads, n, C, reg_opacity, reg_scale);
    } else {
        if (grad_f64) regulariser_kernel<float, double><<<blocks, 256, 0, s>>>((const float *)params, (double *)grads, n, C, reg_opacity, reg_scale);
        else regulariser_kernel<float, float><<<blocks, 256, 0, s>>>((const float *)params, (float *)grads, n, C, reg_opacity, reg_scale);
    }
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" int ubs_regulariser_value(const void *params, int32_t param_f64, int64_t n, int32_t n_dims, double *sums,
                                     ubs_stream_t stream) {
    if (!params || !sums) return UBS_E_ARGS;
    if (n_dims != 3 && n_dims != 6 && n_dims != 7) return UBS_E_ARGS;
    if (n == 0) return UBS_OK;
    const int C = n_dims - 3;
    const unsigned blocks = (unsigned)min((int64_t)148 * 8, (n + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    if (param_f64) regulariser_value_kernel<double><<<blocks, 256, 0, s>>>((const double *)params, n, C, sums);
    else regulariser_value_kernel<float><<<blocks, 256, 0, s>>>((const float *)params, n, C, sums);
    UBS_CUDA_CHECK();
    return UBS_OK;
}

UBS_CHECKED_ACCESSOR(optim)
