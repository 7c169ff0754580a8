// Tile binning: depth order + per-tile depth-ordered id lists.
//
// Reference: raster.py:274-275 (order = ids[lexsort((ids, depth[ids]))]) and
// raster.py:252-266 (build_tiles, an O(tiles x N) mask loop on the CPU).
//
// Device algorithm:
//   1. stable LSD radix sort of (f64 depth bits, id) over all n primitives;
//      invisible primitives carry an all-ones key and sort to the back.  With
//      values emitted in id order the stable sort reproduces lexsort.
//   2. gather each rank's tile count, exclusive scan in rank order.
//   3. emit (tile, id) pairs rank-major, row-major inside each rect.
//   4. stable radix sort on the tile bits only (ceil(log2 n_tiles) bits, two
//      8-bit digit passes at 1080p): since emission is already rank ordered,
//      this equals a full (tile, rank) sort.
//   5. [start, end) per tile without touching the pairs: the preprocess
//      kernel adds each visible rect's corners to a 2D difference array, whose
//      prefix sums are the per-tile counts (tile_scan_kernel).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "ubs_common.cuh"

namespace ubs {

__global__ void iota_kernel(uint32_t *out, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint32_t)i;
}

__global__ void gather_counts_kernel(const uint32_t *__restrict__ order, const uint32_t *__restrict__ tile_count,
                                     uint32_t *__restrict__ counts_by_rank, int64_t n) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) counts_by_rank[r] = tile_count[order[r]];
}

// One warp per 32 consecutive ranks; for each rank the whole warp writes its
// pairs cooperatively, so a primitive covering thousands of tiles does not
// serialise on one thread and every store instruction is coalesced.
__global__ void emit_pairs_kernel(const uint32_t *__restrict__ order, const uint32_t *__restrict__ offsets,
                                  const uint64_t *__restrict__ rect, const uint32_t *__restrict__ tile_count,
                                  const uint32_t *__restrict__ n_visible, int tiles_x,
                                  uint32_t *__restrict__ pair_keys, uint32_t *__restrict__ pair_vals) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nv = *n_visible;
    const int64_t r0 = warp * 32;
    if (r0 >= nv) return;
    const int64_t r = r0 + lane;
    uint32_t id = 0, cnt = 0, off = 0;
    uint64_t rc = 0;
    if (r < nv) {
        id = order[r];
        off = offsets[r];
        cnt = tile_count[id];
        rc = rect[id];
    }
    for (int j = 0; j < 32; ++j) {
        const uint32_t c = __shfl_sync(0xffffffffu, cnt, j);
        if (c == 0) continue;
        const uint32_t pid = __shfl_sync(0xffffffffu, id, j);
        const uint32_t o = __shfl_sync(0xffffffffu, off, j);
        const uint64_t q = __shfl_sync(0xffffffffu, rc, j);
        const uint32_t tx0 = (uint32_t)(q & 0xFFFF), ty0 = (uint32_t)((q >> 16) & 0xFFFF);
        const uint32_t tx1 = (uint32_t)((q >> 32) & 0xFFFF);
        const uint32_t w = tx1 - tx0 + 1;
        // floor((k + 0.5) / w) in fp32 is exact here: (k + 0.5)/w is >= 0.5/w
        // away from an integer, far more than the rounding of two fp32 ops
        const float inv_w = 1.0f / (float)w;
        for (uint32_t k = lane; k < c; k += 32) {
            const uint32_t dy = (uint32_t)(((float)k + 0.5f) * inv_w);
            const uint32_t ty = ty0 + dy, tx = tx0 + (k - dy * w);
            pair_keys[o + k] = ty * (uint32_t)tiles_x + tx;
            pair_vals[o + k] = pid;
        }
    }
}

// Per-tile [start, end) from the rect-corner difference array (one CTA):
// row prefix, column prefix -> per-tile pair counts, then an exclusive scan
// in row-major tile order.  Equals the ranges of the tile-sorted pair array
// because every visible primitive contributes exactly its rect.
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads)
tile_scan_kernel(int32_t *__restrict__ grid, int TX, int TY, uint32_t *__restrict__ ranges) {
    const int gw = TX + 1;
    for (int r = threadIdx.x; r <= TY; r += kScanThreads) {
        int acc = 0;
        for (int c = 0; c <= TX; ++c) {
            acc += grid[r * gw + c];
            grid[r * gw + c] = acc;
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c <= TX; c += kScanThreads) {
        int acc = 0;
        for (int r = 0; r <= TY; ++r) {
            acc += grid[r * gw + c];
            grid[r * gw + c] = acc;
        }
    }
    __syncthreads();
    __shared__ uint32_t warp_tot[kScanThreads / 32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int n_tiles = TX * TY;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < n_tiles; base += kScanThreads) {
        const int t = base + threadIdx.x;
        uint32_t c = 0;
        if (t < n_tiles) c = (uint32_t)grid[(t / TX) * gw + (t % TX)];
        uint32_t x = c;  // inclusive warp scan
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t w = warp_tot[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            warp_tot[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const uint32_t excl = carry + (wid ? warp_tot[wid - 1] : 0u) + x - c;
        if (t < n_tiles) {
            ranges[2 * t] = excl;
            ranges[2 * t + 1] = excl + c;
        }
        __syncthreads();
        if (threadIdx.x == kScanThreads - 1) carry = excl + c;
        __syncthreads();
    }
}

static int tile_bits(int n_tiles) {
    int b = 1;
    while ((1 << b) < n_tiles) ++b;
    return b;
}

}  // namespace ubs

using namespace ubs;

extern "C" size_t ubs_bin_temp_bytes(int64_t n, int64_t pair_capacity, int32_t n_tiles) {
    size_t a = 0, b = 0, c = 0;
    const int nn = (int)(n > 0 ? n : 1);
    const int kk = (int)(pair_capacity > 0 ? pair_capacity : 1);
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, nn, 0, 64);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint32_t *)nullptr, (uint32_t *)nullptr, nn);
    cub::DeviceRadixSort::SortPairs(nullptr, c, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, kk, 0,
                                    tile_bits(n_tiles > 1 ? n_tiles : 2));
    size_t m = a > b ? a : b;
    return (m > c ? m : c) + 256;
}

extern "C" int ubs_bin_depth(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                             ubs_stream_t stream) {
    if (!v || !pb || !bb || !bb->temp || !pb->tile_grid || !bb->tile_ranges) return UBS_E_ARGS;
    const int64_t n = v->n;
    if (n >= (int64_t)1 << 31) return UBS_E_ARGS;
    cudaStream_t s = (cudaStream_t)stream;
    const int TX = (v->cam.width + kTile - 1) / kTile, TY = (v->cam.height + kTile - 1) / kTile;
    tile_scan_kernel<<<1, kScanThreads, 0, s>>>(pb->tile_grid, TX, TY, bb->tile_ranges);
    if (n == 0) {
        UBS_CUDA_CHECK();
        return UBS_OK;
    }
    const int thr = 256;
    const unsigned blocks = (unsigned)((n + thr - 1) / thr);
    iota_kernel<<<blocks, thr, 0, s>>>(bb->ids_iota, n);
    size_t bytes = bb->temp_bytes;
    if (cub::DeviceRadixSort::SortPairs(bb->temp, bytes, pb->depth_key, bb->keys_sorted, bb->ids_iota,
                                        bb->order, (int)n, 0, 64, s) != cudaSuccess)
        return UBS_E_CUDA;
    // ids_iota is free again: reuse it for the rank-ordered counts
    gather_counts_kernel<<<blocks, thr, 0, s>>>(bb->order, pb->tile_count, bb->ids_iota, n);
    bytes = bb->temp_bytes;
    if (cub::DeviceScan::ExclusiveSum(bb->temp, bytes, bb->ids_iota, bb->offsets, (int)n, s) != cudaSuccess)
        return UBS_E_CUDA;
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" int ubs_bin_tiles(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                             int64_t n_pairs, ubs_stream_t stream) {
    if (!v || !pb || !bb) return UBS_E_ARGS;
    const int W = v->cam.width, H = v->cam.height;
    const int TX = (W + kTile - 1) / kTile, TY = (H + kTile - 1) / kTile;
    const int n_tiles = TX * TY;
    cudaStream_t s = (cudaStream_t)stream;
    if (n_pairs == 0 || v->n == 0) return UBS_OK;
    if (n_pairs > bb->pair_capacity || n_pairs >= ((int64_t)1 << 31)) return UBS_E_CAPACITY;
    const int64_t n = v->n;
    const int thr = 256;
    const int64_t warps = (n + 31) / 32;
    emit_pairs_kernel<<<(unsigned)((warps * 32 + thr - 1) / thr), thr, 0, s>>>(
        bb->order, bb->offsets, pb->rect, pb->tile_count, pb->n_visible, TX, bb->pair_keys, bb->pair_vals);
    size_t bytes = bb->temp_bytes;
    if (cub::DeviceRadixSort::SortPairs(bb->temp, bytes, bb->pair_keys, bb->pair_keys_sorted, bb->pair_vals,
                                        bb->tile_ids, (int)n_pairs, 0, tile_bits(n_tiles > 1 ? n_tiles : 2),
                                        s) != cudaSuccess)
        return UBS_E_CUDA;
    UBS_CUDA_CHECK();
    return UBS_OK;
}
