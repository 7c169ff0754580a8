// Tile binning: depth order + per-tile depth-ordered id lists.
//
// Reference: raster.py:274-275 (order = ids[lexsort((ids, depth[ids]))]) and
// raster.py:252-266 (build_tiles, an O(tiles x N) mask loop on the CPU).
//
// Device algorithm:
//   1. bucket sort of the visible primitives by (f64 depth bits, id): range-
//      normalised key histogram, scan, scatter, exact rank inside each bucket
//      (reproduces lexsort, ties by id).
//   2. per-tile [start, end): the preprocess kernel adds each visible rect's
//      corners to a 2D difference array whose prefix sums are the per-tile
//      counts (tile_scan_kernel); no pass over the K pairs.
//   3. per-tile depth-ordered lists without a global pair sort: see the
//      "Sort-free stable binning" block below.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include "ubs_common.cuh"

// At most 2^20 depth buckets: their 4 MB of cursors stay L2-resident under the
// scatter's one random atomic per element (2^24 buckets at 10M primitives:
// depth scatter 656 us; capped: bin_depth 0.98 -> 0.59 ms, 390 -> 457 fps).
#ifndef UBS_SORT_MAX_LOG
#define UBS_SORT_MAX_LOG 20
#endif
namespace ubs {

// Depth order = lexsort((ids, depth)) (raster.py:274-275) as a bucket sort.
// key32 = (f64 depth bits - min) >> shift (< 2^31, monotone in depth); its top
// log2(B) bits pick one of B ~ n buckets.  (1) histogram, (2) exclusive
// scan (CUB), (3) scatter of (f64 bits, id) into bucket slots in arrival
// order, (4) inside each bucket every element counts the elements that
// precede it by (f64 bits, id) -- the exact lexsort order, ties by id -- and
// writes its id there.  O(n) traffic in four light passes; the rank step is
// O(s) per element for a bucket of s elements (a few on average; thousands
// only if that many primitives share nearly the same depth bits).
constexpr uint64_t kNoRect = ~0ull;  // rect_sorted entry of a primitive that touches no tile

__host__ __device__ inline int sort_log_buckets(int64_t n) {
    int l = 12;
    while (l < UBS_SORT_MAX_LOG && ((int64_t)1 << l) < n) ++l;
    return l;
}

struct DepthBuckets {
    unsigned long long lo;
    int shift, bshift;
};

__device__ __forceinline__ DepthBuckets depth_buckets(const unsigned long long *range, int logB) {
    DepthBuckets d;
    d.lo = range[0];
    const unsigned long long hi = range[1];
    const unsigned long long span = hi >= d.lo ? hi - d.lo : 0ull;
    const int bits = span ? 64 - __clzll((long long)span) : 0;
    d.shift = bits > 31 ? bits - 31 : 0;
    d.bshift = 31 - logB;
    return d;
}

__device__ __forceinline__ uint32_t depth_bucket(const DepthBuckets &d, uint64_t k) {
    return (uint32_t)((k - d.lo) >> d.shift) >> d.bshift;
}

__global__ void depth_hist_kernel(const uint64_t *__restrict__ key64, const unsigned long long *__restrict__ range,
                                  int64_t n, int logB, uint32_t *__restrict__ hist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = key64[i];
    if (k == kInvisibleKey) return;
    atomicAdd(hist + depth_bucket(depth_buckets(range, logB), k), 1u);
}

// hist[b] counts down to 0 while slots [start[b], start[b] + count) fill
__global__ void depth_scatter_kernel(const uint64_t *__restrict__ key64, const unsigned long long *__restrict__ range,
                                     int64_t n, int logB, const uint32_t *__restrict__ start,
                                     uint32_t *__restrict__ hist, uint64_t *__restrict__ tkey,
                                     uint32_t *__restrict__ tid) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = key64[i];
    if (k == kInvisibleKey) return;
    const uint32_t b = depth_bucket(depth_buckets(range, logB), k);
    const uint32_t pos = start[b] + atomicSub(hist + b, 1u) - 1u;
    if (!UBS_GUARD(pos < (uint32_t)n, kChkRank)) return;
    tkey[pos] = k;
    tid[pos] = (uint32_t)i;
}

// also writes each primitive's tile rect at its rank (all-ones: no tile), so
// the level-1 binning reads rects coalesced in depth order
__global__ void depth_rank_kernel(const unsigned long long *__restrict__ range, int logB,
                                  const uint32_t *__restrict__ start, const uint64_t *__restrict__ tkey,
                                  const uint32_t *__restrict__ tid, const uint32_t *__restrict__ n_visible,
                                  const uint64_t *__restrict__ rect, const uint32_t *__restrict__ tile_count,
                                  uint32_t *__restrict__ order, uint64_t *__restrict__ rect_sorted) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (int64_t)*n_visible) return;
    const uint64_t k = tkey[p];
    const uint32_t id = tid[p];
    const uint32_t b = depth_bucket(depth_buckets(range, logB), k);
    const uint32_t s0 = start[b], s1 = start[b + 1];
    uint32_t rank = 0;
    for (uint32_t q = s0; q < s1; ++q) {
        const uint64_t kq = tkey[q];
        rank += (kq < k || (kq == k && tid[q] < id)) ? 1u : 0u;
    }
    if (!UBS_GUARD(s0 + rank < s1 && s1 <= *n_visible, kChkRank)) return;
    order[s0 + rank] = id;
    rect_sorted[s0 + rank] = tile_count[id] != 0 ? rect[id] : kNoRect;
}

// Per-tile [start, end) from the rect-corner difference array (one CTA):
// row prefix, column prefix -> per-tile pair counts, then an exclusive scan
// in row-major tile order.  Equals the ranges of the tile-sorted pair array
// because every visible primitive contributes exactly its rect.
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads)
tile_scan_kernel(const int32_t *__restrict__ grid_in, int TX, int TY, uint32_t *__restrict__ ranges) {
    extern __shared__ int32_t g[];
    const int gw = TX + 1, gsz = (TX + 1) * (TY + 1);
    for (int i = threadIdx.x; i < gsz; i += kScanThreads) g[i] = grid_in[i];
    __syncthreads();
    for (int r = threadIdx.x; r <= TY; r += kScanThreads) {
        int acc = 0;
        for (int c = 0; c <= TX; ++c) acc = (g[r * gw + c] += acc);
    }
    __syncthreads();
    for (int c = threadIdx.x; c <= TX; c += kScanThreads) {
        int acc = 0;
        for (int r = 0; r <= TY; ++r) acc = (g[r * gw + c] += acc);
    }
    __syncthreads();
    // exclusive scan of the per-tile counts in row-major order: warp w owns
    // a contiguous span of tiles (a multiple of 32); pass 1 sums each span
    // (REDUX), one scan over the 32 span totals, pass 2 rescans each span in
    // 32-tile chunks and writes the ranges coalesced (3 barriers in all)
    __shared__ uint32_t warp_tot[kScanThreads / 32];
    const int n_tiles = TX * TY;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int kWarps = kScanThreads / 32;
    const int span = ((n_tiles + 32 * kWarps - 1) / (32 * kWarps)) * 32;
    const int w0 = min(n_tiles, wid * span), w1 = min(n_tiles, w0 + span);
    // this lane's first tile w0 + lane as (row, column), advanced 32 tiles per chunk
    const int ty0 = (w0 + lane) / TX, tx0 = (w0 + lane) - ty0 * TX;
    int ty = ty0, tx = tx0;
    uint32_t tot = 0;
    for (int t = w0 + lane; t - lane < w1; t += 32) {
        if (t < w1) tot += (uint32_t)g[ty * gw + tx];
        tx += 32;
        while (tx >= TX) { tx -= TX; ++ty; }
    }
    tot = __reduce_add_sync(0xffffffffu, tot);
    if (lane == 0) warp_tot[wid] = tot;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    uint32_t carry = wid ? warp_tot[wid - 1] : 0u;
    ty = ty0;
    tx = tx0;
    for (int t = w0 + lane; t - lane < w1; t += 32) {
        const uint32_t c = t < w1 ? (uint32_t)g[ty * gw + tx] : 0u;
        uint32_t x = c;  // inclusive warp scan of the chunk
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t excl = carry + x - c;
        if (t < w1) {
            ranges[2 * t] = excl;
            ranges[2 * t + 1] = excl + c;
        }
        carry += __shfl_sync(0xffffffffu, x, 31);
        tx += 32;
        while (tx >= TX) { tx -= TX; ++ty; }
    }
}

// Large frames (grid beyond one CTA's shared memory): the same three steps in
// global memory -- row prefix (a warp per row), column prefix (a thread per
// column), then a three-phase exclusive scan of the per-tile counts.
__global__ void grid_row_prefix_kernel(int32_t *__restrict__ g, int gw, int rows) {
    const int r = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (r >= rows) return;
    int32_t carry = 0;
    for (int c0 = 0; c0 < gw; c0 += 32) {
        const int c = c0 + lane;
        int32_t x = c < gw ? g[(int64_t)r * gw + c] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (c < gw) g[(int64_t)r * gw + c] = x + carry;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
}

__global__ void grid_col_prefix_kernel(int32_t *__restrict__ g, int gw, int rows) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= gw) return;
    int32_t acc = 0;
    for (int r = 0; r < rows; ++r) acc = (g[(int64_t)r * gw + c] += acc);
}

__device__ __forceinline__ uint32_t block_excl_scan1024(uint32_t v, uint32_t *warp_tot, uint32_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    total = warp_tot[31];
    const uint32_t ex = (wid ? warp_tot[wid - 1] : 0u) + x - v;
    __syncthreads();
    return ex;
}

__device__ __forceinline__ uint32_t tile_count_at(const int32_t *g, int TX, int t) {
    return (uint32_t)g[(int64_t)(t / TX) * (TX + 1) + (t % TX)];
}

__global__ void __launch_bounds__(1024) tile_block_sums_kernel(const int32_t *__restrict__ g, int TX, int n_tiles,
                                                               uint32_t *__restrict__ bsum) {
    __shared__ uint32_t warp_tot[32];
    const int t = blockIdx.x * 1024 + threadIdx.x;
    uint32_t total;
    block_excl_scan1024(t < n_tiles ? tile_count_at(g, TX, t) : 0u, warp_tot, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) tile_block_scan_kernel(uint32_t *__restrict__ bsum, int nb) {
    __shared__ uint32_t warp_tot[32];
    uint32_t carry = 0;
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nb ? bsum[i] : 0u;
        uint32_t total;
        const uint32_t ex = block_excl_scan1024(v, warp_tot, total);
        if (i < nb) bsum[i] = carry + ex;
        carry += total;
    }
}

__global__ void __launch_bounds__(1024) tile_ranges_kernel(const int32_t *__restrict__ g, int TX, int n_tiles,
                                                           const uint32_t *__restrict__ bsum,
                                                           uint32_t *__restrict__ ranges) {
    __shared__ uint32_t warp_tot[32];
    const int t = blockIdx.x * 1024 + threadIdx.x;
    const uint32_t c = t < n_tiles ? tile_count_at(g, TX, t) : 0u;
    uint32_t total;
    const uint32_t ex = bsum[blockIdx.x] + block_excl_scan1024(c, warp_tot, total);
    if (t < n_tiles) {
        ranges[2 * t] = ex;
        ranges[2 * t + 1] = ex + c;
    }
}

// ---------------------------------------------------------------------------
// Sort-free stable binning.
//
// Per-tile lists are built in two levels so that every large write is
// contiguous:
//   level 1: rank-ordered entries (id, mask of the bucket tiles its rect
//            covers) are stably distributed into coarse buckets of kRows x
//            kBand tiles.  Ranks are cut into G chunks of kCtaRanks;
//            per-chunk bucket histograms, offsets from a scan over chunks,
//            then an ordered scatter (flattened rank-major (rank, bucket)
//            walk, see below).
//   level 2: one warp per tile scans its bucket (staged in shared memory
//            once per tile row) and appends, in order, the entries whose mask
//            has the tile's bit, stopping at the list cap.
// Bucket shape: 8 x 4 tiles cuts level-1 entries ~2.6x against 8 x 1 for
// ~1.4x more level-2 reads (bench scene: 7.3M -> 2.8M entries, 14.5M ->
// 20.7M reads), and the per-CTA bucket counters shrink 4x.
// Every tile list is the rank-ordered set of visible primitives whose rect
// contains the tile == build_tiles (raster.py:252-266).
// HBM: 8 B per bucket entry written + read (L2-resident at 1080p), 4 B per
// pair written once; no global sort of the K pairs.
// ---------------------------------------------------------------------------
constexpr int kBand = 8;  // tile columns per bucket
constexpr int kRows = 4;  // tile rows per bucket

// Level-1 work unit: one warp per chunk of kChunkRanks consecutive ranks
// (8 warps per CTA), each with a private shared-memory counter per bucket.
constexpr int kChunkRanks = 128;             // ranks per warp slice
constexpr int kCtaRanks = kChunkRanks * 8;   // ranks per CTA chunk (one histogram row)
constexpr int kBinWarps = 8;

// The (rank, bucket) pairs of a batch of 32 consecutive ranks, flattened in
// rank-major order (and row-major bucket order inside a rank): lane j holds
// rank j's rect; after a warp inclusive scan of the per-rank bucket counts,
// flat index f belongs to the rank j with incl[j-1] <= f < incl[j] (found by
// a 5-step shuffle binary search).  A warp step thus covers 32 pairs instead
// of one rank's ~9 buckets.
struct FlatBatch {
    uint64_t q;      // this lane's rect
    int nb, incl;    // this lane's bucket count and inclusive prefix
    int total;       // pairs in the batch
    bool fast;       // owner[] holds the lane of every flat index
};

// Per-warp shared staging of a 32-rank batch: each lane's rect, flat offset
// and id, plus owner[f] = lane of flat index f when the batch has at most
// kOwnerCap pairs (then a flat index resolves with two dependent shared loads
// instead of a 5-step shuffle binary search).
constexpr int kOwnerCap = 512;
struct FlatStage {
    uint64_t q[32];
    int excl[32];
    uint32_t id[32];
    uint8_t owner[kOwnerCap];
};

__device__ __forceinline__ int rank_bucket_count(uint64_t q, bool has) {
    if (!has) return 0;
    const int b0 = (int)(q & 0xFFFF) / kBand, g0 = (int)((q >> 16) & 0xFFFF) / kRows;
    const int b1 = (int)((q >> 32) & 0xFFFF) / kBand, g1 = (int)((q >> 48) & 0xFFFF) / kRows;
    return (b1 - b0 + 1) * (g1 - g0 + 1);
}

// level-1 entry: id | mask of the bucket's kBand x kRows tiles the rect
// covers (bit ly * kBand + lx) << 32
__device__ __forceinline__ uint64_t bucket_entry(uint32_t id, uint64_t q, int band, int grp) {
    static_assert(kBand * kRows == 32, "tile mask is 32 bits");
    const int bx = band * kBand, by = grp * kRows;
    const int x0 = max((int)(q & 0xFFFF) - bx, 0), x1 = min((int)((q >> 32) & 0xFFFF) - bx, kBand - 1);
    const int y0 = max((int)((q >> 16) & 0xFFFF) - by, 0), y1 = min((int)(q >> 48) - by, kRows - 1);
    const uint32_t row = ((2u << x1) - 1u) & ~((1u << x0) - 1u);  // bits x0..x1
    // the row replicated into bytes y0..y1 (kBand = 8 bits per tile row)
    const uint32_t rows = (0xFFFFFFFFu >> (8 * (kRows - 1 - y1))) & (0xFFFFFFFFu << (8 * y0));
    const uint32_t mask = (row * 0x01010101u) & rows;
    return (uint64_t)id | ((uint64_t)mask << 32);
}

__device__ __forceinline__ FlatBatch flat_batch(uint64_t q, bool has, uint32_t id, int lane, FlatStage &st) {
    FlatBatch fb;
    fb.q = q;
    fb.nb = rank_bucket_count(q, has);
    int x = fb.nb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    fb.incl = x;
    fb.total = __shfl_sync(0xffffffffu, x, 31);
    fb.fast = fb.total <= kOwnerCap;
    __syncwarp();  // the previous batch's readers are done
    const int excl = x - fb.nb;
    st.q[lane] = q;
    st.excl[lane] = excl;
    st.id[lane] = id;
    if (fb.fast)
        for (int i = 0; i < fb.nb; ++i)
            if (UBS_GUARD(excl + i < kOwnerCap, kChkOwner)) st.owner[excl + i] = (uint8_t)lane;
    __syncwarp();
    return fb;
}

// (rank lane j, bucket k = grp * NB + band) of flat index f (all lanes
// participate: the slow path shuffles); q = rank j's rect
__device__ __forceinline__ int flat_locate(const FlatBatch &fb, const FlatStage &st, int f, int NB, int &j,
                                           uint64_t &q, int &band, int &grp) {
    if (fb.fast) {
        j = st.owner[f];
    } else {
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int incl_mid = __shfl_sync(0xffffffffu, fb.incl, lo + step - 1);
            if (incl_mid <= f) lo += step;
        }
        j = lo;  // first lane whose inclusive prefix exceeds f
    }
    if (!UBS_GUARD(j >= 0 && j < 32, kChkLocate)) j = 0;
    q = st.q[j];
    const int excl = st.excl[j];
    const int b0 = (int)(q & 0xFFFF) / kBand, g0 = (int)((q >> 16) & 0xFFFF) / kRows;
    const int nbw = (int)((q >> 32) & 0xFFFF) / kBand - b0 + 1;
    const int i = f - excl;
    // floor((i + 0.5) / nbw) with the MUFU reciprocal: (i + 0.5) / nbw is at
    // least 0.5 / nbw from an integer and the product's relative error is
    // < 3 * 2^-24, so the floor is exact while i < 2^24 / 6 (i < buckets of one
    // rect: 32k at 16K x 16K)
    float rc;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"((float)nbw));
    const int r = (int)(((float)i + 0.5f) * rc);
    band = b0 + (i - r * nbw);
    grp = g0 + r;
    return grp * NB + band;
}

// count the (rank, bucket) pairs of ranks [r0, r1) into cnt (shared atomics)
__device__ __forceinline__ void count_slice(const uint64_t *__restrict__ rect_sorted, int64_t r0, int64_t r1,
                                            int NB, int nbk, uint32_t *cnt, int lane, FlatStage &st) {
    for (int64_t rb = r0; rb < r1; rb += 32) {
        const int64_t r = rb + lane;
        uint64_t q = 0;
        bool has = false;
        if (r < r1) {
            q = rect_sorted[r];
            has = q != kNoRect;
            if (!has) q = 0;
        }
        const FlatBatch fb = flat_batch(q, has, 0u, lane, st);
        for (int f0 = 0; f0 < fb.total; f0 += 32) {
            const int f = f0 + lane;
            int j, band, grp;
            uint64_t q;
            const int k = flat_locate(fb, st, min(f, fb.total - 1), NB, j, q, band, grp);
            if (f < fb.total && UBS_GUARD(k >= 0 && k < nbk, kChkBucket)) atomicAdd(&cnt[k], 1u);
        }
    }
}

// (1) per-CTA-chunk bucket counts (8 warps count 128-rank slices into one array)
__global__ void __launch_bounds__(kBinWarps * 32)
bucket_hist_kernel(const uint64_t *__restrict__ rect_sorted, const uint32_t *__restrict__ n_visible, int G, int NB,
                   int nbk, uint32_t *__restrict__ hist, uint32_t *__restrict__ whist) {
    extern __shared__ uint32_t scnt_all[];  // kBinWarps x nbk: per-warp counts
    __shared__ FlatStage stage[kBinWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < kBinWarps * nbk; k += kBinWarps * 32) scnt_all[k] = 0;
    __syncthreads();
    const int64_t nv = *n_visible;
    const int64_t c0 = (int64_t)blockIdx.x * kCtaRanks;
    const int64_t r0 = min(c0 + (int64_t)w * kChunkRanks, nv), r1 = min(r0 + kChunkRanks, nv);
    count_slice(rect_sorted, r0, r1, NB, nbk, scnt_all + w * nbk, lane, stage[w]);
    __syncthreads();
    // per-warp counts (the scatter's intra-chunk offsets) and the chunk totals
    uint32_t *hw = whist + (int64_t)blockIdx.x * kBinWarps * nbk;
    for (int k = threadIdx.x; k < kBinWarps * nbk; k += kBinWarps * 32) hw[k] = scnt_all[k];
    uint32_t *h = hist + (int64_t)blockIdx.x * nbk;
    for (int k = threadIdx.x; k < nbk; k += kBinWarps * 32) {
        uint32_t t = 0;
#pragma unroll
        for (int ww = 0; ww < kBinWarps; ++ww) t += scnt_all[ww * nbk + k];
        h[k] = t;
    }
}

// (2) one kernel, one CTA per bucket k: off[c][k] = sum_{c' < c} hist[c'][k]
// (a block scan down the chunk column) and total[k]; the last CTA to finish
// (atomic ticket, reset for the next frame) scans the totals into
// bucket_start.  The scatter adds bucket_start[k] to its chunk offsets.
constexpr int kOffThreads = 256;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *warp_tot, uint32_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    uint32_t before = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < kOffThreads / 32; ++w) {
        const uint32_t t = warp_tot[w];
        before += w < wid ? t : 0u;
        total += t;
    }
    __syncthreads();
    return before + x - v;
}

__global__ void __launch_bounds__(kOffThreads)
bucket_offsets_kernel(const uint32_t *__restrict__ hist, int G, int nbk, uint32_t *__restrict__ off,
                      uint32_t *__restrict__ total, uint32_t *__restrict__ bstart, uint32_t *__restrict__ ticket) {
    __shared__ uint32_t warp_tot[kOffThreads / 32];
    __shared__ bool last;
    const int k = blockIdx.x;
    const int L = (G + kOffThreads - 1) / kOffThreads;
    const int c0 = min(G, (int)threadIdx.x * L), c1 = min(G, c0 + L);
    uint32_t sum = 0;
    for (int c = c0; c < c1; ++c) sum += hist[(int64_t)c * nbk + k];
    uint32_t col_total;
    uint32_t run = block_excl_scan(sum, warp_tot, col_total);
    for (int c = c0; c < c1; ++c) {
        const uint32_t v = hist[(int64_t)c * nbk + k];
        off[(int64_t)c * nbk + k] = run;
        run += v;
    }
    if (threadIdx.x == 0) {
        total[k] = col_total;
        __threadfence();
        last = atomicAdd(ticket, 1u) == (uint32_t)nbk - 1u;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    uint32_t carry = 0;
    for (int base = 0; base < nbk; base += kOffThreads) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nbk ? __ldcg(total + i) : 0u;
        uint32_t chunk_total;
        const uint32_t ex = block_excl_scan(v, warp_tot, chunk_total);
        if (i < nbk) bstart[i] = carry + ex;
        carry += chunk_total;
    }
    if (threadIdx.x == 0) {
        bstart[nbk] = carry;
        *ticket = 0u;
    }
}

// (3) ordered scatter.  Each warp recounts its 128-rank slice, a scan over
// the 8 warps turns the CTA offsets into per-warp start offsets, then each
// warp walks its slice in the flattened rank-major (rank, bucket) order;
// lanes of one step that hit the same bucket are ranked with
// __match_any_sync, so every bucket's entries come out in rank order.
__global__ void __launch_bounds__(kBinWarps * 32)
bucket_scatter_kernel(const uint32_t *__restrict__ order, const uint64_t *__restrict__ rect_sorted,
                      const uint32_t *__restrict__ n_visible, int G,
                      int NB, int nbk, const uint32_t *__restrict__ off, const uint32_t *__restrict__ bstart,
                      const uint32_t *__restrict__ whist, uint64_t *__restrict__ entries,
                      const unsigned long long *__restrict__ n_pairs, int64_t capacity, uint32_t *status) {
    if (pairs_overflow(n_pairs, capacity, status)) return;
    extern __shared__ uint32_t sfill_all[];  // kBinWarps x nbk
    __shared__ FlatStage stage[kBinWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nv = *n_visible;
    const int64_t c0 = (int64_t)blockIdx.x * kCtaRanks;
    if (c0 >= nv) return;
    const int64_t r0 = min(c0 + (int64_t)w * kChunkRanks, nv), r1 = min(r0 + kChunkRanks, nv);
    uint32_t *sfill = sfill_all + w * nbk;
    // per-warp start offsets: bucket start + chunk offset + earlier warps' counts
    const uint32_t *o = off + (int64_t)blockIdx.x * nbk;
    const uint32_t *hw = whist + (int64_t)blockIdx.x * kBinWarps * nbk;
    for (int k = threadIdx.x; k < nbk; k += kBinWarps * 32) {
        uint32_t run = bstart[k] + o[k];
#pragma unroll
        for (int ww = 0; ww < kBinWarps; ++ww) {
            sfill_all[ww * nbk + k] = run;
            run += hw[ww * nbk + k];
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t rb = r0; rb < r1; rb += 32) {
        const int64_t r = rb + lane;
        uint64_t q = 0;
        uint32_t id = 0;
        bool has = false;
        if (r < r1) {
            id = order[r];
            q = rect_sorted[r];
            has = q != kNoRect;
            if (!has) q = 0;
        }
        FlatStage &st = stage[w];
        const FlatBatch fb = flat_batch(q, has, id, lane, st);
        for (int f0 = 0; f0 < fb.total; f0 += 32) {
            const int f = f0 + lane;
            const bool act = f < fb.total;
            int j, band, grp;
            uint64_t qj;
            const int k = flat_locate(fb, st, act ? f : fb.total - 1, NB, j, qj, band, grp);
            const uint32_t idj = st.id[j];
            const unsigned same = __match_any_sync(0xffffffffu, act ? k : -1);
            const uint32_t base = sfill[act ? k : 0];
            if (act && UBS_GUARD((int64_t)base + __popc(same & lt) < capacity && k < nbk, kChkEntry))
                entries[base + __popc(same & lt)] = bucket_entry(idj, qj, band, grp);
            __syncwarp();
            if (act && (same >> lane) == 1u) sfill[k] = base + __popc(same);  // highest lane of the group
            __syncwarp();
        }
    }
}

// (4) per-tile lists: one CTA per (bucket, tile row), one warp per tile of
// that row (kBand tiles).  Each round stages kListRound bucket entries in
// shared memory once; every warp scans them in order, keeps the entries whose
// tile mask has its bit (warp ballot compaction, so the list stays
// in rank order) and stops once `cap` ids are written: only the prefix of
// each list a tile can consume is materialised.  The round loop ends when
// every warp is done or the bucket is exhausted.
constexpr int kListThreads = kBand * 32;
constexpr int kListRound = 1024;
__global__ void __launch_bounds__(kListThreads)
tile_lists_kernel(const uint64_t *__restrict__ entries, const uint32_t *__restrict__ bstart,
                  const uint32_t *__restrict__ ranges, int TX, int TY, int NB, uint32_t cap,
                  uint32_t *__restrict__ out, const unsigned long long *__restrict__ n_pairs, int64_t capacity) {
    __shared__ uint64_t sbuf[kListRound];
    if (pairs_overflow(n_pairs, capacity, nullptr)) return;
    const int k = blockIdx.x / kRows, ly = blockIdx.x % kRows;
    const int grp = k / NB, band = k - grp * NB;
    const int lane = threadIdx.x & 31, lx = threadIdx.x >> 5;
    const int tx = band * kBand + lx, ty = grp * kRows + ly;
    uint32_t t0 = 0, want = 0;
    if (tx < TX && ty < TY) {
        const int tile = ty * TX + tx;
        t0 = ranges[2 * tile];
        want = min(cap, ranges[2 * tile + 1] - t0);
    }
    const uint32_t tmask = 1u << (ly * kBand + lx);  // this tile's bit in the entry mask (high word)
    uint32_t *dst = out + t0;
    const uint32_t e0 = bstart[k], e1 = bstart[k + 1];
    const unsigned lt = (1u << lane) - 1u;
    uint32_t written = 0;
    for (uint32_t base = e0; base < e1; base += kListRound) {
        if (__syncthreads_count(written < want) == 0) break;
#pragma unroll
        for (int r = 0; r < kListRound / kListThreads; ++r) {  // zero entries pad the round: mask 0 never matches
            const uint32_t i = base + r * kListThreads + threadIdx.x;
            sbuf[r * kListThreads + threadIdx.x] = i < e1 ? entries[i] : 0ull;
        }
        __syncthreads();
        const int m = (int)min((uint32_t)kListRound, e1 - base);
        // 4 x 32 entries per step: independent loads / tests / ballots, then
        // the ordered appends (no bounds test: the round is zero-padded)
        for (int j0 = 0; j0 < m && written < want; j0 += 128) {
            uint32_t idv[4];
            bool p[4];
            unsigned bal[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t e = sbuf[j0 + 32 * u + lane];
                idv[u] = (uint32_t)e;
                p[u] = ((uint32_t)(e >> 32) & tmask) != 0u;
                bal[u] = __ballot_sync(0xffffffffu, p[u]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t pos = written + __popc(bal[u] & lt);
                if (p[u] && pos < want && UBS_GUARD((int64_t)t0 + pos < capacity, kChkList)) dst[pos] = idv[u];
                written += __popc(bal[u]);
            }
        }
    }
}

}  // namespace ubs

using namespace ubs;

// temp: hist (B + 1) | start (B + 1) | CUB scan scratch
static size_t depth_scan_bytes(int64_t n) {
    const int B = 1 << sort_log_buckets(n);
    size_t a = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (const uint32_t *)nullptr, (uint32_t *)nullptr, B + 1);
    return a;
}

extern "C" size_t ubs_bin_temp_bytes(int64_t n, int64_t pair_capacity, int32_t n_tiles) {
    (void)pair_capacity;
    const size_t B = (size_t)1 << sort_log_buckets(n);
    const size_t depth = 2 * ((B + 1) * sizeof(uint32_t) + 256) + depth_scan_bytes(n) + 256;
    const size_t tiles = sizeof(uint32_t) * (size_t)((n_tiles > 0 ? n_tiles : 0) / 1024 + 1);  // large-frame tile scan
    return depth > tiles ? depth : tiles;
}

extern "C" int ubs_bin_depth(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                             ubs_stream_t stream) {
    if (!v || !pb || !bb || !bb->temp || !pb->tile_grid || !bb->tile_ranges) return UBS_E_ARGS;
    const int64_t n = v->n;
    if (n >= (int64_t)1 << 31) return UBS_E_ARGS;
    cudaStream_t s = (cudaStream_t)stream;
    const int TX = (v->cam.width + kTile - 1) / kTile, TY = (v->cam.height + kTile - 1) / kTile;
    const size_t gbytes = sizeof(int32_t) * (size_t)(TX + 1) * (TY + 1);
    if (gbytes <= 200 * 1024) {  // up to ~50k tiles: one CTA in shared memory
        cudaFuncSetAttribute(tile_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gbytes);
        tile_scan_kernel<<<1, kScanThreads, gbytes, s>>>(pb->tile_grid, TX, TY, bb->tile_ranges);
    } else {  // in place in global memory; block sums in the (not yet used) depth-sort scratch
        const int n_tiles = TX * TY, nb = (n_tiles + 1023) / 1024;
        if (bb->temp_bytes < sizeof(uint32_t) * (size_t)nb) return UBS_E_CAPACITY;
        uint32_t *bsum = reinterpret_cast<uint32_t *>(bb->temp);
        int32_t *g = pb->tile_grid;
        grid_row_prefix_kernel<<<(TY + 1 + 7) / 8, 256, 0, s>>>(g, TX + 1, TY + 1);
        grid_col_prefix_kernel<<<(TX + 1 + 255) / 256, 256, 0, s>>>(g, TX + 1, TY + 1);
        tile_block_sums_kernel<<<nb, 1024, 0, s>>>(g, TX, n_tiles, bsum);
        tile_block_scan_kernel<<<1, 1024, 0, s>>>(bsum, nb);
        tile_ranges_kernel<<<nb, 1024, 0, s>>>(g, TX, n_tiles, bsum, bb->tile_ranges);
    }
    if (n == 0) {
        UBS_CUDA_CHECK();
        return UBS_OK;
    }
    const int logB = sort_log_buckets(n);
    const size_t B = (size_t)1 << logB;
    const size_t arr = ((B + 1) * sizeof(uint32_t) + 255) & ~(size_t)255;
    size_t scan_bytes = depth_scan_bytes(n);
    if (bb->temp_bytes < 2 * arr + scan_bytes) return UBS_E_CAPACITY;
    uint32_t *hist = reinterpret_cast<uint32_t *>(bb->temp);
    uint32_t *start = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(bb->temp) + arr);
    void *scan_tmp = reinterpret_cast<char *>(bb->temp) + 2 * arr;
    uint64_t *tkey = reinterpret_cast<uint64_t *>(bb->keys_sorted);
    const int thr = 256;
    const unsigned blocks = (unsigned)((n + thr - 1) / thr);
    if (cudaMemsetAsync(hist, 0, (B + 1) * sizeof(uint32_t), s) != cudaSuccess) return UBS_E_CUDA;
    depth_hist_kernel<<<blocks, thr, 0, s>>>(pb->depth_key, pb->depth_range, n, logB, hist);
    if (cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, hist, start, (int)(B + 1), s) != cudaSuccess)
        return UBS_E_CUDA;
    depth_scatter_kernel<<<blocks, thr, 0, s>>>(pb->depth_key, pb->depth_range, n, logB, start, hist, tkey,
                                                bb->ids_iota);
    if (!bb->rect_sorted) return UBS_E_ARGS;
    depth_rank_kernel<<<blocks, thr, 0, s>>>(pb->depth_range, logB, start, tkey, bb->ids_iota, pb->n_visible,
                                             pb->rect, pb->tile_count, bb->order, bb->rect_sorted);
    UBS_CUDA_CHECK();
    return UBS_OK;
}

extern "C" int ubs_bin_tiles(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                             int64_t n_pairs, ubs_stream_t stream) {
    if (!v || !pb || !bb) return UBS_E_ARGS;
    const int W = v->cam.width, H = v->cam.height;
    const int TX = (W + kTile - 1) / kTile, TY = (H + kTile - 1) / kTile;
    const int NB = (TX + kBand - 1) / kBand, nbk = ((TY + kRows - 1) / kRows) * NB;
    cudaStream_t s = (cudaStream_t)stream;
    if (n_pairs == 0 || v->n == 0) return UBS_OK;
    if (n_pairs > bb->pair_capacity || bb->pair_capacity >= ((int64_t)1 << 32)) return UBS_E_CAPACITY;
    const int G = bb->chunk_count;
    if (G < 1 || !bb->chunk_hist || !bb->entries || !bb->seg_scratch || !bb->bucket_start || !bb->tile_ids)
        return UBS_E_ARGS;
    if ((2 + kBinWarps) * (int64_t)G * nbk > bb->chunk_hist_capacity || (int64_t)nbk + 1 > bb->bucket_capacity)
        return UBS_E_CAPACITY;
    if ((int64_t)G * kCtaRanks < v->n) return UBS_E_ARGS;  // chunk_count must cover n / kCtaRanks
    const size_t cnt_bytes = sizeof(uint32_t) * (size_t)kBinWarps * nbk;
    if (cnt_bytes > 200 * 1024) return UBS_E_ARGS;
    cudaFuncSetAttribute(bucket_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cnt_bytes);
    const unsigned cta = (unsigned)G;
    if (!bb->rect_sorted) return UBS_E_ARGS;
    // chunk_hist: chunk totals (G x nbk) | chunk offsets (G x nbk) | per-warp counts (G x kBinWarps x nbk)
    uint32_t *whist = bb->chunk_hist + 2 * (size_t)G * nbk;
    cudaFuncSetAttribute(bucket_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cnt_bytes);
    bucket_hist_kernel<<<cta, kBinWarps * 32, cnt_bytes, s>>>(bb->rect_sorted, pb->n_visible, G, NB, nbk,
                                                              bb->chunk_hist, whist);
    // seg_scratch: bucket totals (nbk) | ticket (1)
    uint32_t *total = bb->seg_scratch, *ticket = total + nbk;
    uint32_t *off = bb->chunk_hist + (size_t)G * nbk;  // second half of chunk_hist
    if (cudaMemsetAsync(ticket, 0, sizeof(uint32_t), s) != cudaSuccess) return UBS_E_CUDA;
    bucket_offsets_kernel<<<nbk, kOffThreads, 0, s>>>(bb->chunk_hist, G, nbk, off, total, bb->bucket_start, ticket);
    bucket_scatter_kernel<<<cta, kBinWarps * 32, cnt_bytes, s>>>(bb->order, bb->rect_sorted,
                                                                 pb->n_visible, G, NB, nbk, off, bb->bucket_start,
                                                                 whist, bb->entries,
                                                                 pb->n_pairs, bb->pair_capacity, bb->status);
    tile_lists_kernel<<<nbk * kRows, kListThreads, 0, s>>>(bb->entries, bb->bucket_start, bb->tile_ranges, TX, TY, NB,
                                                   bb->list_cap ? bb->list_cap : 0xFFFFFFFFu, bb->tile_ids,
                                                   pb->n_pairs, bb->pair_capacity);
    UBS_CUDA_CHECK();
    return UBS_OK;
}

UBS_CHECKED_ACCESSOR(binning)
