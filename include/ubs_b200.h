/*
 * ubs_b200.h — C ABI of the B200-native Universal Beta Splatting render path.
 *
 * Drop-in boundary for the reference package `betasplat`
 * (/root/reference/pkg/src/betasplat).  The reference has no plugin registry;
 * its boundary is (i) the Python entry points render / render_with_cache /
 * gradients.backward and (ii) the two numba kernels tile_forward /
 * tile_backward, whose ABI is "caller allocates every array, kernel writes
 * outputs in place, returns a plain int".  This header keeps that ownership
 * model at frame granularity on the device:
 *
 *   - every pointer is a caller-owned DEVICE buffer (the Python host layer
 *     allocates them as torch tensors); the library never allocates;
 *   - every call is stream-ordered on the given cudaStream_t, performs no
 *     host synchronisation and keeps no global mutable state (re-entrant per
 *     stream);
 *   - return value 0 = success, negative = UBS_E_* below.
 *
 * Stage map (reference function -> entry point here):
 *   slice_scene + project_scene        slicing.py:185-235, raster.py:95-134
 *                                      -> ubs_scene_statics (query-invariant
 *                                         half, once per parameter version)
 *                                         + ubs_preprocess
 *   order = lexsort((ids, depth))      raster.py:274-275
 *   build_tiles                        raster.py:252-266
 *                                      -> ubs_bin_depth + ubs_bin_tiles
 *   tile_forward over all tiles        _tiles.py:19-56, raster.py:284-316
 *                                      -> ubs_raster_forward (+ ubs_raster_fixup)
 *   L1 + ssim_and_grad -> g_image      gradients.py:110-116, metrics.py:74-114
 *                                      -> ubs_loss_image_grad
 *   tile_backward + np.add.at scatter  _tiles.py:59-127, gradients.py:142-173
 *                                      -> ubs_raster_backward
 *   _projection_backward/_slice_backward/_clamp_eig_adjoint + regularisers
 *                                      gradients.py:120-123,179-300
 *                                      -> ubs_prim_backward
 *
 * Primitive layout: the UBS1 record (sceneio.py:3-11) — n rows of 14+6C
 * floats (f32, or f64 when param_f64 = 1) in PARAM_FIELDS order
 * (scene.py:17-28): mu_x[3] mu_q[C] rot[3] s_x_raw[3] l_qx[C*3] s_q_raw[C]
 * b_x b_q[C] opacity_raw color[3].  Parameter gradients use the same layout.
 */
#ifndef UBS_B200_H
#define UBS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *ubs_stream_t; /* == cudaStream_t */

#define UBS_ABI_VERSION 7
#define UBS_TILE 16

enum {
    UBS_OK = 0,
    UBS_E_ARGS = -1,      /* bad argument (null pointer, unsupported n_dims/tile size) */
    UBS_E_CUDA = -2,      /* a CUDA launch or CUB call failed */
    UBS_E_CAPACITY = -3,  /* caller-provided pair / temp capacity too small */
};

/* flag bits in UbsPrimBuffers.flags (16 bits per primitive) */
enum {
    UBS_F_VISIBLE = 1,      /* ProjectionCache.visible (raster.py:131) */
    UBS_F_DEGENERATE = 2,   /* ~SliceCache.valid (covariance.py:122-149) */
    UBS_F_FLOOR3 = 4,       /* SliceCache.floored (slicing.py:215) */
    UBS_F_FLOOR2 = 8,       /* ProjectionCache.floored (raster.py:116) */
    UBS_F_THIN = 16,        /* fp32 raster guard: pixels touching this splat are re-done in fp64 */
    UBS_F_GATE_SAT = 32,    /* some d_gate == 1: the gate adjoint is 0 * inf (NaN), gradients.py:225-226 */
};

/* device status bits (UbsBinBuffers.status) */
enum {
    UBS_S_PAIR_OVERFLOW = 1, /* K exceeded the pair capacity */
    UBS_S_LIST_TRUNC = 2,    /* a tile exhausted its capped list with unsaturated pixels */
};

/* Camera (camera.py:15-51): intrinsics + rigid world_to_cam. */
typedef struct UbsCamera {
    double fx, fy, cx, cy;
    double rot[9];   /* world_to_cam[:3,:3], row-major */
    double trans[3]; /* world_to_cam[:3, 3] */
    int32_t width, height;
} UbsCamera;

/* RenderSettings (config.py:9-38); tile_size must be 16. */
typedef struct UbsSettings {
    double tau_sq, alpha_clamp, transmittance_min, near_plane, cull_margin;
    double screen_cov_floor, psd_floor_scale;
    int32_t gate_symmetric, tile_size;
} UbsSettings;

/* One frame = scene + camera + query (slicing.py:36-77: [], [d], or [t, d]). */
typedef struct UbsView {
    const void *params;   /* n x (14+6C) device records */
    int64_t n;
    int32_t n_dims;       /* 3, 6 or 7 */
    int32_t param_f64;    /* 0: f32 records, 1: f64 records */
    double background[3];
    double query[4];
    UbsCamera cam;
    UbsSettings set;
    /* Optional scene statics from ubs_scene_statics for these params and
     * settings.psd_floor_scale (NULL: ubs_preprocess derives them inline). */
    const void *statics;
} UbsView;

/* Per-primitive preprocess outputs (all length n unless noted). */
typedef struct UbsPrimBuffers {
    uint64_t *depth_key;   /* f64 depth bits when visible, else UINT64 sentinel */
    uint64_t *rect;        /* tile rect packed tx0 | ty0<<16 | tx1<<32 | ty1<<48 */
    uint32_t *tile_count;  /* tiles touched (0 if not visible) */
    uint16_t *flags;       /* UBS_F_* | (s_tanh[k] > 0) << (8 + k), k < C (FrameCache.trace_signature) */
    void *rec32;           /* n x 48 B fp32 raster records (may be NULL in fp64 mode) */
    void *rec64;           /* n x 80 B fp64 raster records */
    double *debug;         /* optional n x UBS_DEBUG_STRIDE f64 dump of intermediates, or NULL */
    uint32_t *n_visible;   /* [1] += number of visible primitives (caller zeroes) */
    unsigned long long *n_pairs; /* [1] += total tile pairs K (caller zeroes) */
    int32_t *tile_grid;    /* (TY+1) x (TX+1) 2D difference array of rect corners (zeroed by ubs_preprocess) */
    unsigned long long *depth_range; /* [2] min / max visible depth key (initialised by ubs_preprocess) */
} UbsPrimBuffers;

/* debug row (FrameCache.slices / .proj: SliceCache slicing.py:153-182, ProjectionCache raster.py:46-60):
 * 0 depth | 1-2 mean2 | 3-5 p2 00,01,11 | 6-7 radii | 8 gated opacity | 9 beta_x |
 * 10-12 cov2 00,01,11 | 13-18 cov3 xx,xy,xz,yy,yz,zz | 19-21 t_cam | 22-24 mean3 | 25 gate |
 * 26 opacity | 27-30 s_tanh[4] | 31 floor_eps | then the offsets below (C-sized fields hold 4 slots,
 * matrices row-major; eigenvalues ascending, eigenvectors as columns, up to sign).  The query-
 * invariant fields (l_x, rotation, s_x, s_q, cov3 eigen pair) are filled only when the view has
 * no statics (flags bit 16). */
#define UBS_DEBUG_VMAT 32       /* (2, 3) jacobian @ rotation */
#define UBS_DEBUG_COV2_EIG 38   /* eigval[2], eigvec (2, 2) of the pre-floor cov2 */
#define UBS_DEBUG_COV3_EIG 44   /* eigval[3], eigvec (3, 3) of the symmetrised pre-floor cov3 */
#define UBS_DEBUG_BETA_Q 56
#define UBS_DEBUG_DELTA 60
#define UBS_DEBUG_M_INV 64      /* (4, 4) */
#define UBS_DEBUG_U 80
#define UBS_DEBUG_V 84
#define UBS_DEBUG_SIGMA_XQ 88   /* (3, 4) */
#define UBS_DEBUG_D_RAW 100
#define UBS_DEBUG_D_GATE 104
#define UBS_DEBUG_LX 108        /* (3, 3) */
#define UBS_DEBUG_ROT 117       /* (3, 3) */
#define UBS_DEBUG_SX 126
#define UBS_DEBUG_SQ 129
#define UBS_DEBUG_COLOR 133
#define UBS_DEBUG_FLAGS 136     /* 1 valid | 2 floored3 | 4 floored2 | 8 visible | 16 inline route */
#define UBS_DEBUG_STRIDE 144

/* Binning buffers. */
typedef struct UbsBinBuffers {
    uint64_t *keys_sorted; /* n x 8 B scratch: depth keys scattered into their sort buckets */
    uint32_t *ids_iota;    /* n: scratch (ids scattered alongside) */
    uint32_t *order;       /* n: ids by (depth, id); first n_vis are visible */
    uint32_t *tile_ids;    /* pair_capacity: primitive ids grouped by tile, depth ordered */
    uint32_t *tile_ranges; /* 2 x n_tiles: [start, end) into tile_ids */
    int64_t pair_capacity;
    void *temp;            /* ubs_bin_temp_bytes: depth-bucket histogram, starts, CUB scan scratch */
    size_t temp_bytes;
    uint32_t *chunk_hist;  /* 10 x chunk_count x n_buckets: per-chunk bucket counts, chunk offsets, then the
                              per-warp counts of each chunk (8 warps) */
    int64_t chunk_hist_capacity; /* elements */
    int32_t chunk_count;   /* G rank chunks */
    uint64_t *entries;     /* pair_capacity: bucket entries (id | covered-tile mask of the 8 x 4
                              tile bucket << 32) */
    uint32_t *seg_scratch; /* n_buckets + 1: bucket totals, completion ticket */
    uint32_t *bucket_start;/* n_buckets + 1 */
    int64_t bucket_capacity; /* elements of bucket_start */
    uint32_t *status;      /* [1] |= UBS_S_* (frame must be re-run with more capacity) */
    uint32_t list_cap;     /* per-tile list cap: only the first list_cap ids of each tile are
                              materialised (0xFFFFFFFF = full lists).  Tiles saturate long before
                              their lists end; a raster CTA that runs out of a capped list with
                              unsaturated pixels sets UBS_S_LIST_TRUNC. */
    uint64_t *rect_sorted; /* n: tile rects in depth order (written by ubs_bin_depth; all-ones when the
                              primitive touches no tile), read coalesced by the level-1 binning */
} UbsBinBuffers;

/* Forward outputs.  Image/alpha/T are f32, or f64 in the fp64 raster. */
typedef struct UbsImageBuffers {
    void *image;        /* H x W x 3 */
    void *alpha_sum;    /* H x W */
    void *t_stop;       /* H x W */
    int32_t *n_contrib; /* H x W: splats iterated before the early-out */
    uint8_t *hit_clamp; /* n: FrameCache.alpha_clamped */
    unsigned long long *visits; /* [1]: processed_pixels total */
    uint32_t *fix_list;  /* H*W capacity: pixels re-done in fp64 (fp32 raster only) */
    uint32_t *fix_count; /* [1] */
    int32_t raster_f64;  /* 1 = fp64 raster, 0 = fp32 raster + fp64 fix-up */
    int32_t raster_scalar; /* fp32 raster kernels: 0 = packed fp32x2 (two pixels per lane, default),
                              1 = one pixel per lane; the same per-pixel arithmetic and results */
} UbsImageBuffers;

/* Backward buffers. */
typedef struct UbsGradBuffers {
    const void *g_image; /* H x W x 3 dL/dimage (same float type as the image) */
    void *grad2d;        /* n x 12 accumulators of per-pixel raw moments, h = g_alpha alpha / (1 - m/tau):
                            sum h dx, sum h dy, sum h dx dx, sum h dx dy, sum h dy dy, sum g_alpha alpha,
                            sum g_alpha alpha ln(1 - m/tau), g_color[3], pad[2]; ubs_prim_backward
                            applies the per-primitive factors (-2 P, -beta/tau, 1/og) and consumes
                            the sums: it leaves the buffer all-zero for the next raster backward
                            (which adds into it; the caller zeroes it once before first use) */
    void *grad_params;   /* n x (14+6C) += parameter gradients (f32, or f64 if grad_f64) */
    int32_t grad_f64;
    int32_t grad2d_f64;  /* grad2d accumulators are f64 (must equal UbsImageBuffers.raster_f64) */
    double reg_opacity;  /* loss_scale * lambda_o   (0 to skip, gradients.py:120-123) */
    double reg_scale;    /* loss_scale * lambda_sigma */
    uint32_t *nonfinite; /* [1] set to 1 when any gradient is not finite */
    const uint16_t *flags; /* UbsPrimBuffers.flags of this view (for the skip test), or NULL */
    uint32_t *active;    /* n scratch: primitives the chain must visit, or NULL (visit all) */
    uint32_t *active_count; /* [1] scratch counter */
    int32_t bwd_pixels_per_lane; /* fp32 raster backward layout: 0 or 4 = four pixels per lane as two
                                    packed fp32x2 pairs (fastest), 2 = two pixels per lane, 8 = one warp
                                    per tile (one warp reduction per (tile, splat)); same results up to
                                    the order of the float atomics */
    /* Deterministic mode (raster.py:1-8, gradients.py:164-173: bit-identical gradients run to run):
     * one warp per tile writes each splat's tile partial to a slot of its own (primitive i owns
     * det_slot_off[i] .. + tile_count[i], its rect's tiles in row-major order) and every primitive
     * adds its partials in slot order -- no float atomics.  Needs det_capacity >= K slots of 10
     * floats (f64 for the fp64 raster) and det_temp of ubs_det_temp_bytes(n) bytes. */
    int32_t deterministic;
    uint32_t *det_slot_off; /* n: exclusive prefix of tile_count */
    void *det_partials;     /* det_capacity x 10 */
    int64_t det_capacity;
    void *det_temp;
    size_t det_temp_bytes;
} UbsGradBuffers;

/* --- entry points --- */
int ubs_abi_version(void);
const char *ubs_build_info(void);

/* Query-invariant half of slice_scene (slicing.py:185-235 minus the
 * conditional mean and gate): activations, Sx, the query-block inverse, Sxq,
 * conditional covariance with its PSD floor, opacity, beta_x.  Written to a
 * caller buffer of ubs_statics_bytes(n, n_dims, param_f64) bytes; valid while
 * params and settings.psd_floor_scale are unchanged.  Set UbsView.statics to
 * it and ubs_preprocess only runs the per-view half (same bits either way). */
size_t ubs_statics_bytes(int64_t n, int32_t n_dims, int32_t param_f64);
int ubs_scene_statics(const UbsView *v, void *statics, ubs_stream_t s);

/* slice + project + tile rects (fp64 arithmetic, one thread per primitive) */
int ubs_preprocess(const UbsView *v, const UbsPrimBuffers *pb, int32_t want_rec32, ubs_stream_t s);

/* ubs_preprocess for n_views views of ONE scene (same params, statics, n,
 * n_dims, settings; cameras and queries differ), each into its own
 * UbsPrimBuffers: the scene statics (required) are read once per
 * UBS_MAX_VIEWS views instead of once per view.  Outputs are bit-identical
 * to n_views ubs_preprocess calls.  The same reference functions as
 * ubs_preprocess (slicing.py:185-235, raster.py:95-134, raster.py:252-266),
 * applied to a batch of frames (a sweep or a training batch). */
#define UBS_MAX_VIEWS 8
int ubs_preprocess_views(const UbsView *views, const UbsPrimBuffers *pbs, int32_t n_views, int32_t want_rec32,
                         ubs_stream_t s);

/* scratch bytes (UbsBinBuffers.temp) needed for n primitives */
size_t ubs_bin_temp_bytes(int64_t n, int64_t pair_capacity, int32_t n_tiles);
/* depth order = lexsort((ids, depth)) (raster.py:274-275): bucket sort of the
 * visible primitives on the top bits of (depth bits - min) >> shift, then an
 * exact rank by (f64 depth bits, id) inside each bucket; plus the per-tile
 * [start, end) ranges from the rect-corner difference array */
int ubs_bin_depth(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb, ubs_stream_t s);
/* per-tile depth-ordered id lists (sort-free two-level stable bucketing over
 * buckets of 8 x 4 tiles); n_buckets = ceil(TY / 4) * ceil(TX / 8).
 * n_pairs >= 0: K as read by the host
 * (checked against pair_capacity); n_pairs < 0: K stays on the device, every
 * kernel that touches the pair buffers checks it against pair_capacity and
 * sets UBS_S_PAIR_OVERFLOW instead of writing out of bounds (no host sync). */
int ubs_bin_tiles(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                  int64_t n_pairs, ubs_stream_t s);

/* front-to-back composite, one 16x16 tile per CTA */
int ubs_raster_forward(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                       const UbsImageBuffers *ib, ubs_stream_t s);

/* fp64 replay of the pixels the fp32 raster flagged (no-op for the fp64 raster) */
int ubs_raster_fixup(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                     const UbsImageBuffers *ib, ubs_stream_t s);

/* L1 + SSIM image gradient; loss_parts[0] += sum|diff|, loss_parts[1] += sum ssim_map */
int ubs_loss_image_grad(const void *image, const void *target, int32_t height, int32_t width,
                        int32_t f64, double lambda_ssim, double scale, void *g_image,
                        double *loss_parts, void *scratch, ubs_stream_t s);
size_t ubs_loss_scratch_bytes(int32_t height, int32_t width, int32_t f64);

/* reverse replay of the blend -> per-primitive 2D gradients (grad2d, +=) */
size_t ubs_det_temp_bytes(int64_t n); /* UbsGradBuffers.det_temp bytes for n primitives */
int ubs_raster_backward(const UbsView *v, const UbsPrimBuffers *pb, const UbsBinBuffers *bb,
                        const UbsImageBuffers *ib, const UbsGradBuffers *gb, ubs_stream_t s);

/* chain 2D gradients back to raw parameters (fp64), += into grad_params.
 * With gb->active set, only primitives with a nonzero screen-space gradient
 * or a saturated gate are visited (the chain of an all-zero 2D gradient is
 * exactly zero otherwise, gradients.py:179-280). */
int ubs_prim_backward(const UbsView *v, const UbsGradBuffers *gb, int32_t add_regularisers, ubs_stream_t s);

/* --- training-step epilogue (optim.py:115-135, gradients.py:120-123) --- */

/* Adam on the flat n x (14+6C) record buffer; lr_group = {position, opacity,
 * scale, other}; b_x/b_q clamped to [-5, 5]; m, v are f32 moments (zeroed by
 * the caller before step 1); step is the 1-based Adam step count. */
int ubs_adam_step(void *params, int32_t param_f64, const void *grads, int32_t grad_f64, float *m, float *v,
                  int64_t n, int32_t n_dims, const double *lr_group, int32_t step, int32_t freeze_shapes,
                  ubs_stream_t s);

/* ubs_adam_step, then grads overwritten with the next step's starting
 * gradient: the regulariser gradient of the updated parameters scaled by
 * next_reg_opacity / next_reg_scale (exactly what zeroing the buffer and
 * ubs_add_regularisers would leave; pass 0, 0 for zeros), and, when
 * next_reg_sums is not NULL, the updated parameters' regulariser sums added
 * into it as ubs_regulariser_value does.  One pass instead of four (Adam,
 * zero, regularisers, value) between two training steps. */
int ubs_adam_step_regularised(void *params, int32_t param_f64, void *grads, int32_t grad_f64, float *m, float *v,
                              int64_t n, int32_t n_dims, const double *lr_group, int32_t step,
                              int32_t freeze_shapes, double next_reg_opacity, double next_reg_scale,
                              double *next_reg_sums, ubs_stream_t s);

/* regulariser gradients, once per step (also fused into ubs_prim_backward) */
int ubs_add_regularisers(const void *params, int32_t param_f64, void *grads, int32_t grad_f64, int64_t n,
                         int32_t n_dims, double reg_opacity, double reg_scale, ubs_stream_t s);

/* regulariser value (gradients.py:120-123): sums[0] += sum sigmoid(opacity_raw),
 * sums[1] += sum exp(s_x_raw) + sum exp(s_q_raw), fp64; the caller zeroes sums
 * and forms lambda_o sums[0] + lambda_sigma sums[1] */
int ubs_regulariser_value(const void *params, int32_t param_f64, int64_t n, int32_t n_dims, double *sums,
                          ubs_stream_t s);

#ifdef __cplusplus
}
#endif
#endif /* UBS_B200_H */
