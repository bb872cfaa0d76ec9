/*
 * ta.h -- C ABI of the B200-native latent-Gaussian rasterizer (Tele-Aloha, arXiv 2405.14866).
 *
 * The two calls follow the paper's statement of the problem (PAPER.md = /root/reference/PAPER.md):
 *
 *   ta_unproject : foreground source pixels -> latent Gaussians {x, f, s, alpha}
 *                  PAPER.md l.374 "each point p_i is characterized by four properties:
 *                  position x_i, latent appearance feature f_i, scale s_i, opacity alpha_i.
 *                  The rotation of Gaussian points is set to an identity matrix";
 *                  l.376 "Given camera parameters Pi, 3D positions x of Gaussian points can be
 *                  unprojected from depth maps"; l.358 disparity maps "converted to depth maps";
 *                  l.385 "foreground pixels in source views ... are lifted to pixel-aligned
 *                  Gaussian points {G}".
 *   ta_rasterize : F_novel = R_G({G}, Pi_novel), the Gaussian
 *                  splatting rasterizer of [kerbl20233d]: EWA projection, screen tiles,
 *                  (tile, depth, index) order, front-to-back alpha compositing of the
 *                  C-channel latent feature, plus the accumulated alpha.
 *
 * Every constant the paper leaves to [kerbl20233d] and every arithmetic step is fixed in
 * DESIGN.md ("Readings" R1-R18, "Normative arithmetic"); results match the CPU oracle
 * (oracle/) bit-exactly for tile lists, order and alpha, and within 1e-4 for features.
 *
 * Conventions.  All buffer pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 * unless stated otherwise; the caller owns every input and output buffer; the context owns
 * grow-only scratch.  `stream` is a cudaStream_t (CUstream) passed as void* (NULL = legacy
 * default stream); every call is stream-ordered and asynchronous unless stated.  Cameras use
 * OpenCV axes (x right, y down, z forward), world->camera extrinsics X_c = R X_w + t with R
 * row-major, pixel (x, y) at integer coordinates = pixel centre (R1).  Images are row-major
 * [H][W]; feature images are HWC (channels last).  Thread safety: one context per host thread
 * / stream; ta_gaussians is read-only inside ta_rasterize.
 *
 * Errors.  Every call returns a ta_status; on failure nothing was enqueued unless the status
 * is TA_ERR_CUDA, and ta_last_error() holds a message.  Invalid pixels (mask 0, non-finite or
 * d <= d_min, NaN opacity) are skipped, not errors.
 */
#ifndef TA_H_
#define TA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ta_context ta_context;   /* opaque: device, scratch, last-call debug info */

typedef enum {
    TA_OK = 0,
    TA_ERR_INVALID_ARG = 1,    /* NULL required pointer, bad size, non-finite / non-orthonormal camera */
    TA_ERR_UNSUPPORTED = 2,    /* C not in {8, 16, 32, 64}, unknown dtype, > TA_MAX_VIEWS views */
    TA_ERR_CUDA = 3,           /* a CUDA runtime error (message in ta_last_error) */
    TA_ERR_OUT_OF_MEMORY = 4,  /* scratch growth failed */
    TA_ERR_CAPACITY = 5        /* output Gaussian capacity < sum of view pixels, > 2^28 Gaussians rasterized,
                                  > 2^32-1 tile entries, or (TA_FLAG_ASYNC) reserved entry capacity exceeded */
} ta_status;

typedef enum { TA_F32 = 0, TA_F16 = 1 } ta_dtype;

#define TA_MAX_VIEWS 16
#define TA_TILE 16             /* screen tiles are 16 x 16 pixels ([kerbl20233d]); opt-in 8 x 8 compositing tiles
                                  (environment TA_TILE_PX=8 at context creation, 32 x 32 coarse bins only) are
                                  reported in ta_debug_view.tile_px.  The tile size never changes a result: a
                                  pixel composites every Gaussian whose box holds it, in (depth, id) order */

typedef struct { float fx, fy, cx, cy; } ta_intrinsics;        /* pixels; fx, fy > 0 */
typedef struct { float R[9]; float t[3]; } ta_extrinsics;      /* world -> camera; R orthonormal (1e-4) */

/* One source view (device pointers, row-major [H][W][...]). */
typedef struct {
    int32_t H, W;                /* 1 <= H, W <= 32767 */
    const float* disparity;      /* [H][W] pixels; lifted iff mask != 0, isfinite(d), d > d_min */
    const uint8_t* mask;         /* [H][W] foreground mask, or NULL = all foreground */
    ta_intrinsics K;
    ta_extrinsics RT;
    float baseline;              /* metres, > 0: depth z = fx * baseline / d (R2) */
    const float* scale;          /* [H][W][3] metres, or NULL = params->default_scale (isotropic) */
    const float* quat;           /* [H][W][4] (w,x,y,z), normalised on use; NULL = identity (l.374) */
    const float* opacity;        /* [H][W], clamped to [0,1]; NULL = params->default_opacity */
    const void* feat;            /* [H][W][C] latent feature map M_f, element type = out->feat_dtype */
} ta_source_view;

/*
 * Gaussian set, caller-allocated structure of arrays (16-byte aligned device buffers).
 * Gaussian i (0 <= i < n):
 *   pos_alpha[4*i .. 4*i+3] = world x, y, z, opacity alpha
 *   cov[8*i .. 8*i+7]       = world covariance s00 s01 s02 s11 s12 s22 (Sigma_w = R_q diag(s^2) R_q^T),
 *                             id (uint32 bit pattern), 0
 *   feat[C*i .. C*i+C-1]    = latent feature (feat_dtype)
 * ids must be a permutation of 0..n-1 (ta_unproject writes id = i: view-major, row-major order);
 * the depth tie-break is by id, so permuting the arrays leaves ta_rasterize's output unchanged.
 */
typedef struct {
    int64_t capacity;            /* Gaussians the arrays can hold */
    int64_t* n_dev;              /* device int64: count written by ta_unproject (may be NULL for rasterize
                                    when n >= 0 is passed) */
    float* pos_alpha;            /* [capacity][4] */
    float* cov;                  /* [capacity][8] */
    void* feat;                  /* [capacity][C] */
    int32_t C;                   /* 8, 16, 32 or 64 */
    ta_dtype feat_dtype;
} ta_gaussians;

/* Rasterizer constants (readings R7-R14); ta_default_params() fills the defaults. */
typedef struct {
    float dilation;              /* 0.3 px^2 added to the diagonal of Sigma' (R7) */
    float alpha_max;             /* 0.99 clamp of alpha' (R9) */
    float alpha_min;             /* 1/255: alpha' below it is skipped (R9) */
    float t_eps;                 /* 1e-4: stop before T would drop below it (R10) */
    float cull_sigma;            /* 3: q <= cull_sigma^2 and the cull_sigma-sigma box (R8); (0, 12] */
    float z_near;                /* 0.01 m (R14) */
    float d_min;                 /* 0: lift iff d > d_min */
    float default_scale;         /* used when a view has no scale map */
    float default_opacity;       /* used when a view has no opacity map */
    uint32_t flags;              /* TA_FLAG_* */
    int32_t exact_exp;           /* 1 (default): exp by the fixed fp32 sequence exp_det (R13), identical to the
                                    oracle, so every decision and A are bit-exact.  0: the opt-in fast mode --
                                    the compositor evaluates exp(-q/2) with the SFU (ex2.approx of the same
                                    staged argument times log2 e); alpha' may then differ by a few ulp, which
                                    can move a stop decision (parity reported separately: test_gpu_fast_exp) */
} ta_raster_params;

/* ta_rasterize does not synchronise with the host.  Scratch must already be large enough
   (ta_reserve, or an earlier synchronous call of at least the same size); if the tile-entry
   count exceeds the reserved capacity the output is undefined and ta_check_overflow reports it. */
#define TA_FLAG_ASYNC 1u
/* Write per-pixel composited-pair counts (ta_debug_view.n_contrib) -- test/debug builds of a call. */
#define TA_FLAG_DEBUG_COUNTS 2u

void ta_default_params(ta_raster_params* p);

/* Create a context on CUDA device `device` (makes it current on the calling thread). */
ta_status ta_context_create(int32_t device, ta_context** out);
ta_status ta_context_destroy(ta_context* ctx);

/* Grow scratch for up to `max_gaussians` Gaussians, `max_entries` (coarse bin, Gaussian) pairs
   (ta_debug_view.Kc of a representative call) and an H x W target (synchronous: allocation).
   Needed before TA_FLAG_ASYNC calls / graph capture. */
ta_status ta_reserve(ta_context* ctx, int64_t max_gaussians, int64_t max_entries, int32_t H, int32_t W);

/*
 * a1 -- lift the foreground pixels of V source views into `out`.
 * Gaussians are written in view order, pixels row-major, ids 0..n-1; *out->n_dev = n.
 * Requires out->capacity >= sum_v H_v*W_v (TA_ERR_CAPACITY), 1 <= V <= TA_MAX_VIEWS.
 * Reads params->d_min, default_scale, default_opacity.
 */
ta_status ta_unproject(ta_context* ctx, const ta_source_view* views, int32_t V,
                       const ta_raster_params* params, ta_gaussians* out, void* stream);

/*
 * a2-a6 -- render the Gaussian set into target camera (K_tgt, RT_tgt), H x W pixels
 * (PAPER.md l.386 F_novel = R_G({G}, Pi_novel)).
 *   n          number of Gaussians, or -1 to use the device count *g->n_dev (no host read).
 *   feat_out   device float [H][W][C] (HWC), alpha_out device float [H][W]: written for every pixel
 *              (F = 0, A = 0 where nothing contributes).
 *   K_tgt, RT_tgt are host structs.  Without TA_FLAG_ASYNC the call reads the tile-entry count
 *   back to the host once (stream synchronisation) to size scratch.
 */
ta_status ta_rasterize(ta_context* ctx, const ta_gaussians* g, int64_t n, const ta_intrinsics* K_tgt,
                       const ta_extrinsics* RT_tgt, int32_t H, int32_t W, const ta_raster_params* params,
                       float* feat_out, float* alpha_out, void* stream);

/*
 * The multi-view display workload (the autostereoscopic screen shows every view
 * from leftmost to rightmost): one Gaussian set rendered into T targets, all H x W, in one
 * call.  Equivalent to T calls of ta_rasterize (identical output bits) but the targets are spread
 * round-robin over `lanes` (1..4) lanes: lane 0 = ctx on `stream`, lanes 1.. = child contexts (own
 * scratch) on child streams owned by ctx, forked from and joined back into `stream`, so one target's
 * projection / sort / binning overlaps another's compositing.  ta_reserve on ctx also sizes the child
 * contexts (needed for TA_FLAG_ASYNC).  K_tgt, RT_tgt: host arrays of T; feat_out, alpha_out: host
 * arrays of T device pointers.  ta_debug_last describes the last target of lane 0.  Errors as
 * ta_rasterize; T < 1 or lanes outside [1, 4] is TA_ERR_INVALID_ARG.
 */
ta_status ta_rasterize_views(ta_context* ctx, const ta_gaussians* g, int64_t n, int32_t T, const ta_intrinsics* K_tgt,
                             const ta_extrinsics* RT_tgt, int32_t H, int32_t W, const ta_raster_params* params,
                             float* const* feat_out, float* const* alpha_out, int32_t lanes, void* stream);

/*
 * north_star (a) -- the fused front end: lift the foreground pixels of V source views (a1), project and
 * cull them for T targets (a2) in ONE pass over the source maps (128-bit loads), then bin, sort and
 * composite each target (a3-a6) exactly as ta_rasterize does.  Equivalent to ta_unproject followed by
 * ta_rasterize(n = -1) per target -- same ids (view-major, row-major compaction), same records, same
 * output bits -- but the Gaussians' world position / covariance (48 B each) are never written to or
 * re-read from memory; only the feature rows are compacted (the compositor's operand).  Use it when few
 * targets are rendered per frame (a single view, the paper's two eyes); for many targets per frame
 * (the 32-view display) ta_unproject once + ta_rasterize per view moves fewer bytes.
 *   views / V / params  as ta_unproject (C, feat_dtype describe the views' feature maps)
 *   T                   1 <= T <= 4 targets, all H x W
 *   K_tgt, RT_tgt       host arrays of T cameras
 *   feat_out, alpha_out host arrays of T device pointers: float [H][W][C] (16-byte aligned), float [H][W]
 * Scratch (context-owned, grow-only): sum_v H_v W_v x (C x feature bytes + T x 40 B); targets 1..T-1 run
 * their sort / bin / composite chains on child contexts and streams owned by ctx, concurrently with
 * target 0, and the call completes on `stream`.  ta_debug_last describes target 0.  Errors as
 * ta_unproject + ta_rasterize; T outside [1, 4] is TA_ERR_INVALID_ARG.
 */
ta_status ta_render_sources(ta_context* ctx, const ta_source_view* views, int32_t V, int32_t C, ta_dtype feat_dtype,
                            const ta_raster_params* params, int32_t T, const ta_intrinsics* K_tgt,
                            const ta_extrinsics* RT_tgt, int32_t H, int32_t W, float* const* feat_out,
                            float* const* alpha_out, void* stream);

/*
 * cascade depth initialisation (cam0's disparity "is
 * converted to a depth map and then lifted to a 3D point cloud.  These points are rasterized to the
 * viewpoints of cam2 and cam3.  Z-buffers are extracted and converted back to disparity maps";
 * SPEC.md l.86-94 points_zbuffer; reading R23).
 * Every valid pixel (mask != 0, finite d > params->d_min) of the V source views is lifted (a1
 * arithmetic, opacity / scale / features ignored), projected into (K_tgt, RT_tgt) (a2 arithmetic,
 * culled unless z > params->z_near) and splatted to the (2 r + 1)^2 pixels around its nearest pixel
 * (rint of the pixel centre, ties to even) with r = splat_radius in [0, 8].  Each target pixel keeps
 * the point of minimum camera-space z, ties to the lowest source index (running pixel index over the
 * views, view-major, row-major) -- independent of execution order.
 *   depth_out  device float [H][W]: that z, 0 where no point lands (required)
 *   disp_out   device float [H][W] or NULL: fx_tgt * baseline_tgt / z, 0 where no point lands
 *              (the d_init of the lower pair; baseline_tgt > 0 required when disp_out != NULL)
 * Scratch: one 64-bit z-buffer word per target pixel (context-owned, grown on demand).
 * Errors: TA_ERR_INVALID_ARG for NULL depth_out / views, bad sizes, radius outside [0, 8],
 * non-finite or non-orthonormal cameras, baseline_tgt <= 0 with disp_out.
 */
ta_status ta_zbuffer(ta_context* ctx, const ta_source_view* views, int32_t V, const ta_raster_params* params,
                     const ta_intrinsics* K_tgt, const ta_extrinsics* RT_tgt, int32_t H, int32_t W,
                     int32_t splat_radius, float baseline_tgt, float* depth_out, float* disp_out, void* stream);

/*
 * occlusion-aware input-view blending (Eqs. 6-10;
 * DESIGN.md reading R24).  For every pixel (u, v) of the novel camera (K_tgt, RT_tgt, H x W) with
 * z_fused > 0 (device float [H][W], e.g. ta_zbuffer of all input views into the novel camera):
 * lift (Eq. 6), project into each of the V input views, sample colour and depth bilinearly (Eq. 7),
 * weight w_i = M_i * Occ * cos<r, n_i> / ||x_i^cam|| (Eqs. 8-9) and write
 * I_blend = sum w_i c_i / sum w_i (Eq. 10); sum w_i < w_min leaves a hole (colour 0).
 *   views      the input views: disparity (z = fx*B/d), mask, K, RT, baseline are read
 *   colors     host array of V device pointers, view i's colour image float [H_i][W_i][3]
 *   rgb_out    device float [H][W][3];  wsum_out  device float [H][W] (the denominator) or NULL
 * Reads params->d_min, z_near.  Errors: TA_ERR_INVALID_ARG for NULL pointers, bad sizes, bad cameras,
 * delta <= 0, edge_tau <= 0, w_min < 0, tau_c < 0.
 */
typedef struct {
    float delta;       /* Eq. 9 SDF threshold (m), default 0.01 */
    float edge_tau;    /* edge mask: max central depth gradient (m / px), default 0.02 */
    float w_min;       /* hole threshold on sum w_i (a pixel with sum w_i = 0 is always a hole), default 1e-4 */
    float tau_c;       /* appearance-consistency mask (l.430-433 names it; SPEC.md l.331's reading, DESIGN.md
                          R24): a sample is kept iff its colour is within tau_c (linear RGB distance) of the
                          pixel's weighted median sample (the medoid minimising sum_j w_j |c_j - c_i|);
                          default 0.15, 0 = mask off */
} ta_blend_params;
void ta_default_blend_params(ta_blend_params* bp);
ta_status ta_blend(ta_context* ctx, const ta_source_view* views, int32_t V, const float* const* colors,
                   const ta_raster_params* params, const ta_blend_params* bp, const ta_intrinsics* K_tgt,
                   const ta_extrinsics* RT_tgt, int32_t H, int32_t W, const float* z_fused, float* rgb_out,
                   float* wsum_out, void* stream);

/*
 * backward pass of the compositing step (the
 * differentiable rasterizer of [kerbl20233d]; reading R25).  Gradients of
 * L = sum_p grad_F(p) . F(p) + grad_A(p) A(p) with respect to each Gaussian's 2D splat parameters,
 * with the per-pixel decisions (box, q <= cull_sigma^2, alpha' >= alpha_min, the stop) held fixed and
 * no gradient through a binding alpha clamp.  Must follow the ta_rasterize of the same Gaussian set,
 * n, camera, size and params on the same context (it reuses that call's splat records and tile lists).
 *   grad_F  device float [H][W][C], grad_A device float [H][W]   (inputs)
 *   d_mean2 [n][2]   d/d(pixel centre x, y)
 *   d_conic [n][3]   d/d(ca, cb2, cc) of q = ca dx^2 + cb2 dx dy + cc dy^2 (the record's conic)
 *   d_alpha [n]      d/d(opacity)      d_feat [n][C]  d/d(feature row)       (device float, overwritten)
 * Sums over pixels use fp32 atomics (order not fixed).  fp16-stored features with C in {16, 32, 64}
 * run the tensor-core kernel (contractions by mma.sync, fp32 accumulation); fp32-stored features and
 * C = 8 the plain per-pixel kernel.  Errors: TA_ERR_INVALID_ARG for NULL pointers or no matching
 * forward call.
 */
ta_status ta_rasterize_backward(ta_context* ctx, const ta_gaussians* g, int64_t n, int32_t H, int32_t W,
                                const ta_raster_params* params, const float* grad_F, const float* grad_A,
                                float* d_mean2, float* d_conic, float* d_alpha, float* d_feat, void* stream);

/*
 * Introspection of the LAST ta_rasterize call on this context (device pointers into context
 * scratch, valid until the next call; read them on the same stream after it completes).
 *   records     [n][8] 32-bit words per Gaussian (array order): mean_x, mean_y, conic a, conic 2b,
 *               conic c, alpha (float bits), pixel box x0 | x1 << 16, y0 | y1 << 16 (culled: 1, 1)
 *   depth_keys  [n] uint32 in depth-rank order: camera-space depth bits (0xffffffff when culled;
 *               culled Gaussians carry no tile entries, their rank positions are unspecified)
 *   order       [n] uint32: array index of the Gaussian of depth rank r
 *   tile_offsets [T + 1] uint32: list of tile t (row-major tiles of tile_px x tile_px pixels, T = tiles_x *
 *               tiles_y) is tile_list[tile_offsets[t] .. tile_offsets[t+1])
 *   tile_list   [K] uint32 array indices ordered by (tile, depth, id) -- the sequence the compositor
 *               walks for each tile (k_tile_split's per-tile lists, compacted into one array by this call)
 *   n_contrib   [H][W] int32 composited pairs per pixel (only with TA_FLAG_DEBUG_COUNTS)
 * The host fields (n, K, P, tiles_x, tiles_y, sort_passes) are filled by a synchronising read.
 */
typedef struct {
    int64_t n, K, Kc;            /* Gaussians, (tile, Gaussian) entries, (coarse bin, Gaussian) entries:
                                    32 x 32-pixel bins up to 1024 px per side, 64 x 64 beyond when the
                                    Gaussian indices fit 24 bits */
    int32_t P, tiles_x, tiles_y, sort_passes;
    const uint32_t* records;
    const uint32_t* depth_keys;
    const uint32_t* order;
    const uint32_t* tile_offsets;
    const uint32_t* tile_list;
    const int32_t* n_contrib;
    /* compositor work counters (only with TA_FLAG_DEBUG_COUNTS): [0] tile-list entries read,
       [1] entries staged, [2] staged entries evaluated, [3] evaluated with some q <= q_max,
       [4] accumulated, [5] composited (pixel, Gaussian) pairs, [6] warps, [7] fill rounds */
    int64_t work[8];
    int32_t tile_px;             /* side of the compositing tiles the lists are for: 16, or 8 (opt-in
                                    TA_TILE_PX=8 with 32 x 32-pixel coarse bins) */
    int32_t reserved;
} ta_debug_view;
ta_status ta_debug_last(ta_context* ctx, ta_debug_view* out, void* stream);

/* Synchronise `stream` (and the context's lane streams) and report whether any TA_FLAG_ASYNC call since
   the last check -- on the context or its lanes' child contexts -- overflowed reserved scratch
   (*overflowed = 1); TA_ERR_CAPACITY is also returned in that case. */
ta_status ta_check_overflow(ta_context* ctx, void* stream, int32_t* overflowed);

/*
 * Stage profiling (CUDA events recorded on the call's stream around each stage of ta_unproject /
 * ta_rasterize while enabled).  ta_profile_read synchronises the device, adds the elapsed times of
 * every pending event pair to the totals and returns them (reset != 0 zeroes the totals afterwards).
 */
typedef enum {
    TA_STAGE_UNPROJECT = 0,   /* a1: count + scan + write */
    TA_STAGE_PROJECT = 1,     /* a2: init + projection / cull */
    TA_STAGE_SORT = 2,        /* a4: depth-key radix passes */
    TA_STAGE_BIN_COUNT = 3,   /* a3: per-warp tile histograms */
    TA_STAGE_BIN_SCAN = 4,    /* a3/a5: tile-major offset scan (+ entry-count readback when synchronous) */
    TA_STAGE_BIN_PLACE = 5,   /* a3: ordered list placement */
    TA_STAGE_COMPOSITE = 6,   /* a6 */
    TA_STAGE_COUNT = 7
} ta_stage;
typedef struct { double ms[TA_STAGE_COUNT]; uint64_t calls[TA_STAGE_COUNT]; } ta_profile;
ta_status ta_profile_enable(ta_context* ctx, int32_t enable);
ta_status ta_profile_read(ta_context* ctx, ta_profile* out, int32_t reset);

/* Kernels this context has launched so far (monotone counter; bench "gpu_launches"). */
uint64_t ta_launch_count(const ta_context* ctx);

const char* ta_status_string(ta_status s);
const char* ta_last_error(const ta_context* ctx);   /* message of the last failing call, "" if none */
const char* ta_build_info(void);                     /* "sm_100a ..." */

#ifdef __cplusplus
}
#endif
#endif /* TA_H_ */
