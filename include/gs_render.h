/*
 * gs_render.h -- C-ABI of the B200 (sm_100a) forward 3DGS renderer with
 * GEMM-compatible alpha blending (GEMM-GS, arXiv 2604.02120).
 *
 * Citations: P:n = PAPER.md line n (the paper's LaTeX source).
 *
 * The library computes, for one camera, the four stages of the forward
 * render path the paper names:
 *   (a) preprocessing  -- project 3D Gaussians to 2D ellipses, tile
 *       intersection, depth d and RGB colour c;
 *   (b) duplication    -- one copy per touched 16x16 tile, key = tile index
 *       concatenated with depth;
 *   (c) sorting        -- per-tile depth order;
 *   (d) blending       -- Eq. (1) front-to-back compositing with the
 *       exponent computed as the GEMM of Eq. (6)-(8) on
 *       tcgen05 tensor cores, alpha = o*exp(power), alpha-skip below 1/255,
 *       alpha cap 0.99, early termination at T < 1e-4 (Alg. 1-2, P:128-191,
 *       P:309-383; readings R-1..R-5 in DESIGN.md).
 *
 * Conventions (all entry points):
 *  - Return GS_OK (0) or a negative gs_status. Nothing is silently truncated:
 *    if the duplicated key count K exceeds the context's max_keys the call
 *    fails with GS_ERR_CAPACITY (reported by gs_last_stats / GS_SYNC).
 *  - Unless stated otherwise every array pointer is a DEVICE pointer on the
 *    context's device, owned by the caller, 16-byte aligned, contiguous,
 *    float32 little-endian. The library never frees caller memory.
 *  - Inputs are ACTIVATED values: scales > 0, rotations as unit-norm
 *    quaternions (w,x,y,z) (renormalised in-kernel), opacity in (0,1).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); all work is
 *    enqueued on it, asynchronously. One gs_ctx per (device, host thread).
 *  - Determinism: outputs are bit-identical across runs, batch sizes and GPU
 *    counts for identical inputs.
 */
#ifndef GS_RENDER_H_
#define GS_RENDER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GS_OK = 0,
    GS_ERR_INVALID_ARG = -1,      /* null pointer, N < 0, W/H <= 0 or above ctx max, sh_degree > 3 */
    GS_ERR_ALIGNMENT = -2,        /* a pointer is not 16-byte aligned                               */
    GS_ERR_CAPACITY = -3,         /* N > max_points or K > max_keys (nothing truncated)             */
    GS_ERR_CUDA = -4,             /* a CUDA runtime call failed                                     */
    GS_ERR_UNSUPPORTED_ARCH = -5, /* device is not sm_100 (B200)                                    */
    GS_ERR_NO_DEVICE = -6
} gs_status;

/* Pinhole camera, OpenCV axes (x right, y down, z forward). A world point p
 * maps to camera space as R p + t (R row-major). Pixel (i,j) has its centre
 * at integer coordinates (R-15); the projected mean is (fx x/z + cx, fy y/z + cy).
 * tan_fovx / tan_fovy bound the EWA Jacobian clamp (1.3 tan_fov, R-14);
 * campos is the origin of the SH view direction. Gaussians with camera depth
 * z <= znear are culled. 22 floats, in this order. */
typedef struct {
    float R[9];
    float t[3];
    float fx, fy, cx, cy;
    float znear;
    float tan_fovx, tan_fovy;
    float campos[3];
} gs_camera;

enum {
    GS_BLEND_TC = 0,      /* tcgen05 TF32 hi/lo exponent GEMM (the paper's method, default) */
    GS_BLEND_DIRECT = 1,  /* CUDA-core direct Eq. (3) (vanilla Alg. 1), A/B baseline        */
    GS_BLEND_MMA = 2,     /* the same GEMM with warp-level mma.sync.m16n8k8 TF32 hi/lo, the
                           * paper's kernel shape: A/B against tcgen05          */
    GS_BLEND_TC_COLOR = 3 /* GS_BLEND_TC with the colour sum of Eq. (1) as a second tcgen05
                           * product per batch (extends P:302-304):
                           * C += W . Col^T with W = alpha*T rounded to TF32 (relative error
                           * <= 2^-11 per term) and colours split TF32 hi/lo; 2 CTAs/SM     */
};

enum {
    GS_FLAG_SYNC = 1u,    /* synchronise the stream at the end and report device errors     */
    GS_FLAG_TIMING = 2u,  /* record CUDA events around the stages (read by gs_stage_times)  */
    GS_FLAG_STATS = 4u,   /* count blend work (pairs evaluated / kept) into gs_stats        */
    GS_FLAG_TIGHT = 8u,   /* tile-exact intersection: drop (Gaussian, tile) pairs whose
                           * maximum over the tile's pixel box is alpha < 1/255 (with a margin
                           * larger than the exponent error). Such pairs are alpha-skipped by the
                           * blend anyway, so the image is bit-identical; binning keeps a subset. */
    GS_FLAG_STATIC_SCENE = 32u, /* gs_render_views: no work pending on `stream` writes the scene
                           * arrays (they are resident and unchanged, as in an orbit or serving
                           * loop), so the call's preprocess and binning may start before the
                           * caller's earlier work on `stream` (e.g. the previous call's last
                           * blends) has finished; frames are still written in stream order.
                           * Safe with interleaved single-view calls: the view-group calls use
                           * their own workspaces and error accumulator, never the ones of
                           * gs_render / gs_debug_* (which run in the caller's stream order). */
    GS_FLAG_TILE_LISTS = 64u, /* GS_BLEND_TC(_COLOR): bin into per-tile lists (the two-level
                           * row / column passes) instead of the 4x4-tile supertile lists the
                           * blend filters itself; for kernel A/Bs on the lists the other blends
                           * read. Frames are identical either way.                          */
    GS_FLAG_OBOX = 16u    /* opacity-aware box (cheaper): the vanilla rect clipped to the
                           * bounding box of the ellipse where alpha >= 1/255 can hold (margin
                           * 5e-3 in ln alpha), and Gaussians with 255*opacity < 1 culled; no
                           * per-row masks, so binning takes the plain-rect path. Frames are
                           * bit-identical to the vanilla rect's; docs/preprocess_order.md 10b.
                           * GS_FLAG_TIGHT takes precedence if both are set. */
};

typedef struct {
    float bg[3];           /* background colour added as T*bg (R-17)                         */
    int sh_degree;         /* 0..3; -1 => shs_or_colors holds plain colours [N,3]            */
    int sh_stride;         /* SH coefficients per Gaussian in shs (>= (deg+1)^2)             */
    float scale_modifier;  /* multiplies every scale (1.0)                                   */
    int blend;             /* GS_BLEND_TC | GS_BLEND_DIRECT | GS_BLEND_MMA | GS_BLEND_TC_COLOR */
    unsigned flags;        /* GS_FLAG_*                                                      */
    int batch;             /* GS_BLEND_MMA: Gaussians per shared-memory batch, 32/64/128/256
                            * (0 = 256); output bit-identical for every value. The
                            * tcgen05 blend streams fixed 32-Gaussian batches (ignored). */
    int band, n_bands;     /* row band of a split frame (SURVEY 8(e) option): n_bands > 1
                            * renders only tile rows [band*gy/n_bands, (band+1)*gy/n_bands)
                            * (gy = ceil(H/16)); pixels of the other bands are not written,
                            * the band's pixels are bit-identical to the full frame's. The
                            * preprocess still projects every Gaussian; binning and blending
                            * only cover the band. n_bands <= 1: the whole frame. */
} gs_opts;

typedef struct {
    int64_t n_points;      /* N of the last call                                             */
    int64_t n_visible;     /* Gaussians with tiles_touched > 0                              */
    int64_t n_keys;        /* K = number of (Gaussian, tile) pairs                          */
    int64_t capacity_keys; /* max_keys of the context                                       */
    int status;            /* gs_status of the last frame (device-side checks included)     */
    int64_t launches;      /* kernels launched by this context since creation              */
    int64_t pairs_evaluated;  /* GS_FLAG_STATS: (Gaussian, pixel) exponents the tensor-core MMA
                               * computed in the last frame (256 x the Gaussians of every batch
                               * built; k_blend_tc only) */
    int64_t pairs_kept;       /* GS_FLAG_STATS: of those, alpha >= 1/255 on a live pixel       */
} gs_stats;

typedef struct gs_ctx gs_ctx;

/* Creates a context owning device workspace for up to max_points Gaussians,
 * max_keys duplicated keys and max_w x max_h images on `device`.
 * Limits: max_keys < 2^32, max_points < 2^31, at most 2^20 16x16 tiles
 * (e.g. 16384 x 16384 px); otherwise GS_ERR_INVALID_ARG.
 * Fails with GS_ERR_UNSUPPORTED_ARCH unless the device is sm_100. */
int gs_ctx_create(gs_ctx **out, int device, int64_t max_points, int64_t max_keys,
                  int max_w, int max_h);
int gs_ctx_destroy(gs_ctx *ctx);

/* Renders one view. means3D [N,3], scales [N,3], rots [N,4] (w,x,y,z),
 * opacity [N], shs_or_colors [N,sh_stride,3] (or [N,3] if sh_degree == -1).
 * out_rgb [3,H,W] planar, out_T [H,W] final transmittance; every in-frame pixel
 * of both is written: out_rgb[c] = C_c + T*bg_c (Eq. 1 plus background). */
int gs_render(gs_ctx *ctx, void *stream, int N, const float *means3D, const float *scales,
              const float *rots, const float *opacity, const float *shs_or_colors,
              const gs_camera *cam, int W, int H, const gs_opts *opts,
              float *out_rgb, float *out_T);

/* Renders n_views cameras (host array cams[n_views]) of the same scene into
 * out_rgb [n_views,3,H,W] and out_T [n_views,H,W] (device), on `stream`.
 * Frames are bit-identical to n_views gs_render calls. The views are processed
 * in groups (gs_set_view_group, default 4, at most 16): one preprocess launch reads each
 * Gaussian's record (means, scales, rotation, opacity, SH) from HBM once for
 * the whole group and writes the group's per-view splats; binning and blending
 * then run view by view (P:109-117 per view). */
int gs_render_views(gs_ctx *ctx, void *stream, int N, const float *means3D, const float *scales,
                    const float *rots, const float *opacity, const float *shs_or_colors,
                    const gs_camera *cams, int n_views, int W, int H, const gs_opts *opts,
                    float *out_rgb, float *out_T);

/* End-to-end variant with HOST buffers (pinned memory recommended): copies the
 * scene host->device, renders n_views, copies the frames device->host and
 * synchronises `stream` before returning. The scene is staged in one of two
 * context-owned device buffers (sized for the scene on first use) by a context
 * upload stream; every frame is copied back on a context copy stream as soon as
 * its blend is done (staging slot v % 2G, G the view group size). */
int gs_render_views_host(gs_ctx *ctx, void *stream, int N, const float *means3D,
                         const float *scales, const float *rots, const float *opacity,
                         const float *shs_or_colors, const gs_camera *cams, int n_views,
                         int W, int H, const gs_opts *opts, float *h_out_rgb, float *h_out_T);

/* Sets the view-group size of gs_render_views / gs_render_views_host (g = 1..16;
 * 1 = one preprocess launch per view) and whether the group's per-view binning
 * chains run concurrently on context-owned streams (concurrent != 0, default) or
 * back to back on the caller's stream. Output does not depend on either. The
 * first multi-view call with group g allocates g workspaces per slot set (two
 * sets in the concurrent mode; as gs_ctx_create: about 36 B x max_points + 16 B x
 * max_keys each), separate from the context's single-view workspace. If an
 * allocation fails the call returns GS_ERR_CUDA with nothing half-allocated
 * (a later call retries) and `stream` still orders after any work it enqueued. With
 * GS_FLAG_TIMING and concurrent chains the per-stage times overlap.
 * GS_ERR_INVALID_ARG for g outside 1..16. */
int gs_set_view_group(gs_ctx *ctx, int g, int concurrent);

/* Makes `stream` wait (device-side, cudaStreamWaitEvent) until view group g of
 * the last gs_render_views / gs_render_views_host call has finished blending,
 * i.e. until frames [g*G, min(n_views, (g+1)*G)) are complete (G = the view
 * group size in effect for that call). Lets a consumer of the frames -- the
 * NCCL frame gather of the multi-GPU orbit -- start on early groups while later
 * ones still render. GS_ERR_INVALID_ARG if g is not a group of that call. */
int gs_stream_wait_group(gs_ctx *ctx, void *stream, int g);

/* Makes `stream` wait (device-side) until views [0, v] of the last gs_render_views
 * call are complete (the blends run in view order, so view v's completion implies
 * every earlier view's). Decouples the gather granularity from the view group:
 * a rank can read the scene once per group of 8-16 views and still hand its
 * frames to the NCCL gather two at a time. GS_ERR_INVALID_ARG if v is not a view
 * of that call. */
int gs_stream_wait_view(gs_ctx *ctx, void *stream, int v);

/* Asynchronous form of gs_render_views_host (same arguments): returns once the
 * work is enqueued; `stream` reaches completion only after every frame is in
 * h_out_rgb / h_out_T. The host inputs must stay valid and unmodified, and the
 * outputs unread, until then (cudaMemcpyAsync rules; pinned memory). The scene
 * upload runs on a context stream into one of two device staging buffers, so the
 * upload of the next call overlaps the rendering of this one (a serving loop of
 * back-to-back calls pipelines H2D, compute and D2H). */
int gs_render_views_host_async(gs_ctx *ctx, void *stream, int N, const float *means3D,
                               const float *scales, const float *rots, const float *opacity,
                               const float *shs_or_colors, const gs_camera *cams, int n_views,
                               int W, int H, const gs_opts *opts, float *h_out_rgb, float *h_out_T);

/* Synchronises the last stream used by ctx and reports counts and the status
 * of the last call (e.g. GS_ERR_CAPACITY with the required n_keys). For a
 * multi-view call the status covers every view (any view over capacity gives
 * GS_ERR_CAPACITY and n_keys = the largest K of the call's views); the other
 * counts are the last view's. */
int gs_last_stats(gs_ctx *ctx, gs_stats *out);

/* Sums of the per-stage device times (ms) of all frames rendered with
 * GS_FLAG_TIMING since the previous call (synchronises): ms[0] preprocess,
 * ms[1] binning (compaction, sorts, duplication, ranges), ms[2] blend.
 * *frames receives the number of frames summed. Resets the sums. */
int gs_stage_times(gs_ctx *ctx, double *ms, int64_t *frames);

const char *gs_status_string(int status);

/* Compute capability of `device` as 10*major+minor, or a negative gs_status. */
int gs_device_arch(int device);

/* ---- test-only entry points (bit-exact stage checks, precision study) ---- */

/* Stage (a) only. Outputs [N]: depth, xy [N,2], conic [N,3] = (A,B,C) of the
 * inverse 2D covariance, rgb [N,3], rect [N,4] int32 (xmin,ymin,xmax,ymax,
 * half-open tile ranges), radius [N] int32, touched [N] uint32 (0 = culled;
 * culled rows are all zero). Operation order: docs/preprocess_order.md. */
int gs_debug_preprocess(gs_ctx *ctx, void *stream, int N, const float *means3D,
                        const float *scales, const float *rots, const float *opacity,
                        const float *shs_or_colors, const gs_camera *cam, int W, int H,
                        const gs_opts *opts, float *depth, float *xy, float *conic, float *rgb,
                        int32_t *rect, int32_t *radius, uint32_t *touched);

/* Stages (a)-(c). Writes sorted keys [K] (tile << 32 | depth bits), vals [K]
 * (Gaussian index), ranges [tiles,2] ([start,end) per tile, empty = (0,0)) and
 * the host int64 *n_keys = K. keys/vals must hold `capacity` entries; if
 * K > capacity only *n_keys is written and GS_ERR_CAPACITY returned.
 * Synchronises `stream`. */
int gs_debug_binning(gs_ctx *ctx, void *stream, int N, const float *means3D,
                     const float *scales, const float *rots, const float *opacity,
                     const float *shs_or_colors, const gs_camera *cam, int W, int H,
                     const gs_opts *opts, uint64_t *keys, uint32_t *vals, uint32_t *ranges,
                     int64_t capacity, int64_t *n_keys);

/* Stage (d) alone from caller-supplied splats: xy [N,2], conic [N,3] (A,B,C),
 * opacity [N], rgb [N,3], vals [K] and ranges [tiles,2] as produced by
 * binning. opts->blend selects the kernel. */
int gs_debug_blend(gs_ctx *ctx, void *stream, int N, const float *xy, const float *conic,
                   const float *opacity, const float *rgb, const uint32_t *vals, int64_t K,
                   const uint32_t *ranges, int W, int H, const gs_opts *opts,
                   float *out_rgb, float *out_T);

/* The exponent GEMM of Eq. (8) alone, as the tensor-core blend computes it:
 * for every list entry e of every tile, m[e][p] = log2(alpha) before the 0.99
 * cap, i.e. log2(e)*power + log2(o), for the 256 pixels p of the tile
 * (p = 32*w + lane, pixel (x,y) = (8*(w%2) + lane%8, 4*(w/2) + lane/8)).
 * out_m [K,256] float32. Used to measure |d ln alpha| against the oracle. */
int gs_debug_exponents(gs_ctx *ctx, void *stream, int N, const float *xy, const float *conic,
                       const float *opacity, const uint32_t *vals, int64_t K,
                       const uint32_t *ranges, int W, int H, float *out_m);

/* Debug: the GS_FLAG_TIMING spans recorded since the last gs_stage_times (which
 * clears them): out[3*i .. 3*i+2] = (stage 0/1/2, start ms, end ms), times relative
 * to the first recorded event; *n_spans = count (at most max_spans). Synchronises. */
int gs_debug_timeline(gs_ctx *ctx, double *out, int max_spans, int *n_spans);

/* Debug: while `trace` is non-NULL, the tensor-core blend of CTA 0 records
 * clock64() timestamps of its per-batch pipeline events into trace[b*16 + e]
 * (b < 1024; e: 0/1 producer push begin/end, 2/3/4 builder got-raw /
 * stage-free / done, 5/6 MMA rows-ready / issue, 7/8 and 9/10 compositor warps
 * 0 and 7 start / release). Device buffer of 16384 int64. NULL disables. */
int gs_debug_set_trace(gs_ctx *ctx, long long *trace);

#ifdef __cplusplus
}
#endif
#endif /* GS_RENDER_H_ */
