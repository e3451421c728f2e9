/*
 * ges_b200.h -- C ABI of the B200-native GES forward renderer.
 *
 * The reference has no FFI: its render path is the Python function
 * ges.forward.render (/root/reference/pkg/src/ges/forward.py:403-417) and the
 * two passes it calls.  Each entry point below replaces one of those calls
 * (cited per function); the Python package paper_2504_17545_b200 binds them
 * with ctypes (INTEGRATION.md shows the binding).  All pointers are DEVICE
 * pointers unless stated; all calls are stream-ordered and re-entrant per
 * stream; no global mutable state except the thread-local error string.
 * Memory is owned by the caller (scene blob, frame workspace, outputs).
 *
 * Return codes: 0 ok; GES_EINVAL invalid argument (Python: ValueError);
 * GES_EDEGREE unsupported SH degree (Python: ValueError, as sh.py:24-31);
 * GES_EWORKSPACE workspace too small; GES_ECUDA CUDA error (RuntimeError).
 */
#ifndef GES_B200_H
#define GES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GES_ABI_VERSION 3

#define GES_OK 0
#define GES_EINVAL 1
#define GES_EDEGREE 2
#define GES_EWORKSPACE 3
#define GES_ECUDA 4

#define GES_LAYERS_FULL 0           /* forward.py:417 */
#define GES_LAYERS_SURFELS_ONLY 1   /* forward.py:407-410 */
#define GES_LAYERS_GAUSSIANS_ONLY 2 /* forward.py:412-416 */

/* Pinhole camera, cameras.py:17-80.  w2c is the top 3x4 of world_to_camera,
 * row-major.  width/height are the BASE resolution; supersample=4 renders the
 * surfel pass on the camera scaled by 2 (cameras.py:75-80, forward.py:136). */
typedef struct ges_camera {
    double fx, fy, cx, cy;
    int32_t width, height;
    double w2c[12];
} ges_camera_t;

/* RenderSettings, forward.py:36-58 (dtype selects ges_render or
 * ges_render_f64; threads is meaningless on the GPU). */
typedef struct ges_settings {
    int32_t supersample;      /* 1 or 4 */
    int32_t layers;           /* GES_LAYERS_* */
    int32_t mip;              /* 0/1 */
    int32_t epsilon_mode;     /* 0 adaptive, 1 constant (forward.py:212-215) */
    int32_t with_geometry;    /* 0/1 */
    double epsilon_value;     /* (float64 like the reference; the float32 kernels round it) */
    double background[3];
    int32_t tile_mode;        /* 0 auto; 1: 16x16-pixel tiles; 2: 32x32-pixel tiles,
                                 2x2 pixels per thread (ss=1 without geometry) */
} ges_settings_t;

/* Source scene in the reference's storage layout (primitives.py:42-161),
 * float64 device arrays, row-major.  g_filter3d may be NULL (all zero).
 * s_order / g_order (int32, may be NULL = identity) give the storage order of
 * the packed scene: packed primitive i is source primitive order[i].  A
 * spatially coherent order (the package uses a 3D Morton order) makes the
 * per-frame binning atomics aggregate per warp; results do not depend on it
 * (surfel ids reported and used for z-buffer tie-breaks are SOURCE ids). */
typedef struct ges_scene_src {
    int64_t n_surfels, n_gaussians;
    int32_t sh_degree;        /* 0..3 */
    int32_t gaussian_dim;     /* 3 = GaussianKind.THREE_D, 2 = TWO_D */
    const double *s_pos, *s_quat, *s_log_scale, *s_sh;
    const double *g_pos, *g_raw_opacity, *g_quat, *g_log_scale, *g_sh, *g_filter3d;
    const int32_t *s_order, *g_order;
    /* Bounding box of all primitive centres (xmin, ymin, zmin, xmax, ymax,
     * zmax) and the largest primitive radius; only sets the per-view depth
     * range of the binning slabs (all zero: one slab, still exact). */
    double bounds[7];
} ges_scene_src_t;

/* Packed device scene (float32, 16-byte aligned SoA).  Filled by
 * ges_scene_pack; all pointers point into the caller's scene blob. */
typedef struct ges_scene {
    int64_t n_surfels, n_gaussians;
    int32_t sh_degree, gaussian_dim;
    float *s_pos_s1;      /* n_surfels x 4: pos.xyz, exp(log_scale[0])          */
    float *s_quat;        /* n_surfels x 4: unit (w, x, y, z)                  */
    float *s_s2;          /* n_surfels:     exp(log_scale[1])                  */
    float *s_sh;          /* n_surfels x K x 3                                 */
    int32_t *s_id;        /* n_surfels: source index of packed surfel i        */
    int32_t *s_pack;      /* n_surfels: packed index of source surfel j        */
    float *g_pos_op;      /* n_gaussians x 4: pos.xyz, eff_opacity             */
    float *g_quat;        /* n_gaussians x 4                                   */
    float *g_scale_eps;   /* n_gaussians x 4: eff_scale (s2=0 for 2D), epsilon */
    float *g_sh;          /* n_gaussians rows of 3K floats padded to 4, 12, 28, 52 floats (deg 0-3) */
    double bounds[7];     /* copied from ges_scene_src_t::bounds               */
} ges_scene_t;

/* Output buffers; any may be NULL (not written).  H, W = base resolution.
 * Layouts match SurfelBuffers / GaussianBuffers / RenderResult
 * (forward.py:61-82): colours (H,W,3) f32, depth (H,W) f32 (+inf uncovered),
 * normal (H,W,3) f32, winner (H,W) int32 (-1 uncovered). */
typedef struct ges_outputs {
    float *image;
    float *s_color, *s_depth, *s_normal;
    int32_t *s_winner;
    float *g_color, *g_weight, *g_depth, *g_normal;
    uint8_t *image_rgba8;     /* (H,W,4) clip(image*255+0.5) as datasets.py:54-56, alpha 255 */
} ges_outputs_t;

/* Per-frame counters written by the device (read them after the frame). */
typedef struct ges_frame_status {
    int64_t surfel_pairs;     /* tile/surfel pairs the frame needed   */
    int64_t gaussian_pairs;   /* tile/Gaussian pairs the frame needed */
    int32_t overflow;         /* nonzero: a pair list exceeded capacity, outputs invalid */
    int32_t pad;
} ges_frame_status_t;

int ges_abi_version(void);
const char *ges_last_error(void);

/* Bytes of the packed scene blob (replaces the lazy property math of
 * primitives.py:55-56, :113-131 done once per scene instead of per render). */
size_t ges_scene_bytes(int64_t n_surfels, int64_t n_gaussians, int32_t sh_degree);
int ges_scene_pack(const ges_scene_src_t *src, void *blob, size_t blob_bytes,
                   ges_scene_t *out, void *stream);

/* Frame workspace: per-primitive screen records, tile counters and the two
 * tile lists with the given pair capacities. */
size_t ges_workspace_bytes(const ges_scene_t *scene, const ges_camera_t *cam,
                           const ges_settings_t *st, int64_t surfel_pair_cap,
                           int64_t gaussian_pair_cap);

/* Full two-pass render: forward.py:403-417 (render). */
int ges_render(const ges_scene_t *scene, const ges_camera_t *cam,
               const ges_settings_t *st, const ges_outputs_t *out,
               void *workspace, size_t ws_bytes, int64_t surfel_pair_cap,
               int64_t gaussian_pair_cap, ges_frame_status_t *status_dev,
               void *stream);

/* ges_render that also records 6 CUDA events (cudaEvent_t, may be NULL) on
 * `stream` at the phase boundaries: [0] frame start, [1] after the counter
 * memsets, [2] after the surfel and Gaussian preprocess kernels, [3] after
 * the tile scan, [4] after the tile fill, [5] after the fused tile kernel. */
int ges_render_profiled(const ges_scene_t *scene, const ges_camera_t *cam,
                        const ges_settings_t *st, const ges_outputs_t *out,
                        void *workspace, size_t ws_bytes, int64_t surfel_pair_cap,
                        int64_t gaussian_pair_cap, ges_frame_status_t *status_dev,
                        void *stream, void *const *events);

/* Pass 1 alone: forward.py:127-209 (rasterize_surfels). */
int ges_rasterize_surfels(const ges_scene_t *scene, const ges_camera_t *cam,
                          const ges_settings_t *st, const ges_outputs_t *out,
                          void *workspace, size_t ws_bytes, int64_t surfel_pair_cap,
                          ges_frame_status_t *status_dev, void *stream);

/* Pass 2 alone against a given surfel depth map (H,W) f32:
 * forward.py:218-245 (accumulate_gaussians).  Writes g_* outputs. */
int ges_accumulate_gaussians(const ges_scene_t *scene, const ges_camera_t *cam,
                             const float *surfel_depth, const ges_settings_t *st,
                             const ges_outputs_t *out, void *workspace, size_t ws_bytes,
                             int64_t gaussian_pair_cap, ges_frame_status_t *status_dev,
                             void *stream);

/* forward.py:384-388 (composite): image = (C_s*w + C_G)/(w + W_G); n = H*W. */
int ges_composite(const float *surfel_color, const float *g_color, const float *g_weight,
                  float surfel_weight, float *image, int64_t n, void *stream);

/* forward.py:391-400 (smooth_geometry). */
int ges_smooth_geometry(const float *s_depth, const float *s_normal, const float *g_depth,
                        const float *g_normal, const float *g_weight, float *depth_out,
                        float *normal_out, int64_t n, void *stream);

/* ------------------------------------------------------------------ float64
 * RenderSettings.dtype = float64 (forward.py:44; the reference's own tests
 * render in float64, pkg/tests/test_forward.py:33-35).  The frame is binned
 * exactly like ges_render (float32 records, conservative ranges and depth
 * keys, 16x16 tiles) and the per-pixel passes then run in float64 on the
 * SOURCE arrays `src` the scene was packed from: forward.py:127-209
 * (surfel z-buffer, lowest source id on ties), :248-381 (depth-gated
 * Gaussian sums) and :384-417 (composite, layers), with the reference's
 * formulas.  Outputs are float64 (winner int32); any may be NULL. */
typedef struct ges_outputs_f64 {
    double *image;
    double *s_color, *s_depth, *s_normal;
    int32_t *s_winner;
    double *g_color, *g_weight, *g_depth, *g_normal;
} ges_outputs_f64_t;

/* Workspace of ges_render_f64 (the float32 binning plus the float64
 * per-primitive records). */
size_t ges_workspace_bytes_f64(const ges_scene_t *scene, const ges_camera_t *cam,
                               const ges_settings_t *st, int64_t surfel_pair_cap,
                               int64_t gaussian_pair_cap);

/* mode 3: render (forward.py:403-417); 1: rasterize_surfels (:127-209);
 * 2: accumulate_gaussians (:218-245) against surfel_depth (H,W) float64. */
int ges_render_f64(const ges_scene_t *scene, const ges_scene_src_t *src, const ges_camera_t *cam,
                   const ges_settings_t *st, int32_t mode, const double *surfel_depth,
                   const ges_outputs_f64_t *out, void *workspace, size_t ws_bytes,
                   int64_t surfel_pair_cap, int64_t gaussian_pair_cap,
                   ges_frame_status_t *status_dev, void *stream);

/* float64 composite / smooth_geometry (forward.py:384-400). */
int ges_composite_f64(const double *surfel_color, const double *g_color, const double *g_weight,
                      double surfel_weight, double *image, int64_t n, void *stream);
int ges_smooth_geometry_f64(const double *s_depth, const double *s_normal, const double *g_depth,
                            const double *g_normal, const double *g_weight, double *depth_out,
                            double *normal_out, int64_t n, void *stream);

#define GES_IMAGE_F32_RGB 0   /* (H,W,3) float32: RenderResult.image */
#define GES_IMAGE_RGBA8 1     /* (H,W,4) uint8: the saved frame, datasets.py:54-56 */

/* End-to-end view batch with HOST buffers (the multi-view caller loop of
 * metrics.py:60-66 / cli.py:165-168): for each host camera, render on the
 * device-resident scene and copy the image (format GES_IMAGE_*) into
 * host_images (pinned memory recommended; all views share one resolution).
 * View v runs on lane v % n_lanes: streams[lane] with its own workspace
 * workspaces[lane] (ws_bytes each) and status slot, so views of different
 * lanes overlap; image_dev holds 2 * n_lanes device image buffers and each
 * copy runs on copy_stream, overlapped with later renders.  Returns after
 * enqueueing; synchronise copy_stream before reading host_images.
 * status_dev: n_views ges_frame_status_t (device) or NULL. */
int ges_render_views_host(const ges_scene_t *scene, const ges_camera_t *host_cams,
                          int32_t n_views, const ges_settings_t *st, int32_t format,
                          void *host_images, int32_t n_lanes, void *const *workspaces,
                          size_t ws_bytes, int64_t surfel_pair_cap, int64_t gaussian_pair_cap,
                          void *image_dev, ges_frame_status_t *status_dev, void *const *streams,
                          void *copy_stream);

/* Peer frame buffers for the multi-GPU frame gather without a collective
 * (SURVEY 8(e)): the destination rank allocates one device buffer and
 * exports a CUDA IPC handle (64 bytes, written to ipc_handle); every other
 * rank maps it on its own device (peer access over NVLink enabled) and
 * passes slices of it as ges_outputs_t::image_rgba8, so the tile kernel's
 * RGBA8 stores land in the destination GPU's memory while it renders.
 * ges_peer_open must run on the device given (the caller's current device
 * is restored). */
int ges_peer_alloc(size_t bytes, void **dev_ptr, void *ipc_handle);
int ges_peer_free(void *dev_ptr);
int ges_peer_open(const void *ipc_handle, int32_t device, void **dev_ptr);
int ges_peer_close(void *dev_ptr);

/* Tile-kernel work counters (24 x u64), then reset.  All zero unless the
 * library was built with -DGES_STATS (tuning builds only; synchronous). */
int ges_debug_stats(uint64_t *out24);

/* ------------------------------------------------------------------ training
 * Joint-stage training step of the reference (training.py:358-392 frozen
 * surfel pass, :399-544 Gaussian passes, :547-788 backward): the forward is
 * the deployment kernels above (ges_rasterize_surfels on the supersampled
 * camera, ges_accumulate_gaussians at base resolution) plus the surfel view
 * colours below; the backward pushes image cotangents to the Gaussian
 * parameters (3D EWA and planar 2D) and, through the cached winner map, to
 * the frozen surfels' SH coefficients and positions.
 *
 * Gradients are float64 device arrays in SOURCE order with the layout of the
 * reference GradientSet (primitives.py:195-209), i.e. w.r.t. exposed values:
 * position, opacity sigma (not its logit), the unit quaternion (tangent
 * projected, training.py:890-893), scale (not its log) and SH. */
typedef struct ges_gauss_grads {
    double *pos;       /* n_gaussians x 3 */
    double *opacity;   /* n_gaussians */
    double *quat;      /* n_gaussians x 4 */
    double *scale;     /* n_gaussians x gaussian_dim */
    double *sh;        /* n_gaussians x K x 3 */
    double *screen;    /* n_gaussians: NDC screen-gradient norm (training.py:896-911) */
} ges_gauss_grads_t;

/* View colour of every surfel, (n_surfels, 3) float32 in SOURCE order:
 * _surfel_colors_with_tape (training.py:100-109) / surfel_view_colors
 * (forward.py:99-103). */
int ges_surfel_colors(const ges_scene_t *scene, const ges_camera_t *cam, float *rgb, void *stream);

/* Surfel buffers of the frozen pass from the cached z-buffer of the
 * supersampled camera (training.py:380-392 and :334-346): winner / depth /
 * normal are (H*grid, W*grid[,3]) device arrays (winner: source ids, -1
 * uncovered), colors (n_surfels, 3) the view colours (ges_surfel_colors),
 * background 3 floats on the HOST.  Writes s_color (H,W,3) = box mean of the
 * sub-samples' colour (background where uncovered), s_depth (H,W) = the
 * depth of sub-sample (0,0) (the Gaussian gate depth of the late phase) and,
 * if non-NULL, the blended geometry b_depth (H,W) / b_normal (H,W,3) = box
 * means of the covered sub-samples' depth / normal. */
int ges_frozen_surfel_buffers(const int32_t *winner, const float *depth, const float *normal,
                              const float *colors, int32_t width, int32_t height, int32_t grid,
                              const float *background, float *s_color, float *s_depth, float *b_depth,
                              float *b_normal, void *stream);

/* Scratch of ges_backward_gaussians: 16 float64 accumulators and two
 * float4 ray coefficients per Gaussian. */
size_t ges_backward_scratch_bytes(int64_t n_gaussians);

/* Workspace of ges_backward_gaussians (its own tile binning at 16 px). */
size_t ges_backward_workspace_bytes(const ges_scene_t *scene, const ges_camera_t *cam,
                                    const ges_settings_t *st, int64_t gaussian_pair_cap);

/* Gaussian half of training.backward (training.py:547-609 with
 * _gaussian_backward_3d :646-719 / _gaussian_backward_2d :722-788), given the
 * cotangents of the Gaussian buffers: g_color = dL/dC_G (H,W,3), g_weight =
 * dL/dW_G (H,W) and, optional (NULL = zero), g_depth = dL/dD_G (H,W),
 * g_normal = dL/dN_G (H,W,3), all float32.  surfel_depth (H,W) is the depth
 * the forward's Gaussian pass was gated with.  `src` must hold the float64
 * source arrays the scene was packed from (the chain rule runs in float64 on
 * them).  any_filter: nonzero iff any filter3d entry is nonzero
 * (primitives.py:113-126 switch the effective scale/opacity on globally).
 * The gradient outputs must be zero-initialised: Gaussians without any
 * contributing fragment are not written. */
int ges_backward_gaussians(const ges_scene_t *scene, const ges_scene_src_t *src, int32_t any_filter,
                           const ges_camera_t *cam, const ges_settings_t *st, const float *surfel_depth,
                           const float *g_color, const float *g_weight, const float *g_depth,
                           const float *g_normal, const ges_gauss_grads_t *grads, void *scratch,
                           size_t scratch_bytes, void *workspace, size_t ws_bytes,
                           int64_t gaussian_pair_cap, ges_frame_status_t *status_dev, void *stream);

/* Per-Gaussian contribution score of one view (optim.py:519-533, the joint
 * stage's pruning statistic): scores[j] = max(scores[j], max over the
 * Gaussian's fragments of max_c(colour) * alpha / (1 + W_G)), for source
 * Gaussian j (order from src->g_order; src may be NULL = identity).
 * g_weight = W_G (H,W) of the same view and settings, float32; scores
 * (n_gaussians) float32 >= 0, accumulated across calls.  Workspace as
 * ges_backward_workspace_bytes. */
int ges_gaussian_contributions(const ges_scene_t *scene, const ges_scene_src_t *src, const ges_camera_t *cam,
                               const ges_settings_t *st, const float *surfel_depth, const float *g_weight,
                               float *scores, void *workspace, size_t ws_bytes, int64_t gaussian_pair_cap,
                               ges_frame_status_t *status_dev, void *stream);

/* Frozen-surfel half of training.backward (_surfel_backward_frozen,
 * training.py:612-629): winner (H*grid, W*grid) int32 source ids (-1 =
 * uncovered) of the cached opaque z-buffer, g_color = dL/dC_s (H,W,3)
 * float32.  Writes g_sh (n_surfels x K x 3) and g_pos (n_surfels x 3)
 * float64 for the surfels that received a colour cotangent (the outputs must
 * be zero-initialised; others are not written); col_scratch holds
 * n_surfels x 3 float64. */
int ges_backward_surfels_frozen(const ges_scene_src_t *src, const ges_camera_t *cam, int32_t grid,
                                const int32_t *winner, const float *g_color, double *col_scratch,
                                double *g_sh, double *g_pos, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GES_B200_H */
