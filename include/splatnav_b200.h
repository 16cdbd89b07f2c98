/*
 * splatnav_b200.h -- C ABI of the B200-native splat-observation hot path.
 *
 * This is the drop-in boundary for the reference package "splatnav"
 * (/root/reference/pkg/src/splatnav). Plain C: no torch or CUDA C++ types. Memory arguments
 * are DEVICE pointers unless a parameter says "host". Every function returns SN_OK (0) or an
 * error code; sn_last_error() gives a thread-local message. Launches are asynchronous on the
 * given stream. sn_render() queues both passes without a host round trip (capacity-sized
 * workspace, counts kept on the device) and synchronizes the stream once, at the end, to check
 * the counts against the capacities (re-running the render with larger buffers if one overflowed);
 * sn_render_async / sn_render_wait split the two so the next render is queued before the host
 * waits for the previous one.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/splatnav):
 *   sn_render ................ renderer.render_observation (renderer.py:169-177) batched over
 *                              E environments; with no avatars it is renderer.rasterize
 *                              (renderer.py:135); opts.tiled=0 gives rasterize_reference (:145)
 *   sn_blend_tile_range ...... raster._kernels_cy.blend_tile_range (_kernels_cy.pyx:89-114), the
 *                              reference's only FFI, same arguments (HOST buffers), for
 *                              raster.get_kernel("cuda") (raster/__init__.py:26-36)
 *   sn_composite ............. renderer.composite (renderer.py:151-166)
 *   sn_sample_pose ........... rig.sample_pose (rig.py:78-104) + AvatarRuntime.clock
 *                              (tasks.py:299-305), batched
 *   sn_skin_lbs .............. rig.lbs_deform (rig.py:107-146)
 *   sn_get_* ................. harness views of intermediates the reference computes inside
 *                              project_cloud (projection.py:184 sorted ids) and _bin_tiles
 *                              (renderer.py:80-101 tile CSR)
 */
#ifndef SPLATNAV_B200_H
#define SPLATNAV_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SN_ABI_VERSION 3

enum {
    SN_OK = 0,
    SN_ERR_INVALID = 1, /* bad argument / contract violation (python: ContractViolation) */
    SN_ERR_CUDA = 2,    /* CUDA runtime error */
    SN_ERR_NOMEM = 3    /* device allocation failed */
};

enum { SN_FLOAT32 = 0, SN_FLOAT64 = 1 };

/* Pinhole camera (camera.py:16-56). 208 bytes. `center` is Camera.center as the host computes it
 * (-R^T t, camera.py:43-48); has_background = 0 selects layer mode (renderer.py:69-71). */
typedef struct sn_camera {
    double fx, fy, cx, cy, near_, far_;
    double rot[9];   /* world_to_camera[:3,:3], row-major */
    double trans[3]; /* world_to_camera[:3,3] */
    double center[3];
    double background[3];
    int32_t width, height, has_background, pad;
} sn_camera;

/* RenderStats (projection.py:30-36), one per environment. */
typedef struct sn_stats {
    int64_t n_input, n_culled_depth, n_culled_frame, n_degenerate, n_drawn;
} sn_stats;

/* Device-resident scene cloud, packed once at load:
 *   pos_opacity (n,4): x, y, z, opacity logit      -- float or double (dtype)
 *   log_scales  (n,4): s0, s1, s2, unused          -- dtype
 *   rotations   (n,4): w, x, y, z (raw, renormalized on use like build_cov3d)  -- dtype
 *   sh          (K*3, n) float32, structure-of-arrays (coefficient k, channel c at row 3k+c)
 * Optionally (ABI 3) the rows are a spatially ordered copy of the reference's cloud:
 *   index        (n) uint32: the reference (original) index of each row -- depth ties, gaussian ids
 *                and every order-dependent output use it, so results are those of the original order
 *   block_bounds (ceil(n / 256), 8) float32 per 256-row block: min x y z, max x y z, 0, 0 of the
 *                positions -- the count kernel decides whole blocks per env where the box allows
 * Both NULL: rows in the original order, no block decisions. */
typedef struct sn_cloud {
    int64_t n;
    int32_t sh_k;
    int32_t dtype;
    const void *pos_opacity;
    const void *log_scales;
    const void *rotations;
    const float *sh;
    const uint32_t *index;
    const float *block_bounds;
} sn_cloud;

/* Device-resident avatar set: A avatars concatenated (render_observation's concat_clouds
 * order), canonical data in float64, skinning as the nonzero (joint, weight) influences of each
 * gaussian in ascending joint order (the dense N x J rows of the bundle, avatar.py:127-178;
 * skipping a zero weight leaves the reference's sums unchanged, rig.py:119-132), in one of two
 * layouts:
 *   4-slot (infl_offset == NULL; every row has <= 4 nonzeros): joints (n) uint32 = 4 x uint8
 *     joint ids, weights (n,4) f64 (zero = unused slot);
 *   CSR (infl_offset != NULL; any row width, e.g. dense SMPL-X softmax weights over 55 joints):
 *     row g's influences are [infl_offset[g], infl_offset[g+1]) of infl_joint (uint8) and
 *     infl_weight (f64); joints / weights are then unused (may be NULL).
 *   pos_opacity (n,4) f64, log_scales (n,4) f64, rotations (n,4) f64, sh (K*3, n) f32
 *   avatar_of (n) uint16
 *   inv_bind (A, J, 16) f64, traj_q (sum_a T_a*(J+1)*4) f64, traj_t (sum_a T_a*(J+1)*3) f64
 *   traj_offset (A) int64 frame offsets into traj_*, n_frames (A) int32, fps (A) f64,
 *   start_offset (A) f64, loop (A) int32    -- AvatarRuntime fields (tasks.py:290-297) */
typedef struct sn_avatars {
    int64_t n;
    int32_t n_avatars;
    int32_t n_joints;
    int32_t sh_k;
    int32_t pad;
    const double *pos_opacity;
    const double *log_scales;
    const double *rotations;
    const float *sh;
    const uint32_t *joints;
    const double *weights;
    const uint16_t *avatar_of;
    const double *inv_bind;
    const double *traj_q;
    const double *traj_t;
    const int64_t *traj_offset;
    const int32_t *n_frames;
    const double *fps;
    const double *start_offset;
    const int32_t *loop;
    const uint32_t *infl_offset; /* (n+1) CSR row offsets, or NULL for the 4-slot layout */
    const uint8_t *infl_joint;   /* (nnz) */
    const double *infl_weight;   /* (nnz) */
} sn_avatars;

/* Stages timed by sn_render_opts.stage_ms (per pass: 0 = scene, 1 = layer). */
enum {
    SN_STAGE_POSE = 0,      /* sample_pose + joint matrices (layer pass only) */
    SN_STAGE_COUNT = 1,     /* (skin +) project + cull + visibility counts */
    SN_STAGE_SCAN = 2,      /* per-env block scan */
    SN_STAGE_EMIT = 3,      /* (skin +) project + SH + record write */
    SN_STAGE_DEPTH_SORT = 4,
    SN_STAGE_PERMUTE = 5,
    SN_STAGE_PAIR_SCAN = 6,
    SN_STAGE_BIN_COUNT = 7,    /* radix: duplicate pairs; counting: chunk counts + scans */
    SN_STAGE_BIN_SCATTER = 8,  /* radix: (env|tile) pair sort; counting: stable scatter */
    SN_STAGE_RANGES = 9,
    SN_STAGE_BLEND = 10,
    SN_STAGE_COMPOSITE = 11,   /* layer pass: composite over the scene frame + float64 fixups */
    SN_STAGE_FAR = 12,         /* depth-sliced scene pass: far buckets, continuation, float64 fixups */
    SN_N_STAGES = 13
};

/* Per-call options. Null pointers disable the corresponding output. */
typedef struct sn_render_opts {
    int32_t tiled;          /* 1: tile pipeline (rasterize); 0: rasterize_reference semantics */
    int32_t binning;        /* -1: auto (streaming for the scene pass, lists for the avatar layer);
                               0: no tile lists, the blend streams depth-sorted rectangles;
                               1: materialized lists (duplicate + stable (env|tile) radix sort) */
    const uint8_t *avatar_active; /* device (E, A) 0/1, NULL = all active */
    int32_t *contrib_scene; /* device (E,H,W): splats accumulated per pixel, scene pass */
    int32_t *contrib_layer; /* device (E,H,W): avatar-layer pass */
    sn_stats *stats;        /* device (E): RenderStats accumulated over both passes */
    double *stage_ms;       /* HOST (2 x SN_N_STAGES): GPU ms per stage (CUDA events), accumulated */
    int64_t *work;          /* HOST (2 x 6): visible splats, tile pairs (when lists are built),
                               records gathered by the blend, rectangles the blend examined,
                               (pixel, splat) contributions, pixels recomputed by the float64
                               fixup -- per pass, accumulated. Both arrays are filled asynchronously: they are complete
                               after the next sn_render on the context or sn_context_sync_stats(),
                               and must stay valid until then. */
    int32_t exact;          /* 1: every pixel takes the float64 path (the blend's fixup walk) instead of
                               the float32 chain with error bounds -- validation / reference mode */
    int32_t serialize;      /* 1: the avatar-layer pass runs on the caller's stream after the scene pass
                               instead of concurrently on the context's side stream (stage_ms then sum
                               to the render's time) */
    uint8_t *rgb8;          /* device (E,H,W,3) or NULL: the observation payload's uint8 colour, written
                               by the epilogues that finalize each pixel (blend, composite, fixups) with
                               frame_io.save_color_png's rule (clip, x*255+0.5 in float64, truncation)
                               on the float32 colour the frame holds */
    uint16_t *depth16;      /* device (E,H,W) or NULL: fp16 depth (round to nearest) of the same pixels */
    int32_t views;          /* 1: keep what the harness views need beyond the render itself (each splat's
                               gaussian id and reference tile rectangle: sn_get_sorted_ids,
                               sn_get_tile_csr, sn_get_counts' pair count); 0: the lean throughput path
                               (12 bytes less written per visible splat), those views then fail */
    int32_t near_slice;     /* depth slicing of the scene pass: only each env's near depth slice is
                               sorted and streamed; the few tiles that exhaust it with unsaturated
                               pixels continue through a per-tile bucket of the far splats, in depth
                               order (the same decisions, counts and stats; frames bit-identical
                               without an avatar layer, within float32 rounding with one). -1 auto (scenes of >= 500k
                               gaussians rendered without harness views), 0 off, 1 on (envs with
                               too few visible splats stay unsliced), 2..1000: on for every env with
                               the slice at near_slice / 1000 of its sampled depths (tests, tuning);
                               never with tiled = 0, exact = 1 or materialized scene lists. A
                               sliced pass keeps no full depth order: the views that need it fail. */
} sn_render_opts;

typedef struct sn_context sn_context;

int sn_abi_version(void);
const char *sn_last_error(void);

/* One context per (device, thread). Owns the workspace; grows it on demand. */
int sn_context_create(sn_context **ctx);
int sn_context_destroy(sn_context *ctx);
/* Cumulative number of this library's kernels launched through the context (CUB's radix sort and
 * scan kernels excluded). */
int sn_context_kernel_launches(const sn_context *ctx, int64_t *n);
/* Renders that were run twice because a pass outgrew its capacity-sized buffers (the render is
 * queued without host round trips; its visible-splat / tile-pair counts are checked at the end). */
int sn_context_render_retries(const sn_context *ctx, int64_t *n);
/* Folds pending stage timings / work counters into the arrays last passed in sn_render_opts. */
int sn_context_sync_stats(sn_context *ctx);
/* Bytes of device workspace currently held. */
int sn_context_workspace_bytes(const sn_context *ctx, size_t *bytes);

/*
 * Render E environments: scene pass with the cameras' background (layer mode when the cameras
 * have none), then one layer pass depth-composited over it (render_observation):
 *   layer != NULL   -- an already-deformed cloud (concat_clouds of the avatar clouds), same for
 *                      every env;
 *   avatars != NULL -- the avatar set, skinned on device at each env's sim time (fused LBS).
 * At most one of the two. All cameras must share width/height and background mode. cams and
 * sim_times are HOST arrays (E entries). Outputs are device float32: color (E,H,W,3),
 * alpha (E,H,W), depth (E,H,W).
 */
int sn_render(sn_context *ctx, const sn_cloud *scene, const sn_cloud *layer, const sn_avatars *avatars,
              const sn_camera *cams, const double *sim_times, int32_t n_envs, const sn_render_opts *opts,
              float *color, float *alpha, float *depth, void *stream);

/*
 * Pipelined form of sn_render: sn_render_async queues the render (same arguments) and returns
 * without waiting; sn_render_wait waits for the OLDEST queued render and checks it. At most two
 * renders are in flight per context (queue i + 1, then wait for i). *retry = 1 when a pass of that
 * render outgrew the workspace: the buffers have been enlarged, its frames are invalid and it --
 * like any render queued after it -- must be queued again. opts->work / stage_ms arrays must stay
 * alive until the render has been waited for. sn_render itself requires that no async render is
 * in flight.
 */
int sn_render_async(sn_context *ctx, const sn_cloud *scene, const sn_cloud *layer, const sn_avatars *avatars,
                    const sn_camera *cams, const double *sim_times, int32_t n_envs, const sn_render_opts *opts,
                    float *color, float *alpha, float *depth, void *stream);
int sn_render_wait(sn_context *ctx, int32_t *retry);

/* Intermediates of the last sn_render pass (0 = scene, 1 = avatar layer) for env e, copied to
 * HOST buffers. The workspace holds one env chunk (<= 64 envs): e must lie in the last chunk the
 * render processed (SN_ERR_INVALID otherwise); render a smaller batch to inspect other envs. sn_get_counts: visible splats and tile pairs. sorted_ids: original gaussian
 * index per depth rank (projection.py:184). tile_starts (T+1) / pair_splat (P): the tile CSR
 * with depth ranks as values (renderer.py:80-101). */
int sn_get_counts(sn_context *ctx, int32_t pass, int32_t env, int64_t *n_visible, int64_t *n_pairs);
int sn_get_sorted_ids(sn_context *ctx, int32_t pass, int32_t env, int32_t *ids_host, int64_t capacity);
int sn_get_tile_csr(sn_context *ctx, int32_t pass, int32_t env, int64_t *tile_starts_host, int32_t *pair_splat_host,
                    int64_t capacity);
/* The tile lists the blend of the last pass actually consumed for env e (HOST): tile_starts (T+1)
 * and, per tile in depth order, the depth ranks of its splats -- the radix binner's (env, tile)
 * ranges over pair_vals when that pass built lists, else the streamed lists the blend assembles in
 * shared memory (exported by the same fill routine, without early termination). They hold the
 * splats whose TIGHT rectangle (the support ellipse's reach) covers the tile, so each is an
 * in-order sub-list of the reference list (sn_get_tile_csr) that keeps every splat with a pixel of
 * the tile inside its support. *n_entries = total entries; ranks_host may be NULL (size query). */
int sn_get_device_tiles(sn_context *ctx, int32_t pass, int32_t env, int64_t *tile_starts_host, int32_t *ranks_host,
                        int64_t capacity, int64_t *n_entries);
/* Depth-sorted per-splat projection outputs of the last pass for env e (HOST, capacity M):
 * means2d (M,2), conics (M,3), depths (M), colors (M,3), alphas (M) -- project_cloud's arrays. */
int sn_get_projection(sn_context *ctx, int32_t pass, int32_t env, double *means2d, double *conics, double *depths,
                      double *colors, double *alphas, int64_t capacity);

/*
 * sample_pose + joint preparation for E x A (env, avatar) pairs at HOST sim_times (E):
 * writes device pose_q (E*A, J+1, 4) and pose_t (E*A, J+1, 3), root last, exactly as
 * rig.sample_pose returns them (after AvatarRuntime.clock). Returns SN_ERR_INVALID for a
 * negative sample time (rig.py:80-81).
 */
int sn_sample_pose(sn_context *ctx, const sn_avatars *avatars, const double *sim_times, int32_t n_envs,
                   double *pose_q, double *pose_t, void *stream);

/* lbs_deform for avatar `avatar`, whose gaussians are [g_begin, g_begin + g_count) of the set, at
 * explicit device poses pose_q (J+1,4) / pose_t (J+1,3), root last: writes device float64
 * positions (g_count,3) and rotations (g_count,4). */
int sn_skin_lbs(sn_context *ctx, const sn_avatars *avatars, int32_t avatar, int64_t g_begin, int64_t g_count,
                const double *pose_q, const double *pose_t, double *out_positions, double *out_rotations,
                void *stream);

/* blend_tile_range with the reference's exact argument list; all buffers are HOST memory
 * (float64 / int64 / int32 as in _kernels_cy.pyx:89-114); accumulates into the caller's buffers. */
int sn_blend_tile_range(int32_t t_begin, int32_t t_end, int32_t tiles_x, int32_t tile_size, int32_t width,
                        int32_t height, const int64_t *tile_starts, int64_t n_tiles_plus1, const int32_t *pair_splat,
                        int64_t n_pairs, const double *means2d, const double *conics, const double *depths,
                        const double *colors, const double *alphas, int64_t n_splats, double *color_acc,
                        double *alpha_acc, double *trans, double *depth_acc);

/*
 * Asset ingest on the device. Validation counters (DEVICE, 10 x uint64, zeroed by
 * the caller): [0..4] rows with non-finite positions / sh / opacity / log-scales / rotations,
 * [5] zero-norm rotations, [6] max |quat norm - 1| (float bits), [7] rows with negative weights,
 * [8] rows with more than 4 nonzero weights, [9] max |weight row sum - 1| (double bits); flags
 * (DEVICE, n bytes): per-row bits in the same order (bit 6 negative weight, bit 7 > 4 weights).
 * Rotations are renormalized in float32 exactly as GaussianCloud.validate (cloud.py:80-86) does.
 *
 * sn_unpack_ply -- ply.load_gaussian_ply (ply.py:76-120): `table` is the DEVICE copy of the
 *   row-major float32 vertex payload (n x n_props); cols (HOST, 14 + 3(K-1) int32) are the column
 *   indices of x y z f_dc_0..2 opacity scale_0..2 rot_0..3 f_rest_0..; outputs are the sn_cloud
 *   float32 buffers (pos+opacity (n,4), log-scales (n,4), rotations (n,4), sh (K*3, n)).
 * sn_unpack_bundle -- avatar.load_avatar_bundle (avatar.py:191-254) + AvatarBundle.validate
 *   (:155-176): canonical.f32 and weights.f32 (DEVICE copies) -> rows [row0, row0 + n) of the
 *   sn_avatars float64 canonical buffers, SH SoA (K*3, sh_stride), packed joints and (n,4) float64
 *   influence weights; row_sums (DEVICE, n) receives the numpy-order float64 row sums.
 */
int sn_unpack_ply(int64_t n, int32_t n_props, const float *table, const int32_t *cols, int32_t sh_k,
                  float *pos_opacity, float *log_scales, float *rotations, float *sh, uint8_t *flags,
                  uint64_t *counters, void *stream);
int sn_unpack_bundle(int64_t n, int32_t sh_k, int32_t n_joints, const float *canonical, const float *weights,
                     int64_t row0, int64_t sh_stride, double *pos_opacity, double *log_scales, double *rotations,
                     float *sh, uint32_t *joints, double *weights4, double *row_sums, uint8_t *flags,
                     uint64_t *counters, void *stream);

/* Skins wider than 4 influences (the CSR layout of sn_avatars), after sn_unpack_bundle of the same
 * rows: each row's nonzero weights.f32 entries (DEVICE, n x n_joints), ascending joint, written at
 * offsets[row] (DEVICE, caller-computed row offsets into the set's CSR arrays) as uint8 joint ids
 * and float64 weights, divided by row_sums when counters[9] (sn_unpack_bundle's largest row-sum
 * deviation) exceeds 1e-5 -- AvatarBundle.validate's renormalization (avatar.py:169-170). */
int sn_pack_influences(int64_t n, int32_t n_joints, const float *weights, const double *row_sums,
                       const uint64_t *counters, const uint32_t *offsets, uint8_t *infl_joint, double *infl_weight,
                       void *stream);

/* Observation payload / frame export (frame_io.py:11-31): uint8 RGB exactly as save_color_png
 * evaluates it on the same values (clip, x*255+0.5 in float64, truncation) and fp16 depth; depth16
 * may be NULL. sn_flip_rows writes (frames, H, W) float32 images bottom-to-top (the PFM row order). */
int sn_quantize_frames(int64_t npix, const float *color, const float *depth, uint8_t *rgb8, uint16_t *depth16,
                       void *stream);
int sn_flip_rows(int64_t frames, int32_t height, int32_t width, const float *src, float *dst, void *stream);

/* Self-check of the blend's fast exponential (ex2.approx, float32): largest relative error against
 * float64 exp(-d2/2) over every float d2 in [0, 9.5]. The blend's error budget assumes <= 3.5e-7. */
int sn_selftest_fast_exp(double *max_rel_err);

/* composite(front, back) on device float64 frames of npix pixels (renderer.py:151-166). */
int sn_composite(int64_t npix, const double *front_color, const double *front_alpha, const double *front_depth,
                 const double *back_color, const double *back_alpha, const double *back_depth, double *out_color,
                 double *out_alpha, double *out_depth, void *stream);

#ifdef __cplusplus
}
#endif
#endif
