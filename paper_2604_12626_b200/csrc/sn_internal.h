// sn_internal.h -- host-side declarations shared by the .cu translation units (not exported).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/splatnav_b200.h"

namespace sn {

struct SplatRec;
struct BlendGeo;

// Per-(env, avatar) pose block produced by the pose kernel and read by the skinning code:
// joint_mats (J x 12, rows of the 3x4 M_j = rigid(T_j) B_j^-1), eff_q (J x 4 effective joint
// quats q_root * q(M_j)), root (12: root rotation 3x3 row-major, root translation).
struct PoseView {
    const double *joint_mats;
    const double *eff_q;
    const double *root;
    int32_t n_joints;
    int32_t n_avatars;
};

// Launch parameters for one preprocess pass over an env chunk [e0, e0 + ec).
struct PrepArgs {
    const sn_camera *cams;  // device, indexed by global env id
    int32_t e0, ec;
    int32_t n_blocks;
    uint64_t *vismask;      // (n) bit e set: gaussian visible in env e0 + e
    uint32_t *blk_counts;   // (ec, n_blocks) -> exclusive offsets after scan
    unsigned long long *stats;  // (E, 5) device, may be null
    const uint8_t *avatar_active;  // (E, A), avatars only, may be null
    const uint8_t *avatar_cull;    // (E, A) whole-avatar cull codes, avatars only, may be null
    // emit outputs (unsorted, env-major, index order within env)
    const uint64_t *env_off;  // (ec + 1)
    uint32_t *keys;            // 32-bit depth keys: top bits of (env << z_bits | z_bits - z_base)
    int32_t key_shift;         // right shift that turns the 64-bit key into the 32-bit one
    uint32_t *vals;            // (unused: the depth sort's first pass generates identity values)
    SplatRec *recs;
    BlendGeo *geo;             // the blend's view of each record (same slots as recs)
    ushort4 *rects_tight;      // tiles the support ellipse's bounding box reaches (within rects)
    uint32_t *gid;             // original gaussian id per slot, or null (harness views off)
    ushort4 *rects;            // reference tile rectangle per slot, or null (harness views off)
    int32_t tiles_x, tiles_y;
    uint64_t z_base;
    int32_t z_bits;
    uint64_t cap;              // capacity of the per-splat buffers (writes past it are dropped)
    // depth slicing (scene pass, sn_render_opts.near_slice): z_cut (ec, device) per env -- visible
    // items with z < z_cut are near (full records, depth-sorted, streamed by the blend), the rest
    // far (not emitted: projected again by far_collect, and only where a tile's near list runs out
    // with live pixels); null = no slicing. blk_counts then has 2 ec rows (near, far) and env_off
    // 2 ec + 1 entries.
    const double *z_cut;
    uint64_t *nearmask;        // (n) bit e: visible and near in env e0 + e
    // lazy far (sliced, no RenderStats requested): in-depth items at z >= z_cut are classified far
    // without their projection -- vismask holds them as in-depth, far rows count them, and
    // far_collect applies the frame cull if a tile ever needs them
    int32_t lazy_far;
};

// sn_preprocess.cu
// per-env depth cuts of a sliced scene pass: z_cut[e] = the `frac` quantile of the z of a strided
// sample of the gaussians inside env e's view cone (+inf: no slicing for that env)
cudaError_t launch_near_cut(const sn_cloud &c, const PrepArgs &a, double frac, bool all_envs, double *z_cut,
                            cudaStream_t s);
cudaError_t launch_scene_count(const sn_cloud &c, const PrepArgs &a, cudaStream_t s);
cudaError_t launch_scene_emit(const sn_cloud &c, const PrepArgs &a, cudaStream_t s);
cudaError_t launch_avatar_count(const sn_avatars &av, const PoseView &pv, const PrepArgs &a, cudaStream_t s);
cudaError_t launch_avatar_emit(const sn_avatars &av, const PoseView &pv, const PrepArgs &a, cudaStream_t s);
cudaError_t launch_block_scan(uint32_t *blk_counts, int32_t n_blocks, int32_t ec, uint64_t *env_off,
                              cudaStream_t s);
cudaError_t launch_skin_range(const sn_avatars &av, int64_t g0, int64_t n, const PoseView &pv, double *out_pos,
                              double *out_rot, cudaStream_t s);

// one-thread copies of a device word into mapped pinned host memory (no copy engine)
cudaError_t launch_publish_u64(const uint64_t *src, uint64_t *mapped_dst, cudaStream_t s);
cudaError_t launch_publish_i32(const int32_t *src, int32_t *mapped_dst, cudaStream_t s);

// sn_rig.cu
cudaError_t launch_pose(const sn_avatars &av, const double *sim_times, int32_t n_envs, double *pose_q, double *pose_t,
                        double *joint_mats, double *eff_q, double *root, int32_t *err_flag, cudaStream_t s);
// (env, avatar) whole-avatar cull codes (0 test, kCullDepth, kCullFrame) after launch_pose
cudaError_t launch_avatar_cull(const sn_avatars &av, const PoseView &pv, const double *pose_t, const sn_camera *cams,
                               int32_t n_envs, unsigned long long *ext, uint8_t *codes, cudaStream_t s);
cudaError_t launch_joint_prep(const sn_avatars &av, int32_t avatar, const double *pose_q, const double *pose_t,
                              double *joint_mats, double *eff_q, double *root, cudaStream_t s);

// sn_far.cu (+ launch_far_collect in sn_preprocess.cu): the far buckets of a depth-sliced pass.
// Control words of a sliced pass (u64, PassWs::fctl): [0] unfinished tiles registered, [1] bucket
// items, [2] the continuation's work counter, [3] far-short flag, [4] far records written, [5] mask
// of the envs (in chunk) with unfinished tiles.
constexpr int kFarCtl = 8;
struct FarArgs {
    int32_t e0, ec, tiles_x, n_tiles;
    int32_t ub;                     // bucket-id bits at the top of the 32-bit item keys
    const uint64_t *vismask;        // (n) visible envs per gaussian
    const uint64_t *nearmask;       // (n) of those, the envs where it is in the near slice
    const sn_camera *cams;
    const int32_t *bucket_of;       // (ec * n_tiles): unfinished-tile index, or -1
    unsigned long long *fctl;       // control words (above)
    SplatRec *recs;                 // (cap_f) far splats that reach an unfinished tile: records,
    BlendGeo *geo;                  //   blend geometry
    uint32_t *gid;                  //   and gaussian index (the tie fix's second key)
    uint64_t cap_f;
    uint32_t *keys, *vals;          // (cap_b) bucket items: bucket << (32 - ub) | z key >> ub, far record
    uint64_t cap_b;
    uint2 *ranges;                  // (cap_u) each bucket's item range after the sort (zeroed)
    uint64_t z_base;
    int32_t z_bits;
};
cudaError_t launch_far_collect(const sn_cloud &c, const FarArgs &f, int64_t n, cudaStream_t s);
cudaError_t launch_far_tie_fix(const FarArgs &f, const uint32_t *keys, uint32_t *vals, cudaStream_t s);
cudaError_t launch_far_ranges(const FarArgs &f, const uint32_t *keys, cudaStream_t s);
// sets the conditional handle to (unfinished tiles registered != 0)
cudaError_t launch_far_cond(cudaGraphConditionalHandle h, const unsigned long long *fctl, cudaStream_t s);

// sn_bin.cu
struct BinArgs {
    int32_t ec, tiles_x, tiles_y, tile_bits, z_bits;
    const uint64_t *d_nvis;        // device: visible splats of the chunk (env_off[ec])
    uint64_t cap_v;                // host capacity of the per-splat buffers
    const uint64_t *d_npairs;      // device: tile pairs (binning 1)
    uint64_t cap_p;
    const uint32_t *keys_sorted;   // 32-bit depth keys after the sort
    uint32_t *vals_sorted;         // depth order -> unsorted record slot (tie-fixed in place)
    const SplatRec *recs_un;       // unsorted records (z for the tie fix)
    const uint32_t *gid_un;        // original ids per slot when the slot order is not the original
                                   // order (spatially reordered scene), else null
    const ushort4 *rects_in;
    const uint64_t *env_off;
    ushort4 *rects_out;
    ushort4 *batch_rects;    // (ceil(n_vis / 256)) union rect per 256-splat batch
    uint32_t *tiles_touched;
    uint64_t *pair_off;      // (n_vis + 1)
    uint32_t *pair_keys;
    uint32_t *pair_vals;
    uint2 *ranges;           // (ec << tile_bits)
    uint32_t *tile_list;     // (ec << tile_bits) the (env | tile) keys that hold pairs, in any order
    uint32_t *n_list;        // device count of tile_list (zeroed before ranges_kernel)
};
#ifndef SN_SUPER_BATCH
#define SN_SUPER_BATCH 32
#endif
constexpr int kSuperBatch = SN_SUPER_BATCH;  // batches per super-batch (8192 splats)
cudaError_t launch_permute(const BinArgs &b, cudaStream_t s);
cudaError_t launch_depth_tie_fix(const BinArgs &b, cudaStream_t s);
cudaError_t launch_super_rects(const BinArgs &b, ushort4 *super_rects, cudaStream_t s);
cudaError_t launch_duplicate(const BinArgs &b, cudaStream_t s);
cudaError_t launch_ranges(const BinArgs &b, const uint32_t *keys_sorted, cudaStream_t s);
constexpr int kCountWords = 6;  // published per (chunk, pass): visible, pairs, far records, unfinished
                                // tiles, bucket items, far-short flag
cudaError_t launch_publish_counts(const uint64_t *v, const uint64_t *p, const unsigned long long *fctl,
                                  uint64_t *mapped_dst, cudaStream_t s);

// sn_sort.cu (counts in device memory, grids sized by capacity)
size_t sort_temp_bytes(uint64_t cap);
bool radix_sort_pairs(void *temp, uint32_t *k0, uint32_t *v0, uint32_t *k1, uint32_t *v1, const uint64_t *d_n,
                      uint64_t cap, int bits, cudaStream_t s, int64_t *launches, bool identity_values = false,
                      const uint32_t *k_in = nullptr);
size_t scan_temp_bytes_dev(uint64_t cap);
cudaError_t scan_u32_to_u64(void *temp, const uint32_t *in, const uint64_t *d_n, uint64_t cap, uint64_t *out,
                            uint64_t *total_out, cudaStream_t s, int64_t *launches);

// sn_blend.cu
// Everything a pixel walk needs from one pass (scene or layer) over an env chunk.
struct PassView {
    int32_t source;         // 0: scan the env's depth-sorted rects (no tile lists); 1: tile lists
                            // (ranges + pair_vals); 2: rasterize_reference -- every splat of the env
    int32_t tile_bits;
    const ushort4 *rects;   // depth-sorted tile rectangles (source 0)
    const ushort4 *batch_rects;  // union rectangle of each global 256-splat batch of rects
    const ushort4 *super_rects;  // union rectangle of each kSuperBatch batches
    const uint2 *ranges;
    const uint32_t *pair_vals;
    const uint64_t *env_off;
    const SplatRec *recs;   // unsorted records
    const BlendGeo *geo;    // blend views in depth order (indexed like order)
    const uint32_t *order;  // depth-sorted index -> record slot
    // capacity guard: a pass whose counts exceeded its buffers produced no valid lists; its blend,
    // composite and fixups do nothing (the host re-runs the render with larger buffers)
    const uint64_t *d_nvis, *d_npairs;
    uint64_t cap_v, cap_p;
    // source 1: the non-empty (env | tile) keys and their count (ranges_kernel), and a work counter
    // the listed layer blend / composite take tiles from (zeroed with the count); null = grid mode
    const uint32_t *tile_list;
    const uint32_t *n_list;
    uint32_t *list_next;
    // depth slicing (scene pass, source 0): env_off has 2 ec + 1 entries (near rows, then far rows);
    // the tiles whose near list ran out with live / undecided pixels continue in their far bucket
    // (the far splats reaching the tile, projected by far_collect, sorted by (z, gaussian index))
    int32_t ec;
    int32_t sliced;
    int32_t n_tiles;
    const int32_t *far_bucket_of;           // (ec * n_tiles): bucket (unfinished tile) index, or -1
    const uint2 *far_ranges;                // (cap_u) bucket -> item range in far_order
    const uint32_t *far_order;              // bucket items in depth order (far record index)
    const SplatRec *far_recs;               // (cap_f) far records
    const BlendGeo *far_geo;                // (cap_f)
    const uint32_t *far_unfin_list;         // (cap_u): el << 16 | tile
    const unsigned long long *far_unfin;    // unfinished tiles registered (device)
    const unsigned long long *far_items;    // bucket items (device)
    const unsigned long long *far_nrec;     // far records (device)
    uint32_t far_cap_u;
    uint64_t cap_f, far_cap_b;
    uint32_t *far_next;                     // the continuation's work counter
    int32_t far_phase;                      // 1: the buckets are not built yet (the first fixup pass):
                                            // a float64 walk that needs its tile's bucket reports `out`
    unsigned long long *far_short;          // set by a float64 walk that ran out of a tile's near list
                                            // with no far bucket to continue in (the render is re-run
                                            // unsliced)
};
// A sliced pass whose far half outgrew its buffers (far items, unfinished tiles or bucket items): the
// continuation and the fixups do nothing (the host re-runs the render with larger buffers).
__device__ __forceinline__ bool far_overflow(const PassView &v) {
    return v.sliced && (*v.far_nrec > v.cap_f || *v.far_unfin > v.far_cap_u || *v.far_items > v.far_cap_b);
}
__device__ __forceinline__ bool pass_overflow(const PassView &v) {
    return *v.d_nvis > v.cap_v || (v.source == 1 && *v.d_npairs > v.cap_p);
}
struct BlendArgs {
    const sn_camera *cams;
    int32_t e0, ec, width, height, tiles_x;
    int32_t mode;           // 0 scene (background), 1 layer only, 2 layer composited over outputs
    PassView pv;            // this pass
    PassView back;          // mode 2: the scene pass of the same env chunk (exact composite fixups)
    float *color, *alpha, *depth;  // (E,H,W,[3]) outputs, indexed by global env
    float *derr;            // (E,H,W) error bound of the scene depth: mode 0 writes it (may be null),
                            // mode 2 reads it
    int32_t *contrib;       // (E,H,W) may be null
    // mode 2 (deferred composite): the layer frame -- normalized colour, alpha, depth (NaN = pending
    // fixup) and the error bounds of depth / alpha -- and a per-(env in chunk, tile) "has layer
    // splats" flag, all indexed like the outputs
    float *lcolor, *lalpha, *ldepth, *lderr, *laerr;
    uint8_t *tile_flag;
    uint32_t *fix_list;     // (ec*H*W, x2 when sliced) pixels deferred to the float64 fixup (el*H*W + pixel)
    unsigned *fix_count;    // device counter, zeroed before the blend
    const unsigned *fix_start;  // the first entry this fixup pass takes (null: 0; a sliced pass's second)
    int32_t force_exact;    // every pixel to the float64 fixup (sn_render_opts.exact)
    uint8_t *rgb8;          // (E,H,W,3) observation payload colour, or null (written where a pixel is final)
    uint16_t *depth16;      // (E,H,W) fp16 payload depth, or null
    unsigned long long *loads;  // device counter: records gathered into shared memory (may be null)
    unsigned long long *scans;  // device counter: rectangles examined by source-0 tiles (may be null)
    unsigned long long *contribs;  // device counter: (pixel, splat) contributions (may be null)
    // depth slicing: where an unfinished tile registers and saves its pixels' state (source 0 blend)
    unsigned long long *unfin_count;
    unsigned long long *unfin_envs;  // bit el: env el has an unfinished tile
    uint32_t *unfin_list;
    int32_t *bucket_of;
    float *state;           // (cap_u, kStateF, kBT)
};
// 1: the scene blend (streamed source) resolves its deferred pixels in the same CTA after the tile's
// walk, and a sliced pass needs only the fixup pass after the far buckets. Off: a CTA holding its
// slot for a latency-bound float64 walk (45% of tiles have one) costs the blend more than the
// separate fixup kernel (6,366 vs 6,460 frames/s at config 2)
#ifndef SN_INCTA_FIXUP
#define SN_INCTA_FIXUP 0
#endif
constexpr uint32_t kLateTile = 1u << 31;  // unfinished-list flag: registered by the first fixup pass (no state)
constexpr int kBT = 128;     // scene blend threads per tile (two pixels each, sn_blend.cu)
constexpr int kStateF = 22;  // floats per blend thread of a saved tile (2 pixels)
#ifndef SN_FIXUP_MIN_BLOCKS
#define SN_FIXUP_MIN_BLOCKS 4  // fixup CTAs (256 threads) per SM
#endif
constexpr int kFixupBlocks = 148 * SN_FIXUP_MIN_BLOCKS;
cudaError_t launch_blend(const BlendArgs &b, cudaStream_t s, bool fixup = true);  // blend (+ fixup, modes 0, 1)
cudaError_t launch_continue(const BlendArgs &b, cudaStream_t s);  // sliced pass: the unfinished tiles' far walk
cudaError_t launch_fixup(const BlendArgs &b, cudaStream_t s);     // modes 0, 1: the float64 fixups
cudaError_t launch_layer_composite(const BlendArgs &b, cudaStream_t s);  // mode 2: composite + fixup
cudaError_t fast_exp_selftest(double *max_rel_err);
// harness export of the streamed (source 0) tile lists of env el: counts (offsets == null) or entries
cudaError_t launch_tile_queue(const PassView &v, int el, int n_tiles, int tiles_x, uint32_t *counts,
                              const uint64_t *offsets, uint32_t *out, cudaStream_t s);
cudaError_t launch_composite64(int64_t npix, const double *fc, const double *fa, const double *fd, const double *bc,
                               const double *ba, const double *bd, double *oc, double *oa, double *od, cudaStream_t s);
cudaError_t launch_blend_tile_range(int t_begin, int t_end, int tiles_x, int tile_size, int width, int height,
                                    const int64_t *tile_starts, const int32_t *pair_splat, const double *means2d,
                                    const double *conics, const double *depths, const double *colors,
                                    const double *alphas, double *color_acc, double *alpha_acc, double *trans,
                                    double *depth_acc, cudaStream_t s);

// sn_assets.cu
cudaError_t launch_unpack_ply(int64_t n, int32_t n_props, const float *table, const int32_t *cols_host, int32_t sh_k,
                              float *pos_opacity, float *log_scales, float *rotations, float *sh, uint8_t *flags,
                              unsigned long long *cnt, cudaStream_t s);
cudaError_t launch_unpack_bundle(int64_t n, int32_t sh_k, int32_t J, const float *canonical, const float *weights,
                                 int64_t row0, int64_t sh_stride, double *pos_opacity, double *log_scales,
                                 double *rotations, float *sh, uint32_t *joints, double *wts, double *sums,
                                 uint8_t *flags, unsigned long long *cnt, cudaStream_t s);

cudaError_t launch_pack_csr(int64_t n, int32_t J, const float *weights, const double *sums,
                            const unsigned long long *cnt, const uint32_t *offsets, uint8_t *joint, double *weight,
                            cudaStream_t s);

cudaError_t launch_quantize(int64_t npix, const float *color, const float *depth, uint8_t *rgb8, uint16_t *depth16,
                            cudaStream_t s);
cudaError_t launch_flip_rows(int64_t frames, int32_t h, int32_t w, const float *src, float *dst, cudaStream_t s);

}  // namespace sn
