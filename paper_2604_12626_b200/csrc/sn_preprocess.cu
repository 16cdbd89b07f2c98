// sn_preprocess.cu -- K1/K2: (skinning +) projection, culling, SH colour and stream compaction.
//
// One thread per gaussian, looping over the env chunk's cameras, so a scene gaussian's
// parameters and its 3D covariance are read/built once per chunk instead of once per env.
// Two launches per pass:
//   count: visibility bitmask per gaussian + per-(env, block) visible counts + RenderStats
//          (warp ballots, aggregated in shared memory, one global atomic per block and field);
//   emit:  recomputes geometry only for visible (gaussian, env) pairs and writes 64-byte splat
//          records + 32-byte blend geometry at order-preserving positions (env-major, gaussian
//          index order within env), so a stable depth sort reproduces np.lexsort((idx, z))
//          (projection.py:184).
// A depth-sliced scene pass (sn_render_opts.near_slice) adds near_cut (each env's depth cut), marks
// the near items in the count and emits only those; the far ones are projected again, and only
// where a tile needs them, by far_collect (sn_far.cu). Without RenderStats the count classifies
// in-depth items beyond the cut as far from their depth alone (the lazy far classification).
// Avatars (sn_avatars) run the same pipeline with LBS skinning fused in front of the
// projection (rig.py:107-146): skinned positions/rotations never touch HBM.
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "sn_common.cuh"
#include "sn_internal.h"

#include <type_traits>

namespace sn {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// resident CTAs per SM the emit / avatar kernels are compiled for (register cap 65536 / (256 x N))
#ifndef SN_EMIT_MIN_BLOCKS
#define SN_EMIT_MIN_BLOCKS 3
#endif
#ifndef SN_COUNT_MIN_BLOCKS
#define SN_COUNT_MIN_BLOCKS 4
#endif
#ifndef SN_AVATAR_ENV_GROUP
#define SN_AVATAR_ENV_GROUP 4  // envs whose pose blocks the avatar count kernel stages per barrier pair
#endif
#ifndef SN_AVATAR_COUNT_MIN_BLOCKS
#define SN_AVATAR_COUNT_MIN_BLOCKS 4
#endif
#ifndef SN_AVATAR_MIN_BLOCKS
#define SN_AVATAR_MIN_BLOCKS 3
#endif

template <typename T>
__device__ __forceinline__ void load4(const T *p, double o[4]);
template <>
__device__ __forceinline__ void load4<float>(const float *p, double o[4]) {
    float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
}
template <>
__device__ __forceinline__ void load4<double>(const double *p, double o[4]) {
    double2 a = __ldg(reinterpret_cast<const double2 *>(p));
    double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = b.x;
    o[3] = b.y;
}

__device__ __forceinline__ double cam_z(const double p[3], const sn_camera &c) {
    return dot3_fma(p[0], p[1], p[2], c.rot[6], c.rot[7], c.rot[8]) + c.trans[2];
}

// Warp-aggregated stats: one shared atomic per warp and field.
__device__ __forceinline__ void tally(unsigned (*s_cnt)[5], int e, int code, bool input) {
    int lane = threadIdx.x & 31;
    unsigned b_in = __ballot_sync(kFull, input);
    unsigned b_keep = __ballot_sync(kFull, code == kKeep);
    unsigned b_depth = __ballot_sync(kFull, code == kCullDepth);
    unsigned b_deg = __ballot_sync(kFull, code == kDegenerate);
    unsigned b_frame = __ballot_sync(kFull, code == kCullFrame);
    if (lane == 0) {
        if (b_in) atomicAdd(&s_cnt[e][0], __popc(b_in));
        if (b_depth) atomicAdd(&s_cnt[e][1], __popc(b_depth));
        if (b_frame) atomicAdd(&s_cnt[e][2], __popc(b_frame));
        if (b_deg) atomicAdd(&s_cnt[e][3], __popc(b_deg));
        if (b_keep) atomicAdd(&s_cnt[e][4], __popc(b_keep));
    }
}

__device__ __forceinline__ void flush_counts(unsigned (*s_cnt)[5], const PrepArgs &a, const unsigned *s_near = nullptr,
                                             const unsigned *s_farz = nullptr, int n_input = -1) {
    int t = threadIdx.x;
    // (the input count is the block's gaussians, the same for every env, when the caller passes it)
    if (n_input >= 0 && t < a.ec) s_cnt[t][0] = (unsigned)n_input;
    __syncthreads();
    if (t < a.ec) {
        if (s_near) {  // depth-sliced: rows e (near) and ec + e (far: visible, or in-depth when lazy)
            a.blk_counts[(int64_t)t * a.n_blocks + blockIdx.x] = s_near[t];
            a.blk_counts[(int64_t)(a.ec + t) * a.n_blocks + blockIdx.x] = s_farz ? s_farz[t] : s_cnt[t][4] - s_near[t];
        } else {
            a.blk_counts[(int64_t)t * a.n_blocks + blockIdx.x] = s_cnt[t][4];
        }
    }
    if (a.stats != nullptr) {
        for (int i = t; i < a.ec * 5; i += blockDim.x) {  // ec * 5 can exceed the block (64 envs: 320)
            int e = i / 5, f = i % 5;  // sn_stats field order: input, depth, frame, degenerate, drawn
            unsigned v = s_cnt[e][f];
            if (v) atomicAdd(a.stats + (int64_t)(a.e0 + e) * 5 + f, (unsigned long long)v);
        }
    }
}

__device__ __forceinline__ void init_counts(unsigned (*s_cnt)[5], int ec) {
    for (int i = threadIdx.x; i < ec * 5; i += blockDim.x) s_cnt[i / 5][i % 5] = 0;
    __syncthreads();
}

// The chunk's cameras into shared memory (read per (gaussian, env) item: broadcasts instead of
// L1 round trips). Callers synchronize before use.
__device__ __forceinline__ void stage_cams(const PrepArgs &a, sn_camera *s_cam) {
    static_assert(sizeof(sn_camera) % sizeof(double) == 0, "sn_camera is copied as doubles");
    const double *src = reinterpret_cast<const double *>(a.cams + a.e0);
    double *dst = reinterpret_cast<double *>(s_cam);
    const int nd = a.ec * (int)(sizeof(sn_camera) / sizeof(double));
    for (int i = threadIdx.x; i < nd; i += blockDim.x) dst[i] = __ldg(src + i);
}

// Per-warp exclusive offsets for each env of the chunk; returns via s_woff.
__device__ __forceinline__ void warp_offsets(uint64_t mask, int ec, unsigned (*s_woff)[kBlock / 32]) {
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = 0; e < ec; ++e) {
        unsigned b = __ballot_sync(kFull, (mask >> e) & 1ull);
        if (lane == 0) s_woff[e][warp] = __popc(b);
    }
    __syncthreads();
    if (threadIdx.x < ec) {
        unsigned run = 0;
        for (int w = 0; w < kBlock / 32; ++w) {
            unsigned c = s_woff[threadIdx.x][w];
            s_woff[threadIdx.x][w] = run;
            run += c;
        }
    }
    __syncthreads();
}

// The tiles whose pixel centres the support {d2 <= 9} can reach: its bounding box mean +- (hx, hy)
// (BlendGeo, float, widened far beyond its rounding), intersected with the reference rectangle
// (3 sqrt(lambda_max) circle, renderer.py:83-86, which contains the ellipse). The reference's
// tile lists hold the other tiles of the rectangle too, but no pixel there passes d2 <= 9, so the
// blend and the exact walks skip them; the harness CSR views still report the reference lists.
__device__ __forceinline__ ushort4 tight_rect(const Geo &geo, const BlendGeo &bg, const int rect[4]) {
    int t0 = rect[0], t1 = rect[1], t2 = rect[2], t3 = rect[3];
    if (bg.hx < 1e30f && bg.hy < 1e30f) {
        const double ex = (double)bg.hx * (1.0 + 1e-5) + 1e-3, ey = (double)bg.hy * (1.0 + 1e-5) + 1e-3;
        // pixel p has its centre p + 0.5 inside [m - e, m + e] iff p in [m - e - 0.5, m + e - 0.5]
        t0 = max(t0, (int)floor((geo.mx - ex - 0.5) / kTile));
        t1 = min(t1, (int)floor((geo.mx + ex - 0.5) / kTile));
        t2 = max(t2, (int)floor((geo.my - ey - 0.5) / kTile));
        t3 = min(t3, (int)floor((geo.my + ey - 0.5) / kTile));
    }
    return t0 <= t1 && t2 <= t3 ? make_ushort4((unsigned short)t0, (unsigned short)t1, (unsigned short)t2,
                                               (unsigned short)t3)
                                : make_ushort4(0xffff, 0, 0xffff, 0);  // reaches no pixel
}

__device__ __forceinline__ void write_splat(const PrepArgs &a, int64_t pos, int e, const Geo &geo, double alpha,
                                            const float rgb[3], uint32_t gid) {
    if ((uint64_t)pos >= a.cap) return;  // overflow: the host re-runs the pass with larger buffers
    SplatRec r;
    r.mx = geo.mx;
    r.my = geo.my;
    r.ca = geo.ca;
    r.cb2 = 2.0 * geo.cb;  // exact; _kernels_cy.pyx:73 evaluates (2.0 * cb) first
    r.cc = geo.cc;
    r.alpha = alpha;
    r.z = geo.z;
    r.rgb = pack_rgb21(rgb);
    a.recs[pos] = r;
    const BlendGeo bg = make_blend_geo(r.ca, r.cb2, r.cc);
    a.geo[pos] = bg;
    unsigned long long zb = (unsigned long long)__double_as_longlong(geo.z);
    a.keys[pos] = (uint32_t)((((unsigned long long)e << a.z_bits) | (zb - a.z_base)) >> a.key_shift);
    // (the sort's first pass generates the identity values itself; the gaussian id and the
    // reference rectangle are written only for the harness views, PrepArgs::gid / rects non-null)
    if (a.gid) a.gid[pos] = gid;
    int rect[4];
    tile_rect(geo.mx, geo.my, geo.radius, a.tiles_x, a.tiles_y, rect);
    if (a.rects)
        a.rects[pos] = make_ushort4((unsigned short)rect[0], (unsigned short)rect[1], (unsigned short)rect[2],
                                    (unsigned short)rect[3]);
    a.rects_tight[pos] = tight_rect(geo, bg, rect);
}

// ------------------------------------------------------------------------------- scene

template <typename T>
__device__ __forceinline__ void load_scene(const sn_cloud &c, int64_t g, double p[3], double ls[3], double q[4],
                                           double &opacity) {
    double v[4];
    load4<T>(static_cast<const T *>(c.pos_opacity) + 4 * g, v);
    p[0] = v[0];
    p[1] = v[1];
    p[2] = v[2];
    opacity = v[3];
    load4<T>(static_cast<const T *>(c.log_scales) + 4 * g, v);
    ls[0] = v[0];
    ls[1] = v[1];
    ls[2] = v[2];
    load4<T>(static_cast<const T *>(c.rotations) + 4 * g, q);
}

// Visible (gaussian, env) items of a warp, compacted per round of kEmitRound envs so the
// float64 projection + SH run with full lanes (a scene gaussian is visible in ~1/4 of the envs;
// walking envs per lane would leave ~3/4 of the lanes idle). Item = lane | env << 5 | rank << 11,
// rank = position among the warp's visible lanes for that env (order-preserving output slot).
#ifndef SN_EMIT_ROUND
#define SN_EMIT_ROUND 16
#endif
#ifndef SN_COUNT_ROUND
#define SN_COUNT_ROUND 16
#endif
constexpr int kEmitRound = SN_EMIT_ROUND;
constexpr int kCountRound = SN_COUNT_ROUND;  // the count kernel's rounds (in-depth items)

__device__ __forceinline__ int build_round(uint64_t mask, int e_begin, int e_end, uint16_t *q) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int n = 0;
    for (int e = e_begin; e < e_end; ++e) {
        bool vis = (mask >> e) & 1ull;
        unsigned bal = __ballot_sync(kFull, vis);
        unsigned r = __popc(bal & lt);
        if (vis) q[n + r] = (uint16_t)(lane | (e << 5) | (r << 11));
        n += __popc(bal);
    }
    __syncwarp();
    return n;
}

// Per-item stats with warp aggregation: lanes holding the same (env, field) add once.
__device__ __forceinline__ void tally_item(unsigned (*s_cnt)[5], unsigned active, int e, int field) {
    unsigned same = __match_any_sync(active, e * 8 + field);
    int leader = __ffs(same) - 1;
    if ((int)(threadIdx.x & 31) == leader) atomicAdd(&s_cnt[e][field], __popc(same));
}

template <typename T>
__global__ void __launch_bounds__(kBlock, SN_COUNT_MIN_BLOCKS) scene_count_kernel(sn_cloud c, PrepArgs a) {
    __shared__ unsigned s_cnt[kMaxEnvChunk][5];
    __shared__ double s_geo[kBlock][9];  // position (3), cov3d (6)
    __shared__ unsigned long long s_vis[kBlock];
    __shared__ uint16_t s_q[kBlock / 32][32 * kCountRound];
    __shared__ sn_camera s_cam[kMaxEnvChunk];
    __shared__ unsigned long long s_nearbits[kBlock];  // depth slicing: visible and z < z_cut
    __shared__ unsigned s_near[kMaxEnvChunk];
    __shared__ unsigned s_farz[kMaxEnvChunk];  // lazy far: in-depth items at z >= z_cut
    __shared__ double s_zcut[kMaxEnvChunk];
    __shared__ uint8_t s_bcode[kMaxEnvChunk];  // per env, the whole block: 0 test, 1 out of depth, 2 far
    stage_cams(a, s_cam);
    if (threadIdx.x < a.ec) {
        s_near[threadIdx.x] = 0u;
        s_farz[threadIdx.x] = 0u;
        s_zcut[threadIdx.x] = a.z_cut ? a.z_cut[threadIdx.x] : INFINITY;
    }
    s_nearbits[threadIdx.x] = 0ull;
    init_counts(s_cnt, a.ec);  // (synchronizes)
    if (threadIdx.x < a.ec) {
        // A spatially ordered scene's 256-row block is decided per env from its bounding box where
        // the box is entirely out of (near, far), or (lazy far) entirely in depth at or beyond the
        // cut: the items' float64 z lies within the box's z range (plus a margin far above the
        // rounding of their dot products), so every item's depth test has the block's answer.
        uint8_t code = 0;
        if (c.block_bounds) {
            const float *bb = c.block_bounds + 8 * (int64_t)blockIdx.x;
            const sn_camera &cam = s_cam[threadIdx.x];
            const double cx = 0.5 * ((double)bb[0] + (double)bb[3]), cy = 0.5 * ((double)bb[1] + (double)bb[4]),
                         cz = 0.5 * ((double)bb[2] + (double)bb[5]);
            const double hx = 0.5 * ((double)bb[3] - (double)bb[0]), hy = 0.5 * ((double)bb[4] - (double)bb[1]),
                         hz = 0.5 * ((double)bb[5] - (double)bb[2]);
            const double zc = (cam.rot[6] * cx + cam.rot[7] * cy) + cam.rot[8] * cz + cam.trans[2];
            const double zr = fabs(cam.rot[6]) * hx + fabs(cam.rot[7]) * hy + fabs(cam.rot[8]) * hz;
            const double tol = 1e-9 * (1.0 + fabs(zc) + zr + fabs(cam.trans[2]));
            const double zmin = zc - zr - tol, zmax = zc + zr + tol;
            if (hx >= 0.0 && hy >= 0.0 && hz >= 0.0 && zmin == zmin && zmax == zmax) {  // (NaN: test)
                if (zmax < cam.near_ || zmin > cam.far_)
                    code = 1;
                else if (a.lazy_far && zmin > cam.near_ && zmax < cam.far_ && zmin > s_zcut[threadIdx.x])
                    code = 2;
            }
        }
        s_bcode[threadIdx.x] = code;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    bool valid = g < c.n;
    const int n_input = (int)min((int64_t)kBlock, c.n - (int64_t)blockIdx.x * kBlock);
    double p[3] = {0.0, 0.0, 0.0};
    if (valid) {
        double ls[3], q[4], opacity, cov[6];
        load_scene<T>(c, g, p, ls, q, opacity);
        build_cov3d(ls, q, cov);
        double *d = s_geo[threadIdx.x];
        d[0] = p[0];
        d[1] = p[1];
        d[2] = p[2];
#pragma unroll
        for (int k = 0; k < 6; ++k) d[3 + k] = cov[k];
    }
    s_vis[threadIdx.x] = 0ull;
    // depth cull for every env (4 fp64 ops per env), then full geometry only for in-depth items --
    // with a.lazy_far, only for the near ones: an in-depth item at z >= z_cut is far whatever its
    // frame cull, and far items are projected again (and culled) only if a tile needs them
    // Per-env warp counts are accumulated in registers, lane e & 31 holding env e's (lo: e < 32,
    // hi: e >= 32), and added to shared memory once per warp after the loop: a ballot and a popc
    // per env instead of a shared atomic per env and counter. The depth-culled count is for
    // RenderStats only; the in-depth far count for the lazy far rows only.
    unsigned out_lo = 0, out_hi = 0, fz_lo = 0, fz_hi = 0;
    const bool want_out = a.stats != nullptr;
    // one half (32 envs) of the chunk: 32-bit masks, no 64-bit variable shifts in the loop
    // (branch-free per env: an invalid thread's p is 0, its z finite and masked by `valid`; the
    // counters wanted are compile-time variants of the loop)
    auto depth_half = [&](auto lazy_tag, auto out_tag, const int e0, const int e1, unsigned &in_m, unsigned &fz_m,
                          unsigned &out_c, unsigned &fz_c) {
        constexpr bool kLazy = decltype(lazy_tag)::value, kOut = decltype(out_tag)::value;
        in_m = fz_m = 0u;
        for (int e = e0; e < e1; ++e) {
            const sn_camera &cam = s_cam[e];
            const int bc = s_bcode[e];  // (uniform)
            bool in, fz;
            if (bc == 1) {
                in = fz = false;
            } else if (kLazy && bc == 2) {
                in = fz = valid;
            } else {
                const double z = cam_z(p, cam);
                in = valid && (z > cam.near_) && (z < cam.far_);
                fz = kLazy && in && !(z < s_zcut[e]);
            }
            in_m |= (unsigned)(in && !fz) << (e - e0);
            fz_m |= (unsigned)fz << (e - e0);
            const bool mine = lane == e - e0;
            if (kOut) {
                const unsigned c = __popc(__ballot_sync(kFull, valid && !in));
                if (mine) out_c = c;
            }
            if (kLazy) {
                const unsigned c = __popc(__ballot_sync(kFull, fz));
                if (mine) fz_c = c;
            }
        }
    };
    auto depth_all = [&](auto lazy_tag, auto out_tag, unsigned &in_lo, unsigned &in_hi, unsigned &far_lo,
                         unsigned &far_hi) {
        depth_half(lazy_tag, out_tag, 0, min(a.ec, 32), in_lo, far_lo, out_lo, fz_lo);
        if (a.ec > 32) depth_half(lazy_tag, out_tag, 32, a.ec, in_hi, far_hi, out_hi, fz_hi);
    };
    unsigned in_lo = 0u, in_hi = 0u, far_lo = 0u, far_hi = 0u;
    if (a.lazy_far)
        depth_all(std::true_type{}, std::false_type{}, in_lo, in_hi, far_lo, far_hi);  // (lazy: no RenderStats)
    else if (want_out)
        depth_all(std::false_type{}, std::true_type{}, in_lo, in_hi, far_lo, far_hi);
    else
        depth_all(std::false_type{}, std::false_type{}, in_lo, in_hi, far_lo, far_hi);
    const uint64_t in_depth = ((uint64_t)in_hi << 32) | in_lo, far_z = ((uint64_t)far_hi << 32) | far_lo;
    if (lane < a.ec) {
        if (want_out && out_lo) atomicAdd(&s_cnt[lane][1], out_lo);
        if (fz_lo) atomicAdd(&s_farz[lane], fz_lo);
    }
    if (lane + 32 < a.ec) {
        if (want_out && out_hi) atomicAdd(&s_cnt[lane + 32][1], out_hi);
        if (fz_hi) atomicAdd(&s_farz[lane + 32], fz_hi);
    }
    const int64_t g0 = (int64_t)blockIdx.x * kBlock + warp * 32;
    uint16_t *qq = s_q[warp];
    // an in-depth item's frame cull: the float32 prefilter decides it where certain (a kept item's
    // radius bound < 3000 px also rules out the degenerate case); the undecided ones are queued at
    // the end of this warp's round list and take the float64 projection with full lanes
    auto resolve = [&](const unsigned it, const unsigned active, const int code) {
        const int l = it & 31, e = (it >> 5) & 63;
        // field: 2 frame, 3 degenerate, 4 drawn (sn_stats order); the lazy sliced pass counts its
        // near items below and needs none of these
        const int field = code == kKeep ? 4 : (code == kDegenerate ? 3 : 2);
        if (!a.lazy_far) tally_item(s_cnt, active, e, field);
        if (code == kKeep) {
            atomicOr(&s_vis[warp * 32 + l], 1ull << e);
            if (cam_z(s_geo[warp * 32 + l], s_cam[e]) < s_zcut[e]) atomicOr(&s_nearbits[warp * 32 + l], 1ull << e);
        }
    };
    for (int eb = 0; eb < a.ec; eb += kCountRound) {
        const int n = build_round(in_depth, eb, min(eb + kCountRound, a.ec), qq);
        int nu = 0;  // undecided items, compacted over the list's consumed head (nu <= k0 + 32)
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            unsigned it = 0;
            int code = -2;
            if (k < n) {
                it = qq[k];
                const int l = it & 31, e = (it >> 5) & 63;
                const double *d = s_geo[warp * 32 + l];
                code = frame_prefilter(d, (d[3] + d[6]) + d[8], s_cam[e]);
            }
            const unsigned und = __ballot_sync(kFull, code == -1);
            __syncwarp();  // (every lane has read its entry before the head is overwritten)
            if (code == -1) qq[nu + __popc(und & ((1u << lane) - 1u))] = (uint16_t)it;
            nu += __popc(und);
            const unsigned dec = __ballot_sync(kFull, code >= 0);
            if (code >= 0) resolve(it, dec, code);
        }
        __syncwarp();
        for (int k0 = 0; k0 < nu; k0 += 32) {
            const int k = k0 + lane;
            const unsigned active = __ballot_sync(kFull, k < nu);
            if (k >= nu) continue;
            const unsigned it = qq[k];
            const int l = it & 31, e = (it >> 5) & 63;
            const double *d = s_geo[warp * 32 + l];
            const double pp[3] = {d[0], d[1], d[2]};
            const double cov[6] = {d[3], d[4], d[5], d[6], d[7], d[8]};
            Geo geo;
            resolve(it, active, project_geo(pp, cov, s_cam[e], geo));
        }
        __syncwarp();
    }
    __syncthreads();
    // (lazy far: the far bits are the in-depth far items, not yet frame-culled)
    if (valid) a.vismask[g] = s_vis[threadIdx.x] | far_z;
    (void)g0;
    if (a.z_cut) {  // near items per env of this block (register-accumulated as above)
        const uint64_t nb = s_nearbits[threadIdx.x];
        if (valid) a.nearmask[g] = nb;
        unsigned n_lo = 0, n_hi = 0;
        for (int e = 0; e < a.ec; ++e) {
            const unsigned c = __popc(__ballot_sync(kFull, (nb >> e) & 1ull));
            if (lane == (e & 31)) (e < 32 ? n_lo : n_hi) = c;
        }
        if (lane < a.ec && n_lo) atomicAdd(&s_near[lane], n_lo);
        if (lane + 32 < a.ec && n_hi) atomicAdd(&s_near[lane + 32], n_hi);
        flush_counts(s_cnt, a, s_near, a.lazy_far ? s_farz : nullptr, n_input);
    } else {
        flush_counts(s_cnt, a, nullptr, nullptr, n_input);
    }
}

template <typename T>
__global__ void __launch_bounds__(kBlock, SN_EMIT_MIN_BLOCKS) scene_emit_kernel(sn_cloud c, PrepArgs a) {
    __shared__ unsigned s_woff[kMaxEnvChunk][kBlock / 32];
    __shared__ double s_geo[kBlock][10];  // position (3), cov3d (6), alpha
    __shared__ uint16_t s_q[kBlock / 32][32 * kEmitRound];
    __shared__ sn_camera s_cam[kMaxEnvChunk];
    stage_cams(a, s_cam);
    int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    bool valid = g < c.n;
    const uint64_t vis = valid ? a.vismask[g] : 0ull;
    const uint64_t near_bits = (valid && a.z_cut) ? a.nearmask[g] : ~0ull;
    const uint64_t mask = vis & near_bits;
    warp_offsets(mask, a.ec, s_woff);  // (synchronizes)
    if (!__any_sync(kFull, mask != 0)) return;
    const int warp = threadIdx.x >> 5;
    if (mask) {
        double p[3], ls[3], q[4], opacity, cov[6];
        load_scene<T>(c, g, p, ls, q, opacity);
        build_cov3d(ls, q, cov);
        double *d = s_geo[threadIdx.x];
        d[0] = p[0];
        d[1] = p[1];
        d[2] = p[2];
#pragma unroll
        for (int k = 0; k < 6; ++k) d[3 + k] = cov[k];
        d[9] = sigmoid(opacity);
    }
    const int64_t g0 = (int64_t)blockIdx.x * kBlock + warp * 32;
    uint16_t *q = s_q[warp];
    for (int eb = 0; eb < a.ec; eb += kEmitRound) {
        const int n = build_round(mask, eb, min(eb + kEmitRound, a.ec), q);
        for (int k = threadIdx.x & 31; k < n; k += 32) {
            const unsigned it = q[k];
            const int l = it & 31, e = (it >> 5) & 63, rank = it >> 11;
            const double *d = s_geo[warp * 32 + l];
            const double p[3] = {d[0], d[1], d[2]};
            const double cov[6] = {d[3], d[4], d[5], d[6], d[7], d[8]};
            const int64_t pos =
                (int64_t)a.env_off[e] + a.blk_counts[(int64_t)e * a.n_blocks + blockIdx.x] + s_woff[e][warp] + rank;
            const sn_camera &cam = s_cam[e];
            Geo geo;
            project_geo(p, cov, cam, geo);
            float dir[3], rgb[3];
            view_dir(p, cam, dir);
            eval_sh_f32(c.sh, c.n, g0 + l, c.sh_k, dir[0], dir[1], dir[2], rgb);
            write_splat(a, pos, e, geo, d[9], rgb, c.index ? __ldg(c.index + g0 + l) : (uint32_t)(g0 + l));
        }
        __syncwarp();
    }
    // (depth-sliced pass: the far items are not emitted -- far_collect projects them again, and only
    // for the envs with a tile whose near list ran out with live pixels)
}

// ------------------------------------------------------------------------------- avatars

// lbs_deform's per-gaussian sums over one influence list (get(k, j, w): the k-th nonzero influence,
// ascending joint order). NC = true: pose data in global memory (read-only path); false: generic
// loads (shared memory). ROT = false: the position only (q_out untouched) -- the count kernel's
// visibility test needs the rotation only for the few items its float32 prefilter cannot decide.
// 16-byte loads of pose data (joint matrices, quaternions and the root block are 16-byte aligned in
// global memory and in the count kernel's shared staging): half the load instructions
template <bool NC, int K>
__device__ __forceinline__ void ldp2(const double *p, double o[K]) {
    static_assert(K % 2 == 0, "pairs");
    const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
    for (int i = 0; i < K / 2; ++i) {
        const double2 v = NC ? __ldg(q + i) : q[i];
        o[2 * i] = v.x;
        o[2 * i + 1] = v.y;
    }
}

template <bool NC, bool ROT, typename Get>
__device__ __forceinline__ void skin_core(int n, Get get, const double P[4], const double Q[4], const double *jm,
                                          const double *eq, const double *root, double p_out[3], double q_out[4]) {
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    int dom = -1;
    double wmax = 0.0;
#pragma unroll
    for (int k = 0; k < n; ++k) {
        int j;
        double w;
        get(k, j, w);
        if (w == 0.0) continue;
        double M[12];
        ldp2<NC, 12>(jm + 12 * j, M);
        // einsum("jab,nb->jna") as numpy evaluates it: (r0 p0 + r2 p2) + r1 p1, then + offset;
        // einsum("nj,jnc->nc") accumulates over j sequentially, unfused (measured)
        double t0 = ((M[0] * P[0] + M[2] * P[2]) + M[1] * P[1]) + M[3];
        double t1 = ((M[4] * P[0] + M[6] * P[2]) + M[5] * P[1]) + M[7];
        double t2 = ((M[8] * P[0] + M[10] * P[2]) + M[9] * P[1]) + M[11];
        acc0 = acc0 + w * (t0 - P[0]);
        acc1 = acc1 + w * (t1 - P[1]);
        acc2 = acc2 + w * (t2 - P[2]);
        if (dom < 0 || w > wmax) {  // np.argmax: the first maximum
            wmax = w;
            dom = j;
        }
    }
    if (dom < 0) dom = 0;  // all-zero row: np.argmax picks joint 0
    double b0 = P[0] + acc0, b1 = P[1] + acc1, b2 = P[2] + acc2;
    double R[12];
    ldp2<NC, 12>(root, R);
    p_out[0] = dot3_fma(b0, b1, b2, R[0], R[1], R[2]) + R[9];
    p_out[1] = dot3_fma(b0, b1, b2, R[3], R[4], R[5]) + R[10];
    p_out[2] = dot3_fma(b0, b1, b2, R[6], R[7], R[8]) + R[11];
    if (!ROT) return;

    double qd[4];
    ldp2<NC, 4>(eq + 4 * dom, qd);
    double bq[4] = {0.0, 0.0, 0.0, 0.0};
    // (weights * signs) @ eff_quats: an FMA chain over j (OpenBLAS at production sizes; for
    // K >= 16 and up to ~1k rows OpenBLAS interleaves 8 accumulators instead -- a few-ulp
    // difference before the normalization, inside the 1e-12 LBS tolerance)
#pragma unroll
    for (int k = 0; k < n; ++k) {
        int j;
        double w;
        get(k, j, w);
        if (w == 0.0) continue;
        double qj[4];
        ldp2<NC, 4>(eq + 4 * j, qj);
        double dot = fma(qj[3], qd[3], fma(qj[2], qd[2], fma(qj[1], qd[1], qj[0] * qd[0])));
        double ws = w * (dot < 0.0 ? -1.0 : 1.0);
        bq[0] = fma(ws, qj[0], bq[0]);
        bq[1] = fma(ws, qj[1], bq[1]);
        bq[2] = fma(ws, qj[2], bq[2]);
        bq[3] = fma(ws, qj[3], bq[3]);
    }
    if (norm4(bq[0], bq[1], bq[2], bq[3]) < 1e-12) {
        bq[0] = qd[0];
        bq[1] = qd[1];
        bq[2] = qd[2];
        bq[3] = qd[3];
    }
    double nn = norm4(bq[0], bq[1], bq[2], bq[3]);
    double qn[4] = {bq[0] / nn, bq[1] / nn, bq[2] / nn, bq[3] / nn};
    quat_multiply(qn, Q, q_out);
}

// lbs_deform (rig.py:107-146) for one gaussian under one (env, avatar) pose. The influences are
// the row's nonzeros in ascending joint order, so the sums equal the dense N x J contractions
// (a zero weight adds +-0): the 4-slot layout, or the CSR rows of an arbitrary-width skin.
template <bool NC = true, bool ROT = true>
__device__ __forceinline__ void skin_one(const sn_avatars &av, int64_t g, const double *jm, const double *eq,
                                         const double *root, double p_out[3], double q_out[4]) {
    double P[4], Q[4];
    load4<double>(av.pos_opacity + 4 * g, P);
    if (ROT) load4<double>(av.rotations + 4 * g, Q);
    if (av.infl_offset == nullptr) {
        double W[4];
        load4<double>(av.weights + 4 * g, W);
        const uint32_t J4 = __ldg(av.joints + g);
        skin_core<NC, ROT>(
            4,
            [&](int k, int &j, double &w) {
                j = (J4 >> (8 * k)) & 0xff;
                w = W[k];
            },
            P, Q, jm, eq, root, p_out, q_out);
    } else {
        const uint32_t o0 = __ldg(av.infl_offset + g), o1 = __ldg(av.infl_offset + g + 1);
        const uint8_t *js = av.infl_joint + o0;
        const double *ws = av.infl_weight + o0;
        skin_core<NC, ROT>(
            (int)(o1 - o0),
            [&](int k, int &j, double &w) {
                j = __ldg(js + k);
                w = __ldg(ws + k);
            },
            P, Q, jm, eq, root, p_out, q_out);
    }
}

__device__ __forceinline__ void pose_ptrs(const PoseView &pv, int env, int avatar, const double *&jm,
                                          const double *&eq, const double *&root) {
    int64_t ea = (int64_t)env * pv.n_avatars + avatar;
    jm = pv.joint_mats + ea * pv.n_joints * 12;
    eq = pv.eff_q + ea * pv.n_joints * 4;
    root = pv.root + ea * 12;
}

__device__ __forceinline__ bool avatar_on(const PrepArgs &a, int n_avatars, int env, int avatar) {
    return a.avatar_active == nullptr || a.avatar_active[(int64_t)env * n_avatars + avatar] != 0;
}

// Pose blocks of the (at most two) avatars a CTA's gaussians belong to are staged in shared memory
// for each env, so the per-(gaussian, env) skinning reads joint matrices from shared memory
// instead of hammering L1 (avatars are contiguous and >= 256 gaussians in practice; other
// avatars fall back to global loads).
__host__ __device__ __forceinline__ int pose_block_doubles(int J) { return 16 * J + 12; }

// Pose blocks are staged for `group` envs per barrier pair (group x 2 blocks in shared memory).
__global__ void __launch_bounds__(kBlock, SN_AVATAR_COUNT_MIN_BLOCKS) avatar_count_kernel(sn_avatars av, PoseView pv, PrepArgs a,
                                                                                    int group) {
    __shared__ unsigned s_cnt[kMaxEnvChunk][5];
    __shared__ sn_camera s_cam[kMaxEnvChunk];
    extern __shared__ double s_pose[];  // group x 2 x (J*12 joint mats | J*4 quats | 12 root)
    stage_cams(a, s_cam);
    init_counts(s_cnt, a.ec);  // (synchronizes)
    int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    bool valid = g < av.n;
    int avatar = valid ? av.avatar_of[g] : 0;
    const int64_t g_first = (int64_t)blockIdx.x * kBlock;
    const int64_t g_last = min(av.n, g_first + kBlock) - 1;
    const int a_lo = av.avatar_of[g_first], a_hi = av.avatar_of[g_last];
    const int J = pv.n_joints, pb = pose_block_doubles(J);
    double ls[4];
    double tr_cov = 0.0;  // trace of cov3d = sum of squared scales (rotation-invariant)
    if (valid) {
        load4<double>(av.log_scales + 4 * g, ls);
        const double s0 = exp(ls[0]), s1 = exp(ls[1]), s2 = exp(ls[2]);
        tr_cov = (s0 * s0 + s1 * s1) + s2 * s2;
    }
    uint64_t mask = 0;
    for (int e = 0; e < a.ec; ++e) {
        int env = a.e0 + e;
        const uint8_t *cull = a.avatar_cull ? a.avatar_cull + (int64_t)env * av.n_avatars : nullptr;
        const int gs = e % group;  // this env's staging slot in the group
        if (gs == 0) {  // stage the group's pose blocks (skipping envs whose two avatars are culled whole)
            __syncthreads();
            const int ge = min(group, a.ec - e);
            // (segment by segment: contiguous copies, no per-element index divisions)
            for (int eg = 0; eg < ge; ++eg) {
                const int env_k = env + eg;
                const uint8_t *cull_k = a.avatar_cull ? a.avatar_cull + (int64_t)env_k * av.n_avatars : nullptr;
                if (cull_k && cull_k[a_lo] && cull_k[a_hi]) continue;
                for (int slot = 0; slot < (a_hi == a_lo ? 1 : 2); ++slot) {  // (one avatar: slot 1 is never read)
                    const int64_t ea = (int64_t)env_k * pv.n_avatars + (slot ? a_hi : a_lo);
                    double *dst = s_pose + (size_t)(eg * 2 + slot) * pb;
                    const double *jm = pv.joint_mats + ea * J * 12, *eq = pv.eff_q + ea * J * 4;
                    for (int o = threadIdx.x; o < 12 * J; o += kBlock) dst[o] = __ldg(jm + o);
                    for (int o = threadIdx.x; o < 4 * J; o += kBlock) dst[12 * J + o] = __ldg(eq + o);
                    if (threadIdx.x < 12) dst[16 * J + threadIdx.x] = __ldg(pv.root + ea * 12 + threadIdx.x);
                }
            }
            __syncthreads();
        }
        bool input = valid && avatar_on(a, av.n_avatars, env, avatar);
        int code = -1;
        if (input && cull && cull[avatar]) {
            // the whole avatar is depth- or frame-culled in this env, or wholly visible
            code = cull[avatar] == kWholeVisible ? kKeep : cull[avatar];
            if (code == kKeep) mask |= 1ull << e;
        } else if (input) {
            double p[3], q[4];
            const bool staged = avatar == a_lo || avatar == a_hi;
            const double *blk = s_pose + (size_t)gs * 2 * pb + (avatar == a_lo ? 0 : pb);
            const double *jm, *eq, *root;
            pose_ptrs(pv, env, avatar, jm, eq, root);
            if (staged)
                skin_one<false, false>(av, g, blk, blk + 12 * J, blk + 16 * J, p, q);
            else
                skin_one<true, false>(av, g, jm, eq, root, p, q);
            const sn_camera &cam = s_cam[env - a.e0];
            double z = cam_z(p, cam);
            if (!((z > cam.near_) && (z < cam.far_))) {
                code = kCullDepth;
            } else if ((code = frame_prefilter(p, tr_cov, cam)) < 0) {
                if (staged)
                    skin_one<false>(av, g, blk, blk + 12 * J, blk + 16 * J, p, q);
                else
                    skin_one<true>(av, g, jm, eq, root, p, q);
                double cov[6];
                build_cov3d(ls, q, cov);
                Geo geo;
                code = project_geo(p, cov, cam, geo);
            }
            if (code == kKeep) mask |= 1ull << e;
        }
        tally(s_cnt, e, code, input);
    }
    if (valid) a.vismask[g] = mask;
    flush_counts(s_cnt, a);
}

__global__ void __launch_bounds__(kBlock, SN_AVATAR_MIN_BLOCKS) avatar_emit_kernel(sn_avatars av, PoseView pv, PrepArgs a) {
    __shared__ unsigned s_woff[kMaxEnvChunk][kBlock / 32];
    __shared__ uint16_t s_q[kBlock / 32][32 * kEmitRound];
    __shared__ sn_camera s_cam[kMaxEnvChunk];
    stage_cams(a, s_cam);
    int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    bool valid = g < av.n;
    uint64_t mask = valid ? a.vismask[g] : 0ull;
    warp_offsets(mask, a.ec, s_woff);
    if (!__any_sync(kFull, mask != 0)) return;
    const int warp = threadIdx.x >> 5;
    const int64_t g0 = (int64_t)blockIdx.x * kBlock + warp * 32;
    uint16_t *q = s_q[warp];
    for (int eb = 0; eb < a.ec; eb += kEmitRound) {
        const int n = build_round(mask, eb, min(eb + kEmitRound, a.ec), q);
        for (int k = threadIdx.x & 31; k < n; k += 32) {
            const unsigned it = q[k];
            const int l = it & 31, e = (it >> 5) & 63, rank = it >> 11;
            const int64_t gi = g0 + l;
            const int env = a.e0 + e;
            const int avatar = av.avatar_of[gi];
            const int64_t pos =
                (int64_t)a.env_off[e] + a.blk_counts[(int64_t)e * a.n_blocks + blockIdx.x] + s_woff[e][warp] + rank;
            const double *jm, *eq, *root;
            pose_ptrs(pv, env, avatar, jm, eq, root);
            double p[3], qr[4], ls[4], cov[6];
            skin_one(av, gi, jm, eq, root, p, qr);
            load4<double>(av.log_scales + 4 * gi, ls);
            build_cov3d(ls, qr, cov);
            const sn_camera &cam = s_cam[env - a.e0];
            Geo geo;
            project_geo(p, cov, cam, geo);
            float dir[3], rgb[3];
            view_dir(p, cam, dir);
            eval_sh_f32(av.sh, av.n, gi, av.sh_k, dir[0], dir[1], dir[2], rgb);
            write_splat(a, pos, e, geo, sigmoid(__ldg(av.pos_opacity + 4 * gi + 3)), rgb, (uint32_t)gi);
        }
        __syncwarp();
    }
}

// Standalone skinning (lbs_deform API): float64 positions/rotations of one avatar.
__global__ void __launch_bounds__(kBlock) skin_kernel(sn_avatars av, int64_t g0, int64_t n, PoseView pv,
                                                      double *out_pos, double *out_rot) {
    int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const double *jm, *eq, *root;
    pose_ptrs(pv, 0, 0, jm, eq, root);
    double p[3], q[4];
    skin_one(av, g0 + i, jm, eq, root, p, q);
    out_pos[3 * i] = p[0];
    out_pos[3 * i + 1] = p[1];
    out_pos[3 * i + 2] = p[2];
    out_rot[4 * i] = q[0];
    out_rot[4 * i + 1] = q[1];
    out_rot[4 * i + 2] = q[2];
    out_rot[4 * i + 3] = q[3];
}

// ------------------------------------------------------------------------------- depth slicing

// z_cut per env of the chunk: the `frac` quantile of the depth of a strided sample of the gaussians
// inside the env's view cone (camera-space |x| <= z (cx + 64) / fx, same for y, near < z < far: a
// cheap stand-in for the visible set), from a 64-bins-per-octave log histogram. Envs with too few
// expected visible splats for slicing to pay get +inf (everything near).
constexpr int kCutBins = 1024;
constexpr int kCutPerOctave = 64;
constexpr double kMinSliced = 131072.0;  // expected visible splats below which an env is not sliced
constexpr int kCutThreads = kCutBins;  // one histogram bin per thread for the scan
template <typename T>
__global__ void __launch_bounds__(kCutThreads) near_cut_kernel(sn_cloud c, PrepArgs a, int64_t stride, double frac,
                                                              double min_visible, double *z_cut) {
    using Scan = cub::BlockScan<unsigned, kCutThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned s_h[kCutBins];
    const sn_camera cam = a.cams[a.e0 + blockIdx.x];
    s_h[threadIdx.x] = 0u;
    __syncthreads();
    const double lnear = log2(cam.near_);
    const double mx = (cam.cx + 64.0) / cam.fx, my = (cam.cy + 64.0) / cam.fy;
    for (int64_t g = (int64_t)threadIdx.x * stride; g < c.n; g += (int64_t)kCutThreads * stride) {
        double v[4];
        load4<T>(static_cast<const T *>(c.pos_opacity) + 4 * g, v);
        const double p[3] = {v[0], v[1], v[2]};
        const double *w = cam.rot;
        const double z = dot3_fma(p[0], p[1], p[2], w[6], w[7], w[8]) + cam.trans[2];
        if (!(z > cam.near_ && z < cam.far_)) continue;
        const double x = dot3_fma(p[0], p[1], p[2], w[0], w[1], w[2]) + cam.trans[0];
        const double y = dot3_fma(p[0], p[1], p[2], w[3], w[4], w[5]) + cam.trans[1];
        if (fabs(x) > z * mx || fabs(y) > z * my) continue;
        const int bin = min(kCutBins - 1, max(0, (int)((log2(z) - lnear) * kCutPerOctave)));
        atomicAdd(&s_h[bin], 1u);
    }
    __syncthreads();
    // inclusive prefix over the bins: the cut is the upper edge of the first bin reaching frac
    const unsigned h = s_h[threadIdx.x];
    unsigned excl, tot;
    Scan(tmp).ExclusiveSum(h, excl, tot);
    const bool slice = tot > 0 && (double)tot * (double)stride >= min_visible;
    const double target = frac * (double)tot;
    if (threadIdx.x == 0) z_cut[blockIdx.x] = INFINITY;  // (no bin reaches the target, or no slicing)
    __syncthreads();
    if (slice && (double)(excl + h) >= target && (double)excl < target) {  // exactly one thread
        const double cut = exp2(lnear + (double)(threadIdx.x + 1) / kCutPerOctave);
        z_cut[blockIdx.x] = cut < cam.far_ ? cut : INFINITY;
    }
}

// The far half of a depth-sliced scene pass, for the envs with unfinished tiles (a tile whose near
// list ran out with a live or undecided pixel, fctl[5]): every visible far (gaussian, env) item of
// those envs is projected again exactly as the emit projects a near one; one that reaches an
// unfinished tile of its env gets a far record (SplatRec, BlendGeo, gaussian index) and a bucket
// item per such tile, keyed (bucket << (32 - ub)) | (32-bit depth key >> ub). The items are sorted
// next (sn_far.cu). Reservations are warp-aggregated.
template <typename T>
__global__ void __launch_bounds__(kBlock, SN_EMIT_MIN_BLOCKS) far_collect_kernel(sn_cloud c, FarArgs f) {
    __shared__ double s_geo[kBlock][10];  // position (3), cov3d (6), alpha
    __shared__ uint16_t s_q[kBlock / 32][32 * kEmitRound];
    __shared__ sn_camera s_cam[kMaxEnvChunk];
    const uint64_t envs = *(volatile unsigned long long *)(f.fctl + 5);
    if (envs == 0) return;  // no unfinished tile anywhere (uniform)
    {
        const double *src = reinterpret_cast<const double *>(f.cams + f.e0);
        double *dst = reinterpret_cast<double *>(s_cam);
        const int nd = f.ec * (int)(sizeof(sn_camera) / sizeof(double));
        for (int i = threadIdx.x; i < nd; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    const int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const uint64_t mask = g < c.n ? (f.vismask[g] & ~f.nearmask[g] & envs) : 0ull;
    if (!__syncthreads_or(mask != 0ull)) return;  // (also the barrier after the camera staging)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (mask) {
        double p[3], ls[3], q[4], opacity, cov[6];
        load_scene<T>(c, g, p, ls, q, opacity);
        build_cov3d(ls, q, cov);
        double *d = s_geo[threadIdx.x];
        d[0] = p[0];
        d[1] = p[1];
        d[2] = p[2];
#pragma unroll
        for (int k = 0; k < 6; ++k) d[3 + k] = cov[k];
        d[9] = sigmoid(opacity);
    }
    const int64_t g0 = (int64_t)blockIdx.x * kBlock + warp * 32;
    uint16_t *qq = s_q[warp];
    const uint32_t lt = (1u << lane) - 1u;
    for (int eb = 0; eb < f.ec; eb += kEmitRound) {
        const int n = build_round(mask, eb, min(eb + kEmitRound, f.ec), qq);  // (warp-uniform n)
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            int e = 0, l = 0;
            Geo geo;
            ushort4 r = make_ushort4(0xffff, 0, 0xffff, 0);
            unsigned hits = 0;
            if (k < n) {
                const unsigned it = qq[k];
                l = it & 31;
                e = (it >> 5) & 63;
                const double *d = s_geo[warp * 32 + l];
                const double p[3] = {d[0], d[1], d[2]};
                const double cov[6] = {d[3], d[4], d[5], d[6], d[7], d[8]};
                // kKeep as the count kernel kept it -- or, lazily classified far items (in depth, not
                // yet frame-culled), whatever the reference's cull decides
                if (project_geo(p, cov, s_cam[e], geo) == kKeep) {
                    const BlendGeo bg = make_blend_geo(geo.ca, 2.0 * geo.cb, geo.cc);  // as write_splat
                    int rect[4];
                    tile_rect(geo.mx, geo.my, geo.radius, f.tiles_x, f.n_tiles / f.tiles_x, rect);
                    r = tight_rect(geo, bg, rect);
                    const int32_t *bo = f.bucket_of + (int64_t)e * f.n_tiles;
                    for (int ty = r.z; ty <= (int)r.w && r.x <= r.y; ++ty)
                        for (int tx = r.x; tx <= (int)r.y; ++tx) hits += __ldg(bo + ty * f.tiles_x + tx) >= 0;
                }
            }
            const unsigned hm = __ballot_sync(kFull, hits > 0);
            if (!hm) continue;
            unsigned incl = hits;  // inclusive warp scan of the item counts
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned o = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += o;
            }
            unsigned long long jb = 0, ib = 0;
            if (lane == 31) {
                jb = atomicAdd(f.fctl + 4, (unsigned long long)__popc(hm));
                ib = atomicAdd(f.fctl + 1, (unsigned long long)incl);
            }
            jb = __shfl_sync(kFull, jb, 31);
            ib = __shfl_sync(kFull, ib, 31);
            if (!hits) continue;
            const uint64_t j = jb + __popc(hm & lt);
            if (j >= f.cap_f) continue;  // overflow: the host re-runs with larger buffers
            const double *d = s_geo[warp * 32 + l];
            const double p[3] = {d[0], d[1], d[2]};
            float dir[3], rgb[3];
            view_dir(p, s_cam[e], dir);
            eval_sh_f32(c.sh, c.n, g0 + l, c.sh_k, dir[0], dir[1], dir[2], rgb);
            SplatRec rec;
            rec.mx = geo.mx;
            rec.my = geo.my;
            rec.ca = geo.ca;
            rec.cb2 = 2.0 * geo.cb;
            rec.cc = geo.cc;
            rec.alpha = d[9];
            rec.z = geo.z;
            rec.rgb = pack_rgb21(rgb);
            f.recs[j] = rec;
            f.geo[j] = make_blend_geo(rec.ca, rec.cb2, rec.cc);
            f.gid[j] = c.index ? __ldg(c.index + g0 + l) : (uint32_t)(g0 + l);
            const unsigned long long off = (unsigned long long)__double_as_longlong(geo.z) - f.z_base;
            const uint32_t zkey = (uint32_t)(f.z_bits > 32 ? off >> (f.z_bits - 32) : off << (32 - f.z_bits));
            const uint32_t zlo = zkey >> f.ub;
            uint64_t pos = ib + incl - hits;
            const int32_t *bo = f.bucket_of + (int64_t)e * f.n_tiles;
            for (int ty = r.z; ty <= (int)r.w; ++ty)
                for (int tx = r.x; tx <= (int)r.y; ++tx) {
                    const int32_t u = __ldg(bo + ty * f.tiles_x + tx);
                    if (u < 0) continue;
                    if (pos < f.cap_b) {
                        f.keys[pos] = ((uint32_t)u << (32 - f.ub)) | zlo;
                        f.vals[pos] = (uint32_t)j;
                    }
                    ++pos;
                }
        }
        __syncwarp();
    }
}

// Per-env exclusive scan of the per-block visible counts (in place), then env offsets.
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) block_scan_kernel(uint32_t *blk_counts, int32_t n_blocks,
                                                                  uint64_t *env_tot) {
    using Scan = cub::BlockScan<uint32_t, kScanThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t carry;
    uint32_t *row = blk_counts + (int64_t)blockIdx.x * n_blocks;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n_blocks; base += kScanThreads) {
        int i = base + threadIdx.x;
        uint32_t v = i < n_blocks ? row[i] : 0u, ex, total;
        Scan(tmp).ExclusiveSum(v, ex, total);
        uint32_t c = carry;
        if (i < n_blocks) row[i] = c + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + total;
        __syncthreads();
    }
    if (threadIdx.x == 0) env_tot[blockIdx.x] = carry;
}

__global__ void env_offsets_kernel(int32_t ec, uint64_t *env_off) {
    // env_off holds per-env totals in [1..ec]; make it an exclusive prefix with env_off[0] = 0
    uint64_t run = 0;
    for (int e = 0; e < ec; ++e) {
        uint64_t t = env_off[e + 1];
        env_off[e] = run;
        run += t;
    }
    env_off[ec] = run;
}

__global__ void publish_u64_kernel(const uint64_t *src, volatile uint64_t *dst) { *dst = *src; }
__global__ void publish_i32_kernel(const int32_t *src, volatile int32_t *dst) { *dst = *src; }

}  // namespace

cudaError_t launch_publish_u64(const uint64_t *src, uint64_t *mapped_dst, cudaStream_t s) {
    publish_u64_kernel<<<1, 1, 0, s>>>(src, mapped_dst);
    return cudaGetLastError();
}

cudaError_t launch_publish_i32(const int32_t *src, int32_t *mapped_dst, cudaStream_t s) {
    publish_i32_kernel<<<1, 1, 0, s>>>(src, mapped_dst);
    return cudaGetLastError();
}

cudaError_t launch_scene_count(const sn_cloud &c, const PrepArgs &a, cudaStream_t s) {
    if (c.dtype == SN_FLOAT64)
        scene_count_kernel<double><<<a.n_blocks, kBlock, 0, s>>>(c, a);
    else
        scene_count_kernel<float><<<a.n_blocks, kBlock, 0, s>>>(c, a);
    return cudaGetLastError();
}

cudaError_t launch_scene_emit(const sn_cloud &c, const PrepArgs &a, cudaStream_t s) {
    if (c.dtype == SN_FLOAT64)
        scene_emit_kernel<double><<<a.n_blocks, kBlock, 0, s>>>(c, a);
    else
        scene_emit_kernel<float><<<a.n_blocks, kBlock, 0, s>>>(c, a);
    return cudaGetLastError();
}

cudaError_t launch_avatar_count(const sn_avatars &av, const PoseView &pv, const PrepArgs &a, cudaStream_t s) {
    const size_t blk = sizeof(double) * 2 * (size_t)pose_block_doubles(pv.n_joints);
    const int group = (int)std::max<size_t>(1, std::min<size_t>(SN_AVATAR_ENV_GROUP, (40 * 1024) / blk));
    const size_t smem = blk * group;
    // dynamic + static (cameras, counters) may pass the default 48 KB: opt in to the dynamic size
    // (a function attribute is per device: remember the opted size per device ordinal)
    constexpr int kMaxDevices = 64;
    static size_t opted[kMaxDevices] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices || smem > opted[dev]) {
        e = cudaFuncSetAttribute(avatar_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < kMaxDevices) opted[dev] = smem;
    }
    avatar_count_kernel<<<a.n_blocks, kBlock, smem, s>>>(av, pv, a, group);
    return cudaGetLastError();
}

cudaError_t launch_avatar_emit(const sn_avatars &av, const PoseView &pv, const PrepArgs &a, cudaStream_t s) {
    avatar_emit_kernel<<<a.n_blocks, kBlock, 0, s>>>(av, pv, a);
    return cudaGetLastError();
}

cudaError_t launch_near_cut(const sn_cloud &c, const PrepArgs &a, double frac, bool all_envs, double *z_cut,
                            cudaStream_t s) {
    const int64_t stride = std::max<int64_t>(1, c.n / 65536);  // ~64k samples per env
    const double min_visible = all_envs ? 0.0 : kMinSliced;
    if (c.dtype == SN_FLOAT64)
        near_cut_kernel<double><<<a.ec, kCutThreads, 0, s>>>(c, a, stride, frac, min_visible, z_cut);
    else
        near_cut_kernel<float><<<a.ec, kCutThreads, 0, s>>>(c, a, stride, frac, min_visible, z_cut);
    return cudaGetLastError();
}

cudaError_t launch_far_collect(const sn_cloud &c, const FarArgs &f, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((n + kBlock - 1) / kBlock);
    if (c.dtype == SN_FLOAT64)
        far_collect_kernel<double><<<grid, kBlock, 0, s>>>(c, f);
    else
        far_collect_kernel<float><<<grid, kBlock, 0, s>>>(c, f);
    return cudaGetLastError();
}

cudaError_t launch_block_scan(uint32_t *blk_counts, int32_t n_blocks, int32_t ec, uint64_t *env_off,
                              cudaStream_t s) {
    block_scan_kernel<<<ec, kScanThreads, 0, s>>>(blk_counts, n_blocks, env_off + 1);
    env_offsets_kernel<<<1, 1, 0, s>>>(ec, env_off);
    return cudaGetLastError();
}

cudaError_t launch_skin_range(const sn_avatars &av, int64_t g0, int64_t n, const PoseView &pv, double *out_pos,
                              double *out_rot, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    skin_kernel<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, s>>>(av, g0, n, pv, out_pos, out_rot);
    return cudaGetLastError();
}

}  // namespace sn
