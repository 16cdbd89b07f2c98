// sn_api.cu -- the C ABI (include/splatnav_b200.h): context/workspace and pass orchestration.
//
// A pass (scene, or the concatenated avatar layer) over a chunk of <= 64 envs is:
//   [near cut] -> count -> per-env block scan -> emit -> depth sort + tie fix -> permute
//   -> (avatar layer: pair-offset scan -> duplicate -> pair sort -> ranges) -> blend
//   -> (sliced scene pass: fixups over the near lists -> far collect -> item sort -> continuation)
//   -> fixups, and the layer's deferred composite on the scene stream.
// No host round trip inside a render: buffers are sized by host-side capacities, the counts stay
// on the device and are published to mapped host memory; sn_render_wait checks them afterwards
// and a render that outgrew its buffers is re-run with larger ones (buffers only grow, so a
// steady-state batch loop allocates nothing).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "sn_common.cuh"
#include "sn_internal.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

#define SN_CUDA(expr)                                                                                      \
    do {                                                                                                   \
        cudaError_t _e = (expr);                                                                           \
        if (_e != cudaSuccess)                                                                             \
            return fail(SN_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));                  \
    } while (0)

#define SN_CHECK(cond, msg)                         \
    do {                                            \
        if (!(cond)) return fail(SN_ERR_INVALID, msg); \
    } while (0)

struct Buf {
    void *p = nullptr;
    size_t cap = 0;
    template <typename T>
    T *as() const {
        return static_cast<T *>(p);
    }
};

int ensure(Buf &b, size_t bytes) {
    if (bytes <= b.cap && b.p != nullptr) return SN_OK;
    size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(SN_ERR_NOMEM, std::string("cudaMalloc(") + std::to_string(want) + "): " + cudaGetErrorString(e));
    }
    b.cap = want;
    return SN_OK;
}

#define SN_ENSURE(buf, bytes)                 \
    do {                                      \
        int _r = ensure((buf), (bytes));      \
        if (_r != SN_OK) return _r;           \
    } while (0)

int bit_length(uint64_t v) { return v == 0 ? 0 : 64 - __builtin_clzll(v); }

// Depth slicing (sn_render_opts.near_slice): auto-on for scenes of at least this many gaussians
// (rendered without harness views); the near slice is this quantile of each env's sampled depths
// (SN_NEAR_FRAC overrides it, for tuning).
// the far pipeline as a conditional graph (SN_FAR_GRAPH=0: plain launches)
bool far_graphs_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("SN_FAR_GRAPH");
        return !(e && e[0] == '0');
    }();
    return on;
}
// auto slicing (near_slice = -1) from this scene size up; SN_SLICE_MIN overrides (tuning)
int64_t slice_min_gaussians() {
    static const int64_t m = [] {
        const char *e = std::getenv("SN_SLICE_MIN");
        return e ? (int64_t)std::atoll(e) : (int64_t)500000;
    }();
    return m;
}
double near_frac() {
    static const double f = [] {
        const char *e = std::getenv("SN_NEAR_FRAC");
        const double v = e ? std::atof(e) : 0.0;
        return v > 0.0 && v <= 1.0 ? v : 0.02;
    }();
    return f;
}

uint64_t dbits(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

struct PassWs {
    Buf vismask, blk_counts, env_off, keys_un, keys_s, vals_un, vals_s, recs_un, geo_un, gid_un, rects_un, rects_tun, rects,
        tiles, pair_off, pkeys_a, pkeys_b, pvals_a, pvals_b, ranges, temp, batch_rects, super_rects, fix, counts, tlist,
        tlist_cnt;
    // depth slicing (scene pass): cuts, near bits, control words, unfinished tiles and their state,
    // far records of the splats reaching them, bucket items (sort buffers) and bucket ranges
    Buf zcut, nearmask, fctl, unfin_list, bucket_of, state, frec, fgeo, fgid, franges, bkey_a, bkey_b, bval_a,
        bval_b, ftemp;
    uint64_t cap_f = 0, cap_b = 0;  // far records, bucket items
    uint32_t cap_u = 0;             // unfinished tiles
    int32_t sliced = 0;
    uint32_t *far_order = nullptr;  // where the bucket sort left the item order (far record indices)
    uint64_t cap_v = 0, cap_p = 0;  // capacities of the per-splat / per-pair buffers
    // metadata of the last chunk rendered by this pass
    int32_t e0 = 0, ec = 0, tiles_x = 0, tiles_y = 0, tile_bits = 0, tiled = 1, valid = 0, binning = 0, views = 1;
    int64_t n_vis = 0, n_pairs = 0;
    sn::BlendArgs bl{};        // the last blend's arguments (the deferred composite reuses them)
    int64_t *work = nullptr;   // mode 2: work counters still to be collected after the composite
};

}  // namespace

struct sn_context {
    PassWs pass[2];
    Buf cams, times, derr, jm, eq, root, err, pose_q, pose_t, loads, fixcnt, av_ext, av_cull, rpose_q, rpose_t;
    Buf lcolor, lalpha, ldepth, lderr, laerr, tile_flag;  // deferred-composite layer frame
    // mapped pinned words the device writes with a one-thread kernel: reading a total this way
    // never queues behind other streams' bulk copies on the device->host copy engine
    uint64_t *h_tot = nullptr, *d_tot = nullptr;
    int32_t *h_err = nullptr, *d_err = nullptr;
    // Per-render host state, in a ring of two so a render can be queued while the previous one is
    // still in flight (sn_render_async / sn_render_wait): mapped (chunk, pass) -> (visible splats,
    // tile pairs) words and the pose kernel's error flag, checked after the render; pinned staging
    // for the per-call host inputs (a pageable cudaMemcpyAsync would serialize with copies other
    // streams have in flight, e.g. the caller's frame downloads).
    struct Slot {
        uint64_t *h_counts = nullptr, *d_counts = nullptr;
        size_t counts_cap = 0;  // entries (chunk x pass)
        int32_t *h_err = nullptr, *d_err = nullptr;
        void *h_stage = nullptr;
        size_t h_stage_cap = 0;
        cudaEvent_t done = nullptr;
        bool pending = false;
        int64_t seq = 0;
        int n_chunks = 0;
        bool two_pass = false;
        int64_t *work = nullptr;  // the caller's work counters (accumulated when the check passes)
        uint64_t cap_v[2] = {0, 0}, cap_p[2] = {0, 0};  // the capacities the render ran with
        uint64_t cap_f[2] = {0, 0}, cap_u[2] = {0, 0}, cap_b[2] = {0, 0};
    } slot[2];
    int cur = 0;          // slot of the render being queued
    int64_t seq = 0;      // renders queued so far
    uint64_t *h_work = nullptr; // pinned (2 passes x 4 counters: loads, scans, contributions, fixups)
    // lazily resolved instrumentation: CUDA events per (pass, stage) and the blend's counters,
    // folded into the caller's arrays at the next sn_render / sn_context_sync_stats, so timing
    // adds no host synchronization inside a render
    cudaEvent_t ev[2][SN_N_STAGES][2] = {};
    cudaEvent_t ev_work[2] = {};
    // side stream for the layer pass: its preprocessing overlaps the scene blend
    cudaStream_t side = nullptr;
    // The far pipeline of a sliced pass as a small graph whose body runs only when the render
    // registered an unfinished tile (a conditional node): the dozen kernels it launches are skipped
    // on the device in the common case. Instantiated per distinct set of launch parameters (the
    // graph bakes them in): a few cached, captured on a private stream.
    struct FarGraph {
        std::vector<unsigned char> shape, key;  // kernels + device-resident control words; all parameters
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        std::vector<cudaGraphNode_t> body;  // the body's kernel nodes in launch order
    };
    FarGraph far_graph[4];
    int far_graph_next = 0;
    int64_t far_graph_builds = 0, far_graph_updates = 0;  // instantiations / in-place parameter updates
    int64_t far_body_launches = 0;  // kernels of the body (counted by render_check when it ran)
    cudaStream_t cap_stream = nullptr;
    cudaEvent_t ev_inputs = nullptr, ev_scene = nullptr, ev_layer = nullptr;
    int64_t launches = 0;  // kernels of this library launched through the context
    int64_t retries = 0;   // renders re-run because a pass outgrew its buffers
    bool slice_off_next = false;  // renders run unsliced until one goes through (a sliced one set far_short)
    int64_t slice_fallbacks = 0;  // sliced renders re-run unsliced that way
    double *ms_dst[2][SN_N_STAGES] = {};
    int64_t *work_dst[2] = {};
    bool have_events = false;
};

namespace {

void resolve_stage(sn_context *ctx, int pass, int stage) {
    double *dst = ctx->ms_dst[pass][stage];
    if (!dst) return;
    cudaEventSynchronize(ctx->ev[pass][stage][1]);
    float t = 0.0f;
    if (cudaEventElapsedTime(&t, ctx->ev[pass][stage][0], ctx->ev[pass][stage][1]) == cudaSuccess) *dst += t;
    ctx->ms_dst[pass][stage] = nullptr;
}

void resolve_all(sn_context *ctx) {
    for (int p = 0; p < 2; ++p) {
        for (int s = 0; s < SN_N_STAGES; ++s) resolve_stage(ctx, p, s);
        if (ctx->work_dst[p]) {
            cudaEventSynchronize(ctx->ev_work[p]);
            for (int k = 0; k < 4; ++k) ctx->work_dst[p][2 + k] += (int64_t)ctx->h_work[4 * p + k];
            ctx->work_dst[p] = nullptr;
        }
    }
}

// Stage timer: CUDA events around each stage on the render stream (only when requested).
struct StageTimer {
    sn_context *ctx;
    cudaStream_t st;
    double *ms;  // host (SN_N_STAGES) for this pass, or null
    int pass;
    int open = -1;
    bool nvtx_open = false;
    void begin(int stage) {
        // NVTX range per stage (host side: it brackets the stage's launches; free with no tool attached)
        static const char *const kNames[2][13] = {
            {"scene.pose", "scene.count", "scene.scan", "scene.emit", "scene.depth_sort", "scene.permute",
             "scene.pair_scan", "scene.bin_count", "scene.bin_scatter", "scene.ranges", "scene.blend",
             "scene.composite", "scene.far"},
            {"layer.pose", "layer.count", "layer.scan", "layer.emit", "layer.depth_sort", "layer.permute",
             "layer.pair_scan", "layer.bin_count", "layer.bin_scatter", "layer.ranges", "layer.blend",
             "layer.composite", "layer.far"}};
        if (nvtx_open) nvtxRangePop();
        nvtxRangePushA(kNames[pass ? 1 : 0][stage >= 0 && stage < 13 ? stage : 0]);
        nvtx_open = true;
        if (!ms) return;
        resolve_stage(ctx, pass, stage);  // the event pair is about to be reused (multi-chunk renders)
        open = stage;
        cudaEventRecord(ctx->ev[pass][stage][0], st);
    }
    void end() {
        if (nvtx_open) nvtxRangePop();
        nvtx_open = false;
        if (!ms || open < 0) return;
        cudaEventRecord(ctx->ev[pass][open][1], st);
        ctx->ms_dst[pass][open] = ms + open;
        open = -1;
    }
};

}  // namespace

namespace {

using namespace sn;

struct PassSpec {
    const sn_cloud *scene = nullptr;
    const sn_avatars *avatars = nullptr;
    PoseView pose{};
    const uint8_t *avatar_active = nullptr;
    const uint8_t *avatar_cull = nullptr;
    int mode = 0;
};

PassView view_of(const PassWs &w) {
    PassView v{};
    v.source = !w.tiled ? 2 : (w.binning == 1 ? 1 : 0);
    v.tile_bits = w.tile_bits;
    v.rects = w.rects.as<ushort4>();
    v.batch_rects = w.batch_rects.as<ushort4>();
    v.super_rects = w.super_rects.as<ushort4>();
    v.ranges = w.ranges.as<uint2>();
    v.pair_vals = w.pvals_b.as<uint32_t>();
    v.env_off = w.env_off.as<uint64_t>();
    v.recs = w.recs_un.as<SplatRec>();
    v.geo = w.geo_un.as<BlendGeo>();
    v.order = w.vals_s.as<uint32_t>();
    v.d_nvis = w.env_off.as<uint64_t>() + w.ec;
    v.d_npairs = w.counts.as<uint64_t>() + 1;
    v.cap_v = w.cap_v;
    v.cap_p = w.cap_p;
    if (v.source == 1 && w.tlist.p && w.tlist_cnt.p) {
        v.tile_list = w.tlist.as<uint32_t>();
        v.n_list = w.tlist_cnt.as<uint32_t>();
        v.list_next = w.tlist_cnt.as<uint32_t>() + 1;
    }
    v.ec = w.ec;
    v.n_tiles = w.tiles_x * w.tiles_y;
    v.sliced = w.sliced;
    if (w.sliced) {
        // control words: see kFarCtl (sn_internal.h)
        v.far_bucket_of = w.bucket_of.as<int32_t>();
        v.far_ranges = w.franges.as<uint2>();
        v.far_order = w.far_order;
        v.far_recs = w.frec.as<SplatRec>();
        v.far_geo = w.fgeo.as<BlendGeo>();
        v.far_unfin_list = w.unfin_list.as<uint32_t>();
        v.far_unfin = w.fctl.as<unsigned long long>();
        v.far_items = w.fctl.as<unsigned long long>() + 1;
        v.far_nrec = w.fctl.as<unsigned long long>() + 4;
        v.far_next = reinterpret_cast<uint32_t *>(w.fctl.as<uint64_t>() + 2);
        v.far_short = w.fctl.as<unsigned long long>() + 3;
        v.far_cap_u = w.cap_u;
        v.cap_f = w.cap_f;
        v.far_cap_b = w.cap_b;
    }
    return v;
}

int run_pass(sn_context *ctx, int pass_id, const PassSpec &sp, int e0, int ec, int width, int height, int tiled,
             uint64_t z_base, int z_bits, const sn_render_opts *opts, float *color, float *alpha, float *depth,
             float *derr, cudaStream_t st, int chunk_idx) {
    PassWs &w = ctx->pass[pass_id];
    StageTimer tm{ctx, st, opts && opts->stage_ms ? opts->stage_ms + pass_id * SN_N_STAGES : nullptr, pass_id};
    int64_t *work = opts && opts->work ? opts->work + pass_id * 6 : nullptr;
    const int64_t n = sp.scene ? sp.scene->n : sp.avatars->n;
    const int tiles_x = tiles_of(width), tiles_y = tiles_of(height);
    const int n_tiles = tiles_x * tiles_y;
    const int tile_bits = std::max(1, bit_length((uint64_t)(n_tiles - 1)));
    const int env_bits = bit_length((uint64_t)(ec - 1));
    const int key_bits = z_bits + env_bits;
    const int32_t n_blocks = (int32_t)std::max<int64_t>(1, (n + kBlock - 1) / kBlock);
    // binning 1: materialized tile lists (duplicate + stable (env | tile) radix sort + ranges);
    // 0: no lists -- each blend CTA streams its env's depth-sorted rectangles and stops at
    // saturation. Auto (opts->binning < 0 or no opts): streaming for the scene pass, whose tiles
    // saturate after ~1k rectangles; lists for the composited avatar layer, whose mostly empty
    // tiles never saturate and have few pairs.
    const int req = opts ? opts->binning : -1;
    const int binning = req == 1 ? 1 : (req == 0 ? 0 : (sp.mode == 2 ? 1 : 0));
    // depth slicing: the scene pass only (streamed rectangles, tiled, not the all-float64 mode)
    const int views = opts ? opts->views : 1;
    const int want_slice = opts ? opts->near_slice : -1;
    const bool slice = sp.scene && sp.mode != 2 && tiled && binning == 0 && !(opts && opts->exact) &&
                       !ctx->slice_off_next &&
                       (want_slice >= 1 || (want_slice < 0 && !views && n >= slice_min_gaussians()));
    const double slice_frac = want_slice >= 2 ? std::min(1.0, want_slice / 1000.0) : near_frac();
    const bool slice_all = want_slice >= 2;  // every env sliced, however few splats it sees
    const int rows = slice ? 2 * ec : ec;  // per-(env, block) counts: near rows, then far rows

    SN_ENSURE(w.vismask, sizeof(uint64_t) * std::max<int64_t>(n, 1));
    SN_ENSURE(w.blk_counts, sizeof(uint32_t) * (size_t)rows * n_blocks);
    SN_ENSURE(w.env_off, sizeof(uint64_t) * (2 * ec + 1));
    SN_CUDA(cudaMemsetAsync(w.env_off.p, 0, sizeof(uint64_t) * (2 * ec + 1), st));

    PrepArgs a{};
    a.cams = ctx->cams.as<sn_camera>();
    a.e0 = e0;
    a.ec = ec;
    a.n_blocks = n_blocks;
    a.vismask = w.vismask.as<uint64_t>();
    a.blk_counts = w.blk_counts.as<uint32_t>();
    a.stats = opts && opts->stats ? reinterpret_cast<unsigned long long *>(opts->stats) : nullptr;
    a.avatar_active = sp.avatar_active;
    a.avatar_cull = sp.avatar_cull;
    a.tiles_x = tiles_x;
    a.tiles_y = tiles_y;
    a.z_base = z_base;
    a.z_bits = z_bits;

    // No host round trip inside a pass: the visible count V = env_off[ec] and the pair count P stay
    // on the device; buffers are sized by the host capacities cap_v / cap_p (from earlier renders);
    // sn_render checks the published counts afterwards and re-runs with larger buffers on overflow.
    const uint64_t cap_v = w.cap_v, cap_p = w.cap_p;
    const size_t v1 = (size_t)cap_v + 1;
    SN_ENSURE(w.keys_un, sizeof(uint32_t) * v1);
    SN_ENSURE(w.keys_s, sizeof(uint32_t) * v1);
    SN_ENSURE(w.vals_un, sizeof(uint32_t) * v1);
    SN_ENSURE(w.vals_s, sizeof(uint32_t) * v1);
    SN_ENSURE(w.recs_un, sizeof(SplatRec) * v1);
    SN_ENSURE(w.geo_un, sizeof(BlendGeo) * v1);
    SN_ENSURE(w.gid_un, sizeof(uint32_t) * v1);
    SN_ENSURE(w.rects_un, sizeof(ushort4) * v1);
    SN_ENSURE(w.rects_tun, sizeof(ushort4) * v1);
    SN_ENSURE(w.rects, sizeof(ushort4) * v1);
    SN_ENSURE(w.tiles, sizeof(uint32_t) * v1);
    SN_ENSURE(w.pair_off, sizeof(uint64_t) * v1);
    const uint64_t n_batches = (cap_v + kBlock - 1) / kBlock;
    SN_ENSURE(w.batch_rects, sizeof(ushort4) * std::max<uint64_t>(n_batches, 1));
    SN_ENSURE(w.super_rects, sizeof(ushort4) * std::max<uint64_t>((n_batches + kSuperBatch - 1) / kSuperBatch, 1));
    SN_ENSURE(w.counts, 2 * sizeof(uint64_t));
    SN_CUDA(cudaMemsetAsync(w.counts.p, 0, 2 * sizeof(uint64_t), st));
    SN_ENSURE(w.temp, std::max({sort_temp_bytes(cap_v), scan_temp_bytes_dev(cap_v), sort_temp_bytes(cap_p)}));
    const uint64_t *d_nvis = w.env_off.as<uint64_t>() + ec;

    a.env_off = w.env_off.as<uint64_t>();
    a.keys = w.keys_un.as<uint32_t>();
    a.key_shift = key_bits > 32 ? key_bits - 32 : 0;
    a.vals = w.vals_un.as<uint32_t>();
    a.recs = w.recs_un.as<SplatRec>();
    a.geo = w.geo_un.as<BlendGeo>();
    // the harness views' extras (gaussian id, reference rectangle per splat) only when requested
    // (a spatially reordered scene always keeps the original ids: its depth ties compare them)
    const bool reordered = sp.scene && sp.scene->index;
    a.gid = (views || reordered) ? w.gid_un.as<uint32_t>() : nullptr;
    a.rects = views ? w.rects_un.as<ushort4>() : nullptr;
    a.rects_tight = w.rects_tun.as<ushort4>();
    a.cap = cap_v;
    w.sliced = slice ? 1 : 0;
    if (slice) {
        // starting capacities of the far half (~300 MB), grown by render_check on overflow: sized so
        // the occasional unfinished tiles of a fresh camera set do not cost a re-render
        if (w.cap_u == 0) w.cap_u = 16384;
        if (w.cap_f == 0) w.cap_f = 1u << 20;
        if (w.cap_b == 0) w.cap_b = 1u << 22;
        SN_ENSURE(w.zcut, sizeof(double) * ec);
        SN_ENSURE(w.nearmask, sizeof(uint64_t) * std::max<int64_t>(n, 1));
        a.z_cut = w.zcut.as<double>();
        a.nearmask = w.nearmask.as<uint64_t>();
        a.lazy_far = a.stats == nullptr ? 1 : 0;  // RenderStats need every item's frame cull
    }

    if (n > 0) {
        tm.begin(SN_STAGE_COUNT);
        ctx->launches += 1;
        if (slice) {
            ctx->launches += 1;
            SN_CUDA(launch_near_cut(*sp.scene, a, slice_frac, slice_all, w.zcut.as<double>(), st));
        }
        if (sp.scene)
            SN_CUDA(launch_scene_count(*sp.scene, a, st));
        else
            SN_CUDA(launch_avatar_count(*sp.avatars, sp.pose, a, st));
        tm.end();
        tm.begin(SN_STAGE_SCAN);
        ctx->launches += 2;
        SN_CUDA(launch_block_scan(a.blk_counts, n_blocks, rows, w.env_off.as<uint64_t>(), st));
        tm.end();
    }

    BinArgs b{};
    b.ec = ec;
    b.tiles_x = tiles_x;
    b.tiles_y = tiles_y;
    b.tile_bits = tile_bits;
    b.z_bits = z_bits;
    b.d_nvis = d_nvis;
    b.cap_v = cap_v;
    b.d_npairs = w.counts.as<uint64_t>() + 1;
    b.cap_p = cap_p;
    b.recs_un = w.recs_un.as<SplatRec>();
    b.gid_un = reordered ? w.gid_un.as<uint32_t>() : nullptr;
    b.rects_in = w.rects_tun.as<ushort4>();  // the blend's (tight) rectangles into depth order
    b.env_off = w.env_off.as<uint64_t>();
    b.rects_out = w.rects.as<ushort4>();
    b.batch_rects = w.batch_rects.as<ushort4>();
    b.tiles_touched = binning == 1 ? w.tiles.as<uint32_t>() : nullptr;  // pair counts: tile lists only
    b.pair_off = w.pair_off.as<uint64_t>();
    b.ranges = w.ranges.as<uint2>();

    const size_t n_ranges = (size_t)ec << tile_bits;
    SN_ENSURE(w.ranges, sizeof(uint2) * n_ranges);
    b.ranges = w.ranges.as<uint2>();
    SN_CUDA(cudaMemsetAsync(w.ranges.p, 0, sizeof(uint2) * n_ranges, st));
    if (binning == 1) {  // the non-empty (env, tile) list of the radix binner (listed layer blend)
        SN_ENSURE(w.tlist, sizeof(uint32_t) * n_ranges);
        SN_ENSURE(w.tlist_cnt, 4 * sizeof(uint32_t));
        SN_CUDA(cudaMemsetAsync(w.tlist_cnt.p, 0, 4 * sizeof(uint32_t), st));
        b.tile_list = w.tlist.as<uint32_t>();
        b.n_list = w.tlist_cnt.as<uint32_t>();
    }
    if (n > 0 && cap_v > 0) {
        tm.begin(SN_STAGE_EMIT);
        ctx->launches += 1;
        if (sp.scene)
            SN_CUDA(launch_scene_emit(*sp.scene, a, st));
        else
            SN_CUDA(launch_avatar_emit(*sp.avatars, sp.pose, a, st));
        tm.end();
        tm.begin(SN_STAGE_DEPTH_SORT);
        // 32-bit keys (env + top z bits), then an exact fix of equal-key runs
        const bool in_s = radix_sort_pairs(w.temp.p, w.keys_un.as<uint32_t>(), w.vals_un.as<uint32_t>(),
                                           w.keys_s.as<uint32_t>(), w.vals_s.as<uint32_t>(), d_nvis, cap_v,
                                           std::min(key_bits, 32), st, &ctx->launches, /*identity_values=*/true);
        SN_CUDA(cudaGetLastError());
        if (!in_s) {  // even pass count: the sorted arrays are back in the *_un buffers
            std::swap(w.keys_un, w.keys_s);
            std::swap(w.vals_un, w.vals_s);
        }
        b.keys_sorted = w.keys_s.as<uint32_t>();
        b.vals_sorted = w.vals_s.as<uint32_t>();
        if (key_bits > 32) {
            ctx->launches += 1;
            SN_CUDA(launch_depth_tie_fix(b, st));
        }
        tm.end();
        tm.begin(SN_STAGE_PERMUTE);
        ctx->launches += 2;
        SN_CUDA(launch_permute(b, st));
        SN_CUDA(launch_super_rects(b, w.super_rects.as<ushort4>(), st));
        tm.end();
        if (tiled && binning == 1) {
            tm.begin(SN_STAGE_PAIR_SCAN);
            SN_CUDA(scan_u32_to_u64(w.temp.p, w.tiles.as<uint32_t>(), d_nvis, cap_v, w.pair_off.as<uint64_t>(),
                                    w.counts.as<uint64_t>() + 1, st, &ctx->launches));
            tm.end();
            if (cap_p > 0) {
                SN_ENSURE(w.pkeys_a, sizeof(uint32_t) * cap_p);
                SN_ENSURE(w.pkeys_b, sizeof(uint32_t) * cap_p);
                SN_ENSURE(w.pvals_a, sizeof(uint32_t) * cap_p);
                SN_ENSURE(w.pvals_b, sizeof(uint32_t) * cap_p);
                b.pair_keys = w.pkeys_a.as<uint32_t>();
                b.pair_vals = w.pvals_a.as<uint32_t>();
                tm.begin(SN_STAGE_BIN_COUNT);
                ctx->launches += 1;
                SN_CUDA(launch_duplicate(b, st));
                tm.end();
                tm.begin(SN_STAGE_BIN_SCATTER);
                // duplicate emits pairs env-major and, within an env, in depth order, so a stable sort on
                // the tile bits alone leaves every (tile, env) group contiguous and depth-ordered; the env
                // bits never need a radix pass.
                const bool in_b = radix_sort_pairs(w.temp.p, w.pkeys_a.as<uint32_t>(), w.pvals_a.as<uint32_t>(),
                                                   w.pkeys_b.as<uint32_t>(), w.pvals_b.as<uint32_t>(),
                                                   b.d_npairs, cap_p, tile_bits, st, &ctx->launches);
                SN_CUDA(cudaGetLastError());
                if (!in_b) {
                    std::swap(w.pkeys_a, w.pkeys_b);
                    std::swap(w.pvals_a, w.pvals_b);
                }
                tm.end();
                tm.begin(SN_STAGE_RANGES);
                ctx->launches += 1;
                SN_CUDA(launch_ranges(b, w.pkeys_b.as<uint32_t>(), st));
                tm.end();
            }
        }
    }

    w.e0 = e0;
    w.ec = ec;
    w.views = views;
    w.tiles_x = tiles_x;
    w.tiles_y = tiles_y;
    w.tile_bits = tile_bits;
    w.tiled = tiled;
    w.binning = binning;
    // (a sliced pass may queue a pixel twice: the first fixup pass defers the ones needing a far bucket)
    SN_ENSURE(w.fix, sizeof(uint32_t) * (size_t)ec * width * height * (slice ? 2 : 1));
    SN_ENSURE(ctx->fixcnt, 4 * sizeof(unsigned));  // per pass: count, then [2 + pass] the second pass's start
    BlendArgs bl{};
    bl.cams = ctx->cams.as<sn_camera>();
    bl.e0 = e0;
    bl.ec = ec;
    bl.width = width;
    bl.height = height;
    bl.tiles_x = tiles_x;
    bl.mode = sp.mode;
    bl.pv = view_of(w);
    if (sp.mode == 2) {
        SN_CHECK(ctx->pass[0].valid && ctx->pass[0].e0 == e0 && ctx->pass[0].ec == ec,
                 "layer composite needs the scene pass of the same env chunk");
        bl.back = view_of(ctx->pass[0]);
    }
    bl.color = color;
    bl.alpha = alpha;
    bl.depth = depth;
    bl.derr = derr;
    bl.contrib = opts ? (pass_id == 0 ? opts->contrib_scene : opts->contrib_layer) : nullptr;
    bl.fix_list = w.fix.as<uint32_t>();
    bl.fix_count = ctx->fixcnt.as<unsigned>() + pass_id;
    bl.force_exact = opts ? opts->exact : 0;
    bl.rgb8 = opts ? opts->rgb8 : nullptr;
    bl.depth16 = opts ? opts->depth16 : nullptr;
    SN_CUDA(cudaMemsetAsync(bl.fix_count, 0, sizeof(unsigned), st));
    if (work) {
        if (ctx->work_dst[pass_id]) {  // previous chunk's counters still in flight
            cudaEventSynchronize(ctx->ev_work[pass_id]);
            for (int k = 0; k < 4; ++k) ctx->work_dst[pass_id][2 + k] += (int64_t)ctx->h_work[4 * pass_id + k];
            ctx->work_dst[pass_id] = nullptr;
        }
        SN_ENSURE(ctx->loads, 8 * sizeof(unsigned long long));
        bl.loads = ctx->loads.as<unsigned long long>() + 4 * pass_id;
        bl.scans = bl.loads + 1;
        bl.contribs = bl.loads + 2;
        SN_CUDA(cudaMemsetAsync(bl.loads, 0, 4 * sizeof(unsigned long long), st));
    }
    if (sp.mode == 2) {
        const size_t npix = (size_t)(e0 + ec) * width * height;
        SN_ENSURE(ctx->lcolor, sizeof(float) * 3 * npix);
        SN_ENSURE(ctx->lalpha, sizeof(float) * npix);
        SN_ENSURE(ctx->ldepth, sizeof(float) * npix);
        SN_ENSURE(ctx->lderr, sizeof(float) * npix);
        SN_ENSURE(ctx->laerr, sizeof(float) * npix);
        SN_ENSURE(ctx->tile_flag, (size_t)ec * n_tiles);
        // listed tiles set their flag; every other tile must read "no layer splats"
        SN_CUDA(cudaMemsetAsync(ctx->tile_flag.p, 0, (size_t)ec * n_tiles, st));
        bl.lcolor = ctx->lcolor.as<float>();
        bl.lalpha = ctx->lalpha.as<float>();
        bl.ldepth = ctx->ldepth.as<float>();
        bl.lderr = ctx->lderr.as<float>();
        bl.laerr = ctx->laerr.as<float>();
        bl.tile_flag = ctx->tile_flag.as<uint8_t>();
    }
    const int ub = std::max(1, bit_length((uint64_t)w.cap_u));  // bucket-id bits of the far item keys
    if (slice) {  // unfinished-tile registry (the blend) and the far buffers (after it)
        const size_t cu = w.cap_u, cb = w.cap_b, cf = w.cap_f;
        SN_ENSURE(w.fctl, kFarCtl * sizeof(uint64_t));
        SN_ENSURE(w.unfin_list, sizeof(uint32_t) * cu);
        SN_ENSURE(w.bucket_of, sizeof(int32_t) * (size_t)ec * n_tiles);
        SN_ENSURE(w.state, sizeof(float) * cu * kStateF * kBT);
        SN_ENSURE(w.franges, sizeof(uint2) * cu);
        SN_ENSURE(w.frec, sizeof(SplatRec) * (cf + 1));
        SN_ENSURE(w.fgeo, sizeof(BlendGeo) * (cf + 1));
        SN_ENSURE(w.fgid, sizeof(uint32_t) * (cf + 1));
        SN_ENSURE(w.bkey_a, sizeof(uint32_t) * (cb + 1));
        SN_ENSURE(w.bkey_b, sizeof(uint32_t) * (cb + 1));
        SN_ENSURE(w.bval_a, sizeof(uint32_t) * (cb + 1));
        SN_ENSURE(w.bval_b, sizeof(uint32_t) * (cb + 1));
        SN_ENSURE(w.ftemp, sort_temp_bytes(cb));
        SN_CUDA(cudaMemsetAsync(w.fctl.p, 0, kFarCtl * sizeof(uint64_t), st));
        SN_CUDA(cudaMemsetAsync(w.bucket_of.p, 0xff, sizeof(int32_t) * (size_t)ec * n_tiles, st));
        SN_CUDA(cudaMemsetAsync(w.franges.p, 0, sizeof(uint2) * cu, st));
        // the item sort is 4 radix passes of 8 bits: the order ends where it started (bkey_a, bval_a)
        w.far_order = w.bval_a.as<uint32_t>();
        bl.pv = view_of(w);
        bl.unfin_count = w.fctl.as<unsigned long long>();
        bl.unfin_envs = w.fctl.as<unsigned long long>() + 5;
        bl.unfin_list = w.unfin_list.as<uint32_t>();
        bl.bucket_of = w.bucket_of.as<int32_t>();
        bl.state = w.state.as<float>();
    }
    tm.begin(SN_STAGE_BLEND);
    // the streamed scene blend resolves its deferred pixels itself (SN_INCTA_FIXUP)
    const bool incta = SN_INCTA_FIXUP && sp.mode == 0 && bl.pv.source == 0;
    const bool fix_after = !slice && !incta && sp.mode != 2;
    ctx->launches += fix_after ? 2 : 1;  // blend (+ float64 fixup; mode 2's runs after the composite)
    SN_CUDA(launch_blend(bl, st, /*fixup=*/fix_after));
    tm.end();
    if (slice) {
        // the far buckets of the unfinished tiles, the continuation, then the fixups (sn_far.cu)
        tm.begin(SN_STAGE_FAR);
        // first fixup pass over the near lists (the buckets do not exist yet): a pixel whose float64
        // walk needs its tile's far bucket registers the tile (if the blend did not) and is queued
        // again for the second pass below
        // (the second pass starts where the blend's entries end: the deferred ones come after them)
        // (with in-CTA fixups the blend did this pass itself: the list holds only deferred pixels)
        unsigned *fix_start = nullptr;
        if (!incta) {
            fix_start = ctx->fixcnt.as<unsigned>() + 2 + pass_id;
            SN_CUDA(cudaMemcpyAsync(fix_start, bl.fix_count, sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
            BlendArgs fa = bl;
            fa.pv.far_phase = 1;
            ctx->launches += 1;
            SN_CUDA(launch_fixup(fa, st));
        }
        FarArgs f;
        std::memset(&f, 0, sizeof f);  // (the graph key compares bytes: padding too)
        f.e0 = e0;
        f.ec = ec;
        f.tiles_x = tiles_x;
        f.n_tiles = n_tiles;
        f.ub = ub;
        f.vismask = w.vismask.as<uint64_t>();
        f.nearmask = w.nearmask.as<uint64_t>();
        f.cams = ctx->cams.as<sn_camera>();
        f.bucket_of = w.bucket_of.as<int32_t>();
        f.fctl = w.fctl.as<unsigned long long>();
        f.recs = w.frec.as<SplatRec>();
        f.geo = w.fgeo.as<BlendGeo>();
        f.gid = w.fgid.as<uint32_t>();
        f.cap_f = w.cap_f;
        f.keys = w.bkey_a.as<uint32_t>();
        f.vals = w.bval_a.as<uint32_t>();
        f.cap_b = w.cap_b;
        f.ranges = w.franges.as<uint2>();
        f.z_base = z_base;
        f.z_bits = z_bits;
        BlendArgs cb2 = bl;
        cb2.pv = view_of(w);
        BlendArgs fb = cb2;  // the second fixup pass: the continuation's pixels and the deferred ones
        fb.fix_start = fix_start;
        const sn_cloud scene_c = *sp.scene;
        // the far pipeline: far_collect, the item sort, tie fix, ranges, the continuation, fixup pass 2
        int64_t body_launches = 0;
        auto far_body = [&](cudaStream_t fs) -> int {
            body_launches += 1;
            SN_CUDA(launch_far_collect(scene_c, f, n, fs));
            const bool odd = radix_sort_pairs(w.ftemp.p, w.bkey_a.as<uint32_t>(), w.bval_a.as<uint32_t>(),
                                              w.bkey_b.as<uint32_t>(), w.bval_b.as<uint32_t>(),
                                              w.fctl.as<uint64_t>() + 1, w.cap_b, 32, fs, &body_launches);
            SN_CHECK(!odd, "far item sort: 32-bit keys take an even number of passes");
            body_launches += 4;
            SN_CUDA(launch_far_tie_fix(f, w.bkey_a.as<uint32_t>(), w.bval_a.as<uint32_t>(), fs));
            SN_CUDA(launch_far_ranges(f, w.bkey_a.as<uint32_t>(), fs));
            SN_CUDA(launch_continue(cb2, fs));
            SN_CUDA(launch_fixup(fb, fs));
            return SN_OK;
        };
        if (!far_graphs_enabled()) {
            SN_CHECK(far_body(st) == SN_OK, sn_last_error());
            ctx->launches += body_launches;
        } else {
            // shape: what fixes the graph's kernels (a cached graph of the same shape takes new
            // parameters in place); key: every launch parameter the graph bakes in
            const uint64_t shape_words[5] = {(uint64_t)(uintptr_t)w.fctl.p, (uint64_t)scene_c.dtype,
                                             (uint64_t)cb2.mode, (uint64_t)(n > 0), (uint64_t)(w.cap_b > 0)};
            std::vector<unsigned char> shape(sizeof shape_words);
            std::memcpy(shape.data(), shape_words, sizeof shape_words);
            std::vector<unsigned char> key(sizeof f + 2 * sizeof(BlendArgs) + sizeof(sn_cloud) + 8 * sizeof(uint64_t));
            {
                unsigned char *k = key.data();
                std::memcpy(k, &f, sizeof f);
                k += sizeof f;
                std::memcpy(k, &cb2, sizeof cb2);
                k += sizeof cb2;
                std::memcpy(k, &fb, sizeof fb);
                k += sizeof fb;
                std::memcpy(k, &scene_c, sizeof scene_c);
                k += sizeof scene_c;
                const uint64_t extra[8] = {(uint64_t)n, (uint64_t)(uintptr_t)w.ftemp.p, (uint64_t)(uintptr_t)w.bkey_b.p,
                                           (uint64_t)(uintptr_t)w.bval_b.p, w.cap_b, 0, 0, 0};
                std::memcpy(k, extra, sizeof extra);
            }
            if (!ctx->cap_stream) SN_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
            cudaStream_t cs = ctx->cap_stream;
            // the kernel nodes of a captured linear chain, in launch order
            auto chain = [](cudaGraph_t g, std::vector<cudaGraphNode_t> &out) -> bool {
                out.clear();
                size_t nr = 1;
                cudaGraphNode_t node = nullptr;
                if (cudaGraphGetRootNodes(g, &node, &nr) != cudaSuccess || nr != 1) return false;
                while (node) {
                    cudaGraphNodeType t;
                    if (cudaGraphNodeGetType(node, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) return false;
                    out.push_back(node);
                    size_t nd = 0;
                    if (cudaGraphNodeGetDependentNodes(node, nullptr, &nd) != cudaSuccess || nd > 1) return false;
                    cudaGraphNode_t next = nullptr;
                    if (nd == 1 && cudaGraphNodeGetDependentNodes(node, &next, &nd) != cudaSuccess) return false;
                    node = nd == 1 ? next : nullptr;
                }
                return true;
            };
            sn_context::FarGraph *fg = nullptr;
            for (auto &c : ctx->far_graph)
                if (c.exec && c.key == key) fg = &c;
            if (!fg) {  // same shape: capture the body alone and move its parameters into the cached graph
                for (auto &c : ctx->far_graph)
                    if (!fg && c.exec && c.shape == shape) fg = &c;
                bool updated = false;
                if (fg) {
                    SN_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
                    body_launches = 0;
                    const int rb = far_body(cs);
                    cudaGraph_t tmp = nullptr;
                    const cudaError_t ec2 = cudaStreamEndCapture(cs, &tmp);
                    SN_CHECK(rb == SN_OK, sn_last_error());
                    SN_CUDA(ec2);
                    std::vector<cudaGraphNode_t> nodes;
                    updated = chain(tmp, nodes) && nodes.size() == fg->body.size();
                    for (size_t i = 0; updated && i < nodes.size(); ++i) {
                        cudaKernelNodeParams kp;
                        updated = cudaGraphKernelNodeGetParams(nodes[i], &kp) == cudaSuccess &&
                                  cudaGraphExecKernelNodeSetParams(fg->exec, fg->body[i], &kp) == cudaSuccess;
                    }
                    cudaGraphDestroy(tmp);
                    cudaGetLastError();  // (a refused update falls back to a new instantiation)
                    if (updated) {
                        fg->key = std::move(key);
                        ctx->far_graph_updates += 1;
                    }
                }
                if (!updated) {
                    if (!fg) {
                        fg = &ctx->far_graph[ctx->far_graph_next];
                        ctx->far_graph_next = (ctx->far_graph_next + 1) % 4;
                    }
                    if (fg->exec) cudaGraphExecDestroy(fg->exec);
                    if (fg->graph) cudaGraphDestroy(fg->graph);
                    fg->exec = nullptr;
                    fg->graph = nullptr;
                    cudaGraph_t g = nullptr;
                    SN_CUDA(cudaGraphCreate(&g, 0));
                    fg->graph = g;
                    cudaGraphConditionalHandle h;
                    SN_CUDA(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
                    SN_CUDA(cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
                    SN_CUDA(launch_far_cond(h, w.fctl.as<unsigned long long>(), cs));
                    cudaStreamCaptureStatus cst;
                    const cudaGraphNode_t *deps = nullptr;
                    size_t n_deps = 0;
                    SN_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &n_deps));
                    cudaGraphNodeParams cp = {};
                    cp.type = cudaGraphNodeTypeConditional;
                    cp.conditional.handle = h;
                    cp.conditional.type = cudaGraphCondTypeIf;
                    cp.conditional.size = 1;
                    cudaGraphNode_t cn;
                    SN_CUDA(cudaGraphAddNode(&cn, g, deps, n_deps, &cp));
                    SN_CUDA(cudaStreamUpdateCaptureDependencies(cs, &cn, 1, cudaStreamSetCaptureDependencies));
                    cudaGraph_t g_out = nullptr;
                    SN_CUDA(cudaStreamEndCapture(cs, &g_out));
                    cudaGraph_t body = cp.conditional.phGraph_out[0];
                    SN_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
                    body_launches = 0;
                    const int rb = far_body(cs);
                    cudaGraph_t b_out = nullptr;
                    const cudaError_t ec2 = cudaStreamEndCapture(cs, &b_out);
                    SN_CHECK(rb == SN_OK, sn_last_error());
                    SN_CUDA(ec2);
                    SN_CHECK(chain(body, fg->body), "far pipeline graph: the body is not a chain of kernels");
                    SN_CUDA(cudaGraphInstantiate(&fg->exec, g, 0));
                    fg->shape = std::move(shape);
                    fg->key = std::move(key);
                    ctx->far_graph_builds += 1;
                }
            }
            if (body_launches) ctx->far_body_launches = body_launches;
            SN_CUDA(cudaGraphLaunch(fg->exec, st));
            ctx->launches += 1;  // the condition kernel (the body's kernels run only when needed)
        }
        bl = cb2;
        tm.end();
    }
    w.bl = bl;
    w.work = nullptr;
    if (work && sp.mode == 2) {  // collected by finish_layer, after the fixups
        w.work = work;
    } else if (work) {
        SN_CUDA(cudaMemcpyAsync(ctx->loads.as<unsigned long long>() + 4 * pass_id + 3, bl.fix_count, sizeof(unsigned),
                                cudaMemcpyDeviceToDevice, st));
        SN_CUDA(cudaMemcpyAsync(ctx->h_work + 4 * pass_id, bl.loads, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        SN_CUDA(cudaEventRecord(ctx->ev_work[pass_id], st));
        ctx->work_dst[pass_id] = work;
    }
    // this chunk's (V, P) into mapped host memory: sn_render checks them against the capacities
    ctx->launches += 1;
    SN_CUDA(launch_publish_counts(d_nvis, w.counts.as<uint64_t>() + 1,
                                  slice ? w.fctl.as<unsigned long long>() : nullptr,
                                  ctx->slot[ctx->cur].d_counts + kCountWords * (2 * chunk_idx + pass_id), st));
    w.valid = 1;
    return SN_OK;
}

// The deferred composite of the layer pass (mode 2) over the scene frame, on the scene stream once
// both blends are done: composite_kernel, then the float64 fixups of the layer pass.
int finish_layer(sn_context *ctx, const sn_render_opts *opts, cudaStream_t st) {
    PassWs &w = ctx->pass[1];
    StageTimer tm{ctx, st, opts && opts->stage_ms ? opts->stage_ms + SN_N_STAGES : nullptr, 1};
    tm.begin(SN_STAGE_COMPOSITE);
    ctx->launches += 2;
    SN_CUDA(launch_layer_composite(w.bl, st));
    tm.end();
    if (w.work) {
        SN_CUDA(cudaMemcpyAsync(ctx->loads.as<unsigned long long>() + 4 + 3, w.bl.fix_count, sizeof(unsigned),
                                cudaMemcpyDeviceToDevice, st));
        SN_CUDA(cudaMemcpyAsync(ctx->h_work + 4, w.bl.loads, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        SN_CUDA(cudaEventRecord(ctx->ev_work[1], st));
        ctx->work_dst[1] = w.work;
        w.work = nullptr;
    }
    return SN_OK;
}

int check_cloud(const sn_cloud *c) {
    SN_CHECK(c != nullptr, "scene cloud is null");
    SN_CHECK(c->n >= 0, "negative gaussian count");
    SN_CHECK(c->n == 0 || (c->pos_opacity && c->log_scales && c->rotations && c->sh), "null scene buffer");
    SN_CHECK(c->sh_k == 1 || c->sh_k == 4 || c->sh_k == 9 || c->sh_k == 16, "sh_k must be 1, 4, 9 or 16");
    SN_CHECK(c->dtype == SN_FLOAT32 || c->dtype == SN_FLOAT64, "dtype must be SN_FLOAT32 or SN_FLOAT64");
    SN_CHECK(c->n < (int64_t)0xffffffffLL, "scene too large for 32-bit splat ids");
    return SN_OK;
}

int check_avatars(const sn_avatars *av) {
    SN_CHECK(av->n >= 0 && av->n_avatars >= 1, "avatar set needs at least one avatar");
    SN_CHECK(av->n_joints >= 1 && av->n_joints <= 255, "n_joints must be in [1, 255]");
    SN_CHECK(av->sh_k == 1 || av->sh_k == 4 || av->sh_k == 9 || av->sh_k == 16, "sh_k must be 1, 4, 9 or 16");
    SN_CHECK(av->n == 0 || (av->pos_opacity && av->log_scales && av->rotations && av->sh && av->avatar_of),
             "null avatar buffer");
    if (av->infl_offset)
        SN_CHECK(av->n == 0 || (av->infl_joint && av->infl_weight), "null CSR influence buffer");
    else
        SN_CHECK(av->n == 0 || (av->joints && av->weights), "null 4-slot influence buffer");
    SN_CHECK(av->inv_bind && av->traj_q && av->traj_t && av->traj_offset && av->n_frames && av->fps &&
                 av->start_offset && av->loop,
             "null avatar trajectory buffer");
    return SN_OK;
}

}  // namespace

extern "C" {

int sn_abi_version(void) { return SN_ABI_VERSION; }

const char *sn_last_error(void) { return g_last_error.c_str(); }

int sn_context_create(sn_context **out) {
    SN_CHECK(out != nullptr, "null output pointer");
    sn_context *ctx = new sn_context();
    cudaError_t e = cudaHostAlloc(&ctx->h_tot, sizeof(uint64_t) * 4, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&ctx->d_tot, ctx->h_tot, 0);
    if (e == cudaSuccess) e = cudaHostAlloc(&ctx->h_err, sizeof(int32_t) * 4, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&ctx->d_err, ctx->h_err, 0);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_work, sizeof(uint64_t) * 8);
    if (e != cudaSuccess) {
        delete ctx;
        return fail(SN_ERR_CUDA, std::string("cudaMallocHost: ") + cudaGetErrorString(e));
    }
    *out = ctx;
    return SN_OK;
}

int sn_context_destroy(sn_context *ctx) {
    if (!ctx) return SN_OK;
    cudaDeviceSynchronize();
    auto free_buf = [](Buf &b) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
    };
    for (auto &w : ctx->pass) {
        for (Buf *b : {&w.vismask, &w.blk_counts, &w.env_off, &w.keys_un, &w.keys_s, &w.vals_un, &w.vals_s, &w.recs_un, &w.geo_un,
                       &w.gid_un, &w.rects_un, &w.rects_tun, &w.rects, &w.tiles, &w.pair_off, &w.pkeys_a,
                       &w.pkeys_b, &w.pvals_a, &w.pvals_b, &w.ranges, &w.temp, &w.batch_rects, &w.super_rects,
                       &w.fix, &w.counts, &w.tlist, &w.tlist_cnt, &w.zcut, &w.nearmask, &w.fctl, &w.unfin_list,
                       &w.bucket_of, &w.state, &w.frec, &w.fgeo, &w.fgid, &w.franges, &w.bkey_a, &w.bkey_b,
                       &w.bval_a, &w.bval_b, &w.ftemp})
            free_buf(*b);
    }
    for (Buf *b : {&ctx->cams, &ctx->times, &ctx->derr, &ctx->jm, &ctx->eq, &ctx->root, &ctx->err, &ctx->pose_q,
                   &ctx->pose_t, &ctx->loads, &ctx->fixcnt, &ctx->av_ext, &ctx->av_cull, &ctx->rpose_q, &ctx->rpose_t, &ctx->lcolor, &ctx->lalpha, &ctx->ldepth, &ctx->lderr,
                   &ctx->laerr, &ctx->tile_flag})
        free_buf(*b);
    if (ctx->have_events) {
        for (auto &p : ctx->ev)
            for (auto &st2 : p)
                for (auto &ev : st2) cudaEventDestroy(ev);
        for (auto &ev : ctx->ev_work) cudaEventDestroy(ev);
    }
    for (auto &g : ctx->far_graph) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
    }
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->h_work) cudaFreeHost(ctx->h_work);
    for (auto &S : ctx->slot) {
        if (S.h_stage) cudaFreeHost(S.h_stage);
        if (S.h_counts) cudaFreeHost(S.h_counts);
        if (S.h_err) cudaFreeHost(S.h_err);
        if (S.done) cudaEventDestroy(S.done);
    }
    if (ctx->side) cudaStreamDestroy(ctx->side);
    for (cudaEvent_t ev : {ctx->ev_inputs, ctx->ev_scene, ctx->ev_layer})
        if (ev) cudaEventDestroy(ev);
    if (ctx->h_tot) cudaFreeHost(ctx->h_tot);
    if (ctx->h_err) cudaFreeHost(ctx->h_err);
    delete ctx;
    return SN_OK;
}

int sn_context_kernel_launches(const sn_context *ctx, int64_t *n) {
    SN_CHECK(ctx && n, "null argument");
    *n = ctx->launches;
    return SN_OK;
}

int sn_context_render_retries(const sn_context *ctx, int64_t *n) {
    SN_CHECK(ctx && n, "null argument");
    *n = ctx->retries;
    return SN_OK;
}

int sn_context_sync_stats(sn_context *ctx) {
    SN_CHECK(ctx != nullptr, "null context");
    resolve_all(ctx);
    return SN_OK;
}

int sn_context_workspace_bytes(const sn_context *ctx, size_t *bytes) {
    SN_CHECK(ctx && bytes, "null argument");
    size_t t = 0;
    for (const auto &w : ctx->pass)
        for (const Buf *b : {&w.vismask, &w.blk_counts, &w.env_off, &w.keys_un, &w.keys_s, &w.vals_un, &w.vals_s,
                             &w.recs_un, &w.geo_un, &w.gid_un, &w.rects_un, &w.rects_tun, &w.rects, &w.tiles, &w.pair_off,
                             &w.pkeys_a, &w.pkeys_b, &w.pvals_a, &w.pvals_b, &w.ranges, &w.temp,
                             &w.batch_rects, &w.super_rects, &w.fix})
            t += b->cap;
    for (const Buf *b : {&ctx->cams, &ctx->times, &ctx->derr, &ctx->jm, &ctx->eq, &ctx->root, &ctx->err,
                         &ctx->pose_q, &ctx->pose_t, &ctx->lcolor, &ctx->lalpha, &ctx->ldepth, &ctx->lderr,
                         &ctx->laerr, &ctx->tile_flag})
        t += b->cap;
    *bytes = t;
    return SN_OK;
}

static int render_once(sn_context *ctx, const sn_cloud *scene, const sn_cloud *layer, const sn_avatars *avatars,
                       const sn_camera *cams, const double *sim_times, int32_t n_envs, const sn_render_opts *opts,
                       float *color, float *alpha, float *depth, cudaStream_t st, uint64_t z_lo, int z_bits, int chunk,
                       int tiled, bool with_layer, bool with_avatars);

// Validates a render's arguments and queues it on `stream` into the current slot; no host wait.
static int render_queue(sn_context *ctx, const sn_cloud *scene, const sn_cloud *layer, const sn_avatars *avatars,
                        const sn_camera *cams, const double *sim_times, int32_t n_envs, const sn_render_opts *opts,
                        float *color, float *alpha, float *depth, void *stream) {
    SN_CHECK(ctx != nullptr, "null context");
    SN_CHECK(n_envs >= 1, "need at least one environment");
    SN_CHECK(cams != nullptr && color && alpha && depth, "null camera or output buffer");
    int r = check_cloud(scene);
    if (r != SN_OK) return r;
    SN_CHECK(layer == nullptr || avatars == nullptr, "pass either a layer cloud or an avatar set, not both");
    const bool with_layer = layer != nullptr && layer->n > 0;
    if (layer) {
        r = check_cloud(layer);
        if (r != SN_OK) return r;
    }
    const bool with_avatars = avatars != nullptr && avatars->n > 0;
    if (with_avatars) {
        r = check_avatars(avatars);
        if (r != SN_OK) return r;
        SN_CHECK(sim_times != nullptr, "avatars need per-env sim_times");
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int W = cams[0].width, H = cams[0].height;
    SN_CHECK(W >= 1 && H >= 1, "camera size must be at least 1x1");
    SN_CHECK(tiles_of(W) <= 65535 && tiles_of(H) <= 65535 && tiles_of(W) * tiles_of(H) <= (1 << 16),
             "frame too large (at most 65536 tiles)");
    uint64_t z_lo = ~0ull, z_hi = 0;
    for (int e = 0; e < n_envs; ++e) {
        const sn_camera &c = cams[e];
        SN_CHECK(c.width == W && c.height == H, "all cameras of a batch must share width/height");
        SN_CHECK(c.has_background == cams[0].has_background, "all cameras of a batch must share the background mode");
        SN_CHECK(c.fx > 0 && c.fy > 0, "focal lengths must be positive");
        SN_CHECK(c.near_ > 0 && c.near_ < c.far_, "need 0 < near < far");
        z_lo = std::min(z_lo, dbits(c.near_));
        z_hi = std::max(z_hi, dbits(c.far_));
    }
    const int z_bits = std::max(1, bit_length(z_hi - z_lo));
    const int free_bits = 64 - z_bits;
    const int chunk = free_bits >= 6 ? kMaxEnvChunk : (1 << free_bits);
    const int tiled = opts ? opts->tiled : 1;
    sn_context::Slot &S = ctx->slot[ctx->cur];
    SN_CHECK(!S.pending, "two renders are already in flight: call sn_render_wait first");
    resolve_all(ctx);
    if (opts && (opts->stage_ms || opts->work) && !ctx->have_events) {
        for (auto &p : ctx->ev)
            for (auto &st2 : p)
                for (auto &ev : st2) SN_CUDA(cudaEventCreate(&ev));
        for (auto &ev : ctx->ev_work) SN_CUDA(cudaEventCreate(&ev));
        ctx->have_events = true;
    }
    const int n_chunks = (n_envs + chunk - 1) / chunk;
    if (!S.h_err) {
        SN_CUDA(cudaHostAlloc(&S.h_err, sizeof(int32_t) * 4, cudaHostAllocMapped));
        SN_CUDA(cudaHostGetDevicePointer(&S.d_err, S.h_err, 0));
        SN_CUDA(cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming));
    }
    if ((size_t)(2 * n_chunks) > S.counts_cap) {
        SN_CUDA(cudaDeviceSynchronize());
        if (S.h_counts) cudaFreeHost(S.h_counts);
        S.h_counts = nullptr;
        S.counts_cap = 0;
        SN_CUDA(cudaHostAlloc(&S.h_counts, sizeof(uint64_t) * kCountWords * 2 * n_chunks, cudaHostAllocMapped));
        SN_CUDA(cudaHostGetDevicePointer(&S.d_counts, S.h_counts, 0));
        S.counts_cap = 2 * n_chunks;
    }
    std::memset(S.h_counts, 0, sizeof(uint64_t) * kCountWords * 2 * n_chunks);
    S.h_err[0] = 0;
    r = render_once(ctx, scene, layer, avatars, cams, sim_times, n_envs, opts, color, alpha, depth, st, z_lo, z_bits,
                    chunk, tiled, with_layer, with_avatars);
    if (r != SN_OK) return r;
    SN_CUDA(cudaEventRecord(S.done, st));
    for (int p = 0; p < 2; ++p) {
        S.cap_v[p] = ctx->pass[p].cap_v;
        S.cap_p[p] = ctx->pass[p].cap_p;
        S.cap_f[p] = ctx->pass[p].cap_f;
        S.cap_u[p] = ctx->pass[p].cap_u;
        S.cap_b[p] = ctx->pass[p].cap_b;
    }
    S.pending = true;
    S.seq = ctx->seq++;
    S.n_chunks = n_chunks;
    S.two_pass = with_layer || with_avatars;
    S.work = opts ? opts->work : nullptr;
    ctx->cur ^= 1;
    return SN_OK;
}

// Waits for the oldest queued render and checks it: the pose kernel's error flag, and every pass's
// published (visible, pairs) counts against the workspace capacities. *retry = 1: a pass outgrew
// its buffers, which have been enlarged; that render's frames are invalid and it must be queued
// again (as must any render queued after it with the old capacities).
static int render_check(sn_context *ctx, int32_t *retry) {
    *retry = 0;
    sn_context::Slot *S = nullptr;
    for (auto &c : ctx->slot)
        if (c.pending && (!S || c.seq < S->seq)) S = &c;
    SN_CHECK(S != nullptr, "no render in flight");
    S->pending = false;
    SN_CUDA(cudaEventSynchronize(S->done));
    SN_CHECK(S->h_err[0] == 0, "sample time must be nonnegative");
    bool grow = false;
    for (int p = 0; p < 2; ++p) {
        uint64_t need_v = 0, need_p = 0, sum_v = 0, sum_p = 0, last_v = 0, last_p = 0, need_f = 0, need_u = 0,
                 need_b = 0, sum_f = 0;
        for (int c = 0; c < S->n_chunks; ++c) {
            const uint64_t *h = S->h_counts + kCountWords * (2 * c + p);
            const uint64_t v = h[0], q = h[1];
            need_v = std::max(need_v, v);
            need_p = std::max(need_p, q);
            if (h[5]) {  // a float64 walk ran out of a near list with no far bucket: re-run unsliced
                if (!ctx->slice_off_next) ctx->slice_fallbacks += 1;
                ctx->slice_off_next = true;
                grow = true;
            }
            if (h[3] && far_graphs_enabled()) ctx->launches += ctx->far_body_launches;  // the body ran
            need_f = std::max(need_f, h[2]);
            need_u = std::max(need_u, h[3]);
            need_b = std::max(need_b, h[4]);
            sum_v += v;
            sum_p += q;
            sum_f += h[2];
            last_v = v;
            last_p = q;
        }
        SN_CHECK(need_v < 0xffffffffull, "too many visible splats in one env chunk (limit 2^32)");
        SN_CHECK(need_p < 0x7fffffffull, "too many tile pairs in one env chunk (limit 2^31)");
        // against the capacities this render ran with (a later check may have grown them already)
        PassWs &w = ctx->pass[p];
        if (need_v > S->cap_v[p]) {
            w.cap_v = std::max(w.cap_v, need_v + need_v / 2 + 1024);  // (+50%: fresh camera sets vary)
            grow = true;
        }
        if (need_p > S->cap_p[p]) {
            w.cap_p = std::max(w.cap_p, need_p + need_p / 2 + 1024);
            grow = true;
        }
        // depth slicing: far splats, unfinished tiles (<= one per (env, tile)), far bucket items
        if (need_f > S->cap_f[p]) {
            w.cap_f = std::max(w.cap_f, need_f + need_f / 2 + 1024);  // (+50%: fresh camera sets vary)
            grow = true;
        }
        if (need_u > S->cap_u[p]) {
            // <= one per (env, tile) of the chunk, so this bounds itself; the state is 11 KB per tile
            SN_CHECK(need_u < (1u << 24), "too many unfinished tiles in one env chunk (limit 2^24)");
            w.cap_u = (uint32_t)std::max<uint64_t>(w.cap_u, need_u + need_u / 2 + 256);
            // the bucket items were counted for the registered tiles only: scale the estimate
            if (S->cap_u[p] > 0) need_b = need_b / S->cap_u[p] * need_u + need_b % S->cap_u[p] * need_u / S->cap_u[p];
            grow = true;
        }
        if (need_b > S->cap_b[p]) {
            w.cap_b = std::max(w.cap_b, need_b + need_b / 2 + 1024);
            grow = true;
        }
        w.n_vis = (int64_t)last_v;
        w.n_pairs = (int64_t)last_p;
        if (!grow && S->work && (p == 0 || S->two_pass)) {
            S->work[6 * p] += (int64_t)(sum_v + sum_f);  // near + far visible splats
            S->work[6 * p + 1] += (int64_t)sum_p;
        }
    }
    if (!grow) ctx->slice_off_next = false;  // (a far-short fallback holds until a render goes through)
    if (grow) {
        // larger buffers: drop the partial work counters of the failed attempt
        resolve_all(ctx);
        ctx->retries += 1;
        *retry = 1;
    }
    return SN_OK;
}

int sn_render_async(sn_context *ctx, const sn_cloud *scene, const sn_cloud *layer, const sn_avatars *avatars,
                    const sn_camera *cams, const double *sim_times, int32_t n_envs, const sn_render_opts *opts,
                    float *color, float *alpha, float *depth, void *stream) {
    return render_queue(ctx, scene, layer, avatars, cams, sim_times, n_envs, opts, color, alpha, depth, stream);
}

int sn_render_wait(sn_context *ctx, int32_t *retry) {
    SN_CHECK(ctx != nullptr && retry != nullptr, "null argument");
    return render_check(ctx, retry);
}

int sn_render(sn_context *ctx, const sn_cloud *scene, const sn_cloud *layer, const sn_avatars *avatars,
              const sn_camera *cams, const double *sim_times, int32_t n_envs, const sn_render_opts *opts, float *color,
              float *alpha, float *depth, void *stream) {
    SN_CHECK(ctx != nullptr, "null context");
    SN_CHECK(!ctx->slot[0].pending && !ctx->slot[1].pending,
             "renders queued with sn_render_async are in flight: call sn_render_wait first");
    // a sliced pass can discover its capacities in stages (splats and pairs, then the unfinished
    // tiles, then their bucket items): a few re-runs at most
    for (int attempt = 0; attempt < 6; ++attempt) {
        int r = render_queue(ctx, scene, layer, avatars, cams, sim_times, n_envs, opts, color, alpha, depth, stream);
        if (r != SN_OK) return r;
        int32_t retry = 0;
        r = render_check(ctx, &retry);
        if (r != SN_OK) return r;
        if (!retry) return SN_OK;
    }
    return fail(SN_ERR_NOMEM, "workspace capacity did not converge");
}

static int render_once(sn_context *ctx, const sn_cloud *scene, const sn_cloud *layer, const sn_avatars *avatars,
                       const sn_camera *cams, const double *sim_times, int32_t n_envs, const sn_render_opts *opts,
                       float *color, float *alpha, float *depth, cudaStream_t st, uint64_t z_lo, int z_bits, int chunk,
                       int tiled, bool with_layer, bool with_avatars) {
    const int W = cams[0].width, H = cams[0].height;
    int r = SN_OK;
    SN_ENSURE(ctx->cams, sizeof(sn_camera) * n_envs);
    sn_context::Slot &S = ctx->slot[ctx->cur];
    {
        const size_t need = (sizeof(sn_camera) + sizeof(double)) * n_envs;
        if (need > S.h_stage_cap) {
            SN_CUDA(cudaStreamSynchronize(st));
            if (S.h_stage) cudaFreeHost(S.h_stage);
            S.h_stage = nullptr;
            S.h_stage_cap = 0;
            SN_CUDA(cudaMallocHost(&S.h_stage, need));
            S.h_stage_cap = need;
        }
    }
    // the slot's previous render (two renders back) has been waited for, so its uploads are done
    // and the staging buffer is free to overwrite here
    std::memcpy(S.h_stage, cams, sizeof(sn_camera) * n_envs);
    SN_CUDA(cudaMemcpyAsync(ctx->cams.p, S.h_stage, sizeof(sn_camera) * n_envs, cudaMemcpyHostToDevice, st));
    float *derr = nullptr;  // scene depth error bounds for the compositor
    if (with_avatars || with_layer) {
        SN_ENSURE(ctx->derr, sizeof(float) * (size_t)n_envs * W * H);
        derr = ctx->derr.as<float>();
    }
    if (opts && opts->stats) SN_CUDA(cudaMemsetAsync(opts->stats, 0, sizeof(sn_stats) * n_envs, st));

    // the layer pass runs on the context's side stream: only its blend waits for the scene blend
    const bool two_pass = with_layer || with_avatars;
    cudaStream_t lst = st;
    if (two_pass && !(opts && opts->serialize)) {
        if (!ctx->side) {
            // highest priority: the layer pass is short and its kernels (and host round trips) must
            // not queue behind the scene blend's CTAs, or the composite waits for it
            int lo = 0, hi = 0;
            SN_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            SN_CUDA(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, hi));
            SN_CUDA(cudaEventCreateWithFlags(&ctx->ev_inputs, cudaEventDisableTiming));
            SN_CUDA(cudaEventCreateWithFlags(&ctx->ev_scene, cudaEventDisableTiming));
            SN_CUDA(cudaEventCreateWithFlags(&ctx->ev_layer, cudaEventDisableTiming));
        }
        lst = ctx->side;
        SN_CUDA(cudaEventRecord(ctx->ev_inputs, st));
        SN_CUDA(cudaStreamWaitEvent(lst, ctx->ev_inputs, 0));
    }

    PassSpec scene_spec;
    scene_spec.scene = scene;
    scene_spec.mode = cams[0].has_background ? 0 : 1;
    PassSpec layer_spec;
    layer_spec.mode = 2;
    if (with_layer) layer_spec.scene = layer;
    // Per env chunk: the scene pass on the caller's stream and the layer pass on the side stream run
    // concurrently (the layer blend writes its own frame); then, on the caller's stream, the
    // composite merges the layer frame and the layer's float64 fixups run (they read both passes'
    // workspaces, so the next chunk's passes are queued behind them).
    for (int e0 = 0; e0 < n_envs; e0 += chunk) {
        const int ec = std::min(chunk, n_envs - e0);
        r = run_pass(ctx, 0, scene_spec, e0, ec, W, H, tiled, z_lo, z_bits, opts, color, alpha, depth, derr, st,
                     e0 / chunk);
        if (r != SN_OK) return r;
        if (!two_pass) continue;
        if (with_avatars && e0 == 0) {
            const int A = avatars->n_avatars, J = avatars->n_joints;
            SN_ENSURE(ctx->times, sizeof(double) * n_envs);
            double *h_times =
                reinterpret_cast<double *>(static_cast<char *>(S.h_stage) + sizeof(sn_camera) * n_envs);
            std::memcpy(h_times, sim_times, sizeof(double) * n_envs);
            SN_CUDA(cudaMemcpyAsync(ctx->times.p, h_times, sizeof(double) * n_envs, cudaMemcpyHostToDevice, lst));
            SN_ENSURE(ctx->jm, sizeof(double) * (size_t)n_envs * A * J * 12);
            SN_ENSURE(ctx->eq, sizeof(double) * (size_t)n_envs * A * J * 4);
            SN_ENSURE(ctx->root, sizeof(double) * (size_t)n_envs * A * 12);
            SN_ENSURE(ctx->err, sizeof(int32_t));
            SN_CUDA(cudaMemsetAsync(ctx->err.p, 0, sizeof(int32_t), lst));
            StageTimer ptm{ctx, lst, opts && opts->stage_ms ? opts->stage_ms + SN_N_STAGES : nullptr, 1};
            ptm.begin(SN_STAGE_POSE);
            ctx->launches += 1;
            SN_ENSURE(ctx->rpose_q, sizeof(double) * (size_t)n_envs * A * (J + 1) * 4);
            SN_ENSURE(ctx->rpose_t, sizeof(double) * (size_t)n_envs * A * (J + 1) * 3);
            SN_CUDA(launch_pose(*avatars, ctx->times.as<double>(), n_envs, ctx->rpose_q.as<double>(),
                                ctx->rpose_t.as<double>(), ctx->jm.as<double>(), ctx->eq.as<double>(),
                                ctx->root.as<double>(), ctx->err.as<int32_t>(), lst));
            ptm.end();
            ctx->launches += 1;
            SN_CUDA(launch_publish_i32(ctx->err.as<int32_t>(), S.d_err, lst));  // checked by sn_render_wait
            layer_spec.avatars = avatars;
            layer_spec.pose = PoseView{ctx->jm.as<double>(), ctx->eq.as<double>(), ctx->root.as<double>(), J, A};
            SN_ENSURE(ctx->av_ext, sizeof(unsigned long long) * (2 + J) * A);
            SN_ENSURE(ctx->av_cull, (size_t)n_envs * A);
            ctx->launches += 2;
            SN_CUDA(launch_avatar_cull(*avatars, layer_spec.pose, ctx->rpose_t.as<double>(), ctx->cams.as<sn_camera>(),
                                       n_envs, ctx->av_ext.as<unsigned long long>(), ctx->av_cull.as<uint8_t>(), lst));
            layer_spec.avatar_cull = ctx->av_cull.as<uint8_t>();
            layer_spec.avatar_active = opts ? opts->avatar_active : nullptr;
        }
        r = run_pass(ctx, 1, layer_spec, e0, ec, W, H, tiled, z_lo, z_bits, opts, color, alpha, depth, derr, lst,
                     e0 / chunk);
        if (r != SN_OK) return r;
        if (lst != st) {
            SN_CUDA(cudaEventRecord(ctx->ev_layer, lst));
            SN_CUDA(cudaStreamWaitEvent(st, ctx->ev_layer, 0));  // both blends done: composite on st
        }
        r = finish_layer(ctx, opts, st);
        if (r != SN_OK) return r;
        if (lst != st) {
            SN_CUDA(cudaEventRecord(ctx->ev_scene, st));
            SN_CUDA(cudaStreamWaitEvent(lst, ctx->ev_scene, 0));  // next chunk's layer pass reuses the buffers
        }
    }
    return SN_OK;
}

static int pass_env(sn_context *ctx, int32_t pass, int32_t env, PassWs *&w, int &el, std::vector<uint64_t> &off) {
    SN_CHECK(ctx != nullptr && (pass == 0 || pass == 1), "bad context or pass");
    w = &ctx->pass[pass];
    SN_CHECK(w->valid, "no render recorded for this pass");
    SN_CHECK(env >= w->e0 && env < w->e0 + w->ec, "env not in the last rendered chunk of this pass");
    SN_CHECK(!w->sliced, "the last pass was depth-sliced (no full depth order kept): render with "
                         "sn_render_opts.near_slice = 0 for the harness views");
    el = env - w->e0;
    off.resize(w->ec + 1);
    SN_CUDA(cudaDeviceSynchronize());
    SN_CUDA(cudaMemcpy(off.data(), w->env_off.p, sizeof(uint64_t) * (w->ec + 1), cudaMemcpyDeviceToHost));
    return SN_OK;
}

// Tile CSR of env `el` in the reference's form (tile_starts, depth ranks): every depth-sorted splat
// whose reference tile rectangle (renderer.py:83-86, computed on the device by the emit) covers
// the tile, in depth order -- _bin_tiles' lists. The device's own lists / streamed rectangles are
// the tighter subsets the blend consumes (tiles the support ellipse can reach), so the view is
// rebuilt here from the device's reference rectangles and depth order.
static int env_tile_csr(PassWs *w, int el, const std::vector<uint64_t> &off, std::vector<int64_t> &ts,
                        std::vector<int32_t> &ps) {
    SN_CHECK(w->views, "the last render kept no harness views (sn_render_opts.views = 0)");
    const int n_tiles = w->tiles_x * w->tiles_y;
    ts.assign(n_tiles + 1, 0);
    ps.clear();
    if (!w->tiled || w->n_vis == 0) return SN_OK;
    const uint64_t v0 = off[el], v1 = off[el + 1];
    std::vector<uint32_t> order((size_t)(v1 - v0));
    std::vector<ushort4> ref((size_t)(v1 - v0)), rects((size_t)(v1 - v0));
    if (!order.empty()) {
        SN_CUDA(cudaMemcpy(order.data(), w->vals_s.as<uint32_t>() + v0, sizeof(uint32_t) * order.size(),
                           cudaMemcpyDeviceToHost));
        SN_CUDA(cudaMemcpy(ref.data(), w->rects_un.as<ushort4>() + v0, sizeof(ushort4) * ref.size(),
                           cudaMemcpyDeviceToHost));
    }
    for (size_t i = 0; i < order.size(); ++i) {  // env-major emission: the env's slots are [v0, v1)
        SN_CHECK(order[i] >= v0 && order[i] < v1, "depth order leaves the env's slots");
        rects[i] = ref[order[i] - v0];
    }
    for (const ushort4 &q : rects)
        for (int y = q.z; y <= q.w; ++y)
            for (int x = q.x; x <= q.y; ++x) ts[y * w->tiles_x + x + 1]++;
    for (int t = 0; t < n_tiles; ++t) ts[t + 1] += ts[t];
    std::vector<int64_t> cur(ts.begin(), ts.end() - 1);
    ps.resize((size_t)ts[n_tiles]);
    for (size_t i = 0; i < rects.size(); ++i) {
        const ushort4 &q = rects[i];
        for (int y = q.z; y <= q.w; ++y)
            for (int x = q.x; x <= q.y; ++x) ps[(size_t)cur[y * w->tiles_x + x]++] = (int32_t)i;
    }
    return SN_OK;
}

int sn_get_counts(sn_context *ctx, int32_t pass, int32_t env, int64_t *n_visible, int64_t *n_pairs) {
    PassWs *w;
    int el;
    std::vector<uint64_t> off;
    int r = pass_env(ctx, pass, env, w, el, off);
    if (r != SN_OK) return r;
    int64_t v0 = (int64_t)off[el], v1 = (int64_t)off[el + 1];
    if (n_visible) *n_visible = v1 - v0;
    if (n_pairs) {
        std::vector<int64_t> ts;
        std::vector<int32_t> ps;
        r = env_tile_csr(w, el, off, ts, ps);
        if (r != SN_OK) return r;
        *n_pairs = (int64_t)ps.size();
    }
    return SN_OK;
}

int sn_get_sorted_ids(sn_context *ctx, int32_t pass, int32_t env, int32_t *ids_host, int64_t capacity) {
    PassWs *w;
    int el;
    std::vector<uint64_t> off;
    int r = pass_env(ctx, pass, env, w, el, off);
    if (r != SN_OK) return r;
    int64_t m = (int64_t)(off[el + 1] - off[el]);
    SN_CHECK(w->views, "the last render kept no harness views (sn_render_opts.views = 0)");
    SN_CHECK(capacity >= m, "ids buffer too small");
    if (m) {
        std::vector<uint32_t> order((size_t)m), gid((size_t)m);
        SN_CUDA(cudaMemcpy(order.data(), w->vals_s.as<uint32_t>() + off[el], sizeof(uint32_t) * m, cudaMemcpyDeviceToHost));
        SN_CUDA(cudaMemcpy(gid.data(), w->gid_un.as<uint32_t>() + off[el], sizeof(uint32_t) * m, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < m; ++i) ids_host[i] = (int32_t)gid[order[i] - off[el]];
    }
    return SN_OK;
}

int sn_get_tile_csr(sn_context *ctx, int32_t pass, int32_t env, int64_t *tile_starts_host, int32_t *pair_splat_host,
                    int64_t capacity) {
    PassWs *w;
    int el;
    std::vector<uint64_t> off;
    int r = pass_env(ctx, pass, env, w, el, off);
    if (r != SN_OK) return r;
    SN_CHECK(w->tiled, "last pass was not tiled");
    std::vector<int64_t> ts;
    std::vector<int32_t> ps;
    r = env_tile_csr(w, el, off, ts, ps);
    if (r != SN_OK) return r;
    SN_CHECK(capacity >= (int64_t)ps.size(), "pair buffer too small");
    std::copy(ts.begin(), ts.end(), tile_starts_host);
    std::copy(ps.begin(), ps.end(), pair_splat_host);
    return SN_OK;
}

int sn_get_device_tiles(sn_context *ctx, int32_t pass, int32_t env, int64_t *tile_starts_host, int32_t *ranks_host,
                        int64_t capacity, int64_t *n_entries) {
    PassWs *w;
    int el;
    std::vector<uint64_t> off;
    int r = pass_env(ctx, pass, env, w, el, off);
    if (r != SN_OK) return r;
    SN_CHECK(w->tiled, "last pass was not tiled");
    SN_CHECK(tile_starts_host && n_entries, "null output");
    const int n_tiles = w->tiles_x * w->tiles_y;
    const uint64_t v0 = off[el], v1 = off[el + 1];
    std::vector<int64_t> ts(n_tiles + 1, 0);
    std::vector<int32_t> ranks;
    if (w->binning == 1) {
        // the radix binner's lists: ranges per (env, tile) into pair_vals (record slots, depth order)
        std::vector<uint2> rg(n_tiles);
        SN_CUDA(cudaMemcpy(rg.data(), w->ranges.as<uint2>() + ((size_t)el << w->tile_bits), sizeof(uint2) * n_tiles,
                           cudaMemcpyDeviceToHost));
        uint64_t np = 0;
        SN_CUDA(cudaMemcpy(&np, w->counts.as<uint64_t>() + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost));
        std::vector<uint32_t> pv((size_t)np), order((size_t)(v1 - v0));
        if (np) SN_CUDA(cudaMemcpy(pv.data(), w->pvals_b.p, sizeof(uint32_t) * np, cudaMemcpyDeviceToHost));
        if (!order.empty())
            SN_CUDA(cudaMemcpy(order.data(), w->vals_s.as<uint32_t>() + v0, sizeof(uint32_t) * order.size(),
                               cudaMemcpyDeviceToHost));
        std::vector<int32_t> rank_of(order.size(), -1);  // record slot -> depth rank within the env
        for (size_t i = 0; i < order.size(); ++i) {
            SN_CHECK(order[i] >= v0 && order[i] < v1, "depth order leaves the env's slots");
            rank_of[order[i] - v0] = (int32_t)i;
        }
        for (int t = 0; t < n_tiles; ++t) {
            const uint2 q = rg[t];
            ts[t + 1] = ts[t] + (q.y > q.x ? (int64_t)(q.y - q.x) : 0);
            for (uint32_t k = q.x; k < q.y; ++k) {
                SN_CHECK(k < np && pv[k] >= v0 && pv[k] < v1, "tile list entry outside the env");
                ranks.push_back(rank_of[pv[k] - v0]);
            }
        }
    } else {
        // the streamed lists the blend builds in shared memory, exported by the same fill routine
        cudaStream_t st = 0;
        uint32_t *d_cnt = nullptr, *d_out = nullptr;
        uint64_t *d_off = nullptr;
        SN_CUDA(cudaMalloc(&d_cnt, sizeof(uint32_t) * n_tiles));
        SN_CUDA(cudaMalloc(&d_off, sizeof(uint64_t) * n_tiles));
        PassView v = view_of(*w);
        cudaError_t e = launch_tile_queue(v, el, n_tiles, w->tiles_x, d_cnt, nullptr, nullptr, st);
        std::vector<uint32_t> cnt(n_tiles);
        if (e == cudaSuccess) e = cudaMemcpy(cnt.data(), d_cnt, sizeof(uint32_t) * n_tiles, cudaMemcpyDeviceToHost);
        std::vector<uint64_t> o(n_tiles);
        for (int t = 0; t < n_tiles; ++t) {
            o[t] = (uint64_t)ts[t];
            ts[t + 1] = ts[t] + cnt[t];
        }
        ranks.resize((size_t)ts[n_tiles]);
        if (e == cudaSuccess && !ranks.empty()) {
            e = cudaMalloc(&d_out, sizeof(uint32_t) * ranks.size());
            if (e == cudaSuccess) e = cudaMemcpy(d_off, o.data(), sizeof(uint64_t) * n_tiles, cudaMemcpyHostToDevice);
            if (e == cudaSuccess) e = launch_tile_queue(v, el, n_tiles, w->tiles_x, d_cnt, d_off, d_out, st);
            if (e == cudaSuccess)
                e = cudaMemcpy(ranks.data(), d_out, sizeof(uint32_t) * ranks.size(), cudaMemcpyDeviceToHost);
        }
        cudaFree(d_cnt);
        cudaFree(d_off);
        if (d_out) cudaFree(d_out);
        SN_CUDA(e);
    }
    *n_entries = (int64_t)ranks.size();
    std::copy(ts.begin(), ts.end(), tile_starts_host);
    if (ranks_host) {
        SN_CHECK(capacity >= (int64_t)ranks.size(), "ranks buffer too small");
        std::copy(ranks.begin(), ranks.end(), ranks_host);
    }
    return SN_OK;
}

int sn_get_projection(sn_context *ctx, int32_t pass, int32_t env, double *means2d, double *conics, double *depths,
                      double *colors, double *alphas, int64_t capacity) {
    PassWs *w;
    int el;
    std::vector<uint64_t> off;
    int r = pass_env(ctx, pass, env, w, el, off);
    if (r != SN_OK) return r;
    int64_t m = (int64_t)(off[el + 1] - off[el]);
    SN_CHECK(capacity >= m, "projection buffers too small");
    std::vector<SplatRec> recs((size_t)m);
    std::vector<uint32_t> order((size_t)m);
    if (m) {
        SN_CUDA(cudaMemcpy(recs.data(), w->recs_un.as<SplatRec>() + off[el], sizeof(SplatRec) * m, cudaMemcpyDeviceToHost));
        SN_CUDA(cudaMemcpy(order.data(), w->vals_s.as<uint32_t>() + off[el], sizeof(uint32_t) * m, cudaMemcpyDeviceToHost));
    }
    for (int64_t i = 0; i < m; ++i) {
        const SplatRec &s = recs[order[i] - off[el]];
        means2d[2 * i] = s.mx;
        means2d[2 * i + 1] = s.my;
        conics[3 * i] = s.ca;
        conics[3 * i + 1] = s.cb2 * 0.5;
        conics[3 * i + 2] = s.cc;
        depths[i] = s.z;
        for (int c = 0; c < 3; ++c)
            colors[3 * i + c] = (double)((s.rgb >> (21 * c)) & 0x1FFFFFull) * (1.0 / 2097151.0);
        alphas[i] = s.alpha;
    }
    return SN_OK;
}

int sn_sample_pose(sn_context *ctx, const sn_avatars *avatars, const double *sim_times, int32_t n_envs,
                   double *pose_q, double *pose_t, void *stream) {
    SN_CHECK(ctx && avatars && sim_times && pose_q && pose_t && n_envs >= 1, "null argument");
    int r = check_avatars(avatars);
    if (r != SN_OK) return r;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SN_ENSURE(ctx->times, sizeof(double) * n_envs);
    SN_CUDA(cudaMemcpyAsync(ctx->times.p, sim_times, sizeof(double) * n_envs, cudaMemcpyHostToDevice, st));
    SN_ENSURE(ctx->err, sizeof(int32_t));
    SN_CUDA(cudaMemsetAsync(ctx->err.p, 0, sizeof(int32_t), st));
    ctx->launches += 1;
    SN_CUDA(launch_pose(*avatars, ctx->times.as<double>(), n_envs, pose_q, pose_t, nullptr, nullptr, nullptr,
                        ctx->err.as<int32_t>(), st));
    ctx->launches += 1;
    SN_CUDA(launch_publish_i32(ctx->err.as<int32_t>(), ctx->d_err, st));
    SN_CUDA(cudaStreamSynchronize(st));
    SN_CHECK(ctx->h_err[0] == 0, "sample time must be nonnegative");
    return SN_OK;
}

int sn_skin_lbs(sn_context *ctx, const sn_avatars *avatars, int32_t avatar, int64_t g_begin, int64_t g_count,
                const double *pose_q, const double *pose_t, double *out_positions, double *out_rotations,
                void *stream) {
    SN_CHECK(ctx && avatars && pose_q && pose_t, "null argument");
    int r = check_avatars(avatars);
    if (r != SN_OK) return r;
    SN_CHECK(avatar >= 0 && avatar < avatars->n_avatars, "avatar index out of range");
    SN_CHECK(g_begin >= 0 && g_count >= 0 && g_begin + g_count <= avatars->n, "gaussian range out of bounds");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int J = avatars->n_joints;
    SN_ENSURE(ctx->pose_q, sizeof(double) * (J * 12 + J * 4 + 12));
    double *jm = ctx->pose_q.as<double>(), *eq = jm + J * 12, *root = eq + J * 4;
    ctx->launches += 1;
    SN_CUDA(launch_joint_prep(*avatars, avatar, pose_q, pose_t, jm, eq, root, st));
    PoseView pv{jm, eq, root, J, 1};
    ctx->launches += 1;
    SN_CUDA(launch_skin_range(*avatars, g_begin, g_count, pv, out_positions, out_rotations, st));
    return SN_OK;
}

int sn_unpack_ply(int64_t n, int32_t n_props, const float *table, const int32_t *cols, int32_t sh_k,
                  float *pos_opacity, float *log_scales, float *rotations, float *sh, uint8_t *flags,
                  uint64_t *counters, void *stream) {
    SN_CHECK(n >= 0 && n_props >= 14 && cols != nullptr, "bad PLY table description");
    SN_CHECK(sh_k == 1 || sh_k == 4 || sh_k == 9 || sh_k == 16, "sh_k must be 1, 4, 9 or 16");
    for (int i = 0; i < 14 + 3 * (sh_k - 1); ++i) SN_CHECK(cols[i] >= 0 && cols[i] < n_props, "column out of range");
    SN_CHECK(n == 0 || (table && pos_opacity && log_scales && rotations && sh && flags && counters), "null buffer");
    SN_CUDA(launch_unpack_ply(n, n_props, table, cols, sh_k, pos_opacity, log_scales, rotations, sh, flags,
                              reinterpret_cast<unsigned long long *>(counters), static_cast<cudaStream_t>(stream)));
    return SN_OK;
}

int sn_unpack_bundle(int64_t n, int32_t sh_k, int32_t n_joints, const float *canonical, const float *weights,
                     int64_t row0, int64_t sh_stride, double *pos_opacity, double *log_scales, double *rotations,
                     float *sh, uint32_t *joints, double *weights4, double *row_sums, uint8_t *flags,
                     uint64_t *counters, void *stream) {
    SN_CHECK(n >= 0 && row0 >= 0 && sh_stride >= row0 + n, "bad bundle slice");
    SN_CHECK(sh_k == 1 || sh_k == 4 || sh_k == 9 || sh_k == 16, "sh_k must be 1, 4, 9 or 16");
    SN_CHECK(n_joints >= 1 && n_joints <= 255, "n_joints must be in [1, 255]");
    SN_CHECK(n == 0 || (canonical && weights && pos_opacity && log_scales && rotations && sh && joints && weights4 &&
                        row_sums && flags && counters),
             "null buffer");
    SN_CUDA(launch_unpack_bundle(n, sh_k, n_joints, canonical, weights, row0, sh_stride, pos_opacity, log_scales,
                                 rotations, sh, joints, weights4, row_sums, flags,
                                 reinterpret_cast<unsigned long long *>(counters), static_cast<cudaStream_t>(stream)));
    return SN_OK;
}

int sn_pack_influences(int64_t n, int32_t n_joints, const float *weights, const double *row_sums,
                       const uint64_t *counters, const uint32_t *offsets, uint8_t *infl_joint, double *infl_weight,
                       void *stream) {
    SN_CHECK(n >= 0 && n_joints >= 1 && n_joints <= 255, "bad influence table description");
    SN_CHECK(n == 0 || (weights && row_sums && counters && offsets && infl_joint && infl_weight), "null buffer");
    SN_CUDA(launch_pack_csr(n, n_joints, weights, row_sums, reinterpret_cast<const unsigned long long *>(counters),
                            offsets, infl_joint, infl_weight, static_cast<cudaStream_t>(stream)));
    return SN_OK;
}

int sn_quantize_frames(int64_t npix, const float *color, const float *depth, uint8_t *rgb8, uint16_t *depth16,
                       void *stream) {
    SN_CHECK(npix >= 0, "negative pixel count");
    SN_CHECK(npix == 0 || (color && rgb8 && (depth16 == nullptr || depth != nullptr)), "null buffer");
    SN_CUDA(launch_quantize(npix, color, depth, rgb8, depth16, static_cast<cudaStream_t>(stream)));
    return SN_OK;
}

int sn_flip_rows(int64_t frames, int32_t height, int32_t width, const float *src, float *dst, void *stream) {
    SN_CHECK(frames >= 0 && height >= 0 && width >= 0 && (frames * height * width == 0 || (src && dst && src != dst)),
             "bad frame buffers");
    SN_CUDA(launch_flip_rows(frames, height, width, src, dst, static_cast<cudaStream_t>(stream)));
    return SN_OK;
}

int sn_selftest_fast_exp(double *max_rel_err) {
    SN_CHECK(max_rel_err != nullptr, "null argument");
    SN_CUDA(fast_exp_selftest(max_rel_err));
    return SN_OK;
}

int sn_blend_tile_range(int32_t t_begin, int32_t t_end, int32_t tiles_x, int32_t tile_size, int32_t width,
                        int32_t height, const int64_t *tile_starts, int64_t n_tiles_plus1, const int32_t *pair_splat,
                        int64_t n_pairs, const double *means2d, const double *conics, const double *depths,
                        const double *colors, const double *alphas, int64_t n_splats, double *color_acc,
                        double *alpha_acc, double *trans, double *depth_acc) {
    SN_CHECK(t_begin >= 0 && t_end >= t_begin && t_end < n_tiles_plus1, "tile range out of bounds");
    SN_CHECK(tiles_x >= 1 && tile_size >= 1 && width >= 1 && height >= 1, "bad tiling");
    if (t_end == t_begin) return SN_OK;
    const size_t npix = (size_t)width * height;
    const size_t ms = (size_t)std::max<int64_t>(n_splats, 1), np = (size_t)std::max<int64_t>(n_pairs, 1);
    size_t sizes[] = {sizeof(int64_t) * n_tiles_plus1, sizeof(int32_t) * np, 16 * ms, 24 * ms, 8 * ms, 24 * ms,
                      8 * ms, 24 * npix, 8 * npix, 8 * npix, 8 * npix};
    size_t total = 0;
    for (size_t s : sizes) total += (s + 255) & ~(size_t)255;
    char *base = nullptr;
    SN_CUDA(cudaMalloc(&base, total));
    void *d[11];
    size_t o = 0;
    for (int i = 0; i < 11; ++i) {
        d[i] = base + o;
        o += (sizes[i] + 255) & ~(size_t)255;
    }
    const void *src[] = {tile_starts, pair_splat, means2d, conics, depths, colors, alphas, color_acc, alpha_acc,
                         trans, depth_acc};
    int rc = SN_OK;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 11 && e == cudaSuccess; ++i)
        if (i != 1 || n_pairs > 0) e = cudaMemcpy(d[i], src[i], i < 7 && i >= 2 ? sizes[i] / ms * n_splats : sizes[i],
                                                  cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = launch_blend_tile_range(t_begin, t_end, tiles_x, tile_size, width, height, (const int64_t *)d[0],
                                    (const int32_t *)d[1], (const double *)d[2], (const double *)d[3],
                                    (const double *)d[4], (const double *)d[5], (const double *)d[6], (double *)d[7],
                                    (double *)d[8], (double *)d[9], (double *)d[10], 0);
    if (e == cudaSuccess) e = cudaMemcpy(color_acc, d[7], sizes[7], cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(alpha_acc, d[8], sizes[8], cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(trans, d[9], sizes[9], cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(depth_acc, d[10], sizes[10], cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(SN_ERR_CUDA, std::string("sn_blend_tile_range: ") + cudaGetErrorString(e));
    cudaFree(base);
    return rc;
}

int sn_composite(int64_t npix, const double *front_color, const double *front_alpha, const double *front_depth,
                 const double *back_color, const double *back_alpha, const double *back_depth, double *out_color,
                 double *out_alpha, double *out_depth, void *stream) {
    SN_CHECK(npix >= 0, "negative pixel count");
    SN_CUDA(launch_composite64(npix, front_color, front_alpha, front_depth, back_color, back_alpha, back_depth,
                               out_color, out_alpha, out_depth, static_cast<cudaStream_t>(stream)));
    return SN_OK;
}

}  // extern "C"

// Diagnostic (not part of the ABI): the last scene pass's depth-slicing control words -- unfinished
// tiles registered, far bucket items -- read synchronously, and the sliced renders re-run unsliced.
extern "C" int sn_debug_slice_counts(sn_context *ctx, uint64_t *out) {
    SN_CHECK(ctx != nullptr && out != nullptr, "null argument");
    out[0] = out[1] = 0;
    out[2] = (uint64_t)ctx->slice_fallbacks;
    const PassWs &w = ctx->pass[0];
    if (!w.sliced || !w.fctl.p) return SN_OK;
    SN_CUDA(cudaDeviceSynchronize());
    SN_CUDA(cudaMemcpy(out, w.fctl.p, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return SN_OK;
}

// Test hook (not part of the ABI): the starting capacities of the scene pass's far half (unfinished
// tiles, far records, bucket items), so a test can force their growth path.
// test hook: far-pipeline graph instantiations and in-place updates so far (0 with SN_FAR_GRAPH=0)
extern "C" int sn_debug_far_graph_builds(sn_context *ctx, int64_t *builds, int64_t *updates) {
    SN_CHECK(ctx != nullptr && builds != nullptr && updates != nullptr, "bad argument");
    *builds = ctx->far_graph_builds;
    *updates = ctx->far_graph_updates;
    return SN_OK;
}

extern "C" int sn_debug_far_caps(sn_context *ctx, uint32_t cap_u, uint64_t cap_f, uint64_t cap_b) {
    SN_CHECK(ctx != nullptr && cap_u > 0 && cap_f > 0 && cap_b > 0, "bad argument");
    ctx->pass[0].cap_u = cap_u;
    ctx->pass[0].cap_f = cap_f;
    ctx->pass[0].cap_b = cap_b;
    return SN_OK;
}

// Diagnostic (not part of the ABI): the whole-avatar codes of the last render with an avatar set,
// (env, avatar) row-major: 0 test every gaussian, kCullDepth / kCullFrame, kWholeVisible (4).
// diagnostic: the last render's float64 fixup list of a pass (el * H * W + pixel codes, the last
// env chunk); returns the count in *n (at most cap entries copied)
extern "C" int sn_debug_fix_list(sn_context *ctx, int pass, uint32_t *out, int64_t cap, int64_t *n) {
    SN_CHECK(ctx != nullptr && out != nullptr && n != nullptr && (pass == 0 || pass == 1), "bad argument");
    SN_CHECK(ctx->fixcnt.p != nullptr && ctx->pass[pass].fix.p != nullptr, "no render yet");
    SN_CUDA(cudaDeviceSynchronize());
    unsigned c = 0;
    SN_CUDA(cudaMemcpy(&c, ctx->fixcnt.as<unsigned>() + pass, sizeof c, cudaMemcpyDeviceToHost));
    *n = c;
    SN_CUDA(cudaMemcpy(out, ctx->pass[pass].fix.p, sizeof(uint32_t) * (size_t)std::min<int64_t>(c, cap),
                       cudaMemcpyDeviceToHost));
    return SN_OK;
}

// diagnostic: the pair-list lengths of the listed (env, tile)s of a pass (the last env chunk)
extern "C" int sn_debug_tile_lens(sn_context *ctx, int pass, uint32_t *out, int64_t cap, int64_t *n) {
    SN_CHECK(ctx != nullptr && out != nullptr && n != nullptr && (pass == 0 || pass == 1), "bad argument");
    PassWs &w = ctx->pass[pass];
    SN_CHECK(w.tlist.p && w.tlist_cnt.p && w.ranges.p, "no listed pass yet");
    SN_CUDA(cudaDeviceSynchronize());
    uint32_t cnt = 0;
    SN_CUDA(cudaMemcpy(&cnt, w.tlist_cnt.p, sizeof cnt, cudaMemcpyDeviceToHost));
    const size_t n_ranges = (size_t)w.ec << w.tile_bits;
    std::vector<uint32_t> keys(cnt);
    std::vector<uint2> rg(n_ranges);
    SN_CUDA(cudaMemcpy(keys.data(), w.tlist.p, sizeof(uint32_t) * cnt, cudaMemcpyDeviceToHost));
    SN_CUDA(cudaMemcpy(rg.data(), w.ranges.p, sizeof(uint2) * n_ranges, cudaMemcpyDeviceToHost));
    *n = cnt;
    for (uint32_t i = 0; i < cnt && (int64_t)i < cap; ++i) out[i] = rg[keys[i]].y - rg[keys[i]].x;
    return SN_OK;
}

extern "C" int sn_debug_avatar_codes(sn_context *ctx, uint8_t *out, int64_t n) {
    SN_CHECK(ctx != nullptr && out != nullptr && n >= 0, "bad argument");
    SN_CHECK(ctx->av_cull.p != nullptr, "no render with an avatar set yet");
    SN_CUDA(cudaDeviceSynchronize());
    SN_CUDA(cudaMemcpy(out, ctx->av_cull.p, (size_t)n, cudaMemcpyDeviceToHost));
    return SN_OK;
}
