// sn_blend.cu -- K7/K8: per-tile front-to-back compositing with fused finalize / composite.
//
// One 256-thread CTA per (tile, env); thread = pixel. The tile's depth-ordered splat list is
// walked in batches of 256: each thread gathers one 64-byte record into shared memory, then all
// pixels evaluate the batch from shared memory (broadcast reads, no bank conflicts). A CTA-wide
// vote (__syncthreads_count) stops the walk once every pixel's transmittance fell below 1e-4.
//
// Per-pixel semantics are _kernels_cy.pyx:64-86 in float64 for the decision chain (d2 test,
// alpha, transmittance) so contributor counts equal the reference's; colour accumulates in fp32.
// The epilogue is _finalize (renderer.py:67-77) and, for the avatar layer, composite
// (renderer.py:151-166) against the scene frame already in the output buffers.
#include "sn_common.cuh"
#include "sn_internal.h"

namespace sn {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Shared-memory form of a record: a float32 copy of the geometry relative to the tile origin for
// the pre-filter, the float64 decision-chain fields, colour unpacked to float. 96 bytes.
struct __align__(16) BlendRec {
    float mxr, myr, caf, cb2f;  // mean - tile origin, conic (a, 2b) in float32
    float ccf, r, g, b;
    double mx, my, ca, cb2, cc, alpha, z, pad;
};

// 2^(j/64), j = 0..63 (round to nearest)
__constant__ double kExp2Tbl[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284, 1.0442737824274138, 1.0556451783605572,
    1.0671404006768237, 1.0787607977571199, 1.0905077326652577, 1.102382583307841, 1.1143867425958924,
    1.1265216186082418, 1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
    1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687, 1.241857812073484, 1.255380757024691,
    1.2690509571917332, 1.2828700160787783, 1.2968395546510096, 1.3109612115247644, 1.3252366431597413,
    1.339667524053303, 1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
    1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647, 1.4768261459394993,
    1.4929077282912648, 1.5091644275934228, 1.5255981507445384, 1.5422108254079407, 1.559004400237837,
    1.5759808451078865, 1.593142151342267, 1.6104903319492543, 1.6280274218573478, 1.645755478153965,
    1.6636765803267364, 1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
    1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989, 1.8340080864093424,
    1.8539791250833855, 1.8741676341103, 1.8945759815869656, 1.9152065613971474, 1.9360617934922943,
    1.9571441241754002, 1.978456026387951};

// e^(-d2/2) for the blend's argument range d2 in [~0, 9]: 2^(n/64) * e^r with a 64-entry table in
// shared memory and a degree-5 polynomial in r2 = 2r, |r| <= ln2/128 (+ the slack of a 21-bit
// scale). The -1/2 is folded into the reduction (exact power-of-two scaling). Max error 2 ulp
// (numpy's, libm's and CUDA's exp also differ by ulps). Constants whose low word is zero encode as
// instruction immediates; only ln2/32-lo and 1/48 need full 64-bit operands.
#define SN_EXP_NEG_HALF(d2, tbl, out)                                                              \
    do {                                                                                           \
        const double _t = fma((d2), -46.166229248046875, 6755399441055744.0);                     \
        const int _n = __double2loint(_t);                                                         \
        const double _nd = _t - 6755399441055744.0;                                                \
        double _r = fma(_nd, -0.021660834550857544, -(d2));                                       \
        _r = fma(_nd, -1.4841640746973977e-08, _r);                                                \
        double _p = fma(_r, 0.00026041665114462376, 0.0026041660457849503);                       \
        _p = fma(_p, _r, 0.020833333333333332);                                                    \
        _p = fma(_p, _r, 0.125);                                                                   \
        _p = fma(_p, _r, 0.5);                                                                     \
        _p = fma(_p, _r, 1.0);                                                                     \
        const double _v = (tbl)[_n & 63] * _p;                                                     \
        (out) = __hiloint2double(__double2hiint(_v) + ((_n >> 6) << 20), __double2loint(_v));    \
    } while (0)

// SOURCE 0: no tile lists. The CTA streams its env's depth-sorted tile rectangles (8 B each; the
//           env's 2 MB array stays in L2 while its 1,200 tiles run) and compacts, in depth order,
//           the splats whose rectangle covers this tile into a shared-memory queue. The walk
//           stops with the early-termination vote, so a saturated tile never looks at the rest
//           of the env -- no pair duplication, no sort, no per-pair HBM traffic.
// SOURCE 1: a materialized tile list (ranges + pair_vals from the radix binner).
// SOURCE 2: rasterize_reference -- every splat of the env, in depth order.
#ifndef SN_BLEND_MIN_BLOCKS
#define SN_BLEND_MIN_BLOCKS 1
#endif
template <int MODE, int SOURCE>
__global__ void __launch_bounds__(kBlock, SN_BLEND_MIN_BLOCKS) blend_kernel(BlendArgs b) {
    __shared__ BlendRec s_rec[kBlock];
    __shared__ double s_exp[64];
    __shared__ uint32_t s_queue[2 * kBlock];
    __shared__ uint32_t s_wsum[kBlock / 32];
    const int tile = blockIdx.x, el = blockIdx.y, env = b.e0 + el;
    const int tx = tile % b.tiles_x, ty = tile / b.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // each warp shades an 8 x 4 pixel block (compact footprint: splats that miss the block skip
    // the float64 path for the whole warp more often than with 16 x 2 rows)
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px_i = tx * kTile + lx;
    const int py_i = ty * kTile + ly;
    const bool inside = px_i < b.width && py_i < b.height;
    const double px = px_i + 0.5, py = py_i + 0.5;
    const double x0 = tx * kTile, y0 = ty * kTile;
    const float lxf = (float)lx + 0.5f, lyf = (float)ly + 0.5f;
    if (threadIdx.x < 64) s_exp[threadIdx.x] = kExp2Tbl[threadIdx.x];

    uint32_t cursor, s1;
    if (SOURCE == 1) {
        uint2 r = b.ranges[((uint32_t)el << b.tile_bits) | (uint32_t)tile];
        cursor = r.x;
        s1 = r.y;
        // composite of an empty layer tile: front alpha 0 and depth `far`, and the scene depth is a
        // weighted mean of z < far, so `front.depth < back.depth` never holds -- nothing to do
        if (MODE == 2 && cursor == s1) return;
    } else {
        cursor = (uint32_t)b.env_off[el];
        s1 = (uint32_t)b.env_off[el + 1];
    }

    double T = 1.0, A = 0.0, D = 0.0;
    float cr = 0.0f, cg = 0.0f, cb = 0.0f;
    int nc = 0;
    bool done = !inside;
    uint32_t loaded = 0, scanned = 0;
    int q_len = 0;  // SOURCE 0: entries waiting in s_queue (uniform across the CTA)
    while (true) {
        if (__syncthreads_count(!done) == 0) break;  // also guards s_rec / s_queue reuse
        int n;
        if (SOURCE == 0) {
            while (q_len < kBlock && cursor < s1) {
                // hierarchical cull (uniform across the CTA, no barrier on the skip path):
                // 8192-splat super-batches, then 256-splat batches, by their union rectangles
                const uint32_t bi = cursor / kBlock;
                const ushort4 sr = __ldg(b.super_rects + bi / kSuperBatch);
                if (!((sr.x <= tx) && (tx <= sr.y) && (sr.z <= ty) && (ty <= sr.w))) {
                    cursor = min(s1, (bi / kSuperBatch + 1) * (uint32_t)(kSuperBatch * kBlock));
                    continue;
                }
                const ushort4 br = __ldg(b.batch_rects + bi);
                const uint32_t b_end = min(s1, (bi + 1) * (uint32_t)kBlock);
                if (!((br.x <= tx) && (tx <= br.y) && (br.z <= ty) && (ty <= br.w))) {
                    cursor = b_end;
                    continue;
                }
                uint32_t i = bi * kBlock + threadIdx.x;
                bool hit = false;
                if (i >= cursor && i < b_end) {
                    ushort4 r = __ldg(b.rects + i);
                    hit = (r.x <= tx) && (tx <= r.y) && (r.z <= ty) && (ty <= r.w);
                }
                unsigned bal = __ballot_sync(kFull, hit);
                if (lane == 0) s_wsum[warp] = __popc(bal);
                __syncthreads();
                int woff = 0, tot = 0;
#pragma unroll
                for (int w = 0; w < kBlock / 32; ++w) {
                    int c = s_wsum[w];
                    woff += (w < warp) ? c : 0;
                    tot += c;
                }
                if (hit) s_queue[q_len + woff + __popc(bal & ((1u << lane) - 1u))] = i;
                q_len += tot;
                scanned += b_end - cursor;
                cursor = b_end;
                __syncthreads();
            }
            n = min(q_len, kBlock);
        } else {
            n = (int)min((uint32_t)kBlock, s1 - cursor);
        }
        if (n <= 0) break;
        loaded += n;
        if (threadIdx.x < n) {
            uint32_t rid = SOURCE == 0 ? s_queue[threadIdx.x]
                                       : (SOURCE == 1 ? __ldg(b.pair_vals + cursor + threadIdx.x) : cursor + threadIdx.x);
            const double2 *src = reinterpret_cast<const double2 *>(b.recs + __ldg(b.order + rid));
            double2 m = __ldg(src), c01 = __ldg(src + 1), c2a = __ldg(src + 2), zr = __ldg(src + 3);
            BlendRec &d = s_rec[threadIdx.x];
            d.mxr = (float)(m.x - x0);
            d.myr = (float)(m.y - y0);
            d.caf = (float)c01.x;
            d.cb2f = (float)c01.y;
            d.ccf = (float)c2a.x;
            float rgb[3];
            unpack_rgb21((unsigned long long)__double_as_longlong(zr.y), rgb);
            d.r = rgb[0];
            d.g = rgb[1];
            d.b = rgb[2];
            d.mx = m.x;
            d.my = m.y;
            d.ca = c01.x;
            d.cb2 = c01.y;
            d.cc = c2a.x;
            d.alpha = c2a.y;
            d.z = zr.x;
        }
        __syncthreads();
        if (!done) {
            for (int j = 0; j < n; ++j) {
                const BlendRec &s = s_rec[j];
                // float32 pre-filter: d2f = dx (a dx + 2b dy) + c dy^2 with FMAs. For a positive
                // definite conic |2b dx dy| <= a dx^2 + c dy^2, so every term is bounded by
                // M = 2 (a dx^2 + c dy^2); the float error is far below 2^-14 M + 1e-3, and a splat
                // clearing 9 by that margin is certainly outside the support. Survivors take the
                // exact float64 test.
                const float dxf = s.mxr - lxf, dyf = s.myr - lyf;
                const float cyf = s.ccf * dyf;
                const float d2f = __fmaf_rn(dxf, __fmaf_rn(s.caf, dxf, s.cb2f * dyf), cyf * dyf);
                const float mag = __fmaf_rn(s.caf * dxf, dxf, cyf * dyf);
                if (d2f > __fmaf_rn(mag, 1.220703125e-04f, 9.001f)) continue;
                double dx = s.mx - px, dy = s.my - py;
                double d2 = (s.ca * dx * dx + s.cb2 * dx * dy) + s.cc * dy * dy;
                if (d2 > kSupportD2) continue;
                double e;
                SN_EXP_NEG_HALF(d2, s_exp, e);
                double a = s.alpha * e;
                if (a > kAlphaClip) a = kAlphaClip;
                double w = a * T;
                float wf = (float)w;
                cr = __fmaf_rn(s.r, wf, cr);
                cg = __fmaf_rn(s.g, wf, cg);
                cb = __fmaf_rn(s.b, wf, cb);
                A = A + w;
                D = fma(s.z, w, D);  // one rounding instead of two: ulp-level, inside the depth tolerance
                T = T * (1.0 - a);
                ++nc;
                if (T < kTCutoff) break;  // T only falls on contributions (_kernels_cy.pyx:65-66)
            }
            done = T < kTCutoff;
        }
        if (SOURCE == 0) {  // drop the consumed head of the queue
            int rest = q_len - n;
            uint32_t v = threadIdx.x < rest ? s_queue[n + threadIdx.x] : 0u;
            __syncthreads();
            if (threadIdx.x < rest) s_queue[threadIdx.x] = v;
            q_len = rest;
        } else {
            cursor += n;
        }
    }
    if (b.scans && threadIdx.x == 0 && scanned) atomicAdd(b.scans, (unsigned long long)scanned);
    if (b.contribs) {
        unsigned sum = __reduce_add_sync(kFull, (unsigned)nc);
        if ((threadIdx.x & 31) == 0 && sum) atomicAdd(b.contribs, (unsigned long long)sum);
    }
    if (b.loads && threadIdx.x == 0 && loaded) atomicAdd(b.loads, (unsigned long long)loaded);
    if (!inside) return;

    const sn_camera &cam = b.cams[env];
    const int64_t pix = ((int64_t)env * b.height + py_i) * b.width + px_i;
    if (b.contrib) b.contrib[pix] = nc;
    const double alpha = A < 1.0 ? A : 1.0;
    const double depth = A > 0.0 ? D / A : cam.far_;
    float *oc = b.color + 3 * pix;
    if (MODE == 0) {
        oc[0] = (float)np_clip((double)cr + cam.background[0] * T, 0.0, 1.0);
        oc[1] = (float)np_clip((double)cg + cam.background[1] * T, 0.0, 1.0);
        oc[2] = (float)np_clip((double)cb + cam.background[2] * T, 0.0, 1.0);
        b.alpha[pix] = (float)alpha;
        b.depth[pix] = (float)depth;
        if (b.depth64) b.depth64[pix] = depth;
        return;
    }
    double fc0 = 0.0, fc1 = 0.0, fc2 = 0.0;
    if (A > 0.0) {
        fc0 = np_clip((double)cr / A, 0.0, 1.0);
        fc1 = np_clip((double)cg / A, 0.0, 1.0);
        fc2 = np_clip((double)cb / A, 0.0, 1.0);
    }
    if (MODE == 1) {
        oc[0] = (float)fc0;
        oc[1] = (float)fc1;
        oc[2] = (float)fc2;
        b.alpha[pix] = (float)alpha;
        b.depth[pix] = (float)depth;
        return;
    }
    // MODE 2: composite(front = this layer, back = scene frame in the outputs)
    const double bd = b.depth64 ? b.depth64[pix] : (double)b.depth[pix];
    if (depth < bd) {
        const double ba = b.alpha[pix];
        oc[0] = (float)(fc0 * alpha + (double)oc[0] * (1.0 - alpha));
        oc[1] = (float)(fc1 * alpha + (double)oc[1] * (1.0 - alpha));
        oc[2] = (float)(fc2 * alpha + (double)oc[2] * (1.0 - alpha));
        b.alpha[pix] = (float)(alpha + ba * (1.0 - alpha));
        if (alpha >= 0.5) b.depth[pix] = (float)depth;
    }
}

__global__ void composite64_kernel(int64_t npix, const double *fc, const double *fa, const double *fd,
                                   const double *bc, const double *ba, const double *bd, double *oc, double *oa,
                                   double *od) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix) return;
    bool use_front = fd[i] < bd[i];
    double a = fa[i];
    for (int c = 0; c < 3; ++c) {
        double blended = fc[3 * i + c] * a + bc[3 * i + c] * (1.0 - a);
        oc[3 * i + c] = use_front ? blended : bc[3 * i + c];
    }
    od[i] = (use_front && a >= 0.5) ? fd[i] : bd[i];
    oa[i] = use_front ? a + ba[i] * (1.0 - a) : ba[i];
}

// blend_tile_range with the reference's float64 buffers (_kernels_cy.pyx:21-86), exact.
__global__ void blend_tile_range_kernel(int t_begin, int tiles_x, int tile_size, int width, int height,
                                        const int64_t *tile_starts, const int32_t *pair_splat, const double *means2d,
                                        const double *conics, const double *depths, const double *colors,
                                        const double *alphas, double *color_acc, double *alpha_acc, double *trans,
                                        double *depth_acc) {
    int t = t_begin + blockIdx.x;
    int64_t s0 = tile_starts[t], s1 = tile_starts[t + 1];
    if (s0 == s1) return;
    int x0 = (t % tiles_x) * tile_size, y0 = (t / tiles_x) * tile_size;
    int tw = min(tile_size, width - x0), th = min(tile_size, height - y0);
    if (tw <= 0 || th <= 0) return;
    for (int k = threadIdx.x; k < tw * th; k += blockDim.x) {
        int py_i = y0 + k / tw, px_i = x0 + k % tw;
        double px = px_i + 0.5, py = py_i + 0.5;
        int64_t p = (int64_t)py_i * width + px_i;
        double c0 = color_acc[3 * p], c1 = color_acc[3 * p + 1], c2 = color_acc[3 * p + 2];
        double A = alpha_acc[p], D = depth_acc[p], T = 1.0;
        for (int64_t s = s0; s < s1; ++s) {
            if (T < kTCutoff) break;
            int sid = pair_splat[s];
            double dx = means2d[2 * sid] - px, dy = means2d[2 * sid + 1] - py;
            double ca = conics[3 * sid], cbv = conics[3 * sid + 1], cc = conics[3 * sid + 2];
            double d2 = ca * dx * dx + 2.0 * cbv * dx * dy + cc * dy * dy;
            if (d2 > kSupportD2) continue;
            double a = alphas[sid] * exp(-0.5 * d2);
            if (a > kAlphaClip) a = kAlphaClip;
            double w = a * T;
            c0 = c0 + colors[3 * sid] * w;
            c1 = c1 + colors[3 * sid + 1] * w;
            c2 = c2 + colors[3 * sid + 2] * w;
            A = A + w;
            D = D + depths[sid] * w;
            T = T * (1.0 - a);
        }
        color_acc[3 * p] = c0;
        color_acc[3 * p + 1] = c1;
        color_acc[3 * p + 2] = c2;
        alpha_acc[p] = A;
        depth_acc[p] = D;
        trans[p] = T;
    }
}

}  // namespace

template <int MODE>
static void launch_blend_mode(const BlendArgs &b, dim3 grid, cudaStream_t s) {
    if (b.source == 0)
        blend_kernel<MODE, 0><<<grid, kBlock, 0, s>>>(b);
    else if (b.source == 1)
        blend_kernel<MODE, 1><<<grid, kBlock, 0, s>>>(b);
    else
        blend_kernel<MODE, 2><<<grid, kBlock, 0, s>>>(b);
}

cudaError_t launch_blend(const BlendArgs &b, cudaStream_t s) {
    dim3 grid((unsigned)(tiles_of(b.width) * tiles_of(b.height)), (unsigned)b.ec);
    if (b.mode == 0)
        launch_blend_mode<0>(b, grid, s);
    else if (b.mode == 1)
        launch_blend_mode<1>(b, grid, s);
    else
        launch_blend_mode<2>(b, grid, s);
    return cudaGetLastError();
}

cudaError_t launch_composite64(int64_t npix, const double *fc, const double *fa, const double *fd, const double *bc,
                               const double *ba, const double *bd, double *oc, double *oa, double *od, cudaStream_t s) {
    if (npix == 0) return cudaSuccess;
    composite64_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(npix, fc, fa, fd, bc, ba, bd, oc, oa, od);
    return cudaGetLastError();
}

cudaError_t launch_blend_tile_range(int t_begin, int t_end, int tiles_x, int tile_size, int width, int height,
                                    const int64_t *tile_starts, const int32_t *pair_splat, const double *means2d,
                                    const double *conics, const double *depths, const double *colors,
                                    const double *alphas, double *color_acc, double *alpha_acc, double *trans,
                                    double *depth_acc, cudaStream_t s) {
    if (t_end <= t_begin) return cudaSuccess;
    blend_tile_range_kernel<<<t_end - t_begin, 256, 0, s>>>(t_begin, tiles_x, tile_size, width, height, tile_starts,
                                                            pair_splat, means2d, conics, depths, colors, alphas,
                                                            color_acc, alpha_acc, trans, depth_acc);
    return cudaGetLastError();
}

}  // namespace sn
