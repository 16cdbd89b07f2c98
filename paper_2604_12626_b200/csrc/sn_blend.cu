// sn_blend.cu -- K7/K8: per-tile front-to-back compositing with fused finalize / composite.
//
// Kernels (a tile is 16 x 16 pixels):
//   blend_kernel      -- the scene pass: one 128-thread CTA per (tile, env), two pixels per thread
//                        (rows ly, ly + 4 of the warp's 8 x 8 block) on packed float32-pair chains.
//                        Sources: 0 the env's depth-sorted rectangles streamed with batch culling,
//                        1 materialized tile lists, 2 every splat (rasterize_reference), 3 the
//                        continuation of a depth-sliced pass's unfinished tiles over their far
//                        buckets (sn_far.cu).
//   blend_kernel_lp2  -- the avatar layer's listed blend: 128-thread CTAs taking the non-empty
//                        (env, tile) pairs dynamically, each warp walking two 8 x 4 blocks.
//   blend_kernel_px1  -- the layer's other sources: 256 threads, one pixel per thread.
//   fixup_kernel / fixup_layer_kernel / composite_kernel -- float64 walks, the deferred composite.
// Per batch the CTA gathers the next depth-ordered records into shared memory (their float32
// principal-axis form and a per-warp block mask), each warp walks the entries whose support can
// reach its block, and a CTA-wide vote (__syncthreads_count) stops once every pixel is saturated.
//
// Numerics (the reference is float64, _kernels_cy.pyx:64-86): the per-contribution chain runs in
// float32 with a rigorous running error bound, and every discrete decision is either certain or
// resolved in float64:
//   * d2 <= 9: each gathered splat is re-expressed, in float64, in its conic's principal axes
//     relative to the tile centre: d2 = l1 u1^2 + l2 u2^2, u1 = e1.o + U1, u2 = e2.o + U2
//     (o = pixel - tile centre, |o| <= 7.5). Every float term is then small -- no cancellation
//     even for camera-hugging splats whose mean is thousands of pixels away -- and a per-(splat,
//     tile) bound E9 on |d2_f - d2| over {d2 <= 9.1} is computed at gather time. Pixels with
//     |d2_f - 9| <= E9 recompute d2 exactly in float64 (rare).
//   * alpha = min(.99, o e^(-d2/2)): relative error eps = E9 / 2 + kEpsExp (ex2.approx, argument
//     and product roundings; the ex2 bound is verified by sn_selftest_fast_exp).
//   * T < 1e-4: T' = fma(-a, T, T) (one rounding) and its absolute error is tracked per pixel,
//     err' = err (1 - a) + w eps + 1.25 u T'.
//     When T is within err of 1e-4 the pixel is "ambiguous": it is appended to a fixup list and
//     recomputed by fixup_kernel, a warp-per-pixel float64 walk with the reference's operation
//     order (the previous, fully float64 blend), which also writes its outputs.
//   * composite (mode 2): depth_front < depth_back and alpha >= 0.5 are decided only when the
//     tracked bounds separate them; otherwise the pixel goes to the fixup, which recomputes the
//     scene pixel and the layer pixel in float64 and composites exactly.
// So the discrete outputs (contributor counts, composite choices) are the float64 chain's, and
// the continuous ones carry float32 error (~1e-6, against the 2e-3 RGB / 1e-4 depth bars).
#include "sn_common.cuh"
#include "sn_internal.h"

#include <cuda_fp16.h>

#include <cstring>
#include <type_traits>

#ifdef SN_BLEND_PROF
__device__ unsigned long long g_blend_prof[16];
__device__ unsigned g_env_frac[64];  // per env: largest fraction (1/1000) of the depth list a tile consumed
#endif
#ifdef SN_FIX_PROF
__device__ unsigned long long g_fix_prof[16];  // why the scene blend deferred pixels (scripts/blend_prof.py)
#endif

namespace sn {

__device__ int g_slice_hooks = 0;  // test hooks, see sn_debug_slice_hooks

namespace {

constexpr unsigned kFull = 0xffffffffu;

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

// ---- float32 chain error constants (see the header comment) ----
// ex2.approx incl. its argument's rounding (measured max 2.76e-7 over d2 in [0, 9.5] by
// sn_selftest_fast_exp; the GPU test asserts <= 3.5e-7) + the roundings of alpha and alpha * e
constexpr float kEpsExp = 5.0e-7f;
constexpr float kEpsExact = 8.0e-7f;   // same, when d2 came from float64 (rounded to float: 4.5 u)
constexpr float kU125 = 7.5e-8f;       // 1.25 u: the one rounding of T' = fma(-a, T, T) (+ the err sums')
constexpr float kTLo = 9.99999e-05f;   // 1e-4 (1 - 1e-6): below it (with the bound) T < 1e-4 for sure
constexpr float kTHi = 1.000001e-04f;  // 1e-4 (1 + 1e-6)
constexpr float kNegHalfLog2e = -0.72134752044448170f;
#ifndef SN_WALK_UNROLL
#define SN_WALK_UNROLL 8
#endif
constexpr int kWalkUnroll = SN_WALK_UNROLL;  // walk loop unroll (entries per iteration)
// the blend works on h = d2 log2(e) / 2 (so e^(-d2/2) = 2^-h): its axes carry sqrt(log2(e) / 2)
constexpr double kHalfLog2e = 0.72134752044448170;
constexpr double kSqrtHalfLog2e = 0.84932180028801904272;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Packed float32 pairs (sm_100 FFMA2: two IEEE fmas per issue slot, each rounded exactly like
// __fmaf_rn; a scalar operand is broadcast to both halves without a move).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void unpack2(f32x2 v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// The blend CTA: 128 threads per 16 x 16 tile, each thread two pixels -- rows ly and ly + 4 of its
// warp's 8 x 8 block (warp w: block (w & 1, w >> 1)) -- whose per-contribution chains run as packed
// float32 pairs (FFMA2 / FMUL2 / FADD2: two IEEE operations per issue slot, each rounded exactly
// like its scalar form), so the per-splat loads, the loop and the block mask are shared by two
// pixels and the chain costs about half the issue slots per pixel.
constexpr int kBW = kBT / 32;  // warps (8 x 8 pixel blocks) per tile (kBT: sn_internal.h)
#ifndef SN_EXACT_BLOCK
// tile_entry's warp-block test: separating axes (0), or the exact disc-vs-parallelogram distance (1),
// which removes more empty walk iterations but was measured slower (scene blend 6.04 vs 5.83 ms at
// config 2: its per-record cost exceeds the walk it saves)
#define SN_EXACT_BLOCK 0
#endif

// Shared-memory form of a gathered splat for the float32 chain (80 B): the principal-axis rows (a
// pixel's v_k = row_k . o + V_k, h = v1^2 + v2^2), V1 and V2 twice (register pairs for FFMA2), the
// decision thresholds k (9 -/+ E(9.1)), alpha's error bound coefficients NEGATED (-eps = nka h +
// nkb, nkb twice: the walk carries negated weights, see blend_kernel), -alpha, z and colour.
// k = log2(e) / 2: the chain works on h = k d2, so alpha = o 2^-h.
struct __align__(16) FRec {
    float a1x, a1y, c2x, c2y;
    float V1, V1b, V2, V2b;
    float thr_out, thr_in, nkb, nkbb;
    float nka, alpha, z, pad0;
    float r, g, b, pad1;
};
static_assert(sizeof(FRec) == 80, "FRec layout");

// Which of the tile's four 8 x 8 warp blocks the splat's support {d2 <= 9} can reach: (mx, my) is
// the mean relative to the tile origin, (hx, hy) the support ellipse's bounding-box half-extents
// (already widened far beyond the float rounding of the reference's d2 test), so a pixel whose
// d2 <= 9 is never outside a set bit.
__device__ __forceinline__ unsigned warp_block_mask(float mx, float my, float hx, float hy) {
    const float x0 = mx - hx, x1 = mx + hx, y0 = my - hy, y1 = my + hy;
    unsigned cols = 0, rows = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // pixel centres 8 k + 0.5 .. 8 k + 7.5 in x and in y
        cols |= (x1 >= 8 * k + 0.5f && x0 <= 8 * k + 7.5f) ? (1u << k) : 0u;
        rows |= (y1 >= 8 * k + 0.5f && y0 <= 8 * k + 7.5f) ? (1u << k) : 0u;
    }
    unsigned m = 0;
#pragma unroll
    for (int w = 0; w < kBW; ++w) m |= (((cols >> (w & 1)) & (rows >> (w >> 1))) & 1u) << w;
    return m;
}

// A gathered splat's float32 blend form for this tile, from its BlendGeo (make_blend_geo): d2 in the
// conic's principal axes relative to the tile centre (cx, cy), d2(o) = l1 (e1.o + U1)^2 +
// l2 (e2.o + U2)^2 with U_k = e_k.(centre - mean) formed in float64, the thresholds 9 -/+ E(9.1) and
// the alpha error coefficients, from the float error of d2 at a pixel with |o| <= 7.5 sqrt(2):
//   |u_k error| <= u S_k, S_k = 2 |U_k| + 21.3 + 3.02 / sqrt(l_k)   (valid while d2 <= 9.1),
//   E(d2) = 1.5 [2 u sqrt(d2) (sqrt(l1) S1 + sqrt(l2) S2) + 7 u d2] + 1e-15 (l1 / l2) 9,
//   eps(d2) = E(d2) / 2 + kEpsExp <= ka d2 + kb   (sqrt(d2) <= (d2 + 1) / 2),
// all evaluated in float with a 1% margin. A degenerate conic (l2 <= 0) gets thresholds that send
// every pixel to the float64 test. Returns the 4-bit warp-block mask (warp_block_mask).
__device__ __forceinline__ unsigned tile_entry(double e1x, double e1y, double p1, double p2, float4 gl, float4 gr,
                                               double cx, double cy, FRec &f) {
    const double U1 = fma(e1x, cx, fma(e1y, cy, -p1));
    const double U2 = fma(-e1y, cx, fma(e1x, cy, -p2));
    const float l1 = gl.x, l2 = gl.y;
    const float fU1 = (float)U1, fU2 = (float)U2, fe1x = (float)e1x, fe1y = (float)e1y;
    const float u = 5.9604644775390625e-08f;  // 2^-24
    const float aU1 = fabsf(fU1), aU2 = fabsf(fU2);
    bool ok = l2 > 0.0f;
    float r1v = 0.0f, r2v = 0.0f, sig = 0.0f, kap = 0.0f, e9 = 0.0f;
    if (ok) {
        const float r1 = rsqrtf(l1), r2 = rsqrtf(l2);
        r1v = r1;
        r2v = r2;
        const float s1 = 2.0f * aU1 + 21.3f + 3.02f * r1, s2 = 2.0f * aU2 + 21.3f + 3.02f * r2;
        sig = (l1 * r1) * s1 + (l2 * r2) * s2;
        kap = 9.0e-15f * fminf(l1 / l2, 1e30f);
        e9 = 1.01f * (1.5f * (2.0f * u * 3.0166f * sig + 7.0f * u * 9.1f) + kap);
        ok = e9 < 0.5f;
    }
    // mean - tile origin, from the principal-axis offsets (float error ~ 2u (|U1| + |U2|))
    const float mx = 8.0f - (fU1 * fe1x - fU2 * fe1y), my = 8.0f - (fU1 * fe1y + fU2 * fe1x);
    const float slack = 1e-3f + 4.0f * u * (aU1 + aU2);
    unsigned m = warp_block_mask(mx, my, gr.z * 1.00001f + slack, gr.w * 1.00001f + slack);
    if (ok && m) {
        // Separating axes along the ellipse's own axes (the support's oriented bounding box,
        // |u_k| <= 3 / sqrt(l_k), against each 8 x 8 block of pixel centres projected on e_k):
        // rotated, elongated splats whose axis-aligned box reaches a block often miss it.
        const float ax = fabsf(fe1x), ay = fabsf(fe1y);
        const float marg = 1e-3f + 8.0f * u * (aU1 + aU2 + 16.0f);
        const float ext1 = 3.0f * rsqrtf(l1) * 1.00001f + marg + 3.5f * (ax + ay);
        const float ext2 = 3.0f * rsqrtf(l2) * 1.00001f + marg + 3.5f * (ay + ax);
        // Two more axes, the diagonals of the support's normalized frame: with v_k = sqrt(l_k) u_k
        // the support is the disc |v| <= 3 and a block is a parallelogram, which misses the disc if
        // its projection on d = (1, +-1)/sqrt(2) stays beyond 3 -- the blocks near the corners of
        // the oriented box, which pass the two tests above without holding a single pixel inside.
        const float s1 = l1 * r1v, s2 = l2 * r2v;  // sqrt(l1), sqrt(l2)
        const float hx1 = s1 * 3.5f * fe1x, hx2 = -s2 * 3.5f * fe1y;  // block half-edges in v space
        const float hy1 = s1 * 3.5f * fe1y, hy2 = s2 * 3.5f * fe1x;
        const float hwp = (fabsf(hx1 + hx2) + fabsf(hy1 + hy2)) * 0.70710678f;
        const float hwm = (fabsf(hx1 - hx2) + fabsf(hy1 - hy2)) * 0.70710678f;
        const float lim = 3.0f * 1.00001f + (s1 + s2) * marg;
        // u_k at the block centres (8 bx - 4, 8 by - 4) relative to the tile centre
        const float u1b = fU1 - 4.0f * fe1x - 4.0f * fe1y, u2b = fU2 + 4.0f * fe1y - 4.0f * fe1x;
#if SN_EXACT_BLOCK
        // Exact: the distance from the disc's centre to the block's parallelogram {C + s A + t B,
        // |s|, |t| <= 1} in v space, against 3 (with the same slack). The parallelogram's minimum is
        // its interior point when the unconstrained minimiser lies inside, else on one of its four
        // edges (a clamped 1-D minimum each); the float errors (~1e-6 of |C|^2) stay far inside the
        // slack's 2e-5 |C| R. Subsumes the four separating axes below.
        const float AA = hx1 * hx1 + hx2 * hx2, BB = hy1 * hy1 + hy2 * hy2, AB = hx1 * hy1 + hx2 * hy2;
        const float rdet = 1.0f / (AA * BB - AB * AB), rAA = 1.0f / AA, rBB = 1.0f / BB;
        (void)ext1;
        (void)ext2;
#pragma unroll
        for (int w = 0; w < kBW; ++w) {
            const float bx = (float)(w & 1), by = (float)(w >> 1);
            const float u1c = u1b + 8.0f * bx * fe1x + 8.0f * by * fe1y;
            const float u2c = u2b - 8.0f * bx * fe1y + 8.0f * by * fe1x;
            const float v1c = s1 * u1c, v2c = s2 * u2c;
            const float rad = lim + 1e-5f * (fabsf(v1c) + fabsf(v2c) + hwp + hwm);
            const float AC = hx1 * v1c + hx2 * v2c, BC = hy1 * v1c + hy2 * v2c;
            const float ss = (AB * BC - BB * AC) * rdet, tt = (AB * AC - AA * BC) * rdet;
            if (fabsf(ss) <= 1.0f && fabsf(tt) <= 1.0f) continue;  // the centre projects inside
            float d2m = 3.0e38f;
#pragma unroll
            for (int sg = -1; sg <= 1; sg += 2) {
                {  // edge s = sg
                    const float cx = v1c + sg * hx1, cy = v2c + sg * hx2;
                    const float t = fminf(1.0f, fmaxf(-1.0f, -(hy1 * cx + hy2 * cy) * rBB));
                    const float ex = cx + t * hy1, ey = cy + t * hy2;
                    d2m = fminf(d2m, ex * ex + ey * ey);
                }
                {  // edge t = sg
                    const float cx = v1c + sg * hy1, cy = v2c + sg * hy2;
                    const float t = fminf(1.0f, fmaxf(-1.0f, -(hx1 * cx + hx2 * cy) * rAA));
                    const float ex = cx + t * hx1, ey = cy + t * hx2;
                    d2m = fminf(d2m, ex * ex + ey * ey);
                }
            }
            if (d2m > rad * rad) m &= ~(1u << w);
        }
#else
#pragma unroll
        for (int w = 0; w < kBW; ++w) {
            const float bx = (float)(w & 1), by = (float)(w >> 1);
            const float u1c = u1b + 8.0f * bx * fe1x + 8.0f * by * fe1y;
            const float u2c = u2b - 8.0f * bx * fe1y + 8.0f * by * fe1x;
            const float v1c = s1 * u1c, v2c = s2 * u2c;
            const float slack = lim + 1e-5f * (fabsf(v1c) + fabsf(v2c) + hwp + hwm);
            if (fabsf(u1c) > ext1 || fabsf(u2c) > ext2 || fabsf(v1c + v2c) * 0.70710678f - hwp > slack ||
                fabsf(v1c - v2c) * 0.70710678f - hwm > slack)
                m &= ~(1u << w);
        }
#endif
    }
    if (!m) return 0u;  // reaches none of the tile's warp blocks: the record is never read
    // the axes pre-scaled by sqrt(l_k log2(e) / 2) (float64 products, rounded once):
    // h = v1^2 + v2^2 = d2 log2(e) / 2, the exp argument itself; every float error of d2 scales by
    // the same factor, so the d2 bounds carry over with thresholds and ka scaled
    const double sl1 = sqrt((double)l1) * kSqrtHalfLog2e, sl2 = sqrt((double)fmaxf(l2, 0.0f)) * kSqrtHalfLog2e;
    f.a1x = (float)(sl1 * e1x);
    f.a1y = (float)(sl1 * e1y);
    f.V1 = f.V1b = (float)(sl1 * U1);
    f.c2x = (float)(-sl2 * e1y);
    f.c2y = (float)(sl2 * e1x);
    f.V2 = f.V2b = (float)(sl2 * U2);
    f.alpha = -gl.z;  // negated: the walk multiplies by -alpha (see blend_kernel)
    f.z = gl.w;
    float rgb[3];
    unpack_rgb21(((unsigned long long)__float_as_uint(gr.y) << 32) | __float_as_uint(gr.x), rgb);
    f.r = rgb[0];
    f.g = rgb[1];
    f.b = rgb[2];
    f.pad0 = f.pad1 = 0.0f;
    if (ok) {
        // k (9 -/+ e9) in h units, widened by 1e-6 for the float k and the products' roundings
        const float kf = (float)kHalfLog2e;
        f.thr_in = __fmaf_rn(-kf, e9, kf * 9.0f) - 1.0e-6f;
        f.thr_out = __fmaf_rn(kf, e9, kf * 9.0f) + 1.0e-6f;
        f.nka = -1.4003f * (0.75f * u * sig + 5.25f * u);  // 1.01 / k: eps = ka d2 + kb = ka' h + kb
        f.nkb = f.nkbb = -1.01f * (0.75f * u * sig + kEpsExp + 0.5f * kap);
    } else {  // every pixel that is not certainly outside takes the float64 test
        f.thr_in = -1.0f;
        f.thr_out = 1.0e29f;  // below the finished-pixel offset 1e30, above any real h (< 1e15)
        f.nka = 0.0f;
        f.nkb = f.nkbb = -kEpsExact;
    }
    return m;
}

// ---- the one-pixel-per-thread blend (256 threads per tile, 8 x 4 warp blocks), kept for the
// avatar layer: its tile lists hold small splats that reach few pixels of a tile, where the finer
// 8 x 4 warp blocks walk fewer entries than the two-pixel kernel's 8 x 8 blocks (measured: 2.39 vs
// 2.55 ms per 64-env layer pass). Same numerics as blend_kernel, scalar chain.
// Shared-memory form of a gathered splat for the float32 chain (64 B): the principal-axis rows as
// (axis 1, axis 2) pairs, the decision thresholds k (9 -/+ E(9.1)), alpha, the alpha error bound
// coefficients, colour and z (paired for the FFMA2 accumulation). k = log2(e) / 2: the chain
// works on h = k d2, so alpha = o 2^-h.
struct __align__(16) FRec1 {
    float a1x, c2x, a1y, c2y;  // (v1, v2) = (a1x, c2x) ox + (a1y, c2y) oy + (V1, V2), h = v1^2 + v2^2,
    float V1, V2, thr_out, thr_in;  // v_j = sqrt(k l_j) u_j
    float ka, kb, alpha, pad;  // alpha's relative error bound: eps = ka h + kb
    float r, g, b, z;
};

// Which of the CTA's eight 8 x 4 warp blocks the splat's support {d2 <= 9} can reach: (mx, my) is
// the mean relative to the tile origin, (hx, hy) the support ellipse's bounding-box half-extents
// (already widened far beyond the float rounding of the reference's d2 test), so a pixel whose
// d2 <= 9 is never outside a set bit.
__device__ __forceinline__ unsigned warp_block_mask_8x4(float mx, float my, float hx, float hy) {
    const float x0 = mx - hx, x1 = mx + hx, y0 = my - hy, y1 = my + hy;
    unsigned cols = 0, rows = 0;
#pragma unroll
    for (int bx = 0; bx < 2; ++bx)  // pixel centres 8 bx + 0.5 .. 8 bx + 7.5
        cols |= (x1 >= 8 * bx + 0.5f && x0 <= 8 * bx + 7.5f) ? (1u << bx) : 0u;
#pragma unroll
    for (int by = 0; by < 4; ++by)  // pixel centres 4 by + 0.5 .. 4 by + 3.5
        rows |= (y1 >= 4 * by + 0.5f && y0 <= 4 * by + 3.5f) ? (1u << by) : 0u;
    unsigned m = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m |= (((cols >> (w & 1)) & (rows >> (w >> 1))) & 1u) << w;
    return m;
}

// A gathered splat's float32 blend form for this tile, from its BlendGeo (make_blend_geo): d2 in the
// conic's principal axes relative to the tile centre (cx, cy), d2(o) = l1 (e1.o + U1)^2 +
// l2 (e2.o + U2)^2 with U_k = e_k.(centre - mean) formed in float64, the thresholds 9 -/+ E(9.1) and
// the alpha error coefficients, from the float error of d2 at a pixel with |o| <= 7.5 sqrt(2):
//   |u_k error| <= u S_k, S_k = 2 |U_k| + 21.3 + 3.02 / sqrt(l_k)   (valid while d2 <= 9.1),
//   E(d2) = 1.5 [2 u sqrt(d2) (sqrt(l1) S1 + sqrt(l2) S2) + 7 u d2] + 1e-15 (l1 / l2) 9,
//   eps(d2) = E(d2) / 2 + kEpsExp <= ka d2 + kb   (sqrt(d2) <= (d2 + 1) / 2),
// all evaluated in float with a 1% margin. A degenerate conic (l2 <= 0) gets thresholds that send
// every pixel to the float64 test. Returns the 8-bit warp-block mask (warp_block_mask).
__device__ __forceinline__ unsigned tile_entry_8x4(double e1x, double e1y, double p1, double p2, float4 gl, float4 gr,
                                               double cx, double cy, FRec1 &f) {
    const double U1 = fma(e1x, cx, fma(e1y, cy, -p1));
    const double U2 = fma(-e1y, cx, fma(e1x, cy, -p2));
    const float l1 = gl.x, l2 = gl.y;
    const float fU1 = (float)U1, fU2 = (float)U2, fe1x = (float)e1x, fe1y = (float)e1y;
    const float u = 5.9604644775390625e-08f;  // 2^-24
    const float aU1 = fabsf(fU1), aU2 = fabsf(fU2);
    bool ok = l2 > 0.0f;
    float r1v = 0.0f, r2v = 0.0f, sig = 0.0f, kap = 0.0f, e9 = 0.0f;
    if (ok) {
        const float r1 = rsqrtf(l1), r2 = rsqrtf(l2);
        r1v = r1;
        r2v = r2;
        const float s1 = 2.0f * aU1 + 21.3f + 3.02f * r1, s2 = 2.0f * aU2 + 21.3f + 3.02f * r2;
        sig = (l1 * r1) * s1 + (l2 * r2) * s2;
        kap = 9.0e-15f * fminf(l1 / l2, 1e30f);
        e9 = 1.01f * (1.5f * (2.0f * u * 3.0166f * sig + 7.0f * u * 9.1f) + kap);
        ok = e9 < 0.5f;
    }
    // mean - tile origin, from the principal-axis offsets (float error ~ 2u (|U1| + |U2|))
    const float mx = 8.0f - (fU1 * fe1x - fU2 * fe1y), my = 8.0f - (fU1 * fe1y + fU2 * fe1x);
    const float slack = 1e-3f + 4.0f * u * (aU1 + aU2);
    unsigned m = warp_block_mask_8x4(mx, my, gr.z * 1.00001f + slack, gr.w * 1.00001f + slack);
    if (ok && m) {
        // Separating axes along the ellipse's own axes (the support's oriented bounding box,
        // |u_k| <= 3 / sqrt(l_k), against each 8 x 4 block of pixel centres projected on e_k):
        // rotated, elongated splats whose axis-aligned box reaches a block often miss it.
        const float ax = fabsf(fe1x), ay = fabsf(fe1y);
        const float marg = 1e-3f + 8.0f * u * (aU1 + aU2 + 16.0f);
        const float ext1 = 3.0f * rsqrtf(l1) * 1.00001f + marg + (3.5f * ax + 1.5f * ay);
        const float ext2 = 3.0f * rsqrtf(l2) * 1.00001f + marg + (3.5f * ay + 1.5f * ax);
        // Two more axes, the diagonals of the support's normalized frame: with v_k = sqrt(l_k) u_k
        // the support is the disc |v| <= 3 and a block is a parallelogram, which misses the disc if
        // its projection on d = (1, +-1)/sqrt(2) stays beyond 3 -- the blocks near the corners of
        // the oriented box, which pass the two tests above without holding a single pixel inside.
        const float s1 = l1 * r1v, s2 = l2 * r2v;  // sqrt(l1), sqrt(l2)
        const float hx1 = s1 * 3.5f * fe1x, hx2 = -s2 * 3.5f * fe1y;  // block half-edges in v space
        const float hy1 = s1 * 1.5f * fe1y, hy2 = s2 * 1.5f * fe1x;
        const float hwp = (fabsf(hx1 + hx2) + fabsf(hy1 + hy2)) * 0.70710678f;
        const float hwm = (fabsf(hx1 - hx2) + fabsf(hy1 - hy2)) * 0.70710678f;
        const float lim = 3.0f * 1.00001f + (s1 + s2) * marg;
        // u_k at the block centres (8 bx - 4, 4 by - 6) relative to the tile centre
        const float u1b = fU1 - 4.0f * fe1x - 6.0f * fe1y, u2b = fU2 + 4.0f * fe1y - 6.0f * fe1x;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const float bx = (float)(w & 1), by = (float)(w >> 1);
            const float u1c = u1b + 8.0f * bx * fe1x + 4.0f * by * fe1y;
            const float u2c = u2b - 8.0f * bx * fe1y + 4.0f * by * fe1x;
            const float v1c = s1 * u1c, v2c = s2 * u2c;
            const float slack = lim + 1e-5f * (fabsf(v1c) + fabsf(v2c) + hwp + hwm);
            if (fabsf(u1c) > ext1 || fabsf(u2c) > ext2 || fabsf(v1c + v2c) * 0.70710678f - hwp > slack ||
                fabsf(v1c - v2c) * 0.70710678f - hwm > slack)
                m &= ~(1u << w);
        }
    }
    if (!m) return 0u;  // reaches none of the CTA's warp blocks: the record is never read
    // the axes pre-scaled by sqrt(l_k log2(e) / 2) (float64 products, rounded once):
    // h = v1^2 + v2^2 = d2 log2(e) / 2, the exp argument itself; every float error of d2 scales by
    // the same factor, so the d2 bounds carry over with thresholds and ka scaled
    const double sl1 = sqrt((double)l1) * kSqrtHalfLog2e, sl2 = sqrt((double)fmaxf(l2, 0.0f)) * kSqrtHalfLog2e;
    f.a1x = (float)(sl1 * e1x);
    f.a1y = (float)(sl1 * e1y);
    f.V1 = (float)(sl1 * U1);
    f.c2x = (float)(-sl2 * e1y);
    f.c2y = (float)(sl2 * e1x);
    f.V2 = (float)(sl2 * U2);
    f.alpha = gl.z;
    f.z = gl.w;
    float rgb[3];
    unpack_rgb21(((unsigned long long)__float_as_uint(gr.y) << 32) | __float_as_uint(gr.x), rgb);
    f.r = rgb[0];
    f.g = rgb[1];
    f.b = rgb[2];
    f.pad = 0.0f;
    if (ok) {
        // k (9 -/+ e9) in h units, widened by 1e-6 for the float k and the products' roundings
        const float kf = (float)kHalfLog2e;
        f.thr_in = __fmaf_rn(-kf, e9, kf * 9.0f) - 1.0e-6f;
        f.thr_out = __fmaf_rn(kf, e9, kf * 9.0f) + 1.0e-6f;
        f.ka = 1.4003f * (0.75f * u * sig + 5.25f * u);  // 1.01 / k: eps = ka d2 + kb = ka' h + kb
        f.kb = 1.01f * (0.75f * u * sig + kEpsExp + 0.5f * kap);
    } else {  // every pixel that is not certainly outside takes the float64 test
        f.thr_in = -1.0f;
        f.thr_out = 3.0e38f;
        f.ka = 0.0f;
        f.kb = kEpsExact;
    }
    return m;
}


// The observation payload of a finished pixel (sn_render_opts.rgb8 / depth16), from the float32
// values the frame holds: frame_io.save_color_png's uint8 rule (frame_io.py:13-14: clip, x * 255
// + 0.5 in float64, truncation) and fp16 depth -- the same bytes sn_quantize_frames writes, fused
// into each epilogue that finalizes a pixel so only the quantized frame leaves for the gather.
__device__ __forceinline__ uint8_t quant8(float x) {
    double v = (double)x;
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    return (uint8_t)(v * 255.0 + 0.5);
}
__device__ __forceinline__ void store_payload(const BlendArgs &b, int64_t pix, float r, float g, float bl,
                                              float depth) {
    if (b.rgb8) {
        uint8_t *o = b.rgb8 + 3 * pix;
        o[0] = quant8(r);
        o[1] = quant8(g);
        o[2] = quant8(bl);
    }
    if (b.depth16) b.depth16[pix] = __half_as_ushort(__float2half_rn(depth));
}

__device__ __forceinline__ bool covers(ushort4 r, int tx, int ty) {
    return (r.x <= tx) && (tx <= r.y) && (r.z <= ty) && (ty <= r.w);
}

// Warp-aggregated append of this lane's pixel to the fixup list (all 32 lanes must call).
__device__ __forceinline__ void push_fixup(const BlendArgs &b, bool flag, uint32_t code) {
    const unsigned bal = __ballot_sync(kFull, flag);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == __ffs(bal) - 1) base = atomicAdd(b.fix_count, (unsigned)__popc(bal));
    base = __shfl_sync(kFull, base, __ffs(bal) - 1);
    SN_ASSERT(!flag || base + __popc(bal) <= (unsigned)(b.ec * b.width * b.height));
    if (flag) b.fix_list[base + __popc(bal & ((1u << lane) - 1u))] = code;
}

// The streamed tile list of SOURCE 0 (below): appends to s_queue, in depth order, the depth ranks
// i in [cursor, s1) whose (tight) tile rectangle covers tile (tx, ty), one 256-rectangle batch per
// step (NT threads, 256 / NT rectangles each, in order), until at least `cap` entries wait (the
// queue holds cap + 255) or the env's list ends. Whole 8192-splat super-batches and 256-splat
// batches whose union rectangles miss the tile are skipped without a barrier (the branch is
// uniform across the CTA). Used by the blend and by the harness export of the lists the blend
// consumes (tile_queue_kernel).
template <int NT>
__device__ __forceinline__ void stream_fill(const PassView &v, int tx, int ty, int cap, uint32_t &cursor, uint32_t s1,
                                            int &q_len, uint32_t &scanned, uint32_t *s_queue, uint32_t *s_wsum) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    while (q_len < cap && cursor < s1) {
        const uint32_t bi = cursor / kBlock;
        if (!covers(__ldg(v.super_rects + bi / kSuperBatch), tx, ty)) {
            cursor = min(s1, (bi / kSuperBatch + 1) * (uint32_t)(kSuperBatch * kBlock));
            continue;
        }
        const uint32_t b_end = min(s1, (bi + 1) * (uint32_t)kBlock);
        if (!covers(__ldg(v.batch_rects + bi), tx, ty)) {
            cursor = b_end;
            continue;
        }
#pragma unroll
        for (int r = 0; r < kBlock / NT; ++r) {
            const uint32_t i = bi * kBlock + r * NT + threadIdx.x;
            const bool hit = i >= cursor && i < b_end && covers(__ldg(v.rects + i), tx, ty);
            const unsigned bal = __ballot_sync(kFull, hit);
            if (lane == 0) s_wsum[warp] = __popc(bal);
            __syncthreads();
            int woff = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) {
                const int c = s_wsum[w];
                woff += (w < warp) ? c : 0;
                tot += c;
            }
            SN_ASSERT(q_len + tot < cap + kBlock);  // callers size the queue cap + kBlock
            if (hit) s_queue[q_len + woff + __popc(bal & ((1u << lane) - 1u))] = i;
            q_len += tot;
            __syncthreads();
        }
        scanned += b_end - cursor;
        cursor = b_end;
    }
}

// Harness export (sn_get_device_tiles) of the streamed lists for env `el` of the last pass: one CTA
// per tile runs stream_fill over the whole env (no early termination) and writes, in order, the
// depth ranks (relative to the env) it queued: counts first (out == null), then the entries at
// the caller's offsets.
__global__ void __launch_bounds__(kBlock) tile_queue_kernel(PassView v, int el, int tiles_x, uint32_t *counts,
                                                            const uint64_t *offsets, uint32_t *out) {
    __shared__ uint32_t s_queue[2 * kBlock];
    __shared__ uint32_t s_wsum[kBlock / 32];
    if (pass_overflow(v)) return;
    const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
    const uint32_t e0 = (uint32_t)v.env_off[el];
    uint32_t cursor = e0, s1 = (uint32_t)v.env_off[el + 1], scanned = 0;
    uint64_t total = 0;
    while (true) {
        int q_len = 0;
        stream_fill<kBlock>(v, tx, ty, kBlock, cursor, s1, q_len, scanned, s_queue, s_wsum);
        if (q_len == 0) break;
        if (out)
            for (int i = threadIdx.x; i < q_len; i += kBlock) out[offsets[tile] + total + i] = s_queue[i] - e0;
        total += q_len;
        __syncthreads();
    }
    if (!out && threadIdx.x == 0) counts[tile] = (uint32_t)total;
}

// SOURCE 0: no tile lists. The CTA streams its env's depth-sorted tile rectangles (8 B each; the
//           env's 2 MB array stays in L2 while its 1,200 tiles run) and compacts, in depth order,
//           the splats whose rectangle covers this tile into a shared-memory queue. The walk
//           stops with the early-termination vote, so a saturated tile never looks at the rest
//           of the env -- no pair duplication, no sort, no per-pair HBM traffic.
// SOURCE 1: a materialized tile list (ranges + pair_vals from the radix binner; the values are
//           record slots, in depth order).
// SOURCE 2: rasterize_reference -- every splat of the env, in depth order.
#ifndef SN_BLEND_MIN_BLOCKS
#define SN_BLEND_MIN_BLOCKS 6
#endif
#ifndef SN_LAYER_MIN_BLOCKS
#define SN_LAYER_MIN_BLOCKS 6
#endif
// 1.0f when a <= b, else 0.0f (one FSET)
__device__ __forceinline__ float le_mask(float a, float b) {
    float r;
    asm("set.le.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
// packed float32 pair helpers (sm_100 FMUL2 / FADD2, each half rounded like the scalar op)
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float lo_of(f32x2 v) {
    float a, c;
    unpack2(v, a, c);
    return a;
}
__device__ __forceinline__ float hi_of(f32x2 v) {
    float a, c;
    unpack2(v, a, c);
    return c;
}

// One pixel's float32 chain state, packed with the thread's other pixel (lo = row ly, hi = ly + 4).
struct PixPair {
    f32x2 T, err, A, cr, cg, cb, D, dead, eps_max, z_last, nc;  // nc: contributions (exact floats)
};

// ---- exact (float64) per-pixel walk: the fixup path (defined below) ----

struct ExactPixel {
    float cr, cg, cb;
    double A, D, T;
    int nc;
    bool near;  // the cutoff test met a transmittance within 1e-12 (relative) of 1e-4: re-walk with SEQ
    bool out;   // (far_phase 1) the walk needs the tile's far bucket, not built yet: defer the pixel
};

// The relative window around 1e-4 inside which the warp prefix product's association (<= ~1e-13
// relative from the sequential product after hundreds of contributions) could flip `T < 1e-4`.
constexpr double kNearCut = 1e-12;


// A contribution waiting in a warp's queue (float64 alpha and z, colour).
struct QEntry {
    double a, z;
    float r, g, b, pad;
};
constexpr int kQueue = 64;  // per-warp queue capacity: < 32 waiting + 32 arriving

#ifndef SN_FIXUP_PER
#define SN_FIXUP_PER 2
#endif
template <int kPer>
__device__ __forceinline__ ExactPixel exact_pixel(const PassView &v, int el, int tile, int tiles_x, int px_i, int py_i,
                                                  const double *s_exp, QEntry *q);
__device__ __forceinline__ void write_exact_scene(const BlendArgs &b, const ExactPixel &f, int64_t pix,
                                                  const sn_camera &cam);
__device__ __forceinline__ void defer_to_far(const BlendArgs &b, int el, int tile, uint32_t code);

template <int MODE, int SOURCE>
__global__ void __launch_bounds__(kBT, MODE == 2 ? SN_LAYER_MIN_BLOCKS : SN_BLEND_MIN_BLOCKS) blend_kernel(BlendArgs b) {
    constexpr bool kBound = MODE != 1;  // depth error bounds feed the compositor
    // the layer tracks each pixel's largest alpha bound (it decides the compositor's depth choice);
    // the scene pass uses the CTA's largest bound over every gathered splat -- looser, one
    // instruction less per contribution
    static_assert(MODE != 2, "the avatar layer (mode 2) runs blend_kernel_px1");
    constexpr bool kPixBound = false;      // (mode 2's per-pixel alpha bound lives in blend_kernel_px1)
    constexpr int kPerT = 2;               // records gathered per thread per batch
    constexpr int kBatch = kBT * kPerT;    // 256 records per batch
    __shared__ unsigned s_epsmax;
    __shared__ FRec s_f[kBatch + 1];     // + a record no pixel is inside of (list padding)
    __shared__ uint32_t s_slot[kBatch];  // record slot (the boundary band reads its SplatRec)
    __shared__ uint32_t s_queue[SOURCE == 0 ? kBatch + kBlock : 1];
    __shared__ int s_u;  // sliced pass: this tile's unfinished index (-1: none / overflow)
    __shared__ uint32_t s_wsum[kBW];
    __shared__ uint8_t s_mask[kBatch];  // bit w: the splat's support may reach warp w's 8 x 8 block
    // per warp: byte offsets of its batch entries, in depth order, padded to a multiple of the
    // walk's unroll with the inert record
    __shared__ uint16_t s_wl[kBW][kBatch + kWalkUnroll];
    // the scene pass resolves its deferred pixels itself, after the tile's walk (a warp per pixel,
    // the float64 walk of fixup_kernel): their latency-bound list walks overlap the other CTAs' blends
    constexpr bool kInCta = MODE == 0 && SOURCE == 0 && SN_INCTA_FIXUP;
    __shared__ uint32_t s_fixpix[kInCta ? 2 * kBT : 1];
    __shared__ unsigned s_nfix;
    static_assert(sizeof(s_f) >= 64 * sizeof(double) + kBW * kQueue * sizeof(QEntry), "fixup scratch in s_f");
    const PassView &v = b.pv;
    if (pass_overflow(v)) return;
    if (SOURCE == 3 && far_overflow(v)) return;
    // one (env, tile); u: its unfinished index (the continuation, SOURCE 3), else -1
    auto do_tile = [&](const int tile, const int el, const int u) {
        if (threadIdx.x == 0) {
            s_epsmax = __float_as_uint(kEpsExact);
            s_nfix = 0u;
        }
        if (threadIdx.x < 20) {  // the inert record: h = dead >= 0 > thr_in = thr_out = -1, alpha 0
            float *d = reinterpret_cast<float *>(&s_f[kBatch]);
            d[threadIdx.x] = (threadIdx.x == 8 || threadIdx.x == 9) ? -1.0f : 0.0f;
        }
        const int env = b.e0 + el;
        const int tx = tile % b.tiles_x, ty = tile / b.tiles_x;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 8 + (lane >> 3);  // rows ly, ly + 4
        const int px_i = tx * kTile + lx;
        const int py0 = ty * kTile + ly, py1 = py0 + 4;
        const bool in0 = px_i < b.width && py0 < b.height, in1 = px_i < b.width && py1 < b.height;
        const double px = px_i + 0.5;
        const double x0 = tx * kTile, y0 = ty * kTile;
        const float oxf = (float)lx - 7.5f;  // pixel centre - tile centre
        const f32x2 OX = pack2(oxf, oxf), OY = pack2((float)ly - 7.5f, (float)ly - 3.5f);
    #ifdef SN_BLEND_PROF
        unsigned long long prof[16] = {};
    #define PROF(i, x) (prof[i] += (x))
    #else
    #define PROF(i, x) ((void)0)
    #endif

        uint32_t cursor, s1;
        if (SOURCE == 1) {
            uint2 r = v.ranges[((uint32_t)el << v.tile_bits) | (uint32_t)tile];
            cursor = r.x;
            s1 = r.y;
            // composite of an empty layer tile: front alpha 0 and depth `far`, and the scene depth is a
            // weighted mean of z < far, so `front.depth < back.depth` never holds -- nothing to do
            if (MODE == 2) {
                if (threadIdx.x == 0) b.tile_flag[(int64_t)el * (tiles_of(b.width) * tiles_of(b.height)) + tile] = cursor != s1;
                if (cursor == s1) return;
            }
        } else if (SOURCE == 3) {  // continuation of an unfinished tile: its far bucket, in depth order
            const uint2 r = v.far_ranges[u];
            cursor = r.x;
            s1 = r.y;
        } else {
            cursor = (uint32_t)v.env_off[el];
            s1 = (uint32_t)v.env_off[el + 1];
        }

        // added to h: a finished pixel skips every splat. A pixel is finished when it is outside the
        // frame, forced exact, or past the cutoff test (after which T and err never change, so the
        // cutoff's ambiguity is re-derived from them after the walk). 1e30 (not inf) keeps every
        // product of the chain finite (a finished pixel's alpha is 0 and its eps ~1e24).
        constexpr float kDead = 1.0e30f;
        PixPair P;
        P.T = pack2(1.0f, 1.0f);
        P.err = P.A = P.cr = P.cg = P.cb = P.D = P.eps_max = P.z_last = P.nc = 0ull;
        P.dead = pack2((!in0 || b.force_exact) ? kDead : 0.0f, (!in1 || b.force_exact) ? kDead : 0.0f);
        float z_first = 3.0e38f;
        bool entry_live0 = true, entry_live1 = true;  // SOURCE 3: pixels still live when the tile resumed
        if (SOURCE == 3) {  // the state the near walk saved (save_state below)
            SN_ASSERT(u >= 0 && (uint32_t)u < v.far_cap_u);
            const float *st = b.state + (size_t)u * kStateF * kBT + threadIdx.x;
            f32x2 *f[10] = {&P.T, &P.err, &P.A, &P.cr, &P.cg, &P.cb, &P.D, &P.dead, &P.z_last, &P.nc};
    #pragma unroll
            for (int q = 0; q < 10; ++q) *f[q] = pack2(st[(2 * q) * kBT], st[(2 * q + 1) * kBT]);
            z_first = st[20 * kBT];
            if (threadIdx.x == 0) s_epsmax = __float_as_uint(st[21 * kBT]);
            entry_live0 = lo_of(P.dead) == 0.0f;
            entry_live1 = hi_of(P.dead) == 0.0f;
        }
        uint32_t loaded = 0, scanned = 0;
        int q_len = 0;  // SOURCE 0: entries waiting in s_queue (uniform across the CTA)
        while (true) {
            const bool live = lo_of(P.dead) == 0.0f || hi_of(P.dead) == 0.0f;
            if (__syncthreads_count(live) == 0) break;  // also guards s_f / s_queue reuse
            int n;
            if (SOURCE == 0) {
                stream_fill<kBT>(v, tx, ty, kBatch, cursor, s1, q_len, scanned, s_queue, s_wsum);
                n = min(q_len, kBatch);
            } else {
                n = (int)min((uint32_t)kBatch, s1 - cursor);
            }
            if (n <= 0) break;
            loaded += n;
    #pragma unroll
            for (int r = 0; r < kPerT; ++r) {
                const int jt = threadIdx.x + r * kBT;
                if (jt >= n) break;
                // the record slot: tile lists hold slots; streamed / all-splat sources map depth ranks
                const uint32_t rid = SOURCE == 1   ? __ldg(v.pair_vals + cursor + jt)
                                     : SOURCE == 3 ? __ldg(v.far_order + cursor + jt)
                                                   : __ldg(v.order + (SOURCE == 0 ? s_queue[jt] : cursor + jt));
                SN_ASSERT(SOURCE == 3 ? (uint64_t)rid < v.cap_f : (uint64_t)rid < v.cap_v);
                const GatheredSplat gs = SOURCE == 3 ? gather_splat(v.far_geo, v.far_recs, rid) : gather_splat(v.geo, v.recs, rid);
                FRec f;
                unsigned msk = tile_entry(gs.e1x, gs.e1y, gs.p1, gs.p2, gs.gl, gs.gr, x0 + 8.0, y0 + 8.0, f);
                if (kBound && !kPixBound && msk)  // eps at the support edge bounds eps inside it
                    atomicMax(&s_epsmax, __float_as_uint(-__fmaf_rn(f.nka, fminf(f.thr_out, 7.0f), f.nkb)));
                if (msk) s_f[jt] = f;  // an entry no warp walks is never read
                s_slot[jt] = rid;
                s_mask[jt] = (uint8_t)(msk | (msk && gs.gl.z > 0.99f ? 0x80u : 0u));  // bit 7: opacity > .99
            }
            __syncthreads();
            // each warp walks only the batch entries whose support can reach its 8 x 8 pixel block,
            // in depth order; the per-pixel tests below stay exact, the mask only skips whole warps
            int cnt = 0;
            bool hi_op = false;  // an entry of this warp's list has opacity > .99 (mask bit 7)
            for (int j0 = 0; j0 < n; j0 += 32) {
                const unsigned mk = j0 + lane < n ? s_mask[j0 + lane] : 0u;
                const bool mine = (mk >> warp) & 1u;
                const unsigned bal = __ballot_sync(kFull, mine);
                if (mine) s_wl[warp][cnt + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)((j0 + lane) * sizeof(FRec));
                hi_op |= __any_sync(kFull, mine && (mk & 0x80u));
                cnt += __popc(bal);
            }
            const int cnt_pad = (cnt + kWalkUnroll - 1) / kWalkUnroll * kWalkUnroll;
            SN_ASSERT(cnt_pad <= kBatch + kWalkUnroll);
            if (lane < cnt_pad - cnt) s_wl[warp][cnt + lane] = (uint16_t)(kBatch * sizeof(FRec));
            __syncwarp();
            // depth bounds of the contributions, once per batch instead of per contribution: the warp's
            // entries arrive in depth order, so its first one is a lower bound of every pixel's first
            // contribution, and its last one an upper bound of any contribution a pixel still live at
            // the batch's start makes in it
            const char *fbase = reinterpret_cast<const char *>(s_f);
            if (kBound && cnt > 0) {
                z_first = fminf(z_first, reinterpret_cast<const FRec *>(fbase + s_wl[warp][0])->z);
                const float zb = reinterpret_cast<const FRec *>(fbase + s_wl[warp][cnt - 1])->z;
                float z0, z1, d0, d1;
                unpack2(P.z_last, z0, z1);
                unpack2(P.dead, d0, d1);
                P.z_last = pack2(d0 == 0.0f ? fmaxf(z0, zb) : z0, d1 == 0.0f ? fmaxf(z1, zb) : z1);
            }
            // The walk carries NEGATED weights: na = -a (the record holds -alpha, the inside mask m is
            // 1 / 0), so T (1 - a) = fma(na, T, T) and err (1 - a) = fma(na, err, .) need no negation;
            // nw = -w, and the colour, depth and A sums accumulate negated (flipped once in the epilogue).
            auto walk = [&](auto clamp_tag) {
                constexpr bool kClamp = decltype(clamp_tag)::value;
                for (int k0 = 0; k0 < cnt_pad; k0 += 32) {
                    if (__all_sync(kFull, !(lo_of(P.dead) == 0.0f || hi_of(P.dead) == 0.0f))) break;
                    const int k1 = min(cnt_pad, k0 + 32);
                    for (int k = k0; k < k1; k += kWalkUnroll) {
        #pragma unroll
                    for (int ku = 0; ku < kWalkUnroll; ++ku) {
                        const FRec &s = *reinterpret_cast<const FRec *>(fbase + s_wl[warp][k + ku]);
                        PROF(0, lane == 0);
                        const float4 q0 = *reinterpret_cast<const float4 *>(&s.a1x);      // a1x a1y c2x c2y
                        const float4 q1 = *reinterpret_cast<const float4 *>(&s.V1);       // V1 V1 V2 V2
                        const float4 q2 = *reinterpret_cast<const float4 *>(&s.thr_out);  // thr_out thr_in nkb nkb
                        const float4 q3 = *reinterpret_cast<const float4 *>(&s.nka);      // nka alpha z -
                        // v_k for both pixels (same ox; oy and oy + 4), h = v1^2 + v2^2 (+ the finished offset)
                        const f32x2 v1 = fma2(OY, pack2(q0.y, q0.y), fma2(OX, pack2(q0.x, q0.x), pack2(q1.x, q1.y)));
                        const f32x2 v2 = fma2(OY, pack2(q0.w, q0.w), fma2(OX, pack2(q0.z, q0.z), pack2(q1.z, q1.w)));
                        const f32x2 h = fma2(v1, v1, fma2(v2, v2, P.dead));
                        f32x2 neps = fma2(h, pack2(q3.x, q3.x), pack2(q2.z, q2.w));  // -(alpha's relative bound)
                        float h0, h1;
                        unpack2(h, h0, h1);
        #ifdef SN_BLEND_PROF
                        {  // walk iterations where no pixel of the warp's block (live or not) is inside
                            float g0, g1;
                            unpack2(fma2(v1, v1, mul2(v2, v2)), g0, g1);
                            PROF(3, lane == 0 && !__any_sync(kFull, g0 <= q2.x || g1 <= q2.x));
                        }
        #endif
                        // 1 where the pixel is certainly inside the support, 0 where outside or finished
                        float m0 = le_mask(h0, q2.y), m1 = le_mask(h1, q2.y);
                        if ((h0 > q2.y && h0 <= q2.x) || (h1 > q2.y && h1 <= q2.x)) {
                            // boundary band (rare, divergent): the reference's float64 test (_kernels_cy.pyx:73-75)
                            PROF(1, 1);
                            const int j = (int)((reinterpret_cast<const char *>(&s) - fbase) / sizeof(FRec));
                            const SplatRec &sd = (SOURCE == 3 ? v.far_recs : v.recs)[s_slot[j]];
                            const double ddx = sd.mx - px;
                            float e0, e1;
                            unpack2(neps, e0, e1);
                            if (h0 > q2.y && h0 <= q2.x) {
                                const double ddy = sd.my - (py0 + 0.5);
                                const double d2d = (sd.ca * ddx * ddx + sd.cb2 * ddx * ddy) + sd.cc * ddy * ddy;
                                if (!(d2d > kSupportD2)) {
                                    m0 = 1.0f;
                                    h0 = (float)(d2d * kHalfLog2e);  // h, rounded once (within kEpsExact)
                                    e0 = -kEpsExact;
                                }
                            }
                            if (h1 > q2.y && h1 <= q2.x) {
                                const double ddy = sd.my - (py1 + 0.5);
                                const double d2d = (sd.ca * ddx * ddx + sd.cb2 * ddx * ddy) + sd.cc * ddy * ddy;
                                if (!(d2d > kSupportD2)) {
                                    m1 = 1.0f;
                                    h1 = (float)(d2d * kHalfLog2e);
                                    e1 = -kEpsExact;
                                }
                            }
                            neps = pack2(e0, e1);
                        }
                        const f32x2 m = pack2(m0, m1);
                        // alpha = min(o 2^-h, .99) inside the support, 0 outside: T, err and the sums then
                        // stay exactly as they were (w = 0, T (1 - 0) = T, err (1 - 0) + 0)
                        float e0, e1;
                        unpack2(mul2(pack2(ex2_approx(-h0), ex2_approx(-h1)), pack2(q3.y, q3.y)), e0, e1);  // -o 2^-h
                        // min(., .99) only matters for opacities above .99 (o 2^-h <= o): batches without one skip it
                        const f32x2 na = kClamp ? mul2(pack2(fmaxf(e0, -0.99f), fmaxf(e1, -0.99f)), m)
                                                : mul2(pack2(e0, e1), m);  // -a
                        const f32x2 nw = mul2(na, P.T);                                       // -w
                        const f32x2 Tn = fma2(na, P.T, P.T);  // T (1 - a), rounded once
                        const float4 q4 = *reinterpret_cast<const float4 *>(&s.r);  // r g b -
                        P.cr = fma2(nw, pack2(q4.x, q4.x), P.cr);
                        P.cg = fma2(nw, pack2(q4.y, q4.y), P.cg);
                        P.cb = fma2(nw, pack2(q4.z, q4.z), P.cb);
                        P.D = fma2(nw, pack2(q3.z, q3.z), P.D);
                        P.A = add2(P.A, nw);
                        // err (1 - a) + w eps + 1.25 u T' (the rounding term only where T changed)
                        P.err = fma2(na, P.err, fma2(nw, neps, fma2(Tn, mul2(m, pack2(kU125, kU125)), P.err)));
                        P.T = Tn;
                        P.nc = add2(P.nc, m);
                        // near the cutoff (_kernels_cy.pyx:65-66): stop; decided or deferred after the walk
                        // (+ kDead once per step past it: a finished pixel's offset only grows, ~1e30 per
                        // walked entry, far from overflow; liveness is dead == 0)
                        float g0, g1;
                        unpack2(sub2(Tn, P.err), g0, g1);
                        P.dead = fma2(pack2(le_mask(g0, kTHi), le_mask(g1, kTHi)), pack2(kDead, kDead), P.dead);
                    }
                    }
                }
            };
            if (hi_op)
                walk(std::true_type{});
            else
                walk(std::false_type{});
            if (SOURCE == 0) {  // drop the consumed head of the queue
                const int rest = q_len - n;
                uint32_t qv0 = threadIdx.x < rest ? s_queue[n + threadIdx.x] : 0u;
                uint32_t qv1 = threadIdx.x + kBT < rest ? s_queue[n + kBT + threadIdx.x] : 0u;
                __syncthreads();
                if (threadIdx.x < rest) s_queue[threadIdx.x] = qv0;
                if (threadIdx.x + kBT < rest) s_queue[kBT + threadIdx.x] = qv1;
                q_len = rest;
            } else {
                cursor += n;
            }
        }
    #ifdef SN_BLEND_PROF
        const bool prof_live = __syncthreads_or(lo_of(P.dead) == 0.0f || hi_of(P.dead) == 0.0f) != 0;
        if (SOURCE == 0 && MODE == 0 && threadIdx.x == 0) {
            const uint32_t st = (uint32_t)v.env_off[el], tot = s1 - st;
            // consumed: the list position the walk had reached (queued-but-unwalked entries excluded)
            const uint32_t used = (cursor - st) - (uint32_t)q_len;
            const unsigned fr = tot ? (unsigned)((1000ull * used) / tot) : 0u;
            atomicMax(&g_env_frac[el & 63], fr);
            // log-spaced bins of the consumed fraction (1e-5 units): <=0.1%, 0.2, 0.5, 1, 2, 5, 10, 20,
            // 50, <100%; bin 10: the list ran out with a live (unsaturated) pixel
            const unsigned f5 = tot ? (unsigned)((100000ull * used) / tot) : 0u;
            const unsigned edges[9] = {100, 200, 500, 1000, 2000, 5000, 10000, 20000, 50000};
            unsigned bin = 9;
            for (int k = 8; k >= 0; --k)
                if (f5 <= edges[k]) bin = k;
            if (prof_live && cursor >= s1 && q_len == 0) bin = 10;
            atomicAdd(&g_blend_prof[4 + bin], 1ull);
        }
        for (int i = 0; i < 16; ++i)
            if (prof[i]) atomicAdd(&g_blend_prof[i], prof[i]);
    #endif
        if (b.scans && threadIdx.x == 0 && scanned) atomicAdd(b.scans, (unsigned long long)scanned);
        if (b.loads && threadIdx.x == 0 && loaded) atomicAdd(b.loads, (unsigned long long)loaded);

        // Depth-sliced pass: the near list ran out. A tile with a live pixel (or one whose cutoff is
        // undecided: its float64 walk may need to go on) and far splats in its env registers as
        // unfinished, saves its pixels' state and leaves the live pixels to the continuation (source 3).
        bool saved = false;
        // (Only tiles that reached the end of the near list: a tile whose pixels all stopped before it
        // leaves its undecided pixels' float64 walks the rest of the near list, which ends them but
        // for a pathological few -- those set far_short and the render is re-run unsliced.)
        if (SOURCE == 0 && v.sliced && cursor >= s1 && q_len == 0) {
            float Tq[2], Eq[2], Dq[2];
            unpack2(P.T, Tq[0], Tq[1]);
            unpack2(P.err, Eq[0], Eq[1]);
            unpack2(P.dead, Dq[0], Dq[1]);
            bool need = false;
    #pragma unroll
            for (int p = 0; p < 2; ++p) {
                const bool cutq = Tq[p] - Eq[p] <= kTHi;
                const bool ambq = cutq && (!(Tq[p] + Eq[p] < kTLo) || Eq[p] > 0.0625f * Tq[p]);
                need |= (p ? in1 : in0) && (Dq[p] == 0.0f || (ambq && !(g_slice_hooks & 2)));
            }
            const bool has_far = v.env_off[v.ec + el + 1] > v.env_off[v.ec + el];
            if (__syncthreads_or(need) && has_far) {
                if (threadIdx.x == 0) {
                    const unsigned long long uu = atomicAdd(b.unfin_count, 1ull);
                    s_u = uu < v.far_cap_u ? (int)uu : -1;
                    if (s_u >= 0) {
                        atomicOr(b.unfin_envs, 1ull << el);
                        b.unfin_list[s_u] = ((uint32_t)el << 16) | (uint32_t)tile;
                        b.bucket_of[(int64_t)el * (tiles_of(b.width) * tiles_of(b.height)) + tile] = s_u;
                    }
                }
                __syncthreads();
                const int us = s_u;
                if (us >= 0) {
                    float *st = b.state + (size_t)us * kStateF * kBT + threadIdx.x;
                    const f32x2 f[10] = {P.T, P.err, P.A, P.cr, P.cg, P.cb, P.D, P.dead, P.z_last, P.nc};
    #pragma unroll
                    for (int q = 0; q < 10; ++q) {
                        st[(2 * q) * kBT] = lo_of(f[q]);
                        st[(2 * q + 1) * kBT] = hi_of(f[q]);
                    }
                    st[20 * kBT] = z_first;
                    st[21 * kBT] = __uint_as_float(s_epsmax);
                }
                saved = true;  // (on overflow the render is re-run: these pixels' outputs do not matter)
            }
        }

        const sn_camera &cam = b.cams[env];
        if (!kPixBound) P.eps_max = pack2(__uint_as_float(s_epsmax), __uint_as_float(s_epsmax));
        float T2[2], E2[2], A2[2], CR[2], CG[2], CB[2], DD[2], EM[2], ZL[2];
        unpack2(P.T, T2[0], T2[1]);
        unpack2(P.err, E2[0], E2[1]);
        unpack2(P.A, A2[0], A2[1]);
        unpack2(P.cr, CR[0], CR[1]);
        unpack2(P.cg, CG[0], CG[1]);
        unpack2(P.cb, CB[0], CB[1]);
        unpack2(P.D, DD[0], DD[1]);
        unpack2(P.eps_max, EM[0], EM[1]);
        unpack2(P.z_last, ZL[0], ZL[1]);
        float NCf[2];
        unpack2(P.nc, NCf[0], NCf[1]);
        const int NC[2] = {(int)NCf[0], (int)NCf[1]};
    #pragma unroll
        for (int p = 0; p < 2; ++p) {  // the walk accumulated negated sums (exact: negation is exact)
            A2[p] = -A2[p];
            CR[p] = -CR[p];
            CG[p] = -CG[p];
            CB[p] = -CB[p];
            DD[p] = -DD[p];
        }
        float DL[2];
        unpack2(P.dead, DL[0], DL[1]);
        // the pixels this launch finishes: every pixel, but a saved tile's live ones (the continuation
        // finishes them) and, in the continuation, only the pixels that were live when it resumed
        const bool FIN[2] = {SOURCE == 3 ? entry_live0 : !(saved && DL[0] == 0.0f),
                             SOURCE == 3 ? entry_live1 : !(saved && DL[1] == 0.0f)};
        const bool IN[2] = {in0, in1};
        const int PY[2] = {py0, py1};
        unsigned contrib_sum = 0;
    #pragma unroll
        for (int p = 0; p < 2; ++p) {
            const float T = T2[p], err = E2[p], A = A2[p];
            const int nc = NC[p];
            const bool inside = IN[p];
            const int py_i = PY[p];
            // the cutoff fired (T - err <= 1e-4 (1 + 1e-6)) but T < 1e-4 is not certain: float64 fixup.
            // Also when err > T / 16: the 0.25 u T' margin in kU125 covers the bound's own float
            // roundings (<= 2u err per step) only while err <= T / 8, and err / T never decreases.
            const bool cut = T - err <= kTHi;
            const bool amb = inside && (b.force_exact || (cut && (!(T + err < kTLo) || err > 0.0625f * T)));
            PROF(2, amb);
    #ifdef SN_FIX_PROF
            if (MODE == 0 && amb) {
                atomicAdd(&g_fix_prof[0], 1ull);
                if (b.force_exact) atomicAdd(&g_fix_prof[13], 1ull);
                if (err > 0.0625f * T) atomicAdd(&g_fix_prof[1], 1ull);
                atomicAdd(&g_fix_prof[T >= kTHi ? 2 : T >= kTLo ? 3 : 4], 1ull);
                const float lr = T > 0.0f && err > 0.0f ? log10f(err / T) : -9.0f;
                atomicAdd(&g_fix_prof[5 + min(7, max(0, (int)floorf(lr) + 8))], 1ull);
                if (fabsf(T - 1.0e-4f) <= 1.0e-9f) atomicAdd(&g_fix_prof[14], 1ull);
                if (nc <= 4) atomicAdd(&g_fix_prof[15], 1ull);
            }
    #endif
            const int64_t pix = ((int64_t)env * b.height + py_i) * b.width + px_i;
            const uint32_t code = (uint32_t)(((int64_t)el * b.height + py_i) * b.width + px_i);
            // Error bounds of the outputs the compositor decides on. Every weight w_i = a_i T_(i-1) has
            // relative error <= rho_w (transmittance bound + largest alpha bound + the product's
            // rounding); depth = sum z w / sum w then errs by <= rho_w (z_last - z_first) from the
            // weights (z spans the contributions) plus (2n + 2) u from the float sums and the division;
            // alpha by rho_w + (n + 1) u.
            const float zf = nc == 0 ? 3.0e38f : z_first;  // no contribution: the empty range
            const float rho_w = err / T + EM[p] + 6.0e-8f;
            const float alpha = fminf(A, 1.0f);
            const float depth = A > 0.0f ? DD[p] / A : (float)cam.far_;
            const float d_err = 1.01f * (rho_w * (ZL[p] - zf) + (float)(2 * nc + 2) * 6.0e-8f * depth);
            const bool fin = FIN[p];
            const bool flag = inside && amb && fin;
            contrib_sum += (flag || !fin) ? 0u : (unsigned)nc;
            if (kInCta) {
                if (flag) {
                    const unsigned k = atomicAdd(&s_nfix, 1u);
                    SN_ASSERT(k < 2u * kBT);
                    s_fixpix[k] = code;
                }
            } else {
                push_fixup(b, flag, code);
            }
            if (!inside || !fin) continue;
            if (MODE == 2 && SOURCE != 1 && threadIdx.x == 0 && p == 0) b.tile_flag[(int64_t)el * (tiles_of(b.width) * tiles_of(b.height)) + tile] = 1;
            if (flag) {
                if (MODE == 2) b.ldepth[pix] = __int_as_float(0x7fc00000);  // NaN: pending float64 fixup
                continue;
            }
            if (b.contrib) b.contrib[pix] = nc;
            if (MODE == 0) {
                float *oc = b.color + 3 * pix;
                const float o0 = np_clipf(__fmaf_rn((float)cam.background[0], T, CR[p]), 0.0f, 1.0f);
                const float o1 = np_clipf(__fmaf_rn((float)cam.background[1], T, CG[p]), 0.0f, 1.0f);
                const float o2 = np_clipf(__fmaf_rn((float)cam.background[2], T, CB[p]), 0.0f, 1.0f);
                oc[0] = o0;
                oc[1] = o1;
                oc[2] = o2;
                b.alpha[pix] = alpha;
                b.depth[pix] = depth;
                if (b.derr) b.derr[pix] = A > 0.0f ? d_err : 0.0f;
                store_payload(b, pix, o0, o1, o2, depth);
                continue;
            }
            float fc0 = 0.0f, fc1 = 0.0f, fc2 = 0.0f;
            if (A > 0.0f) {
                fc0 = np_clipf(CR[p] / A, 0.0f, 1.0f);
                fc1 = np_clipf(CG[p] / A, 0.0f, 1.0f);
                fc2 = np_clipf(CB[p] / A, 0.0f, 1.0f);
            }
            if (MODE == 1) {
                float *oc = b.color + 3 * pix;
                oc[0] = fc0;
                oc[1] = fc1;
                oc[2] = fc2;
                b.alpha[pix] = alpha;
                b.depth[pix] = depth;
                store_payload(b, pix, fc0, fc1, fc2, depth);
                continue;
            }
            // MODE 2: the layer frame goes to its own buffers; composite_kernel merges it into the scene
            // frame once the scene pass is done (so this blend runs concurrently with the scene blend)
            float *lc = b.lcolor + 3 * pix;
            lc[0] = fc0;
            lc[1] = fc1;
            lc[2] = fc2;
            b.lalpha[pix] = alpha;
            b.ldepth[pix] = depth;
            b.lderr[pix] = d_err;
            b.laerr[pix] = 1.01f * (rho_w + (float)(nc + 1) * 6.0e-8f) * A + 6.0e-8f;
        }
        if (b.contribs) {
            const unsigned sum = __reduce_add_sync(kFull, contrib_sum);
            if (lane == 0 && sum) atomicAdd(b.contribs, (unsigned long long)sum);
        }
        if (kInCta) {
            __syncthreads();
            const unsigned nfix = s_nfix;
            if (nfix) {
                double *s_exp = reinterpret_cast<double *>(s_f);  // (the batch buffers are free now)
                QEntry *q = reinterpret_cast<QEntry *>(s_exp + 64) + warp * kQueue;
                if (threadIdx.x < 64) s_exp[threadIdx.x] = kExp2Tbl[threadIdx.x];
                __syncthreads();
                PassView fv = v;
                fv.far_phase = v.sliced ? 1 : 0;  // a walk that needs the far bucket goes to the fixup pass
                const unsigned hw = (unsigned)b.width * (unsigned)b.height;
                unsigned long long nc_sum = 0;
                for (unsigned i = warp; i < nfix; i += kBW) {
                    const uint32_t code = s_fixpix[i];
                    const int pp = (int)(code % hw);
                    const int fy = pp / b.width, fx = pp % b.width;
                    const ExactPixel f = exact_pixel<SN_FIXUP_PER>(fv, el, tile, b.tiles_x, fx, fy, s_exp, q);
                    if (f.out) {
                        defer_to_far(b, el, tile, code);
                        continue;
                    }
                    nc_sum += (unsigned)f.nc;
                    if (lane == 0) write_exact_scene(b, f, ((int64_t)env * b.height + fy) * b.width + fx, cam);
                }
                if (b.contribs && lane == 0 && nc_sum) atomicAdd(b.contribs, nc_sum);
            }
        }
#undef PROF
    };
    if (SOURCE == 3) {  // the unfinished tiles, taken dynamically by a few CTAs per SM
        const uint32_t n_items = (uint32_t)min(*v.far_unfin, (unsigned long long)v.far_cap_u);
        while (true) {
            if (threadIdx.x == 0) s_u = (int)atomicAdd(v.far_next, 1u);
            __syncthreads();
            const int item = s_u;
            __syncthreads();
            if ((uint32_t)item >= n_items) break;
            const uint32_t key = v.far_unfin_list[item];
            if (key & kLateTile) continue;  // registered by the first fixup pass: no live pixels
            do_tile((int)(key & 0xffffu), (int)((key >> 16) & 0xffu), item);
            __syncthreads();  // the next tile reuses the shared buffers
        }
    } else {
        do_tile(blockIdx.x, blockIdx.y, -1);
    }
}

#ifndef SN_LAYER_PX1_MIN_BLOCKS
#define SN_LAYER_PX1_MIN_BLOCKS 4
#endif
template <int MODE, int SOURCE>
__global__ void __launch_bounds__(kBlock, SN_LAYER_PX1_MIN_BLOCKS) blend_kernel_px1(BlendArgs b) {
    constexpr bool kBound = MODE != 1;  // depth error bounds feed the compositor
    // the layer tracks each pixel's largest alpha bound (it decides the compositor's depth choice);
    // the scene pass uses the CTA's largest bound over every gathered splat -- looser, one
    // instruction less per contribution
    constexpr bool kPixBound = MODE == 2;
    // records per batch: tile lists (the avatar layer) take 2 per thread -- their warps' walks are
    // very uneven (small splats in a few blocks), and fewer, larger batches wait less at barriers
#ifndef SN_STREAM_PER_THREAD
#define SN_STREAM_PER_THREAD 1
#endif
#ifndef SN_LIST_PER_THREAD
#define SN_LIST_PER_THREAD 2
#endif
    constexpr int kPerT = SOURCE == 1 ? SN_LIST_PER_THREAD : (SOURCE == 0 ? SN_STREAM_PER_THREAD : 1);
    constexpr int kBatch = kBlock * kPerT;
    using WlIndex = typename std::conditional<(kBatch > 256), uint16_t, uint8_t>::type;
    __shared__ unsigned s_epsmax;
    __shared__ FRec1 s_f[kBatch];
    __shared__ uint32_t s_slot[kBatch];  // record slot (the boundary band reads its SplatRec)
    __shared__ uint32_t s_queue[SOURCE == 0 ? kBatch + kBlock : 1];
    __shared__ uint32_t s_wsum[kBlock / 32];
    __shared__ uint8_t s_mask[kBatch];  // bit w: the splat's support may reach warp w's 8 x 4 block
    __shared__ WlIndex s_wl[kBlock / 32][kBatch];  // per warp: its batch entries, in depth order
    const PassView &v = b.pv;
    if (pass_overflow(v)) return;
    const int n_tiles_all = tiles_of(b.width) * tiles_of(b.height);
    // one (env, tile): the whole blend of a tile, as a lambda so the listed mode below can loop
    auto do_tile = [&](const int tile, const int el) {
        if (threadIdx.x == 0) s_epsmax = __float_as_uint(kEpsExact);
        const int env = b.e0 + el;
        const int tx = tile % b.tiles_x, ty = tile / b.tiles_x;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
        const int px_i = tx * kTile + lx;
        const int py_i = ty * kTile + ly;
        const bool inside = px_i < b.width && py_i < b.height;
        const double px = px_i + 0.5, py = py_i + 0.5;
        const double x0 = tx * kTile, y0 = ty * kTile;
        const float oxf = (float)lx - 7.5f, oyf = (float)ly - 7.5f;  // pixel centre - tile centre
    #ifdef SN_BLEND_PROF
        unsigned long long prof[16] = {};
    #define PROF(i, x) (prof[i] += (x))
    #else
    #define PROF(i, x) ((void)0)
    #endif

        uint32_t cursor, s1;
        if (SOURCE == 1) {
            uint2 r = v.ranges[((uint32_t)el << v.tile_bits) | (uint32_t)tile];
            cursor = r.x;
            s1 = r.y;
            // composite of an empty layer tile: front alpha 0 and depth `far`, and the scene depth is a
            // weighted mean of z < far, so `front.depth < back.depth` never holds -- nothing to do
            if (MODE == 2) {
                if (threadIdx.x == 0) b.tile_flag[(int64_t)el * n_tiles_all + tile] = cursor != s1;
                if (cursor == s1) return;
            }
        } else {
            cursor = (uint32_t)v.env_off[el];
            s1 = (uint32_t)v.env_off[el + 1];
        }

        float T = 1.0f, A = 0.0f, err = 0.0f;
        f32x2 crg = 0ull, cbd = 0ull;  // (colour r, g), (colour b, depth sum)
        const f32x2 o2x = pack2(oxf, oxf), o2y = pack2(oyf, oyf);
        float eps_max = 0.0f, z_first = 3.0e38f, z_last = 0.0f;
        int nc = 0;
        // added to d2: a finished pixel skips every splat. A pixel is finished when it is outside the
        // frame, forced exact, or past the cutoff test (after which T and err never change, so the
        // cutoff's ambiguity is re-derived from them after the walk)
        float dead = (!inside || b.force_exact) ? INFINITY : 0.0f;
        uint32_t loaded = 0, scanned = 0;
        int q_len = 0;  // SOURCE 0: entries waiting in s_queue (uniform across the CTA)
        while (true) {
            if (__syncthreads_count(dead == 0.0f) == 0) break;  // also guards s_f / s_queue reuse
            int n;
            if (SOURCE == 0) {
                stream_fill<kBlock>(v, tx, ty, kBatch, cursor, s1, q_len, scanned, s_queue, s_wsum);
                n = min(q_len, kBatch);
            } else {
                n = (int)min((uint32_t)kBatch, s1 - cursor);
            }
            if (n <= 0) break;
            loaded += n;
    #pragma unroll
            for (int r = 0; r < kPerT; ++r) {
                const int jt = threadIdx.x + r * kBlock;
                if (jt >= n) break;
                // the record slot: tile lists hold slots; streamed / all-splat sources map depth ranks
                const uint32_t rid = SOURCE == 1 ? __ldg(v.pair_vals + cursor + jt)
                                                 : __ldg(v.order + (SOURCE == 0 ? s_queue[jt] : cursor + jt));
                const GatheredSplat gs = gather_splat(v.geo, v.recs, rid);
                FRec1 f;
                unsigned msk = tile_entry_8x4(gs.e1x, gs.e1y, gs.p1, gs.p2, gs.gl, gs.gr, x0 + 8.0, y0 + 8.0, f);
                if (kBound && !kPixBound && msk)  // eps at the support edge bounds eps inside it
                    atomicMax(&s_epsmax, __float_as_uint(__fmaf_rn(f.ka, fminf(f.thr_out, 7.0f), f.kb)));
                if (msk) s_f[jt] = f;  // an entry no warp walks is never read
                s_slot[jt] = rid;
                s_mask[jt] = (uint8_t)msk;
            }
            __syncthreads();
            // each warp walks only the batch entries whose support can reach its 8 x 4 pixel block,
            // in depth order; the per-pixel tests below stay exact, the mask only skips whole warps
            int cnt = 0;
            for (int j0 = 0; j0 < n; j0 += 32) {
                const bool mine = j0 + lane < n && ((s_mask[j0 + lane] >> warp) & 1u);
                const unsigned bal = __ballot_sync(kFull, mine);
                if (mine) s_wl[warp][cnt + __popc(bal & ((1u << lane) - 1u))] = (WlIndex)(j0 + lane);
                cnt += __popc(bal);
            }
            __syncwarp();
            // a lower bound on the pixel's first contribution depth, once per batch instead of per
            // contribution: the warp's entries arrive in depth order, so its first one is the nearest
            if (kBound && cnt > 0) z_first = fminf(z_first, s_f[s_wl[warp][0]].z);
            for (int k0 = 0; k0 < cnt && !__all_sync(kFull, dead != 0.0f); k0 += 32) {
                const int k1 = min(cnt, k0 + 32);
    #pragma unroll kWalkUnroll
                for (int k = k0; k < k1; ++k) {
                    const int j = s_wl[warp][k];
                    PROF(0, lane == 0);
                    const FRec1 &s = s_f[j];
                    const float4 q0 = *reinterpret_cast<const float4 *>(&s.a1x);
                    const float4 q1 = *reinterpret_cast<const float4 *>(&s.V1);
                    float v1, v2;
                    unpack2(fma2(pack2(q0.x, q0.y), o2x, fma2(pack2(q0.z, q0.w), o2y, pack2(q1.x, q1.y))), v1, v2);
                    // + dead: exact (v2^2 + 0 rounds like v2 * v2), or +inf for a finished pixel
                    float d2 = __fmaf_rn(v1, v1, __fmaf_rn(v2, v2, dead));
                    if (d2 > q1.z) continue;  // saturated (dead = inf), or certainly outside the support
                    const float4 q2 = *reinterpret_cast<const float4 *>(&s.ka);  // (ka, kb, alpha, -): one load
                    float eps;
                    if (d2 < q1.w) {
                        eps = __fmaf_rn(d2, q2.x, q2.y);
                    } else {  // boundary band: the reference's float64 test (_kernels_cy.pyx:73-75)
                        PROF(1, 1);
                        const SplatRec &sd = v.recs[s_slot[j]];
                        const double ddx = sd.mx - px, ddy = sd.my - py;
                        const double d2d = (sd.ca * ddx * ddx + sd.cb2 * ddx * ddy) + sd.cc * ddy * ddy;
                        if (d2d > kSupportD2) continue;
                        d2 = (float)(d2d * kHalfLog2e);  // h, rounded once (within kEpsExact)
                        eps = kEpsExact;
                    }
                    const float e = ex2_approx(-d2);  // 2^-h: the negation is an operand modifier
                    const float a = fminf(q2.z * e, 0.99f);
                    const float w = a * T;
                    const float Tn = __fmaf_rn(-a, T, T);  // T (1 - a), rounded once
                    const float4 q3 = *reinterpret_cast<const float4 *>(&s.r);
                    crg = fma2(pack2(q3.x, q3.y), pack2(w, w), crg);
                    cbd = fma2(pack2(q3.z, q3.w), pack2(w, w), cbd);
                    A = A + w;
                    err = __fmaf_rn(-a, err, __fmaf_rn(w, eps, __fmaf_rn(Tn, kU125, err)));  // err (1 - a) + ...
                    T = Tn;
                    ++nc;
                    if (kPixBound) eps_max = fmaxf(eps_max, eps);
                    if (kBound) z_last = fmaxf(z_last, q3.w);  // one op into a fixed register (a copy would be two)
                    // near the cutoff (_kernels_cy.pyx:65-66): stop; decided or deferred after the walk
                    if (Tn - err <= kTHi) dead = INFINITY;
                }
            }
            if (SOURCE == 0) {  // drop the consumed head of the queue
                int rest = q_len - n;
                uint32_t qv = threadIdx.x < rest ? s_queue[n + threadIdx.x] : 0u;
                __syncthreads();
                if (threadIdx.x < rest) s_queue[threadIdx.x] = qv;
                q_len = rest;
            } else {
                cursor += n;
            }
        }
        float cr, cg, cb, D;
        unpack2(crg, cr, cg);
        unpack2(cbd, cb, D);
        // the cutoff fired (T - err <= 1e-4 (1 + 1e-6)) but T < 1e-4 is not certain: float64 fixup.
        // Also when err > T / 16: the 0.25 u T' margin in kU125 covers the bound's own float roundings
        // (<= 2u err per step) only while err <= T / 8, and err / T never decreases along the walk.
        const bool cut = T - err <= kTHi;
        const bool amb = inside && (b.force_exact || (cut && (!(T + err < kTLo) || err > 0.0625f * T)));
        PROF(2, amb);
    #ifdef SN_BLEND_PROF
        const bool prof_live = __syncthreads_or(dead == 0.0f) != 0;
        if (SOURCE == 0 && MODE == 0 && threadIdx.x == 0) {
            const uint32_t st = (uint32_t)v.env_off[el], tot = s1 - st;
            // consumed: the list position the walk had reached (queued-but-unwalked entries excluded)
            const uint32_t used = (cursor - st) - (uint32_t)q_len;
            const unsigned fr = tot ? (unsigned)((1000ull * used) / tot) : 0u;
            atomicMax(&g_env_frac[el & 63], fr);
            // log-spaced bins of the consumed fraction (1e-5 units): <=0.1%, 0.2, 0.5, 1, 2, 5, 10, 20,
            // 50, <100%; bin 14: the list ran out with a live (unsaturated) pixel
            const unsigned f5 = tot ? (unsigned)((100000ull * used) / tot) : 0u;
            const unsigned edges[9] = {100, 200, 500, 1000, 2000, 5000, 10000, 20000, 50000};
            unsigned bin = 9;
            for (int k = 8; k >= 0; --k)
                if (f5 <= edges[k]) bin = k;
            if (prof_live && cursor >= s1 && q_len == 0) bin = 10;
            atomicAdd(&g_blend_prof[4 + bin], 1ull);
        }
        for (int i = 0; i < 16; ++i)
            if (prof[i]) atomicAdd(&g_blend_prof[i], prof[i]);
    #endif
        if (b.scans && threadIdx.x == 0 && scanned) atomicAdd(b.scans, (unsigned long long)scanned);
        if (b.loads && threadIdx.x == 0 && loaded) atomicAdd(b.loads, (unsigned long long)loaded);

        const sn_camera &cam = b.cams[env];
        const int64_t pix = ((int64_t)env * b.height + py_i) * b.width + px_i;
        const uint32_t code = (uint32_t)(((int64_t)el * b.height + py_i) * b.width + px_i);
        // Error bounds of the outputs the compositor decides on. Every weight w_i = a_i T_(i-1) has
        // relative error <= rho_w (transmittance bound + largest alpha bound + the product's rounding);
        // depth = sum z w / sum w then errs by <= rho_w (z_last - z_first) from the weights (z spans the
        // contributions) plus (2n + 2) u from the float sums and the division; alpha by rho_w + (n + 1) u.
        if (!kPixBound) eps_max = __uint_as_float(s_epsmax);
        if (nc == 0) z_first = 3.0e38f;  // no contribution: the empty range, as before any batch
        const float rho_w = err / T + eps_max + 6.0e-8f;
        const float alpha = fminf(A, 1.0f);
        const float depth = A > 0.0f ? D / A : (float)cam.far_;
        const float d_err = 1.01f * (rho_w * (z_last - z_first) + (float)(2 * nc + 2) * 6.0e-8f * depth);
        const bool flag = inside && amb;
        if (b.contribs) {
            unsigned sum = __reduce_add_sync(kFull, flag ? 0u : (unsigned)nc);
            if (lane == 0 && sum) atomicAdd(b.contribs, (unsigned long long)sum);
        }
        push_fixup(b, flag, code);
        if (!inside) return;
        if (MODE == 2 && SOURCE != 1 && threadIdx.x == 0) b.tile_flag[(int64_t)el * n_tiles_all + tile] = 1;
        if (flag) {
            if (MODE == 2) b.ldepth[pix] = __int_as_float(0x7fc00000);  // NaN: pending float64 fixup
            return;
        }
        if (b.contrib) b.contrib[pix] = nc;
        if (MODE == 0) {
            float *oc = b.color + 3 * pix;
            const float o0 = np_clipf(__fmaf_rn((float)cam.background[0], T, cr), 0.0f, 1.0f);
            const float o1 = np_clipf(__fmaf_rn((float)cam.background[1], T, cg), 0.0f, 1.0f);
            const float o2 = np_clipf(__fmaf_rn((float)cam.background[2], T, cb), 0.0f, 1.0f);
            oc[0] = o0;
            oc[1] = o1;
            oc[2] = o2;
            b.alpha[pix] = alpha;
            b.depth[pix] = depth;
            if (b.derr) b.derr[pix] = A > 0.0f ? d_err : 0.0f;
            store_payload(b, pix, o0, o1, o2, depth);
            return;
        }
        float fc0 = 0.0f, fc1 = 0.0f, fc2 = 0.0f;
        if (A > 0.0f) {
            fc0 = np_clipf(cr / A, 0.0f, 1.0f);
            fc1 = np_clipf(cg / A, 0.0f, 1.0f);
            fc2 = np_clipf(cb / A, 0.0f, 1.0f);
        }
        if (MODE == 1) {
            float *oc = b.color + 3 * pix;
            oc[0] = fc0;
            oc[1] = fc1;
            oc[2] = fc2;
            b.alpha[pix] = alpha;
            b.depth[pix] = depth;
            store_payload(b, pix, fc0, fc1, fc2, depth);
            return;
        }
        // MODE 2: the layer frame goes to its own buffers; composite_kernel merges it into the scene
        // frame once the scene pass is done (so this blend runs concurrently with the scene blend)
        float *lc = b.lcolor + 3 * pix;
        lc[0] = fc0;
        lc[1] = fc1;
        lc[2] = fc2;
        b.lalpha[pix] = alpha;
        b.ldepth[pix] = depth;
        b.lderr[pix] = d_err;
        b.laerr[pix] = 1.01f * (rho_w + (float)(nc + 1) * 6.0e-8f) * A + 6.0e-8f;
#undef PROF
    };
    if (SOURCE == 1 && MODE == 2 && v.tile_list) {
        // listed mode: only the (env, tile) pairs that hold layer splats (ranges_kernel's list), taken
        // dynamically by a grid of a few CTAs per SM -- most of the layer's tiles are empty, and a
        // CTA per tile would spend the pass launching and retiring them
        __shared__ int s_item;
        const uint32_t n_items = *v.n_list;
        while (true) {
            if (threadIdx.x == 0) s_item = (int)atomicAdd(v.list_next, 1u);
            __syncthreads();
            const int item = s_item;
            __syncthreads();
            if ((uint32_t)item >= n_items) break;
            const uint32_t key = v.tile_list[item];
            do_tile((int)(key & ((1u << v.tile_bits) - 1u)), (int)(key >> v.tile_bits));
            __syncthreads();  // the next tile reuses the shared buffers
        }
    } else {
        do_tile(blockIdx.x, blockIdx.y);
    }
}

// The avatar layer's listed blend with TWO 8 x 4 pixel blocks per warp (SN_LAYER_LP2): 128-thread
// CTAs, warp w owning blocks w and 7 - w of the tile (opposite corners: a cluster of small splats
// loads one corner, so the pair evens out what a warp per block leaves to the slowest warp at each
// barrier). Per batch the CTA gathers the tile list's records once, each warp builds a list per
// block and walks them one after the other with that block's pixel state (no lane idles for the
// other block, unlike a paired-pixel chain). Numerics, outputs and fixups are blend_kernel_px1's
// (MODE 2, SOURCE 1): the same per-pixel float32 chain, in the same order.
#ifndef SN_LAYER_LP2
#define SN_LAYER_LP2 1
#endif
#ifndef SN_LAYER_LP2_MIN_BLOCKS
#define SN_LAYER_LP2_MIN_BLOCKS 8
#endif
#ifndef SN_LP2_UNROLL
#define SN_LP2_UNROLL 1  // the walk's unroll (measured: 1 > 2, 4 -- smaller code beside the scene blend)
#endif
constexpr int kLp2Unroll = SN_LP2_UNROLL;
#ifndef SN_LAYER_LP2_PER_THREAD
#define SN_LAYER_LP2_PER_THREAD 2  // records per thread per batch
#endif
constexpr int kLT = 128;           // threads per layer CTA
constexpr int kLWarps = kLT / 32;  // 4 warps x 2 blocks = the tile's 8 blocks
__global__ void __launch_bounds__(kLT, SN_LAYER_LP2_MIN_BLOCKS) blend_kernel_lp2(BlendArgs b) {
    constexpr int kPerT = SN_LAYER_LP2_PER_THREAD;
    constexpr int kBatch = kLT * kPerT;
    __shared__ FRec1 s_f[kBatch];
    __shared__ uint32_t s_slot[kBatch];
    __shared__ uint8_t s_mask[kBatch];  // bit k: the splat's support may reach block k (8 x 4)
    __shared__ uint16_t s_wl[kLWarps][2][kBatch];
    __shared__ int s_item;
    const PassView &v = b.pv;
    if (pass_overflow(v)) return;
    const int n_tiles_all = tiles_of(b.width) * tiles_of(b.height);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int blk[2] = {warp, 7 - warp};
    const uint32_t n_items = *v.n_list;
    while (true) {
        if (threadIdx.x == 0) s_item = (int)atomicAdd(v.list_next, 1u);
        __syncthreads();
        const int item = s_item;
        __syncthreads();
        if ((uint32_t)item >= n_items) break;
        const uint32_t key = v.tile_list[item];
        const int tile = (int)(key & ((1u << v.tile_bits) - 1u)), el = (int)(key >> v.tile_bits);
        const int env = b.e0 + el;
        const int tx = tile % b.tiles_x, ty = tile / b.tiles_x;
        const uint2 rg = v.ranges[((uint32_t)el << v.tile_bits) | (uint32_t)tile];
        uint32_t cursor = rg.x;
        const uint32_t s1 = rg.y;
        if (threadIdx.x == 0) b.tile_flag[(int64_t)el * n_tiles_all + tile] = cursor != s1;
        const double x0 = tx * kTile, y0 = ty * kTile;
        int px_i[2], py_i[2];
        bool inside[2];
        float T[2], A[2], err[2], eps_max[2], z_first[2], z_last[2], dead[2];
        f32x2 crg[2], cbd[2], o2x[2], o2y[2];
        int nc[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int lx = (blk[q] & 1) * 8 + (lane & 7), ly = (blk[q] >> 1) * 4 + (lane >> 3);
            px_i[q] = tx * kTile + lx;
            py_i[q] = ty * kTile + ly;
            inside[q] = px_i[q] < b.width && py_i[q] < b.height;
            const float oxf = (float)lx - 7.5f, oyf = (float)ly - 7.5f;
            o2x[q] = pack2(oxf, oxf);
            o2y[q] = pack2(oyf, oyf);
            T[q] = 1.0f;
            A[q] = err[q] = eps_max[q] = z_last[q] = 0.0f;
            z_first[q] = 3.0e38f;
            crg[q] = cbd[q] = 0ull;
            nc[q] = 0;
            dead[q] = (!inside[q] || b.force_exact) ? INFINITY : 0.0f;
        }
        uint32_t loaded = 0;
        while (true) {
            if (__syncthreads_count(dead[0] == 0.0f || dead[1] == 0.0f) == 0) break;  // guards s_f reuse
            const int n = (int)min((uint32_t)kBatch, s1 - cursor);
            if (n <= 0) break;
            loaded += n;
#pragma unroll
            for (int r = 0; r < kPerT; ++r) {
                const int jt = threadIdx.x + r * kLT;
                if (jt >= n) break;
                const uint32_t rid = __ldg(v.pair_vals + cursor + jt);
                const GatheredSplat gs = gather_splat(v.geo, v.recs, rid);
                FRec1 f;
                const unsigned msk = tile_entry_8x4(gs.e1x, gs.e1y, gs.p1, gs.p2, gs.gl, gs.gr, x0 + 8.0, y0 + 8.0, f);
                if (msk) s_f[jt] = f;
                s_slot[jt] = rid;
                s_mask[jt] = (uint8_t)msk;
            }
            __syncthreads();
            int cnt[2] = {0, 0};
            for (int j0 = 0; j0 < n; j0 += 32) {
                const unsigned mk = j0 + lane < n ? s_mask[j0 + lane] : 0u;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const bool mine = (mk >> blk[q]) & 1u;
                    const unsigned bal = __ballot_sync(kFull, mine);
                    if (mine) s_wl[warp][q][cnt[q] + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)(j0 + lane);
                    cnt[q] += __popc(bal);
                }
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint16_t *wl = s_wl[warp][q];
                if (cnt[q] > 0) z_first[q] = fminf(z_first[q], s_f[wl[0]].z);
                const double px = px_i[q] + 0.5, py = py_i[q] + 0.5;
                float Tq = T[q], Aq = A[q], errq = err[q], em = eps_max[q], zl = z_last[q], dq = dead[q];
                f32x2 crgq = crg[q], cbdq = cbd[q];
                int ncq = nc[q];
                for (int k0 = 0; k0 < cnt[q] && !__all_sync(kFull, dq != 0.0f); k0 += 32) {
                    const int k1 = min(cnt[q], k0 + 32);
#pragma unroll kLp2Unroll
                    for (int k = k0; k < k1; ++k) {
                        const int j = wl[k];
                        const FRec1 &sr = s_f[j];
                        const float4 q0 = *reinterpret_cast<const float4 *>(&sr.a1x);
                        const float4 q1 = *reinterpret_cast<const float4 *>(&sr.V1);
                        float v1, v2;
                        unpack2(fma2(pack2(q0.x, q0.y), o2x[q], fma2(pack2(q0.z, q0.w), o2y[q], pack2(q1.x, q1.y))), v1,
                                v2);
                        float d2 = __fmaf_rn(v1, v1, __fmaf_rn(v2, v2, dq));
                        if (d2 > q1.z) continue;
                        const float4 q2 = *reinterpret_cast<const float4 *>(&sr.ka);
                        float eps;
                        if (d2 < q1.w) {
                            eps = __fmaf_rn(d2, q2.x, q2.y);
                        } else {  // boundary band: the reference's float64 test (_kernels_cy.pyx:73-75)
                            const SplatRec &sd = v.recs[s_slot[j]];
                            const double ddx = sd.mx - px, ddy = sd.my - py;
                            const double d2d = (sd.ca * ddx * ddx + sd.cb2 * ddx * ddy) + sd.cc * ddy * ddy;
                            if (d2d > kSupportD2) continue;
                            d2 = (float)(d2d * kHalfLog2e);
                            eps = kEpsExact;
                        }
                        const float e = ex2_approx(-d2);
                        const float a = fminf(q2.z * e, 0.99f);
                        const float w = a * Tq;
                        const float Tn = __fmaf_rn(-a, Tq, Tq);
                        const float4 q3 = *reinterpret_cast<const float4 *>(&sr.r);
                        crgq = fma2(pack2(q3.x, q3.y), pack2(w, w), crgq);
                        cbdq = fma2(pack2(q3.z, q3.w), pack2(w, w), cbdq);
                        Aq = Aq + w;
                        errq = __fmaf_rn(-a, errq, __fmaf_rn(w, eps, __fmaf_rn(Tn, kU125, errq)));
                        Tq = Tn;
                        ++ncq;
                        em = fmaxf(em, eps);
                        zl = fmaxf(zl, q3.w);
                        if (Tn - errq <= kTHi) dq = INFINITY;
                    }
                }
                T[q] = Tq;
                A[q] = Aq;
                err[q] = errq;
                eps_max[q] = em;
                z_last[q] = zl;
                dead[q] = dq;
                crg[q] = crgq;
                cbd[q] = cbdq;
                nc[q] = ncq;
            }
            cursor += n;
        }
        if (b.loads && threadIdx.x == 0 && loaded) atomicAdd(b.loads, (unsigned long long)loaded);
        const sn_camera &cam = b.cams[env];
#pragma unroll
        for (int q = 0; q < 2; ++q) {  // blend_kernel_px1's MODE 2 epilogue, per block
            float cr, cg, cb, D;
            unpack2(crg[q], cr, cg);
            unpack2(cbd[q], cb, D);
            const float Tq = T[q], errq = err[q], Aq = A[q];
            const bool cut = Tq - errq <= kTHi;
            const bool amb = inside[q] && (b.force_exact || (cut && (!(Tq + errq < kTLo) || errq > 0.0625f * Tq)));
            const int64_t pix = ((int64_t)env * b.height + py_i[q]) * b.width + px_i[q];
            const uint32_t code = (uint32_t)(((int64_t)el * b.height + py_i[q]) * b.width + px_i[q]);
            const float zf = nc[q] == 0 ? 3.0e38f : z_first[q];
            const float rho_w = errq / Tq + eps_max[q] + 6.0e-8f;
            const float alpha = fminf(Aq, 1.0f);
            const float depth = Aq > 0.0f ? D / Aq : (float)cam.far_;
            const float d_err = 1.01f * (rho_w * (z_last[q] - zf) + (float)(2 * nc[q] + 2) * 6.0e-8f * depth);
            const bool flag = inside[q] && amb;
            if (b.contribs) {
                const unsigned sum = __reduce_add_sync(kFull, flag ? 0u : (unsigned)nc[q]);
                if (lane == 0 && sum) atomicAdd(b.contribs, (unsigned long long)sum);
            }
            push_fixup(b, flag, code);
            if (!inside[q]) continue;
            if (flag) {
                b.ldepth[pix] = __int_as_float(0x7fc00000);  // NaN: pending float64 fixup
                continue;
            }
            if (b.contrib) b.contrib[pix] = nc[q];
            float fc0 = 0.0f, fc1 = 0.0f, fc2 = 0.0f;
            if (Aq > 0.0f) {
                fc0 = np_clipf(cr / Aq, 0.0f, 1.0f);
                fc1 = np_clipf(cg / Aq, 0.0f, 1.0f);
                fc2 = np_clipf(cb / Aq, 0.0f, 1.0f);
            }
            float *lc = b.lcolor + 3 * pix;
            lc[0] = fc0;
            lc[1] = fc1;
            lc[2] = fc2;
            b.lalpha[pix] = alpha;
            b.ldepth[pix] = depth;
            b.lderr[pix] = d_err;
            b.laerr[pix] = 1.01f * (rho_w + (float)(nc[q] + 1) * 6.0e-8f) * Aq + 6.0e-8f;
        }
        __syncthreads();  // the next tile reuses the shared buffers
    }
}

// composite(front = avatar layer, back = scene frame), renderer.py:151-166, for the layer frame the
// mode-2 blend left in its buffers. Decisions (front.depth < back.depth, alpha >= 0.5) are taken
// only when the tracked float32 error bounds separate them; other pixels join the fixup list and
// fixup_kernel<2> recomputes both layers in float64 and composites exactly.
__device__ __forceinline__ void composite_tile(const BlendArgs &b, const int tile, const int el) {
    const int env = b.e0 + el;
    const int tx = tile % b.tiles_x, ty = tile / b.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px_i = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py_i = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = px_i < b.width && py_i < b.height;
    const int64_t pix = ((int64_t)env * b.height + py_i) * b.width + px_i;
    bool flag = false, use_front = false;
    float ld = 0.0f, la = 0.0f, bd = 0.0f;
    if (inside) {
        ld = b.ldepth[pix];
        la = b.lalpha[pix];
        // pending fixup (NaN), or no contribution (front depth = far never wins)
        if (ld == ld && la > 0.0f) {
            bd = b.depth[pix];
            if (fabsf(ld - bd) <= 1.01f * (b.lderr[pix] + b.derr[pix]) + 1e-30f)
                flag = true;
            else if (ld < bd) {
                use_front = true;
                if (fabsf(la - 0.5f) <= b.laerr[pix]) flag = true;
            }
        }
    }
    push_fixup(b, flag, (uint32_t)(((int64_t)el * b.height + py_i) * b.width + px_i));
    if (!use_front || flag) return;
    const float *lc = b.lcolor + 3 * pix;
    float *oc = b.color + 3 * pix;
    const float o0 = __fmaf_rn(lc[0], la, oc[0] * (1.0f - la));
    const float o1 = __fmaf_rn(lc[1], la, oc[1] * (1.0f - la));
    const float o2 = __fmaf_rn(lc[2], la, oc[2] * (1.0f - la));
    oc[0] = o0;
    oc[1] = o1;
    oc[2] = o2;
    b.alpha[pix] = __fmaf_rn(b.alpha[pix], 1.0f - la, la);
    if (la >= 0.5f) b.depth[pix] = ld;
    store_payload(b, pix, o0, o1, o2, la >= 0.5f ? ld : bd);
}

__global__ void __launch_bounds__(kBlock) composite_kernel(BlendArgs b) {
    if (pass_overflow(b.pv) || pass_overflow(b.back) || far_overflow(b.back)) return;
    if (b.pv.source == 1 && b.pv.tile_list) {  // listed: only the tiles that hold layer splats
        const uint32_t n_items = *b.pv.n_list;
        for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
            const uint32_t key = b.pv.tile_list[item];
            composite_tile(b, (int)(key & ((1u << b.pv.tile_bits) - 1u)), (int)(key >> b.pv.tile_bits));
        }
        return;
    }
    const int tile = blockIdx.x, el = blockIdx.y;
    if (!b.tile_flag[(int64_t)el * gridDim.x + tile]) return;
    composite_tile(b, tile, el);
}

// ---- exact (float64) per-pixel walk: the fixup path ----

// One group's transmittances. Fast mode: a warp prefix product (Hillis-Steele, its association
// differs from the sequential product's by a few ulps). SEQ mode: lane l multiplies T by
// (1 - a_j) for j < l itself, in order -- the reference's sequential product (_kernels_cy.pyx:86),
// bit for bit. Returns T before this lane's contribution; t_after = before * (1 - a).
template <bool SEQ>
__device__ __forceinline__ double group_trans_before(double T, double one_minus_a, const QEntry *q, int lane,
                                                     bool act) {
    double before = T;
    if (SEQ) {
        for (int j = 0; j < lane; ++j) before *= 1.0 - q[j].a;  // q[j], j < lane, are active entries
    } else {
        double pp = act ? one_minus_a : 1.0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double o = __shfl_up_sync(kFull, pp, d);
            if (lane >= d) pp *= o;
        }
        double ex = __shfl_up_sync(kFull, pp, 1);
        if (lane == 0) ex = 1.0;
        before = T * ex;
    }
    return before;
}

// exp(-d2 / 2) of a contribution: the table exp (2 ulp), or in SEQ mode the device libm exp (1 ulp)
// on the reference's own argument -0.5 * d2
template <bool SEQ>
__device__ __forceinline__ double exp_neg_half(double d2, const double *s_exp) {
    double ev;
    if (SEQ) {
        ev = exp(-0.5 * d2);
    } else {
        SN_EXP_NEG_HALF(d2, s_exp, ev);
    }
    return ev;
}

// One pixel of one pass, walked by a whole warp with the reference's float64 arithmetic
// (_kernels_cy.pyx:64-86: float64 d2 / alpha / transmittance, T tested after each contribution).
// Lanes gather and test 32 depth-ordered candidates at a time; the contributing ones are queued
// (in order) and consumed 32 at a time: the transmittance through a group is a warp prefix
// product (its rounding differs from the sequential product by a few float64 ulps, like the table
// exp), the first member that takes T below 1e-4 is the last contribution, and the accumulators are
// per-lane partial sums reduced at the end. Groups are the 1st..32nd, 33rd..64th, ... contributions,
// so the result depends only on the contribution sequence -- not on how candidates were listed
// (streamed rectangles, tile lists or every splat of the env give bit-identical pixels). When a
// cutoff test meets a transmittance within kNearCut of 1e-4 the walk reports `near` and the caller
// re-walks the pixel with SEQ = true: sequential transmittance and libm exp, the reference's order.
template <int kPer, bool SEQ = false>  // candidates per lane per step: their gathers are in flight together
__device__ ExactPixel exact_walk(const PassView &v, int el, int tile, int tiles_x, int px_i, int py_i,
                                 const double *s_exp, QEntry *q) {
    const int lane = threadIdx.x & 31;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const double px = px_i + 0.5, py = py_i + 0.5;
    float cr = 0.0f, cg = 0.0f, cb = 0.0f;  // per-lane partial sums, reduced at the end
    double A = 0.0, D = 0.0, T = 1.0;
    int nc = 0, qn = 0;
    bool done = false, near = false, out = false;
    auto consume = [&](int m) {  // the first m <= 32 queued contributions
        const bool act = lane < m;
        QEntry e{};
        if (act) e = q[lane];
        const double before = group_trans_before<SEQ>(T, 1.0 - e.a, q, lane, act);
        const double t_after = before * (1.0 - e.a);
        if (!SEQ && __any_sync(kFull, act && fabs(t_after - kTCutoff) <= kNearCut * kTCutoff)) near = true;
        const unsigned cut = __ballot_sync(kFull, act && t_after < kTCutoff);
        const int last = cut ? __ffs(cut) - 1 : m - 1;
        if (act && lane <= last) {
            const double w = e.a * before;
            const float wf = (float)w;
            cr = __fmaf_rn(e.r, wf, cr);
            cg = __fmaf_rn(e.g, wf, cg);
            cb = __fmaf_rn(e.b, wf, cb);
            A = A + w;
            D = fma(e.z, w, D);
            ++nc;
        }
        T = __shfl_sync(kFull, t_after, last);
        if (cut) done = true;
    };
    uint32_t cur, end;
    if (v.source == 1) {
        uint2 r = v.ranges[((uint32_t)el << v.tile_bits) | (uint32_t)tile];
        cur = r.x;
        end = r.y;
    } else {
        cur = (uint32_t)v.env_off[el];
        end = (uint32_t)v.env_off[el + 1];
    }
    // two segments: the pass's own list, then -- a depth-sliced pass's unfinished tile -- its far
    // bucket (every far z is beyond every near one: the concatenation is the tile's depth order)
    for (int sgm = 0; sgm < 2; ++sgm) {
    const bool far = sgm == 1;
    if (far) {
        if (!v.sliced || done || near) break;
        if (v.far_phase == 1) {  // first fixup pass: the buckets come later -- defer (if there is a far half)
            out = v.env_off[v.ec + el + 1] > v.env_off[v.ec + el];
            break;
        }
        const int32_t ub = v.far_bucket_of[(int64_t)el * v.n_tiles + tile];
        if (ub < 0) {  // unregistered: the env has no far splats, or the tile stopped inside its near list
            if (lane == 0 && v.env_off[v.ec + el + 1] > v.env_off[v.ec + el]) atomicExch(v.far_short, 1ull);
            break;
        }
        cur = v.far_ranges[ub].x;
        end = v.far_ranges[ub].y;
    }
    while (cur < end && !done && !near) {
        uint32_t step;
        uint32_t rid[kPer];
        bool cand[kPer];
        if (!far && v.source == 0) {
            const uint32_t bi = cur / kBlock;
            if (cur % kBlock == 0 || !covers(__ldg(v.batch_rects + bi), tx, ty)) {
                // find the next 256-splat batch whose union rectangle covers the tile, 32 batches
                // per step (the lanes test them in parallel)
                const uint32_t nb = (end + kBlock - 1) / kBlock;
                const uint32_t cand_b = bi + lane;
                const unsigned hit = __ballot_sync(kFull, cand_b < nb && covers(__ldg(v.batch_rects + cand_b), tx, ty));
                if (!hit) {
                    cur = min(end, (bi + 32) * (uint32_t)kBlock);
                    continue;
                }
                const uint32_t first = bi + __ffs(hit) - 1;
                if (first != bi) {
                    cur = first * (uint32_t)kBlock;
                    continue;
                }
            }
            const uint32_t b_end = min(end, (bi + 1) * (uint32_t)kBlock);
            step = min(32u * kPer, b_end - cur);
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                rid[i] = cur + 32 * i + lane;
                cand[i] = rid[i] < cur + step && covers(__ldg(v.rects + rid[i]), tx, ty);
            }
        } else {
            step = min(32u * kPer, end - cur);
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const uint32_t k = cur + 32 * i + lane;
                cand[i] = k < cur + step;
                rid[i] = cand[i] ? (far ? __ldg(v.far_order + k) : v.source == 1 ? __ldg(v.pair_vals + k) : k) : 0u;
            }
        }
        QEntry e[kPer];
        bool contrib[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            contrib[i] = false;
            e[i] = QEntry{};
            if (cand[i]) {
                const SplatRec &s = far ? v.far_recs[rid[i]] : v.recs[v.source == 1 ? rid[i] : __ldg(v.order + rid[i])];
                const double dx = s.mx - px, dy = s.my - py;
                const double d2 = (s.ca * dx * dx + s.cb2 * dx * dy) + s.cc * dy * dy;
                if (!(d2 > kSupportD2)) {
                    contrib[i] = true;
                    e[i].a = s.alpha * exp_neg_half<SEQ>(d2, s_exp);
                    if (e[i].a > kAlphaClip) e[i].a = kAlphaClip;
                    e[i].z = s.z;
                    float rgb[3];
                    unpack_rgb21(s.rgb, rgb);
                    e[i].r = rgb[0];
                    e[i].g = rgb[1];
                    e[i].b = rgb[2];
                }
            }
        }
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            if (done || near) break;
            const unsigned bal = __ballot_sync(kFull, contrib[i]);
            if (contrib[i]) q[qn + __popc(bal & ((1u << lane) - 1u))] = e[i];
            qn += __popc(bal);
            __syncwarp();
            if (qn >= 32) {
                consume(32);
                QEntry rest{};
                const bool mv = lane < qn - 32;
                if (mv) rest = q[32 + lane];
                __syncwarp();
                if (mv) q[lane] = rest;
                __syncwarp();
                qn -= 32;
            }
        }
        cur += step;
    }
    }
    if (!done && !near && qn > 0) consume(qn);
    __syncwarp();
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        cr += __shfl_xor_sync(kFull, cr, d);
        cg += __shfl_xor_sync(kFull, cg, d);
        cb += __shfl_xor_sync(kFull, cb, d);
        A += __shfl_xor_sync(kFull, A, d);
        D += __shfl_xor_sync(kFull, D, d);
    }
    if (v.sliced && (g_slice_hooks & 1) && lane == 0) atomicExch(v.far_short, 1ull);
    return ExactPixel{cr, cg, cb, A, D, T, (int)__reduce_add_sync(kFull, (unsigned)nc), near, out};
}

// exact_walk, then -- only when its cutoff test met a transmittance within kNearCut of 1e-4 -- the
// same pixel again in SEQ mode (sequential transmittance, libm exp): the reference's decision.
template <int kPer>
__device__ __forceinline__ ExactPixel exact_pixel(const PassView &v, int el, int tile, int tiles_x, int px_i, int py_i,
                                                  const double *s_exp, QEntry *q) {
    ExactPixel f = exact_walk<kPer, false>(v, el, tile, tiles_x, px_i, py_i, s_exp, q);
    if (f.near) {
        __syncwarp();
        f = exact_walk<kPer, true>(v, el, tile, tiles_x, px_i, py_i, s_exp, q);
        f.near = true;
    }
    return f;
}

// exact_walk for one pixel by a whole CTA (long, unsaturated lists: avatar-layer fixups). The 8
// warps gather and evaluate up to 1,024 candidates per step (256 per step on the streamed-rectangle
// source), the contributions are compacted in candidate order into a shared queue, and warp 0
// consumes them 32 at a time exactly as exact_walk does -- same groups, bit-identical result.
// Returns the reduced pixel in warp 0 (other warps' return values are unspecified).
#ifndef SN_FIXUP_CTA_PER
#define SN_FIXUP_CTA_PER 4
#endif
constexpr int kCtaPer = SN_FIXUP_CTA_PER;
constexpr int kCtaQueue = kCtaPer * kBlock + 32;
template <bool SEQ>
__device__ ExactPixel exact_walk_cta(const PassView &v, int el, int tile, int tiles_x, int px_i, int py_i,
                                     const double *s_exp, QEntry *q, int *s_i) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const double px = px_i + 0.5, py = py_i + 0.5;
    float cr = 0.0f, cg = 0.0f, cb = 0.0f;
    double A = 0.0, D = 0.0, T = 1.0;
    int nc = 0;
    bool done = false, near = false;  // warp 0's view
    int qn = 0;         // queued contributions (uniform)
    auto consume = [&](int head, int m) {  // warp 0: q[head, head + m), m <= 32
        const bool act = lane < m;
        QEntry e{};
        if (act) e = q[head + lane];
        const double before = group_trans_before<SEQ>(T, 1.0 - e.a, q + head, lane, act);
        const double t_after = before * (1.0 - e.a);
        if (!SEQ && __any_sync(kFull, act && fabs(t_after - kTCutoff) <= kNearCut * kTCutoff)) near = true;
        const unsigned cut = __ballot_sync(kFull, act && t_after < kTCutoff);
        const int last = cut ? __ffs(cut) - 1 : m - 1;
        if (act && lane <= last) {
            const double w = e.a * before;
            const float wf = (float)w;
            cr = __fmaf_rn(e.r, wf, cr);
            cg = __fmaf_rn(e.g, wf, cg);
            cb = __fmaf_rn(e.b, wf, cb);
            A = A + w;
            D = fma(e.z, w, D);
            ++nc;
        }
        T = __shfl_sync(kFull, t_after, last);
        if (cut) done = true;
    };
    uint32_t cur, end;
    if (v.source == 1) {
        uint2 r = v.ranges[((uint32_t)el << v.tile_bits) | (uint32_t)tile];
        cur = r.x;
        end = r.y;
    } else {
        cur = (uint32_t)v.env_off[el];
        end = (uint32_t)v.env_off[el + 1];
    }
    int *s_cnt = s_i;           // [8] per-warp counts
    int *s_flag = s_i + 8;      // [0] done, [1] next cursor (source 0 batch search)
    if (threadIdx.x == 0) s_flag[0] = 0;
    __syncthreads();
    // two segments: the pass's own list, then a depth-sliced pass's far bucket (see exact_walk)
    for (int sgm = 0; sgm < 2; ++sgm) {
    const bool far = sgm == 1;
    if (far) {
        if (!v.sliced || s_flag[0]) break;  // s_flag[0]: the walk already stopped (uniform)
        const int32_t ub = v.far_bucket_of[(int64_t)el * v.n_tiles + tile];
        if (ub < 0) {  // as in exact_walk
            if (threadIdx.x == 0 && v.env_off[v.ec + el + 1] > v.env_off[v.ec + el]) atomicExch(v.far_short, 1ull);
            break;
        }
        cur = v.far_ranges[ub].x;
        end = v.far_ranges[ub].y;
    }
    while (cur < end) {
        uint32_t step;
        int per;
        if (!far && v.source == 0) {  // one 256-splat batch per step; warp 0 finds the next covering batch
            if (warp == 0) {
                uint32_t c = cur;
                while (c < end) {
                    const uint32_t bi = c / kBlock;
                    const uint32_t nb = (end + kBlock - 1) / kBlock;
                    const unsigned hit =
                        __ballot_sync(kFull, bi + lane < nb && covers(__ldg(v.batch_rects + bi + lane), tx, ty));
                    if (hit) {
                        c = max(c, (bi + __ffs(hit) - 1) * (uint32_t)kBlock);
                        break;
                    }
                    c = min(end, (bi + 32) * (uint32_t)kBlock);
                }
                if (lane == 0) s_flag[1] = (int)c;
            }
            __syncthreads();
            cur = (uint32_t)s_flag[1];
            if (cur >= end) break;
            step = min((uint32_t)kBlock - cur % kBlock, end - cur);
            per = 1;
        } else {
            step = min((uint32_t)(kCtaPer * kBlock), end - cur);
            per = kCtaPer;
        }
        for (int i = 0; i < per; ++i) {
            const uint32_t k = cur + (uint32_t)(i * kBlock) + threadIdx.x;
            bool contrib = false;
            QEntry e{};
            if (k < cur + step) {
                uint32_t rid = k;
                bool cand = true;
                if (far) rid = __ldg(v.far_order + k);
                else if (v.source == 0) cand = covers(__ldg(v.rects + k), tx, ty);
                else if (v.source == 1) rid = __ldg(v.pair_vals + k);
                if (cand) {
                    const SplatRec &sr = far ? v.far_recs[rid] : v.recs[v.source == 1 ? rid : __ldg(v.order + rid)];
                    const double dx = sr.mx - px, dy = sr.my - py;
                    const double d2 = (sr.ca * dx * dx + sr.cb2 * dx * dy) + sr.cc * dy * dy;
                    if (!(d2 > kSupportD2)) {
                        contrib = true;
                        e.a = sr.alpha * exp_neg_half<SEQ>(d2, s_exp);
                        if (e.a > kAlphaClip) e.a = kAlphaClip;
                        e.z = sr.z;
                        float rgb[3];
                        unpack_rgb21(sr.rgb, rgb);
                        e.r = rgb[0];
                        e.g = rgb[1];
                        e.b = rgb[2];
                    }
                }
            }
            const unsigned bal = __ballot_sync(kFull, contrib);
            if (lane == 0) s_cnt[warp] = __popc(bal);
            __syncthreads();
            int off = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kBlock / 32; ++w) {
                const int c = s_cnt[w];
                off += w < warp ? c : 0;
                tot += c;
            }
            if (contrib) q[qn + off + __popc(bal & ((1u << lane) - 1u))] = e;
            qn += tot;
            __syncthreads();
        }
        // warp 0 consumes whole groups of 32; the remainder moves to the queue's front
        if (warp == 0) {
            int head = 0;
            while (!done && !near && qn - head >= 32) {
                consume(head, 32);
                head += 32;
            }
            const int rest = (done || near) ? 0 : qn - head;
            QEntry t{};
            if (lane < rest) t = q[head + lane];
            __syncwarp();
            if (lane < rest) q[lane] = t;
            if (lane == 0) {
                s_flag[0] = done || near;
                s_cnt[0] = rest;
            }
        }
        __syncthreads();
        qn = s_cnt[0];
        const bool stop = s_flag[0] != 0;
        __syncthreads();
        if (stop) break;
        cur += step;
    }
    }
    if (warp == 0) {
        if (!done && !near && qn > 0) consume(0, qn);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            cr += __shfl_xor_sync(kFull, cr, d);
            cg += __shfl_xor_sync(kFull, cg, d);
            cb += __shfl_xor_sync(kFull, cb, d);
            A += __shfl_xor_sync(kFull, A, d);
            D += __shfl_xor_sync(kFull, D, d);
        }
        nc = (int)__reduce_add_sync(kFull, (unsigned)nc);
        if (lane == 0) s_flag[2] = near;
    }
    __syncthreads();  // the queue and scratch are reused by the next walk
    near = s_flag[2] != 0;  // uniform across the CTA
    __syncthreads();
    return ExactPixel{cr, cg, cb, A, D, T, nc, near};
}

// exact_walk_cta, re-walked in SEQ mode when the cutoff met a transmittance within kNearCut of 1e-4.
__device__ __forceinline__ ExactPixel exact_pixel_cta(const PassView &v, int el, int tile, int tiles_x, int px_i,
                                                      int py_i, const double *s_exp, QEntry *q, int *s_i) {
    ExactPixel f = exact_walk_cta<false>(v, el, tile, tiles_x, px_i, py_i, s_exp, q, s_i);
    if (f.near) {
        f = exact_walk_cta<true>(v, el, tile, tiles_x, px_i, py_i, s_exp, q, s_i);
        f.near = true;
    }
    return f;
}

// Layer fixups (mode 2): a CTA per listed pixel (their walks are long: near avatars' tile lists
// run to tens of thousands of pairs and rarely saturate).
__global__ void __launch_bounds__(256) fixup_layer_kernel(BlendArgs b) {
    __shared__ double s_exp[64];
    __shared__ QEntry s_q[kCtaQueue];
    __shared__ int s_i[16];
    __shared__ int s_back;
    if (threadIdx.x < 64) s_exp[threadIdx.x] = kExp2Tbl[threadIdx.x];
    __syncthreads();
    if (pass_overflow(b.pv) || pass_overflow(b.back) || far_overflow(b.back)) return;
    const unsigned n_fix = *b.fix_count;
    const unsigned hw = (unsigned)b.width * (unsigned)b.height;
    unsigned long long contribs = 0;
    for (unsigned i = blockIdx.x; i < n_fix; i += gridDim.x) {
        const uint32_t code = b.fix_list[i];
        const int el = (int)(code / hw), p = (int)(code % hw);
        const int py_i = p / b.width, px_i = p % b.width;
        const int env = b.e0 + el;
        const int tile = (py_i / kTile) * b.tiles_x + px_i / kTile;
        const sn_camera &cam = b.cams[env];
        const ExactPixel f = exact_pixel_cta(b.pv, el, tile, b.tiles_x, px_i, py_i, s_exp, s_q, s_i);
        const int64_t pix = ((int64_t)env * b.height + py_i) * b.width + px_i;
        const double alpha = f.A < 1.0 ? f.A : 1.0;
        const double depth = f.A > 0.0 ? f.D / f.A : cam.far_;
        if (threadIdx.x == 0) {
            contribs += (unsigned)f.nc;
            if (b.contrib) b.contrib[pix] = f.nc;
            // the back depth in the frame is within derr of the float64 value: recompute the scene
            // pixel only when the exact front depth falls inside that band
            s_back = f.A > 0.0 && fabs(depth - (double)b.depth[pix]) <= 1.01 * (double)b.derr[pix] + 1e-30;
        }
        __syncthreads();
        const bool exact_back = s_back != 0;
        __syncthreads();
        ExactPixel k{};
        if (exact_back) k = exact_pixel_cta(b.back, el, tile, b.tiles_x, px_i, py_i, s_exp, s_q, s_i);
        if (threadIdx.x != 0 || !(f.A > 0.0)) continue;  // front depth = far: the back is kept
        float *oc = b.color + 3 * pix;
        float bc[3] = {oc[0], oc[1], oc[2]};
        float ba = b.alpha[pix];
        double bd = (double)b.depth[pix];
        if (exact_back) {  // the scene frame exactly as the scene pass stores it (float32)
            bc[0] = (float)np_clip((double)k.cr + cam.background[0] * k.T, 0.0, 1.0);
            bc[1] = (float)np_clip((double)k.cg + cam.background[1] * k.T, 0.0, 1.0);
            bc[2] = (float)np_clip((double)k.cb + cam.background[2] * k.T, 0.0, 1.0);
            ba = (float)(k.A < 1.0 ? k.A : 1.0);
            bd = k.A > 0.0 ? k.D / k.A : cam.far_;
        }
        if (depth < bd) {  // composite, renderer.py:151-166
            const double fc[3] = {np_clip((double)f.cr / f.A, 0.0, 1.0), np_clip((double)f.cg / f.A, 0.0, 1.0),
                                  np_clip((double)f.cb / f.A, 0.0, 1.0)};
            for (int c = 0; c < 3; ++c) oc[c] = (float)(fc[c] * alpha + (double)bc[c] * (1.0 - alpha));
            b.alpha[pix] = (float)(alpha + (double)ba * (1.0 - alpha));
            b.depth[pix] = (float)(alpha >= 0.5 ? depth : bd);
            store_payload(b, pix, oc[0], oc[1], oc[2], b.depth[pix]);
        } else if (exact_back) {
            for (int c = 0; c < 3; ++c) oc[c] = bc[c];
            b.alpha[pix] = ba;
            b.depth[pix] = (float)bd;
            store_payload(b, pix, bc[0], bc[1], bc[2], (float)bd);
        }
    }
    if (b.contribs && threadIdx.x == 0 && contribs) atomicAdd(b.contribs, contribs);
}

// Recomputes the listed pixels exactly (warp per pixel, grid-stride over the device-side count)
// and writes the same outputs the float64 blend epilogue writes. Mode 2 also recomputes the scene
// pixel (the back layer) so the composite's comparisons see float64 depths.
// A scene pixel's float64 result into the frame (fixup_kernel<0> and the blend's in-CTA fixups).
__device__ __forceinline__ void write_exact_scene(const BlendArgs &b, const ExactPixel &f, int64_t pix,
                                                  const sn_camera &cam) {
    const double alpha = f.A < 1.0 ? f.A : 1.0;
    const double depth = f.A > 0.0 ? f.D / f.A : cam.far_;
    if (b.contrib) b.contrib[pix] = f.nc;
    float *oc = b.color + 3 * pix;
    oc[0] = (float)np_clip((double)f.cr + cam.background[0] * f.T, 0.0, 1.0);
    oc[1] = (float)np_clip((double)f.cg + cam.background[1] * f.T, 0.0, 1.0);
    oc[2] = (float)np_clip((double)f.cb + cam.background[2] * f.T, 0.0, 1.0);
    b.alpha[pix] = (float)alpha;
    b.depth[pix] = (float)depth;
    store_payload(b, pix, oc[0], oc[1], oc[2], (float)depth);
    // the stored depth is the float64 walk's rounded to float32 (and the walk's prefix-product
    // transmittance / table exp differ from the sequential reference by a few float64 ulps):
    // a band of ~2 float ulps makes a layer fixup whose exact front depth falls inside it
    // recompute this pixel in float64 (fixup_layer_kernel / fixup_kernel<2>)
    if (b.derr) b.derr[pix] = f.A > 0.0 ? (float)(2.5e-7 * fabs(depth)) : 0.0f;
}

// (sliced pass, far_phase 1) a float64 walk needs the tile's far bucket: register the tile if the
// blend did not (late: no saved state, the continuation skips it) and queue the pixel for the
// fixup pass after the buckets, which walks near list + bucket. Lane 0 acts.
__device__ __forceinline__ void defer_to_far(const BlendArgs &b, int el, int tile, uint32_t code) {
    if ((threadIdx.x & 31) != 0) return;
    int32_t *bo = b.bucket_of + (int64_t)el * b.pv.n_tiles + tile;
    if (atomicCAS(bo, -1, -2) == -1) {
        const unsigned long long u = atomicAdd(b.unfin_count, 1ull);
        if (u < b.pv.far_cap_u) {
            b.unfin_list[u] = kLateTile | ((uint32_t)el << 16) | (uint32_t)tile;
            atomicOr(b.unfin_envs, 1ull << el);
            atomicExch(bo, (int32_t)u);
        }  // (overflow: the render is re-run with more room)
    }
    const unsigned slot = atomicAdd(b.fix_count, 1u);
    SN_ASSERT(slot < 2u * (unsigned)b.ec * (unsigned)b.width * (unsigned)b.height);
    b.fix_list[slot] = code;
}

template <int MODE>
__global__ void __launch_bounds__(256, SN_FIXUP_MIN_BLOCKS) fixup_kernel(BlendArgs b) {
    __shared__ double s_exp[64];
    __shared__ QEntry s_q[8][kQueue];
    if (threadIdx.x < 64) s_exp[threadIdx.x] = kExp2Tbl[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    QEntry *q = s_q[threadIdx.x >> 5];
    if (pass_overflow(b.pv) || far_overflow(b.pv) || (MODE == 2 && (pass_overflow(b.back) || far_overflow(b.back))))
        return;
    const unsigned n_fix = *b.fix_count, i0 = b.fix_start ? *b.fix_start : 0u;
    const unsigned hw = (unsigned)b.width * (unsigned)b.height;
    unsigned long long contribs = 0;
    for (unsigned i = i0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < n_fix;
         i += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t code = b.fix_list[i];
        const int el = (int)(code / hw), p = (int)(code % hw);
        const int py_i = p / b.width, px_i = p % b.width;
        const int env = b.e0 + el;
        const int tile = (py_i / kTile) * b.tiles_x + px_i / kTile;
        const sn_camera &cam = b.cams[env];
        // mode 2 fixups are few and each walks long, unsaturated lists: more gathers in flight
        const ExactPixel f = exact_pixel<MODE == 2 ? 8 : SN_FIXUP_PER>(b.pv, el, tile, b.tiles_x, px_i, py_i, s_exp, q);
        if (MODE != 2 && f.out) {
            defer_to_far(b, el, tile, code);
            continue;
        }
        contribs += (unsigned)f.nc;
        const int64_t pix = ((int64_t)env * b.height + py_i) * b.width + px_i;
        const double alpha = f.A < 1.0 ? f.A : 1.0;
        const double depth = f.A > 0.0 ? f.D / f.A : cam.far_;
        if (MODE == 2) {
            // composite(front = this layer, back = the scene frame), renderer.py:151-166. The back
            // depth in the frame is within derr of the float64 value: only when the exact front
            // depth falls inside that band is the scene pixel recomputed in float64 as well.
            if (lane == 0 && b.contrib) b.contrib[pix] = f.nc;
            if (!(f.A > 0.0)) continue;  // front depth = far: the back is kept
            double bd = (double)b.depth[pix];
            bool exact_back = false;
            ExactPixel k{};
            if (fabs(depth - bd) <= 1.01 * (double)b.derr[pix] + 1e-30) {
                k = exact_pixel<4>(b.back, el, tile, b.tiles_x, px_i, py_i, s_exp, q);
                bd = k.A > 0.0 ? k.D / k.A : cam.far_;
                exact_back = true;
            }
            if (lane != 0) continue;
            float *oc = b.color + 3 * pix;
            float bc[3] = {oc[0], oc[1], oc[2]};
            float ba = b.alpha[pix];
            if (exact_back) {  // the scene frame exactly as the scene pass stores it (float32)
                bc[0] = (float)np_clip((double)k.cr + cam.background[0] * k.T, 0.0, 1.0);
                bc[1] = (float)np_clip((double)k.cg + cam.background[1] * k.T, 0.0, 1.0);
                bc[2] = (float)np_clip((double)k.cb + cam.background[2] * k.T, 0.0, 1.0);
                ba = (float)(k.A < 1.0 ? k.A : 1.0);
            }
            if (depth < bd) {
                const double fc[3] = {np_clip((double)f.cr / f.A, 0.0, 1.0), np_clip((double)f.cg / f.A, 0.0, 1.0),
                                      np_clip((double)f.cb / f.A, 0.0, 1.0)};
                for (int c = 0; c < 3; ++c) oc[c] = (float)(fc[c] * alpha + (double)bc[c] * (1.0 - alpha));
                b.alpha[pix] = (float)(alpha + (double)ba * (1.0 - alpha));
                b.depth[pix] = (float)(alpha >= 0.5 ? depth : bd);
                store_payload(b, pix, oc[0], oc[1], oc[2], b.depth[pix]);
            } else if (exact_back) {
                for (int c = 0; c < 3; ++c) oc[c] = bc[c];
                b.alpha[pix] = ba;
                b.depth[pix] = (float)bd;
                store_payload(b, pix, bc[0], bc[1], bc[2], (float)bd);
            }
            continue;
        }
        if (lane != 0) continue;
        if (MODE == 0) {
            write_exact_scene(b, f, pix, cam);
            continue;
        }
        if (b.contrib) b.contrib[pix] = f.nc;
        float *oc = b.color + 3 * pix;
        double fc[3] = {0.0, 0.0, 0.0};
        if (f.A > 0.0) {
            fc[0] = np_clip((double)f.cr / f.A, 0.0, 1.0);
            fc[1] = np_clip((double)f.cg / f.A, 0.0, 1.0);
            fc[2] = np_clip((double)f.cb / f.A, 0.0, 1.0);
        }
        for (int c = 0; c < 3; ++c) oc[c] = (float)fc[c];
        b.alpha[pix] = (float)alpha;
        b.depth[pix] = (float)depth;
        store_payload(b, pix, oc[0], oc[1], oc[2], (float)depth);
    }
    if (b.contribs && lane == 0 && contribs) atomicAdd(b.contribs, contribs);
}

// Largest relative error of the blend's fast exp, ex2.approx(d2 * -log2(e) / 2) against float64
// exp(-d2 / 2), over every float d2 in [0, 9.5]: the kEpsExp budget assumes <= 3.5e-7.
__global__ void fast_exp_selftest_kernel(unsigned long long *max_err_bits) {
    const uint32_t lo = 0u, hi = __float_as_uint(9.5f);
    double worst = 0.0;
    for (uint32_t u = lo + blockIdx.x * blockDim.x + threadIdx.x; u <= hi; u += gridDim.x * blockDim.x) {
        const float d2 = __uint_as_float(u);
        const float e = ex2_approx(d2 * kNegHalfLog2e);
        const double ref = exp(-0.5 * (double)d2);
        worst = fmax(worst, fabs((double)e - ref) / ref);
    }
    atomicMax(max_err_bits, (unsigned long long)__double_as_longlong(worst));
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
static void launch_blend_mode(const BlendArgs &b, dim3 grid, cudaStream_t s, bool fixup) {
    if constexpr (MODE == 2) {  // the avatar layer: one pixel per thread (see blend_kernel_px1)
        if (b.pv.source == 0)
            blend_kernel_px1<MODE, 0><<<grid, kBlock, 0, s>>>(b);
        else if (b.pv.source == 1 && b.pv.tile_list && SN_LAYER_LP2)  // listed, two blocks per warp
            blend_kernel_lp2<<<148 * SN_LAYER_LP2_MIN_BLOCKS, kLT, 0, s>>>(b);
        else if (b.pv.source == 1 && b.pv.tile_list)  // listed: a few CTAs per SM take the non-empty tiles
            blend_kernel_px1<MODE, 1><<<148 * SN_LAYER_PX1_MIN_BLOCKS, kBlock, 0, s>>>(b);
        else if (b.pv.source == 1)
            blend_kernel_px1<MODE, 1><<<grid, kBlock, 0, s>>>(b);
        else
            blend_kernel_px1<MODE, 2><<<grid, kBlock, 0, s>>>(b);
    } else {
        if (b.pv.source == 0)
            blend_kernel<MODE, 0><<<grid, kBT, 0, s>>>(b);
        else if (b.pv.source == 1)
            blend_kernel<MODE, 1><<<grid, kBT, 0, s>>>(b);
        else
            blend_kernel<MODE, 2><<<grid, kBT, 0, s>>>(b);
        if (fixup) fixup_kernel<MODE><<<kFixupBlocks, 256, 0, s>>>(b);  // mode 2: after the composite
    }
}

cudaError_t launch_tile_queue(const PassView &v, int el, int n_tiles, int tiles_x, uint32_t *counts,
                              const uint64_t *offsets, uint32_t *out, cudaStream_t s) {
    tile_queue_kernel<<<n_tiles, kBlock, 0, s>>>(v, el, tiles_x, counts, offsets, out);
    return cudaGetLastError();
}

cudaError_t launch_layer_composite(const BlendArgs &b, cudaStream_t s) {
    if (b.pv.source == 1 && b.pv.tile_list) {
        composite_kernel<<<148 * 8, kBlock, 0, s>>>(b);
    } else {
        dim3 grid((unsigned)(tiles_of(b.width) * tiles_of(b.height)), (unsigned)b.ec);
        composite_kernel<<<grid, kBlock, 0, s>>>(b);
    }
    fixup_layer_kernel<<<kFixupBlocks, 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_blend(const BlendArgs &b, cudaStream_t s, bool fixup) {
    dim3 grid((unsigned)(tiles_of(b.width) * tiles_of(b.height)), (unsigned)b.ec);
    if (b.mode == 0)
        launch_blend_mode<0>(b, grid, s, fixup);
    else if (b.mode == 1)
        launch_blend_mode<1>(b, grid, s, fixup);
    else
        launch_blend_mode<2>(b, grid, s, fixup);
    return cudaGetLastError();
}

cudaError_t launch_continue(const BlendArgs &b, cudaStream_t s) {
    BlendArgs c = b;
    c.pv.source = 3;
    if (b.mode == 0)
        blend_kernel<0, 3><<<148 * SN_BLEND_MIN_BLOCKS, kBT, 0, s>>>(c);
    else if (b.mode == 1)
        blend_kernel<1, 3><<<148 * SN_BLEND_MIN_BLOCKS, kBT, 0, s>>>(c);
    return cudaGetLastError();
}

cudaError_t launch_fixup(const BlendArgs &b, cudaStream_t s) {
    if (b.mode == 0)
        fixup_kernel<0><<<kFixupBlocks, 256, 0, s>>>(b);
    else if (b.mode == 1)
        fixup_kernel<1><<<kFixupBlocks, 256, 0, s>>>(b);
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

cudaError_t fast_exp_selftest(double *max_rel_err) {
    unsigned long long *d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    cudaMemset(d, 0, sizeof(unsigned long long));
    fast_exp_selftest_kernel<<<1184, 256>>>(d);
    unsigned long long bits = 0;
    e = cudaMemcpy(&bits, d, sizeof(bits), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e == cudaSuccess) std::memcpy(max_rel_err, &bits, sizeof(double));
    return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace sn

// Test hooks (not part of the ABI) for the rare paths of a sliced pass, which the tests check give
// identical frames: bit 0 -- every float64 walk sets far_short as if it had run out of a near list
// with no bucket, so the render is re-run unsliced; bit 1 -- the blend does not register tiles for
// their undecided pixels alone, so those pixels' walks are deferred by the first fixup pass, which
// registers their tiles late.
extern "C" int sn_debug_slice_hooks(int bits) {
    return cudaMemcpyToSymbol(sn::g_slice_hooks, &bits, sizeof(int)) == cudaSuccess ? 0 : 1;
}

#ifdef SN_FIX_PROF
extern "C" int sn_debug_fix_prof(unsigned long long *out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_fix_prof, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_fix_prof, z, sizeof(z));
    }
    return 0;
}
#endif
#ifdef SN_BLEND_PROF
extern "C" int sn_debug_blend_prof(unsigned long long *out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_blend_prof, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_blend_prof, z, sizeof(z));
    }
    return 0;
}
extern "C" int sn_debug_env_frac(unsigned *out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_env_frac, sizeof(unsigned) * 64);
    if (reset) {
        unsigned z[64] = {};
        cudaMemcpyToSymbol(g_env_frac, z, sizeof(z));
    }
    return 0;
}
#endif
