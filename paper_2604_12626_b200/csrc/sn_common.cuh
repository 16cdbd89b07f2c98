// sn_common.cuh -- shared device code for the splat-observation kernels (sm_100a).
//
// Numerics contract: this file is compiled with -fmad=false, so no multiply-add is contracted
// implicitly. Every fma() below is deliberate: it restates an OpenBLAS FMA chain the reference's
// numpy matmuls run (projection.py:123,144-146, rig.py:116,123,130,132); every other product and
// sum rounds separately like a numpy ufunc. Geometry and the blend's decision chain are float64,
// so the visible set, depth order, tile rectangles and contributor counts are the reference's.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cstdio>

#include "../../include/splatnav_b200.h"

namespace sn {

// Device-side bounds checks of the build variant compiled with -DSN_CHECKS (the sanitizer tools are
// unavailable on the GPU pool): a failed check prints its location and traps the kernel, which
// surfaces as a CUDA error from the render. Compiled out otherwise.
#ifdef SN_CHECKS
#define SN_ASSERT(cond)                                                                               \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("SN_ASSERT failed: %s at %s:%d (block %d,%d thread %d)\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                               \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define SN_ASSERT(cond) ((void)0)
#endif

constexpr int kTile = 16;
constexpr int kBlock = 256;
constexpr int kMaxEnvChunk = 64;
constexpr int kMaxJoints = 64;

// projection.py:16-18, _kernels_cy.pyx:10-12
constexpr double kCovReg = 0.3;
constexpr double kSigma = 3.0;
constexpr double kDegDet = 1e-12;
constexpr double kTCutoff = 1e-4;
constexpr double kSupportD2 = 9.0;
constexpr double kAlphaClip = 0.99;

enum { kKeep = 0, kCullDepth = 1, kDegenerate = 2, kCullFrame = 3 };
// whole-avatar cull code (avatar_cull_kernel): every gaussian of the avatar is visible in the env
constexpr int kWholeVisible = 4;

// One depth-sorted splat as the blend reads it: 64 bytes, one gather of four 16-byte vectors.
// The decision chain (mean, conic, alpha) stays float64; colour is 3 x 21-bit unorm (error
// 2.4e-7, far inside the 2e-3 RGB budget); z is float64 for depth accumulation.
struct __align__(16) SplatRec {
    double mx, my;
    double ca, cb2, cc;  // conic (a, 2b, c): d2 = (ca*dx)*dx + (cb2*dx)*dy + (cc*dy)*dy
    double alpha;        // sigmoid(opacity)
    double z;
    unsigned long long rgb;
};
static_assert(sizeof(SplatRec) == 64, "SplatRec must stay 64 bytes");

// The blend's view of a splat, written next to its SplatRec by the emit stage (32 B): the conic's
// principal axes -- float64 major-axis direction e1 (e2 = (-e1y, e1x)) and the eigenvalues
// l1 >= l2 -- and the support ellipse's bounding-box half-extents. The blend reads the mean, alpha,
// z and colour from the SplatRec itself and forms p1 = e1.mean, p2 = e2.mean (blend_geo_p), so a
// tile only has to form e1.(centre - mean) in float64.
struct __align__(16) BlendGeo {
    double e1x, e1y;
    float l1, l2;          // l2 <= 0: degenerate -- the blend tests every pixel in float64
    float hx, hy;          // 3 sqrt(e1x^2 / l1 + e1y^2 / l2), 3 sqrt(e1y^2 / l1 + e1x^2 / l2)
};
static_assert(sizeof(BlendGeo) == 32, "BlendGeo must stay 32 bytes");

// p1 = e1.mean, p2 = e2.mean, rounded as products then sum (compiled with -fmad=false)
__device__ __forceinline__ void blend_geo_p(double e1x, double e1y, double mx, double my, double &p1, double &p2) {
    p1 = e1x * mx + e1y * my;
    p2 = e1x * my - e1y * mx;
}

__device__ __forceinline__ BlendGeo make_blend_geo(double ca, double cb2, double cc) {
    BlendGeo g;
    const double b = 0.5 * cb2;
    const double h = 0.5 * (ca - cc);
    const double r = sqrt(h * h + b * b);
    const double l1 = 0.5 * (ca + cc) + r;
    const double det = ca * cc - b * b;
    const double l2 = det / l1;
    double vx = h >= 0.0 ? h + r : b, vy = h >= 0.0 ? b : r - h;
    const double vn = sqrt(vx * vx + vy * vy);
    if (vn > 0.0) {
        vx /= vn;
        vy /= vn;
    } else {
        vx = 1.0;
        vy = 0.0;
    }
    g.e1x = vx;
    g.e1y = vy;
    const bool ok = det > 0.0 && l2 > 0.0 && l1 < 1e30;
    g.l1 = (float)l1;
    g.l2 = ok ? (float)l2 : 0.0f;
    // support half-extents in float (IEEE ops, relative error ~1e-7): the blend widens them by 1e-5
    const float fx2 = (float)(vx * vx), fy2 = (float)(vy * vy);
    const float il1 = __frcp_rn(g.l1), il2 = __frcp_rn(g.l2);
    g.hx = ok ? 3.0f * __fsqrt_rn(__fmaf_rn(fx2, il1, fy2 * il2)) : 3.0e38f;
    g.hy = ok ? 3.0f * __fsqrt_rn(__fmaf_rn(fy2, il1, fx2 * il2)) : 3.0e38f;
    return g;
}

// A gathered splat for the blend: (e1x, e1y, p1, p2) in float64, gl = (l1, l2, alpha, z) and
// gr = (rgb lo bits, rgb hi bits, hx, hy) -- the inputs of the blend's tile_entry -- from the
// splat's BlendGeo and SplatRec (4 x 16-byte read-only loads, 3 L2 sectors).
struct GatheredSplat {
    double e1x, e1y, p1, p2;
    float4 gl, gr;
};
__device__ __forceinline__ GatheredSplat gather_splat(const BlendGeo *geo, const void *recs, uint32_t rid) {
    GatheredSplat g;
    const double2 e = __ldg(reinterpret_cast<const double2 *>(geo + rid));
    const float4 lh = __ldg(reinterpret_cast<const float4 *>(geo + rid) + 1);
    const double2 *r = reinterpret_cast<const double2 *>(static_cast<const char *>(recs) + 64 * (size_t)rid);
    const double2 mm = __ldg(r);          // mx, my
    const double2 ca = __ldg(r + 2);      // cc, alpha
    const double2 zr = __ldg(r + 3);      // z, rgb bits
    g.e1x = e.x;
    g.e1y = e.y;
    blend_geo_p(e.x, e.y, mm.x, mm.y, g.p1, g.p2);
    const unsigned long long rgb = (unsigned long long)__double_as_longlong(zr.y);
    g.gl = make_float4(lh.x, lh.y, (float)ca.y, (float)zr.x);
    g.gr = make_float4(__uint_as_float((unsigned)(rgb & 0xffffffffull)), __uint_as_float((unsigned)(rgb >> 32)), lh.z,
                       lh.w);
    return g;
}

__host__ __device__ inline int tiles_of(int px) { return (px + kTile - 1) / kTile; }

// numpy.maximum(x, 0.0) / numpy.clip: NaN propagates (fmax would drop it)
__device__ __forceinline__ double np_max0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
    if (x != x) return x;
    x = x < lo ? lo : x;
    return x > hi ? hi : x;
}
__device__ __forceinline__ float np_clipf(float x, float lo, float hi) {
    if (x != x) return x;
    x = x < lo ? lo : x;
    return x > hi ? hi : x;
}

// sum_k a_k b_k for k = 0,1,2 as OpenBLAS evaluates small gemms
__device__ __forceinline__ double dot3_fma(double a0, double a1, double a2, double b0, double b1, double b2) {
    return fma(a2, b2, fma(a1, b1, a0 * b0));
}
__device__ __forceinline__ double norm4(double a, double b, double c, double d) {
    return sqrt(((a * a + b * b) + c * c) + d * d);
}

// transforms.py:17-34
__device__ __forceinline__ void quat_to_matrix(double w, double x, double y, double z, double m[9]) {
    double xx = x * x, yy = y * y, zz = z * z;
    double xy = x * y, xz = x * z, yz = y * z;
    double wx = w * x, wy = w * y, wz = w * z;
    m[0] = 1.0 - 2.0 * (yy + zz);
    m[1] = 2.0 * (xy - wz);
    m[2] = 2.0 * (xz + wy);
    m[3] = 2.0 * (xy + wz);
    m[4] = 1.0 - 2.0 * (xx + zz);
    m[5] = 2.0 * (yz - wx);
    m[6] = 2.0 * (xz - wy);
    m[7] = 2.0 * (yz + wx);
    m[8] = 1.0 - 2.0 * (xx + yy);
}

// transforms.py:56-70
__device__ __forceinline__ void quat_multiply(const double a[4], const double b[4], double o[4]) {
    double r0 = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    double r1 = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    double r2 = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    double r3 = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
    o[0] = r0;
    o[1] = r1;
    o[2] = r2;
    o[3] = r3;
}

// build_cov3d (projection.py:39-51) for one gaussian: 6 unique entries of R diag(e^s)^2 R^T
// (xx, xy, xz, yy, yz, zz). Overflow yields inf/nan on purpose; the det test rejects it.
__device__ __forceinline__ void build_cov3d(const double ls[3], const double q_raw[4], double cov[6]) {
    double s0 = exp(ls[0]), s1 = exp(ls[1]), s2 = exp(ls[2]);
    double qn = norm4(q_raw[0], q_raw[1], q_raw[2], q_raw[3]);
    double r[9];
    quat_to_matrix(q_raw[0] / qn, q_raw[1] / qn, q_raw[2] / qn, q_raw[3] / qn, r);
    double m[9] = {r[0] * s0, r[1] * s1, r[2] * s2, r[3] * s0, r[4] * s1, r[5] * s2, r[6] * s0, r[7] * s1, r[8] * s2};
    cov[0] = dot3_fma(m[0], m[1], m[2], m[0], m[1], m[2]);
    cov[1] = dot3_fma(m[0], m[1], m[2], m[3], m[4], m[5]);
    cov[2] = dot3_fma(m[0], m[1], m[2], m[6], m[7], m[8]);
    cov[3] = dot3_fma(m[3], m[4], m[5], m[3], m[4], m[5]);
    cov[4] = dot3_fma(m[3], m[4], m[5], m[6], m[7], m[8]);
    cov[5] = dot3_fma(m[6], m[7], m[8], m[6], m[7], m[8]);
}

struct Geo {
    double z, mx, my, ca, cb, cc, radius;  // conic (ca, cb, cc) = (c, -b, a) / det
};

// project_cloud's per-gaussian geometry (projection.py:122-176) for one camera.
// Returns kKeep / kCullDepth / kDegenerate / kCullFrame; fills g only for kKeep.
__device__ __forceinline__ int project_geo(const double p[3], const double cov[6], const sn_camera &c, Geo &g) {
    const double *w = c.rot;
    double z = dot3_fma(p[0], p[1], p[2], w[6], w[7], w[8]) + c.trans[2];
    if (!((z > c.near_) && (z < c.far_))) return kCullDepth;
    double x = dot3_fma(p[0], p[1], p[2], w[0], w[1], w[2]) + c.trans[0];
    double y = dot3_fma(p[0], p[1], p[2], w[3], w[4], w[5]) + c.trans[1];
    double inv_z = 1.0 / z;
    double j00 = c.fx * inv_z, j02 = ((-c.fx) * x * inv_z) * inv_z;
    double j11 = c.fy * inv_z, j12 = ((-c.fy) * y * inv_z) * inv_z;
    // jw = J @ W (2x3), J = [[j00, 0, j02], [0, j11, j12]]
    double jw[6];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        jw[b] = dot3_fma(j00, 0.0, j02, w[b], w[3 + b], w[6 + b]);
        jw[3 + b] = dot3_fma(0.0, j11, j12, w[b], w[3 + b], w[6 + b]);
    }
    const double C[9] = {cov[0], cov[1], cov[2], cov[1], cov[3], cov[4], cov[2], cov[4], cov[5]};
    double t1[6];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            t1[a * 3 + b] = dot3_fma(jw[a * 3], jw[a * 3 + 1], jw[a * 3 + 2], C[b], C[3 + b], C[6 + b]);
    double c00 = dot3_fma(t1[0], t1[1], t1[2], jw[0], jw[1], jw[2]);
    double c01 = dot3_fma(t1[0], t1[1], t1[2], jw[3], jw[4], jw[5]);
    double c11 = dot3_fma(t1[3], t1[4], t1[5], jw[3], jw[4], jw[5]);
    double ca = c00 + kCovReg, cb = c01, cc = c11 + kCovReg;
    double det = ca * cc - cb * cb;
    if (!(det > kDegDet)) return kDegenerate;
    double mx = c.fx * x * inv_z + c.cx;
    double my = c.fy * y * inv_z + c.cy;
    double mid = 0.5 * (ca + cc);
    double lam = mid + sqrt(np_max0(mid * mid - det));
    double radius = kSigma * sqrt(np_max0(lam));
    bool on_frame = (mx + radius >= 0.0) && (mx - radius <= (double)c.width) && (my + radius >= 0.0) &&
                    (my - radius <= (double)c.height);
    if (!on_frame) return kCullFrame;
    g.z = z;
    g.mx = mx;
    g.my = my;
    g.ca = cc / det;
    g.cb = (-cb) / det;
    g.cc = ca / det;
    g.radius = radius;
    return kKeep;
}

// The frame cull of project_geo for an in-depth gaussian, decided in float32 where that is certain
// (-1: undecided, run project_geo). Camera coordinates are project_geo's own float64 values;
// the mean's float32 projection errs by far less than `m`; the 3-sigma radius is at most
// r^ = 3 sqrt(||J||_F^2 tr(cov3d) + 0.3) (lambda_max(J W S W^T J^T) <= ||J W||_2^2 lambda_max(S),
// W orthonormal), and at least 0. While r^ < 3000 px the entries of cov2d stay below 1e6, so the
// float64 determinant is >= 0.09 - 1e-4 and the reference's degenerate test cannot fire: a
// mean inside the frame is kept, a footprint bound outside it is culled, anything else (and
// any non-finite value) takes the float64 path.
__device__ __forceinline__ int frame_prefilter(const double p[3], double tr_cov, const sn_camera &c) {
    const double *w = c.rot;
    const double z = dot3_fma(p[0], p[1], p[2], w[6], w[7], w[8]) + c.trans[2];
    const double x = dot3_fma(p[0], p[1], p[2], w[0], w[1], w[2]) + c.trans[0];
    const double y = dot3_fma(p[0], p[1], p[2], w[3], w[4], w[5]) + c.trans[1];
    // approximate float ops (a few ulp each: the margins below are ~17 ulp and 0.03%)
    const float iz = __frcp_rn((float)z), xz = (float)x * iz, yz = (float)y * iz;
    const float fx = (float)c.fx, fy = (float)c.fy;
    const float mx = __fmaf_rn(fx, xz, (float)c.cx), my = __fmaf_rn(fy, yz, (float)c.cy);
    const float jx = fx * iz, jy = fy * iz;
    const float jf2 = jx * jx * __fmaf_rn(xz, xz, 1.0f) + jy * jy * __fmaf_rn(yz, yz, 1.0f);
    const float l = __fmaf_rn(jf2, (float)tr_cov, 0.3f);
    const float r = 3.001f * (l * rsqrtf(l)) + 1e-3f;
    if (!(r < 3000.0f) || !isfinite(mx) || !isfinite(my)) return -1;  // also catches NaN / inf
    const float W = (float)c.width, H = (float)c.height;
    const float m = 1e-3f + 1e-6f * (fabsf(mx) + fabsf(my) + W + H);
    if (mx >= m && mx <= W - m && my >= m && my <= H - m) return kKeep;
    if (mx + r < -m || mx - r > W + m || my + r < -m || my - r > H + m) return kCullFrame;
    return -1;
}

// renderer.py:83-86: inclusive tile rectangle, clipped to the grid
__device__ __forceinline__ void tile_rect(double mx, double my, double r, int tiles_x, int tiles_y, int rect[4]) {
    rect[0] = (int)np_clip(floor((mx - r) / kTile), 0.0, (double)(tiles_x - 1));
    rect[1] = (int)np_clip(floor((mx + r) / kTile), 0.0, (double)(tiles_x - 1));
    rect[2] = (int)np_clip(floor((my - r) / kTile), 0.0, (double)(tiles_y - 1));
    rect[3] = (int)np_clip(floor((my + r) / kTile), 0.0, (double)(tiles_y - 1));
}

// sh.py:20-49 in float32 (colour is tolerance-checked, not part of the decision chain).
// sh: SoA (K*3, n) float32; dir: unit view direction. K is a compile-time constant (1, 4, 9, 16) so
// the basis stays in registers; coefficient rows are walked with a 32-bit element offset (one
// IMAD.WIDE per load) while 3 K n < 2^32, else with 64-bit indices.
template <int K>
__device__ __forceinline__ void eval_sh_k(const float *__restrict__ sh, int64_t n, int64_t g, float x, float y,
                                          float z, float rgb[3]) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    float basis[16];
    basis[0] = C0;
    if (K > 1) {
        basis[1] = -C1 * y;
        basis[2] = C1 * z;
        basis[3] = -C1 * x;
    }
    if (K > 4) {
        float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
        basis[4] = 1.0925484305920792f * xy;
        basis[5] = -1.0925484305920792f * yz;
        basis[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
        basis[7] = -1.0925484305920792f * xz;
        basis[8] = 0.5462742152960396f * (xx - yy);
        if (K > 9) {
            basis[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
            basis[10] = 2.890611442640554f * xy * z;
            basis[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
            basis[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            basis[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
            basis[14] = 1.445305721320277f * z * (xx - yy);
            basis[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
        }
    }
    float acc[3] = {0.0f, 0.0f, 0.0f};
    if ((uint64_t)(3 * K) * (uint64_t)n < (1ull << 32)) {
        const uint32_t un = (uint32_t)n;
        uint32_t off = (uint32_t)g;
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                acc[ch] = __fmaf_rn(basis[k], __ldg(sh + off), acc[ch]);
                off += un;
            }
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
                acc[ch] = __fmaf_rn(basis[k], __ldg(sh + (int64_t)(3 * k + ch) * n + g), acc[ch]);
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) rgb[ch] = np_clipf(acc[ch] + 0.5f, 0.0f, 1.0f);
}

__device__ __forceinline__ void eval_sh_f32(const float *__restrict__ sh, int64_t n, int64_t g, int K, float x,
                                            float y, float z, float rgb[3]) {
    switch (K) {
        case 16: eval_sh_k<16>(sh, n, g, x, y, z, rgb); break;
        case 9: eval_sh_k<9>(sh, n, g, x, y, z, rgb); break;
        case 4: eval_sh_k<4>(sh, n, g, x, y, z, rgb); break;
        default: eval_sh_k<1>(sh, n, g, x, y, z, rgb); break;
    }
}

__device__ __forceinline__ unsigned long long pack_rgb21(const float rgb[3]) {
    const float s = 2097151.0f;  // 2^21 - 1
    unsigned long long r = (unsigned long long)__float2uint_rn(rgb[0] * s);
    unsigned long long g = (unsigned long long)__float2uint_rn(rgb[1] * s);
    unsigned long long b = (unsigned long long)__float2uint_rn(rgb[2] * s);
    return r | (g << 21) | (b << 42);
}
__device__ __forceinline__ void unpack_rgb21(unsigned long long v, float rgb[3]) {
    const float inv = 1.0f / 2097151.0f;
    rgb[0] = (float)(unsigned)(v & 0x1FFFFFull) * inv;
    rgb[1] = (float)(unsigned)((v >> 21) & 0x1FFFFFull) * inv;
    rgb[2] = (float)(unsigned)((v >> 42) & 0x1FFFFFull) * inv;
}

// View direction (projection.py:178-180) for SH, from float64 position and camera centre. The
// difference is float64; the normalization is float32 (colour is tolerance-checked: a direction
// error of ~1e-7 moves an SH colour by far less than the 2e-3 bar).
__device__ __forceinline__ void view_dir(const double p[3], const sn_camera &c, float d[3]) {
    const float v0 = (float)(p[0] - c.center[0]), v1 = (float)(p[1] - c.center[1]), v2 = (float)(p[2] - c.center[2]);
    const float n2 = __fmaf_rn(v0, v0, __fmaf_rn(v1, v1, v2 * v2));
    const float inv = n2 > 0.0f ? rsqrtf(n2) : 1.0f;  // the reference divides by 1 for a zero vector
    d[0] = v0 * inv;
    d[1] = v1 * inv;
    d[2] = v2 * inv;
}

__device__ __forceinline__ double sigmoid(double o) { return 1.0 / (1.0 + exp(-o)); }

}  // namespace sn
