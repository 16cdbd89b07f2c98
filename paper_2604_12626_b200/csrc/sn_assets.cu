// sn_assets.cu -- asset ingest on the device: the reference's on-disk layouts unpacked straight into
// the renderer's device layouts.
//
//   * 3DGS PLY vertex table (ply.py:76-120: row-major float32, f_rest channel-major on disk) ->
//     sn_cloud float32 buffers (pos+opacity, log-scales, rotations (n,4) and SH as a (K*3, n)
//     structure-of-arrays);
//   * avatar bundle canonical.f32 (avatar.py:191-254: field blocks, f_rest coefficient-major) ->
//     the sn_avatars float64 canonical buffers + SH SoA, and weights.f32 (N x J dense) -> up to
//     4 (joint, weight) influences per gaussian in ascending joint order.
//
// Validation follows GaussianCloud.validate (cloud.py:50-87) and AvatarBundle.validate
// (avatar.py:155-176) exactly: non-finite values per field, zero-norm rotations, the float32
// quaternion renormalization (np.linalg.norm = sqrt(((x0^2 + x1^2) + x2^2) + x3^2) in float32,
// applied to every row when any row deviates by more than 1e-5), negative weights, the float64
// row sums in numpy's pairwise order and the renormalization of every row when any row deviates
// by more than 1e-5 (error above 1e-3). Counters and per-row flags go to the caller; the host side
// (assets.py) raises the reference's exceptions from them.
#include "sn_common.cuh"
#include "sn_internal.h"

#include <cuda_fp16.h>

namespace sn {

namespace {

constexpr double kQuatNormTol = 1e-5;  // cloud.py:14 (compared in float64, like numpy)
constexpr double kWeightSumTol = 1e-5;

// counters: [0..4] rows with non-finite positions / sh / opacity / log-scales / rotations,
//           [5] zero-norm rotations, [6] max |norm - 1| (float bits), [7] rows with negative weights,
//           [8] rows with more than 4 nonzero weights, [9] max |row sum - 1| (double bits)
enum { kCntNonFinite = 0, kCntZeroNorm = 5, kCntQuatDev = 6, kCntNegW = 7, kCntManyW = 8, kCntSumDev = 9 };

__device__ __forceinline__ bool finite(float x) { return isfinite(x); }

struct CloudDst {
    int32_t f64;       // 0: float32 (n,4) buffers (scene cloud); 1: float64 (avatar canonical)
    void *pos_opacity, *log_scales, *rotations;
    float *sh;         // (K*3, sh_stride)
    int64_t sh_stride, row0;  // SoA stride (all gaussians of the set) and this cloud's first row
};

__device__ __forceinline__ void store4(const CloudDst &d, void *base, int64_t row, float a, float b, float c,
                                       float e) {
    if (d.f64) {
        double *p = static_cast<double *>(base) + 4 * (d.row0 + row);
        p[0] = a;
        p[1] = b;
        p[2] = c;
        p[3] = e;
    } else {
        reinterpret_cast<float4 *>(base)[d.row0 + row] = make_float4(a, b, c, e);
    }
}

// One gaussian: fields gathered by the caller's accessor, validated, stored unnormalized.
__device__ __forceinline__ void unpack_row(const CloudDst &d, int64_t row, const float pos[3], const float *shv,
                                           int sh_k, float opacity, const float ls[3], const float rot[4],
                                           uint8_t *flags, unsigned long long *cnt) {
    unsigned f = 0;
    if (!(finite(pos[0]) && finite(pos[1]) && finite(pos[2]))) f |= 1u;
    bool sh_ok = true;
    for (int i = 0; i < 3 * sh_k; ++i) sh_ok &= finite(shv[i]);
    if (!sh_ok) f |= 2u;
    if (!finite(opacity)) f |= 4u;
    if (!(finite(ls[0]) && finite(ls[1]) && finite(ls[2]))) f |= 8u;
    if (!(finite(rot[0]) && finite(rot[1]) && finite(rot[2]) && finite(rot[3]))) f |= 16u;
    // np.linalg.norm(rotations, axis=1) in float32: sequential sum of squares, then sqrt
    const float nrm = sqrtf(__fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(rot[0], rot[0]), __fmul_rn(rot[1], rot[1])),
                                                __fmul_rn(rot[2], rot[2])),
                                      __fmul_rn(rot[3], rot[3])));
    if (!(nrm > 0.0f)) f |= 32u;
    for (int b = 0; b < 6; ++b)
        if (f & (1u << b)) atomicAdd(cnt + b, 1ull);
    const float dev = fabsf(__fsub_rn(nrm, 1.0f));
    // warp-aggregated max (one atomic per warp; dev >= 0, so its bits order like the value)
    const unsigned active = __activemask();
    const unsigned m = __reduce_max_sync(active, dev == dev ? __float_as_uint(dev) : 0u);
    if ((threadIdx.x & 31) == __ffs(active) - 1) atomicMax(cnt + kCntQuatDev, (unsigned long long)m);
    flags[row] = (uint8_t)f;
    store4(d, d.pos_opacity, row, pos[0], pos[1], pos[2], opacity);
    store4(d, d.log_scales, row, ls[0], ls[1], ls[2], 0.0f);
    store4(d, d.rotations, row, rot[0], rot[1], rot[2], rot[3]);
    for (int k = 0; k < sh_k; ++k)
        for (int c = 0; c < 3; ++c) d.sh[(int64_t)(3 * k + c) * d.sh_stride + d.row0 + row] = shv[3 * k + c];
}

// ply.py:97-118: row-major float32 table; cols = x y z f_dc_0..2 opacity scale_0..2 rot_0..3
// f_rest_0..f_rest_(3(K-1)-1) (column index of each); f_rest is channel-major on disk.
struct PlyCols {
    int32_t c[14 + 45];
};

constexpr int kPlyRows = 128;  // rows per CTA, staged through shared memory (coalesced loads)

__global__ void __launch_bounds__(kPlyRows) unpack_ply_kernel(int64_t n, int32_t n_props, const float *table,
                                                              PlyCols cl, int32_t sh_k, CloudDst d, uint8_t *flags,
                                                              unsigned long long *cnt) {
    extern __shared__ float s_tab[];  // kPlyRows x n_props
    const int32_t *cols = cl.c;
    const int64_t row0 = (int64_t)blockIdx.x * kPlyRows;
    const int rows = (int)min((int64_t)kPlyRows, n - row0);
    const int64_t words = (int64_t)rows * n_props;
    const float *src = table + row0 * n_props;
    for (int64_t i = threadIdx.x; i < words; i += kPlyRows) s_tab[i] = __ldg(src + i);
    __syncthreads();
    if (threadIdx.x >= rows) return;
    const int64_t row = row0 + threadIdx.x;
    const float *r = s_tab + threadIdx.x * n_props;
    float pos[3], ls[3], rot[4], shv[48];
    for (int i = 0; i < 3; ++i) pos[i] = r[cols[i]];
    for (int c = 0; c < 3; ++c) shv[c] = r[cols[3 + c]];
    const float opacity = r[cols[6]];
    for (int i = 0; i < 3; ++i) ls[i] = r[cols[7 + i]];
    for (int i = 0; i < 4; ++i) rot[i] = r[cols[10 + i]];
    const int rest = sh_k - 1;
    for (int i = 0; i < 3 * rest; ++i) {  // f_rest_i: channel i / rest, coefficient 1 + i % rest
        const int c = i / rest, k = 1 + i % rest;
        shv[3 * k + c] = r[cols[14 + i]];
    }
    unpack_row(d, row, pos, shv, sh_k, opacity, ls, rot, flags, cnt);
}

// avatar.py:217-237: canonical.f32 = positions (n,3) | f_dc (n,3) | f_rest (n,K-1,3) | opacities (n)
// | log_scales (n,3) | rotations (n,4), one block after another.
__global__ void __launch_bounds__(256) unpack_bundle_kernel(int64_t n, const float *blob, int32_t sh_k, CloudDst d,
                                                            uint8_t *flags, unsigned long long *cnt) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const int rest = sh_k - 1;
    const float *pos_b = blob, *dc_b = pos_b + 3 * n, *rest_b = dc_b + 3 * n, *op_b = rest_b + 3 * rest * n;
    const float *ls_b = op_b + n, *rot_b = ls_b + 3 * n;
    float pos[3], ls[3], rot[4], shv[48];
    for (int i = 0; i < 3; ++i) pos[i] = __ldg(pos_b + 3 * row + i);
    for (int c = 0; c < 3; ++c) shv[c] = __ldg(dc_b + 3 * row + c);
    for (int i = 0; i < 3 * rest; ++i) shv[3 + i] = __ldg(rest_b + 3 * rest * row + i);
    const float opacity = __ldg(op_b + row);
    for (int i = 0; i < 3; ++i) ls[i] = __ldg(ls_b + 3 * row + i);
    for (int i = 0; i < 4; ++i) rot[i] = __ldg(rot_b + 4 * row + i);
    unpack_row(d, row, pos, shv, sh_k, opacity, ls, rot, flags, cnt);
}

// cloud.py:85-86: when any row's norm deviates by more than 1e-5, every row is divided by its
// float32 norm (the max deviation is read on the device: no host round trip)
__global__ void __launch_bounds__(256) renorm_rot_kernel(int64_t n, CloudDst d, const unsigned long long *cnt) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    if (!((double)__uint_as_float((unsigned)cnt[kCntQuatDev]) > kQuatNormTol)) return;
    float q[4];
    if (d.f64) {
        const double *p = static_cast<const double *>(d.rotations) + 4 * (d.row0 + row);
        for (int i = 0; i < 4; ++i) q[i] = (float)p[i];
    } else {
        const float4 v = reinterpret_cast<const float4 *>(d.rotations)[d.row0 + row];
        q[0] = v.x, q[1] = v.y, q[2] = v.z, q[3] = v.w;
    }
    const float nrm = sqrtf(__fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(q[0], q[0]), __fmul_rn(q[1], q[1])),
                                                __fmul_rn(q[2], q[2])),
                                      __fmul_rn(q[3], q[3])));
    store4(d, d.rotations, row, __fdiv_rn(q[0], nrm), __fdiv_rn(q[1], nrm), __fdiv_rn(q[2], nrm),
           __fdiv_rn(q[3], nrm));
}

// numpy's pairwise summation of one contiguous float64 row (the order w.sum(axis=1) uses):
// < 8 items sequential; <= 128 items: 8 strided accumulators, tree-combined, tail sequential;
// larger: split at a multiple of 8 and recurse (one level suffices for J <= 255).
__device__ double np_pairwise_sum8(const float *a, int n) {
    if (n < 8) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += (double)a[i];
        return s;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = (double)a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += (double)a[i + j];
    double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) s += (double)a[i];
    return s;
}
__device__ double np_pairwise_sum(const float *a, int n) {
    if (n <= 128) return np_pairwise_sum8(a, n);
    int n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum8(a, n2) + np_pairwise_sum8(a + n2, n - n2);
}

// weights.f32 row -> up to 4 (joint, weight) influences, ascending joint order (rig.py:119-132
// visits joints in that order); the row sum's deviation feeds the all-rows renormalization.
__global__ void __launch_bounds__(256) pack_weights_kernel(int64_t n, int32_t J, const float *w, int64_t row0,
                                                           uint32_t *joints, double *wts, double *sums,
                                                           uint8_t *flags, unsigned long long *cnt) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const float *r = w + row * J;
    uint32_t packed = 0;
    double w4[4] = {0.0, 0.0, 0.0, 0.0};
    int nz = 0;
    bool neg = false;
    for (int j = 0; j < J; ++j) {
        const float v = __ldg(r + j);
        if (v < 0.0f) neg = true;
        if (v != 0.0f) {
            if (nz < 4) {
                packed |= (uint32_t)j << (8 * nz);
                w4[nz] = (double)v;
            }
            ++nz;
        }
    }
    const double s = np_pairwise_sum(r, J);
    sums[row] = s;
    const double dev = fabs(s - 1.0);
    if (dev == dev) atomicMax(cnt + kCntSumDev, (unsigned long long)__double_as_longlong(dev));
    if (neg) atomicAdd(cnt + kCntNegW, 1ull);
    if (nz > 4) atomicAdd(cnt + kCntManyW, 1ull);
    flags[row] |= (uint8_t)((neg ? 64u : 0u) | (nz > 4 ? 128u : 0u));
    joints[row0 + row] = packed;
    for (int k = 0; k < 4; ++k) wts[4 * (row0 + row) + k] = w4[k];
}

// avatar.py:169-170: every row divided by its float64 sum when any row deviates by more than 1e-5
__global__ void __launch_bounds__(256) renorm_weights_kernel(int64_t n, int64_t row0, double *wts, const double *sums,
                                                             const unsigned long long *cnt) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    if (!(__longlong_as_double((long long)cnt[kCntSumDev]) > kWeightSumTol)) return;
    const double s = sums[row];
    for (int k = 0; k < 4; ++k) wts[4 * (row0 + row) + k] = wts[4 * (row0 + row) + k] / s;
}

// Skins wider than 4 influences: row `row` of weights.f32 -> its nonzeros (ascending joint) at
// offsets[row] of the CSR arrays, float64, divided by the float64 row sum when any row of the
// bundle deviated by more than 1e-5 (the same rule as renorm_weights_kernel).
__global__ void __launch_bounds__(256) pack_csr_kernel(int64_t n, int32_t J, const float *w, const double *sums,
                                                       const unsigned long long *cnt, const uint32_t *offsets,
                                                       uint8_t *joint, double *weight) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const bool renorm = __longlong_as_double((long long)cnt[kCntSumDev]) > kWeightSumTol;
    const double s = sums[row];
    const float *r = w + row * J;
    uint32_t o = offsets[row];
    for (int j = 0; j < J; ++j) {
        const float v = __ldg(r + j);
        if (v == 0.0f) continue;
        joint[o] = (uint8_t)j;
        weight[o] = renorm ? (double)v / s : (double)v;
        ++o;
    }
}

unsigned grid_for(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t launch_unpack_ply(int64_t n, int32_t n_props, const float *table, const int32_t *cols, int32_t sh_k,
                              float *pos_opacity, float *log_scales, float *rotations, float *sh, uint8_t *flags,
                              unsigned long long *cnt, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    CloudDst d{0, pos_opacity, log_scales, rotations, sh, n, 0};
    PlyCols cl{};
    for (int i = 0; i < 14 + 3 * (sh_k - 1); ++i) cl.c[i] = cols[i];  // host array, passed by value
    const size_t smem = sizeof(float) * kPlyRows * (size_t)n_props;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(unpack_ply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    unpack_ply_kernel<<<(unsigned)((n + kPlyRows - 1) / kPlyRows), kPlyRows, smem, s>>>(n, n_props, table, cl, sh_k,
                                                                                        d, flags, cnt);
    renorm_rot_kernel<<<grid_for(n), 256, 0, s>>>(n, d, cnt);
    return cudaGetLastError();
}

cudaError_t launch_unpack_bundle(int64_t n, int32_t sh_k, int32_t J, const float *canonical, const float *weights,
                                 int64_t row0, int64_t sh_stride, double *pos_opacity, double *log_scales,
                                 double *rotations, float *sh, uint32_t *joints, double *wts, double *sums,
                                 uint8_t *flags, unsigned long long *cnt, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    CloudDst d{1, pos_opacity, log_scales, rotations, sh, sh_stride, row0};
    unpack_bundle_kernel<<<grid_for(n), 256, 0, s>>>(n, canonical, sh_k, d, flags, cnt);
    renorm_rot_kernel<<<grid_for(n), 256, 0, s>>>(n, d, cnt);
    pack_weights_kernel<<<grid_for(n), 256, 0, s>>>(n, J, weights, row0, joints, wts, sums, flags, cnt);
    renorm_weights_kernel<<<grid_for(n), 256, 0, s>>>(n, row0, wts, sums, cnt);
    return cudaGetLastError();
}

cudaError_t launch_pack_csr(int64_t n, int32_t J, const float *weights, const double *sums,
                            const unsigned long long *cnt, const uint32_t *offsets, uint8_t *joint, double *weight,
                            cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    pack_csr_kernel<<<grid_for(n), 256, 0, s>>>(n, J, weights, sums, cnt, offsets, joint, weight);
    return cudaGetLastError();
}

}  // namespace sn

// ---- frame export (frame_io.py:11-58) and the observation payload ----

namespace sn {

namespace {

// uint8 colour exactly as frame_io.save_color_png (frame_io.py:13-14) evaluates it on the same
// values: clip to [0, 1], x * 255 + 0.5 in float64, truncation; fp16 depth (round to nearest).
__global__ void __launch_bounds__(256) quantize_kernel(int64_t npix, const float *color, const float *depth,
                                                       uint8_t *rgb8, __half *depth16) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix) return;
    for (int c = 0; c < 3; ++c) {
        double x = (double)color[3 * i + c];
        x = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
        rgb8[3 * i + c] = (uint8_t)(x * 255.0 + 0.5);
    }
    if (depth16) depth16[i] = __float2half_rn(depth[i]);
}

// frame_io.save_depth_pfm (:23-31): rows bottom-to-top, little-endian float32
__global__ void __launch_bounds__(256) flip_rows_kernel(int64_t frames, int32_t h, int32_t w, const float *src,
                                                        float *dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t hw = (int64_t)h * w;
    if (i >= frames * hw) return;
    const int64_t f = i / hw, p = i % hw, y = p / w, x = p % w;
    dst[f * hw + (int64_t)(h - 1 - y) * w + x] = src[i];
}

}  // namespace

cudaError_t launch_quantize(int64_t npix, const float *color, const float *depth, uint8_t *rgb8, uint16_t *depth16,
                            cudaStream_t s) {
    if (npix == 0) return cudaSuccess;
    quantize_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(npix, color, depth, rgb8,
                                                                   reinterpret_cast<__half *>(depth16));
    return cudaGetLastError();
}

cudaError_t launch_flip_rows(int64_t frames, int32_t h, int32_t w, const float *src, float *dst, cudaStream_t s) {
    const int64_t n = frames * h * w;
    if (n == 0) return cudaSuccess;
    flip_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(frames, h, w, src, dst);
    return cudaGetLastError();
}

}  // namespace sn
