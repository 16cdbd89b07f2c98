// sn_rig.cu -- per-(env, avatar) pose sampling and joint preparation.
//
// AvatarRuntime.clock (tasks.py:299-305) -> sample_pose (rig.py:78-104, nlerp with hemisphere
// correction, transforms.py:73-81) -> M_j = rigid(q_j, t_j) @ inv_bind_j (rig.py:116) and the
// effective joint quaternions q_root * matrix_to_quat(M_j) (rig.py:127-128, Shepperd,
// transforms.py:37-53). One CTA per (env, avatar), one thread per joint (+ root). The output
// pose block is what the fused skin->project kernels read (a few KB per env and avatar).
#include "sn_common.cuh"
#include "sn_internal.h"

namespace sn {

namespace {

__device__ __forceinline__ void matrix_to_quat(const double m[9], double q[4]) {
    double t = (m[0] + m[4]) + m[8];
    double s;
    if (t > 0.0) {
        s = sqrt(t + 1.0) * 2.0;
        q[0] = 0.25 * s;
        q[1] = (m[7] - m[5]) / s;
        q[2] = (m[2] - m[6]) / s;
        q[3] = (m[3] - m[1]) / s;
    } else if (m[0] >= m[4] && m[0] >= m[8]) {
        s = sqrt(((1.0 + m[0]) - m[4]) - m[8]) * 2.0;
        q[0] = (m[7] - m[5]) / s;
        q[1] = 0.25 * s;
        q[2] = (m[1] + m[3]) / s;
        q[3] = (m[2] + m[6]) / s;
    } else if (m[4] >= m[8]) {
        s = sqrt(((1.0 + m[4]) - m[0]) - m[8]) * 2.0;
        q[0] = (m[2] - m[6]) / s;
        q[1] = (m[1] + m[3]) / s;
        q[2] = 0.25 * s;
        q[3] = (m[5] + m[7]) / s;
    } else {
        s = sqrt(((1.0 + m[8]) - m[0]) - m[4]) * 2.0;
        q[0] = (m[3] - m[1]) / s;
        q[1] = (m[2] + m[6]) / s;
        q[2] = (m[5] + m[7]) / s;
        q[3] = 0.25 * s;
    }
    double n = norm4(q[0], q[1], q[2], q[3]);
    q[0] /= n;
    q[1] /= n;
    q[2] /= n;
    q[3] /= n;
}

// rigid(q, t) @ inv_bind (4x4 @ 4x4, FMA chain over k as OpenBLAS), rows 0..2 -> M (12);
// then the effective quaternion q_root * q(M[:3,:3]).
__device__ __forceinline__ void joint_prep(const double q[4], const double t[3], const double root_q[4],
                                           const double *ib, double *jm_out, double *eq_out) {
    double r[9];
    quat_to_matrix(q[0], q[1], q[2], q[3], r);
    double rm[12] = {r[0], r[1], r[2], t[0], r[3], r[4], r[5], t[1], r[6], r[7], r[8], t[2]};
    double m[12];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
            m[a * 4 + b] = fma(rm[a * 4 + 3], ib[12 + b],
                               fma(rm[a * 4 + 2], ib[8 + b], fma(rm[a * 4 + 1], ib[4 + b], rm[a * 4 + 0] * ib[b])));
#pragma unroll
    for (int i = 0; i < 12; ++i) jm_out[i] = m[i];
    double m3[9] = {m[0], m[1], m[2], m[4], m[5], m[6], m[8], m[9], m[10]};
    double mq[4];
    matrix_to_quat(m3, mq);
    double e[4];
    quat_multiply(root_q, mq, e);
    eq_out[0] = e[0];
    eq_out[1] = e[1];
    eq_out[2] = e[2];
    eq_out[3] = e[3];
}

__device__ __forceinline__ void root_prep(const double q[4], const double t[3], double *root) {
    double r[9];
    quat_to_matrix(q[0], q[1], q[2], q[3], r);
#pragma unroll
    for (int i = 0; i < 9; ++i) root[i] = r[i];
    root[9] = t[0];
    root[10] = t[1];
    root[11] = t[2];
}

// sample_pose for joint j of one trajectory at time t (t >= 0 checked by the caller).
__device__ __forceinline__ void sample_joint(const double *tq, const double *tt, int n_frames, int jp, double fps,
                                             double t, int j, double q[4], double tr[3]) {
    double pos = t * fps;
    double ff = floor(pos);
    int last = n_frames - 1;
    if (ff >= (double)last) {
        const double *a = tq + ((int64_t)last * jp + j) * 4;
        const double *b = tt + ((int64_t)last * jp + j) * 3;
        q[0] = a[0]; q[1] = a[1]; q[2] = a[2]; q[3] = a[3];
        tr[0] = b[0]; tr[1] = b[1]; tr[2] = b[2];
        return;
    }
    int f = (int)ff;
    double lam = pos - ff;
    const double *qa = tq + ((int64_t)f * jp + j) * 4, *qb = tq + ((int64_t)(f + 1) * jp + j) * 4;
    const double *ta = tt + ((int64_t)f * jp + j) * 3, *tb = tt + ((int64_t)(f + 1) * jp + j) * 3;
    if (lam == 0.0) {
        q[0] = qa[0]; q[1] = qa[1]; q[2] = qa[2]; q[3] = qa[3];
        tr[0] = ta[0]; tr[1] = ta[1]; tr[2] = ta[2];
        return;
    }
    double dot = ((qa[0] * qb[0] + qa[1] * qb[1]) + qa[2] * qb[2]) + qa[3] * qb[3];
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double bk = dot < 0.0 ? -qb[k] : qb[k];
        v[k] = qa[k] + lam * (bk - qa[k]);
    }
    double n = norm4(v[0], v[1], v[2], v[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = v[k] / n;
#pragma unroll
    for (int k = 0; k < 3; ++k) tr[k] = ta[k] + lam * (tb[k] - ta[k]);
}

__global__ void pose_kernel(sn_avatars av, const double *sim_times, double *pose_q, double *pose_t,
                            double *joint_mats, double *eff_q, double *root, int32_t *err_flag) {
    __shared__ double s_root_q[4];
    int ea = blockIdx.x;
    int A = av.n_avatars, J = av.n_joints, jp = J + 1;
    int env = ea / A, a = ea % A;
    int j = threadIdx.x;
    // AvatarRuntime.clock (tasks.py:299-305)
    double fps = av.fps[a];
    int nf = av.n_frames[a];
    double t = av.start_offset[a] + sim_times[env];
    double duration = (double)nf / fps;
    if (av.loop[a] && duration > 0)
        t = fmod(t, duration);
    else
        t = t < duration ? t : duration;
    bool bad = !(t >= 0.0);  // rig.py:80-81 (also rejects NaN)
    const double *tq = av.traj_q + av.traj_offset[a] * jp * 4;
    const double *tt = av.traj_t + av.traj_offset[a] * jp * 3;
    double q[4] = {1.0, 0.0, 0.0, 0.0}, tr[3] = {0.0, 0.0, 0.0};
    if (j <= J && !bad) sample_joint(tq, tt, nf, jp, fps, t, j, q, tr);
    if (j == J) {
        s_root_q[0] = q[0]; s_root_q[1] = q[1]; s_root_q[2] = q[2]; s_root_q[3] = q[3];
    }
    __syncthreads();
    if (j > J) return;
    if (bad) {
        if (j == 0) atomicExch(err_flag, 1);
        return;
    }
    if (pose_q) {
        double *oq = pose_q + ((int64_t)ea * jp + j) * 4;
        double *ot = pose_t + ((int64_t)ea * jp + j) * 3;
        oq[0] = q[0]; oq[1] = q[1]; oq[2] = q[2]; oq[3] = q[3];
        ot[0] = tr[0]; ot[1] = tr[1]; ot[2] = tr[2];
    }
    if (joint_mats == nullptr) return;
    if (j < J) {
        double rq[4] = {s_root_q[0], s_root_q[1], s_root_q[2], s_root_q[3]};
        joint_prep(q, tr, rq, av.inv_bind + ((int64_t)a * J + j) * 16, joint_mats + ((int64_t)ea * J + j) * 12,
                   eff_q + ((int64_t)ea * J + j) * 4);
    } else {
        root_prep(q, tr, root + (int64_t)ea * 12);
    }
}

__global__ void joint_prep_kernel(sn_avatars av, int avatar, const double *pose_q, const double *pose_t,
                                  double *joint_mats, double *eff_q, double *root) {
    int J = av.n_joints, j = threadIdx.x;
    if (j > J) return;
    double q[4] = {pose_q[4 * j], pose_q[4 * j + 1], pose_q[4 * j + 2], pose_q[4 * j + 3]};
    double t[3] = {pose_t[3 * j], pose_t[3 * j + 1], pose_t[3 * j + 2]};
    if (j < J) {
        double rq[4] = {pose_q[4 * J], pose_q[4 * J + 1], pose_q[4 * J + 2], pose_q[4 * J + 3]};
        joint_prep(q, t, rq, av.inv_bind + ((int64_t)avatar * J + j) * 16, joint_mats + 12 * j, eff_q + 4 * j);
    } else {
        root_prep(q, t, root);
    }
}

// Per avatar: the largest canonical position norm and the largest 3D standard deviation
// exp(max log-scale); per (avatar, joint): d_j = the largest |inv_bind_j P| over the gaussians the
// joint influences -- the inputs of the (env, avatar) culling bound below.
// ext layout per avatar: [0] |P|max, [1] s_max, [2 .. 2 + J) d_j (non-negative doubles as bits)
__global__ void __launch_bounds__(256) avatar_extent_kernel(sn_avatars av, unsigned long long *ext) {
    // a block's 256 gaussians belong to at most two avatars (contiguous ranges): reduce the maxima
    // in shared memory, then one global atomic per slot and block
    extern __shared__ unsigned long long s_ext[];  // 2 x (2 + J)
    const int J = av.n_joints, slots = 2 + J;
    for (int i = threadIdx.x; i < 2 * slots; i += blockDim.x) s_ext[i] = 0ull;
    __syncthreads();
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t g = g0 + threadIdx.x;
    const int a_lo = av.avatar_of[g0];
    if (g < av.n) {
        const int a = av.avatar_of[g];
        unsigned long long *e = s_ext + (a == a_lo ? 0 : slots);
        const double *p = av.pos_opacity + 4 * g, *l = av.log_scales + 4 * g;
        const double r = sqrt((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2]);
        // (a non-finite rotation poisons the scale bound too: its covariance, hence the reference's
        // degenerate test, cannot be bounded)
        const double *qq = av.rotations + 4 * g;
        const bool q_ok = isfinite(qq[0]) && isfinite(qq[1]) && isfinite(qq[2]) && isfinite(qq[3]);
        const double sm = q_ok ? exp(fmax(fmax(l[0], l[1]), l[2])) : INFINITY;
        // non-negative doubles order like their bit patterns; NaN/inf poison the bound (no culling)
        atomicMax(e, (unsigned long long)__double_as_longlong(r == r ? r : INFINITY));
        atomicMax(e + 1, (unsigned long long)__double_as_longlong(sm == sm ? sm : INFINITY));
        const bool csr = av.infl_offset != nullptr;
        const uint32_t j4 = csr ? 0u : av.joints[g];
        const int64_t k0 = csr ? (int64_t)av.infl_offset[g] : 0, k1 = csr ? (int64_t)av.infl_offset[g + 1] : 4;
        for (int64_t k = k0; k < k1; ++k) {
            if ((csr ? av.infl_weight[k] : av.weights[4 * g + k]) == 0.0) continue;
            const int j = csr ? (int)av.infl_joint[k] : (int)((j4 >> (8 * k)) & 0xff);
            const double *ib = av.inv_bind + ((int64_t)a * J + j) * 16;
            const double x = ((ib[0] * p[0] + ib[1] * p[1]) + ib[2] * p[2]) + ib[3];
            const double y = ((ib[4] * p[0] + ib[5] * p[1]) + ib[6] * p[2]) + ib[7];
            const double z = ((ib[8] * p[0] + ib[9] * p[1]) + ib[10] * p[2]) + ib[11];
            const double d = sqrt((x * x + y * y) + z * z);
            atomicMax(e + 2 + j, (unsigned long long)__double_as_longlong(d == d ? d : INFINITY));
        }
    }
    __syncthreads();
    const int64_t g_last = min(av.n, g0 + (int64_t)blockDim.x) - 1;
    const int a_hi = av.avatar_of[g_last];
    for (int i = threadIdx.x; i < 2 * slots; i += blockDim.x) {
        const int which = i / slots, slot = i % slots;
        const int a = which ? a_hi : a_lo;
        if (which && a_hi == a_lo) continue;
        if (s_ext[i]) atomicMax(ext + (int64_t)a * slots + slot, s_ext[i]);
    }
}

// Whole-avatar culling per (env, avatar), conservative and exact in its RenderStats category.
// Skinned position p' = R_root b + t_root with b = (1 - sum w) P + sum_j w_j rigid_j(inv_bind_j P),
// 0 <= w, |sum w - 1| <= 1e-3 (AvatarBundle validation): rigid_j(inv_bind_j P) lies within d_j of
// the joint's sampled translation t_j, so b lies within rho = max_j (|t_j - c| + d_j) + 1e-3 |P|max of
// any centre c (c = centre of the joints' bounding box), and p' within rho of R_root c + t_root.
// Code kCullDepth: the whole ball is at z <= near or z >= far (projection.py:128-135). Code
// kCullFrame: the ball is strictly inside (near, far), every covariance is finite (so det > 1e-12:
// cov2d >= 0.3 I), and even with the largest projected radius 3 sqrt(||J||_F^2 s_max^2 + 0.3)
// (>= 3 sqrt(lambda_max)) every mean misses the frame on one side (projection.py:160-166).
// kWholeVisible: the ball is strictly inside (near, far), every mean lands inside the frame (so the
// inclusive 3-sigma frame test passes whatever the radius), and that radius bound stays below
// 3000 px, so the cov2d entries stay below 1e6 and the float64 determinant cannot fall to the
// degenerate threshold (>= 0.09 - 1e-4): every gaussian is kept without being skinned.
// 0: test every gaussian.
__global__ void avatar_cull_kernel(sn_avatars av, PoseView pv, const double *pose_t, const sn_camera *cams,
                                   const unsigned long long *ext, int n_envs, uint8_t *codes) {
    const int ea = blockIdx.x * blockDim.x + threadIdx.x;
    const int A = av.n_avatars, J = av.n_joints;
    if (ea >= n_envs * A) return;
    const int env = ea / A, a = ea % A;
    const unsigned long long *e = ext + (int64_t)a * (2 + J);
    const double pmax = __longlong_as_double((long long)e[0]);
    const double smax = __longlong_as_double((long long)e[1]);
    const double *tj = pose_t + (int64_t)ea * (J + 1) * 3, *root = pv.root + (int64_t)ea * 12;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int j = 0; j < J; ++j)
        for (int k = 0; k < 3; ++k) {
            lo[k] = fmin(lo[k], tj[3 * j + k]);
            hi[k] = fmax(hi[k], tj[3 * j + k]);
        }
    const double cb[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    double rb = 0.0;
    for (int j = 0; j < J; ++j) {
        const double dx = tj[3 * j] - cb[0], dy = tj[3 * j + 1] - cb[1], dz = tj[3 * j + 2] - cb[2];
        rb = fmax(rb, sqrt((dx * dx + dy * dy) + dz * dz) + __longlong_as_double((long long)e[2 + j]));
    }
    uint8_t code = 0;
    const double rho = (rb + 1e-3 * pmax) * (1.0 + 1e-9) + 1e-9;
    if (rho < 1e30) {
        // ball centre in the world: R_root cb + t_root
        const double px = ((root[0] * cb[0] + root[1] * cb[1]) + root[2] * cb[2]) + root[9];
        const double py = ((root[3] * cb[0] + root[4] * cb[1]) + root[5] * cb[2]) + root[10];
        const double pz = ((root[6] * cb[0] + root[7] * cb[1]) + root[8] * cb[2]) + root[11];
        const sn_camera &c = cams[env];
        const double *w = c.rot;
        const double xc = ((w[0] * px + w[1] * py) + w[2] * pz) + c.trans[0];
        const double yc = ((w[3] * px + w[4] * py) + w[5] * pz) + c.trans[1];
        const double zc = ((w[6] * px + w[7] * py) + w[8] * pz) + c.trans[2];
        const double tol = 1e-9 * (1.0 + fabs(zc) + rho);
        if (zc + rho < c.near_ - tol || zc - rho > c.far_ + tol) {
            code = kCullDepth;
        } else if (zc - rho > c.near_ + tol && zc + rho < c.far_ - tol && smax < 1e30) {
            const double zl = zc - rho, zh = zc + rho;
            const double xl = xc - rho, xh = xc + rho, yl = yc - rho, yh = yc + rho;
            const double ax = fmax(fabs(xl), fabs(xh)), ay = fmax(fabs(yl), fabs(yh));
            const double jf2 = (c.fx * c.fx + c.fy * c.fy) / (zl * zl) +
                               (c.fx * c.fx * ax * ax + c.fy * c.fy * ay * ay) / (zl * zl * zl * zl);
            const double r = 3.0 * sqrt(jf2 * smax * smax + 0.3) * (1.0 + 1e-9) + 1e-6;
            const double mx_hi = (xh >= 0.0 ? c.fx * xh / zl : c.fx * xh / zh) + c.cx;
            const double mx_lo = (xl <= 0.0 ? c.fx * xl / zl : c.fx * xl / zh) + c.cx;
            const double my_hi = (yh >= 0.0 ? c.fy * yh / zl : c.fy * yh / zh) + c.cy;
            const double my_lo = (yl <= 0.0 ? c.fy * yl / zl : c.fy * yl / zh) + c.cy;
            const double mw = 1e-6 * (1.0 + fabs(mx_hi) + fabs(mx_lo) + fabs(my_hi) + fabs(my_lo));
            if (mx_hi + r < -mw || mx_lo - r > (double)c.width + mw || my_hi + r < -mw ||
                my_lo - r > (double)c.height + mw)
                code = kCullFrame;
            else if (r < 3000.0 && mx_lo > mw && mx_hi < (double)c.width - mw && my_lo > mw &&
                     my_hi < (double)c.height - mw)
                code = kWholeVisible;
        }
    }
    codes[ea] = code;
}

}  // namespace

cudaError_t launch_pose(const sn_avatars &av, const double *sim_times, int32_t n_envs, double *pose_q, double *pose_t,
                        double *joint_mats, double *eff_q, double *root, int32_t *err_flag, cudaStream_t s) {
    int threads = ((av.n_joints + 1 + 31) / 32) * 32;
    pose_kernel<<<n_envs * av.n_avatars, threads, 0, s>>>(av, sim_times, pose_q, pose_t, joint_mats, eff_q, root,
                                                           err_flag);
    return cudaGetLastError();
}

cudaError_t launch_avatar_cull(const sn_avatars &av, const PoseView &pv, const double *pose_t, const sn_camera *cams,
                               int32_t n_envs, unsigned long long *ext, uint8_t *codes, cudaStream_t s) {
    cudaMemsetAsync(ext, 0, sizeof(unsigned long long) * (2 + av.n_joints) * av.n_avatars, s);
    if (av.n > 0)
        avatar_extent_kernel<<<(unsigned)((av.n + 255) / 256), 256, sizeof(unsigned long long) * 2 * (2 + av.n_joints),
                               s>>>(av, ext);
    const int n = n_envs * av.n_avatars;
    avatar_cull_kernel<<<(n + 127) / 128, 128, 0, s>>>(av, pv, pose_t, cams, ext, n_envs, codes);
    return cudaGetLastError();
}

cudaError_t launch_joint_prep(const sn_avatars &av, int32_t avatar, const double *pose_q, const double *pose_t,
                              double *joint_mats, double *eff_q, double *root, cudaStream_t s) {
    int threads = ((av.n_joints + 1 + 31) / 32) * 32;
    joint_prep_kernel<<<1, threads, 0, s>>>(av, avatar, pose_q, pose_t, joint_mats, eff_q, root);
    return cudaGetLastError();
}

}  // namespace sn
