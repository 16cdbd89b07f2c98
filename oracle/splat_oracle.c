/*
 * splat_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A plain-C, float64 restatement of the reference's splat-observation hot path
 * (/root/reference/pkg/src/splatnav, the "splatnav" package). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load
 * this library. The product path (paper_2604_12626_b200) never links or calls it.
 *
 * Every arithmetic step follows the reference's numpy expression order, including the
 * places where numpy hands a contraction to OpenBLAS (which evaluates small matmuls as an
 * FMA chain in k order) and where numpy's einsum uses a pairwise order. Those orders were
 * measured against the reference in this container (tests/golden/make_golden.py pins the
 * result). Compile with -ffp-contract=off: every fused multiply-add below is explicit.
 *
 * The one known ulp-level gap: the reference's numpy exp (AVX-512 SIMD) and this file's
 * libm exp disagree in the last bit for a few percent of arguments. That changes no
 * discrete output (kept set, order, tile lists, contributor counts) on any pinned case;
 * continuous outputs agree to ~1e-15 relative.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_TILE 16

/* projection.py:16-18 */
static const double COV_REGULARIZATION = 0.3;
static const double FOOTPRINT_SIGMA = 3.0;
static const double DEGENERATE_DET = 1e-12;
/* _kernels_cy.pyx:10-12 */
static const double T_CUTOFF = 1e-4;
static const double SUPPORT_D2 = 9.0;
static const double ALPHA_CLIP = 0.99;
/* sh.py:11-15 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* Camera (camera.py:16-48) flattened; layout shared with oracle.py. */
typedef struct {
    double fx, fy, cx, cy, near_, far_;
    double rot[9];    /* world_to_camera[:3,:3], row-major */
    double trans[3];  /* world_to_camera[:3,3] */
    double center[3]; /* Camera.center, computed by the caller exactly as camera.py:43-48 */
    double background[3];
    int32_t width, height, has_background, pad;
} or_camera;

typedef struct {
    int64_t n_input, n_culled_depth, n_culled_frame, n_degenerate, n_drawn;
} or_stats; /* projection.py:30-36 */

/* numpy.maximum(x, 0.0): NaN propagates (unlike fmax). */
static inline double np_max0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }
static inline double np_clip(double x, double lo, double hi) {
    /* np.clip == minimum(maximum(x, lo), hi) with NaN propagation */
    if (x != x) return x;
    if (x < lo) x = lo;
    if (x > hi) x = hi;
    return x;
}

/* transforms.py:17-34 */
static void quat_to_matrix(const double q[4], double m[9]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
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

/* np.linalg.norm over a short last axis: sqrt of a left-to-right sum of squares. */
static inline double norm4(const double q[4]) {
    return sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
}
static inline double norm3(const double v[3]) {
    return sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
}

/* OpenBLAS small gemm element: sum_k a[k]*b[k] as an FMA chain in k order. */
static inline double dot3_fma(double a0, double a1, double a2, double b0, double b1, double b2) {
    return fma(a2, b2, fma(a1, b1, a0 * b0));
}

/* sh.py:20-49 for one splat, float64. coeffs: K x 3 (coefficient-major, channel-minor). */
static void eval_sh(const double *c, int K, const double d[3], double rgb[3]) {
    double x = d[0], y = d[1], z = d[2];
    for (int ch = 0; ch < 3; ++ch) {
        double r = SH_C0 * c[0 * 3 + ch];
        if (K > 1) {
            r = ((r - (SH_C1 * y) * c[1 * 3 + ch]) + (SH_C1 * z) * c[2 * 3 + ch]) - (SH_C1 * x) * c[3 * 3 + ch];
        }
        if (K > 4) {
            double xx = x * x, yy = y * y, zz = z * z;
            double xy = x * y, yz = y * z, xz = x * z;
            r = r + (SH_C2[0] * xy) * c[4 * 3 + ch];
            r = r + (SH_C2[1] * yz) * c[5 * 3 + ch];
            r = r + (SH_C2[2] * ((2.0 * zz - xx) - yy)) * c[6 * 3 + ch];
            r = r + (SH_C2[3] * xz) * c[7 * 3 + ch];
            r = r + (SH_C2[4] * (xx - yy)) * c[8 * 3 + ch];
            if (K > 9) {
                r = r + ((SH_C3[0] * y) * (3.0 * xx - yy)) * c[9 * 3 + ch];
                r = r + ((SH_C3[1] * xy) * z) * c[10 * 3 + ch];
                r = r + ((SH_C3[2] * y) * ((4.0 * zz - xx) - yy)) * c[11 * 3 + ch];
                r = r + ((SH_C3[3] * z) * ((2.0 * zz - 3.0 * xx) - 3.0 * yy)) * c[12 * 3 + ch];
                r = r + ((SH_C3[4] * x) * ((4.0 * zz - xx) - yy)) * c[13 * 3 + ch];
                r = r + ((SH_C3[5] * z) * (xx - yy)) * c[14 * 3 + ch];
                r = r + ((SH_C3[6] * x) * (xx - 3.0 * yy)) * c[15 * 3 + ch];
            }
        }
        r = r + 0.5;
        rgb[ch] = np_clip(r, 0.0, 1.0);
    }
}

typedef struct {
    double z, mx, my, ca, cb, cc, radius, alpha, rgb[3];
} or_splat;

enum { KEEP = 0, CULL_DEPTH = 1, DEGENERATE = 2, CULL_FRAME = 3 };

/* projection.py:100-182 for one gaussian (the vectorized code is elementwise). */
static int project_one(const double p[3], const double ls[3], const double qraw[4], double opacity,
                       const double *sh, int K, const or_camera *cam, or_splat *o) {
    const double *w = cam->rot;
    double cx_ = dot3_fma(p[0], p[1], p[2], w[0], w[1], w[2]) + cam->trans[0];
    double cy_ = dot3_fma(p[0], p[1], p[2], w[3], w[4], w[5]) + cam->trans[1];
    double z = dot3_fma(p[0], p[1], p[2], w[6], w[7], w[8]) + cam->trans[2];
    if (!((z > cam->near_) && (z < cam->far_))) return CULL_DEPTH;

    /* build_cov3d, projection.py:39-51 */
    double s[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double qn = norm4(qraw);
    double q[4] = {qraw[0] / qn, qraw[1] / qn, qraw[2] / qn, qraw[3] / qn};
    double r[9], m[9], cov[9];
    quat_to_matrix(q, r);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m[a * 3 + b] = r[a * 3 + b] * s[b];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            cov[a * 3 + b] = dot3_fma(m[a * 3 + 0], m[a * 3 + 1], m[a * 3 + 2], m[b * 3 + 0], m[b * 3 + 1], m[b * 3 + 2]);

    /* projection.py:137-148 */
    double inv_z = 1.0 / z;
    double j[6] = {cam->fx * inv_z, 0.0, ((-cam->fx) * cx_ * inv_z) * inv_z,
                   0.0, cam->fy * inv_z, ((-cam->fy) * cy_ * inv_z) * inv_z};
    double jw[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            jw[a * 3 + b] = dot3_fma(j[a * 3 + 0], j[a * 3 + 1], j[a * 3 + 2], w[0 * 3 + b], w[1 * 3 + b], w[2 * 3 + b]);
    double t1[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            t1[a * 3 + b] = dot3_fma(jw[a * 3 + 0], jw[a * 3 + 1], jw[a * 3 + 2], cov[0 * 3 + b], cov[1 * 3 + b], cov[2 * 3 + b]);
    double c2[4];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            c2[a * 2 + b] = dot3_fma(t1[a * 3 + 0], t1[a * 3 + 1], t1[a * 3 + 2], jw[b * 3 + 0], jw[b * 3 + 1], jw[b * 3 + 2]);
    double ca = c2[0] + COV_REGULARIZATION;
    double cb = c2[1];
    double cc = c2[3] + COV_REGULARIZATION;
    double det = ca * cc - cb * cb;
    if (!(det > DEGENERATE_DET)) return DEGENERATE;

    double mx = cam->fx * cx_ * inv_z + cam->cx;
    double my = cam->fy * cy_ * inv_z + cam->cy;
    /* _radii_from_cov, projection.py:65-73 */
    double mid = 0.5 * (ca + cc);
    double det2 = ca * cc - cb * cb;
    double lam = mid + sqrt(np_max0(mid * mid - det2));
    double radius = FOOTPRINT_SIGMA * sqrt(np_max0(lam));
    int on_frame = (mx + radius >= 0.0) && (mx - radius <= (double)cam->width) && (my + radius >= 0.0) &&
                   (my - radius <= (double)cam->height);
    if (!on_frame) return CULL_FRAME;

    o->z = z;
    o->mx = mx;
    o->my = my;
    o->ca = cc / det; /* conic = (c, -b, a) / det, projection.py:176 */
    o->cb = (-cb) / det;
    o->cc = ca / det;
    o->radius = radius;
    /* projection.py:178-182 */
    double v[3] = {p[0] - cam->center[0], p[1] - cam->center[1], p[2] - cam->center[2]};
    double nv = norm3(v);
    if (nv == 0.0) nv = 1.0;
    double d[3] = {v[0] / nv, v[1] / nv, v[2] / nv};
    eval_sh(sh, K, d, o->rgb);
    o->alpha = 1.0 / (1.0 + exp(-opacity));
    return KEEP;
}

typedef struct {
    double z;
    int64_t idx;
} zkey;

static int cmp_zkey(const void *a, const void *b) {
    const zkey *x = (const zkey *)a, *y = (const zkey *)b;
    if (x->z < y->z) return -1;
    if (x->z > y->z) return 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

/*
 * project_cloud (projection.py:100-194). Inputs float64, row-major:
 * pos (n,3), log_scales (n,3), rots (n,4), opac (n), sh (n,K,3).
 * Outputs in (depth, index) order, capacity n: means2d (M,2), conics (M,3), depths, colors (M,3),
 * alphas, radii, ids (original index). Returns M.
 */
int64_t or_project(int64_t n, const double *pos, const double *ls, const double *rot, const double *opac,
                   const double *sh, int K, const or_camera *cam, double *means2d, double *conics, double *depths,
                   double *colors, double *alphas, double *radii, int64_t *ids, or_stats *st) {
    or_splat *tmp = (or_splat *)malloc(sizeof(or_splat) * (size_t)(n > 0 ? n : 1));
    zkey *keys = (zkey *)malloc(sizeof(zkey) * (size_t)(n > 0 ? n : 1));
    int64_t m = 0;
    st->n_input += n;
    for (int64_t i = 0; i < n; ++i) {
        or_splat s;
        int r = project_one(pos + 3 * i, ls + 3 * i, rot + 4 * i, opac[i], sh + (size_t)i * K * 3, K, cam, &s);
        if (r == CULL_DEPTH) {
            st->n_culled_depth++;
        } else if (r == DEGENERATE) {
            st->n_degenerate++;
        } else if (r == CULL_FRAME) {
            st->n_culled_frame++;
        } else {
            tmp[i] = s;
            keys[m].z = s.z;
            keys[m].idx = i;
            ++m;
        }
    }
    qsort(keys, (size_t)m, sizeof(zkey), cmp_zkey); /* np.lexsort((idx, z)), projection.py:184 */
    for (int64_t k = 0; k < m; ++k) {
        const or_splat *s = &tmp[keys[k].idx];
        means2d[2 * k] = s->mx;
        means2d[2 * k + 1] = s->my;
        conics[3 * k] = s->ca;
        conics[3 * k + 1] = s->cb;
        conics[3 * k + 2] = s->cc;
        depths[k] = s->z;
        colors[3 * k] = s->rgb[0];
        colors[3 * k + 1] = s->rgb[1];
        colors[3 * k + 2] = s->rgb[2];
        alphas[k] = s->alpha;
        radii[k] = s->radius;
        ids[k] = keys[k].idx;
    }
    st->n_drawn += m;
    free(tmp);
    free(keys);
    return m;
}

/* Per-splat tile rectangle (renderer.py:83-86), inclusive bounds. */
static void tile_rect(double mx, double my, double r, int tiles_x, int tiles_y, int64_t rect[4]) {
    rect[0] = (int64_t)np_clip(floor((mx - r) / OR_TILE), 0.0, (double)(tiles_x - 1));
    rect[1] = (int64_t)np_clip(floor((mx + r) / OR_TILE), 0.0, (double)(tiles_x - 1));
    rect[2] = (int64_t)np_clip(floor((my - r) / OR_TILE), 0.0, (double)(tiles_y - 1));
    rect[3] = (int64_t)np_clip(floor((my + r) / OR_TILE), 0.0, (double)(tiles_y - 1));
}

/* Number of (splat, tile) pairs _bin_tiles will emit. */
int64_t or_count_pairs(int64_t m, const double *means2d, const double *radii, int tiles_x, int tiles_y) {
    int64_t total = 0, rect[4];
    for (int64_t i = 0; i < m; ++i) {
        tile_rect(means2d[2 * i], means2d[2 * i + 1], radii[i], tiles_x, tiles_y, rect);
        total += (rect[1] - rect[0] + 1) * (rect[3] - rect[2] + 1);
    }
    return total;
}

/*
 * _bin_tiles (renderer.py:80-101): stable bucket of depth-ordered splats by tile id.
 * tile_starts: int64[T+1]; pair_splat: int32[P] (indices into the depth-sorted arrays).
 */
void or_bin_tiles(int64_t m, const double *means2d, const double *radii, int tiles_x, int tiles_y,
                  int64_t *tile_starts, int32_t *pair_splat) {
    int64_t n_tiles = (int64_t)tiles_x * tiles_y, rect[4];
    memset(tile_starts, 0, sizeof(int64_t) * (size_t)(n_tiles + 1));
    for (int64_t i = 0; i < m; ++i) {
        tile_rect(means2d[2 * i], means2d[2 * i + 1], radii[i], tiles_x, tiles_y, rect);
        for (int64_t ty = rect[2]; ty <= rect[3]; ++ty)
            for (int64_t tx = rect[0]; tx <= rect[1]; ++tx) tile_starts[ty * tiles_x + tx + 1]++;
    }
    for (int64_t t = 0; t < n_tiles; ++t) tile_starts[t + 1] += tile_starts[t];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_tiles > 0 ? n_tiles : 1));
    memcpy(cursor, tile_starts, sizeof(int64_t) * (size_t)n_tiles);
    for (int64_t i = 0; i < m; ++i) { /* depth order => stable per tile */
        tile_rect(means2d[2 * i], means2d[2 * i + 1], radii[i], tiles_x, tiles_y, rect);
        for (int64_t ty = rect[2]; ty <= rect[3]; ++ty)
            for (int64_t tx = rect[0]; tx <= rect[1]; ++tx) pair_splat[cursor[ty * tiles_x + tx]++] = (int32_t)i;
    }
    free(cursor);
}

/*
 * _kernels_cy._blend (_kernels_cy.pyx:21-86), plus harness-only counters:
 * contrib[px] = splats accumulated (d2 <= 9 while T >= 1e-4), visited[px] = list entries examined.
 * Either counter pointer may be NULL.
 */
void or_blend(int t_begin, int t_end, int tiles_x, int tile_size, int width, int height, const int64_t *tile_starts,
              const int32_t *pair_splat, const double *means2d, const double *conics, const double *depths,
              const double *colors, const double *alphas, double *color_acc, double *alpha_acc, double *trans,
              double *depth_acc, int32_t *contrib, int32_t *visited) {
    for (int t = t_begin; t < t_end; ++t) {
        int64_t s0 = tile_starts[t], s1 = tile_starts[t + 1];
        if (s0 == s1) continue;
        int x0 = (t % tiles_x) * tile_size, y0 = (t / tiles_x) * tile_size;
        int tw = tile_size, th = tile_size;
        if (x0 + tw > width) tw = width - x0;
        if (y0 + th > height) th = height - y0;
        if (tw <= 0 || th <= 0) continue;
        for (int i = 0; i < th; ++i) {
            int py_i = y0 + i;
            double py = py_i + 0.5;
            for (int jx = 0; jx < tw; ++jx) {
                int px_i = x0 + jx;
                double px = px_i + 0.5;
                size_t pix = (size_t)py_i * width + px_i;
                double tcur = 1.0;
                int32_t nc = 0, nv = 0;
                for (int64_t s = s0; s < s1; ++s) {
                    if (tcur < T_CUTOFF) break;
                    ++nv;
                    int32_t sid = pair_splat[s];
                    double dx = means2d[2 * sid] - px;
                    double dy = means2d[2 * sid + 1] - py;
                    double ca = conics[3 * sid], cb = conics[3 * sid + 1], cc = conics[3 * sid + 2];
                    double d2 = ca * dx * dx + 2.0 * cb * dx * dy + cc * dy * dy;
                    if (d2 > SUPPORT_D2) continue;
                    double a = alphas[sid] * exp(-0.5 * d2);
                    if (a > ALPHA_CLIP) a = ALPHA_CLIP;
                    double weight = a * tcur;
                    color_acc[3 * pix + 0] += colors[3 * sid + 0] * weight;
                    color_acc[3 * pix + 1] += colors[3 * sid + 1] * weight;
                    color_acc[3 * pix + 2] += colors[3 * sid + 2] * weight;
                    alpha_acc[pix] += weight;
                    depth_acc[pix] += depths[sid] * weight;
                    tcur *= 1.0 - a;
                    ++nc;
                }
                trans[pix] = tcur;
                if (contrib) contrib[pix] = nc;
                if (visited) visited[pix] = nv;
            }
        }
    }
}

/* _finalize (renderer.py:67-77). background NULL = layer mode. Outputs may alias nothing. */
void or_finalize(int64_t npix, const double *color_acc, const double *alpha_acc, const double *trans,
                 const double *depth_acc, const double *background, double far_, double *color, double *alpha,
                 double *depth) {
    for (int64_t i = 0; i < npix; ++i) {
        double A = alpha_acc[i];
        alpha[i] = A < 1.0 ? A : 1.0;
        for (int c = 0; c < 3; ++c) {
            double v;
            if (background == NULL) {
                double safe = A > 1e-300 ? A : 1e-300;
                v = (A > 0.0) ? color_acc[3 * i + c] / safe : 0.0;
            } else {
                v = color_acc[3 * i + c] + background[c] * trans[i];
            }
            color[3 * i + c] = np_clip(v, 0.0, 1.0);
        }
        double safe = A > 1e-300 ? A : 1e-300;
        depth[i] = (A > 0.0) ? depth_acc[i] / safe : far_;
    }
}

/* composite (renderer.py:151-166), front = avatar layer, back = scene frame; writes out_*. */
void or_composite(int64_t npix, const double *fc, const double *fa, const double *fd, const double *bc,
                  const double *ba, const double *bd, double *oc, double *oa, double *od) {
    for (int64_t i = 0; i < npix; ++i) {
        int use_front = fd[i] < bd[i];
        double a = fa[i];
        for (int c = 0; c < 3; ++c) {
            double blended = fc[3 * i + c] * a + bc[3 * i + c] * (1.0 - a);
            oc[3 * i + c] = use_front ? blended : bc[3 * i + c];
        }
        od[i] = (use_front && (a >= 0.5)) ? fd[i] : bd[i];
        oa[i] = use_front ? a + ba[i] * (1.0 - a) : ba[i];
    }
}

/* ---------------------------------------------------------------- avatar rig (rig.py) */

/* transforms.py:56-70 */
static void quat_multiply(const double a[4], const double b[4], double o[4]) {
    double r0 = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    double r1 = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    double r2 = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    double r3 = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
    o[0] = r0; o[1] = r1; o[2] = r2; o[3] = r3;
}

/* transforms.py:37-53 (Shepperd) on a row-major 3x3 */
static void matrix_to_quat(const double m[9], double q[4]) {
    double t = (m[0] + m[4]) + m[8];
    double s;
    if (t > 0.0) {
        s = sqrt(t + 1.0) * 2.0;
        q[0] = 0.25 * s; q[1] = (m[7] - m[5]) / s; q[2] = (m[2] - m[6]) / s; q[3] = (m[3] - m[1]) / s;
    } else if (m[0] >= m[4] && m[0] >= m[8]) {
        s = sqrt(((1.0 + m[0]) - m[4]) - m[8]) * 2.0;
        q[0] = (m[7] - m[5]) / s; q[1] = 0.25 * s; q[2] = (m[1] + m[3]) / s; q[3] = (m[2] + m[6]) / s;
    } else if (m[4] >= m[8]) {
        s = sqrt(((1.0 + m[4]) - m[0]) - m[8]) * 2.0;
        q[0] = (m[2] - m[6]) / s; q[1] = (m[1] + m[3]) / s; q[2] = 0.25 * s; q[3] = (m[5] + m[7]) / s;
    } else {
        s = sqrt(((1.0 + m[8]) - m[0]) - m[4]) * 2.0;
        q[0] = (m[3] - m[1]) / s; q[1] = (m[2] + m[6]) / s; q[2] = (m[5] + m[7]) / s; q[3] = 0.25 * s;
    }
    double n = norm4(q);
    q[0] /= n; q[1] /= n; q[2] /= n; q[3] /= n;
}

/*
 * sample_pose (rig.py:78-104). traj_q: (T, J+1, 4), traj_t: (T, J+1, 3); root is index J.
 * Writes quats (J+1,4) and trans (J+1,3), root last. Returns 0, or -1 for t < 0.
 */
int or_sample_pose(int n_frames, int n_joints, double fps, const double *traj_q, const double *traj_t, double t,
                   double *out_q, double *out_t) {
    if (t < 0) return -1;
    int jp = n_joints + 1;
    double pos = t * fps;
    double ff = floor(pos);
    int last = n_frames - 1;
    if (ff >= (double)last) {
        memcpy(out_q, traj_q + (size_t)last * jp * 4, sizeof(double) * jp * 4);
        memcpy(out_t, traj_t + (size_t)last * jp * 3, sizeof(double) * jp * 3);
        return 0;
    }
    int f = (int)ff;
    double lam = pos - ff;
    const double *qa = traj_q + (size_t)f * jp * 4, *qb = traj_q + (size_t)(f + 1) * jp * 4;
    const double *ta = traj_t + (size_t)f * jp * 3, *tb = traj_t + (size_t)(f + 1) * jp * 3;
    if (lam == 0.0) {
        memcpy(out_q, qa, sizeof(double) * jp * 4);
        memcpy(out_t, ta, sizeof(double) * jp * 3);
        return 0;
    }
    for (int j = 0; j < jp; ++j) { /* quat_nlerp, transforms.py:73-81 */
        const double *a = qa + 4 * j, *b = qb + 4 * j;
        double dot = ((a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]) + a[3] * b[3];
        double bb[4];
        for (int k = 0; k < 4; ++k) bb[k] = dot < 0.0 ? -b[k] : b[k];
        double q[4];
        for (int k = 0; k < 4; ++k) q[k] = a[k] + lam * (bb[k] - a[k]);
        double n = norm4(q);
        for (int k = 0; k < 4; ++k) out_q[4 * j + k] = q[k] / n;
        for (int k = 0; k < 3; ++k) out_t[3 * j + k] = ta[3 * j + k] + lam * (tb[3 * j + k] - ta[3 * j + k]);
    }
    return 0;
}

/*
 * lbs_deform (rig.py:107-146) with the dense (N, J) float64 weights the reference holds.
 * pose_q (J+1,4) / pose_t (J+1,3), root last; inv_bind (J,4,4) row-major.
 * Outputs positions (N,3) and rotations (N,4), float64.
 */
void or_lbs_deform(int64_t n, int J, const double *pos, const double *rot, const double *weights,
                   const double *inv_bind, const double *pose_q, const double *pose_t, double *out_pos,
                   double *out_rot) {
    double *jm = (double *)malloc(sizeof(double) * 16 * J);
    double *eq = (double *)malloc(sizeof(double) * 4 * J);
    for (int j = 0; j < J; ++j) {
        double r[9], rm[16];
        quat_to_matrix(pose_q + 4 * j, r); /* rigid_matrices, transforms.py:92-101 */
        memset(rm, 0, sizeof(rm));
        for (int a = 0; a < 3; ++a) {
            for (int b = 0; b < 3; ++b) rm[a * 4 + b] = r[a * 3 + b];
            rm[a * 4 + 3] = pose_t[3 * j + a];
        }
        rm[15] = 1.0;
        const double *ib = inv_bind + 16 * j;
        for (int a = 0; a < 4; ++a) /* (J,4,4) @ (J,4,4): BLAS FMA chain over k */
            for (int b = 0; b < 4; ++b)
                jm[16 * j + a * 4 + b] =
                    fma(rm[a * 4 + 3], ib[12 + b], fma(rm[a * 4 + 2], ib[8 + b], fma(rm[a * 4 + 1], ib[4 + b], rm[a * 4 + 0] * ib[b])));
        double m3[9];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) m3[a * 3 + b] = jm[16 * j + a * 4 + b];
        double mq[4];
        matrix_to_quat(m3, mq);
        quat_multiply(pose_q + 4 * J, mq, eq + 4 * j); /* rig.py:127-128 */
    }
    double root_r[9];
    quat_to_matrix(pose_q + 4 * J, root_r);
    const double *root_t = pose_t + 3 * J;
    for (int64_t i = 0; i < n; ++i) {
        const double *p = pos + 3 * i;
        const double *w = weights + (size_t)i * J;
        double acc[3] = {0.0, 0.0, 0.0};
        for (int j = 0; j < J; ++j) {
            const double *M = jm + 16 * j;
            for (int a = 0; a < 3; ++a) {
                /* einsum("jab,nb->jna") measured order: (r0 p0 + r2 p2) + r1 p1, then + offset */
                double tr = (M[a * 4 + 0] * p[0] + M[a * 4 + 2] * p[2]) + M[a * 4 + 1] * p[1];
                tr = tr + M[a * 4 + 3];
                double delta = tr - p[a];
                acc[a] = acc[a] + w[j] * delta; /* einsum("nj,jnc->nc"): sequential, unfused */
            }
        }
        double bl[3] = {p[0] + acc[0], p[1] + acc[1], p[2] + acc[2]};
        for (int a = 0; a < 3; ++a) /* blended @ root_rot.T + root_trans */
            out_pos[3 * i + a] = dot3_fma(bl[0], bl[1], bl[2], root_r[a * 3], root_r[a * 3 + 1], root_r[a * 3 + 2]) + root_t[a];

        int dom = 0; /* np.argmax: first maximum */
        for (int j = 1; j < J; ++j)
            if (w[j] > w[dom]) dom = j;
        const double *qd = eq + 4 * dom;
        double bq[4] = {0.0, 0.0, 0.0, 0.0};
        for (int j = 0; j < J; ++j) {
            const double *qj = eq + 4 * j;
            /* dots = eff @ eff[dom].T: BLAS FMA chain over the 4 components */
            double dot = fma(qj[3], qd[3], fma(qj[2], qd[2], fma(qj[1], qd[1], qj[0] * qd[0])));
            double ws = w[j] * (dot < 0.0 ? -1.0 : 1.0);
            /* (weights * signs) @ eff_quats: BLAS FMA chain over j */
            for (int k = 0; k < 4; ++k) bq[k] = (j == 0) ? ws * qj[k] : fma(ws, qj[k], bq[k]);
        }
        double nb = norm4(bq);
        if (nb < 1e-12) memcpy(bq, qd, sizeof(bq));
        double nn = norm4(bq);
        double qn[4] = {bq[0] / nn, bq[1] / nn, bq[2] / nn, bq[3] / nn};
        quat_multiply(qn, rot + 4 * i, out_rot + 4 * i);
    }
    free(jm);
    free(eq);
}

/* ---------------------------------------------------------------- whole-frame drivers */

typedef struct {
    int64_t n;
    int K;
    const double *pos, *ls, *rot, *opac, *sh;
} or_cloud;

/*
 * rasterize (renderer.py:104-148) for one camera into caller buffers:
 * color (H,W,3), alpha, depth float64; contrib/visited int32 (optional).
 * tiled = 0 reproduces rasterize_reference. Returns number of drawn splats.
 */
int64_t or_rasterize(const or_cloud *c, const or_camera *cam, int tiled, int layer_mode, double *color,
                     double *alpha, double *depth, int32_t *contrib, int32_t *visited, or_stats *st) {
    int64_t n = c->n;
    int W = cam->width, H = cam->height;
    size_t npix = (size_t)W * H;
    int64_t cap = n > 0 ? n : 1;
    double *means2d = malloc(sizeof(double) * 2 * cap), *conics = malloc(sizeof(double) * 3 * cap);
    double *depths = malloc(sizeof(double) * cap), *colors = malloc(sizeof(double) * 3 * cap);
    double *alphas = malloc(sizeof(double) * cap), *radii = malloc(sizeof(double) * cap);
    int64_t *ids = malloc(sizeof(int64_t) * cap);
    double *cacc = calloc(3 * npix, sizeof(double)), *aacc = calloc(npix, sizeof(double));
    double *tr = malloc(sizeof(double) * npix), *dacc = calloc(npix, sizeof(double));
    for (size_t i = 0; i < npix; ++i) tr[i] = 1.0;
    if (contrib) memset(contrib, 0, sizeof(int32_t) * npix);
    if (visited) memset(visited, 0, sizeof(int32_t) * npix);
    int64_t m = or_project(n, c->pos, c->ls, c->rot, c->opac, c->sh, c->K, cam, means2d, conics, depths, colors,
                           alphas, radii, ids, st);
    if (m > 0) {
        if (tiled) {
            int tiles_x = (W + OR_TILE - 1) / OR_TILE, tiles_y = (H + OR_TILE - 1) / OR_TILE;
            int64_t P = or_count_pairs(m, means2d, radii, tiles_x, tiles_y);
            int64_t *ts = malloc(sizeof(int64_t) * ((size_t)tiles_x * tiles_y + 1));
            int32_t *ps = malloc(sizeof(int32_t) * (size_t)(P > 0 ? P : 1));
            or_bin_tiles(m, means2d, radii, tiles_x, tiles_y, ts, ps);
            or_blend(0, tiles_x * tiles_y, tiles_x, OR_TILE, W, H, ts, ps, means2d, conics, depths, colors, alphas,
                     cacc, aacc, tr, dacc, contrib, visited);
            free(ts);
            free(ps);
        } else {
            int64_t ts[2] = {0, m};
            int32_t *ps = malloc(sizeof(int32_t) * (size_t)m);
            for (int64_t i = 0; i < m; ++i) ps[i] = (int32_t)i;
            or_blend(0, 1, 1, W > H ? W : H, W, H, ts, ps, means2d, conics, depths, colors, alphas, cacc, aacc, tr,
                     dacc, contrib, visited);
            free(ps);
        }
    }
    or_finalize((int64_t)npix, cacc, aacc, tr, dacc, layer_mode ? NULL : cam->background, cam->far_, color, alpha,
                depth);
    free(means2d); free(conics); free(depths); free(colors); free(alphas); free(radii); free(ids);
    free(cacc); free(aacc); free(tr); free(dacc);
    return m;
}

/*
 * Batched CPU baseline: E independent environments rendered end to end with render_observation
 * semantics (renderer.py:169-177): scene pass, then (if any avatar cloud is non-empty) one
 * concatenated avatar-layer pass composited over it. Avatar clouds for env e are given already
 * deformed (the caller runs or_lbs_deform per env). Envs are spread over `threads` pthreads.
 */
typedef struct {
    const or_cloud *scene;
    const or_cloud *avatars; /* per env, may have n == 0 */
    const or_camera *cams;
    double *color, *alpha, *depth;
    int E, next_env;
    pthread_mutex_t lock;
} batch_job;

static void render_env(batch_job *b, int e) {
    const or_camera *cam = &b->cams[e];
    size_t npix = (size_t)cam->width * cam->height;
    or_stats st;
    memset(&st, 0, sizeof(st));
    double *c = b->color + 3 * npix * e, *a = b->alpha + npix * e, *d = b->depth + npix * e;
    or_rasterize(b->scene, cam, 1, 0, c, a, d, NULL, NULL, &st);
    if (b->avatars && b->avatars[e].n > 0) {
        double *lc = malloc(sizeof(double) * 3 * npix), *la = malloc(sizeof(double) * npix);
        double *ld = malloc(sizeof(double) * npix);
        or_rasterize(&b->avatars[e], cam, 1, 1, lc, la, ld, NULL, NULL, &st);
        or_composite((int64_t)npix, lc, la, ld, c, a, d, c, a, d);
        free(lc); free(la); free(ld);
    }
}

static void *batch_worker(void *arg) {
    batch_job *b = (batch_job *)arg;
    for (;;) {
        pthread_mutex_lock(&b->lock);
        int e = b->next_env++;
        pthread_mutex_unlock(&b->lock);
        if (e >= b->E) break;
        render_env(b, e);
    }
    return NULL;
}

void or_render_batch(const or_cloud *scene, const or_cloud *avatars_per_env, const or_camera *cams, int E,
                     int threads, double *color, double *alpha, double *depth) {
    batch_job b;
    b.scene = scene; b.avatars = avatars_per_env; b.cams = cams;
    b.color = color; b.alpha = alpha; b.depth = depth;
    b.E = E; b.next_env = 0;
    pthread_mutex_init(&b.lock, NULL);
    if (threads < 1) threads = 1;
    if (threads > E) threads = E;
    pthread_t *tids = malloc(sizeof(pthread_t) * (size_t)(threads > 0 ? threads : 1));
    for (int i = 0; i < threads; ++i) pthread_create(&tids[i], NULL, batch_worker, &b);
    for (int i = 0; i < threads; ++i) pthread_join(tids[i], NULL);
    free(tids);
    pthread_mutex_destroy(&b.lock);
}

int or_abi_version(void) { return 1; }
