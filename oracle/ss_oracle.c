/*
 * ss_oracle.c -- CPU restatement of the 3DSS surface-splatting hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * product path (paper_2605_05876_b200/csrc/ kernels) and the CPU baseline that
 * bench.py reports beside it.  Nothing in the product imports, links or
 * executes it.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.
 *
 * Every function restates the reference algorithm (surfsplat 0.1.0, a
 * CPU-only numpy/numba package) and cites the file:line it follows, with the
 * reference's own mixed precision reproduced operation by operation:
 *   - preprocess is float32 end to end (preprocess.py:231-309); the two
 *     numpy-BLAS product shapes are restated with the FMA chains measured on
 *     the survey host (SURVEY.md §7 hard part 1);
 *   - the rasteriser computes the ray/plane intersection in float32 and
 *     everything downstream of rho^2 in float64 (rasterizer.py:197-224; numba
 *     type promotion of the 2.0 literal);
 *   - shading, the backward kernel, the chain rule and the environment
 *     operators are float64 (shading.py, backward.py).
 * Build with -ffp-contract=off (numba and numpy never contract a*b+c).
 *
 * Parity pin: the tests/golden fixtures were produced by importing the reference
 * itself (tests/golden/make_golden.py) and tests/test_oracle_golden.py checks
 * this file against them.  Two inputs are unpinned at the bit level and are
 * checked with tolerances: numpy's float32 SIMD exp (scales, sigmoids) and
 * BLAS summation order in float64 matmuls.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define DENOM_EPS 1e-9
#define OR_PI 3.141592653589793

/* ------------------------------------------------------------------------- */
/* small helpers                                                              */

static inline float npmaxf(float a, float b) { return (a != a) ? a : (a > b ? a : b); }
static inline double npmax(double a, double b) { return (a != a) ? a : (a > b ? a : b); }
static inline double npclip(double a, double lo, double hi) {
    if (a != a) return a;
    return a < lo ? lo : (a > hi ? hi : a);
}
static inline float npclipf(float a, float lo, float hi) {
    if (a != a) return a;
    return a < lo ? lo : (a > hi ? hi : a);
}
/* float32 exp used where numpy runs its float32 SIMD exp (unpinned at 1 ulp) */
static inline float exp_f32(float x) { return (float)exp((double)x); }
static inline float sigmoid_f32(float x) {
    /* surfels.py:16-23: two-branch stable sigmoid in the input dtype */
    if (x >= 0.0f) return 1.0f / (1.0f + exp_f32(-x));
    float ex = exp_f32(x);
    return ex / (1.0f + ex);
}
static inline long pymod(long a, long m) { long r = a % m; return r < 0 ? r + m : r; }

/* ------------------------------------------------------------------------- */
/* preprocess (preprocess.py:38-309), float32                                  */

/* (N,3)@(3,3): BLAS sgemm inner product, measured as fma(a2,b2,fma(a1,b1,a0*b0)) */
static inline float dot3_gemm(const float a[3], const float b[3]) {
    return fmaf(a[2], b[2], fmaf(a[1], b[1], a[0] * b[0]));
}
/* (N,3)@(3,): BLAS sgemv inner product, measured as fma(a2,v2,fma(a0,v0,a1*v1)) */
static inline float dot3_gemv(const float a[3], const float v[3]) {
    return fmaf(a[2], v[2], fmaf(a[0], v[0], a[1] * v[1]));
}

/* intersect_ray (preprocess.py:108-120) in float32; threshold float32(1e-9)
 * because numpy compares a float32 array with a weak python float. */
static inline int intersect_f32(const float t1[3], const float t2[3], const float t4[3],
                                float x, float y, float *u, float *v) {
    float k0 = x * t4[0] - t1[0], k1 = x * t4[1] - t1[1], k2 = x * t4[2] - t1[2];
    float l0 = y * t4[0] - t2[0], l1 = y * t4[1] - t2[1], l2 = y * t4[2] - t2[2];
    float p0 = k1 * l2 - k2 * l1;
    float p1 = k2 * l0 - k0 * l2;
    float p2 = k0 * l1 - k1 * l0;
    int hit = fabsf(p2) >= (float)DENOM_EPS;
    float safe = hit ? p2 : 1.0f;
    *u = p0 / safe;
    *v = p1 / safe;
    return hit;
}

/* Returns 0, or -1 when any quaternion has zero norm (surfels.py:31-37 raises). */
int or_preprocess(int n, const float *centers, const float *quats, const float *log_scales,
                  const float *albedo_raw, const float *metallic_raw, const float *roughness_raw,
                  const double *view64, const double *proj64, int W, int H,
                  float r_cut, int mip, float mip_sigma,
                  const float *scales_override, /* nullable: (N,2) exp(log_scales) from the host */
                  int8_t *cull, float *t1o, float *t2o, float *t4o, float *view_z, float *eps_z,
                  float *sinv, float *n_f, float *center_ndc, float *jac, uint8_t *jac_ok,
                  int32_t *rect, float *c_cam, float *tu_cam, float *tv_cam)
{
    float view[16], proj[16];
    for (int i = 0; i < 16; ++i) { view[i] = (float)view64[i]; proj[i] = (float)proj64[i]; }
    for (int i = 0; i < n; ++i) {
        const float *q = quats + 4 * i;
        float nrm = sqrtf(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        if (nrm == 0.0f) return -1;
    }
    const float dxp = (float)(1.0 / W), dyp = (float)(1.0 / H);
    const float tiny = FLT_MIN;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        const float *c = centers + 3 * i, *q = quats + 4 * i, *ls = log_scales + 2 * i;
        int finite = 1;
        for (int k = 0; k < 3; ++k) finite &= isfinite(c[k]) && isfinite(albedo_raw[3 * i + k]);
        for (int k = 0; k < 4; ++k) finite &= isfinite(q[k]);
        finite &= isfinite(ls[0]) && isfinite(ls[1]) && isfinite(metallic_raw[i]) && isfinite(roughness_raw[i]);
        int code = finite ? 0 : 1;

        /* quat_to_frame in float32 (surfels.py:40-51) */
        float nrm = sqrtf(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        float w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
        float uh[3] = {1.0f - 2.0f * (y * y + z * z), 2.0f * (x * y + w * z), 2.0f * (x * z - w * y)};
        float vh[3] = {2.0f * (x * y - w * z), 1.0f - 2.0f * (x * x + z * z), 2.0f * (y * z + w * x)};
        float su = scales_override ? scales_override[2 * i] : exp_f32(ls[0]);
        float sv = scales_override ? scales_override[2 * i + 1] : exp_f32(ls[1]);
        float suu[3] = {su * uh[0], su * uh[1], su * uh[2]};
        float svv[3] = {sv * vh[0], sv * vh[1], sv * vh[2]};
        float cc[3], tu[3], tv[3];
        for (int r = 0; r < 3; ++r) {
            const float Rr[3] = {view[4 * r + 0], view[4 * r + 1], view[4 * r + 2]};
            cc[r] = dot3_gemm(c, Rr) + view[4 * r + 3];
            tu[r] = dot3_gemm(suu, Rr);
            tv[r] = dot3_gemm(svv, Rr);
        }
        float vz = -cc[2];
        float rows[3][3];
        const int irs[3] = {0, 1, 3};
        for (int k = 0; k < 3; ++k) {
            const float *Pr = proj + 4 * irs[k];
            rows[k][0] = dot3_gemv(tu, Pr);
            rows[k][1] = dot3_gemv(tv, Pr);
            rows[k][2] = dot3_gemv(cc, Pr) + Pr[3];
        }
        float *t1 = rows[0], *t2 = rows[1], *t4 = rows[2];
        if (code == 0 && !(vz >= 1e-4f)) code = 2;
        int alive = code == 0;
        float ez = r_cut * sqrtf(tu[2] * tu[2] + tv[2] * tv[2]);
        float d4 = t4[2];
        float sd4 = alive ? d4 : 1.0f;
        float cnx = t1[2] / sd4, cny = t2[2] / sd4;

        float j00 = 0, j01 = 0, j10 = 0, j11 = 0;
        int ok = 0;
        float m00 = 1.0f, m01 = 0.0f, m11 = 1.0f, nf = 1.0f;
        float t1b[3], t2b[3], t4b[3];
        if (mip) {
            float cx = t1[2] / t4[2], cy = t2[2] / t4[2];
            float upx, vpx, umx, vmx, upy, vpy, umy, vmy;
            int o0 = intersect_f32(t1, t2, t4, cx + dxp, cy, &upx, &vpx);
            int o1 = intersect_f32(t1, t2, t4, cx - dxp, cy, &umx, &vmx);
            int o2 = intersect_f32(t1, t2, t4, cx, cy + dyp, &upy, &vpy);
            int o3 = intersect_f32(t1, t2, t4, cx, cy - dyp, &umy, &vmy);
            ok = o0 && o1 && o2 && o3;
            if (ok && alive) {
                j00 = upx - umx; j01 = upy - umy; j10 = vpx - vmx; j11 = vpy - vmy;
            }
            float s = mip_sigma;
            float jjt00 = j00 * j00 + j01 * j01;
            float jjt01 = j00 * j10 + j01 * j11;
            float jjt11 = j10 * j10 + j11 * j11;
            float s00 = 1.0f + s * jjt00, s01 = s * jjt01, s11 = 1.0f + s * jjt11;
            float det = s00 * s11 - s01 * s01;
            float inv_det = 1.0f / det;
            m00 = s11 * inv_det; m01 = -s01 * inv_det; m11 = s00 * inv_det;
            nf = sqrtf(inv_det);
            float la = sqrtf(1.0f + s * jjt00);
            float lb = s * jjt01 / la;
            float lc = sqrtf(npmaxf(1.0f + s * jjt11 - lb * lb, tiny));
            const float *src[3] = {t1, t2, t4};
            float *dst[3] = {t1b, t2b, t4b};
            for (int k = 0; k < 3; ++k) {
                dst[k][0] = la * src[k][0] + lb * src[k][1];
                dst[k][1] = lc * src[k][1];
                dst[k][2] = src[k][2];
            }
        } else {
            for (int k = 0; k < 3; ++k) { t1b[k] = t1[k]; t2b[k] = t2[k]; t4b[k] = t4[k]; }
        }
        /* bounding_rect (preprocess.py:77-105) */
        float rr = r_cut * r_cut;
        float f44 = t4b[2] * t4b[2] - rr * (t4b[0] * t4b[0] + t4b[1] * t4b[1]);
        int valid = f44 > 0.0f;
        float f44s = valid ? f44 : 1.0f;
        float ctr[2], half[2];
        const float *ax[2] = {t1b, t2b};
        for (int a = 0; a < 2; ++a) {
            const float *tr = ax[a];
            float fi4 = tr[2] * t4b[2] - rr * (tr[0] * t4b[0] + tr[1] * t4b[1]);
            float fii = tr[2] * tr[2] - rr * (tr[0] * tr[0] + tr[1] * tr[1]);
            float disc = npmaxf(fi4 * fi4 - f44 * fii, 0.0f);
            ctr[a] = fi4 / f44s;
            half[a] = sqrtf(disc) / f44s;
        }
        if (alive && !valid) code = 3;
        alive = code == 0;
        float lo_x = ctr[0] - half[0], hi_x = ctr[0] + half[0];
        float lo_y = ctr[1] - half[1], hi_y = ctr[1] + half[1];
        float fw = (float)W, fh = (float)H;
        float x0 = ceilf((lo_x + 1.0f) * 0.5f * fw - 0.5f - 1e-4f);
        float x1 = floorf((hi_x + 1.0f) * 0.5f * fw - 0.5f + 1e-4f) + 1.0f;
        float y0 = ceilf((1.0f - hi_y) * 0.5f * fh - 0.5f - 1e-4f);
        float y1 = floorf((1.0f - lo_y) * 0.5f * fh - 0.5f + 1e-4f) + 1.0f;
        x0 = npclipf(x0, 0.0f, fw); x1 = npclipf(x1, 0.0f, fw);
        y0 = npclipf(y0, 0.0f, fh); y1 = npclipf(y1, 0.0f, fh);
        if (alive && (x0 >= x1 || y0 >= y1)) code = 4;

        cull[i] = (int8_t)code;
        for (int k = 0; k < 3; ++k) {
            t1o[3 * i + k] = t1[k]; t2o[3 * i + k] = t2[k]; t4o[3 * i + k] = t4[k];
            c_cam[3 * i + k] = cc[k]; tu_cam[3 * i + k] = tu[k]; tv_cam[3 * i + k] = tv[k];
        }
        view_z[i] = vz; eps_z[i] = ez;
        sinv[3 * i] = m00; sinv[3 * i + 1] = m01; sinv[3 * i + 2] = m11; n_f[i] = nf;
        center_ndc[2 * i] = cnx; center_ndc[2 * i + 1] = cny;
        jac[4 * i] = j00; jac[4 * i + 1] = j01; jac[4 * i + 2] = j10; jac[4 * i + 3] = j11;
        jac_ok[i] = (uint8_t)ok;
        if (code == 0) {
            rect[4 * i] = (int32_t)x0; rect[4 * i + 1] = (int32_t)y0;
            rect[4 * i + 2] = (int32_t)x1; rect[4 * i + 3] = (int32_t)y1;
        } else {
            rect[4 * i] = rect[4 * i + 1] = rect[4 * i + 2] = rect[4 * i + 3] = 0;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* bin_and_sort (rasterizer.py:76-116)                                        */

/* Pair count for each record; returns total pairs. */
int64_t or_count_pairs(int nrec, const int32_t *rect, int tile, int64_t *counts)
{
    int64_t tot = 0;
    for (int i = 0; i < nrec; ++i) {
        const int32_t *r = rect + 4 * i;
        int64_t sx = (r[2] - 1) / tile - r[0] / tile + 1;
        int64_t sy = (r[3] - 1) / tile - r[1] / tile + 1;
        counts[i] = sx * sy;
        tot += counts[i];
    }
    return tot;
}

typedef struct { int64_t tile; float z; int32_t rec; } OrPair;

static int cmp_pair(const void *a, const void *b) {
    const OrPair *x = (const OrPair *)a, *y = (const OrPair *)b;
    if (x->tile != y->tile) return x->tile < y->tile ? -1 : 1;
    /* lexsort on float32 keys: -0.0 == +0.0, ties broken by record index */
    if (x->z < y->z) return -1;
    if (x->z > y->z) return 1;
    return x->rec < y->rec ? -1 : (x->rec > y->rec ? 1 : 0);
}

/* Emit pairs record-major / row-major (rasterizer.py:76-89), then order by
 * (tile, z_start, record) as np.lexsort does (rasterizer.py:111). */
void or_bin_sort(int nrec, const int32_t *rect, const float *z_start, int W, int H, int tile,
                 int64_t total, int64_t *tile_offsets, int32_t *pair_rec)
{
    int ntx = (W + tile - 1) / tile, nty = (H + tile - 1) / tile;
    int ntiles = ntx * nty;
    OrPair *pairs = (OrPair *)malloc(sizeof(OrPair) * (total > 0 ? total : 1));
    int64_t pos = 0;
    for (int i = 0; i < nrec; ++i) {
        const int32_t *r = rect + 4 * i;
        int tx0 = r[0] / tile, ty0 = r[1] / tile, tx1 = (r[2] - 1) / tile, ty1 = (r[3] - 1) / tile;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) {
                pairs[pos].tile = (int64_t)ty * ntx + tx;
                pairs[pos].z = z_start[i];
                pairs[pos].rec = i;
                ++pos;
            }
    }
    qsort(pairs, (size_t)total, sizeof(OrPair), cmp_pair);
    memset(tile_offsets, 0, sizeof(int64_t) * (ntiles + 1));
    for (int64_t p = 0; p < total; ++p) { pair_rec[p] = pairs[p].rec; tile_offsets[pairs[p].tile + 1]++; }
    for (int t = 0; t < ntiles; ++t) tile_offsets[t + 1] += tile_offsets[t];
    free(pairs);
}

/* ------------------------------------------------------------------------- */
/* forward kernel, interval mode (rasterizer.py:119-249)                       */

typedef struct {
    const float *t1, *t2, *t4, *sinv, *n_f, *view_z, *z_start, *z_end, *colors;
    const int32_t *rect;
} OrRecords;

/* numba promotion: the fp32 products s0*u*u and s2*v*v stay float, the 2.0
 * literal lifts the cross term and the sum to float64 (rasterizer.py:208). */
static inline double rho2_mixed(const float *s, float u, float v) {
    float a = s[0] * u * u;
    double b = 2.0 * (double)s[1] * (double)u * (double)v;
    float c = s[2] * v * v;
    return ((double)a + b) + (double)c;
}

void or_forward(int W, int H, int tile, const int64_t *tile_offsets, const int32_t *pair_rec,
                const float *t1, const float *t2, const float *t4, const float *sinv, const float *n_f,
                const float *view_z, const float *z_start, const float *z_end, const int32_t *rect,
                const float *colors, const float *bg, int k_max,
                float *rgb, float *alpha, float *depth, int32_t *nlayers,
                int64_t *pair_cover, /* nullable, per pair */
                float *st_w, float *st_c, float *st_z, float *st_z2, int32_t *st_n, /* nullable, (H,W,k_max[,3]) */
                int64_t *tile_discarded)
{
    int ntx = (W + tile - 1) / tile, nty = (H + tile - 1) / tile;
    int ntiles = ntx * nty;
    const double r_cut2 = 9.0, rate = 1.0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < ntiles; ++t) {
        int64_t p0 = tile_offsets[t], p1 = tile_offsets[t + 1];
        tile_discarded[t] = 0;
        int tx = t % ntx, ty = t / ntx;
        int x_lo = tx * tile, y_lo = ty * tile;
        int x_hi = x_lo + tile < W ? x_lo + tile : W, y_hi = y_lo + tile < H ? y_lo + tile : H;
        for (int iy = y_lo; iy < y_hi; ++iy) {
            float y = (float)(1.0 - ((double)iy + 0.5) * (2.0 / H));
            for (int ix = x_lo; ix < x_hi; ++ix) {
                float x = (float)(((double)ix + 0.5) * (2.0 / W) - 1.0);
                int pix = iy * W + ix;
                rgb[3 * pix] = bg[0]; rgb[3 * pix + 1] = bg[1]; rgb[3 * pix + 2] = bg[2];
                alpha[pix] = 0.0f; depth[pix] = 0.0f; nlayers[pix] = 0;
                double w_g = 0, c0 = 0, c1 = 0, c2 = 0, z_g = 0, z2_g = 0, z_max_end = 0;
                int layers = 0, stopped = 0;
                double trans = 1.0, o0 = 0, o1 = 0, o2 = 0, d_num = 0, d_den = 0;
                for (int64_t p = p0; p < p1; ++p) {
                    int r = pair_rec[p];
                    const int32_t *rc = rect + 4 * r;
                    if (ix < rc[0] || ix >= rc[2] || iy < rc[1] || iy >= rc[3]) continue;
                    if (stopped) { tile_discarded[t]++; continue; }
                    if (w_g > 0.0 && (double)z_start[r] > z_max_end) {
                        double a_k = 1.0 - exp(-w_g * rate);
                        double inv_w = 1.0 / w_g;
                        o0 += trans * a_k * c0 * inv_w;
                        o1 += trans * a_k * c1 * inv_w;
                        o2 += trans * a_k * c2 * inv_w;
                        d_num += trans * a_k * z_g * inv_w;
                        d_den += trans * a_k;
                        trans *= 1.0 - a_k;
                        if (st_w) {
                            size_t o = (size_t)pix * k_max + layers;
                            st_w[o] = (float)w_g; st_c[3 * o] = (float)c0; st_c[3 * o + 1] = (float)c1;
                            st_c[3 * o + 2] = (float)c2; st_z[o] = (float)z_g; st_z2[o] = (float)z2_g;
                        }
                        layers += 1;
                        w_g = c0 = c1 = c2 = z_g = z2_g = z_max_end = 0.0;
                        if (layers >= k_max) { stopped = 1; tile_discarded[t]++; continue; }
                    }
                    const float *a1 = t1 + 3 * r, *a2 = t2 + 3 * r, *a4 = t4 + 3 * r;
                    float k0 = x * a4[0] - a1[0], k1 = x * a4[1] - a1[1], k2 = x * a4[2] - a1[2];
                    float l0 = y * a4[0] - a2[0], l1 = y * a4[1] - a2[1], l2 = y * a4[2] - a2[2];
                    float den = k0 * l1 - k1 * l0;
                    if (fabs((double)den) < DENOM_EPS) continue;
                    float u = (k1 * l2 - k2 * l1) / den;
                    float v = (k2 * l0 - k0 * l2) / den;
                    double rho2 = rho2_mixed(sinv + 3 * r, u, v);
                    if (rho2 >= r_cut2) continue;
                    if (pair_cover) pair_cover[p] += 1;
                    double w = (double)n_f[r] * exp(-0.5 * rho2);
                    double z = (double)view_z[r];
                    w_g += w;
                    c0 += w * (double)colors[3 * r];
                    c1 += w * (double)colors[3 * r + 1];
                    c2 += w * (double)colors[3 * r + 2];
                    z_g += w * z;
                    z2_g += w * z * z;
                    if (st_n && layers < k_max) st_n[(size_t)pix * k_max + layers] += 1;
                    if ((double)z_end[r] > z_max_end) z_max_end = (double)z_end[r];
                }
                if (w_g > 0.0) {
                    double a_k = 1.0 - exp(-w_g * rate);
                    double inv_w = 1.0 / w_g;
                    o0 += trans * a_k * c0 * inv_w;
                    o1 += trans * a_k * c1 * inv_w;
                    o2 += trans * a_k * c2 * inv_w;
                    d_num += trans * a_k * z_g * inv_w;
                    d_den += trans * a_k;
                    trans *= 1.0 - a_k;
                    if (st_w) {
                        size_t o = (size_t)pix * k_max + layers;
                        st_w[o] = (float)w_g; st_c[3 * o] = (float)c0; st_c[3 * o + 1] = (float)c1;
                        st_c[3 * o + 2] = (float)c2; st_z[o] = (float)z_g; st_z2[o] = (float)z2_g;
                    }
                    layers += 1;
                }
                if (layers > 0) {
                    rgb[3 * pix] = (float)(o0 + trans * (double)bg[0]);
                    rgb[3 * pix + 1] = (float)(o1 + trans * (double)bg[1]);
                    rgb[3 * pix + 2] = (float)(o2 + trans * (double)bg[2]);
                    alpha[pix] = (float)(1.0 - trans);
                    if (d_den > 0.0) depth[pix] = (float)(d_num / d_den);
                    nlayers[pix] = layers;
                }
            }
        }
    }
}

/* ------------------------------------------------------------------------- */
/* backward kernel (backward.py:48-321) + fixed-order reduction (:382-396)     */

#define KMAXCAP 64

void or_backward_pairs(int W, int H, int tile, const int64_t *tile_offsets, const int32_t *pair_rec,
                       const float *t1, const float *t2, const float *t4, const float *sinv,
                       const float *n_f, const float *view_z, const float *z_start, const float *z_end,
                       const int32_t *rect, const float *colors, const float *bg, int k_max,
                       const double *g_rgb, const double *g_alpha, double cons_scale,
                       double *pb /* P x 17 */, double *ss /* P */, int64_t *touch /* P */,
                       double *cons_out /* ntiles */)
{
    int ntx = (W + tile - 1) / tile, nty = (H + tile - 1) / tile;
    int ntiles = ntx * nty;
    const double r_cut2 = 9.0, rate = 1.0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < ntiles; ++t) {
        int64_t pa = tile_offsets[t], pz = tile_offsets[t + 1];
        cons_out[t] = 0.0;
        if (pa == pz) continue;
        double lw[KMAXCAP], lc[KMAXCAP][3], lz[KMAXCAP], lz2[KMAXCAP], a_arr[KMAXCAP], tbar[KMAXCAP];
        double wm[KMAXCAP], zb_a[KMAXCAP], var_a[KMAXCAP], gw_c[KMAXCAP], gz_c[KMAXCAP], gv_c[KMAXCAP];
        double g_wtot[KMAXCAP], g_craw[KMAXCAP][3], g_zc[KMAXCAP], g_z2c[KMAXCAP];
        double cons_local = 0.0;
        int tx = t % ntx, ty = t / ntx;
        int x_lo = tx * tile, y_lo = ty * tile;
        int x_hi = x_lo + tile < W ? x_lo + tile : W, y_hi = y_lo + tile < H ? y_lo + tile : H;
        for (int iy = y_lo; iy < y_hi; ++iy) {
            float y = (float)(1.0 - ((double)iy + 0.5) * (2.0 / H));
            for (int ix = x_lo; ix < x_hi; ++ix) {
                float x = (float)(((double)ix + 0.5) * (2.0 / W) - 1.0);
                int pix = iy * W + ix;
                int nl = 0, stopped = 0;
                double w_g = 0, c0 = 0, c1 = 0, c2 = 0, z_g = 0, z2_g = 0, z_max_end = 0;
                for (int64_t p = pa; p < pz; ++p) {
                    int r = pair_rec[p];
                    const int32_t *rc = rect + 4 * r;
                    if (ix < rc[0] || ix >= rc[2] || iy < rc[1] || iy >= rc[3]) continue;
                    if (stopped) continue;
                    if (w_g > 0.0 && (double)z_start[r] > z_max_end) {
                        lw[nl] = w_g; lc[nl][0] = c0; lc[nl][1] = c1; lc[nl][2] = c2;
                        lz[nl] = z_g; lz2[nl] = z2_g; nl += 1;
                        w_g = c0 = c1 = c2 = z_g = z2_g = z_max_end = 0.0;
                        if (nl >= k_max) { stopped = 1; continue; }
                    }
                    const float *a1 = t1 + 3 * r, *a2 = t2 + 3 * r, *a4 = t4 + 3 * r;
                    float k0 = x * a4[0] - a1[0], k1 = x * a4[1] - a1[1], k2 = x * a4[2] - a1[2];
                    float l0 = y * a4[0] - a2[0], l1 = y * a4[1] - a2[1], l2 = y * a4[2] - a2[2];
                    float den = k0 * l1 - k1 * l0;
                    if (fabs((double)den) < DENOM_EPS) continue;
                    float u = (k1 * l2 - k2 * l1) / den;
                    float v = (k2 * l0 - k0 * l2) / den;
                    double rho2 = rho2_mixed(sinv + 3 * r, u, v);
                    if (rho2 >= r_cut2) continue;
                    double w = (double)n_f[r] * exp(-0.5 * rho2);
                    double z = (double)view_z[r];
                    w_g += w;
                    c0 += w * (double)colors[3 * r];
                    c1 += w * (double)colors[3 * r + 1];
                    c2 += w * (double)colors[3 * r + 2];
                    z_g += w * z;
                    z2_g += w * z * z;
                    if ((double)z_end[r] > z_max_end) z_max_end = (double)z_end[r];
                }
                if (w_g > 0.0) {
                    lw[nl] = w_g; lc[nl][0] = c0; lc[nl][1] = c1; lc[nl][2] = c2;
                    lz[nl] = z_g; lz2[nl] = z2_g; nl += 1;
                }
                if (nl == 0) continue;
                double trans = 1.0;
                for (int m = 0; m < nl; ++m) {
                    a_arr[m] = 1.0 - exp(-lw[m] * rate);
                    tbar[m] = trans;
                    trans *= 1.0 - a_arr[m];
                }
                for (int m = 0; m < nl; ++m) gw_c[m] = gz_c[m] = gv_c[m] = 0.0;
                if (cons_scale > 0.0) {
                    for (int m = 0; m < nl; ++m) {
                        wm[m] = tbar[m] * a_arr[m];
                        double inv_w = 1.0 / lw[m];
                        double zb = lz[m] * inv_w;
                        double v_raw = lz2[m] * inv_w - zb * zb;
                        zb_a[m] = zb;
                        var_a[m] = v_raw > 0.0 ? v_raw : 0.0;
                        gv_c[m] = v_raw > 0.0 ? cons_scale * wm[m] * wm[m] : 0.0;
                    }
                    double l_pix = 0.0;
                    for (int i = 0; i < nl; ++i) {
                        l_pix += wm[i] * wm[i] * var_a[i];
                        gw_c[i] += cons_scale * 2.0 * wm[i] * var_a[i];
                        for (int j = i + 1; j < nl; ++j) {
                            double dz = zb_a[i] - zb_a[j];
                            double adz = fabs(dz);
                            l_pix += wm[i] * wm[j] * adz;
                            gw_c[i] += cons_scale * wm[j] * adz;
                            gw_c[j] += cons_scale * wm[i] * adz;
                            double sgn = dz > 0.0 ? 1.0 : (dz < 0.0 ? -1.0 : 0.0);
                            gz_c[i] += cons_scale * wm[i] * wm[j] * sgn;
                            gz_c[j] -= cons_scale * wm[i] * wm[j] * sgn;
                        }
                    }
                    cons_local += cons_scale * l_pix;
                }
                double gc0 = g_rgb[3 * pix], gc1 = g_rgb[3 * pix + 1], gc2 = g_rgb[3 * pix + 2];
                double ga = g_alpha[pix];
                double sfx0 = bg[0], sfx1 = bg[1], sfx2 = bg[2], q_sfx = 1.0, rw_sfx = 0.0;
                for (int m = nl - 1; m >= 0; --m) {
                    double inv_w = 1.0 / lw[m];
                    double ch0 = lc[m][0] * inv_w, ch1 = lc[m][1] * inv_w, ch2 = lc[m][2] * inv_w;
                    double zb = lz[m] * inv_w;
                    double v_raw = lz2[m] * inv_w - zb * zb;
                    double g_alpha_m = tbar[m] * (gc0 * (ch0 - sfx0) + gc1 * (ch1 - sfx1)
                                                  + gc2 * (ch2 - sfx2)
                                                  + ga * q_sfx + gw_c[m] - rw_sfx);
                    double gch0 = gc0 * tbar[m] * a_arr[m];
                    double gch1 = gc1 * tbar[m] * a_arr[m];
                    double gch2 = gc2 * tbar[m] * a_arr[m];
                    double g_w = g_alpha_m * rate * (1.0 - a_arr[m]);
                    g_w -= (gch0 * ch0 + gch1 * ch1 + gch2 * ch2) * inv_w;
                    g_w -= gz_c[m] * zb * inv_w;
                    g_w += gv_c[m] * (zb * zb - v_raw) * inv_w;
                    g_wtot[m] = g_w;
                    g_craw[m][0] = gch0 * inv_w; g_craw[m][1] = gch1 * inv_w; g_craw[m][2] = gch2 * inv_w;
                    g_zc[m] = gz_c[m] * inv_w - 2.0 * gv_c[m] * zb * inv_w;
                    g_z2c[m] = gv_c[m] * inv_w;
                    sfx0 = a_arr[m] * ch0 + (1.0 - a_arr[m]) * sfx0;
                    sfx1 = a_arr[m] * ch1 + (1.0 - a_arr[m]) * sfx1;
                    sfx2 = a_arr[m] * ch2 + (1.0 - a_arr[m]) * sfx2;
                    q_sfx *= 1.0 - a_arr[m];
                    rw_sfx = gw_c[m] * a_arr[m] + (1.0 - a_arr[m]) * rw_sfx;
                }
                int m_cur = 0, group_n = 0;
                z_max_end = 0.0;
                stopped = 0;
                for (int64_t p = pa; p < pz; ++p) {
                    int r = pair_rec[p];
                    const int32_t *rc = rect + 4 * r;
                    if (ix < rc[0] || ix >= rc[2] || iy < rc[1] || iy >= rc[3]) continue;
                    if (stopped) continue;
                    if (group_n > 0 && (double)z_start[r] > z_max_end) {
                        m_cur += 1; group_n = 0; z_max_end = 0.0;
                        if (m_cur >= k_max) { stopped = 1; continue; }
                    }
                    const float *a1 = t1 + 3 * r, *a2 = t2 + 3 * r, *a4 = t4 + 3 * r;
                    float k0 = x * a4[0] - a1[0], k1 = x * a4[1] - a1[1], k2 = x * a4[2] - a1[2];
                    float l0 = y * a4[0] - a2[0], l1 = y * a4[1] - a2[1], l2 = y * a4[2] - a2[2];
                    float den = k0 * l1 - k1 * l0;
                    if (fabs((double)den) < DENOM_EPS) continue;
                    float u = (k1 * l2 - k2 * l1) / den;
                    float v = (k2 * l0 - k0 * l2) / den;
                    const float *s = sinv + 3 * r;
                    double rho2 = rho2_mixed(s, u, v);
                    if (rho2 >= r_cut2) continue;
                    double w = (double)n_f[r] * exp(-0.5 * rho2);
                    double z = (double)view_z[r];
                    group_n += 1;
                    if ((double)z_end[r] > z_max_end) z_max_end = (double)z_end[r];
                    const float *col = colors + 3 * r;
                    double g_w = (g_wtot[m_cur] + g_craw[m_cur][0] * (double)col[0]
                                  + g_craw[m_cur][1] * (double)col[1]
                                  + g_craw[m_cur][2] * (double)col[2]
                                  + g_zc[m_cur] * z + g_z2c[m_cur] * z * z);
                    double *b = pb + 17 * p;
                    b[13] += w * g_craw[m_cur][0];
                    b[14] += w * g_craw[m_cur][1];
                    b[15] += w * g_craw[m_cur][2];
                    b[16] += w * (g_zc[m_cur] + 2.0 * z * g_z2c[m_cur]);
                    double g_rho2 = -0.5 * w * g_w;
                    b[12] += exp(-0.5 * rho2) * g_w;
                    double du = u, dv = v;
                    b[9] += g_rho2 * du * du;
                    b[10] += g_rho2 * 2.0 * du * dv;
                    b[11] += g_rho2 * dv * dv;
                    /* the inner sums are float32 in numba (backward.py:293-294) */
                    double g_u = g_rho2 * 2.0 * (double)(s[0] * u + s[1] * v);
                    double g_v = g_rho2 * 2.0 * (double)(s[1] * u + s[2] * v);
                    double dden = den;
                    double gp0 = g_u / dden, gp1 = g_v / dden, gp2 = -(g_u * du + g_v * dv) / dden;
                    double K0 = k0, K1 = k1, K2 = k2, L0 = l0, L1 = l1, L2 = l2;
                    double gk0 = L1 * gp2 - L2 * gp1;
                    double gk1 = L2 * gp0 - L0 * gp2;
                    double gk2 = L0 * gp1 - L1 * gp0;
                    double gl0 = gp1 * K2 - gp2 * K1;
                    double gl1 = gp2 * K0 - gp0 * K2;
                    double gl2 = gp0 * K1 - gp1 * K0;
                    b[0] -= gk0; b[1] -= gk1; b[2] -= gk2;
                    b[3] -= gl0; b[4] -= gl1; b[5] -= gl2;
                    double X = x, Y = y;
                    b[6] += X * gk0 + Y * gl0;
                    b[7] += X * gk1 + Y * gl1;
                    b[8] += X * gk2 + Y * gl2;
                    double gsx = -gk2 * (double)a4[2];
                    double gsy = -gl2 * (double)a4[2];
                    ss[p] += sqrt(gsx * gsx + gsy * gsy);
                    touch[p] += 1;
                }
            }
        }
        cons_out[t] = cons_local;
    }
}

/* serial fixed-order reduction: np.bincount(pair_rec, weights) (backward.py:382-388) */
void or_reduce_pairs(int64_t npairs, int nrec, const int32_t *pair_rec, const double *pb,
                     const double *ss, const int64_t *touch,
                     double *merged /* nrec x 17 */, double *ss_rec, double *touch_rec)
{
    memset(merged, 0, sizeof(double) * 17 * (size_t)nrec);
    memset(ss_rec, 0, sizeof(double) * (size_t)nrec);
    memset(touch_rec, 0, sizeof(double) * (size_t)nrec);
    for (int c = 0; c < 17; ++c)
        for (int64_t p = 0; p < npairs; ++p) merged[17 * (size_t)pair_rec[p] + c] += pb[17 * p + c];
    for (int64_t p = 0; p < npairs; ++p) {
        ss_rec[pair_rec[p]] += ss[p];
        touch_rec[pair_rec[p]] += (double)touch[p];
    }
}

/* ------------------------------------------------------------------------- */
/* MIP chain backward (backward.py:473-548), float64, in place on g_t rows     */

void or_mip_chain_backward(int nrec, int W, int H, double sigma, const float *jac, const uint8_t *jac_ok,
                           const float *t1f, const float *t2f, const float *t4f,
                           const double *g_sinv, const double *g_nf,
                           double *g_t1, double *g_t2, double *g_t4)
{
    const double dx = 1.0 / W, dy = 1.0 / H;
    for (int i = 0; i < nrec; ++i) {
        double j00 = jac[4 * i], j01 = jac[4 * i + 1], j10 = jac[4 * i + 2], j11 = jac[4 * i + 3];
        double s00 = 1.0 + sigma * (j00 * j00 + j01 * j01);
        double s01 = sigma * (j00 * j10 + j01 * j11);
        double s11 = 1.0 + sigma * (j10 * j10 + j11 * j11);
        double det = s00 * s11 - s01 * s01;
        double b00 = s11 / det, b01 = -s01 / det, b11 = s00 / det;
        double nf = 1.0 / sqrt(det);
        double g00 = g_sinv[3 * i], g01 = 0.5 * g_sinv[3 * i + 1], g11 = g_sinv[3 * i + 2];
        double bg00 = b00 * g00 + b01 * g01, bg01 = b00 * g01 + b01 * g11;
        double bg10 = b01 * g00 + b11 * g01, bg11 = b01 * g01 + b11 * g11;
        double gnf = g_nf[i];
        double ga00 = -(bg00 * b00 + bg01 * b01) - 0.5 * gnf * nf * b00;
        double ga01 = -(bg00 * b01 + bg01 * b11) - 0.5 * gnf * nf * b01;
        double ga11 = -(bg10 * b01 + bg11 * b11) - 0.5 * gnf * nf * b11;
        double two_s = 2.0 * sigma;
        double live = jac_ok[i] ? 1.0 : 0.0;
        double gj00 = two_s * (ga00 * j00 + ga01 * j10) * live;
        double gj01 = two_s * (ga00 * j01 + ga01 * j11) * live;
        double gj10 = two_s * (ga01 * j00 + ga11 * j10) * live;
        double gj11 = two_s * (ga01 * j01 + ga11 * j11) * live;
        double T1[3] = {t1f[3 * i], t1f[3 * i + 1], t1f[3 * i + 2]};
        double T2[3] = {t2f[3 * i], t2f[3 * i + 1], t2f[3 * i + 2]};
        double T4[3] = {t4f[3 * i], t4f[3 * i + 1], t4f[3 * i + 2]};
        double d4 = T4[2], cx = T1[2] / d4, cy = T2[2] / d4;
        double gcx = 0.0, gcy = 0.0;
        double probes[4][4] = {{cx + dx, cy, gj00, gj10}, {cx - dx, cy, -gj00, -gj10},
                               {cx, cy + dy, gj01, gj11}, {cx, cy - dy, -gj01, -gj11}};
        double *G1 = g_t1 + 3 * i, *G2 = g_t2 + 3 * i, *G4 = g_t4 + 3 * i;
        for (int pi = 0; pi < 4; ++pi) {
            double px = probes[pi][0], py = probes[pi][1];
            double k[3], l[3];
            for (int c = 0; c < 3; ++c) { k[c] = px * T4[c] - T1[c]; l[c] = py * T4[c] - T2[c]; }
            double p0 = k[1] * l[2] - k[2] * l[1];
            double p1 = k[2] * l[0] - k[0] * l[2];
            double den = k[0] * l[1] - k[1] * l[0];
            int hit = fabs(den) >= DENOM_EPS;
            double safe = hit ? den : 1.0;
            double u = p0 / safe, v = p1 / safe;
            double gu = (hit && jac_ok[i]) ? probes[pi][2] : 0.0;
            double gv = (hit && jac_ok[i]) ? probes[pi][3] : 0.0;
            double gp[3] = {gu / safe, gv / safe, -(gu * u + gv * v) / safe};
            double gk[3] = {l[1] * gp[2] - l[2] * gp[1], l[2] * gp[0] - l[0] * gp[2], l[0] * gp[1] - l[1] * gp[0]};
            double gl[3] = {gp[1] * k[2] - gp[2] * k[1], gp[2] * k[0] - gp[0] * k[2], gp[0] * k[1] - gp[1] * k[0]};
            for (int c = 0; c < 3; ++c) {
                G1[c] -= gk[c];
                G2[c] -= gl[c];
                G4[c] += px * gk[c] + py * gl[c];
            }
            gcx += (gk[0] * T4[0] + gk[1] * T4[1]) + gk[2] * T4[2];
            gcy += (gl[0] * T4[0] + gl[1] * T4[1]) + gl[2] * T4[2];
        }
        G1[2] += gcx / d4;
        G4[2] -= gcx * cx / d4;
        G2[2] += gcy / d4;
        G4[2] -= gcy * cy / d4;
    }
}

/* T rows -> camera -> world (backward.py:405-441); float64.  Outputs per record. */
void or_rows_to_world(int nrec, const double *view64, const double *proj64,
                      const double *g_t1, const double *g_t2, const double *g_t4, const double *g_z,
                      const double *quats64_src /* nrec x 4 */, const double *log_scales_src /* nrec x 2 */,
                      double *g_centers, double *g_log_scales, double *g_u_hat, double *g_v_hat)
{
    const double *pm = proj64;
    for (int i = 0; i < nrec; ++i) {
        double gtu[3], gtv[3], gcc[3];
        for (int c = 0; c < 3; ++c) {
            gtu[c] = g_t1[3 * i] * pm[c] + g_t2[3 * i] * pm[4 + c] + g_t4[3 * i] * pm[12 + c];
            gtv[c] = g_t1[3 * i + 1] * pm[c] + g_t2[3 * i + 1] * pm[4 + c] + g_t4[3 * i + 1] * pm[12 + c];
            gcc[c] = g_t1[3 * i + 2] * pm[c] + g_t2[3 * i + 2] * pm[4 + c] + g_t4[3 * i + 2] * pm[12 + c];
        }
        gcc[2] -= g_z[i];
        double gw[3], guw[3], gvw[3];
        for (int k = 0; k < 3; ++k) {
            gw[k] = (gcc[0] * view64[k] + gcc[1] * view64[4 + k]) + gcc[2] * view64[8 + k];
            guw[k] = (gtu[0] * view64[k] + gtu[1] * view64[4 + k]) + gtu[2] * view64[8 + k];
            gvw[k] = (gtv[0] * view64[k] + gtv[1] * view64[4 + k]) + gtv[2] * view64[8 + k];
        }
        const double *q = quats64_src + 4 * i;
        double nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
        double uh[3] = {1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)};
        double vh[3] = {2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)};
        double su = exp(log_scales_src[2 * i]), sv = exp(log_scales_src[2 * i + 1]);
        double gsu = (guw[0] * uh[0] + guw[1] * uh[1]) + guw[2] * uh[2];
        double gsv = (gvw[0] * vh[0] + gvw[1] * vh[1]) + gvw[2] * vh[2];
        for (int k = 0; k < 3; ++k) {
            g_centers[3 * i + k] = gw[k];
            g_u_hat[3 * i + k] = su * guw[k];
            g_v_hat[3 * i + k] = sv * gvw[k];
        }
        g_log_scales[2 * i] = gsu * su;
        g_log_scales[2 * i + 1] = gsv * sv;
    }
}

/* quat_frame_backward (surfels.py:54-77), float64 */
void or_quat_frame_backward(int n, const double *quats, const double *gu, const double *gv,
                            const double *gn, double *g_out)
{
    for (int i = 0; i < n; ++i) {
        const double *q = quats + 4 * i;
        double nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
        const double *U = gu + 3 * i, *V = gv + 3 * i, *N = gn + 3 * i;
#define D3(g, a0, a1, a2) ((g)[0] * (a0) + (g)[1] * (a1) + (g)[2] * (a2))
        double gw = D3(U, 0.0, 2 * z, -2 * y) + D3(V, -2 * z, 0.0, 2 * x) + D3(N, 2 * y, -2 * x, 0.0);
        double gx = D3(U, 0.0, 2 * y, 2 * z) + D3(V, 2 * y, -4 * x, 2 * w) + D3(N, 2 * z, -2 * w, -4 * x);
        double gy = D3(U, -4 * y, 2 * x, -2 * w) + D3(V, 2 * x, 0.0, 2 * z) + D3(N, 2 * w, 2 * z, -4 * y);
        double gz = D3(U, -4 * z, 2 * w, 2 * x) + D3(V, -2 * w, -4 * z, 2 * y) + D3(N, 2 * x, 2 * y, 0.0);
#undef D3
        double radial = ((gw * w + gx * x) + gy * y) + gz * z;
        g_out[4 * i] = (gw - radial * w) / nrm;
        g_out[4 * i + 1] = (gx - radial * x) / nrm;
        g_out[4 * i + 2] = (gy - radial * y) / nrm;
        g_out[4 * i + 3] = (gz - radial * z) / nrm;
    }
}

/* ------------------------------------------------------------------------- */
/* shading (shading.py), float64                                              */

static double radical_inverse(uint32_t i) {
    i = (i << 16) | (i >> 16);
    i = ((i & 0x55555555u) << 1) | ((i & 0xAAAAAAAAu) >> 1);
    i = ((i & 0x33333333u) << 2) | ((i & 0xCCCCCCCCu) >> 2);
    i = ((i & 0x0F0F0F0Fu) << 4) | ((i & 0xF0F0F0F0u) >> 4);
    i = ((i & 0x00FF00FFu) << 8) | ((i & 0xFF00FF00u) >> 8);
    return (double)i * 2.3283064365386963e-10;
}

static void ggx_h(double xi0, double xi1, double alpha, double h[3]) {
    double phi = 2.0 * OR_PI * xi0;
    double cos_t = sqrt((1.0 - xi1) / (1.0 + (alpha * alpha - 1.0) * xi1));
    double sin_t = sqrt(npmax(1.0 - cos_t * cos_t, 0.0));
    h[0] = sin_t * cos(phi); h[1] = sin_t * sin(phi); h[2] = cos_t;
}

static double smith_g1(double c, double k) { return c / (c * (1.0 - k) + k); }

/* brdf_lut (shading.py:118-156): (res, res, 2) float32, row = roughness */
void or_brdf_lut(int res, int samples, float *lut)
{
    for (int j = 0; j < res; ++j) {
        double r = ((double)j + 0.5) / res;
        double alpha = r * r, k = alpha / 2.0;
        for (int i = 0; i < res; ++i) {
            double cv = ((double)i + 0.5) / res;
            double view[3] = {sqrt(1.0 - cv * cv), 0.0, cv};
            double s1 = 0.0, s2 = 0.0;
            for (int s = 0; s < samples; ++s) {
                double h[3];
                ggx_h(((double)s + 0.5) / samples, radical_inverse((uint32_t)s), alpha, h);
                double vh = (view[0] * h[0] + view[1] * h[1]) + view[2] * h[2];
                double l2 = 2.0 * vh * h[2] - view[2];
                double nh = h[2], nv = cv;
                int good = (l2 > 0.0) && (vh > 0.0);
                double g = smith_g1(nv, k) * smith_g1(npmax(l2, 1e-8), k);
                double gv = good ? g * vh / npmax(nh * nv, 1e-8) : 0.0;
                double fc = pow(1.0 - npclip(vh, 0.0, 1.0), 5.0);
                s1 += gv * (1.0 - fc);
                s2 += gv * fc;
            }
            lut[2 * (j * res + i)] = (float)(s1 / samples);
            lut[2 * (j * res + i) + 1] = (float)(s2 / samples);
        }
    }
}

static int cmp_int_asc(const void *a, const void *b) {
    int x = *(const int *)a, y = *(const int *)b;
    return (x > y) - (x < y);
}

static void texel_dir(int i, int j, int He, int We, double d[3], double *solid) {
    double th = ((double)i + 0.5) * (OR_PI / He);
    double ph = ((double)j + 0.5) * (2.0 * OR_PI / We) - OR_PI;
    d[0] = sin(th) * cos(ph); d[1] = sin(th) * sin(ph); d[2] = cos(th);
    if (solid) *solid = sin(th) * (OR_PI / He) * (2.0 * OR_PI / We);
}

static void dir_coords(const double d[3], int He, int We, double *fu, double *fv) {
    double th = acos(npclip(d[2], -1.0, 1.0));
    double ph = atan2(d[1], d[0]);
    *fu = (ph + OR_PI) * (We / (2.0 * OR_PI)) - 0.5;
    *fv = th * (He / OR_PI) - 0.5;
}

typedef struct { long i0, i1, j0, j1; double tu, tv; int du_ok, dv_ok; } Bil;

static Bil bil_prepare(int h, int w, double fu, double fv, int wrap) {
    Bil b;
    double fvc = npclip(fv, 0.0, h - 1.0);
    double fj = floor(fvc);
    b.j0 = (long)(fj < h - 2 ? fj : h - 2);
    b.tv = fvc - (double)b.j0;
    b.dv_ok = (fv > 0.0) && (fv < h - 1.0);
    b.j1 = b.j0 + 1;
    if (wrap) {
        double i0f = floor(fu);
        b.tu = fu - i0f;
        b.i0 = pymod((long)i0f, w);
        b.i1 = pymod(b.i0 + 1, w);
        b.du_ok = 1;
    } else {
        double fuc = npclip(fu, 0.0, w - 1.0);
        double fi = floor(fuc);
        b.i0 = (long)(fi < w - 2 ? fi : w - 2);
        b.tu = fuc - (double)b.i0;
        b.i1 = b.i0 + 1;
        b.du_ok = (fu > 0.0) && (fu < w - 1.0);
    }
    return b;
}

/* tex is (h, w, C) float64 */
static void bil_lookup(const double *tex, int w, int C, const Bil *b, double *out) {
    double tu = b->tu, tv = b->tv;
    for (int c = 0; c < C; ++c) {
        double A = tex[(b->j0 * w + b->i0) * C + c], B = tex[(b->j0 * w + b->i1) * C + c];
        double Cc = tex[(b->j1 * w + b->i0) * C + c], D = tex[(b->j1 * w + b->i1) * C + c];
        out[c] = (1 - tu) * (1 - tv) * A + tu * (1 - tv) * B + (1 - tu) * tv * Cc + tu * tv * D;
    }
}

static void bil_coord_grads(const double *tex, int w, int C, const Bil *b, double *gu, double *gv) {
    double tu = b->tu, tv = b->tv;
    for (int c = 0; c < C; ++c) {
        double A = tex[(b->j0 * w + b->i0) * C + c], B = tex[(b->j0 * w + b->i1) * C + c];
        double Cc = tex[(b->j1 * w + b->i0) * C + c], D = tex[(b->j1 * w + b->i1) * C + c];
        double u = (1 - tv) * (B - A) + tv * (D - Cc);
        double v = (1 - tu) * (Cc - A) + tu * (D - B);
        gu[c] = b->du_ok ? u : 0.0;
        gv[c] = b->dv_ok ? v : 0.0;
    }
}

static void coord_grad_to_dir(const double d[3], int He, int We, double g_fu, double g_fv, double g[3]) {
    double rxy2 = d[0] * d[0] + d[1] * d[1];
    int safe = rxy2 > 1e-12;
    double inv = safe ? 1.0 / npmax(rxy2, 1e-12) : 0.0;
    double g_phi = g_fu * (We / (2.0 * OR_PI));
    double g_theta = g_fv * (He / OR_PI);
    double sin_t = sqrt(npmax(1.0 - d[2] * d[2], 1e-12));
    g[0] = g_phi * (-d[1]) * inv;
    g[1] = g_phi * d[0] * inv;
    g[2] = safe ? -g_theta / sin_t : 0.0;
}

/* Per-surfel shading context (shading.py:447-503) */
typedef struct {
    double albedo[3], m, r, n[3], wo[3], inv_dist, ndv_raw, refl[3];
    double l_d[3], l_s[3], spec_lo[3], spec_hi[3], b1, b2, f0[3], k_d[3], frac;
    long lvl0, lvl1;
    Bil bd, bs, bl;
    double fx, fy;
} ShadeCtx;

static void shade_one(int i, const float *centers, const float *quats, const float *albedo_raw,
                      const float *metallic_raw, const float *roughness_raw, const double cam_pos[3],
                      int He, int We, int L, const double *diffuse, const double *specular,
                      int lut_res, const double *lut, ShadeCtx *s, double col[3])
{
    for (int c = 0; c < 3; ++c) s->albedo[c] = (double)sigmoid_f32(albedo_raw[3 * i + c]);
    s->m = (double)sigmoid_f32(metallic_raw[i]);
    s->r = (double)sigmoid_f32(roughness_raw[i]);
    double q[4] = {quats[4 * i], quats[4 * i + 1], quats[4 * i + 2], quats[4 * i + 3]};
    double nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
    s->n[0] = 2 * (x * z + w * y); s->n[1] = 2 * (y * z - w * x); s->n[2] = 1 - 2 * (x * x + y * y);
    double tc[3];
    for (int c = 0; c < 3; ++c) tc[c] = cam_pos[c] - (double)centers[3 * i + c];
    double dist = sqrt((tc[0] * tc[0] + tc[1] * tc[1]) + tc[2] * tc[2]);
    s->inv_dist = 1.0 / npmax(dist, 1e-12);
    for (int c = 0; c < 3; ++c) s->wo[c] = tc[c] * s->inv_dist;
    s->ndv_raw = (s->n[0] * s->wo[0] + s->n[1] * s->wo[1]) + s->n[2] * s->wo[2];
    double ndv = npclip(s->ndv_raw, 0.0, 1.0);
    for (int c = 0; c < 3; ++c) s->refl[c] = 2.0 * s->ndv_raw * s->n[c] - s->wo[c];
    double fu, fv;
    dir_coords(s->n, He, We, &fu, &fv);
    s->bd = bil_prepare(He, We, fu, fv, 1);
    bil_lookup(diffuse, We, 3, &s->bd, s->l_d);
    double lvl = npclip(s->r, 0.0, 1.0) * (L - 1);
    long cap = L - 2 > 0 ? L - 2 : 0;
    double fl = floor(lvl);
    s->lvl0 = (long)(fl < cap ? fl : cap);
    s->frac = L > 1 ? lvl - (double)s->lvl0 : 0.0;
    s->lvl1 = s->lvl0 + 1 < L - 1 ? s->lvl0 + 1 : L - 1;
    dir_coords(s->refl, He, We, &fu, &fv);
    s->bs = bil_prepare(He, We, fu, fv, 1);
    size_t lvl_stride = (size_t)He * We * 3;
    bil_lookup(specular + lvl_stride * s->lvl0, We, 3, &s->bs, s->spec_lo);
    bil_lookup(specular + lvl_stride * s->lvl1, We, 3, &s->bs, s->spec_hi);
    for (int c = 0; c < 3; ++c) s->l_s[c] = (1.0 - s->frac) * s->spec_lo[c] + s->frac * s->spec_hi[c];
    s->fx = ndv * (lut_res - 1);
    s->fy = s->r * (lut_res - 1);
    s->bl = bil_prepare(lut_res, lut_res, s->fx, s->fy, 0); /* cols = cos theta, rows = roughness */
    double bb[2];
    bil_lookup(lut, lut_res, 2, &s->bl, bb);
    s->b1 = bb[0]; s->b2 = bb[1];
    for (int c = 0; c < 3; ++c) {
        s->f0[c] = 0.04 * (1.0 - s->m) + s->albedo[c] * s->m;
        s->k_d[c] = (1.0 - s->f0[c]) * (1.0 - s->m);
        col[c] = s->k_d[c] * s->albedo[c] * s->l_d[c] + s->l_s[c] * (s->f0[c] * s->b1 + s->b2);
    }
}

/* shade_surfels: colors (N,3) float32 */
void or_shade(int n, const float *centers, const float *quats, const float *albedo_raw,
              const float *metallic_raw, const float *roughness_raw, const double *cam_pos,
              int He, int We, int L, const double *diffuse, const double *specular,
              int lut_res, const double *lut, float *colors)
{
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        ShadeCtx s;
        double col[3];
        shade_one(i, centers, quats, albedo_raw, metallic_raw, roughness_raw, cam_pos, He, We, L,
                  diffuse, specular, lut_res, lut, &s, col);
        for (int c = 0; c < 3; ++c) colors[3 * i + c] = (float)col[c];
    }
}

/* shade_backward (shading.py:525-621) minus the env adjoint: returns per-surfel
 * grads and the derived-map gradients d_diffuse (He,We,3), d_spec (L,He,We,3). */
void or_shade_backward(int n, const float *centers, const float *quats, const float *albedo_raw,
                       const float *metallic_raw, const float *roughness_raw, const double *cam_pos,
                       int He, int We, int L, const double *diffuse, const double *specular,
                       int lut_res, const double *lut, const double *g_colors,
                       double *g_albedo_raw, double *g_metallic_raw, double *g_roughness_raw,
                       double *g_normals, double *g_centers, double *d_diffuse, double *d_spec)
{
    size_t lvl_stride = (size_t)He * We * 3;
    memset(d_diffuse, 0, sizeof(double) * lvl_stride);
    memset(d_spec, 0, sizeof(double) * lvl_stride * L);
    ShadeCtx *ctx = (ShadeCtx *)malloc(sizeof(ShadeCtx) * (n > 0 ? n : 1));
    double *g_ls = (double *)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
    double *g_ld = (double *)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        ShadeCtx *s = ctx + i;
        double col[3];
        shade_one(i, centers, quats, albedo_raw, metallic_raw, roughness_raw, cam_pos, He, We, L,
                  diffuse, specular, lut_res, lut, s, col);
        const double *g = g_colors + 3 * i;
        double g_kd[3], g_alb[3], g_f0[3];
        double g_b1 = 0.0, g_b2 = 0.0;
        for (int c = 0; c < 3; ++c) {
            g_kd[c] = g[c] * s->albedo[c] * s->l_d[c];
            g_alb[c] = g[c] * s->k_d[c] * s->l_d[c];
            g_ld[3 * i + c] = g[c] * s->k_d[c] * s->albedo[c];
            g_ls[3 * i + c] = g[c] * (s->f0[c] * s->b1 + s->b2);
            g_f0[c] = g[c] * s->l_s[c] * s->b1;
        }
        g_b1 = (g[0] * s->l_s[0] * s->f0[0] + g[1] * s->l_s[1] * s->f0[1]) + g[2] * s->l_s[2] * s->f0[2];
        g_b2 = (g[0] * s->l_s[0] + g[1] * s->l_s[1]) + g[2] * s->l_s[2];
        double g_met = 0.0;
        for (int c = 0; c < 3; ++c) g_f0[c] += g_kd[c] * (-(1.0 - s->m));
        g_met = (g_kd[0] * (-(1.0 - s->f0[0])) + g_kd[1] * (-(1.0 - s->f0[1]))) + g_kd[2] * (-(1.0 - s->f0[2]));
        g_met += (g_f0[0] * (s->albedo[0] - 0.04) + g_f0[1] * (s->albedo[1] - 0.04)) + g_f0[2] * (s->albedo[2] - 0.04);
        for (int c = 0; c < 3; ++c) g_alb[c] += g_f0[c] * s->m;
        double dfx[2], dfy[2];
        bil_coord_grads(lut, lut_res, 2, &s->bl, dfx, dfy);
        double g_ndv = (g_b1 * dfx[0] + g_b2 * dfx[1]) * (lut_res - 1);
        double g_rough = (g_b1 * dfy[0] + g_b2 * dfy[1]) * (lut_res - 1);
        int ndv_active = (s->ndv_raw > 0.0) && (s->ndv_raw < 1.0);
        if (!ndv_active) g_ndv = 0.0;
        if (L > 1) {
            double acc = (g_ls[3 * i] * (s->spec_hi[0] - s->spec_lo[0]) + g_ls[3 * i + 1] * (s->spec_hi[1] - s->spec_lo[1]))
                         + g_ls[3 * i + 2] * (s->spec_hi[2] - s->spec_lo[2]);
            g_rough += acc * (L - 1);
        }
        double g_refl[3] = {0, 0, 0};
        /* lo contribution (level lvl0), then hi (level lvl1) */
        double wts[2] = {1.0 - s->frac, s->frac};
        long lv[2] = {s->lvl0, s->lvl1};
        for (int h = 0; h < 2; ++h) {
            double gu[3], gv[3];
            bil_coord_grads(specular + lvl_stride * lv[h], We, 3, &s->bs, gu, gv);
            double gh[3] = {g_ls[3 * i] * wts[h], g_ls[3 * i + 1] * wts[h], g_ls[3 * i + 2] * wts[h]};
            double gfu = (gh[0] * gu[0] + gh[1] * gu[1]) + gh[2] * gu[2];
            double gfv = (gh[0] * gv[0] + gh[1] * gv[1]) + gh[2] * gv[2];
            double gd[3];
            coord_grad_to_dir(s->refl, He, We, gfu, gfv, gd);
            for (int c = 0; c < 3; ++c) g_refl[c] += gd[c];
        }
        double gu[3], gv[3];
        bil_coord_grads(diffuse, We, 3, &s->bd, gu, gv);
        double gfu = (g_ld[3 * i] * gu[0] + g_ld[3 * i + 1] * gu[1]) + g_ld[3 * i + 2] * gu[2];
        double gfv = (g_ld[3 * i] * gv[0] + g_ld[3 * i + 1] * gv[1]) + g_ld[3 * i + 2] * gv[2];
        double g_n[3];
        coord_grad_to_dir(s->n, He, We, gfu, gfv, g_n);
        double sdot = s->ndv_raw;
        double grn = (g_refl[0] * s->n[0] + g_refl[1] * s->n[1]) + g_refl[2] * s->n[2];
        double g_wo[3];
        for (int c = 0; c < 3; ++c) {
            g_n[c] += 2.0 * grn * s->wo[c] + 2.0 * sdot * g_refl[c];
            g_wo[c] = 2.0 * grn * s->n[c] - g_refl[c];
        }
        double gnd = ndv_active ? g_ndv : 0.0;
        for (int c = 0; c < 3; ++c) { g_n[c] += gnd * s->wo[c]; g_wo[c] += gnd * s->n[c]; }
        double radial = (g_wo[0] * s->wo[0] + g_wo[1] * s->wo[1]) + g_wo[2] * s->wo[2];
        for (int c = 0; c < 3; ++c) {
            g_centers[3 * i + c] = -(g_wo[c] - radial * s->wo[c]) * s->inv_dist;
            g_normals[3 * i + c] = g_n[c];
            g_albedo_raw[3 * i + c] = g_alb[c] * s->albedo[c] * (1.0 - s->albedo[c]);
        }
        g_metallic_raw[i] = g_met * s->m * (1.0 - s->m);
        g_roughness_raw[i] = g_rough * s->r * (1.0 - s->r);
    }
    /* bilinear_scatter order: per level, lo-surfels then hi-surfels; per
     * scatter, corner-major then surfel order (np.add.at semantics). */
    for (int lvl = 0; lvl < L; ++lvl) {
        for (int h = 0; h < 2; ++h) {
            for (int corner = 0; corner < 4; ++corner) {
                for (int i = 0; i < n; ++i) {
                    ShadeCtx *s = ctx + i;
                    long lv = h == 0 ? s->lvl0 : s->lvl1;
                    if (lv != lvl) continue;
                    double wt = h == 0 ? 1.0 - s->frac : s->frac;
                    double tu = s->bs.tu, tv = s->bs.tv, cw;
                    long idx;
                    switch (corner) {
                    case 0: idx = s->bs.j0 * We + s->bs.i0; cw = (1 - tu) * (1 - tv); break;
                    case 1: idx = s->bs.j0 * We + s->bs.i1; cw = tu * (1 - tv); break;
                    case 2: idx = s->bs.j1 * We + s->bs.i0; cw = (1 - tu) * tv; break;
                    default: idx = s->bs.j1 * We + s->bs.i1; cw = tu * tv; break;
                    }
                    for (int c = 0; c < 3; ++c)
                        d_spec[lvl_stride * lvl + 3 * idx + c] += (g_ls[3 * i + c] * wt) * cw;
                }
            }
        }
    }
    for (int corner = 0; corner < 4; ++corner) {
        for (int i = 0; i < n; ++i) {
            ShadeCtx *s = ctx + i;
            double tu = s->bd.tu, tv = s->bd.tv, cw;
            long idx;
            switch (corner) {
            case 0: idx = s->bd.j0 * We + s->bd.i0; cw = (1 - tu) * (1 - tv); break;
            case 1: idx = s->bd.j0 * We + s->bd.i1; cw = tu * (1 - tv); break;
            case 2: idx = s->bd.j1 * We + s->bd.i0; cw = (1 - tu) * tv; break;
            default: idx = s->bd.j1 * We + s->bd.i1; cw = tu * tv; break;
            }
            for (int c = 0; c < 3; ++c) d_diffuse[3 * idx + c] += g_ld[3 * i + c] * cw;
        }
    }
    free(ctx); free(g_ls); free(g_ld);
}

/* ------------------------------------------------------------------------- */
/* environment prefilter operators, applied on the fly (shading.py:275-394)   */

static void texel_table(int He, int We, double *dirs, double *solid) {
    for (int a = 0; a < He * We; ++a) texel_dir(a / We, a % We, He, We, dirs + 3 * a, solid + a);
}

/* Row sums of the clamped-cosine quadrature (shading.py:275-282). */
static void diffuse_rowsums(int T, const double *dirs, const double *solid, double *rowsum) {
#pragma omp parallel for schedule(static)
    for (int a = 0; a < T; ++a) {
        const double *di = dirs + 3 * a;
        double s = 0.0;
        for (int b = 0; b < T; ++b) {
            const double *dj = dirs + 3 * b;
            s += npmax((di[0] * dj[0] + di[1] * dj[1]) + di[2] * dj[2], 0.0) * solid[b];
        }
        rowsum[a] = s;
    }
}

/* One specular operator row (shading.py:285-331) accumulated sample by sample
 * into a dense row buffer; the touched columns are returned sorted.  Returns
 * the weight sum (<= 0 marks the identity fallback, shading.py:324-328). */
static double spec_row(int a, int He, int We, double rough, int samples, const double *dirs,
                       double *row, int *touched, int *list, int *nlist) {
    const double *d = dirs + 3 * a;
    double alpha = rough * rough;
    double up[3] = {0, 0, 1};
    if (!(fabs(d[2]) < 0.999)) { up[0] = 1; up[2] = 0; }
    double tx[3] = {up[1] * d[2] - up[2] * d[1], up[2] * d[0] - up[0] * d[2], up[0] * d[1] - up[1] * d[0]};
    double tn = sqrt((tx[0] * tx[0] + tx[1] * tx[1]) + tx[2] * tx[2]);
    for (int c = 0; c < 3; ++c) tx[c] /= tn;
    double ty[3] = {d[1] * tx[2] - d[2] * tx[1], d[2] * tx[0] - d[0] * tx[2], d[0] * tx[1] - d[1] * tx[0]};
    double wsum = 0.0;
    int m = 0;
    for (int s = 0; s < samples; ++s) {
        double h[3];
        ggx_h(((double)s + 0.5) / samples, radical_inverse((uint32_t)s), alpha, h);
        double hv[3];
        for (int c = 0; c < 3; ++c) hv[c] = h[0] * tx[c] + h[1] * ty[c] + h[2] * d[c];
        double vh = (d[0] * hv[0] + d[1] * hv[1]) + d[2] * hv[2];
        double l[3];
        for (int c = 0; c < 3; ++c) l[c] = 2.0 * vh * hv[c] - d[c];
        double nl = (d[0] * l[0] + d[1] * l[1]) + d[2] * l[2];
        double wgt = npmax(nl, 0.0);
        if (!(wgt > 0)) continue;
        double fu, fv;
        dir_coords(l, He, We, &fu, &fv);
        Bil b = bil_prepare(He, We, fu, fv, 1);
        long idx[4] = {b.j0 * We + b.i0, b.j0 * We + b.i1, b.j1 * We + b.i0, b.j1 * We + b.i1};
        double cw[4] = {wgt * (1 - b.tu) * (1 - b.tv), wgt * b.tu * (1 - b.tv), wgt * (1 - b.tu) * b.tv, wgt * b.tu * b.tv};
        for (int k = 0; k < 4; ++k) {
            if (!touched[idx[k]]) { touched[idx[k]] = 1; row[idx[k]] = 0.0; list[m++] = (int)idx[k]; }
            row[idx[k]] += cw[k];
        }
        wsum += wgt;
    }
    qsort(list, (size_t)m, sizeof(int), cmp_int_asc);
    for (int k = 0; k < m; ++k) touched[list[k]] = 0;
    *nlist = m;
    return wsum;
}

/* refresh (shading.py:369-379): base_log (He,We,3) -> base, diffuse, specular (L,He,We,3) */
void or_env_refresh(int He, int We, int L, int samples, const double *base_log,
                    double *base, double *diffuse, double *specular)
{
    int T = He * We;
    for (int a = 0; a < 3 * T; ++a) base[a] = exp(base_log[a]);
    double *dirs = (double *)malloc(sizeof(double) * 3 * T);
    double *solid = (double *)malloc(sizeof(double) * T);
    double *rowsum = (double *)malloc(sizeof(double) * T);
    texel_table(He, We, dirs, solid);
    diffuse_rowsums(T, dirs, solid, rowsum);
#pragma omp parallel for schedule(static)
    for (int a = 0; a < T; ++a) {
        const double *di = dirs + 3 * a;
        double acc[3] = {0, 0, 0};
        for (int b = 0; b < T; ++b) {
            const double *dj = dirs + 3 * b;
            double wgt = npmax((di[0] * dj[0] + di[1] * dj[1]) + di[2] * dj[2], 0.0) * solid[b] / rowsum[a];
            for (int c = 0; c < 3; ++c) acc[c] += wgt * base[3 * b + c];
        }
        for (int c = 0; c < 3; ++c) diffuse[3 * a + c] = acc[c];
    }
    for (int lvl = 0; lvl < L; ++lvl) {
        double rough = L == 1 ? 0.0 : lvl / (L - 1.0);
        double *out = specular + (size_t)lvl * T * 3;
        if (rough <= 0.0) { memcpy(out, base, sizeof(double) * 3 * T); continue; }
#pragma omp parallel
        {
            double *row = (double *)malloc(sizeof(double) * T);
            int *touched = (int *)calloc(T, sizeof(int));
            int *list = (int *)malloc(sizeof(int) * (4 * samples + 4));
#pragma omp for schedule(static)
            for (int a = 0; a < T; ++a) {
                int m;
                double ws = spec_row(a, He, We, rough, samples, dirs, row, touched, list, &m);
                double acc[3] = {0, 0, 0};
                if (ws <= 0) {
                    for (int c = 0; c < 3; ++c) acc[c] = base[3 * a + c];
                } else {
                    for (int k = 0; k < m; ++k) {
                        double opv = row[list[k]] / ws;
                        for (int c = 0; c < 3; ++c) acc[c] += opv * base[3 * list[k] + c];
                    }
                }
                for (int c = 0; c < 3; ++c) out[3 * a + c] = acc[c];
            }
            free(row); free(touched); free(list);
        }
    }
    free(dirs); free(solid); free(rowsum);
}

/* env_gradient (shading.py:381-394): d_base and d_base_log (He,We,3) */
void or_env_gradient(int He, int We, int L, int samples, const double *base,
                     const double *d_diffuse, const double *d_spec, double *d_base, double *d_base_log)
{
    int T = He * We;
    double *dirs = (double *)malloc(sizeof(double) * 3 * T);
    double *solid = (double *)malloc(sizeof(double) * T);
    double *rowsum = (double *)malloc(sizeof(double) * T);
    texel_table(He, We, dirs, solid);
    diffuse_rowsums(T, dirs, solid, rowsum);
    /* D^T g : column b gathers over rows a */
#pragma omp parallel for schedule(static)
    for (int b = 0; b < T; ++b) {
        const double *dj = dirs + 3 * b;
        double acc[3] = {0, 0, 0};
        for (int a = 0; a < T; ++a) {
            const double *di = dirs + 3 * a;
            double wgt = npmax((di[0] * dj[0] + di[1] * dj[1]) + di[2] * dj[2], 0.0) * solid[b] / rowsum[a];
            for (int c = 0; c < 3; ++c) acc[c] += wgt * d_diffuse[3 * a + c];
        }
        for (int c = 0; c < 3; ++c) d_base[3 * b + c] = acc[c];
    }
    for (int lvl = 0; lvl < L; ++lvl) {
        double rough = L == 1 ? 0.0 : lvl / (L - 1.0);
        const double *g = d_spec + (size_t)lvl * T * 3;
        if (rough <= 0.0) {
            for (int a = 0; a < 3 * T; ++a) d_base[a] += g[a];
            continue;
        }
        double *tmp = (double *)calloc((size_t)3 * T, sizeof(double));
        double *row = (double *)malloc(sizeof(double) * T);
        int *touched = (int *)calloc(T, sizeof(int));
        int *list = (int *)malloc(sizeof(int) * (4 * samples + 4));
        for (int a = 0; a < T; ++a) {
            int m;
            double ws = spec_row(a, He, We, rough, samples, dirs, row, touched, list, &m);
            if (ws <= 0) {
                for (int c = 0; c < 3; ++c) tmp[3 * a + c] += g[3 * a + c];
                continue;
            }
            for (int k = 0; k < m; ++k) {
                double opv = row[list[k]] / ws;
                for (int c = 0; c < 3; ++c) tmp[3 * list[k] + c] += opv * g[3 * a + c];
            }
        }
        for (int a = 0; a < 3 * T; ++a) d_base[a] += tmp[a];
        free(tmp); free(row); free(touched); free(list);
    }
    for (int a = 0; a < 3 * T; ++a) d_base_log[a] = d_base[a] * base[a];
    free(dirs); free(solid); free(rowsum);
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
