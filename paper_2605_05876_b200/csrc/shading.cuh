// shading.cuh -- split-sum IBL shading of one surfel and its adjoint, float64
// like the reference (shading.py:447-621).  Used by the preprocess kernel
// (forward) and the chain-backward kernel (adjoint, recomputing the forward
// state from the parameters instead of storing a per-surfel context).
#pragma once
#include "ss_common.cuh"

__device__ __forceinline__ float ss_sigmoid_f32(float x) {
    // surfels.py:16-23 two-branch sigmoid in float32; exp correctly rounded
    if (x >= 0.0f) return 1.0f / (1.0f + (float)exp((double)-x));
    float ex = (float)exp((double)x);
    return ex / (1.0f + ex);
}

__device__ __forceinline__ double ss_clip(double a, double lo, double hi) {
    if (a != a) return a;
    return a < lo ? lo : (a > hi ? hi : a);
}
__device__ __forceinline__ double ss_npmax(double a, double b) { return (a != a) ? a : (a > b ? a : b); }

struct SsBil {
    int i0, i1, j0, j1;
    double tu, tv;
    bool du_ok, dv_ok;
};

// _bilinear_prepare (shading.py:200-219); fu indexes columns, fv rows.
__device__ __forceinline__ SsBil ss_bil_prepare(int h, int w, double fu, double fv, bool wrap) {
    SsBil b;
    double fvc = ss_clip(fv, 0.0, h - 1.0);
    double fj = floor(fvc);
    b.j0 = (int)(fj < h - 2 ? fj : h - 2);
    b.tv = fvc - (double)b.j0;
    b.dv_ok = (fv > 0.0) && (fv < h - 1.0);
    b.j1 = b.j0 + 1;
    if (wrap) {
        double i0f = floor(fu);
        b.tu = fu - i0f;
        long long ii = (long long)i0f % w;
        if (ii < 0) ii += w;
        b.i0 = (int)ii;
        b.i1 = (b.i0 + 1) % w;
        b.du_ok = true;
    } else {
        double fuc = ss_clip(fu, 0.0, w - 1.0);
        double fi = floor(fuc);
        b.i0 = (int)(fi < w - 2 ? fi : w - 2);
        b.tu = fuc - (double)b.i0;
        b.i1 = b.i0 + 1;
        b.du_ok = (fu > 0.0) && (fu < w - 1.0);
    }
    return b;
}

template <int C>
__device__ __forceinline__ void ss_bil_lookup(const float *__restrict__ tex, int w, const SsBil &b, double *out) {
    const double tu = b.tu, tv = b.tv;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        double A = tex[(b.j0 * w + b.i0) * C + c], B = tex[(b.j0 * w + b.i1) * C + c];
        double Cc = tex[(b.j1 * w + b.i0) * C + c], D = tex[(b.j1 * w + b.i1) * C + c];
        out[c] = (1 - tu) * (1 - tv) * A + tu * (1 - tv) * B + (1 - tu) * tv * Cc + tu * tv * D;
    }
}

template <int C>
__device__ __forceinline__ void ss_bil_grads(const float *__restrict__ tex, int w, const SsBil &b, double *gu, double *gv) {
    const double tu = b.tu, tv = b.tv;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        double A = tex[(b.j0 * w + b.i0) * C + c], B = tex[(b.j0 * w + b.i1) * C + c];
        double Cc = tex[(b.j1 * w + b.i0) * C + c], D = tex[(b.j1 * w + b.i1) * C + c];
        gu[c] = b.du_ok ? (1 - tv) * (B - A) + tv * (D - Cc) : 0.0;
        gv[c] = b.dv_ok ? (1 - tu) * (Cc - A) + tu * (D - B) : 0.0;
    }
}

// dirs_to_coords (shading.py:172-179)
__device__ __forceinline__ void ss_dir_coords(const double d[3], int he, int we, double &fu, double &fv) {
    double th = acos(ss_clip(d[2], -1.0, 1.0));
    double ph = atan2(d[1], d[0]);
    fu = (ph + SS_PI) * (we / (2.0 * SS_PI)) - 0.5;
    fv = th * (he / SS_PI) - 0.5;
}

// coord_grad_to_dir (shading.py:182-197)
__device__ __forceinline__ void ss_coord_grad_to_dir(const double d[3], int he, int we, double gfu, double gfv, double g[3]) {
    double rxy2 = d[0] * d[0] + d[1] * d[1];
    bool safe = rxy2 > 1e-12;
    double inv = safe ? 1.0 / ss_npmax(rxy2, 1e-12) : 0.0;
    double gphi = gfu * (we / (2.0 * SS_PI));
    double gth = gfv * (he / SS_PI);
    double sin_t = sqrt(ss_npmax(1.0 - d[2] * d[2], 1e-12));
    g[0] = gphi * (-d[1]) * inv;
    g[1] = gphi * d[0] * inv;
    g[2] = safe ? -gth / sin_t : 0.0;
}

struct ShadeIn {
    double albedo[3], m, r, n[3], wo[3], inv_dist;
};

struct ShadeState {
    double ndv_raw, refl[3], l_d[3], l_s[3], spec_lo[3], spec_hi[3], b1, b2, f0[3], k_d[3], frac;
    int lvl0, lvl1;
    SsBil bd, bs, bl;
};

// Activated materials, float64 normal and view direction of surfel i.
__device__ __forceinline__ void ss_shade_inputs(const SsCloud &cloud, int i, const double cam_pos[3], ShadeIn &in) {
    in.albedo[0] = (double)ss_sigmoid_f32(cloud.albedo_raw[3 * i]);
    in.albedo[1] = (double)ss_sigmoid_f32(cloud.albedo_raw[3 * i + 1]);
    in.albedo[2] = (double)ss_sigmoid_f32(cloud.albedo_raw[3 * i + 2]);
    in.m = (double)ss_sigmoid_f32(cloud.metallic_raw[i]);
    in.r = (double)ss_sigmoid_f32(cloud.roughness_raw[i]);
    double q0 = cloud.quats[4 * i], q1 = cloud.quats[4 * i + 1], q2 = cloud.quats[4 * i + 2], q3 = cloud.quats[4 * i + 3];
    double nrm = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    double w = q0 / nrm, x = q1 / nrm, y = q2 / nrm, z = q3 / nrm;
    in.n[0] = 2 * (x * z + w * y); in.n[1] = 2 * (y * z - w * x); in.n[2] = 1 - 2 * (x * x + y * y);
    double tc[3];
    for (int c = 0; c < 3; ++c) tc[c] = cam_pos[c] - (double)cloud.centers[3 * i + c];
    double dist = sqrt((tc[0] * tc[0] + tc[1] * tc[1]) + tc[2] * tc[2]);
    in.inv_dist = 1.0 / ss_npmax(dist, 1e-12);
    for (int c = 0; c < 3; ++c) in.wo[c] = tc[c] * in.inv_dist;
}

// shade_surfels body (shading.py:463-488)
__device__ __forceinline__ void ss_shade_forward(const ShadeIn &in, const SsEnv &env, ShadeState &s, double col[3]) {
    const int he = env.he, we = env.we, L = env.levels, R = env.lut_res;
    s.ndv_raw = (in.n[0] * in.wo[0] + in.n[1] * in.wo[1]) + in.n[2] * in.wo[2];
    double ndv = ss_clip(s.ndv_raw, 0.0, 1.0);
    for (int c = 0; c < 3; ++c) s.refl[c] = 2.0 * s.ndv_raw * in.n[c] - in.wo[c];
    double fu, fv;
    ss_dir_coords(in.n, he, we, fu, fv);
    s.bd = ss_bil_prepare(he, we, fu, fv, true);
    ss_bil_lookup<3>(env.diffuse, we, s.bd, s.l_d);
    double lvl = ss_clip(in.r, 0.0, 1.0) * (L - 1);
    int cap = L - 2 > 0 ? L - 2 : 0;
    double fl = floor(lvl);
    s.lvl0 = (int)(fl < cap ? fl : cap);
    s.frac = L > 1 ? lvl - (double)s.lvl0 : 0.0;
    s.lvl1 = s.lvl0 + 1 < L - 1 ? s.lvl0 + 1 : L - 1;
    ss_dir_coords(s.refl, he, we, fu, fv);
    s.bs = ss_bil_prepare(he, we, fu, fv, true);
    const size_t lstride = (size_t)he * we * 3;
    ss_bil_lookup<3>(env.specular + lstride * s.lvl0, we, s.bs, s.spec_lo);
    ss_bil_lookup<3>(env.specular + lstride * s.lvl1, we, s.bs, s.spec_hi);
    for (int c = 0; c < 3; ++c) s.l_s[c] = (1.0 - s.frac) * s.spec_lo[c] + s.frac * s.spec_hi[c];
    s.bl = ss_bil_prepare(R, R, ndv * (R - 1), in.r * (R - 1), false);
    double bb[2];
    ss_bil_lookup<2>(env.lut, R, s.bl, bb);
    s.b1 = bb[0]; s.b2 = bb[1];
    for (int c = 0; c < 3; ++c) {
        s.f0[c] = 0.04 * (1.0 - in.m) + in.albedo[c] * in.m;
        s.k_d[c] = (1.0 - s.f0[c]) * (1.0 - in.m);
        col[c] = s.k_d[c] * in.albedo[c] * s.l_d[c] + s.l_s[c] * (s.f0[c] * s.b1 + s.b2);
    }
}

// Branch signature cells (shading.py:490-497), 15 ints.
__device__ __forceinline__ void ss_shade_cells(const ShadeState &s, const SsEnv &env, int32_t *out) {
    out[0] = s.bd.i0; out[1] = s.bd.j0; out[2] = s.bd.du_ok; out[3] = s.bd.dv_ok;
    out[4] = s.bs.i0; out[5] = s.bs.j0; out[6] = s.bs.du_ok; out[7] = s.bs.dv_ok;
    out[8] = s.lvl0;
    out[9] = s.bl.i0; out[10] = s.bl.j0; out[11] = s.bl.du_ok; out[12] = s.bl.dv_ok;
    out[13] = s.ndv_raw > 0.0; out[14] = s.ndv_raw < 1.0;
}

struct ShadeGrads {
    double albedo_raw[3], metallic_raw, roughness_raw, normal[3], center[3];
    double g_ls[3], g_ld[3];   // derived-map upstreams for the env scatter
};

// shade_backward for one surfel (shading.py:525-615), env adjoint excluded.
__device__ __forceinline__ void ss_shade_backward(const ShadeIn &in, const ShadeState &s, const SsEnv &env,
                                                  const double g[3], ShadeGrads &o) {
    const int he = env.he, we = env.we, L = env.levels, R = env.lut_res;
    double g_kd[3], g_alb[3], g_f0[3];
    for (int c = 0; c < 3; ++c) {
        g_kd[c] = g[c] * in.albedo[c] * s.l_d[c];
        g_alb[c] = g[c] * s.k_d[c] * s.l_d[c];
        o.g_ld[c] = g[c] * s.k_d[c] * in.albedo[c];
        o.g_ls[c] = g[c] * (s.f0[c] * s.b1 + s.b2);
        g_f0[c] = g[c] * s.l_s[c] * s.b1;
    }
    double g_b1 = (g[0] * s.l_s[0] * s.f0[0] + g[1] * s.l_s[1] * s.f0[1]) + g[2] * s.l_s[2] * s.f0[2];
    double g_b2 = (g[0] * s.l_s[0] + g[1] * s.l_s[1]) + g[2] * s.l_s[2];
    for (int c = 0; c < 3; ++c) g_f0[c] += g_kd[c] * (-(1.0 - in.m));
    double g_met = (g_kd[0] * (-(1.0 - s.f0[0])) + g_kd[1] * (-(1.0 - s.f0[1]))) + g_kd[2] * (-(1.0 - s.f0[2]));
    g_met += (g_f0[0] * (in.albedo[0] - 0.04) + g_f0[1] * (in.albedo[1] - 0.04)) + g_f0[2] * (in.albedo[2] - 0.04);
    for (int c = 0; c < 3; ++c) g_alb[c] += g_f0[c] * in.m;
    double dfx[2], dfy[2];
    ss_bil_grads<2>(env.lut, R, s.bl, dfx, dfy);
    double g_ndv = (g_b1 * dfx[0] + g_b2 * dfx[1]) * (R - 1);
    double g_rough = (g_b1 * dfy[0] + g_b2 * dfy[1]) * (R - 1);
    bool active = (s.ndv_raw > 0.0) && (s.ndv_raw < 1.0);
    if (!active) g_ndv = 0.0;
    if (L > 1) {
        double acc = (o.g_ls[0] * (s.spec_hi[0] - s.spec_lo[0]) + o.g_ls[1] * (s.spec_hi[1] - s.spec_lo[1])) +
                     o.g_ls[2] * (s.spec_hi[2] - s.spec_lo[2]);
        g_rough += acc * (L - 1);
    }
    double g_refl[3] = {0.0, 0.0, 0.0};
    const size_t lstride = (size_t)he * we * 3;
    const double wts[2] = {1.0 - s.frac, s.frac};
    const int lv[2] = {s.lvl0, s.lvl1};
    for (int h = 0; h < 2; ++h) {
        double gu[3], gv[3];
        ss_bil_grads<3>(env.specular + lstride * lv[h], we, s.bs, gu, gv);
        double gh0 = o.g_ls[0] * wts[h], gh1 = o.g_ls[1] * wts[h], gh2 = o.g_ls[2] * wts[h];
        double gfu = (gh0 * gu[0] + gh1 * gu[1]) + gh2 * gu[2];
        double gfv = (gh0 * gv[0] + gh1 * gv[1]) + gh2 * gv[2];
        double gd[3];
        ss_coord_grad_to_dir(s.refl, he, we, gfu, gfv, gd);
        for (int c = 0; c < 3; ++c) g_refl[c] += gd[c];
    }
    double gu[3], gv[3];
    ss_bil_grads<3>(env.diffuse, we, s.bd, gu, gv);
    double gfu = (o.g_ld[0] * gu[0] + o.g_ld[1] * gu[1]) + o.g_ld[2] * gu[2];
    double gfv = (o.g_ld[0] * gv[0] + o.g_ld[1] * gv[1]) + o.g_ld[2] * gv[2];
    double g_n[3];
    ss_coord_grad_to_dir(in.n, he, we, gfu, gfv, g_n);
    double grn = (g_refl[0] * in.n[0] + g_refl[1] * in.n[1]) + g_refl[2] * in.n[2];
    double g_wo[3];
    for (int c = 0; c < 3; ++c) {
        g_n[c] += 2.0 * grn * in.wo[c] + 2.0 * s.ndv_raw * g_refl[c];
        g_wo[c] = 2.0 * grn * in.n[c] - g_refl[c];
    }
    double gnd = active ? g_ndv : 0.0;
    for (int c = 0; c < 3; ++c) { g_n[c] += gnd * in.wo[c]; g_wo[c] += gnd * in.n[c]; }
    double radial = (g_wo[0] * in.wo[0] + g_wo[1] * in.wo[1]) + g_wo[2] * in.wo[2];
    for (int c = 0; c < 3; ++c) {
        o.center[c] = -(g_wo[c] - radial * in.wo[c]) * in.inv_dist;
        o.normal[c] = g_n[c];
        o.albedo_raw[c] = g_alb[c] * in.albedo[c] * (1.0 - in.albedo[c]);
    }
    o.metallic_raw = g_met * in.m * (1.0 - in.m);
    o.roughness_raw = g_rough * in.r * (1.0 - in.r);
}
