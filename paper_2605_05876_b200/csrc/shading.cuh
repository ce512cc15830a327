// shading.cuh -- split-sum IBL shading of one surfel and its adjoint,
// templated on the real type (float64 like the reference for the forward
// colours; the backward may run in float32) (shading.py:447-621).  Used by the preprocess kernel
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

// Fast sigmoid for the float32 shading adjoint (gradients: the 1e-3 bar).
__device__ __forceinline__ float ss_sigmoid_fast(float x) {
    const float e = __expf(-fabsf(x));
    return x >= 0.0f ? __fdividef(1.0f, 1.0f + e) : __fdividef(e, 1.0f + e);
}

template <typename R>
__device__ __forceinline__ R ss_act(float x) {
    if constexpr (sizeof(R) == 4) return ss_sigmoid_fast(x);
    else return (R)ss_sigmoid_f32(x);
}

template <typename R>
__device__ __forceinline__ R ss_clip(R a, R lo, R hi) {
    if (a != a) return a;
    return a < lo ? lo : (a > hi ? hi : a);
}
template <typename R>
__device__ __forceinline__ R ss_npmax(R a, R b) { return (a != a) ? a : (a > b ? a : b); }

template <typename R>
struct SsBil {
    int i0, i1, j0, j1;
    R tu, tv;
    bool du_ok, dv_ok;
};

// _bilinear_prepare (shading.py:200-219); fu indexes columns, fv rows.
template <typename R>
__device__ __forceinline__ SsBil<R> ss_bil_prepare(int h, int w, R fu, R fv, bool wrap) {
    SsBil<R> b;
    R fvc = ss_clip<R>(fv, R(0.0), h - R(1.0));
    R fj = floor(fvc);
    b.j0 = (int)(fj < h - 2 ? fj : h - 2);
    b.tv = fvc - (R)b.j0;
    b.dv_ok = (fv > R(0.0)) && (fv < h - R(1.0));
    b.j1 = b.j0 + 1;
    if (wrap) {
        R i0f = floor(fu);
        b.tu = fu - i0f;
        // fu = (phi + pi) w / (2 pi) - 1/2 lies in [-1/2, w - 1/2]: one
        // conditional wrap instead of a 64-bit modulo (the modulo stays for
        // anything outside (-w, 2w))
        long long ii = (long long)i0f;
        if (ii < 0) ii += w;
        else if (ii >= w) ii -= w;
        if (ii < 0 || ii >= w) {
            ii = (long long)i0f % w;
            if (ii < 0) ii += w;
        }
        b.i0 = (int)ii;
        b.i1 = b.i0 + 1 == w ? 0 : b.i0 + 1;
        b.du_ok = true;
    } else {
        R fuc = ss_clip<R>(fu, R(0.0), w - R(1.0));
        R fi = floor(fuc);
        b.i0 = (int)(fi < w - 2 ? fi : w - 2);
        b.tu = fuc - (R)b.i0;
        b.i1 = b.i0 + 1;
        b.du_ok = (fu > R(0.0)) && (fu < w - R(1.0));
    }
    return b;
}

template <int C, typename R, typename T = float>
__device__ __forceinline__ void ss_bil_lookup(const T *__restrict__ tex, int w, const SsBil<R> &b, R *out) {
    const R tu = b.tu, tv = b.tv;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        R A = tex[(b.j0 * w + b.i0) * C + c], B = tex[(b.j0 * w + b.i1) * C + c];
        R Cc = tex[(b.j1 * w + b.i0) * C + c], D = tex[(b.j1 * w + b.i1) * C + c];
        out[c] = (1 - tu) * (1 - tv) * A + tu * (1 - tv) * B + (1 - tu) * tv * Cc + tu * tv * D;
    }
}

// 3-channel lookups on 16-byte texels (the padded copies of the env maps)
template <typename R>
__device__ __forceinline__ void ss_bil_lookup4(const float4 *__restrict__ tex, int w, const SsBil<R> &b, R *out) {
    const float4 A = __ldg(tex + b.j0 * w + b.i0), B = __ldg(tex + b.j0 * w + b.i1);
    const float4 Cc = __ldg(tex + b.j1 * w + b.i0), D = __ldg(tex + b.j1 * w + b.i1);
    const R tu = b.tu, tv = b.tv;
    const R wa = (1 - tu) * (1 - tv), wb = tu * (1 - tv), wc = (1 - tu) * tv, wd = tu * tv;
    out[0] = wa * A.x + wb * B.x + wc * Cc.x + wd * D.x;
    out[1] = wa * A.y + wb * B.y + wc * Cc.y + wd * D.y;
    out[2] = wa * A.z + wb * B.z + wc * Cc.z + wd * D.z;
}

template <typename R>
__device__ __forceinline__ void ss_bil_grads4(const float4 *__restrict__ tex, int w, const SsBil<R> &b, R *gu, R *gv) {
    const float4 A = __ldg(tex + b.j0 * w + b.i0), B = __ldg(tex + b.j0 * w + b.i1);
    const float4 Cc = __ldg(tex + b.j1 * w + b.i0), D = __ldg(tex + b.j1 * w + b.i1);
    const R tu = b.tu, tv = b.tv;
    const R a[3] = {A.x, A.y, A.z}, bb[3] = {B.x, B.y, B.z}, c[3] = {Cc.x, Cc.y, Cc.z}, d[3] = {D.x, D.y, D.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        gu[k] = b.du_ok ? (1 - tv) * (bb[k] - a[k]) + tv * (d[k] - c[k]) : R(0.0);
        gv[k] = b.dv_ok ? (1 - tu) * (c[k] - a[k]) + tu * (d[k] - bb[k]) : R(0.0);
    }
}

// value and coordinate derivatives of one bilinear lookup from ONE read of
// its four texels (the forward and the adjoint of the chain kernel share it)
template <typename R>
__device__ __forceinline__ void ss_bil_lookup_grads4(const float4 *__restrict__ tex, int w, const SsBil<R> &b, R *out,
                                                     R *gu, R *gv) {
    const float4 A = __ldg(tex + b.j0 * w + b.i0), B = __ldg(tex + b.j0 * w + b.i1);
    const float4 Cc = __ldg(tex + b.j1 * w + b.i0), D = __ldg(tex + b.j1 * w + b.i1);
    const R tu = b.tu, tv = b.tv;
    const R wa = (1 - tu) * (1 - tv), wb = tu * (1 - tv), wc = (1 - tu) * tv, wd = tu * tv;
    const R a[3] = {A.x, A.y, A.z}, bb[3] = {B.x, B.y, B.z}, c[3] = {Cc.x, Cc.y, Cc.z}, d[3] = {D.x, D.y, D.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        out[k] = wa * a[k] + wb * bb[k] + wc * c[k] + wd * d[k];
        gu[k] = b.du_ok ? (1 - tv) * (bb[k] - a[k]) + tv * (d[k] - c[k]) : R(0.0);
        gv[k] = b.dv_ok ? (1 - tu) * (c[k] - a[k]) + tu * (d[k] - bb[k]) : R(0.0);
    }
}

template <int C, typename R>
__device__ __forceinline__ void ss_bil_lookup_grads(const float *__restrict__ tex, int w, const SsBil<R> &b, R *out,
                                                    R *gu, R *gv) {
    const R tu = b.tu, tv = b.tv;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        R A = tex[(b.j0 * w + b.i0) * C + c], B = tex[(b.j0 * w + b.i1) * C + c];
        R Cc = tex[(b.j1 * w + b.i0) * C + c], D = tex[(b.j1 * w + b.i1) * C + c];
        out[c] = (1 - tu) * (1 - tv) * A + tu * (1 - tv) * B + (1 - tu) * tv * Cc + tu * tv * D;
        gu[c] = b.du_ok ? (1 - tv) * (B - A) + tv * (D - Cc) : R(0.0);
        gv[c] = b.dv_ok ? (1 - tu) * (Cc - A) + tu * (D - B) : R(0.0);
    }
}

template <int C, typename R>
__device__ __forceinline__ void ss_bil_grads(const float *__restrict__ tex, int w, const SsBil<R> &b, R *gu, R *gv) {
    const R tu = b.tu, tv = b.tv;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        R A = tex[(b.j0 * w + b.i0) * C + c], B = tex[(b.j0 * w + b.i1) * C + c];
        R Cc = tex[(b.j1 * w + b.i0) * C + c], D = tex[(b.j1 * w + b.i1) * C + c];
        gu[c] = b.du_ok ? (1 - tv) * (B - A) + tv * (D - Cc) : R(0.0);
        gv[c] = b.dv_ok ? (1 - tu) * (Cc - A) + tu * (D - B) : R(0.0);
    }
}

// float atan2 with ~3e-7 rad error (range reduction to |t| <= tan(pi/8) and
// the classic 4-term minimax polynomial for atan(t)/t), IEEE signed-zero
// quadrants; finite inputs only (shading directions).  About a sixth of
// atan2f's instruction count.
__device__ __forceinline__ float ss_atan2f(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float a = mx > 0.f ? __fdividef(mn, mx) : 0.f;  // [0, 1]
    const bool big = a > 0.41421356237f;
    const float t = big ? __fdividef(a - 1.f, a + 1.f) : a;  // |t| <= tan(pi/8)
    const float z = t * t;
    const float p = fmaf(fmaf(fmaf(8.05374449538e-2f, z, -1.38776856032e-1f), z, 1.99777106478e-1f), z,
                         -3.33329491539e-1f);
    float r = fmaf(p * z, t, t);
    if (big) r += 0.785398163397448310f;
    if (ay > ax) r = 1.57079632679489662f - r;
    if (signbit(x)) r = 3.14159265358979324f - r;
    return copysignf(r, y);
}

// dirs_to_coords (shading.py:172-179)
template <typename R>
__device__ __forceinline__ void ss_dir_coords(const R d[3], int he, int we, R &fu, R &fv) {
    // float32: theta = atan2(|d_xy|, d_z) instead of acos(d_z) -- the same
    // angle for a unit d but well conditioned at the poles, where acos would
    // amplify the float32 rounding of d_z
    R th;
    if constexpr (sizeof(R) == 4) th = ss_atan2f(sqrtf(d[0] * d[0] + d[1] * d[1]), d[2]);
    else th = acos(ss_clip<R>(d[2], -R(1.0), R(1.0)));
    R ph;
    if constexpr (sizeof(R) == 4) ph = ss_atan2f(d[1], d[0]);
    else ph = atan2(d[1], d[0]);
    fu = (ph + R(SS_PI)) * ((R)we / (R(2) * R(SS_PI))) - R(0.5);
    fv = th * ((R)he / R(SS_PI)) - R(0.5);
}

// coord_grad_to_dir (shading.py:182-197)
template <typename R>
__device__ __forceinline__ void ss_coord_grad_to_dir(const R d[3], int he, int we, R gfu, R gfv, R g[3]) {
    R rxy2 = d[0] * d[0] + d[1] * d[1];
    bool safe = rxy2 > R(1e-12);
    R inv = safe ? R(1.0) / ss_npmax<R>(rxy2, R(1e-12)) : R(0.0);
    R gphi = gfu * ((R)we / (R(2) * R(SS_PI)));
    R gth = gfv * ((R)he / R(SS_PI));
    R sin_t = sqrt(ss_npmax<R>(R(1.0) - d[2] * d[2], R(1e-12)));
    g[0] = gphi * (-d[1]) * inv;
    g[1] = gphi * d[0] * inv;
    g[2] = safe ? -gth / sin_t : R(0.0);
}

template <typename R>
struct ShadeIn {
    R albedo[3], m, r, n[3], wo[3], inv_dist;
};

template <typename R>
struct ShadeState {
    R ndv_raw, refl[3], l_d[3], l_s[3], spec_lo[3], spec_hi[3], b1, b2, f0[3], k_d[3], frac;
    int lvl0, lvl1;
    SsBil<R> bd, bs, bl;
    // texel derivatives of the lookups, when the forward kept them
    // (ss_shade_forward_cells): diffuse, specular lo / hi, LUT
    R dgu[3], dgv[3], sgu[2][3], sgv[2][3], lgu[2], lgv[2];
    // the step's diffuse normal map (PreDiff): dL/dn = (gfu a0, gfu a1, gfv b2)
    bool dpre;
    R da0, da1, db2;
};

// Activated materials and normal of surfel i (view independent).
template <typename R>
__device__ __forceinline__ void ss_shade_material(const SsCloud &cloud, int i, ShadeIn<R> &in) {
    in.albedo[0] = ss_act<R>(cloud.albedo_raw[3 * i]);
    in.albedo[1] = ss_act<R>(cloud.albedo_raw[3 * i + 1]);
    in.albedo[2] = ss_act<R>(cloud.albedo_raw[3 * i + 2]);
    in.m = ss_act<R>(cloud.metallic_raw[i]);
    in.r = ss_act<R>(cloud.roughness_raw[i]);
    R q0 = cloud.quats[4 * i], q1 = cloud.quats[4 * i + 1], q2 = cloud.quats[4 * i + 2], q3 = cloud.quats[4 * i + 3];
    R nrm = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    R w = q0 / nrm, x = q1 / nrm, y = q2 / nrm, z = q3 / nrm;
    in.n[0] = 2 * (x * z + w * y); in.n[1] = 2 * (y * z - w * x); in.n[2] = 1 - 2 * (x * x + y * y);
}

// View direction of surfel i.
template <typename R>
__device__ __forceinline__ void ss_shade_view(const SsCloud &cloud, int i, const double cam_pos[3], ShadeIn<R> &in) {
    R tc[3];
    for (int c = 0; c < 3; ++c) tc[c] = cam_pos[c] - (R)cloud.centers[3 * i + c];
    R dist = sqrt((tc[0] * tc[0] + tc[1] * tc[1]) + tc[2] * tc[2]);
    in.inv_dist = R(1.0) / ss_npmax<R>(dist, R(1e-12));
    for (int c = 0; c < 3; ++c) in.wo[c] = tc[c] * in.inv_dist;
}

// Activated materials, float64 normal and view direction of surfel i.
template <typename R>
__device__ __forceinline__ void ss_shade_inputs(const SsCloud &cloud, int i, const double cam_pos[3], ShadeIn<R> &in) {
    ss_shade_material(cloud, i, in);
    ss_shade_view(cloud, i, cam_pos, in);
}

// The diffuse (irradiance) lookup of shade_surfels (shading.py:469-471):
// view independent -- TrainStep evaluates it once per step (ss_surfel_prepass).
template <typename R>
__device__ __forceinline__ void ss_shade_diffuse(const R n[3], const SsEnv &env, SsBil<R> &bd, R l_d[3]) {
    const int he = env.he, we = env.we;
    R fu, fv;
    ss_dir_coords(n, he, we, fu, fv);
    bd = ss_bil_prepare<R>(he, we, fu, fv, true);
    const float4 *d4 = reinterpret_cast<const float4 *>(env.diffuse4);
    // float64 shading reads the float64 maps (the reference's, shading.py:369-379)
    const bool m64 = sizeof(R) == 8 && env.diffuse64 && env.specular64;
    if (m64) ss_bil_lookup<3>(env.diffuse64, we, bd, l_d);
    else if (d4) ss_bil_lookup4(d4, we, bd, l_d);
    else ss_bil_lookup<3>(env.diffuse, we, bd, l_d);
}

// shade_surfels body (shading.py:463-488) after the diffuse lookup (s.bd,
// s.l_d set): reflection, specular levels, LUT, colour.
template <typename R>
__device__ __forceinline__ void ss_shade_forward_view(const ShadeIn<R> &in, const SsEnv &env, ShadeState<R> &s,
                                                      R col[3]) {
    const int he = env.he, we = env.we, L = env.levels, LR = env.lut_res;
    s.ndv_raw = (in.n[0] * in.wo[0] + in.n[1] * in.wo[1]) + in.n[2] * in.wo[2];
    R ndv = ss_clip<R>(s.ndv_raw, R(0.0), R(1.0));
    for (int c = 0; c < 3; ++c) s.refl[c] = R(2.0) * s.ndv_raw * in.n[c] - in.wo[c];
    R fu, fv;
    const float4 *s4 = reinterpret_cast<const float4 *>(env.specular4);
    const bool m64 = sizeof(R) == 8 && env.diffuse64 && env.specular64;
    R lvl = ss_clip<R>(in.r, R(0.0), R(1.0)) * (L - 1);
    int cap = L - 2 > 0 ? L - 2 : 0;
    R fl = floor(lvl);
    s.lvl0 = (int)(fl < cap ? fl : cap);
    s.frac = L > 1 ? lvl - (R)s.lvl0 : R(0.0);
    s.lvl1 = s.lvl0 + 1 < L - 1 ? s.lvl0 + 1 : L - 1;
    ss_dir_coords(s.refl, he, we, fu, fv);
    s.bs = ss_bil_prepare<R>(he, we, fu, fv, true);
    const size_t lstride = (size_t)he * we * 3;
    if (m64) {
        ss_bil_lookup<3>(env.specular64 + lstride * s.lvl0, we, s.bs, s.spec_lo);
        ss_bil_lookup<3>(env.specular64 + lstride * s.lvl1, we, s.bs, s.spec_hi);
    } else if (s4) {
        ss_bil_lookup4(s4 + (size_t)he * we * s.lvl0, we, s.bs, s.spec_lo);
        ss_bil_lookup4(s4 + (size_t)he * we * s.lvl1, we, s.bs, s.spec_hi);
    } else {
        ss_bil_lookup<3>(env.specular + lstride * s.lvl0, we, s.bs, s.spec_lo);
        ss_bil_lookup<3>(env.specular + lstride * s.lvl1, we, s.bs, s.spec_hi);
    }
    for (int c = 0; c < 3; ++c) s.l_s[c] = (R(1.0) - s.frac) * s.spec_lo[c] + s.frac * s.spec_hi[c];
    s.bl = ss_bil_prepare<R>(LR, LR, ndv * (LR - 1), in.r * (LR - 1), false);
    R bb[2];
    ss_bil_lookup<2>(env.lut, LR, s.bl, bb);
    s.b1 = bb[0]; s.b2 = bb[1];
    for (int c = 0; c < 3; ++c) {
        s.f0[c] = R(0.04) * (R(1.0) - in.m) + in.albedo[c] * in.m;
        s.k_d[c] = (R(1.0) - s.f0[c]) * (R(1.0) - in.m);
        col[c] = s.k_d[c] * in.albedo[c] * s.l_d[c] + s.l_s[c] * (s.f0[c] * s.b1 + s.b2);
    }
}

// shade_surfels body (shading.py:463-488)
template <typename R>
__device__ __forceinline__ void ss_shade_forward(const ShadeIn<R> &in, const SsEnv &env, ShadeState<R> &s, R col[3]) {
    ss_shade_diffuse(in.n, env, s.bd, s.l_d);
    ss_shade_forward_view(in, env, s, col);
}

// Narrow a float64 forward state to float32: the backward then runs in
// float32 on EXACTLY the forward's branch decisions (texel cells, roughness
// level, clip activity), which a float32 recomputation of the forward could
// flip at a cell boundary -- where the bilinear derivatives jump.
__device__ __forceinline__ SsBil<float> ss_bil_narrow(const SsBil<double> &b) {
    SsBil<float> o;
    o.i0 = b.i0; o.i1 = b.i1; o.j0 = b.j0; o.j1 = b.j1;
    o.tu = (float)b.tu; o.tv = (float)b.tv; o.du_ok = b.du_ok; o.dv_ok = b.dv_ok;
    return o;
}
__device__ __forceinline__ void ss_shade_narrow(const ShadeIn<double> &a, const ShadeState<double> &s,
                                                ShadeIn<float> &af, ShadeState<float> &sf) {
    for (int c = 0; c < 3; ++c) {
        af.albedo[c] = (float)a.albedo[c]; af.n[c] = (float)a.n[c]; af.wo[c] = (float)a.wo[c];
        sf.refl[c] = (float)s.refl[c]; sf.l_d[c] = (float)s.l_d[c]; sf.l_s[c] = (float)s.l_s[c];
        sf.spec_lo[c] = (float)s.spec_lo[c]; sf.spec_hi[c] = (float)s.spec_hi[c];
        sf.f0[c] = (float)s.f0[c]; sf.k_d[c] = (float)s.k_d[c];
    }
    af.m = (float)a.m; af.r = (float)a.r; af.inv_dist = (float)a.inv_dist;
    sf.ndv_raw = (float)s.ndv_raw; sf.b1 = (float)s.b1; sf.b2 = (float)s.b2; sf.frac = (float)s.frac;
    // the clip-activity flags follow the float64 ndv (narrowing could move
    // a value within 1 ulp of 0 or 1 across the bound)
    if ((s.ndv_raw > 0.0) != (sf.ndv_raw > 0.f)) sf.ndv_raw = s.ndv_raw > 0.0 ? 1e-30f : 0.f;
    if ((s.ndv_raw < 1.0) != (sf.ndv_raw < 1.f)) sf.ndv_raw = s.ndv_raw < 1.0 ? 0.99999994f : 1.f;
    sf.lvl0 = s.lvl0; sf.lvl1 = s.lvl1;
    sf.bd = ss_bil_narrow(s.bd); sf.bs = ss_bil_narrow(s.bs); sf.bl = ss_bil_narrow(s.bl);
}

// The float64 forward's branch state, packed (SsProjAux.cells_packed).
template <typename R>
__device__ __forceinline__ uint4 ss_shade_pack(const ShadeState<R> &s) {
    const unsigned flags = (s.bd.dv_ok ? 1u : 0u) | (s.bs.dv_ok ? 2u : 0u) | (s.bl.du_ok ? 4u : 0u) |
                           (s.bl.dv_ok ? 8u : 0u) | (s.ndv_raw > R(0.0) ? 16u : 0u) | (s.ndv_raw < R(1.0) ? 32u : 0u);
    return make_uint4((unsigned)s.bd.i0 | ((unsigned)s.bd.j0 << 16), (unsigned)s.bs.i0 | ((unsigned)s.bs.j0 << 16),
                      (unsigned)s.bl.i0 | ((unsigned)s.bl.j0 << 16), (unsigned)s.lvl0 | (flags << 8));
}

// A bilinear cell forced to (i0, j0): the weights from this evaluation's own
// coordinates relative to the forced cell (wrapping columns: the nearest
// image of fu).
__device__ __forceinline__ SsBil<float> ss_bil_forced(int h, int w, float fu, float fv, bool wrap, unsigned cell,
                                                      bool du_ok, bool dv_ok) {
    SsBil<float> b;
    b.i0 = (int)(cell & 0xffffu);
    b.j0 = (int)(cell >> 16);
    b.j1 = b.j0 + 1;
    b.tv = ss_clip<float>(fv, 0.f, h - 1.f) - (float)b.j0;
    if (wrap) {
        float t = fu - (float)b.i0;
        if (t < -0.5f * w) t += (float)w;
        else if (t > 0.5f * w) t -= (float)w;
        b.tu = t;
        b.i1 = b.i0 + 1 == w ? 0 : b.i0 + 1;
    } else {
        b.tu = ss_clip<float>(fu, 0.f, w - 1.f) - (float)b.i0;
        b.i1 = b.i0 + 1;
    }
    b.du_ok = du_ok;
    b.dv_ok = dv_ok;
    return b;
}

// shade_surfels body in float32 on the branch state of the float64 forward
// (ss_shade_pack): the state the adjoint needs, without re-deriving the
// cells in float64.
// pd (nullable): the step's float32 diffuse state (prepass.cuh PreDiff: l_d,
// texel derivatives and the coord_grad_to_dir map of the normal), which the
// lookup and its adjoint then take instead of re-deriving them per view.
__device__ __forceinline__ void ss_shade_forward_cells(const ShadeIn<float> &in, const SsEnv &env, uint4 cells,
                                                       ShadeState<float> &s, const float *pd = nullptr) {
    const int he = env.he, we = env.we, L = env.levels, LR = env.lut_res;
    const unsigned fl = cells.w >> 8;
    s.ndv_raw = (in.n[0] * in.wo[0] + in.n[1] * in.wo[1]) + in.n[2] * in.wo[2];
    // the clip-activity flags are the float64 forward's
    if ((s.ndv_raw > 0.f) != ((fl & 16u) != 0)) s.ndv_raw = (fl & 16u) ? 1e-30f : 0.f;
    if ((s.ndv_raw < 1.f) != ((fl & 32u) != 0)) s.ndv_raw = (fl & 32u) ? 0.99999994f : 1.f;
    const float ndv = ss_clip<float>(s.ndv_raw, 0.f, 1.f);
    for (int c = 0; c < 3; ++c) s.refl[c] = 2.f * s.ndv_raw * in.n[c] - in.wo[c];
    float fu, fv;
    s.dpre = pd != nullptr;
    if (pd) {  // PreDiff: l_d[3] gu[3] gv[3] a0 a1 b2 tu tv
        const float4 p0 = reinterpret_cast<const float4 *>(pd)[0], p1 = reinterpret_cast<const float4 *>(pd)[1];
        const float4 p2 = reinterpret_cast<const float4 *>(pd)[2], p3 = reinterpret_cast<const float4 *>(pd)[3];
        s.l_d[0] = p0.x; s.l_d[1] = p0.y; s.l_d[2] = p0.z;
        s.dgu[0] = p0.w; s.dgu[1] = p1.x; s.dgu[2] = p1.y;
        s.dgv[0] = p1.z; s.dgv[1] = p1.w; s.dgv[2] = p2.x;
        s.da0 = p2.y; s.da1 = p2.z; s.db2 = p2.w;
        s.bd.i0 = (int)(cells.x & 0xffffu); s.bd.j0 = (int)(cells.x >> 16);
        s.bd.i1 = s.bd.i0 + 1 == we ? 0 : s.bd.i0 + 1; s.bd.j1 = s.bd.j0 + 1;
        s.bd.tu = p3.x; s.bd.tv = p3.y; s.bd.du_ok = true; s.bd.dv_ok = (fl & 1u) != 0;
    } else {
        ss_dir_coords(in.n, he, we, fu, fv);
        s.bd = ss_bil_forced(he, we, fu, fv, true, cells.x, true, (fl & 1u) != 0);
        ss_bil_lookup_grads4(reinterpret_cast<const float4 *>(env.diffuse4), we, s.bd, s.l_d, s.dgu, s.dgv);
    }
    const float4 *s4 = reinterpret_cast<const float4 *>(env.specular4);
    const float lvl = ss_clip<float>(in.r, 0.f, 1.f) * (L - 1);
    s.lvl0 = (int)(cells.w & 0xffu);
    s.frac = L > 1 ? lvl - (float)s.lvl0 : 0.f;
    s.lvl1 = s.lvl0 + 1 < L - 1 ? s.lvl0 + 1 : L - 1;
    ss_dir_coords(s.refl, he, we, fu, fv);
    s.bs = ss_bil_forced(he, we, fu, fv, true, cells.y, true, (fl & 2u) != 0);
    ss_bil_lookup_grads4(s4 + (size_t)he * we * s.lvl0, we, s.bs, s.spec_lo, s.sgu[0], s.sgv[0]);
    ss_bil_lookup_grads4(s4 + (size_t)he * we * s.lvl1, we, s.bs, s.spec_hi, s.sgu[1], s.sgv[1]);
    for (int c = 0; c < 3; ++c) s.l_s[c] = (1.f - s.frac) * s.spec_lo[c] + s.frac * s.spec_hi[c];
    s.bl = ss_bil_forced(LR, LR, ndv * (LR - 1), in.r * (LR - 1), false, cells.z, (fl & 4u) != 0, (fl & 8u) != 0);
    float bb[2];
    ss_bil_lookup_grads<2>(env.lut, LR, s.bl, bb, s.lgu, s.lgv);
    s.b1 = bb[0]; s.b2 = bb[1];
    for (int c = 0; c < 3; ++c) {
        s.f0[c] = 0.04f * (1.f - in.m) + in.albedo[c] * in.m;
        s.k_d[c] = (1.f - s.f0[c]) * (1.f - in.m);
    }
}

// Branch signature cells (shading.py:490-497), 15 ints.
template <typename R>
__device__ __forceinline__ void ss_shade_cells(const ShadeState<R> &s, const SsEnv &env, int32_t *out) {
    out[0] = s.bd.i0; out[1] = s.bd.j0; out[2] = s.bd.du_ok; out[3] = s.bd.dv_ok;
    out[4] = s.bs.i0; out[5] = s.bs.j0; out[6] = s.bs.du_ok; out[7] = s.bs.dv_ok;
    out[8] = s.lvl0;
    out[9] = s.bl.i0; out[10] = s.bl.j0; out[11] = s.bl.du_ok; out[12] = s.bl.dv_ok;
    out[13] = s.ndv_raw > R(0.0); out[14] = s.ndv_raw < R(1.0);
}

template <typename R>
struct ShadeGrads {
    R albedo_raw[3], metallic_raw, roughness_raw, normal[3], center[3];
    R g_ls[3], g_ld[3];   // derived-map upstreams for the env scatter
};

// shade_backward for one surfel (shading.py:525-615), env adjoint excluded.
// kStored: the texel derivatives come from the forward state (one texel
// read per lookup); else they are re-read here
template <typename R, bool kStored = false>
__device__ __forceinline__ void ss_shade_backward(const ShadeIn<R> &in, const ShadeState<R> &s, const SsEnv &env,
                                                  const R g[3], ShadeGrads<R> &o) {
    const int he = env.he, we = env.we, L = env.levels, LR = env.lut_res;
    R g_kd[3], g_alb[3], g_f0[3];
    for (int c = 0; c < 3; ++c) {
        g_kd[c] = g[c] * in.albedo[c] * s.l_d[c];
        g_alb[c] = g[c] * s.k_d[c] * s.l_d[c];
        o.g_ld[c] = g[c] * s.k_d[c] * in.albedo[c];
        o.g_ls[c] = g[c] * (s.f0[c] * s.b1 + s.b2);
        g_f0[c] = g[c] * s.l_s[c] * s.b1;
    }
    R g_b1 = (g[0] * s.l_s[0] * s.f0[0] + g[1] * s.l_s[1] * s.f0[1]) + g[2] * s.l_s[2] * s.f0[2];
    R g_b2 = (g[0] * s.l_s[0] + g[1] * s.l_s[1]) + g[2] * s.l_s[2];
    for (int c = 0; c < 3; ++c) g_f0[c] += g_kd[c] * (-(R(1.0) - in.m));
    R g_met = (g_kd[0] * (-(R(1.0) - s.f0[0])) + g_kd[1] * (-(R(1.0) - s.f0[1]))) + g_kd[2] * (-(R(1.0) - s.f0[2]));
    g_met += (g_f0[0] * (in.albedo[0] - R(0.04)) + g_f0[1] * (in.albedo[1] - R(0.04))) + g_f0[2] * (in.albedo[2] - R(0.04));
    for (int c = 0; c < 3; ++c) g_alb[c] += g_f0[c] * in.m;
    R dfx[2], dfy[2];
    if constexpr (kStored) {
        dfx[0] = s.lgu[0]; dfx[1] = s.lgu[1]; dfy[0] = s.lgv[0]; dfy[1] = s.lgv[1];
    } else {
        ss_bil_grads<2>(env.lut, LR, s.bl, dfx, dfy);
    }
    R g_ndv = (g_b1 * dfx[0] + g_b2 * dfx[1]) * (LR - 1);
    R g_rough = (g_b1 * dfy[0] + g_b2 * dfy[1]) * (LR - 1);
    bool active = (s.ndv_raw > R(0.0)) && (s.ndv_raw < R(1.0));
    if (!active) g_ndv = R(0.0);
    if (L > 1) {
        R acc = (o.g_ls[0] * (s.spec_hi[0] - s.spec_lo[0]) + o.g_ls[1] * (s.spec_hi[1] - s.spec_lo[1])) +
                     o.g_ls[2] * (s.spec_hi[2] - s.spec_lo[2]);
        g_rough += acc * (L - 1);
    }
    R g_refl[3] = {R(0.0), R(0.0), R(0.0)};
    const size_t lstride = (size_t)he * we * 3;
    const R wts[2] = {R(1.0) - s.frac, s.frac};
    const int lv[2] = {s.lvl0, s.lvl1};
    for (int h = 0; h < 2; ++h) {
        R gu[3], gv[3];
        if constexpr (kStored) {
            for (int c = 0; c < 3; ++c) { gu[c] = s.sgu[h][c]; gv[c] = s.sgv[h][c]; }
        } else if (env.specular4) {
            ss_bil_grads4(reinterpret_cast<const float4 *>(env.specular4) + (size_t)he * we * lv[h], we, s.bs, gu, gv);
        } else {
            ss_bil_grads<3>(env.specular + lstride * lv[h], we, s.bs, gu, gv);
        }
        R gh0 = o.g_ls[0] * wts[h], gh1 = o.g_ls[1] * wts[h], gh2 = o.g_ls[2] * wts[h];
        R gfu = (gh0 * gu[0] + gh1 * gu[1]) + gh2 * gu[2];
        R gfv = (gh0 * gv[0] + gh1 * gv[1]) + gh2 * gv[2];
        R gd[3];
        ss_coord_grad_to_dir(s.refl, he, we, gfu, gfv, gd);
        for (int c = 0; c < 3; ++c) g_refl[c] += gd[c];
    }
    R gu[3], gv[3];
    if constexpr (kStored) {
        for (int c = 0; c < 3; ++c) { gu[c] = s.dgu[c]; gv[c] = s.dgv[c]; }
    } else if (env.diffuse4) {
        ss_bil_grads4(reinterpret_cast<const float4 *>(env.diffuse4), we, s.bd, gu, gv);
    } else {
        ss_bil_grads<3>(env.diffuse, we, s.bd, gu, gv);
    }
    R gfu = (o.g_ld[0] * gu[0] + o.g_ld[1] * gu[1]) + o.g_ld[2] * gu[2];
    R gfv = (o.g_ld[0] * gv[0] + o.g_ld[1] * gv[1]) + o.g_ld[2] * gv[2];
    R g_n[3];
    if (kStored && s.dpre) {
        g_n[0] = gfu * s.da0; g_n[1] = gfu * s.da1; g_n[2] = gfv * s.db2;
    } else {
        ss_coord_grad_to_dir(in.n, he, we, gfu, gfv, g_n);
    }
    R grn = (g_refl[0] * in.n[0] + g_refl[1] * in.n[1]) + g_refl[2] * in.n[2];
    R g_wo[3];
    for (int c = 0; c < 3; ++c) {
        g_n[c] += R(2.0) * grn * in.wo[c] + R(2.0) * s.ndv_raw * g_refl[c];
        g_wo[c] = R(2.0) * grn * in.n[c] - g_refl[c];
    }
    R gnd = active ? g_ndv : R(0.0);
    for (int c = 0; c < 3; ++c) { g_n[c] += gnd * in.wo[c]; g_wo[c] += gnd * in.n[c]; }
    R radial = (g_wo[0] * in.wo[0] + g_wo[1] * in.wo[1]) + g_wo[2] * in.wo[2];
    for (int c = 0; c < 3; ++c) {
        o.center[c] = -(g_wo[c] - radial * in.wo[c]) * in.inv_dist;
        o.normal[c] = g_n[c];
        o.albedo_raw[c] = g_alb[c] * in.albedo[c] * (R(1.0) - in.albedo[c]);
    }
    o.metallic_raw = g_met * in.m * (R(1.0) - in.m);
    o.roughness_raw = g_rough * in.r * (R(1.0) - in.r);
}
