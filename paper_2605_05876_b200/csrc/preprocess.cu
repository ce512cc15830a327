// preprocess.cu -- per-surfel projection, filter setup, bounding, shading and
// tile counting in ONE pass over the surfel parameters.
//
// Reference: preprocess.py:38-309 (float32 throughout), shading.py:447-503
// (float64), rasterizer.py:92-106 (tile spans).  Compiled with -fmad=false:
// every float32 expression below rounds each operation like numpy does; the
// two BLAS inner products are written as the explicit fmaf chains numpy's
// OpenBLAS kernels evaluate (hard part 1).
//
// HBM: reads 56 B of parameters per surfel (plus a few KB of env/LUT texels
// that stay in L1/L2), writes one 96 B record + 1 B cull + 4 B pair count.
#include "ss_common.cuh"
#include "shading.cuh"
#include "coverage.cuh"
#include "prepass.cuh"

namespace {

__device__ __forceinline__ float dot_gemm(float a0, float a1, float a2, float b0, float b1, float b2) {
    return __fmaf_rn(a2, b2, __fmaf_rn(a1, b1, a0 * b0));
}
__device__ __forceinline__ float dot_gemv(float a0, float a1, float a2, float v0, float v1, float v2) {
    return __fmaf_rn(a2, v2, __fmaf_rn(a0, v0, a1 * v1));
}
__device__ __forceinline__ float npmaxf(float a, float b) { return (a != a) ? a : (a > b ? a : b); }
__device__ __forceinline__ float npclipf(float a, float lo, float hi) {
    if (a != a) return a;
    return a < lo ? lo : (a > hi ? hi : a);
}

struct CamF {
    float view[16], proj[16];
    double cam_pos[3];
    int W, H;
    SsPixelSteps px;
};

// View-independent per-surfel state of one optimisation step
// (ss_surfel_prepass): the float32 scaled tangent frame and the float64
// shading inputs plus the diffuse lookup, computed once per step instead of
// once per view, with exactly the preprocess kernel's operations (this file
// is compiled with -fmad=false), so the records are bit-identical.
// (PreGeom, PreShade, PreDiff: prepass.cuh)

// quat_to_frame + exp(log_scales) in float32 (surfels.py:40-51), the
// preprocess kernel's expressions
__device__ __forceinline__ void scaled_frame(float4 q, float2 ls, float &nrm, float s[6]) {
    nrm = sqrtf(((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w);
    float w = q.x / nrm, x = q.y / nrm, y = q.z / nrm, z = q.w / nrm;
    float uh0 = 1.0f - 2.0f * (y * y + z * z), uh1 = 2.0f * (x * y + w * z), uh2 = 2.0f * (x * z - w * y);
    float vh0 = 2.0f * (x * y - w * z), vh1 = 1.0f - 2.0f * (x * x + z * z), vh2 = 2.0f * (y * z + w * x);
    // numpy's float32 exp is a SIMD kernel; the correctly rounded value is the
    // documented stand-in (oracle/ss_oracle.c does the same).
    float su = (float)exp((double)ls.x), sv = (float)exp((double)ls.y);
    s[0] = su * uh0; s[1] = su * uh1; s[2] = su * uh2;
    s[3] = sv * vh0; s[4] = sv * vh1; s[5] = sv * vh2;
}

__global__ void __launch_bounds__(256) surfel_prepass_kernel(SsCloud cloud, SsEnv env, int shade,
                                                             PreGeom *__restrict__ geom,
                                                             PreShade *__restrict__ sh, PreDiff *__restrict__ pd) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cloud.n) return;
    const float4 q = reinterpret_cast<const float4 *>(cloud.quats)[i];
    const float2 ls = reinterpret_cast<const float2 *>(cloud.log_scales)[i];
    const bool finite = isfinite(cloud.centers[3 * i]) && isfinite(cloud.centers[3 * i + 1]) &&
                        isfinite(cloud.centers[3 * i + 2]) && isfinite(q.x) && isfinite(q.y) && isfinite(q.z) &&
                        isfinite(q.w) && isfinite(ls.x) && isfinite(ls.y) && isfinite(cloud.albedo_raw[3 * i]) &&
                        isfinite(cloud.albedo_raw[3 * i + 1]) && isfinite(cloud.albedo_raw[3 * i + 2]) &&
                        isfinite(cloud.metallic_raw[i]) && isfinite(cloud.roughness_raw[i]);
    float nrm, f[6];
    scaled_frame(q, ls, nrm, f);
    PreGeom g;
    g.su0 = f[0]; g.su1 = f[1]; g.su2 = f[2]; g.sv0 = f[3]; g.sv1 = f[4]; g.sv2 = f[5];
    g.finite = finite;
    g.zero_norm = nrm == 0.0f;
    geom[i] = g;
    if (!shade) return;
    ShadeIn<double> in;
    ss_shade_material(cloud, i, in);
    SsBil<double> bd;
    PreShade o;
    ss_shade_diffuse(in.n, env, bd, o.l_d);
    for (int c = 0; c < 3; ++c) { o.n[c] = in.n[c]; o.alb[c] = (float)in.albedo[c]; }
    o.m = (float)in.m; o.r = (float)in.r;
    o.cell = (unsigned)bd.i0 | ((unsigned)bd.j0 << 16);
    o.dv_ok = bd.dv_ok;
    o.pad = 0;
    sh[i] = o;
    if (!env.diffuse4) return;
    // the chain kernel's float32 diffuse state on this cell (its
    // ss_shade_forward_cells / ss_shade_backward diffuse part, once per step)
    ShadeIn<float> inf;
    ss_shade_material(cloud, i, inf);
    float fu, fv;
    ss_dir_coords(inf.n, env.he, env.we, fu, fv);
    const SsBil<float> b = ss_bil_forced(env.he, env.we, fu, fv, true, o.cell, true, bd.dv_ok);
    PreDiff d;
    ss_bil_lookup_grads4(reinterpret_cast<const float4 *>(env.diffuse4), env.we, b, d.l_d, d.gu, d.gv);
    float ga[3], gb[3];
    ss_coord_grad_to_dir(inf.n, env.he, env.we, 1.f, 0.f, ga);
    ss_coord_grad_to_dir(inf.n, env.he, env.we, 0.f, 1.f, gb);
    d.a0 = ga[0]; d.a1 = ga[1]; d.b2 = gb[2];
    d.tu = b.tu; d.tv = b.tv;
    d.pad[0] = d.pad[1] = 0.f;
    pd[i] = d;
}

#ifndef SS_PRE_MINB
#define SS_PRE_MINB 3  // 80 registers, 3 CTAs per SM (small spill, better latency hiding)
#endif
__global__ void __launch_bounds__(256, SS_PRE_MINB) preprocess_kernel(
    SsCloud cloud, CamF cam, SsPreprocessOpts opt, int color_source, const float *__restrict__ colors_in,
    SsEnv env, SsRecord *__restrict__ records, int8_t *__restrict__ cull_out,
    int32_t *__restrict__ pair_count, int32_t *__restrict__ tile_counts, uint4 *__restrict__ bininfo, SsProjAux aux,
    int32_t *__restrict__ flags, const PreGeom *__restrict__ pre_geom, const PreShade *__restrict__ pre_shade)
{
    const int i_raw = blockIdx.x * blockDim.x + threadIdx.x;
    const bool in_range = i_raw < cloud.n;
    const int i = in_range ? i_raw : cloud.n - 1;  // tail lanes recompute the last row, write nothing
    const float c0 = cloud.centers[3 * i], c1 = cloud.centers[3 * i + 1], c2 = cloud.centers[3 * i + 2];
    float su0, su1, su2, sv0, sv1, sv2;
    bool finite;
    if (pre_geom) {  // this step's prepass (ss_surfel_prepass)
        const PreGeom g = pre_geom[i];
        su0 = g.su0; su1 = g.su1; su2 = g.su2; sv0 = g.sv0; sv1 = g.sv1; sv2 = g.sv2;
        finite = in_range && g.finite;
        if (in_range && g.zero_norm) atomicOr(&flags[0], 1);
    } else {
        const float4 q = reinterpret_cast<const float4 *>(cloud.quats)[i];
        const float2 ls = reinterpret_cast<const float2 *>(cloud.log_scales)[i];
        finite = in_range && isfinite(c0) && isfinite(c1) && isfinite(c2) && isfinite(q.x) && isfinite(q.y) &&
                 isfinite(q.z) && isfinite(q.w) && isfinite(ls.x) && isfinite(ls.y) &&
                 isfinite(cloud.albedo_raw[3 * i]) && isfinite(cloud.albedo_raw[3 * i + 1]) &&
                 isfinite(cloud.albedo_raw[3 * i + 2]) && isfinite(cloud.metallic_raw[i]) &&
                 isfinite(cloud.roughness_raw[i]);
        // quat_to_frame in float32 (surfels.py:40-51)
        float nrm, f[6];
        scaled_frame(q, ls, nrm, f);
        if (in_range && nrm == 0.0f) atomicOr(&flags[0], 1);
        su0 = f[0]; su1 = f[1]; su2 = f[2]; sv0 = f[3]; sv1 = f[4]; sv2 = f[5];
    }
    int code = finite ? 0 : 1;
    float cc[3], tu[3], tv[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const float R0 = cam.view[4 * r], R1 = cam.view[4 * r + 1], R2 = cam.view[4 * r + 2];
        cc[r] = dot_gemm(c0, c1, c2, R0, R1, R2) + cam.view[4 * r + 3];
        tu[r] = dot_gemm(su0, su1, su2, R0, R1, R2);
        tv[r] = dot_gemm(sv0, sv1, sv2, R0, R1, R2);
    }
    const float vz = -cc[2];
    float t[3][3];
    const int irs[3] = {0, 1, 3};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float *P = cam.proj + 4 * irs[k];
        t[k][0] = dot_gemv(tu[0], tu[1], tu[2], P[0], P[1], P[2]);
        t[k][1] = dot_gemv(tv[0], tv[1], tv[2], P[0], P[1], P[2]);
        t[k][2] = dot_gemv(cc[0], cc[1], cc[2], P[0], P[1], P[2]) + P[3];
    }
    const float *t1 = t[0], *t2 = t[1], *t4 = t[2];
    if (code == 0 && !(vz >= SS_VIEW_Z_EPS)) code = 2;
    bool alive = code == 0;
    const float ez = opt.r_cut * sqrtf(tu[2] * tu[2] + tv[2] * tv[2]);
    const float sd4 = alive ? t4[2] : 1.0f;
    const float cnx = t1[2] / sd4, cny = t2[2] / sd4;

    float j00 = 0.f, j01 = 0.f, j10 = 0.f, j11 = 0.f;
    bool ok = false;
    float m00 = 1.f, m01 = 0.f, m11 = 1.f, nf = 1.f;
    float tb[3][3];
    if (opt.mip_enabled) {
        float jj[4];
        ok = ss_center_jacobian(t1, t2, t4, cam.px.dxp, cam.px.dyp, jj);
        if (ok && alive) { j00 = jj[0]; j01 = jj[1]; j10 = jj[2]; j11 = jj[3]; }
        const float s = opt.mip_sigma;
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
        float lc = sqrtf(npmaxf(1.0f + s * jjt11 - lb * lb, 1.17549435e-38f));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            tb[k][0] = la * t[k][0] + lb * t[k][1];
            tb[k][1] = lc * t[k][1];
            tb[k][2] = t[k][2];
        }
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) { tb[k][0] = t[k][0]; tb[k][1] = t[k][1]; tb[k][2] = t[k][2]; }
    }
    // bounding_rect (preprocess.py:77-105)
    const float rr2 = opt.r_cut * opt.r_cut;
    const float *b4 = tb[2];
    float f44 = b4[2] * b4[2] - rr2 * (b4[0] * b4[0] + b4[1] * b4[1]);
    bool valid = f44 > 0.0f;
    float f44s = valid ? f44 : 1.0f;
    float ctr[2], half[2];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        const float *tr = tb[a];
        float fi4 = tr[2] * b4[2] - rr2 * (tr[0] * b4[0] + tr[1] * b4[1]);
        float fii = tr[2] * tr[2] - rr2 * (tr[0] * tr[0] + tr[1] * tr[1]);
        float disc = npmaxf(fi4 * fi4 - f44 * fii, 0.0f);
        ctr[a] = fi4 / f44s;
        half[a] = sqrtf(disc) / f44s;
    }
    if (alive && !valid) code = 3;
    alive = code == 0;
    const float fw = (float)cam.W, fh = (float)cam.H;
    float lo_x = ctr[0] - half[0], hi_x = ctr[0] + half[0];
    float lo_y = ctr[1] - half[1], hi_y = ctr[1] + half[1];
    float x0 = ceilf((lo_x + 1.0f) * 0.5f * fw - 0.5f - 9.99999975e-05f);
    float x1 = floorf((hi_x + 1.0f) * 0.5f * fw - 0.5f + 9.99999975e-05f) + 1.0f;
    float y0 = ceilf((1.0f - hi_y) * 0.5f * fh - 0.5f - 9.99999975e-05f);
    float y1 = floorf((1.0f - lo_y) * 0.5f * fh - 0.5f + 9.99999975e-05f) + 1.0f;
    x0 = npclipf(x0, 0.f, fw); x1 = npclipf(x1, 0.f, fw);
    y0 = npclipf(y0, 0.f, fh); y1 = npclipf(y1, 0.f, fh);
    if (alive && (x0 >= x1 || y0 >= y1)) code = 4;
    alive = code == 0;

    // colour (rasterizer.py:341-353)
    float col[3] = {0.f, 0.f, 0.f};
    if (color_source == SS_COLOR_EXPLICIT) {
        col[0] = colors_in[3 * i]; col[1] = colors_in[3 * i + 1]; col[2] = colors_in[3 * i + 2];
#ifdef SS_EXP_NO_SHADE
    } else if (true) {
        col[0] = ss_sigmoid_f32(cloud.albedo_raw[3 * i]); col[1] = ss_sigmoid_f32(cloud.albedo_raw[3 * i + 1]);
    col[2] = ss_sigmoid_f32(cloud.albedo_raw[3 * i + 2]);
#endif
    } else if (color_source == SS_COLOR_ALBEDO) {
        col[0] = ss_sigmoid_f32(cloud.albedo_raw[3 * i]); col[1] = ss_sigmoid_f32(cloud.albedo_raw[3 * i + 1]);
        col[2] = ss_sigmoid_f32(cloud.albedo_raw[3 * i + 2]);
    } else if (color_source == SS_COLOR_IBL && pre_shade) {
        // materials, normal and the diffuse lookup from this step's prepass
        const PreShade &ps = pre_shade[i];
        ShadeIn<double> in;
        for (int c = 0; c < 3; ++c) { in.n[c] = ps.n[c]; in.albedo[c] = (double)ps.alb[c]; }
        in.m = (double)ps.m; in.r = (double)ps.r;
        ss_shade_view(cloud, i, cam.cam_pos, in);
        ShadeState<double> st;
        for (int c = 0; c < 3; ++c) st.l_d[c] = ps.l_d[c];
        st.bd.i0 = (int)(ps.cell & 0xffffu); st.bd.j0 = (int)(ps.cell >> 16);
        st.bd.du_ok = true; st.bd.dv_ok = ps.dv_ok != 0;
        double out[3];
        ss_shade_forward_view(in, env, st, out);
        col[0] = (float)out[0]; col[1] = (float)out[1]; col[2] = (float)out[2];
        if (aux.cells) ss_shade_cells(st, env, aux.cells + 15 * i);
        if (aux.cells_packed && in_range) reinterpret_cast<uint4 *>(aux.cells_packed)[i] = ss_shade_pack(st);
    } else if (color_source == SS_COLOR_IBL_F32) {
        ShadeIn<float> in;
        ss_shade_inputs(cloud, i, cam.cam_pos, in);
        ShadeState<float> st;
        ss_shade_forward(in, env, st, col);
        if (aux.cells) ss_shade_cells(st, env, aux.cells + 15 * i);
    } else {
        ShadeIn<double> in;
        ss_shade_inputs(cloud, i, cam.cam_pos, in);
        ShadeState<double> st;
        double out[3];
        ss_shade_forward(in, env, st, out);
        col[0] = (float)out[0]; col[1] = (float)out[1]; col[2] = (float)out[2];
        if (aux.cells) ss_shade_cells(st, env, aux.cells + 15 * i);
        if (aux.cells_packed && in_range) reinterpret_cast<uint4 *>(aux.cells_packed)[i] = ss_shade_pack(st);
    }
    if (in_range && !(isfinite(col[0]) && isfinite(col[1]) && isfinite(col[2]))) atomicOr(&flags[1], 1);

    const float zs = vz - ez, ze = vz + ez;
    SsRecord rec;
    rec.a = make_float4(t1[0], t1[1], t1[2], t2[0]);
    rec.b = make_float4(t2[1], t2[2], t4[0], t4[1]);
    rec.c = make_float4(t4[2], m00, m01, m11);
    rec.d = make_float4(nf, vz, zs, ze);
    // e.w: certified fast-coverage margin of this record (coverage.cuh)
#ifdef SS_EXP_NO_MARGIN
    const float cm = alive ? 1.f
#else
    const float cm = alive ? coverage_margin(t1, t2, t4, m00, m01, m11, (int)x0, (int)y0, (int)x1, (int)y1, cam.px.two_w,
                                            cam.px.two_h)
#endif
                           : 0.f;
    rec.e = make_float4(col[0], col[1], col[2], cm);
    int count = 0;
    const int tile = opt.tile;
    const int ntx = (cam.W + tile - 1) / tile;
    int tx0 = 0, ty0 = 0, sx = 1;
    if (alive) {
        int ix0 = (int)x0, iy0 = (int)y0, ix1 = (int)x1, iy1 = (int)y1;
        rec.r = make_int4(ix0, iy0, ix1, iy1);
        tx0 = ix0 / tile; ty0 = iy0 / tile;
        const int tx1 = (ix1 - 1) / tile, ty1 = (iy1 - 1) / tile;
        sx = tx1 - tx0 + 1;
        count = sx * (ty1 - ty0 + 1);
    } else {
        rec.r = make_int4(0, 0, 0, 0);
    }
    // per-tile histogram (one global atomic per (record, tile); records in
    // source order spread over the image, so the counters see little contention)
    for (int s = 0, tx = tx0, ty = ty0; s < count; ++s) {
        atomicAdd(&tile_counts[ty * ntx + tx], 1);
        if (++tx == tx0 + sx) { tx = tx0; ++ty; }
    }
    if (!in_range) return;
    records[i] = rec;
    cull_out[i] = (int8_t)code;
    if (pair_count) pair_count[i] = count;
    // compact binning input (packed rect, sort key): 16 B instead of the 96 B record
    if (bininfo)
        bininfo[i] = alive ? make_uint4((uint32_t)rec.r.x | ((uint32_t)rec.r.y << 16),
                                        (uint32_t)rec.r.z | ((uint32_t)rec.r.w << 16), ss_orderable(zs), 0u)
                           : make_uint4(0u, 0u, 0u, 0u);
    if (aux.c_cam) {
        for (int k = 0; k < 3; ++k) { aux.c_cam[3 * i + k] = cc[k]; aux.tu_cam[3 * i + k] = tu[k]; aux.tv_cam[3 * i + k] = tv[k]; }
    }
    if (aux.eps_z) aux.eps_z[i] = ez;
    if (aux.center_ndc) { aux.center_ndc[2 * i] = cnx; aux.center_ndc[2 * i + 1] = cny; }
    if (aux.jac) {
        aux.jac[4 * i] = j00; aux.jac[4 * i + 1] = j01; aux.jac[4 * i + 2] = j10; aux.jac[4 * i + 3] = j11;
        aux.jac_ok[i] = ok ? 1 : 0;
    }
    if (aux.colors) { aux.colors[3 * i] = col[0]; aux.colors[3 * i + 1] = col[1]; aux.colors[3 * i + 2] = col[2]; }
}

// Records from a compacted ProjectedSurfels (render(proj=...) reuse and
// bin_and_sort(proj)): row k of the projection -> record source_index[k]
// (or k), with the same fields, certified margin, bin info and tile counts
// the preprocess kernel writes for a kept surfel.
__global__ void pack_kernel(int k, const float *__restrict__ t1, const float *__restrict__ t2,
                            const float *__restrict__ t4, const float *__restrict__ sinv, const float *__restrict__ n_f,
                            const float *__restrict__ view_z, const float *__restrict__ eps_z,
                            const int32_t *__restrict__ rect, const int32_t *__restrict__ source_index,
                            const float *__restrict__ colors, int W, int H, int tile, SsRecord *__restrict__ records,
                            uint4 *__restrict__ bininfo, int32_t *__restrict__ tile_counts)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    const int i = source_index ? source_index[j] : j;
    const float a1[3] = {t1[3 * j], t1[3 * j + 1], t1[3 * j + 2]};
    const float a2[3] = {t2[3 * j], t2[3 * j + 1], t2[3 * j + 2]};
    const float a4[3] = {t4[3 * j], t4[3 * j + 1], t4[3 * j + 2]};
    const float m00 = sinv[3 * j], m01 = sinv[3 * j + 1], m11 = sinv[3 * j + 2];
    const float vz = view_z[j], ez = eps_z[j];
    const float zs = vz - ez, ze = vz + ez;  // ProjectedSurfels.z_start / z_end (preprocess.py:217-223)
    const int x0 = rect[4 * j], y0 = rect[4 * j + 1], x1 = rect[4 * j + 2], y1 = rect[4 * j + 3];
    SsRecord rec;
    rec.a = make_float4(a1[0], a1[1], a1[2], a2[0]);
    rec.b = make_float4(a2[1], a2[2], a4[0], a4[1]);
    rec.c = make_float4(a4[2], m00, m01, m11);
    rec.d = make_float4(n_f[j], vz, zs, ze);
    const bool alive = x1 > x0 && y1 > y0;
    const float cm = alive ? coverage_margin(a1, a2, a4, m00, m01, m11, x0, y0, x1, y1, 2.0 / W, 2.0 / H) : 0.f;
    const float c0 = colors ? colors[3 * i] : 0.f, c1 = colors ? colors[3 * i + 1] : 0.f,
                c2 = colors ? colors[3 * i + 2] : 0.f;
    rec.e = make_float4(c0, c1, c2, cm);
    rec.r = alive ? make_int4(x0, y0, x1, y1) : make_int4(0, 0, 0, 0);
    records[i] = rec;
    bininfo[i] = alive ? make_uint4((uint32_t)x0 | ((uint32_t)y0 << 16), (uint32_t)x1 | ((uint32_t)y1 << 16),
                                    ss_orderable(zs), 0u)
                       : make_uint4(0u, 0u, 0u, 0u);
    if (!alive) return;
    const int ntx = (W + tile - 1) / tile;
    for (int ty = y0 / tile; ty <= (y1 - 1) / tile; ++ty)
        for (int tx = x0 / tile; tx <= (x1 - 1) / tile; ++tx) atomicAdd(&tile_counts[ty * ntx + tx], 1);
}

}  // namespace

extern "C" int ss_pack_records(int k, const float *t1, const float *t2, const float *t4, const float *sinv,
                               const float *n_f, const float *view_z, const float *eps_z, const int32_t *rect,
                               const int32_t *source_index, const float *colors, int width, int height, int tile,
                               float *records, uint32_t *bininfo, int32_t *tile_counts, void *stream)
{
    if (k < 0 || width <= 0 || height <= 0 || width > 65535 || height > 65535 || tile <= 0) return SS_ERR_INVALID;
    if (k == 0) return SS_OK;
    if (!t1 || !t2 || !t4 || !sinv || !n_f || !view_z || !eps_z || !rect || !records || !bininfo || !tile_counts)
        return SS_ERR_INVALID;
    pack_kernel<<<(k + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        k, t1, t2, t4, sinv, n_f, view_z, eps_z, rect, source_index, colors, width, height, tile,
        reinterpret_cast<SsRecord *>(records), reinterpret_cast<uint4 *>(bininfo), tile_counts);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" size_t ss_surfel_prepass_bytes(int n) {
    return n < 0 ? 0 : (sizeof(PreGeom) + sizeof(PreShade) + sizeof(PreDiff)) * (size_t)n;
}

extern "C" int ss_surfel_prepass(const SsCloud *cloud, const SsEnv *env, void *prepass, void *stream)
{
    if (!cloud || !prepass) return SS_ERR_INVALID;
    if (cloud->n == 0) return SS_OK;
    const bool shade = env && env->diffuse && env->diffuse64 && env->specular64;
    PreGeom *g = reinterpret_cast<PreGeom *>(prepass);
    PreShade *sh = reinterpret_cast<PreShade *>(g + cloud->n);
    PreDiff *pd = reinterpret_cast<PreDiff *>(sh + cloud->n);
    surfel_prepass_kernel<<<(cloud->n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(*cloud, env ? *env : SsEnv{},
                                                                                     shade ? 1 : 0, g, sh, pd);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

static int preprocess_impl(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                           int color_source, const float *colors_in, const SsEnv *env,
                           float *records, int8_t *cull, int32_t *pair_count, int32_t *tile_counts,
                           uint32_t *bininfo, const SsProjAux *aux, int32_t *flags, const void *prepass,
                           void *stream)
{
    if (!cloud || !cam || !opt || !tile_counts || !flags) return SS_ERR_INVALID;
    if (cam->width <= 0 || cam->height <= 0 || opt->tile <= 0) return SS_ERR_INVALID;
    if (cloud->n == 0) return SS_OK;
    if (!records || !cull) return SS_ERR_INVALID;
    if (color_source == SS_COLOR_EXPLICIT && !colors_in) return SS_ERR_INVALID;
    if ((color_source == SS_COLOR_IBL || color_source == SS_COLOR_IBL_F32) &&
        (!env || !env->diffuse || !env->specular || !env->lut))
        return SS_ERR_INVALID;
    if (color_source < SS_COLOR_EXPLICIT || color_source > SS_COLOR_IBL_F32) return SS_ERR_INVALID;
    CamF cf;
    for (int k = 0; k < 16; ++k) { cf.view[k] = (float)cam->view[k]; cf.proj[k] = (float)cam->proj[k]; }
    // camera.py:69-72: position = -R^T t (float64)
    for (int k = 0; k < 3; ++k)
        cf.cam_pos[k] = -(cam->view[k] * cam->view[3] + cam->view[4 + k] * cam->view[7] + cam->view[8 + k] * cam->view[11]);
    cf.W = cam->width; cf.H = cam->height;
    cf.px = ss_pixel_steps(cf.W, cf.H);
    SsEnv e = env ? *env : SsEnv{};
    SsProjAux a = aux ? *aux : SsProjAux{};
    int blocks = (cloud->n + 255) / 256;
    const PreGeom *pg = reinterpret_cast<const PreGeom *>(prepass);
    // the shading part of the prepass is only written with the float64 maps
    const PreShade *ps = pg && e.diffuse64 && e.specular64 ? reinterpret_cast<const PreShade *>(pg + cloud->n) : nullptr;
    preprocess_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        *cloud, cf, *opt, color_source, colors_in, e, reinterpret_cast<SsRecord *>(records), cull,
        pair_count, tile_counts, reinterpret_cast<uint4 *>(bininfo), a, flags, pg, ps);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_preprocess(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                             int color_source, const float *colors_in, const SsEnv *env,
                             float *records, int8_t *cull, int32_t *pair_count, int32_t *tile_counts,
                             uint32_t *bininfo, const SsProjAux *aux, int32_t *flags, void *stream)
{
    return preprocess_impl(cloud, cam, opt, color_source, colors_in, env, records, cull, pair_count, tile_counts,
                           bininfo, aux, flags, nullptr, stream);
}

extern "C" int ss_preprocess_prepared(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                                      int color_source, const float *colors_in, const SsEnv *env,
                                      float *records, int8_t *cull, int32_t *pair_count, int32_t *tile_counts,
                                      uint32_t *bininfo, const SsProjAux *aux, int32_t *flags, const void *prepass,
                                      void *stream)
{
    if (!prepass) return SS_ERR_INVALID;
    return preprocess_impl(cloud, cam, opt, color_source, colors_in, env, records, cull, pair_count, tile_counts,
                           bininfo, aux, flags, prepass, stream);
}
