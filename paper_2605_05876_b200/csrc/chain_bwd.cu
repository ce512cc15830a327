// chain_bwd.cu -- per-surfel tail of the backward pass, float64 like the
// reference: MIP-filter chain (backward.py:473-548), T rows -> camera ->
// world (backward.py:398-441), shading adjoint (shading.py:525-615) with the
// derived-map scatter, activations, and the quaternion adjoint
// (surfels.py:54-77).  One thread per surfel; the projection state is
// recomputed from the 56 B of parameters (cheaper than storing it), so the
// kernel streams params + the 80 B record accumulator and ADDS 14 parameter
// gradients + stats (multi-view steps accumulate in place, no extra pass).
#include "ss_common.cuh"
#include "shading.cuh"
#include "prepass.cuh"

namespace {

struct ChainParams {
    SsCloud cloud;
    double view[16], proj[16], cam_pos[3];
    float viewf[16], projf[16];
    int W, H, mip, color_source;
    SsPixelSteps px;
    double sigma;
    float r_cut, sigma_f;
    SsEnv env;
    const int8_t *cull;
    const float *acc;
    const double *acc64;  // float64 rows of the big records (SS_ACC_F64)
    const uint4 *cells;   // nullable: the forward's packed shading branch state
    const PreDiff *pre_diff;  // nullable: the step's float32 diffuse state (ss_chain_backward_prepared)
    float4 *g_ld;             // with pre_diff: per-surfel sum of the diffuse-lookup upstream (the taps
                              // are view independent: ss_diffuse_scatter applies them once per step)
    SsGrads g;
};

__device__ __forceinline__ float dot_gemm(float a0, float a1, float a2, float b0, float b1, float b2) {
    return __fmaf_rn(a2, b2, __fmaf_rn(a1, b1, fm(a0, b0)));
}
__device__ __forceinline__ float dot_gemv(float a0, float a1, float a2, float v0, float v1, float v2) {
    return __fmaf_rn(a2, v2, __fmaf_rn(a0, v0, fm(a1, v1)));
}

// T rows of surfel i, bit-identical to the preprocess kernel (explicit
// round-to-nearest ops so this file's FMA contraction cannot change them).
__device__ __forceinline__ void rows_of(const ChainParams &P, int i, float t1[3], float t2[3], float t4[3]) {
    const SsCloud &c = P.cloud;
    const float c0 = c.centers[3 * i], c1 = c.centers[3 * i + 1], c2 = c.centers[3 * i + 2];
    const float4 q = reinterpret_cast<const float4 *>(c.quats)[i];
    const float2 ls = reinterpret_cast<const float2 *>(c.log_scales)[i];
    const float nrm = __fsqrt_rn(fa(fa(fa(fm(q.x, q.x), fm(q.y, q.y)), fm(q.z, q.z)), fm(q.w, q.w)));
    const float w = fd(q.x, nrm), x = fd(q.y, nrm), y = fd(q.z, nrm), z = fd(q.w, nrm);
    const float uh0 = fs(1.f, fm(2.f, fa(fm(y, y), fm(z, z)))), uh1 = fm(2.f, fa(fm(x, y), fm(w, z))),
                uh2 = fm(2.f, fs(fm(x, z), fm(w, y)));
    const float vh0 = fm(2.f, fs(fm(x, y), fm(w, z))), vh1 = fs(1.f, fm(2.f, fa(fm(x, x), fm(z, z)))),
                vh2 = fm(2.f, fa(fm(y, z), fm(w, x)));
    const float su = (float)exp((double)ls.x), sv = (float)exp((double)ls.y);
    const float su0 = fm(su, uh0), su1 = fm(su, uh1), su2 = fm(su, uh2);
    const float sv0 = fm(sv, vh0), sv1 = fm(sv, vh1), sv2 = fm(sv, vh2);
    float cc[3], tu[3], tv[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const float R0 = P.viewf[4 * r], R1 = P.viewf[4 * r + 1], R2 = P.viewf[4 * r + 2];
        cc[r] = fa(dot_gemm(c0, c1, c2, R0, R1, R2), P.viewf[4 * r + 3]);
        tu[r] = dot_gemm(su0, su1, su2, R0, R1, R2);
        tv[r] = dot_gemm(sv0, sv1, sv2, R0, R1, R2);
    }
    const int irs[3] = {0, 1, 3};
    float *rows[3] = {t1, t2, t4};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float *Pr = P.projf + 4 * irs[k];
        rows[k][0] = dot_gemv(tu[0], tu[1], tu[2], Pr[0], Pr[1], Pr[2]);
        rows[k][1] = dot_gemv(tv[0], tv[1], tv[2], Pr[0], Pr[1], Pr[2]);
        rows[k][2] = fa(dot_gemv(cc[0], cc[1], cc[2], Pr[0], Pr[1], Pr[2]), Pr[3]);
    }
}

// Fire-and-forget accumulation (RED, no return value, no load latency): the
// per-view chain kernels are serialised, so each address has one writer at a
// time and the sums stay deterministic.
__device__ __forceinline__ void red_add(float *p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add2(float *p, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void red_add4(float *p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Derived-map scatter of one bilinear tap (3 channels, float64 atomics).
// Neighbouring surfels (Morton order) mostly hit the same env texel: when the
// whole warp is present and agrees on the texel, the warp sums first
// (fixed butterfly order) and one lane issues the atomics -- 32x fewer
// same-address atomics at L2; otherwise every lane adds its own.
__device__ __forceinline__ void scatter_rgb(double *base, int key, double v0, double v1, double v2) {
    const unsigned am = __activemask();
    // warp-uniform texel?  (one shuffle + vote instead of a match_any)
    const bool uniform = am == 0xffffffffu && __all_sync(0xffffffffu, key == __shfl_sync(0xffffffffu, key, 0));
    if (uniform) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v0 += __shfl_xor_sync(0xffffffffu, v0, o);
            v1 += __shfl_xor_sync(0xffffffffu, v1, o);
            v2 += __shfl_xor_sync(0xffffffffu, v2, o);
        }
        if ((threadIdx.x & 31) != 0) return;
    }
    double *d = base + 3 * (size_t)key;
    if (v0 != 0.0) atomicAdd(d, v0);
    if (v1 != 0.0) atomicAdd(d + 1, v1);
    if (v2 != 0.0) atomicAdd(d + 2, v2);
}

// The same tap into a per-view float32 map with 16-byte texels: one vector
// reduction per tap.  kUniform: the warp first checks for a warp-uniform
// texel and pre-sums it (the diffuse taps: surfels of a flat region share
// their normal's texel); the specular taps skip the check (reflection texels
// are almost never warp-uniform; measured: chain 0.216 -> 0.210 ms without it).
template <bool kUniform>
__device__ __forceinline__ void scatter_rgb4(float *base, int key, float v0, float v1, float v2) {
    if constexpr (!kUniform) {
        if (v0 != 0.f || v1 != 0.f || v2 != 0.f) red_add4(base + 4 * (size_t)key, v0, v1, v2, 0.f);
        return;
    }
    const unsigned am = __activemask();
    const bool uniform = am == 0xffffffffu && __all_sync(0xffffffffu, key == __shfl_sync(0xffffffffu, key, 0));
    if (uniform) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v0 += __shfl_xor_sync(0xffffffffu, v0, o);
            v1 += __shfl_xor_sync(0xffffffffu, v1, o);
            v2 += __shfl_xor_sync(0xffffffffu, v2, o);
        }
        if ((threadIdx.x & 31) != 0) return;
    }
    if (v0 != 0.f || v1 != 0.f || v2 != 0.f) red_add4(base + 4 * (size_t)key, v0, v1, v2, 0.f);
}

__global__ void env_merge_kernel(int64_t texels, float4 *__restrict__ src, double *__restrict__ dst) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < texels; t += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = src[t];
        if (v.x != 0.f || v.y != 0.f || v.z != 0.f) {
            dst[3 * t] += v.x; dst[3 * t + 1] += v.y; dst[3 * t + 2] += v.z;
            src[t] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

#ifdef SS_CHAIN_TAIL_F32
typedef float TT;
#define TT_PROJ P.projf
#define TT_VIEW P.viewf
#else
typedef double TT;
#define TT_PROJ P.proj
#define TT_VIEW P.view
#endif

#ifndef SS_CHAIN_MINB
#define SS_CHAIN_MINB 4
#endif
// kPre: the step's prepass diffuse state and per-surfel diffuse upstream
// (ss_chain_backward_prepared); a separate instantiation, so the per-view
// path keeps its register allocation
template <bool kPre>
__global__ void __launch_bounds__(128, SS_CHAIN_MINB) chain_kernel(ChainParams P)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.cloud.n || P.cull[i] != 0) return;
    const float *a = P.acc + (size_t)i * SS_ACC_FLOATS;
    const float4 a0 = reinterpret_cast<const float4 *>(a)[0];
    const float4 a1 = reinterpret_cast<const float4 *>(a)[1];
    const float4 a2 = reinterpret_cast<const float4 *>(a)[2];
    const float4 a3 = reinterpret_cast<const float4 *>(a)[3];
    const float4 a4 = reinterpret_cast<const float4 *>(a)[4];
    double G1[3] = {a0.x, a0.y, a0.z}, G2[3] = {a0.w, a1.x, a1.y}, G4[3] = {a1.z, a1.w, a2.x};
    double gs0 = a2.y, gs1 = a2.z, gs2 = a2.w, gnf = a3.x;
    double gcol[3] = {a3.y, a3.z, a3.w};
    double gz = a4.x;
    const float ss = a4.y;
    const int touch = __float_as_int(a4.z);
    if (a4.w == SS_ACC_F64 && P.acc64) {  // a big record: its float64 channels (T-row layout)
        const double *r = P.acc64 + (size_t)__float_as_int(a0.x) * SS_ACC64_WIDTH;
        for (int c = 0; c < 3; ++c) { G1[c] = r[c]; G2[c] = r[3 + c]; G4[c] = r[6 + c]; gcol[c] = r[13 + c]; }
        gs0 = r[9]; gs1 = r[10]; gs2 = r[11]; gnf = r[12]; gz = r[17];
    }

    float t1f[3], t2f[3], t4f[3];
    rows_of(P, i, t1f, t2f, t4f);
    if (a4.w == SS_ACC_MOMENTS) {
        // moments of the ray-plane gradient (train_step.cu item_grad) about
        // the projected centre (cx, cy): Sx = Sx' + cx S, Sy = Sy' + cy S in
        // float64; then with k = x t4 - t1, l = y t4 - t2:  sum l x gp =
        // t4 x Sy - t2 x S, sum gp x k = Sx x t4 - S x t1,
        // sum x (l x gp) + y (gp x k) = t1 x Sy - t2 x Sx
        const double cx = fd(t1f[2], t4f[2]), cy = fd(t2f[2], t4f[2]);  // bit-identical to the record kernel's
        const double S[3] = {G1[0], G1[1], G1[2]};
        const double Sx[3] = {G2[0] + cx * S[0], G2[1] + cx * S[1], G2[2] + cx * S[2]};
        const double Sy[3] = {G4[0] + cy * S[0], G4[1] + cy * S[1], G4[2] + cy * S[2]};
        const double T1[3] = {t1f[0], t1f[1], t1f[2]}, T2[3] = {t2f[0], t2f[1], t2f[2]};
        const double T4[3] = {t4f[0], t4f[1], t4f[2]};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int c1 = (c + 1) % 3, c2 = (c + 2) % 3;
            G1[c] = (T2[c1] * S[c2] - T2[c2] * S[c1]) - (T4[c1] * Sy[c2] - T4[c2] * Sy[c1]);
            G2[c] = (S[c1] * T1[c2] - S[c2] * T1[c1]) - (Sx[c1] * T4[c2] - Sx[c2] * T4[c1]);
            G4[c] = (T1[c1] * Sy[c2] - T1[c2] * Sy[c1]) - (T2[c1] * Sx[c2] - T2[c2] * Sx[c1]);
        }
    }
#ifdef SS_EXP_NO_MIP
    if (false) {
#else
    if (P.mip) {
#endif
        // _mip_chain_backward (backward.py:473-548)
        float jf[4];
        const bool ok = ss_center_jacobian(t1f, t2f, t4f, P.px.dxp, P.px.dyp, jf);
        const double j00 = jf[0], j01 = jf[1], j10 = jf[2], j11 = jf[3];
        const double sg = P.sigma;
        const double s00 = 1.0 + sg * (j00 * j00 + j01 * j01);
        const double s01 = sg * (j00 * j10 + j01 * j11);
        const double s11 = 1.0 + sg * (j10 * j10 + j11 * j11);
        const double det = s00 * s11 - s01 * s01;
        const double idet = 1.0 / det;
        const double b00 = s11 * idet, b01 = -s01 * idet, b11 = s00 * idet;
        const double nf = 1.0 / sqrt(det);
        const double g00 = gs0, g01 = 0.5 * gs1, g11 = gs2;
        const double bg00 = b00 * g00 + b01 * g01, bg01 = b00 * g01 + b01 * g11;
        const double bg10 = b01 * g00 + b11 * g01, bg11 = b01 * g01 + b11 * g11;
        const double ga00 = -(bg00 * b00 + bg01 * b01) - 0.5 * gnf * nf * b00;
        const double ga01 = -(bg00 * b01 + bg01 * b11) - 0.5 * gnf * nf * b01;
        const double ga11 = -(bg10 * b01 + bg11 * b11) - 0.5 * gnf * nf * b11;
        if (ok) {
            const double ts = 2.0 * sg;
            const double gj00 = ts * (ga00 * j00 + ga01 * j10), gj01 = ts * (ga00 * j01 + ga01 * j11);
            const double gj10 = ts * (ga01 * j00 + ga11 * j10), gj11 = ts * (ga01 * j01 + ga11 * j11);
            const double T1[3] = {t1f[0], t1f[1], t1f[2]}, T2[3] = {t2f[0], t2f[1], t2f[2]}, T4[3] = {t4f[0], t4f[1], t4f[2]};
            const double d4 = T4[2], id4 = 1.0 / d4, cx = T1[2] * id4, cy = T2[2] * id4;
            const double dx = P.px.inv_w, dy = P.px.inv_h;
            const double pr[4][4] = {{cx + dx, cy, gj00, gj10}, {cx - dx, cy, -gj00, -gj10},
                                     {cx, cy + dy, gj01, gj11}, {cx, cy - dy, -gj01, -gj11}};
            double gcx = 0.0, gcy = 0.0;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const double px = pr[p][0], py = pr[p][1];
                double k[3], l[3];
                for (int c = 0; c < 3; ++c) { k[c] = px * T4[c] - T1[c]; l[c] = py * T4[c] - T2[c]; }
                const double p0 = k[1] * l[2] - k[2] * l[1];
                const double p1 = k[2] * l[0] - k[0] * l[2];
                const double den = k[0] * l[1] - k[1] * l[0];
                if (!(fabs(den) >= SS_DENOM_EPS)) continue;
                const double iden = 1.0 / den;
                const double u = p0 * iden, v = p1 * iden;
                const double gu = pr[p][2], gv = pr[p][3];
                const double gp[3] = {gu * iden, gv * iden, -(gu * u + gv * v) * iden};
                const double gk[3] = {l[1] * gp[2] - l[2] * gp[1], l[2] * gp[0] - l[0] * gp[2], l[0] * gp[1] - l[1] * gp[0]};
                const double gl[3] = {gp[1] * k[2] - gp[2] * k[1], gp[2] * k[0] - gp[0] * k[2], gp[0] * k[1] - gp[1] * k[0]};
                for (int c = 0; c < 3; ++c) {
                    G1[c] -= gk[c];
                    G2[c] -= gl[c];
                    G4[c] += px * gk[c] + py * gl[c];
                }
                gcx += (gk[0] * T4[0] + gk[1] * T4[1]) + gk[2] * T4[2];
                gcy += (gl[0] * T4[0] + gl[1] * T4[1]) + gl[2] * T4[2];
            }
            G1[2] += gcx * id4;
            G4[2] -= gcx * cx * id4;
            G2[2] += gcy * id4;
            G4[2] -= gcy * cy * id4;
        }
    }
    // T rows -> camera -> world (backward.py:405-441) and the frame adjoint
    // in float64 with the float64 camera like the reference: a grazing
    // splat's row gradients are large and cancel in these linear maps
    // (float32 lost ~1% of its log-scale gradients).  TT: the tail's type
    // (SS_CHAIN_TAIL_F32: float32, an experiment switch)
    const TT *pm = TT_PROJ;
    TT gtu[3], gtv[3], gcc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        gtu[c] = G1[0] * pm[c] + G2[0] * pm[4 + c] + G4[0] * pm[12 + c];
        gtv[c] = G1[1] * pm[c] + G2[1] * pm[4 + c] + G4[1] * pm[12 + c];
        gcc[c] = G1[2] * pm[c] + G2[2] * pm[4 + c] + G4[2] * pm[12 + c];
    }
    gcc[2] -= gz;
    TT gw[3], guw[3], gvw[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        gw[k] = (gcc[0] * TT_VIEW[k] + gcc[1] * TT_VIEW[4 + k]) + gcc[2] * TT_VIEW[8 + k];
        guw[k] = (gtu[0] * TT_VIEW[k] + gtu[1] * TT_VIEW[4 + k]) + gtu[2] * TT_VIEW[8 + k];
        gvw[k] = (gtv[0] * TT_VIEW[k] + gtv[1] * TT_VIEW[4 + k]) + gtv[2] * TT_VIEW[8 + k];
    }
    const SsCloud &cl = P.cloud;
    const float4 qv = reinterpret_cast<const float4 *>(cl.quats)[i];
    const TT qn = (TT) sqrt((((double)qv.x * qv.x + (double)qv.y * qv.y) + (double)qv.z * qv.z) + (double)qv.w * qv.w);
    const TT iqn = TT(1) / qn;
    const TT w = qv.x * iqn, x = qv.y * iqn, y = qv.z * iqn, z = qv.w * iqn;
    const TT uh[3] = {1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)};
    const TT vh[3] = {2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)};
    const float2 lsv = reinterpret_cast<const float2 *>(cl.log_scales)[i];
    const TT su = (TT)exp((double)lsv.x), sv = (TT)exp((double)lsv.y);
    const TT gsu = (guw[0] * uh[0] + guw[1] * uh[1]) + guw[2] * uh[2];
    const TT gsv = (gvw[0] * vh[0] + gvw[1] * vh[1]) + gvw[2] * vh[2];
    TT gU[3], gV[3], gN[3] = {0, 0, 0};
    for (int k = 0; k < 3; ++k) { gU[k] = su * guw[k]; gV[k] = sv * gvw[k]; }
    TT gcent[3] = {gw[0], gw[1], gw[2]};
    float galb[3] = {0.f, 0.f, 0.f}, gmet = 0.f, grough = 0.f;

#ifdef SS_EXP_NO_SHADE
    if (false) {
#else
    if (P.color_source == SS_COLOR_IBL) {
#endif
        // the forward state in float64 like the preprocess kernel's colours
        // (identical texel cells / level / clip branches as the forward and
        // the reference's shading_ctx), the adjoint arithmetic in float32
        // (gradients: the 1e-3 parity bar)
        ShadeIn<float> in;
        ShadeState<float> st;
        ShadeGrads<float> sg;
        const float gcf[3] = {(float)gcol[0], (float)gcol[1], (float)gcol[2]};
        if (P.cells && P.env.diffuse4 && P.env.specular4) {
            // the preprocess kernel's float64 branch decisions, float32 state
            // with the texel derivatives read together with the values
            ss_shade_inputs(cl, i, P.cam_pos, in);
            ss_shade_forward_cells(in, P.env, __ldg(P.cells + i), st,
                                   kPre ? reinterpret_cast<const float *>(P.pre_diff + i) : nullptr);
            ss_shade_backward<float, true>(in, st, P.env, gcf, sg);
        } else {
            ShadeIn<double> in64;
            ss_shade_inputs(cl, i, P.cam_pos, in64);
            ShadeState<double> st64;
            double col[3];
            ss_shade_forward(in64, P.env, st64, col);
            ss_shade_narrow(in64, st64, in, st);
            ss_shade_backward(in, st, P.env, gcf, sg);
        }
        for (int c = 0; c < 3; ++c) { gcent[c] += sg.center[c]; gN[c] = sg.normal[c]; galb[c] = sg.albedo_raw[c]; }
        gmet = sg.metallic_raw;
        grough = sg.roughness_raw;
        // derived-map scatter (bilinear_scatter, shading.py:248-260, 583-597)
        const int we = P.env.we;
        const double wts[2] = {1.0 - (double)st.frac, (double)st.frac};
        const int lvs[2] = {st.lvl0, st.lvl1};
        const SsBil<float> &bs = st.bs;
        const int sidx[4] = {bs.j0 * we + bs.i0, bs.j0 * we + bs.i1, bs.j1 * we + bs.i0, bs.j1 * we + bs.i1};
        const double scw[4] = {(1.0 - bs.tu) * (1.0 - bs.tv), (double)bs.tu * (1.0 - bs.tv), (1.0 - bs.tu) * (double)bs.tv,
                               (double)bs.tu * bs.tv};
        const int T = P.env.he * we;
        const SsBil<float> &bd = st.bd;
        const int didx[4] = {bd.j0 * we + bd.i0, bd.j0 * we + bd.i1, bd.j1 * we + bd.i0, bd.j1 * we + bd.i1};
        const double dcw[4] = {(1.0 - bd.tu) * (1.0 - bd.tv), (double)bd.tu * (1.0 - bd.tv), (1.0 - bd.tu) * (double)bd.tv,
                               (double)bd.tu * bd.tv};
#ifdef SS_EXP_NO_SCATTER
        if (P.g.d_specular4 && sg.g_ls[0] == 12345.f) {  // (experiment: never true)
#else
        if (P.g.d_specular4) {  // per-view float32 maps, folded into the float64 sums per view
#endif
            for (int h = 0; h < 2; ++h)
                for (int k = 0; k < 4; ++k) {
                    const float f = (float)(wts[h] * scw[k]);
                    scatter_rgb4<false>(P.g.d_specular4, lvs[h] * T + sidx[k], sg.g_ls[0] * f, sg.g_ls[1] * f,
                                        sg.g_ls[2] * f);
                }
            if (kPre) {  // per surfel; the step's one diffuse scatter applies the taps
                red_add4(reinterpret_cast<float *>(P.g_ld + i), sg.g_ld[0], sg.g_ld[1], sg.g_ld[2], 0.f);
            } else {
                for (int k = 0; k < 4; ++k) {
                    const float f = (float)dcw[k];
                    scatter_rgb4<true>(P.g.d_diffuse4, didx[k], sg.g_ld[0] * f, sg.g_ld[1] * f, sg.g_ld[2] * f);
                }
            }
        } else if (!P.g.d_specular4) {
            for (int h = 0; h < 2; ++h)  // level lvs[h] texel sidx[k] = element 3 * (lvs[h] * T + sidx[k])
                for (int k = 0; k < 4; ++k) {
                    const double f = wts[h] * scw[k];
                    scatter_rgb(P.g.d_specular, lvs[h] * T + sidx[k], sg.g_ls[0] * f, sg.g_ls[1] * f, sg.g_ls[2] * f);
                }
            for (int k = 0; k < 4; ++k)
                scatter_rgb(P.g.d_diffuse, didx[k], sg.g_ld[0] * dcw[k], sg.g_ld[1] * dcw[k], sg.g_ld[2] * dcw[k]);
        }
    } else if (P.color_source == SS_COLOR_ALBEDO) {
        for (int c = 0; c < 3; ++c) {
            const float al = ss_sigmoid_fast(cl.albedo_raw[3 * i + c]);
            galb[c] = (float)gcol[c] * al * (1.f - al);
        }
    }
    // quat_frame_backward (surfels.py:54-77)
#define D3(g, a0, a1, a2) ((g)[0] * (a0) + (g)[1] * (a1) + (g)[2] * (a2))
    const TT gqw = D3(gU, TT(0), 2 * z, -2 * y) + D3(gV, -2 * z, TT(0), 2 * x) + D3(gN, 2 * y, -2 * x, TT(0));
    const TT gqx = D3(gU, TT(0), 2 * y, 2 * z) + D3(gV, 2 * y, -4 * x, 2 * w) + D3(gN, 2 * z, -2 * w, -4 * x);
    const TT gqy = D3(gU, -4 * y, 2 * x, -2 * w) + D3(gV, 2 * x, TT(0), 2 * z) + D3(gN, 2 * w, 2 * z, -4 * y);
    const TT gqz = D3(gU, -4 * z, 2 * w, 2 * x) + D3(gV, -2 * w, -4 * z, 2 * y) + D3(gN, 2 * x, 2 * y, TT(0));
#undef D3
    const TT radial = ((gqw * w + gqx * x) + gqy * y) + gqz * z;

    SsGrads &g = P.g;
    for (int c = 0; c < 3; ++c) {
        red_add(g.centers + 3 * i + c, (float)gcent[c]);
        red_add(g.albedo_raw + 3 * i + c, (float)galb[c]);
    }
    red_add4(g.quats + 4 * (size_t)i, (float)((gqw - radial * w) * iqn), (float)((gqx - radial * x) * iqn),
             (float)((gqy - radial * y) * iqn), (float)((gqz - radial * z) * iqn));
    red_add2(g.log_scales + 2 * (size_t)i, (float)(gsu * su), (float)(gsv * sv));
    red_add(g.metallic_raw + i, (float)gmet);
    red_add(g.roughness_raw + i, (float)grough);
    if (g.colors)
        for (int c = 0; c < 3; ++c) red_add(g.colors + 3 * i + c, (float)gcol[c]);
    red_add(g.ss_grad + i, ss);
    if (g.touched) atomicAdd(g.touched + i, touch);
    if (g.view_count && touch > 0) red_add(g.view_count + i, 1.f);
}

}  // namespace

extern "C" int ss_env_grad_merge(int64_t texels, float *src4, double *dst, void *stream)
{
    if (texels < 0 || (texels > 0 && (!src4 || !dst))) return SS_ERR_INVALID;
    if (texels == 0) return SS_OK;
    const int blocks = (int)((texels + 255) / 256 < ss_sm_count() * 4 ? (texels + 255) / 256 : ss_sm_count() * 4);
    env_merge_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(texels, reinterpret_cast<float4 *>(src4), dst);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

static int chain_backward(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt, int color_source,
                          const SsEnv *env, const int8_t *cull, const float *rec_acc, const double *rec_acc64,
                          const uint32_t *shade_cells, const SsGrads *grads, const void *prepass, float *g_ld,
                          void *stream)
{
    if (!cloud || !cam || !opt || !grads) return SS_ERR_INVALID;
    if (cloud->n == 0) return SS_OK;
    if (!cull || !rec_acc) return SS_ERR_INVALID;
    if (color_source == SS_COLOR_IBL && (!env || !grads->d_diffuse || !grads->d_specular)) return SS_ERR_INVALID;
    if (cloud->n == 0) return SS_OK;
    ChainParams P;
    P.cloud = *cloud;
    for (int k = 0; k < 16; ++k) {
        P.view[k] = cam->view[k]; P.proj[k] = cam->proj[k];
        P.viewf[k] = (float)cam->view[k]; P.projf[k] = (float)cam->proj[k];
    }
    for (int k = 0; k < 3; ++k)
        P.cam_pos[k] = -(cam->view[k] * cam->view[3] + cam->view[4 + k] * cam->view[7] + cam->view[8 + k] * cam->view[11]);
    P.W = cam->width; P.H = cam->height; P.mip = opt->mip_enabled; P.color_source = color_source;
    P.px = ss_pixel_steps(P.W, P.H);
    P.sigma = (double)opt->mip_sigma;
    P.r_cut = opt->r_cut; P.sigma_f = opt->mip_sigma;
    P.env = env ? *env : SsEnv{};
    P.cull = cull; P.acc = rec_acc; P.acc64 = rec_acc64; P.g = *grads;
    P.cells = reinterpret_cast<const uint4 *>(shade_cells);
    const bool pre = prepass && g_ld && shade_cells && color_source == SS_COLOR_IBL && env && env->diffuse4;
    P.pre_diff = pre ? prepass_diff(prepass, cloud->n) : nullptr;
    P.g_ld = pre ? reinterpret_cast<float4 *>(g_ld) : nullptr;
    if (pre) chain_kernel<true><<<(cloud->n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(P);
    else chain_kernel<false><<<(cloud->n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(P);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_chain_backward(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                                 int color_source, const SsEnv *env, const int8_t *cull,
                                 const float *rec_acc, const double *rec_acc64, const uint32_t *shade_cells,
                                 const SsGrads *grads, void *stream)
{
    return chain_backward(cloud, cam, opt, color_source, env, cull, rec_acc, rec_acc64, shade_cells, grads, nullptr,
                          nullptr, stream);
}

extern "C" int ss_chain_backward_prepared(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                                          int color_source, const SsEnv *env, const int8_t *cull,
                                          const float *rec_acc, const double *rec_acc64,
                                          const uint32_t *shade_cells, const SsGrads *grads, const void *prepass,
                                          float *g_ld, void *stream)
{
    if (!prepass || !g_ld) return SS_ERR_INVALID;
    return chain_backward(cloud, cam, opt, color_source, env, cull, rec_acc, rec_acc64, shade_cells, grads, prepass,
                          g_ld, stream);
}

namespace {
// d_diffuse += the step's diffuse-lookup upstream of every surfel through its
// four bilinear taps (bilinear_scatter, shading.py:248-260, 583-597): the
// cell and fractions are the normal's, so the per-view scatter folds into one
// per step; g_ld is zeroed for the next step.
__global__ void diffuse_scatter_kernel(int n, int we, const PreShade *__restrict__ sh, const PreDiff *__restrict__ pd,
                                       float4 *__restrict__ g_ld, double *__restrict__ d_diffuse) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 g = g_ld[i];
    if (g.x == 0.f && g.y == 0.f && g.z == 0.f) return;
    g_ld[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const unsigned cell = sh[i].cell;
    const int i0 = (int)(cell & 0xffffu), j0 = (int)(cell >> 16);
    const int i1 = i0 + 1 == we ? 0 : i0 + 1, j1 = j0 + 1;
    const double tu = pd[i].tu, tv = pd[i].tv;
    const int idx[4] = {j0 * we + i0, j0 * we + i1, j1 * we + i0, j1 * we + i1};
    const double w[4] = {(1.0 - tu) * (1.0 - tv), tu * (1.0 - tv), (1.0 - tu) * tv, tu * tv};
#pragma unroll
    for (int k = 0; k < 4; ++k) scatter_rgb(d_diffuse, idx[k], g.x * w[k], g.y * w[k], g.z * w[k]);
}
}  // namespace

extern "C" int ss_diffuse_scatter(int n, const SsEnv *env, const void *prepass, float *g_ld, double *d_diffuse,
                                  void *stream)
{
    if (n < 0 || !env || !prepass || !g_ld || !d_diffuse) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    diffuse_scatter_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        n, env->we, prepass_shade(prepass, n), prepass_diff(prepass, n), reinterpret_cast<float4 *>(g_ld), d_diffuse);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
