// coverage.cuh -- fast coverage decision with a per-record certified margin.
//
// The reference decides coverage of pixel (x, y) by a record with float32
// k = x t4 - t1, l = y t4 - t2, u = (k1 l2 - k2 l1) / den, v = (k2 l0 - k0 l2)
// / den, den = k0 l1 - k1 l0 and the mixed-precision rho^2 < 9
// (rasterizer.py:197-210).  In exact arithmetic NU, NV and DEN are LINEAR in
// (x, y) (the x*y terms of the cross products cancel), and NU = NV = 0 at the
// splat centre (xc, yc) = (t1z / t4z, t2z / t4z).  So per record
//     nu = au dx + bu dy,  nv = av dx + bv dy,  den = dc + ad dx + bd dy,
// with dx = x - xc, dy = y - yc: 6 FMAs, one reciprocal and the quadratic
// form per pixel instead of the reference's ~25 separately rounded ops.
//
// The two evaluations differ by rounding only.  The preprocess kernel bounds
// |rho2_fast - rho2_reference| over the record's whole rect (both rounding
// error budgets, float64, corners of the rect -- everything is bilinear or
// quasi-linear there) and stores the bound M in the record (slot e.w).  A
// pixel whose fast rho^2 lies within M of the cut-off (or whose den is near
// the ray-miss threshold) takes the reference's exact sequence (ss_cover);
// every other decision is provably the reference's.  Records whose bound is
// not small, or whose den changes sign over the rect, carry M = +inf and
// always take the exact path.
#pragma once
#include "ss_common.cuh"

struct FastCov {
    float au, bu, av, bv, ad, bd, dc, xc, yc, m;
};

__device__ __forceinline__ float fc_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * (2.f - x * r);
}

// Coefficients from the record's T rows (a = t1.xyz t2.x, b = t2.yz t4.xy,
// c.x = t4.z) and its margin m.
__device__ __forceinline__ void fast_cov_setup(const float4 &a, const float4 &b, const float4 &c, float m,
                                               FastCov &f) {
    const float t1x = a.x, t1y = a.y, t1z = a.z, t2x = a.w, t2y = b.x, t2z = b.y;
    const float t4x = b.z, t4y = b.w, t4z = c.x;
    f.au = t4z * t2y - t4y * t2z;
    f.bu = t1z * t4y - t1y * t4z;
    f.av = t4x * t2z - t4z * t2x;
    f.bv = t1x * t4z - t1z * t4x;
    f.ad = t4y * t2x - t4x * t2y;
    f.bd = t1y * t4x - t1x * t4y;
    const float it4 = fc_rcp(t4z);
    f.xc = t1z * it4;
    f.yc = t2z * it4;
    const float k0 = f.xc * t4x - t1x, k1 = f.xc * t4y - t1y;
    const float l0 = f.yc * t4x - t2x, l1 = f.yc * t4y - t2y;
    f.dc = k0 * l1 - k1 * l0;
    f.m = m;
}

// 1: covered, 0: not covered (both certified equal to the reference's
// decision), -1: undecided (take the exact path).  u, v, rho2 are the fast
// values (weights: within the margin of the reference's).
__device__ __forceinline__ int fast_cover(const FastCov &f, float s0, float s1, float s2, float x, float y, float &u,
                                          float &v, float &rho2) {
    const float dx = x - f.xc, dy = y - f.yc;
    const float nu = f.au * dx + f.bu * dy;
    const float nv = f.av * dx + f.bv * dy;
    const float den = f.dc + f.ad * dx + f.bd * dy;
    const float inv = fc_rcp(den);
    u = nu * inv;
    v = nv * inv;
    rho2 = s0 * u * u + 2.f * s1 * u * v + s2 * v * v;
    if (!(fabsf(den) > 4e-9f)) return -1;  // near the ray-miss threshold (also NaN)
    if (rho2 < 9.f - f.m) return 1;
    if (rho2 >= 9.f + f.m) return 0;
    return -1;
}

// Certified bound on |rho2_fast - rho2_reference| over the pixel centres of
// rect [x0, x1) x [y0, y1) (float64, first order in the unit roundoff e,
// then doubled).  Reference: k_i = fl(fl(x t4_i) - t1_i) is off by at most
// e(|x t4_i| + |k_i|) <= e a_i with a_i = 2 max|x| |t4_i| + |t1_i| (b_i for
// l), so a cross product nu = fl(fl(k1 l2) - fl(k2 l1)) is off by at most
// 3e(a1 b2 + a2 b1) + e|nu|.  Fast path: the rounded coefficients (2e of
// their term magnitudes), the centre (3e relative), dx, dy and the two FMAs.
// den's bound is the same construction; u = nu/den then moves by
// (E_nu + |u| E_den) / min|den| plus the quotient roundings, and rho^2 by the
// first-order propagation plus both rho^2 evaluation roundings.  +inf when
// den may change sign over the rect or the bound is not small.
__device__ __forceinline__ float coverage_margin(const float t1[3], const float t2[3], const float t4[3], float s0,
                                                 float s1, float s2, int x0, int y0, int x1, int y1, double two_w,
                                                 double two_h) {
    const double e = 5.9604644775390625e-08;  // 2^-24, float32 unit roundoff
    const float INF = __int_as_float(0x7f800000);
    const double T1[3] = {t1[0], t1[1], t1[2]}, T2[3] = {t2[0], t2[1], t2[2]}, T4[3] = {t4[0], t4[1], t4[2]};
    const double xs[2] = {(double)ss_ndc_xs(x0, two_w), (double)ss_ndc_xs(x1 - 1, two_w)};
    const double ys[2] = {(double)ss_ndc_ys(y0, two_h), (double)ss_ndc_ys(y1 - 1, two_h)};
    // den is linear in (x, y): its extremes over the rect are at the corners
    double dmin = 1e300, dmax = -1e300;
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            const double k0 = xs[i] * T4[0] - T1[0], k1 = xs[i] * T4[1] - T1[1];
            const double l0 = ys[j] * T4[0] - T2[0], l1 = ys[j] * T4[1] - T2[1];
            const double den = k0 * l1 - k1 * l0;
            dmin = fmin(dmin, den);
            dmax = fmax(dmax, den);
        }
    if (!(dmin > 0.0 || dmax < 0.0)) return INF;  // den changes sign / vanishes over the rect
    const double dm = fmin(fabs(dmin), fabs(dmax)), dabs = fmax(fabs(dmin), fabs(dmax));
    // Only points near or inside the support matter: a wrong decision needs
    // the reference's rho^2 < 9 or the fast one < 9 + m, i.e. (to first
    // order) a point of the ellipse rho^2 <= 9.5, where |u| <= sqrt(9.5 S^-1_00)
    // and |v| <= sqrt(9.5 S^-1_11); far rect corners are decided "out" by
    // any evaluation, so they do not set the error scale.
    const double S0 = s0, S1 = s1, S2 = s2, det = S0 * S2 - S1 * S1;
    if (!(det > 0.0 && S0 > 0.0)) return INF;
    const double umax = sqrt(9.5 * S2 / det), vmax = sqrt(9.5 * S0 / det);
    const double numax = umax * dabs, nvmax = vmax * dabs;
    const double it4 = 1.0 / T4[2], xc = T1[2] * it4, yc = T2[2] * it4;
    const double xm = fmax(fabs(xs[0]), fabs(xs[1])), ym = fmax(fabs(ys[0]), fabs(ys[1]));
    const double dxm = fmax(fabs(xs[0] - xc), fabs(xs[1] - xc)), dym = fmax(fabs(ys[0] - yc), fabs(ys[1] - yc));
    double a[3], b[3];
    for (int i = 0; i < 3; ++i) {
        a[i] = 2.0 * xm * fabs(T4[i]) + fabs(T1[i]);
        b[i] = 2.0 * ym * fabs(T4[i]) + fabs(T2[i]);
    }
    // reference cross products
    const double r_den = 3.0 * e * (a[0] * b[1] + a[1] * b[0]) + e * dabs;
    const double r_nu = 3.0 * e * (a[1] * b[2] + a[2] * b[1]) + e * numax;
    const double r_nv = 3.0 * e * (a[2] * b[0] + a[0] * b[2]) + e * nvmax;
    // fast linear forms: coefficient term magnitudes c*, centre/dx rounding
    const double cau = fabs(T4[2] * T2[1]) + fabs(T4[1] * T2[2]), cbu = fabs(T1[2] * T4[1]) + fabs(T1[1] * T4[2]);
    const double cav = fabs(T4[0] * T2[2]) + fabs(T4[2] * T2[0]), cbv = fabs(T1[0] * T4[2]) + fabs(T1[2] * T4[0]);
    const double cad = fabs(T4[1] * T2[0]) + fabs(T4[0] * T2[1]), cbd = fabs(T1[1] * T4[0]) + fabs(T1[0] * T4[1]);
    const double gx = 4.0 * dxm + 3.0 * fabs(xc), gy = 4.0 * dym + 3.0 * fabs(yc);
    const double f_nu = e * (cau * gx + cbu * gy + numax);
    const double f_nv = e * (cav * gx + cbv * gy + nvmax);
    // dc is the reference-style cross product at the centre, then two FMAs
    const double f_den = r_den + e * (cad * gx + cbd * gy + 2.0 * dabs);
    const double e_den = r_den + f_den, e_nu = r_nu + f_nu, e_nv = r_nv + f_nv;
    if (!(e_den < 0.05 * dm)) return INF;
    const double iq = 1.0 / (dm - e_den);
    const double du = (e_nu + umax * e_den) * iq + 3.0 * e * umax;
    const double dv = (e_nv + vmax * e_den) * iq + 3.0 * e * vmax;
    const double as1 = fabs(S1);
    const double q = S0 * umax * umax + 2.0 * as1 * umax * vmax + S2 * vmax * vmax;
    const double dr = 2.0 * (S0 * umax + as1 * vmax) * du + 2.0 * (as1 * umax + S2 * vmax) * dv +
                      S0 * du * du + 2.0 * as1 * du * dv + S2 * dv * dv + 6.0 * e * q;
    const double m = 2.0 * dr;  // x2 for the dropped second-order terms
    if (!(m < 1.0)) return INF;
    return (float)m * 1.0000002f;
}
