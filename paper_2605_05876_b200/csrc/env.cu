// env.cu -- environment prefilter operators applied on the fly, their
// adjoint, and the preintegrated BRDF LUT.
//
// Reference: EnvironmentLight.refresh / env_gradient (shading.py:369-394),
// build_diffuse_operator (:275-282, a DENSE T x T float64 matrix),
// build_specular_operator (:285-331), brdf_lut (:118-156).  The reference
// materialises T x T operators (51.5 GB at 128x256, 825 GB at 256x512); here
// the diffuse operator is regenerated on the fly as an O(T^2) FP32 N-body
// pass (column texels staged through shared memory, gather form in both
// directions so no atomics, float64 chunk accumulation), and the specular
// operator is regenerated per output texel from the same Hammersley/GGX
// samples (refresh: gather; adjoint: scatter with float atomics).
#include "ss_common.cuh"
#include "shading.cuh"

namespace {

__device__ __forceinline__ double radical_inverse(uint32_t i) {
    return (double)__brev(i) * 2.3283064365386963e-10;
}

__device__ __forceinline__ void ggx_h(double xi0, double xi1, double alpha, double h[3]) {
    const double phi = 2.0 * SS_PI * xi0;
    const double cos_t = sqrt((1.0 - xi1) / (1.0 + (alpha * alpha - 1.0) * xi1));
    const double sin_t = sqrt(ss_npmax(1.0 - cos_t * cos_t, 0.0));
    h[0] = sin_t * cos(phi); h[1] = sin_t * sin(phi); h[2] = cos_t;
}

__device__ __forceinline__ double smith_g1(double c, double k) { return c / (c * (1.0 - k) + k); }

__global__ void lut_kernel(int res, int samples, float *lut) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= res * res) return;
    const int j = id / res, i = id % res;
    const double r = ((double)j + 0.5) / res, alpha = r * r, k = alpha / 2.0;
    const double cv = ((double)i + 0.5) / res;
    const double vx = sqrt(1.0 - cv * cv), vz = cv;
    double s1 = 0.0, s2 = 0.0;
    for (int s = 0; s < samples; ++s) {
        double h[3];
        ggx_h(((double)s + 0.5) / samples, radical_inverse((uint32_t)s), alpha, h);
        const double vh = vx * h[0] + vz * h[2];
        const double l2 = 2.0 * vh * h[2] - vz;
        const bool good = l2 > 0.0 && vh > 0.0;
        const double g = smith_g1(cv, k) * smith_g1(ss_npmax(l2, 1e-8), k);
        const double gv = good ? g * vh / ss_npmax(h[2] * cv, 1e-8) : 0.0;
        const double fc = pow(1.0 - ss_clip(vh, 0.0, 1.0), 5.0);
        s1 += gv * (1.0 - fc);
        s2 += gv * fc;
    }
    lut[2 * id] = (float)(s1 / samples);
    lut[2 * id + 1] = (float)(s2 / samples);
}

// Texel direction and solid angle (latlong_texel_dirs, shading.py:162-169).
__device__ __forceinline__ void texel(int b, int he, int we, float d[3], float &om) {
    const int r = b / we, c = b % we;
    const double th = ((double)r + 0.5) * (SS_PI / he);
    const double ph = ((double)c + 0.5) * (2.0 * SS_PI / we) - SS_PI;
    const double st = sin(th);
    d[0] = (float)(st * cos(ph)); d[1] = (float)(st * sin(ph)); d[2] = (float)cos(th);
    om = (float)(st * (SS_PI / he) * (2.0 * SS_PI / we));
}

// The clamped-cosine quadrature as an on-the-fly T x T product (N-body form).
// Column texels are staged CHUNK at a time in shared memory as (dir, value)
// with the per-column factor folded into the value, so the inner loop is
// 3 FFMA (dot) + max + 3 FFMA (accumulate):
// mode 0: rowsum_a = sum_b max(d_a.d_b,0) om_b
// mode 1: out_a    = sum_b max(d_a.d_b,0) om_b x_b / rowsum_a          (refresh)
// mode 2: out_b   += om_b sum_a max(d_a.d_b,0) x_a / rowsum_a          (adjoint; roles swapped)
constexpr int kChunk = 512;   // column texels staged per pass
constexpr int kOut = 2;       // output texels per thread (register blocking over the staged columns)
constexpr int kDiffThreads = 128;
constexpr int kSplit = 8;     // column range split across CTAs (fills the GPU: T outputs alone do not)

template <int MODE, typename TIn>
__global__ void __launch_bounds__(kDiffThreads) diffuse_kernel(int he, int we, const TIn *__restrict__ x,
                                                               const double *__restrict__ rowsum,
                                                               double *__restrict__ part) {
    __shared__ float4 sd[kChunk];   // column direction (xyz, w unused)
    __shared__ float4 sv[kChunk];   // column value rgb with its factor folded in (w unused)
    const int T = he * we;
    const int a0 = (blockIdx.x * blockDim.x + threadIdx.x) * kOut;
    const int per = (T + kSplit - 1) / kSplit;
    const int b0 = blockIdx.y * per, b1 = min(T, b0 + per);
    float da[kOut][3], oma[kOut];
#pragma unroll
    for (int q = 0; q < kOut; ++q) {
        da[q][0] = da[q][1] = da[q][2] = 0.f;
        oma[q] = 0.f;
        if (a0 + q < T) texel(a0 + q, he, we, da[q], oma[q]);
    }
    float s[kOut][3];
    double t[kOut][3];
#pragma unroll
    for (int q = 0; q < kOut; ++q) { s[q][0] = s[q][1] = s[q][2] = 0.f; t[q][0] = t[q][1] = t[q][2] = 0.0; }
    for (int base = b0; base < b1; base += kChunk) {
        const int cn = min(kChunk, b1 - base);
        __syncthreads();
        for (int k = threadIdx.x; k < cn; k += blockDim.x) {
            const int b = base + k;
            float db[3], omb;
            texel(b, he, we, db, omb);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (MODE == 0) {
                v.x = omb;
            } else if (MODE == 1) {
                v = make_float4(omb * (float)x[3 * b], omb * (float)x[3 * b + 1], omb * (float)x[3 * b + 2], 0.f);
            } else {
                const double inv = 1.0 / (double)rowsum[b];
                v = make_float4((float)(x[3 * b] * inv), (float)(x[3 * b + 1] * inv), (float)(x[3 * b + 2] * inv), 0.f);
            }
            sd[k] = make_float4(db[0], db[1], db[2], 0.f);
            sv[k] = v;
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < cn; ++k) {
            const float4 d = sd[k];
            const float4 v = sv[k];
#pragma unroll
            for (int q = 0; q < kOut; ++q) {
                const float c = fmaxf(da[q][0] * d.x + da[q][1] * d.y + da[q][2] * d.z, 0.f);
                s[q][0] = fmaf(c, v.x, s[q][0]);
                if (MODE != 0) { s[q][1] = fmaf(c, v.y, s[q][1]); s[q][2] = fmaf(c, v.z, s[q][2]); }
            }
        }
        // flush the chunk partials into float64 (keeps the 32k-term sums accurate)
#pragma unroll
        for (int q = 0; q < kOut; ++q) {
            t[q][0] += s[q][0]; t[q][1] += s[q][1]; t[q][2] += s[q][2];
            s[q][0] = s[q][1] = s[q][2] = 0.f;
        }
    }
#pragma unroll
    for (int q = 0; q < kOut; ++q) {
        const int a = a0 + q;
        if (a >= T) break;
        atomicAdd(part + 3 * a, t[q][0]);
        if (MODE != 0) { atomicAdd(part + 3 * a + 1, t[q][1]); atomicAdd(part + 3 * a + 2, t[q][2]); }
    }
}

// mode 0: rowsum_a = part; mode 1: out_a = part / rowsum_a; mode 2: out_a += om_a part
template <int MODE, typename TOut>
__global__ void diffuse_finish_kernel(int he, int we, const double *__restrict__ part, const double *__restrict__ rowsum,
                                      TOut *__restrict__ out) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= he * we) return;
    if (MODE == 0) {
        out[a] = (TOut)part[3 * a];
    } else if (MODE == 1) {
        const double inv = 1.0 / (double)rowsum[a];
        for (int c = 0; c < 3; ++c) out[3 * a + c] = (TOut)(part[3 * a + c] * inv);
    } else {
        float d[3], om;
        texel(a, he, we, d, om);
        for (int c = 0; c < 3; ++c) out[3 * a + c] += (TOut)(part[3 * a + c] * (double)om);
    }
}

// ---- spectral form of the same quadrature ----------------------------------
// Between lat-long texels, d_a . d_b = s_i s_j cos(phi_a - phi_b) + c_i c_j
// (rows i, j; s = sin theta, c = cos theta) and phi_a - phi_b = 2 pi (c_a -
// c_b) / we: the clamped-cosine kernel depends on the columns only through
// (c_a - c_b) mod we.  Row pair by row pair the T x T product is therefore a
// circular convolution along phi, K_ij(m) = max(s_i s_j cos(2 pi m / we) +
// c_i c_j, 0), and along the DFT of each row
//     y_i^(k) = sum_j K_ij^(k) v_j^(k).
// K_ij is even in m, so K_ij^ is real; it depends on the grid only and is
// built once per shape (float64, he^2 (we/2 + 1) values).  One application
// costs O(he^2 we + he we^2) float64 operations instead of the O(he^2 we^2)
// of the N-body form above (which remains for odd widths).


__device__ __forceinline__ void twiddles(int we, double *tc, double *ts) {
    for (int m = threadIdx.x; m < we; m += blockDim.x) {
        double sv, cv;
        sincospi(2.0 * m / we, &sv, &cv);
        tc[m] = cv;
        ts[m] = sv;
    }
}

// K^_ij(k) = sum_m K_ij(m) cos(2 pi k m / we), stored [k][i][j]; one CTA per
// (i, j), threads over k
__global__ void __launch_bounds__(128) dspec_kernel(int he, int we, double *__restrict__ khat) {
    extern __shared__ double dsm[];
    double *tc = dsm, *ts = dsm + we, *kv = dsm + 2 * we;
    const int i = blockIdx.x / he, j = blockIdx.x % he;
    twiddles(we, tc, ts);
    double si, ci, sj, cj;
    sincospi((i + 0.5) / he, &si, &ci);
    sincospi((j + 0.5) / he, &sj, &cj);
    __syncthreads();
    for (int m = threadIdx.x; m < we; m += blockDim.x) kv[m] = fmax(si * sj * tc[m] + ci * cj, 0.0);
    __syncthreads();
    const int nk = we / 2 + 1;
    for (int k = threadIdx.x; k < nk; k += blockDim.x) {
        double acc = 0.0;
        int idx = 0;
        for (int m = 0; m < we; ++m) {
            acc += kv[m] * tc[idx];
            idx += k;
            if (idx >= we) idx -= we;
        }
        khat[((size_t)k * he + i) * he + j] = acc;
    }
}

// Row DFTs of the weighted input v (mode 0: v = om; 1: om x; 2: x / rowsum),
// packed per (channel, row) as we doubles: re0, re_{we/2}, re1, im1, ...
template <int MODE, typename TIn>
__global__ void __launch_bounds__(256) drow_dft_kernel(int he, int we, const TIn *__restrict__ x,
                                                       const double *__restrict__ rowsum, double *__restrict__ vhat) {
    extern __shared__ double dsm[];
    constexpr int NC = MODE == 0 ? 1 : 3;
    double *tc = dsm, *ts = dsm + we, *sv = dsm + 2 * we;
    const int r = blockIdx.x;
    twiddles(we, tc, ts);
    const double om = sinpi((r + 0.5) / he) * (SS_PI / he) * (2.0 * SS_PI / we);
    for (int t = threadIdx.x; t < NC * we; t += blockDim.x) {
        const int c = t / we, m = t % we, b = r * we + m;
        double v;
        if (MODE == 0) v = om;
        else if (MODE == 1) v = om * (double)x[3 * b + c];
        else v = (double)x[3 * b + c] / (double)rowsum[b];
        sv[c * we + m] = v;
    }
    __syncthreads();
    const int nk = we / 2 + 1;
    for (int t = threadIdx.x; t < NC * nk; t += blockDim.x) {
        const int c = t / nk, k = t % nk;
        const double *v = sv + c * we;
        double re = 0.0, im = 0.0;
        int idx = 0;
        for (int m = 0; m < we; ++m) {
            re += v[m] * tc[idx];
            im -= v[m] * ts[idx];
            idx += k;
            if (idx >= we) idx -= we;
        }
        double *o = vhat + ((size_t)c * he + r) * we;
        if (k == 0) o[0] = re;
        else if (k == we / 2) o[1] = re;
        else { o[2 * k] = re; o[2 * k + 1] = im; }
    }
}

// One CTA per frequency k: y^_i(k) = sum_j K^_ij(k) v^_j(k) for every row i
// and channel, written over v^(k) in place (no other CTA touches column k).
template <int NC>
__global__ void __launch_bounds__(128) dmul_kernel(int he, int we, const double *__restrict__ khat,
                                                   double *__restrict__ vhat) {
    extern __shared__ double dsm[];
    double *vr = dsm, *vi = dsm + NC * he;  // [c][j]
    const int k = blockIdx.x, nk = we / 2 + 1;
    const bool real = k == 0 || k == nk - 1;
    const int ore = k == 0 ? 0 : (k == nk - 1 ? 1 : 2 * k);
    for (int t = threadIdx.x; t < NC * he; t += blockDim.x) {
        const double *v = vhat + (size_t)t * we;  // t = c * he + j
        vr[t] = v[ore];
        vi[t] = real ? 0.0 : v[ore + 1];
    }
    __syncthreads();
    const double *K = khat + (size_t)k * he * he;
    for (int i = threadIdx.x; i < he; i += blockDim.x) {
        double re[NC], im[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) re[c] = im[c] = 0.0;
        const double *row = K + (size_t)i * he;
        for (int j = 0; j < he; ++j) {
            const double kk = __ldg(row + j);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                re[c] = fma(kk, vr[c * he + j], re[c]);
                im[c] = fma(kk, vi[c * he + j], im[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            double *o = vhat + ((size_t)c * he + i) * we;
            o[ore] = re[c];
            if (!real) o[ore + 1] = im[c];
        }
    }
}

// One CTA per output row i: inverse DFT of y^_i, then the mode's finish
// (0: rowsum; 1: out = y / rowsum; 2: out += om y).
template <int MODE, typename TOut>
__global__ void __launch_bounds__(256) dinv_kernel(int he, int we, const double *__restrict__ yhat,
                                                   const double *__restrict__ rowsum, TOut *__restrict__ out) {
    extern __shared__ double dsm[];
    constexpr int NC = MODE == 0 ? 1 : 3;
    double *tc = dsm, *ts = dsm + we, *sy = dsm + 2 * we;  // sy[c][we] packed spectrum
    const int i = blockIdx.x, nk = we / 2 + 1;
    twiddles(we, tc, ts);
    for (int t = threadIdx.x; t < NC * we; t += blockDim.x)
        sy[t] = yhat[((size_t)(t / we) * he + i) * we + t % we];
    __syncthreads();
    const double om = sinpi((i + 0.5) / he) * (SS_PI / he) * (2.0 * SS_PI / we);
    for (int t = threadIdx.x; t < NC * we; t += blockDim.x) {
        const int c = t / we, col = t % we;
        const double *a = sy + c * we;
        double y = a[0] + ((col & 1) ? -a[1] : a[1]);
        double h = 0.0;
        int idx = col;
        for (int k = 1; k < nk - 1; ++k) {
            h += a[2 * k] * tc[idx] - a[2 * k + 1] * ts[idx];
            idx += col;
            if (idx >= we) idx -= we;
        }
        y = (y + 2.0 * h) / we;
        const int b = i * we + col;
        if (MODE == 0) out[b] = (TOut)y;
        else if (MODE == 1) out[3 * b + c] = (TOut)(y / (double)rowsum[b]);
        else out[3 * b + c] += (TOut)(om * y);
    }
}

// Spectral form applicable?  (even widths up to 1024: the row tables fit
// 48 KB of shared memory; K^ of at most 512 MB: 256 x 512 needs 135 MB,
// larger maps take the N-body form)
bool spectral_ok(int he, int we) {
    return (we & 1) == 0 && we <= 1024 && he <= 1024 && (double)he * he * (we / 2 + 1) * 8.0 <= 512.0 * (1 << 20);
}

// Diffuse quadrature: the spectral form with the caller's K^ when given
// (ss_env_khat), else the N-body form.
template <int MODE, typename TIn, typename TOut>
int run_diffuse(int he, int we, const TIn *x, const double *rowsum, TOut *out, double *work, const double *khat,
                cudaStream_t st) {
    const int T = he * we;
    if (khat && spectral_ok(he, we)) {
        const int nk = we / 2 + 1;
        drow_dft_kernel<MODE, TIn><<<he, 256, (2 + (MODE == 0 ? 1 : 3)) * we * sizeof(double), st>>>(he, we, x, rowsum,
                                                                                                      work);
        SS_CUDA_CHECK_LAUNCH();
        constexpr int NC = MODE == 0 ? 1 : 3;
        dmul_kernel<NC><<<nk, 128, 2 * NC * he * sizeof(double), st>>>(he, we, khat, work);
        SS_CUDA_CHECK_LAUNCH();
        dinv_kernel<MODE, TOut><<<he, 256, (2 + NC) * we * sizeof(double), st>>>(he, we, work, rowsum, out);
        SS_CUDA_CHECK_LAUNCH();
        return SS_OK;
    }
    cudaMemsetAsync(work, 0, sizeof(double) * 3 * T, st);
    const dim3 grid((T + kDiffThreads * kOut - 1) / (kDiffThreads * kOut), kSplit);
    diffuse_kernel<MODE, TIn><<<grid, kDiffThreads, 0, st>>>(he, we, x, rowsum, work);
    SS_CUDA_CHECK_LAUNCH();
    diffuse_finish_kernel<MODE, TOut><<<(T + 255) / 256, 256, 0, st>>>(he, we, work, rowsum, out);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

struct SpecSample {
    int idx[4];
    double w[4];
};

// One GGX sample of a specular operator row (shading.py:306-323).
__device__ __forceinline__ bool spec_sample(const double d[3], const double tx[3], const double ty[3], int s,
                                            int samples, double alpha, int he, int we, SpecSample &o, double &wgt) {
    double h[3];
    ggx_h(((double)s + 0.5) / samples, radical_inverse((uint32_t)s), alpha, h);
    double hv[3];
    for (int c = 0; c < 3; ++c) hv[c] = h[0] * tx[c] + h[1] * ty[c] + h[2] * d[c];
    const double vh = (d[0] * hv[0] + d[1] * hv[1]) + d[2] * hv[2];
    double l[3];
    for (int c = 0; c < 3; ++c) l[c] = 2.0 * vh * hv[c] - d[c];
    const double nl = (d[0] * l[0] + d[1] * l[1]) + d[2] * l[2];
    wgt = ss_npmax(nl, 0.0);
    if (!(wgt > 0.0)) return false;
    double fu, fv;
    ss_dir_coords(l, he, we, fu, fv);
    const SsBil<double> b = ss_bil_prepare<double>(he, we, fu, fv, true);
    o.idx[0] = b.j0 * we + b.i0; o.idx[1] = b.j0 * we + b.i1; o.idx[2] = b.j1 * we + b.i0; o.idx[3] = b.j1 * we + b.i1;
    o.w[0] = wgt * (1 - b.tu) * (1 - b.tv); o.w[1] = wgt * b.tu * (1 - b.tv);
    o.w[2] = wgt * (1 - b.tu) * b.tv; o.w[3] = wgt * b.tu * b.tv;
    return true;
}

__device__ __forceinline__ void texel_frame(int a, int he, int we, double d[3], double tx[3], double ty[3]) {
    const int r = a / we, c = a % we;
    const double th = ((double)r + 0.5) * (SS_PI / he);
    const double ph = ((double)c + 0.5) * (2.0 * SS_PI / we) - SS_PI;
    d[0] = sin(th) * cos(ph); d[1] = sin(th) * sin(ph); d[2] = cos(th);
    double up[3] = {0.0, 0.0, 1.0};
    if (!(fabs(d[2]) < 0.999)) { up[0] = 1.0; up[2] = 0.0; }
    tx[0] = up[1] * d[2] - up[2] * d[1]; tx[1] = up[2] * d[0] - up[0] * d[2]; tx[2] = up[0] * d[1] - up[1] * d[0];
    const double tn = sqrt((tx[0] * tx[0] + tx[1] * tx[1]) + tx[2] * tx[2]);
    for (int k = 0; k < 3; ++k) tx[k] /= tn;
    ty[0] = d[1] * tx[2] - d[2] * tx[1]; ty[1] = d[2] * tx[0] - d[0] * tx[2]; ty[2] = d[0] * tx[1] - d[1] * tx[0];
}

// specular[l] = S_l base (l >= 1); level 0 is the identity (shading.py:287-289)
__global__ void __launch_bounds__(128) spec_refresh_kernel(int he, int we, int levels, int samples,
                                                           const double *__restrict__ base, double *__restrict__ spec) {
    const int T = he * we;
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int lv = blockIdx.y + 1;
    if (a >= T) return;
    const double rough = lv / (levels - 1.0), alpha = rough * rough;
    double d[3], tx[3], ty[3];
    texel_frame(a, he, we, d, tx, ty);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, ws = 0.0;
    for (int s = 0; s < samples; ++s) {
        SpecSample o;
        double wgt;
        if (!spec_sample(d, tx, ty, s, samples, alpha, he, we, o, wgt)) continue;
        ws += wgt;
        for (int k = 0; k < 4; ++k) {
            acc0 += o.w[k] * base[3 * o.idx[k]];
            acc1 += o.w[k] * base[3 * o.idx[k] + 1];
            acc2 += o.w[k] * base[3 * o.idx[k] + 2];
        }
    }
    double *out = spec + (size_t)lv * T * 3 + 3 * a;
    if (ws <= 0.0) {
        out[0] = base[3 * a]; out[1] = base[3 * a + 1]; out[2] = base[3 * a + 2];
    } else {
        out[0] = acc0 / ws; out[1] = acc1 / ws; out[2] = acc2 / ws;
    }
}

// d_base += S_l^T g_l (scatter form; atomics), l >= 1
__global__ void __launch_bounds__(128) spec_adjoint_kernel(int he, int we, int levels, int samples,
                                                           const double *__restrict__ g, double *__restrict__ d_base) {
    const int T = he * we;
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int lv = blockIdx.y + 1;
    if (a >= T) return;
    const double *gl = g + (size_t)lv * T * 3;
    const double g0 = gl[3 * a], g1 = gl[3 * a + 1], g2 = gl[3 * a + 2];
    if (g0 == 0.0 && g1 == 0.0 && g2 == 0.0) return;
    const double rough = lv / (levels - 1.0), alpha = rough * rough;
    double d[3], tx[3], ty[3];
    texel_frame(a, he, we, d, tx, ty);
    double ws = 0.0;
    for (int s = 0; s < samples; ++s) {
        SpecSample o;
        double wgt;
        if (spec_sample(d, tx, ty, s, samples, alpha, he, we, o, wgt)) ws += wgt;
    }
    if (ws <= 0.0) {
        atomicAdd(d_base + 3 * a, g0); atomicAdd(d_base + 3 * a + 1, g1); atomicAdd(d_base + 3 * a + 2, g2);
        return;
    }
    const double inv = 1.0 / ws;
    for (int s = 0; s < samples; ++s) {
        SpecSample o;
        double wgt;
        if (!spec_sample(d, tx, ty, s, samples, alpha, he, we, o, wgt)) continue;
        for (int k = 0; k < 4; ++k) {
            const double f = o.w[k] * inv;
            atomicAdd(d_base + 3 * o.idx[k], f * g0);
            atomicAdd(d_base + 3 * o.idx[k] + 1, f * g1);
            atomicAdd(d_base + 3 * o.idx[k] + 2, f * g2);
        }
    }
}

// ---- specular operators as a sparse matrix, built once per env shape ------
// Row r = (l-1)*T + i holds the 4 bilinear corners of every active GGX sample
// of texel i at level l (duplicate columns are kept: the SpMV sums them), each
// weight already divided by the row's weight sum (shading.py:306-329); empty
// rows hold one identity entry.
__global__ void __launch_bounds__(128) spec_count_kernel(int he, int we, int levels, int samples,
                                                         int32_t *__restrict__ nnz) {
    const int T = he * we;
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int lv = blockIdx.y + 1;
    if (a >= T) return;
    const double rough = lv / (levels - 1.0), alpha = rough * rough;
    double d[3], tx[3], ty[3];
    texel_frame(a, he, we, d, tx, ty);
    int act = 0;
    for (int s = 0; s < samples; ++s) {
        SpecSample o;
        double wgt;
        act += spec_sample(d, tx, ty, s, samples, alpha, he, we, o, wgt);
    }
    nnz[(size_t)(lv - 1) * T + a] = act ? 4 * act : 1;
}

__global__ void __launch_bounds__(128) spec_fill_kernel(int he, int we, int levels, int samples,
                                                        const int64_t *__restrict__ row_ptr, int32_t *__restrict__ col,
                                                        double *__restrict__ val) {
    const int T = he * we;
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int lv = blockIdx.y + 1;
    if (a >= T) return;
    const double rough = lv / (levels - 1.0), alpha = rough * rough;
    double d[3], tx[3], ty[3];
    texel_frame(a, he, we, d, tx, ty);
    double ws = 0.0;
    for (int s = 0; s < samples; ++s) {
        SpecSample o;
        double wgt;
        if (spec_sample(d, tx, ty, s, samples, alpha, he, we, o, wgt)) ws += wgt;
    }
    int64_t p = row_ptr[(size_t)(lv - 1) * T + a];
    if (ws <= 0.0) { col[p] = a; val[p] = 1.f; return; }
    const double inv = 1.0 / ws;
    for (int s = 0; s < samples; ++s) {
        SpecSample o;
        double wgt;
        if (!spec_sample(d, tx, ty, s, samples, alpha, he, we, o, wgt)) continue;
        for (int k = 0; k < 4; ++k) { col[p] = o.idx[k]; val[p] = o.w[k] * inv; ++p; }
    }
}

// specular[l][i] = sum_e val_e base[col_e], one warp per row (l >= 1),
// float64 like the reference's dense operator products; the float copy for
// the float32 consumers (nullable)
__global__ void __launch_bounds__(256) spec_apply_kernel(int T, int nrows, const int64_t *__restrict__ row_ptr,
                                                         const int32_t *__restrict__ col, const double *__restrict__ val,
                                                         const double *__restrict__ base, double *__restrict__ spec,
                                                         float *__restrict__ spec_f) {
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= nrows) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int64_t p = row_ptr[r] + lane; p < row_ptr[r + 1]; p += 32) {
        const double w = val[p];
        const int j = col[p];
        s0 = fma(w, base[3 * j], s0); s1 = fma(w, base[3 * j + 1], s1); s2 = fma(w, base[3 * j + 2], s2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
        const size_t o = (size_t)T * 3 + (size_t)r * 3;  // level l = r / T + 1
        spec[o] = s0; spec[o + 1] = s1; spec[o + 2] = s2;
        if (spec_f) { spec_f[o] = (float)s0; spec_f[o + 1] = (float)s1; spec_f[o + 2] = (float)s2; }
    }
}

// d_base[j] += sum_l sum_{e in column j of S_l} val_e g_l[row_e]; the
// transpose (CSC, per level) is the caller's stable sort of the entries by
// (level, column); one warp per output texel.
__global__ void __launch_bounds__(256) spec_apply_t_kernel(int T, int levels, const int64_t *__restrict__ col_ptr,
                                                           const int32_t *__restrict__ row, const double *__restrict__ val,
                                                           const double *__restrict__ g, double *__restrict__ d_base) {
    const int lane = threadIdx.x & 31;
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (j >= T) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int lv = 1; lv < levels; ++lv) {
        const double *gl = g + (size_t)lv * T * 3;
        const size_t c = (size_t)(lv - 1) * T + j;
        for (int64_t p = col_ptr[c] + lane; p < col_ptr[c + 1]; p += 32) {
            const double w = val[p];
            const int i = row[p];
            s0 += w * gl[3 * i]; s1 += w * gl[3 * i + 1]; s2 += w * gl[3 * i + 2];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) { d_base[3 * j] += s0; d_base[3 * j + 1] += s1; d_base[3 * j + 2] += s2; }
}

// base = exp(base_log) in float64 (the reference's base, shading.py:373)
// and its float copies; level 0 of the specular chain is the base itself
template <typename T>
__global__ void exp_kernel(int n, const T *__restrict__ lg, float *__restrict__ base, float *__restrict__ spec0,
                           double *__restrict__ base64, double *__restrict__ spec0_64) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double b = exp((double)lg[k]);
    base[k] = (float)b;
    spec0[k] = (float)b;
    base64[k] = b;
    spec0_64[k] = b;
}

__global__ void narrow_kernel(int n, const double *__restrict__ a, float *__restrict__ b) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) b[k] = (float)a[k];
}

__global__ void adjoint_finish_kernel(int n, const double *__restrict__ g0, const double *__restrict__ base,
                                      double *__restrict__ d_base, float *__restrict__ d_log) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double db = d_base[k] + g0[k];
    d_base[k] = db;
    d_log[k] = (float)(db * base[k]);
}


}  // namespace

extern "C" int ss_brdf_lut(int res, int samples, float *lut, void *stream) {
    if (res < 2 || samples < 1 || !lut) return SS_ERR_INVALID;
    lut_kernel<<<(res * res + 127) / 128, 128, 0, (cudaStream_t)stream>>>(res, samples, lut);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_env_rowsums(int he, int we, const double *khat, double *rowsum, double *work, void *stream) {
    if (he < 2 || we < 2 || !rowsum || !work) return SS_ERR_INVALID;
    return run_diffuse<0, float, double>(he, we, nullptr, nullptr, rowsum, work, khat, (cudaStream_t)stream);
}

extern "C" int ss_spec_apply(int he, int we, int levels, const int64_t *row_ptr, const int32_t *col,
                             const double *val, const double *base, double *specular, float *specular_f,
                             void *stream);
extern "C" int ss_spec_apply_t(int he, int we, int levels, const int64_t *col_ptr, const int32_t *row,
                               const double *val, const double *d_specular, double *d_base, void *stream);

extern "C" size_t ss_env_khat_words(int he, int we) {
    if (he < 2 || we < 2 || !spectral_ok(he, we)) return 0;
    return (size_t)he * he * (we / 2 + 1);
}

extern "C" int ss_env_khat(int he, int we, double *khat, void *stream) {
    if (!khat || ss_env_khat_words(he, we) == 0) return SS_ERR_INVALID;
    dspec_kernel<<<he * he, 128, 3 * we * sizeof(double), (cudaStream_t)stream>>>(he, we, khat);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

template <typename TL>
static int env_refresh(int he, int we, int levels, int samples, const TL *base_log, const SsEnvOps *ops,
                       float *base, float *diffuse, float *specular, double *base64, double *diffuse64,
                       double *specular64, void *stream) {
    if (he < 2 || we < 2 || levels < 1 || !base_log || !ops || !ops->rowsum || !ops->work || !base || !diffuse ||
        !specular || !base64 || !diffuse64 || !specular64)
        return SS_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    const int T = he * we;
    exp_kernel<TL><<<(3 * T + 255) / 256, 256, 0, st>>>(3 * T, base_log, base, specular, base64, specular64);
    SS_CUDA_CHECK_LAUNCH();
    {
        const int rc = run_diffuse<1, double, double>(he, we, base64, ops->rowsum, diffuse64, ops->work, ops->khat, st);
        if (rc != SS_OK) return rc;
        narrow_kernel<<<(3 * T + 255) / 256, 256, 0, st>>>(3 * T, diffuse64, diffuse);
        SS_CUDA_CHECK_LAUNCH();
    }
    if (levels > 1) {
        if (ops->row_ptr && ops->col && ops->rval)
            return ss_spec_apply(he, we, levels, ops->row_ptr, ops->col, ops->rval, base64, specular64, specular,
                                 stream);
        spec_refresh_kernel<<<dim3((T + 127) / 128, levels - 1), 128, 0, st>>>(he, we, levels, samples, base64,
                                                                              specular64);
        SS_CUDA_CHECK_LAUNCH();
        narrow_kernel<<<(int)(((size_t)3 * T * (levels - 1) + 255) / 256), 256, 0, st>>>(
            3 * T * (levels - 1), specular64 + (size_t)3 * T, specular + (size_t)3 * T);
        SS_CUDA_CHECK_LAUNCH();
    }
    return SS_OK;
}

extern "C" int ss_env_refresh(int he, int we, int levels, int samples, const float *base_log, const SsEnvOps *ops,
                              float *base, float *diffuse, float *specular, double *base64, double *diffuse64,
                              double *specular64, void *stream) {
    return env_refresh<float>(he, we, levels, samples, base_log, ops, base, diffuse, specular, base64, diffuse64,
                              specular64, stream);
}

extern "C" int ss_env_refresh64(int he, int we, int levels, int samples, const double *base_log,
                                const SsEnvOps *ops, float *base, float *diffuse, float *specular, double *base64,
                                double *diffuse64, double *specular64, void *stream) {
    return env_refresh<double>(he, we, levels, samples, base_log, ops, base, diffuse, specular, base64, diffuse64,
                               specular64, stream);
}

extern "C" int ss_env_adjoint(int he, int we, int levels, int samples, const double *base, const SsEnvOps *ops,
                              const double *d_diffuse, const double *d_specular, double *d_base, float *d_base_log,
                              void *stream) {
    if (he < 2 || we < 2 || levels < 1 || !base || !ops || !ops->rowsum || !ops->work || !d_diffuse || !d_specular ||
        !d_base || !d_base_log)
        return SS_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    const int T = he * we;
    cudaMemsetAsync(d_base, 0, sizeof(double) * 3 * T, st);
    {
        const int rc = run_diffuse<2, double, double>(he, we, d_diffuse, ops->rowsum, d_base, ops->work, ops->khat, st);
        if (rc != SS_OK) return rc;
    }
    if (levels > 1) {
        if (ops->col_ptr && ops->row && ops->cval) {
            const int rc = ss_spec_apply_t(he, we, levels, ops->col_ptr, ops->row, ops->cval, d_specular, d_base, stream);
            if (rc != SS_OK) return rc;
        } else {
            spec_adjoint_kernel<<<dim3((T + 127) / 128, levels - 1), 128, 0, st>>>(he, we, levels, samples, d_specular,
                                                                                  d_base);
            SS_CUDA_CHECK_LAUNCH();
        }
    }
    adjoint_finish_kernel<<<(3 * T + 255) / 256, 256, 0, st>>>(3 * T, d_specular, base, d_base, d_base_log);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_spec_op_count(int he, int we, int levels, int samples, int32_t *row_nnz, void *stream) {
    if (he < 2 || we < 2 || levels < 2 || samples < 1 || !row_nnz) return SS_ERR_INVALID;
    const int T = he * we;
    spec_count_kernel<<<dim3((T + 127) / 128, levels - 1), 128, 0, (cudaStream_t)stream>>>(he, we, levels, samples, row_nnz);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_spec_op_fill(int he, int we, int levels, int samples, const int64_t *row_ptr, int32_t *col,
                               double *val, void *stream) {
    if (he < 2 || we < 2 || levels < 2 || samples < 1 || !row_ptr || !col || !val) return SS_ERR_INVALID;
    const int T = he * we;
    spec_fill_kernel<<<dim3((T + 127) / 128, levels - 1), 128, 0, (cudaStream_t)stream>>>(he, we, levels, samples,
                                                                                         row_ptr, col, val);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_spec_apply(int he, int we, int levels, const int64_t *row_ptr, const int32_t *col,
                             const double *val, const double *base, double *specular, float *specular_f,
                             void *stream) {
    if (he < 2 || we < 2 || levels < 2 || !row_ptr || !col || !val || !base || !specular) return SS_ERR_INVALID;
    const int T = he * we, nrows = (levels - 1) * T;
    spec_apply_kernel<<<(nrows + 7) / 8, 256, 0, (cudaStream_t)stream>>>(T, nrows, row_ptr, col, val, base, specular,
                                                                         specular_f);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_spec_apply_t(int he, int we, int levels, const int64_t *col_ptr, const int32_t *row,
                               const double *val, const double *d_specular, double *d_base, void *stream) {
    if (he < 2 || we < 2 || levels < 2 || !col_ptr || !row || !val || !d_specular || !d_base) return SS_ERR_INVALID;
    const int T = he * we;
    spec_apply_t_kernel<<<(T + 7) / 8, 256, 0, (cudaStream_t)stream>>>(T, levels, col_ptr, row, val, d_specular, d_base);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
