// losses.cu -- the image losses of the reference fit step on the device:
// tone mapping (shading.py:40-79), L1 + SSIM photometric loss
// (losses.py:45-108) and the silhouette soft-IoU (losses.py:111-123), with
// their input gradients.  SURVEY §8(f) rank 1.
//
// Layout: images (H, W, C) float32 row-major, C in {1, 3}.  Everything is
// evaluated in float64 like the reference (the SSIM variances are
// differences of window means: float32 would cancel).  SSIM = the 11x11
// separable Gaussian window (sigma 1.5, zero boundary), mean over the fully
// windowed interior; its adjoint reuses the same (self-adjoint) window.
//
// Kernels: (1) tone map + L1 sum; (2) SSIM forward on 16x16 output tiles
// (halo 5 staged in shared memory, horizontal then vertical pass for the five
// window moments), writing the three adjoint maps; (3) SSIM adjoint on the
// same tiling, fused with the L1 gradient and the tone-map backward.  The
// scalar results stay on the device (no host sync).
#include "ss_common.cuh"

namespace {

constexpr int kWin = 11, kHalf = 5, kT = 16, kP = kT + 2 * kHalf;  // kP: tile + halo
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;
constexpr double kLinBound = 0.0031308;

struct LossParams {
    int H, W, C, mode;           // mode: -1 identity, 0 ldr, 1 hdr-loss
    double lambda_ssim;
    double win[kWin];
    const float *x, *y;          // (H, W, C)
    double *mx, *my;             // tone-mapped images
    double *gmu, *gx2, *gxy;     // SSIM adjoint maps
    double *sums;                // [0] sum |mx - my|, [1] sum of the SSIM map over the interior
    float *grad;                 // d loss / d x (pre-tone-map input)
    double *grad64;              // nullable: the same in float64
};

__device__ __forceinline__ double srgb(double t) {
    return t <= kLinBound ? t * 12.92 : 1.055 * pow(fmax(t, kLinBound), 1.0 / 2.4) - 0.055;
}
__device__ __forceinline__ double srgb_grad(double t) {
    return t <= kLinBound ? 12.92 : (1.055 / 2.4) * pow(fmax(t, kLinBound), 1.0 / 2.4 - 1.0);
}
__device__ __forceinline__ double tone(double v, int mode) {
    if (mode == 0) return srgb(fmin(fmax(v, 0.0), 1.0));
    if (mode == 1) return srgb(log1p(fmax(v, 0.0)));
    return v;
}
__device__ __forceinline__ double tone_bwd(double v, int mode, double g) {
    if (mode == 0) return (v > 0.0 && v < 1.0) ? g * srgb_grad(fmin(fmax(v, 0.0), 1.0)) : 0.0;
    if (mode == 1) {
        const double xp = fmax(v, 0.0);
        return v > 0.0 ? g * srgb_grad(log1p(xp)) / (1.0 + xp) : 0.0;
    }
    return g;
}

__device__ __forceinline__ void block_add(double v, double *dst) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v != 0.0) atomicAdd(dst, v);
}

__global__ void tone_l1_kernel(LossParams P, int64_t n) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double a = tone((double)P.x[i], P.mode), b = tone((double)P.y[i], P.mode);
        P.mx[i] = a;
        P.my[i] = b;
        acc += fabs(a - b);
    }
    block_add(acc, P.sums);
}

// Load the (kP x kP) halo patch of channel c of up to three maps into smem
// (zero outside the image = the reference's constant boundary).
template <int NM>
__device__ __forceinline__ void load_patch(const LossParams &P, const double *const src[NM], int c, int y0, int x0,
                                           double (*patch)[kP][kP]) {
    for (int k = threadIdx.x; k < kP * kP; k += blockDim.x) {
        const int py = k / kP, px = k % kP;
        const int gy = y0 - kHalf + py, gx = x0 - kHalf + px;
        const bool in = gy >= 0 && gy < P.H && gx >= 0 && gx < P.W;
        const size_t idx = ((size_t)gy * P.W + gx) * P.C + c;
#pragma unroll
        for (int m = 0; m < NM; ++m) patch[m][py][px] = in ? src[m][idx] : 0.0;
    }
}

__global__ void __launch_bounds__(256) ssim_fwd_kernel(LossParams P) {
    __shared__ double patch[2][kP][kP];
    __shared__ double hsum[5][kP][kT];
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;
    const int gx = x0 + tx, gy = y0 + ty;
    const double n_valid = (double)(P.H - 2 * kHalf) * (P.W - 2 * kHalf) * P.C;
    const bool valid = gy >= kHalf && gy < P.H - kHalf && gx >= kHalf && gx < P.W - kHalf;
    double s_acc = 0.0;
    const double *src[2] = {P.mx, P.my};
    for (int c = 0; c < P.C; ++c) {
        load_patch<2>(P, src, c, y0, x0, patch);
        __syncthreads();
        // horizontal pass: rows of the patch x the tile's columns, five moments
        for (int k = threadIdx.x; k < kP * kT; k += blockDim.x) {
            const int r = k / kT, col = k % kT;
            double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
#pragma unroll
            for (int j = 0; j < kWin; ++j) {
                const double a = patch[0][r][col + j], b = patch[1][r][col + j], wj = P.win[j];
                m0 += wj * a; m1 += wj * b; m2 += wj * a * a; m3 += wj * b * b; m4 += wj * a * b;
            }
            hsum[0][r][col] = m0; hsum[1][r][col] = m1; hsum[2][r][col] = m2; hsum[3][r][col] = m3;
            hsum[4][r][col] = m4;
        }
        __syncthreads();
        double mu_x = 0.0, mu_y = 0.0, x2 = 0.0, y2 = 0.0, xy = 0.0;
#pragma unroll
        for (int j = 0; j < kWin; ++j) {
            const double wj = P.win[j];
            mu_x += wj * hsum[0][ty + j][tx]; mu_y += wj * hsum[1][ty + j][tx];
            x2 += wj * hsum[2][ty + j][tx]; y2 += wj * hsum[3][ty + j][tx]; xy += wj * hsum[4][ty + j][tx];
        }
        if (gx < P.W && gy < P.H) {
            const double var_x = x2 - mu_x * mu_x, var_y = y2 - mu_y * mu_y, cov = xy - mu_x * mu_y;
            const double a1 = 2.0 * mu_x * mu_y + kC1, a2 = 2.0 * cov + kC2;
            const double b1 = mu_x * mu_x + mu_y * mu_y + kC1, b2 = var_x + var_y + kC2;
            const double s = (a1 * a2) / (b1 * b2);
            const double e = valid ? -1.0 / n_valid : 0.0;
            if (valid) s_acc += s;
            const double ds_mu = 2.0 * mu_y * a2 / (b1 * b2) - 2.0 * mu_x * s / b1;
            const double ds_var = -s / b2, ds_cov = 2.0 * a1 / (b1 * b2);
            const size_t idx = ((size_t)gy * P.W + gx) * P.C + c;
            P.gmu[idx] = e * (ds_mu - 2.0 * mu_x * ds_var - mu_y * ds_cov);
            P.gx2[idx] = e * ds_var;
            P.gxy[idx] = e * ds_cov;
        }
        __syncthreads();
    }
    block_add(s_acc, P.sums + 1);
}

// SSIM adjoint (window filter of the three adjoint maps) fused with the L1
// gradient, the (1 - lambda, lambda) mix and the tone-map backward.
__global__ void __launch_bounds__(256) ssim_bwd_kernel(LossParams P) {
    __shared__ double patch[3][kP][kP];
    __shared__ double hsum[3][kP][kT];
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;
    const int gx = x0 + tx, gy = y0 + ty;
    const double inv_n = 1.0 / ((double)P.H * P.W * P.C);
    const double *src[3] = {P.gmu, P.gx2, P.gxy};
    for (int c = 0; c < P.C; ++c) {
        load_patch<3>(P, src, c, y0, x0, patch);
        __syncthreads();
        for (int k = threadIdx.x; k < kP * kT; k += blockDim.x) {
            const int r = k / kT, col = k % kT;
            double m0 = 0.0, m1 = 0.0, m2 = 0.0;
#pragma unroll
            for (int j = 0; j < kWin; ++j) {
                const double wj = P.win[j];
                m0 += wj * patch[0][r][col + j]; m1 += wj * patch[1][r][col + j]; m2 += wj * patch[2][r][col + j];
            }
            hsum[0][r][col] = m0; hsum[1][r][col] = m1; hsum[2][r][col] = m2;
        }
        __syncthreads();
        if (gx < P.W && gy < P.H) {
            double w0 = 0.0, w1 = 0.0, w2 = 0.0;
#pragma unroll
            for (int j = 0; j < kWin; ++j) {
                const double wj = P.win[j];
                w0 += wj * hsum[0][ty + j][tx]; w1 += wj * hsum[1][ty + j][tx]; w2 += wj * hsum[2][ty + j][tx];
            }
            const size_t idx = ((size_t)gy * P.W + gx) * P.C + c;
            const double a = P.mx[idx], b = P.my[idx];
            const double g_ssim = w0 + 2.0 * a * w1 + b * w2;
            const double d = a - b;
            const double g_l1 = (d > 0.0 ? inv_n : (d < 0.0 ? -inv_n : 0.0));
            const double g = (1.0 - P.lambda_ssim) * g_l1 + P.lambda_ssim * g_ssim;
            const double gx = tone_bwd((double)P.x[idx], P.mode, g);
            P.grad[idx] = (float)gx;
            if (P.grad64) P.grad64[idx] = gx;
        }
        __syncthreads();
    }
}

__global__ void l1_grad_kernel(LossParams P, int64_t n) {
    const double inv_n = 1.0 / (double)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = P.mx[i] - P.my[i];
        const double g = d > 0.0 ? inv_n : (d < 0.0 ? -inv_n : 0.0);
        const double gx = tone_bwd((double)P.x[i], P.mode, (1.0 - P.lambda_ssim) * g);
        P.grad[i] = (float)gx;
        if (P.grad64) P.grad64[i] = gx;
    }
}

// out[0] = (1 - lambda) mean|mx - my| + lambda (1 - mean SSIM), out[1] = L1, out[2] = 1 - SSIM
__global__ void finish_kernel(const double *sums, int H, int W, int C, double lambda, bool ssim, double *out) {
    const double n = (double)H * W * C;
    const double l1 = sums[0] / n;
    double sl = 0.0;
    if (ssim) sl = 1.0 - sums[1] / ((double)(H - 2 * kHalf) * (W - 2 * kHalf) * C);
    out[0] = (1.0 - lambda) * l1 + lambda * sl;
    out[1] = l1;
    out[2] = sl;
}

__global__ void tone_map_kernel(int64_t n, const float *img, int mode, float *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)tone((double)img[i], mode);
}

__global__ void tone_map_bwd_kernel(int64_t n, const float *img, int mode, const float *g_out, float *g_in) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        g_in[i] = (float)tone_bwd((double)img[i], mode, (double)g_out[i]);
}

__global__ void sil_sums_kernel(int64_t n, const float *alpha, const float *mask, double *sums) {
    double inter = 0.0, uni = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double a = alpha[i], m = mask[i];
        inter += a * m;
        uni += a + m - a * m;
    }
    block_add(inter, sums);
    block_add(uni, sums + 1);
}

__global__ void sil_grad_kernel(int64_t n, const float *mask, const double *sums, float *grad, double *out) {
    const double inter = sums[0], uni = sums[1];
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = uni > 0.0 ? 1.0 - inter / uni : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double m = mask[i];
        grad[i] = uni > 0.0 ? (float)((inter * (1.0 - m) - m * uni) / (uni * uni)) : 0.0f;
    }
}

int grid_for(int64_t n) { return (int)((n + 255) / 256 < ss_sm_count() * 8 ? (n + 255) / 256 : ss_sm_count() * 8); }

}  // namespace

extern "C" size_t ss_photometric_workspace(int height, int width, int channels) {
    return (5 * (size_t)height * width * channels + 8) * sizeof(double);
}

extern "C" int ss_photometric_loss(int height, int width, int channels, const float *x, const float *y, int tone_mode,
                                   double lambda_ssim, double *out, float *grad, double *grad64, double *workspace,
                                   void *stream)
{
    if (height <= 0 || width <= 0 || (channels != 1 && channels != 3) || tone_mode < -1 || tone_mode > 1)
        return SS_ERR_INVALID;
    if (!x || !y || !out || !grad || !workspace || !(lambda_ssim >= 0.0 && lambda_ssim <= 1.0)) return SS_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = (int64_t)height * width * channels;
    LossParams P{};
    P.H = height; P.W = width; P.C = channels; P.mode = tone_mode; P.lambda_ssim = lambda_ssim;
    double ksum = 0.0;
    for (int j = 0; j < kWin; ++j) {
        const double t = (j - (kWin - 1) / 2.0) / 1.5;
        P.win[j] = exp(-0.5 * t * t);
        ksum += P.win[j];
    }
    for (int j = 0; j < kWin; ++j) P.win[j] /= ksum;  // losses.py:24-28
    P.x = x; P.y = y;
    P.mx = workspace; P.my = P.mx + n; P.gmu = P.my + n; P.gx2 = P.gmu + n; P.gxy = P.gx2 + n;
    P.sums = P.gxy + n;
    P.grad = grad;
    P.grad64 = grad64;
    cudaMemsetAsync(P.sums, 0, 8 * sizeof(double), st);
    tone_l1_kernel<<<grid_for(n), 256, 0, st>>>(P, n);
    SS_CUDA_CHECK_LAUNCH();
    // SSIM is zero (and its gradient too) when the image is smaller than the window (losses.py:55-56)
    const bool ssim = lambda_ssim > 0.0 && height >= kWin && width >= kWin;
    if (ssim) {
        const dim3 g((width + kT - 1) / kT, (height + kT - 1) / kT);
        ssim_fwd_kernel<<<g, kT * kT, 0, st>>>(P);
        SS_CUDA_CHECK_LAUNCH();
        ssim_bwd_kernel<<<g, kT * kT, 0, st>>>(P);
        SS_CUDA_CHECK_LAUNCH();
    } else {
        l1_grad_kernel<<<grid_for(n), 256, 0, st>>>(P, n);
        SS_CUDA_CHECK_LAUNCH();
    }
    finish_kernel<<<1, 1, 0, st>>>(P.sums, height, width, channels, lambda_ssim, ssim, out);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_tone_map(int64_t n, const float *img, int tone_mode, float *out, void *stream)
{
    if (n < 0 || tone_mode < 0 || tone_mode > 1 || (n > 0 && (!img || !out))) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    tone_map_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, img, tone_mode, out);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_tone_map_backward(int64_t n, const float *img, int tone_mode, const float *g_out, float *g_in,
                                    void *stream)
{
    if (n < 0 || tone_mode < 0 || tone_mode > 1 || (n > 0 && (!img || !g_out || !g_in))) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    tone_map_bwd_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, img, tone_mode, g_out, g_in);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_silhouette_loss(int64_t n, const float *alpha, const float *mask, double *out, float *grad,
                                  double *workspace, void *stream)
{
    if (n <= 0 || !alpha || !mask || !out || !grad || !workspace) return SS_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(workspace, 0, 2 * sizeof(double), st);
    sil_sums_kernel<<<grid_for(n), 256, 0, st>>>(n, alpha, mask, workspace);
    SS_CUDA_CHECK_LAUNCH();
    sil_grad_kernel<<<grid_for(n), 256, 0, st>>>(n, mask, workspace, grad, out);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
