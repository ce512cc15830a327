// raster_fwd.cu -- per-pixel interval-grouped coverage compositing, forward.
//
// Reference: _forward_kernel, depth_mode 'interval' (rasterizer.py:119-249);
// per-pixel semantics rasterize_pixel/composite_layers (reference.py:133-182).
//
// B200 mapping: one CTA per screen tile (tile*tile threads, one pixel each);
// warps own 8x4 pixel blocks.  The tile's sorted record list is streamed
// through shared memory in CTA-sized chunks (one 96 B record gathered per
// thread with 16-byte loads); each warp then culls 32 staged records at a
// time against its 8x4 block with one ballot and walks only the overlapping
// ones, in list order, all 32 lanes on the same record (shared-memory
// broadcast).  The ray/plane intersection reproduces the reference's float32
// arithmetic exactly (ss_intersect) and the cut-off test rho^2 >= 9 is
// evaluated with numba's float64 promotion (ss_rho2), so coverage and layer
// membership decisions are identical to the reference; the accumulation is
// float32 (outputs are float32 in the reference as well).
//
// kTrain: the training-step variant fuses the L1 photometric loss
// (losses.py:94-108, lambda_ssim = 0) and the per-pixel suffix recursion of
// the backward (backward.py:201-238) into the forward: it writes the loss
// partial sum and, per pixel and layer, the float4 coefficients
// (A, dL/dC_raw rgb) that the pass-2-only backward kernel consumes, so the
// backward never replays the walk a second time.
#include "ss_common.cuh"

namespace {

struct FwdParams {
    int W, H, tile, ntx, k_max;
    float bg0, bg1, bg2;
    const int32_t *offsets;
    const int32_t *pair_rec;
    const SsRecord *records;
    float *rgb, *alpha, *depth;
    int32_t *nlayers;
    int32_t *pair_cover;
    SsStacks st;
    unsigned long long *discarded;
    // training variant
    const float *target;   // (H,W,3)
    float inv_count;       // 1 / (3 H W): mean over all image entries
    float4 *coef;          // (k_max, H*W) float4
    double *loss;          // sum of |rgb - target| (1 double)
};

__device__ __forceinline__ void stage_record(SsRecord *dst, const SsRecord *__restrict__ src) {
    const float4 *s = reinterpret_cast<const float4 *>(src);
    float4 *d = reinterpret_cast<float4 *>(dst);
#pragma unroll
    for (int k = 0; k < 6; ++k) d[k] = __ldg(s + k);
}

template <bool kExtras, bool kTrain>
__global__ void __launch_bounds__(256) raster_fwd_kernel(FwdParams P)
{
    extern __shared__ SsRecord srec[];
    __shared__ double loss_red[32];
    const int t = blockIdx.x;
    const int tx = t % P.ntx, ty = t / P.ntx;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int wpr = P.tile >> 3;  // warps per tile row (8 px wide each)
    const int bx = tx * P.tile + (wid % wpr) * 8, by = ty * P.tile + (wid / wpr) * 4;
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    const bool live = px < P.W && py < P.H;
    const float x = ss_ndc_x(px, P.W), y = ss_ndc_y(py, P.H);

    float Wg = 0.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Zg = 0.f, Z2g = 0.f, zmax = 0.f;
    float T = 1.f, o0 = 0.f, o1 = 0.f, o2 = 0.f, dnum = 0.f, dden = 0.f;
    int layers = 0, members = 0;
    bool stopped = false;
    unsigned discarded = 0;
    const size_t pix = live ? (size_t)py * P.W + px : 0;
    // training: per-layer raw sums for the suffix recursion
    constexpr int KL = kTrain ? SS_KMAX_CAP : 1;
    float lw[KL], lc0[KL], lc1[KL], lc2[KL];

    auto close_layer = [&]() {
        const float a_k = -expm1f(-Wg);
        const float inv_w = 1.f / Wg;
        const float ta = T * a_k;
        o0 += ta * C0 * inv_w; o1 += ta * C1 * inv_w; o2 += ta * C2 * inv_w;
        dnum += ta * Zg * inv_w; dden += ta;
        T *= 1.f - a_k;
        if (kExtras && P.st.w) {
            const size_t o = pix * P.k_max + layers;
            P.st.w[o] = Wg; P.st.c[3 * o] = C0; P.st.c[3 * o + 1] = C1; P.st.c[3 * o + 2] = C2;
            P.st.z[o] = Zg; P.st.z2[o] = Z2g; P.st.n[o] = members;
        }
        if (kTrain) { lw[layers] = Wg; lc0[layers] = C0; lc1[layers] = C1; lc2[layers] = C2; }
        ++layers;
        Wg = C0 = C1 = C2 = Zg = Z2g = zmax = 0.f;
        members = 0;
    };

    const int p0 = P.offsets[t], p1 = P.offsets[t + 1];
    const int nthreads = blockDim.x;
    for (int base = p0; base < p1; base += nthreads) {
        const int cn = min(nthreads, p1 - base);
        __syncthreads();
        if ((int)threadIdx.x < cn) stage_record(&srec[threadIdx.x], P.records + P.pair_rec[base + threadIdx.x]);
        __syncthreads();
        for (int sub = 0; sub < cn; sub += 32) {
            // warp-level cull: which of these 32 records touch my 8x4 block?
            bool ov = false;
            if (sub + lane < cn) {
                const int4 r = srec[sub + lane].r;
                ov = r.x < bx + 8 && r.z > bx && r.y < by + 4 && r.w > by;
            }
            unsigned mask = __ballot_sync(0xffffffffu, ov);
            while (mask) {
                const int j = sub + __ffs(mask) - 1;
                mask &= mask - 1;
                const SsRecord &R = srec[j];
                const int4 r = R.r;
                const bool inr = live && px >= r.x && px < r.z && py >= r.y && py < r.w;
                bool cov = false;
                if (inr) {
                    if (stopped) {
                        ++discarded;
                    } else {
                        bool go = true;
                        if (Wg > 0.f && R.d.z > zmax) {
                            close_layer();  // rasterizer.py:168-196
                            if (layers >= P.k_max) { stopped = true; ++discarded; go = false; }
                        }
                        if (go) {
                            const float t1[3] = {R.a.x, R.a.y, R.a.z};
                            const float t2[3] = {R.a.w, R.b.x, R.b.y};
                            const float t4[3] = {R.b.z, R.b.w, R.c.x};
                            SsHit h;
                            if (ss_intersect(x, y, t1, t2, t4, h)) {
                                const double rho2 = ss_rho2(R.c.y, R.c.z, R.c.w, h.u, h.v);
                                if (rho2 < 9.0) {
                                    cov = true;
                                    const float w = R.d.x * __expf(-0.5f * (float)rho2);
                                    const float z = R.d.y;
                                    Wg += w;
                                    C0 += w * R.e.x; C1 += w * R.e.y; C2 += w * R.e.z;
                                    if (!kTrain) { Zg += w * z; Z2g += w * z * z; }
                                    ++members;
                                    if (R.d.w > zmax) zmax = R.d.w;
                                }
                            }
                        }
                    }
                }
                if (kExtras && P.pair_cover) {
                    const unsigned cm = __ballot_sync(0xffffffffu, cov);
                    if (cm && lane == 0) atomicAdd(&P.pair_cover[base + j], __popc(cm));
                }
            }
        }
    }
    double lsum = 0.0;
    if (live) {
        if (Wg > 0.f) close_layer();
        const float r0 = o0 + T * P.bg0, r1 = o1 + T * P.bg1, r2 = o2 + T * P.bg2;
        if (!kTrain || P.rgb) {
            P.rgb[3 * pix] = r0; P.rgb[3 * pix + 1] = r1; P.rgb[3 * pix + 2] = r2;
        }
        if (!kTrain) {
            P.alpha[pix] = 1.f - T;
            P.depth[pix] = dden > 0.f ? dnum / dden : 0.f;
            P.nlayers[pix] = layers;
        } else {
            // L1 loss and its image gradient (losses.py:100-104)
            const float d0 = r0 - P.target[3 * pix], d1 = r1 - P.target[3 * pix + 1], d2 = r2 - P.target[3 * pix + 2];
            lsum = (double)fabsf(d0) + (double)fabsf(d1) + (double)fabsf(d2);
            const float sg = P.inv_count;
            const float gc0 = d0 > 0.f ? sg : (d0 < 0.f ? -sg : 0.f);
            const float gc1 = d1 > 0.f ? sg : (d1 < 0.f ? -sg : 0.f);
            const float gc2 = d2 > 0.f ? sg : (d2 < 0.f ? -sg : 0.f);
            // suffix recursion over the layers (backward.py:201-238, no
            // consolidation, no coverage loss): per layer A and dL/dC_raw
            float tb[KL], av[KL];
            float tr = 1.f;
            for (int m = 0; m < layers; ++m) {
                av[m] = -expm1f(-lw[m]);
                tb[m] = tr;
                tr *= 1.f - av[m];
            }
            float sf0 = P.bg0, sf1 = P.bg1, sf2 = P.bg2;
            const size_t HW = (size_t)P.W * P.H;
            for (int m = layers - 1; m >= 0; --m) {
                const float inv = 1.f / lw[m];
                const float ch0 = lc0[m] * inv, ch1 = lc1[m] * inv, ch2 = lc2[m] * inv;
                const float a = av[m];
                const float g_am = tb[m] * (gc0 * (ch0 - sf0) + gc1 * (ch1 - sf1) + gc2 * (ch2 - sf2));
                const float ta = tb[m] * a;
                const float gh0 = gc0 * ta, gh1 = gc1 * ta, gh2 = gc2 * ta;
                float4 cf;
                cf.x = g_am * (1.f - a) - (gh0 * ch0 + gh1 * ch1 + gh2 * ch2) * inv;
                cf.y = gh0 * inv; cf.z = gh1 * inv; cf.w = gh2 * inv;
                P.coef[(size_t)m * HW + pix] = cf;
                sf0 = a * ch0 + (1.f - a) * sf0;
                sf1 = a * ch1 + (1.f - a) * sf1;
                sf2 = a * ch2 + (1.f - a) * sf2;
            }
        }
    }
    if (kExtras && P.discarded) {
        unsigned d = discarded;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (lane == 0 && d) atomicAdd(P.discarded, (unsigned long long)d);
    }
    if (kTrain) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        if (lane == 0) loss_red[wid] = lsum;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += loss_red[k];
            atomicAdd(P.loss, s);
        }
    }
}

template <bool kExtras, bool kTrain>
void launch(const FwdParams &P, int ntiles, int threads, cudaStream_t st) {
    raster_fwd_kernel<kExtras, kTrain><<<ntiles, threads, threads * sizeof(SsRecord), st>>>(P);
}

bool fill_common(FwdParams &P, int width, int height, int tile, const int32_t *tile_offsets,
                 const int32_t *pair_rec, const float *records, const float *background, int k_max) {
    if (width <= 0 || height <= 0 || tile < 8 || tile > 16 || (tile & 7) || k_max < 1 || k_max > SS_KMAX_CAP)
        return false;
    if (!tile_offsets || !background) return false;
    P = FwdParams{};
    P.W = width; P.H = height; P.tile = tile; P.ntx = (width + tile - 1) / tile; P.k_max = k_max;
    P.bg0 = background[0]; P.bg1 = background[1]; P.bg2 = background[2];
    P.offsets = tile_offsets; P.pair_rec = pair_rec;
    P.records = reinterpret_cast<const SsRecord *>(records);
    return true;
}

}  // namespace

extern "C" int ss_raster_forward(int width, int height, int tile, const int32_t *tile_offsets,
                                 const int32_t *pair_rec, const float *records, const float *background,
                                 int k_max, float *rgb, float *alpha, float *depth, int32_t *nlayers,
                                 int32_t *pair_cover, const SsStacks *stacks, unsigned long long *discarded,
                                 void *stream)
{
    FwdParams P;
    if (!fill_common(P, width, height, tile, tile_offsets, pair_rec, records, background, k_max)) return SS_ERR_INVALID;
    if (!rgb || !alpha || !depth || !nlayers) return SS_ERR_INVALID;
    P.rgb = rgb; P.alpha = alpha; P.depth = depth; P.nlayers = nlayers;
    P.pair_cover = pair_cover;
    P.st = stacks ? *stacks : SsStacks{};
    P.discarded = discarded;
    const int ntiles = P.ntx * ((height + tile - 1) / tile);
    const bool extras = pair_cover || (stacks && stacks->w) || discarded;
    if (extras) launch<true, false>(P, ntiles, tile * tile, (cudaStream_t)stream);
    else launch<false, false>(P, ntiles, tile * tile, (cudaStream_t)stream);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_train_forward(int width, int height, int tile, const int32_t *tile_offsets,
                                const int32_t *pair_rec, const float *records, const float *background,
                                int k_max, const float *target, float *coef, double *loss_sum, float *rgb,
                                void *stream)
{
    FwdParams P;
    if (!fill_common(P, width, height, tile, tile_offsets, pair_rec, records, background, k_max)) return SS_ERR_INVALID;
    if (!target || !coef || !loss_sum) return SS_ERR_INVALID;
    P.target = target;
    P.inv_count = (float)(1.0 / (3.0 * (double)width * (double)height));
    P.coef = reinterpret_cast<float4 *>(coef);
    P.loss = loss_sum;
    P.rgb = rgb;
    const int ntiles = P.ntx * ((height + tile - 1) / tile);
    launch<false, true>(P, ntiles, tile * tile, (cudaStream_t)stream);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
