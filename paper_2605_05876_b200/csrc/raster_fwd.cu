// raster_fwd.cu -- per-pixel interval-grouped coverage compositing, forward.
//
// Reference: _forward_kernel, depth_mode 'interval' (rasterizer.py:119-249);
// per-pixel semantics rasterize_pixel/composite_layers (reference.py:133-182).
//
// B200 mapping: one CTA per screen tile (tile*tile threads, one pixel each);
// warps own 8x4 pixel blocks and walk the tile's sorted pair list
// independently (raster_walk.cuh: 32 packed rects per ballot, only the
// overlapping records are gathered into the warp's shared-memory slots, no
// CTA barrier), all 32 lanes on the same record in list order.  Coverage
// (raster_walk.cuh ss_cover) reproduces the reference's float32 intersection
// bit for bit and re-takes the decision with numba's float64 rho^2 when the
// float32 value is within 1e-4 of the cut-off, so coverage and layer
// membership are identical to the reference (verified at scale by
// ss_debug_cover_check); accumulation is float32 (the reference's outputs are
// float32 too).
//
// kTrain: the training-step variant fuses the L1 photometric loss
// (losses.py:94-108, lambda_ssim = 0) and the per-pixel suffix recursion of
// the backward (backward.py:201-238) into the forward: it writes the loss
// partial sum and, per pixel and layer, the float4 coefficients
// (A, dL/dC_raw rgb) that the pass-2-only backward kernel consumes, so the
// backward never replays the walk a second time.
#include <type_traits>
#include "ss_common.cuh"
#include "raster_walk.cuh"

#ifdef SS_CTA_TIMING
__device__ unsigned long long *g_fwd_times;  // (3 per CTA): start, end, smid
extern "C" int ss_debug_set_fwd_timing(void *buf) {
    return cudaMemcpyToSymbol(g_fwd_times, &buf, sizeof(buf)) == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}
#else
extern "C" int ss_debug_set_fwd_timing(void *) { return SS_ERR_INVALID; }
#endif

namespace {

struct FwdParams {
    int W, H, tile, ntx, k_max;
    float bg0, bg1, bg2;
    const int32_t *offsets;
    const int32_t *tile_order;  // nullable: launch order of the tiles (heavy first)
    const int32_t *pair_rec;
    const uint2 *pair_rect;
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
    float *thr;            // (k_max, H*W) depth at which layer j >= 3 closed
    int4 *hdr;             // (H*W, 2) packed (closed-layer count, closing depths of layers 0..2), (depths 3..6)
    double *loss;          // sum of |rgb - target| (1 double)
    float4 *zst;           // kCons: (k_max, H*W) per layer (z0, sum w dz, sum w dz^2, 0), dz = view_z - z0
};

// Layer coefficients of the backward, stored without losing the record-
// colour cancellation: g_w(c) = A + sum_c G_c c_c with A = g_am (1 - a) -
// sum_c G_c c_hat_c is a small difference of large terms whenever a record's
// colour is close to its layer's mean colour c_hat, so A is formed from the
// ROUNDED G_c (then g_w = g_am (1 - a) + sum_c G_c (c_c - c_hat_c) exactly)
// and stored as float hi + lo (the lo plane follows the k_max float4 planes
// in `coef`).  The backward evaluates g_w in float64.
__device__ __forceinline__ void store_coef(float4 *coef, size_t o, size_t lo_off, double base, double gh0, double gh1,
                                           double gh2, double inv, double ch0, double ch1, double ch2) {
    const float g0 = (float)(gh0 * inv), g1 = (float)(gh1 * inv), g2 = (float)(gh2 * inv);
    const double A = base - ((double)g0 * ch0 + (double)g1 * ch1 + (double)g2 * ch2);
    const float hi = (float)A;
    coef[o] = make_float4(hi, g0, g1, g2);
    reinterpret_cast<float *>(coef + lo_off)[o] = (float)(A - (double)hi);
}

// CTAs of kFwdWarps warps (a tile is split over tile*tile/32/kFwdWarps
// CTAs; measured 4 > 2 = 8 > 1 with the heavy-first tile order): warps never
// wait for each other.
#ifndef SS_FWD_WARPS
#define SS_FWD_WARPS 4
#endif
constexpr int kFwdWarps = SS_FWD_WARPS;

// kCons (deferred training mode only): also the per-layer depth moments the
// consolidation penalty needs, relative to the layer's first covering member
// like the reference's pass 1 (raster_bwd.cu), parked in P.zst per layer.
// kDeferred (deferred-loss training forward): float64 layer sums, stored
// as float hi + lo parts (the coefficient kernel forms the layer mean colour
// from them)
template <bool kExtras, bool kTrain, bool kCons = false, bool kDeferred = false>
__global__ void __launch_bounds__(32 * kFwdWarps) raster_fwd_kernel(FwdParams P)
{
    __shared__ PackedScratch scratch[kFwdWarps];
#ifdef SS_CTA_TIMING
    const unsigned long long t_start = ss_globaltimer();
#endif
    const int wpc = blockDim.x >> 5;  // kFwdWarps, or fewer for 8x8 tiles
    const int ctas_per_tile = P.tile * P.tile / (32 * wpc);
    const int t = P.tile_order ? P.tile_order[blockIdx.x / ctas_per_tile] : blockIdx.x / ctas_per_tile;
    const int wid_in_tile = (blockIdx.x % ctas_per_tile) * wpc + (threadIdx.x >> 5);
    const WarpPix wp = warp_pixels(t, P.ntx, P.tile, P.W, P.H, wid_in_tile);
    const int lane = wp.lane, wid = threadIdx.x >> 5;
    const bool live = wp.live;
    const size_t pix = wp.pix;
    PackedScratch &sm = scratch[wid];
    packed_init(wp, sm, P.W, P.H);

    // layer sums: float64 in the training modes (the layer's mean colour
    // C / W enters the backward through record colour - mean colour, which
    // float32 sums would blur), float32 for the plain render
#ifdef SS_FWD_F64_SUMS
    using AccT = typename std::conditional<kTrain, double, float>::type;
#else
    using AccT = typename std::conditional<kDeferred, double, float>::type;
#endif
    AccT Wg = 0, C0 = 0, C1 = 0, C2 = 0;
    float Zg = 0.f, Z2g = 0.f, zmax = 0.f;
    float T = 1.f, o0 = 0.f, o1 = 0.f, o2 = 0.f, dnum = 0.f, dden = 0.f;
    int layers = 0, members = 0;
    bool stopped = !live;
    unsigned discarded = 0;
    // training: per-layer raw sums for the suffix recursion
    constexpr int KL = kTrain ? SS_KMAX_CAP : 1;
    AccT lw[KL], lc0[KL], lc1[KL], lc2[KL];
    int ncl = 0;
    float th0 = 0.f, th1 = 0.f, th2 = 0.f;  // first three closing depths (kTrain)
    float z0 = 0.f, Zs = 0.f, Z2s = 0.f;     // kCons: layer depth moments about the first member

    // one layer of the over-compositing (rasterizer.py:168-181)
    auto composite = [&](float w, float c0, float c1, float c2) {
        const float a_k = -expm1f(-w);
        const float inv_w = 1.f / w;
        const float ta = T * a_k;
        o0 += ta * c0 * inv_w; o1 += ta * c1 * inv_w; o2 += ta * c2 * inv_w;
        if (!kTrain) { dnum += ta * Zg * inv_w; dden += ta; }
        T *= 1.f - a_k;
    };
    // closing a layer in the training walk only parks its raw sums: the
    // compositing is replayed (same operations, same order) once per pixel
    // after the walk, off the hot loop
    auto close_layer = [&]() {
        if (!kTrain) composite((float)Wg, (float)C0, (float)C1, (float)C2);
        if (kExtras && P.st.w) {
            const size_t o = pix * P.k_max + layers;
            P.st.w[o] = (float)Wg; P.st.c[3 * o] = (float)C0; P.st.c[3 * o + 1] = (float)C1; P.st.c[3 * o + 2] = (float)C2;
            P.st.z[o] = Zg; P.st.z2[o] = Z2g; P.st.n[o] = members;
        }
        if (kTrain) { lw[layers] = Wg; lc0[layers] = C0; lc1[layers] = C1; lc2[layers] = C2; }
        if (kCons) {
            P.zst[(size_t)layers * P.W * P.H + pix] = make_float4(z0, Zs, Z2s, 0.f);
            Zs = Z2s = 0.f;
        }
        ++layers;
        Wg = C0 = C1 = C2 = 0;
        Zg = Z2g = zmax = 0.f;
        members = 0;
    };

    const int p0 = P.offsets[t], p1 = P.offsets[t + 1];
    // early exit between chunks once every lane of the warp stopped (only
    // when the discard statistic is not requested)
    {
        walk_tile_packed<!kExtras>(wp, p0, p1, P.pair_rec, P.pair_rect, P.records, sm, kExtras ? P.pair_cover : nullptr,
            [&]() { return !kExtras && __all_sync(0xffffffffu, stopped); },
            // the forward keeps the reference's own float32 sequence: its weights
            // then match the reference's to ~1e-7 (the fast linear-form path of
            // coverage.cuh decides coverage identically but its weights carry
            // independent rounding noise of ~1e-4 relative at the support edge)
            [](const RecGeo &R, float x, float y) {
                Cover c;
                return ss_cover(x, y, R, c) ? R.d.x * ss_exp_fast(-0.5f * c.rho2) : -1.f;
            },
            [&](const SlotView &v) {
            if (stopped) {
                ++discarded;
                return;
            }
            if (Wg > 0.f && v.zs > zmax) {
                if (kTrain) {
                    if (ncl == 0) th0 = zmax;
                    else if (ncl == 1) th1 = zmax;
                    else if (ncl == 2) th2 = zmax;
                    else if (ncl < 7) reinterpret_cast<float *>(P.hdr)[8 * pix + 1 + ncl] = zmax;
                    else P.thr[(size_t)ncl * P.W * P.H + pix] = zmax;
                }
                ++ncl;
                close_layer();  // rasterizer.py:168-196
                if (layers >= P.k_max) { stopped = true; ++discarded; return; }
            }
            if (v.w >= 0.f) {
                const float w = v.w;
                if (kCons) {
                    if (Wg == 0.f) z0 = v.vz;
                    const float dz = v.vz - z0;
                    Zs += w * dz;
                    Z2s += w * dz * dz;
                }
                Wg += (AccT)w;
                C0 += (AccT)(w * v.c0); C1 += (AccT)(w * v.c1); C2 += (AccT)(w * v.c2);
                if (!kTrain) { Zg += w * v.vz; Z2g += w * v.vz * v.vz; }
                ++members;
                if (v.ze > zmax) zmax = v.ze;
                if (kExtras && P.pair_cover) atomicAdd(&sm.ncov[v.slot], 1);
            }
        });
    }
    double lsum = 0.0;
    if (live) {
        if (Wg > 0) close_layer();
        if (kTrain)
            for (int m = 0; m < layers; ++m) composite((float)lw[m], (float)lc0[m], (float)lc1[m], (float)lc2[m]);
        const float r0 = o0 + T * P.bg0, r1 = o1 + T * P.bg1, r2 = o2 + T * P.bg2;
        if (!kTrain || P.rgb) {
            P.rgb[3 * pix] = r0; P.rgb[3 * pix + 1] = r1; P.rgb[3 * pix + 2] = r2;
        }
        if (!kTrain) {
            P.alpha[pix] = 1.f - T;
            P.depth[pix] = dden > 0.f ? dnum / dden : 0.f;
            P.nlayers[pix] = layers;
        } else if (!P.target) {
            // deferred loss (ss_train_coefs finishes the layer coefficients
            // once the image-space gradient is known): raw layer sums
            P.hdr[2 * pix] = make_int4(ncl | (layers << 8), __float_as_int(th0), __float_as_int(th1), __float_as_int(th2));
            const size_t HW = (size_t)P.W * P.H;
            // the lo parts go to the third region of `coef` (after the float4
            // planes and the A_lo planes)
            float4 *raw_lo = reinterpret_cast<float4 *>(reinterpret_cast<float *>(P.coef) + (size_t)5 * P.k_max * HW);
            for (int m = 0; m < layers; ++m) {
                const float4 hi = make_float4((float)lw[m], (float)lc0[m], (float)lc1[m], (float)lc2[m]);
                P.coef[(size_t)m * HW + pix] = hi;
                raw_lo[(size_t)m * HW + pix] = make_float4((float)((double)lw[m] - hi.x), (float)((double)lc0[m] - hi.y),
                                                           (float)((double)lc1[m] - hi.z), (float)((double)lc2[m] - hi.w));
            }
            if (P.alpha) P.alpha[pix] = 1.f - T;
        } else {
            P.hdr[2 * pix] = make_int4(ncl | (layers << 8), __float_as_int(th0), __float_as_int(th1), __float_as_int(th2));
            // L1 loss and its image gradient (losses.py:100-104)
            const float d0 = r0 - P.target[3 * pix], d1 = r1 - P.target[3 * pix + 1], d2 = r2 - P.target[3 * pix + 2];
            lsum = (double)fabsf(d0) + (double)fabsf(d1) + (double)fabsf(d2);
            const float sg = P.inv_count;
            const float gc0 = d0 > 0.f ? sg : (d0 < 0.f ? -sg : 0.f);
            const float gc1 = d1 > 0.f ? sg : (d1 < 0.f ? -sg : 0.f);
            const float gc2 = d2 > 0.f ? sg : (d2 < 0.f ? -sg : 0.f);
            // suffix recursion over the layers (backward.py:201-238, no
            // consolidation, no coverage loss) in float64 like the reference:
            // per layer A and dL/dC_raw
            double tb[KL], av[KL];
            double tr = 1.0;
            for (int m = 0; m < layers; ++m) {
                av[m] = -expm1(-(double)lw[m]);
                tb[m] = tr;
                tr *= 1.0 - av[m];
            }
            double sf0 = P.bg0, sf1 = P.bg1, sf2 = P.bg2;
            const size_t HW = (size_t)P.W * P.H;
            for (int m = layers - 1; m >= 0; --m) {
                const double inv = 1.0 / (double)lw[m];
                const double ch0 = lc0[m] * inv, ch1 = lc1[m] * inv, ch2 = lc2[m] * inv;
                const double a = av[m];
                const double g_am = tb[m] * (gc0 * (ch0 - sf0) + gc1 * (ch1 - sf1) + gc2 * (ch2 - sf2));
                const double ta = tb[m] * a;
                const double gh0 = gc0 * ta, gh1 = gc1 * ta, gh2 = gc2 * ta;
                store_coef(P.coef, (size_t)m * HW + pix, (size_t)P.k_max * HW, g_am * (1.0 - a), gh0, gh1, gh2, inv,
                           ch0, ch1, ch2);
                sf0 = a * ch0 + (1.0 - a) * sf0;
                sf1 = a * ch1 + (1.0 - a) * sf1;
                sf2 = a * ch2 + (1.0 - a) * sf2;
            }
        }
    }
    if (kExtras && P.discarded) {
        unsigned d = discarded;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (lane == 0 && d) atomicAdd(P.discarded, (unsigned long long)d);
    }
    if (kTrain && P.target) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        if (lane == 0) atomicAdd(P.loss, lsum);
    }
#ifdef SS_CTA_TIMING
    __syncthreads();
    if (threadIdx.x == 0 && g_fwd_times) {
        unsigned long long *o = g_fwd_times + 3 * (size_t)blockIdx.x;
        o[0] = t_start; o[1] = ss_globaltimer(); o[2] = ss_smid();
    }
#endif
}

// Deferred-loss training step: turn the forward's raw layer sums (W, C) into
// the per-layer backward coefficients (A, dL/dC_raw) once the image-space
// gradients g_rgb (and g_alpha) are known -- the suffix recursion of
// backward.py:201-238 including the coverage term (g_alpha * prod(1 - a)).
__global__ void __launch_bounds__(256) train_coef_kernel(int HW, int k_max, const int4 *__restrict__ hdr, float4 *coef,
                                                         const float *__restrict__ g_rgb, const double *__restrict__ g64,
                                                         const float *__restrict__ g_alpha, float bg0, float bg1,
                                                         float bg2)
{
    const int pix = blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= HW) return;
    const int layers = hdr[2 * pix].x >> 8;
    if (layers == 0) return;
    double a[SS_KMAX_CAP], tb[SS_KMAX_CAP];
    float4 raw[SS_KMAX_CAP];
    double tr = 1.0;
    const float4 *raw_lo = reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(coef) + (size_t)5 * k_max * HW);
    double rw_[SS_KMAX_CAP];
    for (int m = 0; m < layers; ++m) {
        raw[m] = coef[(size_t)m * HW + pix];
        const float4 lo = raw_lo[(size_t)m * HW + pix];
        rw_[m] = (double)raw[m].x + lo.x;
        a[m] = -expm1(-rw_[m]);
        tb[m] = tr;
        tr *= 1.0 - a[m];
    }
    // the float64 image gradient when the loss kept it (ss_photometric_loss grad64)
    const double gc0 = g64 ? g64[3 * (size_t)pix] : (double)g_rgb[3 * (size_t)pix];
    const double gc1 = g64 ? g64[3 * (size_t)pix + 1] : (double)g_rgb[3 * (size_t)pix + 1];
    const double gc2 = g64 ? g64[3 * (size_t)pix + 2] : (double)g_rgb[3 * (size_t)pix + 2];
    const double ga = g_alpha ? (double)g_alpha[pix] : 0.0;
    double sf0 = bg0, sf1 = bg1, sf2 = bg2, q = 1.0;
    for (int m = layers - 1; m >= 0; --m) {
        const double inv = 1.0 / rw_[m];
        const float4 hi = coef[(size_t)m * HW + pix], lo = raw_lo[(size_t)m * HW + pix];
        const double ch0 = ((double)hi.y + lo.y) * inv, ch1 = ((double)hi.z + lo.z) * inv,
                     ch2 = ((double)hi.w + lo.w) * inv;
        const double g_am = tb[m] * (gc0 * (ch0 - sf0) + gc1 * (ch1 - sf1) + gc2 * (ch2 - sf2) + ga * q);
        const double ta = tb[m] * a[m];
        const double gh0 = gc0 * ta, gh1 = gc1 * ta, gh2 = gc2 * ta;
        store_coef(coef, (size_t)m * HW + pix, (size_t)k_max * HW, g_am * (1.0 - a[m]), gh0, gh1, gh2, inv, ch0, ch1,
                   ch2);
        sf0 = a[m] * ch0 + (1.0 - a[m]) * sf0;
        sf1 = a[m] * ch1 + (1.0 - a[m]) * sf1;
        sf2 = a[m] * ch2 + (1.0 - a[m]) * sf2;
        q *= 1.0 - a[m];
    }
}

// train_coef_kernel plus the consolidation penalty (backward.py:160-238 with
// cons_scale > 0, the float64 pixel pass of raster_bwd.cu): from the layer
// depth moments in zst it adds the penalty's weight term to A and rewrites
// zst in place as the per-layer (B, Q, z_bar, var) of the record gradient
//     g_w += B dz + Q (dz^2 - var),  g_vz = w (B + 2 Q dz),  dz = view_z - z_bar;
// the penalty value is block-reduced into cons_loss.
__global__ void __launch_bounds__(256) train_coef_cons_kernel(int HW, int k_max, const int4 *__restrict__ hdr, float4 *coef,
                                                              float4 *zst, const float *__restrict__ g_rgb,
                                                              const double *__restrict__ g64,
                                                              const float *__restrict__ g_alpha, float bg0,
                                                              float bg1, float bg2, double s, double *cons_loss)
{
    __shared__ double red[8];
    const int pix = blockIdx.x * blockDim.x + threadIdx.x;
    double cons_pix = 0.0;
    const int layers = pix < HW ? hdr[2 * pix].x >> 8 : 0;
    if (layers > 0) {
        double a[SS_KMAX_CAP], tb[SS_KMAX_CAP], zb[SS_KMAX_CAP], vr[SS_KMAX_CAP];
        double gw_c[SS_KMAX_CAP], gz_c[SS_KMAX_CAP], gv_c[SS_KMAX_CAP], wm[SS_KMAX_CAP];
        const float4 *raw_lo = reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(coef) + (size_t)5 * k_max * HW);
        double raw[SS_KMAX_CAP][4];  // float64 layer sums W, C (hi + lo)
        double tr = 1.0;
        for (int m = 0; m < layers; ++m) {
            const float4 hi = coef[(size_t)m * HW + pix], lo = raw_lo[(size_t)m * HW + pix];
            raw[m][0] = (double)hi.x + lo.x; raw[m][1] = (double)hi.y + lo.y;
            raw[m][2] = (double)hi.z + lo.z; raw[m][3] = (double)hi.w + lo.w;
            const float4 z = zst[(size_t)m * HW + pix];
            a[m] = -expm1(-raw[m][0]);
            tb[m] = tr;
            tr *= 1.0 - a[m];
            const double inv = 1.0 / raw[m][0];
            const double mz = (double)z.y * inv;
            zb[m] = (double)z.x + mz;
            vr[m] = (double)z.z * inv - mz * mz;
            wm[m] = tb[m] * a[m];
            gv_c[m] = vr[m] > 0.0 ? s * wm[m] * wm[m] : 0.0;
            gw_c[m] = gz_c[m] = 0.0;
        }
        double l_pix = 0.0;
        for (int i = 0; i < layers; ++i) {
            const double var = vr[i] > 0.0 ? vr[i] : 0.0;
            l_pix += wm[i] * wm[i] * var;
            gw_c[i] += s * 2.0 * wm[i] * var;
            for (int j = i + 1; j < layers; ++j) {
                const double dz = zb[i] - zb[j];
                const double adz = fabs(dz);
                l_pix += wm[i] * wm[j] * adz;
                gw_c[i] += s * wm[j] * adz;
                gw_c[j] += s * wm[i] * adz;
                const double sgn = dz > 0.0 ? 1.0 : (dz < 0.0 ? -1.0 : 0.0);
                gz_c[i] += s * wm[i] * wm[j] * sgn;
                gz_c[j] -= s * wm[i] * wm[j] * sgn;
            }
        }
        cons_pix = s * l_pix;
        // the float64 image gradient when the loss kept it (ss_photometric_loss grad64)
        const double gc0 = g64 ? g64[3 * (size_t)pix] : (double)g_rgb[3 * (size_t)pix];
        const double gc1 = g64 ? g64[3 * (size_t)pix + 1] : (double)g_rgb[3 * (size_t)pix + 1];
        const double gc2 = g64 ? g64[3 * (size_t)pix + 2] : (double)g_rgb[3 * (size_t)pix + 2];
        const double ga = g_alpha ? (double)g_alpha[pix] : 0.0;
        double sf0 = bg0, sf1 = bg1, sf2 = bg2, q = 1.0, rw = 0.0;
        for (int m = layers - 1; m >= 0; --m) {
            const double inv = 1.0 / raw[m][0];
            const double ch0 = raw[m][1] * inv, ch1 = raw[m][2] * inv, ch2 = raw[m][3] * inv;
            const double g_am =
                tb[m] * (gc0 * (ch0 - sf0) + gc1 * (ch1 - sf1) + gc2 * (ch2 - sf2) + ga * q + gw_c[m] - rw);
            const double ta = tb[m] * a[m];
            const double gh0 = gc0 * ta, gh1 = gc1 * ta, gh2 = gc2 * ta;
            store_coef(coef, (size_t)m * HW + pix, (size_t)k_max * HW, g_am * (1.0 - a[m]), gh0, gh1, gh2, inv, ch0,
                       ch1, ch2);
            zst[(size_t)m * HW + pix] = make_float4((float)(gz_c[m] * inv), (float)(gv_c[m] * inv), (float)zb[m],
                                                    (float)vr[m]);
            sf0 = a[m] * ch0 + (1.0 - a[m]) * sf0;
            sf1 = a[m] * ch1 + (1.0 - a[m]) * sf1;
            sf2 = a[m] * ch2 + (1.0 - a[m]) * sf2;
            q *= 1.0 - a[m];
            rw = gw_c[m] * a[m] + (1.0 - a[m]) * rw;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cons_pix += __shfl_xor_sync(0xffffffffu, cons_pix, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cons_pix;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
        if (t != 0.0) atomicAdd(cons_loss, t);
    }
}

template <bool kExtras, bool kTrain, bool kCons = false, bool kDeferred = false>
void launch(const FwdParams &P, int ntiles, int threads, cudaStream_t st) {
    const int wpc = threads / 32 < kFwdWarps ? threads / 32 : kFwdWarps;  // tile 8: 2 warps
    const int ctas_per_tile = threads / (32 * wpc);
    raster_fwd_kernel<kExtras, kTrain, kCons, kDeferred><<<ntiles * ctas_per_tile, 32 * wpc, 0, st>>>(P);
}

bool fill_common(FwdParams &P, int width, int height, int tile, const int32_t *tile_offsets,
                 const int32_t *pair_rec, const uint32_t *pair_rect, const float *records, const float *background,
                 int k_max) {
    if (width <= 0 || height <= 0 || tile < 8 || tile > 16 || (tile & 7) || k_max < 1 || k_max > SS_KMAX_CAP)
        return false;
    if (!tile_offsets || !background) return false;
    P = FwdParams{};
    P.W = width; P.H = height; P.tile = tile; P.ntx = (width + tile - 1) / tile; P.k_max = k_max;
    P.bg0 = background[0]; P.bg1 = background[1]; P.bg2 = background[2];
    P.offsets = tile_offsets; P.pair_rec = pair_rec;
    P.pair_rect = reinterpret_cast<const uint2 *>(pair_rect);
    P.records = reinterpret_cast<const SsRecord *>(records);
    return true;
}

}  // namespace

extern "C" int ss_raster_forward(int width, int height, int tile, const int32_t *tile_offsets,
                                 const int32_t *pair_rec, const uint32_t *pair_rect, const float *records, const float *background,
                                 int k_max, float *rgb, float *alpha, float *depth, int32_t *nlayers,
                                 int32_t *pair_cover, const SsStacks *stacks, unsigned long long *discarded,
                                 void *stream)
{
    FwdParams P;
    if (!fill_common(P, width, height, tile, tile_offsets, pair_rec, pair_rect, records, background, k_max)) return SS_ERR_INVALID;
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

static int train_forward(int width, int height, int tile, const int32_t *tile_offsets, const int32_t *pair_rec,
                         const uint32_t *pair_rect, const float *records, const float *background, int k_max,
                         const float *target, float *coef, float *thr, int32_t *pix_hdr, double *loss_sum, float *rgb,
                         float *alpha, const int32_t *tile_order, float *zstats, void *stream)
{
    FwdParams P;
    if (!fill_common(P, width, height, tile, tile_offsets, pair_rec, pair_rect, records, background, k_max)) return SS_ERR_INVALID;
    if (!coef || !thr || !pix_hdr) return SS_ERR_INVALID;
    if (target ? !loss_sum : !rgb) return SS_ERR_INVALID;  // fused L1 needs the loss sum, deferred mode the image
    P.alpha = alpha;
    P.tile_order = tile_order;
    P.target = target;
    P.thr = thr;
    P.hdr = reinterpret_cast<int4 *>(pix_hdr);
    P.inv_count = (float)(1.0 / (3.0 * (double)width * (double)height));
    P.coef = reinterpret_cast<float4 *>(coef);
    P.loss = loss_sum;
    P.rgb = rgb;
    P.zst = reinterpret_cast<float4 *>(zstats);
    const int ntiles = P.ntx * ((height + tile - 1) / tile);
    if (zstats) launch<false, true, true, true>(P, ntiles, tile * tile, (cudaStream_t)stream);
    else if (!target) launch<false, true, false, true>(P, ntiles, tile * tile, (cudaStream_t)stream);
    else launch<false, true>(P, ntiles, tile * tile, (cudaStream_t)stream);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_train_forward(int width, int height, int tile, const int32_t *tile_offsets,
                                const int32_t *pair_rec, const uint32_t *pair_rect, const float *records, const float *background,
                                int k_max, const float *target, float *coef, float *thr, int32_t *pix_hdr,
                                double *loss_sum, float *rgb, float *alpha, const int32_t *tile_order, void *stream)
{
    return train_forward(width, height, tile, tile_offsets, pair_rec, pair_rect, records, background, k_max, target,
                         coef, thr, pix_hdr, loss_sum, rgb, alpha, tile_order, nullptr, stream);
}

extern "C" int ss_train_forward_zstats(int width, int height, int tile, const int32_t *tile_offsets,
                                       const int32_t *pair_rec, const uint32_t *pair_rect, const float *records,
                                       const float *background, int k_max, float *coef, float *thr, int32_t *pix_hdr,
                                       float *rgb, float *alpha, const int32_t *tile_order, float *zstats, void *stream)
{
    if (!zstats) return SS_ERR_INVALID;
    return train_forward(width, height, tile, tile_offsets, pair_rec, pair_rect, records, background, k_max, nullptr,
                         coef, thr, pix_hdr, nullptr, rgb, alpha, tile_order, zstats, stream);
}

extern "C" int ss_train_coefs(int width, int height, int k_max, const int32_t *pix_hdr, float *coef,
                              const float *g_rgb, const double *g_rgb64, const float *g_alpha,
                              const float *background, void *stream)
{
    if (width <= 0 || height <= 0 || k_max < 1 || k_max > SS_KMAX_CAP || !pix_hdr || !coef || !g_rgb || !background)
        return SS_ERR_INVALID;
    const int HW = width * height;
    train_coef_kernel<<<(HW + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        HW, k_max, reinterpret_cast<const int4 *>(pix_hdr), reinterpret_cast<float4 *>(coef), g_rgb, g_rgb64, g_alpha,
        background[0], background[1], background[2]);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_train_coefs_cons(int width, int height, int k_max, const int32_t *pix_hdr, float *coef,
                                   float *zstats, const float *g_rgb, const double *g_rgb64, const float *g_alpha,
                                   const float *background, double cons_scale, double *cons_loss, void *stream)
{
    if (width <= 0 || height <= 0 || k_max < 1 || k_max > SS_KMAX_CAP || !pix_hdr || !coef || !zstats || !g_rgb ||
        !background || !cons_loss || !(cons_scale >= 0.0))
        return SS_ERR_INVALID;
    const int HW = width * height;
    train_coef_cons_kernel<<<(HW + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        HW, k_max, reinterpret_cast<const int4 *>(pix_hdr), reinterpret_cast<float4 *>(coef),
        reinterpret_cast<float4 *>(zstats), g_rgb, g_rgb64, g_alpha, background[0], background[1], background[2],
        cons_scale, cons_loss);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

// ---------------------------------------------------------------------------
// Diagnostic: every (pixel, in-rect record) of a view is tested with the fast
// coverage path (ss_cover) and the exact reference evaluation; counts[0] =
// evaluations, counts[1] = decisions that differ (must be 0), counts[2] =
// evaluations that took the exact fallback.
namespace {
__global__ void __launch_bounds__(256) cover_check_kernel(int W, int H, int tile, int ntx, const int32_t *offsets,
                                                          const int32_t *pair_rec, const uint2 *pair_rect,
                                                          const SsRecord *recs, unsigned long long *counts)
{
    __shared__ SsRecord wbuf_all[8][32];
    const int t = blockIdx.x;
    const WarpPix wp = warp_pixels(t, ntx, tile, W, H);
    unsigned long long n = 0, bad = 0, slow = 0;
    walk_tile(wp, offsets[t], offsets[t + 1], pair_rec, pair_rect, recs, wbuf_all[wp.wid],
              [&](const SsRecord &R, int, int) {
                  if (!in_rect(wp, R.r)) return;
                  ++n;
                  const float t1[3] = {R.a.x, R.a.y, R.a.z}, t2[3] = {R.a.w, R.b.x, R.b.y}, t4[3] = {R.b.z, R.b.w, R.c.x};
                  SsHit h;
                  const bool exact = ss_intersect(wp.x, wp.y, t1, t2, t4, h) && ss_rho2(R.c.y, R.c.z, R.c.w, h.u, h.v) < 9.0;
                  FastCov f;
                  fast_cov_setup(R.a, R.b, R.c, R.e.w, f);
                  float u, v, r2;
                  const int d = fast_cover(f, R.c.y, R.c.z, R.c.w, wp.x, wp.y, u, v, r2);
                  Cover c;
                  const bool cov = d >= 0 ? d == 1 : ss_cover(wp.x, wp.y, R, c);
                  bad += cov != exact;
                  slow += d < 0;
              });
    atomicAdd(&counts[0], n);
    atomicAdd(&counts[1], bad);
    atomicAdd(&counts[2], slow);
}
}  // namespace

extern "C" int ss_debug_cover_check(int width, int height, int tile, const int32_t *tile_offsets,
                                    const int32_t *pair_rec, const uint32_t *pair_rect, const float *records,
                                    unsigned long long *counts, void *stream)
{
    if (width <= 0 || height <= 0 || tile != 16 || !tile_offsets || !counts) return SS_ERR_INVALID;
    const int ntx = (width + tile - 1) / tile, nty = (height + tile - 1) / tile;
    cover_check_kernel<<<ntx * nty, 256, 0, (cudaStream_t)stream>>>(width, height, tile, ntx, tile_offsets, pair_rec,
                                                                    reinterpret_cast<const uint2 *>(pair_rect),
                                                                    reinterpret_cast<const SsRecord *>(records), counts);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
