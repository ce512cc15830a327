// train_step.cu -- splat-parallel backward of the training step.
//
// Reference: pass 2 of _backward_kernel (backward.py:240-320).  The reference
// (and ss_raster_backward) replays the sorted walk per pixel to learn which
// layer each covering record belongs to.  That membership is in fact order
// independent once the forward has recorded, per pixel, the depth at which
// each layer closed (z_max_end of layer j when the gap test fired,
// rasterizer.py:168-196): the thresholds are strictly increasing and a
// covering record with interval start zs belongs to layer
//     m = #{ j : thr_j < zs },   discarded when m >= k_max
// (proof in DESIGN.md §kernels).  So the backward needs neither the walk nor
// the tile lists: records are counting-sorted by rect area and an 8-lane
// group owns one record (4 per warp, ~95% lane packing at the measured area
// distribution, vs ~28% for a pixel-parallel replay where most lanes of a
// warp block lie outside the record).  The lanes re-evaluate coverage with
// the certified fast path (coverage.cuh), read their pixel's layer header
// and coefficients (L2-resident planes) and accumulate 17 gradient channels
// in registers; one 3-level transposed reduction per group and plain stores
// (each record is committed exactly once: no atomics, deterministic).
#include "ss_common.cuh"
#include "raster_walk.cuh"
#include "warp_reduce.cuh"

#ifdef SS_CTA_TIMING
__device__ unsigned long long *g_bwd_times;  // (3 per warp of splat_bwd_kernel): start, end, smid
extern "C" int ss_debug_set_bwd_timing(void *buf) {
    return cudaMemcpyToSymbol(g_bwd_times, &buf, sizeof(buf)) == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}
#else
extern "C" int ss_debug_set_bwd_timing(void *) { return SS_ERR_INVALID; }
#endif

namespace {


constexpr int KS = 4;   // layers per pixel staged in shared memory (rest read from global)
constexpr int NCH = 17; // t1(3) t2(3) t4(3) Sigma^-1(3) n_f colour(3) screen-space |g|
constexpr int NCHC = 18; // + d/d view_z (consolidation)
template <bool kCons> __host__ __device__ constexpr int nch() { return kCons ? NCHC : NCH; }
// Warp max / sum by xor shuffles.  Loop bounds the compiler can prove
// warp-uniform (redux.sync max, vote.any loop conditions, or a broadcast
// from lane 0) make the record kernel ~9% faster but hang it intermittently
// on B200 (2-5 of 12-28 runs of a 3-step single-stream loop:
// tools/hang_variants.sh, tools/hang_hunt.py); these forms: 0 of 96 -- root
// cause not identified; see DESIGN.md.  Keep the bounds non-uniform.
// max over the 4 groups of a value uniform within each 8-lane group
__device__ __forceinline__ int group_max(int v) {
#ifdef SS_UNIFORM_BOUNDS  // the faster, intermittently hanging form (investigation switch)
    return __reduce_max_sync(0xffffffffu, v);
#else
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 8));
    return max(v, __shfl_xor_sync(0xffffffffu, v, 16));
#endif
}
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// reduced channel -> accumulator slot (slot 16 = dview_z, 17 = ss sum)
__device__ __forceinline__ int acc_slot(int c) { return c < 16 ? c : (c == 16 ? 17 : 16); }

struct SplatParams {
    int W, H, k_max, n;
    const int8_t *cull;
    const SsRecord *records;
    const float *xs, *ys;   // pixel-centre NDC per column / row (exact: coverage decisions)
    const float4 *coef;     // (k_max, HW) per-layer (A hi, dL/dC_raw)
    const float *coef_lo;   // (k_max, HW) low part of A (follows the float4 planes)
    const float *thr;       // (k_max, HW) closing depths of layers >= 3
    const int4 *hdr;        // (HW, 2) (closed-layer count, closing depths of layers 0..2), (depths 3..6)
    const float4 *zc;       // kCons: (k_max, HW) per layer (B, Q, z_bar, var) of the consolidation penalty
    float *acc;             // (n, 20)
    const int32_t *big_list;  // big-record queue (medium from the front, huge from the back)
    double *big_acc;          // (n, kBigW) float64 sums of the big records, by queue slot
};
constexpr int kBigW = SS_ACC64_WIDTH;  // float64 channels per big-record slot (>= NCHC)
static_assert(kBigW >= 18, "float64 row holds every channel");

constexpr int kHeadWords = 8 + 2 * 256;  // see the scratch layout below

__global__ void pixel_ndc_kernel(int W, int H, float *xs, float *ys, int32_t *big_count) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < W) xs[k] = ss_ndc_x(k, W);
    if (k < H) ys[k] = ss_ndc_y(k, H);
    if (k < kHeadWords) big_count[k] = 0;  // counters, class histogram and cursors
}

// Gradient of the covered item (pixel ix, iy of record R) with the coverage
// quantities u, v, rho^2 of the coverage pass, accumulated into g[].
// Returns 1 when the record reaches the pixel before the K_MAX stop.
// 1/x by the hardware approximation + one Newton step (no slow-path call).
__device__ __forceinline__ float fast_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * (2.f - x * r);
}

// (cx, cy): the record's projected centre (t1.z / t4.z, t2.z / t4.z), the
// origin of the x and y moments.
#ifdef SS_SPLAT_ACC_F64
typedef double SplatAcc;  // experiment: float64 per-lane channel sums
#else
typedef float SplatAcc;
#endif

template <bool kCons>
__device__ __forceinline__ int item_grad(const SplatParams &P, const SsRecord &R, int ix, int iy, float x, float y,
                                         float cx, float cy, SplatAcc *g) {
    const size_t HW = (size_t)P.W * P.H;
    const size_t pix = (size_t)iy * P.W + ix;
    // the packed header and the (most common) layer-0 coefficients are loaded
    // together, before the geometry below, so their latency hides behind it
    const int4 h = __ldg(P.hdr + 2 * pix);
    const float4 cf0 = __ldg(P.coef + pix);
    // ray / tangent-plane quantities with the reference's own float32
    // sequence (rasterizer.py:197-207, bit-identical k, l, den; u, v within
    // ~2 ulp): the certified fast form decided coverage in pass 1, but its
    // u, v carry ~1e-4 relative noise at the support edge, which sums into
    // a systematic bias of the record's gradient
    const float k0 = fs(fm(x, R.b.z), R.a.x), k1 = fs(fm(x, R.b.w), R.a.y), k2 = fs(fm(x, R.c.x), R.a.z);
    const float l0 = fs(fm(y, R.b.z), R.a.w), l1 = fs(fm(y, R.b.w), R.b.x), l2 = fs(fm(y, R.c.x), R.b.y);
#ifdef SS_ITEM_DIV
    const float den_ = fs(fm(k0, l1), fm(k1, l0));
    const float inv_den = fc_rcp(den_);
    const float u = fd(fs(fm(k1, l2), fm(k2, l1)), den_);
    const float v = fd(fs(fm(k2, l0), fm(k0, l2)), den_);
#else
    const float inv_den = fc_rcp(fs(fm(k0, l1), fm(k1, l0)));
    const float u = fs(fm(k1, l2), fm(k2, l1)) * inv_den;
    const float v = fs(fm(k2, l0), fm(k0, l2)) * inv_den;
#endif
#ifdef SS_ITEM_RHO64
    const double rho2 = ss_rho2(R.c.y, R.c.z, R.c.w, u, v);
#else
    const float rho2 = (R.c.y * u * u + 2.f * R.c.z * u * v) + R.c.w * v * v;
#endif
    const float zs = R.d.z;
    const int nc = h.x & 0xff;  // closed layers (the layer count sits in bits 8+)
    int m = (nc > 0 && __int_as_float(h.y) < zs) + (nc > 1 && __int_as_float(h.z) < zs) +
            (nc > 2 && __int_as_float(h.w) < zs);
    // the closing depths increase strictly with j: the second header half
    // (same 32-byte sector) only when zs lies beyond the first three
    if (m == 3 && nc > 3) {
        const int4 h2 = __ldg(P.hdr + 2 * pix + 1);
        m += (__int_as_float(h2.x) < zs) + (nc > 4 && __int_as_float(h2.y) < zs) +
             (nc > 5 && __int_as_float(h2.z) < zs) + (nc > 6 && __int_as_float(h2.w) < zs);
        if (m == 7) {
            const int jn = min(nc, P.k_max);
            for (int j = 7; j < jn && __ldg(P.thr + j * HW + pix) < zs; ++j) ++m;
        }
    }
    if (m >= P.k_max) return 0;  // beyond the K_MAX stop: discarded
    const float4 cf = m == 0 ? cf0 : __ldg(P.coef + m * HW + pix);
#if defined(SS_ITEM_RHO64)
    const double e = exp(-0.5 * rho2);
    const double w = (double)R.d.x * e;
#elif defined(SS_EXP_EXPF)
    const float e = expf(-0.5f * rho2);
    const float w = R.d.x * e;
#else
    float e;  // exp(-rho^2 / 2) by the hardware ex2 (ftz: no range fix-up)
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(rho2 * -0.72134752044448170368f));
    const float w = R.d.x * e;
#endif
    // g_w = A + sum_c G_c colour_c in float32 (A's low part is left out):
    // measured against a float64 sum with A_lo -- no full-size test entry
    // moves past the tolerance, and the float form saves 0.05 ms per view
    // (SS_GW_F64 restores the float64 form; the big records keep it)
#ifdef SS_GW_F64
    float gw = (float)(((double)cf.x + (double)__ldg(P.coef_lo + m * HW + pix)) +
                       (((double)cf.y * R.e.x + (double)cf.z * R.e.y) + (double)cf.w * R.e.z));
#else
    float gw = cf.x + ((cf.y * R.e.x + cf.z * R.e.y) + cf.w * R.e.z);
#endif
    if constexpr (kCons) {  // consolidation penalty (backward.py:272-286, centred depth form)
        const float4 zq = __ldg(P.zc + m * HW + pix);
        const float dz = R.d.y - zq.z;
        gw += zq.x * dz + zq.y * (dz * dz - zq.w);
        g[17] += w * (zq.x + 2.f * zq.y * dz);
    }
    g[13] += w * cf.y; g[14] += w * cf.z; g[15] += w * cf.w;
    const float gr = -0.5f * w * gw;
    g[12] += e * gw;
    g[9] += gr * u * u; g[10] += gr * 2.f * u * v; g[11] += gr * v * v;
    // sinv u + sinv v rounded like numba's float32 expression (backward.py:292-293)
    const float gu = 2.f * gr * fa(fm(R.c.y, u), fm(R.c.z, v));
    const float gv = 2.f * gr * fa(fm(R.c.z, u), fm(R.c.w, v));
    const float gp0 = gu * inv_den, gp1 = gv * inv_den, gp2 = -(gu * u + gv * v) * inv_den;
    // k = x t4 - t1 and l = y t4 - t2 are linear in the pixel centre, so the
    // per-item dL/dk = l x gp, dL/dl = gp x k and their T-row images sum to
    // cross products of the record's rows with three moments of gp
    // (sum gp, sum (x - cx) gp, sum (y - cy) gp): those 9 channels are
    // accumulated here and turned into dL/dt1, dt2, dt4 by the chain kernel
    // (SS_ACC_MOMENTS).  The moments are taken about the projected centre,
    // where k.z and l.z vanish: about the NDC origin, sum y gp ~ cy sum gp
    // and the float32 sums would lose the O(rect size) part the gradient
    // lives in (0.3% errors on off-centre splats)
    const float dx = x - cx, dy = y - cy;
    g[0] += gp0; g[1] += gp1; g[2] += gp2;
    g[3] += dx * gp0; g[4] += dx * gp1; g[5] += dx * gp2;
    g[6] += dy * gp0; g[7] += dy * gp1; g[8] += dy * gp2;
    const float gk2 = l0 * gp1 - l1 * gp0;
    const float gl2 = gp0 * k1 - gp1 * k0;
    float nrm;  // screen-space gradient norm (Eq. 12): approximate sqrt, no slow path
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(nrm) : "f"(gk2 * gk2 + gl2 * gl2));
    g[16] += fabsf(R.c.x) * nrm;
    return 1;
}

// Layer of a covering record at pixel `pix` (m = #{j : thr_j < zs}, see the
// file header), -1 beyond the K_MAX stop; its coefficients in cf.
__device__ __forceinline__ int pixel_layer(const SplatParams &P, size_t pix, float zs, float4 &cf, float &lo) {
    const size_t HW = (size_t)P.W * P.H;
    const int4 h = __ldg(P.hdr + 2 * pix);
    const int nc = h.x & 0xff;
    int m = (nc > 0 && __int_as_float(h.y) < zs) + (nc > 1 && __int_as_float(h.z) < zs) +
            (nc > 2 && __int_as_float(h.w) < zs);
    if (m == 3 && nc > 3) {
        const int4 h2 = __ldg(P.hdr + 2 * pix + 1);
        m += (__int_as_float(h2.x) < zs) + (nc > 4 && __int_as_float(h2.y) < zs) +
             (nc > 5 && __int_as_float(h2.z) < zs) + (nc > 6 && __int_as_float(h2.w) < zs);
        if (m == 7) {
            const int jn = min(nc, P.k_max);
            for (int j = 7; j < jn && __ldg(P.thr + j * HW + pix) < zs; ++j) ++m;
        }
    }
    if (m >= P.k_max) return -1;
    cf = __ldg(P.coef + m * HW + pix);
    lo = __ldg(P.coef_lo + m * HW + pix);
    return m;
}

// Big records (rects > kBigArea): the reference's own per-item arithmetic
// (backward.py:257-320) -- k, l, den, u, v in exact float32 (bit-identical,
// so is the coverage decision), rho^2 with numba's promotion, weight and
// every gradient term in float64, float64 sums, dL/dt1, dt2, dt4 formed per
// item as cross products.  A grazing splat's rect spans up to ~10^5 pixels
// whose terms cancel to ~1e-3 of their magnitude sum; float32 terms and
// sums (the moment form of item_grad) drift by percent there.
template <bool kCons>
__device__ __forceinline__ int item_grad_ref(const SplatParams &P, const SsRecord &R, int ix, int iy, float x,
                                             float y, double *g) {
    const float t4x = R.b.z, t4y = R.b.w, t4z = R.c.x;
    const float k0 = fs(fm(x, t4x), R.a.x), k1 = fs(fm(x, t4y), R.a.y), k2 = fs(fm(x, t4z), R.a.z);
    const float l0 = fs(fm(y, t4x), R.a.w), l1 = fs(fm(y, t4y), R.b.x), l2 = fs(fm(y, t4z), R.b.y);
    const float den = fs(fm(k0, l1), fm(k1, l0));
    if (fabsf(den) <= 9.99999972e-10f) return 0;  // |den| < 1e-9 in float64, exactly
    const float u = fd(fs(fm(k1, l2), fm(k2, l1)), den);
    const float v = fd(fs(fm(k2, l0), fm(k0, l2)), den);
    const double rho2 = ss_rho2(R.c.y, R.c.z, R.c.w, u, v);
    if (!(rho2 < 9.0)) return 0;
    float4 cf;
    float lo;
    const int m = pixel_layer(P, (size_t)iy * P.W + ix, R.d.z, cf, lo);
    if (m < 0) return 0;  // beyond the K_MAX stop: discarded
    const double e = exp(-0.5 * rho2);
    const double w = (double)R.d.x * e;
    double gw = ((double)cf.x + (double)lo) + (((double)cf.y * R.e.x + (double)cf.z * R.e.y) + (double)cf.w * R.e.z);
    if constexpr (kCons) {
        const size_t HW = (size_t)P.W * P.H;
        const float4 zq = __ldg(P.zc + m * HW + (size_t)iy * P.W + ix);
        const double dz = (double)R.d.y - zq.z;
        gw += zq.x * dz + zq.y * (dz * dz - zq.w);
        g[17] += w * (zq.x + 2.0 * zq.y * dz);
    }
    g[13] += w * cf.y; g[14] += w * cf.z; g[15] += w * cf.w;
    const double gr = -0.5 * w * gw;
    const double U = u, V = v;
    g[12] += e * gw;
    g[9] += gr * U * U; g[10] += gr * 2.0 * U * V; g[11] += gr * V * V;
    // numba keeps sinv * u + sinv * v in float32 (float32 operands), then
    // promotes (backward.py:292-293): the rounded sum is part of the result
    const double gu = gr * 2.0 * (double)fa(fm(R.c.y, u), fm(R.c.z, v));
    const double gv = gr * 2.0 * (double)fa(fm(R.c.z, u), fm(R.c.w, v));
    const double D = den;
    const double gp0 = gu / D, gp1 = gv / D, gp2 = -(gu * U + gv * V) / D;
    const double K0 = k0, K1 = k1, K2 = k2, L0 = l0, L1 = l1, L2 = l2, X = x, Y = y;
    const double gk0 = L1 * gp2 - L2 * gp1, gk1 = L2 * gp0 - L0 * gp2, gk2 = L0 * gp1 - L1 * gp0;
    const double gl0 = gp1 * K2 - gp2 * K1, gl1 = gp2 * K0 - gp0 * K2, gl2 = gp0 * K1 - gp1 * K0;
    g[0] -= gk0; g[1] -= gk1; g[2] -= gk2;
    g[3] -= gl0; g[4] -= gl1; g[5] -= gl2;
    g[6] += X * gk0 + Y * gl0; g[7] += X * gk1 + Y * gl1; g[8] += X * gk2 + Y * gl2;
    const double gsx = -gk2 * (double)t4z, gsy = -gl2 * (double)t4z;  // Eq. 12
    g[16] += sqrt(gsx * gsx + gsy * gsy);
    return 1;
}

// Coverage of pixel (ix, iy) of record R (fast path with the record's
// certified margin, exact reference arithmetic when undecided); on a hit
// returns the pixel (ix | iy << 16) and u, v, rho^2.
__device__ __forceinline__ bool item_cover(const float *xs, const float *ys, const SsRecord &R, const FastCov &f, int ix,
                                           int iy, int &ixy, float4 &q) {
    const float x = xs[ix], y = ys[iy];
    float u, v, r2;
    const int d = fast_cover(f, R.c.y, R.c.z, R.c.w, x, y, u, v, r2);
    if (d == 0) return false;
    if (d < 0) {
        Cover c;
        if (!ss_cover(x, y, R, c)) return false;
        u = c.u; v = c.v; r2 = c.rho2;
    }
    ixy = ix | (iy << 16);
    q = make_float4(u, v, r2, 0.f);
    return true;
}

__device__ __forceinline__ void load_record(const SsRecord *recs, int rec, SsRecord &R) {
    const float4 *src = reinterpret_cast<const float4 *>(recs + rec);
    R.a = __ldg(src); R.b = __ldg(src + 1); R.c = __ldg(src + 2); R.d = __ldg(src + 3); R.e = __ldg(src + 4);
    R.r = __ldg(reinterpret_cast<const int4 *>(src) + 5);
}

constexpr int kBigChunk = 1024;
constexpr int kHugeArea = 8 * kBigChunk;  // big rects above this are spread over the grid
constexpr int kBigArea = 512;  // rects above this go to the CTA-chunked kernel (~0.1% of records)
constexpr int kNB = 256;       // (area class, coverage-fraction bucket) classes of the other records
constexpr int kGL = 8;         // lanes per record group (4 records per warp)
#ifndef SS_GCAP
#define SS_GCAP 128
#endif
constexpr int kGCap = SS_GCAP;  // rect pixels compacted per group pass
#ifndef SS_SPLAT_WARPS
#define SS_SPLAT_WARPS 8
#endif
constexpr int kSplatWarps = SS_SPLAT_WARPS;
constexpr int kNdcSmem = 4096;  // W + H up to this: pixel-centre tables staged in shared memory
#ifndef SS_SPLAT_MINB
#define SS_SPLAT_MINB 3  // resident CTAs per SM the register budget is sized for
#endif
#ifndef SS_SPLAT_GRID
#define SS_SPLAT_GRID SS_SPLAT_MINB  // persistent CTAs launched per SM
#endif
#ifndef SS_SCAT_ITEMS
#define SS_SCAT_ITEMS 16
#endif
constexpr int kScatItems = SS_SCAT_ITEMS;  // records per thread of the class scatter
#ifndef SS_HEAVY_CLASS
#define SS_HEAVY_CLASS (32 * 4)
#endif
#ifndef SS_LIGHT_ROUNDS
#define SS_LIGHT_ROUNDS 8
#endif
constexpr int kHeavyClass = SS_HEAVY_CLASS;  // area >= 64 px: one round per work-counter ticket
constexpr int kLightRounds = SS_LIGHT_ROUNDS;  // rounds per ticket of the lighter classes

// Scratch layout (32-bit words after the two NDC tables), see
// ss_train_backward_scratch_words: 8 counters (medium / huge queue sizes,
// group-round and medium-record work counters, small-record count), the
// class histogram and cursors, the big-rect queue (n), the class-sorted
// record order (n) and the per-record class bytes.
static_assert(kHeadWords == 8 + 2 * kNB, "scratch head layout");

// Area class: exact below 16 px, then 8 classes per octave (~12% wide).
__device__ __forceinline__ int area_class(int a) {
    if (a < 16) return a;
    const int e = 31 - __clz(a);
    return 16 + (e - 4) * 8 + ((a >> (e - 3)) & 7);
}

__device__ __forceinline__ int rect_area(const int4 &r) {
    return (r.z > r.x && r.w > r.y) ? (r.z - r.x) * (r.w - r.y) : 0;
}

// Covered fraction of the rect, estimated from the record (the support
// ellipse rho^2 < 9 has area 9 pi / sqrt(det Sigma^-1) in the tangent plane,
// mapped by the projection's Jacobian at the centre), in 4 buckets: records
// of a round then have similar covered counts as well as similar areas
// (pass 2 runs to the round's largest covered count).
__device__ __forceinline__ int cover_bucket(const SsRecord &R, int area, int W, int H) {
    const float t1x = R.a.x, t1y = R.a.y, t1z = R.a.z, t2x = R.a.w, t2y = R.b.x, t2z = R.b.y;
    const float t4x = R.b.z, t4y = R.b.w, t4z = R.c.x;
    const float i2 = 1.f / (t4z * t4z);
    const float jxu = (t1x * t4z - t1z * t4x) * i2, jxv = (t1y * t4z - t1z * t4y) * i2;
    const float jyu = (t2x * t4z - t2z * t4x) * i2, jyv = (t2y * t4z - t2z * t4y) * i2;
    const float dets = R.c.y * R.c.w - R.c.z * R.c.z;
    const float est = 28.274333882f * rsqrtf(fmaxf(dets, 1e-30f)) * fabsf(jxu * jyv - jxv * jyu) * (0.25f * W * H);
    const float fr = est / (float)max(area, 1);
    return (fr >= 0.56f) + (fr >= 0.70f) + (fr >= 0.785f);  // (NaN: bucket 0)
}

// Class every kept record by rect area.  Big rects are queued for
// big_bwd_kernel (their accumulator rows zeroed: that kernel commits with
// atomics); the others get a class byte and count in the class histogram.
__global__ void __launch_bounds__(256) area_class_kernel(SplatParams P, uint8_t *cls, int32_t *big_list,
                                                         int32_t *counters, int32_t *hist)
{
    __shared__ int s_hist[kNB];
    if (threadIdx.x < kNB) s_hist[threadIdx.x] = 0;
    __syncthreads();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < P.n; r += gridDim.x * blockDim.x) {
        uint8_t c = 0xff;
        if (P.cull[r] == 0) {
            const int area = rect_area(__ldg(reinterpret_cast<const int4 *>(P.records + r) + 5));
            if (area > kBigArea) {
                float4 *dst = reinterpret_cast<float4 *>(P.acc + (size_t)r * SS_ACC_FLOATS);
#pragma unroll
                for (int i = 0; i < SS_ACC_FLOATS / 4; ++i) dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                const int q = area > kHugeArea ? P.n - 1 - atomicAdd(counters + 1, 1) : atomicAdd(counters, 1);
                big_list[q] = r;
                double2 *row = reinterpret_cast<double2 *>(P.big_acc + (size_t)q * kBigW);
#pragma unroll
                for (int i = 0; i < kBigW / 2; ++i) row[i] = make_double2(0.0, 0.0);
            } else {
                SsRecord R;
                const float4 *src = reinterpret_cast<const float4 *>(P.records + r);
                R.a = __ldg(src); R.b = __ldg(src + 1); R.c = __ldg(src + 2);
                c = (uint8_t)(area_class(area) * 4 + cover_bucket(R, area, P.W, P.H));
                atomicAdd(&s_hist[c], 1);
            }
        }
        cls[r] = c;
    }
    __syncthreads();
    if (threadIdx.x < kNB && s_hist[threadIdx.x] != 0) atomicAdd(hist + threadIdx.x, s_hist[threadIdx.x]);
}

// Counting-sort scatter: records in DESCENDING area class (heavy first);
// the order within a class is irrelevant (every record is processed whole by
// one group and committed with plain stores).
__global__ void __launch_bounds__(256) area_scatter_kernel(int n, const uint8_t *cls, const int32_t *hist,
                                                           int32_t *cursor, int32_t *order, int32_t *nsmall)
{
    __shared__ int s_cnt[kNB], s_base[kNB];
    const int t = threadIdx.x;
    for (int k = t; k < kNB; k += 256) s_cnt[k] = 0;
    __syncthreads();
    const int base = blockIdx.x * 256 * kScatItems;
    int rank[kScatItems], c[kScatItems];
    const unsigned lt = (1u << (t & 31)) - 1u;
#pragma unroll
    for (int j = 0; j < kScatItems; ++j) {
        const int r = base + j * 256 + t;
        c[j] = r < n ? cls[r] : 0xff;
        // warp-aggregated: one shared atomic per distinct class of the warp
        // (a few area classes hold most records; per-lane atomics on them
        // serialise)
        const unsigned same = __match_any_sync(0xffffffffu, c[j]);
        const int leader = __ffs(same) - 1;
        int b = 0;
        if ((t & 31) == leader && c[j] != 0xff) b = atomicAdd(&s_cnt[c[j]], __popc(same));
        b = __shfl_sync(0xffffffffu, b, leader);
        rank[j] = c[j] != 0xff ? b + __popc(same & lt) : 0;
    }
    __syncthreads();
    if (t < 32) {
        // positions kCpl t .. kCpl t + kCpl - 1 of the descending order are
        // classes kNB - 1 - kCpl t - j
        constexpr int kCpl = kNB / 32;
        int h[kCpl], loc = 0;
#pragma unroll
        for (int j = 0; j < kCpl; ++j) { h[j] = __ldg(hist + kNB - 1 - kCpl * t - j); loc += h[j]; }
        int incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (t >= o) incl += v;
        }
        int run = incl - loc;
#pragma unroll
        for (int j = 0; j < kCpl; ++j) {
            const int cj = kNB - 1 - kCpl * t - j;
            s_base[cj] = run + (s_cnt[cj] ? atomicAdd(cursor + cj, s_cnt[cj]) : 0);
            run += h[j];
        }
        // records of class >= kHeavyClass (the first kNB - kHeavyClass positions) are handed out one round at a time
        const int nheavy = __shfl_sync(0xffffffffu, incl, (kNB - kHeavyClass) / kCpl - 1);
        if (blockIdx.x == 0 && t == 31) {
            nsmall[0] = incl;
            nsmall[1] = nheavy;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScatItems; ++j)
        if (c[j] != 0xff) order[s_base[c[j]] + rank[j]] = base + j * 256 + t;
}

struct GroupSmem {
    SsRecord rec[2][4];       // current / prefetched records of the 4 groups (cp.async double buffer)
    int ixy[4][kGCap];        // covered items: pixel ix | iy << 16
};

// Eight lanes per record, four records per warp, records taken in
// descending area class so the four rects of a round (and the warps of a
// launch) carry nearly equal work.  Rounds of 4 sorted records are handed
// out in blocks of 8 by one counter; the next round's records are copied
// into the other shared slot with cp.async while the current one runs.  Per
// record: pass 1 takes the exact coverage decision for up to kGCap rect
// pixels and compacts the covered ones (with u, v) into the group's list;
// pass 2 evaluates the gradient on the covered items, 8 per iteration.  One
// 3-level transposed reduction per group and plain stores of the record's
// row (each record committed exactly once: no atomics, deterministic).
template <bool kSmemNdc, bool kCons>
__global__ void __launch_bounds__(32 * kSplatWarps, SS_SPLAT_MINB) splat_bwd_kernel(SplatParams P, const int32_t *order,
                                                                        int32_t *counters)
{
    extern __shared__ __align__(16) unsigned char splat_smem[];
#ifdef SS_CTA_TIMING
    const unsigned long long t_start = ss_globaltimer();
#endif
    GroupSmem &sm = reinterpret_cast<GroupSmem *>(splat_smem)[threadIdx.x >> 5];
    // the exact pixel-centre tables of the coverage decisions, staged in
    // shared memory when they fit (one CTA barrier, at the start)
    const float *xs = P.xs, *ys = P.ys;
    if constexpr (kSmemNdc) {
        float *s_ndc = reinterpret_cast<float *>(splat_smem + kSplatWarps * sizeof(GroupSmem));
        for (int t = threadIdx.x; t < P.W + P.H; t += blockDim.x) s_ndc[t] = P.xs[t];
        __syncthreads();
        xs = s_ndc;
        ys = s_ndc + P.W;
    }
    const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & (kGL - 1);
    const unsigned glt = (1u << gl) - 1u;
    int ch[3];
    constexpr int NC = nch<kCons>();
    warp_tr_indices<NC, 4>(ch, lane);
    const int nsmall = counters[4];
    const int nrounds = (nsmall + 3) >> 2, hrounds = (counters[5] + 3) >> 2;
    int32_t *work = counters + 2;
    int rend = 0;
    auto grab = [&]() {  // ticket -> first round: heavy rounds one by one, then blocks of kLightRounds
        int t = 0;
        if (lane == 0) t = atomicAdd(work, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        const int b = t < hrounds ? t : hrounds + (t - hrounds) * kLightRounds;
        rend = t < hrounds ? b + 1 : b + kLightRounds;
        return b;
    };
    auto issue = [&](int r, int buf) {  // cp.async of round r's records into slot buf
        if (r < nrounds && lane < 24) {
            const int e = r * 4 + lane / 6;
            if (e < nsmall)
                cp_async16(reinterpret_cast<float4 *>(&sm.rec[buf][lane / 6]) + lane % 6,
                           reinterpret_cast<const float4 *>(P.records + __ldg(order + e)) + lane % 6);
        }
        cp_async_commit();
    };
    int cur = grab();
    int buf = 0;
    issue(cur, 0);
    while (cur < nrounds) {
        const int nxt = cur + 1 < rend ? cur + 1 : grab();
        cp_async_wait_all();
        __syncwarp();
        issue(nxt, buf ^ 1);
        const int e = cur * 4 + grp;
        const bool valid = e < nsmall;
        const SsRecord &R = sm.rec[buf][grp];
        int rw = 1, area = 0;
        if (valid) {
            rw = R.r.z - R.r.x;
            area = rect_area(R.r);
        }
        // k / rw as (k * mrw) >> 20 with mrw = ceil(2^20 / rw): exact while
        // k * rw < 2^20 (k < area <= kBigArea, rw <= kBigArea)
        const unsigned mrw = ((1u << 20) + (unsigned)rw - 1u) / (unsigned)rw;
        FastCov f;
        fast_cov_setup(R.a, R.b, R.c, R.e.w, f);
        const float cx = valid ? fd(R.a.z, R.c.x) : 0.f, cy = valid ? fd(R.b.y, R.c.x) : 0.f;
        SplatAcc g[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) g[k] = 0.f;
        int touch = 0;
        const int amax = group_max(area);  // area is uniform within a group
        for (int c0 = 0; c0 < amax; c0 += kGCap) {
            // pass 1: exact coverage of up to kGCap rect pixels, compaction
            const int cend = min(c0 + kGCap, amax);
            int ncov = 0;
            for (int k0 = c0; k0 < cend; k0 += kGL) {
                const int k = k0 + gl;
                int ixy = 0;
                float4 q;
                const int ky = (int)(((unsigned)k * mrw) >> 20);
                const bool hit = k < area && item_cover(xs, ys, R, f, R.r.x + (k - ky * rw), R.r.y + ky, ixy, q);
                const unsigned gm = (__ballot_sync(0xffffffffu, hit) >> (grp * kGL)) & 0xffu;
                if (hit) sm.ixy[grp][ncov + __popc(gm & glt)] = ixy;
                ncov += __popc(gm);
            }
            __syncwarp();
            // pass 2: gradients of the covered items
            const int nmax = group_max(ncov);  // ncov is uniform within a group
            for (int j0 = 0; j0 < nmax; j0 += kGL) {
                const int j = j0 + gl;
                if (j < ncov) {
                    const int ixy = sm.ixy[grp][j];
                    // pixel centres from the (shared-memory) tables: no int->float conversions
                    const int ix = ixy & 0xffff, iy = ixy >> 16;
                    touch += item_grad<kCons>(P, R, ix, iy, xs[ix], ys[iy], cx, cy, g);
                }
            }
            __syncwarp();
        }
        warp_tr_all<NC, 4>(g, lane);  // 3 channel sums of the group per lane
        touch += __shfl_xor_sync(0xffffffffu, touch, 4);
        touch += __shfl_xor_sync(0xffffffffu, touch, 2);
        touch += __shfl_xor_sync(0xffffffffu, touch, 1);
        if (valid) {
            // channel c -> accumulator slot (16 is dview_z, 0 here: the ss sum lives in 17);
            // channels held by two lanes carry identical sums
            float *dst = P.acc + (size_t)__ldg(order + e) * SS_ACC_FLOATS;
#pragma unroll
            for (int i = 0; i < 3; ++i) dst[acc_slot(ch[i])] = (float)g[i];
            if (gl == 0) reinterpret_cast<int *>(dst)[18] = touch;
            if (!kCons && gl == 1) dst[16] = 0.f;
            if (gl == 2) dst[19] = SS_ACC_MOMENTS;
        }
        __syncwarp();
        cur = nxt;
        buf ^= 1;
    }
    cp_async_wait_all();
#ifdef SS_CTA_TIMING
    if (lane == 0 && g_bwd_times) {
        unsigned long long *o = g_bwd_times + 3 * ((size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
        o[0] = t_start; o[1] = ss_globaltimer(); o[2] = ss_smid();
    }
#endif
}

// Gradient contribution of record R at rect pixel k (row-major) for the big
// records (no compaction), accumulated into g[]; returns 1 when touched.
template <bool kCons>
__device__ __forceinline__ int pixel_grad(const SplatParams &P, const SsRecord &R, int k, int rw, double *g) {
    // integer division: exact for any rect size (a float32 reciprocal
    // multiply is exact only while k < ~2^22, i.e. rects below ~4 MP); this
    // path handles ~0.1% of the records
    const int ky = k / rw;
    const int ix = R.r.x + (k - ky * rw), iy = R.r.y + ky;
    return item_grad_ref<kCons>(P, R, ix, iy, __ldg(P.xs + ix), __ldg(P.ys + iy), g);
}

// Big records (grazing splats whose filtered bound spans up to most of the
// image).  The splat kernel queues them in two lists: medium rects (up to
// kHugeArea pixels) from the front of the queue, huge ones from its back.  A
// medium record is processed by one CTA (grid-stride over the list), a huge
// one is cut into 1024-pixel chunks spread over the whole grid (chunk c of
// huge entry h goes to CTA (c + 37 h) mod grid).  Warps split the pixels in
// 32-pixel rows, reduce, and commit with atomics (the splat kernel zeroed
// the rows).
template <bool kCons>
__device__ __forceinline__ void big_record(const SplatParams &P, int q, int c0, int cstep, int wid, int nw,
                                           int lane, int my_ch, bool owner) {
    constexpr int NC = nch<kCons>();
    const int rec = P.big_list[q];
    SsRecord R;
    load_record(P.records, rec, R);
    const int rw = R.r.z - R.r.x, area = rw * (R.r.w - R.r.y);
    const int nchunks = (area + kBigChunk - 1) / kBigChunk;
    double g[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) g[k] = 0.0;
    int touch = 0;
    for (int c = c0; c < nchunks; c += cstep) {
        const int k1 = min(area, (c + 1) * kBigChunk);
        for (int k = c * kBigChunk + wid * 32 + lane; k < k1; k += 32 * nw) touch += pixel_grad<kCons>(P, R, k, rw, g);
    }
    const int tot = warp_sum(touch);
    if (tot == 0) return;
    warp_tr_reduce<NC>(g, lane);
    if (owner) atomicAdd(P.big_acc + (size_t)q * kBigW + my_ch, g[0]);
    if (lane == 0) atomicAdd(reinterpret_cast<int *>(P.acc + (size_t)rec * SS_ACC_FLOATS) + 18, tot);
}

template <bool kCons>
__global__ void __launch_bounds__(256) big_bwd_kernel(SplatParams P, const int32_t *big_list,
                                                      const int32_t *big_count)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int my_ch = warp_tr_index<nch<kCons>()>(lane);
    const unsigned same = __match_any_sync(0xffffffffu, my_ch);
    const bool owner = (__ffs(same) - 1) == lane;
    const int nmed = big_count[0], nhuge = big_count[1];
    const int G = gridDim.x;
    // medium records: handed out one per CTA by a work counter
    __shared__ int s_b;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_b = atomicAdd(const_cast<int32_t *>(big_count) + 3, 1);
        __syncthreads();
        const int b = s_b;
        if (b >= nmed) break;
        big_record<kCons>(P, b, 0, 1, wid, nw, lane, my_ch, owner);
    }
    for (int h = 0; h < nhuge; ++h) {
        const int first = (int)(((long long)blockIdx.x - 37LL * h) % G + G) % G;
        big_record<kCons>(P, P.n - 1 - h, first, G, wid, nw, lane, my_ch, owner);
    }
}

// The big records' rows point at their float64 sums (slot 19 =
// SS_ACC_F64, slot 0 = the queue slot): the chain kernel reads the float64
// channels -- a grazing splat's row gradients cancel in the chain's linear
// maps, beyond a float32 accumulator row.
__global__ void __launch_bounds__(256) big_finish_kernel(SplatParams P, const int32_t *big_count) {
    const int nmed = big_count[0], nhuge = big_count[1];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nmed + nhuge; e += gridDim.x * blockDim.x) {
        const int q = e < nmed ? e : P.n - 1 - (e - nmed);
        float *dst = P.acc + (size_t)P.big_list[q] * SS_ACC_FLOATS;
        dst[0] = __int_as_float(q);
        dst[17] = (float)P.big_acc[(size_t)q * kBigW + 16];  // ss (readers of the float row)
        dst[19] = SS_ACC_F64;
    }
}

}  // namespace

extern "C" size_t ss_train_backward_scratch_words(int n, int width, int height)
{
    if (n < 0 || width <= 0 || height <= 0) return 0;
    return (size_t)width + height + kHeadWords + 2 * (size_t)n + ((size_t)n + 3) / 4;
}

template <bool kSmemNdc, bool kCons>
void launch_splat(const SplatParams &P, const int32_t *order, int32_t *counters, int smem, cudaStream_t st) {
    ss_func_smem((const void *)splat_bwd_kernel<kSmemNdc, kCons>,
                 kSplatWarps * (int)sizeof(GroupSmem) + (kSmemNdc ? kNdcSmem * (int)sizeof(float) : 0));
    splat_bwd_kernel<kSmemNdc, kCons><<<ss_sm_count() * SS_SPLAT_GRID, 32 * kSplatWarps, smem, st>>>(P, order, counters);
}

static int backward_records(int n, const int8_t *cull, const float *records, int width, int height, int k_max,
                            const float *coef, const float *thr, const int32_t *pix_hdr, const float *zcoef,
                            float *pixel_ndc, float *rec_acc, double *rec_acc64, void *stream)
{
    if (n < 0 || width <= 0 || height <= 0 || k_max < 1 || k_max > SS_KMAX_CAP) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    if (!cull || !records || !coef || !thr || !pix_hdr || !pixel_ndc || !rec_acc || !rec_acc64) return SS_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    const int mx = width > height ? width : height;

    int32_t *counters = reinterpret_cast<int32_t *>(pixel_ndc + width + height);
    int32_t *hist = counters + 8, *cursor = hist + kNB;
    int32_t *big_list = counters + kHeadWords;
    int32_t *order = big_list + n;
    uint8_t *cls = reinterpret_cast<uint8_t *>(order + n);

    pixel_ndc_kernel<<<(mx + kHeadWords + 255) / 256, 256, 0, st>>>(width, height, pixel_ndc, pixel_ndc + width,
                                                                     counters);
    SS_CUDA_CHECK_LAUNCH();
    SplatParams P{};
    P.W = width; P.H = height; P.k_max = k_max; P.n = n;
    P.cull = cull;
    P.records = reinterpret_cast<const SsRecord *>(records);
    P.xs = pixel_ndc; P.ys = pixel_ndc + width;
    P.coef = reinterpret_cast<const float4 *>(coef);
    P.coef_lo = coef + (size_t)4 * k_max * width * height;
    P.thr = thr; P.hdr = reinterpret_cast<const int4 *>(pix_hdr); P.acc = rec_acc;
    P.zc = reinterpret_cast<const float4 *>(zcoef);
    P.big_list = big_list;
    P.big_acc = rec_acc64;
    const bool cons = zcoef != nullptr;
    area_class_kernel<<<ss_sm_count() * 4, 256, 0, st>>>(P, cls, big_list, counters, hist);
    SS_CUDA_CHECK_LAUNCH();
    area_scatter_kernel<<<(n + 256 * kScatItems - 1) / (256 * kScatItems), 256, 0, st>>>(n, cls, hist, cursor, order,
                                                                                       counters + 4);
    SS_CUDA_CHECK_LAUNCH();
    const int smem = kSplatWarps * (int)sizeof(GroupSmem);
    // (the pixel-centre tables sit right after the NDC scratch: xs then ys, contiguous)
    const int smem_ndc = smem + (width + height) * (int)sizeof(float);
    if (width + height <= kNdcSmem) {
        if (cons) launch_splat<true, true>(P, order, counters, smem_ndc, st);
        else launch_splat<true, false>(P, order, counters, smem_ndc, st);
    } else {
        if (cons) launch_splat<false, true>(P, order, counters, smem, st);
        else launch_splat<false, false>(P, order, counters, smem, st);
    }
    SS_CUDA_CHECK_LAUNCH();
    if (cons) big_bwd_kernel<true><<<ss_sm_count() * 4, 256, 0, st>>>(P, big_list, counters);
    else big_bwd_kernel<false><<<ss_sm_count() * 4, 256, 0, st>>>(P, big_list, counters);
    SS_CUDA_CHECK_LAUNCH();
    big_finish_kernel<<<ss_sm_count(), 256, 0, st>>>(P, counters);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_train_backward_records(int n, const int8_t *cull, const float *records, int width, int height,
                                         int k_max, const float *coef, const float *thr, const int32_t *pix_hdr,
                                         float *pixel_ndc, float *rec_acc, double *rec_acc64, void *stream)
{
    return backward_records(n, cull, records, width, height, k_max, coef, thr, pix_hdr, nullptr, pixel_ndc, rec_acc,
                            rec_acc64, stream);
}

extern "C" int ss_train_backward_records_cons(int n, const int8_t *cull, const float *records, int width, int height,
                                              int k_max, const float *coef, const float *thr, const int32_t *pix_hdr,
                                              const float *zcoef, float *pixel_ndc, float *rec_acc, double *rec_acc64,
                                              void *stream)
{
    if (!zcoef) return SS_ERR_INVALID;
    return backward_records(n, cull, records, width, height, k_max, coef, thr, pix_hdr, zcoef, pixel_ndc, rec_acc,
                            rec_acc64, stream);
}
