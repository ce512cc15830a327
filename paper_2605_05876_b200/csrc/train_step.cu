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
// (proof in DESIGN.md §kernels).  So the backward needs no walk: one WARP
// owns one (record, tile) pair and its lanes sweep the record's rect inside
// the tile (dense: ~90% lane utilisation for the typical 5x5-10x10 px rects,
// vs ~28% for a pixel-parallel replay where most lanes of a warp block lie
// outside the record).  Each lane re-evaluates coverage with the forward's
// exact-decision fast path, looks its layer up in the tile's shared-memory
// threshold table and accumulates 17 gradient channels in registers; one
// transposed warp reduction and one set of atomics per (record, tile).
#include "ss_common.cuh"
#include "raster_walk.cuh"
#include "warp_reduce.cuh"

namespace {

constexpr int KS = 4;   // layers per pixel staged in shared memory (rest read from global)
constexpr int NCH = 17; // t1(3) t2(3) t4(3) Sigma^-1(3) n_f colour(3) screen-space |g|

struct SplatParams {
    int W, H, tile, ntx, k_max;
    const int32_t *offsets;
    const int32_t *pair_rec;
    const SsRecord *records;
    const float4 *coef;     // (k_max, HW) per-layer (A, dL/dC_raw)
    const float *thr;       // (k_max, HW) layer closing depths
    const int32_t *ncl;     // (HW) number of closed layers (thresholds)
    float *acc;             // (n, 20)
};

__global__ void __launch_bounds__(256, 2) splat_bwd_kernel(SplatParams P)
{
    __shared__ float s_thr[KS][256];
    __shared__ float4 s_cf[KS][256];
    __shared__ int s_ncl[256];
    __shared__ float s_x[32], s_y[32];
    const int t = blockIdx.x;
    const int tx = t % P.ntx, ty = t / P.ntx;
    const int x0 = tx * P.tile, y0 = ty * P.tile;
    const int tw = min(P.tile, P.W - x0), th = min(P.tile, P.H - y0);
    const size_t HW = (size_t)P.W * P.H;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // stage the tile's per-pixel layer tables
    for (int k = threadIdx.x; k < P.tile * P.tile; k += blockDim.x) {
        const int lx = k % P.tile, ly = k / P.tile;
        int nc = 0;
        if (lx < tw && ly < th) {
            const size_t pix = (size_t)(y0 + ly) * P.W + (x0 + lx);
            nc = P.ncl[pix];
            for (int m = 0; m < KS; ++m) {
                s_thr[m][k] = m < nc ? P.thr[m * HW + pix] : 0.f;
                s_cf[m][k] = P.coef[m * HW + pix];
            }
        }
        s_ncl[k] = nc;
    }
    if (threadIdx.x < P.tile) s_x[threadIdx.x] = ss_ndc_x(x0 + threadIdx.x, P.W);
    if (threadIdx.x >= 32 && threadIdx.x < 32 + P.tile) s_y[threadIdx.x - 32] = ss_ndc_y(y0 + threadIdx.x - 32, P.H);
    __syncthreads();

    const int my_ch = warp_tr_index<NCH>(lane);
    const unsigned same = __match_any_sync(0xffffffffu, my_ch);
    const bool owner = (__ffs(same) - 1) == lane;

    // one warp per (record, tile) pair; lanes sweep the record's rect inside the tile
    const int p0 = P.offsets[t], p1 = P.offsets[t + 1];
    for (int p = p0 + wid; p < p1; p += nw) {
        const int rec = __ldg(P.pair_rec + p);
        const float4 *src = reinterpret_cast<const float4 *>(P.records + rec);
        SsRecord R;
        R.a = __ldg(src); R.b = __ldg(src + 1); R.c = __ldg(src + 2); R.d = __ldg(src + 3); R.e = __ldg(src + 4);
        R.r = __ldg(reinterpret_cast<const int4 *>(src) + 5);
        const int ix0 = max(R.r.x, x0), ix1 = min(R.r.z, x0 + tw);
        const int iy0 = max(R.r.y, y0), iy1 = min(R.r.w, y0 + th);
        const int rw = ix1 - ix0, area = rw * (iy1 - iy0);
        const float inv_rw = 1.f / (float)max(rw, 1);  // k < 256: float division is exact after floor
        const float zs = R.d.z, t4z = fabsf(R.c.x);
        float g[NCH];
#pragma unroll
        for (int k = 0; k < NCH; ++k) g[k] = 0.f;
        int touch = 0;
        for (int k = lane; k < area; k += 32) {
            const int ky = (int)(((float)k + 0.5f) * inv_rw);
            const int iy = iy0 + ky, ix = ix0 + (k - ky * rw);
            const float x = s_x[ix - x0], y = s_y[iy - y0];
            Cover c;
            if (!ss_cover(x, y, R, c)) continue;
            const int lp = (iy - y0) * P.tile + (ix - x0);
            const int nc = s_ncl[lp];
            int m = 0;
            for (int j = 0; j < nc; ++j) {
                const float tj = j < KS ? s_thr[j][lp] : P.thr[j * HW + (size_t)iy * P.W + ix];
                m += tj < zs;
            }
            if (m >= P.k_max) continue;  // beyond the K_MAX stop: discarded
            const float4 cf = m < KS ? s_cf[m][lp] : P.coef[m * HW + (size_t)iy * P.W + ix];
            ++touch;
            const float e = __expf(-0.5f * c.rho2);
            const float w = R.d.x * e;
            const float gw = cf.x + cf.y * R.e.x + cf.z * R.e.y + cf.w * R.e.z;
            g[13] += w * cf.y; g[14] += w * cf.z; g[15] += w * cf.w;
            const float gr = -0.5f * w * gw;
            g[12] += e * gw;
            const float u = c.u, v = c.v;
            g[9] += gr * u * u; g[10] += gr * 2.f * u * v; g[11] += gr * v * v;
            const float gu = 2.f * gr * (R.c.y * u + R.c.z * v);
            const float gv = 2.f * gr * (R.c.z * u + R.c.w * v);
            const float gp0 = gu * c.inv_den, gp1 = gv * c.inv_den, gp2 = -(gu * u + gv * v) * c.inv_den;
            const float gk0 = c.l1 * gp2 - c.l2 * gp1;
            const float gk1 = c.l2 * gp0 - c.l0 * gp2;
            const float gk2 = c.l0 * gp1 - c.l1 * gp0;
            const float gl0 = gp1 * c.k2 - gp2 * c.k1;
            const float gl1 = gp2 * c.k0 - gp0 * c.k2;
            const float gl2 = gp0 * c.k1 - gp1 * c.k0;
            g[0] -= gk0; g[1] -= gk1; g[2] -= gk2;
            g[3] -= gl0; g[4] -= gl1; g[5] -= gl2;
            g[6] += x * gk0 + y * gl0; g[7] += x * gk1 + y * gl1; g[8] += x * gk2 + y * gl2;
            g[16] += t4z * sqrtf(gk2 * gk2 + gl2 * gl2);
        }
        const int tot = __reduce_add_sync(0xffffffffu, touch);
        if (tot == 0) continue;
        warp_tr_reduce<NCH>(g, lane);
        float *dst = P.acc + (size_t)rec * SS_ACC_FLOATS;
        // channel c -> accumulator slot (16 is dview_z, unused: the ss sum lives in 17)
        if (owner) atomicAdd(dst + (my_ch == 16 ? 17 : my_ch), g[0]);
        if (lane == 0) atomicAdd(reinterpret_cast<int *>(dst + 18), tot);
    }
}

}  // namespace

extern "C" int ss_train_backward(int width, int height, int tile, const int32_t *tile_offsets,
                                 const int32_t *pair_rec, const uint32_t *pair_rect, const float *records, int k_max,
                                 const float *coef, const float *thr, const int32_t *ncl, float *rec_acc, void *stream)
{
    (void)pair_rect;
    if (width <= 0 || height <= 0 || tile != 16 || k_max < 1 || k_max > SS_KMAX_CAP) return SS_ERR_INVALID;
    if (!tile_offsets || !coef || !thr || !ncl) return SS_ERR_INVALID;
    SplatParams P{};
    P.W = width; P.H = height; P.tile = tile; P.ntx = (width + tile - 1) / tile; P.k_max = k_max;
    P.offsets = tile_offsets; P.pair_rec = pair_rec;
    P.records = reinterpret_cast<const SsRecord *>(records);
    P.coef = reinterpret_cast<const float4 *>(coef);
    P.thr = thr; P.ncl = ncl; P.acc = rec_acc;
    const int ntiles = P.ntx * ((height + tile - 1) / tile);
    splat_bwd_kernel<<<ntiles, 256, 0, (cudaStream_t)stream>>>(P);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
