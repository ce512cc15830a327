// raster_walk.cuh -- the per-warp tile walk shared by the forward and
// backward rasterisers, and the fast coverage test with exact fallback.
#pragma once
#include "ss_common.cuh"

// Warp layout inside a tile CTA: warps own 8x4 pixel blocks.
struct WarpPix {
    int bx, by, px, py, lane, wid;
    bool live;
    float x, y;
    size_t pix;
};

__device__ __forceinline__ WarpPix warp_pixels(int t, int ntx, int tile, int W, int H) {
    WarpPix w;
    w.lane = threadIdx.x & 31;
    w.wid = threadIdx.x >> 5;
    const int tx = t % ntx, ty = t / ntx;
    const int wpr = tile >> 3;
    w.bx = tx * tile + (w.wid % wpr) * 8;
    w.by = ty * tile + (w.wid / wpr) * 4;
    w.px = w.bx + (w.lane & 7);
    w.py = w.by + (w.lane >> 3);
    w.live = w.px < W && w.py < H;
    w.x = ss_ndc_x(w.px, W);
    w.y = ss_ndc_y(w.py, H);
    w.pix = w.live ? (size_t)w.py * W + w.px : 0;
    return w;
}

__device__ __forceinline__ bool in_rect(const WarpPix &w, int4 r) {
    return w.live && w.px >= r.x && w.px < r.z && w.py >= r.y && w.py < r.w;
}

// Walk the tile's sorted pair list [p0, p1) in list order, calling
// f(record, pair_index, record_index) warp-uniformly for every record whose
// rect overlaps this warp's 8x4 block.  32 pairs at a time: the packed rects
// (coalesced, pair order) are culled with one ballot and only the overlapping
// records are gathered (16-byte loads) into this warp's private 32-slot
// shared-memory buffer -- no CTA-wide barrier, warps walk independently.
template <typename F>
__device__ __forceinline__ void walk_tile(const WarpPix &w, int p0, int p1, const int32_t *__restrict__ pair_rec,
                                          const uint2 *__restrict__ pair_rect, const SsRecord *__restrict__ recs,
                                          SsRecord *wbuf, F &&f) {
    for (int base = p0; base < p1; base += 32) {
        const int p = base + w.lane;
        bool ov = false;
        int rec = 0;
        if (p < p1) {
            const uint2 pr = __ldg(pair_rect + p);
            const int x0 = pr.x & 0xffff, y0 = pr.x >> 16, x1 = pr.y & 0xffff, y1 = pr.y >> 16;
            ov = x0 < w.bx + 8 && x1 > w.bx && y0 < w.by + 4 && y1 > w.by;
            if (ov) {
                rec = __ldg(pair_rec + p);
                const float4 *s = reinterpret_cast<const float4 *>(recs + rec);
                float4 *d = reinterpret_cast<float4 *>(wbuf + w.lane);
#pragma unroll
                for (int k = 0; k < 6; ++k) d[k] = __ldg(s + k);
            }
        }
        unsigned mask = __ballot_sync(0xffffffffu, ov);
        __syncwarp();
        while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            const int rj = __shfl_sync(0xffffffffu, rec, j);
            f(wbuf[j], base + j, rj);
        }
        __syncwarp();
    }
}

// Coverage of pixel (x, y) by a record, with everything downstream.
// Fast path: float32 with FMA and an approximate reciprocal.  Whenever the
// decision could differ from the reference's exact float32/float64 evaluation
// (rho^2 within 1% of the cut-off, or a denominator small relative to its
// terms) the exact evaluation (ss_intersect + ss_rho2) decides, so coverage
// and therefore layer membership are identical to the reference; u, v, rho^2
// and the weight are the fast values (a few ulp from the reference's).
struct Cover {
    float k0, k1, k2, l0, l1, l2, den, inv_den, u, v, rho2;
};

__device__ __forceinline__ bool ss_cover(float x, float y, const SsRecord &R, Cover &c) {
    const float t1x = R.a.x, t1y = R.a.y, t1z = R.a.z, t2x = R.a.w, t2y = R.b.x, t2z = R.b.y;
    const float t4x = R.b.z, t4y = R.b.w, t4z = R.c.x;
    c.k0 = __fmaf_rn(x, t4x, -t1x);
    c.k1 = __fmaf_rn(x, t4y, -t1y);
    c.k2 = __fmaf_rn(x, t4z, -t1z);
    c.l0 = __fmaf_rn(y, t4x, -t2x);
    c.l1 = __fmaf_rn(y, t4y, -t2y);
    c.l2 = __fmaf_rn(y, t4z, -t2z);
    const float a = c.k0 * c.l1, b = c.k1 * c.l0;
    c.den = a - b;
    c.inv_den = __fdividef(1.0f, c.den);
    c.u = (c.k1 * c.l2 - c.k2 * c.l1) * c.inv_den;
    c.v = (c.k2 * c.l0 - c.k0 * c.l2) * c.inv_den;
    const float s0 = R.c.y, s1 = R.c.z, s2 = R.c.w;
    c.rho2 = s0 * c.u * c.u + 2.f * s1 * c.u * c.v + s2 * c.v * c.v;
    const bool doubtful = !(fabsf(c.den) > 1e-5f * (fabsf(a) + fabsf(b)) + 1e-8f) ||
                          fabsf(c.rho2 - 9.f) < 0.09f || !(c.rho2 == c.rho2);
    if (!doubtful) return c.rho2 < 9.f;
    const float t1[3] = {t1x, t1y, t1z}, t2[3] = {t2x, t2y, t2z}, t4[3] = {t4x, t4y, t4z};
    SsHit h;
    if (!ss_intersect(x, y, t1, t2, t4, h)) return false;
    const double r2 = ss_rho2(s0, s1, s2, h.u, h.v);
    if (!(r2 < 9.0)) return false;
    c.k0 = h.k0; c.k1 = h.k1; c.k2 = h.k2; c.l0 = h.l0; c.l1 = h.l1; c.l2 = h.l2;
    c.den = h.den; c.inv_den = 1.f / h.den; c.u = h.u; c.v = h.v; c.rho2 = (float)r2;
    return true;
}
