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

__device__ __forceinline__ WarpPix warp_pixels(int t, int ntx, int tile, int W, int H, int wid_in_tile) {
    WarpPix w;
    w.lane = threadIdx.x & 31;
    w.wid = wid_in_tile;
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

__device__ __forceinline__ WarpPix warp_pixels(int t, int ntx, int tile, int W, int H) {
    return warp_pixels(t, ntx, tile, W, H, threadIdx.x >> 5);
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
// k, l, den and the two numerators are evaluated with the reference's exact
// float32 operation sequence (no contraction), so they are bit-identical to
// rasterizer.py:197-205 and the ray-miss test |den| < 1e-9 is exact.  The
// quotient uses an IEEE reciprocal (u, v within 1 ulp of the reference's
// division) and rho^2 is evaluated in float32; when the quadratic form is ill
// conditioned (cancelling terms, |terms| > 32) or rho^2 lies within 2e-4 of
// its term magnitude from the cut-off, the reference's exact u, v and numba's
// float64 rho^2 decide (and are used).  Coverage and layer membership are
// therefore identical to the reference, and weights agree to ~1e-6 relative.
struct Cover {
    float k0, k1, k2, l0, l1, l2, den, inv_den, u, v, rho2;
};

__device__ __forceinline__ bool ss_cover(float x, float y, const SsRecord &R, Cover &c) {
    const float t1x = R.a.x, t1y = R.a.y, t1z = R.a.z, t2x = R.a.w, t2y = R.b.x, t2z = R.b.y;
    const float t4x = R.b.z, t4y = R.b.w, t4z = R.c.x;
    c.k0 = fs(fm(x, t4x), t1x);
    c.k1 = fs(fm(x, t4y), t1y);
    c.k2 = fs(fm(x, t4z), t1z);
    c.l0 = fs(fm(y, t4x), t2x);
    c.l1 = fs(fm(y, t4y), t2y);
    c.l2 = fs(fm(y, t4z), t2z);
    c.den = fs(fm(c.k0, c.l1), fm(c.k1, c.l0));
    if (fabsf(c.den) <= 9.99999972e-10f) return false;  // == (double)|den| < 1e-9 exactly
    const float nu = fs(fm(c.k1, c.l2), fm(c.k2, c.l1));
    const float nv = fs(fm(c.k2, c.l0), fm(c.k0, c.l2));
    c.inv_den = __frcp_rn(c.den);
    c.u = nu * c.inv_den;
    c.v = nv * c.inv_den;
    const float s0 = R.c.y, s1 = R.c.z, s2 = R.c.w;
    const float ta = s0 * c.u * c.u, tb = 2.f * s1 * c.u * c.v, tc = s2 * c.v * c.v;
    c.rho2 = ta + tb + tc;
    // the float32 sum is within ~4e-7 * mag of the reference's mixed-precision
    // value when the quadratic form is well conditioned (mag <= 32); otherwise,
    // or near the cut-off, the reference's exact arithmetic decides
    const float mag = fabsf(ta) + fabsf(tb) + fabsf(tc);
    if (c.rho2 - 9.f >= 2e-4f * mag) return false;                // clearly outside
    if (9.f - c.rho2 >= 2e-4f * mag && mag <= 32.f) return true;  // clearly inside, well conditioned
    // doubtful: the reference's exact quotient and float64 rho^2 decide
    c.u = fd(nu, c.den);
    c.v = fd(nv, c.den);
    const double r2 = ss_rho2(s0, s1, s2, c.u, c.v);
    c.rho2 = (float)r2;
    return r2 < 9.0;
}
