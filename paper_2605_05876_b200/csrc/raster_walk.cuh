// raster_walk.cuh -- the per-warp tile walk shared by the forward and
// backward rasterisers, and the fast coverage test with exact fallback.
#pragma once
#include "ss_common.cuh"
#include "coverage.cuh"

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

// Per-warp shared scratch of the packed walk: the chunk's overlapping records
// (compacted, list order; the 64 bytes coverage needs), the per-slot fields
// the compositing reads (SoA: lanes on different slots hit different banks),
// the per (slot, pixel) weights and the per-pixel slot masks.
struct RecGeo {
    float4 a, b, c, d;    // the first 64 bytes of SsRecord
};

#ifndef SS_PACK_SLOTS
#define SS_PACK_SLOTS 20
#endif
constexpr int kSlots = SS_PACK_SLOTS;  // overlapping records per chunk (<= 32)

// One chunk of overlapping records (double-buffered: the next chunk's
// records stream in with cp.async while the current one is processed).
struct ChunkBuf {
    RecGeo geo[kSlots];       // t1, t2, t4, Sigma^-1, n_f, view_z, z_start, z_end
    float4 ext[kSlots];       // colour r, g, b, coverage margin (record bytes 64..79)
    int meta[32];             // in-block rect: cx0 | cw << 4 | ry0 << 8 | cnt << 12 (lanes >= n: unread)
    int pidx[kSlots];
};

struct PackedScratch {
    ChunkBuf buf[2];
    float wgt[kSlots][32];    // [slot][pixel]: n_f exp(-rho^2/2) when covered, -1 when not (in-rect only)
    unsigned mask[32];        // per pixel: slots whose rect contains it
    int ncov[32];             // covered lanes per slot (pair cover counts)
    float xs[8], ys[4];
};

// What the compositing of one (slot, pixel) sees.
struct SlotView {
    float w;              // >= 0 covered (the weight), < 0 in rect but not covered
    float zs, ze, vz, c0, c1, c2;
    int slot;
};

__device__ __forceinline__ void packed_init(const WarpPix &w, PackedScratch &sm, int W, int H) {
    if (w.lane < 8) sm.xs[w.lane] = ss_ndc_x(w.bx + w.lane, W);
    if (w.lane < 4) sm.ys[w.lane] = ss_ndc_y(w.by + w.lane, H);
    sm.mask[w.lane] = 0u;
    sm.ncov[w.lane] = 0;
    __syncwarp();
}

// kCoveredOnly: phase 2 visits only the COVERED slots of each pixel.  That
// renders identically: an in-rect record that does not cover the pixel adds
// no weight, and the layer it may close by the gap test (z_start > z_max_end,
// rasterizer.py:168) would be closed by the next covering record anyway --
// list order is ascending z_start, so that record's z_start is larger still,
// nothing was accumulated in between, and the K_MAX stop falls on the same
// layer.  Only the discarded-record statistic (counted per in-rect record)
// needs the full in-rect walk.
// Two-phase walk of the tile's sorted pair list [p0, p1) for one 8x4 warp
// block.  Per chunk the next (up to) 32 overlapping records are gathered
// (compacted, list order) into the warp's shared scratch -- scanning as many
// 32-pair windows as that takes, so the per-chunk work is amortised over
// full slot sets; stop() is polled between chunks; phase 1 evaluates coverage and
// weight for every in-rect (record, pixel) item with ONE item per lane (items
// packed across records, so no lane idles outside a record's rect) and marks
// the slot in the pixel's mask; phase 2 lets every lane walk only ITS pixel's
// in-rect slots, in list order, calling f(SlotView) -- the order-dependent
// compositing costs max-over-lanes of the in-rect count instead of the number
// of overlapping records.
template <bool kCoveredOnly, typename Stop, typename Wt, typename F>
__device__ __forceinline__ void walk_tile_packed(const WarpPix &w, int p0, int p1, const int32_t *__restrict__ pair_rec,
                                                 const uint2 *__restrict__ pair_rect,
                                                 const SsRecord *__restrict__ recs, PackedScratch &sm,
                                                 int32_t *pair_cover, Stop &&stop, Wt &&weight, F &&f) {
    const unsigned FULL = 0xffffffffu;
    const unsigned lt = (1u << w.lane) - 1u;
    int cursor = p0;
    // the next window's pair rects and record indices are loaded one window
    // ahead (right after the cursor moves), so their latency hides behind
    // the current window's work
    uint2 pr_next = make_uint2(0u, 0u);
    int rec_next = 0;
    auto prefetch = [&](int c) {
        const int p = c + w.lane;
        if (p < p1) {
            pr_next = __ldg(pair_rect + p);
            rec_next = __ldg(pair_rec + p);
        }
    };
    // fill cb with up to kSlots next overlapping records (list order),
    // scanning as many 32-pair windows as that takes; the records are copied
    // with cp.async (one commit group per chunk)
    auto fill = [&](ChunkBuf &cb) -> int {
        int n = 0;
        while (n < kSlots && cursor < p1) {
            const int p = cursor + w.lane;
            const uint2 pr = pr_next;
            const int rec = rec_next;
            bool ov = false;
            int meta = 0;
            if (p < p1) {
                const int x0 = pr.x & 0xffff, y0 = pr.x >> 16, x1 = pr.y & 0xffff, y1 = pr.y >> 16;
                ov = x0 < w.bx + 8 && x1 > w.bx && y0 < w.by + 4 && y1 > w.by;
                const int cx0 = max(x0 - w.bx, 0), cw = min(x1 - w.bx, 8) - cx0;
                const int ry0 = max(y0 - w.by, 0), ch = min(y1 - w.by, 4) - ry0;
                meta = cx0 | (cw << 4) | (ry0 << 8) | ((cw * ch) << 12);
            }
            unsigned ovm = __ballot_sync(FULL, ov);
            const int room = kSlots - n;
            if (__popc(ovm) > room) {
                // keep the first `room` overlapping pairs; resume after the last kept
                const int last = __fns(ovm, 0, room);
                ovm &= (2u << last) - 1u;
                cursor += last + 1;
            } else {
                cursor += 32;
            }
            prefetch(cursor);
            if ((ovm >> w.lane) & 1u) {
                const int pos = n + __popc(ovm & lt);
                const float4 *src = reinterpret_cast<const float4 *>(recs + rec);
                cp_async16(&cb.geo[pos].a, src);
                cp_async16(&cb.geo[pos].b, src + 1);
                cp_async16(&cb.geo[pos].c, src + 2);
                cp_async16(&cb.geo[pos].d, src + 3);
                cp_async16(&cb.ext[pos], src + 4);
                cb.meta[pos] = meta;
                cb.pidx[pos] = p;
            }
            n += __popc(ovm);
        }
        cp_async_commit();
        return n;
    };
    prefetch(cursor);
    int cur = 0;
    int n = stop() ? 0 : fill(sm.buf[0]);
    while (n > 0) {
        cp_async_wait_all();
        __syncwarp();
        ChunkBuf &cb = sm.buf[cur];
        // the next chunk streams into the other buffer during this one's phases
        const int n_next = cursor < p1 ? fill(sm.buf[cur ^ 1]) : 0;
        // phase 1: inclusive scan of the per-slot item counts, then packed items
        const int my_meta = w.lane < n ? cb.meta[w.lane] : 0;
        const int cnt = my_meta >> 12;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (w.lane >= o) incl += y;
        }
        const int total = __shfl_sync(FULL, incl, 31);
        // geometry | slot's first item << 12 | magic(cw) << 23, where
        // (k * magic) >> 8 == k / cw for k < 32 (magic = ceil(256 / cw))
        const unsigned cwm = (my_meta >> 4) & 15;
        const unsigned magic = cwm ? (unsigned)((0x1F242A333F557FFFull >> ((cwm - 1) * 8)) & 0xFF) + 1u : 0u;
        const unsigned packed = (unsigned)(my_meta & 0xfff) | ((unsigned)(incl - cnt) << 12) | (magic << 23);
        for (int b0 = 0; b0 < total; b0 += 32) {
            const bool bnd = w.lane < n && incl > b0 && incl < b0 + 32;
            const unsigned B = __reduce_or_sync(FULL, bnd ? (1u << (incl - b0)) : 0u);
            const int j0 = __popc(__ballot_sync(FULL, w.lane < n && incl <= b0));
            const int s = min(j0 + __popc(B & ((2u << w.lane) - 1u)), 31);
            const unsigned pk = __shfl_sync(FULL, packed, s);
            const int i = b0 + w.lane;
            if (i < total) {
                const int k = i - (int)((pk >> 12) & 0x7ff);
                const int cx0 = pk & 15, cw = (pk >> 4) & 15, ry0 = (pk >> 8) & 15;
                const int row = (k * (int)(pk >> 23)) >> 8;
                const int col = k - row * cw;
                const int px = (ry0 + row) * 8 + cx0 + col;
                const float wv = weight(cb.geo[s], sm.xs[px & 7], sm.ys[px >> 3]);
                sm.wgt[s][px] = wv;
                if (!kCoveredOnly || wv >= 0.f) atomicOr(&sm.mask[px], 1u << s);
            }
        }
        __syncwarp();
        // phase 2: each lane walks its own pixel's in-rect slots in list order
        unsigned M = sm.mask[w.lane];
        sm.mask[w.lane] = 0u;
        while (__any_sync(FULL, M != 0u)) {
            if (M != 0u) {
                SlotView v;
                v.slot = __ffs(M) - 1;
                M &= M - 1u;
                v.w = sm.wgt[v.slot][w.lane];
                const float4 d = cb.geo[v.slot].d;
                const float4 e = cb.ext[v.slot];
                v.zs = d.z; v.ze = d.w; v.vz = d.y;
                v.c0 = e.x; v.c1 = e.y; v.c2 = e.z;
                f(v);
            }
        }
        __syncwarp();
        if (pair_cover && w.lane < n && sm.ncov[w.lane] > 0) {  // f counted covered lanes per slot
            atomicAdd(&pair_cover[cb.pidx[w.lane]], sm.ncov[w.lane]);
            sm.ncov[w.lane] = 0;
        }
        if (stop()) break;  // polled between chunks
        n = n_next;
        cur ^= 1;
    }
    cp_async_wait_all();
}

// Coverage of pixel (x, y) by a record, with everything downstream.
// k, l, den and the two numerators are evaluated with the reference's exact
// float32 operation sequence (no contraction), so they are bit-identical to
// rasterizer.py:197-205 and the ray-miss test |den| < 1e-9 is exact.  The
// quotient uses a Newton-refined hardware reciprocal (u, v within ~2 ulp of
// the reference's division) and rho^2 is evaluated in float32; when the quadratic form is ill
// conditioned (cancelling terms, |terms| > 32) or rho^2 lies within 2e-4 of
// its term magnitude from the cut-off, the reference's exact u, v and numba's
// float64 rho^2 decide (and are used).  Coverage and layer membership are
// therefore identical to the reference, and weights agree to ~1e-6 relative.
struct Cover {
    float k0, k1, k2, l0, l1, l2, den, inv_den, u, v, rho2;
};

template <typename Rec>
__device__ __forceinline__ bool ss_cover(float x, float y, const Rec &R, Cover &c) {
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
    c.inv_den = fc_rcp(c.den);  // hardware rcp + one Newton step (~1 ulp; no slow-path branch)
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
