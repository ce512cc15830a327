// raster_bwd.cu -- analytic backward of the interval-grouped compositing.
//
// Reference: _backward_kernel (backward.py:48-321) + the fixed-order pair
// reduction (backward.py:382-396).  Two replays of the forward walk per pixel
// like the reference: pass 1 rebuilds the per-layer sums and evaluates the
// suffix recursion over the compositing chain (plus the consolidation penalty
// and its gradients) in float64 per pixel; pass 2 walks the list again and
// distributes per-record gradients.
//
// B200 mapping: same tile CTA / 8x4-pixel warp layout and shared-memory
// staging as the forward.  In pass 2 all 32 lanes of a warp process the SAME
// record (for 32 different pixels), so the 18 per-record gradient channels
// are summed across the warp with a transposed butterfly (20 shuffles instead
// of 90) that leaves one channel total per lane, and 18 lanes issue one
// coalesced fp32 RED each into the record's accumulator row: one atomic
// per (warp, record, channel) instead of the reference's per-(pixel, record)
// 17-float pair buffer.
//
// Depth moments are accumulated relative to the first member of each layer
// (z - z0) so the consolidation variance E[z^2] - E[z]^2 does not cancel in
// float32; the per-record chain uses the algebraically identical centred
// form of backward.py:278-286.
#include "ss_common.cuh"
#include "warp_reduce.cuh"
#include "raster_walk.cuh"

namespace {

constexpr int KC = SS_KMAX_CAP;
constexpr int NCH = 18;  // reduced channels: t1(3) t2(3) t4(3) sinv(3) nf col(3) vz ss

struct BwdParams {
    const float4 *coef;  // kCoef: per-layer (A, dL/dC_raw) from ss_train_forward
    int W, H, tile, ntx, k_max;
    float bg0, bg1, bg2, cons_scale;
    const int32_t *offsets;
    const int32_t *pair_rec;
    const uint2 *pair_rect;
    const SsRecord *records;
    const float *g_rgb, *g_alpha;
    float *acc;
    double *cons_loss;
};

template <bool kCoef>
__global__ void __launch_bounds__(256) raster_bwd_kernel(BwdParams P)
{
    __shared__ SsRecord wbuf_all[8][32];
    __shared__ double cons_red[32];
    const int t = blockIdx.x;
    const WarpPix wp = warp_pixels(t, P.ntx, P.tile, P.W, P.H);
    const int lane = wp.lane, wid = wp.wid;
    const bool live = wp.live;
    const size_t pix = wp.pix;
    const float x = wp.x, y = wp.y;
    SsRecord *wbuf = wbuf_all[wid];

    // owner lane / channel of the transposed warp reduction
    const int my_ch = warp_tr_index<NCH>(lane);
    const unsigned same = __match_any_sync(0xffffffffu, my_ch);
    const bool owner = (__ffs(same) - 1) == lane;

    const int p0 = P.offsets[t], p1 = P.offsets[t + 1];

    // ---------------- pass 1: layer sums (rasterizer walk replay) ----------
    constexpr int KP = kCoef ? 1 : KC;
    float lw[KP], lc0[KP], lc1[KP], lc2[KP], lzs[KP], lz2s[KP], lz0[KP];
    int nl = 0;
    if constexpr (!kCoef) {
        float Wg = 0.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Zs = 0.f, Z2s = 0.f, z0 = 0.f, zmax = 0.f;
        bool stopped = !live;
        walk_tile(wp, p0, p1, P.pair_rec, P.pair_rect, P.records, wbuf, [&](const SsRecord &R, int, int) {
            if (stopped || !in_rect(wp, R.r)) return;
            if (Wg > 0.f && R.d.z > zmax) {
                lw[nl] = Wg; lc0[nl] = C0; lc1[nl] = C1; lc2[nl] = C2;
                lzs[nl] = Zs; lz2s[nl] = Z2s; lz0[nl] = z0;
                ++nl;
                Wg = C0 = C1 = C2 = Zs = Z2s = zmax = 0.f;
                if (nl >= P.k_max) { stopped = true; return; }
            }
            Cover c;
            if (!ss_cover(x, y, R, c)) return;
            const float w = R.d.x * ss_exp_fast(-0.5f * c.rho2);
            const float z = R.d.y;
            if (Wg == 0.f) z0 = z;
            const float dz = z - z0;
            Wg += w;
            C0 += w * R.e.x; C1 += w * R.e.y; C2 += w * R.e.z;
            Zs += w * dz; Z2s += w * dz * dz;
            if (R.d.w > zmax) zmax = R.d.w;
        });
        if (live && Wg > 0.f) {
            lw[nl] = Wg; lc0[nl] = C0; lc1[nl] = C1; lc2[nl] = C2;
            lzs[nl] = Zs; lz2s[nl] = Z2s; lz0[nl] = z0;
            ++nl;
        }
    }

    // ------- per-pixel layer gradients (float64, backward.py:160-238) -------
    // Stored per layer: A (weight term), gC (3), B (depth), Cq (variance),
    // zb (layer mean depth), vr (raw variance): g_w = A + gC.c + B dz + Cq (dz^2 - vr)
    float cA[KP], cC0[KP], cC1[KP], cC2[KP], cB[KP], cQ[KP], cZb[KP], cV[KP];
    double cons_pix = 0.0;
    if (!kCoef && nl > 0) {
        double a[KC], tb[KC], zb[KC], vr[KC], gw_c[KC], gz_c[KC], gv_c[KC];
        double trans = 1.0;
        for (int m = 0; m < nl; ++m) {
            a[m] = -expm1(-(double)lw[m]);
            tb[m] = trans;
            trans *= 1.0 - a[m];
            const double inv = 1.0 / (double)lw[m];
            const double mz = (double)lzs[m] * inv;
            zb[m] = (double)lz0[m] + mz;
            vr[m] = (double)lz2s[m] * inv - mz * mz;
            gw_c[m] = gz_c[m] = gv_c[m] = 0.0;
        }
        const double s = P.cons_scale;
        if (s > 0.0) {
            double wm[KC];
            for (int m = 0; m < nl; ++m) {
                wm[m] = tb[m] * a[m];
                gv_c[m] = vr[m] > 0.0 ? s * wm[m] * wm[m] : 0.0;
            }
            double l_pix = 0.0;
            for (int i = 0; i < nl; ++i) {
                const double var = vr[i] > 0.0 ? vr[i] : 0.0;
                l_pix += wm[i] * wm[i] * var;
                gw_c[i] += s * 2.0 * wm[i] * var;
                for (int j = i + 1; j < nl; ++j) {
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
        }
        const double gc0 = P.g_rgb[3 * pix], gc1 = P.g_rgb[3 * pix + 1], gc2 = P.g_rgb[3 * pix + 2];
        const double ga = P.g_alpha ? (double)P.g_alpha[pix] : 0.0;
        double sf0 = P.bg0, sf1 = P.bg1, sf2 = P.bg2, q = 1.0, rw = 0.0;
        for (int m = nl - 1; m >= 0; --m) {
            const double inv = 1.0 / (double)lw[m];
            const double ch0 = lc0[m] * inv, ch1 = lc1[m] * inv, ch2 = lc2[m] * inv;
            const double g_am = tb[m] * (gc0 * (ch0 - sf0) + gc1 * (ch1 - sf1) + gc2 * (ch2 - sf2) + ga * q + gw_c[m] - rw);
            const double ta = tb[m] * a[m];
            const double gh0 = gc0 * ta, gh1 = gc1 * ta, gh2 = gc2 * ta;
            cA[m] = (float)(g_am * (1.0 - a[m]) - (gh0 * ch0 + gh1 * ch1 + gh2 * ch2) * inv);
            cC0[m] = (float)(gh0 * inv); cC1[m] = (float)(gh1 * inv); cC2[m] = (float)(gh2 * inv);
            cB[m] = (float)(gz_c[m] * inv);
            cQ[m] = (float)(gv_c[m] * inv);
            cZb[m] = (float)zb[m];
            cV[m] = (float)vr[m];
            sf0 = a[m] * ch0 + (1.0 - a[m]) * sf0;
            sf1 = a[m] * ch1 + (1.0 - a[m]) * sf1;
            sf2 = a[m] * ch2 + (1.0 - a[m]) * sf2;
            q *= 1.0 - a[m];
            rw = gw_c[m] * a[m] + (1.0 - a[m]) * rw;
        }
    }

    // ---------------- pass 2: distribute per-record gradients ----------------
    {
        int m_cur = 0, group_n = 0;
        float zmax = 0.f;
        bool stopped = kCoef ? !live : nl == 0;
        const int m_end = kCoef ? P.k_max : nl;
        const size_t HW = (size_t)P.W * P.H;
        float A = 0.f, G0 = 0.f, G1 = 0.f, G2 = 0.f, Bz = 0.f, Qv = 0.f, Zb = 0.f, Vr = 0.f;
        if (kCoef) {
            if (live) { const float4 c = P.coef[pix]; A = c.x; G0 = c.y; G1 = c.z; G2 = c.w; }
        } else if (nl > 0) {
            A = cA[0]; G0 = cC0[0]; G1 = cC1[0]; G2 = cC2[0]; Bz = cB[0]; Qv = cQ[0]; Zb = cZb[0]; Vr = cV[0];
        }
        for (int cb = p0; cb < p1; cb += 32 * 8) {
            if (__all_sync(0xffffffffu, stopped)) break;
            const int ce = min(p1, cb + 32 * 8);
            walk_tile(wp, cb, ce, P.pair_rec, P.pair_rect, P.records, wbuf, [&](const SsRecord &R, int, int rec) {
                float v[NCH];
#pragma unroll
                for (int k = 0; k < NCH; ++k) v[k] = 0.f;
                bool cov = false;
                if (!stopped && in_rect(wp, R.r)) {
                    bool go = true;
                    if (group_n > 0 && R.d.z > zmax) {
                        ++m_cur;
                        group_n = 0;
                        zmax = 0.f;
                        if (m_cur >= P.k_max || m_cur >= m_end) {
                            stopped = true;
                            go = false;
                        } else if (kCoef) {
                            const float4 c = P.coef[(size_t)m_cur * HW + pix];
                            A = c.x; G0 = c.y; G1 = c.z; G2 = c.w;
                        } else {
                            A = cA[m_cur]; G0 = cC0[m_cur]; G1 = cC1[m_cur]; G2 = cC2[m_cur];
                            Bz = cB[m_cur]; Qv = cQ[m_cur]; Zb = cZb[m_cur]; Vr = cV[m_cur];
                        }
                    }
                    Cover c;
                    if (go && ss_cover(x, y, R, c)) {
                        // backward.py:272-320 in the centred depth form
                        cov = true;
                        ++group_n;
                        if (R.d.w > zmax) zmax = R.d.w;
                        const float e = ss_exp_fast(-0.5f * c.rho2);
                        const float w = R.d.x * e;
                        const float dz = R.d.y - Zb;
                        const float gw = A + G0 * R.e.x + G1 * R.e.y + G2 * R.e.z + Bz * dz + Qv * (dz * dz - Vr);
                        v[13] = w * G0; v[14] = w * G1; v[15] = w * G2;
                        v[16] = w * (Bz + 2.f * Qv * dz);
                        const float gr = -0.5f * w * gw;
                        v[12] = e * gw;
                        const float u = c.u, vv = c.v;
                        v[9] = gr * u * u; v[10] = gr * 2.f * u * vv; v[11] = gr * vv * vv;
                        // float32 sums like numba's (backward.py:292-293)
                        const float gu = 2.f * gr * fa(fm(R.c.y, u), fm(R.c.z, vv));
                        const float gv = 2.f * gr * fa(fm(R.c.z, u), fm(R.c.w, vv));
                        const float gp0 = gu * c.inv_den, gp1 = gv * c.inv_den, gp2 = -(gu * u + gv * vv) * c.inv_den;
                        const float gk0 = c.l1 * gp2 - c.l2 * gp1;
                        const float gk1 = c.l2 * gp0 - c.l0 * gp2;
                        const float gk2 = c.l0 * gp1 - c.l1 * gp0;
                        const float gl0 = gp1 * c.k2 - gp2 * c.k1;
                        const float gl1 = gp2 * c.k0 - gp0 * c.k2;
                        const float gl2 = gp0 * c.k1 - gp1 * c.k0;
                        v[0] = -gk0; v[1] = -gk1; v[2] = -gk2;
                        v[3] = -gl0; v[4] = -gl1; v[5] = -gl2;
                        v[6] = x * gk0 + y * gl0; v[7] = x * gk1 + y * gl1; v[8] = x * gk2 + y * gl2;
                        v[17] = fabsf(R.c.x) * sqrtf(gk2 * gk2 + gl2 * gl2);
                    }
                }
                const unsigned cm = __ballot_sync(0xffffffffu, cov);
                if (cm) {
                    warp_tr_reduce<NCH>(v, lane);
                    float *dst = P.acc + (size_t)rec * SS_ACC_FLOATS;
                    if (owner) atomicAdd(dst + my_ch, v[0]);
                    if (lane == 0) atomicAdd(reinterpret_cast<int *>(dst + 18), __popc(cm));
                }
            });
        }
    }

    if (kCoef) return;
    // consolidation value: block reduce, one double atomic per CTA
    double cp = cons_pix;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cp += __shfl_xor_sync(0xffffffffu, cp, o);
    if (lane == 0) cons_red[wid] = cp;
    __syncthreads();
    if (threadIdx.x == 0 && P.cons_scale > 0.f) {
        double s = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += cons_red[k];
        if (s != 0.0) atomicAdd(P.cons_loss, s);
    }
}

}  // namespace

extern "C" int ss_raster_backward(int width, int height, int tile, const int32_t *tile_offsets,
                                  const int32_t *pair_rec, const uint32_t *pair_rect, const float *records, const float *background,
                                  int k_max, const float *g_rgb, const float *g_alpha, float cons_scale,
                                  float *rec_acc, double *cons_loss, void *stream)
{
    if (width <= 0 || height <= 0 || tile != 16 || k_max < 1 || k_max > SS_KMAX_CAP) return SS_ERR_INVALID;
    if (!tile_offsets || !background || !g_rgb || !cons_loss) return SS_ERR_INVALID;
    BwdParams P;
    P.W = width; P.H = height; P.tile = tile; P.ntx = (width + tile - 1) / tile; P.k_max = k_max;
    P.bg0 = background[0]; P.bg1 = background[1]; P.bg2 = background[2];
    P.cons_scale = cons_scale;
    P.offsets = tile_offsets; P.pair_rec = pair_rec;
    P.pair_rect = reinterpret_cast<const uint2 *>(pair_rect);
    P.records = reinterpret_cast<const SsRecord *>(records);
    P.g_rgb = g_rgb; P.g_alpha = g_alpha; P.acc = rec_acc; P.cons_loss = cons_loss;
    const int nty = (height + tile - 1) / tile;
    const int threads = tile * tile;
    P.coef = nullptr;
    raster_bwd_kernel<false><<<P.ntx * nty, threads, 0, (cudaStream_t)stream>>>(P);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
