// refine.cu -- the density-aware refinement scan on the device, with no host
// synchronisation: prune -> split selection -> budget -> compaction -> the
// new cloud and the remapped optimiser state in one pass.
//
// Reference: refine_topology (densify.py:168-202): prune_keep_mask
// (:101-135: stale = grad_sum <= 0, isolated (the isolation kernel of
// optim.cu), floater = front > 0 & outside >= front), select_split (:43-57:
// threshold = max(np.quantile(mean_grad[active], q), grad_floor) with numpy's
// default 'linear' method, i.e. virtual index (m - 1) q and numpy's _lerp;
// candidates mean_grad >= thresh and max scale > mean neighbour distance),
// the budget (:187-198: the `allowed` largest mean_grad, ties in index
// order -- a stable argsort of -mean_grad), split_cloud (:60-98: layout
// [stay..., +children..., -children...]) and Adam.remap (adam.py:43-58:
// rows follow their source, children start from zero moments).
//
// B200 mapping: one flag pass; order statistics by an 8-bit radix select on
// the IEEE bits of the positive float64 mean gradients (8 histogram passes,
// block-privatised histograms); the counts and the chosen digits live in a
// device state block, so the whole sequence is a fixed list of launches
// (stream-ordered, graph-capturable); compaction by a three-kernel scan
// (block counts, one-block scan of the block counts, block-local scan).
// All of it streams a few bytes per surfel: HBM- and launch-bound.
#include "ss_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kScanBlock = 1024;  // elements per scan block (4 per thread)

enum {
    C_OUT = 0, C_KEPT, C_SPLIT, C_STALE, C_ISO, C_FLOAT, C_ACTIVE, C_CAND, C_STAY, C_GT, C_EQ, C_NCOUNT
};

struct RefineState {
    long long counts[16];
    unsigned long long prefix, mask;  // radix select: digits chosen so far
    long long rank;                   // rank still to find inside the prefix class
    long long q_prev;                 // quantile: floor of the virtual index (-1: take the max)
    double q_gamma;                   // quantile: fractional part
    unsigned long long v_prev;        // bits of sorted[q_prev]
    unsigned long long min_gt;        // smallest key above v_prev
    long long count_le;               // keys <= v_prev
    double thresh;                    // the split threshold
    long long budget_on;              // 1 when the budget cut applies
    long long allowed;
    unsigned long long v_cut;         // budget: value of the allowed-th largest candidate
    long long need_eq;                // budget: candidates equal to v_cut still to take
};

// flag bits
constexpr uint8_t F_KEEP = 1, F_ACTIVE = 2, F_CAND = 4, F_CHOSEN = 8, F_EQ = 16;

__device__ __forceinline__ unsigned long long key_of(double v) { return (unsigned long long)__double_as_longlong(v); }

__device__ __forceinline__ float scale_max_f32(const float *ls, int i) {
    // densify.py:56/122: cloud.scales = exp(log_scales) in float32 (correctly rounded here)
    const float s0 = (float)exp((double)ls[2 * i]), s1 = (float)exp((double)ls[2 * i + 1]);
    return s0 > s1 ? s0 : s1;
}

template <int N>
__device__ __forceinline__ void block_add(long long (&v)[N], long long *dst) {
    __shared__ long long s[N];
    if (threadIdx.x < N) s[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) {
        long long x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd((unsigned long long *)&s[k], (unsigned long long)x);
    }
    __syncthreads();
    if (threadIdx.x < N && s[threadIdx.x]) atomicAdd((unsigned long long *)&dst[threadIdx.x], (unsigned long long)s[threadIdx.x]);
}

__global__ void init_kernel(RefineState *st) {
    if (threadIdx.x < 16) st->counts[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        st->prefix = st->mask = 0ull;
        st->rank = 0;
        st->min_gt = ~0ull;
        st->count_le = 0;
        st->thresh = 0.0;
        st->budget_on = 0;
        st->need_eq = 0;
    }
}

// prune_keep_mask + mean gradient + active flag (densify.py:35-57, 101-135)
__global__ void flags_kernel(int n, const double *__restrict__ grad_sum, const int64_t *__restrict__ view_count,
                             const uint8_t *__restrict__ isolated, const int64_t *__restrict__ outside,
                             const int64_t *__restrict__ front, double *__restrict__ mg, uint8_t *__restrict__ fl,
                             RefineState *st) {
    long long c[6] = {0, 0, 0, 0, 0, 0};  // kept, stale, iso, floater, active, (unused)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double gs = grad_sum[i];
        const bool stale = gs <= 0.0;
        const bool iso = n > 1 && isolated[i] != 0;
        bool flo = false;
        if (outside && front) flo = front[i] > 0 && outside[i] >= front[i];
        const bool keep = !(stale || iso || flo);
        const long long vc = view_count[i];
        const double m = gs / (double)(vc > 1 ? vc : 1);
        uint8_t f = 0;
        if (keep) { f |= F_KEEP; ++c[0]; }
        if (keep && m > 0.0) { f |= F_ACTIVE; ++c[4]; }
        c[1] += stale;
        c[2] += iso && !stale;
        c[3] += flo && !stale && !iso;
        mg[i] = m;
        fl[i] = f;
    }
    long long v[5] = {c[0], c[1], c[2], c[3], c[4]};
    __shared__ long long s[5];
    if (threadIdx.x < 5) s[threadIdx.x] = 0;
    __syncthreads();
    for (int k = 0; k < 5; ++k) {
        long long x = v[k];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd((unsigned long long *)&s[k], (unsigned long long)x);
    }
    __syncthreads();
    const int slot[5] = {C_KEPT, C_STALE, C_ISO, C_FLOAT, C_ACTIVE};
    if (threadIdx.x < 5 && s[threadIdx.x]) atomicAdd((unsigned long long *)&st->counts[slot[threadIdx.x]],
                                                     (unsigned long long)s[threadIdx.x]);
}

// numpy linear quantile (virtual index (m - 1) q, _get_indexes, _get_gamma):
// the rank to select and the interpolation weight
__global__ void quantile_setup_kernel(RefineState *st, double q) {
    const long long m = st->counts[C_ACTIVE];
    st->prefix = st->mask = 0ull;
    if (m == 0) { st->q_prev = -2; st->rank = 0; return; }
    const double v = (double)(m - 1) * q;
    if (v >= (double)(m - 1)) {           // above bounds: the largest value
        st->q_prev = -1;
        st->rank = m - 1;
        st->q_gamma = 0.0;
    } else {
        const double pv = floor(v);
        st->q_prev = (long long)pv;
        st->rank = (long long)pv;
        st->q_gamma = v - pv;
    }
}

// One radix-select pass over the keys of the rows whose flags contain
// `want`: histogram of digit `pass` (8 bits, most significant first) among
// the keys matching the digits chosen so far.
__global__ void select_hist_kernel(int n, const double *__restrict__ mg, const uint8_t *__restrict__ fl, uint8_t want,
                                   int pass, const RefineState *st, unsigned int *__restrict__ hist) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long prefix = st->prefix, mask = st->mask;
    const int shift = 56 - 8 * pass;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if ((fl[i] & want) != want) continue;
        const unsigned long long k = key_of(mg[i]);
        if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(hist + threadIdx.x, h[threadIdx.x]);
}

// Choose the digit of this pass that holds the wanted rank; zero the histogram.
__global__ void select_pick_kernel(int pass, RefineState *st, unsigned int *__restrict__ hist, int active_only) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = hist[threadIdx.x];
    hist[threadIdx.x] = 0;
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (active_only == 1 && st->q_prev == -2) return;  // no active rows: nothing to select
    if (active_only == 2 && !st->budget_on) return;    // budget not binding
    long long r = st->rank;
    int b = 0;
    for (; b < 255; ++b) {
        if (r < (long long)h[b]) break;
        r -= h[b];
    }
    const int shift = 56 - 8 * pass;
    st->prefix |= (unsigned long long)b << shift;
    st->mask |= 255ull << shift;
    st->rank = r;
}

// Quantile: sorted[prev] is the selected key; sorted[prev + 1] is the same
// value when more than prev + 1 keys are <= it, else the smallest larger key.
__global__ void quantile_next_kernel(int n, const double *__restrict__ mg, const uint8_t *__restrict__ fl,
                                     RefineState *st) {
    const unsigned long long v = st->prefix;
    long long le = 0;
    unsigned long long mn = ~0ull;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (!(fl[i] & F_ACTIVE)) continue;
        const unsigned long long k = key_of(mg[i]);
        if (k <= v) ++le;
        else mn = k < mn ? k : mn;
    }
    for (int o = 16; o > 0; o >>= 1) {
        le += __shfl_xor_sync(0xffffffffu, le, o);
        const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mn, o);
        mn = m2 < mn ? m2 : mn;
    }
    if ((threadIdx.x & 31) == 0) {
        if (le) atomicAdd((unsigned long long *)&st->count_le, (unsigned long long)le);
        if (mn != ~0ull) atomicMin(&st->min_gt, mn);
    }
}

// The threshold: max(lerp(prev, next, gamma), grad_floor), numpy's _lerp.
__global__ void threshold_kernel(RefineState *st, double grad_floor) {
    if (st->q_prev == -2) { st->thresh = 1.0 / 0.0; return; }  // no active rows: nothing splits
    const double a = __longlong_as_double((long long)st->prefix);
    double b = a;
    if (st->q_prev >= 0 && st->count_le <= st->q_prev + 1 && st->min_gt != ~0ull)
        b = __longlong_as_double((long long)st->min_gt);
    const double t = st->q_gamma;
    const double d = b - a;
    double r = a + d * t;
    if (t >= 0.5) r = b - d * (1.0 - t);
    st->thresh = r > grad_floor ? r : grad_floor;  // max(float(q), grad_floor)
}

// select_split candidates (densify.py:54-57)
__global__ void candidate_kernel(int n, const double *__restrict__ mg, uint8_t *__restrict__ fl,
                                 const float *__restrict__ ls, const double *__restrict__ mnd, RefineState *st) {
    const double th = st->thresh;
    long long c = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint8_t f = fl[i];
        if ((f & F_KEEP) && mg[i] >= th && (double)scale_max_f32(ls, i) > mnd[i]) {
            f |= F_CAND | F_CHOSEN;
            ++c;
        }
        fl[i] = f;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long *)&st->counts[C_CAND], (unsigned long long)c);
}

// budget = max_surfels - kept (densify.py:186-198)
__global__ void budget_setup_kernel(RefineState *st, long long max_surfels) {
    const long long kept = st->counts[C_KEPT], cand = st->counts[C_CAND];
    const long long budget = max_surfels - kept;
    st->prefix = st->mask = 0ull;
    st->budget_on = cand > budget ? 1 : 0;
    st->allowed = budget > 0 ? budget : 0;
    // the allowed-th largest = ascending rank cand - allowed
    st->rank = st->budget_on && st->allowed > 0 ? cand - st->allowed : 0;
}

// Budget cut: keep candidates above the cut value, and the first need_eq of
// those equal to it in index order (stable argsort of -mean_grad).
__global__ void budget_mark_kernel(int n, const double *__restrict__ mg, uint8_t *__restrict__ fl, RefineState *st) {
    if (!st->budget_on) return;
    const bool none = st->allowed == 0;
    const unsigned long long v = st->prefix;
    long long gt = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint8_t f = fl[i];
        if (!(f & F_CAND)) continue;
        f &= ~(F_CHOSEN | F_EQ);
        if (!none) {
            const unsigned long long k = key_of(mg[i]);
            if (k > v) { f |= F_CHOSEN; ++gt; }
            else if (k == v) f |= F_EQ;
        }
        fl[i] = f;
    }
    for (int o = 16; o > 0; o >>= 1) gt += __shfl_xor_sync(0xffffffffu, gt, o);
    if ((threadIdx.x & 31) == 0 && gt) atomicAdd((unsigned long long *)&st->counts[C_GT], (unsigned long long)gt);
}

// ---- three-kernel scan over fixed blocks of kScanBlock rows -------------
// mode 0: rank of the F_EQ rows (tie break of the budget cut);
// mode 1: ranks of the stay rows (keep & !chosen) and of the split rows.
__device__ __forceinline__ int2 scan_flags(uint8_t f, int mode) {
    if (mode == 0) return make_int2((f & F_EQ) ? 1 : 0, 0);
    const bool keep = f & F_KEEP, chosen = f & F_CHOSEN;
    return make_int2(keep && !chosen ? 1 : 0, chosen ? 1 : 0);
}

__global__ void __launch_bounds__(kThreads) scan_count_kernel(int n, const uint8_t *__restrict__ fl, int mode,
                                                              const RefineState *st, int2 *__restrict__ bsum) {
    if (mode == 0 && !st->budget_on) return;
    const int b = blockIdx.x;
    int2 c = make_int2(0, 0);
    for (int k = threadIdx.x; k < kScanBlock; k += kThreads) {
        const int i = b * kScanBlock + k;
        if (i < n) {
            const int2 f = scan_flags(fl[i], mode);
            c.x += f.x; c.y += f.y;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        c.x += __shfl_xor_sync(0xffffffffu, c.x, o);
        c.y += __shfl_xor_sync(0xffffffffu, c.y, o);
    }
    __shared__ int2 w[kThreads / 32];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int2 t = make_int2(0, 0);
        for (int k = 0; k < kThreads / 32; ++k) { t.x += w[k].x; t.y += w[k].y; }
        bsum[b] = t;
    }
}

// exclusive scan of the block sums (one CTA of 1024 threads, any count)
__global__ void __launch_bounds__(1024) scan_blocks_kernel(int nb, int mode, RefineState *st,
                                                           int2 *__restrict__ bsum) {
    if (mode == 0 && !st->budget_on) return;
    __shared__ long long sx[1024], sy[1024];
    __shared__ long long carry_x, carry_y;
    if (threadIdx.x == 0) { carry_x = 0; carry_y = 0; }
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int b = base + threadIdx.x;
        const int2 v = b < nb ? bsum[b] : make_int2(0, 0);
        sx[threadIdx.x] = v.x; sy[threadIdx.x] = v.y;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const long long ax = threadIdx.x >= o ? sx[threadIdx.x - o] : 0, ay = threadIdx.x >= o ? sy[threadIdx.x - o] : 0;
            __syncthreads();
            sx[threadIdx.x] += ax; sy[threadIdx.x] += ay;
            __syncthreads();
        }
        if (b < nb) bsum[b] = make_int2((int)(carry_x + sx[threadIdx.x] - v.x), (int)(carry_y + sy[threadIdx.x] - v.y));
        __syncthreads();
        if (threadIdx.x == 1023) { carry_x += sx[1023]; carry_y += sy[1023]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (mode == 0) {
            st->need_eq = st->allowed - st->counts[C_GT];
        } else {
            st->counts[C_STAY] = carry_x;
            st->counts[C_SPLIT] = carry_y;
            st->counts[C_OUT] = carry_x + 2 * carry_y;
        }
    }
}

// block-local scan + block offset: mode 0 marks the first need_eq F_EQ rows
// chosen; mode 1 writes the destination of every stay row and the rank of
// every split row (kind: 0 removed, 1 stay, 2 split).
__global__ void __launch_bounds__(kThreads) scan_apply_kernel(int n, uint8_t *__restrict__ fl, int mode,
                                                              const RefineState *st, const int2 *__restrict__ boff,
                                                              int32_t *__restrict__ dst, uint8_t *__restrict__ kind) {
    if (mode == 0 && !st->budget_on) return;
    constexpr int PER = kScanBlock / kThreads;  // 4 consecutive rows per thread
    const int b = blockIdx.x;
    const int i0 = b * kScanBlock + threadIdx.x * PER;
    uint8_t f[PER];
    int2 loc = make_int2(0, 0);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        f[k] = i0 + k < n ? fl[i0 + k] : 0;
        const int2 c = scan_flags(f[k], mode);
        loc.x += c.x; loc.y += c.y;
    }
    // exclusive block scan of the per-thread counts
    __shared__ int2 s[kThreads];
    int2 incl = loc;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const int ax = __shfl_up_sync(0xffffffffu, incl.x, o), ay = __shfl_up_sync(0xffffffffu, incl.y, o);
        if (lane >= o) { incl.x += ax; incl.y += ay; }
    }
    if (lane == 31) s[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        int2 acc = make_int2(0, 0);
        for (int k = 0; k < kThreads / 32; ++k) { const int2 t = s[k]; s[k] = acc; acc.x += t.x; acc.y += t.y; }
    }
    __syncthreads();
    int2 run = make_int2(boff[b].x + s[wid].x + incl.x - loc.x, boff[b].y + s[wid].y + incl.y - loc.y);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int i = i0 + k;
        if (i >= n) break;
        const int2 c = scan_flags(f[k], mode);
        if (mode == 0) {
            if (c.x && run.x < st->need_eq) fl[i] = f[k] | F_CHOSEN;
        } else {
            if (c.x) { dst[i] = run.x; kind[i] = 1; }
            else if (c.y) { dst[i] = run.y; kind[i] = 2; }
            else { dst[i] = -1; kind[i] = 0; }
        }
        run.x += c.x; run.y += c.y;
    }
}

// ---- apply: the new rows ---------------------------------------------------
constexpr int kMaxRemap = 32;
struct RemapSet {
    const void *src[kMaxRemap];
    void *dst[kMaxRemap];
    int row_bytes[kMaxRemap];
    int role[kMaxRemap];   // 0 copy to children, 1 zero in children (moments), 2 centres, 3 log scales
    int count;
};

__global__ void apply_kernel(int n, const uint8_t *__restrict__ kind, const int32_t *__restrict__ dst,
                             const float *__restrict__ centers, const float *__restrict__ quats,
                             const float *__restrict__ ls, const RefineState *st, RemapSet R,
                             int64_t *__restrict__ index_map) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int k = kind[i];
    if (k == 0) return;
    const long long nstay = st->counts[C_STAY], nsplit = st->counts[C_SPLIT];
    long long rows[2];
    int nr;
    if (k == 1) { rows[0] = dst[i]; nr = 1; }
    else { rows[0] = nstay + dst[i]; rows[1] = nstay + nsplit + dst[i]; nr = 2; }
    if (index_map) {
        if (k == 1) index_map[rows[0]] = i;
        else { index_map[rows[0]] = -1; index_map[rows[1]] = -1; }
    }
    // children (split_cloud, densify.py:72-96): +-(s_max / 2) along the
    // longer tangent axis, that axis' scale x 0.7, float64 arithmetic
    double off[3] = {0.0, 0.0, 0.0};
    float cl0 = 0.f, cl1 = 0.f;
    if (k == 2) {
        const double q0 = quats[4 * i], q1 = quats[4 * i + 1], q2 = quats[4 * i + 2], q3 = quats[4 * i + 3];
        const double qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
        const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
        const double u[3] = {1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)};
        const double v[3] = {2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)};
        double s0 = (double)(float)exp((double)ls[2 * i]), s1 = (double)(float)exp((double)ls[2 * i + 1]);
        const bool axis_u = s0 >= s1;
        const double smax = axis_u ? s0 : s1;
        if (axis_u) s0 *= 0.7; else s1 *= 0.7;
        cl0 = (float)log(s0); cl1 = (float)log(s1);
        for (int c = 0; c < 3; ++c) off[c] = (smax / 2.0) * (axis_u ? u[c] : v[c]);
    }
    for (int t = 0; t < R.count; ++t) {
        const int rb = R.row_bytes[t];
        const char *s = static_cast<const char *>(R.src[t]) + (size_t)i * rb;
        for (int h = 0; h < nr; ++h) {
            char *d = static_cast<char *>(R.dst[t]) + (size_t)rows[h] * rb;
            const int role = k == 1 ? 0 : R.role[t];
            if (role == 0) {
                for (int b = 0; b < rb; b += 4) *reinterpret_cast<int *>(d + b) = *reinterpret_cast<const int *>(s + b);
            } else if (role == 1) {
                for (int b = 0; b < rb; b += 4) *reinterpret_cast<int *>(d + b) = 0;
            } else if (role == 2) {
                float *dc = reinterpret_cast<float *>(d);
                const double sg = h == 0 ? 1.0 : -1.0;
                for (int c = 0; c < 3; ++c) dc[c] = (float)((double)centers[3 * i + c] + sg * off[c]);
            } else {
                float *dl = reinterpret_cast<float *>(d);
                dl[0] = cl0; dl[1] = cl1;
            }
        }
    }
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

struct Ws {
    double *mg;
    uint8_t *fl;
    int2 *bsum;
    unsigned int *hist;
    RefineState *st;
};

Ws carve(void *ws, int n) {
    char *p = static_cast<char *>(ws);
    Ws w;
    w.st = reinterpret_cast<RefineState *>(p); p += align256(sizeof(RefineState));
    w.hist = reinterpret_cast<unsigned int *>(p); p += align256(256 * sizeof(unsigned int));
    w.mg = reinterpret_cast<double *>(p); p += align256((size_t)n * sizeof(double));
    w.fl = reinterpret_cast<uint8_t *>(p); p += align256((size_t)n);
    w.bsum = reinterpret_cast<int2 *>(p);
    return w;
}

int select_passes(int n, const Ws &w, uint8_t want, int which, int grid, cudaStream_t s) {
    for (int pass = 0; pass < 8; ++pass) {
        select_hist_kernel<<<grid, 256, 0, s>>>(n, w.mg, w.fl, want, pass, w.st, w.hist);
        select_pick_kernel<<<1, 256, 0, s>>>(pass, w.st, w.hist, which);
    }
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

}  // namespace

extern "C" size_t ss_refine_workspace_bytes(int n) {
    if (n < 0) return 0;
    const size_t nb = ((size_t)n + kScanBlock - 1) / kScanBlock + 1;
    return align256(sizeof(RefineState)) + align256(256 * sizeof(unsigned int)) + align256((size_t)n * 8) +
           align256((size_t)n) + align256(nb * sizeof(int2));
}

extern "C" int ss_refine_plan(int n, const double *grad_sum, const int64_t *view_count, const uint8_t *isolated,
                              const int64_t *outside_votes, const int64_t *front_votes, const float *log_scales,
                              const double *mean_neighbor_dist, int64_t max_surfels, double quantile,
                              double grad_floor, int32_t *dst, uint8_t *kind, int64_t *counts, void *workspace,
                              void *stream) {
    if (n < 0 || !(quantile >= 0.0 && quantile <= 1.0)) return SS_ERR_INVALID;
    if (n > 0 && (!grad_sum || !view_count || !isolated || !log_scales || !mean_neighbor_dist || !dst || !kind ||
                  !counts || !workspace))
        return SS_ERR_INVALID;
    if ((outside_votes == nullptr) != (front_votes == nullptr)) return SS_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    Ws w = carve(workspace, n);
    init_kernel<<<1, 32, 0, s>>>(w.st);
    cudaMemsetAsync(w.hist, 0, 256 * sizeof(unsigned int), s);
    SS_CUDA_CHECK_LAUNCH();
    if (n == 0) {
        cudaMemcpyAsync(counts, w.st->counts, 8 * sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
        return SS_OK;
    }
    const int grid = ss_sm_count() * 4;
    flags_kernel<<<grid, kThreads, 0, s>>>(n, grad_sum, view_count, isolated, outside_votes, front_votes, w.mg, w.fl,
                                           w.st);
    quantile_setup_kernel<<<1, 1, 0, s>>>(w.st, quantile);
    SS_CUDA_CHECK_LAUNCH();
    if (select_passes(n, w, F_ACTIVE, 1, grid, s) != SS_OK) return SS_ERR_CUDA;
    quantile_next_kernel<<<grid, kThreads, 0, s>>>(n, w.mg, w.fl, w.st);
    threshold_kernel<<<1, 1, 0, s>>>(w.st, grad_floor);
    candidate_kernel<<<grid, kThreads, 0, s>>>(n, w.mg, w.fl, log_scales, mean_neighbor_dist, w.st);
    budget_setup_kernel<<<1, 1, 0, s>>>(w.st, (long long)max_surfels);
    SS_CUDA_CHECK_LAUNCH();
    if (select_passes(n, w, F_CAND, 2, grid, s) != SS_OK) return SS_ERR_CUDA;
    budget_mark_kernel<<<grid, kThreads, 0, s>>>(n, w.mg, w.fl, w.st);
    const int nb = (n + kScanBlock - 1) / kScanBlock;
    for (int mode = 0; mode < 2; ++mode) {
        scan_count_kernel<<<nb, kThreads, 0, s>>>(n, w.fl, mode, w.st, w.bsum);
        scan_blocks_kernel<<<1, 1024, 0, s>>>(nb, mode, w.st, w.bsum);
        scan_apply_kernel<<<nb, kThreads, 0, s>>>(n, w.fl, mode, w.st, w.bsum, dst, kind);
    }
    SS_CUDA_CHECK_LAUNCH();
    // counts: [n_out, kept, split, stale, isolated, floater, active, candidates] + threshold bits
    cudaMemcpyAsync(counts, w.st->counts, 8 * sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(counts + 8, &w.st->thresh, sizeof(double), cudaMemcpyDeviceToDevice, s);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_refine_apply(int n, const uint8_t *kind, const int32_t *dst, const float *centers,
                               const float *quats, const float *log_scales, int ntensors, const void *const *src,
                               void *const *dst_tensors, const int *row_bytes, const int *roles, int64_t *index_map,
                               const void *workspace, void *stream) {
    if (n < 0 || ntensors < 0 || ntensors > kMaxRemap) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    if (!kind || !dst || !centers || !quats || !log_scales || !workspace) return SS_ERR_INVALID;
    RemapSet R{};
    R.count = ntensors;
    for (int t = 0; t < ntensors; ++t) {
        if (!src[t] || !dst_tensors[t] || row_bytes[t] <= 0 || row_bytes[t] % 4 || roles[t] < 0 || roles[t] > 3)
            return SS_ERR_INVALID;
        R.src[t] = src[t]; R.dst[t] = dst_tensors[t]; R.row_bytes[t] = row_bytes[t]; R.role[t] = roles[t];
    }
    Ws w = carve(const_cast<void *>(workspace), n);
    apply_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, kind, dst, centers, quats, log_scales, w.st, R,
                                                                      index_map);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
