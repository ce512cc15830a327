// optim.cu -- fused Adam step, quaternion renormalisation and the refinement
// scan helpers (isolation query on a uniform grid, split children).
//
// Reference: Adam.step (adam.py:21-41), normalize_quats after the step
// (train.py:246), prune_keep_mask isolation test (densify.py:118-123, scipy
// cKDTree k=2), split_cloud (densify.py:60-98).  All HBM-streaming kernels.
#include "ss_common.cuh"

namespace {

// S: the moment storage type (double like the reference's numpy state,
// adam.py:26-28, or float); the update is evaluated in float64 either way.
template <typename S>
__global__ void adam_kernel(int64_t count, float *__restrict__ p, const float *__restrict__ g,
                            S *__restrict__ m, S *__restrict__ v, double lr, double b1, double b2,
                            double eps, double c1, double c2) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        const double gg = g[k];
        const double mm = b1 * (double)m[k] + (1.0 - b1) * gg;
        const double vv = b2 * (double)v[k] + (1.0 - b2) * gg * gg;
        m[k] = (S)mm;
        v[k] = (S)vv;
        const double mh = mm / c1, vh = vv / c2;
        p[k] = p[k] - (float)(lr * mh / (sqrt(vh) + eps));
    }
}

__global__ void normalize_quats_kernel(int n, float4 *__restrict__ q) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 a = q[i];
    const float nrm = sqrtf(((a.x * a.x + a.y * a.y) + a.z * a.z) + a.w * a.w);
    if (nrm > 0.f) { a.x /= nrm; a.y /= nrm; a.z /= nrm; a.w /= nrm; }
    q[i] = a;
}

// Multi-tensor Adam: up to kMaxTensors (param, grad, m, v) segments in one
// launch.  A segment flagged `quat` is processed one quaternion (4 floats)
// per thread and renormalised right after its update (train.py:241-246).
constexpr int kMaxTensors = 8;
template <typename S>
struct AdamSeg {
    float *p;
    const float *g;
    S *m, *v;
    int64_t count;      // floats
    int64_t first;      // first work item of the segment
    double lr, c1, c2;  // bias corrections 1 - beta^t
    int quat;
};
template <typename S>
struct AdamMulti {
    AdamSeg<S> seg[kMaxTensors];
    int nseg;
    int64_t items;
    double b1, b2, eps;
};

template <typename S>
__device__ __forceinline__ float adam_one(float p, float g, S *m, S *v, const AdamSeg<S> &s, const AdamMulti<S> &A) {
    const double gg = g;
    const double mm = A.b1 * (double)*m + (1.0 - A.b1) * gg;
    const double vv = A.b2 * (double)*v + (1.0 - A.b2) * gg * gg;
    *m = (S)mm;
    *v = (S)vv;
    const double mh = mm / s.c1, vh = vv / s.c2;
    return p - (float)(s.lr * mh / (sqrt(vh) + A.eps));
}

template <typename S>
__global__ void adam_multi_kernel(AdamMulti<S> A) {
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < A.items;
         it += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (k + 1 < A.nseg && it >= A.seg[k + 1].first) ++k;
        const AdamSeg<S> &s = A.seg[k];
        const int64_t j = it - s.first;
        if (s.quat) {
            float4 p = reinterpret_cast<float4 *>(s.p)[j];
            const float4 g = reinterpret_cast<const float4 *>(s.g)[j];
            S *m = s.m + 4 * j, *v = s.v + 4 * j;
            p.x = adam_one(p.x, g.x, m, v, s, A);
            p.y = adam_one(p.y, g.y, m + 1, v + 1, s, A);
            p.z = adam_one(p.z, g.z, m + 2, v + 2, s, A);
            p.w = adam_one(p.w, g.w, m + 3, v + 3, s, A);
            const float nrm = sqrtf(((p.x * p.x + p.y * p.y) + p.z * p.z) + p.w * p.w);
            if (nrm > 0.f) { p.x /= nrm; p.y /= nrm; p.z /= nrm; p.w /= nrm; }
            reinterpret_cast<float4 *>(s.p)[j] = p;
        } else {
            s.p[j] = adam_one(s.p[j], s.g[j], s.m + j, s.v + j, s, A);
        }
    }
}

// Multi-tensor Adam on float64 MASTER parameters (the reference's fit keeps
// its parameters in float64, train.py:168-174): the update is the
// reference's numpy sequence operation by operation (adam.py:31-41, no
// contraction), quaternions are renormalised in float64 like
// normalize_quats (surfels.py:31-37, train.py:246), and the kernels' float32
// copy is the rounded master value.
struct MasterSeg {
    float *p;
    double *p64;
    const float *g;
    double *m, *v;
    int64_t count, first;
    double lr, c1, c2;
    int quat;
};
struct MasterMulti {
    MasterSeg seg[kMaxTensors];
    int nseg;
    int64_t items;
    double b1, b2, eps;
};

__device__ __forceinline__ double adam_master_one(double p, float g, double *m, double *v, const MasterSeg &s,
                                                  const MasterMulti &A) {
    const double gg = g;
    // m *= b1; m += (1 - b1) g;  v *= b2; v += (1 - b2) g g
    const double mm = __dadd_rn(__dmul_rn(*m, A.b1), __dmul_rn(__dsub_rn(1.0, A.b1), gg));
    const double vv = __dadd_rn(__dmul_rn(*v, A.b2), __dmul_rn(__dmul_rn(__dsub_rn(1.0, A.b2), gg), gg));
    *m = mm;
    *v = vv;
    const double mh = __ddiv_rn(mm, s.c1), vh = __ddiv_rn(vv, s.c2);
    return __dsub_rn(p, __ddiv_rn(__dmul_rn(s.lr, mh), __dadd_rn(__dsqrt_rn(vh), A.eps)));
}

__global__ void adam_master_kernel(MasterMulti A) {
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < A.items;
         it += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (k + 1 < A.nseg && it >= A.seg[k + 1].first) ++k;
        const MasterSeg &s = A.seg[k];
        const int64_t j = it - s.first;
        if (s.quat) {
            double q[4];
            for (int c = 0; c < 4; ++c) q[c] = adam_master_one(s.p64[4 * j + c], s.g[4 * j + c], s.m + 4 * j + c,
                                                               s.v + 4 * j + c, s, A);
            const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q[0], q[0]), __dmul_rn(q[1], q[1])),
                                                              __dmul_rn(q[2], q[2])),
                                                    __dmul_rn(q[3], q[3])));
            if (nrm > 0.0)  // (zero norms are reported by the next preprocess, as the reference raises)
                for (int c = 0; c < 4; ++c) q[c] = __ddiv_rn(q[c], nrm);
            for (int c = 0; c < 4; ++c) { s.p64[4 * j + c] = q[c]; s.p[4 * j + c] = (float)q[c]; }
        } else {
            const double p = adam_master_one(s.p64[j], s.g[j], s.m + j, s.v + j, s, A);
            s.p64[j] = p;
            s.p[j] = (float)p;
        }
    }
}

struct Grid { float ox, oy, oz, cell; int dim; };

__device__ __forceinline__ int axis_cell(float c, float o, float cell, int dim) {
    int k = (int)floorf((c - o) / cell);
    return k < 0 ? 0 : (k >= dim ? dim - 1 : k);
}

// device-resident grid (ss_grid_fit): origin, cell, dim at words 0..4
__device__ __forceinline__ Grid load_grid(const Grid &g, const float *gd) {
    if (!gd) return g;
    return Grid{gd[0], gd[1], gd[2], gd[3], __float_as_int(gd[4])};
}

__device__ __forceinline__ unsigned fkey(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// Grid fit without a host round trip: bounding box of the centres and the
// mean isolation support 3 max(scale) (atomics into words 6..13), then
// cell = max(2 x mean support, extent / 1024), dim = ceil(extent / cell) + 1
// (<= 1024) -- the host version's sizing (densify.py isolation query) with
// the mean instead of the median support.
__global__ void grid_fit_kernel(int n, const float *__restrict__ c, const float *__restrict__ ls, float *gd) {
    unsigned lo[3] = {~0u, ~0u, ~0u}, hi[3] = {0u, 0u, 0u};
    double sup = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        for (int k = 0; k < 3; ++k) {
            const unsigned key = fkey(c[3 * i + k]);
            lo[k] = min(lo[k], key);
            hi[k] = max(hi[k], key);
        }
        const float s0 = (float)exp((double)ls[2 * i]), s1 = (float)exp((double)ls[2 * i + 1]);
        sup += 3.0 * (double)(s0 > s1 ? s0 : s1);
    }
    for (int o = 16; o > 0; o >>= 1) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
        sup += __shfl_xor_sync(0xffffffffu, sup, o);
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned *u = reinterpret_cast<unsigned *>(gd);
        for (int k = 0; k < 3; ++k) { atomicMin(u + 6 + k, lo[k]); atomicMax(u + 9 + k, hi[k]); }
        atomicAdd(reinterpret_cast<double *>(gd + 12), sup);
    }
}

__global__ void grid_finish_kernel(int n, float *gd) {
    const unsigned *u = reinterpret_cast<const unsigned *>(gd);
    float lo[3], ext = 0.f;
    for (int k = 0; k < 3; ++k) {
        lo[k] = fkey_inv(u[6 + k]);
        ext = fmaxf(ext, fkey_inv(u[9 + k]) - lo[k]);
    }
    const double mean_sup = *reinterpret_cast<const double *>(gd + 12) / (double)(n > 0 ? n : 1);
    const float cell = fmaxf(fmaxf((float)(2.0 * mean_sup), ext / 1024.f), 1e-12f);
    int dim = (int)ceilf(ext / cell) + 1;
    dim = dim < 1 ? 1 : (dim > 1024 ? 1024 : dim);
    gd[0] = lo[0]; gd[1] = lo[1]; gd[2] = lo[2]; gd[3] = cell; gd[4] = __int_as_float(dim);
}

__global__ void grid_cells_kernel(int n, const float *__restrict__ c, Grid g0, const float *gd,
                                  int32_t *__restrict__ cell_of) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Grid g = load_grid(g0, gd);
    const int x = axis_cell(c[3 * i], g.ox, g.cell, g.dim), y = axis_cell(c[3 * i + 1], g.oy, g.cell, g.dim),
              z = axis_cell(c[3 * i + 2], g.oz, g.cell, g.dim);
    cell_of[i] = (x * g.dim + y) * g.dim + z;
}

__device__ __forceinline__ int lower_bound(const int32_t *a, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (a[mid] < key) lo = mid + 1; else hi = mid; }
    return lo;
}

__global__ void isolation_kernel(int n, const float *__restrict__ c, const float *__restrict__ ls,
                                 const int32_t *__restrict__ order, const int32_t *__restrict__ sorted_cells, Grid g0,
                                 const float *gd, uint8_t *__restrict__ isolated) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Grid g = load_grid(g0, gd);
    if (n <= 1) { isolated[i] = 0; return; }
    // support = R_CUT * max(scales) with numpy's float32 scales (densify.py:122)
    const float s0 = (float)exp((double)ls[2 * i]), s1 = (float)exp((double)ls[2 * i + 1]);
    const double sup = (double)(3.0f * (s0 > s1 ? s0 : s1));  // float32 like the reference
    const double sup2 = sup * sup;
    const double px = c[3 * i], py = c[3 * i + 1], pz = c[3 * i + 2];
    const int x0 = axis_cell((float)(px - sup), g.ox, g.cell, g.dim), x1 = axis_cell((float)(px + sup), g.ox, g.cell, g.dim);
    const int y0 = axis_cell((float)(py - sup), g.oy, g.cell, g.dim), y1 = axis_cell((float)(py + sup), g.oy, g.cell, g.dim);
    const int z0 = axis_cell((float)(pz - sup), g.oz, g.cell, g.dim), z1 = axis_cell((float)(pz + sup), g.oz, g.cell, g.dim);
    for (int x = x0; x <= x1; ++x)
        for (int y = y0; y <= y1; ++y) {
            const int key0 = (x * g.dim + y) * g.dim + z0, key1 = (x * g.dim + y) * g.dim + z1;
            int k = lower_bound(sorted_cells, n, key0);
            for (; k < n && sorted_cells[k] <= key1; ++k) {
                const int j = order[k];
                if (j == i) continue;
                const double dx = px - c[3 * j], dy = py - c[3 * j + 1], dz = pz - c[3 * j + 2];
                if (sqrt(dx * dx + dy * dy + dz * dz) <= sup) { isolated[i] = 0; return; }
            }
        }
    (void)sup2;
    isolated[i] = 1;
}

__global__ void split_kernel(int ns, const int32_t *__restrict__ parents, const float *__restrict__ centers,
                             const float *__restrict__ quats, const float *__restrict__ ls, float *__restrict__ oc,
                             float *__restrict__ ols, int64_t plus0, int64_t minus0) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ns) return;
    const int p = parents[k];
    const double q0 = quats[4 * p], q1 = quats[4 * p + 1], q2 = quats[4 * p + 2], q3 = quats[4 * p + 3];
    const double qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
    const double u[3] = {1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)};
    const double v[3] = {2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)};
    double s0 = (double)(float)exp((double)ls[2 * p]), s1 = (double)(float)exp((double)ls[2 * p + 1]);
    const bool axis_u = s0 >= s1;
    const double smax = axis_u ? s0 : s1;
    if (axis_u) s0 *= 0.7; else s1 *= 0.7;
    const float l0 = (float)log(s0), l1 = (float)log(s1);
    for (int c = 0; c < 3; ++c) {
        const double off = (smax / 2.0) * (axis_u ? u[c] : v[c]);
        const double cc = centers[3 * p + c];
        oc[3 * (plus0 + k) + c] = (float)(cc + off);
        oc[3 * (minus0 + k) + c] = (float)(cc - off);
    }
    ols[2 * (plus0 + k)] = l0; ols[2 * (plus0 + k) + 1] = l1;
    ols[2 * (minus0 + k)] = l0; ols[2 * (minus0 + k) + 1] = l1;
}

}  // namespace

template <typename S>
static int adam_step(int64_t count, float *param, const float *grad, S *m, S *v, int t, float lr, float beta1,
                     float beta2, float eps, void *stream) {
    if (count < 0 || t < 1 || (count > 0 && (!param || !grad || !m || !v))) return SS_ERR_INVALID;
    if (count == 0) return SS_OK;
    const double c1 = 1.0 - pow((double)beta1, t), c2 = 1.0 - pow((double)beta2, t);
    const int64_t cap = (int64_t)ss_sm_count() * 16;
    const int blocks = (int)((count + 255) / 256 < cap ? (count + 255) / 256 : cap);
    adam_kernel<S><<<blocks, 256, 0, (cudaStream_t)stream>>>(count, param, grad, m, v, lr, beta1, beta2, eps, c1, c2);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_adam_step(int64_t count, float *param, const float *grad, float *m, float *v, int t, float lr,
                            float beta1, float beta2, float eps, void *stream) {
    return adam_step<float>(count, param, grad, m, v, t, lr, beta1, beta2, eps, stream);
}

extern "C" int ss_adam_step_f64(int64_t count, float *param, const float *grad, double *m, double *v, int t,
                                float lr, float beta1, float beta2, float eps, void *stream) {
    return adam_step<double>(count, param, grad, m, v, t, lr, beta1, beta2, eps, stream);
}

template <typename S>
static int adam_multi(int ntensors, float *const *params, const float *const *grads, S *const *m, S *const *v,
                      const int64_t *counts, const int *steps, const float *lrs, const int *quat_flags, float beta1,
                      float beta2, float eps, void *stream) {
    if (ntensors < 1 || ntensors > kMaxTensors || !params || !grads || !m || !v || !counts || !steps || !lrs)
        return SS_ERR_INVALID;
    AdamMulti<S> A{};
    A.nseg = ntensors;
    A.b1 = beta1; A.b2 = beta2; A.eps = eps;
    int64_t items = 0;
    for (int k = 0; k < ntensors; ++k) {
        AdamSeg<S> &sg = A.seg[k];
        sg.p = params[k]; sg.g = grads[k]; sg.m = m[k]; sg.v = v[k];
        sg.count = counts[k];
        sg.quat = quat_flags ? quat_flags[k] : 0;
        if (sg.count < 0 || steps[k] < 1 || (sg.quat && sg.count % 4)) return SS_ERR_INVALID;
        if (sg.count > 0 && (!sg.p || !sg.g || !sg.m || !sg.v)) return SS_ERR_INVALID;
        sg.lr = lrs[k];
        sg.c1 = 1.0 - pow((double)beta1, steps[k]);
        sg.c2 = 1.0 - pow((double)beta2, steps[k]);
        sg.first = items;
        items += sg.quat ? sg.count / 4 : sg.count;
    }
    A.items = items;
    if (items == 0) return SS_OK;
    const int64_t cap = (int64_t)ss_sm_count() * 16;
    const int blocks = (int)((items + 255) / 256 < cap ? (items + 255) / 256 : cap);
    adam_multi_kernel<S><<<blocks, 256, 0, (cudaStream_t)stream>>>(A);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_adam_multi(int ntensors, float *const *params, const float *const *grads, float *const *m,
                             float *const *v, const int64_t *counts, const int *steps, const float *lrs,
                             const int *quat_flags, float beta1, float beta2, float eps, void *stream) {
    return adam_multi<float>(ntensors, params, grads, m, v, counts, steps, lrs, quat_flags, beta1, beta2, eps, stream);
}

extern "C" int ss_adam_multi_f64(int ntensors, float *const *params, const float *const *grads, double *const *m,
                                 double *const *v, const int64_t *counts, const int *steps, const float *lrs,
                                 const int *quat_flags, float beta1, float beta2, float eps, void *stream) {
    return adam_multi<double>(ntensors, params, grads, m, v, counts, steps, lrs, quat_flags, beta1, beta2, eps,
                              stream);
}

extern "C" int ss_adam_multi_master(int ntensors, float *const *params, double *const *masters,
                                    const float *const *grads, double *const *m, double *const *v,
                                    const int64_t *counts, const double *c1s, const double *c2s, const double *lrs,
                                    const int *quat_flags, double beta1, double beta2, double eps, void *stream) {
    if (ntensors < 1 || ntensors > kMaxTensors || !params || !masters || !grads || !m || !v || !counts || !c1s ||
        !c2s || !lrs)
        return SS_ERR_INVALID;
    MasterMulti A{};
    A.nseg = ntensors;
    A.b1 = beta1; A.b2 = beta2; A.eps = eps;
    int64_t items = 0;
    for (int k = 0; k < ntensors; ++k) {
        MasterSeg &sg = A.seg[k];
        sg.p = params[k]; sg.p64 = masters[k]; sg.g = grads[k]; sg.m = m[k]; sg.v = v[k];
        sg.count = counts[k];
        sg.quat = quat_flags ? quat_flags[k] : 0;
        if (sg.count < 0 || (sg.quat && sg.count % 4)) return SS_ERR_INVALID;
        if (sg.count > 0 && (!sg.p || !sg.p64 || !sg.g || !sg.m || !sg.v)) return SS_ERR_INVALID;
        sg.lr = lrs[k]; sg.c1 = c1s[k]; sg.c2 = c2s[k];
        sg.first = items;
        items += sg.quat ? sg.count / 4 : sg.count;
    }
    A.items = items;
    if (items == 0) return SS_OK;
    const int64_t cap = (int64_t)ss_sm_count() * 16;
    const int blocks = (int)((items + 255) / 256 < cap ? (items + 255) / 256 : cap);
    adam_master_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(A);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_normalize_quats(int n, float *quats, void *stream) {
    if (n < 0 || (n > 0 && !quats)) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    normalize_quats_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, reinterpret_cast<float4 *>(quats));
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_grid_cells(int n, const float *centers, const float *origin3, float cell, int dim,
                             int32_t *cell_of, void *stream) {
    if (n < 0 || !origin3 || cell <= 0.f || dim < 1 || dim > 1024) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    Grid g{origin3[0], origin3[1], origin3[2], cell, dim};
    grid_cells_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, centers, g, nullptr, cell_of);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_isolation(int n, const float *centers, const float *log_scales, const int32_t *order,
                            const int32_t *sorted_cells, const float *origin3, float cell, int dim,
                            uint8_t *isolated, void *stream) {
    if (n < 0 || !origin3 || cell <= 0.f || dim < 1 || dim > 1024) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    Grid g{origin3[0], origin3[1], origin3[2], cell, dim};
    isolation_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, centers, log_scales, order, sorted_cells, g,
                                                                         nullptr, isolated);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_grid_fit(int n, const float *centers, const float *log_scales, float *grid, void *stream) {
    if (n < 0 || !grid || (n > 0 && (!centers || !log_scales))) return SS_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    // words 6..8 = ~0 (min keys), 9..11 = 0, 12..13 = 0.0
    cudaMemsetAsync(grid + 6, 0xff, 3 * sizeof(float), s);
    cudaMemsetAsync(grid + 9, 0, 5 * sizeof(float), s);
    if (n > 0) grid_fit_kernel<<<ss_sm_count() * 2, 256, 0, s>>>(n, centers, log_scales, grid);
    grid_finish_kernel<<<1, 1, 0, s>>>(n, grid);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_grid_cells_d(int n, const float *centers, const float *grid, int32_t *cell_of, void *stream) {
    if (n < 0 || !grid || (n > 0 && (!centers || !cell_of))) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    grid_cells_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, centers, Grid{}, grid, cell_of);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_isolation_d(int n, const float *centers, const float *log_scales, const int32_t *order,
                              const int32_t *sorted_cells, const float *grid, uint8_t *isolated, void *stream) {
    if (n < 0 || !grid || (n > 0 && (!centers || !log_scales || !order || !sorted_cells || !isolated)))
        return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    isolation_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, centers, log_scales, order, sorted_cells,
                                                                         Grid{}, grid, isolated);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_split_children(int nsplit, const int32_t *parents, const float *centers, const float *quats,
                                 const float *log_scales, float *out_centers, float *out_log_scales,
                                 int64_t plus_row0, int64_t minus_row0, void *stream) {
    if (nsplit < 0) return SS_ERR_INVALID;
    if (nsplit == 0) return SS_OK;
    split_kernel<<<(nsplit + 127) / 128, 128, 0, (cudaStream_t)stream>>>(nsplit, parents, centers, quats, log_scales,
                                                                         out_centers, out_log_scales, plus_row0,
                                                                         minus_row0);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
