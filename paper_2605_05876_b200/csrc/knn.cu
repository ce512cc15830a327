// knn.cu -- oriented K-nearest-neighbour index and the normal-consistency
// loss.
//
// Reference: NeighborIndex.rebuild (knn.py:31-81; scipy cKDTree, float64):
// for every surfel the k nearest OTHER surfels whose normal has a positive
// dot product with its own, in ascending distance, -1 padded; mean_dist =
// the mean distance to them, or the distance to the nearest other surfel of
// any orientation when none qualifies (1.0 for clouds of <= 1 surfel).
// normal_consistency_loss (losses.py:189-220): L = sum_ij w_ij (1 - n_i.n_j)
// / (N k), w_ij = exp(-|c_i - c_j|^2 / (2 sigma_i^2)), gradients through the
// normals only, mapped to quaternion gradients (surfels.py:54-77).
//
// B200 mapping: a uniform grid over the centres (cells sorted by the caller,
// the isolation query's grid of optim.cu), one thread per surfel expanding
// cube shells of cells around its own until the k-th accepted distance is
// within the shell radius (nothing unvisited can be closer); the top-k list
// lives in registers (insertion by (distance, index)).  The loss scatters the
// symmetric normal term with float64 atomics.
#include "ss_common.cuh"

namespace {

constexpr int kMaxK = 16;

struct KnnGrid { float ox, oy, oz, cell; int dim; };

__device__ __forceinline__ int kaxis(double c, float o, float cell, int dim) {
    int k = (int)floor((c - (double)o) / (double)cell);
    return k < 0 ? 0 : (k >= dim ? dim - 1 : k);
}

__device__ __forceinline__ int klower(const int32_t *a, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid; }
    return lo;
}

// unit normal (third frame column) of a float32 quaternion, float64 (surfels.py:40-51)
__device__ __forceinline__ void quat_normal(const float *q4, double n[3]) {
    const double q0 = q4[0], q1 = q4[1], q2 = q4[2], q3 = q4[3];
    const double qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
    n[0] = 2 * (x * z + w * y);
    n[1] = 2 * (y * z - w * x);
    n[2] = 1 - 2 * (x * x + y * y);
}

template <int K>
__global__ void __launch_bounds__(128) knn_kernel(int n, const float *__restrict__ c, const float *__restrict__ q,
                                                  const int32_t *__restrict__ order,
                                                  const int32_t *__restrict__ sorted_cells, KnnGrid g, int k,
                                                  int64_t *__restrict__ neighbors, double *__restrict__ mean_dist) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double px = c[3 * i], py = c[3 * i + 1], pz = c[3 * i + 2];
    double ni[3];
    quat_normal(q + 4 * i, ni);
    double bd[K];
    int bj[K];
    int cnt = 0;
    double any_d = 1e300;  // nearest other surfel of any orientation (the fallback scale)
    int any_j = 0x7fffffff;
    const int cx = kaxis(px, g.ox, g.cell, g.dim), cy = kaxis(py, g.oy, g.cell, g.dim), cz = kaxis(pz, g.oz, g.cell, g.dim);
    auto visit = [&](int x, int y, int z0, int z1) {
        const int base = (x * g.dim + y) * g.dim;
        for (int t = klower(sorted_cells, n, base + z0); t < n && __ldg(sorted_cells + t) <= base + z1; ++t) {
            const int j = __ldg(order + t);
            if (j == i) continue;
            const double dx = px - c[3 * j], dy = py - c[3 * j + 1], dz = pz - c[3 * j + 2];
            const double d = sqrt(dx * dx + dy * dy + dz * dz);
            if (d < any_d || (d == any_d && j < any_j)) { any_d = d; any_j = j; }
            double nj[3];
            quat_normal(q + 4 * j, nj);
            if (!((ni[0] * nj[0] + ni[1] * nj[1]) + ni[2] * nj[2] > 0.0)) continue;
            if (cnt == k && !(d < bd[k - 1] || (d == bd[k - 1] && j < bj[k - 1]))) continue;
            // insertion by (distance, index)
            int s = cnt < k ? cnt++ : k - 1;
            while (s > 0 && (bd[s - 1] > d || (bd[s - 1] == d && bj[s - 1] > j))) {
                bd[s] = bd[s - 1];
                bj[s] = bj[s - 1];
                --s;
            }
            bd[s] = d;
            bj[s] = j;
        }
    };
    for (int r = 0;; ++r) {
        const int x0 = cx - r, x1 = cx + r, y0 = cy - r, y1 = cy + r, z0 = cz - r, z1 = cz + r;
        for (int x = max(x0, 0); x <= min(x1, g.dim - 1); ++x)
            for (int y = max(y0, 0); y <= min(y1, g.dim - 1); ++y) {
                if (x == x0 || x == x1 || y == y0 || y == y1) {
                    visit(x, y, max(z0, 0), min(z1, g.dim - 1));
                } else {
                    if (z0 >= 0) visit(x, y, z0, z0);
                    if (z1 < g.dim && z1 != z0) visit(x, y, z1, z1);
                }
            }
        // every unvisited surfel lies farther than r cells from this one
        const double reach = (double)r * (double)g.cell;
        const bool covered = x0 <= 0 && y0 <= 0 && z0 <= 0 && x1 >= g.dim - 1 && y1 >= g.dim - 1 && z1 >= g.dim - 1;
        if (covered) break;
        if (cnt == k && bd[k - 1] <= reach) break;  // (a short row keeps searching, like knn.py:60-63)
    }
    double sum = 0.0;
    for (int s = 0; s < k; ++s) {
        neighbors[(size_t)i * k + s] = s < cnt ? (int64_t)bj[s] : (int64_t)-1;
        if (s < cnt) sum += bd[s];
    }
    mean_dist[i] = cnt > 0 ? sum / cnt : any_d;
}

__global__ void nc_kernel(int n, int k, const float *__restrict__ c, const float *__restrict__ q,
                          const int64_t *__restrict__ nb, const double *__restrict__ sigma, double inv_count,
                          double *__restrict__ g_n, double *__restrict__ loss) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    if (i < n) {
        double ni[3];
        quat_normal(q + 4 * i, ni);
        const double px = c[3 * i], py = c[3 * i + 1], pz = c[3 * i + 2];
        const double s = fmax(sigma[i], 1e-12);
        const double inv2s2 = 1.0 / (2.0 * s * s);
        double gi0 = 0.0, gi1 = 0.0, gi2 = 0.0;
        for (int t = 0; t < k; ++t) {
            const int64_t j = nb[(size_t)i * k + t];
            if (j < 0) continue;
            const double dx = px - c[3 * j], dy = py - c[3 * j + 1], dz = pz - c[3 * j + 2];
            const double w = exp(-(dx * dx + dy * dy + dz * dz) * inv2s2);
            double nj[3];
            quat_normal(q + 4 * j, nj);
            acc += w * (1.0 - ((ni[0] * nj[0] + ni[1] * nj[1]) + ni[2] * nj[2]));
            const double wk = w * inv_count;
            gi0 -= wk * nj[0]; gi1 -= wk * nj[1]; gi2 -= wk * nj[2];
            atomicAdd(g_n + 3 * j, -wk * ni[0]);
            atomicAdd(g_n + 3 * j + 1, -wk * ni[1]);
            atomicAdd(g_n + 3 * j + 2, -wk * ni[2]);
        }
        atomicAdd(g_n + 3 * i, gi0);
        atomicAdd(g_n + 3 * i + 1, gi1);
        atomicAdd(g_n + 3 * i + 2, gi2);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(loss, acc * inv_count);
}

// quat_frame_backward with only the normal column (surfels.py:54-77)
__global__ void nc_quat_kernel(int n, const float *__restrict__ q, const double *__restrict__ g_n,
                               float *__restrict__ g_q) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double q0 = q[4 * i], q1 = q[4 * i + 1], q2 = q[4 * i + 2], q3 = q[4 * i + 3];
    const double qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
    const double a = g_n[3 * i], b = g_n[3 * i + 1], cc = g_n[3 * i + 2];
    const double gw = a * (2 * y) + b * (-2 * x);
    const double gx = a * (2 * z) + b * (-2 * w) + cc * (-4 * x);
    const double gy = a * (2 * w) + b * (2 * z) + cc * (-4 * y);
    const double gz = a * (2 * x) + b * (2 * y);
    const double radial = ((gw * w + gx * x) + gy * y) + gz * z;
    g_q[4 * i] = (float)((gw - radial * w) / qn);
    g_q[4 * i + 1] = (float)((gx - radial * x) / qn);
    g_q[4 * i + 2] = (float)((gy - radial * y) / qn);
    g_q[4 * i + 3] = (float)((gz - radial * z) / qn);
}

}  // namespace

extern "C" int ss_knn_oriented(int n, const float *centers, const float *quats, const int32_t *order,
                               const int32_t *sorted_cells, const float *origin3, float cell, int dim, int k,
                               int64_t *neighbors, double *mean_dist, void *stream) {
    if (n < 0 || k < 1 || k > kMaxK || !origin3 || !(cell > 0.f) || dim < 1 || dim > 1024) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    if (!centers || !quats || !order || !sorted_cells || !neighbors || !mean_dist) return SS_ERR_INVALID;
    KnnGrid g{origin3[0], origin3[1], origin3[2], cell, dim};
    knn_kernel<kMaxK><<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, centers, quats, order, sorted_cells, g, k,
                                                                         neighbors, mean_dist);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_normal_consistency(int n, int k, const float *centers, const float *quats, const int64_t *neighbors,
                                     const double *mean_dist, double *loss, double *g_normals, float *g_quats,
                                     void *stream) {
    if (n < 0 || k < 1) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    if (!centers || !quats || !neighbors || !mean_dist || !loss || !g_normals || !g_quats) return SS_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(loss, 0, sizeof(double), st);
    cudaMemsetAsync(g_normals, 0, 3 * sizeof(double) * (size_t)n, st);
    nc_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, k, centers, quats, neighbors, mean_dist,
                                              1.0 / ((double)n * (double)k), g_normals, loss);
    SS_CUDA_CHECK_LAUNCH();
    nc_quat_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, quats, g_normals, g_quats);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
