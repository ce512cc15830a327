// grid.cu -- a dense uniform cell grid over the surfel centres for the
// neighbour queries of the refinement pass and the oriented KNN index
// (densify.py:118-123 isolation, knn.py:31-81 NeighborIndex.rebuild; the
// reference uses scipy cKDTree for both).
//
// B200 mapping: no host round trip and no binary searches.  The bounding box
// and the grid parameters are reduced on the device; a counting sort
// (atomic cell counts, a three-kernel exclusive scan over dim^3 cells,
// scatter) yields per-cell [start, end) ranges in a dense table, so a query
// reads its cells' ranges directly.  Queries run in cell order (thread t
// takes the t-th surfel of the sorted order), so a warp's lanes probe
// neighbouring cells and share their loads through L1.  dim is chosen by
// the caller (~sqrt(n / 24): a surface sampling puts a few tens of surfels
// in each occupied cell, and the k nearest usually lie within one shell).
//
// grid words: [0..2] origin, [3] cell (float bits), [4] dim, [5..7] scratch
// (bbox keys), [8..15] scratch, then starts[0 .. dim^3] (int32).
#include "ss_common.cuh"

namespace {

constexpr int kScan = 1024;  // cells per scan block

__device__ __forceinline__ unsigned okey(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float okey_inv(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

struct Grid {
    float ox, oy, oz, cell;
    int dim;
};

__device__ __forceinline__ Grid read_grid(const int32_t *gw) {
    const float *f = reinterpret_cast<const float *>(gw);
    return Grid{f[0], f[1], f[2], f[3], gw[4]};
}

__device__ __forceinline__ int gaxis(double c, float o, float cell, int dim) {
    int k = (int)floor((c - (double)o) / (double)cell);
    return k < 0 ? 0 : (k >= dim ? dim - 1 : k);
}

__global__ void bbox_kernel(int n, const float *__restrict__ c, int32_t *gw) {
    unsigned lo[3] = {~0u, ~0u, ~0u}, hi[3] = {0u, 0u, 0u};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int k = 0; k < 3; ++k) {
            const unsigned key = okey(c[3 * i + k]);
            lo[k] = min(lo[k], key);
            hi[k] = max(hi[k], key);
        }
    for (int o = 16; o > 0; o >>= 1)
        for (int k = 0; k < 3; ++k) {
            lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
    if ((threadIdx.x & 31) == 0) {
        unsigned *u = reinterpret_cast<unsigned *>(gw);
        for (int k = 0; k < 3; ++k) { atomicMin(u + 5 + k, lo[k]); atomicMax(u + 8 + k, hi[k]); }
    }
}

// cubic cells: cell = (largest extent) / dim, padded so the maximum lands
// inside the last cell
__global__ void grid_params_kernel(int32_t *gw, int dim) {
    const unsigned *u = reinterpret_cast<const unsigned *>(gw);
    float lo[3], ext = 0.f;
    for (int k = 0; k < 3; ++k) {
        lo[k] = okey_inv(u[5 + k]);
        ext = fmaxf(ext, okey_inv(u[8 + k]) - lo[k]);
    }
    float *f = reinterpret_cast<float *>(gw);
    const float cell = fmaxf(ext * (1.f + 1e-5f), 1e-30f) / (float)dim;
    f[0] = lo[0]; f[1] = lo[1]; f[2] = lo[2]; f[3] = cell;
    gw[4] = dim;
}

__global__ void cell_count_kernel(int n, const float *__restrict__ c, int32_t *gw, int32_t *__restrict__ cell_of) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Grid g = read_grid(gw);
    const int x = gaxis(c[3 * i], g.ox, g.cell, g.dim), y = gaxis(c[3 * i + 1], g.oy, g.cell, g.dim),
              z = gaxis(c[3 * i + 2], g.oz, g.cell, g.dim);
    const int cid = (x * g.dim + y) * g.dim + z;
    cell_of[i] = cid;
    atomicAdd(gw + 16 + cid, 1);
}

__global__ void __launch_bounds__(256) scan_sum_kernel(int m, const int32_t *__restrict__ v, int32_t *__restrict__ bsum) {
    int s = 0;
    for (int k = threadIdx.x; k < kScan; k += 256) {
        const int i = blockIdx.x * kScan + k;
        if (i < m) s += v[i];
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ int w[8];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int k = 0; k < 8; ++k) t += w[k];
        bsum[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) scan_blocks_kernel(int nb, int32_t *__restrict__ bsum) {
    __shared__ int s[1024];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int b = base + threadIdx.x;
        const int v = b < nb ? bsum[b] : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const int a = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
            __syncthreads();
            s[threadIdx.x] += a;
            __syncthreads();
        }
        if (b < nb) bsum[b] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += s[1023];
        __syncthreads();
    }
}

// in place: counts -> exclusive starts (+ block offsets); the last entry
// (index m) receives the total
__global__ void __launch_bounds__(256) scan_apply_kernel(int m, int32_t *__restrict__ v,
                                                         const int32_t *__restrict__ boff, int n) {
    constexpr int PER = kScan / 256;
    const int i0 = blockIdx.x * kScan + threadIdx.x * PER;
    int x[PER], loc = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) { x[k] = i0 + k < m ? v[i0 + k] : 0; loc += x[k]; }
    int incl = loc;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += a;
    }
    __shared__ int ws[8];
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int k = 0; k < 8; ++k) { const int t = ws[k]; ws[k] = acc; acc += t; }
    }
    __syncthreads();
    int run = boff[blockIdx.x] + ws[wid] + incl - loc;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        if (i0 + k < m) v[i0 + k] = run;
        run += x[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) v[m] = n;
}

__global__ void cell_scatter_kernel(int n, const int32_t *__restrict__ cell_of, const int32_t *__restrict__ starts,
                                    int32_t *__restrict__ cursor, int32_t *__restrict__ order) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int cid = cell_of[i];
    order[starts[cid] + atomicAdd(cursor + cid, 1)] = i;
}

// ---- oriented KNN (knn.py:31-81) on the dense grid ------------------------
constexpr int kMaxK = 16;

__device__ __forceinline__ void quat_normal(const float *q4, double n[3]) {
    const double q0 = q4[0], q1 = q4[1], q2 = q4[2], q3 = q4[3];
    const double qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
    n[0] = 2 * (x * z + w * y);
    n[1] = 2 * (y * z - w * x);
    n[2] = 1 - 2 * (x * x + y * y);
}

template <int K>
__global__ void __launch_bounds__(128) knn_dense_kernel(int n, const float *__restrict__ c, const float *__restrict__ q,
                                                        const int32_t *__restrict__ gw,
                                                        const int32_t *__restrict__ order, int k,
                                                        int64_t *__restrict__ neighbors,
                                                        double *__restrict__ mean_dist) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = __ldg(order + t);  // cell order: a warp's queries are neighbours
    const Grid g = read_grid(gw);
    const int32_t *starts = gw + 16;
    const double px = c[3 * i], py = c[3 * i + 1], pz = c[3 * i + 2];
    double ni[3];
    quat_normal(q + 4 * i, ni);
    double bd[K];
    int bj[K];
    int cnt = 0;
    double any_d = 1e300;  // nearest other surfel of any orientation (the fallback scale)
    int any_j = 0x7fffffff;
    const int cx = gaxis(px, g.ox, g.cell, g.dim), cy = gaxis(py, g.oy, g.cell, g.dim), cz = gaxis(pz, g.oz, g.cell, g.dim);
    auto visit_cell = [&](int cid) {
        const int s1 = __ldg(starts + cid + 1);
        for (int s = __ldg(starts + cid); s < s1; ++s) {
            const int j = __ldg(order + s);
            if (j == i) continue;
            const double dx = px - c[3 * j], dy = py - c[3 * j + 1], dz = pz - c[3 * j + 2];
            const double d = sqrt(dx * dx + dy * dy + dz * dz);
            if (d < any_d || (d == any_d && j < any_j)) { any_d = d; any_j = j; }
            if (cnt == k && !(d < bd[k - 1] || (d == bd[k - 1] && j < bj[k - 1]))) continue;
            double nj[3];
            quat_normal(q + 4 * j, nj);
            if (!((ni[0] * nj[0] + ni[1] * nj[1]) + ni[2] * nj[2] > 0.0)) continue;
            int sl = cnt < k ? cnt++ : k - 1;  // insertion by (distance, index)
            while (sl > 0 && (bd[sl - 1] > d || (bd[sl - 1] == d && bj[sl - 1] > j))) {
                bd[sl] = bd[sl - 1];
                bj[sl] = bj[sl - 1];
                --sl;
            }
            bd[sl] = d;
            bj[sl] = j;
        }
    };
    for (int r = 0;; ++r) {
        const int x0 = cx - r, x1 = cx + r, y0 = cy - r, y1 = cy + r, z0 = cz - r, z1 = cz + r;
        for (int x = max(x0, 0); x <= min(x1, g.dim - 1); ++x)
            for (int y = max(y0, 0); y <= min(y1, g.dim - 1); ++y) {
                const int base = (x * g.dim + y) * g.dim;
                if (x == x0 || x == x1 || y == y0 || y == y1) {
                    for (int z = max(z0, 0); z <= min(z1, g.dim - 1); ++z) visit_cell(base + z);
                } else {
                    if (z0 >= 0) visit_cell(base + z0);
                    if (z1 < g.dim && z1 != z0) visit_cell(base + z1);
                }
            }
        // every unvisited surfel lies more than r cells (r * cell) away
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

// ---- isolation (densify.py:118-123) on the dense grid ----------------------
__global__ void __launch_bounds__(128) isolation_dense_kernel(int n, const float *__restrict__ c,
                                                              const float *__restrict__ ls,
                                                              const int32_t *__restrict__ gw,
                                                              const int32_t *__restrict__ order,
                                                              uint8_t *__restrict__ isolated) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = __ldg(order + t);
    if (n <= 1) { isolated[i] = 0; return; }
    const Grid g = read_grid(gw);
    const int32_t *starts = gw + 16;
    // support = R_CUT * max(scales) with the float32 scales of the cloud (densify.py:122)
    const float s0 = (float)exp((double)ls[2 * i]), s1 = (float)exp((double)ls[2 * i + 1]);
    const double sup = (double)(3.0f * (s0 > s1 ? s0 : s1));
    const double px = c[3 * i], py = c[3 * i + 1], pz = c[3 * i + 2];
    const int x0 = gaxis(px - sup, g.ox, g.cell, g.dim), x1 = gaxis(px + sup, g.ox, g.cell, g.dim);
    const int y0 = gaxis(py - sup, g.oy, g.cell, g.dim), y1 = gaxis(py + sup, g.oy, g.cell, g.dim);
    const int z0 = gaxis(pz - sup, g.oz, g.cell, g.dim), z1 = gaxis(pz + sup, g.oz, g.cell, g.dim);
    // an existence query: the surfel's own cell first (its nearest
    // neighbours almost always share it), then the rest of the ball's cells
    auto near_in = [&](int cid) {
        const int s1e = __ldg(starts + cid + 1);
        for (int s = __ldg(starts + cid); s < s1e; ++s) {
            const int j = __ldg(order + s);
            if (j == i) continue;
            const double dx = px - c[3 * j], dy = py - c[3 * j + 1], dz = pz - c[3 * j + 2];
            if (sqrt(dx * dx + dy * dy + dz * dz) <= sup) return true;
        }
        return false;
    };
    const int cx = gaxis(px, g.ox, g.cell, g.dim), cy = gaxis(py, g.oy, g.cell, g.dim), cz = gaxis(pz, g.oz, g.cell, g.dim);
    const int own = (cx * g.dim + cy) * g.dim + cz;
    if (near_in(own)) { isolated[i] = 0; return; }
    for (int x = x0; x <= x1; ++x)
        for (int y = y0; y <= y1; ++y)
            for (int z = z0; z <= z1; ++z) {
                const int cid = (x * g.dim + y) * g.dim + z;
                if (cid != own && near_in(cid)) { isolated[i] = 0; return; }
            }
    isolated[i] = 1;
}

}  // namespace

extern "C" size_t ss_cell_grid_words(int n, int dim) {
    if (n < 0 || dim < 1 || dim > 512) return 0;
    const size_t cells = (size_t)dim * dim * dim;
    const size_t nb = (cells + kScan - 1) / kScan;
    // params + starts (cells + 1) + block sums + cursors (cells) + cell of (n) + order (n)
    return 16 + (cells + 1) + nb + cells + 2 * (size_t)n;
}

extern "C" int ss_cell_grid_build(int n, const float *centers, int dim, int32_t *grid, void *stream) {
    if (n < 0 || dim < 1 || dim > 512 || !grid || (n > 0 && !centers)) return SS_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t cells = (size_t)dim * dim * dim;
    const int nb = (int)((cells + kScan - 1) / kScan);
    int32_t *starts = grid + 16, *bsum = starts + cells + 1, *cursor = bsum + nb, *cell_of = cursor + cells,
            *order = cell_of + n;
    cudaMemsetAsync(grid + 5, 0xff, 3 * sizeof(int32_t), s);  // bbox min keys
    cudaMemsetAsync(grid + 8, 0, 3 * sizeof(int32_t), s);     // bbox max keys
    cudaMemsetAsync(starts, 0, (cells + 1) * sizeof(int32_t), s);
    cudaMemsetAsync(cursor, 0, cells * sizeof(int32_t), s);
    if (n > 0) bbox_kernel<<<ss_sm_count() * 2, 256, 0, s>>>(n, centers, grid);
    grid_params_kernel<<<1, 1, 0, s>>>(grid, dim);
    if (n > 0) cell_count_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, centers, grid, cell_of);
    scan_sum_kernel<<<nb, 256, 0, s>>>((int)cells, starts, bsum);
    scan_blocks_kernel<<<1, 1024, 0, s>>>(nb, bsum);
    scan_apply_kernel<<<nb, 256, 0, s>>>((int)cells, starts, bsum, n);
    if (n > 0) cell_scatter_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, cell_of, starts, cursor, order);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

static const int32_t *grid_order(const int32_t *grid, int n, int dim) {
    const size_t cells = (size_t)dim * dim * dim;
    const size_t nb = (cells + kScan - 1) / kScan;
    return grid + 16 + (cells + 1) + nb + cells + n;
}

extern "C" int ss_knn_dense(int n, const float *centers, const float *quats, const int32_t *grid, int dim, int k,
                            int64_t *neighbors, double *mean_dist, void *stream) {
    if (n < 0 || k < 1 || k > kMaxK || dim < 1 || dim > 512 || !grid) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    if (!centers || !quats || !neighbors || !mean_dist) return SS_ERR_INVALID;
    knn_dense_kernel<kMaxK><<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
        n, centers, quats, grid, grid_order(grid, n, dim), k, neighbors, mean_dist);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_isolation_dense(int n, const float *centers, const float *log_scales, const int32_t *grid, int dim,
                                  uint8_t *isolated, void *stream) {
    if (n < 0 || dim < 1 || dim > 512 || !grid) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    if (!centers || !log_scales || !isolated) return SS_ERR_INVALID;
    isolation_dense_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, centers, log_scales, grid,
                                                                              grid_order(grid, n, dim), isolated);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
