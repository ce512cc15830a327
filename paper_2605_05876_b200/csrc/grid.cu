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

__global__ void cell_scatter_kernel(int n, const float *__restrict__ c, const int32_t *__restrict__ cell_of,
                                    const int32_t *__restrict__ starts, int32_t *__restrict__ cursor,
                                    int32_t *__restrict__ order, float4 *__restrict__ pk) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int cid = cell_of[i];
    const int at = starts[cid] + atomicAdd(cursor + cid, 1);
    order[at] = i;
    pk[at] = make_float4(c[3 * i], c[3 * i + 1], c[3 * i + 2], __int_as_float(i));
}

// ---- oriented KNN (knn.py:31-81) on the dense grid ------------------------
// The candidates of a query stream from the grid's cell-ordered copy of the
// centres (float4: x, y, z, source index) and a cell-ordered float64 normal
// table built once per call, so the inner loop is a broadcast load, a
// float64 squared distance and a compare against the current k-th best; the
// k best (squared distance, index) pairs live in registers (K is a template
// parameter: the insertion is unrolled, no local-memory arrays).  Ordering
// by the squared distance is cKDTree's own (it compares squared distances
// and takes the root of the results).
constexpr int kMaxK = 16;

// quat_to_frame's normal column (surfels.py:40-51), float64 without contraction
__device__ __forceinline__ void quat_normal(const float *q4, double n[3]) {
    const double q0 = q4[0], q1 = q4[1], q2 = q4[2], q3 = q4[3];
    const double qn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q0, q0), __dmul_rn(q1, q1)), __dmul_rn(q2, q2)),
                                           __dmul_rn(q3, q3)));
    const double w = __ddiv_rn(q0, qn), x = __ddiv_rn(q1, qn), y = __ddiv_rn(q2, qn), z = __ddiv_rn(q3, qn);
    n[0] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
    n[1] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
    n[2] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y))));
}

// cell-ordered float64 normals of the query pass
__global__ void knn_normals_kernel(int n, const float *__restrict__ q, const int32_t *__restrict__ order,
                                   double4 *__restrict__ nrm) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double v[3];
    quat_normal(q + 4 * (size_t)__ldg(order + t), v);
    nrm[t] = make_double4(v[0], v[1], v[2], 0.0);
}

__device__ __forceinline__ double sqdist(double px, double py, double pz, float4 c) {
    const double dx = __dsub_rn(px, (double)c.x), dy = __dsub_rn(py, (double)c.y), dz = __dsub_rn(pz, (double)c.z);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// (d, j) before (e, k): by distance, then index
__device__ __forceinline__ bool before(double d, int j, double e, int k) { return d < e || (d == e && j < k); }

// The k best (squared distance, index) pairs of one query in registers,
// plus the nearest surfel of any orientation (the fallback scale).
template <int K>
struct TopK {
    double bd[K];
    int bj[K];
    double any_d;
    int any_j;
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int s = 0; s < K; ++s) { bd[s] = INFINITY; bj[s] = 0x7fffffff; }
        any_d = INFINITY;
        any_j = 0x7fffffff;
    }
    __device__ __forceinline__ bool full() const { return bj[K - 1] != 0x7fffffff; }
    // unrolled insertion (from the back: bd[m - 1] is still the old value)
    __device__ __forceinline__ void insert(double d, int j) {
#pragma unroll
        for (int m = K - 1; m >= 0; --m) {
            if (before(d, j, bd[m], bj[m])) {
                if (m > 0 && before(d, j, bd[m - 1], bj[m - 1])) { bd[m] = bd[m - 1]; bj[m] = bj[m - 1]; }
                else { bd[m] = d; bj[m] = j; }
            }
        }
    }
    // candidate s of the cell-ordered tables for the query (i, p, ni)
    __device__ __forceinline__ void visit(int i, double px, double py, double pz, const double4 &ni, float4 c,
                                          const double4 *__restrict__ nrm, int s) {
        const int j = __float_as_int(c.w);
        if (j == i) return;
        const double d = sqdist(px, py, pz, c);
        if (before(d, j, any_d, any_j)) { any_d = d; any_j = j; }
        if (!before(d, j, bd[K - 1], bj[K - 1])) return;
        const double4 nj = nrm[s];
        if (!(__dadd_rn(__dadd_rn(__dmul_rn(ni.x, nj.x), __dmul_rn(ni.y, nj.y)), __dmul_rn(ni.z, nj.z)) > 0.0)) return;
        insert(d, j);
    }
    __device__ __forceinline__ void write(int i, int64_t *__restrict__ neighbors, double *__restrict__ mean_dist) const {
        double sum = 0.0;
        int cnt = 0;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            const bool ok = bj[s] != 0x7fffffff;
            neighbors[(size_t)i * K + s] = ok ? (int64_t)bj[s] : (int64_t)-1;
            if (ok) { sum += __dsqrt_rn(bd[s]); ++cnt; }
        }
        mean_dist[i] = cnt > 0 ? sum / cnt : __dsqrt_rn(any_d);
    }
};

// Shells of cells around the query's cell.  A query whose row is not final
// after kMaxShell shells (its k-th oriented neighbour lies far away: a
// surfel facing against its surroundings, an outlier) is deferred to
// knn_far_kernel (a CTA per query, on the coarse grid) instead of expanding
// shells of mostly empty cells one thread at a time (a single such query at
// r ~ 60 visits ~2M cells).
#ifndef SS_KNN_MAX_SHELL
#define SS_KNN_MAX_SHELL 3
#endif
constexpr int kMaxShell = SS_KNN_MAX_SHELL;

template <int K>
__global__ void __launch_bounds__(128) knn_dense_kernel(int n, const int32_t *__restrict__ gw,
                                                        const float4 *__restrict__ pk, const double4 *__restrict__ nrm,
                                                        int64_t *__restrict__ neighbors,
                                                        double *__restrict__ mean_dist, int32_t *__restrict__ defer) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const Grid g = read_grid(gw);
    const int32_t *starts = gw + 16;
    const float4 me = __ldg(pk + t);  // cell order: a warp's queries are neighbours
    const int i = __float_as_int(me.w);
    const double px = me.x, py = me.y, pz = me.z;
    const double4 ni = nrm[t];
    TopK<K> tk;
    tk.init();
    const int cx = gaxis(px, g.ox, g.cell, g.dim), cy = gaxis(py, g.oy, g.cell, g.dim), cz = gaxis(pz, g.oz, g.cell, g.dim);
    auto visit_cell = [&](int cid) {
        const int s1 = __ldg(starts + cid + 1);
        for (int s = __ldg(starts + cid); s < s1; ++s) tk.visit(i, px, py, pz, ni, __ldg(pk + s), nrm, s);
    };
    // distances from the query to its own cell's faces (the block of shell r
    // extends r cells beyond them); faces on the grid boundary bound nothing
    const double cl = g.cell;
    const double fxl = px - ((double)g.ox + cx * cl), fxh = ((double)g.ox + (cx + 1) * cl) - px;
    const double fyl = py - ((double)g.oy + cy * cl), fyh = ((double)g.oy + (cy + 1) * cl) - py;
    const double fzl = pz - ((double)g.oz + cz * cl), fzh = ((double)g.oz + (cz + 1) * cl) - pz;
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
        const bool covered = x0 <= 0 && y0 <= 0 && z0 <= 0 && x1 >= g.dim - 1 && y1 >= g.dim - 1 && z1 >= g.dim - 1;
        if (covered) break;
        // every unvisited surfel lies beyond an interior face of the visited
        // (2r+1)^3 block: at least `reach` away (shrunk by a relative 1e-9 for
        // the rounding of the cell assignment).  A full row whose k-th
        // distance is strictly below it is final (ties could still prefer an
        // unvisited lower index); a short row keeps searching, like knn.py:60-63
        double reach = INFINITY;
        if (x0 > 0) reach = fmin(reach, fxl);
        if (x1 < g.dim - 1) reach = fmin(reach, fxh);
        if (y0 > 0) reach = fmin(reach, fyl);
        if (y1 < g.dim - 1) reach = fmin(reach, fyh);
        if (z0 > 0) reach = fmin(reach, fzl);
        if (z1 < g.dim - 1) reach = fmin(reach, fzh);
        reach = (reach + r * cl) * (1.0 - 1e-9);
        if (tk.full() && tk.bd[K - 1] < reach * reach) break;
        if (r == kMaxShell) {  // far k-th neighbour: the whole-cloud pass
            defer[2 + atomicAdd(defer, 1)] = t;
            return;
        }
    }
    tk.write(i, neighbors, mean_dist);
}

// Deferred queries, one CTA each (taken by a work counter), on a COARSE
// grid of the same centres (cells 4x wider: a far k-th neighbour is a few
// coarse shells away instead of tens of fine ones).  The CTA's threads split
// each shell's cells (the six faces of the (2r+1)^3 block, flattened), keep
// thread-local rows, stop once the smallest thread-local k-th distance lies
// strictly inside the shell's reach (the row's k-th distance can only be
// smaller), and merge the rows pairwise in shared memory in the same
// (distance, index) order -- the row equals the fine search's.
template <int K> __host__ __device__ constexpr int far_threads() { return K > 8 ? 128 : 256; }

// cell of shell r >= 1 number e (0 <= e < 24 r^2 + 2) around (cx, cy, cz)
__device__ __forceinline__ void shell_cell(int r, int e, int cx, int cy, int cz, int &x, int &y, int &z) {
    const int side = 2 * r + 1, inner = 2 * r - 1;
    if (e < 2 * side * side) {  // the two z faces
        const int f = e / (side * side), rem = e - f * side * side;
        x = cx - r + rem / side; y = cy - r + rem % side; z = f ? cz + r : cz - r;
        return;
    }
    e -= 2 * side * side;
    if (e < 2 * side * inner) {  // the two y faces (z inside)
        const int f = e / (side * inner), rem = e - f * side * inner;
        x = cx - r + rem / inner; z = cz - r + 1 + rem % inner; y = f ? cy + r : cy - r;
        return;
    }
    e -= 2 * side * inner;  // the two x faces (y, z inside)
    const int f = e / (inner * inner), rem = e - f * inner * inner;
    y = cy - r + 1 + rem / inner; z = cz - r + 1 + rem % inner; x = f ? cx + r : cx - r;
}

template <int K>
__global__ void __launch_bounds__(far_threads<K>()) knn_far_kernel(const float4 *__restrict__ pk,
                                                                   const double4 *__restrict__ nrm,
                                                                   const int32_t *__restrict__ gwc,
                                                                   const float4 *__restrict__ pkc,
                                                                   const double4 *__restrict__ nrmc,
                                                                   int64_t *__restrict__ neighbors,
                                                                   double *__restrict__ mean_dist,
                                                                   int32_t *__restrict__ defer) {
    constexpr int NT = far_threads<K>();
    __shared__ double sd[NT][K + 1];
    __shared__ int sj[NT][K + 1];
    __shared__ double s_min[NT / 32];
    __shared__ int s_q;
    const Grid g = read_grid(gwc);
    const int32_t *starts = gwc + 16;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_q = atomicAdd(defer + 1, 1);
        __syncthreads();
        const int q = s_q;
        if (q >= defer[0]) return;
        const int t = defer[2 + q];
        const float4 me = __ldg(pk + t);
        const int i = __float_as_int(me.w);
        const double px = me.x, py = me.y, pz = me.z;
        const double4 ni = nrm[t];
        TopK<K> tk;
        tk.init();
        auto visit_cell = [&](int cid) {
            const int s1 = __ldg(starts + cid + 1);
            for (int s = __ldg(starts + cid); s < s1; ++s) tk.visit(i, px, py, pz, ni, __ldg(pkc + s), nrmc, s);
        };
        const int cx = gaxis(px, g.ox, g.cell, g.dim), cy = gaxis(py, g.oy, g.cell, g.dim),
                  cz = gaxis(pz, g.oz, g.cell, g.dim);
        const double cl = g.cell;
        const double fxl = px - ((double)g.ox + cx * cl), fxh = ((double)g.ox + (cx + 1) * cl) - px;
        const double fyl = py - ((double)g.oy + cy * cl), fyh = ((double)g.oy + (cy + 1) * cl) - py;
        const double fzl = pz - ((double)g.oz + cz * cl), fzh = ((double)g.oz + (cz + 1) * cl) - pz;
        for (int r = 0;; ++r) {
            if (r == 0) {
                if (threadIdx.x == 0) visit_cell((cx * g.dim + cy) * g.dim + cz);
            } else {
                const int ncell = 24 * r * r + 2;
                for (int e = threadIdx.x; e < ncell; e += NT) {
                    int x, y, z;
                    shell_cell(r, e, cx, cy, cz, x, y, z);
                    if (x >= 0 && y >= 0 && z >= 0 && x < g.dim && y < g.dim && z < g.dim)
                        visit_cell((x * g.dim + y) * g.dim + z);
                }
            }
            const int x0 = cx - r, x1 = cx + r, y0 = cy - r, y1 = cy + r, z0 = cz - r, z1 = cz + r;
            if (x0 <= 0 && y0 <= 0 && z0 <= 0 && x1 >= g.dim - 1 && y1 >= g.dim - 1 && z1 >= g.dim - 1) break;
            double reach = INFINITY;
            if (x0 > 0) reach = fmin(reach, fxl);
            if (x1 < g.dim - 1) reach = fmin(reach, fxh);
            if (y0 > 0) reach = fmin(reach, fyl);
            if (y1 < g.dim - 1) reach = fmin(reach, fyh);
            if (z0 > 0) reach = fmin(reach, fzl);
            if (z1 < g.dim - 1) reach = fmin(reach, fzh);
            reach = (reach + r * cl) * (1.0 - 1e-9);
            double m = tk.full() ? tk.bd[K - 1] : INFINITY;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) s_min[wid] = m;
            __syncthreads();
            double mm = s_min[0];
#pragma unroll
            for (int w = 1; w < NT / 32; ++w) mm = fmin(mm, s_min[w]);
            __syncthreads();
            if (mm < reach * reach) break;
        }
#pragma unroll
        for (int m = 0; m < K; ++m) { sd[threadIdx.x][m] = tk.bd[m]; sj[threadIdx.x][m] = tk.bj[m]; }
        sd[threadIdx.x][K] = tk.any_d;
        sj[threadIdx.x][K] = tk.any_j;
        for (int half = NT / 2; half > 0; half >>= 1) {
            __syncthreads();
            if (threadIdx.x < half) {  // merge row threadIdx.x + half into row threadIdx.x
                const int o = threadIdx.x + half;
                double md[K];
                int mj[K];
                int a = 0, b = 0;
#pragma unroll
                for (int m = 0; m < K; ++m) {
                    const bool ta = before(sd[threadIdx.x][a], sj[threadIdx.x][a], sd[o][b], sj[o][b]);
                    md[m] = ta ? sd[threadIdx.x][a] : sd[o][b];
                    mj[m] = ta ? sj[threadIdx.x][a] : sj[o][b];
                    a += ta;
                    b += !ta;
                }
#pragma unroll
                for (int m = 0; m < K; ++m) { sd[threadIdx.x][m] = md[m]; sj[threadIdx.x][m] = mj[m]; }
                if (before(sd[o][K], sj[o][K], sd[threadIdx.x][K], sj[threadIdx.x][K])) {
                    sd[threadIdx.x][K] = sd[o][K];
                    sj[threadIdx.x][K] = sj[o][K];
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int m = 0; m < K; ++m) { tk.bd[m] = sd[0][m]; tk.bj[m] = sj[0][m]; }
            tk.any_d = sd[0][K];
            tk.any_j = sj[0][K];
            tk.write(i, neighbors, mean_dist);
        }
    }
}

// ---- isolation (densify.py:118-123) on the dense grid ----------------------
__global__ void __launch_bounds__(128) isolation_dense_kernel(int n, const float *__restrict__ c,
                                                              const float *__restrict__ ls,
                                                              const int32_t *__restrict__ gw,
                                                              const float4 *__restrict__ pk,
                                                              uint8_t *__restrict__ isolated) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = __float_as_int(__ldg(pk + t).w);
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
            const float4 cj = __ldg(pk + s);
            if (__float_as_int(cj.w) == i) continue;
            if (__dsqrt_rn(sqdist(px, py, pz, cj)) <= sup) return true;
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

static size_t pk_offset(size_t cells, size_t nb, int n) {
    return (16 + (cells + 1) + nb + cells + 2 * (size_t)n + 3) & ~(size_t)3;
}

extern "C" size_t ss_cell_grid_words(int n, int dim) {
    if (n < 0 || dim < 1 || dim > 512) return 0;
    const size_t cells = (size_t)dim * dim * dim;
    const size_t nb = (cells + kScan - 1) / kScan;
    // params + starts (cells + 1) + block sums + cursors (cells) + cell of (n) + order (n),
    // then the cell-ordered centres (float4, 16-byte aligned)
    return pk_offset(cells, nb, n) + 4 * (size_t)n;
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
    float4 *pk = reinterpret_cast<float4 *>(grid + pk_offset(cells, nb, n));
    if (n > 0) cell_scatter_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, centers, cell_of, starts, cursor, order, pk);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

static const int32_t *grid_order(const int32_t *grid, int n, int dim) {
    const size_t cells = (size_t)dim * dim * dim;
    const size_t nb = (cells + kScan - 1) / kScan;
    return grid + 16 + (cells + 1) + nb + cells + n;
}

static const float4 *grid_packed(const int32_t *grid, int n, int dim) {
    const size_t cells = (size_t)dim * dim * dim;
    const size_t nb = (cells + kScan - 1) / kScan;
    return reinterpret_cast<const float4 *>(grid + pk_offset(cells, nb, n));
}

template <int K>
static void launch_knn(int n, const int32_t *grid, const float4 *pk, const double4 *nrm, const int32_t *gridc,
                       const float4 *pkc, const double4 *nrmc, int64_t *neighbors, double *mean_dist, int32_t *defer,
                       cudaStream_t s) {
    knn_dense_kernel<K><<<(n + 127) / 128, 128, 0, s>>>(n, grid, pk, nrm, neighbors, mean_dist, defer);
    knn_far_kernel<K><<<ss_sm_count() * 4, far_threads<K>(), 0, s>>>(pk, nrm, gridc, pkc, nrmc, neighbors, mean_dist,
                                                                    defer);
}

extern "C" size_t ss_knn_workspace_bytes(int n) {
    if (n < 0) return 0;
    // the fine and the coarse grid's cell-ordered float64 normals (32 B each),
    // then the deferred-query list (2 counters + n)
    return 64 * (size_t)n + 4 * ((size_t)n + 2);
}

extern "C" int ss_knn_dense(int n, const float *centers, const float *quats, const int32_t *grid, int dim,
                            const int32_t *grid_coarse, int dim_coarse, int k, void *workspace, int64_t *neighbors,
                            double *mean_dist, void *stream) {
    if (n < 0 || k < 1 || k > kMaxK || dim < 1 || dim > 512 || !grid) return SS_ERR_INVALID;
    if (dim_coarse < 1 || dim_coarse > 512 || !grid_coarse) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    if (!centers || !quats || !workspace || !neighbors || !mean_dist) return SS_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    double4 *nrm = reinterpret_cast<double4 *>(workspace), *nrmc = nrm + n;
    int32_t *defer = reinterpret_cast<int32_t *>(nrmc + n);
    cudaMemsetAsync(defer, 0, 2 * sizeof(int32_t), s);
    knn_normals_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, quats, grid_order(grid, n, dim), nrm);
    knn_normals_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, quats, grid_order(grid_coarse, n, dim_coarse), nrmc);
    const float4 *pk = grid_packed(grid, n, dim), *pkc = grid_packed(grid_coarse, n, dim_coarse);
    switch (k) {
#define SS_KNN_CASE(K) \
    case K: launch_knn<K>(n, grid, pk, nrm, grid_coarse, pkc, nrmc, neighbors, mean_dist, defer, s); break;
        SS_KNN_CASE(1) SS_KNN_CASE(2) SS_KNN_CASE(3) SS_KNN_CASE(4) SS_KNN_CASE(5) SS_KNN_CASE(6)
        SS_KNN_CASE(7) SS_KNN_CASE(8) SS_KNN_CASE(9) SS_KNN_CASE(10) SS_KNN_CASE(11) SS_KNN_CASE(12)
        SS_KNN_CASE(13) SS_KNN_CASE(14) SS_KNN_CASE(15) SS_KNN_CASE(16)
#undef SS_KNN_CASE
    }
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_isolation_dense(int n, const float *centers, const float *log_scales, const int32_t *grid, int dim,
                                  uint8_t *isolated, void *stream) {
    if (n < 0 || dim < 1 || dim > 512 || !grid) return SS_ERR_INVALID;
    if (n == 0) return SS_OK;
    if (!centers || !log_scales || !isolated) return SS_ERR_INVALID;
    isolation_dense_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, centers, log_scales, grid,
                                                                              grid_packed(grid, n, dim), isolated);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
