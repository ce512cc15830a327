// binning.cu -- tile binning with a deterministic (tile, z_start, record)
// order, sync-free (all counts stay on the device).
//
// Reference: bin_and_sort (rasterizer.py:92-116) = emit pairs, np.lexsort by
// (tile, z_start[rec], rec), offsets by bincount.  B200 design:
//   1. the preprocess kernel already built the per-tile histogram;
//   2. tile_scan: one CTA scans it into tile_offsets (the output) and checks
//      the pair capacity;
//   3. scatter: each record drops a 64-bit key (orderable z_start << 32 | rec)
//      into every tile bucket of its rect (unordered, atomics);
//   4. tile_sort: one CTA per tile sorts its bucket in shared memory with a
//      padding-free bitonic network.  Keys are unique (rec in the low bits),
//      so the order is total and equals lexsort's stable tie-break exactly.
#include "ss_common.cuh"

namespace {

constexpr int kScanThreads = 1024;
// Per-tile merge sort in shared memory (two ping-pong buffers).  Tiles up to
// kSmallCap keys are sorted by a light CTA so several tiles share an SM; the
// heavier ones by a second launch with a large buffer (each launch skips the
// other's tiles); beyond kHeavyCap a bitonic network runs in global memory.
#ifndef SS_SORT_SMALL_THREADS
#define SS_SORT_SMALL_THREADS 512
#endif
#ifndef SS_SORT_SMALL_CAP
#define SS_SORT_SMALL_CAP 4096
#endif
constexpr int kSmallThreads = SS_SORT_SMALL_THREADS;
constexpr int kSmallCap = SS_SORT_SMALL_CAP;
#ifndef SS_SORT_HEAVY_CAP
#define SS_SORT_HEAVY_CAP 12288
#endif
constexpr int kHeavyThreads = 1024;
constexpr int kHeavyCap = SS_SORT_HEAVY_CAP;


__device__ void tile_order(const int32_t *__restrict__ counts, int ntiles, int32_t *__restrict__ order);

// CTA 0: exclusive scan of the tile counts into the offsets; CTA 1 (when an
// order is requested): the heavy-first launch order of the tiles.
__global__ void __launch_bounds__(kScanThreads) tile_scan_kernel(
    const int32_t *__restrict__ counts, int ntiles, int32_t *__restrict__ offsets,
    int32_t *__restrict__ cursors, int64_t capacity, int32_t *__restrict__ flags, int32_t *__restrict__ order)
{
    if (blockIdx.x == 1) {
        tile_order(counts, ntiles, order);
        return;
    }
    __shared__ int32_t warp_sums[kScanThreads / 32];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < ntiles; base += kScanThreads) {
        int t = base + threadIdx.x;
        int v = t < ntiles ? counts[t] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int s = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        int excl = carry + (wid > 0 ? warp_sums[wid - 1] : 0) + x - v;
        if (t < ntiles) {
            // clamped to the capacity: on overflow every consumer of the
            // offsets (scatter, tile sort, rasterisers) stays inside the pair
            // buffers; the dropped pairs are reported by flags[2]/[3]
            offsets[t] = (int64_t)excl < capacity ? excl : (int32_t)capacity;
            cursors[t] = 0;
        }
        __syncthreads();
        if (threadIdx.x == kScanThreads - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        offsets[ntiles] = (int64_t)carry < capacity ? carry : (int32_t)capacity;
        if ((int64_t)carry > capacity) atomicOr(&flags[2], 1);
        atomicMax(&flags[3], carry);  // pairs the view needs (max over the views sharing these flags)
    }
}

// Launch order for the rasterisers: tiles grouped by descending log2 of
// their pair count (heavy tiles first, so the last wave is made of light
// ones); the order within a group is irrelevant to the results.
__device__ void tile_order(const int32_t *__restrict__ counts, int ntiles, int32_t *__restrict__ order)
{
    __shared__ int32_t hist[33], base[33];
    if (threadIdx.x < 33) hist[threadIdx.x] = 0;
    __syncthreads();
    auto group = [](int c) { return c > 0 ? 32 - __clz(c) : 0; };  // 0 (empty) .. 32, larger = heavier
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) atomicAdd(&hist[group(counts[t])], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int g = 32; g >= 0; --g) { base[g] = acc; acc += hist[g]; }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) order[atomicAdd(&base[group(counts[t])], 1)] = t;
}

// Each record drops its key into every tile bucket of its rect.  Atomics on
// the tile cursors are privatised per CTA: a CTA of 4096 records counts its
// pairs per tile in shared memory, reserves one contiguous block per touched
// tile with a single global atomic, then hands out slots with shared-memory
// atomics.  Global same-address traffic drops from one atomic per pair to one
// per (CTA, tile).  Slot order inside a bucket is arbitrary: the per-tile sort
// that follows keys on (z_start, record), so the result is deterministic.
#ifndef SS_SCATTER_THREADS
#define SS_SCATTER_THREADS 1024
#endif
#ifndef SS_SCATTER_PER_THREAD
#define SS_SCATTER_PER_THREAD 4
#endif
constexpr int kScatterThreads = SS_SCATTER_THREADS;
constexpr int kScatterPerThread = SS_SCATTER_PER_THREAD;

__global__ void __launch_bounds__(kScatterThreads) scatter_kernel(
    int n, const uint4 *__restrict__ bininfo, const int8_t *__restrict__ cull, int ntx, int ntiles, int tile,
    const int32_t *__restrict__ offsets, int32_t *__restrict__ cursors, uint64_t *__restrict__ keys,
    int64_t capacity)
{
    extern __shared__ int32_t s_cnt[];   // ntiles counters, then ntiles block bases
    int32_t *s_base = s_cnt + ntiles;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_cnt[t] = 0;
    __syncthreads();
    const int first = blockIdx.x * kScatterThreads * kScatterPerThread;
    for (int k = 0; k < kScatterPerThread; ++k) {
        const int i = first + k * kScatterThreads + threadIdx.x;
        if (i >= n || cull[i] != 0) continue;
        const uint4 b = bininfo[i];
        const int tx0 = (int)(b.x & 0xffff) / tile, ty0 = (int)(b.x >> 16) / tile;
        const int tx1 = ((int)(b.y & 0xffff) - 1) / tile, ty1 = ((int)(b.y >> 16) - 1) / tile;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(&s_cnt[ty * ntx + tx], 1);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
        const int c = s_cnt[t];
        if (c > 0) s_base[t] = atomicAdd(&cursors[t], c);
        s_cnt[t] = 0;
    }
    __syncthreads();
    for (int k = 0; k < kScatterPerThread; ++k) {
        const int i = first + k * kScatterThreads + threadIdx.x;
        if (i >= n || cull[i] != 0) continue;
        const uint4 b = bininfo[i];
        const uint64_t key = ((uint64_t)b.z << 32) | (uint32_t)i;
        const int tx0 = (int)(b.x & 0xffff) / tile, ty0 = (int)(b.x >> 16) / tile;
        const int tx1 = ((int)(b.y & 0xffff) - 1) / tile, ty1 = ((int)(b.y >> 16) - 1) / tile;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) {
                const int t = ty * ntx + tx;
                const int64_t at = (int64_t)offsets[t] + s_base[t] + atomicAdd(&s_cnt[t], 1);
                if (at < capacity) keys[at] = key;
            }
    }
}

// Ascending bitonic network on n elements padded (virtually) with +inf up to
// a power of two: every comparator is ascending, so a pair whose upper index
// is past the end never exchanges and the padding never has to exist.
template <typename Load, typename Swap>
__device__ __forceinline__ void bitonic_sort(int n, Load ld, Swap sw) {
    int N = 1, lgN = 0;
    while (N < n) { N <<= 1; ++lgN; }
    for (int lk = 1; lk <= lgN; ++lk) {
        const int lh = lk - 1;  // log2(k / 2)
        const int hmask = (1 << lh) - 1;
        for (int p = threadIdx.x; p < (N >> 1); p += blockDim.x) {
            const int off = p & hmask;
            const int lo = ((p >> lh) << lk) + off, hi = lo + (1 << lk) - 1 - 2 * off;
            if (hi < n) sw(lo, hi);
        }
        __syncthreads();
        for (int lj = lh - 1; lj >= 0; --lj) {
            const int jm = (1 << lj) - 1;
            for (int p = threadIdx.x; p < (N >> 1); p += blockDim.x) {
                const int lo = ((p >> lj) << (lj + 1)) + (p & jm), hi = lo + (1 << lj);
                if (hi < n) sw(lo, hi);
            }
            __syncthreads();
        }
    }
    (void)ld;
}

// packed pixel rect of a record, in pair order, for the rasterisers' warp cull
__device__ __forceinline__ uint2 pack_rect(const uint4 *__restrict__ bininfo, int rec) {
    return *reinterpret_cast<const uint2 *>(bininfo + rec);
}

// 32 keys per warp sorted in registers (bitonic network over shuffles).
__device__ __forceinline__ uint64_t warp_sort32(uint64_t v, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint64_t o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = (lane & k) == 0;           // ascending block
            const bool lower = (lane & j) == 0;        // lower element of the pair
            const bool keep_min = lower == up;
            v = keep_min ? (o < v ? o : v) : (o > v ? o : v);
        }
    }
    return v;
}

// Merge path: the split (a, d - a) of diagonal d of runs x[0, la), y[0, lb)
// (unique keys).
__device__ __forceinline__ int merge_split(const uint64_t *x, int la, const uint64_t *y, int lb, int d) {
    int lo = max(0, d - lb), hi = min(d, la);
    while (lo < hi) {
        const int a = (lo + hi) >> 1;
        if (x[a] < y[d - a - 1]) lo = a + 1;
        else hi = a;
    }
    return lo;
}

template <int kThreads, int kCap, bool kHeavy>
__global__ void __launch_bounds__(kThreads) tile_sort_kernel(
    const int32_t *__restrict__ offsets, uint64_t *__restrict__ keys, int32_t *__restrict__ pair_rec,
    uint2 *__restrict__ pair_rect, const uint4 *__restrict__ recs, int64_t capacity,
    const int32_t *__restrict__ order)
{
    extern __shared__ uint64_t skeys[];
    const int t = order ? order[blockIdx.x] : blockIdx.x;  // heavy tiles first when an order is given
    const int64_t o0 = offsets[t];
    int64_t o1 = offsets[t + 1];
    if (o1 > capacity) o1 = capacity;
    if (o0 >= o1) return;
    const int n = (int)(o1 - o0);
    if ((n > kSmallCap) != kHeavy) return;  // the other launch owns this tile
    uint64_t *g = keys + o0;
    if (n <= kCap) {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        const int np = (n + 31) & ~31;  // padded with +inf to whole 32-key runs
        uint64_t *A = skeys, *B = skeys + kCap;
        for (int r = wid * 32; r < np; r += kThreads) {
            const int k = r + lane;
            const uint64_t v = k < n ? g[k] : ~0ull;
            A[k] = warp_sort32(v, lane);
        }
        __syncthreads();
        for (int w = 32; w < np; w <<= 1) {
            const int per = (np + kThreads - 1) / kThreads;
            const int o = threadIdx.x * per;
            if (o < np) {
                const int pair0 = (o / (2 * w)) * (2 * w);
                const int la = min(w, np - pair0), lb = max(0, min(w, np - pair0 - w));
                const uint64_t *x = A + pair0, *y = A + pair0 + la;
                const int d = o - pair0;
                int a = merge_split(x, la, y, lb, d), b = d - a;
                const int e = min(per, np - o);
                // a thread's output may cross into the next pair of runs
                int base = pair0, cla = la, clb = lb;
                for (int q = 0; q < e; ++q) {
                    if (a + b == cla + clb) {  // next pair of runs starts at this output
                        base += 2 * w;
                        cla = min(w, np - base);
                        clb = max(0, min(w, np - base - w));
                        x = A + base; y = A + base + cla;
                        a = 0; b = 0;
                    }
                    const bool take_x = b >= clb || (a < cla && x[a] < y[b]);
                    B[o + q] = take_x ? x[a] : y[b];
                    a += take_x; b += !take_x;
                }
            }
            __syncthreads();
            uint64_t *tmp = A; A = B; B = tmp;
        }
        for (int k = threadIdx.x; k < n; k += kThreads) {
            const int rec = (int32_t)(uint32_t)A[k];
            pair_rec[o0 + k] = rec;
            pair_rect[o0 + k] = pack_rect(recs, rec);
        }
    } else {
        // rare oversized tile: bitonic network directly in global memory
        bitonic_sort(n, 0, [&](int a, int b) {
            uint64_t x = g[a], y = g[b];
            if (x > y) { g[a] = y; g[b] = x; }
        });
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
            const int rec = (int32_t)(uint32_t)g[k];
            pair_rec[o0 + k] = rec;
            pair_rect[o0 + k] = pack_rect(recs, rec);
        }
    }
}

}  // namespace

extern "C" int ss_bin_sort(int n, const uint32_t *bininfo, const int8_t *cull, int width, int height, int tile,
                           const int32_t *tile_counts, int32_t *tile_offsets, int32_t *cursors,
                           uint64_t *keys, int32_t *pair_rec, uint32_t *pair_rect, int64_t pair_capacity,
                           int32_t *flags, int32_t *tile_order, void *stream)
{
    if (width <= 0 || height <= 0 || tile <= 0 || !tile_counts || !tile_offsets || !cursors || !flags)
        return SS_ERR_INVALID;
    if (width > 65535 || height > 65535) return SS_ERR_INVALID;  // rects are packed as uint16
    ss_func_smem((const void *)tile_sort_kernel<kHeavyThreads, kHeavyCap, true>, 2 * kHeavyCap * (int)sizeof(uint64_t));
    ss_func_smem((const void *)tile_sort_kernel<kSmallThreads, kSmallCap, false>, 2 * kSmallCap * (int)sizeof(uint64_t));
    cudaStream_t st = (cudaStream_t)stream;
    const int ntx = (width + tile - 1) / tile, nty = (height + tile - 1) / tile;
    const int ntiles = ntx * nty;
    tile_scan_kernel<<<tile_order ? 2 : 1, kScanThreads, 0, st>>>(tile_counts, ntiles, tile_offsets, cursors,
                                                                  pair_capacity, flags, tile_order);
    SS_CUDA_CHECK_LAUNCH();
    if (n > 0) {
        const size_t smem = 2 * (size_t)ntiles * sizeof(int32_t);
        if (smem > 220 * 1024) return SS_ERR_INVALID;  // > 28k tiles: not supported by the privatised scatter
        ss_func_smem((const void *)scatter_kernel, (int)smem);
        const int per_cta = kScatterThreads * kScatterPerThread;
        scatter_kernel<<<(n + per_cta - 1) / per_cta, kScatterThreads, smem, st>>>(
            n, reinterpret_cast<const uint4 *>(bininfo), cull, ntx, ntiles, tile, tile_offsets, cursors, keys,
            pair_capacity);
        SS_CUDA_CHECK_LAUNCH();
    }
    tile_sort_kernel<kSmallThreads, kSmallCap, false><<<ntiles, kSmallThreads, 2 * kSmallCap * sizeof(uint64_t), st>>>(
        tile_offsets, keys, pair_rec, reinterpret_cast<uint2 *>(pair_rect), reinterpret_cast<const uint4 *>(bininfo),
        pair_capacity, tile_order);
    SS_CUDA_CHECK_LAUNCH();
    tile_sort_kernel<kHeavyThreads, kHeavyCap, true><<<ntiles, kHeavyThreads, 2 * kHeavyCap * sizeof(uint64_t), st>>>(
        tile_offsets, keys, pair_rec, reinterpret_cast<uint2 *>(pair_rect), reinterpret_cast<const uint4 *>(bininfo),
        pair_capacity, tile_order);
    SS_CUDA_CHECK_LAUNCH();
    return SS_OK;
}
