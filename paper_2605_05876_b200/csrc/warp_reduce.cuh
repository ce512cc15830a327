// warp_reduce.cuh -- transposed butterfly reduction of N per-lane channels.
//
// After warp_tr_reduce<N>(v, lane) every lane holds in v[0] the warp-wide sum
// of channel warp_tr_index<N>(lane).  At each of the 5 butterfly levels a lane
// keeps half of its remaining channels and trades the other half with its
// partner, so N channels cost ~N+log2(32) shuffles instead of 5N.  Channels
// left unpaired at a level are all-reduced in both lanes; duplicates are
// resolved by the caller with __match_any_sync (lowest lane owns).
#pragma once
#include <cuda_runtime.h>

template <int N, int O, typename T>
__device__ __forceinline__ void warp_tr_level(T *v, bool upper) {
    constexpr int H = N / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        const T send = upper ? v[i] : v[i + H];
        const T keep = upper ? v[i + H] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
    if constexpr ((N & 1) != 0) v[H] = v[N - 1] + __shfl_xor_sync(0xffffffffu, v[N - 1], O);
}

template <int N, int O, typename T>
__device__ __forceinline__ void warp_tr_all(T *v, int lane) {
    warp_tr_level<N, O>(v, (lane & O) != 0);
    if constexpr (O > 1) warp_tr_all<N / 2 + (N & 1), O / 2>(v, lane);
}

// float or double channels
template <int N, typename T>
__device__ __forceinline__ void warp_tr_reduce(T (&v)[N], int lane) {
    warp_tr_all<N, 16>(v, lane);
}

template <int N, int O>
__device__ __forceinline__ int warp_tr_index_rec(int *idx, int lane) {
    constexpr int H = N / 2;
    const bool upper = (lane & O) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) idx[i] = upper ? idx[i + H] : idx[i];
    if constexpr ((N & 1) != 0) idx[H] = idx[N - 1];
    if constexpr (O > 1) return warp_tr_index_rec<N / 2 + (N & 1), O / 2>(idx, lane);
    else return idx[0];
}

template <int N>
__device__ __forceinline__ int warp_tr_index(int lane) {
    int idx[N];
#pragma unroll
    for (int i = 0; i < N; ++i) idx[i] = i;
    return warp_tr_index_rec<N, 16>(idx, lane);
}

template <int N, int O>
__device__ __forceinline__ void warp_tr_indices_rec(int *idx, int lane) {
    constexpr int H = N / 2;
    const bool upper = (lane & O) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) idx[i] = upper ? idx[i + H] : idx[i];
    if constexpr ((N & 1) != 0) idx[H] = idx[N - 1];
    if constexpr (O > 1) warp_tr_indices_rec<N / 2 + (N & 1), O / 2>(idx, lane);
}

// Channel indices held in v[0 .. M) after warp_tr_all<N, O> (levels O .. 1,
// i.e. a reduction within groups of 2*O lanes).
template <int N, int O, int M>
__device__ __forceinline__ void warp_tr_indices(int (&out)[M], int lane) {
    int idx[N];
#pragma unroll
    for (int i = 0; i < N; ++i) idx[i] = i;
    warp_tr_indices_rec<N, O>(idx, lane);
#pragma unroll
    for (int i = 0; i < M; ++i) out[i] = idx[i];
}
