// Warp / block scan helpers (shuffle based). Internal.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace spc {

constexpr unsigned kFull = 0xffffffffu;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = __shfl_up_sync(kFull, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
    return v;
}

// Block exclusive scan; every thread of the block must call it. `sm` needs 33 T (one slot per
// warp plus the block total, kept apart so that 32-warp blocks do not overwrite warp 31's prefix).
// Returns the exclusive prefix of v; *total receives the block sum (all threads).
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sm, T* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    T inc = warp_incl_scan(v);
    if (lane == 31) sm[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T s = lane < nw ? sm[lane] : T(0);
        T si = warp_incl_scan(s);
        if (lane < nw) sm[lane] = si - s;
        if (lane == nw - 1) sm[32] = si;
    }
    __syncthreads();
    T res = inc - v + sm[wid];
    *total = sm[32];
    __syncthreads();
    return res;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sm) {
    T tot;
    block_excl_scan(v, sm, &tot);
    return tot;
}

}  // namespace spc
