// Deterministic block reductions in fp64 (fixed shuffle tree, fixed warp order).
#pragma once
#include <cuda_runtime.h>

namespace ctkb {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Sum over the whole block; result valid in thread 0.  blockDim.x*y*z <= 1024.
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double ws[32];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    v = warp_sum(v);
    __syncthreads();
    if ((tid & 31) == 0) ws[tid >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (tid < 32) {
        r = (tid < (nthr + 31) / 32) ? ws[tid] : 0.0;
        r = warp_sum(r);
    }
    return r;
}

__device__ __forceinline__ double block_max(double v) {
    __shared__ double wm[32];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    v = warp_max(v);
    __syncthreads();
    if ((tid & 31) == 0) wm[tid >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (tid < 32) {
        r = (tid < (nthr + 31) / 32) ? wm[tid] : 0.0;
        r = warp_max(r);
    }
    return r;
}

}  // namespace ctkb
