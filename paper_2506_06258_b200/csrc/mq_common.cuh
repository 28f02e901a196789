// Shared device helpers for the market_eq_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "market_eq_b200.h"

#define MQ_FULL 0xffffffffu

// Bounds checks of the checked build (-DMQ_DEBUG_BOUNDS; compute-sanitizer is
// not available on the GPU pool): a failed check prints its file and line and
// traps, the launch fails and the caller's NativeError names the call.
#ifdef MQ_DEBUG_BOUNDS
#include <cassert>
#define MQ_CHECK(c) assert(c)
#else
#define MQ_CHECK(c) ((void)0)
#endif
#define MQ_MAX_BLOCKS 1024          // fixed partial-sum width => deterministic sums
#define MQ_SCRATCH_DOUBLES (8 * MQ_MAX_BLOCKS + 64)

namespace mq {

// error bookkeeping (abi.cu)
int set_error(cudaError_t e, const char *where);
int check_launch(const char *where);

inline int grid_for(int64_t work, int per_block, int cap) {
    int64_t g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

// xor-butterfly sum over a G-lane group: every lane ends with the same,
// order-fixed value (commutativity makes both halves of each pair agree).
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(MQ_FULL, v, o);
    return v;
}
template <int G>
__device__ __forceinline__ int group_sum_int(int v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(MQ_FULL, v, o);
    return v;
}
template <int G>
__device__ __forceinline__ double group_max(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(MQ_FULL, v, o));
    return v;
}
template <int G>
__device__ __forceinline__ double group_min(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(MQ_FULL, v, o));
    return v;
}

// Max of nonnegative doubles through their (order-preserving) bit patterns:
// order-free, hence deterministic.
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
    if (v > 0.0)
        atomicMax(reinterpret_cast<unsigned long long *>(addr),
                  (unsigned long long)__double_as_longlong(v));
}

// Block-wide fixed-order sum of one double per thread (blockDim.x <= 1024,
// multiple of 32).  Result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double *smem /*[32]*/) {
    v = group_sum<32>(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (warp == 0) {
        r = lane < (int)(blockDim.x >> 5) ? smem[lane] : 0.0;
        r = group_sum<32>(r);
    }
    return r;
}

__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t *smem /*[32]*/) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MQ_FULL, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    int64_t r = 0;
    if (warp == 0) {
        r = lane < (int)(blockDim.x >> 5) ? smem[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(MQ_FULL, r, o);
    }
    return r;
}

// Positive root of s^2 - A s - tw B = 0 (the fixed point s = A + tw B / s of
// an active set with A = sum u c, B = sum u^2); conjugate form for A < 0.
__device__ __forceinline__ double active_root(double A, double B, double tw) {
    const double d = sqrt(A * A + 4.0 * tw * B);
    return A >= 0.0 ? 0.5 * (A + d) : (2.0 * tw * B) / (d - A);
}

}  // namespace mq
