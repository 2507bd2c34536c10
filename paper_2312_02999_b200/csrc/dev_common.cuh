// Shared device utilities of the CUDA path (not shared with the oracle).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace pdipc {

// Every kernel launch of the library goes through PDI_LAUNCH so that the number of our
// kernels launched inside a timed region can be reported (bench.py "gpu_launches").
void note_launch();
long long launch_count();
#define PDI_LAUNCH(kern, ...) ::pdipc::note_launch(), kern<<<__VA_ARGS__>>>

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum (fixed tree order for a fixed blockDim); result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh /* >= NT/32 */) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < NT / 32 ? sh[lane] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

// Non-negative doubles compare like their bit patterns: atomic min of a TOI in [0, 1].
__device__ __forceinline__ void atomic_min_nonneg(double *addr, double v) {
    atomicMin(reinterpret_cast<unsigned long long *>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace pdipc
