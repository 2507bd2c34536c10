// Whole-GPU FP64 tensor (DMMA, mma.sync.m8n8k4.f64) throughput: every SM runs CTAs of 256
// threads issuing independent register-operand DMMAs back to back; timed with CUDA events over
// a burst (~50 ms) and a sustained (~4 s) run.  The roofline denominator of bench.py's dense
// Schur line (the single-SM figure of fp64_peaks.cu x 148 x max clock is the nominal one).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_gpu_peak dmma_gpu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
__global__ void __launch_bounds__(256) k_dmma(double *out, long long iters, double x) {
    double d[kChains][2];
    for (int k = 0; k < kChains; ++k) d[k][0] = d[k][1] = 0.0;
    const double a = x + threadIdx.x * 1e-9, b = x - threadIdx.x * 1e-9;
    for (long long i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < kChains; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int k = 0; k < kChains; ++k) s += d[k][0] + d[k][1];
    if (s == 1.2345) out[0] = s;      // keep the chains alive
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int per_sm : {1, 2, 4}) {
        const int grid = nsm * per_sm;
        for (long long iters : {20000LL, 1600000LL / per_sm}) {
            k_dmma<<<grid, 256>>>(out, 1000, 1.0);   // warm-up
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            k_dmma<<<grid, 256>>>(out, iters, 1.0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 512.0 * kChains * iters * (grid * 256 / 32);   // 8x8x4 x 2 per warp mma
            printf("DMMA whole GPU: %d SMs x %d CTAs x 256 thr, %lld iters: %.3f ms, %.2f TFLOP/s\n", nsm, per_sm,
                   iters, ms, flops / (ms * 1e-3) / 1e12);
        }
    }
    return cudaGetLastError() != cudaSuccess;
}
