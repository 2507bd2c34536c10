// FP64 latency / throughput micro-benchmark on one SM (DFMA, rsqrt, shfl, DMMA m8n8k4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
// The DMMA figure (flop/clk/SM) x 148 SMs x max SM clock is the FP64 tensor peak bench.py uses.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dfma(double *out, long long *cyc, double x) {
    double a = x, b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr_dfma(double *out, long long *cyc, double x) {
    double a[8]; for (int k = 0; k < 8; ++k) a[k] = x + k;
    double b = 1.0000001, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s; if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void lat_rsqrt(double *out, long long *cyc, double x) {
    double a = x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) a = rsqrt(a) + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_shfl(double *out, long long *cyc, double x) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31);
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr_dmma(double *out, long long *cyc, double x) {
    double d[8][2]; for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = 0;
    double a = x + threadIdx.x, b = 1.0 / (1 + threadIdx.x);
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0; for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s; if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double *o; long long *c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8 * 4096);
    long long h[4];
    lat_dfma<<<1, 32>>>(o, c, 1.0); cudaDeviceSynchronize(); lat_dfma<<<1, 32>>>(o, c, 1.0); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA latency: %.1f cycles\n", h[0] / 4096.0);
    for (int nt : {32, 128, 256, 512, 1024}) {
        thr_dfma<<<1, nt>>>(o, c, 1.0); cudaDeviceSynchronize(); thr_dfma<<<1, nt>>>(o, c, 1.0); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput, 1 CTA x %d thr: %.2f DFMA/clk/SM\n", nt, 8.0 * 1024 * nt / h[0]);
    }
    lat_rsqrt<<<1, 32>>>(o, c, 2.0); cudaDeviceSynchronize(); lat_rsqrt<<<1, 32>>>(o, c, 2.0); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("rsqrt(double)+add latency: %.1f cycles\n", h[0] / 256.0);
    lat_shfl<<<1, 32>>>(o, c, 1.0); cudaDeviceSynchronize(); lat_shfl<<<1, 32>>>(o, c, 1.0); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("shfl(double) latency: %.1f cycles\n", h[0] / 1024.0);
    for (int nt : {32, 128, 256, 512}) {
        thr_dmma<<<1, nt>>>(o, c, 1.0); cudaDeviceSynchronize(); thr_dmma<<<1, nt>>>(o, c, 1.0); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
        printf("DMMA m8n8k4 1 CTA x %d thr: %.3f mma/clk/SM = %.1f flop/clk/SM\n", nt, 8.0 * 256 * (nt / 32) / h[0], 512.0 * 8 * 256 * (nt / 32) / h[0]);
    }
}
