// Probe: cycles of the single-thread 8x8 Cholesky+inverse and of a dependent rsqrt chain
// (debug aid for the Schur tile factorisation).
#include "../../paper_2312_02999_b200/csrc/k_schur.cu"
#include <cstdio>
namespace pdipc { void note_launch() {} long long launch_count() { return 0; } }
using namespace pdipc;
__global__ void kprobe(const double *A, long long *cyc, int *info) {
    __shared__ double S[8 * TS];
    __shared__ double D[8][9];
    for (int e = threadIdx.x; e < 64; e += blockDim.x) S[(e >> 3) * TS + (e & 7)] = A[e];
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        bool bad = chol8_thread(S, D, 8);
        long long t1 = clock64();
        cyc[0] = t1 - t0 + (bad ? 1000000 : 0);
        double x = S[0];
        t0 = clock64();
        for (int i = 0; i < 16; ++i) x = rsqrt(x + 1.0);
        t1 = clock64();
        cyc[1] = (t1 - t0) / 16;
        S[1] = x;
    }
}
int main() {
    double A[64];
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) A[i * 8 + j] = (i == j ? 10.0 : 0.5 / (1 + i + j));
    double *dA;
    long long *dc;
    int *di;
    cudaMalloc(&dA, 512);
    cudaMalloc(&dc, 64);
    cudaMalloc(&di, 4);
    cudaMemcpy(dA, A, 512, cudaMemcpyHostToDevice);
    for (int r = 0; r < 3; ++r) {
        kprobe<<<1, 32>>>(dA, dc, di);
        cudaDeviceSynchronize();
        long long c[2];
        cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
        printf("chol8_thread %lld cycles, rsqrt(double) chain %lld cycles/op\n", c[0], c[1]);
    }
}
