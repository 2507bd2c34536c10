// Micro-benchmark of the 64x64 tile Cholesky used by the fused Schur kernel (debug aid).
#include "../../paper_2312_02999_b200/csrc/k_schur.cu"
#include <cstdio>
#include <vector>
#include <cmath>
namespace pdipc { void note_launch() {} long long launch_count() { return 0; } }
using namespace pdipc;
template <int V>
__global__ void kbench(const double* A, double* Lout, double* Liout, long long* cyc, int* info) {
    extern __shared__ double sm[];
    double *S = sm, *Li = sm + TB * TS;
    long long t0 = clock64();
    ld_tile(S, A, 64, 64, 64);
    __syncthreads();
    long long t1 = clock64();
    tile_chol64(S, Li, 64, 64, info);
    long long t2 = clock64();
    st_tile(S, Lout, 64, 64, 64);
    st_tile(Li, Liout, 64, 64, 64);
    __syncthreads();
    long long t3 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
    std::vector<double> A(64 * 64), M(64 * 64);
    srand(1);
    for (auto& v : M) v = (rand() / (double)RAND_MAX) - 0.5;
    for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) {
        double s = 0; for (int k = 0; k < 64; ++k) s += M[i * 64 + k] * M[j * 64 + k];
        A[i * 64 + j] = s + (i == j ? 64.0 : 0.0);
    }
    double *dA, *dL, *dLi; long long* dc; int* di;
    cudaMalloc(&dA, 8 * 4096); cudaMalloc(&dL, 8 * 4096); cudaMalloc(&dLi, 8 * 4096); cudaMalloc(&dc, 64); cudaMalloc(&di, 4);
    cudaMemcpy(dA, A.data(), 8 * 4096, cudaMemcpyHostToDevice); cudaMemset(di, 0, 4);
    int smem = 3 * TB * TS * 8;
    cudaFuncSetAttribute(kbench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kbench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kbench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int v = 0; v < 1; ++v) {
        for (int rep = 0; rep < 3; ++rep) {
            if (v == 0) kbench<0><<<1, NT, smem>>>(dA, dL, dLi, dc, di);
            else if (v == 1) kbench<1><<<1, NT, smem>>>(dA, dL, dLi, dc, di);
            else kbench<2><<<1, NT, smem>>>(dA, dL, dLi, dc, di);
            cudaDeviceSynchronize();
            long long c[3]; cudaMemcpy(c, dc, 24, cudaMemcpyDeviceToHost);
            printf("v%d cycles: load %lld  chol %lld  store %lld  (err=%s)\n", v, c[0], c[1], c[2], cudaGetErrorString(cudaGetLastError()));
        }
        std::vector<double> L(4096), Li(4096);
        cudaMemcpy(L.data(), dL, 8 * 4096, cudaMemcpyDeviceToHost); cudaMemcpy(Li.data(), dLi, 8 * 4096, cudaMemcpyDeviceToHost);
        double e1 = 0, e2 = 0, e3 = 0;
        for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) {
            double s = 0, t = 0; for (int k = 0; k < 64; ++k) { s += L[i * 64 + k] * L[j * 64 + k]; t += L[i * 64 + k] * Li[k * 64 + j]; }
            if (j <= i) e1 = fmax(e1, fabs(s - A[i * 64 + j]));
            e2 = fmax(e2, fabs(t - (i == j)));
            if (j > i) e3 = fmax(e3, fabs(L[i * 64 + j]) + fabs(Li[i * 64 + j]));
        }
        printf("v%d max |LL^T - A| = %.3e   max |L Li - I| = %.3e  upper %.1e\n", v, e1, e2, e3);
    }
}
