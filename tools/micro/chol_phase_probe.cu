// Probe: per-phase cycles of the 64x64 tile Cholesky (tile_chol64) of the Schur kernel, with
// clock64 stamps taken by thread 0 (debug aid).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 chol_phase_probe.cu
#include "../../paper_2312_02999_b200/csrc/k_schur.cu"
#include <cstdio>
#include <vector>
namespace pdipc { void note_launch() {} long long launch_count() { return 0; } }
using namespace pdipc;

__device__ long long g_st[64];

// copy of tile_chol64 with timestamps
__device__ void tile_chol64_probe(double *S, double *Li, int nb, int free_row, int *info) {
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    __shared__ double DI[2][8][9];
    int ns = 0;
    if (tid == 0) g_st[ns] = clock64();
    ++ns;
    for (int e = tid; e < TB * TB; e += NT) {
        const int r = e >> 6, c = e & 63;
        if (r >= nb || c >= nb) S[r * TS + c] = (r == c) ? 1.0 : 0.0;
        else if (c > r) S[r * TS + c] = 0.0;
        Li[r * TS + c] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    bool bad = false;
    if (tid == 0) bad |= chol8_thread(S, DI[0], free_row);
    __syncthreads();
    if (tid == 0) g_st[ns] = clock64();
    ++ns;
    for (int J = 0; J < 8; ++J) {
        const int j0 = 8 * J;
        const double (*D)[9] = DI[J & 1];
        if (tid < 64) {
            const int i = tid;
            if (i >= j0 + 8) {
                double v[8], o[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = S[i * TS + j0 + q];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    double acc = 0.0;
#pragma unroll
                    for (int q = 0; q <= c; ++q) acc += v[q] * D[c][q];
                    o[c] = acc;
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) S[i * TS + j0 + c] = o[c];
            }
        } else if (tid < 128) {
            const int c = tid - 64;
            if (c < j0 + 8) {
                double v[8], o[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = Li[(j0 + q) * TS + c];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    double acc = 0.0;
#pragma unroll
                    for (int q = 0; q <= r; ++q) acc += D[r][q] * v[q];
                    o[r] = acc;
                }
#pragma unroll
                for (int r = 0; r < 8; ++r) Li[(j0 + r) * TS + c] = o[r];
            }
        }
        __syncthreads();
        if (tid == 0) g_st[ns] = clock64();
        ++ns;
        if (J == 7) break;
        const int T = 7 - J, j1 = j0 + 8;
        if (wid == 0) {
            tile8_sub_xyt(S + j1 * TS + j1, S + j1 * TS + j0, S + j1 * TS + j0, TS, 1, true);
            __syncwarp();
            long long c0 = clock64();
            if (lane == 0) bad |= chol8_thread(S + j1 * TS + j1, DI[(J + 1) & 1], free_row - j1);
            if (lane == 0) g_st[40 + J] = clock64() - c0;
        } else {
            long long c0 = clock64();
            const int nA = T * (T + 1) / 2 - 1, nB = T * (J + 1);
            for (int t = wid - 1; t < nA + nB; t += NT / 32 - 1) {
                if (t < nA) {
                    int u = t + 1, I = 0;
                    while (u > I) { u -= I + 1; ++I; }
                    const int L = u;
                    const int r0 = j1 + 8 * I, c0 = j1 + 8 * L;
                    tile8_sub_xyt(S + r0 * TS + c0, S + r0 * TS + j0, S + c0 * TS + j0, TS, 1, I == L);
                } else {
                    const int u = t - nA, I = u / (J + 1), Lb = u % (J + 1);
                    const int r0 = j1 + 8 * I, c0 = 8 * Lb;
                    tile8_sub_xyt(Li + r0 * TS + c0, S + r0 * TS + j0, Li + j0 * TS + c0, 1, TS, false);
                }
            }
            if (tid == 32) g_st[50 + J] = clock64() - c0;
        }
        __syncthreads();
        if (tid == 0) g_st[ns] = clock64();
        ++ns;
    }
    if (bad) atomicExch(info, 1);
    if (tid == 0) g_st[39] = ns;
}

__global__ void kbench(const double *A, long long *out, int *info) {
    extern __shared__ double sm[];
    double *S = sm, *Li = sm + TB * TS;
    ld_tile(S, A, 64, 64, 64);
    __syncthreads();
    tile_chol64_probe(S, Li, 64, 64, info);
    __syncthreads();
    if (threadIdx.x < 64) out[threadIdx.x] = g_st[threadIdx.x];
}

int main() {
    std::vector<double> A(64 * 64), M(64 * 64);
    srand(1);
    for (auto &v : M) v = (rand() / (double)RAND_MAX) - 0.5;
    for (int i = 0; i < 64; ++i)
        for (int j = 0; j < 64; ++j) {
            double s = 0;
            for (int k = 0; k < 64; ++k) s += M[i * 64 + k] * M[j * 64 + k];
            A[i * 64 + j] = s + (i == j ? 64.0 : 0.0);
        }
    double *dA;
    long long *dout;
    int *di;
    cudaMalloc(&dA, 8 * 4096);
    cudaMalloc(&dout, 8 * 64);
    cudaMalloc(&di, 4);
    cudaMemcpy(dA, A.data(), 8 * 4096, cudaMemcpyHostToDevice);
    int smem = 2 * TB * TS * 8;
    cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        kbench<<<1, NT, smem>>>(dA, dout, di);
        cudaDeviceSynchronize();
        long long o[64];
        cudaMemcpy(o, dout, 8 * 64, cudaMemcpyDeviceToHost);
        int ns = (int)o[39];
        printf("rep %d total %lld cycles; phase intervals:", rep, o[ns - 1] - o[0]);
        for (int i = 1; i < ns; ++i) printf(" %lld", o[i] - o[i - 1]);
        printf("\n  chol8 (warp0 lane0) per J:");
        for (int J = 0; J < 7; ++J) printf(" %lld", o[40 + J]);
        printf("\n  updates (warp1) per J:");
        for (int J = 0; J < 7; ++J) printf(" %lld", o[50 + J]);
        printf("\n");
    }
}
