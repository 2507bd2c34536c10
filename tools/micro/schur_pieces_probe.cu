// Probe: cycles of the Schur kernel's tile building blocks on one CTA (debug aid):
// ld_tile from L2, tile_trsm_d, tile_syrk_lower_sub, tile_xyt, tile_chol64_d, tile_chol64.
#include "../../paper_2312_02999_b200/csrc/k_schur.cu"
#include <cstdio>
#include <vector>
namespace pdipc { void note_launch() {} long long launch_count() { return 0; } }
using namespace pdipc;

__global__ void kprobe(const double *A, double *out, long long *cyc, int *info) {
    extern __shared__ double sm[];
    double *T0 = sm, *T1 = sm + TB * TS, *T2 = sm + 2 * TB * TS, *T3 = sm + 3 * TB * TS;
    __shared__ double Dsh[8][8][9];
    long long t[16];
    int n = 0;
    __syncthreads();
    t[n++] = clock64();
    ld_tile(T0, A, 64, 64, 64);          // 0: load
    __syncthreads();
    t[n++] = clock64();
    for (int e = threadIdx.x; e < TB * TS; e += NT) T1[e] = T0[e];
    __syncthreads();
    t[n++] = clock64();
    tile_chol64_d(T1, Dsh, 64, 64, info);   // 2: chol64_d
    __syncthreads();
    t[n++] = clock64();
    ld_tile(T2, A, 64, 64, 64);
    __syncthreads();
    t[n++] = clock64();
    tile_trsm_d(T2, T1, Dsh);            // 4: trsm
    __syncthreads();
    t[n++] = clock64();
    tile_syrk_lower_sub(T0, T2);         // 5: syrk lower
    t[n++] = clock64();
    tile_xyt(T0, T2, T2, -1.0, true);    // 6: full product
    t[n++] = clock64();
    tile_chol64(T3, T2, 64, 64, info);   // 7: chol64 with inverse (on T3 garbage-free copy)
    __syncthreads();
    t[n++] = clock64();
    st_tile(T1, out, 64, 64, 64);        // 8: store
    __syncthreads();
    t[n++] = clock64();
    if (threadIdx.x == 0)
        for (int i = 0; i + 1 < n; ++i) cyc[i] = t[i + 1] - t[i];
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
    double *dA, *dO;
    long long *dc;
    int *di;
    cudaMalloc(&dA, 8 * 4096);
    cudaMalloc(&dO, 8 * 4096);
    cudaMalloc(&dc, 8 * 16);
    cudaMalloc(&di, 4);
    cudaMemcpy(dA, A.data(), 8 * 4096, cudaMemcpyHostToDevice);
    int smem = 4 * TB * TS * 8;
    cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char *names[] = {"ld_tile", "copy", "chol64_d", "ld_tile", "trsm_d", "syrk_lower", "tile_xyt",
                           "chol64+inv", "st_tile"};
    for (int rep = 0; rep < 2; ++rep) {
        kprobe<<<1, NT, smem>>>(dA, dO, dc, di);
        cudaError_t e = cudaDeviceSynchronize();
        long long c[16];
        cudaMemcpy(c, dc, 8 * 16, cudaMemcpyDeviceToHost);
        printf("rep %d (%s):", rep, cudaGetErrorString(e));
        for (int i = 0; i < 9; ++i) printf(" %s %lld", names[i], c[i]);
        printf("\n");
    }
    // check chol64_d: L L^T = A
    std::vector<double> L(4096);
    cudaMemcpy(L.data(), dO, 8 * 4096, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 64; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = 0;
            for (int k = 0; k < 64; ++k) s += L[i * 64 + k] * L[j * 64 + k];
            err = fmax(err, fabs(s - A[i * 64 + j]));
        }
    printf("chol64_d max |LL^T - A| = %.3e\n", err);
#ifdef CHOL_PROBE
    long long cp[8][64];
    cudaMemcpyFromSymbol(cp, g_cp, sizeof(cp));
    long long t0 = cp[2][0];
    for (int J = 0; J < 7; ++J)
        printf("J%d w0: panel %lld syrk8 %lld chol8 %lld | w1: panel %lld wait %lld upd %lld | end %lld\n", J,
               cp[0][4 * J + 1] - cp[0][4 * J], cp[0][4 * J + 2] - cp[0][4 * J + 1], cp[0][4 * J + 3] - cp[0][4 * J + 2],
               cp[1][4 * J + 1] - cp[1][4 * J], cp[1][4 * J + 2] - cp[1][4 * J + 1], cp[1][4 * J + 3] - cp[1][4 * J + 2],
               cp[2][J + 1] - cp[2][J]);
    (void)t0;
#endif
}
// (per-J stamps of tile_chol64_d when built with -DCHOL_PROBE: printed by chol_d_stamps())
