// Times the 64 x 64 diagonal-tile factor of the large-system Cholesky (tile_chol64: Cholesky +
// explicit inverse, one CTA) and its neighbours on the panel chain (tile_xyt), with clock64 on
// one CTA: the chain element of every tile column of P3.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int TB = 64, TS = 68, NT = 256;
__device__ __forceinline__ void dmma_884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ bool chol8_thread(double *S, double (*D)[9], int free_row) {
    double a[8][8], x[8][8], rinv[8];
    bool bad = false;
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) a[r][c] = c <= r ? S[r * TS + c] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        double p = a[k][k];
        bad |= !(p > 0.0) && k < free_row;
        p = p > 0.0 ? p : 1.0;
        const double rs = rsqrt(p);
        rinv[k] = rs;
        a[k][k] = p * rs;
#pragma unroll
        for (int r = k + 1; r < 8; ++r) a[r][k] *= rs;
#pragma unroll
        for (int r = k + 1; r < 8; ++r)
#pragma unroll
            for (int l = k + 1; l <= r; ++l) a[r][l] -= a[r][k] * a[l][k];
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)                 // x = L^{-1}: column c by forward substitution
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            double acc = r == c ? 1.0 : 0.0;
#pragma unroll
            for (int q = 0; q < r; ++q) acc -= a[r][q] * x[q][c];
            x[r][c] = r >= c ? acc * rinv[r] : 0.0;
        }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (c <= r) S[r * TS + c] = a[r][c];
            D[r][c] = x[r][c];
        }
    return bad;
}

__device__ __forceinline__ void tile8_sub_xyt(double *C, const double *X, const double *Y, int ys_row,
                                              int ys_col, bool lower_only) {
    const int lane = threadIdx.x & 31, gr = lane >> 2, gc = lane & 3;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < 2; ++k4)
        dmma_884(d0, d1, X[gr * TS + 4 * k4 + gc], Y[gr * ys_row + (4 * k4 + gc) * ys_col]);
    const int c = 2 * gc;
    if (!lower_only || c <= gr) C[gr * TS + c] -= d0;
    if (!lower_only || c + 1 <= gr) C[gr * TS + c + 1] -= d1;
}

template <int NTH = NT>
__device__ void tile_chol64(double *S, double *Li, int nb, int free_row, int *info) {
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    __shared__ double DI[2][8][9];
    for (int e = tid; e < TB * TB; e += NTH) {
        const int r = e >> 6, c = e & 63;
        if (r >= nb || c >= nb) S[r * TS + c] = (r == c) ? 1.0 : 0.0;
        else if (c > r) S[r * TS + c] = 0.0;
        Li[r * TS + c] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    bool bad = false;
    if (tid == 0) bad |= chol8_thread(S, DI[0], free_row);
    __syncthreads();
    for (int J = 0; J < 8; ++J) {
        const int j0 = 8 * J;
        const double (*D)[9] = DI[J & 1];
        // (b)
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
        if (J == 7) break;
        // (c)
        const int T = 7 - J, j1 = j0 + 8;
        if (wid == 0) {
            tile8_sub_xyt(S + j1 * TS + j1, S + j1 * TS + j0, S + j1 * TS + j0, TS, 1, true);
            __syncwarp();
            if (lane == 0) bad |= chol8_thread(S + j1 * TS + j1, DI[(J + 1) & 1], free_row - j1);
        } else {
            const int nA = T * (T + 1) / 2 - 1, nB = T * (J + 1);
            for (int t = wid - 1; t < nA + nB; t += NTH / 32 - 1) {
                if (t < nA) {              // A tile (I, L), J+1 <= L <= I, not (J+1, J+1)
                    int u = t + 1, I = 0;
                    while (u > I) { u -= I + 1; ++I; }
                    const int L = u;       // I, L relative to J+1
                    const int r0 = j1 + 8 * I, c0 = j1 + 8 * L;
                    tile8_sub_xyt(S + r0 * TS + c0, S + r0 * TS + j0, S + c0 * TS + j0, TS, 1, I == L);
                } else {                   // B tile (I, Lb), I >= J+1, Lb <= J
                    const int u = t - nA, I = u / (J + 1), Lb = u % (J + 1);
                    const int r0 = j1 + 8 * I, c0 = 8 * Lb;
                    tile8_sub_xyt(Li + r0 * TS + c0, S + r0 * TS + j0, Li + j0 * TS + c0, 1, TS, false);
                }
            }
        }
        __syncthreads();
    }
    if (bad) atomicExch(info, 1);
}
template <int NTH = NT>
__device__ __forceinline__ void tile_xyt(double *C, const double *X, const double *Y, double alpha,
                                         bool accumulate) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    double acc[8][2];
    const bool on = NTH == NT || w < 8;     // 8 warps compute (wider CTAs: the rest only sync)
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
        const int r = 8 * (w & 7) + gr, c = 8 * nb + 2 * gc;
        acc[nb][0] = accumulate && on ? C[r * TS + c] : 0.0;
        acc[nb][1] = accumulate && on ? C[r * TS + c + 1] : 0.0;
    }
#pragma unroll 4
    for (int k4 = 0; k4 < (on ? TB / 4 : 0); ++k4) {
        const double av = alpha * X[(8 * w + gr) * TS + 4 * k4 + gc];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) dmma_884(acc[nb][0], acc[nb][1], av, Y[(8 * nb + gr) * TS + 4 * k4 + gc]);
    }
    __syncthreads();
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
        const int r = 8 * w + gr, c = 8 * nb + 2 * gc;
        if (on) {
            C[r * TS + c] = acc[nb][0];
            C[r * TS + c + 1] = acc[nb][1];
        }
    }
    __syncthreads();
}

// ld_tile without the wait: the caller commits / waits (cp.async groups)
__device__ __forceinline__ void ld_tile_async(double *S, const double *src, int ld, int rows, int cols) {
    for (int e = threadIdx.x; e < TB * TB; e += NT) {
        int r = e >> 6, c = e & 63;
        if (r < rows && c < cols) {
            const unsigned s = (unsigned)__cvta_generic_to_shared(S + r * TS + c);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src + (size_t)r * ld + c));
        } else {
            S[r * TS + c] = 0.0;
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

__device__ __forceinline__ bool chol8_fac(double *S, double *rinv, int free_row) {
    double a[8][8];
    bool bad = false;
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) a[r][c] = c <= r ? S[r * TS + c] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        double p = a[k][k];
        bad |= !(p > 0.0) && k < free_row;
        p = p > 0.0 ? p : 1.0;
        const double rs = rsqrt(p);
        rinv[k] = rs;
        a[k][k] = p * rs;
#pragma unroll
        for (int r = k + 1; r < 8; ++r) a[r][k] *= rs;
#pragma unroll
        for (int r = k + 1; r < 8; ++r)
#pragma unroll
            for (int l = k + 1; l <= r; ++l) a[r][l] -= a[r][k] * a[l][k];
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) S[r * TS + c] = a[r][c];
    return bad;
}

// One thread: row i of a panel block, L_iJ = A_iJ L_JJ^{-T} by forward substitution with the
// factored 8x8 block Ljj (stride TS) and its reciprocal pivots.
__device__ __forceinline__ void panel_row8(double *row, const double *Ljj, const double *rinv) {
    double o[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        double acc = row[c];
#pragma unroll
        for (int q = 0; q < c; ++q) acc -= o[q] * Ljj[c * TS + q];
        o[c] = acc * rinv[c];
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) row[c] = o[c];
}

#ifdef CHOL_PROBE
__device__ long long g_cp[8][64];
#define CP_STAMP(w, i) do { if ((threadIdx.x & 31) == 0) g_cp[w][i] = clock64(); } while (0)
#else
#define CP_STAMP(w, i) do {} while (0)
#endif
__device__ void tile_chol64_d(double *S, double (*Dsh)[8][9], int nb, int free_row, int *info) {
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    __shared__ double rinv[64];
    for (int e = tid; e < TB * TB; e += NT) {
        const int r = e >> 6, c = e & 63;
        if (r >= nb || c >= nb) S[r * TS + c] = (r == c) ? 1.0 : 0.0;
        else if (c > r) S[r * TS + c] = 0.0;
    }
    __syncthreads();
    bool bad = false;
    if (tid == 0) bad |= chol8_fac(S, rinv, free_row);
    __syncthreads();
    const int wk = wid < 4 ? wid - 1 : wid - 2;           // worker index 0..5 (wid 1-3, 5-7)
    for (int J = 0; J < 8; ++J) {
        const int j0 = 8 * J, j1 = j0 + 8;
        if (wid == 0) {
            if (J < 7) {
                CP_STAMP(0, 4 * J);
                if (lane < 8) panel_row8(S + (j1 + lane) * TS + j0, S + j0 * TS + j0, rinv + j0);
                __syncwarp();
                CP_STAMP(0, 4 * J + 1);
                asm volatile("bar.arrive 1, 224;\n" ::: "memory");
                tile8_sub_xyt(S + j1 * TS + j1, S + j1 * TS + j0, S + j1 * TS + j0, TS, 1, true);
                __syncwarp();
                CP_STAMP(0, 4 * J + 2);
                if (lane == 0) bad |= chol8_fac(S + j1 * TS + j1, rinv + j1, free_row - j1);
                CP_STAMP(0, 4 * J + 3);
            }
        } else if (wid != 4) {
            const int wt = wk * 32 + lane;
            if (wid == 1) CP_STAMP(1, 4 * J);
            if (j1 + 8 + wt < 64) panel_row8(S + (j1 + 8 + wt) * TS + j0, S + j0 * TS + j0, rinv + j0);
            if (wt >= 160 && wt < 168) {                    // D_J column c = L_JJ^{-1} e_c
                const int c = wt - 160;
                double x[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    double acc = r == c ? 1.0 : 0.0;
#pragma unroll
                    for (int q = 0; q < r; ++q) acc -= S[(j0 + r) * TS + j0 + q] * x[q];
                    x[r] = r >= c ? acc * rinv[j0 + r] : 0.0;
                    Dsh[J][r][c] = x[r];
                }
            }
            if (wid == 1) CP_STAMP(1, 4 * J + 1);
            if (J < 7) {
                asm volatile("bar.sync 1, 224;\n" ::: "memory");
                if (wid == 1) CP_STAMP(1, 4 * J + 2);
                const int I = J + 2 + wk;                  // block row of this worker
                if (I < 8)
                    for (int L = J + 1; L <= I; ++L)
                        tile8_sub_xyt(S + 8 * I * TS + 8 * L, S + 8 * I * TS + j0, S + 8 * L * TS + j0, TS, 1,
                                      I == L);
                if (wid == 1) CP_STAMP(1, 4 * J + 3);
            }
        }
        __syncthreads();
        if (wid == 2) CP_STAMP(2, J);
    }
    if (bad) atomicExch(info, 1);
}

__device__ __forceinline__ void tile_trsm_d(double *X, const double *L, const double (*Dsh)[8][9]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    double *xr = X + (8 * w + gr) * TS;
    for (int J = 0; J < 8; ++J) {
        double c0 = xr[8 * J + 2 * gc], c1 = xr[8 * J + 2 * gc + 1], e0 = 0.0, e1 = 0.0;
        for (int K = 0; K < J; K += 2) {                   // two independent DMMA chains
#pragma unroll
            for (int k4 = 0; k4 < 2; ++k4)
                dmma_884(c0, c1, -xr[8 * K + 4 * k4 + gc], L[(8 * J + gr) * TS + 8 * K + 4 * k4 + gc]);
            if (K + 1 < J) {
#pragma unroll
                for (int k4 = 0; k4 < 2; ++k4)
                    dmma_884(e0, e1, -xr[8 * K + 8 + 4 * k4 + gc], L[(8 * J + gr) * TS + 8 * K + 8 + 4 * k4 + gc]);
            }
        }
        xr[8 * J + 2 * gc] = c0 + e0;
        xr[8 * J + 2 * gc + 1] = c1 + e1;
        __syncwarp();
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int k4 = 0; k4 < 2; ++k4) dmma_884(d0, d1, xr[8 * J + 4 * k4 + gc], Dsh[J][gr][4 * k4 + gc]);
        __syncwarp();
        xr[8 * J + 2 * gc] = d0;
        xr[8 * J + 2 * gc + 1] = d1;
        __syncwarp();
    }
}

__global__ void __launch_bounds__(NT, 1) k_bench(const double *A, double *out, long long *cyc, int reps) {
    extern __shared__ double smx[];
    double *T0 = smx, *T1 = smx + TB * TS, *T2 = smx + 2 * TB * TS;
    __shared__ int info;
    long long tc = 0, tx = 0, td = 0, tt = 0;
    __shared__ double Dsh[8][8][9];
    for (int r = 0; r < reps; ++r) {
        for (int e = threadIdx.x; e < TB * TB; e += NT) T0[(e >> 6) * TS + (e & 63)] = A[e];
        __syncthreads();
        long long t0 = clock64();
        tile_chol64(T0, T1, 64, 64, &info);
        __syncthreads();
        long long t1 = clock64();
        tile_xyt(T2, T1, T1, 1.0, false);
        long long t2 = clock64();
        tc += t1 - t0;
        tx += t2 - t1;
        for (int e = threadIdx.x; e < TB * TB; e += NT) T0[(e >> 6) * TS + (e & 63)] = A[e];
        __syncthreads();
        long long t3 = clock64();
        tile_chol64_d(T0, Dsh, 64, 64, &info);
        __syncthreads();
        long long t4 = clock64();
        tile_trsm_d(T2, T0, Dsh);
        __syncthreads();
        long long t5 = clock64();
        td += t4 - t3;
        tt += t5 - t4;
    }
    if (threadIdx.x == 0) { cyc[0] = tc / reps; cyc[1] = tx / reps; cyc[2] = td / reps; cyc[3] = tt / reps; }
    for (int e = threadIdx.x; e < TB * TB; e += NT) out[e] = T1[(e >> 6) * TS + (e & 63)];
}
int main() {
    double h[64 * 64];
    for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j ? 64.0 : 0.0) + 1.0 / (1 + i + j);
    double *A, *o; long long *c, hc[4];
    cudaMalloc(&A, sizeof(h)); cudaMalloc(&o, sizeof(h)); cudaMalloc(&c, 32);
    cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * TB * TS * 8);
    k_bench<<<1, NT, 3 * TB * TS * 8>>>(A, o, c, 50);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%s: tile_chol64 %lld cycles = %.2f us, tile_xyt %lld cycles = %.2f us\n", cudaGetErrorString(e), hc[0],
           hc[0] / (clk * 1e-3), hc[1], hc[1] / (clk * 1e-3));
    printf("tile_chol64_d (no inverse) %lld cycles = %.2f us, tile_trsm_d %lld cycles = %.2f us\n", hc[2],
           hc[2] / (clk * 1e-3), hc[3], hc[3] / (clk * 1e-3));
}
