// Fused dense Schur step of the contact-reduced global solve in ONE
// persistent cooperative kernel (grid-wide barriers between phases, no host round trips):
//   P0  y_S = -V_s^T w  and  K_s = V_s^T V_s  (= (L_FF^{-1})_SS)
//   P1  Sigma_s = K_s^{-1}  by the symmetric block sweep (Gauss-Jordan on an SPD matrix)
//   P2  Sigma-hat = Sigma_s (x) I3 + B-check, augmented with the row b^T = ((Sigma_s (x) I3) y_S)^T
//   P3  right-looking blocked Cholesky of the augmented matrix: its last row is (C^{-1} b)^T,
//       i.e. the forward substitution comes for free
//   P4  backward substitution u = C^{-T} (C^{-1} b)    (u = dx_S)
//   P5  t = B-check u;  Z = w + V_s t  (input of the final backward supernodal solve)
// PAPER.md:194-198 (Eq. 8: the Schur complement restricted to the collision region) and
// PAPER.md:241-247 (Eq. 11: the update on the n_c contact vertices), here in the K-Schur form
// that never inverts the singular B-check.
// All O(m^3) work runs in 64x64 tiles on the FP64 tensor pipe: mma.sync.m8n8k4.f64 (DMMA).
#include <cooperative_groups.h>

#include "kernels.h"

#include "dev_common.cuh"

namespace cg = cooperative_groups;

namespace pdipc {

constexpr int TB = 64;          // tile
constexpr int TS = 68;          // smem tile stride (DMMA-friendly)
constexpr int NT = 256;         // threads per CTA

__device__ __forceinline__ void dmma_884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

struct SchurArgs {
    // panel
    const double *V;
    int ldv;
    const double *G;            // w [nf][4]
    const int *qS, *col2sn, *sn_c0, *sn_parent, *lo, *hi;
    int nsn, nf, nS;
    // dense buffers
    double *K;                  // [capS][ldk] -> Sigma_s
    int ldk;
    const double *Bc;           // [3capS][ldb]
    int ldb;
    double *Sh;                 // [3capS+1][ldh] augmented Sigma-hat
    int ldh;
    double *Lstore;             // [nt][64][64] inverses of the diagonal factor tiles
    double *T;                  // 64x64 scratch (sweep pivot inverse)
    double *U;                  // sweep panel [capS+64][64]
    double *yS, *u, *t;         // [3capS]
    double *Kpart;              // [grid][32*32] split-K partial tiles
    double *Z;                  // [nf][4]
    int *info;
    unsigned long long *prof;   // optional phase timestamps (PDIPC_TRACE), [1024]
};

__device__ __forceinline__ unsigned long long gtimer_s() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------- tile helpers -----------
// load a rows x cols block (row-major, ld) into smem S (stride TS), zero padded to 64x64
// (asynchronous copies: all 16 loads of a thread are in flight at once; the caller's
// __syncthreads() publishes the tile)
__device__ __forceinline__ void ld_tile(double *S, const double *src, int ld, int rows, int cols) {
    for (int e = threadIdx.x; e < TB * TB; e += NT) {
        int r = e >> 6, c = e & 63;
        if (r < rows && c < cols) {
            const unsigned s = (unsigned)__cvta_generic_to_shared(S + r * TS + c);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src + (size_t)r * ld + c));
        } else {
            S[r * TS + c] = 0.0;
        }
    }
    asm volatile("cp.async.wait_all;\n" ::);
}
__device__ __forceinline__ void st_tile(const double *S, double *dst, int ld, int rows, int cols) {
    for (int e = threadIdx.x; e < TB * TB; e += NT) {
        int r = e >> 6, c = e & 63;
        if (r < rows && c < cols) dst[(size_t)r * ld + c] = S[r * TS + c];
    }
}

// C (64x64 smem) (+)= alpha * X Y^T  (X, Y 64x64 smem), DMMA; 8 warps x (8 rows x 64 cols)
__device__ __forceinline__ void tile_xyt(double *C, const double *X, const double *Y, double alpha,
                                         bool accumulate) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    double acc[8][2];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
        const int r = 8 * w + gr, c = 8 * nb + 2 * gc;
        acc[nb][0] = accumulate ? C[r * TS + c] : 0.0;
        acc[nb][1] = accumulate ? C[r * TS + c + 1] : 0.0;
    }
#pragma unroll 4
    for (int k4 = 0; k4 < TB / 4; ++k4) {
        const double av = alpha * X[(8 * w + gr) * TS + 4 * k4 + gc];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) dmma_884(acc[nb][0], acc[nb][1], av, Y[(8 * nb + gr) * TS + 4 * k4 + gc]);
    }
    __syncthreads();
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
        const int r = 8 * w + gr, c = 8 * nb + 2 * gc;
        C[r * TS + c] = acc[nb][0];
        C[r * TS + c + 1] = acc[nb][1];
    }
    __syncthreads();
}

// One warp: in-place Cholesky of the n x n (n <= 32) block at S (stride TS); pivots after
// row `free_row` (the augmented right-hand-side row) are not checked.
__device__ void chol32_warp(double *S, int n, int free_row, int *info) {
    const int lane = threadIdx.x & 31;
    for (int j = 0; j < n; ++j) {
        double djj = S[j * TS + j];
        if (!(djj > 0.0)) {
            if (j < free_row && lane == 0) atomicExch(info, 1);
            djj = 1.0;
        }
        const double d = sqrt(djj);
        __syncwarp();
        if (lane == j) S[j * TS + j] = d;
        if (lane > j && lane < n) S[lane * TS + j] /= d;
        __syncwarp();
        if (lane > j && lane < n) {
            const double lij = S[lane * TS + j];
            for (int l = j + 1; l <= lane; ++l) S[lane * TS + l] -= lij * S[l * TS + j];
        }
        __syncwarp();
    }
}

// One warp: Li = L^{-1} for the lower n x n block L (n <= 32), lane = column
__device__ void trinv32_warp(const double *L, double *Li, int n) {
    const int c = threadIdx.x & 31;
    for (int i = 0; i < 32; ++i) {
        double v = 0.0;
        if (c < n && i < n && i >= c) {
            double acc = (i == c) ? 1.0 : 0.0;
            for (int q = c; q < i; ++q) acc -= L[i * TS + q] * Li[q * TS + c];
            v = acc / L[i * TS + i];
        }
        Li[i * TS + c] = v;
        __syncwarp();
    }
}

// CTA: Cholesky of the nb x nb (nb <= 64) tile S in place (lower, upper zeroed) and its inverse
// Li (64x64), blocked in 8x8 blocks: per block column one thread factors and inverts the 8x8
// diagonal block in registers, the CTA does the 8-wide TRSM and the rank-8 trailing update
// (3 barriers per block column); the inverse is assembled block row by block row.  Rows >= nb
// are treated as identity.  Pivots at rows >= free_row are not checked.
__device__ void tile_chol64_fast(double *S, double *Li, int nb, int free_row, int *info) {
    const int tid = threadIdx.x;
    __shared__ double DI[8][8][9];                       // inverses of the 8x8 diagonal blocks
    for (int e = tid; e < TB * TB; e += NT) {            // identity padding, zero upper part
        const int r = e >> 6, c = e & 63;
        if (r >= nb || c >= nb) S[r * TS + c] = (r == c) ? 1.0 : 0.0;
        else if (c > r) S[r * TS + c] = 0.0;
    }
    __syncthreads();
    for (int J = 0; J < 8; ++J) {
        const int j0 = 8 * J;
        if (tid < 32) {
            // warp 0: lane r < 8 holds row r of the 8x8 diagonal block; shuffles carry columns
            const int lane = tid, r = lane & 7;
            double a[8], rinv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = (lane < 8 && k <= r) ? S[(j0 + r) * TS + j0 + k] : 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                double p = __shfl_sync(0xffffffffu, a[k], k);
                if (!(p > 0.0)) {
                    if (lane == 0 && j0 + k < free_row) atomicExch(info, 1);
                    p = 1.0;
                }
                // one reciprocal square root per pivot (no division on the pivot chain)
                const double inv = rsqrt(p);
                rinv[k] = inv;
                if (r == k) a[k] = p * inv;
                else if (r > k) a[k] = a[k] * inv;
#pragma unroll
                for (int l = k + 1; l < 8; ++l) {
                    const double llk = __shfl_sync(0xffffffffu, a[k], l);
                    if (r >= l) a[l] -= a[k] * llk;
                }
            }
            // inverse: lane c < 8 solves L x = e_c; L[i][q] comes from lane i; 1/L_ii = rinv[i]
            const int c = lane & 7;
            double x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double acc = (i == c) ? 1.0 : 0.0;
#pragma unroll
                for (int q = 0; q < i; ++q) acc -= __shfl_sync(0xffffffffu, a[q], i) * x[q];
                x[i] = (i >= c) ? acc * rinv[i] : 0.0;
            }
            if (lane < 8) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    S[(j0 + r) * TS + j0 + k] = k <= r ? a[k] : 0.0;
                    DI[J][k][c] = x[k];
                }
            }
        }
        __syncthreads();
        const int nrem = 64 - j0 - 8;
        // TRSM: rows below, S[i][j0..j0+8) <- S[i][j0..] DI_J^T
        for (int e = tid; e < nrem * 8; e += NT) {
            const int i = j0 + 8 + (e >> 3), c = e & 7;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q <= c) acc += S[i * TS + j0 + q] * DI[J][c][q];
            Li[i * TS + c] = acc;                         // Li rows used as scratch
        }
        __syncthreads();
        for (int e = tid; e < nrem * 8; e += NT) {
            const int i = j0 + 8 + (e >> 3), c = e & 7;
            S[i * TS + j0 + c] = Li[i * TS + c];
        }
        __syncthreads();
        // rank-8 trailing update of the lower part (16 x 16 thread grid, no integer division)
        for (int i = j0 + 8 + (tid >> 4); i < 64; i += 16)
            for (int l = j0 + 8 + (tid & 15); l <= i; l += 16) {
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) acc += S[i * TS + j0 + q] * S[l * TS + j0 + q];
                S[i * TS + l] -= acc;
            }
        __syncthreads();
    }
    // inverse: Li_II = DI_I;  Li_IJ = -DI_I sum_{K=J}^{I-1} L_IK Li_KJ   (block row by block row)
    for (int e = tid; e < TB * TB; e += NT) {
        const int r = e >> 6, c = e & 63;
        Li[r * TS + c] = ((r >> 3) == (c >> 3)) ? DI[r >> 3][r & 7][c & 7] : 0.0;
    }
    __syncthreads();
    __shared__ double Tmp[8][64];
    for (int I = 1; I < 8; ++I) {
        const int i0 = 8 * I;
        {                                                 // Tmp = sum_K L_IK Li_KJ, cols < i0
            const int r = tid >> 5, c0 = tid & 31;        // 8 rows x 32 lanes, 2 columns each
            for (int c = c0; c < i0; c += 32) {
                double acc = 0.0;
#pragma unroll 8
                for (int q = (c & ~7); q < i0; ++q) acc += S[(i0 + r) * TS + q] * Li[q * TS + c];
                Tmp[r][c] = acc;
            }
        }
        __syncthreads();
        {
            const int r = tid >> 5, c0 = tid & 31;
            for (int c = c0; c < i0; c += 32) {
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q <= r) acc += DI[I][r][q] * Tmp[q][c];
                Li[(i0 + r) * TS + c] = -acc;
            }
        }
        __syncthreads();
    }
}

// CTA: Cholesky of the nb x nb (nb <= 64) tile S in place (lower, upper zeroed) and its inverse
// Li (64x64, zero padded).  W is a 64x64 scratch tile.  free_row: see chol32_warp.
__device__ void tile_chol64(double *S, double *Li, double *W, int nb, int free_row, int *info) {
    const int tid = threadIdx.x, w = tid >> 5;
    const int n1 = min(32, nb), n2 = nb - n1;
    for (int e = tid; e < TB * TB; e += NT) Li[(e >> 6) * TS + (e & 63)] = 0.0;
    __syncthreads();
    if (w == 0) chol32_warp(S, n1, free_row, info);
    __syncthreads();
    if (w == 0) trinv32_warp(S, Li, n1);                 // Li11
    __syncthreads();
    if (n2 > 0) {
        // A21 <- A21 Li11^T   (rows 32..nb-1, cols 0..31)
        for (int e = tid; e < 32 * 32; e += NT) {
            const int r = e >> 5, c = e & 31;
            double acc = 0.0;
            if (r < n2)
                for (int q = 0; q <= c; ++q) acc += S[(32 + r) * TS + q] * Li[c * TS + q];
            W[r * TS + c] = acc;
        }
        __syncthreads();
        for (int e = tid; e < 32 * 32; e += NT) {
            const int r = e >> 5, c = e & 31;
            if (r < n2) S[(32 + r) * TS + c] = W[r * TS + c];
        }
        __syncthreads();
        // A22 -= L21 L21^T (lower part)
        for (int e = tid; e < 32 * 32; e += NT) {
            const int r = e >> 5, c = e & 31;
            if (r < n2 && c <= r) {
                double acc = 0.0;
                for (int q = 0; q < 32; ++q) acc += S[(32 + r) * TS + q] * S[(32 + c) * TS + q];
                S[(32 + r) * TS + 32 + c] -= acc;
            }
        }
        __syncthreads();
        if (w == 0) chol32_warp(S + 32 * TS + 32, n2, free_row - 32, info);
        __syncthreads();
        if (w == 0) trinv32_warp(S + 32 * TS + 32, Li + 32 * TS + 32, n2);   // Li22
        __syncthreads();
        // Li21 = -Li22 L21 Li11
        for (int e = tid; e < 32 * 32; e += NT) {       // W = L21 Li11
            const int r = e >> 5, c = e & 31;
            double acc = 0.0;
            if (r < n2)
                for (int q = c; q < 32; ++q) acc += S[(32 + r) * TS + q] * Li[q * TS + c];
            W[r * TS + c] = acc;
        }
        __syncthreads();
        for (int e = tid; e < 32 * 32; e += NT) {
            const int r = e >> 5, c = e & 31;
            double acc = 0.0;
            if (r < n2)
                for (int q = 0; q <= r; ++q) acc += Li[(32 + r) * TS + 32 + q] * W[q * TS + c];
            Li[(32 + r) * TS + c] = -acc;
        }
        __syncthreads();
    }
    for (int e = tid; e < TB * TB; e += NT) {            // clean the upper triangle / padding
        const int r = e >> 6, c = e & 63;
        if (c > r || r >= nb || c >= nb) S[r * TS + c] = 0.0;
    }
    __syncthreads();
}

// ---------------------------------------------------------------- the kernel ---------------
__global__ void __launch_bounds__(NT, 1) k_schur_coop(SchurArgs a) {
    extern __shared__ double sm[];
    double *T0 = sm, *T1 = sm + TB * TS, *T2 = sm + 2 * TB * TS, *T3 = sm + 3 * TB * TS;
    __shared__ double red[32];
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x, bid = blockIdx.x;
    const int nS = a.nS, m = 3 * nS, ma = m + 1;          // augmented size
    int np = 0;                                           // phase-timestamp counter (debug)
    if (a.prof && bid == 0 && tid == 0) a.prof[np++] = gtimer_s();
#define GSYNC()                                                               \
    do {                                                                      \
        grid.sync();                                                          \
        if (a.prof && bid == 0 && tid == 0 && np < 1023) a.prof[np++] = gtimer_s(); \
    } while (0)
    // ------------------------------------------------ P0: y_S and K = V^T V
    for (int c = bid; c < nS; c += G) {
        double acc[3] = {0, 0, 0};
        for (int s = a.col2sn[a.qS[c]]; s >= 0; s = a.sn_parent[s])
            for (int r = a.sn_c0[s] + tid; r < a.sn_c0[s + 1]; r += NT) {
                const double v = a.V[(size_t)r * a.ldv + c];
                acc[0] += v * a.G[(size_t)r * 4 + 0];
                acc[1] += v * a.G[(size_t)r * 4 + 1];
                acc[2] += v * a.G[(size_t)r * 4 + 2];
            }
        for (int i = 0; i < 3; ++i) {
            double tsum = block_sum<NT>(acc[i], red);
            if (tid == 0) a.yS[3 * c + i] = -tsum;
        }
    }
    const int ntk = (nS + 31) / 32;                  // 32x32 tiles of K (lower)
    const int ntiles = ntk * (ntk + 1) / 2;
    // split the supernode (row) loop of each tile over nsplit CTAs when tiles are few;
    // partial tiles are reduced in a fixed order afterwards (deterministic)
    const int nsplit = max(1, min(8, G / max(ntiles, 1)));
    {
        double *Va = T0, *Vb = T1;                   // 32 x 33 each
        for (int bs = bid; bs < ntiles * nsplit; bs += G) {
            const int b = bs / nsplit, split = bs % nsplit;
            int ti = 0, rem = b;
            while (rem > ti) { rem -= ti + 1; ++ti; }
            const int tj = rem;
            const int ia = ti * 32, ja = tj * 32;
            const int tx = tid & 31, ty = tid >> 5;
            double acc[4] = {0, 0, 0, 0};
            for (int s = split; s < a.nsn; s += nsplit) {
                const int l = a.lo[s], h = a.hi[s];
                if (h <= l || l >= min(ia + 32, nS) || h <= ia || l >= ja + 32 || h <= ja) continue;
                const int c0 = a.sn_c0[s], c1 = a.sn_c0[s + 1];
                for (int rb = c0; rb < c1; rb += 32) {
                    const int nrb = min(32, c1 - rb);
                    for (int e = tid; e < 32 * 32; e += NT) {
                        const int rr = e >> 5, cc = e & 31;
                        const int ca = ia + cc, cb = ja + cc;
                        double va = 0, vb = 0;
                        if (rr < nrb) {
                            if (ca >= l && ca < h && ca < nS) va = a.V[(size_t)(rb + rr) * a.ldv + ca];
                            if (cb >= l && cb < h && cb < nS) vb = a.V[(size_t)(rb + rr) * a.ldv + cb];
                        }
                        Va[rr * 33 + cc] = va;
                        Vb[rr * 33 + cc] = vb;
                    }
                    __syncthreads();
                    for (int rr = 0; rr < nrb; ++rr) {
                        const double bv = Vb[rr * 33 + tx];
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc[k] += Va[rr * 33 + ty * 4 + k] * bv;
                    }
                    __syncthreads();
                }
            }
            if (nsplit == 1) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int r = ia + ty * 4 + k, c = ja + tx;
                    if (r < nS && c < nS && c <= r) {
                        a.K[(size_t)r * a.ldk + c] = acc[k];
                        a.K[(size_t)c * a.ldk + r] = acc[k];
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) a.Kpart[(size_t)bs * 1024 + (ty * 4 + k) * 32 + tx] = acc[k];
            }
        }
    }
    if (nsplit > 1) {
        GSYNC();
        for (int b = bid; b < ntiles; b += G) {
            int ti = 0, rem = b;
            while (rem > ti) { rem -= ti + 1; ++ti; }
            const int tj = rem;
            for (int e = tid; e < 1024; e += NT) {
                double acc = 0.0;
                for (int sp = 0; sp < nsplit; ++sp) acc += a.Kpart[((size_t)b * nsplit + sp) * 1024 + e];
                const int r = ti * 32 + (e >> 5), c = tj * 32 + (e & 31);
                if (r < nS && c < nS && c <= r) {
                    a.K[(size_t)r * a.ldk + c] = acc;
                    a.K[(size_t)c * a.ldk + r] = acc;
                }
            }
        }
    }
    GSYNC();
    // ------------------------------------------------ P1: K <- -K^{-1} (block sweep)
    {
        const int nt = (nS + TB - 1) / TB;
        for (int k = 0; k < nt; ++k) {
            const int kc0 = k * TB, kn = min(TB, nS - kc0);
            if (bid == 0) {          // P = A_kk^{-1} = Li^T Li
                ld_tile(T0, a.K + (size_t)kc0 * a.ldk + kc0, a.ldk, kn, kn);
                __syncthreads();
                tile_chol64_fast(T0, T1, kn, kn, a.info);
                for (int e = tid; e < TB * TB; e += NT) {
                    const int r = e >> 6, c = e & 63;
                    double acc = 0.0;
                    for (int q = max(r, c); q < kn; ++q) acc += T1[q * TS + r] * T1[q * TS + c];
                    a.T[e] = acc;
                }
            }
            GSYNC();
            for (int b = bid; b < nt - 1; b += G) {      // U_i = A_ik P, i != k
                const int ti = b < k ? b : b + 1;
                const int r0 = ti * TB, rows = min(TB, nS - r0);
                ld_tile(T0, a.K + (size_t)r0 * a.ldk + kc0, a.ldk, rows, kn);
                ld_tile(T1, a.T, TB, TB, TB);
                __syncthreads();
                tile_xyt(T2, T0, T1, 1.0, false);
                st_tile(T2, a.U + (size_t)r0 * TB, TB, rows, TB);
            }
            GSYNC();
            for (int b = bid; b < (nt - 1) * (nt - 1); b += G) {   // A_ij -= U_i A_jk^T
                const int bi = b / (nt - 1), bj = b % (nt - 1);
                const int ti = bi < k ? bi : bi + 1, tj = bj < k ? bj : bj + 1;
                const int r0 = ti * TB, c0 = tj * TB;
                const int rows = min(TB, nS - r0), cols = min(TB, nS - c0);
                ld_tile(T0, a.U + (size_t)r0 * TB, TB, rows, TB);
                ld_tile(T1, a.K + (size_t)c0 * a.ldk + kc0, a.ldk, cols, kn);
                ld_tile(T2, a.K + (size_t)r0 * a.ldk + c0, a.ldk, rows, cols);
                __syncthreads();
                tile_xyt(T2, T0, T1, -1.0, true);
                st_tile(T2, a.K + (size_t)r0 * a.ldk + c0, a.ldk, rows, cols);
            }
            GSYNC();
            for (size_t e = (size_t)bid * NT + tid; e < (size_t)nS * kn; e += (size_t)G * NT) {
                const int r = (int)(e / kn), c = (int)(e % kn);
                const double v = (r >= kc0 && r < kc0 + kn) ? -a.T[(r - kc0) * TB + c] : a.U[(size_t)r * TB + c];
                a.K[(size_t)r * a.ldk + kc0 + c] = v;
                a.K[(size_t)(kc0 + c) * a.ldk + r] = v;
            }
            GSYNC();
        }
    }
    // ------------------------------------------------ P2: augmented Sigma-hat (Sigma_s = -K)
    for (size_t e = (size_t)bid * NT + tid; e < (size_t)m * m; e += (size_t)G * NT) {
        const int r = (int)(e / m), c = (int)(e % m);
        if (c > r) continue;
        double v = a.Bc[(size_t)r * a.ldb + c];
        if (r % 3 == c % 3) v -= a.K[(size_t)(r / 3) * a.ldk + c / 3];
        a.Sh[(size_t)r * a.ldh + c] = v;
    }
    for (int row = bid * (NT / 32) + wid; row < m; row += G * (NT / 32)) {   // b = Sigma_s yS
        const int ai = row / 3, i = row % 3;
        double acc = 0.0;
        for (int bb = lane; bb < nS; bb += 32) acc -= a.K[(size_t)ai * a.ldk + bb] * a.yS[3 * bb + i];
        acc = warp_sum(acc);
        if (lane == 0) a.Sh[(size_t)m * a.ldh + row] = acc;
    }
    if (bid == 0 && tid == 0) a.Sh[(size_t)m * a.ldh + m] = 1.0;
    GSYNC();
    // ------------------------------------------------ P3: Cholesky of the augmented matrix
    const int nt = (ma + TB - 1) / TB;
    for (int k = 0; k < nt; ++k) {
        const int kc0 = k * TB, kn = min(TB, ma - kc0);
        if (bid == 0) {
            ld_tile(T0, a.Sh + (size_t)kc0 * a.ldh + kc0, a.ldh, kn, kn);
            __syncthreads();
            tile_chol64_fast(T0, T1, kn, m - kc0, a.info);
            st_tile(T0, a.Sh + (size_t)kc0 * a.ldh + kc0, a.ldh, kn, kn);
            for (int e = tid; e < TB * TB; e += NT) a.Lstore[(size_t)k * TB * TB + e] = T1[(e >> 6) * TS + (e & 63)];
        }
        GSYNC();
        for (int b = bid; b < nt - k - 1; b += G) {      // L_ik = A_ik Li^T
            const int ti = k + 1 + b, r0 = ti * TB, rows = min(TB, ma - r0);
            ld_tile(T0, a.Sh + (size_t)r0 * a.ldh + kc0, a.ldh, rows, kn);
            ld_tile(T1, a.Lstore + (size_t)k * TB * TB, TB, TB, TB);
            __syncthreads();
            tile_xyt(T2, T0, T1, 1.0, false);
            st_tile(T2, a.Sh + (size_t)r0 * a.ldh + kc0, a.ldh, rows, kn);
        }
        GSYNC();
        const int rr = nt - k - 1;
        for (int b = bid; b < rr * (rr + 1) / 2; b += G) {   // A_ij -= L_ik L_jk^T, k < j <= i
            int i = 0, bb = b;
            while (bb >= rr - i) { bb -= rr - i; ++i; }
            const int tj = k + 1 + i, ti = tj + bb;
            const int r0 = ti * TB, c0 = tj * TB, rows = min(TB, ma - r0), cols = min(TB, ma - c0);
            ld_tile(T0, a.Sh + (size_t)r0 * a.ldh + kc0, a.ldh, rows, kn);
            ld_tile(T1, a.Sh + (size_t)c0 * a.ldh + kc0, a.ldh, cols, kn);
            ld_tile(T2, a.Sh + (size_t)r0 * a.ldh + c0, a.ldh, rows, cols);
            __syncthreads();
            tile_xyt(T2, T0, T1, -1.0, true);
            st_tile(T2, a.Sh + (size_t)r0 * a.ldh + c0, a.ldh, rows, cols);
        }
        GSYNC();
    }
    // ------------------------------------------------ P4: u = C^{-T} y, y = row m of the factor
    // right-looking on C^T: u_k = Li_k^T y_k, then y_j -= (C_kj)^T u_k for j < k
    for (int e = bid * NT + tid; e < m; e += G * NT) a.u[e] = a.Sh[(size_t)m * a.ldh + e];
    GSYNC();
    const int ntm = (m + TB - 1) / TB;
    for (int k = ntm - 1; k >= 0; --k) {
        const int kc0 = k * TB, kn = min(TB, m - kc0);
        if (bid == 0) {
            double *yk = T3;                      // stage y_k
            for (int i = tid; i < TB; i += NT) yk[i] = i < kn ? a.u[kc0 + i] : 0.0;
            __syncthreads();
            const double *Li = a.Lstore + (size_t)k * TB * TB;
            for (int i = tid; i < kn; i += NT) {  // u_k[i] = sum_r Li[r][i] y_k[r]
                double acc = 0.0;
                for (int r = i; r < kn; ++r) acc += Li[r * TB + i] * yk[r];
                a.u[kc0 + i] = acc;
            }
        }
        GSYNC();
        // y_j -= C_kj^T u_k  for rows j < kc0 (block row k of the factor, columns j)
        for (int j = bid * NT + tid; j < kc0; j += G * NT) {
            double acc = 0.0;
            for (int r = 0; r < kn; ++r) acc += a.Sh[(size_t)(kc0 + r) * a.ldh + j] * a.u[kc0 + r];
            a.u[j] -= acc;
        }
        GSYNC();
    }
    // ------------------------------------------------ P5: t = B u ; Z = w + V t
    for (int row = bid * (NT / 32) + wid; row < m; row += G * (NT / 32)) {
        double acc = 0.0;
        for (int c = lane; c < m; c += 32) acc += a.Bc[(size_t)row * a.ldb + c] * a.u[c];
        acc = warp_sum(acc);
        if (lane == 0) a.t[row] = acc;
    }
    GSYNC();
    for (int r = bid * NT + tid; r < a.nf; r += G * NT) {
        const int s = a.col2sn[r];
        double z0 = a.G[(size_t)r * 4 + 0], z1 = a.G[(size_t)r * 4 + 1], z2 = a.G[(size_t)r * 4 + 2];
        for (int c = a.lo[s]; c < a.hi[s]; ++c) {
            const double v = a.V[(size_t)r * a.ldv + c];
            z0 += v * a.t[3 * c + 0];
            z1 += v * a.t[3 * c + 1];
            z2 += v * a.t[3 * c + 2];
        }
        a.Z[(size_t)r * 4 + 0] = z0;
        a.Z[(size_t)r * 4 + 1] = z1;
        a.Z[(size_t)r * 4 + 2] = z2;
        a.Z[(size_t)r * 4 + 3] = 0.0;
    }
}

constexpr int kSchurSmem = 4 * TB * TS * (int)sizeof(double);
static int g_schur_grid = 0;

void schur_init(int device) {
    cudaFuncSetAttribute(k_schur_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, kSchurSmem);
    int per_sm = 0, nsm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_schur_coop, NT, kSchurSmem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    g_schur_grid = std::max(1, per_sm) * nsm;
}

int launch_schur(const DevFactor &F, const double *V, int ldv, const double *G, const int *qS,
                 const int *lo, const int *hi, int nS, double *K, int ldk, const double *Bc, int ldb,
                 double *Sh, int ldh, double *Lstore, double *T, double *U, double *yS, double *u,
                 double *t, double *Z, int *info, unsigned long long *prof, cudaStream_t st) {
    SchurArgs a;
    a.V = V; a.ldv = ldv; a.G = G; a.qS = qS; a.col2sn = F.col2sn; a.sn_c0 = F.sn_c0;
    a.sn_parent = F.sn_parent; a.lo = lo; a.hi = hi; a.nsn = F.nsn; a.nf = F.nf; a.nS = nS;
    a.K = K; a.ldk = ldk; a.Bc = Bc; a.ldb = ldb; a.Sh = Sh; a.ldh = ldh; a.Lstore = Lstore;
    a.T = T; a.U = U; a.yS = yS; a.u = u; a.t = t; a.Z = Z; a.info = info; a.prof = prof;
    static double *kpart = nullptr;                 // grid x 1024 doubles, allocated once
    if (!kpart) cudaMalloc(&kpart, (size_t)g_schur_grid * 1024 * sizeof(double));
    a.Kpart = kpart;
    void *args[] = {&a};
    note_launch();
    return (int)cudaLaunchCooperativeKernel((const void *)k_schur_coop, dim3(g_schur_grid), dim3(NT),
                                             args, kSchurSmem, st);
}

}  // namespace pdipc
