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
#include "prims.h"
#include <cstring>
#include <cudaTypedefs.h>

#include "dev_common.cuh"

namespace cg = cooperative_groups;

namespace pdipc {

constexpr int TB = 64;          // tile
constexpr int TS = 68;          // smem tile stride (DMMA-friendly)
constexpr int NT = 256;         // threads per CTA
constexpr int kPW = 4;          // P3 panel width in tiles (trailing update once per panel)
constexpr int kPWMinTiles = 21; // ... for systems of at least this many tiles (m >= 1280)
constexpr int kLPTiles = kPWMinTiles;   // small-system P3: panel tiles per step
// 4 tiles (P0-P3); the small-system P4 needs y, u (m each), 2 X tiles and 8 partial rows
constexpr int kSmallMaxM = TB * (kPWMinTiles - 1);
constexpr int kSchurSmemBase = (10 * kSmallMaxM + 8 + 2 * 64 * 65) * (int)sizeof(double);   // y, u, X[2], 8 partials
// large-system trailing updates: kTmaStages stages of one 32-wide k chunk of a 128 x 64 block
// (X: 128 rows, Y: 64 rows, 256 B each, dense with the 128-byte TMA swizzle), 1024-B aligned
constexpr int kTmaStages = 4, kTmaAhead = 3, kTmaStageB = 192 * 256;
constexpr int cmax(int x, int y) { return x > y ? x : y; }
// (P1's update pipeline: two sets of three 64 x 64 tiles)
constexpr int kSchurSmem = cmax(cmax(kSchurSmemBase, kTmaStages * kTmaStageB + 1024), 6 * TB * TS * 8);
static_assert(kSchurSmem >= 4 * TB * TS * (int)sizeof(double), "smem");

__device__ __forceinline__ void dmma_884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}



// Barrier among the `target / k`-member group that shares counter *ctr (k-th use: target =
// k x members).  Members are co-resident (cooperative launch).
__device__ __forceinline__ void group_bar(unsigned *ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        volatile unsigned *v = ctr;
        while (*v < target) __nanosleep(32);
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer_s() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------- tile helpers -----------
// load a rows x cols block (row-major, ld) into smem S (stride TS), zero padded to 64x64
// (asynchronous copies: all 16 loads of a thread are in flight at once; the caller's
// __syncthreads() publishes the tile)
template <int NTH = NT>
__device__ __forceinline__ void ld_tile(double *S, const double *src, int ld, int rows, int cols) {
    for (int e = threadIdx.x; e < TB * TB; e += NTH) {
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
// S[r][c] = src[c * ld + r] (the transposed rows x cols block), zero padded
__device__ __forceinline__ void ld_tile_T(double *S, const double *src, int ld, int rows, int cols) {
    for (int e = threadIdx.x; e < TB * TB; e += NT) {
        const int c = e >> 6, r = e & 63;
        S[r * TS + c] = (r < rows && c < cols) ? src[(size_t)c * ld + r] : 0.0;
    }
}
template <int NTH = NT>
__device__ __forceinline__ void st_tile(const double *S, double *dst, int ld, int rows, int cols) {
    for (int e = threadIdx.x; e < TB * TB; e += NTH) {
        int r = e >> 6, c = e & 63;
        if (r < rows && c < cols) dst[(size_t)r * ld + c] = S[r * TS + c];
    }
}

// C (64x64 smem) (+)= alpha * X Y^T  (X, Y 64x64 smem), DMMA; 8 warps x (8 rows x 64 cols)
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

// acc (warp w: rows 8w..8w+7, all 64 columns, fragment layout of tile_xyt) += X Y^T on DMMA (the
// caller keeps the accumulator negated to subtract: no per-step negation on the operand path)
__device__ __forceinline__ void tile_add_xyt_regs(double (&acc)[8][2], const double *X, const double *Y) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    const double *xr = X + (8 * w + gr) * TS + gc;
    const double *yr = Y + gr * TS + gc;
#pragma unroll 4
    for (int k4 = 0; k4 < TB / 4; ++k4) {
        const double av = xr[4 * k4];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) dmma_884(acc[nb][0], acc[nb][1], av, yr[8 * nb * TS + 4 * k4]);
    }
}

// acc (warp w: rows 8w..8w+7, all 64 columns, fragment layout of tile_xyt) -= X Y^T on DMMA
__device__ __forceinline__ void tile_sub_xyt_regs(double (&acc)[8][2], const double *X, const double *Y) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, gc = lane & 3;
#pragma unroll 4
    for (int k4 = 0; k4 < TB / 4; ++k4) {
        const double av = -X[(8 * w + gr) * TS + 4 * k4 + gc];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) dmma_884(acc[nb][0], acc[nb][1], av, Y[(8 * nb + gr) * TS + 4 * k4 + gc]);
    }
}

// One thread: Cholesky of the 8x8 diagonal block at S (stride TS, lower part read) in
// registers, its inverse into D (8 x 9), L written back to S.  Returns true on a bad pivot
// below free_row (relative to the block).
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

// One warp: C (8x8 at smem, stride TS) -= X Y^T with X, Y 8 x 8 (X[r][k] at X + r*TS + k,
// Y[n][k] at Y + n*ys_row + k*ys_col) on DMMA (2 k-steps); lower_only keeps C's strict upper
// triangle untouched (diagonal tiles).
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

// CTA: Cholesky of the nb x nb (nb <= 64) tile S in place (lower, upper and padding zeroed,
// rows >= nb identity) and its inverse Li, in 8-wide block columns with one block of
// look-ahead.  Per block column J (two barriers):
//   (b) thread per row: L_IJ = A_IJ D_J^{-T}; thread per column: B_J <- D_J^{-1} B_J
//       (B starts as I and ends as L^{-1});
//   (c) warp 0 updates the next diagonal block and ONE thread factors and inverts it in
//       registers, while warps 1..7 apply the rank-8 updates A_IL -= L_IJ L_LJ^T and
//       B_I -= L_IJ B_J on DMMA.
// Pivots at rows >= free_row are not checked.
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


// ---------------------------------------------------------------- small-system tile kernels --
// One thread: Cholesky of the 8x8 diagonal block at S (stride TS, lower part read) in
// registers, L written back to S, the reciprocal pivots to rinv[0..7].  Returns true on a bad
// pivot below free_row (relative to the block).
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

// Diagonal-tile factor without the explicit inverse: L (in place, lower; upper and padding
// zeroed, rows >= nb identity) and the inverses D_J of its eight 8x8 diagonal blocks (Dsh[J]),
// which is all the blocked triangular solves need.  Right-looking over 8-wide block columns
// with the critical chain on warp 0: per block column J, warp 0 forms the panel rows of block
// J+1 (lanes 0..7, forward substitution), updates the diagonal block (J+1, J+1) on DMMA and one
// lane factors it; meanwhile the worker warps 1-3, 5-7 form the other panel rows, D_J, and apply
// the rank-8 updates A_IL -= L_IJ L_LJ^T of block rows I >= J+2 (warp 4 shares warp 0's SM
// sub-partition and FP64 pipe and stays idle).  Named barrier 1 (224 threads) hands warp 0's
// panel rows to the workers.  Pivots at rows >= free_row are not checked.
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

// X <- X L^{-T} for a 64x64 tile X (rows independent) with L the factored diagonal tile and
// Dsh its 8x8 diagonal-block inverses: per 8-wide block column J,
// X_J = (X_J - sum_{K<J} X_K L_JK^T) D_J^T.  Warp w owns rows 8w..8w+7 (no CTA barrier inside;
// the caller's __syncthreads publishes X).
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

// C -= X X^T on the 36 lower 8x8 blocks of a 64x64 tile (the upper blocks are not touched);
// warp w accumulates blocks w, w+8, ... in registers (independent DMMA chains)
__device__ __forceinline__ void tile_syrk_lower_sub(double *C, const double *X) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    double acc[5][2];
    int bi[5], bl[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int b = w + 8 * j;
        int I = 0, u = b < 36 ? b : 0;
        while (u > I) { u -= I + 1; ++I; }
        bi[j] = I;
        bl[j] = u;
        acc[j][0] = b < 36 ? C[(8 * I + gr) * TS + 8 * u + 2 * gc] : 0.0;
        acc[j][1] = b < 36 ? C[(8 * I + gr) * TS + 8 * u + 2 * gc + 1] : 0.0;
    }
#pragma unroll 4
    for (int k4 = 0; k4 < TB / 4; ++k4) {
#pragma unroll
        for (int j = 0; j < 5; ++j)
            if (w + 8 * j < 36)
                dmma_884(acc[j][0], acc[j][1], -X[(8 * bi[j] + gr) * TS + 4 * k4 + gc],
                         X[(8 * bl[j] + gr) * TS + 4 * k4 + gc]);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 5; ++j)
        if (w + 8 * j < 36) {
            C[(8 * bi[j] + gr) * TS + 8 * bl[j] + 2 * gc] = acc[j][0];
            C[(8 * bi[j] + gr) * TS + 8 * bl[j] + 2 * gc + 1] = acc[j][1];
        }
    __syncthreads();
}

__device__ __forceinline__ void st_dblocks(const double (*Dsh)[8][9], double *dst) {
    for (int e = threadIdx.x; e < 512; e += NT) dst[e] = Dsh[e >> 6][(e >> 3) & 7][e & 7];
}
__device__ __forceinline__ void ld_dblocks(double (*Dsh)[8][9], const double *src) {
    for (int e = threadIdx.x; e < 512; e += NT) Dsh[e >> 6][(e >> 3) & 7][e & 7] = src[e];
}

// ---------------------------------------------------------------- the kernel ---------------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                 "@!P1 bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(NT, 1) k_schur_coop(const __grid_constant__ SchurBatch P) {
    extern __shared__ double sm[];
    // TMA ring of the large-system trailing updates: full[s] (TMA bytes landed), empty[s] (the 8
    // warps are done with stage s); phases tracked by the chunk counter tma_g (uniform per CTA)
    __shared__ __align__(8) unsigned long long tma_bar[2 * kTmaStages];
    double *T0 = sm, *T1 = sm + TB * TS, *T2 = sm + 2 * TB * TS, *T3 = sm + 3 * TB * TS;
    // CTA group grp runs system P.s[grp]: group-local CTA index and count, group barriers.  The
    // systems of a launch split the grid in proportion to their work m^wexp (m = 3 n_c + 1, wexp 2.5
    // by default; read from the device-resident |S| of every system, identical on every CTA),
    // so a smaller system does not idle while a larger one finishes.  Group g owns CTAs
    // [start_g, start_{g+1}), start_{g+1} = round(grid x W_<=g / W), at least one CTA each (a system
    // without contact returns at once).  A system's arithmetic does not depend on its CTA count
    // (batched == single runs, bit for bit).
    int grp = 0, gsz = gridDim.x, gbase = 0;
    {
        double w[kMaxSchurSys], W = 0.0;
        for (int g = 0; g < P.nsys; ++g) {
            const double m = 3.0 * min(*P.s[g].nS_ptr, P.s[g].capS) + 1.0;
            w[g] = P.wexp == 3.0 ? m * m * m : pow(m, P.wexp);
            W += w[g];
        }
        double cum = 0.0;
        int start = 0;
        for (int g = 0; g < P.nsys; ++g) {
            cum += w[g];
            const int next = g == P.nsys - 1 ? (int)gridDim.x
                                             : min((int)gridDim.x - (P.nsys - 1 - g),
                                                   max(start + 1, (int)lrint((double)gridDim.x * cum / W)));
            if ((int)blockIdx.x >= start && (int)blockIdx.x < next) {
                grp = g;
                gbase = start;
                gsz = next - start;
            }
            start = next;
        }
    }
    if (grp >= P.nsys) return;
    __shared__ SchurArgs a_sh;
    if (threadIdx.x == 0) {
        a_sh = P.s[grp];
        a_sh.Kpart = P.s[0].Kpart + (size_t)gbase * 1152;   // per-CTA split-K partials of the group
        for (int i = 0; i < kTmaStages; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&tma_bar[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&tma_bar[kTmaStages + i])),
                         "r"(NT / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    unsigned tma_g = 0;                                   // k chunks streamed so far (TMA ring)
    const SchurArgs &a = a_sh;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gsz, bid = blockIdx.x - gbase;
    unsigned nsync = 0;
    const int nS = min(*a.nS_ptr, a.capS), m = 3 * nS, ma = m + 1;   // augmented size
    if (nS == 0) {   // no contact: z = w = w_el (gather backend: the sparse right-hand side is 0)
        for (int r = bid * NT + tid; r < 4 * a.nf; r += G * NT) a.Z[r] = a.mode == kSchurGather ? 0.0 : a.G[r];
        return;
    }
    int np = 0;                                           // phase-timestamp counter (debug)
    const bool large = (ma + TB - 1) / TB >= a.pw_min && a.phase != 0;
    if (a.phase == 2 && !large) return;                   // small system: done in phase 1
    if (a.phase == 2 && a.prof) np = (int)a.prof[999];    // timestamps continue after P3
    if (a.prof && bid == 0 && tid == 0 && a.phase != 2) a.prof[np++] = gtimer_s();
    if (a.phase != 2) {                                   // ---------------- P0 .. P3
#define GSYNC()                                                               \
    do {                                                                      \
        group_bar(a.gbar, ++nsync * (unsigned)G);                             \
        if (a.prof && bid == 0 && tid == 0 && np < 1000) a.prof[np++] = gtimer_s(); \
    } while (0)
    // ------------------------------------------------ P0: y_S = -V_s^T w and K = V_s^T V_s
    // Tile-parallel over the 32x32 lower tiles of K, split over the supernodes (rows) when tiles
    // are few; every CTA streams the 32-row chunks of its supernodes whose active column range
    // [lo_s, hi_s) meets both tile ranges (cp.async double buffer, inactive entries zeroed) and
    // accumulates on DMMA.  Diagonal tiles also accumulate y_S for their columns.  Split partials
    // are reduced in a fixed order (deterministic).
    const bool reuse = *a.same != 0;                 // uniform across the grid
    // S changed by a few vertices: Sigma_s updated by low-rank steps from the slot's previous one
    const bool supd = !reuse && a.uinfo != nullptr && a.uinfo[0] != 0;
    // Small systems with Sigma_s reused: CTA 0 assembles and factors the first diagonal tile of
    // Sigma-hat right away (it needs only B-check and the stored Sigma_s), while the other CTAs
    // run P0 and P2 -- the first tile factorisation leaves the critical path
    const int nt0 = (ma + TB - 1) / TB;
    const bool early0 = reuse && nt0 >= 2 && nt0 < a.pw_min && G > 1;
    const int pb = early0 ? bid - 1 : bid, pG = early0 ? G - 1 : G;   // P0 / P2 workers
    __shared__ double Dsh[2][8][8][9];   // small-system P3: [0] D_k of the step, [1] look-ahead
    if (early0 && bid == 0) {
        for (int e = tid; e < TB * TB; e += NT) {
            const int r = e >> 6, c = e & 63;
            double v = 0.0;
            if (c <= r) {
                v = a.Bc[(size_t)r * a.ldb + c];
                if (r % 3 == c % 3) v -= a.K[(size_t)(r / 3) * a.ldk + c / 3];
            }
            T0[r * TS + c] = v;
        }
        __syncthreads();
        tile_chol64_d(T0, Dsh[0], TB, m, a.info);
        __syncthreads();
        st_tile(T0, a.Sh, a.ldh, TB, TB);
        st_dblocks(Dsh[0], a.Lstore);
        __syncthreads();
    }
    // y_S^el[c] = -sum over the etree path of q_c's supernode of V[r][c] w_el[r] (the elastic
    // part; the contact part -K gc is folded into b below since Sigma_s K = I): one CTA per column,
    // the path rows come from a static per-supernode list (independent loads), fixed-order
    // block reduction: the same bits whether or not K is recomputed
    if (a.mode == kSchurGather) {   // y_S = -(L^-T L^-1 Pi g_el)_S: rows S of the base solve
        for (int e = pb * NT + tid; pb >= 0 && e < 3 * nS; e += pG * NT)
            a.yS[e] = -a.Yel[(size_t)a.qS[e / 3] * 4 + e % 3];
    }
    for (int c = pb; pb >= 0 && a.mode == kSchurPanel && c < nS; c += pG) {
        const int s0 = a.col2sn[a.qS[c]];
        double acc[3] = {0, 0, 0};
        for (int pi = a.path_ptr[s0]; pi < a.path_ptr[s0 + 1]; ++pi) {
            const int sn = a.path_sn[pi];
            for (int r = a.sn_c0[sn] + tid; r < a.sn_c0[sn + 1]; r += NT) {
                const double v = a.V[(size_t)r * a.ldv + c];
                acc[0] += v * a.G[(size_t)r * 4 + 0];
                acc[1] += v * a.G[(size_t)r * 4 + 1];
                acc[2] += v * a.G[(size_t)r * 4 + 2];
            }
        }
        for (int i = 0; i < 3; ++i) {
            const double tsum = block_sum<NT>(acc[i], T3);
            if (tid == 0) a.yS[3 * c + i] = -tsum;
        }
    }
    const int ntk = (nS + 31) / 32;
    // K keeps -Sigma_s when S is unchanged; the gather backend reads K from G2 instead
    const int ntiles = (reuse || a.mode == kSchurGather) ? 0 : ntk * (ntk + 1) / 2;
    if (a.mode == kSchurGather && !reuse && !supd)   // K_s = (L^-1)_SS = G2[r(S), r(S)] (a gather)
        for (size_t e = (size_t)bid * NT + tid; e < (size_t)nS * nS; e += (size_t)G * NT) {
            const int i = (int)(e / nS), j = (int)(e % nS);
            a.K[(size_t)i * a.ldk + j] = a.G2[(size_t)a.rpos[a.qS[i]] * a.n2 + a.rpos[a.qS[j]]];
        }
    const int nsplit = max(1, min(16, G / max(ntk * (ntk + 1) / 2, 1)));
    auto tile_of = [&](int b, int &ti, int &tj) {
        int rem = b;
        ti = 0;
        while (rem > ti) { rem -= ti + 1; ++ti; }
        tj = rem;
    };
    {
        typedef double Chunk[32][36];
        Chunk *Va = reinterpret_cast<Chunk *>(T0), *Vb = reinterpret_cast<Chunk *>(T1);   // [2] each
        const int gr = lane >> 2, gc = lane & 3;
        for (int bs = bid; bs < ntiles * nsplit; bs += G) {
            const int b = bs / nsplit, split = bs % nsplit;
            int ti, tj;
            tile_of(b, ti, tj);
            const int ia = ti * 32, ja = tj * 32;
            const bool diag = ti == tj;
            // chunk iterator over (supernode s, first row rb)
            auto overlaps = [&](int sn) {
                const int l = a.lo[sn], h = a.hi[sn];
                return h > l && l < ia + 32 && h > ia && l < ja + 32 && h > ja;
            };
            auto next_chunk = [&](int &sn, int &rb) -> bool {
                if (sn >= 0) {
                    rb += 32;
                    if (rb < a.sn_c0[sn + 1]) return true;
                    sn += nsplit;
                } else {
                    sn = split;
                }
                for (; sn < a.nsn; sn += nsplit)
                    if (overlaps(sn)) { rb = a.sn_c0[sn]; return true; }
                return false;
            };
            auto stage = [&](int sn, int rb, int buf) {
                const int l = a.lo[sn], h = a.hi[sn], nrb = min(32, a.sn_c0[sn + 1] - rb);
                for (int e = tid; e < 32 * 32; e += NT) {
                    const int rr = e >> 5, cc = e & 31;
                    const int ca = ia + cc, cb = ja + cc;
                    const double *row = a.V + (size_t)(rb + rr) * a.ldv;
                    if (rr < nrb && ca >= l && ca < h) {
                        const unsigned sa = (unsigned)__cvta_generic_to_shared(&Va[buf][rr][cc]);
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(row + ca));
                    } else {
                        Va[buf][rr][cc] = 0.0;
                    }
                    if (!diag) {
                        if (rr < nrb && cb >= l && cb < h) {
                            const unsigned sb = (unsigned)__cvta_generic_to_shared(&Vb[buf][rr][cc]);
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sb), "l"(row + cb));
                        } else {
                            Vb[buf][rr][cc] = 0.0;
                        }
                    }
                }
                asm volatile("cp.async.commit_group;\n" ::);
            };
            double acc[2][2] = {{0, 0}, {0, 0}};
            int sn = -1, rb = 0;
            bool have = next_chunk(sn, rb);
            if (have) stage(sn, rb, 0);
            int buf = 0;
            while (have) {
                int sn2 = sn, rb2 = rb;
                const bool have2 = next_chunk(sn2, rb2);
                if (have2) {
                    stage(sn2, rb2, buf ^ 1);
                    asm volatile("cp.async.wait_group 1;\n" ::);
                } else {
                    asm volatile("cp.async.wait_group 0;\n" ::);
                }
                __syncthreads();
                const Chunk &A = Va[buf];
                const Chunk &B = diag ? Va[buf] : Vb[buf];
#pragma unroll
                for (int j = 0; j < 2; ++j) {        // warp w: 8x8 tiles t = w, w + 8 of 4 x 4
                    const int t = wid + 8 * j, ta = t >> 2, tb = t & 3;
#pragma unroll
                    for (int k4 = 0; k4 < 8; ++k4)
                        dmma_884(acc[j][0], acc[j][1], A[4 * k4 + gc][8 * ta + gr], B[4 * k4 + gc][8 * tb + gr]);
                }
                __syncthreads();
                sn = sn2;
                rb = rb2;
                have = have2;
                buf ^= 1;
            }
            double *dst = a.Kpart + (size_t)bs * 1152;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int t = wid + 8 * j, ta = t >> 2, tb = t & 3;
                const int r = 8 * ta + gr, c = 8 * tb + 2 * gc;
                if (nsplit == 1) {
                    for (int q = 0; q < 2; ++q) {
                        const int R = ia + r, Cc = ja + c + q;
                        if (R < nS && Cc < nS && Cc <= R) {
                            a.K[(size_t)R * a.ldk + Cc] = acc[j][q];
                            a.K[(size_t)Cc * a.ldk + R] = acc[j][q];
                        }
                    }
                } else {
                    dst[r * 32 + c] = acc[j][0];
                    dst[r * 32 + c + 1] = acc[j][1];
                }
            }
        }
    }
    if (ntiles > 0 && nsplit > 1) {
        GSYNC();
        for (int e = bid * NT + tid; e < ntiles * 1024; e += G * NT) {
            const int b = e / 1024, q = e % 1024;
            int ti, tj;
            tile_of(b, ti, tj);
            double acc = 0.0;
            for (int sp = 0; sp < nsplit; ++sp) acc += a.Kpart[((size_t)b * nsplit + sp) * 1152 + q];
            const int r = ti * 32 + (q >> 5), c = tj * 32 + (q & 31);
            if (r < nS && c < nS && c <= r) {
                a.K[(size_t)r * a.ldk + c] = acc;
                a.K[(size_t)c * a.ldk + r] = acc;
            }
        }
    }
    GSYNC();
    if (a.mode == kSchurKOnly) return;        // setup: K = V^T V of the region only
    if (a.prof && bid == 0 && tid == 0) { a.prof[1000 + 1] = np; a.prof[np < 1000 ? np++ : np] = gtimer_s(); }   // phase marker (PDIPC_TRACE)
    // ------------------------------------------------ P1: K <- -K^{-1} (block sweep)
    // Gauss-Jordan sweep over 64-wide pivot blocks k on the SPD K (kept in its LOWER triangle:
    // column k's tile i is (i, k) for i > k and the transpose of (k, i) for i < k):
    //   P_k = A_kk^{-1};  U_i = A_ik P_k (i != k);  A_ij -= U_i A_jk^T (i, j != k);
    //   column k <- U, A_kk <- -P_k;      after all steps K = -K^{-1}.
    // Two grid barriers per step: phase A computes U (double-buffered) and writes the PREVIOUS
    // step's column (its values are in the other U buffer: the one tile of it phase A needs,
    // (k, k-1), is read from there); phase B runs the rank-64 update with a two-deep cp.async
    // tile pipeline per CTA, while CTA 0 updates the next pivot tile and inverts it (look-ahead).
    if (!reuse && supd) {
        // Low-rank update (S changed by at most 64 removed and 64 added vertices; K holds -Sigma_old
        // of the previous S, both triangles).  With Sigma = K_s^{-1} (exact identities):
        //   removal of R:  Sigma' = Sigma_kk - Sigma_kR Sigma_RR^{-1} Sigma_Rk   (kept rows / cols)
        //   addition of A: b = K_s[keep, A], X = Sigma' b, Sc = K_s[A, A] - b^T X,
        //     Sigma_new = [[Sigma' + X Sc^{-1} X^T, -X Sc^{-1}], [-Sc^{-1} X^T, Sc^{-1}]]
        // in the new S order (dpos: old position of each new one).  Sigma' lives in Sh (free until
        // P2); Y / Z / X / P in the two U buffers; Sigma_RR^{-1}, Sc^{-1} in T; the partials of b^T X
        // in Lstore (free until P3).  O(n^2 (|R| + |A|)) instead of the sweep's O(n^3).
        const int nr = a.uinfo[1], nad = a.uinfo[2], nold = a.uinfo[3], ldk = a.ldk;
        const size_t ustride = (size_t)(a.capS + 64) * TB;
        double *Yb = a.U, *Zb = a.U + ustride;             // [n][64] each
        double *Tm = a.T, *Tm2 = a.T + TB * TB;
        double *W = a.Sh;                                   // Sigma' (new order, ld = ldk)
        const int nto = (nold + TB - 1) / TB, ntn = (nS + TB - 1) / TB;
        auto inv_spd = [&](int nb, double *dst) {         // CTA: dst = T0[0:nb, 0:nb]^{-1} (identity pad)
            tile_chol64(T0, T1, nb, nb, a.info);
            for (int e = tid; e < TB * TB; e += NT) {
                const int r = e >> 6, c = e & 63;
                T2[r * TS + c] = T1[c * TS + r];
            }
            __syncthreads();
            tile_xyt(T3, T2, T2, 1.0, false);               // Li^T Li
            st_tile(T3, dst, TB, TB, TB);
        };
        auto g2 = [&](int i, int j) {                      // K_s entry of new positions i, j
            return a.G2[(size_t)a.rpos[a.qS[i]] * a.n2 + a.rpos[a.qS[j]]];
        };
        auto find_al = [&](int i) {
            int lo = 0, hi = nad;
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (a.al[mid] < i) lo = mid + 1; else hi = mid; }
            return lo;
        };
        if (nr > 0) {
            if (bid == 0) {                                 // Sigma_RR^{-1}
                for (int e = tid; e < TB * TB; e += NT) {
                    const int r = e >> 6, c = e & 63;
                    T0[r * TS + c] = (r < nr && c < nr) ? -a.K[(size_t)a.rl[r] * ldk + a.rl[c]] : 0.0;
                }
                __syncthreads();
                inv_spd(nr, Tm);
            }
            GSYNC();
            for (int t = bid; t < nto; t += G) {           // Z = Sigma_old[:, R], Y = Z Sigma_RR^{-1}
                const int p0 = t * TB, rows = min(TB, nold - p0);
                for (int e = tid; e < TB * TB; e += NT) {
                    const int r = e >> 6, c = e & 63;
                    T0[r * TS + c] = (r < rows && c < nr) ? -a.K[(size_t)(p0 + r) * ldk + a.rl[c]] : 0.0;
                }
                ld_tile(T1, Tm, TB, TB, TB);
                __syncthreads();
                tile_xyt(T2, T0, T1, 1.0, false);
                st_tile(T0, Zb + (size_t)p0 * TB, TB, rows, TB);
                st_tile(T2, Yb + (size_t)p0 * TB, TB, rows, TB);
                __syncthreads();
            }
            GSYNC();
        }
        for (int t = bid; t < ntn * ntn; t += G) {         // Sigma' = Sigma_old - Y Z^T, new order
            const int I = t / ntn, J = t % ntn, i0 = I * TB, j0 = J * TB;
            const int rows = min(TB, nS - i0), cols = min(TB, nS - j0);
            for (int e = tid; e < TB * TB; e += NT) {
                const int r = e >> 6, c = e & 63;
                const int pi = r < rows ? a.dpos[i0 + r] : -1, pj = c < cols ? a.dpos[j0 + c] : -1;
                T0[r * TS + c] = (pi >= 0 && pj >= 0) ? -a.K[(size_t)pi * ldk + pj] : 0.0;
                if (nr > 0) {
                    const int pr = r < cols ? a.dpos[j0 + r] : -1;
                    T1[r * TS + c] = pi >= 0 ? Yb[(size_t)pi * TB + c] : 0.0;
                    T2[r * TS + c] = pr >= 0 ? Zb[(size_t)pr * TB + c] : 0.0;
                }
            }
            __syncthreads();
            if (nr > 0) tile_xyt(T0, T1, T2, -1.0, true);
            st_tile(T0, W + (size_t)i0 * ldk + j0, ldk, rows, cols);
            __syncthreads();
        }
        GSYNC();
        if (nad > 0) {
            for (int e = bid * NT + tid; e < nS * TB; e += G * NT) {   // b = K_s[:, A] (0 on added rows)
                const int j = e >> 6, k = e & 63;
                Yb[e] = (k < nad && a.dpos[j] >= 0) ? g2(j, a.al[k]) : 0.0;
            }
            GSYNC();
            for (int I = bid; I < ntn; I += G) {           // X_I = sum_J Sigma'_IJ b_J; Q_I = b_I^T X_I
                const int i0 = I * TB, rows = min(TB, nS - i0);
                for (int J = 0; J < ntn; ++J) {
                    const int j0 = J * TB, cols = min(TB, nS - j0);
                    ld_tile(T0, W + (size_t)i0 * ldk + j0, ldk, rows, cols);
                    ld_tile(T3, Yb + (size_t)j0 * TB, TB, cols, TB);
                    __syncthreads();
                    for (int e = tid; e < TB * TB; e += NT) {
                        const int k = e >> 6, jj = e & 63;
                        T1[k * TS + jj] = T3[jj * TS + k];
                    }
                    __syncthreads();
                    tile_xyt(T2, T0, T1, 1.0, J > 0);
                }
                st_tile(T2, Zb + (size_t)i0 * TB, TB, rows, TB);
                ld_tile(T3, Yb + (size_t)i0 * TB, TB, rows, TB);
                __syncthreads();
                for (int e = tid; e < TB * TB; e += NT) {
                    const int k = e >> 6, ii = e & 63;
                    T1[k * TS + ii] = T3[ii * TS + k];      // b_I^T
                    T0[k * TS + ii] = T2[ii * TS + k];      // X_I^T
                }
                __syncthreads();
                tile_xyt(T3, T1, T0, 1.0, false);
                st_tile(T3, a.Lstore + (size_t)I * TB * TB, TB, TB, TB);
                __syncthreads();
            }
            GSYNC();
            if (bid == 0) {                                 // Sc = K_s[A, A] - sum_I Q_I; its inverse
                for (int e = tid; e < TB * TB; e += NT) {
                    const int k = e >> 6, l = e & 63;
                    double v = 0.0;
                    if (k < nad && l < nad) {
                        v = g2(a.al[k], a.al[l]);
                        for (int I = 0; I < ntn; ++I) v -= a.Lstore[(size_t)I * TB * TB + k * TB + l];
                    }
                    T0[k * TS + l] = v;
                }
                __syncthreads();
                inv_spd(nad, Tm2);
            }
            GSYNC();
            for (int t = bid; t < ntn; t += G) {           // P = X Sc^{-1}
                const int i0 = t * TB, rows = min(TB, nS - i0);
                ld_tile(T0, Zb + (size_t)i0 * TB, TB, rows, TB);
                ld_tile(T1, Tm2, TB, TB, TB);
                __syncthreads();
                tile_xyt(T2, T0, T1, 1.0, false);
                st_tile(T2, Yb + (size_t)i0 * TB, TB, rows, TB);
                __syncthreads();
            }
            GSYNC();
        }
        for (int t = bid; t < ntn * ntn; t += G) {         // K = -Sigma_new
            const int I = t / ntn, J = t % ntn, i0 = I * TB, j0 = J * TB;
            const int rows = min(TB, nS - i0), cols = min(TB, nS - j0);
            ld_tile(T0, W + (size_t)i0 * ldk + j0, ldk, rows, cols);
            if (nad > 0) {
                ld_tile(T1, Yb + (size_t)i0 * TB, TB, rows, TB);
                ld_tile(T2, Zb + (size_t)j0 * TB, TB, cols, TB);
            }
            __syncthreads();
            if (nad > 0) tile_xyt(T0, T1, T2, 1.0, true);  // Sigma' + P X^T
            for (int e = tid; e < TB * TB; e += NT) {
                const int r = e >> 6, c = e & 63;
                if (r < rows && c < cols) {
                    const int i = i0 + r, j = j0 + c;
                    const bool ai = nad > 0 && a.dpos[i] < 0, aj = nad > 0 && a.dpos[j] < 0;
                    double v = T0[r * TS + c];
                    if (ai && aj) v = Tm2[find_al(i) * TB + find_al(j)];
                    else if (ai) v = -Yb[(size_t)j * TB + find_al(i)];
                    else if (aj) v = -Yb[(size_t)i * TB + find_al(j)];
                    a.K[(size_t)i * ldk + j] = -v;
                }
            }
            __syncthreads();
        }
        GSYNC();
    } else if (!reuse) {
        const int nt = (nS + TB - 1) / TB;
        const size_t ustride = (size_t)(a.capS + 64) * TB;
        auto Ubuf = [&](int k) { return a.U + (size_t)(k & 1) * ustride; };
        auto Tbuf = [&](int k) { return a.T + (size_t)(k & 1) * TB * TB; };
        // CTA 0: P_k = (A_kk - [U_k A_k,k-1^T])^{-1} = Li^T Li into Tbuf(k)
        auto pivot_inverse = [&](int k, bool update_first) {
            const int kc0 = k * TB, kn = min(TB, nS - kc0);
            ld_tile(T0, a.K + (size_t)kc0 * a.ldk + kc0, a.ldk, kn, kn);
            if (update_first) {
                ld_tile(T1, Ubuf(k - 1) + (size_t)kc0 * TB, TB, kn, TB);
                ld_tile(T2, a.K + (size_t)kc0 * a.ldk + kc0 - TB, a.ldk, kn, TB);
            }
            __syncthreads();
            if (update_first) {
                tile_xyt(T0, T1, T2, -1.0, true);
                __syncthreads();
            }
            tile_chol64(T0, T1, kn, kn, a.info);
            for (int e = tid; e < TB * TB; e += NT) {      // T2 = Li^T
                const int r = e >> 6, c = e & 63;
                T2[r * TS + c] = T1[c * TS + r];
            }
            __syncthreads();
            tile_xyt(T3, T2, T2, 1.0, false);               // P = Li^T Li on DMMA
            st_tile(T3, Tbuf(k), TB, TB, TB);
        };
        // column k of the swept matrix: (r, k) = U_r for r != k, (k, k) = -P_k (lower storage)
        // mirror (last column): also the transposed entry in the upper triangle, from the lower
        // entry (P2 reads rows of Sigma_s)
        auto write_column = [&](int k, bool mirror) {
            const int kc0 = k * TB, kn = min(TB, nS - kc0);
            const double *Uk = Ubuf(k), *Tk = Tbuf(k);
            for (size_t e = (size_t)bid * NT + tid; e < (size_t)nS * kn; e += (size_t)G * NT) {
                const int r = (int)(e / kn), c = (int)(e % kn);
                const bool diag = r >= kc0 && r < kc0 + kn;
                const double v = diag ? -Tk[(r - kc0) * TB + c] : Uk[(size_t)r * TB + c];
                if (!mirror) {
                    if (r >= kc0) a.K[(size_t)r * a.ldk + kc0 + c] = v;        // lower: (r, k) block
                    else a.K[(size_t)(kc0 + c) * a.ldk + r] = v;                // lower: (k, r) block
                } else if (!diag || r - kc0 >= c) {
                    a.K[(size_t)r * a.ldk + kc0 + c] = v;
                    a.K[(size_t)(kc0 + c) * a.ldk + r] = v;
                }
            }
        };
        if (bid == 0) pivot_inverse(0, false);
        GSYNC();
        double *B0 = sm, *B1 = sm + 3 * TB * TS;             // two sets {X, Y, C} of the pipeline
        for (int k = 0; k < nt; ++k) {
            const int kc0 = k * TB, kn = min(TB, nS - kc0);
            double *Uk = Ubuf(k);
            // ---- phase A: U_i = A_ik P_k (i != k); column k-1 written
            for (int b = bid; b < nt - 1; b += G) {
                const int ti = b < k ? b : b + 1;
                const int r0 = ti * TB, rows = min(TB, nS - r0);
                if (ti > k) ld_tile(T0, a.K + (size_t)r0 * a.ldk + kc0, a.ldk, rows, kn);
                else if (ti == k - 1) {              // (k-1, k) = (k, k-1)^T = U_k(k-1)^T
                    const double *src = Ubuf(k - 1) + (size_t)kc0 * TB;
                    for (int e = tid; e < TB * TB; e += NT) {
                        const int c = e >> 6, r = e & 63;   // T0[r][c] = U_k(k-1)[c][r]
                        T0[r * TS + c] = (r < rows && c < kn) ? src[(size_t)c * TB + r] : 0.0;
                    }
                } else ld_tile_T(T0, a.K + (size_t)kc0 * a.ldk + r0, a.ldk, rows, kn);
                ld_tile(T1, Tbuf(k), TB, TB, TB);
                __syncthreads();
                tile_xyt(T2, T0, T1, 1.0, false);
                st_tile(T2, Uk + (size_t)r0 * TB, TB, rows, TB);
                __syncthreads();
            }
            if (k > 0) write_column(k - 1, false);
            GSYNC();
            // ---- phase B: A_ij -= U_i A_jk^T over the lower tiles (i, j != k); CTA 0 takes the
            // next pivot (k+1, k+1) instead (look-ahead), the others the rest
            const bool la = k + 1 < nt;
            if (la && bid == 0) pivot_inverse(k + 1, true);
            const int w0 = (la && G > 1) ? 1 : 0, nw = G - w0;
            const int ntile = (nt - 1) * nt / 2;
            auto tile_of = [&](int b, int &ti, int &tj) {
                int bi = 0, bj = b;
                while (bj > bi) { bj -= bi + 1; ++bi; }
                ti = bi < k ? bi : bi + 1;
                tj = bj < k ? bj : bj + 1;
            };
            auto next_b = [&](int b) {               // this CTA's next tile index (skips the pivot)
                while (b < ntile && w0 == 1) {
                    int ti, tj;
                    tile_of(b, ti, tj);
                    if (!(ti == k + 1 && tj == k + 1)) break;
                    b += nw;
                }
                return b;
            };
            auto issue = [&](int b, double *Bs) {    // U_i, A_jk (as Y: rows j), A_ij into {X, Y, C}
                int ti, tj;
                tile_of(b, ti, tj);
                const int r0 = ti * TB, c0 = tj * TB, rows = min(TB, nS - r0), cols = min(TB, nS - c0);
                double *X = Bs, *Y = Bs + TB * TS, *C = Bs + 2 * TB * TS;
                // 16-byte pieces (rows of U, K are 16-byte aligned: TB and ldk even); a piece
                // that straddles the valid width is copied element by element
                auto cp16 = [&](double *dst, const double *src, int c, int width) {
                    if (c + 1 < width) {
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
                    } else {
                        if (c < width) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
                        else dst[0] = 0.0;
                        dst[1] = 0.0;
                    }
                };
                for (int e = tid; e < TB * TB / 2; e += NT) {
                    const int r = e >> 5, c = (e & 31) * 2;
                    if (r < rows) cp16(X + r * TS + c, Uk + (size_t)(r0 + r) * TB + c, c, TB);
                    else { X[r * TS + c] = 0.0; X[r * TS + c + 1] = 0.0; }
                    if (r < rows) cp16(C + r * TS + c, a.K + (size_t)(r0 + r) * a.ldk + c0 + c, c, cols);
                    else { C[r * TS + c] = 0.0; C[r * TS + c + 1] = 0.0; }
                    if (tj > k) {                    // Y = tile (j, k)
                        if (r < cols) cp16(Y + r * TS + c, a.K + (size_t)(c0 + r) * a.ldk + kc0 + c, c, kn);
                        else { Y[r * TS + c] = 0.0; Y[r * TS + c + 1] = 0.0; }
                    }
                }
                if (tj < k)                          // Y = (k, j)^T: coalesced reads of (k, j)
                    for (int e = tid; e < TB * TB; e += NT) {
                        const int r = e >> 6, c = e & 63;
                        if (r < kn && c < cols)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(Y + c * TS + r)),
                                         "l"(a.K + (size_t)(kc0 + r) * a.ldk + c0 + c));
                        else Y[c * TS + r] = 0.0;
                    }
                asm volatile("cp.async.commit_group;\n" ::);
            };
            if (bid >= w0) {
                int b = next_b(bid - w0), par = 0;
                if (b < ntile) issue(b, B0);
                while (b < ntile) {
                    const int bn = next_b(b + nw);
                    asm volatile("cp.async.wait_group 0;\n" ::);
                    __syncthreads();                 // tile b landed; the other set is free
                    if (bn < ntile) issue(bn, par ? B0 : B1);
                    double *Bs = par ? B1 : B0;
                    tile_xyt(Bs + 2 * TB * TS, Bs, Bs + TB * TS, -1.0, true);
                    __syncthreads();
                    int ti, tj;
                    tile_of(b, ti, tj);
                    const int rows = min(TB, nS - ti * TB), cols = min(TB, nS - tj * TB);
                    if (k + 1 < nt) {
                        st_tile(Bs + 2 * TB * TS, a.K + (size_t)(ti * TB) * a.ldk + tj * TB, a.ldk, rows, cols);
                    } else {                         // final values: lower entries and their mirror
                        const double *Cs = Bs + 2 * TB * TS;
                        for (int e = tid; e < TB * TB; e += NT) {
                            const int r = e >> 6, cc = e & 63;
                            if (r < rows && cc < cols && (ti > tj || r >= cc)) {
                                const double v = Cs[r * TS + cc];
                                a.K[(size_t)(ti * TB + r) * a.ldk + tj * TB + cc] = v;
                                a.K[(size_t)(tj * TB + cc) * a.ldk + ti * TB + r] = v;
                            }
                        }
                    }
                    b = bn;
                    par ^= 1;
                }
            }
            GSYNC();
        }
        write_column(nt - 1, true);
        GSYNC();
    }
    if (a.prof && bid == 0 && tid == 0) { a.prof[1000 + 2] = np; a.prof[np < 1000 ? np++ : np] = gtimer_s(); }   // phase marker (PDIPC_TRACE)
    // ------------------------------------------------ P2: augmented Sigma-hat (Sigma_s = -K)
    // lower triangle, a warp per row (tile-0 rows: factored by CTA 0 when early0); the Sigma_s
    // entries of row r sit at columns c = r mod 3 + 3 j
    // With the block bits of B-check (a.tbits), the row is written from Sigma_s alone (writes
    // only) and the nonzero 3 x 3 blocks of B-check (b <= a in vertex row a = r / 3) are added
    // after: fl(-k + B) = fl(B - k), bit-identical to reading the dense row.
    for (int r = (early0 ? TB : 0) + pb * (NT / 32) + wid; a.tbits && pb >= 0 && r < m; r += pG * (NT / 32)) {
        const double *brow = a.Bc + (size_t)r * a.ldb;
        double *srow = a.Sh + (size_t)r * a.ldh;
        const int av = r / 3, r3 = r % 3;
        const double *krow = a.K + (size_t)av * a.ldk;
        for (int c0 = 0; c0 <= r; c0 += 512) {           // 16 loads per lane in flight
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int c = c0 + lane + 32 * u;
                v[u] = (c <= r && c % 3 == r3) ? -krow[c / 3] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int c = c0 + lane + 32 * u;
                if (c <= r) srow[c] = v[u];
            }
        }
        __syncwarp();
        const unsigned long long k0 = (unsigned long long)av * a.capS, k1 = k0 + av + 1;
        for (unsigned long long w = (k0 >> 5) + lane; w <= ((k1 - 1) >> 5); w += 32) {
            unsigned bits = a.tbits[w];
            if (w == (k0 >> 5)) bits &= ~0u << (unsigned)(k0 & 31);
            if (w == ((k1 - 1) >> 5) && (k1 & 31)) bits &= (1u << (unsigned)(k1 & 31)) - 1u;
            while (bits) {
                const int bp = __ffs(bits) - 1;
                bits &= bits - 1u;
                const int c3 = 3 * (int)(w * 32 + bp - k0);
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    if (c3 + j <= r) srow[c3 + j] += brow[c3 + j];
            }
        }
    }
    for (int r = (early0 ? TB : 0) + pb * (NT / 32) + wid; !a.tbits && pb >= 0 && r < m; r += pG * (NT / 32)) {
        const double *brow = a.Bc + (size_t)r * a.ldb;
        double *srow = a.Sh + (size_t)r * a.ldh;
        const double *krow = a.K + (size_t)(r / 3) * a.ldk;
        const int r3 = r % 3;
        for (int c0 = 0; c0 <= r; c0 += 256) {           // 8 loads per lane in flight
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = c0 + lane + 32 * u;
                v[u] = c <= r ? brow[c] - (c % 3 == r3 ? krow[c / 3] : 0.0) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = c0 + lane + 32 * u;
                if (c <= r) srow[c] = v[u];
            }
        }
    }
    if (a.prof && bid == 0 && tid == 0) a.prof[996] = gtimer_s();   // CTA 0: assembly rows done
    // b = (Sigma_s (x) I3) y_S with y_S = y_S^el - (K (x) I3) gc, i.e. b = Sigma_s y_S^el - gc
    // (K holds -Sigma_s in both triangles: the sweep mirrors its final values; a warp reads a row
    // once for the three components)
    for (int ai = pb * (NT / 32) + wid; pb >= 0 && ai < nS; ai += pG * (NT / 32)) {
        const double *krow = a.K + (size_t)ai * a.ldk;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
        for (int bb = lane; bb < nS; bb += 32) {
            const double kv = krow[bb];
            acc0 -= kv * a.yS[3 * bb + 0];
            acc1 -= kv * a.yS[3 * bb + 1];
            acc2 -= kv * a.yS[3 * bb + 2];
        }
        acc0 = warp_sum(acc0);
        acc1 = warp_sum(acc1);
        acc2 = warp_sum(acc2);
        if (lane == 0) {
            a.Sh[(size_t)m * a.ldh + 3 * ai + 0] = acc0 - a.gc[3 * ai + 0];
            a.Sh[(size_t)m * a.ldh + 3 * ai + 1] = acc1 - a.gc[3 * ai + 1];
            a.Sh[(size_t)m * a.ldh + 3 * ai + 2] = acc2 - a.gc[3 * ai + 2];
        }
    }
    if (a.prof && bid == 0 && tid == 0) a.prof[995] = gtimer_s();   // CTA 0: b rows done
    if (bid == 0 && tid == 0) a.Sh[(size_t)m * a.ldh + m] = 1.0;
    if (bid == 0)
        for (int e = tid; e < kMaxPanels; e += NT) a.bar[e] = 0u;   // P3 group-barrier counters
    GSYNC();
    if (a.prof && bid == 0 && tid == 0) { a.prof[1000 + 3] = np; a.prof[np < 1000 ? np++ : np] = gtimer_s(); }   // phase marker (PDIPC_TRACE)
    if (large) {                                          // P3 runs in k_chol_large
        if (a.prof && bid == 0 && tid == 0) a.prof[999] = np;
        return;
    }
    // ------------------------------------------------ P3: Cholesky of the augmented matrix
    // Right-looking in panels of kPW tile columns: inside a panel, per tile column k: diagonal
    // tile factor + inverse (CTA 0), L_ik = A_ik Li_k^T, update of the panel's later columns;
    // then ONE trailing update of everything right of the panel with the panel's kPW tile
    // columns (k streamed through shared memory, accumulator in registers): the trailing
    // matrix is read and written once per panel instead of once per tile column.
    const int nt = (ma + TB - 1) / TB;
    const int pw = nt >= a.pw_min ? kPW : nt + 1;  // small systems: look-ahead path below
    if (nt < a.pw_min) {
        // Small systems (latency-bound): ONE grid barrier per tile column.  Step k: every CTA
        // updates one tile (i, j), k < j <= i, recomputing the panel tiles it needs
        // (L_ik = A_ik L_kk^{-T}, blocked triangular solve with the 8x8 diagonal-block inverses
        // D_k of the factored tile) itself; CTA 0 takes (k+1, k+1) and then factors it
        // (look-ahead).  L_ik go to a ping-pong scratch (A_ik is still read by other CTAs in the
        // step) and are written into the factor one step later.  D_k is kept in Lstore[k * 512].
        double *Dst = a.Lstore;
        if (!early0) {                                   // (else factored during P0 / P2)
            if (bid == 0) {
                ld_tile(T0, a.Sh, a.ldh, min(TB, ma), min(TB, ma));
                __syncthreads();
                tile_chol64_d(T0, Dsh[0], min(TB, ma), m, a.info);
                __syncthreads();
                st_tile(T0, a.Sh, a.ldh, min(TB, ma), min(TB, ma));
                st_dblocks(Dsh[0], Dst);
            }
            GSYNC();
        }
        for (int k = 0; k < nt; ++k) {
            const int kc0 = k * TB, kn = min(TB, ma - kc0);
            double *LPk = a.LP + (size_t)(k & 1) * kLPTiles * TB * TB;      // L_ik of this step
            const double *LPp = a.LP + (size_t)((k + 1) & 1) * kLPTiles * TB * TB;   // previous
            const int rr = nt - k - 1;
            const int ntile = rr * (rr + 1) / 2;
            // write back the previous step's L_{i,k-1} (no CTA reads column k-1 any more)
            if (k > 0)
                for (size_t e = (size_t)bid * NT + tid; e < (size_t)(nt - k) * TB * TB; e += (size_t)G * NT) {
                    const int t = (int)(e / (TB * TB)), q = (int)(e % (TB * TB)), r = q >> 6, c = q & 63;
                    const int i = k + t, r0 = i * TB;
                    if (r0 + r < ma && (k - 1) * TB + c < ma)
                        a.Sh[(size_t)(r0 + r) * a.ldh + (k - 1) * TB + c] = LPp[(size_t)t * TB * TB + q];
                }
            // X_k = L_kk^{-T} (for the back substitution P4) on the first CTA without a tile this
            // step (the last CTA when every CTA has one): X = I L_kk^{-T}, blocked solve
            if (bid == (ntile < G ? ntile : G - 1)) {
                ld_tile(T1, a.Sh + (size_t)kc0 * a.ldh + kc0, a.ldh, kn, kn);
                ld_dblocks(Dsh[0], Dst + (size_t)k * 512);
                __syncthreads();
                for (int e = tid; e < TB * TB; e += NT) {
                    const int r = e >> 6, c = e & 63;
                    if (r >= kn || c >= kn) T1[r * TS + c] = (r == c) ? 1.0 : 0.0;
                    T0[r * TS + c] = (r == c) ? 1.0 : 0.0;
                }
                __syncthreads();
                tile_trsm_d(T0, T1, Dsh[0]);
                __syncthreads();
                st_tile(T0, Dst + (size_t)512 * (nt + 1) + (size_t)k * TB * TB, TB, TB, TB);
                __syncthreads();
            }
            if (bid < ntile) {
                // factored diagonal tile k (T1) and its block inverses: copies in flight together
                // with the tile loads below (one wait per step)
                ld_tile_async(T1, a.Sh + (size_t)kc0 * a.ldh + kc0, a.ldh, kn, kn);
                for (int e = tid; e < 512; e += NT) {
                    const unsigned sa = (unsigned)__cvta_generic_to_shared(&Dsh[0][e >> 6][(e >> 3) & 7][e & 7]);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(Dst + (size_t)k * 512 + e));
                }
                asm volatile("cp.async.commit_group;\n" ::);
            }
            for (int b = bid; b < ntile; b += G) {
                // b == 0 -> the look-ahead tile (k+1, k+1) on CTA 0
                int i = 0, bb = b;
                while (bb >= rr - i) { bb -= rr - i; ++i; }
                const int tj = k + 1 + i, ti = tj + bb;
                const int r0 = ti * TB, c0 = tj * TB, rows = min(TB, ma - r0), cols = min(TB, ma - c0);
                // A_ik (T0), A_jk (T3), A_ij (T2): all copies issued, one wait
                ld_tile_async(T0, a.Sh + (size_t)r0 * a.ldh + kc0, a.ldh, rows, kn);
                if (tj != ti) ld_tile_async(T3, a.Sh + (size_t)c0 * a.ldh + kc0, a.ldh, cols, kn);
                ld_tile_async(T2, a.Sh + (size_t)r0 * a.ldh + c0, a.ldh, rows, cols);
                asm volatile("cp.async.wait_all;\n" ::);
                __syncthreads();
                if (kn < TB)                                 // padding rows: identity (as factored)
                    for (int e = tid; e < TB * TB; e += NT) {
                        const int r = e >> 6, c = e & 63;
                        if (r >= kn || c >= kn) T1[r * TS + c] = (r == c) ? 1.0 : 0.0;
                    }
                __syncthreads();
                tile_trsm_d(T0, T1, Dsh[0]);                 // L_ik, L_jk
                if (tj != ti) tile_trsm_d(T3, T1, Dsh[0]);
                __syncthreads();
                if (tj == ti)                                // the diagonal-tile CTA keeps L_ik
                    for (int e = tid; e < TB * TB; e += NT)
                        LPk[(size_t)(ti - k - 1) * TB * TB + e] = T0[(e >> 6) * TS + (e & 63)];
                if (tj == ti) tile_syrk_lower_sub(T2, T0);
                else tile_xyt(T2, T0, T3, -1.0, true);
                if (b == 0) {                                // look-ahead: factor tile k+1 now
                    tile_chol64_d(T2, Dsh[1], rows, m - r0, a.info);
                    __syncthreads();
                    st_tile(T2, a.Sh + (size_t)r0 * a.ldh + c0, a.ldh, rows, cols);
                    st_dblocks(Dsh[1], Dst + (size_t)(k + 1) * 512);
                } else {
                    st_tile(T2, a.Sh + (size_t)r0 * a.ldh + c0, a.ldh, rows, cols);
                }
                __syncthreads();
            }
            GSYNC();
        }
    }
    // Large systems: right-looking in panels of kPW tile columns with LOOK-AHEAD.  Iteration q:
    //   panel group (CTAs [0, npg)): applies panel q-1 to panel q's tile columns, then factors
    //     panel q -- per tile column k: diagonal tile factor + inverse on the group's first CTA,
    //     L_ik = A_ik Li_k^T, update of the panel's later columns -- with group barriers;
    //   update group (CTAs [npg, G)): applies panel q-1 to every tile column right of panel q
    //     (accumulators in registers, k streamed through shared memory, double-buffered).
    // ONE grid barrier per panel: the serial panel chain runs beside the trailing update.  npg
    // balances the two groups' estimated work (identical on every CTA).
    // A_ij -= sum_{k in [k0, k1)} L_ik L_jk^T for one 64 x 64 tile (ti, tj)
    auto update_tile = [&](int ti, int tj, int k0, int k1) {
        const int gr = lane >> 2, gc = lane & 3;
        const int r0 = ti * TB, c0 = tj * TB, rows = min(TB, ma - r0), cols = min(TB, ma - c0);
        // first k-chunk in flight before the accumulator (kept negated: acc = -A_ij) is read
        ld_tile_async(T0, a.Sh + (size_t)r0 * a.ldh + k0 * TB, a.ldh, rows, TB);
        ld_tile_async(T1, a.Sh + (size_t)c0 * a.ldh + k0 * TB, a.ldh, cols, TB);
        double acc[8][2];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
            const int r = 8 * wid + gr, c = 8 * nb + 2 * gc;
            acc[nb][0] = (r < rows && c < cols) ? -a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c] : 0.0;
            acc[nb][1] = (r < rows && c + 1 < cols) ? -a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c + 1] : 0.0;
        }
        for (int k = k0; k < k1; ++k) {
            double *X = ((k - k0) & 1) ? T2 : T0, *Y = ((k - k0) & 1) ? T3 : T1;
            if (k + 1 < k1) {
                double *Xn = ((k - k0) & 1) ? T0 : T2, *Yn = ((k - k0) & 1) ? T1 : T3;
                ld_tile_async(Xn, a.Sh + (size_t)r0 * a.ldh + (k + 1) * TB, a.ldh, rows, TB);
                ld_tile_async(Yn, a.Sh + (size_t)c0 * a.ldh + (k + 1) * TB, a.ldh, cols, TB);
                asm volatile("cp.async.wait_group 2;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncthreads();
            tile_add_xyt_regs(acc, X, Y);
            __syncthreads();
        }
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
            const int r = 8 * wid + gr, c = 8 * nb + 2 * gc;
            if (r < rows && c < cols) a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c] = -acc[nb][0];
            if (r < rows && c + 1 < cols) a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c + 1] = -acc[nb][1];
        }
    };
    // A_ij -= sum_k L_ik L_jk^T for the 128 x 64 block of row tiles (ti, ti + 1) x column tile tj
    // (ti + 1 may lie beyond the matrix: those rows are not stored).  k is streamed in 32-wide
    // chunks by thread 0 with 2-D TMA tensor copies (6 boxes of 16 doubles x 64 rows per chunk,
    // 128-byte swizzle: dense stages, conflict-free fragment loads) into a kTmaStages ring, kTmaAhead
    // chunks ahead, with mbarriers instead of CTA barriers: full[s] completes when the chunk's
    // 48 KB landed, empty[s] when all 8 warps are done with it.  Rows of X or Y beyond the matrix
    // hold whatever Sh holds there (zero beyond the allocation); they only reach accumulator rows /
    // columns that are not stored.  Warp w owns rows 16w .. 16w + 15 x 64 columns: per 4-wide k step
    // 2 + 8 fragment loads feed 16 independent DMMAs; the accumulator is kept negated (adds only).
    constexpr int KC = 32;
    auto update_pair = [&](int ti, int tj, int k0, int k1) {
        const int gr = lane >> 2, gc = lane & 3;
        const int r0 = ti * TB, c0 = tj * TB;
        const int rows = min(2 * TB, ma - r0), cols = min(TB, ma - c0);
        const int kbeg = k0 * TB, nch = (k1 - k0) * TB / KC;
        const unsigned g0 = tma_g;
        const unsigned ring = (smem_u32(sm) + 1023u) & ~1023u;
        const unsigned fullb = smem_u32(tma_bar), emptyb = fullb + 8 * kTmaStages;
        // earlier generic-proxy writes of the ring (other phases) before the async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        auto produce = [&](int ch) {                      // thread 0
            const unsigned g = g0 + ch, st = g % kTmaStages;
            if (g >= (unsigned)kTmaStages) mbar_wait(emptyb + 8 * st, ((g / kTmaStages) - 1) & 1);
            const unsigned fb = fullb + 8 * st, sb = ring + st * kTmaStageB;
            const int kc = kbeg + ch * KC;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(kTmaStageB)
                         : "memory");
            const unsigned long long tm = reinterpret_cast<unsigned long long>(&P.s[grp].tmap_sh);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
                                 "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(sb + h * 16384 + j * 8192),
                                 "l"(tm), "r"(kc + 16 * h), "r"(r0 + 64 * j), "r"(fb)
                                 : "memory");
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
                             "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(sb + 32768 + h * 8192),
                             "l"(tm), "r"(kc + 16 * h), "r"(c0), "r"(fb)
                             : "memory");
            }
        };
        if (tid == 0) {
            // Sh written through the generic proxy (this and other CTAs, ordered by the barriers)
            // before the tensor copies read it
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            for (int ch = 0; ch < min(nch, kTmaAhead); ++ch) produce(ch);
        }
        double acc[2][8][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr, c = 8 * nb + 2 * gc;
                acc[h][nb][0] = (r < rows && c < cols) ? -a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c] : 0.0;
                acc[h][nb][1] = (r < rows && c + 1 < cols) ? -a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c + 1] : 0.0;
            }
        // 128-byte swizzle: the 16-byte unit u of row r sits at u ^ (r & 7); rows of a fragment
        // load have r & 7 = gr (all row bases are multiples of 8)
        unsigned sw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) sw[q] = ((((2 * q) + (gc >> 1)) ^ gr) << 4) + ((gc & 1) << 3);
        const char *smc = reinterpret_cast<const char *>(sm) + (ring - smem_u32(sm));
        for (int ch = 0; ch < nch; ++ch) {
            if (tid == 0 && ch + kTmaAhead < nch) produce(ch + kTmaAhead);
            const unsigned g = g0 + ch, st = g % kTmaStages;
            mbar_wait(fullb + 8 * st, (g / kTmaStages) & 1);
            const char *xa = smc + st * kTmaStageB + (16 * wid + gr) * 128;
            const char *yb = smc + st * kTmaStageB + 32768 + gr * 128;
#pragma unroll
            for (int k4 = 0; k4 < KC / 4; ++k4) {
                const int hx = (k4 >> 2) * 16384 + sw[k4 & 3], hy = (k4 >> 2) * 8192 + sw[k4 & 3];
                const double a0 = *reinterpret_cast<const double *>(xa + hx);
                const double a1 = *reinterpret_cast<const double *>(xa + 1024 + hx);
#pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                    const double bv = *reinterpret_cast<const double *>(yb + nb * 1024 + hy);
                    dmma_884(acc[0][nb][0], acc[0][nb][1], a0, bv);
                    dmma_884(acc[1][nb][0], acc[1][nb][1], a1, bv);
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(emptyb + 8 * st) : "memory");
        }
        tma_g = g0 + nch;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr, c = 8 * nb + 2 * gc;
                if (r < rows && c < cols) a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c] = -acc[h][nb][0];
                if (r < rows && c + 1 < cols) a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c + 1] = -acc[h][nb][1];
            }
        __syncthreads();                                  // the ring is free for the caller's next phase
    };
    // pairs of row tiles (ti, ti + 1), ti = tj + 2p, over the tile columns [ja, jb): linear index b
    auto pair_of = [&](int b, int ja, int &ti, int &tj) {
        int j = ja;
        while (b >= (nt - j + 1) / 2) { b -= (nt - j + 1) / 2; ++j; }
        tj = j;
        ti = j + 2 * b;
    };
    auto pairs_in = [&](int ja, int jb) {
        int t = 0;
        for (int j = ja; j < jb; ++j) t += (nt - j + 1) / 2;
        return t;
    };
    // panel width in tiles: wider panels amortise the trailing updates (k = 64 kpw per pass) and
    // the grid barriers; measured best at n_c ~ 3000 (141 tiles): 10 (tools/gpu_kpw_sweep.sh,
    // profiles/schur_kpw_sweep_r02.txt); narrower for smaller systems
    const int kpw = min(a.kpw, max(4, nt / 14));
    // variable panel widths: the first panel (factored with nothing to overlap) a.kpw0 wide, the
    // last ones narrower (the panel chain is the critical path there): w = min(kpw, max(4,
    // remaining / a.ktail)); identical on every CTA
    auto width = [&](int q, int c0) {
        if (q == 0) return min(nt, max(1, min(kpw, a.kpw0)));
        const int w = a.ktail > 0 ? min(kpw, max(4, (nt - c0) / a.ktail)) : kpw;
        return min(nt - c0, w);
    };
    if (a.prof && bid == 0 && tid == 0) a.prof[997] = (unsigned long long)(a.wu_coef * 1000.0);
    int c0t = 0, pc0 = 0;                                 // panel q: [c0t, c1t); previous: [pc0, c0t)
    for (int q = 0; nt >= a.pw_min && c0t < nt; ++q) {
        const int c1t = c0t + width(q, c0t), ppw = c0t - pc0;
        const int rr = nt - c1t;                                   // tile columns right of panel q
        int npg = G;
        if (q > 0 && rr > 0 && G > 1) {
            // work estimates in units of a 64^3 tile product: a k = 4-tile update ~ 4, a TRSM or
            // single-k update ~ 1.3, the diagonal factor ~ 4 (serial), a barrier ~ 0.3 (serial)
            double wp = 0.0, ws = 0.0;
            for (int j = c0t; j < c1t; ++j) wp += (double)ppw * (nt - j);
            const int mid = c1t - c0t >= 6 && nt - c1t >= a.split_min ? c0t + (c1t - c0t + 1) / 2 : c1t;
            for (int k = c0t; k < c1t; ++k) {
                wp += 1.3 * (nt - k - 1);
                for (int j = k + 1; j < (k < mid ? mid : c1t); ++j) wp += 1.3 * (nt - j);
                ws += 4.0 + 3 * 0.3;
            }
            for (int j = mid; j < c1t; ++j) wp += (double)(mid - c0t) * (nt - j);
            const double wu = 0.25 * a.wu_coef * ppw * rr * (rr + 1) / 2.0;
            double best = 1e300;
            for (int x = 1; x < G; ++x) {
                const double t = fmax(ws + wp / x, wu / (G - x));
                if (t < best) { best = t; npg = x; }
            }
        }
        if (bid < npg) {
            unsigned *ctr = a.bar + q;
            unsigned nbar = 0;
            if (q > 0) {        // panel q-1 applied to panel q's tiles (i, j), c0t <= j < c1t, i >= j
                const int tot = pairs_in(c0t, c1t);
                for (int b = bid; b < tot; b += npg) {
                    int ti, tj;
                    pair_of(b, c0t, ti, tj);
                    update_pair(ti, tj, pc0, c0t);
                }
                group_bar(ctr, ++nbar * npg);
            }
            if (a.prof && bid == 0 && tid == 0 && q < 100) a.prof[500 + q] = gtimer_s();   // panel update done
            // Per tile column k: TRSM of the tiles below the diagonal, then the intra-panel update,
            // with the NEXT diagonal tile taken out of it (look-ahead): CTA 0 updates (k+1, k+1)
            // in shared memory and factors it while the other CTAs update the rest of the panel,
            // so the serial tile factor overlaps the update (one group barrier per step saved).
            // The tile (k+2, k+1), the other half of the pair that holds (k+1, k+1), becomes a
            // single-tile update.
            auto factor_diag = [&](int k, bool update_first) {    // CTA 0
                const int kc0 = k * TB, kn = min(TB, ma - kc0);
                ld_tile(T0, a.Sh + (size_t)kc0 * a.ldh + kc0, a.ldh, kn, kn);
                if (update_first) ld_tile(T1, a.Sh + (size_t)kc0 * a.ldh + kc0 - TB, a.ldh, kn, TB);
                __syncthreads();
                if (update_first) {               // A_kk -= L_k,k-1 L_k,k-1^T
                    tile_xyt(T0, T1, T1, -1.0, true);
                    __syncthreads();
                }
                tile_chol64(T0, T1, kn, m - kc0, a.info);
                st_tile(T0, a.Sh + (size_t)kc0 * a.ldh + kc0, a.ldh, kn, kn);
                for (int e = tid; e < TB * TB; e += NT) a.Lstore[(size_t)k * TB * TB + e] = T1[(e >> 6) * TS + (e & 63)];
            };
            if (bid == 0) factor_diag(c0t, false);
            group_bar(ctr, ++nbar * npg);
            // two halves (panels of >= 6 columns): the first half's intra-panel updates stay in
            // the first half; then ONE update of the second half with all first-half columns
            // (k = 64 x half width: the long, efficient update) and the second half
            const int mid = c1t - c0t >= 6 && nt - c1t >= a.split_min ? c0t + (c1t - c0t + 1) / 2 : c1t;
            for (int k = c0t; k < c1t; ++k) {
                const int kc0 = k * TB, kn = min(TB, ma - kc0);
                // per-column detail of panels 2 and 30 (PDIPC_TRACE): diagonal factored, TRSM
                // done, intra-panel update done
                const int pslot = (q == 0 || q == 12) && a.prof && bid == 0 && tid == 0 && k - c0t < 10
                                      ? 900 + (q == 12 ? 40 : 0) + 3 * (k - c0t) : -1;
                if (pslot >= 0) a.prof[pslot] = gtimer_s();
                for (int b = bid; b < nt - k - 1; b += npg) {      // L_ik = A_ik Li^T
                    const int ti = k + 1 + b, r0 = ti * TB, rows = min(TB, ma - r0);
                    ld_tile(T0, a.Sh + (size_t)r0 * a.ldh + kc0, a.ldh, rows, kn);
                    ld_tile(T1, a.Lstore + (size_t)k * TB * TB, TB, TB, TB);
                    __syncthreads();
                    tile_xyt(T2, T0, T1, 1.0, false);
                    st_tile(T2, a.Sh + (size_t)r0 * a.ldh + kc0, a.ldh, rows, kn);
                }
                group_bar(ctr, ++nbar * npg);
                if (pslot >= 0) a.prof[pslot + 1] = gtimer_s();
                const int kend = k < mid ? mid : c1t;
                if (k + 1 == mid && mid < c1t) {   // second half += first half (k in [c0t, mid))
                    const int tot = pairs_in(mid, c1t);
                    for (int b = bid; b < tot; b += npg) {
                        int ti, tj;
                        pair_of(b, mid, ti, tj);
                        update_pair(ti, tj, c0t, mid);
                    }
                    group_bar(ctr, ++nbar * npg);
                    if (bid == 0) factor_diag(mid, false);
                    group_bar(ctr, ++nbar * npg);
                } else if (k + 1 < kend) {  // A_ij -= L_ik L_jk^T, k < j < kend, i >= j
                    // pair 0 is (k+1, k+2) x (k+1): its diagonal tile goes to CTA 0 (look-ahead),
                    // its lower tile (k+2, k+1) to the last CTA; pairs 1.. to CTAs 1.. (all
                    // CTAs when npg == 1)
                    const int tot = pairs_in(k + 1, kend);
                    if (bid == 0) factor_diag(k + 1, true);
                    if (bid == npg - 1 && k + 2 < nt) update_tile(k + 2, k + 1, k, k + 1);
                    const int w0 = npg > 1 ? 1 : 0, nw = npg > 1 ? npg - 1 : 1;
                    if (bid >= w0)
                        for (int b = 1 + (bid - w0); b < tot; b += nw) {
                            int ti, tj;
                            pair_of(b, k + 1, ti, tj);
                            update_pair(ti, tj, k, k + 1);
                        }
                    group_bar(ctr, ++nbar * npg);
                }
                if (pslot >= 0) a.prof[pslot + 2] = gtimer_s();
            }
            if (a.prof && bid == 0 && tid == 0 && q < 100) { a.prof[600 + q] = gtimer_s(); a.prof[800 + q] = npg; }
        } else if (q > 0) {     // panel q-1 applied to the tile columns right of panel q
            const int ub = bid - npg, nu = G - npg, tot = pairs_in(c1t, nt);
            for (int b = ub; b < tot; b += nu) {
                int ti, tj;
                pair_of(b, c1t, ti, tj);
                update_pair(ti, tj, pc0, c0t);
            }
            if (a.prof && tid == 0 && q < 100) atomicMax(a.prof + 700 + q, gtimer_s());   // update group done
        }
        GSYNC();
        pc0 = c0t;
        c0t = c1t;
    }
    }                                                     // ---------------- end of P0 .. P3
    if (a.prof && bid == 0 && tid == 0) { a.prof[1000 + 4] = np; a.prof[np < 1000 ? np++ : np] = gtimer_s(); }   // phase marker (PDIPC_TRACE)
    // ------------------------------------------------ P4: u = C^{-T} y, y = row m of the factor
    const int ntm = (m + TB - 1) / TB, nt = (ma + TB - 1) / TB;
    if (nt < a.pw_min) {
        // Small systems: CTA 0 alone, no grid barrier.  Per 64-row tile k of C from the last:
        // u_k = X_k y_k with X_k = L_kk^{-T} (formed by P3), then y_j -= sum_r C[kc0+r][j] u_r for
        // j < kc0 (rows of C read from L2, every load of a thread in flight at once).  X_k is
        // prefetched into shared memory one tile ahead (cp.async).
        if (bid == 0) {
            const int mr = (m + 7) & ~7;
            double *yv = sm, *uv = sm + mr;                     // y, u  [mr] each
            double *Xt = sm + 2 * mr;                           // [2][64][65]
            const double *Xg = a.Lstore + (size_t)512 * (nt + 1);
            for (int e = tid; e < mr; e += NT) yv[e] = e < m ? a.Sh[(size_t)m * a.ldh + e] : 0.0;
            auto issue = [&](int k) {
                if (k >= 0)
                    for (int e = tid; e < TB * TB; e += NT) {
                        const unsigned sa = (unsigned)__cvta_generic_to_shared(Xt + (size_t)(k & 1) * 64 * 65 +
                                                                               (e >> 6) * 65 + (e & 63));
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa),
                                     "l"(Xg + (size_t)k * TB * TB + e));
                    }
                asm volatile("cp.async.commit_group;\n" ::);
            };
            const int ntm = (m + TB - 1) / TB;
            issue(ntm - 1);
            __syncthreads();
            for (int k = ntm - 1; k >= 0; --k) {
                issue(k - 1);
                asm volatile("cp.async.wait_group 1;\n" ::);
                __syncthreads();
                const int kc0 = k * TB, kn = min(TB, m - kc0);
                const double *X = Xt + (size_t)(k & 1) * 64 * 65;
                {   // u_i = sum_{r >= i} X[i][r] y_r: 4 partial sums per output
                    const int i = tid & 63, pq = tid >> 6;
                    double acc = 0.0;
                    if (i < kn)
                        for (int r = i + pq; r < kn; r += 4) acc += X[i * 65 + r] * yv[kc0 + r];
                    T3[pq * 64 + i] = acc;
                }
                __syncthreads();
                if (tid < kn) uv[kc0 + tid] = T3[tid] + T3[64 + tid] + T3[128 + tid] + T3[192 + tid];
                __syncthreads();
                if (a.prof && tid == 0 && np < 1000) a.prof[np++] = gtimer_s();
                // y_j -= sum_r C[kc0 + r][j] u_r: warp w takes rows w, w + 8, ..., lane the columns
                // j = lane + 32 q (coalesced rows; 8 rows x 8 columns of loads in flight per chunk);
                // the 8 warp partials are summed in a fixed order (deterministic)
                double *part = Xt + 2 * 64 * 65;                // [8][mr]
                for (int q0 = 0; q0 < kc0; q0 += 256) {
                    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    double v[8][8], ur[8];                      // unconditional loads (clamped
#pragma unroll                                                  // indices): all 64 in flight
                    for (int rr = 0; rr < 8; ++rr) {
                        const int r = wid + 8 * rr, rc = min(r, kn - 1);
                        ur[rr] = r < kn ? uv[kc0 + r] : 0.0;
                        const double *row = a.Sh + (size_t)(kc0 + rc) * a.ldh;
#pragma unroll
                        for (int q = 0; q < 8; ++q) v[rr][q] = __ldcg(row + min(q0 + lane + 32 * q, kc0 - 1));
                    }
#pragma unroll
                    for (int rr = 0; rr < 8; ++rr)
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc[q] += v[rr][q] * ur[rr];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int j = q0 + lane + 32 * q;
                        if (j < kc0) part[wid * mr + j] = acc[q];
                    }
                }
                __syncthreads();
                for (int j = tid; j < kc0; j += NT)
                    yv[j] -= ((part[j] + part[mr + j]) + (part[2 * mr + j] + part[3 * mr + j])) +
                             ((part[4 * mr + j] + part[5 * mr + j]) + (part[6 * mr + j] + part[7 * mr + j]));
                __syncthreads();                                // this stage is refilled next
                if (a.prof && tid == 0 && np < 1000) a.prof[np++] = gtimer_s();
            }
            asm volatile("cp.async.wait_group 0;\n" ::);
            for (int e = tid; e < m; e += NT) a.u[e] = uv[e];
        }
        GSYNC();
    } else if (ntm <= kMaxPanels / 2) {
        // Dataflow back substitution (no grid barrier per tile): CTA b owns the tiles j = b, b+G,
        // ... (descending).  For tile j it accumulates y_j - sum_{k>j} C_kj^T u_k in registers, k
        // descending, each u_k as soon as its flag is set (fixed order: deterministic), then forms
        // u_j = Li_j^T y_j, stores it and sets flag j.  Every dependency points to a higher tile,
        // so the wait chain is acyclic; the critical path is one tile product + one flag hand-off
        // per tile.  Flags: a.bar[512 + j], zeroed in P2.
        volatile unsigned *flag = a.bar + kMaxPanels / 2;
        double *yj = T0, *part = T1;                       // [64], [4][64]
        const int c = tid & 63, rq = tid >> 6;
        const int jtop = bid < ntm ? bid + ((ntm - 1 - bid) / G) * G : -1;
        double *Cl = T2, *Lj = T3;                         // last tile C_{j+1,j}, Li_j (smem)
        for (int j = jtop; j >= 0; j -= G) {
            const int jc0 = j * TB, jn = min(TB, m - jc0);
            double acc = 0.0;                              // column c of y_j, rows r = rq, rq + 4, ...
            for (int k = ntm - 1; k > j + 1; --k) {       // all but the last tile: from L2
                if (tid == 0)
                    while (flag[k] == 0u) __nanosleep(32);
                __syncthreads();
                const int kc0 = k * TB, kn = min(TB, m - kc0);
                const double *Ck = a.Sh + (size_t)kc0 * a.ldh + jc0 + c;
                const double *uk = a.u + kc0;
                if (c < jn)
#pragma unroll 4
                    for (int r = rq; r < kn; r += 4) acc += __ldcg(Ck + (size_t)r * a.ldh) * __ldcg(uk + r);
            }
            // the critical step: C_{j+1,j} and Li_j staged in shared memory before the wait
            const bool has_last = j + 1 < ntm;
            const int lc0 = (j + 1) * TB, ln = has_last ? min(TB, m - lc0) : 0;
            if (has_last) ld_tile_async(Cl, a.Sh + (size_t)lc0 * a.ldh + jc0, a.ldh, ln, jn);
            ld_tile_async(Lj, a.Lstore + (size_t)j * TB * TB, TB, TB, TB);
            asm volatile("cp.async.commit_group;\n" ::);
            if (has_last && tid == 0)
                while (flag[j + 1] == 0u) __nanosleep(20);
            asm volatile("cp.async.wait_group 0;\n" ::);
            __syncthreads();
            if (has_last)
                for (int r = rq; r < ln; r += 4) acc += Cl[r * TS + c] * __ldcg(a.u + lc0 + r);
            part[rq * TB + c] = acc;
            __syncthreads();
            if (tid < TB)
                yj[tid] = tid < jn ? a.Sh[(size_t)m * a.ldh + jc0 + tid] -
                                         ((part[tid] + part[TB + tid]) + (part[2 * TB + tid] + part[3 * TB + tid]))
                                   : 0.0;
            __syncthreads();
            {   // u_j[i] = sum_{r >= i} Li[r][i] y_j[r]: 4 partial sums per output
                const int i = tid & 63, pq = tid >> 6;
                double s = 0.0;
                if (i < jn)
                    for (int r = i + pq; r < jn; r += 4) s += Lj[r * TS + i] * yj[r];
                part[pq * TB + i] = s;
            }
            __syncthreads();
            if (tid < jn) a.u[jc0 + tid] = (part[tid] + part[TB + tid]) + (part[2 * TB + tid] + part[3 * TB + tid]);
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicExch((unsigned *)&flag[j], 1u);
        }
        GSYNC();
    } else {
        {
            // one grid barrier per tile step: every CTA forms u_k = Li_k^T y_k itself (64 x 64, from
            // L2), CTA 0 publishes it, all CTAs update their slice of y_j -= C_kj^T u_k (j < k).
            // y lives in a.y (updated in place), u in a.u.
            for (int e = bid * NT + tid; e < m; e += G * NT) a.y[e] = a.Sh[(size_t)m * a.ldh + e];
            GSYNC();
            double *uk = T0, *part = T1;
            for (int k = ntm - 1; k >= 0; --k) {
                const int kc0 = k * TB, kn = min(TB, m - kc0);
                const double *Li = a.Lstore + (size_t)k * TB * TB;
                {   // u_k[i] = sum_{r >= i} Li[r][i] y_k[r]: 4 partial sums per output
                    const int i = tid & 63, pq = tid >> 6;
                    double acc = 0.0;
                    if (i < kn)
                        for (int r = i + pq; r < kn; r += 4) acc += Li[r * TB + i] * a.y[kc0 + r];
                    part[pq * TB + i] = acc;
                }
                __syncthreads();
                if (tid < TB) {
                    const double v = tid < kn ? part[tid] + part[TB + tid] + part[2 * TB + tid] + part[3 * TB + tid] : 0.0;
                    uk[tid] = v;
                    if (bid == 0 && tid < kn) a.u[kc0 + tid] = v;
                }
                __syncthreads();
                for (int j = bid * NT + tid; j < kc0; j += G * NT) {   // y_j -= sum_r C[kc0 + r][j] u_k[r]
                    double acc = 0.0;
#pragma unroll 8
                    for (int r = 0; r < kn; ++r) acc += a.Sh[(size_t)(kc0 + r) * a.ldh + j] * uk[r];
                    a.y[j] -= acc;
                }
                GSYNC();
            }
        }
    }
    if (a.prof && bid == 0 && tid == 0) { a.prof[1000 + 5] = np; a.prof[np < 1000 ? np++ : np] = gtimer_s(); }   // phase marker (PDIPC_TRACE)
    // ------------------------------------------------ P5: t = B u ; Z = w + V t = w_el + V (gc + t)
    // (w = L^{-1} Pi g = w_el + V gc since the contact gradient is supported on S)
    if (a.tbits) {
        // B-check is block-sparse: a warp per vertex row ab scans the row's block bits (lane per
        // 32-bit word, bits in increasing order) and multiplies only the nonzero 3 x 3 blocks;
        // the lane partials are summed by the fixed xor tree (deterministic)
        for (int ab = bid * (NT / 32) + wid; ab < nS; ab += G * (NT / 32)) {
            const unsigned long long k0 = (unsigned long long)ab * a.capS, k1 = k0 + nS;
            const unsigned long long w0 = k0 >> 5, w1 = (k1 - 1) >> 5;
            double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
            const double *r0 = a.Bc + (size_t)(3 * ab) * a.ldb;
            for (unsigned long long w = w0 + lane; w <= w1; w += 32) {
                unsigned bits = a.tbits[w];
                if (w == w0) bits &= ~0u << (unsigned)(k0 & 31);
                if (w == w1 && (k1 & 31)) bits &= (1u << (unsigned)(k1 & 31)) - 1u;
                while (bits) {
                    const int bp = __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const int b3 = 3 * (int)(w * 32 + bp - k0);
                    const double u0 = a.u[b3], u1 = a.u[b3 + 1], u2 = a.u[b3 + 2];
                    acc0 += r0[b3] * u0 + r0[b3 + 1] * u1 + r0[b3 + 2] * u2;
                    acc1 += r0[a.ldb + b3] * u0 + r0[a.ldb + b3 + 1] * u1 + r0[a.ldb + b3 + 2] * u2;
                    acc2 += r0[2 * (size_t)a.ldb + b3] * u0 + r0[2 * (size_t)a.ldb + b3 + 1] * u1 +
                            r0[2 * (size_t)a.ldb + b3 + 2] * u2;
                }
            }
            acc0 = warp_sum(acc0);
            acc1 = warp_sum(acc1);
            acc2 = warp_sum(acc2);
            if (lane == 0) {
                a.t[3 * ab + 0] = acc0 + a.gc[3 * ab + 0];
                a.t[3 * ab + 1] = acc1 + a.gc[3 * ab + 1];
                a.t[3 * ab + 2] = acc2 + a.gc[3 * ab + 2];
            }
        }
    } else {
        for (int row = bid * (NT / 32) + wid; row < m; row += G * (NT / 32)) {
            double acc = 0.0;
            for (int c = lane; c < m; c += 32) acc += a.Bc[(size_t)row * a.ldb + c] * a.u[c];
            acc = warp_sum(acc);
            if (lane == 0) a.t[row] = acc + a.gc[row];
        }
    }
    if (a.prof && bid == 0 && tid == 0) { a.prof[1000 + 7] = np; a.prof[np < 1000 ? np++ : np] = gtimer_s(); }
    if (a.mode == kSchurGather) {
        // sparse right-hand side E_S (gc + t) of the caller's solve: zero, then the rows of S
        for (size_t e = (size_t)bid * NT + tid; e < (size_t)4 * a.nf; e += (size_t)G * NT) a.Z[e] = 0.0;
        GSYNC();
        for (int e = bid * NT + tid; e < m; e += G * NT) a.Z[(size_t)a.qS[e / 3] * 4 + e % 3] = a.t[e];
        if (a.prof && bid == 0 && tid == 0) { a.prof[1000 + 6] = np; a.prof[np < 1000 ? np++ : np] = gtimer_s(); }
        return;
    }
    GSYNC();
    // Z = w_el + V (gc + t): warp per row, lanes over the row's active columns [lo_s, hi_s)
    // (contiguous in V), fixed xor-tree reduction
    for (int r = bid * (NT / 32) + wid; r < a.nf; r += G * (NT / 32)) {
        const int sn = a.col2sn[r];
        const int c0 = a.lo[sn], c1 = a.hi[sn];
        double z0 = 0.0, z1 = 0.0, z2 = 0.0;
        for (int c = c0 + lane; c < c1; c += 32) {
            const double v = a.V[(size_t)r * a.ldv + c];
            z0 += v * a.t[3 * c + 0];
            z1 += v * a.t[3 * c + 1];
            z2 += v * a.t[3 * c + 2];
        }
        z0 = warp_sum(z0);
        z1 = warp_sum(z1);
        z2 = warp_sum(z2);
        if (lane == 0) {
            a.Z[(size_t)r * 4 + 0] = a.G[(size_t)r * 4 + 0] + z0;
            a.Z[(size_t)r * 4 + 1] = a.G[(size_t)r * 4 + 1] + z1;
            a.Z[(size_t)r * 4 + 2] = a.G[(size_t)r * 4 + 2] + z2;
            a.Z[(size_t)r * 4 + 3] = 0.0;
        }
    }
}

// ---------------------------------------------------------------- large-system Cholesky ---
// P3 of a large system (>= pw_min 64-tiles, C3 / C4) in its own cooperative kernel with 16 warps
// per CTA (the fused Schur kernel's register budget allows only 8): right-looking panels of kPW
// tile columns with look-ahead as in k_schur_coop (panel group / update group, one grid barrier
// per panel); the trailing updates on 128 x 128 blocks (2 x 2 tiles), warp (wr, wc) owning rows
// 16wr .. 16wr + 15 and columns 64wc .. 64wc + 63, k streamed in 32-wide chunks through a 3-stage
// 16-byte cp.async pipeline (per 4-wide k step 2 + 8 fragment loads feed 16 DMMAs per warp).
constexpr int NT2 = 512;
constexpr int XS2 = 36;
constexpr int kCholSmem = 3 * 256 * XS2 * (int)sizeof(double);
static_assert(kCholSmem >= 4 * TB * TS * (int)sizeof(double), "chol tiles");

struct CholArgs {
    double *Sh;
    int ldh;
    const int *nS_ptr;
    int capS, pw_min;
    double *Lstore;
    int *info;
    unsigned *bar;
    unsigned long long *prof;
};

__global__ void __launch_bounds__(NT2, 1) k_chol_large(CholArgs a) {
    extern __shared__ double sm[];
    double *T0 = sm, *T1 = sm + TB * TS, *T2 = sm + 2 * TB * TS;
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x, bid = blockIdx.x;
    const int nS = min(*a.nS_ptr, a.capS), m = 3 * nS, ma = m + 1, nt = (ma + TB - 1) / TB;
    if (nS == 0 || nt < a.pw_min) return;
    int np = a.prof ? (int)a.prof[999] : 0;
    const int wr = wid & 7, wc = wid >> 3, gr = lane >> 2, gc = lane & 3;
    // A_ij -= sum_{k in [k0, k1)} L_ik L_jk^T on the 128 x 128 block of row tiles (ti, ti + 1) x
    // column tiles (tj, tj + 1), columns limited to jlim tiles (and the matrix)
    auto update_block = [&](int ti, int tj, int k0, int k1, int jlim) {
        const int r0 = ti * TB, c0 = tj * TB;
        const int rows = min(2 * TB, ma - r0), cols = min(2 * TB, min(jlim * TB, ma) - c0);
        const int kbeg = k0 * TB, nch = (k1 - k0) * TB / 32;
        auto issue = [&](int ch) {
            if (ch < nch) {
                double *X = sm + (ch % 3) * 256 * XS2;
                const int kc = kbeg + ch * 32;
                for (int e = tid; e < 4096; e += NT2) {            // X rows 0..127, Y rows 128..255
                    const int rr = e >> 4, c2 = (e & 15) * 2;
                    const bool isx = rr < 128;
                    const int r = isx ? rr : rr - 128;
                    double *dst = X + rr * XS2 + c2;
                    if (r < (isx ? rows : cols)) {
                        const double *src = a.Sh + (size_t)((isx ? r0 : c0) + r) * a.ldh + kc + c2;
                        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
                    } else {
                        dst[0] = 0.0;
                        dst[1] = 0.0;
                    }
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        issue(0);
        issue(1);
        double acc[2][8][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wr + 8 * h + gr, c = 64 * wc + 8 * nb + 2 * gc;
                acc[h][nb][0] = (r < rows && c < cols) ? -a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c] : 0.0;
                acc[h][nb][1] = (r < rows && c + 1 < cols) ? -a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c + 1] : 0.0;
            }
        for (int ch = 0; ch < nch; ++ch) {
            issue(ch + 2);
            asm volatile("cp.async.wait_group 2;\n" ::);
            __syncthreads();
            const double *X = sm + (ch % 3) * 256 * XS2 + (16 * wr + gr) * XS2 + gc;
            const double *Y = sm + (ch % 3) * 256 * XS2 + (128 + 64 * wc + gr) * XS2 + gc;
#pragma unroll
            for (int k4 = 0; k4 < 8; ++k4) {
                const double a0 = X[4 * k4], a1 = X[8 * XS2 + 4 * k4];
#pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                    const double bv = Y[8 * nb * XS2 + 4 * k4];
                    dmma_884(acc[0][nb][0], acc[0][nb][1], a0, bv);
                    dmma_884(acc[1][nb][0], acc[1][nb][1], a1, bv);
                }
            }
            __syncthreads();
        }
        asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wr + 8 * h + gr, c = 64 * wc + 8 * nb + 2 * gc;
                if (r < rows && c < cols) a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c] = -acc[h][nb][0];
                if (r < rows && c + 1 < cols) a.Sh[(size_t)(r0 + r) * a.ldh + c0 + c + 1] = -acc[h][nb][1];
            }
    };
    // 2 x 2 blocks over the tile columns [ja, jb): block columns tj = ja, ja + 2, ..., row tiles
    // ti = tj, tj + 2, ...
    auto nblocks = [&](int ja, int jb) {
        int t = 0;
        for (int j = ja; j < jb; j += 2) t += (nt - j + 1) / 2;
        return t;
    };
    auto block_of = [&](int b, int ja, int &ti, int &tj) {
        int j = ja;
        while (b >= (nt - j + 1) / 2) { b -= (nt - j + 1) / 2; j += 2; }
        tj = j;
        ti = j + 2 * b;
    };
    const int npan = (nt + kPW - 1) / kPW;
    for (int q = 0; q < npan; ++q) {
        const int c0t = q * kPW, c1t = min(nt, c0t + kPW);
        int npg = G;
        if (q > 0 && c1t < nt && G > 1) {   // work in 64^3-product units (see k_schur_coop)
            double wp = 16.0 * nblocks(c0t, c1t), ws = 0.0;
            for (int k = c0t; k < c1t; ++k) {
                wp += 1.3 * (nt - k - 1) + 4.0 * 1.3 * nblocks(k + 1, c1t);
                ws += 4.0 + 3 * 0.3;
            }
            const double wu = 16.0 * nblocks(c1t, nt);
            double best = 1e300;
            for (int x = 1; x < G; ++x) {
                const double t = fmax(ws + wp / x, wu / (G - x));
                if (t < best) { best = t; npg = x; }
            }
        }
        if (bid < npg) {
            unsigned *ctr = a.bar + q;
            unsigned nbar = 0;
            if (q > 0) {
                const int tot = nblocks(c0t, c1t);
                for (int b = bid; b < tot; b += npg) {
                    int ti, tj;
                    block_of(b, c0t, ti, tj);
                    update_block(ti, tj, c0t - kPW, c0t, c1t);
                }
                group_bar(ctr, ++nbar * npg);
            }
            for (int k = c0t; k < c1t; ++k) {
                const int kc0 = k * TB, kn = min(TB, ma - kc0);
                if (bid == 0) {
                    ld_tile<NT2>(T0, a.Sh + (size_t)kc0 * a.ldh + kc0, a.ldh, kn, kn);
                    __syncthreads();
                    tile_chol64<NT2>(T0, T1, kn, m - kc0, a.info);
                    st_tile<NT2>(T0, a.Sh + (size_t)kc0 * a.ldh + kc0, a.ldh, kn, kn);
                    for (int e = tid; e < TB * TB; e += NT2) a.Lstore[(size_t)k * TB * TB + e] = T1[(e >> 6) * TS + (e & 63)];
                }
                group_bar(ctr, ++nbar * npg);
                for (int b = bid; b < nt - k - 1; b += npg) {      // L_ik = A_ik Li^T
                    const int ti = k + 1 + b, r0 = ti * TB, rows = min(TB, ma - r0);
                    ld_tile<NT2>(T0, a.Sh + (size_t)r0 * a.ldh + kc0, a.ldh, rows, kn);
                    ld_tile<NT2>(T1, a.Lstore + (size_t)k * TB * TB, TB, TB, TB);
                    __syncthreads();
                    tile_xyt<NT2>(T2, T0, T1, 1.0, false);
                    st_tile<NT2>(T2, a.Sh + (size_t)r0 * a.ldh + kc0, a.ldh, rows, kn);
                }
                group_bar(ctr, ++nbar * npg);
                if (k + 1 < c1t) {          // A_ij -= L_ik L_jk^T, k < j < c1t, i >= j
                    const int tot = nblocks(k + 1, c1t);
                    for (int b = bid; b < tot; b += npg) {
                        int ti, tj;
                        block_of(b, k + 1, ti, tj);
                        update_block(ti, tj, k, k + 1, c1t);
                    }
                    group_bar(ctr, ++nbar * npg);
                }
            }
            if (a.prof && bid == 0 && tid == 0 && q < 100) { a.prof[600 + q] = gtimer_s(); a.prof[800 + q] = npg; }
        } else if (q > 0) {
            const int ub = bid - npg, nu = G - npg, tot = nblocks(c1t, nt);
            for (int b = ub; b < tot; b += nu) {
                int ti, tj;
                block_of(b, c1t, ti, tj);
                update_block(ti, tj, c0t - kPW, c0t, nt);
            }
            if (a.prof && tid == 0 && q < 100) atomicMax(a.prof + 700 + q, gtimer_s());
        }
        grid.sync();
        if (a.prof && bid == 0 && tid == 0 && np < 1000) a.prof[np++] = gtimer_s();
    }
    if (a.prof && bid == 0 && tid == 0) a.prof[999] = np;
}

static int g_schur_grid = 0;
static unsigned *g_gbar = nullptr;  // group barrier counters, kMaxSchurSys x 32 (one cache line each)
// PDIPC_SPLIT_SCHUR=1: large systems factor in k_chol_large (16 warps per CTA, 128 x 128 blocks)
// between two k_schur_coop launches.  Off by default: measured 16.1 vs 14.7 ms for P3 at n_c 3000
// (the fused kernel's 128 x 64 blocks on 8 warps reach the same per-SM DMMA rate, and the split
// adds the spills of a 128-register budget to the diagonal-tile chain).
static bool getenv_fused() {
    static const int v = [] { const char *e = std::getenv("PDIPC_SPLIT_SCHUR"); return e && e[0] == '1' ? 0 : 1; }();
    return v != 0;
}
static double *g_kpart = nullptr;   // split-K partial tiles, grid x 1152 doubles (allocated at init)
static double *g_lp = nullptr;      // small-system P3 panel scratch
static unsigned *g_bar = nullptr;   // large-system P3 group-barrier counters

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;   // driver entry point (no -lcuda)

void schur_init(int device) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&g_encode, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            g_encode = nullptr;
    }
    cudaFuncSetAttribute(k_schur_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, kSchurSmem);
    int per_sm = 0, nsm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_schur_coop, NT, kSchurSmem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    g_schur_grid = std::max(1, per_sm) * nsm;
    if (!g_kpart) cudaMalloc(&g_kpart, (size_t)g_schur_grid * 1152 * sizeof(double));   // split by group
    if (!g_lp) cudaMalloc(&g_lp, (size_t)kMaxSchurSys * 2 * kLPTiles * TB * TB * sizeof(double));
    if (!g_bar) cudaMalloc(&g_bar, (size_t)kMaxSchurSys * kMaxPanels * sizeof(unsigned));
    if (!g_gbar) cudaMalloc(&g_gbar, (size_t)kMaxSchurSys * 32 * sizeof(unsigned));
    cudaFuncSetAttribute(k_chol_large, cudaFuncAttributeMaxDynamicSharedMemorySize, kCholSmem);
}

SchurArgs schur_args(const DevFactor &F, const double *V, int ldv, const double *G, const double *gc,
                     const int *qS, const int *lo, const int *hi, const int *nS, int capS, double *K, int ldk,
                     const double *Bc, int ldb, double *Sh, int ldh, double *Lstore, double *T, double *U,
                     double *yS, double *y, double *u, double *t, double *Z, int *info, const int *same_S,
                     unsigned long long *prof, int large_min_tiles, int mode, const double *G2, int n2,
                     const int *rpos, const double *Yel) {
    SchurArgs a;
    std::memset(&a, 0, sizeof(a));
    a.V = V; a.ldv = ldv; a.G = G; a.gc = gc; a.qS = qS; a.col2sn = F.col2sn; a.sn_c0 = F.sn_c0;
    a.sn_parent = F.sn_parent; a.path_ptr = F.path_ptr; a.path_sn = F.path_sn; a.lo = lo; a.hi = hi; a.nsn = F.nsn; a.nf = F.nf; a.nS_ptr = nS; a.capS = capS;
    a.K = K; a.ldk = ldk; a.Bc = Bc; a.ldb = ldb; a.Sh = Sh; a.ldh = ldh; a.Lstore = Lstore;
    a.T = T; a.U = U; a.yS = yS; a.y = y; a.u = u; a.t = t; a.Z = Z; a.info = info; a.same = same_S; a.prof = prof;
    a.pw_min = large_min_tiles > 0 ? std::min(large_min_tiles, kPWMinTiles) : kPWMinTiles;
    a.mode = mode; a.G2 = G2; a.n2 = n2; a.rpos = rpos; a.Yel = Yel;
    static const double wu = [] { const char *e = std::getenv("PDIPC_SCHUR_WU"); return e ? std::atof(e) : 3.5; }();
    a.wu_coef = wu;
    static const int kpw = [] { const char *e = std::getenv("PDIPC_SCHUR_KPW"); return e ? std::max(1, std::atoi(e)) : 10; }();
    a.kpw = kpw;
    static const int kpw0 = [] { const char *e = std::getenv("PDIPC_SCHUR_KPW0"); return e ? std::max(1, std::atoi(e)) : 10; }();
    static const int ktail = [] { const char *e = std::getenv("PDIPC_SCHUR_KTAIL"); return e ? std::atoi(e) : 0; }();
    a.kpw0 = kpw0;
    // -1: chosen per launch in launch_schur_batch (PDIPC_SCHUR_SPLIT overrides)
    static const int split_min = [] { const char *e = std::getenv("PDIPC_SCHUR_SPLIT"); return e ? std::atoi(e) : -1; }();
    a.split_min = split_min;
    a.ktail = ktail;
    if (g_encode && Sh && ldh > 0 && capS > 0) {
        const cuuint64_t dims[2] = {(cuuint64_t)ldh, (cuuint64_t)(3 * capS + 1)};
        const cuuint64_t strides[1] = {(cuuint64_t)ldh * sizeof(double)};
        const cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
        g_encode(&a.tmap_sh, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Sh, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return a;
}

int launch_schur_batch(const SchurArgs *sys, int nsys, cudaStream_t st) {
    if (nsys < 1 || nsys > kMaxSchurSys) return (int)cudaErrorInvalidValue;
    if (!g_encode) return (int)cudaErrorNotSupported;    // the trailing updates need TMA descriptors
    SchurBatch b;
    std::memset(&b, 0, sizeof(b));
    const int gsz = g_schur_grid / nsys;
    for (int g = 0; g < nsys; ++g) {          // per-group scratch (split-K partials, panels, barriers)
        b.s[g] = sys[g];
        // half-panel split threshold: 80 tile columns for a system on the whole grid (C3 single,
        // profiles/schur_kpw_sweep_r02.txt), 20 in a batched launch where each system has ~1/nsys
        // of the CTAs (C4 4 systems: never / 40 / 30 / 20 / always 70.1 / 73.5 / 73.6 / 73.6 / 73.4
        // it/s, profiles/schur_split_r02.txt)
        if (b.s[g].split_min < 0) b.s[g].split_min = nsys == 1 ? 80 : 20;
        b.s[g].Kpart = g_kpart + (size_t)g * gsz * 1152;
        b.s[g].LP = g_lp + (size_t)g * 2 * kLPTiles * TB * TB;
        b.s[g].bar = g_bar + (size_t)g * kMaxPanels;
        b.s[g].gbar = g_gbar + (size_t)g * 32;
        b.s[g].phase = 0;
    }
    b.nsys = nsys;
    // weights m^2.5 rather than the Cholesky's m^3: a larger system's serial panel chain does not
    // shrink with more CTAs (C4 exponent 2 / 2.25 / 2.5 / 3 / 3.5: 71.9 / 72.3 / 72.7 / 72.4 / 71.1
    // it/s, profiles/schur_split_r02.txt; PDIPC_SCHUR_WEXP)
    static const double wexp = [] { const char *e = std::getenv("PDIPC_SCHUR_WEXP"); return e ? std::atof(e) : 2.5; }();
    b.wexp = wexp;
    cudaError_t e = dev_zero(g_gbar, kMaxSchurSys * 32 * sizeof(unsigned), st);
    if (e != cudaSuccess) return (int)e;
    const bool split = nsys == 1 && !getenv_fused() && sys[0].mode != kSchurKOnly;
    void *args[] = {&b};
    note_launch();
    if (!split)
        return (int)cudaLaunchCooperativeKernel((const void *)k_schur_coop, dim3(g_schur_grid), dim3(NT), args,
                                                 kSchurSmem, st);
    // large systems (PDIPC_SPLIT_SCHUR=1): P0-P2 | P3 in k_chol_large | P4-P5 (each launch checks
    // the size on the device)
    b.s[0].phase = 1;
    e = cudaLaunchCooperativeKernel((const void *)k_schur_coop, dim3(g_schur_grid), dim3(NT), args, kSchurSmem, st);
    if (e != cudaSuccess) return (int)e;
    CholArgs c;
    c.Sh = b.s[0].Sh; c.ldh = b.s[0].ldh; c.nS_ptr = b.s[0].nS_ptr; c.capS = b.s[0].capS; c.pw_min = b.s[0].pw_min;
    c.Lstore = b.s[0].Lstore; c.info = b.s[0].info; c.bar = b.s[0].bar; c.prof = b.s[0].prof;
    void *cargs[] = {&c};
    note_launch();
    e = cudaLaunchCooperativeKernel((const void *)k_chol_large, dim3(g_schur_grid), dim3(NT2), cargs, kCholSmem, st);
    if (e != cudaSuccess) return (int)e;
    b.s[0].phase = 2;
    e = dev_zero(g_gbar, kMaxSchurSys * 32 * sizeof(unsigned), st);
    if (e != cudaSuccess) return (int)e;
    note_launch();
    return (int)cudaLaunchCooperativeKernel((const void *)k_schur_coop, dim3(g_schur_grid), dim3(NT), args,
                                             kSchurSmem, st);
}

int launch_schur(const DevFactor &F, const double *V, int ldv, const double *G, const double *gc,
                 const int *qS,
                 const int *lo, const int *hi, const int *nS, int capS, double *K, int ldk, const double *Bc, int ldb,
                 double *Sh, int ldh, double *Lstore, double *T, double *U, double *yS, double *y, double *u,
                 double *t, double *Z, int *info, const int *same_S, unsigned long long *prof,
                 int large_min_tiles, int mode, const double *G2, int n2, const int *rpos, const double *Yel,
                 cudaStream_t st) {
    const SchurArgs a = schur_args(F, V, ldv, G, gc, qS, lo, hi, nS, capS, K, ldk, Bc, ldb, Sh, ldh, Lstore, T, U,
                                   yS, y, u, t, Z, info, same_S, prof, large_min_tiles, mode, G2, n2, rpos, Yel);
    return launch_schur_batch(&a, 1, st);
}

}  // namespace pdipc
