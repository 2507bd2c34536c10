// Dense FP64 linear algebra of the contact-reduced global step:
//   Sigma_s = K_s^{-1}  (symmetric block sweep = Gauss-Jordan on an SPD matrix),
//   Sigma-hat = Sigma_s (x) I3 + B-check,  Sigma-hat = C C^T (right-looking blocked Cholesky),
//   u = Sigma-hat^{-1} (Sigma_s (x) I3) y_S,  t = B-check u.
// PAPER.md:194-198 (Eq. 8): the dense Schur complement; PAPER.md:241-247 (Eq. 11): the
// low-rank update on the n_c contact vertices, here in the K-Schur form that never inverts
// the (singular) B-check.
// The O(m^3) work runs in 64x64 tiles on the FP64 tensor pipe: mma.sync.m8n8k4.f64 (DMMA;
// tcgen05 has no f64 kind on sm_100a).  Matrices are row-major with a
// leading dimension; the Cholesky factor is the lower triangle.
#include "kernels.h"

#include "dev_common.cuh"

namespace pdipc {

constexpr int NB = 64;          // tile size
constexpr int SST = 68;         // smem row stride (doubles): conflict-free DMMA fragment loads

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

enum TileMode { TM_TRSM = 0, TM_POTRF_UPD = 1, TM_SWEEP_PANEL = 2, TM_SWEEP_UPD = 3 };

struct TileArgs {
    int mode, nt, k, m;
    double *A;
    int ld;
    const double *T;     // 64x64 tile operand (Linv or P), ld = NB
    double *U;           // sweep panel buffer [nt*64][64]
};

// loads a (rows x 64) tile at src (row-major, ld) into smem with zero padding
__device__ __forceinline__ void load_tile(double *S, const double *src, int ld, int rows, int cols) {
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
        int r = e >> 6, c = e & 63;
        S[r * SST + c] = (r < rows && c < cols) ? src[(size_t)r * ld + c] : 0.0;
    }
}

// One CTA (256 threads = 8 warps) computes a 64x64 output tile  Out (+)= alpha X Y^T.
__global__ void __launch_bounds__(256) k_tile_gemm(TileArgs a) {
    extern __shared__ double smem[];
    double *Xs = smem, *Ys = smem + NB * SST;
    int ti, tj;
    const int k = a.k, nt = a.nt;
    int b = blockIdx.x;
    if (a.mode == TM_TRSM || a.mode == TM_SWEEP_PANEL) {
        ti = (a.mode == TM_TRSM) ? k + 1 + b : (b < k ? b : b + 1);
        tj = k;
    } else if (a.mode == TM_POTRF_UPD) {
        // lower tiles k < tj <= ti < nt
        int r = nt - k - 1;                 // trailing tile count
        int i = 0;
        while (b >= r - i) { b -= r - i; ++i; }   // column-wise enumeration
        tj = k + 1 + i;
        ti = tj + b;
    } else {                                // all (ti, tj) != k
        int n1 = nt - 1;
        int bi = b / n1, bj = b % n1;
        ti = bi < k ? bi : bi + 1;
        tj = bj < k ? bj : bj + 1;
    }
    const int m = a.m;
    const int r0 = ti * NB, c0 = tj * NB;
    const int rows = min(NB, m - r0), cols = min(NB, m - c0);
    const int kcols = min(NB, m - k * NB);
    // operands
    const double *Xsrc, *Ysrc;
    int ldx, ldy, xrows, yrows;
    if (a.mode == TM_TRSM || a.mode == TM_SWEEP_PANEL) {
        Xsrc = a.A + (size_t)r0 * a.ld + k * NB; ldx = a.ld; xrows = rows;
        Ysrc = a.T; ldy = NB; yrows = NB;
    } else if (a.mode == TM_POTRF_UPD) {
        Xsrc = a.A + (size_t)r0 * a.ld + k * NB; ldx = a.ld; xrows = rows;
        Ysrc = a.A + (size_t)c0 * a.ld + k * NB; ldy = a.ld; yrows = cols;
    } else {
        Xsrc = a.U + (size_t)r0 * NB; ldx = NB; xrows = rows;
        Ysrc = a.A + (size_t)c0 * a.ld + k * NB; ldy = a.ld; yrows = cols;
    }
    load_tile(Xs, Xsrc, ldx, xrows, kcols);
    load_tile(Ys, Ysrc, ldy, yrows, kcols);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    double acc[8][2];
    const bool accum = a.mode == TM_POTRF_UPD || a.mode == TM_SWEEP_UPD;
    double *Out;
    int ldo;
    if (a.mode == TM_SWEEP_PANEL) { Out = a.U + (size_t)r0 * NB; ldo = NB; }
    else { Out = a.A + (size_t)r0 * a.ld + c0; ldo = a.ld; }
    const double alpha = accum ? -1.0 : 1.0;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
        int r = 8 * w + gr, c = 8 * nb + 2 * gc;
        acc[nb][0] = (accum && r < rows && c < cols) ? Out[(size_t)r * ldo + c] : 0.0;
        acc[nb][1] = (accum && r < rows && c + 1 < cols) ? Out[(size_t)r * ldo + c + 1] : 0.0;
    }
#pragma unroll 4
    for (int k4 = 0; k4 < NB / 4; ++k4) {
        double av = alpha * Xs[(8 * w + gr) * SST + 4 * k4 + gc];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
            double bv = Ys[(8 * nb + gr) * SST + 4 * k4 + gc];
            dmma(acc[nb][0], acc[nb][1], av, bv);
        }
    }
    __syncthreads();   // in-place TRSM: all reads of Xs done before writes (Xs is in smem anyway)
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
        int r = 8 * w + gr, c = 8 * nb + 2 * gc;
        if (r < rows && c < cols) Out[(size_t)r * ldo + c] = acc[nb][0];
        if (r < rows && c + 1 < cols) Out[(size_t)r * ldo + c + 1] = acc[nb][1];
    }
}

// Cholesky of the diagonal tile k in place (lower) and Linv = L_kk^{-1} (64x64, zero padded).
// If spd_inverse, instead writes P = (A_kk)^{-1} = Linv^T Linv to T and leaves A_kk untouched.
__global__ void __launch_bounds__(256) k_tile_potrf(double *A, int ld, int m, int k, double *T,
                                                    int spd_inverse, int *info) {
    extern __shared__ double potrf_sm[];
    double (*S)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(potrf_sm);
    double (*I)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(potrf_sm + NB * (NB + 1));
    const int r0 = k * NB, nb = min(NB, m - r0);
    const int tid = threadIdx.x;
    for (int e = tid; e < NB * NB; e += 256) {
        int r = e >> 6, c = e & 63;
        S[r][c] = (r < nb && c < nb) ? A[(size_t)(r0 + r) * ld + r0 + c] : 0.0;
    }
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
        double d = S[j][j];
        if (!(d > 0.0)) {
            if (tid == 0) atomicExch(info, 1);
            d = 1.0;
        }
        d = sqrt(d);
        __syncthreads();
        if (tid == 0) S[j][j] = d;
        for (int i = j + 1 + tid; i < nb; i += 256) S[i][j] /= d;
        __syncthreads();
        for (int e = tid; e < (nb - j - 1) * (nb - j - 1); e += 256) {
            int i = j + 1 + e / (nb - j - 1), l = j + 1 + e % (nb - j - 1);
            if (l <= i) S[i][l] -= S[i][j] * S[l][j];
        }
        __syncthreads();
    }
    // Linv: solve L X = I, one thread per column
    if (tid < NB) {
        const int c = tid;
        for (int i = 0; i < NB; ++i) {
            double v;
            if (i < c || i >= nb || c >= nb) v = 0.0;
            else {
                double acc = (i == c) ? 1.0 : 0.0;
                for (int q = c; q < i; ++q) acc -= S[i][q] * I[q][c];
                v = acc / S[i][i];
            }
            I[i][c] = v;
        }
    }
    __syncthreads();
    if (!spd_inverse) {
        for (int e = tid; e < nb * nb; e += 256) {
            int r = e / nb, c = e % nb;
            A[(size_t)(r0 + r) * ld + r0 + c] = c <= r ? S[r][c] : 0.0;
        }
        for (int e = tid; e < NB * NB; e += 256) T[e] = I[e >> 6][e & 63];
    } else {
        // P = Linv^T Linv
        for (int e = tid; e < NB * NB; e += 256) {
            int r = e >> 6, c = e & 63;
            double acc = 0.0;
            for (int q = max(r, c); q < nb; ++q) acc += I[q][r] * I[q][c];
            T[e] = acc;
        }
    }
}

// sweep finish: A[i,k] = U_i, A[k,i] = U_i^T (i != k), A[k,k] = -P
__global__ void k_sweep_finish(double *A, int ld, int m, int k, const double *U, const double *P) {
    const int kc0 = k * NB, kn = min(NB, m - kc0);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * kn; e += gridDim.x * blockDim.x) {
        int r = e / kn, c = e % kn;
        double v;
        if (r >= kc0 && r < kc0 + kn) v = -P[(r - kc0) * NB + c];
        else v = U[(size_t)r * NB + c];
        A[(size_t)r * ld + kc0 + c] = v;
        A[(size_t)(kc0 + c) * ld + r] = v;
    }
}

// Sigma-hat = Sigma_s (x) I3 + B  (all 3m x 3m, row-major)
__global__ void k_assemble_sigma_hat(const double *Sig, int lds, const double *Bc, int ldb,
                                     double *Sh, int ldh, int nS) {
    const int m3 = 3 * nS;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)m3 * m3;
         e += (size_t)gridDim.x * blockDim.x) {
        int r = (int)(e / m3), c = (int)(e % m3);
        double v = Bc[(size_t)r * ldb + c];
        if (r % 3 == c % 3) v += Sig[(size_t)(r / 3) * lds + c / 3];
        Sh[(size_t)r * ldh + c] = v;
    }
}

// y = (Sigma_s (x) I3) x  or  y = B x  : one warp per output row
__global__ void k_kron_matvec(const double *Sig, int lds, int nS, const double *x, double *y) {
    int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (row >= 3 * nS) return;
    int a = row / 3, i = row % 3;
    double acc = 0.0;
    for (int b = lane; b < nS; b += 32) acc += Sig[(size_t)a * lds + b] * x[3 * b + i];
    acc = warp_sum(acc);
    if (lane == 0) y[row] = acc;
}

__global__ void k_matvec(const double *M, int ldm, int n, const double *x, double *y) {
    int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (row >= n) return;
    double acc = 0.0;
    for (int c = lane; c < n; c += 32) acc += M[(size_t)row * ldm + c] * x[c];
    acc = warp_sum(acc);
    if (lane == 0) y[row] = acc;
}

// Solve L L^T u = b with the lower Cholesky factor (row-major): one CTA, 64-row blocks.
__global__ void __launch_bounds__(1024) k_chol_solve(const double *L, int ld, int n,
                                                     const double *b, double *u) {
    __shared__ double xb[NB];
    __shared__ double part[32][NB + 1];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // forward: u = L^{-1} b (u used as workspace)
    for (int kb = 0; kb < n; kb += NB) {
        const int nb = min(NB, n - kb);
        // partial dots: rows kb..kb+nb, columns 0..kb
        for (int r = wid; r < nb; r += 32) {
            double acc = 0.0;
            for (int c = lane; c < kb; c += 32) acc += L[(size_t)(kb + r) * ld + c] * u[c];
            acc = warp_sum(acc);
            if (lane == 0) xb[r] = b[kb + r] - acc;
        }
        __syncthreads();
        if (wid == 0) {
            // lane-per-row triangular solve of the nb x nb block, two rows per lane
            double v0 = lane < nb ? xb[lane] : 0.0, v1 = lane + 32 < nb ? xb[lane + 32] : 0.0;
            for (int k = 0; k < nb; ++k) {
                double mine = k < 32 ? v0 : v1;
                double xk = __shfl_sync(0xffffffffu, mine, k & 31);
                xk /= L[(size_t)(kb + k) * ld + kb + k];
                if (lane == (k & 31)) { if (k < 32) v0 = xk; else v1 = xk; }
                if (lane > k && lane < nb) v0 -= L[(size_t)(kb + lane) * ld + kb + k] * xk;
                if (lane + 32 > k && lane + 32 < nb) v1 -= L[(size_t)(kb + lane + 32) * ld + kb + k] * xk;
            }
            if (lane < nb) u[kb + lane] = v0;
            if (lane + 32 < nb) u[kb + lane + 32] = v1;
        }
        __syncthreads();
    }
    // backward: L^T u = y
    for (int kb = ((n - 1) / NB) * NB; kb >= 0; kb -= NB) {
        const int nb = min(NB, n - kb);
        // contributions from rows > kb+nb: sum_{r > kb+nb} L[r][kb + c] u[r]
        for (int c = tid; c < nb; c += 1024) part[0][c] = 0.0;
        __syncthreads();
        {
            const int c = tid & 63, g = tid >> 6;     // 16 row groups
            double acc = 0.0;
            if (c < nb)
                for (int r = kb + nb + g; r < n; r += 16) acc += L[(size_t)r * ld + kb + c] * u[r];
            part[g + 1][c] = acc;
        }
        __syncthreads();
        if (tid < nb) {
            double s = 0.0;
            for (int g = 0; g < 16; ++g) s += part[g + 1][tid];
            xb[tid] = u[kb + tid] - s;
        }
        __syncthreads();
        if (wid == 0) {
            double v0 = lane < nb ? xb[lane] : 0.0, v1 = lane + 32 < nb ? xb[lane + 32] : 0.0;
            for (int k = nb - 1; k >= 0; --k) {
                double mine = k < 32 ? v0 : v1;
                double xk = __shfl_sync(0xffffffffu, mine, k & 31);
                xk /= L[(size_t)(kb + k) * ld + kb + k];
                if (lane == (k & 31)) { if (k < 32) v0 = xk; else v1 = xk; }
                if (lane < k) v0 -= L[(size_t)(kb + k) * ld + kb + lane] * xk;
                if (lane + 32 < k) v1 -= L[(size_t)(kb + k) * ld + kb + lane + 32] * xk;
            }
            if (lane < nb) u[kb + lane] = v0;
            if (lane + 32 < nb) u[kb + lane + 32] = v1;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ host drivers ----------
static void tile_gemm(const TileArgs &a, int nblocks, cudaStream_t st) {
    if (nblocks <= 0) return;
    PDI_LAUNCH(k_tile_gemm, nblocks, 256, 2 * NB * SST * sizeof(double), st)(a);
}

constexpr int kPotrfSmem = 2 * NB * (NB + 1) * (int)sizeof(double);

void dense_init() {
    cudaFuncSetAttribute(k_tile_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * NB * SST * (int)sizeof(double));
    cudaFuncSetAttribute(k_tile_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, kPotrfSmem);
}

// In-place lower Cholesky of the m x m SPD matrix A (row-major, ld).  T: 64*64 scratch.
void dense_potrf(double *A, int ld, int m, double *T, int *info, cudaStream_t st) {
    const int nt = (m + NB - 1) / NB;
    for (int k = 0; k < nt; ++k) {
        PDI_LAUNCH(k_tile_potrf, 1, 256, kPotrfSmem, st)(A, ld, m, k, T, 0, info);
        TileArgs a{TM_TRSM, nt, k, m, A, ld, T, nullptr};
        tile_gemm(a, nt - k - 1, st);
        a.mode = TM_POTRF_UPD;
        int r = nt - k - 1;
        tile_gemm(a, r * (r + 1) / 2, st);
    }
}

// In-place inverse of the m x m SPD matrix A (full symmetric storage) by the block sweep
// operator; U: m_pad x 64 scratch, T: 64*64 scratch.
void dense_spd_inverse(double *A, int ld, int m, double *U, double *T, int *info, cudaStream_t st) {
    const int nt = (m + NB - 1) / NB;
    for (int k = 0; k < nt; ++k) {
        PDI_LAUNCH(k_tile_potrf, 1, 256, kPotrfSmem, st)(A, ld, m, k, T, 1, info);
        TileArgs a{TM_SWEEP_PANEL, nt, k, m, A, ld, T, U};
        tile_gemm(a, nt - 1, st);
        a.mode = TM_SWEEP_UPD;
        tile_gemm(a, (nt - 1) * (nt - 1), st);
        PDI_LAUNCH(k_sweep_finish, 64, 256, 0, st)(A, ld, m, k, U, T);
    }
}

void dense_negate(double *A, int ld, int m, cudaStream_t st);

__global__ void k_negate(double *A, int ld, int m) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)m * m;
         e += (size_t)gridDim.x * blockDim.x)
        A[(e / m) * ld + e % m] = -A[(e / m) * ld + e % m];
}
void dense_negate(double *A, int ld, int m, cudaStream_t st) {
    PDI_LAUNCH(k_negate, 256, 256, 0, st)(A, ld, m);
}

void launch_assemble_sigma_hat(const double *Sig, int lds, const double *Bc, int ldb, double *Sh,
                               int ldh, int nS, cudaStream_t st) {
    PDI_LAUNCH(k_assemble_sigma_hat, 512, 256, 0, st)(Sig, lds, Bc, ldb, Sh, ldh, nS);
}
void launch_kron_matvec(const double *Sig, int lds, int nS, const double *x, double *y,
                        cudaStream_t st) {
    int rows = 3 * nS;
    PDI_LAUNCH(k_kron_matvec, (rows * 32 + 255) / 256, 256, 0, st)(Sig, lds, nS, x, y);
}
void launch_matvec(const double *M, int ldm, int n, const double *x, double *y, cudaStream_t st) {
    PDI_LAUNCH(k_matvec, (n * 32 + 255) / 256, 256, 0, st)(M, ldm, n, x, y);
}
void launch_chol_solve(const double *L, int ld, int n, const double *b, double *u,
                       cudaStream_t st) {
    PDI_LAUNCH(k_chol_solve, 1, 1024, 0, st)(L, ld, n, b, u);
}

}  // namespace pdipc
