// The paper's PCG baseline for the contact global step (PAPER.md:128-134
// Eq. 5): split-preconditioned conjugate gradients on
//     (L^-1 H-hat L^-T) (L^T dx) = -L^-1 g-hat,   H-hat = H + script-B,   L L^T = H,
// i.e. on M = I + L^-1 script-B L^-T (eigenvalues >= 1).  One CG iteration applies M with one
// backward solve (t = L^-T p), the contact Hessian on S (y_S = B-check t_S, the dense 3n_c x 3n_c
// block the direct path assembles), one forward solve of the S-sparse vector E_S y_S, and the
// vector updates below.  Vectors are [nf][4] doubles in factor order (xyz + pad).  Dot products:
// block partials summed in a fixed order by every block that needs them (deterministic).
#include "kernels.h"
#include "prims.h"

#include "dev_common.cuh"

namespace pdipc {

constexpr int kCgNT = 256;
constexpr int kCgBlocks = 296;   // 2 per SM

// r = p = -w, z = 0; part[b] = partial r.r
__global__ void __launch_bounds__(kCgNT) k_cg_init(const double *__restrict__ w, double *__restrict__ r,
                                                   double *__restrict__ p, double *__restrict__ z, int nf,
                                                   double *__restrict__ part) {
    __shared__ double sh[kCgNT / 32];
    double acc = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * nf; e += gridDim.x * blockDim.x) {
        const double v = (e & 3) < 3 ? -w[e] : 0.0;
        r[e] = v;
        p[e] = v;
        z[e] = 0.0;
        acc += v * v;
    }
    acc = block_sum<kCgNT>(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// fixed-order sum of the block partials, broadcast to every thread of the block
__device__ __forceinline__ double sum_parts(const double *part, int n, double *sh) {
    __shared__ double bc;
    double v = 0.0;
    for (int b = threadIdx.x; b < n; b += blockDim.x) v += __ldcg(part + b);
    v = block_sum<kCgNT>(v, sh);            // valid in thread 0
    if (threadIdx.x == 0) bc = v;
    __syncthreads();
    v = bc;
    __syncthreads();
    return v;
}

// out = sparse E_S (B-check t_S): rows of S get B-check (3|S| x 3|S|, ld ldb) times t gathered on S
__global__ void __launch_bounds__(kCgNT) k_cg_bmul(const double *__restrict__ Bc, int ldb, const int *__restrict__ qS,
                                                   const int *__restrict__ nS_ptr, int capS,
                                                   const double *__restrict__ t, double *__restrict__ out) {
    const int nS = min(*nS_ptr, capS), m = 3 * nS;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int row = blockIdx.x * (kCgNT / 32) + wid; row < m; row += gridDim.x * (kCgNT / 32)) {
        double acc = 0.0;
        for (int c = lane; c < m; c += 32) acc += Bc[(size_t)row * ldb + c] * t[4 * (size_t)qS[c / 3] + c % 3];
        acc = warp_sum(acc);
        if (lane == 0) out[4 * (size_t)qS[row / 3] + row % 3] = acc;
    }
}

// q = p + f (f = L^-1 E_S B-check t_S); part[b] = partial p.q
__global__ void __launch_bounds__(kCgNT) k_cg_q(const double *__restrict__ p, const double *__restrict__ f,
                                                double *__restrict__ q, int nf, double *__restrict__ part) {
    __shared__ double sh[kCgNT / 32];
    double acc = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * nf; e += gridDim.x * blockDim.x) {
        const double v = (e & 3) < 3 ? p[e] + f[e] : 0.0;
        q[e] = v;
        acc += p[e] * v;
    }
    acc = block_sum<kCgNT>(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// alpha = rr / pq (rr from the previous iteration's partials rr_old); z += alpha p; r -= alpha q;
// rr_new[b] = partial r.r of the updated residual (double-buffered partial arrays: no block
// overwrites a partial another block may still be summing)
__global__ void __launch_bounds__(kCgNT) k_cg_step(const double *__restrict__ rr_old, const double *__restrict__ part_pq,
                                                   const double *__restrict__ p, const double *__restrict__ q,
                                                   double *__restrict__ z, double *__restrict__ r, int nf,
                                                   double *__restrict__ rr_new) {
    __shared__ double sh[kCgNT / 32];
    const double pq = sum_parts(part_pq, gridDim.x, sh);
    const double alpha = sum_parts(rr_old, gridDim.x, sh) / pq;
    double acc = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * nf; e += gridDim.x * blockDim.x) {
        z[e] += alpha * p[e];
        const double rv = r[e] - alpha * q[e];
        r[e] = rv;
        acc += rv * rv;
    }
    acc = block_sum<kCgNT>(acc, sh);
    if (threadIdx.x == 0) rr_new[blockIdx.x] = acc;
}

// beta = rr_new / rr_old; p = r + beta p; block 0 publishes rr_new in *host_rr (read by the
// host for the convergence test)
__global__ void __launch_bounds__(kCgNT) k_cg_dir(const double *__restrict__ rr_old, const double *__restrict__ rr_new,
                                                  const double *__restrict__ r, double *__restrict__ p, int nf,
                                                  double *__restrict__ host_rr) {
    __shared__ double sh[kCgNT / 32];
    const double rn = sum_parts(rr_new, gridDim.x, sh);
    if (rr_old) {
        const double beta = rn / sum_parts(rr_old, gridDim.x, sh);
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * nf; e += gridDim.x * blockDim.x)
            p[e] = r[e] + beta * p[e];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *host_rr = rn;
}

// Z = -z (the backward solve and the dx scatter negate: dx = -Pi^T L^-T Z = Pi^T L^-T z)
__global__ void k_cg_finish(const double *__restrict__ z, double *__restrict__ Z, int nf) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * nf; e += gridDim.x * blockDim.x)
        Z[e] = -z[e];
}

// part: [3][kCgBlocks] = p.q partials, r.r partials (two buffers, by iteration parity)
void launch_cg_init(const double *w, double *r, double *p, double *z, int nf, double *part, double *host_rr,
                    cudaStream_t st) {
    PDI_LAUNCH(k_cg_init, kCgBlocks, kCgNT, 0, st)(w, r, p, z, nf, part + kCgBlocks);
    PDI_LAUNCH(k_cg_dir, kCgBlocks, kCgNT, 0, st)(nullptr, part + kCgBlocks, r, p, nf, host_rr);
}
void launch_cg_bmul(const double *Bc, int ldb, const int *qS, const int *nS, int capS, const double *t,
                    double *out, int nf, cudaStream_t st) {
    dev_zero(out, sizeof(double) * 4 * (size_t)nf, st);
    PDI_LAUNCH(k_cg_bmul, kCgBlocks, kCgNT, 0, st)(Bc, ldb, qS, nS, capS, t, out);
}
void launch_cg_update(const double *f, double *p, double *q, double *z, double *r, int nf, double *part, int it,
                      double *host_rr, cudaStream_t st) {
    double *pq = part, *rr_old = part + (size_t)(1 + (it & 1)) * kCgBlocks,
           *rr_new = part + (size_t)(1 + ((it + 1) & 1)) * kCgBlocks;
    PDI_LAUNCH(k_cg_q, kCgBlocks, kCgNT, 0, st)(p, f, q, nf, pq);
    PDI_LAUNCH(k_cg_step, kCgBlocks, kCgNT, 0, st)(rr_old, pq, p, q, z, r, nf, rr_new);
    PDI_LAUNCH(k_cg_dir, kCgBlocks, kCgNT, 0, st)(rr_old, rr_new, r, p, nf, host_rr);
}
void launch_cg_finish(const double *z, double *Z, int nf, cudaStream_t st) {
    PDI_LAUNCH(k_cg_finish, kCgBlocks, kCgNT, 0, st)(z, Z, nf);
}
int cg_partials() { return kCgBlocks; }

}  // namespace pdipc
