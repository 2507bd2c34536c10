// Elastic part of the PD+IPC iteration: actuation ingestion, the fused local step (a1),
// the atomics-free elastic gradient gather (a2), surface interpolation s = W x (a3), and the
// per-tet / per-vertex reductions of the line search (a11) and the update x += alpha dx.
//
// PAPER.md:73-79 (Eq. 1): E_i(x) = min_R ||F_i(x) - R A_i||_F^2; "we find the best rotation
// R_i using the polar decomposition of F_i A_i" in parallel over elements.
// PAPER.md:97,113 (Eq. 4): elastic gradient sum_i w_i G_i^T (G_i x - p_i).
// s = W x.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

#include "dev_common.cuh"

namespace pdipc {

// ------------------------------------------------------------------ actuation ingestion ----
// A9 [T][9] row-major (ABI layout) -> SoA A6 [6][T] = (a00, a01, a02, a11, a12, a22).
__global__ void k_ingest_actuation(const double *__restrict__ A9, double *__restrict__ A6, int T) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    const double *a = A9 + 9 * (size_t)t;
    A6[0 * (size_t)T + t] = a[0];
    A6[1 * (size_t)T + t] = a[1];
    A6[2 * (size_t)T + t] = a[2];
    A6[3 * (size_t)T + t] = a[4];
    A6[4 * (size_t)T + t] = a[5];
    A6[5 * (size_t)T + t] = a[8];
}

// Actuation check on the device (pd_ipc_step rejects a call whose A_next has any matrix that is
// non-finite (bit 1), not symmetric to 1e-9 of its largest entry (bit 2) or of det <= 0 (bit 4))
__global__ void k_validate_actuation(const double *__restrict__ A, size_t nmat, int *__restrict__ flag) {
    int bits = 0;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < nmat; t += (size_t)gridDim.x * blockDim.x) {
        const double *a = A + 9 * t;
        double v[9], mx = 0.0;
        bool fin = true;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            v[k] = a[k];
            fin &= isfinite(v[k]);
            mx = fmax(mx, fabs(v[k]));
        }
        if (!fin) { bits |= 1; continue; }
        const double asym = fmax(fmax(fabs(v[1] - v[3]), fabs(v[2] - v[6])), fabs(v[5] - v[7]));
        if (asym > 1e-9 * mx) bits |= 2;
        const double det = v[0] * (v[4] * v[8] - v[5] * v[7]) - v[1] * (v[3] * v[8] - v[5] * v[6]) +
                           v[2] * (v[3] * v[7] - v[4] * v[6]);
        if (!(det > 0)) bits |= 4;
    }
    if (bits) atomicOr(flag, bits);
}

// ------------------------------------------------------------------ 3x3 polar -------------
// Symmetric 3x3 eigen-decomposition by cyclic Jacobi (FP64).  S = V diag(l) V^T.
__device__ __forceinline__ void jacobi_rot(double S[3][3], double V[3][3], int p, int q) {
    double apq = S[p][q];
    if (fabs(apq) < 1e-300) return;
    double tau = (S[q][q] - S[p][p]) / (2.0 * apq);
    double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
    double c = rsqrt(1.0 + t * t);
    double s = t * c;
    // S <- J^T S J
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double skp = S[k][p], skq = S[k][q];
        S[k][p] = c * skp - s * skq;
        S[k][q] = s * skp + c * skq;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double spk = S[p][k], sqk = S[q][k];
        S[p][k] = c * spk - s * sqk;
        S[q][k] = s * spk + c * sqk;
    }
    S[p][q] = S[q][p] = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double vkp = V[k][p], vkq = V[k][q];
        V[k][p] = c * vkp - s * vkq;
        V[k][q] = s * vkp + c * vkq;
    }
}

// Rotation factor R of M with the reflection fix: SVD M = U S V^T, flip the
// smallest singular axis when det < 0, R = U V^T.  Computed from the eigenvectors V of M^T M
// (Jacobi), u1 = M v1/|M v1|, u2 = Gram-Schmidt(M v2), u3 = u1 x u2, v3 = v1 x v2.
__device__ void polar_rotation(const double M[3][3], double R[3][3]) {
    double S[3][3], V[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            S[i][j] = M[0][i] * M[0][j] + M[1][i] * M[1][j] + M[2][i] * M[2][j];
            V[i][j] = i == j ? 1.0 : 0.0;
        }
    const double tr2 = S[0][0] * S[0][0] + S[1][1] * S[1][1] + S[2][2] * S[2][2];
    for (int sweep = 0; sweep < 12; ++sweep) {
        double off = S[0][1] * S[0][1] + S[0][2] * S[0][2] + S[1][2] * S[1][2];
        if (off <= 1e-30 * tr2) break;   // off-diagonal <= 1e-15 of the diagonal (squared)
        jacobi_rot(S, V, 0, 1);
        jacobi_rot(S, V, 0, 2);
        jacobi_rot(S, V, 1, 2);
    }
    // order eigenvalues descending
    int i1 = 0, i2 = 1, i3 = 2;
    double l[3] = {S[0][0], S[1][1], S[2][2]};
    if (l[i1] < l[i2]) { int t = i1; i1 = i2; i2 = t; }
    if (l[i2] < l[i3]) { int t = i2; i2 = i3; i3 = t; }
    if (l[i1] < l[i2]) { int t = i1; i1 = i2; i2 = t; }
    double v1[3] = {V[0][i1], V[1][i1], V[2][i1]};
    double v2[3] = {V[0][i2], V[1][i2], V[2][i2]};
    double u1[3], u2[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        u1[a] = M[a][0] * v1[0] + M[a][1] * v1[1] + M[a][2] * v1[2];
        u2[a] = M[a][0] * v2[0] + M[a][1] * v2[1] + M[a][2] * v2[2];
    }
    double n1 = sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
    if (n1 > 0) {
        for (int a = 0; a < 3; ++a) u1[a] /= n1;
    } else {
        u1[0] = 1; u1[1] = 0; u1[2] = 0;
    }
    double dp = u1[0] * u2[0] + u1[1] * u2[1] + u1[2] * u2[2];
    for (int a = 0; a < 3; ++a) u2[a] -= dp * u1[a];
    double n2 = sqrt(u2[0] * u2[0] + u2[1] * u2[1] + u2[2] * u2[2]);
    if (n2 > 1e-150 && n2 > 1e-14 * n1) {
        for (int a = 0; a < 3; ++a) u2[a] /= n2;
    } else {                                   // rank <= 1: any unit vector orthogonal to u1
        double e[3] = {0, 0, 0};
        int k = fabs(u1[0]) < 0.6 ? 0 : (fabs(u1[1]) < 0.6 ? 1 : 2);
        e[k] = 1.0;
        double d = u1[k];
        for (int a = 0; a < 3; ++a) u2[a] = e[a] - d * u1[a];
        double nn = sqrt(u2[0] * u2[0] + u2[1] * u2[1] + u2[2] * u2[2]);
        for (int a = 0; a < 3; ++a) u2[a] /= nn;
    }
    double u3[3] = {u1[1] * u2[2] - u1[2] * u2[1], u1[2] * u2[0] - u1[0] * u2[2],
                    u1[0] * u2[1] - u1[1] * u2[0]};
    double v3[3] = {v1[1] * v2[2] - v1[2] * v2[1], v1[2] * v2[0] - v1[0] * v2[2],
                    v1[0] * v2[1] - v1[1] * v2[0]};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) R[a][b] = u1[a] * v1[b] + u2[a] * v2[b] + u3[a] * v3[b];
}

// Rotation factor of M by the scaled Newton iteration X <- (g X + X^{-T} / g) / 2 (Higham), with
// X^{-T} from the cofactor matrix and the Frobenius scaling g = (|X^{-1}|_F / |X|_F)^{1/2}.  For
// det M > 0 it converges quadratically to the unique R in SO(3) with M = R U (the same R as the
// SVD route); 4-6 iterations at the strains of the workloads, no eigen-decomposition.  Returns
// false when det M <= 0, with X still equal to M (the caller takes the SVD route with the
// reflection fix).  In place: X = M on entry, R on exit.
__device__ __forceinline__ bool polar_newton(double X[3][3]) {
    for (int it = 0; it < 16; ++it) {
        double C[3][3];
        C[0][0] = X[1][1] * X[2][2] - X[1][2] * X[2][1];
        C[0][1] = X[1][2] * X[2][0] - X[1][0] * X[2][2];
        C[0][2] = X[1][0] * X[2][1] - X[1][1] * X[2][0];
        C[1][0] = X[0][2] * X[2][1] - X[0][1] * X[2][2];
        C[1][1] = X[0][0] * X[2][2] - X[0][2] * X[2][0];
        C[1][2] = X[0][1] * X[2][0] - X[0][0] * X[2][1];
        C[2][0] = X[0][1] * X[1][2] - X[0][2] * X[1][1];
        C[2][1] = X[0][2] * X[1][0] - X[0][0] * X[1][2];
        C[2][2] = X[0][0] * X[1][1] - X[0][1] * X[1][0];
        const double det = X[0][0] * C[0][0] + X[0][1] * C[0][1] + X[0][2] * C[0][2];
        if (!(det > 0.0)) return false;          // Newton keeps the sign of det: only at it == 0
        const double idet = 1.0 / det;
        double a = 0.5, b = 0.5 * idet;
        if (it < 2) {                            // Frobenius scaling for the first steps only
            double nx = 0.0, nc = 0.0;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    nx += X[i][j] * X[i][j];
                    nc += C[i][j] * C[i][j];
                }
            const double z = sqrt(nc / nx) * idet;       // g^2, |X^-1|_F = |C|_F / det
            const double rz = rsqrt(z);                  // a = g/2 = z rz / 2, b = 1/(2 g det)
            a = 0.5 * z * rz;
            b = 0.5 * idet * rz;
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) X[i][j] = a * X[i][j] + b * C[i][j];
        // convergence from the determinant computed anyway: after a (scaled) Newton step every
        // singular value is (g s + 1/(g s))/2 >= 1, so det X - 1 = prod(1 + d_i) - 1 >= sum d_i;
        // det X < 1 + 1e-9 bounds every error d_i by 1e-9, and the step just taken (quadratic,
        // Higham) leaves X at rounding level
        if (it >= 1 && det < 1.0 + 1e-9) break;
    }
    return true;
}

// ------------------------------------------------------------------ a1 local step ---------
// One thread per tet.  Reads tet (int4), x (double4 per vertex, L2-resident gather),
// B (SoA [9][T]), A (SoA [6][T]), w; writes the per-corner elastic forces
// f_{i,c} = w_i (F_i - P_i) g_{i,c} as fc[T][4][3] (coalesced 96 B per tet) and, when
// p != nullptr, p_i = vec(R_i A_i) (SoA [9][T]) for the parity hook.
// L2 policy: the once-per-iteration mesh streams (tets, B, A, w) are read evict-first and the
// forces are written with an evict-last policy, so the forces the gather reads next are the
// lines the L2 keeps (C5 1M: local step 63.3 -> 61.8 us, gather 38.5 -> 36.3 us,
// tools/gather_ab.sh; a persisting-L2 set-aside for the forces measured slower).
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_f64x2_evict_last(double2 *a, double x, double y, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(x), "d"(y), "l"(pol)
                 : "memory");
}
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_local_step(
    const int4 *__restrict__ tets, const double4 *__restrict__ x, const double *__restrict__ B,
    const double *__restrict__ A6, const double *__restrict__ w, int T, double *__restrict__ fc,
    double *__restrict__ p, int *__restrict__ clr, int nseq, long long xs, int clrs) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    // the iteration's device counters of every sequence, cleared by its first kernel: active-pair
    // counts [0, 1] and info / capacity / hash flags [4, 8) (the candidate counts [2, 3] carry
    // over, see R8)
    if (clr)
        for (int i = t; i < 8 * nseq; i += gridDim.x * blockDim.x)
            if ((i & 7) < 2 || (i & 7) >= 4) clr[(i >> 3) * clrs + (i & 7)] = 0;
    if (t >= T) return;
    // the mesh data of the tet is read once for all sequences of the batch
    const int4 tv = __ldcs(tets + t);
    double Bm[3][3];
#pragma unroll
    for (int k = 0; k < 9; ++k) Bm[k / 3][k % 3] = __ldcs(B + (size_t)k * T + t);
    const double wt = __ldcs(w + t);
    for (int sq = 0; sq < nseq; ++sq) {
    const double4 *xq = x + sq * xs;
    const double *A6q = A6 + (size_t)sq * 6 * T;
    const double4 x0 = xq[tv.x], x1 = xq[tv.y], x2 = xq[tv.z], x3 = xq[tv.w];
    const double a00 = __ldcs(A6q + t), a01 = __ldcs(A6q + (size_t)T + t), a02 = __ldcs(A6q + 2 * (size_t)T + t),
                 a11 = __ldcs(A6q + 3 * (size_t)T + t), a12 = __ldcs(A6q + 4 * (size_t)T + t),
                 a22 = __ldcs(A6q + 5 * (size_t)T + t);
    const double A[3][3] = {{a00, a01, a02}, {a01, a11, a12}, {a02, a12, a22}};
    // D_s = [x1-x0, x2-x0, x3-x0] (columns); F = D_s B
    const double Ds[3][3] = {{x1.x - x0.x, x2.x - x0.x, x3.x - x0.x},
                             {x1.y - x0.y, x2.y - x0.y, x3.y - x0.y},
                             {x1.z - x0.z, x2.z - x0.z, x3.z - x0.z}};
    double F[3][3], R[3][3], P[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) F[a][b] = Ds[a][0] * Bm[0][b] + Ds[a][1] * Bm[1][b] + Ds[a][2] * Bm[2][b];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) R[a][b] = F[a][0] * A[0][b] + F[a][1] * A[1][b] + F[a][2] * A[2][b];
    if (!polar_newton(R)) {                          // det <= 0: SVD route, reflection fix
        const double M[3][3] = {{R[0][0], R[0][1], R[0][2]}, {R[1][0], R[1][1], R[1][2]},
                                {R[2][0], R[2][1], R[2][2]}};
        polar_rotation(M, R);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) P[a][b] = R[a][0] * A[0][b] + R[a][1] * A[1][b] + R[a][2] * A[2][b];
    if (p) {
#pragma unroll
        for (int k = 0; k < 9; ++k) p[(size_t)sq * 9 * T + (size_t)k * T + t] = P[k / 3][k % 3];
    }
    // r = w (F - P);  f_c = r g_c, g_c = row c-1 of B (c = 1..3), f_0 = -(f_1 + f_2 + f_3)
    double r[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) r[a][b] = wt * (F[a][b] - P[a][b]);
    double f[4][3];
#pragma unroll
    for (int c = 1; c < 4; ++c)
#pragma unroll
        for (int a = 0; a < 3; ++a)
            f[c][a] = r[a][0] * Bm[c - 1][0] + r[a][1] * Bm[c - 1][1] + r[a][2] * Bm[c - 1][2];
#pragma unroll
    for (int a = 0; a < 3; ++a) f[0][a] = -(f[1][a] + f[2][a] + f[3][a]);
    double2 *o = reinterpret_cast<double2 *>(fc + (size_t)sq * 12 * T + 12 * (size_t)t);
    const unsigned long long pol = l2_policy_evict_last();
    st_f64x2_evict_last(o + 0, f[0][0], f[0][1], pol);
    st_f64x2_evict_last(o + 1, f[0][2], f[1][0], pol);
    st_f64x2_evict_last(o + 2, f[1][1], f[1][2], pol);
    st_f64x2_evict_last(o + 3, f[2][0], f[2][1], pol);
    st_f64x2_evict_last(o + 4, f[2][2], f[3][0], pol);
    st_f64x2_evict_last(o + 5, f[3][1], f[3][2], pol);
    }
}

// ------------------------------------------------------------------ a2 gather -------------
// g_el[q] = sum over incidences (t, c) of vertex q2v[q] of f_{t,c}: transpose-CSR gather in
// factor order, deterministic, no atomics.  Output double4 [nf] (w = 0).
// 8 lanes per free vertex: lane l sums the incident corner forces l, l+8, ... of the vertex's
// transpose-incidence list, then a fixed xor tree over the 8 lanes (deterministic order).  The
// index loads of a lane are issued together (up to kGatherBatch), then all their force loads,
// so the index -> force dependency costs one memory latency per batch, not per incidence.
constexpr int kGatherLanes = 8;
constexpr int kGatherBatch = 4;
__global__ void __launch_bounds__(256) k_gather_elastic(const int *__restrict__ inc_ptr, const int *__restrict__ inc,
                                                        const double *__restrict__ fc, int nf,
                                                        double4 *__restrict__ g, long long fcs) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    fc += (size_t)blockIdx.y * fcs;        // sequence blockIdx.y: its forces and gradient
    g += (size_t)blockIdx.y * nf;
    const int q = gid / kGatherLanes, l = gid % kGatherLanes;
    double gx = 0, gy = 0, gz = 0;
    if (q < nf) {
        const int k0 = __ldg(inc_ptr + q), k1 = __ldg(inc_ptr + q + 1);
        for (int kb = k0 + l; kb < k1; kb += kGatherLanes * kGatherBatch) {
            int tc[kGatherBatch];
#pragma unroll
            for (int u = 0; u < kGatherBatch; ++u) {
                const int k = kb + u * kGatherLanes;
                tc[u] = k < k1 ? __ldg(inc + k) : -1;
            }
            double f[kGatherBatch][3];
#pragma unroll
            for (int u = 0; u < kGatherBatch; ++u) {
                if (tc[u] >= 0) {
                    const double *p = fc + 12 * (size_t)(tc[u] >> 2) + 3 * (tc[u] & 3);
                    f[u][0] = __ldcs(p);
                    f[u][1] = __ldcs(p + 1);
                    f[u][2] = __ldcs(p + 2);
                } else {
                    f[u][0] = f[u][1] = f[u][2] = 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kGatherBatch; ++u) {   // same order as one incidence at a time
                gx += f[u][0];
                gy += f[u][1];
                gz += f[u][2];
            }
        }
    }
#pragma unroll
    for (int o = kGatherLanes / 2; o > 0; o >>= 1) {
        gx += __shfl_xor_sync(0xffffffffu, gx, o);
        gy += __shfl_xor_sync(0xffffffffu, gy, o);
        gz += __shfl_xor_sync(0xffffffffu, gz, o);
    }
    if (q < nf && l == 0) g[q] = make_double4(gx, gy, gz, 0.0);
}

// ------------------------------------------------------------------ a3 s = W x ------------
__global__ void k_surface(const int *__restrict__ Wp, const int *__restrict__ Wc,
                          const double *__restrict__ Wv, const double4 *__restrict__ x, int Ns,
                          double4 *__restrict__ s) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= Ns) return;
    double sx = 0, sy = 0, sz = 0;
    for (int k = Wp[j]; k < Wp[j + 1]; ++k) {
        double wv = Wv[k];
        double4 xv = x[Wc[k]];
        sx += wv * xv.x;
        sy += wv * xv.y;
        sz += wv * xv.z;
    }
    s[j] = make_double4(sx, sy, sz, 0.0);
}

// ds = W dx (dx given per vertex, zero on fixed)
// (same kernel as k_surface applied to dx)

// ------------------------------------------------------------------ a11 reductions ---------
// partial[b] = sum over tets of block b of w ||D_s(dx) B||^2   (= dx^T H dx over all DOFs)
__global__ void __launch_bounds__(256) k_quad_partials(const int4 *__restrict__ tets,
                                                       const double4 *__restrict__ dx,
                                                       const double *__restrict__ B,
                                                       const double *__restrict__ w, int T,
                                                       double *__restrict__ part) {
    __shared__ double sh[8];
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    double v = 0.0;
    if (t < T) {
        const int4 tv = tets[t];
        const double4 x0 = dx[tv.x], x1 = dx[tv.y], x2 = dx[tv.z], x3 = dx[tv.w];
        const double Ds[3][3] = {{x1.x - x0.x, x2.x - x0.x, x3.x - x0.x},
                                 {x1.y - x0.y, x2.y - x0.y, x3.y - x0.y},
                                 {x1.z - x0.z, x2.z - x0.z, x3.z - x0.z}};
        double Bm[3][3];
#pragma unroll
        for (int k = 0; k < 9; ++k) Bm[k / 3][k % 3] = B[(size_t)k * T + t];
        double acc = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                double F = Ds[a][0] * Bm[0][b] + Ds[a][1] * Bm[1][b] + Ds[a][2] * Bm[2][b];
                acc += F * F;
            }
        v = w[t] * acc;
    }
    v = block_sum<256>(v, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// partial[b] = sum over q of block b of g_el[q] . dx[q2v[q]]
__global__ void __launch_bounds__(256) k_gdx_partials(const double4 *__restrict__ g,
                                                      const double4 *__restrict__ dx,
                                                      const int *__restrict__ q2v, int nf,
                                                      double *__restrict__ part) {
    __shared__ double sh[8];
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    double v = 0.0;
    if (q < nf) {
        double4 a = g[q], b = dx[q2v[q]];
        v = a.x * b.x + a.y * b.y + a.z * b.z;
    }
    v = block_sum<256>(v, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// x_F += alpha dx, unless this iteration raised a flag (flags = [Cholesky info, capacity bits,
// static hash overflow, swept hash overflow]) or an earlier iteration of the batch did (abort =
// [sticky, iteration index, why]); the first failing iteration records itself.
// Convergence-terminated frames (SURVEY Z10 option, "while not converged"; cv =
// [converged, iterations applied, block ticket], amax = max |alpha dx| of the iteration as the
// bits of a non-negative double): once an iteration moves no free vertex by tol or more, the
// sequence is converged and the rest of the pd_ipc_step call leaves it untouched.
__global__ void k_update(double4 *__restrict__ x, const double4 *__restrict__ dx,
                         const int *__restrict__ q2v, int nf, const double *__restrict__ alpha,
                         const int *__restrict__ flags, int *__restrict__ abort, int it, int *__restrict__ cv,
                         unsigned long long *__restrict__ amax, double tol) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (cv[0]) return;                                  // converged earlier in this call
    double mv = 0.0;
    bool applied = false;
    if (q < nf) {
    // alpha[3] == 2: the line search saw a non-finite gradient, dx or energy (k_ls_round)
    const int nonfinite = alpha[3] == 2.0 ? 64 : 0;
    const int bad = flags[0] | flags[1] | flags[2] | flags[3] | nonfinite;
    if (bad) {
        if (q == 0 && abort[0] == 0) {
            abort[0] = 1;
            abort[1] = it;
            abort[2] = flags[1] | (flags[2] ? 8 : 0) | (flags[3] ? 16 : 0) | (flags[0] ? 32 : 0) | nonfinite;
        }
        return;
    }
    if (abort[0]) return;
    const int v = q2v[q];
    const double a = *alpha;
    double4 xv = x[v], d = dx[v];
    xv.x += a * d.x;
    xv.y += a * d.y;
    xv.z += a * d.z;
    x[v] = xv;
    mv = fmax(fabs(a * d.x), fmax(fabs(a * d.y), fabs(a * d.z)));
    applied = true;
    }
    // block max of |alpha dx|, then the last block to finish decides (and resets the scratch)
    __shared__ double wm[8];
    __shared__ bool last;
    for (int o = 16; o > 0; o >>= 1) mv = fmax(mv, __shfl_xor_sync(0xffffffffu, mv, o));
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mv;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < (int)blockDim.x / 32; ++w) b = fmax(b, wm[w]);
        atomicMax(amax, (unsigned long long)__double_as_longlong(b));
        __threadfence();
        last = atomicAdd(cv + 2, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    const double m = __longlong_as_double((long long)atomicExch(amax, 0ull));
    cv[2] = 0;
    if (applied || nf == 0) {
        cv[1] += 1;                                     // iterations applied in this call
        if (tol > 0.0 && m < tol) cv[0] = 1;
    }
}

// scatter dx from factor order (solution of the backward solve, [nf][4], negated) to vertices
// (fixed vertices keep dx = 0 from the clear at create); also seeds the CCD minimum *amin = 1
__global__ void k_scatter_dx(const double *__restrict__ z, const int *__restrict__ q2v, int nf,
                             double4 *__restrict__ dx, double *__restrict__ amin, int n, int amin_stride) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    z += (size_t)blockIdx.y * 4 * nf;      // sequence blockIdx.y
    dx += (size_t)blockIdx.y * n;
    if (amin) amin += (size_t)blockIdx.y * amin_stride;
    if (q == 0 && amin) *amin = 1.0;
    if (q >= nf) return;
    const double *r = z + 4 * (size_t)q;
    dx[q2v[q]] = make_double4(-r[0], -r[1], -r[2], 0.0);
}

__global__ void k_set_double(double *p, double v) { *p = v; }

// ------------------------------------------------------------------ f3 true-energy LS -----
// Elastic part of the true-energy line search (SURVEY 8(f) f3, Z7's alternative): for the trials
// alpha_h = am 2^-(h0+h), h < KH, block partials of 1/2 sum_i w_i (e_i(x + alpha_h dx) - e_i(x)),
// e_i(y) = min_{R in SO(3)} ||F_i(y) - R A_i||_F^2 (Eq. 1), R = polar(F_i A_i)
// by the local step's scaled Newton iteration, SVD route with the reflection fix for
// det <= 0.  One thread per tet (grid-stride over a fixed grid: deterministic block sums);
// written to pte[h * gridDim.x + block] and summed in fixed order by k_ls_round's decision.
__device__ __forceinline__ double true_elastic_e(const double F[3][3], const double A[3][3]) {
    double R[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) R[a][b] = F[a][0] * A[0][b] + F[a][1] * A[1][b] + F[a][2] * A[2][b];
    if (!polar_newton(R)) {
        const double M[3][3] = {{R[0][0], R[0][1], R[0][2]}, {R[1][0], R[1][1], R[1][2]},
                                {R[2][0], R[2][1], R[2][2]}};
        polar_rotation(M, R);
    }
    double e = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const double r = F[a][b] - (R[a][0] * A[0][b] + R[a][1] * A[1][b] + R[a][2] * A[2][b]);
            e += r * r;
        }
    return e;
}
template <int KH>
__global__ void __launch_bounds__(256) k_ls_true_elastic(const int4 *__restrict__ tets, const double4 *__restrict__ x,
                                                         const double4 *__restrict__ dx, const double *__restrict__ B,
                                                         const double *__restrict__ A6, const double *__restrict__ w,
                                                         int T, const double *__restrict__ amin,
                                                         const double *__restrict__ ls, int h0,
                                                         double *__restrict__ pte) {
    if (h0 > 0 && ls[1] != 0.0) return;    // accepted (or aborted) in an earlier round
    __shared__ double sh[8];
    const double am = h0 == 0 ? *amin : ls[0];
    double acc[KH];
#pragma unroll
    for (int h = 0; h < KH; ++h) acc[h] = 0.0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        const int4 tv = tets[t];
        double Bm[3][3];
#pragma unroll
        for (int k = 0; k < 9; ++k) Bm[k / 3][k % 3] = B[(size_t)k * T + t];
        const double a00 = A6[t], a01 = A6[(size_t)T + t], a02 = A6[2 * (size_t)T + t], a11 = A6[3 * (size_t)T + t],
                     a12 = A6[4 * (size_t)T + t], a22 = A6[5 * (size_t)T + t];
        const double A[3][3] = {{a00, a01, a02}, {a01, a11, a12}, {a02, a12, a22}};
        const double4 X[4] = {x[tv.x], x[tv.y], x[tv.z], x[tv.w]};
        const double4 D[4] = {dx[tv.x], dx[tv.y], dx[tv.z], dx[tv.w]};
        const double hw = 0.5 * w[t];
        double e0;
        {
            double F[3][3];
            const double Ds[3][3] = {{X[1].x - X[0].x, X[2].x - X[0].x, X[3].x - X[0].x},
                                     {X[1].y - X[0].y, X[2].y - X[0].y, X[3].y - X[0].y},
                                     {X[1].z - X[0].z, X[2].z - X[0].z, X[3].z - X[0].z}};
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) F[a][b] = Ds[a][0] * Bm[0][b] + Ds[a][1] * Bm[1][b] + Ds[a][2] * Bm[2][b];
            e0 = true_elastic_e(F, A);
        }
#pragma unroll 1
        for (int h = 0; h < KH; ++h) {
            const double al = ldexp(am, -(h0 + h));
            double Y[4][3];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                Y[c][0] = X[c].x + al * D[c].x;
                Y[c][1] = X[c].y + al * D[c].y;
                Y[c][2] = X[c].z + al * D[c].z;
            }
            double F[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    F[a][b] = (Y[1][a] - Y[0][a]) * Bm[0][b] + (Y[2][a] - Y[0][a]) * Bm[1][b] +
                              (Y[3][a] - Y[0][a]) * Bm[2][b];
            acc[h] += hw * (true_elastic_e(F, A) - e0);
        }
    }
#pragma unroll 1
    for (int h = 0; h < KH; ++h) {
        const double v = block_sum<256>(acc[h], sh);
        if (threadIdx.x == 0) pte[(size_t)h * gridDim.x + blockIdx.x] = v;
    }
}
int ls_te_blocks(int T) { return std::max(1, std::min((T + 255) / 256, 148 * 4)); }
int launch_ls_true_elastic(const int4 *tets, const double4 *x, const double4 *dx, const double *B, const double *A6,
                           const double *w, int T, const double *amin, const double *ls, int h0, int kh,
                           double *pte, cudaStream_t st) {
    const int nb = ls_te_blocks(T);
    if (kh == 1)
        PDI_LAUNCH(k_ls_true_elastic<1>, nb, 256, 0, st)(tets, x, dx, B, A6, w, T, amin, ls, h0, pte);
    else if (kh == 8)
        PDI_LAUNCH(k_ls_true_elastic<8>, nb, 256, 0, st)(tets, x, dx, B, A6, w, T, amin, ls, h0, pte);
    else
        PDI_LAUNCH(k_ls_true_elastic<22>, nb, 256, 0, st)(tets, x, dx, B, A6, w, T, amin, ls, h0, pte);
    return nb;
}

// ------------------------------------------------------------------ host wrappers ---------
void launch_set_double(double *p, double v, cudaStream_t st) { PDI_LAUNCH(k_set_double, 1, 1, 0, st)(p, v); }

void launch_ingest_actuation(const double *A9, double *A6, int T, cudaStream_t st) {
    PDI_LAUNCH(k_ingest_actuation, (T + 255) / 256, 256, 0, st)(A9, A6, T);
}
void launch_validate_actuation(const double *A, size_t nmat, int *flag, cudaStream_t st) {
    PDI_LAUNCH(k_validate_actuation, 148 * 8, 256, 0, st)(A, nmat, flag);
}
static int g_ls_minb = 4;   // resident CTAs per SM the local step is compiled for (PDIPC_LS_MINB)
void elastic_init(int) {
    if (const char *e = std::getenv("PDIPC_LS_MINB")) g_ls_minb = std::atoi(e);
}
void launch_local_step(const int4 *tets, const double4 *x, const double *B, const double *A6,
                       const double *w, int T, double *fc, double *p, int *clr, int nseq, long long xs,
                       int clrs, cudaStream_t st) {
    if (T <= 0) return;
    // latency-bound small meshes (fewer than ~4 CTAs of 128 per SM): half-size CTAs spread the
    // tets over twice as many CTAs, balancing the SMs
    const int nt = T < 4 * 148 * 128 ? 64 : 128;
    if (g_ls_minb == 5)
        PDI_LAUNCH(k_local_step<5>, (T + nt - 1) / nt, nt, 0, st)(tets, x, B, A6, w, T, fc, p, clr, nseq, xs, clrs);
    else
        PDI_LAUNCH(k_local_step<4>, (T + nt - 1) / nt, nt, 0, st)(tets, x, B, A6, w, T, fc, p, clr, nseq, xs, clrs);
}
void launch_gather_elastic(const int *inc_ptr, const int *inc, const double *fc, int nf,
                           double4 *g, int nseq, long long fcs, cudaStream_t st) {
    if (nf <= 0) return;
    PDI_LAUNCH(k_gather_elastic, dim3((unsigned)(((long long)nf * kGatherLanes + 255) / 256), nseq), 256, 0, st)(
        inc_ptr, inc, fc, nf, g, fcs);
}
void launch_surface(const int *Wp, const int *Wc, const double *Wv, const double4 *x, int Ns,
                    double4 *s, cudaStream_t st) {
    if (Ns > 0) PDI_LAUNCH(k_surface, (Ns + 127) / 128, 128, 0, st)(Wp, Wc, Wv, x, Ns, s);
}
int quad_partials(const int4 *tets, const double4 *dx, const double *B, const double *w, int T,
                  double *part, cudaStream_t st) {
    int nb = (T + 255) / 256;
    PDI_LAUNCH(k_quad_partials, nb, 256, 0, st)(tets, dx, B, w, T, part);
    return nb;
}
int gdx_partials(const double4 *g, const double4 *dx, const int *q2v, int nf, double *part,
                 cudaStream_t st) {
    int nb = (nf + 255) / 256;
    PDI_LAUNCH(k_gdx_partials, nb, 256, 0, st)(g, dx, q2v, nf, part);
    return nb;
}
// both elastic line-search reductions in one launch: blocks [0, nb1) the gradient term,
// [nb1, nb1 + nb2) the quadratic term; part[block] as the two separate kernels write them
__global__ void __launch_bounds__(256) k_elastic_partials(const double4 *__restrict__ g,
                                                          const double4 *__restrict__ dx,
                                                          const int *__restrict__ q2v, int nf,
                                                          const int4 *__restrict__ tets,
                                                          const double *__restrict__ B,
                                                          const double *__restrict__ w, int T, int nb1,
                                                          double *__restrict__ part) {
    __shared__ double sh[8];
    double v = 0.0;
    if ((int)blockIdx.x < nb1) {
        const int q = blockIdx.x * blockDim.x + threadIdx.x;
        if (q < nf) {
            const double4 a = g[q], b = dx[q2v[q]];
            v = a.x * b.x + a.y * b.y + a.z * b.z;
        }
    } else {
        const int t = (blockIdx.x - nb1) * blockDim.x + threadIdx.x;
        if (t < T) {
            const int4 tv = tets[t];
            const double4 x0 = dx[tv.x], x1 = dx[tv.y], x2 = dx[tv.z], x3 = dx[tv.w];
            const double Ds[3][3] = {{x1.x - x0.x, x2.x - x0.x, x3.x - x0.x},
                                     {x1.y - x0.y, x2.y - x0.y, x3.y - x0.y},
                                     {x1.z - x0.z, x2.z - x0.z, x3.z - x0.z}};
            double Bm[3][3];
#pragma unroll
            for (int k = 0; k < 9; ++k) Bm[k / 3][k % 3] = B[(size_t)k * T + t];
            double acc = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    double F = Ds[a][0] * Bm[0][b] + Ds[a][1] * Bm[1][b] + Ds[a][2] * Bm[2][b];
                    acc += F * F;
                }
            v = w[t] * acc;
        }
    }
    v = block_sum<256>(v, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}
void elastic_partials(const double4 *g, const double4 *dx, const int *q2v, int nf, const int4 *tets,
                      const double *B, const double *w, int T, double *part, int *nb1, int *nb2,
                      cudaStream_t st) {
    *nb1 = (nf + 255) / 256;
    *nb2 = (T + 255) / 256;
    PDI_LAUNCH(k_elastic_partials, *nb1 + *nb2, 256, 0, st)(g, dx, q2v, nf, tets, B, w, T, *nb1, part);
}
void launch_update(double4 *x, const double4 *dx, const int *q2v, int nf, const double *alpha,
                   const int *flags, int *abort, int it, int *cv, unsigned long long *amax, double tol,
                   cudaStream_t st) {
    PDI_LAUNCH(k_update, std::max(1, (nf + 255) / 256), 256, 0, st)(x, dx, q2v, nf, alpha, flags, abort, it, cv, amax, tol);
}
void launch_scatter_dx(const double *z, const int *q2v, int nf, double4 *dx, double *amin, int nseq, int n,
                       int amin_stride, cudaStream_t st) {
    PDI_LAUNCH(k_scatter_dx, dim3((nf + 255) / 256, nseq), 256, 0, st)(z, q2v, nf, dx, amin, n, amin_stride);
}

}  // namespace pdipc
