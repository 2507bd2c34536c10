// Supernodal triangular solves against the prefactorised PD matrix.
//
// "Equation 2 could be effectively solved by forward/backward substitution";
// the contact-reduced global step (BASELINE.json north_star; PAPER.md:240-247 generalised)
// additionally needs the panel V_s = L^{-1} Pi E_S (one sparse RHS per contact vertex).
//
// Forward solve: ONE persistent, sync-free kernel over work items (supernode s, RHS tile).
// Tile 0 of every supernode is the 3-column gradient RHS (w = L^{-1} Pi g-hat, in place);
// panel tiles cover the contact columns active in s (contact vertices in s's subtree, a
// contiguous column range because supernodes are postordered and S is sorted by factor
// position).  Left-looking: an item gathers the updates of its descendants through the
// precomputed segment lists, so there are no value atomics and the result is deterministic.
// Items are dispensed in postorder by an atomic ticket; an item waits (spin on a counter) for
// all items of its child supernodes, which were dispensed earlier -> deadlock-free.
// Backward solve: same scheme in reverse postorder, 3 columns, waiting for the parent.
#include "kernels.h"

#include "dev_common.cuh"

namespace pdipc {

constexpr int kTS_NT = 256;            // threads per CTA
constexpr int kTS_W = 128;             // max supernode width (host caps it)
constexpr int kPT = 32;                // panel tile width
// Safety net: a dependency wait longer than ~2 s (at ~2 GHz) means a scheduling bug; the
// waiting CTA records the fault in ticket[1] and proceeds instead of hanging the GPU.
constexpr long long kSpinLimit = 4000000000LL;

// per-iteration item setup: active column ranges and item counts
__global__ void k_ts_items(const int *__restrict__ sn_c0, const int *__restrict__ sn_fd,
                           const int *__restrict__ sn_parent, int nsn, const int *__restrict__ qS,
                           const int *__restrict__ nS_ptr, int *__restrict__ lo,
                           int *__restrict__ hi, int *__restrict__ cnt, int *__restrict__ rem) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsn) return;
    const int nS = *nS_ptr;
    const int a = sn_fd[s], b = sn_c0[s + 1];
    // lower_bound(qS, a), lower_bound(qS, b)
    int l = 0, r = nS;
    while (l < r) { int m = (l + r) >> 1; if (qS[m] < a) l = m + 1; else r = m; }
    int L0 = l;
    r = nS;
    while (l < r) { int m = (l + r) >> 1; if (qS[m] < b) l = m + 1; else r = m; }
    int H0 = l;
    lo[s] = L0;
    hi[s] = H0;
    int c = 1 + (H0 > L0 ? (H0 - 1) / kPT - L0 / kPT + 1 : 0);
    cnt[s] = c;
    int p = sn_parent[s];
    if (p >= 0) atomicAdd(rem + p, c);
}

struct FwdArgs {
    const int *sn_c0, *sn_rowptr, *sn_rows, *sn_parent;
    const long long *sn_valptr;
    const double *L;
    const int *seg_ptr, *seg_d, *seg_klo, *seg_khi;
    const int *lo, *hi, *item_ptr, *qS;
    int nsn;
    int *rem, *ticket;
    double *G;                         // [nf][4] in: Pi g-hat, out: w
    double *V;                         // [nf][ldv] panel
    int ldv;
};

__device__ __forceinline__ int find_sn(const int *item_ptr, int nsn, int item) {
    int l = 0, r = nsn;            // largest s with item_ptr[s] <= item
    while (r - l > 1) { int m = (l + r) >> 1; if (item_ptr[m] <= item) l = m; else r = m; }
    return l;
}

__global__ void __launch_bounds__(kTS_NT) k_forward_solve(FwdArgs A) {
    __shared__ double X[kTS_W][kPT + 1];
    __shared__ int sh_item;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = kTS_NT / 32;
    const int total = A.item_ptr[A.nsn];
    while (true) {
        if (tid == 0) sh_item = atomicAdd(A.ticket, 1);
        __syncthreads();
        const int item = sh_item;
        __syncthreads();
        if (item >= total) return;
        const int s = find_sn(A.item_ptr, A.nsn, item);
        const int tk = item - A.item_ptr[s];
        if (tid == 0) {
            volatile int *rp = A.rem + s;
            long long t0 = clock64();
            while (*rp > 0) {
                __nanosleep(64);
                if (clock64() - t0 > kSpinLimit) { atomicExch(A.ticket + 1, 1); break; }
            }
            __threadfence();
        }
        __syncthreads();
        const int c0 = A.sn_c0[s], w = A.sn_c0[s + 1] - c0;
        const int r0 = A.sn_rowptr[s], nr = A.sn_rowptr[s + 1] - r0;
        const double *Ls = A.L + A.sn_valptr[s];
        const bool grad = tk == 0;
        double *Y = grad ? A.G : A.V;
        const int ld = grad ? 4 : A.ldv;
        const int ncol = grad ? 4 : kPT;
        int ca = 0, cb = 4, tbase = 0;
        if (!grad) {
            int tile = A.lo[s] / kPT + tk - 1;
            tbase = tile * kPT;
            ca = max(tbase, A.lo[s]);
            cb = min(tbase + kPT, A.hi[s]);
        }
        // ---- init the RHS block
        for (int e = tid; e < w * kPT; e += kTS_NT) {
            int r = e / kPT, c = e % kPT;
            double v = 0.0;
            if (grad) {
                if (c < 4) v = __ldcg(A.G + (size_t)(c0 + r) * 4 + c);
            } else {
                int col = tbase + c;
                if (col >= ca && col < cb && A.qS[col] == c0 + r) v = 1.0;
            }
            X[r][c] = v;
        }
        __syncthreads();
        // ---- gather descendant updates (left-looking)
        for (int sg = A.seg_ptr[s]; sg < A.seg_ptr[s + 1]; ++sg) {
            const int d = A.seg_d[sg], klo = A.seg_klo[sg], khi = A.seg_khi[sg];
            int da = ca, db = cb;
            if (!grad) {
                da = max(ca, A.lo[d]);
                db = min(cb, A.hi[d]);
                if (da >= db) continue;
            }
            const int dc0 = A.sn_c0[d], dw = A.sn_c0[d + 1] - dc0;
            const int dr0 = A.sn_rowptr[d], dnr = A.sn_rowptr[d + 1] - dr0;
            const double *Ld = A.L + A.sn_valptr[d];
            const int col = tbase + lane;
            const bool act = lane < ncol && (grad ? lane < 3 : (col >= da && col < db));
            for (int j2 = klo + wid; j2 < khi; j2 += nw) {
                double acc = 0.0;
                if (act) {
                    const double *y = Y + (size_t)dc0 * ld + (grad ? lane : col);
                    for (int k = 0; k < dw; ++k) acc += Ld[j2 + (size_t)k * dnr] * __ldcg(y + (size_t)k * ld);
                    X[A.sn_rows[dr0 + j2] - c0][lane] -= acc;
                }
            }
            __syncthreads();
        }
        // ---- forward substitution with the diagonal block, 32-row blocks
        for (int kb = 0; kb < w; kb += 32) {
            const int nb = min(32, w - kb);
            if (wid == 0 && lane < ncol) {
                for (int k = 0; k < nb; ++k) {
                    const double *lk = Ls + (size_t)(kb + k) * nr;
                    double xk = X[kb + k][lane] / lk[kb + k];
                    X[kb + k][lane] = xk;
                    for (int i = k + 1; i < nb; ++i) X[kb + i][lane] -= lk[kb + i] * xk;
                }
            }
            __syncthreads();
            for (int e = tid; e < (w - kb - nb) * kPT; e += kTS_NT) {
                int i = kb + nb + e / kPT, c = e % kPT;
                if (c >= ncol) continue;
                double acc = 0.0;
                for (int k = 0; k < nb; ++k) acc += Ls[i + (size_t)(kb + k) * nr] * X[kb + k][c];
                X[i][c] -= acc;
            }
            __syncthreads();
        }
        // ---- write back
        for (int e = tid; e < w * kPT; e += kTS_NT) {
            int r = e / kPT, c = e % kPT;
            if (grad) {
                if (c < 4) A.G[(size_t)(c0 + r) * 4 + c] = X[r][c];
            } else {
                int col = tbase + c;
                if (col >= ca && col < cb) A.V[(size_t)(c0 + r) * A.ldv + col] = X[r][c];
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            int p = A.sn_parent[s];
            if (p >= 0) atomicSub(A.rem + p, 1);
        }
    }
}

struct BwdArgs {
    const int *sn_c0, *sn_rowptr, *sn_rows, *sn_parent;
    const long long *sn_valptr;
    const double *L;
    int nsn;
    int *done, *ticket;
    double *Z;                         // [nf][4] in: rhs, out: solution of L^T x = rhs
};

__global__ void __launch_bounds__(kTS_NT) k_backward_solve(BwdArgs A) {
    __shared__ double X[kTS_W][5];
    __shared__ int sh_item;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    while (true) {
        if (tid == 0) sh_item = atomicAdd(A.ticket, 1);
        __syncthreads();
        const int item = sh_item;
        __syncthreads();
        if (item >= A.nsn) return;
        const int s = A.nsn - 1 - item;
        if (tid == 0) {
            int p = A.sn_parent[s];
            if (p >= 0) {
                volatile int *dp = A.done + p;
                long long t0 = clock64();
                while (*dp == 0) {
                    __nanosleep(64);
                    if (clock64() - t0 > kSpinLimit) { atomicExch(A.ticket + 1, 1); break; }
                }
            }
            __threadfence();
        }
        __syncthreads();
        const int c0 = A.sn_c0[s], w = A.sn_c0[s + 1] - c0;
        const int r0 = A.sn_rowptr[s], nr = A.sn_rowptr[s + 1] - r0;
        const double *Ls = A.L + A.sn_valptr[s];
        // X = rhs - L_off^T x_off
        for (int e = tid; e < w * 4; e += kTS_NT) {
            int k = e >> 2, c = e & 3;
            double acc = 0.0;
            const double *lk = Ls + (size_t)k * nr;
            for (int r = w; r < nr; ++r) acc += lk[r] * __ldcg(A.Z + (size_t)A.sn_rows[r0 + r] * 4 + c);
            X[k][c] = __ldcg(A.Z + (size_t)(c0 + k) * 4 + c) - acc;
        }
        __syncthreads();
        // backward substitution with L_ss^T in 32-row blocks, last block first
        for (int kb = ((w - 1) / 32) * 32; kb >= 0; kb -= 32) {
            const int nb = min(32, w - kb);
            for (int e = tid; e < nb * 4; e += kTS_NT) {
                int k = kb + (e >> 2), c = e & 3;
                double acc = 0.0;
                const double *lk = Ls + (size_t)k * nr;
                for (int i = kb + nb; i < w; ++i) acc += lk[i] * X[i][c];
                X[k][c] -= acc;
            }
            __syncthreads();
            if (wid == 0 && lane < 4) {
                for (int k = nb - 1; k >= 0; --k) {
                    const double *lk = Ls + (size_t)(kb + k) * nr;
                    double acc = X[kb + k][lane];
                    for (int i = k + 1; i < nb; ++i) acc -= lk[kb + i] * X[kb + i][lane];
                    X[kb + k][lane] = acc / lk[kb + k];
                }
            }
            __syncthreads();
        }
        for (int e = tid; e < w * 4; e += kTS_NT) A.Z[(size_t)(c0 + (e >> 2)) * 4 + (e & 3)] = X[e >> 2][e & 3];
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicExch(A.done + s, 1);
    }
}

// y_S[a][i] = -sum_{r in reach(a)} V[r][a] w[r][i]: walk the supernode path from q_a's supernode
__global__ void k_panel_yS(const int *__restrict__ qS, const int *__restrict__ nS_ptr,
                           const int *__restrict__ col2sn, const int *__restrict__ sn_c0,
                           const int *__restrict__ sn_parent, const double *__restrict__ V, int ldv,
                           const double *__restrict__ G, double *__restrict__ yS) {
    const int a = blockIdx.x;
    if (a >= *nS_ptr) return;
    double acc[3] = {0, 0, 0};
    for (int s = col2sn[qS[a]]; s >= 0; s = sn_parent[s]) {
        for (int r = sn_c0[s] + threadIdx.x; r < sn_c0[s + 1]; r += blockDim.x) {
            double v = V[(size_t)r * ldv + a];
            acc[0] += v * G[(size_t)r * 4 + 0];
            acc[1] += v * G[(size_t)r * 4 + 1];
            acc[2] += v * G[(size_t)r * 4 + 2];
        }
    }
    __shared__ double sh[8];
    for (int i = 0; i < 3; ++i) {
        double t = block_sum<256>(acc[i], sh);
        if (threadIdx.x == 0) yS[3 * a + i] = -t;
    }
}

// Z[r][i] = w[r][i] + sum_{a active in sn(r)} V[r][a] t[a][i]
__global__ void k_panel_correct(const int *__restrict__ col2sn, const int *__restrict__ lo,
                                const int *__restrict__ hi, int nf, const double *__restrict__ V,
                                int ldv, const double *__restrict__ G, const double *__restrict__ t,
                                double *__restrict__ Z) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nf) return;
    int s = col2sn[r];
    double z0 = G[(size_t)r * 4 + 0], z1 = G[(size_t)r * 4 + 1], z2 = G[(size_t)r * 4 + 2];
    for (int a = lo[s]; a < hi[s]; ++a) {
        double v = V[(size_t)r * ldv + a];
        z0 += v * t[3 * a + 0];
        z1 += v * t[3 * a + 1];
        z2 += v * t[3 * a + 2];
    }
    Z[(size_t)r * 4 + 0] = z0;
    Z[(size_t)r * 4 + 1] = z1;
    Z[(size_t)r * 4 + 2] = z2;
    Z[(size_t)r * 4 + 3] = 0.0;
}

// K[a][b] = sum over rows r active for both a and b of V[r][a] V[r][b]  (SYRK on the panel;
// K = (L_FF^{-1})_SS).  One CTA per 32x32 lower tile; deterministic.
__global__ void __launch_bounds__(256) k_panel_syrk(const int *__restrict__ sn_c0,
                                                    const int *__restrict__ lo,
                                                    const int *__restrict__ hi, int nsn,
                                                    const double *__restrict__ V, int ldv,
                                                    const int *__restrict__ nS_ptr,
                                                    double *__restrict__ K, int ldk) {
    const int nS = *nS_ptr;
    const int ti = blockIdx.x, tj = blockIdx.y;     // tile row, tile col
    if (tj > ti || ti * 32 >= nS) return;
    const int ia = ti * 32, ja = tj * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 8 row groups of 4 rows
    double acc[4] = {0, 0, 0, 0};
    __shared__ double Va[32][33], Vb[32][33];
    for (int s = 0; s < nsn; ++s) {
        const int l = lo[s], h = hi[s];
        if (h <= l || l >= min(ia + 32, nS) || h <= ia || l >= ja + 32 || h <= ja) continue;
        const int c0 = sn_c0[s], c1 = sn_c0[s + 1];
        for (int rb = c0; rb < c1; rb += 32) {
            const int nrb = min(32, c1 - rb);
            for (int e = threadIdx.x; e < 32 * 32; e += 256) {
                int rr = e >> 5, cc = e & 31;
                int ca = ia + cc, cb = ja + cc;
                double va = 0, vb = 0;
                if (rr < nrb) {
                    if (ca >= l && ca < h && ca < nS) va = V[(size_t)(rb + rr) * ldv + ca];
                    if (cb >= l && cb < h && cb < nS) vb = V[(size_t)(rb + rr) * ldv + cb];
                }
                Va[rr][cc] = va;
                Vb[rr][cc] = vb;
            }
            __syncthreads();
            for (int rr = 0; rr < nrb; ++rr) {
                double b = Vb[rr][tx];
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[k] += Va[rr][ty * 4 + k] * b;
            }
            __syncthreads();
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int a = ia + ty * 4 + k, b = ja + tx;
        if (a < nS && b < nS && b <= a) {
            K[(size_t)a * ldk + b] = acc[k];
            K[(size_t)b * ldk + a] = acc[k];
        }
    }
}

// ------------------------------------------------------------------ host wrappers ---------
void launch_ts_items(const int *sn_c0, const int *sn_fd, const int *sn_parent, int nsn,
                     const int *qS, const int *nS_ptr, int *lo, int *hi, int *cnt, int *rem,
                     cudaStream_t st) {
    cudaMemsetAsync(rem, 0, sizeof(int) * nsn, st);
    k_ts_items<<<(nsn + 255) / 256, 256, 0, st>>>(sn_c0, sn_fd, sn_parent, nsn, qS, nS_ptr, lo,
                                                   hi, cnt, rem);
}

void launch_forward_solve(const DevFactor &F, const int *lo, const int *hi, const int *item_ptr,
                          const int *qS, int *rem, int *ticket, double *G, double *V, int ldv,
                          int nsm, cudaStream_t st) {
    FwdArgs A;
    A.sn_c0 = F.sn_c0; A.sn_rowptr = F.sn_rowptr; A.sn_rows = F.sn_rows; A.sn_parent = F.sn_parent;
    A.sn_valptr = F.sn_valptr; A.L = F.L;
    A.seg_ptr = F.seg_ptr; A.seg_d = F.seg_d; A.seg_klo = F.seg_klo; A.seg_khi = F.seg_khi;
    A.lo = lo; A.hi = hi; A.item_ptr = item_ptr; A.qS = qS; A.nsn = F.nsn;
    A.rem = rem; A.ticket = ticket; A.G = G; A.V = V; A.ldv = ldv;
    cudaMemsetAsync(ticket, 0, sizeof(int), st);
    k_forward_solve<<<nsm * 4, kTS_NT, 0, st>>>(A);
}

void launch_backward_solve(const DevFactor &F, int *done, int *ticket, double *Z, int nsm,
                           cudaStream_t st) {
    BwdArgs A;
    A.sn_c0 = F.sn_c0; A.sn_rowptr = F.sn_rowptr; A.sn_rows = F.sn_rows; A.sn_parent = F.sn_parent;
    A.sn_valptr = F.sn_valptr; A.L = F.L; A.nsn = F.nsn; A.done = done; A.ticket = ticket; A.Z = Z;
    cudaMemsetAsync(ticket, 0, sizeof(int), st);
    cudaMemsetAsync(done, 0, sizeof(int) * F.nsn, st);
    k_backward_solve<<<nsm * 4, kTS_NT, 0, st>>>(A);
}

void launch_panel_yS(const int *qS, const int *nS_ptr, int nS_host, const DevFactor &F,
                     const double *V, int ldv, const double *G, double *yS, cudaStream_t st) {
    if (nS_host > 0)
        k_panel_yS<<<nS_host, 256, 0, st>>>(qS, nS_ptr, F.col2sn, F.sn_c0, F.sn_parent, V, ldv, G, yS);
}

void launch_panel_correct(const DevFactor &F, const int *lo, const int *hi, const double *V,
                          int ldv, const double *G, const double *t, double *Z, cudaStream_t st) {
    k_panel_correct<<<(F.nf + 255) / 256, 256, 0, st>>>(F.col2sn, lo, hi, F.nf, V, ldv, G, t, Z);
}

void launch_panel_syrk(const DevFactor &F, const int *lo, const int *hi, const double *V, int ldv,
                       const int *nS_ptr, int nS_host, double *K, int ldk, cudaStream_t st) {
    if (nS_host <= 0) return;
    int nt = (nS_host + 31) / 32;
    k_panel_syrk<<<dim3(nt, nt), 256, 0, st>>>(F.sn_c0, lo, hi, F.nsn, V, ldv, nS_ptr, K, ldk);
}

}  // namespace pdipc
