// Supernodal triangular solves against the prefactorised PD matrix.
//
// "Equation 2 could be effectively solved by forward/backward substitution";
// the contact-reduced global step (BASELINE.json north_star; PAPER.md:240-247 generalised)
// additionally needs the panel V_s = L^{-1} Pi E_S (one sparse RHS per contact vertex).
//
// Forward solve: ONE persistent, sync-free kernel over work items (supernode s, RHS tile),
// multifrontal style.  Tile 0 of every supernode is the 3-column gradient RHS
// (w = L^{-1} Pi g-hat, in place); panel tiles (32 columns) cover the contact columns active in
// s (contact vertices in s's subtree: a contiguous column range because supernodes are
// postordered and S is sorted by factor position).  An item
//   1. extend-adds its children's update blocks: rows landing on s's columns are subtracted
//      from the right-hand side (children in fixed order: deterministic, no value atomics),
//   2. applies the precomputed inverse of its diagonal block (dense product, no sequential
//      substitution),
//   3. forms its own update block U_s = L_off Y_s + (children's rows landing on s's off rows),
//      consumed by its parent.
// All loads of a phase are independent across threads; dense products stage 32-column slabs
// of D^-1 / L_off in shared memory.  Items are dispensed in postorder by an atomic ticket; an
// item waits for all items of its child supernodes, which hold earlier tickets -> deadlock-free.
// Backward solve: reverse postorder, 3 columns: stage the already-solved ancestor rows, column
// dot products with L_off, then the transposed inverse of the diagonal block.
#include "kernels.h"

#include "dev_common.cuh"

namespace pdipc {

constexpr int kTS_NT = 256;            // threads per CTA
constexpr int kTS_W = 128;             // max supernode width (host caps it)
constexpr int kPT = 32;                // panel tile width
constexpr int kLD = kPT + 1;           // smem row stride
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
    const int *sn_c0, *sn_rowptr, *sn_parent;
    const long long *sn_valptr;
    const double *L;
    const int *uoff, *urel, *ch_ptr, *ch;
    const long long *dinv_ptr;
    const double *dinv;
    const int *lo, *hi, *item_ptr, *qS;
    int nsn;
    int *rem, *ticket;
    double *G;                         // [nf][4] in: Pi g-hat, out: w
    double *V;                         // [nf][ldv] panel
    int ldv;
    double *Ug;                        // [nU][4] gradient update rows
    double *Up;                        // [nU][ldu] panel update rows
    int ldu;
    unsigned long long *trace;         // optional [items][4]: s|tk, dispense, ready, done (ns)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double4 ldcg4(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a = __ldcg(q), b = __ldcg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ int find_sn(const int *item_ptr, int nsn, int item) {
    int l = 0, r = nsn;            // largest s with item_ptr[s] <= item
    while (r - l > 1) { int m = (l + r) >> 1; if (item_ptr[m] <= item) l = m; else r = m; }
    return l;
}

__device__ __forceinline__ void wait_zero(volatile int *p, int *fault) {
    long long t0 = clock64();
    while (*p > 0) {
        __nanosleep(32);
        if (clock64() - t0 > kSpinLimit) { atomicExch(fault, 1); break; }
    }
    __threadfence();
}

__device__ __forceinline__ bool has_tile(int lo, int hi, int tbase) {
    return hi > lo && lo < tbase + kPT && hi > tbase;
}

// Asynchronous global->shared copies (LDGSTS): a thread issues all of its copies before any
// completes, so a staging pass costs about one memory latency instead of one per element.
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// FP64 tensor-core MMA (DMMA): D(8x8) += A(8x4) B(4x8).  tcgen05 has no f64 kind on sm_100a
// (SURVEY App. A.5); mma.sync.m8n8k4.f64 lowers to DMMA.8x8x4.
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// shared-memory row strides (doubles): A operands (staged slabs) use a stride = 4 mod 16,
// B operands / outputs a stride = 8 mod 16, so DMMA fragment loads are conflict-free.
constexpr int kSS = 36;
constexpr int kXS = 40;

// Out[i][n] = sum_k M[i][k] In[k][n] for i < m, n < 8*NCT, k < kdim (k <= i if LOWER), on DMMA.
// M[i][k] at M + i*ldm_row + k*ldm_col; 32-column slabs of M are staged in Sg with cp.async.
// In rows >= kdim must be zero (callers zero them).  Warp w owns the 8x8 tiles t = w + 8j of
// the (ceil(m/8) x NCT) tile grid.
// TRI: 0 full, 1 lower (k <= i), 2 upper (k >= i)
template <int TRI>
__device__ __forceinline__ void stage_slab(const double *M, long long ldm_row, long long ldm_col,
                                           int m, int mr, int kc, int kn, double (*Sg)[kSS]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (ldm_row == 1) {                     // column-major source: coalesce over i
        for (int kk = wid; kk < 32; kk += kTS_NT / 32)
            for (int i = lane; i < mr; i += 32) {
                if (i < m && kk < kn && (TRI == 0 || (TRI == 1 ? kc + kk <= i : kc + kk >= i)))
                    cp_async8(&Sg[i][kk], M + (long long)i + (long long)(kc + kk) * ldm_col);
                else
                    Sg[i][kk] = 0.0;
            }
    } else {                                // row-major source: coalesce over k
        for (int i = wid; i < mr; i += kTS_NT / 32) {
            const int kk = lane;
            if (i < m && kk < kn && (TRI == 0 || (TRI == 1 ? kc + kk <= i : kc + kk >= i)))
                cp_async8(&Sg[i][kk], M + (long long)i * ldm_row + (long long)(kc + kk) * ldm_col);
            else
                Sg[i][kk] = 0.0;
        }
    }
    cp_async_commit();
}

// Sg points at TWO slab buffers (double buffering: chunk c+1 is in flight while chunk c runs).
template <int TRI, int NCT, bool ACC = false>
__device__ __forceinline__ void slab_dmma(const double *M, long long ldm_row, long long ldm_col,
                                          int m, int kdim, const double (*In)[kXS],
                                          double (*Sg)[kSS], double (*Out)[kXS]) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int rt = (m + 7) >> 3, ntiles = rt * NCT, mr = rt * 8;
    constexpr int kMaxT = (kTS_W / 8) * NCT / 8;       // tiles per warp (16*NCT/8)
    double acc[kMaxT][2];
#pragma unroll
    for (int j = 0; j < kMaxT; ++j) acc[j][0] = acc[j][1] = 0.0;
    const int gr = lane >> 2, gc = lane & 3;
    const int nch = (kdim + 31) / 32;
    stage_slab<TRI>(M, ldm_row, ldm_col, m, mr, 0, min(32, kdim), Sg);
    for (int ch = 0; ch < nch; ++ch) {
        const int kc = ch * 32;
        double (*B)[kSS] = Sg + (ch & 1) * kTS_W;
        if (ch + 1 < nch) {
            stage_slab<TRI>(M, ldm_row, ldm_col, m, mr, kc + 32, min(32, kdim - kc - 32),
                              Sg + ((ch + 1) & 1) * kTS_W);
            cp_async_wait_group<1>();
        } else {
            cp_async_wait_group<0>();
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
            for (int j = 0; j < kMaxT; ++j) {
                const int t = wid + 8 * j;
                if (t < ntiles) {
                    const int tr = t / NCT, tc = t % NCT;
                    const double a = B[tr * 8 + gr][ks * 4 + gc];
                    const double b = In[kc + ks * 4 + gc][tc * 8 + gr];
                    dmma884(acc[j][0], acc[j][1], a, b);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < kMaxT; ++j) {
        const int t = wid + 8 * j;
        if (t < ntiles) {
            const int tr = t / NCT, tc = t % NCT;
            const int r = tr * 8 + gr, c = tc * 8 + 2 * gc;
            if (r < m) {
                if (ACC) {
                    Out[r][c] += acc[j][0];
                    Out[r][c + 1] += acc[j][1];
                } else {
                    Out[r][c] = acc[j][0];
                    Out[r][c + 1] = acc[j][1];
                }
            }
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kTS_NT) k_forward_solve(FwdArgs A) {
    extern __shared__ double fsm[];
    double (*X)[kXS] = reinterpret_cast<double (*)[kXS]>(fsm);
    double (*Y)[kXS] = reinterpret_cast<double (*)[kXS]>(fsm + kTS_W * kXS);
    double (*Sg)[kSS] = reinterpret_cast<double (*)[kSS]>(fsm + 2 * kTS_W * kXS);
    __shared__ int sh_item;
    __shared__ int prel[kTS_W];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
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
            if (A.trace) {
                A.trace[4 * (size_t)item] = ((unsigned long long)s << 16) | (unsigned)tk;
                A.trace[4 * (size_t)item + 1] = gtimer();
            }
            wait_zero(A.rem + s, A.ticket + 1);
            if (A.trace) A.trace[4 * (size_t)item + 2] = gtimer();
        }
        __syncthreads();
        const int c0 = A.sn_c0[s], w = A.sn_c0[s + 1] - c0;
        const int nr = A.sn_rowptr[s + 1] - A.sn_rowptr[s], noff = nr - w;
        const double *Ls = A.L + A.sn_valptr[s];
        const double *D = A.dinv + A.dinv_ptr[s];
        const int u0 = A.uoff[s];
        const bool grad = tk == 0;
        int lo_s = 0, hi_s = 0, tbase = 0;
        if (!grad) {
            lo_s = A.lo[s];
            hi_s = A.hi[s];
            tbase = (lo_s / kPT + tk - 1) * kPT;
        }
        const int col = tbase + lane;
        const int ncc = grad ? 3 : 32;
        // ---- 1. right-hand side block (rows >= w zeroed: they feed the DMMA k-padding)
        for (int e = tid; e < kTS_W * 32; e += kTS_NT) {
            const int j = e >> 5, c = e & 31;
            double b = 0.0;
            if (j < w) {
                if (grad) b = c < 3 ? __ldcg(A.G + (size_t)(c0 + j) * 4 + c) : 0.0;
                else {
                    const int cc = tbase + c;
                    b = (cc >= lo_s && cc < hi_s && A.qS[cc] == c0 + j) ? 1.0 : 0.0;
                }
            }
            X[j][c] = b;
        }
        __syncthreads();
        // ---- 2. children's update rows landing on s's columns (extend-add, child by child,
        //         128-row chunks staged with cp.async into Y, which is free until step 3)
        const int cb0 = A.ch_ptr[s], cb1 = A.ch_ptr[s + 1];
        for (int ci = cb0; ci < cb1; ++ci) {
            const int c = A.ch[ci];
            if (!grad && !has_tile(A.lo[c], A.hi[c], tbase)) continue;   // zero contribution
            const int uc = A.uoff[c], nc = A.uoff[c + 1] - uc;
            for (int kb = 0; kb < nc; kb += kTS_W) {
                const int m = min(kTS_W, nc - kb);
                for (int k = wid; k < m; k += kTS_NT / 32) {
                    if (lane < ncc) {
                        const double *src = grad ? A.Ug + (size_t)(uc + kb + k) * 4 + lane
                                                 : A.Up + (size_t)(uc + kb + k) * A.ldu + tbase + lane;
                        cp_async8(&Y[k][lane], src);
                    }
                }
                for (int k = tid; k < m; k += kTS_NT) prel[k] = __ldg(A.urel + uc + kb + k);
                cp_async_wait_all();
                __syncthreads();
                for (int k = wid; k < m; k += kTS_NT / 32) {
                    const int p = prel[k];
                    if (p < w && lane < ncc) X[p][lane] -= Y[k][lane];
                }
                __syncthreads();
            }
        }
        // ---- 3. Y = Dinv X  (D row-major w x w, lower).  Panel: DMMA on staged slabs.
        //         Gradient (3 columns, no reuse to exploit): thread per row straight from L2,
        //         all loads independent.
        if (grad) slab_dmma<1, 1>(D, w, 1, w, w, X, Sg, Y);
        else slab_dmma<1, 4>(D, w, 1, w, w, X, Sg, Y);
        for (int e = tid; e < kTS_W * 32; e += kTS_NT) {
            const int i = e >> 5, c = e & 31;
            if (i >= w) { Y[i][c] = 0.0; continue; }        // k-padding of step 4
            if (grad) {
                if (c < 3) A.G[(size_t)(c0 + i) * 4 + c] = Y[i][c];
            } else {
                const int cc = tbase + c;
                if (cc >= lo_s && cc < hi_s) A.V[(size_t)(c0 + i) * A.ldv + cc] = Y[i][c];
            }
        }
        __syncthreads();
        // ---- 4. U_s = L_off Y  (L column-major, ld nr) on DMMA, 128-row blocks through X
        if (grad) {
            for (int rb = 0; rb < noff; rb += kTS_W) {
                const int m = min(kTS_W, noff - rb);
                slab_dmma<0, 1>(Ls + w + rb, 1, nr, m, w, Y, Sg, X);
                for (int e = tid; e < m * 4; e += kTS_NT) {
                    const int r = e >> 2, c = e & 3;
                    A.Ug[(size_t)(u0 + rb + r) * 4 + c] = c < 3 ? X[r][c] : 0.0;
                }
                __syncthreads();
            }
        } else {
            for (int rb = 0; rb < noff; rb += kTS_W) {
                const int m = min(kTS_W, noff - rb);
                slab_dmma<0, 4>(Ls + w + rb, 1, nr, m, w, Y, Sg, X);
                for (int e = tid; e < m * 32; e += kTS_NT) {
                    const int r = e >> 5, c = e & 31;
                    A.Up[(size_t)(u0 + rb + r) * A.ldu + tbase + c] = X[r][c];
                }
                __syncthreads();
            }
        }
        // ---- 5. + children's update rows landing on s's off rows (block-private RMW; the
        //         child rows are staged in X; 16 loads batched per thread)
        for (int ci = cb0; ci < cb1; ++ci) {
            const int c = A.ch[ci];
            if (!grad && !has_tile(A.lo[c], A.hi[c], tbase)) continue;
            const int uc = A.uoff[c], nc = A.uoff[c + 1] - uc;
            for (int kb = 0; kb < nc; kb += kTS_W) {
                const int m = min(kTS_W, nc - kb);
                for (int k = wid; k < m; k += kTS_NT / 32) {
                    if (lane < ncc) {
                        const double *src = grad ? A.Ug + (size_t)(uc + kb + k) * 4 + lane
                                                 : A.Up + (size_t)(uc + kb + k) * A.ldu + tbase + lane;
                        cp_async8(&X[k][lane], src);
                    }
                }
                for (int k = tid; k < m; k += kTS_NT) prel[k] = __ldg(A.urel + uc + kb + k);
                cp_async_wait_all();
                __syncthreads();
                double cur[kTS_W / 8];
                double *dst[kTS_W / 8];
#pragma unroll
                for (int q = 0; q < kTS_W / 8; ++q) {
                    const int k = wid + 8 * q;
                    dst[q] = nullptr;
                    cur[q] = 0.0;
                    if (k < m && lane < ncc) {
                        const int p = prel[k];
                        if (p >= w) {
                            dst[q] = grad ? A.Ug + (size_t)(u0 + p - w) * 4 + lane
                                          : A.Up + (size_t)(u0 + p - w) * A.ldu + tbase + lane;
                            cur[q] = __ldcg(dst[q]);
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < kTS_W / 8; ++q)
                    if (dst[q]) *dst[q] = cur[q] + X[wid + 8 * q][lane];
                __syncthreads();
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            int p = A.sn_parent[s];
            if (p >= 0) atomicSub(A.rem + p, 1);
            if (A.trace) A.trace[4 * (size_t)item + 3] = gtimer();
        }
    }
}

struct BwdArgs {
    const int *sn_c0, *sn_rowptr, *sn_rows, *sn_parent;
    const long long *sn_valptr;
    const double *L;
    const long long *dinv_ptr;
    const double *dinv;
    int nsn;
    int *done, *ticket;
    double *Z;                         // [nf][4] in: rhs, out: solution of L^T x = rhs
};

constexpr int kBwdStage = 256;

__global__ void __launch_bounds__(kTS_NT) k_backward_solve_v1(BwdArgs A) {
    __shared__ double X[kTS_W][4];
    __shared__ double4 xo[kBwdStage];
    __shared__ double Sg[32][kTS_W + 1];
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
                    __nanosleep(32);
                    if (clock64() - t0 > kSpinLimit) { atomicExch(A.ticket + 1, 1); break; }
                }
            }
            __threadfence();
        }
        __syncthreads();
        const int c0 = A.sn_c0[s], w = A.sn_c0[s + 1] - c0;
        const int r0 = A.sn_rowptr[s], nr = A.sn_rowptr[s + 1] - r0, noff = nr - w;
        const double *Ls = A.L + A.sn_valptr[s];
        const double *D = A.dinv + A.dinv_ptr[s];
        const double4 *Z4 = reinterpret_cast<const double4 *>(A.Z);
        for (int k = tid; k < w; k += kTS_NT) {
            const double4 z = ldcg4(Z4 + c0 + k);
            X[k][0] = z.x;
            X[k][1] = z.y;
            X[k][2] = z.z;
        }
        // X[k] -= sum_r L[r][k] x[R(r)]: stage the solved ancestor rows, then warp per k
        for (int rb = 0; rb < noff; rb += kBwdStage) {
            const int m = min(kBwdStage, noff - rb);
            for (int r = tid; r < m; r += kTS_NT) xo[r] = ldcg4(Z4 + A.sn_rows[r0 + w + rb + r]);
            __syncthreads();
            for (int k = wid; k < w; k += kTS_NT / 32) {
                const double *lk = Ls + (size_t)k * nr + w + rb;
                double a0 = 0, a1 = 0, a2 = 0;
                for (int r = lane; r < m; r += 32) {
                    const double l = lk[r];
                    const double4 xv = xo[r];
                    a0 += l * xv.x;
                    a1 += l * xv.y;
                    a2 += l * xv.z;
                }
                a0 = warp_sum(a0);
                a1 = warp_sum(a1);
                a2 = warp_sum(a2);
                if (lane == 0) {
                    X[k][0] -= a0;
                    X[k][1] -= a1;
                    X[k][2] -= a2;
                }
            }
            __syncthreads();
        }
        __syncthreads();
        // x_s[i] = sum_{k >= i} D[k][i] X[k]: thread per i, column i of D read straight from
        // L2 (coalesced across threads), loads independent
        double a[3] = {0, 0, 0};
        if (tid < w) {
            const int i = tid;
#pragma unroll 8
            for (int k = i; k < w; ++k) {
                const double dv = __ldg(D + (size_t)k * w + i);
                a[0] += dv * X[k][0];
                a[1] += dv * X[k][1];
                a[2] += dv * X[k][2];
            }
        }
        if (tid < w) {
            double *zr = A.Z + (size_t)(c0 + tid) * 4;
            zr[0] = a[0];
            zr[1] = a[1];
            zr[2] = a[2];
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicExch(A.done + s, 1);
    }
}

// Backward solve item s (reverse postorder, waits for its parent):
//   X = z_s - L_off^T x_off    (DMMA over 128-row chunks of the solved ancestor rows x_off)
//   x_s = Dinv^T X             (DMMA, upper-triangular slab staging)
__global__ void __launch_bounds__(kTS_NT) k_backward_solve(BwdArgs A) {
    extern __shared__ double bsm[];
    double (*X)[kXS] = reinterpret_cast<double (*)[kXS]>(bsm);
    double (*Y)[kXS] = reinterpret_cast<double (*)[kXS]>(bsm + kTS_W * kXS);
    double (*Sg)[kSS] = reinterpret_cast<double (*)[kSS]>(bsm + 2 * kTS_W * kXS);
    __shared__ int sh_item;
    const int tid = threadIdx.x;
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
                    __nanosleep(32);
                    if (clock64() - t0 > kSpinLimit) { atomicExch(A.ticket + 1, 1); break; }
                }
            }
            __threadfence();
        }
        __syncthreads();
        const int c0 = A.sn_c0[s], w = A.sn_c0[s + 1] - c0;
        const int r0 = A.sn_rowptr[s], nr = A.sn_rowptr[s + 1] - r0, noff = nr - w;
        const double *Ls = A.L + A.sn_valptr[s];
        const double *D = A.dinv + A.dinv_ptr[s];
        // ---- acc = L_off^T x_off, chunks of 128 off rows staged in Y (cols >= 3 and padding 0)
        for (int rb = 0; rb < noff; rb += kTS_W) {
            const int m = min(kTS_W, noff - rb);
            for (int e = tid; e < kTS_W * 8; e += kTS_NT) {
                const int r = e >> 3, c = e & 7;
                Y[r][c] = (r < m && c < 3) ? __ldcg(A.Z + (size_t)A.sn_rows[r0 + w + rb + r] * 4 + c) : 0.0;
            }
            __syncthreads();
            if (rb == 0) slab_dmma<0, 1, false>(Ls + w + rb, nr, 1, w, m, Y, Sg, X);
            else slab_dmma<0, 1, true>(Ls + w + rb, nr, 1, w, m, Y, Sg, X);
        }
        // ---- X = z_s - acc (rows >= w and columns >= 3 zeroed: k-padding of the next product)
        for (int e = tid; e < kTS_W * 8; e += kTS_NT) {
            const int k = e >> 3, c = e & 7;
            double v = 0.0;
            if (k < w && c < 3) v = __ldcg(A.Z + (size_t)(c0 + k) * 4 + c) - (noff > 0 ? X[k][c] : 0.0);
            Y[k][c] = v;
        }
        __syncthreads();
        // ---- x_s = Dinv^T X : element (i, k) = D[k][i] (column-major source, upper triangle)
        slab_dmma<2, 1, false>(D, 1, w, w, w, Y, Sg, X);
        for (int e = tid; e < w * 3; e += kTS_NT) {
            const int i = e / 3, c = e % 3;
            A.Z[(size_t)(c0 + i) * 4 + c] = X[i][c];
        }
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
constexpr int kFwdSmem = (2 * kTS_W * kXS + 2 * kTS_W * kSS) * (int)sizeof(double);

void trisolve_init() {
    cudaFuncSetAttribute(k_forward_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
    cudaFuncSetAttribute(k_backward_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
}

void launch_ts_items(const int *sn_c0, const int *sn_fd, const int *sn_parent, int nsn,
                     const int *qS, const int *nS_ptr, int *lo, int *hi, int *cnt, int *rem,
                     cudaStream_t st) {
    cudaMemsetAsync(rem, 0, sizeof(int) * nsn, st);
    PDI_LAUNCH(k_ts_items, (nsn + 255) / 256, 256, 0, st)(sn_c0, sn_fd, sn_parent, nsn, qS, nS_ptr,
                                                           lo, hi, cnt, rem);
}

void launch_forward_solve(const DevFactor &F, const int *lo, const int *hi, const int *item_ptr,
                          const int *qS, int *rem, int *ticket, double *G, double *V, int ldv,
                          double *Ug, double *Up, int ldu, int nsm, unsigned long long *trace,
                          cudaStream_t st) {
    FwdArgs A;
    A.sn_c0 = F.sn_c0; A.sn_rowptr = F.sn_rowptr; A.sn_parent = F.sn_parent;
    A.sn_valptr = F.sn_valptr; A.L = F.L;
    A.uoff = F.uoff; A.urel = F.urel; A.ch_ptr = F.ch_ptr; A.ch = F.ch;
    A.dinv_ptr = F.dinv_ptr; A.dinv = F.dinv;
    A.lo = lo; A.hi = hi; A.item_ptr = item_ptr; A.qS = qS; A.nsn = F.nsn;
    A.rem = rem; A.ticket = ticket; A.G = G; A.V = V; A.ldv = ldv; A.Ug = Ug; A.Up = Up; A.ldu = ldu;
    A.trace = trace;
    cudaMemsetAsync(ticket, 0, sizeof(int), st);
    PDI_LAUNCH(k_forward_solve, nsm, kTS_NT, kFwdSmem, st)(A);
}

void launch_backward_solve(const DevFactor &F, int *done, int *ticket, double *Z, int nsm,
                           cudaStream_t st) {
    BwdArgs A;
    A.sn_c0 = F.sn_c0; A.sn_rowptr = F.sn_rowptr; A.sn_rows = F.sn_rows; A.sn_parent = F.sn_parent;
    A.sn_valptr = F.sn_valptr; A.L = F.L; A.dinv_ptr = F.dinv_ptr; A.dinv = F.dinv;
    A.nsn = F.nsn; A.done = done; A.ticket = ticket; A.Z = Z;
    cudaMemsetAsync(ticket, 0, sizeof(int), st);
    cudaMemsetAsync(done, 0, sizeof(int) * F.nsn, st);
    PDI_LAUNCH(k_backward_solve, nsm, kTS_NT, kFwdSmem, st)(A);
}

void launch_panel_yS(const int *qS, const int *nS_ptr, int nS_host, const DevFactor &F,
                     const double *V, int ldv, const double *G, double *yS, cudaStream_t st) {
    if (nS_host > 0)
        PDI_LAUNCH(k_panel_yS, nS_host, 256, 0, st)(qS, nS_ptr, F.col2sn, F.sn_c0, F.sn_parent, V,
                                                    ldv, G, yS);
}

void launch_panel_correct(const DevFactor &F, const int *lo, const int *hi, const double *V,
                          int ldv, const double *G, const double *t, double *Z, cudaStream_t st) {
    PDI_LAUNCH(k_panel_correct, (F.nf + 255) / 256, 256, 0, st)(F.col2sn, lo, hi, F.nf, V, ldv, G,
                                                                 t, Z);
}

void launch_panel_syrk(const DevFactor &F, const int *lo, const int *hi, const double *V, int ldv,
                       const int *nS_ptr, int nS_host, double *K, int ldk, cudaStream_t st) {
    if (nS_host <= 0) return;
    int nt = (nS_host + 31) / 32;
    PDI_LAUNCH(k_panel_syrk, dim3(nt, nt), 256, 0, st)(F.sn_c0, lo, hi, F.nsn, V, ldv, nS_ptr, K, ldk);
}

}  // namespace pdipc
