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
#include "prims.h"

#include "dev_common.cuh"

namespace pdipc {

constexpr int kTS_NT = 256;            // threads per CTA
constexpr int kTS_W = 128;             // max supernode width (host caps it)
constexpr int kPT = 32;                // panel tile width
// Safety net: a dependency wait longer than ~2 s (at ~2 GHz) means a scheduling bug; the
// waiting CTA records the fault in ticket[1] and proceeds instead of hanging the GPU.
constexpr long long kSpinLimit = 4000000000LL;

// per-iteration item setup: active column ranges and item counts (row blocks x (1 + tiles)) of
// the supernode at dispatch position k; adds the count to the parent's dependency counter
__device__ __forceinline__ int ts_item_count(int k, const int *__restrict__ ford, const int *__restrict__ sn_c0,
                                             const int *__restrict__ sn_rowptr, const int *__restrict__ sn_fd,
                                             const int *__restrict__ sn_parent, const int *__restrict__ qS,
                                             const int *__restrict__ nS_ptr, int capS,
                                             const int *__restrict__ same_S, int nU, long long up_cap,
                                             int *__restrict__ flags, int mode, int ngt, int *__restrict__ lo,
                                             int *__restrict__ hi, int *__restrict__ rem) {
    const int s = ford[k];
    const int nb = (sn_rowptr[s + 1] - sn_rowptr[s] + kSolveRB - 1) / kSolveRB;
    if (!(mode & 2)) {                     // gradient items only: no contact data read at all
        lo[s] = hi[s] = 0;
        const int p = sn_parent[s];
        if (p >= 0) atomicAdd(rem + p, nb * ngt);
        return nb * ngt;
    }
    const int nS = min(*nS_ptr, capS);
    // panel update rows need nU x round32(|S|) doubles; otherwise flag bit 4 (grow and redo)
    const bool up_ok = (long long)nU * (((nS + 31) / 32) * 32) <= up_cap;
    if (!up_ok && k == 0) atomicOr(flags, 4);
    const int a = sn_fd[s], b = sn_c0[s + 1];
    int l = 0, r = nS;
    while (l < r) { int m = (l + r) >> 1; if (qS[m] < a) l = m + 1; else r = m; }
    int L0 = l;
    r = nS;
    while (l < r) { int m = (l + r) >> 1; if (qS[m] < b) l = m + 1; else r = m; }
    int H0 = l;
    lo[s] = L0;
    hi[s] = H0;
    // panel tiles only when V_s must be recomputed (S changed)
    const int tiles = (up_ok && *same_S == 0 && H0 > L0) ? (H0 - 1) / kPT - L0 / kPT + 1 : 0;
    const int c = nb * ((mode & 1) ? ngt + tiles : tiles);
    const int p = sn_parent[s];
    if (p >= 0) atomicAdd(rem + p, c);
    return c;
}

// The whole per-iteration plan of a solve in ONE block: dependency counters and the item
// dispenser cleared, item counts and column ranges of every supernode, and their exclusive scan
// item_ptr[0..nsn] (replaces a clear, the count kernel and a two-pass scan).
constexpr int kPlanNT = 1024;
__global__ void __launch_bounds__(kPlanNT) k_ts_plan(const int *__restrict__ ford, const int *__restrict__ sn_c0,
                                                     const int *__restrict__ sn_rowptr, const int *__restrict__ sn_fd,
                                                     const int *__restrict__ sn_parent, int nsn,
                                                     const int *__restrict__ qS, const int *__restrict__ nS_ptr,
                                                     int capS, const int *__restrict__ same_S, int nU,
                                                     long long up_cap, int *__restrict__ flags, int mode,
                                                     int ngt, int *__restrict__ lo, int *__restrict__ hi,
                                                     int *__restrict__ cnt, int *__restrict__ rem,
                                                     int *__restrict__ item_ptr, int *__restrict__ ticket) {
    __shared__ int wsum[kPlanNT / 32];
    __shared__ int carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < nsn; i += kPlanNT) rem[i] = 0;
    if (tid == 0) {
        ticket[0] = 0;
        carry = 0;
    }
    __syncthreads();
    for (int k = tid; k < nsn; k += kPlanNT)
        cnt[k] = ts_item_count(k, ford, sn_c0, sn_rowptr, sn_fd, sn_parent, qS, nS_ptr, capS, same_S, nU, up_cap,
                               flags, mode, ngt, lo, hi, rem);
    __syncthreads();
    for (int k0 = 0; k0 <= nsn; k0 += kPlanNT) {          // exclusive scan, item_ptr[nsn] = total
        const int k = k0 + tid;
        const int v = k < nsn ? cnt[k] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int t = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            wsum[lane] = t;
        }
        __syncthreads();
        const int ex = carry + (wid > 0 ? wsum[wid - 1] : 0) + x - v;
        if (k <= nsn) item_ptr[k] = ex;
        __syncthreads();
        if (tid == 0) carry += wsum[kPlanNT / 32 - 1];
        __syncthreads();
    }
}

struct FwdArgs {
    const int *sn_c0, *sn_rowptr, *sn_parent, *uoff, *rc_ptr;
    const int2 *rc_src;
    const long long *sn_valptr;
    const double *Q;
    const int *lo, *hi, *item_ptr, *qS, *ford;
    int nsn;
    int *rem, *ticket;
    const double *G;                   // [nseq][nf][4] Pi g (sequence stride gstride doubles)
    double *Y;                         // [nseq][nf][4] out: w = L^{-1} Pi g (+ Yadd)
    const double *Yadd;                // nullable [nseq][nf][4] added to the solution rows
    double *V;                         // [nf][ldv] panel
    int ldv;
    double *Ug;                        // [nseq][nU][4] gradient update rows (stride ustride)
    long long gstride, ustride;
    int nseq;                          // gradient right-hand sides: 3 columns per sequence
    int ngt, gw;                       // gradient tiles per row block, columns per tile (8 | 32)
    double *Up;                        // [nU][ldu] panel update rows, ldu = round32(|S|)
    const int *nS_ptr;
    int capS;
    int with_grad;                     // 0: panel tiles only (item tile index starts at 1)
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

constexpr int kSgRows = 256;
constexpr int kItemPtrSh = 4096;      // item_ptr entries cached in shared memory
constexpr int kMaxSrc = 4;             // cached extend-add sources per row (more: list walk)           // staged A-operand rows (all k-slabs of one block)

// Issue (without waiting) the cp.async copies of A = M[0..m) x [0..kdim) into Sg as
// ceil(kdim/32) slabs of round8(m) rows; out-of-range entries are zeroed.
// M[i][k] at M + i*ldm_row + k*ldm_col.  Requires ceil(kdim/32) * round8(m) <= kSgRows.
__device__ __forceinline__ void stage_block(const double *M, long long ldm_row, long long ldm_col,
                                            int m, int kdim, double (*Sg)[kSS]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int mr = (m + 7) & ~7, nch = (kdim + 31) >> 5;
    for (int ch = 0; ch < nch; ++ch) {
        double (*S)[kSS] = Sg + ch * mr;
        const int kc = ch * 32;
        if (ldm_row == 1) {                 // column-major source: coalesce over i
            for (int kk = wid; kk < 32; kk += kTS_NT / 32)
                for (int i = lane; i < mr; i += 32) {
                    if (i < m && kc + kk < kdim)
                        cp_async8(&S[i][kk], M + (long long)i + (long long)(kc + kk) * ldm_col);
                    else
                        S[i][kk] = 0.0;
                }
        } else {                            // row-major source: coalesce over k
            for (int i = wid; i < mr; i += kTS_NT / 32) {
                if (i < m && kc + lane < kdim)
                    cp_async8(&S[i][lane], M + (long long)i * ldm_row + (long long)(kc + lane) * ldm_col);
                else
                    S[i][lane] = 0.0;
            }
        }
    }
    cp_async_commit();
}

// Out[i][n] = sum_k A[i][k] In[k][n] (i < m, n < 8*NCT) on DMMA from the staged block; In rows
// in [kdim, 32*ceil(kdim/32)) must be zero.  Warp w owns 8x8 tiles t = w + 8j.  Caller has
// waited for the staging and synchronised.
template <int NCT, int MAXRT>
__device__ __forceinline__ void block_dmma(int m, int kdim, const double (*Sg)[kSS],
                                           const double (*In)[kXS], double (*Out)[kXS]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int rt = (m + 7) >> 3, ntiles = rt * NCT, mr = rt * 8, nch = (kdim + 31) >> 5;
    constexpr int kMaxT = (MAXRT * NCT + 7) / 8;
    double acc[kMaxT][2];
#pragma unroll
    for (int j = 0; j < kMaxT; ++j) acc[j][0] = acc[j][1] = 0.0;
    const int gr = lane >> 2, gc = lane & 3;
    for (int ch = 0; ch < nch; ++ch) {
        const double (*S)[kSS] = Sg + ch * mr;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
            for (int j = 0; j < kMaxT; ++j) {
                const int t = wid + 8 * j;
                if (t < ntiles) {
                    const int tr = t / NCT, tc = t % NCT;
                    dmma884(acc[j][0], acc[j][1], S[tr * 8 + gr][ks * 4 + gc],
                            In[ch * 32 + ks * 4 + gc][tc * 8 + gr]);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kMaxT; ++j) {
        const int t = wid + 8 * j;
        if (t < ntiles) {
            const int tr = t / NCT, tc = t % NCT;
            const int r = tr * 8 + gr, c = tc * 8 + 2 * gc;
            if (r < m) {
                Out[r][c] = acc[j][0];
                Out[r][c + 1] = acc[j][1];
            }
        }
    }
}

// Forward solve.  Item (s, tile tk, row block b): tk = 0 is the 3-column gradient RHS, tk >= 1
// the 32-column panel tiles active in s; rows [64b, 64b + 64) of s's row list R_s.
//   X   = rhs_s - (children's update rows landing on s's columns)      (w x ncols, gathered)
//   O   = Q_s[rows] X                                                   (DMMA)
//   rows < w:  the solution rows of s (w = L^{-1} Pi g, or V);
//   rows >= w: U_s rows = O + children's update rows landing there (consumed by the parent).
// Every item of s depends only on s's children (Q_s folds L_ss^{-1} into the off-diagonal
// block), so the row blocks of one supernode run on different SMs at the same time.
__global__ void __launch_bounds__(kTS_NT) k_forward_solve(FwdArgs A) {
    extern __shared__ double fsm[];
    double (*X)[kXS] = reinterpret_cast<double (*)[kXS]>(fsm);
    double (*O)[kXS] = reinterpret_cast<double (*)[kXS]>(fsm + kTS_W * kXS);
    double (*Sg)[kSS] = reinterpret_cast<double (*)[kSS]>(fsm + (kTS_W + kSolveRB) * kXS);
    __shared__ int sh_item;
    __shared__ int src_n[kTS_W + kSolveRB], src_u[kTS_W + kSolveRB][kMaxSrc];
    __shared__ int ip_sh[kItemPtrSh];                   // item_ptr cached (small factors)
    const int tid = threadIdx.x;
    const bool ip_cached = A.nsn + 1 <= kItemPtrSh;
    if (ip_cached)
        for (int i = tid; i <= A.nsn; i += kTS_NT) ip_sh[i] = A.item_ptr[i];
    const int *item_ptr = ip_cached ? ip_sh : A.item_ptr;
    const int total = A.item_ptr[A.nsn];
    const int ldu = ((min(*A.nS_ptr, A.capS) + 31) / 32) * 32;
    while (true) {
        if (tid == 0) sh_item = atomicAdd(A.ticket, 1);
        __syncthreads();
        const int item = sh_item;
        __syncthreads();
        if (item >= total) return;
        const int kpos = find_sn(item_ptr, A.nsn, item), s = A.ford[kpos];
        const int c0 = A.sn_c0[s], w = A.sn_c0[s + 1] - c0;
        const int slot0 = A.sn_rowptr[s], nr = A.sn_rowptr[s + 1] - slot0;
        const int nb = (nr + kSolveRB - 1) / kSolveRB;
        const int idx = item - item_ptr[kpos], tk = idx / nb;
        const int rb = (idx % nb) * kSolveRB;
        const int m = min(kSolveRB, nr - rb);
        const int ngt = A.with_grad ? A.ngt : 0;
        // tiles 0 .. ngt-1: gradient right-hand sides, gw columns = gw/4 sequences x (xyz + pad);
        // tiles >= ngt: the 32-column panel tiles active in s
        const bool grad = tk < ngt;
        const int gseq0 = grad ? tk * (A.gw >> 2) : 0;
        int lo_s = 0, hi_s = 0, tbase = 0;
        if (!grad) {
            lo_s = A.lo[s];
            hi_s = A.hi[s];
            tbase = (lo_s / kPT + tk - ngt) * kPT;
        }
        const int ncc = grad ? A.gw : 32;
        // Q block rows in flight while we wait for the children and gather the RHS
        stage_block(A.Q + A.sn_valptr[s] + rb, 1, nr, m, w, Sg);
        // ---- extend-add sources of the rows this item touches (static structure: resolved
        //      while the children may still be running): list slot q < w is column row
        //      q (for X), slot w + i is row rb + i (epilogue, off rows only).  Resolved once,
        //      thread per row, so the value gathers below are independent loads.
        // update-row element (row, column c of this tile): gradient rows are per sequence
        auto uelem = [&](int row, int c) -> size_t {
            return grad ? (size_t)(gseq0 + (c >> 2)) * A.ustride + (size_t)row * 4 + (c & 3)
                        : (size_t)row * ldu + tbase + c;
        };
        for (int q = tid; q < w + m; q += kTS_NT) {
            const int row = q < w ? q : rb + q - w;
            int cnt = 0;
            if (q < w || row >= w) {
                const int j0 = A.rc_ptr[slot0 + row], j1 = A.rc_ptr[slot0 + row + 1];
                for (int jb = j0; jb < j1; jb += 4) {
                    int2 sr[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) sr[k] = jb + k < j1 ? A.rc_src[jb + k] : make_int2(-1, -1);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (sr[k].x < 0) continue;
                        if (grad || has_tile(A.lo[sr[k].y], A.hi[sr[k].y], tbase)) {
                            if (cnt < kMaxSrc) src_u[q][cnt] = sr[k].x;
                            ++cnt;
                        }
                    }
                }
            }
            src_n[q] = cnt;
        }
        if (tid == 0) {
            if (A.trace) {
                A.trace[4 * (size_t)item] = ((unsigned long long)s << 16) | (unsigned)tk;
                A.trace[4 * (size_t)item + 1] = gtimer();
            }
            wait_zero(A.rem + s, A.ticket + 1);
            if (A.trace) A.trace[4 * (size_t)item + 2] = gtimer();
        }
        __syncthreads();
        // ---- X: rhs minus the children's rows landing on s's columns (fixed child order)
        const int kpad = (w + 31) & ~31, ncw = ncc, lg = ncw == 8 ? 3 : 5;
        for (int e0 = 0; e0 < kpad * ncw; e0 += 4 * kTS_NT) {
            double v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int e = e0 + k * kTS_NT + tid, p = e >> lg, c = e & (ncw - 1);
                v[k] = 0.0;
                const bool live = !grad || gseq0 + (c >> 2) < A.nseq;
                if (p < w && c < ncc && live) {
                    if (grad) v[k] = __ldcg(A.G + (size_t)(gseq0 + (c >> 2)) * A.gstride + (size_t)(c0 + p) * 4 + (c & 3));
                    else {
                        const int cc = tbase + c;
                        v[k] = (cc >= lo_s && cc < hi_s && A.qS[cc] == c0 + p) ? 1.0 : 0.0;
                    }
                    const int n = src_n[p];
#pragma unroll
                    for (int t = 0; t < kMaxSrc; ++t)
                        if (t < n) v[k] -= __ldcg((grad ? A.Ug : A.Up) + uelem(src_u[p][t], c));
                    if (n > kMaxSrc) {   // rare: more sources than cached, walk the list
                        int t = 0;
                        for (int j = A.rc_ptr[slot0 + p]; j < A.rc_ptr[slot0 + p + 1]; ++j) {
                            const int2 sr = A.rc_src[j];
                            if (grad || has_tile(A.lo[sr.y], A.hi[sr.y], tbase)) {
                                if (t >= kMaxSrc) v[k] -= __ldcg((grad ? A.Ug : A.Up) + uelem(sr.x, c));
                                ++t;
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int e = e0 + k * kTS_NT + tid, p = e >> lg, c = e & (ncw - 1);
                if (p < kpad) X[p][c] = v[k];
            }
        }
        cp_async_wait_group<0>();
        __syncthreads();
        if (ncw == 8) block_dmma<1, kSolveRB / 8>(m, w, Sg, X, O);
        else block_dmma<4, kSolveRB / 8>(m, w, Sg, X, O);
        __syncthreads();
        // ---- epilogue: solution rows, or U rows = O + children's rows landing there
        for (int e0 = 0; e0 < m * ncw; e0 += 4 * kTS_NT) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int e = e0 + k * kTS_NT + tid, i = e >> lg, c = e & (ncw - 1), r = rb + i;
                if (i >= m || c >= ncw || (grad && gseq0 + (c >> 2) >= A.nseq)) continue;
                if (r < w) {
                    if (grad) {
                        const size_t yi = (size_t)(gseq0 + (c >> 2)) * A.gstride + (size_t)(c0 + r) * 4 + (c & 3);
                        A.Y[yi] = (c & 3) < 3 ? O[i][c] + (A.Yadd ? __ldcg(A.Yadd + yi) : 0.0) : 0.0;
                    }
                    else {
                        const int cc = tbase + c;
                        if (cc >= lo_s && cc < hi_s) A.V[(size_t)(c0 + r) * A.ldv + cc] = O[i][c];
                    }
                    continue;
                }
                double u = O[i][c];
                const int q = w + i, n = src_n[q];
                const double *Usrc = grad ? A.Ug : A.Up;
#pragma unroll
                for (int t = 0; t < kMaxSrc; ++t)
                    if (t < n) u += __ldcg(Usrc + uelem(src_u[q][t], c));
                if (n > kMaxSrc) {
                    int t = 0;
                    for (int j = A.rc_ptr[slot0 + r]; j < A.rc_ptr[slot0 + r + 1]; ++j) {
                        const int2 sr = A.rc_src[j];
                        if (grad || has_tile(A.lo[sr.y], A.hi[sr.y], tbase)) {
                            if (t >= kMaxSrc) u += __ldcg(Usrc + uelem(sr.x, c));
                            ++t;
                        }
                    }
                }
                (grad ? A.Ug : A.Up)[uelem(A.uoff[s] + r - w, c)] = u;
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
    const double *Q;
    const int2 *items;                 // [nitems] (s, row block) in reverse postorder
    const int *pbase;                  // [nsn] first partial block of s
    int nitems;
    int *done, *cnt, *ticket;
    double *P;                         // [blocks][kTS_W][kBwCols] partial sums
    double *Z;                         // [nseq][nf][4] in: rhs, out: solution of L^T x = rhs
    long long zstride;                 // sequence stride of Z (doubles)
    int nseq;                          // right-hand sides: 3 columns per sequence, nseq <= 8 ntile
    int ntile;                         // column tiles of 8 sequences: items (s, row block, tile)
    int nsn;                           // done / cnt stride per tile
    long long pstride;                 // P stride per tile (doubles)
};
constexpr int kBwCols = 32;            // columns of one backward-solve launch (8 sequences)

// Backward solve.  x_s = L_ss^{-T}(z_s - L_off^T x_R) = Q_s^T [z_s; -x_R].  Item (s, b, tile)
// forms the partial Q_s[rows]^T v[rows] of its 64-row block for the tile's 8 sequences (DMMA);
// the last block of (s, tile) to finish sums the partials in block order (deterministic) and
// publishes x_s.  Items of (s, tile) wait for (parent, tile) (all of R_s's rows are solved by
// then).  The tiles of one (s, b) are dispensed back to back (the Q block is re-read from L2), so
// one launch covers every sequence of a batch and pays the etree's dependency depth once; each
// tile's arithmetic is that of an 8-sequence launch (bit-identical results).
__global__ void __launch_bounds__(kTS_NT) k_backward_solve(BwdArgs A) {
    extern __shared__ double bsm[];
    double (*Vb)[kXS] = reinterpret_cast<double (*)[kXS]>(bsm);
    double (*O)[kXS] = reinterpret_cast<double (*)[kXS]>(bsm + kSolveRB * kXS);
    double (*Sg)[kSS] = reinterpret_cast<double (*)[kSS]>(bsm + (kTS_W + kSolveRB) * kXS);
    __shared__ int sh_item, sh_last;
    const int tid = threadIdx.x;
    while (true) {
        if (tid == 0) sh_item = atomicAdd(A.ticket, 1);
        __syncthreads();
        const int item = sh_item;
        __syncthreads();
        if (item >= A.nitems * A.ntile) return;
        const int tile = item % A.ntile;
        const int2 it = A.items[item / A.ntile];
        int *const done = A.done + (size_t)tile * A.nsn;
        int *const cntp = A.cnt + (size_t)tile * A.nsn;
        double *const Pt = A.P + (size_t)tile * A.pstride;
        double *const Zt = A.Z + (size_t)tile * 8 * A.zstride;
        const int nseq = min(8, A.nseq - 8 * tile);
        const int s = it.x, rb = it.y * kSolveRB;
        const int c0 = A.sn_c0[s], w = A.sn_c0[s + 1] - c0;
        const int slot0 = A.sn_rowptr[s], nr = A.sn_rowptr[s + 1] - slot0;
        const int nb = (nr + kSolveRB - 1) / kSolveRB;
        const int m = min(kSolveRB, nr - rb);
        // A = Q_s[rb.., :]^T : element (k, i) = Q[rb + i][k]  (w x m)
        stage_block(A.Q + A.sn_valptr[s] + rb, nr, 1, w, m, Sg);
        // source row of every right-hand-side row of this item (independent of the parent: resolved
        // before the dependency wait)
        __shared__ int srow[kSolveRB];
        for (int i = tid; i < kSolveRB; i += kTS_NT) {
            const int r = rb + i;
            srow[i] = i < m ? (r < w ? c0 + r : A.sn_rows[slot0 + r]) : -1;
        }
        if (tid == 0) {
            int p = A.sn_parent[s];
            if (p >= 0) {
                volatile int *dp = done + p;
                long long t0 = clock64();
                while (*dp == 0) {
                    __nanosleep(32);
                    if (clock64() - t0 > kSpinLimit) { atomicExch(A.ticket + 1, 1); break; }
                }
            }
            __threadfence();
        }
        __syncthreads();
        // columns: 4 per sequence (xyz + pad); 8 columns when nseq <= 2, else 32
        const int ncw = nseq <= 2 ? 8 : kBwCols, lg = ncw == 8 ? 3 : 5;
        const int kpad = (m + 31) & ~31;
        for (int e = tid; e < kpad * ncw; e += kTS_NT) {
            const int i = e >> lg, c = e & (ncw - 1), r = rb + i, sq = c >> 2, comp = c & 3;
            double v = 0.0;
            if (i < m && comp < 3 && sq < nseq) {
                v = __ldcg(Zt + (size_t)sq * A.zstride + (size_t)srow[i] * 4 + comp);
                if (r >= w) v = -v;
            }
            Vb[i][c] = v;
        }
        cp_async_wait_group<0>();
        __syncthreads();
        if (ncw == 8) block_dmma<1, kTS_W / 8>(w, m, Sg, Vb, O);
        else block_dmma<4, kTS_W / 8>(w, m, Sg, Vb, O);
        __syncthreads();
        double *Pb = Pt + (size_t)(A.pbase[s] + it.y) * kTS_W * kBwCols;
        const int nout = w * ncw;
        if (nb == 1) {   // single block: publish directly
            for (int e = tid; e < nout; e += kTS_NT) {
                const int i = e >> lg, c = e & (ncw - 1), sq = c >> 2, comp = c & 3;
                if (comp < 3 && sq < nseq) Zt[(size_t)sq * A.zstride + (size_t)(c0 + i) * 4 + comp] = O[i][c];
            }
        } else {
            for (int e = tid; e < nout; e += kTS_NT) {
                const int i = e >> lg, c = e & (ncw - 1);
                Pb[i * kBwCols + c] = O[i][c];
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) sh_last = atomicAdd(cntp + s, 1) == nb - 1;
            __syncthreads();
            if (!sh_last) continue;
            __threadfence();
            const double *P0 = Pt + (size_t)A.pbase[s] * kTS_W * kBwCols;
            for (int e = tid; e < nout; e += kTS_NT) {
                const int i = e >> lg, c = e & (ncw - 1), sq = c >> 2, comp = c & 3;
                if (comp >= 3 || sq >= nseq) continue;
                double x = 0.0;
                for (int b = 0; b < nb; ++b) x += __ldcg(P0 + (size_t)b * kTS_W * kBwCols + i * kBwCols + c);
                Zt[(size_t)sq * A.zstride + (size_t)(c0 + i) * 4 + comp] = x;
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicExch(done + s, 1);
    }
}


// ------------------------------------------------------------------ host wrappers ---------
constexpr int kFwdSmem = ((kTS_W + kSolveRB) * kXS + kSgRows * kSS) * (int)sizeof(double);

void trisolve_init() {
    cudaFuncSetAttribute(k_forward_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
    cudaFuncSetAttribute(k_backward_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
}

int grad_tiles(int nseq) { return nseq <= 2 ? 1 : (nseq + 7) / 8; }

void launch_ts_plan(const DevFactor &F, const int *qS, const int *nS_ptr, int capS, const int *same_S,
                    long long up_cap, int *flags, int mode, int nseq, int *lo, int *hi, int *cnt, int *rem,
                    int *item_ptr, int *ticket, cudaStream_t st) {
    PDI_LAUNCH(k_ts_plan, 1, kPlanNT, 0, st)(F.ford, F.sn_c0, F.sn_rowptr, F.sn_fd, F.sn_parent, F.nsn, qS, nS_ptr,
                                              capS, same_S, F.nU, up_cap, flags, mode, grad_tiles(nseq), lo, hi,
                                              cnt, rem, item_ptr, ticket);
}

void launch_forward_solve(const DevFactor &F, const int *lo, const int *hi, const int *item_ptr,
                          const int *qS, int *rem, int *ticket, const double *G, double *Y, double *V,
                          int ldv, double *Ug, double *Up, const int *nS_ptr, int capS, int with_grad,
                          int nseq, long long gstride, long long ustride,
                          int nsm, unsigned long long *trace, cudaStream_t st, const double *Yadd) {
    FwdArgs A;
    A.sn_c0 = F.sn_c0; A.sn_rowptr = F.sn_rowptr; A.sn_parent = F.sn_parent;
    A.uoff = F.uoff; A.rc_ptr = F.rc_ptr; A.rc_src = F.rc_src;
    A.sn_valptr = F.sn_valptr; A.Q = F.Q;
    A.lo = lo; A.hi = hi; A.item_ptr = item_ptr; A.qS = qS; A.ford = F.ford; A.nsn = F.nsn;
    A.rem = rem; A.ticket = ticket; A.G = G; A.Y = Y; A.V = V; A.ldv = ldv;
    A.Ug = Ug; A.Up = Up; A.nS_ptr = nS_ptr; A.capS = capS; A.with_grad = with_grad; A.trace = trace;
    A.nseq = nseq; A.gstride = gstride; A.ustride = ustride; A.Yadd = Yadd;
    A.ngt = grad_tiles(nseq);
    A.gw = nseq <= 2 ? 8 : 32;
    PDI_LAUNCH(k_forward_solve, nsm, kTS_NT, kFwdSmem, st)(A);
}

void launch_backward_solve(const DevFactor &F, int *done, int *cnt, int *ticket, double *P, double *Z,
                           int nseq, long long zstride, int nsm, cudaStream_t st) {
    BwdArgs A;
    A.sn_c0 = F.sn_c0; A.sn_rowptr = F.sn_rowptr; A.sn_rows = F.sn_rows; A.sn_parent = F.sn_parent;
    A.sn_valptr = F.sn_valptr; A.Q = F.Q; A.items = F.bw_items; A.pbase = F.bw_pbase;
    A.nitems = F.bw_nitems; A.done = done; A.cnt = cnt; A.ticket = ticket; A.P = P; A.Z = Z;
    A.nseq = nseq; A.zstride = zstride;
    A.ntile = (nseq + kBwSeqs - 1) / kBwSeqs;
    A.nsn = F.nsn;
    A.pstride = (long long)F.bw_nblocks * kTS_W * kBwCols;
    dev_zero3(ticket, sizeof(int), done, sizeof(int) * F.nsn * A.ntile, cnt, sizeof(int) * F.nsn * A.ntile, st);
    PDI_LAUNCH(k_backward_solve, nsm, kTS_NT, kFwdSmem, st)(A);
}





}  // namespace pdipc
