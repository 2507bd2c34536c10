// C ABI (include/pd_ipc.h) and the per-iteration orchestration of the PD+IPC hot path.
//
// One iteration of Algorithm 1 on the device, stream-ordered:
//   Misc   : a1 local step (fused polar + per-corner elastic forces), a2 gather -> g_el
//   IPC    : a3 s = W x, a4 hash broad phase, a5 narrow phase + per-pair derivatives + PSD,
//            a6 S, g-hat = g_el + W^T grad_s B, B-check
//   G-Step : a7/a8 forward solves (w_el = L^-1 Pi g_el and the contact panel), a9 dense
//            K_s = V^T V, Sigma_s = K_s^{-1}, Sigma-hat Cholesky, u, t = B u, one backward
//            solve of w + V t  -> dx = -(H + B)^{-1} g-hat exactly
//   CCD    : ds = W dx, swept broad phase, ACCD -> alpha_m
//   LS     : surrogate energy differences at alpha_m 2^-h, first decrease -> alpha; x += alpha dx
//
// Sequences: a handle holds B independent actuation sequences sharing the mesh
// and the factor.  They advance in LOCKSTEP: one lockstep iteration runs a1/a2 over (tet,
// sequence) in one launch each (mesh data read once per tet), ONE forward solve with the 3B
// gradient right-hand sides of all sequences (the factor read once per supernode row block),
// then every sequence's contact stages and its dense Schur step (each with its own n_c), then
// backward solves of 8 sequences' right-hand sides per launch, then every sequence's CCD, line
// search and update.  Per-sequence state: x, A, forces, gradients, candidate lists, counters and
// a reuse slot (V_s, K_s / Sigma_s and the S they belong to).  All counts live on the device;
// a batch of iterations is one captured CUDA graph with one host round trip.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pd_ipc.h"
#include "kernels.h"
#include "prims.h"
#include "setup.h"

namespace pdipc {

struct CudaError : std::runtime_error {
    int code;
    CudaError(const std::string &m, int c) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_),               \
                            e_ == cudaErrorMemoryAllocation ? PD_IPC_E_OOM : PD_IPC_E_CUDA); \
    } while (0)

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    void ensure(size_t m) {
        if (m <= n && p) return;
        if (p) cudaFree(p);
        p = nullptr;
        size_t cap = std::max<size_t>(m, 1);
        if (n) cap = std::max(cap, n + n / 2);
        CK(cudaMalloc(&p, cap * sizeof(T)));
        n = cap;
    }
    void exact(size_t m) {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        ensure(m);
    }
    void upload(const T *h, size_t m) {   // m may be 0 (a 1-element buffer is still allocated)
        exact(std::max<size_t>(m, 1));
        if (m && h) CK(cudaMemcpy(p, h, m * sizeof(T), cudaMemcpyHostToDevice));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

static int bits_for(unsigned long long v) {   // bits to represent values < v (v >= 1)
    int b = 0;
    while (b < 64 && (1ull << b) < v) ++b;
    return std::max(b, 1);
}

constexpr int kMaxBatch = 32;   // iterations enqueued (or captured) before one host round trip
constexpr int kSlotCap = 256;   // (iteration, sequence) slots of one batch: k = kSlotCap / B iterations

// Device int slots of a sequence (32 ints each).  Every count an iteration needs stays on the
// device; the host reads them once per batch.
enum : int {
    D_ACNT = 0,      // [0] n_pt, [1] n_all active pairs
    D_CCNT = 2,      // [2] npt, [3] ntot candidates of the current broad phase
    D_INFO = 4,      // Cholesky info
    D_CAP = 5,       // capacity bits: 1 candidate buffer, 2 |S| > capS, 4 panel update rows
    D_HOVF = 6,      // [6] static, [7] swept hash overflow (outlier box / table) -> sort path
    D_SAME = 9,      // V_s, K_s, Sigma_s of the sequence's reuse slot belong to this S
    D_STAT = 10,     // [10] npt, [11] ntot of the static phase (stats)
    D_ABORT = 12,    // [12] sticky: an iteration of the batch failed, [13] its index, [14] why
    D_REUSED = 15,   // iterations of the batch that reused V_s, K_s, Sigma_s
    D_SORT = 16,     // [16..18] scratch counters of the sort path
    D_LSCTR = 19,    // line-search round: blocks finished (the last one decides; reset by it)
    D_NS = 20,       // |S| of the last iteration
    D_CONV = 21,     // [21] converged in this pd_ipc_step call, [22] iterations applied, [23] ticket
    D_UPDATED = 24,  // iterations of the batch that updated Sigma_s by low-rank steps
    D_STRIDE = 32,
};
constexpr int S_STRIDE = 18;   // doubles per sequence in dscal: [0] unused, [1] amin, [2..4] ls,
                               // [5..8] ls_out, [9..10] scal, [11] max |pair term|, [12] min
                               // active distance, [14..15] broad-phase cell, [16] kappa of the
                               // sequence, [17] previous min active d^2 (adaptive kappa)

struct Seq {
    // captured CUDA graph of a batch run of this sequence alone (debug / redo path)
    pd_ipc_stats stats;
    DBuf<unsigned long long> cand;   // candidate keys: static list, then the previous swept list
    bool force_sort = false;         // the next broad phases take the sort path (hash overflow)
    int slot = 0;                    // reuse slot (V_s, K_s, key)
    int cg_iters = 0;                // pcg backend: CG iterations of the current pd_ipc_step call
    bool converged = false;          // conv_tol reached in the current pd_ipc_step call
    int iters_applied = 0;
    int nS = 0;
    // debug copies of the last iteration
    std::vector<int32_t> pt, ee, S;
    std::vector<double> ghat, gel, dx, proj, pgrad, phess;
};

// Per-kernel-group device timing (CUDA events on the launching stream), for the roofline report.
enum KId { K_LOCAL = 0, K_GATHER, K_BROAD, K_NARROW, K_DERIV, K_ASSEMBLY, K_FWD, K_DENSE, K_BWD,
           K_CCD, K_LS, K_D_SYRK, K_D_INV, K_D_POTRF, K_D_SOLVE, K_NUM };
static const char *kKernelNames[K_NUM] = {"local_step", "gather", "broad_phase", "narrow_phase",
                                          "pair_derivatives", "contact_assembly", "panel_forward",
                                          "dense_schur", "backward_solve", "ccd", "line_search",
                                          "w_el_forward", "unused.1", "dense.potrf",
                                          "dense.solve"};
// During stream capture an event must be recorded as an external event node (a plain record
// would only mark a capture dependency); outside capture a plain record.
static bool g_capturing = false;
static void record_event(cudaEvent_t e, cudaStream_t st) {
    CK(g_capturing ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st));
}

// Table-1 stage boundaries per (iteration, sequence) slot of a batch:
//   [0] batch-iteration start, [1] after a1/a2 (batched), [2] sequence's contact start,
//   [3] after its IPC stages, [4] after its Schur step, [5] backward solves start (batched),
//   [6] after them, [7] sequence's CCD start, [8] after CCD, [9] after line search + update
constexpr int kStageEv = 10;
struct StageTimer {
    std::vector<cudaEvent_t> ev;     // [kSlotCap][kStageEv]
    std::vector<char> used;
    void init() {
        ev.resize((size_t)kSlotCap * kStageEv);
        used.assign(ev.size(), 0);
        for (auto &e : ev) CK(cudaEventCreate(&e));
    }
    void destroy() { for (auto &e : ev) cudaEventDestroy(e); }
    cudaEvent_t &at(int slot, int k) { return ev[(size_t)slot * kStageEv + k]; }
    void rec(int slot, int k, cudaStream_t st) {
        record_event(at(slot, k), st);
        used[(size_t)slot * kStageEv + k] = 1;
    }
    float el(int slot, int a, int b) {
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, at(slot, a), at(slot, b)));
        return f;
    }
};

struct KTimer {
    bool on = false;
    unsigned mask = ~0u;                // timed groups (bit k = group k)
    int slot = 0;                       // (iteration, sequence) slot being enqueued
    std::vector<cudaEvent_t> ev;        // [kSlotCap][K_NUM][2]
    std::vector<char> used;             // [kSlotCap][K_NUM]
    double ms[K_NUM] = {};
    long long cnt[K_NUM] = {};
    void init() {
        ev.resize((size_t)kSlotCap * K_NUM * 2);
        used.assign((size_t)kSlotCap * K_NUM, 0);
        for (auto &e : ev) CK(cudaEventCreate(&e));
    }
    void destroy() { for (auto &e : ev) cudaEventDestroy(e); }
    cudaEvent_t &e(int s, int k, int w) { return ev[((size_t)s * K_NUM + k) * 2 + w]; }
    void start(int k, cudaStream_t st) { if (on && (mask >> k & 1)) record_event(e(slot, k, 0), st); }
    void stop(int k, cudaStream_t st) {
        if (on && (mask >> k & 1)) { record_event(e(slot, k, 1), st); used[(size_t)slot * K_NUM + k] = 1; }
    }
    bool timeline = false;          // PDIPC_TIMELINE=1: print start/stop offsets of every group
    void collect(const std::vector<char> &applied) {   // after a stream synchronize
        if (timeline)
            for (int i = 0; i < kSlotCap; ++i) {
                if (!used[(size_t)i * K_NUM + K_LOCAL] || !applied[i]) continue;
                std::fprintf(stderr, "timeline it %d:", i);
                for (int k = 0; k < K_NUM; ++k)
                    if (used[(size_t)i * K_NUM + k]) {
                        float a, b;
                        CK(cudaEventElapsedTime(&a, e(i, K_LOCAL, 0), e(i, k, 0)));
                        CK(cudaEventElapsedTime(&b, e(i, K_LOCAL, 0), e(i, k, 1)));
                        std::fprintf(stderr, " %s=[%.1f,%.1f]", kKernelNames[k], 1e3 * a, 1e3 * b);
                    }
                std::fprintf(stderr, "\n");
            }
        for (int i = 0; i < kSlotCap; ++i)
            for (int k = 0; k < K_NUM; ++k)
                if (used[(size_t)i * K_NUM + k]) {
                    if (applied[i]) {
                        float f;
                        CK(cudaEventElapsedTime(&f, e(i, k, 0), e(i, k, 1)));
                        ms[k] += f;
                        cnt[k] += 1;
                    }
                    used[(size_t)i * K_NUM + k] = 0;
                }
    }
};

// captured graph of one batch shape (first sequence, sequence count, iterations)
struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    unsigned key = ~0u, mask = 0;
    int b0 = -1, nb = 0, k = 0;
    long long launches = 0;
    std::vector<char> kt_used, st_used;
};

}  // namespace pdipc

using namespace pdipc;

// Scratch of the contact stage (a3-a6) and of the CCD / line-search stage (a10-a11) of one
// sequence: a second set lets pairs of sequences run these stages concurrently on two streams
// (chains of small latency-bound kernels).  X(member) for every per-stage buffer, stream, event.
#define PD_CONTACT_SCRATCH(X)                                                                         \
    X(cand_tmp) X(flag) X(pos) X(ctype) X(cd2) X(iscr) X(akeys) X(atype) X(ad2) X(grad) X(Hp) X(dist) \
    X(ids) X(blo) X(bhi) X(qcnt) X(qoff) X(qlist) X(gsq) X(hcnt) X(hstart) X(hent) X(mark) X(st) X(st3) \
    X(ev_fork3) X(ev_join3) X(ev_S) X(part) X(b0) X(lspart) X(tepart)
struct ContactAlt;

struct pd_ipc {
    std::string err;
    int device = 0, nsm = 148;
    cudaStream_t st = nullptr;
    pd_ipc_options opt{};
    double dh = 0, kappa = 0, dh2 = 0;
    HostMesh hm;
    HostFactor hf;
    int n = 0, T = 0, nf = 0, Ns = 0, Nt = 0, Ne = 0, B = 1;
    int capS = 0, ldv = 0, ldh = 0, ldk = 0;   // ldk: even row stride of K / Sigma_s (16-byte rows)
    int debug = 0;
    double cell0 = 0;
    // mesh (shared by sequences)
    DBuf<int4> tets;
    DBuf<double> B_, w;
    DBuf<int> inc_ptr, inc, q2v, v2q;
    DBuf<int> Wp, Wc, WTp, WTr, tris, edges;
    DBuf<double> Wv, WTv;
    // factor
    DevFactor F;
    DBuf<int> f_c0, f_rowptr, f_rows, f_parent, f_seg_ptr, f_seg_d, f_seg_klo, f_seg_khi, f_fd, f_col2sn;
    DBuf<long long> f_valptr, f_dinv_ptr;
    DBuf<double> f_L, f_dinv, Ug, Up, bw_P;
    DBuf<int2> f_bw_items, f_rc_src;
    DBuf<int> f_bw_pbase, bw_cnt, f_ford, f_path_ptr, f_path_sn;
    DBuf<int> f_uoff, f_urow_sn, f_rc_ptr, f_rc_idx, f_urel, f_ch_ptr, f_ch;
    // sequences: host state + batched device arrays [B][...]
    std::vector<std::unique_ptr<Seq>> seqs;
    DBuf<double4> x_all, gel_all, dx_all, s_all, ds_all, xstage, surf_out;
    DBuf<double> A6_all, p_all, fc_all, G_all, Yw_all, Z_all, dscal_all;
    DBuf<int> dint_all;
    // reuse slots: V_s [nf][ldv], K_s / -Sigma_s [capS][capS], the S they belong to
    int nslots = 1;
    std::vector<DBuf<double>> V_slot, K_slot;
    std::vector<DBuf<int>> qS_slot;
    DBuf<int> nS_slot;                  // [nslots] |S| of the key (0 = invalid)
    DBuf<int> nupd_slot;                // [nslots] low-rank Sigma_s updates since the last full sweep
    // reduced-solve backend: panel (V_s on the fly) or gather (precomputed
    // G2 = (L^-1)_RR over the region R of W-supported free vertices, n2 = |R|)
    bool gather = false;
    bool pcg = false;                   // the paper's PCG baseline
    bool region = false;                // the paper's literal prescribed-region solve (backend 4: S = R)
    ContactAlt *alt = nullptr;          // second contact-stage scratch set (batched Schur groups)
    cudaEvent_t ev_cfork = nullptr, ev_cjoin = nullptr;
    DBuf<int> Rq_dev;                   // region R (factor positions), backend 4
    DBuf<double> cg_r, cg_p, cg_z, cg_q, cg_t, cg_f, cg_R, cg_part;
    double *cg_rr_host = nullptr;       // pinned: r.r of the last CG iteration
    int n2 = 0;
    DBuf<double> G2, Yel_all, Zf_all, bw_P2;
    DBuf<int> rpos, ts_done2, bw_cnt2;
    // shared contact / Schur work buffers (a sequence's contact + Schur stages run in order)
    DBuf<double> A9stage;               // actuation of all sequences (host input), [B][T][9]
    DBuf<int> aflag;                    // actuation check bits
    DBuf<double4> blo, bhi;
    DBuf<int> hcnt, hstart, hent, qcnt, qoff, qlist;
    unsigned hmask = 0;
    size_t pair_cap = 0;                // capacity of the per-pair buffers (>= every cand.n)
    DBuf<unsigned long long> cand_tmp, akeys;
    DBuf<int> flag, pos, ctype, atype, ids, iscr;
    DBuf<double> cd2, ad2, grad, Hp, dist;
    DBuf<int> mark;
    DBuf<double> lspart;    // line-search partial sums [ls_round_width()][ls_blocks()]
    DBuf<double> tepart;    // true-energy line search: elastic partials [ls_round_width()][ls_te_blocks(T)]
    // second stream: w_el = L^-1 Pi g_el of all sequences runs concurrently with the contact
    // stages (it depends on the elastic gradients only)
    cudaStream_t st2 = nullptr;
    bool side_env = false;    // PDIPC_SIDE_CTAS given: use side_ctas for every batch size
    int side_ctas = 74;       // persistent CTAs of the stream-2 solve (PDIPC_SIDE_CTAS); the rest
                              // of the SMs run the contact stages concurrently (74: the w_el solve
                              // and the contact path end together at C2, tools/side_sweep.sh)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // third stream: the contact-gradient pull-back (needs the pair gradients only) runs beside
    // the S / B-check chain of the assembly
    cudaStream_t st3 = nullptr;
    cudaEvent_t ev_fork3 = nullptr, ev_join3 = nullptr, ev_S = nullptr;
    DBuf<double> Ug2;
    DBuf<int> ts_lo2, ts_hi2, ts_cnt2, ts_ptr2, ts_rem2, ticket2, f_bord, iscr2;
    bool graphs = true;       // replay each batch as a CUDA graph (PDIPC_NO_GRAPH=1: off)
    unsigned buf_epoch = 0;   // bumped whenever a buffer the iteration uses is reallocated
    std::vector<GraphEntry> gcache;
    DBuf<int> ts_lo, ts_hi, ts_cnt, ts_ptr, ts_rem, ts_done, ticket;
    DBuf<double> part, b0;
    // per-system buffers of the Schur step: a sequence's contact stages fill the set of its group
    // (b mod nsysb) and the batched Schur launch runs nsysb systems at once (gather backend, B > 1)
    struct SysBufs {
        DBuf<int> qS, spos;                                  // S (factor positions), S positions / |S|
        DBuf<double> Bc, Sh, gcS, Lstore, U, Tt, yS, rhs, u, tv;
        // B-check assembly: fixed-point accumulators (hi, lo words; zero between uses), the bits
        // and list of the lower 3 x 3 blocks touched by the current use, and its count
        DBuf<long long> Bh, Bl;
        DBuf<unsigned> tbits;
        DBuf<int> tlist, tcnt;
        DBuf<int> dpos, rl, al, uinfo;                      // low-rank Sigma_s update plan
    };
    std::vector<SysBufs> sys;
    int nsysb = 1;
    SysBufs &sb(int b) { return sys[b % nsysb]; }
    DBuf<long long> gsq;    // surface gradient, fixed point [Ns][3]
    StageTimer tm;
    KTimer kt;
    // debugging aid: PDIPC_TRACE=<file> appends per-item forward-solve timestamps
    FILE *trace_file = nullptr, *schur_file = nullptr;
    DBuf<unsigned long long> trace, sprof;

    // per-sequence views of the batched arrays
    double4 *x(int b) { return x_all.p + (size_t)b * n; }
    double *A6(int b) { return A6_all.p + (size_t)b * 6 * T; }
    double4 *gel(int b) { return gel_all.p + (size_t)b * nf; }
    double *G(int b) { return G_all.p + (size_t)b * 4 * nf; }
    double *Yw(int b) { return Yw_all.p + (size_t)b * 4 * nf; }
    double *Z(int b) { return Z_all.p + (size_t)b * 4 * nf; }
    double *Yel(int b) { return Yel_all.p + (size_t)b * 4 * nf; }
    double *Zf(int b) { return Zf_all.p + (size_t)b * 4 * nf; }
    double4 *dx(int b) { return dx_all.p + (size_t)b * n; }
    double4 *s(int b) { return s_all.p + (size_t)b * std::max(1, Ns); }
    double4 *ds(int b) { return ds_all.p + (size_t)b * std::max(1, Ns); }
    int *dint(int b) { return dint_all.p + (size_t)b * D_STRIDE; }
    double *dscal(int b) { return dscal_all.p + (size_t)b * S_STRIDE; }
};

static thread_local std::string g_last_error;

static int fail(pd_ipc *h, int code, const std::string &msg) {
    if (h) h->err = msg;
    g_last_error = msg;
    return code;
}

struct ContactAlt {
#define PD_ALT_MEMBER(m) decltype(pd_ipc::m) m{};
    PD_CONTACT_SCRATCH(PD_ALT_MEMBER)
#undef PD_ALT_MEMBER
};
// swap the handle's contact-stage scratch with the second set (host-side pointers only: what the
// kernels enqueued next see)
static void swap_contact_scratch(pd_ipc *h) {
#define PD_SWAP_MEMBER(m) std::swap(h->m, h->alt->m);
    PD_CONTACT_SCRATCH(PD_SWAP_MEMBER)
#undef PD_SWAP_MEMBER
}

// ------------------------------------------------------------------ helpers --------------
static void sync_read_ints(pd_ipc *h, int *dst, const int *src, int k) {
    CK(cudaMemcpyAsync(dst, src, sizeof(int) * k, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
}

// device scalar <- v, stream-ordered, no host staging (a pageable H2D copy would block)
static void set_d(pd_ipc *h, double *dptr, double v) { launch_set_double(dptr, v, h->st); }

// shared per-pair / per-candidate scratch sized for n candidate keys (the largest list of any
// sequence)
static void grow_pair_set(pd_ipc *h, size_t n);
static void ensure_pair_buffers(pd_ipc *h, size_t n) {
    if (n <= h->pair_cap) return;
    ++h->buf_epoch;
    h->pair_cap = n;
    grow_pair_set(h, n);
    if (h->alt) {
        swap_contact_scratch(h);
        grow_pair_set(h, n);
        swap_contact_scratch(h);
    }
}
static void grow_pair_set(pd_ipc *h, size_t n) {
    h->cand_tmp.exact(n);
    h->flag.exact(n + 1);
    h->pos.exact(n + 1);
    h->ctype.exact(n + 1);
    h->cd2.exact(n + 1);
    h->iscr.ensure(std::max(radix_scratch_ints((int)n + 1), scan_scratch_ints((int)n + 1)) + 1024);
    if (h->Nt > 0) {
        h->akeys.exact(n + 1);
        h->atype.exact(n + 1);
        h->ad2.exact(n + 1);
        h->grad.exact(12 * n + 12);
        h->Hp.exact(78 * n + 78);
        h->dist.exact(n + 1);
        h->ids.exact(4 * n + 4);
        h->b0.exact(n + 1);
    }
}

// grow sequence b's candidate list (and the shared pair buffers) to at least n keys (rare;
// synchronising)
static void grow_candidates(pd_ipc *h, int b, size_t n) {
    Seq &q = *h->seqs[b];
    if (n > q.cand.n) {
        ++h->buf_epoch;
        q.cand.exact(n);
    }
    ensure_pair_buffers(h, n);
}

// parity / debugging copies of the last iteration of sequence b (run alone: the shared contact
// buffers hold its data)
static void debug_capture(pd_ipc *h, int b, int n_pt, int n_ee, int nS) {
    Seq &q = *h->seqs[b];
    pd_ipc::SysBufs &SB = h->sb(b);
    const int nf = h->nf;
    std::vector<double> G4(4 * (size_t)nf), g4(4 * (size_t)nf);
    CK(cudaMemcpy(G4.data(), h->G(b), sizeof(double) * 4 * nf, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(g4.data(), h->gel(b), sizeof(double) * 4 * nf, cudaMemcpyDeviceToHost));
    q.ghat.assign(3 * (size_t)h->n, 0.0);
    q.gel.assign(3 * (size_t)h->n, 0.0);
    for (int k = 0; k < nf; ++k)
        for (int a = 0; a < 3; ++a) {
            q.ghat[3 * (size_t)h->hm.q2v[k] + a] = G4[4 * (size_t)k + a];
            q.gel[3 * (size_t)h->hm.q2v[k] + a] = g4[4 * (size_t)k + a];
        }
    const int na = n_pt + n_ee;
    std::vector<unsigned long long> ak(na);
    if (na) CK(cudaMemcpy(ak.data(), h->akeys.p, sizeof(unsigned long long) * na, cudaMemcpyDeviceToHost));
    q.pt.clear();
    q.ee.clear();
    for (int k = 0; k < na; ++k) {
        const unsigned long long nb = k < n_pt ? (unsigned long long)h->Nt : (unsigned long long)h->Ne;
        auto &v = k < n_pt ? q.pt : q.ee;
        v.push_back((int32_t)(ak[k] / nb));
        v.push_back((int32_t)(ak[k] % nb));
    }
    q.pgrad.resize(12 * (size_t)na);
    q.phess.resize(78 * (size_t)na);
    if (na) {
        CK(cudaMemcpy(q.pgrad.data(), h->grad.p, sizeof(double) * q.pgrad.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(q.phess.data(), h->Hp.p, sizeof(double) * q.phess.size(), cudaMemcpyDeviceToHost));
    }
    std::vector<int> qs(nS);
    if (nS) CK(cudaMemcpy(qs.data(), SB.qS.p, sizeof(int) * nS, cudaMemcpyDeviceToHost));
    q.S.clear();
    for (int v : qs) q.S.push_back(h->hm.q2v[v]);
    std::sort(q.S.begin(), q.S.end());
    std::vector<double4> d4(h->n);
    CK(cudaMemcpy(d4.data(), h->dx(b), sizeof(double4) * h->n, cudaMemcpyDeviceToHost));
    q.dx.resize(3 * (size_t)h->n);
    for (int v = 0; v < h->n; ++v) {
        q.dx[3 * v] = d4[v].x;
        q.dx[3 * v + 1] = d4[v].y;
        q.dx[3 * v + 2] = d4[v].z;
    }
}

// debugging aid (PDIPC_TRACE): per-item forward-solve timestamps and Schur phase timestamps
static void dump_traces(pd_ipc *h, int nS) {
    if (!h->trace_file || nS <= 0 || std::ftell(h->trace_file) >= (30l << 20)) return;
    if (h->gather || !h->trace.p) {   // no panel forward solve to trace: Schur phases only
        if (h->schur_file) {
            std::vector<unsigned long long> pr(1024);
            CK(cudaMemcpy(pr.data(), h->sprof.p, 1024 * 8, cudaMemcpyDeviceToHost));
            fwrite(&nS, sizeof(int), 1, h->schur_file);
            fwrite(pr.data(), 8, 1024, h->schur_file);
            fflush(h->schur_file);
        }
        return;
    }
    int nitems;
    CK(cudaMemcpy(&nitems, h->ts_ptr.p + h->F.nsn, sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<unsigned long long> tr(4 * (size_t)nitems);
    CK(cudaMemcpy(tr.data(), h->trace.p, tr.size() * 8, cudaMemcpyDeviceToHost));
    fwrite(&nitems, sizeof(int), 1, h->trace_file);
    fwrite(tr.data(), 8, tr.size(), h->trace_file);
    fflush(h->trace_file);
    if (h->schur_file) {
        std::vector<unsigned long long> pr(1024);
        CK(cudaMemcpy(pr.data(), h->sprof.p, 1024 * 8, cudaMemcpyDeviceToHost));
        fwrite(&nS, sizeof(int), 1, h->schur_file);
        fwrite(pr.data(), 8, 1024, h->schur_file);
        fflush(h->schur_file);
    }
}

static void broad_phase_sort(pd_ipc *h, int b, const double4 *ds, double infl, int *ccnt);

// Broad phase of sequence b: static (ds == nullptr, boxes inflated by infl) or swept.  Produces
// sorted unique PT keys in cand[0..npt) and EE keys in cand[npt..ntot) with ccnt = [npt, ntot] on
// the device, no host round trip.  Sort-free: every query sorts its own (short) partner list, so
// the lists come out globally sorted.  A table overflow raises *hovf; the iteration is then
// redone with the sort path.
// Hash cell = min(max box extent, kCellCap * cell0): one long swept box must not coarsen the grid
// for every query; boxes wider than the cap span several cells (bounded, see k_hash_insert).
constexpr double kCellCap = 2.0;

static void broad_phase(pd_ipc *h, int b, const double4 *ds, double infl, int *ccnt, int *hovf) {
    Seq &q = *h->seqs[b];
    if (q.force_sort || (h->opt.debug_flags & PD_IPC_DBG_SORT_BROAD)) {
        broad_phase_sort(h, b, ds, infl, ccnt);
        return;
    }
    cudaStream_t st = h->st;
    const int Ns = h->Ns, Nt = h->Nt, Ne = h->Ne;
    double *ext = h->dscal(b) + 14;   // cell = [max box extent, cap]
    const unsigned M = h->hmask + 1;
    // PD_IPC_DBG_TINY_HASH: an entry capacity of 1 makes the hash path overflow, so the iteration
    // is redone on the sort path (exercises the overflow -> sort fallback)
    const int nq = Ns + Ne, cap_ent = (h->opt.debug_flags & PD_IPC_DBG_TINY_HASH) ? 1 : (int)h->hent.n;
    // ext = [cell0, cap], overflow flag and both tables' bucket counts cleared in one launch
    launch_broad_prep(ext, h->cell0, kCellCap * h->cell0, hovf, h->hcnt.p, (int)(2 * (M + 1)), st);
    launch_boxes(h->s(b), ds, h->tris.p, h->edges.p, Ns, Nt, Ne, infl, h->blo.p, h->bhi.p, ext, st);
    // both tables (tris, edges) in one pass each: count, scan (which clears the counts for the
    // fill pass's cursors), fill
    launch_hash_insert(h->blo.p, h->bhi.p, Ns, Nt, Ne, ext, h->hmask, h->hcnt.p, nullptr, nullptr, 0, hovf, st);
    scan_exclusive_clear(h->hcnt.p, h->hstart.p, (int)(2 * (M + 1)), h->iscr.p, st);
    launch_hash_insert(h->blo.p, h->bhi.p, Ns, Nt, Ne, ext, h->hmask, h->hcnt.p, h->hstart.p, h->hent.p,
                       cap_ent, hovf, st);
    // one warp per query (PT points, then EE edges): sorted unique partner lists
    launch_hash_query_warp(h->blo.p, h->bhi.p, Ns, Nt, Ne, ext, h->hmask, h->hstart.p, h->hent.p, h->tris.p,
                           h->edges.p, h->qcnt.p, h->qlist.p, hovf, st);
    scan_exclusive(h->qcnt.p, h->qoff.p, nq, h->iscr.p, st);
    launch_hash_emit(Ns, Nt, Ne, h->qcnt.p, h->qoff.p, h->qlist.p, q.cand.p, (int)q.cand.n, ccnt,
                     h->dint(b) + D_CAP, st);
}

// Fallback after a hash overflow: uncapped cells (every box covers at most 8 of them), global
// radix sort + unique.  Host-synchronous (rare path).
static void broad_phase_sort(pd_ipc *h, int b, const double4 *ds, double infl, int *ccnt) {
    Seq &q = *h->seqs[b];
    cudaStream_t st = h->st;
    const int Ns = h->Ns, Nt = h->Nt, Ne = h->Ne;
    double *ext = h->dscal(b) + 14;
    set_d(h, ext, h->cell0);
    set_d(h, ext + 1, 1e300);
    launch_boxes(h->s(b), ds, h->tris.p, h->edges.p, Ns, Nt, Ne, infl, h->blo.p, h->bhi.p, ext, st);
    const unsigned M = h->hmask + 1;
    int *cnt_pt = h->dint(b) + D_SORT, *cnt_ee = h->dint(b) + D_SORT + 1;
    int *ovf = h->dint(b) + D_SORT + 2;   // cannot trip: uncapped cells bound entries by 8 per box
    CK(dev_zero(ovf, sizeof(int), st));
    CK(dev_zero(h->hcnt.p, sizeof(int) * 2 * (M + 1), st));
    launch_hash_insert(h->blo.p, h->bhi.p, Ns, Nt, Ne, ext, h->hmask, h->hcnt.p, nullptr, nullptr, 0, ovf, st);
    scan_exclusive(h->hcnt.p, h->hstart.p, (int)(2 * (M + 1)), h->iscr.p, st);
    CK(dev_zero(h->hcnt.p, sizeof(int) * 2 * (M + 1), st));
    launch_hash_insert(h->blo.p, h->bhi.p, Ns, Nt, Ne, ext, h->hmask, h->hcnt.p, h->hstart.p, h->hent.p,
                       (int)h->hent.n, ovf, st);
    for (int pass = 0; pass < 2; ++pass) {
        int counts[2];
        const int cap = (int)(q.cand.n / 2);
        for (int kind = 0; kind < 2; ++kind) {   // 0 = PT (B = tris), 1 = EE (B = edges)
            const int b0 = kind == 0 ? Ns : Ns + Nt;
            const int a0 = kind == 0 ? 0 : Ns + Nt, na = kind == 0 ? Ns : Ne;
            const int *hs = h->hstart.p + (size_t)kind * (M + 1), *he = h->hent.p;
            int *cnt = kind == 0 ? cnt_pt : cnt_ee;
            CK(dev_zero(cnt, sizeof(int), st));
            unsigned long long *out = q.cand.p + (size_t)kind * cap;
            launch_hash_query(h->blo.p, h->bhi.p, a0, na, b0, kind == 0 ? Nt : Ne, ext, h->hmask, hs,
                              he, kind == 0, h->tris.p, h->edges.p, out, cnt, cap, st);
        }
        sync_read_ints(h, counts, cnt_pt, 2);
        if (counts[0] <= cap && counts[1] <= cap) {
            // sort + unique each list, then pack PT | EE contiguously in cand_tmp -> cand
            int res[2];
            for (int kind = 0; kind < 2; ++kind) {
                unsigned long long *keys = q.cand.p + (size_t)kind * cap;
                int nk = counts[kind];
                unsigned long long range = kind == 0 ? (unsigned long long)Ns * Nt : (unsigned long long)Ne * Ne;
                // sort scratch = this kind's half of cand_tmp (the PT result lives in the other)
                radix_sort_u64(reinterpret_cast<uint64_t *>(keys),
                               reinterpret_cast<uint64_t *>(h->cand_tmp.p + (size_t)kind * cap), nk,
                               bits_for(range), h->iscr.p, st);
                unique_sorted_u64(reinterpret_cast<uint64_t *>(keys), nk,
                                  reinterpret_cast<uint64_t *>(h->cand_tmp.p + (size_t)kind * cap), h->flag.p,
                                  h->pos.p, h->iscr.p, st);
                CK(dev_copy(cnt_pt + kind, h->pos.p + nk, sizeof(int), st));
            }
            sync_read_ints(h, res, cnt_pt, 2);
            CK(cudaMemcpyAsync(q.cand.p, h->cand_tmp.p, sizeof(unsigned long long) * res[0],
                               cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(q.cand.p + res[0], h->cand_tmp.p + cap, sizeof(unsigned long long) * res[1],
                               cudaMemcpyDeviceToDevice, st));
            const int cc[2] = {res[0], res[0] + res[1]};
            CK(cudaMemcpyAsync(ccnt, cc, sizeof(cc), cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));   // cc is a host stack array
            return;
        }
        grow_candidates(h, b, 2 * (size_t)std::max(counts[0], counts[1]) + 1024);
    }
    throw CudaError("broad phase capacity", PD_IPC_E_CAPACITY);
}

// panel V_s = L^-1 Pi E_S of sequence b into its reuse slot (panel tiles only; no items when S is
// unchanged).  Reads S, |S| and the same-S flag; writes V, Up and the panel plan.  Stream 3.
static void enqueue_panel_forward(pd_ipc *h, int b, const int *nS_dev, cudaStream_t sp) {
    const DevFactor &F = h->F;
    pd_ipc::SysBufs &SB = h->sb(b);
    KTimer &kt = h->kt;
    int *di = h->dint(b);
    kt.start(K_FWD, sp);
    launch_ts_plan(F, SB.qS.p, nS_dev, h->capS, di + D_SAME, (long long)h->Up.n, di + D_CAP, 2, 0,
                   h->ts_lo.p, h->ts_hi.p, h->ts_cnt.p, h->ts_rem.p, h->ts_ptr.p, h->ticket.p, sp);
    if (h->trace_file) h->trace.ensure(4 * (size_t)F.bw_nblocks * (2 + (h->capS + 31) / 32));
    launch_forward_solve(F, h->ts_lo.p, h->ts_hi.p, h->ts_ptr.p, SB.qS.p, h->ts_rem.p, h->ticket.p, nullptr,
                         nullptr, h->V_slot[h->seqs[b]->slot].p, h->ldv, nullptr, h->Up.p, nS_dev, h->capS, 0,
                         0, 0, 0, h->nsm, h->trace_file ? h->trace.p : nullptr, sp);
    kt.stop(K_FWD, sp);
}

// ---- one lockstep iteration of sequences [b0, b0 + nb), iteration index it of the batch -----
// (a) a1 + a2 over (tet, sequence); the w_el solve of all nb sequences forks onto stream 2
static void enqueue_elastic(pd_ipc *h, int b0, int nb, int it) {
    cudaStream_t st = h->st;
    KTimer &kt = h->kt;
    const int slot = it * nb;
    h->kt.slot = slot;
    h->tm.rec(slot, 0, st);
    kt.start(K_LOCAL, st);
    launch_local_step(h->tets.p, h->x(b0), h->B_.p, h->A6(b0), h->w.p, h->T, h->fc_all.p,
                      h->debug ? h->p_all.p + (size_t)b0 * 9 * h->T : nullptr, h->dint(b0), nb, h->n, D_STRIDE,
                      st);   // also clears each sequence's active-pair counts and flags
    kt.stop(K_LOCAL, st);
    kt.start(K_GATHER, st);
    launch_gather_elastic(h->inc_ptr.p, h->inc.p, h->fc_all.p, h->nf, h->gel(b0), nb, 12 * (long long)h->T, st);
    kt.stop(K_GATHER, st);
    h->tm.rec(slot, 1, st);
    // fork: w_el = L^-1 Pi g_el of every sequence (3 nb right-hand sides, ONE solve) on stream 2,
    // concurrent with the contact stages (the contact part of w is V_s gc, folded into the Schur
    // step)
    cudaStream_t s2 = h->st2;
    const DevFactor &F2 = h->F;
    // CTAs of the side solve: 74 when it overlaps a single sequence's contact path (C2, tuned by
    // tools/side_sweep.sh); every SM for a batch of >= 4 sequences, where the first Schur step
    // waits for the whole batched solve (C4: 65.3 -> 65.9 it/s, tools/gpu_side_sweep.sh)
    const int side = h->Nt == 0 ? h->nsm : (nb >= 4 && !h->side_env) ? h->nsm : h->side_ctas;
    CK(cudaEventRecord(h->ev_fork, st));
    CK(cudaStreamWaitEvent(s2, h->ev_fork, 0));
    kt.start(K_D_SYRK, s2);
    // ticket2: [0] item dispenser (cleared by the plan), [1] fault (cleared per batch),
    // [2] |S| = 0 (never written), [3] flags (unused in gradient-only mode)
    launch_ts_plan(F2, nullptr, h->ticket2.p + 2, 0, h->ticket2.p + 2, 0, h->ticket2.p + 3, 1, nb, h->ts_lo2.p,
                   h->ts_hi2.p, h->ts_cnt2.p, h->ts_rem2.p, h->ts_ptr2.p, h->ticket2.p, s2);
    launch_forward_solve(F2, h->ts_lo2.p, h->ts_hi2.p, h->ts_ptr2.p, nullptr, h->ts_rem2.p, h->ticket2.p,
                         reinterpret_cast<const double *>(h->gel(b0)), h->Yw(b0), nullptr, h->ldv, h->Ug2.p,
                         nullptr, h->ticket2.p + 2, 0, 1, nb, 4 * (long long)h->nf,
                         4 * (long long)std::max(1, F2.nU), side, nullptr, s2);
    if (h->gather && h->Nt > 0) {
        // gather backend: y_el = L^-T w_el (the base solve), whose rows S give y_S
        CK(dev_copy(h->Yel(b0), h->Yw(b0), sizeof(double) * 4 * h->nf * nb, s2));
        launch_backward_solve(h->F, h->ts_done2.p, h->bw_cnt2.p, h->ticket2.p, h->bw_P2.p, h->Yel(b0), nb,
                              4 * (long long)h->nf, side, s2);
    }
    kt.stop(K_D_SYRK, s2);
    CK(cudaEventRecord(h->ev_join, s2));
}

// The paper's PCG baseline (Eq. 5) for sequence b, in place of
// the a9 Schur step: CG on M = L^-1 H-hat L^-T = I + L^-1 script-B L^-T with rhs -L^-1 Pi g-hat;
// one iteration = backward solve of p, B-check on S, forward solve of the S-sparse result, vector
// updates.  Host-driven (one 8-byte read per iteration for the convergence test).  Writes
// Z_b = -z, so the common backward solve + scatter give dx = Pi^T L^-T z.
static void pcg_solve(pd_ipc *h, int b) {
    cudaStream_t st = h->st;
    pd_ipc::SysBufs &SB = h->sb(b);
    const DevFactor &F = h->F;
    const int nf = h->nf;
    int *nS_dev = SB.spos.p + nf;
    const long long us = 4 * (long long)std::max(1, F.nU);
    auto fwd = [&](const double *rhs, double *out) {
        launch_ts_plan(F, nullptr, h->ticket2.p + 2, 0, h->ticket2.p + 2, 0, h->ticket2.p + 3, 1, 1, h->ts_lo2.p,
                       h->ts_hi2.p, h->ts_cnt2.p, h->ts_rem2.p, h->ts_ptr2.p, h->ticket2.p, st);
        launch_forward_solve(F, h->ts_lo2.p, h->ts_hi2.p, h->ts_ptr2.p, nullptr, h->ts_rem2.p, h->ticket2.p, rhs, out,
                             nullptr, h->ldv, h->Ug2.p, nullptr, h->ticket2.p + 2, 0, 1, 1, 4 * (long long)nf, us,
                             h->nsm, nullptr, st);
    };
    fwd(h->G(b), h->cg_f.p);                                   // w = L^-1 Pi g-hat
    launch_cg_init(h->cg_f.p, h->cg_r.p, h->cg_p.p, h->cg_z.p, nf, h->cg_part.p, h->cg_rr_host, st);
    CK(cudaStreamSynchronize(st));
    const double rr0 = *h->cg_rr_host;
    const double tol = h->opt.cg_tol > 0 ? h->opt.cg_tol : 1e-12;
    const int maxit = h->opt.cg_max_iters > 0 ? h->opt.cg_max_iters : 10000;
    int it = 0;
    while (rr0 > 0 && it < maxit) {
        CK(dev_copy(h->cg_t.p, h->cg_p.p, sizeof(double) * 4 * nf, st));
        launch_backward_solve(F, h->ts_done.p, h->bw_cnt.p, h->ticket.p, h->bw_P.p, h->cg_t.p, 1, 4 * (long long)nf,
                              h->nsm, st);                     // t = L^-T p
        launch_cg_bmul(SB.Bc.p, 3 * h->capS, SB.qS.p, nS_dev, h->capS, h->cg_t.p, h->cg_R.p, nf, st);
        fwd(h->cg_R.p, h->cg_f.p);                             // f = L^-1 E_S B-check t_S
        launch_cg_update(h->cg_f.p, h->cg_p.p, h->cg_q.p, h->cg_z.p, h->cg_r.p, nf, h->cg_part.p, it,
                         h->cg_rr_host, st);
        CK(cudaStreamSynchronize(st));
        ++it;
        if (std::sqrt(*h->cg_rr_host / rr0) <= tol) break;
    }
    launch_cg_finish(h->cg_z.p, h->Z(b), nf, st);
    h->seqs[b]->cg_iters += it;
}

// (b) sequence b: a3-a6 contact stages, a8 panel (stream 3) and the a9 dense Schur step -> Z_b
static void enqueue_contact(pd_ipc *h, int b, int b0, int nb, int it) {
    cudaStream_t st = h->st;
    Seq &q = *h->seqs[b];
    pd_ipc::SysBufs &SB = h->sb(b);
    KTimer &kt = h->kt;
    const int slot = it * nb + (b - b0);
    kt.slot = slot;
    h->tm.rec(slot, 2, st);
    const int nf = h->nf, Ns = h->Ns, Nt = h->Nt, Ne = h->Ne;
    const int cap = (int)q.cand.n;
    int *di = h->dint(b);
    double *ds_ = h->dscal(b);
    int *acnt = di + D_ACNT, *ccnt = di + D_CCNT;
    int *nS_dev = SB.spos.p + nf;     // exclusive scan total of the S marks
    double *dmax = ds_ + 11;
    const int slotr = q.slot;
    if (Nt > 0) {
        kt.start(K_BROAD, st);
        launch_surface(h->Wp.p, h->Wc.p, h->Wv.p, h->x(b), Ns, h->s(b), st);
        // after the first iteration of a batch the previous iteration's swept candidate list
        // (cand, ccnt; boxes over [s, s + ds] inflated by d_hat) contains every pair closer
        // than d_hat at x + alpha dx: the narrow phase filters it exactly (same C)
        if (it == 0 || h->opt.no_cand_reuse) broad_phase(h, b, nullptr, 0.5 * h->dh * 1.01, ccnt, di + D_HOVF);
        kt.stop(K_BROAD, st);
        kt.start(K_NARROW, st);
        // one pass over [PT | EE] candidates; one scan; actives come out as [PT | EE], each sorted
        launch_narrow(q.cand.p, ccnt, cap, h->s(b), h->tris.p, h->edges.p, Nt, Ne, h->dh2, h->flag.p,
                      h->ctype.p, h->cd2.p, di + D_STAT, st);
        scan_exclusive_dev(h->flag.p, h->pos.p, ccnt + 1, cap, h->iscr.p, st);
        launch_compact_active(q.cand.p, ccnt, cap, h->flag.p, h->pos.p, h->ctype.p, h->cd2.p, h->akeys.p,
                              h->atype.p, h->ad2.p, acnt, st);
        kt.stop(K_NARROW, st);
        kt.start(K_DERIV, st);
        launch_contact_prep(h->mark.p, nf, h->gsq.p, 6 * Ns, dmax, st);   // clears of a5-a6
        if (h->opt.kappa_adapt_eps > 0)       // f3: adaptive kappa from this iteration's min active d^2
            launch_kappa_update(h->ad2.p, acnt, ds_ + 16, h->opt.kappa_adapt_eps * h->opt.kappa_adapt_eps,
                                h->opt.kappa_max, st);
        launch_pair_derivs(h->akeys.p, h->atype.p, h->ad2.p, acnt, cap, h->s(b), h->tris.p, h->edges.p, Nt,
                           Ne, h->dh, ds_ + 16, h->grad.p, h->Hp.p, h->dist.p, h->ids.p, dmax, st);
        kt.stop(K_DERIV, st);
        // fork: stream 3 takes the gradient pull-back (reads ids, grad, dmax, g_el; writes gsq,
        // G: deterministic fixed-point accumulation on the surface, then W^T), then -- once S is
        // known -- the contact gradient on S and the panel forward solve, while this stream
        // assembles B-check
        CK(cudaEventRecord(h->ev_fork3, st));
        CK(cudaStreamWaitEvent(h->st3, h->ev_fork3, 0));
        launch_accum_grad_fx(h->ids.p, acnt, cap, h->grad.p, dmax, h->gsq.p, h->st3);
        launch_grad_pullback_fx(h->gel(b), h->WTp.p, h->WTr.p, h->WTv.p, h->gsq.p, dmax, acnt, nf, h->G(b), h->st3);
        kt.start(K_ASSEMBLY, st);
        // S
        launch_mark_S(h->ids.p, acnt, cap, h->Wp.p, h->Wc.p, h->v2q.p, h->mark.p, st);
        if (h->region)   // backend 4 (the paper's prescribed region x_2, Eq. 6-8): S = R every iteration
            launch_mark_list(h->Rq_dev.p, h->n2, h->mark.p, st);
        scan_compact(h->mark.p, SB.spos.p, SB.qS.p, nf, h->iscr.p, st);   // positions and S (sorted)
        // V_s, K_s, Sigma_s depend on S (and the constant factor) only: reuse the slot's while S
        // is bit-identical to the S they were computed for
        launch_same_S(SB.qS.p, nS_dev, h->qS_slot[slotr].p, h->nS_slot.p + slotr, di + D_SAME, h->capS,
                      h->opt.no_sigma_reuse == 0, di + D_CAP, di + D_REUSED, SB.dpos.p, SB.rl.p, SB.al.p,
                      SB.uinfo.p, h->nupd_slot.p + slotr,
                      h->gather && !(h->opt.debug_flags & PD_IPC_DBG_NO_SIGMA_UPDATE), di + D_UPDATED, st);
        CK(dev_copy(di + D_NS, nS_dev, sizeof(int), st));
        CK(cudaEventRecord(h->ev_S, st));
        CK(cudaStreamWaitEvent(h->st3, h->ev_S, 0));
        launch_gather_gc(SB.qS.p, nS_dev, h->capS, h->WTp.p, h->WTr.p, h->WTv.p, h->gsq.p, dmax, acnt, SB.gcS.p,
                         h->st3);
        if (!h->gather && !h->pcg) enqueue_panel_forward(h, b, nS_dev, h->st3);
        CK(cudaEventRecord(h->ev_join3, h->st3));
        // B-check: the previous use's blocks cleared in the dense double B-check, fixed-point
        // accumulation of the lower blocks (recorded in the block list), then the listed blocks
        // converted (with their mirrors) and their accumulators re-zeroed
        const int ldb = 3 * h->capS;
        launch_bc_clear(SB.Bc.p, ldb, h->capS, SB.tlist.p, SB.tcnt.p, SB.tbits.p, st);
        CK(dev_zero(SB.tcnt.p, sizeof(int), st));
        launch_accum_bc_fx(h->ids.p, acnt, cap, h->Wp.p, h->Wc.p, h->Wv.p, h->v2q.p, SB.spos.p, h->Hp.p, dmax,
                           SB.Bh.p, SB.Bl.p, ldb, h->capS, SB.tbits.p, SB.tlist.p, SB.tcnt.p, st);
        launch_bc_convert(SB.Bh.p, SB.Bl.p, SB.Bc.p, ldb, h->capS, SB.tlist.p, SB.tcnt.p, SB.tbits.p, dmax, acnt, st);
        kt.stop(K_ASSEMBLY, st);
        CK(cudaStreamWaitEvent(st, h->ev_join3, 0));     // join stream 3
    } else {
        CK(dev_zero(nS_dev, sizeof(int), st));
        CK(dev_zero(di + D_SAME, sizeof(int), st));
        CK(dev_zero(di + D_STAT, 2 * sizeof(int), st));
        CK(dev_zero(di + D_NS, sizeof(int), st));
        launch_grad_pullback(h->gel(b), h->WTp.p, h->WTr.p, h->WTv.p, nullptr, nf, h->G(b), st);
    }
    h->tm.rec(slot, 3, st);
}

// (b') the a9 G-step of sequences [c0, c1) (one group each): ONE batched Schur launch (gather
// backend), or per sequence the single-system Schur / PCG solve
static void enqueue_schur(pd_ipc *h, int c0, int c1, int b0, int nb, int it) {
    cudaStream_t st = h->st;
    KTimer &kt = h->kt;
    const int nf = h->nf, Nt = h->Nt;
    const DevFactor &F = h->F;
    // join stream 2 (w_el of all sequences) before the first Schur step of the iteration
    if (c0 == b0) CK(cudaStreamWaitEvent(st, h->ev_join, 0));
    kt.slot = it * nb + (c0 - b0);
    kt.start(K_DENSE, st);
    if (Nt > 0 && h->pcg) {
        for (int b = c0; b < c1; ++b) pcg_solve(h, b);
    } else if (Nt > 0) {
        if (h->trace_file) {
            h->sprof.ensure(1024);
            CK(dev_zero(h->sprof.p, 1024 * 8, st));
        }
        SchurArgs args[kMaxSchurSys];
        for (int b = c0; b < c1; ++b) {
            pd_ipc::SysBufs &SB = h->sb(b);
            const int slotr = h->seqs[b]->slot;
            int *di = h->dint(b);
            args[b - c0] = schur_args(F, h->V_slot[slotr].p, h->ldv, h->Yw(b), SB.gcS.p, SB.qS.p, h->ts_lo.p,
                                      h->ts_hi.p, SB.spos.p + nf, h->capS, h->K_slot[slotr].p, h->ldk, SB.Bc.p,
                                      3 * h->capS, SB.Sh.p, h->ldh, SB.Lstore.p, SB.Tt.p, SB.U.p, SB.yS.p,
                                      SB.rhs.p, SB.u.p, SB.tv.p, h->Z(b), di + D_INFO, di + D_SAME,
                                      h->trace_file ? h->sprof.p : nullptr,
                                      (h->opt.debug_flags & PD_IPC_DBG_LARGE_SCHUR) ? 1 : 0,
                                      h->gather ? kSchurGather : kSchurPanel, h->G2.p, h->n2, h->rpos.p,
                                      h->gather ? h->Yel(b) : nullptr);
            args[b - c0].tbits = SB.tbits.p;   // B-check block bits: t = B u over the nonzero blocks
            if (h->gather) {                // the low-rank Sigma_s update plan of k_same_S
                args[b - c0].uinfo = SB.uinfo.p;
                args[b - c0].dpos = SB.dpos.p;
                args[b - c0].rl = SB.rl.p;
                args[b - c0].al = SB.al.p;
            }
        }
        CK((cudaError_t)launch_schur_batch(args, c1 - c0, st));
    } else {
        for (int b = c0; b < c1; ++b) CK(dev_copy(h->Z(b), h->Yw(b), sizeof(double) * 4 * nf, st));
    }
    kt.stop(K_DENSE, st);
    for (int b = c0; b < c1; ++b) h->tm.rec(it * nb + (b - b0), 4, st);
}

// (c) backward solves of every sequence (8 sequences' right-hand sides per launch), dx scatter
static void enqueue_backward(pd_ipc *h, int b0, int nb, int it) {
    cudaStream_t st = h->st;
    KTimer &kt = h->kt;
    const int slot = it * nb;
    kt.slot = slot;
    h->tm.rec(slot, 5, st);
    double *Zb = h->Z(b0);
    if (h->gather && h->Nt > 0) {
        // gather backend: Zf = w_el + L^-1 Pi E_S (gc + t) -- one forward solve of every sequence's
        // sparse right-hand side (the Schur step left it in Z), added to w_el
        kt.start(K_FWD, st);
        launch_ts_plan(h->F, nullptr, h->ticket2.p + 2, 0, h->ticket2.p + 2, 0, h->ticket2.p + 3, 1, nb, h->ts_lo2.p,
                       h->ts_hi2.p, h->ts_cnt2.p, h->ts_rem2.p, h->ts_ptr2.p, h->ticket2.p, st);
        launch_forward_solve(h->F, h->ts_lo2.p, h->ts_hi2.p, h->ts_ptr2.p, nullptr, h->ts_rem2.p, h->ticket2.p,
                             h->Z(b0), h->Zf(b0), nullptr, h->ldv, h->Ug2.p, nullptr, h->ticket2.p + 2, 0, 1, nb,
                             4 * (long long)h->nf, 4 * (long long)std::max(1, h->F.nU), h->nsm, nullptr, st,
                             h->Yw(b0));
        kt.stop(K_FWD, st);
        Zb = h->Zf(b0);
    }
    kt.start(K_BWD, st);
    launch_backward_solve(h->F, h->ts_done.p, h->bw_cnt.p, h->ticket.p, h->bw_P.p, Zb, nb, 4 * (long long)h->nf,
                          h->nsm, st);
    kt.stop(K_BWD, st);
    launch_scatter_dx(Zb, h->q2v.p, h->nf, h->dx(b0), h->dscal(b0) + 1, nb, h->n, S_STRIDE,
                      st);   // also seeds each sequence's CCD minimum amin = 1
    h->tm.rec(slot, 6, st);
}

// (d) sequence b: CCD, line search, update
static void enqueue_ccd_ls(pd_ipc *h, int b, int b0, int nb, int it) {
    cudaStream_t st = h->st;
    Seq &q = *h->seqs[b];
    KTimer &kt = h->kt;
    const int slot = it * nb + (b - b0);
    kt.slot = slot;
    h->tm.rec(slot, 7, st);
    const int T = h->T, nf = h->nf, Ns = h->Ns, Nt = h->Nt, Ne = h->Ne;
    int *di = h->dint(b);
    double *dsc = h->dscal(b);
    int *ccnt = di + D_CCNT;
    double *amin = dsc + 1, *ls = dsc + 2, *ls_out = dsc + 5, *scal = dsc + 9;
    kt.start(K_CCD, st);
    if (Nt > 0) {
        launch_surface(h->Wp.p, h->Wc.p, h->Wv.p, h->dx(b), Ns, h->ds(b), st);
        broad_phase(h, b, h->ds(b), h->dh, ccnt, di + D_HOVF + 1);
        launch_accd(q.cand.p, ccnt, (int)q.cand.n, h->s(b), h->tris.p, h->edges.p, Nt, Ne, h->ds(b), h->opt.accd_s,
                    h->opt.accd_max_iters, amin, st);
    } else {
        CK(dev_zero(ccnt, 2 * sizeof(int), st));
    }
    kt.stop(K_CCD, st);
    h->tm.rec(slot, 8, st);
    kt.start(K_LS, st);
    {
        // elastic terms: block partials here, summed (fixed order) by the first line-search round
        int nb1 = 0, nb2 = 0;
        elastic_partials(h->gel(b), h->dx(b), h->q2v.p, nf, h->tets.p, h->B_.p, h->w.p, T, h->part.p, &nb1, &nb2,
                         st);
        const int hmax = h->opt.ls_max_halvings;
        const bool te = h->opt.ls_energy == 1;
        for (int h0 = 0; h0 <= hmax; h0 = ls_round_next(h0)) {
            int nte = 0;
            if (te)   // f3: true elastic energy differences of the round's trials (block partials)
                nte = launch_ls_true_elastic(h->tets.p, h->x(b), h->dx(b), h->B_.p, h->A6(b), h->w.p, T, amin, ls,
                                             h0, ls_round_width_at(h0), h->tepart.p, st);
            launch_ls_round(q.cand.p, ccnt, h->s(b), h->tris.p, h->edges.p, Nt, Ne, h->ds(b), h->dh, h->b0.p, ls,
                            h0, h->lspart.p, scal, dsc + 16, hmax, ls_out, di + D_LSCTR, h->part.p, nb1,
                            h->part.p + nb1, nb2, amin, te ? h->tepart.p : nullptr, nte, st);
        }
        launch_update(h->x(b), h->dx(b), h->q2v.p, nf, ls_out, di + D_INFO, di + D_ABORT, it, di + D_CONV,
                      reinterpret_cast<unsigned long long *>(dsc + 13), h->opt.conv_tol, st);
    }
    kt.stop(K_LS, st);
    h->tm.rec(slot, 9, st);
}

static void enqueue_lockstep_iteration(pd_ipc *h, int b0, int nb, int it) {
    enqueue_elastic(h, b0, nb, it);
    for (int c0 = b0; c0 < b0 + nb; c0 += h->nsysb) {      // groups of nsysb sequences (c0 = 0 mod nsysb)
        const int c1 = std::min(b0 + nb, c0 - c0 % h->nsysb + h->nsysb);
        if (h->alt && c1 - c0 >= 2) {
            // the group's contact stages on two streams: even members on the main stream's
            // scratch, odd ones on the second set (its own main / side streams), joined before
            // the Schur launch
            CK(cudaEventRecord(h->ev_cfork, h->st));
            CK(cudaStreamWaitEvent(h->alt->st, h->ev_cfork, 0));
            for (int b = c0; b < c1; b += 2) enqueue_contact(h, b, b0, nb, it);
            swap_contact_scratch(h);
            for (int b = c0 + 1; b < c1; b += 2) enqueue_contact(h, b, b0, nb, it);
            CK(cudaEventRecord(h->ev_cjoin, h->st));
            swap_contact_scratch(h);
            CK(cudaStreamWaitEvent(h->st, h->ev_cjoin, 0));
        } else {
            for (int b = c0; b < c1; ++b) enqueue_contact(h, b, b0, nb, it);
        }
        enqueue_schur(h, c0, c1, b0, nb, it);
        c0 = c1 - h->nsysb;
    }
    enqueue_backward(h, b0, nb, it);
    if (h->alt && nb >= 2) {   // CCD / line search of even sequences on the main set, odd ones on the second
        CK(cudaEventRecord(h->ev_cfork, h->st));
        CK(cudaStreamWaitEvent(h->alt->st, h->ev_cfork, 0));
        for (int b = b0; b < b0 + nb; b += 2) enqueue_ccd_ls(h, b, b0, nb, it);
        swap_contact_scratch(h);
        for (int b = b0 + 1; b < b0 + nb; b += 2) enqueue_ccd_ls(h, b, b0, nb, it);
        CK(cudaEventRecord(h->ev_cjoin, h->st));
        swap_contact_scratch(h);
        CK(cudaStreamWaitEvent(h->st, h->ev_cjoin, 0));
    } else {
        for (int b = b0; b < b0 + nb; ++b) enqueue_ccd_ls(h, b, b0, nb, it);
    }
}

// Run k lockstep iterations of sequences [b0, b0 + nb) with ONE host round trip: replay the
// captured CUDA graph of the batch when possible (every launch configuration is static: all
// sizes live on the device), else enqueue stream-ordered.  A failing iteration of a sequence
// (capacity / hash overflow, Cholesky breakdown, non-finite values) raises that sequence's
// sticky device flag: it and every later iteration of the batch leave its x untouched, so x is
// its last accepted iterate.  applied[b - b0] = iterations applied; ms[b - b0][6] accumulates the
// Table-1 stage times.  Buffers are grown here; the caller runs the rest.
static void run_lockstep(pd_ipc *h, int b0, int nb, int k, std::vector<int> &applied,
                         std::vector<std::array<double, 6>> &ms) {
    cudaStream_t st = h->st;
    KTimer &kt = h->kt;
    bool any_sort = false;
    for (int b = b0; b < b0 + nb; ++b) any_sort |= h->seqs[b]->force_sort;
    const bool graph = h->graphs && !h->debug && !h->trace_file && !any_sort && !h->pcg &&
                       !(h->opt.debug_flags & PD_IPC_DBG_SORT_BROAD);
    const unsigned key = (h->buf_epoch << 1) | (kt.on ? 1u : 0u);
    const unsigned key_mask = kt.on ? kt.mask : 0u;
    auto enqueue_batch = [&]() {
        for (int b = b0; b < b0 + nb; ++b) {
            CK(dev_zero(h->dint(b) + D_ABORT, 4 * sizeof(int), st));   // abort, index, why, reused
            CK(dev_zero(h->dint(b) + D_UPDATED, sizeof(int), st));
        }
        CK(dev_zero(h->ticket.p + 1, sizeof(int), st));               // solve fault flags of the batch
        CK(dev_zero(h->ticket2.p + 1, sizeof(int), st));
        for (int i = 0; i < k; ++i) enqueue_lockstep_iteration(h, b0, nb, i);
    };
    GraphEntry *ge = nullptr;
    if (graph) {
        for (auto &g : h->gcache)
            if (g.b0 == b0 && g.nb == nb && g.k == k) ge = &g;
        if (!ge) {
            h->gcache.emplace_back();
            ge = &h->gcache.back();
            ge->b0 = b0;
            ge->nb = nb;
            ge->k = k;
        }
        if (!ge->exec || ge->key != key || ge->mask != key_mask) {
            if (ge->exec) {
                cudaGraphExecDestroy(ge->exec);
                ge->exec = nullptr;
            }
            cudaGraph_t g = nullptr;
            const long long l0 = launch_count();
            bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                g_capturing = true;
                try {
                    enqueue_batch();
                } catch (const CudaError &) {
                    ok = false;
                }
                g_capturing = false;
                ok = (cudaStreamEndCapture(st, &g) == cudaSuccess) && ok;
            }
            if (ok) ok = cudaGraphInstantiate(&ge->exec, g, 0) == cudaSuccess;
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            const long long n_captured = launch_count() - l0;
            add_launches(-n_captured);                     // counted on every replay instead
            if (ok) {
                ge->launches = n_captured;
                ge->key = key;
                ge->mask = key_mask;
                ge->kt_used = kt.used;
                ge->st_used = h->tm.used;
            } else {
                ge->exec = nullptr;
                h->graphs = false;                         // capture unsupported: stream path from now on
            }
        }
        if (!ge->exec) ge = nullptr;
    }
    if (ge) {
        CK(cudaGraphLaunch(ge->exec, st));
        add_launches(ge->launches);
        kt.used = ge->kt_used;
        h->tm.used = ge->st_used;
    } else {
        enqueue_batch();
    }
    // ---------------- the one host round trip of the batch: counters and scalars of every sequence
    std::vector<int> di((size_t)nb * D_STRIDE);
    std::vector<double> sc((size_t)nb * S_STRIDE);
    CK(cudaMemcpyAsync(di.data(), h->dint(b0), sizeof(int) * di.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(sc.data(), h->dscal(b0), sizeof(double) * sc.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int fault = 0, f2 = 0;
    CK(cudaMemcpy(&fault, h->ticket.p + 1, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&f2, h->ticket2.p + 1, sizeof(int), cudaMemcpyDeviceToHost));
    fault |= f2;
    if (fault) throw CudaError("triangular solve dependency wait timed out", PD_IPC_E_CUDA);
    applied.assign(nb, k);
    std::vector<char> slot_ok((size_t)kSlotCap, 0);
    for (int j = 0; j < nb; ++j) {
        const int *d = di.data() + (size_t)j * D_STRIDE;
        if (d[D_ABORT]) applied[j] = d[D_ABORT + 1];
        for (int i = 0; i < applied[j]; ++i) slot_ok[(size_t)i * nb + j] = 1;
    }
    // Table-1 stage times of each sequence: its own contact / Schur / CCD / LS events, plus its
    // share (1 / nb) of the batched a1/a2 and backward-solve stages
    for (int j = 0; j < nb; ++j)
        for (int i = 0; i < applied[j]; ++i) {
            const int sl = i * nb + j, s0 = i * nb;
            const float misc = h->tm.el(s0, 0, 1) / nb, bw = h->tm.el(s0, 5, 6) / nb;
            const float ipc = h->tm.el(sl, 2, 3), gst = h->tm.el(sl, 3, 4) + bw;
            const float ccd = h->tm.el(sl, 7, 8), lsm = h->tm.el(sl, 8, 9);
            ms[j][0] += ipc;
            ms[j][1] += gst;
            ms[j][2] += ccd;
            ms[j][3] += lsm;
            ms[j][4] += misc;
            ms[j][5] += ipc + gst + ccd + lsm + misc;
        }
    // kernel-group timers: a batched group is recorded on the slot of sequence 0 of an iteration
    {
        std::vector<char> okk((size_t)kSlotCap, 0);
        for (int i = 0; i < kSlotCap; ++i) okk[i] = slot_ok[i];
        for (int i = 0; i < k; ++i) okk[(size_t)i * nb] = 1;   // batched groups of applied iterations
        kt.collect(okk);
    }
    for (int j = 0; j < nb; ++j) {
        const int b = b0 + j;
        Seq &q = *h->seqs[b];
        const int *d = di.data() + (size_t)j * D_STRIDE;
        const double *s = sc.data() + (size_t)j * S_STRIDE;
        q.stats.sigma_reused += d[D_REUSED];
        q.stats.sigma_updated += d[D_UPDATED];
        q.nS = d[D_NS];
        q.converged = d[D_CONV] != 0;
        q.iters_applied = d[D_CONV + 1];
        if (d[D_ABORT]) {   // why: 1 cand, 2 |S|, 4 Up, 8/16 hash, 32 info, 64 NaN
            const int why = d[D_ABORT + 2];
            // V_s, K_s, Sigma_s of the aborted iteration (and of the batch's later, skipped ones)
            // may not have been computed for the S recorded by k_same_S: invalidate the slot key
            CK(dev_zero(h->nS_slot.p + q.slot, sizeof(int), st));
            CK(cudaStreamSynchronize(st));
            if (why & 64) throw CudaError("non-finite value in step (dx, gradient or energy)", PD_IPC_E_NONFINITE);
            if (why & 2) throw CudaError("contact vertex set exceeds capacity", PD_IPC_E_CAPACITY);
            if (why & 32) throw CudaError("dense Cholesky: matrix not SPD", PD_IPC_E_NOT_SPD);
            if (why & 1) grow_candidates(h, b, 2 * (size_t)q.cand.n);
            if (why & 4) {
                h->Up.exact((size_t)std::max(1, h->F.nU) * (((std::min(q.nS, h->capS) + 31) / 32) * 32 + 64));
                ++h->buf_epoch;
            }
            if (why & 24) q.force_sort = true;      // the next iteration takes the sort broad phase
            continue;
        }
        q.force_sort = false;
        // stats of the last iteration
        const int n_pt = d[D_ACNT], n_all = d[D_ACNT + 1];
        pd_ipc_stats &S = q.stats;
        S.n_cand = d[D_STAT + 1];
        S.n_active = n_all;
        S.n_S = q.nS;
        S.alpha_max = s[2];
        S.alpha = s[5];
        S.ls_trials = (int)s[6];
        S.dE = s[7];
        S.flags = (int)s[8];
        const double min_dist = n_all > 0 ? s[12] : 0.0;
        if (n_all > 0 && !(min_dist > 0))
            throw CudaError("non-positive distance in the active set", PD_IPC_E_NONFINITE);
        S.min_dist = min_dist;
        S.kappa = s[16];
        if (!std::isfinite(s[5]) || !std::isfinite(s[9]) || !std::isfinite(s[10]))
            throw CudaError("non-finite value in step", PD_IPC_E_NONFINITE);
        if (h->debug && nb == 1) debug_capture(h, b, n_pt, n_all - n_pt, q.nS);
    }
    if (nb == 1) dump_traces(h, h->seqs[b0]->nS);
}

// ------------------------------------------------------------------ ABI -------------------
// host check of the create-time actuation (the same predicate as k_validate_actuation)
static int validate_actuation(const double *A, size_t nmat, std::string &err) {
    for (size_t t = 0; t < nmat; ++t) {
        const double *a = A + 9 * t;
        double mx = 0, asym = 0;
        for (int k = 0; k < 9; ++k) {
            if (!std::isfinite(a[k])) { err = "non-finite actuation"; return PD_IPC_E_ACTUATION; }
            mx = std::max(mx, std::fabs(a[k]));
        }
        asym = std::max({std::fabs(a[1] - a[3]), std::fabs(a[2] - a[6]), std::fabs(a[5] - a[7])});
        if (asym > 1e-9 * mx) { err = "actuation not symmetric"; return PD_IPC_E_ACTUATION; }
        double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
                     a[2] * (a[3] * a[7] - a[4] * a[6]);
        if (!(det > 0)) { err = "actuation det <= 0"; return PD_IPC_E_ACTUATION; }
    }
    return 0;
}

// A_next of all sequences checked on the device (non-finite / asymmetric / det <= 0) BEFORE any
// sequence ingests it: a rejected call leaves the state untouched.  Host input: one H2D copy into
// a staging buffer; device input (A_on_device): checked in place.
static int stage_actuation(pd_ipc *h, const double *A, bool on_device, std::string &err) {
    const int T = h->T;
    const size_t nm = h->seqs.size() * (size_t)T;
    const double *dA = A;
    if (!on_device) {
        h->A9stage.ensure(9 * nm);
        CK(cudaMemcpyAsync(h->A9stage.p, A, sizeof(double) * 9 * nm, cudaMemcpyHostToDevice, h->st));
        dA = h->A9stage.p;
    }
    h->aflag.ensure(1);
    CK(dev_zero(h->aflag.p, sizeof(int), h->st));
    launch_validate_actuation(dA, nm, h->aflag.p, h->st);
    int bits = 0;
    CK(cudaMemcpyAsync(&bits, h->aflag.p, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (bits & 1) { err = "non-finite actuation"; return PD_IPC_E_ACTUATION; }
    if (bits & 2) { err = "actuation not symmetric"; return PD_IPC_E_ACTUATION; }
    if (bits & 4) { err = "actuation det <= 0"; return PD_IPC_E_ACTUATION; }
    for (size_t sq = 0; sq < h->seqs.size(); ++sq)
        launch_ingest_actuation(dA + 9 * (size_t)T * sq, h->A6((int)sq), T, h->st);
    return 0;
}

// Intersection-free check of a state (SURVEY.md 8(b) E_INTERSECTING; 8(c) O0 rest-state check):
// (1) no surface edge strictly crosses a surface triangle (host, uniform grid), (2) every
// non-incident PT / EE pair closer than d_hat has a positive distance (device: exact sort broad
// phase + the canonical narrow phase, host-checked).  xd: the state on the device; x: the same
// state on the host [n][3].  Uses the handle's contact work buffers (not on the timed path).
static int check_intersection_free(pd_ipc *h, int b, const double4 *xd, const double *x, std::string &why) {
    if (h->Nt == 0) return 0;
    const long long nx = surface_edge_triangle_crossings(h->hm, x);
    if (nx > 0) {
        why = "intersecting state: " + std::to_string(nx) + " surface edge-triangle crossings";
        return PD_IPC_E_INTERSECTING;
    }
    // sequence b's surface, candidate list and counters are the scratch (its next iteration
    // starts with a static broad phase)
    launch_surface(h->Wp.p, h->Wc.p, h->Wv.p, xd, h->Ns, h->s(b), h->st);
    Seq &q = *h->seqs[b];
    const bool fs = q.force_sort;
    q.force_sort = true;             // exact and host-checked: this is a validation path
    int *ccnt = h->dint(b) + D_CCNT;
    broad_phase(h, b, nullptr, 0.5 * h->dh * 1.01, ccnt, h->dint(b) + D_HOVF);
    q.force_sort = fs;
    launch_narrow(q.cand.p, ccnt, (int)q.cand.n, h->s(b), h->tris.p, h->edges.p, h->Nt, h->Ne, h->dh2,
                  h->flag.p, h->ctype.p, h->cd2.p, nullptr, h->st);
    int cc[2];
    sync_read_ints(h, cc, ccnt, 2);
    std::vector<double> d2(cc[1]);
    if (cc[1]) CK(cudaMemcpy(d2.data(), h->cd2.p, sizeof(double) * cc[1], cudaMemcpyDeviceToHost));
    for (double v : d2)
        if (!(v > 0)) {
            why = "intersecting state: a surface pair at distance <= 0";
            return PD_IPC_E_INTERSECTING;
        }
    return 0;
}

extern "C" {

int pd_ipc_create(const pd_ipc_mesh *mesh, const double *rest_pos, const double *A, double d_hat,
                  double kappa, const pd_ipc_options *opt, pd_ipc **out) {
    if (out) *out = nullptr;
    if (!mesh || !rest_pos || !A || !out) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    if (!(d_hat > 0) || !(kappa > 0)) return fail(nullptr, PD_IPC_E_ARG, "d_hat and kappa must be > 0");
    std::unique_ptr<pd_ipc> h(new pd_ipc());
    pd_ipc_options o{};
    o.n_seq = 1;
    o.device = 0;
    o.ls_max_halvings = 30;
    o.accd_max_iters = 10000;
    o.A_on_device = 0;
    o.max_pairs = 0;
    o.accd_s = 0.1;
    if (opt) {
        o = *opt;
        if (o.n_seq <= 0) o.n_seq = 1;
        if (o.ls_max_halvings <= 0) o.ls_max_halvings = 30;
        if (o.accd_max_iters <= 0) o.accd_max_iters = 10000;
        if (!(o.accd_s > 0 && o.accd_s < 1)) o.accd_s = 0.1;
    }
    if (o.reduced_backend < 0 || o.reduced_backend > 4) return fail(nullptr, PD_IPC_E_ARG, "reduced_backend must be 0..4");
    if (o.ls_energy != 0 && o.ls_energy != 1) return fail(nullptr, PD_IPC_E_ARG, "ls_energy must be 0 or 1");
    if (!(o.kappa_adapt_eps >= 0)) return fail(nullptr, PD_IPC_E_ARG, "kappa_adapt_eps must be >= 0");
    if (!(o.kappa_max > 0)) o.kappa_max = 100.0 * kappa;
    h->opt = o;
    h->dh = d_hat;
    h->kappa = kappa;
    h->dh2 = d_hat * d_hat;
    std::string err;
    int rc = build_host_mesh(mesh->n_verts, mesh->n_tets, mesh->tets, mesh->n_fixed, mesh->fixed,
                             rest_pos, mesh->n_surf_verts, mesh->n_surf_tris, mesh->surf_tris,
                             mesh->embed_tet, mesh->embed_w, h->hm, err);
    if (rc) return fail(nullptr, rc, err);
    rc = validate_actuation(A, (size_t)o.n_seq * mesh->n_tets, err);
    if (rc) return fail(nullptr, rc, err);
    rc = factorize(h->hm, h->hf, err);
    if (rc) return fail(nullptr, rc, err);
    try {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
            return fail(nullptr, PD_IPC_E_CUDA, "no CUDA device");
        if (o.device < 0 || o.device >= ndev) return fail(nullptr, PD_IPC_E_ARG, "bad device ordinal");
        CK(cudaSetDevice(o.device));
        h->device = o.device;
        const int bw_tiles = (o.n_seq + kBwSeqs - 1) / kBwSeqs;   // backward solve: one launch, all sequences
        CK(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, o.device));
        CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&h->st3, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->ev_fork3, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_join3, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_S, cudaEventDisableTiming));
        h->tm.init();
        h->kt.init();
        if (const char *ng = std::getenv("PDIPC_NO_GRAPH")) h->graphs = !(ng[0] == '1');
        if (const char *tl = std::getenv("PDIPC_TIMELINE")) h->kt.timeline = tl[0] == '1';
        if (const char *sc = std::getenv("PDIPC_SIDE_CTAS")) {
            h->side_ctas = std::max(1, std::atoi(sc));
            h->side_env = true;
        }
        if (const char *tp = std::getenv("PDIPC_TRACE")) {
            h->trace_file = std::fopen(tp, "wb");
            h->schur_file = std::fopen((std::string(tp) + ".schur").c_str(), "wb");
        }
        contact_init();
        trisolve_init();
        elastic_init(o.device);
        schur_init(o.device);
        HostMesh &m = h->hm;
        HostFactor &f = h->hf;
        h->n = m.n;
        h->T = m.T;
        h->nf = m.nf;
        h->Ns = m.Ns;
        h->Nt = m.Nt;
        h->Ne = m.Ne;
        // mesh SoA
        {
            std::vector<double> Bs(9 * (size_t)m.T);
            for (int t = 0; t < m.T; ++t)
                for (int k = 0; k < 9; ++k) Bs[(size_t)k * m.T + t] = m.B[9 * (size_t)t + k];
            h->B_.upload(Bs.data(), Bs.size());
            h->w.upload(m.w.data(), m.w.size());
            h->tets.upload(reinterpret_cast<const int4 *>(m.tets.data()), m.T);
        }
        h->inc_ptr.upload(m.inc_ptr.data(), m.inc_ptr.size());
        h->inc.upload(m.inc.data(), std::max<size_t>(m.inc.size(), 1));
        h->q2v.upload(m.q2v.data(), m.q2v.size());
        h->v2q.upload(m.v2q.data(), m.v2q.size());
        h->Wp.upload(m.W_ptr.data(), m.W_ptr.size());
        h->Wc.upload(m.W_col.data(), std::max<size_t>(m.W_col.size(), 1));
        h->Wv.upload(m.W_val.data(), std::max<size_t>(m.W_val.size(), 1));
        h->WTp.upload(m.WT_ptr.data(), m.WT_ptr.size());
        h->WTr.upload(m.WT_row.data(), std::max<size_t>(m.WT_row.size(), 1));
        h->WTv.upload(m.WT_val.data(), std::max<size_t>(m.WT_val.size(), 1));
        h->tris.upload(m.tris.data(), std::max<size_t>(m.tris.size(), 1));
        h->edges.upload(m.edges.data(), std::max<size_t>(m.edges.size(), 1));
        // factor
        h->f_c0.upload(f.sn_c0.data(), f.sn_c0.size());
        h->f_rowptr.upload(f.sn_rowptr.data(), f.sn_rowptr.size());
        h->f_rows.upload(f.sn_rows.data(), f.sn_rows.size());
        h->f_parent.upload(f.sn_parent.data(), f.sn_parent.size());
        h->f_seg_ptr.upload(f.seg_ptr.data(), f.seg_ptr.size());
        h->f_seg_d.upload(f.seg_d.data(), std::max<size_t>(f.seg_d.size(), 1));
        h->f_seg_klo.upload(f.seg_klo.data(), std::max<size_t>(f.seg_klo.size(), 1));
        h->f_seg_khi.upload(f.seg_khi.data(), std::max<size_t>(f.seg_khi.size(), 1));
        h->f_fd.upload(f.sn_fd.data(), f.sn_fd.size());
        h->f_col2sn.upload(f.col2sn.data(), f.col2sn.size());
        {
            std::vector<long long> vp(f.sn_valptr.begin(), f.sn_valptr.end());
            h->f_valptr.upload(vp.data(), vp.size());
        }
        h->f_L.upload(f.Q.data(), f.Q.size());
        {   // etree path of every supernode (itself first, then its ancestors): y_S column walks
            std::vector<int> pp(f.nsn + 1, 0), ps;
            for (int s = 0; s < f.nsn; ++s) {
                for (int t = s; t >= 0; t = f.sn_parent[t]) ps.push_back(t);
                pp[s + 1] = (int)ps.size();
            }
            h->f_path_ptr.upload(pp.data(), pp.size());
            h->f_path_sn.upload(ps.data(), ps.size());
        }
        {   // Item dispatch orders (list scheduling on the elimination tree).  Forward: by
            // decreasing cost-to-root (a child always precedes its parent), so the items on the
            // longest chains start first.  Backward: by decreasing height (a parent precedes
            // its children).  cost(s) = its row blocks.
            const int nsn = f.nsn;
            std::vector<int> nbk(nsn);
            std::vector<double> ctr(nsn, 0.0), hgt(nsn, 0.0);
            for (int s = 0; s < nsn; ++s)
                nbk[s] = (f.sn_rowptr[s + 1] - f.sn_rowptr[s] + kSolveRB - 1) / kSolveRB;
            for (int s = nsn - 1; s >= 0; --s)    // parents have larger postorder indices
                ctr[s] = nbk[s] + (f.sn_parent[s] >= 0 ? ctr[f.sn_parent[s]] : 0.0);
            for (int s = 0; s < nsn; ++s) {
                hgt[s] += nbk[s];
                if (f.sn_parent[s] >= 0) hgt[f.sn_parent[s]] = std::max(hgt[f.sn_parent[s]], hgt[s]);
            }
            std::vector<int> ford(nsn), bord(nsn);
            for (int s = 0; s < nsn; ++s) ford[s] = bord[s] = s;
            std::stable_sort(ford.begin(), ford.end(), [&](int a, int b) { return ctr[a] > ctr[b]; });
            std::stable_sort(bord.begin(), bord.end(), [&](int a, int b) { return hgt[a] > hgt[b]; });
            h->f_ford.upload(ford.data(), ford.size());
            h->f_bord.upload(bord.data(), bord.size());
            std::vector<int2> items;
            std::vector<int> pbase(nsn);
            int nblk = 0;
            for (int s : bord) {
                pbase[s] = nblk;
                nblk += nbk[s];
                for (int b = 0; b < nbk[s]; ++b) items.push_back(make_int2(s, b));
            }
            h->f_bw_items.upload(items.data(), items.size());
            h->f_bw_pbase.upload(pbase.data(), pbase.size());
            h->F.bw_nitems = (int)items.size();
            h->F.bw_nblocks = nblk;
            h->bw_P.exact((size_t)nblk * 128 * 32 * bw_tiles);   // kTS_W x kBwCols partials per row block and tile
            h->bw_cnt.exact((size_t)f.nsn * bw_tiles);
        }
        h->f_uoff.upload(f.uoff.data(), f.uoff.size());
        h->f_urow_sn.upload(f.urow_sn.data(), f.urow_sn.size());
        h->f_rc_ptr.upload(f.rc_ptr.data(), f.rc_ptr.size());
        h->f_rc_idx.upload(f.rc_idx.data(), f.rc_idx.size());
        {   // (U row, owner child) per extend-add source
            std::vector<int2> src(f.rc_idx.size());
            for (size_t j = 0; j < src.size(); ++j) src[j] = make_int2(f.rc_idx[j], f.urow_sn[f.rc_idx[j]]);
            h->f_rc_src.upload(src.data(), src.size());
        }
        h->f_urel.upload(f.urel.data(), f.urel.size());
        h->f_ch_ptr.upload(f.ch_ptr.data(), f.ch_ptr.size());
        h->f_ch.upload(f.ch.data(), f.ch.size());
        {
            std::vector<long long> dp(f.dinv_ptr.begin(), f.dinv_ptr.end());
            h->f_dinv_ptr.upload(dp.data(), dp.size());
        }
        h->f_dinv.upload(f.dinv.data(), f.dinv.size());
        h->Ug.exact(4 * (size_t)std::max(1, f.uoff[f.nsn]));
        h->Ug2.exact(4 * (size_t)std::max(1, f.uoff[f.nsn]) * std::max(1, o.n_seq));
        h->iscr2.exact(scan_scratch_ints(f.nsn + 1) + 64);
        DevFactor &F = h->F;
        F.uoff = h->f_uoff.p; F.urow_sn = h->f_urow_sn.p; F.rc_ptr = h->f_rc_ptr.p; F.rc_idx = h->f_rc_idx.p;
        F.rc_src = h->f_rc_src.p;
        F.dinv_ptr = h->f_dinv_ptr.p; F.dinv = h->f_dinv.p; F.nU = f.uoff[f.nsn];
        F.urel = h->f_urel.p; F.ch_ptr = h->f_ch_ptr.p; F.ch = h->f_ch.p;
        F.nf = f.nf; F.nsn = f.nsn;
        F.sn_c0 = h->f_c0.p; F.sn_rowptr = h->f_rowptr.p; F.sn_rows = h->f_rows.p; F.sn_parent = h->f_parent.p;
        F.sn_valptr = h->f_valptr.p; F.Q = h->f_L.p;
        F.bw_items = h->f_bw_items.p; F.bw_pbase = h->f_bw_pbase.p; F.ford = h->f_ford.p;
        F.path_ptr = h->f_path_ptr.p; F.path_sn = h->f_path_sn.p; F.bord = h->f_bord.p;
        F.seg_ptr = h->f_seg_ptr.p; F.seg_d = h->f_seg_d.p; F.seg_klo = h->f_seg_klo.p; F.seg_khi = h->f_seg_khi.p;
        F.sn_fd = h->f_fd.p; F.col2sn = h->f_col2sn.p;
        // contact capacity: S is a subset of the free vertices in the W support (n2)
        {
            std::vector<char> sup(m.nf, 0);
            int n2 = 0;
            for (size_t k = 0; k < m.W_col.size(); ++k) {
                int qv = m.v2q[m.W_col[k]];
                if (qv >= 0 && !sup[qv]) { sup[qv] = 1; ++n2; }
            }
            h->capS = std::max(1, std::min(n2, 6144));
        }
        h->ldv = ((h->capS + 31) / 32) * 32;
        const int nf = m.nf;
        // sequences: host state + batched device arrays [B][...]
        const int Bq = o.n_seq;
        h->B = Bq;
        {
            std::vector<double4> x4((size_t)m.n * Bq);
            for (int sq = 0; sq < Bq; ++sq)
                for (int v = 0; v < m.n; ++v)
                    x4[(size_t)sq * m.n + v] =
                        make_double4(rest_pos[3 * v], rest_pos[3 * v + 1], rest_pos[3 * v + 2], 0.0);
            h->x_all.upload(x4.data(), x4.size());
        }
        h->A6_all.exact(6 * (size_t)m.T * Bq);
        h->fc_all.exact(12 * (size_t)m.T * Bq);
        h->gel_all.exact((size_t)nf * Bq);
        h->G_all.exact(4 * (size_t)nf * Bq);
        h->Yw_all.exact(4 * (size_t)nf * Bq);
        h->Z_all.exact(4 * (size_t)nf * Bq);
        h->dx_all.exact((size_t)m.n * Bq);
        CK(cudaMemset(h->dx_all.p, 0, sizeof(double4) * m.n * Bq));   // fixed vertices keep dx = 0
        h->s_all.exact((size_t)std::max(1, m.Ns) * Bq);
        h->ds_all.exact((size_t)std::max(1, m.Ns) * Bq);
        h->dscal_all.exact((size_t)S_STRIDE * Bq);
        h->dint_all.exact((size_t)D_STRIDE * Bq);
        CK(cudaMemset(h->dscal_all.p, 0, sizeof(double) * S_STRIDE * Bq));   // flags / counters start cleared
        {   // per-sequence kappa (constant unless adaptive) and the previous min active d^2 (+inf)
            std::vector<double> kk(2 * (size_t)Bq);
            for (int sq = 0; sq < Bq; ++sq) {
                kk[2 * sq] = kappa;
                kk[2 * sq + 1] = HUGE_VAL;
            }
            CK(cudaMemcpy2D(h->dscal_all.p + 16, S_STRIDE * sizeof(double), kk.data(), 2 * sizeof(double),
                            2 * sizeof(double), Bq, cudaMemcpyHostToDevice));
        }
        CK(cudaMemset(h->dint_all.p, 0, sizeof(int) * D_STRIDE * Bq));
        const size_t cap_cand = o.max_pairs > 0 ? (size_t)o.max_pairs
                                                : std::max<size_t>(1 << 16, 16 * (size_t)(m.Ns + m.Ne));
        for (int sq = 0; sq < Bq; ++sq) {
            std::unique_ptr<Seq> sp(new Seq());
            std::memset(&sp->stats, 0, sizeof(sp->stats));
            sp->cand.exact(2 * cap_cand);
            h->seqs.push_back(std::move(sp));
        }
        h->ts_lo2.exact(f.nsn);
        h->ts_hi2.exact(f.nsn);
        h->ts_cnt2.exact(f.nsn + 1);
        h->ts_ptr2.exact(f.nsn + 1);
        h->ts_rem2.exact(f.nsn);
        h->ticket2.exact(4);
        CK(cudaMemset(h->ticket2.p, 0, 4 * sizeof(int)));
        h->mark.exact(nf + 1);
        // per-system Schur buffers: group 0 now, more groups once the backend is known
        auto alloc_sys = [&](pd_ipc::SysBufs &g) {
            g.spos.exact(nf + 1);
            g.qS.exact(nf + 1);
            g.Tt.exact(2 * 64 * 64);                 // P1 pivot inverses, double-buffered
            if (m.Nt > 0) {
                const int cS = h->capS;
                g.gcS.exact(3 * (size_t)cS + 3);
                g.Bc.exact((size_t)9 * cS * cS);
                g.Bh.exact((size_t)9 * cS * cS);
                g.Bl.exact((size_t)9 * cS * cS);
                g.tbits.exact(((size_t)cS * cS + 31) / 32);
                g.tlist.exact((size_t)cS * (cS + 1) / 2);
                g.tcnt.exact(1);
                g.dpos.exact((size_t)cS + 1);
                g.rl.exact(64);
                g.al.exact(64);
                g.uinfo.exact(4);
                CK(cudaMemset(g.uinfo.p, 0, 4 * sizeof(int)));
                CK(cudaMemset(g.Bc.p, 0, g.Bc.n * sizeof(double)));
                CK(cudaMemset(g.Bh.p, 0, g.Bh.n * sizeof(long long)));
                CK(cudaMemset(g.Bl.p, 0, g.Bl.n * sizeof(long long)));
                CK(cudaMemset(g.tbits.p, 0, g.tbits.n * sizeof(unsigned)));
                CK(cudaMemset(g.tcnt.p, 0, sizeof(int)));
                g.Sh.exact((size_t)(3 * cS + 1) * ((3 * cS + 8 + 1) & ~1));
                // large systems: Li tiles [nt+1][64][64]; small: D blocks [nt+1][512] + X tiles [nt][64][64]
                g.Lstore.exact((size_t)((3 * cS + 1 + 63) / 64 + 1) * (64 * 64 + 512));
                g.U.exact((size_t)2 * (cS + 64) * 64);   // P1 sweep panels, double-buffered
                g.yS.exact(3 * (size_t)cS);
                g.rhs.exact(3 * (size_t)cS);
                g.u.exact(3 * (size_t)cS);
                g.tv.exact(3 * (size_t)cS);
            }
        };
        h->sys.resize(1);
        alloc_sys(h->sys[0]);
        h->ts_lo.exact(f.nsn);
        h->ts_hi.exact(f.nsn);
        h->ts_cnt.exact(f.nsn + 1);
        h->ts_ptr.exact(f.nsn + 1);
        h->ts_rem.exact(f.nsn);
        h->ts_done.exact((size_t)f.nsn * bw_tiles);
        h->ticket.exact(4);
        CK(cudaMemset(h->ticket.p, 0, 4 * sizeof(int)));
        // pre-size the per-pair buffers so that no allocation happens inside the iteration
        // (an allocation synchronises the device); they still grow on demand.  Active pairs <=
        // candidates: same capacity, no overflow check needed
        ensure_pair_buffers(h.get(), 2 * cap_cand);
        if (m.Nt > 0) {
            h->blo.exact((size_t)m.Ns + m.Nt + m.Ne);
            h->bhi.exact((size_t)m.Ns + m.Nt + m.Ne);
            h->qcnt.exact((size_t)m.Ns + m.Ne + 1);
            h->qoff.exact((size_t)m.Ns + m.Ne + 1);
            h->qlist.exact((size_t)(m.Ns + m.Ne) * hash_query_cap());
            h->gsq.exact(6 * (size_t)m.Ns + 6);
        }
        h->lspart.exact((size_t)ls_round_width() * ls_blocks());
        if (h->opt.ls_energy == 1) h->tepart.exact((size_t)ls_round_width() * ls_te_blocks(h->T));
        h->iscr.ensure(std::max({radix_scratch_ints((int)(2 * cap_cand)), scan_scratch_ints(nf + 1),
                                 scan_scratch_ints(f.nsn + 1)}) + 1024);
        {
            unsigned M = 1024;
            while (M < 16u * (unsigned)std::max(m.Nt, m.Ne)) M <<= 1;
            h->hmask = M - 1;
            h->hcnt.exact(2 * (size_t)(M + 1));
            h->hstart.exact(2 * (size_t)(M + 1) + 1);
            h->hent.exact(64 * (size_t)std::max(1, m.Nt + m.Ne));
            h->iscr.ensure(scan_scratch_ints(2 * (M + 1)) + scan_scratch_ints(m.Ns + m.Ne + 1) + 1024);
        }
        h->cell0 = std::max(m.mean_edge, 2.0 * d_hat);
        if (m.Nt > 0) {
            const int cS = h->capS;
            h->ldh = (3 * cS + 8 + 1) & ~1;   // even: 16-byte aligned rows (cp.async 16 B)
            h->ldk = (cS + 1) & ~1;           // even: 16-byte aligned rows of K / Sigma_s
            h->Up.exact((size_t)std::max(1, f.uoff[f.nsn]) * (((cS + 31) / 32) * 32));
        }
        h->part.exact(std::max<size_t>(4096, (size_t)(m.T + 255) / 256 + (nf + 255) / 256 + 64));
        std::vector<int> Rq;   // region R: factor positions of the W-supported free vertices, sorted
        {
            std::vector<char> sup(m.nf, 0);
            for (size_t k = 0; k < m.W_col.size(); ++k) {
                const int qv = m.v2q[m.W_col[k]];
                if (qv >= 0) sup[qv] = 1;
            }
            for (int qv = 0; qv < m.nf; ++qv)
                if (sup[qv]) Rq.push_back(qv);
            h->n2 = (int)Rq.size();
            // reduced-solve backend: 1 panel, 2 gather, 0 auto (gather for regions of >= 1024
            // vertices: there the panel and K_s = V_s^T V_s dominate an iteration whenever S changes)
            const int be = o.reduced_backend;
            const bool want = be == 2 || be == 4 || (be == 0 && h->n2 >= 1024);
            h->gather = m.Nt > 0 && want && h->n2 <= h->capS;
            h->region = h->gather && be == 4;
            if (h->region) h->Rq_dev.upload(Rq.data(), Rq.size());
            h->pcg = m.Nt > 0 && be == 3;
            // batched Schur: with the gather backend and several sequences, 4 systems per launch
            // (the grid split in proportion to their work: the systems' serial panel chains overlap
            // each other's updates; C4 2 / 3 / 4 / 6 / 8 systems: 70.7 / 71.9 / 72.3 / 71.7 / 70.3
            // it/s, profiles/schur_split_r02.txt)
            h->nsysb = (h->gather && Bq > 1) ? std::min(Bq, 4) : 1;
            if (const char *sbv = std::getenv("PDIPC_SCHUR_BATCH"))
                h->nsysb = std::max(1, std::min(std::min(Bq, (int)kMaxSchurSys), std::atoi(sbv)));
            if (!h->gather) h->nsysb = 1;                  // (panel mode: split-K sums depend on the grid)
            h->sys.resize(h->nsysb);
            for (int g = 1; g < h->nsysb; ++g) alloc_sys(h->sys[g]);
            if (h->pcg) {
                for (auto *bf : {&h->cg_r, &h->cg_p, &h->cg_z, &h->cg_q, &h->cg_t, &h->cg_f, &h->cg_R})
                    bf->exact(4 * (size_t)nf);
                h->cg_part.exact(3 * (size_t)cg_partials());
                CK(cudaMallocHost(&h->cg_rr_host, sizeof(double)));
            }
        }
        {   // reuse slots (V_s, K_s / -Sigma_s and the S they belong to): one per sequence when 40 %
            // of the free HBM holds them, else fewer, shared round-robin (the bit-exact key check
            // keeps sharing exact; a shared slot only reuses less often)
            const size_t vbytes = m.Nt > 0 ? (h->gather ? 0 : (size_t)nf * h->ldv * 8) + (size_t)h->capS * h->capS * 8 +
                                                 (size_t)(nf + 1) * 4
                                           : 256;
            size_t fr = 0, tot = 0;
            CK(cudaMemGetInfo(&fr, &tot));
            const size_t fit = std::max<size_t>(1, (size_t)(0.4 * (double)fr) / std::max<size_t>(vbytes, 1));
            h->nslots = m.Nt > 0 ? (int)std::min<size_t>((size_t)Bq, fit) : 1;
            if (const char *ns = std::getenv("PDIPC_REUSE_SLOTS")) h->nslots = std::max(1, std::min(Bq, std::atoi(ns)));
            h->V_slot.resize(h->nslots);
            h->K_slot.resize(h->nslots);
            h->qS_slot.resize(h->nslots);
            for (int r = 0; r < h->nslots; ++r) {
                h->V_slot[r].exact(m.Nt > 0 && !h->gather ? (size_t)nf * h->ldv : 32);
                h->K_slot[r].exact(m.Nt > 0 ? (size_t)h->capS * h->ldk : 1);
                h->qS_slot[r].exact(nf + 1);
            }
            h->nS_slot.exact(h->nslots);
            CK(cudaMemset(h->nS_slot.p, 0, sizeof(int) * h->nslots));
            h->nupd_slot.exact(h->nslots);
            CK(cudaMemset(h->nupd_slot.p, 0, sizeof(int) * h->nslots));
            for (int sq = 0; sq < Bq; ++sq) h->seqs[sq]->slot = sq % h->nslots;
        }
        if (h->gather) {
            // one-time (untimed) precompute of G2 = (L^-1)_RR = V_R^T V_R with V_R = L^-1 Pi E_R: the
            // panel forward solve and the K-only Schur phase with S = R (the
            // paper's precomputed Sigma^-1 of the collision region)
            const int n2 = h->n2;
            std::vector<int> rp(nf, -1);
            for (int i = 0; i < n2; ++i) rp[Rq[i]] = i;
            h->rpos.upload(rp.data(), rp.size());
            CK(cudaMemcpy(h->sys[0].qS.p, Rq.data(), sizeof(int) * n2, cudaMemcpyHostToDevice));
            int *nS_dev = h->sys[0].spos.p + nf;
            CK(cudaMemcpy(nS_dev, &n2, sizeof(int), cudaMemcpyHostToDevice));
            DBuf<double> Vtmp;
            Vtmp.exact((size_t)nf * h->ldv);
            h->G2.exact((size_t)n2 * n2);
            int *zero = h->ticket2.p + 2, *flags = h->dint(0) + D_CAP;
            launch_ts_plan(F, h->sys[0].qS.p, nS_dev, h->capS, zero, (long long)h->Up.n, flags, 2, 0, h->ts_lo.p, h->ts_hi.p,
                           h->ts_cnt.p, h->ts_rem.p, h->ts_ptr.p, h->ticket.p, h->st);
            launch_forward_solve(F, h->ts_lo.p, h->ts_hi.p, h->ts_ptr.p, h->sys[0].qS.p, h->ts_rem.p, h->ticket.p, nullptr,
                                 nullptr, Vtmp.p, h->ldv, nullptr, h->Up.p, nS_dev, h->capS, 0, 0, 0, 0, h->nsm,
                                 nullptr, h->st);
            CK((cudaError_t)launch_schur(F, Vtmp.p, h->ldv, h->Yw(0), h->sys[0].gcS.p, h->sys[0].qS.p, h->ts_lo.p, h->ts_hi.p,
                                         nS_dev, h->capS, h->G2.p, n2, h->sys[0].Bc.p, 3 * h->capS, h->sys[0].Sh.p, h->ldh,
                                         h->sys[0].Lstore.p, h->sys[0].Tt.p, h->sys[0].U.p, h->sys[0].yS.p, h->sys[0].rhs.p, h->sys[0].u.p, h->sys[0].tv.p, h->Z(0),
                                         h->dint(0) + D_INFO, zero, nullptr, 0, kSchurKOnly, nullptr, 0, nullptr,
                                         nullptr, h->st));
            CK(cudaStreamSynchronize(h->st));
            int cap_flags = 0;
            CK(cudaMemcpy(&cap_flags, flags, sizeof(int), cudaMemcpyDeviceToHost));
            if (cap_flags) throw CudaError("region precompute: panel capacity", PD_IPC_E_CAPACITY);
            CK(cudaMemset(flags, 0, sizeof(int)));
            Vtmp.release();
            h->Yel_all.exact(4 * (size_t)nf * Bq);
            h->Zf_all.exact(4 * (size_t)nf * Bq);
            h->bw_P2.exact(h->bw_P.n);
            h->ts_done2.exact((size_t)f.nsn * bw_tiles);
            h->bw_cnt2.exact((size_t)f.nsn * bw_tiles);
        }
        // second contact-stage scratch set: the sequences of a batched Schur group run their contact
        // stages concurrently (PDIPC_SERIAL_CONTACT=1 keeps them on one stream)
        const char *sc_env = std::getenv("PDIPC_SERIAL_CONTACT");
        // (the members of a group must own distinct reuse slots: their k_same_S run concurrently)
        if (m.Nt > 0 && h->gather && !h->pcg && h->nsysb >= 2 && h->nslots >= h->nsysb &&
            !(sc_env && sc_env[0] == '1')) {
            h->alt = new ContactAlt();
            ContactAlt &a = *h->alt;
#define PD_ALT_ALLOC(b) a.b.exact(h->b.n);
            PD_ALT_ALLOC(cand_tmp) PD_ALT_ALLOC(flag) PD_ALT_ALLOC(pos) PD_ALT_ALLOC(ctype) PD_ALT_ALLOC(cd2)
            PD_ALT_ALLOC(iscr) PD_ALT_ALLOC(akeys) PD_ALT_ALLOC(atype) PD_ALT_ALLOC(ad2) PD_ALT_ALLOC(grad)
            PD_ALT_ALLOC(Hp) PD_ALT_ALLOC(dist) PD_ALT_ALLOC(ids) PD_ALT_ALLOC(blo) PD_ALT_ALLOC(bhi)
            PD_ALT_ALLOC(qcnt) PD_ALT_ALLOC(qoff) PD_ALT_ALLOC(qlist) PD_ALT_ALLOC(gsq) PD_ALT_ALLOC(hcnt)
            PD_ALT_ALLOC(hstart) PD_ALT_ALLOC(hent) PD_ALT_ALLOC(mark) PD_ALT_ALLOC(part) PD_ALT_ALLOC(b0)
            PD_ALT_ALLOC(lspart)
            if (h->tepart.n) PD_ALT_ALLOC(tepart)
#undef PD_ALT_ALLOC
            CK(cudaStreamCreateWithFlags(&a.st, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&a.st3, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&a.ev_fork3, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&a.ev_join3, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&a.ev_S, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&h->ev_cfork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&h->ev_cjoin, cudaEventDisableTiming));
        }
        {
            std::string e2;
            if (stage_actuation(h.get(), A, false, e2)) throw CudaError(e2.c_str(), PD_IPC_E_ACTUATION);
        }
        CK(cudaStreamSynchronize(h->st));
        {   // the rest state must be intersection-free (SURVEY.md 8(b) E_INTERSECTING at create)
            std::string why;
            const int rc = check_intersection_free(h.get(), 0, h->x(0), rest_pos, why);
            if (rc) {
                pd_ipc_destroy(h.release());
                return fail(nullptr, rc, why);
            }
        }
    } catch (const CudaError &e) {
        int code = e.code;
        std::string msg = e.what();
        if (h->st) cudaStreamDestroy(h->st);
        return fail(nullptr, code, msg);
    }
    *out = h.release();
    return PD_IPC_OK;
}

int pd_ipc_step(pd_ipc *h, const double *A_next, int32_t n_iters, pd_ipc_stats *stats) {
    if (!h) return fail(nullptr, PD_IPC_E_ARG, "NULL handle");
    if (n_iters < 0) return fail(h, PD_IPC_E_ARG, "n_iters < 0");
    try {
        CK(cudaSetDevice(h->device));
        if (A_next) {
            std::string err;
            const int rc = stage_actuation(h, A_next, h->opt.A_on_device != 0, err);
            if (rc) return fail(h, rc, err);
        }
        // Sequences advance in lockstep (one batch = k iterations of all of them, k * B <= kSlotCap);
        // with debug capture on, each sequence runs alone so the shared contact buffers hold its
        // data.  A sequence whose iteration aborted (capacity / hash overflow: buffers grown, or the
        // sort broad phase next) runs its remaining iterations of the batch alone.
        const int Bq = h->B;
        std::vector<std::array<double, 6>> ms(Bq, std::array<double, 6>{0, 0, 0, 0, 0, 0});
        for (int b = 0; b < Bq; ++b) {
            Seq &sq = *h->seqs[b];
            sq.stats.sigma_reused = 0;
            sq.stats.sigma_updated = 0;
            sq.cg_iters = 0;
            sq.converged = false;
            sq.iters_applied = 0;
            CK(dev_zero(h->dint(b) + D_CONV, 3 * sizeof(int), h->st));        // convergence state
            CK(dev_zero(h->dscal(b) + 13, sizeof(double), h->st));
        }
        const bool conv = h->opt.conv_tol > 0;
        auto run_alone = [&](int b, int iters) {
            int done = 0, tries = 0;
            std::vector<int> ap;
            std::vector<std::array<double, 6>> m1(1, std::array<double, 6>{0, 0, 0, 0, 0, 0});
            while (done < iters && !(conv && h->seqs[b]->converged)) {
                const int k = std::min(iters - done, kMaxBatch);
                run_lockstep(h, b, 1, k, ap, m1);
                done += ap[0];
                if (ap[0] < k && ++tries > 8)            // buffers grown / sort path: redo the rest
                    throw CudaError("capacity growth did not converge", PD_IPC_E_CAPACITY);
            }
            for (int c = 0; c < 6; ++c) ms[b][c] += m1[0][c];
        };
        if (h->debug || Bq == 1) {
            for (int b = 0; b < Bq; ++b) run_alone(b, n_iters);
        } else {
            const int kb = std::max(1, std::min(kMaxBatch, kSlotCap / Bq));
            std::vector<int> ap;
            for (int done = 0; done < n_iters;) {
                const int k = std::min(n_iters - done, kb);
                run_lockstep(h, 0, Bq, k, ap, ms);
                for (int b = 0; b < Bq; ++b)
                    if (ap[b] < k) run_alone(b, k - ap[b]);
                done += k;
                bool all = conv;
                for (int b = 0; b < Bq && all; ++b) all = h->seqs[b]->converged;
                if (all) break;                    // every sequence converged (conv_tol)
            }
        }
        for (int b = 0; b < Bq; ++b) {
            h->seqs[b]->stats.cg_iters = h->seqs[b]->cg_iters;
            h->seqs[b]->stats.iters = h->seqs[b]->iters_applied;
            for (int c = 0; c < 6; ++c) h->seqs[b]->stats.ms[c] = ms[b][c];
        }
        if (stats)
            for (size_t sq = 0; sq < h->seqs.size(); ++sq) stats[sq] = h->seqs[sq]->stats;
    } catch (const CudaError &e) {
        return fail(h, e.code, e.what());
    }
    return PD_IPC_OK;
}

int pd_ipc_positions(const pd_ipc *h, int32_t seq, double *out) {
    if (!h || !out) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    if (seq < 0 || seq >= (int)h->seqs.size()) return fail(const_cast<pd_ipc *>(h), PD_IPC_E_ARG, "bad sequence");
    try {
        std::vector<double4> x4(h->n);
        CK(cudaMemcpy(x4.data(), const_cast<pd_ipc *>(h)->x(seq), sizeof(double4) * h->n, cudaMemcpyDeviceToHost));
        for (int v = 0; v < h->n; ++v) {
            out[3 * v] = x4[v].x;
            out[3 * v + 1] = x4[v].y;
            out[3 * v + 2] = x4[v].z;
        }
    } catch (const CudaError &e) {
        return fail(const_cast<pd_ipc *>(h), e.code, e.what());
    }
    return PD_IPC_OK;
}

void pd_ipc_destroy(pd_ipc *h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    // DBuf members free in their own scope via release; explicit for clarity
    for (auto &g : h->gcache)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    h->tm.destroy();
    h->kt.destroy();
    if (h->trace_file) std::fclose(h->trace_file);
    if (h->schur_file) std::fclose(h->schur_file);
    h->trace.release();
    h->sprof.release();
    if (h->st2) cudaStreamDestroy(h->st2);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->st3) cudaStreamDestroy(h->st3);
    if (h->ev_fork3) cudaEventDestroy(h->ev_fork3);
    if (h->ev_join3) cudaEventDestroy(h->ev_join3);
    if (h->ev_S) cudaEventDestroy(h->ev_S);
    if (h->st) cudaStreamDestroy(h->st);
    if (h->alt) {
        ContactAlt &a = *h->alt;
        if (a.st) cudaStreamDestroy(a.st);
        if (a.st3) cudaStreamDestroy(a.st3);
        for (cudaEvent_t e : {a.ev_fork3, a.ev_join3, a.ev_S})
            if (e) cudaEventDestroy(e);
        for (auto *b : {&a.cand_tmp, &a.akeys}) b->release();
        for (auto *b : {&a.flag, &a.pos, &a.ctype, &a.atype, &a.ids, &a.iscr, &a.mark, &a.hcnt, &a.hstart, &a.hent,
                        &a.qcnt, &a.qoff, &a.qlist})
            b->release();
        for (auto *b : {&a.cd2, &a.ad2, &a.grad, &a.Hp, &a.dist, &a.part, &a.b0, &a.lspart, &a.tepart}) b->release();
        a.blo.release();
        a.bhi.release();
        a.gsq.release();
        delete h->alt;
        h->alt = nullptr;
    }
    if (h->ev_cfork) cudaEventDestroy(h->ev_cfork);
    if (h->ev_cjoin) cudaEventDestroy(h->ev_cjoin);
    auto rel = [](auto &b) { b.release(); };
    rel(h->tets); rel(h->B_); rel(h->w); rel(h->inc_ptr); rel(h->inc); rel(h->q2v); rel(h->v2q);
    rel(h->Wp); rel(h->Wc); rel(h->WTp); rel(h->WTr); rel(h->tris); rel(h->edges); rel(h->Wv); rel(h->WTv);
    rel(h->f_c0); rel(h->f_rowptr); rel(h->f_rows); rel(h->f_parent); rel(h->f_seg_ptr); rel(h->f_seg_d);
    rel(h->f_seg_klo); rel(h->f_seg_khi); rel(h->f_fd); rel(h->f_col2sn); rel(h->f_valptr); rel(h->f_L);
    rel(h->f_dinv_ptr); rel(h->f_dinv); rel(h->Ug); rel(h->Up); rel(h->bw_P); rel(h->f_bw_items); rel(h->f_ford); rel(h->f_bord); rel(h->Ug2); rel(h->f_path_ptr); rel(h->f_path_sn); rel(h->f_rc_src); rel(h->f_bw_pbase); rel(h->bw_cnt); rel(h->f_uoff); rel(h->f_urow_sn);
    rel(h->f_rc_ptr); rel(h->f_rc_idx); rel(h->f_urel); rel(h->f_ch_ptr); rel(h->f_ch);
    for (auto &s : h->seqs) rel(s->cand);
    for (auto &b : h->V_slot) rel(b);
    for (auto &b : h->K_slot) rel(b);
    for (auto &b : h->qS_slot) rel(b);
    rel(h->nS_slot);
    rel(h->nupd_slot);
    rel(h->x_all); rel(h->gel_all); rel(h->dx_all); rel(h->s_all); rel(h->ds_all); rel(h->A6_all); rel(h->p_all);
    rel(h->fc_all); rel(h->G_all); rel(h->Yw_all); rel(h->Z_all); rel(h->dscal_all); rel(h->dint_all);
    rel(h->xstage); rel(h->surf_out); rel(h->A9stage); rel(h->aflag); rel(h->blo);
    for (auto *bf : {&h->cg_r, &h->cg_p, &h->cg_z, &h->cg_q, &h->cg_t, &h->cg_f, &h->cg_R, &h->cg_part}) rel(*bf);
    if (h->cg_rr_host) cudaFreeHost(h->cg_rr_host);
    rel(h->G2); rel(h->Rq_dev); rel(h->Yel_all); rel(h->Zf_all); rel(h->bw_P2); rel(h->rpos); rel(h->ts_done2); rel(h->bw_cnt2); rel(h->bhi); rel(h->hcnt); rel(h->hstart); rel(h->hent);
    rel(h->qcnt); rel(h->qoff); rel(h->qlist); rel(h->gsq);
    rel(h->cand_tmp); rel(h->akeys); rel(h->flag); rel(h->pos); rel(h->ctype); rel(h->atype); rel(h->ids);
    rel(h->iscr); rel(h->cd2); rel(h->ad2); rel(h->grad); rel(h->Hp); rel(h->dist); rel(h->mark);
    for (auto &g : h->sys) {
        for (auto *bf : {&g.Bc, &g.Sh, &g.gcS, &g.Lstore, &g.U, &g.Tt, &g.yS, &g.rhs, &g.u, &g.tv}) rel(*bf);
        rel(g.Bh);
        rel(g.Bl);
        rel(g.tbits);
        rel(g.tlist);
        rel(g.tcnt);
        rel(g.dpos);
        rel(g.rl);
        rel(g.al);
        rel(g.uinfo);
    }
    for (auto &g : h->sys) { rel(g.qS); rel(g.spos); }
    rel(h->lspart); rel(h->tepart); rel(h->ts_lo);
    rel(h->ts_hi); rel(h->ts_cnt); rel(h->ts_ptr); rel(h->ts_rem); rel(h->ts_done); rel(h->ticket);
    rel(h->part); rel(h->b0);
    delete h;
}

const char *pd_ipc_last_error(const pd_ipc *h) {
    return h ? h->err.c_str() : g_last_error.c_str();
}

int pd_ipc_set_positions(pd_ipc *h, int32_t seq, const double *x) {
    if (!h || !x) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    if (seq < 0 || seq >= (int)h->seqs.size()) return fail(h, PD_IPC_E_ARG, "bad sequence");
    for (int v = 0; v < h->n; ++v)
        if (h->hm.is_fixed[v])
            for (int a = 0; a < 3; ++a)
                if (x[3 * v + a] != h->hm.rest[3 * v + a])
                    return fail(h, PD_IPC_E_ARG, "fixed vertex moved");
    try {
        // the candidate state is staged and checked first; the sequence keeps its state when
        // the check fails
        std::vector<double4> x4(h->n);
        for (int v = 0; v < h->n; ++v) x4[v] = make_double4(x[3 * v], x[3 * v + 1], x[3 * v + 2], 0.0);
        h->xstage.ensure(h->n);
        CK(cudaMemcpy(h->xstage.p, x4.data(), sizeof(double4) * h->n, cudaMemcpyHostToDevice));
        std::string why;
        const int rc = check_intersection_free(h, seq, h->xstage.p, x, why);
        if (rc) return fail(h, rc, why);
        CK(cudaMemcpy(h->x(seq), h->xstage.p, sizeof(double4) * h->n, cudaMemcpyDeviceToDevice));
    } catch (const CudaError &e) {
        return fail(h, e.code, e.what());
    }
    return PD_IPC_OK;
}

int pd_ipc_set_debug(pd_ipc *h, int32_t level) {
    if (!h) return fail(nullptr, PD_IPC_E_ARG, "NULL handle");
    h->debug = level;
    if (level > 0 && !h->p_all.p) {
        try {
            CK(cudaSetDevice(h->device));
            h->p_all.exact(9 * (size_t)h->T * h->B);   // projections of the local step (parity hook)
        } catch (const CudaError &e) {
            return fail(h, e.code, e.what());
        }
    }
    return PD_IPC_OK;
}

int pd_ipc_get_projections(const pd_ipc *h, int32_t seq, double *p) {
    if (!h || !p) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    if (seq < 0 || seq >= (int)h->seqs.size()) return fail(const_cast<pd_ipc *>(h), PD_IPC_E_ARG, "bad sequence");
    if (!h->debug) return fail(const_cast<pd_ipc *>(h), PD_IPC_E_ARG, "enable pd_ipc_set_debug first");
    try {
        std::vector<double> soa(9 * (size_t)h->T);
        CK(cudaMemcpy(soa.data(), h->p_all.p + (size_t)seq * 9 * h->T, sizeof(double) * soa.size(),
                      cudaMemcpyDeviceToHost));
        for (int t = 0; t < h->T; ++t)
            for (int k = 0; k < 9; ++k) p[9 * (size_t)t + k] = soa[(size_t)k * h->T + t];
    } catch (const CudaError &e) {
        return fail(const_cast<pd_ipc *>(h), e.code, e.what());
    }
    return PD_IPC_OK;
}

int pd_ipc_get_pair_terms(const pd_ipc *h, int32_t seq, double *grad, double *Hp, int32_t *n) {
    if (!h || !n) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    if (seq < 0 || seq >= (int)h->seqs.size()) return fail(const_cast<pd_ipc *>(h), PD_IPC_E_ARG, "bad sequence");
    const Seq &q = *h->seqs[seq];
    *n = (int32_t)(q.pgrad.size() / 12);
    if (grad) std::copy(q.pgrad.begin(), q.pgrad.end(), grad);
    if (Hp) std::copy(q.phess.begin(), q.phess.end(), Hp);
    return PD_IPC_OK;
}

int pd_ipc_get_contacts(const pd_ipc *h, int32_t seq, int32_t *pt, int32_t *n_pt, int32_t *ee,
                        int32_t *n_ee, int32_t *S, int32_t *n_S) {
    if (!h || !n_pt || !n_ee || !n_S) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    if (seq < 0 || seq >= (int)h->seqs.size()) return fail(const_cast<pd_ipc *>(h), PD_IPC_E_ARG, "bad sequence");
    const Seq &q = *h->seqs[seq];
    *n_pt = (int32_t)(q.pt.size() / 2);
    *n_ee = (int32_t)(q.ee.size() / 2);
    *n_S = (int32_t)q.S.size();
    if (pt) std::copy(q.pt.begin(), q.pt.end(), pt);
    if (ee) std::copy(q.ee.begin(), q.ee.end(), ee);
    if (S) std::copy(q.S.begin(), q.S.end(), S);
    return PD_IPC_OK;
}

int pd_ipc_get_vector(const pd_ipc *h, int32_t seq, int32_t which, double *out) {
    if (!h || !out) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    if (seq < 0 || seq >= (int)h->seqs.size()) return fail(const_cast<pd_ipc *>(h), PD_IPC_E_ARG, "bad sequence");
    const Seq &q = *h->seqs[seq];
    const std::vector<double> &v = which == 0 ? q.ghat : which == 1 ? q.dx : q.gel;
    if (v.size() != 3 * (size_t)h->n) return fail(const_cast<pd_ipc *>(h), PD_IPC_E_ARG, "not available (debug off?)");
    std::copy(v.begin(), v.end(), out);
    return PD_IPC_OK;
}

const char *pd_ipc_build_info(void) {
    return "pd_ipc sm_100a build " __DATE__ " " __TIME__;
}

int pd_ipc_set_timing(pd_ipc *h, int32_t on) {
    if (!h) return fail(nullptr, PD_IPC_E_ARG, "NULL handle");
    h->kt.on = on != 0;
    h->kt.mask = on < 0 ? (unsigned)(-(long long)on) : ~0u;
    return PD_IPC_OK;
}

int pd_ipc_kernel_times(pd_ipc *h, double *ms, int64_t *counts, int32_t reset) {
    if (!h) return fail(nullptr, PD_IPC_E_ARG, "NULL handle");
    for (int k = 0; k < K_NUM; ++k) {
        if (ms) ms[k] = h->kt.ms[k];
        if (counts) counts[k] = h->kt.cnt[k];
        if (reset) { h->kt.ms[k] = 0; h->kt.cnt[k] = 0; }
    }
    return K_NUM;
}

const char *pd_ipc_kernel_name(int32_t id) {
    return (id >= 0 && id < K_NUM) ? kKernelNames[id] : "";
}

int64_t pd_ipc_launch_count(void) { return pdipc::launch_count(); }

int pd_ipc_get_info(const pd_ipc *h, int64_t *info, int32_t n) {
    if (!h || !info) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    const int64_t v[17] = {h->n, h->T, h->nf, h->Ns, h->Nt, h->Ne, h->hf.nsn, h->hf.nnzL, h->hf.depth,
                           h->capS, h->nslots, h->B, h->F.bw_nblocks, h->F.nU, h->pcg ? 3 : h->region ? 4 : h->gather ? 2 : 1, h->n2,
                           h->nsysb};
    const int k = std::max(0, std::min<int>(n, 17));
    for (int i = 0; i < k; ++i) info[i] = v[i];
    return k;
}

int pd_ipc_build_embedding(const int32_t *tets, int32_t n_tets, const double *rest_pos, int32_t n_verts,
                           const double *points, int32_t n_points, double tol, int32_t *embed_tet,
                           double *embed_w) {
    std::string err;
    const int rc = build_embedding(n_verts, n_tets, tets, rest_pos, n_points, points, tol > 0 ? tol : 1e-9,
                                   embed_tet, embed_w, err);
    return rc ? fail(nullptr, rc, err) : PD_IPC_OK;
}

int pd_ipc_surface_positions(const pd_ipc *h_, int32_t seq, double *out) {
    pd_ipc *h = const_cast<pd_ipc *>(h_);
    if (!h || !out) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    if (seq < 0 || seq >= (int)h->seqs.size()) return fail(h, PD_IPC_E_ARG, "bad sequence");
    if (h->Ns == 0) return PD_IPC_OK;
    try {
        CK(cudaSetDevice(h->device));
        h->surf_out.ensure(h->Ns);
        launch_surface(h->Wp.p, h->Wc.p, h->Wv.p, h->x(seq), h->Ns, h->surf_out.p, h->st);
        std::vector<double4> s4(h->Ns);
        CK(cudaMemcpyAsync(s4.data(), h->surf_out.p, sizeof(double4) * h->Ns, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        for (int j = 0; j < h->Ns; ++j) {
            out[3 * (size_t)j] = s4[j].x;
            out[3 * (size_t)j + 1] = s4[j].y;
            out[3 * (size_t)j + 2] = s4[j].z;
        }
    } catch (const CudaError &e) {
        return fail(h, e.code, e.what());
    }
    return PD_IPC_OK;
}

int64_t pd_ipc_debug_crossings(const pd_ipc_mesh *mesh, const double *rest_pos, const double *x) {
    if (!mesh || !rest_pos || !x) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    HostMesh m;
    std::string err;
    int rc = build_host_mesh(mesh->n_verts, mesh->n_tets, mesh->tets, mesh->n_fixed, mesh->fixed, rest_pos,
                             mesh->n_surf_verts, mesh->n_surf_tris, mesh->surf_tris, mesh->embed_tet,
                             mesh->embed_w, m, err);
    if (rc) return fail(nullptr, rc, err);
    return surface_edge_triangle_crossings(m, x);
}

// Host-only debug entry (no GPU needed): runs setup + factorisation and solves L_FF x = b on
// the host with the supernodal factor; reports factor statistics.  Used by CPU tests of the
// setup logic.  b, x: [n_verts] (values on fixed vertices ignored / set to 0).
int pd_ipc_debug_factor_solve(const pd_ipc_mesh *mesh, const double *rest_pos, const double *b,
                              double *x, int64_t *stats /* [nsn, nnzL, max_width, depth] */) {
    if (!mesh || !rest_pos) return fail(nullptr, PD_IPC_E_ARG, "NULL argument");
    HostMesh m;
    HostFactor f;
    std::string err;
    int rc = build_host_mesh(mesh->n_verts, mesh->n_tets, mesh->tets, mesh->n_fixed, mesh->fixed, rest_pos,
                             mesh->n_surf_verts, mesh->n_surf_tris, mesh->surf_tris, mesh->embed_tet,
                             mesh->embed_w, m, err);
    if (rc) return fail(nullptr, rc, err);
    rc = factorize(m, f, err);
    if (rc) return fail(nullptr, rc, err);
    if (stats) {
        stats[0] = f.nsn;
        stats[1] = f.nnzL;
        stats[2] = f.max_width;
        stats[3] = f.depth;
        int64_t maxseg = 0, segrows = 0;
        for (int s = 0; s < f.nsn; ++s) {
            maxseg = std::max<int64_t>(maxseg, f.seg_ptr[s + 1] - f.seg_ptr[s]);
            for (int g = f.seg_ptr[s]; g < f.seg_ptr[s + 1]; ++g) segrows += f.seg_khi[g] - f.seg_klo[g];
        }
        stats[4] = (int64_t)f.seg_d.size();
        stats[5] = maxseg;
        stats[6] = segrows;
        int64_t offrows = 0;
        for (int s = 0; s < f.nsn; ++s)
            offrows += (f.sn_rowptr[s + 1] - f.sn_rowptr[s]) - (f.sn_c0[s + 1] - f.sn_c0[s]);
        stats[7] = offrows;
    }
    if (const char *dump = std::getenv("PDIPC_DUMP_SUPERNODES")) {   // debugging aid
        if (FILE *fp = std::fopen(dump, "w")) {
            for (int s = 0; s < f.nsn; ++s)
                std::fprintf(fp, "%d %d %d %d %d\n", s, f.sn_c0[s], f.sn_c0[s + 1] - f.sn_c0[s],
                             f.sn_rowptr[s + 1] - f.sn_rowptr[s], f.sn_parent[s]);
            std::fclose(fp);
        }
    }
    if (b && x) {
        std::vector<double> y(f.nf);
        for (int q = 0; q < f.nf; ++q) y[q] = b[m.q2v[q]];
        for (int s = 0; s < f.nsn; ++s) {        // forward
            int c0 = f.sn_c0[s], w = f.sn_c0[s + 1] - c0, r0 = f.sn_rowptr[s], nr = f.sn_rowptr[s + 1] - r0;
            const double *L = &f.vals[f.sn_valptr[s]];
            for (int k = 0; k < w; ++k) {
                y[c0 + k] /= L[k + (size_t)k * nr];
                for (int i = k + 1; i < nr; ++i) y[f.sn_rows[r0 + i]] -= L[i + (size_t)k * nr] * y[c0 + k];
            }
        }
        for (int s = f.nsn - 1; s >= 0; --s) {  // backward
            int c0 = f.sn_c0[s], w = f.sn_c0[s + 1] - c0, r0 = f.sn_rowptr[s], nr = f.sn_rowptr[s + 1] - r0;
            const double *L = &f.vals[f.sn_valptr[s]];
            for (int k = w - 1; k >= 0; --k) {
                double acc = y[c0 + k];
                for (int i = k + 1; i < nr; ++i) acc -= L[i + (size_t)k * nr] * y[f.sn_rows[r0 + i]];
                y[c0 + k] = acc / L[k + (size_t)k * nr];
            }
        }
        for (int v = 0; v < m.n; ++v) x[v] = 0.0;
        for (int q = 0; q < f.nf; ++q) x[m.q2v[q]] = y[q];
    }
    return PD_IPC_OK;
}

}  // extern "C"
