// Host-callable launchers of the CUDA kernels (internal to the library).
#pragma once
#include <cuda_runtime.h>
#include <cuda.h>
#include <cstdint>

namespace pdipc {

struct DevFactor {
    int nf = 0, nsn = 0;
    int *sn_c0 = nullptr, *sn_rowptr = nullptr, *sn_rows = nullptr, *sn_parent = nullptr;
    long long *sn_valptr = nullptr;
    double *Q = nullptr;               // per supernode [L_ss^-1; L_off L_ss^-1], layout of L
    const int2 *bw_items = nullptr;    // backward items (s, row block), reverse postorder
    int *bw_pbase = nullptr;           // first partial block of each supernode
    int *ford = nullptr;               // forward dispatch order of the supernodes
    int *bord = nullptr;               // backward dispatch order (parents first)
    int *path_ptr = nullptr, *path_sn = nullptr;   // etree path (self, ancestors) per supernode
    int bw_nitems = 0, bw_nblocks = 0;
    int *seg_ptr = nullptr, *seg_d = nullptr, *seg_klo = nullptr, *seg_khi = nullptr;
    int *sn_fd = nullptr, *col2sn = nullptr;
    int *uoff = nullptr, *urow_sn = nullptr, *rc_ptr = nullptr, *rc_idx = nullptr;
    const int2 *rc_src = nullptr;      // [rc entries] (U row, child supernode owning it)
    int *urel = nullptr, *ch_ptr = nullptr, *ch = nullptr;
    long long *dinv_ptr = nullptr;
    double *dinv = nullptr;
    int nU = 0;
};

long long launch_count();   // prims.cu: kernels launched so far (PDI_LAUNCH)
void add_launches(long long n);   // graph replays account their captured launches

// ---- k_elastic.cu
void launch_set_double(double *p, double v, cudaStream_t st);
// bits of *flag (or-ed): 1 non-finite, 2 asymmetric, 4 det <= 0 (the caller zeroes it)
void launch_validate_actuation(const double *A, size_t nmat, int *flag, cudaStream_t st);
void launch_ingest_actuation(const double *A9, double *A6, int T, cudaStream_t st);
void elastic_init(int device);
// clr (nullable): device ints clr[0..1] and clr[4..7] zeroed by the kernel (the iteration's
// active-pair counts and flags, engine.cu D_ACNT / D_INFO..)
// a1 / a2 over (tet, sequence) for nseq sequences: x [nseq][xs] double4, A6 [nseq][6][T],
// fc [nseq][T][12], p [nseq][9][T], counters clr [nseq][clrs]; g [nseq][nf] double4
void launch_local_step(const int4 *tets, const double4 *x, const double *B, const double *A6,
                       const double *w, int T, double *fc, double *p, int *clr, int nseq, long long xs,
                       int clrs, cudaStream_t st);
void launch_gather_elastic(const int *inc_ptr, const int *inc, const double *fc, int nf,
                           double4 *g, int nseq, long long fcs, cudaStream_t st);
void launch_surface(const int *Wp, const int *Wc, const double *Wv, const double4 *x, int Ns,
                    double4 *s, cudaStream_t st);
int quad_partials(const int4 *tets, const double4 *dx, const double *B, const double *w, int T,
                  double *part, cudaStream_t st);
int gdx_partials(const double4 *g, const double4 *dx, const int *q2v, int nf, double *part,
                 cudaStream_t st);
// gTdx and dx^T H dx block partials in one launch: part[0..nb1) and part[nb1..nb1+nb2)
void elastic_partials(const double4 *g, const double4 *dx, const int *q2v, int nf, const int4 *tets,
                      const double *B, const double *w, int T, double *part, int *nb1, int *nb2,
                      cudaStream_t st);
// cv = [converged, iterations applied, block ticket]; amax scratch; tol <= 0: fixed iteration count
void launch_update(double4 *x, const double4 *dx, const int *q2v, int nf, const double *alpha,
                   const int *flags, int *abort, int it, int *cv, unsigned long long *amax, double tol,
                   cudaStream_t st);
// f3 true-energy line search: block partials pte[h][b] of 1/2 sum w (e_i(alpha_h) - e_i(0)),
// e_i = min_R ||F_i - R A_i||^2, for the round's trials alpha_h = am 2^-(h0+h), h < kh; am = *amin
// in the first round, ls[0] after; a round after acceptance (ls[1] != 0) returns at once.
// Returns the number of blocks (ls_te_blocks(T)).
int launch_ls_true_elastic(const int4 *tets, const double4 *x, const double4 *dx, const double *B, const double *A6,
                           const double *w, int T, const double *amin, const double *ls, int h0, int kh,
                           double *pte, cudaStream_t st);
int ls_te_blocks(int T);
// z [nseq][nf][4] -> dx [nseq][n]; seeds amin[sq * amin_stride] = 1
void launch_scatter_dx(const double *z, const int *q2v, int nf, double4 *dx, double *amin, int nseq, int n,
                       int amin_stride, cudaStream_t st);

// ---- k_trisolve.cu
constexpr int kSolveRB = 64;   // rows of a supernode per solve work item
// mode: bit 0 gradient items, bit 1 panel tiles
// per-iteration plan of a solve (one block): clears rem and ticket[0], item counts, lo/hi,
// item_ptr = exclusive scan of the counts
// nseq: gradient right-hand sides (3 columns each) of a mode-1 solve
int grad_tiles(int nseq);
void launch_ts_plan(const DevFactor &F, const int *qS, const int *nS_ptr, int capS, const int *same_S,
                    long long up_cap, int *flags, int mode, int nseq, int *lo, int *hi, int *cnt, int *rem,
                    int *item_ptr, int *ticket, cudaStream_t st);
void trisolve_init();
void launch_forward_solve(const DevFactor &F, const int *lo, const int *hi, const int *item_ptr,
                          const int *qS, int *rem, int *ticket, const double *G, double *Y, double *V,
                          int ldv, double *Ug, double *Up, const int *nS_ptr, int capS, int with_grad,
                          int nseq, long long gstride, long long ustride,
                          int nsm, unsigned long long *trace, cudaStream_t st, const double *Yadd = nullptr);
// backward solve of nseq sequences' right-hand sides Z[sq][nf][4] (stride zstride) in ONE launch:
// column tiles of kBwSeqs sequences; done / cnt hold ceil(nseq / kBwSeqs) x nsn ints and P that many
// x bw_nblocks x 128 x 32 doubles
constexpr int kBwSeqs = 8;
void launch_backward_solve(const DevFactor &F, int *done, int *cnt, int *ticket, double *P, double *Z,
                           int nseq, long long zstride, int nsm, cudaStream_t st);

// ---- k_pcg.cu (the paper's PCG baseline)
// part: [3][cg_partials()] doubles; host_rr: one double the host reads (r.r of the iteration)
void launch_cg_init(const double *w, double *r, double *p, double *z, int nf, double *part, double *host_rr,
                    cudaStream_t st);
void launch_cg_bmul(const double *Bc, int ldb, const int *qS, const int *nS, int capS, const double *t,
                    double *out, int nf, cudaStream_t st);
// CG iteration it >= 0 after f = L^-1 E_S B-check (L^-T p)_S: q = p + f, alpha, z, r, beta, p
void launch_cg_update(const double *f, double *p, double *q, double *z, double *r, int nf, double *part, int it,
                      double *host_rr, cudaStream_t st);
void launch_cg_finish(const double *z, double *Z, int nf, cudaStream_t st);
int cg_partials();

// ---- k_schur.cu (fused cooperative dense Schur step, a9)
constexpr int kMaxPanels = 1024;   // [0, 512): P3 panel barriers, [512, 1024): P4 tile flags
struct SchurArgs {
    // panel
    const double *V;
    int ldv;
    const double *G;            // w_el = L^{-1} Pi g_el [nf][4] (elastic part only)
    const double *gc;           // [3|S|] contact part of the gradient on S (Pi g = Pi g_el + E_S gc)
    const int *qS, *col2sn, *sn_c0, *sn_parent, *lo, *hi, *path_ptr, *path_sn;
    int nsn, nf, capS;
    const int *nS_ptr;          // |S| (device); clamped to capS
    // dense buffers
    double *K;                  // [capS][ldk] -> Sigma_s
    int ldk;
    const double *Bc;           // [3capS][ldb]
    int ldb;
    double *Sh;                 // [3capS+1][ldh] augmented Sigma-hat
    int ldh;
    double *Lstore;             // [nt][64][64] inverses of the diagonal factor tiles
    double *LP;                 // [2][kLPTiles][64][64] panel scratch of the small-system P3
    double *T;                  // 64x64 scratch (sweep pivot inverse)
    double *U;                  // sweep panel [capS+64][64]
    double *yS, *y, *u, *t;     // [3capS]
    double *Kpart;              // [grid][1152] split-K partial tiles (+ y_S partials)
    double *Z;                  // [nf][4]
    int *info;
    const int *same;            // 1: S unchanged, K holds the previous -Sigma_s (reuse it)
    unsigned long long *prof;   // optional phase timestamps (PDIPC_TRACE), [1024]
    int pw_min;                 // systems of >= pw_min 64-tiles take the large-system path
    // reduced-solve backend (the paper's precomputed-inverse variant):
    //   kSchurPanel  : K_s = V_s^T V_s and y_S = -V_s^T w_el from the panel; Z = w_el + V_s (gc + t)
    //   kSchurKOnly  : setup: K = V_s^T V_s only (S = the region R), then return
    //   kSchurGather : K_s = G2[r(S), r(S)] gathered from the precomputed (L^-1)_RR, y_S = rows S of
    //                  the base solve y_el = L^-T L^-1 Pi g_el (y_S = -y_el[S]); output Z = the
    //                  sparse right-hand side E_S (gc + t) (zero off S), solved by the caller
    int mode;
    const double *G2;           // [n2][n2] (L^-1)_RR (gather mode)
    int n2;
    const int *rpos;            // [nf] index of a factor position in R, -1 outside (gather mode)
    const double *Yel;          // [nf][4] y_el (gather mode)
    unsigned *bar;              // [kMaxPanels] group-barrier counters of the large-system P3
    int phase;                  // 0: P0-P5; large systems split over three launches: 1 = P0-P2,
                                // then k_chol_large (P3), then 2 = P4-P5 (small systems: the
                                // phase-1 launch does everything, the others return at once)
    unsigned *gbar;             // barrier counter of the CTA group that runs this system
    int kpw0, ktail;            // first-panel width; tail narrowing divisor (0: off)
    int split_min;              // panels split in two halves while >= split_min tile columns remain right of them
    int kpw;                    // large-system P3 panel width in 64-tiles (PDIPC_SCHUR_KPW, default 10)
    double wu_coef;             // large-system P3 split: work of a trailing 128x64 k=256 update (units of
                                // a 64^3 tile product; PDIPC_SCHUR_WU, default 3.5)
    // TMA descriptor of Sh ([3capS+1] rows x ldh doubles, boxes of 16 doubles x 64 rows, 128-byte
    // swizzle): the large-system trailing updates stream their k chunks with tensor copies.
    // Encoded on the host by schur_args(); read by the kernel from the (grid-constant) parameter.
    alignas(64) CUtensorMap tmap_sh;
    // low-rank Sigma_s update instead of the full sweep (gather backend; null: never): uinfo =
    // {update?, |removed|, |added|, n_old}, dpos = old position of each new position (-1 added),
    // rl / al = removed old / added new positions (ordered, <= 64 each)
    const int *uinfo, *dpos, *rl, *al;
    // bits of the 3 x 3 blocks of B-check that are nonzero this iteration (both triangles; row a
    // at bits [a capS, a capS + capS)): t = B u by row scans (null: dense rows)
    const unsigned *tbits;
};
// Several systems (sequences) per launch: the grid splits into nsys equal CTA groups, group g
// running system s[g] with group barriers (the batched variable-n_c Schur step of SURVEY 8(e)).
constexpr int kMaxSchurSys = 8;
struct SchurBatch {
    SchurArgs s[kMaxSchurSys];
    int nsys;
    double wexp;                  // the CTA split weighs system g by m_g^wexp (default 2.5)
};
SchurArgs schur_args(const DevFactor &F, const double *V, int ldv, const double *G, const double *gc,
                     const int *qS, const int *lo, const int *hi, const int *nS, int capS, double *K, int ldk,
                     const double *Bc, int ldb, double *Sh, int ldh, double *Lstore, double *T, double *U,
                     double *yS, double *y, double *u, double *t, double *Z, int *info, const int *same_S,
                     unsigned long long *prof, int large_min_tiles, int mode, const double *G2, int n2,
                     const int *rpos, const double *Yel);
// nsys systems in one cooperative launch (nsys <= kMaxSchurSys; the grid splits into groups in
// proportion to the systems' work m^wexp)
int launch_schur_batch(const SchurArgs *sys, int nsys, cudaStream_t st);
void schur_init(int device);
int launch_schur(const DevFactor &F, const double *V, int ldv, const double *G, const double *gc,
                 const int *qS,
                 const int *lo, const int *hi, const int *nS, int capS, double *K, int ldk, const double *Bc, int ldb,
                 double *Sh, int ldh, double *Lstore, double *T, double *U, double *yS, double *y, double *u,
                 double *t, double *Z, int *info, const int *same_S, unsigned long long *prof,
                 int large_min_tiles, int mode, const double *G2, int n2, const int *rpos, const double *Yel,
                 cudaStream_t st);
void note_launch();
constexpr int kSchurPanel = 0, kSchurKOnly = 1, kSchurGather = 2;   // launch_schur modes

// ---- k_contact.cu
void contact_init();
void launch_boxes(const double4 *s, const double4 *ds, const int *tris, const int *edges, int Ns,
                  int Nt, int Ne, double infl, double4 *lo, double4 *hi, double *ext,
                  cudaStream_t st);
void launch_hash_insert(const double4 *lo, const double4 *hi, int Ns, int Nt, int Ne,
                        const double *cell, unsigned mask, int *cnt, const int *start, int *entries,
                        int cap_entries, int *ovf, cudaStream_t st);
void launch_hash_query(const double4 *lo, const double4 *hi, int a0, int na, int b0, int nB,
                       const double *cell, unsigned mask, const int *start, const int *entries,
                       int is_pt, const int *tris, const int *edges, unsigned long long *out,
                       int *count, int cap, cudaStream_t st);
int hash_query_cap();
void launch_hash_query_warp(const double4 *lo, const double4 *hi, int Ns, int Nt, int Ne,
                            const double *cell, unsigned mask, const int *start, const int *entries,
                            const int *tris, const int *edges, int *cnt, int *qlist, int *ovf,
                            cudaStream_t st);
void launch_hash_emit(int Ns, int Nt, int Ne, const int *cnt, const int *off, const int *qlist,
                      unsigned long long *out, int cap, int *ccnt, int *flags, cudaStream_t st);
// Device-resident counts: ccnt = [npt, ntot] candidate keys (PT block then EE block), acnt =
// [n_pt, n_all] active pairs, nS = |S|; `cap` sizes the (grid-stride) launch only.
void launch_narrow(const unsigned long long *keys, const int *ccnt, int cap, const double4 *s,
                   const int *tris, const int *edges, int Nt, int Ne, double dh2, int *flag,
                   int *type, double *d2, int *stat, cudaStream_t st);
void launch_compact_active(const unsigned long long *keys, const int *ccnt, int cap, const int *flag,
                           const int *pos, const int *type, const double *d2, unsigned long long *akeys,
                           int *atype, double *ad2, int *acnt, cudaStream_t st);
void launch_pair_derivs(const unsigned long long *akeys, const int *atype, const double *ad2,
                        const int *acnt, int cap, const double4 *s, const int *tris, const int *edges,
                        int Nt, int Ne, double dh, const double *kappa, double *grad, double *Hp,
                        double *dist, int *ids, double *dmax, cudaStream_t st);
// f3 adaptive kappa: kd = [kappa, previous min active d^2] of the sequence (see k_contact.cu)
void launch_kappa_update(const double *ad2, const int *acnt, double *kd, double eps2, double kmax, cudaStream_t st);
void launch_mark_S(const int *ids, const int *acnt, int cap, const int *Wp, const int *Wc, const int *v2q,
                   int *mark, cudaStream_t st);
void launch_mark_list(const int *list, int n, int *mark, cudaStream_t st);   // mark[list[i]] = 1
// S against the slot's previous S: bit-identical (reuse), or the plan of a low-rank Sigma_s update
// (dpos / rl / al / uinfo, gather backend, allow_upd) -- see k_contact.cu
void launch_same_S(const int *qS, const int *nS_ptr, int *qS_prev, int *nS_prev, int *same, int cap,
                   bool enabled, int *flags, int *reused, int *dpos, int *rl, int *al, int *uinfo, int *nupd,
                   bool allow_upd, int *updated, cudaStream_t st);
void launch_accum_grad_fx(const int *ids, const int *acnt, int cap, const double *grad, const double *dmax,
                          long long *gsq, cudaStream_t st);
void launch_accum_bc_fx(const int *ids, const int *acnt, int cap, const int *Wp, const int *Wc, const double *Wv,
                        const int *v2q, const int *sidx, const double *Hp, const double *dmax,
                        long long *Bq, long long *Bl, int ldb, int capS, unsigned *tbits, int *tlist, int *tcnt,
                        cudaStream_t st);
// B-check blocks: clear the previous use's blocks in the dense double B-check; convert the listed
// fixed-point blocks (and their mirrors), re-zeroing the accumulators and the block bits
void launch_bc_clear(double *Bc, int ld, int capS, const int *tlist, const int *tcnt, unsigned *tbits,
                     cudaStream_t st);
void launch_bc_convert(long long *Bh, long long *Bl, double *Bc, int ld, int capS, const int *tlist, const int *tcnt,
                       unsigned *tbits, const double *dmax, const int *acnt, cudaStream_t st);
void launch_grad_pullback_fx(const double4 *g_el, const int *WTp, const int *WTr, const double *WTv,
                             const long long *gsq, const double *dmax, const int *acnt, int nf, double *G,
                             cudaStream_t st);
void launch_grad_pullback(const double4 *g_el, const int *WTp, const int *WTr, const double *WTv,
                          const double4 *gs, int nf, double *G, cudaStream_t st);
void launch_broad_prep(double *ext, double cell0, double cap, int *ovf, int *hcnt, int n, cudaStream_t st);
void launch_contact_prep(int *mark, int nf, long long *gsq, int ngsq, double *dmax, cudaStream_t st);
void launch_gather_gc(const int *qS, const int *nS, int capS, const int *WTp, const int *WTr, const double *WTv,
                      const long long *gsq, const double *dmax, const int *acnt, double *gc, cudaStream_t st);
void launch_accd(const unsigned long long *keys, const int *ccnt, int cap, const double4 *s,
                 const int *tris, const int *edges, int Nt, int Ne, const double4 *ds, double s_gap,
                 int max_iters, double *amin, cudaStream_t st);
int ls_blocks();
// round h0 == 0 also sums the elastic partials pg[0..ng), pq[0..nq) into scal and takes
// alpha_max from *amin
void launch_ls_round(const unsigned long long *keys, const int *ccnt, const double4 *s, const int *tris,
                     const int *edges, int Nt, int Ne, const double4 *ds, double dh, double *b0, double *ls,
                     int h0, double *part, double *scal, const double *kappa, int hmax, double *out,
                     int *done_ctr, const double *pg, int ng, const double *pq, int nq, const double *amin,
                     const double *pte, int nte, cudaStream_t st);
int ls_round_width();
int ls_round_width_at(int h0);   // trial alphas of the round starting at h0 (1, 8, 22)
int ls_round_next(int h0);   // first halving of the round after the one starting at h0

}  // namespace pdipc
