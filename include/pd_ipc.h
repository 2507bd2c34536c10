/*
 * pd_ipc.h -- C ABI of the B200 (sm_100a) PD+IPC iteration library.
 *
 * What it computes: Algorithm 1 of arXiv 2312.02999 ("Efficient Incremental Potential Contact
 * for Actuated Face Simulation"): per iteration the projective-dynamics local
 * step (Eq. 1), the elastic gradient (Eq. 2/4, :82-98), the IPC barrier
 * terms on the embedded surface s = W x (Eq. 3, :88-93 and :143), the contact global step
 * (Eq. 4, :95-98) solved exactly through the contact-reduced Schur complement onto the
 * contact vertex set S (section 3, :129-247, generalised as SURVEY.md 8(a) a7-a9), CCD
 * (:99, :115), the backtracking line search (:116) and the update x <- x + alpha dx (:117,
 * read with the current iterate).  Readings of silent points are SURVEY.md
 * section 8(c) Z1-Z28 and are listed in DESIGN.md.
 *
 * Conventions.  All reals are float64 (meters); all indices int32, zero-based; host-side
 * arrays are row-major AoS ("[n][3]" means n consecutive xyz triples).  Every entry point
 * returns 0 on success or a negative PD_IPC_E_* code; no C++ exception crosses the ABI.
 * The caller owns all inputs; the library deep-copies what it needs at create time, so the
 * caller may free its arrays as soon as a call returns.  The handle owns every device buffer
 * and the factorisation.  A handle is single-threaded: use one handle per process and GPU.
 * There is no CPU fallback: every iteration runs in the library's CUDA kernels, and create
 * fails with PD_IPC_E_CUDA when no CUDA device is present.
 */
#ifndef PD_IPC_H
#define PD_IPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes; SPEC.md:48,57,101-102,115,166,285,294 name the cases */
#define PD_IPC_OK              0
#define PD_IPC_E_ARG          -1  /* NULL pointer, d_hat <= 0, kappa <= 0, bad sequence index */
#define PD_IPC_E_MESH         -2  /* index out of range, det(D_m) <= 0, W row not convex /
                                     not summing to 1 within 1e-12, degenerate surface tri */
#define PD_IPC_E_ACTUATION    -3  /* |A - A^T|max > 1e-9 |A|max, det A <= 0, or non-finite  */
#define PD_IPC_E_NOT_SPD      -4  /* no fixed vertices, or the Cholesky factorisation failed */
#define PD_IPC_E_INTERSECTING -5  /* at create / set_positions: a surface pair at distance <= 0
                                     or a surface edge crossing a surface triangle            */
#define PD_IPC_E_NONFINITE    -6  /* a NaN/Inf appeared during step (state = last iterate)   */
#define PD_IPC_E_CUDA         -7  /* CUDA runtime error or no device                         */
#define PD_IPC_E_OOM          -8  /* device or host allocation failed                        */
#define PD_IPC_E_CAPACITY     -9  /* a contact buffer capacity was exceeded                  */

/* stats flags */
#define PD_IPC_FLAG_STALL      1  /* line search found no decrease in 31 trials: alpha = 0   */

typedef struct pd_ipc pd_ipc;     /* opaque handle */

/* Mesh + collision proxy ("mesh" of the north_star create call).
 *   tets      [n_tets][4]  vertex ids; each tet must have det(D_m) > 0
 *   fixed     [n_fixed]    Dirichlet vertex ids, n_fixed >= 1
 *   surf_tris [n_surf_tris][3] surface-vertex ids of the embedded surface
 *   embed_tet [n_surf_verts]   host tet of each surface vertex
 *   embed_w   [n_surf_verts][4] barycentric weights in [0,1] summing to 1: row j of W
 *   n_surf_tris == 0 means pure PD (no contact). */
typedef struct {
    int32_t n_verts, n_tets;
    const int32_t *tets;
    int32_t n_fixed;
    const int32_t *fixed;
    int32_t n_surf_verts, n_surf_tris;
    const int32_t *surf_tris;
    const int32_t *embed_tet;
    const double *embed_w;
} pd_ipc_mesh;

typedef struct {
    int32_t n_seq;            /* independent actuation sequences sharing the mesh (>= 1)      */
    int32_t device;           /* CUDA device ordinal                                          */
    int32_t ls_max_halvings;  /* line search halvings (default 30)                 */
    int32_t accd_max_iters;   /* ACCD iteration cap (default 10000)                */
    int32_t A_on_device;      /* 0: A_next is host memory; 1: device pointer [n_seq][T][9]    */
    int32_t max_pairs;        /* capacity of candidate / active pair buffers (0 = auto)       */
    double accd_s;            /* ACCD gap fraction s_gap (default 0.1)                        */
    int32_t no_sigma_reuse;   /* 0 (default): V_s, K_s and Sigma_s = K_s^{-1} -- functions of S
                                 and the constant factor only -- are recomputed only when S
                                 differs bit for bit from the S they were last computed for;
                                 1: recompute them every iteration                             */
    int32_t no_cand_reuse;    /* 0 (default): iterations after the first of a pd_ipc_step batch
                                 take the previous iteration's SWEPT candidate list (boxes over
                                 [s, s + W dx] inflated by d_hat) as the candidate set of the
                                 narrow phase: x_new = x + alpha dx with alpha in [0, 1], so every
                                 pair closer than d_hat at x_new is in it (the
                                 active set C is then identical, the narrow phase being exact);
                                 1: static broad phase every iteration                         */
    int32_t debug_flags;      /* test hooks that force rarely taken paths (0 = none):
                                 PD_IPC_DBG_LARGE_SCHUR  every dense Schur system takes the
                                   large-system (panel, all-CTA back substitution) path;
                                 PD_IPC_DBG_SORT_BROAD   every broad phase takes the sort path;
                                 PD_IPC_DBG_TINY_HASH    the hash broad phase overflows, so each
                                   iteration is redone on the sort path;
                                 PD_IPC_DBG_NO_SIGMA_UPDATE  Sigma_s is swept afresh whenever S
                                   changed (the exact reuse for an unchanged S stays)           */
    int32_t reduced_backend;  /* how K_s = (L^-1)_SS and the contact part of dx are formed (the
                                 same dx either way):
                                 1 panel: V_s = L^-1 Pi E_S per S (reach-limited forward solve),
                                   K_s = V_s^T V_s, dx from w_el + V_s (gc + t);
                                 2 gather: G2 = (L^-1)_RR over the region R of W-supported free
                                   vertices precomputed at create (the paper's precomputed inverse
                                   of the collision region), K_s gathered from
                                   G2, y_S from the base solve, dx from one more forward solve of
                                   the S-sparse right-hand side;
                                 3 pcg: the paper's baseline (Eq. 5, SURVEY 8(f)
                                   f2) -- conjugate gradients on L^-1 H-hat L^-T, preconditioned by
                                   the prefactorised L, to a relative residual cg_tol (iterative:
                                   dx agrees with the direct backends to ~cg_tol x conditioning);
                                 4 region: the paper's literal prescribed-region solve (PAPER.md
                                   :161-198 Eq. 6-8, SURVEY 8(f) f1 "square"): the gather backend
                                   with S = R, the whole W-supported region, every iteration --
                                   Sigma_R = ((L^-1)_RR)^-1 computed once, the dense 3|R| x 3|R|
                                   Sigma-hat refactorised each iteration (3.7x the K-Schur form's
                                   largest system at C3); the same dx;
                                 0 auto: gather when |R| >= 1024, else panel
                                 (any other value: PD_IPC_E_ARG)                                 */
    double cg_tol;            /* pcg: relative residual ||r|| / ||r0|| to stop at (<= 0: 1e-12)  */
    int32_t cg_max_iters;     /* pcg: iteration cap per solve (<= 0: 10000)                      */
    double conv_tol;          /* > 0: "while not converged" (SURVEY Z10 option): a
                                 sequence stops at the first iteration whose update moves no free
                                 vertex by conv_tol or more (max |alpha dx|, meters); its later
                                 iterations in the call leave it untouched.  0: the fixed n_iters
                                 count (the default, used by every benchmark)                   */
    int32_t ls_energy;        /* line-search energy: 0 (default) the
                                 surrogate E_p with p fixed at x (a closed-form quadratic elastic
                                 part); 1 the true energy E = 1/2 sum w_i min_R ||F_i - R A_i||^2
                                 (Eq. 1), R re-minimised (polar of F_i A_i) at every
                                 trial alpha, summed as per-element differences e_i(x + alpha dx)
                                 - e_i(x)                                                        */
    double kappa_adapt_eps;   /* > 0: adaptive barrier stiffness ("kappa is
                                 initialized according to the average stiffness ... and
                                 adaptively adjusted", IPC's rule, reading R-kappa):
                                 before the barrier terms of an iteration, kappa of the sequence
                                 doubles (capped at kappa_max) when the minimum active-pair
                                 distance is below kappa_adapt_eps (meters) and smaller than the
                                 previous iteration's; kappa persists across step calls.
                                 0 (default): kappa fixed                                        */
    double kappa_max;         /* cap of the adaptive kappa (<= 0: 100 x the create-time kappa)   */
} pd_ipc_options;

#define PD_IPC_DBG_LARGE_SCHUR 1
#define PD_IPC_DBG_SORT_BROAD  2
#define PD_IPC_DBG_TINY_HASH   4
#define PD_IPC_DBG_NO_SIGMA_UPDATE 8   /* full Sigma_s sweep whenever S changed (no low-rank update) */

/* Per sequence, describing the LAST iteration of the last pd_ipc_step call. */
typedef struct {
    int32_t iters;            /* iterations applied in the last step call (n_iters, or fewer
                                 when conv_tol stopped the sequence)                          */
    int32_t n_cand;           /* broad-phase candidates (static, d_hat-inflated)              */
    int32_t n_active;         /* |C| = PT + EE active pairs                                   */
    int32_t n_S;              /* n_c = |S|                                                     */
    int32_t ls_trials;        /* line-search energy evaluations                               */
    int32_t flags;            /* PD_IPC_FLAG_*                                                 */
    double alpha_max;         /* alpha_m from CCD                                              */
    double alpha;             /* accepted step                                                 */
    double dE;                /* line-search energy change at the accepted step (surrogate, or
                                 true energy with ls_energy = 1)                                 */
    double min_dist;          /* min active-pair distance before the step (0 if C empty)      */
    double ms[6];             /* device time per stage over the call: IPC, G-Step, CCD, LS,
                                 Misc, total (Table 1 categories)               */
    int32_t sigma_reused;     /* iterations of the call that reused V_s, K_s, Sigma_s (S same) */
    int32_t cg_iters;         /* pcg backend: CG iterations summed over the call's iterations    */
    int32_t sigma_updated;    /* iterations of the call that updated Sigma_s = K_s^-1 by low-rank
                                 steps (S changed by <= 64 removed / added vertices, gather
                                 backend) instead of the full sweep; exact in exact arithmetic, a
                                 full sweep every 32 consecutive updates bounds the rounding drift */
    double kappa;             /* barrier stiffness of the last iteration (= the create-time kappa
                                 unless kappa_adapt_eps > 0)                                      */
} pd_ipc_stats;

/* Create a solver: validates the mesh, computes B_i = D_m^{-1} and w_i = det/6, assembles the
 * scalar PD matrix L (H = L (x) I3, Eq. 2), eliminates the Dirichlet vertices, orders and
 * factorises L_FF = L L^T on the host (supernodal Cholesky, the paper's one-time
 * prefactorisation), uploads everything to HBM.  rest_pos [n_verts][3] is both
 * the rest shape and the start state x_0 of every sequence.  A [n_seq][n_tets][9] row-major
 * symmetric actuation of the first frame.  d_hat > 0 activation distance (d_0,
 * PAPER.md:88), kappa > 0 barrier stiffness.  opt may be NULL (defaults).
 * On failure *out is NULL and the return code says why (pd_ipc_last_error(NULL) has text). */
int pd_ipc_create(const pd_ipc_mesh *mesh, const double *rest_pos, const double *A,
                  double d_hat, double kappa, const pd_ipc_options *opt, pd_ipc **out);

/* Run n_iters iterations of Algorithm 1 (a fixed count) on every sequence.
 * A_next: NULL keeps the current actuation; otherwise [n_seq][n_tets][9] on the host, or on
 * the device when opt.A_on_device = 1.  Every matrix of every sequence is checked
 * on the device before any sequence takes the new actuation: a non-finite, asymmetric
 * (|A - A^T|max > 1e-9 |A|max) or det <= 0 matrix fails the call with PD_IPC_E_ACTUATION and the
 * state is unchanged.  stats: NULL or [n_seq].  Blocks until done. */
int pd_ipc_step(pd_ipc *h, const double *A_next, int32_t n_iters, pd_ipc_stats *stats);

/* Copy positions x of sequence seq (all vertices, fixed ones at rest) into out [n_verts][3]
 * ("Output x_{t+1}": the state after the last pd_ipc_step).  out is caller
 * owned.  PD_IPC_E_ARG on a NULL argument or a bad sequence index, PD_IPC_E_CUDA on a copy
 * failure. */
int pd_ipc_positions(const pd_ipc *h, int32_t seq, double *out);

/* Free the handle and every device buffer it owns (factor, mesh, states, work buffers).
 * NULL is a no-op.  (Setup/teardown of the one-time prefactorisation.) */
void pd_ipc_destroy(pd_ipc *h);

/* Last error text: owned by h, or by a thread-local buffer when h == NULL. */
const char *pd_ipc_last_error(const pd_ipc *h);

/* ---- parity / test hooks (not on the timed path) ------------------------------------- */

/* Overwrite the state of sequence seq with x [n_verts][3] (fixed vertices must be at rest;
 * PAPER.md:103-104 "Input x_t").  The state is staged and checked first: every non-incident
 * surface pair closer than d_hat must have a positive distance and no surface edge may cross a
 * surface triangle; on PD_IPC_E_INTERSECTING the sequence keeps its state. */
int pd_ipc_set_positions(pd_ipc *h, int32_t seq, const double *x);

/* p_i = vec_rowmajor(R_i A_i) of the last local step of sequence seq: [n_tets][9]. */
int pd_ipc_get_projections(const pd_ipc *h, int32_t seq, double *p);

/* Active set C and contact vertex set S of the last iteration of sequence seq.
 * pt [n_pt][2] = (surface vertex j, triangle f) sorted; ee [n_ee][2] = (edge e, edge e'),
 * e < e', sorted, edges = unique sorted surface-vertex pairs in lexicographic order;
 * S [n_S] sorted simulation vertex ids.  Pass NULL arrays to query the sizes only. */
int pd_ipc_get_contacts(const pd_ipc *h, int32_t seq, int32_t *pt, int32_t *n_pt,
                        int32_t *ee, int32_t *n_ee, int32_t *S, int32_t *n_S);

/* Per active pair of the last iteration (order of pd_ipc_get_contacts: PT pairs, then EE
 * pairs): grad [n][12] = kappa b'(d) grad d over the pair's 4 surface
 * points (p, a, b, c) / (a, b, c, d), Hp [n][78] = packed upper triangle (row-major i <= j) of
 * the PSD-projected 12x12 Hessian H+.  Pass NULL arrays to query n only.  Needs debug >= 1. */
int pd_ipc_get_pair_terms(const pd_ipc *h, int32_t seq, double *grad, double *Hp, int32_t *n);

/* Vectors of the last iteration of sequence seq, each [n_verts][3] with zeros on fixed
 * vertices: which = 0 g-hat (elastic + barrier gradient), 1 dx, 2 elastic gradient only. */
int pd_ipc_get_vector(const pd_ipc *h, int32_t seq, int32_t which, double *out);

/* Debug level: 1 makes step keep p, C, S, g-hat, dx of the last iteration for the hooks
 * above (extra device->host copies; off by default and on the timed path never used). */
int pd_ipc_set_debug(pd_ipc *h, int32_t level);

/* Host-only check of the one-time setup (no GPU used): builds L_FF, orders and factorises it,
 * and solves L_FF x = b on the host with the supernodal factor.  b, x: [n_verts] (entries on
 * fixed vertices ignored / returned as 0).  stats (may be NULL): [supernodes, nnz(L), max
 * supernode width, supernodal etree depth]. */
int pd_ipc_debug_factor_solve(const pd_ipc_mesh *mesh, const double *rest_pos, const double *b,
                              double *x, int64_t *stats);

/* Embedding construction (host only, no GPU used): the rows of W for points
 * embedded in the rest tet mesh -- the paper's embedded collision surface s = W x (PAPER.md:143,
 * :161; SPEC.md:53-61 build_embedding).  For point q, embed_tet[q] = the LOWEST-index tet whose
 * barycentric coordinates of the point are all >= -tol (SPEC.md:81 tie rule: a point on a shared
 * face goes to the lower-index tet), embed_w[q][4] = those coordinates with the negatives clamped
 * to 0 and renormalised to sum 1 (so W rest_pos reproduces the point within ~tol x edge length).
 * tets [n_tets][4], rest_pos [n_verts][3], points [n_points][3]; outputs caller-owned
 * embed_tet [n_points], embed_w [n_points][4] (the pd_ipc_mesh fields).  tol <= 0 means 1e-9.
 * PD_IPC_E_ARG on NULL / negative sizes, PD_IPC_E_MESH on a bad tet index or a point outside
 * every tet. */
int pd_ipc_build_embedding(const int32_t *tets, int32_t n_tets, const double *rest_pos, int32_t n_verts,
                           const double *points, int32_t n_points, double tol, int32_t *embed_tet,
                           double *embed_w);

/* Export of the embedded surface of sequence seq at its current positions: out [n_surf_verts][3]
 * = s = W x, computed on the device.  Caller-owned out. */
int pd_ipc_surface_positions(const pd_ipc *h, int32_t seq, double *out);

/* Host-only check (no GPU used): number of (surface edge, surface triangle) pairs sharing no
 * vertex whose segment strictly crosses the triangle, with the surface at s = W x
 * (PAPER.md:143), x [n_verts][3].  This is the crossing half of the intersection-free check
 * that create and set_positions run (SURVEY.md 8(b) PD_IPC_E_INTERSECTING; 8(c) O0).
 * Returns the count (>= 0) or a negative PD_IPC_E_* code for an invalid mesh. */
int64_t pd_ipc_debug_crossings(const pd_ipc_mesh *mesh, const double *rest_pos, const double *x);

/* Device timing of kernel groups (CUDA events on the library stream around each group, every
 * iteration; on = 1 enables all groups, on < 0 only the groups in the bit mask -on (bit k =
 * group k), on = 0 disables).  pd_ipc_kernel_times copies the accumulated milliseconds and
 * launch counts of the K groups (returns K) into ms[K], counts[K] (either may be NULL) and
 * resets them if reset != 0; pd_ipc_kernel_name(i) names group i (0 = "local_step"). */
int pd_ipc_set_timing(pd_ipc *h, int32_t on);
int pd_ipc_kernel_times(pd_ipc *h, double *ms, int64_t *counts, int32_t reset);
const char *pd_ipc_kernel_name(int32_t id);

/* Sizes of the handle (for measurement reports): info[0..n) of
 *   [n_verts, n_tets, n_free, n_surf_verts, n_surf_tris, n_surf_edges, supernodes, nnz(L),
 *    supernodal etree depth, capS (max |S|), reuse slots, n_seq, backward row blocks, nU,
 *    reduced backend (1 panel, 2 gather, 3 pcg, 4 region), |R|, Schur systems per launch]
 * (nnz(L): the prefactorised PD matrix).  Returns the number of fields written. */
int pd_ipc_get_info(const pd_ipc *h, int64_t *info, int32_t n);

/* Number of CUDA kernels this library has launched in the process so far. */
int64_t pd_ipc_launch_count(void);

/* Library build identification (for the bench record). */
const char *pd_ipc_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* PD_IPC_H */
