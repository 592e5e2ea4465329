/*
 * thetis.h — C ABI of libthetis, the B200-native hot path of Thetis
 * (Bittorf, Re, Wright et al., arXiv 1311.2661): build a relaxed 0/1 LP,
 * solve its quadratic-penalty form (Eq. 5) by stochastic coordinate descent
 * (Alg. 1), reduce residual / objective / infeasibility, round (§2, App. C).
 *
 * Citations: P:L = PAPER.md line of the paper's LaTeX source.  Readings of
 * points the paper leaves open are DESIGN.md §Readings R-1..R-20.
 *
 * Conventions (all entry points):
 *  - Every call returns an int status, THETIS_OK (0) or a negative
 *    thetis_status; thetis_error_string(status) names it and
 *    thetis_last_error(lp) gives the detail of the last failure on lp.
 *  - Array arguments are DEVICE pointers unless the comment says otherwise;
 *    the build calls and thetis_set_x / thetis_round_x also accept HOST
 *    pointers (pinned or pageable; detected with cudaPointerGetAttributes)
 *    and copy them in.  The library never allocates device memory: all device
 *    state lives in the caller-owned workspace passed at build, which must
 *    stay alive until thetis_free.
 *  - All device work is enqueued on the cudaStream_t given at build (passed
 *    as void*; NULL = legacy default stream).  Calls that return host
 *    structs (build, objective, round, solve with stats) synchronise that
 *    stream before returning; thetis_solve with stats == NULL does not.
 *  - Validation errors are returned synchronously and leave the handle
 *    unchanged.  Kernel faults surface as THETIS_ERR_CUDA at the next call
 *    that synchronises (sticky for the CUDA context, as CUDA faults are).
 *  - A handle is not thread-safe; distinct handles are independent.
 *
 * Internal standard form (Eq. 3, with box bounds, R-1/R-2):
 *   z = (x, s): x = n_struct structural columns, s = one slack per
 *   inequality row (App. C): a_i^T x - s_i = b_i (GE),
 *   a_i^T x + s_i = b_i (LE), no slack for EQ.  x in [lo, hi] (default
 *   [0,1]), s >= 0.  MAX objectives are stored as MIN of -c.
 * Update units: n_blocks k-blocks (columns u*k .. u*k+k-1, projected on the
 *   simplex, App. E), then the scalar structural columns, then
 *   the slacks.  Units whose columns all have lo == hi are fixed (skipped).
 */
#ifndef THETIS_H
#define THETIS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define THETIS_API
#else
#define THETIS_API __attribute__((visibility("default")))
#endif

typedef struct thetis_lp thetis_lp; /* opaque handle (host struct) */

typedef enum {
    THETIS_OK = 0,
    THETIS_ERR_INVALID_ARG = -1,        /* null pointer, size mismatch, index out of range,
                                           lo > hi, beta <= 0, epochs < 0, unknown enum */
    THETIS_ERR_WORKSPACE_TOO_SMALL = -2,/* ws_bytes below the queried size */
    THETIS_ERR_CUDA = -3,               /* CUDA launch / runtime error (see thetis_last_error) */
    THETIS_ERR_NOT_SUPPORTED = -4,      /* e.g. VC rounding on an MIS LP, k > 32 */
    THETIS_ERR_DIVERGED = -5,           /* non-finite iterate or objective */
    THETIS_ERR_ROUND_PRECONDITION = -6  /* MWC rounding on a block off the simplex */
} thetis_status;

enum { THETIS_EQ = 0, THETIS_GE = 1, THETIS_LE = 2 };          /* row sense */
enum { THETIS_MIN = 0, THETIS_MAX = 1 };                       /* objective sense */
enum { THETIS_PROB_GENERIC = 0, THETIS_PROB_VC = 1, THETIS_PROB_MIS = 2, THETIS_PROB_MWC = 3 };
enum { THETIS_MODE_DETERMINISTIC = 0,
       THETIS_MODE_ASYNC = 1,        /* Alg. 1's permuted sweep, Hogwild (R-6) */
       THETIS_MODE_ASYNC_SERIAL = 2, /* diagnostic: the THETIS_MODE_ASYNC kernel with one tile in flight */
       THETIS_MODE_ASYNC_HUBLAG = 3, /* throughput variant: row pass + lagged hub step (R-22) */
       THETIS_MODE_ASYNC_HUBLAG_SERIAL = 4 /* diagnostic: the hub-lag kernels with one tile in flight */ };
enum { THETIS_STEP_LMAX = 0, /* Alg. 1: 1/L_max, Eq. 7 */
       THETIS_STEP_LJ = 1    /* 1/L_j per unit: extension, not the paper's (R-4) */ };
enum { THETIS_ROUND_VC_HALF = 1,   /* Lemma-1 threshold (1-eps)/2 + fix-up */
       THETIS_ROUND_VC_FIXUP = 2,  /* threshold 1/2 on raw x + fix-up */
       THETIS_ROUND_MIS_GREEDY = 3,/* packing alpha + greedy repair */
       THETIS_ROUND_MWC_CKR = 4,   /* CKR region growing, best of reps */
       THETIS_ROUND_SC_THRESHOLD = 5, /* set cover: x_s >= (1-eps)/f + fix-up (App. B.1; R-20) */
       THETIS_ROUND_SC_RANDOM = 6,    /* set cover: keep s w.p. min(1, d x_s) + fix-up (App. B.1; R-20) */
       THETIS_ROUND_MIS_BANSAL = 7    /* MIS: Bansal et al.'s Alg. 2 with theta = 1/k on x/(1+alpha), best of reps
                                         (R-21) */ };

#define THETIS_MAX_EPOCH_TIMES 64

typedef struct {
    int64_t epochs;
    int64_t coordinate_updates; /* scalar coordinates updated (a k-block counts k) */
    int64_t nnz_processed;      /* sum of nnz of updated columns (slack = 1) */
    double ms_total;            /* device time of the epochs (CUDA events) */
    float ms_per_epoch[THETIS_MAX_EPOCH_TIMES]; /* first 64 epochs */
    double L_max;               /* Eq. 7 */
    int64_t n_colours;          /* deterministic mode: classes before the slack class */
    int32_t mode, step_rule;
    /* async mode, over the first 64 epochs (CUDA events on the solve stream): device
     * time of the row passes (plus the call's final application of the pending steps;
     * without a hub step: the slack sweeps), of the hub updates, and of the permuted
     * tiles */
    double ms_row_pass, ms_hub_update, ms_tiles;
    int64_t row_pass_launches;
} thetis_solve_stats;

typedef struct {
    double lp_obj;            /* c^T x in the original sense (Eq. 3 objective)      */
    double f_beta;            /* Eq. 5 at z, with r recomputed from z               */
    double resid_l2;          /* ||A z - b||_2 (standard form, slacks included)     */
    double resid_inf;         /* ||A z - b||_inf  (Def. 2's epsilon)         */
    double max_violation_eps; /* max structural row violation with x only (R-8)     */
    double drift_inf;         /* ||r_maintained - (A z - b)||_inf                   */
    int64_t nonfinite;        /* 1 if some z or r is NaN / Inf                      */
} thetis_objective_t;

typedef struct {
    double cost;          /* VC: sum c_v selected; MIS: sum w_v selected; MWC: cut cost */
    int64_t feasible;     /* 1 if the integral solution is feasible for the IP          */
    int64_t n_selected;   /* VC/MIS: vertices selected; MWC: edges cut                 */
    double eps_or_alpha;  /* VC: eps (Lemma 1); MIS: alpha (App. C.2); MWC: 0          */
    int64_t best_rep;     /* MWC: repetition achieving the min cost                    */
    int64_t fallback;     /* VC_HALF: 1 if eps >= 1 forced the plain 1/2 threshold      */
    int64_t rounds;       /* VC: fix-up vertices added; MIS: parallel greedy rounds     */
} thetis_round_result;

typedef struct {
    int64_t m, n_struct, N, U, nnz_struct, n_blocks, block_k, m_edges, n_vertices, n_ineq;
    int32_t problem, obj_sense;
} thetis_dims;

#define THETIS_MAX_ALM_ROUNDS 64

typedef struct {
    int64_t rounds;                  /* outer rounds run (inner solves)                         */
    int64_t epochs_total;            /* inner epochs over all rounds                            */
    double ms_total;                 /* device time of the inner solves (CUDA events)           */
    float beta[THETIS_MAX_ALM_ROUNDS];        /* beta_t of round t                               */
    double eps[THETIS_MAX_ALM_ROUNDS];        /* max structural violation after round t (R-8)   */
    double resid_inf[THETIS_MAX_ALM_ROUNDS];  /* ||A z - b||_inf after round t                   */
    double lp_obj[THETIS_MAX_ALM_ROUNDS];     /* c^T x after round t (original sense)            */
} thetis_alm_stats;

/* ---- build ------------------------------------------------------------ */

/* Workspace bytes for thetis_build_graph_lp on n vertices and n_edges input
 * edges (an upper bound: dedup decides the final row count). */
THETIS_API int thetis_build_graph_lp_workspace(int problem, int64_t n, int64_t n_edges, int k,
                                               size_t* bytes);

/* Graph -> LP (P:126-138 VC; App. B.2 MIS edge rows; App. B.3 MWC).
 *  src, dst   int32[n_edges] endpoints in [0, n); orientation free; self-loops
 *             dropped; duplicate pairs kept once (the first occurrence's
 *             edge weight is used).  Rows follow the unique canonical pairs
 *             (u < v) (R-17): VC / MIS rows with an endpoint in a
 *             hub tile (32 consecutive ids with > 512 incidences) first, sorted
 *             by (u >> 14, v, u); then the other rows (all MWC rows) sorted by
 *             (v, u).  Each CSC column lists the rows where the
 *             vertex is the larger endpoint, then those where it is the smaller,
 *             each in ascending row order.  n must satisfy
 *             ((n-2) >> 14) * n * 2^14 + ... < 2^64 (n <= 2^32), else
 *             THETIS_ERR_NOT_SUPPORTED.
 *  vertex_w   float[n]: VC costs c_v (min) / MIS weights w_v (max).
 *  edge_w     float[n_edges]: MWC edge costs c_uv (objective 1/2 sum c_uv sum_l x_uv^l).
 *  k          MWC labels (2..32); terminals int32[k * t_per_label], label-major
 *             (label l owns terminals[l*t .. l*t+t-1]); terminal blocks are fixed at e_l.
 * Pointers may be host or device; inputs are copied into the workspace. */
THETIS_API int thetis_build_graph_lp(thetis_lp** out, void* workspace, size_t ws_bytes, void* stream,
                                     int problem, int64_t n, int64_t n_edges, const int32_t* src,
                                     const int32_t* dst, const float* vertex_w, const float* edge_w,
                                     int k, const int32_t* terminals, int t_per_label);

THETIS_API int thetis_build_lp_workspace(int64_t m, int64_t n, int64_t nnz, size_t* bytes);

/* Generic LP min/max c^T x s.t. A x (sense) b, lo <= x <= hi (Eq. 3 + slacks).
 *  A is m x n with nnz entries, given twice: CSC (csc_colptr int64[n+1],
 *  csc_rowidx int32[nnz], rows strictly ascending within a column) and CSR
 *  (csr_rowptr int64[m+1], csr_colidx int32[nnz], columns strictly ascending
 *  within a row) with the same entries; *_val float[nnz] or NULL (all 1).
 *  b float[m]; c float[n]; sense int8[m] (NULL = all EQ); lo / hi float[n]
 *  (NULL = 0 / 1); block_k > 0 makes the first n_blocks*block_k columns
 *  simplex blocks.  m, n < 2^31. */
THETIS_API int thetis_build_lp(thetis_lp** out, void* workspace, size_t ws_bytes, void* stream,
                               int64_t m, int64_t n, int64_t nnz, const int64_t* csc_colptr,
                               const int32_t* csc_rowidx, const float* csc_val,
                               const int64_t* csr_rowptr, const int32_t* csr_colidx,
                               const float* csr_val, const float* b, const float* c,
                               const int8_t* sense, const float* lo, const float* hi,
                               int obj_sense, int block_k, int64_t n_blocks);

THETIS_API int thetis_get_dims(const thetis_lp* lp, thetis_dims* out /* host */);

/* ---- state ------------------------------------------------------------ */

/* Anchors of Eq. 5: zbar float[N] and ubar float[m] DEVICE arrays
 * owned by the caller and kept alive while used; NULL = 0 (the default). */
THETIS_API int thetis_set_anchors(thetis_lp* lp, const float* zbar, const float* ubar);
/* z float[N] (host or device); recomputes r = A z - b.  Does not project. */
THETIS_API int thetis_set_x(thetis_lp* lp, const float* z);
/* copy min(count, N) entries of z (resp. m of r) to dst (host or device) */
THETIS_API int thetis_get_x(const thetis_lp* lp, float* dst, int64_t count);
THETIS_API int thetis_get_r(const thetis_lp* lp, float* dst, int64_t count);

/* ---- solve ------------------------------------------------------------ */

/* `epochs` sweeps of Alg. 1 on f_beta (Eq. 5), continuing from the
 * current z.  One epoch updates every non-fixed unit once:
 *  THETIS_MODE_DETERMINISTIC: graph-coloured classes 0..K-1 then the slack
 *    class, each class one conflict-free launch (R-5); bit-identical to the
 *    sequential sweep in that order.
 *  THETIS_MODE_ASYNC: tiles of 32 units in a per-epoch keyed permutation
 *    (R-6), processed concurrently Hogwild-style with atomic
 *    updates, a bounded window of tiles in flight.  Generic LPs and MWC keep the
 *    residual r current (red.global.add.f32); VC / MIS LPs keep the column sums
 *    A^T r current instead (fp64; R-23) and recompute r = A z - b before
 *    returning: same order, same result within rounding.  The environment variable
 *    THETIS_ASYNC_FORM=residual (read at every call) keeps the residual form there.
 *  THETIS_MODE_ASYNC_SERIAL: the async kernel with a single tile in flight,
 *    i.e. the tile-synchronous replay of the permutation (diagnostic / tests).
 * seed keys the colouring (det) or the permutations (async).  stats (host)
 * may be NULL; if given, the call synchronises and fills it. */
THETIS_API int thetis_solve(thetis_lp* lp, float beta, int epochs, int mode, uint64_t seed,
                            int step_rule, thetis_solve_stats* stats);

/* Fused reductions at the current z (Def. 2, Eq. 5); fp64 results. */
THETIS_API int thetis_objective(thetis_lp* lp, float beta, thetis_objective_t* out /* host */);

/* The augmented-Lagrangian outer loop ("proximal method of multipliers", §3.4
 * "Augmented Lagrangian Framework"; R-19): round t solves
 * f_beta (Eq. 5) with (beta_t, ubar_t, zbar_t) for `inner_epochs` epochs of
 * thetis_solve (mode, seed + t, step_rule), then measures eps_t (max structural
 * violation, R-8) and ||A z - b||_inf; it stops when eps_t <= target_eps or after
 * max_outer rounds, else updates
 *     ubar_{t+1} = ubar_t - beta_t (A z_t - b)   (the maintained r; fp32, two roundings)
 *     zbar_{t+1} = z_t                            (structural and slack coordinates)
 *     beta_{t+1} = beta_t * beta_growth if ||A z_t - b||_inf > ||A z_{t-1} - b||_inf / 2,
 *                  else beta_t                    (rounded to float)
 *  ubar  float[m] device, in/out: the multiplier estimate (caller-initialised, e.g. 0)
 *  zbar  float[N] device, in/out: the proximal anchor (caller-initialised, e.g. 0)
 *  Both stay registered as the LP's anchors (thetis_set_anchors) on return.
 *  Errors: INVALID_ARG (null anchors, beta0 <= 0, beta_growth < 1, max_outer < 1 or
 *  > THETIS_MAX_ALM_ROUNDS, inner_epochs < 0, unknown mode / rule); DIVERGED (a
 *  non-finite objective); CUDA.  stats (host) may be NULL. */
THETIS_API int thetis_solve_alm(thetis_lp* lp, float* ubar, float* zbar, float beta0, float beta_growth,
                                int max_outer, int inner_epochs, int mode, uint64_t seed, int step_rule,
                                double target_eps, thetis_alm_stats* stats);

/* ---- round ------------------------------------------------------------ */

/* Round the current x.  out_assign (device or host, may be NULL): uint8[n]
 * vertex selection (VC/MIS) or label (MWC); for the set-cover rules uint8[n_struct]
 * set selection.  seed: MWC_CKR and SC_RANDOM; reps: MWC_CKR only.
 * Set cover (NEXT-3, R-20): a generic LP whose rows all read sum_{s in row} x_s >= 1
 * (GE, b = 1, coefficients 1; else THETIS_ERR_ROUND_PRECONDITION), columns = sets,
 * rows = elements, f = the largest row count.  eps = max_rows (1 - sum x)_+ in fp32
 * (sum in CSR order); SC_THRESHOLD selects x_s >= (1 - eps)/f (f-approximation of
 * Hochbaum, on x/(1 - eps)), or 1/f with fallback = 1 when eps >= 1;
 * SC_RANDOM keeps s iff u_s < min(1, d x_s), d = ceil(ln(2 m)), u_s counter-based
 * (SplitMix64 of seed ^ 0x5851F42D4C957F2D (s + 1)), fallback = 1 when that sample
 * left an element uncovered.  Both then add, for every uncovered element, its set
 * with the largest x (ties: smaller cost, then smaller index), judged against the
 * pre-fix-up selection; rounds = sets added, eps_or_alpha = eps.
 * MIS_BANSAL (NEXT-2, R-21): alpha and x~ = x/(1+alpha) as MIS_GREEDY; repetition t keeps
 * vertex v iff u_{t,v} < x~_v (Alg. 2 step 2 with k theta = 1), u_{t,v} the v-th SplitMix64
 * output seeded seed ^ 0xC2B2AE3D27D4EB4F (t+1), as ((h >> 40) + 1/2) 2^-24; a kept vertex
 * with a kept neighbour is deleted (steps 3-4 for unit weights: E_{a,v} when another chosen
 * set holds a); the best of `reps` (1..64) by weight (ties: smaller t) is returned;
 * best_rep = t, eps_or_alpha = alpha. */
THETIS_API int thetis_round(thetis_lp* lp, int rule, uint64_t seed, int reps, uint8_t* out_assign,
                            thetis_round_result* out /* host */);
/* Same on an explicit structural point x float[n_struct] (host or device). */
THETIS_API int thetis_round_x(thetis_lp* lp, const float* x, int rule, uint64_t seed, int reps,
                              uint8_t* out_assign, thetis_round_result* out);

/* ---- inspection (tests / tooling) ------------------------------------- */

/* structural CSC of A decoded to (colptr int64[n_struct+1], rowidx int32[nnz],
 * val float[nnz]); graph LPs also export the unique edges (eu, ev int32[m_edges]).
 * Any pointer may be NULL; destinations host or device. */
THETIS_API int thetis_get_csc(const thetis_lp* lp, int64_t* colptr, int32_t* rowidx, float* val);
THETIS_API int thetis_get_edges(const thetis_lp* lp, int32_t* eu, int32_t* ev);
/* deterministic-mode colouring for `seed` (computed if not cached): colour
 * int32[U] (slack units = K, fixed = -1); *n_colours = K. */
THETIS_API int thetis_get_colouring(thetis_lp* lp, uint64_t seed, int32_t* colour, int64_t* n_colours);
/* the async tile permutation pi_epoch on [0, n_tiles) as the update kernels
 * compute it inline (out: DEVICE int64[n_tiles]); enqueued on `stream`. */
THETIS_API int thetis_tile_perm(int64_t n_tiles, uint64_t seed, int64_t epoch, int64_t* out,
                                void* stream);

/* ---- lifetime / errors ------------------------------------------------ */
THETIS_API int thetis_sync(thetis_lp* lp);
THETIS_API void thetis_free(thetis_lp* lp); /* does not free the caller's workspace */
THETIS_API const char* thetis_error_string(int status);
THETIS_API const char* thetis_last_error(const thetis_lp* lp);
THETIS_API const char* thetis_version(void);

#ifdef __cplusplus
}
#endif
#endif /* THETIS_H */
