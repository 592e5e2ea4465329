/*
 * thetis_ref — the ORACLE for the Thetis hot path (arXiv 1311.2661).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  The product path (paper_1311_2661_b200/, libthetis.so) never
 * does, and shares no code, header, table or helper with it.
 *
 * A plain, slow, sequential CPU implementation written from the paper:
 *   - LP encodings: Eq. 2 (VC), App. B.2 packing rows (MIS,
 *     P:1036-1061), App. B.3 linearised multiway cut, put in
 *     the standard form Eq. 3 with explicit slack columns for
 *     inequality rows (App. C);
 *   - the penalty f_beta, Eq. 5 and its partial derivatives;
 *   - L_max, Eq. 7;
 *   - Alg. 1 SCD, its block / simplex variant (App. E,
 *     P:1570-1578), in the sweep orders of DESIGN.md §Readings R-5/R-6;
 *   - reductions from Def. 2;
 *   - rounding: P:139-146 + Lemma 1 for VC, App. C.2's alpha
 *      + greedy repair for MIS, CKR region growing
 *      best of `reps` for MWC.
 *
 * Built twice from one source: REAL = double (libthetis_ref64.so, the
 * invariant / pin build) and REAL = float (libthetis_ref32.so, the same
 * plain sequential arithmetic in fp32, which the CUDA deterministic mode is
 * compared against bit for bit).  All pointers are HOST pointers.
 *
 * Parity status per function: see DESIGN.md §Oracle pins.  Async-mode
 * trajectories at scale: parity unpinned beyond the sequential replay.
 */
#ifndef THETIS_REF_H
#define THETIS_REF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ref_lp ref_lp;

typedef struct {
    int64_t epochs, coordinate_updates, nnz_processed;
    double L_max;
    int64_t n_colours;
} ref_stats;

typedef struct {
    double lp_obj, f_beta, resid_l2, resid_inf, max_violation_eps, drift_inf;
    int64_t nonfinite;
} ref_objective;

typedef struct {
    double cost;
    int64_t feasible, n_selected;
    double eps_or_alpha;
    int64_t best_rep, fallback, rounds;
} ref_round_result;

/* codes (same numeric meaning as the product ABI, defined independently) */
enum { REF_OK = 0, REF_INVALID_ARG = -1, REF_NOT_SUPPORTED = -4, REF_DIVERGED = -5,
       REF_ROUND_PRECONDITION = -6 };

int ref_real_bytes(void); /* 4 or 8: which build this is */

int thetis_ref_build_lp(ref_lp** out, int64_t m, int64_t n, int64_t nnz, const int64_t* colptr,
                        const int32_t* rowidx, const float* val, const float* b, const float* c,
                        const int8_t* sense, const float* lo, const float* hi, int obj_sense,
                        int block_k, int64_t n_blocks);
int thetis_ref_build_graph_lp(ref_lp** out, int problem, int64_t n, int64_t n_edges,
                              const int32_t* src, const int32_t* dst, const float* vertex_w,
                              const float* edge_w, int k, const int32_t* terminals,
                              int t_per_label);
void thetis_ref_free(ref_lp* lp);

/* sizes: [m, n_struct, N, U, nnz_struct, n_blocks, block_k, m_edges, n_vertices, n_ineq] */
void thetis_ref_dims(const ref_lp* lp, int64_t* out10);
/* structural CSC of A (m x n_struct), ascending rows within columns */
void thetis_ref_get_csc(const ref_lp* lp, int64_t* colptr, int32_t* rowidx, double* val);
void thetis_ref_get_rows(const ref_lp* lp, double* b, int8_t* sense, double* c_int);
/* unique canonical edges (u < v) in row order, graph LPs only */
void thetis_ref_get_edges(const ref_lp* lp, int32_t* eu, int32_t* ev);

int thetis_ref_set_anchors(ref_lp* lp, const double* zbar, const double* ubar);
int thetis_ref_set_x(ref_lp* lp, const double* z);
void thetis_ref_get_x(const ref_lp* lp, double* z);
void thetis_ref_get_r(const ref_lp* lp, double* r);
void thetis_ref_get_x_f32(const ref_lp* lp, float* z);
void thetis_ref_get_r_f32(const ref_lp* lp, float* r);

/* one coordinate (or block) update of Alg. 1 on unit u; returns REF_OK */
int thetis_ref_step_unit(ref_lp* lp, float beta, int64_t u, int step_rule);
/* partial derivative of f_beta w.r.t. column j at the current point */
double thetis_ref_grad(const ref_lp* lp, float beta, int64_t j);

/* mode 0 = deterministic coloured sweep (R-5);
 * mode 1 = Alg. 1 one unit at a time in the permuted order: tiles
 *          of 32 consecutive units (blocks, scalars, slacks) in the order pi_e,
 *          units of a tile ascending -- THE ASYNC REFERENCE TRAJECTORY (R-6):
 *          the GPU's THETIS_MODE_ASYNC is compared against it within the
 *          BASELINE tolerances;
 * mode 2 = plain cyclic sweep;
 * mode 3 = replay of the hub-lag schedule (R-22, THETIS_MODE_ASYNC_HUBLAG), per
 *          epoch: (1) the hub steps pending from the previous epoch enter r,
 *          then every slack takes its step (slacks share no row); (2) VC / MIS:
 *          the scalar columns of the hub tiles (tiles of 32 structural units
 *          whose columns hold > 512 nonzeros, R-22's definition) take one
 *          synchronous step, z moves and the step d stays pending; (3) the tiles
 *          of 32 structural units in permutation order (pi_e over the structural
 *          tiles), each one synchronous step of its units (every unit steps from
 *          the state at the tile's start; r without the pending d), hub tiles
 *          skipped.  After the call's last epoch d enters r (r = A z - b on
 *          return).  Exact-arithmetic reference of THETIS_MODE_ASYNC_HUBLAG_SERIAL;
 *          a different algorithm from mode 1 with the same fixed point x(beta);
 * mode 4 = mode 1's order with each tile's units in three groups: its k-blocks one
 *          at a time (as in mode 1), then its scalar columns synchronously (all step
 *          from the same state, then apply in unit order), then its slacks likewise:
 *          the exact-arithmetic reference of THETIS_MODE_ASYNC_SERIAL. */
int thetis_ref_solve(ref_lp* lp, float beta, int epochs, int mode, uint64_t seed,
                     int step_rule, ref_stats* st);
int thetis_ref_objective(const ref_lp* lp, float beta, ref_objective* out);

/* augmented-Lagrangian outer loop (§3.4 "Augmented Lagrangian Framework",
 * P:480-496; R-19), the same rounds as thetis_solve_alm: solve with
 * (beta_t, ubar_t, zbar_t) for inner_epochs (mode, seed + t); measure; stop when
 * eps <= target_eps or after max_outer rounds; else ubar -= beta_t r, zbar = z,
 * beta grows by beta_growth when ||A z - b||_inf did not halve.  ubar0 / zbar0
 * may be NULL (zero).  Per round: beta, eps, ||r||_inf, c^T x (up to 64 rounds). */
typedef struct {
    int64_t rounds;
    float beta[64];
    double eps[64], resid_inf[64], lp_obj[64];
} ref_alm_stats;
int thetis_ref_solve_alm(ref_lp* lp, const double* ubar0, const double* zbar0, float beta0, float beta_growth,
                         int max_outer, int inner_epochs, int mode, uint64_t seed, int step_rule,
                         double target_eps, ref_alm_stats* st);
/* the current anchors (zero if unset): ubar (m), zbar (N) */
void thetis_ref_get_anchors(const ref_lp* lp, double* ubar, double* zbar);

/* colouring used by mode 0 for `seed`: colour per unit (slack units = K,
 * fixed units = -1); returns K (the slack class index) */
int64_t thetis_ref_colouring(ref_lp* lp, uint64_t seed, int32_t* colour_out);
/* tile permutation pi_e(t) for t in [0, n_tiles) */
void thetis_ref_tile_perm(int64_t n_tiles, uint64_t seed, int64_t epoch, int64_t* out);
/* Euclidean projection of y (length k) onto the simplex, fp of this build */
void thetis_ref_project_simplex(const double* y, int k, double* out);

/* rounding of an explicit fp32 point x (length n_struct): decisions in fp32 */
int thetis_ref_round_x(const ref_lp* lp, const float* x, int rule, uint64_t seed, int reps,
                       uint8_t* out_assign, ref_round_result* res);
/* rounding of the current iterate (cast to fp32 first) */
int thetis_ref_round(const ref_lp* lp, int rule, uint64_t seed, int reps, uint8_t* out_assign,
                     ref_round_result* res);

#ifdef __cplusplus
}
#endif
#endif
