/*
 * thetis_ref.c — ORACLE (test infrastructure only; see thetis_ref.h).
 *
 * Plain sequential C, written from PAPER.md (cited as P:line) and the
 * readings listed in DESIGN.md §Readings.  No blocking, no fusion, no
 * reordering beyond what the cited definitions state.  Compiled with
 * -ffp-contract=off so that every REAL operation is rounded on its own.
 *
 * REAL is double (libthetis_ref64.so) or float (libthetis_ref32.so).
 */
#include "thetis_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef REAL
#define REAL double
#endif

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define HUB_NNZ 512 /* R-17 / R-22: tiles whose scalar columns hold more nonzeros are hub tiles (the row
                         layout and the hub-lag variant; Alg. 1 (mode 1) does not depend on it) */

enum { PROB_GENERIC = 0, PROB_VC = 1, PROB_MIS = 2, PROB_MWC = 3 };
enum { SENSE_EQ = 0, SENSE_GE = 1, SENSE_LE = 2 };
enum { OBJ_MIN = 0, OBJ_MAX = 1 };
enum { MODE_DET = 0, MODE_ASYNC = 1, MODE_CYCLIC = 2, MODE_HUBLAG_REPLAY = 3, MODE_PI_TILE_SYNC = 4 };
enum { STEP_LMAX = 0, STEP_LJ = 1 };
enum { ROUND_VC_HALF = 1, ROUND_VC_FIXUP = 2, ROUND_MIS_GREEDY = 3, ROUND_MWC_CKR = 4, ROUND_SC_THRESHOLD = 5,
       ROUND_SC_RANDOM = 6, ROUND_MIS_BANSAL = 7 };

struct ref_lp {
    int problem;
    int obj_sense;
    int64_t m;        /* rows of A                                     */
    int64_t n_s;      /* structural columns                            */
    int64_t n_ineq;   /* inequality rows = slack columns               */
    int64_t N;        /* n_s + n_ineq coordinates of z = (x, s)        */
    int64_t nnz_s;    /* structural nonzeros                           */
    /* A, structural part, CSC with ascending rows (Eq. 3 data d = (A,b,c)) */
    int64_t* colptr;
    int32_t* rowidx;
    REAL* val;
    /* the same entries by rows, ascending columns (for r = Az - b row by row) */
    int64_t* rowptr;
    int32_t* rcol;
    REAL* rval;
    REAL* b;
    int8_t* sense;
    int64_t* row_slack;  /* slack column of row i, or -1 for EQ rows   */
    int64_t* slack_row;  /* row of slack q                             */
    REAL* slack_sign;    /* -1 for GE (a x - s = b), +1 for LE (a x + s = b) */
    REAL* c_int;         /* internal (minimisation) cost of structural columns */
    REAL* c_orig;        /* cost as given (original sense)             */
    REAL* lo;            /* bounds of structural columns               */
    REAL* hi;
    /* units: n_blocks k-blocks, then scalar structural columns, then slacks */
    int block_k;
    int64_t n_blocks, n_scalar, U;
    /* graph data (graph LPs) */
    int64_t n_vert, m_edges;
    int32_t* eu;
    int32_t* ev;
    float* vw;
    float* ew;
    int32_t* term_label; /* MWC: terminal label of vertex or -1 */
    /* state */
    REAL* z; /* length N */
    REAL* r; /* length m, maintained r = A z - b */
    REAL* zbar;
    REAL* ubar;
    REAL* ua; /* ubar^T a_j per structural column */
};

/* ------------------------------------------------------------------ */
/* hashing: SplitMix64 (Steele et al. 2014) and MurmurHash3's fmix32   */
/* ------------------------------------------------------------------ */
static uint64_t sm64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* i-th (0-based) output of SplitMix64 seeded with s */
static uint64_t sm64_out(uint64_t s, uint64_t i) { return sm64_mix(s + (i + 1) * GOLDEN); }
static uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6BU;
    h ^= h >> 13;
    h *= 0xC2B2AE35U;
    h ^= h >> 16;
    return h;
}

int ref_real_bytes(void) { return (int)sizeof(REAL); }

static void* xcalloc(int64_t count, size_t size) {
    if (count <= 0) count = 1;
    return calloc((size_t)count, size);
}

void thetis_ref_free(ref_lp* lp) {
    if (!lp) return;
    free(lp->colptr); free(lp->rowidx); free(lp->val);
    free(lp->rowptr); free(lp->rcol); free(lp->rval);
    free(lp->b); free(lp->sense); free(lp->row_slack); free(lp->slack_row); free(lp->slack_sign);
    free(lp->c_int); free(lp->c_orig); free(lp->lo); free(lp->hi);
    free(lp->eu); free(lp->ev); free(lp->vw); free(lp->ew); free(lp->term_label);
    free(lp->z); free(lp->r); free(lp->zbar); free(lp->ubar); free(lp->ua);
    free(lp);
}

/* ------------------------------------------------------------------ */
/* columns of the standard form [A | slack columns] (Eq. 3, App. C)    */
/* ------------------------------------------------------------------ */
static int64_t col_nnz(const ref_lp* lp, int64_t j) {
    return j < lp->n_s ? lp->colptr[j + 1] - lp->colptr[j] : 1;
}
/* sequential sum_i a_ij * v_i in ascending row order */
/* a_j^T v in the deterministic arithmetic contract (R-7; SURVEY §8(c).4's
 * "strided, butterfly-combined" dot, with 2^17 virtual lanes since round 2): virtual
 * lane l in [0, 2^17) sums the column's entries t = l, l + 2^17, l + 2^18, ...
 * (position in CSC order) from +0, each product rounded before the addition; then the
 * lanes combine by halving, p[l] = p[l] + p[l + off] for l < off, off = 2^16, ..., 1;
 * the dot is p[0].  Lanes at or past the column length hold +0, and x + (+0) = x for
 * every lane value x (no lane ever holds -0: a sum starting from +0 is never -0), so
 * the halving may start at the first off below the column length. */
static REAL col_dot(const ref_lp* lp, int64_t j, const REAL* v) {
    if (j >= lp->n_s) {
        int64_t q = j - lp->n_s;
        REAL acc = 0;
        acc = acc + lp->slack_sign[q] * v[lp->slack_row[q]];
        return acc;
    }
    enum { LANES = 1 << 17 };
    static REAL p[LANES];
    const int64_t len = lp->colptr[j + 1] - lp->colptr[j];
    const int64_t used = len < LANES ? len : LANES;
    for (int64_t l = 0; l < used; l++) p[l] = 0;
    for (int64_t t = 0; t < len; t++) {
        const int64_t e = lp->colptr[j] + t;
        p[t % LANES] = p[t % LANES] + lp->val[e] * v[lp->rowidx[e]];
    }
    if (used == 0) return 0;
    for (int64_t off = LANES / 2; off >= 1; off /= 2)
        for (int64_t l = 0; l < off && l + off < used; l++) p[l] = p[l] + p[l + off];
    return p[0];
}
/* r_i += a_ij * d for every nonzero of column j */
static void col_axpy(ref_lp* lp, int64_t j, REAL d) {
    if (j >= lp->n_s) {
        int64_t q = j - lp->n_s;
        int64_t i = lp->slack_row[q];
        lp->r[i] = lp->r[i] + lp->slack_sign[q] * d;
        return;
    }
    for (int64_t t = lp->colptr[j]; t < lp->colptr[j + 1]; t++) {
        int64_t i = lp->rowidx[t];
        lp->r[i] = lp->r[i] + lp->val[t] * d;
    }
}
/* ||a_j||^2 in fp64 */
static double col_norm2(const ref_lp* lp, int64_t j) {
    if (j >= lp->n_s) return 1.0;
    double s = 0.0;
    for (int64_t t = lp->colptr[j]; t < lp->colptr[j + 1]; t++) s += (double)lp->val[t] * (double)lp->val[t];
    return s;
}
static REAL col_lo(const ref_lp* lp, int64_t j) { return j < lp->n_s ? lp->lo[j] : (REAL)0; }
static REAL col_hi(const ref_lp* lp, int64_t j) { return j < lp->n_s ? lp->hi[j] : (REAL)INFINITY; }

/* first column and column count of unit u (blocks, scalars, slacks) */
static void unit_cols(const ref_lp* lp, int64_t u, int64_t* first, int64_t* count) {
    if (u < lp->n_blocks) { *first = u * lp->block_k; *count = lp->block_k; return; }
    u -= lp->n_blocks;
    if (u < lp->n_scalar) { *first = lp->n_blocks * lp->block_k + u; *count = 1; return; }
    u -= lp->n_scalar;
    *first = lp->n_s + u;
    *count = 1;
}
static int unit_fixed(const ref_lp* lp, int64_t u) {
    int64_t f, c;
    unit_cols(lp, u, &f, &c);
    for (int64_t j = f; j < f + c; j++)
        if (col_lo(lp, j) != col_hi(lp, j)) return 0;
    return 1;
}

/* r = A_std z - b, row by row: acc = -b_i, then + a_ij z_j over the row's
 * structural entries in ascending column order, then the slack. */
static void recompute_r(ref_lp* lp) {
    for (int64_t i = 0; i < lp->m; i++) {
        REAL acc = -lp->b[i];
        for (int64_t t = lp->rowptr[i]; t < lp->rowptr[i + 1]; t++)
            acc = acc + lp->rval[t] * lp->z[lp->rcol[t]];
        if (lp->row_slack[i] >= 0) {
            int64_t q = lp->row_slack[i] - lp->n_s;
            acc = acc + lp->slack_sign[q] * lp->z[lp->row_slack[i]];
        }
        lp->r[i] = acc;
    }
}

static void recompute_ua(ref_lp* lp) {
    for (int64_t j = 0; j < lp->n_s; j++) lp->ua[j] = lp->ubar ? col_dot(lp, j, lp->ubar) : (REAL)0;
}

/* ------------------------------------------------------------------ */
/* finishing a build: rows view, slacks, units, initial point          */
/* ------------------------------------------------------------------ */
static int finish_build(ref_lp* lp) {
    int64_t m = lp->m, n = lp->n_s;
    /* by-row view of A (transpose of the CSC, ascending columns) */
    lp->rowptr = (int64_t*)xcalloc(m + 1, sizeof(int64_t));
    lp->rcol = (int32_t*)xcalloc(lp->nnz_s, sizeof(int32_t));
    lp->rval = (REAL*)xcalloc(lp->nnz_s, sizeof(REAL));
    int64_t* fill = (int64_t*)xcalloc(m + 1, sizeof(int64_t));
    if (!lp->rowptr || !lp->rcol || !lp->rval || !fill) { free(fill); return REF_INVALID_ARG; }
    for (int64_t t = 0; t < lp->nnz_s; t++) lp->rowptr[lp->rowidx[t] + 1]++;
    for (int64_t i = 0; i < m; i++) lp->rowptr[i + 1] += lp->rowptr[i];
    for (int64_t i = 0; i < m; i++) fill[i] = lp->rowptr[i];
    for (int64_t j = 0; j < n; j++)
        for (int64_t t = lp->colptr[j]; t < lp->colptr[j + 1]; t++) {
            int64_t i = lp->rowidx[t];
            lp->rcol[fill[i]] = (int32_t)j;
            lp->rval[fill[i]] = lp->val[t];
            fill[i]++;
        }
    free(fill);
    /* slack columns: one per inequality row, in row order (App. C) */
    lp->row_slack = (int64_t*)xcalloc(m, sizeof(int64_t));
    lp->n_ineq = 0;
    for (int64_t i = 0; i < m; i++) lp->n_ineq += lp->sense[i] != SENSE_EQ;
    lp->slack_row = (int64_t*)xcalloc(lp->n_ineq, sizeof(int64_t));
    lp->slack_sign = (REAL*)xcalloc(lp->n_ineq, sizeof(REAL));
    int64_t q = 0;
    for (int64_t i = 0; i < m; i++) {
        if (lp->sense[i] == SENSE_EQ) { lp->row_slack[i] = -1; continue; }
        lp->row_slack[i] = n + q;
        lp->slack_row[q] = i;
        lp->slack_sign[q] = lp->sense[i] == SENSE_GE ? (REAL)-1 : (REAL)1;
        q++;
    }
    lp->N = n + lp->n_ineq;
    lp->n_scalar = n - lp->n_blocks * lp->block_k;
    lp->U = lp->n_blocks + lp->n_scalar + lp->n_ineq;
    lp->z = (REAL*)xcalloc(lp->N, sizeof(REAL));
    lp->r = (REAL*)xcalloc(m, sizeof(REAL));
    lp->ua = (REAL*)xcalloc(n, sizeof(REAL));
    if (!lp->z || !lp->r || !lp->ua) return REF_INVALID_ARG;
    /* initial point (R-3): free scalars at clamp(0, lo, hi); blocks
     * on the simplex barycentre (1/k,...,1/k); fixed columns at lo; slacks 0 */
    for (int64_t j = 0; j < n; j++) {
        REAL z0 = 0;
        if (z0 < lp->lo[j]) z0 = lp->lo[j];
        if (z0 > lp->hi[j]) z0 = lp->hi[j];
        lp->z[j] = z0;
    }
    for (int64_t bk = 0; bk < lp->n_blocks; bk++) {
        int64_t f, c;
        unit_cols(lp, bk, &f, &c);
        if (unit_fixed(lp, bk)) continue;
        for (int64_t j = f; j < f + c; j++) lp->z[j] = (REAL)(1.0 / (double)lp->block_k);
    }
    recompute_r(lp);
    return REF_OK;
}

int thetis_ref_build_lp(ref_lp** out, int64_t m, int64_t n, int64_t nnz, const int64_t* colptr,
                        const int32_t* rowidx, const float* val, const float* b, const float* c,
                        const int8_t* sense, const float* lo, const float* hi, int obj_sense,
                        int block_k, int64_t n_blocks) {
    if (!out || m < 0 || n < 0 || nnz < 0 || !colptr || (nnz > 0 && !rowidx) || (m > 0 && !b) ||
        (n > 0 && !c) || (obj_sense != OBJ_MIN && obj_sense != OBJ_MAX) || block_k < 0 ||
        n_blocks < 0 || (n_blocks > 0 && block_k < 1) || n_blocks * (int64_t)block_k > n ||
        m >= ((int64_t)1 << 31) || n >= ((int64_t)1 << 31))
        return REF_INVALID_ARG;
    if (colptr[0] != 0 || colptr[n] != nnz) return REF_INVALID_ARG;
    for (int64_t j = 0; j < n; j++) {
        if (colptr[j + 1] < colptr[j]) return REF_INVALID_ARG;
        for (int64_t t = colptr[j]; t < colptr[j + 1]; t++) {
            if (rowidx[t] < 0 || rowidx[t] >= m) return REF_INVALID_ARG;
            if (t > colptr[j] && rowidx[t] <= rowidx[t - 1]) return REF_INVALID_ARG;
        }
        if (lo && hi && lo[j] > hi[j]) return REF_INVALID_ARG;
    }
    if (sense)
        for (int64_t i = 0; i < m; i++)
            if (sense[i] < 0 || sense[i] > 2) return REF_INVALID_ARG;
    ref_lp* lp = (ref_lp*)calloc(1, sizeof(ref_lp));
    lp->problem = PROB_GENERIC;
    lp->obj_sense = obj_sense;
    lp->m = m; lp->n_s = n; lp->nnz_s = nnz;
    lp->block_k = block_k; lp->n_blocks = n_blocks;
    lp->colptr = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
    lp->rowidx = (int32_t*)xcalloc(nnz, sizeof(int32_t));
    lp->val = (REAL*)xcalloc(nnz, sizeof(REAL));
    lp->b = (REAL*)xcalloc(m, sizeof(REAL));
    lp->sense = (int8_t*)xcalloc(m, sizeof(int8_t));
    lp->c_int = (REAL*)xcalloc(n, sizeof(REAL));
    lp->c_orig = (REAL*)xcalloc(n, sizeof(REAL));
    lp->lo = (REAL*)xcalloc(n, sizeof(REAL));
    lp->hi = (REAL*)xcalloc(n, sizeof(REAL));
    for (int64_t j = 0; j <= n; j++) lp->colptr[j] = colptr[j];
    for (int64_t t = 0; t < nnz; t++) { lp->rowidx[t] = rowidx[t]; lp->val[t] = val ? (REAL)val[t] : (REAL)1; }
    for (int64_t i = 0; i < m; i++) { lp->b[i] = (REAL)b[i]; lp->sense[i] = sense ? sense[i] : SENSE_EQ; }
    for (int64_t j = 0; j < n; j++) {
        lp->c_orig[j] = (REAL)c[j];
        lp->c_int[j] = obj_sense == OBJ_MAX ? -(REAL)c[j] : (REAL)c[j];
        lp->lo[j] = lo ? (REAL)lo[j] : (REAL)0;
        lp->hi[j] = hi ? (REAL)hi[j] : (REAL)1;
    }
    int rc = finish_build(lp);
    if (rc != REF_OK) { thetis_ref_free(lp); return rc; }
    *out = lp;
    return REF_OK;
}

/* ------------------------------------------------------------------ */
/* graph LPs: VC (Eq. 2), MIS (App. B.2 edge rows), MWC (App. B.3)     */
/* ------------------------------------------------------------------ */
/* rows of graph LPs (R-17): (u < v) pairs sorted by
 * (floor(u / 2^ROW_RANGE_SHIFT), v, u) */
#define ROW_RANGE_SHIFT 14
typedef struct { uint64_t key; int64_t idx; } keyed_edge; /* key = (v << 32) | u */
static int cmp_keyed(const void* a, const void* b) {
    const keyed_edge* x = (const keyed_edge*)a;
    const keyed_edge* y = (const keyed_edge*)b;
    uint64_t gx = (x->key & 0xFFFFFFFFu) >> ROW_RANGE_SHIFT, gy = (y->key & 0xFFFFFFFFu) >> ROW_RANGE_SHIFT;
    if (gx != gy) return gx < gy ? -1 : 1;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}
static int cmp_vranged_key(const void* a, const void* b) { /* (v >> ROW_RANGE_SHIFT, u, v) */
    const keyed_edge* x = (const keyed_edge*)a;
    const keyed_edge* y = (const keyed_edge*)b;
    uint64_t gx = (x->key >> 32) >> ROW_RANGE_SHIFT, gy = (y->key >> 32) >> ROW_RANGE_SHIFT;
    if (gx != gy) return gx < gy ? -1 : 1;
    uint64_t ux = x->key & 0xFFFFFFFFu, uy = y->key & 0xFFFFFFFFu;
    if (ux != uy) return ux < uy ? -1 : 1;
    return (x->key >> 32) < (y->key >> 32) ? -1 : ((x->key >> 32) > (y->key >> 32));
}
static int cmp_plain_key(const void* a, const void* b) { /* (v, u); keys are unique here */
    const keyed_edge* x = (const keyed_edge*)a;
    const keyed_edge* y = (const keyed_edge*)b;
    return x->key < y->key ? -1 : (x->key > y->key);
}

int thetis_ref_build_graph_lp(ref_lp** out, int problem, int64_t n, int64_t n_edges,
                              const int32_t* src, const int32_t* dst, const float* vertex_w,
                              const float* edge_w, int k, const int32_t* terminals,
                              int t_per_label) {
    if (!out || n < 0 || n_edges < 0 || (n_edges > 0 && (!src || !dst))) return REF_INVALID_ARG;
    if (problem != PROB_VC && problem != PROB_MIS && problem != PROB_MWC) return REF_INVALID_ARG;
    if ((problem == PROB_VC || problem == PROB_MIS) && n > 0 && !vertex_w) return REF_INVALID_ARG;
    if (problem == PROB_MWC && (k < 2 || k > 32 || (n_edges > 0 && !edge_w) || t_per_label < 0 ||
                                (t_per_label > 0 && !terminals)))
        return REF_INVALID_ARG;
    for (int64_t e = 0; e < n_edges; e++)
        if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n) return REF_INVALID_ARG;

    /* canonicalise (u < v), drop self-loops, sort by (u >> 14, v, u), keep the
     * first occurrence of each pair; then the hub partition below: the row order
     * (R-17) */
    keyed_edge* ke = (keyed_edge*)xcalloc(n_edges, sizeof(keyed_edge));
    int64_t cnt = 0;
    for (int64_t e = 0; e < n_edges; e++) {
        uint64_t u = (uint64_t)src[e], v = (uint64_t)dst[e];
        if (u == v) continue;
        if (u > v) { uint64_t t = u; u = v; v = t; }
        ke[cnt].key = (v << 32) | u;
        ke[cnt].idx = e;
        cnt++;
    }
    qsort(ke, (size_t)cnt, sizeof(keyed_edge), cmp_keyed);
    int64_t me = 0;
    for (int64_t t = 0; t < cnt; t++)
        if (t == 0 || ke[t].key != ke[t - 1].key) ke[me++] = ke[t];
    {
        /* R-17: the rows whose larger endpoint lies in a hub tile (VC / MIS: a tile
         * of 32 vertices with more than HUB_NNZ incidences) keep this order; then the
         * other rows whose smaller endpoint lies in a hub tile, sorted by
         * (v >> ROW_RANGE_SHIFT, u, v); then the remaining rows, sorted by (v, u) */
        int64_t n_tiles = (n + 31) / 32;
        int64_t* tnz = (int64_t*)xcalloc(n_tiles + 1, sizeof(int64_t));
        for (int64_t e = 0; e < me; e++) {
            tnz[(ke[e].key & 0xFFFFFFFFu) >> 5]++;
            tnz[(ke[e].key >> 32) >> 5]++;
        }
        int hubs = problem == PROB_VC || problem == PROB_MIS;
        keyed_edge* ord = (keyed_edge*)xcalloc(me + 1, sizeof(keyed_edge));
        int64_t m1 = 0;
        for (int64_t e = 0; e < me; e++)
            if (hubs && tnz[(ke[e].key >> 32) >> 5] > HUB_NNZ) ord[m1++] = ke[e];
        int64_t m2 = m1;
        for (int64_t e = 0; e < me; e++)
            if (!(hubs && tnz[(ke[e].key >> 32) >> 5] > HUB_NNZ) && hubs && tnz[(ke[e].key & 0xFFFFFFFFu) >> 5] > HUB_NNZ)
                ord[m2++] = ke[e];
        int64_t q = m2;
        for (int64_t e = 0; e < me; e++)
            if (!(hubs && tnz[(ke[e].key >> 32) >> 5] > HUB_NNZ) && !(hubs && tnz[(ke[e].key & 0xFFFFFFFFu) >> 5] > HUB_NNZ))
                ord[q++] = ke[e];
        qsort(ord + m1, (size_t)(m2 - m1), sizeof(keyed_edge), cmp_vranged_key);
        qsort(ord + m2, (size_t)(me - m2), sizeof(keyed_edge), cmp_plain_key);
        memcpy(ke, ord, (size_t)me * sizeof(keyed_edge));
        free(ord);
        free(tnz);
    }

    ref_lp* lp = (ref_lp*)calloc(1, sizeof(ref_lp));
    lp->problem = problem;
    lp->n_vert = n;
    lp->m_edges = me;
    lp->eu = (int32_t*)xcalloc(me, sizeof(int32_t));
    lp->ev = (int32_t*)xcalloc(me, sizeof(int32_t));
    for (int64_t e = 0; e < me; e++) {
        lp->eu[e] = (int32_t)(ke[e].key & 0xFFFFFFFFu);
        lp->ev[e] = (int32_t)(ke[e].key >> 32);
    }
    if (problem == PROB_MWC) {
        lp->ew = (float*)xcalloc(me, sizeof(float));
        for (int64_t e = 0; e < me; e++) lp->ew[e] = edge_w[ke[e].idx];
    } else {
        lp->vw = (float*)xcalloc(n, sizeof(float));
        for (int64_t v = 0; v < n; v++) lp->vw[v] = vertex_w[v];
    }
    free(ke);

    /* incident edges of each vertex (R-17): the rows where it is the larger
     * endpoint in ascending row order, then the rows where it is the smaller one */
    int64_t* iptr = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
    for (int64_t e = 0; e < me; e++) { iptr[lp->eu[e] + 1]++; iptr[lp->ev[e] + 1]++; }
    for (int64_t v = 0; v < n; v++) iptr[v + 1] += iptr[v];
    int64_t* ifill = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
    int64_t* inc = (int64_t*)xcalloc(2 * me, sizeof(int64_t));
    for (int64_t v = 0; v < n; v++) ifill[v] = iptr[v];
    for (int64_t e = 0; e < me; e++) inc[ifill[lp->ev[e]]++] = e;
    for (int64_t e = 0; e < me; e++) inc[ifill[lp->eu[e]]++] = e;
    free(ifill);

    if (problem == PROB_VC || problem == PROB_MIS) {
        /* x_v in [0,1] per vertex; row e: x_u + x_v >= 1 (VC, Eq. 2) or <= 1 (MIS) */
        lp->obj_sense = problem == PROB_VC ? OBJ_MIN : OBJ_MAX;
        lp->m = me; lp->n_s = n; lp->nnz_s = 2 * me;
        lp->colptr = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
        lp->rowidx = (int32_t*)xcalloc(2 * me, sizeof(int32_t));
        lp->val = (REAL*)xcalloc(2 * me, sizeof(REAL));
        for (int64_t v = 0; v <= n; v++) lp->colptr[v] = iptr[v];
        for (int64_t t = 0; t < 2 * me; t++) { lp->rowidx[t] = (int32_t)inc[t]; lp->val[t] = 1; }
        lp->b = (REAL*)xcalloc(me, sizeof(REAL));
        lp->sense = (int8_t*)xcalloc(me, sizeof(int8_t));
        for (int64_t e = 0; e < me; e++) { lp->b[e] = 1; lp->sense[e] = problem == PROB_VC ? SENSE_GE : SENSE_LE; }
        lp->c_int = (REAL*)xcalloc(n, sizeof(REAL));
        lp->c_orig = (REAL*)xcalloc(n, sizeof(REAL));
        lp->lo = (REAL*)xcalloc(n, sizeof(REAL));
        lp->hi = (REAL*)xcalloc(n, sizeof(REAL));
        for (int64_t v = 0; v < n; v++) {
            lp->c_orig[v] = (REAL)vertex_w[v];
            lp->c_int[v] = problem == PROB_VC ? (REAL)vertex_w[v] : -(REAL)vertex_w[v];
            lp->lo[v] = 0; lp->hi[v] = 1;
        }
    } else {
        /* structural: x_v^l at v*k + l, then x_e^l at n*k + e*k + l (App. B.3).
         * rows 2(ek+l): x_e^l + x_u^l - x_v^l >= 0 ; 2(ek+l)+1: x_e^l - x_u^l + x_v^l >= 0 */
        lp->obj_sense = OBJ_MIN;
        int64_t nk = n * k, ns = nk + me * k, m = 2 * me * k;
        lp->m = m; lp->n_s = ns; lp->nnz_s = 2 * (2 * me) * k + 2 * me * k;
        lp->block_k = k; lp->n_blocks = n;
        lp->colptr = (int64_t*)xcalloc(ns + 1, sizeof(int64_t));
        lp->rowidx = (int32_t*)xcalloc(lp->nnz_s, sizeof(int32_t));
        lp->val = (REAL*)xcalloc(lp->nnz_s, sizeof(REAL));
        int64_t t = 0;
        for (int64_t v = 0; v < n; v++)
            for (int l = 0; l < k; l++) {
                lp->colptr[v * k + l] = t;
                for (int64_t p = iptr[v]; p < iptr[v + 1]; p++) {
                    int64_t e = inc[p];
                    int lower = lp->eu[e] == v; /* v is the smaller endpoint u */
                    lp->rowidx[t] = (int32_t)(2 * (e * k + l));
                    lp->val[t] = lower ? 1 : -1;
                    t++;
                    lp->rowidx[t] = (int32_t)(2 * (e * k + l) + 1);
                    lp->val[t] = lower ? -1 : 1;
                    t++;
                }
            }
        for (int64_t e = 0; e < me; e++)
            for (int l = 0; l < k; l++) {
                lp->colptr[nk + e * k + l] = t;
                lp->rowidx[t] = (int32_t)(2 * (e * k + l)); lp->val[t] = 1; t++;
                lp->rowidx[t] = (int32_t)(2 * (e * k + l) + 1); lp->val[t] = 1; t++;
            }
        lp->colptr[ns] = t;
        lp->b = (REAL*)xcalloc(m, sizeof(REAL));
        lp->sense = (int8_t*)xcalloc(m, sizeof(int8_t));
        for (int64_t i = 0; i < m; i++) { lp->b[i] = 0; lp->sense[i] = SENSE_GE; }
        lp->c_int = (REAL*)xcalloc(ns, sizeof(REAL));
        lp->c_orig = (REAL*)xcalloc(ns, sizeof(REAL));
        lp->lo = (REAL*)xcalloc(ns, sizeof(REAL));
        lp->hi = (REAL*)xcalloc(ns, sizeof(REAL));
        /* objective (1/2) sum_e c_e sum_l x_e^l */
        for (int64_t j = 0; j < ns; j++) { lp->lo[j] = 0; lp->hi[j] = 1; }
        for (int64_t e = 0; e < me; e++)
            for (int l = 0; l < k; l++) {
                REAL ce = (REAL)(lp->ew[e] * 0.5f);
                lp->c_int[nk + e * k + l] = ce;
                lp->c_orig[nk + e * k + l] = ce;
            }
        /* terminals V_1..V_k: block fixed at e_l through lo = hi */
        lp->term_label = (int32_t*)xcalloc(n, sizeof(int32_t));
        for (int64_t v = 0; v < n; v++) lp->term_label[v] = -1;
        for (int l = 0; l < k; l++)
            for (int i = 0; i < t_per_label; i++) {
                int32_t v = terminals[l * t_per_label + i];
                if (v < 0 || v >= n || lp->term_label[v] >= 0) { free(iptr); free(inc); thetis_ref_free(lp); return REF_INVALID_ARG; }
                lp->term_label[v] = l;
                for (int l2 = 0; l2 < k; l2++) {
                    lp->lo[v * k + l2] = l2 == l ? 1 : 0;
                    lp->hi[v * k + l2] = l2 == l ? 1 : 0;
                }
            }
    }
    free(iptr);
    free(inc);
    int rc = finish_build(lp);
    if (rc != REF_OK) { thetis_ref_free(lp); return rc; }
    *out = lp;
    return REF_OK;
}

/* ------------------------------------------------------------------ */
/* accessors                                                           */
/* ------------------------------------------------------------------ */
void thetis_ref_dims(const ref_lp* lp, int64_t* o) {
    o[0] = lp->m; o[1] = lp->n_s; o[2] = lp->N; o[3] = lp->U; o[4] = lp->nnz_s;
    o[5] = lp->n_blocks; o[6] = lp->block_k; o[7] = lp->m_edges; o[8] = lp->n_vert; o[9] = lp->n_ineq;
}
void thetis_ref_get_csc(const ref_lp* lp, int64_t* colptr, int32_t* rowidx, double* val) {
    for (int64_t j = 0; j <= lp->n_s; j++) colptr[j] = lp->colptr[j];
    for (int64_t t = 0; t < lp->nnz_s; t++) { rowidx[t] = lp->rowidx[t]; val[t] = (double)lp->val[t]; }
}
void thetis_ref_get_rows(const ref_lp* lp, double* b, int8_t* sense, double* c_int) {
    for (int64_t i = 0; i < lp->m; i++) { b[i] = (double)lp->b[i]; sense[i] = lp->sense[i]; }
    for (int64_t j = 0; j < lp->n_s; j++) c_int[j] = (double)lp->c_int[j];
}
void thetis_ref_get_edges(const ref_lp* lp, int32_t* eu, int32_t* ev) {
    for (int64_t e = 0; e < lp->m_edges; e++) { eu[e] = lp->eu[e]; ev[e] = lp->ev[e]; }
}
int thetis_ref_set_anchors(ref_lp* lp, const double* zbar, const double* ubar) {
    free(lp->zbar); free(lp->ubar);
    lp->zbar = NULL; lp->ubar = NULL;
    if (zbar) {
        lp->zbar = (REAL*)xcalloc(lp->N, sizeof(REAL));
        for (int64_t j = 0; j < lp->N; j++) lp->zbar[j] = (REAL)zbar[j];
    }
    if (ubar) {
        lp->ubar = (REAL*)xcalloc(lp->m, sizeof(REAL));
        for (int64_t i = 0; i < lp->m; i++) lp->ubar[i] = (REAL)ubar[i];
    }
    recompute_ua(lp);
    return REF_OK;
}
int thetis_ref_set_x(ref_lp* lp, const double* z) {
    for (int64_t j = 0; j < lp->N; j++) lp->z[j] = (REAL)z[j];
    recompute_r(lp);
    return REF_OK;
}
void thetis_ref_get_x(const ref_lp* lp, double* z) { for (int64_t j = 0; j < lp->N; j++) z[j] = (double)lp->z[j]; }
void thetis_ref_get_r(const ref_lp* lp, double* r) { for (int64_t i = 0; i < lp->m; i++) r[i] = (double)lp->r[i]; }
void thetis_ref_get_x_f32(const ref_lp* lp, float* z) { for (int64_t j = 0; j < lp->N; j++) z[j] = (float)lp->z[j]; }
void thetis_ref_get_r_f32(const ref_lp* lp, float* r) { for (int64_t i = 0; i < lp->m; i++) r[i] = (float)lp->r[i]; }

/* ------------------------------------------------------------------ */
/* Eq. 5 gradient and Alg. 1 step                                      */
/* ------------------------------------------------------------------ */
/* [grad f_beta(z)]_j = c_j - ubar^T a_j + beta a_j^T (A z - b) + (z_j - zbar_j)/beta
 * (Eq. 5 differentiated; r = A z - b is maintained) */
static REAL grad_col(const ref_lp* lp, REAL beta, int64_t j) {
    REAL c = j < lp->n_s ? lp->c_int[j] : (REAL)0;
    REAL ua = 0;
    if (lp->ubar) ua = j < lp->n_s ? lp->ua[j] : col_dot(lp, j, lp->ubar);
    REAL D = col_dot(lp, j, lp->r);
    REAL zb = lp->zbar ? lp->zbar[j] : (REAL)0;
    REAL g = c - ua;
    g = g + beta * D;
    g = g + (lp->z[j] - zb) / beta;
    return g;
}

double thetis_ref_grad(const ref_lp* lp, float beta, int64_t j) {
    return (double)grad_col(lp, (REAL)beta, j);
}

/* Euclidean projection onto the simplex {x >= 0, sum x = 1} (App. E,
 * P:1572-1575): sort descending (ties: smaller index first), rho = largest i
 * with u_i - (s_i - 1)/i > 0, tau = (s_rho - 1)/rho, x = max(y - tau, 0). */
static void project_simplex(const REAL* y, int k, REAL* x) {
    int idx[64];
    for (int l = 0; l < k; l++) idx[l] = l;
    for (int a = 1; a < k; a++) { /* insertion sort, descending, stable */
        int cur = idx[a], b = a - 1;
        while (b >= 0 && y[idx[b]] < y[cur]) { idx[b + 1] = idx[b]; b--; }
        idx[b + 1] = cur;
    }
    REAL s = 0, s_rho = y[idx[0]];
    int rho = 1;
    for (int i = 1; i <= k; i++) {
        REAL u = y[idx[i - 1]];
        s = s + u;
        if (u - (s - (REAL)1) / (REAL)i > 0) { rho = i; s_rho = s; }
    }
    REAL tau = (s_rho - (REAL)1) / (REAL)rho;
    for (int l = 0; l < k; l++) {
        REAL v = y[l] - tau;
        x[l] = v > 0 ? v : (REAL)0;
    }
}

void thetis_ref_project_simplex(const double* y, int k, double* out) {
    REAL yy[64], xx[64];
    for (int l = 0; l < k; l++) yy[l] = (REAL)y[l];
    project_simplex(yy, k, xx);
    for (int l = 0; l < k; l++) out[l] = (double)xx[l];
}

typedef struct { REAL beta; double Lmax; REAL invL; int rule; } step_ctx;

static step_ctx make_ctx(const ref_lp* lp, float beta_f, int rule) {
    step_ctx s;
    s.beta = (REAL)beta_f;
    s.rule = rule;
    /* Eq. 7: L_max = beta * max_i ||A_:i||^2 + 1/beta, over every column of
     * the standard form (slack columns have ||a||^2 = 1) */
    double mx = lp->n_ineq > 0 ? 1.0 : 0.0;
    for (int64_t j = 0; j < lp->n_s; j++) {
        double q = col_norm2(lp, j);
        if (q > mx) mx = q;
    }
    s.Lmax = (double)beta_f * mx + 1.0 / (double)beta_f;
    s.invL = (REAL)(1.0 / s.Lmax);
    return s;
}

/* step size 1/L for unit u: Alg. 1's 1/L_max, or 1/L_j (per-unit curvature
 * bound, R-4, an extension flagged as not the paper's) */
static REAL unit_invL(const ref_lp* lp, const step_ctx* s, int64_t first, int64_t count) {
    if (s->rule == STEP_LMAX) return s->invL;
    double mx = 0.0;
    for (int64_t j = first; j < first + count; j++) {
        double q = col_norm2(lp, j);
        if (q > mx) mx = q;
    }
    return (REAL)(1.0 / ((double)s->beta * mx + 1.0 / (double)s->beta));
}

/* Alg. 1 line 4 on unit u, generalised to the box [lo, hi] (R-2) and to
 * k-blocks with simplex projection (App. E): the new values of the unit's
 * columns, from the current z and r (nothing is modified). */
static void unit_new_values(const ref_lp* lp, const step_ctx* s, int64_t u, REAL* out) {
    int64_t f, c;
    unit_cols(lp, u, &f, &c);
    REAL invL = unit_invL(lp, s, f, c);
    if (u < lp->n_blocks) {
        REAL y[64];
        for (int64_t l = 0; l < c; l++) {
            REAL g = grad_col(lp, s->beta, f + l);
            y[l] = lp->z[f + l] - g * invL;
        }
        project_simplex(y, (int)c, out);
        return;
    }
    REAL g = grad_col(lp, s->beta, f);
    REAL t = lp->z[f] - g * invL;
    REAL lo = col_lo(lp, f), hi = col_hi(lp, f);
    REAL zn = t < lo ? lo : t;
    out[0] = zn > hi ? hi : zn;
}
/* z_j <- new value, r += a_j (new - old) for the unit's columns; returns nnz touched */
static int64_t apply_unit(ref_lp* lp, int64_t u, const REAL* nv) {
    int64_t f, c, nz = 0;
    unit_cols(lp, u, &f, &c);
    for (int64_t l = 0; l < c; l++) {
        REAL d = nv[l] - lp->z[f + l];
        col_axpy(lp, f + l, d);
        lp->z[f + l] = nv[l];
        nz += col_nnz(lp, f + l);
    }
    return nz;
}
/* one step of Alg. 1 on unit u; returns the nnz touched (0 if the unit is fixed) */
static int64_t step_unit(ref_lp* lp, const step_ctx* s, int64_t u) {
    if (unit_fixed(lp, u)) return 0;
    REAL nv[64];
    unit_new_values(lp, s, u, nv);
    return apply_unit(lp, u, nv);
}

int thetis_ref_step_unit(ref_lp* lp, float beta, int64_t u, int step_rule) {
    if (u < 0 || u >= lp->U || beta <= 0) return REF_INVALID_ARG;
    step_ctx s = make_ctx(lp, beta, step_rule);
    step_unit(lp, &s, u);
    return REF_OK;
}

/* ------------------------------------------------------------------ */
/* sweep orders (R-5, R-6)                                   */
/* ------------------------------------------------------------------ */
/* priority order of the colouring (R-5): more nonzeros first (largest degree
 * first), then the larger hash, then the smaller id */
typedef struct { int64_t deg; uint32_t prio; int64_t id; } prio_unit;
static int cmp_prio(const void* a, const void* b) {
    const prio_unit* x = (const prio_unit*)a;
    const prio_unit* y = (const prio_unit*)b;
    if (x->deg != y->deg) return x->deg > y->deg ? -1 : 1;
    if (x->prio != y->prio) return x->prio > y->prio ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}

/* Sequential greedy colouring in priority order (largest degree first, R-5):
 * colour(u) = smallest colour
 * not used by an already-coloured unit that shares a row of A with u.
 * Only non-fixed structural units take part; slacks form class K. */
int64_t thetis_ref_colouring(ref_lp* lp, uint64_t seed, int32_t* colour) {
    int64_t S = lp->n_blocks + lp->n_scalar; /* structural units */
    uint32_t key = fmix32((uint32_t)seed) ^ (uint32_t)(seed >> 32);
    /* units of each row */
    int64_t* uptr = (int64_t*)xcalloc(lp->m + 1, sizeof(int64_t));
    int64_t* ulist = (int64_t*)xcalloc(lp->nnz_s, sizeof(int64_t));
    int64_t* fill = (int64_t*)xcalloc(lp->m + 1, sizeof(int64_t));
    int64_t* col_unit = (int64_t*)xcalloc(lp->n_s, sizeof(int64_t));
    for (int64_t u = 0; u < S; u++) {
        int64_t f, c;
        unit_cols(lp, u, &f, &c);
        for (int64_t j = f; j < f + c; j++) col_unit[j] = u;
    }
    for (int64_t t = 0; t < lp->nnz_s; t++) uptr[lp->rowidx[t] + 1]++;
    for (int64_t i = 0; i < lp->m; i++) uptr[i + 1] += uptr[i];
    for (int64_t i = 0; i < lp->m; i++) fill[i] = uptr[i];
    for (int64_t j = 0; j < lp->n_s; j++)
        for (int64_t t = lp->colptr[j]; t < lp->colptr[j + 1]; t++) ulist[fill[lp->rowidx[t]]++] = col_unit[j];
    free(fill);

    prio_unit* order = (prio_unit*)xcalloc(S, sizeof(prio_unit));
    int64_t cnt = 0;
    for (int64_t u = 0; u < S; u++) {
        colour[u] = -1;
        if (unit_fixed(lp, u)) continue;
        int64_t f, c, deg = 0;
        unit_cols(lp, u, &f, &c);
        for (int64_t j = f; j < f + c; j++) deg += col_nnz(lp, j);
        order[cnt].deg = deg;
        order[cnt].prio = fmix32((uint32_t)u ^ key);
        order[cnt].id = u;
        cnt++;
    }
    qsort(order, (size_t)cnt, sizeof(prio_unit), cmp_prio);
    int64_t* stamp = (int64_t*)xcalloc(S + 2, sizeof(int64_t));
    for (int64_t q = 0; q < S + 2; q++) stamp[q] = -1;
    int64_t K = 0;
    for (int64_t p = 0; p < cnt; p++) {
        int64_t u = order[p].id, f, c;
        unit_cols(lp, u, &f, &c);
        for (int64_t j = f; j < f + c; j++)
            for (int64_t t = lp->colptr[j]; t < lp->colptr[j + 1]; t++) {
                int64_t i = lp->rowidx[t];
                for (int64_t q = uptr[i]; q < uptr[i + 1]; q++) {
                    int64_t w = ulist[q];
                    if (w != u && colour[w] >= 0) stamp[colour[w]] = u;
                }
            }
        int32_t col = 0;
        while (stamp[col] == u) col++;
        colour[u] = col;
        if (col + 1 > K) K = col + 1;
    }
    for (int64_t u = S; u < lp->U; u++) colour[u] = (int32_t)K;
    free(stamp); free(order); free(uptr); free(ulist); free(col_unit);
    return K;
}

/* pi_e on [0, n_tiles): 4-round balanced Feistel network on B bits,
 * B = smallest even integer >= max(2, ceil(log2 n_tiles)), round keys =
 * successive SplitMix64 outputs seeded with seed ^ (GOLDEN * (e+1)),
 * cycle-walking until the value is < n_tiles. */
static uint64_t feistel(uint64_t x, int h, const uint64_t* keys) {
    uint64_t mask = (h >= 32) ? 0xFFFFFFFFULL : ((1ULL << h) - 1);
    uint64_t L = x >> h, R = x & mask;
    for (int rd = 0; rd < 4; rd++) {
        uint64_t F = (uint64_t)fmix32((uint32_t)R ^ (uint32_t)keys[rd]) & mask;
        uint64_t nl = R, nr = L ^ F;
        L = nl; R = nr;
    }
    return (L << h) | R;
}
static int perm_bits(int64_t n_tiles) {
    int B = 0;
    while (((int64_t)1 << B) < n_tiles) B++;
    if (B < 2) B = 2;
    if (B & 1) B++;
    return B;
}
void thetis_ref_tile_perm(int64_t n_tiles, uint64_t seed, int64_t epoch, int64_t* out) {
    int h = perm_bits(n_tiles) / 2;
    uint64_t st = seed ^ (GOLDEN * (uint64_t)(epoch + 1));
    uint64_t keys[4];
    for (int rd = 0; rd < 4; rd++) keys[rd] = sm64_out(st, (uint64_t)rd);
    for (int64_t t = 0; t < n_tiles; t++) {
        uint64_t y = feistel((uint64_t)t, h, keys);
        while (y >= (uint64_t)n_tiles) y = feistel(y, h, keys);
        out[t] = (int64_t)y;
    }
}

/* Tile-synchronous replay (test reference for the kernel's semantics at one
 * tile in flight): every unit of the tile takes its step from the state at the
 * tile's start, then all changes are applied in unit order. */
static int64_t step_tile_sync(ref_lp* lp, const step_ctx* s, int64_t u0, int64_t u1, int64_t* updates,
                              REAL* nv) {
    int64_t nz = 0, kk = lp->block_k > 0 ? lp->block_k : 1;
    for (int64_t u = u0; u < u1; u++)
        if (!unit_fixed(lp, u)) unit_new_values(lp, s, u, nv + (u - u0) * kk);
    for (int64_t u = u0; u < u1; u++) {
        if (unit_fixed(lp, u)) continue;
        int64_t f, c;
        unit_cols(lp, u, &f, &c);
        nz += apply_unit(lp, u, nv + (u - u0) * kk);
        *updates += c;
    }
    return nz;
}

int thetis_ref_solve(ref_lp* lp, float beta, int epochs, int mode, uint64_t seed, int step_rule,
                     ref_stats* st) {
    if (!(beta > 0) || epochs < 0 || mode < 0 || mode > 4 || step_rule < 0 || step_rule > 1)
        return REF_INVALID_ARG;
    step_ctx s = make_ctx(lp, beta, step_rule);
    if (lp->ubar) recompute_ua(lp);
    int64_t updates = 0, nnz = 0, K = 0;
    int32_t* colour = NULL;
    int64_t* order = NULL;
    int64_t n_order = 0;
    if (mode == MODE_DET) {
        /* epoch = classes 0..K in order, members in ascending unit id */
        colour = (int32_t*)xcalloc(lp->U, sizeof(int32_t));
        K = thetis_ref_colouring(lp, seed, colour);
        order = (int64_t*)xcalloc(lp->U, sizeof(int64_t));
        for (int64_t cl = 0; cl <= K; cl++)
            for (int64_t u = 0; u < lp->U; u++)
                if (colour[u] == cl) order[n_order++] = u;
    }
    int64_t n_tiles = (lp->U + 31) / 32;
    const int64_t n_struct_units = lp->n_blocks + lp->n_scalar;
    const int64_t n_struct_tiles = (n_struct_units + 31) / 32;
    int64_t* perm = mode != MODE_DET && mode != MODE_CYCLIC ? (int64_t*)xcalloc(n_tiles, sizeof(int64_t)) : NULL;
    /* hub tiles of the async reference (R-6): VC / MIS tiles whose scalar
     * columns hold more than HUB_NNZ nonzeros */
    uint8_t* hub_tile = NULL;
    int64_t* hub_cols = NULL;
    REAL* hub_new = NULL;
    int64_t n_hub_cols = 0;
    if (mode == MODE_HUBLAG_REPLAY && (lp->problem == PROB_VC || lp->problem == PROB_MIS)) {
        hub_tile = (uint8_t*)xcalloc(n_struct_tiles, 1);
        hub_cols = (int64_t*)xcalloc(n_struct_tiles * 32, sizeof(int64_t));
        for (int64_t t = 0; t < n_struct_tiles; t++) {
            int64_t nz = 0;
            for (int64_t u = t * 32; u < t * 32 + 32 && u < lp->n_scalar; u++) nz += col_nnz(lp, u);
            if (nz > HUB_NNZ) {
                hub_tile[t] = 1;
                for (int64_t u = t * 32; u < t * 32 + 32 && u < lp->n_scalar; u++) hub_cols[n_hub_cols++] = u;
            }
        }
        hub_new = (REAL*)xcalloc(n_hub_cols, sizeof(REAL));
    }
    for (int e = 0; e < epochs; e++) {
        if (mode == MODE_DET) {
            for (int64_t p = 0; p < n_order; p++) {
                int64_t f, c;
                unit_cols(lp, order[p], &f, &c);
                nnz += step_unit(lp, &s, order[p]);
                updates += c;
            }
        } else if (mode == MODE_ASYNC) {
            thetis_ref_tile_perm(n_tiles, seed, e, perm);
            for (int64_t t = 0; t < n_tiles; t++)
                for (int64_t u = perm[t] * 32; u < perm[t] * 32 + 32 && u < lp->U; u++) {
                    if (unit_fixed(lp, u)) continue;
                    int64_t f, c;
                    unit_cols(lp, u, &f, &c);
                    nnz += step_unit(lp, &s, u);
                    updates += c;
                }
        } else if (mode == MODE_PI_TILE_SYNC) {
            /* the permuted sweep of MODE_ASYNC, a tile's units in three groups: its
             * k-blocks one at a time, then its scalar columns synchronously (all take
             * their steps from the state at that point, then apply in unit order), then
             * its slacks synchronously (the THETIS_MODE_ASYNC kernel with one tile in
             * flight; test reference for its arithmetic) */
            REAL nv[32 * 64];
            thetis_ref_tile_perm(n_tiles, seed, e, perm);
            for (int64_t t = 0; t < n_tiles; t++) {
                int64_t u0 = perm[t] * 32, u1 = u0 + 32 < lp->U ? u0 + 32 : lp->U;
                /* k-blocks one at a time (as in mode 1), then the scalar columns
                 * synchronously, then the slacks synchronously */
                for (; u0 < u1 && u0 < lp->n_blocks; u0++) {
                    if (unit_fixed(lp, u0)) continue;
                    nnz += step_unit(lp, &s, u0);
                    updates += lp->block_k;
                }
                int64_t us = u0 < n_struct_units ? (u1 < n_struct_units ? u1 : n_struct_units) : u0;
                nnz += step_tile_sync(lp, &s, u0, us, &updates, nv);
                nnz += step_tile_sync(lp, &s, us, u1, &updates, nv);
            }
        } else if (mode == MODE_HUBLAG_REPLAY) {
            REAL nv[32 * 64];
            /* (1) the row pass: the pending hub steps of the previous epoch enter r
             * (none in the first), then every slack takes its step (slacks share no
             * row, so any order gives the same result) */
            if (hub_cols && e > 0)
                for (int64_t q = 0; q < n_hub_cols; q++) col_axpy(lp, hub_cols[q], hub_new[q]);
            for (int64_t u = n_struct_units; u < lp->U; u++) {
                nnz += step_unit(lp, &s, u);
                updates += 1;
            }
            /* (2) hub step (VC / MIS): the scalar columns of every hub tile take one
             * synchronous step from this state; z_j moves, d_j stays pending (r does
             * not see it until the next row pass) */
            if (hub_cols) {
                for (int64_t q = 0; q < n_hub_cols; q++) {
                    REAL v[1];
                    unit_new_values(lp, &s, hub_cols[q], v);
                    hub_new[q] = unit_fixed(lp, hub_cols[q]) ? lp->z[hub_cols[q]] : v[0];
                }
                for (int64_t q = 0; q < n_hub_cols; q++) {
                    int64_t u = hub_cols[q];
                    REAL d = hub_new[q] - lp->z[u];
                    lp->z[u] = hub_new[q];
                    hub_new[q] = d;
                    nnz += col_nnz(lp, u);
                    updates += 1;
                }
            }
            /* (3) tiles of structural units in permutation order, each one synchronous
             * step of its units from r without the pending hub steps (hub tiles have
             * no units left) */
            thetis_ref_tile_perm(n_struct_tiles, seed, e, perm);
            for (int64_t t = 0; t < n_struct_tiles; t++) {
                if (hub_tile && hub_tile[perm[t]]) continue;
                int64_t u0 = perm[t] * 32, u1 = u0 + 32 < n_struct_units ? u0 + 32 : n_struct_units;
                nnz += step_tile_sync(lp, &s, u0, u1, &updates, nv);
            }
            /* after the last epoch the pending steps enter r: r = A z - b again */
            if (hub_cols && e == epochs - 1)
                for (int64_t q = 0; q < n_hub_cols; q++) col_axpy(lp, hub_cols[q], hub_new[q]);
        } else {
            for (int64_t u = 0; u < lp->U; u++) {
                if (unit_fixed(lp, u)) continue;
                int64_t f, c;
                unit_cols(lp, u, &f, &c);
                nnz += step_unit(lp, &s, u);
                updates += c;
            }
        }
    }
    free(colour); free(order); free(perm); free(hub_tile); free(hub_cols); free(hub_new);
    if (st) {
        st->epochs = epochs;
        st->coordinate_updates = updates;
        st->nnz_processed = nnz;
        st->L_max = s.Lmax;
        st->n_colours = K;
    }
    for (int64_t j = 0; j < lp->N; j++)
        if (!isfinite((double)lp->z[j])) return REF_DIVERGED;
    return REF_OK;
}

/* ------------------------------------------------------------------ */
/* reductions: Eq. 5 value, Def. 2 residual measures                   */
/* ------------------------------------------------------------------ */
int thetis_ref_objective(const ref_lp* lp, float beta_f, ref_objective* o) {
    double beta = (double)beta_f;
    memset(o, 0, sizeof(*o));
    double lp_obj = 0.0, lin = 0.0, prox = 0.0, ur = 0.0, r2 = 0.0, rinf = 0.0, eps = 0.0, drift = 0.0;
    int64_t nonfinite = 0;
    for (int64_t j = 0; j < lp->n_s; j++) {
        lp_obj += (double)lp->c_orig[j] * (double)lp->z[j];
        lin += (double)lp->c_int[j] * (double)lp->z[j];
    }
    for (int64_t j = 0; j < lp->N; j++) {
        double d = (double)lp->z[j] - (lp->zbar ? (double)lp->zbar[j] : 0.0);
        prox += d * d;
        if (!isfinite((double)lp->z[j])) nonfinite = 1;
    }
    for (int64_t i = 0; i < lp->m; i++) {
        double ax = 0.0;
        for (int64_t t = lp->rowptr[i]; t < lp->rowptr[i + 1]; t++)
            ax += (double)lp->rval[t] * (double)lp->z[lp->rcol[t]];
        double sl = 0.0;
        if (lp->row_slack[i] >= 0)
            sl = (double)lp->slack_sign[lp->row_slack[i] - lp->n_s] * (double)lp->z[lp->row_slack[i]];
        double ri = ax + sl - (double)lp->b[i]; /* (A z - b)_i */
        r2 += ri * ri;
        if (fabs(ri) > rinf) rinf = fabs(ri);
        if (lp->ubar) ur += (double)lp->ubar[i] * ri;
        double dr = fabs((double)lp->r[i] - ri);
        if (dr > drift || isnan(dr)) drift = dr;
        if (!isfinite((double)lp->r[i])) nonfinite = 1;
        double viol; /* structural violation with x only (R-8) */
        if (lp->sense[i] == SENSE_GE) viol = (double)lp->b[i] - ax;
        else if (lp->sense[i] == SENSE_LE) viol = ax - (double)lp->b[i];
        else viol = fabs(ax - (double)lp->b[i]);
        if (viol > eps) eps = viol;
    }
    o->lp_obj = lp_obj;
    o->f_beta = lin - ur + 0.5 * beta * r2 + prox / (2.0 * beta); /* Eq. 5 */
    o->resid_l2 = sqrt(r2);
    o->resid_inf = rinf;
    o->max_violation_eps = eps;
    o->drift_inf = drift;
    o->nonfinite = nonfinite;
    return nonfinite ? REF_DIVERGED : REF_OK;
}

/* ------------------------------------------------------------------ */
/* rounding                                                            */
/* ------------------------------------------------------------------ */
typedef struct { float x, w; int64_t id; } mis_key;
static int cmp_mis(const void* a, const void* b) {
    const mis_key* p = (const mis_key*)a;
    const mis_key* q = (const mis_key*)b;
    if (p->x != q->x) return p->x > q->x ? -1 : 1;
    if (p->w != q->w) return p->w > q->w ? -1 : 1;
    return p->id < q->id ? -1 : (p->id > q->id);
}

/* set cover (App. B.1; R-20) on a generic covering LP, rows
 * sum_{s in row} x_s >= 1, columns = sets: eps = max_rows (1 - sum x)_+ in fp32 (row sum
 * in ascending set order); SC_THRESHOLD picks x_s >= (1 - eps)/f, f = the largest row
 * count (Hochbaum's f-approximation "pick all sets with x_s > 1/f", on the
 * feasible point x/(1 - eps); >= for the boundary, SPEC's reading), or 1/f with
 * fallback when eps >= 1; SC_RANDOM keeps s iff u_s < min(1, d x_s), d = ceil(ln 2m)
 * (Srinivasan's scheme, with the repetitions of SPEC's ledger folded into
 * d), u_s = the first SplitMix64 output seeded seed ^ (0x5851F42D4C957F2D (s+1)) as
 * ((h >> 40) + 1/2) 2^-24; fallback = 1 if that sample left an element uncovered.
 * Both then add, for each uncovered element, its set with the largest x (ties:
 * smaller cost, then smaller index), judged against the pre-fix-up selection. */
static int round_set_cover(const ref_lp* lp, const float* x, int rule, uint64_t seed, uint8_t* out,
                           ref_round_result* res) {
    if (lp->problem != PROB_GENERIC || lp->n_blocks > 0 || lp->obj_sense != OBJ_MIN) return REF_NOT_SUPPORTED;
    const int64_t ns = lp->n_s, m = lp->m;
    for (int64_t i = 0; i < m; i++) {
        if (lp->sense[i] != SENSE_GE || lp->b[i] != (REAL)1) return REF_ROUND_PRECONDITION;
        for (int64_t t = lp->rowptr[i]; t < lp->rowptr[i + 1]; t++)
            if (lp->rval[t] != (REAL)1) return REF_ROUND_PRECONDITION;
    }
    float eps = 0.0f;
    int64_t f = 0;
    for (int64_t i = 0; i < m; i++) {
        float sum = 0.0f;
        for (int64_t t = lp->rowptr[i]; t < lp->rowptr[i + 1]; t++) sum = sum + x[lp->rcol[t]];
        float v = 1.0f - sum;
        if (v > eps) eps = v;
        if (lp->rowptr[i + 1] - lp->rowptr[i] > f) f = lp->rowptr[i + 1] - lp->rowptr[i];
    }
    res->eps_or_alpha = (double)eps;
    if (rule == ROUND_SC_THRESHOLD) {
        float tau = f > 0 ? 1.0f / (float)f : 1.0f;
        if (eps < 1.0f) tau = (1.0f - eps) / (float)f;
        else res->fallback = 1;
        for (int64_t s = 0; s < ns; s++) out[s] = x[s] >= tau ? 1 : 0;
    } else {
        const float d = (float)ceil(log(2.0 * (double)(m > 0 ? m : 1)));
        for (int64_t s = 0; s < ns; s++) {
            float p = d * x[s];
            if (p > 1.0f) p = 1.0f;
            uint64_t h = sm64_out(seed ^ (0x5851F42D4C957F2DULL * (uint64_t)(s + 1)), 0);
            float u = ((float)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
            out[s] = u < p ? 1 : 0;
        }
    }
    uint8_t* add = (uint8_t*)xcalloc(ns + 1, 1);
    int64_t uncovered = 0;
    for (int64_t i = 0; i < m; i++) {
        const int64_t a = lp->rowptr[i], b = lp->rowptr[i + 1];
        int covered = 0;
        for (int64_t t = a; t < b; t++) if (out[lp->rcol[t]]) covered = 1;
        if (covered || a == b) continue;
        uncovered++;
        int32_t pick = lp->rcol[a];
        for (int64_t t = a + 1; t < b; t++) {
            int32_t s = lp->rcol[t];
            if (x[s] > x[pick] || (x[s] == x[pick] && (lp->c_orig[s] < lp->c_orig[pick] ||
                                                       (lp->c_orig[s] == lp->c_orig[pick] && s < pick))))
                pick = s;
        }
        add[pick] = 1;
    }
    if (rule == ROUND_SC_RANDOM) res->fallback = uncovered > 0;
    for (int64_t s = 0; s < ns; s++) if (add[s] && !out[s]) { out[s] = 1; res->rounds++; }
    free(add);
    double cost = 0.0;
    int64_t sel = 0;
    for (int64_t s = 0; s < ns; s++) if (out[s]) { cost += (double)lp->c_orig[s]; sel++; }
    int64_t feas = 1;
    for (int64_t i = 0; i < m; i++) {
        int covered = 0;
        for (int64_t t = lp->rowptr[i]; t < lp->rowptr[i + 1]; t++) if (out[lp->rcol[t]]) covered = 1;
        if (!covered) feas = 0;
    }
    res->cost = cost; res->n_selected = sel; res->feasible = feas;
    return REF_OK;
}

/* MIS by Bansal et al.'s Alg. 2 as the paper ran it (
 * DESIGN.md R-21): x~ = x/(1+alpha) (the packing lemma's feasible point, tight alpha of
 * P:1313-1315); theta = 1/k, so step 2 keeps vertex v with probability x~_v / (k theta)
 * = x~_v, drawn as u_{t,v} < x~_v with u_{t,v} = ((h >> 40) + 1/2) 2^-24, h the v-th
 * SplitMix64 output seeded seed ^ 0xC2B2AE3D27D4EB4F (t+1); steps 3-4 with unit weights
 * (w_{a,s} = 1 for an edge a at vertex s): a kept vertex with a kept neighbour is deleted
 * (the event that the other chosen sets holding a exceed the capacity left by s; the
 * literal strict "> w_{a,s}" never fires for unit weights, A-10); the best of `reps`
 * repetitions by weight, ties to the smaller t. */
static int round_mis_bansal(const ref_lp* lp, const float* x, uint64_t seed, int reps, uint8_t* out,
                            ref_round_result* res) {
    if (lp->problem != PROB_MIS) return REF_NOT_SUPPORTED;
    if (reps < 1 || reps > 64) return REF_INVALID_ARG;
    const int64_t n = lp->n_vert, me = lp->m_edges;
    float alpha = 0.0f;
    for (int64_t e = 0; e < me; e++) {
        float v = (x[lp->eu[e]] + x[lp->ev[e]]) - 1.0f;
        if (v > alpha) alpha = v;
    }
    const float scale = 1.0f + alpha;
    uint8_t* keep = (uint8_t*)xcalloc(n + 1, 1);
    uint8_t* best_sel = (uint8_t*)xcalloc(n + 1, 1);
    double best_w = -1.0;
    int best_t = 0;
    for (int t = 0; t < reps; t++) {
        const uint64_t st = seed ^ (0xC2B2AE3D27D4EB4FULL * (uint64_t)(t + 1));
        for (int64_t v = 0; v < n; v++) {
            float p = x[v] / scale;
            float u = ((float)(sm64_out(st, (uint64_t)v) >> 40) + 0.5f) * (1.0f / 16777216.0f);
            keep[v] = u < p ? 1 : 0;
        }
        uint8_t* sel = (uint8_t*)xcalloc(n + 1, 1);
        for (int64_t v = 0; v < n; v++) sel[v] = keep[v];
        for (int64_t e = 0; e < me; e++)
            if (keep[lp->eu[e]] && keep[lp->ev[e]]) { sel[lp->eu[e]] = 0; sel[lp->ev[e]] = 0; }
        double w = 0.0;
        for (int64_t v = 0; v < n; v++) if (sel[v]) w += (double)lp->vw[v];
        if (w > best_w) { best_w = w; best_t = t; memcpy(best_sel, sel, (size_t)n); }
        free(sel);
    }
    int64_t cnt = 0;
    for (int64_t v = 0; v < n; v++) { out[v] = best_sel[v]; cnt += best_sel[v]; }
    int64_t feas = 1;
    for (int64_t e = 0; e < me; e++) if (out[lp->eu[e]] && out[lp->ev[e]]) feas = 0;
    res->cost = best_w; res->n_selected = cnt; res->best_rep = best_t; res->eps_or_alpha = (double)alpha;
    res->feasible = feas;
    free(keep); free(best_sel);
    return REF_OK;
}

int thetis_ref_round_x(const ref_lp* lp, const float* x, int rule, uint64_t seed, int reps,
                       uint8_t* out, ref_round_result* res) {
    memset(res, 0, sizeof(*res));
    if (rule == ROUND_MIS_BANSAL) return round_mis_bansal(lp, x, seed, reps, out, res);
    if (rule == ROUND_SC_THRESHOLD || rule == ROUND_SC_RANDOM) return round_set_cover(lp, x, rule, seed, out, res);
    int64_t n = lp->n_vert, me = lp->m_edges;
    if (rule == ROUND_VC_HALF || rule == ROUND_VC_FIXUP) {
        if (lp->problem != PROB_VC) return REF_NOT_SUPPORTED;
        /* eps = max_e (1 - (x_u + x_v))_+ in fp32 (Def. 2 / App. C form) */
        float eps = 0.0f;
        for (int64_t e = 0; e < me; e++) {
            float s = x[lp->eu[e]] + x[lp->ev[e]];
            float v = 1.0f - s;
            if (v > eps) eps = v;
        }
        float tau = 0.5f;
        if (rule == ROUND_VC_HALF) {
            if (eps < 1.0f) tau = (1.0f - eps) * 0.5f; /* Lemma 1: Pi(x/(1-eps)) >= 1/2 */
            else res->fallback = 1;
        }
        res->eps_or_alpha = (double)eps;
        /* threshold */
        for (int64_t v = 0; v < n; v++) out[v] = x[v] >= tau ? 1 : 0;
        /* fix-up against the pre-fix-up set: an uncovered edge adds its endpoint
         * with larger x (ties: smaller cost, then smaller id) */
        uint8_t* add = (uint8_t*)xcalloc(n, 1);
        for (int64_t e = 0; e < me; e++) {
            int32_t u = lp->eu[e], v = lp->ev[e];
            if (out[u] || out[v]) continue;
            int32_t pick;
            if (x[u] != x[v]) pick = x[u] > x[v] ? u : v;
            else if (lp->vw[u] != lp->vw[v]) pick = lp->vw[u] < lp->vw[v] ? u : v;
            else pick = u < v ? u : v;
            add[pick] = 1;
        }
        for (int64_t v = 0; v < n; v++) if (add[v]) { out[v] = 1; res->rounds++; }
        free(add);
        double cost = 0.0;
        int64_t sel = 0;
        for (int64_t v = 0; v < n; v++) if (out[v]) { cost += (double)lp->vw[v]; sel++; }
        int64_t feas = 1;
        for (int64_t e = 0; e < me; e++) if (!out[lp->eu[e]] && !out[lp->ev[e]]) feas = 0;
        res->cost = cost; res->n_selected = sel; res->feasible = feas;
        return REF_OK;
    }
    if (rule == ROUND_MIS_GREEDY) {
        if (lp->problem != PROB_MIS) return REF_NOT_SUPPORTED;
        /* alpha = max_e (x_u + x_v - 1)_+ (App. C.2 tight alpha, c = 1) */
        float alpha = 0.0f;
        for (int64_t e = 0; e < me; e++) {
            float s = x[lp->eu[e]] + x[lp->ev[e]];
            float v = s - 1.0f;
            if (v > alpha) alpha = v;
        }
        res->eps_or_alpha = (double)alpha;
        /* greedy repair: scan (x desc, w desc, id asc), accept v iff no accepted neighbour */
        int64_t* iptr = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
        int32_t* adj = (int32_t*)xcalloc(2 * me, sizeof(int32_t));
        int64_t* fill = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
        for (int64_t e = 0; e < me; e++) { iptr[lp->eu[e] + 1]++; iptr[lp->ev[e] + 1]++; }
        for (int64_t v = 0; v < n; v++) iptr[v + 1] += iptr[v];
        for (int64_t v = 0; v < n; v++) fill[v] = iptr[v];
        for (int64_t e = 0; e < me; e++) { adj[fill[lp->eu[e]]++] = lp->ev[e]; adj[fill[lp->ev[e]]++] = lp->eu[e]; }
        mis_key* ord = (mis_key*)xcalloc(n, sizeof(mis_key));
        for (int64_t v = 0; v < n; v++) { ord[v].x = x[v]; ord[v].w = lp->vw[v]; ord[v].id = v; out[v] = 0; }
        qsort(ord, (size_t)n, sizeof(mis_key), cmp_mis);
        for (int64_t p = 0; p < n; p++) {
            int64_t v = ord[p].id;
            int ok = 1;
            for (int64_t q = iptr[v]; q < iptr[v + 1]; q++) if (out[adj[q]]) { ok = 0; break; }
            if (ok) out[v] = 1;
        }
        double wsum = 0.0;
        int64_t sel = 0;
        for (int64_t v = 0; v < n; v++) if (out[v]) { wsum += (double)lp->vw[v]; sel++; }
        int64_t feas = 1;
        for (int64_t e = 0; e < me; e++) if (out[lp->eu[e]] && out[lp->ev[e]]) feas = 0;
        res->cost = wsum; res->n_selected = sel; res->feasible = feas;
        free(iptr); free(adj); free(fill); free(ord);
        return REF_OK;
    }
    if (rule == ROUND_MWC_CKR) {
        if (lp->problem != PROB_MWC) return REF_NOT_SUPPORTED;
        int k = lp->block_k;
        if (reps < 1) return REF_INVALID_ARG;
        /* precondition: every free vertex block lies on the simplex (App. C.3) */
        for (int64_t v = 0; v < n; v++) {
            if (lp->term_label[v] >= 0) continue;
            double s = 0.0;
            for (int l = 0; l < k; l++) {
                if (!(x[v * k + l] >= 0.0f)) return REF_ROUND_PRECONDITION;
                s += (double)x[v * k + l];
            }
            if (fabs(s - 1.0) > 1e-4) return REF_ROUND_PRECONDITION;
        }
        uint8_t* lab = (uint8_t*)xcalloc(n, 1);
        double best = INFINITY;
        int64_t best_t = -1;
        for (int t = 0; t < reps; t++) {
            /* CKR region growing (Vazirani Alg. 19.4): radius rho
             * uniform, theta = 1 - rho; random order sigma of the labels */
            uint64_t st = seed ^ (0xD1B54A32D192ED03ULL * (uint64_t)(t + 1));
            uint64_t h0 = sm64_out(st, 0);
            float theta = (float)(((double)(h0 >> 41) + 0.5) * 0x1p-23);
            int sigma[64];
            for (int l = 0; l < k; l++) sigma[l] = l;
            for (int i = k - 1; i >= 1; i--) {
                uint64_t h = sm64_out(st, (uint64_t)(k - i));
                int j = (int)(h % (uint64_t)(i + 1));
                int tmp = sigma[i]; sigma[i] = sigma[j]; sigma[j] = tmp;
            }
            for (int64_t v = 0; v < n; v++) {
                int l = sigma[k - 1];
                for (int i = 0; i < k - 1; i++)
                    if (x[v * k + sigma[i]] >= theta) { l = sigma[i]; break; }
                if (lp->term_label[v] >= 0) l = lp->term_label[v];
                lab[v] = (uint8_t)l;
            }
            double cost = 0.0;
            for (int64_t e = 0; e < me; e++)
                if (lab[lp->eu[e]] != lab[lp->ev[e]]) cost += (double)lp->ew[e];
            if (cost < best) { best = cost; best_t = t; if (out) memcpy(out, lab, (size_t)n); }
        }
        int64_t cut = 0;
        if (out)
            for (int64_t e = 0; e < me; e++) cut += out[lp->eu[e]] != out[lp->ev[e]];
        res->cost = best; res->best_rep = best_t; res->feasible = 1; res->n_selected = cut;
        free(lab);
        return REF_OK;
    }
    return REF_INVALID_ARG;
}

int thetis_ref_round(const ref_lp* lp, int rule, uint64_t seed, int reps, uint8_t* out,
                     ref_round_result* res) {
    float* x = (float*)xcalloc(lp->n_s, sizeof(float));
    for (int64_t j = 0; j < lp->n_s; j++) x[j] = (float)lp->z[j];
    int rc = thetis_ref_round_x(lp, x, rule, seed, reps, out, res);
    free(x);
    return rc;
}

/* ------------------------------------------------------------------ */
/* augmented-Lagrangian outer loop (§3.4; R-19)   */
/* ------------------------------------------------------------------ */
/* The method of multipliers for Eq. 3 with the proximal term of Eq. 5: the
 * multiplier estimate moves against the residual, ubar <- ubar - beta (A z - b)
 * (the step consistent with the -ubar^T (A x - b) term of Eq. 5), the proximal
 * anchor moves to the last iterate, zbar <- z; beta grows by beta_growth while
 * the residual does not halve between rounds. */
void thetis_ref_get_anchors(const ref_lp* lp, double* ubar, double* zbar) {
    for (int64_t i = 0; i < lp->m; i++) ubar[i] = lp->ubar ? (double)lp->ubar[i] : 0.0;
    for (int64_t j = 0; j < lp->N; j++) zbar[j] = lp->zbar ? (double)lp->zbar[j] : 0.0;
}
int thetis_ref_solve_alm(ref_lp* lp, const double* ubar0, const double* zbar0, float beta0, float beta_growth,
                         int max_outer, int inner_epochs, int mode, uint64_t seed, int step_rule,
                         double target_eps, ref_alm_stats* st) {
    if (!(beta0 > 0) || !(beta_growth >= 1) || max_outer < 1 || max_outer > 64 || inner_epochs < 0)
        return REF_INVALID_ARG;
    free(lp->ubar); free(lp->zbar);
    lp->ubar = (REAL*)xcalloc(lp->m + 1, sizeof(REAL));
    lp->zbar = (REAL*)xcalloc(lp->N + 1, sizeof(REAL));
    for (int64_t i = 0; i < lp->m; i++) lp->ubar[i] = ubar0 ? (REAL)ubar0[i] : (REAL)0;
    for (int64_t j = 0; j < lp->N; j++) lp->zbar[j] = zbar0 ? (REAL)zbar0[j] : (REAL)0;
    recompute_ua(lp);
    if (st) memset(st, 0, sizeof(*st));
    float beta = beta0;
    double prev_res = INFINITY;
    for (int t = 0; t < max_outer; t++) {
        int rc = thetis_ref_solve(lp, beta, inner_epochs, mode, seed + (uint64_t)t, step_rule, NULL);
        if (rc != REF_OK) return rc;
        ref_objective ob;
        rc = thetis_ref_objective(lp, beta, &ob);
        if (st) {
            st->rounds = t + 1;
            st->beta[t] = beta;
            st->eps[t] = ob.max_violation_eps;
            st->resid_inf[t] = ob.resid_inf;
            st->lp_obj[t] = ob.lp_obj;
        }
        if (rc != REF_OK) return rc;
        if (ob.max_violation_eps <= target_eps || t + 1 == max_outer) break;
        for (int64_t i = 0; i < lp->m; i++) {
            REAL step = (REAL)beta * lp->r[i]; /* rounded on its own (-ffp-contract=off) */
            lp->ubar[i] = lp->ubar[i] - step;
        }
        for (int64_t j = 0; j < lp->N; j++) lp->zbar[j] = lp->z[j];
        recompute_ua(lp);
        if (ob.resid_inf > 0.5 * prev_res) beta = (float)((double)beta * (double)beta_growth);
        prev_res = ob.resid_inf;
    }
    return REF_OK;
}
