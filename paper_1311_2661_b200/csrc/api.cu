// The C ABI of libthetis (include/thetis.h): argument validation, handle and
// workspace management, and dispatch to the kernels in build.cu, colour.cu,
// scd.cu, reduce.cu and round.cu.
#include <cstdarg>
#include <cstdlib>
#include <new>

#include "thetis_internal.cuh"

namespace thetis {

int set_error(thetis_lp* lp, int code, const char* fmt, ...) {
    if (lp) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(lp->err, sizeof(lp->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

int check_cuda(thetis_lp* lp, const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(lp, THETIS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return THETIS_OK;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace thetis

using namespace thetis;

namespace {

int new_handle(thetis_lp** out, void* ws, size_t ws_bytes, void* stream, thetis_lp** lp_out) {
    thetis_lp* lp = new (std::nothrow) thetis_lp();
    if (!lp) return THETIS_ERR_INVALID_ARG;
    lp->ws = (char*)ws;
    lp->ws_bytes = ws_bytes;
    lp->stream = (cudaStream_t)stream;
    if (cudaStreamCreateWithFlags(&lp->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&lp->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&lp->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        delete lp;
        return THETIS_ERR_CUDA;
    }
    *lp_out = lp;
    (void)out;
    return THETIS_OK;
}

void destroy(thetis_lp* lp) {
    if (!lp) return;
    if (lp->det_graph) {
        cudaStreamSynchronize(lp->stream);
        cudaGraphExecDestroy(lp->det_graph);
    }
    if (lp->side) cudaStreamDestroy(lp->side);
    if (lp->ev_fork) cudaEventDestroy(lp->ev_fork);
    if (lp->ev_join) cudaEventDestroy(lp->ev_join);
    for (auto q : lp->det_s) if (q) cudaStreamDestroy(q);
    for (auto e : lp->det_ev) if (e) cudaEventDestroy(e);
    for (auto e : lp->ev_epoch) cudaEventDestroy(e);
    for (auto e : lp->ev_kern) cudaEventDestroy(e);
    delete lp;
}

thread_local char g_err[512];

int fail_global(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

}  // namespace

extern "C" {

THETIS_API const char* thetis_version(void) { return "thetis-b200 0.1 (sm_100a)"; }

THETIS_API const char* thetis_error_string(int status) {
    switch (status) {
        case THETIS_OK: return "THETIS_OK";
        case THETIS_ERR_INVALID_ARG: return "THETIS_ERR_INVALID_ARG";
        case THETIS_ERR_WORKSPACE_TOO_SMALL: return "THETIS_ERR_WORKSPACE_TOO_SMALL";
        case THETIS_ERR_CUDA: return "THETIS_ERR_CUDA";
        case THETIS_ERR_NOT_SUPPORTED: return "THETIS_ERR_NOT_SUPPORTED";
        case THETIS_ERR_DIVERGED: return "THETIS_ERR_DIVERGED";
        case THETIS_ERR_ROUND_PRECONDITION: return "THETIS_ERR_ROUND_PRECONDITION";
        default: return "THETIS_ERR_UNKNOWN";
    }
}

THETIS_API const char* thetis_last_error(const thetis_lp* lp) { return lp ? lp->err : g_err; }

THETIS_API int thetis_build_graph_lp_workspace(int problem, int64_t n, int64_t n_edges, int k, size_t* bytes) {
    if (!bytes || n < 0 || n >= ((int64_t)1 << 31) || n_edges < 0 || n_edges >= ((int64_t)1 << 31) ||
        (problem != THETIS_PROB_VC && problem != THETIS_PROB_MIS && problem != THETIS_PROB_MWC) ||
        (problem == THETIS_PROB_MWC && (k < 2 || k > kMaxK)))
        return fail_global(THETIS_ERR_INVALID_ARG, "bad arguments to thetis_build_graph_lp_workspace");
    *bytes = graph_workspace(problem, n, n_edges, k, false, nullptr, nullptr);
    return THETIS_OK;
}

THETIS_API int thetis_build_graph_lp(thetis_lp** out, void* workspace, size_t ws_bytes, void* stream, int problem,
                                     int64_t n, int64_t n_edges, const int32_t* src, const int32_t* dst,
                                     const float* vertex_w, const float* edge_w, int k, const int32_t* terminals,
                                     int t_per_label) {
    thetis::NvtxRange nvtx_("thetis_build_graph_lp");
    if (!out) return fail_global(THETIS_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    size_t need = 0;
    THETIS_TRY(thetis_build_graph_lp_workspace(problem, n, n_edges, k, &need));
    if (!workspace) return fail_global(THETIS_ERR_INVALID_ARG, "workspace is NULL");
    if (n_edges > 0 && (!src || !dst)) return fail_global(THETIS_ERR_INVALID_ARG, "src / dst NULL");
    if (problem != THETIS_PROB_MWC && n > 0 && !vertex_w) return fail_global(THETIS_ERR_INVALID_ARG, "vertex_w NULL");
    if (problem == THETIS_PROB_MWC) {
        if (n_edges > 0 && !edge_w) return fail_global(THETIS_ERR_INVALID_ARG, "edge_w NULL");
        if (t_per_label < 0 || (t_per_label > 0 && !terminals) || (int64_t)k * t_per_label > n ||
            (int64_t)k * t_per_label > 32 * 4096)
            return fail_global(THETIS_ERR_INVALID_ARG, "bad terminals");
    }
    if (ws_bytes < need) return fail_global(THETIS_ERR_WORKSPACE_TOO_SMALL, "workspace below the queried size");
    thetis_lp* lp = nullptr;
    THETIS_TRY(new_handle(out, workspace, ws_bytes, stream, &lp));
    int rc = build_graph(lp, problem, n, n_edges, src, dst, vertex_w, edge_w, k, terminals, t_per_label);
    if (rc != THETIS_OK) {
        fail_global(rc, lp->err);
        destroy(lp);
        return rc;
    }
    *out = lp;
    return THETIS_OK;
}

THETIS_API int thetis_build_lp_workspace(int64_t m, int64_t n, int64_t nnz, size_t* bytes) {
    if (!bytes || m < 0 || n < 0 || nnz < 0 || m >= ((int64_t)1 << 31) || n >= ((int64_t)1 << 31))
        return fail_global(THETIS_ERR_INVALID_ARG, "bad arguments to thetis_build_lp_workspace");
    *bytes = generic_workspace(m, n, nnz, true, false, nullptr, nullptr);
    return THETIS_OK;
}

THETIS_API int thetis_build_lp(thetis_lp** out, void* workspace, size_t ws_bytes, void* stream, int64_t m, int64_t n,
                               int64_t nnz, const int64_t* csc_colptr, const int32_t* csc_rowidx, const float* csc_val,
                               const int64_t* csr_rowptr, const int32_t* csr_colidx, const float* csr_val,
                               const float* b, const float* c, const int8_t* sense, const float* lo, const float* hi,
                               int obj_sense, int block_k, int64_t n_blocks) {
    thetis::NvtxRange nvtx_("thetis_build_lp");
    if (!out) return fail_global(THETIS_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    size_t need = 0;
    THETIS_TRY(thetis_build_lp_workspace(m, n, nnz, &need));
    if (!workspace || !csc_colptr || !csr_rowptr || (nnz > 0 && (!csc_rowidx || !csr_colidx)) || (m > 0 && !b) ||
        (n > 0 && !c) || ((csc_val == nullptr) != (csr_val == nullptr)) ||
        (obj_sense != THETIS_MIN && obj_sense != THETIS_MAX) || block_k < 0 || block_k > kMaxK || n_blocks < 0 ||
        (n_blocks > 0 && block_k < 1) || n_blocks * (int64_t)block_k > n)
        return fail_global(THETIS_ERR_INVALID_ARG, "bad arguments to thetis_build_lp");
    if (ws_bytes < need) return fail_global(THETIS_ERR_WORKSPACE_TOO_SMALL, "workspace below the queried size");
    thetis_lp* lp = nullptr;
    THETIS_TRY(new_handle(out, workspace, ws_bytes, stream, &lp));
    int rc = build_generic(lp, m, n, nnz, csc_colptr, csc_rowidx, csc_val, csr_rowptr, csr_colidx, csr_val, b, c,
                           sense, lo, hi, obj_sense, block_k, n_blocks);
    if (rc != THETIS_OK) {
        fail_global(rc, lp->err);
        destroy(lp);
        return rc;
    }
    *out = lp;
    return THETIS_OK;
}

THETIS_API int thetis_get_dims(const thetis_lp* lp, thetis_dims* o) {
    if (!lp || !o) return THETIS_ERR_INVALID_ARG;
    const DevLP& d = lp->d;
    o->m = d.m; o->n_struct = d.n_s; o->N = d.N; o->U = d.U; o->nnz_struct = d.nnz_s; o->n_blocks = d.n_blocks;
    o->block_k = d.k; o->m_edges = d.m_edges; o->n_vertices = d.n_vert; o->n_ineq = d.n_ineq;
    o->problem = d.problem; o->obj_sense = d.obj_sense;
    return THETIS_OK;
}

THETIS_API int thetis_set_anchors(thetis_lp* lp, const float* zbar, const float* ubar) {
    if (!lp) return THETIS_ERR_INVALID_ARG;
    if ((zbar && !is_device_ptr(zbar)) || (ubar && !is_device_ptr(ubar)))
        return set_error(lp, THETIS_ERR_INVALID_ARG, "anchors must be device arrays");
    lp->d.zbar = zbar;
    lp->d.ubar = ubar;
    lp->anchors = zbar || ubar;
    return recompute_ua(lp);
}

THETIS_API int thetis_set_x(thetis_lp* lp, const float* z) {
    if (!lp || !z) return THETIS_ERR_INVALID_ARG;
    if (lp->d.N > 0)
        CUDA_TRY(lp, cudaMemcpyAsync(lp->d.z, z, (size_t)lp->d.N * 4, cudaMemcpyDefault, lp->stream));
    return recompute_r(lp);
}

static int copy_out(const thetis_lp* lp, void* dst, const void* src, size_t bytes) {
    thetis_lp* l = const_cast<thetis_lp*>(lp);
    if (bytes == 0) return THETIS_OK;
    CUDA_TRY(l, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, lp->stream));
    CUDA_TRY(l, cudaStreamSynchronize(lp->stream));
    return THETIS_OK;
}

THETIS_API int thetis_get_x(const thetis_lp* lp, float* dst, int64_t count) {
    if (!lp || !dst || count < 0) return THETIS_ERR_INVALID_ARG;
    int64_t c = count < lp->d.N ? count : lp->d.N;
    return copy_out(lp, dst, lp->d.z, (size_t)c * 4);
}

THETIS_API int thetis_get_r(const thetis_lp* lp, float* dst, int64_t count) {
    if (!lp || !dst || count < 0) return THETIS_ERR_INVALID_ARG;
    int64_t c = count < lp->d.m ? count : lp->d.m;
    return copy_out(lp, dst, lp->d.r, (size_t)c * 4);
}

THETIS_API int thetis_solve(thetis_lp* lp, float beta, int epochs, int mode, uint64_t seed, int step_rule,
                            thetis_solve_stats* stats) {
    thetis::NvtxRange nvtx_("thetis_solve");
    if (!lp) return THETIS_ERR_INVALID_ARG;
    if (!(beta > 0.0f) || !isfinite(beta) || epochs < 0 ||
        (mode < THETIS_MODE_DETERMINISTIC || mode > THETIS_MODE_ASYNC_HUBLAG_SERIAL) ||
        (step_rule != THETIS_STEP_LMAX && step_rule != THETIS_STEP_LJ))
        return set_error(lp, THETIS_ERR_INVALID_ARG, "bad arguments to thetis_solve");
    if (lp->anchors) THETIS_TRY(recompute_ua(lp));
    THETIS_TRY(solve_epochs(lp, beta, epochs, mode, seed, step_rule, stats));
    if (stats) {
        stats->coordinate_updates = lp->epoch_updates * epochs;
        stats->nnz_processed = lp->epoch_nnz * epochs;
    }
    return THETIS_OK;
}

THETIS_API int thetis_solve_alm(thetis_lp* lp, float* ubar, float* zbar, float beta0, float beta_growth,
                                int max_outer, int inner_epochs, int mode, uint64_t seed, int step_rule,
                                double target_eps, thetis_alm_stats* stats) {
    thetis::NvtxRange nvtx_("thetis_solve_alm");
    if (!lp) return THETIS_ERR_INVALID_ARG;
    if (!ubar || !zbar || !is_device_ptr(ubar) || !is_device_ptr(zbar) || !(beta0 > 0.0f) || !isfinite(beta0) ||
        !(beta_growth >= 1.0f) || !isfinite(beta_growth) || max_outer < 1 || max_outer > THETIS_MAX_ALM_ROUNDS ||
        inner_epochs < 0 ||
        (mode < THETIS_MODE_DETERMINISTIC || mode > THETIS_MODE_ASYNC_HUBLAG_SERIAL) ||
        (step_rule != THETIS_STEP_LMAX && step_rule != THETIS_STEP_LJ))
        return set_error(lp, THETIS_ERR_INVALID_ARG, "bad arguments to thetis_solve_alm");
    THETIS_TRY(thetis_set_anchors(lp, zbar, ubar));
    if (stats) memset(stats, 0, sizeof(*stats));
    float beta = beta0;
    double prev_res = INFINITY;
    for (int t = 0; t < max_outer; t++) {
        thetis_solve_stats st;
        THETIS_TRY(solve_epochs(lp, beta, inner_epochs, mode, seed + (uint64_t)t, step_rule, stats ? &st : nullptr));
        thetis_objective_t ob;
        const int rc = objective(lp, beta, &ob);
        if (stats) {
            stats->rounds = t + 1;
            stats->epochs_total += inner_epochs;
            stats->ms_total += st.ms_total;
            stats->beta[t] = beta;
            stats->eps[t] = ob.max_violation_eps;
            stats->resid_inf[t] = ob.resid_inf;
            stats->lp_obj[t] = ob.lp_obj;
        }
        if (rc != THETIS_OK) return rc;
        if (ob.max_violation_eps <= target_eps || t + 1 == max_outer) break;
        THETIS_TRY(alm_update(lp, ubar, zbar, beta));  // ubar -= beta r, zbar = z, then u^T a_j
        if (ob.resid_inf > 0.5 * prev_res) beta = (float)((double)beta * (double)beta_growth);
        prev_res = ob.resid_inf;
    }
    return THETIS_OK;
}

THETIS_API int thetis_objective(thetis_lp* lp, float beta, thetis_objective_t* out) {
    thetis::NvtxRange nvtx_("thetis_objective");
    if (!lp || !out || !(beta > 0.0f)) return lp ? set_error(lp, THETIS_ERR_INVALID_ARG, "bad arguments") : THETIS_ERR_INVALID_ARG;
    return objective(lp, beta, out);
}

THETIS_API int thetis_round_x(thetis_lp* lp, const float* x, int rule, uint64_t seed, int reps, uint8_t* out_assign,
                              thetis_round_result* out) {
    thetis::NvtxRange nvtx_("thetis_round_x");
    if (!lp || !x || !out) return THETIS_ERR_INVALID_ARG;
    const float* xd = x;
    if (!is_device_ptr(x)) {
        float* stage = (float*)lp->temp; // first slot of the rounding temp layout
        if (lp->d.n_s > 0)
            CUDA_TRY(lp, cudaMemcpyAsync(stage, x, (size_t)lp->d.n_s * 4, cudaMemcpyHostToDevice, lp->stream));
        xd = stage;
    }
    return round_x(lp, xd, rule, seed, reps, out_assign, out);
}

THETIS_API int thetis_round(thetis_lp* lp, int rule, uint64_t seed, int reps, uint8_t* out_assign,
                            thetis_round_result* out) {
    thetis::NvtxRange nvtx_("thetis_round");
    if (!lp || !out) return THETIS_ERR_INVALID_ARG;
    return round_x(lp, lp->d.z, rule, seed, reps, out_assign, out);
}

THETIS_API int thetis_get_csc(const thetis_lp* lp, int64_t* colptr, int32_t* rowidx, float* val) {
    if (!lp) return THETIS_ERR_INVALID_ARG;
    const DevLP& d = lp->d;
    if (colptr) THETIS_TRY(copy_out(lp, colptr, d.colptr, (size_t)(d.n_s + 1) * 8));
    if (rowidx) THETIS_TRY(copy_out(lp, rowidx, d.rowidx, (size_t)d.nnz_s * 4));
    if (val) {
        if (d.val) {
            THETIS_TRY(copy_out(lp, val, d.val, (size_t)d.nnz_s * 4));
        } else {
            std::vector<int32_t> ri(d.nnz_s);
            std::vector<float> v(d.nnz_s);
            THETIS_TRY(copy_out(lp, ri.data(), d.rowidx, (size_t)d.nnz_s * 4));
            for (int64_t t = 0; t < d.nnz_s; t++) v[t] = ((uint32_t)ri[t] & kSignBit) ? -1.0f : 1.0f;
            thetis_lp* l = const_cast<thetis_lp*>(lp);
            if (d.nnz_s > 0) CUDA_TRY(l, cudaMemcpy(val, v.data(), (size_t)d.nnz_s * 4, cudaMemcpyDefault));
        }
    }
    return THETIS_OK;
}

THETIS_API int thetis_get_edges(const thetis_lp* lp, int32_t* eu, int32_t* ev) {
    if (!lp) return THETIS_ERR_INVALID_ARG;
    const DevLP& d = lp->d;
    if (!d.edges || d.m_edges == 0) return THETIS_OK;
    std::vector<int2> e(d.m_edges);
    THETIS_TRY(copy_out(lp, e.data(), d.edges, (size_t)d.m_edges * 8));
    std::vector<int32_t> a(d.m_edges), b(d.m_edges);
    for (int64_t i = 0; i < d.m_edges; i++) { a[i] = e[i].x; b[i] = e[i].y; }
    thetis_lp* l = const_cast<thetis_lp*>(lp);
    if (eu) CUDA_TRY(l, cudaMemcpy(eu, a.data(), (size_t)d.m_edges * 4, cudaMemcpyDefault));
    if (ev) CUDA_TRY(l, cudaMemcpy(ev, b.data(), (size_t)d.m_edges * 4, cudaMemcpyDefault));
    return THETIS_OK;
}

THETIS_API int thetis_get_colouring(thetis_lp* lp, uint64_t seed, int32_t* colour, int64_t* n_colours) {
    if (!lp || !colour) return THETIS_ERR_INVALID_ARG;
    THETIS_TRY(ensure_colouring(lp, seed));
    const DevLP& d = lp->d;
    const int64_t S = d.n_blocks + d.n_scalar;
    std::vector<int32_t> h(d.U);
    if (S > 0) THETIS_TRY(copy_out(lp, h.data(), lp->colour, (size_t)S * 4));
    for (int64_t u = 0; u < S; u++) h[u] = h[u] < 0 ? -1 : h[u];
    for (int64_t u = S; u < d.U; u++) h[u] = (int32_t)lp->K;
    if (d.U > 0) CUDA_TRY(lp, cudaMemcpy(colour, h.data(), (size_t)d.U * 4, cudaMemcpyDefault));
    if (n_colours) *n_colours = lp->K;
    return THETIS_OK;
}

THETIS_API int thetis_tile_perm(int64_t n_tiles, uint64_t seed, int64_t epoch, int64_t* out, void* stream) {
    if (n_tiles < 0 || (n_tiles > 0 && !out) || epoch < 0) return THETIS_ERR_INVALID_ARG;
    return launch_tile_perm(n_tiles, seed, epoch, out, (cudaStream_t)stream);
}

THETIS_API int thetis_sync(thetis_lp* lp) {
    if (!lp) return THETIS_ERR_INVALID_ARG;
    CUDA_TRY(lp, cudaStreamSynchronize(lp->stream));
    return check_cuda(lp, "sync");
}

THETIS_API void thetis_free(thetis_lp* lp) {
    if (!lp) return;
    cudaStreamSynchronize(lp->stream);
    if (lp->side) cudaStreamSynchronize(lp->side);
    destroy(lp);
}

}  // extern "C"
