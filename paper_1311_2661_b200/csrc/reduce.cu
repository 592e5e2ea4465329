// K9: fused reductions at the current point (Def. 2, Eq. 5).
// One pass over the coordinates and one over the rows (r recomputed from z in
// fp64, so f_beta follows its definition and the maintained r is checked for
// drift), fp64 accumulation with a fixed grid and fixed combine order, so the
// result is identical from run to run.
#include "thetis_internal.cuh"

namespace thetis {
namespace {

enum Q { Q_LIN = 0, Q_OBJ, Q_PROX, Q_R2, Q_UR, Q_SUMS, Q_RINF = Q_SUMS, Q_DRIFT, Q_EPS, Q_NONFIN, Q_ALL };

__device__ __forceinline__ double row_ax(const DevLP& L, int64_t i) {
    if (L.problem == THETIS_PROB_VC || L.problem == THETIS_PROB_MIS) {
        int2 e = L.edges[i];
        return (double)L.z[e.x] + (double)L.z[e.y];
    }
    if (L.problem == THETIS_PROB_MWC) {
        int64_t k = L.k, e = i / (2 * k), rem = i % (2 * k), l = rem >> 1;
        double sgn = (rem & 1) ? -1.0 : 1.0;
        int2 uv = L.edges[e];
        return sgn * ((double)L.z[(int64_t)uv.x * k + l] - (double)L.z[(int64_t)uv.y * k + l]) +
               (double)L.z[L.n_vert * k + e * k + l];
    }
    double s = 0.0;
    for (int64_t t = L.rowptr[i]; t < L.rowptr[i + 1]; t++)
        s += (L.rval ? (double)L.rval[t] : 1.0) * (double)L.z[L.rcol[t]];
    return s;
}

__global__ void __launch_bounds__(kRedThreads) k_reduce(DevLP L, double beta, double* partial) {
    double q[Q_ALL];
    for (int i = 0; i < Q_ALL; i++) q[i] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t j = tid; j < L.N; j += stride) {
        double z = (double)L.z[j];
        if (j < L.n_s) {
            q[Q_LIN] += (double)c_int(L, j) * z;
            q[Q_OBJ] += (double)L.c[j] * z;
        }
        double d = z - (L.zbar ? (double)L.zbar[j] : 0.0);
        q[Q_PROX] += d * d;
        if (!isfinite(z)) q[Q_NONFIN] = 1.0;
    }
    // rows four at a time: the edge and z gathers of four rows are in flight together
    constexpr int kU = 4;
    for (int64_t i0 = tid; i0 < L.m; i0 += kU * stride) {
        double axs[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const int64_t i = i0 + u * stride;
            axs[u] = i < L.m ? row_ax(L, i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
        const int64_t i = i0 + u * stride;
        if (i >= L.m) break;
        const double ax = axs[u];
        int64_t sl = row_slack_of(L, i);
        double sv = sl >= 0 ? (double)row_sigma(L, i) * (double)L.z[sl] : 0.0;
        double b = (double)row_b(L, i);
        double ri = ax + sv - b; // (A z - b)_i
        q[Q_R2] += ri * ri;
        q[Q_RINF] = fmax(q[Q_RINF], fabs(ri));
        if (L.ubar) q[Q_UR] += (double)L.ubar[i] * ri;
        double dr = fabs((double)L.r[i] - ri);
        if (dr > q[Q_DRIFT] || isnan(dr)) q[Q_DRIFT] = isnan(dr) ? (double)INFINITY : dr;
        if (!isfinite((double)L.r[i])) q[Q_NONFIN] = 1.0;
        int s = row_sense(L, i);
        double viol = s == THETIS_GE ? b - ax : (s == THETIS_LE ? ax - b : fabs(ax - b));
        q[Q_EPS] = fmax(q[Q_EPS], viol);
        }
    }
    __shared__ double sh[Q_ALL][kRedThreads];
    for (int i = 0; i < Q_ALL; i++) sh[i][threadIdx.x] = q[i];
    __syncthreads();
    for (int off = kRedThreads / 2; off > 0; off >>= 1) {
        if ((int)threadIdx.x < off)
            for (int i = 0; i < Q_ALL; i++) {
                double a = sh[i][threadIdx.x], b = sh[i][threadIdx.x + off];
                sh[i][threadIdx.x] = i < Q_SUMS ? a + b : fmax(a, b);
            }
        __syncthreads();
    }
    if (threadIdx.x < Q_ALL) partial[blockIdx.x * 16 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void k_reduce_final(int blocks, const double* partial, double* out) {
    int i = threadIdx.x;
    if (i >= Q_ALL) return;
    double acc = 0.0;
    for (int b = 0; b < blocks; b++) {
        double v = partial[b * 16 + i];
        acc = i < Q_SUMS ? acc + v : fmax(acc, v);
    }
    out[i] = acc;
}

}  // namespace

int objective(thetis_lp* lp, float beta, thetis_objective_t* out) {
    cudaStream_t s = lp->stream;
    double* partial = lp->red;
    double* res = lp->red + kRedBlocks * 16;
    k_reduce<<<kRedBlocks, kRedThreads, 0, s>>>(lp->d, (double)beta, partial);
    k_reduce_final<<<1, 32, 0, s>>>(kRedBlocks, partial, res);
    double h[Q_ALL];
    CUDA_TRY(lp, cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(lp, cudaStreamSynchronize(s));
    THETIS_TRY(check_cuda(lp, "objective"));
    const double b = (double)beta;
    out->lp_obj = h[Q_OBJ];
    out->f_beta = h[Q_LIN] - h[Q_UR] + 0.5 * b * h[Q_R2] + h[Q_PROX] / (2.0 * b); // Eq. 5
    out->resid_l2 = sqrt(h[Q_R2]);
    out->resid_inf = h[Q_RINF];
    out->max_violation_eps = h[Q_EPS];
    out->drift_inf = h[Q_DRIFT];
    out->nonfinite = h[Q_NONFIN] != 0.0;
    return out->nonfinite ? THETIS_ERR_DIVERGED : THETIS_OK;
}

}  // namespace thetis
