// K10-K12: rounding of a fractional point (§2, App. C).
//   VC_HALF  : eps = max_e (1 - (x_u + x_v))_+ ; select x_v >= (1 - eps)/2 (Lemma 1,
//              Pi(x/(1-eps)) >= 1/2), fall back to 1/2 when eps >= 1;
//              then every uncovered edge adds its endpoint with larger x (ties:
//              smaller cost, then smaller id), judged against the pre-fix-up set.
//   VC_FIXUP : threshold 1/2 on x, same fix-up.
//   MIS      : alpha = max_e (x_u + x_v - 1)_+ (App. C.2); greedy repair
//              = the lexicographically-first maximal independent set in the order
//              (x desc, w desc, id asc), computed by parallel rounds.
//   MWC_CKR  : CKR region growing (Vazirani Alg. 19.4): theta = 1 - rho,
//              random label order sigma; best of `reps`.
// Decisions are taken in fp32 on the given x; sums in fp64 with fixed combine order.
#include "thetis_internal.cuh"

namespace thetis {
namespace {

constexpr int T = 256;
constexpr int kMaxReps = 64;

struct CkrParams {
    float theta[kMaxReps];
    uint8_t sigma[kMaxReps][kMaxK];
};

__device__ __forceinline__ void atomic_max_nonneg(float* p, float v) {
    if (v > 0.0f) atomicMax((int*)p, __float_as_int(v));
}
// max over the block (non-negative floats compare like their bit patterns), one
// atomic per block
__device__ __forceinline__ void block_max_nonneg(float* p, float v) {
    __shared__ float sh[32];
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0f;
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) atomic_max_nonneg(p, v);
    }
}

// ---------------- VC
__global__ void k_vc_eps(int64_t m, const int2* __restrict__ edges, const float* __restrict__ x, float* eps) {
    float best = 0.0f;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        int2 uv = edges[e];
        best = fmaxf(best, __fsub_rn(1.0f, __fadd_rn(x[uv.x], x[uv.y])));
    }
    block_max_nonneg(eps, best);
}
__global__ void k_vc_select(int64_t n, int rule, const float* __restrict__ x, const float* eps_p, uint8_t* sel,
                            uint8_t* add, int32_t* fallback) {
    const float eps = *eps_p;
    float tau = 0.5f;
    if (rule == THETIS_ROUND_VC_HALF) {
        if (eps < 1.0f) tau = __fmul_rn(__fsub_rn(1.0f, eps), 0.5f);
        else if (blockIdx.x == 0 && threadIdx.x == 0) *fallback = 1;
    }
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        sel[v] = x[v] >= tau ? 1 : 0;
        add[v] = 0;
    }
}
__global__ void k_vc_fixup(int64_t m, const int2* __restrict__ edges, const float* __restrict__ x,
                           const float* __restrict__ c, const uint8_t* __restrict__ sel, uint8_t* add) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        int2 uv = edges[e];
        if (sel[uv.x] || sel[uv.y]) continue;
        int pick;
        float xu = x[uv.x], xv = x[uv.y];
        if (xu != xv) pick = xu > xv ? uv.x : uv.y;
        else if (c[uv.x] != c[uv.y]) pick = c[uv.x] < c[uv.y] ? uv.x : uv.y;
        else pick = uv.x < uv.y ? uv.x : uv.y;
        add[pick] = 1;
    }
}

// per-vertex merge + deterministic partial sums of (cost, selected, added)
__global__ void __launch_bounds__(T) k_vc_merge(int64_t n, const float* __restrict__ c, uint8_t* sel,
                                                const uint8_t* __restrict__ add, double* partial) {
    double cost = 0.0, cnt = 0.0, added = 0.0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        uint8_t s = sel[v];
        if (add[v] && !s) { s = 1; sel[v] = 1; added += 1.0; }
        if (s) { cost += (double)c[v]; cnt += 1.0; }
    }
    __shared__ double sh[3][T];
    sh[0][threadIdx.x] = cost; sh[1][threadIdx.x] = cnt; sh[2][threadIdx.x] = added;
    __syncthreads();
    for (int off = T / 2; off > 0; off >>= 1) {
        if ((int)threadIdx.x < off)
            for (int q = 0; q < 3; q++) sh[q][threadIdx.x] += sh[q][threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x < 3) partial[blockIdx.x * 4 + threadIdx.x] = sh[threadIdx.x][0];
}
__global__ void k_count_bad_edges(int64_t m, const int2* __restrict__ edges, const uint8_t* __restrict__ sel,
                                  int want_cover, unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        int2 uv = edges[e];
        bool s = sel[uv.x], t = sel[uv.y];
        b += want_cover ? (!s && !t) : (s && t);
    }
    for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, b);
}
__global__ void k_sum_partials(int blocks, int width, const double* partial, double* out) {
    int q = threadIdx.x;
    if (q >= width) return;
    double acc = 0.0;
    for (int b = 0; b < blocks; b++) acc += partial[b * 4 + q];
    out[q] = acc;
}

// ---------------- set cover (generic covering LP: rows sum_{s in row} x_s >= 1)
// precondition, eps = max_rows (1 - sum x)_+ (fp32, CSR order) and f = max row count
__global__ void __launch_bounds__(T) k_sc_rows(const DevLP L, const float* __restrict__ x, float* eps, int32_t* f,
                                               int32_t* bad) {
    float best = 0.0f;
    int fm = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.m; i += (int64_t)gridDim.x * blockDim.x) {
        if (L.sense[i] != THETIS_GE || L.b[i] != 1.0f) atomicOr(bad, 1);
        float sum = 0.0f;
        for (int64_t t = L.rowptr[i]; t < L.rowptr[i + 1]; t++) {
            if (L.rval && L.rval[t] != 1.0f) atomicOr(bad, 1);
            sum = __fadd_rn(sum, x[L.rcol[t]]);
        }
        best = fmaxf(best, __fsub_rn(1.0f, sum));
        const int cnt = (int)(L.rowptr[i + 1] - L.rowptr[i]);
        fm = cnt > fm ? cnt : fm;
    }
    for (int o = 16; o; o >>= 1) fm = max(fm, __shfl_xor_sync(0xffffffffu, fm, o));
    if ((threadIdx.x & 31) == 0 && fm) atomicMax(f, fm);
    block_max_nonneg(eps, best);
}
__device__ __forceinline__ float sc_uniform(uint64_t seed, int64_t s) {
    uint64_t z = seed ^ (0x5851F42D4C957F2DULL * (uint64_t)(s + 1));
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return ((float)(z >> 40) + 0.5f) * (1.0f / 16777216.0f);  // exact: 24-bit integer + 1/2, times 2^-24
}
__global__ void k_sc_select(int64_t n, int rule, const float* __restrict__ x, const float* eps_p, const int32_t* f_p,
                            float d, uint64_t seed, uint8_t* sel, uint8_t* add, int32_t* fallback) {
    const float eps = *eps_p;
    const float f = (float)*f_p;
    float tau = f > 0.0f ? __fdiv_rn(1.0f, f) : 1.0f;
    if (rule == THETIS_ROUND_SC_THRESHOLD) {
        if (eps < 1.0f) tau = __fdiv_rn(__fsub_rn(1.0f, eps), f);
        else if (blockIdx.x == 0 && threadIdx.x == 0) *fallback = 1;
    }
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        if (rule == THETIS_ROUND_SC_THRESHOLD) {
            sel[s] = x[s] >= tau ? 1 : 0;
        } else {
            const float p = fminf(1.0f, __fmul_rn(d, x[s]));
            sel[s] = sc_uniform(seed, s) < p ? 1 : 0;
        }
        add[s] = 0;
    }
}
// every element without a selected set adds its set with the largest x (ties: smaller
// cost, then smaller index); counts the uncovered elements
__global__ void k_sc_fixup(const DevLP L, const float* __restrict__ x, const uint8_t* __restrict__ sel, uint8_t* add,
                           unsigned long long* uncovered) {
    unsigned long long u = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = L.rowptr[i], b = L.rowptr[i + 1];
        bool covered = false;
        for (int64_t t = a; t < b && !covered; t++) covered = sel[L.rcol[t]];
        if (covered || a == b) continue;
        u++;
        int32_t pick = L.rcol[a];
        for (int64_t t = a + 1; t < b; t++) {
            const int32_t s = L.rcol[t];
            const float xs = x[s], xp = x[pick];
            if (xs > xp || (xs == xp && (L.c[s] < L.c[pick] || (L.c[s] == L.c[pick] && s < pick)))) pick = s;
        }
        add[pick] = 1;
    }
    for (int o = 16; o; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
    if ((threadIdx.x & 31) == 0 && u) atomicAdd(uncovered, u);
}
__global__ void k_sc_bad_rows(const DevLP L, const uint8_t* __restrict__ sel, unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.m; i += (int64_t)gridDim.x * blockDim.x) {
        bool covered = false;
        for (int64_t t = L.rowptr[i]; t < L.rowptr[i + 1] && !covered; t++) covered = sel[L.rcol[t]];
        b += !covered;
    }
    for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, b);
}

// ---------------- MIS, Bansal et al.'s Alg. 2 (theta = 1/k): bit t of mask[v] = v
// chosen in repetition t; a chosen vertex with a chosen neighbour is deleted
__device__ __forceinline__ float bansal_uniform(uint64_t seed, int t, int64_t v) {
    const uint64_t st = seed ^ (0xC2B2AE3D27D4EB4FULL * (uint64_t)(t + 1));
    return ((float)(sm64_mix(st + (uint64_t)(v + 1) * kGolden) >> 40) + 0.5f) * (1.0f / 16777216.0f);
}
__global__ void k_bansal_sample(int64_t n, const float* __restrict__ x, const float* alpha_p, uint64_t seed, int reps,
                                unsigned long long* mask, unsigned long long* del) {
    const float scale = __fadd_rn(1.0f, *alpha_p);
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const float p = __fdiv_rn(x[v], scale);  // x~ = x / (1 + alpha), probability x~ / (k theta)
        unsigned long long b = 0;
        for (int t = 0; t < reps; t++)
            if (bansal_uniform(seed, t, v) < p) b |= 1ull << t;
        mask[v] = b;
        del[v] = 0;
    }
}
__global__ void k_bansal_conflicts(int64_t m, const int2* __restrict__ edges, const unsigned long long* __restrict__ mask,
                                   unsigned long long* del) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const int2 uv = edges[e];
        const unsigned long long c = mask[uv.x] & mask[uv.y];
        if (c) {
            atomicOr(del + uv.x, c);
            atomicOr(del + uv.y, c);
        }
    }
}
__global__ void __launch_bounds__(T) k_bansal_weight(int64_t n, const float* __restrict__ w,
                                                     const unsigned long long* __restrict__ mask,
                                                     const unsigned long long* __restrict__ del, double* partial) {
    const int t = blockIdx.y;
    double acc = 0.0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (((mask[v] & ~del[v]) >> t) & 1ull) acc += (double)w[v];
    __shared__ double sh[T];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int off = T / 2; off > 0; off >>= 1) {
        if ((int)threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[(int64_t)t * gridDim.x + blockIdx.x] = sh[0];
}
__global__ void k_bansal_select(int64_t n, const unsigned long long* __restrict__ mask,
                                const unsigned long long* __restrict__ del, int best, uint8_t* sel) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        sel[v] = (uint8_t)(((mask[v] & ~del[v]) >> best) & 1ull);
}

// ---------------- MIS
__global__ void k_mis_alpha(int64_t m, const int2* __restrict__ edges, const float* __restrict__ x, float* alpha) {
    float best = 0.0f;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        int2 uv = edges[e];
        best = fmaxf(best, __fsub_rn(__fadd_rn(x[uv.x], x[uv.y]), 1.0f));
    }
    block_max_nonneg(alpha, best);
}
// w precedes v in (x desc, w desc, id asc)
__device__ __forceinline__ bool mis_precedes(float xw, float ww, int64_t w, float xv, float wv, int64_t v) {
    if (xw != xv) return xw > xv;
    if (ww != wv) return ww > wv;
    return w < v;
}
// state: 0 undecided, 1 in, 2 out
__global__ void k_mis_join(const DevLP L, const float* __restrict__ x, uint8_t* state) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < L.n_vert; v += (int64_t)gridDim.x * blockDim.x) {
        if (state[v] != 0) continue;
        const float xv = x[v], wv = L.c[v];
        bool join = true;
        for (int64_t t = L.colptr[v]; t < L.colptr[v + 1] && join; t++) {
            int2 e = L.edges[L.rowidx[t] & kRowMask];
            int64_t w = e.x == (int32_t)v ? e.y : e.x;
            uint8_t sw = ((volatile uint8_t*)state)[w];
            if (sw == 1) join = false;
            else if (sw == 0 && mis_precedes(x[w], L.c[w], w, xv, wv, v)) join = false;
        }
        if (join) state[v] = 1;
    }
}
__global__ void k_mis_drop(const DevLP L, uint8_t* state, unsigned long long* undecided) {
    unsigned long long left = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < L.n_vert; v += (int64_t)gridDim.x * blockDim.x) {
        if (state[v] != 0) continue;
        bool out = false;
        for (int64_t t = L.colptr[v]; t < L.colptr[v + 1] && !out; t++) {
            int2 e = L.edges[L.rowidx[t] & kRowMask];
            int64_t w = e.x == (int32_t)v ? e.y : e.x;
            if (state[w] == 1) out = true;
        }
        if (out) state[v] = 2;
        else left++;
    }
    for (int o = 16; o; o >>= 1) left += __shfl_xor_sync(0xffffffffu, left, o);
    if ((threadIdx.x & 31) == 0 && left) atomicAdd(undecided, left);
}
__global__ void k_mis_finish(int64_t n, uint8_t* state) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        state[v] = state[v] == 1 ? 1 : 0;
}

// ---------------- MWC
__global__ void k_mwc_check(const DevLP L, const float* __restrict__ x, int32_t* bad) {
    const int k = L.k;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < L.n_vert; v += (int64_t)gridDim.x * blockDim.x) {
        if (L.term_label[v] >= 0) continue;
        double s = 0.0;
        bool neg = false;
        for (int l = 0; l < k; l++) {
            float xv = x[v * k + l];
            if (!(xv >= 0.0f)) neg = true;
            s += (double)xv;
        }
        if (neg || fabs(s - 1.0) > 1e-4) atomicOr(bad, 1);
    }
}
__device__ __forceinline__ int ckr_label(const DevLP& L, const float* x, int64_t v, const CkrParams& C, int t) {
    int tl = L.term_label[v];
    if (tl >= 0) return tl;
    const int k = L.k;
    const float th = C.theta[t];
    for (int i = 0; i < k - 1; i++) {
        int l = C.sigma[t][i];
        if (x[v * k + l] >= th) return l;
    }
    return C.sigma[t][k - 1];
}
// blockIdx.y = repetition; deterministic per-block partial cut costs
__global__ void __launch_bounds__(T) k_mwc_cost(const DevLP L, const float* __restrict__ x, CkrParams C,
                                                double* partial) {
    const int t = blockIdx.y;
    double cost = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L.m_edges; e += (int64_t)gridDim.x * blockDim.x) {
        int2 uv = L.edges[e];
        if (ckr_label(L, x, uv.x, C, t) != ckr_label(L, x, uv.y, C, t)) cost += (double)L.ew[e];
    }
    __shared__ double sh[T];
    sh[threadIdx.x] = cost;
    __syncthreads();
    for (int off = T / 2; off > 0; off >>= 1) {
        if ((int)threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[(int64_t)t * gridDim.x + blockIdx.x] = sh[0];
}
__global__ void k_mwc_cost_final(int reps, int blocks, const double* partial, double* out) {
    int t = threadIdx.x;
    if (t >= reps) return;
    double acc = 0.0;
    for (int b = 0; b < blocks; b++) acc += partial[(int64_t)t * blocks + b];
    out[t] = acc;
}
__global__ void k_mwc_labels(const DevLP L, const float* __restrict__ x, CkrParams C, int t, uint8_t* lab) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < L.n_vert; v += (int64_t)gridDim.x * blockDim.x)
        lab[v] = (uint8_t)ckr_label(L, x, v, C, t);
}
__global__ void k_mwc_cut(const DevLP L, const uint8_t* __restrict__ lab, unsigned long long* cut) {
    unsigned long long c = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L.m_edges; e += (int64_t)gridDim.x * blockDim.x) {
        int2 uv = L.edges[e];
        c += lab[uv.x] != lab[uv.y];
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cut, c);
}

}  // namespace

int round_x(thetis_lp* lp, const float* x, int rule, uint64_t seed, int reps, uint8_t* out_assign,
            thetis_round_result* res) {
    const DevLP& L = lp->d;
    cudaStream_t s = lp->stream;
    memset(res, 0, sizeof(*res));
    const bool sc = rule == THETIS_ROUND_SC_THRESHOLD || rule == THETIS_ROUND_SC_RANDOM;
    const int64_t n = sc ? L.n_s : L.n_vert, m = L.m_edges;
    Carver C(lp->temp);
    C.take<float>(L.n_s); // staging of a host x (see thetis_round_x)
    uint8_t* sel = C.take<uint8_t>(n);
    uint8_t* add = C.take<uint8_t>(n);
    double* partial = C.take<double>(4 * (int64_t)kRedBlocks > (int64_t)kMaxReps * kRedBlocks
                                         ? 4 * (int64_t)kRedBlocks : (int64_t)kMaxReps * kRedBlocks);
    double* sums = C.take<double>(kMaxReps);
    int32_t* small = C.take<int32_t>(16); // eps/alpha as float, fallback, bad
    unsigned long long* cnt = C.take<unsigned long long>(4);
    if (C.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "rounding temp");
    const bool dev_out = out_assign && is_device_ptr(out_assign);
    uint8_t* selp = dev_out ? out_assign : sel;
    CUDA_TRY(lp, cudaMemsetAsync(small, 0, 64, s));
    CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 32, s));
    const int gv = grid_for(n, T), ge = grid_for(m, T);

    if (rule == THETIS_ROUND_VC_HALF || rule == THETIS_ROUND_VC_FIXUP) {
        if (L.problem != THETIS_PROB_VC) return set_error(lp, THETIS_ERR_NOT_SUPPORTED, "VC rounding needs a VC LP");
        float* eps = (float*)small;
        if (m > 0) k_vc_eps<<<ge, T, 0, s>>>(m, L.edges, x, eps);
        if (n > 0) k_vc_select<<<gv, T, 0, s>>>(n, rule, x, eps, selp, add, small + 1);
        if (m > 0) k_vc_fixup<<<ge, T, 0, s>>>(m, L.edges, x, L.c, selp, add);
        k_vc_merge<<<kRedBlocks, T, 0, s>>>(n, L.c, selp, add, partial);
        k_sum_partials<<<1, 32, 0, s>>>(kRedBlocks, 3, partial, sums);
        if (m > 0) k_count_bad_edges<<<ge, T, 0, s>>>(m, L.edges, selp, 1, cnt);
        double h[3];
        float he;
        int32_t fb;
        unsigned long long bad;
        CUDA_TRY(lp, cudaMemcpyAsync(h, sums, 24, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&he, eps, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&fb, small + 1, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&bad, cnt, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        res->cost = h[0];
        res->n_selected = (int64_t)h[1];
        res->rounds = (int64_t)h[2];
        res->eps_or_alpha = he;
        res->fallback = rule == THETIS_ROUND_VC_HALF ? fb : 0;
        res->feasible = bad == 0;
    } else if (rule == THETIS_ROUND_MIS_GREEDY) {
        if (L.problem != THETIS_PROB_MIS) return set_error(lp, THETIS_ERR_NOT_SUPPORTED, "MIS rounding needs an MIS LP");
        float* alpha = (float*)small;
        if (m > 0) k_mis_alpha<<<ge, T, 0, s>>>(m, L.edges, x, alpha);
        CUDA_TRY(lp, cudaMemsetAsync(selp, 0, (size_t)(n > 0 ? n : 1), s));
        int64_t rounds = 0;
        while (n > 0) {
            CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 8, s));
            k_mis_join<<<gv, T, 0, s>>>(L, x, selp);
            k_mis_drop<<<gv, T, 0, s>>>(L, selp, cnt);
            unsigned long long left = 0;
            CUDA_TRY(lp, cudaMemcpyAsync(&left, cnt, 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(lp, cudaStreamSynchronize(s));
            rounds++;
            if (left == 0) break;
        }
        if (n > 0) k_mis_finish<<<gv, T, 0, s>>>(n, selp);
        CUDA_TRY(lp, cudaMemsetAsync(add, 0, (size_t)(n > 0 ? n : 1), s));
        k_vc_merge<<<kRedBlocks, T, 0, s>>>(n, L.c, selp, add, partial);
        k_sum_partials<<<1, 32, 0, s>>>(kRedBlocks, 2, partial, sums);
        CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 8, s));
        if (m > 0) k_count_bad_edges<<<ge, T, 0, s>>>(m, L.edges, selp, 0, cnt);
        double h[2];
        float ha;
        unsigned long long bad;
        CUDA_TRY(lp, cudaMemcpyAsync(h, sums, 16, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&ha, alpha, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&bad, cnt, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        res->cost = h[0];
        res->n_selected = (int64_t)h[1];
        res->eps_or_alpha = ha;
        res->rounds = rounds;
        res->feasible = bad == 0;
    } else if (rule == THETIS_ROUND_MIS_BANSAL) {
        if (L.problem != THETIS_PROB_MIS) return set_error(lp, THETIS_ERR_NOT_SUPPORTED, "MIS rounding needs an MIS LP");
        if (reps < 1 || reps > kMaxReps) return set_error(lp, THETIS_ERR_INVALID_ARG, "reps must be in [1, 64]");
        float* alpha = (float*)small;
        Carver C2(lp->temp);
        C2.take<char>((int64_t)C.off);  // after this call's rounding temporaries
        unsigned long long* mask = C2.take<unsigned long long>(n > 0 ? n : 1);
        unsigned long long* del = C2.take<unsigned long long>(n > 0 ? n : 1);
        if (C2.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "rounding temp");
        if (m > 0) k_mis_alpha<<<ge, T, 0, s>>>(m, L.edges, x, alpha);
        if (n > 0) k_bansal_sample<<<gv, T, 0, s>>>(n, x, alpha, seed, reps, mask, del);
        if (m > 0) k_bansal_conflicts<<<ge, T, 0, s>>>(m, L.edges, mask, del);
        const int blocks = kRedBlocks;
        dim3 grid(blocks, reps);
        k_bansal_weight<<<grid, T, 0, s>>>(n, L.c, mask, del, partial);
        k_mwc_cost_final<<<1, kMaxReps, 0, s>>>(reps, blocks, partial, sums);
        double hw[kMaxReps];
        float ha;
        CUDA_TRY(lp, cudaMemcpyAsync(hw, sums, (size_t)reps * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&ha, alpha, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        int best = 0;
        for (int t = 1; t < reps; t++)
            if (hw[t] > hw[best]) best = t;
        if (n > 0) k_bansal_select<<<gv, T, 0, s>>>(n, mask, del, best, selp);
        CUDA_TRY(lp, cudaMemsetAsync(add, 0, (size_t)(n > 0 ? n : 1), s));
        k_vc_merge<<<kRedBlocks, T, 0, s>>>(n, L.c, selp, add, partial);
        k_sum_partials<<<1, 32, 0, s>>>(kRedBlocks, 2, partial, sums);
        CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 8, s));
        if (m > 0) k_count_bad_edges<<<ge, T, 0, s>>>(m, L.edges, selp, 0, cnt);
        double h[2];
        unsigned long long bad;
        CUDA_TRY(lp, cudaMemcpyAsync(h, sums, 16, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&bad, cnt, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        res->cost = hw[best];
        res->n_selected = (int64_t)h[1];
        res->eps_or_alpha = ha;
        res->best_rep = best;
        res->feasible = bad == 0;
    } else if (rule == THETIS_ROUND_MWC_CKR) {
        if (L.problem != THETIS_PROB_MWC) return set_error(lp, THETIS_ERR_NOT_SUPPORTED, "MWC rounding needs an MWC LP");
        if (reps < 1 || reps > kMaxReps) return set_error(lp, THETIS_ERR_INVALID_ARG, "reps must be in [1, 64]");
        int32_t* bad = small + 2;
        if (n > 0) k_mwc_check<<<gv, T, 0, s>>>(L, x, bad);
        int32_t hb = 0;
        CUDA_TRY(lp, cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        if (hb) return set_error(lp, THETIS_ERR_ROUND_PRECONDITION, "a free vertex block is not on the simplex");
        // (theta_t, sigma_t) from SplitMix64 seeded with seed ^ (0xD1B54A32D192ED03 (t+1))
        CkrParams P{};
        const int k = L.k;
        for (int t = 0; t < reps; t++) {
            uint64_t st = seed ^ (0xD1B54A32D192ED03ULL * (uint64_t)(t + 1));
            uint64_t h0 = sm64_mix(st + kGolden);
            P.theta[t] = (float)(((double)(h0 >> 41) + 0.5) * 0x1p-23);
            int sg[kMaxK];
            for (int l = 0; l < k; l++) sg[l] = l;
            for (int i = k - 1; i >= 1; i--) {
                uint64_t h = sm64_mix(st + (uint64_t)(k - i + 1) * kGolden);
                int j = (int)(h % (uint64_t)(i + 1));
                int tmp = sg[i]; sg[i] = sg[j]; sg[j] = tmp;
            }
            for (int l = 0; l < k; l++) P.sigma[t][l] = (uint8_t)sg[l];
        }
        const int blocks = kRedBlocks;
        dim3 grid(blocks, reps);
        k_mwc_cost<<<grid, T, 0, s>>>(L, x, P, partial);
        k_mwc_cost_final<<<1, kMaxReps, 0, s>>>(reps, blocks, partial, sums);
        double hc[kMaxReps];
        CUDA_TRY(lp, cudaMemcpyAsync(hc, sums, (size_t)reps * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        int best = 0;
        for (int t = 1; t < reps; t++)
            if (hc[t] < hc[best]) best = t;
        if (n > 0) k_mwc_labels<<<gv, T, 0, s>>>(L, x, P, best, selp);
        if (m > 0) k_mwc_cut<<<ge, T, 0, s>>>(L, selp, cnt);
        unsigned long long cut = 0;
        CUDA_TRY(lp, cudaMemcpyAsync(&cut, cnt, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        res->cost = hc[best];
        res->best_rep = best;
        res->feasible = 1;
        res->n_selected = (int64_t)cut;
    } else if (sc) {
        if (L.problem != THETIS_PROB_GENERIC || L.n_blocks > 0 || L.obj_sense != THETIS_MIN)
            return set_error(lp, THETIS_ERR_NOT_SUPPORTED, "set-cover rounding needs a generic covering LP");
        float* eps = (float*)small;
        int32_t* f = small + 2;
        int32_t* bad_in = small + 3;
        const int gr = grid_for(L.m, T);
        if (L.m > 0) k_sc_rows<<<gr, T, 0, s>>>(L, x, eps, f, bad_in);
        int32_t hb = 0;
        CUDA_TRY(lp, cudaMemcpyAsync(&hb, bad_in, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        if (hb) return set_error(lp, THETIS_ERR_ROUND_PRECONDITION, "set-cover rounding: a row is not sum x >= 1");
        const float d = (float)ceil(log(2.0 * (double)(L.m > 0 ? L.m : 1)));
        if (n > 0) k_sc_select<<<gv, T, 0, s>>>(n, rule, x, eps, f, d, seed, selp, add, small + 1);
        if (L.m > 0) k_sc_fixup<<<gr, T, 0, s>>>(L, x, selp, add, cnt + 1);
        k_vc_merge<<<kRedBlocks, T, 0, s>>>(n, L.c, selp, add, partial);
        k_sum_partials<<<1, 32, 0, s>>>(kRedBlocks, 3, partial, sums);
        if (L.m > 0) k_sc_bad_rows<<<gr, T, 0, s>>>(L, selp, cnt);
        double h[3];
        float he;
        int32_t fb;
        unsigned long long bad[2];
        CUDA_TRY(lp, cudaMemcpyAsync(h, sums, 24, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&he, eps, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(&fb, small + 1, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(bad, cnt, 16, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        res->cost = h[0];
        res->n_selected = (int64_t)h[1];
        res->rounds = (int64_t)h[2];
        res->eps_or_alpha = he;
        res->fallback = rule == THETIS_ROUND_SC_THRESHOLD ? fb : (bad[1] > 0);
        res->feasible = bad[0] == 0;
    } else {
        return set_error(lp, THETIS_ERR_INVALID_ARG, "unknown rounding rule %d", rule);
    }
    if (out_assign && !dev_out && n > 0) {
        CUDA_TRY(lp, cudaMemcpyAsync(out_assign, selp, (size_t)n, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
    }
    return check_cuda(lp, "round");
}

}  // namespace thetis
