// K5-K8: the SCD hot loop (Alg. 1) on f_beta (Eq. 5).
//
// Per unit j (a column of A_std, or a k-block of columns):
//   D   = a_j^T r                      (r = A z - b kept resident in HBM / L2)
//   g   = c_j - ubar^T a_j + beta D + (z_j - zbar_j) / beta    (Eq. 5 differentiated)
//   z_j <- clamp(z_j - g / L, lo_j, hi_j)  (Alg. 1 line 4; blocks: simplex projection,
//                                           App. E)
//   r  += a_j (z_j' - z_j)
//
// Deterministic mode (R-5): one launch per colour class; units of a class share no
// row, so plain loads / stores on r are race free and the result equals the
// sequential sweep.  The fp32 operation sequence is fixed (DESIGN.md §Arithmetic
// contract): sequential sum over the column in CSC order, each op rounded
// separately (__fadd_rn / __fmul_rn / __fdiv_rn), so it is bit-identical to the
// fp32 build of the oracle.
//
// Async mode (R-6): tiles of 32 consecutive units in a per-epoch keyed
// permutation; one persistent kernel, a warp per tile, tile-synchronous inside
// the tile (all gathers, then all scatters), Hogwild across tiles: r is read
// with L2 loads (ld.global.cg; stale values allowed) and written with
// red.global.add.f32, so no update is lost.  Scalar-column tiles are processed
// cooperatively: the tile's nonzeros are one contiguous CSC range, read
// coalesced 32 at a time; a tile with more than kHeavy nonzeros is finished by
// its whole CTA at its place in the sequence.  The grid bounds the number of
// tiles in flight to ~n_tiles / kAsyncDepth (bounded staleness).
#include "thetis_internal.cuh"

namespace thetis {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int64_t kHeavy = 2048;    // async: scalar nnz per tile above which a CTA takes it
constexpr int64_t kDetWarpCol = 64; // det: columns longer than this use the warp path

struct StepParams {
    float beta;       // caller's beta
    float inv_beta_unused;
    float invLmax;    // (float)(1 / L_max), L_max in fp64 (Eq. 7)
    double beta_d;    // (double)beta
    int rule;         // THETIS_STEP_LMAX / THETIS_STEP_LJ
};

__device__ __forceinline__ float ld_cg(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void red_add(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__device__ __forceinline__ float unit_invL(const StepParams& P, double norm2) {
    if (P.rule == THETIS_STEP_LMAX) return P.invLmax;
    return (float)(1.0 / (P.beta_d * norm2 + 1.0 / P.beta_d));
}

// g = c - ua + beta D + (z - zbar)/beta, each operation rounded on its own
__device__ __forceinline__ float grad_from(float c, float ua, float D, float z, float zb, float beta) {
    float g = __fsub_rn(c, ua);
    g = __fadd_rn(g, __fmul_rn(beta, D));
    g = __fadd_rn(g, __fdiv_rn(__fsub_rn(z, zb), beta));
    return g;
}
__device__ __forceinline__ float clamp_lohi(float t, float lo, float hi) {
    float zn = t < lo ? lo : t;
    return zn > hi ? hi : zn;
}

// sequential dot over column j in CSC order (the arithmetic contract)
template <bool kAsync>
__device__ __forceinline__ float col_dot_seq(const DevLP& L, int64_t j) {
    float D = 0.0f;
    for (int64_t t = L.colptr[j]; t < L.colptr[j + 1]; t++) {
        int64_t row;
        float a;
        entry(L, t, row, a);
        float rv = kAsync ? ld_cg(L.r + row) : L.r[row];
        D = __fadd_rn(D, L.val ? __fmul_rn(a, rv) : (a < 0.0f ? -rv : rv));
    }
    return D;
}
template <bool kAsync>
__device__ __forceinline__ void col_scatter(const DevLP& L, int64_t j, float d) {
    if (d == 0.0f) return;
    for (int64_t t = L.colptr[j]; t < L.colptr[j + 1]; t++) {
        int64_t row;
        float a;
        entry(L, t, row, a);
        float ad = L.val ? __fmul_rn(a, d) : (a < 0.0f ? -d : d);
        if (kAsync) red_add(L.r + row, ad);
        else L.r[row] = __fadd_rn(L.r[row], ad);
    }
}

__device__ __forceinline__ float zbar_of(const DevLP& L, int64_t j) { return L.zbar ? L.zbar[j] : 0.0f; }
__device__ __forceinline__ float ua_of(const DevLP& L, int64_t j) { return L.ubar ? L.ua[j] : 0.0f; }

// scalar structural column, one thread
template <bool kAsync>
__device__ __forceinline__ void update_scalar_seq(const DevLP& L, const StepParams& P, int64_t j) {
    float D = col_dot_seq<kAsync>(L, j);
    float z = L.z[j];
    float g = grad_from(c_int(L, j), ua_of(L, j), D, z, zbar_of(L, j), P.beta);
    float invL = unit_invL(P, col_norm2(L, j));
    float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), col_lo(L, j), col_hi(L, j));
    float d = __fsub_rn(zn, z);
    col_scatter<kAsync>(L, j, d);
    L.z[j] = zn;
}

// Euclidean projection onto the simplex (sort descending, ties: smaller index first)
__device__ __forceinline__ void project_simplex(const float* y, int k, float* x) {
    int idx[kMaxK];
    for (int l = 0; l < k; l++) idx[l] = l;
    for (int a = 1; a < k; a++) {
        int cur = idx[a], b = a - 1;
        while (b >= 0 && y[idx[b]] < y[cur]) { idx[b + 1] = idx[b]; b--; }
        idx[b + 1] = cur;
    }
    float s = 0.0f, s_rho = y[idx[0]];
    int rho = 1;
    for (int i = 1; i <= k; i++) {
        float u = y[idx[i - 1]];
        s = __fadd_rn(s, u);
        if (__fsub_rn(u, __fdiv_rn(__fsub_rn(s, 1.0f), (float)i)) > 0.0f) { rho = i; s_rho = s; }
    }
    float tau = __fdiv_rn(__fsub_rn(s_rho, 1.0f), (float)rho);
    for (int l = 0; l < k; l++) {
        float v = __fsub_rn(y[l], tau);
        x[l] = v > 0.0f ? v : 0.0f;
    }
}

// k-block (App. E): gradient step on the k columns, then projection on the simplex
template <bool kAsync>
__device__ __forceinline__ void update_block_seq(const DevLP& L, const StepParams& P, int64_t u) {
    const int k = L.k;
    const int64_t f = u * k;
    float y[kMaxK], x[kMaxK];
    double mx = 0.0;
    if (P.rule == THETIS_STEP_LJ)
        for (int l = 0; l < k; l++) {
            double q = col_norm2(L, f + l);
            mx = q > mx ? q : mx;
        }
    const float invL = unit_invL(P, mx);
    for (int l = 0; l < k; l++) {
        int64_t j = f + l;
        float D = col_dot_seq<kAsync>(L, j);
        float g = grad_from(c_int(L, j), ua_of(L, j), D, L.z[j], zbar_of(L, j), P.beta);
        y[l] = __fsub_rn(L.z[j], __fmul_rn(g, invL));
    }
    project_simplex(y, k, x);
    for (int l = 0; l < k; l++) {
        int64_t j = f + l;
        float d = __fsub_rn(x[l], L.z[j]);
        col_scatter<kAsync>(L, j, d);
        L.z[j] = x[l];
    }
}

// slack q of row i: a = sigma_i e_i, cost 0, bounds [0, inf)
template <bool kAsync>
__device__ __forceinline__ void update_slack(const DevLP& L, const StepParams& P, int64_t q) {
    const int64_t i = slack_row_of(L, q);
    const int64_t j = L.n_s + q;
    const float sig = row_sigma(L, i);
    float rv = kAsync ? ld_cg(L.r + i) : L.r[i];
    float D = __fadd_rn(0.0f, sig < 0.0f ? -rv : rv);
    float ua = 0.0f;
    if (L.ubar) ua = __fadd_rn(0.0f, sig < 0.0f ? -L.ubar[i] : L.ubar[i]);
    float z = L.z[j];
    float g = grad_from(0.0f, ua, D, z, zbar_of(L, j), P.beta);
    float invL = unit_invL(P, 1.0);
    float t = __fsub_rn(z, __fmul_rn(g, invL));
    float zn = t < 0.0f ? 0.0f : t;
    float d = __fsub_rn(zn, z);
    if (d != 0.0f) {
        float ad = sig < 0.0f ? -d : d;
        if (kAsync) red_add(L.r + i, ad);
        else L.r[i] = __fadd_rn(L.r[i], ad);
    }
    L.z[j] = zn;
}

// ------------------------------------------------------------ deterministic
// one colour class: members are structural units; long scalar columns are
// finished by their warp cooperatively with the same sequential summation order
__global__ void __launch_bounds__(256) k_det_class(DevLP L, StepParams P, const int32_t* __restrict__ members,
                                                   int64_t count) {
    const int lane = threadIdx.x & 31;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t warp_base = idx - lane;
    if (warp_base >= count) return;
    int64_t u = idx < count ? (int64_t)members[idx] : -1;
    bool deferred = false;
    if (u >= 0) {
        if (u < L.n_blocks) {
            update_block_seq<false>(L, P, u);
        } else {
            int64_t j = L.n_blocks * L.k + (u - L.n_blocks);
            if (L.colptr[j + 1] - L.colptr[j] > kDetWarpCol) deferred = true;
            else update_scalar_seq<false>(L, P, j);
        }
    }
    unsigned pending = __ballot_sync(0xffffffffu, deferred);
    while (pending) {
        const int src = __ffs(pending) - 1;
        pending &= pending - 1;
        const int64_t us = __shfl_sync(0xffffffffu, u, src);
        const int64_t j = L.n_blocks * L.k + (us - L.n_blocks);
        const int64_t beg = L.colptr[j], end = L.colptr[j + 1];
        float D = 0.0f;
        for (int64_t base = beg; base < end; base += 32) {
            int64_t t = base + lane;
            float v = 0.0f;
            if (t < end) {
                int64_t row;
                float a;
                entry(L, t, row, a);
                float rv = L.r[row];
                v = L.val ? __fmul_rn(a, rv) : (a < 0.0f ? -rv : rv);
            }
            const int lim = (int)((end - base) < 32 ? (end - base) : 32);
            for (int q = 0; q < lim; q++) D = __fadd_rn(D, __shfl_sync(0xffffffffu, v, q));
        }
        float z = L.z[j];
        float g = grad_from(c_int(L, j), ua_of(L, j), D, z, zbar_of(L, j), P.beta);
        float invL = unit_invL(P, col_norm2(L, j));
        float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), col_lo(L, j), col_hi(L, j));
        float d = __fsub_rn(zn, z);
        if (d != 0.0f)
            for (int64_t t = beg + lane; t < end; t += 32) {
                int64_t row;
                float a;
                entry(L, t, row, a);
                float ad = L.val ? __fmul_rn(a, d) : (a < 0.0f ? -d : d);
                L.r[row] = __fadd_rn(L.r[row], ad);
            }
        if (lane == 0) L.z[j] = zn;
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256) k_det_slacks(DevLP L, StepParams P) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L.n_ineq; q += (int64_t)gridDim.x * blockDim.x)
        update_slack<false>(L, P, q);
}

// ------------------------------------------------------------ async
// scalar sub-range [a, b) of the tile's lanes
__device__ __forceinline__ void scalar_lanes(const DevLP& L, int64_t u0, int& a, int& b) {
    const int64_t s0 = L.n_blocks, s1 = L.n_blocks + L.n_scalar;
    int64_t lo = u0 > s0 ? u0 : s0, hi = u0 + 32 < s1 ? u0 + 32 : s1;
    if (hi < lo) hi = lo;
    a = (int)(lo - u0);
    b = (int)(hi - u0);
}

// new values of a k-block from the current (possibly stale) residual
__device__ __forceinline__ void block_values(const DevLP& L, const StepParams& P, int64_t u, float* x) {
    const int k = L.k;
    const int64_t f = u * k;
    float y[kMaxK];
    double mx = 0.0;
    if (P.rule == THETIS_STEP_LJ)
        for (int l = 0; l < k; l++) {
            double q = col_norm2(L, f + l);
            mx = q > mx ? q : mx;
        }
    const float invL = unit_invL(P, mx);
    for (int l = 0; l < k; l++) {
        int64_t j = f + l;
        float D = col_dot_seq<true>(L, j);
        float g = grad_from(c_int(L, j), ua_of(L, j), D, L.z[j], zbar_of(L, j), P.beta);
        y[l] = __fsub_rn(L.z[j], __fmul_rn(g, invL));
    }
    project_simplex(y, k, x);
}

struct WarpSmem {
    float acc[32];
    float d[32];
    int32_t head[32];
};

// column (lane index) of the nonzero at position base + lane: the segment heads
// falling in the chunk, max-scanned, carried over from the previous chunk
__device__ __forceinline__ int chunk_col(int lane, int ncols, int64_t cp, int64_t base, int64_t end, int32_t* head,
                                         int& carry) {
    head[lane] = -1;
    __syncwarp();
    if (lane < ncols && cp >= base && cp < base + 32 && cp < end) atomicMax(&head[(int)(cp - base)], lane);
    __syncwarp();
    int col = head[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int x = __shfl_up_sync(0xffffffffu, col, o);
        if (lane >= o) col = x > col ? x : col;
    }
    col = col > carry ? col : carry;
    carry = __shfl_sync(0xffffffffu, col, 31);
    __syncwarp();
    return col;
}

// One tile, one warp, tile-synchronous: every unit of the tile gathers from the
// residual as it is when the tile starts (stale w.r.t. other tiles in flight),
// then all units scatter.  Scalar columns are processed cooperatively over the
// tile's contiguous CSC range.  Returns true (warp-uniform) when the scalar range
// has more than heavy_limit nonzeros: the whole CTA then finishes it.
__device__ __forceinline__ bool async_tile_warp(const DevLP& L, const StepParams& P, int64_t tile, int lane,
                                                WarpSmem& sm, int64_t heavy_limit) {
    const int64_t u0 = tile * 32, u = u0 + lane;
    const bool is_block = u < L.U && u < L.n_blocks && !(L.unit_fixed && L.unit_fixed[u]);
    const bool is_slack = u < L.U && u >= L.n_blocks + L.n_scalar;
    float xb[kMaxK];
    if (is_block) block_values(L, P, u, xb);
    float ds = 0.0f, sig = 0.0f;
    int64_t srow = 0;
    if (is_slack) {
        const int64_t q = u - L.n_blocks - L.n_scalar, j = L.n_s + q;
        srow = slack_row_of(L, q);
        sig = row_sigma(L, srow);
        float rv = ld_cg(L.r + srow);
        float D = __fadd_rn(0.0f, sig < 0.0f ? -rv : rv);
        float ua = 0.0f;
        if (L.ubar) ua = __fadd_rn(0.0f, sig < 0.0f ? -L.ubar[srow] : L.ubar[srow]);
        float z = L.z[j];
        float g = grad_from(0.0f, ua, D, z, zbar_of(L, j), P.beta);
        float t = __fsub_rn(z, __fmul_rn(g, unit_invL(P, 1.0)));
        float zn = t < 0.0f ? 0.0f : t;
        ds = __fsub_rn(zn, z);
        L.z[j] = zn;
    }
    // scalar columns
    int a, b;
    scalar_lanes(L, u0, a, b);
    const int ncols = b - a;
    bool heavy = false, coop = false;
    int64_t j0 = 0, cp = 0, beg = 0, end = 0;
    if (ncols > 0) {
        j0 = L.n_blocks * L.k + (u0 + a - L.n_blocks);
        cp = lane < ncols ? L.colptr[j0 + lane] : 0;
        beg = __shfl_sync(0xffffffffu, cp, 0);
        end = L.colptr[j0 + ncols];
        heavy = end - beg > heavy_limit;
        coop = !heavy;
    }
    unsigned moved = 0;
    if (coop) {
        sm.acc[lane] = 0.0f;
        __syncwarp();
        int carry = 0;
        for (int64_t base = beg; base < end; base += 32) {
            const int col = chunk_col(lane, ncols, cp, base, end, sm.head, carry);
            const int64_t t = base + lane;
            if (t < end) {
                int64_t row;
                float av;
                entry(L, t, row, av);
                float rv = ld_cg(L.r + row);
                atomicAdd(&sm.acc[col], L.val ? av * rv : (av < 0.0f ? -rv : rv));
            }
        }
        __syncwarp();
        float d = 0.0f;
        if (lane < ncols && !(L.unit_fixed && L.unit_fixed[u0 + a + lane])) {
            const int64_t j = j0 + lane;
            float z = L.z[j];
            float g = grad_from(c_int(L, j), ua_of(L, j), sm.acc[lane], z, zbar_of(L, j), P.beta);
            float invL = unit_invL(P, col_norm2(L, j));
            float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), col_lo(L, j), col_hi(L, j));
            d = __fsub_rn(zn, z);
            L.z[j] = zn;
        }
        sm.d[lane] = d;
        moved = __ballot_sync(0xffffffffu, d != 0.0f);
    }
    __syncwarp();
    // scatter phase
    if (is_block) {
        for (int l = 0; l < L.k; l++) {
            const int64_t j = u * L.k + l;
            float d = __fsub_rn(xb[l], L.z[j]);
            col_scatter<true>(L, j, d);
            L.z[j] = xb[l];
        }
    }
    if (is_slack && ds != 0.0f) red_add(L.r + srow, sig < 0.0f ? -ds : ds);
    if (moved) {
        int carry = 0;
        for (int64_t base = beg; base < end; base += 32) {
            const int col = chunk_col(lane, ncols, cp, base, end, sm.head, carry);
            const int64_t t = base + lane;
            const float dc = sm.d[col];
            if (t < end && dc != 0.0f) {
                int64_t row;
                float av;
                entry(L, t, row, av);
                red_add(L.r + row, L.val ? av * dc : (av < 0.0f ? -dc : dc));
            }
        }
    }
    return heavy;
}

struct CtaSmem {
    float acc[32];
    float d[32];
    int64_t cp[33];
};

// the scalar range of a heavy tile, by the whole CTA (all threads call this)
__device__ __forceinline__ void async_tile_cta(const DevLP& L, const StepParams& P, int64_t tile, CtaSmem& sm) {
    const int64_t u0 = tile * 32;
    int a, b;
    scalar_lanes(L, u0, a, b);
    const int64_t j0 = L.n_blocks * L.k + (u0 + a - L.n_blocks);
    const int ncols = b - a;
    if (threadIdx.x <= (unsigned)ncols) sm.cp[threadIdx.x] = L.colptr[j0 + threadIdx.x];
    if (threadIdx.x < 32) sm.acc[threadIdx.x] = 0.0f;
    __syncthreads();
    const int64_t beg = sm.cp[0], end = sm.cp[ncols];
    for (int64_t t = beg + threadIdx.x; t < end; t += blockDim.x) {
        int lo = 0, hi = ncols - 1; // last column with start <= t
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (sm.cp[mid] <= t) lo = mid; else hi = mid - 1;
        }
        int64_t row;
        float av;
        entry(L, t, row, av);
        float rv = ld_cg(L.r + row);
        atomicAdd(&sm.acc[lo], L.val ? av * rv : (av < 0.0f ? -rv : rv));
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        float d = 0.0f;
        const int lane = threadIdx.x;
        if (lane < ncols && !(L.unit_fixed && L.unit_fixed[u0 + a + lane])) {
            const int64_t j = j0 + lane;
            float z = L.z[j];
            float g = grad_from(c_int(L, j), ua_of(L, j), sm.acc[lane], z, zbar_of(L, j), P.beta);
            float invL = unit_invL(P, col_norm2(L, j));
            float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), col_lo(L, j), col_hi(L, j));
            d = __fsub_rn(zn, z);
            L.z[j] = zn;
        }
        sm.d[lane] = d;
    }
    __syncthreads();
    for (int64_t t = beg + threadIdx.x; t < end; t += blockDim.x) {
        int lo = 0, hi = ncols - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (sm.cp[mid] <= t) lo = mid; else hi = mid - 1;
        }
        float dc = sm.d[lo];
        if (dc == 0.0f) continue;
        int64_t row;
        float av;
        entry(L, t, row, av);
        red_add(L.r + row, L.val ? av * dc : (av < 0.0f ? -dc : dc));
    }
    __syncthreads();
}

// Persistent: the CTA takes the next `group` consecutive positions of the
// permuted tile sequence per round (one per warp), then finishes their heavy
// scalar ranges together, in position order.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_async(DevLP L, StepParams P, PermKeys K, int64_t n_tiles,
                                                               int group, int64_t heavy_limit,
                                                               unsigned long long* next) {
    __shared__ WarpSmem wsm[kWarpsPerBlock];
    __shared__ CtaSmem csm;
    __shared__ int64_t heavy_tile[kWarpsPerBlock];
    __shared__ int64_t base_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (;;) {
        // dynamic scheduling: positions are handed out in sequence order
        if (threadIdx.x == 0) base_s = (int64_t)atomicAdd(next, (unsigned long long)group);
        __syncthreads();
        const int64_t base = base_s;
        if (base >= n_tiles) break;
        const int64_t t_idx = base + w;
        bool heavy = false;
        int64_t tile = -1;
        if (w < group && t_idx < n_tiles) {
            tile = (int64_t)tile_perm((uint64_t)t_idx, K);
            heavy = async_tile_warp(L, P, tile, lane, wsm[w], heavy_limit);
        }
        if (lane == 0) heavy_tile[w] = heavy ? tile : -1;
        __syncthreads();
        for (int h = 0; h < group; h++) {
            const int64_t ht = heavy_tile[h];
            if (ht >= 0) async_tile_cta(L, P, ht, csm);
        }
        __syncthreads();
    }
}

__global__ void k_tile_perm(PermKeys K, int64_t n, int64_t* out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = (int64_t)tile_perm((uint64_t)t, K);
}

}  // namespace

int launch_tile_perm(int64_t n_tiles, uint64_t seed, int64_t epoch, int64_t* out, cudaStream_t s) {
    if (n_tiles <= 0) return THETIS_OK;
    PermKeys K = make_perm_keys(n_tiles, seed, epoch);
    k_tile_perm<<<grid_for(n_tiles, 256), 256, 0, s>>>(K, n_tiles, out);
    return cudaGetLastError() == cudaSuccess ? THETIS_OK : THETIS_ERR_CUDA;
}

// Bounded staleness (the async scheme needs the number of concurrent
// updaters small relative to n): at most ~n_tiles / kAsyncDepth warps are in
// flight (< 0.8% of the tiles), and never more than the device holds at once
// (persistent grid); large LPs are bounded by the device, not by the depth.
constexpr int64_t kAsyncDepth = 128;
static int64_t async_blocks(thetis_lp* lp, int64_t n_tiles) {
    static int per_sm = 0, sms = 0;
    if (!per_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async, kWarpsPerBlock * 32, 0);
        if (per_sm < 1) per_sm = 1;
    }
    (void)lp;
    int64_t depth_cap = (n_tiles + kWarpsPerBlock * kAsyncDepth - 1) / (kWarpsPerBlock * kAsyncDepth);
    int64_t dev_cap = (int64_t)per_sm * sms;
    int64_t b = depth_cap < dev_cap ? depth_cap : dev_cap;
    return b < 1 ? 1 : b;
}

int solve_epochs(thetis_lp* lp, float beta, int epochs, int mode, uint64_t seed, int step_rule,
                 thetis_solve_stats* st) {
    const DevLP& L = lp->d;
    cudaStream_t s = lp->stream;
    StepParams P{};
    P.beta = beta;
    P.beta_d = (double)beta;
    P.rule = step_rule;
    const double Lmax = (double)beta * lp->maxnorm2 + 1.0 / (double)beta; // Eq. 7
    P.invLmax = (float)(1.0 / Lmax);
    if (mode == THETIS_MODE_DETERMINISTIC) THETIS_TRY(ensure_colouring(lp, seed));
    const bool timed = st != nullptr;
    if (timed) {
        if (lp->ev_epoch.empty()) {
            lp->ev_epoch.resize(THETIS_MAX_EPOCH_TIMES + 2);
            for (auto& e : lp->ev_epoch) CUDA_TRY(lp, cudaEventCreate(&e));
        }
    }
    const int64_t n_tiles = (L.U + 31) / 32;
    cudaEvent_t ev_start = timed ? lp->ev_epoch[0] : nullptr;
    if (timed) CUDA_TRY(lp, cudaEventRecord(ev_start, s));
    for (int e = 0; e < epochs; e++) {
        if (mode == THETIS_MODE_DETERMINISTIC) {
            for (int64_t c = 0; c < lp->K; c++) {
                int64_t beg = lp->class_ptr[c], cnt = lp->class_ptr[c + 1] - beg;
                if (cnt > 0) k_det_class<<<grid_for(cnt, 256, 1 << 30), 256, 0, s>>>(L, P, lp->members + beg, cnt);
            }
            if (L.n_ineq > 0) k_det_slacks<<<grid_for(L.n_ineq, 256), 256, 0, s>>>(L, P);
        } else {
            PermKeys K = make_perm_keys(n_tiles, seed, e);
            if (n_tiles > 0) {
                const bool serial = mode == THETIS_MODE_ASYNC_SERIAL;
                int64_t blocks = serial ? 1 : async_blocks(lp, n_tiles);
                unsigned long long* next = (unsigned long long*)(lp->flags + 56);
                CUDA_TRY(lp, cudaMemsetAsync(next, 0, 8, s));
                k_async<<<(unsigned)blocks, kWarpsPerBlock * 32, 0, s>>>(L, P, K, n_tiles,
                                                                         serial ? 1 : kWarpsPerBlock, kHeavy, next);
            }
        }
        if (timed && e < THETIS_MAX_EPOCH_TIMES) CUDA_TRY(lp, cudaEventRecord(lp->ev_epoch[e + 1], s));
    }
    THETIS_TRY(check_cuda(lp, "solve"));
    if (timed) {
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        memset(st, 0, sizeof(*st));
        st->epochs = epochs;
        st->L_max = Lmax;
        st->n_colours = mode == THETIS_MODE_DETERMINISTIC ? lp->K : 0;
        st->mode = mode;
        st->step_rule = step_rule;
        int last = epochs < THETIS_MAX_EPOCH_TIMES ? epochs : THETIS_MAX_EPOCH_TIMES;
        for (int e = 0; e < last; e++) {
            float ms = 0;
            CUDA_TRY(lp, cudaEventElapsedTime(&ms, lp->ev_epoch[e], lp->ev_epoch[e + 1]));
            st->ms_per_epoch[e] = ms;
            st->ms_total += ms;
        }
    }
    return THETIS_OK;
}

}  // namespace thetis
