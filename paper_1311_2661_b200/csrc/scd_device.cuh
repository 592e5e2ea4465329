// Device helpers shared by the SCD kernels (scd.cu: deterministic classes, the
// hub-lag async schedule; async_pi.cu: the permutation-ordered async schedule).
// Product side; shares nothing with oracle/.  Included inside an anonymous
// namespace by each translation unit (internal linkage).
#pragma once
#include "thetis_internal.cuh"

namespace thetis {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int64_t kDetWarpCol = 32;  // det: columns longer than this use the warp path
constexpr int64_t kDetCtaCol = 1024; // ... and longer than this a CTA per 1024 contract lanes (k_det_long_*);
                                     // (8192 until round 2: a warp walking an 8192-entry column took ~0.12 ms per
                                     // class on config 3, 344 classes per epoch)

struct StepParams {
    float beta;       // caller's beta
    float inv_beta;   // fl(1 / beta), async kernels only
    float invLmax;    // (float)(1 / L_max), L_max in fp64 (Eq. 7)
    double beta_d;    // (double)beta
    int rule;         // THETIS_STEP_LMAX / THETIS_STEP_LJ
};

__device__ __forceinline__ float ld_cg(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
// streaming load of CSC indices (read once per pass; do not keep in L1)
__device__ __forceinline__ int32_t ld_cs_i32(const int32_t* p) {
    int32_t v;
    asm volatile("ld.global.cs.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void red_add(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__device__ __forceinline__ float unit_invL(const StepParams& P, double norm2) {
    if (P.rule == THETIS_STEP_LMAX) return P.invLmax;
    return (float)(1.0 / (P.beta_d * norm2 + 1.0 / P.beta_d));
}

// g = c - ua + beta D + (z - zbar)/beta, each operation rounded on its own (the
// deterministic contract); the async kernels (not bit-exact by nature) multiply
// by inv_beta = fl(1/beta) instead of dividing
__device__ __forceinline__ float grad_from(float c, float ua, float D, float z, float zb, float beta) {
    float g = __fsub_rn(c, ua);
    g = __fadd_rn(g, __fmul_rn(beta, D));
    g = __fadd_rn(g, __fdiv_rn(__fsub_rn(z, zb), beta));
    return g;
}
__device__ __forceinline__ float grad_fast(float c, float ua, float D, float z, float zb, float beta, float inv_beta) {
    float g = __fsub_rn(c, ua);
    g = __fadd_rn(g, __fmul_rn(beta, D));
    g = __fadd_rn(g, __fmul_rn(__fsub_rn(z, zb), inv_beta));
    return g;
}
__device__ __forceinline__ float clamp_lohi(float t, float lo, float hi) {
    float zn = t < lo ? lo : t;
    return zn > hi ? hi : zn;
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

// scalar structural column, one thread (the contract's column dot, thetis_internal.cuh)
template <bool kAsync>
__device__ __forceinline__ void update_scalar_seq(const DevLP& L, const StepParams& P, int64_t j) {
    float D = col_dot_tree_thread(L, j, L.r);
    float z = L.z[j];
    float g = grad_from(c_int(L, j), ua_of(L, j), D, z, zbar_of(L, j), P.beta);
    float invL = unit_invL(P, col_norm2(L, j));
    float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), col_lo(L, j), col_hi(L, j));
    float d = __fsub_rn(zn, z);
    col_scatter<kAsync>(L, j, d);
    L.z[j] = zn;
}

// Euclidean projection onto the simplex (sort descending, ties: smaller index first).
// KC >= k is the compile-time capacity: every loop runs to KC with a guard, so for
// small blocks the arrays stay in registers; the sorted order comes from ranks
// (rank_l = #{m : y_m > y_l, or y_m = y_l and m < l}), and the prefix sums add the
// sorted values one at a time in that order (the same operation sequence as a sort).
template <int KC>
__device__ __forceinline__ void project_simplex(const float* y, int k, float* x) {
    int rk[KC];
#pragma unroll
    for (int l = 0; l < KC; l++) {
        int c = 0;
#pragma unroll
        for (int m = 0; m < KC; m++)
            if (l < k && m < k && (y[m] > y[l] || (y[m] == y[l] && m < l))) c++;
        rk[l] = c;
    }
    float s = 0.0f, s_rho = 0.0f;
    int rho = 1;
#pragma unroll
    for (int i = 1; i <= KC; i++) {
        if (i > k) break;
        float u = 0.0f;
#pragma unroll
        for (int l = 0; l < KC; l++)
            if (l < k && rk[l] == i - 1) u = y[l];
        s = __fadd_rn(s, u);
        if (i == 1) s_rho = s;
        if (__fsub_rn(u, __fdiv_rn(__fsub_rn(s, 1.0f), (float)i)) > 0.0f) { rho = i; s_rho = s; }
    }
    float tau = __fdiv_rn(__fsub_rn(s_rho, 1.0f), (float)rho);
#pragma unroll
    for (int l = 0; l < KC; l++)
        if (l < k) {
            float v = __fsub_rn(y[l], tau);
            x[l] = v > 0.0f ? v : 0.0f;
        }
}

// k-block (App. E): gradient step on the k columns, then projection on the simplex
template <bool kAsync, int KC>
__device__ __forceinline__ void update_block_seq(const DevLP& L, const StepParams& P, int64_t u) {
    const int k = L.k;
    const int64_t f = u * k;
    float y[KC], x[KC];
    double mx = 0.0;
    if (P.rule == THETIS_STEP_LJ)
        for (int l = 0; l < k; l++) {
            double q = col_norm2(L, f + l);
            mx = q > mx ? q : mx;
        }
    const float invL = unit_invL(P, mx);
#pragma unroll
    for (int l = 0; l < KC; l++)
        if (l < k) {
            int64_t j = f + l;
            float D = col_dot_tree_thread(L, j, L.r);
            float g = grad_from(c_int(L, j), ua_of(L, j), D, L.z[j], zbar_of(L, j), P.beta);
            y[l] = __fsub_rn(L.z[j], __fmul_rn(g, invL));
        }
    project_simplex<KC>(y, k, x);
#pragma unroll
    for (int l = 0; l < KC; l++)
        if (l < k) {
            int64_t j = f + l;
            float d = __fsub_rn(x[l], L.z[j]);
            col_scatter<kAsync>(L, j, d);
            L.z[j] = x[l];
        }
}

// slack of row i (column j): a = sigma_i e_i, cost 0, bounds [0, inf); the new
// value from the row's residual rv
template <bool kFast>
__device__ __forceinline__ float slack_new(const DevLP& L, const StepParams& P, int64_t i, int64_t j, float sig,
                                           float rv, float z) {
    float D = __fadd_rn(0.0f, sig < 0.0f ? -rv : rv);
    float ua = 0.0f;
    if (L.ubar) ua = __fadd_rn(0.0f, sig < 0.0f ? -L.ubar[i] : L.ubar[i]);
    float g = kFast ? grad_fast(0.0f, ua, D, z, zbar_of(L, j), P.beta, P.inv_beta)
                    : grad_from(0.0f, ua, D, z, zbar_of(L, j), P.beta);
    float t = __fsub_rn(z, __fmul_rn(g, unit_invL(P, 1.0)));
    return t < 0.0f ? 0.0f : t;
}
// one slack step with a plain read-modify-write of r (rows of distinct slacks differ)
template <bool kFast>
__device__ __forceinline__ void update_slack(const DevLP& L, const StepParams& P, int64_t q) {
    const int64_t i = slack_row_of(L, q);
    const int64_t j = L.n_s + q;
    const float sig = row_sigma(L, i);
    const float rv = L.r[i];
    const float z = L.z[j];
    const float zn = slack_new<kFast>(L, P, i, j, sig, rv, z);
    const float d = __fsub_rn(zn, z);
    if (d != 0.0f) L.r[i] = __fadd_rn(rv, sig < 0.0f ? -d : d);
    L.z[j] = zn;
}

// ------------------------------------------------------------ async
constexpr int kBatch = 16;         // permuted positions drawn per atomic by a warp (large grids)

// scalar sub-range [a, b) of the tile's lanes (tiles cover the structural units)
__device__ __forceinline__ void scalar_lanes(const DevLP& L, int64_t u0, int& a, int& b) {
    const int64_t s0 = L.n_blocks, s1 = L.n_blocks + L.n_scalar;
    int64_t lo = u0 > s0 ? u0 : s0, hi = u0 + 32 < s1 ? u0 + 32 : s1;
    if (hi < lo) hi = lo;
    a = (int)(lo - u0);
    b = (int)(hi - u0);
}

// coefficient of CSC entry t (raw = its row word)
__device__ __forceinline__ float entry_val(const DevLP& L, int64_t t, uint32_t raw) {
    return L.val ? L.val[t] : ((raw & kSignBit) ? -1.0f : 1.0f);
}

// async column dot / scatter with the loads of eight entries in flight together
__device__ __forceinline__ float col_dot_async(const DevLP& L, int64_t j) {
    const int64_t cb = L.colptr[j], ce = L.colptr[j + 1];
    float D = 0.0f;
    for (int64_t q0 = cb; q0 < ce; q0 += 8) {
        uint32_t raw[8];
        float rv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) raw[u] = q0 + u < ce ? (uint32_t)L.rowidx[q0 + u] : 0u;
#pragma unroll
        for (int u = 0; u < 8; u++) rv[u] = q0 + u < ce ? ld_cg(L.r + (raw[u] & kRowMask)) : 0.0f;
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (q0 + u < ce) D += L.val ? L.val[q0 + u] * rv[u] : ((raw[u] & kSignBit) ? -rv[u] : rv[u]);
    }
    return D;
}
__device__ __forceinline__ void col_scatter_async(const DevLP& L, int64_t j, float d) {
    if (d == 0.0f) return;
    const int64_t cb = L.colptr[j], ce = L.colptr[j + 1];
    for (int64_t q0 = cb; q0 < ce; q0 += 8) {
        uint32_t raw[8];
#pragma unroll
        for (int u = 0; u < 8; u++) raw[u] = q0 + u < ce ? (uint32_t)L.rowidx[q0 + u] : 0u;
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (q0 + u < ce) {
                const float ad = L.val ? __fmul_rn(L.val[q0 + u], d) : ((raw[u] & kSignBit) ? -d : d);
                red_add(L.r + (raw[u] & kRowMask), ad);
            }
    }
}

// new values of a k-block from the current (possibly stale) residual
template <int KC>
__device__ __forceinline__ void block_values(const DevLP& L, const StepParams& P, int64_t u, float* x) {
    const int k = L.k;
    const int64_t f = u * k;
    float y[KC];
    double mx = 0.0;
    if (P.rule == THETIS_STEP_LJ)
        for (int l = 0; l < k; l++) {
            double q = col_norm2(L, f + l);
            mx = q > mx ? q : mx;
        }
    const float invL = unit_invL(P, mx);
#pragma unroll
    for (int l = 0; l < KC; l++)
        if (l < k) {
            int64_t j = f + l;
            float D = col_dot_async(L, j);
            float g = grad_fast(c_int(L, j), ua_of(L, j), D, L.z[j], zbar_of(L, j), P.beta, P.inv_beta);
            y[l] = __fsub_rn(L.z[j], __fmul_rn(g, invL));
        }
    project_simplex<KC>(y, k, x);
}

// per-warp shared state
struct WarpSmem {
    int64_t cp[33];   // column starts of the tile's scalar range (cp[ncols] = end)
    float acc[32];    // per-column partial dots
    float d[32];      // per-column steps
};

struct TileCols {
    int64_t j0, u0;
    int a, ncols;
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// largest column index c with cp[c] <= t (uniform over the warp)
__device__ __forceinline__ int col_of(const WarpSmem& sm, int ncols, int64_t t) {
    int lo = 0, hi = ncols - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (sm.cp[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}
// partial dots of the tile's columns over the nonzero range [c0, c1), added into
// sm.acc.  Sub-chunks of 32 lying inside one column accumulate in registers;
// mixed sub-chunks locate each lane's column and add with shared atomics.
// (rows below m_defer are left out: the row pass accumulated them into lv)
__device__ __forceinline__ void gather_range(const DevLP& L, WarpSmem& sm, int ncols, int64_t c0, int64_t c1,
                                             int lane, int64_t m_defer) {
    constexpr int U = 4; // sub-chunks in flight: their loads are issued before any use
    int c = col_of(sm, ncols, c0);
    int64_t nb = sm.cp[c + 1];
    float acc = 0.0f;
    for (int64_t b0 = c0; b0 < c1; b0 += 32 * U) {
        uint32_t raw[U];
        float v[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int64_t t = b0 + 32 * q + lane;
            raw[q] = t < c1 ? (uint32_t)L.rowidx[t] : 0u;  // re-read by the scatter: keep cached
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int64_t t = b0 + 32 * q + lane;
            v[q] = 0.0f;
            if (t < c1 && (int64_t)(raw[q] & kRowMask) >= m_defer) {
                const float rv = ld_cg(L.r + (raw[q] & kRowMask));
                v[q] = L.val ? L.val[t] * rv : ((raw[q] & kSignBit) ? -rv : rv);
            }
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int64_t base = b0 + 32 * q;
            if (base >= c1) break;
            if (nb <= base) {
                acc = warp_sum(acc);
                if (lane == 0 && acc != 0.0f) atomicAdd(&sm.acc[c], acc);
                acc = 0.0f;
                do { c++; nb = sm.cp[c + 1]; } while (nb <= base);
            }
            const int64_t t = base + lane;
            if (base + 32 <= nb || c1 <= nb) {
                acc += v[q];
            } else if (t < c1 && v[q] != 0.0f) {
                int col = c;
                while (sm.cp[col + 1] <= t) col++;
                atomicAdd(&sm.acc[col], v[q]);
            }
        }
    }
    acc = warp_sum(acc);
    if (lane == 0 && acc != 0.0f) atomicAdd(&sm.acc[c], acc);
    __syncwarp();
}
// r += a_j d_j over the nonzero range [c0, c1), d_j = sm.d[column]; rows below
// m_defer are left out (the next row pass applies d_j there)
__device__ __forceinline__ void scatter_range(const DevLP& L, WarpSmem& sm, int ncols, int64_t c0, int64_t c1,
                                              int lane, int64_t m_defer) {
    constexpr int U = 4;
    int c = col_of(sm, ncols, c0);
    int64_t nb = sm.cp[c + 1];
    float dc = sm.d[c];
    for (int64_t b0 = c0; b0 < c1; b0 += 32 * U) {
        uint32_t raw[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int64_t t = b0 + 32 * q + lane;
            raw[q] = t < c1 ? (uint32_t)ld_cs_i32(L.rowidx + t) : 0u;
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int64_t base = b0 + 32 * q;
            if (base >= c1) break;
            if (nb <= base) {
                do { c++; nb = sm.cp[c + 1]; } while (nb <= base);
                dc = sm.d[c];
            }
            const int64_t t = base + lane;
            float d = dc;
            const bool live = t < c1 && (int64_t)(raw[q] & kRowMask) >= m_defer;
            if (!(base + 32 <= nb || c1 <= nb) && live) {
                int col = c;
                while (sm.cp[col + 1] <= t) col++;
                d = sm.d[col];
            }
            if (live && d != 0.0f) {
                const float a = L.val ? L.val[t] : ((raw[q] & kSignBit) ? -1.0f : 1.0f);
                red_add(L.r + (raw[q] & kRowMask), L.val ? a * d : (a < 0.0f ? -d : d));
            }
        }
    }
}

// the coordinate step of lane's column from D = sm.acc[lane]; returns the change
// (z, c: the column's value and cost, loaded ahead by prefetch_tile)
__device__ __forceinline__ float scalar_step(const DevLP& L, const StepParams& P, const TileCols& tc, float D,
                                             int lane, float z, float c) {
    if (lane >= tc.ncols || (L.unit_fixed && L.unit_fixed[tc.u0 + tc.a + lane])) return 0.0f;
    const int64_t j = tc.j0 + lane;
    float g = grad_fast(c, ua_of(L, j), D, z, zbar_of(L, j), P.beta, P.inv_beta);
    float invL = unit_invL(P, col_norm2(L, j));
    float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), col_lo(L, j), col_hi(L, j));
    L.z[j] = zn;
    return __fsub_rn(zn, z);
}

}  // namespace
}  // namespace thetis
