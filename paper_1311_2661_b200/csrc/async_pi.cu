// THETIS_MODE_ASYNC: Alg. 1 on f_beta (Eq. 5), run Hogwild-style
// (many updaters share x, "each thread runs Alg. 1") in the order of the
// oracle's sequential reference trajectory (R-6):
//
//   units  = k-blocks, scalar structural columns, slacks (ids in that order);
//   tiles  = 32 consecutive unit ids, n_tiles = ceil(U / 32);
//   epoch e visits the tiles in the order pi_e (4-round Feistel keyed by
//            (seed, e), thetis_internal.cuh), every unit once.
//
// The GPU hands out the permuted positions in order and runs a small window of them
// concurrently.  Inside a tile, k-blocks step one at a time (neighbouring MWC vertices
// share rows), then the scalar columns synchronously (all read r, then all write it with
// red.global.add.f32, so no update is lost), then the slacks likewise; tiles in flight
// read r stale by at most the window.  With one worker (THETIS_MODE_ASYNC_SERIAL) this is exactly the
// replay of oracle mode 4.
//
// Big tiles (scalar columns holding more than kJobMin nonzeros: power-law hubs) are
// cut into chunks of kJobChunk nonzeros that many warps process: per epoch the
// sequence of positions is expanded into *slots* -- a big tile at position p becomes
// its gather chunks (partial column dots added into the tile's accumulators; the last
// one takes the tile's steps), and its scatter chunks are inserted G positions later
// (G = a quarter of the window; a scatter drawn before its tile's steps are known is
// kept by its warp and run as soon as they are).
// A hub is thus gathered at its position within microseconds by many warps and its
// step reaches r G positions later: a bounded delay, the async model of P:463-476.
//
// Edge-incidence LPs (VC / MIS: every row is x_u + x_v + sigma_i s_i = 1) run the same order in
// the *column-sum form* (kGD, R-23): instead of the m residuals the kernel keeps
// per-vertex state -- x by degree rank and the slack sums S_u = sum_i sigma_i s_i (fp64,
// red.global.add.f64) -- and forms D_u = a_u^T r = deg_u (x_u - 1) + sum_w x_w + S_u at u's
// turn.  A vertex tile gathers its neighbours' x (one random read per nonzero, no scatter: a
// step is visible through x); a slack tile forms r_i = x_u + x_v + sigma s_i - 1 from x (one
// coalesced read of its 32 rows' endpoint slots, two L2 reads of x) and adds its step to S_u
// and S_v.  r itself is not touched during the epochs and is recomputed from z on return
// (r = A z - b, the A2 kernel).  Why: Alg. 1's order makes every nonzero a random access; on r
// (4 B x 1.05e9 rows, uniformly accessed) nearly all of them miss the 126 MB L2, on x (n values,
// accessed in proportion to degree) the hot set of a power-law graph is L2-resident.
// THETIS_GD_PULL=0 builds the earlier push form (D_u maintained, every step pushed into the
// neighbours' D with one RED per nonzero: bound by the L2's atomic rate).
//
// Work distribution: slot batches of kPiBatch; batch b belongs to CTA b mod gridDim,
// whose warps draw that CTA's batches in order from a shared-memory counter, so all
// CTAs sweep the slots together without a global atomic per tile, and the slots in
// flight are ~ (warps in the grid) x kPiBatch consecutive ones.
#include <cub/cub.cuh>

#include "scd_device.cuh"

namespace thetis {
namespace {

constexpr int kPiWarps = 8;           // warps per CTA
constexpr int kPiBatch = 4;           // consecutive slots a warp draws at once
constexpr int64_t kJobChunk = 2048;   // nonzeros per big-tile chunk
constexpr int64_t kJobMin = 4096;     // a tile whose scalar range holds more is big
constexpr int kVShift = 7;            // slot index: one entry per 128 slots

// one big tile (static per solve) and its per-epoch state
struct PiJob {
    int64_t tile, cb, ce;             // tile, its scalar CSC range [cb, ce)
    int32_t n_chunks;
    int32_t gdone;                    // gather chunks finished this epoch
    uint32_t ready;                   // = stamp once d[] holds this epoch's steps
    int32_t pad[3];
    float acc[32];                    // column dots D_j (device-scope atomics)
    float d[32];                      // steps of the tile's columns
};

// scatter chunks whose tile's steps were not ready when drawn: kept per warp and run
// as soon as they are (a warp never waits while it has other slots to run)
constexpr int kDefer = 8;
struct Deferred {
    int32_t b[kDefer], c[kDefer];
    int n;
};

struct PiCtx {
    PermKeys K;                       // pi_e on [0, n_tiles)
    int64_t n_tiles;
    int64_t n_struct;                 // structural units n_blocks + n_scalar
    PiJob* jobs;
    int64_t n_ev;                     // events (2 per big tile), sorted by (position, kind)
    const int64_t* ev_pos;            // position the event sits at
    const int64_t* ev_vstart;         // its first slot
    const int32_t* ev_val;            // 2 b + kind (kind 1 = gathers of big tile b, 0 = scatters)
    const int32_t* vindex;            // per 2^kVShift slots: last event starting at or before, or -1
    const int64_t* n_slots;           // slots this epoch (device)
    uint32_t stamp;                   // epoch stamp of the call (1, 2, ...)
    // kGD (column-sum form): vertices addressed by degree rank
    const int32_t* rank;              // rank of vertex u
    const int32_t* nbr;               // rank of the neighbour of CSC entry t
    const int2* erank;                // ranks of the endpoints of row i
    float* xr;                        // x by rank (kept current)
    double* Dg;                       // by rank, fp64, kept current: the slack sums S_u (pull form) or D_u (push form)
    int64_t hot;                      // slots below this are kept in L2 (evict_last)
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {  // polls: no L1 invalidation
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_release(int32_t* p, int v) {
    int old;
    asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ double ld_cg_f64(const double* p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
// L2 eviction policies of the column-sum form: the slots below `hot` (the largest-degree
// vertices) are kept with evict_last, everything colder passes through with evict_first, so
// that the ~10^10 bytes streamed per epoch do not turn the hot set over
struct L2Pol {
    uint64_t last, first;
    int64_t hot;
};
__device__ __forceinline__ L2Pol make_l2pol(int64_t hot) {
    L2Pol p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p.last));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p.first));
    p.hot = hot;
    return p;
}
// THETIS_GD_EXP (measurement builds only, results wrong by design): 1 drops the REDs into D,
// 2 drops the slack tiles' reads of x, 4 / 8 drop only the REDs into cold / hot slots
#ifndef THETIS_GD_EXP
#define THETIS_GD_EXP 0
#endif
__device__ __forceinline__ float ld_x_slot(const float* xr, int slot, const L2Pol& pol) {
    if (THETIS_GD_EXP & 2) return 0.25f;
    float v;
    asm volatile("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(v) : "l"(xr + slot), "l"(slot < pol.hot ? pol.last : pol.first));
    return v;
}
// D_u lives in HBM / L2 as fp64 (THETIS_GD_DTYPE 0).  Measurement-only alternatives: 1 = fp32
// (loses small steps against hub sums of ~10^6), 2 = 64-bit fixed point, 2^-32 resolution
#ifndef THETIS_GD_DTYPE
#define THETIS_GD_DTYPE 0
#endif
// THETIS_GD_PULL 1 (default): a vertex forms D_u = deg_u (x_u - 1) + sum_w x_w + S_u at its turn
// from its neighbours' x (random *reads*, one per nonzero) and the maintained slack sum
// S_u = sum_i sigma_i s_i (REDs only when a slack moves).  0: D_u itself is maintained, every
// step pushed into the neighbours' D (one RED per nonzero; the L2's RED rate is 220 G/s)
#ifndef THETIS_GD_PULL
#define THETIS_GD_PULL 1
#endif
__device__ __forceinline__ void red_D_slot(double* Dg, int slot, double v, const L2Pol& pol) {
    if (THETIS_GD_EXP & 1) return;
    if ((THETIS_GD_EXP & 4) && slot >= pol.hot) return;
    if ((THETIS_GD_EXP & 8) && slot < pol.hot) return;
    const uint64_t hint = slot < pol.hot ? pol.last : pol.first;
#if THETIS_GD_DTYPE == 1
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"((float*)Dg + slot), "f"((float)v), "l"(hint) : "memory");
#elif THETIS_GD_DTYPE == 2
    asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;"
                 ::"l"((unsigned long long*)Dg + slot), "l"((unsigned long long)__double2ll_rn(v * 4294967296.0)), "l"(hint) : "memory");
#else
    asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(Dg + slot), "d"(v), "l"(hint) : "memory");
#endif
}
__device__ __forceinline__ float ld_D_slot(const double* Dg, int slot) {
#if THETIS_GD_DTYPE == 1
    return ld_cg((const float*)Dg + slot);
#elif THETIS_GD_DTYPE == 2
    long long q;
    asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(q) : "l"((const long long*)Dg + slot));
    return (float)((double)q * (1.0 / 4294967296.0));
#else
    return (float)ld_cg_f64(Dg + slot);
#endif
}
__device__ __forceinline__ float ld_cs_f32(const float* p) {
    float v;
    asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_cs_f32(float* p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ int2 ld_cs_int2(const int2* p) {  // streamed once per epoch
    int2 v;
    asm volatile("ld.global.cs.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// the tile's scalar columns: lanes [a, b), first column j0
__device__ __forceinline__ TileCols tile_cols(const DevLP& L, int64_t tile) {
    TileCols tc;
    tc.u0 = tile * 32;
    int b;
    scalar_lanes(L, tc.u0, tc.a, b);
    tc.ncols = b - tc.a;
    tc.j0 = L.n_blocks * L.k + (tc.u0 + tc.a - L.n_blocks);
    return tc;
}
// column starts of the tile's scalar range into sm.cp (cp[ncols] = end)
__device__ __forceinline__ void load_cp(const DevLP& L, const TileCols& tc, WarpSmem& sm, int lane) {
    if (lane < tc.ncols) sm.cp[lane] = L.colptr[tc.j0 + lane];
    if (lane == 0) sm.cp[tc.ncols] = L.colptr[tc.j0 + tc.ncols];
    __syncwarp();
}

// slack lanes of a tile: new value from r_i (gather side); returns the change of r_i
__device__ __forceinline__ float slack_lane_gather(const DevLP& L, const StepParams& P, int64_t q, int64_t& row) {
    row = slack_row_of(L, q);
    const int64_t j = L.n_s + q;
    const float sig = row_sigma(L, row);
    const float rv = ld_cg(L.r + row);
    const float z = L.z[j];
    const float zn = slack_new<true>(L, P, row, j, sig, rv, z);
    L.z[j] = zn;
    const float d = __fsub_rn(zn, z);
    return sig < 0.0f ? -d : d;
}

// column-sum form (VC / MIS): the slack of row q = (u, v) from x; its step enters the sums of u and v
__device__ __forceinline__ void slack_lane_gd(const DevLP& L, const StepParams& P, const PiCtx& C, const L2Pol& pol,
                                              int64_t q) {
    const int64_t j = L.n_s + q;
    const float sig = row_sigma(L, q);
    const int2 e = ld_cs_int2(C.erank + q);
    const float xu = ld_x_slot(C.xr, e.x, pol), xv = ld_x_slot(C.xr, e.y, pol);
    const float z = ld_cs_f32(L.z + j);
    // r_i = -1 + x_u + x_v + sigma s_i, the operation order of A2 (k_recompute_r)
    float rv = __fadd_rn(__fadd_rn(-1.0f, xu), xv);
    rv = __fadd_rn(rv, sig < 0.0f ? -z : z);
    const float zn = slack_new<true>(L, P, q, j, sig, rv, z);
    if (zn != z) {
        st_cs_f32(L.z + j, zn);
        const float d = __fsub_rn(zn, z);
        const double dr = (double)(sig < 0.0f ? -d : d);
        red_D_slot(C.Dg, e.x, dr, pol);
        red_D_slot(C.Dg, e.y, dr, pol);
    }
}
// X_col += x_w over the neighbours w of the tile's columns, nonzero range [c0, c1), into sm.acc
// (sub-chunks of 32 inside one column accumulate in registers, mixed ones add per lane)
__device__ __forceinline__ void gather_x_range(const PiCtx& C, const L2Pol& pol, WarpSmem& sm, int ncols, int64_t c0,
                                               int64_t c1, int lane) {
    constexpr int U = 4;
    int c = col_of(sm, ncols, c0);
    int64_t nb = sm.cp[c + 1];
    float acc = 0.0f;
    for (int64_t b0 = c0; b0 < c1; b0 += 32 * U) {
        int32_t w[U];
        float v[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int64_t t = b0 + 32 * q + lane;
            w[q] = t < c1 ? ld_cs_i32(C.nbr + t) : 0;
        }
#pragma unroll
        for (int q = 0; q < U; q++) v[q] = b0 + 32 * q + lane < c1 ? ld_x_slot(C.xr, w[q], pol) : 0.0f;
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
// D_u of the pull form from the column's degree, its x, the gathered neighbour sum and S_u
__device__ __forceinline__ float pull_D(int64_t deg, float z, float X, double S) {
    return (float)((double)deg * ((double)z - 1.0) + (double)X + S);
}
// D_v += d_col for the neighbours v of the tile's columns over the nonzero range [c0, c1)
__device__ __forceinline__ void push_range(const PiCtx& C, const L2Pol& pol, WarpSmem& sm, int ncols, int64_t c0,
                                           int64_t c1, int lane) {
    constexpr int U = 4;
    int c = col_of(sm, ncols, c0);
    int64_t nb = sm.cp[c + 1];
    float dc = sm.d[c];
    for (int64_t b0 = c0; b0 < c1; b0 += 32 * U) {
        int32_t v[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int64_t t = b0 + 32 * q + lane;
            v[q] = t < c1 ? ld_cs_i32(C.nbr + t) : 0;
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
            const bool live = t < c1;
            if (!(base + 32 <= nb || c1 <= nb) && live) {
                int col = c;
                while (sm.cp[col + 1] <= t) col++;
                d = sm.d[col];
            }
            if (live && d != 0.0f) red_D_slot(C.Dg, v[q], (double)d, pol);
        }
    }
}

// ---- k-blocks (MWC vertex blocks, App. E): one block at a time in unit order, each by
// the whole warp (neighbouring vertices share rows, so a tile-synchronous step of
// coupled blocks would leave Alg. 1's sequential trajectory).  The block's k columns
// are one contiguous CSC range; lane q takes entries q, q + 32, ... of it.
template <int KC>
__device__ void block_step_warp(const DevLP& L, const StepParams& P, int64_t u, WarpSmem& sm, int lane) {
    const int k = L.k;
    const int64_t f = u * k;
    if (lane <= k) sm.cp[lane] = L.colptr[f + lane];
    float zl = 0.0f, cl = 0.0f, ul = 0.0f, zbl = 0.0f;
    double nrm = 0.0;
    if (lane < k) {
        zl = L.z[f + lane];
        cl = c_int(L, f + lane);
        ul = ua_of(L, f + lane);
        zbl = zbar_of(L, f + lane);
        nrm = col_norm2(L, f + lane);
        sm.acc[lane] = 0.0f;
    }
    __syncwarp();
    const int64_t cb = sm.cp[0], ce = sm.cp[k];
    // D_l = a_l^T r: lane q adds its entries into its column's slot
    for (int64_t t0 = cb; t0 < ce; t0 += 64) {
        uint32_t raw[2];
        float v[2];
#pragma unroll
        for (int e = 0; e < 2; e++) {
            const int64_t t = t0 + lane + 32 * e;
            raw[e] = t < ce ? (uint32_t)L.rowidx[t] : 0u;
        }
#pragma unroll
        for (int e = 0; e < 2; e++) {
            const int64_t t = t0 + lane + 32 * e;
            v[e] = 0.0f;
            if (t < ce) {
                const float rv = ld_cg(L.r + (raw[e] & kRowMask));
                v[e] = L.val ? L.val[t] * rv : ((raw[e] & kSignBit) ? -rv : rv);
            }
        }
#pragma unroll
        for (int e = 0; e < 2; e++) {
            const int64_t t = t0 + lane + 32 * e;
            if (t < ce && v[e] != 0.0f) atomicAdd(&sm.acc[col_of(sm, k, t)], v[e]);
        }
    }
    __syncwarp();
    // step: y_l = z_l - g_l / L (L_max, or the block's largest L_j), projection on the simplex
    double mx = nrm;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double q = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = q > mx ? q : mx;
    }
    const float invL = unit_invL(P, mx);
    const float Dl = lane < k ? sm.acc[lane] : 0.0f;
    const float yl = __fsub_rn(zl, __fmul_rn(grad_fast(cl, ul, Dl, zl, zbl, P.beta, P.inv_beta), invL));
    float y[KC], x[KC];
#pragma unroll
    for (int l = 0; l < KC; l++) y[l] = __shfl_sync(0xffffffffu, yl, l & 31);
    project_simplex<KC>(y, k, x);
    float xl = 0.0f;
#pragma unroll
    for (int l = 0; l < KC; l++)
        if (l == lane) xl = x[l];
    if (lane < k) {
        sm.d[lane] = __fsub_rn(xl, zl);
        L.z[f + lane] = xl;
    }
    __syncwarp();
    // scatter: r_i += a_ij d_col
    for (int64_t t = cb + lane; t < ce; t += 32) {
        const float d = sm.d[col_of(sm, k, t)];
        const uint32_t rw = (uint32_t)L.rowidx[t];
        if (d != 0.0f) red_add(L.r + (rw & kRowMask), L.val ? __fmul_rn(L.val[t], d) : ((rw & kSignBit) ? -d : d));
    }
    __syncwarp();  // the next block's loads come after these (same-warp ordering)
}

// ---- one tile.  scalars = false: the scalar columns are a big tile's (done by chunks)
template <bool kBlocks, int KC, bool kGD>
__device__ void process_tile_pi(const DevLP& L, const StepParams& P, const PiCtx& C, const L2Pol& pol, int64_t tile,
                                WarpSmem& sm, int lane, bool scalars) {
    const int64_t u = tile * 32 + lane;
    if (tile * 32 >= C.n_struct) {  // slack tile
        if (kGD) {
            if (u < L.U) slack_lane_gd(L, P, C, pol, u - C.n_struct);
            return;
        }
        float dr = 0.0f;
        int64_t row = 0;
        if (u < L.U) dr = slack_lane_gather(L, P, u - C.n_struct, row);
        if (dr != 0.0f) red_add(L.r + row, dr);
        return;
    }
    // k-blocks of the tile: one at a time, in unit order (Alg. 1's order inside the tile)
    if (kBlocks && tile * 32 < L.n_blocks) {
        const int nb = (int)(L.n_blocks - tile * 32 < 32 ? L.n_blocks - tile * 32 : 32);
        unsigned live = __ballot_sync(0xffffffffu, lane < nb && !(L.unit_fixed && L.unit_fixed[u]));
        // the blocks step one after the other, each a chain column starts -> row words -> r -> step:
        // bring the tile's static data (one contiguous CSC range, its column starts, values and
        // costs) into L1 once, so that only the read of r is a long round trip per block
        {
            const int64_t c0 = tile * 32 * L.k, c1 = c0 + (int64_t)nb * L.k;
            const int64_t rb = L.colptr[c0], re = L.colptr[c1];
            for (int64_t q = c0 + 16 * lane; q <= c1; q += 16 * 32) prefetch_l1(L.colptr + q);
            for (int64_t q = c0 + 32 * lane; q < c1; q += 32 * 32) {
                prefetch_l1(L.z + q);
                prefetch_l1(L.c + q);
            }
            for (int64_t t = rb + 32 * lane; t < re; t += 32 * 32) prefetch_l1(L.rowidx + t);
        }
        while (live) {
            const int i = __ffs(live) - 1;
            live &= live - 1;
            block_step_warp<KC>(L, P, tile * 32 + i, sm, lane);
        }
    }
    // then the tile's scalar columns synchronously (all read r before any write), then its
    // slacks (a tile mixing both is the one at the structural / slack boundary)
    const TileCols tc = tile_cols(L, tile);
    bool lane_path = false;
    int64_t beg = 0, end = 0, cb = 0, ce = 0;
    unsigned moved = 0;
    if (tc.ncols > 0 && scalars) {
        load_cp(L, tc, sm, lane);
        beg = sm.cp[0];
        end = sm.cp[tc.ncols];
        const int cl = lane - tc.a;  // this lane's scalar column, if any
        if (cl >= 0 && cl < tc.ncols) {
            cb = sm.cp[cl];
            ce = sm.cp[cl + 1];
        }
        lane_path = __reduce_max_sync(0xffffffffu, (unsigned)(ce - cb)) <= 48u;
        float z = 0.0f, cj = 0.0f;
        if (cl >= 0 && cl < tc.ncols) {
            z = L.z[tc.j0 + cl];
            cj = c_int(L, tc.j0 + cl);
        }
        // scalar_step indexes lanes 0..ncols-1 = columns: shuffle the column's data there
        z = __shfl_sync(0xffffffffu, z, (lane + tc.a) & 31);
        cj = __shfl_sync(0xffffffffu, cj, (lane + tc.a) & 31);
        float D = 0.0f;
        int rk = 0;
        if (kGD && THETIS_GD_PULL) {  // pull form: the neighbours' x, then D from it (lane = column index)
            float X = 0.0f;
            if (lane_path) {
                for (int64_t q0 = cb; q0 < ce; q0 += 8) {
                    int32_t w[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) w[q] = q0 + q < ce ? C.nbr[q0 + q] : 0;
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        if (q0 + q < ce) X += ld_x_slot(C.xr, w[q], pol);
                }
                X = __shfl_sync(0xffffffffu, X, (lane + tc.a) & 31);
            } else {
                sm.acc[lane] = 0.0f;
                __syncwarp();
                gather_x_range(C, pol, sm, tc.ncols, beg, end, lane);
                X = sm.acc[lane];
            }
            if (lane < tc.ncols) {
                rk = C.rank[tc.j0 + lane];
                D = pull_D(sm.cp[lane + 1] - sm.cp[lane], z, X, ld_cg_f64(C.Dg + rk));
            }
        } else if (kGD) {  // push form: D_j is kept current
            if (lane < tc.ncols) {
                rk = C.rank[tc.j0 + lane];
                D = ld_D_slot(C.Dg, rk);
            }
        } else if (lane_path) {  // one lane per column, eight loads in flight
            for (int64_t q0 = cb; q0 < ce; q0 += 8) {
                uint32_t raw[8];
                float rv[8];
#pragma unroll
                for (int q = 0; q < 8; q++) raw[q] = q0 + q < ce ? (uint32_t)L.rowidx[q0 + q] : 0u;
#pragma unroll
                for (int q = 0; q < 8; q++) rv[q] = q0 + q < ce ? ld_cg(L.r + (raw[q] & kRowMask)) : 0.0f;
#pragma unroll
                for (int q = 0; q < 8; q++)
                    if (q0 + q < ce) D += L.val ? L.val[q0 + q] * rv[q] : ((raw[q] & kSignBit) ? -rv[q] : rv[q]);
            }
            D = __shfl_sync(0xffffffffu, D, (lane + tc.a) & 31);
        } else {  // the warp walks the tile's CSC range coalesced
            sm.acc[lane] = 0.0f;
            __syncwarp();
            gather_range(L, sm, tc.ncols, beg, end, lane, 0);
            D = sm.acc[lane];
        }
        const float d = scalar_step(L, P, tc, D, lane, z, cj);  // lane = column index
        sm.d[lane] = d;
        moved = __ballot_sync(0xffffffffu, d != 0.0f);
        // x by rank, and the column's own sum: D_j += ||a_j||^2 d_j (||a_j||^2 = its nonzero count)
        if (kGD && d != 0.0f) {
            C.xr[rk] = L.z[tc.j0 + lane];
            if (!THETIS_GD_PULL) red_D_slot(C.Dg, rk, (double)(sm.cp[lane + 1] - sm.cp[lane]) * (double)d, pol);
        }
    }
    __syncwarp();
    // scatters (none in the pull form: a step is visible through x)
    if (moved && !(kGD && THETIS_GD_PULL)) {
        if (kGD) {
            if (lane_path) {
                const int cl = lane - tc.a;
                const float d = cl >= 0 && cl < 32 ? sm.d[cl] : 0.0f;
                if (d != 0.0f)
                    for (int64_t q0 = cb; q0 < ce; q0 += 8) {
                        int32_t v[8];
#pragma unroll
                        for (int q = 0; q < 8; q++) v[q] = q0 + q < ce ? C.nbr[q0 + q] : 0;
#pragma unroll
                        for (int q = 0; q < 8; q++)
                            if (q0 + q < ce) red_D_slot(C.Dg, v[q], (double)d, pol);
                    }
            } else {
                push_range(C, pol, sm, tc.ncols, beg, end, lane);
            }
        } else if (lane_path) {
            const int cl = lane - tc.a;
            const float d = cl >= 0 && cl < 32 ? sm.d[cl] : 0.0f;
            if (d != 0.0f)
                for (int64_t q = cb; q < ce; q++) {
                    const uint32_t raw = (uint32_t)L.rowidx[q];
                    const float a = entry_val(L, q, raw);
                    red_add(L.r + (raw & kRowMask), L.val ? a * d : (a < 0.0f ? -d : d));
                }
        } else {
            scatter_range(L, sm, tc.ncols, beg, end, lane, 0);
        }
    }
    __syncwarp();  // the slacks' loads come after the scalars' writes (same-warp ordering)
    if (u >= C.n_struct && u < L.U) {
        if (kGD) {
            slack_lane_gd(L, P, C, pol, u - C.n_struct);
        } else {
            int64_t srow = 0;
            const float dr = slack_lane_gather(L, P, u - C.n_struct, srow);
            if (dr != 0.0f) red_add(L.r + srow, dr);
        }
    }
    __syncwarp();
}

// ---- big tiles
// gather chunk c of big tile b: partial dots of its columns over the chunk; the last
// one takes the tile's steps (tile-synchronous) and marks them ready
template <bool kBlocks, int KC, bool kGD>
__device__ void job_gather(const DevLP& L, const StepParams& P, const PiCtx& C, const L2Pol& pol, int32_t b, int c,
                           WarpSmem& sm, int lane) {
    PiJob& J = C.jobs[b];
    if (c == 0) process_tile_pi<kBlocks, KC, kGD>(L, P, C, pol, J.tile, sm, lane, false);  // its other units
    const TileCols tc = tile_cols(L, J.tile);
    if (kGD && THETIS_GD_PULL) {  // pull form: partial neighbour sums of x; the last chunk takes the steps
        load_cp(L, tc, sm, lane);
        sm.acc[lane] = 0.0f;
        __syncwarp();
        const int64_t c0 = J.cb + (int64_t)c * kJobChunk;
        const int64_t c1 = c0 + kJobChunk < J.ce ? c0 + kJobChunk : J.ce;
        gather_x_range(C, pol, sm, tc.ncols, c0, c1, lane);
        if (lane < tc.ncols && sm.acc[lane] != 0.0f) atomicAdd(&J.acc[lane], sm.acc[lane]);
        __syncwarp();
        int g = 0;
        if (lane == 0) g = atom_add_release(&J.gdone, 1);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g != J.n_chunks - 1) return;
        if (lane == 0) (void)ld_acquire_u32((const uint32_t*)&J.gdone);
        __syncwarp();
        const float X = ld_cg(&J.acc[lane]);
        float D = 0.0f, z = 0.0f, cj = 0.0f;
        int rk = 0;
        if (lane < tc.ncols) {
            rk = C.rank[tc.j0 + lane];
            z = L.z[tc.j0 + lane];
            cj = c_int(L, tc.j0 + lane);
            D = pull_D(sm.cp[lane + 1] - sm.cp[lane], z, X, ld_cg_f64(C.Dg + rk));
        }
        const float d = scalar_step(L, P, tc, D, lane, z, cj);
        if (d != 0.0f) C.xr[rk] = L.z[tc.j0 + lane];
        return;
    }
    if (kGD) {  // push form: nothing to gather; the first chunk's slot takes the tile's steps
        if (c != 0) return;
        load_cp(L, tc, sm, lane);
        float D = 0.0f, z = 0.0f, cj = 0.0f;
        int rk = 0;
        if (lane < tc.ncols) {
            rk = C.rank[tc.j0 + lane];
            D = ld_D_slot(C.Dg, rk);
            z = L.z[tc.j0 + lane];
            cj = c_int(L, tc.j0 + lane);
        }
        const float d = scalar_step(L, P, tc, D, lane, z, cj);
        J.d[lane] = d;
        if (d != 0.0f) {
            C.xr[rk] = L.z[tc.j0 + lane];
            red_D_slot(C.Dg, rk, (double)(sm.cp[lane + 1] - sm.cp[lane]) * (double)d, pol);
        }
        __syncwarp();
        if (lane == 0) st_release_u32(&J.ready, C.stamp);
        return;
    }
    load_cp(L, tc, sm, lane);
    sm.acc[lane] = 0.0f;
    __syncwarp();
    const int64_t c0 = J.cb + (int64_t)c * kJobChunk;
    const int64_t c1 = c0 + kJobChunk < J.ce ? c0 + kJobChunk : J.ce;
    gather_range(L, sm, tc.ncols, c0, c1, lane, 0);
    if (lane < tc.ncols && sm.acc[lane] != 0.0f) atomicAdd(&J.acc[lane], sm.acc[lane]);
    __syncwarp();  // (the warp barrier orders every lane's partial before lane 0's release)
    int g = 0;
    if (lane == 0) g = atom_add_release(&J.gdone, 1);  // orders this chunk's partials before it
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g != J.n_chunks - 1) return;
    if (lane == 0) (void)ld_acquire_u32((const uint32_t*)&J.gdone);  // every partial is in
    __syncwarp();
    const float D = ld_cg(&J.acc[lane]);
    float z = 0.0f, cj = 0.0f;
    if (lane < tc.ncols) {
        z = L.z[tc.j0 + lane];
        cj = c_int(L, tc.j0 + lane);
    }
    J.d[lane] = scalar_step(L, P, tc, D, lane, z, cj);
    __syncwarp();
    if (lane == 0) st_release_u32(&J.ready, C.stamp);
}
// scatter chunk c of big tile b, whose steps are ready
template <bool kGD>
__device__ void job_scatter(const DevLP& L, const PiCtx& C, const L2Pol& pol, int32_t b, int c, WarpSmem& sm, int lane) {
    if (kGD && THETIS_GD_PULL) return;  // pull form: a big tile's steps are visible through x
    const PiJob& J = C.jobs[b];
    if (lane == 0) (void)ld_acquire_u32(&J.ready);  // the steps and z written before `ready`
    __syncwarp();
    const float d = ld_cg(&J.d[lane]);
    if (!__any_sync(0xffffffffu, d != 0.0f)) return;
    const TileCols tc = tile_cols(L, J.tile);
    load_cp(L, tc, sm, lane);
    sm.d[lane] = d;
    __syncwarp();
    const int64_t c0 = J.cb + (int64_t)c * kJobChunk;
    const int64_t c1 = c0 + kJobChunk < J.ce ? c0 + kJobChunk : J.ce;
    if (kGD) push_range(C, pol, sm, tc.ncols, c0, c1, lane);
    else scatter_range(L, sm, tc.ncols, c0, c1, lane, 0);
}
__device__ __forceinline__ bool job_ready(const PiCtx& C, int32_t b, int lane) {
    int ok = 0;
    if (lane == 0) ok = ld_relaxed_u32(&C.jobs[b].ready) == C.stamp;
    return __shfl_sync(0xffffffffu, ok, 0);
}
// run the deferred scatters that are ready (all of them, waiting, when `drain`)
template <bool kGD>
__device__ void run_deferred(const DevLP& L, const PiCtx& C, const L2Pol& pol, Deferred& df, WarpSmem& sm, int lane,
                             bool drain) {
    int i = 0;
    while (i < df.n) {
        if (job_ready(C, df.b[i], lane)) {
            job_scatter<kGD>(L, C, pol, df.b[i], df.c[i], sm, lane);
            __syncwarp();
            if (lane == 0) {
                df.b[i] = df.b[df.n - 1];
                df.c[i] = df.c[df.n - 1];
                df.n--;
            }
            __syncwarp();
        } else if (drain) {
            __nanosleep(256);
        } else {
            i++;
        }
    }
}

// slot v -> a plain position (returns the tile, kind = 2) or a chunk of an event
// (kind 1 = gather, 0 = scatter; b = big tile, c = chunk)
__device__ __forceinline__ int64_t resolve_slot(const PiCtx& C, int64_t v, int& kind, int32_t& b, int& c) {
    int64_t e = C.n_ev ? C.vindex[v >> kVShift] : -1;
    while (e + 1 < C.n_ev && C.ev_vstart[e + 1] <= v) e++;
    int64_t p = v;
    if (e >= 0) {
        const int32_t val = C.ev_val[e];
        const int k = val & 1;
        b = val >> 1;
        const int64_t vs = C.ev_vstart[e], n = C.jobs[b].n_chunks;
        if (v < vs + n) {
            kind = k;
            c = (int)(v - vs);
            return -1;
        }
        p = C.ev_pos[e] + k + (v - vs - n);
    }
    kind = 2;
    return (int64_t)tile_perm((uint64_t)p, C.K);
}

// resident CTAs per SM of the scalar variant (a register cap of 65536 / (minB * 256)); the
// block variant keeps its registers (k-block arrays)
#ifndef THETIS_PI_MINB
#define THETIS_PI_MINB 6
#endif
#ifndef THETIS_PI_MINB_GD
#define THETIS_PI_MINB_GD 6
#endif
template <bool kBlocks, int KC, bool kGD>
__global__ void __launch_bounds__(kPiWarps * 32, kBlocks ? 3 : kGD ? THETIS_PI_MINB_GD : THETIS_PI_MINB)
    k_async_pi(DevLP L, StepParams P, PiCtx C, int batch) {
    __shared__ WarpSmem wsm[kPiWarps];
    __shared__ Deferred wdf[kPiWarps];
    __shared__ unsigned s_next;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSmem& sm = wsm[w];
    Deferred& df = wdf[w];
    if (threadIdx.x == 0) s_next = 0;
    if (lane == 0) df.n = 0;
    __syncthreads();
    const int64_t V = *C.n_slots;
    const L2Pol pol = make_l2pol(C.hot);
    for (int it = 0;; it++) {
        if (df.n && (it & 3) == 0) run_deferred<kGD>(L, C, pol, df, sm, lane, false);
        unsigned k = 0;
        if (lane == 0) k = atomicAdd(&s_next, 1u);
        k = __shfl_sync(0xffffffffu, k, 0);
        const int64_t first = ((int64_t)k * gridDim.x + blockIdx.x) * batch;
        if (first >= V) break;
        int kind = 2, c = 0;
        int32_t b = 0;
        int64_t tile = -1;
        if (lane < batch && first + lane < V) tile = resolve_slot(C, first + lane, kind, b, c);
        else kind = 3;  // past the end
        for (int i = 0; i < batch; i++) {
            const int ki = __shfl_sync(0xffffffffu, kind, i);
            if (ki == 3) break;
            if (ki == 2) {
                process_tile_pi<kBlocks, KC, kGD>(L, P, C, pol, __shfl_sync(0xffffffffu, tile, i), sm, lane, true);
            } else {
                const int32_t bi = __shfl_sync(0xffffffffu, b, i);
                const int ci = __shfl_sync(0xffffffffu, c, i);
                if (ki == 1) {
                    job_gather<kBlocks, KC, kGD>(L, P, C, pol, bi, ci, sm, lane);
                } else if ((kGD && THETIS_GD_PULL) || job_ready(C, bi, lane)) {
                    job_scatter<kGD>(L, C, pol, bi, ci, sm, lane);
                } else {  // not ready: keep it (wait only when the list is full)
                    if (df.n == kDefer) run_deferred<kGD>(L, C, pol, df, sm, lane, true);
                    __syncwarp();
                    if (lane == 0) {
                        df.b[df.n] = bi;
                        df.c[df.n] = ci;
                        df.n++;
                    }
                    __syncwarp();
                }
            }
        }
    }
    run_deferred<kGD>(L, C, pol, df, sm, lane, true);
}

// ---- column-sum form: per-LP ranks and neighbour lists, per-call column sums
// sort key of vertex u: larger degree first (ties: smaller id, the sort is stable)
__global__ void k_rank_keys(DevLP L, uint32_t* __restrict__ key, int32_t* __restrict__ id) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < L.n_s; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t deg = L.colptr[u + 1] - L.colptr[u];
        key[u] = 0xFFFFFFFFu - (uint32_t)(deg < 0xFFFFFFFFLL ? deg : 0xFFFFFFFFLL);
        id[u] = (int32_t)u;
    }
}
// slot of the vertex at degree rank p.  The hot prefix [0, hot) is transposed in blocks of 32
// (slot = (p mod hot/32) * 32 + p / (hot/32)): consecutive ranks lie 32 slots (256 B of D) apart, so
// the REDs into the very largest hubs spread over the L2 slices instead of queueing on one
// (measured on R-MAT 26: 46.8 -> 26.5 ms per epoch).  The colder vertices keep their rank as
// slot (id order among them measured the same).
__global__ void k_rank_of(int64_t n, int64_t hot, const int32_t* __restrict__ order, int32_t* __restrict__ rank) {
    const int64_t hb = hot / 32;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        rank[order[p]] = (int32_t)(p < hot ? (p % hb) * 32 + p / hb : p);
}
// nbr[t] = rank of the other endpoint of the row of CSC entry t (column j = vertex j); a warp
// per chunk of kNbrChunk entries, so that hub columns spread over many warps
constexpr int64_t kNbrChunk = 2048;
__global__ void k_fill_nbr(DevLP L, const int32_t* __restrict__ rank, int32_t* __restrict__ nbr) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t n_chunks = (L.nnz_s + kNbrChunk - 1) / kNbrChunk;
    for (int64_t c = w0; c < n_chunks; c += nw) {
        const int64_t c0 = c * kNbrChunk, c1 = c0 + kNbrChunk < L.nnz_s ? c0 + kNbrChunk : L.nnz_s;
        int64_t lo = 0, hi = L.n_s - 1;  // the column holding entry c0: largest j with colptr[j] <= c0
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (L.colptr[mid] <= c0) lo = mid; else hi = mid - 1;
        }
        int64_t j = lo, nb = L.colptr[j + 1];
        for (int64_t t = c0 + lane; t < c1; t += 32) {
            while (nb <= t) nb = L.colptr[++j + 1];
            const int2 e = L.edges[(uint32_t)L.rowidx[t] & kRowMask];
            nbr[t] = rank[e.x == (int32_t)j ? e.y : e.x];
        }
    }
}
__global__ void k_fill_erank(DevLP L, const int32_t* __restrict__ rank, int2* __restrict__ erank) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.m; i += (int64_t)gridDim.x * blockDim.x) {
        const int2 e = L.edges[i];
        erank[i] = make_int2(rank[e.x], rank[e.y]);
    }
}
// per call: x by rank, and the maintained sums from the rows (both endpoints of each)
__global__ void k_init_xr(DevLP L, const int32_t* __restrict__ rank, float* __restrict__ xr) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < L.n_s; u += (int64_t)gridDim.x * blockDim.x)
        xr[rank[u]] = L.z[u];
}
__global__ void k_init_colsum(DevLP L, const int2* __restrict__ erank, double* __restrict__ Dg, int64_t hot) {
    const L2Pol pol = make_l2pol(hot);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.m; i += (int64_t)gridDim.x * blockDim.x) {
        const int2 e = ld_cs_int2(erank + i);
        // push form: D = A^T r (r_i into both endpoints); pull form: S = sum of sigma_i s_i
        double rv;
        if (THETIS_GD_PULL) {
            const float sl = ld_cs_f32(L.z + L.n_s + i);
            rv = (double)(row_sigma(L, i) < 0.0f ? -sl : sl);
        } else {
            rv = (double)ld_cs_f32(L.r + i);
        }
        if (rv != 0.0) {
            red_D_slot(Dg, e.x, rv, pol);
            red_D_slot(Dg, e.y, rv, pol);
        }
    }
}

// ---- per-solve and per-epoch preparation of the big tiles' events
__global__ void k_list_big(DevLP L, int64_t n_struct_tiles, PiJob* jobs, unsigned long long* count,
                           unsigned long long* chunks) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_struct_tiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        int a, b;
        scalar_lanes(L, t * 32, a, b);
        if (a >= b) continue;
        const int64_t j0 = L.n_blocks * L.k + (t * 32 + a - L.n_blocks);
        const int64_t cb = L.colptr[j0], ce = L.colptr[j0 + (b - a)];
        if (ce - cb <= kJobMin) continue;
        const int32_t n = (int32_t)((ce - cb + kJobChunk - 1) / kJobChunk);
        if (jobs) {
            const unsigned long long i = atomicAdd(count, 1ull);
            jobs[i].tile = t;
            jobs[i].cb = cb;
            jobs[i].ce = ce;
            jobs[i].n_chunks = n;
        } else {
            atomicAdd(count, 1ull);
            atomicAdd(chunks, (unsigned long long)n);
        }
    }
}
// per epoch: the events of big tile b -- gathers at its position, scatters G later --
// and the reset of its accumulators
__global__ void k_events(PiJob* jobs, int64_t nb, PermKeys K, int64_t G, uint64_t* keys, int32_t* vals) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        PiJob& J = jobs[b];
        const uint64_t p = tile_perm_inv((uint64_t)J.tile, K);
        const uint64_t ps = p + (uint64_t)G < K.n_tiles ? p + (uint64_t)G : K.n_tiles;
        keys[2 * b] = (p << 1) | 1u;
        vals[2 * b] = (int32_t)(2 * b + 1);
        keys[2 * b + 1] = ps << 1;
        vals[2 * b + 1] = (int32_t)(2 * b);
        J.gdone = 0;
        for (int l = 0; l < 32; l++) J.acc[l] = 0.0f;
    }
}
// first slots of the sorted events and the slot count (one CTA)
__global__ void __launch_bounds__(1024) k_event_slots(const PiJob* jobs, int64_t n_ev, int64_t n_tiles,
                                                      const uint64_t* keys, const int32_t* vals, int64_t* ev_pos,
                                                      int64_t* ev_vstart, int64_t* n_slots) {
    typedef cub::BlockScan<int64_t, 1024> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t e0 = 0; e0 < n_ev; e0 += 1024) {
        const int64_t e = e0 + threadIdx.x;
        int64_t delta = 0, pos = 0;
        if (e < n_ev) {
            const int32_t v = vals[e];
            pos = (int64_t)(keys[e] >> 1);
            delta = jobs[v >> 1].n_chunks - (v & 1);  // slots added (a gather replaces its position)
        }
        int64_t excl, total;
        Scan(tmp).ExclusiveSum(delta, excl, total);
        if (e < n_ev) {
            ev_pos[e] = pos;
            ev_vstart[e] = pos + carry + excl;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_slots = n_tiles + carry;
}
__global__ void k_vindex(const int64_t* ev_vstart, int64_t n_ev, const int64_t* n_slots, int64_t n_blocks,
                         int32_t* vindex) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_blocks; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i << kVShift;
        if (v >= *n_slots) continue;
        int64_t lo = 0, hi = n_ev;  // first event with vstart > v
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ev_vstart[mid] <= v) lo = mid + 1;
            else hi = mid;
        }
        vindex[i] = (int32_t)(lo - 1);
    }
}

}  // namespace

// window: at most n_tiles / depth slots drawn and unfinished (bounded staleness),
// filled with as many warps as fit (each warp works on one tile at a time and draws
// window / warps slots at once).  The depth depends on the step rule -- 1/L_j steps are up to
// max_j ||a_j||^2 times longer than 1/L_max's, and the admissible number of concurrent
// updaters "depends on ... the diagonal dominance properties of the Hessian" -- and
// on the form: the residual form delays a big tile's scatter behind its gather and steps
// coupled simplex blocks, and needs a window a quarter as wide as the column-sum form, whose
// hub sums are always current.  Values measured against Alg. 1 (R-6): R-MAT 22 under
// 1/L_max with n_tiles / 512 slots: residual form 1.2e-3 off in c^T x, column-sum form 3.1e-4;
// config 4 at full size (MWC): rounded cut 2% off with n_tiles / 1024, inside 1% with / 2048.
#ifndef THETIS_PI_DEPTH
#define THETIS_PI_DEPTH 2048
#endif
#ifndef THETIS_PI_DEPTH_LJ
#define THETIS_PI_DEPTH_LJ 16384
#endif
#ifndef THETIS_PI_DEPTH_GD
#define THETIS_PI_DEPTH_GD 512
#endif
#ifndef THETIS_PI_DEPTH_GD_LJ   // (R-MAT 24 under 1/L_j: c^T x 1.39e-3 off at 4096, 8.3e-4 at 8192, 6.1e-4 at 16384)
#define THETIS_PI_DEPTH_GD_LJ 16384
#endif

int solve_async_pi(thetis_lp* lp, float beta, int step_rule, int epochs, bool serial, uint64_t seed,
                   cudaEvent_t* epoch_marks, int n_marks) {
    const DevLP& L = lp->d;
    cudaStream_t s = lp->stream;
    StepParams P{};
    P.beta = beta;
    P.beta_d = (double)beta;
    P.inv_beta = (float)(1.0 / (double)beta);
    P.invLmax = (float)(1.0 / ((double)beta * lp->maxnorm2 + 1.0 / (double)beta));  // Eq. 7
    P.rule = step_rule;
    const int64_t n_tiles = (L.U + 31) / 32;
    const int64_t n_struct = L.n_blocks + L.n_scalar;
    const int64_t n_struct_tiles = (n_struct + 31) / 32;
    // column-sum form on edge-incidence LPs (R-23).  THETIS_ASYNC_FORM=residual keeps the
    // residual form there too (same order, same result within rounding: tests run both, A/B timing)
    const char* env_form = getenv("THETIS_ASYNC_FORM");
    const bool gd_ok = (L.problem == THETIS_PROB_VC || L.problem == THETIS_PROB_MIS) && lp->nbr && L.val == nullptr;
    const bool gd = gd_ok && !(env_form && !strcmp(env_form, "residual"));
    // hot prefix: the slots kept in L2 with evict_last (12 B each: x and D), a multiple of 32
#ifndef THETIS_GD_HOT
#define THETIS_GD_HOT (1 << 22)
#endif
    const int64_t hot = (L.n_s < THETIS_GD_HOT ? L.n_s : (int64_t)THETIS_GD_HOT) / 32 * 32;
#ifdef THETIS_GD_FETCH
    if (gd) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, THETIS_GD_FETCH);
#endif
    // (the setup below uses the scratch region before the big-tile lists are carved from it)
    if (gd) {
        if (!lp->nbr_valid) {  // per LP: degree ranks (stable radix sort), neighbour and row ranks
            NvtxRange nvtx_("async column-sum setup");
            Carver Tv(lp->temp);
            uint32_t* rk_key = Tv.take<uint32_t>(2 * L.n_s);
            int32_t* rk_id = Tv.take<int32_t>(2 * L.n_s);
            size_t rb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, rb, rk_key, rk_key + L.n_s, rk_id, rk_id + L.n_s, L.n_s, 0, 32);
            void* rtmp = Tv.take<char>((int64_t)rb);
            if (Tv.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "async rank sort");
            if (L.n_s > 0) {
                k_rank_keys<<<grid_for(L.n_s, 256), 256, 0, s>>>(L, rk_key, rk_id);
                CUDA_TRY(lp, cub::DeviceRadixSort::SortPairs(rtmp, rb, rk_key, rk_key + L.n_s, rk_id, rk_id + L.n_s,
                                                             L.n_s, 0, 32, s));
                k_rank_of<<<grid_for(L.n_s, 256), 256, 0, s>>>(L.n_s, hot, rk_id + L.n_s, lp->rank);
            }
            if (L.nnz_s > 0) k_fill_nbr<<<grid_for((L.nnz_s + kNbrChunk - 1) / kNbrChunk * 32, 256), 256, 0, s>>>(L, lp->rank, lp->nbr);
            if (L.m > 0) k_fill_erank<<<grid_for(L.m, 256), 256, 0, s>>>(L, lp->rank, lp->erank);
            lp->nbr_valid = true;
        }
        CUDA_TRY(lp, cudaMemsetAsync(lp->Dg, 0, sizeof(double) * (size_t)(L.n_s > 0 ? L.n_s : 1), s));
        if (L.n_s > 0) k_init_xr<<<grid_for(L.n_s, 256), 256, 0, s>>>(L, lp->rank, lp->xr);
        if (L.m > 0) k_init_colsum<<<grid_for(L.m, 256), 256, 0, s>>>(L, lp->erank, lp->Dg, hot);
    }
    // big tiles (static per LP): count, then list
    Carver Cv(lp->temp);
    unsigned long long* cnt = Cv.take<unsigned long long>(2);
    CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 16, s));
    if (n_struct_tiles > 0)
        k_list_big<<<grid_for(n_struct_tiles, 256), 256, 0, s>>>(L, n_struct_tiles, nullptr, cnt, cnt + 1);
    unsigned long long hc[2] = {0, 0};
    CUDA_TRY(lp, cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(lp, cudaStreamSynchronize(s));
    const int64_t nb = (int64_t)hc[0], n_ev = 2 * nb;
    const int64_t max_slots = n_tiles + 2 * (int64_t)hc[1];
    const int64_t n_vblocks = (max_slots >> kVShift) + 1;
    PiJob* jobs = Cv.take<PiJob>(nb);
    uint64_t* keys = Cv.take<uint64_t>(2 * n_ev);
    int32_t* vals = Cv.take<int32_t>(2 * n_ev);
    int64_t* ev_pos = Cv.take<int64_t>(n_ev);
    int64_t* ev_vstart = Cv.take<int64_t>(n_ev);
    int32_t* vindex = Cv.take<int32_t>(n_vblocks);
    int64_t* n_slots = Cv.take<int64_t>(1);
    int end_bit = 1;
    while (((int64_t)1 << (end_bit - 1)) <= n_tiles) end_bit++;
    size_t sort_bytes = 0;
    if (n_ev) cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys, keys + n_ev, vals, vals + n_ev, n_ev, 0, end_bit);
    void* sort_tmp = Cv.take<char>((int64_t)sort_bytes);
    if (Cv.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "async big tiles");
    if (nb) {
        CUDA_TRY(lp, cudaMemsetAsync(jobs, 0, nb * sizeof(PiJob), s));
        CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 8, s));
        k_list_big<<<grid_for(n_struct_tiles, 256), 256, 0, s>>>(L, n_struct_tiles, jobs, cnt, nullptr);
    }
    const bool blocks = L.n_blocks > 0;
    const int kind = gd ? 3 : !blocks ? 0 : L.k <= 8 ? 1 : 2;
    // grid: the device's resident warps, or fewer so that the window stays ~n_tiles / depth
    int dev = 0, sms = 0, per_sm = 0;
    CUDA_TRY(lp, cudaGetDevice(&dev));
    CUDA_TRY(lp, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (kind == 0) CUDA_TRY(lp, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async_pi<false, 1, false>, kPiWarps * 32, 0));
    else if (kind == 1) CUDA_TRY(lp, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async_pi<true, 8, false>, kPiWarps * 32, 0));
    else if (kind == 2) CUDA_TRY(lp, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async_pi<true, kMaxK, false>, kPiWarps * 32, 0));
    else CUDA_TRY(lp, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async_pi<false, 1, true>, kPiWarps * 32, 0));
    if (per_sm < 1) per_sm = 1;
    int64_t warps = (int64_t)per_sm * sms * kPiWarps;
    int batch = kPiBatch;
    int64_t depth = gd ? (step_rule == THETIS_STEP_LJ ? THETIS_PI_DEPTH_GD_LJ : THETIS_PI_DEPTH_GD)
                       : (step_rule == THETIS_STEP_LJ ? THETIS_PI_DEPTH_LJ : THETIS_PI_DEPTH);
    // graphs without hubs (largest degree within 8x the average: the ER configs): every column's
    // curvature L_j is within 8x of L_max (so 1/L_j steps are no longer than 8 / L_max), no
    // unit's step moves many rows, and the measured distance to Alg. 1 at the general depth is
    // 300x inside the tolerance (config 2: 3e-6) -- the column-sum form runs them with
    // n_tiles / 64 positions under both step rules (config 2: 2.3e-5 under 1/L_max)
#ifndef THETIS_PI_DEPTH_GD_FLAT
#define THETIS_PI_DEPTH_GD_FLAT 64
#endif
    if (gd && L.n_s > 0 && lp->maxnorm2 * (double)L.n_s <= 8.0 * (double)L.nnz_s) depth = THETIS_PI_DEPTH_GD_FLAT;
    int64_t window = n_tiles / depth;
    if (window < 1) window = 1;
    if (warps * batch > window) {  // the window binds: as many warps as fit, each drawing fewer slots at once
        batch = (int)(window / warps);
        if (batch < 1) batch = 1;
        if (warps * batch > window) warps = window / batch;
        if (warps < 1) warps = 1;
    }
    if (serial) {
        warps = 1;
        batch = 1;
    }
    const int64_t grid = warps >= kPiWarps ? warps / kPiWarps : 1;
    const int threads = warps >= kPiWarps ? kPiWarps * 32 : (int)warps * 32;
    // scatters of a big tile follow its gathers by G positions: a quarter of the window
    // (a scatter drawn before the steps are known waits in its warp's list), one with a
    // single worker (right after them)
#ifndef THETIS_PI_GDIV
#define THETIS_PI_GDIV 4
#endif
    const int64_t G = serial ? 1 : grid * (threads / 32) * batch / THETIS_PI_GDIV + 1;
    PiCtx C{};
    C.n_tiles = n_tiles;
    C.n_struct = n_struct;
    C.jobs = jobs;
    C.n_ev = n_ev;
    C.ev_pos = ev_pos;
    C.ev_vstart = ev_vstart;
    C.ev_val = vals + n_ev;
    C.vindex = vindex;
    C.n_slots = n_slots;
    C.rank = lp->rank;
    C.nbr = lp->nbr;
    C.erank = lp->erank;
    C.xr = lp->xr;
    C.Dg = lp->Dg;
    C.hot = hot;
    for (int e = 0; e < epochs; e++) {
        NvtxRange nvtx_("async epoch");
        C.K = make_perm_keys(n_tiles, seed, e);
        C.stamp = (uint32_t)(e + 1);
        if (nb) {
            k_events<<<grid_for(nb, 256), 256, 0, s>>>(jobs, nb, C.K, G, keys, vals);
            CUDA_TRY(lp, cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, keys, keys + n_ev, vals, vals + n_ev,
                                                         n_ev, 0, end_bit, s));
            k_event_slots<<<1, 1024, 0, s>>>(jobs, n_ev, n_tiles, keys + n_ev, vals + n_ev, ev_pos, ev_vstart, n_slots);
            k_vindex<<<grid_for(n_vblocks, 256), 256, 0, s>>>(ev_vstart, n_ev, n_slots, n_vblocks, vindex);
        } else if (e == 0) {
            CUDA_TRY(lp, cudaMemcpyAsync(n_slots, &n_tiles, 8, cudaMemcpyHostToDevice, s));
            CUDA_TRY(lp, cudaStreamSynchronize(s));  // (pageable source)
        }
        if (n_tiles > 0) {
            if (kind == 0) k_async_pi<false, 1, false><<<(unsigned)grid, threads, 0, s>>>(L, P, C, batch);
            else if (kind == 1) k_async_pi<true, 8, false><<<(unsigned)grid, threads, 0, s>>>(L, P, C, batch);
            else if (kind == 2) k_async_pi<true, kMaxK, false><<<(unsigned)grid, threads, 0, s>>>(L, P, C, batch);
            else k_async_pi<false, 1, true><<<(unsigned)grid, threads, 0, s>>>(L, P, C, batch);
        }
        if (epoch_marks && e < n_marks) CUDA_TRY(lp, cudaEventRecord(epoch_marks[e], s));
    }
    if (gd) THETIS_TRY(recompute_r(lp));  // r = A z - b on return (the epochs never touched r)
    return check_cuda(lp, "async epochs");
}

}  // namespace thetis
