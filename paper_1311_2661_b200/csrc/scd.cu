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
// sequential sweep.  The fp32 operation sequence is fixed (R-7, SURVEY
// §8(c).4): the column dot is 2^17 virtual lanes, lane l summing the column's entries
// at CSC positions l, l + 2^17, ... from +0, combined by halving (off = 2^16 .. 1);
// every operation rounded on its own (__fadd_rn / __fmul_rn / __fdiv_rn), so a thread,
// a warp, a 1024-thread CTA or a hub column split over many CTAs (1024 lanes each,
// k_det_long_lanes / _step / _scatter) gives the bits of the fp32 build of the oracle.
//
// THETIS_MODE_ASYNC (Alg. 1's permuted sweep, Hogwild) lives in async_pi.cu.  This file
// holds the hub-lag throughput variant THETIS_MODE_ASYNC_HUBLAG (R-22), per
// epoch: (1) the row pass -- one stream over the rows with a hub endpoint: the hub
// steps pending from the previous epoch enter r, every slack takes its step, and r is
// accumulated into the hub (and light) columns' D; (2) the hub step -- every hub column
// steps from its D, the step stays pending; (3) the permuted light tiles -- a persistent
// Hogwild kernel (stale reads of r with ld.global.cg, red.global.add.f32 writes, no lost
// update), tile-synchronous within a tile.
#include <algorithm>
#include <array>

#include <cub/cub.cuh>

#include "scd_device.cuh"

namespace thetis {
namespace {

// ------------------------------------------------------------ deterministic
// one colour class: members are structural units; long scalar columns are
// finished by their warp cooperatively with the same sequential summation order
template <int KC>
__global__ void __launch_bounds__(256) k_det_class(DevLP L, StepParams P, const int32_t* __restrict__ members,
                                                   int64_t count) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= count) return;
    const int64_t u = members[idx];
    if (u < L.n_blocks) {
        update_block_seq<false, KC>(L, P, u);
    } else {
        const int64_t j = L.n_blocks * L.k + (u - L.n_blocks);
        if (L.colptr[j + 1] - L.colptr[j] <= kDetWarpCol) update_scalar_seq<false>(L, P, j);
        // longer columns: k_det_mid (one warp each) and k_det_long (one CTA each)
    }
}

// det: one warp per scalar column with kDetWarpCol < nnz <= kDetCtaCol (= 1024: one entry per
// virtual lane slot, lane q holds the contract's lanes q + 32 i).  The row words and the r
// values of the gather stay in registers for the scatter: no unit of the class shares a row,
// so r_i is still the value read (two dependent round trips per column instead of ten).
__global__ void __launch_bounds__(256) k_det_mid(DevLP L, StepParams P, const int32_t* __restrict__ cols, int64_t n) {
    static_assert(kDetCtaCol == 1024, "k_det_mid holds one entry per lane slot");
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    const int64_t j = cols[w];
    const int64_t beg = L.colptr[j], len = L.colptr[j + 1] - beg;
    uint32_t raw[32];
    float rv[32], p[32];
#pragma unroll
    for (int i = 0; i < 32; i++) {
        const int64_t t = lane + 32 * i;
        raw[i] = t < len ? (uint32_t)L.rowidx[beg + t] : 0u;
    }
#pragma unroll
    for (int i = 0; i < 32; i++) {
        const int64_t t = lane + 32 * i;
        rv[i] = t < len ? L.r[raw[i] & kRowMask] : 0.0f;
    }
    const float z = L.z[j], cj = c_int(L, j), ua = ua_of(L, j), zb = zbar_of(L, j);
    const float invL = unit_invL(P, col_norm2(L, j));
    const float lo = col_lo(L, j), hi = col_hi(L, j);
#pragma unroll
    for (int i = 0; i < 32; i++) {
        const int64_t t = lane + 32 * i;
        float term = 0.0f;
        if (t < len) term = L.val ? __fmul_rn(L.val[beg + t], rv[i]) : ((raw[i] & kSignBit) ? -rv[i] : rv[i]);
        p[i] = t < len ? __fadd_rn(0.0f, term) : 0.0f;
    }
#pragma unroll
    for (int s2 = 16; s2 >= 1; s2 >>= 1)  // off = 512 .. 32: within the lane
#pragma unroll
        for (int i = 0; i < s2; i++) p[i] = __fadd_rn(p[i], p[i + s2]);
    float q = p[0];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {  // off = 16 .. 1: across lanes
        const float o = __shfl_down_sync(0xffffffffu, q, off);
        if (lane < off) q = __fadd_rn(q, o);
    }
    const float D = __shfl_sync(0xffffffffu, q, 0);
    const float g = grad_from(cj, ua, D, z, zb, P.beta);
    const float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), lo, hi);
    const float d = __fsub_rn(zn, z);
    if (d != 0.0f) {
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const int64_t t = lane + 32 * i;
            if (t < len) {
                const float ad = L.val ? __fmul_rn(L.val[beg + t], d) : ((raw[i] & kSignBit) ? -d : d);
                L.r[raw[i] & kRowMask] = __fadd_rn(rv[i], ad);
            }
        }
    }
    if (lane == 0) L.z[j] = zn;
}

// det: scalar columns longer than kDetCtaCol (power-law hubs) span many CTAs -- one per
// 1024 virtual lanes of the contract's 2^17 (R-7): a single CTA runs on a single SM, whose
// random-access rate capped a hub column (config 3: 110 ms per epoch); in three launches
// per class:
//   lanes:   CTA (column, b): thread l' computes lane l = 1024 b + l' (its entries l,
//            l + 2^17, ... in order) into P[pbase + l];
//   step:    CTA per column: thread l' combines the lanes l' + 1024 b over b with the
//            tree's offsets 2^16 .. 1024 (b-halving, bit-reversal stack), then the 1024-lane
//            halving through shared memory and shuffles; thread 0 takes the step (z, d);
//   scatter: CTA (column, b): r_i += a_ij d_j over a share of the column's entries
//            (rows of one class are distinct: plain read-modify-write)
struct LongBlk { int32_t col, b, nblk; int64_t pbase; };
// the contract's offsets 2^16 .. 1024 on one 1024-lane slot: with 2^LGB blocks of lanes, the
// halving p_b += p_{b+h} (h = 2^(LGB-1) .. 1) is the binary tree G(r, 2^LG) = G(r, 2^(LG+1)) +
// G(r + 2^LG, 2^(LG+1)) over the residues of b, leaves G(r, 2^LGB) = lane value of block r
// (+0 past the column); Pl points at the slot's value in block 0, blocks are 1024 floats apart
template <int LG, int LGB>
__device__ __forceinline__ float tree_b(const float* __restrict__ Pl, int r, int nblk) {
    if constexpr (LG == LGB) {
        return r < nblk ? Pl[1024 * (int64_t)r] : 0.0f;
    } else {
        const float lo = tree_b<LG + 1, LGB>(Pl, r, nblk);
        const float hi = tree_b<LG + 1, LGB>(Pl, r + (1 << LG), nblk);
        return __fadd_rn(lo, hi);
    }
}
__global__ void __launch_bounds__(1024) k_det_long_lanes(DevLP L, const LongBlk* __restrict__ blk, float* __restrict__ Pbuf) {
    const LongBlk B = blk[blockIdx.x];
    const int64_t cb = L.colptr[B.col], len = L.colptr[B.col + 1] - cb;
    const int64_t l = 1024 * (int64_t)B.b + threadIdx.x;
    Pbuf[B.pbase + l] = l < len ? dot_lane(L, cb, len, l, L.r) : 0.0f;
}
__global__ void __launch_bounds__(1024) k_det_long_step(DevLP L, StepParams P, const LongBlk* __restrict__ cols,
                                                        const float* __restrict__ Pbuf, float* __restrict__ dcol) {
    __shared__ float sp[1024];
    const LongBlk B = cols[blockIdx.x];
    const int l = threadIdx.x, lane = l & 31;
    int lgb = 0;
    while ((1 << lgb) < B.nblk) lgb++;
    const float* Pl = Pbuf + B.pbase + l;
    float comb;
    switch (lgb) {  // the tree over b fully unrolled per depth: loads independent, partial sums in registers
        case 0: comb = tree_b<0, 0>(Pl, 0, B.nblk); break;
        case 1: comb = tree_b<0, 1>(Pl, 0, B.nblk); break;
        case 2: comb = tree_b<0, 2>(Pl, 0, B.nblk); break;
        case 3: comb = tree_b<0, 3>(Pl, 0, B.nblk); break;
        case 4: comb = tree_b<0, 4>(Pl, 0, B.nblk); break;
        case 5: comb = tree_b<0, 5>(Pl, 0, B.nblk); break;
        case 6: comb = tree_b<0, 6>(Pl, 0, B.nblk); break;
        default: comb = tree_b<0, 7>(Pl, 0, B.nblk); break;
    }
    sp[l] = comb;
    __syncthreads();
    for (int off = 512; off >= 32; off >>= 1) {
        if (l < off) sp[l] = __fadd_rn(sp[l], sp[l + off]);
        __syncthreads();
    }
    if (l < 32) {
        float q = sp[l];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const float o = __shfl_down_sync(0xffffffffu, q, off);
            if (lane < off) q = __fadd_rn(q, o);
        }
        if (l == 0) {
            const int64_t j = B.col;
            const float z = L.z[j];
            const float g = grad_from(c_int(L, j), ua_of(L, j), q, z, zbar_of(L, j), P.beta);
            const float invL = unit_invL(P, col_norm2(L, j));
            const float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), col_lo(L, j), col_hi(L, j));
            dcol[blockIdx.x] = __fsub_rn(zn, z);
            L.z[j] = zn;
        }
    }
}
__global__ void __launch_bounds__(1024) k_det_long_scatter(DevLP L, const LongBlk* __restrict__ blk,
                                                           const int32_t* __restrict__ blk_col_idx,
                                                           const float* __restrict__ dcol) {
    const LongBlk B = blk[blockIdx.x];
    const float d = dcol[blk_col_idx[blockIdx.x]];
    if (d == 0.0f) return;
    const int64_t cb = L.colptr[B.col], len = L.colptr[B.col + 1] - cb;
    const int64_t per = (len + B.nblk - 1) / B.nblk, t0 = per * B.b, t1 = t0 + per < len ? t0 + per : len;
    for (int64_t t = t0 + threadIdx.x; t < t1; t += 1024) {
        int64_t row;
        float a;
        entry(L, cb + t, row, a);
        L.r[row] = __fadd_rn(L.r[row], L.val ? __fmul_rn(a, d) : (a < 0.0f ? -d : d));
    }
}
// the class members' scalar columns longer than kDetWarpCol (unordered): (member
// position, column, 1 if longer than kDetCtaCol, its CTAs of 1024 contract lanes)
__global__ void k_det_long_list(DevLP L, int64_t S, const int32_t* __restrict__ members, int32_t* pos,
                                unsigned long long* count) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < S; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = members[p];
        if (u < L.n_blocks) continue;
        const int64_t j = L.n_blocks * L.k + (u - L.n_blocks);
        const int64_t len = L.colptr[j + 1] - L.colptr[j];
        if (len > kDetWarpCol) {
            const unsigned long long i = atomicAdd(count, 1ull);
            pos[4 * i] = (int32_t)p;
            pos[4 * i + 1] = (int32_t)j;
            pos[4 * i + 2] = len > kDetCtaCol;
            pos[4 * i + 3] = (int32_t)((len < kDotLanes ? len : kDotLanes) + 1023) / 1024;  // CTAs of lanes
        }
    }
}

__global__ void __launch_bounds__(256) k_det_slacks(DevLP L, StepParams P) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L.n_ineq; q += (int64_t)gridDim.x * blockDim.x)
        update_slack<false>(L, P, q);
}



// Hub step (R-6): tiles whose scalar columns hold more than kHeavy nonzeros take
// one synchronous step per epoch.  For VC / MIS (every row = one edge (u, v) with
// coefficients +1) it runs as one stream over the rows plus a small update:
//   row pass:  r_e += d_u + d_v (the pending hub steps of the previous epoch),
//              the row's slack step, then r_e into the accumulators D of its hub
//              endpoints;
//   update:    z_j -= (grad_j from D_j) / L for every hub column; d_j pending.
// Rows are grouped by the range of 2^14 ids of their min endpoint (R-17), so one
// block works on one range at a time: the min side's d and D live in shared
// memory (no global atomics for that side); the max side comes in runs of equal
// endpoint inside a range and adds with one atomic per warp run.
// Accumulators and pending steps are compact, hub-major: slot = 32 hub_id + lane.
__device__ __forceinline__ float* acc_of(const float2* hv, int32_t slot) { return (float*)hv + 2 * (int64_t)slot; }
__device__ __forceinline__ float pend_of(const float2* hv, int32_t slot) { return __ldg((const float*)hv + 2 * (int64_t)slot + 1); }
struct HubCtx {
    int64_t n_heavy;
    const int32_t* heavy_tiles;  // sorted tile ids
    const int32_t* hub_id;       // per structural tile: index in heavy_tiles, or -1
    float2* hv;                  // per slot {D_j (accumulated A^T r), d_j (pending step)}:
                                 // the max side reads d and adds into D in one sector
    const int4* items;           // row pass work items {range, row begin, row end, shared}
    int n_items;
    unsigned long long* next;    // work item counter
    const int2* pk;              // per-row keys of the row pass (k_pass_keys)
    float2* lv;                  // hv + 32 n_heavy: per scalar column {D_j from the row pass, pending
                                 // light step d_j}: a light column's rows with a hub endpoint
    int64_t m_defer;             // rows [0, m_defer) have a hub endpoint (R-17)
};
// row-pass keys: an entry of hv (hub slots, then with lv the light columns: lv = hv +
// 32 n_heavy) or, for .x in a shared item, the index into the range's shared arrays;
// -1 nothing
__device__ __forceinline__ float* key_acc(const HubCtx& H, int k) { return (float*)H.hv + 2 * (int64_t)k; }
#ifndef THETIS_PEND_LD
#define THETIS_PEND_LD 1  // L2-only loads (ld.global.cg): 8.28 vs 8.36 ms with __ldg, 9.36 with L1::no_allocate
#endif
__device__ __forceinline__ float key_pend(const HubCtx& H, int k) {
    const float* p = key_acc(H, k) + 1;
#if THETIS_PEND_LD == 1
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
#elif THETIS_PEND_LD == 2
    float v;
    asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ int32_t hub_slot(const HubCtx& H, int32_t v) {
    const int32_t h = H.hub_id[v >> 5];
    return h < 0 ? -1 : h * 32 + (v & 31);
}

__global__ void k_hub_ids(int64_t n_heavy, const int32_t* heavy_tiles, int32_t* hub_id) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < n_heavy; h += (int64_t)gridDim.x * blockDim.x)
        hub_id[heavy_tiles[h]] = (int32_t)h;
}
// first row of every range of min endpoints (rows are sorted by range): lower bound
// (rows [r0, r1) ranged by their min (side 0) or max (side 1) endpoint)
__global__ void k_range_starts(DevLP L, int64_t r0, int64_t r1, int side, int64_t n_ranges, int32_t* start) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g <= n_ranges; g += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = r0, hi = r1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            const int2 uv = L.edges[mid];
            if ((int64_t)((side ? uv.y : uv.x) >> kRowRangeShift) < g) lo = mid + 1;
            else hi = mid;
        }
        start[g] = (int32_t)lo;
    }
}

constexpr int kPassThreads = 1024;             // one block per SM, shared d / D of one range
#ifndef THETIS_ITEM_SHIFT
#define THETIS_ITEM_SHIFT 19
#endif
constexpr int64_t kItemRows = 1 << THETIS_ITEM_SHIFT;  // rows per work item
constexpr int64_t kSharedMinRows = 1 << 14;    // smaller ranges: min side through global memory
constexpr int64_t kSharedMinRowsA = 1 << 12;   // the same for the ranges of the rows with a hub min endpoint only

// v-side of a row: rows come in runs of equal max endpoint (equal key, -1 = none);
// add the warp's run segments with one atomic each.  Fast path when the whole warp
// is one run.
__device__ __forceinline__ void add_max_side(const HubCtx& H, int key, float val, int lane, bool skip = false) {
    const int k0 = __shfl_sync(0xffffffffu, key, 0);
    if (__all_sync(0xffffffffu, key == k0)) {
        if (k0 == -1) return;
#pragma unroll
        for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        if (lane == 0 && !skip) atomicAdd(key_acc(H, k0), val);
        return;
    }
    // segmented suffix sums over the contiguous runs only: a key may come back later in
    // the warp (merged small ranges restart the key sequence), so a lane adds from
    // lane + o only while lane + o lies before the next run head
    const int prev = __shfl_up_sync(0xffffffffu, key, 1);
    const bool head = lane == 0 || prev != key;
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    const unsigned after = lane == 31 ? 0u : heads & (0xFFFFFFFEu << lane);
    const int seg_end = after ? __ffs(after) - 1 : 32;
    float sv = key != -1 ? val : 0.0f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float x = __shfl_down_sync(0xffffffffu, sv, o);
        if (lane + o < seg_end) sv += x;
    }
    if (key != -1 && head && !skip) atomicAdd(key_acc(H, key), sv);
}

// per-row keys of the row pass, built once per solve: .x = the min endpoint's
// index in its range's shared arrays (rows of shared items) or its global key (other
// rows), .y = the max endpoint's global key; rows without a hub endpoint: (-1, -1)
__device__ __forceinline__ int32_t global_key(const HubCtx& H, int32_t v) {
    const int32_t h = hub_slot(H, v);
    return h >= 0 ? h : H.lv ? (int32_t)(H.n_heavy * 32) + v : -1;
}
// .x is the ranged endpoint (rows [0, m_hub_rows): the min one; rows [m_hub_rows,
// m_defer_rows): the max one), .y the other
__global__ void k_pass_keys(DevLP L, HubCtx H, const uint8_t* __restrict__ range_shared,
                            const uint8_t* __restrict__ range_shared_a, int2* __restrict__ pk) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L.m; e += (int64_t)gridDim.x * blockDim.x) {
        if (e >= H.m_defer) {
            pk[e] = make_int2(-1, -1);
            continue;
        }
        const int2 uv = L.edges[e];
        const bool a = e >= L.m_hub_rows && e < L.m_defer_rows;
        const int32_t x = a ? uv.y : uv.x, y = a ? uv.x : uv.y;
        const int32_t g = x >> kRowRangeShift;
        const int32_t gx = global_key(H, x);
        const bool sh = gx != -1 && e < L.m_defer_rows && (a ? range_shared_a[g] : range_shared[g]);
        pk[e] = make_int2(sh ? x - (g << kRowRangeShift) : gx, global_key(H, y));
    }
}

// The row pass (kSlack) or, after a call's last epoch, the application of the
// pending steps alone (!kSlack).  Persistent blocks take work items in order; an
// item with `shared` set stages d of its range in shared memory and accumulates
// the min side of D there, flushed with one atomic per hub column at the end.
// kAnchor: the LP has anchors (zbar / ubar), else both are zero.  The slack step
// is slack_new<true> written out for graph rows (sigma = sg for every row).
// shared memory: d of the range (float) and the min side of D in fixed point with
// resolution 2^-22, kept as two integer sums so that every addition is one native
// shared atomic without a carry (a float add is a CAS loop): x 2^22 = h 2^12 + l with
// h = floor(x 2^10) (signed) and l in [0, 2^12].  An item holds <= 2^19 rows, so
// neither sum can wrap for |x| < 4; larger values go to the global accumulator.
constexpr size_t kPassSmem = 3 * kRowRange * sizeof(float);
constexpr float kFixBound = 4.0f;
__device__ __forceinline__ bool fix_add(uint32_t* lo, int32_t* hi, int i, float x) {
    if (!(fabsf(x) < kFixBound)) return false;
    const float t = x * 1024.0f;                       // exact (power of two)
    const float f = floorf(t);
    atomicAdd(hi + i, (int32_t)f);
    atomicAdd(lo + i, (uint32_t)__float2int_rn((t - f) * 4096.0f));  // t - f exact, in [0, 1)
    return true;
}
__device__ __forceinline__ float fix_value(uint32_t lo, int32_t hi) {
    return (float)(((double)hi * 4096.0 + (double)lo) * (1.0 / 4194304.0));
}
// the keys of rows g .. g + 3 of item w ((-1, -1) outside it)
__device__ __forceinline__ void load_keys4(const int2* __restrict__ pk, int64_t m, const int4& w, int64_t g, int4& k01,
                                           int4& k23) {
    if (g + 4 <= m && g >= w.y && g + 4 <= w.z) {
        k01 = __ldcs((const int4*)(pk + g));
        k23 = __ldcs((const int4*)(pk + g + 2));
        return;
    }
    int2 k[4];
#pragma unroll
    for (int j = 0; j < 4; j++) k[j] = g + j >= w.y && g + j < w.z ? __ldcs(pk + g + j) : make_int2(-1, -1);
    k01 = make_int4(k[0].x, k[0].y, k[1].x, k[1].y);
    k23 = make_int4(k[2].x, k[2].y, k[3].x, k[3].y);
}
template <bool kSlack, bool kAnchor>
__global__ void __launch_bounds__(kPassThreads, 1) k_rows_pass(DevLP L, StepParams P, HubCtx H, int apply, int exp) {
    extern __shared__ float smem[];
    float* s_pend = smem;                                    // d of the range's columns
    uint32_t* s_lo = (uint32_t*)(smem + kRowRange);          // D (min side), fixed point
    int32_t* s_hi = (int32_t*)(smem + 2 * kRowRange);
    __shared__ int32_t s_hub[kRowRange / 32];
    __shared__ int s_it;
    const int lane = threadIdx.x & 31;
    const float sg = row_sigma(L, 0);
    const float invLs = unit_invL(P, 1.0);
    const float beta = P.beta, inv_beta = P.inv_beta;
    float* __restrict__ r = L.r;
    float* __restrict__ zs = L.z + L.n_s;
    const int2* __restrict__ pk = H.pk;
    const bool zvec = (L.n_s & 3) == 0;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_it = (int)atomicAdd(H.next, 1ull);
        __syncthreads();
        const int it = s_it;
        if (it >= H.n_items) return;
        const int4 w = H.items[it];
        if (!kSlack && w.y >= H.m_defer) continue;  // no pending step reaches these rows
        const int32_t base = w.x << kRowRangeShift;
        const bool sh = w.w != 0;
        if (sh) {
            for (int t = threadIdx.x; t < kRowRange / 32; t += blockDim.x)
                s_hub[t] = (int64_t)base + t * 32 < L.n_scalar ? H.hub_id[(base >> 5) + t] : -2;
            __syncthreads();
            constexpr int kPer = (kRowRange + kPassThreads - 1) / kPassThreads;
            float pv[kPer];
#pragma unroll
            for (int q = 0; q < kPer; q++) {  // all loads in flight together
                const int i = threadIdx.x + q * kPassThreads;
                const int32_t h = i < kRowRange ? s_hub[i >> 5] : -2;  // -2: past the columns
                pv[q] = !apply || h == -2 || (h < 0 && !H.lv) ? 0.0f
                        : h >= 0                           ? pend_of(H.hv, h * 32 + (i & 31))
                                                           : pend_of(H.lv, base + i);
            }
#pragma unroll
            for (int q = 0; q < kPer; q++) {
                const int i = threadIdx.x + q * kPassThreads;
                if (i < kRowRange) {
                    s_pend[i] = pv[q];
                    s_lo[i] = 0u;
                    s_hi[i] = 0;
                }
            }
            __syncthreads();
        }
        // four consecutive rows per thread (vector loads; the max side merges its runs in
        // the thread first, then across the warp), groups 4-aligned from a0
        const int64_t a0 = w.y & ~(int64_t)3;
        for (int64_t g0 = a0 + 4 * (int64_t)threadIdx.x; g0 - 4 * lane < w.z; g0 += 4 * (int64_t)blockDim.x) {
            int2 key[4];
            {
                int4 k01, k23;
                load_keys4(pk, L.m, w, g0, k01, k23);
                key[0] = make_int2(k01.x, k01.y); key[1] = make_int2(k01.z, k01.w);
                key[2] = make_int2(k23.x, k23.y); key[3] = make_int2(k23.z, k23.w);
            }
            float r0[4], z[4];
            bool ok[4];
            if (g0 + 4 <= L.m && g0 >= w.y && g0 + 4 <= w.z) {
                const float4 rr = __ldcs((const float4*)(r + g0));
                r0[0] = rr.x; r0[1] = rr.y; r0[2] = rr.z; r0[3] = rr.w;
                if (kSlack) {
                    if (zvec) {
                        const float4 zz = __ldcs((const float4*)(zs + g0));
                        z[0] = zz.x; z[1] = zz.y; z[2] = zz.z; z[3] = zz.w;
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; j++) z[j] = __ldcs(zs + g0 + j);
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; j++) ok[j] = true;
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int64_t e = g0 + j;
                    ok[j] = e >= w.y && e < w.z;
                    r0[j] = ok[j] ? __ldcs(r + e) : 0.0f;
                    z[j] = kSlack && ok[j] ? __ldcs(zs + e) : 0.0f;
                }
            }
            float rv[4];
            float dvp = 0.0f;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                float du = 0.0f, dv = 0.0f;
                if (apply) {
                    if (key[j].x != -1) du = sh ? s_pend[key[j].x] : key_pend(H, key[j].x);
                    if (key[j].y != -1 && !(exp & 4)) {
                        // the thread's rows are sorted by max endpoint: reuse the previous load
                        dv = (j > 0 && key[j].y == key[j - 1].y) ? dvp : key_pend(H, key[j].y);
                        dvp = dv;
                    }
                }
                const float delta = __fadd_rn(du, dv);
                float x = delta != 0.0f ? __fadd_rn(r0[j], delta) : r0[j];
                if (kSlack && ok[j]) {
                    // slack_new<true>: D = sigma r, g = -ua + beta D + (z - zbar) / beta
                    const int64_t e = g0 + j;
                    float ua = 0.0f, zb = 0.0f;
                    if (kAnchor) {
                        if (L.ubar) ua = __fadd_rn(0.0f, sg < 0.0f ? -L.ubar[e] : L.ubar[e]);
                        if (L.zbar) zb = L.zbar[L.n_s + e];
                    }
                    const float D = __fadd_rn(0.0f, sg < 0.0f ? -x : x);
                    float g = __fsub_rn(0.0f, ua);
                    g = __fadd_rn(g, __fmul_rn(beta, D));
                    g = __fadd_rn(g, __fmul_rn(__fsub_rn(z[j], zb), inv_beta));
                    float t = __fsub_rn(z[j], __fmul_rn(g, invLs));
                    t = t < 0.0f ? 0.0f : t;
                    const float d = __fsub_rn(t, z[j]);
                    if (d != 0.0f) {
                        x = __fadd_rn(x, sg < 0.0f ? -d : d);
                        __stcs(zs + e, t);
                    }
                }
                rv[j] = x;
            }
            if (ok[0] && ok[1] && ok[2] && ok[3]) {
                __stcs((float4*)(r + g0), make_float4(rv[0], rv[1], rv[2], rv[3]));
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (ok[j] && rv[j] != r0[j]) __stcs(r + g0 + j, rv[j]);
            }
            if (kSlack) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    if (key[j].x != -1 && !(exp & 2)) {
                        if (!sh) atomicAdd(key_acc(H, key[j].x), rv[j]);
                        else if (!fix_add(s_lo, s_hi, key[j].x, rv[j])) {
                            const int i = key[j].x, h = s_hub[i >> 5];
                            atomicAdd(h >= 0 ? acc_of(H.hv, h * 32 + (i & 31)) : acc_of(H.lv, base + i), rv[j]);
                        }
                    }
                }
                if (!(exp & 1)) {
                    // max side: runs inside the thread; the first run may continue the
                    // previous lane's last run, the last run may continue into the next lane
                    const int k0 = key[0].y, k1 = key[1].y, k2 = key[2].y, k3 = key[3].y;
                    const bool b1 = k1 != k0, b2 = k2 != k1, b3 = k3 != k2;  // run heads at 1, 2, 3
                    const bool single = !b1 && !b2 && !b3;
                    float head = rv[0];
                    if (!b1) head += rv[1];
                    if (!b1 && !b2) head += rv[2];
                    if (single) head += rv[3];
                    float tail = rv[3];
                    if (!b3) tail += rv[2];
                    if (!b3 && !b2) tail += rv[1];
                    if (single) tail = head;
                    // complete runs strictly inside the thread: {1}, {1, 2} or {2}
                    if (b1 && b2 && k1 != -1) atomicAdd(key_acc(H, k1), rv[1]);
                    if (b1 && !b2 && b3 && k1 != -1) atomicAdd(key_acc(H, k1), rv[1] + rv[2]);
                    if (b2 && b3 && k2 != -1) atomicAdd(key_acc(H, k2), rv[2]);
                    // a non-single next lane hands its head to my tail when the run continues
                    const int nk0 = __shfl_down_sync(0xffffffffu, key[0].y, 1);
                    const float nh = __shfl_down_sync(0xffffffffu, head, 1);
                    const bool nsingle = __shfl_down_sync(0xffffffffu, (int)single, 1);
                    if (lane < 31 && !nsingle && nk0 == key[3].y) tail += nh;
                    const int pk3 = __shfl_up_sync(0xffffffffu, key[3].y, 1);
                    if (!single && !(lane > 0 && key[0].y == pk3) && key[0].y != -1) atomicAdd(key_acc(H, key[0].y), head);
                    add_max_side(H, key[3].y, tail, lane, exp & 8);
                }
            }
        }
        if (kSlack && sh) {
            __syncthreads();
            for (int i = threadIdx.x; i < kRowRange; i += blockDim.x) {
                const int32_t h = s_hub[i >> 5];
                const uint32_t lo = s_lo[i];
                const int32_t hi = s_hi[i];
                if ((lo | (uint32_t)hi) && (h >= 0 || H.lv))
                    atomicAdd(h >= 0 ? acc_of(H.hv, h * 32 + (i & 31)) : acc_of(H.lv, base + i), fix_value(lo, hi));
            }
        }
    }
}
// the hub steps from the accumulated A^T r: z_j takes the step, d_j becomes
// pending (applied to r by the next row pass)
__global__ void k_hub_update(DevLP L, StepParams P, HubCtx H) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= H.n_heavy * 32) return;
    const int64_t j = (int64_t)H.heavy_tiles[i >> 5] * 32 + (i & 31);
    if (j >= L.n_scalar) { H.hv[i] = make_float2(0.0f, 0.0f); return; }
    float z = L.z[j];
    float g = grad_fast(c_int(L, j), ua_of(L, j), H.hv[i].x, z, zbar_of(L, j), P.beta, P.inv_beta);
    float invL = P.rule == THETIS_STEP_LMAX ? P.invLmax : unit_invL(P, col_norm2(L, j));
    float zn = clamp_lohi(__fsub_rn(z, __fmul_rn(g, invL)), col_lo(L, j), col_hi(L, j));
    L.z[j] = zn;
    H.hv[i] = make_float2(0.0f, __fsub_rn(zn, z));  // D restarts at 0 for the next row pass
}
// (2) without a hub step: the slack sweep
__global__ void __launch_bounds__(256) k_slack_sweep(DevLP L, StepParams P) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L.n_ineq; q += (int64_t)gridDim.x * blockDim.x)
        update_slack<true>(L, P, q);
}

struct AsyncCtx {
    PermKeys K;
    int64_t n_tiles, heavy_limit;  // tiles above heavy_limit were done by the hub step
    unsigned long long* next;      // position counters (one per stream, 256 B apart)
    int streams;
    const int32_t* hub_id;         // per tile: >= 0 for hub tiles (skipped), or null
    int exp;                       // experiment switches (THETIS_EXP; 0 in production)
    float2* lv;                    // with a hub step: per scalar column {D from the row pass, pending step}
    int64_t m_defer;               // rows [0, m_defer) reach the tiles through lv (R-6), others directly
    const int64_t* ll_off;         // with lv: per scalar column, its rows >= m_defer are
    const int32_t* ll_row;         //   ll_row[ll_off[j] .. ll_off[j + 1])
};

// The loads of a tile that do not depend on r, issued one tile ahead: its column
// starts (lane i: column i; every lane: the end) and the lane's column z and c.
// z_j has a single writer per epoch (the tile's own worker), so the early read
// sees the same value as a late one.
struct TilePre {
    TileCols tc;
    int64_t cp, cp_end;
    float z, c, acc;  // acc: the row pass's part of D (lv), 0 without a hub step
};
__device__ __forceinline__ TilePre prefetch_tile(const DevLP& L, const AsyncCtx& C, int64_t tile, int lane) {
    TilePre t;
    t.tc.u0 = tile * 32;
    int b;
    scalar_lanes(L, t.tc.u0, t.tc.a, b);
    t.tc.ncols = b - t.tc.a;
    t.tc.j0 = L.n_blocks * L.k + (t.tc.u0 + t.tc.a - L.n_blocks);
    t.cp = t.cp_end = 0;
    t.z = t.c = t.acc = 0.0f;
    if (t.tc.ncols > 0) {
        if (lane < t.tc.ncols) {
            const int64_t j = t.tc.j0 + lane;
            t.z = L.z[j];
            t.c = c_int(L, j);
            if (C.lv) {  // with lv: the lane's own rows >= m_defer
                t.acc = C.lv[j].x;
                t.cp = C.ll_off[j];
                t.cp_end = C.ll_off[j + 1];
            } else {
                t.cp = L.colptr[j];
            }
        }
        if (!C.lv) t.cp_end = L.colptr[t.tc.j0 + t.tc.ncols];
    }
    return t;
}

// a light tile with lv (VC / MIS rows, coefficients +1): D = the row pass's part plus
// the lane's few rows without a hub endpoint; the step reaches the rows with a hub
// endpoint through the next row pass (lv.y), the others directly
__device__ __forceinline__ void process_light_tile(const DevLP& L, const StepParams& P, const AsyncCtx& C,
                                                   const TilePre& t, int lane) {
    const TileCols& tc = t.tc;
    float D = t.acc;
    for (int64_t q = t.cp; q < t.cp_end; q++) D += ld_cg(L.r + C.ll_row[q]);
    const float d = scalar_step(L, P, tc, D, lane, t.z, t.c);
    if (lane < tc.ncols) C.lv[tc.j0 + lane] = make_float2(0.0f, d);
    __syncwarp();  // tile-synchronous: every gather of the tile before any scatter
    if (d != 0.0f)
        for (int64_t q = t.cp; q < t.cp_end; q++) red_add(L.r + C.ll_row[q], d);
}

// A tile of short scalar columns without lv: one lane per column walks its own CSC
// range (kLaneCol entries at most; the loads of eight entries go out together)
constexpr int kLaneCol = 48;
__device__ __forceinline__ bool lane_tile(const TilePre& t, int lane, int64_t& cb, int64_t& ce) {
    const int64_t nx = __shfl_down_sync(0xffffffffu, t.cp, 1);
    cb = t.cp;
    ce = lane + 1 < t.tc.ncols ? nx : (lane + 1 == t.tc.ncols ? t.cp_end : t.cp);
    if (lane >= t.tc.ncols) ce = cb;
    return __reduce_max_sync(0xffffffffu, (unsigned)(ce - cb)) <= (unsigned)kLaneCol;
}
__device__ __forceinline__ void process_lane_tile(const DevLP& L, const StepParams& P, const TilePre& t, int lane,
                                                  int64_t cb, int64_t ce) {
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
    const float d = scalar_step(L, P, t.tc, D, lane, t.z, t.c);
    __syncwarp();  // tile-synchronous: every gather of the tile before any scatter
    if (d != 0.0f)
        for (int64_t q = cb; q < ce; q++) {
            const uint32_t raw = (uint32_t)L.rowidx[q];
            const float a = entry_val(L, q, raw);
            red_add(L.r + (raw & kRowMask), L.val ? a * d : (a < 0.0f ? -d : d));
        }
}

// (3) One tile of structural units by one warp, tile-synchronous: all units
// gather (stale w.r.t. other tiles in flight), then all scatter.  A hub tile's
// scalar range was stepped by the hub step of this epoch and is skipped.
template <bool kBlocks, int KC>
__device__ void process_tile(const DevLP& L, const StepParams& P, const AsyncCtx& C, const TilePre& t,
                             WarpSmem& sm, int lane) {
    const TileCols& tc = t.tc;
    const int64_t u = tc.u0 + lane;
    const bool is_block = kBlocks && u < L.n_blocks && !(L.unit_fixed && L.unit_fixed[u]);
    float xb[KC];
    if (is_block) block_values<KC>(L, P, u, xb);
    unsigned moved = 0;
    int64_t beg = 0, end = 0;
    if (tc.ncols > 0) {
        beg = __shfl_sync(0xffffffffu, t.cp, 0);
        end = t.cp_end;
        if (end - beg <= C.heavy_limit) {
            if (lane < tc.ncols) sm.cp[lane] = t.cp;
            if (lane == 0) sm.cp[tc.ncols] = end;
            sm.acc[lane] = t.acc;
            __syncwarp();
            if (!(C.exp & 16)) gather_range(L, sm, tc.ncols, beg, end, lane, C.m_defer);
            const float d = scalar_step(L, P, tc, sm.acc[lane], lane, t.z, t.c);
            sm.d[lane] = d;
            // the row pass applies d to the rows below m_defer and accumulates D anew
            if (C.lv && lane < tc.ncols) C.lv[tc.j0 + lane] = make_float2(0.0f, d);
            moved = __ballot_sync(0xffffffffu, d != 0.0f);
        }
    }
    __syncwarp();
    if (is_block) {
#pragma unroll
        for (int l = 0; l < KC; l++)
            if (l < L.k) {
                const int64_t j = u * L.k + l;
                float d = __fsub_rn(xb[l], L.z[j]);
                col_scatter_async(L, j, d);
                L.z[j] = xb[l];
            }
    }
    if (moved && !(C.exp & 32)) scatter_range(L, sm, tc.ncols, beg, end, lane, C.m_defer);
    __syncwarp();
}

// Persistent, one warp = one worker: draw the next `batch` positions of the
// permuted tile sequence (a stream = a contiguous part of the sequence; one
// stream unless the grid is large) and process them.
// resident blocks per SM: the tile loop is latency-bound, so the VC / MIS variant is
// held to few registers for high occupancy; the block variant keeps its
// registers (its simplex arrays would spill); 6 blocks (40 registers) measured best
#ifndef THETIS_ASYNC_MINB
#define THETIS_ASYNC_MINB 6
#endif
#ifndef THETIS_BLOCKS_MINB
#define THETIS_BLOCKS_MINB 3
#endif
// kPath: kPathBlocks (the LP has simplex blocks: MWC), kPathScalar (scalar columns,
// no lv: lane-per-column or warp-cooperative tiles), kPathLight (light tiles with lv)
enum { kPathBlocks = 0, kPathScalar = 1, kPathLight = 2, kPathBlocks8 = 3 /* host side: blocks, k <= 8 */ };
// KC: block capacity (kPathBlocks: 8 for k <= 8, registers; kMaxK otherwise)
template <int kPath, int KC = 1>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kPath == kPathBlocks ? (KC <= 8 ? THETIS_BLOCKS_MINB : 1) : THETIS_ASYNC_MINB)
    k_async(DevLP L, StepParams P, AsyncCtx C, int batch, int64_t n_workers) {
    constexpr bool kBlocks = kPath == kPathBlocks;
    __shared__ WarpSmem wsm[kWarpsPerBlock];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSmem& sm = wsm[w];
    const int64_t gw = blockIdx.x * (int64_t)(blockDim.x >> 5) + w;
    if (gw >= n_workers) return;
    int st = (int)(gw % C.streams);
    const int64_t per = (C.n_tiles + C.streams - 1) / C.streams;
    for (int tries = 0; tries < C.streams;) {
        const int64_t lo = st * per, hi = lo + per < C.n_tiles ? lo + per : C.n_tiles;
        unsigned long long p0 = 0;
        if (lane == 0) p0 = atomicAdd(C.next + st * 32, (unsigned long long)batch);
        p0 = __shfl_sync(0xffffffffu, p0, 0);
        const int64_t first = lo + (int64_t)p0;
        if (first >= hi) { // this stream is exhausted: help the next one
            st = (st + 1) % C.streams;
            tries++;
            continue;
        }
        // the batch's permuted tiles, one Feistel evaluation per lane
        const bool mine_ok = lane < batch && first + lane < hi;
        const int64_t mine = mine_ok ? (int64_t)tile_perm((uint64_t)(first + lane), C.K) : 0;
        // hub tiles were stepped by the hub step of this epoch: drop them up front
        unsigned todo = __ballot_sync(0xffffffffu, mine_ok && !(C.hub_id && C.hub_id[mine] >= 0));
        if (!todo) continue;
        TilePre cur = prefetch_tile(L, C, __shfl_sync(0xffffffffu, mine, __ffs(todo) - 1), lane);
        while (todo) {
            todo &= todo - 1;
            TilePre nxt = cur;  // the next tile's loads go out before this tile's work
            if (todo) nxt = prefetch_tile(L, C, __shfl_sync(0xffffffffu, mine, __ffs(todo) - 1), lane);
            int64_t cb, ce;
            if (kPath == kPathLight) process_light_tile(L, P, C, cur, lane);
            else if ((kPath == kPathScalar || cur.tc.u0 >= L.n_blocks) && lane_tile(cur, lane, cb, ce))
                process_lane_tile(L, P, cur, lane, cb, ce);  // (tiles past the blocks are scalar)
            else process_tile<kBlocks, KC>(L, P, C, cur, sm, lane);
            cur = nxt;
        }
    }
}

__global__ void k_find_heavy(DevLP L, int64_t n_tiles, int64_t limit, int32_t* heavy, uint8_t* flags,
                             unsigned long long* count) {
    for (int64_t tile = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; tile < n_tiles;
         tile += (int64_t)gridDim.x * blockDim.x) {
        int a, b;
        scalar_lanes(L, tile * 32, a, b);
        bool hv = false;
        if (a < b) {
            int64_t j0 = L.n_blocks * L.k + (tile * 32 + a - L.n_blocks);
            hv = L.colptr[j0 + (b - a)] - L.colptr[j0] > limit;
        }
        flags[tile] = hv;
        if (hv) heavy[atomicAdd(count, 1ull)] = (int32_t)tile;
    }
}

// the rows >= m_defer of every light scalar column (lv mode): counts, then the list
__global__ void k_ll_count(DevLP L, const int32_t* __restrict__ hub_id, int64_t m_defer, int64_t* __restrict__ cnt) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < L.n_scalar; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        if (hub_id[j >> 5] < 0)
            for (int64_t t = L.colptr[j]; t < L.colptr[j + 1]; t++) c += (int64_t)(L.rowidx[t] & kRowMask) >= m_defer;
        cnt[j] = c;
    }
}
__global__ void k_ll_fill(DevLP L, const int32_t* __restrict__ hub_id, int64_t m_defer, const int64_t* __restrict__ off,
                          int32_t* __restrict__ rows) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < L.n_scalar; j += (int64_t)gridDim.x * blockDim.x) {
        if (hub_id[j >> 5] >= 0) continue;
        int64_t o = off[j];
        for (int64_t t = L.colptr[j]; t < L.colptr[j + 1]; t++) {
            const int32_t row = (int32_t)(L.rowidx[t] & kRowMask);
            if (row >= m_defer) rows[o++] = row;
        }
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
// updaters small relative to n): at most ~n_tiles / depth warps work at once, and
// never more than the device holds (persistent grid); large LPs are bounded by the
// device, not by the depth.  The bound "depends on n and on the diagonal dominance properties of the
// Hessian": scalar columns (VC / MIS / generic) work with up to n_tiles / 32 tiles in
// flight, the coupled simplex blocks of MWC with n_tiles / 128 (at n_tiles / 32 the
// reduced config-4 run leaves the async tolerance; measured)
constexpr int64_t kAsyncDepth = 32, kAsyncDepthBlocks = 128;
static int64_t async_workers(int64_t n_tiles, int path) {
    // queried per call: occupancy and SM count are per-device properties (a process may
    // solve on several devices), and the queries are cheap next to a solve
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (path == kPathBlocks)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async<kPathBlocks, kMaxK>, kWarpsPerBlock * 32, 0);
    else if (path == kPathBlocks8)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async<kPathBlocks, 8>, kWarpsPerBlock * 32, 0);
    else if (path == kPathScalar) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async<kPathScalar>, kWarpsPerBlock * 32, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async<kPathLight>, kWarpsPerBlock * 32, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t depth_cap = n_tiles / (path == kPathBlocks || path == kPathBlocks8 ? kAsyncDepthBlocks : kAsyncDepth);
    int64_t dev_cap = (int64_t)per_sm * sms * kWarpsPerBlock;
    int64_t w = depth_cap < dev_cap ? depth_cap : dev_cap;
    return w < 1 ? 1 : w;
}

// persistent grid of the row pass: one block per SM (shared d / D of one range); the
// dynamic shared-memory attribute is per device, so it is set on every call
static int64_t pass_blocks() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_rows_pass<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPassSmem);
    cudaFuncSetAttribute(k_rows_pass<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPassSmem);
    cudaFuncSetAttribute(k_rows_pass<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPassSmem);
    return sms;
}

// hub tiles (VC / MIS only, see the hub step): per-tile flags and the sorted
// list, cached per LP in the persistent `heavy` region (8 n_tiles + 8 bytes:
// flags in the first n_tiles bytes, then the list)
static bool hub_step_enabled(const DevLP& L) {
    return L.problem == THETIS_PROB_VC || L.problem == THETIS_PROB_MIS;
}
static uint8_t* hub_flags(thetis_lp* lp) { return (uint8_t*)lp->heavy; }
static int64_t struct_tiles(const DevLP& L) { return (L.n_blocks + L.n_scalar + 31) / 32; }
static int32_t* hub_list(thetis_lp* lp) {
    const int64_t n_tiles = struct_tiles(lp->d);
    return lp->heavy + (n_tiles + 3) / 4;
}
static int ensure_heavy(thetis_lp* lp) {
    if (lp->heavy_valid) return THETIS_OK;
    const DevLP& L = lp->d;
    cudaStream_t s = lp->stream;
    const int64_t n_tiles = struct_tiles(L);
    lp->n_heavy = 0;
    if (hub_step_enabled(L) && n_tiles > 0) {
        Carver C(lp->temp);
        int32_t* unsorted = C.take<int32_t>(n_tiles);
        unsigned long long* cnt = C.take<unsigned long long>(1);
        CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 8, s));
        k_find_heavy<<<grid_for(n_tiles, 256), 256, 0, s>>>(L, n_tiles, kHeavy, unsorted, hub_flags(lp), cnt);
        unsigned long long h = 0;
        CUDA_TRY(lp, cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        lp->n_heavy = (int64_t)h;
        if (h > 0) {
            size_t cb = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, cb, unsorted, hub_list(lp), (int64_t)h, 0, 32);
            void* cubp = C.take<char>((int64_t)cb);
            if (C.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "heavy list temp");
            CUDA_TRY(lp, cub::DeviceRadixSort::SortKeys(cubp, cb, unsorted, hub_list(lp), (int64_t)h, 0, 32, s));
        }
    }
    lp->heavy_valid = true;
    return check_cuda(lp, "heavy tiles");
}

// Diagnostics: THETIS_EXP switches parts of the hub-lag epoch off to split
// its cost, so results are wrong by design; only a library built with -DTHETIS_DIAG reads
// it (tools/diag_rows.py), the production library never does.
#ifdef THETIS_DIAG
static int g_exp = getenv("THETIS_EXP") ? atoi(getenv("THETIS_EXP")) : 0;
#else
static constexpr int g_exp = 0;
#endif
int solve_epochs(thetis_lp* lp, float beta, int epochs, int mode, uint64_t seed, int step_rule,
                 thetis_solve_stats* st) {
    const DevLP& L = lp->d;
    cudaStream_t s = lp->stream;
    if (mode == THETIS_MODE_ASYNC || mode == THETIS_MODE_ASYNC_SERIAL) {
        // the permutation-ordered schedule (async_pi.cu)
        if (st && lp->ev_epoch.empty()) {
            lp->ev_epoch.resize(THETIS_MAX_EPOCH_TIMES + 2);
            for (auto& e : lp->ev_epoch) CUDA_TRY(lp, cudaEventCreate(&e));
        }
        if (st) CUDA_TRY(lp, cudaEventRecord(lp->ev_epoch[0], s));
        THETIS_TRY(solve_async_pi(lp, beta, step_rule, epochs, mode == THETIS_MODE_ASYNC_SERIAL, seed,
                                  st ? lp->ev_epoch.data() + 1 : nullptr, st ? THETIS_MAX_EPOCH_TIMES : 0));
        if (st) {
            CUDA_TRY(lp, cudaStreamSynchronize(s));
            memset(st, 0, sizeof(*st));
            st->epochs = epochs;
            st->L_max = (double)beta * lp->maxnorm2 + 1.0 / (double)beta;
            st->mode = mode;
            st->step_rule = step_rule;
            const int last = epochs < THETIS_MAX_EPOCH_TIMES ? epochs : THETIS_MAX_EPOCH_TIMES;
            for (int e = 0; e < last; e++) {
                float ms = 0;
                CUDA_TRY(lp, cudaEventElapsedTime(&ms, lp->ev_epoch[e], lp->ev_epoch[e + 1]));
                st->ms_per_epoch[e] = ms;
                st->ms_total += ms;
                st->ms_tiles += ms;
            }
        }
        return THETIS_OK;
    }
    StepParams P{};
    P.beta = beta;
    P.beta_d = (double)beta;
    P.inv_beta = (float)(1.0 / (double)beta);
    P.rule = step_rule;
    const double Lmax = (double)beta * lp->maxnorm2 + 1.0 / (double)beta; // Eq. 7
    P.invLmax = (float)(1.0 / Lmax);
    // det: the class members' scalar columns longer than kDetWarpCol, grouped by class
    // (ascending member position): medium ones for k_det_mid, long ones for k_det_long
    std::vector<int64_t> mid_ptr, long_ptr, lblk_ptr;
    int32_t *mid_cols = nullptr, *lblk_col = nullptr;
    LongBlk *lblk = nullptr, *lcols = nullptr;
    float *Pbuf = nullptr, *dcol = nullptr;
    if (mode == THETIS_MODE_DETERMINISTIC) {
        THETIS_TRY(ensure_colouring(lp, seed));
        const int64_t S = L.n_blocks + L.n_scalar;
        mid_ptr.assign(lp->K + 1, 0);
        long_ptr.assign(lp->K + 1, 0);
        lblk_ptr.assign(lp->K + 1, 0);
        if (S > 0 && L.nnz_s > kDetWarpCol) {
            Carver C(lp->temp);
            int32_t* pos = C.take<int32_t>(4 * S);
            unsigned long long* cnt = C.take<unsigned long long>(1);
            mid_cols = C.take<int32_t>(S);
            if (C.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "det long columns");
            CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 8, s));
            const int64_t n_class = lp->class_ptr[lp->K];
            if (n_class > 0) k_det_long_list<<<grid_for(n_class, 256), 256, 0, s>>>(L, n_class, lp->members, pos, cnt);
            unsigned long long h = 0;
            CUDA_TRY(lp, cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(lp, cudaStreamSynchronize(s));
            std::vector<std::array<int32_t, 4>> lst(h);
            if (h) {
                CUDA_TRY(lp, cudaMemcpyAsync(lst.data(), pos, h * 16, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(lp, cudaStreamSynchronize(s));
            }
            std::sort(lst.begin(), lst.end());
            // per class: the mid columns (a warp each), the long columns and their lane CTAs
            std::vector<int32_t> mc, bci;
            std::vector<LongBlk> lc, lb;
            int64_t pmax = 0;
            size_t q = 0;
            for (int64_t c = 0; c < lp->K; c++) {
                mid_ptr[c] = (int64_t)mc.size();
                long_ptr[c] = (int64_t)lc.size();
                lblk_ptr[c] = (int64_t)lb.size();
                int64_t pb = 0;
                for (; q < lst.size() && lst[q][0] < lp->class_ptr[c + 1]; q++) {
                    if (!lst[q][2]) {
                        mc.push_back(lst[q][1]);
                        continue;
                    }
                    const int32_t nblk = lst[q][3];
                    lc.push_back(LongBlk{lst[q][1], 0, nblk, pb});
                    for (int32_t b = 0; b < nblk; b++) {
                        lb.push_back(LongBlk{lst[q][1], b, nblk, pb});
                        bci.push_back((int32_t)(lc.size() - 1 - long_ptr[c]));
                    }
                    pb += 1024 * (int64_t)nblk;
                }
                pmax = pb > pmax ? pb : pmax;
            }
            mid_ptr[lp->K] = (int64_t)mc.size();
            long_ptr[lp->K] = (int64_t)lc.size();
            lblk_ptr[lp->K] = (int64_t)lb.size();
            lcols = C.take<LongBlk>((int64_t)lc.size());
            lblk = C.take<LongBlk>((int64_t)lb.size());
            lblk_col = C.take<int32_t>((int64_t)bci.size());
            Pbuf = C.take<float>(pmax);
            int64_t lmax = 0;
            for (int64_t c = 0; c < lp->K; c++) lmax = std::max(lmax, long_ptr[c + 1] - long_ptr[c]);
            dcol = C.take<float>(lmax);
            if (C.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "det long columns");
            if (!mc.empty()) CUDA_TRY(lp, cudaMemcpyAsync(mid_cols, mc.data(), mc.size() * 4, cudaMemcpyHostToDevice, s));
            if (!lc.empty()) {
                CUDA_TRY(lp, cudaMemcpyAsync(lcols, lc.data(), lc.size() * sizeof(LongBlk), cudaMemcpyHostToDevice, s));
                CUDA_TRY(lp, cudaMemcpyAsync(lblk, lb.data(), lb.size() * sizeof(LongBlk), cudaMemcpyHostToDevice, s));
                CUDA_TRY(lp, cudaMemcpyAsync(lblk_col, bci.data(), bci.size() * 4, cudaMemcpyHostToDevice, s));
            }
            CUDA_TRY(lp, cudaStreamSynchronize(s));  // `mc`, `lc`, `lb`, `bci` are pageable host memory
        }
    }
    const int64_t n_tiles = struct_tiles(L); // (3) permutes the tiles of structural units
    const bool serial = mode == THETIS_MODE_ASYNC_HUBLAG_SERIAL;
    AsyncCtx AC{};
    HubCtx H{};
    int64_t blocks = 1, hub_blocks = 1, workers = 1;
    int path = kPathScalar;
    bool anchored = false;
    int batch = 1;
    if (mode != THETIS_MODE_DETERMINISTIC) {
        THETIS_TRY(ensure_heavy(lp));
        H.n_heavy = lp->n_heavy;
        H.heavy_tiles = hub_list(lp);
        // light columns reach their rows with a hub endpoint through the row pass (R-6):
        // their accumulators follow the hub slots in hv (keys must fit int32)
        const bool defer = H.n_heavy > 0 && H.n_heavy * 32 + L.n_scalar < (int64_t)INT32_MAX && L.n_blocks == 0;
        path = L.n_blocks > 0 ? (L.k <= 8 ? kPathBlocks8 : kPathBlocks) : defer ? kPathLight : kPathScalar;
        workers = serial ? 1 : async_workers(n_tiles, path);
        blocks = (workers + kWarpsPerBlock - 1) / kWarpsPerBlock;
        AC.streams = blocks >= 128 ? (int)(blocks / 64) : 1;
        batch = blocks >= 128 ? kBatch : 1;
        Carver C(lp->temp);
        AC.next = C.take<unsigned long long>(32 * (int64_t)AC.streams);
        int32_t* hub_id = C.take<int32_t>(n_tiles);
        H.hub_id = hub_id;
        H.hv = C.take<float2>(H.n_heavy * 32 + (defer ? L.n_scalar : 0));
        H.lv = defer ? H.hv + H.n_heavy * 32 : nullptr;
        H.next = C.take<unsigned long long>(32 * 2);
        const int64_t n_ranges = (L.n_scalar + kRowRange - 1) / kRowRange;
        int32_t* rstart = C.take<int32_t>(2 * (n_ranges + 1));
        const int64_t max_items = 2 * (L.m / kItemRows) + 4 * n_ranges + 8;
        int4* items = C.take<int4>(H.n_heavy > 0 ? max_items : 1);
        H.items = items;
        uint8_t* range_shared = C.take<uint8_t>(2 * (n_ranges + 1));
        int2* pk = C.take<int2>(H.n_heavy > 0 ? L.m : 1);
        H.pk = pk;
        H.m_defer = defer ? L.m_defer_rows : L.m;  // without lv every row keeps its hub keys
        int64_t* ll_off = defer ? C.take<int64_t>(L.n_scalar + 1) : nullptr;
        int32_t* ll_row = nullptr;
        size_t ll_cub = 0;
        void* ll_cubp = nullptr;
        if (defer) {
            cub::DeviceScan::ExclusiveSum(nullptr, ll_cub, ll_off, ll_off, L.n_scalar + 1);
            ll_cubp = C.take<char>((int64_t)ll_cub);
        }
        if (C.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "async temp");
        if (H.n_heavy > 0) {
            CUDA_TRY(lp, cudaMemsetAsync(hub_id, 0xFF, (size_t)n_tiles * 4, s));
            CUDA_TRY(lp, cudaMemsetAsync(H.hv, 0, (size_t)H.n_heavy * 32 * 8, s));
            if (H.lv) CUDA_TRY(lp, cudaMemsetAsync(H.lv, 0, (size_t)L.n_scalar * 8, s));
            k_hub_ids<<<grid_for(H.n_heavy, 256), 256, 0, s>>>(H.n_heavy, H.heavy_tiles, hub_id);
            // work items of the row pass: ranges of the ranged endpoint, split into chunks
            // of kItemRows; consecutive small ranges merge into one global-memory item
            const int64_t ma0 = L.m_hub_rows, ma1 = L.m_defer_rows;
            k_range_starts<<<grid_for(n_ranges + 1, 256), 256, 0, s>>>(L, 0, ma0, 0, n_ranges, rstart);
            k_range_starts<<<grid_for(n_ranges + 1, 256), 256, 0, s>>>(L, ma0, ma1, 1, n_ranges, rstart + n_ranges + 1);
            std::vector<int32_t> hs(2 * (n_ranges + 1));
            CUDA_TRY(lp, cudaMemcpyAsync(hs.data(), rstart, hs.size() * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(lp, cudaStreamSynchronize(s));
            std::vector<int4> it;
            std::vector<uint8_t> rsh(2 * (n_ranges + 1), 0);
            for (int part = 0; part < 2; part++) {
                const int32_t* st = hs.data() + part * (n_ranges + 1);
                uint8_t* sh = rsh.data() + part * (n_ranges + 1);
                // ranged by the max endpoint: only light columns gain from the shared side
                const int64_t min_rows = part == 0 ? kSharedMinRows : (H.lv ? kSharedMinRowsA : INT64_MAX);
                for (int64_t g = 0; g < n_ranges; g++) {
                    const int32_t b0 = st[g], b1 = st[g + 1];
                    if (b1 <= b0) continue;
                    if (b1 - b0 >= min_rows) {
                        sh[g] = 1;
                        for (int64_t p = b0; p < b1; p += kItemRows)
                            it.push_back(make_int4((int)g, (int)p, (int)(p + kItemRows < b1 ? p + kItemRows : b1), 1));
                    } else if (!it.empty() && it.back().w == 0 && it.back().z == b0 && b1 - it.back().y <= kItemRows) {
                        it.back().z = b1;
                    } else {
                        it.push_back(make_int4((int)g, b0, b1, 0));
                    }
                }
            }
            // rows without a hub endpoint (R-17: the last part): global items
            for (int64_t p = ma1; p < L.m; p += kItemRows)
                it.push_back(make_int4(0, (int)p, (int)(p + kItemRows < L.m ? p + kItemRows : L.m), 0));
            if ((int64_t)it.size() > max_items) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "row pass items");
            H.n_items = (int)it.size();
            if (!it.empty())
                CUDA_TRY(lp, cudaMemcpyAsync(items, it.data(), it.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
            CUDA_TRY(lp, cudaMemcpyAsync(range_shared, rsh.data(), rsh.size(), cudaMemcpyHostToDevice, s));
            k_pass_keys<<<grid_for(L.m, 256), 256, 0, s>>>(L, H, range_shared, range_shared + n_ranges + 1, pk);
            if (H.lv) {  // the light columns' rows without a hub endpoint
                CUDA_TRY(lp, cudaMemsetAsync(ll_off + L.n_scalar, 0, 8, s));
                k_ll_count<<<grid_for(L.n_scalar, 256), 256, 0, s>>>(L, hub_id, H.m_defer, ll_off);
                CUDA_TRY(lp, cub::DeviceScan::ExclusiveSum(ll_cubp, ll_cub, ll_off, ll_off, L.n_scalar + 1, s));
                int64_t n_ll = 0;
                CUDA_TRY(lp, cudaMemcpyAsync(&n_ll, ll_off + L.n_scalar, 8, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(lp, cudaStreamSynchronize(s));
                ll_row = C.take<int32_t>(n_ll > 0 ? n_ll : 1);
                if (C.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "async temp (ll)");
                k_ll_fill<<<grid_for(L.n_scalar, 256), 256, 0, s>>>(L, hub_id, H.m_defer, ll_off, ll_row);
            }
            CUDA_TRY(lp, cudaStreamSynchronize(s));  // `it`, `rsh` are pageable host memory
        }
        AC.n_tiles = n_tiles;
        AC.heavy_limit = hub_step_enabled(L) ? kHeavy : INT64_MAX;
        AC.hub_id = H.n_heavy > 0 ? H.hub_id : nullptr;
        AC.lv = H.lv;
        AC.m_defer = H.lv ? H.m_defer : 0;
        AC.ll_off = ll_off;
        AC.ll_row = ll_row;
        AC.exp = g_exp;
        hub_blocks = pass_blocks();
        anchored = L.zbar != nullptr || L.ubar != nullptr;
    }
    const bool timed = st != nullptr;
    if (timed) {
        if (lp->ev_epoch.empty()) {
            lp->ev_epoch.resize(THETIS_MAX_EPOCH_TIMES + 2);
            for (auto& e : lp->ev_epoch) CUDA_TRY(lp, cudaEventCreate(&e));
        }
    }
    const int n_timed = epochs < THETIS_MAX_EPOCH_TIMES ? epochs : THETIS_MAX_EPOCH_TIMES;
    if (timed && lp->ev_kern.empty()) {
        lp->ev_kern.resize(3 * THETIS_MAX_EPOCH_TIMES);
        for (auto& e : lp->ev_kern) CUDA_TRY(lp, cudaEventCreate(&e));
    }
    // per timed epoch e: [3e] after the row pass, [3e+1] after the hub update, [3e+2]
    // after the tiles (before the final application of the pending steps)
    auto kern_mark = [&](int e, int k) -> int {
        if (timed && e < n_timed) CUDA_TRY(lp, cudaEventRecord(lp->ev_kern[3 * e + k], s));
        return THETIS_OK;
    };
    // det: one epoch = the class launches (identical every epoch), captured once into a
    // CUDA graph (on the side stream) and replayed per epoch: a launch-bound epoch on small
    // LPs pays one graph launch instead of K + 1 kernel launches
    // fork = true (graph capture only): a class's thread columns, warp columns and CTA columns
    // are independent (units of a class share no row), so they are captured as three parallel
    // branches and joined before the next class
    auto det_epoch = [&](cudaStream_t q, bool fork) {
        for (int64_t c = 0; c < lp->K; c++) {
            int64_t beg = lp->class_ptr[c], cnt = lp->class_ptr[c + 1] - beg;
            const int64_t nm = mid_ptr[c + 1] - mid_ptr[c], nl = long_ptr[c + 1] - long_ptr[c];
            const int64_t nb = lblk_ptr[c + 1] - lblk_ptr[c];
            const bool f = fork && (nm > 0 || nl > 0);
            cudaStream_t qm = f ? lp->det_s[0] : q, ql = f ? lp->det_s[1] : q;
            if (f) {
                cudaEventRecord(lp->det_ev[0], q);
                if (nm > 0) cudaStreamWaitEvent(qm, lp->det_ev[0], 0);
                if (nl > 0) cudaStreamWaitEvent(ql, lp->det_ev[0], 0);
            }
            if (cnt > 0 && L.k <= 8) k_det_class<8><<<grid_for(cnt, 256, 1 << 30), 256, 0, q>>>(L, P, lp->members + beg, cnt);
            else if (cnt > 0) k_det_class<kMaxK><<<grid_for(cnt, 256, 1 << 30), 256, 0, q>>>(L, P, lp->members + beg, cnt);
            if (nm > 0) k_det_mid<<<grid_for(32 * nm, 256, 1 << 30), 256, 0, qm>>>(L, P, mid_cols + mid_ptr[c], nm);
            if (nl > 0) {
                k_det_long_lanes<<<(unsigned)nb, 1024, 0, ql>>>(L, lblk + lblk_ptr[c], Pbuf);
                k_det_long_step<<<(unsigned)nl, 1024, 0, ql>>>(L, P, lcols + long_ptr[c], Pbuf, dcol);
                k_det_long_scatter<<<(unsigned)nb, 1024, 0, ql>>>(L, lblk + lblk_ptr[c], lblk_col + lblk_ptr[c], dcol);
            }
            if (f) {
                if (nm > 0) {
                    cudaEventRecord(lp->det_ev[1], qm);
                    cudaStreamWaitEvent(q, lp->det_ev[1], 0);
                }
                if (nl > 0) {
                    cudaEventRecord(lp->det_ev[2], ql);
                    cudaStreamWaitEvent(q, lp->det_ev[2], 0);
                }
            }
        }
        if (L.n_ineq > 0) k_det_slacks<<<grid_for(L.n_ineq, 256), 256, 0, q>>>(L, P);
    };
    // (the previous call's graph is released here, after its launches completed; the last
    // one by thetis_free)
    if (lp->det_graph) {
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        cudaGraphExecDestroy(lp->det_graph);
        lp->det_graph = nullptr;
    }
    cudaGraphExec_t det_graph = nullptr;
    if (mode == THETIS_MODE_DETERMINISTIC && epochs > 1 && lp->side) {
        cudaGraph_t g = nullptr;
        bool fork = true;  // the branch streams and events of the capture (created once per handle)
        for (auto& q : lp->det_s)
            if (!q && cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking) != cudaSuccess) fork = false;
        for (auto& ev : lp->det_ev)
            if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) fork = false;
        cudaGetLastError();
        if (cudaStreamBeginCapture(lp->side, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            det_epoch(lp->side, fork);
            if (cudaStreamEndCapture(lp->side, &g) == cudaSuccess && g) {
                if (cudaGraphInstantiate(&det_graph, g, 0) != cudaSuccess) det_graph = nullptr;
                lp->det_graph = det_graph;  // owned by the handle from here (released on every path)
                cudaGraphDestroy(g);
            }
        }
        cudaGetLastError();  // a failed capture falls back to direct launches
    }
    cudaEvent_t ev_start = timed ? lp->ev_epoch[0] : nullptr;
    if (timed) CUDA_TRY(lp, cudaEventRecord(ev_start, s));
    for (int e = 0; e < epochs; e++) {
        NvtxRange nvtx_(mode == THETIS_MODE_DETERMINISTIC ? "det epoch" : "hub-lag epoch");
        if (mode == THETIS_MODE_DETERMINISTIC) {
            if (det_graph) CUDA_TRY(lp, cudaGraphLaunch(det_graph, s));
            else det_epoch(s, false);
        } else {
            // (1) hub step + (2) slack sweep, fused; or (2) alone
            if (H.n_heavy > 0) {
                const unsigned hb = (unsigned)((H.n_heavy * 32 + 255) / 256);
                CUDA_TRY(lp, cudaMemsetAsync(H.next, 0, 8, s));
                if (anchored) k_rows_pass<true, true><<<(unsigned)hub_blocks, kPassThreads, kPassSmem, s>>>(L, P, H, e > 0, 0);
                else k_rows_pass<true, false><<<(unsigned)hub_blocks, kPassThreads, kPassSmem, s>>>(L, P, H, e > 0, g_exp);
                THETIS_TRY(kern_mark(e, 0));
                k_hub_update<<<hb, 256, 0, s>>>(L, P, H);
                THETIS_TRY(kern_mark(e, 1));
            } else {
                if (L.n_ineq > 0) k_slack_sweep<<<grid_for(L.n_ineq, 256, 148 * 8), 256, 0, s>>>(L, P);
                THETIS_TRY(kern_mark(e, 0));  // (no hub step: the slack sweep stands for the row pass)
                THETIS_TRY(kern_mark(e, 1));
            }
            // (3) the permuted tiles of structural units
            if (n_tiles > 0) {
                CUDA_TRY(lp, cudaMemsetAsync(AC.next, 0, (size_t)AC.streams * 32 * 8, s));
                AC.K = make_perm_keys(n_tiles, seed, e);
                if (path == kPathBlocks8) k_async<kPathBlocks, 8><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, s>>>(L, P, AC, batch, workers);
                else if (path == kPathBlocks) k_async<kPathBlocks, kMaxK><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, s>>>(L, P, AC, batch, workers);
                else if (path == kPathScalar) k_async<kPathScalar><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, s>>>(L, P, AC, batch, workers);
                else k_async<kPathLight><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, s>>>(L, P, AC, batch, workers);
            }
        }
        if (mode != THETIS_MODE_DETERMINISTIC) THETIS_TRY(kern_mark(e, 2));
        // the last epoch's hub steps are still pending: apply them, r = A z - b again
        if (e == epochs - 1 && mode != THETIS_MODE_DETERMINISTIC && H.n_heavy > 0) {
            CUDA_TRY(lp, cudaMemsetAsync(H.next, 0, 8, s));
            k_rows_pass<false, false><<<(unsigned)hub_blocks, kPassThreads, kPassSmem, s>>>(L, P, H, 1, 0);
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
            if (mode != THETIS_MODE_DETERMINISTIC) {
                float a = 0, b = 0, c = 0;
                CUDA_TRY(lp, cudaEventElapsedTime(&a, lp->ev_epoch[e], lp->ev_kern[3 * e]));
                CUDA_TRY(lp, cudaEventElapsedTime(&b, lp->ev_kern[3 * e], lp->ev_kern[3 * e + 1]));
                CUDA_TRY(lp, cudaEventElapsedTime(&c, lp->ev_kern[3 * e + 1], lp->ev_kern[3 * e + 2]));
                st->ms_row_pass += a;
                st->ms_hub_update += b;
                st->ms_tiles += c;
                st->row_pass_launches += 1;
                if (e == epochs - 1 && H.n_heavy > 0) {  // the final application of the pending steps
                    float f = 0;
                    CUDA_TRY(lp, cudaEventElapsedTime(&f, lp->ev_kern[3 * e + 2], lp->ev_epoch[e + 1]));
                    st->ms_row_pass += f;
                    st->row_pass_launches += 1;
                }
            }
        }
    }
    return THETIS_OK;
}

}  // namespace thetis
