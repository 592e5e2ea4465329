// LP builder (kernels K1-K3): graph edge list -> standard-form
// LP in HBM (CSC with sign-bit coefficients, unique edge rows, costs, bounds), the
// initial point z0 with r0 = A z0 - b, and max ||a_j||^2 for L_max (Eq. 7).
//
//   rows: one per unique undirected non-loop edge (u < v) (R-17).  VC / MIS: first
//   the rows with a hub max endpoint, ordered by (u >> kRowRangeShift, v, u) (the
//   rows whose min endpoint lies in one range of 2^14 ids are contiguous: the row
//   pass accumulates that side in shared memory; within a range a vertex's edges to
//   smaller ids are one run); then the other rows with a hub min endpoint, ordered
//   by (v >> kRowRangeShift, u, v) (the same, with the roles of the endpoints
//   swapped); then the rest in (v, u) order.  MWC: all rows in (v, u) order
//   VC  (Eq. 2):   row e = (u < v): x_u + x_v - s_e = 1
//   MIS (App. B.2):           row e:           x_u + x_v + s_e = 1, max w^T x
//   MWC (App. B.3): x_v^l at v*k+l, x_e^l at n*k+e*k+l;
//        row 2(ek+l):   x_e^l + x_u^l - x_v^l - s = 0
//        row 2(ek+l)+1: x_e^l - x_u^l + x_v^l - s = 0
//
// Sort / unique / scan steps use CUB (header-only, part of the CUDA toolkit);
// every LP-specific step is a kernel below.
#include <cub/cub.cuh>

#include "thetis_internal.cuh"

namespace thetis {

namespace {

constexpr int T = 256;

// CUB's onesweep radix sort of 64-bit keys with a tile shape measured on B200
// (256 threads x 32 keys: 54.6 ms vs 77.6 ms for the stock sm_90 tuning on the
// 1.07e9 R-MAT 26 row keys, scratch microbenchmark); everything else as stock
struct KeySortHub {
    using Base = cub::detail::radix::policy_hub<uint64_t, cub::NullType, unsigned long long>;
    using P9 = Base::Policy900;
    struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, P9> {
        static constexpr bool ONESWEEP = true;
        static constexpr int ONESWEEP_RADIX_BITS = 8;
        using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, uint64_t, 8>;
        using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, 8>;
        using OnesweepPolicy = cub::AgentRadixSortOnesweepPolicy<256, 32, uint64_t, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                                                 cub::BLOCK_SCAN_RAKING_MEMOIZE,
                                                                 cub::RADIX_SORT_STORE_DIRECT, 8>;
        using ScanPolicy = P9::ScanPolicy;
        using DownsweepPolicy = P9::DownsweepPolicy;
        using AltDownsweepPolicy = P9::AltDownsweepPolicy;
        using UpsweepPolicy = P9::UpsweepPolicy;
        using AltUpsweepPolicy = P9::AltUpsweepPolicy;
        using SingleTilePolicy = P9::SingleTilePolicy;
        using SegmentedPolicy = P9::SegmentedPolicy;
        using AltSegmentedPolicy = P9::AltSegmentedPolicy;
    };
    using MaxPolicy = Policy1000;
};
cudaError_t sort_keys_u64(void* tmp, size_t& bytes, cub::DoubleBuffer<uint64_t>& keys, int64_t n, int end_bit,
                          cudaStream_t s) {
    cub::DoubleBuffer<cub::NullType> none;
    return cub::DispatchRadixSort<false, uint64_t, cub::NullType, unsigned long long, KeySortHub>::Dispatch(
        tmp, bytes, keys, none, (unsigned long long)n, 0, end_bit, true, s);
}

enum Flag { FLAG_BAD_INPUT = 0, FLAG_DUP_TERMINAL = 1, FLAG_BAD_CSC = 2, FLAG_BAD_CSR = 3, FLAG_BAD_BOUNDS = 4 };

// ---------------------------------------------------------------- K1: keys
// key(u < v) = ((u >> kRowRangeShift) n + v) 2^kRowRangeShift + (u mod 2^kRowRangeShift):
// (range of u, v, u) in 2 log2(n) bits; invalid pairs and self-loops take `sent`
// (> every key) and sort last
// ranged = false (MWC): key = v n + u, (v, u) order
__global__ void k_make_keys(int64_t E, int64_t n, bool ranged, uint64_t sent, const int32_t* __restrict__ src,
                            const int32_t* __restrict__ dst, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ idx, int32_t* flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t u = src[i], v = dst[i];
        if (u < 0 || v < 0 || u >= n || v >= n) {
            atomicOr(&flags[FLAG_BAD_INPUT], 1);
            keys[i] = sent;
        } else if (u == v) {
            keys[i] = sent; // self-loop: sorts last, dropped
        } else {
            uint64_t a = (uint64_t)(u < v ? u : v), b = (uint64_t)(u < v ? v : u);
            keys[i] = ranged ? ((((a >> kRowRangeShift) * (uint64_t)n + b)) << kRowRangeShift) | (a & (kRowRange - 1))
                             : b * (uint64_t)n + a;
        }
        if (idx) idx[i] = (int32_t)i;
    }
}

__global__ void k_decode_edges(int64_t m, int64_t n, bool ranged, const uint64_t* __restrict__ keys,
                               int2* __restrict__ edges) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[e];
        if (!ranged) {
            edges[e] = make_int2((int32_t)(k % (uint64_t)n), (int32_t)(k / (uint64_t)n));
            continue;
        }
        const uint64_t gv = k >> kRowRangeShift;    // g n + max
        const uint64_t g = gv / (uint64_t)n;
        edges[e] = make_int2((int32_t)((g << kRowRangeShift) | (k & (kRowRange - 1))), (int32_t)(gv - g * (uint64_t)n));
    }
}
// R-17 hub partition (VC / MIS): incidences per tile of 32 vertices.  The rows are
// in ranged order here, so a chunk's min endpoints mostly lie in the range of its
// first row: those count in shared memory; max endpoints come in runs (one atomic
// per warp run)
constexpr int kCountChunk = 8192;
__global__ void __launch_bounds__(256) k_tile_counts(int64_t m, const int2* __restrict__ edges, int32_t* cnt) {
    __shared__ int32_t sh[kRowRange / 32];
    const int lane = threadIdx.x & 31;
    for (int64_t c0 = blockIdx.x * (int64_t)kCountChunk; c0 < m; c0 += (int64_t)gridDim.x * kCountChunk) {
        const int g0 = edges[c0].x >> kRowRangeShift;
        for (int t = threadIdx.x; t < kRowRange / 32; t += blockDim.x) sh[t] = 0;
        __syncthreads();
        const int64_t c1 = c0 + kCountChunk < m ? c0 + kCountChunk : m;
        for (int64_t e = c0 + threadIdx.x; e - lane < c1; e += blockDim.x) {
            const int2 uv = e < c1 ? edges[e] : make_int2(-32, -32);
            const int tv = uv.y >> 5;
            const unsigned same = __match_any_sync(0xffffffffu, tv);
            if (tv >= 0 && lane == __ffs(same) - 1) atomicAdd(cnt + tv, __popc(same));
            if (uv.x >= 0) {
                if ((uv.x >> kRowRangeShift) == g0) atomicAdd(sh + ((uv.x & (kRowRange - 1)) >> 5), 1);
                else atomicAdd(cnt + (uv.x >> 5), 1);
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < kRowRange / 32; t += blockDim.x)
            if (sh[t]) atomicAdd(cnt + ((int64_t)g0 << (kRowRangeShift - 5)) + t, sh[t]);
        __syncthreads();
    }
}
struct HubMaxRow {  // the row's max endpoint lies in a hub tile; row = (min, max) as uint64
    const int32_t* cnt;
    __device__ __forceinline__ bool operator()(uint64_t row) const { return cnt[(int32_t)(row >> 32) >> 5] > kHeavy; }
};
// rows with a light max endpoint (R-17): those with a hub min endpoint first, in
// (v >> kRowRangeShift, u, v) order: key = ((v >> shift) n + u) 2^shift + (v mod 2^shift)
// < ka; then the others in (v, u) order: key = ka + v n + u.  Counts the first part.
__global__ void k_light_keys(int64_t m, int64_t n, uint64_t ka, const int2* __restrict__ rows,
                             const int32_t* __restrict__ cnt, uint64_t* __restrict__ keys, unsigned long long* n_a) {
    unsigned long long c = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const int2 uv = rows[e];
        const uint64_t u = (uint64_t)uv.x, v = (uint64_t)uv.y;
        if (cnt[uv.x >> 5] > kHeavy) {
            c++;
            keys[e] = (((v >> kRowRangeShift) * (uint64_t)n + u) << kRowRangeShift) | (v & (kRowRange - 1));
        } else {
            keys[e] = ka + v * (uint64_t)n + u;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(n_a, c);
}
__global__ void k_decode_light(int64_t m, int64_t n, uint64_t ka, const uint64_t* __restrict__ keys,
                               int2* __restrict__ edges) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[e];
        if (k < ka) {
            const uint64_t gu = k >> kRowRangeShift;  // (v >> shift) n + u
            const uint64_t g = gu / (uint64_t)n;
            edges[e] = make_int2((int32_t)(gu - g * (uint64_t)n), (int32_t)((g << kRowRangeShift) | (k & (kRowRange - 1))));
        } else {
            const uint64_t q = k - ka, v = q / (uint64_t)n;
            edges[e] = make_int2((int32_t)(q - v * (uint64_t)n), (int32_t)v);
        }
    }
}

// (endpoint, e) pairs for the stable by-endpoint sorts (side 0: min, 1: max)
__global__ void k_vkeys(int64_t m, const int2* __restrict__ edges, int side, int32_t* __restrict__ vkey,
                        int32_t* __restrict__ eval) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const int2 uv = edges[e];
        vkey[e] = side ? uv.y : uv.x;
        eval[e] = (int32_t)e;
    }
}
// rows per max endpoint: runs of equal max within a warp add with one atomic
__global__ void k_count_max(int64_t m, const int2* __restrict__ edges, int32_t* cnt) {
    const int lane = threadIdx.x & 31;
    for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 - lane < m;
         e0 += (int64_t)gridDim.x * blockDim.x) {
        const int v = e0 < m ? edges[e0].y : -1;
        const unsigned same = __match_any_sync(0xffffffffu, v);
        if (v >= 0 && lane == __ffs(same) - 1) atomicAdd(cnt + v, __popc(same));
    }
}
// run boundaries of a sorted key sequence: start[key] = first pos, end[key] = last pos + 1
__global__ void k_runs_key(int64_t m, const int32_t* __restrict__ key, int32_t* start, int32_t* end) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        int v = key[p];
        if (p == 0 || key[p - 1] != v) start[v] = (int32_t)p;
        if (end && (p == m - 1 || key[p + 1] != v)) end[v] = (int32_t)(p + 1);
    }
}
__global__ void k_degrees(int64_t n, const int32_t* cnt_max, const int32_t* ls, const int32_t* le, int64_t* deg) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n; v += (int64_t)gridDim.x * blockDim.x)
        deg[v] = v < n ? (int64_t)cnt_max[v] + (int64_t)(le[v] - ls[v]) : 0;
}
// incidence lists in ascending row order (R-17): the rows where the vertex is the
// max endpoint (ranges of smaller ids, then its own) come first, then the rows where
// it is the min endpoint (all in its own range, after its max run).  Each part comes
// from a stable by-endpoint sort of the rows; `skip` = count of the first part.
__global__ void k_fill_part(int64_t m, const int32_t* __restrict__ vkey, const int32_t* __restrict__ eval,
                            const int32_t* __restrict__ start, const int32_t* __restrict__ skip,
                            const int64_t* __restrict__ iptr, int32_t* inc) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        int v = vkey[p];
        inc[iptr[v] + (skip ? skip[v] : 0) + (p - start[v])] = eval[p];
    }
}

__global__ void k_max_deg(int64_t n, const int64_t* __restrict__ colptr, unsigned long long* out) {
    unsigned long long best = 0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long d = (unsigned long long)(colptr[j + 1] - colptr[j]);
        best = d > best ? d : best;
    }
    for (int o = 16; o; o >>= 1) {
        unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

// ---------------------------------------------------------------- MWC
__global__ void k_gather_ew(int64_t m, const int32_t* __restrict__ first, const float* __restrict__ ew_in,
                            float* __restrict__ ew) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
        ew[e] = ew_in[first[e]];
}

__global__ void k_mwc_colptr(int64_t n, int64_t m, int k, const int64_t* __restrict__ iptr, int64_t* colptr) {
    const int64_t nk = n * k, ns = nk + m * k;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= ns; j += (int64_t)gridDim.x * blockDim.x) {
        if (j < nk) {
            int64_t v = j / k, l = j % k;
            int64_t deg = iptr[v + 1] - iptr[v];
            colptr[j] = 2 * (int64_t)k * iptr[v] + 2 * l * deg;
        } else {
            colptr[j] = 4 * (int64_t)k * m + 2 * (j - nk);
        }
    }
}
__global__ void k_mwc_fill_vertex(int64_t n, int k, const int64_t* __restrict__ iptr, const int32_t* __restrict__ inc,
                                  const int2* __restrict__ edges, const int64_t* __restrict__ colptr,
                                  int32_t* __restrict__ rowidx) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t p = iptr[v]; p < iptr[v + 1]; p++) {
            int64_t e = inc[p], q = p - iptr[v];
            bool lower = edges[e].x == (int32_t)v;
            for (int l = 0; l < k; l++) {
                int64_t base = colptr[v * k + l] + 2 * q;
                uint32_t r0 = (uint32_t)(2 * (e * k + l)), r1 = r0 + 1;
                rowidx[base] = (int32_t)(lower ? r0 : (r0 | kSignBit));
                rowidx[base + 1] = (int32_t)(lower ? (r1 | kSignBit) : r1);
            }
        }
    }
}
__global__ void k_mwc_fill_edge(int64_t m, int k, int64_t nnz_vertex, int32_t* __restrict__ rowidx,
                                const float* __restrict__ ew, float* __restrict__ c, int64_t nk) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m * k; q += (int64_t)gridDim.x * blockDim.x) {
        rowidx[nnz_vertex + 2 * q] = (int32_t)(2 * q);
        rowidx[nnz_vertex + 2 * q + 1] = (int32_t)(2 * q + 1);
        c[nk + q] = ew[q / k] * 0.5f; // objective (1/2) sum_e c_e sum_l x_e^l
    }
}
__global__ void k_mwc_terminals(int64_t n, int k, int t, const int32_t* __restrict__ terms, int32_t* term_label,
                                int32_t* flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)k * t) return;
    int32_t v = terms[i];
    if (v < 0 || v >= n) { atomicOr(&flags[FLAG_BAD_INPUT], 1); return; }
    if (atomicCAS(&term_label[v], -1, (int32_t)(i / t)) != -1) atomicOr(&flags[FLAG_DUP_TERMINAL], 1);
}
// initial point (R-3): free blocks at the simplex barycentre, terminal blocks at e_l
__global__ void k_mwc_init(int64_t n, int k, const int32_t* __restrict__ term_label, float* __restrict__ z,
                           uint8_t* __restrict__ unit_fixed, int64_t S) {
    const float bary = (float)(1.0 / (double)k);
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x) {
        if (u < n) {
            int tl = term_label[u];
            unit_fixed[u] = tl >= 0;
            for (int l = 0; l < k; l++) z[u * k + l] = tl >= 0 ? (l == tl ? 1.0f : 0.0f) : bary;
        } else {
            unit_fixed[u] = 0;
        }
    }
}

// ---------------------------------------------------------------- generic
__global__ void k_check_csc(int64_t n, int64_t m, int64_t nnz, const int64_t* __restrict__ colptr,
                            const int32_t* __restrict__ rowidx, int32_t* flags, int flag) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = colptr[j], b = colptr[j + 1];
        if ((j == 0 && a != 0) || (j == n - 1 && b != nnz) || b < a || a < 0 || b > nnz) {
            atomicOr(&flags[flag], 1);
            continue;
        }
        for (int64_t t = a; t < b; t++) {
            int32_t i = rowidx[t];
            if (i < 0 || i >= m || (t > a && i <= rowidx[t - 1])) { atomicOr(&flags[flag], 1); break; }
        }
    }
}
// order-independent fingerprint of the entry set, to check CSC == CSR
__device__ __forceinline__ unsigned long long entry_hash(int64_t i, int64_t j, float v) {
    return sm64_mix(((uint64_t)i << 32 | (uint64_t)(uint32_t)j) ^ ((uint64_t)__float_as_uint(v) * 0x9E3779B97F4A7C15ULL));
}
__global__ void k_fp_csc(int64_t n, const int64_t* colptr, const int32_t* rowidx, const float* val,
                         unsigned long long* out) {
    unsigned long long h = 0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        for (int64_t t = colptr[j]; t < colptr[j + 1]; t++) h += entry_hash(rowidx[t], j, val ? val[t] : 1.0f);
    atomicAdd(out, h);
}
__global__ void k_fp_csr(int64_t m, const int64_t* rowptr, const int32_t* rcol, const float* rval,
                         unsigned long long* out) {
    unsigned long long h = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t t = rowptr[i]; t < rowptr[i + 1]; t++) h += entry_hash(i, rcol[t], rval ? rval[t] : 1.0f);
    atomicAdd(out, h);
}
__global__ void k_slack_flags(int64_t m, const int8_t* __restrict__ sense, int32_t* __restrict__ isq,
                              int32_t* flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == m) { isq[i] = 0; continue; }
        int s = sense[i];
        if (s < 0 || s > 2) atomicOr(&flags[FLAG_BAD_INPUT], 1);
        isq[i] = s != THETIS_EQ;
    }
}
__global__ void k_slack_maps(int64_t m, int64_t n, const int8_t* __restrict__ sense, const int32_t* __restrict__ pos,
                             int64_t* __restrict__ row_slack, int32_t* __restrict__ slack_row) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (sense[i] != THETIS_EQ) {
            row_slack[i] = n + pos[i];
            slack_row[pos[i]] = (int32_t)i;
        } else {
            row_slack[i] = -1;
        }
    }
}
__global__ void k_colnorm2(int64_t n, const int64_t* __restrict__ colptr, const float* __restrict__ val,
                           double* __restrict__ out, unsigned long long* max_bits) {
    double best = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t t = colptr[j]; t < colptr[j + 1]; t++) {
            double v = val ? (double)val[t] : 1.0;
            s += v * v;
        }
        if (out) out[j] = s;
        best = s > best ? s : best;
    }
    // non-negative doubles order like their bit patterns
    atomicMax(max_bits, (unsigned long long)__double_as_longlong(best));
}
__global__ void k_generic_init(int64_t n, int64_t n_blocks, int k, const float* __restrict__ lo,
                               const float* __restrict__ hi, float* __restrict__ z, uint8_t* __restrict__ unit_fixed,
                               int32_t* flags) {
    const int64_t S = n_blocks + (n - n_blocks * k);
    const float bary = k > 0 ? (float)(1.0 / (double)k) : 0.0f;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x) {
        int64_t f = u < n_blocks ? u * k : n_blocks * k + (u - n_blocks);
        int64_t cnt = u < n_blocks ? k : 1;
        bool fixed = true;
        for (int64_t j = f; j < f + cnt; j++) {
            float l = lo ? lo[j] : 0.0f, h = hi ? hi[j] : 1.0f;
            if (!(l <= h)) atomicOr(&flags[FLAG_BAD_BOUNDS], 1);
            fixed = fixed && (l == h);
        }
        unit_fixed[u] = fixed;
        for (int64_t j = f; j < f + cnt; j++) {
            float l = lo ? lo[j] : 0.0f, h = hi ? hi[j] : 1.0f;
            float z0;
            if (u < n_blocks && !fixed) {
                z0 = bary;
            } else {
                z0 = 0.0f < l ? l : 0.0f;
                z0 = z0 > h ? h : z0;
            }
            z[j] = z0;
        }
    }
}

// ---------------------------------------------------------------- r0, ua
// r_i = -b_i + sum_j a_ij z_j (ascending columns) + sigma_i s_i, row-sequential fp32
__global__ void k_recompute_r(DevLP L) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.m; i += (int64_t)gridDim.x * blockDim.x) {
        float acc = -row_b(L, i);
        if (L.problem == THETIS_PROB_VC || L.problem == THETIS_PROB_MIS) {
            int2 e = L.edges[i];
            acc = __fadd_rn(acc, L.z[e.x]);
            acc = __fadd_rn(acc, L.z[e.y]);
        } else if (L.problem == THETIS_PROB_MWC) {
            int64_t k = L.k, e = i / (2 * k), rem = i % (2 * k), l = rem >> 1;
            bool second = rem & 1;
            int2 uv = L.edges[e];
            float zu = L.z[(int64_t)uv.x * k + l], zv = L.z[(int64_t)uv.y * k + l];
            float ze = L.z[L.n_vert * k + e * k + l];
            acc = __fadd_rn(acc, second ? -zu : zu);
            acc = __fadd_rn(acc, second ? zv : -zv);
            acc = __fadd_rn(acc, ze);
        } else {
            for (int64_t t = L.rowptr[i]; t < L.rowptr[i + 1]; t++) {
                float a = L.rval ? L.rval[t] : 1.0f;
                acc = __fadd_rn(acc, __fmul_rn(a, L.z[L.rcol[t]]));
            }
        }
        int64_t sl = row_slack_of(L, i);
        if (sl >= 0) acc = __fadd_rn(acc, __fmul_rn(row_sigma(L, i), L.z[sl]));
        L.r[i] = acc;
    }
}
// ua_j = ubar^T a_j, sequential over the column (same contract as the gradient dot)
// ua_j = ubar^T a_j with the contract's column dot, one warp per column
__global__ void k_recompute_ua(DevLP L) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = w0; j < L.n_s; j += nw) {
        const float acc = L.ubar ? col_dot_tree_warp(L, j, L.ubar, lane) : 0.0f;
        if (lane == 0) L.ua[j] = acc;
    }
}

// per-epoch work: every non-fixed unit once (coordinates, nonzeros incl. slacks)
__global__ void k_epoch_work(DevLP L, unsigned long long* out) {
    unsigned long long upd = 0, nnz = 0;
    const int64_t S = L.n_blocks + L.n_scalar;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x) {
        if (L.unit_fixed && L.unit_fixed[u]) continue;
        const int64_t f = u < L.n_blocks ? u * L.k : L.n_blocks * L.k + (u - L.n_blocks);
        const int64_t c = u < L.n_blocks ? L.k : 1;
        upd += (unsigned long long)c;
        nnz += (unsigned long long)(L.colptr[f + c] - L.colptr[f]);
    }
    for (int o = 16; o; o >>= 1) {
        upd += __shfl_xor_sync(0xffffffffu, upd, o);
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
    }
    if ((threadIdx.x & 31) == 0 && (upd || nnz)) {
        atomicAdd(out, upd);
        atomicAdd(out + 1, nnz);
    }
}

// the largest row key + 1 (R-17 key of the pair (n - 2, n - 1), see k_make_keys);
// graph_keys_fit(n): representable in 64 bits
static unsigned __int128 graph_key_end(int64_t n) {
    if (n <= 1) return 1;
    const unsigned __int128 nn = (unsigned __int128)n, u = nn - 2, v = nn - 1;
    return ((((u >> kRowRangeShift) * nn + v)) << kRowRangeShift) + (u & (kRowRange - 1)) + 1;
}
bool graph_keys_fit(int64_t n) {
    // also the keys of the rows with a light max endpoint (k_light_keys): ka + n^2
    const unsigned __int128 nn = (unsigned __int128)(n > 0 ? n : 1);
    const unsigned __int128 ka = (((nn - 1) >> kRowRangeShift) + 1) * nn << kRowRangeShift;
    return graph_key_end(n) <= (unsigned __int128)UINT64_MAX && ka + nn * nn <= (unsigned __int128)UINT64_MAX;
}
uint64_t graph_key_sentinel(int64_t n) { return (uint64_t)graph_key_end(n); }

int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b) != 0) b++;
    return b < 1 ? 1 : b;
}

struct GraphTemps {
    uint64_t *keys, *keys2;
    int32_t *idx, *idx2;
    int32_t *vkey, *vkey2, *eval, *eval2;
    int32_t *us, *ue, *ls, *le;
    int64_t* deg;
    int64_t* iptr;   // MWC: vertex incidence pointers
    int32_t* inc;    // MWC: incidence lists
    float* ew_in;
    int32_t* terms;
    int32_t *src_stage, *dst_stage;
    void* cub;
    size_t cub_bytes;
    int64_t* nsel;
};

size_t cub_bytes_graph(int64_t n, int64_t E, bool pairs) {
    size_t mx = 0, b = 0;
    cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
    cub::DoubleBuffer<int32_t> di(nullptr, nullptr);
    if (pairs) cub::DeviceRadixSort::SortPairs(nullptr, b, dk, di, E, 0, 64);
    cub::DoubleBuffer<uint64_t> dk2(nullptr, nullptr);
    size_t b2 = 0;
    sort_keys_u64(nullptr, b2, dk2, E, 64, 0);
    b = b2 > b ? b2 : b;
    mx = b > mx ? b : mx;
    b = 0;
    if (pairs)
        cub::DeviceSelect::UniqueByKey(nullptr, b, (uint64_t*)nullptr, (int32_t*)nullptr, (uint64_t*)nullptr,
                                       (int32_t*)nullptr, (int64_t*)nullptr, E);
    else
        cub::DeviceSelect::Unique(nullptr, b, (uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t*)nullptr, E);
    mx = b > mx ? b : mx;
    b = 0;
    cub::DevicePartition::If(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t*)nullptr, E,
                             HubMaxRow{nullptr});
    mx = b > mx ? b : mx;
    b = 0;
    cub::DoubleBuffer<int32_t> dv(nullptr, nullptr), de(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, b, dv, de, E, 0, 32);
    mx = b > mx ? b : mx;
    b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, n + 1);
    mx = b > mx ? b : mx;
    return mx;
}

// temporaries needed by the colouring (class lists) and the rounding passes
size_t post_build_temp(int64_t S, int64_t n_struct, int64_t n_vert) {
    size_t b = 0, mx = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, S, 0, 32);
    mx = b;
    // colouring: keys, ids, sorted keys, class start / end (<= S + 2 each), CUB temp
    size_t colour = 8 * 256 + 5 * ((size_t)S + 2) * 4 + mx + 4 * 256;
    // (selection bytes: per vertex, or per set for the set-cover rules)
    size_t round = 8 * 256 + (size_t)n_struct * 4 + 2 * (size_t)(n_vert > n_struct ? n_vert : n_struct) +
                   (size_t)64 * kRedBlocks * 8 + 64 * 8 + 64 + 32 + 16 * (size_t)n_vert + 512;  // + MIS_BANSAL masks
    return colour > round ? colour : round;
}

}  // namespace


// --------------------------------------------------------------------------
// workspace layouts: the size query and the carve run the same code
// --------------------------------------------------------------------------
static size_t graph_layout(int problem, int64_t n, int64_t E, int k, thetis_lp* lp, void* ws, GraphTemps* tp) {
    const bool carve = lp != nullptr;
    Carver C(carve ? ws : nullptr);
    const bool mwc = problem == THETIS_PROB_MWC;
    const int64_t K = mwc ? k : 1;
    const int64_t n_s = mwc ? n * K + E * K : n;
    const int64_t m = mwc ? 2 * K * E : E;
    const int64_t nnz = mwc ? 6 * K * E : 2 * E;
    const int64_t S = mwc ? n + E * K : n;
    const int64_t U = S + m;
    int64_t* colptr = C.take<int64_t>(n_s + 1);
    int32_t* rowidx = C.take<int32_t>(nnz);
    int2* edges = C.take<int2>(E);
    float* c = C.take<float>(n_s);
    float* z = C.take<float>(n_s + m);
    float* r = C.take<float>(m);
    float* ua = C.take<float>(n_s);
    float* ew = mwc ? C.take<float>(E) : nullptr;
    int32_t* term_label = mwc ? C.take<int32_t>(n) : nullptr;
    uint8_t* unit_fixed = mwc ? C.take<uint8_t>(S) : nullptr;
    int32_t* colour = C.take<int32_t>(S);
    int32_t* members = C.take<int32_t>(S);
    int32_t* heavy = C.take<int32_t>(2 * ((U + kTile - 1) / kTile) + 2);
    double* red = C.take<double>(kRedBlocks * 16 + 256);
    int32_t* flags = C.take<int32_t>(64);
    // THETIS_MODE_ASYNC on edge-incidence LPs (async_pi.cu): neighbour lists, column sums
    int32_t* rank = mwc ? nullptr : C.take<int32_t>(n);
    int32_t* nbr = mwc ? nullptr : C.take<int32_t>(nnz);
    int2* erank = mwc ? nullptr : C.take<int2>(E);
    float* xr = mwc ? nullptr : C.take<float>(n);
    double* Dg = mwc ? nullptr : C.take<double>(n);
    // temporaries of the build, reused afterwards by colouring and rounding
    size_t temp_start = (C.off + 255) & ~(size_t)255;
    GraphTemps t{};
    t.keys = C.take<uint64_t>(E);
    t.keys2 = C.take<uint64_t>(E);
    if (mwc) {
        t.idx = C.take<int32_t>(E);
        t.idx2 = C.take<int32_t>(E);
        t.ew_in = C.take<float>(E);
        t.terms = C.take<int32_t>(32 * 4096);
        t.iptr = C.take<int64_t>(n + 1);
        t.inc = C.take<int32_t>(2 * E);
    }
    t.us = C.take<int32_t>(n);
    t.ue = C.take<int32_t>(n);
    t.ls = C.take<int32_t>(n);
    t.le = C.take<int32_t>(n);
    t.deg = C.take<int64_t>(n + 1);
    t.nsel = C.take<int64_t>(4);
    t.cub_bytes = cub_bytes_graph(n, E, mwc);
    t.cub = C.take<char>((int64_t)t.cub_bytes);
    size_t total = C.off;
    size_t post = post_build_temp(S, n_s, n);
    if (!mwc) {  // THETIS_MODE_ASYNC's per-LP setup (async_pi.cu): the degree sort over n (keys, ids, CUB)
        size_t sb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, sb, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                        (int32_t*)nullptr, n, 0, 32);
        const size_t gdt = 16 * (size_t)n + sb + 8 * 256;
        if (gdt > post) post = gdt;
    }
    if (!mwc) {  // the async solve's row pass (scd.cu): row keys, hub slots, light slots, items
        const size_t asy = 8 * (size_t)E + 16 * ((size_t)n + 32) + 4 * (size_t)((n + 31) / 32) +
                           16 * (size_t)(2 * (E >> 19) + 2 * ((n >> 14) + 1) + 4) + (size_t)(n >> 14) + (1 << 20);
        if (asy > post) post = asy;
    }
    if (temp_start + post > total) total = temp_start + post;
    if (carve) {
        DevLP& d = lp->d;
        d.colptr = colptr; d.rowidx = rowidx; d.edges = edges; d.c = c; d.z = z; d.r = r; d.ua = ua;
        d.ew = ew; d.term_label = term_label; d.unit_fixed = unit_fixed;
        lp->colour = colour; lp->members = members; lp->heavy = heavy; lp->red = red; lp->flags = flags;
        lp->rank = rank; lp->nbr = nbr; lp->erank = erank; lp->xr = xr; lp->Dg = Dg; lp->nbr_valid = false;
        lp->temp = (char*)ws + temp_start;
        lp->temp_bytes = total - temp_start;
        // the by-v sort reuses the key double buffers (2 x 8E bytes); host
        // inputs are staged in the second key buffer
        t.vkey = (int32_t*)t.keys;
        t.eval = (int32_t*)t.keys + E;
        t.vkey2 = (int32_t*)t.keys2;
        t.eval2 = (int32_t*)t.keys2 + E;
        t.src_stage = (int32_t*)t.keys2;
        t.dst_stage = (int32_t*)t.keys2 + E;
        *tp = t;
    }
    return total + 256;
}

size_t graph_workspace(int problem, int64_t n, int64_t n_edges, int k, bool, thetis_lp*, void*) {
    return graph_layout(problem, n, n_edges, k, nullptr, nullptr, nullptr);
}

static size_t generic_layout(int64_t m, int64_t n, int64_t nnz, bool has_val, thetis_lp* lp, void* ws,
                             int32_t** scan_buf, void** cub_buf, size_t* cub_bytes) {
    const bool carve = lp != nullptr;
    Carver C(carve ? ws : nullptr);
    const int64_t S = n; // upper bound on structural units
    const int64_t U = n + m;
    int64_t* colptr = C.take<int64_t>(n + 1);
    int32_t* rowidx = C.take<int32_t>(nnz);
    float* val = has_val ? C.take<float>(nnz) : nullptr;
    double* colnorm2 = has_val ? C.take<double>(n) : nullptr;
    int64_t* rowptr = C.take<int64_t>(m + 1);
    int32_t* rcol = C.take<int32_t>(nnz);
    float* rval = has_val ? C.take<float>(nnz) : nullptr;
    float* b = C.take<float>(m);
    int8_t* sense = C.take<int8_t>(m);
    int64_t* row_slack = C.take<int64_t>(m);
    int32_t* slack_row = C.take<int32_t>(m);
    float* c = C.take<float>(n);
    float* lo = C.take<float>(n);
    float* hi = C.take<float>(n);
    uint8_t* unit_fixed = C.take<uint8_t>(S);
    float* z = C.take<float>(n + m);
    float* r = C.take<float>(m);
    float* ua = C.take<float>(n);
    int32_t* colour = C.take<int32_t>(S);
    int32_t* members = C.take<int32_t>(S);
    int32_t* heavy = C.take<int32_t>(2 * ((U + kTile - 1) / kTile) + 2);
    double* red = C.take<double>(kRedBlocks * 16 + 256);
    int32_t* flags = C.take<int32_t>(64);
    size_t temp_start = (C.off + 255) & ~(size_t)255;
    int32_t* scan = C.take<int32_t>(2 * (m + 1));
    size_t cb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cb, (int32_t*)nullptr, (int32_t*)nullptr, m + 1);
    void* cubp = C.take<char>((int64_t)cb);
    size_t total = C.off;
    size_t post = post_build_temp(S, n, 0);
    if (temp_start + post > total) total = temp_start + post;
    if (carve) {
        DevLP& d = lp->d;
        d.colptr = colptr; d.rowidx = rowidx; d.val = val; d.colnorm2 = colnorm2; d.rowptr = rowptr;
        d.rcol = rcol; d.rval = rval; d.b = b; d.sense = sense; d.row_slack = row_slack; d.slack_row = slack_row;
        d.c = c; d.lo = lo; d.hi = hi; d.unit_fixed = unit_fixed; d.z = z; d.r = r; d.ua = ua;
        lp->colour = colour; lp->members = members; lp->heavy = heavy; lp->red = red; lp->flags = flags;
        lp->rank = nullptr; lp->nbr = nullptr; lp->erank = nullptr; lp->xr = nullptr; lp->Dg = nullptr; lp->nbr_valid = false;
        lp->temp = (char*)ws + temp_start;
        lp->temp_bytes = total - temp_start;
        *scan_buf = scan;
        *cub_buf = cubp;
        *cub_bytes = cb;
    }
    return total + 256;
}

size_t generic_workspace(int64_t m, int64_t n, int64_t nnz, bool has_val, bool, thetis_lp*, void*) {
    return generic_layout(m, n, nnz, has_val, nullptr, nullptr, nullptr, nullptr, nullptr);
}

// --------------------------------------------------------------------------
int recompute_r(thetis_lp* lp) {
    if (lp->d.m > 0) k_recompute_r<<<grid_for(lp->d.m, T), T, 0, lp->stream>>>(lp->d);
    return check_cuda(lp, "recompute_r");
}
// ALM anchor update (thetis_solve_alm): ubar_i -= beta r_i (fp32, product then
// difference, each rounded), zbar_j = z_j
__global__ void k_alm_update(DevLP L, float* __restrict__ ubar, float* __restrict__ zbar, float beta) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.m; i += stride)
        ubar[i] = __fsub_rn(ubar[i], __fmul_rn(beta, L.r[i]));
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < L.N; j += stride) zbar[j] = L.z[j];
}
int alm_update(thetis_lp* lp, float* ubar, float* zbar, float beta) {
    const int64_t n = lp->d.m > lp->d.N ? lp->d.m : lp->d.N;
    if (n > 0) k_alm_update<<<grid_for(n, T), T, 0, lp->stream>>>(lp->d, ubar, zbar, beta);
    THETIS_TRY(check_cuda(lp, "alm_update"));
    return recompute_ua(lp);
}
int recompute_ua(thetis_lp* lp) {
    if (lp->d.n_s > 0) k_recompute_ua<<<grid_for(32 * lp->d.n_s, T), T, 0, lp->stream>>>(lp->d);
    return check_cuda(lp, "recompute_ua");
}

static int copy_in(thetis_lp* lp, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return THETIS_OK;
    CUDA_TRY(lp, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, lp->stream));
    return THETIS_OK;
}
// device pointers are used in place, host inputs are staged into `buf`
static const void* stage(thetis_lp* lp, const void* src, void* buf, size_t bytes, int* rc) {
    *rc = THETIS_OK;
    if (!src || bytes == 0 || is_device_ptr(src)) return src;
    *rc = copy_in(lp, buf, src, bytes);
    return buf;
}

static int read_flags(thetis_lp* lp, int32_t* h) {
    CUDA_TRY(lp, cudaMemcpyAsync(h, lp->flags, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, lp->stream));
    CUDA_TRY(lp, cudaStreamSynchronize(lp->stream));
    return THETIS_OK;
}

static void fill_units(thetis_lp* lp) {
    DevLP& d = lp->d;
    d.N = d.n_s + d.n_ineq;
    d.n_scalar = d.n_s - d.n_blocks * (d.n_blocks > 0 ? d.k : 0);
    d.U = d.n_blocks + d.n_scalar + d.n_ineq;
}

// the work of one epoch (stats), counted once per LP after the bounds are known
static int count_epoch_work(thetis_lp* lp) {
    unsigned long long* w = (unsigned long long*)(lp->flags + 24);
    CUDA_TRY(lp, cudaMemsetAsync(w, 0, 16, lp->stream));
    const int64_t S = lp->d.n_blocks + lp->d.n_scalar;
    if (S > 0) k_epoch_work<<<grid_for(S, T), T, 0, lp->stream>>>(lp->d, w);
    unsigned long long h[2] = {0, 0};
    CUDA_TRY(lp, cudaMemcpyAsync(h, w, 16, cudaMemcpyDeviceToHost, lp->stream));
    CUDA_TRY(lp, cudaStreamSynchronize(lp->stream));
    lp->epoch_updates = (int64_t)h[0] + lp->d.n_ineq;
    lp->epoch_nnz = (int64_t)h[1] + lp->d.n_ineq;
    return THETIS_OK;
}

int build_graph(thetis_lp* lp, int problem, int64_t n, int64_t E, const int32_t* src, const int32_t* dst,
                const float* vertex_w, const float* edge_w, int k, const int32_t* terminals, int t_per_label) {
    GraphTemps t{};
    graph_layout(problem, n, E, k, lp, lp->ws, &t);
    cudaStream_t s = lp->stream;
    DevLP& d = lp->d;
    const bool mwc = problem == THETIS_PROB_MWC;
    int rc;
    d.problem = problem;
    d.obj_sense = problem == THETIS_PROB_MIS ? THETIS_MAX : THETIS_MIN;
    d.c_sign = problem == THETIS_PROB_MIS ? -1.0f : 1.0f;
    d.k = mwc ? k : 0;
    d.n_vert = n;
    CUDA_TRY(lp, cudaMemsetAsync(lp->flags, 0, 64 * sizeof(int32_t), s));
    const int32_t* srcd = (const int32_t*)stage(lp, src, t.src_stage, (size_t)E * 4, &rc);
    THETIS_TRY(rc);
    const int32_t* dstd = (const int32_t*)stage(lp, dst, t.dst_stage, (size_t)E * 4, &rc);
    THETIS_TRY(rc);
    if (!mwc) THETIS_TRY(copy_in(lp, (void*)d.c, vertex_w, (size_t)n * 4));
    if (mwc) THETIS_TRY(copy_in(lp, t.ew_in, edge_w, (size_t)E * 4));
    if (mwc && t_per_label > 0) THETIS_TRY(copy_in(lp, t.terms, terminals, (size_t)k * t_per_label * 4));

    // ---- K1: canonical keys (u < v, R-17), sort, unique -> rows
    int64_t m = 0;
    if (!graph_keys_fit(n))
        return set_error(lp, THETIS_ERR_NOT_SUPPORTED, "n = %lld: row keys exceed 64 bits", (long long)n);
    if (E > 0) {
        const bool ranged = !mwc;
        const uint64_t sent = ranged ? graph_key_sentinel(n) : (uint64_t)n * (uint64_t)n;
        k_make_keys<<<grid_for(E, T), T, 0, s>>>(E, n, ranged, sent, srcd, dstd, t.keys, mwc ? t.idx : nullptr,
                                                 lp->flags);
        const int end_bit = bits_for(sent);
        size_t cb = t.cub_bytes;
        cub::DoubleBuffer<uint64_t> dk(t.keys, t.keys2);
        const uint64_t* uniq;
        const int32_t* first_idx = nullptr;
        if (mwc) {
            cub::DoubleBuffer<int32_t> di(t.idx, t.idx2);
            CUDA_TRY(lp, cub::DeviceRadixSort::SortPairs(t.cub, cb, dk, di, E, 0, end_bit, s));
            cb = t.cub_bytes;
            CUDA_TRY(lp, cub::DeviceSelect::UniqueByKey(t.cub, cb, dk.Current(), di.Current(), dk.Alternate(),
                                                         di.Alternate(), t.nsel, E, s));
            uniq = dk.Alternate();
            first_idx = di.Alternate(); // stable sort: the first occurrence of each pair
        } else {
            CUDA_TRY(lp, sort_keys_u64(t.cub, cb, dk, E, end_bit, s));
            cb = t.cub_bytes;
            CUDA_TRY(lp, cub::DeviceSelect::Unique(t.cub, cb, dk.Current(), dk.Alternate(), t.nsel, E, s));
            uniq = dk.Alternate();
        }
        int64_t nsel = 0;
        uint64_t last = 0;
        CUDA_TRY(lp, cudaMemcpyAsync(&nsel, t.nsel, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        if (nsel > 0) {
            CUDA_TRY(lp, cudaMemcpyAsync(&last, uniq + nsel - 1, 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(lp, cudaStreamSynchronize(s));
        }
        m = nsel - (nsel > 0 && last == sent ? 1 : 0);
        int64_t rows = mwc ? 2 * (int64_t)k * m : m;
        if (rows >= ((int64_t)1 << 31))
            return set_error(lp, THETIS_ERR_NOT_SUPPORTED, "too many rows (%lld) for int32 row indices", (long long)rows);
        if (m > 0) k_decode_edges<<<grid_for(m, T), T, 0, s>>>(m, n, ranged, uniq, (int2*)d.edges);
        if (mwc && m > 0) k_gather_ew<<<grid_for(m, T), T, 0, s>>>(m, first_idx, t.ew_in, (float*)d.ew);
    }
    d.m_edges = m;
    d.m_hub_rows = 0;
    d.m_defer_rows = 0;
    if (!mwc && m > 0) {
        // ---- R-17 hub partition: rows with a hub max endpoint keep the ranged order;
        // then the rows with a hub min endpoint, ranged by the max endpoint; then the rest
        int32_t* tcnt = t.us;  // n_tiles <= n counters, rewritten below
        const int64_t n_tiles = (n + 31) / 32;
        CUDA_TRY(lp, cudaMemsetAsync(tcnt, 0, (size_t)n_tiles * 4, s));
        k_tile_counts<<<grid_for((m + kCountChunk - 1) / kCountChunk, 1, 148 * 8), T, 0, s>>>(m, d.edges, tcnt);
        size_t cb = t.cub_bytes;
        uint64_t* part = t.keys;
        CUDA_TRY(lp, cub::DevicePartition::If(t.cub, cb, (const uint64_t*)d.edges, part, t.nsel, m, HubMaxRow{tcnt}, s));
        int64_t m1 = 0;
        CUDA_TRY(lp, cudaMemcpyAsync(&m1, t.nsel, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        d.m_hub_rows = m1;
        d.m_defer_rows = m1;
        const int64_t m2 = m - m1;
        if (m1 > 0) CUDA_TRY(lp, cudaMemcpyAsync((void*)d.edges, part, (size_t)m1 * 8, cudaMemcpyDeviceToDevice, s));
        if (m2 > 0) {
            const uint64_t ka = ((((uint64_t)n - 1) >> kRowRangeShift) + 1) * (uint64_t)n << kRowRangeShift;
            CUDA_TRY(lp, cudaMemsetAsync(t.nsel, 0, 8, s));
            k_light_keys<<<grid_for(m2, T), T, 0, s>>>(m2, n, ka, (const int2*)(part + m1), tcnt, t.keys2,
                                                       (unsigned long long*)t.nsel);
            cub::DoubleBuffer<uint64_t> dk(t.keys2, t.keys);
            cb = t.cub_bytes;
            CUDA_TRY(lp, sort_keys_u64(t.cub, cb, dk, m2, bits_for(ka + (uint64_t)n * (uint64_t)n), s));
            k_decode_light<<<grid_for(m2, T), T, 0, s>>>(m2, n, ka, dk.Current(), (int2*)d.edges + m1);
            int64_t ma = 0;
            CUDA_TRY(lp, cudaMemcpyAsync(&ma, t.nsel, 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(lp, cudaStreamSynchronize(s));
            d.m_defer_rows = m1 + ma;
        }
    }
    THETIS_TRY(check_cuda(lp, "build: keys"));

    // ---- incidence lists, ascending row order per vertex
    int64_t* iptr = mwc ? t.iptr : (int64_t*)d.colptr;
    int32_t* inc = mwc ? t.inc : (int32_t*)d.rowidx;
    if (n > 0) {
        CUDA_TRY(lp, cudaMemsetAsync(t.us, 0, (size_t)n * 4, s));
        CUDA_TRY(lp, cudaMemsetAsync(t.ue, 0, (size_t)n * 4, s));
        CUDA_TRY(lp, cudaMemsetAsync(t.ls, 0, (size_t)n * 4, s));
        CUDA_TRY(lp, cudaMemsetAsync(t.le, 0, (size_t)n * 4, s));
    }
    // max side: counts now, positions after the by-max sort below; min side: the
    // by-min sort gives counts and positions
    if (m > 0) {
        k_count_max<<<grid_for(m, T), T, 0, s>>>(m, d.edges, t.ue);
        k_vkeys<<<grid_for(m, T), T, 0, s>>>(m, d.edges, 0, t.vkey, t.eval);
        cub::DoubleBuffer<int32_t> dv(t.vkey, t.vkey2), de(t.eval, t.eval2);
        size_t cb = t.cub_bytes;
        CUDA_TRY(lp, cub::DeviceRadixSort::SortPairs(t.cub, cb, dv, de, m, 0, bits_for((uint64_t)n), s));
        k_runs_key<<<grid_for(m, T), T, 0, s>>>(m, dv.Current(), t.ls, t.le);
        k_degrees<<<grid_for(n + 1, T), T, 0, s>>>(n, t.ue, t.ls, t.le, t.deg);
        cb = t.cub_bytes;
        CUDA_TRY(lp, cub::DeviceScan::ExclusiveSum(t.cub, cb, t.deg, iptr, n + 1, s));
        k_fill_part<<<grid_for(m, T), T, 0, s>>>(m, dv.Current(), de.Current(), t.ls, t.ue, iptr, inc);
        k_vkeys<<<grid_for(m, T), T, 0, s>>>(m, d.edges, 1, t.vkey, t.eval);
        dv = cub::DoubleBuffer<int32_t>(t.vkey, t.vkey2);
        de = cub::DoubleBuffer<int32_t>(t.eval, t.eval2);
        cb = t.cub_bytes;
        CUDA_TRY(lp, cub::DeviceRadixSort::SortPairs(t.cub, cb, dv, de, m, 0, bits_for((uint64_t)n), s));
        k_runs_key<<<grid_for(m, T), T, 0, s>>>(m, dv.Current(), t.us, nullptr);
        k_fill_part<<<grid_for(m, T), T, 0, s>>>(m, dv.Current(), de.Current(), t.us, nullptr, iptr, inc);
    } else {
        CUDA_TRY(lp, cudaMemsetAsync(iptr, 0, (size_t)(n + 1) * 8, s));
    }
    THETIS_TRY(check_cuda(lp, "build: incidence"));

    unsigned long long* maxdeg = (unsigned long long*)(lp->flags + 16);
    if (!mwc) {
        // ---- K2 VC / MIS: the incidence lists are the CSC (all coefficients +1)
        d.m = m;
        d.n_s = n;
        d.nnz_s = 2 * m;
        d.n_ineq = m;
        d.n_blocks = 0;
        if (n > 0) k_max_deg<<<grid_for(n, T), T, 0, s>>>(n, d.colptr, maxdeg);
        CUDA_TRY(lp, cudaMemsetAsync(d.z, 0, (size_t)(n + m) * 4, s));
    } else {
        // ---- K2 MWC: expand the incidence into the k label columns + edge-label columns
        const int64_t nk = n * k;
        d.m = 2 * (int64_t)k * m;
        d.n_s = nk + m * k;
        d.nnz_s = 6 * (int64_t)k * m;
        d.n_ineq = d.m;
        d.n_blocks = n;
        k_mwc_colptr<<<grid_for(d.n_s + 1, T), T, 0, s>>>(n, m, k, iptr, (int64_t*)d.colptr);
        if (n > 0) k_mwc_fill_vertex<<<grid_for(n, 128), 128, 0, s>>>(n, k, iptr, inc, d.edges, d.colptr,
                                                                       (int32_t*)d.rowidx);
        CUDA_TRY(lp, cudaMemsetAsync((void*)d.c, 0, (size_t)nk * 4, s));
        if (m > 0) k_mwc_fill_edge<<<grid_for(m * k, T), T, 0, s>>>(m, k, 4 * (int64_t)k * m, (int32_t*)d.rowidx,
                                                                     d.ew, (float*)d.c, nk);
        CUDA_TRY(lp, cudaMemsetAsync((void*)d.term_label, 0xFF, (size_t)n * 4, s));
        if (t_per_label > 0)
            k_mwc_terminals<<<grid_for((int64_t)k * t_per_label, T), T, 0, s>>>(n, k, t_per_label, t.terms,
                                                                                (int32_t*)d.term_label, lp->flags);
        CUDA_TRY(lp, cudaMemsetAsync(d.z, 0, (size_t)(d.n_s + d.m) * 4, s));
        const int64_t S = n + m * k;
        if (S > 0) k_mwc_init<<<grid_for(S, T), T, 0, s>>>(n, k, d.term_label, d.z, (uint8_t*)d.unit_fixed, S);
        if (d.n_s > 0) k_max_deg<<<grid_for(d.n_s, T), T, 0, s>>>(d.n_s, d.colptr, maxdeg);
    }
    fill_units(lp);
    CUDA_TRY(lp, cudaMemsetAsync(d.ua, 0, (size_t)(d.n_s > 0 ? d.n_s : 1) * 4, s));
    THETIS_TRY(recompute_r(lp));
    int32_t h[8];
    unsigned long long md = 0;
    CUDA_TRY(lp, cudaMemcpyAsync(&md, maxdeg, 8, cudaMemcpyDeviceToHost, s));
    THETIS_TRY(read_flags(lp, h));
    if (h[FLAG_BAD_INPUT]) return set_error(lp, THETIS_ERR_INVALID_ARG, "vertex id out of range [0, n)");
    if (h[FLAG_DUP_TERMINAL]) return set_error(lp, THETIS_ERR_INVALID_ARG, "a vertex is a terminal twice");
    lp->maxnorm2 = (double)md;
    if (d.n_ineq > 0 && lp->maxnorm2 < 1.0) lp->maxnorm2 = 1.0; // slack columns
    return count_epoch_work(lp);
}

int build_generic(thetis_lp* lp, int64_t m, int64_t n, int64_t nnz, const int64_t* colptr, const int32_t* rowidx,
                  const float* val, const int64_t* rowptr, const int32_t* rcol, const float* rval, const float* b,
                  const float* c, const int8_t* sense, const float* lo, const float* hi, int obj_sense, int block_k,
                  int64_t n_blocks) {
    int32_t* scan = nullptr;
    void* cubp = nullptr;
    size_t cb = 0;
    generic_layout(m, n, nnz, val != nullptr, lp, lp->ws, &scan, &cubp, &cb);
    cudaStream_t s = lp->stream;
    DevLP& d = lp->d;
    d.problem = THETIS_PROB_GENERIC;
    d.obj_sense = obj_sense;
    d.c_sign = obj_sense == THETIS_MAX ? -1.0f : 1.0f;
    d.k = block_k;
    d.m = m;
    d.n_s = n;
    d.nnz_s = nnz;
    d.n_blocks = n_blocks;
    d.n_vert = 0;
    d.m_edges = 0;
    if (!lo) d.lo = nullptr;
    if (!hi) d.hi = nullptr;
    CUDA_TRY(lp, cudaMemsetAsync(lp->flags, 0, 64 * sizeof(int32_t), s));
    THETIS_TRY(copy_in(lp, (void*)d.colptr, colptr, (size_t)(n + 1) * 8));
    THETIS_TRY(copy_in(lp, (void*)d.rowidx, rowidx, (size_t)nnz * 4));
    if (val) THETIS_TRY(copy_in(lp, (void*)d.val, val, (size_t)nnz * 4));
    THETIS_TRY(copy_in(lp, (void*)d.rowptr, rowptr, (size_t)(m + 1) * 8));
    THETIS_TRY(copy_in(lp, (void*)d.rcol, rcol, (size_t)nnz * 4));
    if (val) THETIS_TRY(copy_in(lp, (void*)d.rval, rval, (size_t)nnz * 4));
    THETIS_TRY(copy_in(lp, (void*)d.b, b, (size_t)m * 4));
    THETIS_TRY(copy_in(lp, (void*)d.c, c, (size_t)n * 4));
    if (sense) THETIS_TRY(copy_in(lp, (void*)d.sense, sense, (size_t)m));
    else if (m > 0) CUDA_TRY(lp, cudaMemsetAsync((void*)d.sense, 0, (size_t)m, s));
    if (lo) THETIS_TRY(copy_in(lp, (void*)d.lo, lo, (size_t)n * 4));
    if (hi) THETIS_TRY(copy_in(lp, (void*)d.hi, hi, (size_t)n * 4));
    // validation: CSC and CSR well formed, same entry set (fingerprint)
    unsigned long long* fp = (unsigned long long*)(lp->flags + 16);
    CUDA_TRY(lp, cudaMemsetAsync(fp, 0, 32, s));
    if (n > 0) {
        k_check_csc<<<grid_for(n, T), T, 0, s>>>(n, m, nnz, d.colptr, d.rowidx, lp->flags, FLAG_BAD_CSC);
        k_fp_csc<<<grid_for(n, T), T, 0, s>>>(n, d.colptr, d.rowidx, d.val, fp);
    }
    if (m > 0) {
        k_check_csc<<<grid_for(m, T), T, 0, s>>>(m, n, nnz, d.rowptr, d.rcol, lp->flags, FLAG_BAD_CSR);
        k_fp_csr<<<grid_for(m, T), T, 0, s>>>(m, d.rowptr, d.rcol, d.rval, fp + 1);
    }
    // slack columns in row order (App. C)
    int64_t n_ineq = 0;
    if (m > 0) {
        k_slack_flags<<<grid_for(m + 1, T), T, 0, s>>>(m, d.sense, scan, lp->flags);
        size_t c2 = cb;
        CUDA_TRY(lp, cub::DeviceScan::ExclusiveSum(cubp, c2, scan, scan + (m + 1), m + 1, s));
        k_slack_maps<<<grid_for(m, T), T, 0, s>>>(m, n, d.sense, scan + (m + 1), (int64_t*)d.row_slack,
                                                  (int32_t*)d.slack_row);
        int32_t ni = 0;
        CUDA_TRY(lp, cudaMemcpyAsync(&ni, scan + (m + 1) + m, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        n_ineq = ni;
    }
    d.n_ineq = n_ineq;
    fill_units(lp);
    unsigned long long* mx = fp + 2;
    if (n > 0) k_colnorm2<<<grid_for(n, T), T, 0, s>>>(n, d.colptr, d.val, (double*)d.colnorm2, mx);
    const int64_t S = d.n_blocks + d.n_scalar;
    CUDA_TRY(lp, cudaMemsetAsync(d.z, 0, (size_t)(d.N > 0 ? d.N : 1) * 4, s));
    if (S > 0) k_generic_init<<<grid_for(S, T), T, 0, s>>>(n, n_blocks, block_k, d.lo, d.hi, d.z,
                                                         (uint8_t*)d.unit_fixed, lp->flags);
    CUDA_TRY(lp, cudaMemsetAsync(d.ua, 0, (size_t)(n > 0 ? n : 1) * 4, s));
    THETIS_TRY(recompute_r(lp));
    int32_t h[8];
    unsigned long long hfp[3] = {0, 0, 0};
    CUDA_TRY(lp, cudaMemcpyAsync(hfp, fp, 24, cudaMemcpyDeviceToHost, s));
    THETIS_TRY(read_flags(lp, h));
    if (h[FLAG_BAD_CSC]) return set_error(lp, THETIS_ERR_INVALID_ARG, "malformed CSC (pointers or row indices)");
    if (h[FLAG_BAD_CSR]) return set_error(lp, THETIS_ERR_INVALID_ARG, "malformed CSR (pointers or column indices)");
    if (h[FLAG_BAD_INPUT]) return set_error(lp, THETIS_ERR_INVALID_ARG, "row sense not in {EQ, GE, LE}");
    if (h[FLAG_BAD_BOUNDS]) return set_error(lp, THETIS_ERR_INVALID_ARG, "lo > hi");
    if (hfp[0] != hfp[1]) return set_error(lp, THETIS_ERR_INVALID_ARG, "CSC and CSR hold different entries");
    double mxd;
    memcpy(&mxd, &hfp[2], 8);
    lp->maxnorm2 = mxd;
    if (d.n_ineq > 0 && lp->maxnorm2 < 1.0) lp->maxnorm2 = 1.0;
    return count_epoch_work(lp);
}

}  // namespace thetis
