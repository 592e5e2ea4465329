// K4: colouring of the unit conflict graph for the deterministic mode (R-5).
// Units conflict when they share a row of A.  Jones-Plassmann rounds: an
// uncoloured unit whose higher-priority conflict neighbours are all coloured
// takes the smallest colour none of them uses.  A unit is coloured exactly when
// all units preceding it in priority order among its neighbours are, so the
// result equals the sequential first-fit greedy in priority order.
// Priorities (R-5): largest degree (nonzeros of the unit's columns) first, then
// fmix32(u ^ key), key = fmix32(lo32 seed) ^ hi32 seed, then the smaller id.
// Largest-degree-first colours power-law hubs in the first rounds.
#include <cub/cub.cuh>

#include "thetis_internal.cuh"

namespace thetis {
namespace {

constexpr int T = 256;

__device__ __forceinline__ int64_t unit_of_col(const DevLP& L, int64_t j) {
    const int64_t nbk = L.n_blocks * L.k;
    return j < nbk ? j / L.k : L.n_blocks + (j - nbk);
}
// rank(u) = (nonzeros of u's columns << 32) | fmix32(u ^ key): largest degree
// first, then the larger hash; equal ranks (impossible for distinct hashes) by id
__device__ __forceinline__ bool precedes(uint64_t rw, int64_t w, uint64_t ru, int64_t u) {
    return rw > ru || (rw == ru && w < u);
}
__global__ void k_colour_rank(DevLP L, int64_t S, uint32_t key, uint64_t* rank) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x) {
        int64_t first, cnt;
        if (u < L.n_blocks) { first = u * L.k; cnt = L.k; }
        else { first = L.n_blocks * L.k + (u - L.n_blocks); cnt = 1; }
        const uint64_t deg = (uint64_t)(L.colptr[first + cnt] - L.colptr[first]);
        rank[u] = (deg << 32) | fmix32((uint32_t)u ^ key);
    }
}

// visit the conflict neighbours of unit u (units sharing a row), f(w) returns
// false to stop early
template <class F>
__device__ __forceinline__ void for_each_neighbour(const DevLP& L, int64_t u, F&& f) {
    int64_t first, cnt;
    if (u < L.n_blocks) { first = u * L.k; cnt = L.k; }
    else { first = L.n_blocks * L.k + (u - L.n_blocks); cnt = 1; }
    for (int64_t j = first; j < first + cnt; j++) {
        for (int64_t t = L.colptr[j]; t < L.colptr[j + 1]; t++) {
            int64_t i = (int64_t)((uint32_t)L.rowidx[t] & kRowMask);
            if (L.problem == THETIS_PROB_VC || L.problem == THETIS_PROB_MIS) {
                int2 e = L.edges[i];
                int64_t w = e.x == (int32_t)u ? e.y : e.x;
                if (!f(w)) return;
            } else if (L.problem == THETIS_PROB_MWC) {
                int64_t k = L.k, e = i / (2 * k), l = (i >> 1) % k;
                int2 uv = L.edges[e];
                if ((int64_t)uv.x != u && !f((int64_t)uv.x)) return;
                if ((int64_t)uv.y != u && !f((int64_t)uv.y)) return;
                int64_t we = L.n_blocks + e * k + l;
                if (we != u && !f(we)) return;
            } else {
                for (int64_t q = L.rowptr[i]; q < L.rowptr[i + 1]; q++) {
                    int64_t w = unit_of_col(L, L.rcol[q]);
                    if (w != u && !f(w)) return;
                }
            }
        }
    }
}

// colour[u]: -2 fixed (no part), -1 uncoloured, >= 0 colour
__global__ void k_colour_init(DevLP L, int64_t S, int32_t* colour) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x)
        colour[u] = (L.unit_fixed && L.unit_fixed[u]) ? -2 : -1;
}

// units whose columns hold more than kLongUnit nonzeros are scanned by a warp each
// (k_jp_round_long); the others by one thread
constexpr int64_t kLongUnit = 256;
__device__ __forceinline__ int64_t unit_nnz(const DevLP& L, int64_t u) {
    int64_t first, cnt;
    if (u < L.n_blocks) { first = u * L.k; cnt = L.k; }
    else { first = L.n_blocks * L.k + (u - L.n_blocks); cnt = 1; }
    return L.colptr[first + cnt] - L.colptr[first];
}
__global__ void k_jp_round(DevLP L, int64_t S, const uint64_t* __restrict__ rank, int32_t* colour,
                           unsigned long long* remaining) {
    unsigned long long left = 0;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x) {
        if (colour[u] != -1 || unit_nnz(L, u) > kLongUnit) continue;
        const uint64_t pu = rank[u];
        int32_t base = 0;
        bool ready = true, done = false;
        while (!done) {
            unsigned long long mask = 0;
            for_each_neighbour(L, u, [&](int64_t w) {
                if (!precedes(rank[w], w, pu, u)) return true;
                int32_t cw = ((volatile int32_t*)colour)[w];
                if (cw == -2) return true;
                if (cw == -1) { ready = false; return false; }
                if (cw >= base && cw < base + 64) mask |= 1ull << (cw - base);
                return true;
            });
            if (!ready) break;
            if (mask != ~0ull) {
                colour[u] = base + __ffsll((long long)~mask) - 1;
                done = true;
            } else {
                base += 64;
            }
        }
        if (!done) left++;
    }
    for (int o = 16; o; o >>= 1) left += __shfl_xor_sync(0xffffffffu, left, o);
    if ((threadIdx.x & 31) == 0 && left) atomicAdd(remaining, left);
}

// the same round for the long units (a list), one warp per unit: the lanes scan the
// unit's entries strided, the warp combines "every higher-priority neighbour is
// coloured" and the used colours of each 64-colour window
__global__ void k_jp_round_long(DevLP L, const int32_t* __restrict__ units, int64_t n_units,
                                const uint64_t* __restrict__ rank, int32_t* colour, unsigned long long* remaining) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = w0; q < n_units; q += nw) {
        const int64_t u = units[q];
        if (colour[u] != -1) continue;
        const uint64_t pu = rank[u];
        int64_t first, cnt;
        if (u < L.n_blocks) { first = u * L.k; cnt = L.k; }
        else { first = L.n_blocks * L.k + (u - L.n_blocks); cnt = 1; }
        int32_t base = 0;
        bool done = false, ready = true;
        while (!done && ready) {
            unsigned long long mask = 0;
            bool lane_ready = true;
            for (int64_t j = first; j < first + cnt && lane_ready; j++)
                for (int64_t t = L.colptr[j] + lane; t < L.colptr[j + 1] && lane_ready; t += 32) {
                    const int64_t i = (int64_t)((uint32_t)L.rowidx[t] & kRowMask);
                    auto visit = [&](int64_t w) {
                        if (w == u || !precedes(rank[w], w, pu, u)) return;
                        const int32_t cw = ((volatile int32_t*)colour)[w];
                        if (cw == -2) return;
                        if (cw == -1) { lane_ready = false; return; }
                        if (cw >= base && cw < base + 64) mask |= 1ull << (cw - base);
                    };
                    if (L.problem == THETIS_PROB_VC || L.problem == THETIS_PROB_MIS) {
                        const int2 e = L.edges[i];
                        visit(e.x == (int32_t)u ? e.y : e.x);
                    } else if (L.problem == THETIS_PROB_MWC) {
                        const int64_t k = L.k, e = i / (2 * k), l = (i >> 1) % k;
                        const int2 uv = L.edges[e];
                        visit((int64_t)uv.x);
                        visit((int64_t)uv.y);
                        visit(L.n_blocks + e * k + l);
                    } else {
                        for (int64_t p = L.rowptr[i]; p < L.rowptr[i + 1]; p++) visit(unit_of_col(L, L.rcol[p]));
                    }
                }
            ready = __all_sync(0xffffffffu, lane_ready);
            if (!ready) break;
            const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)mask);
            const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(mask >> 32));
            const unsigned long long m = ((unsigned long long)hi << 32) | lo;
            if (m != ~0ull) {
                if (lane == 0) colour[u] = base + __ffsll((long long)~m) - 1;
                done = true;
            } else {
                base += 64;
            }
        }
        if (!done && lane == 0) atomicAdd(remaining, 1ull);
    }
}
// the long units (unordered list)
__global__ void k_long_units(DevLP L, int64_t S, int32_t* units, unsigned long long* count) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x)
        if (unit_nnz(L, u) > kLongUnit) units[atomicAdd(count, 1ull)] = (int32_t)u;
}

__global__ void k_colour_max(int64_t S, const int32_t* colour, int32_t* out) {
    int32_t best = -1;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x)
        best = colour[u] > best ? colour[u] : best;
    for (int o = 16; o; o >>= 1) {
        int32_t x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

__global__ void k_class_keys(int64_t S, int32_t K, const int32_t* colour, int32_t* keys, int32_t* ids) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < S; u += (int64_t)gridDim.x * blockDim.x) {
        keys[u] = colour[u] >= 0 ? colour[u] : K; // fixed units sort last, dropped
        ids[u] = (int32_t)u;
    }
}
__global__ void k_class_bounds(int64_t S, const int32_t* keys, int32_t* start, int32_t* end) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < S; p += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = keys[p];
        if (p == 0 || keys[p - 1] != c) start[c] = (int32_t)p;
        if (p == S - 1 || keys[p + 1] != c) end[c] = (int32_t)(p + 1);
    }
}

}  // namespace

int ensure_colouring(thetis_lp* lp, uint64_t seed) {
    if (lp->colour_valid && lp->colour_seed == seed) return THETIS_OK;
    const DevLP& L = lp->d;
    cudaStream_t s = lp->stream;
    const int64_t S = L.n_blocks + L.n_scalar;
    const uint32_t key = fmix32((uint32_t)seed) ^ (uint32_t)(seed >> 32);
    lp->colour_valid = false;
    lp->class_ptr.clear();
    int32_t K = 0;
    if (S > 0) {
        unsigned long long* remaining = (unsigned long long*)(lp->flags + 32);
        uint64_t* rank = (uint64_t*)lp->temp;
        if ((size_t)S * 8 > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "colouring ranks");
        k_colour_rank<<<grid_for(S, T), T, 0, s>>>(L, S, key, rank);
        k_colour_init<<<grid_for(S, T), T, 0, s>>>(L, S, lp->colour);
        int32_t* long_units = (int32_t*)(rank + S);
        unsigned long long n_long = 0;
        if ((size_t)S * 12 > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "colouring ranks");
        {
            unsigned long long* cnt = (unsigned long long*)(lp->flags + 34);
            CUDA_TRY(lp, cudaMemsetAsync(cnt, 0, 8, s));
            k_long_units<<<grid_for(S, T), T, 0, s>>>(L, S, long_units, cnt);
            CUDA_TRY(lp, cudaMemcpyAsync(&n_long, cnt, 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(lp, cudaStreamSynchronize(s));
        }
        for (int round = 0;; round++) {
            CUDA_TRY(lp, cudaMemsetAsync(remaining, 0, 8, s));
            k_jp_round<<<grid_for(S, T), T, 0, s>>>(L, S, rank, lp->colour, remaining);
            if (n_long > 0)
                k_jp_round_long<<<grid_for(32 * (int64_t)n_long, T), T, 0, s>>>(L, long_units, (int64_t)n_long, rank,
                                                                               lp->colour, remaining);
            unsigned long long left = 0;
            CUDA_TRY(lp, cudaMemcpyAsync(&left, remaining, 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(lp, cudaStreamSynchronize(s));
            if (left == 0) break;
            if (round > 1000000) return set_error(lp, THETIS_ERR_CUDA, "colouring did not terminate");
        }
        int32_t* kmax = lp->flags + 40;
        CUDA_TRY(lp, cudaMemsetAsync(kmax, 0xFF, 4, s));
        k_colour_max<<<grid_for(S, T), T, 0, s>>>(S, lp->colour, kmax);
        int32_t mx = -1;
        CUDA_TRY(lp, cudaMemcpyAsync(&mx, kmax, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        K = mx + 1;
        // class lists: stable sort of (colour, id) -> members ascending within class
        Carver C(lp->temp);
        int32_t* keys = C.take<int32_t>(S);
        int32_t* ids = C.take<int32_t>(S);
        int32_t* keys_out = C.take<int32_t>(S);
        int32_t* start = C.take<int32_t>(K + 2);
        int32_t* end = C.take<int32_t>(K + 2);
        size_t cb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, cb, keys, keys_out, ids, lp->members, S, 0, 32);
        void* cubp = C.take<char>((int64_t)cb);
        if (C.off > lp->temp_bytes) return set_error(lp, THETIS_ERR_WORKSPACE_TOO_SMALL, "colouring temp");
        k_class_keys<<<grid_for(S, T), T, 0, s>>>(S, K, lp->colour, keys, ids);
        int bits = 1;
        while (bits < 31 && ((int64_t)1 << bits) <= K) bits++;
        CUDA_TRY(lp, cub::DeviceRadixSort::SortPairs(cubp, cb, keys, keys_out, ids, lp->members, S, 0, bits, s));
        CUDA_TRY(lp, cudaMemsetAsync(start, 0, (size_t)(K + 2) * 4, s));
        CUDA_TRY(lp, cudaMemsetAsync(end, 0, (size_t)(K + 2) * 4, s));
        k_class_bounds<<<grid_for(S, T), T, 0, s>>>(S, keys_out, start, end);
        std::vector<int32_t> hs(K + 2), he(K + 2);
        CUDA_TRY(lp, cudaMemcpyAsync(hs.data(), start, (size_t)(K + 2) * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaMemcpyAsync(he.data(), end, (size_t)(K + 2) * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(lp, cudaStreamSynchronize(s));
        lp->class_ptr.resize(K + 1);
        lp->class_ptr[0] = 0;
        for (int32_t c = 0; c < K; c++) lp->class_ptr[c + 1] = he[c];
    } else {
        lp->class_ptr.assign(1, 0);
    }
    lp->K = K;
    lp->colour_seed = seed;
    lp->colour_valid = true;
    return check_cuda(lp, "colouring");
}

}  // namespace thetis
