// microbenchmark (experiments only): CUB onesweep tunings for the builder's sorts on B200
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>

template <int THREADS, int ITEMS, typename K, typename V, typename Off, int RB = 8>
struct Hub {
    using Base = cub::detail::radix::policy_hub<K, V, Off>;
    using P9 = typename Base::Policy900;
    struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, P9> {
        static constexpr bool ONESWEEP = true;
        static constexpr int ONESWEEP_RADIX_BITS = RB;
        using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, K, RB>;
        using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, RB>;
        using OnesweepPolicy = cub::AgentRadixSortOnesweepPolicy<THREADS, ITEMS, K, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                                                 cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, RB>;
        using ScanPolicy = typename P9::ScanPolicy;
        using DownsweepPolicy = typename P9::DownsweepPolicy;
        using AltDownsweepPolicy = typename P9::AltDownsweepPolicy;
        using UpsweepPolicy = typename P9::UpsweepPolicy;
        using AltUpsweepPolicy = typename P9::AltUpsweepPolicy;
        using SingleTilePolicy = typename P9::SingleTilePolicy;
        using SegmentedPolicy = typename P9::SegmentedPolicy;
        using AltSegmentedPolicy = typename P9::AltSegmentedPolicy;
    };
    using MaxPolicy = Policy1000;
};

__global__ void fill(int32_t* k, int32_t* v, int64_t n, int bits) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull; h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
        k[i] = (int32_t)(h & ((1u << bits) - 1)); v[i] = (int32_t)i;
    }
}

template <int TH, int IT, typename Off>
void run_pairs(const char* name, int32_t* k0, int32_t* k1, int32_t* v0, int32_t* v1, int64_t n, int bits, void* tmp, size_t tmpb) {
    cub::DoubleBuffer<int32_t> dk(k0, k1), dv(v0, v1);
    size_t b = 0;
    using D = cub::DispatchRadixSort<false, int32_t, int32_t, Off, Hub<TH, IT, int32_t, int32_t, Off>>;
    D::Dispatch(nullptr, b, dk, dv, (Off)n, 0, bits, true, 0);
    if (b > tmpb) { printf("%s: temp %zu too big\n", name, b); return; }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        fill<<<148 * 8, 256>>>(k0, v0, n, bits);
        dk = cub::DoubleBuffer<int32_t>(k0, k1); dv = cub::DoubleBuffer<int32_t>(v0, v1);
        cudaEventRecord(e0);
        D::Dispatch(tmp, b, dk, dv, (Off)n, 0, bits, true, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("pairs %-28s %8.2f ms  (%s)\n", name, best, cudaGetErrorString(cudaGetLastError()));
}
void run_stock(int32_t* k0, int32_t* k1, int32_t* v0, int32_t* v1, int64_t n, int bits, void* tmp, size_t tmpb) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        fill<<<148 * 8, 256>>>(k0, v0, n, bits);
        cub::DoubleBuffer<int32_t> dk(k0, k1), dv(v0, v1);
        size_t b = tmpb;
        cudaEventRecord(e0);
        cub::DeviceRadixSort::SortPairs(tmp, b, dk, dv, n, 0, bits, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("pairs %-28s %8.2f ms\n", "stock int64 n", best);
}

__global__ void fill64(uint64_t* k, int64_t n, int bits) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull; h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
        k[i] = h & ((1ull << bits) - 1);
    }
}
template <int TH, int IT, typename Off, int RB = 8>
void run_keys(const char* name, uint64_t* k0, uint64_t* k1, int64_t n, int bits, void* tmp, size_t tmpb) {
    cub::DoubleBuffer<uint64_t> dk(k0, k1);
    cub::DoubleBuffer<cub::NullType> none;
    size_t b = 0;
    using D = cub::DispatchRadixSort<false, uint64_t, cub::NullType, Off, Hub<TH, IT, uint64_t, cub::NullType, Off, RB>>;
    D::Dispatch(nullptr, b, dk, none, (Off)n, 0, bits, true, 0);
    if (b > tmpb) { printf("%s: temp %zu too big\n", name, b); return; }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        fill64<<<148 * 8, 256>>>(k0, n, bits);
        dk = cub::DoubleBuffer<uint64_t>(k0, k1);
        cudaEventRecord(e0);
        D::Dispatch(tmp, b, dk, none, (Off)n, 0, bits, true, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("keys64 %-27s %8.2f ms  (%s)\n", name, best, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int64_t n = 1051915249;
    const int bits = 26;
    int32_t *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    size_t tmpb = (size_t)2 << 30; void* tmp; cudaMalloc(&tmp, tmpb);
    run_stock(k0, k1, v0, v1, n, bits, tmp, tmpb);
    cudaFree(v0); cudaFree(v1); cudaFree(k0); cudaFree(k1);
    const int64_t E = 1073741824;
    uint64_t *q0, *q1;
    cudaMalloc(&q0, E * 8); cudaMalloc(&q1, E * 8);
    run_keys<256, 32, unsigned long long>("256x32 off64 (current)", q0, q1, E, 52, tmp, tmpb);
    run_keys<256, 32, uint32_t>("256x32 off32", q0, q1, E, 52, tmp, tmpb);
    run_keys<256, 32, unsigned long long, 9>("256x32 rb9", q0, q1, E, 52, tmp, tmpb);
    run_keys<256, 32, unsigned long long, 10>("256x32 rb10", q0, q1, E, 52, tmp, tmpb);
    return 0;
}
