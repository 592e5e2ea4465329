// microbenchmark: random fp32 / fp64 RED into an L2-resident array (22 MB, 48 MB: the hot set of
// the column-sum async form); coalesced streaming read.  Reference rates for the RED sector
// counts in profiles/*ncu*: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench_l2_red.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_red(float* acc, int64_t n_acc, int64_t ops, uint64_t seed, int per_thread) {
    int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < ops; i += nt) {
        uint64_t h = (i + seed) * 0x9E3779B97F4A7C15ULL; h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ULL; h ^= h >> 32;
        atomicAdd(acc + (h % n_acc), 1.0f);
    }
}
__global__ void k_red64(double* acc, int64_t n_acc, int64_t ops, uint64_t seed) {
    int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < ops; i += nt) {
        uint64_t h = (i + seed) * 0x9E3779B97F4A7C15ULL; h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ULL; h ^= h >> 32;
        atomicAdd(acc + (h % n_acc), 1.0);
    }
}
// random 4-byte reads (ld.global.cg: L2 only) of an L2-resident array, eight in flight per thread
__global__ void k_read(const float* acc, int64_t n_acc, int64_t ops, uint64_t seed, float* out) {
    int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    float s = 0;
    for (int64_t i = tid; i < ops; i += 8 * nt) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            uint64_t h = (i + q * nt + seed) * 0x9E3779B97F4A7C15ULL; h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ULL; h ^= h >> 32;
            asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v[q]) : "l"(acc + (h % n_acc)));
        }
#pragma unroll
        for (int q = 0; q < 8; q++) s += v[q];
    }
    if (s == 12345.f) *out = s;
}
__global__ void k_stream(const float4* a, int64_t n, float* out) {
    float s = 0; int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < n; i += nt) { float4 v = a[i]; s += v.x + v.y + v.z + v.w; }
    if (s == 12345.f) *out = s;
}
int main() {
    int64_t n_acc = 22LL << 20 >> 2;  // 22 MB of floats
    float* acc; cudaMalloc(&acc, n_acc * 4); cudaMemset(acc, 0, n_acc * 4);
    int64_t big = 4LL << 30; float* a; cudaMalloc(&a, big); cudaMemset(a, 0, big);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int64_t ops = 1LL << 30;
    for (int it = 0; it < 3; it++) {
        for (int blocks : {148 * 8, 148 * 32}) {
            cudaEventRecord(e0); k_red<<<blocks, 256>>>(acc, n_acc, ops, it, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("red random 22MB: blocks %d  %.2f ms  %.1f G/s\n", blocks, ms, ops / ms / 1e6);
        }
        for (int64_t mb : {22, 48}) {
            const int64_t n64 = (mb << 20) >> 3;
            double* acc64; cudaMalloc(&acc64, n64 * 8); cudaMemset(acc64, 0, n64 * 8);
            cudaEventRecord(e0); k_red64<<<148 * 32, 256>>>(acc64, n64, ops, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms64; cudaEventElapsedTime(&ms64, e0, e1);
            printf("red.f64 random %lld MB: blocks %d  %.2f ms  %.1f G/s\n", (long long)mb, 148 * 32, ms64, ops / ms64 / 1e6);
            cudaFree(acc64);
        }
        for (int64_t mb : {22, 48}) {
            const int64_t nr = (mb << 20) >> 2;
            float* accr; cudaMalloc(&accr, nr * 4); cudaMemset(accr, 0, nr * 4);
            k_read<<<148 * 32, 256>>>(accr, nr, ops / 8, 99, acc);  // warm the L2
            cudaEventRecord(e0); k_read<<<148 * 32, 256>>>(accr, nr, ops, it, acc); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float msr; cudaEventElapsedTime(&msr, e0, e1);
            printf("ld.cg.f32 random %lld MB: blocks %d  %.2f ms  %.1f G/s\n", (long long)mb, 148 * 32, msr, ops / msr / 1e6);
            cudaFree(accr);
        }
        cudaEventRecord(e0); k_stream<<<148 * 8, 256>>>((float4*)a, big / 16, acc); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("stream read 4 GB: %.2f ms %.0f GB/s\n", ms, big / ms / 1e6);
    }
    return 0;
}
