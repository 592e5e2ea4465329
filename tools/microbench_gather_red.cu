// microbenchmark: a warp gathers 8 random fp32 of a 4 GB array per lane, then adds to the
// same 8 addresses -- do the adds find the gathered lines in L2?  Variants of the gather
// load (cache operator) and of the add (red vs atom).  Read with ncu:
//   lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum / lts__t_sectors_srcunit_tex_op_red.sum
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t h) {
    h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ULL; h ^= h >> 32; return h;
}
template <int LD, int ADD>
__global__ void k_gather_add(float* r, int64_t n, int64_t per_thread, uint64_t seed) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t it = 0; it < per_thread; it += 8) {
        int64_t idx[8];
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) idx[q] = (int64_t)(mix((tid * per_thread + it + q) * 0x9E3779B97F4A7C15ULL + seed) % (uint64_t)n);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (LD == 0) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v[q]) : "l"(r + idx[q]));
            else if (LD == 1) v[q] = r[idx[q]];
            else if (LD == 2) asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v[q]) : "l"(r + idx[q]));
            else v[q] = atomicAdd(r + idx[q], 0.0f);  // LD == 3: the gather as an atomic
        }
        float d = 0.f;
#pragma unroll
        for (int q = 0; q < 8; q++) d += v[q];
        d = d * 1e-30f + 1e-7f;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (ADD == 0) asm volatile("red.global.add.f32 [%0], %1;" ::"l"(r + idx[q]), "f"(d) : "memory");
            else if (ADD == 1) atomicAdd(r + idx[q], d);
            else r[idx[q]] = v[q] + d;  // ADD == 2: plain store (not Hogwild-safe; cache behaviour only)
        }
    }
}
int main() {
    const int64_t n = 1LL << 30;  // 4 GB of floats
    float* r;
    cudaMalloc(&r, n * 4);
    cudaMemset(r, 0, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256;
    const int64_t per = 256;
    const double ops = (double)blocks * threads * per;
    auto run = [&](const char* name, void (*k)(float*, int64_t, int64_t, uint64_t)) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            k<<<blocks, threads>>>(r, n, per, rep);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%-22s %.3f ms  %.2f G gathers+adds/s\n", name, ms, ops / ms / 1e6);
        }
    };
    run("ld.cg + red", k_gather_add<0, 0>);
    run("ld (ca) + red", k_gather_add<1, 0>);
    run("ld.relaxed.gpu + red", k_gather_add<2, 0>);
    run("ld.cg + atom", k_gather_add<0, 1>);
    run("atom(+0) + red", k_gather_add<3, 0>);
    run("ld.cg + st", k_gather_add<0, 2>);
    return 0;
}
