// Device twin of inputs/gen.c for the inputs too large to generate on the
// host inside a bench run (R-MAT scale 26: 1.07e9 edges).  Same counter-based
// definitions, bit for bit (tests/test_inputs.py::test_device_twin_matches_host checks
// it against the host generator).  Holds none of the method's arithmetic.
#include <cstdint>
#include <cuda_runtime.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

__device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t i) {
    return sm64_mix(seed + (i + 1) * GOLDEN);
}

__global__ void rmat_kernel(int scale, int64_t samples, uint32_t ta, uint32_t tab, uint32_t tabc,
                            uint64_t seed, int32_t* __restrict__ src, int32_t* __restrict__ dst) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < samples;
         s += (int64_t)gridDim.x * blockDim.x) {
        uint32_t a = 0, b = 0;
        uint64_t h = 0;
        for (int t = 0; t < scale; t++) {
            if ((t & 1) == 0) h = draw(seed, 16 * (uint64_t)s + (uint64_t)(t >> 1));
            uint32_t x = (t & 1) ? (uint32_t)h : (uint32_t)(h >> 32);
            uint32_t sb, db;
            if (x < ta) { sb = 0; db = 0; }
            else if (x < tab) { sb = 0; db = 1; }
            else if (x < tabc) { sb = 1; db = 0; }
            else { sb = 1; db = 1; }
            a = (a << 1) | sb;
            b = (b << 1) | db;
        }
        src[s] = (int32_t)a;
        dst[s] = (int32_t)b;
    }
}

__global__ void uniform_weights_kernel(int64_t n, uint64_t seed, float* __restrict__ w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        w[i] = (float)(1.0 + 9.0 * ((double)(draw(seed, (uint64_t)i) >> 40) * 0x1p-24));
}

extern "C" int inputs_rmat_device(int scale, int64_t samples, uint32_t ta, uint32_t tab,
                                  uint32_t tabc, uint64_t seed, int32_t* src, int32_t* dst,
                                  void* stream) {
    if (scale < 1 || scale > 31 || samples < 0) return -1;
    if (samples == 0) return 0;
    rmat_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(scale, samples, ta, tab, tabc, seed, src, dst);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int inputs_uniform_weights_device(int64_t n, uint64_t seed, float* w, void* stream) {
    if (n <= 0) return 0;
    uniform_weights_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(n, seed, w);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
