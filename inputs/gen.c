/*
 * Seeded synthetic input generators (host side) shared by the CUDA path's
 * tests/bench and by the oracle.  This file holds NONE of the method's
 * arithmetic: it only produces raw graph edge lists (possibly with self-loops
 * and duplicates, in the orientation drawn), vertex / edge weights and
 * terminal sets.  Canonicalisation, dedup and LP construction are the
 * method's work and are done separately by oracle/ and by the CUDA library.
 *
 * Recipes: SURVEY.md §8(d) "Concrete synthetic inputs"; DESIGN.md §Inputs.
 *
 * Counter-based randomness: draw(seed, i) is the (i+1)-th output of the
 * SplitMix64 generator seeded with `seed` (Steele, Lea, Flood 2014):
 *     state_i = seed + (i+1)*0x9E3779B97F4A7C15,  out = mix(state_i).
 * inputs/gen_cuda.cu implements the same function on the device for the
 * large bench inputs; tests/test_inputs.py (its GPU test) checks the two agree.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t sm64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t draw(uint64_t seed, uint64_t i) {
    return sm64_mix(seed + (i + 1) * GOLDEN);
}

/* uniform integer in [0, n) from 32 random bits (multiply-shift) */
static inline int64_t below(uint32_t x, int64_t n) {
    return (int64_t)(((uint64_t)x * (uint64_t)n) >> 32);
}

uint64_t inputs_draw(uint64_t seed, uint64_t i) { return draw(seed, i); }

/* ---------- Erdos-Renyi G(n, m), exact m, rejection of loops/duplicates --- */
/* Attempt c uses draw(seed, c): u = hi32 scaled to n, v = lo32 scaled to n.
 * Accepted pairs are written in the orientation drawn. Returns attempts used
 * (>= m), or -1 on bad arguments / allocation failure. */
int64_t inputs_er(int64_t n, int64_t m, uint64_t seed, int32_t* src, int32_t* dst) {
    if (n < 2 || m < 0 || m > n * (n - 1) / 2) return -1;
    uint64_t cap = 16;
    while (cap < (uint64_t)(4 * m + 16)) cap <<= 1;
    uint64_t* table = (uint64_t*)malloc(cap * sizeof(uint64_t));
    if (!table) return -1;
    memset(table, 0xff, cap * sizeof(uint64_t)); /* empty = all ones */
    int64_t got = 0;
    uint64_t c = 0;
    while (got < m) {
        uint64_t h = draw(seed, c++);
        int64_t u = below((uint32_t)(h >> 32), n);
        int64_t v = below((uint32_t)h, n);
        if (u == v) continue;
        uint64_t lo = (uint64_t)(u < v ? u : v), hi = (uint64_t)(u < v ? v : u);
        uint64_t key = (lo << 32) | hi;
        uint64_t slot = sm64_mix(key) & (cap - 1);
        int dup = 0;
        while (table[slot] != ~0ULL) {
            if (table[slot] == key) { dup = 1; break; }
            slot = (slot + 1) & (cap - 1);
        }
        if (dup) continue;
        table[slot] = key;
        src[got] = (int32_t)u;
        dst[got] = (int32_t)v;
        got++;
    }
    free(table);
    return (int64_t)c;
}

/* ---------- Chung-Lu power law ------------------------------------------- */
/* w_i = (i+1)^(-1/(gamma-1)), i = 0..n-1; every one of `samples` edges draws
 * both endpoints independently with probability proportional to w (inverse
 * CDF on the prefix sums, upper_bound).  Sample s uses draw(seed, 2s) for the
 * first endpoint and draw(seed, 2s+1) for the second.  Self-loops and
 * duplicates are kept (the LP builder drops them). */
int inputs_chung_lu(int64_t n, double gamma, int64_t samples, uint64_t seed,
                    int32_t* src, int32_t* dst) {
    if (n < 1 || gamma <= 1.0 || samples < 0) return -1;
    double* cum = (double*)malloc((size_t)n * sizeof(double));
    if (!cum) return -1;
    double acc = 0.0, ex = -1.0 / (gamma - 1.0);
    for (int64_t i = 0; i < n; i++) {
        acc += pow((double)(i + 1), ex);
        cum[i] = acc;
    }
    const double total = acc;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < samples; s++) {
        for (int e = 0; e < 2; e++) {
            double u = (double)(draw(seed, 2 * (uint64_t)s + (uint64_t)e) >> 11) * 0x1p-53 * total;
            int64_t lo = 0, hi = n - 1; /* first i with cum[i] > u */
            while (lo < hi) {
                int64_t mid = lo + (hi - lo) / 2;
                if (cum[mid] > u) hi = mid; else lo = mid + 1;
            }
            if (e == 0) src[s] = (int32_t)lo; else dst[s] = (int32_t)lo;
        }
    }
    free(cum);
    return 0;
}

/* ---------- 4-neighbour grid --------------------------------------------- */
/* id = row*side + col; for v ascending: (v, v+1) if col < side-1, then
 * (v, v+side) if row < side-1.  Returns the number of edges 2*side*(side-1). */
int64_t inputs_grid(int64_t side, int32_t* src, int32_t* dst) {
    int64_t e = 0;
    for (int64_t r = 0; r < side; r++)
        for (int64_t c = 0; c < side; c++) {
            int64_t v = r * side + c;
            if (c + 1 < side) { src[e] = (int32_t)v; dst[e] = (int32_t)(v + 1); e++; }
            if (r + 1 < side) { src[e] = (int32_t)v; dst[e] = (int32_t)(v + side); e++; }
        }
    return e;
}

/* ---------- R-MAT --------------------------------------------------------- */
/* Sample s, level t (t = 0 is the most significant bit): x = 32 random bits,
 * the hi half of draw(seed, 16*s + t/2) for even t, the lo half for odd t.
 * Quadrant: x < ta -> (0,0); x < tab -> (0,1); x < tabc -> (1,0); else (1,1)
 * (src bit, dst bit); thresholds are floor(p * 2^32) computed by the caller.
 * No noise, no relabelling; loops and duplicates kept. */
int inputs_rmat(int scale, int64_t samples, uint32_t ta, uint32_t tab, uint32_t tabc,
                uint64_t seed, int32_t* src, int32_t* dst) {
    if (scale < 1 || scale > 31 || samples < 0) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < samples; s++) {
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
    return 0;
}

/* ---------- weights ------------------------------------------------------- */
/* U[1,10): w_i = fp32(1 + 9*u), u = (draw(seed,i) >> 40) * 2^-24 (exact in fp64,
 * single rounding to fp32). */
void inputs_uniform_weights(int64_t n, uint64_t seed, float* w) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        w[i] = (float)(1.0 + 9.0 * ((double)(draw(seed, (uint64_t)i) >> 40) * 0x1p-24));
}

/* Exp(1): w_i = fp32(-ln(1-u)), u = (draw(seed,i) >> 11) * 2^-53, fp64 math. */
void inputs_exp_weights(int64_t n, uint64_t seed, float* w) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double u = (double)(draw(seed, (uint64_t)i) >> 11) * 0x1p-53;
        w[i] = (float)(-log(1.0 - u));
    }
}

/* ---------- terminals ----------------------------------------------------- */
/* `count` distinct vertex ids: attempt c -> id = hi32(draw(seed,c)) scaled to n,
 * rejected if already chosen.  Label l owns ids [l*t, (l+1)*t). */
int inputs_terminals(int64_t n, int64_t count, uint64_t seed, int32_t* out) {
    if (count > n) return -1;
    int64_t got = 0;
    uint64_t c = 0;
    while (got < count) {
        int32_t id = (int32_t)below((uint32_t)(draw(seed, c++) >> 32), n);
        int dup = 0;
        for (int64_t j = 0; j < got; j++)
            if (out[j] == id) { dup = 1; break; }
        if (!dup) out[got++] = id;
    }
    return 0;
}
