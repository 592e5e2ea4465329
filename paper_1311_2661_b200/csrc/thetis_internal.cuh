// Internal declarations of libthetis (product side; shares nothing with oracle/).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "thetis.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX 3: no-ops unless a profiler is attached

namespace thetis {

constexpr int kTile = 32;          // units per async tile (R-6)
constexpr int kRowRangeShift = 14; // graph LP rows grouped by min endpoint >> 14 (R-17)
constexpr int kRowRange = 1 << kRowRangeShift;
constexpr int64_t kHeavy = 512;    // a tile whose scalar columns hold more nonzeros is a hub tile (R-6, R-17)
constexpr int kMaxK = 32;          // max simplex block size
constexpr uint32_t kSignBit = 0x80000000u;
constexpr uint32_t kRowMask = 0x7FFFFFFFu;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr int kRedBlocks = 1184;   // fixed reduction grid (8 x 148 SMs): deterministic partials
constexpr int kRedThreads = 256;

// ---------------------------------------------------------------------------
// Device view of one LP in standard form (z = (x, s), r = A z - b).
// ---------------------------------------------------------------------------
struct DevLP {
    int problem, obj_sense, k;
    int64_t m, n_s, n_ineq, N, nnz_s, U, n_blocks, n_scalar, n_vert, m_edges;
    int64_t m_hub_rows;        // VC / MIS: rows [0, m_hub_rows) have a hub max endpoint (R-17), ranged by u
    int64_t m_defer_rows;      // rows [m_hub_rows, m_defer_rows) have a hub min endpoint only, ranged
                               // by v; rows [0, m_defer_rows) belong to the row pass, light steps reach
                               // them through it (R-6)
    // A, structural part: CSC, rows ascending.  val == nullptr: coefficient
    // +1, or -1 when bit 31 of rowidx is set.
    const int64_t* colptr;
    const int32_t* rowidx;
    const float* val;
    const double* colnorm2;    // ||a_j||^2 (generic with values), else nullptr (= nnz_j)
    // rows: generic CSR, or implicit from the unique edge list (graph LPs)
    const int64_t* rowptr;
    const int32_t* rcol;
    const float* rval;
    const int2* edges;         // unique canonical edges (u < v), row order
    const float* b;            // generic only
    const int8_t* sense;       // generic only
    const int64_t* row_slack;  // generic only: slack column of row i or -1
    const int32_t* slack_row;  // generic only: row of slack q
    const float* c;            // cost as given (original sense), n_s
    float c_sign;              // +1 MIN, -1 MAX
    const float* lo;           // generic only (nullptr: [0, 1])
    const float* hi;
    const uint8_t* unit_fixed; // per structural unit, or nullptr (none fixed)
    const float* ew;           // MWC edge weights (unique edges)
    const int32_t* term_label; // MWC terminal label per vertex or -1
    float* z;
    float* r;
    const float* zbar;         // anchors (caller-owned) or nullptr
    const float* ubar;
    float* ua;                 // ubar^T a_j per structural column
};

// ---- small device helpers ------------------------------------------------
__device__ __forceinline__ bool graph_rows(const DevLP& L) { return L.problem != THETIS_PROB_GENERIC; }

__device__ __forceinline__ float row_b(const DevLP& L, int64_t i) {
    if (L.problem == THETIS_PROB_GENERIC) return L.b[i];
    return L.problem == THETIS_PROB_MWC ? 0.0f : 1.0f;
}
// slack coefficient of inequality row i: -1 (GE) / +1 (LE)
__device__ __forceinline__ float row_sigma(const DevLP& L, int64_t i) {
    int s = L.problem == THETIS_PROB_GENERIC ? L.sense[i]
                                             : (L.problem == THETIS_PROB_MIS ? THETIS_LE : THETIS_GE);
    return s == THETIS_GE ? -1.0f : 1.0f;
}
__device__ __forceinline__ int row_sense(const DevLP& L, int64_t i) {
    if (L.problem == THETIS_PROB_GENERIC) return L.sense[i];
    return L.problem == THETIS_PROB_MIS ? THETIS_LE : THETIS_GE;
}
__device__ __forceinline__ int64_t slack_row_of(const DevLP& L, int64_t q) {
    return L.problem == THETIS_PROB_GENERIC ? (int64_t)L.slack_row[q] : q;
}
__device__ __forceinline__ int64_t row_slack_of(const DevLP& L, int64_t i) {
    return L.problem == THETIS_PROB_GENERIC ? L.row_slack[i] : L.n_s + i;
}
__device__ __forceinline__ float col_lo(const DevLP& L, int64_t j) { return L.lo ? L.lo[j] : 0.0f; }
__device__ __forceinline__ float col_hi(const DevLP& L, int64_t j) { return L.hi ? L.hi[j] : 1.0f; }
__device__ __forceinline__ float c_int(const DevLP& L, int64_t j) { return L.c_sign * L.c[j]; }

// decode one CSC entry
__device__ __forceinline__ void entry(const DevLP& L, int64_t t, int64_t& row, float& a) {
    uint32_t raw = (uint32_t)L.rowidx[t];
    row = (int64_t)(raw & kRowMask);
    a = L.val ? L.val[t] : ((raw & kSignBit) ? -1.0f : 1.0f);
}

// ---- the column dot a_j^T v of the deterministic arithmetic contract (R-7,
// SURVEY §8(c).4, widened to kDotLanes lanes in round 2): virtual lane l in [0, 2^17) sums
// the column's entries at positions t = l, l + 2^17, ... (CSC order) from +0, each product
// rounded on its own; then p[l] += p[l + off] for l < off, off = 2^16, ..., 1; the dot is
// p[0].  Lanes past the column hold +0 and adding +0 changes no lane value, so every
// evaluation below skips them and gives the same bits.  (Columns of <= 2048 entries give
// the bits of round 1's 1024-lane contract.)
constexpr int kDotLgLanes = 17;
constexpr int64_t kDotLanes = (int64_t)1 << kDotLgLanes;
__device__ __forceinline__ float dot_term(const DevLP& L, int64_t t, const float* v) {
    int64_t row;
    float a;
    entry(L, t, row, a);
    const float x = v[row];
    return L.val ? __fmul_rn(a, x) : (a < 0.0f ? -x : x);
}
// the value of virtual lane l: its entries l, l + 2^17, ... summed in order from +0
__device__ __forceinline__ float dot_lane(const DevLP& L, int64_t cb, int64_t len, int64_t l, const float* v) {
    float x = 0.0f;
    for (int64_t t = l; t < len; t += kDotLanes) x = __fadd_rn(x, dot_term(L, cb + t, v));
    return x;
}
// one thread, columns of at most W entries (registers)
template <int W>
__device__ __forceinline__ float col_dot_tree_small(const DevLP& L, int64_t cb, int64_t len, const float* v) {
    float p[W];
#pragma unroll
    for (int i = 0; i < W; i++) p[i] = i < len ? __fadd_rn(0.0f, dot_term(L, cb + i, v)) : 0.0f;
#pragma unroll
    for (int s = W / 2; s >= 1; s >>= 1)
#pragma unroll
        for (int i = 0; i < s; i++) p[i] = __fadd_rn(p[i], p[i + s]);
    return p[0];
}
__device__ __forceinline__ float col_dot_tree16(const DevLP& L, int64_t cb, int64_t len, const float* v) {
    if (len <= 4) return col_dot_tree_small<4>(L, cb, len, v);
    if (len <= 8) return col_dot_tree_small<8>(L, cb, len, v);
    if (len <= 16) return col_dot_tree_small<16>(L, cb, len, v);
    return col_dot_tree_small<32>(L, cb, len, v);
}
// partial sums of a halving tree visited in lane bit-reversal order: a stack by level
struct TreeStack {
    float st[20];
    int lv[20], sp = 0;
    __device__ __forceinline__ void push(float x) {
        st[sp] = x;
        lv[sp++] = 0;
        while (sp >= 2 && lv[sp - 1] == lv[sp - 2]) {
            st[sp - 2] = __fadd_rn(st[sp - 2], st[sp - 1]);
            lv[sp - 2]++;
            sp--;
        }
    }
};
// one thread, any column: the lanes in the order the halving combines them (lane
// bit-reversal), partial sums on a stack by level
__device__ __forceinline__ float col_dot_tree_thread(const DevLP& L, int64_t j, const float* v) {
    const int64_t cb = L.colptr[j], len = L.colptr[j + 1] - cb;
    if (len <= 32) return col_dot_tree16(L, cb, len, v);
    int lg = 0;
    while ((1LL << lg) < len && lg < kDotLgLanes) lg++;
    const int64_t P = (int64_t)1 << lg;
    TreeStack ts;
    for (int64_t k = 0; k < P; k++) ts.push(dot_lane(L, cb, len, (int64_t)(__brevll((unsigned long long)k) >> (64 - lg)), v));
    return ts.st[0];
}
// one warp, any column: lane q holds the virtual lanes l = q + 32 i + 1024 k (i < 32,
// k < 128): per i the k's combine first (the tree's offsets 2^16 .. 1024), then the i's
// inside the lane (512 .. 32), then the lanes by shuffles (16 .. 1); returns the dot on
// every lane
__device__ __forceinline__ float col_dot_tree_warp(const DevLP& L, int64_t j, const float* v, int lane) {
    const int64_t cb = L.colptr[j], len = L.colptr[j + 1] - cb;
    const int64_t span = len < kDotLanes ? len : kDotLanes;
    const int K = (int)((span + 1023) / 1024);
    float p[32];
    if (K <= 1) {  // at most 1024 entries: one per lane slot
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const int64_t t = lane + 32 * i;
            p[i] = t < len ? __fadd_rn(0.0f, dot_term(L, cb + t, v)) : 0.0f;
        }
    } else if (K <= 8 && len <= kDotLanes) {  // the k's in registers, a fixed 8-wide halving
#pragma unroll 4
        for (int i = 0; i < 32; i++) {
            float x[8];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const int64_t t = lane + 32 * i + 1024 * k;
                x[k] = t < len ? __fadd_rn(0.0f, dot_term(L, cb + t, v)) : 0.0f;
            }
#pragma unroll
            for (int s = 4; s >= 1; s >>= 1)
#pragma unroll
                for (int k = 0; k < s; k++) x[k] = __fadd_rn(x[k], x[k + s]);
            p[i] = x[0];
        }
    } else {  // long columns (ALM anchors): the k's in bit-reversal order on a stack
        int lgK = 0;
        while ((1 << lgK) < K) lgK++;
        for (int i = 0; i < 32; i++) {
            TreeStack ts;
            for (int kk = 0; kk < (1 << lgK); kk++) {
                const int k = lgK ? (int)(__brev((unsigned)kk) >> (32 - lgK)) : 0;
                ts.push(dot_lane(L, cb, len, lane + 32 * i + 1024 * (int64_t)k, v));
            }
            p[i] = ts.st[0];
        }
    }
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1)  // off = 512 .. 32: within the lane
#pragma unroll
        for (int i = 0; i < s; i++) p[i] = __fadd_rn(p[i], p[i + s]);
    float q = p[0];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {  // off = 16 .. 1: across lanes
        const float o = __shfl_down_sync(0xffffffffu, q, off);
        if (lane < off) q = __fadd_rn(q, o);
    }
    return __shfl_sync(0xffffffffu, q, 0);
}
__device__ __forceinline__ double col_norm2(const DevLP& L, int64_t j) {
    return L.colnorm2 ? L.colnorm2[j] : (double)(L.colptr[j + 1] - L.colptr[j]);
}

// ---- hashing (SplitMix64 finaliser, MurmurHash3 fmix32), Feistel permutation
__host__ __device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6BU;
    h ^= h >> 13;
    h *= 0xC2B2AE35U;
    h ^= h >> 16;
    return h;
}

struct PermKeys {
    uint32_t k[4];
    uint64_t n_tiles;
    int h;
};

inline PermKeys make_perm_keys(int64_t n_tiles, uint64_t seed, int64_t epoch) {
    PermKeys p;
    int B = 0;
    while (((int64_t)1 << B) < n_tiles) B++;
    if (B < 2) B = 2;
    if (B & 1) B++;
    p.h = B / 2;
    uint64_t st = seed ^ (kGolden * (uint64_t)(epoch + 1));
    for (int r = 0; r < 4; r++) p.k[r] = (uint32_t)sm64_mix(st + (uint64_t)(r + 1) * kGolden);
    p.n_tiles = (uint64_t)n_tiles;
    return p;
}

__device__ __forceinline__ uint64_t feistel_round4(uint64_t x, const PermKeys& p) {
    const uint32_t mask = p.h >= 32 ? 0xFFFFFFFFu : ((1u << p.h) - 1u);
    uint32_t L = (uint32_t)(x >> p.h), R = (uint32_t)(x & mask);
#pragma unroll
    for (int r = 0; r < 4; r++) {
        uint32_t F = fmix32(R ^ p.k[r]) & mask;
        uint32_t nl = R, nr = L ^ F;
        L = nl;
        R = nr;
    }
    return ((uint64_t)L << p.h) | R;
}
// pi_e(t) on [0, n_tiles) by cycle-walking
__device__ __forceinline__ uint64_t tile_perm(uint64_t t, const PermKeys& p) {
    uint64_t y = feistel_round4(t, p);
    while (y >= p.n_tiles) y = feistel_round4(y, p);
    return y;
}
// the inverse rounds: (L, R) <- (R ^ F(L, k_r), L) for r = 3 .. 0
__device__ __forceinline__ uint64_t feistel_inv4(uint64_t y, const PermKeys& p) {
    const uint32_t mask = p.h >= 32 ? 0xFFFFFFFFu : ((1u << p.h) - 1u);
    uint32_t L = (uint32_t)(y >> p.h), R = (uint32_t)(y & mask);
#pragma unroll
    for (int r = 3; r >= 0; r--) {
        uint32_t nl = R ^ (fmix32(L ^ p.k[r]) & mask), nr = L;
        L = nl;
        R = nr;
    }
    return ((uint64_t)L << p.h) | R;
}
// pi_e^{-1}(y): the position of tile y in epoch e (cycle-walking the inverse)
__device__ __forceinline__ uint64_t tile_perm_inv(uint64_t y, const PermKeys& p) {
    uint64_t x = feistel_inv4(y, p);
    while (x >= p.n_tiles) x = feistel_inv4(x, p);
    return x;
}

// ---- workspace carving (bump allocator; same code for size query and carve)
struct Carver {
    char* base;
    size_t off = 0;
    explicit Carver(void* b) : base((char*)b) {}
    template <class T>
    T* take(int64_t count) {
        off = (off + 255) & ~(size_t)255;
        T* p = base ? (T*)(base + off) : nullptr;
        off += (size_t)(count > 0 ? count : 1) * sizeof(T);
        return p;
    }
};

// NVTX range over a scope (build, solve, epoch, objective, round; host-side enqueue)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace thetis

// ---------------------------------------------------------------------------
// Host handle
// ---------------------------------------------------------------------------
struct thetis_lp {
    thetis::DevLP d{};
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;   // second stream: hub-hub row pass beside the light tiles
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t det_s[2] = {nullptr, nullptr};  // branches of a captured det class (warp columns, CTA columns)
    cudaEvent_t det_ev[3] = {nullptr, nullptr, nullptr};
    cudaGraphExec_t det_graph = nullptr;  // the last deterministic solve's epoch graph
    std::vector<cudaEvent_t> ev_epoch;
    std::vector<cudaEvent_t> ev_kern;   // per-kernel marks of timed async epochs
    char* ws = nullptr;
    size_t ws_bytes = 0;
    // regions inside ws
    char* temp = nullptr;          // scratch region (build temporaries, colouring, rounding)
    size_t temp_bytes = 0;
    double* red = nullptr;         // reduction partials
    int32_t* flags = nullptr;      // small device flags / counters (64 ints)
    int32_t* colour = nullptr;     // per structural unit
    int32_t* members = nullptr;    // class members, grouped by class
    int32_t* heavy = nullptr;      // heavy async tiles
    // VC / MIS, THETIS_MODE_ASYNC in column-sum form (async_pi.cu, R-23); vertices are
    // addressed by their degree rank (0 = largest degree) so that the hot ones share L2 lines
    int32_t* rank = nullptr;       // rank of vertex u
    int32_t* nbr = nullptr;        // rank of the neighbour of CSC entry t (the other endpoint of its row)
    int2* erank = nullptr;         // ranks of the endpoints of row i
    float* xr = nullptr;           // x by rank (a copy of z[0, n) kept current during the epochs)
    double* Dg = nullptr;          // per-vertex sums by rank kept current during the epochs (S_u = sum sigma s; R-23)
    bool nbr_valid = false;
    double maxnorm2 = 0;           // max_j ||a_j||^2 over all standard-form columns
    int64_t epoch_updates = 0;     // coordinates updated per epoch (stats)
    int64_t epoch_nnz = 0;         // nonzeros processed per epoch (slack = 1)
    // colouring cache
    bool colour_valid = false;
    uint64_t colour_seed = 0;
    int64_t K = 0;
    std::vector<int64_t> class_ptr; // K+2 entries: classes 0..K-1, then slacks
    // heavy tile list (async)
    bool heavy_valid = false;
    int64_t n_heavy = 0;
    int64_t n_hub_chunks = 0;
    bool anchors = false;
    char err[512] = {0};
};

// internal entry points implemented across the .cu files
namespace thetis {
int set_error(thetis_lp* lp, int code, const char* fmt, ...);
int check_cuda(thetis_lp* lp, const char* what);
bool is_device_ptr(const void* p);

// build.cu
int build_graph(thetis_lp* lp, int problem, int64_t n, int64_t n_edges, const int32_t* src,
                const int32_t* dst, const float* vertex_w, const float* edge_w, int k,
                const int32_t* terminals, int t_per_label);
size_t graph_workspace(int problem, int64_t n, int64_t n_edges, int k, bool carve, thetis_lp* lp, void* ws);
size_t generic_workspace(int64_t m, int64_t n, int64_t nnz, bool has_val, bool carve, thetis_lp* lp, void* ws);
int build_generic(thetis_lp* lp, int64_t m, int64_t n, int64_t nnz, const int64_t* colptr,
                  const int32_t* rowidx, const float* val, const int64_t* rowptr, const int32_t* rcol,
                  const float* rval, const float* b, const float* c, const int8_t* sense,
                  const float* lo, const float* hi, int obj_sense, int block_k, int64_t n_blocks);
int recompute_r(thetis_lp* lp);
int recompute_ua(thetis_lp* lp);
int alm_update(thetis_lp* lp, float* ubar, float* zbar, float beta);  // ALM anchors (thetis_solve_alm)
// colour.cu
int ensure_colouring(thetis_lp* lp, uint64_t seed);
// scd.cu
int solve_epochs(thetis_lp* lp, float beta, int epochs, int mode, uint64_t seed, int step_rule,
                 thetis_solve_stats* st);
// async_pi.cu: THETIS_MODE_ASYNC / _SERIAL epochs (epoch_marks[e] recorded after epoch e)
int solve_async_pi(thetis_lp* lp, float beta, int step_rule, int epochs, bool serial, uint64_t seed,
                   cudaEvent_t* epoch_marks, int n_marks);
int launch_tile_perm(int64_t n_tiles, uint64_t seed, int64_t epoch, int64_t* out, cudaStream_t s);
// reduce.cu
int objective(thetis_lp* lp, float beta, thetis_objective_t* out);
// round.cu
int round_x(thetis_lp* lp, const float* x_dev, int rule, uint64_t seed, int reps, uint8_t* out_assign,
            thetis_round_result* out);
}  // namespace thetis

#define THETIS_TRY(expr)              \
    do {                              \
        int _rc = (expr);             \
        if (_rc != THETIS_OK) return _rc; \
    } while (0)

#define CUDA_TRY(lp, expr)                                                               \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            return thetis::set_error(lp, THETIS_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

inline int grid_for(int64_t n, int threads, int cap = 148 * 32) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}
