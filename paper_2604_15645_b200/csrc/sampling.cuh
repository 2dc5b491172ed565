// sampling.cuh -- collocation designs generated on the device
// (sampling.cpp:10-103), written straight into the interior segment of the
// axis-major coordinate array, so resampling (trainer.cpp:421-434) and the
// 64M-point sweep need no host point set and no upload.
//
//   SAMPLE_UNIFORM       sample_uniform: tensor grid of linspace axes, last axis
//                        fastest (sampling.cpp:22-54) -- bit-exact: the same
//                        FP64 operations, no FMA contraction
//   SAMPLE_LHS           sample_lhs: per axis a random permutation of the n
//                        strata plus a uniform jitter in each (sampling.cpp:56-73)
//   SAMPLE_LHS_PER_AXIS  sample_lhs_per_axis: per axis one jittered point per
//                        stratum, then the tensor product (sampling.cpp:75-103)
//
// Randomness is counter-based (a keyed 64-bit mixer of (seed, axis, index)), so
// any row of a design -- in particular a worker's shard [lo, hi) of the global
// design -- is computed independently. It is not the reference's mt19937_64
// stream (libstdc++ std::shuffle + uniform_real_distribution); the host mirror
// (host/) keeps that stream bit-exact for parity. The permutation of the joint
// LHS is a 4-round Feistel bijection on [0, 4^b) with cycle walking onto [0, n).
#pragma once
#include <cstdint>

namespace pnx {

enum { SAMPLE_UNIFORM = 0, SAMPLE_LHS = 1, SAMPLE_LHS_PER_AXIS = 2 };
constexpr int kSampleMaxAxes = 4;

struct SampleArgs {
    int mode, d;
    double lo[kSampleMaxAxes], hi[kSampleMaxAxes];
    int64_t dims[kSampleMaxAxes];  // uniform / per-axis LHS
    int64_t n;                     // design size
    uint64_t seed;
    int64_t row0;                  // first design row written (shard offset)
    int64_t nrows;
    double* out;                   // coords + interior offset; axis a at out + a * ld
    int64_t ld;
};

__host__ __device__ inline uint64_t mix64(uint64_t x) {  // splitmix64 finalizer
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}
__host__ __device__ inline uint64_t key3(uint64_t seed, uint64_t a, uint64_t b) {
    return mix64(seed ^ mix64(a * 0x9e3779b97f4a7c15ull + mix64(b + 0x632be59bd9b4e019ull)));
}
// uniform double in [0, 1) with 53 random bits
__host__ __device__ inline double unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

// bijection of [0, n) keyed by k (Feistel on 2b bits, cycle walking)
__host__ __device__ inline uint64_t permute(uint64_t x, uint64_t n, uint64_t k) {
    int b = 1;
    while ((1ull << (2 * b)) < n) ++b;
    const uint64_t mask = (1ull << b) - 1ull;
    do {
        uint64_t L = x >> b, R = x & mask;
        for (int r = 0; r < 4; ++r) {
            const uint64_t F = key3(k, (uint64_t)r, R) & mask;
            const uint64_t t = R;
            R = L ^ F;
            L = t;
        }
        x = (L << b) | R;
    } while (x >= n);
    return x;
}

// linspace(lo, hi, n)[i] exactly as sampling.cpp:10-20 (no contraction)
__device__ inline double linspace_at(double lo, double hi, int64_t n, int64_t i) {
    if (n == 1) return lo;
    if (i == n - 1) return hi;
    const double h = __ddiv_rn(__dsub_rn(hi, lo), (double)(n - 1));
    return __dadd_rn(lo, __dmul_rn((double)i, h));
}

static __global__ void k_sample(SampleArgs s) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < s.nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = s.row0 + r;
        if (s.mode == SAMPLE_LHS) {
            for (int a = 0; a < s.d; ++a) {
                const double h = __ddiv_rn(__dsub_rn(s.hi[a], s.lo[a]), (double)s.n);
                const uint64_t stratum = permute((uint64_t)idx, (uint64_t)s.n, key3(s.seed, 1000 + a, 0));
                const double u = unit(key3(s.seed, 2000 + a, (uint64_t)idx));
                s.out[a * s.ld + r] = __dadd_rn(s.lo[a], __dmul_rn(__dadd_rn((double)stratum, u), h));
            }
        } else {
            int64_t rem = idx;
            for (int a = s.d - 1; a >= 0; --a) {  // row-major enumeration, last axis fastest
                const int64_t k = rem % s.dims[a];
                rem /= s.dims[a];
                double v;
                if (s.mode == SAMPLE_UNIFORM) {
                    v = linspace_at(s.lo[a], s.hi[a], s.dims[a], k);
                } else {
                    const double h = __ddiv_rn(__dsub_rn(s.hi[a], s.lo[a]), (double)s.dims[a]);
                    v = __dadd_rn(s.lo[a], __dmul_rn(__dadd_rn((double)k, unit(key3(s.seed, 3000 + a, (uint64_t)k))), h));
                }
                s.out[a * s.ld + r] = v;
            }
        }
    }
}

// points per causality segment of the last coordinate (split_time_segments,
// trainer.cpp:156-177): integer counts accumulated in FP64 (exact, order-free)
static __global__ void k_segment_counts(const double* __restrict__ t, int64_t n, int M, double tlo, double span,
                                        double* __restrict__ cnt) {
    __shared__ unsigned long long c[64];
    for (int i = threadIdx.x; i < M; i += blockDim.x) c[i] = 0ull;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double frac = (t[i] - tlo) / span;
        int sg = (int)(frac * M);
        sg = sg < 0 ? 0 : (sg > M - 1 ? M - 1 : sg);
        atomicAdd(&c[sg], 1ull);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < M; i += blockDim.x)
        if (c[i]) atomicAdd(&cnt[i], (double)c[i]);
}

}  // namespace pnx
