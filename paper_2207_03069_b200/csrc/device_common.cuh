// device_common.cuh -- shared device helpers for the DABS sm_100a kernels.
// Citations: P:n = PAPER.md line n; R-x = DESIGN.md section 2 readings.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dabs {

constexpr int ALG_MAXMIN = 0, ALG_CYCLIC = 1, ALG_RANDOM = 2, ALG_POSMIN = 3, ALG_TWO = 4;
constexpr int N_ALG = 5, N_GEN = 9;
// the paper's eight genops + the ABS solver's mutation after crossover (R-27)
constexpr int GEN_MUTATION = 0, GEN_CROSSOVER = 1, GEN_XROSSOVER = 2, GEN_ZERO = 3, GEN_ONE = 4,
              GEN_INTERVALZERO = 5, GEN_BEST = 6, GEN_RANDOM = 7, GEN_MUTCROSS = 8;
constexpr int TABU_RING = 32;   // ring slots kept per search (R-11); tabu period <= 31
constexpr uint32_t PUR_POOL_INIT = 1, PUR_GA_CHOICE = 2, PUR_GA_PARENT = 3, PUR_GA_MASK = 4,
                   PUR_MAXMIN = 5, PUR_RANDMIN = 6, PUR_POSMIN = 7, PUR_POOL_TAGS = 8;
constexpr int64_t E_INF = INT64_MAX;

// Philox4x32-10 (R-16): 10 rounds of (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1,
// lo(M0*c0)), Weyl key schedule.  Counter = (purpose<<24 | sub, id, gen, step).
__device__ __forceinline__ uint4 philox4(uint4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; r++) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

__device__ __forceinline__ uint4 rng4(uint64_t seed, uint32_t purpose, uint32_t sub, uint32_t id,
                                      uint32_t gen, uint32_t step)
{
    return philox4(make_uint4((purpose << 24) | (sub & 0xFFFFFFu), id, gen, step), (uint32_t)seed,
                   (uint32_t)(seed >> 32));
}

// lowbias32 mixer (R-8): bijective 32-bit hash, used per bit pair by RandomMin
__device__ __forceinline__ uint32_t lowbias32(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// RandomMin candidate bits of 4 consecutive bit pairs j0..j0+3 (R-8): bit 2h / 2h+1
// = (low / high 16 bits of lowbias32(K + (j0 + h) * 0x9E3779B9)) < p16, p16 < 65536.
// Both halves are compared at once with the SIMD-within-register __vsetltu2.
__device__ __forceinline__ uint32_t randmin_byte(uint32_t K, uint32_t j0, uint32_t p16)
{
    const uint32_t P = p16 | (p16 << 16);
    uint32_t acc = 0;
#pragma unroll
    for (int h = 0; h < 4; h++) acc |= __vsetltu2(lowbias32(K + (j0 + h) * 0x9E3779B9u), P) << (2 * h);
    return (acc & 0x55u) | ((acc >> 15) & 0xAAu);
}

// floor(u * m / 2^32)  (R-15)
__device__ __forceinline__ uint32_t pick_u(uint32_t u, uint32_t m)
{
    return (uint32_t)(((uint64_t)u * m) >> 32);
}

// 0-based rank-biased row floor(u^3 m / 2^96)  (R-17)
__device__ __forceinline__ uint32_t rank_pick(uint32_t u, uint32_t m)
{
    unsigned __int128 u3 = (unsigned __int128)u * u * u;
    return (uint32_t)((u3 * m) >> 96);
}

__device__ __forceinline__ int warp_min(int v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ int warp_max(int v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ unsigned warp_add(unsigned v) { return __reduce_add_sync(0xffffffffu, v); }
__device__ __forceinline__ unsigned warp_or(unsigned v) { return __reduce_or_sync(0xffffffffu, v); }

}  // namespace dabs
