// jump_kernels.cuh -- jump-start batches (R-30): every
// slot of a generation starts its batch AT its target D instead of walking
// there with Straight's flips.  E(D) and Delta(D) for all slots at once need
// C = W . [D_1 .. D_S], one dense contraction: fp16 tensor-core GEMMs with fp32
// accumulation (cuBLAS) on W split into bytes, W = 256*hi + (lo - 128) + 128.
// Every operand is an integer in [-128, 127] or {0, 1} (exact in fp16) and every
// partial sum is an integer of magnitude <= n * 128 <= 2^23 (exact in fp32, in
// any summation order), so the GEMMs are exact:
//   C_k = 256 * (Whi D)_k + (Wlo' D)_k + 128 * popcount(D)      (exact, int32)
//   Delta_k = (1 - 2 d_k)(W_kk + C_k)                          (Eq.(3))
//   E(D) = sum_k d_k (W_kk + C_k / 2)                           (Eq.(2))
// Citations: P:n = PAPER.md line n; R-x = DESIGN.md readings.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace dabs {

// W (int16 [n][n_pad], symmetric, zero diagonal) -> hi, lo' bytes ([n_pad][n_pad], rows >= n zero)
__global__ void jump_split_kernel(const int16_t* __restrict__ W, int n, int n_pad, __half* __restrict__ hi,
                                  __half* __restrict__ lo)
{
    const size_t total = (size_t)n_pad * n_pad;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t k = i / n_pad;
        const int w = k < (size_t)n ? (int)W[i] : 0;
        hi[i] = __int2half_rn(w >> 8);            // arithmetic shift: floor(w / 256)
        lo[i] = __int2half_rn((w & 255) - 128);
    }
}

// packed targets D [slots][nwp] -> bytes Dx [slots][n_pad] (0/1), the GEMM's B operand
__global__ void jump_expand_kernel(const uint32_t* __restrict__ D, int nwp, int n_pad, __half* __restrict__ Dx)
{
    const int s = blockIdx.x;
    const uint32_t* d = D + (size_t)s * nwp;
    __half* o = Dx + (size_t)s * n_pad;
    for (int k = threadIdx.x; k < n_pad; k += blockDim.x)
        o[k] = ((d[k >> 5] >> (k & 31)) & 1u) ? __float2half(1.0f) : __float2half(0.0f);
}

// one CTA per slot: X = D, Delta and E from C (see the header)
__global__ void jump_finish_kernel(const uint32_t* __restrict__ D, const float* __restrict__ Chi,
                                   const float* __restrict__ Clo, const int32_t* __restrict__ diag, int n,
                                   int n_pad, int nwp, uint32_t* __restrict__ X, int32_t* __restrict__ delta,
                                   int64_t* __restrict__ E)
{
    const int s = blockIdx.x;
    const uint32_t* d = D + (size_t)s * nwp;
    __shared__ int pop_s;
    __shared__ long long e_s;
    if (threadIdx.x == 0) { pop_s = 0; e_s = 0; }
    __syncthreads();
    int pop = 0;
    for (int w = threadIdx.x; w < nwp; w += blockDim.x) {
        pop += __popc(d[w]);
        X[(size_t)s * nwp + w] = d[w];
    }
    atomicAdd(&pop_s, pop);
    __syncthreads();
    const int32_t p128 = 128 * pop_s;
    const float* ch = Chi + (size_t)s * n_pad;
    const float* cl = Clo + (size_t)s * n_pad;
    int32_t* dl = delta + (size_t)s * n_pad;
    long long e2 = 0;   // 2 E = sum_k d_k (2 W_kk + C_k)
    for (int k = threadIdx.x; k < n_pad; k += blockDim.x) {
        if (k >= n) { dl[k] = diag[k]; continue; }
        const int32_t c = 256 * __float2int_rn(ch[k]) + __float2int_rn(cl[k]) + p128;
        const int32_t g = diag[k] + c;
        const bool x = (d[k >> 5] >> (k & 31)) & 1u;
        dl[k] = x ? -g : g;
        if (x) e2 += 2ll * diag[k] + c;
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(&e_s), (unsigned long long)e2);   // two's complement sum
    __syncthreads();
    if (threadIdx.x == 0) E[s] = (int64_t)(e_s / 2);   // sum_k d_k C_k counts every pair twice: even
}

}  // namespace dabs
