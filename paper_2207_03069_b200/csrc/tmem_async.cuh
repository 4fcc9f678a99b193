// tmem_async.cuh -- the asynchronous schedule on the TMEM tier:
// one persistent 256-thread CTA per slot, two per SM, looping the TMEM tier's
// batch (tm_batch_body, Delta in tensor memory) -> async_commit (merge, log,
// seed the next packet under the pool's ticket lock; async_kernel.cuh).
// The TMEM columns, the sigma table and the row mbarriers are set up once per
// CTA and live across batches.
#pragma once
#include "async_kernel.cuh"
#include "tmem_kernel.cuh"

namespace dabs {

template <int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 1) tm_async_kernel(const AsyncArgs a)
{
    const int s = (int)blockIdx.x;
    const unsigned long long t_start = globaltimer();
    unsigned long long t_body = 0, t_commit = 0;
    tm_cta_setup<NT>();
    for (uint32_t k = 0;; k++) {
        const unsigned long long tb = globaltimer();
        tm_batch_body<NT, false, true>(a.bp, s, k);
        __syncthreads();
        const unsigned long long tc = globaltimer();
        t_body += tc - tb;
        const bool more = async_commit<1>(a, s, k);
        t_commit += globaltimer() - tc;
        if (!more) break;
    }
    tm_cta_teardown<NT>();
    if (a.profile && threadIdx.x == 0) {
        atomicAdd(a.lock_ns + 7, t_body);                    // time in batches
        atomicAdd(a.lock_ns + 8, globaltimer() - t_start);   // CTA lifetime
        atomicAdd(a.lock_ns + 9, t_commit);                  // time in commits
    }
}

}  // namespace dabs
