// probe.cuh -- measurement probe: the achievable W-row stream bandwidth on
// this GPU (the denominator of the L2 roofline).
//
// Every CTA copies random rows of a resident [rows][row_bytes] buffer into
// shared memory with cp.async.bulk (the batch kernel's row transfer: TMA
// engine, 4 pieces, mbarrier completion), `inflight` rows outstanding, no
// compute.  With a buffer that fits L2 (126 MB) this is the L2 row-stream
// peak the L2-resident workloads (GS800, TSP32, K2000s, QASP) are measured
// against; with a 2 GiB buffer it is the HBM row stream.
#pragma once
#include "device_common.cuh"

namespace dabs {

__global__ void probe_rows_kernel(const char* W, uint32_t row_bytes, uint32_t rows, int iters, int inflight,
                                  unsigned long long* sink)
{
    extern __shared__ __align__(128) char pbuf[];
    __shared__ __align__(8) uint64_t mb[2][4];
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; b++)
            for (int q = 0; q < 4; q++)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mb[b][q])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t piece = row_bytes / 4;
    uint32_t x = blockIdx.x * 2654435761u + 12345u;
    uint32_t par[2] = {0u, 0u};
    auto issue = [&](int b) {
        x = x * 1664525u + 1013904223u;
        const char* src = W + (size_t)(x % rows) * row_bytes;
        for (int q = 0; q < 4; q++)
            asm volatile(
                "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(pbuf + (size_t)b * row_bytes + q * piece)),
                "l"(src + q * piece), "r"(piece), "r"((uint32_t)__cvta_generic_to_shared(&mb[b][q]))
                : "memory");
    };
    auto wait = [&](int b) {
        for (int q = 0; q < 4; q++)
            asm volatile(
                "{\n\t.reg .pred p;\n\tPW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra PW_%=;\n\t}" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(&mb[b][q])),
                "r"(par[b])
                : "memory");
        par[b] ^= 1u;
    };
    unsigned long long acc = 0;
    for (int b = 0; b < inflight; b++) issue(b);
    for (int it = 0; it < iters; it++) {
        const int b = it % inflight;
        wait(b);
        acc += (unsigned char)pbuf[(size_t)b * row_bytes + (it & 127)];
        if (it + inflight < iters) issue(b);
    }
    atomicAdd(sink, acc);
}

}  // namespace dabs
