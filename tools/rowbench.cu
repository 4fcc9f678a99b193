// rowbench.cu -- achievable W-row stream bandwidth on B200: every CTA copies
// random 2*n-byte rows of a [n][n] int16 matrix into shared memory with
// cp.async.bulk (4 pieces, mbarrier completion), back to back, with `inflight`
// rows outstanding per CTA and no compute.  This is the memory side of the
// batch kernel's per-flip chain.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void rows(const char* W, size_t row_bytes, int n, int iters, int inflight, unsigned long long* sink)
{
    extern __shared__ __align__(128) char buf[];
    __shared__ __align__(8) uint64_t mb[2][4];
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; b++)
            for (int q = 0; q < 4; q++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[b][q])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const uint32_t piece = (uint32_t)(row_bytes / 4);
    uint32_t x = blockIdx.x * 2654435761u + 12345u;
    unsigned par[2] = {0, 0};
    auto issue = [&](int b) {
        x = x * 1664525u + 1013904223u;
        const char* src = W + (size_t)(x % (uint32_t)n) * row_bytes;
        for (int q = 0; q < 4; q++)
            asm volatile(
                "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(buf + b * row_bytes + q * piece)),
                "l"(src + q * piece), "r"(piece), "r"(su32(&mb[b][q]))
                : "memory");
    };
    auto wait = [&](int b) {
        for (int q = 0; q < 4; q++)
            asm volatile(
                "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                    su32(&mb[b][q])),
                "r"(par[b])
                : "memory");
        par[b] ^= 1;
    };
    unsigned long long acc = 0;
    if (threadIdx.x == 0) {
        for (int b = 0; b < inflight; b++) issue(b);
        for (int it = 0; it < iters; it++) {
            const int b = it % inflight;
            wait(b);
            acc += buf[b * row_bytes + (it & 127)];
            if (it + inflight < iters) issue(b);
        }
        atomicAdd(sink, acc);
    }
}

int main(int argc, char** argv)
{
    // rowbench [n] [max_ctas_per_sm]: n = 32768 streams 2 GiB from HBM; n = 2048
    // keeps the 8 MiB matrix in L2 (the K2000s-class workloads)
    const int n = argc > 1 ? atoi(argv[1]) : 32768;
    const int max_per_sm = argc > 2 ? atoi(argv[2]) : 2;
    const size_t row = 2 * (size_t)n;
    char* W;
    cudaMalloc(&W, row * n);
    cudaMemset(W, 1, row * n);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaFuncSetAttribute(rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * row));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    for (int inflight = 1; inflight <= 2; inflight++)
        for (int per_sm = 1; per_sm <= max_per_sm; per_sm *= 2) {
            const int grid = sms * per_sm;
            rows<<<grid, 32, 2 * row>>>(W, row, n, 50, inflight, sink);
            cudaEventRecord(a);
            rows<<<grid, 32, 2 * row>>>(W, row, n, iters, inflight, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double bytes = (double)grid * iters * row;
            printf("{\"n\": %d, \"row_bytes\": %zu, \"rows_in_flight_per_cta\": %d, \"ctas_per_sm\": %d, "
                   "\"GBps\": %.1f, \"us_per_row_per_cta\": %.3f}\n",
                   n, row, inflight, per_sm, bytes / ms / 1e6, ms * 1e3 / iters);
        }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
