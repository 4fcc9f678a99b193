// redbench: cycles per CTA-wide reduction step on one SM (512 threads), the
// building block of every batch-kernel selection.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/redbench tools/redbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ int wmin(int v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ int wmax(int v) { return __reduce_max_sync(0xffffffffu, v); }

template <int MODE, int K>
__global__ void __launch_bounds__(512, 1) bench(int iters, int* out, long long* cyc)
{
    __shared__ int red[2][32][8];
    __shared__ int ared[2][8];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    int d[64];
#pragma unroll
    for (int k = 0; k < 64; k++) d[k] = (t * 2654435761u + k * 40503u) & 0xFFFFF;
    if (t < 16) (&ared[0][0])[t] = (t & 1) ? INT32_MIN : INT32_MAX;
    __syncthreads();
    int acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        const int par = it & 1;
        int v[K];
        // "pass": K partial values over 64 registers
#pragma unroll
        for (int j = 0; j < K; j++) {
            int m = (j & 1) ? INT32_MIN : INT32_MAX;
#pragma unroll
            for (int k = 0; k < 64; k += 2) m = (j & 1) ? max(m, max(d[k], d[k + 1] + j)) : min(m, min(d[k], d[k + 1] + j));
            v[j] = m;
        }
        if (MODE == 0) {          // redux + smem + barrier + redux
#pragma unroll
            for (int j = 0; j < K; j++) v[j] = (j & 1) ? wmax(v[j]) : wmin(v[j]);
            if (lane == 0)
#pragma unroll
                for (int j = 0; j < K; j++) red[par][wid][j] = v[j];
            __syncthreads();
#pragma unroll
            for (int j = 0; j < K; j++) {
                const int x = lane < 16 ? red[par][lane][j] : ((j & 1) ? INT32_MIN : INT32_MAX);
                v[j] = (j & 1) ? wmax(x) : wmin(x);
            }
        } else if (MODE == 1) {   // redux + smem atomics + barrier + one load
#pragma unroll
            for (int j = 0; j < K; j++) v[j] = (j & 1) ? wmax(v[j]) : wmin(v[j]);
            if (lane == 0)
#pragma unroll
                for (int j = 0; j < K; j++) {
                    if (j & 1) atomicMax(&ared[par][j], v[j]);
                    else atomicMin(&ared[par][j], v[j]);
                }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < K; j++) v[j] = ared[par][j];
            if (t < K) ared[par ^ 1][t] = (t & 1) ? INT32_MIN : INT32_MAX;   // reset the other buffer
        } else if (MODE == 2) {   // barrier only (no values)
            __syncthreads();
        } else {                  // no barrier, pass only
        }
#pragma unroll
        for (int j = 0; j < K; j++) acc += v[j];
        // "update": perturb d so the pass is not hoisted
#pragma unroll
        for (int k = 0; k < 64; k++) d[k] += (acc >> (k & 7)) & 3;
    }
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * 512 + t] = acc;
}

template <int MODE, int K>
void run(const char* name)
{
    int* out; long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
    const int iters = 20000;
    bench<MODE, K><<<148, 512>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; i++) s += h[i];
    printf("%-34s K=%d  %7.1f cycles/iter\n", name, K, s / 148 / iters);
    cudaFree(out); cudaFree(cyc);
}

int main()
{
    run<3, 1>("pass only (64 el, no barrier)");
    run<2, 1>("pass + bar.sync");
    run<0, 1>("pass + redux/smem/bar/redux");
    run<1, 1>("pass + redux/smem-atomic/bar");
    run<3, 4>("pass only (64 el, no barrier)");
    run<2, 4>("pass + bar.sync");
    run<0, 4>("pass + redux/smem/bar/redux");
    run<1, 4>("pass + redux/smem-atomic/bar");
    return 0;
}
