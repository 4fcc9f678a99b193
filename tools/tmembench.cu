// tmembench.cu -- TMEM load/store throughput per SM (tcgen05.ld/st 32x32b.x64):
// 16 warps (512 threads) of one CTA per SM stream 128 KB of their TMEM columns
// per iteration, the access pattern a search with Delta held in TMEM would use.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld64(uint32_t taddr, uint32_t (&v)[64])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,"
        "%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]),
          "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]),
          "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]),
          "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]),
          "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
        : "r"(taddr));
}
__device__ __forceinline__ void st64(uint32_t taddr, const uint32_t (&v)[64])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,"
        "%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};"
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
          "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
          "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
          "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]), "r"(v[32]),
          "r"(v[33]), "r"(v[34]), "r"(v[35]), "r"(v[36]), "r"(v[37]), "r"(v[38]), "r"(v[39]), "r"(v[40]),
          "r"(v[41]), "r"(v[42]), "r"(v[43]), "r"(v[44]), "r"(v[45]), "r"(v[46]), "r"(v[47]), "r"(v[48]),
          "r"(v[49]), "r"(v[50]), "r"(v[51]), "r"(v[52]), "r"(v[53]), "r"(v[54]), "r"(v[55]), "r"(v[56]),
          "r"(v[57]), "r"(v[58]), "r"(v[59]), "r"(v[60]), "r"(v[61]), "r"(v[62]), "r"(v[63]));
}

__global__ void __launch_bounds__(512, 1) tmem_kernel(int iters, int mode, unsigned long long* out)
{
    __shared__ uint32_t base_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&base_s)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = base_s;
    // warp w: lane quarter w % 4, columns 64 * (w / 4) .. + 64 (of the first 256)
    const uint32_t taddr = base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(64 * (warp >> 2));
    uint32_t v[64];
    for (int j = 0; j < 64; j++) v[j] = threadIdx.x * 64 + j;
    st64(taddr, v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        if (mode != 1) {
            ld64(taddr, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        for (int j = 0; j < 64; j++) v[j] += 1u;
        if (mode != 0) {
            st64(taddr, v);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    for (int j = 0; j < 64; j++) acc ^= v[j];
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x * 2] = (unsigned long long)(t1 - t0); }
    atomicXor((unsigned int*)&out[blockIdx.x * 2 + 1], acc);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

int main()
{
    unsigned long long* out;
    cudaMalloc(&out, 148 * 16);
    const int iters = 2000;
    const char* names[3] = {"load", "store", "load+store"};
    for (int mode = 0; mode < 3; mode++) {
        cudaMemset(out, 0, 148 * 16);
        tmem_kernel<<<148, 512>>>(iters, mode, out);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[296];
        cudaMemcpy(h, out, 148 * 16, cudaMemcpyDeviceToHost);
        const double cyc = (double)h[0] / iters;
        // bytes per iteration per SM: 512 threads x 64 x 4 B = 128 KB (each direction)
        printf("{\"mode\": \"%s\", \"cycles_per_128KB\": %.1f, \"bytes_per_cycle\": %.1f, \"err\": \"%s\"}\n", names[mode],
               cyc, 131072.0 / cyc, cudaGetErrorString(e));
    }
    return 0;
}
