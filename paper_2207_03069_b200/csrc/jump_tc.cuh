// jump_tc.cuh -- the jump-start contraction on the 5th-generation tensor cores
// (R-30 and section 5.2): one hand-written sm_100a
// kernel computes, for every slot s of a generation and every bit k,
//     C_sk = sum_j D_sj W_jk                    (W symmetric, zero diagonal)
// with tcgen05.mma kind::i8 (int8 x int8 -> int32 accumulators in TMEM) and
// writes the slot state the batch starts from (P:498-500 read as R-30):
//     Delta_sk = (1 - 2 d_sk)(W_kk + C_sk)       (Eq.(3))
//     2 E(D_s) = sum_k d_sk (2 W_kk + C_sk)      (Eq.(2))
// Exactness: W = 256 hi + lo with hi = W >> 8 (int8) and lo = W & 255 (uint8);
// D in {0, 1} (uint8).  Both products accumulate in int32 exactly
// (|sum| <= 128 n and 255 n), and C = 256 C_hi + C_lo is taken in wrapping
// 32-bit arithmetic, exact because |C| < 2^31 (dabs_create's range check).
//
// Tiling: UMMA M = 128 slots, N = 256 bits, K = 32 bytes per instruction; a
// CTA owns one 128 x 256 output tile with the hi and lo accumulators in TMEM
// columns [0, 256) and [256, 512) (all 512 columns, one CTA per SM) and walks
// K in 128-byte stages, double-buffered: warp 0 streams the stage's operands
// into shared memory with cp.async.bulk (TMA engine; the operands are stored
// pre-tiled in the canonical no-swizzle K-major core-matrix order, so a stage
// is three contiguous bulk copies), warp 1 issues the MMAs from one thread and
// frees the stage with tcgen05.commit.  The epilogue (all 4 warps, one TMEM
// lane = one slot per thread) reads the accumulators with tcgen05.ld and
// writes Delta and the energy partial sums directly: C never goes to HBM.
// Tiles with the same N block run side by side (blockIdx order), so their W
// stages are shared through L2.
// Citations: P:n = PAPER.md line n; R-x = DESIGN.md readings.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dabs {

constexpr int JT_M = 128;                       // slots per tile (UMMA M)
constexpr int JT_N = 256;                       // bits per tile (UMMA N)
constexpr int JT_K = 128;                       // K bytes per stage
constexpr int JT_STAGES = 2;
constexpr int JT_A_BYTES = JT_M * JT_K;         // 16 KB
constexpr int JT_B_BYTES = JT_N * JT_K;         // 32 KB (each of hi, lo)
constexpr int JT_STAGE_BYTES = JT_A_BYTES + 2 * JT_B_BYTES;
constexpr size_t JT_SMEM = (size_t)JT_STAGES * JT_STAGE_BYTES + 1024;

// byte offset of (row r, K byte kb) inside a rows x 128-byte tile stored as
// core matrices of 8 rows x 16 bytes: [r / 8][kb / 16][r % 8][kb % 16]
__host__ __device__ __forceinline__ uint32_t jt_off(int r, int kb)
{
    return (uint32_t)((((r >> 3) * (JT_K / 16) + (kb >> 4)) << 7) | ((r & 7) << 4) | (kb & 15));
}

// W (int16 [n][n_pad] symmetric) -> tiled hi / lo operands: block (nt, kt) of
// JT_N x JT_K bytes at ((nt * KT + kt) * JT_B_BYTES); row = bit k of the
// output, column = j of the contraction.  Rows >= n and columns >= n are zero.
__global__ void jt_tile_w_kernel(const int16_t* __restrict__ W, int n, int n_pad, int8_t* __restrict__ hi,
                                 uint8_t* __restrict__ lo)
{
    const int KT = n_pad / JT_K;
    const size_t total = (size_t)n_pad * n_pad;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / n_pad), j = (int)(i % n_pad);
        const int w = (k < n && j < n) ? (int)W[(size_t)k * n_pad + j] : 0;
        const size_t o = ((size_t)(k / JT_N) * KT + j / JT_K) * JT_B_BYTES + jt_off(k % JT_N, j % JT_K);
        hi[o] = (int8_t)(w >> 8);          // arithmetic shift: floor(w / 256)
        lo[o] = (uint8_t)(w & 255);
    }
}

// packed targets D [slots][nwp] -> tiled A operand (uint8 0/1): block (mt, kt)
// of JT_M x JT_K bytes; slots >= S are zero rows.  One CTA per (mt, kt) block.
__global__ void jt_tile_d_kernel(const uint32_t* __restrict__ D, int S, int nwp, int n_pad,
                                 uint8_t* __restrict__ A)
{
    const int KT = n_pad / JT_K;
    const int mt = blockIdx.x / KT, kt = blockIdx.x % KT;
    uint8_t* blk = A + (size_t)blockIdx.x * JT_A_BYTES;
    for (int i = threadIdx.x; i < JT_M * JT_K / 4; i += blockDim.x) {
        const int r = i / (JT_K / 4), kb = (i % (JT_K / 4)) * 4;    // 4 consecutive K bytes
        const int s = mt * JT_M + r;
        uint32_t v = 0;
        if (s < S) {
            const uint32_t w = D[(size_t)s * nwp + ((kt * JT_K + kb) >> 5)];
            const int sh = (kt * JT_K + kb) & 31;
            v = ((w >> sh) & 1u) | (((w >> (sh + 1)) & 1u) << 8) | (((w >> (sh + 2)) & 1u) << 16) |
                (((w >> (sh + 3)) & 1u) << 24);
        }
        *reinterpret_cast<uint32_t*>(blk + jt_off(r, kb)) = v;
    }
}

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t jt_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void jt_mbar_init(uint64_t* m, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(jt_smem(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void jt_mbar_wait(uint64_t* m, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "JTW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra JTW_%=;\n\t}" ::"r"(jt_smem(m)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void jt_expect(uint64_t* m, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(jt_smem(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void jt_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* m)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(jt_smem(dst)),
        "l"(src), "r"(bytes), "r"(jt_smem(m))
        : "memory");
}
// UMMA shared-memory descriptor, K-major, no swizzle (canonical interleaved
// layout ((8, m), 2) : ((16 B, SBO), LBO)): LBO = distance between the two
// 16-byte K chunks of one instruction, SBO = distance between 8-row groups;
// bits 46-47 = 1 (the sm_100 descriptor version)
__device__ __forceinline__ uint64_t jt_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// instruction descriptor, kind::i8: D s32, A / B signedness, K-major both, N, M
__host__ __device__ constexpr uint32_t jt_idesc(bool a_signed, bool b_signed)
{
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(JT_N >> 3) << 17) |
           ((uint32_t)(JT_M >> 4) << 24);
}
__device__ __forceinline__ void jt_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void jt_commit(uint64_t* m)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(jt_smem(m))
                 : "memory");
}
__device__ __forceinline__ void jt_ld32(uint32_t taddr, uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// One 128 x 256 output tile per CTA (128 threads).  A_t: tiled D (uint8);
// Bhi_t / Blo_t: tiled W bytes; writes delta [S][n_pad] for the tile's
// columns, adds the tile's part of 2 E(D_s) to e2[s].
__global__ void __launch_bounds__(128, 1)
jt_gemm_kernel(const uint8_t* __restrict__ A_t, const int8_t* __restrict__ Bhi_t, const uint8_t* __restrict__ Blo_t,
               const uint32_t* __restrict__ D, const int32_t* __restrict__ diag, int n, int n_pad, int nwp, int S,
               int MT, int32_t* __restrict__ delta, unsigned long long* __restrict__ e2)
{
    extern __shared__ __align__(1024) uint8_t jsm[];
    __shared__ __align__(8) uint64_t full[JT_STAGES], empty[JT_STAGES], accf;
    __shared__ uint32_t tmem_base_s;
    const int KT = n_pad / JT_K;
    const int mt = (int)blockIdx.x % MT, nt = (int)blockIdx.x / MT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(jsm) + 1023) & ~(uintptr_t)1023);

    if (threadIdx.x == 0) {
        for (int s = 0; s < JT_STAGES; s++) { jt_mbar_init(&full[s], 1); jt_mbar_init(&empty[s], 1); }
        jt_mbar_init(&accf, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {   // TMEM: all 512 columns (hi accumulator at 0, lo at 256)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(jt_smem(&tmem_base_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;

    if (warp == 0 && lane == 0) {
        // producer: stage kt <- A block (mt, kt), B blocks (nt, kt) of hi and lo
        for (int kt = 0; kt < KT; kt++) {
            const int s = kt % JT_STAGES;
            if (kt >= JT_STAGES) jt_mbar_wait(&empty[s], (uint32_t)((kt / JT_STAGES - 1) & 1));
            uint8_t* st = base + (size_t)s * JT_STAGE_BYTES;
            jt_expect(&full[s], (uint32_t)JT_STAGE_BYTES);
            jt_bulk(st, A_t + ((size_t)mt * KT + kt) * JT_A_BYTES, JT_A_BYTES, &full[s]);
            jt_bulk(st + JT_A_BYTES, Bhi_t + ((size_t)nt * KT + kt) * JT_B_BYTES, JT_B_BYTES, &full[s]);
            jt_bulk(st + JT_A_BYTES + JT_B_BYTES, Blo_t + ((size_t)nt * KT + kt) * JT_B_BYTES, JT_B_BYTES, &full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        // MMA issuer: 4 K steps of 32 bytes per stage, hi and lo
        constexpr uint32_t ID_HI = jt_idesc(false, true), ID_LO = jt_idesc(false, false);
        constexpr uint32_t LBO = 128, SBO = (JT_K / 16) * 128;
        for (int kt = 0; kt < KT; kt++) {
            const int s = kt % JT_STAGES;
            jt_mbar_wait(&full[s], (uint32_t)((kt / JT_STAGES) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = jt_smem(base + (size_t)s * JT_STAGE_BYTES);
#pragma unroll
            for (int kk = 0; kk < JT_K / 32; kk++) {
                const uint32_t ko = (uint32_t)kk * 256;   // two 16-byte K chunks = two core matrices
                const uint64_t a = jt_desc(sa + ko, LBO, SBO);
                const uint64_t bh = jt_desc(sa + JT_A_BYTES + ko, LBO, SBO);
                const uint64_t bl = jt_desc(sa + JT_A_BYTES + JT_B_BYTES + ko, LBO, SBO);
                const uint32_t acc = (kt | kk) != 0;
                jt_mma(tmem, a, bh, ID_HI, acc);
                jt_mma(tmem + JT_N, a, bl, ID_LO, acc);
            }
            jt_commit(&empty[s]);      // frees the stage once these MMAs have read it
        }
        jt_commit(&accf);              // accumulators complete
    }
    __syncwarp();

    // ---------------- epilogue: thread = TMEM lane = slot row of the tile
    jt_mbar_wait(&accf, 0u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int r = warp * 32 + lane;
    const int s = mt * JT_M + r;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    long long e2p = 0;
#pragma unroll 1
    for (int c0 = 0; c0 < JT_N; c0 += 32) {
        uint32_t h[32], l[32];
        jt_ld32(lane_addr + (uint32_t)c0, h);
        jt_ld32(lane_addr + (uint32_t)(JT_N + c0), l);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (s < S) {
            const int k0 = nt * JT_N + c0;
            const uint32_t dw = D[(size_t)s * nwp + (k0 >> 5)];      // the 32 target bits of these columns
            int32_t out[32];
#pragma unroll
            for (int j = 0; j < 32; j++) {
                const int k = k0 + j;
                const int32_t dk = diag[k];
                const int32_t c = (int32_t)(256u * h[j] + l[j]);       // wrapping; exact (see header)
                const int32_t g = dk + c;
                const bool x = (dw >> j) & 1u;
                out[j] = k >= n ? dk : (x ? -g : g);
                if (x && k < n) e2p += 2ll * dk + c;
            }
            int4* dst = reinterpret_cast<int4*>(delta + (size_t)s * n_pad + k0);
#pragma unroll
            for (int q = 0; q < 8; q++) dst[q] = make_int4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
        }
    }
    if (s < S && e2p != 0) atomicAdd(&e2[s], (unsigned long long)e2p);   // two's complement sum
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// X = D, E = (2 E) / 2 (sum_k d_k C_k counts every pair twice: even), clear 2E
__global__ void jt_finish_kernel(const uint32_t* __restrict__ D, int S, int nwp, uint32_t* __restrict__ X,
                                 unsigned long long* __restrict__ e2, int64_t* __restrict__ E)
{
    const int s = blockIdx.x;
    for (int w = threadIdx.x; w < nwp; w += blockDim.x) X[(size_t)s * nwp + w] = D[(size_t)s * nwp + w];
    if (threadIdx.x == 0) {
        E[s] = (int64_t)e2[s] / 2;
        e2[s] = 0ull;
    }
}

}  // namespace dabs
