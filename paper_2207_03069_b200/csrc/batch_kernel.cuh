// batch_kernel.cuh -- the DABS hot loop on sm_100a: one batch search per CTA.
//
// A CTA of NT threads owns one search (one slot).  Element k of the search
// lives in thread t = (k/8) mod NT, chunk c = (k/8) / NT, lane-of-chunk e = k mod 8,
// so every thread holds EPT = 8*C flip gains Delta_k in REGISTERS and the bits
// x_k, d_k of its elements in one bits_t word.
//
// Per flip (Step 3):  one elected thread streams row i of the
// symmetric int16 W (2*n_pad bytes) from L2/HBM into shared
// memory with cp.async.bulk (TMA engine, mbarrier completion, NP pieces so the
// update of the first chunks overlaps the tail of the transfer); every thread
// then applies Eq.(4) to its registers.  Step 1 (scan, BEST;
// P:376-379) and Step 2 (selection) reduce over the CTA with
// redux.sync + one shared-memory exchange (one __syncthreads per argmin).
//
// MW=false: one warp per search (n <= 2048), no CTA barriers at all.
// MW=true : NT in {64..512} threads per search (n <= 32768).
// CL=2    : a cluster of two CTAs of NT threads per search (n <= 65536,
//           SURVEY 8(f) f2).  Each CTA holds half of every chunk (thread
//           tq = rank*NT + t of the search's 2*NT), streams its half of the
//           row, and every CTA-wide reduction is completed by one DSMEM swap
//           with the peer CTA (cl_swap).
//
// Citations: P:n = PAPER.md line n; R-x = DESIGN.md readings.
#pragma once
#include <type_traits>

#include "device_common.cuh"

namespace dabs {

struct BatchParams {
    const int16_t* W;        // [n][n_pad] symmetric, zero diagonal, zero padding
    const int32_t* wtab;     // [T+1] CyclicMin width w(t)       (R-7)
    const int32_t* ptab;     // [T+1] RandomMin threshold p16(t) (R-8)
    const int32_t* rmax;     // [n] max_k |W_ik|: bounds how far any Delta can fall per flip
    double invT3;            // 1 / T^3 (MaxMin span estimate, corrected exactly)
    const uint64_t* mtab;    // [T+1] floor(2^64 (T-t)^3 / T^3) (MaxMin span estimate, TMEM tier)
    int n, n_pad, nwp;       // nwp = n_pad / 32 words per bit vector
    int T, B, tabu;
    uint64_t seed;
    uint32_t gen;
    const uint32_t* gen_ptr; // graph replays: the generation index in device memory (else gen)
    uint32_t slot_base;      // global id of local slot 0
    int slot0;               // first local slot of this launch (blockIdx.x offset)
    int count;               // searches in this launch (the TMEM warp tier packs 4 per CTA)
    const int32_t* order;    // optional launch order of the slots (longest batches first)
    uint32_t* X;             // [slots][nwp]   persistent x (R-14)
    int32_t* delta;          // [slots][n_pad] persistent Delta (pads = INT32_MAX)
    int64_t* E;              // [slots]
    int32_t* ring;           // [slots][32] tabu ring, most recent first, -1 empty
    const uint32_t* D;       // [slots][nwp] target vectors (packets in)
    const uint8_t* algo;     // [slots]
    uint32_t* best;          // [slots][nwp] packets out: BEST
    int64_t* ebest;          // [slots]
    int64_t* flips;          // [slots]
    unsigned long long* flip_total;
    int trace_slot;
    int32_t* tr_bit;
    int64_t* tr_E;
    int8_t* tr_phase;
    int64_t tr_cap;
};

// warp tier: sigma words from a 256-entry table instead of 16 sign registers
// (A/B on B200, tools/gpu_ab_warp.sh: K2000s +4.7 %, TSP32 +4.9 %, GS800 +4.0 %)
#ifndef DABS_WARP_LUT
#define DABS_WARP_LUT 1
#endif

#ifndef DABS_NP_MAX
#define DABS_NP_MAX 4   // W-row pieces (one mbarrier each) per flip in the CTA tiers (A/B: -DDABS_NP_MAX=8)
#endif

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// one elected thread: expect `bytes` on mbarrier m and start the bulk copy
__device__ __forceinline__ void bulk_row_piece(void* dst, const void* src, uint32_t bytes, uint64_t* m)
{
    asm volatile(
        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(m))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}

// expect `bytes` more on mbarrier m (the copies that deliver them follow)
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* m)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(m))
        : "memory");
}

// ---- thread-block cluster (CL = 2 CTAs per search, DSMEM exchange)
__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_peer(uint32_t addr, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_peer(uint32_t addr, int v)
{
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_peer(uint32_t addr)
{
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* m, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Swap K uniform values with the peer CTA of the cluster.  Thread 0 stores them
// into the peer's xv[par] and arrives (release.cluster) on the peer's xbar[par];
// every thread waits (acquire.cluster) on its own xbar[par].  Callers reach
// this right after a __syncthreads, so the peer can only reuse xv[par] (two
// swaps later) once every thread here has read it.
template <int K>
__device__ __forceinline__ void cl_swap(const int (&mine)[K], int (&theirs)[K], int32_t (*xv)[8], uint64_t* xbar,
                                        int& xc, uint32_t peer, int t)
{
    const int par = xc & 1;
    const uint32_t ph = (uint32_t)(xc >> 1) & 1u;
    xc++;
    if (t == 0) {
        const uint32_t base = mapa_peer(smem_u32(&xv[par][0]), peer);
#pragma unroll
        for (int k = 0; k < K; k++) st_peer(base + 4u * k, mine[k]);
        mbar_arrive_peer(mapa_peer(smem_u32(&xbar[par]), peer));
    }
    mbar_wait_cluster(&xbar[par], ph);
#pragma unroll
    for (int k = 0; k < K; k++) theirs[k] = xv[par][k];
}

enum : int { OP_MIN = 0, OP_MAX = 1, OP_ADD = 2, OP_OR = 3 };

__device__ __forceinline__ int wop(int op, int v)
{
    switch (op) {
    case OP_MIN: return warp_min(v);
    case OP_MAX: return warp_max(v);
    case OP_ADD: return (int)warp_add((unsigned)v);
    default: return (int)warp_or((unsigned)v);
    }
}
__device__ __forceinline__ int op2(int op, int a, int b)
{
    switch (op) {
    case OP_MIN: return min(a, b);
    case OP_MAX: return max(a, b);
    case OP_ADD: return a + b;
    default: return a | b;
    }
}
__device__ __forceinline__ int op_ident(int op)
{
    return op == OP_MIN ? INT32_MAX : (op == OP_MAX ? INT32_MIN : 0);
}

constexpr int RED_W = 10;   // values per warp in one shared-memory exchange

// Reduce K values over the CTA; every thread gets the results.  Slots marked
// OP_ARGKEY-style pairs are handled by the caller.  One __syncthreads (MW).
template <bool MW, int K>
__device__ __forceinline__ void block_reduce(int (&v)[K], const int (&ops)[K],
                                             int32_t (*red)[32][RED_W], int& rc, int lane, int wid,
                                             int NW)
{
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = wop(ops[k], v[k]);
    if constexpr (MW) {
        const int par = rc & 1;
        rc++;
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < K; k++) red[par][wid][k] = v[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int x = lane < NW ? red[par][lane][k] : op_ident(ops[k]);
            v[k] = wop(ops[k], x);
        }
    }
}

// d[k] for a runtime k: jump table (one lane of a warp executes these)
template <int EPT>
__device__ __forceinline__ int get_at(const int32_t (&d)[EPT], int k)
{
    int v = 0;
    switch (k) {
#define DABS_CASE(j) \
    case j:          \
        if constexpr (j < EPT) v = d[j]; \
        break;
        DABS_CASE(0) DABS_CASE(1) DABS_CASE(2) DABS_CASE(3) DABS_CASE(4) DABS_CASE(5) DABS_CASE(6) DABS_CASE(7)
        DABS_CASE(8) DABS_CASE(9) DABS_CASE(10) DABS_CASE(11) DABS_CASE(12) DABS_CASE(13) DABS_CASE(14) DABS_CASE(15)
        DABS_CASE(16) DABS_CASE(17) DABS_CASE(18) DABS_CASE(19) DABS_CASE(20) DABS_CASE(21) DABS_CASE(22) DABS_CASE(23)
        DABS_CASE(24) DABS_CASE(25) DABS_CASE(26) DABS_CASE(27) DABS_CASE(28) DABS_CASE(29) DABS_CASE(30) DABS_CASE(31)
        DABS_CASE(32) DABS_CASE(33) DABS_CASE(34) DABS_CASE(35) DABS_CASE(36) DABS_CASE(37) DABS_CASE(38) DABS_CASE(39)
        DABS_CASE(40) DABS_CASE(41) DABS_CASE(42) DABS_CASE(43) DABS_CASE(44) DABS_CASE(45) DABS_CASE(46) DABS_CASE(47)
        DABS_CASE(48) DABS_CASE(49) DABS_CASE(50) DABS_CASE(51) DABS_CASE(52) DABS_CASE(53) DABS_CASE(54) DABS_CASE(55)
        DABS_CASE(56) DABS_CASE(57) DABS_CASE(58) DABS_CASE(59) DABS_CASE(60) DABS_CASE(61) DABS_CASE(62) DABS_CASE(63)
#undef DABS_CASE
    default: break;
    }
    return v;
}
template <int EPT>
__device__ __forceinline__ void neg_at(int32_t (&d)[EPT], int k)
{
    switch (k) {
#define DABS_CASE(j) \
    case j:          \
        if constexpr (j < EPT) d[j] = -d[j]; \
        break;
        DABS_CASE(0) DABS_CASE(1) DABS_CASE(2) DABS_CASE(3) DABS_CASE(4) DABS_CASE(5) DABS_CASE(6) DABS_CASE(7)
        DABS_CASE(8) DABS_CASE(9) DABS_CASE(10) DABS_CASE(11) DABS_CASE(12) DABS_CASE(13) DABS_CASE(14) DABS_CASE(15)
        DABS_CASE(16) DABS_CASE(17) DABS_CASE(18) DABS_CASE(19) DABS_CASE(20) DABS_CASE(21) DABS_CASE(22) DABS_CASE(23)
        DABS_CASE(24) DABS_CASE(25) DABS_CASE(26) DABS_CASE(27) DABS_CASE(28) DABS_CASE(29) DABS_CASE(30) DABS_CASE(31)
        DABS_CASE(32) DABS_CASE(33) DABS_CASE(34) DABS_CASE(35) DABS_CASE(36) DABS_CASE(37) DABS_CASE(38) DABS_CASE(39)
        DABS_CASE(40) DABS_CASE(41) DABS_CASE(42) DABS_CASE(43) DABS_CASE(44) DABS_CASE(45) DABS_CASE(46) DABS_CASE(47)
        DABS_CASE(48) DABS_CASE(49) DABS_CASE(50) DABS_CASE(51) DABS_CASE(52) DABS_CASE(53) DABS_CASE(54) DABS_CASE(55)
        DABS_CASE(56) DABS_CASE(57) DABS_CASE(58) DABS_CASE(59) DABS_CASE(60) DABS_CASE(61) DABS_CASE(62) DABS_CASE(63)
#undef DABS_CASE
    default: break;
    }
}
// The owner of flipped element k: Delta_k <- -Delta_k (Eq.(5)) and sigma(x_k)
// byte flipped, one jump table for both
template <int EPT>
__device__ __forceinline__ void owner_flip(int32_t (&d)[EPT], uint32_t (&sg)[EPT / 4], int k)
{
    const uint32_t m = 0xFEu << (8 * (k & 3));
    switch (k) {
#define DABS_CASE(j) \
    case j:          \
        if constexpr (j < EPT) { d[j] = -d[j]; sg[j >> 2] ^= m; } \
        break;
        DABS_CASE(0) DABS_CASE(1) DABS_CASE(2) DABS_CASE(3) DABS_CASE(4) DABS_CASE(5) DABS_CASE(6) DABS_CASE(7)
        DABS_CASE(8) DABS_CASE(9) DABS_CASE(10) DABS_CASE(11) DABS_CASE(12) DABS_CASE(13) DABS_CASE(14) DABS_CASE(15)
        DABS_CASE(16) DABS_CASE(17) DABS_CASE(18) DABS_CASE(19) DABS_CASE(20) DABS_CASE(21) DABS_CASE(22) DABS_CASE(23)
        DABS_CASE(24) DABS_CASE(25) DABS_CASE(26) DABS_CASE(27) DABS_CASE(28) DABS_CASE(29) DABS_CASE(30) DABS_CASE(31)
        DABS_CASE(32) DABS_CASE(33) DABS_CASE(34) DABS_CASE(35) DABS_CASE(36) DABS_CASE(37) DABS_CASE(38) DABS_CASE(39)
        DABS_CASE(40) DABS_CASE(41) DABS_CASE(42) DABS_CASE(43) DABS_CASE(44) DABS_CASE(45) DABS_CASE(46) DABS_CASE(47)
        DABS_CASE(48) DABS_CASE(49) DABS_CASE(50) DABS_CASE(51) DABS_CASE(52) DABS_CASE(53) DABS_CASE(54) DABS_CASE(55)
        DABS_CASE(56) DABS_CASE(57) DABS_CASE(58) DABS_CASE(59) DABS_CASE(60) DABS_CASE(61) DABS_CASE(62) DABS_CASE(63)
#undef DABS_CASE
    default: break;
    }
}

// min over all EPT values with 4 independent accumulators (ILP)
template <int EPT>
__device__ __forceinline__ int min_all(const int32_t (&d)[EPT])
{
    int a[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
#pragma unroll
    for (int k = 0; k < EPT; k++) a[k & 3] = min(a[k & 3], d[k]);
    return min(min(a[0], a[1]), min(a[2], a[3]));
}

// sigma(x_k) of element k is byte k%4 of sg[k/4] (0x01 = +1, 0xFF = -1); flip it
template <int NG>
__device__ __forceinline__ void flip_sign_at(uint32_t (&sg)[NG], int k)
{
    const uint32_t m = 0xFEu << (8 * (k & 3));
    switch (k >> 2) {
#define DABS_G(j) \
    case j:       \
        if constexpr (j < NG) sg[j] ^= m; \
        break;
        DABS_G(0) DABS_G(1) DABS_G(2) DABS_G(3) DABS_G(4) DABS_G(5) DABS_G(6) DABS_G(7)
        DABS_G(8) DABS_G(9) DABS_G(10) DABS_G(11) DABS_G(12) DABS_G(13) DABS_G(14) DABS_G(15)
#undef DABS_G
    default: break;
    }
}

// first lane-of-chunk e in chunk c with mask bit set and d == m (or -1)
template <int EPT, typename bits_t>
__device__ __forceinline__ int first_in_chunk(const int32_t (&d)[EPT], bits_t M, int c, int m)
{
    int r = -1;
    switch (c) {
#define DABS_CHUNK(cc)                                                                    \
    case cc:                                                                              \
        if constexpr (8 * cc < EPT) {                                                     \
            _Pragma("unroll") for (int e = 7; e >= 0; e--) if (((M >> (8 * cc + e)) & 1) && \
                                                                  d[8 * cc + e] == m) r = e; \
        }                                                                                 \
        break;
        DABS_CHUNK(0) DABS_CHUNK(1) DABS_CHUNK(2) DABS_CHUNK(3)
        DABS_CHUNK(4) DABS_CHUNK(5) DABS_CHUNK(6) DABS_CHUNK(7)
#undef DABS_CHUNK
    default: break;
    }
    return r;
}

// floor(a * f / q) exactly, a < 2^32, f, q <= 2^48 (MaxMin span, R-6): a double
// estimate (inv_q = 1/q precomputed; relative error ~2^-50, so the estimate is
// off by at most one) corrected once with the remainder a*f - est*q, whose
// true value is tiny, computed exactly in wrapping 64-bit arithmetic.
__device__ __forceinline__ uint64_t muldiv_floor(uint64_t a, uint64_t f, uint64_t q, double inv_q)
{
    uint64_t est = (uint64_t)((double)a * (double)f * inv_q);
    const int64_t rem = (int64_t)(a * f - est * q);
    if (rem < 0) est--;
    else if ((uint64_t)rem >= q) est++;
    return est;
}

#ifdef DABS_TIMING
// diagnostic build only (-DDABS_TIMING): per bucket (main phase of algorithm 0-4,
// 5 = Straight/Greedy) SM cycles of thread 0 in [selection, wait for the first
// row piece, rest of transfer + update, loop head], and flips
__device__ unsigned long long g_tstat[6][5];
__device__ unsigned long long g_tstat2[10];   // MaxMin/PositiveMin selection sub-steps
#define DABS_TS(k) do { if (t == 0) { const long long now_ = clock64(); ts2_s[k] += now_ - tlast; tlast = now_; } } while (0)
#else
#define DABS_TS(k) do { } while (0)
#endif

__device__ __forceinline__ void mbar_inval(uint64_t* m)
{
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(m)) : "memory");
}

// One batch search of slot s: load the slot's persistent state,
// Straight(D) -> Greedy -> {main -> Greedy} until B flips, write back the
// state and the result packet.  `gen` is the Philox generation field (the
// generation, or the slot's batch index under the asynchronous schedule,
// R-29).  REUSE: the CTA runs further batches afterwards (persistent kernel),
// so the row mbarriers are invalidated at the end.
template <int C, int NTT, int CL, bool TRACE, bool REUSE>
__device__ __forceinline__ void batch_body(const BatchParams& p, const int s, const uint32_t gen, const bool first = true)
{
    static_assert(CL == 1 || (CL == 2 && NTT > 32), "cluster tier needs the CTA tier");
    constexpr bool MW = NTT > 32;                    // more than one warp per search
    constexpr int EPT = 8 * C;
    constexpr int NP = MW ? (C >= DABS_NP_MAX ? DABS_NP_MAX : C) : 1;   // row pieces, one mbarrier each
    constexpr int CPP = C / NP;                      // chunks per piece
    constexpr int CW = (C + 1) / 2;                  // packed count words (two 16-bit fields)
    using bits_t = typename std::conditional<(EPT > 32), unsigned long long, uint32_t>::type;
    constexpr bits_t ONE = 1;
    constexpr bits_t ALL = ~(bits_t)0;
    constexpr unsigned FULL = 0xffffffffu;
    const int t = threadIdx.x;
    constexpr int NT = NTT;                          // threads per search (compile time)
    constexpr int lgNT = NT == 32 ? 5 : NT == 64 ? 6 : NT == 128 ? 7 : NT == 256 ? 8 : 9;
    constexpr int NTG = NT * CL;                     // threads of the whole search
    constexpr int lgNTG = lgNT + (CL == 2 ? 1 : 0);
    constexpr int NW = NT >> 5;
    const int lane = t & 31, wid = t >> 5;
    const uint32_t rank = CL == 2 ? cluster_rank() : 0u;   // CTA within the search's cluster
    const int tq = (int)rank * NT + t;                      // thread within the search
    const uint32_t gslot = p.slot_base + (uint32_t)s;
    const int n = p.n;

    extern __shared__ __align__(128) uint8_t dyn_smem[];
    const int nl = p.n_pad / CL;              // elements held by this CTA
    const uint4* row_s = reinterpret_cast<const uint4*>(dyn_smem);   // this CTA's part of a W row, 2*nl bytes
    uint8_t* tcnt = dyn_smem + 2 * nl;        // per local element: occurrences in the last `tabu` flips
    __shared__ __align__(8) uint64_t mbar[NP];
    __shared__ int32_t ring_s[TABU_RING];
    __shared__ int32_t red_s[2][32][RED_W];
    __shared__ int32_t bc_s[2][4];
    __shared__ int32_t sel_s[4];   // MaxMin/PositiveMin pick, published through the row mbarrier
    __shared__ int32_t xv_s[2][8];                 // CL = 2: the peer CTA's values of a swap
    __shared__ __align__(8) uint64_t xbar[2];
    int xc = 0;
    const uint32_t peer = rank ^ 1u;

    // ---------------- load the slot's persistent state (R-14)
    int32_t d[EPT];
    bits_t xb = 0, db = 0, vb = 0;
    {
        const uint8_t* Xb = reinterpret_cast<const uint8_t*>(p.X + (size_t)s * p.nwp);
        const uint8_t* Db = reinterpret_cast<const uint8_t*>(p.D + (size_t)s * p.nwp);
        const int32_t* dp = p.delta + (size_t)s * p.n_pad;
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int ch = (c << lgNTG) + tq;
            xb |= (bits_t)Xb[ch] << (8 * c);
            // REUSE: the packet was written by the commit warp (on the cluster's
            // other SM for CL = 2): read it from L2, not a stale L1 line
            db |= (bits_t)(REUSE ? __ldcg(Db + ch) : Db[ch]) << (8 * c);
            const int nv = min(max(n - ch * 8, 0), 8);
            vb |= (bits_t)((1u << nv) - 1u) << (8 * c);
            const int4 a = reinterpret_cast<const int4*>(dp + ch * 8)[0];
            const int4 b = reinterpret_cast<const int4*>(dp + ch * 8)[1];
            d[8 * c + 0] = a.x; d[8 * c + 1] = a.y; d[8 * c + 2] = a.z; d[8 * c + 3] = a.w;
            d[8 * c + 4] = b.x; d[8 * c + 5] = b.y; d[8 * c + 6] = b.z; d[8 * c + 7] = b.w;
        }
    }
    // sigma(x_k) as signed bytes (0x01 = +1, 0xFF = -1), 4 elements per word:
    // the int8 operand of the IDP.2A dot products that apply Eq.(4).  One warp
    // per search: in registers.  CTA tiers (registers are the limit): in shared
    // memory, [2][ceil(C/2)][NT] uint4 (16 bytes = two chunks per thread,
    // conflict-free), copy 0 as is for sigma(x_i) = +1 and copy 1 negated for
    // sigma(x_i) = -1, so the update needs no per-word negation.
    // DABS_WARP_LUT: the warp tier takes the four IDP.2A sign words of a chunk
    // from a 256-entry table indexed by the chunk's 8 x bits (as the TMEM tier)
    // instead of keeping sigma bytes in 16 registers
    constexpr bool WLUT = !MW && DABS_WARP_LUT;
    __shared__ uint4 lutw_s[WLUT ? 256 : 1];
    if constexpr (WLUT) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t v = (uint32_t)(j * 32 + t);
            uint32_t w[4];
#pragma unroll
            for (int h = 0; h < 4; h++)
                w[h] = (((v >> (2 * h)) & 1u) ? 0x01u : 0xFFu) | ((((v >> (2 * h + 1)) & 1u) ? 0x01u : 0xFFu) << 24);
            lutw_s[v] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        __syncwarp();
    }
    uint32_t sg[(MW || WLUT) ? 1 : EPT / 4];
    uint4* sgs = reinterpret_cast<uint4*>(dyn_smem + 3 * nl);
    constexpr int SGC = ((C + 1) / 2) << lgNT;   // uint4s per copy
#pragma unroll
    for (int g = 0; g < ((MW || !WLUT) ? EPT / 4 : 0); g++) {
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) w |= (((xb >> (4 * g + j)) & 1) ? 0x01u : 0xFFu) << (8 * j);
        if constexpr (MW) {
            uint32_t* s32 = reinterpret_cast<uint32_t*>(sgs);
            s32[(((g >> 2) << lgNT) + t) * 4 + (g & 3)] = w;
            s32[(SGC + ((g >> 2) << lgNT) + t) * 4 + (g & 3)] = w ^ 0xFEFEFEFEu;
        } else {
            sg[g] = w;
        }
    }
    if (t < TABU_RING) ring_s[t] = REUSE ? __ldcg(p.ring + (size_t)s * TABU_RING + t) : p.ring[(size_t)s * TABU_RING + t];
    // REUSE (persistent CTA, CL = 1): the row mbarriers live across batches
    // (initialised by the first batch, phase parity kept in par_keep) -- no
    // invalidate / re-init between batches
    constexpr bool KEEP = REUSE && CL == 1;
    __shared__ uint32_t par_keep;
    if (t == 0 && (!KEEP || first)) {
#pragma unroll
        for (int qq = 0; qq < NP; qq++) mbar_init(&mbar[qq], 1);
        if constexpr (CL == 2) { mbar_init(&xbar[0], 1); mbar_init(&xbar[1], 1); }
        fence_mbar_init();
    }
    int pos = 0;   // ring_s[(pos + j) & 31] = j-th most recent flip
    int64_t E = REUSE ? (int64_t)__ldcg(reinterpret_cast<const long long*>(p.E + s)) : p.E[s];
    const int algo = REUSE ? (int)__ldcg(p.algo + s) : (int)p.algo[s];
    const int tabu = p.tabu;
    const int T = p.T;
    // tabu state (R-11): each thread counts its own elements' occurrences in
    // the last `tabu` flips (shared memory) and keeps the bits count > 0 in tm
#pragma unroll
    for (int c = 0; c < C; c++) reinterpret_cast<uint2*>(tcnt)[(c << lgNT) + t] = make_uint2(0u, 0u);
    const uint32_t piece_bytes = (uint32_t)(2 * nl / NP);
    uint32_t par_row = (KEEP && !first) ? par_keep : 0u;
    int flips = 0;
    int64_t ebest = E_INF;
    bits_t bdiff = 0;              // BEST = X xor bdiff
    int rc = 0;                    // exchange parity counter
    if constexpr (CL == 2) cluster_sync_all();      // the peer's barriers exist before any swap
    else if constexpr (MW) __syncthreads();
    else __syncwarp();

    auto gidx = [&](int c, int e) { return (((c << lgNTG) + tq) << 3) | e; };
    auto owns = [&](int k) { return ((k >> 3) & (NTG - 1)) == tq; };
    auto lbit = [&](int k) { return (((k >> 3) >> lgNTG) << 3) | (k & 7); };
    // shared-memory index of an owned element (= k for CL = 1)
    auto lidx = [&](int k) { return (((k >> 3) >> lgNTG) << (lgNT + 3)) | (t << 3) | (k & 7); };
    // start the copy of this CTA's part of row i (every chunk's NT*8 elements)
    auto issue_row = [&](int i) {
        fence_proxy_async();
        const char* src = reinterpret_cast<const char*>(p.W) + (size_t)i * (size_t)(2 * p.n_pad);
#pragma unroll
        for (int qq = 0; qq < NP; qq++) {
            if constexpr (CL == 1) {
                bulk_row_piece(dyn_smem + qq * piece_bytes, src + qq * piece_bytes, piece_bytes, &mbar[qq]);
            } else {
                mbar_expect(&mbar[qq], piece_bytes);
#pragma unroll
                for (int cc = 0; cc < CPP; cc++) {
                    const int c = qq * CPP + cc;
                    bulk_copy(dyn_smem + ((size_t)c << (lgNT + 4)), src + ((size_t)((c << lgNTG) + (int)rank * NT) << 4),
                              (uint32_t)(NT * 16), &mbar[qq]);
                }
            }
        }
    };
    // complete a CTA-wide reduction over the cluster (CL = 2; no-op otherwise)
    auto cl_combine = [&](auto& v, const auto& ops) {
        if constexpr (CL == 2) {
            constexpr int K = sizeof(ops) / sizeof(ops[0]);
            int o[K];
            cl_swap<K>(v, o, xv_s, xbar, xc, peer, t);
#pragma unroll
            for (int k = 0; k < K; k++) v[k] = op2(ops[k], v[k], o[k]);
        }
    };

    // phases: 0 Straight, 1 Greedy, 2 main (R-12)
    int phase = 0, round = 0, tt = 0, cursor = 0;
    bool after_main = false;
    bits_t tm = 0;                 // tabu mask of this thread's elements (R-11)
    // Lower bound on min_k Delta_k.  Step 1 can only improve BEST if
    // E + min Delta < E(BEST); while E + glb >= E(BEST) the exact global
    // minimum is not needed (the paper's "BEST updates are rare").
    // After flipping i: Delta_k moves by at most |W_ik|, Delta_i becomes -Delta_i.
    int64_t glb = INT64_MIN / 4;

    // RandomMin candidates of main step ttv at batch flip fl (R-8): u16(k) = half
    // (k mod 2) of lowbias32(K + (k/2) * 0x9E3779B9), K = one Philox word per flip
    // The main rule's Philox draw of batch step fl (R-6, R-8, R-9): every warp
    // computes the draws of 32 consecutive steps at once, lane j holding step
    // base + j, and hands out the one a step needs with a shuffle (one Philox
    // per lane per 32 flips instead of one per thread per flip).
    const uint32_t pur = algo == ALG_MAXMIN ? PUR_MAXMIN : (algo == ALG_RANDOM ? PUR_RANDMIN : PUR_POSMIN);
    int rng_base = -1;
    uint32_t rng_x = 0, rng_y = 0;
    auto draw = [&](int fl) -> uint2 {
        if ((fl >> 5) != rng_base) {
            rng_base = fl >> 5;
            const uint4 r = rng4(p.seed, pur, 0, gslot, gen, (uint32_t)((rng_base << 5) + lane));
            rng_x = r.x;
            rng_y = r.y;
        }
        return make_uint2(__shfl_sync(FULL, rng_x, fl & 31), __shfl_sync(FULL, rng_y, fl & 31));
    };
    auto rand_cand = [&](int ttv, int fl) -> bits_t {
        const uint32_t p16 = (uint32_t)p.ptab[ttv];
        if (p16 >= 65536u) return vb;
        const uint32_t K = draw(fl).x;
        bits_t cand = 0;
#pragma unroll
        for (int c = 0; c < C; c++) {
            const uint32_t j0 = (uint32_t)(((c << lgNTG) + tq) << 2);   // first pair of the chunk
            cand |= (bits_t)randmin_byte(K, j0, p16) << (8 * c);
        }
        return cand;
    };
    // (MW) the next main step's draws, computed while the row is in flight
    int pre_for = -1;

    bits_t cand_pre = 0;
    for (int j = 0; j < tabu; j++) {
        const int r = ring_s[j];
        if (r >= 0 && owns(r)) { tcnt[lidx(r)]++; tm |= ONE << lbit(r); }
    }

#ifdef DABS_TIMING
    __shared__ unsigned int ts_s[6][5];
    __shared__ unsigned int ts2_s[10];
    long long tlast = 0;
    if (t == 0) {
        for (int j = 0; j < 30; j++) (&ts_s[0][0])[j] = 0u;
        for (int j = 0; j < 10; j++) ts2_s[j] = 0u;
    }
    long long tA = clock64(), tB = 0, tC = 0, tD = tA;
    int tbk = 5;
#endif
    while (true) {
#ifdef DABS_TIMING
        tA = clock64();
#endif
        // ---------------- phase transitions
        if (phase == 2 && tt == (algo == ALG_TWO ? 2 * n - 1 : T)) {
            phase = 1;
            after_main = true;
        }
        // ---------------- Step 2 setup: candidate masks (uniform control)
        // kind 0: argmin over M1 (masked) or over all bits (!masked)
        // kind 1: uniform pick among candidates (MaxMin, PositiveMin)
        // kind 2: fixed bit (TwoNeighbor)
        int kind = 0;
        bool masked = true;
        bits_t M1 = vb, M2 = 0;
        int fb = 0;                    // fallback: 1 drop tabu in the window, 2 RandomMin
        int fixed_i = 0;
        if (phase == 0) {
            M1 = (xb ^ db) & vb;                                   // Straight
        } else if (phase == 1) {
            masked = false;                                        // Greedy
        } else {
            tt++;
            if (tt == 1) cursor = 0;                               // main run starts
            if (algo == ALG_CYCLIC) {                              // CyclicMin (R-7)
                const int w = p.wtab[tt];
                const int b0 = min(cursor + w, n), b1 = cursor + w - n;
                bits_t wm = 0;
#pragma unroll
                for (int c = 0; c < C; c++) {
                    // uniform: does the window meet chunk c at all (its span is NT*8 elements)?
                    const int s0 = (c << lgNTG) << 3, s1 = s0 + (NTG << 3);
                    if ((cursor < s1 && b0 > s0) || b1 > s0) {
                        const int base = gidx(c, 0);
                        const int lo = max(cursor - base, 0), hi = min(b0 - base, 8);
                        if (lo < hi) wm |= (bits_t)((((1u << (hi - lo)) - 1u) << lo)) << (8 * c);
                        const int hi2 = min(b1 - base, 8);
                        if (hi2 > 0) wm |= (bits_t)((1u << hi2) - 1u) << (8 * c);
                    }
                }
                cursor += w;                                       // w <= n: one conditional subtract
                if (cursor >= n) cursor -= n;
                M1 = wm & ~tm;
                M2 = wm;
                fb = 1;
            } else if (algo == ALG_RANDOM) {                       // RandomMin (R-8)
                const bits_t cand = (MW && pre_for == flips) ? cand_pre : rand_cand(tt, flips);
                M1 = cand & ~tm & vb;
                M2 = ~tm & vb;
                fb = 2;
            } else if (algo == ALG_TWO) {                          // TwoNeighbor (R-10)
                kind = 2;
                const int q = tt - 1;
                fixed_i = q == 0 ? 0 : ((q & 1) ? (q + 1) >> 1 : (q >> 1) - 1);
            } else {
                kind = 1;                                          // MaxMin / PositiveMin
            }
        }

        // ---------------- Step 1 + Step 2: scans and one exchange
        const bool skip_g = E + glb >= ebest;   // no 1-bit neighbour can beat BEST (uniform)
        int si = 0, sv = 0, sx = 0;     // selected bit, its Delta, its x (uniform)
        int gmin = 0, tg = INT32_MAX;
        int key = INT32_MAX;            // argmin key of the rule (kind 0)
        if (kind == 0) {
            int gm[C];
            int tsel = INT32_MAX;
            if (!masked) {
#pragma unroll
                for (int c = 0; c < C; c++) {
                    int mc = INT32_MAX;
#pragma unroll
                    for (int e = 0; e < 8; e++) mc = min(mc, d[8 * c + e]);
                    gm[c] = mc;
                    tg = min(tg, mc);
                }
                tsel = tg;
                M1 = ALL;
            } else {
                if (!skip_g) tg = min_all(d);
#pragma unroll
                for (int c = 0; c < C; c++) gm[c] = INT32_MAX;
                if (__any_sync(FULL, M1 != 0)) {      // warps without candidates skip
#pragma unroll
                    for (int c = 0; c < C; c++) {
                        int mc = INT32_MAX;
#pragma unroll
                        for (int e = 0; e < 8; e++)
                            if ((M1 >> (8 * c + e)) & 1) mc = min(mc, d[8 * c + e]);
                        gm[c] = mc;
                        tsel = min(tsel, mc);
                    }
                }
            }
            // warp argmin with a lazy key: only the lane(s) holding the minimum search
            const int wmin = warp_min(tsel);
            int k = INT32_MAX;
            if (__any_sync(FULL, tsel == wmin && wmin != INT32_MAX)) {
                if (tsel == wmin && wmin != INT32_MAX) {
                    int cs = 0;
#pragma unroll
                    for (int c = C - 1; c >= 0; c--)
                        if (gm[c] == wmin) cs = c;
                    const int e = first_in_chunk(d, M1, cs, wmin);
                    k = (gidx(cs, e) << 1) | (int)((xb >> (8 * cs + e)) & 1);
                }
            }
            k = warp_min(k);
            int g = warp_min(tg);
            int m;
            if constexpr (MW) {
                const int par = rc & 1;
                rc++;
                if (lane == 0) { red_s[par][wid][0] = wmin; red_s[par][wid][1] = k; red_s[par][wid][2] = g; }
                __syncthreads();
                const int a = lane < NW ? red_s[par][lane][0] : INT32_MAX;
                const int b = lane < NW ? red_s[par][lane][1] : INT32_MAX;
                const int c2 = lane < NW ? red_s[par][lane][2] : INT32_MAX;
                m = warp_min(a);
                key = warp_min(a == m ? b : INT32_MAX);
                gmin = warp_min(c2);
                if constexpr (CL == 2) {
                    const int mine[3] = {m, key, gmin};
                    int o[3];
                    cl_swap<3>(mine, o, xv_s, xbar, xc, peer, t);
                    const int m2 = min(m, o[0]);
                    key = min(m == m2 ? key : INT32_MAX, o[0] == m2 ? o[1] : INT32_MAX);
                    m = m2;
                    gmin = min(gmin, o[2]);
                }
            } else {
                m = wmin;
                key = k;
                gmin = g;
            }
            if (m == INT32_MAX) {
                if (phase == 0) {                   // X == D: Straight ends (no scan, R-3)
                    phase = 1;
                    after_main = false;
                    continue;
                }
                // empty candidate set (R-7, R-8, R-11): argmin over M2, then over all bits
                int t2 = INT32_MAX;
#pragma unroll
                for (int kk = 0; kk < EPT; kk++)
                    if ((M2 >> kk) & 1) t2 = min(t2, d[kk]);
                int v2[1] = {t2};
                const int ops1[1] = {OP_MIN};
                block_reduce<MW>(v2, ops1, red_s, rc, lane, wid, NW);
                cl_combine(v2, ops1);
                bits_t MM = M2;
                if (v2[0] == INT32_MAX) {
                    if (skip_g) {                   // exact global minimum needed after all
                        tg = min_all(d);
                        int v3[1] = {tg};
                        block_reduce<MW>(v3, ops1, red_s, rc, lane, wid, NW);
                        cl_combine(v3, ops1);
                        gmin = v3[0];
                    }
                    MM = vb; t2 = tg; v2[0] = gmin;
                }
                m = v2[0];
                int k2 = INT32_MAX;
                if (__any_sync(FULL, t2 == m))
                    if (t2 == m) {
#pragma unroll
                        for (int c = C - 1; c >= 0; c--)
#pragma unroll
                            for (int e = 7; e >= 0; e--) {
                                const int kk = 8 * c + e;
                                if (((MM >> kk) & 1) && d[kk] == m) k2 = (gidx(c, e) << 1) | (int)((xb >> kk) & 1);
                            }
                    }
                int kv[1] = {k2};
                block_reduce<MW>(kv, ops1, red_s, rc, lane, wid, NW);
                cl_combine(kv, ops1);
                key = kv[0];
            }
            si = key >> 1;
            sx = key & 1;
            sv = m;
        } else if (kind == 2) {
            // TwoNeighbor: scan, and the owner of fixed_i publishes Delta_i and x_i
            if (!skip_g) tg = min_all(d);
            int ov = 0, ox = 0;
            const bool own = owns(fixed_i);
            if (__any_sync(FULL, own)) {
                if (own) {
                    ov = get_at(d, lbit(fixed_i));
                    ox = (int)((xb >> lbit(fixed_i)) & 1);
                }
            }
            if constexpr (MW) {
                if (own) { bc_s[rc & 1][0] = ov; bc_s[rc & 1][1] = ox; }
            }
            int v[1] = {tg};
            const int ops[1] = {OP_MIN};
            block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
            if constexpr (MW) {
                ov = bc_s[(rc - 1) & 1][0];
                ox = bc_s[(rc - 1) & 1][1];
                if constexpr (CL == 2) {
                    // the owner of fixed_i is in one CTA of the two
                    const bool own_cta = (((fixed_i >> 3) & (NTG - 1)) >> lgNT) == (int)rank;
                    int w3[3] = {v[0], own_cta ? ov : 0, own_cta ? ox : 0};
                    const int ops3[3] = {OP_MIN, OP_ADD, OP_ADD};
                    cl_combine(w3, ops3);
                    v[0] = w3[0]; ov = w3[1]; ox = w3[2];
                }
            } else {
                const int src = (fixed_i >> 3) & 31;
                ov = __shfl_sync(FULL, ov, src);
                ox = __shfl_sync(FULL, ox, src);
            }
            gmin = v[0];
            si = fixed_i; sv = ov; sx = ox;
        } else {
            // MaxMin (R-6) / PositiveMin (R-9)
            const bits_t el = ~tm & vb;
            const bool lane_plain = (el == ALL);        // no tabu bit, no padding in this lane
            int a1 = INT32_MAX, a2 = INT32_MIN;         // MaxMin: lo, hi; PositiveMin: pm, unused
            if (algo == ALG_MAXMIN) {
                if (__all_sync(FULL, lane_plain)) {
                    int m4[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
                    int x4[4] = {INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN};
#pragma unroll
                    for (int kk = 0; kk < EPT; kk++) { m4[kk & 3] = min(m4[kk & 3], d[kk]); x4[kk & 3] = max(x4[kk & 3], d[kk]); }
                    tg = min(min(m4[0], m4[1]), min(m4[2], m4[3]));
                    a2 = max(max(x4[0], x4[1]), max(x4[2], x4[3]));
                    a1 = tg;
                } else {
#pragma unroll
                    for (int kk = 0; kk < EPT; kk++) {
                        tg = min(tg, d[kk]);
                        if ((el >> kk) & 1) { a1 = min(a1, d[kk]); a2 = max(a2, d[kk]); }
                    }
                }
            } else {
                unsigned tp = 0xFFFFFFFFu;   // min over eligible positive Delta as (Delta - 1), unsigned
                if (__all_sync(FULL, (el | ~vb) == ALL)) {
                    unsigned p4[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
#pragma unroll
                    for (int kk = 0; kk < EPT; kk++) p4[kk & 3] = min(p4[kk & 3], (unsigned)(d[kk] - 1));
                    tp = min(min(p4[0], p4[1]), min(p4[2], p4[3]));
                    if (!skip_g) tg = min_all(d);
                } else {
#pragma unroll
                    for (int kk = 0; kk < EPT; kk++) {
                        tg = min(tg, d[kk]);
                        if ((el >> kk) & 1) tp = min(tp, (unsigned)(d[kk] - 1));
                    }
                }
                a1 = tp < 0x7FFFFFFEu ? (int)tp + 1 : INT32_MAX;   // pads / non-positive never count
            }
            int v[4] = {tg, a1, a2, el != 0};
            const int ops[4] = {OP_MIN, OP_MIN, OP_MAX, OP_OR};
            DABS_TS(0);
            block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
            cl_combine(v, ops);
            DABS_TS(1);
            gmin = v[0];
            bits_t EL = el;
            int thr;
            const uint2 r = draw(flips);
            if (!v[3]) {
                // every bit tabu: drop tabu (R-11)
                EL = vb;
                int b1 = INT32_MIN;
                unsigned b2 = 0xFFFFFFFFu;
#pragma unroll
                for (int kk = 0; kk < EPT; kk++)
                    if ((vb >> kk) & 1) { b1 = max(b1, d[kk]); b2 = min(b2, (unsigned)(d[kk] - 1)); }
                int w2[2] = {b1, b2 < 0x7FFFFFFEu ? (int)b2 + 1 : INT32_MAX};
                const int ops2[2] = {OP_MAX, OP_MIN};
                block_reduce<MW>(w2, ops2, red_s, rc, lane, wid, NW);
                cl_combine(w2, ops2);
                v[1] = algo == ALG_MAXMIN ? gmin : w2[1];
                v[2] = w2[0];
            }
            uint32_t u;
            if (algo == ALG_MAXMIN) {
                const uint64_t uu = (uint64_t)(T - tt);
                const uint64_t span = muldiv_floor((uint64_t)((int64_t)v[2] - v[1]), uu * uu * uu,
                                                   (uint64_t)T * T * T, p.invT3);
                thr = (int)((int64_t)v[1] + (int64_t)(((unsigned __int128)r.x * (span + 1)) >> 32));
                u = r.y;
            } else {
                thr = v[1];                               // INT32_MAX = "+inf": all eligible
                u = r.x;
            }
            // count candidates (Delta <= thr, eligible) per chunk, packed 2 x 16 bits per word
            DABS_TS(2);
            uint32_t pk[CW];
#pragma unroll
            for (int w = 0; w < CW; w++) pk[w] = 0;
            if (__all_sync(FULL, EL == ALL)) {
#pragma unroll
                for (int c = 0; c < C; c++) {
                    uint32_t cnt = 0;
#pragma unroll
                    for (int e = 0; e < 8; e++) cnt += (uint32_t)(d[8 * c + e] <= thr);
                    pk[c >> 1] += cnt << (16 * (c & 1));
                }
            } else {
#pragma unroll
                for (int c = 0; c < C; c++) {
                    uint32_t byte = 0;
#pragma unroll
                    for (int e = 0; e < 8; e++) byte |= (uint32_t)(d[8 * c + e] <= thr) << e;
                    byte &= (uint32_t)(EL >> (8 * c)) & 0xFFu;
                    pk[c >> 1] += (uint32_t)__popc(byte) << (16 * (c & 1));
                }
            }
            DABS_TS(3);
            uint32_t wt[CW];
#pragma unroll
            for (int w = 0; w < CW; w++) wt[w] = warp_add(pk[w]);
            uint32_t bt[CW];
            int par = 0;
            if constexpr (MW) {
                par = rc & 1;
                rc++;
                if (lane == 0) {
#pragma unroll
                    for (int w = 0; w < CW; w++) red_s[par][wid][w] = (int)wt[w];
                }
                __syncthreads();
#pragma unroll
                for (int w = 0; w < CW; w++) bt[w] = warp_add(lane < NW ? (uint32_t)red_s[par][lane][w] : 0u);
            } else {
#pragma unroll
                for (int w = 0; w < CW; w++) bt[w] = wt[w];
            }
            // chunk-major order: chunk 0 of all threads, then chunk 1, ...
            // (CL = 2: within a chunk, CTA 0's threads come before CTA 1's)
            uint32_t bo[CW];                      // the peer CTA's counts
#pragma unroll
            for (int w = 0; w < CW; w++) bo[w] = 0;
            if constexpr (CL == 2) {
                int mine[CW], o[CW];
#pragma unroll
                for (int w = 0; w < CW; w++) mine[w] = (int)bt[w];
                cl_swap<CW>(mine, o, xv_s, xbar, xc, peer, t);
#pragma unroll
                for (int w = 0; w < CW; w++) bo[w] = (uint32_t)o[w];
            }
            DABS_TS(4);
            uint32_t tot = 0;
#pragma unroll
            for (int c = 0; c < C; c++)
                tot += ((bt[c >> 1] >> (16 * (c & 1))) & 0xFFFFu) + ((bo[c >> 1] >> (16 * (c & 1))) & 0xFFFFu);
            int r1 = (int)pick_u(u, tot);
            int cs = 0;
#pragma unroll
            for (int c = 0; c < C; c++) {
                const int tc = (int)(((bt[c >> 1] >> (16 * (c & 1))) & 0xFFFFu) + ((bo[c >> 1] >> (16 * (c & 1))) & 0xFFFFu));
                if (cs == c && r1 >= tc) { r1 -= tc; cs = c + 1; }
            }
            bool locate = true;                   // does this CTA hold rank r1 of chunk cs?
            if constexpr (CL == 2) {
                uint32_t mc = 0, oc = 0;
#pragma unroll
                for (int c = 0; c < C; c++)
                    if (c == cs) {
                        mc = (bt[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                        oc = (bo[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                    }
                const int c0 = (int)(rank == 0 ? mc : oc);
                if (rank == 0) locate = r1 < c0;
                else { locate = r1 >= c0; r1 -= c0; }
            }
            // which warp holds rank r1 of chunk cs
            DABS_TS(5);
            int wsel = locate ? 0 : -1;
            if (MW && locate) {
                // every warp: the chunk-cs count of the warps before it (one redux)
                // and its own; the warp whose range holds rank r1 locates it
                const int x = lane < NW ? (int)(((uint32_t)red_s[par][lane][cs >> 1] >> (16 * (cs & 1))) & 0xFFFFu) : 0;
                const int pre = (int)warp_add(lane < wid ? (uint32_t)x : 0u);
                const int own = __shfl_sync(FULL, x, wid);
                wsel = (r1 >= pre && r1 < pre + own) ? wid : -1;
                r1 -= pre;
            }
            DABS_TS(6);
            int gi = -1, lv = 0, lx = 0;
            if (wid == wsel) {
                uint32_t mybyte = 0;
                switch (cs) {
#define DABS_MYBYTE(cc)                                                                           \
    case cc:                                                                                      \
        if constexpr (cc < C) {                                                                   \
            _Pragma("unroll") for (int e = 0; e < 8; e++) mybyte |= (uint32_t)(d[8 * cc + e] <= thr) << e; \
            mybyte &= (uint32_t)(EL >> (8 * cc)) & 0xFFu;                                         \
        }                                                                                         \
        break;
                    DABS_MYBYTE(0) DABS_MYBYTE(1) DABS_MYBYTE(2) DABS_MYBYTE(3)
                    DABS_MYBYTE(4) DABS_MYBYTE(5) DABS_MYBYTE(6) DABS_MYBYTE(7)
#undef DABS_MYBYTE
                default: break;
                }
                // rank of this lane's first candidate in index order (lane-major,
                // then element): per-bit ballots instead of a shuffle scan
                const uint32_t lt = (1u << lane) - 1u;
                int y0 = 0;
#pragma unroll
                for (int e = 0; e < 8; e++) y0 += __popc(__ballot_sync(FULL, (mybyte >> e) & 1u) & lt);
                const int x = __popc(mybyte);
                if (r1 >= y0 && r1 < y0 + x) {
                    uint32_t byte = mybyte;
                    for (int j = 0; j < r1 - y0; j++) byte &= byte - 1;
                    const int e = __ffs(byte) - 1;
                    const int li = 8 * cs + e;
                    gi = gidx(cs, e);
                    lv = get_at(d, li);
                    lx = (int)((xb >> li) & 1);
                }
            }
            if constexpr (CL == 2) {
                // the pick is in one CTA: one more reduction + swap makes it uniform
                int q3[3] = {gi, gi >= 0 ? lv : 0, gi >= 0 ? lx : 0};
                const int ops3[3] = {OP_MAX, OP_ADD, OP_ADD};
                block_reduce<MW>(q3, ops3, red_s, rc, lane, wid, NW);
                cl_combine(q3, ops3);
                si = q3[0]; sv = q3[1]; sx = q3[2];
            } else if constexpr (MW) {
                // the locating thread publishes the pick and starts the row copy
                // itself; everybody else learns (i, Delta_i, x_i) from the row's
                // mbarrier (arrive = release, try_wait = acquire): no CTA barrier
                if (gi >= 0) {
                    sel_s[0] = gi; sel_s[1] = lv; sel_s[2] = lx;
                    issue_row(gi);
                }
            } else {
                const int src = __ffs(__ballot_sync(FULL, gi >= 0)) - 1;
                si = __shfl_sync(FULL, gi, src);
                sv = __shfl_sync(FULL, lv, src);
                sx = __shfl_sync(FULL, lx, src);
            }
        }

        // ---------------- Step 1: BEST (R-2, R-3)
        const bool g_exact = !skip_g || phase == 1 || (kind == 1 && algo == ALG_MAXMIN);
        if (g_exact) glb = gmin;
        else gmin = INT32_MAX;                  // not computed: cannot improve BEST
        if (E + gmin < ebest) {
            int bk = key;
            if (kind != 0 || masked) {
                // key of the lowest index holding gmin (rare: BEST improves)
                int k3 = INT32_MAX;
                if (__any_sync(FULL, tg == gmin))
                    if (tg == gmin) {
#pragma unroll
                        for (int c = C - 1; c >= 0; c--)
#pragma unroll
                            for (int e = 7; e >= 0; e--) {
                                const int kk = 8 * c + e;
                                if (d[kk] == gmin) k3 = (gidx(c, e) << 1) | (int)((xb >> kk) & 1);
                            }
                    }
                int kv[1] = {k3};
                const int ops1[1] = {OP_MIN};
                block_reduce<MW>(kv, ops1, red_s, rc, lane, wid, NW);
                cl_combine(kv, ops1);
                bk = kv[0];
            }
            ebest = E + gmin;
            const int j = bk >> 1;
            bdiff = owns(j) ? (ONE << lbit(j)) : (bits_t)0;
        }
        if (phase == 1 && gmin >= 0) {
            // Greedy reached a local minimum (R-4): next round, or the batch ends (R-12)
            if (after_main && (algo == ALG_TWO || flips >= p.B)) break;
            if (after_main) round++;
            phase = 2;
            tt = 0;
            continue;
        }

        // ---------------- Step 3: flip bit si, Eqs.(4)-(5)
#ifdef DABS_TIMING
        tB = clock64();
        tbk = phase == 2 ? algo : 5;
        if (t == 0 && rank == 0) { ts_s[tbk][0] += tB - tA; ts_s[tbk][3] += tA - tD; ts_s[tbk][4] += 1; }
#endif
        // every thread has passed the last exchange: the row buffer is free
        const bool pre_issued = MW && CL == 1 && kind == 1;
        // warp tier: every lane has consumed the previous row (explicit for racecheck;
        // the shuffles of the selection already order it)
        if constexpr (!MW) __syncwarp();
        if (pre_issued) {
            mbar_wait(&mbar[0], par_row);
            DABS_TS(7);
            si = sel_s[0]; sv = sel_s[1]; sx = sel_s[2];
        } else if (t == 0) {
            issue_row(si);
        }
        E += sv;
        const int rmax_si = p.rmax[si];   // consumed after the update: its latency hides there
        // sigma(x_i) = -1 (x_i = 0 before the flip): negate every sigma(x_k) byte
        const uint32_t cmask = sx ? 0u : 0xFEFEFEFEu;
        const uint4* sgn = sgs + (sx ? 0 : SGC);   // CTA tiers: the sign copy for sigma(x_i)
        if (__any_sync(FULL, owns(si))) {
            if (owns(si)) {
                const int kk = lbit(si);
                if constexpr (MW) {
                    neg_at(d, kk);               // Eq.(5); W_ii = 0, so the update leaves Delta_i alone
                    // sigma(x_k) byte of element kk in both sign copies
                    uint8_t* b8 = reinterpret_cast<uint8_t*>(sgs);
                    const int g = kk >> 2;
                    const int off = ((((g >> 2) << lgNT) + t) * 4 + (g & 3)) * 4 + (kk & 3);
                    b8[off] ^= 0xFEu;
                    b8[off + SGC * 16] ^= 0xFEu;
                } else {
                    if constexpr (WLUT) neg_at(d, kk);
                    else owner_flip(d, sg, kk);  // Eq.(5); W_ii = 0, so the update leaves Delta_i alone
                }
                xb ^= ONE << kk;
                bdiff ^= ONE << kk;
            }
        }
        pos = (pos + TABU_RING - 1) & (TABU_RING - 1);
        ring_s[pos] = si;
        if constexpr (!MW) __syncwarp();
        if (tabu > 0) {
            // tabu window (R-11): si enters, the (tabu+1)-th most recent flip leaves
            if (owns(si)) { tcnt[lidx(si)]++; tm |= ONE << lbit(si); }
            const int r = ring_s[(pos + tabu) & (TABU_RING - 1)];
            if (r >= 0 && owns(r) && --tcnt[lidx(r)] == 0) tm &= ~(ONE << lbit(r));
        }
        if constexpr (TRACE) {
            if (tq == 0 && s == p.trace_slot && flips < p.tr_cap) {
                p.tr_bit[flips] = si;
                p.tr_E[flips] = E;
                p.tr_phase[flips] = (int8_t)(phase == 2 ? 2 + min(round, 100) : phase);
            }
        }
        flips++;
        if constexpr (MW) {
            if (phase == 2 && tt < T && algo == ALG_RANDOM) {
                cand_pre = rand_cand(tt + 1, flips);
                pre_for = flips;
            }
        }
#pragma unroll
        for (int qq = 0; qq < NP; qq++) {
            mbar_wait(&mbar[qq], par_row);
#ifdef DABS_TIMING
            if (qq == 0) tC = clock64();
#endif
            uint4 rw[CPP];
#pragma unroll
            for (int cc = 0; cc < CPP; cc++) rw[cc] = row_s[((qq * CPP + cc) << lgNT) + t];
            if constexpr (MW) {
                uint4 sw[(CPP + 1) / 2];
#pragma unroll
                for (int j = 0; j < (CPP + 1) / 2; j++) sw[j] = sgn[(((qq * CPP) / 2 + j) << lgNT) + t];
#pragma unroll
                for (int cc = 0; cc < CPP; cc++) {
                    const int c = qq * CPP + cc;
                    // Eq.(4): Delta_k += W_ik sigma(x_i) sigma(x_k); the row word holds
                    // (W_i,k0, W_i,k1) as int16x2, B holds (+-s_k0, 0, 0, +-s_k1) as int8x4
                    const uint4 q4 = sw[cc >> 1];
                    const uint32_t g0 = (c & 1) ? q4.z : q4.x, g1 = (c & 1) ? q4.w : q4.y;
                    const uint32_t B0 = __byte_perm(g0, 0, 0x1440), B1 = __byte_perm(g0, 0, 0x3442);
                    const uint32_t B2 = __byte_perm(g1, 0, 0x1440), B3 = __byte_perm(g1, 0, 0x3442);
                    d[8 * c + 0] = __dp2a_lo((int)rw[cc].x, (int)B0, d[8 * c + 0]);
                    d[8 * c + 1] = __dp2a_hi((int)rw[cc].x, (int)B0, d[8 * c + 1]);
                    d[8 * c + 2] = __dp2a_lo((int)rw[cc].y, (int)B1, d[8 * c + 2]);
                    d[8 * c + 3] = __dp2a_hi((int)rw[cc].y, (int)B1, d[8 * c + 3]);
                    d[8 * c + 4] = __dp2a_lo((int)rw[cc].z, (int)B2, d[8 * c + 4]);
                    d[8 * c + 5] = __dp2a_hi((int)rw[cc].z, (int)B2, d[8 * c + 5]);
                    d[8 * c + 6] = __dp2a_lo((int)rw[cc].w, (int)B3, d[8 * c + 6]);
                    d[8 * c + 7] = __dp2a_hi((int)rw[cc].w, (int)B3, d[8 * c + 7]);
                }
            } else {
#pragma unroll
                for (int cc = 0; cc < CPP; cc++) {
                    const int c = qq * CPP + cc;
                    // Eq.(4) as above; B holds (s_k0, 0, 0, s_k1) as int8x4, byte-permuted here
                    uint32_t B0, B1, B2, B3;
                    if constexpr (WLUT) {
                        const uint4 Bq = lutw_s[(uint32_t)((xb >> (8 * c)) & 0xFFu) ^ (cmask ? 0xFFu : 0u)];
                        B0 = Bq.x; B1 = Bq.y; B2 = Bq.z; B3 = Bq.w;
                    } else {
                        const uint32_t g0 = sg[2 * c] ^ cmask, g1 = sg[2 * c + 1] ^ cmask;
                        B0 = __byte_perm(g0, 0, 0x1440); B1 = __byte_perm(g0, 0, 0x3442);
                        B2 = __byte_perm(g1, 0, 0x1440); B3 = __byte_perm(g1, 0, 0x3442);
                    }
                    d[8 * c + 0] = __dp2a_lo((int)rw[cc].x, (int)B0, d[8 * c + 0]);
                    d[8 * c + 1] = __dp2a_hi((int)rw[cc].x, (int)B0, d[8 * c + 1]);
                    d[8 * c + 2] = __dp2a_lo((int)rw[cc].y, (int)B1, d[8 * c + 2]);
                    d[8 * c + 3] = __dp2a_hi((int)rw[cc].y, (int)B1, d[8 * c + 3]);
                    d[8 * c + 4] = __dp2a_lo((int)rw[cc].z, (int)B2, d[8 * c + 4]);
                    d[8 * c + 5] = __dp2a_hi((int)rw[cc].z, (int)B2, d[8 * c + 5]);
                    d[8 * c + 6] = __dp2a_lo((int)rw[cc].w, (int)B3, d[8 * c + 6]);
                    d[8 * c + 7] = __dp2a_hi((int)rw[cc].w, (int)B3, d[8 * c + 7]);
                }
            }
        }
#ifdef DABS_TIMING
        tD = clock64();
        if (t == 0 && rank == 0) { ts_s[tbk][1] += tC - tB; ts_s[tbk][2] += tD - tC; }
#endif
        par_row ^= 1u;
        glb = min(glb - (int64_t)rmax_si, (int64_t)-sv);
    }

    // ---------------- write back state and the result packet
    {
        uint8_t* Xb = reinterpret_cast<uint8_t*>(p.X + (size_t)s * p.nwp);
        uint8_t* Bb = reinterpret_cast<uint8_t*>(p.best + (size_t)s * p.nwp);
        int32_t* dp = p.delta + (size_t)s * p.n_pad;
        const bits_t bb = xb ^ bdiff;
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int ch = (c << lgNTG) + tq;
            Xb[ch] = (uint8_t)(xb >> (8 * c));
            Bb[ch] = (uint8_t)(bb >> (8 * c));
            reinterpret_cast<int4*>(dp + ch * 8)[0] = make_int4(d[8 * c], d[8 * c + 1], d[8 * c + 2], d[8 * c + 3]);
            reinterpret_cast<int4*>(dp + ch * 8)[1] = make_int4(d[8 * c + 4], d[8 * c + 5], d[8 * c + 6], d[8 * c + 7]);
        }
        if (tq < TABU_RING) p.ring[(size_t)s * TABU_RING + t] = ring_s[(pos + t) & (TABU_RING - 1)];
        if (tq == 0) {
            p.E[s] = E;
            p.ebest[s] = ebest;
            p.flips[s] = flips;
            atomicAdd(p.flip_total, (unsigned long long)flips);
        }
    }
#ifdef DABS_TIMING
    if (t == 0 && rank == 0)
        for (int j = 0; j < 30; j++) atomicAdd(&g_tstat[0][0] + j, (unsigned long long)(&ts_s[0][0])[j]);
    if (t == 0 && rank == 0)
        for (int j = 0; j < 10; j++) atomicAdd(&g_tstat2[j], (unsigned long long)ts2_s[j]);
#endif
    if constexpr (CL == 2) cluster_sync_all();   // no CTA leaves while its peer may still write to it
    if constexpr (REUSE) {
        if constexpr (MW) __syncthreads(); else __syncwarp();
        if (t == 0) {
            if constexpr (KEEP) {
                par_keep = par_row;
            } else {
#pragma unroll
                for (int qq = 0; qq < NP; qq++) mbar_inval(&mbar[qq]);
                mbar_inval(&xbar[0]);
                mbar_inval(&xbar[1]);
            }
        }
    }
}

// Warp tier: minimum resident searches per SM, i.e. a register cap.  The tier
// is issue/latency bound, more resident warps beat the few spills the cap
// costs (A/B on B200, tools/gpu_ab_libs.sh: uncapped 167 / 128 registers ->
// 128 / 80: K2000s +13 %, TSP32 +7 %, GS800 +6 % flips/s).
#ifndef DABS_MINB8
#define DABS_MINB8 16   // C = 8 (1024 < n <= 2048): 128 registers, 16 searches per SM
#endif
#ifndef DABS_MINB4
#define DABS_MINB4 24   // C = 4 (512 < n <= 1024): 80 registers, 24 searches per SM
#endif
template <int C, int NTT, int CL>
constexpr int batch_min_blocks()
{
    return (CL == 2 && NTT <= 256) ? 2 : (NTT == 32 && C == 8) ? DABS_MINB8 : (NTT == 32 && C == 4) ? DABS_MINB4 : 0;
}

template <int C, int NTT, int CL, bool TRACE>
__global__ void __launch_bounds__(NTT, batch_min_blocks<C, NTT, CL>()) batch_kernel(const BatchParams p)
{
    const int sidx = (int)blockIdx.x / CL;
    const int s = p.order ? p.order[sidx] : p.slot0 + sidx;
    batch_body<C, NTT, CL, TRACE, false>(p, s, p.gen_ptr ? *p.gen_ptr : p.gen);
}

}  // namespace dabs
