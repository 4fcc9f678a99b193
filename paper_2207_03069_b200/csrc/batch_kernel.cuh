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
    int n, n_pad, nwp;       // nwp = n_pad / 32 words per bit vector
    int T, B, tabu;
    uint64_t seed;
    uint32_t gen;
    uint32_t slot_base;      // global id of local slot 0
    int slot0;               // first local slot of this launch (blockIdx.x offset)
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

template <int C, bool MW, bool TRACE>
__global__ void __launch_bounds__(MW ? 512 : 32) batch_kernel(const BatchParams p)
{
    constexpr int EPT = 8 * C;
    constexpr int NP = MW ? (C >= 4 ? 4 : C) : 1;   // row pieces, one mbarrier each
    constexpr int CPP = C / NP;                      // chunks per piece
    using bits_t = typename std::conditional<(EPT > 32), unsigned long long, uint32_t>::type;
    constexpr bits_t ONE = 1;
    const int t = threadIdx.x;
    const int NT = MW ? (int)blockDim.x : 32;
    const int lgNT = 31 - __clz(NT);
    const int lane = t & 31, wid = t >> 5, NW = NT >> 5;
    const int s = p.slot0 + (int)blockIdx.x;
    const uint32_t gslot = p.slot_base + (uint32_t)s;
    const int n = p.n;

    extern __shared__ __align__(128) uint8_t dyn_smem[];
    const uint4* row_s = reinterpret_cast<const uint4*>(dyn_smem);   // one W row, 2*n_pad bytes
    __shared__ __align__(8) uint64_t mbar[NP];
    __shared__ int32_t ring_s[TABU_RING];
    __shared__ int32_t red_s[2][32][RED_W];
    __shared__ int32_t bc_s[2][4];

    // ---------------- load the slot's persistent state (R-14)
    int32_t d[EPT];
    bits_t xb = 0, db = 0, vb = 0;
    {
        const uint8_t* Xb = reinterpret_cast<const uint8_t*>(p.X + (size_t)s * p.nwp);
        const uint8_t* Db = reinterpret_cast<const uint8_t*>(p.D + (size_t)s * p.nwp);
        const int32_t* dp = p.delta + (size_t)s * p.n_pad;
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int ch = (c << lgNT) + t;
            xb |= (bits_t)Xb[ch] << (8 * c);
            db |= (bits_t)Db[ch] << (8 * c);
            const int nv = min(max(n - ch * 8, 0), 8);
            vb |= (bits_t)((1u << nv) - 1u) << (8 * c);
            const int4 a = reinterpret_cast<const int4*>(dp + ch * 8)[0];
            const int4 b = reinterpret_cast<const int4*>(dp + ch * 8)[1];
            d[8 * c + 0] = a.x; d[8 * c + 1] = a.y; d[8 * c + 2] = a.z; d[8 * c + 3] = a.w;
            d[8 * c + 4] = b.x; d[8 * c + 5] = b.y; d[8 * c + 6] = b.z; d[8 * c + 7] = b.w;
        }
    }
    if (t < TABU_RING) ring_s[t] = p.ring[(size_t)s * TABU_RING + t];
    if (t == 0) {
#pragma unroll
        for (int q = 0; q < NP; q++) mbar_init(&mbar[q], 1);
        fence_mbar_init();
    }
    int pos = 0;   // ring_s[(pos + j) & 31] = j-th most recent flip
    int64_t E = p.E[s];
    const int algo = p.algo[s];
    const uint32_t piece_bytes = (uint32_t)(2 * p.n_pad / NP);
    const char* Wbytes = reinterpret_cast<const char*>(p.W);
    uint32_t par_row = 0;
    if constexpr (MW) __syncthreads(); else __syncwarp();

    auto gidx = [&](int c, int e) { return (((c << lgNT) + t) << 3) | e; };
    auto owns = [&](int k) { return ((k >> 3) & (NT - 1)) == t; };
    auto lbit = [&](int k) { return (((k >> 3) >> lgNT) << 3) | (k & 7); };

    // lowest (index<<1 | x) among this thread's elements in M with d == m (full scan; rare use)
    auto first_key_full = [&](bits_t M, int m) -> int {
        int key = INT32_MAX;
#pragma unroll
        for (int c = C - 1; c >= 0; c--) {
#pragma unroll
            for (int e = 7; e >= 0; e--) {
                const int k = 8 * c + e;
                if (((M >> k) & 1) && d[k] == m) key = (gidx(c, e) << 1) | (int)((xb >> k) & 1);
            }
        }
        return key;
    };
    // key of the first element with value m, given per-chunk minima gm[] (one lane runs it)
    auto key_from_chunks = [&](const int (&gm)[C], bits_t M, int m) -> int {
        int cs = 0;
#pragma unroll
        for (int c = C - 1; c >= 0; c--)
            if (gm[c] == m) cs = c;
        const int e = first_in_chunk(d, M, cs, m);
        const int k = 8 * cs + e;
        return (gidx(cs, e) << 1) | (int)((xb >> k) & 1);
    };
    // tabu set = the last `tabu` flips (R-11)
    auto tabu_mask = [&]() -> bits_t {
        bits_t m = 0;
        for (int j = 0; j < p.tabu; j++) {
            const int r = ring_s[(pos + j) & (TABU_RING - 1)];
            if (r >= 0 && owns(r)) m |= ONE << lbit(r);
        }
        return m;
    };

    int phase = 0;                 // 0 Straight, 1 Greedy, 2 main, 3 done
    bool after_main = false;
    int round = 0, tt = 0, cursor = 0, q = 0;
    int flips = 0;
    int64_t ebest = E_INF;
    bits_t bdiff = 0;              // BEST = X xor bdiff
    int rc = 0;

    auto set_best = [&](int key, int m) {
        ebest = E + m;
        const int j = key >> 1;
        bdiff = owns(j) ? (ONE << lbit(j)) : (bits_t)0;
    };
    auto end_phase = [&]() {
        if (phase == 0) {
            phase = 1;
            after_main = false;
        } else if (phase == 1) {
            if (after_main && (algo == ALG_TWO || flips >= p.B)) {   // R-12
                phase = 3;
            } else {
                if (after_main) round++;
                phase = 2; tt = 0; cursor = 0; q = 0;
            }
        } else {
            phase = 1;
            after_main = true;
        }
    };

    // CTA-wide (min, key) reduction of K1 argmin pairs plus K2 plain values,
    // one exchange.  A pair is (tmin, key) where each thread contributes the
    // key of its first element at the warp minimum (computed lazily by the
    // lanes holding it).
    auto reduce_pairs = [&](int (&vmin)[2], int (&vkey)[2], int np_, int (&ext)[4], const int (&eops)[4],
                            int ne) {
        // warp stage (vmin already warp-reduced, vkey already computed by the caller)
#pragma unroll
        for (int k = 0; k < 2; k++)
            if (k < np_) vkey[k] = warp_min(vkey[k]);
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (k < ne) ext[k] = wop(eops[k], ext[k]);
        if constexpr (MW) {
            const int par = rc & 1;
            rc++;
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 2; k++)
                    if (k < np_) { red_s[par][wid][2 * k] = vmin[k]; red_s[par][wid][2 * k + 1] = vkey[k]; }
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if (k < ne) red_s[par][wid][4 + k] = ext[k];
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < 2; k++) {
                if (k < np_) {
                    const int a = lane < NW ? red_s[par][lane][2 * k] : INT32_MAX;
                    const int b = lane < NW ? red_s[par][lane][2 * k + 1] : INT32_MAX;
                    vmin[k] = warp_min(a);
                    vkey[k] = warp_min(a == vmin[k] ? b : INT32_MAX);
                }
            }
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (k < ne) ext[k] = wop(eops[k], lane < NW ? red_s[par][lane][4 + k] : op_ident(eops[k]));
        }
    };

    // count + uniform pick in index order (MaxMin R-6, PositiveMin R-9):
    // returns the pick via (si, sv, sx); kb = BEST key (lowest gmin index).
    auto locate_pick = [&](bits_t cb, uint32_t u, int kb_local, int& si, int& sv, int& sx, int& kb) {
        int incl[C];   // warp-inclusive prefix of this lane's candidate count, per chunk
#pragma unroll
        for (int c = 0; c < C; c++) {
            int x = __popc((uint32_t)((cb >> (8 * c)) & 0xFFu));
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            incl[c] = x;
        }
        int par = 0;
        if constexpr (MW) {
            par = rc & 1;
            rc++;
            const int kw = warp_min(kb_local);
            if (lane == 31) {
#pragma unroll
                for (int c = 0; c < C; c++) red_s[par][wid][c] = incl[c];
            }
            if (lane == 0) red_s[par][wid][RED_W - 1] = kw;
            __syncthreads();
            kb = warp_min(lane < NW ? red_s[par][lane][RED_W - 1] : INT32_MAX);
        } else {
            kb = warp_min(kb_local);
        }
        // chunk-major order: all of chunk 0 (thread order), then chunk 1, ...
        int tot = 0;
        int li = -1;
#pragma unroll
        for (int c = 0; c < C; c++) {
            int woff = 0, Tc;
            if constexpr (MW) {
                const int x = lane < NW ? red_s[par][lane][c] : 0;
                int y = x;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int z = __shfl_up_sync(0xffffffffu, y, off);
                    if (lane >= off) y += z;
                }
                woff = __shfl_sync(0xffffffffu, y - x, wid);
                Tc = __shfl_sync(0xffffffffu, y, 31);
            } else {
                Tc = __shfl_sync(0xffffffffu, incl[c], 31);
            }
            const int cnt = __popc((uint32_t)((cb >> (8 * c)) & 0xFFu));
            const int lo = tot + woff + incl[c] - cnt;
            incl[c] = lo;                          // reuse: start rank of this lane's chunk c
            tot += Tc;
        }
        const int r = (int)pick_u(u, (uint32_t)tot);
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int cnt = __popc((uint32_t)((cb >> (8 * c)) & 0xFFu));
            const int lo = incl[c];
            if (r >= lo && r < lo + cnt) {
                uint32_t byte = (uint32_t)((cb >> (8 * c)) & 0xFFu);
                for (int j = 0; j < r - lo; j++) byte &= byte - 1;   // drop lower set bits
                li = 8 * c + (__ffs(byte) - 1);
            }
        }
        int gi = -1, lv = 0, lx = 0;
        if (__any_sync(0xffffffffu, li >= 0)) {
            if (li >= 0) {
                gi = gidx(li >> 3, li & 7);
                lv = get_at(d, li);
                lx = (int)((xb >> li) & 1);
            }
        }
        if constexpr (MW) {
            const int par2 = rc & 1;
            rc++;
            if (li >= 0) { bc_s[par2][0] = gi; bc_s[par2][1] = lv; bc_s[par2][2] = lx; }
            __syncthreads();
            si = bc_s[par2][0]; sv = bc_s[par2][1]; sx = bc_s[par2][2];
        } else {
            const int src = __ffs(__ballot_sync(0xffffffffu, li >= 0)) - 1;
            si = __shfl_sync(0xffffffffu, gi, src);
            sv = __shfl_sync(0xffffffffu, lv, src);
            sx = __shfl_sync(0xffffffffu, lx, src);
        }
    };

    // lazy key of the global-min element for BEST (rare): lanes holding gmin
    auto best_key = [&](int tg, int gmin) -> int {
        int k = INT32_MAX;
        if (__any_sync(0xffffffffu, tg == gmin)) {
            if (tg == gmin) k = first_key_full(vb, gmin);
        }
        int v[1] = {k};
        const int ops[1] = {OP_MIN};
        block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
        return v[0];
    };

    while (true) {
        int si = -1, sv = 0, sx = 0;       // selected bit, its Delta, its x (uniform)
        if (phase == 3) break;

        // ---------------- Step 1 + Step 2 per phase
        if (phase == 1 || phase == 0 || (phase == 2 && (algo == ALG_CYCLIC || algo == ALG_RANDOM))) {
            // argmin rules: Greedy, Straight, CyclicMin
            // (R-7), RandomMin (R-8).  One exchange:
            // (rule min, key), (global min, -), flags.
            bits_t M1, M2 = 0;     // primary mask, fallback mask
            int fb_mode = 0;       // 0 none, 1 fallback to M2, 2 fallback M2 then all
            if (phase == 1) {
                M1 = vb;
            } else if (phase == 0) {
                M1 = (xb ^ db) & vb;
            } else {
                if (tt == p.T) { end_phase(); continue; }
                tt++;
                const bits_t tm = tabu_mask();
                if (algo == ALG_CYCLIC) {
                    const int w = p.wtab[tt];
                    const int b0 = min(cursor + w, n), b1 = cursor + w - n;
                    bits_t wm = 0;
#pragma unroll
                    for (int c = 0; c < C; c++) {
                        const int base = gidx(c, 0);
                        const int lo = max(cursor - base, 0), hi = min(b0 - base, 8);
                        if (lo < hi) wm |= (bits_t)((((1u << (hi - lo)) - 1u) << lo)) << (8 * c);
                        const int hi2 = min(b1 - base, 8);
                        if (hi2 > 0) wm |= (bits_t)((1u << hi2) - 1u) << (8 * c);
                    }
                    cursor = (cursor + w) % n;
                    M1 = wm & ~tm;
                    M2 = wm;
                    fb_mode = 1;
                } else {
                    const uint32_t p16 = (uint32_t)p.ptab[tt];
                    bits_t cand;
                    if (p16 >= 65536u) {
                        cand = vb;
                    } else {
                        cand = 0;
#pragma unroll
                        for (int c = 0; c < C; c++) {
                            const uint4 r = rng4(p.seed, PUR_RANDMIN, (uint32_t)((c << lgNT) + t), gslot,
                                                 p.gen, (uint32_t)flips);
                            const uint32_t wds[4] = {r.x, r.y, r.z, r.w};
                            uint32_t byte = 0;
#pragma unroll
                            for (int e = 0; e < 8; e++) {
                                const uint32_t u16 = (wds[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
                                byte |= (uint32_t)(u16 < p16) << e;
                            }
                            cand |= (bits_t)byte << (8 * c);
                        }
                    }
                    M1 = cand & ~tm & vb;
                    M2 = ~tm & vb;
                    fb_mode = 2;
                }
            }
            // scan: the global minimum (Step 1) and per-chunk minima of the
            // rule's candidate set M1 (Greedy: all bits).  Warps whose lanes
            // hold no candidate skip the masked scan (CyclicMin reads only its
            // window).  The fallback set M2 is scanned lazily.
            const bool use_g = (phase == 1);
            int gsel[C];
            int tg = INT32_MAX, t1 = INT32_MAX;
            if (use_g) {
#pragma unroll
                for (int c = 0; c < C; c++) {
                    int mg = INT32_MAX;
#pragma unroll
                    for (int e = 0; e < 8; e++) mg = min(mg, d[8 * c + e]);
                    gsel[c] = mg;
                    tg = min(tg, mg);
                }
                t1 = tg;
            } else {
#pragma unroll
                for (int k = 0; k < EPT; k++) tg = min(tg, d[k]);
#pragma unroll
                for (int c = 0; c < C; c++) gsel[c] = INT32_MAX;
                if (__any_sync(0xffffffffu, M1 != 0)) {
#pragma unroll
                    for (int c = 0; c < C; c++) {
                        int m1 = INT32_MAX;
#pragma unroll
                        for (int e = 0; e < 8; e++)
                            if ((M1 >> (8 * c + e)) & 1) m1 = min(m1, d[8 * c + e]);
                        gsel[c] = m1;
                        t1 = min(t1, m1);
                    }
                }
            }
            // warp minimum and lazy key (only the lanes holding it search)
            int vmin[2], vkey[2] = {INT32_MAX, INT32_MAX};
            vmin[0] = warp_min(t1);
            if (__any_sync(0xffffffffu, t1 == vmin[0] && vmin[0] != INT32_MAX))
                if (t1 == vmin[0] && vmin[0] != INT32_MAX)
                    vkey[0] = key_from_chunks(gsel, use_g ? ~(bits_t)0 : M1, vmin[0]);
            int ext[4] = {tg, 0, 0, 0};
            const int eops[4] = {OP_MIN, OP_MIN, OP_MIN, OP_MIN};
            reduce_pairs(vmin, vkey, 1, ext, eops, 1);
            const int gmin = ext[0];
            int m = vmin[0], key = vkey[0];
            if (m == INT32_MAX && fb_mode) {
                // empty candidate set: CyclicMin window all tabu (R-7) / RandomMin
                // with no candidate (R-8) -> argmin over M2 (then over all bits)
                int t2 = INT32_MAX;
#pragma unroll
                for (int k = 0; k < EPT; k++)
                    if ((M2 >> k) & 1) t2 = min(t2, d[k]);
                int v2[1] = {t2};
                const int ops1[1] = {OP_MIN};
                block_reduce<MW>(v2, ops1, red_s, rc, lane, wid, NW);
                if (v2[0] != INT32_MAX) {
                    m = v2[0];
                    int k2 = INT32_MAX;
                    if (__any_sync(0xffffffffu, t2 == m))
                        if (t2 == m) k2 = first_key_full(M2, m);
                    int kv[1] = {k2};
                    block_reduce<MW>(kv, ops1, red_s, rc, lane, wid, NW);
                    key = kv[0];
                } else {
                    m = gmin;
                    key = best_key(tg, gmin);
                }
            }
            if (phase == 0 && m == INT32_MAX) { end_phase(); continue; }   // X == D
            const bool best_upd = E + gmin < ebest;
            if (best_upd) set_best(use_g ? key : best_key(tg, gmin), gmin);
            if (phase == 1 && gmin >= 0) { end_phase(); continue; }       // R-4
            si = key >> 1; sx = key & 1; sv = m;
        } else if (algo == ALG_TWO) {
            // TwoNeighbor (R-10): 0, then (k, k-1) for k = 1..n-1
            if (q == 2 * n - 1) { end_phase(); continue; }
            const int i = q == 0 ? 0 : ((q & 1) ? (q + 1) >> 1 : (q >> 1) - 1);
            q++;
            int tg = INT32_MAX;
#pragma unroll
            for (int k = 0; k < EPT; k++) tg = min(tg, d[k]);
            int ov = 0, ox = 0;
            const bool own = owns(i);
            if (__any_sync(0xffffffffu, own)) {
                if (own) {
                    ov = get_at(d, lbit(i));
                    ox = (int)((xb >> lbit(i)) & 1);
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
            } else {
                const int src = (i >> 3) & 31;
                ov = __shfl_sync(0xffffffffu, ov, src);
                ox = __shfl_sync(0xffffffffu, ox, src);
            }
            const int gmin = v[0];
            if (E + gmin < ebest) set_best(best_key(tg, gmin), gmin);
            si = i; sv = ov; sx = ox;
        } else {
            if (tt == p.T) { end_phase(); continue; }
            tt++;
            const bits_t tm = tabu_mask();
            const bits_t el = ~tm & vb;
            int tg = INT32_MAX;
            if (algo == ALG_MAXMIN) {
                // MaxMin (R-6)
                int lo = INT32_MAX, hi = INT32_MIN, hv = INT32_MIN;
#pragma unroll
                for (int k = 0; k < EPT; k++) {
                    tg = min(tg, d[k]);
                    if ((el >> k) & 1) { lo = min(lo, d[k]); hi = max(hi, d[k]); }
                    if ((vb >> k) & 1) hv = max(hv, d[k]);
                }
                int v[5] = {tg, lo, hi, el != 0, hv};
                const int ops[5] = {OP_MIN, OP_MIN, OP_MAX, OP_OR, OP_MAX};
                block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
                const int gmin = v[0];
                const bool best_upd = E + gmin < ebest;
                const bits_t EL = v[3] ? el : vb;
                const int64_t LO = v[3] ? v[1] : gmin, HI = v[3] ? v[2] : v[4];
                const uint4 r = rng4(p.seed, PUR_MAXMIN, 0, gslot, p.gen, (uint32_t)flips);
                const uint64_t T = (uint64_t)p.T, u = (uint64_t)(p.T - tt);
                const unsigned __int128 num = (unsigned __int128)(uint64_t)(HI - LO) * (u * u * u);
                const uint64_t span = (uint64_t)(num / (unsigned __int128)(T * T * T));
                const int64_t thr = LO + (int64_t)(((unsigned __int128)r.x * (span + 1)) >> 32);
                bits_t cb = 0;
#pragma unroll
                for (int k = 0; k < EPT; k++)
                    if ((int64_t)d[k] <= thr) cb |= ONE << k;
                cb &= EL;
                int kbl = INT32_MAX;
                if (best_upd && __any_sync(0xffffffffu, tg == gmin))
                    if (tg == gmin) kbl = first_key_full(vb, gmin);
                int kb;
                locate_pick(cb, r.y, kbl, si, sv, sx, kb);
                if (best_upd) set_best(kb, gmin);
            } else {
                // PositiveMin (R-9)
                int tp = INT32_MAX, tpv = INT32_MAX;
#pragma unroll
                for (int k = 0; k < EPT; k++) {
                    tg = min(tg, d[k]);
                    if (d[k] > 0) {
                        if ((el >> k) & 1) tp = min(tp, d[k]);
                        if ((vb >> k) & 1) tpv = min(tpv, d[k]);
                    }
                }
                int v[4] = {tg, tp, el != 0, tpv};
                const int ops[4] = {OP_MIN, OP_MIN, OP_OR, OP_MIN};
                block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
                const int gmin = v[0];
                const bool best_upd = E + gmin < ebest;
                const bits_t EL = v[2] ? el : vb;
                const int pm = v[2] ? v[1] : v[3];     // INT32_MAX = "+inf"
                bits_t cb = 0;
#pragma unroll
                for (int k = 0; k < EPT; k++)
                    if (d[k] <= pm) cb |= ONE << k;
                cb &= EL;
                const uint4 r = rng4(p.seed, PUR_POSMIN, 0, gslot, p.gen, (uint32_t)flips);
                int kbl = INT32_MAX;
                if (best_upd && __any_sync(0xffffffffu, tg == gmin))
                    if (tg == gmin) kbl = first_key_full(vb, gmin);
                int kb;
                locate_pick(cb, r.x, kbl, si, sv, sx, kb);
                if (best_upd) set_best(kb, gmin);
            }
        }

        // ---------------- Step 3: flip bit si
        // (every thread has passed the last exchange, so the row buffer is free)
        if (t == 0) {
            fence_proxy_async();
            const char* src = Wbytes + (size_t)si * (size_t)(2 * p.n_pad);
#pragma unroll
            for (int qq = 0; qq < NP; qq++)
                bulk_row_piece(dyn_smem + qq * piece_bytes, src + qq * piece_bytes, piece_bytes, &mbar[qq]);
        }
        E += sv;
        // s_k = sigma(x_i) sigma(x_k) = -1 on these elements (Eq.(4))
        const bits_t negm = sx ? ~xb : xb;
        if (__any_sync(0xffffffffu, owns(si))) {
            if (owns(si)) {
                const int k = lbit(si);
                neg_at(d, k);                  // Eq.(5)
                xb ^= ONE << k;
                bdiff ^= ONE << k;
            }
        }
        pos = (pos + TABU_RING - 1) & (TABU_RING - 1);
        ring_s[pos] = si;
        if constexpr (TRACE) {
            if (t == 0 && s == p.trace_slot && flips < p.tr_cap) {
                p.tr_bit[flips] = si;
                p.tr_E[flips] = E;
                p.tr_phase[flips] = (int8_t)(phase == 2 ? 2 + min(round, 100) : phase);
            }
        }
        flips++;
#pragma unroll
        for (int qq = 0; qq < NP; qq++) {
            mbar_wait(&mbar[qq], par_row);
            uint4 rw[CPP];
#pragma unroll
            for (int cc = 0; cc < CPP; cc++) rw[cc] = row_s[((qq * CPP + cc) << lgNT) + t];
#pragma unroll
            for (int cc = 0; cc < CPP; cc++) {
                const int c = qq * CPP + cc;
                const uint32_t wv[4] = {rw[cc].x, rw[cc].y, rw[cc].z, rw[cc].w};
#pragma unroll
                for (int h = 0; h < 4; h++) {
                    const int lo = (int)(int16_t)(wv[h] & 0xFFFFu);
                    const int hi = (int)wv[h] >> 16;
                    const int k0 = 8 * c + 2 * h, k1 = k0 + 1;
                    d[k0] += ((negm >> k0) & 1) ? -lo : lo;
                    d[k1] += ((negm >> k1) & 1) ? -hi : hi;
                }
            }
        }
        par_row ^= 1u;
    }

    // ---------------- write back state and the result packet
    {
        uint8_t* Xb = reinterpret_cast<uint8_t*>(p.X + (size_t)s * p.nwp);
        uint8_t* Bb = reinterpret_cast<uint8_t*>(p.best + (size_t)s * p.nwp);
        int32_t* dp = p.delta + (size_t)s * p.n_pad;
        const bits_t bb = xb ^ bdiff;
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int ch = (c << lgNT) + t;
            Xb[ch] = (uint8_t)(xb >> (8 * c));
            Bb[ch] = (uint8_t)(bb >> (8 * c));
            reinterpret_cast<int4*>(dp + ch * 8)[0] = make_int4(d[8 * c], d[8 * c + 1], d[8 * c + 2], d[8 * c + 3]);
            reinterpret_cast<int4*>(dp + ch * 8)[1] = make_int4(d[8 * c + 4], d[8 * c + 5], d[8 * c + 6], d[8 * c + 7]);
        }
        if (t < TABU_RING) p.ring[(size_t)s * TABU_RING + t] = ring_s[(pos + t) & (TABU_RING - 1)];
        if (t == 0) {
            p.E[s] = E;
            p.ebest[s] = ebest;
            p.flips[s] = flips;
            atomicAdd(p.flip_total, (unsigned long long)flips);
        }
    }
}

}  // namespace dabs
