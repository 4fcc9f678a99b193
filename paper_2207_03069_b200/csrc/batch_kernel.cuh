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
    constexpr unsigned FULL = 0xffffffffu;
    const int t = threadIdx.x;
    const int NT = MW ? (int)blockDim.x : 32;
    const int lgNT = MW ? 31 - __clz(NT) : 5;
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
        for (int qq = 0; qq < NP; qq++) mbar_init(&mbar[qq], 1);
        fence_mbar_init();
    }
    int pos = 0;   // ring_s[(pos + j) & 31] = j-th most recent flip
    int64_t E = p.E[s];
    const int algo = p.algo[s];
    const int tabu = p.tabu;
    const uint32_t piece_bytes = (uint32_t)(2 * p.n_pad / NP);
    uint32_t par_row = 0;
    int flips = 0;
    int64_t ebest = E_INF;
    bits_t bdiff = 0;              // BEST = X xor bdiff
    int rc = 0;                    // exchange parity counter
    int phase_code = 0;            // for the trace: 0 Straight, 1 Greedy, 2+r main round r
    if constexpr (MW) __syncthreads(); else __syncwarp();

    auto gidx = [&](int c, int e) { return (((c << lgNT) + t) << 3) | e; };
    auto owns = [&](int k) { return ((k >> 3) & (NT - 1)) == t; };
    auto lbit = [&](int k) { return (((k >> 3) >> lgNT) << 3) | (k & 7); };

    // ---------------- scans (Step 1 and the argmin rules of Step 2)
    auto scan_min = [&]() -> int {            // min over all elements (pads are INT32_MAX)
        int m = INT32_MAX;
#pragma unroll
        for (int k = 0; k < EPT; k++) m = min(m, d[k]);
        return m;
    };
    auto scan_chunks = [&](int (&gm)[C]) -> int {   // per-chunk minima, all elements
        int m = INT32_MAX;
#pragma unroll
        for (int c = 0; c < C; c++) {
            int mc = INT32_MAX;
#pragma unroll
            for (int e = 0; e < 8; e++) mc = min(mc, d[8 * c + e]);
            gm[c] = mc;
            m = min(m, mc);
        }
        return m;
    };
    auto scan_chunks_masked = [&](bits_t M, int (&gm)[C]) -> int {   // per-chunk minima over M
        int m = INT32_MAX;
#pragma unroll
        for (int c = 0; c < C; c++) {
            int mc = INT32_MAX;
#pragma unroll
            for (int e = 0; e < 8; e++)
                if ((M >> (8 * c + e)) & 1) mc = min(mc, d[8 * c + e]);
            gm[c] = mc;
            m = min(m, mc);
        }
        return m;
    };
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
    // key of the first element with value m, from per-chunk minima (one lane runs it)
    auto key_from_chunks = [&](const int (&gm)[C], bits_t M, int m) -> int {
        int cs = 0;
#pragma unroll
        for (int c = C - 1; c >= 0; c--)
            if (gm[c] == m) cs = c;
        const int e = first_in_chunk(d, M, cs, m);
        const int k = 8 * cs + e;
        return (gidx(cs, e) << 1) | (int)((xb >> k) & 1);
    };
    // One exchange: argmin (value, lowest key) of the rule + min of tg (Step 1).
    auto argmin_exchange = [&](int tsel, const int (&gm)[C], bits_t M, int tg, int& m, int& key,
                               int& gmin) {
        const int wmin = warp_min(tsel);
        int k = INT32_MAX;
        if (__any_sync(FULL, tsel == wmin && wmin != INT32_MAX))
            if (tsel == wmin && wmin != INT32_MAX) k = key_from_chunks(gm, M, wmin);
        k = warp_min(k);
        int g = warp_min(tg);
        if constexpr (MW) {
            const int par = rc & 1;
            rc++;
            if (lane == 0) { red_s[par][wid][0] = wmin; red_s[par][wid][1] = k; red_s[par][wid][2] = g; }
            __syncthreads();
            const int a = lane < NW ? red_s[par][lane][0] : INT32_MAX;
            const int b = lane < NW ? red_s[par][lane][1] : INT32_MAX;
            const int c = lane < NW ? red_s[par][lane][2] : INT32_MAX;
            m = warp_min(a);
            key = warp_min(a == m ? b : INT32_MAX);
            gmin = warp_min(c);
        } else {
            m = wmin;
            key = k;
            gmin = g;
        }
    };
    // lazy key of the global-min element (BEST update, rare)
    auto best_key = [&](int tg, int gmin) -> int {
        int k = INT32_MAX;
        if (__any_sync(FULL, tg == gmin))
            if (tg == gmin) k = first_key_full(vb, gmin);
        int v[1] = {k};
        const int ops[1] = {OP_MIN};
        block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
        return v[0];
    };
    // masked argmin over M with a full-scan key (fallback paths, rare)
    auto argmin_slow = [&](bits_t M, int& m, int& key) {
        int tm_ = INT32_MAX;
#pragma unroll
        for (int k = 0; k < EPT; k++)
            if ((M >> k) & 1) tm_ = min(tm_, d[k]);
        int v[1] = {tm_};
        const int ops[1] = {OP_MIN};
        block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
        m = v[0];
        int kk = INT32_MAX;
        if (__any_sync(FULL, tm_ == m && m != INT32_MAX))
            if (tm_ == m && m != INT32_MAX) kk = first_key_full(M, m);
        int kv[1] = {kk};
        block_reduce<MW>(kv, ops, red_s, rc, lane, wid, NW);
        key = kv[0];
    };
    auto set_best = [&](int key, int m) {
        ebest = E + m;
        const int j = key >> 1;
        bdiff = owns(j) ? (ONE << lbit(j)) : (bits_t)0;
    };

    // ---------------- Step 3: flip bit si, Eqs.(4)-(5)
    auto do_flip = [&](int si, int sv, int sx) {
        // every thread has passed the last exchange: the row buffer is free
        if (t == 0) {
            fence_proxy_async();
            const char* src = reinterpret_cast<const char*>(p.W) + (size_t)si * (size_t)(2 * p.n_pad);
#pragma unroll
            for (int qq = 0; qq < NP; qq++)
                bulk_row_piece(dyn_smem + qq * piece_bytes, src + qq * piece_bytes, piece_bytes, &mbar[qq]);
        }
        E += sv;
        const bits_t negm = sx ? ~xb : xb;   // s_k = sigma(x_i) sigma(x_k) = -1 here
        if (__any_sync(FULL, owns(si))) {
            if (owns(si)) {
                const int k = lbit(si);
                neg_at(d, k);                    // Eq.(5)
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
                p.tr_phase[flips] = (int8_t)phase_code;
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
                    d[k0] += ((negm >> k0) & 1) ? -lo : lo;   // Eq.(4)
                    d[k1] += ((negm >> k1) & 1) ? -hi : hi;
                }
            }
        }
        par_row ^= 1u;
    };

    // ---------------- tabu mask (R-11): bits of the last `tabu` flips
    auto tabu_full = [&]() -> bits_t {
        bits_t m = 0;
        for (int j = 0; j < tabu; j++) {
            const int r = ring_s[(pos + j) & (TABU_RING - 1)];
            if (r >= 0 && owns(r)) m |= ONE << lbit(r);
        }
        return m;
    };
    // after a flip: the new flip enters, the (tabu+1)-th most recent leaves
    auto tabu_step = [&](bits_t& tm, int si) {
        if (tabu == 0) return;
        if (owns(si)) tm |= ONE << lbit(si);
        const int r = ring_s[(pos + tabu) & (TABU_RING - 1)];
        if (r >= 0 && owns(r)) {
            bool still = false;
            for (int j = 0; j < tabu; j++) still |= ring_s[(pos + j) & (TABU_RING - 1)] == r;
            if (!still) tm &= ~(ONE << lbit(r));
        }
    };

    // ---------------- phases
    // Straight (R-5): argmin over bits with x != d until X == D
    auto run_straight = [&]() {
        phase_code = 0;
        while (true) {
            const bits_t cm = (xb ^ db) & vb;
            const int tg = scan_min();
            int gm[C];
            int t1 = INT32_MAX;
#pragma unroll
            for (int c = 0; c < C; c++) gm[c] = INT32_MAX;
            if (__any_sync(FULL, cm != 0)) t1 = scan_chunks_masked(cm, gm);
            int m, key, gmin;
            argmin_exchange(t1, gm, cm, tg, m, key, gmin);
            if (m == INT32_MAX) return;                         // X == D
            if (E + gmin < ebest) set_best(best_key(tg, gmin), gmin);
            do_flip(key >> 1, m, key & 1);
        }
    };
    // Greedy (R-4): argmin over all bits while min < 0
    auto run_greedy = [&]() {
        phase_code = 1;
        while (true) {
            int gm[C];
            const int tg = scan_chunks(gm);
            int m, key, gmin;
            argmin_exchange(tg, gm, ~(bits_t)0, tg, m, key, gmin);
            if (E + gmin < ebest) set_best(key, gmin);
            if (gmin >= 0) return;
            do_flip(key >> 1, gmin, key & 1);
        }
    };
    // CyclicMin (R-7)
    auto run_cyclic = [&]() {
        bits_t tm = tabu_full();
        int cursor = 0;
        for (int tt = 1; tt <= p.T; tt++) {
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
            const bits_t M1 = wm & ~tm;
            const int tg = scan_min();
            int gm[C];
            int t1 = INT32_MAX;
#pragma unroll
            for (int c = 0; c < C; c++) gm[c] = INT32_MAX;
            if (__any_sync(FULL, M1 != 0)) t1 = scan_chunks_masked(M1, gm);
            int m, key, gmin;
            argmin_exchange(t1, gm, M1, tg, m, key, gmin);
            if (m == INT32_MAX) argmin_slow(wm, m, key);      // window all tabu: drop tabu
            if (E + gmin < ebest) set_best(best_key(tg, gmin), gmin);
            const int si = key >> 1;
            do_flip(si, m, key & 1);
            tabu_step(tm, si);
        }
    };
    // RandomMin (R-8)
    auto run_random = [&]() {
        bits_t tm = tabu_full();
        for (int tt = 1; tt <= p.T; tt++) {
            const uint32_t p16 = (uint32_t)p.ptab[tt];
            bits_t cand;
            if (p16 >= 65536u) {
                cand = vb;
            } else {
                cand = 0;
#pragma unroll
                for (int c = 0; c < C; c++) {
                    const uint4 r = rng4(p.seed, PUR_RANDMIN, (uint32_t)((c << lgNT) + t), gslot, p.gen,
                                         (uint32_t)flips);
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
            const bits_t M1 = cand & ~tm & vb;
            const int tg = scan_min();
            int gm[C];
            int t1 = INT32_MAX;
#pragma unroll
            for (int c = 0; c < C; c++) gm[c] = INT32_MAX;
            if (__any_sync(FULL, M1 != 0)) t1 = scan_chunks_masked(M1, gm);
            int m, key, gmin;
            argmin_exchange(t1, gm, M1, tg, m, key, gmin);
            if (m == INT32_MAX) {                               // no candidate (R-8)
                argmin_slow(~tm & vb, m, key);
                if (m == INT32_MAX) { m = gmin; key = best_key(tg, gmin); }   // all tabu (R-11)
            }
            if (E + gmin < ebest) set_best(best_key(tg, gmin), gmin);
            const int si = key >> 1;
            do_flip(si, m, key & 1);
            tabu_step(tm, si);
        }
    };

    // count + uniform pick in index order (MaxMin R-6, PositiveMin R-9):
    // picks the floor(u |C| / 2^32)-th member of cb in ascending index order.
    auto locate_pick = [&](bits_t cb, uint32_t u, int& si, int& sv, int& sx) {
        int incl[C];   // warp-inclusive prefix of this lane's candidate count, per chunk
#pragma unroll
        for (int c = 0; c < C; c++) {
            int x = __popc((uint32_t)((cb >> (8 * c)) & 0xFFu));
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(FULL, x, off);
                if (lane >= off) x += y;
            }
            incl[c] = x;
        }
        int par = 0;
        if constexpr (MW) {
            par = rc & 1;
            rc++;
            if (lane == 31) {
#pragma unroll
                for (int c = 0; c < C; c++) red_s[par][wid][c] = incl[c];
            }
            __syncthreads();
        }
        // chunk-major order: all of chunk 0 (thread order), then chunk 1, ...
        int tot = 0;
#pragma unroll
        for (int c = 0; c < C; c++) {
            int woff = 0, Tc;
            if constexpr (MW) {
                const int x = lane < NW ? red_s[par][lane][c] : 0;
                int y = x;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int z = __shfl_up_sync(FULL, y, off);
                    if (lane >= off) y += z;
                }
                woff = __shfl_sync(FULL, y - x, wid);
                Tc = __shfl_sync(FULL, y, 31);
            } else {
                Tc = __shfl_sync(FULL, incl[c], 31);
            }
            const int cnt = __popc((uint32_t)((cb >> (8 * c)) & 0xFFu));
            incl[c] = tot + woff + incl[c] - cnt;   // rank of this lane's first candidate in chunk c
            tot += Tc;
        }
        const int r = (int)pick_u(u, (uint32_t)tot);
        int li = -1;
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
        if (__any_sync(FULL, li >= 0)) {
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
            const int src = __ffs(__ballot_sync(FULL, li >= 0)) - 1;
            si = __shfl_sync(FULL, gi, src);
            sv = __shfl_sync(FULL, lv, src);
            sx = __shfl_sync(FULL, lx, src);
        }
    };

    // MaxMin (R-6)
    auto run_maxmin = [&]() {
        bits_t tm = tabu_full();
        for (int tt = 1; tt <= p.T; tt++) {
            const bits_t el = ~tm & vb;
            int tg = INT32_MAX, lo = INT32_MAX, hi = INT32_MIN;
            if (__any_sync(FULL, el != ~(bits_t)0)) {   // lanes with tabu bits or pads: masked
#pragma unroll
                for (int k = 0; k < EPT; k++) {
                    tg = min(tg, d[k]);
                    if ((el >> k) & 1) { lo = min(lo, d[k]); hi = max(hi, d[k]); }
                }
            } else {
#pragma unroll
                for (int k = 0; k < EPT; k++) {
                    tg = min(tg, d[k]);
                    hi = max(hi, d[k]);
                }
                lo = tg;
            }
            int v[4] = {tg, lo, hi, el != 0};
            const int ops[4] = {OP_MIN, OP_MIN, OP_MAX, OP_OR};
            block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
            const int gmin = v[0];
            bits_t EL = el;
            int64_t LO = v[1], HI = v[2];
            if (!v[3]) {                                // every bit tabu: drop tabu (R-11)
                EL = vb;
                int hv = INT32_MIN;
#pragma unroll
                for (int k = 0; k < EPT; k++)
                    if ((vb >> k) & 1) hv = max(hv, d[k]);
                int v2[1] = {hv};
                const int ops2[1] = {OP_MAX};
                block_reduce<MW>(v2, ops2, red_s, rc, lane, wid, NW);
                LO = gmin;
                HI = v2[0];
            }
            const uint4 r = rng4(p.seed, PUR_MAXMIN, 0, gslot, p.gen, (uint32_t)flips);
            const uint64_t T = (uint64_t)p.T, u = (uint64_t)(p.T - tt);
            const unsigned __int128 num = (unsigned __int128)(uint64_t)(HI - LO) * (u * u * u);
            const uint64_t span = (uint64_t)(num / (unsigned __int128)(T * T * T));
            const int thr = (int)(LO + (int64_t)(((unsigned __int128)r.x * (span + 1)) >> 32));
            bits_t cb = 0;
#pragma unroll
            for (int k = 0; k < EPT; k++)
                if (d[k] <= thr) cb |= ONE << k;
            cb &= EL;
            const bool bu = E + gmin < ebest;
            int bk = INT32_MAX;
            if (bu) bk = best_key(tg, gmin);
            int si, sv, sx;
            locate_pick(cb, r.y, si, sv, sx);
            if (bu) set_best(bk, gmin);
            do_flip(si, sv, sx);
            tabu_step(tm, si);
        }
    };
    // PositiveMin (R-9)
    auto run_posmin = [&]() {
        bits_t tm = tabu_full();
        for (int tt = 1; tt <= p.T; tt++) {
            const bits_t el = ~tm & vb;
            int tg = INT32_MAX;
            unsigned tp = 0xFFFFFFFFu;   // min over eligible positive Delta, as Delta-1 unsigned
            if (__any_sync(FULL, (el | ~vb) != ~(bits_t)0)) {   // lanes with tabu bits
#pragma unroll
                for (int k = 0; k < EPT; k++) {
                    tg = min(tg, d[k]);
                    if ((el >> k) & 1) tp = min(tp, (unsigned)(d[k] - 1));
                }
            } else {
#pragma unroll
                for (int k = 0; k < EPT; k++) {
                    tg = min(tg, d[k]);
                    tp = min(tp, (unsigned)(d[k] - 1));   // pads (INT32_MAX) never win
                }
            }
            // Delta <= 0 maps to >= 2^31 - 1 (as unsigned); keep only real positives
            int tpi = tp < 0x7FFFFFFEu ? (int)tp + 1 : INT32_MAX;
            int v[3] = {tg, tpi, el != 0};
            const int ops[3] = {OP_MIN, OP_MIN, OP_OR};
            block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
            const int gmin = v[0];
            bits_t EL = el;
            int pm = v[1];                              // INT32_MAX = "+inf"
            if (!v[2]) {                                // every bit tabu (R-11)
                EL = vb;
                unsigned t2 = 0xFFFFFFFFu;
#pragma unroll
                for (int k = 0; k < EPT; k++) t2 = min(t2, (unsigned)(d[k] - 1));
                int v2[1] = {t2 < 0x7FFFFFFEu ? (int)t2 + 1 : INT32_MAX};
                const int ops2[1] = {OP_MIN};
                block_reduce<MW>(v2, ops2, red_s, rc, lane, wid, NW);
                pm = v2[0];
            }
            bits_t cb = 0;
#pragma unroll
            for (int k = 0; k < EPT; k++)
                if (d[k] <= pm) cb |= ONE << k;
            cb &= EL;
            const uint4 r = rng4(p.seed, PUR_POSMIN, 0, gslot, p.gen, (uint32_t)flips);
            const bool bu = E + gmin < ebest;
            int bk = INT32_MAX;
            if (bu) bk = best_key(tg, gmin);
            int si, sv, sx;
            locate_pick(cb, r.x, si, sv, sx);
            if (bu) set_best(bk, gmin);
            do_flip(si, sv, sx);
            tabu_step(tm, si);
        }
    };
    // TwoNeighbor (R-10): 0, then (k, k-1) for k = 1..n-1
    auto run_two = [&]() {
        for (int q = 0; q < 2 * n - 1; q++) {
            const int i = q == 0 ? 0 : ((q & 1) ? (q + 1) >> 1 : (q >> 1) - 1);
            const int tg = scan_min();
            int ov = 0, ox = 0;
            const bool own = owns(i);
            if (__any_sync(FULL, own)) {
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
                ov = __shfl_sync(FULL, ov, src);
                ox = __shfl_sync(FULL, ox, src);
            }
            const int gmin = v[0];
            if (E + gmin < ebest) set_best(best_key(tg, gmin), gmin);
            do_flip(i, ov, ox);
        }
    };

    // ---------------- batch control (R-12)
    run_straight();
    run_greedy();
    int round = 0;
    do {
        phase_code = 2 + min(round, 100);
        switch (algo) {
        case ALG_MAXMIN: run_maxmin(); break;
        case ALG_CYCLIC: run_cyclic(); break;
        case ALG_RANDOM: run_random(); break;
        case ALG_POSMIN: run_posmin(); break;
        default: run_two(); break;
        }
        run_greedy();
        round++;
    } while (algo != ALG_TWO && flips < p.B);

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
