// batch_kernel.cuh -- the DABS hot loop on sm_100a: one batch search per CTA.
//
// A CTA of NT threads owns one search (one slot).  Element k of the search
// lives in thread t = (k/8) mod NT, chunk c = (k/8) / NT, lane-of-chunk e = k mod 8,
// so every thread holds EPT = 8*C flip gains Delta_k in REGISTERS and the bits
// x_k, d_k of its elements in one bits_t word.  A flip of bit i streams row i
// of the symmetric int16 W (2*n_pad bytes) with one coalesced 128-bit load per
// thread and chunk, updates every Delta_k (Eq.(4)),
// then Step 1 (scan, BEST) and Step 2 (selection) reduce
// over the CTA with redux.sync + one shared-memory exchange.
//
// MW=false: one warp per search (n <= 2048), no shared-memory reductions.
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

// Reduce K values over the CTA; every thread gets the results.  One
// __syncthreads per call (MW); the buffer parity alternates with rc.
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

// d[k] for a runtime k (one thread per warp at most executes these)
template <int EPT>
__device__ __forceinline__ int get_at(const int32_t (&d)[EPT], int k)
{
    int v = 0;
#pragma unroll
    for (int j = 0; j < EPT; j++)
        if (j == k) v = d[j];
    return v;
}
template <int EPT>
__device__ __forceinline__ void neg_at(int32_t (&d)[EPT], int k)
{
#pragma unroll
    for (int j = 0; j < EPT; j++)
        if (j == k) d[j] = -d[j];
}

template <int C, bool MW, bool TRACE>
__global__ void __launch_bounds__(MW ? 512 : 32) batch_kernel(const BatchParams p)
{
    constexpr int EPT = 8 * C;
    using bits_t = typename std::conditional<(EPT > 32), unsigned long long, uint32_t>::type;
    constexpr bits_t ONE = 1;
    const int t = threadIdx.x;
    const int NT = MW ? (int)blockDim.x : 32;
    const int lgNT = 31 - __clz(NT);
    const int lane = t & 31, wid = t >> 5, NW = NT >> 5;
    const int s = p.slot0 + (int)blockIdx.x;
    const uint32_t gslot = p.slot_base + (uint32_t)s;
    const int n = p.n;

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
    int pos = 0;   // ring_s[(pos + j) & 31] = j-th most recent flip
    int64_t E = p.E[s];
    const int algo = p.algo[s];
    if constexpr (MW) __syncthreads(); else __syncwarp();

    // element index of (chunk c, lane-of-chunk e) owned by this thread
    auto gidx = [&](int c, int e) { return (((c << lgNT) + t) << 3) | e; };
    // bit position (in bits_t) of global element k, if this thread owns it
    auto owns = [&](int k) { return ((k >> 3) & (NT - 1)) == t; };
    auto lbit = [&](int k) { return (((k >> 3) >> lgNT) << 3) | (k & 7); };

    // lowest (index<<1 | x) among this thread's elements in M with d == m
    auto first_key = [&](bits_t M, int m) -> int {
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

    // count + uniform pick in index order (MaxMin R-6, PositiveMin R-9):
    // returns the pick via (si, sv, sx); kb = BEST key (lowest gmin index) if wanted.
    auto locate_pick = [&](bits_t cb, uint32_t u, int kb_local, int& si, int& sv, int& sx,
                           int& kb) {
        int cnt[C], incl[C], woff[C], Tc[C];
#pragma unroll
        for (int c = 0; c < C; c++) {
            cnt[c] = __popc((uint32_t)((cb >> (8 * c)) & 0xFFu));
            int x = cnt[c];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            incl[c] = x;
        }
        if constexpr (MW) {
            const int par = rc & 1;
            rc++;
            const int kw = warp_min(kb_local);
            if (lane == 31) {
#pragma unroll
                for (int c = 0; c < C; c++) red_s[par][wid][c] = incl[c];
            }
            if (lane == 0) red_s[par][wid][RED_W - 1] = kw;
            __syncthreads();
#pragma unroll
            for (int c = 0; c < C; c++) {
                const int x = lane < NW ? red_s[par][lane][c] : 0;
                int y = x;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int z = __shfl_up_sync(0xffffffffu, y, off);
                    if (lane >= off) y += z;
                }
                woff[c] = __shfl_sync(0xffffffffu, y - x, wid);
                Tc[c] = __shfl_sync(0xffffffffu, y, 31);
            }
            kb = warp_min(lane < NW ? red_s[par][lane][RED_W - 1] : INT32_MAX);
        } else {
#pragma unroll
            for (int c = 0; c < C; c++) {
                woff[c] = 0;
                Tc[c] = __shfl_sync(0xffffffffu, incl[c], 31);
            }
            kb = warp_min(kb_local);
        }
        uint32_t tot = 0;
        int li = -1;
        int Pc[C];
#pragma unroll
        for (int c = 0; c < C; c++) { Pc[c] = (int)tot; tot += (uint32_t)Tc[c]; }
        const int r = (int)pick_u(u, tot);
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int lo = Pc[c] + woff[c] + incl[c] - cnt[c];
            if (r >= lo && r < lo + cnt[c]) {
                uint32_t byte = (uint32_t)((cb >> (8 * c)) & 0xFFu);
                for (int j = 0; j < r - lo; j++) byte &= byte - 1;   // drop lower set bits
                const int e = __ffs(byte) - 1;
                li = 8 * c + e;
            }
        }
        int gi = -1, lv = 0, lx = 0;
        if (li >= 0) {
            gi = gidx(li >> 3, li & 7);
            lv = get_at(d, li);
            lx = (int)((xb >> li) & 1);
        }
        if constexpr (MW) {
            const int par = rc & 1;
            rc++;
            if (li >= 0) { bc_s[par][0] = gi; bc_s[par][1] = lv; bc_s[par][2] = lx; }
            __syncthreads();
            si = bc_s[par][0]; sv = bc_s[par][1]; sx = bc_s[par][2];
        } else {
            const int src = __ffs(__ballot_sync(0xffffffffu, li >= 0)) - 1;
            si = __shfl_sync(0xffffffffu, gi, src);
            sv = __shfl_sync(0xffffffffu, lv, src);
            sx = __shfl_sync(0xffffffffu, lx, src);
        }
    };

    while (true) {
        int si = -1, sv = 0, sx = 0;       // selected bit, its Delta, its x (uniform)
        if (phase == 3) break;

        // ---------------- Step 1 + Step 2 per phase
        if (phase == 1) {
            // Greedy: argmin over all bits; stop when min >= 0 (R-4)
            int tg = INT32_MAX;
#pragma unroll
            for (int k = 0; k < EPT; k++) tg = min(tg, d[k]);
            int v[1] = {tg};
            const int ops[1] = {OP_MIN};
            block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
            const int gmin = v[0];
            const bool best_upd = E + gmin < ebest;
            if (gmin >= 0 && !best_upd) { end_phase(); continue; }
            int kv[1] = {tg == gmin ? first_key(vb, gmin) : INT32_MAX};
            block_reduce<MW>(kv, ops, red_s, rc, lane, wid, NW);
            if (best_upd) set_best(kv[0], gmin);
            if (gmin >= 0) { end_phase(); continue; }
            si = kv[0] >> 1; sx = kv[0] & 1; sv = gmin;
        } else if (phase == 0) {
            // Straight: argmin over bits with x != d (R-5)
            const bits_t cm = (xb ^ db) & vb;
            int tg = INT32_MAX, ts = INT32_MAX;
#pragma unroll
            for (int k = 0; k < EPT; k++) {
                tg = min(tg, d[k]);
                if ((cm >> k) & 1) ts = min(ts, d[k]);
            }
            int v[3] = {tg, ts, cm != 0};
            const int ops[3] = {OP_MIN, OP_MIN, OP_OR};
            block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
            if (!v[2]) { end_phase(); continue; }
            const int gmin = v[0];
            const bool best_upd = E + gmin < ebest;
            int kv[2] = {ts == v[1] ? first_key(cm, v[1]) : INT32_MAX,
                         (best_upd && tg == gmin) ? first_key(vb, gmin) : INT32_MAX};
            const int ops2[2] = {OP_MIN, OP_MIN};
            block_reduce<MW>(kv, ops2, red_s, rc, lane, wid, NW);
            if (best_upd) set_best(kv[1], gmin);
            si = kv[0] >> 1; sx = kv[0] & 1; sv = v[1];
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
            if (own) {
                ov = get_at(d, lbit(i));
                ox = (int)((xb >> lbit(i)) & 1);
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
            if (E + gmin < ebest) {
                int kv[1] = {tg == gmin ? first_key(vb, gmin) : INT32_MAX};
                block_reduce<MW>(kv, ops, red_s, rc, lane, wid, NW);
                set_best(kv[0], gmin);
            }
            si = i; sv = ov; sx = ox;
        } else {
            if (tt == p.T) { end_phase(); continue; }
            tt++;
            const bits_t tm = tabu_mask();
            const bits_t el = ~tm & vb;
            int tg = INT32_MAX;
            if (algo == ALG_CYCLIC) {
                // CyclicMin (R-7): window [cursor, cursor + w) mod n
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
                const bits_t m1 = wm & ~tm;
                int t1 = INT32_MAX, t2 = INT32_MAX;
#pragma unroll
                for (int k = 0; k < EPT; k++) {
                    tg = min(tg, d[k]);
                    if ((m1 >> k) & 1) t1 = min(t1, d[k]);
                    if ((wm >> k) & 1) t2 = min(t2, d[k]);
                }
                int v[4] = {tg, t1, m1 != 0, t2};
                const int ops[4] = {OP_MIN, OP_MIN, OP_OR, OP_MIN};
                block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
                const int gmin = v[0];
                const bool best_upd = E + gmin < ebest;
                const bool use1 = v[2] != 0;
                const int m = use1 ? v[1] : v[3];
                const int tmine = use1 ? t1 : t2;
                int kv[2] = {tmine == m ? first_key(use1 ? m1 : wm, m) : INT32_MAX,
                             (best_upd && tg == gmin) ? first_key(vb, gmin) : INT32_MAX};
                const int ops2[2] = {OP_MIN, OP_MIN};
                block_reduce<MW>(kv, ops2, red_s, rc, lane, wid, NW);
                if (best_upd) set_best(kv[1], gmin);
                si = kv[0] >> 1; sx = kv[0] & 1; sv = m;
            } else if (algo == ALG_RANDOM) {
                // RandomMin (R-8): Philox candidates, argmin
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
                const bits_t m1 = cand & el;
                int t1 = INT32_MAX, t2 = INT32_MAX;
#pragma unroll
                for (int k = 0; k < EPT; k++) {
                    tg = min(tg, d[k]);
                    if ((m1 >> k) & 1) t1 = min(t1, d[k]);
                    if ((el >> k) & 1) t2 = min(t2, d[k]);
                }
                int v[5] = {tg, t1, m1 != 0, t2, el != 0};
                const int ops[5] = {OP_MIN, OP_MIN, OP_OR, OP_MIN, OP_OR};
                block_reduce<MW>(v, ops, red_s, rc, lane, wid, NW);
                const int gmin = v[0];
                const bool best_upd = E + gmin < ebest;
                const int which = v[2] ? 0 : (v[4] ? 1 : 2);
                const int m = which == 0 ? v[1] : (which == 1 ? v[3] : gmin);
                const bits_t M = which == 0 ? m1 : (which == 1 ? el : vb);
                const int tmine = which == 0 ? t1 : (which == 1 ? t2 : tg);
                int kv[2] = {tmine == m ? first_key(M, m) : INT32_MAX,
                             (best_upd && tg == gmin) ? first_key(vb, gmin) : INT32_MAX};
                const int ops2[2] = {OP_MIN, OP_MIN};
                block_reduce<MW>(kv, ops2, red_s, rc, lane, wid, NW);
                if (best_upd) set_best(kv[1], gmin);
                si = kv[0] >> 1; sx = kv[0] & 1; sv = m;
            } else if (algo == ALG_MAXMIN) {
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
                int kb;
                locate_pick(cb, r.y, (best_upd && tg == gmin) ? first_key(vb, gmin) : INT32_MAX,
                            si, sv, sx, kb);
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
                int kb;
                locate_pick(cb, r.x, (best_upd && tg == gmin) ? first_key(vb, gmin) : INT32_MAX,
                            si, sv, sx, kb);
                if (best_upd) set_best(kb, gmin);
            }
        }

        // ---------------- Step 3: flip bit si
        const uint4* row = reinterpret_cast<const uint4*>(p.W + (size_t)si * p.n_pad);
        uint4 rw[C];
#pragma unroll
        for (int c = 0; c < C; c++) rw[c] = __ldg(row + (c << lgNT) + t);
        E += sv;
        // s_k = sigma(x_i) sigma(x_k) = -1 on these elements (Eq.(4))
        const bits_t negm = sx ? ~xb : xb;
        if (owns(si)) {
            const int k = lbit(si);
            neg_at(d, k);                  // Eq.(5)
            xb ^= ONE << k;
            bdiff ^= ONE << k;
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
        for (int c = 0; c < C; c++) {
            const uint32_t wv[4] = {rw[c].x, rw[c].y, rw[c].z, rw[c].w};
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
