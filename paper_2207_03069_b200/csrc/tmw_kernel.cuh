// tmw_kernel.cuh -- the TMEM warp tier of the DABS hot loop (512 < n <= 2048) on sm_100a.
//
// One warp per search as in the register warp tier (batch_body, MW = false),
// but Delta (8C int32 per lane) lives in tensor memory, so a thread needs no
// registers for it and 32 searches fit on an SM (8 CTAs of 4 independent
// warps, 64 registers per thread) instead of the 16 / 24 that registers allow.
// The register warp tier is issue/latency bound at 52 % issue-active
// (profiles/r02_ncu_batch_k2000s.json): more resident searches hide more of
// the per-flip dependency chains.
//
// Warp w of a CTA is the search of slot order[4*blockIdx.x + w]; it owns TMEM
// lanes 32w..32w+31, columns 0..8C-1 of the CTA's allocation: element
// k = ((c*32 + lane)*8 + e) is column 8c + e of lane `lane` (the register warp
// tier's element order).  The four searches never synchronise with each other
// inside the batch loop; the CTA synchronises only at TMEM alloc / dealloc.
//
// Per flip: selection by warp reductions, the W row by one TMA bulk copy into
// this warp's shared-memory row buffer (mbarrier completion), Eq.(5) by the
// owner lane through one TMEM column, then Delta streams through registers in
// x16 half-pieces (2 chunks, load-ahead): IDP.2A update with sigma words from
// the shared 256-entry table, the next step's Step 1 + Step 2 scans, store.
// Semantics are batch_body's bit for bit (GPU parity tests vs the oracle).
// P:n = PAPER.md line n; R-x = DESIGN.md readings.
#pragma once
#include "tmem_kernel.cuh"

namespace dabs {

constexpr int TMW_SPC = 4;   // searches (warps) per CTA

template <int C, bool TRACE>
__global__ void __launch_bounds__(32 * TMW_SPC, 8) tmw_batch_kernel(const BatchParams p)
{
    static_assert(C == 4 || C == 8, "TMEM warp tier: 4 or 8 chunks per lane");
    constexpr int lgNT = 5, NT = 32, EPT = 8 * C, HP = C / 2, CW = C / 2;
    constexpr int TCOLS = EPT < 32 ? 32 : EPT;   // TMEM columns per CTA (a power of two >= 32)
    constexpr unsigned FULL = 0xffffffffu;
    using bits_t = uint64_t;
    constexpr bits_t ONE = 1;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int t = lane;                                       // thread within the search
    const int sidx = (int)blockIdx.x * TMW_SPC + w;
    const bool active = sidx < p.count;
    const uint32_t gen = p.gen_ptr ? *p.gen_ptr : p.gen;
    const int n = p.n;

    extern __shared__ __align__(128) uint8_t dyn_smem[];
    __shared__ __align__(8) uint64_t mbar_all[TMW_SPC];
    __shared__ uint32_t tbase_s;
    __shared__ int32_t ring_all[TMW_SPC][TABU_RING];
    __shared__ uint4 lut_s[256];
    __shared__ bits_t pm_all[TMW_SPC][3][32];   // [0] D bits, [1] M2, [2] BEST xor X

    if (w == 0) tm_alloc(&tbase_s, TCOLS);
    for (int v = tid; v < 256; v += 32 * TMW_SPC) {
        uint32_t q[4];
#pragma unroll
        for (int j = 0; j < 4; j++)
            q[j] = (((uint32_t)v >> (2 * j)) & 1u ? 0x01u : 0xFFu) | ((((uint32_t)v >> (2 * j + 1)) & 1u ? 0x01u : 0xFFu) << 24);
        lut_s[v] = make_uint4(q[0], q[1], q[2], q[3]);
    }
    if (lane == 0) {
        mbar_init(&mbar_all[w], 1);
        fence_mbar_init();
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();

    if (active) {
        const int s = p.order ? p.order[sidx] : p.slot0 + sidx;
        const uint32_t gslot = p.slot_base + (uint32_t)s;
        const uint32_t tw = tbase_s + ((uint32_t)(32 * w) << 16);
        uint64_t* mbar = &mbar_all[w];
        int32_t* ring_s = ring_all[w];
        bits_t (*pm_s)[32] = pm_all[w];
        const uint4* row_s = reinterpret_cast<const uint4*>(dyn_smem + (size_t)w * 2 * p.n_pad);

        // ---------------- the slot's persistent state (R-14)
        bits_t xb = 0, vb = 0;
        {
            const uint8_t* Xb = reinterpret_cast<const uint8_t*>(p.X + (size_t)s * p.nwp);
            const uint8_t* Db = reinterpret_cast<const uint8_t*>(p.D + (size_t)s * p.nwp);
            const int32_t* dp = p.delta + (size_t)s * p.n_pad;
            bits_t db = 0;
#pragma unroll
            for (int h = 0; h < HP; h++) {
                int32_t v[16];
#pragma unroll
                for (int cc = 0; cc < 2; cc++) {
                    const int c = 2 * h + cc;
                    const int ch = (c << lgNT) + t;
                    xb |= (bits_t)Xb[ch] << (8 * c);
                    db |= (bits_t)Db[ch] << (8 * c);
                    const int nv = min(max(n - ch * 8, 0), 8);
                    vb |= (bits_t)((1u << nv) - 1u) << (8 * c);
                    const int4 a = reinterpret_cast<const int4*>(dp + ch * 8)[0];
                    const int4 b = reinterpret_cast<const int4*>(dp + ch * 8)[1];
                    v[8 * cc + 0] = a.x; v[8 * cc + 1] = a.y; v[8 * cc + 2] = a.z; v[8 * cc + 3] = a.w;
                    v[8 * cc + 4] = b.x; v[8 * cc + 5] = b.y; v[8 * cc + 6] = b.z; v[8 * cc + 7] = b.w;
                }
                tm_st16(tw + 16 * h, v);
            }
            pm_s[0][t] = db;
            pm_s[2][t] = 0;
        }
        tm_wait_st();
        ring_s[t] = p.ring[(size_t)s * TABU_RING + t];
        __syncwarp();
        int pos = 0;
        int64_t E = p.E[s];
        const int algo = (int)p.algo[s];
        const int tabu = p.tabu;
        const int T = p.T;
        uint32_t par_row = 0;
        int flips = 0;
        int64_t ebest = E_INF;

        auto gidx = [&](int c, int e) { return (((c << lgNT) + t) << 3) | e; };
        auto owns = [&](int k) { return ((k >> 3) & (NT - 1)) == t; };
        auto lbit = [&](int k) { return (((k >> 3) >> lgNT) << 3) | (k & 7); };
        auto byte_of = [&](bits_t m, int c) { return (uint32_t)(m >> (8 * c)) & 0xFFu; };
        const uint32_t row_bytes = (uint32_t)(2 * p.n_pad);
        auto issue_row = [&](int i) {
            fence_proxy_async();
            bulk_row_piece(dyn_smem + (size_t)w * row_bytes,
                           reinterpret_cast<const char*>(p.W) + (size_t)i * row_bytes, row_bytes, mbar);
        };

        int phase = 0, round = 0, tt = 0, cursor = 0;
        bool after_main = false;
        bits_t tm = 0;
        int64_t glb = INT64_MIN / 4;
        for (int j = 0; j < tabu; j++) {
            const int r = ring_s[j];
            if (r >= 0 && owns(r)) tm |= ONE << lbit(r);
        }

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

        // ---------------- Step 2 setup (uniform) and scan modes (as tm_batch_kernel)
        constexpr int SM_G = 0, SM_M = 1, SM_R = 2, SM_T = 3, SM_MM = 4, SM_PM = 5;
        int kind = 0;
        bool masked = true;
        bits_t M1 = vb;
        int smode = SM_G;
        uint32_t cmeet = 0xFFu;
        uint32_t rK = 0, rp16 = 0;
        auto setup = [&]() {
            if (phase == 2 && tt == (algo == ALG_TWO ? 2 * n - 1 : T)) {
                phase = 1;
                after_main = true;
            }
            kind = 0;
            masked = true;
            cmeet = 0xFFu;
            if (phase == 0) {
                M1 = (xb ^ pm_s[0][t]) & vb;                               // Straight
            } else if (phase == 1) {
                masked = false;                                            // Greedy
                M1 = ~(bits_t)0;
            } else {
                tt++;
                if (tt == 1) cursor = 0;
                if (algo == ALG_CYCLIC) {                                  // CyclicMin (R-7)
                    const int wdt = p.wtab[tt];
                    const int b0 = min(cursor + wdt, n), b1 = cursor + wdt - n;
                    bits_t wm = 0;
                    cmeet = 0;
#pragma unroll
                    for (int c = 0; c < C; c++) {
                        const int s0 = (c << lgNT) << 3, s1 = s0 + (NT << 3);
                        if ((cursor < s1 && b0 > s0) || b1 > s0) {
                            cmeet |= 1u << c;
                            const int base = gidx(c, 0);
                            const int lo = max(cursor - base, 0), hi = min(b0 - base, 8);
                            uint32_t byte = 0;
                            if (lo < hi) byte |= ((1u << (hi - lo)) - 1u) << lo;
                            const int hi2 = min(b1 - base, 8);
                            if (hi2 > 0) byte |= (1u << hi2) - 1u;
                            wm |= (bits_t)byte << (8 * c);
                        }
                    }
                    cursor += wdt;
                    if (cursor >= n) cursor -= n;
                    M1 = wm & ~tm;
                    pm_s[1][t] = wm;
                } else if (algo == ALG_RANDOM) {                           // RandomMin (R-8)
                    rp16 = (uint32_t)p.ptab[tt];
                    rK = rp16 >= 65536u ? 0u : draw(flips).x;
                    M1 = 0;
                    pm_s[1][t] = vb & ~tm;
                } else if (algo == ALG_TWO) {                              // TwoNeighbor (R-10)
                    kind = 2;
                } else {
                    kind = 1;                                              // MaxMin / PositiveMin
                    M1 = vb & ~tm;
                }
            }
            smode = kind == 2 ? SM_T
                  : kind == 1 ? (algo == ALG_MAXMIN ? SM_MM : SM_PM)
                  : !masked ? SM_G
                  : (algo == ALG_RANDOM && phase == 2) ? SM_R : SM_M;
        };

        int tg = INT32_MAX, tsel = INT32_MAX, tcs = 0, a1 = INT32_MAX, a2 = INT32_MIN;
        unsigned tp = 0xFFFFFFFFu;
        auto reset_partials = [&]() {
            tg = INT32_MAX; tsel = INT32_MAX; tcs = 0; a1 = INT32_MAX; a2 = INT32_MIN; tp = 0xFFFFFFFFu;
        };
        auto scan_chunk = [&](auto MODE, const int c, const int32_t* dc, const uint32_t mb) {
            constexpr int md = decltype(MODE)::value;
            const int mn = min(min(min(dc[0], dc[1]), min(dc[2], dc[3])), min(min(dc[4], dc[5]), min(dc[6], dc[7])));
            if constexpr (md == SM_G) {
                if (mn < tsel) { tsel = mn; tcs = c; }
            } else if constexpr (md == SM_T) {
                tg = min(tg, mn);
            } else if constexpr (md == SM_M || md == SM_R) {
                tg = min(tg, mn);
                if (md == SM_R || ((cmeet >> c) & 1u)) {
                    int mc = INT32_MAX;
#pragma unroll
                    for (int e = 0; e < 8; e++)
                        if ((mb >> e) & 1u) mc = min(mc, dc[e]);
                    if (mc < tsel) { tsel = mc; tcs = c; }
                }
            } else if constexpr (md == SM_MM) {
                tg = min(tg, mn);
                if (mb == 0xFFu) {
                    const int mx = max(max(max(dc[0], dc[1]), max(dc[2], dc[3])), max(max(dc[4], dc[5]), max(dc[6], dc[7])));
                    a1 = min(a1, mn);
                    a2 = max(a2, mx);
                } else {
#pragma unroll
                    for (int e = 0; e < 8; e++)
                        if ((mb >> e) & 1u) { a1 = min(a1, dc[e]); a2 = max(a2, dc[e]); }
                }
            } else {
                tg = min(tg, mn);
                unsigned q = 0xFFFFFFFFu;
#pragma unroll
                for (int e = 0; e < 8; e++)
                    if ((mb >> e) & 1u) q = min(q, (unsigned)(dc[e] - 1));
                tp = min(tp, q);
            }
        };
        // the mask byte of chunk c for MODE (SM_R: the RandomMin candidates, R-8, added to M1)
        auto chunk_mask = [&](auto MODE, const int c) -> uint32_t {
            constexpr int md = decltype(MODE)::value;
            if constexpr (md == SM_R) {
                const uint32_t cb = rp16 >= 65536u ? byte_of(vb, c)
                                                   : randmin_byte(rK, (uint32_t)(((c << lgNT) + t) << 2), rp16);
                const uint32_t mb = cb & byte_of(vb, c) & ~byte_of(tm, c);
                M1 |= (bits_t)mb << (8 * c);
                return mb;
            } else if constexpr (md == SM_M || md == SM_MM || md == SM_PM) {
                return byte_of(M1, c);
            } else {
                return 0u;
            }
        };
        auto scan_full = [&](auto MODE) {
#pragma unroll
            for (int h = 0; h < HP; h++) {
                int32_t v[16];
                tm_ld16(tw + 16 * h, v);
                const uint32_t m0 = chunk_mask(MODE, 2 * h), m1 = chunk_mask(MODE, 2 * h + 1);
                tm_wait_ld16(v);
                scan_chunk(MODE, 2 * h, v, m0);
                scan_chunk(MODE, 2 * h + 1, v + 8, m1);
            }
        };
        // f(c, v8) over every chunk's Delta values (rare full passes)
        auto for_chunks = [&](auto f) {
#pragma unroll 1
            for (int h = 0; h < HP; h++) {
                int32_t v[16];
                tm_ld16(tw + 16 * h, v);
                tm_wait_ld16(v);
                f(2 * h, v);
                f(2 * h + 1, v + 8);
            }
        };
        using IG = std::integral_constant<int, SM_G>;
        using IM = std::integral_constant<int, SM_M>;
        using IR = std::integral_constant<int, SM_R>;
        using IT = std::integral_constant<int, SM_T>;
        using IMM = std::integral_constant<int, SM_MM>;
        using IPM = std::integral_constant<int, SM_PM>;

        bool have = false;
        while (true) {
            const bool skip_g = E + glb >= ebest;
            if (!have) {
                setup();
                reset_partials();
                switch (smode) {
                case SM_G: scan_full(IG{}); break;
                case SM_M: scan_full(IM{}); break;
                case SM_R: scan_full(IR{}); break;
                case SM_T: scan_full(IT{}); break;
                case SM_MM: scan_full(IMM{}); break;
                default: scan_full(IPM{}); break;
                }
            }
            have = false;

            // ---------------- Step 1 + Step 2: warp reductions (R-2..R-11)
            int si = 0, sv = 0, sx = 0;
            int gmin = 0;
            int key = INT32_MAX;
            if (kind == 0) {
                if (!masked) tg = tsel;
                const int wmin = warp_min(tsel);
                int k = INT32_MAX;
                const bool holds = tsel == wmin && wmin != INT32_MAX;
                if (__any_sync(FULL, holds)) {
                    const int cmin = warp_min(holds ? tcs : INT32_MAX);
                    int32_t v[8];
                    tm_ld8(tw + 8 * cmin, v);
                    tm_wait_ld8(v);
                    if (holds && tcs == cmin) {
                        const int e = first_eq8(v, byte_of(M1, cmin), wmin);
                        k = (gidx(cmin, e) << 1) | (int)((xb >> (8 * cmin + e)) & 1);
                    }
                }
                key = warp_min(k);
                gmin = warp_min(tg);
                int m = wmin;
                if (m == INT32_MAX) {
                    if (phase == 0) {                   // X == D: Straight ends (R-3)
                        phase = 1;
                        after_main = false;
                        continue;
                    }
                    // empty candidate set (R-7, R-8, R-11): argmin over M2, then over all bits
                    const bits_t M2 = pm_s[1][t];
                    int t2 = INT32_MAX;
                    for_chunks([&](int c, const int32_t* dc) {
                        const uint32_t mb = byte_of(M2, c);
#pragma unroll
                        for (int e = 0; e < 8; e++)
                            if ((mb >> e) & 1u) t2 = min(t2, dc[e]);
                    });
                    int m2 = warp_min(t2);
                    bits_t MM = M2;
                    if (m2 == INT32_MAX) { MM = vb; t2 = tg; m2 = gmin; }
                    m = m2;
                    int k2 = INT32_MAX;
                    if (__any_sync(FULL, t2 == m)) {
                        const bool mine = t2 == m;
                        for_chunks([&](int c, const int32_t* dc) {
                            const uint32_t mb = byte_of(MM, c);
#pragma unroll
                            for (int e = 0; e < 8; e++)
                                if (mine && ((mb >> e) & 1u) && dc[e] == m)
                                    k2 = min(k2, (gidx(c, e) << 1) | (int)((xb >> (8 * c + e)) & 1));
                        });
                    }
                    key = warp_min(k2);
                }
                si = key >> 1;
                sx = key & 1;
                sv = m;
            } else if (kind == 2) {
                // TwoNeighbor: the owner lane of fixed_i publishes Delta_i and x_i
                const int q = tt - 1;
                const int fixed_i = q == 0 ? 0 : ((q & 1) ? (q + 1) >> 1 : (q >> 1) - 1);
                int32_t v1;
                tm_ld1(tw + lbit(fixed_i), v1);
                const int src = (fixed_i >> 3) & 31;
                gmin = warp_min(tg);
                si = fixed_i;
                sv = __shfl_sync(FULL, v1, src);
                sx = __shfl_sync(FULL, (int)((xb >> lbit(fixed_i)) & 1), src);
            } else {
                // MaxMin (R-6) / PositiveMin (R-9)
                if (algo != ALG_MAXMIN) a1 = tp < 0x7FFFFFFEu ? (int)tp + 1 : INT32_MAX;
                gmin = warp_min(tg);
                int lo = warp_min(a1), hi = warp_max(a2);
                const bool any_el = __any_sync(FULL, M1 != 0);
                bits_t EL = M1;
                int thr;
                const uint2 r = draw(flips);
                if (!any_el) {
                    // every bit tabu: drop tabu (R-11)
                    EL = vb;
                    int b1 = INT32_MIN;
                    unsigned b2 = 0xFFFFFFFFu;
                    for_chunks([&](int c, const int32_t* dc) {
                        const uint32_t mb = byte_of(vb, c);
#pragma unroll
                        for (int e = 0; e < 8; e++)
                            if ((mb >> e) & 1u) { b1 = max(b1, dc[e]); b2 = min(b2, (unsigned)(dc[e] - 1)); }
                    });
                    b1 = warp_max(b1);
                    const int bp = (int)warp_min((int)(b2 < 0x7FFFFFFEu ? b2 + 1 : INT32_MAX));
                    lo = algo == ALG_MAXMIN ? gmin : bp;
                    hi = b1;
                }
                uint32_t u;
                if (algo == ALG_MAXMIN) {
                    // span = floor((hi - lo) u^3 / T^3) exactly (R-6), as tm_batch_kernel
                    const uint64_t uu = (uint64_t)(T - tt);
                    const uint64_t a = (uint64_t)((int64_t)hi - lo), f = uu * uu * uu, qd = (uint64_t)T * T * T;
                    uint64_t span = __umul64hi(a, p.mtab[tt]);
                    if (a * f - span * qd >= qd) span++;
                    thr = (int)((int64_t)lo + (int64_t)(((unsigned __int128)r.x * (span + 1)) >> 32));
                    u = r.y;
                } else {
                    thr = lo;
                    u = r.x;
                }
                // candidates (Delta <= thr, eligible) per chunk, packed 2 x 16 bits per word
                uint32_t pk[CW];
#pragma unroll
                for (int j = 0; j < CW; j++) pk[j] = 0;
#pragma unroll
                for (int h = 0; h < HP; h++) {
                    int32_t v[16];
                    tm_ld16(tw + 16 * h, v);
                    tm_wait_ld16(v);
#pragma unroll
                    for (int cc = 0; cc < 2; cc++) {
                        const int c = 2 * h + cc;
                        uint32_t byte = 0;
#pragma unroll
                        for (int e = 0; e < 8; e++) byte |= (uint32_t)(v[8 * cc + e] <= thr) << e;
                        byte &= byte_of(EL, c);
                        pk[c >> 1] += (uint32_t)__popc(byte) << (16 * (c & 1));
                    }
                }
                uint32_t bt[CW];
#pragma unroll
                for (int j = 0; j < CW; j++) bt[j] = warp_add(pk[j]);
                uint32_t tot = 0;
#pragma unroll
                for (int c = 0; c < C; c++) tot += (bt[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                int r1 = (int)pick_u(u, tot);
                int cs = 0;
#pragma unroll
                for (int c = 0; c < C; c++) {
                    const int tc = (int)((bt[c >> 1] >> (16 * (c & 1))) & 0xFFFFu);
                    if (cs == c && r1 >= tc) { r1 -= tc; cs = c + 1; }
                }
                int32_t v8[8];
                tm_ld8(tw + 8 * cs, v8);
                tm_wait_ld8(v8);
                uint32_t mybyte = 0;
#pragma unroll
                for (int e = 0; e < 8; e++) mybyte |= (uint32_t)(v8[e] <= thr) << e;
                mybyte &= byte_of(EL, cs);
                const uint32_t lt = (1u << lane) - 1u;
                int y0 = 0;
#pragma unroll
                for (int e = 0; e < 8; e++) y0 += __popc(__ballot_sync(FULL, (mybyte >> e) & 1u) & lt);
                const int xc = __popc(mybyte);
                const bool mine = r1 >= y0 && r1 < y0 + xc;
                int gi = -1, lv = 0, lx = 0;
                if (mine) {
                    uint32_t byte = mybyte;
                    for (int j = 0; j < r1 - y0; j++) byte &= byte - 1;
                    const int e = __ffs(byte) - 1;
                    gi = gidx(cs, e);
                    lv = pick8(v8, e);
                    lx = (int)((xb >> (8 * cs + e)) & 1);
                }
                const int src = __ffs(__ballot_sync(FULL, mine)) - 1;
                si = __shfl_sync(FULL, gi, src);
                sv = __shfl_sync(FULL, lv, src);
                sx = __shfl_sync(FULL, lx, src);
            }

            // ---------------- Step 1: BEST (R-2, R-3)
            const bool g_exact = !skip_g || phase == 1 || (kind == 1 && algo == ALG_MAXMIN);
            if (g_exact) glb = gmin;
            else gmin = INT32_MAX;
            if (E + gmin < ebest) {
                int bk = key;
                if (kind != 0 || masked) {
                    int k3 = INT32_MAX;
                    if (__any_sync(FULL, tg == gmin)) {
                        const bool mine = tg == gmin;
                        for_chunks([&](int c, const int32_t* dc) {
#pragma unroll
                            for (int e = 0; e < 8; e++)
                                if (mine && dc[e] == gmin) k3 = min(k3, (gidx(c, e) << 1) | (int)((xb >> (8 * c + e)) & 1));
                        });
                    }
                    bk = warp_min(k3);
                }
                ebest = E + gmin;
                const int j = bk >> 1;
                pm_s[2][t] = owns(j) ? (ONE << lbit(j)) : (bits_t)0;
            }
            if (phase == 1 && gmin >= 0) {
                // Greedy reached a local minimum (R-4): next round, or the batch ends (R-12)
                if (after_main && (algo == ALG_TWO || flips >= p.B)) break;
                if (TRACE && after_main) round++;
                phase = 2;
                tt = 0;
                continue;
            }

            // ---------------- Step 3: flip bit si, Eqs.(4)-(5)
            __syncwarp();                     // every lane has consumed the previous row
            if (lane == 0) issue_row(si);
            E += sv;
            const int rmax_si = p.rmax[si];
            {
                // Eq.(5) by the owner lane (W_ii = 0, so the update leaves Delta_i alone)
                const int kk = lbit(si);
                const bool own = owns(si);
                int32_t v1;
                tm_ld1(tw + kk, v1);
                tm_st1(tw + kk, own ? -v1 : v1);
                if (own) {
                    xb ^= ONE << kk;
                    pm_s[2][t] ^= ONE << kk;
                }
                tm_wait_st();
            }
            pos = (pos + TABU_RING - 1) & (TABU_RING - 1);
            ring_s[pos] = si;
            __syncwarp();
            if (tabu > 0) {
                if (owns(si)) tm |= ONE << lbit(si);
                const int r = ring_s[(pos + tabu) & (TABU_RING - 1)];
                if (r >= 0) {
                    const bool inwin = __any_sync(FULL, lane < tabu && ring_s[(pos + lane) & (TABU_RING - 1)] == r);
                    if (owns(r) && !inwin) tm &= ~(ONE << lbit(r));
                }
            }
            if constexpr (TRACE) {
                if (lane == 0 && s == p.trace_slot && flips < p.tr_cap) {
                    p.tr_bit[flips] = si;
                    p.tr_E[flips] = E;
                    p.tr_phase[flips] = (int8_t)(phase == 2 ? 2 + min(round, 100) : phase);
                }
            }
            flips++;
            setup();
            reset_partials();
            const uint32_t sxm = sx ? 0u : 0xFFu;
            auto upd_scan = [&](auto MODE) {
                int32_t va[16], vb2[16];
                tm_ld16(tw, va);
                // the chunks' mask bytes (RandomMin: the hashes) while the row is in flight
                uint32_t mbs[C];
#pragma unroll
                for (int c = 0; c < C; c++) mbs[c] = chunk_mask(MODE, c);
                auto chunk = [&](int32_t* d8, const int c, const uint4 rw) {
                    const uint32_t mb = mbs[c];
                    const uint4 B = lut_s[byte_of(xb, c) ^ sxm];
                    d8[0] = __dp2a_lo((int)rw.x, (int)B.x, d8[0]);
                    d8[1] = __dp2a_hi((int)rw.x, (int)B.x, d8[1]);
                    d8[2] = __dp2a_lo((int)rw.y, (int)B.y, d8[2]);
                    d8[3] = __dp2a_hi((int)rw.y, (int)B.y, d8[3]);
                    d8[4] = __dp2a_lo((int)rw.z, (int)B.z, d8[4]);
                    d8[5] = __dp2a_hi((int)rw.z, (int)B.z, d8[5]);
                    d8[6] = __dp2a_lo((int)rw.w, (int)B.w, d8[6]);
                    d8[7] = __dp2a_hi((int)rw.w, (int)B.w, d8[7]);
                    scan_chunk(MODE, c, d8, mb);
                };
                mbar_wait(mbar, par_row);
#pragma unroll
                for (int h = 0; h < HP; h += 2) {
                    tm_wait_ld16(va);
                    if (h + 1 < HP) tm_ld16(tw + 16 * (h + 1), vb2);
                    chunk(va, 2 * h, row_s[((2 * h) << lgNT) + t]);
                    chunk(va + 8, 2 * h + 1, row_s[((2 * h + 1) << lgNT) + t]);
                    tm_st16(tw + 16 * h, va);
                    if (h + 1 < HP) {
                        tm_wait_ld16(vb2);
                        if (h + 2 < HP) tm_ld16(tw + 16 * (h + 2), va);
                        chunk(vb2, 2 * h + 2, row_s[((2 * h + 2) << lgNT) + t]);
                        chunk(vb2 + 8, 2 * h + 3, row_s[((2 * h + 3) << lgNT) + t]);
                        tm_st16(tw + 16 * (h + 1), vb2);
                    }
                }
            };
            switch (smode) {
            case SM_G: upd_scan(IG{}); break;
            case SM_M: upd_scan(IM{}); break;
            case SM_R: upd_scan(IR{}); break;
            case SM_T: upd_scan(IT{}); break;
            case SM_MM: upd_scan(IMM{}); break;
            default: upd_scan(IPM{}); break;
            }
            tm_wait_st();
            have = true;
            par_row ^= 1u;
            glb = min(glb - (int64_t)rmax_si, (int64_t)-sv);
        }

        // ---------------- write back state and the result packet
        {
            uint8_t* Xb = reinterpret_cast<uint8_t*>(p.X + (size_t)s * p.nwp);
            uint8_t* Bb = reinterpret_cast<uint8_t*>(p.best + (size_t)s * p.nwp);
            int32_t* dp = p.delta + (size_t)s * p.n_pad;
            const bits_t bb = xb ^ pm_s[2][t];
            for_chunks([&](int c, const int32_t* dc) {
                const int ch = (c << lgNT) + t;
                Xb[ch] = (uint8_t)byte_of(xb, c);
                Bb[ch] = (uint8_t)byte_of(bb, c);
                reinterpret_cast<int4*>(dp + ch * 8)[0] = make_int4(dc[0], dc[1], dc[2], dc[3]);
                reinterpret_cast<int4*>(dp + ch * 8)[1] = make_int4(dc[4], dc[5], dc[6], dc[7]);
            });
            p.ring[(size_t)s * TABU_RING + t] = ring_s[(pos + t) & (TABU_RING - 1)];
            if (lane == 0) {
                p.E[s] = E;
                p.ebest[s] = ebest;
                p.flips[s] = flips;
                atomicAdd(p.flip_total, (unsigned long long)flips);
            }
        }
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if (w == 0) tm_dealloc(tbase_s, TCOLS);
}

}  // namespace dabs
