// tmem_kernel.cuh -- the TMEM tier of the DABS hot loop (16384 < n <= 32768) on sm_100a.
//
// One 256-thread CTA per search and TWO searches per SM.  Delta (int32, 128 KB
// per search at n = 32768) does not fit twice in the register file, so it lives
// in tensor memory: each CTA allocates 256 TMEM columns (all 128 lanes), warp w
// owns lanes 32*(w%4).. and columns 128*(w/4)..+128, so thread t holds its 128
// elements as 128 columns of its lane.  Per flip every thread streams its
// Delta through registers once (tcgen05.ld 32 columns, Eq.(4) update with the
// W row piece, the next step's Step 1 + Step 2 scans, tcgen05.st back), so the
// row fetch and selection of one search overlap the other search's update:
// the one-search-per-SM register tier (batch_kernel<8,512,1>) leaves HBM idle
// while it selects (DESIGN 5, profiles/r01_timing_r32k.txt).
//
// Element k lives in thread t = (k/8) mod 256, chunk c = (k/8) / 256, e = k mod 8
// (the same chunk-major order as the register tiers, C = 16 chunks), at TMEM
// column 8c + e of the thread's lane.  sigma(x_k) bytes for the IDP.2A update
// come from a 256-entry table indexed by 8 x bits (no per-element sign copy).
// Tabu bits (R-11) are kept without per-element counts: when a flip leaves the
// tabu window its owner checks the window in one warp vote.
//
// Semantics are those of batch_body (batch_kernel.cuh) bit for bit; the GPU
// parity tests compare both against the oracle.  P:n = PAPER.md line n.
#pragma once
#include "batch_kernel.cuh"

namespace dabs {

constexpr int TM_NT = 256;   // threads per search (R32K tier; the n > 32768 variant runs 512)
constexpr int TM_C = 16;     // chunks of 8 elements per thread
constexpr int TM_NP = 4;     // W-row pieces per flip (one mbarrier each)
constexpr int TM_COLS = 256; // TMEM columns per CTA (= threads per search)
// dynamic shared memory of a TMEM-tier CTA: the W row, then the mask and chunk-minimum arrays
inline size_t tm_dyn_smem(int n_pad, int nt) { return 2 * (size_t)n_pad + (3 * 16 + TM_C * 4) * (size_t)nt; }

// ---------------------------------------------------------------- tcgen05 helpers
__device__ __forceinline__ void tm_alloc(uint32_t* dst_smem, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_dealloc(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

#define DABS_R8(v, o) "=r"(v[o + 0]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), "=r"(v[o + 5]), \
                      "=r"(v[o + 6]), "=r"(v[o + 7])
#define DABS_W8(v, o) "+r"(v[o + 0]), "+r"(v[o + 1]), "+r"(v[o + 2]), "+r"(v[o + 3]), "+r"(v[o + 4]), "+r"(v[o + 5]), \
                      "+r"(v[o + 6]), "+r"(v[o + 7])
#define DABS_S8(v, o) "r"(v[o + 0]), "r"(v[o + 1]), "r"(v[o + 2]), "r"(v[o + 3]), "r"(v[o + 4]), "r"(v[o + 5]), \
                      "r"(v[o + 6]), "r"(v[o + 7])

// 32 consecutive columns of this warp's 32 lanes (thread = lane): v[j] = column j
__device__ __forceinline__ void tm_ld32(uint32_t ta, int32_t (&v)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : DABS_R8(v, 0), DABS_R8(v, 8), DABS_R8(v, 16), DABS_R8(v, 24)
        : "r"(ta));
}
// wait for this thread's TMEM loads (ptxas tracks the LDTM destinations on a
// scoreboard; the wait orders the load against later TMEM stores of the thread)
__device__ __forceinline__ void tm_wait_ld32(int32_t (&)[32])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_st32(uint32_t ta, const int32_t (&v)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        DABS_S8(v, 0), DABS_S8(v, 8), DABS_S8(v, 16), DABS_S8(v, 24)
        : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t ta, int32_t (&v)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : DABS_R8(v, 0), DABS_R8(v, 8)
                 : "r"(ta));
}
__device__ __forceinline__ void tm_wait_ld16(int32_t (&)[16])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_st16(uint32_t ta, const int32_t (&v)[16])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(ta), DABS_S8(v, 0), DABS_S8(v, 8)
                 : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, int32_t (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : DABS_R8(v, 0) : "r"(ta));
}
__device__ __forceinline__ void tm_wait_ld8(int32_t (&v)[8])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;" : DABS_W8(v, 0) : : "memory");
}
__device__ __forceinline__ void tm_ld1(uint32_t ta, int32_t& v)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v) : : "memory");
}
__device__ __forceinline__ void tm_st1(uint32_t ta, int32_t v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta), "r"(v) : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
#undef DABS_R8
#undef DABS_W8
#undef DABS_S8

// 128-bit per-thread masks, byte c = chunk c
struct M128 {
    uint64_t lo, hi;
};
__device__ __forceinline__ uint32_t mbyte(const M128& m, int c)
{
    return (uint32_t)((c < 8 ? m.lo : m.hi) >> (8 * (c & 7))) & 0xFFu;
}
__device__ __forceinline__ M128 mand(M128 a, M128 b) { return {a.lo & b.lo, a.hi & b.hi}; }
__device__ __forceinline__ M128 mandn(M128 a, M128 b) { return {a.lo & ~b.lo, a.hi & ~b.hi}; }
__device__ __forceinline__ M128 mxor(M128 a, M128 b) { return {a.lo ^ b.lo, a.hi ^ b.hi}; }
__device__ __forceinline__ bool mnz(M128 a) { return (a.lo | a.hi) != 0; }
__device__ __forceinline__ bool mtest(const M128& m, int k) { return ((k < 64 ? m.lo : m.hi) >> (k & 63)) & 1; }
__device__ __forceinline__ void mflip(M128& m, int k)
{
    const uint64_t b = 1ull << (k & 63);
    if (k < 64) m.lo ^= b; else m.hi ^= b;
}
__device__ __forceinline__ void mset(M128& m, int k)
{
    const uint64_t b = 1ull << (k & 63);
    if (k < 64) m.lo |= b; else m.hi |= b;
}
__device__ __forceinline__ void mclr(M128& m, int k)
{
    const uint64_t b = 1ull << (k & 63);
    if (k < 64) m.lo &= ~b; else m.hi &= ~b;
}
__device__ __forceinline__ void mor_byte(M128& m, int c, uint32_t b)
{
    if (c < 8) m.lo |= (uint64_t)b << (8 * c); else m.hi |= (uint64_t)b << (8 * (c - 8));
}

// chunks 4q..4q+3 of a mask as one word (byte cc = chunk 4q+cc)
__device__ __forceinline__ uint32_t pword(const M128& m, int q)
{
    return (uint32_t)((q < 2 ? m.lo : m.hi) >> (32 * (q & 1)));
}
__device__ __forceinline__ void mor_word(M128& m, int q, uint32_t w)
{
    if (q < 2) m.lo |= (uint64_t)w << (32 * (q & 1)); else m.hi |= (uint64_t)w << (32 * (q & 1));
}

// first e in 0..7 with mask bit e set and v[e] == m (or -1)
__device__ __forceinline__ int first_eq8(const int32_t (&v)[8], uint32_t mask, int m)
{
    int r = -1;
#pragma unroll
    for (int e = 7; e >= 0; e--)
        if (((mask >> e) & 1u) && v[e] == m) r = e;
    return r;
}
__device__ __forceinline__ int pick8(const int32_t (&v)[8], int e)
{
    int r = v[0];
#pragma unroll
    for (int j = 1; j < 8; j++)
        if (e == j) r = v[j];
    return r;
}

#ifdef DABS_TIMING
// diagnostic build only: per flip, thread 0's SM cycles in each row piece of the
// update: [3q] TMEM load, [3q+1] wait for the row piece, [3q+2] update + scan; [12] store drain
__device__ unsigned long long g_tstat3[16];
#endif

// CTA-wide state that outlives one batch (the persistent asynchronous kernel
// runs many): the TMEM allocation, the sigma table, the row mbarriers and
// their phase parity
__shared__ __align__(8) uint64_t tm_mbar_s[TM_NP];
__shared__ uint32_t tm_tbase_s;
__shared__ uint32_t tm_par_s;
__shared__ uint4 tm_lut_s[256];   // sigma bytes of 8 elements as the four IDP.2A B words

// once per CTA: NT TMEM columns, the sigma table, the row mbarriers
template <int NT>
__device__ __forceinline__ void tm_cta_setup()
{
    const int t = threadIdx.x, wid = t >> 5;
    if (wid == 0) tm_alloc(&tm_tbase_s, NT);
    // sigma table: entry v = x bits of 8 elements, word j = (s_2j, 0, 0, s_2j+1),
    // s = 0x01 for x = 1 (+1), 0xFF for x = 0 (-1)
    {
        const uint32_t v = (uint32_t)t;
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t s0 = ((v >> (2 * j)) & 1u) ? 0x01u : 0xFFu, s1 = ((v >> (2 * j + 1)) & 1u) ? 0x01u : 0xFFu;
            w[j] = s0 | (s1 << 24);
        }
        if (t < 256) tm_lut_s[t] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (t == 0) {
#pragma unroll
        for (int q = 0; q < TM_NP; q++) mbar_init(&tm_mbar_s[q], 1);
        fence_mbar_init();
        tm_par_s = 0;
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
}
template <int NT>
__device__ __forceinline__ void tm_cta_teardown()
{
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if ((threadIdx.x >> 5) == 0) tm_dealloc(tm_tbase_s, NT);
}

// One batch search of slot s with Delta in TMEM.  REUSE: the CTA
// runs further batches (persistent asynchronous kernel): packets written by
// the commit warp are read from L2, the row mbarriers' parity carries over.
// NT = 256 (n <= 32768, 256 TMEM columns, two CTAs per SM) or 512 (n <= 65536,
// all 512 columns, one CTA per SM); warp w: lanes 32(w%4).., columns 128(w/4)..
template <int NT, bool TRACE, bool REUSE>
__device__ __forceinline__ void tm_batch_body(const BatchParams& p, const int s, const uint32_t gen)
{
    constexpr int lgNT = NT == 512 ? 9 : 8, C = TM_C, NW = NT / 32, NP = TM_NP, CPP = C / NP, CW = C / 2;
    constexpr unsigned FULL = 0xffffffffu;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const uint32_t gslot = p.slot_base + (uint32_t)s;
    const int n = p.n;

    extern __shared__ __align__(128) uint8_t dyn_smem[];
    const uint4* row_s = reinterpret_cast<const uint4*>(dyn_smem);   // one W row, 2*n_pad bytes
    uint64_t* mbar = tm_mbar_s;
    const uint4* lut_s = tm_lut_s;
    __shared__ int32_t ring_s[TABU_RING];
    __shared__ int32_t red_s[2][32][RED_W];
    __shared__ int32_t bc_s[2][4];
    __shared__ int32_t sel_s[4];
    // after the row in dynamic shared memory (48 KB static limit at NT = 512):
    // [0] D bits, [1] M2, [2] BEST xor X; MaxMin / PositiveMin chunk minima of the last scan
    M128 (*pm_s)[NT] = reinterpret_cast<M128 (*)[NT]>(dyn_smem + 2 * (size_t)p.n_pad);
    int32_t (*cmin_s)[NT] = reinterpret_cast<int32_t (*)[NT]>(dyn_smem + 2 * (size_t)p.n_pad + 3 * NT * sizeof(M128));
    const uint32_t tw = tm_tbase_s + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)(128 * (wid >> 2));   // this warp's base

    // ---------------- load the slot's persistent state (R-14)
    M128 xb{0, 0}, vb{0, 0};
    {
        const uint8_t* Xb = reinterpret_cast<const uint8_t*>(p.X + (size_t)s * p.nwp);
        const uint8_t* Db = reinterpret_cast<const uint8_t*>(p.D + (size_t)s * p.nwp);
        const int32_t* dp = p.delta + (size_t)s * p.n_pad;
        M128 db{0, 0};
#pragma unroll
        for (int q = 0; q < NP; q++) {
            int32_t v[32];
#pragma unroll
            for (int cc = 0; cc < CPP; cc++) {
                const int c = q * CPP + cc;
                const int ch = (c << lgNT) + t;
                mor_byte(xb, c, Xb[ch]);
                mor_byte(db, c, REUSE ? __ldcg(Db + ch) : Db[ch]);
                const int nv = min(max(n - ch * 8, 0), 8);
                mor_byte(vb, c, (1u << nv) - 1u);
                const int4 a = reinterpret_cast<const int4*>(dp + ch * 8)[0];
                const int4 b = reinterpret_cast<const int4*>(dp + ch * 8)[1];
                v[8 * cc + 0] = a.x; v[8 * cc + 1] = a.y; v[8 * cc + 2] = a.z; v[8 * cc + 3] = a.w;
                v[8 * cc + 4] = b.x; v[8 * cc + 5] = b.y; v[8 * cc + 6] = b.z; v[8 * cc + 7] = b.w;
            }
            tm_st32(tw + 32 * q, v);
        }
        pm_s[0][t] = db;
        pm_s[2][t] = M128{0, 0};
    }
    tm_wait_st();
    if (t < TABU_RING) ring_s[t] = REUSE ? __ldcg(p.ring + (size_t)s * TABU_RING + t) : p.ring[(size_t)s * TABU_RING + t];
    int pos = 0;   // ring_s[(pos + j) & 31] = j-th most recent flip
    int64_t E = REUSE ? (int64_t)__ldcg(reinterpret_cast<const long long*>(p.E + s)) : p.E[s];
    const int algo = REUSE ? (int)__ldcg(p.algo + s) : (int)p.algo[s];
    const int tabu = p.tabu;
    const int T = p.T;
    uint32_t par_row = tm_par_s;   // 0 at every launch; carried across batches (REUSE)
    int flips = 0;
    int64_t ebest = E_INF;
    int rc = 0;
    __syncthreads();

    auto gidx = [&](int c, int e) { return (((c << lgNT) + t) << 3) | e; };
    auto owns = [&](int k) { return ((k >> 3) & (NT - 1)) == t; };
    auto lbit = [&](int k) { return (((k >> 3) >> lgNT) << 3) | (k & 7); };   // local element = TMEM column
    const uint32_t piece_bytes = (uint32_t)(2 * p.n_pad / NP);
    auto issue_row = [&](int i) {
        fence_proxy_async();
        const char* src = reinterpret_cast<const char*>(p.W) + (size_t)i * (size_t)(2 * p.n_pad);
#pragma unroll
        for (int q = 0; q < NP; q++) bulk_row_piece(dyn_smem + q * piece_bytes, src + q * piece_bytes, piece_bytes, &mbar[q]);
    };

    int phase = 0, round = 0, tt = 0, cursor = 0;
    bool after_main = false;
    M128 tm{0, 0};                 // tabu bits of this thread's elements (R-11)
    int64_t glb = INT64_MIN / 4;   // lower bound on min Delta (batch_body)
    for (int j = 0; j < tabu; j++) {
        const int r = ring_s[j];
        if (r >= 0 && owns(r)) mset(tm, lbit(r));
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
    // RandomMin candidates of chunk c (R-8)
    auto cand_byte = [&](int c, uint32_t K, uint32_t p16) -> uint32_t {
        if (p16 >= 65536u) return mbyte(vb, c);
        return randmin_byte(K, (uint32_t)(((c << lgNT) + t) << 2), p16);
    };

#ifdef DABS_TIMING
    __shared__ unsigned int ts_s[6][5];
    __shared__ unsigned int ts2_s[10];
    __shared__ unsigned long long ts3_s[16];
    long long tlast = 0, tp3 = 0;
    if (t == 0) {
        for (int j = 0; j < 30; j++) (&ts_s[0][0])[j] = 0u;
        for (int j = 0; j < 10; j++) ts2_s[j] = 0u;
        for (int j = 0; j < 16; j++) ts3_s[j] = 0u;
    }
#define DABS_T3(k) do { if (t == 0) { const long long now_ = clock64(); ts3_s[k] += now_ - tp3; tp3 = now_; } } while (0)
    long long tA = clock64(), tB = 0, tC = 0, tD = tA;
    int tbk = 5;
#else
#define DABS_T3(k) do { } while (0)
#endif

    // ---------------- Step 2 setup (uniform) and the scan modes
    constexpr int SM_G = 0, SM_M = 1, SM_R = 2, SM_T = 3, SM_MM = 4, SM_PM = 5;
    int kind = 0;
    bool masked = true;
    M128 M1 = vb;                  // candidates (kind 0) / eligible bits (kind 1)
    int smode = SM_G;
    uint32_t cmeet = 0xFFFFu;      // chunks the CyclicMin window meets (uniform)
    uint32_t rK = 0, rp16 = 0;
    auto setup = [&]() {
        if (phase == 2 && tt == (algo == ALG_TWO ? 2 * n - 1 : T)) {   // main run ends
            phase = 1;
            after_main = true;
        }
        kind = 0;
        masked = true;
        cmeet = 0xFFFFu;
        if (phase == 0) {
            M1 = mand(mxor(xb, pm_s[0][t]), vb);                       // Straight
        } else if (phase == 1) {
            masked = false;                                            // Greedy
            M1 = M128{~0ull, ~0ull};
        } else {
            tt++;
            if (tt == 1) cursor = 0;
            if (algo == ALG_CYCLIC) {                                  // CyclicMin (R-7)
                const int w = p.wtab[tt];
                const int b0 = min(cursor + w, n), b1 = cursor + w - n;
                M128 wm{0, 0};
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
                        mor_byte(wm, c, byte);
                    }
                }
                cursor += w;
                if (cursor >= n) cursor -= n;
                M1 = mandn(wm, tm);
                pm_s[1][t] = wm;
            } else if (algo == ALG_RANDOM) {                           // RandomMin (R-8)
                rp16 = (uint32_t)p.ptab[tt];
                rK = rp16 >= 65536u ? 0u : draw(flips).x;
                M1 = M128{0, 0};                                       // filled by the scan
                pm_s[1][t] = mandn(vb, tm);
            } else if (algo == ALG_TWO) {                              // TwoNeighbor (R-10)
                kind = 2;
            } else {
                kind = 1;                                              // MaxMin / PositiveMin
                M1 = mandn(vb, tm);
            }
        }
        smode = kind == 2 ? SM_T
              : kind == 1 ? (algo == ALG_MAXMIN ? SM_MM : SM_PM)
              : !masked ? SM_G
              : (algo == ALG_RANDOM && phase == 2) ? SM_R : SM_M;
    };

    // per-thread scan partials
    int tg = INT32_MAX, tsel = INT32_MAX, tcs = 0, a1 = INT32_MAX, a2 = INT32_MIN;
    unsigned tp = 0xFFFFFFFFu;
    auto reset_partials = [&]() {
        tg = INT32_MAX; tsel = INT32_MAX; tcs = 0; a1 = INT32_MAX; a2 = INT32_MIN; tp = 0xFFFFFFFFu;
    };
    // scan of chunk c (values dc[0..7]) for mode MODE; cb = RandomMin candidate byte
    // the scan of chunk c (values dc[0..7]) for mode MODE; mb = the chunk's mask
    // byte: candidates (SM_M, SM_R) or eligible bits (SM_MM, SM_PM)
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
            cmin_s[c][t] = mn;          // the counting pass skips chunks whose minimum exceeds thr
            if (mb == 0xFFu) {
                const int mx = max(max(max(dc[0], dc[1]), max(dc[2], dc[3])), max(max(dc[4], dc[5]), max(dc[6], dc[7])));
                a1 = min(a1, mn);
                a2 = max(a2, mx);
            } else {
#pragma unroll
                for (int e = 0; e < 8; e++)
                    if ((mb >> e) & 1u) { a1 = min(a1, dc[e]); a2 = max(a2, dc[e]); }
            }
        } else {   // SM_PM
            tg = min(tg, mn);
            cmin_s[c][t] = mn;
            unsigned q = 0xFFFFFFFFu;
            if (mb == 0xFFu) {          // no tabu bit, no padding in the chunk (the common case)
#pragma unroll
                for (int e = 0; e < 8; e++) q = min(q, (unsigned)(dc[e] - 1));
            } else {
#pragma unroll
                for (int e = 0; e < 8; e++)
                    if ((mb >> e) & 1u) q = min(q, (unsigned)(dc[e] - 1));
            }
            tp = min(tp, q);
        }
    };
    // per piece q (chunks 4q..4q+3): the mask word the scans of MODE use (byte cc = chunk 4q+cc)
    auto piece_mask = [&](auto MODE, const int q, uint32_t (&cb)[CPP]) -> uint32_t {
        constexpr int md = decltype(MODE)::value;
        if constexpr (md == SM_R) {
            // RandomMin candidates (R-8) of the piece, restricted to valid non-tabu bits
            uint32_t w = 0;
#pragma unroll
            for (int cc = 0; cc < CPP; cc++) w |= cand_byte(q * CPP + cc, rK, rp16) << (8 * cc);
            return w & pword(vb, q) & ~pword(tm, q);
        } else if constexpr (md == SM_M || md == SM_MM || md == SM_PM) {
            return pword(M1, q);
        } else {
            return 0u;
        }
    };
    // the whole scan, reading Delta from TMEM (first step, after a phase change)
    auto scan_full = [&](auto MODE) {
        constexpr int md = decltype(MODE)::value;
#pragma unroll 1
        for (int q = 0; q < NP; q++) {
            uint32_t cb[CPP];
            const uint32_t pm = piece_mask(MODE, q, cb);
            if constexpr (md == SM_R) mor_word(M1, q, pm);
            int32_t v[32];
            tm_ld32(tw + 32 * q, v);
            tm_wait_ld32(v);
#pragma unroll
            for (int cc = 0; cc < CPP; cc++) scan_chunk(MODE, q * CPP + cc, v + 8 * cc, (pm >> (8 * cc)) & 0xFFu);
        }
    };
    // apply f(c, v8) to every chunk's 8 Delta values (rare full passes)
    auto for_chunks = [&](auto f) {
#pragma unroll 1
        for (int q = 0; q < NP; q++) {
            int32_t v[32];
            tm_ld32(tw + 32 * q, v);
            tm_wait_ld32(v);
#pragma unroll
            for (int cc = 0; cc < CPP; cc++) f(q * CPP + cc, v + 8 * cc);
        }
    };
    using IG = std::integral_constant<int, SM_G>;
    using IM = std::integral_constant<int, SM_M>;
    using IR = std::integral_constant<int, SM_R>;
    using IT = std::integral_constant<int, SM_T>;
    using IMM = std::integral_constant<int, SM_MM>;
    using IPM = std::integral_constant<int, SM_PM>;

    bool have = false;             // this step's partials came from the fused update
    while (true) {
#ifdef DABS_TIMING
        tA = clock64();
#endif
        const bool skip_g = E + glb >= ebest;   // no 1-bit neighbour can beat BEST (uniform)
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

        // ---------------- Step 1 + Step 2: exchange the partials (R-2..R-11)
        int si = 0, sv = 0, sx = 0;
        int gmin = 0;
        int key = INT32_MAX;
        if (kind == 0) {
            if (!masked) tg = tsel;
            const int wmin = warp_min(tsel);
            int k = INT32_MAX;
            const bool holds = tsel == wmin && wmin != INT32_MAX;
            if (__any_sync(FULL, holds)) {
                // the lowest chunk among the lanes holding the warp minimum: one
                // warp-wide TMEM load of that chunk, those lanes locate their key
                const int cmin = warp_min(holds ? tcs : INT32_MAX);
                int32_t v[8];
                tm_ld8(tw + 8 * cmin, v);
                tm_wait_ld8(v);
                if (holds && tcs == cmin) {
                    const int e = first_eq8(v, mbyte(M1, cmin), wmin);
                    k = (gidx(cmin, e) << 1) | (int)mtest(xb, 8 * cmin + e);
                }
            }
            k = warp_min(k);
            const int g = warp_min(tg);
            const int par = rc & 1;
            rc++;
            if (lane == 0) { red_s[par][wid][0] = wmin; red_s[par][wid][1] = k; red_s[par][wid][2] = g; }
            __syncthreads();
            const int a = lane < NW ? red_s[par][lane][0] : INT32_MAX;
            const int b = lane < NW ? red_s[par][lane][1] : INT32_MAX;
            const int c2 = lane < NW ? red_s[par][lane][2] : INT32_MAX;
            int m = warp_min(a);
            key = warp_min(a == m ? b : INT32_MAX);
            gmin = warp_min(c2);
            if (m == INT32_MAX) {
                if (phase == 0) {                   // X == D: Straight ends (R-3)
                    phase = 1;
                    after_main = false;
                    continue;
                }
                // empty candidate set (R-7, R-8, R-11): argmin over M2, then over all bits
                const M128 M2 = pm_s[1][t];
                int t2 = INT32_MAX;
                for_chunks([&](int c, const int32_t* dc) {
                    const uint32_t mb = mbyte(M2, c);
#pragma unroll
                    for (int e = 0; e < 8; e++)
                        if ((mb >> e) & 1u) t2 = min(t2, dc[e]);
                });
                int v2[1] = {t2};
                const int ops1[1] = {OP_MIN};
                block_reduce<true>(v2, ops1, red_s, rc, lane, wid, NW);
                M128 MM = M2;
                if (v2[0] == INT32_MAX) { MM = vb; t2 = tg; v2[0] = gmin; }
                m = v2[0];
                int k2 = INT32_MAX;
                if (__any_sync(FULL, t2 == m)) {
                    const bool mine = t2 == m;
                    for_chunks([&](int c, const int32_t* dc) {
                        const uint32_t mb = mbyte(MM, c);
#pragma unroll
                        for (int e = 0; e < 8; e++)
                            if (mine && ((mb >> e) & 1u) && dc[e] == m) k2 = min(k2, (gidx(c, e) << 1) | (int)mtest(xb, 8 * c + e));
                    });
                }
                int kv[1] = {k2};
                block_reduce<true>(kv, ops1, red_s, rc, lane, wid, NW);
                key = kv[0];
            }
            si = key >> 1;
            sx = key & 1;
            sv = m;
        } else if (kind == 2) {
            // TwoNeighbor: the owner of fixed_i publishes Delta_i and x_i
            const int q = tt - 1;
            const int fixed_i = q == 0 ? 0 : ((q & 1) ? (q + 1) >> 1 : (q >> 1) - 1);
            const bool own = owns(fixed_i);
            if (__any_sync(FULL, own)) {
                int32_t v1;
                tm_ld1(tw + lbit(fixed_i), v1);
                if (own) { bc_s[rc & 1][0] = v1; bc_s[rc & 1][1] = (int)mtest(xb, lbit(fixed_i)); }
            }
            int v[1] = {tg};
            const int ops[1] = {OP_MIN};
            block_reduce<true>(v, ops, red_s, rc, lane, wid, NW);
            gmin = v[0];
            si = fixed_i;
            sv = bc_s[(rc - 1) & 1][0];
            sx = bc_s[(rc - 1) & 1][1];
        } else {
            // MaxMin (R-6) / PositiveMin (R-9)
            if (algo != ALG_MAXMIN) a1 = tp < 0x7FFFFFFEu ? (int)tp + 1 : INT32_MAX;
            int v[4] = {tg, a1, a2, (int)mnz(M1)};
            const int ops[4] = {OP_MIN, OP_MIN, OP_MAX, OP_OR};
            DABS_TS(0);
            block_reduce<true>(v, ops, red_s, rc, lane, wid, NW);
            DABS_TS(1);
            gmin = v[0];
            M128 EL = M1;
            int thr;
            const uint2 r = draw(flips);
            if (!v[3]) {
                // every bit tabu: drop tabu (R-11)
                EL = vb;
                int b1 = INT32_MIN;
                unsigned b2 = 0xFFFFFFFFu;
                for_chunks([&](int c, const int32_t* dc) {
                    const uint32_t mb = mbyte(vb, c);
#pragma unroll
                    for (int e = 0; e < 8; e++)
                        if ((mb >> e) & 1u) { b1 = max(b1, dc[e]); b2 = min(b2, (unsigned)(dc[e] - 1)); }
                });
                int w2[2] = {b1, b2 < 0x7FFFFFFEu ? (int)b2 + 1 : INT32_MAX};
                const int ops2[2] = {OP_MAX, OP_MIN};
                block_reduce<true>(w2, ops2, red_s, rc, lane, wid, NW);
                v[1] = algo == ALG_MAXMIN ? gmin : w2[1];
                v[2] = w2[0];
            }
            uint32_t u;
            if (algo == ALG_MAXMIN) {
                // span = floor((hi - lo) u^3 / T^3) exactly (R-6): the estimate from the
                // step's 64-bit fraction is floor or floor - 1; one remainder test fixes it
                const uint64_t uu = (uint64_t)(T - tt);
                const uint64_t a = (uint64_t)((int64_t)v[2] - v[1]), f = uu * uu * uu, qd = (uint64_t)T * T * T;
                uint64_t span = __umul64hi(a, p.mtab[tt]);
                if (a * f - span * qd >= qd) span++;
                thr = (int)((int64_t)v[1] + (int64_t)(((unsigned __int128)r.x * (span + 1)) >> 32));
                u = r.y;
            } else {
                thr = v[1];
                u = r.x;
            }
            // count candidates (Delta <= thr, eligible) per chunk, packed 2 x 16 bits per word
            DABS_TS(2);
            uint32_t pk[CW];
#pragma unroll
            for (int w = 0; w < CW; w++) pk[w] = 0;
            {
                // x16 half-pieces (chunks c0, c0 + 1), the next load in flight
                auto count16 = [&](const int32_t (&v16)[16], const int c0) {
#pragma unroll
                    for (int cc = 0; cc < 2; cc++) {
                        const int c = c0 + cc;
                        uint32_t byte = 0;
#pragma unroll
                        for (int e = 0; e < 8; e++) byte |= (uint32_t)(v16[8 * cc + e] <= thr) << e;
                        byte &= mbyte(EL, c);
                        pk[c >> 1] += (uint32_t)__popc(byte) << (16 * (c & 1));
                    }
                };
                // a half-piece whose chunk minima (all elements, from the scan) exceed
                // thr in every lane of the warp holds no candidate: skip its TMEM
                // load (PositiveMin: thr = the least positive gain, so most are skipped)
#pragma unroll
                for (int hp = 0; hp < C / 2; hp++) {
                    const bool need = (cmin_s[2 * hp][t] <= thr) || (cmin_s[2 * hp + 1][t] <= thr);
                    if (__any_sync(FULL, need)) {
                        int32_t v16[16];
                        tm_ld16(tw + 16 * hp, v16);
                        tm_wait_ld16(v16);
                        count16(v16, 2 * hp);
                    }
                }
            }
            DABS_TS(3);
            uint32_t wt[CW];
#pragma unroll
            for (int w = 0; w < CW; w++) wt[w] = warp_add(pk[w]);
            const int par = rc & 1;
            rc++;
            if (lane == 0) {
#pragma unroll
                for (int w = 0; w < CW; w++) red_s[par][wid][w] = (int)wt[w];
            }
            __syncthreads();
            uint32_t bt[CW];
#pragma unroll
            for (int w = 0; w < CW; w++) bt[w] = warp_add(lane < NW ? (uint32_t)red_s[par][lane][w] : 0u);
            DABS_TS(4);
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
            DABS_TS(5);
            // which warp holds rank r1 of chunk cs (chunk-major order, then thread)
            const int x = lane < NW ? (int)(((uint32_t)red_s[par][lane][cs >> 1] >> (16 * (cs & 1))) & 0xFFFFu) : 0;
            const int pre = (int)warp_add(lane < wid ? (uint32_t)x : 0u);
            const int own = __shfl_sync(FULL, x, wid);
            const bool wsel = r1 >= pre && r1 < pre + own;
            r1 -= pre;
            DABS_TS(6);
            if (wsel) {
                int32_t v8[8];
                tm_ld8(tw + 8 * cs, v8);
                tm_wait_ld8(v8);
                uint32_t mybyte = 0;
#pragma unroll
                for (int e = 0; e < 8; e++) mybyte |= (uint32_t)(v8[e] <= thr) << e;
                mybyte &= mbyte(EL, cs);
                const uint32_t lt = (1u << lane) - 1u;
                int y0 = 0;
#pragma unroll
                for (int e = 0; e < 8; e++) y0 += __popc(__ballot_sync(FULL, (mybyte >> e) & 1u) & lt);
                const int xc = __popc(mybyte);
                if (r1 >= y0 && r1 < y0 + xc) {
                    uint32_t byte = mybyte;
                    for (int j = 0; j < r1 - y0; j++) byte &= byte - 1;
                    const int e = __ffs(byte) - 1;
                    sel_s[0] = gidx(cs, e);
                    sel_s[1] = pick8(v8, e);
                    sel_s[2] = (int)mtest(xb, 8 * cs + e);
                    issue_row(sel_s[0]);     // published through the row mbarrier
                }
            }
        }

        // ---------------- Step 1: BEST (R-2, R-3)
        const bool g_exact = !skip_g || phase == 1 || (kind == 1 && algo == ALG_MAXMIN);
        if (g_exact) glb = gmin;
        else gmin = INT32_MAX;
        if (E + gmin < ebest) {
            int bk = key;
            if (kind != 0 || masked) {
                // key of the lowest index holding gmin (rare: BEST improves)
                int k3 = INT32_MAX;
                if (__any_sync(FULL, tg == gmin)) {
                    const bool mine = tg == gmin;
                    for_chunks([&](int c, const int32_t* dc) {
#pragma unroll
                        for (int e = 0; e < 8; e++)
                            if (mine && dc[e] == gmin) k3 = min(k3, (gidx(c, e) << 1) | (int)mtest(xb, 8 * c + e));
                    });
                }
                int kv[1] = {k3};
                const int ops1[1] = {OP_MIN};
                block_reduce<true>(kv, ops1, red_s, rc, lane, wid, NW);
                bk = kv[0];
            }
            ebest = E + gmin;
            const int j = bk >> 1;
            M128 bd{0, 0};
            if (owns(j)) mset(bd, lbit(j));
            pm_s[2][t] = bd;
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
#ifdef DABS_TIMING
        tB = clock64();
        tbk = phase == 2 ? algo : 5;
        if (t == 0) { ts_s[tbk][0] += tB - tA; ts_s[tbk][3] += tA - tD; ts_s[tbk][4] += 1; }
#endif
        if (kind == 1) {
            mbar_wait(&mbar[0], par_row);
            DABS_TS(7);
            si = sel_s[0]; sv = sel_s[1]; sx = sel_s[2];
        } else if (t == 0) {
            issue_row(si);
        }
        E += sv;
        const int rmax_si = p.rmax[si];
        // Eq.(5) by the owner: Delta_i <- -Delta_i (W_ii = 0, so the update leaves it alone)
        if (__any_sync(FULL, owns(si))) {
            const int kk = lbit(si);
            int32_t v1;
            tm_ld1(tw + kk, v1);
            tm_st1(tw + kk, owns(si) ? -v1 : v1);
            if (owns(si)) {
                mflip(xb, kk);
                M128 bd = pm_s[2][t];
                mflip(bd, kk);
                pm_s[2][t] = bd;
            }
            tm_wait_st();
        }
        pos = (pos + TABU_RING - 1) & (TABU_RING - 1);
        ring_s[pos] = si;
        if (tabu > 0) {
            // tabu window (R-11): si enters, the (tabu+1)-th most recent flip leaves;
            // its bit clears unless it is still inside the window (one warp vote)
            if (owns(si)) mset(tm, lbit(si));
            const int r = ring_s[(pos + tabu) & (TABU_RING - 1)];
            if (r >= 0 && __any_sync(FULL, owns(r))) {
                const bool inwin = __any_sync(FULL, lane < tabu && ring_s[(pos + lane) & (TABU_RING - 1)] == r);
                if (owns(r) && !inwin) mclr(tm, lbit(r));
            }
        }
        if constexpr (TRACE) {
            if (t == 0 && s == p.trace_slot && flips < p.tr_cap) {
                p.tr_bit[flips] = si;
                p.tr_E[flips] = E;
                p.tr_phase[flips] = (int8_t)(phase == 2 ? 2 + min(round, 100) : phase);
            }
        }
        flips++;
        // the next step's setup while the row is in flight, then the update with
        // the next step's scans folded in
        setup();
        reset_partials();
        const uint32_t sxm = sx ? 0u : 0xFFFFFFFFu;   // sigma(x_i) = -1: complement the table indices
        // Delta streams through registers in x16 half-pieces (2 chunks), the TMEM
        // load of the next half-piece in flight while this one is updated
        auto upd_scan = [&](auto MODE) {
            constexpr int md = decltype(MODE)::value;
            int32_t va[16], vb2[16];
#ifdef DABS_TIMING
            if (t == 0) tp3 = clock64();
#endif
            tm_ld16(tw, va);
            // Eq.(4) on chunk c: Delta_k += W_ik sigma(x_i) sigma(x_k), then its scans
            auto chunk = [&](int32_t* d8, const int c, const uint32_t xbyte, const uint32_t mbyte_) {
                const uint4 rw = row_s[(c << lgNT) + t];
                const uint4 B = lut_s[xbyte];
                d8[0] = __dp2a_lo((int)rw.x, (int)B.x, d8[0]);
                d8[1] = __dp2a_hi((int)rw.x, (int)B.x, d8[1]);
                d8[2] = __dp2a_lo((int)rw.y, (int)B.y, d8[2]);
                d8[3] = __dp2a_hi((int)rw.y, (int)B.y, d8[3]);
                d8[4] = __dp2a_lo((int)rw.z, (int)B.z, d8[4]);
                d8[5] = __dp2a_hi((int)rw.z, (int)B.z, d8[5]);
                d8[6] = __dp2a_lo((int)rw.w, (int)B.w, d8[6]);
                d8[7] = __dp2a_hi((int)rw.w, (int)B.w, d8[7]);
                scan_chunk(MODE, c, d8, mbyte_);
            };
#pragma unroll 1
            for (int q = 0; q < NP; q++) {
                uint32_t cb[CPP];
                const uint32_t pm = piece_mask(MODE, q, cb);
                if constexpr (md == SM_R) mor_word(M1, q, pm);
                const uint32_t px = pword(xb, q) ^ sxm;   // sigma table indices of the piece's chunks
                tm_wait_ld16(va);
                tm_ld16(tw + 32 * q + 16, vb2);
                DABS_T3(3 * q);
                mbar_wait(&mbar[q], par_row);
                DABS_T3(3 * q + 1);
#ifdef DABS_TIMING
                if (q == 0) tC = clock64();
#endif
                chunk(va, 4 * q, px & 0xFFu, pm & 0xFFu);
                chunk(va + 8, 4 * q + 1, (px >> 8) & 0xFFu, (pm >> 8) & 0xFFu);
                tm_st16(tw + 32 * q, va);
                tm_wait_ld16(vb2);
                if (q + 1 < NP) tm_ld16(tw + 32 * q + 32, va);
                chunk(vb2, 4 * q + 2, (px >> 16) & 0xFFu, (pm >> 16) & 0xFFu);
                chunk(vb2 + 8, 4 * q + 3, px >> 24, pm >> 24);
                tm_st16(tw + 32 * q + 16, vb2);
                DABS_T3(3 * q + 2);
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
        DABS_T3(12);
        have = true;
#ifdef DABS_TIMING
        tD = clock64();
        if (t == 0) { ts_s[tbk][1] += tC - tB; ts_s[tbk][2] += tD - tC; }
#endif
        par_row ^= 1u;
        glb = min(glb - (int64_t)rmax_si, (int64_t)-sv);
    }

    // ---------------- write back state and the result packet
    {
        uint8_t* Xb = reinterpret_cast<uint8_t*>(p.X + (size_t)s * p.nwp);
        uint8_t* Bb = reinterpret_cast<uint8_t*>(p.best + (size_t)s * p.nwp);
        int32_t* dp = p.delta + (size_t)s * p.n_pad;
        const M128 bb = mxor(xb, pm_s[2][t]);
        for_chunks([&](int c, const int32_t* dc) {
            const int ch = (c << lgNT) + t;
            Xb[ch] = (uint8_t)mbyte(xb, c);
            Bb[ch] = (uint8_t)mbyte(bb, c);
            reinterpret_cast<int4*>(dp + ch * 8)[0] = make_int4(dc[0], dc[1], dc[2], dc[3]);
            reinterpret_cast<int4*>(dp + ch * 8)[1] = make_int4(dc[4], dc[5], dc[6], dc[7]);
        });
        if (t < TABU_RING) p.ring[(size_t)s * TABU_RING + t] = ring_s[(pos + t) & (TABU_RING - 1)];
        if (t == 0) {
            p.E[s] = E;
            p.ebest[s] = ebest;
            p.flips[s] = flips;
            atomicAdd(p.flip_total, (unsigned long long)flips);
        }
    }
#ifdef DABS_TIMING
    if (t == 0)
        for (int j = 0; j < 30; j++) atomicAdd(&g_tstat[0][0] + j, (unsigned long long)(&ts_s[0][0])[j]);
    if (t == 0)
        for (int j = 0; j < 10; j++) atomicAdd(&g_tstat2[j], (unsigned long long)ts2_s[j]);
    if (t == 0)
        for (int j = 0; j < 16; j++) atomicAdd(&g_tstat3[j], ts3_s[j]);
#endif
#undef DABS_T3
    __syncthreads();                 // every thread read tm_par_s at the start
    if (t == 0) tm_par_s = par_row;
}

template <int NT, bool TRACE>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 1) tm_batch_kernel(const BatchParams p)
{
    tm_cta_setup<NT>();
    const int s = p.order ? p.order[blockIdx.x] : p.slot0 + (int)blockIdx.x;
    tm_batch_body<NT, TRACE, false>(p, s, p.gen_ptr ? *p.gen_ptr : p.gen);
    tm_cta_teardown<NT>();
}

}  // namespace dabs
