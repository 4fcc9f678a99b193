// ga_pool_kernels.cuh -- W ingest, slot/pool init, GA seeding, pool merge,
// exchange packing and direct energy evaluation (SURVEY 8(a) rows a1, a2, a3,
// a8, a9).  Citations: P:n = PAPER.md line n; R-x = DESIGN.md readings.
#pragma once
#include "device_common.cuh"

namespace dabs {

// ------------------------------------------------------------------ a1 ingest
// Checks of the host upper-triangular input U (row-major n x n): lower
// triangle must be zero (flags[0]); per-row |W_kk| + sum_{j!=k} |W_jk| (int64)
// max into flags[1] (Delta must fit int32).
__global__ void check_kernel(const int16_t* __restrict__ U, int n, unsigned long long* flags)
{
    const int i = blockIdx.x;
    long long acc = 0;
    int lower_nz = 0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int16_t a = U[(size_t)i * n + j];
        if (j < i && a != 0) lower_nz = 1;
        const int16_t w = j >= i ? a : U[(size_t)j * n + i];   // coefficient of x_i x_j
        acc += w < 0 ? -(long long)w : (long long)w;
    }
    __shared__ long long red[32];
    __shared__ int lz[32];
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_down_sync(0xffffffffu, acc, o);
        lower_nz |= __shfl_down_sync(0xffffffffu, lower_nz, o);
    }
    if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = acc; lz[threadIdx.x >> 5] = lower_nz; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long tot = 0;
        int z = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) { tot += red[w]; z |= lz[w]; }
        if (z) atomicOr(&flags[0], 1ull);
        atomicMax(&flags[1], (unsigned long long)tot);
    }
}

// W[i][k] = coefficient of x_i x_k for i != k, 0 on the diagonal and in the
// padding (k >= n).  32x32 tiles through shared memory: the transposed half is
// read coalesced.  diag[k] = U_kk (Delta at X = 0), pads INT32_MAX.
__global__ void symmetrize_kernel(const int16_t* __restrict__ U, int n, int n_pad,
                                  int16_t* __restrict__ W, int32_t* __restrict__ diag)
{
    __shared__ int16_t tile[32][33];
    const int bi = blockIdx.y * 32, bk = blockIdx.x * 32;   // W tile rows bi.., cols bk..
    const int tx = threadIdx.x, ty = threadIdx.y;            // 32 x 8
    // transposed source tile U[bk.., bi..]
    for (int r = ty; r < 32; r += 8) {
        const int row = bk + r, col = bi + tx;
        tile[r][tx] = (row < n && col < n) ? U[(size_t)row * n + col] : (int16_t)0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = bi + r, k = bk + tx;
        if (i >= n) continue;
        int16_t v = 0;
        if (k < n && k != i) v = (k > i) ? U[(size_t)i * n + k] : tile[tx][r];
        W[(size_t)i * n_pad + k] = v;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0) {
        for (int k = ty * 32 + tx; k < n_pad; k += 256)
            diag[k] = k < n ? (int32_t)U[(size_t)k * n + k] : INT32_MAX;
    }
}

// CSR upper triangle -> symmetric dense rows (one CTA per row), diag, pads
__global__ void csr_scatter_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                   const int16_t* __restrict__ val, const int16_t* __restrict__ dg, int n,
                                   int n_pad, int16_t* __restrict__ W, int32_t* __restrict__ diag)
{
    const int i = blockIdx.x;
    for (int e = rp[i] + threadIdx.x; e < rp[i + 1]; e += blockDim.x) {
        const int j = col[e];
        W[(size_t)i * n_pad + j] = val[e];
        W[(size_t)j * n_pad + i] = val[e];
    }
    if (threadIdx.x == 0) diag[i] = dg[i];
    if (i == 0)
        for (int k = n + threadIdx.x; k < n_pad; k += blockDim.x) diag[k] = INT32_MAX;
}

// rmax[i] = max_{k != i} |W_ik| (one CTA per row): how far any Delta_k can
// move in one flip of bit i (batch kernel's lower bound on min Delta)
__global__ void rowmax_kernel(const int16_t* __restrict__ W, int n, int n_pad, int32_t* __restrict__ rmax)
{
    const int i = blockIdx.x;
    int m = 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) m = max(m, abs((int)W[(size_t)i * n_pad + k]));
    m = __reduce_max_sync(0xffffffffu, m);
    __shared__ int red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t = max(t, red[w]);
        rmax[i] = t;
    }
}

// ------------------------------------------------------------------ a2 init
// Slots: X = 0, E = 0, Delta = diag (pads INT32_MAX), empty tabu ring (R-14).
__global__ void init_slots_kernel(int slots, int n_pad, int nwp, const int32_t* __restrict__ diag,
                                  uint32_t* X, int32_t* delta, int64_t* E, int32_t* ring)
{
    const int s = blockIdx.x;
    for (int k = threadIdx.x; k < n_pad; k += blockDim.x) delta[(size_t)s * n_pad + k] = diag[k];
    for (int w = threadIdx.x; w < nwp; w += blockDim.x) X[(size_t)s * nwp + w] = 0u;
    if (threadIdx.x < TABU_RING) ring[(size_t)s * TABU_RING + threadIdx.x] = -1;
    if (threadIdx.x == 0) E[s] = 0;
}

struct PoolView {
    uint32_t* X;      // [cap][nwp]
    int64_t* E;       // [cap]
    uint64_t* seq;    // [cap]
    uint8_t* algo;    // [cap]
    uint8_t* genop;   // [cap]
};

struct GaConst {
    int n, nwp, cap, P, S;
    uint64_t eps_thr;   // floor(eps 2^32): 2^32 at eps = 1, so 64-bit (R-15)
    int n_gen, n_alg;
    int gens[N_GEN];
    int algs[N_ALG];
    uint64_t seed;
};

// Pools start as random vectors with +inf energy and random tags (P:601-602,
// R-19).  blockIdx.x = local pool p (p == P: the successor snapshot, global
// id nbr_gid); blockIdx.y = row.
__global__ void init_pools_kernel(GaConst g, PoolView* pools, uint32_t gid0, uint32_t nbr_gid, uint32_t gen)
{
    const int p = blockIdx.x, r = blockIdx.y;
    const uint32_t gp = (p < g.P) ? gid0 + (uint32_t)p : nbr_gid;
    PoolView pv = pools[p];
    const int full = g.n >> 5, rem = g.n & 31;
    for (int w = threadIdx.x; w < g.nwp; w += blockDim.x) {
        uint32_t v = rng4(g.seed, PUR_POOL_INIT, (uint32_t)w, gp, gen, (uint32_t)r).x;
        if (w > full || (w == full && rem == 0)) v = 0;
        else if (w == full) v &= (1u << rem) - 1u;
        pv.X[(size_t)r * g.nwp + w] = v;
    }
    if (threadIdx.x == 0) {
        const uint4 o = rng4(g.seed, PUR_POOL_TAGS, 0, gp, gen, (uint32_t)r);
        pv.genop[r] = (uint8_t)g.gens[pick_u(o.x, (uint32_t)g.n_gen)];
        pv.algo[r] = (uint8_t)g.algs[pick_u(o.y, (uint32_t)g.n_alg)];
        pv.E[r] = E_INF;
        pv.seq[r] = (uint64_t)r;
    }
}

// ------------------------------------------------------------------ a3 GA seeding
// One warp seeds one slot: adaptive choice of genop and algorithm (P:600-615,
// R-15), rank-biased parents (R-17), one of the genetic operations
// (R-20; Xrossover P:628-630, R-23) -> target D and tags.
// `ord` / `ord_succ` (may be NULL = identity) map a pool rank to its physical
// row (asynchronous schedule, R-29); `ord` lives in shared memory, `ord_succ`
// in global memory unless `succ_ord_shared`.  Pool reads go to L2 (ld.cg)
// because other SMs may have written the pools during the same kernel.
__device__ __forceinline__ void ga_seed_warp(const GaConst& g, const PoolView& pool, const int32_t* ord,
                                             const PoolView& succ, const int32_t* ord_succ, bool succ_ord_shared,
                                             int p, uint32_t gs, uint32_t gen, uint32_t* __restrict__ Dout,
                                             uint8_t* palgo_s, uint8_t* pgenop_s,
                                             unsigned long long* __restrict__ dispatch, int lane)
{
    auto row = [&](const int32_t* o, uint32_t r) { return o ? (uint32_t)o[r] : r; };
    auto row_succ = [&](uint32_t r) {
        return ord_succ ? (uint32_t)(succ_ord_shared ? ord_succ[r] : __ldcg(ord_succ + r)) : r;
    };
    const uint4 a = rng4(g.seed, PUR_GA_CHOICE, 0, gs, gen, 0);
    const int genop = ((uint64_t)a.x < g.eps_thr) ? g.gens[pick_u(a.y, (uint32_t)g.n_gen)]
                                        : (int)__ldcg(pool.genop + row(ord, pick_u(a.y, (uint32_t)g.cap)));
    const int algo = ((uint64_t)a.z < g.eps_thr) ? g.algs[pick_u(a.w, (uint32_t)g.n_alg)]
                                       : (int)__ldcg(pool.algo + row(ord, pick_u(a.w, (uint32_t)g.cap)));
    const uint4 b = rng4(g.seed, PUR_GA_PARENT, 0, gs, gen, 0);
    const uint32_t r1 = rank_pick(b.x, (uint32_t)g.cap), r2 = rank_pick(b.y, (uint32_t)g.cap);
    const uint32_t* A = pool.X + (size_t)row(ord, r1) * g.nwp;
    const uint32_t* Bv = genop == GEN_XROSSOVER ? succ.X + (size_t)row_succ(r2) * g.nwp
                                                : pool.X + (size_t)row(ord, r2) * g.nwp;
    const uint32_t* B0 = pool.X + (size_t)row(ord, 0) * g.nwp;   // the pool's best (GEN_BEST)
    const uint32_t n = (uint32_t)g.n;
    const uint32_t lo = n < 32u ? n : 32u;
    const uint32_t hi = (n / 2 > lo) ? n / 2 : lo;
    const uint32_t L = lo + pick_u(b.z, hi - lo + 1);
    const uint32_t start = pick_u(b.w, n);
    // IntervalZero segment as up to two index ranges [start, e0) and [0, e1)
    const uint32_t e0 = min(start + L, n);
    const int64_t e1 = (int64_t)start + L - n;
    for (int w = lane; w < g.nwp; w += 32) {
        const uint4 m = rng4(g.seed, PUR_GA_MASK, (uint32_t)w, gs, gen, 0);
        const uint32_t p8 = m.x & m.y & m.z;
        uint32_t v;
        switch (genop) {
        case GEN_MUTATION: v = __ldcg(A + w) ^ p8; break;
        case GEN_CROSSOVER:
        case GEN_XROSSOVER: v = (__ldcg(A + w) & m.x) | (__ldcg(Bv + w) & ~m.x); break;
        case GEN_ZERO: v = __ldcg(A + w) & ~p8; break;
        case GEN_ONE: v = __ldcg(A + w) | p8; break;
        case GEN_INTERVALZERO: {
            const int64_t base = (int64_t)w * 32;
            uint32_t clr = 0;
            int64_t lo1 = max((int64_t)start - base, (int64_t)0), hi1 = min((int64_t)e0 - base, (int64_t)32);
            if (lo1 < hi1) clr |= (uint32_t)((((uint64_t)1 << (hi1 - lo1)) - 1) << lo1);
            const int64_t hi2 = min(e1 - base, (int64_t)32);
            if (hi2 > 0) clr |= (uint32_t)(((uint64_t)1 << hi2) - 1);
            v = __ldcg(A + w) & ~clr;
            break;
        }
        case GEN_BEST: v = __ldcg(B0 + w); break;
        case GEN_MUTCROSS: v = ((__ldcg(A + w) & m.w) | (__ldcg(Bv + w) & ~m.w)) ^ p8; break;
        default: v = m.x; break;   // GEN_RANDOM
        }
        const int64_t rem = (int64_t)n - (int64_t)w * 32;   // clear bits >= n
        if (rem <= 0) v = 0;
        else if (rem < 32) v &= (1u << rem) - 1u;
        Dout[w] = v;
    }
    if (lane == 0) {
        *palgo_s = (uint8_t)algo;
        *pgenop_s = (uint8_t)genop;
        atomicAdd(&dispatch[((size_t)p * N_ALG + algo) * N_GEN + genop], 1ull);
    }
}

// One warp per slot, every slot of the generation (bulk-synchronous schedule).
// gen_ptr (CUDA-graph replays of the generation): the generation index is read
// from device memory instead of the by-value argument.
__global__ void ga_seed_kernel(GaConst g, const PoolView* __restrict__ pools, uint32_t slot_base,
                               uint32_t gen, int nslots, uint32_t* __restrict__ D,
                               uint8_t* __restrict__ palgo, uint8_t* __restrict__ pgenop,
                               unsigned long long* __restrict__ dispatch, const uint32_t* __restrict__ gen_ptr)
{
    if (gen_ptr) gen = *gen_ptr;
    const int warps = blockDim.x >> 5;
    const int s = blockIdx.x * warps + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s >= nslots) return;
    const int p = s / g.S;
    const PoolView pool = pools[p];
    const PoolView succ = pools[p + 1];      // pools[P] is the successor snapshot
    ga_seed_warp(g, pool, nullptr, succ, nullptr, false, p, slot_base + (uint32_t)s, gen, D + (size_t)s * g.nwp,
                 palgo + s, pgenop + s, dispatch, lane);
}

// Launch order for the batch kernel: slots whose batches cost the most start
// first (longest-processing-time order; the results do not depend on it).
// Cost classes from measured per-algorithm flip rates: TwoNeighbor (2n-1 main
// flips), MaxMin, PositiveMin, RandomMin, CyclicMin.  One CTA, stable.
__global__ void order_kernel(const uint8_t* __restrict__ palgo, int nslots, int32_t* __restrict__ order)
{
    __shared__ int cnt[5];
    __shared__ int base[5];
    const int cls_of[5] = {1, 4, 3, 2, 0};   // by algorithm id: MaxMin, CyclicMin, RandomMin, PositiveMin, Two
    if (threadIdx.x < 5) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int s = threadIdx.x; s < nslots; s += blockDim.x) atomicAdd(&cnt[cls_of[palgo[s]]], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int a = 0;
        for (int c = 0; c < 5; c++) { base[c] = a; a += cnt[c]; }
    }
    __syncthreads();
    // stable scatter: one warp per class walks the slots in order
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w < 5) {
        int pos = base[w];
        for (int s0 = 0; s0 < nslots; s0 += 32) {
            const int s = s0 + lane;
            const bool m = s < nslots && cls_of[palgo[s]] == w;
            const unsigned bal = __ballot_sync(0xffffffffu, m);
            if (m) order[pos + __popc(bal & ((1u << lane) - 1u))] = s;
            pos += __popc(bal);
        }
    }
}

// ------------------------------------------------------------------ a8 pool merge
// One CTA (1024 threads) per local pool (R-18).  The new pool
// is the first cap entries of the (E, seq)-sorted old ++ new list with
// (E, X)-duplicates of earlier finite entries dropped.  Only results with
// E < E(worst old) can enter (they sort after every old entry otherwise).
struct MergeArgs {
    PoolView* pools;
    const uint32_t* best;     // [slots][nwp]
    const int64_t* ebest;     // [slots]
    const uint8_t* palgo;
    const uint8_t* pgenop;
    int32_t* order;           // scratch [P][S]
    int32_t* acc;             // scratch [P][cap]
    uint32_t* sX;             // scratch [P][cap][nwp]
    int64_t* sE;              // scratch [P][cap]
    uint64_t* sSeq;
    uint8_t* sAlgo;
    uint8_t* sGenop;
    unsigned long long* inserted;
    int32_t* mcount;          // [P] qualifying results per pool (merge_rank_kernel)
    uint64_t* hq;             // scratch [P][S]: hashes of the qualifiers' vectors
    uint64_t* hold;           // scratch [P][cap]: hashes of the old entries' vectors
    uint8_t* dupf;            // scratch [P][S]: duplicate flags
    uint32_t slot_base;
    uint32_t gen;
    const uint32_t* gen_ptr;  // graph replays: the generation index in device memory (else gen)
    int S, cap, nwp;
};

// Rank the results that can enter pool p (E < E(worst entry)) by (E, slot):
// order[rank] = slot.  One WARP per result (blockIdx.y = pool), its lanes
// striding over the pool's S result energies: O(S^2) compares spread over
// S warps of the whole GPU (one thread per result left most SMs idle).
__global__ void __launch_bounds__(256) merge_rank_kernel(MergeArgs a)
{
    const int p = blockIdx.y;
    const int S = a.S;
    const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= S) return;
    const int64_t* eb = a.ebest + (size_t)p * S;
    const int64_t Eworst = a.pools[p].E[a.cap - 1];
    const int64_t e = eb[j];
    if (!(e < Eworst)) return;                       // uniform per warp
    int rank = 0;
    for (int i = lane; i < S; i += 32) {
        const int64_t e2 = eb[i];
        rank += (e2 < Eworst) && (e2 < e || (e2 == e && i < j));
    }
    rank = __reduce_add_sync(0xffffffffu, (unsigned)rank);
    if (lane == 0) {
        a.order[(size_t)p * S + rank] = j;
        atomicAdd(&a.mcount[p], 1);
    }
}

__device__ __forceinline__ bool vec_equal_warp(const uint32_t* a, const uint32_t* b, int nwp, int lane)
{
    bool eq = true;
    for (int w = lane; w < nwp; w += 32) eq &= (a[w] == b[w]);
    return __all_sync(0xffffffffu, eq);
}

__device__ __forceinline__ uint64_t vec_hash_warp(const uint32_t* x, int nwp, int lane)
{
    uint64_t h = 0;
    for (int w = lane; w < nwp; w += 32) {
        uint64_t z = ((uint64_t)x[w] << 32 | (uint32_t)w) + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        h ^= z ^ (z >> 31);
    }
    const uint32_t lo = __reduce_xor_sync(0xffffffffu, (uint32_t)h);
    const uint32_t hi = __reduce_xor_sync(0xffffffffu, (uint32_t)(h >> 32));
    return (uint64_t)hi << 32 | lo;
}

// (1) hashes of the qualifiers' vectors (hq, in rank order) and of the old
// entries (hold), one warp per vector, the whole grid (blockIdx.y = pool)
__global__ void __launch_bounds__(256) merge_hash_kernel(MergeArgs a)
{
    const int p = blockIdx.y;
    const int S = a.S, cap = a.cap, nwp = a.nwp;
    const int o = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    const int M = a.mcount[p];
    if (o >= M + cap) return;
    const uint32_t* xj = o < M ? a.best + ((size_t)p * S + a.order[(size_t)p * S + o]) * nwp
                               : a.pools[p].X + (size_t)(o - M) * nwp;
    const uint64_t h = vec_hash_warp(xj, nwp, lane);
    if (lane == 0) {
        if (o < M) a.hq[(size_t)p * S + o] = h;
        else a.hold[(size_t)p * cap + (o - M)] = h;
    }
}

// (2) duplicate flags, one warp per qualifier, the whole grid (R-18): a
// qualifier is dropped iff its (E, X) equals an old entry or an EARLIER
// qualifier (equality is transitive, so "an earlier accepted result" reduces
// to "an earlier qualifier").  Candidates by ballot on equal (E, hash); full
// vectors compared only for those.
__global__ void __launch_bounds__(256) merge_dup_kernel(MergeArgs a)
{
    const int p = blockIdx.y;
    const int S = a.S, cap = a.cap, nwp = a.nwp;
    const int o = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    const int M = a.mcount[p];
    if (o >= M) return;
    const PoolView pool = a.pools[p];
    const int64_t* eb = a.ebest + (size_t)p * S;
    const int32_t* order = a.order + (size_t)p * S;
    const uint64_t* hq = a.hq + (size_t)p * S;
    const uint64_t* hold = a.hold + (size_t)p * cap;
    const int j = order[o];
    const int64_t e = eb[j];
    const uint64_t h = hq[o];
    const uint32_t* xj = a.best + ((size_t)p * S + j) * nwp;
    bool dup = false;
    for (int r0 = 0; r0 < cap && !dup; r0 += 32) {    // old entries
        const int r = r0 + lane;
        unsigned mk = __ballot_sync(0xffffffffu, r < cap && pool.E[r] == e && hold[r] == h);
        while (mk && !dup) {
            const int rr = r0 + __ffs(mk) - 1;
            mk &= mk - 1;
            if (vec_equal_warp(pool.X + (size_t)rr * nwp, xj, nwp, lane)) dup = true;
        }
    }
    // earlier qualifiers with the same energy are contiguous just before o
    for (int q0 = o - 1; q0 >= 0 && !dup; q0 -= 32) {
        const int q = q0 - lane;
        const bool sameE = q >= 0 && eb[order[q]] == e;
        const unsigned stopm = __ballot_sync(0xffffffffu, q >= 0 && !sameE);
        unsigned mk = __ballot_sync(0xffffffffu, sameE && hq[q] == h);
        if (stopm) mk &= (__ffs(stopm) == 1) ? 0u : ((1u << (__ffs(stopm) - 1)) - 1u);   // lanes before the first E change
        while (mk && !dup) {
            const int qq = q0 - (__ffs(mk) - 1);
            mk &= mk - 1;
            if (vec_equal_warp(a.best + ((size_t)p * S + order[qq]) * nwp, xj, nwp, lane)) dup = true;
        }
        if (stopm) break;
    }
    if (lane == 0) a.dupf[(size_t)p * S + o] = dup ? 1 : 0;
}

__global__ void __launch_bounds__(1024) pool_merge_kernel(MergeArgs a)
{
    const int p = blockIdx.x;
    const int S = a.S, cap = a.cap, nwp = a.nwp;
    const PoolView pool = a.pools[p];
    const int64_t* eb = a.ebest + (size_t)p * S;
    int32_t* order = a.order + (size_t)p * S;
    int32_t* acc = a.acc + (size_t)p * cap;
    __shared__ int s_nacc;
    if (threadIdx.x == 0) s_nacc = 0;
    __syncthreads();
    // qualifying results, ranked by (E, slot) into order[] by merge_rank_kernel,
    // duplicate flags from merge_hash_kernel + merge_dup_kernel
    const int M = a.mcount[p];
    const int lane = threadIdx.x & 31;
    const uint8_t* dupf = a.dupf + (size_t)p * S;
    // (3) the first cap non-duplicates in order (warp 0)
    if (threadIdx.x < 32) {
        int nacc = 0;
        for (int o0 = 0; o0 < M && nacc < cap; o0 += 32) {
            const int o = o0 + lane;
            const bool keep = o < M && !dupf[o];
            const unsigned mk = __ballot_sync(0xffffffffu, keep);
            const int pos = nacc + __popc(mk & ((1u << lane) - 1u));
            if (keep && pos < cap) acc[pos] = order[o];
            nacc += __popc(mk);
        }
        if (lane == 0) s_nacc = nacc < cap ? nacc : cap;
    }
    __syncthreads();
    const int nacc = s_nacc;
    // merge old (sorted) with accepted (sorted; all seq larger) -> first cap
    __shared__ int src[1024];   // >= 0: old row; < 0: -(q+1) accepted index
    if (threadIdx.x == 0) {
        int io = 0, in = 0;
        for (int r = 0; r < cap; r++) {
            const bool take_new = in < nacc && (io >= cap || eb[acc[in]] < pool.E[io]);
            src[r] = take_new ? -(in + 1) : io;
            if (take_new) in++; else io++;
        }
    }
    __syncthreads();
    uint32_t* sX = a.sX + (size_t)p * cap * nwp;
    int64_t* sE = a.sE + (size_t)p * cap;
    uint64_t* sSeq = a.sSeq + (size_t)p * cap;
    uint8_t* sA = a.sAlgo + (size_t)p * cap;
    uint8_t* sG = a.sGenop + (size_t)p * cap;
    for (int r = threadIdx.x >> 5; r < cap; r += blockDim.x >> 5) {
        const int sr = src[r];
        const uint32_t* from;
        if (sr >= 0) {
            from = pool.X + (size_t)sr * nwp;
        } else {
            const int j = acc[-sr - 1];
            from = a.best + ((size_t)p * S + j) * nwp;
        }
        for (int w = threadIdx.x & 31; w < nwp; w += 32) sX[(size_t)r * nwp + w] = from[w];
        if ((threadIdx.x & 31) == 0) {
            if (sr >= 0) {
                sE[r] = pool.E[sr]; sSeq[r] = pool.seq[sr]; sA[r] = pool.algo[sr]; sG[r] = pool.genop[sr];
            } else {
                const int j = acc[-sr - 1];
                const int ls = p * S + j;
                sE[r] = eb[j];
                const uint32_t gen = a.gen_ptr ? *a.gen_ptr : a.gen;
                sSeq[r] = ((uint64_t)(gen + 1) << 32) | (uint64_t)(a.slot_base + (uint32_t)ls);
                sA[r] = a.palgo[ls];
                sG[r] = a.pgenop[ls];
                atomicAdd(&a.inserted[((size_t)p * N_ALG + sA[r]) * N_GEN + sG[r]], 1ull);
            }
        }
    }
    __syncthreads();
    for (size_t w = threadIdx.x; w < (size_t)cap * nwp; w += blockDim.x) pool.X[w] = sX[w];
    for (int r = threadIdx.x; r < cap; r += blockDim.x) {
        pool.E[r] = sE[r]; pool.seq[r] = sSeq[r]; pool.algo[r] = sA[r]; pool.genop[r] = sG[r];
    }
}

// ------------------------------------------------------------------ a9 exchange payload
// Payload of one rank (all 8-byte aligned):
//   X[cap][nwp] u32 | E[cap] i64 | seq[cap] u64 | algo[cap] u8 | genop[cap] u8 | pad |
//   summary: bestE i64, bestSeq u64, bestPool i32, algo i32, genop i32, pad i32, flips u64 |
//   bestX[nwp] u32
struct PayloadLayout {
    size_t oX, oE, oSeq, oAlgo, oGenop, oSum, oBestX, bytes;
};

struct Summary {
    int64_t bestE;
    uint64_t bestSeq;
    int32_t bestPool;     // global pool id
    int32_t algo, genop, pad;
    unsigned long long flips;
};

__global__ void pack_payload_kernel(const PoolView* __restrict__ pools, int P, int cap, int nwp,
                                    uint32_t gpool0, const unsigned long long* __restrict__ flip_total,
                                    uint8_t* __restrict__ out, PayloadLayout L)
{
    const PoolView p0 = pools[0];
    uint32_t* X = reinterpret_cast<uint32_t*>(out + L.oX);
    for (size_t w = threadIdx.x; w < (size_t)cap * nwp; w += blockDim.x) X[w] = p0.X[w];
    int64_t* E = reinterpret_cast<int64_t*>(out + L.oE);
    uint64_t* sq = reinterpret_cast<uint64_t*>(out + L.oSeq);
    for (int r = threadIdx.x; r < cap; r += blockDim.x) {
        E[r] = p0.E[r];
        sq[r] = p0.seq[r];
        out[L.oAlgo + r] = p0.algo[r];
        out[L.oGenop + r] = p0.genop[r];
    }
    // best over local pools: lowest (E, pool)
    int bp = 0;
    for (int q = 1; q < P; q++)
        if (pools[q].E[0] < pools[bp].E[0]) bp = q;
    const PoolView b = pools[bp];
    if (threadIdx.x == 0) {
        Summary* sm = reinterpret_cast<Summary*>(out + L.oSum);
        sm->bestE = b.E[0];
        sm->bestSeq = b.seq[0];
        sm->bestPool = (int32_t)(gpool0 + (uint32_t)bp);
        sm->algo = b.algo[0];
        sm->genop = b.genop[0];
        sm->pad = 0;
        sm->flips = *flip_total;
    }
    uint32_t* BX = reinterpret_cast<uint32_t*>(out + L.oBestX);
    for (int w = threadIdx.x; w < nwp; w += blockDim.x) BX[w] = b.X[w];
}

// The successor's first pool becomes the Xrossover snapshot (R-23).
__global__ void import_snapshot_kernel(const uint8_t* __restrict__ in, PoolView nbr, int cap, int nwp,
                                       PayloadLayout L)
{
    const uint32_t* X = reinterpret_cast<const uint32_t*>(in + L.oX);
    for (size_t w = threadIdx.x + (size_t)blockIdx.x * blockDim.x; w < (size_t)cap * nwp;
         w += (size_t)blockDim.x * gridDim.x)
        nbr.X[w] = X[w];
    if (blockIdx.x == 0) {
        const int64_t* E = reinterpret_cast<const int64_t*>(in + L.oE);
        const uint64_t* sq = reinterpret_cast<const uint64_t*>(in + L.oSeq);
        for (int r = threadIdx.x; r < cap; r += blockDim.x) {
            nbr.E[r] = E[r];
            nbr.seq[r] = sq[r];
            nbr.algo[r] = in[L.oAlgo + r];
            nbr.genop[r] = in[L.oGenop + r];
        }
    }
}

// ------------------------------------------------------------------ Eq.(2) direct
// E(X) = sum_k d_k x_k + sum_{i<k} W_ik x_i x_k, W symmetric with zero diagonal.
__global__ void energy_kernel(const int16_t* __restrict__ W, const int32_t* __restrict__ diag, int n,
                              int n_pad, const uint8_t* __restrict__ x, long long* out)
{
    const int i = blockIdx.x;
    if (!x[i]) return;
    long long acc = 0;
    for (int k = i + 1 + threadIdx.x; k < n; k += blockDim.x)
        if (x[k]) acc += W[(size_t)i * n_pad + k];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    __shared__ long long red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = diag[i];
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
        atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)t);
    }
}

}  // namespace dabs
