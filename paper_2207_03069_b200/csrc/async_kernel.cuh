// async_kernel.cuh -- the asynchronous packet schedule (SURVEY 8(f) f1,
// DESIGN.md R-29): one persistent CTA per slot runs batch after batch with no
// generation barrier, the paper's packet flow moved onto
// the device.  After each batch the CTA takes the rank's pool lock, merges its
// result into its pool (R-18 with one newcomer), updates the run best, appends
// (slot | seeded<<31) to the event log, and -- unless the run is stopping --
// seeds its next packet from the pools as they are now (GA).  The
// log makes the run replayable by the CPU oracle (orc_world_async_replay).
// Citations: P:n = PAPER.md line n; R-x = DESIGN.md readings.
#pragma once
#include "batch_kernel.cuh"
#include "ga_pool_kernels.cuh"

namespace dabs {

struct AsyncArgs {
    BatchParams bp;
    GaConst g;
    const PoolView* pools;            // [P] local pools (rows in physical order)
    int32_t* ord;                     // [P][cap] pool rank -> physical row
    uint64_t* hash;                   // [P][cap] per physical row: hash of X (duplicate pre-check)
    uint32_t* D;                      // [slots][nwp] packets (written here, read by the batch)
    uint8_t *palgo, *pgenop;          // [slots]
    unsigned long long *dispatch, *inserted;
    uint32_t* ticket;                 // [P*32] per-pool ticket locks: next ticket (one 128-B line per pool)
    uint32_t* serving;                // [P*32] ticket being served
    uint32_t* evcount;                // events so far (the event index, taken under the locks)
    int32_t* best_lock;               // guards the run best
    uint32_t* log;                    // [log_cap]; a longer run keeps going, its log is truncated
    uint32_t log_cap;
    int slots;
    unsigned long long* flips_cum;    // flips of merged batches
    unsigned long long budget;
    int64_t target;                   // INT64_MIN = none
    unsigned long long time_limit_ns; // 0 = none
    unsigned long long* t0;           // globaltimer at the start of the run
    int32_t* stop;                    // sticky stop flag
    int64_t* bestE;                   // run best
    uint32_t* bestX;                  // [nwp]
    int32_t* brec;                    // algo, genop, event, slot
    unsigned long long* best_t;       // globaltimer of the last improvement
    unsigned long long* lock_ns;      // [10] summed lock wait/hold times, phase and CTA-time breakdown (device clock)
    int profile;                      // 1: also accumulate the phase / CTA-time breakdown (DABS_ASYNC_PHASES)
};

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}

// 64-bit hash of a bit vector (warp-cooperative): xor of splitmix64(word, index)
__device__ __forceinline__ uint64_t xhash_warp(const uint32_t* X, int nwp, int lane)
{
    uint64_t h = 0;
    for (int w = lane; w < nwp; w += 32) {
        uint64_t z = ((uint64_t)__ldcg(X + w) << 32 | (uint32_t)w) + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        h ^= z ^ (z >> 31);
    }
    const uint32_t lo = __reduce_xor_sync(0xffffffffu, (uint32_t)h);
    const uint32_t hi = __reduce_xor_sync(0xffffffffu, (uint32_t)(h >> 32));
    return (uint64_t)hi << 32 | lo;
}

__global__ void async_init_kernel(int32_t* ord, uint64_t* hash, int P, int cap, unsigned long long* t0)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P * cap; i += gridDim.x * blockDim.x) {
        ord[i] = i % cap;
        hash[i] = 0;   // sentinel rows (E = +inf) are never compared
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *t0 = globaltimer();
}

// bytes of dynamic shared memory the commit needs (ord_s, ord_n, eqf)
inline size_t async_commit_smem(int cap) { return (size_t)cap * 9; }

// Merge + log + seed for slot s after its batch k (warp 0 of the CTA), under
// its pool's ticket lock (an Xrossover partner in another pool is read later,
// by the XREAD event, under that pool's lock).  The lock is held for three
// dependent rounds of L2 loads: (A) pool order, run best, stop flag; (B)
// energies and hashes of the pool entries -> rank of the newcomer; (C) the
// chosen tags and every candidate parent row at once.  Everything that does not read the pools (own result, its hash, the
// Philox draws of packet k+1) happens before the lock.  The GA below is the
// same arithmetic as ga_seed_warp (R-15, R-17, R-20, R-29).
// Returns whether a next packet was seeded (CTA-uniform).
template <int CL>
__device__ __forceinline__ bool async_commit(const AsyncArgs& a, int s, uint32_t k)
{
    // commit scratch in the dynamic shared memory of the batch's row buffer
    // (idle between batches; the launch sizes it to fit, async_commit_smem):
    // static arrays here would shrink the L1 the batches use
    extern __shared__ __align__(128) uint8_t dyn_smem[];
    int32_t* ord_s = reinterpret_cast<int32_t*>(dyn_smem);   // pool order before the merge
    int32_t* ord_n = ord_s + a.g.cap;                         // after
    uint8_t* eqf = reinterpret_cast<uint8_t*>(ord_n + a.g.cap);   // round B: 1 = same E, 3 = same E and hash
    __shared__ int sh_seeded;
    const int t = threadIdx.x, lane = t & 31;
    const BatchParams& bp = a.bp;
    const GaConst& g = a.g;
    const int nwp = bp.nwp, cap = g.cap;
    // cluster tier: the cluster's rank-0 CTA commits; the other waits
    if (t < 32 && (CL == 1 || cluster_rank() == 0)) {
        const int p = s / g.S;
        const int pn = (p + 1) % g.P;   // live ring successor (R-29)
        const PoolView pool = a.pools[p];
        const PoolView succ = a.pools[pn];
        int32_t* ord = a.ord + (size_t)p * cap;
        const int64_t Er = bp.ebest[s];
        const unsigned long long fls = (unsigned long long)bp.flips[s];
        const uint32_t* Xr = bp.best + (size_t)s * nwp;
        const uint8_t alg = a.palgo[s], gop = a.pgenop[s];
        const uint32_t gs = bp.slot_base + (uint32_t)s;
        const uint64_t hr = xhash_warp(Xr, nwp, lane);
        uint64_t* hash = a.hash + (size_t)p * cap;
        // packet k+1 draws (R-15, R-17, R-20)
        const uint32_t gen1 = k + 1;
        const uint4 ga = rng4(g.seed, PUR_GA_CHOICE, 0, gs, gen1, 0);
        const uint4 gb = rng4(g.seed, PUR_GA_PARENT, 0, gs, gen1, 0);
        const bool g_rand = (uint64_t)ga.x < g.eps_thr, a_rand = (uint64_t)ga.z < g.eps_thr;
        const uint32_t pg = pick_u(ga.y, (uint32_t)cap), pa = pick_u(ga.w, (uint32_t)cap);
        const uint32_t r1 = rank_pick(gb.x, (uint32_t)cap), r2 = rank_pick(gb.y, (uint32_t)cap);
        const uint32_t n = (uint32_t)g.n;
        const uint32_t lo = n < 32u ? n : 32u;
        const uint32_t hi = (n / 2 > lo) ? n / 2 : lo;
        const uint32_t L = lo + pick_u(gb.z, hi - lo + 1);
        const uint32_t start = pick_u(gb.w, n);
        const uint32_t e0 = min(start + L, n);
        const int64_t e1 = (int64_t)start + L - n;
        // GA mask words of this lane's first two D words, before the lock
        uint4 mpre[2];
#pragma unroll
        for (int j = 0; j < 2; j++)
            mpre[j] = lane + 32 * j < nwp ? rng4(g.seed, PUR_GA_MASK, (uint32_t)(lane + 32 * j), gs, gen1, 0)
                                         : make_uint4(0, 0, 0, 0);

        // Per-pool ticket locks.  Every event holds exactly one pool's lock and
        // takes its event index under it.  Two events that touch the same pool
        // are then ordered the same way by that pool's lock and by their
        // indices, so replaying the log in index order reproduces every pool's
        // history.  An Xrossover packet whose partner is another pool is
        // finished by a second event (XREAD) under the partner's lock after
        // this one is released (R-29): no lock is ever held while waiting.
        auto lock = [&](int q) {
            const uint32_t tk = atomicAdd(a.ticket + 32 * q, 1u);
            // poll with relaxed loads (an acquire load would invalidate the SM's L1
            // on every poll), then one acquire fence
            for (;;) {
                uint32_t sv;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(sv) : "l"(a.serving + 32 * q) : "memory");
                if (sv == tk) break;
                __nanosleep(min(256u * (tk - sv), 20000u));
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            return tk;
        };
        auto unlock = [&](int q, uint32_t tk) {
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.serving + 32 * q), "r"(tk + 1) : "memory");
        };
        uint32_t tk_own = 0;
        const unsigned long long t_req = globaltimer();
        unsigned long long t_acq = 0, t_B = 0, t_D = 0;
        int64_t bE = 0;
        int32_t bev = 0;
        int stop0 = 0, pos = 0, genop = 0;
        bool ins = false;
        {
            if (lane == 0) tk_own = lock(p);
            __syncwarp();
            t_acq = globaltimer();
            // round A
            for (int r0 = lane; r0 < cap; r0 += 128) {   // four loads in flight per lane
                int32_t o[4];
#pragma unroll
                for (int j = 0; j < 4; j++) o[j] = r0 + 32 * j < cap ? __ldcg(ord + r0 + 32 * j) : 0;
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (r0 + 32 * j < cap) ord_s[r0 + 32 * j] = o[j];
            }
            // the run best and the stop flag change under other locks: one lane
            // reads them and broadcasts, so every branch on them is warp-uniform
            if (lane == 0) {
                bE = __ldcg(a.bestE);
                bev = __ldcg(a.brec + 2);
                stop0 = __ldcg(a.stop);
            }
            bE = __shfl_sync(0xffffffffu, bE, 0);
            bev = __shfl_sync(0xffffffffu, bev, 0);
            stop0 = __shfl_sync(0xffffffffu, stop0, 0);
            __syncwarp();
            t_B = globaltimer();
            // round B: rank of the newcomer = entries with E <= Er (older seq first, R-18);
            // (E, X) duplicates: only entries with E == Er and the same hash are compared
            pos = 0;
            bool cand = false;
            for (int r0 = lane; r0 < cap; r0 += 128) {
                int64_t Eo[4];
                uint64_t ho[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const bool in = r0 + 32 * j < cap;
                    const int32_t o = in ? ord_s[r0 + 32 * j] : 0;
                    Eo[j] = in ? __ldcg(pool.E + o) : E_INF;
                    ho[j] = in ? __ldcg(hash + o) : 0;
                }
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const bool in = r0 + 32 * j < cap;
                    pos += (in && Eo[j] <= Er) ? 1 : 0;
                    const bool sameE = in && Eo[j] == Er, c = sameE && ho[j] == hr;
                    cand |= c;
                    if (in) eqf[r0 + 32 * j] = (uint8_t)((sameE ? 1 : 0) | (c ? 2 : 0));
                }
            }
            pos = (int)warp_add((unsigned)pos);
            ins = pos < cap && Er != E_INF;
            t_D = globaltimer();
            if (ins && __any_sync(0xffffffffu, cand)) {
                __syncwarp();
                for (int r = pos - 1; ins && r >= 0 && (eqf[r] & 1); r--) {
                    if (!(eqf[r] & 2)) continue;
                    const int32_t o = ord_s[r];
                    bool eq = true;
#pragma unroll 4
                    for (int w = lane; w < nwp; w += 32) eq &= (__ldcg(pool.X + (size_t)o * nwp + w) == __ldcg(Xr + w));
                    if (__all_sync(0xffffffffu, eq)) ins = false;
                }
            }
            // the next packet's genetic operation (R-15): the tag at rank pg of the
            // pool as it is after this merge
            if (g_rand) {
                genop = g.gens[pick_u(ga.y, (uint32_t)g.n_gen)];
            } else if (ins && pg == (uint32_t)pos) {
                genop = gop;
            } else {
                const uint32_t q = (ins && pg > (uint32_t)pos) ? pg - 1 : pg;
                genop = (int)__ldcg(pool.genop + ord_s[q]);
            }
        }
        const bool xpend = genop == GEN_XROSSOVER && pn != p;   // finished by an XREAD event
        uint32_t e = 0;
        unsigned long long fl = 0;
        if (lane == 0) {
            e = atomicAdd(a.evcount, 1u);
            fl = atomicAdd(a.flips_cum, fls) + fls;
        }
        e = __shfl_sync(0xffffffffu, e, 0);
        fl = __shfl_sync(0xffffffffu, fl, 0);
        unsigned long long t0 = a.time_limit_ns ? __ldcg(a.t0) : 0ull;
        t0 = __shfl_sync(0xffffffffu, t0, 0);
        const int32_t victim = ord_s[cap - 1];
        if (ins) {
            for (int w = lane; w < nwp; w += 32) __stcg(pool.X + (size_t)victim * nwp + w, __ldcg(Xr + w));
            if (lane == 0) {
                __stcg(pool.E + victim, Er);
                __stcg(hash + victim, hr);
                __stcg(pool.seq + victim, ((uint64_t)(e + 1) << 32) | (uint64_t)gs);
                pool.algo[victim] = alg;
                pool.genop[victim] = gop;
                atomicAdd(&a.inserted[((size_t)p * N_ALG + alg) * N_GEN + gop], 1ull);
            }
            for (int r = lane; r < cap; r += 32) {
                const int32_t o = r < pos ? ord_s[r] : (r == pos ? victim : ord_s[r - 1]);
                ord_n[r] = o;
                __stcg(ord + r, o);
            }
        } else {
            for (int r = lane; r < cap; r += 32) ord_n[r] = ord_s[r];
        }
        __syncwarp();
        // run best (strict improvement), flips, stop rule
        const unsigned long long now = __shfl_sync(0xffffffffu, globaltimer(), 0);   // one clock read: uniform stop
        // run best = the lexicographic minimum of (E, event) over all events, i.e.
        // the first event (in log order) that reached the best energy
        // (racy pre-check: an equal energy already recorded by an earlier event needs no lock)
        if (Er != E_INF && (Er < bE || (Er == bE && (bev < 0 || (uint32_t)bev > e)))) {
            int upd = 0;
            if (lane == 0) {
                while (atomicCAS(a.best_lock, 0, 1) != 0) __nanosleep(64);
                __threadfence();
                const int64_t cE = __ldcg(a.bestE);
                const int32_t ce = __ldcg(a.brec + 2);
                upd = (Er < cE || (Er == cE && (ce < 0 || (uint32_t)ce > e))) ? 1 : 0;
            }
            upd = __shfl_sync(0xffffffffu, upd, 0);
            if (upd) {
                for (int w = lane; w < nwp; w += 32) __stcg(a.bestX + w, __ldcg(Xr + w));
                if (lane == 0) {
                    __stcg(a.bestE, Er);
                    __stcg(a.brec + 0, (int32_t)alg);
                    __stcg(a.brec + 1, (int32_t)gop);
                    __stcg(a.brec + 2, (int32_t)e);
                    __stcg(a.brec + 3, (int32_t)gs);
                    __stcg(a.best_t, now);
                }
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                atomicExch(a.best_lock, 0);
            }
        }
        const int64_t bE2 = Er < bE ? Er : bE;
        const bool stop = stop0 != 0 || fl >= a.budget || (a.target != INT64_MIN && bE2 <= a.target) ||
                          (a.time_limit_ns && now - t0 >= a.time_limit_ns);
        const bool seeded = !stop;
        if (lane == 0) {
            if (stop) __stcg(a.stop, 1);
            if (e < a.log_cap) __stcg(a.log + e, (uint32_t)s | (seeded ? 0x80000000u : 0u));   // full: truncated
        }
        const unsigned long long t_G = globaltimer();
        if (seeded) {
            // round C: tags and all candidate parent rows.  The newcomer's row and
            // tags are this slot's own (the pool copies were just written).
            const bool newA = ins && r1 == (uint32_t)pos, newB = ins && r2 == (uint32_t)pos, new0 = ins && pos == 0;
            const uint32_t* A = newA ? Xr : pool.X + (size_t)ord_n[r1] * nwp;
            const uint32_t* Bo = newB ? Xr : pool.X + (size_t)ord_n[r2] * nwp;
            const uint32_t* Bs = Bo;   // Xrossover: own pool (P = 1); across pools the XREAD fills it
            const uint32_t* B0 = new0 ? Xr : pool.X + (size_t)ord_n[0] * nwp;
            const int algo = a_rand ? g.algs[pick_u(ga.w, (uint32_t)g.n_alg)]
                                    : (ins && pa == (uint32_t)pos ? (int)alg : (int)__ldcg(pool.algo + ord_n[pa]));
            uint32_t* Dout = a.D + (size_t)s * nwp;
            auto emit = [&](int w, const uint4 m) {
                const uint32_t va = __ldcg(A + w), vbo = __ldcg(Bo + w), vbs = __ldcg(Bs + w), v0 = __ldcg(B0 + w);
                const uint32_t vb = genop == GEN_XROSSOVER ? (xpend ? 0u : vbs) : vbo;
                const uint32_t p8 = m.x & m.y & m.z;
                uint32_t v;
                switch (genop) {
                case GEN_MUTATION: v = va ^ p8; break;
                case GEN_CROSSOVER:
                case GEN_XROSSOVER: v = (va & m.x) | (vb & ~m.x); break;
                case GEN_ZERO: v = va & ~p8; break;
                case GEN_ONE: v = va | p8; break;
                case GEN_INTERVALZERO: {
                    const int64_t base = (int64_t)w * 32;
                    uint32_t clr = 0;
                    int64_t lo1 = max((int64_t)start - base, (int64_t)0), hi1 = min((int64_t)e0 - base, (int64_t)32);
                    if (lo1 < hi1) clr |= (uint32_t)((((uint64_t)1 << (hi1 - lo1)) - 1) << lo1);
                    const int64_t hi2 = min(e1 - base, (int64_t)32);
                    if (hi2 > 0) clr |= (uint32_t)(((uint64_t)1 << hi2) - 1);
                    v = va & ~clr;
                    break;
                }
                case GEN_BEST: v = v0; break;
                case GEN_MUTCROSS: v = ((va & m.w) | (vb & ~m.w)) ^ p8; break;
                default: v = m.x; break;   // GEN_RANDOM
                }
                const int64_t rem = (int64_t)n - (int64_t)w * 32;   // clear bits >= n
                if (rem <= 0) v = 0;
                else if (rem < 32) v &= (1u << rem) - 1u;
                Dout[w] = v;
            };
            if (lane < nwp) emit(lane, mpre[0]);
            if (lane + 32 < nwp) emit(lane + 32, mpre[1]);
            for (int w = lane + 64; w < nwp; w += 32) emit(w, rng4(g.seed, PUR_GA_MASK, (uint32_t)w, gs, gen1, 0));
            if (lane == 0) {
                a.palgo[s] = (uint8_t)algo;
                a.pgenop[s] = (uint8_t)genop;
                atomicAdd(&a.dispatch[((size_t)p * N_ALG + algo) * N_GEN + genop], 1ull);
            }
        }
        __syncwarp();   // orders every lane's pool writes before lane 0's release
        const unsigned long long t_R = globaltimer();
        if (lane == 0) {
            unlock(p, tk_own);
            sh_seeded = seeded ? 1 : 0;
            const unsigned long long t_rel = globaltimer();
            atomicAdd(a.lock_ns, t_acq - t_req);
            if (a.profile) {
                atomicAdd(a.lock_ns + 2, t_B - t_acq);
                atomicAdd(a.lock_ns + 3, t_D - t_B);
                atomicAdd(a.lock_ns + 4, t_G - t_D);
                atomicAdd(a.lock_ns + 5, t_R - t_G);
                atomicAdd(a.lock_ns + 6, t_rel - t_R);
            }
            atomicAdd(a.lock_ns + 1, t_rel - t_acq);
        }
        // XREAD (R-29): the partner pool's rank-r2 row fills the bits the mask
        // does not take from the own parent
        if (seeded && xpend) {
            uint32_t tk = 0, e2 = 0;
            if (lane == 0) {
                tk = lock(pn);
                e2 = atomicAdd(a.evcount, 1u);
            }
            __syncwarp();
            const int32_t o2 = __ldcg(a.ord + (size_t)pn * cap + r2);
            const uint32_t* Bx = succ.X + (size_t)o2 * nwp;
            uint32_t* Dout = a.D + (size_t)s * nwp;
            for (int w = lane; w < nwp; w += 32) {
                const uint4 m = w < 64 ? (w < 32 ? mpre[0] : mpre[1]) : rng4(g.seed, PUR_GA_MASK, (uint32_t)w, gs, gen1, 0);
                Dout[w] |= __ldcg(Bx + w) & ~m.x;   // bits >= n: zero in every pool row
            }
            __syncwarp();
            if (lane == 0) {
                if (e2 < a.log_cap) __stcg(a.log + e2, (uint32_t)s | 0x40000000u);
                unlock(pn, tk);
            }
        }
    }
    if constexpr (CL == 2) {
        // publish the decision to the peer CTA (its shared memory), then a
        // cluster barrier (release/acquire: the packet in global memory too)
        if (t == 0 && cluster_rank() == 0) {
            const uint32_t peer = mapa_peer(smem_u32(&sh_seeded), 1u);
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer), "r"((uint32_t)sh_seeded) : "memory");
        }
        cluster_sync_all();
    } else {
        __syncthreads();
    }
    return sh_seeded != 0;
}

// register budget of the batch kernel of the same tier: warp tier C <= 4 -> 16
// CTAs per SM (128 registers), C = 8 -> 12; CTA tiers unconstrained
template <int C, int NTT, int CL>
__global__ void __launch_bounds__(NTT, NTT == 32 ? 16 : 0) async_kernel(const AsyncArgs a)
{
    const int s = (int)blockIdx.x / CL;
    const unsigned long long t_start = globaltimer();
    unsigned long long t_body = 0, t_commit = 0;
    for (uint32_t k = 0;; k++) {
        const unsigned long long tb = globaltimer();
        batch_body<C, NTT, CL, false, true>(a.bp, s, k, k == 0);
        __syncthreads();
        const unsigned long long tc = globaltimer();
        t_body += tc - tb;
        const bool more = async_commit<CL>(a, s, k);
        t_commit += globaltimer() - tc;
        if (!more) break;
    }
    if (a.profile && threadIdx.x == 0 && (CL == 1 || cluster_rank() == 0)) {
        atomicAdd(a.lock_ns + 7, t_body);                    // time in batches
        atomicAdd(a.lock_ns + 8, globaltimer() - t_start);   // CTA lifetime
        atomicAdd(a.lock_ns + 9, t_commit);                  // time in commits
    }
}

// Pools back to rank order after the run (what dabs_read_pool and the
// exchange expect): one CTA per pool gathers rows through ord into scratch,
// then copies them back.
__global__ void async_compact_kernel(const PoolView* __restrict__ pools, const int32_t* __restrict__ ord, int cap,
                                     int nwp, uint32_t* sX, int64_t* sE, uint64_t* sSeq, uint8_t* sA, uint8_t* sG)
{
    const int p = blockIdx.x;
    const PoolView pool = pools[p];
    const int32_t* o = ord + (size_t)p * cap;
    uint32_t* X = sX + (size_t)p * cap * nwp;
    for (size_t i = threadIdx.x; i < (size_t)cap * nwp; i += blockDim.x) {
        const size_t r = i / nwp, w = i % nwp;
        X[i] = pool.X[(size_t)o[r] * nwp + w];
    }
    for (int r = threadIdx.x; r < cap; r += blockDim.x) {
        sE[(size_t)p * cap + r] = pool.E[o[r]];
        sSeq[(size_t)p * cap + r] = pool.seq[o[r]];
        sA[(size_t)p * cap + r] = pool.algo[o[r]];
        sG[(size_t)p * cap + r] = pool.genop[o[r]];
    }
    __syncthreads();
    for (size_t i = threadIdx.x; i < (size_t)cap * nwp; i += blockDim.x) pool.X[i] = X[i];
    for (int r = threadIdx.x; r < cap; r += blockDim.x) {
        pool.E[r] = sE[(size_t)p * cap + r];
        pool.seq[r] = sSeq[(size_t)p * cap + r];
        pool.algo[r] = sA[(size_t)p * cap + r];
        pool.genop[r] = sG[(size_t)p * cap + r];
    }
}

}  // namespace dabs
