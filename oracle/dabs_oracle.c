/*
 * oracle/dabs_oracle.c -- CPU ORACLE for the DABS hot path (arXiv 2207.03069).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` legs may load this library.  The product
 * path (paper_2207_03069_b200/) never imports, links or calls it, and the two
 * share no code: this file has its own Philox, its own one-byte-per-bit
 * layouts and its own plain loops.
 *
 * Plain, slow, obviously correct.  Every function cites the passage it
 * follows:  P:n = /root/reference/PAPER.md line n (section / equation named),
 * R-x = the reading listed in DESIGN.md section "Readings" where the paper is
 * silent, garbled or ambiguous.  All arithmetic is integer: W int16, Delta
 * int32, E int64 (R-1, R-13).
 *
 * Pins (tests/test_oracle_*.py): brute force over all 2^n vectors (n<=20),
 * the reconstructed Fig. 1 fixture, SPEC worked examples, the paper's
 * TwoNeighbor n=6 trace, the 2300>=2000 batch example
 * (P:526-531), Philox KAT vectors, closed-form rank-bias probability
 * (P:576-578), and the checked mode below (Delta recomputed from scratch by
 * direct energy differences after every flip).  The asynchronous schedule
 * (R-29, orc_world_async_*) is pinned by its one-slot equivalence with the
 * generation schedule and the XREAD step recomputed from Philox in the test;
 * jump-start (R-30) by equality with Straight's incremental path.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define ORC_TABU_MAX 32
#define ORC_E_INF INT64_MAX

/* main search algorithms, in the paper's order */
enum { ALG_MAXMIN = 0, ALG_CYCLICMIN = 1, ALG_RANDOMMIN = 2, ALG_POSITIVEMIN = 3,
       ALG_TWONEIGHBOR = 4, N_ALG = 5 };
/* genetic operations, in the paper's order, then the ABS solver's
   single operation "mutation after crossover" (ablation mode, R-27) */
enum { GEN_MUTATION = 0, GEN_CROSSOVER = 1, GEN_XROSSOVER = 2, GEN_ZERO = 3, GEN_ONE = 4,
       GEN_INTERVALZERO = 5, GEN_BEST = 6, GEN_RANDOM = 7, GEN_MUTCROSS = 8, N_GEN = 9 };
/* phases recorded in the trace: 0 Straight, 1 Greedy, 2+r main round r */
enum { PH_STRAIGHT = 0, PH_GREEDY = 1, PH_MAIN = 2 };
/* Philox purposes (R-16) */
enum { PUR_POOL_INIT = 1, PUR_GA_CHOICE = 2, PUR_GA_PARENT = 3, PUR_GA_MASK = 4,
       PUR_MAXMIN = 5, PUR_RANDMIN = 6, PUR_POSMIN = 7, PUR_POOL_TAGS = 8 };

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11), written out from its definition:    */
/* 10 rounds; round: (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2),           */
/*                                     hi(M0*c0)^c3^k1, lo(M0*c0));          */
/* key bumped by the Weyl constants between rounds.  Replaces the paper's    */
/* MT19937-seeded xorshift so runs are replayable (R-16).        */
/* ------------------------------------------------------------------------ */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* counter layout (R-16): (purpose<<24 | sub, id, generation, step); key = seed */
static void rng4(uint64_t seed, uint32_t purpose, uint32_t sub, uint32_t id, uint32_t gen,
                 uint32_t step, uint32_t out[4])
{
    uint32_t ctr[4] = {(purpose << 24) | (sub & 0xFFFFFFu), id, gen, step};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox(ctr, key, out);
}

/* floor(u * m / 2^32): a uniform pick in [0, m) from one 32-bit word (R-15) */
static uint32_t pick(uint32_t u, uint32_t m) { return (uint32_t)(((uint64_t)u * m) >> 32); }

/* ------------------------------------------------------------------------ */
/* Energy, Eq.(2), read as the upper triangle incl. the diagonal   */
/* with each unordered pair once (R-1).  U is row-major n*n; only i<=j read. */
/* ------------------------------------------------------------------------ */
static int16_t Uij(const int16_t* U, int n, int i, int j) { return U[(size_t)i * n + j]; }
/* S_ik = the coefficient of x_i x_k (i != k) */
static int32_t S(const int16_t* U, int n, int i, int k)
{
    return i < k ? Uij(U, n, i, k) : Uij(U, n, k, i);
}

int64_t orc_energy(const int16_t* U, int n, const uint8_t* x)
{
    int64_t e = 0;
    for (int i = 0; i < n; i++)
        for (int j = i; j < n; j++)
            e += (int64_t)Uij(U, n, i, j) * x[i] * x[j];
    return e;
}

/* Eq.(3): Delta_k = -sigma(x_k) * (sum_{j!=k} W_jk x_j + W_kk),  */
/* sigma(x)=2x-1.                                               */
void orc_delta_closed(const int16_t* U, int n, const uint8_t* x, int32_t* delta)
{
    for (int k = 0; k < n; k++) {
        int64_t field = Uij(U, n, k, k);
        for (int j = 0; j < n; j++)
            if (j != k) field += (int64_t)S(U, n, j, k) * x[j];
        int sig = 2 * x[k] - 1;
        delta[k] = (int32_t)(-sig * field);
    }
}

/* ------------------------------------------------------------------------ */
/* One search (one CUDA block in the paper): X, E(X), Delta, the  */
/* tabu ring (R-11), and the batch-scope BEST / E(BEST) (R-3).    */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n;
    const int16_t* U;
    uint8_t* x;       /* n, one byte per bit */
    int32_t* delta;   /* n */
    int64_t E;
    int32_t* ring;    /* ORC_TABU_MAX, ring[0] = most recent flip, -1 = empty */
    int tabu;         /* tabu period t; 8 in the experiments */
    /* batch scope */
    uint8_t* best;
    int64_t ebest;
    int64_t flips;    /* flips in this batch */
    int T, B;
    int64_t flip_limit;   /* sampling bound for timing only (0 = none): stop after this many flips */
    /* randomness */
    uint64_t seed;
    uint32_t slot, gen;
    /* trace */
    int32_t* tr_bit;
    int64_t* tr_E;
    int8_t* tr_phase;
    int64_t tr_cap;
    int phase;
    /* checked mode: recompute E and Delta from scratch after every flip */
    int checked;
    int jump;          /* jump-start (R-30): X <- D before the batch instead of Straight's flips */
    int err;
    int32_t* scratch;  /* n, for checked mode */
    uint8_t* scratch_x;
} search_t;

static int is_tabu(const search_t* s, int k)
{
    /* a flipped bit may not be flipped again in the next t flips */
    for (int j = 0; j < s->tabu; j++)
        if (s->ring[j] == k) return 1;
    return 0;
}

static void check_state(search_t* s)
{
    /* Checked mode: E must equal Eq.(2) evaluated directly, and every Delta_k
       must equal E(f_k(X)) - E(X) (the definition) -- evaluated by
       direct energy differences for n <= 64, else via Eq.(3). */
    int n = s->n;
    int64_t e = orc_energy(s->U, n, s->x);
    if (e != s->E) { s->err = 1; return; }
    if (n <= 64) {
        memcpy(s->scratch_x, s->x, n);
        for (int k = 0; k < n; k++) {
            s->scratch_x[k] ^= 1;
            int64_t d = orc_energy(s->U, n, s->scratch_x) - e;
            s->scratch_x[k] ^= 1;
            if (d != s->delta[k]) { s->err = 2; return; }
        }
    } else {
        orc_delta_closed(s->U, n, s->x, s->scratch);
        for (int k = 0; k < n; k++)
            if (s->scratch[k] != s->delta[k]) { s->err = 2; return; }
    }
}

/* Step 3: X <- f_i(X), E <- E + Delta_i; Eq.(4) for k != i,      */
/* Eq.(5) for k == i.  Then push i on the tabu ring (R-11).                   */
static void flip(search_t* s, int i)
{
    int n = s->n;
    int sig_i = 2 * s->x[i] - 1;            /* sigma(x_i) before the flip */
    s->E += s->delta[i];
    for (int k = 0; k < n; k++) {
        if (k == i) continue;
        int sig_k = 2 * s->x[k] - 1;
        s->delta[k] += S(s->U, n, i, k) * sig_i * sig_k;   /* Eq.(4) */
    }
    s->delta[i] = -s->delta[i];                              /* Eq.(5) */
    s->x[i] ^= 1;
    for (int j = ORC_TABU_MAX - 1; j > 0; j--) s->ring[j] = s->ring[j - 1];
    s->ring[0] = i;
    if (s->tr_bit && s->flips < s->tr_cap) {
        s->tr_bit[s->flips] = i;
        s->tr_E[s->flips] = s->E;
        s->tr_phase[s->flips] = (int8_t)s->phase;
    }
    s->flips++;
    if (s->checked) check_state(s);
    if (s->flip_limit && s->flips >= s->flip_limit && !s->err) s->err = 4;
}

/* Step 1 (typos read as R-2): minE over all 1-bit neighbours,     */
/* j = the lowest index attaining it; strict improvement updates BEST.        */
static int scan(search_t* s, int32_t* m_out)
{
    int j = 0;
    int32_t m = s->delta[0];
    for (int k = 1; k < s->n; k++)
        if (s->delta[k] < m) { m = s->delta[k]; j = k; }
    if (s->E + m < s->ebest) {
        s->ebest = s->E + m;
        memcpy(s->best, s->x, s->n);
        s->best[j] ^= 1;
    }
    if (m_out) *m_out = m;
    return j;
}

/* Greedy: flip argmin Delta until all Delta >= 0 (R-4). */
static void greedy(search_t* s)
{
    s->phase = PH_GREEDY;
    for (;;) {
        int32_t m;
        int j = scan(s, &m);
        if (m >= 0) return;
        flip(s, j);
        if (s->err) return;
    }
}

/* Straight: flip the minimum-Delta bit among bits with x != d     */
/* (lowest index on ties, R-5) until X == D.                                  */
static void straight(search_t* s, const uint8_t* D)
{
    s->phase = PH_STRAIGHT;
    for (;;) {
        int any = 0, j = -1;
        for (int k = 0; k < s->n; k++)
            if (s->x[k] != D[k]) { any = 1; break; }
        if (!any) return;
        scan(s, NULL);
        for (int k = 0; k < s->n; k++)
            if (s->x[k] != D[k] && (j < 0 || s->delta[k] < s->delta[j])) j = k;
        flip(s, j);
        if (s->err) return;
    }
}

/* eligible = non-tabu bits; if that set is empty, tabu is dropped (R-11) */
static void eligible_set(const search_t* s, uint8_t* elig)
{
    int any = 0;
    for (int k = 0; k < s->n; k++) { elig[k] = !is_tabu(s, k); any |= elig[k]; }
    if (!any)
        for (int k = 0; k < s->n; k++) elig[k] = 1;
}

/* choose the pick-th member (0-based, ascending index) of a candidate set */
static int nth_member(const uint8_t* c, int n, uint32_t pick_idx)
{
    uint32_t seen = 0;
    for (int k = 0; k < n; k++)
        if (c[k]) { if (seen == pick_idx) return k; seen++; }
    return -1;
}

/* MaxMin, integer form R-6:
   lo/hi over eligible bits; u = T - t; span = floor((hi-lo) u^3 / T^3);
   thr = lo + floor(r1 (span+1) / 2^32); candidates = eligible with Delta<=thr;
   pick the floor(r2 |C| / 2^32)-th candidate in index order. */
static int sel_maxmin(search_t* s, int t, uint8_t* elig, uint8_t* cand)
{
    int n = s->n;
    eligible_set(s, elig);
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    for (int k = 0; k < n; k++)
        if (elig[k]) { if (s->delta[k] < lo) lo = s->delta[k]; if (s->delta[k] > hi) hi = s->delta[k]; }
    uint64_t T = (uint64_t)s->T, u = (uint64_t)(s->T - t);
    u128 num = (u128)(uint64_t)((int64_t)hi - (int64_t)lo) * (u * u * u);
    uint64_t span = (uint64_t)(num / (u128)(T * T * T));
    uint32_t r[4];
    rng4(s->seed, PUR_MAXMIN, 0, s->slot, s->gen, (uint32_t)s->flips, r);
    int64_t thr = (int64_t)lo + (int64_t)(((u128)r[0] * (span + 1)) >> 32);
    uint32_t cnt = 0;
    for (int k = 0; k < n; k++) { cand[k] = elig[k] && (int64_t)s->delta[k] <= thr; cnt += cand[k]; }
    return nth_member(cand, n, pick(r[1], cnt));
}

/* CyclicMin, integer form R-7:
   w(t) = max(ceil(n t^3 / T^3), min(32, n)); window [cursor, cursor+w) mod n;
   argmin over non-tabu window bits (tabu dropped if none), lowest index. */
static int sel_cyclicmin(search_t* s, int t, int* cursor, uint8_t* elig)
{
    int n = s->n;
    uint64_t T3 = (uint64_t)s->T * s->T * s->T;
    uint64_t t3 = (uint64_t)t * t * t;
    u128 num = (u128)(uint64_t)n * t3;
    uint64_t w = (uint64_t)((num + T3 - 1) / T3);
    uint64_t c = n < 32 ? (uint64_t)n : 32u;
    if (w < c) w = c;
    if (w > (uint64_t)n) w = n;
    memset(elig, 0, n);
    for (uint64_t j = 0; j < w; j++) elig[(*cursor + j) % n] = 1;
    int j = -1;
    for (int k = 0; k < n; k++)
        if (elig[k] && !is_tabu(s, k) && (j < 0 || s->delta[k] < s->delta[j])) j = k;
    if (j < 0)
        for (int k = 0; k < n; k++)
            if (elig[k] && (j < 0 || s->delta[k] < s->delta[j])) j = k;
    *cursor = (int)((*cursor + w) % n);
    return j;
}

/* lowbias32 (C. Wellons' hash prospector): a bijective 32-bit mixer */
static uint32_t lowbias32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
uint32_t orc_lowbias32(uint32_t x) { return lowbias32(x); }

/* RandomMin, integer form R-8:
   p16 = min(65536, max(floor(65536 t^3/T^3), floor(2^21/n)));
   bit k is a candidate iff non-tabu and u16(k) < p16, where u16(k) is the
   16-bit half (k mod 2) of lowbias32(K + (k/2) * 0x9E3779B9) and
   K = word 0 of Philox(RANDMIN, 0, slot, gen, step) -- one keyed counter per
   flip, a cheap mixer per bit pair (the paper draws per-thread xorshift
   numbers); argmin over candidates (lowest index); empty -> argmin
   over eligible bits. */
static int sel_randommin(search_t* s, int t, uint8_t* elig)
{
    int n = s->n;
    uint64_t T3 = (uint64_t)s->T * s->T * s->T;
    uint64_t t3 = (uint64_t)t * t * t;
    uint64_t p = (uint64_t)(((u128)65536u * t3) / T3);
    uint64_t floor_p = (uint64_t)(2097152u / (uint32_t)n);
    if (p < floor_p) p = floor_p;
    if (p > 65536u) p = 65536u;
    int j = -1;
    uint32_t r[4];
    rng4(s->seed, PUR_RANDMIN, 0, s->slot, s->gen, (uint32_t)s->flips, r);
    const uint32_t K = r[0];
    for (int k = 0; k < n; k++) {
        uint32_t h = lowbias32(K + (uint32_t)(k / 2) * 0x9E3779B9u);
        uint32_t u16 = (h >> (16 * (k % 2))) & 0xFFFFu;
        if (!is_tabu(s, k) && u16 < p && (j < 0 || s->delta[k] < s->delta[j])) j = k;
    }
    if (j < 0) {
        eligible_set(s, elig);
        for (int k = 0; k < n; k++)
            if (elig[k] && (j < 0 || s->delta[k] < s->delta[j])) j = k;
    }
    return j;
}

/* PositiveMin, R-9: pm = min positive Delta over eligible bits
   (+inf if none); candidates = eligible with Delta <= pm; uniform pick in
   index order with floor(r |C| / 2^32). */
static int sel_positivemin(search_t* s, uint8_t* elig, uint8_t* cand)
{
    int n = s->n;
    eligible_set(s, elig);
    int64_t pm = INT64_MAX;
    for (int k = 0; k < n; k++)
        if (elig[k] && s->delta[k] > 0 && s->delta[k] < pm) pm = s->delta[k];
    uint32_t cnt = 0;
    for (int k = 0; k < n; k++) { cand[k] = elig[k] && (int64_t)s->delta[k] <= pm; cnt += cand[k]; }
    uint32_t r[4];
    rng4(s->seed, PUR_POSMIN, 0, s->slot, s->gen, (uint32_t)s->flips, r);
    return nth_member(cand, n, pick(r[0], cnt));
}

/* one main-search run: T flips, or the 2n-1 TwoNeighbor flips       */
static void main_search(search_t* s, int algo, int round, uint8_t* elig, uint8_t* cand)
{
    int n = s->n;
    s->phase = PH_MAIN + (round < 100 ? round : 100);
    if (algo == ALG_TWONEIGHBOR) {
        /* flip 0, then (k, k-1) for k = 1..n-1 -- 2n-1 flips (R-10) */
        scan(s, NULL);
        flip(s, 0);
        for (int k = 1; k < n && !s->err; k++) {
            scan(s, NULL); flip(s, k);
            if (s->err) return;
            scan(s, NULL); flip(s, k - 1);
        }
        return;
    }
    int cursor = 0;   /* CyclicMin window starts at bit 0 each run (R-7) */
    for (int t = 1; t <= s->T && !s->err; t++) {
        scan(s, NULL);
        int i = -1;
        switch (algo) {
        case ALG_MAXMIN: i = sel_maxmin(s, t, elig, cand); break;
        case ALG_CYCLICMIN: i = sel_cyclicmin(s, t, &cursor, elig); break;
        case ALG_RANDOMMIN: i = sel_randommin(s, t, elig); break;
        case ALG_POSITIVEMIN: i = sel_positivemin(s, elig, cand); break;
        }
        if (i < 0) { s->err = 3; return; }
        flip(s, i);
    }
}

/* Batch search (R-12): E(BEST)=+inf; Straight(D); Greedy;
   do { main; Greedy } while (algo != TwoNeighbor && flips < B). */
static void batch(search_t* s, const uint8_t* D, int algo)
{
    int n = s->n;
    uint8_t* elig = (uint8_t*)malloc(n);
    uint8_t* cand = (uint8_t*)malloc(n);
    s->ebest = ORC_E_INF;
    s->flips = 0;
    if (s->jump) {
        /* jump-start (P:498-500 read with SURVEY f4, R-30): the batch starts AT
           the target: X = D, E = E(D) by Eq.(2), Delta by Eq.(3) from scratch;
           no flips, no scans, the tabu ring untouched.  Straight then has
           nothing to do. */
        memcpy(s->x, D, n);
        s->E = orc_energy(s->U, n, s->x);
        orc_delta_closed(s->U, n, s->x, s->delta);
    }
    straight(s, D);
    if (!s->err) greedy(s);
    int round = 0;
    if (!s->err) {
        do {
            main_search(s, algo, round++, elig, cand);
            if (s->err) break;
            greedy(s);
            if (s->err) break;
        } while (algo != ALG_TWONEIGHBOR && s->flips < s->B);
    }
    free(elig);
    free(cand);
}

/* T = max(1, ceil(s_milli n / 1000)), B = max(1, ceil(b_milli n / 1000)) (R-13) */
int orc_flip_factor(int milli, int n)
{
    int64_t v = ((int64_t)milli * n + 999) / 1000;
    return v < 1 ? 1 : (int)v;
}

/*
 * Batch-level entry point (one slot, one packet).  In/out: x, delta, E, ring
 * (the slot's persistent state, R-14).  Out: best, ebest, flips.
 * trace arrays (optional, may be NULL) receive (bit, E after flip, phase) per
 * flip.  Returns 0, or an error code: 1/2 checked-mode mismatch, 3 empty
 * selection.
 */
int orc_batch_limited(const int16_t* U, int n, int T, int B, int tabu,
                      uint8_t* x, int32_t* delta, int64_t* E, int32_t* ring,
                      const uint8_t* D, int algo, uint64_t seed, uint32_t slot, uint32_t gen,
                      uint8_t* best, int64_t* ebest, int64_t* flips,
                      int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase, int64_t tr_cap, int checked,
                      int64_t flip_limit);

int orc_batch(const int16_t* U, int n, int T, int B, int tabu,
              uint8_t* x, int32_t* delta, int64_t* E, int32_t* ring,
              const uint8_t* D, int algo, uint64_t seed, uint32_t slot, uint32_t gen,
              uint8_t* best, int64_t* ebest, int64_t* flips,
              int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase, int64_t tr_cap, int checked)
{
    return orc_batch_limited(U, n, T, B, tabu, x, delta, E, ring, D, algo, seed, slot, gen, best, ebest,
                             flips, tr_bit, tr_E, tr_phase, tr_cap, checked, 0);
}

/* orc_batch with the jump-start variant (jump = 1, R-30) and a flip limit
   (> 0: stop after that many flips, returns 4; a bounded sample of a batch,
   used only to time the oracle in bench cpu_baseline). */
int orc_batch_ex(const int16_t* U, int n, int T, int B, int tabu,
                 uint8_t* x, int32_t* delta, int64_t* E, int32_t* ring,
                 const uint8_t* D, int algo, uint64_t seed, uint32_t slot, uint32_t gen,
                 uint8_t* best, int64_t* ebest, int64_t* flips,
                 int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase, int64_t tr_cap, int checked,
                 int64_t flip_limit, int jump);

int orc_batch_limited(const int16_t* U, int n, int T, int B, int tabu,
                      uint8_t* x, int32_t* delta, int64_t* E, int32_t* ring,
                      const uint8_t* D, int algo, uint64_t seed, uint32_t slot, uint32_t gen,
                      uint8_t* best, int64_t* ebest, int64_t* flips,
                      int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase, int64_t tr_cap, int checked,
                      int64_t flip_limit)
{
    return orc_batch_ex(U, n, T, B, tabu, x, delta, E, ring, D, algo, seed, slot, gen, best, ebest, flips,
                        tr_bit, tr_E, tr_phase, tr_cap, checked, flip_limit, 0);
}

int orc_batch_ex(const int16_t* U, int n, int T, int B, int tabu,
                 uint8_t* x, int32_t* delta, int64_t* E, int32_t* ring,
                 const uint8_t* D, int algo, uint64_t seed, uint32_t slot, uint32_t gen,
                 uint8_t* best, int64_t* ebest, int64_t* flips,
                 int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase, int64_t tr_cap, int checked,
                 int64_t flip_limit, int jump)
{
    search_t s;
    memset(&s, 0, sizeof s);
    s.flip_limit = flip_limit;
    s.jump = jump;
    s.n = n; s.U = U; s.x = x; s.delta = delta; s.E = *E; s.ring = ring; s.tabu = tabu;
    s.best = best; s.T = T; s.B = B; s.seed = seed; s.slot = slot; s.gen = gen;
    s.tr_bit = tr_bit; s.tr_E = tr_E; s.tr_phase = tr_phase; s.tr_cap = tr_cap;
    s.checked = checked;
    if (checked) {
        s.scratch = (int32_t*)malloc(sizeof(int32_t) * n);
        s.scratch_x = (uint8_t*)malloc(n);
    }
    batch(&s, D, algo);
    *E = s.E; *ebest = s.ebest; *flips = s.flips;
    free(s.scratch); free(s.scratch_x);
    return s.err;
}

/* Exposed single steps, used by the pin tests to script phases. */
int orc_step_flip(const int16_t* U, int n, uint8_t* x, int32_t* delta, int64_t* E, int32_t* ring, int i)
{
    search_t s;
    memset(&s, 0, sizeof s);
    s.n = n; s.U = U; s.x = x; s.delta = delta; s.E = *E; s.ring = ring;
    flip(&s, i);
    *E = s.E;
    return 0;
}

/* ======================================================================== */
/* GA, solution pools, island ring                              */
/* ======================================================================== */
typedef struct {
    uint8_t* X;     /* cap * n */
    int64_t* E;     /* cap */
    uint64_t* seq;  /* cap: (generation+1)<<32 | global slot; sentinels: row */
    uint8_t* algo;
    uint8_t* genop;
} pool_t;

typedef struct {
    int n, T, B, tabu, cap;
    int16_t* U;
    uint64_t eps_thr;             /* floor(eps * 2^32) (R-15); 2^32 at eps = 1, so 64-bit */
    int n_gen, gens[N_GEN];
    int n_alg, algs[N_ALG];
    int P, S, rank, world;        /* pools per rank, slots per pool */
    uint64_t seed;
    uint32_t gen;                 /* current generation */
    pool_t* pools;                /* P */
    pool_t nbr;                   /* successor snapshot for the last local pool (R-23) */
    /* slots (P*S) */
    uint8_t* sx; int32_t* sdelta; int64_t* sE; int32_t* sring;
    /* packets */
    uint8_t* D; uint8_t* palgo; uint8_t* pgenop;
    uint8_t* rbest; int64_t* rE; int64_t* rflips;
    /* statistics */
    uint64_t* dispatch;   /* P * N_ALG * N_GEN */
    uint64_t* inserted;   /* P * N_ALG * N_GEN */
    /* restart-on-merge (R-28): generations without a box-wide
       improvement, the limit (0 = off), restarts so far */
    uint32_t stall, restart_gens, restarts;
    /* run-level */
    int64_t best_E; uint8_t* best_X; int best_algo, best_genop; int64_t best_gen; int64_t best_slot;
    uint64_t total_flips;
    uint64_t gen_flips;
    int checked;
    int err;
    /* asynchronous schedule (R-29): per-slot batch index, finished, XREAD pending */
    uint32_t* a_k; uint8_t* a_done; uint8_t* a_pending; int64_t a_events;
    int jump;   /* jump-start batches (R-30) */
} world_t;

static void pool_alloc(pool_t* p, int cap, int n)
{
    p->X = (uint8_t*)calloc((size_t)cap * n, 1);
    p->E = (int64_t*)calloc(cap, sizeof(int64_t));
    p->seq = (uint64_t*)calloc(cap, sizeof(uint64_t));
    p->algo = (uint8_t*)calloc(cap, 1);
    p->genop = (uint8_t*)calloc(cap, 1);
}
static void pool_free(pool_t* p) { free(p->X); free(p->E); free(p->seq); free(p->algo); free(p->genop); }

/* a pool starts as random vectors with +inf energy and random
   algorithm / genop columns (R-19).  `gen` = 0 at reset, the generation
   counter at a restart (R-28). */
static void pool_init(const world_t* w, pool_t* p, uint32_t gpool, uint32_t gen)
{
    int n = w->n;
    for (int r = 0; r < w->cap; r++) {
        for (int k = 0; k < n; k++) {
            uint32_t o[4];
            rng4(w->seed, PUR_POOL_INIT, (uint32_t)(k / 32), gpool, gen, (uint32_t)r, o);
            p->X[(size_t)r * n + k] = (uint8_t)((o[0] >> (k % 32)) & 1u);
        }
        uint32_t o[4];
        rng4(w->seed, PUR_POOL_TAGS, 0, gpool, gen, (uint32_t)r, o);
        p->genop[r] = (uint8_t)w->gens[pick(o[0], (uint32_t)w->n_gen)];
        p->algo[r] = (uint8_t)w->algs[pick(o[1], (uint32_t)w->n_alg)];
        p->E[r] = ORC_E_INF;
        p->seq[r] = (uint64_t)r;
    }
}

void* orc_world_new(const int16_t* U, int n, int s_milli, int b_milli, int tabu, int cap,
                    uint32_t eps_ppm, uint32_t genop_mask, uint32_t algo_mask,
                    int P, int S, int rank, int world)
{
    world_t* w = (world_t*)calloc(1, sizeof(world_t));
    w->n = n; w->tabu = tabu; w->cap = cap; w->P = P; w->S = S; w->rank = rank; w->world = world;
    w->T = orc_flip_factor(s_milli, n);
    w->B = orc_flip_factor(b_milli, n);
    w->U = (int16_t*)malloc(sizeof(int16_t) * (size_t)n * n);
    memcpy(w->U, U, sizeof(int16_t) * (size_t)n * n);
    w->eps_thr = ((uint64_t)eps_ppm << 32) / 1000000u;
    for (int g = 0; g < N_GEN; g++) if (genop_mask >> g & 1) w->gens[w->n_gen++] = g;
    for (int a = 0; a < N_ALG; a++) if (algo_mask >> a & 1) w->algs[w->n_alg++] = a;
    w->pools = (pool_t*)calloc(P, sizeof(pool_t));
    for (int p = 0; p < P; p++) pool_alloc(&w->pools[p], cap, n);
    pool_alloc(&w->nbr, cap, n);
    int ns = P * S;
    w->sx = (uint8_t*)calloc((size_t)ns * n, 1);
    w->sdelta = (int32_t*)calloc((size_t)ns * n, sizeof(int32_t));
    w->sE = (int64_t*)calloc(ns, sizeof(int64_t));
    w->sring = (int32_t*)calloc((size_t)ns * ORC_TABU_MAX, sizeof(int32_t));
    w->D = (uint8_t*)calloc((size_t)ns * n, 1);
    w->palgo = (uint8_t*)calloc(ns, 1);
    w->pgenop = (uint8_t*)calloc(ns, 1);
    w->rbest = (uint8_t*)calloc((size_t)ns * n, 1);
    w->rE = (int64_t*)calloc(ns, sizeof(int64_t));
    w->rflips = (int64_t*)calloc(ns, sizeof(int64_t));
    w->dispatch = (uint64_t*)calloc((size_t)P * N_ALG * N_GEN, sizeof(uint64_t));
    w->inserted = (uint64_t*)calloc((size_t)P * N_ALG * N_GEN, sizeof(uint64_t));
    w->best_X = (uint8_t*)calloc(n, 1);
    return w;
}

void orc_world_free(void* vw)
{
    world_t* w = (world_t*)vw;
    if (!w) return;
    for (int p = 0; p < w->P; p++) pool_free(&w->pools[p]);
    pool_free(&w->nbr);
    free(w->pools); free(w->U);
    free(w->sx); free(w->sdelta); free(w->sE); free(w->sring);
    free(w->D); free(w->palgo); free(w->pgenop); free(w->rbest); free(w->rE); free(w->rflips);
    free(w->dispatch); free(w->inserted); free(w->best_X);
    free(w->a_k); free(w->a_done); free(w->a_pending);
    free(w);
}

void orc_world_set_checked(void* vw, int checked) { ((world_t*)vw)->checked = checked; }
void orc_world_set_restart(void* vw, uint32_t gens) { ((world_t*)vw)->restart_gens = gens; }
void orc_world_set_jump(void* vw, int jump) { ((world_t*)vw)->jump = jump; }
uint32_t orc_world_restarts(void* vw) { return ((world_t*)vw)->restarts; }

/* pools from Philox (counter generation `gen`), slots at X=0, E=0,
   Delta_k=W_kk, empty tabu rings */
static void start_pools_and_slots(world_t* w, uint32_t gen)
{
    int n = w->n, ns = w->P * w->S;
    for (int p = 0; p < w->P; p++) pool_init(w, &w->pools[p], (uint32_t)(w->rank * w->P + p), gen);
    uint32_t succ = (uint32_t)(((w->rank + 1) * w->P) % (w->world * w->P));
    pool_init(w, &w->nbr, succ, gen);
    memset(w->sx, 0, (size_t)ns * n);
    for (int s = 0; s < ns; s++) {
        for (int k = 0; k < n; k++) w->sdelta[(size_t)s * n + k] = Uij(w->U, n, k, k);
        w->sE[s] = 0;
        for (int j = 0; j < ORC_TABU_MAX; j++) w->sring[(size_t)s * ORC_TABU_MAX + j] = -1;
    }
}

/* Reset: pools and slots as above, counters zero, generation 0. */
void orc_world_reset(void* vw, uint64_t seed)
{
    world_t* w = (world_t*)vw;
    int n = w->n;
    w->seed = seed;
    w->gen = 0;
    start_pools_and_slots(w, 0);
    w->stall = 0;
    w->restarts = 0;
    memset(w->dispatch, 0, sizeof(uint64_t) * w->P * N_ALG * N_GEN);
    memset(w->inserted, 0, sizeof(uint64_t) * w->P * N_ALG * N_GEN);
    w->best_E = ORC_E_INF; w->best_algo = -1; w->best_genop = -1; w->best_gen = -1; w->best_slot = -1;
    memset(w->best_X, 0, n);
    w->total_flips = 0;
    w->gen_flips = 0;
    w->err = 0;
}

/* rank-biased parent (R-17): 0-based row floor(u^3 m / 2^96) */
static uint32_t rank_pick(uint32_t u, uint32_t m)
{
    u128 u3 = (u128)u * u * u;
    return (uint32_t)((u3 * m) >> 96);
}

uint32_t orc_rank_pick(uint32_t u, uint32_t m) { return rank_pick(u, m); }

/* Apply one genetic operation (R-20) to parents A (and B for the
   crossovers; B comes from the successor pool for Xrossover).
   Bit k uses mask word k/32 of Philox(GA_MASK, k/32, gslot, gen, 0);
   IntervalZero clears the L bits start, start+1, ... (mod n). */
void orc_build_target(int genop, const uint8_t* A, const uint8_t* Bp, const uint8_t* best0, int n,
                      uint64_t seed, uint32_t gs, uint32_t gen, uint32_t L, uint32_t start, uint8_t* D)
{
    for (int k = 0; k < n; k++) {
        uint32_t m[4];
        rng4(seed, PUR_GA_MASK, (uint32_t)(k / 32), gs, gen, 0, m);
        int bit = k % 32;
        int m0 = (m[0] >> bit) & 1, m1 = (m[1] >> bit) & 1, m2 = (m[2] >> bit) & 1;
        int m3 = (m[3] >> bit) & 1;
        int p8 = m0 & m1 & m2;   /* probability 1/8 (R-20) */
        int v = 0;
        switch (genop) {
        case GEN_MUTATION: v = A[k] ^ p8; break;
        case GEN_CROSSOVER:
        case GEN_XROSSOVER: v = m0 ? A[k] : Bp[k]; break;
        case GEN_ZERO: v = p8 ? 0 : A[k]; break;
        case GEN_ONE: v = p8 ? 1 : A[k]; break;
        case GEN_INTERVALZERO:
            v = ((uint32_t)((k - (int)start + n) % n) < L) ? 0 : A[k]; break;
        case GEN_BEST: v = best0[k]; break;
        case GEN_RANDOM: v = m0; break;
        case GEN_MUTCROSS: v = (m3 ? A[k] : Bp[k]) ^ p8; break;        /* P:188-189, R-27 */
        }
        D[k] = (uint8_t)v;
    }
}

/* GA seeding for one slot (R-15, R-17, R-20, R-23).  `gen` is the
   Philox generation field: the generation (bulk-synchronous schedule) or the
   slot's batch index (asynchronous schedule, R-29).  `live_ring`: the last
   pool's Xrossover partner is local pool 0 as it is now (R-29) instead of the
   successor snapshot (R-23). */
static void ga_seed_g(world_t* w, int s, uint32_t gen, int live_ring)
{
    int n = w->n, cap = w->cap;
    int p = s / w->S;
    uint32_t gs = (uint32_t)(w->rank * w->P * w->S + s);
    const pool_t* pool = &w->pools[p];
    const pool_t* succ = (p + 1 < w->P) ? &w->pools[p + 1] : (live_ring ? &w->pools[0] : &w->nbr);
    uint32_t a[4], b[4];
    rng4(w->seed, PUR_GA_CHOICE, 0, gs, gen, 0, a);
    int genop = ((uint64_t)a[0] < w->eps_thr) ? w->gens[pick(a[1], (uint32_t)w->n_gen)]
                                    : pool->genop[pick(a[1], (uint32_t)cap)];
    int algo = ((uint64_t)a[2] < w->eps_thr) ? w->algs[pick(a[3], (uint32_t)w->n_alg)]
                                   : pool->algo[pick(a[3], (uint32_t)cap)];
    rng4(w->seed, PUR_GA_PARENT, 0, gs, gen, 0, b);
    uint32_t r1 = rank_pick(b[0], (uint32_t)cap), r2 = rank_pick(b[1], (uint32_t)cap);
    const uint8_t* A = pool->X + (size_t)r1 * n;
    const uint8_t* Bp = (genop == GEN_XROSSOVER ? succ->X : pool->X) + (size_t)r2 * n;
    /* IntervalZero (R-20): L in [lo, hi], start in [0, n), cyclic */
    uint32_t lo = n < 32 ? (uint32_t)n : 32u;
    uint32_t hi = (uint32_t)(n / 2) > lo ? (uint32_t)(n / 2) : lo;
    uint32_t L = lo + pick(b[2], hi - lo + 1);
    uint32_t start = pick(b[3], (uint32_t)n);
    uint8_t* D = w->D + (size_t)s * n;
    orc_build_target(genop, A, Bp, pool->X, n, w->seed, gs, gen, L, start, D);
    w->palgo[s] = (uint8_t)algo;
    w->pgenop[s] = (uint8_t)genop;
    w->dispatch[((size_t)p * N_ALG + algo) * N_GEN + genop]++;
}

static void ga_seed(world_t* w, int s) { ga_seed_g(w, s, w->gen, 0); }

/* Asynchronous schedule, R-29: an Xrossover packet whose partner is another
   pool is built in two steps.  At the merge event only the bits the mask
   takes from the own parent A are set (D = A where m0, 0 elsewhere; i.e.
   orc_build_target with an all-zero B); the slot's next XREAD event fills
   the others from the partner pool's rank-r2 row as the pool is then.
   Returns 1 if the packet is pending. */
static int ga_seed_async(world_t* w, int s, uint32_t gen)
{
    int p = s / w->S;
    int pn = (p + 1) % w->P;
    if (pn == p) { ga_seed_g(w, s, gen, 1); return 0; }
    /* same draws as ga_seed_g; the partner row is replaced by zeros */
    pool_t saved = w->pools[pn];
    pool_t zero;
    pool_alloc(&zero, w->cap, w->n);   /* calloc: all-zero rows */
    w->pools[pn] = zero;
    ga_seed_g(w, s, gen, 1);
    w->pools[pn] = saved;
    pool_free(&zero);
    return w->pgenop[s] == GEN_XROSSOVER;
}

/* the XREAD step: D[k] = partner row r2, bit k, wherever mask word bit m0 = 0 */
static void xread_async(world_t* w, int s, uint32_t gen)
{
    int n = w->n;
    int p = s / w->S;
    int pn = (p + 1) % w->P;
    uint32_t gs = (uint32_t)(w->rank * w->P * w->S + s);
    uint32_t b[4];
    rng4(w->seed, PUR_GA_PARENT, 0, gs, gen, 0, b);
    uint32_t r2 = rank_pick(b[1], (uint32_t)w->cap);
    const uint8_t* B = w->pools[pn].X + (size_t)r2 * n;
    uint8_t* D = w->D + (size_t)s * n;
    for (int k = 0; k < n; k++) {
        uint32_t m[4];
        rng4(w->seed, PUR_GA_MASK, (uint32_t)(k / 32), gs, gen, 0, m);
        if (!((m[0] >> (k % 32)) & 1)) D[k] = B[k];
    }
}

/* merge one pool (R-18): stable sort of old ++ new by (E, seq),
   drop results equal in (E, X) to an earlier finite entry, keep `cap`. */
typedef struct { int64_t E; uint64_t seq; int src; /* <0: old row -(r+1); >=0: slot */ } cand_t;

static int cand_cmp(const void* a, const void* b)
{
    const cand_t* x = (const cand_t*)a; const cand_t* y = (const cand_t*)b;
    if (x->E != y->E) return x->E < y->E ? -1 : 1;
    if (x->seq != y->seq) return x->seq < y->seq ? -1 : 1;
    return 0;
}

/* merge the results of slots slot[0..m-1] (their packets) with sequence
   numbers seqs[] into pool p */
static void merge_results(world_t* w, int p, const int* slot, const uint64_t* seqs, int m)
{
    int n = w->n, cap = w->cap;
    pool_t* pool = &w->pools[p];
    int M = cap + m;
    cand_t* c = (cand_t*)malloc(sizeof(cand_t) * M);
    for (int r = 0; r < cap; r++) { c[r].E = pool->E[r]; c[r].seq = pool->seq[r]; c[r].src = -(r + 1); }
    for (int j = 0; j < m; j++) {
        c[cap + j].E = w->rE[slot[j]];
        c[cap + j].seq = seqs[j];
        c[cap + j].src = slot[j];
    }
    qsort(c, M, sizeof(cand_t), cand_cmp);
    pool_t np;
    pool_alloc(&np, cap, n);
    int kept = 0;
    for (int j = 0; j < M && kept < cap; j++) {
        const uint8_t* X = c[j].src < 0 ? pool->X + (size_t)(-c[j].src - 1) * n
                                         : w->rbest + (size_t)c[j].src * n;
        int dup = 0;
        if (c[j].E != ORC_E_INF)
            for (int q = 0; q < kept && !dup; q++)
                if (np.E[q] == c[j].E && memcmp(np.X + (size_t)q * n, X, n) == 0) dup = 1;
        if (dup) continue;
        memcpy(np.X + (size_t)kept * n, X, n);
        np.E[kept] = c[j].E;
        np.seq[kept] = c[j].seq;
        if (c[j].src < 0) {
            np.algo[kept] = pool->algo[-c[j].src - 1];
            np.genop[kept] = pool->genop[-c[j].src - 1];
        } else {
            np.algo[kept] = w->palgo[c[j].src];
            np.genop[kept] = w->pgenop[c[j].src];
            w->inserted[((size_t)p * N_ALG + np.algo[kept]) * N_GEN + np.genop[kept]]++;
        }
        kept++;
    }
    pool_free(pool);
    *pool = np;
    free(c);
}

/* the generation's merge: pool p takes its S slots' results, in slot order,
   with seq = (generation+1)<<32 | global slot */
static void merge_pool(world_t* w, int p)
{
    int S = w->S;
    int* slot = (int*)malloc(sizeof(int) * S);
    uint64_t* seqs = (uint64_t*)malloc(sizeof(uint64_t) * S);
    for (int j = 0; j < S; j++) {
        slot[j] = p * S + j;
        seqs[j] = ((uint64_t)(w->gen + 1) << 32) | (uint32_t)(w->rank * w->P * S + slot[j]);
    }
    merge_results(w, p, slot, seqs, S);
    free(slot);
    free(seqs);
}

/* The local part of one generation: GA seeding for every slot, one batch per
   slot (slot order), then the per-pool merge.  Returns 0 or an error. */
int orc_world_generation_local(void* vw)
{
    world_t* w = (world_t*)vw;
    int n = w->n, ns = w->P * w->S;
    for (int s = 0; s < ns; s++) ga_seed(w, s);
    w->gen_flips = 0;
    for (int s = 0; s < ns; s++) {
        uint32_t gs = (uint32_t)(w->rank * ns + s);
        int err = orc_batch_ex(w->U, n, w->T, w->B, w->tabu,
                               w->sx + (size_t)s * n, w->sdelta + (size_t)s * n, &w->sE[s],
                               w->sring + (size_t)s * ORC_TABU_MAX,
                               w->D + (size_t)s * n, w->palgo[s], w->seed, gs, w->gen,
                               w->rbest + (size_t)s * n, &w->rE[s], &w->rflips[s],
                               NULL, NULL, NULL, 0, w->checked, 0, w->jump);
        if (err) { w->err = err; return err; }
        w->gen_flips += (uint64_t)w->rflips[s];
    }
    for (int p = 0; p < w->P; p++) merge_pool(w, p);
    return 0;
}

/* Asynchronous schedule (reading R-29), replayed from a log.
   The paper's host hands each block a new packet as soon as its previous batch
   returns; there is no generation barrier.  Each slot s
   runs batches k = 0, 1, 2, ...; batch k uses the Philox generation field k.
   Every slot's packet 0 is seeded from the freshly initialised pools (k = 0)
   before any batch.  log[e] = s | seeded<<31 is the e-th merge event, in the
   order the device serialised them: slot s's current batch result enters its
   pool as one result with seq = (e+1)<<32 | global slot (rule R-18 with one
   newcomer); the run best and its record (event index as `generation`) are
   updated on strict improvement; then, if `seeded`, packet k+1 is drawn from
   the pools as they are after this merge, with the last pool's Xrossover
   partner = local pool 0, live (R-29).  Single rank only.
   An Xrossover packet whose partner is another pool is completed by the
   slot's XREAD event (log entry s | 1<<30), which reads the partner pool as
   it is at that point of the log (ga_seed_async / xread_async above).
   Returns 0, or 20 (bad slot), 21 (event after the slot's last batch),
   22 (a slot without a final unseeded event), 24 (a batch or XREAD out of
   turn), or a batch error. */
static void async_free(world_t* w)
{
    free(w->a_k); free(w->a_done); free(w->a_pending);
    w->a_k = NULL; w->a_done = NULL; w->a_pending = NULL;
}

/* start of an asynchronous run (after orc_world_reset): packet 0 of every slot */
int orc_world_async_begin(void* vw)
{
    world_t* w = (world_t*)vw;
    int ns = w->P * w->S;
    if (w->world != 1) return 23;
    async_free(w);
    w->a_k = (uint32_t*)calloc(ns, sizeof(uint32_t));
    w->a_done = (uint8_t*)calloc(ns, 1);
    w->a_pending = (uint8_t*)calloc(ns, 1);
    w->a_events = 0;
    for (int s = 0; s < ns; s++) ga_seed_g(w, s, 0, 1);
    return 0;
}

/* one log entry; returns 0 / 1 (the slot's packet now waits for its XREAD)
   or -error */
int orc_world_async_event(void* vw, uint32_t entry)
{
    world_t* w = (world_t*)vw;
    int n = w->n, ns = w->P * w->S;
    int s = (int)(entry & 0x3FFFFFFFu);
    int seeded = (int)(entry >> 31);
    int xread = (int)((entry >> 30) & 1u);
    int64_t e = w->a_events;
    if (!w->a_k) return -25;
    if (s >= ns) return -20;
    if (w->a_done[s]) return -21;
    if (xread != w->a_pending[s]) return -24;
    w->a_events++;
    if (xread) {
        xread_async(w, s, w->a_k[s]);
        w->a_pending[s] = 0;
        return 0;
    }
    uint32_t gs = (uint32_t)s;
    int err = orc_batch(w->U, n, w->T, w->B, w->tabu,
                        w->sx + (size_t)s * n, w->sdelta + (size_t)s * n, &w->sE[s],
                        w->sring + (size_t)s * ORC_TABU_MAX,
                        w->D + (size_t)s * n, w->palgo[s], w->seed, gs, w->a_k[s],
                        w->rbest + (size_t)s * n, &w->rE[s], &w->rflips[s],
                        NULL, NULL, NULL, 0, w->checked);
    if (err) return -err;
    w->total_flips += (uint64_t)w->rflips[s];
    uint64_t seq = ((uint64_t)(e + 1) << 32) | gs;
    merge_results(w, s / w->S, &s, &seq, 1);
    if (w->rE[s] < w->best_E) {
        w->best_E = w->rE[s];
        memcpy(w->best_X, w->rbest + (size_t)s * n, n);
        w->best_algo = w->palgo[s]; w->best_genop = w->pgenop[s];
        w->best_gen = e; w->best_slot = gs;
    }
    if (seeded) {
        w->a_k[s]++;
        w->a_pending[s] = (uint8_t)ga_seed_async(w, s, w->a_k[s]);
        return w->a_pending[s];
    }
    w->a_done[s] = 1;
    return 0;
}

/* end of the log: every slot has merged its final batch */
int orc_world_async_end(void* vw)
{
    world_t* w = (world_t*)vw;
    int ns = w->P * w->S;
    if (!w->a_k) return 25;
    for (int s = 0; s < ns; s++) if (!w->a_done[s]) return 22;
    return 0;
}

int orc_world_async_replay(void* vw, const uint32_t* log, int64_t len)
{
    world_t* w = (world_t*)vw;
    int err = orc_world_async_begin(vw);
    for (int64_t e = 0; e < len && !err; e++) {
        int r = orc_world_async_event(vw, log[e]);
        if (r < 0) err = -r;
    }
    if (!err) err = orc_world_async_end(vw);
    if (err) w->err = err;
    return err;
}

/* Exchange payload (oracle format): first local pool + this rank's best
   entry + this generation's flips.  Layout (bytes):
     cap*n X | cap int64 E | cap uint64 seq | cap algo | cap genop |
     int64 bestE | uint64 bestSeq | int32 bestPool | int32 algo | int32 genop | n X | uint64 flips */
long orc_world_payload_bytes(void* vw)
{
    world_t* w = (world_t*)vw;
    long cap = w->cap, n = w->n;
    return cap * n + cap * 8 + cap * 8 + cap + cap + 8 + 8 + 4 + 4 + 4 + n + 8;
}

void orc_world_export(void* vw, uint8_t* buf)
{
    world_t* w = (world_t*)vw;
    int cap = w->cap, n = w->n;
    const pool_t* p0 = &w->pools[0];
    uint8_t* q = buf;
    memcpy(q, p0->X, (size_t)cap * n); q += (size_t)cap * n;
    memcpy(q, p0->E, cap * 8); q += cap * 8;
    memcpy(q, p0->seq, cap * 8); q += cap * 8;
    memcpy(q, p0->algo, cap); q += cap;
    memcpy(q, p0->genop, cap); q += cap;
    /* best entry over local pools: lowest (E, pool id) */
    int bp = 0;
    for (int p = 1; p < w->P; p++) if (w->pools[p].E[0] < w->pools[bp].E[0]) bp = p;
    int64_t be = w->pools[bp].E[0];
    uint64_t bs = w->pools[bp].seq[0];
    int32_t gpool = w->rank * w->P + bp, ba = w->pools[bp].algo[0], bg = w->pools[bp].genop[0];
    memcpy(q, &be, 8); q += 8;
    memcpy(q, &bs, 8); q += 8;
    memcpy(q, &gpool, 4); q += 4;
    memcpy(q, &ba, 4); q += 4;
    memcpy(q, &bg, 4); q += 4;
    memcpy(q, w->pools[bp].X, n); q += n;
    memcpy(q, &w->gen_flips, 8); q += 8;
}

/* Import all ranks' payloads (concatenated, rank order): the successor snapshot
   for Xrossover (R-23), the run's best and first-best record, total flips.
   Then the generation counter advances. */
void orc_world_import(void* vw, const uint8_t* all)
{
    world_t* w = (world_t*)vw;
    int cap = w->cap, n = w->n;
    long pb = orc_world_payload_bytes(vw);
    const uint8_t* s = all + pb * ((w->rank + 1) % w->world);
    memcpy(w->nbr.X, s, (size_t)cap * n); s += (size_t)cap * n;
    memcpy(w->nbr.E, s, cap * 8); s += cap * 8;
    memcpy(w->nbr.seq, s, cap * 8); s += cap * 8;
    memcpy(w->nbr.algo, s, cap); s += cap;
    memcpy(w->nbr.genop, s, cap); s += cap;
    int64_t gbE = ORC_E_INF; int gbr = -1;
    for (int r = 0; r < w->world; r++) {
        const uint8_t* q = all + pb * r + (long)cap * n + cap * 18;
        int64_t be; uint64_t fl;
        memcpy(&be, q, 8);
        memcpy(&fl, q + 28 + n, 8);
        w->total_flips += fl;
        if (gbr < 0 || be < gbE) { gbE = be; gbr = r; }
    }
    if (gbE < w->best_E) {
        const uint8_t* q = all + pb * gbr + (long)cap * n + cap * 18;
        uint64_t bs; int32_t ba, bg;
        memcpy(&bs, q + 8, 8);
        memcpy(&ba, q + 20, 4);
        memcpy(&bg, q + 24, 4);
        w->best_E = gbE;
        memcpy(w->best_X, q + 28, n);
        w->best_algo = ba; w->best_genop = bg;
        w->best_gen = (int64_t)(bs >> 32) - 1;
        w->best_slot = (int64_t)(bs & 0xFFFFFFFFu);
        w->stall = 0;
    } else {
        w->stall++;
    }
    w->gen++;
    /* restart-on-merge (R-28): after restart_gens generations
       without a box-wide improvement, every rank re-initialises its pools and
       slots (the decision uses only gathered data, so all ranks agree); the
       run's best is kept */
    if (w->restart_gens && w->stall >= w->restart_gens) {
        start_pools_and_slots(w, w->gen);
        w->stall = 0;
        w->restarts++;
    }
}

/* ---- accessors for the Python wrapper ---- */
int orc_world_T(void* vw) { return ((world_t*)vw)->T; }
int orc_world_B(void* vw) { return ((world_t*)vw)->B; }
uint32_t orc_world_gen(void* vw) { return ((world_t*)vw)->gen; }
uint64_t orc_world_total_flips(void* vw) { return ((world_t*)vw)->total_flips; }
uint64_t orc_world_gen_flips(void* vw) { return ((world_t*)vw)->gen_flips; }

void orc_world_get_pool(void* vw, int p, uint8_t* X, int64_t* E, uint64_t* seq, uint8_t* algo, uint8_t* genop)
{
    world_t* w = (world_t*)vw;
    pool_t* q = (p < w->P) ? &w->pools[p] : &w->nbr;
    memcpy(X, q->X, (size_t)w->cap * w->n);
    memcpy(E, q->E, w->cap * 8);
    memcpy(seq, q->seq, w->cap * 8);
    memcpy(algo, q->algo, w->cap);
    memcpy(genop, q->genop, w->cap);
}

void orc_world_get_slot(void* vw, int s, uint8_t* x, int32_t* delta, int64_t* E, int32_t* ring)
{
    world_t* w = (world_t*)vw;
    int n = w->n;
    memcpy(x, w->sx + (size_t)s * n, n);
    memcpy(delta, w->sdelta + (size_t)s * n, sizeof(int32_t) * n);
    *E = w->sE[s];
    memcpy(ring, w->sring + (size_t)s * ORC_TABU_MAX, sizeof(int32_t) * ORC_TABU_MAX);
}

void orc_world_get_packet(void* vw, int s, uint8_t* D, int32_t* algo, int32_t* genop,
                          uint8_t* best, int64_t* ebest, int64_t* flips)
{
    world_t* w = (world_t*)vw;
    int n = w->n;
    memcpy(D, w->D + (size_t)s * n, n);
    *algo = w->palgo[s]; *genop = w->pgenop[s];
    memcpy(best, w->rbest + (size_t)s * n, n);
    *ebest = w->rE[s]; *flips = w->rflips[s];
}

void orc_world_get_stats(void* vw, uint64_t* dispatch, uint64_t* inserted)
{
    world_t* w = (world_t*)vw;
    memcpy(dispatch, w->dispatch, sizeof(uint64_t) * w->P * N_ALG * N_GEN);
    memcpy(inserted, w->inserted, sizeof(uint64_t) * w->P * N_ALG * N_GEN);
}

void orc_world_get_best(void* vw, int64_t* E, uint8_t* X, int32_t* rec /* algo, genop, gen, slot */)
{
    world_t* w = (world_t*)vw;
    *E = w->best_E;
    memcpy(X, w->best_X, w->n);
    rec[0] = w->best_algo; rec[1] = w->best_genop; rec[2] = (int32_t)w->best_gen; rec[3] = (int32_t)w->best_slot;
}
