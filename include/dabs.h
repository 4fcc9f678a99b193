/*
 * dabs.h -- C ABI of the B200-native DABS hot path (Nakano et al., "Diverse
 * Adaptive Bulk Search: a Framework for Solving QUBO Problems on Multiple
 * GPUs", arXiv 2207.03069).
 *
 * Citations: P:n = PAPER.md line n.  R-x = reading x in DESIGN.md section 2.
 *
 * Problem (Eq.(2), R-1): minimise E(X) = sum_{i<=j} W_ij x_i x_j
 * over X in {0,1}^n, W an integer upper-triangular matrix.  The library runs
 * many independent incremental local searches (Sec. III) seeded by a
 * GA over solution pools (Sec. IV), bulk-synchronously by
 * generations (R-25, R-26), entirely in hand-written sm_100a CUDA kernels.
 *
 * Conventions
 *  - Every pointer argument named *_host is host memory owned by the caller;
 *    the library copies what it needs before returning.  No pointer is
 *    retained across calls.
 *  - Bit vectors cross the ABI as n bytes, each 0 or 1 (bit k = byte k).
 *  - Every function returns a dabs_status and never throws; on failure,
 *    dabs_last_error() gives a thread-local message (CUDA errors carry their
 *    cudaGetErrorString text).  After DABS_E_CUDA the context must be
 *    destroyed.
 *  - A context must not be used from two threads at once; contexts are
 *    independent of each other.
 *  - There is no CPU fallback: without a usable sm_100a device every call
 *    that needs one returns DABS_E_CUDA.
 */
#ifndef DABS_H
#define DABS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DABS_OK = 0,
    DABS_E_ARG = 1,       /* bad argument (NULL, n out of range, bad config) */
    DABS_E_TRIANGLE = 2,  /* nonzero entry below the diagonal of W */
    DABS_E_RANGE = 3,     /* max_k sum_j |W_kj| would overflow int32 Delta */
    DABS_E_NOMEM = 4,     /* device allocation failed */
    DABS_E_CUDA = 5,      /* CUDA runtime / kernel error */
    DABS_E_COMM = 6,      /* the exchange hook reported an error */
    DABS_E_STATE = 7      /* call out of order (e.g. dabs_generation before dabs_reset) */
} dabs_status;

typedef struct dabs_ctx dabs_ctx;

/* Exchange hook (Sec. IV-B island ring across GPUs, R-23):
 * an all-gather of `bytes` bytes from every rank, in rank order, on the given
 * CUDA stream: recv_dev[r*bytes .. (r+1)*bytes) = rank r's send_dev.  Both
 * buffers are device memory owned by the library.  Return 0 on success.
 * The Python binding implements it with torch.distributed (NCCL). */
typedef int (*dabs_exchange_fn)(void* user, const void* send_dev, void* recv_dev, size_t bytes,
                                void* cuda_stream);

/* Optional device allocator hook (e.g. torch's caching allocator). */
typedef void* (*dabs_alloc_fn)(void* user, size_t bytes, void* cuda_stream);
typedef void (*dabs_free_fn)(void* user, void* ptr, void* cuda_stream);

typedef struct {
    uint32_t struct_size;     /* sizeof(dabs_config) */
    uint32_t s_milli;         /* search flip factor s x 1000 (R-13); default 100 */
    uint32_t b_milli;         /* batch flip factor b x 1000; default 1000 */
    uint32_t tabu_period;     /* P:487-489; default 8; <= 31 */
    uint32_t pool_capacity;   /* P:703; default 100 */
    uint32_t eps_ppm;         /* exploration probability; default 50000 = 5% */
    uint32_t genop_mask;      /* enabled genetic operations, bit g (P:174 order); default 0xFF.
                                 Bit 8 = mutation after crossover, the ABS solver's only
                                 operation (R-27): genop_mask = 0x100 with
                                 algo_mask = 0x2 (CyclicMin) is the ABS ablation mode */
    uint32_t algo_mask;       /* enabled main algorithms, bit a (P:169 order); default 0x1F */
    uint32_t pools_per_gpu;   /* solution pools on this rank; default 1 */
    uint32_t slots_per_pool;  /* concurrent searches per pool; 0 = auto (fill the GPU) */
    int64_t target_energy;    /* dabs_run stops once best <= target; INT64_MIN = none */
    uint64_t time_limit_ns;   /* dabs_run wall-clock limit; 0 = none */
    int32_t rank, world;      /* this rank and the number of ranks (one per GPU) */
    int32_t device;           /* CUDA device ordinal; -1 = current */
    void* cuda_stream;        /* cudaStream_t to run on; NULL = a private stream */
    dabs_exchange_fn exchange;/* required when world > 1 */
    dabs_alloc_fn alloc;      /* NULL = cudaMalloc */
    dabs_free_fn free;
    void* user;               /* passed to the hooks */
    uint32_t restart_gens;    /* restart-on-merge (R-28): after this many
                                 generations without a box-wide improvement, pools and
                                 slots start afresh (the best is kept); 0 = off (default) */
    uint32_t flags;           /* DABS_FLAG_ONE_WAVE: slots_per_pool = 0 sizes ONE wave of
                                 co-resident searches (the persistent CTAs of
                                 dabs_run_async) instead of four waves per generation */
} dabs_config;

#define DABS_FLAG_ONE_WAVE 1u
/* Jump-start batches (R-30): in every generation each
 * slot starts its batch AT its target D (X = D, E(D) and Delta(D) from one
 * exact int8 tensor-core contraction (tcgen05) of W's bytes against all
 * targets) instead of walking there with Straight's flips.  A method variant
 * (fewer flips per batch, no scans along the Straight path).  Generation
 * schedule only; needs 2 n_pad^2 + 128 ceil(slots/128) n_pad bytes more device
 * memory. */
#define DABS_FLAG_JUMP_START 2u

/* Fills the defaults listed above. */
void dabs_config_default(dabs_config* cfg);

/* Create a solver for W (host, row-major n x n int16, upper triangular
 * including the diagonal, E(X) = sum_{i<=j} W_ij x_i x_j).  Only i <= j is
 * read for the model; any nonzero below the diagonal -> DABS_E_TRIANGLE.
 * 1 <= n <= 65536 else DABS_E_ARG (n <= 2048: one warp per search; n <=
 * 16384: one CTA; n <= 32768: one 256-thread CTA with Delta in tensor memory,
 * two per SM; n > 32768: one 512-thread CTA per SM with Delta in all of its
 * tensor memory, or a cluster of two CTAs with DABS_TMEM64=0).  T = ceil(s n) > 65536
 * or B = ceil(b n) > 2^30 -> DABS_E_ARG (the exact MaxMin span and the
 * flip counters are sized for those).  eps_ppm = 1000000 means "always
 * uniform" (R-15).  If max_k (|W_kk| +
 * sum_{j!=k} |W_jk|) >= 2^31 - 1 -> DABS_E_RANGE (Delta is int32; reachable
 * only at n = 65536 with weights of -32768).  Uploads W, lays it out as
 * symmetric int16 rows with zero diagonal, allocates slots
 * and pools.  *out receives the context (NULL on failure). */
dabs_status dabs_create(const int16_t* W_host, int32_t n, const dabs_config* cfg, dabs_ctx** out);

/* Same, from a sparse upper triangle in CSR form (host arrays, caller-owned,
 * copied): row i's off-diagonal coefficients W_ij, j > i, are
 * val[row_ptr[i] .. row_ptr[i+1]) at columns col[...] (strictly increasing,
 * each > i; zero values allowed), diag[i] = W_ii.  A column <= its row ->
 * DABS_E_TRIANGLE; a column out of range, a non-increasing row, a bad row_ptr
 * -> DABS_E_ARG; the same int32 range check as dabs_create -> DABS_E_RANGE.
 * The device keeps the same symmetric dense rows. */
dabs_status dabs_create_csr(int32_t n, const int32_t* row_ptr, const int32_t* col, const int16_t* val,
                            const int16_t* diag, const dabs_config* cfg, dabs_ctx** out);

/* Reset to the start of a run: slots X=0, E=0, Delta_k=W_kk,
 * empty tabu rings; pools = random +inf sentinels drawn from `seed`
 * (R-19); generation 0. */
dabs_status dabs_reset(dabs_ctx* ctx, uint64_t seed);

/* One generation (R-25): GA seeding of every slot, one batch
 * search per slot, pool merge (R-18), then the exchange
 * (world > 1) and the box-wide best / flip count.  Requires dabs_reset. */
dabs_status dabs_generation(dabs_ctx* ctx);

/* dabs_reset(seed), then generations until the box-wide total of flips
 * >= flip_budget, best <= target_energy, or the time limit.  Writes the best
 * vector found (n bytes, host) and its energy.  SPMD: every rank calls it
 * with identical arguments. */
dabs_status dabs_run(dabs_ctx* ctx, uint64_t seed, uint64_t flip_budget, uint8_t* best_x_host,
                     int64_t* best_e);

/* Asynchronous schedule (reading R-29; the paper's
 * packet flow without a generation barrier).
 * dabs_reset(seed); packet 0 of every slot is seeded from the fresh pools;
 * then ONE persistent kernel, one CTA per slot, runs batch after batch: after
 * batch k a slot takes its pool's lock, merges its result into its pool
 * (R-18 with one newcomer, seq = (event+1)<<32 | slot), updates the run best,
 * appends (slot | seeded<<31) to the event log and, unless the run is
 * stopping, seeds packet k+1 (Philox generation field = k+1) from its pool as
 * it is.  An Xrossover packet whose partner (local pool (p+1) mod P, live) is
 * another pool is completed by a second event (XREAD) under the partner's
 * lock, after the own lock is released: no lock is held while waiting.  The
 * run stops seeding once the merged flips >= flip_budget, best <=
 * target_energy, or the time limit has passed (device clock); every slot then
 * merges its running batch and exits.  Deterministic given the log: the CPU
 * oracle replays it (orc_world_async_replay).  Slots are persistent CTAs, so
 * create the context with flags = DABS_FLAG_ONE_WAVE (slots beyond the
 * resident capacity start only after the stop).  Every tier (on the cluster
 * tier the cluster's rank-0 CTA commits).  Requires world == 1,
 * restart_gens == 0, tracing off and no jump-start, else DABS_E_ARG.
 * Writes the best vector (n bytes, host) and energy; dabs_get_stats then
 * reports the run (generations = events, time_to_best_ns from the
 * kernel's start on the device clock, batch_ms_last = the kernel's time). */
dabs_status dabs_run_async(dabs_ctx* ctx, uint64_t seed, uint64_t flip_budget, uint8_t* best_x_host,
                           int64_t* best_e);

/* The last dabs_run_async's event log, in event order: a merge is local slot
 * | (1<<31 if a next packet was seeded); an XREAD is local slot | (1<<30).
 * Copies min(cap, kept) entries to `log` (host, caller-owned; may be NULL);
 * *len = the number of events.  The device keeps the first
 * max(2^20, 64 * slots) events; a longer run is not cut short, but its log
 * is truncated and this call then returns DABS_E_STATE (after copying). */
dabs_status dabs_async_log(const dabs_ctx* ctx, uint32_t* log, int64_t cap, int64_t* len);

/* Device time (CUDA events, ms) of the last generation's jump-start step
 * (target expansion, the two GEMMs, Delta/E assembly); 0 without the flag. */
dabs_status dabs_jump_ms(const dabs_ctx* ctx, float* ms);

/* The last dabs_run_async's pool-lock profile (device clock): the sum over
 * merge events of the time spent waiting for the lock and holding it. */
dabs_status dabs_async_lock_ns(const dabs_ctx* ctx, uint64_t* wait_ns, uint64_t* hold_ns);

/* Best vector and energy seen so far (box-wide after the last exchange). */
dabs_status dabs_best(const dabs_ctx* ctx, uint8_t* best_x_host, int64_t* best_e);

/* Direct evaluation of Eq.(2) on the device for one host vector (n bytes). */
dabs_status dabs_energy(const dabs_ctx* ctx, const uint8_t* x_host, int64_t* e);

typedef struct {
    uint64_t total_flips;        /* box-wide flips since reset (every executed flip) */
    uint64_t local_flips;        /* this rank's flips since reset */
    uint64_t generations;
    uint64_t wall_ns;            /* host wall time inside dabs_generation since reset */
    uint64_t time_to_best_ns;    /* wall time from reset to the generation that found best */
    float batch_ms_last;         /* device time of the last batch launch (CUDA events) */
    float ga_ms_last, merge_ms_last;
    int64_t best_energy;
    int32_t best_algo, best_genop;   /* first-best record */
    int32_t best_generation, best_slot;
    uint64_t dispatch[5][9];     /* [algorithm][genop] packets issued (Table V) */
    uint64_t inserted[5][9];     /* [algorithm][genop] results that entered a pool */
    uint64_t restarts;           /* restart-on-merge events since reset */
    int32_t n, n_pad, threads_per_search, slots, pools, T, B;
    int32_t cap;
    uint64_t kernel_launches;    /* kernels of this library launched by the context since create
                                    (library GEMMs not counted) */
} dabs_stats;

dabs_status dabs_get_stats(const dabs_ctx* ctx, dabs_stats* out);

/* ---- parity hooks (used by the tests against the CPU oracle) ---- */

/* Run ONE batch search on the device for local slot `slot` from the given
 * state (host: x n bytes, delta n int32, E, ring[32] most-recent-first, -1 =
 * empty), target D (n bytes) and algorithm, with the Philox stream of
 * (seed, global slot id, gen).  Writes the updated state back into the same
 * host arrays, the batch's BEST/E(BEST)/flips, and (if trace_cap > 0) the
 * per-flip trace (bit, E after the flip, phase: 0 Straight, 1 Greedy, 2+r main
 * round r).  Uses the production kernel for this n (traced instantiation). */
dabs_status dabs_debug_batch(dabs_ctx* ctx, uint32_t slot, uint8_t* x, int32_t* delta, int64_t* E,
                             int32_t* ring, const uint8_t* D, int32_t algo, uint64_t seed,
                             uint32_t gen, uint8_t* best, int64_t* ebest, int64_t* flips,
                             int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase, int64_t trace_cap);

/* Read local slot / pool / packet state (host outputs, layouts as above).
 * pool == pools_per_gpu reads the successor snapshot used by Xrossover. */
dabs_status dabs_read_slot(const dabs_ctx* ctx, uint32_t slot, uint8_t* x, int32_t* delta,
                           int64_t* E, int32_t* ring);
dabs_status dabs_read_pool(const dabs_ctx* ctx, uint32_t pool, uint8_t* X /* cap*n */,
                           int64_t* E, uint64_t* seq, uint8_t* algo, uint8_t* genop);
dabs_status dabs_read_packet(const dabs_ctx* ctx, uint32_t slot, uint8_t* D, int32_t* algo,
                             int32_t* genop, uint8_t* best, int64_t* ebest, int64_t* flips);
dabs_status dabs_read_stats_pool(const dabs_ctx* ctx, uint32_t pool, uint64_t* dispatch /*5*9*/,
                                 uint64_t* inserted /*5*9*/);

/* Enable per-flip tracing of one local slot in production generations
 * (trace_cap flips per batch; -1 slot disables).  Read after a generation. */
dabs_status dabs_trace_enable(dabs_ctx* ctx, int32_t slot, int64_t trace_cap);
dabs_status dabs_trace_read(const dabs_ctx* ctx, int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase,
                            int64_t* count);

/* ---- measurement probe (bench.py's roofline denominators) ----
 * The achievable W-row stream bandwidth of this GPU: `ctas_per_sm` CTAs per
 * SM copy random rows of a device buffer of rows x row_bytes bytes into
 * shared memory with TMA bulk copies (4 pieces per row, `inflight` rows in
 * flight per CTA, no compute), `iters` rows each; *gbps = bytes / event time.
 * A buffer that fits L2 gives the L2 row-stream peak.  device < 0: the current
 * device.  row_bytes must be a multiple of 64 and inflight*row_bytes <= 200 KiB,
 * inflight in {1, 2}, else DABS_E_ARG; the buffer is allocated and freed here. */
dabs_status dabs_probe_row_stream(int32_t device, int64_t rows, int32_t row_bytes, int32_t ctas_per_sm,
                                  int32_t inflight, int32_t iters, double* gbps);

const char* dabs_last_error(void);
void dabs_destroy(dabs_ctx* ctx);   /* NULL-safe */

#ifdef __cplusplus
}
#endif
#endif /* DABS_H */
