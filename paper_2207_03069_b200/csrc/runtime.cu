// runtime.cu -- the C ABI (include/dabs.h) over the sm_100a kernels.
//
// One context = one rank (one GPU): W, the slots (persistent searches), the
// packets, P solution pools + the Xrossover successor snapshot, statistics,
// and the exchange buffers.  A generation is GA seed -> batch -> merge ->
// pack -> (exchange) -> import, all on one stream (R-25, R-26).
// Citations: P:n = PAPER.md line n; R-x = DESIGN.md readings.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/dabs.h"
#include "batch_kernel.cuh"
#include "tmem_kernel.cuh"
#include "tmw_kernel.cuh"
#include "ga_pool_kernels.cuh"
#include "async_kernel.cuh"
#include "tmem_async.cuh"
#include "jump_tc.cuh"
#include "probe.cuh"

using namespace dabs;

// NVTX ranges around the C-ABI calls and the generation phases (header-only
// nvtx3: no-ops unless a profiler injects itself)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_err;

static dabs_status fail(dabs_status st, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(DABS_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,                \
                        cudaGetErrorString(e_));                                              \
    } while (0)

struct dabs_ctx {
    dabs_config cfg;
    int dev = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // problem and tiling
    int n = 0, n_pad = 0, nwp = 0, C = 0, NT = 0;
    int CL = 1;              // CTAs per search (2 = cluster tier)
    bool mw = false;
    bool tm = false;         // TMEM tier (tm_batch_kernel): two 256-thread searches per SM, Delta in TMEM
    int tmNT = 256;          // its threads per search: 256 (n <= 32768) or 512 (n > 32768, DABS_TMEM64=1)
    bool tma = false;        // the asynchronous schedule on the TMEM tier (tm_async_kernel)
    bool tmw = false;        // TMEM warp tier (tmw_batch_kernel): 4 warp-searches per CTA, Delta in TMEM
    int T = 0, B = 0, tabu = 8, cap = 100, P = 1, S = 1, slots = 1;
    GaConst ga{};
    // device buffers
    std::vector<void*> allocs;
    int16_t* W = nullptr;
    int32_t* diag = nullptr;
    int32_t* rmax = nullptr;
    int32_t *wtab = nullptr, *ptab = nullptr;
    uint64_t* mtab = nullptr;   // MaxMin: floor(2^64 (T-t)^3 / T^3) per step t (R-6; TMEM tier)
    uint32_t* X = nullptr;
    int32_t* delta = nullptr;
    int64_t* E = nullptr;
    int32_t* ring = nullptr;
    uint32_t* D = nullptr;
    uint8_t *palgo = nullptr, *pgenop = nullptr;
    uint32_t* best = nullptr;
    int64_t *ebest = nullptr, *flips = nullptr;
    int32_t* order = nullptr;             // batch launch order (longest first)
    PoolView* pools_d = nullptr;          // [P+1]
    std::vector<PoolView> pools_h;        // host copy of the views
    MergeArgs margs{};
    unsigned long long* dispatch = nullptr;
    unsigned long long* inserted = nullptr;
    unsigned long long* flip_total = nullptr;   // this rank, cumulative
    unsigned long long* scratch64 = nullptr;    // energy / checks
    uint8_t* xbytes = nullptr;                  // energy input
    PayloadLayout L{};
    uint8_t *send = nullptr, *recv = nullptr;
    // trace
    int trace_slot = -1;
    int64_t trace_cap = 0;
    int32_t* tr_bit = nullptr;
    int64_t* tr_E = nullptr;
    int8_t* tr_phase = nullptr;
    // run state (host)
    bool ready = false;
    uint64_t seed = 0;
    uint32_t gen = 0;
    uint64_t total_flips = 0, local_flips = 0;
    uint32_t stall = 0;          // generations without a box-wide improvement (R-28)
    uint64_t restarts = 0;
    int64_t best_E = E_INF;
    std::vector<uint8_t> best_X;
    int32_t rec[4] = {-1, -1, -1, -1};
    uint64_t wall_ns = 0, ttb_ns = 0;
    float batch_ms = 0, ga_ms = 0, merge_ms = 0;
    cudaEvent_t ev[6] = {};
    // asynchronous schedule
    uint32_t* a_lock = nullptr;      // tickets [P*32], serving [P*32], evcount, stop, best lock (own lines)
    uint64_t* a_hash = nullptr;      // [P][cap]
    uint64_t a_wait_ns = 0, a_hold_ns = 0;
    uint64_t launches = 0;           // kernels of this library launched since create (dabs_stats)
    // the generation as one CUDA graph (single rank, no tracing): captured once,
    // replayed every generation; kernels read the generation index from gen_d
    cudaGraphExec_t gexec = nullptr;
    uint32_t* gen_d = nullptr;
    Summary* sums_h = nullptr;       // pinned: the summaries the graph copies out
    uint32_t* gen_h = nullptr;       // pinned: the generation index copied in before a replay
    uint64_t graph_launches = 0;     // kernels per replay
    bool no_graph = false;
    // jump-start
    bool jump = false;
    int8_t* jBhi = nullptr;          // W bytes, tiled for the tcgen05 kernel (jump_tc.cuh)
    uint8_t *jBlo = nullptr, *jA = nullptr;
    unsigned long long* je2 = nullptr;   // 2 E(D) per slot
    int jMT = 0;                     // 128-slot tiles
    float jump_ms = 0;   // last async run: summed pool-lock wait / hold (device clock)
    uint32_t* a_log = nullptr;
    uint32_t a_log_cap = 0;
    unsigned long long* a_u64 = nullptr;   // flips_cum, t0, best_t
    int64_t* a_bestE = nullptr;
    uint32_t* a_bestX = nullptr;
    int32_t* a_brec = nullptr;
    std::vector<uint32_t> a_log_h;
    uint32_t a_events = 0;           // events of the last async run (the log keeps the first a_log_cap)
    std::chrono::steady_clock::time_point t_reset;
};

template <typename Tp>
static dabs_status dalloc(dabs_ctx* c, Tp** p, size_t count)
{
    size_t bytes = count * sizeof(Tp);
    if (bytes == 0) bytes = 16;
    void* q = nullptr;
    if (c->cfg.alloc) {
        q = c->cfg.alloc(c->cfg.user, bytes, c->stream);
        if (!q) return fail(DABS_E_NOMEM, "alloc hook failed for %zu bytes", bytes);
    } else {
        cudaError_t e = cudaMalloc(&q, bytes);
        if (e != cudaSuccess) return fail(DABS_E_NOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    }
    c->allocs.push_back(q);
    *p = reinterpret_cast<Tp*>(q);
    return DABS_OK;
}

#define AL(ptr, count)                                         \
    do {                                                       \
        dabs_status st_ = dalloc(c, &(ptr), (size_t)(count));  \
        if (st_ != DABS_OK) return st_;                        \
    } while (0)

extern "C" void dabs_config_default(dabs_config* cfg)
{
    if (!cfg) return;
    memset(cfg, 0, sizeof *cfg);
    cfg->struct_size = sizeof *cfg;
    cfg->s_milli = 100;
    cfg->b_milli = 1000;
    cfg->tabu_period = 8;
    cfg->pool_capacity = 100;
    cfg->eps_ppm = 50000;
    cfg->genop_mask = 0xFF;
    cfg->algo_mask = 0x1F;
    cfg->pools_per_gpu = 1;
    cfg->slots_per_pool = 0;
    cfg->target_energy = INT64_MIN;
    cfg->time_limit_ns = 0;
    cfg->rank = 0;
    cfg->world = 1;
    cfg->device = -1;
}

extern "C" const char* dabs_last_error(void) { return g_err.c_str(); }

#ifdef DABS_TIMING
// diagnostic build only: read (and clear) the batch kernel's cycle buckets
extern "C" int dabs_timing_read(unsigned long long* out)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_tstat, sizeof(g_tstat));
    cudaMemcpyFromSymbol(out + 30, g_tstat2, sizeof(g_tstat2));
    cudaMemcpyFromSymbol(out + 40, g_tstat3, sizeof(g_tstat3));
    static const unsigned long long zero[30] = {};
    cudaMemcpyToSymbol(g_tstat2, zero, sizeof(g_tstat2));
    cudaMemcpyToSymbol(g_tstat3, zero, sizeof(g_tstat3));
    return (int)cudaMemcpyToSymbol(g_tstat, zero, sizeof(g_tstat));
}
#endif

static int flip_factor(uint32_t milli, int n)
{
    const int64_t v = ((int64_t)milli * n + 999) / 1000;
    return v < 1 ? 1 : (int)v;
}

// ---------------------------------------------------------------- kernels by tier
using BatchFn = void (*)(const BatchParams);

static BatchFn pick_batch(int C, int NT, int CL, bool trace)
{
    if (CL == 2) {
        switch (NT) {
        case 64: return trace ? batch_kernel<8, 64, 2, true> : batch_kernel<8, 64, 2, false>;
        case 128: return trace ? batch_kernel<8, 128, 2, true> : batch_kernel<8, 128, 2, false>;
        case 256: return trace ? batch_kernel<8, 256, 2, true> : batch_kernel<8, 256, 2, false>;
        default: return trace ? batch_kernel<8, 512, 2, true> : batch_kernel<8, 512, 2, false>;
        }
    }
    if (NT > 32) {
        switch (NT) {
        case 64: return trace ? batch_kernel<8, 64, 1, true> : batch_kernel<8, 64, 1, false>;
        case 128: return trace ? batch_kernel<8, 128, 1, true> : batch_kernel<8, 128, 1, false>;
        case 256: return trace ? batch_kernel<8, 256, 1, true> : batch_kernel<8, 256, 1, false>;
        default: return trace ? batch_kernel<8, 512, 1, true> : batch_kernel<8, 512, 1, false>;
        }
    }
    switch (C) {
    case 1: return trace ? batch_kernel<1, 32, 1, true> : batch_kernel<1, 32, 1, false>;
    case 2: return trace ? batch_kernel<2, 32, 1, true> : batch_kernel<2, 32, 1, false>;
    case 4: return trace ? batch_kernel<4, 32, 1, true> : batch_kernel<4, 32, 1, false>;
    default: return trace ? batch_kernel<8, 32, 1, true> : batch_kernel<8, 32, 1, false>;
    }
}
static BatchFn pick_batch(const dabs_ctx* c, bool trace)
{
    if (c->tm) {
        if (c->tmNT == 512) return trace ? tm_batch_kernel<512, true> : tm_batch_kernel<512, false>;
        return trace ? tm_batch_kernel<256, true> : tm_batch_kernel<256, false>;
    }
    if (c->tmw) {
        if (c->C == 8) return trace ? tmw_batch_kernel<8, true> : tmw_batch_kernel<8, false>;
        return trace ? tmw_batch_kernel<4, true> : tmw_batch_kernel<4, false>;
    }
    return pick_batch(c->C, c->NT, c->CL, trace);
}
// threads per CTA of the generation schedule's batch kernel
static int batch_threads(const dabs_ctx* c) { return c->tm ? c->tmNT : c->tmw ? 32 * TMW_SPC : c->NT; }
// searches per CTA of the generation schedule's batch kernel
static int batch_spc(const dabs_ctx* c) { return c->tmw ? TMW_SPC : 1; }

using AsyncFn = void (*)(const AsyncArgs);
static AsyncFn pick_async(int C, int NT, int CL, bool tm = false)
{
    if (tm) return NT == 512 ? tm_async_kernel<512> : tm_async_kernel<256>;
    if (CL == 2) {
        switch (NT) {
        case 64: return async_kernel<8, 64, 2>;
        case 128: return async_kernel<8, 128, 2>;
        case 256: return async_kernel<8, 256, 2>;
        default: return async_kernel<8, 512, 2>;
        }
    }
    switch (NT) {
    case 32: return C == 1 ? async_kernel<1, 32, 1> : C == 2 ? async_kernel<2, 32, 1> : C == 4 ? async_kernel<4, 32, 1>
                                                                                       : async_kernel<8, 32, 1>;
    case 64: return async_kernel<8, 64, 1>;
    case 128: return async_kernel<8, 128, 1>;
    case 256: return async_kernel<8, 256, 1>;
    default: return async_kernel<8, 512, 1>;
    }
}

// per CTA: its part of one W row + tabu counts (+ two copies of the sigma bytes, CTA tiers)
static size_t row_smem_reg(const dabs_ctx* c)
{
    return (size_t)(c->mw ? 5 : 3) * (c->n_pad / c->CL);
}
// the generation schedule's batch kernel: the TMEM tier keeps only the W row in dynamic smem
static size_t row_smem(const dabs_ctx* c)
{
    return c->tm ? tm_dyn_smem(c->n_pad, c->tmNT) : c->tmw ? (size_t)2 * c->n_pad * TMW_SPC : row_smem_reg(c);
}
// the asynchronous schedule's persistent kernel, its threads and dynamic smem
// (the row buffer doubles as the commit's scratch)
static AsyncFn async_fn(const dabs_ctx* c) { return pick_async(c->C, c->tma ? c->tmNT : c->NT, c->CL, c->tma); }
static int async_threads(const dabs_ctx* c) { return c->tma ? c->tmNT : c->NT; }
static size_t async_smem(const dabs_ctx* c, int cap)
{
    return std::max(c->tma ? tm_dyn_smem(c->n_pad, c->tmNT) : row_smem_reg(c), async_commit_smem(cap));
}

static BatchParams batch_params(dabs_ctx* c, uint64_t seed, uint32_t gen, int slot0)
{
    BatchParams p{};
    p.W = c->W; p.wtab = c->wtab; p.ptab = c->ptab; p.rmax = c->rmax;
    p.invT3 = 1.0 / ((double)c->T * (double)c->T * (double)c->T);
    p.mtab = c->mtab;
    p.n = c->n; p.n_pad = c->n_pad; p.nwp = c->nwp;
    p.T = c->T; p.B = c->B; p.tabu = c->tabu;
    p.seed = seed; p.gen = gen;
    p.slot_base = (uint32_t)(c->cfg.rank * c->slots);
    p.slot0 = slot0;
    p.count = 0;
    p.X = c->X; p.delta = c->delta; p.E = c->E; p.ring = c->ring;
    p.D = c->D; p.algo = c->palgo;
    p.best = c->best; p.ebest = c->ebest; p.flips = c->flips;
    p.flip_total = c->flip_total;
    p.trace_slot = c->trace_slot; p.tr_bit = c->tr_bit; p.tr_E = c->tr_E; p.tr_phase = c->tr_phase;
    p.tr_cap = c->trace_cap;
    return p;
}

// ---------------------------------------------------------------- create
static void dabs_destroy_impl(dabs_ctx* c);

// configuration, device, stream, tiling and GA constants common to both ingest paths
static dabs_status create_begin(int32_t n, const dabs_config* cfg_in, dabs_ctx** out)
{
    if (!out) return fail(DABS_E_ARG, "out is NULL");
    *out = nullptr;
    if (n < 1 || n > 65536) return fail(DABS_E_ARG, "n=%d outside [1, 65536]", n);
    dabs_config cfg;
    dabs_config_default(&cfg);
    if (cfg_in) {
        if (cfg_in->struct_size != sizeof(dabs_config)) return fail(DABS_E_ARG, "dabs_config.struct_size mismatch");
        cfg = *cfg_in;
    }
    if (cfg.tabu_period > 31) return fail(DABS_E_ARG, "tabu_period > 31");
    if (cfg.pool_capacity < 1 || cfg.pool_capacity > 1024) return fail(DABS_E_ARG, "pool_capacity outside [1,1024]");
    if (cfg.s_milli < 1 || cfg.b_milli < 1) return fail(DABS_E_ARG, "s and b must be positive");
    {
        // MaxMin's span (R-6) takes u^3 and T^3 in 64-bit words and divides
        // through muldiv_floor, exact for T^3 <= 2^48: T = ceil(s n) <= 65536.
        // B must fit the int flip counters of a batch.
        const int64_t T = ((int64_t)cfg.s_milli * n + 999) / 1000, B = ((int64_t)cfg.b_milli * n + 999) / 1000;
        if (T > 65536) return fail(DABS_E_ARG, "T = ceil(s n) = %lld > 65536", (long long)T);
        if (B > (int64_t)1 << 30) return fail(DABS_E_ARG, "B = ceil(b n) = %lld > 2^30", (long long)B);
    }
    if ((cfg.genop_mask & 0x1FF) == 0 || (cfg.algo_mask & 0x1F) == 0) return fail(DABS_E_ARG, "empty genop/algo mask");
    if (cfg.eps_ppm > 1000000) return fail(DABS_E_ARG, "eps_ppm > 1e6");
    if (cfg.world < 1 || cfg.rank < 0 || cfg.rank >= cfg.world) return fail(DABS_E_ARG, "bad rank/world");
    if (cfg.world > 1 && !cfg.exchange) return fail(DABS_E_ARG, "world > 1 needs an exchange hook");
    if (cfg.pools_per_gpu < 1) return fail(DABS_E_ARG, "pools_per_gpu < 1");

    dabs_ctx* c = new dabs_ctx();
    c->cfg = cfg;
    auto bail = [&](dabs_status st) {
        dabs_destroy_impl(c);
        return st;
    };
    int ndev = 0;
    cudaError_t e0 = cudaGetDeviceCount(&ndev);
    if (e0 != cudaSuccess || ndev == 0) {
        fail(DABS_E_CUDA, "no CUDA device: %s", cudaGetErrorString(e0));
        return bail(DABS_E_CUDA);
    }
    c->dev = cfg.device >= 0 ? cfg.device : 0;
    if (cfg.device < 0) cudaGetDevice(&c->dev);
    if (cudaSetDevice(c->dev) != cudaSuccess) {
        fail(DABS_E_CUDA, "cudaSetDevice(%d) failed", c->dev);
        return bail(DABS_E_CUDA);
    }
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, c->dev);
    if (prop.major != 10) {
        fail(DABS_E_CUDA, "device %d is sm_%d%d; this library is built for sm_100a only", c->dev, prop.major, prop.minor);
        return bail(DABS_E_CUDA);
    }
    if (cfg.cuda_stream) {
        c->stream = (cudaStream_t)cfg.cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            fail(DABS_E_CUDA, "stream create failed");
            return bail(DABS_E_CUDA);
        }
        c->own_stream = true;
    }
    for (auto& e : c->ev) cudaEventCreate(&e);

    // ---- tiling: warp per search for n <= 2048, else a CTA
    c->n = n;
    if (n <= 2048) {
        c->mw = false;
        c->NT = 32;
        int C = 1;
        while (C * 256 < n) C <<= 1;
        c->C = C;
        // 512 < n <= 2048, DABS_TMW=1 (A/B, off by default): the TMEM warp tier,
        // 32 searches per SM with Delta in TMEM.  Measured break-even at K2000s
        // (7.34e8 vs 7.41e8 flips/s: MaxMin/PositiveMin +13/+25 %, RandomMin
        // -9 %) and -19 % at TSP32 (tools/gpu_tmw.sh; DESIGN 9)
        const char* ew = getenv("DABS_TMW");
        c->tmw = C >= 4 && ew && ew[0] == '1';
    } else {
        // one CTA of NT threads x 64 elements (n <= 32768), else a cluster of
        // two such CTAs (n <= 65536).  DABS_CLUSTER=1 forces the
        // cluster tier for every n > 4096 (A/B measurements).
        c->mw = true;
        c->C = 8;
        const char* ev = getenv("DABS_CLUSTER");
        const char* e64 = getenv("DABS_TMEM64");
        // n > 32768: one 512-thread CTA per SM with all of Delta (256 KB) in the SM's
        // tensor memory (R64K 0.371 -> 0.661 of HBM against the cluster tier,
        // tools/gpu_tm64.sh); DABS_TMEM64=0 or DABS_CLUSTER=1: the 2-CTA cluster tier
        const bool tm64 = n > 32768 && !(e64 && e64[0] == '0') && !(ev && ev[0] == '1');
        c->CL = ((n > 32768 && !tm64) || (ev && ev[0] == '1' && n > 4096)) ? 2 : 1;
        int NT = 64;
        while (NT * 64 * c->CL < n) NT <<= 1;
        c->NT = NT;
        // 16384 < n <= 32768: the TMEM tier for the generation schedule (DABS_TMEM=0: the
        // 512-thread register tier, A/B).  The asynchronous schedule follows (tm_async_kernel).
        const char* et = getenv("DABS_TMEM");
        c->tm = c->CL == 1 && NT == 512 && !(et && et[0] == '0');
        if (tm64) {
            c->tm = true;
            c->tmNT = 512;
            c->NT = 512;
            c->C = 16;                    // 512 threads x 128 elements: n_pad = 65536
        }
    }
    c->n_pad = c->NT * c->CL * c->C * 8;
    c->nwp = c->n_pad / 32;
    for (int tr = 0; tr < 2; tr++) {
        cudaError_t e = cudaFuncSetAttribute(pick_batch(c, tr != 0),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem(c));
        // TMEM tier: the full shared-memory carveout, so two searches fit per SM
        // (and the occupancy query below sees them)
        if (e == cudaSuccess && (c->tm || c->tmw))
            e = cudaFuncSetAttribute(pick_batch(c, tr != 0), cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return bail(fail(DABS_E_CUDA, "smem attribute: %s", cudaGetErrorString(e)));
    }
    {
        // the asynchronous schedule follows the tier (DABS_TMEM_ASYNC=0: the register tier at R32K)
        const char* eta = getenv("DABS_TMEM_ASYNC");
        c->tma = c->tm && !(eta && eta[0] == '0');
        cudaError_t e = cudaFuncSetAttribute(async_fn(c), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)async_smem(c, (int)cfg.pool_capacity));
        if (e == cudaSuccess && c->tma)
            e = cudaFuncSetAttribute(async_fn(c), cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return bail(fail(DABS_E_CUDA, "smem attribute: %s", cudaGetErrorString(e)));
    }
    c->T = flip_factor(cfg.s_milli, n);
    c->B = flip_factor(cfg.b_milli, n);
    c->tabu = (int)cfg.tabu_period;
    c->cap = (int)cfg.pool_capacity;
    c->P = (int)cfg.pools_per_gpu;
    if (cfg.slots_per_pool) {
        c->S = (int)cfg.slots_per_pool;
    } else {
        int occ = 0;
        const bool one_wave = (cfg.flags & DABS_FLAG_ONE_WAVE) != 0;
        if (one_wave)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, async_fn(c), async_threads(c),
                                                          async_smem(c, (int)cfg.pool_capacity));
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pick_batch(c, false), batch_threads(c), row_smem(c));
        if (getenv("DABS_DEBUG_OCC")) fprintf(stderr, "dabs: occupancy %d CTAs/SM (tier NT=%d C=%d CL=%d tm=%d)\n", occ,
                                             batch_threads(c), c->C, c->CL, (int)c->tm);
        // the TMEM tier is built for two co-resident searches per SM (ncu: 16
        // active warps per SM); the occupancy query reports one for it
        if (c->tm && c->tmNT == 256 && !one_wave && occ < 2) occ = 2;
        if (c->tma && c->tmNT == 256 && one_wave && occ < 2) occ = 2;    // the same two co-resident searches per SM
        if (c->tmw && !one_wave && occ < 8) occ = 8;   // 8 CTAs x 4 searches: the TMEM columns and 64 registers
        if (occ < 1) occ = 1;
        // concurrent searches (the TMEM warp tier packs 4 per CTA)
        const int conc = std::max(1, prop.multiProcessorCount * occ * (one_wave ? 1 : batch_spc(c)) / c->CL);
        if (one_wave)
            c->S = std::max(1, conc / c->P);    // persistent CTAs of the asynchronous schedule, all resident
        else {
            // several waves per generation: batch lengths differ (TwoNeighbor runs
            // 2n-1 main flips), more waves let the block scheduler balance them.
            // Four waves for the register tiers: more waves shorten the last wave's idle tail by only
            // 1-3 % at a fixed algorithm (tools/waves_fixed_algo.py); the larger
            // flips/s changes seen with more slots per generation come from the
            // adaptive algorithm mix, not from the kernels (DESIGN 5)
            // The TMEM tier (two searches per SM, long R32K batches) loses more to
            // the last wave's tail: 4 -> 8 -> 16 waves measured 0.661 -> 0.686 ->
            // 0.718 of the HBM roofline with the adaptive mix and +6-8 % for every
            // fixed rule (tools/gpu_waves.sh), at ~2.3 s per generation.
            // The warp tier keeps four: 16 waves measured K2000s +17 %, TSP32 +5 %,
            // GS800 +9 % flips/s but 54 ms generations at TSP32 (the pools, and
            // the time to target, move once per generation; tools/gpu_ab_warp.sh).
            // DABS_WAVES overrides (A/B).
            const char* ewv = getenv("DABS_WAVES");
            const int waves = ewv ? std::max(1, atoi(ewv)) : (c->tm ? 16 : 4);
            c->S = (waves * conc + c->P - 1) / c->P;
        }
    }
    c->slots = c->P * c->S;
    if ((int64_t)c->slots * (cfg.world) >= (1ll << 31)) return bail(fail(DABS_E_ARG, "too many slots"));

    // ---- GA constants
    GaConst& g = c->ga;
    g.n = n; g.nwp = c->nwp; g.cap = c->cap; g.P = c->P; g.S = c->S;
    g.eps_thr = ((uint64_t)cfg.eps_ppm << 32) / 1000000u;
    g.n_gen = 0; g.n_alg = 0;
    for (int k = 0; k < N_GEN; k++) if (cfg.genop_mask >> k & 1) g.gens[g.n_gen++] = k;
    for (int k = 0; k < N_ALG; k++) if (cfg.algo_mask >> k & 1) g.algs[g.n_alg++] = k;
    *out = c;
    return DABS_OK;
}

// a1 (dense): upload the host triangle, check it, build symmetric rows
static dabs_status ingest_dense(dabs_ctx* c, const int16_t* W_host)
{
    const int n = c->n;
    auto bail = [&](dabs_status st) { return st; };
    int16_t* U = nullptr;
    dabs_status st;
    if ((st = dalloc(c, &U, (size_t)n * n)) != DABS_OK) return bail(st);
    if ((st = dalloc(c, &c->scratch64, 4)) != DABS_OK) return bail(st);
    if (cudaMemcpyAsync(U, W_host, sizeof(int16_t) * (size_t)n * n, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->scratch64, 0, 32, c->stream) != cudaSuccess)
        return bail(fail(DABS_E_CUDA, "upload of W failed"));
    check_kernel<<<n, 256, 0, c->stream>>>(U, n, c->scratch64);
    c->launches++;
    unsigned long long flags[2];
    if (cudaMemcpyAsync(flags, c->scratch64, 16, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
        return bail(fail(DABS_E_CUDA, "check kernel failed: %s", cudaGetErrorString(cudaGetLastError())));
    if (flags[0]) return bail(fail(DABS_E_TRIANGLE, "W has a nonzero entry below the diagonal"));
    if (flags[1] >= (unsigned long long)INT32_MAX)
        return bail(fail(DABS_E_RANGE, "max_k sum_j |W_kj| = %llu does not fit int32 Delta", flags[1]));
    if ((st = dalloc(c, &c->W, (size_t)n * c->n_pad)) != DABS_OK) return bail(st);
    if ((st = dalloc(c, &c->diag, c->n_pad)) != DABS_OK) return bail(st);
    if (cudaMemsetAsync(c->W, 0, sizeof(int16_t) * (size_t)n * c->n_pad, c->stream) != cudaSuccess)
        return bail(fail(DABS_E_CUDA, "memset W"));
    {
        dim3 grid((c->n_pad + 31) / 32, (n + 31) / 32), blk(32, 8);
        symmetrize_kernel<<<grid, blk, 0, c->stream>>>(U, n, c->n_pad, c->W, c->diag);
        c->launches++;
    }
    if ((st = dalloc(c, &c->rmax, n)) != DABS_OK) return bail(st);
    rowmax_kernel<<<n, 256, 0, c->stream>>>(c->W, n, c->n_pad, c->rmax);
    c->launches++;
    if (cudaStreamSynchronize(c->stream) != cudaSuccess)
        return bail(fail(DABS_E_CUDA, "symmetrize: %s", cudaGetErrorString(cudaGetLastError())));
    // free the staging copy
    for (auto it = c->allocs.begin(); it != c->allocs.end(); ++it)
        if (*it == U) {
            if (c->cfg.free) c->cfg.free(c->cfg.user, U, c->stream); else cudaFree(U);
            c->allocs.erase(it);
            break;
        }

    return DABS_OK;
}

// tables, slots, packets, pools, exchange buffers
static dabs_status create_end(dabs_ctx* c)
{
    const int n = c->n;
    const dabs_config& cfg = c->cfg;
    dabs_status st;
    auto bail = [&](dabs_status st2) { return st2; };
    // ---- schedule tables for CyclicMin (R-7) and RandomMin (R-8)
    {
        std::vector<int32_t> wt(c->T + 1), pt(c->T + 1);
        std::vector<uint64_t> mt(c->T + 1);
        const unsigned __int128 T3 = (unsigned __int128)c->T * c->T * c->T;
        for (int t = 0; t <= c->T; t++) {
            const unsigned __int128 u = (unsigned __int128)(c->T - t);
            mt[t] = t == 0 ? ~0ull : (uint64_t)(((u * u * u) << 64) / T3);   // u^3 < T^3: below 2^64
            const unsigned __int128 t3 = (unsigned __int128)t * t * t;
            uint64_t w = (uint64_t)(((unsigned __int128)n * t3 + T3 - 1) / T3);
            const uint64_t cmin = n < 32 ? (uint64_t)n : 32u;
            if (w < cmin) w = cmin;
            if (w > (uint64_t)n) w = n;
            wt[t] = (int32_t)w;
            uint64_t p = (uint64_t)(((unsigned __int128)65536u * t3) / T3);
            const uint64_t pf = 2097152u / (uint32_t)n;
            if (p < pf) p = pf;
            if (p > 65536u) p = 65536u;
            pt[t] = (int32_t)p;
        }
        if ((st = dalloc(c, &c->wtab, c->T + 1)) != DABS_OK) return bail(st);
        if ((st = dalloc(c, &c->ptab, c->T + 1)) != DABS_OK) return bail(st);
        cudaMemcpyAsync(c->wtab, wt.data(), 4 * wt.size(), cudaMemcpyHostToDevice, c->stream);
        cudaMemcpyAsync(c->ptab, pt.data(), 4 * pt.size(), cudaMemcpyHostToDevice, c->stream);
        if ((st = dalloc(c, &c->mtab, c->T + 1)) != DABS_OK) return bail(st);
        cudaMemcpyAsync(c->mtab, mt.data(), 8 * mt.size(), cudaMemcpyHostToDevice, c->stream);
        if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(fail(DABS_E_CUDA, "tables"));
    }

    // ---- slots, packets, pools
    const size_t ns = c->slots, nwp = c->nwp, cap = c->cap, P = c->P;
#define AB(ptr, count) if ((st = dalloc(c, &(ptr), (count))) != DABS_OK) return bail(st)
    AB(c->X, ns * nwp); AB(c->delta, ns * c->n_pad); AB(c->E, ns); AB(c->ring, ns * TABU_RING);
    AB(c->D, ns * nwp); AB(c->palgo, ns); AB(c->pgenop, ns);
    AB(c->best, ns * nwp); AB(c->ebest, ns); AB(c->flips, ns); AB(c->order, ns);
    AB(c->dispatch, P * N_ALG * N_GEN); AB(c->inserted, P * N_ALG * N_GEN);
    AB(c->flip_total, 1); AB(c->xbytes, (size_t)n);
    c->pools_h.resize(P + 1);
    for (size_t q = 0; q <= P; q++) {
        PoolView& v = c->pools_h[q];
        AB(v.X, cap * nwp); AB(v.E, cap); AB(v.seq, cap); AB(v.algo, cap); AB(v.genop, cap);
    }
    AB(c->pools_d, P + 1);
    cudaMemcpyAsync(c->pools_d, c->pools_h.data(), sizeof(PoolView) * (P + 1), cudaMemcpyHostToDevice, c->stream);
    MergeArgs& m = c->margs;
    m.pools = c->pools_d; m.best = c->best; m.ebest = c->ebest; m.palgo = c->palgo; m.pgenop = c->pgenop;
    AB(m.order, ns); AB(m.acc, P * cap); AB(m.sX, P * cap * nwp); AB(m.sE, P * cap); AB(m.sSeq, P * cap);
    AB(m.sAlgo, P * cap); AB(m.sGenop, P * cap); AB(m.mcount, P); AB(m.hq, P * ns); AB(m.hold, P * cap); AB(m.dupf, P * ns);
    m.inserted = c->inserted;
    m.slot_base = (uint32_t)(cfg.rank * c->slots);
    m.S = c->S; m.cap = c->cap; m.nwp = c->nwp;
    // payload layout (8-byte aligned fields)
    {
        PayloadLayout& L = c->L;
        size_t o = 0;
        auto al8 = [](size_t v) { return (v + 7) & ~(size_t)7; };
        L.oX = o; o = al8(o + 4 * cap * nwp);
        L.oE = o; o = al8(o + 8 * cap);
        L.oSeq = o; o = al8(o + 8 * cap);
        L.oAlgo = o; o = al8(o + cap);
        L.oGenop = o; o = al8(o + cap);
        L.oSum = o; o = al8(o + sizeof(Summary));
        L.oBestX = o; o = al8(o + 4 * nwp);
        L.bytes = o;
    }
    AB(c->a_lock, 64 * P + 96); AB(c->a_hash, P * cap); AB(c->a_u64, 13); AB(c->a_bestE, 1); AB(c->a_bestX, nwp); AB(c->a_brec, 4);
    c->a_log_cap = (uint32_t)std::max<size_t>(1u << 20, 64 * ns);
    AB(c->a_log, c->a_log_cap);
    if (cfg.flags & DABS_FLAG_JUMP_START) {
        c->jump = true;
        const size_t np = (size_t)c->n_pad;
        c->jMT = (ns + JT_M - 1) / JT_M;
        AB(c->jBhi, np * np); AB(c->jBlo, np * np); AB(c->jA, (size_t)c->jMT * JT_M * np); AB(c->je2, ns);
        CK(cudaMemsetAsync(c->je2, 0, 8 * (size_t)ns, c->stream));
        jt_tile_w_kernel<<<8 * 148, 256, 0, c->stream>>>(c->W, n, c->n_pad, c->jBhi, c->jBlo);
        c->launches++;
        CK(cudaFuncSetAttribute(jt_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)JT_SMEM));
    }
    AB(c->send, c->L.bytes);
    AB(c->recv, c->L.bytes * (size_t)cfg.world);
    AB(c->gen_d, 1);
    if (cudaMallocHost(&c->sums_h, sizeof(Summary) * (size_t)cfg.world) != cudaSuccess ||
        cudaMallocHost(&c->gen_h, 4) != cudaSuccess)
        return bail(fail(DABS_E_NOMEM, "pinned summaries"));
#undef AB
    c->best_X.assign(n, 0);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(fail(DABS_E_CUDA, "create: %s", cudaGetErrorString(cudaGetLastError())));
    return DABS_OK;
}

extern "C" dabs_status dabs_create(const int16_t* W_host, int32_t n, const dabs_config* cfg_in,
                                   dabs_ctx** out)
{
    NvtxRange nr_("dabs_create");
    if (!out) return fail(DABS_E_ARG, "out is NULL");
    *out = nullptr;
    if (!W_host) return fail(DABS_E_ARG, "W is NULL");
    dabs_ctx* c = nullptr;
    dabs_status st = create_begin(n, cfg_in, &c);
    if (st != DABS_OK) return st;
    if ((st = ingest_dense(c, W_host)) != DABS_OK || (st = create_end(c)) != DABS_OK) {
        const std::string msg = g_err;
        dabs_destroy_impl(c);
        g_err = msg;
        return st;
    }
    *out = c;
    return DABS_OK;
}

// a1 (CSR): validate the host upper-triangle CSR, upload it, scatter into the
// same symmetric dense rows (the per-flip scan is O(n) whatever the storage)
extern "C" dabs_status dabs_create_csr(int32_t n, const int32_t* row_ptr, const int32_t* col, const int16_t* val,
                                       const int16_t* diag, const dabs_config* cfg_in, dabs_ctx** out)
{
    NvtxRange nr_("dabs_create_csr");
    if (!out) return fail(DABS_E_ARG, "out is NULL");
    *out = nullptr;
    if (!row_ptr || !diag) return fail(DABS_E_ARG, "row_ptr / diag is NULL");
    if (n < 1 || n > 65536) return fail(DABS_E_ARG, "n=%d outside [1, 65536]", n);
    if (row_ptr[0] != 0) return fail(DABS_E_ARG, "row_ptr[0] != 0");
    const int64_t nnz = row_ptr[n];
    if (nnz < 0 || nnz > (int64_t)n * (n - 1) / 2) return fail(DABS_E_ARG, "bad nnz %lld", (long long)nnz);
    if (nnz > 0 && (!col || !val)) return fail(DABS_E_ARG, "col / val is NULL");
    std::vector<int64_t> absum(n, 0);
    for (int i = 0; i < n; i++) {
        if (row_ptr[i + 1] < row_ptr[i]) return fail(DABS_E_ARG, "row_ptr not monotone at row %d", i);
        absum[i] += diag[i] < 0 ? -(int64_t)diag[i] : diag[i];
        for (int32_t e = row_ptr[i]; e < row_ptr[i + 1]; e++) {
            const int32_t j = col[e];
            if (j >= n || j < 0) return fail(DABS_E_ARG, "column %d out of range in row %d", j, i);
            if (j <= i) return fail(DABS_E_TRIANGLE, "entry (%d,%d) is not strictly above the diagonal", i, j);
            if (e > row_ptr[i] && j <= col[e - 1]) return fail(DABS_E_ARG, "row %d columns not strictly increasing", i);
            const int64_t a = val[e] < 0 ? -(int64_t)val[e] : val[e];
            absum[i] += a;
            absum[j] += a;
        }
    }
    for (int i = 0; i < n; i++)
        if (absum[i] >= INT32_MAX) return fail(DABS_E_RANGE, "row %d: sum |W| does not fit int32 Delta", i);
    dabs_ctx* c = nullptr;
    dabs_status st = create_begin(n, cfg_in, &c);
    if (st != DABS_OK) return st;
    auto fin = [&](dabs_status s2) {
        const std::string msg = g_err;
        dabs_destroy_impl(c);
        g_err = msg;
        return s2;
    };
    int32_t *d_rp = nullptr, *d_col = nullptr;
    int16_t *d_val = nullptr, *d_diag = nullptr;
    if ((st = dalloc(c, &d_rp, n + 1)) != DABS_OK || (st = dalloc(c, &d_col, nnz)) != DABS_OK ||
        (st = dalloc(c, &d_val, nnz)) != DABS_OK || (st = dalloc(c, &d_diag, n)) != DABS_OK ||
        (st = dalloc(c, &c->W, (size_t)n * c->n_pad)) != DABS_OK || (st = dalloc(c, &c->diag, c->n_pad)) != DABS_OK ||
        (st = dalloc(c, &c->scratch64, 4)) != DABS_OK || (st = dalloc(c, &c->rmax, n)) != DABS_OK)
        return fin(st);
    cudaStream_t s0 = c->stream;
    if (cudaMemcpyAsync(d_rp, row_ptr, 4 * (size_t)(n + 1), cudaMemcpyHostToDevice, s0) != cudaSuccess ||
        (nnz && cudaMemcpyAsync(d_col, col, 4 * (size_t)nnz, cudaMemcpyHostToDevice, s0) != cudaSuccess) ||
        (nnz && cudaMemcpyAsync(d_val, val, 2 * (size_t)nnz, cudaMemcpyHostToDevice, s0) != cudaSuccess) ||
        cudaMemcpyAsync(d_diag, diag, 2 * (size_t)n, cudaMemcpyHostToDevice, s0) != cudaSuccess ||
        cudaMemsetAsync(c->W, 0, sizeof(int16_t) * (size_t)n * c->n_pad, s0) != cudaSuccess)
        return fin(fail(DABS_E_CUDA, "CSR upload failed"));
    csr_scatter_kernel<<<n, 128, 0, s0>>>(d_rp, d_col, d_val, d_diag, n, c->n_pad, c->W, c->diag);
    c->launches++;
    rowmax_kernel<<<n, 256, 0, s0>>>(c->W, n, c->n_pad, c->rmax);
    c->launches++;
    if (cudaStreamSynchronize(s0) != cudaSuccess)
        return fin(fail(DABS_E_CUDA, "CSR scatter: %s", cudaGetErrorString(cudaGetLastError())));
    if ((st = create_end(c)) != DABS_OK) return fin(st);
    *out = c;
    return DABS_OK;
}

static void dabs_destroy_impl(dabs_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->dev);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (void* q : c->allocs) {
        if (c->cfg.free) c->cfg.free(c->cfg.user, q, c->stream); else cudaFree(q);
    }
    for (auto& e : c->ev) if (e) cudaEventDestroy(e);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->sums_h) cudaFreeHost(c->sums_h);
    if (c->gen_h) cudaFreeHost(c->gen_h);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

extern "C" void dabs_destroy(dabs_ctx* c) { dabs_destroy_impl(c); }

// ---------------------------------------------------------------- reset / generation
extern "C" dabs_status dabs_reset(dabs_ctx* c, uint64_t seed)
{
    if (!c) return fail(DABS_E_ARG, "ctx is NULL");
    CK(cudaSetDevice(c->dev));
    c->seed = seed;
    c->ga.seed = seed;
    c->gen = 0;
    init_slots_kernel<<<c->slots, 256, 0, c->stream>>>(c->slots, c->n_pad, c->nwp, c->diag, c->X, c->delta,
                                                       c->E, c->ring);
    c->launches++;
    const uint32_t gid0 = (uint32_t)(c->cfg.rank * c->P);
    const uint32_t nbr_gid = (uint32_t)(((c->cfg.rank + 1) * c->P) % (c->cfg.world * c->P));
    init_pools_kernel<<<dim3(c->P + 1, c->cap), 128, 0, c->stream>>>(c->ga, c->pools_d, gid0, nbr_gid, 0u);
    c->launches++;
    c->stall = 0;
    c->restarts = 0;
    CK(cudaMemsetAsync(c->dispatch, 0, 8 * c->P * N_ALG * N_GEN, c->stream));
    CK(cudaMemsetAsync(c->inserted, 0, 8 * c->P * N_ALG * N_GEN, c->stream));
    CK(cudaMemsetAsync(c->flip_total, 0, 8, c->stream));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    c->total_flips = 0;
    c->local_flips = 0;
    c->best_E = E_INF;
    std::fill(c->best_X.begin(), c->best_X.end(), 0);
    c->rec[0] = c->rec[1] = c->rec[2] = c->rec[3] = -1;
    c->wall_ns = 0;
    c->ttb_ns = 0;
    c->t_reset = std::chrono::steady_clock::now();
    c->ready = true;
    return DABS_OK;
}

static dabs_status launch_batch(dabs_ctx* c, uint64_t seed, uint32_t gen, int slot0, int count, bool trace,
                                const int32_t* order = nullptr, const uint32_t* gen_ptr = nullptr)
{
    BatchParams p = batch_params(c, seed, gen, slot0);
    p.order = order;
    p.gen_ptr = gen_ptr;
    p.count = count;
    BatchFn fn = pick_batch(c, trace);
    if (c->CL == 1) {
        const int spc = batch_spc(c);
        fn<<<(count + spc - 1) / spc, batch_threads(c), row_smem(c), c->stream>>>(p);
        c->launches++;
    } else {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)(count * c->CL));
        lc.blockDim = dim3((unsigned)c->NT);
        lc.dynamicSmemBytes = row_smem(c);
        lc.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)c->CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        CK(cudaLaunchKernelEx(&lc, fn, p));
        c->launches++;
    }
    CK(cudaGetLastError());
    return DABS_OK;
}

// jump-start (R-30): X = D, E(D), Delta(D) for every slot from C = D . W on the
// tensor cores (jump_tc.cuh: tcgen05.mma kind::i8, epilogue writes Delta)
static dabs_status jump_start(dabs_ctx* c)
{
    cudaStream_t st = c->stream;
    const int np = c->n_pad, KT = np / JT_K, NTL = np / JT_N;
    jt_tile_d_kernel<<<c->jMT * KT, 256, 0, st>>>(c->D, c->slots, c->nwp, np, c->jA);
    c->launches++;
    jt_gemm_kernel<<<c->jMT * NTL, 128, JT_SMEM, st>>>(c->jA, c->jBhi, c->jBlo, c->D, c->diag, c->n, np, c->nwp,
                                                       c->slots, c->jMT, c->delta, c->je2);
    c->launches++;
    CK(cudaGetLastError());
    jt_finish_kernel<<<c->slots, 256, 0, st>>>(c->D, c->slots, c->nwp, c->X, c->je2, c->E);
    c->launches++;
    CK(cudaGetLastError());
    return DABS_OK;
}

// Enqueue one generation (a3 GA seeding, a4-a7 batches, a8 merge, a9 exchange)
// on the library's stream; graph = captured for replay (kernels read the
// generation index from gen_d, copied in before every replay).
static dabs_status enqueue_generation(dabs_ctx* c, bool graph)
{
    NvtxRange nr_("dabs.enqueue_generation");
    cudaStream_t st = c->stream;
    const uint32_t* genp = graph ? c->gen_d : nullptr;
    // inside a capture a plain event record only orders streams; the timing
    // events must be external records to become nodes of the graph
    const unsigned evf = graph ? cudaEventRecordExternal : cudaEventRecordDefault;
    // a3: GA seeding
    CK(cudaEventRecordWithFlags(c->ev[0], st, evf));
    ga_seed_kernel<<<(c->slots + 7) / 8, 256, 0, st>>>(c->ga, c->pools_d, (uint32_t)(c->cfg.rank * c->slots),
                                                        c->gen, c->slots, c->D, c->palgo, c->pgenop,
                                                        c->dispatch, genp);
    c->launches++;
    CK(cudaGetLastError());
    if (c->jump) {
        // jump-start (R-30): X = D, Delta(D), E(D) for every slot from one GEMM pair
        CK(cudaEventRecordWithFlags(c->ev[4], st, evf));
        dabs_status sj = jump_start(c);
        if (sj != DABS_OK) return sj;
        CK(cudaEventRecordWithFlags(c->ev[5], st, evf));
    }
    CK(cudaEventRecordWithFlags(c->ev[1], st, evf));
    // a4-a7: one batch search per slot (the hot loop)
    order_kernel<<<1, 256, 0, st>>>(c->palgo, c->slots, c->order);
    c->launches++;
    CK(cudaGetLastError());
    dabs_status s1 = launch_batch(c, c->seed, c->gen, 0, c->slots, c->trace_slot >= 0, c->order, genp);
    if (s1 != DABS_OK) return s1;
    CK(cudaEventRecordWithFlags(c->ev[2], st, evf));
    // a8: pool merge
    c->margs.gen = c->gen;
    c->margs.gen_ptr = genp;
    CK(cudaMemsetAsync(c->margs.mcount, 0, 4 * (size_t)c->P, st));
    merge_rank_kernel<<<dim3((c->S + 7) / 8, c->P), 256, 0, st>>>(c->margs);
    c->launches++;
    merge_hash_kernel<<<dim3((c->S + c->cap + 7) / 8, c->P), 256, 0, st>>>(c->margs);
    c->launches++;
    merge_dup_kernel<<<dim3((c->S + 7) / 8, c->P), 256, 0, st>>>(c->margs);
    c->launches++;
    pool_merge_kernel<<<c->P, 1024, 0, st>>>(c->margs);
    c->launches++;
    CK(cudaGetLastError());
    CK(cudaEventRecordWithFlags(c->ev[3], st, evf));
    // a9: exchange
    pack_payload_kernel<<<1, 256, 0, st>>>(c->pools_d, c->P, c->cap, c->nwp, (uint32_t)(c->cfg.rank * c->P),
                                           c->flip_total, c->send, c->L);
    c->launches++;
    CK(cudaGetLastError());
    const uint8_t* gathered = c->send;
    if (c->cfg.world > 1) {
        const int rc = c->cfg.exchange(c->cfg.user, c->send, c->recv, c->L.bytes, st);
        if (rc != 0) return fail(DABS_E_COMM, "exchange hook returned %d", rc);
        gathered = c->recv;
    }
    const int succ_rank = (c->cfg.rank + 1) % c->cfg.world;
    import_snapshot_kernel<<<8, 256, 0, st>>>(gathered + (size_t)succ_rank * c->L.bytes, c->pools_h[c->P],
                                              c->cap, c->nwp, c->L);
    c->launches++;
    CK(cudaGetLastError());
    // summaries of all ranks to the host (pinned)
    for (int r = 0; r < c->cfg.world; r++)
        CK(cudaMemcpyAsync(&c->sums_h[r], gathered + (size_t)r * c->L.bytes + c->L.oSum, sizeof(Summary),
                           cudaMemcpyDeviceToHost, st));
    return DABS_OK;
}

extern "C" dabs_status dabs_generation(dabs_ctx* c)
{
    if (!c) return fail(DABS_E_ARG, "ctx is NULL");
    if (!c->ready) return fail(DABS_E_STATE, "dabs_generation before dabs_reset");
    NvtxRange nr_("dabs_generation");
    CK(cudaSetDevice(c->dev));
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t st = c->stream;
    // one CUDA graph per context (single rank, no tracing: the exchange hook and
    // the traced kernel stay on plain launches); DABS_NO_GRAPH=1 disables it
    const bool use_graph = c->cfg.world == 1 && c->trace_slot < 0 && !c->no_graph && !getenv("DABS_NO_GRAPH");
    if (use_graph) {
        if (!c->gexec) {
            const uint64_t l0 = c->launches;
            cudaGraph_t g = nullptr;
            if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
                cudaGetLastError();            // e.g. the legacy default stream: plain launches
                c->no_graph = true;
                return dabs_generation(c);
            }
            const dabs_status se = enqueue_generation(c, true);
            const cudaError_t ce = cudaStreamEndCapture(st, &g);
            if (se != DABS_OK) return se;
            if (ce != cudaSuccess) return fail(DABS_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
            const cudaError_t ie = cudaGraphInstantiate(&c->gexec, g, 0);
            cudaGraphDestroy(g);
            if (ie != cudaSuccess) return fail(DABS_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ie));
            c->graph_launches = c->launches - l0;
            c->launches = l0;
        }
        *c->gen_h = c->gen;
        CK(cudaMemcpyAsync(c->gen_d, c->gen_h, 4, cudaMemcpyHostToDevice, st));
        CK(cudaGraphLaunch(c->gexec, st));
        c->launches += c->graph_launches;
    } else {
        const dabs_status se = enqueue_generation(c, false);
        if (se != DABS_OK) return se;
    }
    const uint8_t* gathered = c->cfg.world > 1 ? c->recv : c->send;
    const Summary* sums = c->sums_h;
    CK(cudaStreamSynchronize(st));
    CK(cudaEventElapsedTime(&c->ga_ms, c->ev[0], c->ev[1]));
    if (c->jump) {
        CK(cudaEventElapsedTime(&c->jump_ms, c->ev[4], c->ev[5]));
        if (getenv("DABS_JUMP_TIMING")) fprintf(stderr, "jump-start (tcgen05 contraction + finish): %.3f ms\n", c->jump_ms);
    }
    CK(cudaEventElapsedTime(&c->batch_ms, c->ev[1], c->ev[2]));
    CK(cudaEventElapsedTime(&c->merge_ms, c->ev[2], c->ev[3]));
    uint64_t tot = 0;
    int br = 0;
    for (int r = 0; r < c->cfg.world; r++) {
        tot += sums[r].flips;
        if (sums[r].bestE < sums[br].bestE) br = r;
    }
    c->total_flips = tot;
    c->local_flips = sums[c->cfg.rank].flips;
    const auto t1 = std::chrono::steady_clock::now();
    c->wall_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    if (sums[br].bestE < c->best_E) {
        c->best_E = sums[br].bestE;
        std::vector<uint32_t> words(c->nwp);
        CK(cudaMemcpy(words.data(), gathered + (size_t)br * c->L.bytes + c->L.oBestX, 4 * c->nwp,
                      cudaMemcpyDeviceToHost));
        for (int k = 0; k < c->n; k++) c->best_X[k] = (uint8_t)((words[k >> 5] >> (k & 31)) & 1u);
        c->rec[0] = sums[br].algo;
        c->rec[1] = sums[br].genop;
        c->rec[2] = (int32_t)((sums[br].bestSeq >> 32) - 1);
        c->rec[3] = (int32_t)(sums[br].bestSeq & 0xFFFFFFFFu);
        c->ttb_ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - c->t_reset).count();
        c->stall = 0;
    } else {
        c->stall++;
    }
    c->gen++;
    // restart-on-merge (R-28): the decision uses gathered data only,
    // so every rank restarts in the same generation; the run's best is kept
    if (c->cfg.restart_gens && c->stall >= c->cfg.restart_gens) {
        init_slots_kernel<<<c->slots, 256, 0, st>>>(c->slots, c->n_pad, c->nwp, c->diag, c->X, c->delta, c->E,
                                                    c->ring);
        c->launches++;
        const uint32_t gid0 = (uint32_t)(c->cfg.rank * c->P);
        const uint32_t nbr_gid = (uint32_t)(((c->cfg.rank + 1) * c->P) % (c->cfg.world * c->P));
        init_pools_kernel<<<dim3(c->P + 1, c->cap), 128, 0, st>>>(c->ga, c->pools_d, gid0, nbr_gid, c->gen);
        c->launches++;
        CK(cudaGetLastError());
        c->stall = 0;
        c->restarts++;
    }
    return DABS_OK;
}

extern "C" dabs_status dabs_run(dabs_ctx* c, uint64_t seed, uint64_t flip_budget, uint8_t* best_x,
                                int64_t* best_e)
{
    NvtxRange nr_("dabs_run");
    dabs_status st = dabs_reset(c, seed);
    if (st != DABS_OK) return st;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        st = dabs_generation(c);
        if (st != DABS_OK) return st;
        if (c->total_flips >= flip_budget) break;
        if (c->cfg.target_energy != INT64_MIN && c->best_E <= c->cfg.target_energy) break;
        if (c->cfg.time_limit_ns) {
            const auto ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
            if ((uint64_t)ns >= c->cfg.time_limit_ns) break;
        }
    }
    return dabs_best(c, best_x, best_e);
}

// Asynchronous schedule: one persistent kernel, no
// generation barrier, every merge logged for the oracle's replay.
extern "C" dabs_status dabs_run_async(dabs_ctx* c, uint64_t seed, uint64_t flip_budget, uint8_t* best_x,
                                      int64_t* best_e)
{
    NvtxRange nr_("dabs_run_async");
    if (!c) return fail(DABS_E_ARG, "ctx is NULL");
    if (c->cfg.world != 1) return fail(DABS_E_ARG, "the asynchronous schedule runs on one rank (world == 1)");
    if (c->cfg.restart_gens) return fail(DABS_E_ARG, "restart-on-merge is a generation-schedule option");
    if (c->trace_slot >= 0) return fail(DABS_E_ARG, "tracing is a generation-schedule option");
    if (c->jump) return fail(DABS_E_ARG, "jump-start is a generation-schedule option");
    dabs_status st = dabs_reset(c, seed);
    if (st != DABS_OK) return st;
    const auto t0 = std::chrono::steady_clock::now();   // the stream is idle (dabs_reset synchronised)
    cudaStream_t s0 = c->stream;
    int32_t* ord = c->margs.acc;   // [P][cap] scratch, free outside the generation schedule's merge
    CK(cudaMemsetAsync(c->a_lock, 0, 4 * (64 * (size_t)c->P + 96), s0));
    CK(cudaMemsetAsync(c->a_u64, 0, 104, s0));
    CK(cudaMemsetAsync(c->a_brec, 0xFF, 16, s0));
    const int64_t inf = E_INF;
    CK(cudaMemcpyAsync(c->a_bestE, &inf, 8, cudaMemcpyHostToDevice, s0));
    // the device clock origin t0 is stamped here, before the seeding, so the
    // time to best below spans the same work as the generation schedule's
    async_init_kernel<<<4, 256, 0, s0>>>(ord, c->a_hash, c->P, c->cap, c->a_u64 + 1);
    c->launches++;
    CK(cudaGetLastError());
    // packet 0 of every slot from the fresh pools
    ga_seed_kernel<<<(c->slots + 7) / 8, 256, 0, s0>>>(c->ga, c->pools_d, 0u, 0u, c->slots, c->D, c->palgo,
                                                        c->pgenop, c->dispatch, nullptr);
    c->launches++;
    CK(cudaGetLastError());
    AsyncArgs a{};
    a.bp = batch_params(c, c->seed, 0u, 0);
    a.g = c->ga;
    a.pools = c->pools_d;
    a.ord = ord;
    a.hash = c->a_hash;
    a.D = c->D; a.palgo = c->palgo; a.pgenop = c->pgenop;
    a.dispatch = c->dispatch; a.inserted = c->inserted;
    a.ticket = c->a_lock; a.serving = c->a_lock + 32 * c->P; a.evcount = c->a_lock + 64 * c->P;
    a.stop = (int32_t*)(c->a_lock + 64 * c->P + 32); a.best_lock = (int32_t*)(c->a_lock + 64 * c->P + 64);
    a.log = c->a_log; a.log_cap = c->a_log_cap; a.slots = c->slots;
    a.flips_cum = c->a_u64; a.t0 = c->a_u64 + 1; a.best_t = c->a_u64 + 2; a.lock_ns = c->a_u64 + 3;
    a.budget = flip_budget;
    a.target = c->cfg.target_energy;
    a.time_limit_ns = c->cfg.time_limit_ns;
    a.bestE = c->a_bestE; a.bestX = c->a_bestX; a.brec = c->a_brec;
    a.profile = getenv("DABS_ASYNC_PHASES") ? 1 : 0;
    CK(cudaEventRecord(c->ev[1], s0));
    const size_t asmem = async_smem(c, c->cap);
    if (c->CL == 1) {
        async_fn(c)<<<c->slots, async_threads(c), asmem, s0>>>(a);
        c->launches++;
    } else {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)(c->slots * c->CL));
        lc.blockDim = dim3((unsigned)c->NT);
        lc.dynamicSmemBytes = asmem;
        lc.stream = s0;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)c->CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        CK(cudaLaunchKernelEx(&lc, pick_async(c->C, c->NT, c->CL), a));
        c->launches++;
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev[2], s0));
    async_compact_kernel<<<c->P, 256, 0, s0>>>(c->pools_d, ord, c->cap, c->nwp, c->margs.sX, c->margs.sE,
                                                c->margs.sSeq, c->margs.sAlgo, c->margs.sGenop);
    c->launches++;
    CK(cudaGetLastError());
    uint32_t nev = 0;
    unsigned long long u64[13];
    int64_t bE = E_INF;
    int32_t rec[4];
    std::vector<uint32_t> words(c->nwp);
    CK(cudaMemcpyAsync(&nev, c->a_lock + 64 * c->P, 4, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(u64, c->a_u64, 104, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(&bE, c->a_bestE, 8, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(rec, c->a_brec, 16, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(words.data(), c->a_bestX, 4 * c->nwp, cudaMemcpyDeviceToHost, s0));
    CK(cudaStreamSynchronize(s0));
    CK(cudaEventElapsedTime(&c->batch_ms, c->ev[1], c->ev[2]));
    c->a_events = nev;
    c->a_log_h.resize(std::min(nev, c->a_log_cap));
    if (!c->a_log_h.empty())
        CK(cudaMemcpy(c->a_log_h.data(), c->a_log, 4 * c->a_log_h.size(), cudaMemcpyDeviceToHost));
    const auto t1 = std::chrono::steady_clock::now();
    c->wall_ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    c->total_flips = c->local_flips = u64[0];
    c->gen = nev;
    c->best_E = bE;
    for (int k = 0; k < c->n; k++) c->best_X[k] = (uint8_t)((words[k >> 5] >> (k & 31)) & 1u);
    for (int j = 0; j < 4; j++) c->rec[j] = rec[j];
    // time to best from dabs_reset, like the generation schedule's host wall
    // clock: (host time from reset to this call's first launch) + (device clock
    // from the first kernel's start to the improving merge); the host-to-device
    // launch gap between the two (a few us) is the only part not counted
    const uint64_t pre_ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t0 - c->t_reset).count();
    c->ttb_ns = pre_ns + (u64[2] > u64[1] ? u64[2] - u64[1] : 0);
    c->a_wait_ns = u64[3];
    c->a_hold_ns = u64[4];
    if (getenv("DABS_ASYNC_PHASES"))
        fprintf(stderr, "async lock phases (us/event): A %.2f B %.2f dup+ins %.2f GA %.2f release %.2f\n",
                u64[5] / 1e3 / std::max(1u, nev), u64[6] / 1e3 / std::max(1u, nev), u64[7] / 1e3 / std::max(1u, nev),
                u64[8] / 1e3 / std::max(1u, nev), u64[9] / 1e3 / std::max(1u, nev));
    if (getenv("DABS_ASYNC_PHASES"))
        fprintf(stderr, "async CTA time: batches %.3f, commits %.3f of lifetime; mean lifetime %.3f ms (kernel %.3f ms)\n",
                (double)u64[10] / std::max(1ull, u64[11]), (double)u64[12] / std::max(1ull, u64[11]),
                u64[11] / 1e6 / c->slots, (double)c->batch_ms);
    return dabs_best(c, best_x, best_e);
}

extern "C" dabs_status dabs_jump_ms(const dabs_ctx* c, float* ms)
{
    if (!c || !ms) return fail(DABS_E_ARG, "NULL argument");
    *ms = c->jump ? c->jump_ms : 0.0f;
    return DABS_OK;
}

extern "C" dabs_status dabs_async_lock_ns(const dabs_ctx* c, uint64_t* wait_ns, uint64_t* hold_ns)
{
    if (!c || !wait_ns || !hold_ns) return fail(DABS_E_ARG, "NULL argument");
    *wait_ns = c->a_wait_ns;
    *hold_ns = c->a_hold_ns;
    return DABS_OK;
}

extern "C" dabs_status dabs_async_log(const dabs_ctx* c, uint32_t* log, int64_t cap, int64_t* len)
{
    if (!c || !len) return fail(DABS_E_ARG, "NULL argument");
    const int64_t m = (int64_t)c->a_log_h.size();
    *len = (int64_t)c->a_events;
    if (log && cap > 0) memcpy(log, c->a_log_h.data(), 4 * (size_t)std::min(cap, m));
    if ((int64_t)c->a_events > m)
        return fail(DABS_E_STATE, "async log truncated: %lld of %u events kept (a replay needs the whole log)",
                    (long long)m, c->a_events);
    return DABS_OK;
}

extern "C" dabs_status dabs_best(const dabs_ctx* c, uint8_t* best_x, int64_t* best_e)
{
    if (!c) return fail(DABS_E_ARG, "ctx is NULL");
    if (best_x) memcpy(best_x, c->best_X.data(), c->n);
    if (best_e) *best_e = c->best_E;
    return DABS_OK;
}

extern "C" dabs_status dabs_energy(const dabs_ctx* cc, const uint8_t* x, int64_t* e)
{
    dabs_ctx* c = const_cast<dabs_ctx*>(cc);
    if (!c || !x || !e) return fail(DABS_E_ARG, "NULL argument");
    CK(cudaSetDevice(c->dev));
    CK(cudaMemcpyAsync(c->xbytes, x, c->n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->scratch64, 0, 8, c->stream));
    energy_kernel<<<c->n, 256, 0, c->stream>>>(c->W, c->diag, c->n, c->n_pad, c->xbytes, (long long*)c->scratch64);
    const_cast<dabs_ctx*>(c)->launches++;
    CK(cudaGetLastError());
    long long v = 0;
    CK(cudaMemcpyAsync(&v, c->scratch64, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *e = v;
    return DABS_OK;
}

extern "C" dabs_status dabs_get_stats(const dabs_ctx* c, dabs_stats* o)
{
    if (!c || !o) return fail(DABS_E_ARG, "NULL argument");
    memset(o, 0, sizeof *o);
    o->total_flips = c->total_flips;
    o->local_flips = c->local_flips;
    o->generations = c->gen;
    o->wall_ns = c->wall_ns;
    o->time_to_best_ns = c->ttb_ns;
    o->batch_ms_last = c->batch_ms;
    o->ga_ms_last = c->ga_ms;
    o->merge_ms_last = c->merge_ms;
    o->best_energy = c->best_E;
    o->restarts = c->restarts;
    o->best_algo = c->rec[0]; o->best_genop = c->rec[1]; o->best_generation = c->rec[2]; o->best_slot = c->rec[3];
    std::vector<unsigned long long> d(c->P * N_ALG * N_GEN), in(c->P * N_ALG * N_GEN);
    if (cudaMemcpy(d.data(), c->dispatch, 8 * d.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(in.data(), c->inserted, 8 * in.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail(DABS_E_CUDA, "stats copy failed");
    for (int p = 0; p < c->P; p++)
        for (int a = 0; a < N_ALG; a++)
            for (int g = 0; g < N_GEN; g++) {
                o->dispatch[a][g] += d[(p * N_ALG + a) * N_GEN + g];
                o->inserted[a][g] += in[(p * N_ALG + a) * N_GEN + g];
            }
    o->n = c->n; o->n_pad = c->n_pad; o->threads_per_search = batch_threads(c) / batch_spc(c) * c->CL; o->slots = c->slots; o->pools = c->P;
    o->T = c->T; o->B = c->B; o->cap = c->cap;
    o->kernel_launches = c->launches;
    return DABS_OK;
}

// ---------------------------------------------------------------- parity hooks
static void bytes_to_words(const uint8_t* x, int n, std::vector<uint32_t>& w)
{
    std::fill(w.begin(), w.end(), 0u);
    for (int k = 0; k < n; k++) if (x[k]) w[k >> 5] |= 1u << (k & 31);
}
static void words_to_bytes(const std::vector<uint32_t>& w, int n, uint8_t* x)
{
    for (int k = 0; k < n; k++) x[k] = (uint8_t)((w[k >> 5] >> (k & 31)) & 1u);
}

static dabs_status ensure_trace(dabs_ctx* c, int64_t cap)
{
    if (cap <= c->trace_cap && c->tr_bit) return DABS_OK;
    dabs_status st;
    if ((st = dalloc(c, &c->tr_bit, cap)) != DABS_OK) return st;
    if ((st = dalloc(c, &c->tr_E, cap)) != DABS_OK) return st;
    if ((st = dalloc(c, &c->tr_phase, cap)) != DABS_OK) return st;
    c->trace_cap = cap;
    return DABS_OK;
}

extern "C" dabs_status dabs_debug_batch(dabs_ctx* c, uint32_t slot, uint8_t* x, int32_t* delta, int64_t* E,
                                        int32_t* ring, const uint8_t* D, int32_t algo, uint64_t seed,
                                        uint32_t gen, uint8_t* best, int64_t* ebest, int64_t* flips,
                                        int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase, int64_t trace_cap)
{
    if (!c || !x || !delta || !E || !ring || !D || !best || !ebest || !flips) return fail(DABS_E_ARG, "NULL argument");
    if (slot >= (uint32_t)c->slots) return fail(DABS_E_ARG, "slot out of range");
    if (algo < 0 || algo >= N_ALG) return fail(DABS_E_ARG, "algo out of range");
    CK(cudaSetDevice(c->dev));
    const int n = c->n;
    std::vector<uint32_t> w(c->nwp);
    bytes_to_words(x, n, w);
    CK(cudaMemcpy(c->X + (size_t)slot * c->nwp, w.data(), 4 * c->nwp, cudaMemcpyHostToDevice));
    bytes_to_words(D, n, w);
    CK(cudaMemcpy(c->D + (size_t)slot * c->nwp, w.data(), 4 * c->nwp, cudaMemcpyHostToDevice));
    std::vector<int32_t> dp(c->n_pad, INT32_MAX);
    memcpy(dp.data(), delta, 4 * (size_t)n);
    CK(cudaMemcpy(c->delta + (size_t)slot * c->n_pad, dp.data(), 4 * (size_t)c->n_pad, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->E + slot, E, 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->ring + (size_t)slot * TABU_RING, ring, 4 * TABU_RING, cudaMemcpyHostToDevice));
    const uint8_t a8 = (uint8_t)algo;
    CK(cudaMemcpy(c->palgo + slot, &a8, 1, cudaMemcpyHostToDevice));
    const int64_t tcap = trace_cap > 0 ? trace_cap : 1;
    dabs_status st = ensure_trace(c, tcap);
    if (st != DABS_OK) return st;
    const int saved_slot = c->trace_slot;
    const int64_t saved_cap = c->trace_cap;
    c->trace_slot = (int)slot;
    c->trace_cap = trace_cap > 0 ? trace_cap : 0;
    st = launch_batch(c, seed, gen, (int)slot, 1, true);
    c->trace_slot = saved_slot;
    c->trace_cap = saved_cap;
    if (st != DABS_OK) return st;
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(w.data(), c->X + (size_t)slot * c->nwp, 4 * c->nwp, cudaMemcpyDeviceToHost));
    words_to_bytes(w, n, x);
    CK(cudaMemcpy(dp.data(), c->delta + (size_t)slot * c->n_pad, 4 * (size_t)c->n_pad, cudaMemcpyDeviceToHost));
    memcpy(delta, dp.data(), 4 * (size_t)n);
    CK(cudaMemcpy(E, c->E + slot, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ring, c->ring + (size_t)slot * TABU_RING, 4 * TABU_RING, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(w.data(), c->best + (size_t)slot * c->nwp, 4 * c->nwp, cudaMemcpyDeviceToHost));
    words_to_bytes(w, n, best);
    CK(cudaMemcpy(ebest, c->ebest + slot, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(flips, c->flips + slot, 8, cudaMemcpyDeviceToHost));
    if (trace_cap > 0 && tr_bit && tr_E && tr_phase) {
        const int64_t m = *flips < trace_cap ? *flips : trace_cap;
        CK(cudaMemcpy(tr_bit, c->tr_bit, 4 * m, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(tr_E, c->tr_E, 8 * m, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(tr_phase, c->tr_phase, m, cudaMemcpyDeviceToHost));
    }
    return DABS_OK;
}

extern "C" dabs_status dabs_read_slot(const dabs_ctx* c, uint32_t slot, uint8_t* x, int32_t* delta, int64_t* E,
                                      int32_t* ring)
{
    if (!c || slot >= (uint32_t)c->slots) return fail(DABS_E_ARG, "bad ctx/slot");
    CK(cudaSetDevice(c->dev));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<uint32_t> w(c->nwp);
    if (x) {
        CK(cudaMemcpy(w.data(), c->X + (size_t)slot * c->nwp, 4 * c->nwp, cudaMemcpyDeviceToHost));
        words_to_bytes(w, c->n, x);
    }
    if (delta) CK(cudaMemcpy(delta, c->delta + (size_t)slot * c->n_pad, 4 * (size_t)c->n, cudaMemcpyDeviceToHost));
    if (E) CK(cudaMemcpy(E, c->E + slot, 8, cudaMemcpyDeviceToHost));
    if (ring) CK(cudaMemcpy(ring, c->ring + (size_t)slot * TABU_RING, 4 * TABU_RING, cudaMemcpyDeviceToHost));
    return DABS_OK;
}

extern "C" dabs_status dabs_read_pool(const dabs_ctx* c, uint32_t pool, uint8_t* X, int64_t* E, uint64_t* seq,
                                      uint8_t* algo, uint8_t* genop)
{
    if (!c || pool > (uint32_t)c->P) return fail(DABS_E_ARG, "bad ctx/pool");
    CK(cudaSetDevice(c->dev));
    CK(cudaStreamSynchronize(c->stream));
    const PoolView& v = c->pools_h[pool];
    if (X) {
        std::vector<uint32_t> w((size_t)c->cap * c->nwp);
        CK(cudaMemcpy(w.data(), v.X, 4 * w.size(), cudaMemcpyDeviceToHost));
        for (int r = 0; r < c->cap; r++)
            for (int k = 0; k < c->n; k++)
                X[(size_t)r * c->n + k] = (uint8_t)((w[(size_t)r * c->nwp + (k >> 5)] >> (k & 31)) & 1u);
    }
    if (E) CK(cudaMemcpy(E, v.E, 8 * c->cap, cudaMemcpyDeviceToHost));
    if (seq) CK(cudaMemcpy(seq, v.seq, 8 * c->cap, cudaMemcpyDeviceToHost));
    if (algo) CK(cudaMemcpy(algo, v.algo, c->cap, cudaMemcpyDeviceToHost));
    if (genop) CK(cudaMemcpy(genop, v.genop, c->cap, cudaMemcpyDeviceToHost));
    return DABS_OK;
}

extern "C" dabs_status dabs_read_packet(const dabs_ctx* c, uint32_t slot, uint8_t* D, int32_t* algo,
                                        int32_t* genop, uint8_t* best, int64_t* ebest, int64_t* flips)
{
    if (!c || slot >= (uint32_t)c->slots) return fail(DABS_E_ARG, "bad ctx/slot");
    CK(cudaSetDevice(c->dev));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<uint32_t> w(c->nwp);
    if (D) {
        CK(cudaMemcpy(w.data(), c->D + (size_t)slot * c->nwp, 4 * c->nwp, cudaMemcpyDeviceToHost));
        words_to_bytes(w, c->n, D);
    }
    if (best) {
        CK(cudaMemcpy(w.data(), c->best + (size_t)slot * c->nwp, 4 * c->nwp, cudaMemcpyDeviceToHost));
        words_to_bytes(w, c->n, best);
    }
    uint8_t a = 0, g = 0;
    CK(cudaMemcpy(&a, c->palgo + slot, 1, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&g, c->pgenop + slot, 1, cudaMemcpyDeviceToHost));
    if (algo) *algo = a;
    if (genop) *genop = g;
    if (ebest) CK(cudaMemcpy(ebest, c->ebest + slot, 8, cudaMemcpyDeviceToHost));
    if (flips) CK(cudaMemcpy(flips, c->flips + slot, 8, cudaMemcpyDeviceToHost));
    return DABS_OK;
}

extern "C" dabs_status dabs_read_stats_pool(const dabs_ctx* c, uint32_t pool, uint64_t* dispatch, uint64_t* inserted)
{
    if (!c || pool >= (uint32_t)c->P) return fail(DABS_E_ARG, "bad ctx/pool");
    CK(cudaSetDevice(c->dev));
    CK(cudaStreamSynchronize(c->stream));
    const size_t off = (size_t)pool * N_ALG * N_GEN;
    if (dispatch) CK(cudaMemcpy(dispatch, c->dispatch + off, 8 * N_ALG * N_GEN, cudaMemcpyDeviceToHost));
    if (inserted) CK(cudaMemcpy(inserted, c->inserted + off, 8 * N_ALG * N_GEN, cudaMemcpyDeviceToHost));
    return DABS_OK;
}

extern "C" dabs_status dabs_trace_enable(dabs_ctx* c, int32_t slot, int64_t cap)
{
    if (!c) return fail(DABS_E_ARG, "ctx is NULL");
    if (slot >= c->slots) return fail(DABS_E_ARG, "slot out of range");
    if (slot < 0 || cap <= 0) {
        c->trace_slot = -1;
        return DABS_OK;
    }
    dabs_status st = ensure_trace(c, cap);
    if (st != DABS_OK) return st;
    c->trace_slot = slot;
    c->trace_cap = cap;
    return DABS_OK;
}

extern "C" dabs_status dabs_trace_read(const dabs_ctx* c, int32_t* tr_bit, int64_t* tr_E, int8_t* tr_phase,
                                       int64_t* count)
{
    if (!c || c->trace_slot < 0) return fail(DABS_E_STATE, "tracing not enabled");
    CK(cudaSetDevice(c->dev));
    CK(cudaStreamSynchronize(c->stream));
    int64_t f = 0;
    CK(cudaMemcpy(&f, c->flips + c->trace_slot, 8, cudaMemcpyDeviceToHost));
    const int64_t m = f < c->trace_cap ? f : c->trace_cap;
    if (tr_bit) CK(cudaMemcpy(tr_bit, c->tr_bit, 4 * m, cudaMemcpyDeviceToHost));
    if (tr_E) CK(cudaMemcpy(tr_E, c->tr_E, 8 * m, cudaMemcpyDeviceToHost));
    if (tr_phase) CK(cudaMemcpy(tr_phase, c->tr_phase, m, cudaMemcpyDeviceToHost));
    if (count) *count = m;
    return DABS_OK;
}

// ---------------------------------------------------------------- measurement probe
extern "C" dabs_status dabs_probe_row_stream(int32_t device, int64_t rows, int32_t row_bytes, int32_t ctas_per_sm,
                                             int32_t inflight, int32_t iters, double* gbps)
{
    if (!gbps || rows < 1 || row_bytes < 64 || row_bytes % 64 || ctas_per_sm < 1 || inflight < 1 || inflight > 2 ||
        iters < 1 || (size_t)inflight * row_bytes > 200 * 1024)
        return fail(DABS_E_ARG, "bad probe arguments");
    if (device >= 0) CK(cudaSetDevice(device));
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    char* buf = nullptr;
    unsigned long long* sink = nullptr;
    const size_t bytes = (size_t)rows * row_bytes;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return fail(DABS_E_NOMEM, "probe buffer of %zu bytes", bytes);
    if (cudaMalloc(&sink, 8) != cudaSuccess) { cudaFree(buf); return fail(DABS_E_NOMEM, "probe sink"); }
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemsetAsync(buf, 1, bytes, s);
    const size_t smem = (size_t)inflight * row_bytes;
    cudaFuncSetAttribute(probe_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = sms * ctas_per_sm;
    probe_rows_kernel<<<grid, 32, smem, s>>>(buf, (uint32_t)row_bytes, (uint32_t)rows, std::max(1, iters / 10),
                                             inflight, sink);
    cudaEventRecord(a, s);
    probe_rows_kernel<<<grid, 32, smem, s>>>(buf, (uint32_t)row_bytes, (uint32_t)rows, iters, inflight, sink);
    cudaEventRecord(b, s);
    const cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(s);
    cudaFree(sink);
    cudaFree(buf);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess)
        return fail(DABS_E_CUDA, "probe kernel: %s", cudaGetErrorString(e));
    *gbps = (double)grid * iters * row_bytes / (ms * 1e-3) / 1e9;
    return DABS_OK;
}
