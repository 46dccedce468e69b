// C ABI (include/egt_b200.h): device layout upload, solver drivers, graphs.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only; the library is opened at run time (egt_shard)

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

// EGT_TRACE=1 in the environment: host-side phase timings of loading and initialisation on
// stderr (wall clock; device work is synchronised where a phase ends in a host wait)
namespace {
struct Trace {
    bool on;
    std::chrono::steady_clock::time_point t;
    const char* what;
    explicit Trace(const char* w) : on(std::getenv("EGT_TRACE") != nullptr), t(std::chrono::steady_clock::now()), what(w) {}
    void mark(const char* phase) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[egt] %s: %s %.2f ms\n", what, phase, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};
}  // namespace

#include "../../include/egt_b200.h"
#include "game.h"
#include "kernels.cuh"

using namespace egt;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                                 \
    do {                                                                                         \
        cudaError_t _e = (call);                                                                 \
        if (_e != cudaSuccess) return fail(EGT_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

enum SolverKind { SOLVER_NONE = 0, SOLVER_EGT = 1, SOLVER_CFR = 2 };

struct egt_game {
    HostGame host;
    DevGame dg{};
    DevPlayer dp[2]{};              // the view the solver launches (a row slice when sharded)
    DevPlayer dp_full[2]{};         // all rows
    // sharding (egt_shard): this rank computes a slice of every gradient's rows, then one
    // NCCL all-reduce (sum) per gradient gives every rank the full gradient
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    // fused all-gather (egt_shard_peers): the gradient kernels store their rows into every
    // rank's gradient buffer over NVLink; a one-element NCCL all-reduce then orders the ranks
    bool p2p = false;
    DevPeers peers[2];
    std::vector<void*> ipc_opened;
    double* barrier_word = nullptr;
    // rows [shard_lo[p], shard_hi[p]] of player p's gradient hold this rank's slice; with the
    // NCCL all-reduce every other row is zeroed before each sharded gradient (the previous
    // all-reduce left the full gradient there)
    int shard_lo[2] = {0, 0}, shard_hi[2] = {0, 0};
    // emulated ranks on one device (egt_shard_emulate, tests): every rank's slice kernel runs
    // into its own buffer and the collective is a local kernel over the `emu_world` buffers
    int emu_world = 0, emu_fused = 0;
    std::vector<DevPlayer> emu_dp[2];
    std::vector<double*> emu_buf[2];   // [0] is GR[p]
    double** emu_ptrs[2] = {nullptr, nullptr};  // device copy of emu_buf
    int esz = 8;                    // bytes per vector element (8: fp64, 4: fp32 mode)
    std::vector<void*> allocs;
    std::vector<void*> pool_allocs;  // stream-ordered allocations from the library pool (lib_pool)
    bool gr_ipc[2] = {false, false};  // GR[p] is a plain cudaMalloc buffer (exportable over IPC)
    cudaStream_t st = nullptr;      // internal stream (graphs are captured here)
    cudaStream_t user = nullptr;    // caller's stream (nullptr = legacy default)
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaStream_t st2 = nullptr;     // second stream for independent chains inside the graph
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    long long V[2] = {0, 0};        // doubles per game per player vector
    // scratch
    double* partial = nullptr;
    unsigned* counter = nullptr;
    double* partial2 = nullptr;     // reduction scratch of the second stream
    unsigned* counter2 = nullptr;
    double *partial_br = nullptr, *partial2_br = nullptr;  // fused best-response reductions
    unsigned *counter_br = nullptr, *counter2_br = nullptr;
    // solver state
    int solver = SOLVER_NONE;
    int variant = 0;
    DevScalars sc{};
    double* gapval = nullptr;       // [2][G]
    double* gapout = nullptr;       // [G]
    double* gapcur = nullptr;       // [G] eps_sad of the current EGT/as iterate (maintained)
    double* S[2] = {nullptr, nullptr};   // EGT state, 2 slots
    double* C[2] = {nullptr, nullptr};   // EGT cache (smoothed BR as behavioural logs, R16), 2 slots
    double* XQ[2] = {nullptr, nullptr};  // the same smoothed BR in sequence form (x_hat = (1-tau) x + tau XQ), 2 slots
    double* HAT[2] = {nullptr, nullptr};
    double* RESP[2] = {nullptr, nullptr};
    double* GR[2] = {nullptr, nullptr};
    double* R[2] = {nullptr, nullptr};   // CFR regrets
    double* Z[2] = {nullptr, nullptr};   // CFR behavioural strategy
    double* Q[2] = {nullptr, nullptr};   // CFR sequence-form strategy
    double* AVG[2] = {nullptr, nullptr}; // CFR average
    cudaGraphExec_t graph = nullptr;
    long long grads = 0;            // gradient evaluations per game
    long long h2d_bytes = 0;        // uploaded by egt_load_game
    int grads_per_iter = 0;
    // kernel timing mode (egt_timing): eager launches bracketed by CUDA events
    int timing = 0;
    std::vector<int> focus_host;    // per-game focus of the current EGT iteration (timing mode)
    struct Pending { int kind; long long active; double bytes; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> ev_pool;
    double t_ms[EGT_N_KERNEL_KINDS] = {0};
    double t_launch[EGT_N_KERNEL_KINDS] = {0};
    double t_active[EGT_N_KERNEL_KINDS] = {0};
    double t_bytes[EGT_N_KERNEL_KINDS] = {0};
};

const char* egt_last_error(void) { return g_err.c_str(); }

// The library's device memory pool (one per device, created on first use): the large
// per-game vectors are stream-ordered allocations from it, and memory a freed game returns
// stays reserved for the next game (release threshold: unlimited), so loading a batch after
// another one does not pay the page mapping of several GB again.
static cudaMemPool_t lib_pool(cudaError_t* err) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    *err = cudaGetDevice(&dev);
    if (*err != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool = nullptr;
        *err = cudaMemPoolCreate(&pool, &props);
        if (*err != cudaSuccess) return nullptr;
        uint64_t keep = UINT64_MAX;
        *err = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        if (*err != cudaSuccess) return nullptr;
        pools[dev] = pool;
    }
    return pools[dev];
}

// n elements of T: from the library pool on the game's stream (plain cudaMalloc before the
// stream exists)
template <class T>
static int dalloc(egt_game* G, T** p, size_t n) {
    void* q = nullptr;
    if (n == 0) n = 1;
    if (!G->st) {
        cudaError_t e = cudaMalloc(&q, n * sizeof(T));
        if (e != cudaSuccess) return fail(EGT_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        G->allocs.push_back(q);
    } else {
        cudaError_t e = cudaSuccess;
        cudaMemPool_t pool = lib_pool(&e);
        if (pool) e = cudaMallocFromPoolAsync(&q, n * sizeof(T), pool, G->st);
        if (e != cudaSuccess) return fail(EGT_E_CUDA, std::string("cudaMallocFromPoolAsync: ") + cudaGetErrorString(e));
        G->pool_allocs.push_back(q);
    }
    *p = (T*)q;
    return 0;
}

extern "C" int egt_pool_trim(void) {
    cudaError_t e = cudaSuccess;
    cudaMemPool_t pool = lib_pool(&e);
    if (pool) e = cudaMemPoolTrimTo(pool, 0);
    if (e != cudaSuccess) return fail(EGT_E_CUDA, std::string("pool trim: ") + cudaGetErrorString(e));
    return 0;
}

// a per-game vector buffer of n elements in the game's precision (base address only):
// from the library pool on the game's stream, or a plain cudaMalloc when the buffer is
// shared with other processes through CUDA IPC (pool memory has no IPC handle)
static int dalloc_vec(egt_game* G, double** p, size_t n, bool ipc = false) {
    void* q = nullptr;
    if (n == 0) n = 1;
    const size_t bytes = n * (size_t)G->esz;
    if (ipc || !G->st) {
        cudaError_t e = cudaMalloc(&q, bytes);
        if (e != cudaSuccess) return fail(EGT_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        G->allocs.push_back(q);
    } else {
        cudaError_t e = cudaSuccess;
        cudaMemPool_t pool = lib_pool(&e);
        if (pool) e = cudaMallocFromPoolAsync(&q, bytes, pool, G->st);
        if (e != cudaSuccess) return fail(EGT_E_CUDA, std::string("cudaMallocFromPoolAsync: ") + cudaGetErrorString(e));
        G->pool_allocs.push_back(q);
    }
    *p = (double*)q;
    return 0;
}

template <class T>
static int upload(egt_game* G, T** p, const std::vector<T>& v) {
    int r = dalloc(G, p, v.size());
    if (r) return r;
    // stream-ordered after the pool allocation; a pageable source is staged before the call returns
    if (!v.empty()) CK(cudaMemcpyAsync(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, G->st));
    G->h2d_bytes += (long long)(v.size() * sizeof(T));
    return 0;
}

static VecRef vec(double* base, long long stride) {
    VecRef r;
    r.base = base;
    r.game_stride = stride;
    return r;
}

// 2-slot buffers are laid out [slot][G][V]; the slot of game g is cur[g] ^ x
static VecRef slot2(egt_game* G, double* base, int p, int x) {
    VecRef r;
    r.base = base;
    r.game_stride = G->V[p];
    r.slot_stride = (long long)G->host.n_games * G->V[p];
    r.slot_sel = G->sc.cur;
    r.slot_xor = x;
    return r;
}

static int begin(egt_game* G) {
    CK(cudaEventRecord(G->ev_in, G->user));
    CK(cudaStreamWaitEvent(G->st, G->ev_in, 0));
    return 0;
}

static int end(egt_game* G) {
    CK(cudaEventRecord(G->ev_out, G->st));
    CK(cudaStreamWaitEvent(G->user, G->ev_out, 0));
    return 0;
}

// ----------------------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
};

static NcclApi* nccl_api(std::string& err) {
    static NcclApi api;
    static std::once_flag once;
    static std::string load_err;
    std::call_once(once, [] {
        // an NCCL already in the process (e.g. torch's) is reused by soname
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            load_err = std::string("dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
        api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
        api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
        api.errStr = (decltype(api.errStr))dlsym(h, "ncclGetErrorString");
        if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.commDestroy || !api.errStr) {
            load_err = "libnccl.so.2 lacks a required symbol";
            return;
        }
        api.lib = h;
    });
    if (!api.lib) {
        err = load_err;
        return nullptr;
    }
    return &api;
}

static void nccl_destroy(ncclComm_t c) {
    std::string e;
    if (NcclApi* a = nccl_api(e)) a->commDestroy(c);
}

// Rows of player p's gradient that shard `rank` of `world` computes: a contiguous range of
// the sequences that end a terminal, balanced by terminal count, split into chunks of
// ~grad_chunk_terms(n_games) terminals (relative to the range) for the staged kernel.
static void shard_rows(const PlayerLayout& L, int rank, int world, int chunk_terms, int& r0, int& r1,
                       std::vector<int>& chunks) {
    const int n = (int)L.rows_term.size();
    std::vector<long long> cum(n + 1, 0);
    for (int r = 0; r < n; ++r) cum[r + 1] = cum[r] + (L.term_off[L.rows_term[r] + 1] - L.term_off[L.rows_term[r]]);
    auto bound = [&](int k) {
        const long long target = cum[n] * k / world;
        int i = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        if (i > 0 && i < n && L.pair_next[i - 1]) ++i;  // never split a swapped pair of rows
        return i;
    };
    r0 = rank == 0 ? 0 : bound(rank);
    r1 = rank + 1 == world ? n : bound(rank + 1);
    chunks.assign(1, 0);
    for (int r = r0, cnt = 0; r < r1; ++r) {
        cnt += (int)(cum[r + 1] - cum[r]);
        if ((cnt >= chunk_terms && !L.pair_next[r]) || r + 1 == r1) {
            chunks.push_back(r + 1 - r0);
            cnt = 0;
        }
    }
}

static int max_chunk_terms(const PlayerLayout& L, int r0, const std::vector<int>& chunks) {
    int mx = 0;
    for (size_t c = 0; c + 1 < chunks.size(); ++c) {
        int n = 0;
        for (int r = r0 + chunks[c]; r < r0 + chunks[c + 1]; ++r)
            n += L.term_off[L.rows_term[r] + 1] - L.term_off[L.rows_term[r]];
        mx = std::max(mx, n);
    }
    return mx;
}

// A DevPlayer view restricted to shard `rank` of `world` (device chunk table allocated into allocs).
static int make_slice(egt_game* G, int p, int rank, int world, DevPlayer& out, std::vector<void*>& allocs) {
    int r0, r1;
    std::vector<int> chunks;
    shard_rows(G->host.pl[p], rank, world, grad_chunk_terms(G->host.n_games), r0, r1, chunks);
    out = G->dp_full[p];
    out.rows_term = G->dp_full[p].rows_term + r0;
    out.n_rows_term = r1 - r0;
    out.n_chunks = (int)chunks.size() - 1;
    out.max_chunk_terms = max_chunk_terms(G->host.pl[p], r0, chunks);
    void* d = nullptr;
    if (cudaMalloc(&d, sizeof(int) * chunks.size()) != cudaSuccess)
        return fail(EGT_E_CUDA, "cudaMalloc (shard chunks)");
    allocs.push_back(d);
    if (cudaMemcpy(d, chunks.data(), sizeof(int) * chunks.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(EGT_E_CUDA, "cudaMemcpy (shard chunks)");
    out.chunk_off = (const int*)d;
    return 0;
}

// sequence bounds [lo, hi] of a slice's rows (lo > hi: the slice is empty)
static void slice_bounds(const egt_game* G, int p, const DevPlayer& P, int& lo, int& hi) {
    const PlayerLayout& L = G->host.pl[p];
    const int r0 = (int)(P.rows_term - G->dp_full[p].rows_term);
    if (P.n_rows_term == 0) {
        lo = L.n_pub;
        hi = L.n_pub - 1;
        return;
    }
    // (rows_term is in processing order: a swapped pair of rows is never split between slices)
    lo = *std::min_element(L.rows_term.begin() + r0, L.rows_term.begin() + r0 + P.n_rows_term);
    hi = *std::max_element(L.rows_term.begin() + r0, L.rows_term.begin() + r0 + P.n_rows_term);
}

// zero every row of a gradient buffer outside [lo, hi] (all games): before a sharded
// gradient whose result is summed over the ranks
static cudaError_t zero_outside(const egt_game* G, int p, double* base, int lo, int hi, cudaStream_t st) {
    const size_t es = (size_t)G->esz, Hp = (size_t)G->host.H_pad, pitch = es * (size_t)G->V[p];
    const int np = G->host.pl[p].n_pub, Gn = G->host.n_games;
    cudaError_t e = cudaSuccess;
    if (lo > 0) e = cudaMemset2DAsync(base, pitch, 0, es * Hp * (size_t)std::min(lo, np), Gn, st);
    if (e == cudaSuccess && hi + 1 < np && hi + 1 >= 0) {
        char* b = reinterpret_cast<char*>(base) + es * Hp * (size_t)(hi + 1);
        e = cudaMemset2DAsync(b, pitch, 0, es * Hp * (size_t)(np - hi - 1), Gn, st);
    }
    return e;
}

// ----------------------------------------------------------------------------- load
extern "C" int egt_load_game(const egt_game_spec* spec, egt_game** out) {
    if (!spec || !out) return fail(EGT_E_ARG, "null argument");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(EGT_E_CUDA, "no CUDA device");
    if (spec->precision != EGT_F64 && spec->precision != EGT_F32) return fail(EGT_E_ARG, "bad precision");
    Trace tr("load");
    egt_game* G = new egt_game();
    G->esz = spec->precision == EGT_F32 ? 4 : 8;
    std::string err = build_host_game(*spec, G->host);
    tr.mark("host build (trees, strengths, tables)");
    if (!err.empty()) {
        delete G;
        return fail(EGT_E_ARG, err);
    }
    HostGame& H = G->host;
    const int Gn = H.n_games, Hp = H.H_pad, nbs = H.tree.n_board_states;
    int r = 0;
#define TRY(x)                    \
    do {                          \
        r = (x);                  \
        if (r) {                  \
            egt_free_game(G);     \
            return r;             \
        }                         \
    } while (0)
    {
        cudaError_t e = cudaStreamCreateWithFlags(&G->st, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&G->ev_in, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&G->ev_out, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&G->st2, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&G->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&G->ev_join, cudaEventDisableTiming);
        if (e == cudaSuccess) e = kernels_prepare();
        if (e != cudaSuccess) {
            egt_free_game(G);
            return fail(EGT_E_CUDA, std::string("stream/event: ") + cudaGetErrorString(e));
        }
    }
    tr.mark("streams, events, kernel attributes");
    // tables
    std::vector<int> nvalid;
    std::vector<int16_t> order;
    std::vector<uint16_t> cent;
    std::vector<uint32_t> lohi, pcard;
    std::vector<uint8_t> valid;
    for (const BoardTable& tb : H.tables) {
        nvalid.push_back(tb.nvalid);
        order.insert(order.end(), tb.order.begin(), tb.order.end());
        lohi.insert(lohi.end(), tb.lohi.begin(), tb.lohi.end());
        cent.insert(cent.end(), tb.cent.begin(), tb.cent.end());
        pcard.insert(pcard.end(), tb.pcard.begin(), tb.pcard.end());
        valid.insert(valid.end(), tb.valid.begin(), tb.valid.end());
    }
    int* d_nvalid;
    int16_t* d_order;
    uint16_t* d_cent;
    uint32_t *d_lohi, *d_pcard;
    uint8_t* d_valid;
    TRY(upload(G, &d_nvalid, nvalid));
    TRY(upload(G, &d_order, order));
    TRY(upload(G, &d_lohi, lohi));
    TRY(upload(G, &d_cent, cent));
    TRY(upload(G, &d_pcard, pcard));
    TRY(upload(G, &d_valid, valid));
    // the card-domain gradient kernel's per-board plans (river games, one board state)
    bool plans = nbs == 1;
    for (const BoardTable& tb : H.tables) plans = plans && tb.plan.tab.size() == (size_t)CARD_TAB_WORDS;
    if (plans) {
        std::vector<uint32_t> tab;
        tab.reserve(H.tables.size() * (size_t)CARD_TAB_WORDS);
        for (const BoardTable& tb : H.tables) tab.insert(tab.end(), tb.plan.tab.begin(), tb.plan.tab.end());
        uint32_t* d_tab;
        TRY(upload(G, &d_tab, tab));
        G->dg.card_tab = d_tab;
    }
    G->dg.card_plan = plans ? 1 : 0;
    double *d_p0, *d_p1, *d_kg;
    if (G->esz == 8) {
        TRY(upload(G, &d_p0, H.prior[0]));
        TRY(upload(G, &d_p1, H.prior[1]));
    } else {  // fp32 mode: priors in the vectors' precision
        std::vector<float> f0(H.prior[0].begin(), H.prior[0].end()), f1(H.prior[1].begin(), H.prior[1].end());
        float *q0, *q1;
        TRY(upload(G, &q0, f0));
        TRY(upload(G, &q1, f1));
        d_p0 = (double*)q0;
        d_p1 = (double*)q1;
    }
    TRY(upload(G, &d_kg, H.kappa_game));
    std::vector<DevTerm> terms;
    for (const Terminal& t : H.terms) {
        DevTerm d;
        d.amount = t.amount;
        d.kappa = t.kappa;
        d.kind = t.kind;
        d.bs = t.board_state;
        d.seq[0] = t.last_seq[0];
        d.seq[1] = t.last_seq[1];
        terms.push_back(d);
    }
    DevTerm* d_terms;
    TRY(upload(G, &d_terms, terms));
    G->dg.n_games = Gn;
    G->dg.H = H.H;
    G->dg.H_pad = Hp;
    G->dg.hand_size = H.hand_size;
    G->dg.n_bs = nbs;
    G->dg.n_cards = H.n_cards;
    G->dg.esz = G->esz;
    G->dg.all_valid = H.all_valid;
    G->dg.tab_nvalid = d_nvalid;
    G->dg.tab_order = d_order;
    G->dg.tab_lohi = d_lohi;
    G->dg.tab_cent = d_cent;
    G->dg.tab_pcard = reinterpret_cast<const uint2*>(d_pcard);
    G->dg.n_ce = H.n_ce;
    G->dg.seg_w = H.seg_w;
    G->dg.ident = 1;
    for (const BoardTable& tb : H.tables)
        for (int i = 0; i < H.H; ++i)
            if (tb.order[i] != i) G->dg.ident = 0;
    G->dg.tab_valid = d_valid;
    G->dg.prior[0] = d_p0;
    G->dg.prior[1] = d_p1;
    G->dg.kappa_game = d_kg;
    G->dg.terms = d_terms;
    for (int p = 0; p < 2; ++p) {
        const PlayerLayout& L = H.pl[p];
        DevPlayer& P = G->dp[p];
        P.n_pub = L.n_pub;
        P.n_nodes = (int)L.first.size();
        P.n_levels = (int)L.lvl_off.size() - 1;
        P.n_rows_term = (int)L.rows_term.size();
        int *a, *b, *c, *d, *e, *f, *lo, *ln, *ko, *kd, *rt, *co, *so, *sn, *rs, *ss;
        double* be;
        TRY(upload(G, &a, L.first));
        TRY(upload(G, &b, L.nact));
        TRY(upload(G, &c, L.parent_seq));
        TRY(upload(G, &d, L.board_state));
        TRY(upload(G, &be, H.beta[p]));
        TRY(upload(G, &e, L.term_off));
        TRY(upload(G, &f, L.term_idx));
        TRY(upload(G, &lo, L.lvl_off));
        TRY(upload(G, &ln, L.lvl_nodes));
        TRY(upload(G, &ko, L.kid_off));
        TRY(upload(G, &kd, L.kids));
        TRY(upload(G, &rt, L.rows_term));
        TRY(upload(G, &co, L.chunk_off));
        TRY(upload(G, &so, L.sched_off));
        TRY(upload(G, &sn, L.sched_nodes));
        TRY(upload(G, &rs, L.root_slot));
        TRY(upload(G, &ss, L.seq_slot));
        P.seq_slot = ss;
        P.n_int = L.n_int;
        P.sched_off = so;
        P.sched_nodes = sn;
        P.root_slot = rs;
        P.n_root = L.n_root;
        P.n_chunks = (int)L.chunk_off.size() - 1;
        P.chunk_off = co;
        P.max_chunk_terms = max_chunk_terms(L, 0, L.chunk_off);
        P.node_first = a;
        P.node_nact = b;
        P.node_parent = c;
        P.node_bs = d;
        P.beta = be;
        P.term_off = e;
        P.term_idx = f;
        P.lvl_off = lo;
        P.lvl_nodes = ln;
        P.kid_off = ko;
        P.kids = kd;
        P.rows_term = rt;
        if (tree_smem_bytes(P, G->esz) > 200 * 1024) {
            egt_free_game(G);
            return fail(EGT_E_ARG, "public tree too large for the treeplex kernel's shared-memory tile");
        }
        G->V[p] = (long long)L.n_pub * Hp;
    }
    G->dp_full[0] = G->dp[0];
    G->dp_full[1] = G->dp[1];
    const int max_tiles = (H.H + 31) / 32;
    TRY(dalloc(G, &G->partial, (size_t)Gn * max_tiles));
    TRY(dalloc(G, &G->counter, (size_t)Gn));
    TRY(dalloc(G, &G->partial2, (size_t)Gn * max_tiles));
    TRY(dalloc(G, &G->counter2, (size_t)Gn));
    TRY(dalloc(G, &G->partial_br, (size_t)Gn * max_tiles));
    TRY(dalloc(G, &G->counter_br, (size_t)Gn));
    TRY(dalloc(G, &G->partial2_br, (size_t)Gn * max_tiles));
    TRY(dalloc(G, &G->counter2_br, (size_t)Gn));
    if (cudaMemsetAsync(G->counter, 0, sizeof(unsigned) * Gn, G->st) != cudaSuccess ||
        cudaMemsetAsync(G->counter2, 0, sizeof(unsigned) * Gn, G->st) != cudaSuccess ||
        cudaMemsetAsync(G->counter_br, 0, sizeof(unsigned) * Gn, G->st) != cudaSuccess ||
        cudaMemsetAsync(G->counter2_br, 0, sizeof(unsigned) * Gn, G->st) != cudaSuccess) {
        egt_free_game(G);
        return fail(EGT_E_CUDA, "memset");
    }
    // scalars
    DevScalars& S = G->sc;
    TRY(dalloc(G, &S.mu, 2 * (size_t)Gn));
    TRY(dalloc(G, &S.mu_cand, 2 * (size_t)Gn));
    TRY(dalloc(G, &S.tau, (size_t)Gn));
    TRY(dalloc(G, &S.step, (size_t)Gn));
    TRY(dalloc(G, &S.val, 2 * (size_t)Gn));
    TRY(dalloc(G, &S.egv, (size_t)Gn));
    TRY(dalloc(G, &S.focus, (size_t)Gn));
    TRY(dalloc(G, &S.cur, (size_t)Gn));
    TRY(dalloc(G, &S.t, (size_t)Gn));
    TRY(dalloc(G, &S.attempts, (size_t)Gn));
    TRY(dalloc(G, &S.backtracks, (size_t)Gn));
    TRY(dalloc(G, &S.fail, (size_t)Gn));
    TRY(dalloc(G, &S.live, (size_t)Gn));
    {
        double* tg = nullptr;
        TRY(dalloc(G, &tg, (size_t)Gn));
        if (cudaMemsetAsync(tg, 0, sizeof(double) * Gn, G->st) != cudaSuccess) {
            egt_free_game(G);
            return fail(EGT_E_CUDA, "memset");
        }
        S.target = tg;
    }
    TRY(dalloc(G, &G->gapval, 2 * (size_t)Gn));
    TRY(dalloc(G, &G->gapcur, (size_t)Gn));
    S.brval = G->gapval;
    S.gap = G->gapcur;
    TRY(dalloc(G, &G->gapout, (size_t)Gn));
    for (int p = 0; p < 2; ++p) {
        const size_t n = (size_t)Gn * G->V[p];
        TRY(dalloc_vec(G, &G->GR[p], n));
        TRY(dalloc_vec(G, &G->HAT[p], n));
        // rows that end no terminal are never written by the solver's gradient launches
        if (cudaMemsetAsync(G->GR[p], 0, n * G->esz, G->st) != cudaSuccess) {
            egt_free_game(G);
            return fail(EGT_E_CUDA, "memset");
        }
    }
    if (cudaDeviceSynchronize() != cudaSuccess) {
        egt_free_game(G);
        return fail(EGT_E_CUDA, "sync after load");
    }
#undef TRY
    tr.mark("device tables (allocate + copy)");
    *out = G;
    return 0;
}

extern "C" void egt_free_game(egt_game* G) {
    if (!G) return;
    if (G->graph) cudaGraphExecDestroy(G->graph);
    if (G->st) cudaStreamSynchronize(G->st);
    for (auto& p : G->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (cudaEvent_t e : G->ev_pool) cudaEventDestroy(e);
    for (void* q : G->ipc_opened) cudaIpcCloseMemHandle(q);
    if (G->comm) nccl_destroy(G->comm);
    for (void* p : G->allocs) cudaFree(p);
    if (G->st) {
        for (void* p : G->pool_allocs) cudaFreeAsync(p, G->st);
        cudaStreamSynchronize(G->st);
    }
    if (G->ev_in) cudaEventDestroy(G->ev_in);
    if (G->ev_out) cudaEventDestroy(G->ev_out);
    if (G->ev_fork) cudaEventDestroy(G->ev_fork);
    if (G->ev_join) cudaEventDestroy(G->ev_join);
    if (G->st2) {
        cudaStreamSynchronize(G->st2);
        cudaStreamDestroy(G->st2);
    }
    if (G->st) cudaStreamDestroy(G->st);
    delete G;
}

extern "C" int egt_set_stream(egt_game* G, void* stream) {
    if (!G) return fail(EGT_E_ARG, "null game");
    G->user = (cudaStream_t)stream;
    return 0;
}

extern "C" int egt_game_info_get(const egt_game* G, egt_game_info* o) {
    if (!G || !o) return fail(EGT_E_ARG, "null argument");
    const HostGame& H = G->host;
    memset(o, 0, sizeof(*o));
    o->n_games = H.n_games;
    o->H = H.H;
    o->H_pad = H.H_pad;
    o->n_combos = H.n_combos;
    for (int p = 0; p < 2; ++p) {
        o->n_pub[p] = H.pl[p].n_pub;
        o->n_nodes[p] = (int)H.pl[p].first.size();
        o->depth[p] = H.pl[p].depth;
        o->vec_stride[p] = G->V[p];
    }
    o->n_terminals = (int)H.terms.size();
    o->max_abs_A[0] = 0.0;
    o->h2d_bytes = G->h2d_bytes;
    o->precision = G->esz == 4 ? EGT_F32 : EGT_F64;
    for (int p = 0; p < 2; ++p) {
        std::vector<char> seen(H.pl[1 - p].n_pub, 0);
        for (const Terminal& t : H.terms)
            if (t.last_seq[1 - p] != 0) seen[t.last_seq[1 - p]] = 1;
        int n = 0;
        for (char c : seen) n += c;
        o->grad_rows_read[p] = n;
        o->grad_rows_written[p] = (int)H.pl[p].rows_term.size();
    }
    return 0;
}

extern "C" int egt_hand_cards(const egt_game* G, int32_t g, int32_t* out) {
    if (!G || !out || g < 0 || g >= G->host.n_games) return fail(EGT_E_ARG, "bad argument");
    const HostGame& H = G->host;
    for (int h = 0; h < H.H; ++h) {
        out[2 * h] = H.hand_cards[((size_t)g * H.H + h) * 2];
        out[2 * h + 1] = H.hand_size == 2 ? H.hand_cards[((size_t)g * H.H + h) * 2 + 1] : -1;
    }
    return 0;
}

extern "C" int egt_pub_history(const egt_game* G, int32_t player, int32_t s, char* buf, int32_t buflen) {
    if (!G || !buf || buflen < 1 || player < 0 || player > 1) return fail(EGT_E_ARG, "bad argument");
    const PlayerLayout& L = G->host.pl[player];
    if (s < 0 || s >= L.n_pub) return fail(EGT_E_ARG, "sequence out of range");
    const std::string& h = L.seq_hist[s];
    if ((int)h.size() + 1 > buflen) return fail(EGT_E_ARG, "buffer too small");
    memcpy(buf, h.c_str(), h.size() + 1);
    return 0;
}

// ----------------------------------------------------------------------------- kernel-level
static cudaError_t allreduce_grad(egt_game* G, int p, VecRef out);

extern "C" int egt_gradient(egt_game* G, int32_t player, const double* din, double* dout) {
    if (!G || !din || !dout || player < 0 || player > 1) return fail(EGT_E_ARG, "bad argument");
    if (begin(G)) return EGT_E_CUDA;
    VecRef out = vec(dout, G->V[player]);
    CK(launch_gradient(G->dg, G->dp[player], player, vec(const_cast<double*>(din), G->V[1 - player]), out,
                       nullptr, 0, 1, G->st));
    CK(allreduce_grad(G, player, out));
    return end(G);
}

extern "C" int egt_gradient_rows(egt_game* G, int32_t player, int32_t rank, int32_t world, const double* din,
                                 double* dout) {
    if (!G || !din || !dout || player < 0 || player > 1 || world < 1 || rank < 0 || rank >= world)
        return fail(EGT_E_ARG, "bad argument");
    std::vector<void*> tmp;
    DevPlayer P;
    int r = make_slice(G, player, rank, world, P, tmp);
    if (!r && begin(G)) r = EGT_E_CUDA;
    if (!r) {
        cudaError_t e = launch_gradient(G->dg, P, player, vec(const_cast<double*>(din), G->V[1 - player]),
                                        vec(dout, G->V[player]), nullptr, 0, 1, G->st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(G->st);
        if (e != cudaSuccess) r = fail(EGT_E_CUDA, std::string("egt_gradient_rows: ") + cudaGetErrorString(e));
    }
    for (void* q : tmp) cudaFree(q);
    if (r) return r;
    return end(G);
}

extern "C" int egt_gradient_rows_to(egt_game* G, int32_t player, int32_t rank, int32_t world, const double* din,
                                    const uint64_t* dsts, int32_t n_dst) {
    if (!G || !din || !dsts || player < 0 || player > 1 || world < 1 || rank < 0 || rank >= world || n_dst < 1 ||
        n_dst > EGT_MAX_PEERS)
        return fail(EGT_E_ARG, "bad argument");
    DevPeers pr;
    pr.n = n_dst;
    for (int d = 0; d < n_dst; ++d) pr.base[d] = reinterpret_cast<void*>(dsts[d]);
    std::vector<void*> tmp;
    DevPlayer P;
    int r = make_slice(G, player, rank, world, P, tmp);
    if (!r && begin(G)) r = EGT_E_CUDA;
    if (!r) {
        cudaError_t e = launch_gradient(G->dg, P, player, vec(const_cast<double*>(din), G->V[1 - player]),
                                        vec(reinterpret_cast<double*>(dsts[0]), G->V[player]), nullptr, 0, 0, G->st,
                                        &pr);
        if (e == cudaSuccess) e = cudaStreamSynchronize(G->st);
        if (e != cudaSuccess) r = fail(EGT_E_CUDA, std::string("egt_gradient_rows_to: ") + cudaGetErrorString(e));
    }
    for (void* q : tmp) cudaFree(q);
    if (r) return r;
    return end(G);
}

extern "C" int egt_ipc_handles(egt_game* G, uint8_t* out) {
    if (!G || !out) return fail(EGT_E_ARG, "bad argument");
    for (int p = 0; p < 2; ++p) {
        if (!G->gr_ipc[p]) {
            // pool memory has no IPC handle: move this gradient buffer to a plain allocation
            // (its contents are scratch except the rows no terminal ends, which stay 0)
            const size_t n = (size_t)G->host.n_games * G->V[p];
            double* q = nullptr;
            if (dalloc_vec(G, &q, n, true)) return EGT_E_CUDA;
            CK(cudaMemset(q, 0, n * G->esz));
            CK(cudaStreamSynchronize(G->st));
            auto it = std::find(G->pool_allocs.begin(), G->pool_allocs.end(), (void*)G->GR[p]);
            if (it != G->pool_allocs.end()) {
                CK(cudaFreeAsync(*it, G->st));
                G->pool_allocs.erase(it);
            }
            G->GR[p] = q;
            G->gr_ipc[p] = true;
            if (G->graph) {  // a captured iteration would still name the old buffer
                cudaGraphExecDestroy(G->graph);
                G->graph = nullptr;
            }
        }
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, G->GR[p]));
        static_assert(sizeof(h) == EGT_IPC_HANDLE_BYTES, "IPC handle size");
        memcpy(out + p * sizeof(h), &h, sizeof(h));
    }
    return 0;
}

extern "C" int egt_shard_peers(egt_game* G, const uint8_t* handles) {
    if (!G || !handles) return fail(EGT_E_ARG, "bad argument");
    if (!G->comm) return fail(EGT_E_STATE, "egt_shard_peers needs egt_shard with an NCCL id first");
    if (G->world > EGT_MAX_PEERS) return fail(EGT_E_ARG, "too many ranks for the fused all-gather");
    if (G->solver != SOLVER_NONE) return fail(EGT_E_STATE, "egt_shard_peers must precede egt_init / cfr_init");
    if (!G->barrier_word && dalloc(G, &G->barrier_word, 1)) return EGT_E_CUDA;
    CK(cudaMemsetAsync(G->barrier_word, 0, sizeof(double), G->st));
    CK(cudaStreamSynchronize(G->st));
    for (int p = 0; p < 2; ++p) {
        G->peers[p].n = G->world;
        for (int r = 0; r < G->world; ++r) {
            if (r == G->rank) {
                G->peers[p].base[r] = G->GR[p];
                continue;
            }
            cudaIpcMemHandle_t h;
            memcpy(&h, handles + ((size_t)r * 2 + p) * sizeof(h), sizeof(h));
            void* q = nullptr;
            CK(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
            G->ipc_opened.push_back(q);
            G->peers[p].base[r] = q;
        }
    }
    G->p2p = true;
    if (G->graph) {
        cudaGraphExecDestroy(G->graph);
        G->graph = nullptr;
    }
    return 0;
}

extern "C" int egt_nccl_unique_id(uint8_t* out) {
    if (!out) return fail(EGT_E_ARG, "null argument");
    std::string err;
    NcclApi* a = nccl_api(err);
    if (!a) return fail(EGT_E_CUDA, err);
    ncclUniqueId id;
    ncclResult_t r = a->getUniqueId(&id);
    if (r != ncclSuccess) return fail(EGT_E_CUDA, std::string("ncclGetUniqueId: ") + a->errStr(r));
    static_assert(sizeof(ncclUniqueId) == EGT_NCCL_ID_BYTES, "NCCL unique id size");
    memcpy(out, &id, sizeof(id));
    return 0;
}

extern "C" int egt_shard(egt_game* G, int32_t rank, int32_t world, const uint8_t* id) {
    if (!G || world < 1 || rank < 0 || rank >= world || (world > 1 && !id)) return fail(EGT_E_ARG, "bad argument");
    if (G->solver != SOLVER_NONE) return fail(EGT_E_STATE, "egt_shard must precede egt_init / cfr_init");
    if (G->comm) {
        nccl_destroy(G->comm);
        G->comm = nullptr;
    }
    G->rank = rank;
    G->world = world;
    for (int p = 0; p < 2; ++p) {
        int r = make_slice(G, p, rank, world, G->dp[p], G->allocs);
        if (r) return r;
        slice_bounds(G, p, G->dp[p], G->shard_lo[p], G->shard_hi[p]);
    }
    if (id) {  // world == 1 with an id still builds a (1-rank) communicator: the same path
        std::string err;
        NcclApi* a = nccl_api(err);
        if (!a) return fail(EGT_E_CUDA, err);
        ncclUniqueId uid;
        memcpy(&uid, id, sizeof(uid));
        ncclResult_t r = a->commInitRank(&G->comm, world, uid, rank);
        if (r != ncclSuccess) return fail(EGT_E_CUDA, std::string("ncclCommInitRank: ") + a->errStr(r));
    }
    if (G->graph) {
        cudaGraphExecDestroy(G->graph);
        G->graph = nullptr;
    }
    return 0;
}

static TreeArgs base_args() { return TreeArgs(); }

extern "C" int egt_smoothed_br(egt_game* G, int32_t player, const double* dg, double gsign, const double* dmu,
                               double* dq, double* db, double* dlb, double* dval) {
    if (!G || !dg || !dmu || player < 0 || player > 1) return fail(EGT_E_ARG, "bad argument");
    TreeArgs A = base_args();
    A.mode = TM_SBR;
    A.g = vec(const_cast<double*>(dg), G->V[player]);
    A.gsign = gsign;
    A.mu = dmu;
    if (dq) A.out_q = vec(dq, G->V[player]);
    if (db) A.out_b = vec(db, G->V[player]);
    if (dlb) A.out_lb = vec(dlb, G->V[player]);
    A.value = dval;
    A.partial = G->partial;
    A.counter = G->counter;
    if (begin(G)) return EGT_E_CUDA;
    CK(launch_tree(G->dg, G->dp[player], player, A, G->st));
    return end(G);
}

extern "C" int egt_prox(egt_game* G, int32_t player, const double* dg, double gsign, const double* dstep,
                        const double* dcenter_lb, double* dq) {
    if (!G || !dg || !dstep || !dcenter_lb || !dq || player < 0 || player > 1) return fail(EGT_E_ARG, "bad argument");
    TreeArgs A = base_args();
    A.mode = TM_PROX;
    A.g = vec(const_cast<double*>(dg), G->V[player]);
    A.gsign = gsign;
    A.mu = dstep;
    A.center = vec(const_cast<double*>(dcenter_lb), G->V[player]);
    A.out_q = vec(dq, G->V[player]);
    if (begin(G)) return EGT_E_CUDA;
    CK(launch_tree(G->dg, G->dp[player], player, A, G->st));
    return end(G);
}

extern "C" int egt_best_response(egt_game* G, int32_t player, const double* dg, double gsign, double* dval) {
    if (!G || !dg || !dval || player < 0 || player > 1) return fail(EGT_E_ARG, "bad argument");
    TreeArgs A = base_args();
    A.mode = TM_BR;
    A.g = vec(const_cast<double*>(dg), G->V[player]);
    A.gsign = gsign;
    A.value = dval;
    A.partial = G->partial;
    A.counter = G->counter;
    if (begin(G)) return EGT_E_CUDA;
    CK(launch_tree(G->dg, G->dp[player], player, A, G->st));
    return end(G);
}

// ----------------------------------------------------------------------------- EGT
static const double GSIGN[2] = {+1.0, -1.0};  // min-form objective of each player (R5)

static int ensure_egt_buffers(egt_game* G) {
    const int Gn = G->host.n_games;
    for (int p = 0; p < 2; ++p) {
        const size_t n = (size_t)Gn * G->V[p];
        if (!G->S[p] && dalloc_vec(G, &G->S[p], 2 * n)) return EGT_E_CUDA;
        if (!G->C[p] && dalloc_vec(G, &G->C[p], 2 * n)) return EGT_E_CUDA;
        if (!G->XQ[p] && dalloc_vec(G, &G->XQ[p], 2 * n)) return EGT_E_CUDA;
        if (!G->RESP[p] && dalloc_vec(G, &G->RESP[p], n)) return EGT_E_CUDA;
    }
    return 0;
}

// ---- kernel timing (egt_timing): every launch bracketed by a pair of events on G->st
static cudaEvent_t pool_event(egt_game* G) {
    if (!G->ev_pool.empty()) {
        cudaEvent_t e = G->ev_pool.back();
        G->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

static cudaError_t timing_flush(egt_game* G) {
    if (G->pending.empty()) return cudaSuccess;
    cudaError_t e = cudaStreamSynchronize(G->st);
    if (e != cudaSuccess) return e;
    for (auto& p : G->pending) {
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, p.a, p.b);
        if (e != cudaSuccess) return e;
        G->t_ms[p.kind] += ms;
        G->t_launch[p.kind] += 1;
        G->t_active[p.kind] += (double)p.active;
        G->t_bytes[p.kind] += p.bytes;
        G->ev_pool.push_back(p.a);
        G->ev_pool.push_back(p.b);
    }
    G->pending.clear();
    return cudaSuccess;
}

// games that do work under (mask, want); only known on the host in timing mode
static long long active_games(egt_game* G, const int* mask, int want) {
    const int Gn = G->host.n_games;
    if (!mask) return Gn;
    if ((int)G->focus_host.size() != Gn) return Gn;
    long long n = 0;
    if (mask == G->sc.focus)
        for (int g = 0; g < Gn; ++g) n += G->focus_host[g] == want;
    else if (mask == G->sc.live)  // a stopped game has focus -1; live games have 0 or 1
        for (int g = 0; g < Gn; ++g) n += (G->focus_host[g] >= 0) == (want == 1);
    else
        return Gn;
    return n;
}

template <class F>
static cudaError_t timed(egt_game* G, int kind, long long active, F&& launch, double bytes_per_game = 0.0) {
    if (!G->timing) return launch();
    cudaEvent_t a = pool_event(G), b = pool_event(G);
    cudaError_t e = cudaEventRecord(a, G->st);
    if (e == cudaSuccess) e = launch();
    if (e == cudaSuccess) e = cudaEventRecord(b, G->st);
    if (e != cudaSuccess) return e;
    G->pending.push_back({kind, active, bytes_per_game * (double)active, a, b});
    if (G->pending.size() >= 1024) return timing_flush(G);
    return cudaSuccess;
}

// compulsory HBM bytes of one treeplex pass of one game: every vector the
// pass reads or writes, n_pub x H elements each (read-modify-write vectors count twice)
static double tree_bytes_per_game(const egt_game* G, int p, const TreeArgs& A) {
    int n = 0;
    const bool has_grad = A.mode == TM_SBR || A.mode == TM_PROX || A.mode == TM_BR || A.mode == TM_CFR;
    n += has_grad;
    if (A.center.ok()) n += A.mode == TM_CFR ? 2 : 1;
    n += A.regret.ok() ? 2 : 0;
    n += A.avg.ok() ? 2 : 0;
    n += A.out_b.ok() + A.out_q.ok() + A.out_lb.ok() + A.comb_in.ok() + A.comb_out.ok();
    return (double)n * G->host.pl[p].n_pub * G->host.H * G->esz;
}

// compulsory HBM bytes of one gradient of one game
static double grad_bytes_per_game(const egt_game* G, int p, bool comb = false) {
    const HostGame& H = G->host;
    std::vector<char> seen(H.pl[1 - p].n_pub, 0);
    int rd = 0;
    for (const Terminal& t : H.terms)
        if (t.last_seq[1 - p] != 0 && !seen[t.last_seq[1 - p]]) {
            seen[t.last_seq[1 - p]] = 1;
            ++rd;
        }
    // comb: the input is formed from two vectors' rows (Alg. 2 line 1 fused into the gradient)
    return (double)((comb ? 2 : 1) * rd + (int)H.pl[p].rows_term.size() + 2) * H.H * G->esz;
}

static cudaError_t tree(egt_game* G, int p, const TreeArgs& A) {
    return timed(
        G, EGT_KERNEL_TREE, active_games(G, A.mask, A.want),
        [&] { return launch_tree(G->dg, G->dp[p], p, A, G->st); }, G->timing ? tree_bytes_per_game(G, p, A) : 0.0);
}
// the other ranks' rows of a sharded gradient, summed in by an in-place NCCL all-reduce
static cudaError_t allreduce_grad(egt_game* G, int p, VecRef out) {
    if (!G->comm) return cudaSuccess;
    std::string err;
    NcclApi* a = nccl_api(err);
    if (!a || out.slot_sel) return cudaErrorInvalidValue;
    const size_t count = (size_t)G->host.n_games * G->V[p];
    return timed(G, EGT_KERNEL_COMM, G->host.n_games, [&] {
        return a->allReduce(out.base, out.base, count, G->esz == 8 ? ncclDouble : ncclFloat, ncclSum, G->comm,
                            G->st) == ncclSuccess
                   ? cudaSuccess
                   : cudaErrorUnknown;
    });
}

// ranks' barrier after a fused all-gather: a one-element all-reduce on the stream
static cudaError_t peer_barrier(egt_game* G) {
    std::string err;
    NcclApi* a = nccl_api(err);
    if (!a) return cudaErrorInvalidValue;
    return timed(G, EGT_KERNEL_COMM, 0, [&] {
        return a->allReduce(G->barrier_word, G->barrier_word, 1, ncclDouble, ncclSum, G->comm, G->st) == ncclSuccess
                   ? cudaSuccess
                   : cudaErrorUnknown;
    });
}

static cudaError_t emu_grad(egt_game* G, int p, VecRef in, VecRef out, const int* mask, int want, int all_rows,
                            const GradComb* comb);

// One gradient of the solver.  Sharded (egt_shard), this rank computes its slice of the rows:
//  * fused all-gather (egt_shard_peers): the kernel stores its rows into every rank's buffer;
//    a peer barrier BEFORE the launch orders those stores after every rank's last read of
//    the buffer (the previous gradient's consumers), one AFTER it makes every rank's rows
//    visible before anyone reads them -- correct by construction whatever the launch order;
//  * NCCL all-reduce: the rows outside the slice are zeroed first (they hold the previous
//    gradient's sum), so the in-place sum adds exact zeros to every other rank's rows.
// all_rows: every row is written (rows no terminal ends are 0), for buffers that are not
// the solver's gradient buffers.
static cudaError_t grad(egt_game* G, int p, VecRef in, VecRef out, const int* mask = nullptr, int want = 0,
                        int all_rows = 0, const GradComb* comb = nullptr) {
    if (G->emu_world > 1) return emu_grad(G, p, in, out, mask, want, all_rows, comb);
    const bool fused = G->p2p && out.base == G->GR[p] && !out.slot_sel && !all_rows;
    if (fused) {
        cudaError_t e = peer_barrier(G);
        if (e != cudaSuccess) return e;
    } else if (G->comm && !all_rows) {
        cudaError_t e = zero_outside(G, p, out.base, G->shard_lo[p], G->shard_hi[p], G->st);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = timed(
        G, p == 0 ? EGT_KERNEL_GRAD_AY : EGT_KERNEL_GRAD_ATX, active_games(G, mask, want),
        [&] {
            return launch_gradient(G->dg, G->dp[p], p, in, out, mask, want, all_rows, G->st,
                                   fused ? &G->peers[p] : nullptr, comb);
        },
        G->timing ? grad_bytes_per_game(G, p, comb != nullptr) : 0.0);
    if (e != cudaSuccess) return e;
    return fused ? peer_barrier(G) : allreduce_grad(G, p, out);
}

// Emulated ranks (egt_shard_emulate): rank r's slice kernel writes buffer r (rank 0's is the
// solver's output) exactly as on rank r; the collective is a local kernel over the buffers.
static cudaError_t emu_grad(egt_game* G, int p, VecRef in, VecRef out, const int* mask, int want, int all_rows,
                            const GradComb* comb) {
    const int W = G->emu_world;
    if (all_rows || out.slot_sel || out.base != G->GR[p]) {  // not a solver gradient buffer: unsharded
        return launch_gradient(G->dg, G->dp_full[p], p, in, out, mask, want, all_rows, G->st, nullptr, comb);
    }
    cudaError_t e = cudaSuccess;
    for (int r = 0; r < W && e == cudaSuccess; ++r) {
        const DevPlayer& P = G->emu_dp[p][r];
        VecRef o = out;
        o.base = G->emu_buf[p][r];
        if (G->emu_fused) {
            DevPeers pr;
            pr.n = W;
            for (int d = 0; d < W; ++d) pr.base[d] = G->emu_buf[p][d];
            e = launch_gradient(G->dg, P, p, in, o, mask, want, 0, G->st, &pr, comb);
        } else {
            int lo, hi;
            slice_bounds(G, p, P, lo, hi);
            e = zero_outside(G, p, o.base, lo, hi, G->st);
            if (e == cudaSuccess) e = launch_gradient(G->dg, P, p, in, o, mask, want, 0, G->st, nullptr, comb);
        }
    }
    if (e == cudaSuccess && !G->emu_fused)
        e = launch_emu_allreduce(G->emu_ptrs[p], W, (size_t)G->host.n_games * G->V[p], G->esz, G->st);
    return e;
}

extern "C" int egt_shard_emulate(egt_game* G, int32_t world, int32_t fused) {
    if (!G || world < 1 || world > EGT_MAX_PEERS) return fail(EGT_E_ARG, "bad argument");
    if (G->solver != SOLVER_NONE) return fail(EGT_E_STATE, "egt_shard_emulate must precede egt_init / cfr_init");
    if (G->comm || G->p2p) return fail(EGT_E_STATE, "game is already sharded over real ranks");
    G->emu_world = world > 1 ? world : 0;
    G->emu_fused = fused != 0;
    for (int p = 0; p < 2; ++p) {
        G->emu_dp[p].assign(world, DevPlayer());
        G->emu_buf[p].assign(world, nullptr);
        G->emu_buf[p][0] = G->GR[p];
        for (int r = 0; r < world; ++r) {
            int rc = make_slice(G, p, r, world, G->emu_dp[p][r], G->allocs);
            if (rc) return rc;
            if (r > 0) {
                const size_t n = (size_t)G->host.n_games * G->V[p];
                if (dalloc_vec(G, &G->emu_buf[p][r], n)) return EGT_E_CUDA;
                CK(cudaMemsetAsync(G->emu_buf[p][r], 0, n * G->esz, G->st));
            }
        }
        if (!G->emu_ptrs[p] && dalloc(G, &G->emu_ptrs[p], (size_t)EGT_MAX_PEERS)) return EGT_E_CUDA;
        CK(cudaMemcpyAsync(G->emu_ptrs[p], G->emu_buf[p].data(), sizeof(double*) * world, cudaMemcpyHostToDevice, G->st));
    }
    CK(cudaStreamSynchronize(G->st));
    if (G->graph) {
        cudaGraphExecDestroy(G->graph);
        G->graph = nullptr;
    }
    return 0;
}
template <class F>
static cudaError_t scalar_k(egt_game* G, F&& launch) {
    return timed(G, EGT_KERNEL_SCALAR, G->host.n_games, launch);
}

// EGT initial point (Alg. 1/3 lines 1-2, R4) at the current per-game mu;
// leaves val[0] = phi_{mu_x}(y0), val[1] = -f_{mu_y}(x0) and the caches C[.][cur].
// A^T x_omega, x_omega the uniform behavioural strategy in sequence form (into HAT[0]);
// independent of mu, so the mu search evaluates it once (into `out`)
static int egt_omega_gradient(egt_game* G, double* out) {
    TreeArgs U = base_args();
    U.mode = TM_UNIFORM;
    U.out_q = vec(G->HAT[0], G->V[0]);
    CK(tree(G, 0, U));
    // every row written: `out` is scratch whose terminal-free rows would otherwise be stale
    CK(grad(G, 1, vec(G->HAT[0], G->V[0]), vec(out, G->V[1]), nullptr, 0, 1));
    return 0;
}

// Alg. 1 / 3 initialisation at the current mu: y0 = y_mu(x_omega), x0 = x_mu(y0) (cache C[0]),
// y_mu(x0) (cache C[1]) and the values the excessive-gap check needs.  g_omega: A^T x_omega
// already evaluated (the mu search), or nullptr to evaluate it here.  mask: only the games
// with mask[g] == 1 (the mu scan's games still scanning), or nullptr for all.
// With a mask (a round of the practical-mu scan) only the values the excessive-gap test reads
// are produced: the caches C and XQ come from the final, unmasked call.
static int egt_initial_point(egt_game* G, double* g_omega, const int* mask = nullptr) {
    const int Gn = G->host.n_games;
    DevScalars& S = G->sc;
    if (!g_omega) {
        if (egt_omega_gradient(G, G->GR[1])) return EGT_E_CUDA;
        g_omega = G->GR[1];
    }
    // y0 = y_{mu_y}(x_omega)
    TreeArgs A = base_args();
    A.mode = TM_SBR;
    A.g = vec(g_omega, G->V[1]);
    A.gsign = GSIGN[1];
    A.mu = S.mu + Gn;
    A.out_q = slot2(G, G->S[1], 1, 0);
    A.mask = mask;
    A.want = 1;
    CK(tree(G, 1, A));
    // x0 = x_{mu_x}(y0) (also the cache C[0]); phi_{mu_x}(y0)
    CK(grad(G, 0, slot2(G, G->S[1], 1, 0), vec(G->GR[0], G->V[0]), mask, 1));
    A = base_args();
    A.mode = TM_SBR;
    A.g = vec(G->GR[0], G->V[0]);
    A.gsign = GSIGN[0];
    A.mu = S.mu;
    A.out_q = slot2(G, G->S[0], 0, 0);
    if (!mask) A.out_lb = slot2(G, G->C[0], 0, 0);
    A.value = S.val;
    A.partial = G->partial;
    A.counter = G->counter;
    A.mask = mask;
    A.want = 1;
    CK(tree(G, 0, A));
    // y_{mu_y}(x0) (cache C[1]) and -f_{mu_y}(x0)
    CK(grad(G, 1, slot2(G, G->S[0], 0, 0), vec(G->GR[1], G->V[1]), mask, 1));
    A = base_args();
    A.mode = TM_SBR;
    A.g = vec(G->GR[1], G->V[1]);
    A.gsign = GSIGN[1];
    A.mu = S.mu + Gn;
    if (!mask) {
        A.out_lb = slot2(G, G->C[1], 1, 0);
        A.out_q = slot2(G, G->XQ[1], 1, 0);
    }
    A.value = S.val + Gn;
    A.partial = G->partial;
    A.counter = G->counter;
    A.mask = mask;
    A.want = 1;
    CK(tree(G, 1, A));
    // x0 = x_mu(y0) is also the sequence-form cache of player 0 (every game's slot is 0 here)
    if (!mask)
        CK(cudaMemcpyAsync(G->XQ[0], G->S[0], (size_t)G->esz * Gn * G->V[0], cudaMemcpyDeviceToDevice, G->st));
    return 0;
}

static int record_egt_iteration(egt_game* G) {
    const int Gn = G->host.n_games;
    DevScalars& S = G->sc;
    const int var = G->variant;
    CK(scalar_k(G, [&] { return launch_egt_prepare(var, Gn, S, G->st); }));
    if (G->timing) {
        // timing mode only: learn each game's focus so masked launches report their active games
        G->focus_host.assign(Gn, 0);
        CK(cudaMemcpyAsync(G->focus_host.data(), S.focus, sizeof(int) * Gn, cudaMemcpyDeviceToHost, G->st));
        CK(cudaStreamSynchronize(G->st));
    }
    // The two focus chains touch disjoint games (every launch is masked by the game's focus
    // player), so in graph mode player 2's chain runs on the second stream beside player 1's:
    // the half-empty masked launches of one chain fill the SMs the other leaves idle.  Not in
    // timing mode (per-kernel events) and not when sharded (one all-reduce order on all ranks).
    const bool fork_focus = !G->timing && !G->comm && !G->emu_world;
    cudaStream_t main_st = G->st;
    struct Restore {  // G->st is the main stream again on every exit path
        egt_game* g;
        cudaStream_t s;
        ~Restore() { g->st = s; }
    } restore{G, main_st};
    if (fork_focus) {
        CK(cudaEventRecord(G->ev_fork, main_st));
        CK(cudaStreamWaitEvent(G->st2, G->ev_fork, 0));
    }
    for (int p = 0; p < 2; ++p) {
        const int o = 1 - p;
        if (fork_focus) G->st = p == 0 ? main_st : G->st2;
        if (var != EGT_AS) {
            // x_{mu_x}(y) for the focused player (not cached without the EGC check)
            CK(grad(G, p, slot2(G, G->S[o], o, 0), vec(G->GR[p], G->V[p]), S.focus, p));
            TreeArgs A = base_args();
            A.mode = TM_SBR;
            A.g = vec(G->GR[p], G->V[p]);
            A.gsign = GSIGN[p];
            A.mu = S.mu + (size_t)p * Gn;
            A.out_lb = slot2(G, G->C[p], p, 0);
            A.out_q = slot2(G, G->XQ[p], p, 0);
            A.mask = S.focus;
            A.want = p;
            CK(tree(G, p, A));
        }
        // Alg. 2 line 1: p_hat = (1 - tau) p + tau p_mu(o), formed by the gradient of line 2 on
        // the rows it reads (p_mu(o) in sequence form, cached by the SBR that produced it)
        GradComb hat;
        hat.b = slot2(G, G->XQ[p], p, 0);
        hat.tau = S.tau;
        // line 2: o_plus = (1 - tau) o + tau o_mu(p_hat)
        CK(grad(G, o, slot2(G, G->S[p], p, 0), vec(G->GR[o], G->V[o]), S.focus, p, 0, &hat));
        TreeArgs A = base_args();
        A.mode = TM_SBR;
        A.g = vec(G->GR[o], G->V[o]);
        A.gsign = GSIGN[o];
        A.mu = S.mu + (size_t)o * Gn;
        A.out_q = vec(G->RESP[o], G->V[o]);
        A.comb_in = slot2(G, G->S[o], o, 0);
        A.comb_out = slot2(G, G->S[o], o, 1);
        A.tau = S.tau;
        A.mask = S.focus;
        A.want = p;
        CK(tree(G, o, A));
        // line 3-4: p_til = prox_{p_mu(o)}(s grad f(p_hat)), p_plus = (1 - tau) p + tau p_til
        CK(grad(G, p, vec(G->RESP[o], G->V[o]), vec(G->GR[p], G->V[p]), S.focus, p));
        A = base_args();
        A.mode = TM_PROX;
        A.g = vec(G->GR[p], G->V[p]);
        A.gsign = GSIGN[p];
        A.mu = S.step;
        A.center = slot2(G, G->C[p], p, 0);
        A.comb_in = slot2(G, G->S[p], p, 0);
        A.comb_out = slot2(G, G->S[p], p, 1);
        A.tau = S.tau;
        A.mask = S.focus;
        A.want = p;
        CK(tree(G, p, A));
        G->st = main_st;
    }
    if (fork_focus) {
        CK(cudaEventRecord(G->ev_join, G->st2));
        CK(cudaStreamWaitEvent(main_st, G->ev_join, 0));
    }
    if (var == EGT_AS) {
        // excessive gap at the candidate: phi_{mu_x+}(y+) and -f_{mu_y+}(x+) (refreshes the
        // caches), then the stopping test (Alg. 3 line 5) at the candidate from the same
        // gradients A y+ and A^T x+.  The two players' chains are independent: in graph mode
        // player 1's runs on a second stream (own reduction scratch) beside player 0's -- not
        // when sharded, where both chains' all-reduces must keep one order on every rank.
        const bool fork = !G->timing && !G->comm && !G->emu_world;
        if (fork) {
            CK(cudaEventRecord(G->ev_fork, main_st));
            CK(cudaStreamWaitEvent(G->st2, G->ev_fork, 0));
        }
        for (int p = 0; p < 2; ++p) {
            const int o = 1 - p;
            if (fork) G->st = p == 0 ? main_st : G->st2;
            double* partial = (fork && p == 1) ? G->partial2 : G->partial;
            unsigned* counter = (fork && p == 1) ? G->counter2 : G->counter;
            double* br_partial = (fork && p == 1) ? G->partial2_br : G->partial_br;
            unsigned* br_counter = (fork && p == 1) ? G->counter2_br : G->counter_br;
            int r = 0;
            cudaError_t e = grad(G, p, slot2(G, G->S[o], o, 1), vec(G->GR[p], G->V[p]), S.live, 1);
            if (e == cudaSuccess) {
                // one pass: the smoothed response (cache + EGV term) and the best response of
                // the same gradient (the stopping test at the candidate)
                TreeArgs A = base_args();
                A.mode = TM_SBR;
                A.g = vec(G->GR[p], G->V[p]);
                A.gsign = GSIGN[p];
                A.mu = S.mu_cand + (size_t)p * Gn;
                A.out_lb = slot2(G, G->C[p], p, 1);
                A.out_q = slot2(G, G->XQ[p], p, 1);
                A.value = S.val + (size_t)p * Gn;
                A.partial = partial;
                A.counter = counter;
                A.br_value = G->gapval + (size_t)p * Gn;
                A.br_partial = br_partial;
                A.br_counter = br_counter;
                A.mask = S.live;  // games that reached their target (egt_set_target) stop
                A.want = 1;
                e = tree(G, p, A);
            }
            G->st = main_st;
            if (e != cudaSuccess) r = fail(EGT_E_CUDA, std::string("excessive-gap check: ") + cudaGetErrorString(e));
            if (r) return r;
        }
        if (fork) {
            CK(cudaEventRecord(G->ev_join, G->st2));
            CK(cudaStreamWaitEvent(main_st, G->ev_join, 0));
        }
    }
    CK(scalar_k(G, [&] { return launch_egt_accept(var, Gn, S, G->st); }));
    return 0;
}

static int build_graph(egt_game* G, int (*rec)(egt_game*)) {
    if (G->graph) {
        cudaGraphExecDestroy(G->graph);
        G->graph = nullptr;
    }
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(G->st, cudaStreamCaptureModeThreadLocal));
    int r = rec(G);
    cudaError_t e = cudaStreamEndCapture(G->st, &graph);
    if (r) return r;
    if (e != cudaSuccess) return fail(EGT_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&G->graph, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(EGT_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    return 0;
}

static int zero_scalars(egt_game* G) {
    const int Gn = G->host.n_games;
    DevScalars& S = G->sc;
    CK(cudaMemsetAsync(S.cur, 0, sizeof(int) * Gn, G->st));
    CK(cudaMemsetAsync(S.t, 0, sizeof(int) * Gn, G->st));
    CK(cudaMemsetAsync(S.attempts, 0, sizeof(int) * Gn, G->st));
    CK(cudaMemsetAsync(S.backtracks, 0, sizeof(int) * Gn, G->st));
    CK(cudaMemsetAsync(S.fail, 0, sizeof(int) * Gn, G->st));
    CK(cudaMemsetAsync(S.egv, 0, sizeof(double) * Gn, G->st));
    std::vector<double> half(Gn, 0.5);
    CK(cudaMemcpyAsync(S.tau, half.data(), sizeof(double) * Gn, cudaMemcpyHostToDevice, G->st));
    std::vector<int> ones(Gn, 1);
    CK(cudaMemcpyAsync(S.live, ones.data(), sizeof(int) * Gn, cudaMemcpyHostToDevice, G->st));
    CK(cudaStreamSynchronize(G->st));
    return 0;
}

static int enqueue_gap(egt_game* G, int which, double* dev_out);

extern "C" int egt_init(egt_game* G, int32_t variant, double mu_x, double mu_y) {
    if (!G || variant < EGT_THEORY || variant > EGT_AS) return fail(EGT_E_ARG, "bad argument");
    const HostGame& H = G->host;
    const int Gn = H.n_games;
    Trace tr("egt_init");
    if (ensure_egt_buffers(G)) return EGT_E_CUDA;
    tr.mark("solver buffers");
    if (begin(G)) return EGT_E_CUDA;
    if (zero_scalars(G)) return EGT_E_CUDA;
    G->solver = SOLVER_EGT;
    G->variant = variant;
    if (G->graph) {
        cudaGraphExecDestroy(G->graph);
        G->graph = nullptr;
    }
    std::vector<double> mu(2 * (size_t)Gn);
    const bool given = mu_x > 0 && mu_y > 0;
    double* omega = nullptr;  // A^T x_omega once the mu search has evaluated it
    std::vector<double> mth(Gn);
    if (!given) {
        // mu_x = mu_y = ||A|| / sqrt(phi_X phi_Y), phi = 1/M
        const std::vector<double> amax = compute_max_abs_A_all(H);
        for (int g = 0; g < Gn; ++g) mth[g] = amax[g] * std::sqrt(H.M[0][g] * H.M[1][g]);
        tr.mark("max |A| (host)");
    }
    for (int g = 0; g < Gn; ++g) {
        mu[g] = given ? mu_x : mth[g];
        mu[Gn + g] = given ? mu_y : mth[g];
    }
    CK(cudaMemcpyAsync(G->sc.mu, mu.data(), sizeof(double) * 2 * Gn, cudaMemcpyHostToDevice, G->st));
    G->grads = 0;
    if (!given && variant != EGT_THEORY) {
        // DESIGN.md R14: mu = mu_theory * 2^-k with k the last of 0, 1, ..., 30 before the EGC
        // at the initial point first fails -- a plain scan, every k evaluated in turn (no
        // monotonicity assumed).  One round per k on the device for the games still scanning
        // (masked launches: a game that failed costs nothing more); the host looks at the
        // scan flags every few rounds to stop early.  A^T x_omega, independent of mu, once.
        int *scan = nullptr, *kbest = nullptr;
        double* mth_d = nullptr;
        if (dalloc(G, &scan, (size_t)Gn) || dalloc(G, &kbest, (size_t)Gn) || dalloc(G, &mth_d, 2 * (size_t)Gn))
            return EGT_E_CUDA;
        std::vector<int> ones(Gn, 1), flags(Gn, 0);
        CK(cudaMemcpyAsync(scan, ones.data(), sizeof(int) * Gn, cudaMemcpyHostToDevice, G->st));
        CK(cudaMemsetAsync(kbest, 0, sizeof(int) * Gn, G->st));
        CK(cudaMemcpyAsync(mth_d, mu.data(), sizeof(double) * 2 * Gn, cudaMemcpyHostToDevice, G->st));
        if (egt_omega_gradient(G, G->RESP[1])) return EGT_E_CUDA;  // RESP is scratch until the first step
        G->grads += 1;
        omega = G->RESP[1];
        int rounds = 0;
        for (int k = 0; k <= EGT_MU_SCAN_KMAX; ++k) {
            CK(launch_mu_scan(Gn, k, 0, mth_d, G->sc.mu, scan, kbest, G->sc.val, G->st));
            if (egt_initial_point(G, omega, scan)) return EGT_E_CUDA;
            CK(launch_mu_scan(Gn, k, 1, mth_d, G->sc.mu, scan, kbest, G->sc.val, G->st));
            ++rounds;
            if (k % 4 == 3 || k == EGT_MU_SCAN_KMAX) {
                CK(cudaMemcpyAsync(flags.data(), scan, sizeof(int) * Gn, cudaMemcpyDeviceToHost, G->st));
                CK(cudaStreamSynchronize(G->st));
                if (std::find(flags.begin(), flags.end(), 1) == flags.end()) break;
            }
        }
        G->grads += 2LL * rounds;
        CK(launch_mu_scan(Gn, 0, 2, mth_d, G->sc.mu, scan, kbest, G->sc.val, G->st));
        CK(cudaStreamSynchronize(G->st));
        for (void* q : {(void*)scan, (void*)kbest, (void*)mth_d}) {
            auto it = std::find(G->pool_allocs.begin(), G->pool_allocs.end(), q);
            if (it != G->pool_allocs.end()) {
                CK(cudaFreeAsync(*it, G->st));
                G->pool_allocs.erase(it);
            }
        }
        tr.mark("practical mu scan (device, host looks every 4 rounds)");
    }
    if (egt_initial_point(G, omega)) return EGT_E_CUDA;
    G->grads += omega ? 2 : 3;
    G->grads_per_iter = variant == EGT_AS ? 4 : 3;
    if (variant == EGT_AS) {
        int r = enqueue_gap(G, 0, G->gapcur);  // eps_sad(x0, y0); steps keep it current
        if (r) return r;
    }
    return end(G);
}

extern "C" int egt_set_target(egt_game* G, const double* host_eps) {
    if (!G) return fail(EGT_E_ARG, "null game");
    const int Gn = G->host.n_games;
    std::vector<double> t(Gn, 0.0);
    if (host_eps)
        for (int g = 0; g < Gn; ++g) t[g] = host_eps[g] > 0.0 ? host_eps[g] : 0.0;
    std::vector<int> ones(Gn, 1);
    if (begin(G)) return EGT_E_CUDA;
    CK(cudaMemcpyAsync(const_cast<double*>(G->sc.target), t.data(), sizeof(double) * Gn, cudaMemcpyHostToDevice, G->st));
    CK(cudaMemcpyAsync(G->sc.live, ones.data(), sizeof(int) * Gn, cudaMemcpyHostToDevice, G->st));
    CK(cudaStreamSynchronize(G->st));
    return end(G);
}

extern "C" int egt_step(egt_game* G, int32_t n_iters) {
    if (!G) return fail(EGT_E_ARG, "null game");
    if (G->solver != SOLVER_EGT) return fail(EGT_E_STATE, "egt_step before egt_init");
    if (n_iters <= 0) return 0;
    if (!G->timing && !G->graph && build_graph(G, record_egt_iteration)) return EGT_E_CUDA;
    if (begin(G)) return EGT_E_CUDA;
    for (int i = 0; i < n_iters; ++i) {
        if (G->timing) {
            int r = record_egt_iteration(G);
            if (r) return r;
        } else {
            CK(cudaGraphLaunch(G->graph, G->st));
        }
    }
    G->grads += (long long)G->grads_per_iter * n_iters;
    return end(G);
}

// ----------------------------------------------------------------------------- CFR
static int record_cfr_iteration(egt_game* G) {
    const int Gn = G->host.n_games;
    for (int p = 0; p < 2; ++p) {
        const int o = 1 - p;
        // Gen-CFR line 29 / 35: g = -A y^{t-1} (x), g = A^T x^t (y, alternating); games that
        // reached their target (egt_set_target) are skipped
        CK(grad(G, p, vec(G->Q[o], G->V[o]), vec(G->GR[p], G->V[p]), G->sc.live, 1));
        TreeArgs A = base_args();
        A.mode = TM_CFR;
        A.g = vec(G->GR[p], G->V[p]);
        A.gsign = p == 0 ? -1.0 : 1.0;
        A.center = vec(G->Z[p], G->V[p]);
        A.regret = vec(G->R[p], G->V[p]);
        A.out_q = vec(G->Q[p], G->V[p]);
        A.avg = vec(G->AVG[p], G->V[p]);
        A.iter = G->sc.t;
        A.cfr_plus = G->variant != CFR_RM;
        A.avg_linear = G->variant == CFR_PLUS;
        A.mask = G->sc.live;
        A.want = 1;
        CK(tree(G, p, A));
    }
    CK(scalar_k(G, [&] { return launch_tick(Gn, G->sc.t, G->sc.live, G->st); }));
    return 0;
}

extern "C" int cfr_init(egt_game* G, int32_t variant) {
    if (!G || variant < CFR_RM || variant > CFR_PLUS) return fail(EGT_E_ARG, "bad argument");
    const int Gn = G->host.n_games;
    for (int p = 0; p < 2; ++p) {
        const size_t n = (size_t)Gn * G->V[p];
        if (!G->R[p] && dalloc_vec(G, &G->R[p], n)) return EGT_E_CUDA;
        if (!G->Z[p] && dalloc_vec(G, &G->Z[p], n)) return EGT_E_CUDA;
        if (!G->Q[p] && dalloc_vec(G, &G->Q[p], n)) return EGT_E_CUDA;
        if (!G->AVG[p] && dalloc_vec(G, &G->AVG[p], n)) return EGT_E_CUDA;
    }
    if (begin(G)) return EGT_E_CUDA;
    if (zero_scalars(G)) return EGT_E_CUDA;
    if (G->graph) {
        cudaGraphExecDestroy(G->graph);
        G->graph = nullptr;
    }
    G->solver = SOLVER_CFR;
    G->variant = variant;
    G->focus_host.clear();  // timing mode counts every game of a CFR launch as active
    G->grads = 0;
    G->grads_per_iter = 2;
    std::vector<int> one(Gn, 1);
    CK(cudaMemcpyAsync(G->sc.t, one.data(), sizeof(int) * Gn, cudaMemcpyHostToDevice, G->st));
    for (int p = 0; p < 2; ++p) {
        const size_t n = (size_t)Gn * G->V[p];
        CK(cudaMemsetAsync(G->R[p], 0, n * G->esz, G->st));
        CK(cudaMemsetAsync(G->AVG[p], 0, n * G->esz, G->st));
        TreeArgs U = base_args();
        U.mode = TM_UNIFORM;  // x^0 uniform at every simplex (Gen-CFR line 1)
        U.out_b = vec(G->Z[p], G->V[p]);
        U.out_q = vec(G->Q[p], G->V[p]);
        CK(tree(G, p, U));
    }
    CK(cudaStreamSynchronize(G->st));
    return end(G);
}

extern "C" int cfr_step(egt_game* G, int32_t n_iters) {
    if (!G) return fail(EGT_E_ARG, "null game");
    if (G->solver != SOLVER_CFR) return fail(EGT_E_STATE, "cfr_step before cfr_init");
    if (n_iters <= 0) return 0;
    if (!G->timing && !G->graph && build_graph(G, record_cfr_iteration)) return EGT_E_CUDA;
    if (begin(G)) return EGT_E_CUDA;
    for (int i = 0; i < n_iters; ++i) {
        if (G->timing) {
            int r = record_cfr_iteration(G);
            if (r) return r;
        } else {
            CK(cudaGraphLaunch(G->graph, G->st));
        }
    }
    G->grads += 2LL * n_iters;
    return end(G);
}

// ----------------------------------------------------------------------------- gap / strategies
static int strategy_refs(egt_game* G, int which, VecRef out[2]) {
    if (G->solver == SOLVER_EGT) {
        out[0] = slot2(G, G->S[0], 0, 0);
        out[1] = slot2(G, G->S[1], 1, 0);
    } else if (G->solver == SOLVER_CFR) {
        for (int p = 0; p < 2; ++p) {
            double* b = which == 1 ? G->AVG[p] : which == 2 ? G->R[p] : which == 3 ? G->Z[p] : G->Q[p];
            out[p] = vec(b, G->V[p]);
        }
    } else {
        return fail(EGT_E_STATE, "no solver initialised");
    }
    return 0;
}

// eps_sad = max_y <x, A y> - min_x <x, A y>, enqueued on G->st:
// gapval[0][g] = min_x <x, A y>, gapval[1][g] = min_y <y, -A^T x>, dev_out[g] = -(both).
static int enqueue_gap(egt_game* G, int which, double* dev_out) {
    VecRef s[2];
    if (strategy_refs(G, which, s)) return EGT_E_STATE;
    const int Gn = G->host.n_games;
    for (int p = 0; p < 2; ++p) {
        CK(grad(G, p, s[1 - p], vec(G->GR[p], G->V[p])));
        TreeArgs A = base_args();
        A.mode = TM_BR;
        A.g = vec(G->GR[p], G->V[p]);
        A.gsign = GSIGN[p];
        A.value = G->gapval + (size_t)p * Gn;
        A.partial = G->partial;
        A.counter = G->counter;
        CK(tree(G, p, A));
    }
    CK(scalar_k(G, [&] { return launch_gap_combine(Gn, G->gapval, dev_out, G->st); }));
    G->grads += 2;
    return 0;
}

// EGT/as keeps eps_sad of its current iterate up to date (from the excessive-gap check's
// gradients); other solvers and the CFR averages evaluate it (2 gradients + 2 best responses).
static int gap_into(egt_game* G, int which, double* dev_out) {
    if (G->solver == SOLVER_EGT && G->variant == EGT_AS && which == 0) {
        CK(cudaMemcpyAsync(dev_out, G->gapcur, sizeof(double) * G->host.n_games, cudaMemcpyDeviceToDevice, G->st));
        return 0;
    }
    int r = enqueue_gap(G, which, dev_out);
    if (!r && G->solver == SOLVER_CFR && which == 1)
        CK(launch_stop_at_target(G->host.n_games, dev_out, G->sc.target, G->sc.live, G->st));
    return r;
}

extern "C" int saddle_gap(egt_game* G, int32_t which, double* host_out) {
    if (!G || !host_out) return fail(EGT_E_ARG, "bad argument");
    const int Gn = G->host.n_games;
    if (begin(G)) return EGT_E_CUDA;
    int r = gap_into(G, which, G->gapout);
    if (r) return r;
    CK(cudaMemcpyAsync(host_out, G->gapout, sizeof(double) * Gn, cudaMemcpyDeviceToHost, G->st));
    CK(cudaStreamSynchronize(G->st));
    return end(G);
}

extern "C" int saddle_gap_device(egt_game* G, int32_t which, double* dev_out) {
    if (!G || !dev_out) return fail(EGT_E_ARG, "bad argument");
    if (begin(G)) return EGT_E_CUDA;
    int r = gap_into(G, which, dev_out);
    if (r) return r;
    return end(G);
}

extern "C" int egt_timing(egt_game* G, int32_t enable) {
    if (!G) return fail(EGT_E_ARG, "null game");
    CK(timing_flush(G));
    for (int k = 0; k < EGT_N_KERNEL_KINDS; ++k) G->t_ms[k] = G->t_launch[k] = G->t_active[k] = G->t_bytes[k] = 0.0;
    G->timing = enable != 0;
    if (!G->timing) G->focus_host.clear();
    return 0;
}

extern "C" int egt_timing_get(egt_game* G, double* host_out) {
    if (!G || !host_out) return fail(EGT_E_ARG, "bad argument");
    CK(timing_flush(G));
    for (int k = 0; k < EGT_N_KERNEL_KINDS; ++k) {
        host_out[4 * k + 0] = G->t_ms[k];
        host_out[4 * k + 1] = G->t_launch[k];
        host_out[4 * k + 2] = G->t_active[k];
        host_out[4 * k + 3] = G->t_bytes[k];
    }
    return 0;
}

extern "C" int get_strategy_device(egt_game* G, int32_t player, int32_t which, double* dev_out) {
    if (!G || !dev_out || player < 0 || player > 1) return fail(EGT_E_ARG, "bad argument");
    VecRef s[2];
    if (strategy_refs(G, which, s)) return EGT_E_STATE;
    const int Gn = G->host.n_games;
    std::vector<int> cur(Gn, 0);
    if (begin(G)) return EGT_E_CUDA;
    if (s[player].slot_sel) {
        CK(cudaMemcpyAsync(cur.data(), G->sc.cur, sizeof(int) * Gn, cudaMemcpyDeviceToHost, G->st));
        CK(cudaStreamSynchronize(G->st));
    }
    const size_t es = (size_t)G->esz;
    for (int g = 0; g < Gn; ++g) {
        const char* src = reinterpret_cast<const char*>(s[player].base) +
                          es * ((size_t)g * G->V[player] +
                                (s[player].slot_sel ? (size_t)(cur[g] & 1) * s[player].slot_stride : 0));
        CK(cudaMemcpyAsync(reinterpret_cast<char*>(dev_out) + es * (size_t)g * G->V[player], src,
                           es * G->V[player], cudaMemcpyDeviceToDevice, G->st));
    }
    return end(G);
}

extern "C" int get_avg_strategy(egt_game* G, int32_t player, double* host_out) {
    if (!G || !host_out || player < 0 || player > 1) return fail(EGT_E_ARG, "bad argument");
    const HostGame& H = G->host;
    const int Gn = H.n_games, Hp = H.H_pad, np = H.pl[player].n_pub;
    double* tmp = nullptr;
    const size_t ne = (size_t)Gn * G->V[player];
    CK(cudaMalloc(&tmp, (size_t)G->esz * ne));
    int r = get_strategy_device(G, player, 1, tmp);
    std::vector<double> h(ne);
    std::vector<float> hf(G->esz == 4 ? ne : 0);
    if (!r) {
        cudaError_t e = G->esz == 8
                            ? cudaMemcpyAsync(h.data(), tmp, sizeof(double) * ne, cudaMemcpyDeviceToHost, G->user)
                            : cudaMemcpyAsync(hf.data(), tmp, sizeof(float) * ne, cudaMemcpyDeviceToHost, G->user);
        if (e == cudaSuccess) e = cudaStreamSynchronize(G->user);
        if (e != cudaSuccess) r = fail(EGT_E_CUDA, cudaGetErrorString(e));
    }
    cudaFree(tmp);
    if (r) return r;
    if (G->esz == 4) std::copy(hf.begin(), hf.end(), h.begin());
    const int nc = H.n_combos;
    for (int g = 0; g < Gn; ++g)
        for (int s = 0; s < np; ++s) {
            double* o = host_out + ((size_t)g * np + s) * nc;
            for (int c = 0; c < nc; ++c) o[c] = 0.0;
            for (int hh = 0; hh < H.H; ++hh)
                o[H.hand_combo[(size_t)g * H.H + hh]] = h[(size_t)g * G->V[player] + (size_t)s * Hp + hh];
        }
    return 0;
}

extern "C" int egt_scalars(egt_game* G, double* host_out) {
    if (!G || !host_out) return fail(EGT_E_ARG, "bad argument");
    const int Gn = G->host.n_games;
    std::vector<double> mu(2 * Gn), tau(Gn), egv(Gn);
    std::vector<int> t(Gn), att(Gn), bt(Gn);
    if (begin(G)) return EGT_E_CUDA;
    CK(cudaMemcpyAsync(mu.data(), G->sc.mu, sizeof(double) * 2 * Gn, cudaMemcpyDeviceToHost, G->st));
    CK(cudaMemcpyAsync(tau.data(), G->sc.tau, sizeof(double) * Gn, cudaMemcpyDeviceToHost, G->st));
    CK(cudaMemcpyAsync(egv.data(), G->sc.egv, sizeof(double) * Gn, cudaMemcpyDeviceToHost, G->st));
    CK(cudaMemcpyAsync(t.data(), G->sc.t, sizeof(int) * Gn, cudaMemcpyDeviceToHost, G->st));
    CK(cudaMemcpyAsync(att.data(), G->sc.attempts, sizeof(int) * Gn, cudaMemcpyDeviceToHost, G->st));
    CK(cudaMemcpyAsync(bt.data(), G->sc.backtracks, sizeof(int) * Gn, cudaMemcpyDeviceToHost, G->st));
    CK(cudaStreamSynchronize(G->st));
    for (int g = 0; g < Gn; ++g) {
        double* o = host_out + (size_t)g * 8;
        o[0] = mu[g];
        o[1] = mu[Gn + g];
        o[2] = tau[g];
        o[3] = t[g];
        o[4] = att[g];
        o[5] = bt[g];
        o[6] = egv[g];
        o[7] = (double)G->grads;
    }
    return end(G);
}
