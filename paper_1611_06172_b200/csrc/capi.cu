// capi.cu — the C-ABI of include/w2v.h: context, options, training driver (setup → epochs →
// sync intervals → fused step launches), embeddings I/O, statistics, debug export, and the
// NCCL data-parallel layer (dlopen'd libnccl.so.2, reading R13, C13).
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys, no-ops without a tool

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/w2v.h"
#include "w2v_internal.h"

using namespace w2v;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess) return fail(W2V_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_));  \
    } while (0)

// ------------------------------------------------------------------ NCCL (dlopen) ----------
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
    bool load() {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) return false;
        getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
        commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
        allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
        commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
        getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
        commGetAsyncError = (decltype(commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
        return getUniqueId && commInitRank && allReduce && commDestroy && getErrorString;
    }
} g_nccl;

#define NC(expr)                                                                                         \
    do {                                                                                                 \
        ncclResult_t r_ = (expr);                                                                        \
        if (r_ != ncclSuccess) return fail(W2V_ENCCL, "%s: %s", #expr, g_nccl.getErrorString(r_));      \
    } while (0)

// ------------------------------------------------------------------ context ----------------
struct Ctx {
    bool live = false;
    int device = 0, sms = 148;
    int64_t V = 0;
    int32_t D = 0, Ds = 0, window = 0, K = 0;  // Ds: half-row stride of the model (floats)
    float alpha = 0.f, t = 0.f;
    uint64_t seed = 0;
    // options
    int mode = 0;
    int32_t L = 1000;
    int64_t sync_period = 1 << 20;
    int64_t sync_hot_rows = 0;   // C14: hot prefix averaged every interval (0 = all rows)
    int64_t sync_cold_every = 1; // C14: the other rows every this many intervals (and the last)
    int sync_overlap = 0;        // C15: average in flight during the next interval (one late)
    float *syS = nullptr, *syC = nullptr;  // C15: average (S) of the snapshot (C), out of place
    int sync_device = 0;         // C17: a9 as one kernel over NCCL's symmetric window (sync_dev.cu)
    DevSync ds;                  // ... its window + device communicator (open after w2v_dist_init)
    bool M_nccl = false;         // the model lives in ncclMemAlloc memory (freed by ncclMemFree)
    bool sy_nccl = false;        // ... and so do C15's snapshot / average buffers (C17 + C15)
    unsigned long long* ds_owned = nullptr;  // floats this rank reduced in the C17 kernel (stats)
    cudaStream_t comm_stream = nullptr;
    // w2v_prefetch: up to two host corpora copied ahead on the copy stream into their own device
    // buffers; a w2v_train on the same host pointer and size consumes the oldest (FIFO)
    cudaStream_t copy_stream = nullptr;
    struct Prefetch {
        const void* host = nullptr;
        int64_t n = 0;
        uint64_t seq = 0;
        bool pending = false;
        int32_t* buf = nullptr;
        size_t cap = 0;
        cudaEvent_t done = nullptr;
    } pf[2];
    uint64_t pf_seq = 0;
    int64_t Q = 10000;
    int allow_tn = 0;
    int64_t dbg_base = 0, dbg_len = 0;
    int l2_persist = 0;          // persisting-L2 window (measured harmful: the bulk copies ignore it)
    int l2_hint = 1;             // a8 cache-policy hints on the row copies (StepParams::l2_hint)
    int64_t l2_hot_rows = -1;    // hot prefix for the hints (-1 = auto)
    int64_t l2_hot_rows_in = -1; // ... for the M_in (context) rows of the rows kernel (-1 = all)
    int64_t l2_window_rows = 0;  // hot-prefix rows under the persisting window (0 = auto)
    int64_t l2_carve_mb = 0;     // persisting-L2 carve-out, MB (0 = device maximum)
    int64_t l2_hit_pct = 100;    // hitRatio of the window, percent
    int ctas_per_sm = 0;
    int32_t epochs_total = 0;
    int32_t epoch_base = 0;  // RNG epoch field / schedule position of this call's first epoch (resume)
    int64_t launch_words = 1ll << 26;
    int64_t loss_tail_from = INT64_MAX;
    int kernel = 0;  // 0 auto, 1 per-target rows (hogbatch.cu), 2 window-resident (hogbatch_win.cu)
    int algorithm = 0;  // 0 HogBatch, 1 Alg.1 (alg1.cu)
    int rowpath_only = 0;  // measurement mode of the rows kernel (StepParams::rowpath_only)
    int ring_writeback = 0;
    int scatter_wait = 1;    // StepParams::scatter_wait  // ring kernel, deterministic mode: 0 store the slot, 1 reduce slot - original
    // device state
    cudaStream_t own_stream = nullptr, stream = nullptr;
    float* M = nullptr;  // V rows of [M_in | M_out]
    int32_t* corpus = nullptr;
    size_t corpus_cap = 0;
    unsigned long long* counts = nullptr;
    uint64_t *thr = nullptr, *P = nullptr, *scratch = nullptr;
    int32_t* G = nullptr;
    int gbits = 0;
    SetupInfo* info = nullptr;
    DevStats* dstats = nullptr;
    unsigned long long* chunk_ctr = nullptr;
    int64_t* dp_tmp = nullptr;
    uint32_t* tick = nullptr;               // mode 2: [issue 2V | done 2V] ticket counters
    uint32_t* tick_tab = nullptr;           // mode 2: per-CTA ticket tables in global memory
    size_t tick_tab_cap = 0;
    unsigned long long* turn = nullptr;     // mode 2: chunk turn of the current launch
    // batch stream of one launch range (batch.cu -> step kernels), capacity in chunks
    // two sets: the batch kernel fills set (j+1)&1 on the side stream while the step kernel
    // consumes set j&1 on the main stream
    struct BtSet {
        int32_t *nk = nullptr, *kid = nullptr, *kinfo = nullptr, *neg = nullptr;
        size_t cap_nk = 0, cap_kid = 0, cap_neg = 0;
    } bt[2];
    uint32_t* bt_redo = nullptr;
    cudaStream_t side = nullptr;
    int check_finite = 1;   // NaN/Inf scan of the model after every w2v_train (W2V_ENUMERIC)
    int tma_gather = 1;     // rows kernel: TMA tile::gather4 where step_tma_gather_ok (option)
    int overlap_batch = 0;  // option "overlap_batch" (measured slower on B200: DESIGN.md §8)
    // debug
    uint8_t *dbg_keep = nullptr, *dbg_b = nullptr, *dbg_N = nullptr;
    int32_t *dbg_ctx = nullptr, *dbg_neg = nullptr, *dbg_a1neg = nullptr;
    int64_t dbg_rec_len = 0;
    // dist
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    // stats
    w2v_stats_t st{};

} g;

void free_bt() {
    for (auto& b : g.bt) {
        cudaFree(b.nk); cudaFree(b.kid); cudaFree(b.kinfo); cudaFree(b.neg);
        b = Ctx::BtSet{};
    }
    cudaFree(g.bt_redo);
    g.bt_redo = nullptr;
}

void free_dbg() {
    cudaFree(g.dbg_keep); cudaFree(g.dbg_b); cudaFree(g.dbg_N); cudaFree(g.dbg_ctx); cudaFree(g.dbg_neg);
    cudaFree(g.dbg_a1neg);
    g.dbg_keep = g.dbg_b = g.dbg_N = nullptr;
    g.dbg_ctx = g.dbg_neg = g.dbg_a1neg = nullptr;
    g.dbg_rec_len = 0;
}

int dmalloc(void** p, size_t bytes, const char* what) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(W2V_ENOMEM, "cudaMalloc of %zu bytes for %s failed: %s", bytes, what, cudaGetErrorString(e));
    }
    return W2V_OK;
}

// batch stream buffers for `chunks` chunks of Lp slots (batch.cu layout); the negatives are
// padded by kSampGrp (8) targets because the step kernels prefetch a fixed group past nk
int ensure_bt(int64_t chunks, int32_t Lp, int32_t KS, int sets) {
    const size_t nk = (size_t)chunks, kid = (size_t)chunks * Lp, neg = (size_t)chunks * Lp * KS + 8 * (size_t)KS;
    int rc;
    for (int si = 0; si < sets; ++si) {
        auto& b = g.bt[si];
        if (nk > b.cap_nk) {
            cudaFree(b.nk); b.nk = nullptr; b.cap_nk = 0;
            if ((rc = dmalloc((void**)&b.nk, nk * 4, "batch stream (kept counts)"))) return rc;
            b.cap_nk = nk;
        }
        if (kid > b.cap_kid) {
            cudaFree(b.kid); cudaFree(b.kinfo); b.kid = b.kinfo = nullptr; b.cap_kid = 0;
            if ((rc = dmalloc((void**)&b.kid, kid * 4, "batch stream (kept words)"))) return rc;
            if ((rc = dmalloc((void**)&b.kinfo, kid * 4, "batch stream (offsets, b)"))) return rc;
            b.cap_kid = kid;
        }
        if (neg > b.cap_neg) {
            cudaFree(b.neg); b.neg = nullptr; b.cap_neg = 0;
            if ((rc = dmalloc((void**)&b.neg, neg * 4, "batch stream (negatives)"))) return rc;
            b.cap_neg = neg;
        }
    }
    if (!g.bt_redo && (rc = dmalloc((void**)&g.bt_redo, batch_redo_words(g.sms) * 4, "batch kernel scratch"))) return rc;
    return W2V_OK;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// NVTX range for the host-side phases of a call (SURVEY.md §5 tracing); pops on every exit path.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Every CUDA event of one w2v_train call; destroyed on every exit path (errors included).
struct EventPool {
    std::vector<cudaEvent_t> v;
    cudaError_t make(cudaEvent_t* e, unsigned flags = cudaEventDefault) {
        cudaError_t r = cudaEventCreateWithFlags(e, flags);
        if (r == cudaSuccess) v.push_back(*e);
        return r;
    }
    ~EventPool() {
        for (auto e : v) cudaEventDestroy(e);
    }
};

// a8 option l2_persist: the persisting-L2 carve-out and the stream's access-policy window are
// process-wide state; undo both (window off, persisting lines reset, previous limit) on every
// exit path of w2v_train so later calls and other work get the whole L2 back.
struct L2WindowGuard {
    bool window_set = false, limit_set = false;
    size_t prev_limit = 0;
    cudaStream_t stream = nullptr;
    ~L2WindowGuard() {
        if (window_set) {
            cudaStreamAttrValue a{};
            a.accessPolicyWindow.num_bytes = 0;
            cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &a);
            cudaCtxResetPersistingL2Cache();
        }
        if (limit_set) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev_limit);
        cudaGetLastError();
    }
};

// C13 host plan
struct Plan {
    int64_t S, lo, hi, start, end, J, I;
};
Plan make_plan(int64_t n, int32_t L, int32_t W, int32_t r, int64_t P) {
    Plan p{};
    p.S = (n + L - 1) / L;
    p.lo = (int64_t)r * p.S / W;
    p.hi = ((int64_t)r + 1) * p.S / W;
    p.start = p.lo * L;
    p.end = std::min(p.hi * L, n);
    p.I = std::max<int64_t>(1, P / L);
    int64_t mins = INT64_MAX;
    for (int q = 0; q < W; ++q) mins = std::min(mins, ((int64_t)q + 1) * p.S / W - (int64_t)q * p.S / W);
    p.J = std::max<int64_t>(1, mins / p.I);
    return p;
}

// The data-parallel path runs whenever a communicator exists: world > 1, or a 1-rank NCCL
// communicator created by w2v_dist_init(0, 1, id) (test hook: exercises every collective on one
// GPU; averaging over one replica is the identity).
bool dp() { return g.comm != nullptr; }

// a9: replace rows [row_lo, row_hi) of both matrices (one contiguous range of the interleaved
// model) by their mean over ranks
int sync_models(int64_t row_lo = 0, int64_t row_hi = -1, int* launches = nullptr) {
    if (!dp()) return W2V_OK;
    NvtxRange nvtx("a9 model average");
    if (row_hi < 0) row_hi = g.V;
    if (row_hi <= row_lo) return W2V_OK;
    if (g.ds.devcomm) {  // C17: one kernel, in place over the symmetric window (sync_dev.cu)
        CU(devsync_launch(g.ds, 0, 0, (size_t)row_lo * 2 * g.Ds, (size_t)(row_hi - row_lo) * 2 * g.Ds, g.ds_owned,
                          kDevSyncCtas, g.stream));
        if (launches) ++*launches;
    } else {
        NC(g_nccl.allReduce(g.M + (size_t)row_lo * 2 * g.Ds, g.M + (size_t)row_lo * 2 * g.Ds,
                            (size_t)(row_hi - row_lo) * 2 * g.Ds, ncclFloat32, ncclAvg, g.comm, g.stream));
    }
    if (row_lo == 0 && row_hi == g.V) g.st.syncs += 1;
    else g.st.syncs_hot += 1;
    if (g_nccl.commGetAsyncError) {  // a peer that failed surfaces here instead of as a hang later
        ncclResult_t ae = ncclSuccess;
        NC(g_nccl.commGetAsyncError(g.comm, &ae));
        NC(ae);
    }
    return W2V_OK;
}

// Data-parallel error consensus: every rank passes its local status; if any rank failed, all
// ranks return (the failing ones their own error, the others W2V_EPEER) instead of leaving peers
// blocked in the next collective (DESIGN.md §2 C13). No-op without a communicator.
int dp_agree(int rc_local, cudaStream_t st) {
    if (!dp()) return rc_local;
    const std::string own = g_err;
    std::vector<int64_t> h(g.world, 0);
    h[g.rank] = rc_local != 0 ? 1 : 0;
    CU(cudaMemcpyAsync(g.dp_tmp, h.data(), (size_t)g.world * 8, cudaMemcpyHostToDevice, st));
    NC(g_nccl.allReduce(g.dp_tmp, g.dp_tmp, (size_t)g.world, ncclInt64, ncclSum, g.comm, st));
    CU(cudaMemcpyAsync(h.data(), g.dp_tmp, (size_t)g.world * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (rc_local != 0) { g_err = own; return rc_local; }
    for (int q = 0; q < g.world; ++q)
        if (h[q]) return fail(W2V_EPEER, "w2v_train: rank %d failed during setup; nothing trained on any rank", q);
    return W2V_OK;
}

}  // namespace

extern "C" {

const char* w2v_last_error(void) { return g_err.c_str(); }

int w2v_init(int64_t V, int32_t D, int32_t window, int32_t K, float alpha, float subsample, uint64_t seed) {
    if (g.live) return fail(W2V_ESTATE, "w2v_init: already initialised (call w2v_finalize first)");
    if (V < 1 || V > 2147483647ll) return fail(W2V_EINVAL, "w2v_init: V=%lld out of [1, 2^31)", (long long)V);
    if (D < 4 || D % 4 != 0 || D > 512) return fail(W2V_EINVAL, "w2v_init: D=%d must be a multiple of 4 in [4,512]", D);
    if (window < 1 || window > 254) return fail(W2V_EINVAL, "w2v_init: window=%d out of [1,254]", window);
    if (K < 0 || K > 31) return fail(W2V_EINVAL, "w2v_init: K=%d out of [0,31]", K);
    if (!(alpha > 0.f) || !std::isfinite(alpha)) return fail(W2V_EINVAL, "w2v_init: alpha must be > 0");
    if (!(subsample >= 0.f) || !std::isfinite(subsample)) return fail(W2V_EINVAL, "w2v_init: subsample must be >= 0");
    if (!step_supported(D, K)) return fail(W2V_EINVAL, "w2v_init: (D=%d, K=%d) exceeds the register tiles (DESIGN.md §8)", D, K);
    Ctx fresh;
    g = fresh;
    CU(cudaGetDevice(&g.device));
    CU(cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, g.device));
    g.V = V; g.D = D; g.window = window;
    {   // model layout: each half-row padded to 128 B (W2V_ROW_ALIGN=0 packs them; experiment)
        const char* ra = getenv("W2V_ROW_ALIGN");
        const bool align = !(ra && ra[0] == '0');
        g.Ds = align ? (D + 31) / 32 * 32 : D;
    } g.K = K; g.alpha = alpha; g.t = subsample; g.seed = seed;
    CU(cudaStreamCreateWithFlags(&g.own_stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&g.side, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&g.comm_stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&g.copy_stream, cudaStreamNonBlocking));
    for (auto& f : g.pf) CU(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming));
    g.stream = g.own_stream;
    int rc;
    if ((rc = dmalloc((void**)&g.M, (size_t)V * 2 * g.Ds * sizeof(float), "the model [M_in|M_out]"))) return rc;
    CU(cudaMemsetAsync(g.M, 0, (size_t)V * 2 * g.Ds * sizeof(float), g.stream));  // padding stays 0
    if ((rc = dmalloc((void**)&g.counts, (size_t)V * 8, "counts"))) return rc;
    if ((rc = dmalloc((void**)&g.thr, (size_t)V * 8, "keep thresholds"))) return rc;
    if ((rc = dmalloc((void**)&g.P, (size_t)(V + 1) * 8, "sampler prefix"))) return rc;
    const int64_t nb = (V + 2047) / 2048;
    if ((rc = dmalloc((void**)&g.scratch, (size_t)(nb + 1) * 8, "scan scratch"))) return rc;
    g.gbits = 1;
    while ((1ll << g.gbits) < V) ++g.gbits;
    g.gbits += 1;
    if ((rc = dmalloc((void**)&g.G, (size_t)((1ll << g.gbits) + 2) * 4, "guide table"))) return rc;
    if ((rc = dmalloc((void**)&g.info, sizeof(SetupInfo), "setup info"))) return rc;
    if ((rc = dmalloc((void**)&g.dstats, sizeof(DevStats), "stats"))) return rc;
    if ((rc = dmalloc((void**)&g.chunk_ctr, 64, "chunk counter"))) return rc;
    CU(launch_init(g.M, V, D, g.Ds, seed, g.sms, g.stream));
    CU(cudaStreamSynchronize(g.stream));
    g.live = true;
    return W2V_OK;
}

int w2v_set_option(const char* key, int64_t v) {
    if (!g.live) return fail(W2V_ESTATE, "w2v_set_option before w2v_init");
    if (!key) return fail(W2V_EINVAL, "w2v_set_option: null key");
    std::string k(key);
    if (k == "mode") { if (v < 0 || v > 2) return fail(W2V_EINVAL, "mode must be 0 (Hogwild), 1 (deterministic, one unit) or 2 (deterministic, conflict-ticketed)"); g.mode = (int)v; }
    else if (k == "sentence_len") { if (v < 1 || v > 4096) return fail(W2V_EINVAL, "sentence_len out of [1,4096]"); g.L = (int32_t)v; }
    else if (k == "sync_period_words") { if (v < 1) return fail(W2V_EINVAL, "sync_period_words must be >= 1"); g.sync_period = v; }
    else if (k == "sync_hot_rows") { if (v < 0) return fail(W2V_EINVAL, "sync_hot_rows must be >= 0"); g.sync_hot_rows = v; }
    else if (k == "sync_cold_every") { if (v < 1) return fail(W2V_EINVAL, "sync_cold_every must be >= 1"); g.sync_cold_every = v; }
    else if (k == "sync_device") {
        if (v != 0 && v != 1) return fail(W2V_EINVAL, "sync_device must be 0/1");
        if (g.comm) return fail(W2V_ESTATE, "sync_device must be set before w2v_dist_init (it places the model in NCCL symmetric memory)");
        g.sync_device = (int)v;
    }
    else if (k == "sync_overlap") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "sync_overlap must be 0/1"); g.sync_overlap = (int)v; }
    else if (k == "lr_quantum") { if (v < 1) return fail(W2V_EINVAL, "lr_quantum must be >= 1"); g.Q = v; }
    else if (k == "allow_target_negative") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "allow_target_negative must be 0/1"); g.allow_tn = (int)v; }
    else if (k == "debug_base") { if (v < 0) return fail(W2V_EINVAL, "debug_base must be >= 0"); g.dbg_base = v; }
    else if (k == "debug_len") { if (v < 0) return fail(W2V_EINVAL, "debug_len must be >= 0"); g.dbg_len = v; }
    else if (k == "l2_persist") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "l2_persist must be 0/1"); g.l2_persist = (int)v; }
    else if (k == "l2_hint") { if (v < 0 || v > 3) return fail(W2V_EINVAL, "l2_hint out of [0,3]"); g.l2_hint = (int)v; }
    else if (k == "l2_hot_rows_in") { if (v < -1) return fail(W2V_EINVAL, "l2_hot_rows_in must be >= -1"); g.l2_hot_rows_in = v; }
    else if (k == "l2_hot_rows") { if (v < -1) return fail(W2V_EINVAL, "l2_hot_rows must be >= -1"); g.l2_hot_rows = v; }
    else if (k == "l2_window_rows") { if (v < 0) return fail(W2V_EINVAL, "l2_window_rows must be >= 0"); g.l2_window_rows = v; }
    else if (k == "l2_carve_mb") { if (v < 0) return fail(W2V_EINVAL, "l2_carve_mb must be >= 0"); g.l2_carve_mb = v; }
    else if (k == "l2_hit_pct") { if (v < 1 || v > 100) return fail(W2V_EINVAL, "l2_hit_pct out of [1,100]"); g.l2_hit_pct = v; }
    else if (k == "ctas_per_sm") { if (v < 0 || v > 32) return fail(W2V_EINVAL, "ctas_per_sm out of [0,32]"); g.ctas_per_sm = (int)v; }
    else if (k == "loss_tail_from") { if (v < 0) return fail(W2V_EINVAL, "loss_tail_from must be >= 0"); g.loss_tail_from = v; }
    else if (k == "algorithm") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "algorithm must be 0 (HogBatch) or 1 (Alg.1)"); g.algorithm = (int)v; }
    else if (k == "rowpath_only") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "rowpath_only must be 0/1"); g.rowpath_only = (int)v; }
    else if (k == "scatter_wait") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "scatter_wait must be 0/1"); g.scatter_wait = (int)v; }
    else if (k == "ring_writeback") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "ring_writeback must be 0/1"); g.ring_writeback = (int)v; }
    else if (k == "tma_gather") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "tma_gather must be 0/1"); g.tma_gather = (int)v; }
    else if (k == "check_finite") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "check_finite must be 0/1"); g.check_finite = (int)v; }
    else if (k == "overlap_batch") { if (v != 0 && v != 1) return fail(W2V_EINVAL, "overlap_batch must be 0/1"); g.overlap_batch = (int)v; }
    else if (k == "kernel") { if (v < 0 || v > 4) return fail(W2V_EINVAL, "kernel must be 0 (auto), 1 (rows), 2 (window), 3 (window, warp-specialised) or 4 (ring, TMEM originals)"); g.kernel = (int)v; }
    else if (k == "launch_words") { if (v < 1 || v > (1ll << 31)) return fail(W2V_EINVAL, "launch_words out of [1, 2^31]"); g.launch_words = v; }
    else if (k == "epoch_base") { if (v < 0 || v > 255) return fail(W2V_EINVAL, "epoch_base out of [0,255]"); g.epoch_base = (int32_t)v; }
    else if (k == "epochs_total") { if (v < 0) return fail(W2V_EINVAL, "epochs_total must be >= 0"); g.epochs_total = (int32_t)v; }
    else return fail(W2V_EINVAL, "w2v_set_option: unknown key '%s'", key);
    return W2V_OK;
}

int w2v_set_stream(void* s) {
    if (!g.live) return fail(W2V_ESTATE, "w2v_set_stream before w2v_init");
    g.stream = s ? (cudaStream_t)s : g.own_stream;
    return W2V_OK;
}

int w2v_train(const int32_t* ids_in, int64_t n, int32_t epochs) {
    NvtxRange nvtx_train("w2v_train");
    if (!g.live) return fail(W2V_ESTATE, "w2v_train before w2v_init");
    if (epochs < 1) return fail(W2V_EINVAL, "w2v_train: epochs=%d must be >= 1", epochs);
    if (n < 0) return fail(W2V_EINVAL, "w2v_train: n_tokens < 0");
    g.st.launches = 0;
    g.st.ms_total = g.st.ms_step = g.st.ms_setup = g.st.ms_sync = g.st.ms_h2d = g.st.ms_batch = 0;
    g.st.step_launches = 0;
    g.st.bytes_row = 0;
    // the union of the shards may be non-empty while this rank's shard is empty: only a
    // world-1 empty corpus is a pure no-op
    if (n == 0 && !dp()) return W2V_OK;
    if (!ids_in && n > 0) return fail(W2V_EINVAL, "w2v_train: null corpus");
    cudaStream_t st = g.stream;
    int launches = 0;
    cudaEvent_t ev0, ev_h2d, ev_setup, ev_end;
    EventPool pool;
    CU(pool.make(&ev0)); CU(pool.make(&ev_h2d)); CU(pool.make(&ev_setup)); CU(pool.make(&ev_end));
    CU(cudaEventRecord(ev0, st));
    // ---- corpus placement
    const int32_t* ids = ids_in;
    int local_fail = 0;  // a rank-local failure before the first collective (reported through it)
    if (n > 0 && !is_device_ptr(ids_in)) {
        Ctx::Prefetch* hit = nullptr;  // the oldest pending prefetch of this corpus (w2v_prefetch)
        for (auto& f : g.pf)
            if (f.pending && f.host == (const void*)ids_in && f.n == n && (!hit || f.seq < hit->seq)) hit = &f;
        if (hit) {   // its H2D copy ran on the copy stream, overlapped with earlier work
            CU(cudaStreamWaitEvent(st, hit->done, 0));
            hit->pending = false;
            ids = hit->buf;
        } else {
            if ((size_t)n > g.corpus_cap) {
                cudaFree(g.corpus);
                g.corpus = nullptr;
                g.corpus_cap = 0;
                local_fail = dmalloc((void**)&g.corpus, (size_t)n * 4, "the device copy of a host corpus");
                if (local_fail && !dp()) return local_fail;
                if (!local_fail) g.corpus_cap = (size_t)n;
            }
            if (!local_fail) {
                CU(cudaMemcpyAsync(g.corpus, ids_in, (size_t)n * 4, cudaMemcpyHostToDevice, st));
                ids = g.corpus;
            }
        }
    }
    CU(cudaEventRecord(ev_h2d, st));
    // ---- a0: shard geometry (C13), counts, thresholds, sampler
    int64_t n_global = n, shard_start = 0;
    bool bad_shard = false;
    if (dp()) {
        if (!g.dp_tmp) { int rc = dmalloc((void**)&g.dp_tmp, (size_t)g.world * 8, "dp scratch"); if (rc) return rc; }
        std::vector<int64_t> h(g.world, 0);
        h[g.rank] = local_fail ? -1 : n;   // -1: this rank failed before the collectives
        CU(cudaMemcpyAsync(g.dp_tmp, h.data(), (size_t)g.world * 8, cudaMemcpyHostToDevice, st));
        NC(g_nccl.allReduce(g.dp_tmp, g.dp_tmp, (size_t)g.world, ncclInt64, ncclSum, g.comm, st));
        CU(cudaMemcpyAsync(h.data(), g.dp_tmp, (size_t)g.world * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (local_fail) return local_fail;
        for (int q = 0; q < g.world; ++q)
            if (h[q] < 0) return fail(W2V_EPEER, "w2v_train: rank %d failed to place its corpus; nothing trained", q);
        n_global = 0;
        for (int q = 0; q < g.world; ++q) { if (q < g.rank) shard_start += h[q]; n_global += h[q]; }
        if (n_global == 0) return W2V_OK;
        const Plan pl = make_plan(n_global, g.L, g.world, g.rank, g.sync_period);
        if (pl.start != shard_start || pl.end - pl.start != n) {
            // rank-local error: reported after the setup collectives below, which every rank
            // still joins, so no peer is left blocked
            bad_shard = true;
            fail(W2V_EINVAL, "w2v_train: rank %d shard [%lld,%lld) is not the C13 shard [%lld,%lld) of n=%lld, L=%d",
                 g.rank, (long long)shard_start, (long long)(shard_start + n), (long long)pl.start,
                 (long long)pl.end, (long long)n_global, g.L);
        }
    }
    CU(cudaMemsetAsync(g.counts, 0, (size_t)g.V * 8, st));
    CU(cudaMemsetAsync(g.info, 0, sizeof(SetupInfo), st));
    CU(launch_hist(ids, n, g.V, g.counts, g.info, g.sms, st, &launches));
    if (dp()) NC(g_nccl.allReduce(g.counts, g.counts, (size_t)g.V, ncclUint64, ncclSum, g.comm, st));
    CU(launch_tables(g.counts, g.V, n_global, g.t, g.thr, g.P, g.scratch, g.G, g.gbits, g.info, st, &launches));
    SetupInfo hinfo{};
    CU(cudaMemcpyAsync(&hinfo, g.info, sizeof hinfo, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (dp()) {
        // every rank must take the same exit: combine the bad-id and bad-shard flags
        std::vector<int64_t> h(g.world, 0);
        h[g.rank] = hinfo.bad_id | (bad_shard ? 2 : 0);
        CU(cudaMemcpyAsync(g.dp_tmp, h.data(), (size_t)g.world * 8, cudaMemcpyHostToDevice, st));
        NC(g_nccl.allReduce(g.dp_tmp, g.dp_tmp, (size_t)g.world, ncclInt64, ncclSum, g.comm, st));
        CU(cudaMemcpyAsync(h.data(), g.dp_tmp, (size_t)g.world * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (bad_shard) return W2V_EINVAL;  // message set above
        for (int q = 0; q < g.world; ++q) {
            hinfo.bad_id |= (int)(h[q] & 1);
            if (h[q] & 2) return fail(W2V_EPEER, "w2v_train: rank %d passed a shard that is not its C13 shard", q);
        }
    }
    if (hinfo.bad_id) return fail(W2V_EINVAL, "w2v_train: corpus contains an id outside [0,%lld); nothing trained", (long long)g.V);
    if (hinfo.PV == 0) return fail(W2V_EINVAL, "w2v_train: sampler mass P[V] is 0");
    CU(cudaEventRecord(ev_setup, st));
    // Everything from here to the first step launch may fail on one rank only (allocation,
    // occupancy): with a communicator, every exit of this region goes through one consensus
    // collective (dp_agree), so a failing rank never leaves its peers blocked in an all-reduce.
    auto bail = [&](int rc) -> int { return dp() ? dp_agree(rc, st) : rc; };
#define CUB(expr)                                                                                 \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess) return bail(fail(W2V_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_))); \
    } while (0)
    // ---- debug buffers
    free_dbg();
    if (g.dbg_len > 0) {
        const int64_t Lq = g.dbg_len, kk = g.K > 0 ? g.K : 1;
        int rc;
        if ((rc = dmalloc((void**)&g.dbg_keep, Lq, "debug keep"))) return bail(rc);
        if ((rc = dmalloc((void**)&g.dbg_b, Lq, "debug b"))) return bail(rc);
        if ((rc = dmalloc((void**)&g.dbg_N, Lq, "debug N"))) return bail(rc);
        if ((rc = dmalloc((void**)&g.dbg_ctx, (size_t)Lq * 2 * g.window * 4, "debug ctx"))) return bail(rc);
        if ((rc = dmalloc((void**)&g.dbg_neg, (size_t)Lq * kk * 4, "debug neg"))) return bail(rc);
        CUB(cudaMemsetAsync(g.dbg_keep, 0, Lq, st));
        CUB(cudaMemsetAsync(g.dbg_b, 0, Lq, st));
        CUB(cudaMemsetAsync(g.dbg_N, 0, Lq, st));
        CUB(cudaMemsetAsync(g.dbg_ctx, 0xff, (size_t)Lq * 2 * g.window * 4, st));
        CUB(cudaMemsetAsync(g.dbg_neg, 0xff, (size_t)Lq * kk * 4, st));
        if (g.algorithm == 1) {
            if ((rc = dmalloc((void**)&g.dbg_a1neg, (size_t)Lq * 2 * g.window * kk * 4, "debug Alg.1 negatives"))) return bail(rc);
            CUB(cudaMemsetAsync(g.dbg_a1neg, 0xff, (size_t)Lq * 2 * g.window * kk * 4, st));
        }
        g.dbg_rec_len = Lq;
    }
    // ---- a8: persisting-L2 window over the hot prefix rows of [M_in|M_out] (option; measured
    // harmful). The carve-out limit and the stream window are restored on every exit path.
    L2WindowGuard l2guard;
    bool& window_set = l2guard.window_set;
    g.st.l2_window_bytes = g.st.l2_carve_bytes = 0;
    if (g.l2_persist && g.mode == 0) {
        int maxp = 0, maxwin = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, g.device);
        cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, g.device);
        if (maxp > 0 && maxwin > 0) {
            const size_t rowb = (size_t)2 * g.Ds * 4;
            size_t carve = g.l2_carve_mb > 0 ? std::min<size_t>((size_t)g.l2_carve_mb << 20, (size_t)maxp) : (size_t)maxp;
            size_t bytes = g.l2_window_rows > 0 ? (size_t)g.l2_window_rows * rowb : carve;
            bytes = std::min<size_t>(bytes, (size_t)maxwin);
            bytes = std::min<size_t>(bytes, (size_t)g.V * rowb);
            size_t prev = 0;
            if (cudaDeviceGetLimit(&prev, cudaLimitPersistingL2CacheSize) == cudaSuccess &&
                cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve) == cudaSuccess) {
                l2guard.limit_set = true;
                l2guard.prev_limit = prev;
                l2guard.stream = st;
                cudaStreamAttrValue a{};
                a.accessPolicyWindow.base_ptr = g.M;
                a.accessPolicyWindow.num_bytes = bytes;
                a.accessPolicyWindow.hitRatio = (float)g.l2_hit_pct / 100.0f;
                a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                window_set = cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a) == cudaSuccess;
            }
            g.st.l2_window_bytes = window_set ? (int64_t)bytes : 0;
            g.st.l2_carve_bytes = window_set ? (int64_t)carve : 0;
        }
        cudaGetLastError();
    }
    // ---- epochs × sync intervals of fused steps
    StepParams p{};
    p.ids = ids;
    p.ids_base = shard_start;
    p.shard_start = shard_start;
    p.n_local = n;
    p.n_global = n_global;
    p.L = g.L; p.window = g.window; p.K = g.K; p.D = g.D; p.Ds = g.Ds;
    p.epochs = g.epochs_total > 0 ? g.epochs_total : epochs;
    p.world = g.world;
    p.allow_tn = g.allow_tn;
    p.deterministic = g.mode;
    p.alpha0 = g.alpha; p.Q = g.Q; p.seed = g.seed; p.V = g.V;
    p.thr = g.thr; p.P = g.P; p.G = g.G; p.info = g.info; p.M = g.M;
    p.chunk_ctr = g.chunk_ctr; p.stats = g.dstats;
    p.loss_tail_from = g.loss_tail_from;
    p.l2_hint = g.l2_hint;
    p.hot_rows = g.l2_hot_rows >= 0 ? g.l2_hot_rows : (int64_t)(64ll << 20) / ((int64_t)2 * g.Ds * 4);
    // a chunk's context rows are re-read by its next targets within microseconds: all M_in rows
    // get evict_last by default (profiles/r01_ablations.md §2)
    p.hot_rows_in = g.l2_hot_rows_in >= 0 ? g.l2_hot_rows_in : g.V;
    p.dbg_base = g.dbg_base; p.dbg_len = g.dbg_len;
    p.dbg_keep = g.dbg_keep; p.dbg_b = g.dbg_b; p.dbg_N = g.dbg_N; p.dbg_ctx = g.dbg_ctx; p.dbg_neg = g.dbg_neg;
    p.dbg_a1neg = g.dbg_a1neg;
    p.algorithm = g.algorithm;
    p.rowpath_only = g.rowpath_only;
    p.ring_delta = g.ring_writeback;
    p.scatter_wait = g.scatter_wait;
    // rows kernel gathers through TMA tile::gather4 (4 rows per instruction) where the slab
    // layout allows it: the model as a 2-D fp32 tensor [V][2*Ds], box D x 1
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof tmap);
    p.tma_gather = 0;
    if (g.tma_gather && g.algorithm == 0 && step_tma_gather_ok(g.D, g.K, g.window)) {
        typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        static Encode encode = nullptr;
        if (!encode) {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess)
                encode = (Encode)fn;
            cudaGetLastError();
        }
        const cuuint64_t dims[2] = {(cuuint64_t)2 * g.Ds, (cuuint64_t)g.V};
        const cuuint64_t strides[1] = {(cuuint64_t)2 * g.Ds * sizeof(float)};
        const cuuint32_t box[2] = {(cuuint32_t)g.D, 1}, es[2] = {1, 1};
        if (encode && encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g.M, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
            p.tma_gather = 1;
    }
    {   // cache-aware roofline statistics: the hot prefix whose half-rows of both matrices fill L2
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g.device);
        p.cold_from = (int64_t)l2 / ((int64_t)8 * g.D);
        g.st.cold_from_row = p.cold_from;
    }
    if (g.rowpath_only && (g.algorithm != 0 || g.kernel == 2 || g.kernel == 3))
        return bail(fail(W2V_EINVAL, "w2v_train: rowpath_only applies to the rows and ring kernels (kernel 0/1/4, algorithm 0)"));
    if (g.algorithm == 1 && !alg1_supported(g.D, g.K))
        return bail(fail(W2V_EINVAL, "w2v_train: Alg.1 kernel does not cover D=%d, K=%d", g.D, g.K));
    // kernel choice: 1 per-target rows, 2 window-resident (one warp per unit),
    // 3 window-resident warp-specialised (a CTA of column warps + an IO warp per unit)
    const size_t kSmemMax = 227 * 1024;
    int32_t off_win = 0, off_row = 0, off_wg = 0;
    const size_t wb_win = win_warp_bytes(g.L, g.window, g.K, g.D, &off_win);
    int32_t off_tick = 0;
    size_t wb_row = step_warp_bytes(g.L, g.window, g.K, g.D, &off_row, g.mode == 2 ? &off_tick : nullptr);
    if (g.mode == 2 && wb_row > kSmemMax) {  // the ticket table goes to global memory instead
        wb_row = step_warp_bytes(g.L, g.window, g.K, g.D, &off_row, nullptr);
        off_tick = -1;
    }
    const size_t wb_wg = wg_cta_bytes(g.L, g.window, g.K, g.D, &off_wg);
    int32_t off_ring = 0;
    const size_t wb_ring = ring_warp_bytes(g.L, g.window, g.K, g.D, &off_ring);
    int kern = g.kernel == 0 ? 1 : g.kernel;
    if (g.algorithm == 1) kern = 0;  // alg1.cu
    if (g.mode == 2) {  // NEXT-4: the rows kernel with per-row tickets (hogbatch.cu)
        if (kern != 1 || 2 * g.window + g.K + 1 > 32)
            return bail(fail(W2V_EINVAL, "w2v_train: mode 2 (conflict-ticketed) needs the rows kernel (kernel 0/1, "
                             "algorithm 0) and 2*window+K+1 <= 32"));
        if (!g.tick) {
            int rc = dmalloc((void**)&g.tick, (size_t)g.V * 4 * sizeof(uint32_t), "mode-2 ticket counters");
            if (rc) return bail(rc);
            rc = dmalloc((void**)&g.turn, 64, "mode-2 chunk turn");
            if (rc) return bail(rc);
        }
        CUB(cudaMemsetAsync(g.tick, 0, (size_t)g.V * 4 * sizeof(uint32_t), st));
        p.tick_issue = g.tick;
        p.tick_done = g.tick + 2 * g.V;
        p.turn = g.turn;
        p.tick_off = off_tick;
    }
    int ring_units = 0;  // kernel 4: work units (warps) per CTA, one CTA per SM
    if (kern == 4) {
        ring_units = g.mode == 1 ? 1 : ring_units_per_cta(g.window, g.D, g.K, wb_ring, kSmemMax);
        if (g.mode == 0 && g.ctas_per_sm > 0 && g.ctas_per_sm < ring_units) ring_units = g.ctas_per_sm;
        if (!ring_supported(g.window, g.D, g.K) || wb_ring == 0 || ring_units < 1)
            return bail(fail(W2V_EINVAL, "w2v_train: kernel=4 (ring) unsupported for window=%d, D=%d, K=%d, L=%d (window <= 15)",
                             g.window, g.D, g.K, g.L));
    }
    if (kern == 2 && !(wb_win > 0 && wb_win <= kSmemMax))
        return bail(fail(W2V_EINVAL, "w2v_train: kernel=2 (window) unsupported for window=%d, D=%d, K=%d, L=%d", g.window, g.D, g.K, g.L));
    if (kern == 3 && !(wb_wg > 0 && wb_wg <= kSmemMax))
        return bail(fail(W2V_EINVAL, "w2v_train: kernel=3 (window, warp-specialised) unsupported for window=%d, D=%d, K=%d, L=%d", g.window, g.D, g.K, g.L));
    const bool use_win = kern == 2;
    size_t wb = kern == 4 ? wb_ring : kern == 3 ? wb_wg : use_win ? wb_win : wb_row;
    if (kern == 0) wb = alg1_warp_bytes(g.L);
    p.slab_offset = kern == 4 ? off_ring : kern == 3 ? off_wg : use_win ? off_win : off_row;
    if (wb == 0 || wb > kSmemMax) return bail(fail(W2V_EINVAL, "w2v_train: shared memory per work unit %zu B exceeds 227 KB (reduce sentence_len/window/K/D)", wb));
    p.warp_bytes = (int32_t)wb;
    int ctas = 1;
    if (kern == 4) {
        ctas = g.mode == 0 ? g.sms : 1;   // one CTA of ring_units warps per SM (its TMEM block)
    } else if (g.mode != 1) {
        int occ = kern == 0 ? alg1_max_ctas_per_sm(p) : kern == 3 ? wg_max_ctas_per_sm(p)
                : use_win ? win_max_ctas_per_sm(p) : step_max_ctas_per_sm(p);
        if (occ < 1) return bail(fail(W2V_ECUDA, "w2v_train: step kernel cannot be resident (%zu B smem per work unit)", wb));
        if (g.ctas_per_sm > 0 && g.ctas_per_sm < occ) occ = g.ctas_per_sm;
        ctas = g.sms * occ;
    }
    if (g.mode == 2 && off_tick < 0) {  // global ticket tables, one per CTA of this launch grid
        const size_t need = (size_t)ctas * ((g.L + 3) & ~3) * (2 * g.window + g.K + 1);
        if (need > g.tick_tab_cap) {
            cudaFree(g.tick_tab);
            g.tick_tab = nullptr;
            g.tick_tab_cap = 0;
            int rc = dmalloc((void**)&g.tick_tab, need * sizeof(uint32_t), "mode-2 ticket tables");
            if (rc) return bail(rc);
            g.tick_tab_cap = need;
        }
    }
    p.tick_glob = g.tick_tab;
    g.st.units_per_sm = kern == 4 ? ring_units : ctas >= g.sms ? ctas / g.sms : 1;
    // stats: 1 rows, 2 window, 3 window warp-specialised, 4 alg1, 5 ring
    g.st.kernel = kern == 0 ? 4 : kern == 4 ? 5 : kern;
    CUB(cudaMemsetAsync(g.dstats, 0, sizeof(DevStats), st));
    const Plan pl = make_plan(n_global, g.L, g.world, g.rank, g.sync_period);
    const int64_t chunk_lo = shard_start / g.L;
    const int64_t chunk_hi = (shard_start + n + g.L - 1) / g.L;
    // an interval is issued as launches of at most launch_words raw words (bounded kernel
    // duration and batch-stream size); chunks are still claimed in corpus order in each launch
    int64_t per = std::max<int64_t>(1, g.launch_words / g.L);
    p.Lp = (g.L + 3) & ~3;
    // negatives per kept slot: K shared (HogBatch) or 2*window*K per-input (Alg.1); Alg.1
    // launches are shortened so that its larger negative buffer stays <= 1 GiB
    const int32_t negs_per_slot = g.algorithm == 1 ? 2 * g.window * (g.K > 0 ? g.K : 1) : (g.K > 0 ? g.K : 1);
    if (g.algorithm == 1)
        per = std::max<int64_t>(1, std::min<int64_t>(per, (1ll << 30) / ((int64_t)p.Lp * negs_per_slot * 4)));
    {
        int rc = ensure_bt(std::min<int64_t>(per, std::max<int64_t>(chunk_hi - chunk_lo, 1)), p.Lp, negs_per_slot,
                           g.overlap_batch ? 2 : 1);
        if (rc) return bail(rc);
    }
    p.bt_redo = g.bt_redo;
    auto use_set = [&](StepParams& q, int set) {
        q.bt_nk = g.bt[set].nk; q.bt_kid = g.bt[set].kid; q.bt_kinfo = g.bt[set].kinfo; q.bt_neg = g.bt[set].neg;
    };
    // the batch kernel of launch j+1 runs on the side stream while the step kernel of launch j
    // runs on the main one (the step kernel's slabs leave room for one batch block per SM)
    const bool ovl = g.overlap_batch != 0;
    cudaEvent_t ev_tables, ev_bdone[2], ev_sdone[2];
    CUB(pool.make(&ev_tables, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
        CUB(pool.make(&ev_bdone[i], cudaEventDisableTiming));
        CUB(pool.make(&ev_sdone[i], cudaEventDisableTiming));
    }
    CUB(cudaEventRecord(ev_tables, st));
    if (ovl) {
        CUB(cudaStreamWaitEvent(g.side, ev_tables, 0));
        for (int i = 0; i < 2; ++i) CUB(cudaEventRecord(ev_sdone[i], st));
    }
    std::vector<cudaEvent_t> bev;  // (start, end) pairs of the batch launches on the side stream
    // C15 state: rows [0, pend_hi) of the model have an average in flight on the comm stream
    cudaEvent_t ev_snap, ev_ar;
    CUB(pool.make(&ev_snap, cudaEventDisableTiming));
    CUB(pool.make(&ev_ar, cudaEventDisableTiming));
    int64_t pend_hi = 0;
    if (dp() && g.sync_overlap && !g.syS) {
        const size_t bytes = (size_t)g.V * 2 * g.Ds * sizeof(float);
        int rc;
        if ((rc = dmalloc((void**)&g.syS, bytes, "C15 average"))) return bail(rc);
        if ((rc = dmalloc((void**)&g.syC, bytes, "C15 snapshot"))) return bail(rc);
    }
    {
        const int rc = bail(W2V_OK);  // every rank reached the training loop
        if (rc) return rc;
    }
#undef CUB
    int64_t jl = 0;                // launch counter (buffer set = jl & 1)
    std::vector<cudaEvent_t> evs;
    std::vector<int> ev_kind;  // 0 step, 1 sync, 2 batch
    auto mark = [&](int kind) -> cudaError_t {
        cudaEvent_t e;
        cudaError_t r = pool.make(&e);
        if (r != cudaSuccess) return r;
        evs.push_back(e);
        ev_kind.push_back(kind);
        return cudaEventRecord(e, st);
    };
    for (int32_t e = 0; e < epochs; ++e) {
        p.epoch = g.epoch_base + e;  // C1 epoch field and C8 progress of the global epoch
        const int64_t J = dp() ? pl.J : 1;
        for (int64_t k = 0; k < J; ++k) {
            const int64_t ilo = dp() ? chunk_lo + k * pl.I : chunk_lo;
            const int64_t ihi = (dp() && k < J - 1) ? chunk_lo + (k + 1) * pl.I : chunk_hi;
            for (int64_t a = ilo; a < ihi; a += per, ++jl) {
                p.chunk_lo = a;
                p.chunk_hi = std::min(ihi, a + per);
                const int set = ovl ? (int)(jl & 1) : 0;
                use_set(p, set);
                if (ovl) {  // a1 + a2 -> batch stream set `set`, once step jl-2 has consumed it
                    CU(cudaStreamWaitEvent(g.side, ev_sdone[set], 0));
                    cudaEvent_t b0, b1;
                    CU(pool.make(&b0)); CU(pool.make(&b1));
                    bev.push_back(b0); bev.push_back(b1);
                    CU(cudaEventRecord(b0, g.side));
                    CU(launch_batch(p, g.sms, 1, g.side));
                    CU(cudaEventRecord(b1, g.side));
                    CU(cudaEventRecord(ev_bdone[set], g.side));
                    CU(cudaStreamWaitEvent(st, ev_bdone[set], 0));
                } else {
                    CU(mark(2));
                    CU(launch_batch(p, g.sms, 8, st));
                    CU(mark(2));
                }
                CU(cudaMemsetAsync(g.chunk_ctr, 0, 8, st));
                if (g.mode == 2) CU(cudaMemsetAsync(g.turn, 0, 8, st));
                CU(mark(0));
                CU(kern == 0 ? launch_alg1(p, ctas, st) : kern == 4 ? launch_ring(p, ctas, ring_units, st)
                   : kern == 3 ? launch_wg(p, ctas, st)
                      : use_win ? launch_win(p, ctas, st) : launch_step(p, ctas, st, p.tma_gather ? &tmap : nullptr));  // a3-a8
                CU(mark(0));
                if (ovl) CU(cudaEventRecord(ev_sdone[set], st));
                launches += 2;
                ++g.st.step_launches;
            }
            if (dp()) {  // C13 / C14: full average, or the hot prefix with the cold rows every C-th
                CU(mark(1));
                const int64_t H = (g.sync_hot_rows <= 0 || g.sync_hot_rows >= g.V) ? g.V : g.sync_hot_rows;
                const bool full = H == g.V || g.sync_cold_every <= 1 || (k + 1) % g.sync_cold_every == 0 || k == J - 1;
                if (!g.sync_overlap) {
                    int rc = full ? sync_models(0, -1, &launches) : sync_models(0, H, &launches);
                    if (rc) return rc;
                } else {
                    // C15: apply the average in flight (its correction), then put this interval's
                    // rows in flight; the last interval ends with the plain (blocking) mean
                    const size_t rowf = (size_t)2 * g.Ds;
                    if (pend_hi > 0) {
                        CU(cudaStreamWaitEvent(st, ev_ar, 0));
                        CU(launch_sync_apply(g.M, g.syS, g.syC, (size_t)pend_hi * rowf, g.sms, st));
                        pend_hi = 0;
                    }
                    if (k == J - 1) {
                        int rc = sync_models(0, -1, &launches);
                        if (rc) return rc;
                    } else {
                        const int64_t hi_r = full ? g.V : H;
                        // snapshot C = M[rows]; out-of-place average C -> S in flight
                        CU(launch_sync_snap(g.M, g.syC, (size_t)hi_r * rowf, g.sms, st));
                        CU(cudaEventRecord(ev_snap, st));
                        CU(cudaStreamWaitEvent(g.comm_stream, ev_snap, 0));
                        if (g.ds.devcomm && g.ds.nwin == 3) {   // C17: the device kernel, C -> S, small grid
                            CU(devsync_launch(g.ds, 1, 2, 0, (size_t)hi_r * rowf, g.ds_owned, kDevSyncOverlapCtas,
                                              g.comm_stream));
                            ++launches;
                        } else {
                            NC(g_nccl.allReduce(g.syC, g.syS, (size_t)hi_r * rowf, ncclFloat32, ncclAvg, g.comm,
                                                g.comm_stream));
                        }
                        CU(cudaEventRecord(ev_ar, g.comm_stream));
                        pend_hi = hi_r;
                        if (full) g.st.syncs += 1; else g.st.syncs_hot += 1;
                    }
                }
                CU(mark(1));
            }
        }
    }
    if (g.check_finite) {  // failure detection: a diverged model is an error
        CU(launch_finite_check(g.M, (size_t)g.V * 2 * g.Ds, &g.info->nonfinite, g.sms, st));
        ++launches;
    }
    CU(cudaEventRecord(ev_end, st));
    DevStats hs{};
    SetupInfo hend{};
    CU(cudaMemcpyAsync(&hs, g.dstats, sizeof hs, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(&hend, g.info, sizeof hend, cudaMemcpyDeviceToHost, st));
    unsigned long long owned = 0;
    if (g.ds_owned) CU(cudaMemcpyAsync(&owned, g.ds_owned, 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (g.ds_owned) g.st.sync_floats_owned = (int64_t)owned;
    step_phase_report();
    win_phase_report();
    wg_phase_report();
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, ev0, ev_end)); g.st.ms_total = ms;
    CU(cudaEventElapsedTime(&ms, ev0, ev_h2d)); g.st.ms_h2d = ms;
    CU(cudaEventElapsedTime(&ms, ev_h2d, ev_setup)); g.st.ms_setup = ms;
    for (size_t i = 0; i + 1 < evs.size(); i += 2) {
        CU(cudaEventElapsedTime(&ms, evs[i], evs[i + 1]));
        if (ev_kind[i] == 0) g.st.ms_step += ms;
        else if (ev_kind[i] == 1) g.st.ms_sync += ms;
        else g.st.ms_batch += ms;
    }
    for (size_t i = 0; i + 1 < bev.size(); i += 2) {
        CU(cudaEventElapsedTime(&ms, bev[i], bev[i + 1]));
        g.st.ms_batch += ms;
    }
    // (events are destroyed by `pool`)
    g.st.words += (int64_t)hs.words;
    g.st.targets += (int64_t)hs.targets;
    g.st.row_touches += (int64_t)hs.row_touches;
    g.st.loss_pairs += (int64_t)hs.loss_pairs;
    g.st.loss_sum += hs.loss_sum;
    g.st.loss_tail_sum += hs.loss_tail_sum;
    g.st.loss_tail_pairs += (int64_t)hs.loss_tail_pairs;
    g.st.launches = launches;
    g.st.bytes_row = (int64_t)hs.row_touches * 4 * g.D * 2;
    g.st.row_touches_cold = (int64_t)hs.row_touches_cold;
    g.st.bytes_moved = (kern == 4 ? (int64_t)hs.rows_moved : 2 * (int64_t)hs.row_touches) * 4 * g.D;
    if (g.check_finite && hend.nonfinite)
        return fail(W2V_ENUMERIC, "w2v_train: the model holds NaN/Inf after training (diverged; lower alpha)");
    return W2V_OK;
}

int w2v_prefetch(const int32_t* ids, int64_t n) {
    NvtxRange nvtx("w2v_prefetch");
    if (!g.live) return fail(W2V_ESTATE, "w2v_prefetch before w2v_init");
    if (n < 0 || (!ids && n > 0)) return fail(W2V_EINVAL, "w2v_prefetch: bad corpus");
    if (n == 0) return W2V_OK;
    if (is_device_ptr(ids)) return fail(W2V_EINVAL, "w2v_prefetch: the corpus is already on the device");
    Ctx::Prefetch* f = !g.pf[0].pending ? &g.pf[0] : !g.pf[1].pending ? &g.pf[1] : nullptr;
    if (!f) return fail(W2V_ESTATE, "w2v_prefetch: two prefetched corpora are already pending (train on them first)");
    if ((size_t)n > f->cap) {
        cudaFree(f->buf);
        f->buf = nullptr;
        f->cap = 0;
        int rc = dmalloc((void**)&f->buf, (size_t)n * 4, "a prefetched corpus");
        if (rc) return rc;
        f->cap = (size_t)n;
    }
    // the copy engine moves it while the compute stream trains on the previous corpus; the
    // buffer is free: w2v_train is synchronous and consumed this slot's last corpus already
    CU(cudaMemcpyAsync(f->buf, ids, (size_t)n * 4, cudaMemcpyHostToDevice, g.copy_stream));
    CU(cudaEventRecord(f->done, g.copy_stream));
    f->host = ids;
    f->n = n;
    f->seq = ++g.pf_seq;
    f->pending = true;
    return W2V_OK;
}

int w2v_sync(void) {
    NvtxRange nvtx_sync("w2v_sync");
    if (!g.live) return fail(W2V_ESTATE, "w2v_sync before w2v_init");
    int rc = sync_models();
    if (rc) return rc;
    unsigned long long owned = 0;
    if (g.ds_owned) CU(cudaMemcpyAsync(&owned, g.ds_owned, 8, cudaMemcpyDeviceToHost, g.stream));
    CU(cudaStreamSynchronize(g.stream));
    if (g.ds_owned) g.st.sync_floats_owned = (int64_t)owned;
    return W2V_OK;
}

int w2v_get_embeddings(int32_t which, float* dst) {
    if (!g.live) return fail(W2V_ESTATE, "w2v_get_embeddings before w2v_init");
    if ((which != 0 && which != 1) || !dst) return fail(W2V_EINVAL, "w2v_get_embeddings: which must be 0/1, dst non-null");
    const size_t row = (size_t)g.D * 4;
    CU(cudaMemcpy2DAsync(dst, row, g.M + (which ? g.Ds : 0), (size_t)2 * g.Ds * 4, row, (size_t)g.V, cudaMemcpyDefault, g.stream));
    CU(cudaStreamSynchronize(g.stream));
    return W2V_OK;
}

int w2v_set_embeddings(int32_t which, const float* src) {
    if (!g.live) return fail(W2V_ESTATE, "w2v_set_embeddings before w2v_init");
    if ((which != 0 && which != 1) || !src) return fail(W2V_EINVAL, "w2v_set_embeddings: which must be 0/1, src non-null");
    const size_t row = (size_t)g.D * 4;
    CU(cudaMemcpy2DAsync(g.M + (which ? g.Ds : 0), (size_t)2 * g.Ds * 4, src, row, row, (size_t)g.V, cudaMemcpyDefault, g.stream));
    CU(cudaStreamSynchronize(g.stream));
    return W2V_OK;
}

int w2v_get_stats(w2v_stats_t* out) {
    if (!g.live) return fail(W2V_ESTATE, "w2v_get_stats before w2v_init");
    if (!out) return fail(W2V_EINVAL, "w2v_get_stats: null out");
    *out = g.st;
    return W2V_OK;
}

int w2v_debug_batches(uint8_t* keep, uint8_t* b, uint8_t* N, int32_t* ctx, int32_t* neg) {
    if (!g.live || g.dbg_rec_len == 0) return fail(W2V_ESTATE, "w2v_debug_batches: nothing recorded");
    const int64_t Lq = g.dbg_rec_len, kk = g.K > 0 ? g.K : 1;
    if (keep) CU(cudaMemcpyAsync(keep, g.dbg_keep, Lq, cudaMemcpyDefault, g.stream));
    if (b) CU(cudaMemcpyAsync(b, g.dbg_b, Lq, cudaMemcpyDefault, g.stream));
    if (N) CU(cudaMemcpyAsync(N, g.dbg_N, Lq, cudaMemcpyDefault, g.stream));
    if (ctx) CU(cudaMemcpyAsync(ctx, g.dbg_ctx, (size_t)Lq * 2 * g.window * 4, cudaMemcpyDefault, g.stream));
    if (neg) CU(cudaMemcpyAsync(neg, g.dbg_neg, (size_t)Lq * kk * 4, cudaMemcpyDefault, g.stream));
    CU(cudaStreamSynchronize(g.stream));
    return W2V_OK;
}

int w2v_debug_alg1_negatives(int32_t* neg) {
    if (!g.live || g.dbg_rec_len == 0 || !g.dbg_a1neg)
        return fail(W2V_ESTATE, "w2v_debug_alg1_negatives: nothing recorded (needs algorithm=1 and debug_len > 0)");
    if (!neg) return fail(W2V_EINVAL, "w2v_debug_alg1_negatives: null out");
    const int64_t kk = g.K > 0 ? g.K : 1;
    CU(cudaMemcpyAsync(neg, g.dbg_a1neg, (size_t)g.dbg_rec_len * 2 * g.window * kk * 4, cudaMemcpyDefault, g.stream));
    CU(cudaStreamSynchronize(g.stream));
    return W2V_OK;
}

int w2v_dist_unique_id(uint8_t out[128]) {
    if (!out) return fail(W2V_EINVAL, "w2v_dist_unique_id: null out");
    if (!g_nccl.load()) return fail(W2V_ENCCL, "cannot dlopen libnccl.so.2: %s", dlerror());
    ncclUniqueId id;
    NC(g_nccl.getUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return W2V_OK;
}

int w2v_dist_init(int32_t rank, int32_t world, const uint8_t id[128]) {
    if (!g.live) return fail(W2V_ESTATE, "w2v_dist_init before w2v_init");
    if (world < 1 || rank < 0 || rank >= world) return fail(W2V_EINVAL, "w2v_dist_init: rank %d / world %d", rank, world);
    if (g.comm) return fail(W2V_ESTATE, "w2v_dist_init: already initialised");
    g.rank = rank;
    g.world = world;
    if (world == 1 && !id) return W2V_OK;  // no communicator, no collective calls
    if (!id) return fail(W2V_EINVAL, "w2v_dist_init: null id with world > 1");
    if (!g_nccl.load()) return fail(W2V_ENCCL, "cannot dlopen libnccl.so.2: %s", dlerror());
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    NC(g_nccl.commInitRank(&g.comm, world, uid, rank));
    if (!g.dp_tmp) {  // scratch of the consensus collectives, allocated here so w2v_train cannot fail on it
        int rc = dmalloc((void**)&g.dp_tmp, (size_t)world * 8, "dp scratch");
        if (rc) return rc;
    }
    g.st.sync_path = 1;
    // every model average moves 2*V*Ds floats: at world > 1 drop the 128-B row padding (worth
    // ~0.7% on one GPU) so the average covers exactly the 2*V*D model floats; with
    // sync_device (C17) the model moves into ncclMemAlloc memory (the symmetric window)
    const bool repack = world > 1 && g.Ds != g.D;
    if (repack || g.sync_device) {
        const int32_t Dn = repack ? g.D : g.Ds;
        const size_t bytes = (size_t)g.V * 2 * Dn * sizeof(float);
        float* M2 = nullptr;
        int rc;
        if (g.sync_device) {
            std::string e;
            void* b = nullptr;
            rc = devsync_alloc(bytes, &b, &e) ? fail(W2V_ENCCL, "%s", e.c_str()) : W2V_OK;
            M2 = (float*)b;
            if (!rc) rc = dmalloc((void**)&g.ds_owned, 8, "sync_device counter");
        } else {
            rc = dmalloc((void**)&M2, bytes, "the unpadded data-parallel model");
        }
        rc = dp_agree(rc, g.stream);  // a rank that cannot allocate must not leave peers in a collective
        if (rc) {
            if (g.sync_device) devsync_free(M2); else cudaFree(M2);
            return rc;
        }
        if (repack) {
            const size_t half = (size_t)g.D * 4;
            for (int h = 0; h < 2; ++h)
                CU(cudaMemcpy2DAsync(M2 + h * g.D, 2 * half, g.M + h * g.Ds, (size_t)2 * g.Ds * 4, half, (size_t)g.V,
                                     cudaMemcpyDeviceToDevice, g.stream));
        } else {
            CU(cudaMemcpyAsync(M2, g.M, bytes, cudaMemcpyDeviceToDevice, g.stream));
        }
        if (g.ds_owned) CU(cudaMemsetAsync(g.ds_owned, 0, 8, g.stream));
        CU(cudaStreamSynchronize(g.stream));
        if (g.M_nccl) devsync_free(g.M); else cudaFree(g.M);
        g.M = M2;
        g.M_nccl = g.sync_device != 0;
        g.Ds = Dn;
        if (g.sync_device && g.sync_overlap && !g.syS) {
            // C15 with C17: the snapshot C and the average S are symmetric windows too
            std::string e;
            void *bc = nullptr, *bs = nullptr;
            int lrc = devsync_alloc(bytes, &bc, &e) || devsync_alloc(bytes, &bs, &e) ? fail(W2V_ENCCL, "%s", e.c_str())
                                                                                    : W2V_OK;
            lrc = dp_agree(lrc, g.stream);
            if (lrc) {
                devsync_free(bc);
                devsync_free(bs);
                return lrc;
            }
            g.syC = (float*)bc;
            g.syS = (float*)bs;
            g.sy_nccl = true;
        }
        if (g.sync_device) {  // collective: window registration + device communicator
            std::string e;
            auto agree_min = [](int v) -> int {  // min over ranks (NCCL all-reduce on the scratch)
                int64_t h = v;
                if (cudaMemcpyAsync(g.dp_tmp, &h, 8, cudaMemcpyHostToDevice, g.stream) != cudaSuccess) return -1;
                if (g_nccl.allReduce(g.dp_tmp, g.dp_tmp, 1, ncclInt64, ncclMin, g.comm, g.stream) != ncclSuccess)
                    return -1;
                if (cudaMemcpyAsync(&h, g.dp_tmp, 8, cudaMemcpyDeviceToHost, g.stream) != cudaSuccess) return -1;
                if (cudaStreamSynchronize(g.stream) != cudaSuccess) return -1;
                return (int)h;
            };
            void* bufs[3] = {g.M, g.syC, g.syS};
            const size_t sizes[3] = {bytes, bytes, bytes};
            if (devsync_open(g.comm, bufs, sizes, g.sy_nccl ? 3 : 1, world, 1, +agree_min, &g.ds, &e))
                return fail(W2V_ENCCL, "%s", e.c_str());
            g.st.sync_path = g.ds.multimem ? 3 : 2;
        }
    }
    return W2V_OK;
}

int w2v_dist_sync_slice(int64_t off, int64_t n, int32_t world, int32_t rank, int64_t out[4]) {
    if (off < 0 || n < 0 || world < 1 || rank < 0 || rank >= world || !out)
        return fail(W2V_EINVAL, "w2v_dist_sync_slice: bad arguments");
    size_t s0, a0, a1, s1;
    devsync_slice((size_t)off, (size_t)n, rank, world, &s0, &a0, &a1, &s1);
    out[0] = (int64_t)s0; out[1] = (int64_t)a0; out[2] = (int64_t)a1; out[3] = (int64_t)s1;
    return W2V_OK;
}

int64_t w2v_dist_plan(int64_t n_global, int32_t L, int32_t world, int32_t rank, int64_t P, int64_t* out,
                      int64_t max_out) {
    if (n_global < 0 || L < 1 || world < 1 || rank < 0 || rank >= world || P < 1 || !out)
        return fail(W2V_EINVAL, "w2v_dist_plan: bad arguments");
    const Plan pl = make_plan(n_global, L, world, rank, P);
    out[0] = pl.start;
    out[1] = pl.end;
    out[2] = pl.J;
    for (int64_t k = 0; k < pl.J && k < max_out; ++k) {
        out[3 + 2 * k] = pl.lo + k * pl.I;
        out[4 + 2 * k] = (k == pl.J - 1) ? pl.hi : pl.lo + (k + 1) * pl.I;
    }
    return pl.J;
}

int w2v_finalize(void) {
    if (!g.live) return W2V_OK;
    cudaStreamSynchronize(g.stream);
    devsync_close(&g.ds);
    if (g.comm) g_nccl.commDestroy(g.comm);
    free_dbg();
    free_bt();
    if (g.M_nccl) devsync_free(g.M); else cudaFree(g.M);
    cudaFree(g.ds_owned);
    cudaFree(g.corpus); cudaFree(g.counts); cudaFree(g.thr); cudaFree(g.P); cudaFree(g.scratch);
    cudaFree(g.G); cudaFree(g.info); cudaFree(g.dstats); cudaFree(g.chunk_ctr); cudaFree(g.dp_tmp);
    cudaFree(g.tick); cudaFree(g.turn); cudaFree(g.tick_tab);
    cudaStreamSynchronize(g.side);
    cudaStreamSynchronize(g.comm_stream);
    cudaStreamSynchronize(g.copy_stream);
    cudaStreamDestroy(g.side);
    cudaStreamDestroy(g.comm_stream);
    cudaStreamDestroy(g.copy_stream);
    for (auto& f : g.pf) {
        cudaFree(f.buf);
        if (f.done) cudaEventDestroy(f.done);
    }
    if (g.sy_nccl) { devsync_free(g.syS); devsync_free(g.syC); } else { cudaFree(g.syS); cudaFree(g.syC); }
    cudaStreamDestroy(g.own_stream);
    Ctx fresh;
    g = fresh;
    return W2V_OK;
}

}  // extern "C"
