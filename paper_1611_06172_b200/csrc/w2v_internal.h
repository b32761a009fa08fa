// w2v_internal.h — structures shared by the library's translation units (not part of the ABI).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <string>

struct ncclComm;

namespace w2v {

// Written by the setup kernels, read by the step kernel and (once per w2v_train) by the host.
struct SetupInfo {
    uint64_t PV;       // P[V], total sampler mass (C3)
    int32_t gshift;    // guide-table bucket shift
    int32_t bad_id;    // 1 if an id outside [0,V) was seen
    int32_t nonfinite; // 1 if the model holds a NaN/Inf after training (option check_finite)
    int64_t first_bad; // (unused by kernels; host diagnostics)
};

struct DevStats {
    unsigned long long words, targets, row_touches, loss_pairs;
    double loss_sum;
    double loss_tail_sum;
    unsigned long long loss_tail_pairs;
    unsigned long long row_touches_cold;  // row touches with id >= StepParams::cold_from
    unsigned long long rows_moved;        // rows actually gathered + reduced (ring kernel)
};

struct StepParams {
    const int32_t* ids;   // ids[k] = token at global position ids_base + k
    int64_t ids_base;
    int64_t shard_start, n_local, n_global;
    int64_t chunk_lo, chunk_hi;  // global chunk range of this launch
    int32_t L, window, K, D;
    int32_t epoch, epochs, world;
    int32_t allow_tn, deterministic;
    float alpha0;
    int64_t Q;
    uint64_t seed;
    int64_t V;
    const uint64_t* thr;
    const uint64_t* P;
    const int32_t* G;
    const SetupInfo* info;
    float* M;  // interleaved model: row w = [M_in[w] (D, padded to Ds) | M_out[w] (D, padded to Ds)]
    int32_t Ds;  // half-row stride in floats (>= D)
    unsigned long long* chunk_ctr;
    DevStats* stats;
    int64_t loss_tail_from;
    int64_t dbg_base, dbg_len;
    uint8_t *dbg_keep, *dbg_b, *dbg_N;
    int32_t *dbg_ctx, *dbg_neg;
    int32_t warp_bytes;   // dynamic shared memory per warp
    int32_t slab_offset;  // byte offset of the row slab inside a warp's region
    // batch stream of the launch range (batch.cu), rel = chunk - chunk_lo, Lp = L rounded to 4
    int32_t Lp;
    int32_t* bt_nk;       // [chunks]          kept positions per chunk
    int32_t* bt_kid;      // [chunks][Lp]      kept words, corpus order
    int32_t* bt_kinfo;    // [chunks][Lp]      (offset << 8) | b
    int32_t* bt_neg;      // [chunks][Lp][KS]  shared negatives of each kept target
    uint32_t* bt_redo;    // batch kernel scratch: per-warp rejection masks
    // a8: L2 eviction-priority hints on the row copies: rows with id < hot_rows (the Zipf-hot
    // prefix) get evict_last if l2_hint & 1; the others evict_first if l2_hint & 2
    int64_t hot_rows;     // M_out rows (targets, negatives; and both halves in the window kernels)
    int64_t hot_rows_in;  // M_in rows (contexts) in the rows kernel
    int32_t l2_hint;
    int32_t rowpath_only; // measurement mode: rows kernel without a4-a6 (zero deltas; model unchanged)
    // mode 2 (NEXT-4, conflict-ticketed deterministic; rows kernel): per (matrix, row) the next
    // ticket to hand out and the number of completed accesses ([0,V) M_in, [V,2V) M_out), the
    // launch's chunk turn, and the byte offset of the warp's ticket table in shared memory
    uint32_t* tick_issue;
    uint32_t* tick_done;
    unsigned long long* turn;
    int32_t tick_off;     // >= 0: byte offset of the table in the warp's smem; -1: in tick_glob
    uint32_t* tick_glob;  // mode 2 ticket tables in global memory, [CTA][Lp][2w+K+1], when the
                          // table does not fit beside the slab (long chunks x many rows)
    int32_t scatter_wait; // 1: a target waits for its reductions to complete before the next
                          // target's gathers (R11); 0 (Hogwild only): until they are read
    int32_t ring_delta;   // ring kernel, deterministic mode: 1 = write back slot - original
                          // (the Hogwild path) instead of the slot value (option ring_writeback)
    int64_t cold_from;    // statistics: row touches with id >= cold_from are counted as "cold" (the
                          // ids beyond an L2-sized hot prefix; the cache-aware roofline's B_cold)
    int32_t algorithm;    // 0 HogBatch (shared negatives), 1 Alg.1 (per-input negatives, alg1.cu)
    int32_t tma_gather;   // rows kernel: gather 4 rows per TMA tile::gather4 (step_tma_gather_ok)
    int32_t* dbg_a1neg;   // Alg.1 debug: [len][2*window][K] per-input negatives
};

// setup.cu
cudaError_t launch_hist(const int32_t* ids, int64_t n, int64_t V, unsigned long long* counts, SetupInfo* info,
                        int sms, cudaStream_t st, int* launches);
cudaError_t launch_tables(const unsigned long long* counts, int64_t V, int64_t T, float t, uint64_t* thr,
                          uint64_t* P, uint64_t* scratch, int32_t* G, int gbits, SetupInfo* info, cudaStream_t st,
                          int* launches);
cudaError_t launch_finite_check(const float* M, size_t n, int32_t* flag, int sms, cudaStream_t st);
cudaError_t launch_init(float* M, int64_t V, int32_t D, int32_t Ds, uint64_t seed, int sms, cudaStream_t st);

// batch.cu (a1 subsampling + window batching, a2 negative sampler)
size_t batch_redo_words(int sms);
cudaError_t launch_batch(const StepParams& p, int sms, int blocks_per_sm, cudaStream_t st);

// hogbatch_win.cu (window-resident rows; window <= 15)
size_t win_warp_bytes(int L, int window, int K, int D, int32_t* slab_offset);
int win_max_ctas_per_sm(const StepParams& p);
cudaError_t launch_win(const StepParams& p, int ctas, cudaStream_t st);
void win_phase_report();  // (experiment builds with W2V_PHASE_TIMING)

// hogbatch_wg.cu (window-resident, warp-specialised: NW column warps + 1 IO warp per CTA)
size_t wg_cta_bytes(int L, int window, int K, int D, int32_t* slab_offset);
int wg_threads(int D);
int wg_max_ctas_per_sm(const StepParams& p);
cudaError_t launch_wg(const StepParams& p, int ctas, cudaStream_t st);
void wg_phase_report();  // (experiment builds with W2V_PHASE_TIMING)

// sync.cu (C15 overlapped averaging)
cudaError_t launch_sync_apply(float* M, const float* S, const float* C, size_t n, int sms, cudaStream_t st);
cudaError_t launch_sync_snap(const float* M, float* C, size_t n, int sms, cudaStream_t st);

// sync_dev.cu: a9 as one kernel over NCCL's symmetric window (option "sync_device", C17)
constexpr int kDevSyncCtas = 296;  // 2 per SM; also the LSA barrier count
// rank r of W owns floats [s0, s1) = [off + n*r/W, off + n*(r+1)/W) of an averaged range: a scalar
// head [s0, a0) up to the first 16-B aligned float, a float4 body [a0, a1), a scalar tail [a1, s1)
__host__ __device__ inline void devsync_slice(size_t off, size_t n, int r, int W, size_t* s0, size_t* a0, size_t* a1,
                                              size_t* s1) {
    *s0 = off + n * (size_t)r / (size_t)W;
    *s1 = off + n * (size_t)(r + 1) / (size_t)W;
    *a0 = *s0 + 3 < *s1 ? (*s0 + 3) & ~(size_t)3 : *s1;
    *a1 = *a0 + ((*s1 - *a0) & ~(size_t)3);
}
constexpr int kDevSyncOverlapCtas = 32;  // C15's in-flight average: a small grid beside the step kernel
constexpr int kDevSyncMaxWin = 3;        // windows: 0 the model, 1 C15 snapshot C, 2 C15 average S
struct DevSync {
    void* comm = nullptr;                 // ncclComm_t
    void* win[kDevSyncMaxWin] = {};       // ncclWindow_t per registered buffer
    int nwin = 0;
    void* devcomm = nullptr;              // heap ncclDevComm
    int multimem = 0;                     // 1: NVLS multicast path, 0: LSA peer loads/stores
    int lsa_size = 0;
};
int devsync_alloc(size_t bytes, void** buf, std::string* err);
void devsync_free(void* buf);
int devsync_open(ncclComm* comm, void* const* bufs, const size_t* bytes, int nwin, int world, int want_mm,
                 int (*agree_min)(int), DevSync* ds, std::string* err);
void devsync_close(DevSync* ds);
cudaError_t devsync_launch(const DevSync& ds, int src, int dst, size_t off, size_t n, unsigned long long* counted,
                           int ctas, cudaStream_t st);

// alg1.cu (Algorithm 1, the level-1 baseline)
bool alg1_supported(int D, int K);
size_t alg1_warp_bytes(int L);
int alg1_max_ctas_per_sm(const StepParams& p);
cudaError_t launch_alg1(const StepParams& p, int ctas, cudaStream_t st);

// hogbatch_ring.cu (window ring of M_in rows, originals in TMEM; window <= 15)
size_t ring_warp_bytes(int L, int window, int K, int D, int32_t* slab_offset);
int ring_units_per_cta(int window, int D, int K, size_t warp_bytes, size_t smem_max);
bool ring_supported(int window, int D, int K);
cudaError_t launch_ring(const StepParams& p, int ctas, int units, cudaStream_t st);

// hogbatch.cu (per-target rows; any window)
bool step_supported(int D, int K);
cudaError_t launch_step(const StepParams& p, int ctas, cudaStream_t st, const CUtensorMap* tmap);
bool step_tma_gather_ok(int D, int K, int window);
int step_max_ctas_per_sm(const StepParams& p);
size_t step_warp_bytes(int L, int window, int K, int D, int32_t* slab_offset, int32_t* tick_offset = nullptr);
void step_phase_report();  // (experiment builds with W2V_PHASE_TIMING) prints per-phase cycles

}  // namespace w2v
