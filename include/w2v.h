/*
 * w2v.h — C-ABI of libw2v.so, the B200-native HogBatch skip-gram negative-sampling SGD step
 * (arXiv 1611.06172). Citations: PAPER.md:L = /root/reference/PAPER.md line L; "Alg.1 l.k" =
 * PAPER.md line 38+k; C1..C15 and R1..R18 are the contract and readings in DESIGN.md §2-§3.
 *
 * Conventions for every call:
 *  - Returns int: W2V_OK (0) or a negative W2V_E* code; w2v_last_error() then describes it
 *    (thread-local string, valid until the next call on that thread).
 *  - One process-global context = one model on the CUDA device current at w2v_init.
 *  - Pointers marked "host or device" are classified with cudaPointerGetAttributes; they are
 *    read/written during the call only and never retained. The library owns M_in, M_out,
 *    the sampler tables and all work buffers (cudaMalloc'd in w2v_init / w2v_train, freed in
 *    w2v_finalize).
 *  - Model layout in HBM: one buffer of V rows, row w = [M_in[w] | M_out[w]],
 *    each half padded to a multiple of 32 fp32 (128 B), so the Zipf-hot rows of BOTH matrices
 *    form one contiguous prefix and every row starts on a cache line.
 *  - All work is enqueued on the library stream (w2v_set_stream, default: a private stream);
 *    every call returns after its work has completed (synchronous API).
 */
#ifndef W2V_H_
#define W2V_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define W2V_OK 0
#define W2V_EINVAL (-1)   /* bad argument, id outside [0,V), unknown option key, P[V]==0    */
#define W2V_ESTATE (-2)   /* call out of order (e.g. train before init)                      */
#define W2V_ENOMEM (-3)   /* device allocation failed; message names the requested bytes      */
#define W2V_ECUDA  (-4)   /* CUDA runtime error                                               */
#define W2V_ENCCL  (-5)   /* NCCL error or NCCL library not loadable                          */
#define W2V_ENUMERIC (-6) /* the model holds NaN/Inf after w2v_train (option check_finite)     */
#define W2V_EPEER  (-7)   /* data-parallel: another rank failed before the first model average;
                           * every rank returns (no collective is left waiting)              */

typedef struct {
    int64_t words;        /* raw corpus tokens processed (R14: the unit of words/s)           */
    int64_t targets;      /* trained targets (kept, N > 0)                                     */
    int64_t row_touches;  /* sum over targets of N + K + 1 (C12)             */
    int64_t loss_pairs;   /* sum over targets of N * (K + 1)                                   */
    double  loss_sum;     /* SGNS loss of the pre-update snapshots (C11), fp64 accumulator     */
    int64_t syncs;        /* model averagings performed (C13)                                  */
    int64_t launches;     /* kernels launched by the library in the last w2v_train             */
    double  ms_total;     /* last w2v_train wall time on the stream (CUDA events), ms          */
    double  ms_step;      /* ... of which inside the fused hogbatch_step launches, ms          */
    double  ms_setup;     /* ... of which setup (a0: validate, counts, tables), ms             */
    double  ms_sync;      /* ... of which model averaging (a9), ms                             */
    double  ms_h2d;       /* ... of which corpus host->device copy (host-pointer calls), ms    */
    int64_t step_launches;/* hogbatch_step launches in the last w2v_train                      */
    int64_t bytes_row;    /* algorithmic row bytes of the last w2v_train: row_touches*4D*2      */
    double  loss_tail_sum;   /* loss of targets at global positions >= option loss_tail_from    */
    int64_t loss_tail_pairs; /* ... and their pair count (the "final-10%" training loss)         */
    int64_t kernel;          /* step kernel of the last w2v_train: 1 rows, 2 window, 3 window
                                warp-specialised, 4 Alg.1                                       */
    double  ms_batch;        /* ... of which the a1/a2 batch kernel (subsampling, windows,
                                negatives; batch.cu), ms — not included in ms_step              */
    int64_t l2_window_bytes; /* a8: bytes of the hot-row prefix under the persisting-L2 window  */
    int64_t l2_carve_bytes;  /* a8: persisting-L2 carve-out set for the last w2v_train (0 = off) */
    int64_t syncs_hot;       /* C14 averagings of the hot-row prefix only (syncs counts full ones) */
    int64_t units_per_sm;    /* step-kernel work units (1-warp CTAs) resident per SM, last train   */
    int64_t row_touches_cold;/* row touches (gathered rows) of the last w2v_train whose id is >=
                                cold_from_row: outside the Zipf-hot prefix that fits the 126 MB L2
                                (ids are frequency ranks), i.e. the rows that must come from DRAM
                                under an ideal static cache — B_cold of SURVEY.md §8(d)           */
    int64_t cold_from_row;   /* that prefix: L2 bytes / (8 D) rows, last train                    */
    int64_t bytes_moved;     /* row bytes the step kernel actually gathered + reduced in the last
                                w2v_train: bytes_row for the per-target kernels; fewer for the ring
                                kernel, which keeps M_in rows of the window on chip             */
    int64_t sync_path;       /* how a9 averages: 0 no communicator, 1 NCCL all-reduce (ncclAvg),
                                2 one kernel over NCCL's symmetric window with peer loads/stores,
                                3 the same kernel through the NVSwitch multicast address (NVLS
                                multimem.ld_reduce / multimem.st) — option "sync_device"       */
    int64_t sync_floats_owned; /* sync_path 2/3: floats this rank reduced and broadcast since
                                w2v_dist_init (its 1/W slice of every averaged range)           */
} w2v_stats_t;

/* Create the model (Alg.1 l.1 "Given model parameter Omega = {M_in, M_out}").
 * V vocabulary size (>=1), D embedding width (>=4, D % 4 == 0, D <= 512), window (>=1, the
 * maximum half-window of C4; N <= 2*window), K shared negatives (0..31; K=0 degenerates to
 * logistic regression), alpha initial learning rate (>0, C8), subsample t (>=0,
 * C2; 0 disables), seed (C1 key). Initialises M_in ~ U[-0.5/D, 0.5/D) and M_out = 0 per C9.
 * Supported (D, K) envelope of the register tiles: D <= 64 with K <= 31, D <= 192 with
 * K <= 15, D <= 320 with K <= 7, D <= 512 with K <= 5 (covers the paper's D=300, K=5).
 * Errors: EINVAL on out-of-range arguments or (D, K) outside the envelope,
 * ENOMEM naming the 2*V*D*4 bytes requested, ESTATE if already initialised. */
int w2v_init(int64_t V, int32_t D, int32_t window, int32_t K, float alpha, float subsample,
             uint64_t seed);

/* Set an integer option before w2v_train (SURVEY.md §5 "Config / flags"). Keys:
 *  "mode"                  0 = Hogwild (default), 1 = deterministic
 *                          (one work unit, targets in corpus order, R17), 2 = deterministic
 *                          and parallel ("dependence
 *                          between iterations"): all SMs, every row access waits on a per-row
 *                          ticket taken in corpus order — bit-identical to mode 1 (rows kernel,
 *                          2*window+K+1 <= 32; a chunk's ticket table, sentence_len x
 *                          (2*window+K+1) u32, lives in shared memory, or in global memory when
 *                          it does not fit beside the slab)
 *  "sentence_len"          chunk length L of C5 (1..4096; default 1000)
 *  "sync_period_words"     P of C13 (>=1; default 2^20)
 *  "sync_hot_rows"         C14: rows [0,H) of both matrices (the Zipf-hot prefix)
 *                          are averaged after every interval (default 0 = all rows, i.e. C13)
 *  "sync_cold_every"       C14: rows [H,V) only after every this many intervals and after the
 *                          last interval of each epoch (>=1; default 1)
 *  "sync_device"           C17 (default 0; set BEFORE w2v_dist_init): the model is
 *                          placed in ncclMemAlloc memory registered as an NCCL symmetric window
 *                          and every C13/C14 average runs as ONE kernel (sync_dev.cu): each rank
 *                          reduces its 1/W slice — through the NVSwitch multicast address
 *                          (multimem.ld_reduce / multimem.st, NVLS) when NCCL provides one, else
 *                          by peer loads/stores over NVLink — between two device-side barriers.
 *                          Needs NCCL >= 2.28 and all ranks in one NVLink domain (else ENCCL
 *                          from w2v_dist_init). With "sync_overlap" also set before
 *                          w2v_dist_init, C15's snapshot and average buffers are symmetric
 *                          windows too and each in-flight average is the same kernel, out of
 *                          place, on the library's comm stream (32 CTAs beside the step kernel).
 *  "tma_gather"            1 (default): the rows kernel gathers 4 rows per TMA tile::gather4
 *                          instruction where its slab allows (D <= 256 packed, 2*window and the
 *                          output tile multiples of 4: cfg4's D = 128, K = 15, window 8); 0 =
 *                          one cp.async.bulk per row everywhere. Same data either way.
 *  "sync_overlap"          C15 (default 0): the rows due are snapshot and averaged
 *                          on a communication stream while the next interval trains; their
 *                          correction M += avg - snapshot is applied one interval late; the last
 *                          interval of an epoch ends with the plain blocking mean
 *  "lr_quantum"            Q of C8 (>=1; default 10000)
 *  "allow_target_negative" 0/1 (R2; default 0)
 *  "debug_base","debug_len" record the batch stream (C5-C7) for global positions
 *                          [base, base+len) during the next w2v_train (len 0 = off)
 *  "algorithm"             0 = HogBatch (default), 1 = Algorithm 1, the
 *                          "original" level-1 SGNS update: per-input negatives
 *                          on the A1NEG stream, one dot + immediate update per (input, output)
 *                          pair, N(K+1)+N row updates per target
 *  "l2_hint"               a8 L2 eviction-priority hints on the row copies: bit 0 = evict_last
 *                          on the hot prefix, bit 1 = evict_first on the other rows (default 1)
 *  "l2_hot_rows"           hot prefix for l2_hint (-1 = the rows that fit 64 MB; default -1)
 *  "l2_hot_rows_in"        ... for the M_in (context) rows of the rows kernel (-1 = all rows:
 *                          a chunk's next targets re-read them within microseconds)
 *  "l2_persist"            0/1 persisting-L2 access-policy window over the hot-row prefix
 *                          (default 0: measured harmful on B200, the bulk copies ignore it and
 *                          the carve-out only shrinks L2; profiles/r01_ablations.md §2)
 *  "l2_window_rows", "l2_carve_mb", "l2_hit_pct"  that window's rows (0 = carve-out size),
 *                          carve-out in MB (0 = device maximum) and hitRatio in percent
 *  "ctas_per_sm"           0 = occupancy maximum (default), else that many 1-warp CTAs per SM
 *  "launch_words"          raw words per hogbatch_step launch (>=1; default 2^26): bounds a
 *                          launch's duration; results do not depend on it in deterministic mode
 *  "kernel"                0 auto (default), 1 per-target rows (hogbatch.cu),
 *                          2 window-resident rows (hogbatch_win.cu; window <= 15), 3 window-
 *                          resident warp-specialised (hogbatch_wg.cu; window <= 15), 4 window
 *                          ring with the originals in tensor memory (hogbatch_ring.cu; window
 *                          <= 15): ~1 gather + 1 reduction per kept position for M_in. In
 *                          Hogwild mode a slot holds a row for 2*window+1 targets, so with
 *                          long windows the deltas of stale Zipf-hot rows overshoot (cfg4,
 *                          window 8: final loss +2.6%); exact in modes 1/2
 *  "ring_writeback"        kernel 4 in deterministic mode: 0 (default) stores the slot value
 *                          (the exact sequential row), 1 reduces slot - original as Hogwild does
 *  "check_finite"          1 (default): scan the model for NaN/Inf after every w2v_train (one
 *                          streaming pass, ~0.5 ms at cfg3) and return W2V_ENUMERIC if found
 *  "overlap_batch"         1: the a1/a2 batch kernel of launch j+1 runs on a side stream
 *                          concurrently with the step kernel of launch j (double-buffered batch
 *                          stream); 0 (default): serialised on the library stream — the
 *                          co-resident batch block slows the step kernel by more than it hides
 *  "rowpath_only"          measurement mode (default 0): the rows kernel issues exactly the same
 *                          gathers and scatters but skips a4-a6 and reduces zero deltas (model
 *                          unchanged) — the achievable rate of the row path, for the roofline
 *  "loss_tail_from"        global position from which targets also accumulate into
 *                          loss_tail_sum / loss_tail_pairs (default: never)
 *  "epochs_total"          E used by the alpha schedule when training is split over several
 *                          w2v_train calls (0 = the epochs argument of each call; default 0)
 *  "epoch_base"            global index of this call's first epoch: the C1 RNG epoch field and
 *                          the C8 schedule position (0..255; default 0). With epochs_total it
 *                          makes checkpoint/resume exact: w2v_get_embeddings after epoch e,
 *                          w2v_set_embeddings + epoch_base = e+1 later (deterministic mode:
 *                          bit-identical to one uninterrupted call)
 * Unknown key or bad value -> EINVAL. */
int w2v_set_option(const char* key, int64_t value);

/* Use this CUDA stream (a cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream) for all
 * subsequent work; NULL restores the library's private stream. Plumbing, not a step of the
 * method (PyTorch supplies device memory, streams and process groups). */
int w2v_set_stream(void* cuda_stream);

/* Train (PAPER.md:116-126 HogBatch; PAPER.md:135-138 Hogwild across work units).
 * corpus_ids: int32[n_tokens], host or device, ids in [0,V), this rank's contiguous shard of
 * the global corpus (C13; with world 1 the whole corpus). Runs, per call: id validation and
 * counts (global over ranks), thresholds, sampler, then `epochs` epochs of subsampling +
 * window batching + negative sampling + the fused step, syncing every sync_period_words per
 * rank (C13). Counts/thresholds/sampler come from this call's corpus. Epoch e of this call
 * uses RNG epoch field e. n_tokens == 0: no-op success, model unchanged.
 * Errors: EINVAL (id outside [0,V): nothing trained; P[V] == 0; epochs < 1; shard not
 * chunk-aligned per C13), ESTATE, ENOMEM, ECUDA, ENCCL. */
int w2v_train(const int32_t* corpus_ids, int64_t n_tokens, int32_t epochs);

/* Start copying a HOST corpus (int32[n_tokens], ideally pinned) to the device on the library's
 * copy stream and return at once; a later w2v_train with the same pointer and n_tokens trains on
 * that copy instead of copying again (the oldest matching prefetch first). Lets a caller overlap
 * the next corpus's host->device transfer with the current w2v_train (plumbing around the step,
 * the corpus arrives from the host). The host data must not change until the
 * consuming w2v_train returns. At most two prefetches may be pending. Errors: ESTATE (before
 * w2v_init, or two pending), EINVAL (NULL with n > 0, a device pointer), ENOMEM, ECUDA. */
int w2v_prefetch(const int32_t* corpus_ids, int64_t n_tokens);

/* Collective (all ranks must call): replace M_in and M_out by their elementwise mean over
 * ranks (R13). World 1: no-op. */
int w2v_sync(void);

/* Copy M_in (which = 0) or M_out (which = 1) into dst, V x D fp32 row-major, host or device.
 * M_in / M_out are the input and output embedding matrices of the problem statement
 * (Alg.1 l.1 "model parameter Omega = {M_in, M_out}"); M_in is the
 * word embedding (R15). Errors: ESTATE before w2v_init, EINVAL for which not 0/1 or dst NULL. */
int w2v_get_embeddings(int32_t which, float* dst);

/* Overwrite M_in (which = 0) or M_out (which = 1) from src, V x D fp32 row-major, host or
 * device (resume / test setup): the same Omega restored from a checkpoint
 * (SURVEY.md §5). Errors as w2v_get_embeddings. */
int w2v_set_embeddings(int32_t which, const float* src);

/* Statistics of the last w2v_train (counters are cumulative since w2v_init; ms_* and
 * launches refer to the last call). */
int w2v_get_stats(w2v_stats_t* out);

/* Copy the batch stream recorded by the last w2v_train for [debug_base, debug_base+debug_len)
 * (C5-C7: the subsampling, window and negative-sampling decisions of Alg.1 l.3-11,
 * PAPER.md:41-49, as shared per target by HogBatch): keep u8[len], b u8[len] (0 = not kept), N u8[len] (0 = not trained), ctx
 * int32[len][2*window] (-1 padded), neg int32[len][max(K,1)] (-1 padded). Host or device;
 * any pointer may be NULL. ESTATE if nothing was recorded. */
int w2v_debug_batches(uint8_t* keep, uint8_t* b, uint8_t* N, int32_t* ctx, int32_t* neg);

/* Algorithm 1 only (option "algorithm" = 1): copy the per-input negatives recorded by the last
 * w2v_train for [debug_base, debug_base+debug_len): int32[len][2*window][max(K,1)], entry
 * [q][i][k] = the k-th negative of input i of the target at position base+q (Alg.1 l.10),
 * -1 padded. Host or device. ESTATE if nothing was recorded. */
int w2v_debug_alg1_negatives(int32_t* neg);

/* Data-parallel bootstrap (C13). Rank 0 creates a 128-byte NCCL unique id; the caller
 * broadcasts it (torch.distributed) and every rank calls w2v_dist_init. world == 1 with a NULL id
 * creates no communicator and makes no NCCL call; world == 1 WITH an id creates a 1-rank NCCL
 * communicator so that every collective of the data-parallel path runs on one GPU (test hook;
 * averaging one replica is the identity). Requires libnccl.so.2 (dlopen) when an id is given. */
int w2v_dist_unique_id(uint8_t out[128]);
int w2v_dist_init(int32_t rank, int32_t world, const uint8_t id[128]);

/* Pure host planner (no device needed): shard of rank r per C13 and its sync intervals.
 * out[0..1] = [start, end) global raw positions; out[2] = J intervals per epoch; then
 * out[3+2k], out[4+2k] = chunk range of interval k, for k < min(J, max_out). Returns J. */
int64_t w2v_dist_plan(int64_t n_global, int32_t L, int32_t world, int32_t rank,
                      int64_t sync_period_words, int64_t* out, int64_t max_out);

/* Pure host (no device needed): the part of an averaged float range [off, off+n) of the model
 * that rank `rank` of `world` reduces and broadcasts in the C17 device average (option
 * "sync_device"; PAPER.md:154-157 periodic synchronisation, reading R13): out[0..3] = s0, a0, a1,
 * s1 — its floats [s0, s1) = [off + n*rank/world, off + n*(rank+1)/world), a scalar head
 * [s0, a0) up to the first 16-B aligned float, a float4 body [a0, a1), a scalar tail [a1, s1).
 * The kernel uses exactly this arithmetic. EINVAL on negative sizes or rank outside [0, world). */
int w2v_dist_sync_slice(int64_t off, int64_t n, int32_t world, int32_t rank, int64_t out[4]);

/* Free everything (model, tables, buffers, NCCL communicator). Safe to call twice. */
int w2v_finalize(void);

const char* w2v_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* W2V_H_ */
