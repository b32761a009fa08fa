// hogbatch.cu — the fused HogBatch step, sm_100a.
//
// One WARP is one work unit. It claims whole chunks (C5) from a global counter in increasing
// corpus order. The chunk's batch stream (kept words, offsets/b, shared negatives: rows a1/a2,
// batch.cu) arrives by cp.async; then per kept target, in chunk order (targets of a chunk are
// sequential, R11):
//   a3  gather the N context rows of M_in and the K+1 rows of M_out into the warp's smem slab:
//       one bulk copy (cp.async.bulk, the TMA engine) per row, completing on an mbarrier —
//       the snapshot of R11, no register staging, ~1 instruction per row
//   a4  C = A·Bᵀ: lane owns float2 columns d = 2·lane + 64c; B and the ΔOut accumulators live
//       in registers; rows are zero-padded to 64·CP2 floats in smem so no predicates remain;
//       packed fp32 FMA (FFMA2, fma.rn.f32x2 — two IEEE fmaf per issue slot); the N x (K+1)
//       partial dots are finished by a butterfly reduce-scatter (lane ends with one dot). No
//       tensor cores: the tiles are <= 16x16 (fp32 parity would also need 3xTF32)
//   a5  E = [j=0] − σ(C) once per lane, G = αE through smem; loss in fp64
//   a6  ΔIn_i = G_i·B written over A_i in smem; ΔOut_j += G_ij·A_i in registers, then over B_j
//   a7  Hogwild scatter: one bulk fp32 reduce-add per row
//       (cp.reduce.async.bulk .add.f32, element-atomic at L2); the warp waits for completion
//       before the next target's gather so a chunk's targets see each other's updates.
// The next target's row list and negatives are prepared while the rows fly.
// Paper mapping: Alg.1 loops over inputs and outputs one dot at a time;
// HogBatch batches them into C = A·Bᵀ and the two update GEMMs; the
// "write back at the end of the GEMM" is the scatter of a7.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "hogbatch_common.cuh"

namespace w2v {

#if defined(W2V_PHASE_TIMING)
// (experiment) cycles per phase summed over warps: chunk load, gather issue->landed, compute,
// scatter issue->complete, targets
__device__ unsigned long long g_phase[8];
#define W2V_T(...) __VA_ARGS__
#else
#define W2V_T(...)
#endif

namespace {

// ---- mode 2 (NEXT-4): acquire/release on the ticket counters and the chunk turn
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* a) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* a, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_add_u32(uint32_t* a, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
// order this thread's async-proxy (bulk copy) global accesses with its generic ones
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

constexpr int kSmemChunk = 256;  // chunks up to this many (padded) kept slots are staged in smem
// long chunks: ring of kept slots (ids, offsets) in smem, staged kKBlock = 8 slots at a time up to
// slot m+4+w at iteration m; the slots still read after that span [m+1-w, m+w+11], so the ring
// needs >= 2w + 11 slots: 32 up to window 10 (cfg4's window 8: 512 B less per unit than a
// 64-slot ring, which is what lets a 12th unit fit at D = 128), 64 up to 26, 128 up to 32.
constexpr int kKBlock = 8;
// negatives of the next targets, staged by cp.async: a ring of 8 targets refilled 4 at a time
// (load_chunk brings the first 8), so a target's group is >= 3 iterations old when it is read
constexpr int kNegRows = 8;
constexpr int kNegGrp = 4;
__host__ __device__ constexpr int kring_slots(int window) {
    return 2 * window + 11 <= 32 ? 32 : 2 * window + 11 <= 64 ? 64 : 128;
}

#ifndef W2V_MINB
#define W2V_MINB 12  // resident 1-warp CTAs per SM the register budget is sized for: 168 registers
                     // (3 warps per SM sub-partition) whether 11 or 12 fit; smem decides (D=300:
                     // 11; cfg4's D=128: 12)
#endif

// CP2 = float2 columns per lane (lane owns d = 2*(lane + 32*c2) + {0,1}, D <= 64*CP2);
// KP1MAX >= K+1 (register tile of the K+1 output rows).
// RSC: compile-time smem row stride of the slab (floats); 0 = padded to 64*CP2 (predicate-free).
// The packed instance for the paper's D=300 (RSC=300) saves 20 floats per row — what lets an 11th
// work unit fit per SM — at the cost of a predicate on each lane's last float2 column.
// TK: the mode-2 (NEXT-4) ticketed instance; the others carry none of its code or registers
// tmap (p.tma_gather): the model as a 2-D fp32 tensor [V][2*Ds] with a box of D x 1; a group of 4
// rows of one matrix lands as 4 consecutive slab rows (RS == D) with one tile::gather4
template <int CP2, int KP1MAX, int RSC, bool TK>
__global__ void __launch_bounds__(32, W2V_MINB) hogbatch_step_kernel(const StepParams p,
                                                                     const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int TI = 32 / KP1MAX;  // inputs per reduce-scatter tile
    const int lane = threadIdx.x & 31;
    unsigned char* wbase = smem + (threadIdx.x >> 5) * p.warp_bytes;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase);
    int32_t* nk_s = reinterpret_cast<int32_t*>(wbase + 8);   // kept count of the chunk
    const int D = p.D, Ds = p.Ds, K = p.K, KP1 = K + 1, window = p.window, RMAX = 2 * window + KP1;
    const int KS = K > 0 ? K : 1;
    // kept ids / (offset << 8) | b of the chunk: staged in smem for short chunks; long ones (L >
    // kSmemChunk) are read in place from the batch stream (global, generic loads), which keeps a
    // unit's smem at the slab's size — at L = 1000 that is 8 KB, i.e. 3 more units per SM
    const bool chunk_smem = p.Lp <= kSmemChunk;
    // long chunks with window <= 32: a ring of kring_slots kept slots (ids and offsets), staged 8
    // slots at a time by cp.async ahead of the targets that read them (an L2 round trip per
    // slot on the critical path otherwise: DESIGN.md §8, cfg4)
    const bool kring_on = !chunk_smem && window <= 32;
    int32_t* kid_s = reinterpret_cast<int32_t*>(wbase + 16);
    const int KR = kring_slots(window);
    const int Lps = chunk_smem ? p.Lp : kring_on ? KR : 0;
    int32_t* rowid0 = kid_s + 2 * Lps;                        // 2 x RMAX: ctx ids, target, negatives
    int32_t* negs = rowid0 + 2 * RMAX;                        // kNegRows x KS negatives ring
    float* gs = reinterpret_cast<float*>(negs + kNegRows * KS);  // G of the target, [N][KP1MAX]
    constexpr int RS = RSC > 0 ? RSC : 64 * CP2;             // smem row stride (floats)
    // wide output tiles finish their dots through a transpose in the B slab (see a4); it needs
    // 32 x 36 floats of it
#ifndef W2V_TRANSPOSE_MIN_KP1
#define W2V_TRANSPOSE_MIN_KP1 16
#endif
    constexpr bool kTransposeDots = KP1MAX >= W2V_TRANSPOSE_MIN_KP1 && KP1MAX * RS >= 32 * 36;
    const bool lastok = RS >= 64 * CP2 || 2 * lane + 64 * (CP2 - 1) < D;  // lane's last float2 column exists
    float* Bs = reinterpret_cast<float*>(wbase + p.slab_offset);  // KP1MAX rows: target, negatives
    float* As = Bs + KP1MAX * RS;                             // 2*window rows: context
    const uint32_t rowbytes = (uint32_t)D * 4u;

    const int64_t shard_end = p.shard_start + p.n_local;

    const uint64_t pol_hot = (p.l2_hint & 1) ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_cold = (p.l2_hint & 2) ? policy_evict_first() : policy_evict_normal();
    if (lane == 0) mbar_init(mbar, 1);
    for (int i = lane; i < (KP1MAX + 2 * window) * RS / 4; i += 32)
        reinterpret_cast<float4*>(Bs)[i] = make_float4(0.f, 0.f, 0.f, 0.f);  // padding stays 0
    __syncwarp();
    uint32_t phase = 0;

    W2V_T(unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};)
    unsigned long long st_words = 0, st_targets = 0, st_touch = 0, st_pairs = 0, st_tail_pairs = 0;
    unsigned st_cold = 0;  // this lane's gathered rows with id >= cold_from
    float st_loss_f = 0.f;
    double st_loss = 0.0, st_tail = 0.0;

    // ---- C6: context ids, target and its (already sampled) negatives of kept target m
    const int32_t* kid = kid_s;    // set per chunk: the whole chunk in smem, the ring, or global
    const int32_t* kinfo = kid_s + Lps;
    int kmask = -1;                // slot index mask (KR - 1 for the ring)
    const int32_t* kid_g = nullptr;    // the chunk's kept list in the batch stream (global)
    const int32_t* kinfo_g = nullptr;
    int kb_hi = 0;                 // ring: 32-slot blocks staged so far
    auto stage_block = [&](int blk) {  // ring: slots [8 blk, 8 blk + 8) of ids and offsets
        const int q = kKBlock * blk + 4 * (lane & 1);
        if (lane < 4 && q < p.Lp) {
            const int32_t* src = (lane < 2 ? kid_g : kinfo_g) + q;
            cp_async16(kid_s + (lane < 2 ? 0 : KR) + (q & (KR - 1)), src);
        }
    };
    auto gather_list = [&](int m, int nk, int32_t* rowid) -> int {
        const int b = kinfo[m & kmask] & 255;
        const int lo = m - b < 0 ? 0 : m - b;
        const int hi = m + b > nk - 1 ? nk - 1 : m + b;
        const int N = hi - lo;
        for (int i = lane; i < N; i += 32) rowid[i] = kid[(lo + i + (lo + i >= m ? 1 : 0)) & kmask];
        if (lane == 0) rowid[N] = kid[m & kmask];
        const int32_t* ng = negs + (m % kNegRows) * KS;
        for (int k = lane; k < K; k += 32) rowid[N + 1 + k] = ng[k];
        return N;
    };

    for (;;) {
        long long s = 0;
        if (lane == 0) s = (long long)atomicAdd(p.chunk_ctr, 1ull) + p.chunk_lo;
        s = __shfl_sync(kFull, s, 0);
        if (s >= p.chunk_hi) break;
        int64_t c0 = s * (int64_t)p.L, c1 = c0 + p.L;
        if (c1 > shard_end) c1 = shard_end;
        if (c0 < p.shard_start) c0 = p.shard_start;
        const int cnt = (int)(c1 - c0);
        const int64_t rel = s - p.chunk_lo;
        constexpr bool ticketed = TK;
        if (cnt <= 0) {
            if (ticketed) {  // an empty chunk still passes the turn on
                if (lane == 0) {
                    while (ld_acquire_u64(p.turn) != (unsigned long long)rel) __nanosleep(20);
                    st_release_u64(p.turn, (unsigned long long)rel + 1);
                }
                __syncwarp();
            }
            continue;
        }

        // ---------------- the chunk's batch stream (a1/a2 rows, batch.cu)
        W2V_T(long long t0 = clock64();)
        kid_g = p.bt_kid + rel * p.Lp;
        kinfo_g = p.bt_kinfo + rel * p.Lp;
        if (chunk_smem) {
            kid = kid_s;
            kinfo = kid_s + Lps;
            kmask = -1;
        } else {
            if (lane == 0) {  // the chunk's kept list, read target by target below, into L2 now
                bulk_prefetch_l2(kid_g, (uint32_t)p.Lp * 4u);
                bulk_prefetch_l2(kinfo_g, (uint32_t)p.Lp * 4u);
            }
            if (kring_on) {   // first blocks: every slot gather_list(0) and (1) can read
                kid = kid_s;
                kinfo = kid_s + KR;
                kmask = KR - 1;
                for (kb_hi = 0; kKBlock * kb_hi < p.Lp && kKBlock * kb_hi <= window + 3; ++kb_hi) stage_block(kb_hi);
            } else {
                kid = kid_g;
                kinfo = kinfo_g;
                kmask = -1;
            }
        }
        load_chunk<kNegRows>(p, rel, chunk_smem ? kid_s : nullptr, kid_s + Lps, nk_s, negs, lane);
        cp_async_wait_all();
        __syncwarp();
        W2V_T(ph[0] += clock64() - t0;)
        const int nk = *nk_s;
        if (lane == 0) st_words += (unsigned long long)cnt;
        uint32_t* tick = p.tick_off >= 0 ? reinterpret_cast<uint32_t*>(wbase + p.tick_off)  // [nk][RMAX] (mode 2)
                                         : p.tick_glob + (size_t)blockIdx.x * p.Lp * RMAX;
        if (ticketed) {
            // NEXT-4 (dependences between iterations): chunks take their turn in
            // corpus order; during its turn a chunk takes one ticket per row access of each of
            // its targets, in sequential order. A target later waits, per row, until every
            // earlier access of that row has completed (done == its first ticket), so each row
            // sees exactly the sequential order of updates while non-conflicting targets of
            // different chunks run in parallel — bit-identical to mode 1.
            if (lane == 0)
                while (ld_acquire_u64(p.turn) != (unsigned long long)rel) __nanosleep(20);
            __syncwarp();
            if (nk >= 2) {
                const int32_t* kidx = chunk_smem ? kid_s : kid_g;   // the whole chunk
                const int32_t* kinfx = chunk_smem ? kid_s + Lps : kinfo_g;
                for (int m = 0; m < nk; ++m) {
                    const int b = kinfx[m] & 255;
                    const int lo = m - b < 0 ? 0 : m - b;
                    const int hi = m + b > nk - 1 ? nk - 1 : m + b;
                    const int N = hi - lo;
                    for (int r = lane; r < N + KP1; r += 32) {
                        const int32_t id = r < N ? kidx[lo + r + (lo + r >= m ? 1 : 0)]
                                         : r == N ? kidx[m] : p.bt_neg[(rel * p.Lp + m) * KS + (r - N - 1)];
                        tick[m * RMAX + r] = atomicAdd(p.tick_issue + (r < N ? 0 : p.V) + id, 1u);
                    }
                }
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) st_release_u64(p.turn, (unsigned long long)rel + 1);
        }
        if (nk < 2) continue;  // N = 0 for every kept target iff the chunk keeps < 2 words

        // alpha (C8): recomputed only when a target crosses into the next Q-quantum
        int64_t q_next = -1;
        float alpha = 0.f;

        int samp_hi = nk < kNegRows ? nk : kNegRows;  // negatives of [0, samp_hi) are in the ring (load_chunk)
        int buf = 0;
        int N = gather_list(0, nk, rowid0);
        __syncwarp();
        for (int m = 0; m < nk; ++m) {
            int32_t* rowid = rowid0 + buf * RMAX;
            const int R = N + KP1;
            const int64_t pp = c0 + (kinfo[m & kmask] >> 8);
            // mode 2: wait until every earlier access of each of this target's rows completed
            uint32_t my_first = 0, my_mult = 0;   // lane r < R: first ticket of row r's (matrix, id), multiplicity
            if (ticketed) {
                if (lane < R) {
                    const int32_t id = rowid[lane];
                    const bool outside = lane >= N;
                    my_first = tick[m * RMAX + lane];
                    for (int r2 = 0; r2 < R; ++r2)
                        if ((r2 >= N) == outside && rowid[r2] == id) {
                            const uint32_t t2 = tick[m * RMAX + r2];
                            my_first = t2 < my_first ? t2 : my_first;
                            ++my_mult;
                        }
                    if (my_first != tick[m * RMAX + lane]) my_mult = 0;  // released by the first occurrence
                    const uint32_t* dn = p.tick_done + (outside ? p.V : 0) + id;
                    while (ld_acquire_u32(dn) != my_first) __nanosleep(20);
                }
                __syncwarp();
                fence_proxy_async_global();
            }
            // ---------------- a3: gather the snapshot rows (one bulk copy per row)
            W2V_T(long long t1 = clock64();)
            if (p.tma_gather) {
                // groups of 4 rows per TMA instruction (SURVEY.md §8(a) "Gather engines"); a
                // group's missing rows repeat its last row (landing in slab rows the compute
                // and the scatter never use: the slab holds 2w >= 4*ceil(N/4) A rows and
                // KP1MAX >= 4*ceil((K+1)/4) B rows, step_tma_gather_ok)
                const int ga = (N + 3) >> 2, gb = (KP1 + 3) >> 2;
                if (lane == 0) mbar_arrive_expect_tx(mbar, (uint32_t)(4 * (ga + gb)) * rowbytes);
                __syncwarp();
                if (lane < ga + gb) {
                    const bool isA = lane < ga;
                    const int r0 = isA ? 4 * lane : N + 4 * (lane - ga), rend = isA ? N : R;
                    int32_t id[4];
                    bool hot = false;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        id[k] = rowid[r0 + k < rend ? r0 + k : rend - 1];
                        hot |= id[k] < (isA ? p.hot_rows_in : p.hot_rows);
                    }
                    tma_gather4_hint(isA ? As + 4 * lane * RS : Bs + 4 * (lane - ga) * RS, &tmap, isA ? 0 : Ds,
                                     id, mbar, hot ? pol_hot : pol_cold);
                }
                for (int r = lane; r < R; r += 32) st_cold += rowid[r] >= p.cold_from;
            } else {
#ifndef W2V_ABL_NOGATHER
            if (lane == 0) mbar_arrive_expect_tx(mbar, (uint32_t)R * rowbytes);
#else
            if (lane == 0) mbar_arrive_expect_tx(mbar, 0u);
#endif
            __syncwarp();
            for (int r = lane; r < R; r += 32) {
                const int32_t id = rowid[r];
                st_cold += id >= p.cold_from;
                float* dst = r < N ? As + r * RS : Bs + (r - N) * RS;
#ifndef W2V_ABL_NOGATHER
                bulk_g2s_hint(dst, p.M + (size_t)id * 2 * Ds + (r < N ? 0 : Ds), rowbytes, mbar,
                              id < (r < N ? p.hot_rows_in : p.hot_rows) ? pol_hot : pol_cold);
#else
                (void)dst; (void)id;
#endif
            }
            }
            // while the rows fly: fetch negatives ahead, build the next target's row list, alpha.
            // One cp.async group per target (possibly empty); targets fetched at iteration m' are
            // >= m'+4 (a group of 4 when fewer than 4 remain ahead of m'+1), so waiting only for
            // the groups at least 3 iterations old covers target m+1 without stalling on the
            // fetch just issued, and the 8-target ring never overwrites one before gather_list
            // has read it.
            if (K > 0 && samp_hi < nk && samp_hi - (m + 1) < kNegGrp) {
                const int c = nk - samp_hi < kNegGrp ? nk - samp_hi : kNegGrp;
                fetch_negs<kNegRows>(p, rel, samp_hi, c, negs, lane);
                samp_hi += c;
            }
            // ring: stage the blocks up to slot m+4+w now — gather_list(m+4) reads up to there at
            // iteration m+3, when this group is 3 iterations old and waited for; the oldest slot
            // still read, m+1-w, stays within KR of the newest staged slot (<= m+w+11; KR >=
            // 2w + 11). The chunk start stages up to w+3 (iterations 0-2) and waits for it.
            if (kring_on)
                for (; kKBlock * kb_hi < nk && kKBlock * kb_hi <= m + 4 + window; ++kb_hi) stage_block(kb_hi);
            cp_async_commit();
            cp_async_wait_but_3();
            __syncwarp();
            const int Nn = (m + 1 < nk) ? gather_list(m + 1, nk, rowid0 + (buf ^ 1) * RMAX) : 0;
            const int64_t pi = (int64_t)p.epoch * p.n_local + (pp - p.shard_start);
            if (pi >= q_next) {
                const int64_t qi = pi / p.Q;
                q_next = (qi + 1) * p.Q;
                alpha = alpha_at(p, qi);
            }
            W2V_T(long long t2 = clock64(); ph[5] += t2 - t1;)
            mbar_wait(mbar, phase);
            phase ^= 1u;
            W2V_T(long long t3 = clock64(); ph[1] += t3 - t1;)

            // ---------------- a4-a6: C = A·Bᵀ, E, G, ΔIn (over A), ΔOut (registers, then over B)
            // Rows are padded to RS floats and B to KP1MAX rows with zeros (never written by
            // the bulk copies), so the compute needs no column or row predicates. Inputs go in
            // tiles of TI = 32/KP1MAX: the TI*KP1MAX partial dots of a tile are finished by ONE
            // butterfly reduce-scatter (lane l ends with dot l = t*KP1MAX + j), σ/G/loss once per
            // lane, G through smem; then per input: ΔOut += G·A (snapshot) and ΔIn over A.
#ifndef W2V_ABL_NOCOMPUTE
            if (p.rowpath_only) {
                // measurement mode (option "rowpath_only"): the same gathers and scatters with
                // a4-a6 skipped — zero deltas are reduced, the model is unchanged
                float4* z = reinterpret_cast<float4*>(Bs);
                for (int u = lane; u < (KP1MAX + 2 * window) * RS / 4; u += 32) z[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
            float2 bq[KP1MAX][CP2], dq[KP1MAX][CP2];
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CP2; ++c) {
                    bq[j][c] = (c < CP2 - 1 || lastok) ? *reinterpret_cast<const float2*>(Bs + j * RS + 2 * lane + 64 * c)
                                                       : make_float2(0.f, 0.f);
                    dq[j][c] = make_float2(0.f, 0.f);
                }
            const int tt = lane / KP1MAX, tj = lane - tt * KP1MAX;  // dot held after the reduce-scatter
            for (int i0 = 0; i0 < N; i0 += TI) {
                float v[32];
#pragma unroll
                for (int t = 0; t < TI; ++t) {
#if !defined(W2V_DOT_FULL_TILE)
                    if (i0 + t >= N) {  // warp-uniform: the last tile's missing inputs cost nothing
#pragma unroll
                        for (int j = 0; j < KP1MAX; ++j) v[t * KP1MAX + j] = 0.f;
                        continue;
                    }
#endif
                    const float* Ai = As + (i0 + t < N ? i0 + t : 0) * RS + 2 * lane;
                    float2 a[CP2];
#pragma unroll
                    for (int c = 0; c < CP2; ++c)
                        a[c] = (c < CP2 - 1 || lastok) ? *reinterpret_cast<const float2*>(Ai + 64 * c) : make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < KP1MAX; ++j) {
                        float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int c = 0; c < CP2; ++c) s2 = ffma2(a[c], bq[j][c], s2);
                        v[t * KP1MAX + j] = s2.x + s2.y;
                    }
                }
#pragma unroll
                for (int u = TI * KP1MAX; u < 32; ++u) v[u] = 0.f;
                float dot;
                if constexpr (kTransposeDots) {
                    // many outputs per tile (K+1 >= 16: two inputs per tile, ~4.5 tiles per
                    // target at cfg4): finish the 32 dots through a 32 x 36 transpose in the B
                    // slab, whose rows are already in registers (bq) and are only rewritten with
                    // ΔOut after a6 — 8 STS.128 + 32 LDS + 31 FADD instead of the butterfly's
                    // 31 SHFL + 62 FSEL + 31 FADD. Lane l sums column l = dot l, as below.
                    float* T = Bs;
                    __syncwarp();  // the previous tile's column reads are done
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        *reinterpret_cast<float4*>(T + lane * 36 + 4 * k) =
                            make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    __syncwarp();
                    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int r = 0; r < 32; ++r) acc[r & 3] += T[r * 36 + lane];
                    dot = (acc[0] + acc[1]) + (acc[2] + acc[3]);
                } else {
#pragma unroll
                for (int st = 0; st < 5; ++st) {
                    const int o = 16 >> st;
                    const bool up = lane & o;
#pragma unroll
                    for (int u = 0; u < o; ++u) {
                        const float send = up ? v[u] : v[u + o];
                        const float keep = up ? v[u + o] : v[u];
                        v[u] = keep + __shfl_xor_sync(kFull, send, o);
                    }
                }
                dot = v[0];
                }
                const bool valid = tt < TI && i0 + tt < N && tj < KP1;
                const float ex = expf(-fabsf(dot));
                const float rc = __frcp_rn(1.0f + ex);
                const float sg = dot >= 0.f ? rc : ex * rc;
                const bool pos = (tj == 0);
                if (lane < TI * KP1MAX) gs[i0 * KP1MAX + lane] = valid ? alpha * ((pos ? 1.0f : 0.0f) - sg) : 0.f;
                if (valid) st_loss_f += fmaxf(pos ? -dot : dot, 0.f) - __logf(rc);
            }
            __syncwarp();
            for (int i = 0; i < N; ++i) {
                float* Ai = As + i * RS + 2 * lane;
                float2 a[CP2];
#pragma unroll
                for (int c = 0; c < CP2; ++c)
                    a[c] = (c < CP2 - 1 || lastok) ? *reinterpret_cast<const float2*>(Ai + 64 * c) : make_float2(0.f, 0.f);
                float2 g2[KP1MAX];
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) {
                    const float gj = gs[i * KP1MAX + j];
                    g2[j] = make_float2(gj, gj);
                }
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                    for (int c = 0; c < CP2; ++c) dq[j][c] = ffma2(g2[j], a[c], dq[j][c]);
#pragma unroll
                for (int c = 0; c < CP2; ++c) {
                    // ΔIn_i = Σ_j G_ij B_j: with many outputs and few columns (cfg4: 16 x 2) the
                    // single FFMA2 chain is latency-bound, so it runs as NCH interleaved chains
                    constexpr int NCH = (KP1MAX >= 8 && CP2 <= 2) ? 4 : 1;
                    float2 s2[NCH];
#pragma unroll
                    for (int h = 0; h < NCH; ++h) s2[h] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < KP1MAX; ++j) s2[j % NCH] = ffma2(g2[j], bq[j][c], s2[j % NCH]);
#pragma unroll
                    for (int h = 1; h < NCH; ++h) s2[0] = fadd2(s2[0], s2[h]);
                    if (c < CP2 - 1 || lastok) *reinterpret_cast<float2*>(Ai + 64 * c) = s2[0];
                }
            }
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CP2; ++c)
                    if (c < CP2 - 1 || lastok) *reinterpret_cast<float2*>(Bs + j * RS + 2 * lane + 64 * c) = dq[j][c];
            }
#endif  // W2V_ABL_NOCOMPUTE
            fence_proxy_async_smem();
            __syncwarp();

            W2V_T(long long t4 = clock64(); ph[2] += t4 - t3;)
            // ---------------- a7: Hogwild scatter-add, one bulk fp32 reduction per row at L2
            for (int r = lane; r < R; r += 32) {
                const int32_t id = rowid[r];
                const float* src = r < N ? As + r * RS : Bs + (r - N) * RS;
#if defined(W2V_ABL_NOHOT)
                if (id < W2V_ABL_NOHOT) continue;
#endif
#ifndef W2V_ABL_NOSCATTER
                bulk_red_add_s2g_hint(p.M + (size_t)id * 2 * Ds + (r < N ? 0 : Ds), src, rowbytes,
                                      id < (r < N ? p.hot_rows_in : p.hot_rows) ? pol_hot : pol_cold);
#else
                (void)src; (void)id;
#endif
            }
            bulk_commit();
            st_loss += (double)st_loss_f;   // per-target partial (<= N terms) into fp64 (C11)
            if (pp >= p.loss_tail_from) {
                st_tail += (double)st_loss_f;
                if (lane == 0) st_tail_pairs += (unsigned long long)N * KP1;
            }
            st_loss_f = 0.f;
            if (lane == 0) {
                st_targets += 1;
                st_touch += (unsigned long long)R;
                st_pairs += (unsigned long long)N * KP1;
            }
            if (p.dbg_len && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len) {
                const int64_t q = pp - p.dbg_base;
                if (lane == 0) p.dbg_N[q] = (uint8_t)N;
                for (int i = lane; i < N; i += 32) p.dbg_ctx[q * 2 * window + i] = rowid[i];
                for (int k = lane; k < K; k += 32) p.dbg_neg[q * K + k] = rowid[N + 1 + k];
            }
            // the next target's gather must see these updates (R11: targets of a chunk are
            // sequential) and the slab must be free: wait for the reductions to complete
#if !defined(W2V_ABL_NOWAIT)
            // (option scatter_wait = 0, Hogwild only: wait just until the sources are read; see
            // hogbatch_ring.cu)
            if (p.deterministic || p.scatter_wait) bulk_wait_all();
            else bulk_wait_read_all();
#else
            bulk_wait_read_all();
#endif
            if (p.deterministic) __threadfence();
            if (ticketed) {  // mode 2: this target's accesses are complete: release the rows
                fence_proxy_async_global();
                __threadfence();
                if (lane < R && my_mult) red_release_add_u32(p.tick_done + (lane >= N ? p.V : 0) + rowid[lane], my_mult);
            }
            __syncwarp();
            W2V_T(ph[3] += clock64() - t4; ph[4] += 1;)
            N = Nn;
            buf ^= 1;
        }
    }

    // flush per-warp statistics
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        st_loss += __shfl_xor_sync(kFull, st_loss, o);
        st_tail += __shfl_xor_sync(kFull, st_tail, o);
        st_cold += __shfl_xor_sync(kFull, st_cold, o);
    }
    W2V_T(if (lane == 0) for (int i = 0; i < 8; ++i) atomicAdd(&g_phase[i], ph[i]);)
    if (lane == 0) {
        atomicAdd(&p.stats->words, st_words);
        atomicAdd(&p.stats->targets, st_targets);
        atomicAdd(&p.stats->row_touches, st_touch);
        atomicAdd(&p.stats->loss_pairs, st_pairs);
        atomicAdd(&p.stats->loss_sum, st_loss);
        atomicAdd(&p.stats->row_touches_cold, (unsigned long long)st_cold);
        if (st_tail_pairs) {
            atomicAdd(&p.stats->loss_tail_sum, st_tail);
            atomicAdd(&p.stats->loss_tail_pairs, st_tail_pairs);
        }
    }
}

using KernelFn = void (*)(const StepParams, const CUtensorMap);

struct Inst {
    int cp2, kp1, rs;  // rs: packed row stride (the instance serves D == rs only), 0 = padded
    KernelFn fn, fn_tk;  // Hogwild / mode 1, and the mode-2 (ticketed) instance
};

#define W2V_INST(C, KK) {C, KK, 0, hogbatch_step_kernel<C, KK, 0, false>, hogbatch_step_kernel<C, KK, 0, true>}
// (float2 columns per lane, max K+1) instantiations; register tile ~ 4*CP2*KP1MAX floats.
const Inst kInst[] = {
    W2V_INST(1, 2), W2V_INST(1, 4), W2V_INST(1, 6), W2V_INST(1, 8), W2V_INST(1, 16), W2V_INST(1, 32),
    W2V_INST(2, 2), W2V_INST(2, 4), W2V_INST(2, 6), W2V_INST(2, 8), W2V_INST(2, 16),
    W2V_INST(3, 2), W2V_INST(3, 4), W2V_INST(3, 6), W2V_INST(3, 8), W2V_INST(3, 16),
    W2V_INST(4, 2), W2V_INST(4, 4), W2V_INST(4, 6), W2V_INST(4, 8),
    W2V_INST(5, 2), W2V_INST(5, 4), W2V_INST(5, 6), W2V_INST(5, 8),
    W2V_INST(8, 2), W2V_INST(8, 4), W2V_INST(8, 6),
    {5, 6, 300, hogbatch_step_kernel<5, 6, 300, false>, hogbatch_step_kernel<5, 6, 300, true>},  // D=300, K<=5, packed
};
// Supported envelope (w2v_init rejects the rest): ceil(D/64) float2 columns per lane times
// the padded K+1 tile must be one of the rows above, i.e. D <= 64 with K <= 31; D <= 128 with
// K <= 15; D <= 192 with K <= 15; D <= 320 with K <= 7; D <= 512 with K <= 5.
#undef W2V_INST

const Inst* pick(int D, int K) {
    const int need = (D + 63) / 64, kp1 = K + 1;
    const char* pad = getenv("W2V_SLAB_PAD");
    const bool packed_ok = !(pad && pad[0] == '1');
    for (const Inst& in : kInst)  // a packed instance made for exactly this D wins
        if (packed_ok && in.rs == D && in.cp2 >= need && in.kp1 >= kp1) return &in;
    const Inst* best = nullptr;
    for (const Inst& in : kInst) {
        if (in.rs != 0 || in.cp2 < need || in.kp1 < kp1) continue;
        if (!best || in.cp2 * in.kp1 < best->cp2 * best->kp1) best = &in;
    }
    return best;
}

}  // namespace

bool step_supported(int D, int K) { return pick(D, K) != nullptr; }

void step_phase_report() {
#if defined(W2V_PHASE_TIMING)
    unsigned long long h[8];
    cudaMemcpyFromSymbol(h, g_phase, sizeof h);
    if (!h[4]) return;
    const double T = (double)h[4];
    fprintf(stderr, "[phase] per target (cycles): chunk-load %.0f  gather->landed %.0f (issue+prep %.0f)  compute %.0f  scatter->done %.0f  targets %llu\n",
            h[0] / T, h[1] / T, h[5] / T, h[2] / T, h[3] / T, h[4]);
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase, z, sizeof z);
#endif
}

size_t step_warp_bytes(int L, int window, int K, int D, int32_t* slab_offset, int32_t* tick_offset) {
    // [mbarrier 8 B | nk 4 B][kid Lp][kinfo Lp][rowid 2 x (2w+K+1)][negs 32 x max(K,1)][G tiles x 32]
    // [slab: KP1MAX B rows + 2w A rows, stride RS fp32]. RS = 64*CP2 (zero padding), or D for a
    // packed instance (W2V_SLAB_PAD=1 forces the padded one; experiments).
    const Inst* in = pick(D, K);
    if (!in) return 0;
    const int RS = in->rs > 0 ? in->rs : 64 * in->cp2;
    const int R = 2 * window + K + 1;
    const int TI = 32 / in->kp1;
    const size_t gfl = (size_t)((2 * window + TI - 1) / TI) * 32;
    const int Lp = (L + 3) & ~3;
    // long chunks: a kring_slots(window)-slot ring (window <= 32), else read from the batch stream
    const int Lps = Lp <= kSmemChunk ? Lp : window <= 32 ? kring_slots(window) : 0;
    const size_t ids = 16 + (size_t)(2 * Lps + 2 * R + kNegRows * (K > 0 ? K : 1)) * 4 + gfl * 4;
    // 16-B aligned slab (bulk copies; every byte counts), 128-B aligned where the TMA gather4
    // path may run (tensor destinations)
    const size_t align = step_tma_gather_ok(D, K, window) ? 128 : 16;
    const size_t off = (ids + align - 1) / align * align;
    if (slab_offset) *slab_offset = (int32_t)off;
    const size_t end = off + (size_t)(in->kp1 + 2 * window) * RS * 4;
    if (tick_offset) {  // mode 2: + a ticket table [Lp][2w+K+1] u32 after the slab
        *tick_offset = (int32_t)end;
        return end + (size_t)Lp * R * 4;
    }
    return end;
}

int step_max_ctas_per_sm(const StepParams& p) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return 0;
    const KernelFn fn = p.deterministic == 2 ? in->fn_tk : in->fn;
    int n = 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, 32, p.warp_bytes) != cudaSuccess) return 0;
    return n;
}

cudaError_t launch_step(const StepParams& p, int ctas, cudaStream_t st, const CUtensorMap* tmap) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return cudaErrorInvalidValue;
    if (p.tma_gather && !tmap) return cudaErrorInvalidValue;
    const KernelFn fn = p.deterministic == 2 ? in->fn_tk : in->fn;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (e != cudaSuccess) return e;
    CUtensorMap none;
    std::memset(&none, 0, sizeof none);
    fn<<<ctas, 32, p.warp_bytes, st>>>(p, tmap ? *tmap : none);
    return cudaGetLastError();
}

// TMA tile::gather4 for the rows kernel: one box of D fp32 columns per row (D <= 256, 16-B
// multiple), slab rows packed at RS == D, and whole groups of 4 fitting the slab: 2*window and
// KP1MAX multiples of 4
bool step_tma_gather_ok(int D, int K, int window) {
    const Inst* in = pick(D, K);
    if (!in) return false;
    const int RS = in->rs > 0 ? in->rs : 64 * in->cp2;
    return D <= 256 && RS == D && (2 * window) % 4 == 0 && in->kp1 % 4 == 0;
}

}  // namespace w2v
