// hogbatch_ring.cu — the fused HogBatch step with a window RING of M_in rows whose original
// values live in TENSOR MEMORY (SURVEY.md §8(a) rows a3-a7 and §8(f) NEXT-1 "sentence-tiled row
// reuse"), sm_100a. Same math, contract and per-target order as hogbatch.cu; different M_in
// data movement:
//
//  * The context of kept target m is a subset of kept positions [m-w, m+w] of its chunk. Those
//    positions' M_in rows stay in a ring of S = 2w+1 shared-memory slots (one slot per distinct
//    word: repeated words share it, reference-counted). Position q ENTERS when target q-w starts
//    (one bulk copy unless its word is already in the ring) and LEAVES after target q+w — the
//    last one whose window can reach it (b <= w, C4).
//  * Targets update the slot in place (slot += ΔIn_i), so the chunk's later targets read the
//    updated rows exactly as the sequential algorithm does (R11).
//  * On entry the row's ORIGINAL value is also written to the warp's columns of TMEM
//    (tcgen05.st; 256 KB per SM that this path would otherwise leave idle). On leaving, the
//    slot's total update is recovered as  delta = slot - original  (tcgen05.ld) and written
//    back with ONE bulk fp32 reduce-add (cp.reduce.async.bulk .add.f32), so concurrent work
//    units' updates to the same row are never lost (Hogwild). In the
//    deterministic mode the global row still holds the original when the slot leaves, and
//    original + (slot - original) == slot exactly whenever slot/original lies in [1/2, 2]
//    (Sterbenz): the result is the sequential one up to that last rounding.
//  * M_out rows (target + K shared negatives) are gathered and reduced per target exactly as in
//    hogbatch.cu, and each target waits for its reductions before the next gather.
// So M_in costs ~1 gather + 1 reduction per kept position instead of N per target: at cfg3
// the rows moved per target fall from N+K+1 = 11.05 to ~K+1+1.
//
// TMEM layout: the CTA (one per SM, UPC warps = work units) allocates the TMEM columns once;
// warp u may address lanes 32*(u%4)..+31 (its sub-partition) and owns columns
// [(u/4)*CW, (u/4)*CW + CW), CW = S * 2*CP2 — slot s, lane l holds the lane's 2*CP2 floats of
// the row (d = 2l + 64c + {0,1}, c < CP2), the same layout the compute keeps in registers.
// Paper mapping: PAPER.md:116-126 (HogBatch GEMMs, write-back at the end), :140-149 ("cut down
// on the total number of updates"), :135-138 (Hogwild across work units).
#include <cstdio>

#include "hogbatch_common.cuh"

namespace w2v {

namespace {

constexpr int kRingSmemChunk = 256;  // chunks up to this many (padded) kept slots are staged in smem
#ifndef W2V_RING_WARPS
#define W2V_RING_WARPS 11
#endif
constexpr int kRingMaxWarps = W2V_RING_WARPS;  // work units per CTA (one CTA per SM in Hogwild mode)
constexpr int kRingNegRows = 8;      // ring of targets whose negatives are staged in smem
constexpr int kRingNegGrp = 4;       // fetched 4 at a time, >= 3 targets ahead of use

// ---- tcgen05 (TMEM) primitives: all are .sync.aligned (the whole warp, converged) ----------
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st2(uint32_t ta, float a, float b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(ta), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b))
                 : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t ta, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta), "r"(__float_as_uint(v[0])),
                 "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3]))
                 : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t ta, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(ta),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
        : "memory");
}
__device__ __forceinline__ void tmem_ld2(uint32_t ta, float* v) {
    uint32_t a, b;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(ta) : "memory");
    v[0] = __uint_as_float(a); v[1] = __uint_as_float(b);
}
__device__ __forceinline__ void tmem_ld4(uint32_t ta, float* v) {
    uint32_t a, b, c, d;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(ta)
                 : "memory");
    v[0] = __uint_as_float(a); v[1] = __uint_as_float(b); v[2] = __uint_as_float(c); v[3] = __uint_as_float(d);
}
__device__ __forceinline__ void tmem_ld8(uint32_t ta, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta)
                 : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// N = 2*CP2 consecutive columns from/to v[0..N): decomposed into x8 / x4 / x2 pieces
template <int N>
__device__ __forceinline__ void tmem_store_row(uint32_t ta, const float* v) {
    int c = 0;
#pragma unroll
    for (; c + 8 <= N; c += 8) tmem_st8(ta + c, v + c);
    if (N - c >= 4) { tmem_st4(ta + c, v + c); c += 4; }
    if (N - c >= 2) tmem_st2(ta + c, v[c], v[c + 1]);
}
template <int N>
__device__ __forceinline__ void tmem_load_row(uint32_t ta, float* v) {
    int c = 0;
#pragma unroll
    for (; c + 8 <= N; c += 8) tmem_ld8(ta + c, v + c);
    if (N - c >= 4) { tmem_ld4(ta + c, v + c); c += 4; }
    if (N - c >= 2) tmem_ld2(ta + c, v + c);
}

constexpr int ring_tmem_cols(int window, int cp2) { return (2 * window + 1) * 2 * cp2; }

uint32_t pow2_cols(uint32_t c) {
    uint32_t n = 32;
    while (n < c) n <<= 1;
    return n;
}

// CP2 = float2 columns per lane (D <= 64*CP2); KP1MAX >= K+1; RSC: packed smem row stride (0 =
// padded to 64*CP2). One WARP = one work unit; a CTA holds `units` of them and one TMEM block.
template <int CP2, int KP1MAX, int RSC>
// registers are partitioned per SM sub-partition (16,384 each): 11 warps put 3 on some
// sub-partitions, so <= 170 per thread (168; the rows kernel's budget too)
__global__ void __launch_bounds__(32 * kRingMaxWarps, 1) hogbatch_ring_kernel(const StepParams p, int units_cols) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int TI = 32 / KP1MAX;  // inputs per reduce-scatter tile
    constexpr int NC = 2 * CP2;      // TMEM columns per slot (the lane's floats of one row)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ uint32_t tmem_base_s;
    const int D = p.D, Ds = p.Ds, K = p.K, KP1 = K + 1, w = p.window, S = 2 * w + 1;
    const int KS = K > 0 ? K : 1;
    const int nwarps = blockDim.x >> 5;
    const uint32_t tm_cols = (uint32_t)units_cols;   // allocated per CTA (power of 2 >= 32)

    if (wid == 0) tmem_alloc(&tmem_base_s, tm_cols);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    // this warp's TMEM: lanes of its sub-partition, its own column block
    const uint32_t tbase = tmem_base_s + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)((wid >> 2) * S * NC);

    unsigned char* wbase = smem + (size_t)wid * p.warp_bytes;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase);
    int32_t* nk_s = reinterpret_cast<int32_t*>(wbase + 8);
    const bool chunk_smem = p.Lp <= kRingSmemChunk;
    // per-warp launch statistics live in shared memory (lane 0 updates them once per target):
    // registers are the scarce resource at 11 warps per SM
    unsigned long long* wst = reinterpret_cast<unsigned long long*>(wbase + 16);  // [6]
    int32_t* kid_s = reinterpret_cast<int32_t*>(wbase + 64);
    const int Lps = chunk_smem ? p.Lp : 0;
    int32_t* negs = kid_s + 2 * Lps;                           // kRingNegRows x KS negatives ring
    float* gs = reinterpret_cast<float*>(negs + kRingNegRows * KS);  // G of the target, [tiles][32]
    constexpr int RS = RSC > 0 ? RSC : 64 * CP2;
#ifndef W2V_TRANSPOSE_MIN_KP1
#define W2V_TRANSPOSE_MIN_KP1 16
#endif
    constexpr bool kTransposeDots = KP1MAX >= W2V_TRANSPOSE_MIN_KP1 && KP1MAX * RS >= 32 * 36;
    const bool lastok = RS >= 64 * CP2 || 2 * lane + 64 * (CP2 - 1) < D;
    float* Bs = reinterpret_cast<float*>(wbase + p.slab_offset);  // KP1MAX rows: target, negatives
    float* Ring = Bs + KP1MAX * RS;                               // S slots of M_in rows
    const uint32_t rowbytes = (uint32_t)D * 4u;
    const int64_t shard_end = p.shard_start + p.n_local;
    const uint64_t pol_hot = (p.l2_hint & 1) ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_cold = (p.l2_hint & 2) ? policy_evict_first() : policy_evict_normal();
    if (lane == 0) mbar_init(mbar, 1);
    for (int i = lane; i < (KP1MAX + S) * RS / 4; i += 32)
        reinterpret_cast<float4*>(Bs)[i] = make_float4(0.f, 0.f, 0.f, 0.f);  // padding stays 0
    fence_proxy_async_smem();
    __syncwarp();
    uint32_t phase = 0;

    // per-warp counters of one launch; 32 bits where a launch (launch_words <= 2^31 raw words, one
    // unit in deterministic mode) cannot overflow them
    enum { kWords, kTargets, kTouch, kPairs, kTailPairs, kMoved };
    if (lane < 6) wst[lane] = 0;
    unsigned st_cold = 0;
    float st_loss_f = 0.f;
    double st_loss = 0.0, st_tail = 0.0;

    const int32_t* kid = kid_s;
    const int32_t* kinfo = kid_s + Lps;

    for (;;) {
        long long s = 0;
        if (lane == 0) s = (long long)atomicAdd(p.chunk_ctr, 1ull) + p.chunk_lo;
        s = __shfl_sync(kFull, s, 0);
        if (s >= p.chunk_hi) break;
        int64_t c0 = s * (int64_t)p.L, c1 = c0 + p.L;
        if (c1 > shard_end) c1 = shard_end;
        if (c0 < p.shard_start) c0 = p.shard_start;
        const int cnt = (int)(c1 - c0);
        if (cnt <= 0) continue;
        const int64_t rel = s - p.chunk_lo;
        if (chunk_smem) {
            kid = kid_s;
            kinfo = kid_s + Lps;
        } else {
            kid = p.bt_kid + rel * p.Lp;
            kinfo = p.bt_kinfo + rel * p.Lp;
            if (lane == 0) {
                bulk_prefetch_l2(kid, (uint32_t)p.Lp * 4u);
                bulk_prefetch_l2(kinfo, (uint32_t)p.Lp * 4u);
            }
        }
        load_chunk<kRingNegRows>(p, rel, chunk_smem ? kid_s : nullptr, kid_s + Lps, nk_s, negs, lane);
        cp_async_wait_all();
        __syncwarp();
        const int nk = *nk_s;
        if (lane == 0) wst[kWords] += (unsigned long long)cnt;
        if (nk < 2) continue;  // N = 0 for every kept target iff the chunk keeps < 2 words

        // ring state, in registers: lane s < S holds slot s (word id, reference count); lane
        // r holds the slot of the window position q with q & 31 == r (the window spans 2w+1 <= 31
        // positions, so the low five bits are unique in it; no division by S)
        int32_t slot_word = -1, slot_ref = 0, pos_slot = 0;
        uint32_t freem = (S >= 32) ? kFull : ((1u << S) - 1u);
        int next_in = 0;  // next kept position to enter

        int64_t q_next = -1;
        float alpha = 0.f;
        int samp_hi = nk < kSampGrp ? nk : kSampGrp;

        for (int m = 0; m < nk; ++m) {
            const int b = kinfo[m] & 255;
            const int lo = m - b < 0 ? 0 : m - b;
            const int hi = m + b > nk - 1 ? nk - 1 : m + b;
            const int N = hi - lo;
            const int64_t pp = c0 + (kinfo[m] >> 8);
            // ---------------- entries: positions up to m + w join the ring
            uint32_t newm = 0;
            const int in_hi = m + w < nk - 1 ? m + w : nk - 1;
            for (; next_in <= in_hi; ++next_in) {
                const int32_t id = kid[next_in];
                const unsigned hit = __ballot_sync(kFull, lane < S && slot_ref > 0 && slot_word == id);
                int sl;
                if (hit) {
                    sl = __ffs(hit) - 1;
                } else {
                    sl = __ffs(freem) - 1;
                    freem &= ~(1u << sl);
                    newm |= 1u << sl;
                    if (lane == sl) slot_word = id;
                }
                if (lane == sl) slot_ref += 1;
                if (lane == (next_in & 31)) pos_slot = sl;
            }
            // ---------------- a3: gather new ring rows + the K+1 output rows (one bulk copy each)
            const int nnew = __popc(newm);
            if (lane == 0) mbar_arrive_expect_tx(mbar, (uint32_t)(nnew + KP1) * rowbytes);
            __syncwarp();
            if ((newm >> lane) & 1u) {
                st_cold += slot_word >= p.cold_from;
                bulk_g2s_hint(Ring + lane * RS, p.M + (size_t)slot_word * 2 * Ds, rowbytes, mbar,
                              slot_word < p.hot_rows_in ? pol_hot : pol_cold);
            }
            // output rows: target word and its negatives (C7, from the batch stream's ring)
            // (target m's negatives were fetched >= 3 targets ago: complete, see the fetch below)
            const int32_t* ng = negs + (m % kRingNegRows) * KS;
            int32_t oid = 0;
            if (lane < KP1) {
                oid = lane == 0 ? kid[m] : ng[lane - 1];
                st_cold += oid >= p.cold_from;
                bulk_g2s_hint(Bs + lane * RS, p.M + (size_t)oid * 2 * Ds + Ds, rowbytes, mbar,
                              oid < p.hot_rows ? pol_hot : pol_cold);
            }
            // while the rows fly: negatives ahead, context slots and ids, alpha
            // negatives ahead: the chunk load brought targets [0, 8); a group of 4 more is fetched
            // when fewer than 4 remain ahead of m+1, so every group is >= 3 iterations old (its
            // cp.async group long complete) when its first target is read, and the 8-row ring
            // never overwrites a target before it ran
            if (K > 0 && samp_hi < nk && samp_hi - (m + 1) < kRingNegGrp) {
                const int c = nk - samp_hi < kRingNegGrp ? nk - samp_hi : kRingNegGrp;
                fetch_negs<kRingNegRows>(p, rel, samp_hi, c, negs, lane);
                samp_hi += c;
            }
            cp_async_commit();
            // lane i < N: context i = kept position lo + i (+1 past m), its slot and word
            int my_cs = 0;
            {
                const int qpos = lo + lane + (lo + lane >= m ? 1 : 0);
                const int src = (lane < N ? qpos : 0) & 31;
                const int cs = __shfl_sync(kFull, pos_slot, src);
                if (lane < N) {
                    my_cs = cs;
                    st_cold += kid[qpos] >= p.cold_from;
                }
            }
            const int64_t pi = (int64_t)p.epoch * p.n_local + (pp - p.shard_start);
            if (pi >= q_next) {
                const int64_t qi = pi / p.Q;
                q_next = (qi + 1) * p.Q;
                alpha = alpha_at(p, qi);
            }
            cp_async_wait_but_3();   // negatives are fetched >= 4 targets ahead
            mbar_wait(mbar, phase);
            phase ^= 1u;
            __syncwarp();
            // originals of the new slots into TMEM (the rows just landed)
            for (uint32_t nm = newm; nm; nm &= nm - 1) {
                const int sl = __ffs(nm) - 1;
                float v[NC];
#pragma unroll
                for (int c = 0; c < CP2; ++c) {
                    const float2 x = (c < CP2 - 1 || lastok)
                                         ? *reinterpret_cast<const float2*>(Ring + sl * RS + 2 * lane + 64 * c)
                                         : make_float2(0.f, 0.f);
                    v[2 * c] = x.x;
                    v[2 * c + 1] = x.y;
                }
                tmem_store_row<NC>(tbase + (uint32_t)(sl * NC), v);
            }
            if (newm) tmem_wait_st();

            // ---------------- a4-a6 (as hogbatch.cu; A rows are ring slots)
            if (p.rowpath_only) {
                float4* z = reinterpret_cast<float4*>(Bs);
                for (int u = lane; u < KP1MAX * RS / 4; u += 32) z[u] = make_float4(0.f, 0.f, 0.f, 0.f);
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
                const int tt = lane / KP1MAX, tj = lane - tt * KP1MAX;
                for (int i0 = 0; i0 < N; i0 += TI) {
                    float v[32];
#pragma unroll
                    for (int t = 0; t < TI; ++t) {
                        const int slt = __shfl_sync(kFull, my_cs, (i0 + t) & 31);
                        if (i0 + t >= N) {
#pragma unroll
                            for (int j = 0; j < KP1MAX; ++j) v[t * KP1MAX + j] = 0.f;
                            continue;
                        }
                        const float* Ai = Ring + slt * RS + 2 * lane;
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
                    if constexpr (kTransposeDots) {  // as hogbatch.cu: through the idle B slab
                        float* T = Bs;
                        __syncwarp();
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
                // a6 per input i: ΔOut_j += G_ij A_i (A over the SNAPSHOT) and slot(i) += ΔIn_i =
                // Σ_j G_ij B_j, in input order (M_in[ctx_i] += ΔIn_i, C10). When a word repeats
                // inside the window two contexts share a slot, and a later input must still read
                // the snapshot: then all ΔOut first, all slot updates second
                // (conservative and cheap: some slot is shared by two window positions)
                const bool dup = __any_sync(kFull, lane < S && slot_ref > 1);
                auto delta_in = [&](int i, float2 (&din)[CP2]) {
                    float2 g2[KP1MAX];
#pragma unroll
                    for (int j = 0; j < KP1MAX; ++j) {
                        const float gj = gs[i * KP1MAX + j];
                        g2[j] = make_float2(gj, gj);
                    }
#pragma unroll
                    for (int c = 0; c < CP2; ++c) {
                        constexpr int NCH = (KP1MAX >= 8 && CP2 <= 2) ? 4 : 1;
                        float2 s2[NCH];
#pragma unroll
                        for (int h = 0; h < NCH; ++h) s2[h] = make_float2(0.f, 0.f);
#pragma unroll
                        for (int j = 0; j < KP1MAX; ++j) s2[j % NCH] = ffma2(g2[j], bq[j][c], s2[j % NCH]);
#pragma unroll
                        for (int h = 1; h < NCH; ++h) s2[0] = fadd2(s2[0], s2[h]);
                        din[c] = s2[0];
                    }
                };
                for (int i = 0; i < N; ++i) {
                    const int slt = __shfl_sync(kFull, my_cs, i);
                    float* Ai = Ring + slt * RS + 2 * lane;
                    float2 a[CP2];
#pragma unroll
                    for (int c = 0; c < CP2; ++c)
                        a[c] = (c < CP2 - 1 || lastok) ? *reinterpret_cast<const float2*>(Ai + 64 * c) : make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < KP1MAX; ++j) {
                        const float gj = gs[i * KP1MAX + j];
                        const float2 g2 = make_float2(gj, gj);
#pragma unroll
                        for (int c = 0; c < CP2; ++c) dq[j][c] = ffma2(g2, a[c], dq[j][c]);
                    }
                    if (!dup) {   // the common case: fused, A_i still in registers
                        float2 din[CP2];
                        delta_in(i, din);
#pragma unroll
                        for (int c = 0; c < CP2; ++c)
                            if (c < CP2 - 1 || lastok)
                                *reinterpret_cast<float2*>(Ai + 64 * c) =
                                    make_float2(__fadd_rn(a[c].x, din[c].x), __fadd_rn(a[c].y, din[c].y));
                    }
                }
                if (dup) {
                    __syncwarp();
                    for (int i = 0; i < N; ++i) {
                        const int slt = __shfl_sync(kFull, my_cs, i);
                        float* Ai = Ring + slt * RS + 2 * lane;
                        float2 din[CP2];
                        delta_in(i, din);
#pragma unroll
                        for (int c = 0; c < CP2; ++c)
                            if (c < CP2 - 1 || lastok) {
                                float2 x = *reinterpret_cast<float2*>(Ai + 64 * c);
                                x.x = __fadd_rn(x.x, din[c].x);
                                x.y = __fadd_rn(x.y, din[c].y);
                                *reinterpret_cast<float2*>(Ai + 64 * c) = x;
                            }
                        __syncwarp();
                    }
                }
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                    for (int c = 0; c < CP2; ++c)
                        if (c < CP2 - 1 || lastok) *reinterpret_cast<float2*>(Bs + j * RS + 2 * lane + 64 * c) = dq[j][c];
            }
            __syncwarp();

            // ---------------- leaves: position m-w (or, at the chunk's last target, every
            // position still in the ring); a slot whose count drops to 0 is written back
            uint32_t outm = 0;
            {
                const int q_lo = m - w < 0 ? 0 : m - w;
                const int q_hi = (m == nk - 1) ? nk - 1 : m - w;
                for (int q = q_lo; q <= q_hi; ++q) {
                    const int sl = __shfl_sync(kFull, pos_slot, q & 31);
                    int left = 0;
                    if (lane == sl) {
                        slot_ref -= 1;
                        left = slot_ref == 0;
                    }
                    if (__shfl_sync(kFull, left, sl)) outm |= 1u << sl;
                }
            }
            // write-back of the leaving slots. Hogwild: delta = slot - original (TMEM), reduced
            // into the row so concurrent units' updates survive. Deterministic (one unit, no
            // concurrent writer) with option ring_writeback = 0: the slot VALUE is stored, exactly
            // the sequential row (bit-identical to the rows kernel's mode 1)
            const bool store_back = p.deterministic && !p.ring_delta;
            for (uint32_t om = store_back ? 0u : outm; om; om &= om - 1) {   // delta = slot - original, in place
                const int sl = __ffs(om) - 1;
                float v[NC];
                tmem_load_row<NC>(tbase + (uint32_t)(sl * NC), v);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < CP2; ++c)
                    if (c < CP2 - 1 || lastok) {
                        float2* x = reinterpret_cast<float2*>(Ring + sl * RS + 2 * lane + 64 * c);
                        float2 y = *x;
                        y.x = __fsub_rn(y.x, v[2 * c]);
                        y.y = __fsub_rn(y.y, v[2 * c + 1]);
                        *x = y;
                    }
            }
            fence_proxy_async_smem();
            __syncwarp();

            // ---------------- a7: Hogwild scatter-add: K+1 output rows + the written-back slots
            if (lane < KP1)
                bulk_red_add_s2g_hint(p.M + (size_t)oid * 2 * Ds + Ds, Bs + lane * RS, rowbytes,
                                      oid < p.hot_rows ? pol_hot : pol_cold);
            if ((outm >> lane) & 1u) {
                if (store_back)
                    bulk_s2g(p.M + (size_t)slot_word * 2 * Ds, Ring + lane * RS, rowbytes);
                else
                    bulk_red_add_s2g_hint(p.M + (size_t)slot_word * 2 * Ds, Ring + lane * RS, rowbytes,
                                          slot_word < p.hot_rows_in ? pol_hot : pol_cold);
                slot_word = -1;
            }
            bulk_commit();
            freem |= outm;
            st_loss += (double)st_loss_f;
            if (pp >= p.loss_tail_from) {
                st_tail += (double)st_loss_f;
                if (lane == 0) wst[kTailPairs] += (unsigned long long)(N * KP1);
            }
            st_loss_f = 0.f;
            if (lane == 0) {
                wst[kTargets] += 1;
                wst[kTouch] += (unsigned long long)(N + KP1);
                wst[kPairs] += (unsigned long long)(N * KP1);
                wst[kMoved] += (unsigned long long)(2 * KP1 + nnew + __popc(outm));
            }
            if (p.dbg_len && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len) {
                const int64_t qd = pp - p.dbg_base;
                if (lane == 0) p.dbg_N[qd] = (uint8_t)N;
                if (lane < N) p.dbg_ctx[qd * 2 * w + lane] = kid[lo + lane + (lo + lane >= m ? 1 : 0)];
                for (int k = lane; k < K; k += 32) p.dbg_neg[qd * K + k] = ng[k];
            }
            // the next target's gathers must see these reductions (R11) and the slab must be free
            // (option scatter_wait = 0, Hogwild only: just free — wait until the engine has read
            // the sources; the chunk's next target may then read a row before this target's
            // update to it lands, the same staleness Hogwild allows between units)
            if (p.deterministic || p.scatter_wait) bulk_wait_all();
            else bulk_wait_read_all();
            if (p.deterministic) __threadfence();
            __syncwarp();
        }
    }

#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        st_loss += __shfl_xor_sync(kFull, st_loss, o);
        st_tail += __shfl_xor_sync(kFull, st_tail, o);
        st_cold += __shfl_xor_sync(kFull, st_cold, o);
    }
    if (lane == 0) {
        atomicAdd(&p.stats->words, wst[kWords]);
        atomicAdd(&p.stats->targets, wst[kTargets]);
        atomicAdd(&p.stats->row_touches, wst[kTouch]);
        atomicAdd(&p.stats->loss_pairs, wst[kPairs]);
        atomicAdd(&p.stats->loss_sum, st_loss);
        atomicAdd(&p.stats->row_touches_cold, (unsigned long long)st_cold);
        atomicAdd(&p.stats->rows_moved, wst[kMoved]);
        if (wst[kTailPairs]) {
            atomicAdd(&p.stats->loss_tail_sum, st_tail);
            atomicAdd(&p.stats->loss_tail_pairs, wst[kTailPairs]);
        }
    }
    // every warp of the CTA is done with TMEM before warp 0 frees it
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (wid == 0) tmem_dealloc(tmem_base_s, tm_cols);
    (void)nwarps;
}

using KernelFn = void (*)(const StepParams, int);

struct Inst {
    int cp2, kp1, rs;
    KernelFn fn;
};

#define W2V_RINST(C, KK) {C, KK, 0, hogbatch_ring_kernel<C, KK, 0>}
const Inst kInst[] = {
    W2V_RINST(1, 2), W2V_RINST(1, 4), W2V_RINST(1, 6), W2V_RINST(1, 8), W2V_RINST(1, 16), W2V_RINST(1, 32),
    W2V_RINST(2, 2), W2V_RINST(2, 4), W2V_RINST(2, 6), W2V_RINST(2, 8), W2V_RINST(2, 16),
    W2V_RINST(3, 2), W2V_RINST(3, 4), W2V_RINST(3, 6), W2V_RINST(3, 8), W2V_RINST(3, 16),
    W2V_RINST(4, 2), W2V_RINST(4, 4), W2V_RINST(4, 6), W2V_RINST(4, 8),
    W2V_RINST(5, 2), W2V_RINST(5, 4), W2V_RINST(5, 6), W2V_RINST(5, 8),
    W2V_RINST(8, 2), W2V_RINST(8, 4), W2V_RINST(8, 6),
    {5, 6, 300, hogbatch_ring_kernel<5, 6, 300>},  // the paper's D=300, K<=5, packed rows
};
#undef W2V_RINST

const Inst* pick(int D, int K) {
    const int need = (D + 63) / 64, kp1 = K + 1;
    for (const Inst& in : kInst)
        if (in.rs == D && in.cp2 >= need && in.kp1 >= kp1) return &in;
    const Inst* best = nullptr;
    for (const Inst& in : kInst) {
        if (in.rs != 0 || in.cp2 < need || in.kp1 < kp1) continue;
        if (!best || in.cp2 * in.kp1 < best->cp2 * best->kp1) best = &in;
    }
    return best;
}

}  // namespace

size_t ring_warp_bytes(int L, int window, int K, int D, int32_t* slab_offset) {
    // [mbarrier 8 | nk 4 | pad 4 | stats 6 x 8 B][kid Lp][kinfo Lp][negs 8 x max(K,1)][G tiles x 32]
    // [slab: KP1MAX B rows + (2w+1) ring rows, stride RS] — 21,040 B at cfg3: 11 units per SM
    const Inst* in = pick(D, K);
    if (!in || window > 15) return 0;  // the ring's slot and position masks are one warp wide
    const int RS = in->rs > 0 ? in->rs : 64 * in->cp2;
    const int TI = 32 / in->kp1;
    const size_t gfl = (size_t)((2 * window + TI - 1) / TI) * 32;
    const int Lp = (L + 3) & ~3;
    const int Lps = Lp <= kRingSmemChunk ? Lp : 0;
    const size_t ids = 64 + (size_t)(2 * Lps + kRingNegRows * (K > 0 ? K : 1)) * 4 + gfl * 4;
    const size_t off = (ids + 15) / 16 * 16;
    if (slab_offset) *slab_offset = (int32_t)off;
    return off + (size_t)(in->kp1 + 2 * window + 1) * RS * 4;
}

// work units per CTA the TMEM columns and shared memory allow (one CTA per SM); 0 = unsupported
int ring_units_per_cta(int window, int D, int K, size_t warp_bytes, size_t smem_max) {
    const Inst* in = pick(D, K);
    if (!in || window > 15 || warp_bytes == 0) return 0;
    const int cw = ring_tmem_cols(window, in->cp2);   // columns per warp
    int u = (int)(smem_max / warp_bytes);
    if (u > kRingMaxWarps) u = kRingMaxWarps;
    while (u > 0 && ((u + 3) / 4) * cw > 512) --u;
    return u;
}

cudaError_t launch_ring(const StepParams& p, int ctas, int units, cudaStream_t st) {
    const Inst* in = pick(p.D, p.K);
    if (!in || units < 1) return cudaErrorInvalidValue;
    const int cw = ring_tmem_cols(p.window, in->cp2);
    const uint32_t cols = pow2_cols((uint32_t)(((units + 3) / 4) * cw));
    size_t smem = (size_t)units * p.warp_bytes;
    // one CTA per SM: a second co-resident CTA would block in tcgen05.alloc until the first one
    // exits, so ask for more than half of the SM's shared memory when the grid is persistent
    if (ctas > 1 && smem < 116 * 1024) smem = 116 * 1024;
    cudaError_t e = cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    in->fn<<<ctas, 32 * units, smem, st>>>(p, (int)cols);
    return cudaGetLastError();
}

bool ring_supported(int window, int D, int K) { return pick(D, K) != nullptr && window <= 15; }

}  // namespace w2v
