// hogbatch_win.cu — the fused HogBatch step with WINDOW-RESIDENT rows (SURVEY.md §8(a) rows
// a1-a7; §8(f) NEXT-1 "sentence-tiled row reuse"), sm_100a. Same math and contract as
// hogbatch.cu; different data movement:
//
//  * M_in rows. The context of kept target m is a subset of kept positions [m-w, m+w]. Those
//    positions live in a ring of S = 2w+2 smem slots (value row + delta-accumulator row). A
//    position enters one step ahead (one bulk copy) and leaves w steps later; on leaving, its
//    accumulated ΔIn is written back with ONE bulk fp32 reduce-add. Positions holding the same
//    word share a slot (reference count), so a chunk's targets read each other's updates
//    exactly as the sequential algorithm does (R11), with ~1 gather + 1 scatter per kept
//    position instead of N per target.
//  * M_out rows (target + K negatives) are prefetched one target ahead into a double buffer;
//    rows of target m+1 that repeat a row of target m receive target m's ΔOut in smem
//    ("patch"), and every gather is issued only after all of this warp's earlier reductions
//    completed — so the warp's view of the model is exactly the sequential one, while the
//    copies of target m+1 overlap the compute of target m.
//  * Compute per target: all N·(K+1) dots first (FFMA2), ONE butterfly reduce-scatter per
//    32 dots (lane l ends with dot l), σ/G/loss once per lane, G through smem, then ΔOut
//    (pass A, reads the snapshot) and ΔIn (pass B, writes value + accumulator rows).
// Paper mapping: PAPER.md:116-126 (HogBatch GEMMs, write-back at the end), :140-149 (fewer
// model updates), :135-138 (Hogwild across work units).
#include <cstdio>

#include "hogbatch_common.cuh"

namespace w2v {

#if defined(W2V_PHASE_TIMING)
// (experiment) cycles per target summed over warps: waits for this target's rows, prefetch of
// the next target (incl. conflict waits), compute, scatter issue; targets
__device__ unsigned long long g_wphase[8];
#define W2V_T(...) __VA_ARGS__
#else
#define W2V_T(...)
#endif

namespace {

#ifndef W2V_WIN_MINB
#define W2V_WIN_MINB 4
#endif

constexpr int kWinMaxSlots = 32;  // S = 2*window + 2 <= 32 (window <= 15)

template <int CP2, int KP1MAX>
__global__ void __launch_bounds__(32, W2V_WIN_MINB) hogbatch_win_kernel(const StepParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int P2 = Pow2<KP1MAX>::v, LG = Pow2<KP1MAX>::lg;
    constexpr int TI = 32 / P2;  // inputs per reduce-scatter tile
    constexpr int RS = 64 * CP2;
    const int lane = threadIdx.x & 31;
    unsigned char* wbase = smem + (threadIdx.x >> 5) * p.warp_bytes;
    const int D = p.D, Ds = p.Ds, K = p.K, KP1 = K + 1, w = p.window, S = 2 * w + 2, KS = K > 0 ? K : 1;
    const uint32_t rowbytes = (uint32_t)D * 4u;

    uint64_t* mbarA = reinterpret_cast<uint64_t*>(wbase);  // window entries
    uint64_t* mbarB = mbarA + 1;                           // [2] target/negative buffers
    int32_t* nk_s = reinterpret_cast<int32_t*>(wbase + 24);  // kept count of the chunk
    int32_t* kid = reinterpret_cast<int32_t*>(wbase + 32);
    int32_t* kinfo = kid + p.Lp;
    int32_t* pslot = kinfo + p.Lp;     // slot of kept position (valid while in the window)
    int32_t* slot_id = pslot + p.L;    // [S]
    int32_t* slot_ref = slot_id + S;   // [S]
    int32_t* negs = slot_ref + S;      // [kSampWin][KS]
    int32_t* bid = negs + kSampWin * KS;  // [2][KP1MAX]
    int32_t* cslot = bid + 2 * KP1MAX;    // [2w] context slots of the current target
    float* gs = reinterpret_cast<float*>(cslot + 2 * w);  // G, [tiles*TI][P2]
    float* val = reinterpret_cast<float*>(wbase + p.slab_offset);  // [S][RS]
    float* acc = val + S * RS;                                      // [S][RS]
    float* Bb = acc + S * RS;                                       // [2][KP1MAX][RS]

    const int64_t shard_end = p.shard_start + p.n_local;

    const uint64_t pol_hot = (p.l2_hint & 1) ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_cold = (p.l2_hint & 2) ? policy_evict_first() : policy_evict_normal();
    if (lane == 0) {
        mbar_init(mbarA, 1);
        mbar_init(mbarB, 1);
        mbar_init(mbarB + 1, 1);
    }
    {   // zero value rows (their padding columns stay 0) and both B buffers (padding rows stay 0)
        float4* z = reinterpret_cast<float4*>(val);
        for (int i = lane; i < S * RS / 4; i += 32) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        z = reinterpret_cast<float4*>(Bb);
        for (int i = lane; i < 2 * KP1MAX * RS / 4; i += 32) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    fence_proxy_async_smem();  // the bulk engine writes these rows later
    __syncwarp();
    uint32_t phA = 0, phB0 = 0, phB1 = 0;
    unsigned gstep = 0;

    W2V_T(unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};)
    unsigned long long st_words = 0, st_targets = 0, st_touch = 0, st_pairs = 0, st_tail_pairs = 0;
    float st_loss_f = 0.f;
    double st_loss = 0.0, st_tail = 0.0;
    uint32_t freem = 0, newslots = 0, bytesA = 0;
    int32_t pend_exit = -1;  // M_in row whose write-back is in the most recent bulk group

    // ---- window bookkeeping (uniform: every lane executes it with identical values)
    auto enter = [&](int q) {  // plan the entry of kept position q; the copy is issued later
        const int32_t id = kid[q];
        const unsigned hit = __ballot_sync(kFull, lane < S && slot_ref[lane] > 0 && slot_id[lane] == id);
        int s;
        if (hit) {
            s = __ffs(hit) - 1;
            if (lane == 0) slot_ref[s] += 1;
        } else {
            s = __ffs(freem) - 1;
            freem &= ~(1u << s);
            newslots |= 1u << s;
            bytesA += rowbytes;
            if (lane == 0) { slot_id[s] = id; slot_ref[s] = 1; }
            float4* a4 = reinterpret_cast<float4*>(acc + s * RS);
            for (int i = lane; i < RS / 4; i += 32) a4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (lane == 0) pslot[q] = s;
        __syncwarp();
    };
    auto issue_entries = [&]() {  // one expect_tx (possibly 0 bytes) + the planned copies
        if (lane == 0) mbar_arrive_expect_tx(mbarA, bytesA);
        __syncwarp();
        if ((newslots >> lane) & 1u)
            bulk_g2s_hint(val + lane * RS, p.M + (size_t)slot_id[lane] * 2 * Ds, rowbytes, mbarA,
                          slot_id[lane] < p.hot_rows ? pol_hot : pol_cold);
        newslots = 0;
        bytesA = 0;
    };
    auto leave = [&](int q) {  // kept position q leaves; write back the slot when unreferenced
        const int s = pslot[q];
        const int ref = slot_ref[s] - 1;
        __syncwarp();
        if (lane == 0) {
            slot_ref[s] = ref;
            if (ref == 0)
                bulk_red_add_s2g_hint(p.M + (size_t)slot_id[s] * 2 * Ds, acc + s * RS, rowbytes,
                                      slot_id[s] < p.hot_rows ? pol_hot : pol_cold);
        }
        if (ref == 0) {
            freem |= 1u << s;
            pend_exit = slot_id[s];
        }
        __syncwarp();
    };
    auto issue_B = [&](int m, int buf) {  // target + negatives of kept target m into Bb[buf]
        int32_t* ids = bid + buf * KP1MAX;
        const int32_t* ng = negs + (m % kSampWin) * KS;
        if (lane == 0) ids[0] = kid[m];
        if (lane >= 1 && lane <= K) ids[lane] = ng[lane - 1];
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(mbarB + buf, (uint32_t)KP1 * rowbytes);
        __syncwarp();
        if (lane < KP1)
            bulk_g2s_hint(Bb + (buf * KP1MAX + lane) * RS, p.M + (size_t)ids[lane] * 2 * Ds + Ds, rowbytes, mbarB + buf,
                          ids[lane] < p.hot_rows ? pol_hot : pol_cold);
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
        if (cnt <= 0) continue;

        // ---------------- the chunk's batch stream (a1/a2 rows, batch.cu)
        const int64_t rel = s - p.chunk_lo;
        load_chunk(p, rel, kid, kinfo, nk_s, negs, lane);
        cp_async_wait_all();
        __syncwarp();
        const int nk = *nk_s;
        if (lane == 0) st_words += (unsigned long long)cnt;
        if (nk < 2) continue;  // N = 0 for every kept target iff the chunk keeps < 2 words

        int samp_hi = nk < kSampGrp ? nk : kSampGrp;  // negatives of [0, samp_hi) are in the ring
        // every gather below must see all of this warp's earlier reductions
        bulk_wait_all();
        pend_exit = -1;
        __syncwarp();
        for (int i = lane; i < S; i += 32) slot_ref[i] = 0;
        freem = (S >= 32) ? 0xffffffffu : ((1u << S) - 1u);
        __syncwarp();
        for (int q = 0; q <= w && q < nk; ++q) enter(q);
        issue_entries();
        issue_B(0, gstep & 1);

        int64_t q_next = -1;
        float alpha = 0.f;
        for (int m = 0; m < nk; ++m, ++gstep) {
            W2V_T(long long t0 = clock64();)
            const int cur = gstep & 1, nxt = cur ^ 1;
            float* Bc = Bb + cur * KP1MAX * RS;
            const float* Bp = Bb + nxt * KP1MAX * RS;
            const int32_t* bidc = bid + cur * KP1MAX;
            mbar_wait(mbarB + cur, cur ? phB1 : phB0);
            if (cur) phB1 ^= 1u; else phB0 ^= 1u;
            mbar_wait(mbarA, phA);
            phA ^= 1u;
            W2V_T(long long t1 = clock64(); ph[0] += t1 - t0;)
            // exactness: rows of target m repeated from target m-1 get its ΔOut (still in Bp)
            if (m > 0) {
                const int32_t* bidp = bid + nxt * KP1MAX;
                for (int j = 0; j < KP1; ++j) {
                    unsigned pm = __ballot_sync(kFull, lane < KP1 && bidp[lane] == bidc[j]);
                    while (pm) {
                        const int jp = __ffs(pm) - 1;
                        pm &= pm - 1;
#pragma unroll
                        for (int c = 0; c < CP2; ++c) {
                            float2* d2 = reinterpret_cast<float2*>(Bc + j * RS + 2 * lane + 64 * c);
                            *d2 = fadd2(*d2, *reinterpret_cast<const float2*>(Bp + jp * RS + 2 * lane + 64 * c));
                        }
                    }
                }
            }
            // ---------------- prefetch for target m+1 (overlaps this target's compute)
            // (one cp.async group per target; after iteration m the ring holds targets up to
            // >= m+10, so waiting for all groups but this one covers target m+1)
            if (K > 0 && samp_hi < nk && samp_hi - (m + 2) < kSampGrp) {
                const int c = nk - samp_hi < kSampGrp ? nk - samp_hi : kSampGrp;
                fetch_negs(p, rel, samp_hi, c, negs, lane);
                samp_hi += c;
            }
            cp_async_commit();
            cp_async_wait_but_last();
            __syncwarp();
            // Sources of earlier reductions must be read before Bp / freed slots are reused, and
            // every group but target m-1's must be complete; a gather that touches a row still in
            // target m-1's group (same M_out id, or the M_in row it wrote back) waits for it.
            bulk_wait_read_all();
            bulk_wait_all_but_last();
            if (m + 1 < nk) {
                bool conf = false;
                if (lane < KP1) {
                    const int32_t id = lane == 0 ? kid[m + 1] : negs[((m + 1) % kSampWin) * KS + lane - 1];
                    const int32_t* bidp = bid + nxt * KP1MAX;
                    for (int jp = 0; jp < KP1; ++jp) conf |= (id == bidp[jp]);
                }
                if (lane == 0 && m + w + 1 < nk) conf |= (kid[m + w + 1] == pend_exit);
                if (__any_sync(kFull, conf)) bulk_wait_all();
            }
            pend_exit = -1;
            __syncwarp();
            if (m + 1 < nk) {  // one arrival per wait on each barrier
                issue_B(m + 1, nxt);
                if (m + w + 1 < nk) enter(m + w + 1);
                issue_entries();
            }

            // ---------------- target m: context slots, alpha
            const int b = kinfo[m] & 255;
            const int64_t pp = c0 + (kinfo[m] >> 8);
            const int lo = m - b < 0 ? 0 : m - b;
            const int hi = m + b > nk - 1 ? nk - 1 : m + b;
            const int N = hi - lo;
            for (int i = lane; i < N; i += 32) cslot[i] = pslot[lo + i + (lo + i >= m ? 1 : 0)];
            const int64_t pi = (int64_t)p.epoch * p.n_local + (pp - p.shard_start);
            if (pi >= q_next) {
                const int64_t qi = pi / p.Q;
                q_next = (qi + 1) * p.Q;
                alpha = alpha_at(p, qi);
            }
            __syncwarp();

            W2V_T(long long t2 = clock64(); ph[1] += t2 - t1;)
            // ---------------- a4/a5: all N x (K+1) dots, reduce-scatter, E, G, loss
            float2 bq[KP1MAX][CP2];
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CP2; ++c) bq[j][c] = *reinterpret_cast<const float2*>(Bc + j * RS + 2 * lane + 64 * c);
            const int tj = lane & (P2 - 1);  // after the reduce-scatter lane holds dot (tile input lane>>LG, tj)
            for (int i0 = 0; i0 < N; i0 += TI) {
                float v[32];
#pragma unroll
                for (int t = 0; t < TI; ++t) {
                    const int i = i0 + t;
                    float2 a[CP2];
                    const float* Ai = val + (i < N ? cslot[i] : 0) * RS + 2 * lane;
#pragma unroll
                    for (int c = 0; c < CP2; ++c) a[c] = *reinterpret_cast<const float2*>(Ai + 64 * c);
#pragma unroll
                    for (int j = 0; j < P2; ++j) {
                        float2 s2 = make_float2(0.f, 0.f);
                        if (j < KP1MAX) {
#pragma unroll
                            for (int c = 0; c < CP2; ++c) s2 = ffma2(a[c], bq[j][c], s2);
                        }
                        v[t * P2 + j] = s2.x + s2.y;
                    }
                }
#pragma unroll
                for (int st = 0; st < 5; ++st) {
                    const int o = 16 >> st;
                    const int half = 16 >> st;
                    const bool up = lane & o;
#pragma unroll
                    for (int u = 0; u < half; ++u) {
                        const float send = up ? v[u] : v[u + half];
                        const float keep = up ? v[u + half] : v[u];
                        v[u] = keep + __shfl_xor_sync(kFull, send, o);
                    }
                }
                const float dot = v[0];
                const bool valid = (i0 + (lane >> LG) < N) && tj < KP1;
                const float ex = expf(-fabsf(dot));
                const float rc = __frcp_rn(1.0f + ex);
                const float sg = dot >= 0.f ? rc : ex * rc;
                const bool pos = (tj == 0);
                gs[i0 * P2 + lane] = valid ? alpha * ((pos ? 1.0f : 0.0f) - sg) : 0.f;
                if (valid) st_loss_f += fmaxf(pos ? -dot : dot, 0.f) - __logf(rc);
            }
            __syncwarp();

            // ---------------- a6 pass A: ΔOut_j = Σ_i G_ij A_i (A = snapshot, nothing written yet)
            float2 dq[KP1MAX][CP2];
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CP2; ++c) dq[j][c] = make_float2(0.f, 0.f);
            for (int i = 0; i < N; ++i) {
                const float* Ai = val + cslot[i] * RS + 2 * lane;
                float2 a[CP2];
#pragma unroll
                for (int c = 0; c < CP2; ++c) a[c] = *reinterpret_cast<const float2*>(Ai + 64 * c);
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) {
                    const float gj = gs[i * P2 + j];
                    const float2 g2 = make_float2(gj, gj);
#pragma unroll
                    for (int c = 0; c < CP2; ++c) dq[j][c] = ffma2(g2, a[c], dq[j][c]);
                }
            }
            // ---------------- a6 pass B: ΔIn_i = Σ_j G_ij B_j into value + accumulator rows
            for (int i = 0; i < N; ++i) {
                float2 d[CP2];
#pragma unroll
                for (int c = 0; c < CP2; ++c) d[c] = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) {
                    const float gj = gs[i * P2 + j];
                    const float2 g2 = make_float2(gj, gj);
#pragma unroll
                    for (int c = 0; c < CP2; ++c) d[c] = ffma2(g2, bq[j][c], d[c]);
                }
                float* Vi = val + cslot[i] * RS + 2 * lane;
                float* Ci = acc + cslot[i] * RS + 2 * lane;
#pragma unroll
                for (int c = 0; c < CP2; ++c) {
                    float2* v2 = reinterpret_cast<float2*>(Vi + 64 * c);
                    float2* c2 = reinterpret_cast<float2*>(Ci + 64 * c);
                    *v2 = fadd2(*v2, d[c]);
                    *c2 = fadd2(*c2, d[c]);
                }
            }
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CP2; ++c) *reinterpret_cast<float2*>(Bc + j * RS + 2 * lane + 64 * c) = dq[j][c];
            fence_proxy_async_smem();
            __syncwarp();

            W2V_T(long long t3 = clock64(); ph[2] += t3 - t2;)
            // ---------------- a7: ΔOut rows now; position m-w leaves the window
            if (lane < KP1)
                bulk_red_add_s2g_hint(p.M + (size_t)bidc[lane] * 2 * Ds + Ds, Bc + lane * RS, rowbytes,
                                      bidc[lane] < p.hot_rows ? pol_hot : pol_cold);
            if (m - w >= 0) leave(m - w);
            bulk_commit();

            st_loss += (double)st_loss_f;
            if (pp >= p.loss_tail_from) {
                st_tail += (double)st_loss_f;
                if (lane == 0) st_tail_pairs += (unsigned long long)N * KP1;
            }
            st_loss_f = 0.f;
            if (lane == 0) {
                st_targets += 1;
                st_touch += (unsigned long long)(N + KP1);
                st_pairs += (unsigned long long)N * KP1;
            }
            if (p.dbg_len && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len) {
                const int64_t q = pp - p.dbg_base;
                if (lane == 0) p.dbg_N[q] = (uint8_t)N;
                for (int i = lane; i < N; i += 32) p.dbg_ctx[q * 2 * w + i] = kid[lo + i + (lo + i >= m ? 1 : 0)];
                for (int k = lane; k < K; k += 32) p.dbg_neg[q * K + k] = bidc[1 + k];
            }
            W2V_T(ph[3] += clock64() - t3; ph[4] += 1;)
            if (p.deterministic) __threadfence();
            __syncwarp();
        }
        // chunk end: the positions still in the window leave
        for (int q = nk - w > 0 ? nk - w : 0; q < nk; ++q) leave(q);
        bulk_commit();
    }
    bulk_wait_all();  // the smem sources of the last reductions must be read before exit

#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        st_loss += __shfl_xor_sync(kFull, st_loss, o);
        st_tail += __shfl_xor_sync(kFull, st_tail, o);
    }
    W2V_T(if (lane == 0) for (int i = 0; i < 8; ++i) atomicAdd(&g_wphase[i], ph[i]);)
    if (lane == 0) {
        atomicAdd(&p.stats->words, st_words);
        atomicAdd(&p.stats->targets, st_targets);
        atomicAdd(&p.stats->row_touches, st_touch);
        atomicAdd(&p.stats->loss_pairs, st_pairs);
        atomicAdd(&p.stats->loss_sum, st_loss);
        if (st_tail_pairs) {
            atomicAdd(&p.stats->loss_tail_sum, st_tail);
            atomicAdd(&p.stats->loss_tail_pairs, st_tail_pairs);
        }
    }
}

using KernelFn = void (*)(const StepParams);
struct Inst {
    int cp2, kp1;
    KernelFn fn;
};
#define W2V_INST(C, KK) {C, KK, hogbatch_win_kernel<C, KK>}
const Inst kInst[] = {
    W2V_INST(1, 2), W2V_INST(1, 4), W2V_INST(1, 6), W2V_INST(1, 8), W2V_INST(1, 16), W2V_INST(1, 32),
    W2V_INST(2, 2), W2V_INST(2, 4), W2V_INST(2, 6), W2V_INST(2, 8), W2V_INST(2, 16),
    W2V_INST(3, 4), W2V_INST(3, 6), W2V_INST(3, 8), W2V_INST(3, 16),
    W2V_INST(4, 4), W2V_INST(4, 6), W2V_INST(4, 8),
    W2V_INST(5, 4), W2V_INST(5, 6), W2V_INST(5, 8),
    W2V_INST(8, 4), W2V_INST(8, 6),
};
#undef W2V_INST

const Inst* pick(int D, int K) {
    const int need = (D + 63) / 64, kp1 = K + 1;
    const Inst* best = nullptr;
    for (const Inst& in : kInst) {
        if (in.cp2 < need || in.kp1 < kp1) continue;
        if (!best || in.cp2 * in.kp1 < best->cp2 * best->kp1) best = &in;
    }
    return best;
}

}  // namespace

void win_phase_report() {
#if defined(W2V_PHASE_TIMING)
    unsigned long long h[8];
    cudaMemcpyFromSymbol(h, g_wphase, sizeof h);
    if (!h[4]) return;
    const double T = (double)h[4];
    fprintf(stderr, "[phase] win per target (cycles): wait rows %.0f  prefetch next %.0f  compute %.0f  scatter issue %.0f  targets %llu\n",
            h[0] / T, h[1] / T, h[2] / T, h[3] / T, h[4]);
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_wphase, z, sizeof z);
#endif
}

size_t win_warp_bytes(int L, int window, int K, int D, int32_t* slab_offset) {
    const Inst* in = pick(D, K);
    const int S = 2 * window + 2;
    if (!in || S > kWinMaxSlots) return 0;
    const int P2 = in->kp1 <= 2 ? 2 : in->kp1 <= 4 ? 4 : in->kp1 <= 8 ? 8 : in->kp1 <= 16 ? 16 : 32;
    const int TI = 32 / P2;
    const int tiles = (2 * window + TI - 1) / TI;
    const int Lp = (L + 3) & ~3;
    const size_t ints = (size_t)2 * Lp + L + 2 * S + kSampWin * (K > 0 ? K : 1) + 2 * in->kp1 + 2 * window;
    const size_t head = 32 + ints * 4 + (size_t)tiles * 32 * 4;
    const size_t off = (head + 127) / 128 * 128;
    if (slab_offset) *slab_offset = (int32_t)off;
    return off + (size_t)(2 * S + 2 * in->kp1) * 64 * in->cp2 * 4;
}

int win_max_ctas_per_sm(const StepParams& p) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return 0;
    int n = 0;
    cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, in->fn, 32, p.warp_bytes) != cudaSuccess) return 0;
    return n;
}

cudaError_t launch_win(const StepParams& p, int ctas, cudaStream_t st) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (e != cudaSuccess) return e;
    in->fn<<<ctas, 32, p.warp_bytes, st>>>(p);
    return cudaGetLastError();
}

}  // namespace w2v
