// hogbatch_wg.cu — the fused HogBatch step, window-resident and WARP-SPECIALISED (SURVEY.md §8(a)
// rows a3-a8, §8(f) NEXT-1), sm_100a. Same math, contract and data movement as hogbatch_win.cu —
// a chunk's kept positions [m-w, m+w+1] live in smem slots (value + ΔIn accumulator, written back
// once when the position leaves the window), M_out rows are prefetched one target ahead and
// patched — so ~1 gather + 1 scatter per kept position for M_in instead of N per target
// (≈36% fewer row bytes than hogbatch.cu). What changes is who does the work:
//
//  * One CTA = one work unit (chunks in corpus order, targets sequential, R11) with NW+1 warps.
//  * NW compute warps split the COLUMNS: warp c owns float2 column 2*lane + 64c of every row
//    (NW = ceil(D/64): 5 at the paper's D=300). Every row operation of the step (dots, ΔOut,
//    ΔIn, patches) touches only the warp's own columns, so the compute warps never wait on each
//    other's data — except for the dot products, whose per-warp partials (after an in-warp
//    butterfly reduce-scatter) meet once per target in smem behind one named barrier.
//  * One IO warp runs the window bookkeeping and every bulk copy/reduction (the TMA engine),
//    one target ahead of the compute warps: while they compute target m it waits for the row
//    conflicts of target m+1, issues its M_out rows and entering M_in row, then issues target m's
//    ΔOut reductions and the leaving row's write-back as soon as the compute warps signal.
//  * Hand-offs are mbarriers: rows landed (TMA complete_tx + IO arrive, which also publishes the
//    IO warp's slot tables), patch done and compute done (one arrive per compute warp), each
//    double-buffered by target parity so neither side can lap the other.
// Per-target latency drops ~NW-fold against the one-warp window kernel, whose compute phase
// (≈5,300 cycles) made it latency-bound (profiles/r01_ablations.md).
#include <cstdio>

#include "hogbatch_common.cuh"

namespace w2v {

#if defined(W2V_PHASE_TIMING)
// (experiment) cycles summed over CTAs: IO [0] wait patch, [1] bulk/conflict waits, [2] issue,
// [3] wait compute-done, [4] scatter issue; compute warp 0 [5] wait rows, [6] dots incl. barrier,
// [7] rest of compute; [8] targets
__device__ unsigned long long g_gphase[16];
#define W2V_T(...) __VA_ARGS__
#else
#define W2V_T(...)
#endif

namespace {

constexpr int kWgMaxSlots = 32;  // S = 2*window + 2 <= 32

#ifndef W2V_WG_MINB
#define W2V_WG_MINB 4  // resident CTAs per SM the register budget is sized for (smem allows 4 at D=300)
#endif

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_sync_id(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int NW, int KP1MAX>
__global__ void __launch_bounds__(32 * (NW + 1), W2V_WG_MINB) hogbatch_wg_kernel(const StepParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int TI = 32 / KP1MAX;  // inputs per reduce-scatter tile
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool io = warp == NW;
    const int D = p.D, Ds = p.Ds, K = p.K, KP1 = K + 1, w = p.window, S = 2 * w + 2, KS = K > 0 ? K : 1, RS = p.D;
    const int tiles = (2 * w + TI - 1) / TI;
    const uint32_t rowbytes = (uint32_t)D * 4u;

    // ---- shared memory (layout mirrored by wg_cta_bytes)
    uint64_t* mbarA = reinterpret_cast<uint64_t*>(smem);  // [2] entering M_in rows of a target
    uint64_t* mbarB = mbarA + 2;                          // [2] M_out rows of a target
    uint64_t* mbarP = mbarA + 4;                          // [2] patch done
    uint64_t* mbarD = mbarA + 6;                          // [2] compute done
    int32_t* hdr = reinterpret_cast<int32_t*>(smem + 64);  // [0] nk, [1] chunk claimed (rel), [2] cnt
    int32_t* kid = reinterpret_cast<int32_t*>(smem + 80);
    int32_t* kinfo = kid + p.Lp;
    int32_t* pslot = kinfo + p.Lp;                      // [L] slot of a kept position
    int32_t* slot_id = pslot + p.Lp;                    // [S]
    int32_t* slot_ref = slot_id + kWgMaxSlots;          // [S]
    int32_t* negs = slot_ref + kWgMaxSlots;             // [kSampWin][KS]
    int32_t* bid = negs + kSampWin * KS;                // [2][KP1MAX]
    int32_t* cslot = bid + 2 * KP1MAX;                  // [2][2w] context slots of a target
    float* part = reinterpret_cast<float*>(cslot + 4 * w);  // [2][NW][tiles][32] partial dots
    float* gsh = part + 2 * NW * tiles * 32;                // [NW][tiles][32] G (one copy per warp)
    float* val = reinterpret_cast<float*>(smem + p.slab_offset);  // [S][RS]
    float* acc = val + S * RS;                                    // [S][RS]
    float* Bb = acc + S * RS;                                     // [2][KP1MAX][RS]

    const uint64_t pol_hot = (p.l2_hint & 1) ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_cold = (p.l2_hint & 2) ? policy_evict_first() : policy_evict_normal();
    if (threadIdx.x == 0) {
        mbar_init(mbarA, 1);
        mbar_init(mbarA + 1, 1);
        mbar_init(mbarB, 1);
        mbar_init(mbarB + 1, 1);
        mbar_init(mbarP, NW);
        mbar_init(mbarP + 1, NW);
        mbar_init(mbarD, NW);
        mbar_init(mbarD + 1, NW);
    }
    {   // zero the B buffers (rows a copy never writes stay 0: K+1 < KP1MAX)
        float4* z = reinterpret_cast<float4*>(Bb);
        for (int i = threadIdx.x; i < 2 * KP1MAX * RS / 4; i += blockDim.x) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    fence_proxy_async_smem();
    __syncthreads();

    const int64_t shard_end = p.shard_start + p.n_local;
    unsigned gstep = 0;                         // targets processed by this CTA (buffer parity)
    uint32_t phA0 = 0, phA1 = 0, phB0 = 0, phB1 = 0;  // compute warps: parities of the row barriers
    uint32_t phP0 = 0, phP1 = 0, phD0 = 0, phD1 = 0;  // IO warp: parities of the signal barriers

    W2V_T(unsigned long long ph[16] = {0};)
    // IO-warp state (uniform in the IO warp)
    uint32_t freem = 0, newslots = 0, bytesA = 0;
    int32_t pend_exit = -1;
    // compute-warp statistics (warp 0 counts: every compute warp sees the same dots)
    unsigned long long st_words = 0, st_targets = 0, st_touch = 0, st_pairs = 0, st_tail_pairs = 0;
    double st_loss = 0.0, st_tail = 0.0;

    // ---- IO warp: window bookkeeping (same rules as hogbatch_win.cu)
    auto enter = [&](int q) {
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
            fence_proxy_async_smem();  // the bulk engine reduces this accumulator later
        }
        if (lane == 0) pslot[q] = s;
        __syncwarp();
    };
    auto issue_entries = [&](int buf) {  // rows entering for the target of parity buf
        if (lane == 0) mbar_arrive_expect_tx(mbarA + buf, bytesA);
        __syncwarp();
        if ((newslots >> lane) & 1u)
            bulk_g2s_hint(val + lane * RS, p.M + (size_t)slot_id[lane] * 2 * Ds, rowbytes, mbarA + buf,
                          slot_id[lane] < p.hot_rows ? pol_hot : pol_cold);
        newslots = 0;
        bytesA = 0;
    };
    auto leave = [&](int q) {
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
    // target m's M_out rows into Bb[buf] and its context slots into cslot[buf]; the arrive on
    // mbarB[buf] publishes bid / cslot to the compute warps
    auto issue_B = [&](int m, int buf, int nk) {
        int32_t* ids = bid + buf * KP1MAX;
        const int32_t* ng = negs + (m % kSampWin) * KS;
        if (lane == 0) ids[0] = kid[m];
        if (lane >= 1 && lane <= K) ids[lane] = ng[lane - 1];
        const int b = kinfo[m] & 255;
        const int lo = m - b < 0 ? 0 : m - b, hi = m + b > nk - 1 ? nk - 1 : m + b;
        for (int i = lane; i < hi - lo; i += 32) cslot[buf * 2 * w + i] = pslot[lo + i + (lo + i >= m ? 1 : 0)];
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(mbarB + buf, (uint32_t)KP1 * rowbytes);
        __syncwarp();
        if (lane < KP1)
            bulk_g2s_hint(Bb + (buf * KP1MAX + lane) * RS, p.M + (size_t)ids[lane] * 2 * Ds + Ds, rowbytes,
                          mbarB + buf, ids[lane] < p.hot_rows ? pol_hot : pol_cold);
    };

    for (;;) {
        // ---------------- claim a chunk, load its batch stream (IO warp), publish (CTA barrier)
        if (io) {
            long long s = 0;
            if (lane == 0) s = (long long)atomicAdd(p.chunk_ctr, 1ull) + p.chunk_lo;
            s = __shfl_sync(kFull, s, 0);
            int nk = -1, cnt = 0;
            if (s < p.chunk_hi) {
                int64_t c0 = s * (int64_t)p.L, c1 = c0 + p.L;
                if (c1 > shard_end) c1 = shard_end;
                if (c0 < p.shard_start) c0 = p.shard_start;
                cnt = (int)(c1 - c0);
                nk = 0;
                if (cnt > 0) {
                    load_chunk(p, s - p.chunk_lo, kid, kinfo, hdr, negs, lane);
                    cp_async_wait_all();
                    __syncwarp();
                    nk = hdr[0];
                }
            }
            if (lane == 0) { hdr[0] = nk; hdr[1] = (int32_t)(s - p.chunk_lo); hdr[2] = cnt; }
        }
        __syncthreads();
        const int nk = hdr[0];
        if (nk < 0) break;  // no chunk left
        const int64_t rel = hdr[1];
        const int64_t s = rel + p.chunk_lo;
        int64_t c0 = s * (int64_t)p.L;
        if (c0 < p.shard_start) c0 = p.shard_start;
        if (!io && warp == 0 && lane == 0) st_words += (unsigned long long)hdr[2];
        __syncthreads();  // hdr is rewritten by the next claim only after everyone read it
        if (nk < 2) continue;

        if (io) {
            // every gather of this chunk must see all of this CTA's earlier reductions
            bulk_wait_all();
            pend_exit = -1;
            for (int i = lane; i < S; i += 32) slot_ref[i] = 0;
            freem = (S >= 32) ? 0xffffffffu : ((1u << S) - 1u);
            __syncwarp();
            for (int q = 0; q <= w && q < nk; ++q) enter(q);
            issue_entries(gstep & 1);
            issue_B(0, gstep & 1, nk);
            int samp_hi = nk < kSampGrp ? nk : kSampGrp;
            for (int m = 0; m < nk; ++m, ++gstep) {
                const int cur = gstep & 1, nxt = cur ^ 1;
                W2V_T(long long t0 = clock64();)
                // the compute warps patched target m from Bp: Bp may now take target m+1's rows
                if (m > 0) {
                    mbar_wait(mbarP + cur, cur ? phP1 : phP0);
                    if (cur) phP1 ^= 1u; else phP0 ^= 1u;
                }
                W2V_T(long long t1 = clock64(); ph[0] += t1 - t0;)
                if (K > 0 && samp_hi < nk && samp_hi - (m + 2) < kSampGrp) {
                    const int c = nk - samp_hi < kSampGrp ? nk - samp_hi : kSampGrp;
                    fetch_negs(p, rel, samp_hi, c, negs, lane);
                    samp_hi += c;
                }
                cp_async_commit();
                cp_async_wait_but_last();
                __syncwarp();
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
                W2V_T(long long t2 = clock64(); ph[1] += t2 - t1;)
                if (m + 1 < nk) {
                    if (m + w + 1 < nk) enter(m + w + 1);
                    issue_B(m + 1, nxt, nk);
                    issue_entries(nxt);
                }
                // target m computed: its ΔOut rows and the leaving position's write-back
                W2V_T(long long t3 = clock64(); ph[2] += t3 - t2;)
                mbar_wait(mbarD + cur, cur ? phD1 : phD0);
                if (cur) phD1 ^= 1u; else phD0 ^= 1u;
                W2V_T(long long t4 = clock64(); ph[3] += t4 - t3;)
                if (lane < KP1) {
                    const int32_t id = bid[cur * KP1MAX + lane];
                    bulk_red_add_s2g_hint(p.M + (size_t)id * 2 * Ds + Ds, Bb + (cur * KP1MAX + lane) * RS, rowbytes,
                                          id < p.hot_rows ? pol_hot : pol_cold);
                }
                if (m - w >= 0) leave(m - w);
                bulk_commit();
                W2V_T(ph[4] += clock64() - t4;)
                if (p.deterministic) {
                    bulk_wait_all();
                    __threadfence();
                }
            }
            for (int q = nk - w > 0 ? nk - w : 0; q < nk; ++q) leave(q);
            bulk_commit();
            continue;
        }

        // ---------------- compute warps: target m on columns 2*lane + 64*warp (+0, +1)
        const int col = 2 * lane + 64 * warp;
        const bool cok = col < D;
        int64_t q_next = -1;
        float alpha = 0.f;
        for (int m = 0; m < nk; ++m, ++gstep) {
            const int cur = gstep & 1, nxt = cur ^ 1;
            float* Bc = Bb + cur * KP1MAX * RS;
            const float* Bp = Bb + nxt * KP1MAX * RS;
            const int32_t* bidc = bid + cur * KP1MAX;
            W2V_T(long long t5 = clock64();)
            mbar_wait(mbarB + cur, cur ? phB1 : phB0);
            if (cur) phB1 ^= 1u; else phB0 ^= 1u;
            mbar_wait(mbarA + cur, cur ? phA1 : phA0);
            if (cur) phA1 ^= 1u; else phA0 ^= 1u;
            W2V_T(long long t6 = clock64(); ph[5] += t6 - t5;)
            // exactness: rows of target m repeated from target m-1 get its ΔOut (still in Bp)
            if (m > 0) {
                const int32_t* bidp = bid + nxt * KP1MAX;
                for (int j = 0; j < KP1; ++j) {
                    unsigned pm = __ballot_sync(kFull, lane < KP1 && bidp[lane] == bidc[j]);
                    while (pm) {
                        const int jp = __ffs(pm) - 1;
                        pm &= pm - 1;
                        if (cok) {
                            float2* d2 = reinterpret_cast<float2*>(Bc + j * RS + col);
                            *d2 = fadd2(*d2, *reinterpret_cast<const float2*>(Bp + jp * RS + col));
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(mbarP + cur);
            }
            const int b = kinfo[m] & 255;
            const int64_t pp = c0 + (kinfo[m] >> 8);
            const int lo = m - b < 0 ? 0 : m - b;
            const int hi = m + b > nk - 1 ? nk - 1 : m + b;
            const int N = hi - lo;
            const int32_t* cs = cslot + cur * 2 * w;
            const int64_t pi = (int64_t)p.epoch * p.n_local + (pp - p.shard_start);
            if (pi >= q_next) {
                const int64_t qi = pi / p.Q;
                q_next = (qi + 1) * p.Q;
                alpha = alpha_at(p, qi);
            }
            // ---- a4: partial dots over this warp's columns, butterfly reduce-scatter per tile
            float2 bq[KP1MAX];
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
                bq[j] = cok ? *reinterpret_cast<const float2*>(Bc + j * RS + col) : make_float2(0.f, 0.f);
            float* pw = part + ((size_t)(m & 1) * NW + warp) * tiles * 32;
            for (int i0 = 0, tl = 0; i0 < N; i0 += TI, ++tl) {
                float v[32];
#pragma unroll
                for (int t = 0; t < TI; ++t) {
                    const int i = i0 + t;
                    const float2 a = (cok && i < N) ? *reinterpret_cast<const float2*>(val + cs[i] * RS + col)
                                                    : make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < KP1MAX; ++j) {
                        const float2 s2 = ffma2(a, bq[j], make_float2(0.f, 0.f));
                        v[t * KP1MAX + j] = s2.x + s2.y;
                    }
                }
#pragma unroll
                for (int u = TI * KP1MAX; u < 32; ++u) v[u] = 0.f;
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
                pw[tl * 32 + lane] = v[0];
            }
            bar_sync_id(1, 32 * NW);
            W2V_T(long long t7 = clock64(); ph[6] += t7 - t6;)
            // ---- a5: full dots (partials summed in warp order: identical in every warp), σ, G
            const int tt = lane / KP1MAX, tj = lane - tt * KP1MAX;
            float* gw = gsh + (size_t)warp * tiles * 32;
            float loss_f = 0.f;
            for (int i0 = 0, tl = 0; i0 < N; i0 += TI, ++tl) {
                float dot = 0.f;
#pragma unroll
                for (int q = 0; q < NW; ++q) dot += part[((size_t)(m & 1) * NW + q) * tiles * 32 + tl * 32 + lane];
                const bool valid = tt < TI && i0 + tt < N && tj < KP1;
                const float ex = expf(-fabsf(dot));
                const float rc = __frcp_rn(1.0f + ex);
                const float sg = dot >= 0.f ? rc : ex * rc;
                const bool pos = (tj == 0);
                gw[tl * 32 + lane] = valid ? alpha * ((pos ? 1.0f : 0.0f) - sg) : 0.f;
                if (valid) loss_f += fmaxf(pos ? -dot : dot, 0.f) - __logf(rc);
            }
            __syncwarp();
            // ---- a6: ΔOut_j = Σ_i G_ij A_i (snapshot), then ΔIn_i = Σ_j G_ij B_j into value + acc
            float2 dq[KP1MAX];
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j) dq[j] = make_float2(0.f, 0.f);
            for (int i = 0; i < N; ++i) {
                const float2 a = cok ? *reinterpret_cast<const float2*>(val + cs[i] * RS + col) : make_float2(0.f, 0.f);
                const float* gi = gw + (i / TI) * 32 + (i % TI) * KP1MAX;
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) dq[j] = ffma2(make_float2(gi[j], gi[j]), a, dq[j]);
            }
            for (int i = 0; i < N; ++i) {
                const float* gi = gw + (i / TI) * 32 + (i % TI) * KP1MAX;
                float2 d = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) d = ffma2(make_float2(gi[j], gi[j]), bq[j], d);
                if (cok) {
                    float2* v2 = reinterpret_cast<float2*>(val + cs[i] * RS + col);
                    float2* c2 = reinterpret_cast<float2*>(acc + cs[i] * RS + col);
                    *v2 = fadd2(*v2, d);
                    *c2 = fadd2(*c2, d);
                }
            }
            if (cok) {
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) *reinterpret_cast<float2*>(Bc + j * RS + col) = dq[j];
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(mbarD + cur);
            W2V_T(ph[7] += clock64() - t7; ph[8] += 1;)

            if (warp == 0) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) loss_f += __shfl_xor_sync(kFull, loss_f, o);
                st_loss += (double)loss_f;
                if (pp >= p.loss_tail_from) {
                    st_tail += (double)loss_f;
                    st_tail_pairs += (unsigned long long)N * KP1;
                }
                st_targets += 1;
                st_touch += (unsigned long long)(N + KP1);
                st_pairs += (unsigned long long)N * KP1;
                if (p.dbg_len && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len) {
                    const int64_t q = pp - p.dbg_base;
                    if (lane == 0) p.dbg_N[q] = (uint8_t)N;
                    for (int i = lane; i < N; i += 32) p.dbg_ctx[q * 2 * w + i] = kid[lo + i + (lo + i >= m ? 1 : 0)];
                    for (int k = lane; k < K; k += 32) p.dbg_neg[q * K + k] = bidc[1 + k];
                }
            }
        }
    }
    if (io) bulk_wait_all();  // smem sources of the last reductions must be read before exit
    W2V_T(if (lane == 0 && (io || warp == 0)) for (int i = 0; i < 16; ++i) if (ph[i]) atomicAdd(&g_gphase[i], ph[i]);)
    if (warp == 0 && lane == 0) {
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
    int nw, kp1;
    KernelFn fn;
};
#define W2V_INST(C, KK) {C, KK, hogbatch_wg_kernel<C, KK>}
const Inst kInst[] = {
    W2V_INST(1, 2), W2V_INST(1, 4), W2V_INST(1, 6), W2V_INST(1, 8), W2V_INST(1, 16),
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
        if (in.nw != need || in.kp1 < kp1) continue;
        if (!best || in.kp1 < best->kp1) best = &in;
    }
    return best;
}

}  // namespace

void wg_phase_report() {
#if defined(W2V_PHASE_TIMING)
    unsigned long long h[16];
    cudaMemcpyFromSymbol(h, g_gphase, sizeof h);
    if (!h[8]) return;
    const double T = (double)h[8];
    fprintf(stderr, "[phase] wg per target (cycles): IO wait-patch %.0f waits %.0f issue %.0f wait-done %.0f scatter %.0f | "
            "C0 wait-rows %.0f dots+bar %.0f rest %.0f  targets %llu\n",
            h[0] / T, h[1] / T, h[2] / T, h[3] / T, h[4] / T, h[5] / T, h[6] / T, h[7] / T, h[8]);
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_gphase, z, sizeof z);
#endif
}

size_t wg_cta_bytes(int L, int window, int K, int D, int32_t* slab_offset) {
    const Inst* in = pick(D, K);
    const int S = 2 * window + 2;
    if (!in || S > kWgMaxSlots) return 0;
    const int TI = 32 / in->kp1;
    const int tiles = (2 * window + TI - 1) / TI;
    const int Lp = (L + 3) & ~3;
    const size_t ints = (size_t)3 * Lp + 2 * kWgMaxSlots + kSampWin * (K > 0 ? K : 1) + 2 * in->kp1 + 4 * window;
    const size_t floats = (size_t)3 * in->nw * tiles * 32;
    const size_t head = 80 + ints * 4 + floats * 4;  // 64 B of mbarriers, 16 B header, then ints
    const size_t off = (head + 127) / 128 * 128;
    if (slab_offset) *slab_offset = (int32_t)off;
    return off + (size_t)(2 * S + 2 * in->kp1) * D * 4;
}

int wg_threads(int D) { return 32 * ((D + 63) / 64 + 1); }

int wg_max_ctas_per_sm(const StepParams& p) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return 0;
    int n = 0;
    cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, in->fn, 32 * (in->nw + 1), p.warp_bytes) != cudaSuccess) return 0;
    return n;
}

cudaError_t launch_wg(const StepParams& p, int ctas, cudaStream_t st) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (e != cudaSuccess) return e;
    in->fn<<<ctas, 32 * (in->nw + 1), p.warp_bytes, st>>>(p);
    return cudaGetLastError();
}

}  // namespace w2v
