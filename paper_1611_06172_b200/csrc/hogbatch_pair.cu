// hogbatch_pair.cu — the fused HogBatch step with TWO warps per work unit, the K+1 output rows
// split between them, sm_100a. Same contract, batch stream, data
// movement and per-target order as hogbatch.cu (one bulk copy per row in, one bulk reduce-add
// per row out, each target waiting for its reductions — R11); only the compute is divided.
//
// Why: with many outputs per target (cfg4: K+1 = 16 shared negatives, N <= 16 inputs, D = 128)
// the one-warp kernel is bound by the latency of a4-a6 (~7,500 cycles per target):
// N·16 dots finished by butterfly reduce-scatters, then N·16·2 FFMA2 per lane for ΔOut and
// ΔIn. Here warp h owns outputs [h·H, h·H + H):
//   a4  its N·H dots (C = A·B_hᵀ; a butterfly per 32/H inputs), σ, G and loss of its outputs;
//   a6  ΔOut_j (j in its half) = Σ_i G_ij A_i over the snapshot A, in registers;
//       ΔIn_i = Σ_{all j} G_ij B_j = partial_0 + partial_1: after both warps have read A,
//       warp 0 writes its partial over A_i, warp 1 adds its own (the same two-term sum for
//       every i; the order of the halves is fixed, so runs are reproducible);
//   a7  warp 0 issues the bulk reduce-adds of all N + K + 1 rows.
// Both halves of the per-target critical path shrink by ~2x; the CTA (the unit) synchronises
// with __syncthreads (64 threads) three times per target.
// Paper mapping: PAPER.md:116-126 (the HogBatch minibatch GEMMs), :135-138 (Hogwild).
#include <cstdio>

#include "hogbatch_common.cuh"

namespace w2v {

namespace {

constexpr int kPairSmemChunk = 256;  // chunks up to this many (padded) kept slots are staged in smem

#ifndef W2V_PAIR_MINB
#define W2V_PAIR_MINB 10  // resident 2-warp units per SM the register budget is sized for
#endif

// CP2 float2 columns per lane (D <= 64*CP2); H outputs per warp (K+1 <= 2H); RSC packed stride
template <int CP2, int H, int RSC>
__global__ void __launch_bounds__(64, W2V_PAIR_MINB) hogbatch_pair_kernel(const StepParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int KP1MAX = 2 * H;
    constexpr int TI = 32 / H;  // inputs per reduce-scatter tile of one warp
    const int lane = threadIdx.x & 31, h = threadIdx.x >> 5;
    unsigned char* wbase = smem;  // one unit per CTA
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase);
    int32_t* nk_s = reinterpret_cast<int32_t*>(wbase + 8);
    long long* chunk_s = reinterpret_cast<long long*>(wbase + 16);
    const int D = p.D, Ds = p.Ds, K = p.K, KP1 = K + 1, window = p.window, RMAX = 2 * window + KP1;
    const int KS = K > 0 ? K : 1;
    const bool chunk_smem = p.Lp <= kPairSmemChunk;
    int32_t* kid_s = reinterpret_cast<int32_t*>(wbase + 32);
    const int Lps = chunk_smem ? p.Lp : 0;
    int32_t* rowid0 = kid_s + 2 * Lps;                        // 2 x RMAX: ctx ids, target, negatives
    int32_t* negs = rowid0 + 2 * RMAX;                        // kSampWinRows x KS negatives ring
    const int gtile = ((2 * window + TI - 1) / TI) * 32;      // G floats per warp
    float* gs = reinterpret_cast<float*>(negs + kSampWinRows * KS) + h * gtile;  // this warp's G
    constexpr int RS = RSC > 0 ? RSC : 64 * CP2;
    const bool lastok = RS >= 64 * CP2 || 2 * lane + 64 * (CP2 - 1) < D;
    float* Bs = reinterpret_cast<float*>(wbase + p.slab_offset);  // KP1MAX rows: target, negatives
    float* As = Bs + KP1MAX * RS;                                 // 2*window rows: context
    float* Bh = Bs + h * H * RS;                                  // this warp's output rows
    const uint32_t rowbytes = (uint32_t)D * 4u;
    const int64_t shard_end = p.shard_start + p.n_local;
    const uint64_t pol_hot = (p.l2_hint & 1) ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_cold = (p.l2_hint & 2) ? policy_evict_first() : policy_evict_normal();
    if (threadIdx.x == 0) mbar_init(mbar, 1);
    for (int i = threadIdx.x; i < (KP1MAX + 2 * window) * RS / 4; i += 64)
        reinterpret_cast<float4*>(Bs)[i] = make_float4(0.f, 0.f, 0.f, 0.f);  // padding stays 0
    __syncthreads();
    uint32_t phase = 0;

    unsigned long long st_words = 0, st_targets = 0, st_touch = 0, st_pairs = 0, st_tail_pairs = 0;
    unsigned st_cold = 0;
    float st_loss_f = 0.f;
    double st_loss = 0.0, st_tail = 0.0;

    const int32_t* kid = kid_s;
    const int32_t* kinfo = kid_s + Lps;
    auto gather_list = [&](int m, int nk, int32_t* rowid) -> int {  // warp 0 (C6, C7)
        const int b = kinfo[m] & 255;
        const int lo = m - b < 0 ? 0 : m - b;
        const int hi = m + b > nk - 1 ? nk - 1 : m + b;
        const int N = hi - lo;
        for (int i = lane; i < N; i += 32) rowid[i] = kid[lo + i + (lo + i >= m ? 1 : 0)];
        if (lane == 0) rowid[N] = kid[m];
        const int32_t* ng = negs + (m % kSampWinRows) * KS;
        for (int k = lane; k < K; k += 32) rowid[N + 1 + k] = ng[k];
        return N;
    };
    auto count_N = [&](int m, int nk) -> int {
        const int b = kinfo[m] & 255;
        const int lo = m - b < 0 ? 0 : m - b;
        const int hi = m + b > nk - 1 ? nk - 1 : m + b;
        return hi - lo;
    };

    for (;;) {
        if (threadIdx.x == 0) *chunk_s = (long long)atomicAdd(p.chunk_ctr, 1ull) + p.chunk_lo;
        __syncthreads();
        const long long s = *chunk_s;
        __syncthreads();  // (chunk_s is rewritten by the next claim)
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
            if (threadIdx.x == 0) {
                bulk_prefetch_l2(kid, (uint32_t)p.Lp * 4u);
                bulk_prefetch_l2(kinfo, (uint32_t)p.Lp * 4u);
            }
        }
        if (h == 0) {
            load_chunk<kSampWinRows>(p, rel, chunk_smem ? kid_s : nullptr, kid_s + Lps, nk_s, negs, lane);
            cp_async_wait_all();
        }
        __syncthreads();
        const int nk = *nk_s;
        if (threadIdx.x == 0) st_words += (unsigned long long)cnt;
        if (nk < 2) continue;

        int64_t q_next = -1;
        float alpha = 0.f;
        int samp_hi = nk < kSampGrp ? nk : kSampGrp;
        int buf = 0;
        int N = (h == 0) ? gather_list(0, nk, rowid0) : count_N(0, nk);
        __syncthreads();
        for (int m = 0; m < nk; ++m) {
            int32_t* rowid = rowid0 + buf * RMAX;
            const int R = N + KP1;
            const int64_t pp = c0 + (kinfo[m] >> 8);
            // ---------------- a3 (warp 0): one bulk copy per row into the slab
            if (h == 0) {
                if (lane == 0) mbar_arrive_expect_tx(mbar, (uint32_t)R * rowbytes);
                __syncwarp();
                for (int r = lane; r < R; r += 32) {
                    const int32_t id = rowid[r];
                    st_cold += id >= p.cold_from;
                    float* dst = r < N ? As + r * RS : Bs + (r - N) * RS;
                    bulk_g2s_hint(dst, p.M + (size_t)id * 2 * Ds + (r < N ? 0 : Ds), rowbytes, mbar,
                                  id < (r < N ? p.hot_rows_in : p.hot_rows) ? pol_hot : pol_cold);
                }
                if (K > 0 && samp_hi < nk && samp_hi - (m + 1) < kSampGrp) {
                    const int c = nk - samp_hi < kSampGrp ? nk - samp_hi : kSampGrp;
                    fetch_negs<kSampWinRows>(p, rel, samp_hi, c, negs, lane);
                    samp_hi += c;
                }
                cp_async_commit();
                cp_async_wait_but_last();
                __syncwarp();
            }
            // next target's row list (warp 0) / size (warp 1), alpha, while the rows fly
            const int Nn = (m + 1 < nk) ? (h == 0 ? gather_list(m + 1, nk, rowid0 + (buf ^ 1) * RMAX) : count_N(m + 1, nk))
                                        : 0;
            const int64_t pi = (int64_t)p.epoch * p.n_local + (pp - p.shard_start);
            if (pi >= q_next) {
                const int64_t qi = pi / p.Q;
                q_next = (qi + 1) * p.Q;
                alpha = alpha_at(p, qi);
            }
            mbar_wait(mbar, phase);
            phase ^= 1u;

            // ---------------- a4-a6 on this warp's H outputs
            if (p.rowpath_only) {
                if (h == 0) {
                    float4* z = reinterpret_cast<float4*>(Bs);
                    for (int u = lane; u < (KP1MAX + 2 * window) * RS / 4; u += 32) z[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            } else {
                float2 bq[H][CP2], dq[H][CP2];
#pragma unroll
                for (int j = 0; j < H; ++j)
#pragma unroll
                    for (int c = 0; c < CP2; ++c) {
                        bq[j][c] = (c < CP2 - 1 || lastok) ? *reinterpret_cast<const float2*>(Bh + j * RS + 2 * lane + 64 * c)
                                                           : make_float2(0.f, 0.f);
                        dq[j][c] = make_float2(0.f, 0.f);
                    }
                const int tt = lane / H, tj = lane - tt * H;  // dot held after the reduce-scatter
                const int jg = h * H + tj;                    // its global output index
                for (int i0 = 0; i0 < N; i0 += TI) {
                    float v[32];
#pragma unroll
                    for (int t = 0; t < TI; ++t) {
                        if (i0 + t >= N) {
#pragma unroll
                            for (int j = 0; j < H; ++j) v[t * H + j] = 0.f;
                            continue;
                        }
                        const float* Ai = As + (i0 + t) * RS + 2 * lane;
                        float2 a[CP2];
#pragma unroll
                        for (int c = 0; c < CP2; ++c)
                            a[c] = (c < CP2 - 1 || lastok) ? *reinterpret_cast<const float2*>(Ai + 64 * c) : make_float2(0.f, 0.f);
#pragma unroll
                        for (int j = 0; j < H; ++j) {
                            float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
                            for (int c = 0; c < CP2; ++c) s2 = ffma2(a[c], bq[j][c], s2);
                            v[t * H + j] = s2.x + s2.y;
                        }
                    }
#pragma unroll
                    for (int u = TI * H; u < 32; ++u) v[u] = 0.f;
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
                    const float dot = v[0];
                    const bool valid = tt < TI && i0 + tt < N && jg < KP1;
                    const float ex = expf(-fabsf(dot));
                    const float rc = __frcp_rn(1.0f + ex);
                    const float sg = dot >= 0.f ? rc : ex * rc;
                    const bool pos = (jg == 0);
                    if (lane < TI * H) gs[i0 * H + lane] = valid ? alpha * ((pos ? 1.0f : 0.0f) - sg) : 0.f;
                    if (valid) st_loss_f += fmaxf(pos ? -dot : dot, 0.f) - __logf(rc);
                }
                __syncwarp();
                // ΔOut_j = Σ_i G_ij A_i (snapshot A) for this warp's outputs
                for (int i = 0; i < N; ++i) {
                    const float* Ai = As + i * RS + 2 * lane;
                    float2 a[CP2];
#pragma unroll
                    for (int c = 0; c < CP2; ++c)
                        a[c] = (c < CP2 - 1 || lastok) ? *reinterpret_cast<const float2*>(Ai + 64 * c) : make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < H; ++j) {
                        const float gj = gs[i * H + j];
                        const float2 g2 = make_float2(gj, gj);
#pragma unroll
                        for (int c = 0; c < CP2; ++c) dq[j][c] = ffma2(g2, a[c], dq[j][c]);
                    }
                }
                __syncthreads();  // both warps are done reading A (snapshot)
                // ΔIn_i = partial_0 + partial_1 written over A_i: warp 0 stores, then warp 1 adds
                for (int pass = 0; pass < 2; ++pass) {
                    if (h == pass) {
                        for (int i = 0; i < N; ++i) {
                            float* Ai = As + i * RS + 2 * lane;
                            float2 g2[H];
#pragma unroll
                            for (int j = 0; j < H; ++j) {
                                const float gj = gs[i * H + j];
                                g2[j] = make_float2(gj, gj);
                            }
#pragma unroll
                            for (int c = 0; c < CP2; ++c) {
                                constexpr int NCH = (H >= 8 && CP2 <= 2) ? 4 : (H >= 4 ? 2 : 1);
                                float2 s2[NCH];
#pragma unroll
                                for (int q = 0; q < NCH; ++q) s2[q] = make_float2(0.f, 0.f);
#pragma unroll
                                for (int j = 0; j < H; ++j) s2[j % NCH] = ffma2(g2[j], bq[j][c], s2[j % NCH]);
#pragma unroll
                                for (int q = 1; q < NCH; ++q) s2[0] = fadd2(s2[0], s2[q]);
                                if (c < CP2 - 1 || lastok) {
                                    float2* x = reinterpret_cast<float2*>(Ai + 64 * c);
                                    *x = pass == 0 ? s2[0] : fadd2(*x, s2[0]);
                                }
                            }
                        }
                    }
                    __syncthreads();
                }
#pragma unroll
                for (int j = 0; j < H; ++j)
#pragma unroll
                    for (int c = 0; c < CP2; ++c)
                        if (c < CP2 - 1 || lastok) *reinterpret_cast<float2*>(Bh + j * RS + 2 * lane + 64 * c) = dq[j][c];
            }
            fence_proxy_async_smem();
            __syncthreads();  // every ΔIn / ΔOut row written (and visible to the bulk engine)
            st_loss += (double)st_loss_f;
            if (pp >= p.loss_tail_from) st_tail += (double)st_loss_f;
            st_loss_f = 0.f;
            if (h == 0) {
                // ---------------- a7: Hogwild scatter-add, one bulk fp32 reduction per row
                for (int r = lane; r < R; r += 32) {
                    const int32_t id = rowid[r];
                    const float* src = r < N ? As + r * RS : Bs + (r - N) * RS;
                    bulk_red_add_s2g_hint(p.M + (size_t)id * 2 * Ds + (r < N ? 0 : Ds), src, rowbytes,
                                          id < (r < N ? p.hot_rows_in : p.hot_rows) ? pol_hot : pol_cold);
                }
                bulk_commit();
                if (lane == 0) {
                    st_targets += 1;
                    st_touch += (unsigned long long)R;
                    st_pairs += (unsigned long long)N * KP1;
                    if (pp >= p.loss_tail_from) st_tail_pairs += (unsigned long long)N * KP1;
                }
                if (p.dbg_len && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len) {
                    const int64_t q = pp - p.dbg_base;
                    if (lane == 0) p.dbg_N[q] = (uint8_t)N;
                    for (int i = lane; i < N; i += 32) p.dbg_ctx[q * 2 * window + i] = rowid[i];
                    for (int k = lane; k < K; k += 32) p.dbg_neg[q * K + k] = rowid[N + 1 + k];
                }
                // the next target's gathers must see these reductions (R11), the slab be free
                if (p.deterministic || p.scatter_wait) bulk_wait_all();
                else bulk_wait_read_all();
                if (p.deterministic) __threadfence();
            }
            __syncthreads();  // warp 1 must not touch the slab before the next gather lands
            N = Nn;
            buf ^= 1;
        }
    }

#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        st_loss += __shfl_xor_sync(kFull, st_loss, o);
        st_tail += __shfl_xor_sync(kFull, st_tail, o);
        st_cold += __shfl_xor_sync(kFull, st_cold, o);
    }
    if (lane == 0) {
        atomicAdd(&p.stats->loss_sum, st_loss);
        if (st_tail != 0.0) atomicAdd(&p.stats->loss_tail_sum, st_tail);
        if (h == 0) {
            atomicAdd(&p.stats->words, st_words);
            atomicAdd(&p.stats->targets, st_targets);
            atomicAdd(&p.stats->row_touches, st_touch);
            atomicAdd(&p.stats->loss_pairs, st_pairs);
            atomicAdd(&p.stats->row_touches_cold, (unsigned long long)st_cold);
            if (st_tail_pairs) atomicAdd(&p.stats->loss_tail_pairs, st_tail_pairs);
        }
    }
}

using KernelFn = void (*)(const StepParams);
struct Inst {
    int cp2, h, rs;
    KernelFn fn;
};
#define W2V_PINST(C, HH) {C, HH, 0, hogbatch_pair_kernel<C, HH, 0>}
const Inst kInst[] = {
    W2V_PINST(1, 4), W2V_PINST(1, 8), W2V_PINST(1, 16),
    W2V_PINST(2, 4), W2V_PINST(2, 8),
    W2V_PINST(3, 4), W2V_PINST(3, 8),
    W2V_PINST(4, 4),
    W2V_PINST(5, 3), W2V_PINST(5, 4),
    {5, 3, 300, hogbatch_pair_kernel<5, 3, 300>},  // the paper's D=300, K<=5, packed rows
};
#undef W2V_PINST

const Inst* pick(int D, int K) {
    const int need = (D + 63) / 64, kp1 = K + 1;
    for (const Inst& in : kInst)
        if (in.rs == D && in.cp2 >= need && 2 * in.h >= kp1) return &in;
    const Inst* best = nullptr;
    for (const Inst& in : kInst) {
        if (in.rs != 0 || in.cp2 < need || 2 * in.h < kp1) continue;
        if (!best || in.cp2 * in.h < best->cp2 * best->h) best = &in;
    }
    return best;
}

}  // namespace

bool pair_supported(int D, int K) { return pick(D, K) != nullptr; }

size_t pair_cta_bytes(int L, int window, int K, int D, int32_t* slab_offset) {
    // [mbarrier 8 | nk 4 | pad 4 | chunk 8 | pad 8][kid Lp][kinfo Lp][rowid 2 x (2w+K+1)]
    // [negs 16 x max(K,1)][G: 2 warps x tiles x 32][slab: 2H B rows + 2w A rows, stride RS]
    const Inst* in = pick(D, K);
    if (!in) return 0;
    const int RS = in->rs > 0 ? in->rs : 64 * in->cp2;
    const int R = 2 * window + K + 1;
    const int TI = 32 / in->h;
    const size_t gfl = (size_t)((2 * window + TI - 1) / TI) * 32 * 2;
    const int Lp = (L + 3) & ~3;
    const int Lps = Lp <= kPairSmemChunk ? Lp : 0;
    const size_t ids = 32 + (size_t)(2 * Lps + 2 * R + kSampWinRows * (K > 0 ? K : 1)) * 4 + gfl * 4;
    const size_t off = (ids + 15) / 16 * 16;
    if (slab_offset) *slab_offset = (int32_t)off;
    return off + (size_t)(2 * in->h + 2 * window) * RS * 4;
}

int pair_max_ctas_per_sm(const StepParams& p) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return 0;
    int n = 0;
    cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, in->fn, 64, p.warp_bytes) != cudaSuccess) return 0;
    return n;
}

cudaError_t launch_pair(const StepParams& p, int ctas, cudaStream_t st) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (e != cudaSuccess) return e;
    in->fn<<<ctas, 64, p.warp_bytes, st>>>(p);
    return cudaGetLastError();
}

}  // namespace w2v
