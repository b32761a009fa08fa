// hogbatch.cu — the fused HogBatch step, sm_100a.
//
// One WARP is one work unit. It claims whole chunks (C5) from a global counter in increasing
// corpus order and, per chunk:
//   a1  keep flags (C2) + in-order compaction (ballot/popc) + half-window b (C4), in smem
//   per kept target, in chunk order (targets of a chunk are sequential, R11):
//   a2  K shared negatives (C7): lane d evaluates draw d in parallel, a ballot picks the
//       first K accepted draws (exactly C7's sequential redraw rule when >= K of the first
//       32 draws are accepted; otherwise a literal sequential fallback). Drawn for target m+1
//       while the rows of target m are in flight (the sampler's dependent L2 loads overlap
//       the gather).
//   a3  gather the N context rows of M_in and the K+1 rows of M_out into the warp's smem slab:
//       one bulk copy (cp.async.bulk, the TMA engine) per row, completing on an mbarrier —
//       the snapshot of R11, no register staging, ~1 instruction per row
//   a4  C = A·Bᵀ: lane owns columns d = lane + 32c; B and the ΔOut accumulators live in
//       registers; the N x (K+1) partial dots are finished by a butterfly reduce-scatter
//       (lane ends with one dot), fp32 FMA — no tensor cores: tiles are <= 16x16
//   a5  E = [j=0] − σ(C) once per lane, G = αE broadcast by shuffles; loss in fp64
//   a6  ΔIn_i = G_i·B written over A_i in smem; ΔOut_j += G_ij·A_i in registers, then over B_j
//   a7  Hogwild scatter: one bulk fp32 reduce-add per row
//       (cp.reduce.async.bulk .add.f32, element-atomic at L2); the warp waits for completion
//       before the next target's gather so a chunk's targets see each other's updates.
// Paper mapping: Alg.1 loops over inputs and outputs one dot at a time;
// HogBatch batches them into C = A·Bᵀ and the two update GEMMs; the
// "write back at the end of the GEMM" is the scatter of a7.
#include <cstdio>

#include "w2v_device.cuh"
#include "w2v_internal.h"

namespace w2v {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int KP1MAX>
struct Pow2 {
    static constexpr int v = KP1MAX <= 1 ? 1 : KP1MAX <= 2 ? 2 : KP1MAX <= 4 ? 4 : KP1MAX <= 8 ? 8 : KP1MAX <= 16 ? 16 : 32;
    static constexpr int lg = v == 1 ? 0 : v == 2 ? 1 : v == 4 ? 2 : v == 8 ? 3 : v == 16 ? 4 : 5;
};

// Per-target state produced ahead of time by prepare() (double-buffered rowid lists).
struct Tgt {
    int m, N;
    int64_t pp;
};

#ifndef W2V_MINB
#define W2V_MINB 11  // resident 1-warp CTAs per SM the register budget is sized for
#endif
template <int CPL, int KP1MAX>
__global__ void __launch_bounds__(32, W2V_MINB) hogbatch_step_kernel(const StepParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int P2 = Pow2<KP1MAX>::v, LG = Pow2<KP1MAX>::lg, SH = 5 - LG;
    const int lane = threadIdx.x & 31;
    unsigned char* wbase = smem + (threadIdx.x >> 5) * p.warp_bytes;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase);
    const int D = p.D, K = p.K, KP1 = K + 1, window = p.window, RMAX = 2 * window + KP1;
    int32_t* kid = reinterpret_cast<int32_t*>(wbase + 16);   // kept ids of the chunk
    int32_t* kinfo = kid + p.L;                               // (offset << 8) | b
    int32_t* rowid0 = kinfo + p.L;                            // 2 x RMAX: ctx ids, target, negatives
    float* slab = reinterpret_cast<float*>(wbase + p.slab_offset);
    const uint32_t rowbytes = (uint32_t)D * 4u;

    const uint64_t PV = p.info->PV;
    const int gshift = p.info->gshift;
    const int64_t shard_end = p.shard_start + p.n_local;
    const uint32_t e = (uint32_t)p.epoch;
    const int64_t alpha_den = (int64_t)p.epochs * p.n_global + 1;

    if (lane == 0) mbar_init(mbar, 1);
    __syncwarp();
    uint32_t phase = 0;

    unsigned long long st_words = 0, st_targets = 0, st_touch = 0, st_pairs = 0;
    float st_loss_f = 0.f;
    double st_loss = 0.0, st_tail = 0.0;
    unsigned long long st_tail_pairs = 0;

    // C7 negatives + C6 context of kept target m into rowid[0..N+K]
    auto prepare = [&](int m, int nk, int64_t c0, int32_t* rowid) -> Tgt {
        const int info = kinfo[m];
        const int b = info & 255;
        const int64_t pp = c0 + (info >> 8);
        const int32_t tw = kid[m];
        const int lo = m - b < 0 ? 0 : m - b;
        const int hi = m + b > nk - 1 ? nk - 1 : m + b;
        const int N = hi - lo;
        for (int i = lane; i < N; i += 32) {
            const int mm = lo + i + (lo + i >= m ? 1 : 0);
            rowid[i] = kid[mm];
        }
        if (K > 0) {
            const U4 r = philox(p.seed, kTagNeg, e, (uint64_t)pp, (uint32_t)(lane >> 1));
            const uint64_t u = (lane & 1) ? (((uint64_t)r.w << 32) | r.z) : (((uint64_t)r.y << 32) | r.x);
            const int32_t x = invcdf_guided(p.P, p.G, gshift, __umul64hi(u, PV));
            const bool acc = (x != tw) || p.allow_tn;
            const unsigned am = __ballot_sync(kFull, acc);
            if (__popc(am) >= K) {
                const int rank = __popc(am & lanemask_lt());
                if (acc && rank < K) rowid[N + 1 + rank] = x;
            } else if (lane == 0) {
                // literal C7 (only reached when fewer than K of the first 32 draws are accepted)
                uint32_t d = 0;
                for (int k = 1; k <= K; ++k) {
                    int32_t y = (int32_t)((tw + 1) % p.V);
                    for (int tries = 0; tries < 100; ++tries, ++d) {
                        const U4 rr = philox(p.seed, kTagNeg, e, (uint64_t)pp, d >> 1);
                        const uint64_t uu = (d & 1) ? (((uint64_t)rr.w << 32) | rr.z) : (((uint64_t)rr.y << 32) | rr.x);
                        const int32_t z = invcdf_guided(p.P, p.G, gshift, __umul64hi(uu, PV));
                        if (z != tw || p.allow_tn) { y = z; ++d; break; }
                    }
                    rowid[N + k] = y;
                }
            }
        }
        if (lane == 0) rowid[N] = tw;
        return Tgt{m, N, pp};
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

        // ---------------- a1: subsampling (C2) + in-order compaction + window (C4)
        int nk = 0;
        for (int k0 = 0; k0 < cnt; k0 += 32) {
            const int k = k0 + lane;
            bool keep = false;
            int32_t w = 0;
            uint32_t u1 = 0;
            const int64_t pp = c0 + k;
            if (k < cnt) {
                w = __ldg(p.ids + (pp - p.ids_base));
                const U4 r = philox(p.seed, kTagPos, e, (uint64_t)pp, 0u);
                keep = (uint64_t)r.x < __ldg(p.thr + w);
                u1 = r.y;
            }
            const unsigned m = __ballot_sync(kFull, keep);
            const int b = 1 + (int)(((uint64_t)u1 * (uint64_t)window) >> 32);
            if (keep) {
                const int slot = nk + __popc(m & lanemask_lt());
                kid[slot] = w;
                kinfo[slot] = (k << 8) | b;
            }
            if (p.dbg_len && k < cnt && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len) {
                const int64_t q = pp - p.dbg_base;
                const int kk = K > 0 ? K : 1;
                p.dbg_keep[q] = keep;
                p.dbg_b[q] = keep ? (uint8_t)b : 0;
                p.dbg_N[q] = 0;
                for (int u = 0; u < 2 * window; ++u) p.dbg_ctx[q * 2 * window + u] = -1;
                for (int u = 0; u < kk; ++u) p.dbg_neg[q * kk + u] = -1;
            }
            nk += __popc(m);
        }
        if (lane == 0) st_words += (unsigned long long)cnt;
        __syncwarp();
        if (nk < 2) continue;  // N = 0 for every kept target iff the chunk keeps < 2 words

        // alpha (C8) for the chunk's first quantum and the next one (a chunk spans <= 2 quanta
        // only when L > Q; the general case is handled by recomputing below)
        const int64_t pi0 = (int64_t)p.epoch * p.n_local + (c0 - p.shard_start);
        int64_t qcur = pi0 / p.Q;
        auto alpha_of = [&](int64_t qidx) -> float {
            const int64_t num = (int64_t)p.world * qidx * p.Q;
            const double frac = __ddiv_rn((double)num, (double)alpha_den);
            return (float)__dmul_rn((double)p.alpha0, fmax(1.0 - frac, 1e-4));
        };
        float alpha_cur = alpha_of(qcur);

        // ---------------- per kept target, in order; negatives of target m+1 are drawn while
        // the rows of target m are in flight
        int buf = 0;
        Tgt t = prepare(0, nk, c0, rowid0);
        __syncwarp();
        for (;;) {
            int32_t* rowid = rowid0 + buf * RMAX;
            const int N = t.N, R = N + KP1;
            // ---------------- a3: gather the snapshot rows (one bulk copy per row)
            if (lane == 0) mbar_arrive_expect_tx(mbar, (uint32_t)R * rowbytes);
            __syncwarp();
            for (int r = lane; r < R; r += 32) {
                const int32_t id = rowid[r];
                bulk_g2s(slab + r * D, p.M + (size_t)id * 2 * D + (r < N ? 0 : D), rowbytes, mbar);
            }
            const bool has_next = t.m + 1 < nk;
            Tgt tn{};
            if (has_next) tn = prepare(t.m + 1, nk, c0, rowid0 + (buf ^ 1) * RMAX);
            const int64_t pi = (int64_t)p.epoch * p.n_local + (t.pp - p.shard_start);
            if (pi / p.Q != qcur) { qcur = pi / p.Q; alpha_cur = alpha_of(qcur); }
            const float alpha = alpha_cur;
            mbar_wait(mbar, phase);
            phase ^= 1u;

            // ---------------- a4-a6: C = A·Bᵀ, E, G, ΔIn (over A), ΔOut (registers, then over B)
            float bq[KP1MAX][CPL], dq[KP1MAX][CPL];
            float* Bs = slab + N * D;
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int d = lane + 32 * c;
                    bq[j][c] = (j < KP1 && d < D) ? Bs[j * D + d] : 0.f;
                    dq[j][c] = 0.f;
                }
            const int jj = (lane >> SH) & (P2 - 1);   // the dot this lane holds after the reduce-scatter
            for (int i = 0; i < N; ++i) {
                float* Ai = slab + i * D;
                float a[CPL];
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int d = lane + 32 * c;
                    a[c] = d < D ? Ai[d] : 0.f;
                }
                float v[P2];
#pragma unroll
                for (int j = 0; j < P2; ++j) {
                    float s2 = 0.f;
                    if (j < KP1MAX) {
#pragma unroll
                        for (int c = 0; c < CPL; ++c) s2 = fmaf(a[c], bq[j][c], s2);
                    }
                    v[j] = s2;
                }
                // butterfly reduce-scatter: after LG halving steps lane holds dot jj (partial over
                // the lanes sharing jj), then plain xor-sums finish it
#pragma unroll
                for (int st = 0; st < LG; ++st) {
                    const int o = 16 >> st;
                    const int half = P2 >> (st + 1);
                    const bool up = lane & o;
#pragma unroll
                    for (int u = 0; u < half; ++u) {
                        const float send = up ? v[u] : v[u + half];
                        const float keep = up ? v[u + half] : v[u];
                        v[u] = keep + __shfl_xor_sync(kFull, send, o);
                    }
                }
                float dot = v[0];
#pragma unroll
                for (int o = (1 << SH) >> 1; o > 0; o >>= 1) dot += __shfl_xor_sync(kFull, dot, o);
                // E = label - sigma(C) (exact sigma, one per lane), G = alpha * E
                const float sg = 1.0f / (1.0f + expf(-dot));
                const float gl = (jj < KP1) ? alpha * ((jj == 0 ? 1.0f : 0.0f) - sg) : 0.f;
                if (jj < KP1 && (lane & ((1 << SH) - 1)) == 0) st_loss_f += softplus_f(jj == 0 ? -dot : dot);
                float g[KP1MAX];
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) g[j] = __shfl_sync(kFull, gl, j << SH);
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int d = lane + 32 * c;
                    float s2 = 0.f;
#pragma unroll
                    for (int j = 0; j < KP1MAX; ++j) s2 = fmaf(g[j], bq[j][c], s2);
                    if (d < D) Ai[d] = s2;
                }
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                    for (int c = 0; c < CPL; ++c) dq[j][c] = fmaf(g[j], a[c], dq[j][c]);
            }
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int d = lane + 32 * c;
                    if (j < KP1 && d < D) Bs[j * D + d] = dq[j][c];
                }
            fence_proxy_async_smem();
            __syncwarp();

            // ---------------- a7: Hogwild scatter-add, one bulk fp32 reduction per row at L2
            for (int r = lane; r < R; r += 32) {
                const int32_t id = rowid[r];
                bulk_red_add_s2g(p.M + (size_t)id * 2 * D + (r < N ? 0 : D), slab + r * D, rowbytes);
            }
            bulk_commit();
            st_loss += (double)st_loss_f;   // per-target partial (<= N terms) into fp64 (C11)
            if (t.pp >= p.loss_tail_from) {
                st_tail += (double)st_loss_f;
                if (lane == 0) st_tail_pairs += (unsigned long long)N * KP1;
            }
            st_loss_f = 0.f;
            if (lane == 0) {
                st_targets += 1;
                st_touch += (unsigned long long)R;
                st_pairs += (unsigned long long)N * KP1;
            }
            if (p.dbg_len && t.pp >= p.dbg_base && t.pp < p.dbg_base + p.dbg_len) {
                const int64_t q = t.pp - p.dbg_base;
                if (lane == 0) p.dbg_N[q] = (uint8_t)N;
                for (int i = lane; i < N; i += 32) p.dbg_ctx[q * 2 * window + i] = rowid[i];
                for (int k = lane; k < K; k += 32) p.dbg_neg[q * K + k] = rowid[N + 1 + k];
            }
            // the next target's gather must see these updates (R11: targets of a chunk are
            // sequential) and the slab must be free: wait for the reductions to complete
            bulk_wait_all();
            if (p.deterministic) __threadfence();
            __syncwarp();
            if (!has_next) break;
            t = tn;
            buf ^= 1;
        }
    }

    // flush per-warp statistics
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        st_loss += __shfl_xor_sync(kFull, st_loss, o);
        st_tail += __shfl_xor_sync(kFull, st_tail, o);
    }
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
    int cpl, kp1;
    KernelFn fn;
};

#define W2V_INST(C, KK) {C, KK, hogbatch_step_kernel<C, KK>}
// (columns-per-lane, max K+1) instantiations; register footprint ~ 2*CPL*KP1MAX floats.
const Inst kInst[] = {
    W2V_INST(1, 2),  W2V_INST(1, 4),  W2V_INST(1, 6),  W2V_INST(1, 8),  W2V_INST(1, 16), W2V_INST(1, 32),
    W2V_INST(2, 2),  W2V_INST(2, 4),  W2V_INST(2, 6),  W2V_INST(2, 8),  W2V_INST(2, 16), W2V_INST(2, 32),
    W2V_INST(4, 2),  W2V_INST(4, 4),  W2V_INST(4, 6),  W2V_INST(4, 8),  W2V_INST(4, 16),
    W2V_INST(8, 2),  W2V_INST(8, 4),  W2V_INST(8, 6),  W2V_INST(8, 8),
    W2V_INST(10, 2), W2V_INST(10, 4), W2V_INST(10, 6), W2V_INST(10, 8),
    W2V_INST(16, 2), W2V_INST(16, 4), W2V_INST(16, 6),
};
#undef W2V_INST

const Inst* pick(int D, int K) {
    const int cpl_need = (D + 31) / 32, kp1 = K + 1;
    const Inst* best = nullptr;
    for (const Inst& in : kInst) {
        if (in.cpl < cpl_need || in.kp1 < kp1) continue;
        if (!best || in.cpl * in.kp1 < best->cpl * best->kp1) best = &in;
    }
    return best;
}

}  // namespace

bool step_supported(int D, int K) { return pick(D, K) != nullptr; }

size_t step_warp_bytes(int L, int window, int K, int D, int32_t* slab_offset) {
    // [mbarrier 16 B][kid L][kinfo L][rowid 2 x (2w+K+1)] [slab (2w+K+1) x D fp32]
    const size_t ids = 16 + (size_t)(2 * L + 2 * (2 * window + K + 1)) * 4;
    const size_t off = (ids + 127) / 128 * 128;
    if (slab_offset) *slab_offset = (int32_t)off;
    return off + (size_t)(2 * window + K + 1) * D * 4;
}

int step_max_ctas_per_sm(const StepParams& p) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return 0;
    int n = 0;
    cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, in->fn, 32, p.warp_bytes) != cudaSuccess) return 0;
    return n;
}

cudaError_t launch_step(const StepParams& p, int ctas, cudaStream_t st) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (e != cudaSuccess) return e;
    in->fn<<<ctas, 32, p.warp_bytes, st>>>(p);
    return cudaGetLastError();
}

}  // namespace w2v
