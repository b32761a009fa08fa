// hogbatch.cu — the fused HogBatch step, sm_100a.
//
// One WARP is one work unit. It claims whole chunks (C5) from a global counter in increasing
// corpus order and, per chunk:
//   a1  keep flags (C2) + in-order compaction (ballot/popc) + half-window b (C4), in smem
//   per kept target, in chunk order (targets of a chunk are sequential, R11):
//   a2  K shared negatives (C7): lane d evaluates draw d in parallel, a ballot picks the
//       first K accepted draws (exactly C7's sequential redraw rule when >= K of the first
//       32 draws are accepted; otherwise a literal sequential fallback)
//   a3  gather the N context rows of M_in and the K+1 rows of M_out into the warp's smem slab
//       with 16-byte cp.async.cg (L2-only, no register staging) — the snapshot of R11
//   a4  C = A·Bᵀ: lane owns columns d = lane + 32c; B and the ΔOut accumulators live in
//       registers; each dot is finished with a 5-step xor butterfly (fp32 FMA, no tensor
//       cores: the tiles are ≤ 16x16, PAPER.md:116-126 GEMMs of this size waste a tcgen05 tile)
//   a5  E = [j=0] − σ(C), G = αE, loss (fp64 accumulation)
//   a6  ΔIn_i = G_i·B written over A_i in smem; ΔOut_j += G_ij·A_i in registers
//   a7  Hogwild scatter: red.global.add.v4.f32 of every slab row at L2,
//       same lane ↔ same 16-B column as its gather, so a warp always reads its own earlier
//       updates of a row in program order (deterministic mode adds a gpu-scope fence).
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

template <int CPL, int KP1MAX>
__global__ void __launch_bounds__(32) hogbatch_step_kernel(const StepParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    unsigned char* wbase = smem + (threadIdx.x >> 5) * p.warp_bytes;
    int32_t* kid = reinterpret_cast<int32_t*>(wbase);   // kept ids of the chunk
    int32_t* kinfo = kid + p.L;                          // (offset << 8) | b
    int32_t* rowid = kinfo + p.L;                        // ctx ids, then target + negatives
    float* slab = reinterpret_cast<float*>(wbase + p.slab_offset);

    const int D = p.D, D4 = D >> 2, K = p.K, KP1 = K + 1, window = p.window;
    const uint64_t PV = p.info->PV;
    const int gshift = p.info->gshift;
    const int64_t shard_end = p.shard_start + p.n_local;
    const uint32_t e = (uint32_t)p.epoch;

    unsigned long long st_words = 0, st_targets = 0, st_touch = 0, st_pairs = 0;
    double st_loss = 0.0;

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

        // ---------------- a1: subsampling (C2) + compaction + window (C4)
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
                p.dbg_keep[q] = keep;
                p.dbg_b[q] = keep ? (uint8_t)b : 0;
                p.dbg_N[q] = 0;
                for (int u = 0; u < 2 * window; ++u) p.dbg_ctx[q * 2 * window + u] = -1;
                for (int u = 0; u < (K > 0 ? K : 1); ++u) p.dbg_neg[q * (K > 0 ? K : 1) + u] = -1;
            }
            nk += __popc(m);
        }
        if (lane == 0) st_words += (unsigned long long)cnt;
        __syncwarp();

        // ---------------- per kept target, in order
        for (int m = 0; m < nk; ++m) {
            const int info = kinfo[m];
            const int b = info & 255;
            const int64_t pp = c0 + (info >> 8);
            const int32_t tw = kid[m];
            const int lo = m - b < 0 ? 0 : m - b;
            const int hi = m + b > nk - 1 ? nk - 1 : m + b;
            const int N = hi - lo;  // neighbours in [lo, hi] except m itself
            if (N == 0) continue;
            for (int i = lane; i < N; i += 32) {
                const int mm = lo + i + (lo + i >= m ? 1 : 0);
                rowid[i] = kid[mm];
            }
            // ---------------- a2: K shared negatives (C7)
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
                    // literal C7 (only reached when fewer than K of 32 draws are accepted)
                    uint32_t d = 0;
                    for (int k = 1; k <= K; ++k) {
                        int32_t y = (int32_t)((tw + 1) % p.V);
                        for (int tries = 0; tries < 100; ++tries, ++d) {
                            const U4 rr = philox(p.seed, kTagNeg, e, (uint64_t)pp, d >> 1);
                            const uint64_t uu = (d & 1) ? (((uint64_t)rr.w << 32) | rr.z)
                                                        : (((uint64_t)rr.y << 32) | rr.x);
                            const int32_t z = invcdf_guided(p.P, p.G, gshift, __umul64hi(uu, PV));
                            if (z != tw || p.allow_tn) { y = z; ++d; break; }
                        }
                        rowid[N + k] = y;
                    }
                }
            }
            if (lane == 0) rowid[N] = tw;
            __syncwarp();

            // ---------------- a3: gather snapshot rows into the slab (16-B cp.async.cg)
            const int R = N + KP1;
            for (int r = 0; r < R; ++r) {
                const int32_t id = rowid[r];
                const float* src = p.M + (size_t)id * 2 * D + (r < N ? 0 : D);
                float* dst = slab + r * D;
                for (int f = lane; f < D4; f += 32) cp_async16(dst + 4 * f, src + 4 * f);
            }
            // alpha (C8), computed while the copies fly
            const int64_t pi = (int64_t)p.epoch * p.n_local + (pp - p.shard_start);
            const int64_t num = (int64_t)p.world * (pi / p.Q) * p.Q;
            const double frac = __ddiv_rn((double)num, (double)((int64_t)p.epochs * p.n_global + 1));
            const float alpha = (float)__dmul_rn((double)p.alpha0, fmax(1.0 - frac, 1e-4));
            cp_async_wait_all();
            __syncwarp();

            // ---------------- a4-a6: C = A·Bᵀ, E, G, ΔIn, ΔOut
            float bq[KP1MAX][CPL], dq[KP1MAX][CPL];
            const float* Bs = slab + N * D;
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int d = lane + 32 * c;
                    bq[j][c] = (j < KP1 && d < D) ? Bs[j * D + d] : 0.f;
                    dq[j][c] = 0.f;
                }
            float lossacc = 0.f;
            for (int i = 0; i < N; ++i) {
                float* Ai = slab + i * D;
                float a[CPL];
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int d = lane + 32 * c;
                    a[c] = d < D ? Ai[d] : 0.f;
                }
                float dot[KP1MAX];
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) {
                    float s = 0.f;
#pragma unroll
                    for (int c = 0; c < CPL; ++c) s = fmaf(a[c], bq[j][c], s);
                    dot[j] = s;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int j = 0; j < KP1MAX; ++j) dot[j] += __shfl_xor_sync(kFull, dot[j], o);
                float g[KP1MAX];
                float mine = 0.f;
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j) {
                    const float sg = 1.0f / (1.0f + expf(-dot[j]));
                    g[j] = (j < KP1) ? alpha * ((j == 0 ? 1.0f : 0.0f) - sg) : 0.f;
                    if (lane == j) mine = dot[j];
                }
                if (lane < KP1) lossacc += softplus_f(lane == 0 ? -mine : mine);
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int d = lane + 32 * c;
                    float s = 0.f;
#pragma unroll
                    for (int j = 0; j < KP1MAX; ++j) s = fmaf(g[j], bq[j][c], s);
                    if (d < D) Ai[d] = s;
                }
#pragma unroll
                for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                    for (int c = 0; c < CPL; ++c) dq[j][c] = fmaf(g[j], a[c], dq[j][c]);
            }
            float* Bw = slab + N * D;
#pragma unroll
            for (int j = 0; j < KP1MAX; ++j)
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int d = lane + 32 * c;
                    if (j < KP1 && d < D) Bw[j * D + d] = dq[j][c];
                }
            __syncwarp();

            // ---------------- a7: Hogwild scatter-add (vector red at L2)
            for (int r = 0; r < R; ++r) {
                const int32_t id = rowid[r];
                float* dstg = p.M + (size_t)id * 2 * D + (r < N ? 0 : D);
                const float* src = slab + r * D;
                for (int f = lane; f < D4; f += 32) red_add_v4(dstg + 4 * f, lds4(src + 4 * f));
            }
            st_loss += (double)lossacc;
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
            if (p.deterministic) __threadfence();
            __syncwarp();
        }
    }

    // flush per-warp statistics
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) st_loss += __shfl_xor_sync(kFull, st_loss, o);
    if (lane == 0) {
        atomicAdd(&p.stats->words, st_words);
        atomicAdd(&p.stats->targets, st_targets);
        atomicAdd(&p.stats->row_touches, st_touch);
        atomicAdd(&p.stats->loss_pairs, st_pairs);
        atomicAdd(&p.stats->loss_sum, st_loss);
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
    const size_t ids = (size_t)(2 * L + 2 * window + K + 1) * 4;
    const size_t off = (ids + 15) / 16 * 16;
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
