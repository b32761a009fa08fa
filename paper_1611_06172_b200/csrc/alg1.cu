// alg1.cu — Algorithm 1, the "original" word2vec SGNS update (SURVEY.md §8(f)
// NEXT-3), on B200, sm_100a: the level-1 baseline HogBatch is compared against (PAPER.md:186,
// Fig. 3a). Same chunks, subsampling, windows and learning rate as the HogBatch path (C2-C8);
// what differs is the paper's point:
//   * every input word i of a target draws its OWN K negatives (Alg.1 l.10; A1NEG stream,
//     drawn by batch.cu), and
//   * every (input, output) pair is one dot product followed by an immediate update of that
//     output row (l.13-17), the input row is updated once per input (l.20): N(K+1) + N row
//     updates per target instead of HogBatch's N + K + 1.
//
// One warp = one work unit (a chunk, targets in order, like hogbatch.cu). The lane owns float2
// columns d = 2*lane + 64c of every row; rows live in registers (no shared-memory slab, so the
// occupancy is set by registers alone). Per input: the input row and its K negative rows are
// loaded together (ld.relaxed.gpu: one round trip), the target row M_out[tw] stays in
// registers for the whole target. Each dot is a warp all-reduce (5 shuffles); each update goes
// to the model as red.relaxed.gpu.add.v2.f32 AND to the register copy, so later pairs of the
// same target see it exactly as the sequential algorithm does (duplicate rows inside one input's
// output list are kept in sync in registers). A lane only ever touches its own columns, so its
// later loads of a row are ordered after its own earlier reductions of that row (same thread,
// same address, both morally strong) — the warp's view of the model is the sequential one.
#include <cstdio>

#include "hogbatch_common.cuh"

namespace w2v {

namespace {

#ifndef W2V_A1_MINB
#define W2V_A1_MINB 16  // resident warps per SM the register budget is sized for (<= 128 registers)
#endif

__device__ __forceinline__ float2 ld_relaxed2(const float* p) {
    float2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_add2(float* p, float2 v) {
    asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

// Alg.1 l.13 on one (input, output) pair: the full dot product, in every lane
template <int CP2>
__device__ __forceinline__ float warp_dot(const float2 (&a)[CP2], const float2 (&b)[CP2]) {
    float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < CP2; ++c) s2 = ffma2(a[c], b[c], s2);
    float s = s2.x + s2.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    return s;
}

template <int CP2, int KMAX>
__global__ void __launch_bounds__(32, W2V_A1_MINB) alg1_kernel(const StepParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    unsigned char* wbase = smem + (threadIdx.x >> 5) * p.warp_bytes;
    int32_t* nk_s = reinterpret_cast<int32_t*>(wbase + 8);
    int32_t* kid = reinterpret_cast<int32_t*>(wbase + 16);
    int32_t* kinfo = kid + p.Lp;
    const int D = p.D, Ds = p.Ds, K = p.K, W2 = 2 * p.window;
    const int64_t shard_end = p.shard_start + p.n_local;

    // lane's columns: float2 c at d = 2*lane + 64c; the last float2 columns may be past D
    bool colok[CP2];
#pragma unroll
    for (int c = 0; c < CP2; ++c) colok[c] = 2 * lane + 64 * c < D;

    unsigned long long st_words = 0, st_targets = 0, st_touch = 0, st_pairs = 0, st_tail_pairs = 0;
    double st_loss = 0.0, st_tail = 0.0;

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
        {   // the chunk's kept words and (offset << 8) | b (batch.cu)
            const int q = p.Lp >> 2;
            const int4* sk = reinterpret_cast<const int4*>(p.bt_kid + rel * p.Lp);
            const int4* si = reinterpret_cast<const int4*>(p.bt_kinfo + rel * p.Lp);
            for (int i = lane; i < q; i += 32) {
                cp_async16(kid + 4 * i, sk + i);
                cp_async16(kinfo + 4 * i, si + i);
            }
            if (lane == 0) cp_async4(nk_s, p.bt_nk + rel);
            cp_async_wait_all();
            __syncwarp();
        }
        const int nk = *nk_s;
        if (lane == 0) st_words += (unsigned long long)cnt;
        if (nk < 2) continue;

        int64_t q_next = -1;
        float alpha = 0.f;
        for (int m = 0; m < nk; ++m) {
            const int b = kinfo[m] & 255;
            const int64_t pp = c0 + (kinfo[m] >> 8);
            const int lo = m - b < 0 ? 0 : m - b;
            const int hi = m + b > nk - 1 ? nk - 1 : m + b;
            const int N = hi - lo;
            const int32_t tw = kid[m];
            const int64_t pi = (int64_t)p.epoch * p.n_local + (pp - p.shard_start);
            if (pi >= q_next) {
                const int64_t qi = pi / p.Q;
                q_next = (qi + 1) * p.Q;
                alpha = alpha_at(p, qi);
            }
            const int32_t* negm = p.bt_neg + (rel * p.Lp + m) * (int64_t)W2 * K;
            // l.8: the target row, in registers for the whole target (its updates go to both)
            float* pt = p.M + (size_t)tw * 2 * Ds + Ds + 2 * lane;
            float2 bt[CP2];
#pragma unroll
            for (int c = 0; c < CP2; ++c) bt[c] = colok[c] ? ld_relaxed2(pt + 64 * c) : make_float2(0.f, 0.f);
            double loss_t = 0.0;
            for (int i = 0; i < N; ++i) {                                   // l.2
                const int32_t in = kid[lo + i + (lo + i >= m ? 1 : 0)];     // l.3
                // l.10 ids of this input's K negatives (lane k holds id k), then all loads
                int32_t myneg = lane < K ? __ldg(negm + i * K + lane) : -1;
                int32_t nid[KMAX];
#pragma unroll
                for (int k = 0; k < KMAX; ++k) nid[k] = __shfl_sync(kFull, myneg, k < K ? k : 0);
                float* pa = p.M + (size_t)in * 2 * Ds + 2 * lane;
                float2 a[CP2], bn[KMAX][CP2];
#pragma unroll
                for (int c = 0; c < CP2; ++c) a[c] = colok[c] ? ld_relaxed2(pa + 64 * c) : make_float2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
#pragma unroll
                    for (int c = 0; c < CP2; ++c)
                        bn[k][c] = (k < K && colok[c]) ? ld_relaxed2(p.M + (size_t)nid[k] * 2 * Ds + Ds + 2 * lane + 64 * c)
                                                       : make_float2(0.f, 0.f);
                // duplicates: a negative equal to the target, or to an earlier negative of
                // this input, must read the value as updated by the earlier pairs (l.17)
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    if (k >= K) break;
                    if (nid[k] == tw) {
#pragma unroll
                        for (int c = 0; c < CP2; ++c) bn[k][c] = bt[c];
                    }
                }
                float2 tmp[CP2];                                            // l.4
#pragma unroll
                for (int c = 0; c < CP2; ++c) tmp[c] = make_float2(0.f, 0.f);
                // ---- k = 0: the target (label 1), l.8 and l.12-17
                {
                    const float inn = warp_dot<CP2>(a, bt);
                    const float ex = expf(-fabsf(inn));
                    const float rc = __frcp_rn(1.0f + ex);
                    const float sg = inn >= 0.f ? rc : ex * rc;
                    const float err = 1.0f - sg;                            // l.14
                    loss_t += (double)(fmaxf(-inn, 0.f) - __logf(rc));
                    const float g = __fmul_rn(alpha, err);
#pragma unroll
                    for (int c = 0; c < CP2; ++c) {
                        tmp[c] = ffma2(make_float2(err, err), bt[c], tmp[c]);  // l.15
                        const float2 dl = make_float2(__fmul_rn(g, a[c].x), __fmul_rn(g, a[c].y));
                        bt[c] = make_float2(__fadd_rn(bt[c].x, dl.x), __fadd_rn(bt[c].y, dl.y));  // l.17
                        if (colok[c]) red_add2(pt + 64 * c, dl);
                    }
#pragma unroll
                    for (int k = 0; k < KMAX; ++k)
                        if (k < K && nid[k] == tw) {
#pragma unroll
                            for (int c = 0; c < CP2; ++c) bn[k][c] = bt[c];
                        }
                }
                // ---- k = 1..K: the negatives (label 0)
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    if (k >= K) break;
                    const float inn = warp_dot<CP2>(a, bn[k]);
                    const float ex = expf(-fabsf(inn));
                    const float rc = __frcp_rn(1.0f + ex);
                    const float sg = inn >= 0.f ? rc : ex * rc;
                    const float err = 0.0f - sg;
                    loss_t += (double)(fmaxf(inn, 0.f) - __logf(rc));
                    const float g = __fmul_rn(alpha, err);
                    float* pn = p.M + (size_t)nid[k] * 2 * Ds + Ds + 2 * lane;
#pragma unroll
                    for (int c = 0; c < CP2; ++c) {
                        tmp[c] = ffma2(make_float2(err, err), bn[k][c], tmp[c]);
                        const float2 dl = make_float2(__fmul_rn(g, a[c].x), __fmul_rn(g, a[c].y));
                        bn[k][c] = make_float2(__fadd_rn(bn[k][c].x, dl.x), __fadd_rn(bn[k][c].y, dl.y));
                        if (colok[c]) red_add2(pn + 64 * c, dl);
                    }
                    // keep every copy of this row in sync (later duplicates, and the target row)
#pragma unroll
                    for (int k2 = k + 1; k2 < KMAX; ++k2)
                        if (k2 < K && nid[k2] == nid[k]) {
#pragma unroll
                            for (int c = 0; c < CP2; ++c) bn[k2][c] = bn[k][c];
                        }
                    if (nid[k] == tw) {
#pragma unroll
                        for (int c = 0; c < CP2; ++c) bt[c] = bn[k][c];
                    }
                }
                // l.20: the input row once per input
#pragma unroll
                for (int c = 0; c < CP2; ++c)
                    if (colok[c]) red_add2(pa + 64 * c, make_float2(__fmul_rn(alpha, tmp[c].x), __fmul_rn(alpha, tmp[c].y)));
                if (p.dbg_len && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len && lane < K)
                    p.dbg_a1neg[((pp - p.dbg_base) * W2 + i) * K + lane] = myneg;
            }
            st_loss += loss_t;
            if (pp >= p.loss_tail_from) {
                st_tail += loss_t;
                if (lane == 0) st_tail_pairs += (unsigned long long)N * (K + 1);
            }
            if (lane == 0) {
                st_targets += 1;
                st_touch += (unsigned long long)N * (K + 1) + N;
                st_pairs += (unsigned long long)N * (K + 1);
            }
            if (p.dbg_len && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len) {
                const int64_t q = pp - p.dbg_base;
                if (lane == 0) p.dbg_N[q] = (uint8_t)N;
                for (int i = lane; i < N; i += 32) p.dbg_ctx[q * W2 + i] = kid[lo + i + (lo + i >= m ? 1 : 0)];
            }
            if (p.deterministic) __threadfence();
        }
    }
    if (lane == 0) {  // loss was accumulated identically in every lane: count it once
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
    int cp2, kmax;
    KernelFn fn;
};
#define W2V_INST(C, KK) {C, KK, alg1_kernel<C, KK>}
const Inst kInst[] = {
    W2V_INST(1, 1), W2V_INST(1, 3), W2V_INST(1, 5), W2V_INST(1, 15), W2V_INST(1, 31),
    W2V_INST(2, 1), W2V_INST(2, 3), W2V_INST(2, 5), W2V_INST(2, 15),
    W2V_INST(3, 1), W2V_INST(3, 3), W2V_INST(3, 5), W2V_INST(3, 15),
    W2V_INST(5, 1), W2V_INST(5, 3), W2V_INST(5, 5), W2V_INST(5, 7),
    W2V_INST(8, 1), W2V_INST(8, 3), W2V_INST(8, 5),
};
#undef W2V_INST

const Inst* pick(int D, int K) {
    const int need = (D + 63) / 64, kk = K < 1 ? 1 : K;
    const Inst* best = nullptr;
    for (const Inst& in : kInst) {
        if (in.cp2 < need || in.kmax < kk) continue;
        if (!best || in.cp2 * in.kmax < best->cp2 * best->kmax) best = &in;
    }
    return best;
}

}  // namespace

bool alg1_supported(int D, int K) { return pick(D, K) != nullptr; }

size_t alg1_warp_bytes(int L) {
    const int Lp = (L + 3) & ~3;
    return ((size_t)16 + (size_t)2 * Lp * 4 + 15) / 16 * 16;
}

int alg1_max_ctas_per_sm(const StepParams& p) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return 0;
    int n = 0;
    cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, in->fn, 32, p.warp_bytes) != cudaSuccess) return 0;
    return n;
}

cudaError_t launch_alg1(const StepParams& p, int ctas, cudaStream_t st) {
    const Inst* in = pick(p.D, p.K);
    if (!in) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(in->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.warp_bytes);
    if (e != cudaSuccess) return e;
    in->fn<<<ctas, 32, p.warp_bytes, st>>>(p);
    return cudaGetLastError();
}

}  // namespace w2v
