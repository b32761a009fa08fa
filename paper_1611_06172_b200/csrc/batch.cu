// batch.cu — SURVEY.md §8(a) rows a1 (frequency subsampling + window batching) and a2 (the
// counter-based-RNG unigram^0.75 negative sampler) as their own kernel, run once per launch
// range of chunks just before the fused step kernel consumes its output.
//
// Why a separate kernel: both rows are chains of dependent L2 loads (thr[ids[p]]; guide table
// then a binary search over the u64 prefix P). Inside the fused step, whose occupancy is capped
// by its row slabs (~10 warps/SM), those chains sat on every warp's critical path (r01 ablation:
// removing the sampler from the step kernel raised cfg3 throughput by 41%). Here they run at
// full occupancy, where the latency is hidden by other warps, and the step kernel reads a
// compact batch stream (~30 B per kept target, <0.3% of the row traffic).
//
// Output, per chunk s of the launch range (rel = s - chunk_lo; Lp = L rounded up to 4):
//   bt_nk[rel]                       number of kept positions of the chunk (C2, C5)
//   bt_kid[rel*Lp + m]               word of kept position m, in corpus order (C6)
//   bt_kinfo[rel*Lp + m]             (offset of m inside the chunk) << 8 | b   (C4)
//   bt_neg[(rel*Lp + m)*KS + k]      k-th shared negative of kept target m (C7), written only
//                                    when the chunk keeps >= 2 positions (else N = 0 for all)
// plus the keep / b debug records (w2v_debug_batches) for positions in the debug range.
#include "w2v_device.cuh"
#include "w2v_internal.h"

namespace w2v {

namespace {

constexpr unsigned kAll = 0xffffffffu;
constexpr int kBatchWarps = 8;            // warps per CTA
constexpr int kMaskWords = 4096 / 32;     // sentence_len <= 4096

__device__ __forceinline__ unsigned lane_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// draw d of the NEG stream at position pp (C1: block idx = d >> 1, half d & 1) through C3
__device__ __forceinline__ int32_t neg_draw(const StepParams& p, uint32_t e, int64_t pp, uint32_t d, uint64_t PV,
                                            int gshift) {
    const U4 r = philox(p.seed, kTagNeg, e, (uint64_t)pp, d >> 1);
    const uint64_t u = (d & 1) ? (((uint64_t)r.w << 32) | r.z) : (((uint64_t)r.y << 32) | r.x);
    return invcdf_guided(p.P, p.G, gshift, __umul64hi(u, PV));
}

// No shared memory (the redo masks live in a small global scratch): with ~1 KB of smem left by
// the step kernel's slabs, one block of this kernel can co-reside on every SM and run the NEXT
// launch range's batch stream while the step kernel consumes the current one (capi.cu).
__global__ void __launch_bounds__(32 * kBatchWarps) batch_kernel(const StepParams p) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // targets whose first K draws hit a rejection (one bit each), per warp
    uint32_t* fix = p.bt_redo + ((size_t)blockIdx.x * kBatchWarps + wid) * kMaskWords;
    const uint32_t e = (uint32_t)p.epoch;
    const int window = p.window, K = p.K, KS = K > 0 ? K : 1, Lp = p.Lp;
    const int64_t shard_end = p.shard_start + p.n_local;
    const uint64_t PV = p.info->PV;
    const int gshift = p.info->gshift;
    const int64_t nwarps = (int64_t)gridDim.x * kBatchWarps;

    for (int64_t s = p.chunk_lo + (int64_t)blockIdx.x * kBatchWarps + wid; s < p.chunk_hi; s += nwarps) {
        const int64_t rel = s - p.chunk_lo;
        int64_t c0 = s * (int64_t)p.L, c1 = c0 + p.L;
        if (c1 > shard_end) c1 = shard_end;
        if (c0 < p.shard_start) c0 = p.shard_start;
        const int cnt = c1 > c0 ? (int)(c1 - c0) : 0;
        int32_t* kid = p.bt_kid + rel * Lp;
        int32_t* kinfo = p.bt_kinfo + rel * Lp;

        // ---- a1: keep iff u32(POS,e,p)[0] < thr[ids[p]] (C2); compaction in order; b (C4)
        int nk = 0;
        for (int k0 = 0; k0 < cnt; k0 += 32) {
            const int k = k0 + lane;
            const int64_t pp = c0 + k;
            bool keep = false;
            int32_t w = 0;
            uint32_t u1 = 0;
            if (k < cnt) {
                w = __ldg(p.ids + (pp - p.ids_base));
                const U4 r = philox(p.seed, kTagPos, e, (uint64_t)pp, 0u);
                keep = (uint64_t)r.x < __ldg(p.thr + w);
                u1 = r.y;
            }
            const unsigned m = __ballot_sync(kAll, keep);
            const int b = 1 + (int)(((uint64_t)u1 * (uint64_t)window) >> 32);
            if (keep) {
                const int slot = nk + __popc(m & lane_lt());
                kid[slot] = w;
                kinfo[slot] = (k << 8) | b;
            }
            if (p.dbg_len && k < cnt && pp >= p.dbg_base && pp < p.dbg_base + p.dbg_len) {
                const int64_t q = pp - p.dbg_base;
                p.dbg_keep[q] = keep;
                p.dbg_b[q] = keep ? (uint8_t)b : 0;
                p.dbg_N[q] = 0;  // the step kernel fills N / ctx / negatives of trained targets
                for (int u = 0; u < 2 * window; ++u) p.dbg_ctx[q * 2 * window + u] = -1;
                for (int u = 0; u < KS; ++u) p.dbg_neg[q * KS + u] = -1;
                if (p.dbg_a1neg)
                    for (int u = 0; u < 2 * window * KS; ++u) p.dbg_a1neg[q * 2 * window * KS + u] = -1;
            }
            nk += __popc(m);
        }
        if (lane == 0) p.bt_nk[rel] = nk;
        if (nk < 2 || K == 0) continue;  // N = 0 for every kept target iff nk < 2
        __syncwarp();                    // kid / kinfo written by other lanes are visible below

        if (p.algorithm == 1) {
            // ---- Alg.1 l.10: K negatives per (target m, input i) on the A1NEG stream, draw
            // counter d restarting at 0 per input, block idx = i << 12 | d >> 1 (C1). One lane
            // per (m, i) runs C7's redraw rule literally.
            const int W2 = 2 * window;
            for (int u = lane; u < nk * W2; u += 32) {
                const int m = u / W2, i = u - m * W2;
                const int bm = kinfo[m] & 255;
                const int lo = m - bm < 0 ? 0 : m - bm, hi = m + bm > nk - 1 ? nk - 1 : m + bm;
                if (i >= hi - lo) continue;
                const int64_t pp = c0 + (kinfo[m] >> 8);
                const int32_t tw = kid[m];
                int32_t* out = p.bt_neg + ((rel * Lp + m) * W2 + i) * K;
                uint32_t d = 0;
                for (int k = 0; k < K; ++k) {
                    int32_t y = (int32_t)((tw + 1) % p.V);
                    for (int tries = 0; tries < 100; ++tries, ++d) {
                        const U4 r = philox(p.seed, kTagA1Neg, e, (uint64_t)pp, ((uint32_t)i << 12) | (d >> 1));
                        const uint64_t uu = (d & 1) ? (((uint64_t)r.w << 32) | r.z) : (((uint64_t)r.y << 32) | r.x);
                        const int32_t z = invcdf_guided(p.P, p.G, gshift, __umul64hi(uu, PV));
                        if (z != tw || p.allow_tn) { y = z; ++d; break; }
                    }
                    out[k] = y;
                }
            }
            continue;
        }

        // ---- a2: K negatives per kept target (C7). Lane u handles Philox block j = u % KB of
        // target m = u / KB (KB = ceil(K/2)): its two u64 halves are draws 2j and 2j+1 (C1), so
        // each block is computed once and each lane runs two independent inverse-CDF chains —
        // assuming no rejection before them; a target whose first K draws contain a rejection
        // (x == target) is redone by one lane with the literal sequential rule.
        for (int i = lane; i < (nk + 31) / 32; i += 32) fix[i] = 0u;
        __syncwarp();
        int32_t* neg = p.bt_neg + rel * Lp * KS;
        const int KB = (K + 1) >> 1;
        for (int u = lane; u < nk * KB; u += 32) {
            const int m = u / KB, j = u - m * KB;
            const int64_t pp = c0 + (kinfo[m] >> 8);
            const int32_t tw = kid[m];
            const U4 r = philox(p.seed, kTagNeg, e, (uint64_t)pp, (uint32_t)j);
            const int32_t x0 = invcdf_guided(p.P, p.G, gshift, __umul64hi(((uint64_t)r.y << 32) | r.x, PV));
            const bool two = 2 * j + 1 < K;
            const int32_t x1 = two ? invcdf_guided(p.P, p.G, gshift, __umul64hi(((uint64_t)r.w << 32) | r.z, PV)) : 0;
            bool bad = false;
            if (x0 != tw || p.allow_tn) neg[m * KS + 2 * j] = x0;
            else bad = true;
            if (two) {
                if (x1 != tw || p.allow_tn) neg[m * KS + 2 * j + 1] = x1;
                else bad = true;
            }
            if (bad) atomicOr(fix + (m >> 5), 1u << (m & 31));
        }
        __syncwarp();
        for (int m = lane; m < nk; m += 32) {
            if (!((fix[m >> 5] >> (m & 31)) & 1u)) continue;
            const int64_t pp = c0 + (kinfo[m] >> 8);
            const int32_t tw = kid[m];
            uint32_t d = 0;
            for (int k = 0; k < K; ++k) {
                int32_t y = (int32_t)((tw + 1) % p.V);
                for (int tries = 0; tries < 100; ++tries) {
                    const int32_t z = neg_draw(p, e, pp, d++, PV, gshift);
                    if (z != tw || p.allow_tn) { y = z; break; }
                }
                neg[m * KS + k] = y;
            }
        }
        __syncwarp();
    }
}

}  // namespace

size_t batch_redo_words(int sms) { return (size_t)sms * 8 * kBatchWarps * kMaskWords; }

cudaError_t launch_batch(const StepParams& p, int sms, int blocks_per_sm, cudaStream_t st) {
    const int64_t chunks = p.chunk_hi - p.chunk_lo;
    if (chunks <= 0) return cudaSuccess;
    int64_t blocks = (chunks + kBatchWarps - 1) / kBatchWarps;
    if (blocks_per_sm < 1 || blocks_per_sm > 8) blocks_per_sm = 8;
    if (blocks > (int64_t)sms * blocks_per_sm) blocks = (int64_t)sms * blocks_per_sm;
    batch_kernel<<<(int)blocks, 32 * kBatchWarps, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace w2v
