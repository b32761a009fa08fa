// hogbatch_common.cuh — device pieces shared by the two fused-step kernels (hogbatch.cu: per-
// target gather/scatter; hogbatch_win.cu: window-resident rows). Rows a1/a2 of SURVEY.md §8(a).
#pragma once
#include "w2v_device.cuh"
#include "w2v_internal.h"

namespace w2v {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSampWin = 32;  // ring of sampled targets (negatives staged in smem)
constexpr int kSampGrp = 8;   // targets sampled together (independent L2 chains in flight)

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

// Blackwell packed fp32 FMA (FFMA2): two IEEE fmaf's, one issue slot.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&d);
}

// a1 (C2, C4, C5): subsampling of chunk positions [c0, c0+cnt), in-order compaction into
// kid/kinfo ((offset << 8) | b), debug stream. Returns the number of kept positions.
__device__ __forceinline__ int compact_chunk(const StepParams& p, int64_t c0, int cnt, int32_t* kid,
                                             int32_t* kinfo, int lane) {
    const uint32_t e = (uint32_t)p.epoch;
    const int window = p.window, KS = p.K > 0 ? p.K : 1;
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
            for (int u = 0; u < KS; ++u) p.dbg_neg[q * KS + u] = -1;
        }
        nk += __popc(m);
    }
    return nk;
}

// a2 (C7): negatives of kept targets [m_lo, m_lo+cnt) (cnt <= kSampGrp) into the negs ring
// (slot (m % kSampWin) * KS). Lane d evaluates draw d of every target; the guide-table and
// prefix loads of all targets are issued together; a ballot then keeps the first K accepted
// draws of each target (= C7's sequential redraw rule whenever >= K of the first 32 draws are
// accepted; otherwise a literal sequential fallback on lane 0).
__device__ __forceinline__ void sample_group(const StepParams& p, int m_lo, int cnt, int64_t c0,
                                             const int32_t* kid, const int32_t* kinfo, int32_t* negs,
                                             uint64_t PV, int gshift, int lane) {
    const uint32_t e = (uint32_t)p.epoch;
    const int K = p.K, KS = K > 0 ? K : 1;
    int32_t lo[kSampGrp], hi[kSampGrp], tw[kSampGrp];
    uint64_t x[kSampGrp];
#pragma unroll
    for (int t = 0; t < kSampGrp; ++t) {
        lo[t] = hi[t] = 0;
        tw[t] = -1;
        x[t] = 0;
        if (t < cnt) {
            const int64_t pp = c0 + (kinfo[m_lo + t] >> 8);
            tw[t] = kid[m_lo + t];
            const U4 r = philox(p.seed, kTagNeg, e, (uint64_t)pp, (uint32_t)(lane >> 1));
            const uint64_t u = (lane & 1) ? (((uint64_t)r.w << 32) | r.z) : (((uint64_t)r.y << 32) | r.x);
            x[t] = __umul64hi(u, PV);
            const uint64_t kb = x[t] >> gshift;
            lo[t] = __ldg(p.G + kb);
            hi[t] = __ldg(p.G + kb + 1);
        }
    }
    for (;;) {  // batched binary search: smallest w in [lo,hi] with P[w+1] > x (C3)
        bool act = false;
        int32_t mid[kSampGrp];
        uint64_t pv[kSampGrp];
#pragma unroll
        for (int t = 0; t < kSampGrp; ++t) {
            mid[t] = lo[t] + ((hi[t] - lo[t]) >> 1);
            pv[t] = 0;
            if (lo[t] < hi[t]) {
                pv[t] = __ldg(p.P + mid[t] + 1);
                act = true;
            }
        }
        if (!__any_sync(kFull, act)) break;
#pragma unroll
        for (int t = 0; t < kSampGrp; ++t)
            if (lo[t] < hi[t]) {
                if (pv[t] > x[t]) hi[t] = mid[t];
                else lo[t] = mid[t] + 1;
            }
    }
#pragma unroll
    for (int t = 0; t < kSampGrp; ++t) {
        if (t >= cnt) break;
        int32_t* out = negs + ((m_lo + t) % kSampWin) * KS;
        const bool acc = (lo[t] != tw[t]) || p.allow_tn;
        const unsigned am = __ballot_sync(kFull, acc);
        if (__popc(am) >= K) {
            const int rank = __popc(am & lanemask_lt());
            if (acc && rank < K) out[rank] = lo[t];
        } else if (lane == 0) {
            const int64_t pp = c0 + (kinfo[m_lo + t] >> 8);
            uint32_t d = 0;
            for (int k = 0; k < K; ++k) {
                int32_t y = (int32_t)((tw[t] + 1) % p.V);
                for (int tries = 0; tries < 100; ++tries, ++d) {
                    const U4 rr = philox(p.seed, kTagNeg, e, (uint64_t)pp, d >> 1);
                    const uint64_t uu = (d & 1) ? (((uint64_t)rr.w << 32) | rr.z) : (((uint64_t)rr.y << 32) | rr.x);
                    const int32_t z = invcdf_guided(p.P, p.G, gshift, __umul64hi(uu, PV));
                    if (z != tw[t] || p.allow_tn) {
                        y = z;
                        ++d;
                        break;
                    }
                }
                out[k] = y;
            }
        }
    }
}

// C8: alpha for rank-local progress pi (quantised by Q), fp64, rounded to fp32
__device__ __forceinline__ float alpha_at(const StepParams& p, int64_t qidx) {
    const int64_t den = (int64_t)p.epochs * p.n_global + 1;
    const double frac = __ddiv_rn((double)((int64_t)p.world * qidx * p.Q), (double)den);
    return (float)__dmul_rn((double)p.alpha0, fmax(1.0 - frac, 1e-4));
}

}  // namespace w2v
