// hogbatch_common.cuh — device pieces shared by the two fused-step kernels (hogbatch.cu: per-
// target gather/scatter; hogbatch_win.cu: window-resident rows): reading the batch stream of
// rows a1/a2 (batch.cu), packed fp32 math, the learning-rate schedule.
#pragma once
#include "w2v_device.cuh"
#include "w2v_internal.h"

namespace w2v {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSampWin = 32;  // ring of targets whose negatives are staged in smem
constexpr int kSampWinRows = 16;  // hogbatch.cu's ring: it fetches at most 16 targets ahead
constexpr int kSampGrp = 8;   // targets whose negatives are fetched together (one async group)

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

// Chunk rel of the launch's batch stream (batch.cu: a1 subsampling + window batching, a2
// negatives) into the warp's smem: kid / kinfo (Lp ints each, 16-B async copies), the kept count
// nk, and the negatives of kept targets [0, kSampGrp) into the ring — one cp.async group.
// Reading past nk (stale slots, or the next chunk's) is harmless: the buffers are padded.
template <int RING = kSampWin>
__device__ __forceinline__ void fetch_negs(const StepParams& p, int64_t rel, int m_lo, int cnt, int32_t* negs,
                                           int lane) {
    const int K = p.K;  // K > 0 here, so KS == K and a group of targets is contiguous
    const int32_t* src = p.bt_neg + (rel * p.Lp + m_lo) * K;
    int32_t* dst = negs + (m_lo % RING) * K;
    for (int u = lane; u < cnt * K; u += 32) cp_async4(dst + u, src + u);
}
template <int RING = kSampWin>
__device__ __forceinline__ void load_chunk(const StepParams& p, int64_t rel, int32_t* kid, int32_t* kinfo,
                                           int32_t* nk_s, int32_t* negs, int lane) {
    const int q = kid ? p.Lp >> 2 : 0;  // kid == nullptr: the caller reads kid/kinfo from global
    const int4* sk = reinterpret_cast<const int4*>(p.bt_kid + rel * p.Lp);
    const int4* si = reinterpret_cast<const int4*>(p.bt_kinfo + rel * p.Lp);
    for (int i = lane; i < q; i += 32) {
        cp_async16(kid + 4 * i, sk + i);
        cp_async16(kinfo + 4 * i, si + i);
    }
    if (lane == 0) cp_async4(nk_s, p.bt_nk + rel);
    if (p.K > 0) fetch_negs<RING>(p, rel, 0, kSampGrp, negs, lane);
    cp_async_commit();
}

// C8: alpha for rank-local progress pi (quantised by Q), fp64, rounded to fp32
__device__ __forceinline__ float alpha_at(const StepParams& p, int64_t qidx) {
    const int64_t den = (int64_t)p.epochs * p.n_global + 1;
    const double frac = __ddiv_rn((double)((int64_t)p.world * qidx * p.Q), (double)den);
    return (float)__dmul_rn((double)p.alpha0, fmax(1.0 - frac, 1e-4));
}

}  // namespace w2v
