// setup.cu — SURVEY.md §8(a) row a0 (once per w2v_train): id validation + counts, keep
// thresholds (C2), unigram^0.75 sampler prefix (C3) + guide table, and model init (C9).
// All on the device; the host reads back only SetupInfo (P[V], bad-id flag).
#include "w2v_device.cuh"
#include "w2v_internal.h"

namespace w2v {

namespace {

constexpr int kHot = 12288;  // smem-privatised counters for the Zipf-hot id prefix

// Counts c[w] = #{p : ids[p] = w}; flags ids outside [0,V) (SPEC.md:253 precondition).
__global__ void __launch_bounds__(512) hist_kernel(const int32_t* __restrict__ ids, int64_t n, int64_t V,
                                                   unsigned long long* __restrict__ counts, SetupInfo* info) {
    __shared__ unsigned int hot[kHot];
    const int H = (int)(V < kHot ? V : kHot);
    for (int i = threadIdx.x; i < H; i += blockDim.x) hot[i] = 0;
    __syncthreads();
    int bad = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int32_t w = __ldcs(ids + i);
        if (w < 0 || (int64_t)w >= V) { bad = 1; continue; }
        if (w < H) atomicAdd(&hot[w], 1u);
        else atomicAdd(&counts[w], 1ull);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(&info->bad_id, 1);
    for (int i = threadIdx.x; i < H; i += blockDim.x)
        if (hot[i]) atomicAdd(&counts[i], (unsigned long long)hot[i]);
}

// thr[w] (C2) and the raw sampler weight q[w] (C3) into P[w+1].
__global__ void weights_kernel(const unsigned long long* __restrict__ counts, int64_t V, int64_t T, float t,
                               uint64_t* __restrict__ thr, uint64_t* __restrict__ P) {
    const double t64 = (double)t;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < V; w += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long c = counts[w];
        uint64_t th = 4294967296ull;
        if (t64 != 0.0 && c != 0) {
            const double z = __ddiv_rn((double)c, __dmul_rn(t64, (double)T));
            const double k = __ddiv_rn(__dadd_rn(__dsqrt_rn(z), 1.0), z);
            if (k < 1.0) th = (uint64_t)floor(__dmul_rn(k, 4294967296.0));
        }
        thr[w] = th;
        const double x = (double)c;
        const double wgt = __dmul_rn(__dsqrt_rn(x), __dsqrt_rn(__dsqrt_rn(x)));
        P[w + 1] = (uint64_t)floor(__dmul_rn(wgt, 1048576.0));
        if (w == 0) P[0] = 0;
    }
}

constexpr int kScanT = 256, kScanI = 8, kScanTile = kScanT * kScanI;

// Block-wide inclusive scan of kScanTile u64 items held as v[kScanI] per thread (blocked order).
__device__ __forceinline__ uint64_t block_scan(uint64_t (&v)[kScanI], uint64_t* warp_tot) {
#pragma unroll
    for (int i = 1; i < kScanI; ++i) v[i] += v[i - 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t s = v[kScanI - 1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
    }
    if (lane == 31) warp_tot[wid] = s;
    __syncthreads();
    uint64_t off = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kScanT / 32; ++w) {
        if (w < wid) off += warp_tot[w];
        total += warp_tot[w];
    }
    off += s - v[kScanI - 1];
#pragma unroll
    for (int i = 0; i < kScanI; ++i) v[i] += off;
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(kScanT) scan_reduce_kernel(const uint64_t* __restrict__ x, int64_t n,
                                                             uint64_t* __restrict__ bsum) {
    __shared__ uint64_t wt[kScanT / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanI;
    uint64_t v[kScanI];
#pragma unroll
    for (int i = 0; i < kScanI; ++i) v[i] = (base + i < n) ? x[base + i] : 0;
    const uint64_t tot = block_scan(v, wt);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanT) scan_bsum_kernel(uint64_t* __restrict__ bsum, int64_t nb) {
    __shared__ uint64_t wt[kScanT / 32];
    uint64_t carry = 0;
    for (int64_t t0 = 0; t0 < nb; t0 += kScanTile) {
        const int64_t base = t0 + threadIdx.x * kScanI;
        uint64_t v[kScanI], raw[kScanI];
#pragma unroll
        for (int i = 0; i < kScanI; ++i) raw[i] = v[i] = (base + i < nb) ? bsum[base + i] : 0;
        const uint64_t tot = block_scan(v, wt);
#pragma unroll
        for (int i = 0; i < kScanI; ++i)
            if (base + i < nb) bsum[base + i] = carry + v[i] - raw[i];  // exclusive
        carry += tot;
    }
}

__global__ void __launch_bounds__(kScanT) scan_apply_kernel(uint64_t* __restrict__ x, int64_t n,
                                                            const uint64_t* __restrict__ bsum) {
    __shared__ uint64_t wt[kScanT / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanI;
    uint64_t v[kScanI];
#pragma unroll
    for (int i = 0; i < kScanI; ++i) v[i] = (base + i < n) ? x[base + i] : 0;
    block_scan(v, wt);
    const uint64_t off = bsum[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanI; ++i)
        if (base + i < n) x[base + i] = v[i] + off;
}

// Guide table G[k] = invcdf(min(k << gshift, P[V]-1)), k in [0, 2^gbits + 1]. gshift is the
// smallest shift with ((P[V]-1) >> gshift) < 2^gbits.
__global__ void guide_kernel(const uint64_t* __restrict__ P, int64_t V, int32_t* __restrict__ G, int gbits,
                             SetupInfo* info) {
    const uint64_t PV = P[V];
    const int bl = PV > 1 ? 64 - __clzll((long long)(PV - 1)) : 0;
    const int gshift = bl > gbits ? bl - gbits : 0;
    const int64_t nk = (1ll << gbits) + 2;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        info->PV = PV;
        info->gshift = gshift;
    }
    if (PV == 0) return;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nk; k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t x = (uint64_t)k << gshift;
        if (x > PV - 1) x = PV - 1;
        G[k] = (int32_t)invcdf_range(P, 0, V - 1, x);
    }
}

// C9: M_in[r][d] = ((float)(u32>>8)*2^-24 - 0.5f) / (float)D, M_out = 0. D % 4 == 0, so the
// 4 words of one Philox block land in one row.
__global__ void init_kernel(float* __restrict__ M, int64_t V, int32_t D, int32_t Ds, uint64_t seed) {
    const int64_t groups = V * (int64_t)D / 4;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const U4 r = philox(seed, kTagInit, 0u, (uint64_t)g, 0u);
        const int64_t e = g * 4, row = e / D, d = e % D;
        const uint32_t u[4] = {r.x, r.y, r.z, r.w};
        float4 v;
        float* vp = &v.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float f = __fmul_rn((float)(u[j] >> 8), 5.9604644775390625e-08f);
            vp[j] = __fdiv_rn(__fsub_rn(f, 0.5f), (float)D);
        }
        float* rowp = M + row * 2 * (int64_t)Ds;
        *reinterpret_cast<float4*>(rowp + d) = v;
        *reinterpret_cast<float4*>(rowp + Ds + d) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// flag |= 1 if any element of M[0, n) is NaN or Inf (divergence check)
__global__ void finite_kernel(const float4* __restrict__ M, size_t n4, int32_t* flag) {
    int bad = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = M[i];
        bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace

cudaError_t launch_finite_check(const float* M, size_t n, int32_t* flag, int sms, cudaStream_t st) {
    size_t b = (n / 4 + 255) / 256;
    if (b > (size_t)sms * 8) b = (size_t)sms * 8;
    if (b < 1) b = 1;
    finite_kernel<<<(int)b, 256, 0, st>>>(reinterpret_cast<const float4*>(M), n / 4, flag);
    return cudaGetLastError();
}

cudaError_t launch_hist(const int32_t* ids, int64_t n, int64_t V, unsigned long long* counts, SetupInfo* info,
                        int sms, cudaStream_t st, int* launches) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 511) / 512;
    if (blocks > (int64_t)sms * 2) blocks = (int64_t)sms * 2;
    hist_kernel<<<(int)blocks, 512, 0, st>>>(ids, n, V, counts, info);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_tables(const unsigned long long* counts, int64_t V, int64_t T, float t, uint64_t* thr,
                          uint64_t* P, uint64_t* scratch, int32_t* G, int gbits, SetupInfo* info, cudaStream_t st,
                          int* launches) {
    int64_t wb = (V + 255) / 256;
    if (wb > 65535) wb = 65535;
    weights_kernel<<<(int)wb, 256, 0, st>>>(counts, V, T, t, thr, P);
    const int64_t nb = (V + kScanTile - 1) / kScanTile;
    scan_reduce_kernel<<<(int)nb, kScanT, 0, st>>>(P + 1, V, scratch);
    scan_bsum_kernel<<<1, kScanT, 0, st>>>(scratch, nb);
    scan_apply_kernel<<<(int)nb, kScanT, 0, st>>>(P + 1, V, scratch);
    int64_t gb = (((int64_t)1 << gbits) + 2 + 255) / 256;
    if (gb > 65535) gb = 65535;
    guide_kernel<<<(int)gb, 256, 0, st>>>(P, V, G, gbits, info);
    *launches += 5;
    return cudaGetLastError();
}

cudaError_t launch_init(float* M, int64_t V, int32_t D, int32_t Ds, uint64_t seed, int sms, cudaStream_t st) {
    const int64_t groups = V * (int64_t)D / 4;
    int64_t blocks = (groups + 255) / 256;
    if (blocks > (int64_t)sms * 32) blocks = (int64_t)sms * 32;
    if (blocks < 1) blocks = 1;
    init_kernel<<<(int)blocks, 256, 0, st>>>(M, V, D, Ds, seed);
    return cudaGetLastError();
}

}  // namespace w2v
