/*
 * inputs/gen_cuda.cu — the SAME seeded synthetic corpus as gen.c, generated on the GPU (test and
 * bench INPUTS only; holds none of the method's arithmetic). BASELINE.json cfg5 asks for its 8B
 * tokens to be "generated on-device from seed": a 32 GB corpus per replica is never staged
 * through the host.
 *
 * Bit-exact with gen.c by construction: the only floating point of the recipe (the Zipf weights
 * pow(w+1,-s), quantised to u64) is computed ONCE on the host by gen.c's own table builders and
 * uploaded; everything here is integer: Philox4x32-10 (GEN tag), mulhi64, and an inverse CDF
 * over those u64 prefix tables. A guide table over the prefix (bucket k of x >> shift -> the
 * candidate range) keeps the search to ~1-3 probes per token; it only narrows the range of the
 * same "smallest k with pre[k+1] > x" search, so it cannot change a result.
 */
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr uint32_t kGenTag = 4u;

__device__ __forceinline__ uint64_t gen_u64(uint64_t seed, uint64_t ctr, uint32_t idx) {
    uint32_t c0 = (uint32_t)ctr, c1 = (uint32_t)(ctr >> 32), c2 = 0u, c3 = (kGenTag << 24) | idx;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return ((uint64_t)c1 << 32) | c0;
}

// smallest k in [lo, hi] with pre[k+1] > x (the answer is known to lie in the range)
__device__ __forceinline__ int64_t search(const uint64_t* __restrict__ pre, int64_t lo, int64_t hi, uint64_t x) {
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(pre + mid + 1) > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// guide[k] = invcdf(min(k << shift, total-1)), k in [0, 2^bits]
__global__ void guide_kernel(const uint64_t* __restrict__ pre, int64_t n, int bits, int shift, int32_t* guide) {
    const uint64_t total = pre[n];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= ((int64_t)1 << bits);
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t x = (uint64_t)k << shift;
        if (x >= total) x = total - 1;
        guide[k] = (int32_t)search(pre, 0, n - 1, x);
    }
}

__device__ __forceinline__ int64_t invcdf_g(const uint64_t* pre, const int32_t* guide, int shift, uint64_t x) {
    const uint64_t k = x >> shift;
    return search(pre, __ldg(guide + k), __ldg(guide + k + 1), x);
}

__global__ void iid_kernel(uint64_t seed, const uint64_t* __restrict__ pre, int64_t V, const int32_t* __restrict__ guide,
                           int shift, int64_t i0, int64_t n, int32_t* __restrict__ out) {
    const uint64_t Z = pre[V];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = __umul64hi(gen_u64(seed, (uint64_t)(i0 + k), 0u), Z);
        out[k] = (int32_t)invcdf_g(pre, guide, shift, x);
    }
}

__global__ void planted_kernel(uint64_t seed, int64_t V, int64_t C, int64_t Lg, const uint64_t* __restrict__ cl_pre,
                               const uint64_t* __restrict__ mem_pre, const int64_t* __restrict__ off, int64_t i0,
                               int64_t n, int32_t* __restrict__ out) {
    const uint64_t Zc = cl_pre[C];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + k, s = i / Lg;
        const int64_t c = search(cl_pre, 0, C - 1, __umul64hi(gen_u64(seed, (uint64_t)s, 1u), Zc));
        const int64_t M = (V - 1 - c) / C + 1;
        const uint64_t* mp = mem_pre + __ldg(off + c);
        const int64_t m = search(mp, 0, M - 1, __umul64hi(gen_u64(seed, (uint64_t)i, 0u), __ldg(mp + M)));
        out[k] = (int32_t)(c + m * C);
    }
}

int grid_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t b = (n + 255) / 256;
    const int64_t cap = (int64_t)sms * 16;
    return (int)(b < 1 ? 1 : b > cap ? cap : b);
}

}  // namespace

extern "C" {

/* Guide table for an iid prefix pre[0..V] (device): bits chosen by the caller, guide int32[2^bits+1]. */
int gen_cuda_guide(const uint64_t* pre, int64_t V, int bits, int shift, int32_t* guide, void* stream) {
    guide_kernel<<<grid_for(((int64_t)1 << bits) + 1), 256, 0, (cudaStream_t)stream>>>(pre, V, bits, shift, guide);
    return (int)cudaGetLastError();
}

/* tokens i0 .. i0+n-1 of the iid Zipf corpus into out (device) */
int gen_cuda_iid(uint64_t seed, const uint64_t* pre, int64_t V, const int32_t* guide, int shift, int64_t i0, int64_t n,
                 int32_t* out, void* stream) {
    if (n <= 0) return 0;
    iid_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(seed, pre, V, guide, shift, i0, n, out);
    return (int)cudaGetLastError();
}

/* tokens i0 .. i0+n-1 of the planted-cluster corpus into out (device) */
int gen_cuda_planted(uint64_t seed, int64_t V, int64_t C, int64_t Lg, const uint64_t* cl_pre, const uint64_t* mem_pre,
                     const int64_t* off, int64_t i0, int64_t n, int32_t* out, void* stream) {
    if (n <= 0) return 0;
    planted_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(seed, V, C, Lg, cl_pre, mem_pre, off, i0, n, out);
    return (int)cudaGetLastError();
}

}  // extern "C"
