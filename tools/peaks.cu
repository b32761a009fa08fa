// tools/peaks.cu — in-run roofline denominators for bench.py (measurement only, not the product
// path): libw2v_peaks.so, C-ABI, built by __graft_entry__.build().
//
//  peaks_l2_rowpath  the L2 ceiling of the step kernel's own access pattern: every
//                    warp of a persistent grid repeatedly bulk-copies a batch of R rows of
//                    `row_bytes` into shared memory (cp.async.bulk + mbarrier), waits, then
//                    bulk-reduces them back (cp.reduce.async.bulk .add.f32) and waits — row ids
//                    hashed over an L2-resident working set (32 MB), so DRAM is not involved.
//                    Returns row bytes moved (gathered + reduced) per second.
//  peaks_ffma2       fp32 FMA-pipe peak: independent FFMA2 (fma.rn.f32x2) chains, all SMs.
//                    Returns FLOP/s (2 per fma, 2 fma per FFMA2).
//  peaks_l2_read / peaks_l2_red   pure ld.global.cg.v4 reads / pure red.global.add.v4.f32 over the
//                    same working set (the two sides of the mixed cap).
// Times are CUDA events around the second of two identical launches (the first warms L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared -o tools/libw2v_peaks.so tools/peaks.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// one warp = one unit: batches of R rows gathered then reduced, like one target of the step
__global__ void rowpath_kernel(float* base, uint32_t nrows, uint32_t row_floats, uint32_t row_bytes, int R,
                               int batches, int warp_bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wb = smem + (size_t)w * warp_bytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(wb);
    float* rows = reinterpret_cast<float*>(wb + 128);
    const uint32_t mb = smem_u32(bar);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + w;
    uint32_t phase = 0;
    for (int it = 0; it < batches; ++it) {
        const uint32_t key = hash32(gw * 7919u + (uint32_t)it * 104729u);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(row_bytes * (uint32_t)R));
        __syncwarp();
        uint32_t id = 0;
        if (lane < R) {
            id = hash32(key + lane) % nrows;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(rows + (size_t)lane * row_floats)),
                "l"(base + (size_t)id * row_floats), "r"(row_bytes), "r"(mb)
                : "memory");
        }
        asm volatile(
            "{\n .reg .pred q;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W_%=;\n}" ::"r"(mb),
            "r"(phase)
            : "memory");
        phase ^= 1u;
        if (lane < R)
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                             base + (size_t)id * row_floats),
                         "r"(smem_u32(rows + (size_t)lane * row_floats)), "r"(row_bytes)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
}

__global__ void ffma2_kernel(float* out, int iters) {
    float2 a[8], b = make_float2(1.0000001f, 0.9999999f), c = make_float2(1e-7f, -1e-7f);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = make_float2((float)threadIdx.x * 1e-3f + i, (float)i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            unsigned long long d;
            asm volatile("fma.rn.f32x2 %0, %1, %2, %3;"
                         : "=l"(d)
                         : "l"(*reinterpret_cast<unsigned long long*>(&a[i])),
                           "l"(*reinterpret_cast<unsigned long long*>(&b)),
                           "l"(*reinterpret_cast<unsigned long long*>(&c)));
            a[i] = *reinterpret_cast<float2*>(&d);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
    if (s == 1234.5f) out[0] = s;
}

__global__ void rd_kernel(const float4* __restrict__ p, size_t n4, int reps, float* out) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
            float4 v;
            asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p + i));
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 1234.5f) out[0] = acc;
}

__global__ void red_kernel(float4* p, size_t n4, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
            asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "f"(0.f), "f"(0.f),
                         "f"(0.f), "f"(0.f)
                         : "memory");
}

struct Timer {
    cudaEvent_t a, b;
    Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
    ~Timer() { cudaEventDestroy(a); cudaEventDestroy(b); }
};

int sm_count() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

constexpr size_t kWorkingSet = 32u << 20;  // L2-resident (126 MB L2)

}  // namespace

extern "C" {

// row_bytes % 16 == 0; R rows per batch (<= 32); warps_per_sm resident 1-warp... units per SM.
// Returns 0 and *gbs = (gathered + reduced row bytes) / s, or a CUDA error code.
int peaks_l2_rowpath(int row_bytes, int R, int warps_per_sm, double* gbs) {
    if (row_bytes <= 0 || row_bytes % 16 || R < 1 || R > 32 || warps_per_sm < 1) return -1;
    const int sms = sm_count();
    const uint32_t row_floats = (uint32_t)((row_bytes + 127) / 128 * 32);   // 128-B row stride
    const uint32_t nrows = (uint32_t)(kWorkingSet / (row_floats * 4));
    float* base = nullptr;
    if (cudaMalloc(&base, kWorkingSet) != cudaSuccess) return (int)cudaGetLastError();
    cudaMemset(base, 0, kWorkingSet);
    const int warp_bytes = 128 + R * (int)row_floats * 4;
    int wpc = warps_per_sm, cpsm = 1;           // CTAs of up to 8 warps
    while (wpc > 8) { wpc = (wpc + 1) / 2; cpsm *= 2; }
    const int smem = wpc * warp_bytes;
    cudaFuncSetAttribute(rowpath_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int batches = 2000;
    Timer t;
    float ms = 0.f;
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(t.a);
        rowpath_kernel<<<sms * cpsm, 32 * wpc, smem>>>(base, nrows, row_floats, (uint32_t)row_bytes, R, batches,
                                                       warp_bytes);
        cudaEventRecord(t.b);
        cudaEventSynchronize(t.b);
        cudaEventElapsedTime(&ms, t.a, t.b);
    }
    const cudaError_t e = cudaGetLastError();
    cudaFree(base);
    if (e != cudaSuccess) return (int)e;
    *gbs = (double)sms * cpsm * wpc * batches * R * row_bytes * 2.0 / (ms * 1e-3) / 1e9;
    return 0;
}

int peaks_ffma2(double* tflops) {
    const int sms = sm_count();
    float* out = nullptr;
    cudaMalloc(&out, 4);
    const int iters = 1 << 16, blocks = sms * 8, threads = 256;
    Timer t;
    float ms = 0.f;
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(t.a);
        ffma2_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(t.b);
        cudaEventSynchronize(t.b);
        cudaEventElapsedTime(&ms, t.a, t.b);
    }
    const cudaError_t e = cudaGetLastError();
    cudaFree(out);
    if (e != cudaSuccess) return (int)e;
    *tflops = (double)blocks * threads * iters * 8 * 2 * 2 / (ms * 1e-3) / 1e12;   // 8 FFMA2 x 2 fma x 2 flop
    return 0;
}

int peaks_l2_read(double* gbs) {
    const int sms = sm_count();
    float *p = nullptr, *out = nullptr;
    if (cudaMalloc(&p, kWorkingSet) != cudaSuccess) return (int)cudaGetLastError();
    cudaMalloc(&out, 4);
    cudaMemset(p, 0, kWorkingSet);
    const int reps = 100;
    Timer t;
    float ms = 0.f;
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(t.a);
        rd_kernel<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(p), kWorkingSet / 16, reps, out);
        cudaEventRecord(t.b);
        cudaEventSynchronize(t.b);
        cudaEventElapsedTime(&ms, t.a, t.b);
    }
    const cudaError_t e = cudaGetLastError();
    cudaFree(p); cudaFree(out);
    if (e != cudaSuccess) return (int)e;
    *gbs = (double)kWorkingSet * reps / (ms * 1e-3) / 1e9;
    return 0;
}

int peaks_l2_red(double* gbs) {
    const int sms = sm_count();
    float* p = nullptr;
    if (cudaMalloc(&p, kWorkingSet) != cudaSuccess) return (int)cudaGetLastError();
    cudaMemset(p, 0, kWorkingSet);
    const int reps = 25;
    Timer t;
    float ms = 0.f;
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(t.a);
        red_kernel<<<sms * 8, 256>>>(reinterpret_cast<float4*>(p), kWorkingSet / 16, reps);
        cudaEventRecord(t.b);
        cudaEventSynchronize(t.b);
        cudaEventElapsedTime(&ms, t.a, t.b);
    }
    const cudaError_t e = cudaGetLastError();
    cudaFree(p);
    if (e != cudaSuccess) return (int)e;
    *gbs = (double)kWorkingSet * reps / (ms * 1e-3) / 1e9;
    return 0;
}

}  // extern "C"
