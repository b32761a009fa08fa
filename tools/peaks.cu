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
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// one warp = one unit: batches of R rows gathered then reduced, like one target of the step
// (rows [0, n_store) of a batch are written back by a plain bulk store instead of the reduction)
__global__ void rowpath_kernel(float* base, uint32_t nrows, uint32_t row_floats, uint32_t row_bytes, int R,
                               int batches, int warp_bytes, int n_store, unsigned long long* clk) {
    if (clk && blockIdx.x == 0 && threadIdx.x == 0) clk[0] = clock64();   // SM cycles over the run
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
        if (lane < R && lane >= n_store)
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                             base + (size_t)id * row_floats),
                         "r"(smem_u32(rows + (size_t)lane * row_floats)), "r"(row_bytes)
                         : "memory");
        if (lane < R && lane < n_store)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                             base + (size_t)id * row_floats),
                         "r"(smem_u32(rows + (size_t)lane * row_floats)), "r"(row_bytes)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    if (clk && blockIdx.x == 0 && threadIdx.x == 0) clk[1] = clock64();
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

// ---- gather-engine comparison (SURVEY.md §8(a) "Gather engines"): every warp
// gathers R rows of `row_bytes` (random rows of an L2-resident working set) into shared memory
// with one of four engines, then (reduce = 1) bulk-reduces them back, like one target of the
// step kernel. Engine 0: one cp.async.bulk per row (the step kernel's); 1: LSU ld.global.cg.v4 +
// st.shared; 2: cp.async.cg 16-B (LDGSTS); 3: TMA cp.async.bulk.tensor tile::gather4 (4 rows per
// instruction, box of 100 fp32 columns: 3 instructions per 4 rows of 300 floats).
template <int ENGINE>
__global__ void engine_kernel(float* base, uint32_t nrows, uint32_t row_floats, uint32_t row_bytes, int R, int batches,
                              int warp_bytes, int reduce, const __grid_constant__ CUtensorMap tmap, int* bad) {
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
    const uint32_t rf = row_bytes / 4, n16 = row_bytes / 16;
    uint32_t phase = 0;
    for (int it = 0; it < batches; ++it) {
        const uint32_t key = hash32(gw * 7919u + (uint32_t)it * 104729u);
        const uint32_t my_id = hash32(key + lane) % nrows;   // lane r < R: row r of this batch
        if (ENGINE == 0 || ENGINE == 3) {
            const uint32_t nrow_tx = ENGINE == 3 ? (uint32_t)((R + 3) / 4) * 4u : (uint32_t)R;  // gather4: whole groups
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(row_bytes * nrow_tx));
            __syncwarp();
        }
        if (ENGINE == 0) {
            if (lane < R)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(rows + (size_t)lane * rf)),
                    "l"(base + (size_t)my_id * row_floats), "r"(row_bytes), "r"(mb)
                    : "memory");
        } else if (ENGINE == 1 || ENGINE == 2) {
            for (int r = 0; r < R; ++r) {
                const uint32_t id = __shfl_sync(0xffffffffu, my_id, r);
                const float4* src = reinterpret_cast<const float4*>(base + (size_t)id * row_floats);
                float4* dst = reinterpret_cast<float4*>(rows + (size_t)r * rf);
                for (uint32_t u = lane; u < n16; u += 32) {
                    if (ENGINE == 1) {
                        float4 v;
                        asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(src + u));
                        dst[u] = v;
                    } else {
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + u)), "l"(src + u) : "memory");
                    }
                }
            }
            if (ENGINE == 2) asm volatile("cp.async.wait_all;" ::: "memory");
        } else {  // ENGINE 3: groups of 4 rows, 100-column boxes; segment s of rows 4g..4g+3 is
                  // [4 rows][100 floats] at rows + g * 1248 + s * 416 floats (128-B aligned:
                  // TMA tensor destinations must be)
            const int groups = (R + 3) / 4;
            if (lane < groups * 3) {
                const int g = lane / 3, sgm = lane % 3;
                int32_t r4[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) r4[k] = 0;
                (void)r4;
                const uint32_t id0 = hash32(key + 4 * g + 0) % nrows, id1 = hash32(key + 4 * g + 1) % nrows;
                const uint32_t id2 = hash32(key + 4 * g + 2) % nrows, id3 = hash32(key + 4 * g + 3) % nrows;
                float* dst = rows + (size_t)g * 1248 + (size_t)sgm * 416;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                        smem_u32(dst)),
                    "l"(&tmap), "r"(100 * sgm), "r"((int)id0), "r"((int)id1), "r"((int)id2), "r"((int)id3), "r"(mb)
                    : "memory");
            }
        }
        if (ENGINE == 0 || ENGINE == 3) {
            asm volatile(
                "{\n .reg .pred q;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W_%=;\n}" ::"r"(mb),
                "r"(phase)
                : "memory");
            phase ^= 1u;
        }
        __syncwarp();
        if (it == 0 && bad) {  // data check of the first batch (the base holds id*1e-3 in every float)
            for (int r = 0; r < R && ENGINE != 3; ++r) {
                const uint32_t id = __shfl_sync(0xffffffffu, my_id, r);
                for (uint32_t u = lane; u < rf; u += 32)
                    if (rows[(size_t)r * rf + u] != base[(size_t)id * row_floats + u]) atomicAdd(bad, 1);
            }
            if (ENGINE == 3)
                for (int g = 0; g < (R + 3) / 4; ++g)
                    for (int k = 0; k < 4 && 4 * g + k < R; ++k) {
                        const uint32_t id = hash32(key + 4 * g + k) % nrows;
                        for (int sgm = 0; sgm < 3; ++sgm)
                            for (uint32_t u = lane; u < 100; u += 32)
                                if (rows[(size_t)g * 1248 + sgm * 416 + k * 100 + u] != base[(size_t)id * row_floats + 100 * sgm + u])
                                    atomicAdd(bad, 1);
                    }
            __syncwarp();
        }
        if (reduce) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane < R)
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                                 base + (size_t)my_id * row_floats),
                             "r"(smem_u32(rows + (size_t)lane * rf)), "r"(row_bytes)
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
        __syncwarp();
    }
}

__global__ void fill_kernel(float* p, size_t n, uint32_t row_floats) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (float)(i / row_floats) * 1e-3f;
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
int peaks_l2_rowpath_clk(int row_bytes, int R, int warps_per_sm, int n_store, double* gbs, double* mhz);
int peaks_l2_rowpath_store(int row_bytes, int R, int warps_per_sm, int n_store, double* gbs) {
    return peaks_l2_rowpath_clk(row_bytes, R, warps_per_sm, n_store, gbs, nullptr);
}
int peaks_l2_rowpath(int row_bytes, int R, int warps_per_sm, double* gbs) {
    return peaks_l2_rowpath_clk(row_bytes, R, warps_per_sm, 0, gbs, nullptr);
}

// the same with the first n_store rows of every batch written back by a plain bulk store
// (cp.async.bulk.global.shared::cta) instead of the fp32 reduce-add; *mhz (if given) = the SM
// clock the timed run ran at (block 0's clock64 span over the launch's CUDA-event time)
int peaks_l2_rowpath_clk(int row_bytes, int R, int warps_per_sm, int n_store, double* gbs, double* mhz) {
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
    const char* nb = getenv("W2V_CAP_BATCHES");
    const int batches = nb ? atoi(nb) : 2000;
    unsigned long long* clk = nullptr;
    cudaMalloc(&clk, 16);
    Timer t;
    float ms = 0.f;
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(t.a);
        rowpath_kernel<<<sms * cpsm, 32 * wpc, smem>>>(base, nrows, row_floats, (uint32_t)row_bytes, R, batches,
                                                       warp_bytes, n_store, clk);
        cudaEventRecord(t.b);
        cudaEventSynchronize(t.b);
        cudaEventElapsedTime(&ms, t.a, t.b);
    }
    unsigned long long hc[2] = {0, 0};
    cudaMemcpy(hc, clk, 16, cudaMemcpyDeviceToHost);
    cudaFree(clk);
    const cudaError_t e = cudaGetLastError();
    cudaFree(base);
    if (e != cudaSuccess) return (int)e;
    *gbs = (double)sms * cpsm * wpc * batches * R * row_bytes * 2.0 / (ms * 1e-3) / 1e9;
    if (mhz) *mhz = hc[1] > hc[0] ? (double)(hc[1] - hc[0]) / (ms * 1e3) : 0.0;
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

// Gather-engine comparison: out[e] = gathered row bytes per second for engine e in 0..3, out[4+e]
// = gathered + reduced row bytes per second; bad[e] = mismatching floats in the first batch's data check (-1: the
// engine could not run, e.g. the tensor map was rejected). 300-float rows (D = 300), 320-float
// stride, R rows per batch, warps_per_sm units.
int peaks_gather_engines(int R, int warps_per_sm, double* out, int* bad) {
    const int sms = sm_count();
    const uint32_t row_floats = 320, row_bytes = 1200;
    const uint32_t nrows = (uint32_t)(kWorkingSet / (row_floats * 4));
    float* base = nullptr;
    int* dbad = nullptr;
    if (cudaMalloc(&base, kWorkingSet) != cudaSuccess) return (int)cudaGetLastError();
    cudaMalloc(&dbad, 4 * sizeof(int));
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof tmap);
    bool tmap_ok = false;
    {   // 2-D fp32 tensor [nrows][320], box 100 columns x 1 row (gather4 supplies 4 row coordinates)
        typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess && fn) {
            const cuuint64_t dims[2] = {row_floats, nrows}, strides[1] = {row_floats * 4};
            const cuuint32_t box[2] = {100, 1}, es[2] = {1, 1};
            tmap_ok = ((Encode)fn)(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        cudaGetLastError();
    }
    const int warp_bytes = 128 + ((R + 3) / 4) * 1248 * 4;  // >= R rows of 320 floats; gather4 groups
    int wpc = warps_per_sm, cpsm = 1;
    while (wpc > 8) { wpc = (wpc + 1) / 2; cpsm *= 2; }
    const int smem = wpc * warp_bytes;
    const int batches = 1000;
    Timer t;
    for (int e = 0; e < 4; ++e) {  // engine 3 last: a rejected tensor copy leaves a sticky error
        out[e] = out[4 + e] = 0.0;
        bad[e] = -1;
        if (e == 3 && !tmap_ok) continue;
        fill_kernel<<<sms * 4, 256>>>(base, kWorkingSet / 4, row_floats);
        cudaMemset(dbad, 0, 4 * sizeof(int));
        float ms = 0.f;
        int reduce = 0;
        auto run = [&](int chk) {
            switch (e) {
            case 0: cudaFuncSetAttribute(engine_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                engine_kernel<0><<<sms * cpsm, 32 * wpc, smem>>>(base, nrows, row_floats, row_bytes, R, chk ? 1 : batches, warp_bytes, chk ? 0 : reduce, tmap, chk ? dbad + e : nullptr); break;
            case 1: cudaFuncSetAttribute(engine_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                engine_kernel<1><<<sms * cpsm, 32 * wpc, smem>>>(base, nrows, row_floats, row_bytes, R, chk ? 1 : batches, warp_bytes, chk ? 0 : reduce, tmap, chk ? dbad + e : nullptr); break;
            case 2: cudaFuncSetAttribute(engine_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                engine_kernel<2><<<sms * cpsm, 32 * wpc, smem>>>(base, nrows, row_floats, row_bytes, R, chk ? 1 : batches, warp_bytes, chk ? 0 : reduce, tmap, chk ? dbad + e : nullptr); break;
            default: cudaFuncSetAttribute(engine_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                engine_kernel<3><<<sms * cpsm, 32 * wpc, smem>>>(base, nrows, row_floats, row_bytes, R, chk ? 1 : batches, warp_bytes, chk ? 0 : reduce, tmap, chk ? dbad + e : nullptr); break;
            }
        };
        run(1);  // data check on the unmodified fill (no reduction)
        if (cudaDeviceSynchronize() != cudaSuccess) { cudaGetLastError(); continue; }
        cudaMemcpy(&bad[e], dbad + e, sizeof(int), cudaMemcpyDeviceToHost);
        for (reduce = 0; reduce < 2; ++reduce) {   // out[e]: gather only; out[4 + e]: + bulk reduce
            for (int pass = 0; pass < 2; ++pass) {
                cudaEventRecord(t.a);
                run(0);
                cudaEventRecord(t.b);
                cudaEventSynchronize(t.b);
                cudaEventElapsedTime(&ms, t.a, t.b);
            }
            if (cudaGetLastError() != cudaSuccess) { bad[e] = -1; break; }
            out[4 * reduce + e] = (double)sms * cpsm * wpc * batches * R * row_bytes * (reduce ? 2.0 : 1.0) / (ms * 1e-3) / 1e9;
        }
    }
    cudaFree(base);
    cudaFree(dbad);
    return 0;
}

}  // extern "C"
