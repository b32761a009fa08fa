// tools/l2cap.cu — L2 slice (LTS) throughput cap on this GPU: all SMs stream an L2-resident
// working set (32 MB) with 16-B L2-only loads, then with 16-B fp32 vector reductions, then with
// the bulk copy / bulk reduce engine (the step kernel's path). Prints bytes/s per pattern from
// CUDA events; run under `ncu --metrics lts__t_sectors.sum,lts__cycles_elapsed.avg` for B/cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2cap tools/l2cap.cu && ./l2cap
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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
            asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "f"(1e-9f), "f"(1e-9f),
                         "f"(1e-9f), "f"(1e-9f) : "memory");
}

// one warp per 1200-B "row": bulk copy global->smem then bulk reduce smem->global (the step's path)
__global__ void bulk_kernel(float* p, size_t rows, int reps) {
    __shared__ __align__(128) float buf[8][320];
    __shared__ __align__(8) uint64_t bar[8];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&buf[w][0]);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[w]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    uint32_t phase = 0;
    const size_t nw = (size_t)gridDim.x * 8;
    for (int r = 0; r < reps; ++r)
        for (size_t row = (size_t)blockIdx.x * 8 + w; row < rows; row += nw) {
            if (lane == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 1200;" ::"r"(mb));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1200, [%2];"
                             ::"r"(sb), "l"(p + row * 320), "r"(mb) : "memory");
                asm volatile("{\n .reg .pred q;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W;\n}"
                             ::"r"(mb), "r"(phase) : "memory");
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 1200;"
                             ::"l"(p + row * 320), "r"(sb) : "memory");
                asm volatile("cp.async.bulk.commit_group;");
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            }
            phase ^= 1u;
            __syncwarp();
        }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = 32u << 20, n4 = bytes / 16, rows = bytes / 1280;
    float* p;
    float* out;
    cudaMalloc(&p, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(p, 0, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 200;
    float ms;
    for (int pass = 0; pass < 2; ++pass) {  // pass 0 warms up
        cudaEventRecord(a);
        rd_kernel<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(p), n4, reps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (pass) printf("ld.cg.v4 reads        : %.2f TB/s\n", bytes * (double)reps / (ms * 1e-3) / 1e12);
        cudaEventRecord(a);
        red_kernel<<<sms * 8, 256>>>(reinterpret_cast<float4*>(p), n4, reps / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (pass) printf("red.add.v4 reductions : %.2f TB/s\n", bytes * (double)(reps / 4) / (ms * 1e-3) / 1e12);
        cudaEventRecord(a);
        bulk_kernel<<<sms * 8, 256>>>(p, rows, reps / 8);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (pass)
            printf("bulk gather+reduce    : %.2f TB/s (1200-B rows, both directions)\n",
                   rows * 2400.0 * (reps / 8) / (ms * 1e-3) / 1e12);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
