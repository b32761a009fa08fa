// sync.cu — C15: the element-wise halves of the overlapped model average (a9,
// SURVEY.md §8(f) NEXT-2). After interval k the rows due are snapshot (C = M) and averaged by an
// OUT-OF-PLACE NCCL all-reduce (C -> S) on the comm stream while interval k+1 trains; after
// interval k+1 the replica applies the average's correction M += S - C. Both passes are HBM-bound streams over the
// contiguous row range of the interleaved model (float4, grid-stride, sized to the SM count).
#include "w2v_internal.h"

namespace w2v {

namespace {

__global__ void apply_kernel(float4* __restrict__ M, const float4* __restrict__ S, const float4* __restrict__ C,
                             size_t n4) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 m = M[i];
        const float4 s = S[i], c = C[i];
        m.x = __fadd_rn(m.x, __fsub_rn(s.x, c.x));
        m.y = __fadd_rn(m.y, __fsub_rn(s.y, c.y));
        m.z = __fadd_rn(m.z, __fsub_rn(s.z, c.z));
        m.w = __fadd_rn(m.w, __fsub_rn(s.w, c.w));
        M[i] = m;
    }
}

__global__ void snap_kernel(const float4* __restrict__ M, float4* __restrict__ C, size_t n4) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        C[i] = M[i];
}

int grid(size_t n4, int sms) {
    size_t b = (n4 + 255) / 256;
    const size_t cap = (size_t)sms * 8;
    return (int)(b < 1 ? 1 : b > cap ? cap : b);
}

}  // namespace

// M[i] += S[i] - C[i] over n floats (n % 4 == 0, 16-B aligned)
cudaError_t launch_sync_apply(float* M, const float* S, const float* C, size_t n, int sms, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    apply_kernel<<<grid(n / 4, sms), 256, 0, st>>>(reinterpret_cast<float4*>(M), reinterpret_cast<const float4*>(S),
                                                   reinterpret_cast<const float4*>(C), n / 4);
    return cudaGetLastError();
}

// C[i] = M[i] over n floats
cudaError_t launch_sync_snap(const float* M, float* C, size_t n, int sms, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    snap_kernel<<<grid(n / 4, sms), 256, 0, st>>>(reinterpret_cast<const float4*>(M), reinterpret_cast<float4*>(C),
                                                  n / 4);
    return cudaGetLastError();
}

}  // namespace w2v
