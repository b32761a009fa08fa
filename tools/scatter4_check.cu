// Does cp.reduce.async.bulk.tensor ... .add.tile::scatter4 add (or store)? ptxas 12.9 prints its
// SASS as UTMASTG.2D.SCATTER4 (the plain store's opcode), unlike tile mode's UTMAREDG.2D.ADD.
// Rows of a [16][128] fp32 tensor hold 1.0; rows 1, 3, 3, 8 receive a reduce-scatter4 of 4 rows
// of 2.0 (row 3 twice). A true reduction leaves 3, 5, 3 in rows 1, 3, 8; a store leaves 2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/scatter4_check tools/scatter4_check.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>

__global__ void k(const __grid_constant__ CUtensorMap tmap, int mode) {
    __shared__ __align__(128) float s[4 * 128];
    for (int i = threadIdx.x; i < 4 * 128; i += blockDim.x) s[i] = 2.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(s);
        if (mode == 0)
            asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                         :: "l"(&tmap), "r"(0), "r"(1), "r"(3), "r"(3), "r"(8), "r"(sa) : "memory");
        else
            for (int r : {1, 3, 3, 8})
                asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
                             :: "l"(&tmap), "r"(0), "r"(r), "r"(sa) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    float* d = nullptr;
    cudaMalloc(&d, 16 * 128 * 4);
    typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    for (int mode = 0; mode < 2; ++mode) {
        float h[16 * 128];
        for (int i = 0; i < 16 * 128; ++i) h[i] = 1.0f;
        cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
        CUtensorMap tm;
        std::memset(&tm, 0, sizeof tm);
        const cuuint64_t dims[2] = {128, 16}, strides[1] = {128 * 4};
        const cuuint32_t box[2] = {128, 1}, es[2] = {1, 1};
        CUresult r = ((Encode)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        k<<<1, 128>>>(tm, mode);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        printf("%s: encode %d, kernel %s, rows 0/1/3/8 = %.1f %.1f %.1f %.1f (reduction: 1 3 5 3)\n",
               mode == 0 ? "reduce tile::scatter4" : "reduce tile x4 (reference)", (int)r, cudaGetErrorString(e), h[0],
               h[128], h[3 * 128], h[8 * 128]);
    }
    return 0;
}
