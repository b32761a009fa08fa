// NVLS / multimem capability probe for one B200 (not part of the library).
//   1. CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED;
//   2. a 1-device multicast object (driver VMM API) bound to local memory, and a
//      multimem.ld_reduce / multimem.st kernel through its multicast address;
//   3. NCCL's symmetric-window device API on a 1-rank communicator (ncclMemAlloc,
//      ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC), ncclDevCommCreate with lsaMultimem).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -I<nccl>/include tools/nvls_probe.cu
//        -L<nccl>/lib -l:libnccl.so.2 -lcuda -o tools/nvls_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <cstdio>
#include <cstring>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s = nullptr; cuGetErrorString(r_, &s); \
    printf("  %s -> %d %s\n", #x, (int)r_, s ? s : "?"); return 1; } } while (0)
#define NK(x) do { ncclResult_t r_ = (x); if (r_ != ncclSuccess) { printf("  %s -> %s\n", #x, ncclGetErrorString(r_)); \
    return 1; } } while (0)

__global__ void mm_avg(float* mc, size_t n4, float scale) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float a, b, c, d;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + 4 * i) : "memory");
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                     :: "l"(mc + 4 * i), "f"(a * scale), "f"(b * scale), "f"(c * scale), "f"(d * scale) : "memory");
    }
}

__global__ void nccl_avg(ncclWindow_t win, ncclDevComm dc, size_t n4, float scale) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, true);
    bar.sync(ncclCoopCta(), cuda::memory_order_relaxed);
    float* mc = (float*)ncclGetLsaMultimemPointer(win, 0, dc);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float a, b, c, d;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + 4 * i) : "memory");
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                     :: "l"(mc + 4 * i), "f"(a * scale), "f"(b * scale), "f"(c * scale), "f"(d * scale) : "memory");
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_release);
}

static int probe_driver() {
    CK(cuInit(0));
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
    int mc = 0; CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    int fab = 0; cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    printf("multicast_supported=%d fabric_handle_supported=%d\n", mc, fab);
    if (!mc) return 1;
    size_t n = (size_t)64 << 20;  // floats
    CUmulticastObjectProp mp; memset(&mp, 0, sizeof mp);
    mp.numDevices = 1; mp.size = n * 4; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    size_t mgran = 0; CK(cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
    printf("mc granularity recommended=%zu minimum=%zu\n", gran, mgran);
    mp.size = (mp.size + mgran - 1) / mgran * mgran;
    CUmemGenericAllocationHandle mch;
    CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE,
                                        CU_MEM_HANDLE_TYPE_FABRIC};
    CUresult cr = CUDA_ERROR_INVALID_VALUE;
    for (int t = 0; t < 3 && cr != CUDA_SUCCESS; ++t) {
        mp.handleTypes = hts[t];
        cr = cuMulticastCreate(&mch, &mp);
        printf("cuMulticastCreate(numDevices 1, handleTypes %d, size %zu) -> %d\n", (int)hts[t], mp.size, (int)cr);
    }
    if (cr != CUDA_SUCCESS) {
        mp.numDevices = 2; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        cr = cuMulticastCreate(&mch, &mp);
        printf("cuMulticastCreate(numDevices 2) -> %d (create only; one device present, not used)\n", (int)cr);
        if (cr == CUDA_SUCCESS) printf("  addDevice -> %d\n", (int)cuMulticastAddDevice(mch, dev));
        return 1;
    }
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap; memset(&ap, 0, sizeof ap);
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = dev;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
    CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, mp.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, ph, 0, mp.size, 0));
    CUdeviceptr uc, mcp;
    CUmemAccessDesc acc; memset(&acc, 0, sizeof acc);
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = dev; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    gran = mgran;
    CK(cuMemAddressReserve(&uc, mp.size, gran, 0, 0)); CK(cuMemMap(uc, mp.size, 0, ph, 0));
    CK(cuMemSetAccess(uc, mp.size, &acc, 1));
    CK(cuMemAddressReserve(&mcp, mp.size, gran, 0, 0)); CK(cuMemMap(mcp, mp.size, 0, mch, 0));
    CK(cuMemSetAccess(mcp, mp.size, &acc, 1));
    float* h = new float[n];
    for (size_t i = 0; i < n; ++i) h[i] = (float)(i % 1000) * 0.5f;
    cudaMemcpy((void*)uc, h, n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    mm_avg<<<148 * 4, 512>>>((float*)mcp, n / 4, 0.5f);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) mm_avg<<<148 * 4, 512>>>((float*)mcp, n / 4, 1.0f);
    cudaEventRecord(e1);
    cudaError_t ce = cudaDeviceSynchronize();
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    printf("multimem kernel: %s, %.3f ms per %zu MB pass (%.1f GB/s read+write)\n", cudaGetErrorString(ce), ms / 10,
           n * 4 >> 20, 2.0 * n * 4 / (ms / 10 * 1e6));
    float* g = new float[n];
    cudaMemcpy(g, (void*)uc, n * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < n; ++i) bad += g[i] != h[i] * 0.5f;
    printf("multimem 1-device avg check: %zu mismatches of %zu\n", bad, n);
    return 0;
}

static int probe_nccl() {
    cudaSetDevice(0);
    ncclUniqueId id; NK(ncclGetUniqueId(&id));
    ncclComm_t comm; NK(ncclCommInitRank(&comm, 1, id, 0));
    size_t n = (size_t)16 << 20;
    void* buf = nullptr; NK(ncclMemAlloc(&buf, n * 4));
    ncclWindow_t win; NK(ncclCommWindowRegister(comm, buf, n * 4, &win, NCCL_WIN_COLL_SYMMETRIC));
    printf("nccl window registered\n");
    ncclDevCommRequirements req; memset(&req, 0, sizeof req);
    req.lsaMultimem = true; req.lsaBarrierCount = 148;
    ncclDevComm dc;
    ncclResult_t r = ncclDevCommCreate(comm, &req, &dc);
    printf("ncclDevCommCreate(lsaMultimem) -> %s (lsaSize %d, mcBase %p)\n", ncclGetErrorString(r),
           r == ncclSuccess ? dc.lsaSize : -1, r == ncclSuccess ? dc.lsaMultimem.mcBasePtr : nullptr);
    if (r != ncclSuccess || !dc.lsaMultimem.mcBasePtr) {
        req.lsaMultimem = false;
        r = ncclDevCommCreate(comm, &req, &dc);
        printf("ncclDevCommCreate(no multimem) -> %s\n", ncclGetErrorString(r));
        return 0;
    }
    cudaMemset(buf, 0, n * 4);
    nccl_avg<<<148, 512>>>(win, dc, n / 4, 1.0f);
    printf("nccl multimem kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

int main() {
    int a = probe_driver();
    printf("driver probe rc %d\n", a);
    int b = probe_nccl();
    printf("nccl probe rc %d\n", b);
    return 0;
}
