// sync_dev.cu — a9 as ONE device kernel over NCCL's symmetric memory (option "sync_device";
// SURVEY.md §8(f) NEXT-2, DESIGN.md §2 C17). PAPER.md:154-157 (§2.2): each node trains its own
// replica and "the model is synchronized across nodes periodically" — reading R13 / C13: rows
// [lo, hi) of the interleaved model [M_in | M_out] become their mean over the W replicas.
//
// The model lives in ncclMemAlloc memory registered as a symmetric window
// (NCCL_WIN_COLL_SYMMETRIC), so every replica is load/store-addressable from every GPU of the
// NVLink domain (NCCL's "LSA" team) and, on NVSwitch systems with multicast, through one
// multicast (NVLS) address. Each rank owns 1/W of the float range:
//   NVLS:  multimem.ld_reduce.add.v4.f32 returns the sum over the W replicas (the switch reduces),
//          one multimem.st writes sum * (1/W) into all W replicas (the switch fans out);
//   LSA:   (no multicast object) the slice is loaded from every peer in rank order, summed,
//          scaled by 1/W and stored into every peer.
// An LSA barrier opens the pass (every replica finished its interval) and closes it with release
// order (every store landed before any rank trains on). No host round trip, no staging copy,
// no second buffer: the in-place mean of C13/C14 in one launch on the training stream. With C15
// (sync_overlap) the same kernel runs OUT of place — snapshot window C -> average window S — on
// the comm stream with a small grid, concurrently with the next interval's training.
//
// Built against the NCCL 2.28 device headers of the nvidia-nccl wheel that torch loads (the
// ncclDevComm layout is version-specific: devsync_alloc checks the runtime's major.minor).
#include <nccl.h>
#include <nccl_device.h>
#include <dlfcn.h>
#include <cstdio>
#include <cstring>

#include "w2v_internal.h"

namespace w2v {

namespace {

struct NcclDev {
    bool ok = false;
    ncclResult_t (*getVersion)(int*) = nullptr;
    ncclResult_t (*memAlloc)(void**, size_t) = nullptr;
    ncclResult_t (*memFree)(void*) = nullptr;
    ncclResult_t (*winRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
    ncclResult_t (*winDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
    ncclResult_t (*devCommCreate)(ncclComm_t, ncclDevCommRequirements_t const*, ncclDevComm_t*) = nullptr;
    ncclResult_t (*devCommDestroy)(ncclComm_t, ncclDevComm_t const*) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
    bool load() {
        if (ok) return true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        getVersion = (decltype(getVersion))dlsym(h, "ncclGetVersion");
        memAlloc = (decltype(memAlloc))dlsym(h, "ncclMemAlloc");
        memFree = (decltype(memFree))dlsym(h, "ncclMemFree");
        winRegister = (decltype(winRegister))dlsym(h, "ncclCommWindowRegister");
        winDeregister = (decltype(winDeregister))dlsym(h, "ncclCommWindowDeregister");
        devCommCreate = (decltype(devCommCreate))dlsym(h, "ncclDevCommCreate");
        devCommDestroy = (decltype(devCommDestroy))dlsym(h, "ncclDevCommDestroy");
        errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
        ok = getVersion && memAlloc && memFree && winRegister && winDeregister && devCommCreate && devCommDestroy &&
             errStr;
        return ok;
    }
} g_dev;

// every CTA must be resident at once: CTA i of each rank meets CTA i of every peer in the LSA
// barrier, so a CTA left waiting for a slot could block a peer forever (2 x 512 threads per SM,
// <= 64 registers; kDevSyncCtas = 2 x 148)
constexpr int kThreads = 512;
constexpr int kUnroll = 4;  // float4 per thread per peer in flight

__device__ __forceinline__ float4 mm_ld_reduce4(const float4* p) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void mm_st4(float4* p, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float mm_ld_reduce1(const float* p) {
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void mm_st1(float* p, float v) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" :: "l"(p), "f"(v) : "memory");
}

__device__ __forceinline__ float4 scale4(float4 a, float s) {
    return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s), __fmul_rn(a.w, s));
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// floats [off, off+n) of the window: this rank's slice [s0, s1) = [off + n*r/W, off + n*(r+1)/W)
// (W = LSA team size, r = LSA rank); a scalar head up to 16-B alignment, a float4 body, a scalar tail.
// dst[off, off+n) := mean over the W replicas of src[off, off+n) (src == dst: in place)
template <bool MM>
__global__ void __launch_bounds__(kThreads, 2) avg_kernel(ncclWindow_t src, ncclWindow_t dst, ncclDevComm dc,
                                                       size_t off, size_t n, unsigned long long* counted) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, MM);
    bar.sync(ncclCoopCta(), cuda::memory_order_relaxed);  // every replica finished its interval

    const int W = dc.lsaSize, r = dc.lsaRank;
    const float inv = 1.0f / (float)W;
    size_t s0, a0, a1, s1;
    devsync_slice(off, n, r, W, &s0, &a0, &a1, &s1);
    const size_t T = (size_t)gridDim.x * kThreads, tid = (size_t)blockIdx.x * kThreads + threadIdx.x;
    uint32_t mine = 0;

    if constexpr (MM) {
        const float* ms = (const float*)ncclGetLsaMultimemPointer(src, 0, dc);
        float* md = (float*)ncclGetLsaMultimemPointer(dst, 0, dc);
        for (size_t i = s0 + tid; i < a0; i += T) { mm_st1(md + i, __fmul_rn(mm_ld_reduce1(ms + i), inv)); ++mine; }
        for (size_t i = a1 + tid; i < s1; i += T) { mm_st1(md + i, __fmul_rn(mm_ld_reduce1(ms + i), inv)); ++mine; }
        const float4* s4 = reinterpret_cast<const float4*>(ms);
        float4* d4 = reinterpret_cast<float4*>(md);
        const size_t v0 = a0 / 4, v1 = a1 / 4;
        for (size_t b = v0 + tid; b < v1; b += T * kUnroll) {
            float4 s[kUnroll];
#pragma unroll
            for (int k = 0; k < kUnroll; ++k)
                if (b + k * T < v1) s[k] = mm_ld_reduce4(s4 + b + k * T);
#pragma unroll
            for (int k = 0; k < kUnroll; ++k)
                if (b + k * T < v1) { mm_st4(d4 + b + k * T, scale4(s[k], inv)); mine += 4; }
        }
    } else {
        // rank-order sum of the peers' copies (the same order on every rank)
        auto one = [&](size_t i) {
            float s = __ldcg((const float*)ncclGetLsaPointer(src, 0, 0) + i);
            for (int p = 1; p < W; ++p) s = __fadd_rn(s, __ldcg((const float*)ncclGetLsaPointer(src, 0, p) + i));
            s = __fmul_rn(s, inv);
            for (int p = 0; p < W; ++p) __stcg((float*)ncclGetLsaPointer(dst, 0, p) + i, s);
            ++mine;
        };
        for (size_t i = s0 + tid; i < a0; i += T) one(i);
        for (size_t i = a1 + tid; i < s1; i += T) one(i);
        const size_t v0 = a0 / 4, v1 = a1 / 4;
        for (size_t b = v0 + tid; b < v1; b += T * kUnroll) {
            float4 s[kUnroll];
            const float4* p0 = (const float4*)ncclGetLsaPointer(src, 0, 0);
#pragma unroll
            for (int k = 0; k < kUnroll; ++k)
                if (b + k * T < v1) s[k] = __ldcg(p0 + b + k * T);
            for (int p = 1; p < W; ++p) {
                const float4* pp = (const float4*)ncclGetLsaPointer(src, 0, p);
                float4 x[kUnroll];
#pragma unroll
                for (int k = 0; k < kUnroll; ++k)
                    if (b + k * T < v1) x[k] = __ldcg(pp + b + k * T);
#pragma unroll
                for (int k = 0; k < kUnroll; ++k)
                    if (b + k * T < v1) s[k] = add4(s[k], x[k]);
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) s[k] = scale4(s[k], inv);
            for (int p = 0; p < W; ++p) {
                float4* pp = (float4*)ncclGetLsaPointer(dst, 0, p);
#pragma unroll
                for (int k = 0; k < kUnroll; ++k)
                    if (b + k * T < v1) __stcg(pp + b + k * T, s[k]);
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k)
                if (b + k * T < v1) mine += 4;
        }
    }
    // floats this rank averaged (stats; the test checks the slices tile the range exactly)
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(counted, (unsigned long long)mine);

    bar.sync(ncclCoopCta(), cuda::memory_order_release);  // every store landed before anyone trains on
}

void set_err(std::string* err, const char* what, ncclResult_t r) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s: %s", what, g_dev.errStr ? g_dev.errStr(r) : "?");
    *err = buf;
}

}  // namespace

int devsync_alloc(size_t bytes, void** buf, std::string* err) {
    if (!g_dev.load()) { *err = "sync_device: libnccl.so.2 lacks the symmetric-memory API (needs NCCL >= 2.28)"; return 1; }
    int v = 0;
    g_dev.getVersion(&v);
    if (v / 100 != NCCL_VERSION_CODE / 100) {
        char b[160];
        snprintf(b, sizeof b, "sync_device: runtime NCCL %d, built against %d (the device-communicator layout is "
                 "version-specific)", v, NCCL_VERSION_CODE);
        *err = b;
        return 1;
    }
    ncclResult_t r = g_dev.memAlloc(buf, bytes);
    if (r != ncclSuccess) { *buf = nullptr; set_err(err, "sync_device: ncclMemAlloc of the model", r); return 1; }
    return 0;
}

void devsync_free(void* buf) {
    if (buf && g_dev.ok) g_dev.memFree(buf);
}

// Collective over the communicator: register the model buffer as a symmetric window and create
// the device communicator (NVLS multicast if NCCL can give it, else LSA loads/stores).
// agree_min(v): the minimum of v over all ranks (a collective supplied by the caller), so that a
// multicast team that only some ranks could create is dropped on every rank (the fallback
// creation is collective too and must be called by all or none)
int devsync_open(ncclComm_t comm, void* const* bufs, const size_t* bytes, int nwin, int world, int want_mm,
                 int (*agree_min)(int), DevSync* ds, std::string* err) {
    // every window is registered BEFORE the device communicator is created (its multicast
    // mapping then covers them all)
    ncclWindow_t wins[kDevSyncMaxWin] = {};
    auto drop_wins = [&]() {
        for (int k = 0; k < nwin; ++k)
            if (wins[k]) g_dev.winDeregister(comm, wins[k]);
    };
    if (nwin < 1 || nwin > kDevSyncMaxWin) { *err = "sync_device: bad window count"; return 1; }
    ncclResult_t r = ncclSuccess;
    for (int k = 0; k < nwin; ++k) {
        r = g_dev.winRegister(comm, bufs[k], bytes[k], &wins[k], NCCL_WIN_COLL_SYMMETRIC);
        if (r != ncclSuccess) {
            wins[k] = nullptr;
            drop_wins();
            set_err(err, "sync_device: ncclCommWindowRegister", r);
            return 1;
        }
    }
    auto* dc = new ncclDevComm;
    ncclDevCommRequirements req;
    std::memset(&req, 0, sizeof req);
    req.lsaBarrierCount = kDevSyncCtas;
    int mm = 0;
    if (want_mm) {  // also at W = 1: exercises the failed-attempt fallback on one-GPU boxes
        req.lsaMultimem = true;
        const bool made = g_dev.devCommCreate(comm, &req, dc) == ncclSuccess;
        mm = made && dc->lsaMultimem.mcBasePtr != nullptr;
        const int all = agree_min(mm);
        if (all < 0) {
            if (made) g_dev.devCommDestroy(comm, dc);
            delete dc;
            drop_wins();
            *err = "sync_device: the multicast agreement collective failed";
            return 1;
        }
        if (made && !all) g_dev.devCommDestroy(comm, dc);
        mm = all;
        req.lsaMultimem = false;
    }
    if (!mm) {
        r = g_dev.devCommCreate(comm, &req, dc);
        if (r != ncclSuccess) {
            delete dc;
            drop_wins();
            set_err(err, "sync_device: ncclDevCommCreate", r);
            return 1;
        }
    }
    if (dc->lsaSize != world) {
        char b[200];
        snprintf(b, sizeof b, "sync_device: %d of the %d ranks are load/store-reachable (one NVLink domain is "
                 "required; use the NCCL all-reduce path)", dc->lsaSize, world);
        g_dev.devCommDestroy(comm, dc);
        delete dc;
        drop_wins();
        *err = b;
        return 1;
    }
    ds->comm = comm;
    for (int k = 0; k < nwin; ++k) ds->win[k] = (void*)wins[k];
    ds->nwin = nwin;
    ds->devcomm = (void*)dc;
    ds->multimem = mm;
    ds->lsa_size = dc->lsaSize;
    return 0;
}

void devsync_close(DevSync* ds) {
    if (!ds->devcomm) return;
    auto* dc = (ncclDevComm*)ds->devcomm;
    g_dev.devCommDestroy((ncclComm_t)ds->comm, dc);
    delete dc;
    for (int k = 0; k < ds->nwin; ++k) g_dev.winDeregister((ncclComm_t)ds->comm, (ncclWindow_t)ds->win[k]);
    *ds = DevSync{};
}

// floats [off, off + n) of window `dst` := the mean over the LSA team of the same floats of
// window `src` (src == dst: in place), on `ctas` <= kDevSyncCtas CTAs
cudaError_t devsync_launch(const DevSync& ds, int src, int dst, size_t off, size_t n, unsigned long long* counted,
                           int ctas, cudaStream_t st) {
    if (src < 0 || src >= ds.nwin || dst < 0 || dst >= ds.nwin || ctas < 1 || ctas > kDevSyncCtas)
        return cudaErrorInvalidValue;
    const ncclDevComm& dc = *(const ncclDevComm*)ds.devcomm;
    const ncclWindow_t ws = (ncclWindow_t)ds.win[src], wd = (ncclWindow_t)ds.win[dst];
    if (ds.multimem)
        avg_kernel<true><<<ctas, kThreads, 0, st>>>(ws, wd, dc, off, n, counted);
    else
        avg_kernel<false><<<ctas, kThreads, 0, st>>>(ws, wd, dc, off, n, counted);
    return cudaGetLastError();
}

}  // namespace w2v
