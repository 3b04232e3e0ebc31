// merf_comm.cu -- multi-GPU plumbing of libmerf: the NCCL frame gather to a
// root rank, the single-frame shard assembly kernel, and communicator error handling.
//
// The render path has no collective (rays are independent and the scene is replicated): the
// only exchange is the gather of FINISHED frames.  NCCL is loaded at run time (dlopen of
// libnccl.so.2, or MERF_NCCL_LIB), so libmerf itself has no link-time NCCL dependency and a
// process without NCCL gets MERF_ENCCL from these calls instead of a loader error.  When torch
// has already loaded its NCCL, dlopen returns that same library (soname match).
#include <dlfcn.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/merf.h"
#include "merf_kernels.h"

merf_status merf_set_error(merf_status s, const char* msg);   // merf_api.cu

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    char err[256] = {0};
};

NcclApi g_api;

NcclApi* nccl() {
    NcclApi& api = g_api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* path = getenv("MERF_NCCL_LIB");
        void* h = dlopen(path && path[0] ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            snprintf(api.err, sizeof(api.err), "cannot load NCCL (%s)", dlerror());
            return;
        }
        bool ok = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) {
                ok = false;
                snprintf(api.err, sizeof(api.err), "NCCL symbol %s missing", name);
            }
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommAbort, "ncclCommAbort");
        sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
        sym(api.GetVersion, "ncclGetVersion");
        if (ok) api.h = h;
    });
    return api.h ? &api : nullptr;
}

merf_status nccl_fail(const char* what, ncclResult_t r) {
    char buf[384];
    NcclApi* a = nccl();
    snprintf(buf, sizeof(buf), "%s: %s", what, a ? a->GetErrorString(r) : "NCCL unavailable");
    return merf_set_error(MERF_ENCCL, buf);
}

merf_status no_nccl() {
    char buf[320];
    snprintf(buf, sizeof(buf), "NCCL unavailable: %s (set MERF_NCCL_LIB to a libnccl.so.2)", g_api.err);
    return merf_set_error(MERF_ENCCL, buf);
}

struct DevScope {
    int prev = -1;
    explicit DevScope(int dev) {
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DevScope() { if (prev >= 0) cudaSetDevice(prev); }
};

}  // namespace

struct merf_comm {
    ncclComm_t comm = nullptr;
    int n_ranks = 0, rank = 0, device = 0;
    bool aborted = false;
};

extern "C" merf_status merf_comm_unique_id(uint8_t* id_out) {
    if (!id_out) return merf_set_error(MERF_EINVAL, "id_out is NULL");
    NcclApi* a = nccl();
    if (!a) return no_nccl();
    ncclUniqueId id;
    ncclResult_t r = a->GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
    memcpy(id_out, id.internal, MERF_COMM_ID_BYTES);
    return MERF_OK;
}

extern "C" merf_status merf_comm_init(const uint8_t* id, int32_t n_ranks, int32_t rank, int32_t device,
                                      merf_comm** out) {
    if (!id || !out) return merf_set_error(MERF_EINVAL, "NULL id/out");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return merf_set_error(MERF_EINVAL, "need 0 <= rank < n_ranks");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return merf_set_error(MERF_EINVAL, "device out of range");
    NcclApi* a = nccl();
    if (!a) return no_nccl();
    DevScope ds(device);
    ncclUniqueId uid;
    memcpy(uid.internal, id, MERF_COMM_ID_BYTES);
    merf_comm* c = new merf_comm();
    c->n_ranks = n_ranks;
    c->rank = rank;
    c->device = device;
    ncclResult_t r = a->CommInitRank(&c->comm, n_ranks, uid, rank);   // blocking: all ranks join
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail("ncclCommInitRank", r);
    }
    *out = c;
    return MERF_OK;
}

extern "C" merf_status merf_comm_free(merf_comm* c) {
    if (!c) return MERF_OK;
    NcclApi* a = nccl();
    if (a && c->comm) {
        DevScope ds(c->device);
        if (c->aborted) {
            // already torn down by merf_comm_wait's abort
        } else {
            a->CommDestroy(c->comm);
        }
    }
    delete c;
    return MERF_OK;
}

// The async error state of the communicator (ncclCommGetAsyncError): a failed peer or network
// error surfaces here, not as a return code of the enqueueing call.
static merf_status comm_state(merf_comm* c) {
    if (c->aborted) return merf_set_error(MERF_ENCCL, "communicator was aborted (earlier error or timeout)");
    ncclResult_t st = ncclSuccess;
    ncclResult_t r = nccl()->CommGetAsyncError(c->comm, &st);
    if (r != ncclSuccess) return nccl_fail("ncclCommGetAsyncError", r);
    if (st != ncclSuccess && st != ncclInProgress) return nccl_fail("NCCL async error", st);
    return MERF_OK;
}

extern "C" merf_status merf_gather_frames(merf_comm* c, const void* local, void* root_buf, int64_t bytes,
                                          int32_t root, void* stream) {
    if (!c || !c->comm) return merf_set_error(MERF_EINVAL, "NULL communicator");
    if (bytes < 0 || root < 0 || root >= c->n_ranks) return merf_set_error(MERF_EINVAL, "bad bytes / root");
    if (bytes > 0 && !local) return merf_set_error(MERF_EINVAL, "local is NULL");
    if (bytes > 0 && c->rank == root && !root_buf) return merf_set_error(MERF_EINVAL, "root_buf is NULL on the root");
    if (bytes == 0) return MERF_OK;
    NcclApi* a = nccl();
    if (!a) return no_nccl();
    merf_status s = comm_state(c);
    if (s) return s;
    DevScope ds(c->device);
    nvtxRangePushA("merf.gather_frames");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)bytes;
    ncclResult_t r = a->GroupStart();
    if (r != ncclSuccess) return nccl_fail("ncclGroupStart", r);
    if (c->rank == root) {
        // the root's own frames: a device copy into its slot; every other rank's by ncclRecv
        cudaError_t ce = cudaMemcpyAsync((char*)root_buf + (size_t)root * n, local, n, cudaMemcpyDeviceToDevice, st);
        if (ce != cudaSuccess) {
            a->GroupEnd();
            return merf_set_error(MERF_ECUDA, cudaGetErrorString(ce));
        }
        for (int p = 0; p < c->n_ranks && r == ncclSuccess; p++)
            if (p != root) r = a->Recv((char*)root_buf + (size_t)p * n, n, ncclUint8, p, c->comm, st);
    } else {
        r = a->Send(local, n, ncclUint8, root, c->comm, st);
    }
    ncclResult_t r2 = a->GroupEnd();
    if (r != ncclSuccess) return nccl_fail("ncclSend/ncclRecv", r);
    if (r2 != ncclSuccess) return nccl_fail("ncclGroupEnd", r2);
    return comm_state(c);
}

extern "C" merf_status merf_comm_wait(merf_comm* c, void* stream, int32_t timeout_ms) {
    if (!c || !c->comm) return merf_set_error(MERF_EINVAL, "NULL communicator");
    NcclApi* a = nccl();
    if (!a) return no_nccl();
    DevScope ds(c->device);
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
        cudaError_t q = cudaStreamQuery((cudaStream_t)stream);
        if (q == cudaSuccess) return comm_state(c);
        if (q != cudaErrorNotReady) return merf_set_error(MERF_ECUDA, cudaGetErrorString(q));
        merf_status s = comm_state(c);
        if (s) {
            a->CommAbort(c->comm);           // unblock the stream; the communicator is unusable
            c->aborted = true;
            return s;
        }
        const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
        if (timeout_ms >= 0 && ms > timeout_ms) {
            a->CommAbort(c->comm);
            c->aborted = true;
            char buf[160];
            snprintf(buf, sizeof(buf), "frame gather did not complete within %d ms: communicator aborted", timeout_ms);
            return merf_set_error(MERF_ENCCL, buf);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

extern "C" merf_status merf_comm_info(const merf_comm* c, int32_t* n_ranks, int32_t* rank, int32_t* nccl_version) {
    if (!c) return merf_set_error(MERF_EINVAL, "NULL communicator");
    if (n_ranks) *n_ranks = c->n_ranks;
    if (rank) *rank = c->rank;
    if (nccl_version) {
        int v = 0;
        NcclApi* a = nccl();
        if (a) a->GetVersion(&v);
        *nccl_version = v;
    }
    return MERF_OK;
}

// ------------------------------------------------------------------------------------
// single-frame shards: assembling the gathered 64x64 blocks into frames
// ------------------------------------------------------------------------------------
namespace {

// One thread per pixel of every gathered block slot: [part][view][slot][64][64] -> frame.
// Block b of the frame belongs to part b % part_count, slot b / part_count (row-major blocks).
template <int PX>
__global__ void shard_assemble_kernel(const uint8_t* __restrict__ blocks, int n_views, int W, int H,
                                      int part_count, int slots, int nbx, int n_blocks, uint8_t* __restrict__ frame) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_part = (int64_t)n_views * slots * 4096;
    if (i >= per_part * part_count) return;
    const int part = (int)(i / per_part);
    int64_t rem = i - (int64_t)part * per_part;
    const int view = (int)(rem / ((int64_t)slots * 4096));
    rem -= (int64_t)view * slots * 4096;
    const int slot = (int)(rem >> 12);
    const int p = (int)(rem & 4095);
    const int b = part + part_count * slot;
    if (b >= n_blocks) return;
    const int by = b / nbx, bx = b - by * nbx;
    const int x = bx * 64 + (p & 63), y = by * 64 + (p >> 6);
    if (x >= W || y >= H) return;
    const uint8_t* src = blocks + (size_t)i * PX;
    uint8_t* dst = frame + (((size_t)view * H + y) * W + x) * PX;
    if (PX == 4) {
        *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(src);
    } else {
        const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
        uint32_t* d = reinterpret_cast<uint32_t*>(dst);
        d[0] = s[0]; d[1] = s[1]; d[2] = s[2];
    }
}

}  // namespace

extern "C" int32_t merf_shard_slots(int32_t W, int32_t H, int32_t part_count) {
    if (W <= 0 || H <= 0 || part_count < 1) return 0;
    const int nb = ((W + 63) / 64) * ((H + 63) / 64);
    return (nb + part_count - 1) / part_count;
}

extern "C" merf_status merf_shard_assemble(const void* blocks, int32_t n_views, int32_t W, int32_t H,
                                           int32_t part_count, int32_t format, void* frame_out, void* stream) {
    if (!blocks || !frame_out) return merf_set_error(MERF_EINVAL, "NULL blocks/frame_out");
    if (n_views <= 0 || W <= 0 || H <= 0 || part_count < 1) return merf_set_error(MERF_EINVAL, "bad n_views/W/H/part_count");
    if (format != MERF_RGB_F32 && format != MERF_RGBA_U8) return merf_set_error(MERF_EINVAL, "bad format");
    const int slots = merf_shard_slots(W, H, part_count);
    const int nbx = (W + 63) / 64;
    const int n_blocks = nbx * ((H + 63) / 64);
    const int64_t n = (int64_t)part_count * n_views * slots * 4096;
    const unsigned grid = (unsigned)((n + 255) / 256);
    if (format == MERF_RGBA_U8)
        shard_assemble_kernel<4><<<grid, 256, 0, (cudaStream_t)stream>>>((const uint8_t*)blocks, n_views, W, H, part_count,
                                                                         slots, nbx, n_blocks, (uint8_t*)frame_out);
    else
        shard_assemble_kernel<12><<<grid, 256, 0, (cudaStream_t)stream>>>((const uint8_t*)blocks, n_views, W, H, part_count,
                                                                          slots, nbx, n_blocks, (uint8_t*)frame_out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return merf_set_error(MERF_ECUDA, cudaGetErrorString(e));
    return MERF_OK;
}
