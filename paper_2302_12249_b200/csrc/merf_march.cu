// merf_march.cu -- instantiations + launcher of the persistent march kernel.
#include <cstdio>
#include <cstdlib>

#include "merf_render_kernel.cuh"

namespace merf {

constexpr int kMaxDevices = 64;

template <int KF>
static cudaError_t march_v(const DevScene& S, int64_t n, const Workspace& ws, uint32_t rflags,
                           const TraceArgs& ta, unsigned long long* stats, cudaStream_t st,
                           const RaySource& rs, void* out) {
    if (n <= 0) return cudaSuccess;
    // persistent grid: resident CTAs x SMs, cached per variant and per device (the caller's
    // entry point has made the scene's device current)
    static int cache[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int blocks = (dev >= 0 && dev < kMaxDevices) ? cache[dev] : 0;
    if (blocks == 0) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march_kernel<KF>, kMarchThreads, 0);
        blocks = sms * (per_sm > 0 ? per_sm : 1);
        if (dev >= 0 && dev < kMaxDevices) cache[dev] = blocks;
    }
    int64_t need = (n + kMarchThreads - 1) / kMarchThreads;
    int grid = (int)(need < blocks ? need : blocks);
    // the tile queue is reset by the setup kernel that always precedes the march; launched as a
    // programmatic dependent of it (the march waits for the setup grid with griddepcontrol.wait)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kMarchThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, march_kernel<KF>, S, n, ws, rflags, ta, stats, rs, out);
    return cudaGetLastError();
}

// fold one launch's (start, dry, end) timestamps into the busy / tail sums and re-arm them
__global__ void stats_fold_kernel(unsigned long long* st) {
    if (st[16] != ~0ull && st[17] != ~0ull && st[18] >= st[17] && st[17] >= st[16]) {
        st[19] += st[17] - st[16];
        st[20] += st[18] - st[17];
    }
    st[16] = ~0ull;
    st[17] = ~0ull;
    st[18] = 0;
}

cudaError_t launch_stats_fold(unsigned long long* stats, cudaStream_t st) {
    stats_fold_kernel<<<1, 1, 0, st>>>(stats);
    return cudaGetLastError();
}

static bool env_flag(const char* name) {
    const char* e = getenv(name);
    return e && e[0] && e[0] != '0';
}

// the per-cell skip table is used when the scene has one, unless MERF_NO_SKIPTAB is set (tests
// and ablations run both traversals)
static bool use_skiptab(const DevScene& S) {
    if (!S.skiptab) return false;
    const char* e = getenv("MERF_NO_SKIPTAB");
    return !(e && e[0] && e[0] != '0');
}

static bool paper_geometry(const DevScene& S) {
    return S.L == kPaperL && S.R == kPaperR && S.n_fin == kPaperNf && !env_flag("MERF_NO_PAPER");
}

bool fused_march_ok(const DevScene& S) {
    return S.n_src == 4 && use_skiptab(S) && paper_geometry(S) && S.mlp_frag != nullptr;
}

cudaError_t launch_march(int kf, const DevScene& S, int64_t n, const Workspace& ws, uint32_t rflags,
                         const TraceArgs& ta, unsigned long long* stats, cudaStream_t st,
                         const RaySource& rs, void* out) {
    if (kf & KF_FUSED) {                              // production + fused MLP epilogue (paper geometry)
        if (kf & KF_U8) return march_v<KF_ALLSRC | KF_SKIPTAB | KF_PAPER | KF_FUSED | KF_U8>(S, n, ws, rflags, ta, stats, st, rs, out);
        return march_v<KF_ALLSRC | KF_SKIPTAB | KF_PAPER | KF_FUSED>(S, n, ws, rflags, ta, stats, st, rs, out);
    }
    if (kf & KF_SPH) {                                // NEXT-2 like-for-like variant
        if (S.n_src == 4 && paper_geometry(S)) {
            if (kf & KF_COUNT) return march_v<KF_SPH | KF_ALLSRC | KF_PAPER | KF_COUNT>(S, n, ws, rflags, ta, stats, st, rs, out);
            return march_v<KF_SPH | KF_ALLSRC | KF_PAPER>(S, n, ws, rflags, ta, stats, st, rs, out);
        }
        if (kf & KF_COUNT) return march_v<KF_SPH | KF_COUNT>(S, n, ws, rflags, ta, stats, st, rs, out);
        return march_v<KF_SPH>(S, n, ws, rflags, ta, stats, st, rs, out);
    }
    const bool tab = use_skiptab(S);
    if (S.n_src == 4 && !(kf & (KF_TRACE | KF_DENSE))) {    // production variants
        if (tab) {
            if (paper_geometry(S)) {
                if (kf & KF_COUNT) return march_v<KF_ALLSRC | KF_SKIPTAB | KF_PAPER | KF_COUNT>(S, n, ws, rflags, ta, stats, st, rs, out);
                return march_v<KF_ALLSRC | KF_SKIPTAB | KF_PAPER>(S, n, ws, rflags, ta, stats, st, rs, out);
            }
            if (kf & KF_COUNT) return march_v<KF_ALLSRC | KF_SKIPTAB | KF_COUNT>(S, n, ws, rflags, ta, stats, st, rs, out);
            return march_v<KF_ALLSRC | KF_SKIPTAB>(S, n, ws, rflags, ta, stats, st, rs, out);
        }
        if (kf & KF_COUNT) return march_v<KF_ALLSRC | KF_COUNT>(S, n, ws, rflags, ta, stats, st, rs, out);
        return march_v<KF_ALLSRC>(S, n, ws, rflags, ta, stats, st, rs, out);
    }
    // traces: the production instances (the ones merf_render times) plus the trace writes, so
    // the traversal and gather code of the timed kernel is what the bit-exact trace tests check
    if (tab && S.n_src == 4 && (kf & (KF_TRACE | KF_DENSE | KF_COUNT)) == KF_TRACE) {
        if (paper_geometry(S)) return march_v<KF_TRACE | KF_ALLSRC | KF_SKIPTAB | KF_PAPER>(S, n, ws, rflags, ta, stats, st, rs, out);
        return march_v<KF_TRACE | KF_ALLSRC | KF_SKIPTAB>(S, n, ws, rflags, ta, stats, st, rs, out);
    }
    if (tab && (kf & (KF_TRACE | KF_DENSE | KF_COUNT)) == KF_TRACE)
        return march_v<KF_TRACE | KF_SKIPTAB>(S, n, ws, rflags, ta, stats, st, rs, out);
    if (tab && (kf & (KF_TRACE | KF_DENSE | KF_COUNT)) == 0)
        return march_v<KF_SKIPTAB>(S, n, ws, rflags, ta, stats, st, rs, out);
    if (tab && (kf & (KF_TRACE | KF_DENSE | KF_COUNT)) == KF_COUNT)
        return march_v<KF_SKIPTAB | KF_COUNT>(S, n, ws, rflags, ta, stats, st, rs, out);
    switch (kf & (KF_TRACE | KF_DENSE | KF_COUNT)) {
        case 0: return march_v<0>(S, n, ws, rflags, ta, stats, st, rs, out);
        case KF_COUNT: return march_v<KF_COUNT>(S, n, ws, rflags, ta, stats, st, rs, out);
        case KF_DENSE: return march_v<KF_DENSE>(S, n, ws, rflags, ta, stats, st, rs, out);
        case KF_DENSE | KF_COUNT: return march_v<KF_DENSE | KF_COUNT>(S, n, ws, rflags, ta, stats, st, rs, out);
        case KF_TRACE: return march_v<KF_TRACE>(S, n, ws, rflags, ta, stats, st, rs, out);
        case KF_TRACE | KF_DENSE: return march_v<KF_TRACE | KF_DENSE>(S, n, ws, rflags, ta, stats, st, rs, out);
        default: return cudaErrorInvalidValue;
    }
}

template <int KF>
static cudaError_t sph_v(const DevScene& S, const RaySource& rs, const Workspace& ws, uint32_t rflags,
                         const TraceArgs& ta, unsigned long long* stats, cudaStream_t st) {
    if (rs.n <= 0) return cudaSuccess;
    dim3 grid((unsigned)((rs.n + kSetupThreads - 1) / kSetupThreads));
    march_sph_kernel<KF><<<grid, kSetupThreads, 0, st>>>(S, rs, ws, rflags, ta, stats);
    return cudaGetLastError();
}

cudaError_t launch_march_sph(int kf, const DevScene& S, const RaySource& rs, const Workspace& ws,
                             uint32_t rflags, const TraceArgs& ta, unsigned long long* stats, cudaStream_t st) {
    switch (kf & (KF_TRACE | KF_RAYS | KF_COUNT)) {
        case 0: return sph_v<0>(S, rs, ws, rflags, ta, stats, st);
        case KF_COUNT: return sph_v<KF_COUNT>(S, rs, ws, rflags, ta, stats, st);
        case KF_RAYS: return sph_v<KF_RAYS>(S, rs, ws, rflags, ta, stats, st);
        case KF_RAYS | KF_COUNT: return sph_v<KF_RAYS | KF_COUNT>(S, rs, ws, rflags, ta, stats, st);
        case KF_TRACE: return sph_v<KF_TRACE>(S, rs, ws, rflags, ta, stats, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace merf
