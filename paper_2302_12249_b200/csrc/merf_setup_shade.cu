// merf_setup_shade.cu -- instantiations + launchers of the setup and shade kernels.
#include "merf_render_kernel.cuh"

namespace merf {

template <int KF>
static cudaError_t setup_v(const DevScene& S, const RaySource& rs, const Workspace& ws, const TraceArgs& ta,
                           unsigned long long* stats, cudaStream_t st) {
    if (rs.n <= 0) return cudaSuccess;
    dim3 grid((unsigned)((rs.n + kSetupThreads - 1) / kSetupThreads));
    setup_kernel<KF><<<grid, kSetupThreads, 0, st>>>(S, rs, ws, ta, stats);
    return cudaGetLastError();
}

cudaError_t launch_setup(int kf, const DevScene& S, const RaySource& rs, const Workspace& ws,
                         const TraceArgs& ta, unsigned long long* stats, cudaStream_t st) {
    switch (kf & (KF_RAYS | KF_TRACE | KF_SEGS | KF_COUNT | KF_SPH | KF_LPT)) {
        case KF_LPT: return setup_v<KF_LPT>(S, rs, ws, ta, stats, st);
        case KF_LPT | KF_COUNT: return setup_v<KF_LPT | KF_COUNT>(S, rs, ws, ta, stats, st);
        case KF_SPH: return setup_v<KF_SPH>(S, rs, ws, ta, stats, st);
        case KF_SPH | KF_COUNT: return setup_v<KF_SPH | KF_COUNT>(S, rs, ws, ta, stats, st);
        case 0: return setup_v<0>(S, rs, ws, ta, stats, st);
        case KF_COUNT: return setup_v<KF_COUNT>(S, rs, ws, ta, stats, st);
        case KF_RAYS: return setup_v<KF_RAYS>(S, rs, ws, ta, stats, st);
        case KF_RAYS | KF_COUNT: return setup_v<KF_RAYS | KF_COUNT>(S, rs, ws, ta, stats, st);
        case KF_TRACE: return setup_v<KF_TRACE>(S, rs, ws, ta, stats, st);
        case KF_SEGS: return setup_v<KF_SEGS>(S, rs, ws, ta, stats, st);
        default: return cudaErrorInvalidValue;
    }
}

template <int KF>
static cudaError_t shade_v(const DevScene& S, const RaySource& rs, const Workspace& ws, void* out,
                           const MlpParams& mlp, cudaStream_t st) {
    if (rs.n <= 0) return cudaSuccess;
    dim3 grid((unsigned)((rs.n + kSetupThreads - 1) / kSetupThreads));
    shade_kernel<KF><<<grid, kSetupThreads, 0, st>>>(S, rs, ws, out, mlp);
    return cudaGetLastError();
}

cudaError_t launch_shade(int kf, const DevScene& S, const RaySource& rs, const Workspace& ws, void* out,
                         const MlpParams& mlp, bool ffma, cudaStream_t st) {
    // the tensor-core MLP when the scene has its fragment table (activation bound checked at
    // upload), unless the caller asked for the FFMA kernel (MERF_MLP_FFMA)
    if (S.mlp_frag && !ffma) return launch_shade_mma(kf, S, rs, ws, out, st);
    switch (kf & (KF_RAYS | KF_U8)) {
        case 0: return shade_v<0>(S, rs, ws, out, mlp, st);
        case KF_U8: return shade_v<KF_U8>(S, rs, ws, out, mlp, st);
        case KF_RAYS: return shade_v<KF_RAYS>(S, rs, ws, out, mlp, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace merf
