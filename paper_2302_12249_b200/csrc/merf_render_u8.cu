// merf_render_u8.cu -- launchers (explicit instantiations) of the render kernel.
#include "merf_render_kernel.cuh"

namespace merf {
// ------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------
template <int KF>
static cudaError_t launch_frames(const DevScene& S, const CamBatch& cb, int W, int H, void* out,
                                 uint32_t rflags, unsigned long long* stats, cudaStream_t st) {
    dim3 grid((W + 15) / 16, (H + 7) / 8, cb.n);
    RayArgs ra{};
    TraceArgs ta{};
    render_kernel<KF><<<grid, 128, 0, st>>>(S, cb, W, H, out, rflags, ra, ta, stats);
    return cudaGetLastError();
}

cudaError_t launch_render_frames_u8(const DevScene& S, const CamBatch& cb, int W, int H, void* out,
                                    uint32_t rflags, unsigned long long* stats, cudaStream_t st) {
    const bool cnt = stats != nullptr;
    if (rflags & MERF_DENSE)
        return cnt ? launch_frames<KF_U8 | KF_COUNT | KF_DENSE>(S, cb, W, H, out, rflags, stats, st)
                   : launch_frames<KF_U8 | KF_DENSE>(S, cb, W, H, out, rflags, stats, st);
    return cnt ? launch_frames<KF_U8 | KF_COUNT>(S, cb, W, H, out, rflags, stats, st)
               : launch_frames<KF_U8>(S, cb, W, H, out, rflags, stats, st);
}

}  // namespace merf
