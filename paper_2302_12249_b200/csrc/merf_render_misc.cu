// merf_render_misc.cu -- launchers (explicit instantiations) of the render kernel.
#include "merf_render_kernel.cuh"

namespace merf {
cudaError_t launch_render_frames(const DevScene& S, const CamBatch& cb, int W, int H, int format,
                                 void* out, uint32_t rflags, unsigned long long* stats,
                                 cudaStream_t st) {
    return format == MERF_RGBA_U8 ? launch_render_frames_u8(S, cb, W, H, out, rflags, stats, st)
                                  : launch_render_frames_f32(S, cb, W, H, out, rflags, stats, st);
}

cudaError_t launch_render_rays(const DevScene& S, const double* o, const double* d,
                               const double* t_near, int64_t n, float* rgb, uint32_t rflags,
                               unsigned long long* stats, cudaStream_t st) {
    CamBatch cb{};
    RayArgs ra{o, d, t_near, nullptr, n};
    TraceArgs ta{};
    dim3 grid((unsigned)((n + 127) / 128));
    if (rflags & MERF_DENSE) {
        if (stats) render_kernel<KF_RAYS | KF_COUNT | KF_DENSE><<<grid, 128, 0, st>>>(S, cb, 0, 0, rgb, rflags, ra, ta, stats);
        else render_kernel<KF_RAYS | KF_DENSE><<<grid, 128, 0, st>>>(S, cb, 0, 0, rgb, rflags, ra, ta, stats);
    } else {
        if (stats) render_kernel<KF_RAYS | KF_COUNT><<<grid, 128, 0, st>>>(S, cb, 0, 0, rgb, rflags, ra, ta, stats);
        else render_kernel<KF_RAYS><<<grid, 128, 0, st>>>(S, cb, 0, 0, rgb, rflags, ra, ta, stats);
    }
    return cudaGetLastError();
}

cudaError_t launch_trace(const DevScene& S, const merf_camera& cam, int W, const int64_t* pixel_ids,
                         int64_t n, int max_per_ray, uint64_t* cells, float* T, int32_t* counts,
                         uint32_t rflags, cudaStream_t st) {
    CamBatch cb{};
    cb.cam[0] = cam;
    cb.n = 1;
    RayArgs ra{nullptr, nullptr, nullptr, pixel_ids, n};
    TraceArgs ta{cells, T, counts, max_per_ray, nullptr};
    dim3 grid((unsigned)((n + 127) / 128));
    if (rflags & MERF_DENSE)
        render_kernel<KF_TRACE | KF_DENSE><<<grid, 128, 0, st>>>(S, cb, W, 0, nullptr, rflags, ra, ta, nullptr);
    else
        render_kernel<KF_TRACE><<<grid, 128, 0, st>>>(S, cb, W, 0, nullptr, rflags, ra, ta, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_segments(const DevScene& S, const merf_camera& cam, int W, const int64_t* pixel_ids,
                            int64_t n, int max_seg, merf_segment* segs, int32_t* counts, cudaStream_t st) {
    CamBatch cb{};
    cb.cam[0] = cam;
    cb.n = 1;
    RayArgs ra{nullptr, nullptr, nullptr, pixel_ids, n};
    TraceArgs ta{nullptr, nullptr, counts, max_seg, segs};
    dim3 grid((unsigned)((n + 127) / 128));
    render_kernel<KF_SEGS><<<grid, 128, 0, st>>>(S, cb, W, 0, nullptr, 0, ra, ta, nullptr);
    return cudaGetLastError();
}

}  // namespace merf
