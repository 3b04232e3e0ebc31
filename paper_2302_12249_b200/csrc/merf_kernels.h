// merf_kernels.h -- host-callable launchers of the device kernels (internal to libmerf).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "merf_device.cuh"

namespace merf {

cudaError_t launch_render_frames(const DevScene& S, const CamBatch& cb, int W, int H, int format,
                                 void* out, uint32_t rflags, unsigned long long* stats,
                                 cudaStream_t st);
cudaError_t launch_render_frames_f32(const DevScene& S, const CamBatch& cb, int W, int H, void* out,
                                     uint32_t rflags, unsigned long long* stats, cudaStream_t st);
cudaError_t launch_render_frames_u8(const DevScene& S, const CamBatch& cb, int W, int H, void* out,
                                    uint32_t rflags, unsigned long long* stats, cudaStream_t st);
cudaError_t launch_render_rays(const DevScene& S, const double* o, const double* d,
                               const double* t_near, int64_t n, float* rgb, uint32_t rflags,
                               unsigned long long* stats, cudaStream_t st);
cudaError_t launch_trace(const DevScene& S, const merf_camera& cam, int W, const int64_t* pixel_ids,
                         int64_t n, int max_per_ray, uint64_t* cells, float* T, int32_t* counts,
                         uint32_t rflags, cudaStream_t st);

cudaError_t launch_segments(const DevScene& S, const merf_camera& cam, int W, const int64_t* pixel_ids,
                            int64_t n, int max_seg, merf_segment* segs, int32_t* counts, cudaStream_t st);

// K0: coarse[N^3 bits] = OR over each (f/N)^3 block of fine[f^3 bits]
cudaError_t launch_maxpool_bits(const uint32_t* fine, int f, uint32_t* coarse, int N, cudaStream_t st);
// K1 part 1: need[(L/8)^3] = 1 for every block slot some occupied finest cell can reach
cudaError_t launch_block_need(const uint32_t* finest, int N, int L, uint8_t* need, cudaStream_t st);
// K1 part 2: index[slot] = need ? exclusive_scan(need)[slot] : -1 ; returns count via *d_count
cudaError_t launch_block_number(const uint8_t* need, int64_t slots, int32_t* index, int64_t* d_count,
                                void* d_temp, size_t* temp_bytes, int32_t* d_scan, cudaStream_t st);
// upload check: *d_bad += slots that are needed but not stored, or entries out of range
cudaError_t launch_block_check(const uint8_t* need, const int32_t* index, int64_t slots,
                               int64_t n_blocks, unsigned long long* d_bad, cudaStream_t st);
// internal density-first layouts (quads per plane texel, octets per grid base voxel)
cudaError_t launch_pack_density(const uint8_t* planes, int R, uint32_t* pdens, const uint8_t* atlas,
                                int64_t n_blocks, uint2* vdens, cudaStream_t st);
cudaError_t launch_contract(const double* x, int64_t n, double* y, int32_t* region, cudaStream_t st);

}  // namespace merf
