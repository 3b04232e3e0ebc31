// merf_kernels.h -- host-callable launchers of the device kernels (internal to libmerf).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "merf_device.cuh"

namespace merf {

// The render pipeline (merf_render_kernel.cuh).  kf = KF_* flags of the variant.
struct RaySource;
struct Workspace;
struct TraceArgs;
cudaError_t launch_setup(int kf, const DevScene& S, const RaySource& rs, const Workspace& ws,
                         const TraceArgs& ta, unsigned long long* stats, cudaStream_t st);
cudaError_t launch_march(int kf, const DevScene& S, int64_t n, const Workspace& ws, uint32_t rflags,
                         const TraceArgs& ta, unsigned long long* stats, cudaStream_t st,
                         const RaySource& rs, void* out);
// the fused-epilogue march instance applies to this scene (paper geometry, all sources, skip
// table, tensor-core MLP table)
bool fused_march_ok(const DevScene& S);
cudaError_t launch_march_sph(int kf, const DevScene& S, const RaySource& rs, const Workspace& ws,
                             uint32_t rflags, const TraceArgs& ta, unsigned long long* stats, cudaStream_t st);
cudaError_t launch_shade(int kf, const DevScene& S, const RaySource& rs, const Workspace& ws, void* out,
                         const MlpParams& mlp, bool ffma, cudaStream_t st);
// deferred MLP on the tensor cores (merf_shade_mma.cu; needs S.mlp_frag)
cudaError_t launch_shade_mma(int kf, const DevScene& S, const RaySource& rs, const Workspace& ws, void* out,
                             cudaStream_t st);
cudaError_t launch_mlp_frag(const float* w, uint32_t* frag, cudaStream_t st);

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
// NEXT-1 baking helpers
cudaError_t launch_bake_occupancy(const double* x, const double* tau, const double* w, int64_t n,
                                  double tau_thr, double w_thr, int N, uint32_t* bits, cudaStream_t st);
cudaError_t launch_pack_atlas(const uint8_t* dense, int L, const int32_t* index, int64_t n_blocks,
                              uint8_t* atlas, cudaStream_t st);
// appearance pair layouts from the AoS planes / atlas (see DevScene)
cudaError_t launch_pack_pairs(const uint8_t* planes, int R, uint4* plane_pairs, const uint8_t* atlas,
                              int64_t n_blocks, uint4* atlas_pairs, cudaStream_t st);
// skip table of the march (one 4-bit code per finest cell over all dyadic levels; Nf >= 2),
// bordered: (Nf + 2)^3 entries (see merf_build.cu)
inline int64_t skiptab_words(int Nf) { const int64_t b = Nf + 2; return (b * b * b + 3) / 4; }
cudaError_t launch_skiptab(const uint32_t* finest, int Nf, uint32_t* tab, cudaStream_t st);
cudaError_t launch_contract(const double* x, int64_t n, double* y, int32_t* region, cudaStream_t st);

// NEXT-3 quantisation-aware forward/backward (merf_qat.cu)
struct DevScene;
struct RaySource;
struct Workspace;
cudaError_t launch_qat(const DevScene& S, const RaySource& rs, const Workspace& ws, const float* theta_v,
                       const float* theta_p, float* vv, float* vp, int quant, const float* target, float* rgb,
                       float* gvals_v, float* gvals_p, float* grad_v, float* grad_p, float* samp, int smax,
                       float* rayb, const float* mlp, double* loss, unsigned int* overflow,
                       unsigned long long* n_samples, int L, int R, int Nf, const uint32_t* occf, float md, float ma,
                       cudaStream_t st);
cudaError_t launch_stats_fold(unsigned long long* stats, cudaStream_t st);
cudaError_t launch_apron_edge(const int32_t* index, int L, int64_t n_blocks, uint8_t* atlas, cudaStream_t st);

}  // namespace merf
