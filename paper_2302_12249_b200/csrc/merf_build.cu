// merf_build.cu -- upload-time structure kernels (sm_100a):
//   K0 occupancy pyramid by max-pooling the finest binary grid,
//   K1 canonical block allocation of the sparse 3D grid (reading D11),
//   and the contract_pi helper.
#include <cstdint>
#include <cub/device/device_scan.cuh>
#include <cstdlib>
#include <cuda_runtime.h>

#include "merf_device.cuh"
#include "merf_kernels.h"

namespace merf {

static __host__ __device__ __forceinline__ int ilog2(int v) {
    int n = 0;
    while ((1 << n) < v) n++;
    return n;
}

// One thread per 32-bit word of the coarse level: OR over the r^3 fine cells of each of its
// 32 coarse cells.  No atomics; deterministic.
__global__ void maxpool_bits_kernel(const uint32_t* __restrict__ fine, int f,
                                    uint32_t* __restrict__ coarse, int N) {
    int64_t word = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = ((int64_t)N * N * N + 31) / 32;
    if (word >= total) return;
    const int r = f / N;
    uint32_t out = 0;
    for (int b = 0; b < 32; b++) {
        int64_t lin = word * 32 + b;
        if (lin >= (int64_t)N * N * N) break;
        int x = (int)(lin % N), y = (int)((lin / N) % N), z = (int)(lin / ((int64_t)N * N));
        bool any = false;
        for (int dz = 0; dz < r && !any; dz++)
            for (int dy = 0; dy < r && !any; dy++) {
                // the r fine cells along x of one (z, y) row are contiguous bits
                int64_t l0 = ((int64_t)(z * r + dz) * f + (y * r + dy)) * f + (int64_t)x * r;
                for (int dx = 0; dx < r; dx += 32) {
                    int64_t l = l0 + dx;
                    int nbits = min(32, r - dx);
                    int64_t w0 = l >> 5;
                    int sh = (int)(l & 31);
                    uint64_t v = __ldg(fine + w0);
                    if (sh + nbits > 32) v |= (uint64_t)__ldg(fine + w0 + 1) << 32;
                    uint64_t mask = (nbits == 64) ? ~0ull : ((1ull << nbits) - 1);
                    if ((v >> sh) & mask) { any = true; break; }
                }
            }
        if (any) out |= 1u << b;
    }
    coarse[word] = out;
}

// OR-pool by 2 in x, y and z (fine resolution 2N, N >= 32): one thread per coarse 32-bit
// word = 32 coarse cells of one (z, y) row; it reads the 2 x 2 rows of 2 fine words,
// ORs them, ORs adjacent bit pairs and compacts the even bits.  Every fine word is read
// exactly once (bandwidth-bound); repeated halvings give the max-pool of any power-of-two
// factor exactly (OR is associative).
__device__ __forceinline__ uint32_t compact_even(uint32_t x) {
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    x = (x | (x >> 8)) & 0x0000FFFFu;
    return x;
}

__global__ void halve_bits_kernel(const uint32_t* __restrict__ fine, uint32_t* __restrict__ coarse, int N) {
    const int64_t words = (int64_t)N * N * N / 32;
    const int64_t wi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (wi >= words) return;
    const int wpr = N / 32;                          // coarse words per row
    const int wx = (int)(wi % wpr);
    const int64_t row = wi / wpr;                    // z * N + y
    const int y = (int)(row % N), z = (int)(row / N);
    const int F = 2 * N, fwpr = F / 32;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int dz = 0; dz < 2; dz++)
#pragma unroll
        for (int dy = 0; dy < 2; dy++) {
            const int64_t frow = (int64_t)(2 * z + dz) * F + (2 * y + dy);
            const uint32_t* p = fine + frow * fwpr + 2 * wx;
            lo |= __ldg(p);
            hi |= __ldg(p + 1);
        }
    lo |= lo >> 1;
    hi |= hi >> 1;
    coarse[wi] = compact_even(lo) | (compact_even(hi) << 16);
}

// Lower trilinear base voxel of lattice coordinate Q on the L grid (clamped, as the render
// kernel's texel()).
__device__ __forceinline__ int base_voxel(int64_t Q, int s, int L) {
    int64_t P = Q + kTwo - (int64_t(1) << (s - 1));
    int64_t i = P >> s;
    if (i < 0) i = 0;
    if (i > L - 2) i = L - 2;
    return (int)i;
}

// One thread per finest cell: mark every block slot a sample inside an occupied cell can use.
__global__ void block_need_kernel(const uint32_t* __restrict__ finest, int N, int L,
                                  uint8_t* __restrict__ need) {
    int64_t lin = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lin >= (int64_t)N * N * N) return;
    if (!((__ldg(finest + (lin >> 5)) >> (lin & 31)) & 1u)) return;
    const int cc[3] = {(int)(lin % N), (int)((lin / N) % N), (int)(lin / ((int64_t)N * N))};
    const int so = kF + 2 - ilog2(N);
    const int sv = kF + 2 - ilog2(L);
    const int nb = L / 8;
    int blo[3], bhi[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        int lo = (cc[a] == 0) ? 0 : base_voxel(((int64_t)cc[a] << so) - kTwo, sv, L);
        int hi = (cc[a] == N - 1) ? L - 2 : base_voxel((((int64_t)cc[a] + 1) << so) - kTwo - 1, sv, L);
        blo[a] = lo >> 3;
        bhi[a] = hi >> 3;
    }
    for (int bz = blo[2]; bz <= bhi[2]; bz++)
        for (int by = blo[1]; by <= bhi[1]; by++)
            for (int bx = blo[0]; bx <= bhi[0]; bx++)
                need[((int64_t)bz * nb + by) * nb + bx] = 1;
}

__global__ void to_int_kernel(const uint8_t* __restrict__ need, int32_t* __restrict__ flags, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = need[i];
}

__global__ void number_kernel(const uint8_t* __restrict__ need, const int32_t* __restrict__ scan,
                              int32_t* __restrict__ index, int64_t n, int64_t* count) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) index[i] = need[i] ? scan[i] : -1;
    if (i == n - 1) *count = (int64_t)scan[i] + need[i];
}

__global__ void block_check_kernel(const uint8_t* __restrict__ need, const int32_t* __restrict__ index,
                                   int64_t n, int64_t n_blocks, unsigned long long* bad) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t v = index[i];
    bool b = (v < -1) || (v >= n_blocks) || (need[i] && v < 0);
    if (b) atomicAdd(bad, 1ull);
}

__global__ void contract_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ y,
                                int32_t* __restrict__ region) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]}, c[3];
    int g = region_of(p[0], p[1], p[2]);
    contract_region(g, p, c);
    y[3 * i] = c[0];
    y[3 * i + 1] = c[1];
    y[3 * i + 2] = c[2];
    if (region) region[i] = g;
}

// NEXT-1 baking: one thread per weighted point; a point with w > w_thr and
// tau > tau_thr (i.e. alpha = 1 - exp(-tau Delta) > 0.005 with the renderer's step)
// marks the eight voxels around its contracted position (trilinear corners of the
// cell-centred grid, reading D9) with atomicOr.  Contraction in canonical fp64 (D8).
__global__ void bake_occupancy_kernel(const double* __restrict__ x, const double* __restrict__ tau,
                                      const double* __restrict__ w, int64_t n, double tau_thr,
                                      double w_thr, int N, uint32_t* __restrict__ bits) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (!(w[i] > w_thr) || !(tau[i] > tau_thr)) return;
    const double p[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    double c[3];
    contract_region(region_of(p[0], p[1], p[2]), p, c);
    const int s = kF + 2 - ilog2(N);
    int lo[3];
#pragma unroll
    for (int a = 0; a < 3; a++) lo[a] = base_voxel(__double2ll_rn(mul_rn(c[a], (double)kOne)), s, N);
#pragma unroll
    for (int cz = 0; cz < 2; cz++)
#pragma unroll
        for (int cy = 0; cy < 2; cy++)
#pragma unroll
            for (int cx = 0; cx < 2; cx++) {
                const int64_t lin = ((int64_t)(lo[2] + cz) * N + (lo[1] + cy)) * N + (lo[0] + cx);
                atomicOr(bits + (lin >> 5), 1u << (lin & 31));
            }
}

// Block-sparse storage of a dense V (D11): one thread per (block, voxel of 9^3).
__global__ void pack_atlas_kernel(const uint8_t* __restrict__ dense, int L, const int32_t* __restrict__ index,
                                  int64_t n_slots, int64_t n_blocks, uint8_t* __restrict__ atlas) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_slots * 729) return;
    const int64_t slot = i / 729;
    const int l = (int)(i - slot * 729);
    const int32_t b = index[slot];
    if (b < 0 || b >= n_blocks) return;
    const int nb = L / 8;
    const int bx = (int)(slot % nb), by = (int)((slot / nb) % nb), bz = (int)(slot / ((int64_t)nb * nb));
    const int lx = l % 9, ly = (l / 9) % 9, lz = l / 81;
    const int gx = min(bx * 8 + lx, L - 1), gy = min(by * 8 + ly, L - 1), gz = min(bz * 8 + lz, L - 1);
    const uint2 v = *reinterpret_cast<const uint2*>(dense + (((size_t)gz * L + gy) * L + gx) * 8);
    *reinterpret_cast<uint2*>(atlas + ((size_t)b * 729 + l) * 8) = v;
}

static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_maxpool_bits(const uint32_t* fine, int f, uint32_t* coarse, int N, cudaStream_t st) {
    if (N < 32 || f / N <= 2) {                      // small levels / single halving: direct
        if (N >= 32 && f == 2 * N) {
            halve_bits_kernel<<<blocks_for((int64_t)N * N * N / 32, 256), 256, 0, st>>>(fine, coarse, N);
            return cudaGetLastError();
        }
        int64_t words = ((int64_t)N * N * N + 31) / 32;
        maxpool_bits_kernel<<<blocks_for(words, 256), 256, 0, st>>>(fine, f, coarse, N);
        return cudaGetLastError();
    }
    // successive halvings f -> f/2 -> ... -> N through stream-ordered temporaries
    const uint32_t* src = fine;
    uint32_t* tmp[2] = {nullptr, nullptr};
    int cur = f, t = 0;
    cudaError_t e = cudaSuccess;
    while (cur / 2 > N) {
        const int n2 = cur / 2;
        const size_t bytes = (size_t)n2 * n2 * n2 / 8;
        if (tmp[t] == nullptr && (e = cudaMallocAsync(&tmp[t], (size_t)(cur / 2) * (cur / 2) * (cur / 2) / 8, st)) != cudaSuccess)
            break;
        (void)bytes;
        halve_bits_kernel<<<blocks_for((int64_t)n2 * n2 * n2 / 32, 256), 256, 0, st>>>(src, tmp[t], n2);
        src = tmp[t];
        t ^= 1;
        if (tmp[t]) { cudaFreeAsync(tmp[t], st); tmp[t] = nullptr; }
        cur = n2;
    }
    if (e == cudaSuccess) {
        halve_bits_kernel<<<blocks_for((int64_t)N * N * N / 32, 256), 256, 0, st>>>(src, coarse, N);
        e = cudaGetLastError();
    }
    for (int i = 0; i < 2; i++)
        if (tmp[i]) cudaFreeAsync(tmp[i], st);
    return e;
}

cudaError_t launch_block_need(const uint32_t* finest, int N, int L, uint8_t* need, cudaStream_t st) {
    int64_t slots = (int64_t)(L / 8) * (L / 8) * (L / 8);
    cudaError_t e = cudaMemsetAsync(need, 0, slots, st);
    if (e != cudaSuccess) return e;
    int64_t cells = (int64_t)N * N * N;
    block_need_kernel<<<blocks_for(cells, 256), 256, 0, st>>>(finest, N, L, need);
    return cudaGetLastError();
}

cudaError_t launch_block_number(const uint8_t* need, int64_t slots, int32_t* index, int64_t* d_count,
                                void* d_temp, size_t* temp_bytes, int32_t* d_scan, cudaStream_t st) {
    // d_scan holds 2*slots int32: flags then exclusive scan
    if (d_temp == nullptr) {
        return cub::DeviceScan::ExclusiveSum(nullptr, *temp_bytes, (const int32_t*)nullptr,
                                             (int32_t*)nullptr, (int)slots, st);
    }
    to_int_kernel<<<blocks_for(slots, 256), 256, 0, st>>>(need, d_scan, slots);
    cudaError_t e = cub::DeviceScan::ExclusiveSum(d_temp, *temp_bytes, d_scan, d_scan + slots,
                                                  (int)slots, st);
    if (e != cudaSuccess) return e;
    number_kernel<<<blocks_for(slots, 256), 256, 0, st>>>(need, d_scan + slots, index, slots, d_count);
    return cudaGetLastError();
}

cudaError_t launch_block_check(const uint8_t* need, const int32_t* index, int64_t slots,
                               int64_t n_blocks, unsigned long long* d_bad, cudaStream_t st) {
    block_check_kernel<<<blocks_for(slots, 256), 256, 0, st>>>(need, index, slots, n_blocks, d_bad);
    return cudaGetLastError();
}

cudaError_t launch_bake_occupancy(const double* x, const double* tau, const double* w, int64_t n,
                                  double tau_thr, double w_thr, int N, uint32_t* bits, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(bits, 0, (size_t)(((int64_t)N * N * N + 31) / 32) * 4, st);
    if (e != cudaSuccess || n <= 0) return e;
    bake_occupancy_kernel<<<blocks_for(n, 256), 256, 0, st>>>(x, tau, w, n, tau_thr, w_thr, N, bits);
    return cudaGetLastError();
}

cudaError_t launch_pack_atlas(const uint8_t* dense, int L, const int32_t* index, int64_t n_blocks,
                              uint8_t* atlas, cudaStream_t st) {
    const int64_t slots = (int64_t)(L / 8) * (L / 8) * (L / 8);
    pack_atlas_kernel<<<blocks_for(slots * 729, 256), 256, 0, st>>>(dense, L, index, slots, n_blocks, atlas);
    return cudaGetLastError();
}

cudaError_t launch_contract(const double* x, int64_t n, double* y, int32_t* region, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    contract_kernel<<<blocks_for(n, 256), 256, 0, st>>>(x, n, y, region);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Skip table: for every finest cell, code = lattice shift of the coarsest EMPTY dyadic cell
// containing it, minus 16, or 0 if the finest cell is occupied.  The dyadic levels are the
// OR-pools of the finest level at every power-of-two resolution N_f/2, ..., 1 -- the
// multi-level occupancy grid of P:307-308 completed to all scales, so each skip leaves the
// largest aligned empty cell around the sample.  Only empty space is skipped, so the set of
// evaluated samples (and every trace) is the one of dense stepping.  One byte per entry, one
// thread per 4 entries.
// ------------------------------------------------------------------------------------
constexpr int kMaxDyadic = 16;
struct LevelSet {
    const uint32_t* occ[kMaxDyadic];   // coarse -> fine, res 1, 2, 4, ..., N_f
    int n;
};

// The table is BORDERED: (N + 2)^3 entries, entry (x + 1, y + 1, z + 1) for cell (x, y, z) and
// a one-cell border that repeats the clamped edge cell, so the march indexes it with the
// unclamped cell Qb >> s_fin.  Lattice drift never leaves the cube by a whole finest cell:
// sample k of a segment is within 0.5 + 0.5 k lattice units of its exact position (rounded
// Qa and U), the exact positions lie in [-2, 2]^3, and k < K <= 4 sqrt(3) / Delta <= 3.7e6
// for the smallest accepted Delta = 2^-19 -- below the finest cell of 2^21 units at the
// largest table resolution N = 512 (2^22 at N = 256).
// Chebyshev (L-inf) distance, in finest cells, from every cell to the nearest occupied one,
// capped at kChebCap: three separable passes (x, y, z) over byte grids, each cell scanning its
// row outwards until the running minimum cannot improve.  dist = 0 for occupied cells.
constexpr int kChebCap = 128;
__global__ void cheb_pass_kernel(const uint32_t* __restrict__ occ, const uint8_t* __restrict__ src,
                                 uint8_t* __restrict__ dst, int N, int axis) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)N * N * N) return;
    const int x = (int)(i % N), y = (int)((i / N) % N), z = (int)(i / ((int64_t)N * N));
    const int c = axis == 0 ? x : (axis == 1 ? y : z);
    const int64_t stride = axis == 0 ? 1 : (axis == 1 ? N : (int64_t)N * N);
    int best = kChebCap;
    if (axis == 0) {
        for (int d = 0; d < best && d < N; d++) {          // 1D distance to an occupied cell in the row
            if (c - d >= 0 && ((__ldg(occ + ((i - d) >> 5)) >> ((i - d) & 31)) & 1u)) { best = d; break; }
            if (c + d < N && ((__ldg(occ + ((i + d) >> 5)) >> ((i + d) & 31)) & 1u)) { best = d; break; }
        }
    } else {
        // L-inf composition: min over offsets t of max(|t|, previous distance at c + t)
        for (int t = 0; t < best && t < N; t++) {
            if (c - t >= 0) best = min(best, max(t, (int)src[i - t * stride]));
            if (c + t < N) best = min(best, max(t, (int)src[i + t * stride]));
        }
    }
    dst[i] = (uint8_t)best;
}

__global__ void skiptab_kernel(LevelSet ls, const uint8_t* __restrict__ cheb, uint32_t* __restrict__ tab) {
    const int nl = ls.n;
    const int N = 1 << (nl - 1);
    const int Nb = N + 2;
    const int64_t entries = (int64_t)Nb * Nb * Nb;
    const int64_t words = (entries + 3) / 4;
    const int64_t wi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (wi >= words) return;
    uint32_t out = 0;
    for (int q = 0; q < 4; q++) {
        const int64_t e = wi * 4 + q;
        if (e >= entries) break;
        const int x = min(max((int)(e % Nb) - 1, 0), N - 1);
        const int y = min(max((int)((e / Nb) % Nb) - 1, 0), N - 1);
        const int z = min(max((int)(e / ((int64_t)Nb * Nb)) - 1, 0), N - 1);
        const int64_t c = ((int64_t)z * N + y) * N + x;
        uint32_t code = 0;
        if (!((__ldg(ls.occ[nl - 1] + (c >> 5)) >> (c & 31)) & 1u)) {
            int lev = nl - 1;                    // the finest (known empty) unless a coarser one is
            for (int l = 0; l < nl - 1; l++) {
                const int sft = nl - 1 - l, M = 1 << l;
                const int64_t li = ((int64_t)(z >> sft) * M + (y >> sft)) * M + (x >> sft);
                if (!((__ldg(ls.occ[l] + (li >> 5)) >> (li & 31)) & 1u)) {
                    lev = l;
                    break;
                }
            }
            code = (uint32_t)(kF + 2 - lev - 16);   // lattice shift of resolution 2^lev, - 16
            // the cube of Chebyshev radius D - 1 around the cell is empty too (D = distance to
            // the nearest occupied cell); take it when it is larger than the dyadic cell
            if (cheb) {
                const int r = (int)cheb[c] - 1;
                if (2 * r + 1 > (1 << (nl - 1 - lev))) code = 128u + (uint32_t)min(r, 127);
            }
        }
        out |= code << (8 * q);
    }
    tab[wi] = out;
}

cudaError_t launch_skiptab(const uint32_t* finest, int Nf, uint32_t* tab, cudaStream_t st) {
    int nl = 0;
    while ((1 << nl) < Nf) nl++;
    nl += 1;                                   // resolutions 1 .. Nf
    if (nl > kMaxDyadic) return cudaErrorInvalidValue;
    LevelSet ls{};
    ls.n = nl;
    ls.occ[nl - 1] = finest;
    uint32_t* tmp[kMaxDyadic] = {};
    cudaError_t e = cudaSuccess;
    for (int l = nl - 2; l >= 0 && e == cudaSuccess; l--) {   // each level from the next finer
        const int M = 1 << l;
        e = cudaMallocAsync(&tmp[l], (((size_t)M * M * M + 31) / 32) * 4, st);
        if (e == cudaSuccess) e = launch_maxpool_bits(ls.occ[l + 1], 2 * M, tmp[l], M, st);
        ls.occ[l] = tmp[l];
    }
    // Chebyshev distances (MERF_SKIP_DYADIC=1: dyadic cells only, the r01 table, for A/B)
    uint8_t* dist[2] = {nullptr, nullptr};
    const char* env = getenv("MERF_SKIP_DYADIC");
    const bool use_cheb = !(env && env[0] == '1');
    const int64_t cells = (int64_t)Nf * Nf * Nf;
    if (use_cheb && e == cudaSuccess) {
        e = cudaMallocAsync(&dist[0], cells, st);
        if (e == cudaSuccess) e = cudaMallocAsync(&dist[1], cells, st);
        const unsigned g = (unsigned)((cells + 255) / 256);
        if (e == cudaSuccess) cheb_pass_kernel<<<g, 256, 0, st>>>(finest, nullptr, dist[0], Nf, 0);
        if (e == cudaSuccess) cheb_pass_kernel<<<g, 256, 0, st>>>(finest, dist[0], dist[1], Nf, 1);
        if (e == cudaSuccess) cheb_pass_kernel<<<g, 256, 0, st>>>(finest, dist[1], dist[0], Nf, 2);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        const int64_t words = skiptab_words(Nf);
        skiptab_kernel<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(ls, use_cheb ? dist[0] : nullptr, tab);
        e = cudaGetLastError();
    }
    for (int q = 0; q < 2; q++)
        if (dist[q]) cudaFreeAsync(dist[q], st);
    for (int l = 0; l < kMaxDyadic; l++)
        if (tmp[l]) cudaFreeAsync(tmp[l], st);
    return e;
}

// ------------------------------------------------------------------------------------
// Appearance pair layouts (see DevScene): word k of entry u = bytes (c_{2k+1}(u),
// c_{2k+1}(u+1), c_{2k+2}(u), c_{2k+2}(u+1)) with c8 := c0 (density, unused by the pass).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 pair_entry(uint2 a, uint2 b) {
    // a.x = c0 c1 c2 c3, a.y = c4 c5 c6 c7 (texel u); b the same for texel u + 1
    uint4 o;
    o.x = __byte_perm(a.x, b.x, 0x6251);                                   // c1 c1' c2 c2'
    o.y = __byte_perm(__byte_perm(a.x, b.x, 0x0073), __byte_perm(a.y, b.y, 0x0040), 0x5410);   // c3 c3' c4 c4'
    o.z = __byte_perm(a.y, b.y, 0x6251);                                   // c5 c5' c6 c6'
    o.w = __byte_perm(__byte_perm(a.y, b.y, 0x0073), __byte_perm(a.x, b.x, 0x0040), 0x5410);   // c7 c7' c0 c0'
    return o;
}

__global__ void pack_plane_pairs_kernel(const uint2* __restrict__ planes, int R, uint4* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // entry (a, v, u), v <= R
    const int64_t n = (int64_t)3 * (R + 1) * R;
    if (i >= n) return;
    const int u = (int)(i % R);
    const int a_ = (int)(i / ((int64_t)(R + 1) * R));
    const int v = min((int)((i / R) % (R + 1)), R - 1);                  // row R repeats row R - 1
    const int64_t src = ((int64_t)a_ * R + v) * R + u;
    const uint2 a = planes[src];
    const uint2 b = u + 1 < R ? planes[src + 1] : a;  // u + 1 = R repeats texel R - 1 (edge)
    out[i] = pair_entry(a, b);
}

__global__ void pack_atlas_pairs_kernel(const uint2* __restrict__ atlas, int64_t n_blocks, uint4* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // entry (b, z, y, x < 8)
    if (i >= n_blocks * 648) return;
    const int64_t row = i / 8;                                          // (b, z, y)
    const int x = (int)(i % 8);
    const uint2* src = atlas + row * 9 + x;
    out[i] = pair_entry(src[0], src[1]);
}

// The + side apron (local index 8) of a block on the grid's upper edge lies outside the grid;
// the renderer's texel() reads it as the corner past texel L-1, which must repeat texel L-1
// (clamp to edge, D9).  Rewrite those apron voxels of the staging atlas (our device copy of the
// caller's AoS atlas) from the edge voxels before the packed layouts are built.
__global__ void apron_edge_kernel(const int32_t* __restrict__ index, int64_t slots, int nb, int64_t n_blocks,
                                  uint2* __restrict__ atlas) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // (slot, voxel of 9^3)
    if (i >= slots * 729) return;
    const int64_t slot = i / 729;
    const int l = (int)(i - slot * 729);
    const int bx = (int)(slot % nb), by = (int)((slot / nb) % nb), bz = (int)(slot / ((int64_t)nb * nb));
    if (bx != nb - 1 && by != nb - 1 && bz != nb - 1) return;
    const int32_t b = index[slot];
    if (b < 0 || b >= n_blocks) return;
    const int lx = l % 9, ly = (l / 9) % 9, lz = l / 81;
    const int sx = (bx == nb - 1) ? min(lx, 7) : lx, sy = (by == nb - 1) ? min(ly, 7) : ly,
              sz = (bz == nb - 1) ? min(lz, 7) : lz;
    if (sx == lx && sy == ly && sz == lz) return;                    // not an outside-the-grid apron voxel
    atlas[(size_t)b * 729 + l] = atlas[(size_t)b * 729 + (sz * 9 + sy) * 9 + sx];
}

cudaError_t launch_apron_edge(const int32_t* index, int L, int64_t n_blocks, uint8_t* atlas, cudaStream_t st) {
    const int nb = L / 8;
    const int64_t slots = (int64_t)nb * nb * nb;
    if (n_blocks <= 0) return cudaSuccess;
    apron_edge_kernel<<<(unsigned)((slots * 729 + 255) / 256), 256, 0, st>>>(index, slots, nb, n_blocks,
                                                                          reinterpret_cast<uint2*>(atlas));
    return cudaGetLastError();
}

cudaError_t launch_pack_pairs(const uint8_t* planes, int R, uint4* plane_pairs, const uint8_t* atlas,
                              int64_t n_blocks, uint4* atlas_pairs, cudaStream_t st) {
    if (planes && R > 0) {
        const int64_t n = (int64_t)3 * (R + 1) * R;
        pack_plane_pairs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
            reinterpret_cast<const uint2*>(planes), R, plane_pairs);
    }
    if (atlas && n_blocks > 0) {
        const int64_t n = n_blocks * 648;
        pack_atlas_pairs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
            reinterpret_cast<const uint2*>(atlas), n_blocks, atlas_pairs);
    }
    return cudaGetLastError();
}

}  // namespace merf
