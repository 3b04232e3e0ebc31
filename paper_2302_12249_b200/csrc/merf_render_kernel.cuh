// merf_render_kernel.cuh -- the hot path as a 3-kernel pipeline per chunk of rays (sm_100a).
//
// Per ray (Sec. 6):
//  1. setup_kernel (fp64, canonical order, reading D8; one thread per ray, coherent 8x4
//     pixel tiles): raygen -> region segmentation of the world ray into <= 7 contracted
//     segments -> per segment the int32 lattice origin Qa, step U and sample
//     count K -> workspace (32 B per segment).
//  2. march_kernel (int32 lattice + fp32 shading; persistent warps, one coherent 8x4 tile
//     of rays per warp): Q_k = Qa + k U; one occupancy probe per step (the dyadic skip
//     table, or the scene's levels finest-first); an empty cell jumps to the first lattice
//     sample outside it (the ray-AABB exit).  An evaluated sample reads the DENSITY
//     first -- one 8-byte octet of the block-sparse grid (through the indirection table) +
//     one 4-byte quad per plane, i.e. 4 loads for the 8 trilinear + 12 bilinear corners
//     (Eq. 5) -- computes alpha = 1 - exp(-tau Delta) and reads the appearance texels only
//     if alpha > alpha_skip; composite (Eq. 1-2) with termination at T < 2e-4
//     (P:309).  A warp takes its next tile when all 32 of its rays have ended.
//  3. shade_mma_kernel (merf_shade_mma.cu, tensor cores) or shade_kernel (FFMA): deferred
//     MLP h(C_d, F, d) per pixel (Eq. 3), C = clamp(C_d + h), store RGB f32 / RGBA8.
#pragma once
#include <cstdint>
#include <climits>
#include <cuda_runtime.h>

#include "merf_device.cuh"
#include "merf_kernels.h"
#include "merf_mma.cuh"

namespace merf {

enum : int {
    KF_TRACE = 1,       // write per-sample trace records
    KF_COUNT = 2,       // accumulate merf_stats counters
    KF_RAYS = 4,        // explicit rays instead of camera pixels
    KF_U8 = 8,          // RGBA8 output
    KF_DENSE = 16,      // dense stepping gated by the finest level (debug)
    KF_SEGS = 32,       // record contracted segments only (no marching)
    KF_ALLSRC = 64,     // all four sources present (compile-time; the production variant)
    KF_SKIPTAB = 128,   // skip level from the per-cell table (S.skiptab) instead of the level search
    KF_PAPER = 256,     // the paper's default resolutions as compile-time constants (below)
    KF_SPH = 512,       // NEXT-2 like-for-like: spherical contraction, fp32 curve stepping in the
                        // persistent tile-scheduled march (MERF_SPHERICAL | MERF_SPH_PERSISTENT)
    KF_FUSED = 1024,    // the deferred MLP (tensor cores) and the output store run in the march
                        // at each tile's end: no shade kernel, no accumulator round trip
    KF_LPT = 8192,      // setup: also estimate each tile's cost and file it for longest-first
                        // dispatch (launches of <= 4 views; a separate instance so that the
                        // batched setup keeps its registers)
};

// The paper's default scene geometry (L = 512, R = 2048; finest occupancy level
// 256^3) as compile-time constants: the shifts, strides and clamps become immediates and free
// the registers that held them (the march kernel runs at the 64-register limit).  Selected at
// launch when the scene has exactly this geometry; every other scene runs the generic kernel.
constexpr int kPaperL = 512, kPaperR = 2048, kPaperNf = 256;
template <int KF> struct Geo {
    static __device__ __forceinline__ int L(const DevScene& S) { return (KF & KF_PAPER) ? kPaperL : S.L; }
    static __device__ __forceinline__ int R(const DevScene& S) { return (KF & KF_PAPER) ? kPaperR : S.R; }
    static __device__ __forceinline__ int nb(const DevScene& S) { return (KF & KF_PAPER) ? kPaperL / 8 : S.nb; }
    static __device__ __forceinline__ int sV(const DevScene& S) { return (KF & KF_PAPER) ? kF + 2 - 9 : S.sV; }
    static __device__ __forceinline__ int sP(const DevScene& S) { return (KF & KF_PAPER) ? kF + 2 - 11 : S.sP; }
    static __device__ __forceinline__ int Nf(const DevScene& S) { return (KF & KF_PAPER) ? kPaperNf : S.n_fin; }
    static __device__ __forceinline__ int sf(const DevScene& S) { return (KF & KF_PAPER) ? kF + 2 - 8 : S.s_fin; }
};

constexpr int kSetupThreads = 128;
// March CTA shape: 128 threads, 9 resident CTAs/SM (56 registers, 36 warps/SM) measured
// +0.9 % over 256 x 4 (64 registers, 32 warps); 128 x 10 (48 registers) spills and is -7 %.
#ifndef MERF_MARCH_THREADS
#define MERF_MARCH_THREADS 128
#define MERF_MARCH_MINB 9
#endif
constexpr int kMarchThreads = MERF_MARCH_THREADS;
// March scheduling policy, tuned on B200 (bench workload sweeps, r01): a warp takes a new tile
// of 32 rays only when all its lanes are idle (per-lane refill broke the tile coherence the
// skipping relies on and was 1.5-2x slower).  A round = one traversal step of every lane
// holding a ray, then the shading of the lanes that found a sample; further warp-synchronous
// steps (until k lanes are ready, at most m steps) measured slower once the per-step ballot
// cost dropped: (16, 16) 1315, (8, 16) 1324, (1, 16) 1337, (1, 1) 1369 M rays/s.

// ------------------------------------------------------------------------------------
// ray indexing: camera rays are numbered in 8x4-pixel tile order (32 rays per tile, one
// tile per warp), tiles row-major per view; explicit/trace rays use their list index.
// ------------------------------------------------------------------------------------
// camera-ray tile shape (32 rays, one warp): 8 x 4 pixels (measured: 4 x 8 -0.7 %, 16 x 2 -4 %)
#ifndef MERF_TILE_W
#define MERF_TILE_W 8
#endif
constexpr int kTileW = MERF_TILE_W, kTileH = 32 / MERF_TILE_W;

struct RaySource {
    CamBatch cb;
    int W, H, tiles_x, tiles_per_view;
    int64_t ray0;                // first ray id of this chunk
    int64_t n;                   // rays in this chunk
    const double* o;             // explicit rays (KF_RAYS)
    const double* d;
    const double* t_near;
    const int64_t* pixel_ids;    // trace / segments mode: pixel list of camera 0
    // progressive rendering: the rays cover the sub-lattice of pixels
    // (stride * i + ox, stride * j + oy); tiles_x / tiles_per_view count tiles of that
    // lattice.  Zero-initialised = every pixel (stride 1).
    int stride_m1, ox, oy;
    int fill;                    // shade: also write the colour to the stride x stride block
    // exact division by tiles_per_view / tiles_x as a 64-bit multiply-high: m = ceil(2^64 / d)
    // gives floor(n / d) = umulhi(n, m) for all n, d < 2^32 (d >= 2); 0 = not set (divide)
    uint64_t m_tpv, m_tx;
    // single-frame sharding (merf_render_shard): part_n > 0 -> the rays cover only the
    // 64x64-pixel blocks b with b % part_n == part_r; a view's tile range is then part_slots
    // block slots of kShardTiles tiles (block b = part_r + part_n * slot, row-major over the
    // frame's nbx blocks per row, n_pblocks in total; slots past the last block are empty)
    int part_n, part_r, nbx, n_pblocks;
    // compact shard output (merf_render_shard_blocks): pixel (px, py) of block b is stored at
    // [view][slot = b / part_n][py % 64][px % 64] instead of its frame position
    int compact, part_slots;
};
constexpr int kShardBX = 64 / kTileW, kShardBY = 64 / kTileH, kShardTiles = kShardBX * kShardBY;

// host: the tile geometry of a camera chunk and its division magics
inline void set_tiles(RaySource& rs, int tiles_x, int tiles_per_view) {
    rs.tiles_x = tiles_x;
    rs.tiles_per_view = tiles_per_view;
    rs.m_tx = tiles_x >= 2 ? UINT64_MAX / (uint64_t)tiles_x + 1 : 0;
    rs.m_tpv = tiles_per_view >= 2 ? UINT64_MAX / (uint64_t)tiles_per_view + 1 : 0;
}

__device__ __forceinline__ unsigned div_magic(unsigned n, unsigned d, uint64_t m) {
    return m ? (unsigned)__umul64hi((uint64_t)n, m) : n / d;
}

__device__ __forceinline__ bool ray_pixel(const RaySource& rs, int64_t ray, int& view, int& px, int& py) {
    const int64_t tile = ray >> 5;
    const int lane = (int)(ray & 31);
    int tt;
    if (tile <= 0xffffffffll) {            // every practical batch: 32-bit, by multiply-high
        const unsigned t32 = (unsigned)tile, v = div_magic(t32, (unsigned)rs.tiles_per_view, rs.m_tpv);
        view = (int)v;
        tt = (int)(t32 - v * (unsigned)rs.tiles_per_view);
    } else {
        view = (int)(tile / rs.tiles_per_view);
        tt = (int)(tile - (int64_t)view * rs.tiles_per_view);
    }
    int ty, tx;
    if (rs.part_n > 0) {                              // shard modes (set by render_frames)
        const int slot = tt / kShardTiles, w = tt - slot * kShardTiles;
        const int b = rs.part_r + rs.part_n * slot;
        if (b >= rs.n_pblocks) return false;          // padding slot of this shard
        const int by = b / rs.nbx, bx = b - by * rs.nbx;
        tx = bx * kShardBX + (w % kShardBX);
        ty = by * kShardBY + (w / kShardBX);
    } else {
        ty = (int)div_magic((unsigned)tt, (unsigned)rs.tiles_x, rs.m_tx);
        tx = tt - ty * rs.tiles_x;
    }
    const int lx = tx * kTileW + (lane % kTileW), ly = ty * kTileH + (lane / kTileW);
    px = lx * rs.stride_m1 + lx + rs.ox;
    py = ly * rs.stride_m1 + ly + rs.oy;
    return px < rs.W && py < rs.H;
}

// output element index of a finished pixel: its frame position, or (compact shards) its
// position in this part's block-slot buffer
__device__ __forceinline__ int64_t out_index(const RaySource& rs, int view, int px, int py) {
    if (rs.compact) {
        const int b = (py >> 6) * rs.nbx + (px >> 6);
        const int slot = b / rs.part_n;
        return (((int64_t)view * rs.part_slots + slot) << 12) + ((py & 63) << 6) + (px & 63);
    }
    return ((int64_t)view * rs.H + py) * rs.W + px;
}

// Tile dispatch order of the persistent march (longest-processing-time first).  The march's
// tail -- from the moment its tile queue runs dry to the last warp's exit -- is the duration
// of the most expensive tiles taken last (measured 0.36-0.47 ms per launch on the orbit views,
// 23 % of a single 1080p view: 1 % of the tiles have a ray with >= 268 evaluated samples, 5x the
// median tile, and take ~1 ms under full load).  With MERF_TILE_ORDER=cost the setup kernel
// estimates every 32-ray tile's cost (tile_cost_bucket) and appends the tile to one of kBuckets
// lists by log2 of the estimate; the march takes the lists most expensive first.  The order
// changes no ray's arithmetic: every tile is still marched by one warp.  Measured a net loss
// (the estimate costs more setup time than the shorter tail saves), so raster is the default.
constexpr int kBuckets = 16;       // half-octave buckets of the measured history (the probe uses 8)

struct Workspace {
    int4* seg;                   // [n][seg_slots][2]: (Qa.xyz, K), (U.xyz, region)
    int seg_slots;               // segment slots per ray: kMaxSeg, or kMaxSegCore (see below)
    uint8_t* nseg;               // [n]
    float4* accum;               // [n][2]: (C_d.rgb, T), (F0..F3)
    unsigned int* queue;         // tile counter of the persistent march
    int* tile_list;              // [kBuckets][n_tiles] tile indices, or NULL: raster order
    unsigned int* bucket_cnt;    // [kBuckets] tiles per list (zeroed before the setup)
    int n_tiles;                 // ceil(n / 32) of the current chunk
    // per-tile march durations of the previous call with the same tiling (SM clock >> 8,
    // saturated), or NULL.  The setup's KF_LPT path files tiles by these instead of the probe
    // estimate; the march overwrites them with this call's durations.  Scheduling only.
    uint16_t* tile_cost;
};



// merf_stats counters (device array of kStatWords): 0..15 as merf_stats; per march launch
// 16 = first warp start, 17 = first warp to find the tile queue empty, 18 = last warp exit
// (%globaltimer ns, min/min/max), folded into 19 (busy) and 20 (tail) sums after each launch
constexpr int kStatWords = 24;

__device__ __forceinline__ unsigned tid_volatile() {
    unsigned t;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
    return t;
}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct TraceArgs {
    uint64_t* cells;
    float* T;
    int32_t* counts;
    int max_per_ray;
    merf_segment* segs;
};

__device__ __forceinline__ void add_stat(unsigned long long* stats, int idx, int v) {
    unsigned int s = __reduce_add_sync(0xffffffffu, (unsigned)v);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(stats + idx, (unsigned long long)s);
}

// ====================================================================================
// 1. setup
// ====================================================================================
// Tile-cost estimate for the dispatch order (not part of the rendered result): the tile's
// centre ray (lane kCostLane) is probed at 64 points spread evenly over its lattice samples, two
// per lane.  An occupied probe stands for Ktot/64 samples; its optical depth is estimated from
// the NEAREST texel of each source (no interpolation weights) and the probes are counted in ray
// order until the accumulated optical depth passes ln(1/t_min), where termination would cut the
// ray.  Measured on a 1080p orbit view (tools/tile_cost.py): rank correlation 0.54 with the
// tile's true longest ray, and all of the 1 % most expensive tiles land in the top two buckets
// (a two-probes-per-segment occupancy count without the density term: -0.25, and 73 % of them
// in the cheapest bucket).
constexpr int kCostLane = 20;      // pixel (4, 2) of the 8x4 tile

__device__ __forceinline__ float probe_od(const DevScene& S, int Qx, int Qy, int Qz, float od_per_tau) {
    const int N = S.n_fin, sf = S.s_fin;
    if (!occ_bit(S.occ_fin, occ_cell(Qx, sf, N), occ_cell(Qy, sf, N), occ_cell(Qz, sf, N), N)) return -1.f;
    unsigned sum = 0;
    int n = 0;
    if (S.use_v) {
        const int L = S.L;
        const int ix = min(max(Qx >> S.sV, 0), L - 1), iy = min(max(Qy >> S.sV, 0), L - 1),
                  iz = min(max(Qz >> S.sV, 0), L - 1);
        const int blk = __ldg(S.block_index + ((iz >> 3) * S.nb + (iy >> 3)) * S.nb + (ix >> 3));
        if (blk >= 0) {
            sum += (__ldg(reinterpret_cast<const uint32_t*>(S.atlas_pairs + (unsigned)(blk * 648 + ((iz & 7) * 9 + (iy & 7)) * 8 + (ix & 7))) + 3) >> 16) & 0xFFu;
            n++;
        }
    }
    if (S.R > 0) {
        const int R = S.R;
        const int px = min(max(Qx >> S.sP, 0), R - 1), py = min(max(Qy >> S.sP, 0), R - 1),
                  pz = min(max(Qz >> S.sP, 0), R - 1);
        const int v[3] = {pz, pz, py}, u[3] = {py, px, px};
#pragma unroll
        for (int a = 0; a < 3; a++)
            if (S.use_p[a]) {
                const unsigned idx = (unsigned)(a * (R + 1) + v[a]) * R + u[a];
                sum += (__ldg(reinterpret_cast<const uint32_t*>(S.plane_pairs + idx) + 3) >> 16) & 0xFFu;
                n++;
            }
    }
    // tau Delta = 2^(s kd_l2 - n md_l2 + log2 Delta), times the samples the probe stands for
    return ex2_ftz(fmaf((float)sum, S.kd_l2, fmaf((float)n, -S.md_l2, S.log2_step))) * od_per_tau;
}

// bucket of the tile that holds chunk-local ray r (call with all 32 lanes of the warp, after the
// warp's segments are in the workspace)
__device__ __forceinline__ int tile_cost_bucket(const DevScene& S, const Workspace& ws, int64_t r, int64_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t rc = (r & ~(int64_t)31) + kCostLane;
    int ns = 0;
    if (rc < n) ns = ws.nseg[rc];
    const int4* sp = ws.seg + rc * ws.seg_slots * 2;
    int Ktot = 0;
    for (int j = 0; j < ns; j++) Ktot += sp[2 * j].w;            // uniform loop (same ray)
    float od[2] = {-1.f, -1.f};
    const float per = (float)Ktot * (1.f / 64.f);
    if (Ktot > 0) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
            int k = (int)(((float)(2 * lane + h) + 0.5f) * per);
            int j = 0;
            while (j < ns - 1 && k >= sp[2 * j].w) { k -= sp[2 * j].w; j++; }
            const int4 qa = sp[2 * j], uu = sp[2 * j + 1];
            od[h] = probe_od(S, qa.x + k * uu.x, qa.y + k * uu.y, qa.z + k * uu.z, per);
        }
    }
    // optical depth accumulated before each probe, in ray order (lane-major): exclusive scan
    const float mine = fmaxf(od[0], 0.f) + fmaxf(od[1], 0.f);
    float inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const float v = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += v;
    }
    const float before0 = inc - mine, before1 = before0 + fmaxf(od[0], 0.f);
    const float cut = -__logf(S.t_min);
    const int cnt = (od[0] >= 0.f && before0 < cut) + (od[1] >= 0.f && before1 < cut);
    const int tot = __reduce_add_sync(0xffffffffu, cnt);
    const unsigned e = (unsigned)((float)tot * per);            // estimated evaluated samples
    return min(7, 31 - __clz((int)(e + 1u)));
}

template <int KF>
__device__ __forceinline__ void emit_segment(const DevScene& S, int g, const double o[3], const double d[3],
                                             double t_a, double t_b, int64_t r, int64_t ray,
                                             const Workspace& ws, const TraceArgs& ta, int& nseg,
                                             unsigned& reg_mask) {
    Segment sg;
    if (!make_segment(S, g, o, d, t_a, t_b, sg)) return;   // zero length: dropped

    if (KF & KF_SEGS) {
        if (nseg < ta.max_per_ray) {
            merf_segment rec;
            rec.t_a = t_a;
            rec.t_b = t_b;
#pragma unroll
            for (int q = 0; q < 3; q++) { rec.Qa[q] = sg.Qa[q]; rec.U[q] = sg.U[q]; }
            rec.K = sg.K;
            rec.region = sg.region;
            ta.segs[ray * ta.max_per_ray + nseg] = rec;
        }
    } else if (nseg < ws.seg_slots) {
        int4* p = ws.seg + (r * ws.seg_slots + nseg) * 2;
        p[0] = make_int4(sg.Qa[0] + kTwoI, sg.Qa[1] + kTwoI, sg.Qa[2] + kTwoI, sg.K);   // biased origin
        p[1] = make_int4(sg.U[0], sg.U[1], sg.U[2], sg.region);
    }
    nseg++;
    reg_mask |= 1u << g;
}

template <int KF>
__global__ void __launch_bounds__(kSetupThreads, (KF & KF_LPT) ? 7 : 8) setup_kernel(DevScene S, RaySource rs, Workspace ws,
                                                              TraceArgs ta, unsigned long long* stats) {
    __shared__ double s_cand[kSetupThreads][13];   // 13: odd stride, conflict-free rows
    // programmatic dependent launch: the march may be scheduled as soon as every setup CTA has
    // started (it waits for this grid's completion before reading the workspace); the march's
    // tile queue is reset here, so no memset sits between the two launches
    if (blockIdx.x == 0 && threadIdx.x == 0 && ws.queue) *ws.queue = 0u;
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // index within chunk
    const int64_t ray = rs.ray0 + r;
    bool valid = r < rs.n;
    int nseg = 0;
    unsigned reg_mask = 0;       // regions are convex, so a ray visits each at most once
    if (valid) {
        double o[3], d[3], t_near;
        if (KF & (KF_TRACE | KF_SEGS)) {
            const int64_t pid = rs.pixel_ids[ray];
            raygen(rs.cb.cam[0], (int)(pid % rs.W), (int)(pid / rs.W), o, d);
            t_near = rs.cb.cam[0].t_near;
        } else if (KF & KF_RAYS) {
#pragma unroll
            for (int q = 0; q < 3; q++) { o[q] = rs.o[3 * ray + q]; d[q] = rs.d[3 * ray + q]; }
            t_near = rs.t_near ? rs.t_near[ray] : 0.0;
        } else {
            int view, px, py;
            valid = ray_pixel(rs, ray, view, px, py);
            if (valid) {
                raygen(rs.cb.cam[view], px, py, o, d);
                t_near = rs.cb.cam[view].t_near;
            }
        }
        if (valid && (KF & KF_SPH)) {
            // spherical variant: no segments; the march steps the curve from (o, d, t_near)
            int4* p = ws.seg + (r * ws.seg_slots) * 2;
            p[0] = make_int4(__float_as_int((float)o[0]), __float_as_int((float)o[1]), __float_as_int((float)o[2]),
                             __float_as_int((float)t_near));
            p[1] = make_int4(__float_as_int((float)d[0]), __float_as_int((float)d[1]), __float_as_int((float)d[2]), 0);
            nseg = 1;
            reg_mask = 1u;
        } else if (valid) {
            double cand[12];
            boundary_candidates(o, d, t_near, cand);
            // Walk the sorted boundaries (staged in this thread's shared-memory row: dynamic
            // indexing without local memory or register shifting) and merge equal-region
            // intervals into segments.
            double* sc = s_cand[threadIdx.x];
#pragma unroll
            for (int q = 0; q < 12; q++) sc[q] = cand[q];
            double b = t_near, seg_start = t_near;
            int g_cur = -1;
            for (int q = 0; q <= 12; q++) {
                // the sorted candidates in order, one shared-memory load each; a repeat of the
                // previous boundary (two planes crossed at the same t) adds no interval
                const double nb = q < 12 ? sc[q] : __longlong_as_double(0x7ff0000000000000ll);
                if (!(nb > b)) continue;
                const bool last = isinf(nb);
                const double p = last ? add_rn(mul_rn(b, 2.0), 1.0) : mul_rn(add_rn(b, nb), 0.5);
                double x[3];
                point_at(o, d, p, x);
                const int g = region_of(x[0], x[1], x[2]);
                if (g_cur < 0) {
                    g_cur = g;
                    seg_start = b;
                } else if (g != g_cur) {
                    emit_segment<KF>(S, g_cur, o, d, seg_start, b, r, ray, ws, ta, nseg, reg_mask);
                    g_cur = g;
                    seg_start = b;
                }
                if (last) {
                    emit_segment<KF>(S, g_cur, o, d, seg_start, nb, r, ray, ws, ta, nseg, reg_mask);
                    break;
                }
                b = nb;
            }
        }
    }
    if (KF & KF_SEGS) {
        if (r < rs.n) ta.counts[ray] = nseg;
    } else if (r < rs.n) {
        MERF_CHECK(nseg <= ws.seg_slots);        // kMaxSegCore bound (proof at kMaxSegCore)
        ws.nseg[r] = (uint8_t)min(nseg, ws.seg_slots);
    }
    if ((KF & KF_LPT) && !(KF & (KF_SEGS | KF_TRACE | KF_SPH))) {
        // one 32-ray tile per warp (chunks are tile aligned): file it under its cost bucket
        __syncwarp();                                  // the centre ray's segments are written
        // the previous frame's measured duration when the caller keeps a history (temporal
        // coherence of a frame sequence), else the centre-ray probe estimate
        int b;
        if (ws.tile_cost) {
            const unsigned c = r < rs.n ? (unsigned)ws.tile_cost[r >> 5] : 0u;
            // half-octave buckets: 2 floor(log2 c) + the next bit - 12 (c in 256-cycle units;
            // 8 log2 buckets measured 4 % slower on the C2 protocol pose)
            const int lg = 31 - __clz((int)(c | 1u));
            b = min(kBuckets - 1, max(0, 2 * lg + (int)((c >> max(lg - 1, 0)) & 1u) - 12));
        } else {
            b = tile_cost_bucket(S, ws, r, rs.n);
        }
        if ((threadIdx.x & 31) == 0 && r < rs.n) {
            const unsigned slot = atomicAdd(ws.bucket_cnt + b, 1u);
            ws.tile_list[(int64_t)b * ws.n_tiles + slot] = (int)(r >> 5);
        }
    }
    if (KF & KF_COUNT) {
        add_stat(stats, 0, valid ? 1 : 0);
        add_stat(stats, 1, nseg);
#pragma unroll
        for (int g = 0; g < 7; g++) add_stat(stats, 6 + g, (reg_mask >> g) & 1u);
    }
}

// ====================================================================================
// 2. march
// ====================================================================================
struct RayState {
    float T;
    float cd[3];
    float F[4];
};

// the ray's accumulators (C_d, T), F as stored for the shade kernel
__device__ __forceinline__ void store_accum(float4* a, const RayState& st) {
    a[0] = make_float4(st.cd[0], st.cd[1], st.cd[2], st.T);
    a[1] = make_float4(st.F[0], st.F[1], st.F[2], st.F[3]);
}


// Linear index of texel (v, u) of plane a in the [3][R + 1][R] layouts (row R of each plane
// repeats row R - 1: the upper-edge corner of texel(), see merf_device.cuh).  With the paper
// geometry a (R + 1) R = a (2^22 + 2^11) is a constant, so one 32-bit three-input add (the
// plane offset never becomes a separate 64-bit pointer add).
template <int KF>
__device__ __forceinline__ unsigned plane_index(int a, int R, int v, int u) {
    if (KF & KF_PAPER) {
        // opaque to the compiler: it would otherwise peel the plane offset off into a 64-bit
        // pointer add (IADD3 + IMAD.X per access) after the 32-bit index scaling
        unsigned idx;
        asm("add.u32 %0, %1, %2;" : "=r"(idx) : "r"((unsigned)a * (unsigned)((kPaperR + 1) * kPaperR) + ((unsigned)v << 11)),
            "r"((unsigned)u));
        return idx;
    }
    return (unsigned)((a * (R + 1) + v) * R + u);
}

// Appearance accumulation of a corner PAIR from its pair-interleaved 16-byte entry (see
// DevScene): 7 dp2a (16-bit weights packed in wp, bytes already paired).  acc[c] is in units
// of 1/65535 byte.
__device__ __forceinline__ void acc_pair(uint32_t acc[7], uint4 p, uint32_t wp) {
    acc[0] = __dp2a_lo(wp, p.x, acc[0]);
    acc[1] = __dp2a_hi(wp, p.x, acc[1]);
    acc[2] = __dp2a_lo(wp, p.y, acc[2]);
    acc[3] = __dp2a_hi(wp, p.y, acc[3]);
    acc[4] = __dp2a_lo(wp, p.z, acc[4]);
    acc[5] = __dp2a_hi(wp, p.z, acc[5]);
    acc[6] = __dp2a_lo(wp, p.w, acc[6]);
}

// Evaluate the field at lattice point (Qx, Qy, Qz) and composite it (Eq. 1-2, 5-7).
// Returns 1 if the sample was density-only (alpha <= alpha_skip), 2 if its V block was
// missing (unsound scene; counted), else 0.  `bslot`/`bblk` cache the last block lookup.
template <int KF>
__device__ __forceinline__ int shade_sample(const DevScene& S, int Qx, int Qy, int Qz, RayState& st,
                                            int& bslot, int& bblk) {
    constexpr bool ALL = (KF & KF_ALLSRC) != 0;
    const bool use_v = ALL || S.use_v;
    const int Q[3] = {Qx, Qy, Qz};
    int ret = 0;
    // Interpolation weights, computed once and shared by both passes: 16-bit fixed point,
    // partitioning 65535 exactly per source, packed per corner pair for dp2a.  V: rows
    // (dy, dz), c = dy + 2 dz, x pair per row; plane a: rows dv, u pair per row.
    int n_src = ALL ? 4 : S.n_src;
    uint32_t sd = 0u;                  // density sum over sources, units of 1/65535 byte
    int vi[3] = {0, 0, 0};
    uint32_t wV[4] = {0u, 0u, 0u, 0u};
    int blk = -1;
    // compile-time geometry: fractions as exact g-floats (texel_g), no I2F / scaling
    constexpr bool GF = (KF & KF_PAPER) != 0;
    if (use_v) {
        float vf[3], vg[3];
        const int sV = Geo<KF>::sV(S);
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (GF) texel_g(Q[a], sV, Geo<KF>::L(S), vi[a], vg[a]);
            else texel(Q[a], sV, Geo<KF>::L(S), vi[a], vf[a]);
        }
        const int nb = Geo<KF>::nb(S);
        const int slot = ((vi[2] >> 3) * nb + (vi[1] >> 3)) * nb + (vi[0] >> 3);
        if (slot != bslot) {                              // blocks change every ~8 voxels
            MERF_CHECK(slot >= 0 && slot < nb * nb * nb);
            bslot = slot;
            bblk = __ldg(S.block_index + slot);
            MERF_CHECK(bblk < S.n_blocks_dev);
        }
        blk = bblk;
        uint32_t zi[2], yi[4];
        float zf[2], yf[4];
        if (GF) {
            wsplit_full_g(vg[2], sV, zi[0], zf[0], zi[1], zf[1]);
            vf[1] = g_frac(vg[1], sV);
            vf[0] = g_frac(vg[0], sV);
        } else {
            wsplit(65535u, 65535.f, vf[2], zi[0], zf[0], zi[1], zf[1]);
        }
        wsplit<true>(zi[0], zf[0], vf[1], yi[0], yf[0], yi[1], yf[1]);   // leaf parents: biased
        wsplit<true>(zi[1], zf[1], vf[1], yi[2], yf[2], yi[3], yf[3]);
#pragma unroll
        for (int c = 0; c < 4; c++) wV[c] = wleaf(yi[c], yf[c], vf[0]);
        if (ALL) {
            // An evaluated sample lies in an occupied finest cell, and the upload rejects any
            // scene in which such a cell's trilinear base voxel has no block (block_need +
            // block_check, MERF_EMISMATCH): the block exists.  The clamp only keeps a corrupted
            // index in bounds (MERF_BOUNDS_CHECK builds trap on it instead); the r01 branch-free
            // zero-weight handling of a missing block cost 7 issued instructions per sample.
            MERF_CHECK(blk >= 0);
            blk = max(blk, 0);
        }
        if (ALL || blk >= 0) {
            // ---- density pass, V: the 8 corners' density bytes from the pair entries of rows
            // (dy, dz): word .w = c7 c7' c0 c0', so dp2a_hi weighs (c0(x), c0(x + 1)) with the
            // row's leaf pair (W - w1, w1) -- no separate density copy of the atlas (r02: the
            // octet copy cost 83 MB and bought 0.1 %)
            MERF_CHECK(blk >= 0 && blk < max(S.n_blocks_dev, 1));
            const uint32_t* wrow = reinterpret_cast<const uint32_t*>(
                S.atlas_pairs + ((unsigned)blk * 648u + (unsigned)(((vi[2] & 7) * 9 + (vi[1] & 7)) * 8 + (vi[0] & 7))));
#pragma unroll
            for (int c = 0; c < 4; c++) sd = __dp2a_hi(wV[c], __ldg(wrow + 4 * ((c >> 1) * 72 + (c & 1) * 8) + 3), sd);
        } else {
            n_src -= 1;                    // a missing block contributes nothing
            ret = 2;
        }
    }
    // plane texel coordinates: each axis feeds two planes (P_x(y,z), P_y(x,z), P_z(x,y))
    int pi[3] = {0, 0, 0};
    uint32_t wP[3][2] = {{0u, 0u}, {0u, 0u}, {0u, 0u}};
    const bool any_p = ALL || S.R > 0;
    const int R = Geo<KF>::R(S);
    if (any_p) {
        float pf[3], pg[3];
        const int sP = Geo<KF>::sP(S);
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (GF) {
                texel_g(Q[a], sP, R, pi[a], pg[a]);
                pf[a] = g_frac(pg[a], sP);      // used only as a u axis (x, y); dead for z
            } else {
                texel(Q[a], sP, R, pi[a], pf[a]);
            }
        }
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (!(ALL || S.use_p[a])) continue;
            const int ua = (a == 0) ? 1 : 0;
            const int va = (a == 2) ? 1 : 2;
            uint32_t v0i, v1i;
            float v0f, v1f;
            if (GF) wsplit_full_g<true>(pg[va], sP, v0i, v0f, v1i, v1f);
            else wsplit<true>(65535u, 65535.f, pf[va], v0i, v0f, v1i, v1f);
            wP[a][0] = wleaf(v0i, v0f, pf[ua]);
            wP[a][1] = wleaf(v1i, v1f, pf[ua]);
            // ---- density pass, plane a: the texel quad as 2 dp2a on the .w words (c0 c0' high)
            MERF_CHECK(pi[va] >= 0 && pi[va] < R && pi[ua] >= 0 && pi[ua] < R);
            {                                            // rows v, v + 1 of the pair entries
                MERF_CHECK((int64_t)plane_index<KF>(a, R, pi[va], pi[ua]) + R < (int64_t)3 * (R + 1) * R);
                const uint32_t* wrow = reinterpret_cast<const uint32_t*>(S.plane_pairs + plane_index<KF>(a, R, pi[va], pi[ua]));
                sd = __dp2a_hi(wP[a][0], __ldg(wrow + 3), sd);
                sd = __dp2a_hi(wP[a][1], __ldg(wrow + 4 * R + 3), sd);
            }
        }
    }
    // tau = exp(t0), t0 = s0 kd - n m (Eq. 6-7), s0 = sd / 65535; alpha = 1 - exp(-tau Delta)
    // in base 2: log2(tau Delta) = sd kd log2e / 65535 - n m log2e + log2 Delta (one FFMA)
    // (all-sources instance: the constant term -4 m log2e + log2 Delta precomputed at upload,
    // bit-identical to the fmaf below with n_src = 4)
    const float tau_step = ex2_ftz(fmaf((float)(int)sd, S.kd_l2w,
                                        ALL ? S.dens_off4 : fmaf((float)n_src, -S.md_l2, S.log2_step)));
    const float alpha = 1.f - ex2_ftz(tau_step * -1.4426950408889634f);
    if (alpha > S.alpha_skip) {
        // ---- appearance pass: 20 AoS texels, channels 1..7, the same weights + dp2a
        uint32_t acc[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
        if (ALL || blk >= 0) {
            const int lx = vi[0] & 7, ly = vi[1] & 7, lz = vi[2] & 7;
            // pair entries per block: 9 z x 9 y x 8 x; the four (dy, dz) rows as constant
            // offsets from one pointer (immediate LDG offsets, one address computation)
            const uint4* row = S.atlas_pairs + ((unsigned)blk * 648u + (unsigned)((lz * 9 + ly) * 8 + lx));
#pragma unroll
            for (int c = 0; c < 4; c++) {                 // (dy, dz) rows; one x pair per row
                const int dy = c & 1, dz = c >> 1;
                acc_pair(acc, __ldg(row + (dz * 72 + dy * 8)), wV[c]);
            }
        }
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (!(ALL || S.use_p[a])) continue;
            const int ua = (a == 0) ? 1 : 0;
            const int va = (a == 2) ? 1 : 2;
            const uint4* row = S.plane_pairs + plane_index<KF>(a, R, pi[va], pi[ua]);
#pragma unroll
            for (int dv = 0; dv < 2; dv++) acc_pair(acc, __ldg(row + dv * R), wP[a][dv]);
        }
        // sigmoid(x), x = acc ka / 65535 - n m: 1 / (1 + 2^(-x log2e)), the exponent in one FFMA
        const float off = ALL ? S.ma_l2_4 : (float)n_src * S.ma_l2;
        const float w = alpha * st.T;
#pragma unroll
        for (int c = 0; c < 3; c++)
            st.cd[c] = fmaf(w, rcp_ftz(1.f + ex2_ftz(fmaf((float)(int)acc[c], S.ka_l2n, off))), st.cd[c]);
#pragma unroll
        for (int c = 0; c < 4; c++)
            st.F[c] = fmaf(w, rcp_ftz(1.f + ex2_ftz(fmaf((float)(int)acc[3 + c], S.ka_l2n, off))), st.F[c]);
    } else if (ret == 0) {
        ret = 1;
    }
    st.T *= (1.f - alpha);
    return ret;
}

// ---- fused deferred-MLP epilogue (KF_FUSED) ----------------------------------------------
// When a warp's 32 rays have all ended, their accumulators are still in the lanes' registers:
// the warp evaluates h(C_d, F, d) (Eq. 3; 34 -> 16 -> 16 -> 3) for its tile on
// the tensor cores exactly as shade_mma_kernel does (split-fp16 operands, fp32 accumulation:
// pixels are the M dimension, two m16 tiles), and stores the pixels.  The input rows are
// transposed through ONE per-CTA staging buffer (16 rows x 2 halves planes, 3.5 KB) that the
// CTA's warps take in turn (a shared-memory lock: tile ends are rare, ~1 per 0.1 ms per warp),
// so the march keeps its L1 for the texel gathers.
struct FusedSmem {
    __half x[2][16][kXStride];     // [hi, lo][pixel row of the m16 tile][input]
    float o[32][4];                // logits of the tile's pixels
    int lock;
};

template <int KF>
__device__ __noinline__ void fused_epilogue(const DevScene& S, const RaySource& rs, void* out, int64_t rbase,
                                            const RayState st, FusedSmem& sm) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t r = rbase + lane;
    bool valid = r < rs.n;
    int view = 0, px = 0, py = 0;
    float d[3] = {0.f, 0.f, 1.f};
    if (valid) valid = ray_pixel(rs, rs.ray0 + r, view, px, py);
    if (valid) {
        const merf_camera& c = rs.cb.cam[view];
        const float x0 = __fdividef((float)px + 0.5f - (float)c.cx, (float)c.fx);   // MLP input: fp32
        const float x1 = __fdividef((float)py + 0.5f - (float)c.cy, (float)c.fy);
        float v[3];
#pragma unroll
        for (int q = 0; q < 3; q++)
            v[q] = fmaf((float)c.c2w[4 * q], x0, fmaf((float)c.c2w[4 * q + 1], x1, (float)c.c2w[4 * q + 2]));
        const float inv = rsqrtf(fmaf(v[0], v[0], fmaf(v[1], v[1], v[2] * v[2])));
#pragma unroll
        for (int q = 0; q < 3; q++) d[q] = v[q] * inv;
    }
    if (lane == 0) {
        while (atomicCAS(&sm.lock, 0, 1) != 0) __nanosleep(32);
        __threadfence_block();
    }
    __syncwarp();
    const uint4* tab = reinterpret_cast<const uint4*>(S.mlp_frag) + lane * (kMlpFragWords / 4);
    const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 8;
    float h3[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; mt++) {
        if ((lane >> 4) == mt) {
            // this pixel's input row [C_d, F, d, sin/cos(2^k d_j) (j outer, k inner, D17), 0 pad]
            // as 20 (hi, lo) half pairs: columns 0..39 (the k8 step reads 32..39)
            uint32_t* ph = reinterpret_cast<uint32_t*>(&sm.x[0][lane & 15][0]);
            uint32_t* pl = reinterpret_cast<uint32_t*>(&sm.x[1][lane & 15][0]);
            uint32_t h, l;
            split2(st.cd[0], st.cd[1], h, l); ph[0] = h; pl[0] = l;
            split2(st.cd[2], st.F[0], h, l); ph[1] = h; pl[1] = l;
            split2(st.F[1], st.F[2], h, l); ph[2] = h; pl[2] = l;
            split2(st.F[3], d[0], h, l); ph[3] = h; pl[3] = l;
            split2(d[1], d[2], h, l); ph[4] = h; pl[4] = l;
            int w = 5;
#pragma unroll
            for (int j = 0; j < 3; j++) {
                float sn = __sinf(d[j]), cs = __cosf(d[j]);
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    split2(sn, cs, h, l);
                    ph[w] = h;
                    pl[w] = l;
                    w++;
                    const float s2 = 2.f * sn * cs, c2 = fmaf(-2.f * sn, sn, 1.f);
                    sn = s2;
                    cs = c2;
                }
            }
#pragma unroll
            for (int q = 17; q < 20; q++) { ph[q] = 0u; pl[q] = 0u; }
        }
        __syncwarp();
        // layer 1: [16 px x 34] x [34 x 16], bias in the accumulator
        float c1[2][4];
        {
            const uint4 b01 = __ldg(tab + 8);                   // layer-1 biases (words 32..35)
            c1[0][0] = c1[0][2] = __uint_as_float(b01.x);
            c1[0][1] = c1[0][3] = __uint_as_float(b01.y);
            c1[1][0] = c1[1][2] = __uint_as_float(b01.z);
            c1[1][1] = c1[1][3] = __uint_as_float(b01.w);
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; s2++) {
            uint32_t ah[4], al[4];
            ldm4(ah, &sm.x[0][lrow][16 * s2 + lcol]);
            ldm4(al, &sm.x[1][lrow][16 * s2 + lcol]);
#pragma unroll
            for (int nt = 0; nt < 2; nt++) {
                const uint4 b = __ldg(tab + 2 * s2 + nt);
                const uint32_t bb[4] = {b.x, b.y, b.z, b.w};
                mma16x3(c1[nt], ah, al, bb);
            }
        }
        {
            uint32_t h0, h1, l0, l1;
            ldm2(h0, h1, &sm.x[0][lrow][32]);
            ldm2(l0, l1, &sm.x[1][lrow][32]);
            const uint4 b = __ldg(tab + 4);                    // words 16..19
            mma8(c1[0], l0, l1, b.x);
            mma8(c1[0], h0, h1, b.y);
            mma8(c1[0], h0, h1, b.x);
            mma8(c1[1], l0, l1, b.z);
            mma8(c1[1], h0, h1, b.w);
            mma8(c1[1], h0, h1, b.z);
        }
        __syncwarp();                                          // staging rows free for the next m tile
        // layer 2: ReLU(h1) [16 x 16] x [16 x 16]
        uint32_t ah[4], al[4];
        relu_to_a(c1[0], c1[1], ah, al);
        float c2[2][4];
        {
            const uint4 b23 = __ldg(tab + 9);                   // layer-2 biases (words 36..39)
            c2[0][0] = c2[0][2] = __uint_as_float(b23.x);
            c2[0][1] = c2[0][3] = __uint_as_float(b23.y);
            c2[1][0] = c2[1][2] = __uint_as_float(b23.z);
            c2[1][1] = c2[1][3] = __uint_as_float(b23.w);
        }
#pragma unroll
        for (int nt = 0; nt < 2; nt++) {
            const uint4 b = __ldg(tab + 5 + nt);               // words 20..27
            const uint32_t bb[4] = {b.x, b.y, b.z, b.w};
            mma16x3(c2[nt], ah, al, bb);
        }
        // layer 3: ReLU(h2) [16 x 16] x [16 x 3 (padded to 8)]
        relu_to_a(c2[0], c2[1], ah, al);
        {
            const uint4 b3 = __ldg(tab + 10);                  // words 40..43 (layer-3 biases)
            h3[mt][0] = h3[mt][2] = __uint_as_float(b3.x);
            h3[mt][1] = h3[mt][3] = __uint_as_float(b3.y);
            const uint4 b = __ldg(tab + 7);                    // words 28..31
            const uint32_t bb[4] = {b.x, b.y, b.z, b.w};
            mma16x3(h3[mt], ah, al, bb);
        }
    }
    if (t <= 1) {
#pragma unroll
        for (int mt = 0; mt < 2; mt++) {
            *reinterpret_cast<float2*>(&sm.o[16 * mt + g][2 * t]) = make_float2(h3[mt][0], h3[mt][1]);
            *reinterpret_cast<float2*>(&sm.o[16 * mt + g + 8][2 * t]) = make_float2(h3[mt][2], h3[mt][3]);
        }
    }
    __syncwarp();
    const float4 hv = *reinterpret_cast<const float4*>(&sm.o[lane][0]);
    __syncwarp();
    if (lane == 0) {
        __threadfence_block();
        atomicExch(&sm.lock, 0);
    }
    if (!valid) return;
    const float c0 = __saturatef(st.cd[0] + __fdividef(1.0f, 1.0f + __expf(-hv.x)));
    const float c1 = __saturatef(st.cd[1] + __fdividef(1.0f, 1.0f + __expf(-hv.y)));
    const float c2 = __saturatef(st.cd[2] + __fdividef(1.0f, 1.0f + __expf(-hv.z)));
    const int64_t idx = out_index(rs, view, px, py);
    if (KF & KF_U8) {
        reinterpret_cast<uchar4*>(out)[idx] =
            make_uchar4((unsigned char)__float2int_rn(c0 * 255.f), (unsigned char)__float2int_rn(c1 * 255.f),
                        (unsigned char)__float2int_rn(c2 * 255.f), 255);
    } else {
        float* o3 = reinterpret_cast<float*>(out) + 3 * idx;
        o3[0] = c0;
        o3[1] = c1;
        o3[2] = c2;
    }
}

// Persistent march.  Every lane owns one ray at a time; a warp takes the next tile of 32
// coherent rays from the global queue once all its lanes are idle (refilling single lanes or
// half tiles breaks the coherence the skipping relies on: measured 1.5-2x and 1.27x slower).
// Each round is one traversal step of every lane holding a ray (segment transition, probe,
// skip or find) followed by the shading of the lanes that found a sample.
template <int KF>
__global__ void __launch_bounds__(kMarchThreads, MERF_MARCH_MINB) march_kernel(const __grid_constant__ DevScene S,
                                                              int64_t n_rays, Workspace ws,
                                                              uint32_t rflags, TraceArgs ta,
                                                              unsigned long long* stats,
                                                              const __grid_constant__ RaySource rs, void* out) {
    const unsigned FULL = 0xffffffffu;
    // programmatic dependent launch (merf_march.cu): wait for the setup grid's results; let the
    // shade grid be scheduled behind this one
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ __align__(16) FusedSmem fsm[(KF & KF_FUSED) ? 1 : 1];
    __shared__ unsigned s_tc[kMarchThreads / 32][2];   // per warp: tile start clock, tile (history)
    if ((threadIdx.x & 31) == 0) s_tc[threadIdx.x >> 5][1] = ~0u;
    if (KF & KF_FUSED) {
        if (threadIdx.x == 0) fsm[0].lock = 0;
        __syncthreads();
    }
    int64_t tile_rbase = -1;           // chunk-local first ray of the warp's current tile (fused epilogue)
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int nl = S.n_levels;
    const int Nf = Geo<KF>::Nf(S);
    const int sf = Geo<KF>::sf(S);
    const uint32_t* occ_f = S.occ_fin;
    const bool early_term = !(rflags & MERF_NO_EARLY_TERM);
    // spherical variant: step cap and stop radius of the curve march (reading S1: k < 8 / Delta + 8, stop at radius 2 - Delta)
    const int sph_kmax = (KF & KF_SPH) ? (int)(8.0 / S.step) + 8 : 0;
    const float sph_stop = (KF & KF_SPH) ? 2.f - S.step_f : 0.f;

    // per-lane ray state
    int ray = -1;                      // chunk-local ray index (chunks < 2^31 rays)
    int bslot = -1, bblk = -1;         // last V block lookup
    int j = 0, ns = 0, k = 0, last_cell = -1, n_eval = 0;
    int4 qa = make_int4(0, 0, 0, 0), uu = make_int4(0, 0, 0, 0);
    RayState st;
    st.T = 1.f;
    st.cd[0] = st.cd[1] = st.cd[2] = 0.f;
    st.F[0] = st.F[1] = st.F[2] = st.F[3] = 0.f;
    int c_eval = 0, c_donly = 0, c_skip = 0, c_miss = 0, c_rounds = 0, c_steps = 0, c_lanes = 0;

    if (KF & KF_COUNT) {
        if (lane == 0) atomicMin(stats + 16, gtime());
    }

    auto finish = [&]() {
        if (!(KF & KF_FUSED)) store_accum(ws.accum + (int64_t)ray * 2, st);
        if (KF & KF_TRACE) ta.counts[ray] = n_eval;
        ray = -1;
    };

    while (true) {
        // ---------------- tile scheduling: a new tile of 32 rays when the warp is empty -------
        unsigned act = __ballot_sync(FULL, ray >= 0);
        if (act == 0) {
            if ((KF & KF_FUSED) && tile_rbase >= 0) fused_epilogue<KF>(S, rs, out, tile_rbase, st, fsm[0]);
            int tile = 0;
            if (lane == 0) {
                if (ws.tile_cost) {
                    // the finished tile's duration, for the next call's dispatch order (kept in
                    // shared memory, not in registers: the loop is at its register cap; the warp
                    // index is re-read, not hoisted into a register across the loop)
                    const unsigned w = tid_volatile() >> 5;
                    if (s_tc[w][1] != ~0u)
                        ws.tile_cost[s_tc[w][1]] = (uint16_t)min((unsigned)(clock() - s_tc[w][0]) >> 8, 65535u);
                }
                int t = (int)atomicAdd(ws.queue, 1u);
                tile = t;
                if (ws.tile_list && t < ws.n_tiles) {
                    // the cost-ordered lists, most expensive bucket first
                    for (int b = kBuckets - 1; b >= 0; b--) {
                        const int c = (int)__ldg(ws.bucket_cnt + b);
                        if (t < c) { tile = __ldg(ws.tile_list + (int64_t)b * ws.n_tiles + t); break; }
                        t -= c;
                    }
                }
            }
            tile = __shfl_sync(FULL, tile, 0);
            const unsigned base = (unsigned)tile << 5;
            tile_rbase = base;
            if (ws.tile_cost && lane == 0) {
                const unsigned w = tid_volatile() >> 5;
                s_tc[w][0] = (unsigned)clock();
                s_tc[w][1] = tile < ws.n_tiles ? (unsigned)tile : ~0u;
            }
            if (tile >= ws.n_tiles) {
                if ((KF & KF_COUNT) && lane == 0) atomicMin(stats + 17, gtime());
                break;
            }
            if ((int64_t)base + lane < n_rays) {
                ray = (int)base + lane;
                ns = ws.nseg[ray];
                j = 0;
                k = 0;
                n_eval = 0;
                last_cell = -1;
                st.T = 1.f;
                st.cd[0] = st.cd[1] = st.cd[2] = 0.f;
                st.F[0] = st.F[1] = st.F[2] = st.F[3] = 0.f;
                if (ns > 0) {
                    const int4* p = ws.seg + ((int64_t)ray * ws.seg_slots) * 2;
                    qa = p[0];
                    uu = p[1];
                } else {
                    qa.w = 0;
                }
            }
            act = __ballot_sync(FULL, ray >= 0);
        }

        // ---------------- traversal: advance lanes towards their next evaluated sample ----
        // One step per lane per round; lanes in long empty stretches keep skipping in the next
        // rounds, so one lane's skip chain never idles the warp.
        bool found = false;
        int Qx, Qy, Qz, fcell;             // set by the step that finds a sample (read only then)
        // one traversal step of a lane that wants a sample
        auto step = [&]() {
            if (KF & KF_SPH) {
                // Eq. 4 contraction: sample k at t, then t += Delta / sigma(t)
                // (reading S1) in fp32; every sample is tested against the finest level -- lines
                // map to curves, so there is no AABB skip.  qa = (o, t), uu = d (fp32 bits).
                if (ns == 0 || k >= sph_kmax) { finish(); return; }
                const float t = __int_as_float(qa.w);
                const float dx = __int_as_float(uu.x), dy = __int_as_float(uu.y), dz = __int_as_float(uu.z);
                const float x0 = fmaf(t, dx, __int_as_float(qa.x)), x1 = fmaf(t, dy, __int_as_float(qa.y)),
                            x2 = fmaf(t, dz, __int_as_float(qa.z));
                const float r2 = fmaf(x0, x0, fmaf(x1, x1, x2 * x2));
                const float r = sqrtf(r2);
                float cr = r, sc = 1.f, speed = 1.f;
                if (r > 1.f) {
                    const float inv = __fdividef(1.f, r);
                    cr = 2.f - inv;
                    sc = cr * inv;
                    const float dr = fmaf(dx, x0, fmaf(dy, x1, dz * x2)) * inv;   // radial speed
                    const float inv2 = inv * inv;
                    const float ra = dr * inv2, rb = fmaf(2.f, r, -1.f) * inv2;
                    const float perp = fmaxf(fmaf(-dr, dr, 1.f), 0.f);
                    speed = sqrtf(fmaf(ra, ra, rb * rb * perp));
                }
                if (cr >= sph_stop) { finish(); return; }
                const float q = sc * (float)kOne;
                Qx = __float2int_rn(x0 * q) + kTwoI;
                Qy = __float2int_rn(x1 * q) + kTwoI;
                Qz = __float2int_rn(x2 * q) + kTwoI;
                qa.w = __float_as_int(fmaf(S.step_f, __fdividef(1.f, speed), t));
                k++;
                if (occ_bit(occ_f, occ_cell(Qx, sf, Nf), occ_cell(Qy, sf, Nf), occ_cell(Qz, sf, Nf), Nf)) found = true;
                return;
            }
            if (k >= qa.w) {                                  // segment exhausted
                j++;
                if (j >= ns) { finish(); return; }
                const int4* p = ws.seg + ((int64_t)ray * ws.seg_slots + j) * 2;
                qa = p[0];
                uu = p[1];
                k = 0;
                return;
            }
            Qx = qa.x + k * uu.x;
            Qy = qa.y + k * uu.y;
            Qz = qa.z + k * uu.z;
            if (KF & KF_SKIPTAB) {
                // bordered skip table: the unclamped finest cell indexes it directly (no clamps;
                // multiply-adds on the FMA pipe).  fcell holds this entry index as the cell key.
                const int Nb = Nf + 2;
                fcell = ((Qz >> sf) * Nb + (Qy >> sf)) * Nb + (Qx >> sf) + (Nb * Nb + Nb + 1);
                if (fcell == last_cell) { found = true; return; }  // same finest cell: all levels set
                // one probe: 0 = occupied, else the shift of the coarsest empty level - 16
                MERF_CHECK(fcell >= 0 && (int64_t)fcell < (int64_t)Nb * Nb * Nb);
                const unsigned code = __ldg(reinterpret_cast<const uint8_t*>(S.skiptab) + (unsigned)fcell);
                if (code == 0u) { found = true; return; }
                // the empty cube to leave (the larger of the two the table offers, reading D23):
                //  code < 128: the aligned dyadic cell of lattice shift code + 16 containing the sample;
                //  code >= 128: the cube of Chebyshev radius r = code - 128 finest cells centred on the
                //  sample's finest cell.  Either as [lo, lo + w) per axis, lo = (Q & ~(2^a - 1)) - b.
                const bool cheb = code >= 128u;
                const int r = (int)code - 128;
                const int a = cheb ? sf : (int)code + 16;
                const int b = cheb ? (r << sf) : 0;
                const int w = cheb ? ((2 * r + 1) << sf) : (1 << a);
                const int msk = -(1 << a);
                const int lx = (Qx & msk) - b, ly = (Qy & msk) - b, lz = (Qz & msk) - b;
                // one convergent exit computation for every skipping lane: jump to the first
                // lattice sample outside that empty cube (ray-AABB exit)
                const int K = qa.w;
                int e = min(K, exit_axis(qa.x, uu.x, lx, lx + w, K));
                e = min(e, exit_axis(qa.y, uu.y, ly, ly + w, K));
                e = min(e, exit_axis(qa.z, uu.z, lz, lz + w, K));
                k = min(max(k + 1, e), K);
                if (KF & KF_COUNT) c_skip++;
                return;
            }
            const int fx = occ_cell(Qx, sf, Nf), fy = occ_cell(Qy, sf, Nf), fz = occ_cell(Qz, sf, Nf);
            fcell = (fz * Nf + fy) * Nf + fx;
            if (KF & KF_DENSE) {
                if (occ_bit(occ_f, fx, fy, fz, Nf)) found = true;
                else k++;
                return;
            }
            if (fcell == last_cell) { found = true; return; }  // same finest cell: all levels set
            // level search (no skip table): finest level first -- an occupied finest cell means
            // every coarser (max-pooled) cell is occupied too, so the sample is evaluated after
            // one probe; only an empty finest cell searches coarse -> fine for the coarsest empty
            // level, whose cell exit is the skip target of P:308 (identical result to probing
            // coarse -> fine throughout)
            int e = -1;
            int sh = sf, cx = fx, cy = fy, cz = fz;
            const bool skip = !occ_bit(occ_f, fx, fy, fz, Nf);
            if (skip) {
                // coarsest empty level (default: the finest, known empty)
                bool chosen = false;
    #pragma unroll
                for (int lev = 0; lev < MERF_MAX_LEVELS - 1; lev++) {
                    if (lev < nl - 1 && !chosen) {
                        const int N = S.level_res[lev];
                        const int shl = S.level_shift[lev];
                        const int x = occ_cell(Qx, shl, N), y = occ_cell(Qy, shl, N), z = occ_cell(Qz, shl, N);
                        if (!occ_bit(S.occ[lev], x, y, z, N)) {
                            sh = shl;
                            cx = x;
                            cy = y;
                            cz = z;
                            chosen = true;
                        }
                    }
                }
            }
            if (skip) {
                // one convergent exit computation for every skipping lane: jump to the first
                // lattice sample outside that empty cell (ray-AABB exit)
                const int K = qa.w;
                e = min(K, exit_axis(qa.x, uu.x, cx << sh, (cx + 1) << sh, K));
                e = min(e, exit_axis(qa.y, uu.y, cy << sh, (cy + 1) << sh, K));
                e = min(e, exit_axis(qa.z, uu.z, cz << sh, (cz + 1) << sh, K));
            }
            if (e >= 0) {
                k = min(max(k + 1, e), qa.w);
                if (KF & KF_COUNT) c_skip++;
            } else {
                found = true;
            }
        };
        // one step for every lane holding a ray, then the shading (a round; §6 Rounds: further
        // warp-synchronous steps before shading measured slower, so the r01 tuning knob is gone)
        if (KF & KF_COUNT) c_steps += lane == 0;
        if (ray >= 0) step();

        // ---------------- shading (converged) ----------------
        if (KF & KF_COUNT) {
            const bool any_found = __any_sync(FULL, found);   // every lane votes (no short circuit)
            c_rounds += (lane == 0 && any_found) ? 1 : 0;
            c_lanes += (lane == 0) ? __popc(act) : 0;         // lanes holding a ray this round
        }
        if (found) {
            last_cell = fcell;
            const int kind = shade_sample<KF>(S, Qx, Qy, Qz, st, bslot, bblk);
            if (KF & KF_COUNT) {
                c_eval++;
                c_donly += kind == 1;
                c_miss += kind == 2;
            }
            if (KF & KF_TRACE) {
                if (n_eval < ta.max_per_ray) {
                    const int64_t idx = (int64_t)ray * ta.max_per_ray + n_eval;
                    const int tcell = (KF & KF_SKIPTAB)   // fcell is the bordered table index there
                        ? (occ_cell(Qz, sf, Nf) * Nf + occ_cell(Qy, sf, Nf)) * Nf + occ_cell(Qx, sf, Nf)
                        : fcell;
                    ta.cells[idx] = ((uint64_t)j << 61) | ((uint64_t)k << 40) | (uint64_t)tcell;
                    if (ta.T) ta.T[idx] = st.T;
                }
            }
            n_eval++;
            if (!(KF & KF_SPH)) k++;                          // (the curve step advanced k already)
            if (early_term && st.T < S.t_min) finish();
        }
    }
    if (KF & KF_COUNT) {
        if (lane == 0) atomicMax(stats + 18, gtime());
        add_stat(stats, 2, c_eval);
        add_stat(stats, 3, c_donly);
        add_stat(stats, 4, c_skip);
        add_stat(stats, 5, c_miss);
        add_stat(stats, 13, c_rounds);
        add_stat(stats, 14, c_steps);
        add_stat(stats, 15, c_lanes);
    }
}

// ====================================================================================
// 2b. NEXT-2 comparison variant: the spherical contraction of Eq. 4.  Lines
// map to curves, so there is no ray-AABB skip: one thread per ray takes Euler
// steps of uniform contracted arc length, t += Delta / sigma(t) (reading S1), tests every
// sample against the finest occupancy level and shades occupied samples with the same
// gather/composite code.  Canonical fp64 stepping (reading D8: bit-reproducible traces).
// ====================================================================================
__device__ __forceinline__ double contract_sph(const double x[3], double c[3]) {
    const double r = __dsqrt_rn(add_rn(add_rn(mul_rn(x[0], x[0]), mul_rn(x[1], x[1])), mul_rn(x[2], x[2])));
    if (r <= 1.0) {
        c[0] = x[0]; c[1] = x[1]; c[2] = x[2];
        return r;
    }
    const double sc = sub_rn(2.0, div_rn(1.0, r));
#pragma unroll
    for (int q = 0; q < 3; q++) c[q] = mul_rn(sc, div_rn(x[q], r));
    return r;
}

__device__ __forceinline__ double sph_speed(const double x[3], const double d[3], double r) {
    if (r <= 1.0) return 1.0;
    double xh[3];
#pragma unroll
    for (int q = 0; q < 3; q++) xh[q] = div_rn(x[q], r);
    const double dr = add_rn(add_rn(mul_rn(d[0], xh[0]), mul_rn(d[1], xh[1])), mul_rn(d[2], xh[2]));
    const double rr = mul_rn(r, r);
    const double a = div_rn(dr, rr);
    const double b = div_rn(sub_rn(mul_rn(2.0, r), 1.0), rr);
    double perp = sub_rn(1.0, mul_rn(dr, dr));
    if (perp < 0.0) perp = 0.0;
    return __dsqrt_rn(add_rn(mul_rn(a, a), mul_rn(mul_rn(b, b), perp)));
}

template <int KF>
__global__ void __launch_bounds__(kSetupThreads) march_sph_kernel(DevScene S, RaySource rs, Workspace ws,
                                                                  uint32_t rflags, TraceArgs ta,
                                                                  unsigned long long* stats) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ray = rs.ray0 + r;
    bool valid = r < rs.n;
    double o[3] = {0, 0, 0}, d[3] = {0, 0, 1}, t = 0.0;
    if (valid) {
        if (KF & KF_TRACE) {
            const int64_t pid = rs.pixel_ids[ray];
            raygen(rs.cb.cam[0], (int)(pid % rs.W), (int)(pid / rs.W), o, d);
            t = rs.cb.cam[0].t_near;
        } else if (KF & KF_RAYS) {
#pragma unroll
            for (int q = 0; q < 3; q++) { o[q] = rs.o[3 * ray + q]; d[q] = rs.d[3 * ray + q]; }
            t = rs.t_near ? rs.t_near[ray] : 0.0;
        } else {
            int view, px, py;
            valid = ray_pixel(rs, ray, view, px, py);
            if (valid) {
                raygen(rs.cb.cam[view], px, py, o, d);
                t = rs.cb.cam[view].t_near;
            }
        }
    }
    RayState st;
    st.T = 1.f;
    st.cd[0] = st.cd[1] = st.cd[2] = 0.f;
    st.F[0] = st.F[1] = st.F[2] = st.F[3] = 0.f;
    int n_eval = 0, c_donly = 0, c_miss = 0;
    int bslot = -1, bblk = -1;
    if (valid) {
        const int nl = S.n_levels;
        const int Nf = S.n_fin;
        const int sf = S.s_fin;
        const double stop = sub_rn(2.0, S.step);
        const int kmax = (int)(8.0 / S.step) + 8;
        for (int k = 0; k < kmax; k++) {
            double x[3], c[3];
            point_at(o, d, t, x);
            const double rad = contract_sph(x, c);
            const double cr = rad <= 1.0 ? rad : sub_rn(2.0, div_rn(1.0, rad));
            if (cr >= stop) break;
            const int Qx = (int)__double2ll_rn(mul_rn(c[0], (double)kOne)) + kTwoI;   // biased
            const int Qy = (int)__double2ll_rn(mul_rn(c[1], (double)kOne)) + kTwoI;
            const int Qz = (int)__double2ll_rn(mul_rn(c[2], (double)kOne)) + kTwoI;
            const int fx = occ_cell(Qx, sf, Nf), fy = occ_cell(Qy, sf, Nf), fz = occ_cell(Qz, sf, Nf);
            if (occ_bit(S.occ_fin, fx, fy, fz, Nf)) {
                const int kind = shade_sample<KF>(S, Qx, Qy, Qz, st, bslot, bblk);
                c_donly += kind == 1;
                c_miss += kind == 2;
                if (KF & KF_TRACE) {
                    if (n_eval < ta.max_per_ray) {
                        const int64_t idx = ray * ta.max_per_ray + n_eval;
                        ta.cells[idx] = ((uint64_t)k << 40) | (uint64_t)((fz * Nf + fy) * Nf + fx);
                        if (ta.T) ta.T[idx] = st.T;
                    }
                }
                n_eval++;
                if (!(rflags & MERF_NO_EARLY_TERM) && st.T < S.t_min) break;
            }
            t = add_rn(t, div_rn(S.step, sph_speed(x, d, rad)));
        }
    }
    if (r < rs.n) {
        store_accum(ws.accum + r * 2, st);
        if (KF & KF_TRACE) ta.counts[ray] = n_eval;
    }
    if (KF & KF_COUNT) {
        add_stat(stats, 0, valid ? 1 : 0);
        add_stat(stats, 1, valid ? 1 : 0);
        add_stat(stats, 2, n_eval);
        add_stat(stats, 3, c_donly);
        add_stat(stats, 5, c_miss);
        add_stat(stats, 6, valid ? 1 : 0);
    }
}

// ====================================================================================
// 3. deferred MLP + store
// ====================================================================================
__device__ __forceinline__ void deferred_mlp(const MlpParams& mp, const float x7[7], const float d[3],
                                             float out[3]) {
    const float* w = mp.w;
    float x[34];
#pragma unroll
    for (int i = 0; i < 7; i++) x[i] = x7[i];
    x[7] = d[0]; x[8] = d[1]; x[9] = d[2];
    int n = 10;
    // sin/cos(2^k d_j), k = 0..3, by angle doubling from |d_j| <= 1 (no slow-path range
    // reduction, no local memory); error ~1e-6, far inside the colour tolerance
#pragma unroll
    for (int j = 0; j < 3; j++) {
        float s = __sinf(d[j]), c = __cosf(d[j]);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            x[n++] = s;
            x[n++] = c;
            const float s2 = 2.f * s * c, c2 = fmaf(-2.f * s, s, 1.f);
            s = s2;
            c = c2;
        }
    }
    const float* W0 = w;
    const float* b0 = w + 544;
    const float* W1 = w + 560;
    const float* b1 = w + 816;
    const float* W2 = w + 832;
    const float* b2 = w + 880;
    float h0[16], h1[16];
#pragma unroll
    for (int o = 0; o < 16; o++) {
        float s = b0[o];
#pragma unroll
        for (int i = 0; i < 34; i++) s = fmaf(W0[o * 34 + i], x[i], s);
        h0[o] = fmaxf(s, 0.f);
    }
#pragma unroll
    for (int o = 0; o < 16; o++) {
        float s = b1[o];
#pragma unroll
        for (int i = 0; i < 16; i++) s = fmaf(W1[o * 16 + i], h0[i], s);
        h1[o] = fmaxf(s, 0.f);
    }
#pragma unroll
    for (int o = 0; o < 3; o++) {
        float s = b2[o];
#pragma unroll
        for (int i = 0; i < 16; i++) s = fmaf(W2[o * 16 + i], h1[i], s);
        out[o] = __fdividef(1.0f, 1.0f + __expf(-s));
    }
}

template <int KF>
__global__ void __launch_bounds__(kSetupThreads) shade_kernel(DevScene S, RaySource rs, Workspace ws,
                                                              void* out, const __grid_constant__ MlpParams mlp) {
    asm volatile("griddepcontrol.wait;" ::: "memory");    // the march's accumulators (PDL)
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rs.n) return;
    const int64_t ray = rs.ray0 + r;
    float d[3];
    int64_t out_idx;
    int view = 0, px = 0, py = 0;
    if (KF & KF_RAYS) {
#pragma unroll
        for (int q = 0; q < 3; q++) d[q] = (float)rs.d[3 * ray + q];
        out_idx = ray;
    } else {
        if (!ray_pixel(rs, ray, view, px, py)) return;
        double od[3], dd[3];
        raygen(rs.cb.cam[view], px, py, od, dd);
#pragma unroll
        for (int q = 0; q < 3; q++) d[q] = (float)dd[q];
        out_idx = out_index(rs, view, px, py);
    }
    const float4 a0 = ws.accum[r * 2], a1 = ws.accum[r * 2 + 1];
    const float x7[7] = {a0.x, a0.y, a0.z, a1.x, a1.y, a1.z, a1.w};
    float h[3];
    deferred_mlp(mlp, x7, d, h);
    const float c0 = __saturatef(a0.x + h[0]), c1 = __saturatef(a0.y + h[1]), c2 = __saturatef(a0.z + h[2]);
    auto put = [&](int64_t idx) {
        if (KF & KF_U8) {
            reinterpret_cast<uchar4*>(out)[idx] =
                make_uchar4((unsigned char)__float2int_rn(c0 * 255.f), (unsigned char)__float2int_rn(c1 * 255.f),
                            (unsigned char)__float2int_rn(c2 * 255.f), 255);
        } else {
            float* o3 = reinterpret_cast<float*>(out) + 3 * idx;
            o3[0] = c0;
            o3[1] = c1;
            o3[2] = c2;
        }
    };
    put(out_idx);
    if (!(KF & KF_RAYS) && rs.fill) {
        // progressive preview: nearest upsampling of the sub-lattice pixel to its
        // stride x stride block (clipped to the frame)
        const int sd = rs.stride_m1 + 1;
        for (int dy = 0; dy < sd; dy++)
            for (int dx = 0; dx < sd; dx++)
                if ((dx | dy) != 0 && px + dx < rs.W && py + dy < rs.H)
                    put(((int64_t)view * rs.H + py + dy) * rs.W + px + dx);
    }
}

}  // namespace merf
