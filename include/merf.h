/*
 * merf.h -- C ABI of the B200-native MERF baked-scene renderer (libmerf.so).
 *
 * The library renders a baked MERF scene (Reiser et al., arXiv 2302.12249; "P:<n>" below is
 * line n of the paper text /root/reference/PAPER.md) with hand-written sm_100a CUDA kernels:
 * per ray, piecewise-projective contraction and region clipping (Sec. 4.2),
 * hierarchical occupancy skipping in contracted space, block-sparse 3D grid +
 * tri-plane gather of uint8 features, dequantised and summed (Eq. 5, Eq. 7
 * P:254-258), decode (Eq. 6), front-to-back compositing with early termination
 * (Eq. 1-2) and one deferred MLP per pixel (Eq. 3).
 * Readings of the paper where it is silent (D1..D22) are listed in DESIGN.md.
 *
 * Conventions
 *   - Plain C, no exceptions cross the ABI, nothing aborts.  Every call returns a
 *     merf_status; on failure merf_last_error() returns a thread-local message.
 *   - Host pointers are marked [host], device pointers [device].  Device pointers must be
 *     allocations on the scene's device (e.g. torch tensors' data_ptr()).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Compute
 *     calls are asynchronous on that stream unless documented otherwise.
 *   - Ownership: inputs are caller-owned and only read; merf_scene_upload copies everything
 *     it needs, so the caller may free its arrays after it returns.  The scene handle owns
 *     all device memory it allocated until merf_scene_free.  Output buffers are caller-owned.
 *   - Thread safety: a scene is immutable after upload; concurrent renders of one scene on
 *     different streams are safe.  merf_scene_free must not race with renders.
 *
 * Layouts (all little-endian, C order)
 *   occupancy bits : level of resolution N is N^3 bits, linear index (z*N + y)*N + x,
 *                    packed LSB-first into uint32 words ((N^3 + 31) / 32 words).
 *   planes         : uint8 [3][R][R][C]; plane 0 = P_x indexed [z][y], plane 1 = P_y [z][x],
 *                    plane 2 = P_z [y][x].  Texel i is centred at
 *                    -2 + (i + 1/2) * 4/R in contracted space (reading D9).
 *   block_index    : int32 [(L/8)^3], slot (bz*nb + by)*nb + bx, -1 = block not stored.
 *   atlas          : uint8 [n_blocks][9][9][9][C], (z,y,x): block data voxels 8b..8b+7 plus a
 *                    1-voxel apron at 8b+8 (clamped to L-1) so trilinear corners never cross
 *                    blocks (reading D11).
 *   channels       : C = 8: [density, r, g, b, f0, f1, f2, f3] (reading D12); byte b
 *                    decodes to 2m*b/255 - m with m = 14 (density) / 7 (others) (Eq. 7).
 *   mlp            : float32 [883] = W0[16][34] b0[16] W1[16][16] b1[16] W2[3][16] b2[3];
 *                    input [C_d(3), F(4), d(3), sin/cos(2^k d_j) j outer, k = 0..3 inner,
 *                    sin before cos] (readings D16-D17).
 *   camera         : merf_camera below; OpenCV pinhole, pixel centres (reading D18).
 *   output         : MERF_RGB_F32 -> float [n_cams][H][W][3]; MERF_RGBA_U8 -> uint8
 *                    [n_cams][H][W][4], round(255*C), alpha = 255.
 */
#ifndef MERF_H_
#define MERF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MERF_OK = 0,
    MERF_EINVAL = 1,     /* invalid argument (null pointer, bad size, bad descriptor)     */
    MERF_ENOMEM = 2,     /* device allocation failed                                      */
    MERF_ECUDA = 3,      /* a CUDA runtime call or kernel launch failed                   */
    MERF_ENCCL = 4,      /* NCCL missing, a communicator error, or a gather timeout       */
    MERF_EMISMATCH = 5,  /* scene arrays inconsistent (unsound block index, bad entries)  */
    MERF_EIO = 6         /* bundle / camera file missing, unreadable, malformed or corrupt */
} merf_status;

enum { MERF_RGB_F32 = 0, MERF_RGBA_U8 = 1 };

enum {
    MERF_NO_EARLY_TERM = 1u,   /* disable termination at T < t_min                */
    MERF_COUNTERS = 2u,        /* accumulate merf_stats (adds device atomics)             */
    MERF_DENSE = 4u,           /* debug: dense stepping gated by the finest level only     */
    MERF_TIMED = 8u,           /* record CUDA events around every pipeline kernel launch     */
    MERF_SPHERICAL = 16u,      /* NEXT-2 comparison variant: the scene's grids live in the
                                  space of the spherical contraction of Eq. 4;
                                  fixed contracted-arc-length Euler steps, t += Delta/sigma(t),
                                  every sample tested against the finest level, no AABB skip
                                  (P:222-226).  Accepted by merf_render, merf_render_rays,
                                  merf_trace (segment ordinal 0, k = step index).            */
    MERF_MLP_FFMA = 32u,       /* run the deferred MLP (Eq. 3) as FFMA chains instead of
                                  the default tensor-core kernel (split-fp16 mma.sync, fp32-class
                                  accuracy); cross-check / ablation.  Scenes whose MLP weights
                                  could overflow fp16 always use the FFMA kernel.              */
    MERF_SPH_PERSISTENT = 64u  /* with MERF_SPHERICAL in merf_render / merf_render_rays: the
                                  same curve march in fp32 inside the persistent tile-scheduled
                                  march kernel with the production gather -- the like-for-like
                                  speed comparison with the piecewise-projective contraction.
                                  fp32 sample positions differ slightly from the canonical fp64
                                  steps, so its parity is statistical (traces: fp64 kernel).  */
};

#define MERF_MAX_LEVELS 4
#define MERF_FIXED_BITS 28     /* lattice fraction bits F (reading D8): int32 lattice     */

typedef struct {
    int32_t L;                  /* 3D grid resolution: power of two >= 8, or 0 = no grid      */
    int32_t R;                  /* plane resolution: power of two >= 2, or 0 = no planes      */
    int32_t C;                  /* channels, must be 8                                        */
    int32_t n_levels;           /* occupancy levels, 1..MERF_MAX_LEVELS                      */
    int32_t level_res[MERF_MAX_LEVELS]; /* coarse -> fine, powers of two, each divides next;
                                   the last (finest) level gates field evaluation  */
    float m_density;            /* 14                                                 */
    float m_appearance;         /* 7                                                 */
    double step;                /* uniform contracted step Delta, power of two (D5)   */
    float t_min;                /* termination transmittance, 2e-4                   */
    float alpha_skip;           /* appearance read iff alpha > alpha_skip, 0 (D14)     */
    uint32_t source_mask;       /* bit0 V, bit1 P_x, bit2 P_y, bit3 P_z (config-5 variants)  */
} merf_scene_desc;

typedef struct {
    double c2w[12];             /* camera-to-world, row-major 3x4 [R | t]; OpenCV axes       */
    double fx, fy, cx, cy;      /* pinhole intrinsics in pixels                              */
    double t_near;              /* ray start parameter, >= 0                                 */
} merf_camera;

typedef struct {
    int64_t rays;
    int64_t segments;           /* kept contracted segments (<= 7 per ray)                    */
    int64_t evaluated;          /* samples whose finest occupancy bit is set (field read)    */
    int64_t density_only;       /* evaluated samples with alpha <= alpha_skip (20 B read)     */
    int64_t skips;              /* empty-cell jumps                                   */
    int64_t missing_blocks;     /* evaluated samples whose V block is absent (must be 0)      */
    int64_t region_segments[7]; /* kept segments per region (core, +x, -x, +y, -y, +z, -z)   */
    int64_t march_rounds;       /* warp shading rounds of the persistent march (perf counter) */
    int64_t march_steps;        /* warp traversal iterations (perf counter)                   */
    int64_t march_lane_rounds;  /* sum over rounds of lanes holding a ray (perf counter)      */
    int64_t march_busy_ns;      /* per march launch, summed: first warp start -> tile queue dry */
    int64_t march_tail_ns;      /* per march launch, summed: tile queue dry -> last warp exit   */
} merf_stats;

typedef struct {
    int32_t L, R, C, n_levels;
    int32_t level_res[MERF_MAX_LEVELS];
    int64_t n_blocks;
    int64_t canonical_blocks;   /* blocks the canonical allocation needs (<= n_blocks)        */
    int64_t device_bytes;       /* device memory owned by the scene                           */
    int32_t device;
} merf_scene_info;

typedef struct merf_scene merf_scene;

/* Device time of the render pipeline's kernels launched with MERF_TIMED since the last
 * reset (CUDA events on the launch stream; reading synchronises them). */
typedef struct {
    double setup_ms, march_ms, shade_ms;     /* summed device time per kernel kind        */
    int64_t setup_launches, march_launches, shade_launches;
} merf_kernel_times;

/* Thread-local description of the last failure ("" if none). */
const char *merf_last_error(void);

/* Library/ABI version (major*10000 + minor*100 + patch). */
int32_t merf_version(void);

/*
 * Copy a baked scene to `device` and build its acceleration structures:
 * the coarser occupancy levels by max-pooling the finest and the canonical
 * block allocation (reading D11).
 *   desc        [host] scene descriptor (validated: L, R powers of two, C == 8, levels
 *               powers of two dividing each other, step a power of two > 0).
 *   planes      [host] uint8 [3][R][R][C] (ignored if R == 0).
 *   block_index [host] int32 [(L/8)^3] or NULL: NULL means "atlas is in canonical order"
 *               and requires n_blocks == the canonical count.  A non-NULL index is checked:
 *               entries in [-1, n_blocks) and every canonically needed block stored
 *               (soundness: every evaluated sample has its block), else MERF_EMISMATCH.
 *   atlas       [host] uint8 [n_blocks][9][9][9][C] (ignored if L == 0).
 *   occ_finest  [host] uint32 bits of the finest level (level_res[n_levels-1]).
 *   mlp         [host] float [883].
 *   out         [host] receives the handle.
 * Synchronous.  Errors: MERF_EINVAL, MERF_ENOMEM, MERF_ECUDA, MERF_EMISMATCH.
 */
merf_status merf_scene_upload(const merf_scene_desc *desc, const uint8_t *planes,
                              const int32_t *block_index, const uint8_t *atlas, int64_t n_blocks,
                              const uint32_t *occ_finest, const float *mlp, int32_t device,
                              merf_scene **out);

/* Release the scene's device memory (synchronises its device).  NULL is a no-op. */
merf_status merf_scene_free(merf_scene *scene);

/* Scene facts (host struct). */
merf_status merf_scene_info_get(const merf_scene *scene, merf_scene_info *info);

/* Device copy of occupancy level `level` (0 = coarsest) into `bits_out` [device]
 * ((N^3+31)/32 words), asynchronous on `stream`. */
merf_status merf_scene_occupancy(const merf_scene *scene, int32_t level, uint32_t *bits_out,
                                 void *stream);

/* Device copy of the scene's block index [(L/8)^3] int32 into `index_out` [device]. */
merf_status merf_scene_block_index(const merf_scene *scene, int32_t *index_out, void *stream);

/*
 * Render n_cams full frames of W x H pixels (the hot path, Sec. 6).
 *   cams   [host] n_cams cameras (copied into the launch; the caller may reuse them).
 *   format MERF_RGB_F32 or MERF_RGBA_U8; out [device] caller-owned output (see Layouts).
 *   flags  MERF_NO_EARLY_TERM | MERF_COUNTERS | MERF_DENSE.
 *   stats  [host] optional; if non-NULL the call enables counters, synchronises `stream`
 *          and fills *stats (so it is no longer asynchronous).
 * Scheduling state: a call of at most 4 views in one chunk records its per-tile march
 * durations in the scene (a few hundred KB of device memory, allocated on first use); the
 * next such call with the same W, H and n_cams dispatches its tiles longest first by them.
 * Only the order in which warps take tiles changes, never a pixel (results are byte-identical
 * to raster order; MERF_TILE_ORDER=raster in the environment disables it).
 * Errors: MERF_EINVAL (null, W/H/n_cams <= 0, W*H*n_cams > 2^31, bad format), MERF_ENOMEM,
 * MERF_ECUDA.
 */
merf_status merf_render(const merf_scene *scene, const merf_camera *cams, int32_t n_cams,
                        int32_t W, int32_t H, int32_t format, void *out, uint32_t flags,
                        void *stream, merf_stats *stats);

/*
 * Device workspace a merf_render(scene, cams, n_cams views of W x H) call allocates from the
 * stream-ordered pool for its chunk of rays (segments, accumulators, queue, tile lists):
 * *bytes, and the rays of one chunk in *rays_per_chunk (optional).  cams [host] may be NULL
 * (worst case: 7 segment slots per ray; cameras whose origins are all in the core need 4).
 * Host-only arithmetic, no device work.  Errors: MERF_EINVAL.
 */
merf_status merf_render_workspace_bytes(const merf_scene *scene, const merf_camera *cams, int32_t n_cams,
                                        int32_t W, int32_t H, int64_t *bytes, int64_t *rays_per_chunk);

/* Collect (and, if reset != 0, clear) the MERF_TIMED kernel times of `scene`. */
merf_status merf_kernel_times_get(merf_scene *scene, merf_kernel_times *out, int32_t reset);

/*
 * Single-frame sharding for multi-GPU rendering ("image tiles of 64x64
 * interleaved by rank, to balance the uneven samples/ray"): renders exactly the pixels of the
 * 64x64-pixel blocks b (row-major over the frame, b = bx + by * ceil(W / 64)) with
 * b % part_count == part_rank, of every view, each with the same arithmetic as merf_render,
 * into the full-resolution `out` (layout as merf_render); all other pixels are left
 * untouched.  The part_count shards of one frame therefore write disjoint pixel sets whose
 * union is the whole frame: zero-filled RGBA8 shards combine by a byte-wise sum (e.g. an
 * NCCL reduce to the root).  part_count = 1 is merf_render.  MERF_COUNTERS is ignored.
 * Asynchronous.  Errors: those of merf_render, MERF_EINVAL (part_count < 1 or part_rank not
 * in [0, part_count)).
 */
merf_status merf_render_shard(const merf_scene *scene, const merf_camera *cams, int32_t n_cams,
                              int32_t W, int32_t H, int32_t part_rank, int32_t part_count,
                              int32_t format, void *out, uint32_t flags, void *stream);

/*
 * Compact single-frame shard: the same rays as merf_render_shard, but the output
 * holds only this part's blocks, packed by slot: blocks_out [device] [n_cams][S][64][64] pixels
 * (RGB f32 or RGBA8), S = merf_shard_slots(W, H, part_count), slot s = block part_rank +
 * part_count * s (row-major blocks).  Pixels of edge blocks outside the frame and slots past
 * the last block are not written.  This is what a rank sends to the root (merf_gather_frames);
 * the root rebuilds the frames with merf_shard_assemble.  Asynchronous.  Errors: those of
 * merf_render_shard.
 */
merf_status merf_render_shard_blocks(const merf_scene *scene, const merf_camera *cams, int32_t n_cams,
                                     int32_t W, int32_t H, int32_t part_rank, int32_t part_count,
                                     int32_t format, void *blocks_out, uint32_t flags, void *stream);

/* Block slots per part of a W x H frame split into part_count parts (0 on bad arguments). */
int32_t merf_shard_slots(int32_t W, int32_t H, int32_t part_count);

/*
 * Rebuild frames from the gathered compact shards: blocks [device] [part_count][n_views][S]
 * [64][64] pixels (merf_gather_frames of every part's merf_render_shard_blocks output, part p
 * at offset p) -> frame_out [device] [n_views][H][W] pixels (format as rendered).  Every frame
 * pixel is written exactly once (the parts partition the blocks).  Asynchronous; one kernel.
 * Errors: MERF_EINVAL (null, sizes, format), MERF_ECUDA.
 */
merf_status merf_shard_assemble(const void *blocks, int32_t n_views, int32_t W, int32_t H, int32_t part_count,
                                int32_t format, void *frame_out, void *stream);

/*
 * Multi-GPU frame gather (the only collective of the design: rays are
 * independent and the scene is replicated, so finished frames are the one thing exchanged;
 * throughput context P:329).  One process per GPU.  NCCL is loaded at run time
 * (libnccl.so.2, or the path in MERF_NCCL_LIB): without it these calls return MERF_ENCCL.
 *
 * merf_comm_unique_id: rank 0 creates the 128-byte id [host]; the caller distributes it to the
 *   other ranks by any channel (e.g. a TCP store).
 * merf_comm_init: every rank joins (blocking until all n_ranks have called it), on `device`.
 * merf_gather_frames: rank r's `bytes` bytes at local [device] land at root_buf + r * bytes on
 *   the root (root_buf [device], n_ranks * bytes, ignored elsewhere).  Grouped ncclSend (ranks
 *   != root) / ncclRecv (root; its own part is a device copy), enqueued on `stream`
 *   (asynchronous; the caller orders buffer reuse by stream events).  The communicator's async
 *   error state (ncclCommGetAsyncError) is checked before and after enqueueing.
 * merf_comm_wait: wait for `stream` while polling the async error state; on an error, or if
 *   the stream has not completed after timeout_ms (< 0: no limit), the communicator is aborted
 *   (ncclCommAbort, so the stream is released) and MERF_ENCCL returned; the communicator is then
 *   unusable (free it).
 * merf_comm_info: rank count, own rank and the loaded NCCL version code.
 * Errors: MERF_EINVAL (null, rank/root out of range, device), MERF_ENCCL, MERF_ECUDA.
 */
#define MERF_COMM_ID_BYTES 128
typedef struct merf_comm merf_comm;
merf_status merf_comm_unique_id(uint8_t *id_out);
merf_status merf_comm_init(const uint8_t *id, int32_t n_ranks, int32_t rank, int32_t device, merf_comm **out);
merf_status merf_comm_free(merf_comm *comm);
merf_status merf_comm_info(const merf_comm *comm, int32_t *n_ranks, int32_t *rank, int32_t *nccl_version);
merf_status merf_gather_frames(merf_comm *comm, const void *local, void *root_buf, int64_t bytes,
                               int32_t root, void *stream);
merf_status merf_comm_wait(merf_comm *comm, void *stream, int32_t timeout_ms);

/*
 * Progressive rendering ("the image is first rendered at a
 * lower resolution ... additional low resolution images are rendered that are dynamically
 * combined into the final high resolution image"): pass p in [0, stride^2) renders exactly
 * the pixels (stride * i + p % stride, stride * j + p / stride) of every view -- each pixel
 * with the same arithmetic as merf_render, so the stride^2 passes together write a frame
 * identical to merf_render's -- into the full-resolution `out` (layout as merf_render);
 * other pixels are left untouched unless `fill` != 0, which also writes each rendered colour
 * to its stride x stride block (pixels (x, y) with x in [px, px + stride), y in [py, py +
 * stride), clipped to the frame): the nearest-upsampled preview.  stride 1 = merf_render.
 * A pass whose offset lies outside a tiny frame renders nothing.  MERF_COUNTERS is ignored.
 * Asynchronous.  Errors: those of merf_render, MERF_EINVAL (stride not in [1, 64], pass not
 * in [0, stride^2)).
 */
merf_status merf_render_progressive(const merf_scene *scene, const merf_camera *cams, int32_t n_cams,
                                    int32_t W, int32_t H, int32_t stride, int32_t pass, int32_t fill,
                                    int32_t format, void *out, uint32_t flags, void *stream);

/*
 * End-to-end variant with HOST output: renders into scene-owned device staging buffers in
 * chunks (up to 14 views, then a last chunk of 2) and copies each finished chunk to
 * `out_host` [host] (pinned memory recommended) while the next chunk renders, so only the
 * last short copy is exposed.  Synchronous on return.  Same layouts/errors as merf_render.
 */
merf_status merf_render_host(const merf_scene *scene, const merf_camera *cams, int32_t n_cams,
                             int32_t W, int32_t H, int32_t format, void *out_host,
                             uint32_t flags, void *stream);

/*
 * Asynchronous end-to-end variant for frame streams: renders the n_cams views into one of two
 * scene-owned device buffers (alternating between calls) and enqueues their copy to `out_host`
 * [host, pinned for an asynchronous copy] on the scene's copy stream; returns at once.  The
 * next call renders into the other buffer while this copy runs, so a stream of calls keeps the
 * GPU rendering; a call reuses a buffer only after its previous copy completed (device-side
 * ordering, no host wait).  `out_host` must stay allocated and must not be read until
 * merf_host_wait(scene) returns.  One host thread per scene for these calls.  Same layouts /
 * errors as merf_render.
 */
merf_status merf_render_host_async(const merf_scene *scene, const merf_camera *cams, int32_t n_cams,
                                   int32_t W, int32_t H, int32_t format, void *out_host,
                                   uint32_t flags, void *stream);

/* Wait until every copy enqueued by merf_render_host_async on `scene` has landed in host memory. */
merf_status merf_host_wait(merf_scene *scene);

/*
 * Render explicit rays: o, d [device] double [n][3] (d unit length), t_near [device] double [n]
 * or NULL (0).  rgb [device] float [n][3].  Errors: MERF_EINVAL, MERF_ECUDA.
 */
merf_status merf_render_rays(const merf_scene *scene, const double *o, const double *d,
                             const double *t_near, int64_t n, float *rgb, uint32_t flags,
                             void *stream, merf_stats *stats);

/*
 * Per-ray visited-cell trace (debug/parity) for pixels `pixel_ids` [device] int64 [n]
 * (id = j*W + i) of camera `cam` [host].  For each evaluated sample, in march order:
 *   cells_out [device] uint64 [n][max_per_ray]: (segment ordinal << 61) | (k << 40) | cell,
 *             cell = finest-level linear index (z*N + y)*N + x;
 *   T_out     [device] float [n][max_per_ray]: transmittance after the sample (may be NULL);
 *   counts_out[device] int32 [n]: number of evaluated samples (may exceed max_per_ray; only
 *             the first max_per_ray are stored).
 * Errors: MERF_EINVAL, MERF_ECUDA.
 */
merf_status merf_trace(const merf_scene *scene, const merf_camera *cam, int32_t W,
                       const int64_t *pixel_ids, int64_t n, int32_t max_per_ray,
                       uint64_t *cells_out, float *T_out, int32_t *counts_out, uint32_t flags,
                       void *stream);

/* One contracted segment of a ray: world interval [t_a, t_b] (t_b = +inf for the
 * unbounded last one), region (0 core, 1 + 2j + (s < 0)), lattice origin Qa = llrint(c_a 2^28),
 * lattice step U = llrint(u Delta 2^28) and sample count K = ceil(l / Delta) (readings D5-D8). */
typedef struct {
    double t_a, t_b;
    int64_t Qa[3];
    int64_t U[3];
    int32_t K;
    int32_t region;
} merf_segment;

/*
 * Per-ray contracted segments (debug/parity of the clipping step) for pixels `pixel_ids`
 * [device] int64 [n] of camera `cam` [host]: segs_out [device] merf_segment [n][max_seg]
 * (kept segments in order, zero-length ones dropped), counts_out [device] int32 [n].
 * Errors: MERF_EINVAL, MERF_ECUDA.
 */
merf_status merf_segments(const merf_scene *scene, const merf_camera *cam, int32_t W,
                          const int64_t *pixel_ids, int64_t n, int32_t max_seg,
                          merf_segment *segs_out, int32_t *counts_out, void *stream);

/*
 * contract_pi of n points: x, y [device] double [n][3]; region [device] int32 [n]
 * or NULL (0 = core, 1 + 2j + (x_j < 0) for the outer region of axis j, reading D1-D2).
 */
merf_status merf_contract(const double *x, int64_t n, double *y, int32_t *region, void *stream);

/*
 * Occupancy pyramid (K0): max-pool the finest level `finest_bits` [device] into every
 * coarser level of `desc`, written coarse -> fine, concatenated, to `levels_out` [device]
 * (sum over levels 0..n_levels-2 of (N^3+31)/32 words).  Asynchronous.
 */
merf_status merf_build_occupancy(const uint32_t *finest_bits, const merf_scene_desc *desc,
                                 uint32_t *levels_out, void *stream);

/*
 * Canonical block allocation (K1, reading D11): a block slot is needed iff some occupied
 * finest cell can produce a sample whose trilinear base voxel lies in it; needed slots are
 * numbered in raster order.  finest_bits [device]; index_out [device] int32 [(L/8)^3];
 * n_blocks [host] receives the count.  Synchronises `stream`.
 */
merf_status merf_build_block_index(const uint32_t *finest_bits, const merf_scene_desc *desc,
                                   int32_t *index_out, int64_t *n_blocks, void *stream);

/*
 * Baking helpers (upstream of the render path).
 *
 * merf_bake_occupancy: binary grid A of resolution N from weighted points:
 * point i (world position x[i], density tau[i], volume-rendering weight w[i]) marks the eight
 * voxels around its contracted position (cell-centred trilinear corners, clamped; readings
 * D2, D8, D9) iff w[i] > w_thr and alpha_i = 1 - exp(-tau[i] step) > alpha_thr with the
 * renderer's step.  The alpha test is evaluated as tau[i] > -ln(1 - alpha_thr)
 * / step (monotone, exact).  x [device] double [n][3], tau, w [device] double [n];
 * bits_out [device] uint32 ((N^3+31)/32 words), zeroed by the call.  Asynchronous.
 * Errors: MERF_EINVAL (N not a power of two in [2, 4096], step <= 0, null pointers).
 */
merf_status merf_bake_occupancy(const double *x, const double *tau, const double *w, int64_t n,
                                int32_t N, double step, double w_thr, double alpha_thr,
                                uint32_t *bits_out, void *stream);

/*
 * merf_pack_atlas: block-sparse storage of a dense grid (reading D11): for every stored
 * block b = index[slot], atlas[b] = dense voxels 8*slot .. 8*slot + 8 per axis (apron clamped
 * to L - 1).  dense [device] uint8 [L][L][L][8]; index [device] int32 [(L/8)^3];
 * atlas_out [device] uint8 [n_blocks][9][9][9][8].  Asynchronous.
 */
merf_status merf_pack_atlas(const uint8_t *dense, int32_t L, const int32_t *index, int64_t n_blocks,
                            uint8_t *atlas_out, void *stream);

/*
 * Asset ingestion (Sec. 5.3, "we encode textures as PNGs";
 * SPEC S:430-465 bundle layout).  A bundle is a directory:
 *   manifest.txt  "merf_bundle 1", L, R, C, block_size 8, level_res (coarse -> fine),
 *                 m_density, m_appearance, step (%.17g), t_min, alpha_skip, source_mask,
 *                 n_blocks, "background none", mlp_dims 34 16 16 3, the 883 MLP weights in
 *                 decimal (%.9g, exact for fp32), and "file <name> <bytes> <crc32 hex>" per
 *                 payload;
 *   plane<a>_{density,diffuse,features}.png (a = 0..2, if R > 0): lossless 8-bit gray / RGB
 *                 / RGBA rasters R x R (channels 0 / 1-3 / 4-7 of [R][R][8]);
 *   atlas_{density,diffuse,features}.png (if L > 0 and n_blocks > 0): the atlas as a Z-major
 *                 stack of 9 x 9 slices (slice q = 9 b + z), 455 slices per raster row
 *                 (<= 4095 px wide), same channel split;
 *   block_index.bin (if L > 0): int32 little-endian [(L/8)^3];
 *   occupancy<i>.bin: level i packed little-endian bits, bit k of byte n = cell 8n + k, x
 *                 fastest, ceil(N^3/8) bytes; coarse levels = OR-pool of the
 *                 finest.
 *
 * merf_bundle_write: write the host arrays of merf_scene_upload (block_index required when
 * L > 0) into `dir` (created if missing; files overwritten).  Coarse occupancy levels are
 * pooled from occ_finest.  Errors: MERF_EINVAL, MERF_EMISMATCH (an index entry outside
 * [-1, n_blocks): payload/manifest mismatch refuses to write), MERF_EIO.
 *
 * merf_bundle_read: parse `dir`; desc and *n_blocks are always filled; when every array
 * pointer is NULL the call only queries them, otherwise planes [3][R][R][8] (if R > 0),
 * block_index and atlas [n_blocks][9][9][9][8] (if L > 0), occ_finest ((N^3+31)/32 words)
 * and mlp [883] (host, caller-owned, sized from the query) are filled.  Every payload's size
 * and CRC-32 are checked, every raster's dimensions against the manifest, every coarse
 * level against the pool of the finest.  Errors: MERF_EINVAL, MERF_EIO (missing file,
 * checksum / size / version mismatch, malformed manifest or PNG), MERF_EMISMATCH.
 *
 * merf_scene_load: merf_bundle_read + merf_scene_upload (synchronous).
 */
merf_status merf_bundle_write(const char *dir, const merf_scene_desc *desc, const uint8_t *planes,
                              const int32_t *block_index, const uint8_t *atlas, int64_t n_blocks,
                              const uint32_t *occ_finest, const float *mlp);
merf_status merf_bundle_read(const char *dir, merf_scene_desc *desc, int64_t *n_blocks, uint8_t *planes,
                             int32_t *block_index, uint8_t *atlas, uint32_t *occ_finest, float *mlp);
merf_status merf_scene_load(const char *dir, int32_t device, merf_scene **out);

/*
 * Camera file: one camera per line, '#' comments and blank lines skipped,
 * 20 numbers: W H fx fy cx cy r00 r01 r02 t0 r10 r11 r12 t1 r20 r21 r22 t2 near far
 * (camera-to-world [R | t] row-major, OpenCV axes, reading D18; `near` becomes t_near; far
 * must exceed near and is otherwise unused: rays end at the contracted scene boundary).
 * cams [host] (max_cams entries) or NULL to count; widths / heights [host] or NULL.
 * Errors: MERF_EINVAL (NULL path / n_cams, more than max_cams cameras), MERF_EIO (unreadable
 * file; a malformed line, non-positive size or focal length, far <= near, or a rotation
 * that is not orthonormal with det +1 -- the message names the line).
 */
merf_status merf_cameras_read(const char *path, merf_camera *cams, int32_t max_cams, int32_t *n_cams,
                              int32_t *widths, int32_t *heights);

/*
 * Quantisation-aware training step (Sec. 5.2, Eq. 7-8) on
 * toy DENSE grids: continuous pre-sigmoid parameters theta of a dense L^3 grid and three R^2
 * planes (C = 8 channels, channel fastest, same axis conventions as the baked arrays) are
 * turned into stored values v = 2m q(sigma(theta)) - m (Eq. 7; q = round to 1/255 when
 * `quantize`, else identity), rendered with the renderer's lattice (readings D5-D8) at every
 * sample inside an occupied cell of `occ` (dense mode, no early termination), composited
 * (Eq. 1-2) and shaded by the fixed deferred MLP (Eq. 3) into C = clamp(C_d + h, 0, 1).
 * Texel lookup clamps the lower corner to [0, M-2] (same values as reading D9's clamp, and
 * gradients never leave the grid).  loss = sum over pixels and channels (C - target)^2; the
 * gradient of the loss w.r.t. theta uses the straight-through estimator dq/dx = 1 (Eq. 8).
 */
typedef struct {
    int32_t L;                  /* dense grid resolution (power of two, 2..1024)              */
    int32_t R;                  /* plane resolution (power of two, 2..8192)                   */
    int32_t occ_res;            /* occupancy grid resolution N (power of two, 2..4096)        */
    int32_t quantize;           /* 1: Eq. 7-8 with STE; 0: continuous sigma(theta)            */
    int32_t max_samples;        /* per-ray sample records kept for the backward pass (>= 1)   */
    int32_t pad_;
    double step;                /* Delta (power of two in (0, 1])                             */
    double m_density, m_appearance;   /* decode ranges m: 14 and 7                     */
} merf_qat_desc;

/*
 * merf_qat_step: forward + backward of one batch of n_cams views (<= 16).
 *   theta_v [device] float [L][L][L][8]; theta_p [device] float [3][R][R][8];
 *   occ [device] uint32 bits of the N^3 occupancy grid (x fastest, LSB first);
 *   mlp [device] float [883]; cams [host] merf_camera [n_cams];
 *   target [device] float [n_cams][H][W][3];
 *   rgb_out [device] float [n_cams][H][W][3] (written);
 *   grad_v, grad_p [device] float, shaped like theta (overwritten, not accumulated);
 *   loss [device] double (overwritten);
 *   overflow [device] int32 or NULL: rays whose sample count exceeded max_samples (their
 *   colour and loss are exact, their gradient contribution is dropped; 0 on a valid call);
 *   n_samples [device] int64 or NULL: total evaluated samples of the batch.
 * Scratch (~48 B x max_samples per ray) is stream-ordered device memory owned by the call.
 * Asynchronous on `stream`.  Errors: MERF_EINVAL (null pointers, bad sizes), MERF_ENOMEM,
 * MERF_ECUDA.
 */
merf_status merf_qat_step(const merf_qat_desc *desc, const float *theta_v, const float *theta_p,
                          const uint32_t *occ, const float *mlp, const merf_camera *cams,
                          int32_t n_cams, int32_t W, int32_t H, const float *target, float *rgb_out,
                          float *grad_v, float *grad_p, double *loss, int32_t *overflow, int64_t *n_samples,
                          void *stream);

#ifdef __cplusplus
}
#endif

#endif /* MERF_H_ */
