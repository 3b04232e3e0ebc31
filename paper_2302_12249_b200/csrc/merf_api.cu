// merf_api.cu -- the C ABI of libmerf (include/merf.h): validation, device memory, launch
// plumbing.  No compute happens here; every step of the path runs in the kernels of
// merf_render.cu / merf_build.cu.
#include <cstdarg>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: no-ops unless a tool (nsys, ncu --nvtx) attaches

#include "../../include/merf.h"
#include "merf_device.cuh"
#include "merf_kernels.h"
#include "merf_render_kernel.cuh"

using namespace merf;

struct merf_scene {
    merf_scene_desc desc;
    DevScene dev;
    MlpParams mlp_params;          // host copy of the MLP weights (shade kernel parameter)
    int device;
    int64_t n_blocks;
    int64_t canonical_blocks;
    int64_t device_bytes;
    std::vector<void*> allocs;
    // staging for merf_render_host (lazily allocated, guarded by the caller's usage)
    void* stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    // merf_render_host_async: two device frame buffers alternating between calls, each with
    // the event of its last device -> host copy (on copy_stream)
    void* astage[2] = {nullptr, nullptr};
    size_t astage_bytes = 0;
    int abuf = 0;
    cudaEvent_t acopied[2] = {nullptr, nullptr};
    bool apending[2] = {false, false};
    // per-tile march durations of the last single-chunk small call (Workspace::tile_cost):
    // the next call with the same W, H and views dispatches its tiles longest first
    uint16_t* hist = nullptr;
    int64_t hist_cap = 0;
    int hist_W = 0, hist_H = 0, hist_views = 0;
    bool hist_valid = false;
    std::mutex hmu;
    // MERF_TIMED bookkeeping: (kind, start, end) of launches not yet collected
    struct Timed { int kind; cudaEvent_t a, b; };
    std::mutex tmu;
    std::vector<Timed> timed;
    merf_kernel_times acc{};
};

// Every entry point that takes a scene runs on the scene's device: the guard makes it current
// for the call (kernels, stream-ordered workspaces, grid-size caches) and restores the caller's.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const merf_scene* s);
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

static thread_local std::string g_err;

DeviceGuard::DeviceGuard(const merf_scene* s) {
    if (!s) return;
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != s->device && cudaSetDevice(s->device) == cudaSuccess)
        prev = cur;
}

static merf_status fail(merf_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

merf_status merf_set_error(merf_status s, const char* msg) {   // for the other translation units
    g_err = msg;
    return s;
}

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            return fail(_e == cudaErrorMemoryAllocation ? MERF_ENOMEM : MERF_ECUDA,       \
                        "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
    } while (0)

static const int kSkipTabMaxRes = 512;



static bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
static int ilog2i(int64_t v) { int n = 0; while ((int64_t(1) << n) < v) n++; return n; }
static int64_t occ_words(int N) { return ((int64_t)N * N * N + 31) / 32; }

extern "C" const char* merf_last_error(void) { return g_err.c_str(); }
extern "C" int32_t merf_version(void) { return 100; }

// keep call workspaces cached in the device's stream-ordered pool between calls (no
// re-mapping of pages per call)
static int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

static void keep_pool_cached(int device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
}

static merf_status validate_desc(const merf_scene_desc* d) {
    if (!d) return fail(MERF_EINVAL, "desc is NULL");
    if (d->C != 8) return fail(MERF_EINVAL, "C must be 8 (got %d)", d->C);
    if (d->L != 0 && (!is_pow2(d->L) || d->L < 8))
        return fail(MERF_EINVAL, "L must be 0 or a power of two >= 8 (got %d)", d->L);
    if (d->R != 0 && (!is_pow2(d->R) || d->R < 2))
        return fail(MERF_EINVAL, "R must be 0 or a power of two >= 2 (got %d)", d->R);
    if (d->L == 0 && d->R == 0) return fail(MERF_EINVAL, "scene has neither grid nor planes");
    if (d->L > 4096 || d->R > 65536) return fail(MERF_EINVAL, "L or R too large");
    if (d->n_levels < 1 || d->n_levels > MERF_MAX_LEVELS)
        return fail(MERF_EINVAL, "n_levels must be in [1, %d]", MERF_MAX_LEVELS);
    for (int i = 0; i < d->n_levels; i++) {
        int N = d->level_res[i];
        if (!is_pow2(N) || N > 4096) return fail(MERF_EINVAL, "level_res[%d] = %d not a power of two <= 4096", i, N);
        if (i > 0 && (N % d->level_res[i - 1]) != 0)
            return fail(MERF_EINVAL, "level_res[%d] does not divide level_res[%d]", i - 1, i);
    }
    if (!(d->step > 0.0)) return fail(MERF_EINVAL, "step must be > 0");
    int e;
    double m = frexp(d->step, &e);
    if (m != 0.5 || d->step > 1.0 || d->step < 1e-6)
        return fail(MERF_EINVAL, "step must be a power of two in [2^-19, 1] (got %g)", d->step);
    if (!(d->t_min >= 0.f && d->t_min < 1.f)) return fail(MERF_EINVAL, "t_min must be in [0, 1)");
    if (!(d->m_density > 0.f && d->m_appearance > 0.f)) return fail(MERF_EINVAL, "m must be > 0");
    return MERF_OK;
}

static void fill_dev(merf_scene* s) {
    const merf_scene_desc& d = s->desc;
    DevScene& S = s->dev;
    S.L = (d.source_mask & 1u) ? d.L : 0;
    S.R = (d.source_mask & 14u) ? d.R : 0;
    S.nb = S.L / 8;
    S.n_levels = d.n_levels;
    for (int i = 0; i < MERF_MAX_LEVELS; i++) {
        S.level_res[i] = i < d.n_levels ? d.level_res[i] : 1;
        S.level_shift[i] = kF + 2 - ilog2i(S.level_res[i]);
    }
    S.n_fin = S.level_res[S.n_levels - 1];
    S.s_fin = S.level_shift[S.n_levels - 1];
    S.sV = S.L ? kF + 2 - ilog2i(S.L) : 0;
    S.sP = S.R ? kF + 2 - ilog2i(S.R) : 0;
    S.kd = (float)(2.0 * d.m_density / 255.0);
    S.ka = (float)(2.0 * d.m_appearance / 255.0);
    S.md = d.m_density;
    S.ma = d.m_appearance;
    {
        const double l2e = 1.4426950408889634;
        S.kd_l2 = (float)(2.0 * d.m_density / 255.0 * l2e);
        S.kd_l2w = (float)(2.0 * d.m_density / 255.0 * l2e / 65535.0);
        S.md_l2 = (float)(d.m_density * l2e);
        S.log2_step = (float)std::log2(d.step);
        S.ka_l2n = (float)(-2.0 * d.m_appearance / 255.0 / 65535.0 * l2e);
        S.ma_l2 = (float)(d.m_appearance * l2e);
        // the device's fp32 fmaf / product with n = 4, evaluated exactly as the kernel would
        // (fma rounds once: std::fma on floats), so the folded constants change no bit
        S.dens_off4 = std::fma(4.0f, -S.md_l2, S.log2_step);
        S.ma_l2_4 = 4.0f * S.ma_l2;
    }
    S.use_v = S.L > 0;
    for (int a = 0; a < 3; a++) S.use_p[a] = S.R > 0 && ((d.source_mask >> (1 + a)) & 1u);
    S.n_src = S.use_v + S.use_p[0] + S.use_p[1] + S.use_p[2];
    S.step = d.step;
    S.lattice_step = d.step * (double)kOne;
    S.inv_step = 1.0 / d.step;
    S.step_f = (float)d.step;
    S.t_min = d.t_min;
    S.alpha_skip = d.alpha_skip;
}

// Bound on every operand the tensor-core MLP (merf_shade_mma.cu) converts to fp16: the inputs
// are in [-1, 1] (C_d, F in [0, 1] since sum w <= 1; |d| = 1; sin, cos), so layer l's
// pre-activations are bounded by max_o |b_o| + sum_i |W_oi| * (bound of layer l - 1).
// NaN/inf weights give +inf (FFMA kernel).
static double mlp_mma_bound(const float* w) {
    const int nin[3] = {34, 16, 16}, nout[3] = {16, 16, 3}, woff[3] = {0, 560, 832}, boff[3] = {544, 816, 880};
    double in = 1.0, worst = 1.0;
    for (int l = 0; l < 3; l++) {
        double m = 0.0;
        for (int o = 0; o < nout[l]; o++) {
            double a = fabs((double)w[boff[l] + o]);
            for (int i = 0; i < nin[l]; i++) a += fabs((double)w[woff[l] + o * nin[l] + i]) * in;
            if (!(a <= 1e30)) return INFINITY;
            m = fmax(m, a);
        }
        in = m;
        worst = fmax(worst, m);
    }
    return worst;
}

template <typename T>
static merf_status dalloc(merf_scene* s, T** p, size_t bytes) {
    void* q = nullptr;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) return fail(MERF_ENOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    s->allocs.push_back(q);
    s->device_bytes += (int64_t)bytes;
    *p = reinterpret_cast<T*>(q);
    return MERF_OK;
}

extern "C" merf_status merf_scene_free(merf_scene* s) {
    if (!s) return MERF_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    cudaDeviceSynchronize();
    for (void* p : s->allocs) cudaFree(p);
    for (int i = 0; i < 2; i++) {
        if (s->stage[i]) cudaFree(s->stage[i]);
        if (s->ev[i]) cudaEventDestroy(s->ev[i]);
        if (s->astage[i]) cudaFree(s->astage[i]);
        if (s->acopied[i]) cudaEventDestroy(s->acopied[i]);
    }
    if (s->hist) cudaFree(s->hist);
    if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
    cudaSetDevice(prev);
    delete s;
    return MERF_OK;
}

extern "C" merf_status merf_scene_upload(const merf_scene_desc* desc, const uint8_t* planes,
                                         const int32_t* block_index, const uint8_t* atlas,
                                         int64_t n_blocks, const uint32_t* occ_finest,
                                         const float* mlp, int32_t device, merf_scene** out) {
    merf_status st = validate_desc(desc);
    if (st) return st;
    if (!out || !occ_finest || !mlp) return fail(MERF_EINVAL, "NULL out/occ_finest/mlp");
    const bool use_v = desc->L > 0 && (desc->source_mask & 1u);
    const bool use_p = desc->R > 0 && (desc->source_mask & 14u);
    if (!use_v && !use_p) return fail(MERF_EINVAL, "source_mask selects no stored source");
    if (use_p && !planes) return fail(MERF_EINVAL, "planes is NULL");
    if (use_v && (!atlas || n_blocks < 0)) return fail(MERF_EINVAL, "atlas is NULL or n_blocks < 0");
    if (use_v && n_blocks > (int64_t)INT32_MAX) return fail(MERF_EINVAL, "n_blocks too large");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(MERF_EINVAL, "device %d out of range", device);
    int prev = 0;
    cudaGetDevice(&prev);
    CUDA_TRY(cudaSetDevice(device));

    merf_scene* s = new merf_scene();
    s->desc = *desc;
    s->device = device;
    s->n_blocks = use_v ? n_blocks : 0;
    s->dev.n_blocks_dev = (int)s->n_blocks;
    fill_dev(s);
    DevScene& S = s->dev;
    auto bail = [&](merf_status e) { merf_scene_free(s); cudaSetDevice(prev); return e; };
#define UP_TRY(expr) do { merf_status _s = (expr); if (_s) return bail(_s); } while (0)
#define UPC_TRY(expr) do { cudaError_t _e = (expr); if (_e != cudaSuccess) \
        return bail(fail(_e == cudaErrorMemoryAllocation ? MERF_ENOMEM : MERF_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e))); } while (0)

    // Every upload step (host->device copies included) is ordered on this one stream:
    // a blocking cudaMemcpy from pageable memory may return before its DMA lands, so a
    // kernel on another stream could read stale device memory.
    cudaStream_t cs;
    UPC_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    keep_pool_cached(device);
    // ---- MLP weights
    float* d_mlp;
    UP_TRY(dalloc(s, &d_mlp, kMlpFloats * sizeof(float)));
    UPC_TRY(cudaMemcpyAsync(d_mlp, mlp, kMlpFloats * sizeof(float), cudaMemcpyHostToDevice, cs));
    S.mlp = d_mlp;
    memcpy(s->mlp_params.w, mlp, sizeof(s->mlp_params.w));
    S.mlp_frag = nullptr;
    if (mlp_mma_bound(mlp) < 3e4) {        // fp16 operand range of the tensor-core MLP
        uint32_t* d_frag;
        UP_TRY(dalloc(s, &d_frag, 32 * kMlpFragWords * sizeof(uint32_t)));
        UPC_TRY(launch_mlp_frag(d_mlp, d_frag, cs));
        S.mlp_frag = d_frag;
    }
    // ---- planes
    if (use_p) {
        size_t pb = (size_t)3 * desc->R * desc->R * 8;
        uint8_t* d_pl;                         // AoS staging, freed once the layouts are built
        UPC_TRY(cudaMallocAsync((void**)&d_pl, pb, cs));
        UPC_TRY(cudaMemcpyAsync(d_pl, planes, pb, cudaMemcpyHostToDevice, cs));
        uint4* d_pp;
        // [3][R + 1][R]: row R of each plane repeats row R - 1 (the upper-edge corner, texel())
        const size_t ppb = (size_t)3 * (desc->R + 1) * desc->R * 16;
        UP_TRY(dalloc(s, &d_pp, ppb));
        UPC_TRY(launch_pack_pairs(d_pl, desc->R, d_pp, nullptr, 0, nullptr, cs));
        S.plane_pairs = d_pp;
        UPC_TRY(cudaFreeAsync(d_pl, cs));
    }
    // ---- occupancy pyramid (K0)
    const int nl = desc->n_levels;
    const int Nf = desc->level_res[nl - 1];
    uint32_t* d_occ[MERF_MAX_LEVELS] = {nullptr, nullptr, nullptr, nullptr};
    for (int i = 0; i < nl; i++) UP_TRY(dalloc(s, &d_occ[i], occ_words(desc->level_res[i]) * 4));
    UPC_TRY(cudaMemcpyAsync(d_occ[nl - 1], occ_finest, occ_words(Nf) * 4, cudaMemcpyHostToDevice, cs));
    for (int i = nl - 2; i >= 0; i--)       // each level from the next finer one (nested)
        UPC_TRY(launch_maxpool_bits(d_occ[i + 1], desc->level_res[i + 1], d_occ[i], desc->level_res[i], cs));
    for (int i = 0; i < MERF_MAX_LEVELS; i++) S.occ[i] = d_occ[i < nl ? i : nl - 1];
    S.occ_fin = d_occ[nl - 1];
    S.skiptab = nullptr;
    if (Nf <= kSkipTabMaxRes && Nf >= 2) {    // 1 byte per bordered finest cell (136 MB at 512^3)
        uint32_t* d_tab;
        UP_TRY(dalloc(s, &d_tab, (size_t)skiptab_words(Nf) * 4));
        UPC_TRY(launch_skiptab(d_occ[nl - 1], Nf, d_tab, cs));
        S.skiptab = d_tab;
    }
    // ---- block index (K1) + atlas
    if (use_v) {
        const int64_t slots = (int64_t)(desc->L / 8) * (desc->L / 8) * (desc->L / 8);
        uint8_t* d_need;
        int32_t* d_idx;
        int32_t* d_scan;
        int64_t* d_count;
        unsigned long long* d_bad;
        UPC_TRY(cudaMalloc(&d_need, slots));
        UPC_TRY(cudaMalloc(&d_scan, slots * 8));
        UPC_TRY(cudaMalloc(&d_count, 16));
        UPC_TRY(cudaMalloc(&d_bad, 16));
        UP_TRY(dalloc(s, &d_idx, slots * 4));
        size_t tb = 0;
        UPC_TRY(launch_block_number(nullptr, slots, nullptr, nullptr, nullptr, &tb, nullptr, cs));
        void* d_tmp;
        UPC_TRY(cudaMalloc(&d_tmp, tb + 16));
        UPC_TRY(launch_block_need(d_occ[nl - 1], Nf, desc->L, d_need, cs));
        int64_t canon = 0;
        if (block_index) {
            UPC_TRY(cudaMemcpyAsync(d_idx, block_index, slots * 4, cudaMemcpyHostToDevice, cs));
            int32_t* d_canon;
            UPC_TRY(cudaMalloc(&d_canon, slots * 4));
            UPC_TRY(launch_block_number(d_need, slots, d_canon, d_count, d_tmp, &tb, d_scan, cs));
            UPC_TRY(cudaStreamSynchronize(cs));
            cudaFree(d_canon);
        } else {
            UPC_TRY(launch_block_number(d_need, slots, d_idx, d_count, d_tmp, &tb, d_scan, cs));
        }
        UPC_TRY(cudaMemsetAsync(d_bad, 0, 8, cs));
        UPC_TRY(launch_block_check(d_need, d_idx, slots, n_blocks, d_bad, cs));
        unsigned long long bad = 0;
        UPC_TRY(cudaMemcpyAsync(&canon, d_count, 8, cudaMemcpyDeviceToHost, cs));
        UPC_TRY(cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, cs));
        UPC_TRY(cudaStreamSynchronize(cs));
        cudaFree(d_need); cudaFree(d_scan); cudaFree(d_count); cudaFree(d_bad); cudaFree(d_tmp);
        s->canonical_blocks = canon;
        if (!block_index && canon != n_blocks)
            return bail(fail(MERF_EMISMATCH, "canonical allocation needs %lld blocks, atlas has %lld",
                             (long long)canon, (long long)n_blocks));
        if (bad)
            return bail(fail(MERF_EMISMATCH, "block index unsound or out of range at %llu slots "
                                             "(an occupied cell's block is missing)", bad));
        size_t ab = (size_t)n_blocks * 729 * 8;
        uint8_t* d_at = nullptr;               // AoS staging, freed once the layouts are built
        if (ab) {
            UPC_TRY(cudaMallocAsync((void**)&d_at, ab, cs));
            UPC_TRY(cudaMemcpyAsync(d_at, atlas, ab, cudaMemcpyHostToDevice, cs));
        }
        S.block_index = d_idx;
        // outside-the-grid aprons of edge blocks repeat the edge voxels (texel(), D9)
        if (d_at) UPC_TRY(launch_apron_edge(d_idx, desc->L, n_blocks, d_at, cs));
        uint4* d_ap;
        UP_TRY(dalloc(s, &d_ap, (size_t)n_blocks * 648 * 16));
        if (n_blocks) UPC_TRY(launch_pack_pairs(nullptr, 0, nullptr, d_at, n_blocks, d_ap, cs));
        S.atlas_pairs = d_ap;
        if (d_at) UPC_TRY(cudaFreeAsync(d_at, cs));
    }
    UPC_TRY(cudaStreamSynchronize(cs));
    cudaStreamDestroy(cs);
    cudaSetDevice(prev);
    *out = s;
    return MERF_OK;
#undef UP_TRY
#undef UPC_TRY
}

extern "C" merf_status merf_scene_info_get(const merf_scene* s, merf_scene_info* info) {
    if (!s || !info) return fail(MERF_EINVAL, "NULL argument");
    memset(info, 0, sizeof(*info));
    info->L = s->dev.L;
    info->R = s->dev.R;
    info->C = 8;
    info->n_levels = s->desc.n_levels;
    for (int i = 0; i < MERF_MAX_LEVELS; i++) info->level_res[i] = s->desc.level_res[i];
    info->n_blocks = s->n_blocks;
    info->canonical_blocks = s->canonical_blocks;
    info->device_bytes = s->device_bytes;
    info->device = s->device;
    return MERF_OK;
}

extern "C" merf_status merf_scene_occupancy(const merf_scene* s, int32_t level, uint32_t* bits_out,
                                            void* stream) {
    if (!s || !bits_out) return fail(MERF_EINVAL, "NULL argument");
    DeviceGuard dg(s);
    if (level < 0 || level >= s->desc.n_levels) return fail(MERF_EINVAL, "level out of range");
    CUDA_TRY(cudaMemcpyAsync(bits_out, s->dev.occ[level], occ_words(s->desc.level_res[level]) * 4,
                             cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return MERF_OK;
}

extern "C" merf_status merf_scene_block_index(const merf_scene* s, int32_t* index_out, void* stream) {
    if (!s || !index_out) return fail(MERF_EINVAL, "NULL argument");
    DeviceGuard dg(s);
    if (!s->dev.L) return fail(MERF_EINVAL, "scene has no 3D grid");
    int64_t slots = (int64_t)s->dev.nb * s->dev.nb * s->dev.nb;
    CUDA_TRY(cudaMemcpyAsync(index_out, s->dev.block_index, slots * 4, cudaMemcpyDeviceToDevice,
                             (cudaStream_t)stream));
    return MERF_OK;
}

static merf_status check_frames(const merf_scene* s, const merf_camera* cams, int32_t n_cams,
                                int32_t W, int32_t H, int32_t format, const void* out) {
    if (!s || !cams || !out) return fail(MERF_EINVAL, "NULL scene/cams/out");
    if (n_cams <= 0 || W <= 0 || H <= 0) return fail(MERF_EINVAL, "n_cams, W, H must be > 0");
    if ((int64_t)W * H * n_cams > ((int64_t)1 << 31)) return fail(MERF_EINVAL, "W*H*n_cams too large");
    if (H > 65535 * 8) return fail(MERF_EINVAL, "H too large");
    if (format != MERF_RGB_F32 && format != MERF_RGBA_U8) return fail(MERF_EINVAL, "bad format %d", format);
    for (int i = 0; i < n_cams; i++)
        if (!(cams[i].fx > 0 && cams[i].fy > 0 && cams[i].t_near >= 0))
            return fail(MERF_EINVAL, "camera %d: fx, fy must be > 0 and t_near >= 0", i);
    return MERF_OK;
}

static void to_stats(const unsigned long long* h, merf_stats* st) {
    st->rays = (int64_t)h[0];
    st->segments = (int64_t)h[1];
    st->evaluated = (int64_t)h[2];
    st->density_only = (int64_t)h[3];
    st->skips = (int64_t)h[4];
    st->missing_blocks = (int64_t)h[5];
    for (int g = 0; g < 7; g++) st->region_segments[g] = (int64_t)h[6 + g];
    st->march_rounds = (int64_t)h[13];
    st->march_steps = (int64_t)h[14];
    st->march_lane_rounds = (int64_t)h[15];
    st->march_busy_ns = (int64_t)h[19];
    st->march_tail_ns = (int64_t)h[20];
}

// ------------------------------------------------------------------------------------
// render pipeline orchestration: per chunk of rays, setup -> persistent march -> shade
// ------------------------------------------------------------------------------------
// views per pipeline chunk (one persistent march launch): 16 1080p views = 33 M rays, an
// 8.6 GB workspace (~257 B per ray in flight); fewer, longer launches amortise the tail of
// the persistent march (measured: 4 -> 937, 8 -> 960, 16 -> 973 M rays/s)
static const int64_t kChunkRays = int64_t(1) << 25;
static const int kViewsPerChunk = 16;
// experiment hook: MERF_CHUNK_VIEWS=<n> overrides the views per chunk (and scales the ray cap)
static int chunk_views() {
    static const int v = [] {
        const char* e = getenv("MERF_CHUNK_VIEWS");
        const int n = e ? atoi(e) : 0;
        return (n >= 1 && n <= kMaxCams) ? n : kViewsPerChunk;
    }();
    return v;
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// workspace bytes of a chunk of n rays (shared with
// merf_render_workspace_bytes so that the reported figure is the allocated one)
static size_t ws_tiles(int64_t n) { return (size_t)((n + 31) / 32); }
static size_t ws_bytes(int64_t n, int slots) {
    return align256((size_t)n * slots * 32) + align256((size_t)n) + align256((size_t)n * 32) + 256
           + align256(ws_tiles(n) * kBuckets * 4) + 256;
}

// segment slots per ray for a chunk of these cameras: kMaxSegCore if every origin is in the
// core (||o||_inf <= 1, o = the c2w translation), else kMaxSeg (merf_device.cuh)
static int seg_slots_for(const merf_camera* cams, int n) {
    if (!cams) return kMaxSeg;
    for (int i = 0; i < n; i++) {
        const double* m = cams[i].c2w;
        if (!(std::fabs(m[3]) <= 1.0 && std::fabs(m[7]) <= 1.0 && std::fabs(m[11]) <= 1.0)) return kMaxSeg;
    }
    return kMaxSegCore;
}

// Tile dispatch order.  Single-chunk calls of at most kHistMaxViews views keep the march's
// per-tile durations in the scene (Workspace::tile_cost); the next such call with the same W, H
// and views -- the next frame of a sequence -- dispatches its tiles longest first by them
// (exact costs of the previous frame: its heaviest tiles start at once instead of at 65 % of
// the queue).  MERF_TILE_ORDER=raster turns this off; MERF_TILE_ORDER=cost uses the
// centre-ray probe estimate (below) for every call instead.  Otherwise raster order.  Measured on 1080p orbit views (tools/view_scaling.py, r02 final
// kernels): the march's tail (tile queue dry -> last warp exit) drops from 0.33-0.45 ms to
// 0.09-0.29 ms and the march per view by 0.5-3 %, but the estimate adds 0.05 ms of setup per
// view, so the call is 0.5-3 % slower at every batch size from 1 to 16 views.  (An earlier
// policy used it for <= 4 views on a measurement that predates the setup-instance split.)
static const int kLptMaxViews = 0;
static const int kHistMaxViews = 4;
static bool fused_mlp() {
    static const bool v = [] { const char* e = getenv("MERF_FUSED_MLP"); return e && e[0] == '1'; }();
    return v;
}
static int tile_order_override() {                   // 0 = policy, 1 = raster, 2 = cost
    static const int v = [] {
        const char* e = getenv("MERF_TILE_ORDER");
        if (!e) return 0;
        if (!strcmp(e, "raster")) return 1;
        if (!strcmp(e, "cost")) return 2;
        return 0;
    }();
    return v;
}
static bool cost_order(int views_per_chunk) {
    const int o = tile_order_override();
    return o == 2 || (o == 0 && views_per_chunk <= kLptMaxViews);
}

static merf_status ws_alloc(int64_t n, cudaStream_t st, Workspace& ws, void** base, int slots = kMaxSeg) {
    const size_t seg = align256((size_t)n * slots * 32);
    ws.seg_slots = slots;
    const size_t ns = align256((size_t)n);
    const size_t acc = align256((size_t)n * 32);
    CUDA_TRY(cudaMallocAsync(base, ws_bytes(n, slots), st));
    static const bool poison = getenv("MERF_DEBUG_POISON") != nullptr;   // debug: NaN-fill
    if (poison) CUDA_TRY(cudaMemsetAsync(*base, 0xFF, ws_bytes(n, slots), st));
    char* b = (char*)*base;
    ws.seg = (int4*)b;
    ws.nseg = (uint8_t*)(b + seg);
    ws.accum = (float4*)(b + seg + ns);
    ws.queue = (unsigned int*)(b + seg + ns + acc);
    ws.bucket_cnt = (unsigned int*)(b + seg + ns + acc + 128);
    ws.tile_list = (int*)(b + seg + ns + acc + 256);   // cost order available; the caller may clear it
    ws.n_tiles = (int)ws_tiles(n);
    ws.tile_cost = nullptr;
    return MERF_OK;
}

// NVTX range over a host scope (pipeline stage names: "merf_render", "setup", "march", ...),
// so nsys timelines and `ncu --nvtx --nvtx-include` select the paper's pipeline stages
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static merf_status timed_launch(const merf_scene* cs, uint32_t flags, int kind, cudaStream_t st,
                                cudaError_t (*fn)(void*), void* arg) {
    static const char* const kStage[3] = {"merf.setup", "merf.march", "merf.shade"};
    NvtxRange nv(kStage[kind < 0 || kind > 2 ? 1 : kind]);
    merf_scene* s = const_cast<merf_scene*>(cs);
    if (!(flags & MERF_TIMED)) {
        CUDA_TRY(fn(arg));
        return MERF_OK;
    }
    merf_scene::Timed t{kind, nullptr, nullptr};
    CUDA_TRY(cudaEventCreate(&t.a));
    CUDA_TRY(cudaEventCreate(&t.b));
    CUDA_TRY(cudaEventRecord(t.a, st));
    CUDA_TRY(fn(arg));
    CUDA_TRY(cudaEventRecord(t.b, st));
    std::lock_guard<std::mutex> g(s->tmu);
    s->timed.push_back(t);
    return MERF_OK;
}

struct ChunkCall {
    const merf_scene* s;
    int kf_setup, kf_march, kf_shade;
    const RaySource* rs;
    const Workspace* ws;
    void* out;
    uint32_t flags;
    const TraceArgs* ta;
    unsigned long long* d_stats;
    cudaStream_t st;
};

static cudaError_t call_setup(void* p) {
    ChunkCall* c = (ChunkCall*)p;
    return launch_setup(c->kf_setup, c->s->dev, *c->rs, *c->ws, *c->ta, c->d_stats, c->st);
}
static cudaError_t call_march(void* p) {
    ChunkCall* c = (ChunkCall*)p;
    return launch_march(c->kf_march, c->s->dev, c->rs->n, *c->ws, c->flags, *c->ta, c->d_stats, c->st, *c->rs, c->out);
}
static cudaError_t call_march_sph(void* p) {
    ChunkCall* c = (ChunkCall*)p;
    // the setup-variant flags carry RAYS/TRACE/COUNT for the single-kernel spherical path
    return launch_march_sph(c->kf_setup, c->s->dev, *c->rs, *c->ws, c->flags, *c->ta, c->d_stats, c->st);
}
static cudaError_t call_shade(void* p) {
    ChunkCall* c = (ChunkCall*)p;
    return launch_shade(c->kf_shade, c->s->dev, *c->rs, *c->ws, c->out, c->s->mlp_params,
                        (c->flags & MERF_MLP_FFMA) != 0, c->st);
}

static merf_status run_chunk(const merf_scene* s, int kf_setup, int kf_march, int kf_shade,
                             const RaySource& rs, const Workspace& ws_in, void* out, uint32_t flags,
                             const TraceArgs& ta, unsigned long long* d_stats, cudaStream_t st) {
    Workspace ws = ws_in;
    ws.n_tiles = (int)ws_tiles(rs.n);                 // this chunk's tiles
    // fused deferred-MLP epilogue in the march (KF_FUSED): camera rays of the production
    // instance, not the progressive preview fill nor the FFMA ablation (MERF_FUSED_MLP=0/1)
    if (fused_mlp() && kf_march >= 0 && kf_shade >= 0 && !(kf_march & (KF_DENSE | KF_TRACE)) &&
        !(kf_setup & (KF_RAYS | KF_TRACE | KF_SEGS)) && !rs.fill && !(flags & (MERF_MLP_FFMA | MERF_SPHERICAL)) &&
        fused_march_ok(s->dev) && !(kf_march & KF_COUNT)) {
        kf_march = KF_FUSED | (kf_shade & KF_U8);
        kf_shade = -1;
    }
    if ((flags & MERF_SPHERICAL) && (flags & MERF_SPH_PERSISTENT) && !(kf_setup & (KF_TRACE | KF_SEGS))) {
        kf_setup |= KF_SPH;                // like-for-like: the persistent pipeline, fp32 curve steps
        if (kf_march >= 0) kf_march = KF_SPH | (kf_march & KF_COUNT);
        flags &= ~(uint32_t)MERF_SPHERICAL;
    }
    // longest-first dispatch: the setup instance that also files every tile under its cost bucket
    if (ws.tile_list && !(kf_setup & (KF_RAYS | KF_TRACE | KF_SEGS | KF_SPH))) kf_setup |= KF_LPT;
    ChunkCall c{s, kf_setup, kf_march, kf_shade, &rs, &ws, out, flags, &ta, d_stats, st};
    if (flags & MERF_SPHERICAL) {          // NEXT-2 variant: no setup kernel, one march kernel
        merf_status e = timed_launch(s, flags, 1, st, call_march_sph, &c);
        if (e) return e;
        if (kf_shade >= 0 && (e = timed_launch(s, flags, 2, st, call_shade, &c))) return e;
        return MERF_OK;
    }
    if (ws.tile_list) CUDA_TRY(cudaMemsetAsync(ws.bucket_cnt, 0, kBuckets * sizeof(unsigned int), st));
    merf_status e = timed_launch(s, flags, 0, st, call_setup, &c);
    if (e) return e;
    if (kf_march >= 0 && (e = timed_launch(s, flags, 1, st, call_march, &c))) return e;
    if (kf_march >= 0 && d_stats) CUDA_TRY(launch_stats_fold(d_stats, st));
    if (kf_shade >= 0 && (e = timed_launch(s, flags, 2, st, call_shade, &c))) return e;
    return MERF_OK;
}

extern "C" merf_status merf_kernel_times_get(merf_scene* s, merf_kernel_times* out, int32_t reset) {
    if (!s || !out) return fail(MERF_EINVAL, "NULL argument");
    DeviceGuard dg(s);
    std::lock_guard<std::mutex> g(s->tmu);
    for (auto& t : s->timed) {
        CUDA_TRY(cudaEventSynchronize(t.b));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, t.a, t.b));
        if (t.kind == 0) { s->acc.setup_ms += ms; s->acc.setup_launches++; }
        if (t.kind == 1) { s->acc.march_ms += ms; s->acc.march_launches++; }
        if (t.kind == 2) { s->acc.shade_ms += ms; s->acc.shade_launches++; }
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    s->timed.clear();
    *out = s->acc;
    if (reset) s->acc = merf_kernel_times{};
    return MERF_OK;
}

static int march_flags(uint32_t flags, bool count) {
    return ((flags & MERF_DENSE) ? KF_DENSE : 0) | (count ? KF_COUNT : 0);
}

struct Progressive {
    int stride, ox, oy, fill;
};

struct Shard {
    int rank, count;
    bool compact;          // output = this part's block slots (merf_render_shard_blocks)
};

static merf_status render_frames(const merf_scene* s, const merf_camera* cams, int32_t n_cams,
                                 int32_t W, int32_t H, int32_t format, void* out, uint32_t flags,
                                 cudaStream_t st, unsigned long long* d_stats,
                                 const Progressive* prog = nullptr, const Shard* shard = nullptr) {
    const size_t px_bytes = format == MERF_RGBA_U8 ? 4 : 12;
    RaySource rs{};
    rs.W = W;
    rs.H = H;
    int Wl = W, Hl = H;                    // pixel lattice covered by the rays
    if (prog) {
        rs.stride_m1 = prog->stride - 1;
        rs.ox = prog->ox;
        rs.oy = prog->oy;
        rs.fill = prog->fill;
        Wl = (W - prog->ox + prog->stride - 1) / prog->stride;
        Hl = (H - prog->oy + prog->stride - 1) / prog->stride;
    }
    set_tiles(rs, (Wl + kTileW - 1) / kTileW, ((Wl + kTileW - 1) / kTileW) * ((Hl + kTileH - 1) / kTileH));
    if (shard && (shard->count > 1 || shard->compact)) {   // 64x64 blocks interleaved by rank
        rs.part_n = shard->count;
        rs.part_r = shard->rank;
        rs.nbx = (W + 63) / 64;
        rs.n_pblocks = rs.nbx * ((H + 63) / 64);
        const int slots = (rs.n_pblocks + shard->count - 1) / shard->count;
        set_tiles(rs, rs.tiles_x, slots * kShardTiles);
        rs.compact = shard->compact ? 1 : 0;
        rs.part_slots = slots;
    }
    const int64_t rays_per_view = (int64_t)rs.tiles_per_view * 32;
    const int cv = chunk_views();
    int vpc = (int)(kChunkRays * cv / kViewsPerChunk / rays_per_view);
    vpc = vpc < 1 ? 1 : (vpc > cv ? cv : vpc);
    if (vpc > n_cams) vpc = n_cams;
    Workspace ws;
    void* base = nullptr;
    merf_status e = ws_alloc(rays_per_view * vpc, st, ws, &base, seg_slots_for(cams, n_cams));
    if (e) return e;
    int* const lists = ws.tile_list;
    if (!cost_order(vpc)) ws.tile_list = nullptr;
    // frame-sequence history (see kHistMaxViews): one chunk, small, full frames
    if (tile_order_override() == 0 && n_cams <= vpc && vpc <= kHistMaxViews && !prog && !shard &&
        !(flags & MERF_SPHERICAL)) {     // (the spherical variant's march records nothing)
        merf_scene* ms = const_cast<merf_scene*>(s);
        std::lock_guard<std::mutex> g(ms->hmu);
        const int64_t nt = (int64_t)ws_tiles(rays_per_view * n_cams);
        if (ms->hist_cap < nt) {
            if (ms->hist) {
                cudaError_t ce = cudaFree(ms->hist);   // (synchronises: no launch still uses it)
                if (ce != cudaSuccess) { cudaFreeAsync(base, st); return fail(MERF_ECUDA, "%s", cudaGetErrorString(ce)); }
            }
            ms->hist = nullptr;
            ms->hist_cap = 0;
            ms->hist_valid = false;
            if (cudaMalloc(&ms->hist, (size_t)nt * sizeof(uint16_t)) != cudaSuccess) {
                ms->hist = nullptr;
                cudaFreeAsync(base, st);
                return fail(MERF_ENOMEM, "tile-cost history allocation failed");
            }
            CUDA_TRY(cudaMemsetAsync(ms->hist, 0, (size_t)nt * sizeof(uint16_t), st));
            ms->hist_cap = nt;
        }
        const bool match = ms->hist_valid && ms->hist_W == W && ms->hist_H == H && ms->hist_views == n_cams;
        ws.tile_cost = ms->hist;
        ws.tile_list = match ? lists : nullptr;     // cost-ordered lists, else raster (recording)
        ms->hist_W = W;
        ms->hist_H = H;
        ms->hist_views = n_cams;
        ms->hist_valid = true;           // the march below records every tile (stream order)
    }
    const bool count = d_stats != nullptr;
    for (int c0 = 0; c0 < n_cams; c0 += vpc) {
        const int nv = n_cams - c0 < vpc ? n_cams - c0 : vpc;
        rs.cb.n = nv;
        for (int i = 0; i < nv; i++) rs.cb.cam[i] = cams[c0 + i];
        rs.ray0 = 0;
        rs.n = rays_per_view * nv;
        const size_t view_px = rs.compact ? (size_t)rs.part_slots * 4096 : (size_t)W * H;
        void* o = (char*)out + (size_t)c0 * view_px * px_bytes;
        TraceArgs ta{};
        e = run_chunk(s, count ? KF_COUNT : 0, march_flags(flags, count),
                      format == MERF_RGBA_U8 ? KF_U8 : 0, rs, ws, o, flags, ta, d_stats, st);
        if (e) { cudaFreeAsync(base, st); return e; }
    }
    CUDA_TRY(cudaFreeAsync(base, st));
    return MERF_OK;
}

extern "C" merf_status merf_render(const merf_scene* s, const merf_camera* cams, int32_t n_cams,
                                   int32_t W, int32_t H, int32_t format, void* out, uint32_t flags,
                                   void* stream, merf_stats* stats) {
    merf_status e = check_frames(s, cams, n_cams, W, H, format, out);
    if (e) return e;
    DeviceGuard dg(s);
    NvtxRange nv("merf_render");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* d_stats = nullptr;
    if (stats || (flags & MERF_COUNTERS)) {
        CUDA_TRY(cudaMallocAsync(&d_stats, kStatWords * sizeof(unsigned long long), st));
        CUDA_TRY(cudaMemsetAsync(d_stats, 0, kStatWords * sizeof(unsigned long long), st));
        CUDA_TRY(cudaMemsetAsync(d_stats + 16, 0xFF, 2 * sizeof(unsigned long long), st));   // min slots
    }
    e = render_frames(s, cams, n_cams, W, H, format, out, flags, st, d_stats);
    if (e) return e;
    if (d_stats) {
        unsigned long long h[kStatWords];
        CUDA_TRY(cudaMemcpyAsync(h, d_stats, sizeof(h), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaFreeAsync(d_stats, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (stats) to_stats(h, stats);
    }
    return MERF_OK;
}

extern "C" merf_status merf_render_workspace_bytes(const merf_scene* s, const merf_camera* cams, int32_t n_cams,
                                                   int32_t W, int32_t H, int64_t* bytes, int64_t* rays_per_chunk) {
    if (!s || !bytes || n_cams <= 0 || W <= 0 || H <= 0) return fail(MERF_EINVAL, "bad arguments");
    const int64_t tiles = (int64_t)((W + kTileW - 1) / kTileW) * ((H + kTileH - 1) / kTileH);
    const int64_t rays_per_view = tiles * 32;
    const int cv = chunk_views();
    int64_t vpc = kChunkRays * cv / kViewsPerChunk / rays_per_view;
    vpc = vpc < 1 ? 1 : (vpc > cv ? cv : vpc);
    if (vpc > n_cams) vpc = n_cams;
    *bytes = (int64_t)ws_bytes(rays_per_view * vpc, seg_slots_for(cams, n_cams));
    if (rays_per_chunk) *rays_per_chunk = rays_per_view * vpc;
    return MERF_OK;
}

extern "C" merf_status merf_render_shard(const merf_scene* s, const merf_camera* cams, int32_t n_cams,
                                         int32_t W, int32_t H, int32_t part_rank, int32_t part_count,
                                         int32_t format, void* out, uint32_t flags, void* stream) {
    merf_status e = check_frames(s, cams, n_cams, W, H, format, out);
    if (e) return e;
    DeviceGuard dg(s);
    NvtxRange nv("merf_render_shard");
    if (part_count < 1 || part_rank < 0 || part_rank >= part_count)
        return fail(MERF_EINVAL, "need 0 <= part_rank < part_count (got %d of %d)", part_rank, part_count);
    Shard sh{part_rank, part_count, false};
    return render_frames(s, cams, n_cams, W, H, format, out, flags & ~(uint32_t)MERF_COUNTERS,
                         (cudaStream_t)stream, nullptr, nullptr, &sh);
}

extern "C" merf_status merf_render_shard_blocks(const merf_scene* s, const merf_camera* cams, int32_t n_cams,
                                                int32_t W, int32_t H, int32_t part_rank, int32_t part_count,
                                                int32_t format, void* blocks_out, uint32_t flags, void* stream) {
    merf_status e = check_frames(s, cams, n_cams, W, H, format, blocks_out);
    if (e) return e;
    DeviceGuard dg(s);
    NvtxRange nv("merf_render_shard_blocks");
    if (part_count < 1 || part_rank < 0 || part_rank >= part_count)
        return fail(MERF_EINVAL, "need 0 <= part_rank < part_count (got %d of %d)", part_rank, part_count);
    Shard sh{part_rank, part_count, true};
    return render_frames(s, cams, n_cams, W, H, format, blocks_out, flags & ~(uint32_t)MERF_COUNTERS,
                         (cudaStream_t)stream, nullptr, nullptr, &sh);
}

extern "C" merf_status merf_render_progressive(const merf_scene* s, const merf_camera* cams, int32_t n_cams,
                                               int32_t W, int32_t H, int32_t stride, int32_t pass, int32_t fill,
                                               int32_t format, void* out, uint32_t flags, void* stream) {
    merf_status e = check_frames(s, cams, n_cams, W, H, format, out);
    if (e) return e;
    DeviceGuard dg(s);
    NvtxRange nv("merf_render_progressive");
    if (stride < 1 || stride > 64) return fail(MERF_EINVAL, "stride must be in [1, 64]");
    if (pass < 0 || pass >= stride * stride) return fail(MERF_EINVAL, "pass must be in [0, stride^2)");
    Progressive p{stride, pass % stride, pass / stride, fill ? 1 : 0};
    if (p.ox >= W || p.oy >= H) return MERF_OK;   // an empty sub-lattice (frame smaller than stride)
    return render_frames(s, cams, n_cams, W, H, format, out, flags, (cudaStream_t)stream, nullptr, &p);
}

extern "C" merf_status merf_render_host(const merf_scene* cs, const merf_camera* cams, int32_t n_cams,
                                        int32_t W, int32_t H, int32_t format, void* out_host,
                                        uint32_t flags, void* stream) {
    merf_status e = check_frames(cs, cams, n_cams, W, H, format, out_host);
    if (e) return e;
    DeviceGuard dg(cs);
    NvtxRange nv("merf_render_host");
    merf_scene* s = const_cast<merf_scene*>(cs);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t px_bytes = format == MERF_RGBA_U8 ? 4 : 12;
    const size_t frame = (size_t)W * H * px_bytes;
    // Chunk plan: big chunks (efficient persistent-march launches) whose copies hide behind
    // the next chunk's render, then a small last chunk so that only its short copy is exposed.
    static const int kTail = [] {
        const char* e = getenv("MERF_HOST_TAIL");
        const int v = e ? atoi(e) : 2;
        return v >= 1 ? v : 2;
    }();
    static const int kBig = [] {   // measured e2e (16 views): 4x4 960, 12+4 980, 14+2 989 M rays/s
        const char* e = getenv("MERF_HOST_BIG");
        const int v = e ? atoi(e) : 14;
        return v >= 1 ? v : 14;
    }();
    std::vector<int> plan;
    {
        const int tail = n_cams < kTail ? n_cams : kTail;
        int rem = n_cams - tail;
        while (rem > 0) {
            const int c = rem < kBig ? rem : kBig;
            plan.push_back(c);
            rem -= c;
        }
        plan.push_back(tail);
    }
    int chunk = 0;
    for (int c : plan) chunk = c > chunk ? c : chunk;
    const size_t need = frame * chunk;
    if (s->stage_bytes < need) {
        for (int i = 0; i < 2; i++) {
            if (s->stage[i]) cudaFree(s->stage[i]);
            s->stage[i] = nullptr;
        }
        s->stage_bytes = 0;
        for (int i = 0; i < 2; i++) CUDA_TRY(cudaMalloc(&s->stage[i], need));
        s->stage_bytes = need;
    }
    if (!s->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; i++)
        if (!s->ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&s->ev[i], cudaEventDisableTiming));
    cudaEvent_t copied[2];
    for (int i = 0; i < 2; i++) CUDA_TRY(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    bool pending[2] = {false, false};
    int b = 0;
    int c0 = 0;
    for (size_t pi = 0; pi < plan.size(); c0 += plan[pi], pi++, b ^= 1) {
        const int n = plan[pi];
        if (pending[b]) CUDA_TRY(cudaStreamWaitEvent(st, copied[b], 0));   // buffer free again
        e = render_frames(s, cams + c0, n, W, H, format, s->stage[b], flags, st, nullptr);
        if (e) return e;
        CUDA_TRY(cudaEventRecord(s->ev[b], st));
        CUDA_TRY(cudaStreamWaitEvent(s->copy_stream, s->ev[b], 0));
        CUDA_TRY(cudaMemcpyAsync((char*)out_host + (size_t)c0 * frame, s->stage[b], frame * n,
                                 cudaMemcpyDeviceToHost, s->copy_stream));
        CUDA_TRY(cudaEventRecord(copied[b], s->copy_stream));
        pending[b] = true;
    }
    CUDA_TRY(cudaStreamSynchronize(s->copy_stream));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int i = 0; i < 2; i++) cudaEventDestroy(copied[i]);
    return MERF_OK;
}

extern "C" merf_status merf_render_host_async(const merf_scene* cs, const merf_camera* cams, int32_t n_cams,
                                              int32_t W, int32_t H, int32_t format, void* out_host, uint32_t flags,
                                              void* stream) {
    merf_status e = check_frames(cs, cams, n_cams, W, H, format, out_host);
    if (e) return e;
    DeviceGuard dg(cs);
    NvtxRange nv("merf_render_host_async");
    merf_scene* s = const_cast<merf_scene*>(cs);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t px_bytes = format == MERF_RGBA_U8 ? 4 : 12;
    const size_t bytes = (size_t)W * H * px_bytes * n_cams;
    if (!s->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; i++)
        if (!s->acopied[i]) CUDA_TRY(cudaEventCreateWithFlags(&s->acopied[i], cudaEventDisableTiming));
    if (s->astage_bytes < bytes) {                 // grow both buffers once no copy reads them
        CUDA_TRY(cudaStreamSynchronize(s->copy_stream));
        for (int i = 0; i < 2; i++) {
            if (s->astage[i]) cudaFree(s->astage[i]);
            s->astage[i] = nullptr;
            s->apending[i] = false;
        }
        s->astage_bytes = 0;
        for (int i = 0; i < 2; i++) CUDA_TRY(cudaMalloc(&s->astage[i], bytes));
        s->astage_bytes = bytes;
    }
    const int b = s->abuf;
    s->abuf ^= 1;
    // the render may overwrite buffer b only after ITS previous copy (two calls back) is done
    if (s->apending[b]) CUDA_TRY(cudaStreamWaitEvent(st, s->acopied[b], 0));
    e = render_frames(s, cams, n_cams, W, H, format, s->astage[b], flags, st, nullptr);
    if (e) return e;
    cudaEvent_t rendered;
    CUDA_TRY(cudaEventCreateWithFlags(&rendered, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(rendered, st));
    CUDA_TRY(cudaStreamWaitEvent(s->copy_stream, rendered, 0));
    cudaEventDestroy(rendered);                    // released once the wait has been enqueued
    CUDA_TRY(cudaMemcpyAsync(out_host, s->astage[b], bytes, cudaMemcpyDeviceToHost, s->copy_stream));
    CUDA_TRY(cudaEventRecord(s->acopied[b], s->copy_stream));
    s->apending[b] = true;
    return MERF_OK;
}

extern "C" merf_status merf_host_wait(merf_scene* s) {
    if (!s) return fail(MERF_EINVAL, "NULL scene");
    DeviceGuard dg(s);
    if (s->copy_stream) CUDA_TRY(cudaStreamSynchronize(s->copy_stream));
    return MERF_OK;
}

extern "C" merf_status merf_render_rays(const merf_scene* s, const double* o, const double* d,
                                        const double* t_near, int64_t n, float* rgb, uint32_t flags,
                                        void* stream, merf_stats* stats) {
    if (!s || !o || !d || !rgb) return fail(MERF_EINVAL, "NULL argument");
    DeviceGuard dg(s);
    if (n < 0 || n > ((int64_t)1 << 31)) return fail(MERF_EINVAL, "bad ray count");
    if (n == 0) return MERF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* d_stats = nullptr;
    if (stats) {
        CUDA_TRY(cudaMallocAsync(&d_stats, kStatWords * sizeof(unsigned long long), st));
        CUDA_TRY(cudaMemsetAsync(d_stats, 0, kStatWords * sizeof(unsigned long long), st));
        CUDA_TRY(cudaMemsetAsync(d_stats + 16, 0xFF, 2 * sizeof(unsigned long long), st));   // min slots
    }
    {
        RaySource rs{};
        rs.o = o;
        rs.d = d;
        rs.t_near = t_near;
        const int64_t chunk = n < kChunkRays ? n : kChunkRays;
        Workspace ws;
        void* base = nullptr;
        merf_status e = ws_alloc(chunk, st, ws, &base);
        if (e) return e;
        if (tile_order_override() != 2) ws.tile_list = nullptr;   // explicit rays: caller's order
        const bool count = d_stats != nullptr;
        for (int64_t c0 = 0; c0 < n; c0 += chunk) {
            rs.ray0 = c0;
            rs.n = n - c0 < chunk ? n - c0 : chunk;
            TraceArgs ta{};
            e = run_chunk(s, KF_RAYS | (count ? KF_COUNT : 0), march_flags(flags, count), KF_RAYS, rs, ws,
                          rgb, flags, ta, d_stats, st);
            if (e) { cudaFreeAsync(base, st); return e; }
        }
        CUDA_TRY(cudaFreeAsync(base, st));
    }
    if (d_stats) {
        unsigned long long h[kStatWords];
        CUDA_TRY(cudaMemcpyAsync(h, d_stats, sizeof(h), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaFreeAsync(d_stats, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        to_stats(h, stats);
    }
    return MERF_OK;
}

extern "C" merf_status merf_trace(const merf_scene* s, const merf_camera* cam, int32_t W,
                                  const int64_t* pixel_ids, int64_t n, int32_t max_per_ray,
                                  uint64_t* cells_out, float* T_out, int32_t* counts_out,
                                  uint32_t flags, void* stream) {
    if (!s || !cam || !pixel_ids || !cells_out || !counts_out) return fail(MERF_EINVAL, "NULL argument");
    DeviceGuard dg(s);
    if (n < 0 || n > ((int64_t)1 << 31) || W <= 0 || max_per_ray < 0)
        return fail(MERF_EINVAL, "bad n / W / max_per_ray");
    if (!(cam->fx > 0 && cam->fy > 0 && cam->t_near >= 0)) return fail(MERF_EINVAL, "bad camera");
    if (n == 0) return MERF_OK;
    {
        cudaStream_t st = (cudaStream_t)stream;
        RaySource rs{};
        rs.cb.cam[0] = *cam;
        rs.cb.n = 1;
        rs.W = W;
        rs.pixel_ids = pixel_ids;
        rs.ray0 = 0;
        rs.n = n;
        Workspace ws;
        void* base = nullptr;
        merf_status e = ws_alloc(n, st, ws, &base);
        if (e) return e;
        ws.tile_list = nullptr;                      // pixel lists: the caller's order
        TraceArgs ta{cells_out, T_out, counts_out, max_per_ray, nullptr};
        e = run_chunk(s, KF_TRACE, KF_TRACE | ((flags & MERF_DENSE) ? KF_DENSE : 0), -1, rs, ws, nullptr,
                      flags, ta, nullptr, st);
        cudaFreeAsync(base, st);
        if (e) return e;
    }
    return MERF_OK;
}

extern "C" merf_status merf_segments(const merf_scene* s, const merf_camera* cam, int32_t W,
                                     const int64_t* pixel_ids, int64_t n, int32_t max_seg,
                                     merf_segment* segs_out, int32_t* counts_out, void* stream) {
    if (!s || !cam || !pixel_ids || !segs_out || !counts_out) return fail(MERF_EINVAL, "NULL argument");
    DeviceGuard dg(s);
    if (n < 0 || n > ((int64_t)1 << 31) || W <= 0 || max_seg < 0) return fail(MERF_EINVAL, "bad n / W / max_seg");
    if (!(cam->fx > 0 && cam->fy > 0 && cam->t_near >= 0)) return fail(MERF_EINVAL, "bad camera");
    if (n == 0) return MERF_OK;
    {
        RaySource rs{};
        rs.cb.cam[0] = *cam;
        rs.cb.n = 1;
        rs.W = W;
        rs.pixel_ids = pixel_ids;
        rs.ray0 = 0;
        rs.n = n;
        Workspace ws{};
        TraceArgs ta{nullptr, nullptr, counts_out, max_seg, segs_out};
        CUDA_TRY(launch_setup(KF_SEGS, s->dev, rs, ws, ta, nullptr, (cudaStream_t)stream));
    }
    return MERF_OK;
}

extern "C" merf_status merf_contract(const double* x, int64_t n, double* y, int32_t* region, void* stream) {
    if (n < 0) return fail(MERF_EINVAL, "n < 0");
    if (n > 0 && (!x || !y)) return fail(MERF_EINVAL, "NULL argument");
    CUDA_TRY(launch_contract(x, n, y, region, (cudaStream_t)stream));
    return MERF_OK;
}

extern "C" merf_status merf_build_occupancy(const uint32_t* finest_bits, const merf_scene_desc* desc,
                                            uint32_t* levels_out, void* stream) {
    merf_status e = validate_desc(desc);
    if (e) return e;
    if (!finest_bits || (!levels_out && desc->n_levels > 1)) return fail(MERF_EINVAL, "NULL argument");
    const int nl = desc->n_levels;
    keep_pool_cached(current_device());   // stream-ordered temporaries of the halving chain
    // offsets of the coarser levels in levels_out (coarse -> fine), built fine -> coarse, each
    // from the next finer one (levels are nested: each divides the next)
    int64_t off[MERF_MAX_LEVELS] = {0, 0, 0, 0};
    for (int i = 1; i < nl - 1; i++) off[i] = off[i - 1] + occ_words(desc->level_res[i - 1]);
    for (int i = nl - 2; i >= 0; i--) {
        const uint32_t* src = (i == nl - 2) ? finest_bits : levels_out + off[i + 1];
        CUDA_TRY(launch_maxpool_bits(src, desc->level_res[i + 1], levels_out + off[i], desc->level_res[i],
                                     (cudaStream_t)stream));
    }
    return MERF_OK;
}

extern "C" merf_status merf_build_block_index(const uint32_t* finest_bits, const merf_scene_desc* desc,
                                              int32_t* index_out, int64_t* n_blocks, void* stream) {
    merf_status e = validate_desc(desc);
    if (e) return e;
    if (!finest_bits || !index_out || !n_blocks) return fail(MERF_EINVAL, "NULL argument");
    if (desc->L <= 0) return fail(MERF_EINVAL, "L must be > 0");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t slots = (int64_t)(desc->L / 8) * (desc->L / 8) * (desc->L / 8);
    const int Nf = desc->level_res[desc->n_levels - 1];
    uint8_t* d_need = nullptr;
    int32_t* d_scan = nullptr;
    int64_t* d_count = nullptr;
    void* d_tmp = nullptr;
    size_t tb = 0;
    CUDA_TRY(launch_block_number(nullptr, slots, nullptr, nullptr, nullptr, &tb, nullptr, st));
    // stream-ordered temporaries from the (cached) default pool: no device-wide
    // cudaMalloc/cudaFree synchronisation per call
    keep_pool_cached(current_device());
    CUDA_TRY(cudaMallocAsync(&d_need, slots, st));
    CUDA_TRY(cudaMallocAsync(&d_scan, slots * 8, st));
    CUDA_TRY(cudaMallocAsync(&d_count, 16, st));
    CUDA_TRY(cudaMallocAsync(&d_tmp, tb + 16, st));
    CUDA_TRY(launch_block_need(finest_bits, Nf, desc->L, d_need, st));
    CUDA_TRY(launch_block_number(d_need, slots, index_out, d_count, d_tmp, &tb, d_scan, st));
    int64_t cnt = 0;
    CUDA_TRY(cudaMemcpyAsync(&cnt, d_count, 8, cudaMemcpyDeviceToHost, st));
    cudaFreeAsync(d_need, st); cudaFreeAsync(d_scan, st); cudaFreeAsync(d_count, st); cudaFreeAsync(d_tmp, st);
    CUDA_TRY(cudaStreamSynchronize(st));
    *n_blocks = cnt;
    return MERF_OK;
}

extern "C" merf_status merf_bake_occupancy(const double* x, const double* tau, const double* w, int64_t n,
                                           int32_t N, double step, double w_thr, double alpha_thr,
                                           uint32_t* bits_out, void* stream) {
    if (!bits_out || (n > 0 && (!x || !tau || !w))) return fail(MERF_EINVAL, "NULL argument");
    if (n < 0 || !is_pow2(N) || N < 2 || N > 4096) return fail(MERF_EINVAL, "bad n or N");
    if (!(step > 0.0) || !(alpha_thr > 0.0 && alpha_thr < 1.0)) return fail(MERF_EINVAL, "bad step / alpha_thr");
    const double tau_thr = -log1p(-alpha_thr) / step;
    CUDA_TRY(launch_bake_occupancy(x, tau, w, n, tau_thr, w_thr, N, bits_out, (cudaStream_t)stream));
    return MERF_OK;
}

extern "C" merf_status merf_pack_atlas(const uint8_t* dense, int32_t L, const int32_t* index, int64_t n_blocks,
                                       uint8_t* atlas_out, void* stream) {
    if (!dense || !index || (!atlas_out && n_blocks > 0)) return fail(MERF_EINVAL, "NULL argument");
    if (!is_pow2(L) || L < 8 || n_blocks < 0) return fail(MERF_EINVAL, "bad L or n_blocks");
    if (n_blocks == 0) return MERF_OK;
    CUDA_TRY(launch_pack_atlas(dense, L, index, n_blocks, atlas_out, (cudaStream_t)stream));
    return MERF_OK;
}

// ------------------------------------------------------------------------------------
// NEXT-3: quantisation-aware training step on toy dense grids (Eq. 7-8)
// ------------------------------------------------------------------------------------
extern "C" merf_status merf_qat_step(const merf_qat_desc* d, const float* theta_v, const float* theta_p,
                                     const uint32_t* occ, const float* mlp, const merf_camera* cams,
                                     int32_t n_cams, int32_t W, int32_t H, const float* target, float* rgb_out,
                                     float* grad_v, float* grad_p, double* loss, int32_t* overflow,
                                     int64_t* n_samples, void* stream) {
    if (!d || !theta_v || !theta_p || !occ || !mlp || !cams || !target || !rgb_out || !grad_v || !grad_p || !loss)
        return fail(MERF_EINVAL, "NULL argument");
    if (!is_pow2(d->L) || d->L < 2 || d->L > 1024 || !is_pow2(d->R) || d->R < 2 || d->R > 8192)
        return fail(MERF_EINVAL, "L, R must be powers of two in [2, 1024] / [2, 8192]");
    if (!is_pow2(d->occ_res) || d->occ_res < 2 || d->occ_res > 4096)
        return fail(MERF_EINVAL, "occ_res must be a power of two in [2, 4096]");
    if (d->max_samples < 1 || d->max_samples > (1 << 20)) return fail(MERF_EINVAL, "bad max_samples");
    int ex = 0;
    if (!(d->step > 0.0 && d->step <= 1.0) || std::frexp(d->step, &ex) != 0.5)
        return fail(MERF_EINVAL, "step must be a power of two in (0, 1]");
    if (!(d->m_density > 0.0) || !(d->m_appearance > 0.0)) return fail(MERF_EINVAL, "bad decode range m");
    if (n_cams <= 0 || n_cams > kMaxCams || W <= 0 || H <= 0) return fail(MERF_EINVAL, "bad n_cams, W or H");
    RaySource rs{};
    rs.W = W;
    rs.H = H;
    set_tiles(rs, (W + kTileW - 1) / kTileW, ((W + kTileW - 1) / kTileW) * ((H + kTileH - 1) / kTileH));
    rs.n = (int64_t)rs.tiles_per_view * 32 * n_cams;
    if (rs.n * d->max_samples > (int64_t(1) << 31)) return fail(MERF_EINVAL, "n_rays * max_samples > 2^31");
    rs.cb.n = n_cams;
    for (int i = 0; i < n_cams; i++) rs.cb.cam[i] = cams[i];
    DevScene S{};
    S.step = d->step;
    S.lattice_step = std::ldexp(d->step, kF);
    S.inv_step = 1.0 / d->step;
    cudaStream_t st = (cudaStream_t)stream;
    {
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        keep_pool_cached(dev);
    }
    const int64_t nv = (int64_t)d->L * d->L * d->L * 8, np = (int64_t)3 * d->R * d->R * 8;
    const size_t samp_b = align256((size_t)rs.n * d->max_samples * 48 + (size_t)rs.n * 64);   // + per-ray rows
    const size_t grid_b = align256((size_t)(nv + np) * 4);
    void* base = nullptr;
    Workspace ws;
    merf_status e = ws_alloc(rs.n, st, ws, &base);
    if (e) return e;
    char* scratch = nullptr;
    if (cudaMallocAsync((void**)&scratch, samp_b + 2 * grid_b + 256, st) != cudaSuccess) {
        cudaFreeAsync(base, st);
        return fail(MERF_ENOMEM, "QAT scratch allocation failed");
    }
    float* samp = (float*)scratch;
    float* rayb = samp + (size_t)rs.n * d->max_samples * 12;
    float* vv = (float*)(scratch + samp_b);
    float* vp = vv + nv;
    float* gvv = (float*)(scratch + samp_b + grid_b);
    float* gvp = gvv + nv;
    unsigned int* ovf = overflow ? (unsigned int*)overflow : (unsigned int*)(scratch + samp_b + 2 * grid_b);
    cudaError_t ce = cudaMemsetAsync(ovf, 0, 4, st);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(loss, 0, 8, st);
    if (ce == cudaSuccess && n_samples) ce = cudaMemsetAsync(n_samples, 0, 8, st);
    TraceArgs ta{};
    ws.tile_list = nullptr;                          // the QAT kernels walk rays in raster order
    if (ce == cudaSuccess) ce = launch_setup(0, S, rs, ws, ta, nullptr, st);
    if (ce == cudaSuccess)
        ce = launch_qat(S, rs, ws, theta_v, theta_p, vv, vp, d->quantize ? 1 : 0, target, rgb_out, gvv, gvp,
                        grad_v, grad_p, samp, d->max_samples, rayb, mlp, loss, ovf,
                        (unsigned long long*)n_samples, d->L, d->R, d->occ_res, occ,
                        (float)d->m_density, (float)d->m_appearance, st);
    cudaFreeAsync(scratch, st);
    cudaFreeAsync(base, st);
    if (ce != cudaSuccess) return fail(MERF_ECUDA, "%s", cudaGetErrorString(ce));
    return MERF_OK;
}
