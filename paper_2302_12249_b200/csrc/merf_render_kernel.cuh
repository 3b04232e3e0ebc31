// merf_render_kernel.cuh -- the hot path: one fused kernel per batch of views (sm_100a).
//
// Per ray (Sec. 6):
//   raygen (fp64)  ->  region segmentation of the world ray into <= 7 contracted segments
//     ->  per segment, integer lattice stepping Q_k = Qa + k U (reading D7-D8)
//   with coarse-to-fine occupancy probes; an empty cell jumps to the first lattice sample
//   outside it (the ray-AABB exit)  ->  evaluated samples gather 8 trilinear corners
//   of the block-sparse grid through the indirection table and 3 x 4 bilinear plane texels
//   (Eq. 5), density first; alpha = 1 - exp(-tau Delta); appearance only if
//   alpha > alpha_skip  ->  composite (Eq. 1-2) with termination at T < 2e-4
//   ->  deferred MLP h(C_d, F, d) per pixel (Eq. 3)  ->  store.
//
// Layout: one thread per ray; a warp covers an 8 x 4 pixel tile and a CTA 16 x 8 pixels so
// the 32 rays of a warp are spatially coherent (shared texels, shared occupancy words).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "merf_device.cuh"
#include "merf_kernels.h"

namespace merf {

enum : int {
    KF_TRACE = 1,       // write per-sample trace records
    KF_COUNT = 2,       // accumulate merf_stats counters
    KF_RAYS = 4,        // explicit rays instead of camera pixels
    KF_U8 = 8,          // RGBA8 output
    KF_DENSE = 16,      // dense stepping gated by the finest level (debug)
    KF_SEGS = 32,       // record contracted segments only (no marching)
};

struct RayArgs {
    const double* o;
    const double* d;
    const double* t_near;
    const int64_t* pixel_ids;   // trace mode: pixel list of camera 0
    int64_t n;
};

struct TraceArgs {
    uint64_t* cells;
    float* T;
    int32_t* counts;
    int max_per_ray;
    merf_segment* segs;
};

struct RayState {
    float T;
    float cd[3];
    float F[4];
    bool done;
    int last_cell;          // finest cell of the last evaluated sample (all levels known set)
    int n_eval;             // evaluated samples (trace index)
    // counters
    int c_eval, c_donly, c_skip, c_miss;
};

__device__ __forceinline__ void acc_texel(float acc[8], uint2 t, float w) {
    acc[0] = fmaf(w, (float)(t.x & 0xffu), acc[0]);
    acc[1] = fmaf(w, (float)((t.x >> 8) & 0xffu), acc[1]);
    acc[2] = fmaf(w, (float)((t.x >> 16) & 0xffu), acc[2]);
    acc[3] = fmaf(w, (float)(t.x >> 24), acc[3]);
    acc[4] = fmaf(w, (float)(t.y & 0xffu), acc[4]);
    acc[5] = fmaf(w, (float)((t.y >> 8) & 0xffu), acc[5]);
    acc[6] = fmaf(w, (float)((t.y >> 16) & 0xffu), acc[6]);
    acc[7] = fmaf(w, (float)(t.y >> 24), acc[7]);
}

__device__ __forceinline__ float sigmoidf_(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

// Evaluate the field at lattice point Q and composite it (Eq. 1-2, 5-7).
template <int KF>
__device__ __forceinline__ void shade_sample(const DevScene& S, const int64_t Q[3], RayState& st) {
    uint2 tv[8];
    uint2 tp[3][4];
    float wv[8];
    float wp[3][4];
    bool have_v = false;
    int n_src = S.n_src;
    if (S.use_v) {
        int i0[3];
        float f[3];
#pragma unroll
        for (int a = 0; a < 3; a++) texel(Q[a], S.sV, S.L, i0[a], f[a]);
        int slot = ((i0[2] >> 3) * S.nb + (i0[1] >> 3)) * S.nb + (i0[0] >> 3);
        int blk = __ldg(S.block_index + slot);
        if (blk >= 0) {
            have_v = true;
            const uint8_t* base = S.atlas + (size_t)blk * (729 * 8);
            int lx = i0[0] & 7, ly = i0[1] & 7, lz = i0[2] & 7;
#pragma unroll
            for (int c = 0; c < 8; c++) {
                int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
                const uint2* p = reinterpret_cast<const uint2*>(
                    base + (((lz + dz) * 9 + (ly + dy)) * 9 + (lx + dx)) * 8);
                tv[c] = __ldg(p);
                wv[c] = (dx ? f[0] : 1.f - f[0]) * (dy ? f[1] : 1.f - f[1]) *
                        (dz ? f[2] : 1.f - f[2]);
            }
        } else {
            n_src -= 1;                    // a missing block contributes nothing
            if (KF & KF_COUNT) st.c_miss++;
        }
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (!S.use_p[a]) continue;
        const int ua = (a == 0) ? 1 : 0;
        const int va = (a == 2) ? 1 : 2;
        int iu, iv;
        float fu, fv;
        texel(Q[ua], S.sP, S.R, iu, fu);
        texel(Q[va], S.sP, S.R, iv, fv);
        const uint8_t* pl = S.planes + (size_t)a * S.R * S.R * 8;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            int du = c & 1, dv = c >> 1;
            tp[a][c] = __ldg(reinterpret_cast<const uint2*>(pl + ((size_t)(iv + dv) * S.R + (iu + du)) * 8));
            wp[a][c] = (du ? fu : 1.f - fu) * (dv ? fv : 1.f - fv);
        }
    }
    // density first
    float s0 = 0.f;
    if (have_v) {
#pragma unroll
        for (int c = 0; c < 8; c++) s0 = fmaf(wv[c], (float)(tv[c].x & 0xffu), s0);
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (!S.use_p[a]) continue;
#pragma unroll
        for (int c = 0; c < 4; c++) s0 = fmaf(wp[a][c], (float)(tp[a][c].x & 0xffu), s0);
    }
    float t0 = fmaf(s0, S.kd, -(float)n_src * S.md);
    float tau = __expf(t0);
    float alpha = 1.f - __expf(-tau * S.step_f);
    if (alpha > S.alpha_skip) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (have_v) {
#pragma unroll
            for (int c = 0; c < 8; c++) acc_texel(acc, tv[c], wv[c]);
        }
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (!S.use_p[a]) continue;
#pragma unroll
            for (int c = 0; c < 4; c++) acc_texel(acc, tp[a][c], wp[a][c]);
        }
        float off = -(float)n_src * S.ma;
        float w = alpha * st.T;
#pragma unroll
        for (int c = 0; c < 3; c++) st.cd[c] = fmaf(w, sigmoidf_(fmaf(acc[1 + c], S.ka, off)), st.cd[c]);
#pragma unroll
        for (int c = 0; c < 4; c++) st.F[c] = fmaf(w, sigmoidf_(fmaf(acc[4 + c], S.ka, off)), st.F[c]);
    } else if (KF & KF_COUNT) {
        st.c_donly++;
    }
    st.T *= (1.f - alpha);
}

// March one contracted segment.
template <int KF>
__device__ __forceinline__ void march_segment(const DevScene& S, const Segment& sg, int ordinal,
                                              RayState& st, uint32_t rflags, const TraceArgs& ta,
                                              int64_t ray) {
    const int nl = S.n_levels;
    const int Nf = S.level_res[nl - 1];
    const int sf = S.level_shift[nl - 1];
    int k = 0;
    while (k < sg.K) {
        int64_t Q[3];
#pragma unroll
        for (int a = 0; a < 3; a++) Q[a] = sg.Qa[a] + (int64_t)k * sg.U[a];
        int fx = occ_cell(Q[0], sf, Nf), fy = occ_cell(Q[1], sf, Nf), fz = occ_cell(Q[2], sf, Nf);
        int fcell = (fz * Nf + fy) * Nf + fx;
        if (KF & KF_DENSE) {
            if (!occ_bit(S.occ[nl - 1], fx, fy, fz, Nf)) { k++; continue; }
        } else if (fcell != st.last_cell) {
            bool empty = false;
            for (int lev = 0; lev < nl; lev++) {
                const int N = S.level_res[lev];
                const int sh = S.level_shift[lev];
                int cx = occ_cell(Q[0], sh, N), cy = occ_cell(Q[1], sh, N), cz = occ_cell(Q[2], sh, N);
                if (!occ_bit(S.occ[lev], cx, cy, cz, N)) {
                    // jump to the first lattice sample outside this empty cell (ray-AABB exit)
                    int64_t e = INT64_MAX;
                    const int cc[3] = {cx, cy, cz};
#pragma unroll
                    for (int a = 0; a < 3; a++) {
                        if (sg.U[a] == 0) continue;
                        int64_t lo = ((int64_t)cc[a] << sh) - kTwo;
                        int64_t hi = ((int64_t)(cc[a] + 1) << sh) - kTwo;
                        int64_t ea = exit_axis(sg.Qa[a], sg.U[a], lo, hi);
                        e = ea < e ? ea : e;
                    }
                    int64_t kn = (int64_t)k + 1;
                    if (e > kn) kn = e;
                    if (kn > sg.K) kn = sg.K;
                    k = (int)kn;
                    if (KF & KF_COUNT) st.c_skip++;
                    empty = true;
                    break;
                }
            }
            if (empty) continue;
        }
        st.last_cell = fcell;
        shade_sample<KF>(S, Q, st);
        if (KF & KF_COUNT) st.c_eval++;
        if (KF & KF_TRACE) {
            if (st.n_eval < ta.max_per_ray) {
                int64_t idx = ray * ta.max_per_ray + st.n_eval;
                ta.cells[idx] = ((uint64_t)ordinal << 61) | ((uint64_t)k << 40) | (uint64_t)fcell;
                if (ta.T) ta.T[idx] = st.T;
            }
        }
        st.n_eval++;
        if (!(rflags & MERF_NO_EARLY_TERM) && st.T < S.t_min) { st.done = true; return; }
        k++;
    }
}

// Deferred MLP (Eq. 3; 3 layers x 16 hidden, 4 frequencies).
__device__ __forceinline__ void deferred_mlp(const float* __restrict__ w, const RayState& st,
                                             const double d[3], float out[3]) {
    float x[34];
    x[0] = st.cd[0]; x[1] = st.cd[1]; x[2] = st.cd[2];
    x[3] = st.F[0]; x[4] = st.F[1]; x[5] = st.F[2]; x[6] = st.F[3];
    int n = 7;
#pragma unroll
    for (int j = 0; j < 3; j++) x[n++] = (float)d[j];
#pragma unroll
    for (int j = 0; j < 3; j++) {
        float dj = (float)d[j];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            float s, c;
            sincosf(dj * (float)(1 << k), &s, &c);
            x[n++] = s;
            x[n++] = c;
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
        out[o] = __fdividef(1.0f, 1.0f + expf(-s));
    }
}

__device__ __forceinline__ void record_segment(const TraceArgs& ta, int64_t ray, int ordinal,
                                               const Segment& sg, double t_a, double t_b) {
    if (ordinal >= ta.max_per_ray) return;
    merf_segment r;
    r.t_a = t_a;
    r.t_b = t_b;
#pragma unroll
    for (int q = 0; q < 3; q++) { r.Qa[q] = sg.Qa[q]; r.U[q] = sg.U[q]; }
    r.K = sg.K;
    r.region = sg.region;
    ta.segs[ray * ta.max_per_ray + ordinal] = r;
}

__device__ __forceinline__ void add_stat(unsigned long long* stats, int idx, int v) {
    unsigned int s = __reduce_add_sync(0xffffffffu, (unsigned)v);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(stats + idx, (unsigned long long)s);
}

template <int KF>
__global__ void __launch_bounds__(128) render_kernel(DevScene S, CamBatch cb, int W, int H,
                                                     void* out, uint32_t rflags, RayArgs ra,
                                                     TraceArgs ta, unsigned long long* stats) {
    __shared__ float s_mlp[kMlpFloats];
    for (int i = threadIdx.x; i < kMlpFloats; i += blockDim.x) s_mlp[i] = S.mlp[i];
    __syncthreads();

    bool valid;
    int64_t ray;
    double o[3], d[3], t_near;
    int cam_i = 0, px = 0, py = 0;
    if (KF & (KF_RAYS | KF_TRACE | KF_SEGS)) {
        ray = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        valid = ray < ra.n;
        if (valid) {
            if (KF & (KF_TRACE | KF_SEGS)) {
                int64_t pid = ra.pixel_ids[ray];
                px = (int)(pid % W);
                py = (int)(pid / W);
                raygen(cb.cam[0], px, py, o, d);
                t_near = cb.cam[0].t_near;
            } else {
#pragma unroll
                for (int q = 0; q < 3; q++) { o[q] = ra.o[3 * ray + q]; d[q] = ra.d[3 * ray + q]; }
                t_near = ra.t_near ? ra.t_near[ray] : 0.0;
            }
        }
    } else {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        px = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
        py = blockIdx.y * 8 + (warp >> 1) * 4 + (lane >> 3);
        cam_i = blockIdx.z;
        valid = px < W && py < H;
        ray = ((int64_t)cam_i * H + py) * W + px;
        if (valid) {
            raygen(cb.cam[cam_i], px, py, o, d);
            t_near = cb.cam[cam_i].t_near;
        }
    }

    RayState st;
    st.T = 1.f;
#pragma unroll
    for (int c = 0; c < 3; c++) st.cd[c] = 0.f;
#pragma unroll
    for (int c = 0; c < 4; c++) st.F[c] = 0.f;
    st.done = false;
    st.last_cell = -1;
    st.n_eval = 0;
    st.c_eval = st.c_donly = st.c_skip = st.c_miss = 0;
    int c_seg = 0;
    unsigned reg_mask = 0;   // regions are convex, so a ray visits each at most once

    if (valid) {
        double cand[12];
        boundary_candidates(o, d, t_near, cand);
        // Walk the sorted boundaries; merge equal-region intervals into segments.  The
        // candidates are consumed as a register shift queue (constant indices only): no
        // dynamically indexed local array anywhere in the kernel.
        double b = t_near, seg_start = t_near;
        int g_cur = -1, ordinal = 0;
        const bool keep_counting = (KF & KF_COUNT) != 0;
        for (int it = 0; it < 13; it++) {
            for (int pop = 0; pop < 12 && cand[0] <= b; pop++) {
#pragma unroll
                for (int q = 0; q < 11; q++) cand[q] = cand[q + 1];
                cand[11] = __longlong_as_double(0x7ff0000000000000ll);
            }
            const double nb = cand[0];
            const bool last = isinf(nb);
            double p = last ? add_rn(mul_rn(b, 2.0), 1.0) : mul_rn(add_rn(b, nb), 0.5);
            double x[3];
            point_at(o, d, p, x);
            int g = region_of(x[0], x[1], x[2]);
            if (g_cur < 0) {
                g_cur = g;
                seg_start = b;
            } else if (g != g_cur) {
                Segment sg;
                if (make_segment(S, g_cur, o, d, seg_start, b, sg)) {
                    if (KF & KF_SEGS) record_segment(ta, ray, ordinal, sg, seg_start, b);
                    else if (!st.done) march_segment<KF>(S, sg, ordinal, st, rflags, ta, ray);
                    ordinal++;
                    c_seg++;
                    reg_mask |= 1u << g_cur;
                }
                g_cur = g;
                seg_start = b;
                if (st.done && !keep_counting) break;
            }
            if (last) {
                Segment sg;
                if (make_segment(S, g_cur, o, d, seg_start, nb, sg)) {
                    if (KF & KF_SEGS) record_segment(ta, ray, ordinal, sg, seg_start, nb);
                    else if (!st.done) march_segment<KF>(S, sg, ordinal, st, rflags, ta, ray);
                    ordinal++;
                    c_seg++;
                    reg_mask |= 1u << g_cur;
                }
                break;
            }
            b = nb;
        }
        float rgb[3];
        deferred_mlp(s_mlp, st, d, rgb);
#pragma unroll
        for (int c = 0; c < 3; c++) rgb[c] = __saturatef(st.cd[c] + rgb[c]);
        if (KF & KF_SEGS) {
            ta.counts[ray] = ordinal;
        } else if (KF & KF_TRACE) {
            ta.counts[ray] = st.n_eval;
        } else if (KF & KF_U8) {
            uchar4 v = make_uchar4((unsigned char)__float2int_rn(rgb[0] * 255.f),
                                   (unsigned char)__float2int_rn(rgb[1] * 255.f),
                                   (unsigned char)__float2int_rn(rgb[2] * 255.f), 255);
            reinterpret_cast<uchar4*>(out)[ray] = v;
        } else {
            float* o3 = reinterpret_cast<float*>(out) + 3 * ray;
            o3[0] = rgb[0];
            o3[1] = rgb[1];
            o3[2] = rgb[2];
        }
    }
    if (KF & KF_COUNT) {
        add_stat(stats, 0, valid ? 1 : 0);
        add_stat(stats, 1, c_seg);
        add_stat(stats, 2, st.c_eval);
        add_stat(stats, 3, st.c_donly);
        add_stat(stats, 4, st.c_skip);
        add_stat(stats, 5, st.c_miss);
#pragma unroll
        for (int g = 0; g < 7; g++) add_stat(stats, 6 + g, (reg_mask >> g) & 1u);
    }
}

}  // namespace merf
