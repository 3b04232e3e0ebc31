// merf_render_kernel.cuh -- the hot path: one fused kernel per batch of views (sm_100a).
//
// Per ray (Sec. 6), in two phases inside one kernel:
//  A. setup (fp64, canonical order, reading D8): raygen -> region segmentation of the world
//     ray into <= 7 contracted segments -> per segment the int32 lattice origin
//     Qa, step U and sample count K, written to shared memory.  No fp64 state survives A.
//  B. march (int32 lattice + fp32 shading): Q_k = Qa + k U; coarse-to-fine occupancy probes;
//     an empty cell jumps to the first lattice sample outside it (the ray-AABB exit);
//     an evaluated sample reads the DENSITY first -- one 8-byte octet of the block-sparse
//     grid (through the indirection table) + one 4-byte quad per plane, i.e. 4 loads for the
//     8 trilinear + 12 bilinear corners (Eq. 5) -- computes alpha = 1 - exp(-tau Delta) and
//     reads the appearance texels only if alpha > alpha_skip; composite (Eq. 1-2)
//     with termination at T < 2e-4.
//  C. deferred MLP h(C_d, F, d) per pixel (Eq. 3) and the store.
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

constexpr int kThreads = 128;

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
    int last_cell;          // finest cell of the last evaluated sample (all levels known set)
    int n_eval;             // evaluated samples (trace index)
    int c_eval, c_donly, c_skip, c_miss;
};

__device__ __forceinline__ float sigmoidf_(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

// accumulate channels 1..7 of an 8-byte AoS texel with weight w
__device__ __forceinline__ void acc_appearance(float acc[7], uint2 t, float w) {
    acc[0] = fmaf(w, byte_f(t.x, 1), acc[0]);
    acc[1] = fmaf(w, byte_f(t.x, 2), acc[1]);
    acc[2] = fmaf(w, byte_f(t.x, 3), acc[2]);
    acc[3] = fmaf(w, byte_f(t.y, 0), acc[3]);
    acc[4] = fmaf(w, byte_f(t.y, 1), acc[4]);
    acc[5] = fmaf(w, byte_f(t.y, 2), acc[5]);
    acc[6] = fmaf(w, byte_f(t.y, 3), acc[6]);
}

// Evaluate the field at lattice point (Qx, Qy, Qz) and composite it (Eq. 1-2, 5-7).
template <int KF>
__device__ __forceinline__ void shade_sample(const DevScene& S, int Qx, int Qy, int Qz, RayState& st) {
    const int Q[3] = {Qx, Qy, Qz};
    // ---- density pass: 1 octet (V) + 3 quads (planes)
    int n_src = S.n_src;
    float s0 = 0.f;
    int vi[3] = {0, 0, 0};
    float vf[3] = {0.f, 0.f, 0.f};
    int blk = -1;
    if (S.use_v) {
#pragma unroll
        for (int a = 0; a < 3; a++) texel(Q[a], S.sV, S.L, vi[a], vf[a]);
        const int slot = ((vi[2] >> 3) * S.nb + (vi[1] >> 3)) * S.nb + (vi[0] >> 3);
        blk = __ldg(S.block_index + slot);
        if (blk >= 0) {
            const uint2 oct = __ldg(S.vdens + ((size_t)blk * 512 + ((vi[2] & 7) * 8 + (vi[1] & 7)) * 8 + (vi[0] & 7)));
            const float gx = 1.f - vf[0], gy = 1.f - vf[1], gz = 1.f - vf[2];
            const float w00 = gy * gz, w10 = vf[1] * gz, w01 = gy * vf[2], w11 = vf[1] * vf[2];
            s0 = fmaf(gx * w00, byte_f(oct.x, 0), s0);
            s0 = fmaf(vf[0] * w00, byte_f(oct.x, 1), s0);
            s0 = fmaf(gx * w10, byte_f(oct.x, 2), s0);
            s0 = fmaf(vf[0] * w10, byte_f(oct.x, 3), s0);
            s0 = fmaf(gx * w01, byte_f(oct.y, 0), s0);
            s0 = fmaf(vf[0] * w01, byte_f(oct.y, 1), s0);
            s0 = fmaf(gx * w11, byte_f(oct.y, 2), s0);
            s0 = fmaf(vf[0] * w11, byte_f(oct.y, 3), s0);
        } else {
            n_src -= 1;                    // a missing block contributes nothing
            if (KF & KF_COUNT) st.c_miss++;
        }
    }
    int pu[3], pv[3];
    float fu[3], fv[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (!S.use_p[a]) continue;
        const int ua = (a == 0) ? 1 : 0;
        const int va = (a == 2) ? 1 : 2;
        texel(Q[ua], S.sP, S.R, pu[a], fu[a]);
        texel(Q[va], S.sP, S.R, pv[a], fv[a]);
        const uint32_t quad = __ldg(S.pdens + ((size_t)a * S.R + pv[a]) * S.R + pu[a]);
        const float gu = 1.f - fu[a], gv = 1.f - fv[a];
        s0 = fmaf(gu * gv, byte_f(quad, 0), s0);
        s0 = fmaf(fu[a] * gv, byte_f(quad, 1), s0);
        s0 = fmaf(gu * fv[a], byte_f(quad, 2), s0);
        s0 = fmaf(fu[a] * fv[a], byte_f(quad, 3), s0);
    }
    const float t0 = fmaf(s0, S.kd, -(float)n_src * S.md);
    const float tau = __expf(t0);
    const float alpha = 1.f - __expf(-tau * S.step_f);
    if (alpha > S.alpha_skip) {
        // ---- appearance pass: 20 AoS texels, channels 1..7
        float acc[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (blk >= 0) {
            const uint8_t* base = S.atlas + (size_t)blk * (729 * 8);
            const int lx = vi[0] & 7, ly = vi[1] & 7, lz = vi[2] & 7;
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
                const uint2 t = __ldg(reinterpret_cast<const uint2*>(
                    base + (((lz + dz) * 9 + (ly + dy)) * 9 + (lx + dx)) * 8));
                const float w = (dx ? vf[0] : 1.f - vf[0]) * (dy ? vf[1] : 1.f - vf[1]) *
                                (dz ? vf[2] : 1.f - vf[2]);
                acc_appearance(acc, t, w);
            }
        }
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (!S.use_p[a]) continue;
            const uint2* pl = reinterpret_cast<const uint2*>(S.planes) + (size_t)a * S.R * S.R;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int du = c & 1, dv = c >> 1;
                const uint2 t = __ldg(pl + (size_t)(pv[a] + dv) * S.R + (pu[a] + du));
                const float w = (du ? fu[a] : 1.f - fu[a]) * (dv ? fv[a] : 1.f - fv[a]);
                acc_appearance(acc, t, w);
            }
        }
        const float off = -(float)n_src * S.ma;
        const float w = alpha * st.T;
#pragma unroll
        for (int c = 0; c < 3; c++) st.cd[c] = fmaf(w, sigmoidf_(fmaf(acc[c], S.ka, off)), st.cd[c]);
#pragma unroll
        for (int c = 0; c < 4; c++) st.F[c] = fmaf(w, sigmoidf_(fmaf(acc[3 + c], S.ka, off)), st.F[c]);
    } else if (KF & KF_COUNT) {
        st.c_donly++;
    }
    st.T *= (1.f - alpha);
}

// March one contracted segment.  Returns true when the ray terminated.
template <int KF>
__device__ __forceinline__ bool march_segment(const DevScene& S, int4 qa, int4 uu, int ordinal,
                                              RayState& st, uint32_t rflags, const TraceArgs& ta,
                                              int64_t ray) {
    const int nl = S.n_levels;
    const int Nf = S.level_res[nl - 1];
    const int sf = S.level_shift[nl - 1];
    const uint32_t* occ_f = S.occ[nl - 1];
    const int K = qa.w;
    int k = 0;
    while (k < K) {
        const int Qx = qa.x + k * uu.x, Qy = qa.y + k * uu.y, Qz = qa.z + k * uu.z;
        const int fx = occ_cell(Qx, sf, Nf), fy = occ_cell(Qy, sf, Nf), fz = occ_cell(Qz, sf, Nf);
        const int fcell = (fz * Nf + fy) * Nf + fx;
        if (KF & KF_DENSE) {
            if (!occ_bit(occ_f, fx, fy, fz, Nf)) { k++; continue; }
        } else if (fcell != st.last_cell) {
            int e = -1;
#pragma unroll
            for (int lev = 0; lev < MERF_MAX_LEVELS; lev++) {
                if (lev < nl && e < 0) {
                    const int N = S.level_res[lev];
                    const int sh = S.level_shift[lev];
                    const int cx = occ_cell(Qx, sh, N), cy = occ_cell(Qy, sh, N), cz = occ_cell(Qz, sh, N);
                    if (!occ_bit(S.occ[lev], cx, cy, cz, N)) {
                        // jump to the first lattice sample outside this empty cell (ray-AABB exit)
                        e = K;
                        if (uu.x != 0) e = min(e, exit_axis(qa.x, uu.x, (cx << sh) - kTwoI, ((cx + 1) << sh) - kTwoI, K));
                        if (uu.y != 0) e = min(e, exit_axis(qa.y, uu.y, (cy << sh) - kTwoI, ((cy + 1) << sh) - kTwoI, K));
                        if (uu.z != 0) e = min(e, exit_axis(qa.z, uu.z, (cz << sh) - kTwoI, ((cz + 1) << sh) - kTwoI, K));
                    }
                }
            }
            if (e >= 0) {
                k = min(max(k + 1, e), K);
                if (KF & KF_COUNT) st.c_skip++;
                continue;
            }
        }
        st.last_cell = fcell;
        shade_sample<KF>(S, Qx, Qy, Qz, st);
        if (KF & KF_COUNT) st.c_eval++;
        if (KF & KF_TRACE) {
            if (st.n_eval < ta.max_per_ray) {
                const int64_t idx = ray * ta.max_per_ray + st.n_eval;
                ta.cells[idx] = ((uint64_t)ordinal << 61) | ((uint64_t)k << 40) | (uint64_t)fcell;
                if (ta.T) ta.T[idx] = st.T;
            }
        }
        st.n_eval++;
        if (!(rflags & MERF_NO_EARLY_TERM) && st.T < S.t_min) return true;
        k++;
    }
    return false;
}

// Deferred MLP (Eq. 3; 3 layers x 16 hidden, 4 frequencies).
__device__ __forceinline__ void deferred_mlp(const float* __restrict__ w, const RayState& st,
                                             const float d[3], float out[3]) {
    float x[34];
    x[0] = st.cd[0]; x[1] = st.cd[1]; x[2] = st.cd[2];
    x[3] = st.F[0]; x[4] = st.F[1]; x[5] = st.F[2]; x[6] = st.F[3];
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
        out[o] = __fdividef(1.0f, 1.0f + expf(-s));
    }
}

__device__ __forceinline__ void add_stat(unsigned long long* stats, int idx, int v) {
    unsigned int s = __reduce_add_sync(0xffffffffu, (unsigned)v);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(stats + idx, (unsigned long long)s);
}

template <int KF>
__global__ void __launch_bounds__(kThreads, 4) render_kernel(DevScene S, CamBatch cb, int W, int H,
                                                             void* out, uint32_t rflags, RayArgs ra,
                                                             TraceArgs ta, unsigned long long* stats) {
    __shared__ float s_mlp[kMlpFloats];
    __shared__ int4 s_qa[kMaxSeg][kThreads];    // Qa.xyz, K
    __shared__ int4 s_u[kMaxSeg][kThreads];     // U.xyz, region
    for (int i = threadIdx.x; i < kMlpFloats; i += blockDim.x) s_mlp[i] = S.mlp[i];
    __syncthreads();
    const int tid = threadIdx.x;

    bool valid;
    int64_t ray;
    int cam_i = 0, px = 0, py = 0;
    if (KF & (KF_RAYS | KF_TRACE | KF_SEGS)) {
        ray = (int64_t)blockIdx.x * blockDim.x + tid;
        valid = ray < ra.n;
    } else {
        const int warp = tid >> 5, lane = tid & 31;
        px = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
        py = blockIdx.y * 8 + (warp >> 1) * 4 + (lane >> 3);
        cam_i = blockIdx.z;
        valid = px < W && py < H;
        ray = ((int64_t)cam_i * H + py) * W + px;
    }

    // ---------------- phase A: fp64 setup -> segments in shared memory ----------------
    int nseg = 0;
    unsigned reg_mask = 0;       // regions are convex, so a ray visits each at most once
    float df[3] = {0.f, 0.f, 1.f};
    if (valid) {
        double o[3], d[3], t_near;
        if (KF & (KF_TRACE | KF_SEGS)) {
            const int64_t pid = ra.pixel_ids[ray];
            px = (int)(pid % W);
            py = (int)(pid / W);
            raygen(cb.cam[0], px, py, o, d);
            t_near = cb.cam[0].t_near;
        } else if (KF & KF_RAYS) {
#pragma unroll
            for (int q = 0; q < 3; q++) { o[q] = ra.o[3 * ray + q]; d[q] = ra.d[3 * ray + q]; }
            t_near = ra.t_near ? ra.t_near[ray] : 0.0;
        } else {
            raygen(cb.cam[cam_i], px, py, o, d);
            t_near = cb.cam[cam_i].t_near;
        }
        df[0] = (float)d[0];
        df[1] = (float)d[1];
        df[2] = (float)d[2];
        double cand[12];
        boundary_candidates(o, d, t_near, cand);
        // Walk the sorted boundaries; merge equal-region intervals into segments.  The
        // candidates are consumed as a register shift queue (constant indices only).
        auto emit = [&](int g, double t_a, double t_b) {
            Segment sg;
            if (!make_segment(S, g, o, d, t_a, t_b, sg)) return;   // zero length: dropped
            if (KF & KF_SEGS) {
                if (nseg < ta.max_per_ray) {
                    merf_segment r;
                    r.t_a = t_a;
                    r.t_b = t_b;
#pragma unroll
                    for (int q = 0; q < 3; q++) { r.Qa[q] = sg.Qa[q]; r.U[q] = sg.U[q]; }
                    r.K = sg.K;
                    r.region = sg.region;
                    ta.segs[ray * ta.max_per_ray + nseg] = r;
                }
            } else if (nseg < kMaxSeg) {
                s_qa[nseg][tid] = make_int4(sg.Qa[0], sg.Qa[1], sg.Qa[2], sg.K);
                s_u[nseg][tid] = make_int4(sg.U[0], sg.U[1], sg.U[2], sg.region);
            }
            nseg++;
            reg_mask |= 1u << g;
        };
        double b = t_near, seg_start = t_near;
        int g_cur = -1;
        for (int it = 0; it < 13; it++) {
            for (int pop = 0; pop < 12 && cand[0] <= b; pop++) {
#pragma unroll
                for (int q = 0; q < 11; q++) cand[q] = cand[q + 1];
                cand[11] = __longlong_as_double(0x7ff0000000000000ll);
            }
            const double nb = cand[0];
            const bool last = isinf(nb);
            const double p = last ? add_rn(mul_rn(b, 2.0), 1.0) : mul_rn(add_rn(b, nb), 0.5);
            double x[3];
            point_at(o, d, p, x);
            const int g = region_of(x[0], x[1], x[2]);
            if (g_cur < 0) {
                g_cur = g;
                seg_start = b;
            } else if (g != g_cur) {
                emit(g_cur, seg_start, b);
                g_cur = g;
                seg_start = b;
            }
            if (last) {
                emit(g_cur, seg_start, nb);
                break;
            }
            b = nb;
        }
    }

    // ---------------- phase B: march (int32 lattice, fp32 shading) ----------------
    RayState st;
    st.T = 1.f;
#pragma unroll
    for (int c = 0; c < 3; c++) st.cd[c] = 0.f;
#pragma unroll
    for (int c = 0; c < 4; c++) st.F[c] = 0.f;
    st.last_cell = -1;
    st.n_eval = 0;
    st.c_eval = st.c_donly = st.c_skip = st.c_miss = 0;
    if (valid && !(KF & KF_SEGS)) {
        const int ns = min(nseg, kMaxSeg);
        for (int j = 0; j < ns; j++) {
            if (march_segment<KF>(S, s_qa[j][tid], s_u[j][tid], j, st, rflags, ta, ray)) break;
        }
        // ---------------- phase C: deferred MLP + store ----------------
        float rgb[3];
        deferred_mlp(s_mlp, st, df, rgb);
#pragma unroll
        for (int c = 0; c < 3; c++) rgb[c] = __saturatef(st.cd[c] + rgb[c]);
        if (KF & KF_TRACE) {
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
    if ((KF & KF_SEGS) && valid) ta.counts[ray] = nseg;
    if (KF & KF_COUNT) {
        add_stat(stats, 0, valid ? 1 : 0);
        add_stat(stats, 1, nseg);
        add_stat(stats, 2, st.c_eval);
        add_stat(stats, 3, st.c_donly);
        add_stat(stats, 4, st.c_skip);
        add_stat(stats, 5, st.c_miss);
#pragma unroll
        for (int g = 0; g < 7; g++) add_stat(stats, 6 + g, (reg_mask >> g) & 1u);
    }
}

}  // namespace merf
