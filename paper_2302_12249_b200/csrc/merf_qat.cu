// merf_qat.cu -- NEXT-3: quantisation-aware differentiable forward/backward of the render path
// on toy dense grids (Sec. 5.2, Eq. 7-8).
//
//  1. prequant_kernel: stored value v = 2m q(sigma(theta)) - m per grid element (Eq. 7), with
//     q(x) = floor(255 x + 1/2)/255 (Eq. 8) evaluated in fp64 so byte decisions are exact.
//  2. qat_ray_kernel (one thread per ray; lattice from the render setup kernel, every sample
//     in an occupied finest cell, no early termination): forward gather (Eq. 5), decode
//     (Eq. 6), composite (Eq. 1-2) storing per-sample records; deferred MLP (Eq. 3) forward
//     and backward; loss sum (C - C*)^2; then the reverse compositing pass
//        dL/dalpha_i = T_i (G . x_i - G . R_i),  R_i = sum_{j>i} alpha_j prod_{i<k<j}(1-alpha_k) x_j
//     (division-free), chained to dL/dt and scattered to the grid corners with atomics.
//  3. ste_kernel: dL/dtheta = dL/dv * 2m sigma'(theta) -- the straight-through estimator
//     treats q as the identity in the backward pass (Eq. 8).
#include <cstdint>
#include <cuda_runtime.h>

#include "merf_render_kernel.cuh"
#include "merf_kernels.h"

namespace merf {

struct QatArgs {
    const float* vv;        // [L^3][8] stored (quantised) values of V
    const float* vp;        // [3][R^2][8] stored values of the planes
    const float* target;    // [H*W][3]
    float* rgb;             // [H*W][3]
    float* gv;              // [L^3][8] dL/dv (accumulated)
    float* gp;              // [3][R^2][8]
    float* samp;            // [n][smax][12]
    const float* mlp;       // [883]
    double* loss;
    unsigned int* overflow;
    unsigned long long* n_samples;   // total evaluated samples (optional)
    int L, R, smax, Nf, sf;
    const uint32_t* occf;
    float step;
};

__device__ __forceinline__ void coord_qat(int Q, int M, int& i0, float& f) {
    // lower texel index in [0, M-2] and fraction (cell-centred, clamp to edge; reading D9)
    const int s = kF + 2 - (31 - __clz(M));
    const int P = Q - (1 << (s - 1));          // Q biased (workspace segments, see occ_cell)
    int i = P >> s;
    float fr = (float)(P & ((1 << s) - 1)) * __int_as_float((127 - s) << 23);
    if (i < 0) { i = 0; fr = 0.f; }
    if (i > M - 2) { i = M - 2; fr = 1.f; }
    i0 = i;
    f = fr;
}

__global__ void prequant_kernel(const float* __restrict__ theta, int64_t n, int quant, float md, float ma,
                                float* __restrict__ v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double m = (i % 8 == 0) ? (double)md : (double)ma;
    const double s = 1.0 / (1.0 + exp(-(double)theta[i]));
    const double q = quant ? floor(255.0 * s + 0.5) / 255.0 : s;
    v[i] = (float)(2.0 * m * q - m);
}

__global__ void ste_kernel(const float* __restrict__ theta, const float* __restrict__ gvals, int64_t n,
                           float md, float ma, float* __restrict__ gtheta) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float m = (i % 8 == 0) ? md : ma;
    const float s = 1.f / (1.f + expf(-theta[i]));
    gtheta[i] = gvals[i] * 2.f * m * s * (1.f - s);
}

// per-ray scratch row (16 floats): [0..6] C_d, F accumulated; [7] sample count (int bits);
// [8] overflow flag; [9..15] G = dL/d(C_d, F)
constexpr int kRayRow = 16;

// 2a. forward: composite every occupied lattice sample, storing the per-sample records
__global__ void __launch_bounds__(128) qat_fwd_kernel(RaySource rs, Workspace ws, QatArgs A, float* rayb) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rs.n) return;
    int view, px, py;
    if (!ray_pixel(rs, r, view, px, py)) return;
    float* rec0 = A.samp + (size_t)r * A.smax * 12;
    float acc[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float T = 1.f;
    int n = 0;
    bool over = false;
    float vc[8][8];                    // the current V cell's corner values
    int cur_e0 = -1;
    float pc[3][4][8];                 // the current plane cells' corner values
    int cur_p[3] = {-1, -1, -1};
    const int ns = ws.nseg[r];
    for (int j = 0; j < ns; j++) {
        const int4 qa = ws.seg[(r * ws.seg_slots + j) * 2], uu = ws.seg[(r * ws.seg_slots + j) * 2 + 1];
        const int K = qa.w;
        for (int k = 0; k < K; k++) {
            const int Qx = qa.x + k * uu.x, Qy = qa.y + k * uu.y, Qz = qa.z + k * uu.z;
            const int cx = occ_cell(Qx, A.sf, A.Nf), cy = occ_cell(Qy, A.sf, A.Nf), cz = occ_cell(Qz, A.sf, A.Nf);
            if (!occ_bit(A.occf, cx, cy, cz, A.Nf)) {
                // empty finest cell: jump to the first lattice sample outside it (the render
                // march's lattice-snapped exit) -- the same evaluated-sample set as
                // testing every step; only when the sample lies inside the (unclamped) cell
                const int w = 1 << A.sf, lx = cx << A.sf, ly = cy << A.sf, lz = cz << A.sf;
                if (Qx >= lx && Qx < lx + w && Qy >= ly && Qy < ly + w && Qz >= lz && Qz < lz + w) {
                    int e = min(K, exit_axis(qa.x, uu.x, lx, lx + w, K));
                    e = min(e, exit_axis(qa.y, uu.y, ly, ly + w, K));
                    e = min(e, exit_axis(qa.z, uu.z, lz, lz + w, K));
                    k = max(k, e - 1);                     // the loop's k++ lands on e
                }
                continue;
            }
            float t[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            // V and each plane: the corners' values are kept in registers for the run of
            // samples that share that source's cell (8 lattice steps per voxel at L = 128, ~2
            // per plane texel), reloaded when it changes (247 registers, no spills)
            {
                int vi[3];
                float vf[3];
                coord_qat(Qx, A.L, vi[0], vf[0]);
                coord_qat(Qy, A.L, vi[1], vf[1]);
                coord_qat(Qz, A.L, vi[2], vf[2]);
                const int e0 = (vi[2] * A.L + vi[1]) * A.L + vi[0];
                if (e0 != cur_e0) {
                    cur_e0 = e0;
#pragma unroll
                    for (int c = 0; c < 8; c++) {
                        const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
                        const float4* src = reinterpret_cast<const float4*>(A.vv + (size_t)(e0 + (dz * A.L + dy) * A.L + dx) * 8);
                        const float4 a = __ldg(src), b = __ldg(src + 1);
                        vc[c][0] = a.x; vc[c][1] = a.y; vc[c][2] = a.z; vc[c][3] = a.w;
                        vc[c][4] = b.x; vc[c][5] = b.y; vc[c][6] = b.z; vc[c][7] = b.w;
                    }
                }
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
                    const float w = (dx ? vf[0] : 1.f - vf[0]) * (dy ? vf[1] : 1.f - vf[1]) * (dz ? vf[2] : 1.f - vf[2]);
#pragma unroll
                    for (int q = 0; q < 8; q++) t[q] = fmaf(w, vc[c][q], t[q]);
                }
            }
            {
                int pi[3];
                float pf[3];
                coord_qat(Qx, A.R, pi[0], pf[0]);
                coord_qat(Qy, A.R, pi[1], pf[1]);
                coord_qat(Qz, A.R, pi[2], pf[2]);
#pragma unroll
                for (int a = 0; a < 3; a++) {
                    const int ua = (a == 0) ? 1 : 0, va = (a == 2) ? 1 : 2;
                    const int e = pi[va] * A.R + pi[ua];
                    if (e != cur_p[a]) {
                        cur_p[a] = e;
#pragma unroll
                        for (int c = 0; c < 4; c++) {
                            const int du = c & 1, dv = c >> 1;
                            const float4* src = reinterpret_cast<const float4*>(
                                A.vp + ((size_t)a * A.R * A.R + (pi[va] + dv) * A.R + (pi[ua] + du)) * 8);
                            const float4 a4 = __ldg(src), b4 = __ldg(src + 1);
                            pc[a][c][0] = a4.x; pc[a][c][1] = a4.y; pc[a][c][2] = a4.z; pc[a][c][3] = a4.w;
                            pc[a][c][4] = b4.x; pc[a][c][5] = b4.y; pc[a][c][6] = b4.z; pc[a][c][7] = b4.w;
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        const int du = c & 1, dv = c >> 1;
                        const float w = (du ? pf[ua] : 1.f - pf[ua]) * (dv ? pf[va] : 1.f - pf[va]);
#pragma unroll
                        for (int q = 0; q < 8; q++) t[q] = fmaf(w, pc[a][c][q], t[q]);
                    }
                }
            }
            const float tau = expf(t[0]);
            const float alpha = 1.f - expf(-tau * A.step);
            float xs[7];
#pragma unroll
            for (int c = 0; c < 7; c++) {
                xs[c] = 1.f / (1.f + expf(-t[1 + c]));
                acc[c] = fmaf(alpha * T, xs[c], acc[c]);
            }
            if (n < A.smax) {
                float4* rec = reinterpret_cast<float4*>(rec0 + (size_t)n * 12);
                rec[0] = make_float4(__int_as_float(Qx), __int_as_float(Qy), __int_as_float(Qz), t[0]);
                rec[1] = make_float4(T, xs[0], xs[1], xs[2]);
                rec[2] = make_float4(xs[3], xs[4], xs[5], xs[6]);
            } else {
                over = true;
            }
            T *= (1.f - alpha);
            n++;
        }
    }
    if (over) atomicAdd(A.overflow, 1u);
    if (A.n_samples) atomicAdd(A.n_samples, (unsigned long long)n);
    float* row = rayb + r * kRayRow;
#pragma unroll
    for (int c = 0; c < 7; c++) row[c] = acc[c];
    row[7] = __int_as_float(n);
    row[8] = over ? 1.f : 0.f;
}

// 2b. deferred MLP (Eq. 3) forward + backward per ray: colour, loss, G = dL/d(C_d, F)
__global__ void __launch_bounds__(128) qat_mlp_kernel(RaySource rs, QatArgs A, float* rayb) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rs.n) return;
    int view, px, py;
    if (!ray_pixel(rs, r, view, px, py)) return;
    const int64_t pix = ((int64_t)view * rs.H + py) * rs.W + px;
    float* row = rayb + r * kRayRow;
    double od[3], dd[3];
    raygen(rs.cb.cam[view], px, py, od, dd);
    float x[34];
#pragma unroll
    for (int c = 0; c < 7; c++) x[c] = row[c];
#pragma unroll
    for (int q = 0; q < 3; q++) x[7 + q] = (float)dd[q];
    int m = 10;
#pragma unroll
    for (int jj = 0; jj < 3; jj++)
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
            const float a = (float)dd[jj] * (float)(1 << kk);
            x[m++] = sinf(a);
            x[m++] = cosf(a);
        }
    const float* W0 = A.mlp;
    const float* b0 = A.mlp + 544;
    const float* W1 = A.mlp + 560;
    const float* b1 = A.mlp + 816;
    const float* W2 = A.mlp + 832;
    const float* b2 = A.mlp + 880;
    float h0[16], h1[16], h[3];
#pragma unroll
    for (int o = 0; o < 16; o++) {
        float s = __ldg(b0 + o);
#pragma unroll
        for (int i = 0; i < 34; i++) s = fmaf(__ldg(W0 + o * 34 + i), x[i], s);
        h0[o] = fmaxf(s, 0.f);
    }
#pragma unroll
    for (int o = 0; o < 16; o++) {
        float s = __ldg(b1 + o);
#pragma unroll
        for (int i = 0; i < 16; i++) s = fmaf(__ldg(W1 + o * 16 + i), h0[i], s);
        h1[o] = fmaxf(s, 0.f);
    }
#pragma unroll
    for (int o = 0; o < 3; o++) {
        float s = __ldg(b2 + o);
#pragma unroll
        for (int i = 0; i < 16; i++) s = fmaf(__ldg(W2 + o * 16 + i), h1[i], s);
        h[o] = 1.f / (1.f + expf(-s));
    }
    float dC[3];
    double lsum = 0.0;
#pragma unroll
    for (int c = 0; c < 3; c++) {
        const float raw = x[c] + h[c];
        const float C = fminf(fmaxf(raw, 0.f), 1.f);
        A.rgb[pix * 3 + c] = C;
        const float e = C - A.target[pix * 3 + c];
        lsum += (double)e * e;
        dC[c] = (raw > 0.f && raw < 1.f) ? 2.f * e : 0.f;
    }
    atomicAdd(A.loss, lsum);
    float dz2[3], dh1[16], dh0[16];
#pragma unroll
    for (int o = 0; o < 3; o++) dz2[o] = dC[o] * h[o] * (1.f - h[o]);
#pragma unroll
    for (int i = 0; i < 16; i++) {
        float s = 0.f;
#pragma unroll
        for (int o = 0; o < 3; o++) s = fmaf(__ldg(W2 + o * 16 + i), dz2[o], s);
        dh1[i] = h1[i] > 0.f ? s : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 16; i++) {
        float s = 0.f;
#pragma unroll
        for (int o = 0; o < 16; o++) s = fmaf(__ldg(W1 + o * 16 + i), dh1[o], s);
        dh0[i] = h0[i] > 0.f ? s : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 7; i++) {
        float s = (i < 3) ? dC[i] : 0.f;
#pragma unroll
        for (int o = 0; o < 16; o++) s = fmaf(__ldg(W0 + o * 34 + i), dh0[o], s);
        row[9 + i] = s;
    }
}

// 2c. reverse compositing pass + scatter of dL/dv to the grid corners
__global__ void __launch_bounds__(128) qat_bwd_kernel(RaySource rs, QatArgs A, const float* rayb) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rs.n) return;
    int view, px, py;
    if (!ray_pixel(rs, r, view, px, py)) return;
    const float* row = rayb + r * kRayRow;
    if (row[8] != 0.f) return;                     // overflowed: gradient dropped (documented)
    const int n = __float_as_int(row[7]);
    float G[7];
#pragma unroll
    for (int c = 0; c < 7; c++) G[c] = row[9 + c];
    const float* rec0 = A.samp + (size_t)r * A.smax * 12;
    float Rt[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    // Run merging: consecutive samples of a ray usually share their V cell (8 lattice steps per
    // voxel at L = 128) and each plane's texel cell (~2 steps at R = 4L, longer for the plane
    // facing the ray), so the corners' gradients are summed in registers while a cell stays the
    // same and reduced to memory once per run (2 red.v4 per corner per run instead of per
    // sample).  The reductions are the kernel's bound (L2 reduction units, conflicts between a
    // ray's consecutive samples), DESIGN.md NEXT-3.  (8 + 12 corners x 8 channels = 160 fp32
    // accumulators: 226 registers, no spills; fewer resident warps, far fewer reductions.)
    float vacc[8][8];
#pragma unroll
    for (int c = 0; c < 8; c++)
#pragma unroll
        for (int q = 0; q < 8; q++) vacc[c][q] = 0.f;
    int cur_e0 = -1;
    unsigned touched = 0u;
    auto flush_v = [&]() {
        if (cur_e0 < 0) return;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            if (touched & (1u << c)) {
                const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
                float4* dst = reinterpret_cast<float4*>(A.gv + (size_t)(cur_e0 + (dz * A.L + dy) * A.L + dx) * 8);
                atomicAdd(dst, make_float4(vacc[c][0], vacc[c][1], vacc[c][2], vacc[c][3]));
                atomicAdd(dst + 1, make_float4(vacc[c][4], vacc[c][5], vacc[c][6], vacc[c][7]));
            }
#pragma unroll
            for (int q = 0; q < 8; q++) vacc[c][q] = 0.f;
        }
        touched = 0u;
    };
    float pacc[3][4][8];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int c = 0; c < 4; c++)
#pragma unroll
            for (int q = 0; q < 8; q++) pacc[a][c][q] = 0.f;
    int cur_p[3] = {-1, -1, -1};
    unsigned ptouched = 0u;
    auto flush_p = [&](int a) {
        if (cur_p[a] < 0) return;
        const int pu = cur_p[a] % A.R, pv = cur_p[a] / A.R;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            if (ptouched & (1u << (4 * a + c))) {
                const int du = c & 1, dv = c >> 1;
                float4* dst = reinterpret_cast<float4*>(A.gp + ((size_t)a * A.R * A.R + (pv + dv) * A.R + (pu + du)) * 8);
                atomicAdd(dst, make_float4(pacc[a][c][0], pacc[a][c][1], pacc[a][c][2], pacc[a][c][3]));
                atomicAdd(dst + 1, make_float4(pacc[a][c][4], pacc[a][c][5], pacc[a][c][6], pacc[a][c][7]));
            }
#pragma unroll
            for (int q = 0; q < 8; q++) pacc[a][c][q] = 0.f;
        }
        ptouched &= ~(15u << (4 * a));
    };
    for (int i = n - 1; i >= 0; i--) {
        const float4* rec4 = reinterpret_cast<const float4*>(rec0 + (size_t)i * 12);
        const float4 r0 = rec4[0], r1 = rec4[1], r2 = rec4[2];
        const float xs[7] = {r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
        const float tau = expf(r0.w);
        const float alpha = 1.f - expf(-tau * A.step);
        const float Ti = r1.x;
        float gx = 0.f, gr = 0.f;
#pragma unroll
        for (int c = 0; c < 7; c++) {
            gx = fmaf(G[c], xs[c], gx);
            gr = fmaf(G[c], Rt[c], gr);
        }
        const float dalpha = Ti * (gx - gr);
#pragma unroll
        for (int c = 0; c < 7; c++) Rt[c] = fmaf(alpha, xs[c] - Rt[c], Rt[c]);   // a x + (1-a) R
        float dt[8];
        dt[0] = dalpha * A.step * (1.f - alpha) * tau;
        const float w = alpha * Ti;
#pragma unroll
        for (int c = 0; c < 7; c++) dt[1 + c] = w * G[c] * xs[c] * (1.f - xs[c]);
        const int Q[3] = {__float_as_int(r0.x), __float_as_int(r0.y), __float_as_int(r0.z)};
        {
            int vi[3];
            float vf[3];
#pragma unroll
            for (int a = 0; a < 3; a++) coord_qat(Q[a], A.L, vi[a], vf[a]);
            const int e0 = (vi[2] * A.L + vi[1]) * A.L + vi[0];
            if (e0 != cur_e0) {
                flush_v();
                cur_e0 = e0;
            }
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
                const float wc = (dx ? vf[0] : 1.f - vf[0]) * (dy ? vf[1] : 1.f - vf[1]) * (dz ? vf[2] : 1.f - vf[2]);
                touched |= (wc != 0.f ? 1u : 0u) << c;
#pragma unroll
                for (int q = 0; q < 8; q++) vacc[c][q] = fmaf(wc, dt[q], vacc[c][q]);
            }
        }
        {
            int pi[3];
            float pf[3];
#pragma unroll
            for (int a = 0; a < 3; a++) coord_qat(Q[a], A.R, pi[a], pf[a]);
#pragma unroll
            for (int a = 0; a < 3; a++) {
                const int ua = (a == 0) ? 1 : 0, va = (a == 2) ? 1 : 2;
                const int e = pi[va] * A.R + pi[ua];
                if (e != cur_p[a]) {
                    flush_p(a);
                    cur_p[a] = e;
                }
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const int du = c & 1, dv = c >> 1;
                    const float wc = (du ? pf[ua] : 1.f - pf[ua]) * (dv ? pf[va] : 1.f - pf[va]);
                    ptouched |= (wc != 0.f ? 1u : 0u) << (4 * a + c);
#pragma unroll
                    for (int q = 0; q < 8; q++) pacc[a][c][q] = fmaf(wc, dt[q], pacc[a][c][q]);
                }
            }
        }
    }
    flush_v();
#pragma unroll
    for (int a = 0; a < 3; a++) flush_p(a);
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_qat(const DevScene& S, const RaySource& rs, const Workspace& ws, const float* theta_v,
                       const float* theta_p, float* vv, float* vp, int quant, const float* target, float* rgb,
                       float* gvals_v, float* gvals_p, float* grad_v, float* grad_p, float* samp, int smax,
                       float* rayb, const float* mlp, double* loss, unsigned int* overflow,
                       unsigned long long* n_samples, int L, int R, int Nf, const uint32_t* occf, float md, float ma,
                       cudaStream_t st) {
    const int64_t nv = (int64_t)L * L * L * 8, np = (int64_t)3 * R * R * 8;
    prequant_kernel<<<nblk(nv, 256), 256, 0, st>>>(theta_v, nv, quant, md, ma, vv);
    prequant_kernel<<<nblk(np, 256), 256, 0, st>>>(theta_p, np, quant, md, ma, vp);
    cudaMemsetAsync(gvals_v, 0, nv * 4, st);
    cudaMemsetAsync(gvals_p, 0, np * 4, st);
    QatArgs A{vv, vp, target, rgb, gvals_v, gvals_p, samp, mlp, loss, overflow, n_samples, L, R, smax, Nf,
              kF + 2 - (31 - __builtin_clz((unsigned)Nf)), occf, (float)S.step};
    qat_fwd_kernel<<<nblk(rs.n, 128), 128, 0, st>>>(rs, ws, A, rayb);
    qat_mlp_kernel<<<nblk(rs.n, 128), 128, 0, st>>>(rs, A, rayb);
    qat_bwd_kernel<<<nblk(rs.n, 128), 128, 0, st>>>(rs, A, rayb);
    ste_kernel<<<nblk(nv, 256), 256, 0, st>>>(theta_v, gvals_v, nv, md, ma, grad_v);
    ste_kernel<<<nblk(np, 256), 256, 0, st>>>(theta_p, gvals_p, np, md, ma, grad_p);
    return cudaGetLastError();
}

}  // namespace merf
