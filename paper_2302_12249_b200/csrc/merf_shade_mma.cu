// merf_shade_mma.cu -- the deferred MLP epilogue on the tensor cores (warp-level mma.sync).
//
// The deferred shading network h(C_d, F, d) (Eq. 3; 34 -> 16 -> 16 -> 3 with ReLU,
// ReLU, sigmoid) runs once per pixel.  The FFMA kernel (shade_kernel) spends ~850 FFMA
// and ~1100 instructions per pixel on it (4.5 % of a bench step, profiles/r01_launches_summary).
// Here one warp evaluates the network for its tile of 32 pixels as three small GEMMs on the
// tensor cores: pixels are the M dimension (two m16 tiles), so the f32 accumulator fragment of
// one layer is, after ReLU, exactly the A fragment of the next (no shuffles); only the input
// layer is transposed through shared memory (ldmatrix).
//
// Precision: operands are fp16 PAIRS, x = x_hi + x_lo with x_hi = fp16(x) and
// x_lo = fp16(x - x_hi) (likewise for the weights), and each product is evaluated as
// x_hi w_hi + x_hi w_lo + x_lo w_hi in fp32 accumulation (3 mma per tile).  The dropped
// x_lo w_lo term and the rounding of x_lo, w_lo are ~2^-22 relative: fp32-class results
// (measured against the FFMA kernel in tests/test_gpu_parity.py).  fp16 needs every operand
// below 65504: the inputs are bounded (C_d, F in [0, 1], |d| = 1, |sin|, |cos| <= 1), and the
// upload computes a bound on every hidden activation from the weights
// (mlp_mma_bound in merf_api.cu); scenes whose bound exceeds 3e4 use the FFMA kernel.
#include <cuda_fp16.h>

#include "merf_render_kernel.cuh"
#include "merf_mma.cuh"

namespace merf {

// Per-lane B fragments (m16n8k16 / m16n8k8 "col" operands: B[k][n] = W[n][k], lane (g, t)
// holds n = g, k = 2t, 2t+1 (+8, +9)) of the three layers as hi/lo pairs, and the lane's bias
// columns (2t, 2t+1 of each n tile).  Layout per lane, kMlpFragWords words:
//   [0,16)  layer 1, k16 steps s = 0,1 x n tiles 0,1: hi(k..k+1), hi(k+8..k+9), lo(..), lo(..)
//   [16,20) layer 1, k8 step (k = 32..39) x n tiles 0,1: hi, lo
//   [20,28) layer 2 x n tiles 0,1          [28,32) layer 3 (n = 0..2 of one n8 tile)
//   [32,36) layer-1 biases (nt 0: 2t, 2t+1; nt 1: 8+2t, 9+2t)   [36,40) layer 2   [40,42) layer 3
__global__ void mlp_frag_kernel(const float* w, uint32_t* frag) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    uint32_t* f = frag + lane * kMlpFragWords;
    int q = 0;
    auto quad = [&](int off, int nin, int nout, int n, int k) {
        uint32_t h0, l0, h1, l1;
        split2(wnk(w, off, nin, nout, n, k), wnk(w, off, nin, nout, n, k + 1), h0, l0);
        split2(wnk(w, off, nin, nout, n, k + 8), wnk(w, off, nin, nout, n, k + 9), h1, l1);
        f[q++] = h0; f[q++] = h1; f[q++] = l0; f[q++] = l1;
    };
    for (int s = 0; s < 2; s++)
        for (int nt = 0; nt < 2; nt++) quad(0, 34, 16, 8 * nt + g, 16 * s + 2 * t);
    for (int nt = 0; nt < 2; nt++) {
        uint32_t h, l;
        split2(wnk(w, 0, 34, 16, 8 * nt + g, 32 + 2 * t), wnk(w, 0, 34, 16, 8 * nt + g, 33 + 2 * t), h, l);
        f[q++] = h; f[q++] = l;
    }
    for (int nt = 0; nt < 2; nt++) quad(560, 16, 16, 8 * nt + g, 2 * t);
    quad(832, 16, 3, g, 2 * t);
    const float* b0 = w + 544;
    const float* b1 = w + 816;
    const float* b2 = w + 880;
    for (int nt = 0; nt < 2; nt++) {
        f[q++] = __float_as_uint(b0[8 * nt + 2 * t]);
        f[q++] = __float_as_uint(b0[8 * nt + 2 * t + 1]);
    }
    for (int nt = 0; nt < 2; nt++) {
        f[q++] = __float_as_uint(b1[8 * nt + 2 * t]);
        f[q++] = __float_as_uint(b1[8 * nt + 2 * t + 1]);
    }
    f[q++] = __float_as_uint(2 * t < 3 ? b2[2 * t] : 0.f);
    f[q++] = __float_as_uint(2 * t + 1 < 3 ? b2[2 * t + 1] : 0.f);
    while (q < kMlpFragWords) f[q++] = 0u;
}

template <int KF>
__global__ void __launch_bounds__(128) shade_mma_kernel(DevScene S, RaySource rs, Workspace ws, void* out) {
    __shared__ __align__(16) __half s_x[4][2][32][kXStride];   // [warp][hi, lo][pixel][input]
    __shared__ __align__(16) float s_o[4][32][4];               // [warp][pixel][h0 h1 h2 -]
    asm volatile("griddepcontrol.wait;" ::: "memory");    // the march's accumulators (PDL)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // index within chunk
    const int64_t ray = rs.ray0 + r;

    // ---- this lane's pixel: direction (fp32: an MLP input, not a lattice decision) and inputs
    bool valid = r < rs.n;
    int view = 0, px = 0, py = 0;
    float d[3] = {0.f, 0.f, 1.f};
    float4 a0 = make_float4(0.f, 0.f, 0.f, 1.f), a1 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
        if (KF & KF_RAYS) {
#pragma unroll
            for (int q = 0; q < 3; q++) d[q] = (float)rs.d[3 * ray + q];
        } else {
            valid = ray_pixel(rs, ray, view, px, py);
            if (valid) {
                const merf_camera& c = rs.cb.cam[view];
                const float x0 = __fdividef((float)px + 0.5f - (float)c.cx, (float)c.fx);   // an MLP input:
                const float x1 = __fdividef((float)py + 0.5f - (float)c.cy, (float)c.fy);   // ~1 ulp is plenty
                float v[3];
#pragma unroll
                for (int q = 0; q < 3; q++)
                    v[q] = fmaf((float)c.c2w[4 * q], x0, fmaf((float)c.c2w[4 * q + 1], x1, (float)c.c2w[4 * q + 2]));
                const float inv = rsqrtf(fmaf(v[0], v[0], fmaf(v[1], v[1], v[2] * v[2])));
#pragma unroll
                for (int q = 0; q < 3; q++) d[q] = v[q] * inv;
            }
        }
        if (valid) {
            a0 = ws.accum[r * 2];
            a1 = ws.accum[r * 2 + 1];
        }
    }
    {
        float x[40];
        x[0] = a0.x; x[1] = a0.y; x[2] = a0.z;
        x[3] = a1.x; x[4] = a1.y; x[5] = a1.z; x[6] = a1.w;
        x[7] = d[0]; x[8] = d[1]; x[9] = d[2];
        int n = 10;
#pragma unroll
        for (int j = 0; j < 3; j++) {        // [sin, cos](2^k d_j), j outer, k inner (reading D17)
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
#pragma unroll
        for (int i = 34; i < 40; i++) x[i] = 0.f;
        uint32_t hi[24], lo[24];
#pragma unroll
        for (int w = 0; w < 20; w++) split2(x[2 * w], x[2 * w + 1], hi[w], lo[w]);
#pragma unroll
        for (int w = 20; w < 24; w++) hi[w] = lo[w] = 0u;
        uint4* ph = reinterpret_cast<uint4*>(&s_x[warp][0][lane][0]);
        uint4* pl = reinterpret_cast<uint4*>(&s_x[warp][1][lane][0]);
#pragma unroll
        for (int v = 0; v < 6; v++) {
            ph[v] = make_uint4(hi[4 * v], hi[4 * v + 1], hi[4 * v + 2], hi[4 * v + 3]);
            pl[v] = make_uint4(lo[4 * v], lo[4 * v + 1], lo[4 * v + 2], lo[4 * v + 3]);
        }
    }
    __syncwarp();

    // ---- weights: this lane's B fragments and bias columns (4 KB table, L1/L2 resident)
    uint32_t f[44];
    {
        const uint4* tab = reinterpret_cast<const uint4*>(S.mlp_frag) + lane * (kMlpFragWords / 4);
#pragma unroll
        for (int v = 0; v < kMlpFragWords / 4; v++) {
            const uint4 u = __ldg(tab + v);
            f[4 * v] = u.x; f[4 * v + 1] = u.y; f[4 * v + 2] = u.z; f[4 * v + 3] = u.w;
        }
    }
    const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 8;   // ldmatrix row address
    float h3[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; mt++) {
        // ---- layer 1: [16 px x 34] x [34 x 16], bias in the accumulator
        float c1[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; nt++) {
            c1[nt][0] = c1[nt][2] = __uint_as_float(f[32 + 2 * nt]);
            c1[nt][1] = c1[nt][3] = __uint_as_float(f[33 + 2 * nt]);
        }
#pragma unroll
        for (int s = 0; s < 2; s++) {
            uint32_t ah[4], al[4];
            ldm4(ah, &s_x[warp][0][16 * mt + lrow][16 * s + lcol]);
            ldm4(al, &s_x[warp][1][16 * mt + lrow][16 * s + lcol]);
#pragma unroll
            for (int nt = 0; nt < 2; nt++) mma16x3(c1[nt], ah, al, &f[8 * s + 4 * nt]);
        }
        {
            uint32_t h0, h1, l0, l1;
            ldm2(h0, h1, &s_x[warp][0][16 * mt + lrow][32]);
            ldm2(l0, l1, &s_x[warp][1][16 * mt + lrow][32]);
#pragma unroll
            for (int nt = 0; nt < 2; nt++) {
                mma8(c1[nt], l0, l1, f[16 + 2 * nt]);
                mma8(c1[nt], h0, h1, f[17 + 2 * nt]);
                mma8(c1[nt], h0, h1, f[16 + 2 * nt]);
            }
        }
        // ---- layer 2: ReLU(h1) [16 x 16] x [16 x 16]
        uint32_t ah[4], al[4];
        relu_to_a(c1[0], c1[1], ah, al);
        float c2[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; nt++) {
            c2[nt][0] = c2[nt][2] = __uint_as_float(f[36 + 2 * nt]);
            c2[nt][1] = c2[nt][3] = __uint_as_float(f[37 + 2 * nt]);
            mma16x3(c2[nt], ah, al, &f[20 + 4 * nt]);
        }
        // ---- layer 3: ReLU(h2) [16 x 16] x [16 x 3 (padded to 8)]
        relu_to_a(c2[0], c2[1], ah, al);
        h3[mt][0] = h3[mt][2] = __uint_as_float(f[40]);
        h3[mt][1] = h3[mt][3] = __uint_as_float(f[41]);
        mma16x3(h3[mt], ah, al, &f[28]);
    }
    // ---- logits back to their pixels' lanes: lane (g, t <= 1) holds columns 2t, 2t+1 of
    // pixels 16 mt + g and 16 mt + g + 8
    if (t <= 1) {
#pragma unroll
        for (int mt = 0; mt < 2; mt++) {
            *reinterpret_cast<float2*>(&s_o[warp][16 * mt + g][2 * t]) = make_float2(h3[mt][0], h3[mt][1]);
            *reinterpret_cast<float2*>(&s_o[warp][16 * mt + g + 8][2 * t]) = make_float2(h3[mt][2], h3[mt][3]);
        }
    }
    __syncwarp();
    if (!valid) return;
    const float4 hv = *reinterpret_cast<const float4*>(&s_o[warp][lane][0]);
    const float c0 = __saturatef(a0.x + __fdividef(1.0f, 1.0f + __expf(-hv.x)));
    const float c1 = __saturatef(a0.y + __fdividef(1.0f, 1.0f + __expf(-hv.y)));
    const float c2 = __saturatef(a0.z + __fdividef(1.0f, 1.0f + __expf(-hv.z)));
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
    if (KF & KF_RAYS) {
        put(ray);
        return;
    }
    put(out_index(rs, view, px, py));
    if (rs.fill) {
        // progressive preview: nearest upsampling of the sub-lattice pixel to its
        // stride x stride block (clipped to the frame)
        const int sd = rs.stride_m1 + 1;
        for (int dy = 0; dy < sd; dy++)
            for (int dx = 0; dx < sd; dx++)
                if ((dx | dy) != 0 && px + dx < rs.W && py + dy < rs.H)
                    put(((int64_t)view * rs.H + py + dy) * rs.W + px + dx);
    }
}

cudaError_t launch_mlp_frag(const float* w, uint32_t* frag, cudaStream_t st) {
    mlp_frag_kernel<<<1, 32, 0, st>>>(w, frag);
    return cudaGetLastError();
}

template <int KF>
static cudaError_t shade_mma_v(const DevScene& S, const RaySource& rs, const Workspace& ws, void* out,
                               cudaStream_t st) {
    if (rs.n <= 0) return cudaSuccess;
    dim3 grid((unsigned)((rs.n + 127) / 128));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // behind the march (PDL)
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, shade_mma_kernel<KF>, S, rs, ws, out);
    return cudaGetLastError();
}

cudaError_t launch_shade_mma(int kf, const DevScene& S, const RaySource& rs, const Workspace& ws, void* out,
                             cudaStream_t st) {
    switch (kf & (KF_RAYS | KF_U8)) {
        case 0: return shade_mma_v<0>(S, rs, ws, out, st);
        case KF_U8: return shade_mma_v<KF_U8>(S, rs, ws, out, st);
        case KF_RAYS: return shade_mma_v<KF_RAYS>(S, rs, ws, out, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace merf
